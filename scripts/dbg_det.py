"""Debug aid: one deterministic-mode fwd+bwd at a given shape, compared with the default mode."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_15780_b200 as ua
N, H, D = (int(x) for x in sys.argv[1:4])
torch.manual_seed(0)
q, k, v, do = (torch.randn(1, N, H, D, device="cuda").bfloat16() for _ in range(4))
c = ua.Context(P=1)
r = ua.ulysses_attn_fwd(c, q, k, v)
g0 = ua.ulysses_attn_bwd(c, q, k, v, r.out, r.lse, do)
c.set_deterministic(True)
g1 = ua.ulysses_attn_bwd(c, q, k, v, r.out, r.lse, do)
torch.cuda.synchronize()
print(N, H, D, "maxdiff", [float((a.float() - b.float()).abs().max()) for a, b in zip(g0, g1)], flush=True)
