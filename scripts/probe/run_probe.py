"""Run the tcgen05 descriptor probes on a GPU and report max errors vs torch."""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libprobe.so"))
torch.manual_seed(0)
dev = "cuda"


def p(t):
    return ctypes.c_void_p(t.data_ptr())


ok = True
for D in (64, 128):
    q = torch.randn(128, D, device=dev).bfloat16()
    k = torch.randn(128, D, device=dev).bfloat16()
    s = torch.zeros(128, 128, device=dev)
    rc = lib.probe_qk(p(q), p(k), p(s), D)
    ref = q.float() @ k.float().T
    e = (s - ref).abs().max().item()
    print(f"qk D={D} rc={rc} maxerr={e:.3e}")
    ok &= rc == 0 and e < 1e-3
    P = torch.rand(128, 128, device=dev).bfloat16()
    v = torch.randn(128, D, device=dev).bfloat16()
    ref = P.float() @ v.float()
    for mode in (0, 1):
        o = torch.zeros(128, D, device=dev)
        rc = lib.probe_pv(p(P), p(v), p(o), D, mode)
        e = (o - ref).abs().max().item()
        print(f"pv D={D} mode={'TS' if mode == 0 else 'SS'} rc={rc} maxerr={e:.3e}")
        if e > 1e-3:
            print("  got[0,:8]", o[0, :8].tolist(), "\n  ref[0,:8]", ref[0, :8].tolist())
        ok &= rc == 0 and e < 1e-3
    x = torch.randn(128, 128, device=dev).bfloat16()
    y = torch.randn(128, D, device=dev).bfloat16()
    ref = x.float().T @ y.float()
    for mode in (0, 1):
        c = torch.zeros(128, D, device=dev)
        rc = lib.probe_atb(p(x), p(y), p(c), D, mode)
        e = (c - ref).abs().max().item()
        print(f"atb D={D} mode={'TMA' if mode == 0 else 'manual'} rc={rc} maxerr={e:.3e}")
        ok &= rc == 0 and e < 1e-3
print("ALL_OK" if ok else "SOME_FAILED")
sys.exit(0 if ok else 1)
