"""The input generator is counter-based: any shard / head subset equals the
corresponding slice of the global draw (P-invariance of the inputs)."""
import numpy as np

import synth


def test_shards_are_slices_of_the_global_tensor():
    B, N, H, D = 2, 3000, 4, 32
    full = synth.normal_f32(B, N, H, D, 5, "k")
    for n0, n1 in ((0, 1500), (1500, 3000), (1000, 2048), (2999, 3000)):
        assert np.array_equal(synth.normal_f32(B, N, H, D, 5, "k", n0=n0, n1=n1), full[:, n0:n1])
    assert np.array_equal(synth.normal_f32(B, N, H, D, 5, "k", heads=[3, 1]), full[:, :, [3, 1]])
    q, k, v = synth.qkv(B, N, H, D, seed=5)
    assert np.array_equal(k.float().numpy(), synth.normal_bf16(B, N, H, D, 5, "k").float().numpy())


def test_distribution_and_independence():
    x = synth.normal_f32(1, 8192, 2, 64, 9, "q")
    y = synth.normal_f32(1, 8192, 2, 64, 9, "v")
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1) < 0.01
    assert abs(np.corrcoef(x.ravel(), y.ravel())[0, 1]) < 0.01
    assert not np.array_equal(x[:, :1024], x[:, 1024:2048])
