"""Host-only checks of the C-ABI library: it loads, exports every symbol
include/ulysses_attn.h declares, validates shapes with the documented status
codes, plans workspaces, and fails loudly (no CPU fallback) without a GPU."""
import os
import re

import pytest
import torch

import paper_2405_15780_b200 as ua
from paper_2405_15780_b200 import build as ua_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ulysses_attn.h")


@pytest.fixture(scope="module", autouse=True)
def built():
    ua_build.build()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ua_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_exports():
    assert declared_functions() == sorted(ua.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = ua.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    # and nm agrees (extern "C", unmangled, defined)
    import subprocess
    syms = subprocess.run(["nm", "-D", "--defined-only", ua.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}$", syms, flags=re.M), name


def test_version_and_status_strings():
    assert "sm_100a" in ua.version()
    for code, name in ua.STATUS.items():
        assert ua.lib().ua_status_string(code).decode() == name


@pytest.mark.parametrize("args,status", [
    ((1, 16, 4, 64, 8), 2),      # H=4, P=8 -> HeadDivisibility
    ((1, 12, 6, 64, 4), 2),      # P does not divide H
    ((1, 10, 4, 64, 4), 3),      # N % P != 0 -> SeqDivisibility
    ((1, 16, 4, 72, 2), 0),      # D=72: ViT-10B, 4608 / 64 heads (Table 1)
    ((1, 16, 4, 80, 2), 4),      # D=80 unsupported
    ((1, 16, 4, 160, 2), 4),     # D=160 (2560 / 16) unsupported: TMEM cannot hold S and two O tiles
    ((0, 16, 4, 64, 1), 1),
    ((1, 0, 4, 64, 1), 1),
    ((1, 1 << 31, 32, 64, 8), 4),
    ((1, 256, 4, 32, 1), 0),     # c1
    ((1, 188416, 32, 64, 8), 0),  # c4 at P=8
    ((1, 1048576, 32, 128, 8), 0),  # c5
])
def test_validate_codes(args, status):
    assert ua.lib().ua_validate(*args) == status
    if status:
        assert ua.lib().ua_last_error().decode() != ""


def test_python_errors():
    with pytest.raises(ua.HeadDivisibilityError):
        ua.validate(1, 16, 4, 64, 8)
    with pytest.raises(ua.SeqDivisibilityError):
        ua.validate(1, 10, 4, 64, 4)


def test_workspace_plan():
    B, N, H, D = 1, 188416, 32, 64
    shard = B * N * H * D * 2
    f1, b1 = ua.workspace_size(B, N, H, D, 1)
    assert f1 == 0 and b1 >= B * N * H * 4 + B * N * H * D * 4
    for P in (2, 4, 8):
        f, b = ua.workspace_size(B, N, H, D, P)
        s = shard // P
        assert 7 * s <= f <= 7 * s + 4096
        assert b >= 11 * s + 2 * s + 2 * B * (N // P) * H * 4


def test_no_cpu_fallback():
    """Without a CUDA device every compute entry point fails loudly."""
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import ctypes
    h = ctypes.c_void_p(0)
    st = ua.lib().ua_ctx_create(None, 1, 0, 0, ctypes.byref(h))
    assert st in (4, 5) and not h.value
    st = ua.lib().ua_attn_fwd_segment(*(ctypes.c_void_p(16),) * 5, 1, 256, 4, 64, 0, 256, None)
    assert st in (4, 5)
    with pytest.raises(ValueError):
        ua.ulysses_attn_fwd(None, torch.zeros(1, 4, 1, 64), torch.zeros(1, 4, 1, 64), torch.zeros(1, 4, 1, 64))


@pytest.mark.parametrize("args,status", [
    ((1, 16, 4, 64, 8), 0),       # LSS has no head limit: H=4, P=8 is fine
    ((1, 12, 6, 64, 4), 0),       # P need not divide H
    ((1, 10, 4, 64, 4), 3),       # N % P != 0 -> SeqDivisibility
    ((1, 16, 4, 72, 2), 0),
    ((1, 16, 4, 96, 2), 4),
    ((0, 16, 4, 64, 1), 1),
    ((1, 188416, 32, 64, 8), 0),
    ((1, 1048576, 32, 128, 64), 0),
])
def test_lss_validate_codes(args, status):
    assert ua.lib().ua_lss_validate(*args) == status


def test_lss_workspace_plan():
    """LSS forward gathers K, V ([2][N][B][H][D] bf16 + local send copy); the
    backward adds fp32 partial dK, dV for all N keys and their reduced shard."""
    B, N, H, D = 1, 188416, 32, 64
    full = B * N * H * D
    assert ua.lss_workspace_size(B, N, H, D, 1) == ua.workspace_size(B, N, H, D, 1)
    for P in (2, 4, 8):
        f, b = ua.lss_workspace_size(B, N, H, D, P)
        s = full // P
        assert 2 * 2 * full + 2 * 2 * s <= f <= 2 * 2 * full + 2 * 2 * s + 4096
        assert b >= f + 2 * 4 * full + 2 * 4 * s + (N // P) * H * 4
    # P > H works for LSS, not for Ulysses
    assert ua.lss_workspace_size(1, 4096, 2, 64, 4)[0] > 0
    with pytest.raises(ua.HeadDivisibilityError):
        ua.workspace_size(1, 4096, 2, 64, 4)


def test_ctx_mode_setters_validate_arguments():
    """Host-side argument checks of the ctx mode entry points (no device needed)."""
    import ctypes
    L = ua.lib()
    assert L.ua_ctx_set_deterministic(None, 1) == 1          # UA_ERR_INVALID_ARG
    assert L.ua_ctx_get_deterministic(None, ctypes.byref(ctypes.c_int(0))) == 1
    assert L.ua_ctx_set_a2a_mode(None, 0) == 1
    assert "ctx" in L.ua_last_error().decode()


def test_rank_local_steps_validate_before_any_launch():
    """The rank-local step entry points check shapes (the same codes as
    ua_validate) and pointers on the host before touching the device."""
    import ctypes
    L = ua.lib()
    arr = (ctypes.c_void_p * 4)(16, 32, 48, 64)
    # S:248 head limit (H=4, P=8) and S:244 N % P, before anything else
    assert L.ua_pack_seq_to_head(arr, arr, 1, 1, 16, 4, 64, 8, None, None, None, None) == 2
    assert L.ua_unpack_head_to_seq(arr, arr, 1, 1, 10, 4, 64, 4, None) == 3
    assert L.ua_head_attn_fwd(None, None, None, None, None, 1, 16, 4, 64, 8, 0, None, None) == 2
    # bad counts / ranks / pointers
    assert L.ua_pack_seq_to_head(arr, arr, 5, 1, 16, 4, 64, 2, None, None, None, None) == 1
    assert L.ua_pack_seq_to_head(arr, arr, 0, 1, 16, 4, 64, 2, None, None, None, None) == 1   # 0 tensors, no Delta
    assert L.ua_unpack_head_to_seq(arr, arr, 0, 1, 16, 4, 64, 2, None) == 1
    assert L.ua_push_seq_to_head(arr, 1, arr, 1, 16, 4, 64, 2, 2, None, None, None) == 1      # rank >= P
    assert L.ua_head_attn_fwd(None, None, None, None, None, 1, 16, 4, 64, 2, 0, None, None) == 1
    assert L.ua_head_attn_fwd(*(ctypes.c_void_p(16),) * 5, 1, 16, 4, 64, 2, 3, None, None) == 1  # rank >= P
    assert L.ua_head_attn_bwd(*(ctypes.c_void_p(16),) * 9, 1, 16, 4, 64, 2, 0, None, 0, ctypes.c_void_p(16), 0,
                              None) == 1                                                      # workspace too small
    misaligned = (ctypes.c_void_p * 1)(18)
    assert L.ua_unpack_head_to_seq(misaligned, arr, 1, 1, 16, 4, 64, 2, None) == 1


def test_head_attn_bwd_workspace_size():
    """fp32 dQ accumulator [B*Hl][N_pad][D] + (lse, Delta) table [B*Hl][N_pad] float2."""
    import ctypes
    n = ctypes.c_size_t(0)
    B, N, H, D, P = 2, 1000, 8, 64, 4
    assert ua.lib().ua_head_attn_bwd_workspace_size(B, N, H, D, P, ctypes.byref(n)) == 0
    n_pad = 1024
    need = B * (H // P) * n_pad * (D * 4 + 8)
    assert need <= n.value <= need + 512
    # the P = 1 backward's workspace holds Delta plus exactly this region
    _, b1 = ua.workspace_size(B, N, H, D, 1)
    assert ua.lib().ua_head_attn_bwd_workspace_size(B, N, H, D, 1, ctypes.byref(n)) == 0
    assert b1 >= n.value + B * N * H * 4


def test_gemm_validates_before_launch():
    """ua_gemm_bf16 checks segment counts, pointers and 16-byte row alignment on the host."""
    import ctypes
    L = ua.lib()
    arr = (ctypes.c_void_p * 3)(256, 512, 768)
    c = ctypes.c_void_p(1024)
    assert L.ua_gemm_bf16(0, 0, 128, 128, 64, arr, arr, 0, c, 0, None) == 1      # nseg = 0
    assert L.ua_gemm_bf16(0, 0, 128, 128, 64, arr, arr, 4, c, 0, None) == 1      # nseg > 3
    assert L.ua_gemm_bf16(0, 0, 128, 128, 60, arr, arr, 1, c, 0, None) == 1      # K-major rows of 60 bf16
    assert L.ua_gemm_bf16(1, 1, 100, 128, 64, arr, arr, 1, c, 0, None) == 1      # MN-major A with M = 100
    bad = (ctypes.c_void_p * 1)(258)
    assert L.ua_gemm_bf16(0, 0, 128, 128, 64, bad, arr, 1, c, 0, None) == 1      # misaligned A
    assert L.ua_gemm_bf16(0, 0, 0, 128, 64, arr, arr, 1, c, 0, None) == 1        # M = 0


def test_no_vendor_blas_linked():
    """The projection GEMMs run on the library's own tcgen05 kernel: the
    shared object links NCCL and the CUDA runtime only, no cuBLAS / cuBLASLt."""
    import subprocess
    out = subprocess.run(["readelf", "-d", ua.LIB_PATH], capture_output=True, text=True).stdout
    needed = [line for line in out.splitlines() if "(NEEDED)" in line]
    assert needed and not any("cublas" in line.lower() for line in needed), needed
    syms = subprocess.run(["nm", "-D", "--undefined-only", ua.LIB_PATH], capture_output=True, text=True).stdout
    assert "cublas" not in syms.lower()
