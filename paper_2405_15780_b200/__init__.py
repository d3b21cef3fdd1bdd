"""Python binding of libulysses_attn.so (B200-native Ulysses sequence-parallel
exact attention, arXiv 2405.15780).

Argument marshalling only: every step of the hot path (pack, all-to-all,
attention, unpack, Delta, dQ finalisation, LSE merge) runs inside the C-ABI
library.  torch is used for device memory, streams and process groups.  There
is no CPU fallback: importing works anywhere (so tests can check the library
loads and exports its symbols), but every compute call raises if the CUDA
extension is missing or no sm_100 device is present.

Names follow include/ulysses_attn.h (§2.5).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libulysses_attn.so")

UA_OK = 0
STATUS = {0: "UA_OK", 1: "UA_ERR_INVALID_ARG", 2: "UA_ERR_HEAD_DIVISIBILITY", 3: "UA_ERR_SEQ_DIVISIBILITY",
          4: "UA_ERR_UNSUPPORTED", 5: "UA_ERR_CUDA", 6: "UA_ERR_NCCL"}

# Every symbol include/ulysses_attn.h declares.
EXPORTS = ("ua_version", "ua_status_string", "ua_last_error", "ua_validate", "ua_workspace_size",
           "ua_get_unique_id", "ua_ctx_create", "ua_ctx_destroy", "ua_ctx_comm_stats",
           "ua_ctx_enable_timing", "ua_ctx_phase_times", "ua_ctx_set_a2a_mode", "ua_ctx_get_a2a_mode",
           "ua_ctx_set_deterministic", "ua_ctx_get_deterministic",
           "ua_ulysses_attn_fwd", "ua_ulysses_attn_bwd", "ua_attn_fwd_segment", "ua_lse_merge",
           "ua_f32_to_bf16_bnhd", "ua_lss_validate", "ua_lss_workspace_size", "ua_lss_attn_fwd", "ua_lss_attn_bwd",
           "ua_layer_sizes", "ua_layer_fwd", "ua_layer_bwd",
           "ua_pack_seq_to_head", "ua_unpack_head_to_seq", "ua_push_seq_to_head", "ua_head_attn_fwd",
           "ua_head_attn_bwd_workspace_size", "ua_head_attn_bwd", "ua_gemm_bf16",
           "ua_lss_rank_fwd", "ua_lss_rank_bwd_workspace_size", "ua_lss_rank_bwd")

PHASES = ("pack_fwd", "a2a_fwd_in", "attn_fwd", "a2a_fwd_out", "unpack_fwd", "pack_bwd", "a2a_bwd_in",
          "attn_bwd", "dq_finalize", "a2a_bwd_out", "unpack_bwd")


class UlyssesError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        self.name = STATUS.get(status, f"status {status}")
        super().__init__(f"{self.name}: {detail}")


class HeadDivisibilityError(UlyssesError):
    pass


class SeqDivisibilityError(UlyssesError):
    pass


_lib = None


def lib():
    """Load libulysses_attn.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2405_15780_b200/build.py (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
        L.ua_version.restype = ctypes.c_char_p
        L.ua_status_string.restype = ctypes.c_char_p
        L.ua_status_string.argtypes = [i32]
        L.ua_last_error.restype = ctypes.c_char_p
        L.ua_validate.argtypes = [i64, i64, i32, i32, i32]
        L.ua_workspace_size.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(sz), ctypes.POINTER(sz)]
        L.ua_get_unique_id.argtypes = [ctypes.c_char_p]
        L.ua_ctx_create.argtypes = [ctypes.c_char_p, i32, i32, i32, ctypes.POINTER(vp)]
        L.ua_ctx_destroy.argtypes = [vp]
        L.ua_ctx_comm_stats.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.ua_ctx_enable_timing.argtypes = [vp, i32]
        L.ua_ctx_set_a2a_mode.argtypes = [vp, i32]
        L.ua_ctx_get_a2a_mode.argtypes = [vp, ctypes.POINTER(i32)]
        L.ua_ctx_set_deterministic.argtypes = [vp, i32]
        L.ua_ctx_get_deterministic.argtypes = [vp, ctypes.POINTER(i32)]
        L.ua_ctx_phase_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
        L.ua_ulysses_attn_fwd.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
        L.ua_ulysses_attn_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
        L.ua_lss_validate.argtypes = [i64, i64, i32, i32, i32]
        L.ua_lss_workspace_size.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(sz), ctypes.POINTER(sz)]
        L.ua_lss_attn_fwd.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
        L.ua_lss_attn_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
        L.ua_layer_sizes.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(sz), ctypes.POINTER(sz), ctypes.POINTER(sz)]
        L.ua_layer_fwd.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
        L.ua_layer_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
        L.ua_attn_fwd_segment.argtypes = [vp, vp, vp, vp, vp, i64, i64, i32, i32, i64, i64, vp]
        L.ua_lse_merge.argtypes = [vp, vp, vp, vp, i64, i32, vp]
        L.ua_f32_to_bf16_bnhd.argtypes = [vp, vp, i64, i64, i32, i32, vp]
        pp = ctypes.POINTER(vp)
        L.ua_pack_seq_to_head.argtypes = [pp, pp, i32, i64, i64, i32, i32, i32, vp, vp, vp, vp]
        L.ua_unpack_head_to_seq.argtypes = [pp, pp, i32, i64, i64, i32, i32, i32, vp]
        L.ua_push_seq_to_head.argtypes = [pp, i32, pp, i64, i64, i32, i32, i32, i32, vp, vp, vp]
        L.ua_head_attn_fwd.argtypes = [vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, i32, pp, vp]
        L.ua_gemm_bf16.argtypes = [i32, i32, i64, i64, i64, pp, pp, i32, vp, i32, vp]
        L.ua_lss_rank_fwd.argtypes = [vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp]
        L.ua_lss_rank_bwd_workspace_size.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(sz)]
        L.ua_lss_rank_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, i32, vp, sz, vp]
        L.ua_head_attn_bwd_workspace_size.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(sz)]
        L.ua_head_attn_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, i32, pp, i32, vp,
                                       sz, vp]
        for name in EXPORTS:
            getattr(L, name).restype = getattr(L, name).restype if name in (
                "ua_version", "ua_status_string", "ua_last_error") else i32
        _lib = L
    return _lib


def _check(status: int):
    if status != UA_OK:
        detail = lib().ua_last_error().decode()
        cls = {2: HeadDivisibilityError, 3: SeqDivisibilityError}.get(status, UlyssesError)
        raise cls(status, detail)


def version() -> str:
    return lib().ua_version().decode()


def validate(B: int, N: int, H: int, D: int, P: int) -> None:
    """Host-only shape check (raises HeadDivisibilityError etc.)."""
    _check(lib().ua_validate(B, N, H, D, P))


def workspace_size(B: int, N: int, H: int, D: int, P: int) -> tuple[int, int]:
    f, b = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(lib().ua_workspace_size(B, N, H, D, P, ctypes.byref(f), ctypes.byref(b)))
    return f.value, b.value


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().ua_get_unique_id(buf))
    return buf.raw


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda_bf16(*ts):
    for t in ts:
        if not (t.is_cuda and t.dtype == torch.bfloat16 and t.is_contiguous()):
            raise ValueError("expected contiguous bf16 CUDA tensors [B][N/P][H][D]")


class Context:
    """Owns a ua_ctx (and, for P > 1, the library's NCCL communicator).

    For P > 1 pass ``group`` (a torch.distributed process group, any backend)
    to broadcast rank 0's NCCL unique id; the data path never uses torch's
    collectives."""

    def __init__(self, P: int = 1, rank: int = 0, device: int | None = None, group=None, uid: bytes | None = None):
        self.P, self.rank = P, rank
        self.device = torch.cuda.current_device() if device is None else device
        if P > 1 and uid is None:
            import torch.distributed as dist
            obj = [get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = obj[0]
        h = ctypes.c_void_p(0)
        _check(lib().ua_ctx_create(uid if P > 1 else None, P, rank, self.device, ctypes.byref(h)))
        self._h = h
        self._ws = {}

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h and self._h.value:
            _check(lib().ua_ctx_destroy(self._h))
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def comm_stats(self) -> tuple[int, int]:
        c, b = ctypes.c_int64(0), ctypes.c_int64(0)
        _check(lib().ua_ctx_comm_stats(self._h, ctypes.byref(c), ctypes.byref(b)))
        return c.value, b.value

    A2A_MODES = {"nccl": 0, "peer": 1}

    def set_a2a_mode(self, mode: str):
        """'nccl' (pack -> NCCL send/recv -> unpack) or 'peer' (kernels store
        straight into the owning GPU's buffers over NVLink).  Collective."""
        _check(lib().ua_ctx_set_a2a_mode(self._h, self.A2A_MODES[mode]))

    def a2a_mode(self) -> str:
        m = ctypes.c_int(0)
        _check(lib().ua_ctx_get_a2a_mode(self._h, ctypes.byref(m)))
        return {v: k for k, v in self.A2A_MODES.items()}[m.value]

    def set_deterministic(self, on: bool = True):
        """Bitwise-reproducible backward: query-stationary dQ kernel instead of
        the fp32 reduce-add of key-tile partials (ua_ctx_set_deterministic)."""
        _check(lib().ua_ctx_set_deterministic(self._h, 1 if on else 0))

    def deterministic(self) -> bool:
        m = ctypes.c_int(0)
        _check(lib().ua_ctx_get_deterministic(self._h, ctypes.byref(m)))
        return bool(m.value)

    def enable_timing(self, on: bool = True):
        _check(lib().ua_ctx_enable_timing(self._h, 1 if on else 0))

    def phase_times(self) -> dict:
        """{phase: (ms summed since last query, launches)}; synchronises."""
        n = len(PHASES)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        _check(lib().ua_ctx_phase_times(self._h, ms, cnt))
        return {PHASES[i]: (ms[i], cnt[i]) for i in range(n)}

    def workspace(self, nbytes: int) -> torch.Tensor:
        """Cached device workspace of at least nbytes."""
        ws = self._ws.get("buf")
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=f"cuda:{self.device}")
            self._ws["buf"] = ws
        return ws


@dataclass
class FwdOut:
    out: torch.Tensor
    lse: torch.Tensor


def ulysses_attn_fwd(ctx: Context, q, k, v, H: int | None = None, out=None, lse=None, stream=None) -> FwdOut:
    """q, k, v: bf16 [B][N/P][H][D] (this rank's sequence shard).
    Returns out [B][N/P][H][D] bf16 and lse [B][H/P][N] fp32."""
    _need_cuda_bf16(q, k, v)
    B, Nl, H_, D = q.shape
    P = ctx.P
    N = Nl * P
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((B, H_ // P if H_ % P == 0 else 1, N), dtype=torch.float32, device=q.device)
    validate(B, N, H_, D, P)
    fb, _ = workspace_size(B, N, H_, D, P)
    ws = ctx.workspace(fb)
    _check(lib().ua_ulysses_attn_fwd(ctx.handle, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), B, N, H_, D, P,
                                     _ptr(ws), ws.numel(), _stream(stream)))
    return FwdOut(out, lse)


def ulysses_attn_bwd(ctx: Context, q, k, v, out, lse, dout, dq=None, dk=None, dv=None, stream=None):
    """Gradients (dq, dk, dv) bf16 [B][N/P][H][D] of this rank's shard."""
    _need_cuda_bf16(q, k, v, out, dout)
    B, Nl, H, D = q.shape
    P = ctx.P
    N = Nl * P
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    validate(B, N, H, D, P)
    _, bb = workspace_size(B, N, H, D, P)
    ws = ctx.workspace(bb)
    _check(lib().ua_ulysses_attn_bwd(ctx.handle, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _ptr(dout),
                                     _ptr(dq), _ptr(dk), _ptr(dv), B, N, H, D, P, _ptr(ws), ws.numel(),
                                     _stream(stream)))
    return dq, dk, dv


def lss_validate(B: int, N: int, H: int, D: int, P: int) -> None:
    """Host-only shape check of the LSS strategy (no head limit)."""
    _check(lib().ua_lss_validate(B, N, H, D, P))


def lss_workspace_size(B: int, N: int, H: int, D: int, P: int) -> tuple[int, int]:
    f, b = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(lib().ua_lss_workspace_size(B, N, H, D, P, ctypes.byref(f), ctypes.byref(b)))
    return f.value, b.value


def lss_attn_fwd(ctx: Context, q, k, v, out=None, lse=None, stream=None) -> FwdOut:
    """LSS sequence parallelism: q, k, v bf16 [B][N/P][H][D]
    (this rank's segment).  Returns out [B][N/P][H][D] bf16 and lse [B][H][N/P] fp32."""
    _need_cuda_bf16(q, k, v)
    B, Nl, H, D = q.shape
    P = ctx.P
    N = Nl * P
    out = torch.empty_like(q) if out is None else out
    lse = torch.empty((B, H, Nl), dtype=torch.float32, device=q.device) if lse is None else lse
    lss_validate(B, N, H, D, P)
    fb, _ = lss_workspace_size(B, N, H, D, P)
    ws = ctx.workspace(fb)
    _check(lib().ua_lss_attn_fwd(ctx.handle, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), B, N, H, D, P,
                                 _ptr(ws), ws.numel(), _stream(stream)))
    return FwdOut(out, lse)


def lss_attn_bwd(ctx: Context, q, k, v, out, lse, dout, dq=None, dk=None, dv=None, stream=None):
    """LSS backward: gradients (dq, dk, dv) bf16 [B][N/P][H][D] of this rank's segment."""
    _need_cuda_bf16(q, k, v, out, dout)
    B, Nl, H, D = q.shape
    P = ctx.P
    N = Nl * P
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    lss_validate(B, N, H, D, P)
    _, bb = lss_workspace_size(B, N, H, D, P)
    ws = ctx.workspace(bb)
    _check(lib().ua_lss_attn_bwd(ctx.handle, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _ptr(dout), _ptr(dq),
                                 _ptr(dk), _ptr(dv), B, N, H, D, P, _ptr(ws), ws.numel(), _stream(stream)))
    return dq, dk, dv


def layer_sizes(B: int, N: int, H: int, D: int, P: int) -> tuple[int, int, int]:
    """(saved_bytes, fwd_workspace_bytes, bwd_workspace_bytes) of the attention layer."""
    a, f, b = ctypes.c_size_t(0), ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(lib().ua_layer_sizes(B, N, H, D, P, ctypes.byref(a), ctypes.byref(f), ctypes.byref(b)))
    return a.value, f.value, b.value


def layer_fwd(ctx: Context, x, w_qkv, w_o, H: int, stream=None):
    """Attention layer forward on this rank's sequence shard x bf16 [B][N/P][E]
    (E = H*D; w_qkv [3E][E], w_o [E][E] bf16).  Returns (y, saved); saved is the
    opaque uint8 buffer the backward needs."""
    _need_cuda_bf16(x, w_qkv, w_o)
    B, Nl, E = x.shape
    D = E // H
    P = ctx.P
    N = Nl * P
    sb, fb, _ = layer_sizes(B, N, H, D, P)
    saved = torch.empty(sb, dtype=torch.uint8, device=x.device)
    y = torch.empty_like(x)
    ws = ctx.workspace(fb)
    _check(lib().ua_layer_fwd(ctx.handle, _ptr(x), _ptr(w_qkv), _ptr(w_o), _ptr(y), _ptr(saved), B, N, H, D, P,
                              _ptr(ws), ws.numel(), _stream(stream)))
    return y, saved


def layer_bwd(ctx: Context, x, w_qkv, w_o, saved, dy, H: int, stream=None):
    """Attention layer backward: (dx bf16 [B][N/P][E], dw_qkv fp32 [3E][E], dw_o fp32 [E][E]);
    the weight gradients are summed over the SP group (one all-reduce)."""
    _need_cuda_bf16(x, w_qkv, w_o, dy)
    B, Nl, E = x.shape
    D = E // H
    P = ctx.P
    N = Nl * P
    _, _, bb = layer_sizes(B, N, H, D, P)
    dx = torch.empty_like(x)
    dw_qkv = torch.empty((3 * E, E), dtype=torch.float32, device=x.device)
    dw_o = torch.empty((E, E), dtype=torch.float32, device=x.device)
    ws = ctx.workspace(bb)
    _check(lib().ua_layer_bwd(ctx.handle, _ptr(x), _ptr(w_qkv), _ptr(w_o), _ptr(saved), _ptr(dy), _ptr(dx),
                              _ptr(dw_qkv), _ptr(dw_o), B, N, H, D, P, _ptr(ws), ws.numel(), _stream(stream)))
    return dx, dw_qkv, dw_o


def attn_fwd_segment(q, k, v, kv_begin: int, kv_end: int, o_seg=None, lse_seg=None, stream=None):
    """One LSS key segment on head-layout tensors q, k, v bf16 [B][N][Hx][D].
    Returns (o_seg fp32 [B][Hx][N][D], lse_seg fp32 [B][Hx][N])."""
    _need_cuda_bf16(q, k, v)
    B, N, Hx, D = q.shape
    if o_seg is None:
        o_seg = torch.empty((B, Hx, N, D), dtype=torch.float32, device=q.device)
    if lse_seg is None:
        lse_seg = torch.empty((B, Hx, N), dtype=torch.float32, device=q.device)
    _check(lib().ua_attn_fwd_segment(_ptr(q), _ptr(k), _ptr(v), _ptr(o_seg), _ptr(lse_seg), B, N, Hx, D, kv_begin,
                                     kv_end, _stream(stream)))
    return o_seg, lse_seg


def lse_merge(o_a, lse_a, o_b, lse_b, stream=None):
    """In-place exact merge of segment b into segment a."""
    D = o_a.shape[-1]
    _check(lib().ua_lse_merge(_ptr(o_a), _ptr(lse_a), _ptr(o_b), _ptr(lse_b), lse_a.numel(), D, _stream(stream)))
    return o_a, lse_a


def f32_to_bf16_bnhd(src, stream=None):
    """fp32 [B][Hx][N][D] -> bf16 [B][N][Hx][D]."""
    B, Hx, N, D = src.shape
    dst = torch.empty((B, N, Hx, D), dtype=torch.bfloat16, device=src.device)
    _check(lib().ua_f32_to_bf16_bnhd(_ptr(src), _ptr(dst), B, N, Hx, D, _stream(stream)))
    return dst


def lss_chunked_fwd(q, k, v, seg_len: int, stream=None):
    """Exact attention over head-layout q, k, v [B][N][Hx][D] computed as
    contiguous key segments of seg_len (multiple of 128) merged by LSE
    (P:72).  Returns (out bf16 [B][N][Hx][D], lse fp32 [B][Hx][N])."""
    B, N, Hx, D = q.shape
    if seg_len % 128 != 0 or seg_len < 128:
        raise ValueError("seg_len must be a positive multiple of 128")
    o_acc, l_acc = attn_fwd_segment(q, k, v, 0, min(seg_len, N), stream=stream)
    o_tmp = torch.empty_like(o_acc)
    l_tmp = torch.empty_like(l_acc)
    for j0 in range(seg_len, N, seg_len):
        attn_fwd_segment(q, k, v, j0, min(j0 + seg_len, N), o_tmp, l_tmp, stream=stream)
        lse_merge(o_acc, l_acc, o_tmp, l_tmp, stream=stream)
    return f32_to_bf16_bnhd(o_acc, stream=stream), l_acc


# ---------------------------------------------------------------- rank-local steps
# (include/ulysses_attn.h "rank-local steps": what one rank computes between the
# all-to-alls; no communication, no ctx.)
def _ptr_array(ts):
    return (ctypes.c_void_p * max(1, len(ts)))(*[t.data_ptr() if t is not None else 0 for t in ts])


def pack_seq_to_head(srcs, P: int, dout=None, out=None, stream=None):
    """A1 / B1: srcs = list of bf16 [B][N/P][H][D] shards of one rank.  Returns
    (send list of bf16 [P][N/P][B][H/P][D], delta fp32 [P][N/P][B][H/P] or None)."""
    ref = srcs[0] if srcs else dout
    B, Nl, H, D = ref.shape
    dsts = [torch.empty((P, Nl, B, H // P, D), dtype=torch.bfloat16, device=ref.device) for _ in srcs]
    delta = None
    if dout is not None:
        delta = torch.empty((P, Nl, B, H // P), dtype=torch.float32, device=ref.device)
    _check(lib().ua_pack_seq_to_head(_ptr_array(srcs), _ptr_array(dsts), len(srcs), B, Nl * P, H, D, P, _ptr(dout),
                                     _ptr(out), _ptr(delta), _stream(stream)))
    return dsts, delta


def unpack_head_to_seq(srcs, P: int, stream=None):
    """A6 / B6: srcs = list of bf16 [P][N/P][B][H/P][D] (chunk s from rank s).
    Returns list of bf16 [B][N/P][H][D]."""
    _, Nl, B, Hl, D = srcs[0].shape
    H = Hl * P
    dsts = [torch.empty((B, Nl, H, D), dtype=torch.bfloat16, device=srcs[0].device) for _ in srcs]
    _check(lib().ua_unpack_head_to_seq(_ptr_array(srcs), _ptr_array(dsts), len(srcs), B, Nl * P, H, D, P,
                                       _stream(stream)))
    return dsts


def push_seq_to_head(srcs, dst_ranks, P: int, rank: int, dout=None, out=None, stream=None):
    """A1 + A2 fused (the peer transport's kernel): store rank `rank`'s chunks into
    every destination's receive buffer dst_ranks[j] (uint8 tensors of
    ntensors*N*B*Hl*D*2 (+ N*B*Hl*4 with Delta) bytes)."""
    B, Nl, H, D = srcs[0].shape
    _check(lib().ua_push_seq_to_head(_ptr_array(srcs), len(srcs), _ptr_array(dst_ranks), B, Nl * P, H, D, P, rank,
                                     _ptr(dout), _ptr(out), _stream(stream)))


def head_attn_fwd(q, k, v, P: int, rank: int, o=None, lse=None, o_owner=None, stream=None):
    """A3 on rank `rank`'s head shard: q, k, v bf16 [N][B][H/P][D].  Returns (o
    [N][B][H/P][D], or None when o_owner (P token-owner tensors [B][N/P][H][D]) is
    given; lse fp32 [B][H/P][N])."""
    N, B, Hl, D = q.shape
    if lse is None:
        lse = torch.empty((B, Hl, N), dtype=torch.float32, device=q.device)
    if o is None and o_owner is None:
        o = torch.empty_like(q)
    owners = _ptr_array(o_owner) if o_owner is not None else None
    _check(lib().ua_head_attn_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), B, N, Hl * P, D, P, rank, owners,
                                  _stream(stream)))
    return o, lse


def head_attn_bwd(q, k, v, dout, lse, delta, P: int, rank: int, owners=None, deterministic=False, stream=None):
    """B3 + B4 on rank `rank`'s head shard (layouts as head_attn_fwd; delta fp32
    [N][B][H/P]).  Returns (dq, dk, dv) bf16 [N][B][H/P][D], or None when owners
    (3P token-owner tensors: dq owners, dk owners, dv owners) is given."""
    N, B, Hl, D = q.shape
    n = ctypes.c_size_t(0)
    _check(lib().ua_head_attn_bwd_workspace_size(B, N, Hl * P, D, P, ctypes.byref(n)))
    ws = torch.empty(max(n.value, 256), dtype=torch.uint8, device=q.device)
    grads = (None, None, None) if owners is not None else tuple(torch.empty_like(q) for _ in range(3))
    _check(lib().ua_head_attn_bwd(_ptr(q), _ptr(k), _ptr(v), _ptr(dout), _ptr(lse), _ptr(delta), _ptr(grads[0]),
                                  _ptr(grads[1]), _ptr(grads[2]), B, N, Hl * P, D, P, rank,
                                  _ptr_array(owners) if owners is not None else None, 1 if deterministic else 0,
                                  _ptr(ws), ws.numel(), _stream(stream)))
    return None if owners is not None else grads


def lss_rank_fwd(q, k_full, v_full, P: int, out=None, lse=None, stream=None):
    """LSS compute of one rank (no communication): q bf16 [B][N/P][H][D] (its
    query segment), k_full, v_full bf16 [N][B][H][D] (all ranks' keys, rank
    order).  Returns (out [B][N/P][H][D] bf16, lse [B][H][N/P] fp32)."""
    B, Nl, H, D = q.shape
    out = torch.empty_like(q) if out is None else out
    lse = torch.empty((B, H, Nl), dtype=torch.float32, device=q.device) if lse is None else lse
    _check(lib().ua_lss_rank_fwd(_ptr(q), _ptr(k_full), _ptr(v_full), _ptr(out), _ptr(lse), B, Nl * P, H, D, P,
                                 _stream(stream)))
    return out, lse


def lss_rank_bwd(q, k_full, v_full, out, lse, dout, P: int, deterministic=False, stream=None):
    """LSS backward compute of one rank: returns (dq bf16 [B][N/P][H][D],
    dk_part, dv_part fp32 [N][B][H][D] = partial sums over this rank's queries)."""
    B, Nl, H, D = q.shape
    N = Nl * P
    n = ctypes.c_size_t(0)
    _check(lib().ua_lss_rank_bwd_workspace_size(B, N, H, D, P, ctypes.byref(n)))
    ws = torch.empty(max(n.value, 256), dtype=torch.uint8, device=q.device)
    dq = torch.empty_like(q)
    dk_part = torch.empty((N, B, H, D), dtype=torch.float32, device=q.device)
    dv_part = torch.empty_like(dk_part)
    _check(lib().ua_lss_rank_bwd(_ptr(q), _ptr(k_full), _ptr(v_full), _ptr(out), _ptr(lse), _ptr(dout), _ptr(dq),
                                 _ptr(dk_part), _ptr(dv_part), B, N, H, D, P, 1 if deterministic else 0, _ptr(ws),
                                 ws.numel(), _stream(stream)))
    return dq, dk_part, dv_part


def gemm(As, Bs, a_mn: bool, b_mn: bool, out_f32: bool = False, stream=None):
    """C = sum_s op(A_s) op(B_s) on the library's tcgen05 GEMM (ua_gemm_bf16):
    a_mn: A_s is [K][M] (transposed), else [M][K]; b_mn: B_s is [K][N], else
    [N][K] (transposed).  Returns C [M][N] bf16 (or fp32)."""
    A0, B0 = As[0], Bs[0]
    M, K = (A0.shape[1], A0.shape[0]) if a_mn else (A0.shape[0], A0.shape[1])
    N = B0.shape[1] if b_mn else B0.shape[0]
    C = torch.empty((M, N), dtype=torch.float32 if out_f32 else torch.bfloat16, device=A0.device)
    _check(lib().ua_gemm_bf16(int(a_mn), int(b_mn), M, N, K, _ptr_array(As), _ptr_array(Bs), len(As), _ptr(C),
                              int(out_f32), _stream(stream)))
    return C


class UlyssesAttention(torch.autograd.Function):
    """autograd wrapper: y = ulysses_attn(q, k, v) on this rank's shard."""

    @staticmethod
    def forward(ctx_, q, k, v, uctx: Context):
        r = ulysses_attn_fwd(uctx, q, k, v)
        ctx_.save_for_backward(q, k, v, r.out, r.lse)
        ctx_.uctx = uctx
        return r.out

    @staticmethod
    def backward(ctx_, dout):
        q, k, v, out, lse = ctx_.saved_tensors
        dq, dk, dv = ulysses_attn_bwd(ctx_.uctx, q, k, v, out, lse, dout.contiguous())
        return dq, dk, dv, None
