// capi.cpp — the C ABI (include/ulysses_attn.h): validation, workspace plan,
// NCCL all-to-all, and the launch sequence of the Ulysses forward / backward.
#include "../../include/ulysses_attn.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "tma_host.h"

namespace {
// RAII phase marker: records an event pair around a phase when timing is on.
struct Phase {
  ua_ctx* ctx;
  cudaStream_t stream;
  ua_ctx::Rec rec{};
  Phase(ua_ctx* c, int phase, cudaStream_t s) : ctx(c), stream(s) {
    if (ctx && ctx->timing) {
      rec.phase = phase;
      rec.a = ctx->get_event();
      rec.b = ctx->get_event();
      cudaEventRecord(rec.a, stream);
    }
  }
  ~Phase() {
    if (ctx && ctx->timing) {
      cudaEventRecord(rec.b, stream);
      ctx->pending.push_back(rec);
    }
  }
};
}  // namespace

namespace {
thread_local std::string g_err;
}  // namespace

namespace ua_internal {
ua_status fail(ua_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}
}  // namespace ua_internal

namespace {
using ua_internal::fail;

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

ua_status ua_internal::check_device() {
  static std::mutex mu;
  static int checked[64] = {0};  // 0 unknown, 1 ok, 2 bad
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return fail(UA_ERR_UNSUPPORTED, "no CUDA device available (%s); this library has no CPU fallback",
                cudaGetErrorString(e));
  }
  std::lock_guard<std::mutex> lk(mu);
  if (checked[dev] == 0) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    checked[dev] = (major == 10 && minor == 0) ? 1 : 2;
  }
  if (checked[dev] != 1) return fail(UA_ERR_UNSUPPORTED, "device %d is not sm_100 (B200); kernels are sm_100a only", dev);
  return UA_OK;
}

namespace {
using ua_internal::check_device;

struct Shape {
  int64_t B, N, Nl;
  int H, Hl, D, P;
  int64_t shard() const { return B * Nl * H * D; }  // elements of one [B][N/P][H][D] shard
  int64_t chunk() const { return Nl * B * Hl * D; }  // elements per (tensor, peer) in the a2a
};

Shape make_shape(int64_t B, int64_t N, int H, int D, int P) {
  Shape s;
  s.B = B; s.N = N; s.H = H; s.D = D; s.P = P;
  s.Nl = N / P; s.Hl = H / P;
  return s;
}

// 4-D map {D, N, heads, B} over a bf16 view with token / head / batch strides (elements).
ua_status make_map(CUtensorMap* m, const void* base, int D, int64_t N, int heads, int64_t B, int64_t sn, int64_t sh,
                   int64_t sb, uint32_t box_rows = 128) {
  const uint64_t dims[4] = {uint64_t(D), uint64_t(N), uint64_t(heads), uint64_t(B)};
  const uint64_t strides[3] = {uint64_t(sn) * 2, uint64_t(sh) * 2, uint64_t(sb) * 2};
  // one box per smem atom (attn_common.cuh TileGeom): 64 columns SW128 (D = 64, 128), 32 columns SW64
  // (D = 32), 16 columns SW32 (D = 72: five atoms, columns 72..79 of the last zero-filled by TMA)
  const uint32_t box0 = D % 64 == 0 ? 64 : (D % 32 == 0 ? 32 : 16);
  const CUtensorMapSwizzle sw = D % 64 == 0 ? CU_TENSOR_MAP_SWIZZLE_128B
                                            : (D % 32 == 0 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  if (!ua::make_tmap_bf16_4d(m, base, dims, strides, box0, box_rows, sw))
    return fail(UA_ERR_CUDA, "cuTensorMapEncodeTiled failed (D=%d N=%lld heads=%d)", D, (long long)N, heads);
  return UA_OK;
}

// Workspace plans (byte offsets).
struct FwdPlan {
  size_t send = 0, recv = 0, o_head = 0, total = 0;
};
FwdPlan plan_fwd(const Shape& s) {
  FwdPlan p;
  if (s.P == 1) return p;
  const size_t S = size_t(s.shard()) * 2;
  p.send = 0;                         // [3][P][Nl][B][Hl][D]; reused as recv_o [P][Nl][B][Hl][D]
  p.recv = align_up(p.send + 3 * S);  // [3][N][B][Hl][D]
  p.o_head = align_up(p.recv + 3 * S);
  p.total = align_up(p.o_head + S);
  return p;
}
struct BwdPlan {
  size_t send = 0, send_delta = 0, recv = 0, recv_delta = 0, grad = 0, delta = 0, head = 0, total = 0;
};
size_t head_bwd_bytes(const Shape& s);
BwdPlan plan_bwd(const Shape& s) {
  BwdPlan p;
  const size_t S = size_t(s.shard()) * 2;
  const size_t DL = size_t(s.B * s.Nl * s.H) * 4;  // Delta of one shard
  if (s.P == 1) {
    p.delta = 0;                                  // [N][B][H] fp32
    p.head = align_up(DL);                        // head_bwd workspace: dq_acc, (lse, Delta) table
    p.total = align_up(p.head + head_bwd_bytes(s));
    return p;
  }
  p.send = 0;                                     // [4][P][Nl][B][Hl][D]; reused as recv_grad [3][P]...
  p.send_delta = align_up(4 * S);                 // [P][Nl][B][Hl]
  p.recv = align_up(p.send_delta + DL);           // [4][N][B][Hl][D]
  p.recv_delta = align_up(p.recv + 4 * S);        // [N][B][Hl]
  p.grad = align_up(p.recv_delta + DL);           // [3][N][B][Hl][D] bf16
  p.head = align_up(p.grad + 3 * S);
  p.total = align_up(p.head + head_bwd_bytes(s));
  return p;
}

// LSS plans (P > 1).  KV gathered layout [N][B][H][D] (rank p's tokens at rows p*Nl..).
// Rank-local LSS backward workspace: Delta [Nl][B][H] fp32, dq_acc [B*H][Nl_pad][D] fp32,
// (lse, Delta) table [B*H][Nl_pad] float2.
struct LssRankPlan {
  size_t delta = 0, dq_acc = 0, lsed = 0, total = 0;
};
LssRankPlan plan_lss_rank(const Shape& s) {
  LssRankPlan p;
  const int64_t n_pad = (s.Nl + 127) / 128 * 128;
  p.delta = 0;
  p.dq_acc = align_up(p.delta + size_t(s.B * s.Nl * s.H) * 4);
  p.lsed = align_up(p.dq_acc + size_t(s.B * s.H * n_pad * s.D) * 4);
  p.total = align_up(p.lsed + size_t(s.B * s.H * n_pad) * 8);
  return p;
}
struct LssPlan {
  size_t kv_send = 0, kv_full = 0, rank = 0, part = 0, red = 0, total = 0;
};
LssPlan plan_lss(const Shape& s, bool bwd) {
  LssPlan p;
  if (s.P == 1) return p;
  const size_t S = size_t(s.shard()) * 2;          // one bf16 [B][Nl][H][D] shard
  p.kv_send = 0;                                    // [2][Nl][B][H][D] bf16 (B > 1: local K, V re-laid)
  p.kv_full = align_up(p.kv_send + 2 * S);          // [2][N][B][H][D] bf16
  p.total = align_up(p.kv_full + 2 * S * s.P);
  if (!bwd) return p;
  p.rank = p.total;                                 // rank-local backward workspace (LssRankPlan)
  p.part = align_up(p.rank + plan_lss_rank(s).total);                   // [2][N][B][H][D] fp32 partial dK, dV
  p.red = align_up(p.part + 2 * S * 2 * s.P);                          // [2][Nl][B][H][D] fp32 reduced
  p.total = align_up(p.red + 2 * S * 2);
  return p;
}

// Fused all-to-all of `nt` equally-shaped tensors: peer chunk i of tensor w is
// `count` elements at send[w] + i*count (bytes elem_size).  One NCCL group =
// one collective call in the S:274 sense.
ua_status a2a(ua_ctx* ctx, void* const* send, void* const* recv, int nt, size_t count, ncclDataType_t dt,
              size_t elem_size, cudaStream_t stream) {
  UA_NCCL(ncclGroupStart());
  for (int peer = 0; peer < ctx->P; ++peer) {
    for (int w = 0; w < nt; ++w) {
      const char* sp = static_cast<const char*>(send[w]) + size_t(peer) * count * elem_size;
      char* rp = static_cast<char*>(recv[w]) + size_t(peer) * count * elem_size;
      ncclResult_t r1 = ncclSend(sp, count, dt, peer, ctx->comm, stream);
      ncclResult_t r2 = ncclRecv(rp, count, dt, peer, ctx->comm, stream);
      if (r1 != ncclSuccess || r2 != ncclSuccess) {
        ncclGroupEnd();
        return fail(UA_ERR_NCCL, "ncclSend/Recv: %s", ncclGetErrorString(r1 != ncclSuccess ? r1 : r2));
      }
    }
  }
  UA_NCCL(ncclGroupEnd());
  ctx->a2a_bytes += int64_t(ctx->P - 1) * int64_t(count * elem_size) * nt;
  return UA_OK;
}

ua_status check_async(ua_ctx* ctx) {
  if (ctx) {  // kernels launch on the current device; a ctx is bound to one
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != ctx->device)
      return fail(UA_ERR_INVALID_ARG, "current CUDA device %d is not the ctx's device %d (cudaSetDevice first)", dev,
                  ctx->device);
  }
  if (ctx && ctx->peer_err_host && *static_cast<volatile int*>(ctx->peer_err_host) != 0)
    return fail(UA_ERR_CUDA, "a peer all-to-all wait timed out (a peer rank failed, died or diverged); "
                             "outputs of that call are undefined and this ctx must be destroyed");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(UA_ERR_CUDA, "pending CUDA error: %s", cudaGetErrorString(e));
  if (ctx && ctx->comm) {
    ncclResult_t ar = ncclSuccess;
    ncclCommGetAsyncError(ctx->comm, &ar);
    if (ar != ncclSuccess) return fail(UA_ERR_NCCL, "NCCL async error: %s", ncclGetErrorString(ar));
  }
  return UA_OK;
}

// Rows of a bf16 [.][rows][heads][D] view: base + token / head / batch strides (elements).
struct Rows {
  const void* base;
  int64_t sn, sh, sb, n;
};

ua_status launch_attention_fwd(Rows q, const void* k, const void* v, Rows kv, ua::ViewArg o, float* o_f32,
                               int64_t of_sn, int64_t of_sh, int64_t of_sb, float* lse, int64_t l_sh, int64_t l_sb,
                               int64_t B, int heads, int D, int64_t kv_begin, int64_t kv_end, cudaStream_t stream,
                               const ua::PeerOut* o_peer = nullptr) {
  ua::FwdParams p;
  std::memset(&p, 0, sizeof(p));
  UA_TRY(make_map(&p.tm_q, q.base, D, q.n, heads, B, q.sn, q.sh, q.sb));
  UA_TRY(make_map(&p.tm_k, k, D, kv.n, heads, B, kv.sn, kv.sh, kv.sb));
  UA_TRY(make_map(&p.tm_v, v, D, kv.n, heads, B, kv.sn, kv.sh, kv.sb));
  p.o = o;
  if (o_peer) p.o_peer = *o_peer;
  p.o_f32 = o_f32;
  p.of_sn = of_sn; p.of_sh = of_sh; p.of_sb = of_sb;
  p.lse = lse;
  p.l_sh = l_sh; p.l_sb = l_sb;
  p.n_q = int(q.n);
  p.kv_begin = int(kv_begin);
  p.kv_end = int(kv_end);
  p.scale_log2 = float(1.4426950408889634 / std::sqrt(double(D)));
  p.d_io = D;
  UA_CUDA(ua::launch_attn_fwd(p, D, int(B), heads, stream));
  return UA_OK;
}

// Square problem (queries and keys share N and strides).
ua_status launch_attention_fwd(const void* q, const void* k, const void* v, int64_t sn, int64_t sh, int64_t sb,
                               ua::ViewArg o, float* o_f32, int64_t of_sn, int64_t of_sh, int64_t of_sb, float* lse,
                               int64_t l_sh, int64_t l_sb, int64_t B, int64_t N, int heads, int D, int64_t kv_begin,
                               int64_t kv_end, cudaStream_t stream, const ua::PeerOut* o_peer = nullptr) {
  const Rows r{q, sn, sh, sb, N};
  return launch_attention_fwd(r, k, v, r, o, o_f32, of_sn, of_sh, of_sb, lse, l_sh, l_sb, B, heads, D, kv_begin,
                              kv_end, stream, o_peer);
}

// Backward over queries q.n (q, dout share q's strides) and keys kv.n (k, v).
// kv_f32: dk / dv views are fp32 partial sums.
ua_status launch_attention_bwd(Rows q, const void* dout, const void* k, const void* v, Rows kv, ua::ViewArg dk,
                               ua::ViewArg dv, int kv_f32, float* dq_acc, const float* lse, int64_t l_sh,
                               int64_t l_sb, const float* delta, int64_t d_sn, int64_t d_sh, int64_t d_sb, int64_t B,
                               int heads, int D, float2* lsed, int deterministic, cudaStream_t stream,
                               const ua::PeerOut* dk_peer = nullptr, const ua::PeerOut* dv_peer = nullptr) {
  ua::BwdParams p;
  std::memset(&p, 0, sizeof(p));
  if (dk_peer) p.dk_peer = *dk_peer;
  if (dv_peer) p.dv_peer = *dv_peer;
  const int64_t N = q.n;
  // (-lse*log2e, Delta) per query row, contiguous per head (bulk-loaded by the kernel)
  UA_CUDA(ua::launch_bwd_prep(lse, l_sh, l_sb, delta, d_sn, d_sh, d_sb, lsed, B, heads, N, stream));
  p.lsed = lsed;
  UA_TRY(make_map(&p.tm_q, q.base, D, N, heads, B, q.sn, q.sh, q.sb));
  UA_TRY(make_map(&p.tm_do, dout, D, N, heads, B, q.sn, q.sh, q.sb));
  UA_TRY(make_map(&p.tm_qh, q.base, D, N, heads, B, q.sn, q.sh, q.sb, 64));
  UA_TRY(make_map(&p.tm_doh, dout, D, N, heads, B, q.sn, q.sh, q.sb, 64));
  UA_TRY(make_map(&p.tm_k, k, D, kv.n, heads, B, kv.sn, kv.sh, kv.sb));
  UA_TRY(make_map(&p.tm_v, v, D, kv.n, heads, B, kv.sn, kv.sh, kv.sb));
  const int64_t n_pad = (N + 127) / 128 * 128;
  if (!ua::make_tmap_f32_2d(&p.tm_dq, dq_acc, uint64_t(D), uint64_t(B * heads * n_pad), 128))
    return fail(UA_ERR_CUDA, "cuTensorMapEncodeTiled failed for dq_acc");
  p.dk = dk;
  p.dv = dv;
  p.kv_f32 = kv_f32;
  p.dq_acc = dq_acc;
  p.lse = lse;
  p.l_sh = l_sh; p.l_sb = l_sb;
  p.delta = delta;
  p.d_sn = d_sn; p.d_sh = d_sh; p.d_sb = d_sb;
  p.n = int(N);
  p.n_kv = int(kv.n);
  p.heads = heads;
  p.batch = int(B);
  p.scale = float(1.0 / std::sqrt(double(D)));
  p.scale_log2 = float(1.4426950408889634 / std::sqrt(double(D)));
  p.d_io = D;
  p.deterministic = deterministic;
  UA_CUDA(ua::launch_attn_bwd_ws(p, D, stream));
  return UA_OK;
}

// Square problem.
ua_status launch_attention_bwd(const void* q, const void* k, const void* v, const void* dout, int64_t sn, int64_t sh,
                               int64_t sb, ua::ViewArg dk, ua::ViewArg dv, float* dq_acc, const float* lse,
                               int64_t l_sh, int64_t l_sb, const float* delta, int64_t d_sn, int64_t d_sh,
                               int64_t d_sb, int64_t B, int64_t N, int heads, int D, float2* lsed,
                               int deterministic, cudaStream_t stream, const ua::PeerOut* dk_peer = nullptr,
                               const ua::PeerOut* dv_peer = nullptr) {
  const Rows r{q, sn, sh, sb, N};
  return launch_attention_bwd(r, dout, k, v, r, dk, dv, 0, dq_acc, lse, l_sh, l_sb, delta, d_sn, d_sh, d_sb, B, heads,
                              D, lsed, deterministic, stream, dk_peer, dv_peer);
}

// ------------------------------------------------------------ peer all-to-all
// Library-owned receive buffers in NCCL symmetric memory: allocated with ncclMemAlloc, registered
// collectively as a window (NCCL_WIN_COLL_SYMMETRIC), and every rank's copy addressed through the
// window's load/store-accessible peer pointers (once per shape, not per call).
ua_status peer_map(ua_ctx* ctx, ua_ctx::PeerBuf& pb, cudaStream_t stream) {
  UA_NCCL(ncclCommWindowRegister(ctx->comm, pb.local, pb.bytes, &pb.win, NCCL_WIN_COLL_SYMMETRIC));
  const int P = ctx->P;
  void** d = nullptr;
  UA_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), sizeof(void*) * P));
  UA_CUDA(ua_internal::launch_lsa_ptrs(pb.win, P, d, stream));
  UA_CUDA(cudaMemcpyAsync(pb.peer, d, sizeof(void*) * P, cudaMemcpyDeviceToHost, stream));
  UA_CUDA(cudaStreamSynchronize(stream));
  cudaFree(d);
  for (int k = 0; k < P; ++k)
    if (!pb.peer[k]) return fail(UA_ERR_NCCL, "NCCL window: no load/store pointer for rank %d", k);
  return UA_OK;
}

void peer_release(ua_ctx* ctx, ua_ctx::PeerBuf& pb) {
  if (pb.win) ncclCommWindowDeregister(ctx->comm, pb.win);
  if (pb.local) ncclMemFree(pb.local);
  pb = ua_ctx::PeerBuf();
}

// Collective (all ranks call with the same shape): make sure `pb` holds at
// least `bytes`, re-allocating and re-registering when it grows.
ua_status peer_ensure(ua_ctx* ctx, ua_ctx::PeerBuf& pb, size_t bytes, cudaStream_t stream) {
  if (pb.local && pb.bytes >= bytes) return UA_OK;
  // every rank has drained its previous steps before anyone deregisters / frees
  UA_CUDA(cudaDeviceSynchronize());
  int* dummy = nullptr;
  UA_CUDA(cudaMalloc(&dummy, sizeof(int)));
  UA_NCCL(ncclAllReduce(dummy, dummy, 1, ncclInt32, ncclSum, ctx->comm, stream));
  UA_CUDA(cudaStreamSynchronize(stream));
  cudaFree(dummy);
  peer_release(ctx, pb);
  const size_t align = NCCL_WIN_REQUIRED_ALIGNMENT;
  bytes = (bytes + align - 1) / align * align;
  UA_NCCL(ncclMemAlloc(&pb.local, bytes));
  UA_CUDA(cudaMemset(pb.local, 0, bytes));
  pb.bytes = bytes;
  return peer_map(ctx, pb, stream);
}

ua::PeerFlags peer_flags(const ua_ctx* ctx) {
  ua::PeerFlags f{};
  for (int k = 0; k < ctx->P; ++k) f.peer[k] = static_cast<int64_t*>(ctx->flags.peer[k]);
  return f;
}

ua::PeerOut peer_out(const ua_ctx::PeerBuf& pb, size_t offset, const Shape& s, int rank) {
  ua::PeerOut o{};
  for (int k = 0; k < s.P; ++k) o.base[k] = static_cast<char*>(pb.peer[k]) + offset;
  o.nl = s.Nl;
  o.H = s.H;
  o.h0 = rank * s.Hl;
  return o;
}

enum { kSlotFwdIn = 0, kSlotFwdOut = 1, kSlotBwdIn = 2, kSlotBwdOut = 3 };

// ------------------------------------------------------------ rank-local steps
// Strides (elements) of the bf16 tensors a head-shard step reads: the a2a receive
// layout [N][B][Hl][D], or the user layout [B][N][H][D] at P = 1.
struct Strides {
  int64_t sn, sh, sb;
};
Strides head_layout(int64_t B, int Hl, int D) { return {B * int64_t(Hl) * D, D, int64_t(Hl) * D}; }

// A3 on one rank's head shard: O into the view o (a2a #2 send layout) or, with
// o_peer, straight into the token owners' tensors (A3 + A5 fused).
ua_status head_fwd(ua_ctx* ctx, const void* q, const void* k, const void* v, Strides st, void* o,
                   const ua::PeerOut* o_peer, float* lse, int64_t B, int64_t N, int Hl, int D, cudaStream_t stream) {
  const ua::ViewArg ov{o_peer ? nullptr : o, st.sn, st.sh, st.sb};
  Phase ph(ctx, UA_PHASE_ATTN_FWD, stream);
  return launch_attention_fwd(q, k, v, st.sn, st.sh, st.sb, ov, nullptr, 0, 0, 0, lse, N, int64_t(Hl) * N, B, N, Hl,
                              D, 0, N, stream, o_peer);
}

// Workspace of head_bwd: fp32 dQ accumulator [B*Hl][N_pad][D] + (lse, Delta) table [B*Hl][N_pad].
struct HeadBwdPlan {
  size_t dq_acc = 0, lsed = 0, total = 0;
};
HeadBwdPlan plan_head_bwd(int64_t B, int64_t N, int Hl, int D) {
  HeadBwdPlan p;
  const int64_t n_pad = (N + 127) / 128 * 128;
  p.lsed = align_up(size_t(B * Hl * n_pad * D) * 4);
  p.total = align_up(p.lsed + size_t(B * Hl * n_pad) * 8);
  return p;
}
size_t head_bwd_bytes(const Shape& s) { return plan_head_bwd(s.B, s.N, s.Hl, s.D).total; }

// B3 + B4 on one rank's head shard: delta [N][B][Hl] (strides B*Hl, 1, Hl);
// dq, dk, dv into views with the inputs' strides, or (peers = {dq, dk, dv}
// owner maps) straight into the token owners' tensors (B3 + B5 fused).
ua_status head_bwd(ua_ctx* ctx, const void* q, const void* k, const void* v, const void* dout, Strides st,
                   const float* lse, const float* delta, void* dq, void* dk, void* dv, const ua::PeerOut* peers,
                   int64_t B, int64_t N, int Hl, int D, int deterministic, char* ws, cudaStream_t stream) {
  const HeadBwdPlan plan = plan_head_bwd(B, N, Hl, D);
  float* dq_acc = reinterpret_cast<float*>(ws + plan.dq_acc);
  const int64_t n_pad = (N + 127) / 128 * 128;
  const float scale = float(1.0 / std::sqrt(double(D)));
  {
    Phase ph(ctx, UA_PHASE_ATTN_BWD, stream);
    UA_CUDA(cudaMemsetAsync(dq_acc, 0, size_t(B * Hl * n_pad * D) * 4, stream));
    const ua::ViewArg vdk{peers ? nullptr : dk, st.sn, st.sh, st.sb}, vdv{peers ? nullptr : dv, st.sn, st.sh, st.sb};
    UA_TRY(launch_attention_bwd(q, k, v, dout, st.sn, st.sh, st.sb, vdk, vdv, dq_acc, lse, N, int64_t(Hl) * N, delta,
                                B * int64_t(Hl), 1, Hl, B, N, Hl, D, reinterpret_cast<float2*>(ws + plan.lsed),
                                deterministic, stream, peers ? &peers[1] : nullptr, peers ? &peers[2] : nullptr));
  }
  Phase ph(ctx, UA_PHASE_DQ_FINALIZE, stream);
  if (peers) {
    UA_CUDA(ua::launch_finalize_push(dq_acc, peers[0], B, N, Hl, D, scale, stream));
  } else {
    UA_CUDA(ua::launch_dq_finalize(dq_acc, ua::ViewArg{dq, st.sn, st.sh, st.sb}, B, N, Hl, D, scale, stream));
  }
  return UA_OK;
}

ua_status check_ptrs(std::initializer_list<const void*> ptrs) {
  for (const void* ptr : ptrs) {
    if (!ptr) return fail(UA_ERR_INVALID_ARG, "null tensor pointer");
    if (!aligned16(ptr)) return fail(UA_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  }
  return UA_OK;
}

}  // namespace

extern "C" {

const char* ua_version(void) { return "ulysses_attn 0.1 sm_100a"; }

const char* ua_status_string(ua_status s) {
  switch (s) {
    case UA_OK: return "UA_OK";
    case UA_ERR_INVALID_ARG: return "UA_ERR_INVALID_ARG";
    case UA_ERR_HEAD_DIVISIBILITY: return "UA_ERR_HEAD_DIVISIBILITY";
    case UA_ERR_SEQ_DIVISIBILITY: return "UA_ERR_SEQ_DIVISIBILITY";
    case UA_ERR_UNSUPPORTED: return "UA_ERR_UNSUPPORTED";
    case UA_ERR_CUDA: return "UA_ERR_CUDA";
    case UA_ERR_NCCL: return "UA_ERR_NCCL";
  }
  return "UA_ERR_UNKNOWN";
}

const char* ua_last_error(void) { return g_err.c_str(); }

ua_status ua_validate(int64_t B, int64_t N, int H, int D, int P) {
  if (B < 1 || N < 1 || H < 1 || D < 1 || P < 1)
    return fail(UA_ERR_INVALID_ARG, "B, N, H, D, P must be >= 1 (got B=%lld N=%lld H=%d D=%d P=%d)", (long long)B,
                (long long)N, H, D, P);
  if (P > H || H % P != 0)
    return fail(UA_ERR_HEAD_DIVISIBILITY, "Ulysses needs P <= H and H %% P == 0 (H=%d, P=%d)", H, P);
  if (N % P != 0) return fail(UA_ERR_SEQ_DIVISIBILITY, "Ulysses needs N %% P == 0 (N=%lld, P=%d)", (long long)N, P);
  if (D != 32 && D != 64 && D != 72 && D != 128)
    return fail(UA_ERR_UNSUPPORTED, "head dim D=%d not in {32, 64, 72, 128}", D);
  if (N >= (int64_t(1) << 31)) return fail(UA_ERR_UNSUPPORTED, "N=%lld >= 2^31", (long long)N);
  if (B * N * H >= (int64_t(1) << 40)) return fail(UA_ERR_UNSUPPORTED, "problem too large");
  return UA_OK;
}

ua_status ua_workspace_size(int64_t B, int64_t N, int H, int D, int P, size_t* fwd_bytes, size_t* bwd_bytes) {
  UA_TRY(ua_validate(B, N, H, D, P));
  Shape s = make_shape(B, N, H, D, P);
  if (fwd_bytes) *fwd_bytes = plan_fwd(s).total;
  if (bwd_bytes) *bwd_bytes = plan_bwd(s).total;
  return UA_OK;
}

ua_status ua_get_unique_id(unsigned char uid[128]) {
  if (!uid) return fail(UA_ERR_INVALID_ARG, "uid is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  UA_NCCL(ncclGetUniqueId(&id));
  std::memcpy(uid, &id, 128);
  return UA_OK;
}

ua_status ua_ctx_create(const unsigned char* uid, int P, int rank, int cuda_device, ua_ctx** out) {
  if (!out) return fail(UA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (P < 1 || rank < 0 || rank >= P) return fail(UA_ERR_INVALID_ARG, "bad P=%d rank=%d", P, rank);
  if (P > 1 && !uid) return fail(UA_ERR_INVALID_ARG, "uid is NULL for P=%d", P);
  UA_CUDA(cudaSetDevice(cuda_device));
  UA_TRY(check_device());
  ua_ctx* c = new ua_ctx();
  c->P = P;
  c->rank = rank;
  c->device = cuda_device;
  if (P > 1) {
    ncclUniqueId id;
    std::memcpy(&id, uid, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, P, id, rank);
    if (r != ncclSuccess) {
      delete c;
      return fail(UA_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
  }
  *out = c;
  return UA_OK;
}

ua_status ua_ctx_set_a2a_mode(ua_ctx* ctx, int mode) {
  if (!ctx) return fail(UA_ERR_INVALID_ARG, "ctx is NULL");
  if (mode != UA_A2A_NCCL && mode != UA_A2A_PEER) return fail(UA_ERR_INVALID_ARG, "bad a2a mode %d", mode);
  if (mode == UA_A2A_PEER) {
    if (ctx->P == 1) return fail(UA_ERR_UNSUPPORTED, "peer all-to-all needs P > 1");
    if (ctx->P > ua::kMaxPeers) return fail(UA_ERR_UNSUPPORTED, "peer all-to-all supports P <= %d", ua::kMaxPeers);
    if (!ctx->peer_err_host) {
      UA_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->peer_err_host), sizeof(int), cudaHostAllocMapped));
      *ctx->peer_err_host = 0;
      UA_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->peer_err), ctx->peer_err_host, 0));
    }
    if (!ctx->flags.local) {
      cudaStream_t s;
      UA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      ua_status st = peer_ensure(ctx, ctx->flags, sizeof(int64_t) * 4 * ua::kMaxPeers, s);
      cudaStreamDestroy(s);
      if (st != UA_OK) return st;
    }
  }
  ctx->a2a_mode = mode;
  return UA_OK;
}

ua_status ua_ctx_set_deterministic(ua_ctx* ctx, int enable) {
  if (!ctx) return fail(UA_ERR_INVALID_ARG, "ctx is NULL");
  ctx->deterministic = enable ? 1 : 0;
  return UA_OK;
}

ua_status ua_ctx_get_deterministic(const ua_ctx* ctx, int* enable) {
  if (!ctx || !enable) return fail(UA_ERR_INVALID_ARG, "null argument");
  *enable = ctx->deterministic;
  return UA_OK;
}

ua_status ua_ctx_get_a2a_mode(const ua_ctx* ctx, int* mode) {
  if (!ctx || !mode) return fail(UA_ERR_INVALID_ARG, "null argument");
  *mode = ctx->a2a_mode;
  return UA_OK;
}

ua_status ua_ctx_destroy(ua_ctx* ctx) {
  if (!ctx) return UA_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != ctx->device) cudaSetDevice(ctx->device);  // release on the ctx's device, restore below
  if (ctx->flags.local) {
    cudaDeviceSynchronize();
    for (auto* pb : {&ctx->flags, &ctx->fwd_in, &ctx->fwd_out, &ctx->bwd_in, &ctx->bwd_out}) peer_release(ctx, *pb);
  }
  ua_internal::layer_release(ctx);
  if (ctx->peer_err_host) cudaFreeHost(ctx->peer_err_host);
  ncclResult_t r = ncclSuccess;
  if (ctx->comm) r = ncclCommDestroy(ctx->comm);
  for (auto& rec : ctx->pending) {
    cudaEventDestroy(rec.a);
    cudaEventDestroy(rec.b);
  }
  for (cudaEvent_t e : ctx->pool) cudaEventDestroy(e);
  const int dev = ctx->device;
  delete ctx;
  if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  if (r != ncclSuccess) return fail(UA_ERR_NCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return UA_OK;
}

ua_status ua_ctx_comm_stats(const ua_ctx* ctx, int64_t* a2a_calls, int64_t* a2a_bytes_sent) {
  if (!ctx) return fail(UA_ERR_INVALID_ARG, "ctx is NULL");
  if (a2a_calls) *a2a_calls = ctx->a2a_calls;
  if (a2a_bytes_sent) *a2a_bytes_sent = ctx->a2a_bytes;
  return UA_OK;
}

ua_status ua_ulysses_attn_fwd(ua_ctx* ctx, const void* q, const void* k, const void* v, void* out, float* lse,
                              int64_t B, int64_t N, int H, int D, int P, void* workspace, size_t workspace_bytes,
                              ua_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  UA_TRY(ua_validate(B, N, H, D, P));
  if (!ctx) return fail(UA_ERR_INVALID_ARG, "ctx is NULL");
  if (P != ctx->P) return fail(UA_ERR_INVALID_ARG, "P=%d differs from ctx P=%d", P, ctx->P);
  if (!q || !k || !v || !out || !lse) return fail(UA_ERR_INVALID_ARG, "null tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out) || !aligned16(lse))
    return fail(UA_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  const Shape s = make_shape(B, N, H, D, P);
  const FwdPlan plan = plan_fwd(s);
  if (workspace_bytes < plan.total || (plan.total > 0 && !workspace))
    return fail(UA_ERR_INVALID_ARG, "workspace too small: need %zu bytes, got %zu", plan.total, workspace_bytes);
  UA_TRY(check_device());
  UA_TRY(check_async(ctx));

  if (P == 1) return head_fwd(ctx, q, k, v, Strides{int64_t(H) * D, D, N * H * D}, out, nullptr, lse, B, N, H, D, stream);

  if (ctx->a2a_mode == UA_A2A_PEER) {
    // Fused all-to-alls over NVLink peer stores (no NCCL on the data path).
    const size_t S = size_t(s.shard()) * 2;
    UA_TRY(peer_ensure(ctx, ctx->fwd_in, 3 * S, stream));   // [3][N][B][Hl][D] on every rank
    UA_TRY(peer_ensure(ctx, ctx->fwd_out, S, stream));      // [B][Nl][H][D] token-owner output
    const int64_t step = ++ctx->step_fwd;
    const ua::PeerFlags fl = peer_flags(ctx);
    {  // 1+2. pack straight into every head owner's receive buffer, then flag it
      Phase ph(ctx, UA_PHASE_PACK_FWD, stream);
      ua::PeerPack pk{};
      pk.src[0] = q; pk.src[1] = k; pk.src[2] = v;
      for (int j = 0; j < P; ++j) pk.dst[j] = ctx->fwd_in.peer[j];
      pk.ntensors = 3;
      UA_CUDA(ua::launch_pack_push(pk, B, s.Nl, H, D, P, ctx->rank, stream));
      UA_CUDA(ua::launch_signal(fl, kSlotFwdIn, ctx->rank, P, step, stream));
    }
    {
      Phase ph(ctx, UA_PHASE_A2A_FWD_IN, stream);
      UA_CUDA(ua::launch_wait_copy(static_cast<const int64_t*>(ctx->flags.local), kSlotFwdIn, P, step, nullptr,
                                   nullptr, 0, ctx->peer_err, stream));
      ctx->a2a_calls += 1;
      ctx->a2a_bytes += int64_t(P - 1) * int64_t(s.chunk()) * 2 * 3;
    }
    char* rin = static_cast<char*>(ctx->fwd_in.local);
    const ua::PeerOut po = peer_out(ctx->fwd_out, 0, s, ctx->rank);
    // 3+4. attention; the epilogue stores O rows into the token owners' buffers
    UA_TRY(head_fwd(ctx, rin, rin + S, rin + 2 * S, head_layout(B, s.Hl, D), nullptr, &po, lse, B, N, s.Hl, D, stream));
    {
      Phase ph(ctx, UA_PHASE_A2A_FWD_OUT, stream);
      UA_CUDA(ua::launch_signal(fl, kSlotFwdOut, ctx->rank, P, step, stream));
    }
    {  // 5. all owners' rows are in: copy into the caller's out
      Phase ph(ctx, UA_PHASE_UNPACK_FWD, stream);
      UA_CUDA(ua::launch_wait_copy(static_cast<const int64_t*>(ctx->flags.local), kSlotFwdOut, P, step,
                                   ctx->fwd_out.local, out, int64_t(S), ctx->peer_err, stream));
      ctx->a2a_calls += 1;
      ctx->a2a_bytes += int64_t(P - 1) * int64_t(s.chunk()) * 2;
    }
    return UA_OK;
  }

  char* ws = static_cast<char*>(workspace);
  const size_t S = size_t(s.shard()) * 2;
  void* send[3] = {ws + plan.send, ws + plan.send + S, ws + plan.send + 2 * S};
  void* recv[3] = {ws + plan.recv, ws + plan.recv + S, ws + plan.recv + 2 * S};
  const void* src[3] = {q, k, v};
  {  // 1. pack (sequence shard -> per-destination head chunks)
    Phase ph(ctx, UA_PHASE_PACK_FWD, stream);
    UA_CUDA(ua::launch_pack(src, send, 3, B, s.Nl, H, D, P, nullptr, nullptr, nullptr, stream));
  }
  {  // 2. all-to-all #1 (fused q, k, v): rank j receives all N tokens of its head block
    Phase ph(ctx, UA_PHASE_A2A_FWD_IN, stream);
    UA_TRY(a2a(ctx, send, recv, 3, size_t(s.chunk()), ncclBfloat16, 2, stream));
    ctx->a2a_calls += 1;
  }
  // 3. attention on the head shard, layout [N][B][Hl][D]; O straight into the send layout of #2
  void* o_head = ws + plan.o_head;
  UA_TRY(head_fwd(ctx, recv[0], recv[1], recv[2], head_layout(B, s.Hl, D), o_head, nullptr, lse, B, N, s.Hl, D,
                  stream));
  void* recv_o = ws + plan.send;
  {  // 4. all-to-all #2: token block i of every local head goes back to rank i
    Phase ph(ctx, UA_PHASE_A2A_FWD_OUT, stream);
    UA_TRY(a2a(ctx, &o_head, &recv_o, 1, size_t(s.chunk()), ncclBfloat16, 2, stream));
    ctx->a2a_calls += 1;
  }
  {  // 5. unpack head chunks -> [B][Nl][H][D]
    Phase ph(ctx, UA_PHASE_UNPACK_FWD, stream);
    const void* usrc[1] = {recv_o};
    void* udst[1] = {out};
    UA_CUDA(ua::launch_unpack(usrc, udst, 1, B, s.Nl, H, D, P, stream));
  }
  return UA_OK;
}

ua_status ua_ulysses_attn_bwd(ua_ctx* ctx, const void* q, const void* k, const void* v, const void* out,
                              const float* lse, const void* dout, void* dq, void* dk, void* dv, int64_t B, int64_t N,
                              int H, int D, int P, void* workspace, size_t workspace_bytes, ua_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  UA_TRY(ua_validate(B, N, H, D, P));
  if (!ctx) return fail(UA_ERR_INVALID_ARG, "ctx is NULL");
  if (P != ctx->P) return fail(UA_ERR_INVALID_ARG, "P=%d differs from ctx P=%d", P, ctx->P);
  const void* ptrs[] = {q, k, v, out, lse, dout, dq, dk, dv};
  for (const void* ptr : ptrs) {
    if (!ptr) return fail(UA_ERR_INVALID_ARG, "null tensor pointer");
    if (!aligned16(ptr)) return fail(UA_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  }
  const Shape s = make_shape(B, N, H, D, P);
  const BwdPlan plan = plan_bwd(s);
  if (workspace_bytes < plan.total || !workspace)
    return fail(UA_ERR_INVALID_ARG, "workspace too small: need %zu bytes, got %zu", plan.total, workspace_bytes);
  UA_TRY(check_device());
  UA_TRY(check_async(ctx));
  char* ws = static_cast<char*>(workspace);

  if (P == 1) {
    float* delta = reinterpret_cast<float*>(ws + plan.delta);
    {  // Delta[n][b][h] = sum_d dO.O (fp32)
      Phase ph(ctx, UA_PHASE_PACK_BWD, stream);
      UA_CUDA(ua::launch_pack(nullptr, nullptr, 0, B, N, H, D, 1, dout, out, delta, stream));
    }
    return head_bwd(ctx, q, k, v, dout, Strides{int64_t(H) * D, D, N * H * D}, lse, delta, dq, dk, dv, nullptr, B, N,
                    H, D, ctx->deterministic, ws + plan.head, stream);
  }

  if (ctx->a2a_mode == UA_A2A_PEER) {
    // Fused all-to-alls over NVLink peer stores (no NCCL on the data path).
    const size_t S = size_t(s.shard()) * 2;
    const size_t DL = size_t(B * s.Nl * H) * 4;  // Delta bytes received per rank
    UA_TRY(peer_ensure(ctx, ctx->bwd_in, 4 * S + DL, stream));  // [4][N][B][Hl][D] + Delta [N][B][Hl]
    UA_TRY(peer_ensure(ctx, ctx->bwd_out, 3 * S, stream));      // [3][B][Nl][H][D]: dq, dk, dv of the owner
    const int64_t step = ++ctx->step_bwd;
    const ua::PeerFlags fl = peer_flags(ctx);
    {  // 1+2. q, k, v, dO + Delta straight into every head owner's receive buffer
      Phase ph(ctx, UA_PHASE_PACK_BWD, stream);
      ua::PeerPack pk{};
      pk.src[0] = q; pk.src[1] = k; pk.src[2] = v; pk.src[3] = dout;
      for (int j = 0; j < P; ++j) pk.dst[j] = ctx->bwd_in.peer[j];
      pk.ntensors = 4;
      pk.dout = dout;
      pk.out = out;
      UA_CUDA(ua::launch_pack_push(pk, B, s.Nl, H, D, P, ctx->rank, stream));
      UA_CUDA(ua::launch_signal(fl, kSlotBwdIn, ctx->rank, P, step, stream));
    }
    {
      Phase ph(ctx, UA_PHASE_A2A_BWD_IN, stream);
      UA_CUDA(ua::launch_wait_copy(static_cast<const int64_t*>(ctx->flags.local), kSlotBwdIn, P, step, nullptr,
                                   nullptr, 0, ctx->peer_err, stream));
      ctx->a2a_calls += 1;
      ctx->a2a_bytes += int64_t(P - 1) * (int64_t(s.chunk()) * 2 * 4 + int64_t(s.Nl * B * s.Hl) * 4);
    }
    char* rin = static_cast<char*>(ctx->bwd_in.local);
    const float* rdelta = reinterpret_cast<const float*>(rin + 4 * S);
    const ua::PeerOut owners[3] = {peer_out(ctx->bwd_out, 0, s, ctx->rank), peer_out(ctx->bwd_out, S, s, ctx->rank),
                                   peer_out(ctx->bwd_out, 2 * S, s, ctx->rank)};
    // 3+4. attention backward; dK, dV rows (epilogue) and dQ rows (finaliser) go straight to the token owners
    UA_TRY(head_bwd(ctx, rin, rin + S, rin + 2 * S, rin + 3 * S, head_layout(B, s.Hl, D), lse, rdelta, nullptr,
                    nullptr, nullptr, owners, B, N, s.Hl, D, ctx->deterministic, ws + plan.head, stream));
    {
      Phase ph(ctx, UA_PHASE_A2A_BWD_OUT, stream);
      UA_CUDA(ua::launch_signal(fl, kSlotBwdOut, ctx->rank, P, step, stream));
    }
    {  // 5. all heads' rows are in: copy into the caller's dq, dk, dv
      Phase ph(ctx, UA_PHASE_UNPACK_BWD, stream);
      char* rout = static_cast<char*>(ctx->bwd_out.local);
      UA_CUDA(ua::launch_wait_copy(static_cast<const int64_t*>(ctx->flags.local), kSlotBwdOut, P, step, rout, dq,
                                   int64_t(S), ctx->peer_err, stream));
      UA_CUDA(cudaMemcpyAsync(dk, rout + S, S, cudaMemcpyDeviceToDevice, stream));
      UA_CUDA(cudaMemcpyAsync(dv, rout + 2 * S, S, cudaMemcpyDeviceToDevice, stream));
      ctx->a2a_calls += 1;
      ctx->a2a_bytes += int64_t(P - 1) * int64_t(s.chunk()) * 2 * 3;
    }
    return UA_OK;
  }

  const size_t S = size_t(s.shard()) * 2;
  void* send[4] = {ws + plan.send, ws + plan.send + S, ws + plan.send + 2 * S, ws + plan.send + 3 * S};
  void* recv[4] = {ws + plan.recv, ws + plan.recv + S, ws + plan.recv + 2 * S, ws + plan.recv + 3 * S};
  float* send_delta = reinterpret_cast<float*>(ws + plan.send_delta);
  float* recv_delta = reinterpret_cast<float*>(ws + plan.recv_delta);
  void* grad[3] = {ws + plan.grad, ws + plan.grad + S, ws + plan.grad + 2 * S};
  const void* src[4] = {q, k, v, dout};
  {  // 1. pack q, k, v, dO + Delta = rowsum(dO * O) in sequence space
    Phase ph(ctx, UA_PHASE_PACK_BWD, stream);
    UA_CUDA(ua::launch_pack(src, send, 4, B, s.Nl, H, D, P, dout, out, send_delta, stream));
  }
  {  // 2. all-to-all #3 (fused q, k, v, dO, Delta)
    Phase ph(ctx, UA_PHASE_A2A_BWD_IN, stream);
    UA_NCCL(ncclGroupStart());
    ua_status st = a2a(ctx, send, recv, 4, size_t(s.chunk()), ncclBfloat16, 2, stream);
    if (st != UA_OK) { ncclGroupEnd(); return st; }
    void* sd = send_delta;
    void* rd = recv_delta;
    st = a2a(ctx, &sd, &rd, 1, size_t(s.Nl * B * s.Hl), ncclFloat32, 4, stream);
    if (st != UA_OK) { ncclGroupEnd(); return st; }
    UA_NCCL(ncclGroupEnd());
    ctx->a2a_calls += 1;
  }
  // 3+4. attention backward on the head shard [N][B][Hl][D]; dq, dk, dv into the send layout of #4
  UA_TRY(head_bwd(ctx, recv[0], recv[1], recv[2], recv[3], head_layout(B, s.Hl, D), lse, recv_delta, grad[0], grad[1],
                  grad[2], nullptr, B, N, s.Hl, D, ctx->deterministic, ws + plan.head, stream));
  void* rgrad[3] = {ws + plan.send, ws + plan.send + S, ws + plan.send + 2 * S};
  {  // 4. all-to-all #4 (fused dq, dk, dv) back to the token owners
    Phase ph(ctx, UA_PHASE_A2A_BWD_OUT, stream);
    UA_TRY(a2a(ctx, grad, rgrad, 3, size_t(s.chunk()), ncclBfloat16, 2, stream));
    ctx->a2a_calls += 1;
  }
  {  // 5. unpack -> dq, dk, dv [B][Nl][H][D]
    Phase ph(ctx, UA_PHASE_UNPACK_BWD, stream);
    const void* usrc[3] = {rgrad[0], rgrad[1], rgrad[2]};
    void* udst[3] = {dq, dk, dv};
    UA_CUDA(ua::launch_unpack(usrc, udst, 3, B, s.Nl, H, D, P, stream));
  }
  return UA_OK;
}

// ------------------------------------------------------------ rank-local steps (no communication)
ua_status ua_pack_seq_to_head(const void* const* src, void* const* dst, int ntensors, int64_t B, int64_t N, int H,
                              int D, int P, const void* dout, const void* out, float* delta, ua_stream_t stream) {
  UA_TRY(ua_validate(B, N, H, D, P));
  const bool with_delta = dout || out || delta;
  if (ntensors < 0 || ntensors > 4 || (ntensors == 0 && !with_delta))
    return fail(UA_ERR_INVALID_ARG, "ntensors=%d (0..4; 0 only with Delta)", ntensors);
  if (ntensors > 0 && (!src || !dst)) return fail(UA_ERR_INVALID_ARG, "src / dst arrays are NULL");
  for (int w = 0; w < ntensors; ++w) UA_TRY(check_ptrs({src[w], dst[w]}));
  if (with_delta) UA_TRY(check_ptrs({dout, out, delta}));
  UA_TRY(check_device());
  UA_TRY(check_async(nullptr));
  UA_CUDA(ua::launch_pack(src, dst, ntensors, B, N / P, H, D, P, dout, out, delta,
                          reinterpret_cast<cudaStream_t>(stream)));
  return UA_OK;
}

ua_status ua_unpack_head_to_seq(const void* const* src, void* const* dst, int ntensors, int64_t B, int64_t N, int H,
                                int D, int P, ua_stream_t stream) {
  UA_TRY(ua_validate(B, N, H, D, P));
  if (ntensors < 1 || ntensors > 4 || !src || !dst) return fail(UA_ERR_INVALID_ARG, "ntensors=%d (1..4)", ntensors);
  for (int w = 0; w < ntensors; ++w) UA_TRY(check_ptrs({src[w], dst[w]}));
  UA_TRY(check_device());
  UA_TRY(check_async(nullptr));
  UA_CUDA(ua::launch_unpack(src, dst, ntensors, B, N / P, H, D, P, reinterpret_cast<cudaStream_t>(stream)));
  return UA_OK;
}

ua_status ua_push_seq_to_head(const void* const* src, int ntensors, void* const* dst_rank, int64_t B, int64_t N, int H,
                              int D, int P, int rank, const void* dout, const void* out, ua_stream_t stream) {
  UA_TRY(ua_validate(B, N, H, D, P));
  if (P > ua::kMaxPeers) return fail(UA_ERR_UNSUPPORTED, "P=%d > %d", P, ua::kMaxPeers);
  if (rank < 0 || rank >= P) return fail(UA_ERR_INVALID_ARG, "rank=%d not in [0, %d)", rank, P);
  if (ntensors < 1 || ntensors > 4 || !src || !dst_rank)
    return fail(UA_ERR_INVALID_ARG, "ntensors=%d (1..4)", ntensors);
  if ((dout == nullptr) != (out == nullptr)) return fail(UA_ERR_INVALID_ARG, "dout and out: both or neither");
  ua::PeerPack pk{};
  for (int w = 0; w < ntensors; ++w) {
    UA_TRY(check_ptrs({src[w]}));
    pk.src[w] = src[w];
  }
  for (int j = 0; j < P; ++j) {
    UA_TRY(check_ptrs({dst_rank[j]}));
    pk.dst[j] = dst_rank[j];
  }
  if (dout) UA_TRY(check_ptrs({dout, out}));
  pk.ntensors = ntensors;
  pk.dout = dout;
  pk.out = out;
  UA_TRY(check_device());
  UA_TRY(check_async(nullptr));
  UA_CUDA(ua::launch_pack_push(pk, B, N / P, H, D, P, rank, reinterpret_cast<cudaStream_t>(stream)));
  return UA_OK;
}

namespace {
// Owner maps of the token-owner tensors [B][N/P][H][D] (o_owner[i] = rank i's tensor).
ua_status owner_map(void* const* owners, const Shape& s, int rank, ua::PeerOut* o) {
  if (s.P > ua::kMaxPeers) return fail(UA_ERR_UNSUPPORTED, "P=%d > %d", s.P, ua::kMaxPeers);
  *o = ua::PeerOut{};
  for (int i = 0; i < s.P; ++i) {
    UA_TRY(check_ptrs({owners[i]}));
    o->base[i] = owners[i];
  }
  o->nl = s.Nl;
  o->H = s.H;
  o->h0 = rank * s.Hl;
  return UA_OK;
}
}  // namespace

ua_status ua_head_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t B, int64_t N,
                           int H, int D, int P, int rank, void* const* o_owner, ua_stream_t stream) {
  UA_TRY(ua_validate(B, N, H, D, P));
  if (rank < 0 || rank >= P) return fail(UA_ERR_INVALID_ARG, "rank=%d not in [0, %d)", rank, P);
  UA_TRY(check_ptrs({q, k, v, lse}));
  const Shape s = make_shape(B, N, H, D, P);
  ua::PeerOut po;
  if (o_owner) {
    if (o) return fail(UA_ERR_INVALID_ARG, "o must be NULL when o_owner is given");
    UA_TRY(owner_map(o_owner, s, rank, &po));
  } else {
    UA_TRY(check_ptrs({o}));
  }
  UA_TRY(check_device());
  UA_TRY(check_async(nullptr));
  return head_fwd(nullptr, q, k, v, head_layout(B, s.Hl, D), o, o_owner ? &po : nullptr, lse, B, N, s.Hl, D,
                  reinterpret_cast<cudaStream_t>(stream));
}

ua_status ua_head_attn_bwd_workspace_size(int64_t B, int64_t N, int H, int D, int P, size_t* bytes) {
  UA_TRY(ua_validate(B, N, H, D, P));
  if (!bytes) return fail(UA_ERR_INVALID_ARG, "bytes is NULL");
  *bytes = head_bwd_bytes(make_shape(B, N, H, D, P));
  return UA_OK;
}

ua_status ua_head_attn_bwd(const void* q, const void* k, const void* v, const void* dout, const float* lse,
                           const float* delta, void* dq, void* dk, void* dv, int64_t B, int64_t N, int H, int D, int P,
                           int rank, void* const* owners, int deterministic, void* workspace, size_t workspace_bytes,
                           ua_stream_t stream) {
  UA_TRY(ua_validate(B, N, H, D, P));
  if (rank < 0 || rank >= P) return fail(UA_ERR_INVALID_ARG, "rank=%d not in [0, %d)", rank, P);
  UA_TRY(check_ptrs({q, k, v, dout, lse, delta, workspace}));
  const Shape s = make_shape(B, N, H, D, P);
  if (workspace_bytes < head_bwd_bytes(s))
    return fail(UA_ERR_INVALID_ARG, "workspace too small: need %zu bytes, got %zu", head_bwd_bytes(s),
                workspace_bytes);
  ua::PeerOut po[3];
  if (owners) {
    if (dq || dk || dv) return fail(UA_ERR_INVALID_ARG, "dq, dk, dv must be NULL when owners are given");
    for (int w = 0; w < 3; ++w) UA_TRY(owner_map(owners + w * P, s, rank, &po[w]));
  } else {
    UA_TRY(check_ptrs({dq, dk, dv}));
  }
  UA_TRY(check_device());
  UA_TRY(check_async(nullptr));
  return head_bwd(nullptr, q, k, v, dout, head_layout(B, s.Hl, D), lse, delta, dq, dk, dv, owners ? po : nullptr, B, N,
                  s.Hl, D, deterministic ? 1 : 0, static_cast<char*>(workspace), reinterpret_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------ LSS sequence parallelism
ua_status ua_lss_validate(int64_t B, int64_t N, int H, int D, int P) {
  if (B < 1 || N < 1 || H < 1 || D < 1 || P < 1)
    return fail(UA_ERR_INVALID_ARG, "B, N, H, D, P must be >= 1 (got B=%lld N=%lld H=%d D=%d P=%d)", (long long)B,
                (long long)N, H, D, P);
  if (N % P != 0) return fail(UA_ERR_SEQ_DIVISIBILITY, "LSS needs N %% P == 0 (N=%lld, P=%d)", (long long)N, P);
  if (D != 32 && D != 64 && D != 72 && D != 128)
    return fail(UA_ERR_UNSUPPORTED, "head dim D=%d not in {32, 64, 72, 128}", D);
  if (N >= (int64_t(1) << 31)) return fail(UA_ERR_UNSUPPORTED, "N=%lld >= 2^31", (long long)N);
  if (B * N * H >= (int64_t(1) << 40)) return fail(UA_ERR_UNSUPPORTED, "problem too large");
  return UA_OK;
}

ua_status ua_lss_workspace_size(int64_t B, int64_t N, int H, int D, int P, size_t* fwd_bytes, size_t* bwd_bytes) {
  UA_TRY(ua_lss_validate(B, N, H, D, P));
  const Shape s = make_shape(B, N, H, D, P);
  if (P == 1) {  // plain attention on the whole sequence: the Ulysses P = 1 plan
    if (fwd_bytes) *fwd_bytes = plan_fwd(s).total;
    if (bwd_bytes) *bwd_bytes = plan_bwd(s).total;
    return UA_OK;
  }
  if (fwd_bytes) *fwd_bytes = plan_lss(s, false).total;
  if (bwd_bytes) *bwd_bytes = plan_lss(s, true).total;
  return UA_OK;
}

namespace {
// K, V of every rank into kv_full [2][N][B][H][D]: one fused all-gather (NCCL group of two).
ua_status lss_gather_kv(ua_ctx* ctx, const Shape& s, const void* k, const void* v, char* ws, const LssPlan& plan,
                        int ph_pack, int ph_gather, cudaStream_t stream) {
  const size_t S = size_t(s.shard()) * 2;
  const void* kv_src[2] = {k, v};
  void* kv_send[2] = {ws + plan.kv_send, ws + plan.kv_send + S};
  if (s.B > 1) {  // [B][Nl][H][D] -> [Nl][B][H][D] (pack with one destination)
    Phase ph(ctx, ph_pack, stream);
    UA_CUDA(ua::launch_pack(kv_src, kv_send, 2, s.B, s.Nl, s.H, s.D, 1, nullptr, nullptr, nullptr, stream));
  } else {
    kv_send[0] = const_cast<void*>(k);
    kv_send[1] = const_cast<void*>(v);
  }
  Phase ph(ctx, ph_gather, stream);
  UA_NCCL(ncclGroupStart());
  for (int w = 0; w < 2; ++w) {
    ncclResult_t r = ncclAllGather(kv_send[w], ws + plan.kv_full + size_t(w) * S * s.P, size_t(s.shard()),
                                   ncclBfloat16, ctx->comm, stream);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return fail(UA_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
    }
  }
  UA_NCCL(ncclGroupEnd());
  ctx->a2a_calls += 1;
  ctx->a2a_bytes += int64_t(s.P - 1) * int64_t(S) * 2;
  return UA_OK;
}

// LSS compute of one rank (no communication): its N/P queries of every head over all N keys.
//   q, dout, out [B][Nl][H][D] bf16 (sequence shard); kf, vf [N][B][H][D] bf16 (the gathered keys);
//   lse [B][H][Nl]; dk_part, dv_part fp32 [N][B][H][D] (partial sums over this rank's queries).
ua_status lss_rank_fwd(ua_ctx* ctx, const Shape& s, const void* q, const void* kf, const void* vf, void* out,
                       float* lse, cudaStream_t stream) {
  const int64_t H = s.H, D = s.D;
  const int64_t qsn = H * D, qsh = D, qsb = s.Nl * H * D;
  const Rows qr{q, qsn, qsh, qsb, s.Nl};
  const Rows kvr{nullptr, s.B * H * D, D, H * D, s.N};
  ua::ViewArg o{out, qsn, qsh, qsb};
  Phase ph(ctx, UA_PHASE_ATTN_FWD, stream);
  return launch_attention_fwd(qr, kf, vf, kvr, o, nullptr, 0, 0, 0, lse, s.Nl, H * s.Nl, s.B, s.H, s.D, 0, s.N, stream);
}

ua_status lss_rank_bwd(ua_ctx* ctx, const Shape& s, const void* q, const void* kf, const void* vf, const void* out,
                       const float* lse, const void* dout, void* dq, float* dk_part, float* dv_part, int deterministic,
                       char* ws, cudaStream_t stream) {
  const int64_t H = s.H, D = s.D, Nl = s.Nl;
  const LssRankPlan plan = plan_lss_rank(s);
  const int64_t n_pad = (Nl + 127) / 128 * 128;
  const float scale = float(1.0 / std::sqrt(double(D)));
  float* delta = reinterpret_cast<float*>(ws + plan.delta);
  float* dq_acc = reinterpret_cast<float*>(ws + plan.dq_acc);
  {  // Delta[t][b][h] = sum_d dO.O (fp32), local queries
    Phase ph(ctx, UA_PHASE_PACK_BWD, stream);
    UA_CUDA(ua::launch_pack(nullptr, nullptr, 0, s.B, Nl, s.H, s.D, 1, dout, out, delta, stream));
  }
  const int64_t qsn = H * D, qsh = D, qsb = Nl * H * D;
  const int64_t ksn = s.B * H * D, ksh = D, ksb = H * D;
  {  // local dQ; dK, dV partial sums over the local queries for all N keys (fp32)
    Phase ph(ctx, UA_PHASE_ATTN_BWD, stream);
    UA_CUDA(cudaMemsetAsync(dq_acc, 0, size_t(s.B * H * n_pad * D) * 4, stream));
    const Rows qr{q, qsn, qsh, qsb, Nl};
    const Rows kvr{nullptr, ksn, ksh, ksb, s.N};
    ua::ViewArg vdk{dk_part, ksn, ksh, ksb}, vdv{dv_part, ksn, ksh, ksb};
    UA_TRY(launch_attention_bwd(qr, dout, kf, vf, kvr, vdk, vdv, 1, dq_acc, lse, Nl, H * Nl, delta, s.B * H, 1, s.H,
                                s.B, s.H, s.D, reinterpret_cast<float2*>(ws + plan.lsed), deterministic, stream));
  }
  Phase ph(ctx, UA_PHASE_DQ_FINALIZE, stream);
  ua::ViewArg vdq{dq, qsn, qsh, qsb};
  UA_CUDA(ua::launch_dq_finalize(dq_acc, vdq, s.B, Nl, s.H, s.D, scale, stream));
  return UA_OK;
}

ua_status lss_check_call(ua_ctx* ctx, int64_t B, int64_t N, int H, int D, int P, std::initializer_list<const void*> ptrs,
                         size_t need, void* workspace, size_t workspace_bytes) {
  UA_TRY(ua_lss_validate(B, N, H, D, P));
  if (!ctx) return fail(UA_ERR_INVALID_ARG, "ctx is NULL");
  if (P != ctx->P) return fail(UA_ERR_INVALID_ARG, "P=%d differs from ctx P=%d", P, ctx->P);
  for (const void* ptr : ptrs) {
    if (!ptr) return fail(UA_ERR_INVALID_ARG, "null tensor pointer");
    if (!aligned16(ptr)) return fail(UA_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  }
  if (workspace_bytes < need || (need > 0 && !workspace))
    return fail(UA_ERR_INVALID_ARG, "workspace too small: need %zu bytes, got %zu", need, workspace_bytes);
  UA_TRY(check_device());
  return check_async(ctx);
}
}  // namespace

ua_status ua_lss_attn_fwd(ua_ctx* ctx, const void* q, const void* k, const void* v, void* out, float* lse, int64_t B,
                          int64_t N, int H, int D, int P, void* workspace, size_t workspace_bytes, ua_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const Shape s = make_shape(B, N, H, D, P);
  const LssPlan plan = plan_lss(s, false);
  UA_TRY(lss_check_call(ctx, B, N, H, D, P, {q, k, v, out, lse}, plan.total, workspace, workspace_bytes));
  if (P == 1) return ua_ulysses_attn_fwd(ctx, q, k, v, out, lse, B, N, H, D, 1, workspace, workspace_bytes, stream_);
  char* ws = static_cast<char*>(workspace);
  UA_TRY(lss_gather_kv(ctx, s, k, v, ws, plan, UA_PHASE_PACK_FWD, UA_PHASE_A2A_FWD_IN, stream));
  // exact attention of the local query segment over all N keys, every head
  const size_t S = size_t(s.shard()) * 2;
  return lss_rank_fwd(ctx, s, q, ws + plan.kv_full, ws + plan.kv_full + S * P, out, lse, stream);
}

ua_status ua_lss_attn_bwd(ua_ctx* ctx, const void* q, const void* k, const void* v, const void* out, const float* lse,
                          const void* dout, void* dq, void* dk, void* dv, int64_t B, int64_t N, int H, int D, int P,
                          void* workspace, size_t workspace_bytes, ua_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const Shape s = make_shape(B, N, H, D, P);
  const LssPlan plan = plan_lss(s, true);
  UA_TRY(lss_check_call(ctx, B, N, H, D, P, {q, k, v, out, lse, dout, dq, dk, dv}, plan.total, workspace,
                        workspace_bytes));
  if (P == 1)
    return ua_ulysses_attn_bwd(ctx, q, k, v, out, lse, dout, dq, dk, dv, B, N, H, D, 1, workspace, workspace_bytes,
                               stream_);
  char* ws = static_cast<char*>(workspace);
  const size_t S = size_t(s.shard()) * 2;
  const int64_t Nl = s.Nl;
  UA_TRY(lss_gather_kv(ctx, s, k, v, ws, plan, UA_PHASE_PACK_BWD, UA_PHASE_A2A_BWD_IN, stream));
  float* part = reinterpret_cast<float*>(ws + plan.part);
  float* red = reinterpret_cast<float*>(ws + plan.red);
  const size_t PE = size_t(s.shard()) * s.P;  // elements of one [N][B][H][D] tensor
  UA_TRY(lss_rank_bwd(ctx, s, q, ws + plan.kv_full, ws + plan.kv_full + S * P, out, lse, dout, dq, part, part + PE,
                      ctx->deterministic, ws + plan.rank, stream));
  {  // dK, dV partials summed over ranks into the key owners (one fused reduce-scatter)
    Phase ph(ctx, UA_PHASE_A2A_BWD_OUT, stream);
    UA_NCCL(ncclGroupStart());
    for (int w = 0; w < 2; ++w) {
      ncclResult_t r = ncclReduceScatter(part + w * PE, red + w * size_t(s.shard()), size_t(s.shard()), ncclFloat32,
                                         ncclSum, ctx->comm, stream);
      if (r != ncclSuccess) {
        ncclGroupEnd();
        return fail(UA_ERR_NCCL, "ncclReduceScatter: %s", ncclGetErrorString(r));
      }
    }
    UA_NCCL(ncclGroupEnd());
    ctx->a2a_calls += 1;
    ctx->a2a_bytes += int64_t(s.P - 1) * int64_t(s.shard()) * 4 * 2;
  }
  {  // [Nl][B][H][D] fp32 -> bf16 [B][Nl][H][D]
    Phase ph(ctx, UA_PHASE_UNPACK_BWD, stream);
    void* dsts[2] = {dk, dv};
    for (int w = 0; w < 2; ++w) {
      ua::ViewArg vo{dsts[w], D, Nl * H * D, int64_t(H) * D};
      UA_CUDA(ua::launch_f32_to_view(red + w * size_t(s.shard()), vo, Nl, H, int(B), D, stream));
    }
  }
  return UA_OK;
}

ua_status ua_lss_rank_fwd(const void* q, const void* k_full, const void* v_full, void* out, float* lse, int64_t B,
                          int64_t N, int H, int D, int P, ua_stream_t stream) {
  UA_TRY(ua_lss_validate(B, N, H, D, P));
  UA_TRY(check_ptrs({q, k_full, v_full, out, lse}));
  UA_TRY(check_device());
  UA_TRY(check_async(nullptr));
  return lss_rank_fwd(nullptr, make_shape(B, N, H, D, P), q, k_full, v_full, out, lse,
                      reinterpret_cast<cudaStream_t>(stream));
}

ua_status ua_lss_rank_bwd_workspace_size(int64_t B, int64_t N, int H, int D, int P, size_t* bytes) {
  UA_TRY(ua_lss_validate(B, N, H, D, P));
  if (!bytes) return fail(UA_ERR_INVALID_ARG, "bytes is NULL");
  *bytes = plan_lss_rank(make_shape(B, N, H, D, P)).total;
  return UA_OK;
}

ua_status ua_lss_rank_bwd(const void* q, const void* k_full, const void* v_full, const void* out, const float* lse,
                          const void* dout, void* dq, float* dk_part, float* dv_part, int64_t B, int64_t N, int H,
                          int D, int P, int deterministic, void* workspace, size_t workspace_bytes,
                          ua_stream_t stream) {
  UA_TRY(ua_lss_validate(B, N, H, D, P));
  UA_TRY(check_ptrs({q, k_full, v_full, out, lse, dout, dq, dk_part, dv_part, workspace}));
  const Shape s = make_shape(B, N, H, D, P);
  if (workspace_bytes < plan_lss_rank(s).total)
    return fail(UA_ERR_INVALID_ARG, "workspace too small: need %zu bytes, got %zu", plan_lss_rank(s).total,
                workspace_bytes);
  UA_TRY(check_device());
  UA_TRY(check_async(nullptr));
  return lss_rank_bwd(nullptr, s, q, k_full, v_full, out, lse, dout, dq, dk_part, dv_part, deterministic ? 1 : 0,
                      static_cast<char*>(workspace), reinterpret_cast<cudaStream_t>(stream));
}

ua_status ua_ctx_enable_timing(ua_ctx* ctx, int enable) {
  if (!ctx) return fail(UA_ERR_INVALID_ARG, "ctx is NULL");
  ctx->timing = enable != 0;
  return UA_OK;
}

ua_status ua_ctx_phase_times(ua_ctx* ctx, double* ms, int64_t* launches) {
  if (!ctx) return fail(UA_ERR_INVALID_ARG, "ctx is NULL");
  for (auto& r : ctx->pending) {
    UA_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    UA_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    if (ms) ms[r.phase] += double(t);
    if (launches) launches[r.phase] += 1;
    ctx->pool.push_back(r.a);
    ctx->pool.push_back(r.b);
  }
  ctx->pending.clear();
  return UA_OK;
}

ua_status ua_attn_fwd_segment(const void* q, const void* k, const void* v, float* o_seg, float* lse_seg, int64_t B,
                              int64_t N, int Hx, int D, int64_t kv_begin, int64_t kv_end, ua_stream_t stream_) {
  UA_TRY(ua_validate(B, N, Hx, D, 1));
  if (!q || !k || !v || !o_seg || !lse_seg) return fail(UA_ERR_INVALID_ARG, "null tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o_seg) || !aligned16(lse_seg))
    return fail(UA_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  if (kv_begin < 0 || kv_begin % 128 != 0 || kv_end <= kv_begin || kv_end > N)
    return fail(UA_ERR_INVALID_ARG, "bad key segment [%lld, %lld) for N=%lld", (long long)kv_begin,
                (long long)kv_end, (long long)N);
  UA_TRY(check_device());
  UA_TRY(check_async(nullptr));
  const int64_t sn = int64_t(Hx) * D, sh = D, sb = N * Hx * D;
  ua::ViewArg o{nullptr, 0, 0, 0};
  return launch_attention_fwd(q, k, v, sn, sh, sb, o, o_seg, D, N * D, int64_t(Hx) * N * D, lse_seg, N,
                              int64_t(Hx) * N, B, N, Hx, D, kv_begin, kv_end, reinterpret_cast<cudaStream_t>(stream_));
}

ua_status ua_lse_merge(float* o_a, float* lse_a, const float* o_b, const float* lse_b, int64_t rows, int D,
                       ua_stream_t stream_) {
  if (!o_a || !lse_a || !o_b || !lse_b || rows < 1 || D < 1) return fail(UA_ERR_INVALID_ARG, "bad lse_merge args");
  UA_TRY(check_device());
  UA_CUDA(ua::launch_lse_merge(o_a, lse_a, o_b, lse_b, rows, D, reinterpret_cast<cudaStream_t>(stream_)));
  return UA_OK;
}

ua_status ua_f32_to_bf16_bnhd(const float* src, void* dst, int64_t B, int64_t N, int Hx, int D, ua_stream_t stream_) {
  UA_TRY(ua_validate(B, N, Hx, D, 1));
  if (!src || !dst || !aligned16(src) || !aligned16(dst)) return fail(UA_ERR_INVALID_ARG, "bad pointers");
  UA_TRY(check_device());
  ua::ViewArg v{dst, int64_t(Hx) * D, D, N * Hx * D};
  UA_CUDA(ua::launch_f32_to_view(src, v, B, N, Hx, D, reinterpret_cast<cudaStream_t>(stream_)));
  return UA_OK;
}

}  // extern "C"
