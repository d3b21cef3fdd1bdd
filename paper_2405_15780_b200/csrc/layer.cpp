// layer.cpp — the rest of the attention layer around the Ulysses attention
// (SURVEY §8(f)-3): Q/K/V and output projections and the SP group's
// weight-gradient all-reduce (§5.4, §6.1: "two all-to-all
// calls in the forward pass and two all-to-all calls + all reduce in the
// backward pass per layer").
//
// The projections are dense GEMMs (bf16 operands, fp32 accumulation) on this
// library's own tcgen05 GEMM kernel (kernels/gemm.cu); the attention in between
// is the Ulysses path.  Row-major shapes, M = B * N/P tokens of this rank, E = H * D:
//   forward   q = x Wq^T, k = x Wk^T, v = x Wv^T    ([M][E] each; W_qkv = [Wq; Wk; Wv], [3E][E])
//             o = UlyssesAttention(q, k, v)
//             y = o Wo^T                             (Wo [E][E])
//   backward  do = dy Wo,  dWo = dy^T o
//             (dq, dk, dv) = UlyssesAttentionBackward(q, k, v, o, lse, do)
//             dx = dq Wq + dk Wk + dv Wv   (one GEMM over three K segments: fp32 accumulate, one bf16 rounding)
//             dW_qkv = [dq^T x; dk^T x; dv^T x]
//             dW_qkv, dWo summed over the P ranks of the SP group (one fused NCCL all-reduce, fp32)
#include <cstdint>
#include <cstring>
#include <initializer_list>

#include "capi_internal.h"
#include "tma_host.h"

namespace {

using ua_internal::fail;

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct LayerPlan {
  // saved (caller-owned, forward -> backward): q, k, v, o bf16 [M][E]; lse fp32 [B][H/P][N]
  size_t s_q = 0, s_k = 0, s_v = 0, s_o = 0, s_lse = 0, saved = 0;
  // forward workspace: the attention forward's workspace
  size_t f_attn = 0, fwd = 0;
  // backward workspace: do, dq, dk, dv bf16 [M][E], attention bwd ws
  size_t b_do = 0, b_dq = 0, b_dk = 0, b_dv = 0, b_attn = 0, bwd = 0;
  size_t attn_fwd = 0, attn_bwd = 0;
};

ua_status plan_layer(int64_t B, int64_t N, int H, int D, int P, LayerPlan* pl) {
  UA_TRY(ua_validate(B, N, H, D, P));
  size_t af = 0, ab = 0;
  UA_TRY(ua_workspace_size(B, N, H, D, P, &af, &ab));
  const size_t M = size_t(B) * size_t(N / P), E = size_t(H) * D;
  const size_t T = M * E * 2;  // one bf16 [M][E] tensor
  LayerPlan p;
  p.s_q = 0;
  p.s_k = align_up(p.s_q + T);
  p.s_v = align_up(p.s_k + T);
  p.s_o = align_up(p.s_v + T);
  p.s_lse = align_up(p.s_o + T);
  p.saved = align_up(p.s_lse + size_t(B) * size_t(H / P) * size_t(N) * 4);
  p.f_attn = 0;
  p.fwd = align_up(p.f_attn + af);
  p.b_do = 0;
  p.b_dq = align_up(p.b_do + T);
  p.b_dk = align_up(p.b_dq + T);
  p.b_dv = align_up(p.b_dk + T);
  p.b_attn = align_up(p.b_dv + T);
  p.bwd = align_up(p.b_attn + ab);
  p.attn_fwd = af;
  p.attn_bwd = ab;
  *pl = p;
  return UA_OK;
}

// Row-major C[M][N] = sum_s op(A_s) op(B_s) on the tcgen05 GEMM (kernels/gemm.cu):
// a_mn: A_s stored [K][M] (op = transpose), else [M][K]; b_mn: B_s stored [K][N],
// else [N][K] (op = transpose).  C bf16 or fp32 with leading dimension N.
ua_status gemm(bool a_mn, bool b_mn, int64_t M, int64_t N, int64_t K, std::initializer_list<const void*> As,
               std::initializer_list<const void*> Bs, void* C, bool c_f32, cudaStream_t stream) {
  if (As.size() != Bs.size() || As.size() < 1 || As.size() > size_t(ua::kGemmMaxSeg))
    return fail(UA_ERR_INVALID_ARG, "gemm: %zu A / %zu B segments", As.size(), Bs.size());
  if (M < 1 || N < 1 || K < 1) return fail(UA_ERR_INVALID_ARG, "gemm: M, N, K must be >= 1");
  if ((a_mn ? M : K) % 8 != 0 || (b_mn ? N : K) % 8 != 0)
    return fail(UA_ERR_INVALID_ARG, "gemm: operand rows must be 16-byte multiples (leading dims %% 8)");
  for (const void* a : As)
    if (!a || (reinterpret_cast<uintptr_t>(a) & 15u)) return fail(UA_ERR_INVALID_ARG, "gemm: bad A pointer");
  for (const void* b : Bs)
    if (!b || (reinterpret_cast<uintptr_t>(b) & 15u)) return fail(UA_ERR_INVALID_ARG, "gemm: bad B pointer");
  if (!C || (reinterpret_cast<uintptr_t>(C) & 15u) || (N * (c_f32 ? 4 : 2)) % 16 != 0)
    return fail(UA_ERR_INVALID_ARG, "gemm: bad C pointer or row size");
  if (M >= (int64_t(1) << 31) || N >= (int64_t(1) << 31) || K >= (int64_t(1) << 31))
    return fail(UA_ERR_UNSUPPORTED, "gemm: dimension >= 2^31");
  ua::GemmParams p;
  std::memset(&p, 0, sizeof(p));
  const uint32_t bn = uint32_t(ua::gemm_bn(int(N)));
  int s = 0;
  for (const void* a : As) {
    const bool ok = a_mn ? ua::make_tmap_bf16_2d(&p.tm_a[s], a, uint64_t(M), uint64_t(K), uint64_t(M), 64, 64)
                         : ua::make_tmap_bf16_2d(&p.tm_a[s], a, uint64_t(K), uint64_t(M), uint64_t(K), 64, 128);
    if (!ok) return fail(UA_ERR_CUDA, "cuTensorMapEncodeTiled failed (gemm A, %lldx%lld)", (long long)M, (long long)K);
    ++s;
  }
  s = 0;
  for (const void* b : Bs) {
    const bool ok = b_mn ? ua::make_tmap_bf16_2d(&p.tm_b[s], b, uint64_t(N), uint64_t(K), uint64_t(N), 64, 64)
                         : ua::make_tmap_bf16_2d(&p.tm_b[s], b, uint64_t(K), uint64_t(N), uint64_t(K), 64, bn);
    if (!ok) return fail(UA_ERR_CUDA, "cuTensorMapEncodeTiled failed (gemm B, %lldx%lld)", (long long)N, (long long)K);
    ++s;
  }
  p.c = C;
  p.ldc = N;
  p.c_f32 = c_f32 ? 1 : 0;
  p.M = int(M);
  p.N = int(N);
  p.K = int(K);
  p.nseg = int(As.size());
  p.a_mn = a_mn;
  p.b_mn = b_mn;
  UA_TRY(ua_internal::check_device());
  UA_CUDA(ua::launch_gemm(p, stream));
  return UA_OK;
}

ua_status check_layer_args(ua_ctx* ctx, int P, std::initializer_list<const void*> ptrs) {
  if (!ctx) return fail(UA_ERR_INVALID_ARG, "ctx is NULL");
  if (P != ctx->P) return fail(UA_ERR_INVALID_ARG, "P=%d differs from ctx P=%d", P, ctx->P);
  for (const void* p : ptrs) {
    if (!p) return fail(UA_ERR_INVALID_ARG, "null tensor pointer");
    if ((reinterpret_cast<uintptr_t>(p) & 15u) != 0) return fail(UA_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  }
  return UA_OK;
}

}  // namespace

namespace ua_internal {
void layer_release(ua_ctx*) {}  // the projections hold no library handles
}  // namespace ua_internal

extern "C" {

ua_status ua_layer_sizes(int64_t B, int64_t N, int H, int D, int P, size_t* saved_bytes, size_t* fwd_bytes,
                         size_t* bwd_bytes) {
  LayerPlan pl;
  UA_TRY(plan_layer(B, N, H, D, P, &pl));
  if (saved_bytes) *saved_bytes = pl.saved;
  if (fwd_bytes) *fwd_bytes = pl.fwd;
  if (bwd_bytes) *bwd_bytes = pl.bwd;
  return UA_OK;
}

ua_status ua_layer_fwd(ua_ctx* ctx, const void* x, const void* w_qkv, const void* w_o, void* y, void* saved,
                       int64_t B, int64_t N, int H, int D, int P, void* workspace, size_t workspace_bytes,
                       ua_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  LayerPlan pl;
  UA_TRY(plan_layer(B, N, H, D, P, &pl));
  UA_TRY(check_layer_args(ctx, P, {x, w_qkv, w_o, y, saved, workspace}));
  if (workspace_bytes < pl.fwd) return fail(UA_ERR_INVALID_ARG, "workspace too small: need %zu bytes, got %zu", pl.fwd, workspace_bytes);
  const int64_t M = B * (N / P), E = int64_t(H) * D;
  char* sv = static_cast<char*>(saved);
  char* ws = static_cast<char*>(workspace);
  void* q = sv + pl.s_q;
  void* k = sv + pl.s_k;
  void* v = sv + pl.s_v;
  void* o = sv + pl.s_o;
  float* lse = reinterpret_cast<float*>(sv + pl.s_lse);
  const char* w = static_cast<const char*>(w_qkv);
  const size_t WE = size_t(E) * E * 2;  // bytes of one [E][E] bf16 block of W_qkv
  void* qkv[3] = {q, k, v};
  for (int i = 0; i < 3; ++i)  // q = x Wq^T, k = x Wk^T, v = x Wv^T
    UA_TRY(gemm(false, false, M, E, E, {x}, {w + i * WE}, qkv[i], false, stream));
  UA_TRY(ua_ulysses_attn_fwd(ctx, q, k, v, o, lse, B, N, H, D, P, ws + pl.f_attn, pl.attn_fwd, stream_));
  return gemm(false, false, M, E, E, {o}, {w_o}, y, false, stream);
}

ua_status ua_layer_bwd(ua_ctx* ctx, const void* x, const void* w_qkv, const void* w_o, const void* saved,
                       const void* dy, void* dx, float* dw_qkv, float* dw_o, int64_t B, int64_t N, int H, int D, int P,
                       void* workspace, size_t workspace_bytes, ua_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  LayerPlan pl;
  UA_TRY(plan_layer(B, N, H, D, P, &pl));
  UA_TRY(check_layer_args(ctx, P, {x, w_qkv, w_o, saved, dy, dx, dw_qkv, dw_o, workspace}));
  if (workspace_bytes < pl.bwd) return fail(UA_ERR_INVALID_ARG, "workspace too small: need %zu bytes, got %zu", pl.bwd, workspace_bytes);
  const int64_t M = B * (N / P), E = int64_t(H) * D;
  const char* sv = static_cast<const char*>(saved);
  char* ws = static_cast<char*>(workspace);
  const void* q = sv + pl.s_q;
  const void* k = sv + pl.s_k;
  const void* v = sv + pl.s_v;
  const void* o = sv + pl.s_o;
  const float* lse = reinterpret_cast<const float*>(sv + pl.s_lse);
  void* dout = ws + pl.b_do;
  void* dq = ws + pl.b_dq;
  void* dk = ws + pl.b_dk;
  void* dv = ws + pl.b_dv;
  const char* w = static_cast<const char*>(w_qkv);
  const size_t WE = size_t(E) * E * 2;
  // output projection: do = dy Wo, dWo = dy^T o (this rank's tokens)
  UA_TRY(gemm(false, true, M, E, E, {dy}, {w_o}, dout, false, stream));
  UA_TRY(gemm(true, true, E, E, M, {dy}, {o}, dw_o, true, stream));
  // attention backward (two all-to-alls inside)
  UA_TRY(ua_ulysses_attn_bwd(ctx, q, k, v, o, lse, dout, dq, dk, dv, B, N, H, D, P, ws + pl.b_attn, pl.attn_bwd,
                             stream_));
  // input projections: dx = sum_i dqkv_i W_i (three K segments, one rounding), dW_i = dqkv_i^T x
  UA_TRY(gemm(false, true, M, E, E, {dq, dk, dv}, {w, w + WE, w + 2 * WE}, dx, false, stream));
  const void* g[3] = {dq, dk, dv};
  for (int i = 0; i < 3; ++i) UA_TRY(gemm(true, true, E, E, M, {g[i]}, {x}, dw_qkv + size_t(i) * E * E, true, stream));
  if (P > 1) {  // the SP group's weight-gradient all-reduce, one fused call
    UA_NCCL(ncclGroupStart());
    ncclResult_t r1 = ncclAllReduce(dw_qkv, dw_qkv, size_t(3) * E * E, ncclFloat32, ncclSum, ctx->comm, stream);
    ncclResult_t r2 = ncclAllReduce(dw_o, dw_o, size_t(E) * E, ncclFloat32, ncclSum, ctx->comm, stream);
    UA_NCCL(ncclGroupEnd());
    if (r1 != ncclSuccess || r2 != ncclSuccess)
      return fail(UA_ERR_NCCL, "ncclAllReduce: %s", ncclGetErrorString(r1 != ncclSuccess ? r1 : r2));
    ctx->a2a_calls += 1;
    ctx->a2a_bytes += int64_t(2) * (P - 1) * int64_t(4) * E * E * 4 / P;  // ring all-reduce bytes sent per rank
  }
  return UA_OK;
}

ua_status ua_gemm_bf16(int a_mn, int b_mn, int64_t M, int64_t N, int64_t K, const void* const* A,
                       const void* const* Bm, int nseg, void* C, int c_f32, ua_stream_t stream) {
  if (!A || !Bm || nseg < 1 || nseg > ua::kGemmMaxSeg) return fail(UA_ERR_INVALID_ARG, "gemm: nseg=%d", nseg);
  const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (nseg) {
    case 1: return gemm(a_mn != 0, b_mn != 0, M, N, K, {A[0]}, {Bm[0]}, C, c_f32 != 0, st);
    case 2: return gemm(a_mn != 0, b_mn != 0, M, N, K, {A[0], A[1]}, {Bm[0], Bm[1]}, C, c_f32 != 0, st);
    default: return gemm(a_mn != 0, b_mn != 0, M, N, K, {A[0], A[1], A[2]}, {Bm[0], Bm[1], Bm[2]}, C, c_f32 != 0, st);
  }
}

}  // extern "C"
