// layer.cpp — the rest of the attention layer around the Ulysses attention
// (SURVEY §8(f)-3): Q/K/V and output projections and the SP group's
// weight-gradient all-reduce (§5.4, §6.1: "two all-to-all
// calls in the forward pass and two all-to-all calls + all reduce in the
// backward pass per layer").
//
// The projections are plain dense GEMMs (bf16 operands, fp32 accumulation), so
// they run on cuBLASLt (the same library copy torch loads); the attention in
// between is this library's Ulysses path.  Row-major shapes, M = B * N/P tokens
// of this rank, E = H * D:
//   forward   q = x Wq^T, k = x Wk^T, v = x Wv^T    ([M][E] each; W_qkv = [Wq; Wk; Wv], [3E][E])
//             o = UlyssesAttention(q, k, v)
//             y = o Wo^T                             (Wo [E][E])
//   backward  do = dy Wo,  dWo = dy^T o
//             (dq, dk, dv) = UlyssesAttentionBackward(q, k, v, o, lse, do)
//             dx = dq Wq + dk Wk + dv Wv   (fp32 accumulate, one bf16 rounding)
//             dW_qkv = [dq^T x; dk^T x; dv^T x]
//             dW_qkv, dWo summed over the P ranks of the SP group (one fused NCCL all-reduce, fp32)
#include <cublasLt.h>

#include <cstdint>
#include <cstring>
#include <initializer_list>

#include "capi_internal.h"

namespace {

using ua_internal::fail;

#define UA_LT(expr)                                                                  \
  do {                                                                               \
    cublasStatus_t st_ = (expr);                                                     \
    if (st_ != CUBLAS_STATUS_SUCCESS) return fail(UA_ERR_CUDA, "%s: cublasLt status %d", #expr, int(st_)); \
  } while (0)

constexpr size_t kAlign = 256;
constexpr size_t kLtWorkspace = size_t(32) << 20;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct LayerPlan {
  // saved (caller-owned, forward -> backward): q, k, v, o bf16 [M][E]; lse fp32 [B][H/P][N]
  size_t s_q = 0, s_k = 0, s_v = 0, s_o = 0, s_lse = 0, saved = 0;
  // forward workspace: cuBLASLt scratch + the attention forward's workspace
  size_t f_lt = 0, f_attn = 0, fwd = 0;
  // backward workspace: cuBLASLt scratch, do, dq, dk, dv bf16 [M][E], dx fp32 [M][E], attention bwd ws
  size_t b_lt = 0, b_do = 0, b_dq = 0, b_dk = 0, b_dv = 0, b_dx = 0, b_attn = 0, bwd = 0;
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
  p.f_lt = 0;
  p.f_attn = align_up(kLtWorkspace);
  p.fwd = align_up(p.f_attn + af);
  p.b_lt = 0;
  p.b_do = align_up(kLtWorkspace);
  p.b_dq = align_up(p.b_do + T);
  p.b_dk = align_up(p.b_dq + T);
  p.b_dv = align_up(p.b_dk + T);
  p.b_dx = align_up(p.b_dv + T);
  p.b_attn = align_up(p.b_dx + 2 * T);
  p.bwd = align_up(p.b_attn + ab);
  p.attn_fwd = af;
  p.attn_bwd = ab;
  *pl = p;
  return UA_OK;
}

ua_status lt_handle(ua_ctx* ctx, cublasLtHandle_t* h) {
  if (!ctx->lt) {
    cublasLtHandle_t lt = nullptr;
    UA_LT(cublasLtCreate(&lt));
    ctx->lt = lt;
  }
  *h = static_cast<cublasLtHandle_t>(ctx->lt);
  return UA_OK;
}

// Row-major C[M][N] = op(A) op(B) + beta C with op(A) [M][K], op(B) [K][N]; A, B bf16,
// fp32 accumulation, C bf16 or fp32.  ta: A is stored [K][M]; tb: B is stored [N][K].
// cuBLASLt is column-major, so this issues C^T = op(B)^T op(A)^T.
ua_status gemm_rm(cublasLtHandle_t lt, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const void* A,
                  const void* Bm, void* C, cudaDataType_t ctype, float beta, void* ws, size_t ws_bytes,
                  cudaStream_t stream) {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  ua_status st = UA_OK;
  auto done = [&](ua_status s) {
    if (pref) cublasLtMatmulPreferenceDestroy(pref);
    if (lc) cublasLtMatrixLayoutDestroy(lc);
    if (lb) cublasLtMatrixLayoutDestroy(lb);
    if (la) cublasLtMatrixLayoutDestroy(la);
    if (op) cublasLtMatmulDescDestroy(op);
    return s;
  };
#define UA_LT_OR(expr)                                                                             \
  do {                                                                                             \
    cublasStatus_t s_ = (expr);                                                                    \
    if (s_ != CUBLAS_STATUS_SUCCESS) return done(fail(UA_ERR_CUDA, "%s: cublasLt status %d", #expr, int(s_))); \
  } while (0)
  const cublasOperation_t opa = tb ? CUBLAS_OP_T : CUBLAS_OP_N;  // column-major first operand = B storage
  const cublasOperation_t opb = ta ? CUBLAS_OP_T : CUBLAS_OP_N;  // column-major second operand = A storage
  UA_LT_OR(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  UA_LT_OR(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &opa, sizeof(opa)));
  UA_LT_OR(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &opb, sizeof(opb)));
  // first operand (B storage): op N -> [N rows][K cols] ld N; op T -> stored [K][N] col-major, ld K
  UA_LT_OR(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, tb ? K : N, tb ? N : K, tb ? K : N));
  // second operand (A storage): op N -> [K][M] ld K; op T -> stored [M][K] col-major, ld M
  UA_LT_OR(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, ta ? M : K, ta ? K : M, ta ? M : K));
  UA_LT_OR(cublasLtMatrixLayoutCreate(&lc, ctype, N, M, N));
  UA_LT_OR(cublasLtMatmulPreferenceCreate(&pref));
  UA_LT_OR(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes,
                                                sizeof(ws_bytes)));
  cublasLtMatmulHeuristicResult_t heur;
  int found = 0;
  UA_LT_OR(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 1, &heur, &found));
  if (found == 0) return done(fail(UA_ERR_UNSUPPORTED, "cublasLt: no algorithm for %lldx%lldx%lld", (long long)M,
                                   (long long)N, (long long)K));
  const float alpha = 1.f;
  UA_LT_OR(cublasLtMatmul(lt, op, &alpha, Bm, la, A, lb, &beta, C, lc, C, lc, &heur.algo, ws, ws_bytes, stream));
#undef UA_LT_OR
  return done(st);
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
void layer_release(ua_ctx* ctx) {
  if (ctx && ctx->lt) {
    cublasLtDestroy(static_cast<cublasLtHandle_t>(ctx->lt));
    ctx->lt = nullptr;
  }
}
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
  cublasLtHandle_t lt;
  UA_TRY(lt_handle(ctx, &lt));
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
    UA_TRY(gemm_rm(lt, false, true, M, E, E, x, w + i * WE, qkv[i], CUDA_R_16BF, 0.f, ws + pl.f_lt, kLtWorkspace,
                   stream));
  UA_TRY(ua_ulysses_attn_fwd(ctx, q, k, v, o, lse, B, N, H, D, P, ws + pl.f_attn, pl.attn_fwd, stream_));
  return gemm_rm(lt, false, true, M, E, E, o, w_o, y, CUDA_R_16BF, 0.f, ws + pl.f_lt, kLtWorkspace, stream);
}

ua_status ua_layer_bwd(ua_ctx* ctx, const void* x, const void* w_qkv, const void* w_o, const void* saved,
                       const void* dy, void* dx, float* dw_qkv, float* dw_o, int64_t B, int64_t N, int H, int D, int P,
                       void* workspace, size_t workspace_bytes, ua_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  LayerPlan pl;
  UA_TRY(plan_layer(B, N, H, D, P, &pl));
  UA_TRY(check_layer_args(ctx, P, {x, w_qkv, w_o, saved, dy, dx, dw_qkv, dw_o, workspace}));
  if (workspace_bytes < pl.bwd) return fail(UA_ERR_INVALID_ARG, "workspace too small: need %zu bytes, got %zu", pl.bwd, workspace_bytes);
  cublasLtHandle_t lt;
  UA_TRY(lt_handle(ctx, &lt));
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
  float* dx32 = reinterpret_cast<float*>(ws + pl.b_dx);
  void* ltws = ws + pl.b_lt;
  const char* w = static_cast<const char*>(w_qkv);
  const size_t WE = size_t(E) * E * 2;
  // output projection: do = dy Wo, dWo = dy^T o (this rank's tokens)
  UA_TRY(gemm_rm(lt, false, false, M, E, E, dy, w_o, dout, CUDA_R_16BF, 0.f, ltws, kLtWorkspace, stream));
  UA_TRY(gemm_rm(lt, true, false, E, E, M, dy, o, dw_o, CUDA_R_32F, 0.f, ltws, kLtWorkspace, stream));
  // attention backward (two all-to-alls inside)
  UA_TRY(ua_ulysses_attn_bwd(ctx, q, k, v, o, lse, dout, dq, dk, dv, B, N, H, D, P, ws + pl.b_attn, pl.attn_bwd,
                             stream_));
  // input projections: dx = sum_i dqkv_i W_i (fp32), dW_i = dqkv_i^T x
  const void* g[3] = {dq, dk, dv};
  for (int i = 0; i < 3; ++i) {
    UA_TRY(gemm_rm(lt, false, false, M, E, E, g[i], w + i * WE, dx32, CUDA_R_32F, i == 0 ? 0.f : 1.f, ltws,
                   kLtWorkspace, stream));
    UA_TRY(gemm_rm(lt, true, false, E, E, M, g[i], x, dw_qkv + size_t(i) * E * E, CUDA_R_32F, 0.f, ltws,
                   kLtWorkspace, stream));
  }
  ua::ViewArg vdx{dx, E, 0, 0};
  UA_CUDA(ua::launch_f32_to_view(dx32, vdx, 1, M, 1, int(E), stream));
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

}  // extern "C"
