// attn_kernels.h — internal (C++) launch interface of the CUDA kernels.  Not
// part of the C ABI; csrc/capi.cpp is the only caller.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ua {

struct ViewArg {
  void* base;
  int64_t sn, sh, sb;  // element strides of token, head, batch (d contiguous)
};

// ---- NVLink peer-store all-to-all (peer.cu) -----------------------------------
constexpr int kMaxPeers = 8;
// Token-owner output buffers: rank k's base[k] is a [B][nl][H][D] bf16 tensor
// (CUDA IPC mapping); a head-shard row (b, global token n, local head h) goes to
// base[n / nl] at ((b*nl + n % nl)*H + h0 + h)*D.  base[0] == nullptr: unused.
struct PeerOut {
  void* base[kMaxPeers];
  int64_t nl;
  int H;
  int h0;
};
struct PeerPack {
  const void* src[4];     // local shards [B][Nl][H][D]
  void* dst[kMaxPeers];   // each rank's receive buffer: [ntensors][N][B][Hl][D] (+ Delta [N][B][Hl] fp32)
  int ntensors;
  const void* dout;       // non-null: also push Delta = rowsum(dout * out)
  const void* out;
};
struct PeerFlags {
  int64_t* peer[kMaxPeers];  // every rank's flag array [4 slots][kMaxPeers]
};

struct alignas(64) FwdParams {
  CUtensorMap tm_q;  // 4-D maps {D, N, heads, B} over the Q / K / V views
  CUtensorMap tm_k;
  CUtensorMap tm_v;
  ViewArg o;          // bf16 output (used when o_f32 == nullptr and o_peer.base[0] == nullptr)
  PeerOut o_peer;     // peer mode: O rows straight into the token owner's buffer
  float* o_f32;       // optional fp32 normalised output (LSS segments)
  int64_t of_sn, of_sh, of_sb;
  float* lse;         // lse[b*l_sb + h*l_sh + n]
  int64_t l_sh, l_sb;
  int n_q;            // number of query rows
  int kv_begin, kv_end;  // key range; kv_begin % 128 == 0
  float scale_log2;   // log2(e) / sqrt(D)
  int d_io;           // head dim of the I/O tensors (72 runs in the D = 80 kernel; else == D)
};

struct alignas(64) BwdParams {
  CUtensorMap tm_q;   // {D, N, heads, B}
  CUtensorMap tm_k;
  CUtensorMap tm_v;
  CUtensorMap tm_do;
  CUtensorMap tm_dq;  // fp32 2-D {D, B*heads*N_pad} over dq_acc, box {32, 128}, SW128 (reduce-add target)
  CUtensorMap tm_qh;  // Q / dO with 64-row boxes (half-tile ring of the ws kernel)
  CUtensorMap tm_doh;
  ViewArg dk, dv;     // bf16 outputs (used when dk_peer.base[0] == nullptr)
  PeerOut dk_peer, dv_peer;  // peer mode: dK, dV rows straight into the token owner's buffers
  float* dq_acc;      // fp32 [B*heads][N_pad][D] accumulator, N_pad = ceil(N/128)*128 (zeroed by caller)
  const float* lse;   // lse[b*l_sb + h*l_sh + n]
  int64_t l_sh, l_sb;
  const float* delta; // Delta[b*d_sb + h*d_sh + n*d_sn]
  int64_t d_sn, d_sh, d_sb;
  const float2* lsed; // per head, per 128-row tile: [128 x -lse*log2(e)][128 x -Delta]; rows >= N: (-inf, 0)
  int n;              // number of queries (rows of Q, dO, lse, Delta, dq_acc)
  int n_kv;           // number of keys (rows of K, V, dK, dV); == n except for LSS (local queries, all keys)
  int kv_f32;         // 1: dk / dv views are fp32 (unrounded partial sums, LSS reduce-scatter input)
  int heads;
  int batch;
  float scale;        // 1/sqrt(D)
  float scale_log2;   // log2(e)/sqrt(D)
  int d_io;           // head dim of the I/O tensors and of dq_acc rows (72 runs in the D = 80 kernel)
  int deterministic;  // 1: dQ by the query-stationary kernel, stored (not reduce-added) into dq_acc
};

// Launch setup that is correct in a process driving several GPUs: the dynamic
// shared-memory opt-in is a per-device function attribute, so launchers set it
// on every launch (a cheap driver call) instead of caching it process-wide, and
// persistent grids are sized from the current device's SM count.
template <class Kernel>
inline cudaError_t set_max_smem(Kernel kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
inline int current_num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  return n;
}

cudaError_t launch_attn_fwd(const FwdParams& p, int D, int B, int heads, cudaStream_t stream);

// ---- projection GEMMs of the attention layer (gemm.cu) ---------------------------
// C[M][N] = sum_{s < nseg} op(A_s) op(B_s), bf16 operands, fp32 accumulation.
// tm_a[s]: a_mn ? A stored [K][M] (2-D map {M, K}, box {64, 64})
//               : A stored [M][K] (map {K, M}, box {64, 128});
// tm_b[s]: b_mn ? B stored [K][N] (map {N, K}, box {64, 64})
//               : B stored [N][K] (map {K, N}, box {64, gemm_bn(N)}); all SWIZZLE_128B.
constexpr int kGemmMaxSeg = 3;
struct alignas(64) GemmParams {
  CUtensorMap tm_a[kGemmMaxSeg];
  CUtensorMap tm_b[kGemmMaxSeg];
  void* c;          // row-major [M][ldc], bf16 (c_f32 == 0) or fp32
  int64_t ldc;
  int c_f32;
  int M, N, K;      // K per segment
  int nseg;
  bool a_mn, b_mn;
};
int gemm_bn(int N);   // CTA tile width used for N (the K-major B map's box rows)
cudaError_t launch_gemm(const GemmParams& p, cudaStream_t stream);
// D <= 64 column-split forward (attn_fwd_split.cu); launch_attn_fwd dispatches to it when enabled.
cudaError_t launch_attn_fwd_split(const FwdParams& p, int D, int B, int heads, cudaStream_t stream);
// The backward (attn_bwd_ws.cu): persistent KV-stationary kernel (+ the query-stationary dQ kernel
// in deterministic mode).
cudaError_t launch_attn_bwd_ws(const BwdParams& p, int D, cudaStream_t stream);
// Deterministic dQ (attn_bwd_dq.cu): query-stationary, dq_acc rows = sum_j dS_ij k_j (unscaled, fp32,
// plain stores, fixed key order).  Called by launch_attn_bwd_ws when p.deterministic.
cudaError_t launch_attn_bwd_dq(const BwdParams& p, int D, cudaStream_t stream);

// ---- layout / elementwise kernels (layout.cu) --------------------------------
// Sequence shard -> per-destination send chunks, for `ntensors` tensors:
//   src[w]  : [B][Nl][H][D]          (rank-local sequence shard, user layout)
//   dst[w]  : [P][Nl][B][Hl][D]      (chunk j = heads j*Hl.. of every token)
// If delta_dst != nullptr, also Delta[b,t,h] = sum_d dO.O in fp32 from
// (dout, out) [B][Nl][H][D] into delta_dst [P][Nl][B][Hl] (P == 1: [Nl][B][H]).
cudaError_t launch_pack(const void* const* src, void* const* dst, int ntensors, int64_t B, int64_t Nl, int H, int D,
                        int P, const void* dout, const void* out, float* delta_dst, cudaStream_t stream);
// Received head chunks -> sequence shard, for `ntensors` tensors:
//   src[w]  : [P][Nl][B][Hl][D]      (chunk s = source rank s)
//   dst[w]  : [B][Nl][H][D]
cudaError_t launch_unpack(const void* const* src, void* const* dst, int ntensors, int64_t B, int64_t Nl, int H,
                          int D, int P, cudaStream_t stream);
// dq = bf16(scale * dq_acc), dq_acc [B*heads][N_pad][D] fp32 (N_pad = N rounded up to 128) -> view
cudaError_t launch_dq_finalize(const float* dq_acc, ViewArg dq, int64_t B, int64_t N, int heads, int D, float scale,
                               cudaStream_t stream);
// Backward prep: per head bh and 128-row tile, [128 x -lse*log2(e)][128 x -Delta]
// (rows N <= n < N_pad: -inf, 0).
cudaError_t launch_bwd_prep(const float* lse, int64_t l_sh, int64_t l_sb, const float* delta, int64_t d_sn,
                            int64_t d_sh, int64_t d_sb, float2* lsed, int64_t B, int heads, int64_t N,
                            cudaStream_t stream);
// Peer all-to-all pieces (peer.cu).
cudaError_t launch_pack_push(const PeerPack& pk, int64_t B, int64_t Nl, int H, int D, int P, int rank,
                             cudaStream_t stream);
cudaError_t launch_signal(const PeerFlags& f, int slot, int rank, int P, int64_t step, cudaStream_t stream);
// Spins (bounded: 60 s, then sets *err = 1 and skips the copy) until every peer's flag reached step.
cudaError_t launch_wait_copy(const int64_t* flags, int slot, int P, int64_t step, const void* src, void* dst,
                             int64_t bytes, int* err, cudaStream_t stream);
cudaError_t launch_finalize_push(const float* dq_acc, const PeerOut& o, int64_t B, int64_t N, int heads, int D,
                                 float scale, cudaStream_t stream);
// Exact merge of two LSS segment results (in place into a):
//   lse = logaddexp(lse_a, lse_b); O = e^{lse_a-lse} O_a + e^{lse_b-lse} O_b
cudaError_t launch_lse_merge(float* o_a, float* lse_a, const float* o_b, const float* lse_b, int64_t rows, int D,
                             cudaStream_t stream);
// fp32 [rows][D] -> bf16 view rows (row r = (b, h, n) of [B][heads][N])
cudaError_t launch_f32_to_view(const float* src, ViewArg dst, int64_t B, int64_t N, int heads, int D,
                               cudaStream_t stream);

}  // namespace ua
