// attn_bwd_dq.cu — query-stationary dQ for the deterministic backward (sm_100a),
// D in {32, 64, 80 (= head dim 72 padded), 128}.
//
// Mathematics (recompute form S:209):
//   P_ij = exp(s_ij - lse_i),  dP_ij = dO_i . v_j,  dS_ij = P_ij (dP_ij - Delta_i),
//   dq_acc_i = sum_j dS_ij k_j       (unscaled fp32; dq_finalize applies 1/sqrt(D))
// The KV-stationary backward (attn_bwd_ws_kernel<D, false>) then only produces dK,
// dV.  Here every dQ row is owned by one CTA and summed over the key tiles in
// ascending order inside one TMEM accumulator, so dQ is bitwise reproducible run
// to run and identical for every P ("in the first forward pass,
// all matrices are the same") — the price is recomputing S and dP (3 GEMMs per
// tile pair instead of the fused kernel's one dQ GEMM).
//
// Design: one CTA = one 128-row query tile of one (b, h), 4 + 4 kGroups warps:
//   warp 0      TMA producer (Q, dO once; K/V ring of kStages tiles)
//   warp 1      tcgen05.mma issuer + TMEM owner
//   warps 4..   kGroups elementwise warpgroups, group g owns key columns
//               [kCols g, kCols (g+1)) of each tile (thread = query row);
//               kGroups = 4 (32 columns each, 4 warps per SM sub-partition) by default
// TMEM: S[0] [0,128)  S[1] [128,256)  dP [256,384)  dQ [384, 384+D).
//   S[j&1] = Q K_j^T and dP = dO V_j^T are SS MMAs; the elementwise warpgroups
//   load both, release dP (the next dP GEMM may start), and write bf16 dS into
//   the first kCols/2 of their own S[j&1] columns; dQ += dS K_j is a TS MMA
//   (A = dS from TMEM, B = K_j MN-major, the same smem tile the S GEMM read
//   K-major).  S is double-buffered, so S_{j+1} and dP_{j+1} run under the
//   elementwise work of tile j.
// Keys >= n_kv: K, V rows are zero-filled by TMA, so their dS is finite and
// multiplies a zero K row (no masking needed); query rows >= n get
// -lse*log2e = -inf from the prep array (P = 0) and are not stored.
#include "attn_common.cuh"
#include "attn_kernels.h"

#ifndef UA_BWD_DQ_GROUPS
#define UA_BWD_DQ_GROUPS 4     // elementwise warpgroups per query tile (2: 64 key columns each, 4: 32 each)
#endif
#ifndef UA_BWD_DQ_POLY_MOD
#define UA_BWD_DQ_POLY_MOD 4   // every UA_BWD_DQ_POLY_MOD-th exp2 pair on the FMA pipe (D <= 64; 0: none)
#endif

namespace ua {

namespace {

template <int D>
struct BwdDqCfg {
  using G = TileGeom<D>;
  static constexpr int kStages = D == 128 ? 2 : 3;
  static constexpr int kGroups = UA_BWD_DQ_GROUPS;             // elementwise warpgroups
  static constexpr int kCols = 128 / kGroups;                    // key columns per thread and tile
  static constexpr int kThreads = 128 * (1 + kGroups);
  static constexpr int kSmemBytes = 1024 + (2 + 2 * kStages) * G::kTileBytes + 256;
  static constexpr uint32_t kColS = 0, kColDP = 256, kColDQ = 384;
  static constexpr bool kPolyExp = UA_BWD_DQ_POLY_MOD > 0 && D <= 64;
  // setmaxnreg.inc can only take what the CTA's own warps released: the launch
  // gives every thread kRegsLaunch, the producer / MMA warpgroup drops to kRegsLow.
  static constexpr int kRegsLaunch = (65536 / kThreads) / 8 * 8 > 255 ? 248 : (65536 / kThreads) / 8 * 8;
  static constexpr int kRegsLow = 56;
  static constexpr int kRegsHigh = ((1 + kGroups) * kRegsLaunch - kRegsLow) / kGroups / 8 * 8 > 232
                                       ? 232 : ((1 + kGroups) * kRegsLaunch - kRegsLow) / kGroups / 8 * 8;
  static_assert(kColDQ + D <= 512, "TMEM budget");
  static_assert(kSmemBytes <= 232448, "smem budget");
};

template <int D>
__global__ void __launch_bounds__(BwdDqCfg<D>::kThreads, 1) attn_bwd_dq_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdDqCfg<D>;
  using G = TileGeom<D>;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-B aligned
  uint8_t* sQ = smem;
  uint8_t* sdO = sQ + G::kTileBytes;
  uint8_t* sK = sdO + G::kTileBytes;                   // [kStages]
  uint8_t* sV = sK + kStages * G::kTileBytes;          // [kStages]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kStages * G::kTileBytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;                        // [kStages]
  uint64_t* kv_empty = kv_full + kStages;              // [kStages]
  uint64_t* sdp_full = kv_empty + kStages;             // [2] S[b] and dP computed
  uint64_t* dp_free = sdp_full + 2;                    // dP loaded by both warpgroups
  uint64_t* ds_ready = dp_free + 1;                    // [2] dS stored into S[b]
  uint64_t* dq_done = ds_ready + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tile = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int n_kt = (p.n_kv + 127) / 128;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sdp_full[i], 1);
      mbar_init(&ds_ready[i], 128 * C::kGroups);
    }
    mbar_init(dp_free, 128 * C::kGroups);
    mbar_init(dq_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    setmaxnreg_dec<C::kRegsLow>();
    if (elect_one()) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_do);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      mbar_arrive_expect_tx(q_full, 2 * G::kTileBytes);
      for (int a = 0; a < G::kAtoms; ++a) {
        tma_load_4d(sQ + a * G::kAtomBytes, &p.tm_q, q_full, a * G::kAtomCols, tile * 128, h, b, kEvictFirst);
        tma_load_4d(sdO + a * G::kAtomBytes, &p.tm_do, q_full, a * G::kAtomCols, tile * 128, h, b, kEvictFirst);
      }
      for (int j = 0; j < n_kt; ++j) {
        const int s = j % kStages;
        if (j >= kStages) mbar_wait(&kv_empty[s], ((j / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[s], 2 * G::kTileBytes);
        for (int a = 0; a < G::kAtoms; ++a) {
          tma_load_4d(sK + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_k, &kv_full[s], a * G::kAtomCols, j * 128,
                      h, b, kEvictLast);
          tma_load_4d(sV + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_v, &kv_full[s], a * G::kAtomCols, j * 128,
                      h, b, kEvictLast);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    setmaxnreg_dec<C::kRegsLow>();
    if (elect_one()) {
      const uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);  // S, dP: A, B K-major
      const uint32_t idesc_q = idesc_bf16_f32(128, D, false, true);     // dQ: A = TMEM, B MN-major
      const uint32_t sQa = smem_u32(sQ), sdOa = smem_u32(sdO), sKa = smem_u32(sK), sVa = smem_u32(sV);
      auto issue_dq = [&](int j) {  // dQ += dS(j) K_j; the tile's K/V stage is free afterwards
        const int jb = j & 1;
        mbar_wait(&ds_ready[jb], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t kt = sKa + (j % kStages) * G::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dS keys [16kk, 16kk+16): packed by their warpgroup at the start of its columns
          mma_ts(tbase + C::kColDQ, tbase + C::kColS + jb * 128 + (16 * kk / C::kCols) * C::kCols + (kk * 8) % (C::kCols / 2),
                 mnmajor_desc<D>(kt, kk), idesc_q, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&kv_empty[j % kStages]);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j < n_kt; ++j) {
        const int s = j % kStages, jb = j & 1;
        mbar_wait(&kv_full[s], (j / kStages) & 1);
        tc_fence_after();
        const uint32_t kt = sKa + s * G::kTileBytes, vt = sVa + s * G::kTileBytes;
        // S[jb] = Q K_j^T.  S[jb] last held dS(j-2), whose dQ GEMM was issued
        // before this one: tcgen05.mma from one thread execute in order.
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tbase + C::kColS + jb * 128, kmajor_desc<D>(sQa, kk), kmajor_desc<D>(kt, kk), idesc_s,
                 kk > 0 ? 1u : 0u);
        if (j > 0) {  // dP(j-1) has been loaded by both warpgroups
          mbar_wait(dp_free, (j - 1) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tbase + C::kColDP, kmajor_desc<D>(sdOa, kk), kmajor_desc<D>(vt, kk), idesc_s, kk > 0 ? 1u : 0u);
        mma_commit(&sdp_full[jb]);
        if (j > 0) issue_dq(j - 1);
      }
      issue_dq(n_kt - 1);
      mma_commit(dq_done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ elementwise
    setmaxnreg_inc<C::kRegsHigh>();
    const int g = (warp - 4) / 4;              // key columns [kCols g, kCols (g+1)) of every tile
    const int quad = warp % 4;
    const int r = quad * 32 + lane;            // query row within the tile
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const int64_t bh = int64_t(b) * p.heads + h;
    const int n_pad = (p.n + 127) / 128 * 128;
    const float* lsed_tile = reinterpret_cast<const float*>(p.lsed) + bh * n_pad * 2 + int64_t(tile) * 256;
    const float nl = lsed_tile[r], nd = lsed_tile[128 + r];   // -lse*log2(e), -Delta
    const float2 c2 = make_float2(p.scale_log2, p.scale_log2), nl2 = make_float2(nl, nl), nd2 = make_float2(nd, nd);
    for (int j = 0; j < n_kt; ++j) {
      const int jb = j & 1;
      const uint32_t colS = C::kColS + jb * 128 + C::kCols * g;
      mbar_wait(&sdp_full[jb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t rs[C::kCols], rd[C::kCols];
#pragma unroll
      for (int cc = 0; cc < C::kCols; cc += 32) {
        tmem_ld32(t_lane + colS + cc, rs + cc);
        tmem_ld32(t_lane + C::kColDP + C::kCols * g + cc, rd + cc);
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(dp_free);
      uint32_t pk[C::kCols / 2];
#pragma unroll
      for (int i = 0; i < C::kCols / 2; ++i) {
        const float2 arg = __ffma2_rn(make_float2(__uint_as_float(rs[2 * i]), __uint_as_float(rs[2 * i + 1])), c2, nl2);
        const bool poly = C::kPolyExp && (i % (UA_BWD_DQ_POLY_MOD > 0 ? UA_BWD_DQ_POLY_MOD : 1)) == 1;
        const float2 pp = poly ? exp2_poly2(arg) : make_float2(ex2(arg.x), ex2(arg.y));
        const float2 dd = __fadd2_rn(make_float2(__uint_as_float(rd[2 * i]), __uint_as_float(rd[2 * i + 1])), nd2);
        const float2 ds = __fmul2_rn(pp, dd);
        pk[i] = pack_bf16x2(ds.x, ds.y);
      }
      if constexpr (C::kCols == 64) tmem_st32(t_lane + colS, pk);   // own columns only (already loaded)
      else tmem_st16(t_lane + colS, pk);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&ds_ready[jb]);
    }
    // ------------------------------------------------------------ epilogue: dq_acc row (unscaled)
    mbar_wait(dq_done, 0);
    tc_fence_after();
    const int q_row = tile * 128 + r;
    const int d_io = D % 32 == 0 ? D : p.d_io;
    float* dst = p.dq_acc + (bh * n_pad + q_row) * d_io;
#pragma unroll
    for (int cc = 0; cc < D; cc += 16) {
      if ((cc / 16) % C::kGroups != g) continue;
      uint32_t x[16];
      tmem_ld16(t_lane + C::kColDQ + cc, x);
      tmem_ld_wait();
      if (q_row < p.n) {
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          if (cc + e < d_io)
            *reinterpret_cast<float4*>(dst + cc + e) =
                make_float4(__uint_as_float(x[e]), __uint_as_float(x[e + 1]), __uint_as_float(x[e + 2]),
                            __uint_as_float(x[e + 3]));
      }
    }
  } else {
    setmaxnreg_dec<C::kRegsLow>();  // warps 2, 3: idle members of the producer / MMA warpgroup
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tbase);
}

template <int D>
cudaError_t launch_bwd_dq_impl(const BwdParams& p, cudaStream_t stream) {
  using C = BwdDqCfg<D>;
  cudaError_t e = set_max_smem(attn_bwd_dq_kernel<D>, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  dim3 grid((p.n + 127) / 128, p.heads, p.batch);
  attn_bwd_dq_kernel<D><<<grid, C::kThreads, C::kSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_bwd_dq(const BwdParams& p, int D, cudaStream_t stream) {
  switch (D) {
    case 32: return launch_bwd_dq_impl<32>(p, stream);
    case 64: return launch_bwd_dq_impl<64>(p, stream);
    case 72: return launch_bwd_dq_impl<80>(p, stream);   // padded MMA head dim, p.d_io = 72
    case 128: return launch_bwd_dq_impl<128>(p, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ua
