// attn_bwd_v2.cu — attention backward for D <= 64 with the elementwise work
// overlapped against the tensor core (sm_100a).
//
// Same mathematics as attn_bwd.cu:
//   P = exp(S - lse), dV += P^T dO, dS = P (dP - Delta), dK += scale dS^T Q,
//   dQ += scale dS K.
// Differences from v1 (attn_bwd.cu), all scheduling:
//  * each 128-query tile is processed as two 64-query halves h whose S^T / dP^T
//    live in separate TMEM buffers: while the elementwise warpgroup turns half
//    h into P^T / dS^T, the tensor core runs the other half's GEMMs;
//  * dS^T is double-buffered in smem (one buffer per query tile parity), so the
//    next tile's elementwise never waits for the previous dQ GEMM;
//  * dQ partials leave through an fp32 smem staging tile and ONE bulk
//    cp.reduce.async.bulk (.add.f32) of 128*D*4 contiguous bytes per tile,
//    instead of per-thread vector atomics;
//  * each CTA starts its sweep over query tiles at a different tile
//    (i0 = key_tile * n_q / n_key_tiles) so concurrent CTAs reduce into
//    different dq rows (no same-line contention in L2).
// TMEM: S^T[h] [64h, 64h+64)  dP^T[h] [128+64h, ..)  dV [256, 256+D)
//       dK [256+D, 256+2D)  dQ [256+2D, 256+3D)   (<= 448 columns).
#include "attn_common.cuh"
#include "attn_kernels.h"

namespace ua {

namespace {

template <int D>
struct BwdV2Cfg {
  using G = TileGeom<D>;
  static constexpr int kStages = 2;
  static constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + D, kColDQ = 256 + 2 * D;
  static constexpr int kDsBytes = 128 * 128 * 2;
  static constexpr int kStageBytes = 128 * D * 4;
  static constexpr int kSmemBytes =
      1024 + (2 + 2 * kStages) * G::kTileBytes + 2 * kDsBytes + kStageBytes + kStages * 128 * 8 + 256;
  static_assert(256 + 3 * D <= 512, "TMEM budget");
};

template <int D>
__global__ void __launch_bounds__(384, 1) attn_bwd_v2_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdV2Cfg<D>;
  using G = TileGeom<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + G::kTileBytes;
  uint8_t* sQ = sV + G::kTileBytes;               // [2]
  uint8_t* sdO = sQ + 2 * G::kTileBytes;          // [2]
  uint8_t* sdS = sdO + 2 * G::kTileBytes;         // [2] dS^T [128 keys][128 q] bf16 (2 SW128 atoms)
  float* sStage = reinterpret_cast<float*>(sdS + 2 * C::kDsBytes);  // dQ tile [128][D] fp32
  float* s_nlse = sStage + 128 * D;               // [2][128]
  float* s_dlt = s_nlse + 2 * 128;                // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_dlt + 2 * 128);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;      // [2]
  uint64_t* qdo_empty = bars + 3;     // [2]
  uint64_t* sdp_full = bars + 5;      // [2] per half
  uint64_t* ds_ready = bars + 7;      // [2] per half
  uint64_t* ds_free = bars + 9;       // [2] per dS buffer
  uint64_t* dq_full = bars + 11;
  uint64_t* dq_empty = bars + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int h_ = blockIdx.y, b = blockIdx.z;
  const int k0 = blockIdx.x * 128;
  const int n_q = (p.n + 127) / 128;
  const int i0 = int((int64_t(blockIdx.x) * n_q) / gridDim.x);

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qdo_full[s], 32);
      mbar_init(&qdo_empty[s], 1);
      mbar_init(&sdp_full[s], 1);
      mbar_init(&ds_ready[s], 128);
      mbar_init(&ds_free[s], 1);
    }
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 128);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      tma_prefetch_desc(&p.tm_do);
      mbar_arrive_expect_tx(kv_full, 2 * G::kTileBytes);
      for (int a = 0; a < G::kAtoms; ++a) {
        tma_load_4d(sK + a * G::kAtomBytes, &p.tm_k, kv_full, a * G::kAtomCols, k0, h_, b, kEvictFirst);
        tma_load_4d(sV + a * G::kAtomBytes, &p.tm_v, kv_full, a * G::kAtomCols, k0, h_, b, kEvictFirst);
      }
    }
    const float* lse_bh = p.lse + b * p.l_sb + h_ * p.l_sh;
    const float* dlt_bh = p.delta + b * p.d_sb + h_ * p.d_sh;
    for (int t = 0; t < n_q; ++t) {
      const int s = t & 1;
      const int tile = (i0 + t) % n_q;
      if (t >= 2) mbar_wait(&qdo_empty[s], ((t >> 1) & 1) ^ 1);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = r * 32 + lane;
        const int qi = tile * 128 + row;
        const bool ok = qi < p.n;
        s_nlse[s * 128 + row] = ok ? -lse_bh[qi] * kLog2e : -INFINITY;
        s_dlt[s * 128 + row] = ok ? dlt_bh[int64_t(qi) * p.d_sn] : 0.f;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(&qdo_full[s], 2 * G::kTileBytes);
        for (int a = 0; a < G::kAtoms; ++a) {
          tma_load_4d(sQ + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_q, &qdo_full[s], a * G::kAtomCols,
                      tile * 128, h_, b, kEvictLast);
          tma_load_4d(sdO + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_do, &qdo_full[s], a * G::kAtomCols,
                      tile * 128, h_, b, kEvictLast);
        }
      } else {
        mbar_arrive(&qdo_full[s]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc_s = idesc_bf16_f32(128, 64, false, false);  // S^T, dP^T half: N = 64 queries
      const uint32_t idesc_g = idesc_bf16_f32(128, D, false, true);    // dV, dK: A = TMEM, B MN-major
      const uint32_t idesc_q = idesc_bf16_f32(128, D, true, true);     // dQ: A, B MN-major
      const uint32_t sKa = smem_u32(sK), sVa = smem_u32(sV), sQa = smem_u32(sQ), sdOa = smem_u32(sdO);
      const uint32_t sdSa = smem_u32(sdS);
      auto issue_sdp = [&](int t, int h) {
        const int s = t & 1;
        const uint32_t qt = sQa + s * G::kTileBytes + 64 * h * G::kSw;
        const uint32_t dot = sdOa + s * G::kTileBytes + 64 * h * G::kSw;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tbase + C::kColS + 64 * h, kmajor_desc<D>(sKa, kk), kmajor_desc<D>(qt, kk), idesc_s,
                 kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tbase + C::kColDP + 64 * h, kmajor_desc<D>(sVa, kk), kmajor_desc<D>(dot, kk), idesc_s,
                 kk > 0 ? 1u : 0u);
        mma_commit(&sdp_full[h]);
      };
      mbar_wait(kv_full, 0);
      mbar_wait(&qdo_full[0], 0);
      tc_fence_after();
      issue_sdp(0, 0);
      issue_sdp(0, 1);
      for (int t = 0; t < n_q; ++t) {
        const int s = t & 1;
        const uint32_t qt = sQa + s * G::kTileBytes, dot = sdOa + s * G::kTileBytes;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&ds_ready[h], t & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts(tbase + C::kColDV, tbase + C::kColS + 64 * h + kk * 8, mnmajor_desc<D>(dot, 4 * h + kk),
                   idesc_g, (t > 0 || h > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts(tbase + C::kColDK, tbase + C::kColDP + 64 * h + kk * 8, mnmajor_desc<D>(qt, 4 * h + kk),
                   idesc_g, (t > 0 || h > 0 || kk > 0) ? 1u : 0u);
          if (h == 1) {
            if (t > 0) {
              mbar_wait(dq_empty, (t - 1) & 1);
              tc_fence_after();
            }
            const uint32_t ds = sdSa + (t & 1) * C::kDsBytes;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_ss(tbase + C::kColDQ, mnmajor_desc<128>(ds, kk), mnmajor_desc<D>(sKa, kk), idesc_q,
                     kk > 0 ? 1u : 0u);
            mma_commit(dq_full);
            mma_commit(&ds_free[t & 1]);
            mma_commit(&qdo_empty[s]);
          }
          if (t + 1 < n_q) {
            if (h == 0) {
              mbar_wait(&qdo_full[(t + 1) & 1], ((t + 1) >> 1) & 1);
              tc_fence_after();
            }
            issue_sdp(t + 1, h);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ elementwise
    const int quad = warp % 4;
    const int j = quad * 32 + lane;  // key row within the tile
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const float c = p.scale_log2;
    for (int t = 0; t < n_q; ++t) {
      const int s = t & 1;
      mbar_wait(&qdo_full[s], (t >> 1) & 1);                    // lse / Delta visibility
      if (t >= 2) mbar_wait(&ds_free[t & 1], ((t >> 1) & 1) ^ 1);  // dS buffer consumed by dQ(t-2)
      uint8_t* ds_row = sdS + (t & 1) * C::kDsBytes + j * 128;
      const float4* nl4 = reinterpret_cast<const float4*>(s_nlse + s * 128);
      const float4* dl4 = reinterpret_cast<const float4*>(s_dlt + s * 128);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mbar_wait(&sdp_full[h], t & 1);
        tc_fence_after();
        uint8_t* atom = ds_row + h * (128 * 128);
#pragma unroll
        for (int cc = 0; cc < 64; cc += 32) {
          uint32_t rs[32], rd[32];
          tmem_ld32(t_lane + C::kColS + 64 * h + cc, rs);
          tmem_ld32(t_lane + C::kColDP + 64 * h + cc, rd);
          tmem_ld_wait();
          uint32_t pk_p[16], pk_ds[16];
#pragma unroll
          for (int x = 0; x < 32; x += 4) {
            const float4 nl = nl4[(64 * h + cc + x) / 4];
            const float4 dl = dl4[(64 * h + cc + x) / 4];
            const float p0 = ex2(fmaf(__uint_as_float(rs[x + 0]), c, nl.x));
            const float p1 = ex2(fmaf(__uint_as_float(rs[x + 1]), c, nl.y));
            const float p2 = ex2(fmaf(__uint_as_float(rs[x + 2]), c, nl.z));
            const float p3 = ex2(fmaf(__uint_as_float(rs[x + 3]), c, nl.w));
            pk_p[x / 2] = pack_bf16x2(p0, p1);
            pk_p[x / 2 + 1] = pack_bf16x2(p2, p3);
            pk_ds[x / 2] = pack_bf16x2(p0 * (__uint_as_float(rd[x + 0]) - dl.x), p1 * (__uint_as_float(rd[x + 1]) - dl.y));
            pk_ds[x / 2 + 1] = pack_bf16x2(p2 * (__uint_as_float(rd[x + 2]) - dl.z), p3 * (__uint_as_float(rd[x + 3]) - dl.w));
          }
          tmem_st16(t_lane + C::kColS + 64 * h + cc / 2, pk_p);
          tmem_st16(t_lane + C::kColDP + 64 * h + cc / 2, pk_ds);
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {
            const int chunk = ((cc / 8) + qd) ^ (j & 7);
            *reinterpret_cast<uint4*>(atom + chunk * 16) =
                make_uint4(pk_ds[4 * qd], pk_ds[4 * qd + 1], pk_ds[4 * qd + 2], pk_ds[4 * qd + 3]);
          }
        }
        fence_proxy_async_smem();
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&ds_ready[h]);
      }
    }
    // -------------------------------------------------------- dK, dV epilogue
    mbar_wait(dq_full, (n_q - 1) & 1);
    tc_fence_after();
    const int krow = k0 + j;
    const bool valid = krow < p.n;
    __nv_bfloat16* dv_row = reinterpret_cast<__nv_bfloat16*>(p.dv.base) + b * p.dv.sb + h_ * p.dv.sh + int64_t(krow) * p.dv.sn;
    __nv_bfloat16* dk_row = reinterpret_cast<__nv_bfloat16*>(p.dk.base) + b * p.dk.sb + h_ * p.dk.sh + int64_t(krow) * p.dk.sn;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t col = which == 0 ? C::kColDV : C::kColDK;
      const float sc = which == 0 ? 1.f : p.scale;
      __nv_bfloat16* dst = which == 0 ? dv_row : dk_row;
#pragma unroll
      for (int cc = 0; cc < D; cc += 32) {
        uint32_t r[32];
        tmem_ld32(t_lane + col + cc, r);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int x = 0; x < 16; ++x) pk[x] = pack_bf16x2(__uint_as_float(r[2 * x]) * sc, __uint_as_float(r[2 * x + 1]) * sc);
        if (valid) {
#pragma unroll
          for (int x = 0; x < 16; x += 4)
            *reinterpret_cast<uint4*>(dst + cc + 2 * x) = make_uint4(pk[x], pk[x + 1], pk[x + 2], pk[x + 3]);
        }
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ dQ drain
    const int quad = warp % 4;
    const int r = quad * 32 + lane;  // query row within the tile
    const bool leader = threadIdx.x == 256;
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const int n_pad = n_q * 128;
    for (int t = 0; t < n_q; ++t) {
      const int tile = (i0 + t) % n_q;
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
      float acc[D];
#pragma unroll
      for (int cc = 0; cc < D; cc += 32) {
        uint32_t x[32];
        tmem_ld32(t_lane + C::kColDQ + cc, x);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) acc[cc + e] = __uint_as_float(x[e]);
      }
      tc_fence_before();
      mbar_arrive(dq_empty);
      if (leader) bulk_wait_read<0>();   // previous reduction has read the staging tile
      named_bar_sync(1, 128);
      // staging = D/32 SW128 boxes [128 rows][32 fp32]; 16-B chunk q of row r
      // sits at chunk q ^ (r & 7): conflict-free stores across the warp
      uint8_t* srow = reinterpret_cast<uint8_t*>(sStage) + r * 128;
#pragma unroll
      for (int cb = 0; cb < D / 32; ++cb)
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4)
          *reinterpret_cast<float4*>(srow + cb * 16384 + ((q4 ^ (r & 7)) * 16)) =
              make_float4(acc[32 * cb + 4 * q4], acc[32 * cb + 4 * q4 + 1], acc[32 * cb + 4 * q4 + 2],
                          acc[32 * cb + 4 * q4 + 3]);
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (leader) {
        const int row0 = (b * p.heads + h_) * n_pad + tile * 128;
#pragma unroll
        for (int cb = 0; cb < D / 32; ++cb)
          tma_reduce_add_2d(&p.tm_dq, reinterpret_cast<uint8_t*>(sStage) + cb * 16384, 32 * cb, row0);
        bulk_commit();
      }
    }
    if (leader) bulk_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tbase);
}

template <int D>
cudaError_t launch_bwd_v2_impl(const BwdParams& p, int B, int heads, cudaStream_t stream) {
  using C = BwdV2Cfg<D>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e =
        cudaFuncSetAttribute(attn_bwd_v2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((p.n + 127) / 128, heads, B);
  attn_bwd_v2_kernel<D><<<grid, 384, C::kSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_bwd_v2(const BwdParams& p, int D, int B, int heads, cudaStream_t stream) {
  switch (D) {
    case 32: return launch_bwd_v2_impl<32>(p, B, heads, stream);
    case 64: return launch_bwd_v2_impl<64>(p, B, heads, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ua
