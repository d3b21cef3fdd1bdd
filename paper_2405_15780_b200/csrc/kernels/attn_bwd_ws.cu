// attn_bwd_ws.cu — persistent, warp-specialised attention backward for D <= 64
// (sm_100a).
//
// Mathematics as attn_bwd.cu:
//   P = exp(S - lse), dV += P^T dO, dS = P (dP - Delta), dK += scale dS^T Q,
//   dQ += scale dS K   (dQ partials reduced in fp32; scale applied later).
//
// Scheduling (the B200-specific part):
//  * persistent grid (<= one CTA per SM); work item = one 128-key tile of one
//    (b, h), items in head-major order, CTA c takes items c, c+G, ...  All
//    CTAs sweep their query tiles at the same rate, so at any moment they
//    touch a narrow window of Q / dO / dq rows of the same head (L2-resident
//    even at N = 188K where one head's Q, dO and dq are ~96 MB).  Start tiles
//    are staggered over a window of kStagger tiles so that only ~G/kStagger
//    CTAs reduce into the same dq tile at once.
//  * 16 warps: 0 TMA producer, 1 tcgen05.mma issuer, 4-7 elementwise for the
//    even 64-query half, 8-11 for the odd half, 12-15 dQ drain.  Each query
//    tile's halves have separate TMEM S^T / dP^T buffers, so the two
//    elementwise warpgroups and the tensor core work on different halves at
//    the same time.
//  * dQ: TMEM -> swizzled fp32 smem tile -> TMA tensor reduce-add
//    (cp.reduce.async.bulk.tensor .add) into dq_acc.
// TMEM: S^T[h] [64h, +64)  dP^T[h] [128+64h, +64)  dV [256, +D)  dK [256+D, +D)
//       dQ [256+2D, +D).
#include "attn_common.cuh"
#include "attn_kernels.h"

#ifndef UA_BWD_POLY_MOD
#define UA_BWD_POLY_MOD 4   // every UA_BWD_POLY_MOD-th exp2 pair on the FMA pipe (0: none)
#endif
#ifndef UA_BWD_STAGGER
#define UA_BWD_STAGGER 16   // query-tile window the persistent CTAs' start tiles are spread over
#endif

namespace ua {

namespace {

template <int D>
struct BwdWsCfg {
  using G = TileGeom<D>;
  static constexpr int kThreads = 512;
  static constexpr int kStagger = UA_BWD_STAGGER;
  static constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + D, kColDQ = 256 + 2 * D;
  static constexpr int kDsBytes = 128 * 128 * 2;
  static constexpr int kStages = 3;                 // Q / dO / (lse, Delta) ring depth
  static constexpr bool kPolyExp = true;            // 1/4 of exp2 on the FMA pipe
  static constexpr int kStageBytes = 128 * 32 * 4;  // one 32-column fp32 box of the dQ tile
  static constexpr int kLsedBytes = 128 * 8;        // (-lse*log2e, Delta) per query row
  static constexpr int kSmemBytes = 1024 + (2 + 2 * kStages) * G::kTileBytes + 2 * kDsBytes + kStageBytes +
                                    kStages * kLsedBytes + 256;
  static_assert(256 + 3 * D <= 512, "TMEM budget");
};

template <int D>
__global__ void __launch_bounds__(512, 1) attn_bwd_ws_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdWsCfg<D>;
  using G = TileGeom<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + G::kTileBytes;
  constexpr int kS = C::kStages;
  uint8_t* sQ = sV + G::kTileBytes;               // [kS]
  uint8_t* sdO = sQ + kS * G::kTileBytes;         // [kS]
  uint8_t* sdS = sdO + kS * G::kTileBytes;        // [2] dS^T [128 keys][128 q] bf16 (2 SW128 atoms)
  uint8_t* sStage = sdS + 2 * C::kDsBytes;        // one SW128 box [128][32] fp32 of the dQ tile
  float2* s_lsed = reinterpret_cast<float2*>(sStage + C::kStageBytes);  // [kS][128] (-lse*log2e, Delta)
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_lsed + kS * 128);
  uint64_t* kv_full = bars + 0;
  uint64_t* kv_empty = bars + 1;
  uint64_t* sdp_full = bars + 2;      // [2] per half
  uint64_t* ds_ready = bars + 4;      // [2] per half
  uint64_t* ds_free = bars + 6;       // [2] per dS buffer
  uint64_t* dq_full = bars + 8;
  uint64_t* dq_empty = bars + 9;
  uint64_t* acc_full = bars + 10;
  uint64_t* acc_free = bars + 11;
  uint64_t* qdo_full = bars + 12;     // [kS]
  uint64_t* qdo_empty = qdo_full + kS;  // [kS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qdo_empty + kS);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_q = (p.n + 127) / 128;
  const int n_kt = n_q;
  const int n_items = p.batch * p.heads * n_kt;
  const int start = int((int64_t(blockIdx.x) * C::kStagger) / gridDim.x) % n_q;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    for (int s = 0; s < kS; ++s) {
      mbar_init(&qdo_full[s], 1);
      mbar_init(&qdo_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sdp_full[s], 1);
      mbar_init(&ds_ready[s], 128);
      mbar_init(&ds_free[s], 1);
    }
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 128);
    mbar_init(acc_full, 1);
    mbar_init(acc_free, 256);
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
    }
    if (lane == 0) {
      int T = 0, it = 0;
      const int n_pad = n_q * 128;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int kt = item % n_kt, bh = item / n_kt;
        const int b = bh / p.heads, h = bh % p.heads;
        if (it > 0) mbar_wait(kv_empty, (it - 1) & 1);
        mbar_arrive_expect_tx(kv_full, 2 * G::kTileBytes);
        for (int a = 0; a < G::kAtoms; ++a) {
          tma_load_4d(sK + a * G::kAtomBytes, &p.tm_k, kv_full, a * G::kAtomCols, kt * 128, h, b, kEvictFirst);
          tma_load_4d(sV + a * G::kAtomBytes, &p.tm_v, kv_full, a * G::kAtomCols, kt * 128, h, b, kEvictFirst);
        }
        const float2* lsed_bh = p.lsed + int64_t(bh) * n_pad;
        for (int t = 0; t < n_q; ++t, ++T) {
          const int s = T % kS;
          const int tile = (start + t) % n_q;
          if (T >= kS) mbar_wait(&qdo_empty[s], ((T / kS) & 1) ^ 1);
          mbar_arrive_expect_tx(&qdo_full[s], 2 * G::kTileBytes + C::kLsedBytes);
          for (int a = 0; a < G::kAtoms; ++a) {
            tma_load_4d(sQ + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_q, &qdo_full[s], a * G::kAtomCols,
                        tile * 128, h, b, kEvictLast);
            tma_load_4d(sdO + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_do, &qdo_full[s], a * G::kAtomCols,
                        tile * 128, h, b, kEvictLast);
          }
          bulk_load(s_lsed + s * 128, lsed_bh + tile * 128, C::kLsedBytes, &qdo_full[s]);
        }
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
      auto issue_sdp = [&](int T, int hh) {
        const int s = T % kS;
        const uint32_t qt = sQa + s * G::kTileBytes + 64 * hh * G::kSw;
        const uint32_t dot = sdOa + s * G::kTileBytes + 64 * hh * G::kSw;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tbase + C::kColS + 64 * hh, kmajor_desc<D>(sKa, kk), kmajor_desc<D>(qt, kk), idesc_s,
                 kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tbase + C::kColDP + 64 * hh, kmajor_desc<D>(sVa, kk), kmajor_desc<D>(dot, kk), idesc_s,
                 kk > 0 ? 1u : 0u);
        mma_commit(&sdp_full[hh]);
      };
      int T = 0, it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        mbar_wait(kv_full, it & 1);
        mbar_wait(&qdo_full[T % kS], (T / kS) & 1);
        tc_fence_after();
        issue_sdp(T, 0);
        issue_sdp(T, 1);
        if (it > 0) {
          mbar_wait(acc_free, (it - 1) & 1);  // previous item's dV / dK drained
          tc_fence_after();
        }
        for (int t = 0; t < n_q; ++t, ++T) {
          const int s = T % kS;
          const uint32_t qt = sQa + s * G::kTileBytes, dot = sdOa + s * G::kTileBytes;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            mbar_wait(&ds_ready[hh], T & 1);
            tc_fence_after();
            const uint32_t acc = (t > 0 || hh > 0) ? 1u : 0u;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ts(tbase + C::kColDV, tbase + C::kColS + 64 * hh + kk * 8, mnmajor_desc<D>(dot, 4 * hh + kk),
                     idesc_g, (acc || kk > 0) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ts(tbase + C::kColDK, tbase + C::kColDP + 64 * hh + kk * 8, mnmajor_desc<D>(qt, 4 * hh + kk),
                     idesc_g, (acc || kk > 0) ? 1u : 0u);
            if (hh == 1) {
              if (T > 0) {
                mbar_wait(dq_empty, (T - 1) & 1);
                tc_fence_after();
              }
              const uint32_t ds = sdSa + (T & 1) * C::kDsBytes;
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                mma_ss(tbase + C::kColDQ, mnmajor_desc<128>(ds, kk), mnmajor_desc<D>(sKa, kk), idesc_q,
                       kk > 0 ? 1u : 0u);
              mma_commit(dq_full);
              mma_commit(&ds_free[T & 1]);
              mma_commit(&qdo_empty[s]);
            }
            if (t + 1 < n_q) {
              if (hh == 0) {
                mbar_wait(&qdo_full[(T + 1) % kS], ((T + 1) / kS) & 1);
                tc_fence_after();
              }
              issue_sdp(T + 1, hh);
            }
          }
        }
        mma_commit(acc_full);
        mma_commit(kv_empty);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 12) {
    // ------------------------------------------------------------ elementwise (half hh)
    const int hh = (warp - 4) / 4;
    const int quad = warp % 4;
    const int j = quad * 32 + lane;  // key row within the tile
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const uint32_t colS = C::kColS + 64 * hh, colDP = C::kColDP + 64 * hh;
    const float c = p.scale_log2;
    int T = 0, it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const int kt = item % n_kt, bh = item / n_kt;
      const int b = bh / p.heads, h = bh % p.heads;
      for (int t = 0; t < n_q; ++t, ++T) {
        const int s = T % kS;
        mbar_wait(&qdo_full[s], (T / kS) & 1);                       // (lse, Delta) landed
        if (T >= 2) mbar_wait(&ds_free[T & 1], ((T >> 1) & 1) ^ 1);  // dS buffer consumed by dQ(T-2)
        mbar_wait(&sdp_full[hh], T & 1);
        tc_fence_after();
        uint8_t* atom = sdS + (T & 1) * C::kDsBytes + hh * (128 * 128) + j * 128;
        const float* tl = reinterpret_cast<const float*>(s_lsed + s * 128);  // [128 -lse*log2e][128 -Delta]
        const float4* nl4 = reinterpret_cast<const float4*>(tl + 64 * hh);
        const float4* nd4 = reinterpret_cast<const float4*>(tl + 128 + 64 * hh);
        const float2 c2 = make_float2(c, c);
#pragma unroll
        for (int cc = 0; cc < 64; cc += 16) {
          uint32_t rs[16], rd[16];
          tmem_ld16(t_lane + colS + cc, rs);
          tmem_ld16(t_lane + colDP + cc, rd);
          tmem_ld_wait();
          uint32_t pk_p[8], pk_ds[8];
#pragma unroll
          for (int x = 0; x < 16; x += 4) {
            const float4 nl = nl4[(cc + x) / 4];
            const float4 nd = nd4[(cc + x) / 4];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float2 arg = __ffma2_rn(make_float2(__uint_as_float(rs[x + 2 * u]), __uint_as_float(rs[x + 2 * u + 1])),
                                            c2, u == 0 ? make_float2(nl.x, nl.y) : make_float2(nl.z, nl.w));
              // a quarter of the pairs on the FMA-pipe polynomial
              const bool poly = C::kPolyExp && UA_BWD_POLY_MOD > 0 &&
                                ((x / 2 + u) % (UA_BWD_POLY_MOD > 0 ? UA_BWD_POLY_MOD : 1)) == 1;
              const float2 pp = poly ? exp2_poly2(arg) : make_float2(ex2(arg.x), ex2(arg.y));
              const float2 dd = __fadd2_rn(make_float2(__uint_as_float(rd[x + 2 * u]), __uint_as_float(rd[x + 2 * u + 1])),
                                           u == 0 ? make_float2(nd.x, nd.y) : make_float2(nd.z, nd.w));
              const float2 ds = __fmul2_rn(pp, dd);
              pk_p[x / 2 + u] = pack_bf16x2(pp.x, pp.y);
              pk_ds[x / 2 + u] = pack_bf16x2(ds.x, ds.y);
            }
          }
          tmem_st8(t_lane + colS + cc / 2, pk_p);
          tmem_st8(t_lane + colDP + cc / 2, pk_ds);
#pragma unroll
          for (int qd = 0; qd < 2; ++qd) {
            const int chunk = ((cc / 8) + qd) ^ (j & 7);
            *reinterpret_cast<uint4*>(atom + chunk * 16) =
                make_uint4(pk_ds[4 * qd], pk_ds[4 * qd + 1], pk_ds[4 * qd + 2], pk_ds[4 * qd + 3]);
          }
        }
        fence_proxy_async_smem();
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&ds_ready[hh]);
      }
      // ------------------------------------------------ dV (hh=0) / dK (hh=1) epilogue
      mbar_wait(acc_full, it & 1);
      tc_fence_after();
      const int krow = kt * 128 + j;
      const bool valid = krow < p.n;
      const ViewArg& dst_v = hh == 0 ? p.dv : p.dk;
      const uint32_t col = hh == 0 ? C::kColDV : C::kColDK;
      const float sc = hh == 0 ? 1.f : p.scale;
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(dst_v.base) + b * dst_v.sb + h * dst_v.sh +
                           int64_t(krow) * dst_v.sn;
#pragma unroll
      for (int cc = 0; cc < D; cc += 16) {
        uint32_t r[16];
        tmem_ld16(t_lane + col + cc, r);
        tmem_ld_wait();
        uint32_t pk[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) pk[x] = pack_bf16x2(__uint_as_float(r[2 * x]) * sc, __uint_as_float(r[2 * x + 1]) * sc);
        if (valid) {
          *reinterpret_cast<uint4*>(dst + cc) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(dst + cc + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      tc_fence_before();
      mbar_arrive(acc_free);
    }
  } else if (warp >= 12) {
    // ------------------------------------------------------------ dQ drain
    const int quad = warp % 4;
    const int r = quad * 32 + lane;  // query row within the tile
    const bool leader = threadIdx.x == 384;
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const int n_pad = n_q * 128;
    int T = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int bh = item / n_kt;
      for (int t = 0; t < n_q; ++t, ++T) {
        const int tile = (start + t) % n_q;
        mbar_wait(dq_full, T & 1);
        tc_fence_after();
        float acc[D];
#pragma unroll
        for (int cc = 0; cc < D; cc += 16) {
          uint32_t x[16];
          tmem_ld16(t_lane + C::kColDQ + cc, x);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[cc + e] = __uint_as_float(x[e]);
        }
        tc_fence_before();
        mbar_arrive(dq_empty);
        uint8_t* srow = sStage + r * 128;
#pragma unroll
        for (int cb = 0; cb < D / 32; ++cb) {
          if (leader) bulk_wait_read<0>();   // previous reduction has read the staging box
          named_bar_sync(1, 128);
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            *reinterpret_cast<float4*>(srow + ((q4 ^ (r & 7)) * 16)) =
                make_float4(acc[32 * cb + 4 * q4], acc[32 * cb + 4 * q4 + 1], acc[32 * cb + 4 * q4 + 2],
                            acc[32 * cb + 4 * q4 + 3]);
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (leader) {
            tma_reduce_add_2d(&p.tm_dq, sStage, 32 * cb, bh * n_pad + tile * 128);
            bulk_commit();
          }
        }
      }
    }
    if (leader) bulk_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tbase);
}

template <int D>
cudaError_t launch_bwd_ws_impl(const BwdParams& p, cudaStream_t stream) {
  using C = BwdWsCfg<D>;
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e =
        cudaFuncSetAttribute(attn_bwd_ws_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
  }
  const int64_t items = int64_t(p.batch) * p.heads * ((p.n + 127) / 128);
  const int grid = int(items < num_sms ? items : num_sms);
  attn_bwd_ws_kernel<D><<<grid, C::kThreads, C::kSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_bwd_ws(const BwdParams& p, int D, cudaStream_t stream) {
  switch (D) {
    case 32: return launch_bwd_ws_impl<32>(p, stream);
    case 64: return launch_bwd_ws_impl<64>(p, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ua
