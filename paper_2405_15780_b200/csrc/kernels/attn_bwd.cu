// attn_bwd.cu — exact attention backward for one head shard, sm_100a.
//
// For every (b, h) and key j / query i of the launch (SPEC.md S:181-183,
// FlashAttention-2 recompute backward):
//   P_ij  = exp(s_ij - lse_i),          s_ij = q_i.k_j / sqrt(D)
//   dV_j  = sum_i P_ij dO_i
//   dS_ij = P_ij (dO_i.v_j - Delta_i),  Delta_i = dO_i.o_i (precomputed)
//   dK_j  = scale sum_i dS_ij q_i
//   dQ_i  = scale sum_j dS_ij k_j       (fp32 partials reduced in dq_acc)
//
// Design (KV-stationary): one CTA owns a 128-key tile of one (b, h); K and V
// stay in smem; it sweeps all 128-query tiles i.  Warps:
//   warp 0       TMA producer (Q_i, dO_i ring; lse_i, Delta_i vectors)
//   warp 1       tcgen05.mma issuer + TMEM owner
//   warps 4-7    elementwise: thread = key row j; P^T, dS^T from S^T, dP^T
//   warps 8-11   dQ drain: thread = query row; TMEM -> red.global.add.v4.f32
// Per query tile (all MMAs M=128, fp32 accumulation in TMEM):
//   S^T  = K Q_i^T     (SS)              TMEM cols [0,128)
//   dP^T = V dO_i^T    (SS)              TMEM cols [128,256)
//   elementwise -> P^T bf16 over S^T cols [0,64), dS^T bf16 over dP^T [0,64),
//                  dS^T also to smem (MN-major A operand of the dQ GEMM)
//   dV  += P^T dO_i    (TS, A = P^T from TMEM, B = dO_i MN-major)
//   dK  += dS^T Q_i    (TS, A = dS^T from TMEM, B = Q_i MN-major)
//   dQ_i = dS K        (SS, A = dS MN-major from smem, B = K MN-major)
// Rows past N need no masking: out-of-range keys have K = V = 0 (TMA zero
// fill) so they add nothing to dQ and their dK/dV rows are not stored;
// out-of-range queries get lse = +inf (P = 0) and Delta = 0.
#include <cstdlib>
#include <cstring>

#include "attn_common.cuh"
#include "attn_kernels.h"

namespace ua {

namespace {

template <int D>
struct BwdCfg {
  using G = TileGeom<D>;
  static constexpr int kStages = D == 128 ? 1 : 2;
  static constexpr int kThreads = 384;
  static constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + D;
  static constexpr bool kDqAliasDp = (256 + 3 * D) > 512;
  static constexpr uint32_t kColDQ = kDqAliasDp ? kColDP : 256 + 2 * D;
  static constexpr int kDsBytes = 128 * 128 * 2;
  static constexpr int kSmemBytes = 1024 + (2 + 2 * kStages) * G::kTileBytes + kDsBytes + kStages * 128 * 8 + 256;
};

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(384, 1) attn_bwd_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdCfg<D>;
  using G = TileGeom<D>;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-B aligned, stays in the shared window
  uint8_t* sK = smem;
  uint8_t* sV = sK + G::kTileBytes;
  uint8_t* sQ = sV + G::kTileBytes;                 // [kStages]
  uint8_t* sdO = sQ + kStages * G::kTileBytes;      // [kStages]
  uint8_t* sdS = sdO + kStages * G::kTileBytes;     // dS^T [128 keys][128 queries] bf16, 2 SW128 atoms
  float* s_nlse = reinterpret_cast<float*>(sdS + C::kDsBytes);  // [kStages][128]  -lse_i*log2(e)
  float* s_dlt = s_nlse + kStages * 128;                       // [kStages][128]  Delta_i
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_dlt + kStages * 128);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;              // [kStages]
  uint64_t* qdo_empty = qdo_full + kStages;   // [kStages]
  uint64_t* sdp_full = qdo_empty + kStages;
  uint64_t* ds_ready = sdp_full + 1;
  uint64_t* dq_full = ds_ready + 1;
  uint64_t* dq_empty = dq_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_empty + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int h = blockIdx.y, b = blockIdx.z;
  const int k0 = blockIdx.x * 128;
  const int n_q = (p.n + 127) / 128;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&qdo_full[s], 32);
      mbar_init(&qdo_empty[s], 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(ds_ready, 128);
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
        tma_load_4d(sK + a * G::kAtomBytes, &p.tm_k, kv_full, a * G::kAtomCols, k0, h, b, kEvictFirst);
        tma_load_4d(sV + a * G::kAtomBytes, &p.tm_v, kv_full, a * G::kAtomCols, k0, h, b, kEvictFirst);
      }
    }
    const float* lse_bh = p.lse + b * p.l_sb + h * p.l_sh;
    const float* dlt_bh = p.delta + b * p.d_sb + h * p.d_sh;
    for (int i = 0; i < n_q; ++i) {
      const int s = i % kStages;
      if (i >= kStages) mbar_wait(&qdo_empty[s], ((i / kStages) & 1) ^ 1);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = r * 32 + lane;
        const int qi = i * 128 + row;
        const bool ok = qi < p.n;
        s_nlse[s * 128 + row] = ok ? -lse_bh[qi] * kLog2e : -INFINITY;
        s_dlt[s * 128 + row] = ok ? dlt_bh[int64_t(qi) * p.d_sn] : 0.f;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(&qdo_full[s], 2 * G::kTileBytes);
        for (int a = 0; a < G::kAtoms; ++a) {
          tma_load_4d(sQ + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_q, &qdo_full[s], a * G::kAtomCols, i * 128,
                      h, b, kEvictLast);
          tma_load_4d(sdO + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_do, &qdo_full[s], a * G::kAtomCols,
                      i * 128, h, b, kEvictLast);
        }
      } else {
        mbar_arrive(&qdo_full[s]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);
      const uint32_t idesc_g = idesc_bf16_f32(128, D, false, true);   // dV, dK: A from TMEM, B MN-major
      const uint32_t idesc_q = idesc_bf16_f32(128, D, true, true);    // dQ: A, B MN-major
      const uint32_t sKa = smem_u32(sK), sVa = smem_u32(sV), sQa = smem_u32(sQ), sdOa = smem_u32(sdO);
      const uint32_t sdSa = smem_u32(sdS);
      mbar_wait(kv_full, 0);
      tc_fence_after();
      for (int i = 0; i < n_q; ++i) {
        const int s = i % kStages;
        mbar_wait(&qdo_full[s], (i / kStages) & 1);
        tc_fence_after();
        const uint32_t qt = sQa + s * G::kTileBytes, dot = sdOa + s * G::kTileBytes;
        if (C::kDqAliasDp && i > 0) {
          mbar_wait(dq_empty, (i - 1) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tbase + C::kColS, kmajor_desc<D>(sKa, kk), kmajor_desc<D>(qt, kk), idesc_s, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tbase + C::kColDP, kmajor_desc<D>(sVa, kk), kmajor_desc<D>(dot, kk), idesc_s, kk > 0 ? 1u : 0u);
        mma_commit(sdp_full);
        mbar_wait(ds_ready, i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tbase + C::kColDV, tbase + C::kColS + kk * 8, mnmajor_desc<D>(dot, kk), idesc_g,
                 (i > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tbase + C::kColDK, tbase + C::kColDP + kk * 8, mnmajor_desc<D>(qt, kk), idesc_g,
                 (i > 0 || kk > 0) ? 1u : 0u);
        if (!C::kDqAliasDp && i > 0) {
          mbar_wait(dq_empty, (i - 1) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tbase + C::kColDQ, mnmajor_desc<128>(sdSa, kk), mnmajor_desc<D>(sKa, kk), idesc_q,
                 kk > 0 ? 1u : 0u);
        mma_commit(dq_full);
        mma_commit(&qdo_empty[s]);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ elementwise
    const int quad = warp % 4;
    const int j = quad * 32 + lane;  // key row within the tile
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const float c = p.scale_log2;
    uint8_t* ds_row = sdS + j * 128;
    for (int i = 0; i < n_q; ++i) {
      const int s = i % kStages;
      mbar_wait(&qdo_full[s], (i / kStages) & 1);  // lse / Delta visibility
      if (i > 0) mbar_wait(dq_full, (i - 1) & 1);  // dS smem free (dQ(i-1) consumed it)
      mbar_wait(sdp_full, i & 1);
      tc_fence_after();
      const float4* nl4 = reinterpret_cast<const float4*>(s_nlse + s * 128);
      const float4* dl4 = reinterpret_cast<const float4*>(s_dlt + s * 128);
#pragma unroll
      for (int cc = 0; cc < 128; cc += 32) {
        uint32_t rs[32], rd[32];
        tmem_ld32(t_lane + C::kColS + cc, rs);
        tmem_ld32(t_lane + C::kColDP + cc, rd);
        tmem_ld_wait();
        uint32_t pk_p[16], pk_ds[16];
#pragma unroll
        for (int x = 0; x < 32; x += 4) {
          const float4 nl = nl4[(cc + x) / 4];
          const float4 dl = dl4[(cc + x) / 4];
          const float p0 = ex2(fmaf(__uint_as_float(rs[x + 0]), c, nl.x));
          const float p1 = ex2(fmaf(__uint_as_float(rs[x + 1]), c, nl.y));
          const float p2 = ex2(fmaf(__uint_as_float(rs[x + 2]), c, nl.z));
          const float p3 = ex2(fmaf(__uint_as_float(rs[x + 3]), c, nl.w));
          const float d0 = p0 * (__uint_as_float(rd[x + 0]) - dl.x);
          const float d1 = p1 * (__uint_as_float(rd[x + 1]) - dl.y);
          const float d2 = p2 * (__uint_as_float(rd[x + 2]) - dl.z);
          const float d3 = p3 * (__uint_as_float(rd[x + 3]) - dl.w);
          pk_p[x / 2] = pack_bf16x2(p0, p1);
          pk_p[x / 2 + 1] = pack_bf16x2(p2, p3);
          pk_ds[x / 2] = pack_bf16x2(d0, d1);
          pk_ds[x / 2 + 1] = pack_bf16x2(d2, d3);
        }
        tmem_st16(t_lane + C::kColS + cc / 2, pk_p);
        tmem_st16(t_lane + C::kColDP + cc / 2, pk_ds);
        // dS^T row j, query columns cc..cc+31 -> SW128 atom cc/64, chunks (cc%64)/8 .. +3
        uint8_t* atom = ds_row + (cc / 64) * (128 * 128);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          const int chunk = (((cc % 64) / 8) + qd) ^ (j & 7);
          *reinterpret_cast<uint4*>(atom + chunk * 16) =
              make_uint4(pk_ds[4 * qd], pk_ds[4 * qd + 1], pk_ds[4 * qd + 2], pk_ds[4 * qd + 3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(ds_ready);
    }
    // -------------------------------------------------------- dK, dV epilogue
    mbar_wait(dq_full, (n_q - 1) & 1);
    tc_fence_after();
    const int krow = k0 + j;
    const bool valid = krow < p.n;
    __nv_bfloat16* dv_row = reinterpret_cast<__nv_bfloat16*>(p.dv.base) + b * p.dv.sb + h * p.dv.sh + int64_t(krow) * p.dv.sn;
    __nv_bfloat16* dk_row = reinterpret_cast<__nv_bfloat16*>(p.dk.base) + b * p.dk.sb + h * p.dk.sh + int64_t(krow) * p.dk.sn;
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
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const int n_pad = n_q * 128;
    float* dq_bh = p.dq_acc + (int64_t(b) * p.heads + h) * n_pad * D;
    for (int i = 0; i < n_q; ++i) {
      mbar_wait(dq_full, i & 1);
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
      float* dst = dq_bh + int64_t(i * 128 + r) * D;
#pragma unroll
      for (int e = 0; e < D; e += 4) red_add_v4(dst + e, acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tbase);
}

template <int D>
cudaError_t launch_bwd_impl(const BwdParams& p, int B, int heads, cudaStream_t stream) {
  using C = BwdCfg<D>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((p.n + 127) / 128, heads, B);
  attn_bwd_kernel<D><<<grid, C::kThreads, C::kSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_bwd(const BwdParams& p, int D, int B, int heads, cudaStream_t stream) {
  // D <= 64: the persistent warp-specialised kernel (attn_bwd_ws.cu); UA_BWD_KERNEL=v1 forces
  // this file's kernel (kept for D = 128 and for A/B measurements).
  static const bool force_v1 = [] {
    const char* e = std::getenv("UA_BWD_KERNEL");
    return e != nullptr && std::strcmp(e, "v1") == 0;
  }();
  if (!force_v1) return launch_attn_bwd_ws(p, D, stream);
  if (p.n_kv != p.n || p.kv_f32 || D == 72) return cudaErrorInvalidValue;  // v1: square, bf16 out, D in {32, 64, 128}
  switch (D) {
    case 32: return launch_bwd_impl<32>(p, B, heads, stream);
    case 64: return launch_bwd_impl<64>(p, B, heads, stream);
    case 128: return launch_bwd_impl<128>(p, B, heads, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ua
