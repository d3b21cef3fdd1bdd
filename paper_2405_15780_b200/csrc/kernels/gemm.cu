// gemm.cu — the attention layer's projection GEMMs on the 5th-generation tensor
// cores (§5.4, §6.1): bf16 operands staged
// by TMA into 128B-swizzled shared memory, tcgen05.mma issued by one thread,
// fp32 accumulation in TMEM, epilogue TMEM -> registers -> global.
//
//   C[M][N] = sum_{s < nseg} op(A_s) op(B_s)          (fp32 accumulate)
//     A_s K-major : stored [M][K] (row-major)          op(A) = A
//     A_s MN-major: stored [K][M]                      op(A) = A^T   (weight gradients dW = g^T x)
//     B_s K-major : stored [N][K]                      op(B) = B^T   (y = x W^T)
//     B_s MN-major: stored [K][N]                      op(B) = B     (dx = g W)
//   C bf16 or fp32, row-major [M][N] with leading dimension ldc.
// Segments concatenate the reduction dimension over separate buffers, e.g.
// dx = dq Wq + dk Wk + dv Wv accumulates in one TMEM tile and is rounded once.
//
// CTA tile 128 x BN (BN = 256, or 128 for narrow N) x 64, kStages-deep smem
// ring, warp roles: 0 TMA producer, 1 MMA issuer (+ TMEM owner), 4-7 epilogue
// (thread = output row, TMEM lane).  Two CTAs per SM (96 / 72 KB of smem each)
// so one CTA's epilogue overlaps the other's main loop.
#include <cuda_bf16.h>

#include <cstdint>

#include "attn_common.cuh"
#include "attn_kernels.h"

namespace ua {

namespace {

template <int BN>
struct GemmCfg {
  static constexpr int kBM = 128, kBK = 64;
  static constexpr int kStages = 2;
  static constexpr int kABytes = kBM * kBK * 2;   // 16 KB: [128][64] K-major or 2 x [64 K][64 M] MN-major
  static constexpr int kBBytes = BN * kBK * 2;    // 32 KB (BN = 256)
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + 256;
  static constexpr int kThreads = 256;
};

template <int BN, bool kAmn, bool kBmn>
__global__ void __launch_bounds__(256, 2) gemm_kernel(const __grid_constant__ GemmParams p) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* full = bars;                 // [kStages]
  uint64_t* empty = bars + C::kStages;   // [kStages]
  uint64_t* acc_full = bars + 2 * C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  auto sA = [&](int s) { return smem + s * C::kStageBytes; };
  auto sB = [&](int s) { return smem + s * C::kStageBytes + C::kABytes; };

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * C::kBM;
  const int nk_seg = (p.K + C::kBK - 1) / C::kBK;
  const int nk = nk_seg * p.nseg;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<BN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tacc = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::kStages;
        if (kb >= C::kStages) mbar_wait(&empty[s], ((kb / C::kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], C::kStageBytes);
        const int seg = kb / nk_seg, k0 = (kb % nk_seg) * C::kBK;
        if constexpr (kAmn) {   // [64 K rows][64 M] atoms, two along M
          for (int a = 0; a < 2; ++a) tma_load_2d(sA(s) + a * 8192, &p.tm_a[seg], &full[s], m0 + 64 * a, k0);
        } else {
          tma_load_2d(sA(s), &p.tm_a[seg], &full[s], k0, m0);
        }
        if constexpr (kBmn) {   // [64 K rows][64 N] atoms along N
          for (int a = 0; a < BN / 64; ++a) tma_load_2d(sB(s) + a * 8192, &p.tm_b[seg], &full[s], n0 + 64 * a, k0);
        } else {
          tma_load_2d(sB(s), &p.tm_b[seg], &full[s], k0, n0);
        }
      }
    }
  } else if (warp == 1) {  // ---------------------------------------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, BN, kAmn, kBmn);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::kStages;
        mbar_wait(&full[s], (kb / C::kStages) & 1);
        tc_fence_after();
        const uint32_t a = smem_u32(sA(s)), b = smem_u32(sB(s));
#pragma unroll
        for (int kk = 0; kk < C::kBK / 16; ++kk) {
          const uint64_t ad = kAmn ? mnmajor_desc_r<128, 64>(a, kk) : kmajor_desc_r<64, 128>(a, kk);
          const uint64_t bd = kBmn ? mnmajor_desc_r<BN, 64>(b, kk) : kmajor_desc_r<64, BN>(b, kk);
          mma_ss(tacc, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(acc_full);
    }
    __syncwarp();
  } else if (warp >= 4) {  // ---------------------------------------------- epilogue
    const int quad = warp % 4;
    const int row = m0 + quad * 32 + lane;
    const uint32_t t_lane = tacc + (uint32_t(quad * 32) << 16);
    mbar_wait(acc_full, 0);
    tc_fence_after();
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(t_lane + c0, r);
      tmem_ld_wait();
      const int col = n0 + c0;
      if (row >= p.M || col >= p.N) continue;
      const bool full_chunk = col + 32 <= p.N;
      if (p.c_f32) {
        float* dst = static_cast<float*>(p.c) + int64_t(row) * p.ldc + col;
        if (full_chunk) {
#pragma unroll
          for (int x = 0; x < 32; x += 4)
            *reinterpret_cast<float4*>(dst + x) = make_float4(__uint_as_float(r[x]), __uint_as_float(r[x + 1]),
                                                              __uint_as_float(r[x + 2]), __uint_as_float(r[x + 3]));
        } else {
          for (int x = 0; x < 32 && col + x < p.N; ++x) dst[x] = __uint_as_float(r[x]);
        }
      } else {
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.c) + int64_t(row) * p.ldc + col;
        if (full_chunk) {
#pragma unroll
          for (int x = 0; x < 32; x += 8)
            *reinterpret_cast<uint4*>(dst + x) =
                make_uint4(pack_bf16x2(__uint_as_float(r[x]), __uint_as_float(r[x + 1])),
                           pack_bf16x2(__uint_as_float(r[x + 2]), __uint_as_float(r[x + 3])),
                           pack_bf16x2(__uint_as_float(r[x + 4]), __uint_as_float(r[x + 5])),
                           pack_bf16x2(__uint_as_float(r[x + 6]), __uint_as_float(r[x + 7])));
        } else {
          for (int x = 0; x < 32 && col + x < p.N; ++x) dst[x] = __float2bfloat16_rn(__uint_as_float(r[x]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<BN>(tacc);
}

template <int BN, bool kAmn, bool kBmn>
cudaError_t launch_gemm_impl(const GemmParams& p, cudaStream_t stream) {
  using C = GemmCfg<BN>;
  cudaError_t e = set_max_smem(gemm_kernel<BN, kAmn, kBmn>, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  dim3 grid((p.N + BN - 1) / BN, (p.M + C::kBM - 1) / C::kBM);
  gemm_kernel<BN, kAmn, kBmn><<<grid, C::kThreads, C::kSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

int gemm_bn(int N) { return N % 256 == 0 ? 256 : 128; }

cudaError_t launch_gemm(const GemmParams& p, cudaStream_t stream) {
  if (p.nseg < 1 || p.nseg > kGemmMaxSeg || p.M < 1 || p.N < 1 || p.K < 1) return cudaErrorInvalidValue;
  const int bn = gemm_bn(p.N);
#define UA_GEMM_CASE(BN_, AMN, BMN) \
  if (bn == BN_ && p.a_mn == AMN && p.b_mn == BMN) return launch_gemm_impl<BN_, AMN, BMN>(p, stream);
  UA_GEMM_CASE(256, false, false)   // y = x W^T
  UA_GEMM_CASE(256, false, true)    // dx = g W
  UA_GEMM_CASE(256, true, true)     // dW = g^T x
  UA_GEMM_CASE(128, false, false)
  UA_GEMM_CASE(128, false, true)
  UA_GEMM_CASE(128, true, true)
#undef UA_GEMM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace ua
