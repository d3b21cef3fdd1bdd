// probe_tcgen05.cu — isolated checks of the tcgen05 / TMA / descriptor
// encodings the attention kernels rely on.  Each probe is one CTA computing a
// small GEMM that tests/… compare against torch on the GPU.
//   probe_qk : S[128][128] = Q[128][D] K[128][D]^T   (SS, A,B K-major SW128)
//   probe_pv_ts : O[128][D] = P[128][128] V[128][D]   (TS: P in TMEM, V MN-major)
//   probe_pv_ss : same with P written to smem by threads (manual SW128 K-major)
//   probe_at_b : C[128][D] = X[128][128]^T Y[128][D] (SS, A MN-major via TMA)
//   probe_at_b_manual : same with X^T rows written by threads (manual SW128 MN-major)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../../paper_2405_15780_b200/csrc/kernels/sm100_ptx.cuh"
#include "../../paper_2405_15780_b200/csrc/tma_host.h"

using namespace ua;

struct __align__(8) Bars {
  uint64_t tma;
  uint64_t mma;
  uint32_t tmem_base;
};

// Byte offset of element (r, c) inside a [rows][64] bf16 SW128 atom column.
__device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t c) {
  uint32_t chunk = (c >> 3) ^ (r & 7);
  return r * 128 + chunk * 16 + (c & 7) * 2;
}

__device__ void read_tmem_rows(uint32_t tbase, int ncols, float* out, int ld) {
  int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c = 0; c < ncols; c += 32) {
    uint32_t r[32];
    tmem_ld32(tbase + ((w * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) out[(w * 32 + lane) * ld + c + i] = __uint_as_float(r[i]);
  }
}

__global__ void __launch_bounds__(128) k_qk(const __grid_constant__ CUtensorMap tq,
                                            const __grid_constant__ CUtensorMap tk, float* s, int D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = smem + 32768;
  Bars* bars = reinterpret_cast<Bars*>(smem + 65536);
  if (threadIdx.x == 0) {
    mbar_init(&bars->tma, 1);
    mbar_init(&bars->mma, 1);
    fence_mbar_init();
  }
  if (threadIdx.x / 32 == 0) tmem_alloc<256>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = bars->tmem_base;
  if (threadIdx.x == 0) {
    int natoms = D / 64;
    mbar_arrive_expect_tx(&bars->tma, 2 * 128 * D * 2);
    for (int a = 0; a < natoms; ++a) {
      tma_load_4d(sQ + a * 16384, &tq, &bars->tma, a * 64, 0, 0, 0, kEvictNormal);
      tma_load_4d(sK + a * 16384, &tk, &bars->tma, a * 64, 0, 0, 0, kEvictNormal);
    }
    mbar_wait(&bars->tma, 0);
    tc_fence_after();
    uint32_t idesc = idesc_bf16_f32(128, 128, false, false);
    for (int k = 0; k < D / 16; ++k) {
      uint32_t off = (k / 4) * 16384 + (k % 4) * 32;
      mma_ss(tb, sdesc_sw128(smem_u32(sQ) + off, 16, 1024), sdesc_sw128(smem_u32(sK) + off, 16, 1024), idesc,
             k > 0);
    }
    mma_commit(&bars->mma);
  }
  __syncwarp();
  mbar_wait(&bars->mma, 0);
  tc_fence_after();
  read_tmem_rows(tb, 128, s, 128);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x / 32 == 0) tmem_free<256>(tb);
}

// mode 0: P via TMEM (TS).  mode 1: P via smem (SS, manual swizzle).
__global__ void __launch_bounds__(128) k_pv(const __nv_bfloat16* P, const __grid_constant__ CUtensorMap tv,
                                            float* o, int D, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sV = smem;
  uint8_t* sP = smem + 32768;
  Bars* bars = reinterpret_cast<Bars*>(smem + 65536);
  if (threadIdx.x == 0) {
    mbar_init(&bars->tma, 1);
    mbar_init(&bars->mma, 1);
    fence_mbar_init();
  }
  if (threadIdx.x / 32 == 0) tmem_alloc<256>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = bars->tmem_base;
  const uint32_t pcol = 128, ocol = 0;
  int row = threadIdx.x, w = threadIdx.x / 32;
  if (mode == 0) {
    uint32_t packed[64];
    for (int c = 0; c < 64; ++c) {
      __nv_bfloat162 v;
      v.x = P[row * 128 + 2 * c];
      v.y = P[row * 128 + 2 * c + 1];
      packed[c] = *reinterpret_cast<uint32_t*>(&v);
    }
    tmem_st32(tb + ((w * 32) << 16) + pcol, packed);
    tmem_st32(tb + ((w * 32) << 16) + pcol + 32, packed + 32);
    tmem_st_wait();
  } else {
    for (int c = 0; c < 128; ++c)
      *reinterpret_cast<__nv_bfloat16*>(sP + (c / 64) * 16384 + sw128_off(row, c % 64)) = P[row * 128 + c];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    int natoms = D / 64;
    mbar_arrive_expect_tx(&bars->tma, 128 * D * 2);
    for (int a = 0; a < natoms; ++a) tma_load_4d(sV + a * 16384, &tv, &bars->tma, a * 64, 0, 0, 0, kEvictNormal);
    mbar_wait(&bars->tma, 0);
    tc_fence_after();
    uint32_t idesc = idesc_bf16_f32(128, D, false, true);
    for (int kk = 0; kk < 8; ++kk) {
      uint64_t bdesc = sdesc_sw128(smem_u32(sV) + kk * 2048, 16384, 1024);
      if (mode == 0) {
        mma_ts(tb + ocol, tb + pcol + kk * 8, bdesc, idesc, kk > 0);
      } else {
        uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
        mma_ss(tb + ocol, sdesc_sw128(smem_u32(sP) + off, 16, 1024), bdesc, idesc, kk > 0);
      }
    }
    mma_commit(&bars->mma);
  }
  __syncwarp();
  mbar_wait(&bars->mma, 0);
  tc_fence_after();
  read_tmem_rows(tb + ocol, D, o, D);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x / 32 == 0) tmem_free<256>(tb);
}

// C[128][D] = X^T Y, X [128 k][128 m] (m contiguous), Y [128 k][D] (n contiguous).
// mode 0: X via TMA (SW128 boxes of 64 m).  mode 1: X rows written by threads.
__global__ void __launch_bounds__(128) k_atb(const __nv_bfloat16* X, const __grid_constant__ CUtensorMap tx,
                                             const __grid_constant__ CUtensorMap ty, float* c, int D, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sX = smem;
  uint8_t* sY = smem + 32768;
  Bars* bars = reinterpret_cast<Bars*>(smem + 65536);
  if (threadIdx.x == 0) {
    mbar_init(&bars->tma, 1);
    mbar_init(&bars->mma, 1);
    fence_mbar_init();
  }
  if (threadIdx.x / 32 == 0) tmem_alloc<256>(&bars->tmem_base);
  if (mode == 1) {
    int r = threadIdx.x;  // row = k index
    for (int m = 0; m < 128; ++m)
      *reinterpret_cast<__nv_bfloat16*>(sX + (m / 64) * 16384 + sw128_off(r, m % 64)) = X[r * 128 + m];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = bars->tmem_base;
  if (threadIdx.x == 0) {
    uint32_t bytes = 128 * D * 2 + (mode == 0 ? 128 * 128 * 2 : 0);
    mbar_arrive_expect_tx(&bars->tma, bytes);
    if (mode == 0)
      for (int a = 0; a < 2; ++a) tma_load_4d(sX + a * 16384, &tx, &bars->tma, a * 64, 0, 0, 0, kEvictNormal);
    for (int a = 0; a < D / 64; ++a) tma_load_4d(sY + a * 16384, &ty, &bars->tma, a * 64, 0, 0, 0, kEvictNormal);
    mbar_wait(&bars->tma, 0);
    tc_fence_after();
    uint32_t idesc = idesc_bf16_f32(128, D, true, true);
    for (int kk = 0; kk < 8; ++kk) {
      uint64_t adesc = sdesc_sw128(smem_u32(sX) + kk * 2048, 16384, 1024);
      uint64_t bdesc = sdesc_sw128(smem_u32(sY) + kk * 2048, 16384, 1024);
      mma_ss(tb, adesc, bdesc, idesc, kk > 0);
    }
    mma_commit(&bars->mma);
  }
  __syncwarp();
  mbar_wait(&bars->mma, 0);
  tc_fence_after();
  read_tmem_rows(tb, D, c, D);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x / 32 == 0) tmem_free<256>(tb);
}

static bool map2d(CUtensorMap* m, const void* p, int rows, int cols) {
  uint64_t dims[4] = {(uint64_t)cols, (uint64_t)rows, 1, 1};
  uint64_t str[3] = {(uint64_t)cols * 2, (uint64_t)cols * 2 * rows, (uint64_t)cols * 2 * rows};
  return make_tmap_bf16_4d(m, p, dims, str, 64, rows);
}

extern "C" int probe_qk(const void* q, const void* k, float* s, int D) {
  CUtensorMap tq, tk;
  if (!map2d(&tq, q, 128, D) || !map2d(&tk, k, 128, D)) return -1;
  cudaFuncSetAttribute(k_qk, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k_qk<<<1, 128, 70000>>>(tq, tk, s, D);
  return (int)cudaDeviceSynchronize();
}
extern "C" int probe_pv(const void* P, const void* v, float* o, int D, int mode) {
  CUtensorMap tv;
  if (!map2d(&tv, v, 128, D)) return -1;
  cudaFuncSetAttribute(k_pv, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k_pv<<<1, 128, 70000>>>((const __nv_bfloat16*)P, tv, o, D, mode);
  return (int)cudaDeviceSynchronize();
}
extern "C" int probe_atb(const void* x, const void* y, float* c, int D, int mode) {
  CUtensorMap tx, ty;
  if (!map2d(&tx, x, 128, 128) || !map2d(&ty, y, 128, D)) return -1;
  cudaFuncSetAttribute(k_atb, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k_atb<<<1, 128, 70000>>>((const __nv_bfloat16*)x, tx, ty, c, D, mode);
  return (int)cudaDeviceSynchronize();
}
