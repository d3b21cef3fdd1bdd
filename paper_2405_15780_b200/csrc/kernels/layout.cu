// layout.cu — HBM-bound permutation and elementwise kernels around the
// all-to-all (sequence shards <-> head shards).
//
// All kernels move 16-byte vectors with 64-bit indexing; one row = D bf16
// (64..256 B, always a whole number of vectors).  Reads are in source order
// (pack) or writes in destination order (unpack) so one side is perfectly
// coalesced and the other moves contiguous H_l*D*2-byte runs.
#include <cuda_bf16.h>

#include <cstdint>

#include "attn_kernels.h"

namespace ua {

namespace {

struct Ptrs4 {
  const uint4* src[4];
  uint4* dst[4];
};

// send chunk j <- heads [j*Hl, (j+1)*Hl) of every local token (+ fused Delta).
template <int VPR>  // 16-B vectors per row = D / 8
__global__ void __launch_bounds__(256) pack_kernel(Ptrs4 ptrs, int ntensors, int64_t B, int64_t Nl, int H, int Hl,
                                                   const uint4* __restrict__ dout, const uint4* __restrict__ out,
                                                   float* __restrict__ delta) {
  const int64_t total = B * Nl * H * VPR;
  const int lane = threadIdx.x % 32;
  const int64_t warp0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int64_t nwarps = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t base = warp0 * 32; base < total; base += nwarps * 32) {
    const int64_t v = base + lane;
    const bool ok = v < total;
    const int64_t r = v / VPR;                 // source row (b, t, h)
    const int dv = int(v % VPR);
    const int h = int(r % H);
    const int64_t t = (r / H) % Nl;
    const int64_t b = r / (int64_t(H) * Nl);
    const int j = h / Hl, hp = h % Hl;
    const int64_t drow = ((int64_t(j) * Nl + t) * B + b) * Hl + hp;
    if (ok) {
#pragma unroll 4
      for (int w = 0; w < ntensors; ++w) ptrs.dst[w][drow * VPR + dv] = ptrs.src[w][v];
    }
    if (delta != nullptr) {
      float acc = 0.f;
      if (ok) {
        uint4 a = dout[v], o = out[v];
        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
        const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&o);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float2 fa = __bfloat1622float2(a2[i]), fo = __bfloat1622float2(o2[i]);
          acc = fmaf(fa.x, fo.x, acc);
          acc = fmaf(fa.y, fo.y, acc);
        }
      }
#pragma unroll
      for (int off = VPR / 2; off > 0; off /= 2) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (ok && dv == 0) delta[drow] = acc;
    }
  }
}

// Delta = sum_d dO.O in fp32 for one (b, t, h) row per thread (head dims whose
// row is not a power-of-two number of 16-B vectors, e.g. D = 72); same
// destination index as pack_kernel's fused Delta.
__global__ void __launch_bounds__(256) delta_kernel(int64_t B, int64_t Nl, int H, int Hl, int vpr,
                                                    const uint4* __restrict__ dout, const uint4* __restrict__ out,
                                                    float* __restrict__ delta) {
  const int64_t rows = B * Nl * H;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    const int h = int(r % H);
    const int64_t t = (r / H) % Nl;
    const int64_t b = r / (int64_t(H) * Nl);
    const int j = h / Hl, hp = h % Hl;
    float acc = 0.f;
    for (int i = 0; i < vpr; ++i) {
      uint4 a = dout[r * vpr + i], o = out[r * vpr + i];
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&o);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 fa = __bfloat1622float2(a2[k]), fo = __bfloat1622float2(o2[k]);
        acc = fmaf(fa.x, fo.x, acc);
        acc = fmaf(fa.y, fo.y, acc);
      }
    }
    delta[((int64_t(j) * Nl + t) * B + b) * Hl + hp] = acc;
  }
}

template <int VPR>
__global__ void __launch_bounds__(256) unpack_kernel(Ptrs4 ptrs, int ntensors, int64_t B, int64_t Nl, int H, int Hl) {
  const int64_t total = B * Nl * H * VPR;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < total; v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = v / VPR;                 // destination row (b, t, h)
    const int dv = int(v % VPR);
    const int h = int(r % H);
    const int64_t t = (r / H) % Nl;
    const int64_t b = r / (int64_t(H) * Nl);
    const int s = h / Hl, hp = h % Hl;
    const int64_t srow = ((int64_t(s) * Nl + t) * B + b) * Hl + hp;
#pragma unroll 4
    for (int w = 0; w < ntensors; ++w) ptrs.dst[w][v] = ptrs.src[w][srow * VPR + dv];
  }
}

// src rows (bh, n) at (bh * n_stride + n) * D, n < N  ->  bf16 view (scaled).
__global__ void __launch_bounds__(256) f32_to_bf16_view_kernel(const float4* __restrict__ src, ViewArg dst, int64_t N,
                                                               int64_t n_stride, int heads, int D, float scale,
                                                               int64_t total_vec) {
  const int vpr = D / 8;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < total_vec;
       v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = v / vpr;                  // (bh, n)
    const int dv = int(v % vpr);
    const int64_t n = r % N, bh = r / N;
    const int64_t b = bh / heads, h = bh % heads;
    const int64_t so = ((bh * n_stride + n) * D + dv * 8) / 4;
    float4 x0 = src[so], x1 = src[so + 1];
    __nv_bfloat162 o[4] = {__floats2bfloat162_rn(x0.x * scale, x0.y * scale),
                           __floats2bfloat162_rn(x0.z * scale, x0.w * scale),
                           __floats2bfloat162_rn(x1.x * scale, x1.y * scale),
                           __floats2bfloat162_rn(x1.z * scale, x1.w * scale)};
    __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(dst.base) + b * dst.sb + h * dst.sh + n * dst.sn + dv * 8;
    *reinterpret_cast<uint4*>(base) = *reinterpret_cast<uint4*>(o);
  }
}

// One warp per row: lse = logaddexp(lse_a, lse_b); O = wa O_a + wb O_b.
__global__ void __launch_bounds__(256) lse_merge_kernel(float* __restrict__ o_a, float* __restrict__ lse_a,
                                                        const float* __restrict__ o_b, const float* __restrict__ lse_b,
                                                        int64_t rows, int D) {
  const int lane = threadIdx.x % 32;
  const int64_t nwarps = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; r < rows; r += nwarps) {
    const float la = lse_a[r], lb = lse_b[r];
    const float mx = fmaxf(la, lb);
    const float l = mx + log1pf(expf(fminf(la, lb) - mx));
    const float wa = expf(la - l), wb = expf(lb - l);
    for (int d = lane; d < D; d += 32) o_a[r * D + d] = wa * o_a[r * D + d] + wb * o_b[r * D + d];
    __syncwarp();
    if (lane == 0) lse_a[r] = l;
  }
}

__global__ void __launch_bounds__(256) bwd_prep_kernel(const float* __restrict__ lse, int64_t l_sh, int64_t l_sb,
                                                       const float* __restrict__ delta, int64_t d_sn, int64_t d_sh,
                                                       int64_t d_sb, float2* __restrict__ lsed, int heads, int64_t N,
                                                       int64_t n_pad, int64_t total) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n = i % n_pad, bh = i / n_pad;
    const int64_t b = bh / heads, h = bh % heads;
    float nl = -INFINITY, nd = 0.f;
    if (n < N) {
      nl = -lse[b * l_sb + h * l_sh + n] * 1.4426950408889634f;
      nd = -delta[b * d_sb + h * d_sh + n * d_sn];
    }
    // planar per 128-row tile: [128 x (-lse*log2e)][128 x (-Delta)]
    float* tile = reinterpret_cast<float*>(lsed) + (bh * n_pad + (n / 128) * 128) * 2;
    tile[n % 128] = nl;
    tile[128 + n % 128] = nd;
  }
}

int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = 148 * 16;  // 16 resident 256-thread blocks per SM
  return int(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

cudaError_t launch_pack(const void* const* src, void* const* dst, int ntensors, int64_t B, int64_t Nl, int H, int D,
                        int P, const void* dout, const void* out, float* delta_dst, cudaStream_t stream) {
  if (ntensors < 0 || ntensors > 4 || D % 8 != 0) return cudaErrorInvalidValue;
  Ptrs4 ptrs{};
  for (int w = 0; w < ntensors; ++w) {
    ptrs.src[w] = static_cast<const uint4*>(src[w]);
    ptrs.dst[w] = static_cast<uint4*>(dst[w]);
  }
  const int Hl = H / P;
  const int64_t total = B * Nl * H * (D / 8);
  const int grid = grid_for(total, 256);
  const uint4* dv = static_cast<const uint4*>(dout);
  const uint4* ov = static_cast<const uint4*>(out);
  switch (D / 8) {
    case 4: pack_kernel<4><<<grid, 256, 0, stream>>>(ptrs, ntensors, B, Nl, H, Hl, dv, ov, delta_dst); break;
    case 8: pack_kernel<8><<<grid, 256, 0, stream>>>(ptrs, ntensors, B, Nl, H, Hl, dv, ov, delta_dst); break;
    case 16: pack_kernel<16><<<grid, 256, 0, stream>>>(ptrs, ntensors, B, Nl, H, Hl, dv, ov, delta_dst); break;
    case 9:  // D = 72: rows of 9 vectors straddle warps, Delta in its own pass
      if (ntensors > 0) pack_kernel<9><<<grid, 256, 0, stream>>>(ptrs, ntensors, B, Nl, H, Hl, nullptr, nullptr, nullptr);
      if (delta_dst != nullptr)
        delta_kernel<<<grid_for(B * Nl * H, 256), 256, 0, stream>>>(B, Nl, H, Hl, 9, dv, ov, delta_dst);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_unpack(const void* const* src, void* const* dst, int ntensors, int64_t B, int64_t Nl, int H,
                          int D, int P, cudaStream_t stream) {
  if (ntensors < 1 || ntensors > 4 || D % 8 != 0) return cudaErrorInvalidValue;
  Ptrs4 ptrs{};
  for (int w = 0; w < ntensors; ++w) {
    ptrs.src[w] = static_cast<const uint4*>(src[w]);
    ptrs.dst[w] = static_cast<uint4*>(dst[w]);
  }
  const int Hl = H / P;
  const int64_t total = B * Nl * H * (D / 8);
  const int grid = grid_for(total, 256);
  switch (D / 8) {
    case 4: unpack_kernel<4><<<grid, 256, 0, stream>>>(ptrs, ntensors, B, Nl, H, Hl); break;
    case 8: unpack_kernel<8><<<grid, 256, 0, stream>>>(ptrs, ntensors, B, Nl, H, Hl); break;
    case 16: unpack_kernel<16><<<grid, 256, 0, stream>>>(ptrs, ntensors, B, Nl, H, Hl); break;
    case 9: unpack_kernel<9><<<grid, 256, 0, stream>>>(ptrs, ntensors, B, Nl, H, Hl); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_dq_finalize(const float* dq_acc, ViewArg dq, int64_t B, int64_t N, int heads, int D, float scale,
                               cudaStream_t stream) {
  const int64_t total_vec = B * heads * N * (D / 8);
  const int64_t n_pad = (N + 127) / 128 * 128;
  f32_to_bf16_view_kernel<<<grid_for(total_vec, 256), 256, 0, stream>>>(reinterpret_cast<const float4*>(dq_acc), dq,
                                                                         N, n_pad, heads, D, scale, total_vec);
  return cudaGetLastError();
}

cudaError_t launch_f32_to_view(const float* src, ViewArg dst, int64_t B, int64_t N, int heads, int D,
                               cudaStream_t stream) {
  const int64_t total_vec = B * heads * N * (D / 8);
  f32_to_bf16_view_kernel<<<grid_for(total_vec, 256), 256, 0, stream>>>(reinterpret_cast<const float4*>(src), dst, N,
                                                                         N, heads, D, 1.0f, total_vec);
  return cudaGetLastError();
}

cudaError_t launch_bwd_prep(const float* lse, int64_t l_sh, int64_t l_sb, const float* delta, int64_t d_sn,
                            int64_t d_sh, int64_t d_sb, float2* lsed, int64_t B, int heads, int64_t N,
                            cudaStream_t stream) {
  const int64_t n_pad = (N + 127) / 128 * 128;
  const int64_t total = B * heads * n_pad;
  bwd_prep_kernel<<<grid_for(total, 256), 256, 0, stream>>>(lse, l_sh, l_sb, delta, d_sn, d_sh, d_sb, lsed, heads, N,
                                                            n_pad, total);
  return cudaGetLastError();
}

cudaError_t launch_lse_merge(float* o_a, float* lse_a, const float* o_b, const float* lse_b, int64_t rows, int D,
                             cudaStream_t stream) {
  lse_merge_kernel<<<grid_for(rows * 32, 256), 256, 0, stream>>>(o_a, lse_a, o_b, lse_b, rows, D);
  return cudaGetLastError();
}

}  // namespace ua
