// peer.cu — the all-to-all of PAPER.md P:165 done with NVLink peer stores
// instead of NCCL: kernels write each element straight into
// the receive buffer of the GPU that needs it (CUDA IPC mappings of
// library-owned buffers), then raise a system-scope flag on every peer.
//
//   pack_push   : sequence shard -> every destination rank's head-shard
//                 receive buffer (fwd: q,k,v; bwd: q,k,v,dO + Delta)
//   signal      : flags[peer][slot][rank] = step   (release, system scope)
//   wait_copy   : spin until flags[slot][*] >= step on this GPU, then
//                 optionally copy a received buffer into the caller's tensor
//   finalize_push: dq = bf16(scale * dq_acc) into the token owner's buffer
// The attention kernels' epilogues write O (fwd) and dK, dV (bwd) rows into
// the token owner's buffer directly (FwdParams::o_peer, BwdParams::dk_peer).
#include <cuda_bf16.h>

#include <cstdint>

#include "attn_kernels.h"

namespace ua {

namespace {

__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Source row (b, t, h) of the local shard [B][Nl][H][D] goes to rank j = h / Hl,
// row ((r*Nl + t)*B + b)*Hl + h%Hl of that rank's receive tensor [N][B][Hl][D].
template <int VPR>
__global__ void __launch_bounds__(256) pack_push_kernel(PeerPack pk, int64_t B, int64_t Nl, int H, int Hl, int rank,
                                                        int64_t tensor_vecs) {
  const int64_t total = B * Nl * H * VPR;
  const int lane = threadIdx.x % 32;
  const int64_t warp0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int64_t nwarps = int64_t(gridDim.x) * blockDim.x / 32;
  for (int64_t base = warp0 * 32; base < total; base += nwarps * 32) {
    const int64_t v = base + lane;
    const bool ok = v < total;
    const int64_t r = v / VPR;
    const int dv = int(v % VPR);
    const int h = int(r % H);
    const int64_t t = (r / H) % Nl;
    const int64_t b = r / (int64_t(H) * Nl);
    const int j = h / Hl, hp = h % Hl;
    const int64_t drow = ((int64_t(rank) * Nl + t) * B + b) * Hl + hp;
    uint4* dst = static_cast<uint4*>(pk.dst[j]);
    if (ok) {
#pragma unroll 4
      for (int w = 0; w < pk.ntensors; ++w)
        dst[int64_t(w) * tensor_vecs + drow * VPR + dv] = static_cast<const uint4*>(pk.src[w])[v];
    }
    if (pk.dout != nullptr) {  // Delta = rowsum(dO * O), fp32, into the destination's Delta block
      float acc = 0.f;
      if (ok) {
        uint4 a = static_cast<const uint4*>(pk.dout)[v], o = static_cast<const uint4*>(pk.out)[v];
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
      if (ok && dv == 0) {
        float* dd = reinterpret_cast<float*>(static_cast<uint4*>(pk.dst[j]) + int64_t(pk.ntensors) * tensor_vecs);
        dd[drow] = acc;
      }
    }
  }
}

__global__ void signal_kernel(PeerFlags f, int slot, int rank, int P, int64_t step) {
  __threadfence_system();
  const int p = threadIdx.x;
  if (p < P) st_release_sys(f.peer[p] + slot * kMaxPeers + rank, step);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// A peer that never raises its flag (it failed validation, died, or diverged)
// must not hang this GPU: after kPeerWaitNs the wait gives up, records the
// timeout in the ctx's host-mapped error word and skips its copy; the next
// library call on that ctx returns UA_ERR_CUDA.
constexpr uint64_t kPeerWaitNs = 60ull * 1000 * 1000 * 1000;

__global__ void __launch_bounds__(256) wait_copy_kernel(const int64_t* flags, int slot, int P, int64_t step,
                                                        const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                        int64_t n_vec, volatile int* err) {
  __shared__ int timed_out;
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  if (threadIdx.x < P) {
    const int64_t* f = flags + slot * kMaxPeers + threadIdx.x;
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(f) < step) {
      if (globaltimer_ns() - t0 > kPeerWaitNs) {
        timed_out = 1;
        if (err != nullptr) *err = 1;
        break;
      }
    }
  }
  __syncthreads();
  if (timed_out) return;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_vec; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// dq_acc [B*Hl][N_pad][D] fp32 (head-local) -> bf16 rows of the owner's
// [B][Nl][H][D] buffer (global head = h0 + h).
__global__ void __launch_bounds__(256) finalize_push_kernel(const float4* __restrict__ src, PeerOut o, int64_t N,
                                                            int64_t n_stride, int heads, int D, float scale,
                                                            int64_t total_vec) {
  const int vpr = D / 8;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < total_vec;
       v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = v / vpr;
    const int dv = int(v % vpr);
    const int64_t n = r % N, bh = r / N;
    const int64_t b = bh / heads, h = bh % heads;
    const int64_t so = ((bh * n_stride + n) * D + dv * 8) / 4;
    float4 x0 = src[so], x1 = src[so + 1];
    __nv_bfloat162 ov[4] = {__floats2bfloat162_rn(x0.x * scale, x0.y * scale),
                            __floats2bfloat162_rn(x0.z * scale, x0.w * scale),
                            __floats2bfloat162_rn(x1.x * scale, x1.y * scale),
                            __floats2bfloat162_rn(x1.z * scale, x1.w * scale)};
    const int owner = int(n / o.nl);
    __nv_bfloat16* base = static_cast<__nv_bfloat16*>(o.base[owner]) +
                          ((b * o.nl + (n - owner * o.nl)) * o.H + o.h0 + h) * D + dv * 8;
    *reinterpret_cast<uint4*>(base) = *reinterpret_cast<uint4*>(ov);
  }
}

// Delta = rowsum(dO * O) in fp32, one (b, t, h) row per thread, into the head
// owner's Delta block, for head dims whose rows are not a power-of-two number
// of 16-B vectors (D = 72).  Same arithmetic (sequential fmaf over the row) as
// layout.cu's delta_kernel, so the Delta bits do not depend on the transport.
__global__ void __launch_bounds__(256) delta_push_kernel(PeerPack pk, int64_t B, int64_t Nl, int H, int Hl, int rank,
                                                         int vpr, int64_t tensor_vecs) {
  const int64_t rows = B * Nl * H;
  const uint4* dout = static_cast<const uint4*>(pk.dout);
  const uint4* out = static_cast<const uint4*>(pk.out);
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
    float* dd = reinterpret_cast<float*>(static_cast<uint4*>(pk.dst[j]) + int64_t(pk.ntensors) * tensor_vecs);
    dd[((int64_t(rank) * Nl + t) * B + b) * Hl + hp] = acc;
  }
}

int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  return int(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

cudaError_t launch_pack_push(const PeerPack& pk, int64_t B, int64_t Nl, int H, int D, int P, int rank,
                             cudaStream_t stream) {
  const int Hl = H / P;
  const int64_t total = B * Nl * H * (D / 8);
  const int64_t tensor_vecs = B * Nl * P * Hl * (D / 8);  // one receive tensor [N][B][Hl][D]
  const int grid = grid_for(total, 256);
  switch (D / 8) {
    case 4: pack_push_kernel<4><<<grid, 256, 0, stream>>>(pk, B, Nl, H, Hl, rank, tensor_vecs); break;
    case 8: pack_push_kernel<8><<<grid, 256, 0, stream>>>(pk, B, Nl, H, Hl, rank, tensor_vecs); break;
    case 16: pack_push_kernel<16><<<grid, 256, 0, stream>>>(pk, B, Nl, H, Hl, rank, tensor_vecs); break;
    case 9: {  // D = 72: rows of 9 vectors straddle warps; Delta in its own pass
      PeerPack data = pk;
      data.dout = nullptr;
      pack_push_kernel<9><<<grid, 256, 0, stream>>>(data, B, Nl, H, Hl, rank, tensor_vecs);
      if (pk.dout != nullptr)
        delta_push_kernel<<<grid_for(B * Nl * H, 256), 256, 0, stream>>>(pk, B, Nl, H, Hl, rank, 9, tensor_vecs);
      break;
    }
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_signal(const PeerFlags& f, int slot, int rank, int P, int64_t step, cudaStream_t stream) {
  signal_kernel<<<1, 32, 0, stream>>>(f, slot, rank, P, step);
  return cudaGetLastError();
}

cudaError_t launch_wait_copy(const int64_t* flags, int slot, int P, int64_t step, const void* src, void* dst,
                             int64_t bytes, int* err, cudaStream_t stream) {
  const int64_t n_vec = bytes / 16;
  wait_copy_kernel<<<n_vec > 0 ? grid_for(n_vec, 256) : 1, 256, 0, stream>>>(
      flags, slot, P, step, static_cast<const uint4*>(src), static_cast<uint4*>(dst), n_vec, err);
  return cudaGetLastError();
}

cudaError_t launch_finalize_push(const float* dq_acc, const PeerOut& o, int64_t B, int64_t N, int heads, int D,
                                 float scale, cudaStream_t stream) {
  const int64_t total_vec = B * heads * N * (D / 8);
  const int64_t n_pad = (N + 127) / 128 * 128;
  finalize_push_kernel<<<grid_for(total_vec, 256), 256, 0, stream>>>(reinterpret_cast<const float4*>(dq_acc), o, N,
                                                                      n_pad, heads, D, scale, total_vec);
  return cudaGetLastError();
}

}  // namespace ua
