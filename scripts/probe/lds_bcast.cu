// Shared-memory wavefronts of warp-uniform (broadcast) loads on sm_100a: what does the
// backward's per-column (lse, Delta) read cost per instruction, by width and address pattern?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_bcast lds_bcast.cu
// Run under: ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,
//   smsp__sass_inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum ./lds_bcast
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

// mode 0: v4 uniform; 1: v2 uniform; 2: scalar uniform; 3: v4, 4 groups of 8 lanes (t % 4) on 4
// consecutive 16 B chunks; 4: v4, 2 groups (t % 2); 5: v4, lanes t / 8 -> chunk (4 groups of 8
// consecutive lanes); 6: v2, 4 groups (t % 4) on 4 consecutive 8 B chunks
template <int kMode>
__global__ void __launch_bounds__(512) lds_kernel(float* out) {
  __shared__ __align__(16) float buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = float(i);
  __syncthreads();
  const int t = threadIdx.x % 32;
  uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 8
  for (int it = 0; it < kIters; ++it) {
    const uint32_t a = base + ((it * 16) & 8191);
    if constexpr (kMode == 0 || kMode == 3 || kMode == 4 || kMode == 5) {
      const uint32_t ad = a + (kMode == 3 ? (t % 4) * 16 : kMode == 4 ? (t % 2) * 16 : kMode == 5 ? (t / 8) * 16 : 0);
      float x, y, z, w;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(ad));
      a0 += x; a1 += y; a2 += z; a3 += w;
    } else if constexpr (kMode == 1 || kMode == 6) {
      const uint32_t ad = a + (kMode == 6 ? (t % 4) * 8 : 0);
      float x, y;
      asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(ad));
      a0 += x; a1 += y;
    } else {
      float x;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a));
      a0 += x;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

template <int kMode>
void run(float* out, const char* name) {
  lds_kernel<kMode><<<148, 512>>>(out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) lds_kernel<kMode><<<148, 512>>>(out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  // warp-instructions per SM per launch: 16 warps x kIters
  const double inst = 16.0 * kIters;
  printf("mode %d %-34s %.3f us/launch  %.2f ns per warp-LDS per SM\n", kMode, name, ms * 100.0,
         ms * 1e6 / 10.0 / inst);
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 512 * sizeof(float));
  run<0>(out, "v4 uniform");
  run<1>(out, "v2 uniform");
  run<2>(out, "f32 uniform");
  run<3>(out, "v4, lane%4 -> 4 chunks (64 B)");
  run<4>(out, "v4, lane%2 -> 2 chunks (32 B)");
  run<5>(out, "v4, lane/8 -> 4 chunks (64 B)");
  run<6>(out, "v2, lane%4 -> 4 chunks (32 B)");
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
