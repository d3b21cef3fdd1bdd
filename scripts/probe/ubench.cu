// ubench.cu — per-SM throughput of MUFU.EX2, FFMA, FFMA2, FMNMX3 and F2FP on
// the B200 (calibrates the softmax cost model in DESIGN.md).  Each thread runs
// 8 independent chains; one CTA per SM x 4 warps per SMSP.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kIters = 4096;

__global__ void k_ex2(float* out, float seed) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3f + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, float seed) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3f + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(0.999f), "f"(seed));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float seed) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(seed + threadIdx.x * 1e-3f + i, seed - i);
  const float2 m = make_float2(0.999f, 0.998f), c = make_float2(seed, seed);
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], m, c);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mix(float* out, float seed) {  // 2 ex2 + 1 ffma2 per pair: MUFU/FMA overlap
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(seed + threadIdx.x * 1e-3f + i, seed - i);
  const float2 m = make_float2(0.999f, 0.998f), c = make_float2(seed, seed);
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = __ffma2_rn(a[i], m, c);
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i].x));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i].y));
    }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// packed half-precision exponentials: 2 results per instruction
__global__ void k_ex2_h2(float* out, float seed) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) {
    __half2 h = __floats2half2_rn(-(seed + i * 0.1f), -(seed + threadIdx.x * 1e-3f));
    a[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __low2float(*reinterpret_cast<__half2*>(&a[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ex2_bf2(float* out, float seed) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(-(seed + i * 0.1f), -(seed + threadIdx.x * 1e-3f));
    a[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __low2float(*reinterpret_cast<__nv_bfloat162*>(&a[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, int ops_per_iter_per_thread, int threads, int sms, float* d) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<sms, threads>>>(d, 0.5f);
  cudaEventRecord(a);
  kern<<<sms, threads>>>(d, 0.5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double ops = double(sms) * threads * kIters * ops_per_iter_per_thread;
  double per_sm_per_ns = ops / sms / (ms * 1e6);
  printf("%-8s threads/SM=%4d  %.2f ms  %.2f ops/ns/SM  (%.1f ops/clk/SM at max clock %.0f MHz)\n", name, threads, ms,
         per_sm_per_ns, per_sm_per_ns / (clk_khz * 1e-6), clk_khz / 1e3);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d;
  cudaMalloc(&d, sms * 1024 * sizeof(float));
  for (int th : {128, 256, 512}) {
    run("ex2", k_ex2, 8, th, sms, d);
    run("ffma", k_ffma, 8, th, sms, d);
    run("ffma2", k_ffma2, 16, th, sms, d);   // 2 FMA per lane per instruction
    run("mix", k_mix, 16, th, sms, d);       // ex2 count (2 per pair)
    run("ex2_h2", k_ex2_h2, 16, th, sms, d);   // results (2 per instruction)
    run("ex2_bf2", k_ex2_bf2, 16, th, sms, d);
  }
  return 0;
}
