// Microbenchmark: FP32 FMA throughput with scalar FFMA vs packed FFMA2 (fma.rn.f32x2) on B200.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pk(float2 v){ unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(v.x), "f"(v.y)); return r; }
__device__ __forceinline__ float2 upk(unsigned long long r){ float2 v; asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b, int iters) {
  unsigned long long x[8];
  for (int i = 0; i < 8; ++i) x[i] = pk(make_float2(threadIdx.x + i, i));
  unsigned long long A = pk(make_float2(a, a)), B = pk(make_float2(b, b));
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = upk(x[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000, blocks = 148 * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ffma<<<blocks, threads>>>(out, 0.999f, 0.001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)blocks * threads;
    printf("FFMA : %.1f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(e0); k_ffma2<<<blocks, threads>>>(out, 0.999f, 0.001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2: %.1f TFLOP/s\n", fl / ms / 1e9);
  }
  return 0;
}
