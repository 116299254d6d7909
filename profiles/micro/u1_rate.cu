// Microbenchmark: packed-FP32 rate of the specialised kernels' one-qubit apply pattern
// (lsq_prims.cuh fx/fmix/mx chains on 16 register amplitudes) at the kernels' occupancy.
// Forward: 1 vector; adjoint: 2 vectors + 3 coupling components per group.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2506_04891_b200/csrc/lsq_prims.cuh"
using namespace lsq;

template <int K>
__device__ __forceinline__ void u1(float2 (&v)[16], const float* g) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if ((i >> K) & 1) continue;
    const int j = i | (1 << K);
    const float2 x0 = v[i], x1 = v[j];
    v[i] = fmix(x1, g[5], fx(x1, g[4], fmix(x0, g[1], mx(x0, g[0]))));
    v[j] = fmix(x1, g[7], fx(x1, g[6], fmix(x0, g[3], mx(x0, g[2]))));
  }
}
template <int K>
__device__ __forceinline__ float3 coup(const float2 (&p)[16], const float2 (&l)[16]) {
  float2 a = make_float2(0.f, 0.f), b = a, c = a;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if ((i >> K) & 1) continue;
    const int j = i | (1 << K);
    a = vf_j(l[j], p[j], vf_mj(l[i], p[i], a));
    b = vf_mj(l[j], p[i], vf_mj(l[i], p[j], b));
    c = vf_n(l[i], p[j], vf_p(l[j], p[i], c));
  }
  return make_float3(a.x + a.y, b.x + b.y, c.x + c.y);
}

__global__ void __launch_bounds__(256, 3) k_fwd(float2* out, const float* gm, int iters) {
  __shared__ float s[64];
  if (threadIdx.x < 64) s[threadIdx.x] = gm[threadIdx.x];
  __syncthreads();
  float2 v[16];
  for (int i = 0; i < 16; ++i) v[i] = make_float2(threadIdx.x * 1e-3f + i, i * 1e-3f);
  for (int it = 0; it < iters; ++it) {
    u1<0>(v, s + 0); u1<1>(v, s + 8); u1<2>(v, s + 16); u1<3>(v, s + 24);
  }
  float2 acc = make_float2(0.f, 0.f);
  for (int i = 0; i < 16; ++i) { acc.x += v[i].x; acc.y += v[i].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(256, 2) k_bwd(float2* out, const float* gm, int iters) {
  __shared__ float s[64];
  if (threadIdx.x < 64) s[threadIdx.x] = gm[threadIdx.x];
  __syncthreads();
  float2 p[16], l[16];
  for (int i = 0; i < 16; ++i) { p[i] = make_float2(threadIdx.x * 1e-3f + i, i * 1e-3f); l[i] = make_float2(i * 1e-3f, threadIdx.x * 1e-3f); }
  float sum = 0.f;
  for (int it = 0; it < iters; ++it) {
    float3 c;
    c = coup<0>(p, l); sum += c.x + c.y + c.z; u1<0>(p, s + 0); u1<0>(l, s + 0);
    c = coup<1>(p, l); sum += c.x + c.y + c.z; u1<1>(p, s + 8); u1<1>(l, s + 8);
    c = coup<2>(p, l); sum += c.x + c.y + c.z; u1<2>(p, s + 16); u1<2>(l, s + 16);
    c = coup<3>(p, l); sum += c.x + c.y + c.z; u1<3>(p, s + 24); u1<3>(l, s + 24);
  }
  float2 acc = make_float2(sum, 0.f);
  for (int i = 0; i < 16; ++i) { acc.x += p[i].x + l[i].x; acc.y += p[i].y + l[i].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  float2* out; float* gm;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(float2));
  cudaMalloc(&gm, 64 * sizeof(float));
  float h[64]; for (int i = 0; i < 64; ++i) h[i] = 0.5f * ((i * 37) % 11) / 11.f;
  cudaMemcpy(gm, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  for (int bpsm = 1; bpsm <= 3; ++bpsm) {
    for (int rep = 0; rep < 2; ++rep) {
      float ms;
      const int blocks = 148 * bpsm;
      cudaEventRecord(e0); k_fwd<<<blocks, 256>>>(out, gm, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      // 4 groups x 16 amps x 4 packed ops per amp per iteration, 2 FMA each
      double fma = 4.0 * 16 * 4 * 2 * iters * (double)blocks * 256;
      if (rep) printf("fwd  %d CTA/SM: %.1f TFMA/s (%.0f%% of 37.2)\n", bpsm, fma / ms / 1e9, 100 * fma / ms / 1e9 / 37.2);
      if (bpsm > 2) continue;
      cudaEventRecord(e0); k_bwd<<<blocks, 256>>>(out, gm, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      // per group: 2 x 16 x 4 (apply) + 3 x 16 (coupling, 2 per pair) packed ops
      double fmb = 4.0 * (2 * 16 * 4 + 3 * 16) * 2 * iters * (double)blocks * 256;
      if (rep) printf("bwd  %d CTA/SM: %.1f TFMA/s (%.0f%% of 37.2)\n", bpsm, fmb / ms / 1e9, 100 * fmb / ms / 1e9 / 37.2);
    }
  }
  return 0;
}
