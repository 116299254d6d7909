// Accuracy of the diagonal-run phase evaluations on the GPU: MUFU __sincosf of the full angle,
// MUFU on the exactly quadrant-reduced angle (|x| <= pi/4), the fixed-point polynomial of
// lsq_prims.cuh, and sincospif -- worst absolute error against fp64 sincos over 2^26 angles.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "../../paper_2506_04891_b200/csrc/lsq_prims.cuh"

__global__ void k(double* worst) {
  double w[4] = {0, 0, 0, 0};
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < (1u << 26); u += gridDim.x * blockDim.x) {
    const int32_t ph = (int32_t)(u * 64u + 17u);
    double sd, cd;
    sincospi((double)ph / 2147483648.0, &sd, &cd);
    float s, c;
    __sincosf((float)ph * 1.4629180792671596e-09f, &s, &c);
    w[0] = fmax(w[0], fmax(fabs(c - cd), fabs(s - sd)));
    const int32_t q = (int32_t)((uint32_t)ph + 0x20000000u) >> 30;
    const int32_t r = (int32_t)((uint32_t)ph - ((uint32_t)q << 30));
    float sr, cr;
    __sincosf((float)r * 1.4629180792671596e-09f, &sr, &cr);
    const int qq = q & 3;
    float c2 = (qq & 1) ? sr : cr, s2 = (qq & 1) ? cr : sr;
    if (qq == 1 || qq == 2) c2 = -c2;
    if (qq >= 2) s2 = -s2;
    w[1] = fmax(w[1], fmax(fabs(c2 - cd), fabs(s2 - sd)));
    const float2 p = lsq::phase_cs(ph);
    w[2] = fmax(w[2], fmax(fabs(p.x - cd), fabs(p.y - sd)));
    float s3, c3;
    sincospif((float)ph * 4.656612873077393e-10f, &s3, &c3);
    w[3] = fmax(w[3], fmax(fabs(c3 - cd), fabs(s3 - sd)));
  }
  for (int i = 0; i < 4; ++i) {
    unsigned long long* a = (unsigned long long*)&worst[i];
    unsigned long long old = *a, assumed;
    do {
      assumed = old;
      if (__longlong_as_double(assumed) >= w[i]) break;
      old = atomicCAS(a, assumed, __double_as_longlong(w[i]));
    } while (assumed != old);
  }
}

int main() {
  double* d;
  cudaMalloc(&d, 4 * sizeof(double));
  cudaMemset(d, 0, 4 * sizeof(double));
  k<<<1184, 256>>>(d);
  double h[4];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("worst abs error: MUFU full %.3e | MUFU reduced %.3e | fixed-point polynomial %.3e | sincospif %.3e\n",
         h[0], h[1], h[2], h[3]);
  return 0;
}
