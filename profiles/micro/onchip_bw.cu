// Microbenchmark behind the "keep n=16 on chip" decision (on-chip row): what an
// inter-pass exchange costs on B200 through each level a pass boundary could use instead of HBM:
//   1. distributed shared memory (cluster of C CTAs, every CTA reads 16-byte words of the
//      other CTAs' 64 KB buffers: the all-to-all a tile re-partition between passes needs),
//   2. local shared memory (the exchange the pass kernels already do inside a pass),
//   3. L2-resident global reads + writes (a working set of 48 MB, below the 126 MB L2),
//   4. HBM-streaming reads + writes (a working set of 4 GB).
// Aggregate GB/s over the whole GPU; nvcc -O3 -gencode arch=compute_100a,code=sm_100a.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int TILE_BYTES = 64 * 1024;  // 2^13 complex64 amplitudes: one n=16 row over 8 CTAs
constexpr int NT = 512;

template <bool REMOTE>
__global__ void __launch_bounds__(NT, 1) k_smem(float* out, int iters) {
  extern __shared__ __align__(16) unsigned char raw[];
  float4* mine = reinterpret_cast<float4*>(raw);
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), r = cl.block_rank();
  for (int i = threadIdx.x; i < TILE_BYTES / 16; i += NT) mine[i] = make_float4(i, r, 1.f, 2.f);
  cl.sync();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  // every thread walks the 64 KB tile once per iteration (8 x 16 bytes), slice k of it from
  // CTA (r + 1 + k C / 8) mod C of the cluster (REMOTE) or all of it from its own CTA
  constexpr int K = TILE_BYTES / 16 / NT;
  const float4* p[K];
#pragma unroll
  for (int k = 0; k < K; ++k) p[k] = REMOTE ? cl.map_shared_rank(mine, (r + 1 + (k * C) / K) % C) : mine;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float4 v = p[k][(threadIdx.x + k * NT + it * 32) & (TILE_BYTES / 16 - 1)];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  cl.sync();
  out[blockIdx.x * NT + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

__global__ void __launch_bounds__(256) k_copy(const float4* __restrict__ src, float4* __restrict__ dst,
                                              size_t n16, int iters) {
  for (int it = 0; it < iters; ++it)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
      dst[i] = src[i];
}

template <bool REMOTE>
static double run_smem(int C, int iters, float* out) {
  cudaFuncSetAttribute(k_smem<REMOTE>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_BYTES);
  if (C > 8) cudaFuncSetAttribute(k_smem<REMOTE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cfg.blockDim = dim3(NT); cfg.dynamicSmemBytes = TILE_BYTES;
  int nclusters = 0;
  cfg.gridDim = dim3(C);
  cudaOccupancyMaxActiveClusters(&nclusters, k_smem<REMOTE>, &cfg);
  if (nclusters <= 0) return -1.0;
  cfg.gridDim = dim3(nclusters * C);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0.f;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cudaError_t rc = cudaLaunchKernelEx(&cfg, k_smem<REMOTE>, out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    if (rc != cudaSuccess || cudaGetLastError() != cudaSuccess) return -1.0;
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double bytes = (double)TILE_BYTES * iters * nclusters * C;
  printf("  %s cluster=%2d: %3d clusters resident (%3d SMs), %8.1f GB/s aggregate, %6.1f GB/s per SM\n",
         REMOTE ? "DSMEM all-to-all" : "local shared    ", C, nclusters, nclusters * C, bytes / ms / 1e6,
         bytes / ms / 1e6 / (nclusters * C));
  return bytes / ms / 1e6;
}

int main() {
  float* out; cudaMalloc(&out, 148 * NT * 4 * 4);
  printf("shared-memory tile reads (64 KB per CTA per iteration, 16-byte loads, 512 threads):\n");
  run_smem<false>(1, 400, out);
  for (int C : {2, 4, 8, 16}) run_smem<true>(C, 100, out);
  printf("global copy (read + write bytes), 148 x 8 CTAs of 256 threads:\n");
  for (size_t mb : {48, 4096}) {
    const size_t n16 = mb * 1024 * 1024 / 2 / 16;  // src + dst together are `mb` MB
    float4 *a, *b; cudaMalloc(&a, n16 * 16); cudaMalloc(&b, n16 * 16);
    cudaMemset(a, 0, n16 * 16); cudaMemset(b, 0, n16 * 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = mb < 128 ? 50 : 2;
    float ms = 0.f;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); k_copy<<<148 * 8, 256>>>(a, b, n16, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("  working set %4zu MB (%s): %8.1f GB/s\n", mb, mb < 128 ? "L2-resident" : "HBM-streaming",
           2.0 * n16 * 16 * iters / ms / 1e6);
    cudaFree(a); cudaFree(b);
  }
  return 0;
}
