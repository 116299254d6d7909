// lsq_inst.cu -- one pass-kernel instantiation per translation unit (LSQ_M, LSQ_NV given on
// the nvcc command line) so the sm_100a build runs in parallel (see Makefile).
#include "lsq_pass.cuh"
#include "lsq_kernels.h"

#ifndef LSQ_M
#error "LSQ_M must be defined"
#endif
#ifndef LSQ_NV
#error "LSQ_NV must be defined"
#endif

#define LSQ_CAT2(a, b, c) a##b##_##c
#define LSQ_CAT(a, b, c) LSQ_CAT2(a, b, c)

extern "C" lsq::KernelEntry LSQ_CAT(lsq_kernel_entry_, LSQ_M, LSQ_NV)(void) {
  constexpr int R = lsq::r_of(LSQ_M);
  lsq::KernelEntry e;
  e.fn = (const void*)&lsq::lsq_pass_kernel<LSQ_M, R, LSQ_NV>;
  e.M = LSQ_M;
  e.R = R;
  e.NV = LSQ_NV;
  e.NT = 1 << (LSQ_M - R);
  return e;
}
