// lsq_kernels.h -- registry of the separately compiled pass-kernel instantiations.
#pragma once

namespace lsq {

struct KernelEntry {
  const void* fn;  // __global__ lsq_pass_kernel<M,R,NV>(PassArgs)
  int M, R, NV, NT;
};

// register bits per thread for a tile of M bits (schedule.default_r)
constexpr int r_of(int M) { return M <= 1 ? M : (M - 5 < 2 ? 2 : (M - 5 > 5 ? 5 : M - 5)); }

}  // namespace lsq

#define LSQ_FOR_EACH_KERNEL(X) \
  X(1, 1) X(1, 2) X(2, 1) X(2, 2) X(3, 1) X(3, 2) X(4, 1) X(4, 2) X(5, 1) X(5, 2) X(6, 1) X(6, 2) \
  X(7, 1) X(7, 2) X(8, 1) X(8, 2) X(9, 1) X(9, 2) X(10, 1) X(10, 2) X(11, 1) X(11, 2)         \
  X(12, 1) X(12, 2) X(13, 1) X(13, 2) X(14, 1)

#define LSQ_DECLARE_ENTRY(m, nv) extern "C" lsq::KernelEntry lsq_kernel_entry_##m##_##nv(void);
LSQ_FOR_EACH_KERNEL(LSQ_DECLARE_ENTRY)
