/*
 * layersim_cuda.h -- C ABI of the B200 (sm_100a) engine for the TQml layer-wise
 * state-vector simulator (arXiv 2506.04891).
 *
 * Drop-in boundary.  The reference path is pure Python + a Cython primitive module:
 *   - circuit seam : layersim.core.apply_circuit          pkg/src/layersim/core.py:46-72
 *                    layersim.grad.backward_sweep         pkg/src/layersim/grad.py:169-204
 *                    layersim.grad.gradient               pkg/src/layersim/grad.py:207-218
 *                    layersim.states.expectation_z_sum    pkg/src/layersim/states.py:100-102
 *   - primitive seam: layersim.backend.ops() -> _fastops  pkg/src/layersim/backend.py:25,53-55
 *                    (_fastops.pyx:17-205, 14 in-place ops on host complex128 arrays)
 * The Python package paper_2506_04891_b200 keeps the circuit seam's signatures and calls
 * the entry points below through ctypes.  No torch types cross this
 * boundary: device buffers are plain pointers the caller allocated (PyTorch, cudaMalloc,
 * ...), streams are cudaStream_t passed as void*.
 *
 * Status codes: 0 ok, 1 invalid argument (-> ValueError), 2 plan/program mismatch
 * (-> PlanMismatchError), 3 capacity (-> CapacityError), 4 CUDA error (-> RuntimeError).
 * lsq_last_error() returns a thread-local message for the last failing call.
 *
 * Layouts.  A state batch is (batch, 2^n) complex64 (float2), row-major, wire 0 = most
 * significant index bit (reference states.py:3-6).  Parameters are float64 in the
 * reference's units (radians for rz/rzz/rx/ry/rot, turns for gpi/gpi2/ms).
 *
 * Programs.  lsq_program_create() takes the int32 "program words" + float64 constants
 * produced by the host compiler (paper_2506_04891_b200/schedule.py: fused gate groups,
 * tile passes, register phases).  Word layout: a 32-word header (magic 0x4C535131,
 * version, n, T, E, coupling floats, #passes, #groups, then (offset,count) for the
 * sections gates/groups/passes/phases/ops/subs/pass-groups).  Programs are immutable and
 * may be shared by concurrent streams.
 */
#ifndef LAYERSIM_CUDA_H
#define LAYERSIM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSQ_OK 0
#define LSQ_EINVAL 1
#define LSQ_EPLAN 2
#define LSQ_ECAPACITY 3
#define LSQ_ECUDA 4

typedef struct lsq_program lsq_program;

/* Library / device information. */
int lsq_version(void);
const char* lsq_last_error(void);
/* Writes "name|sm_count|cc_major.cc_minor|driver" into buf (machine id for plans). */
int lsq_device_info(int device, char* buf, int buflen);

/* Build an immutable program on the current device (replaces the per-layer
 * kernels.prepare(...) appliers, reference kernels.py:1006-1023). */
int lsq_program_create(const int32_t* words, int64_t n_words, const double* fvals,
                       int64_t n_fvals, lsq_program** out);
void lsq_program_destroy(lsq_program* prog);
int lsq_program_info(const lsq_program* prog, int64_t* out8); /* n,T,E,passes,groups,slots,..*/

/* Device workspace needed for one call on `batch` rows. */
int64_t lsq_workspace_bytes(const lsq_program* prog, int batch);

/* Forward pass (reference apply_circuit, core.py:46-72).
 *   psi_in : (batch,2^n) input state, or NULL for |0..0> (reference zero_state)
 *   psi_out: (batch,2^n) output state (may equal psi_in; the reference returns a copy,
 *            which the Python layer guarantees by passing a fresh buffer)
 *   zq     : optional (batch,n) float64 <Z_q> of the output state
 *   value  : optional (batch,) float64 sum_q w_q <Z_q>  (w=NULL -> all ones)
 *   theta  : (T,) float64 device, x: (batch, x_stride) float64 device (encoding rows) */
int lsq_forward(const lsq_program* prog, int batch, const double* theta, const double* x,
                int x_stride, const double* w, const void* psi_in, void* psi_out,
                double* zq, double* value, void* workspace, void* stream);

/* Forward from |0..0> + adjoint backward (reference gradient, grad.py:207-218, with the
 * weighted observable sum_q w_q Z_q; w=NULL reproduces sum_k Z_k, states.py:88-97).
 *   psi, lam   : (batch,2^n) scratch state buffers (contents overwritten)
 *   zq, value  : optional outputs as in lsq_forward
 *   grad_rows  : optional (batch,T) float64, d value[b] / d theta  (GradResult.grads)
 *   grad_sum   : optional (T,) float64, sum over the batch rows (fixed summation order)
 *   egrad_rows : optional (batch,E) float64 (GradResult.encoding_grads) */
int lsq_fwd_bwd(const lsq_program* prog, int batch, const double* theta, const double* x,
                int x_stride, const double* w, void* psi, void* lam, double* zq,
                double* value, double* grad_rows, double* grad_sum, double* egrad_rows,
                void* workspace, void* stream);

/* Adjoint backward from a given final state (reference backward_sweep, grad.py:169-204):
 * final_state (batch,2^n) is read only; psi/lam are scratch; outputs as lsq_fwd_bwd. The
 * sweep un-computes psi layer group by layer group exactly like the reference. */
int lsq_bwd_from_state(const lsq_program* prog, int batch, const double* theta, const double* x,
                       int x_stride, const double* w, const void* final_state, void* psi, void* lam,
                       double* zq, double* value, double* grad_rows, double* grad_sum,
                       double* egrad_rows, void* workspace, void* stream);

/* Per-launch timing of the last call on this program (CUDA events on the call's stream):
 * fills up to `cap` floats with milliseconds per pass-kernel launch (kinds[i] = mode*1000 +
 * pass index, mode 0 fwd / 1 turnaround / 2 adjoint), returns the count. Events are
 * recorded without synchronisation; this call waits for the last one. Only active after
 * lsq_set_profiling(prog, 1). */
int lsq_set_profiling(lsq_program* prog, int on);
int lsq_last_pass_times(const lsq_program* prog, float* ms, int cap, int* kinds);
/* Number of kernels (pass kernels + auxiliary reductions) launched by the last call. */
int lsq_last_launch_count(const lsq_program* prog);

#ifdef __cplusplus
}
#endif
#endif /* LAYERSIM_CUDA_H */
