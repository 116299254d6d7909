// lsq_lib.cu -- C ABI of the engine (include/layersim_cuda.h): program objects, the
// forward / forward+adjoint drivers, and the small auxiliary kernels (group tables,
// deterministic fp64 reductions, coupling contraction).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>
#include <limits.h>
#include <nvrtc.h>
#include <stdlib.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <atomic>
#include <fstream>
#include <sstream>
#include <functional>
#include <vector>

#include "../../include/layersim_cuda.h"
#include "lsq_common.cuh"
#include "lsq_prims.cuh"

using namespace lsq;

namespace {

thread_local std::string g_err;

// Per-call bookkeeping lives with the CALLING HOST THREAD, never in the program: a program is
// immutable once lsq_program_jit has attached its kernels, so any number of host threads and
// streams can run it concurrently (each thread sees the launch count / pass timings of its
// own last call).
struct CallState {
  bool profiling = false;
  std::vector<cudaEvent_t> ev;  // pool: 2 events per profiled pass launch
  int ev_used = 0;
  std::vector<int> kinds;
  int launches = 0;
  ~CallState() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};
thread_local CallState g_call;

void begin_call() {
  g_call.ev_used = 0;
  g_call.kinds.clear();
  g_call.launches = 0;
}

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(LSQ_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));        \
  } while (0)

// ---- auxiliary kernels -----------------------------------------------------------------

// shared (non per-row) group tables: 32 floats per group
__global__ void k_group_table(const int* W, const double* fvals, const double* theta, float* gmats) {
  const int ng = sec_cnt(W, SEC_GROUPS);
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
    const int* grp = W + sec_off(W, SEC_GROUPS) + g * GROUP_WORDS;
    if (grp[GW_PERROW]) continue;
    group_table_entry(W, g, fvals, theta, nullptr, gmats + (size_t)g * 32);
  }
}

// per-row (encoding) group tables: [row][nperrow][32]
__global__ void k_row_table(const int* W, const double* fvals, const double* theta, const double* x,
                            int x_stride, int batch, float* rowtab) {
  const int ng = sec_cnt(W, SEC_GROUPS);
  const int npr = W[HDR_NPERROW];
  const int64_t total = (int64_t)batch * ng;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(id / ng), g = (int)(id % ng);
    const int* grp = W + sec_off(W, SEC_GROUPS) + g * GROUP_WORDS;
    if (!grp[GW_PERROW]) continue;
    group_table_entry(W, g, fvals, theta, x + (size_t)b * x_stride,
                      rowtab + ((size_t)b * npr + grp[GW_ROWIDX]) * 32);
  }
}

// product-state prefix vectors: ptab[row][w] = U_w |0> (column 0 of the wire's prefix group),
// |0> for wires without one
__global__ void k_prefix_table(const int* W, const double* fvals, const double* theta, const double* x,
                               int x_stride, int batch, float* ptab) {
  const int n = W[2];
  const int64_t total = (int64_t)batch * n;
  const int* pre = W + sec_off(W, SEC_PREFIX);
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(id / n), w = (int)(id % n);
    float* o = ptab + id * 4;
    const int gid = pre[w * 4];
    if (gid < 0) {
      o[0] = 1.f; o[1] = 0.f; o[2] = 0.f; o[3] = 0.f;
      continue;
    }
    cd U[16];
    group_unitary(W, gid, fvals, theta, x ? x + (size_t)b * x_stride : nullptr, U);
    o[0] = (float)U[0].r; o[1] = (float)U[0].i; o[2] = (float)U[2].r; o[3] = (float)U[2].i;
  }
}

// Macc[b][first + f] = sum_c part[(b*cpr + c)*slotf + f]   (fixed order)
__global__ void k_reduce_part(const double* part, int cpr, int slotf, double* macc, int slot_total,
                              int first, int batch) {
  const int64_t total = (int64_t)batch * slotf;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(id / slotf), f = (int)(id % slotf);
    double s = 0.0;
    const double* src = part + (size_t)b * cpr * slotf + f;
    for (int c = 0; c < cpr; ++c) s += src[(size_t)c * slotf];
    macc[(size_t)b * slot_total + first + f] = s;
  }
}

// zq[b][q] and value[b] from per-CTA partials indexed by physical bit
__global__ void k_reduce_z(const double* zpart, int cpr, int n, const double* wts, double* zq,
                           double* value, int batch) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < batch; b += gridDim.x * blockDim.x) {
    double val = 0.0;
    for (int q = 0; q < n; ++q) {
      const int p = n - 1 - q;
      double s = 0.0;
      for (int c = 0; c < cpr; ++c) s += zpart[((size_t)b * cpr + c) * (n + 1) + p];
      if (zq) zq[(size_t)b * n + q] = s;
      val += (wts ? wts[q] : 1.0) * s;
    }
    if (value) value[b] = val;
  }
}

#ifndef K_CONTRACT_1Q
#define K_CONTRACT_1Q 1
#endif
// 2x2 complex helpers on register arrays (the one-qubit groups of k_contract)
__device__ __forceinline__ void mul2(const cd* a, const cd* b, cd* o) {  // o = a b (o may alias)
  const cd t0 = cadd(cmulx(a[0], b[0]), cmulx(a[1], b[2])), t1 = cadd(cmulx(a[0], b[1]), cmulx(a[1], b[3]));
  const cd t2 = cadd(cmulx(a[2], b[0]), cmulx(a[3], b[2])), t3 = cadd(cmulx(a[2], b[1]), cmulx(a[3], b[3]));
  o[0] = t0; o[1] = t1; o[2] = t2; o[3] = t3;
}
__device__ __forceinline__ void gate2(int code, const double* p, cd* o) {
  cd m[16];
  gate_matrix_dev(code, p, m);
  o[0] = m[0]; o[1] = m[1]; o[2] = m[2]; o[3] = m[3];
}
__device__ __forceinline__ void dgate2(int code, const double* p, int k, cd* o) {
  cd m[16];
  gate_deriv_dev(code, p, k, m);
  o[0] = m[0]; o[1] = m[1]; o[2] = m[2]; o[3] = m[3];
}

// one-qubit group of k_contract with register-resident 2x2 matrices (the generic path below
// keeps 16-entry arrays in local memory for every group)
__device__ void contract1q(const int* grp, const int* gates, const double* fvals, const double* theta,
                           const double* xrow, const cd* M, int b, double* grows, int T, double* erows, int E) {
  const int ngt = grp[GW_NG];
  cd U[4] = {cd{1, 0}, cd{0, 0}, cd{0, 0}, cd{1, 0}};
  for (int j = 0; j < ngt; ++j) {
    const int* gw = gates + (grp[GW_G0] + j) * GATE_WORDS;
    double p[3] = {0, 0, 0};
    for (int k = 0; k < gw[7]; ++k) p[k] = gate_param(gw, k, fvals, theta, xrow);
    cd G[4];
    gate2(gw[0], p, G);
    mul2(G, U, U);
  }
  const cd Ud[4] = {cd{U[0].r, -U[0].i}, cd{U[2].r, -U[2].i}, cd{U[1].r, -U[1].i}, cd{U[3].r, -U[3].i}};
  cd A[4] = {cd{1, 0}, cd{0, 0}, cd{0, 0}, cd{1, 0}};
  for (int j = 0; j < ngt; ++j) {
    const int* gw = gates + (grp[GW_G0] + j) * GATE_WORDS;
    double p[3] = {0, 0, 0};
    for (int k = 0; k < gw[7]; ++k) p[k] = gate_param(gw, k, fvals, theta, xrow);
    cd G[4], Bm[4] = {cd{1, 0}, cd{0, 0}, cd{0, 0}, cd{1, 0}};
    gate2(gw[0], p, G);
    for (int jj = j + 1; jj < ngt; ++jj) {
      const int* gw2 = gates + (grp[GW_G0] + jj) * GATE_WORDS;
      double p2[3] = {0, 0, 0};
      for (int k = 0; k < gw2[7]; ++k) p2[k] = gate_param(gw2, k, fvals, theta, xrow);
      cd G2[4];
      gate2(gw2[0], p2, G2);
      mul2(G2, Bm, Bm);
    }
    for (int k = 0; k < gw[7]; ++k) {
      const int s = gw[2 + k];
      if (s == -1) continue;
      cd Wm[4];
      dgate2(gw[0], p, k, Wm);
      mul2(Wm, A, Wm);
      mul2(Bm, Wm, Wm);
      mul2(Wm, Ud, Wm);
      double g = 0.0;
      for (int e = 0; e < 4; ++e) g += Wm[e].r * M[e].r - Wm[e].i * M[e].i;
      g *= 2.0;
      if (s & ENC_FLAG) {
        if (erows) erows[(size_t)b * E + (s & ~ENC_FLAG)] = g;
      } else {
        if (grows) grows[(size_t)b * T + s] = g;
      }
    }
    mul2(G, A, A);
  }
}

// per (row, group): grads of every parameter of every gate in the group,
// g = 2 Re sum_ab W_ab M_ab,  W = (G_s..G_{j+1}) dG_j (G_{j-1}..G_1) U^dag
__global__ void k_contract(const int* W, const double* fvals, const double* theta, const double* x,
                           int x_stride, const double* macc, int slot_total, int batch,
                           double* grows, int T, double* erows, int E) {
  const int ng = sec_cnt(W, SEC_GROUPS);
  const int64_t total = (int64_t)batch * ng;
  const int* gates = W + sec_off(W, SEC_GATES);
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(id / ng), gid = (int)(id % ng);
    const int* grp = W + sec_off(W, SEC_GROUPS) + gid * GROUP_WORDS;
    if (!grp[GW_GRAD] || grp[GW_SLOT] < 0) continue;
    const double* xrow = x ? x + (size_t)b * x_stride : nullptr;
    const int d = 1 << grp[GW_ARITY];
    const double* mrow = macc + (size_t)b * slot_total + grp[GW_SLOT];
    cd Mm[16];
    mat_zero(Mm, d);
    if (grp[GW_PREFIX]) {
      // prefix group at the prefix boundary: M_ab = Lambda(a) v(b), v = U|0>
      cd U0[16];
      group_unitary(W, gid, fvals, theta, xrow, U0);
      const cd v[2] = {U0[0], U0[2]};
      for (int a = 0; a < 2; ++a)
        for (int bb = 0; bb < 2; ++bb) Mm[a * 2 + bb] = cmulx(cd{mrow[2 * a], mrow[2 * a + 1]}, v[bb]);
    } else if (grp[GW_DIAG]) {
      for (int e = 0; e < d; ++e) Mm[e * d + e] = cd{mrow[2 * e], mrow[2 * e + 1]};
    } else {
      for (int e = 0; e < d * d; ++e) Mm[e] = cd{mrow[2 * e], mrow[2 * e + 1]};
    }
    if (d == 2 && K_CONTRACT_1Q) {
      const cd M2[4] = {Mm[0], Mm[1], Mm[2], Mm[3]};
      contract1q(grp, gates, fvals, theta, xrow, M2, b, grows, T, erows, E);
      continue;
    }
    cd U[16], Ud[16], A[16], Bm[16], G[16], dG[16], Wm[16];
    group_unitary(W, gid, fvals, theta, xrow, U);
    mat_dag(U, Ud, d);
    mat_eye(A, d);
    const int ngt = grp[GW_NG];
    for (int j = 0; j < ngt; ++j) {
      const int* gw = gates + (grp[GW_G0] + j) * GATE_WORDS;
      double p[3] = {0, 0, 0};
      for (int k = 0; k < gw[7]; ++k) p[k] = gate_param(gw, k, fvals, theta, xrow);
      gate_matrix_dev(gw[0], p, G);
      if (d == 4 && gw[1]) mat_swap_wires(G);
      // B = G_s ... G_{j+1}
      mat_eye(Bm, d);
      for (int jj = j + 1; jj < ngt; ++jj) {
        const int* gw2 = gates + (grp[GW_G0] + jj) * GATE_WORDS;
        double p2[3] = {0, 0, 0};
        for (int k = 0; k < gw2[7]; ++k) p2[k] = gate_param(gw2, k, fvals, theta, xrow);
        cd G2[16];
        gate_matrix_dev(gw2[0], p2, G2);
        if (d == 4 && gw2[1]) mat_swap_wires(G2);
        mat_mul(G2, Bm, Bm, d);
      }
      for (int k = 0; k < gw[7]; ++k) {
        const int s = gw[2 + k];
        if (s == -1) continue;
        gate_deriv_dev(gw[0], p, k, dG);
        if (d == 4 && gw[1]) mat_swap_wires(dG);
        mat_mul(dG, A, Wm, d);
        mat_mul(Bm, Wm, Wm, d);
        mat_mul(Wm, Ud, Wm, d);
        double g = 0.0;
        for (int e = 0; e < d * d; ++e) g += Wm[e].r * Mm[e].r - Wm[e].i * Mm[e].i;
        g *= 2.0;
        if (s & ENC_FLAG) {
          if (erows) erows[(size_t)b * E + (s & ~ENC_FLAG)] = g;
        } else {
          if (grows) grows[(size_t)b * T + s] = g;
        }
      }
      mat_mul(G, A, A, d);
    }
  }
}

__global__ void k_zero(double* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

// grad_sum[t] = sum_b grows[b][t]: one block per t, fixed-shape tree (deterministic)
__global__ void k_sum_rows(const double* grows, int batch, int T, double* out) {
  __shared__ double red[256];
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    double s = 0.0;
    for (int b = threadIdx.x; b < batch; b += blockDim.x) s += grows[(size_t)b * T + t];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[t] = red[0];
    __syncthreads();
  }
}

int pow2floor(int64_t v) {
  int r = 1;
  while ((int64_t)r * 2 <= v) r *= 2;
  return r;
}

}  // namespace

struct PassInfo {
  int M, R, nph, slotf, matf, nops, nsubs, first_slot;
};

struct JitKernel {
  const void* fn = nullptr;  // cudaKernel_t usable as a function handle
  int NT = 0;
  size_t smem_set = 0;
  int occ = 0;  // resident CTAs per SM at smem_set (cudaOccupancyMaxActiveBlocksPerMultiprocessor)
};

struct lsq_program {
  std::vector<JitKernel> jit;  // [pass * 3 + mode]: the specialised kernel of each pass and mode
  std::vector<cudaLibrary_t> jit_libs;
  int n, T, E, npasses, ngroups, slot_total, nperrow, prefix = 0, obs = 0;
  int* d_words = nullptr;
  double* d_fvals = nullptr;
  std::vector<int> words;
  std::vector<PassInfo> passes;
  int sm_count = 148;
};

namespace {

size_t smem_bytes(const lsq_program* P, const PassInfo& pi, int NV) {
  (void)NV;
  const int NT = 1 << (pi.M - pi.R);
  const int NW = (NT + 31) / 32;
  size_t b = sizeof(float2) * ((size_t)1 << pi.M);
  b += sizeof(int) * ((size_t)pi.nph * PHASE_WORDS + (size_t)pi.nops * OP_WORDS + (size_t)pi.nsubs * SUB_WORDS + 64);
  b += sizeof(float) * (((pi.matf + 3) & ~3) + ((NW * pi.slotf + 3) & ~3));
  b += sizeof(double) * 34;
  b += sizeof(float) * NW * 32;  // per-warp <Z> / reduction scratch (n + 1 <= 32, M + 1 <= 32)
  b += sizeof(float) * NW * 8;   // specialised kernels: coupling half-block padding per warp
  return (b + 15) & ~(size_t)15;
}

struct Geometry {
  int tpc, cpr;
};

// Tiles per CTA. With the resident capacity G = occ x SMs of the specialised kernel known,
// tpc minimises waves x (tpc + 1/2): whole waves of equal CTAs (a partial last wave leaves
// SMs idle) against the per-CTA prologue (table staging, first tile load, partial flush),
// costed at half a tile. Without it: about 4 CTAs per SM of 64 tiles at most.
// per-CTA prologue cost in tiles (LSQ_GEOM_PROLOGUE overrides; A/B runs)
double geom_prologue() {
  static const double v = [] {
    const char* e = getenv("LSQ_GEOM_PROLOGUE");
    return e ? atof(e) : 0.5;
  }();
  return v;
}

Geometry geometry(const lsq_program* P, int pidx, int mode, int batch) {
  const PassInfo& pi = P->passes[pidx];
  const int ntiles = 1 << (P->n - pi.M);
  const int64_t total = (int64_t)batch * ntiles;
  int occ = 0;
  if (!P->jit.empty() && mode >= 0 && P->jit[pidx * 3 + mode].fn) occ = P->jit[pidx * 3 + mode].occ;
  if (occ > 0) {
    const int64_t G = (int64_t)occ * P->sm_count;
    int best_t = 1;
    double best = 1e300;
    for (int t = std::min(ntiles, 64); t >= 1; t >>= 1) {
      const int64_t units = total / t;
      const int64_t waves = (units + G - 1) / G;
      const double cost = (double)waves * (t + geom_prologue());
      if (cost < best * (1 - 1e-9)) {
        best = cost;
        best_t = t;
      }
    }
    return Geometry{best_t, ntiles / best_t};
  }
  const int64_t target = (int64_t)P->sm_count * 4;
  int tpc = total > target ? pow2floor(total / target) : 1;
  if (tpc > ntiles) tpc = ntiles;
  if (tpc > 64) tpc = 64;
  return Geometry{tpc, ntiles / tpc};
}

struct WS {
  float* gmats;
  float* rowtab;
  float* ptab;
  double* part;
  double* zpart;
  double* macc;
  double* grows;
  double* erows;
  size_t bytes;
};

WS carve(const lsq_program* P, int batch, void* base) {
  WS w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  size_t maxpart = 0, maxz = 0;
  for (int p = 0; p < (int)P->passes.size(); ++p)
    for (int mode = -1; mode < 3; ++mode) {
      const PassInfo& pi = P->passes[p];
      Geometry g = geometry(P, p, mode, batch);
      maxpart = std::max(maxpart, (size_t)batch * g.cpr * pi.slotf);
      maxz = std::max(maxz, (size_t)batch * g.cpr * (P->n + 1));
    }
  size_t o_g = take(sizeof(float) * 32 * (size_t)std::max(P->ngroups, 1));
  size_t o_r = take(sizeof(float) * 32 * (size_t)batch * std::max(P->nperrow, 1));
  size_t o_pt = take(sizeof(float) * 4 * (size_t)batch * (P->prefix ? P->n : 1));
  size_t o_p = take(sizeof(double) * std::max(maxpart, (size_t)1));
  size_t o_z = take(sizeof(double) * std::max(maxz, (size_t)1));
  size_t o_m = take(sizeof(double) * (size_t)batch * std::max(P->slot_total, 1));
  size_t o_gr = take(sizeof(double) * (size_t)batch * std::max(P->T, 1));
  size_t o_er = take(sizeof(double) * (size_t)batch * std::max(P->E, 1));
  w.bytes = off;
  if (base) {
    char* c = (char*)base;
    w.gmats = (float*)(c + o_g);
    w.rowtab = (float*)(c + o_r);
    w.ptab = (float*)(c + o_pt);
    w.part = (double*)(c + o_p);
    w.zpart = (double*)(c + o_z);
    w.macc = (double*)(c + o_m);
    w.grows = (double*)(c + o_gr);
    w.erows = (double*)(c + o_er);
  }
  return w;
}

int launch_pass(const lsq_program* P, int pi_idx, int mode, int flags, int batch, const double* theta,
                const double* x, int x_stride, const double* w, const float2* psi_in, float2* psi_out,
                float2* lam, const WS& ws, cudaStream_t st) {
  const PassInfo& pi = P->passes[pi_idx];
  const JitKernel* jk = P->jit.empty() ? nullptr : &P->jit[pi_idx * 3 + mode];
  if (!jk || !jk->fn)
    return fail(LSQ_EPLAN, "no kernel for pass " + std::to_string(pi_idx) + " mode " + std::to_string(mode) +
                               ": attach the program's specialised kernels first (lsq_program_jit)");
  Geometry g = geometry(P, pi_idx, mode, batch);
  PassArgs A{};
  A.prog = P->d_words;
  A.fvals = P->d_fvals;
  A.pass = pi_idx;
  A.mode = mode;
  A.flags = flags;
  A.n = P->n;
  A.psi_in = psi_in;
  A.psi_out = psi_out;
  A.lam = lam;
  A.tiles_per_cta = g.tpc;
  A.ctas_per_row = g.cpr;
  A.gmats = ws.gmats;
  A.rowtab = ws.rowtab;
  A.nperrow = P->nperrow;
  A.ptab = ws.ptab;
  A.theta = theta;
  A.x = x;
  A.x_stride = x_stride;
  A.wts = w;
  A.part = ws.part;
  A.zpart = ws.zpart;
  CallState& C = g_call;
  // NVTX range per pass launch ("lsq p<pass> <mode>"): host-side, free without an attached tool
  static const char* const kModeName[3] = {"fwd", "turn", "adj"};
  char nvtx_name[32];
  snprintf(nvtx_name, sizeof nvtx_name, "lsq p%d %s", pi_idx, kModeName[mode]);
  nvtxRangePushA(nvtx_name);
  struct NvtxPop {
    ~NvtxPop() { nvtxRangePop(); }
  } nvtx_pop;
  if (C.profiling) {
    while ((int)C.ev.size() < 2 * (C.ev_used + 1)) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      C.ev.push_back(e);
    }
    CUDA_TRY(cudaEventRecord(C.ev[2 * C.ev_used], st));
  }
  void* args[] = {&A};
  CUDA_TRY(cudaLaunchKernel(jk->fn, dim3((unsigned)((int64_t)batch * g.cpr)), dim3(jk->NT), args, jk->smem_set, st));
  C.launches++;
  if (C.profiling) {
    CUDA_TRY(cudaEventRecord(C.ev[2 * C.ev_used + 1], st));
    C.kinds.push_back(mode * 1000 + pi_idx);
    C.ev_used++;
  }
  if (pi.slotf > 0 && mode != MODE_FWD) {
    const int64_t tot = (int64_t)batch * pi.slotf;
    const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 4096);
    k_reduce_part<<<blocks, 256, 0, st>>>(ws.part, g.cpr, pi.slotf, ws.macc, P->slot_total, pi.first_slot, batch);
    CUDA_TRY(cudaGetLastError());
    C.launches++;
  }
  return LSQ_OK;
}

int finish_grads(const lsq_program* P, int batch, const double* theta, const double* x, int x_stride,
                 const WS& ws, double* grad_rows, double* grad_sum, double* egrad_rows, cudaStream_t st) {
  double* grows = grad_rows ? grad_rows : ws.grows;
  double* erows = egrad_rows ? egrad_rows : (P->E ? ws.erows : nullptr);
  if (P->T) {
    const int64_t t = (int64_t)batch * P->T;
    k_zero<<<(int)std::min<int64_t>((t + 255) / 256, 4096), 256, 0, st>>>(grows, t);
    g_call.launches++;
  }
  if (erows) {
    const int64_t t = (int64_t)batch * P->E;
    k_zero<<<(int)std::min<int64_t>((t + 255) / 256, 4096), 256, 0, st>>>(erows, t);
    g_call.launches++;
  }
  {
    const int64_t tot = (int64_t)batch * P->ngroups;
    const int blocks = (int)std::min<int64_t>((tot + 127) / 128, 8192);
    k_contract<<<std::max(blocks, 1), 128, 0, st>>>(P->d_words, P->d_fvals, theta, x, x_stride, ws.macc,
                                                   P->slot_total, batch, grows, P->T, erows, P->E);
    g_call.launches++;
    CUDA_TRY(cudaGetLastError());
  }
  if (grad_sum && P->T) {
    k_sum_rows<<<std::min(P->T, 4096), 256, 0, st>>>(grows, batch, P->T, grad_sum);
    g_call.launches++;
    CUDA_TRY(cudaGetLastError());
  }
  return LSQ_OK;
}

}  // namespace

extern "C" {

int lsq_version(void) { return 1; }

const char* lsq_last_error(void) { return g_err.c_str(); }

int lsq_device_info(int device, char* buf, int buflen) {
  cudaDeviceProp p;
  CUDA_TRY(cudaGetDeviceProperties(&p, device));
  int drv = 0;
  cudaDriverGetVersion(&drv);
  snprintf(buf, buflen, "%s|%d|%d.%d|%d", p.name, p.multiProcessorCount, p.major, p.minor, drv);
  return LSQ_OK;
}

int lsq_program_create(const int32_t* words, int64_t n_words, const double* fvals, int64_t n_fvals,
                       lsq_program** out) {
  if (!words || n_words < HDR_WORDS || !out) return fail(LSQ_EINVAL, "bad program words");
  if (words[0] != MAGIC) return fail(LSQ_EINVAL, "program magic mismatch");
  if (words[1] != 1) return fail(LSQ_EPLAN, "program version mismatch");
  auto* P = new lsq_program();
  P->words.assign(words, words + n_words);
  const int* W = P->words.data();
  P->n = W[2];
  P->T = W[3];
  P->E = W[4];
  P->slot_total = W[5];
  P->npasses = W[6];
  P->ngroups = W[7];
  P->nperrow = W[HDR_NPERROW];
  P->prefix = W[HDR_PREFIX];
  P->obs = W[HDR_OBS];
  if (P->n < 1 || P->n > 30) {
    delete P;
    return fail(LSQ_EINVAL, "n out of range (1..30)");
  }
  for (int s = 0; s < N_SECTIONS; ++s) {
    if (sec_off(W, s) < HDR_WORDS || sec_off(W, s) > n_words) {
      delete P;
      return fail(LSQ_EINVAL, "corrupt program section table");
    }
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&P->sm_count, cudaDevAttrMultiProcessorCount, dev);
  for (int i = 0; i < P->npasses; ++i) {
    const int* pw = W + sec_off(W, SEC_PASSES) + i * PASS_WORDS;
    PassInfo pi{};
    pi.M = pw[PW_M];
    pi.R = pw[PW_R];
    pi.nph = pw[PW_NPH];
    pi.slotf = pw[PW_SLOTF];
    pi.matf = pw[PW_MATF];
    pi.nops = pw[PW_OPN];
    pi.nsubs = pw[PW_SUBN];
    pi.first_slot = pw[PW_FIRSTSLOT];
    P->passes.push_back(pi);
  }
  cudaError_t e1 = cudaMalloc(&P->d_words, sizeof(int) * n_words);
  cudaError_t e2 = cudaMalloc(&P->d_fvals, sizeof(double) * std::max<int64_t>(n_fvals, 1));
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    delete P;
    return fail(LSQ_ECUDA, "cudaMalloc failed for program tables");
  }
  cudaMemcpy(P->d_words, words, sizeof(int) * n_words, cudaMemcpyHostToDevice);
  if (n_fvals > 0) cudaMemcpy(P->d_fvals, fvals, sizeof(double) * n_fvals, cudaMemcpyHostToDevice);
  CUDA_TRY(cudaGetLastError());
  *out = P;
  return LSQ_OK;
}

namespace {

uint64_t fnv1a(const char* s, size_t n) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= (unsigned char)s[i];
    h *= 1099511628211ull;
  }
  return h;
}

bool read_file(const std::string& path, std::string& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::stringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return !out.empty();
}

// NVRTC is resolved at run time from the CUDA toolkit this library was built against (absolute
// path, RTLD_LOCAL): a process that imported torch first already has torch's bundled
// libnvrtc.so.12 (an older 12.x) loaded under the same SONAME, and that ptxas does not fold the
// FFMA2 lane swap/negation into operand modifiers (measured: 1148 MOVs vs 6 in one kernel).
struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcVersion) version = nullptr;
  std::string path, err;
  bool ok = false;
};

#ifndef LSQ_NVRTC_DEFAULT
#define LSQ_NVRTC_DEFAULT "/usr/local/cuda/lib64/libnvrtc.so.12"
#endif

const Nvrtc& nvrtc() {
  static Nvrtc N;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("LSQ_NVRTC");
    std::string want = env && *env ? env : LSQ_NVRTC_DEFAULT;
    char real[PATH_MAX];
    if (realpath(want.c_str(), real)) want = real;
    void* h = dlopen(want.c_str(), RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      N.err = std::string("dlopen(") + want + "): " + dlerror();
      return;
    }
    N.path = want;
    N.create = (decltype(N.create))dlsym(h, "nvrtcCreateProgram");
    N.compile = (decltype(N.compile))dlsym(h, "nvrtcCompileProgram");
    N.log_size = (decltype(N.log_size))dlsym(h, "nvrtcGetProgramLogSize");
    N.log = (decltype(N.log))dlsym(h, "nvrtcGetProgramLog");
    N.cubin_size = (decltype(N.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    N.cubin = (decltype(N.cubin))dlsym(h, "nvrtcGetCUBIN");
    N.destroy = (decltype(N.destroy))dlsym(h, "nvrtcDestroyProgram");
    N.version = (decltype(N.version))dlsym(h, "nvrtcVersion");
    N.ok = N.create && N.compile && N.log_size && N.log && N.cubin_size && N.cubin && N.destroy;
    if (!N.ok) N.err = "missing NVRTC symbols in " + want;
  });
  return N;
}

// NVRTC: source -> sm_100a cubin (with an optional on-disk cache keyed by the source hash)
int jit_compile(const std::string& src, const std::string& cache_dir, std::string& cubin, std::string& log) {
  const Nvrtc& R = nvrtc();
  if (!R.ok) {
    log = R.err;
    return 1;
  }
  std::string key;
  if (!cache_dir.empty()) {
    char buf[40];
    int maj = 0, min = 0;
    if (R.version) R.version(&maj, &min);
    const std::string keyed = src + "\n// nvrtc " + std::to_string(maj) + "." + std::to_string(min);
    snprintf(buf, sizeof buf, "%016llx", (unsigned long long)fnv1a(keyed.data(), keyed.size()));
    key = cache_dir + "/lsq_" + buf + ".cubin";
    if (read_file(key, cubin)) return 0;
  }
  nvrtcProgram prog;
  if (R.create(&prog, src.c_str(), "lsq_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    log = "nvrtcCreateProgram failed";
    return 1;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-DNDEBUG"};
  nvrtcResult rc = R.compile(prog, 4, opts);
  size_t ls = 0;
  R.log_size(prog, &ls);
  if (ls > 1) {
    log.resize(ls);
    R.log(prog, &log[0]);
  }
  if (rc != NVRTC_SUCCESS) {
    R.destroy(&prog);
    return 1;
  }
  size_t cs = 0;
  R.cubin_size(prog, &cs);
  cubin.resize(cs);
  R.cubin(prog, &cubin[0]);
  R.destroy(&prog);
  if (!key.empty()) {
    // unique per process AND thread: the ranks of a torchrun job compile the same kernels at the
    // same time into one cache directory, and equal thread ids across processes would let one
    // rank truncate the file another is about to rename
    std::string tmp = key + ".tmp" + std::to_string((long long)getpid()) + "_" +
                      std::to_string((unsigned long long)std::hash<std::thread::id>{}(std::this_thread::get_id()));
    std::ofstream f(tmp, std::ios::binary);
    if (f) {
      f.write(cubin.data(), (std::streamsize)cubin.size());
      f.close();
      std::rename(tmp.c_str(), key.c_str());
    }
  }
  return 0;
}

}  // namespace

int lsq_program_jit(lsq_program* P, int nk, const char* const* sources, const int* pass_idx,
                    const int* modes, const int* stage_vecs, const int* reg_bits, const char* const* names,
                    const char* cache_dir, int threads) {
  if (!P || nk < 0 || (nk && (!sources || !pass_idx || !modes || !names)))
    return fail(LSQ_EINVAL, "bad JIT arguments");
  std::vector<std::string> cubins(nk), logs(nk);
  std::vector<int> rcs(nk, 0);
  std::atomic<int> next{0};
  const std::string cdir = cache_dir ? cache_dir : "";
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  nt = std::max(1, std::min(nt, nk));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&]() {
      for (int i = next++; i < nk; i = next++) rcs[i] = jit_compile(sources[i], cdir, cubins[i], logs[i]);
    });
  for (auto& th : pool) th.join();
  for (int i = 0; i < nk; ++i)
    if (rcs[i]) return fail(LSQ_EINVAL, std::string("NVRTC failed for ") + names[i] + ":\n" + logs[i].substr(0, 4000));
  P->jit.assign((size_t)P->npasses * 3, JitKernel{});
  for (int i = 0; i < nk; ++i) {
    if (pass_idx[i] < 0 || pass_idx[i] >= P->npasses || modes[i] < 0 || modes[i] > 2)
      return fail(LSQ_EINVAL, "bad JIT kernel index");
    cudaLibrary_t lib;
    CUDA_TRY(cudaLibraryLoadData(&lib, cubins[i].data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    P->jit_libs.push_back(lib);
    cudaKernel_t kern;
    CUDA_TRY(cudaLibraryGetKernel(&kern, lib, names[i]));
    JitKernel& jk = P->jit[pass_idx[i] * 3 + modes[i]];
    jk.fn = (const void*)kern;
    const PassInfo& pi = P->passes[pass_idx[i]];
    // a kernel may tile its registers differently from the program's phase plan (forward kernels
    // with 2^5 amplitudes per thread): reg_bits[i] sets its thread count
    const int kr = reg_bits && reg_bits[i] > 0 ? reg_bits[i] : pi.R;
    if (kr < 1 || kr > pi.M || kr > MAX_R) return fail(LSQ_EINVAL, "bad register bits for a JIT kernel");
    jk.NT = 1 << (pi.M - kr);
    // specialised kernels may add a next-tile prefetch stage of stage_vecs[i] x 2^M amplitudes
    const int NV = modes[i] == 0 ? 1 : 2;
    const int sv = stage_vecs ? stage_vecs[i] : NV;
    const size_t sm = smem_bytes(P, pi, NV) + (size_t)sv * sizeof(float2) * ((size_t)1 << pi.M);
    CUDA_TRY(cudaFuncSetAttribute(jk.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    jk.smem_set = sm;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&jk.occ, jk.fn, jk.NT, sm));
    const char* geo = getenv("LSQ_GEOM_OCC");  // "0": fixed 4-CTAs-per-SM heuristic (A/B runs)
    if (geo && geo[0] == '0') jk.occ = 0;
  }
  return LSQ_OK;
}

int lsq_program_load(const char* path, const char* cache_dir, lsq_program** out) {
  if (!path || !out) return fail(LSQ_EINVAL, "null argument");
  std::string blob;
  if (!read_file(path, blob)) return fail(LSQ_EINVAL, std::string("cannot read program artifact ") + path);
  size_t off = 0;
  auto take = [&](void* dst, size_t n) {
    if (off + n > blob.size()) return false;
    memcpy(dst, blob.data() + off, n);
    off += n;
    return true;
  };
  char magic[4];
  uint32_t version = 0;
  int64_t nw = 0, nf = 0;
  int32_t nk = 0;
  if (!take(magic, 4) || memcmp(magic, "LSQP", 4) != 0) return fail(LSQ_EINVAL, "not a program artifact (magic)");
  if (!take(&version, 4)) return fail(LSQ_EINVAL, "truncated program artifact");
  if (version != 1 && version != 2)
    return fail(LSQ_EPLAN, "program artifact version " + std::to_string(version) + " not in {1, 2}");
  if (!take(&nw, 8) || !take(&nf, 8) || !take(&nk, 4) || nw < HDR_WORDS || nf < 0 || nk < 0 ||
      (size_t)nw > blob.size() / 4 || (size_t)nf > blob.size() / 8)
    return fail(LSQ_EINVAL, "corrupt program artifact header");
  std::vector<int32_t> words((size_t)nw);
  std::vector<double> fvals((size_t)std::max<int64_t>(nf, 1));
  if (!take(words.data(), 4 * (size_t)nw) || !take(fvals.data(), 8 * (size_t)nf))
    return fail(LSQ_EINVAL, "truncated program artifact (words)");
  std::vector<std::string> srcs((size_t)nk), names((size_t)nk);
  std::vector<int> pidx((size_t)nk), modes((size_t)nk), stages((size_t)nk), regs((size_t)nk, 0);
  for (int i = 0; i < nk; ++i) {
    int32_t nl = 0;
    int64_t sl = 0;
    if (!take(&pidx[i], 4) || !take(&modes[i], 4) || !take(&stages[i], 4) || (version >= 2 && !take(&regs[i], 4)) ||
        !take(&nl, 4) || nl < 1 || (size_t)nl > blob.size() - off)
      return fail(LSQ_EINVAL, "corrupt program artifact (kernel header)");
    names[i].resize((size_t)nl);
    if (!take(&names[i][0], (size_t)nl) || !take(&sl, 8) || sl < 1 || (size_t)sl > blob.size() - off)
      return fail(LSQ_EINVAL, "corrupt program artifact (kernel source)");
    srcs[i].resize((size_t)sl);
    take(&srcs[i][0], (size_t)sl);
  }
  if (off != blob.size()) return fail(LSQ_EINVAL, "trailing bytes in program artifact");
  lsq_program* P = nullptr;
  int rc = lsq_program_create(words.data(), nw, fvals.data(), nf, &P);
  if (rc) return rc;
  std::vector<const char*> sp((size_t)nk), np((size_t)nk);
  for (int i = 0; i < nk; ++i) {
    sp[i] = srcs[i].c_str();
    np[i] = names[i].c_str();
  }
  rc = lsq_program_jit(P, nk, sp.data(), pidx.data(), modes.data(), stages.data(), regs.data(), np.data(),
                       cache_dir, 0);
  if (rc) {
    lsq_program_destroy(P);
    return rc;
  }
  *out = P;
  return LSQ_OK;
}

void lsq_program_destroy(lsq_program* P) {
  if (!P) return;
  for (auto l : P->jit_libs) cudaLibraryUnload(l);
  cudaFree(P->d_words);
  cudaFree(P->d_fvals);
  delete P;
}

int lsq_program_info(const lsq_program* P, int64_t* o) {
  if (!P || !o) return fail(LSQ_EINVAL, "null argument");
  o[0] = P->n; o[1] = P->T; o[2] = P->E; o[3] = P->npasses; o[4] = P->ngroups; o[5] = P->slot_total;
  o[6] = P->sm_count; o[7] = 0;
  return LSQ_OK;
}

int64_t lsq_workspace_bytes(const lsq_program* P, int batch) {
  if (!P || batch < 1) return -1;
  return (int64_t)carve(P, batch, nullptr).bytes;
}

int lsq_set_profiling(const lsq_program* P, int on) {
  if (!P) return fail(LSQ_EINVAL, "null program");
  g_call.profiling = on != 0;
  return LSQ_OK;
}

int lsq_last_pass_times(const lsq_program* P, float* ms, int cap, int* kinds) {
  if (!P) return -1;
  const CallState& C = g_call;
  const int n = C.ev_used;
  if (n > 0 && cudaEventSynchronize(C.ev[2 * n - 1]) != cudaSuccess) return -1;
  for (int i = 0; i < n && i < cap; ++i) {
    float t = 0.f;
    cudaEventElapsedTime(&t, C.ev[2 * i], C.ev[2 * i + 1]);
    if (ms) ms[i] = t;
    if (kinds) kinds[i] = C.kinds[i];
  }
  return n;
}

int lsq_last_launch_count(const lsq_program* P) { return P ? g_call.launches : -1; }

int lsq_jit_compiler(char* buf, int buflen) {
  const Nvrtc& R = nvrtc();
  int maj = 0, min = 0;
  if (R.ok && R.version) R.version(&maj, &min);
  snprintf(buf, buflen, "%s|%d.%d|%s", R.ok ? R.path.c_str() : "unavailable", maj, min, R.err.c_str());
  return R.ok ? LSQ_OK : LSQ_ECUDA;
}

int lsq_forward(const lsq_program* Pc, int batch, const double* theta, const double* x, int x_stride,
                const double* w, const void* psi_in, void* psi_out, double* zq, double* value,
                void* workspace, void* stream) {
  const lsq_program* P = Pc;
  if (!P || batch < 1 || !psi_out || !workspace) return fail(LSQ_EINVAL, "null argument");
  if (P->T && !theta) return fail(LSQ_EINVAL, "circuit has trainable parameters but none given");
  if (P->E && !x) return fail(LSQ_EINVAL, "circuit has encoding parameters but none given");
  cudaStream_t st = (cudaStream_t)stream;
  WS ws = carve(P, batch, workspace);
  begin_call();
  k_group_table<<<std::max(1, (P->ngroups + 127) / 128), 128, 0, st>>>(P->d_words, P->d_fvals, theta, ws.gmats);
  g_call.launches++;
  if (P->nperrow && x) {
    const int64_t tot = (int64_t)batch * P->ngroups;
    k_row_table<<<(int)std::min<int64_t>((tot + 127) / 128, 8192), 128, 0, st>>>(P->d_words, P->d_fvals, theta, x, x_stride, batch, ws.rowtab);
    g_call.launches++;
  }
  if (P->prefix) {
    const int64_t tot = (int64_t)batch * P->n;
    k_prefix_table<<<(int)std::min<int64_t>((tot + 127) / 128, 8192), 128, 0, st>>>(P->d_words, P->d_fvals, theta, x, x_stride, batch, ws.ptab);
    g_call.launches++;
  }
  CUDA_TRY(cudaGetLastError());
  const float2* src = (const float2*)psi_in;
  float2* dst = (float2*)psi_out;
  const bool want_z = zq || value;
  if (P->npasses == 0) return fail(LSQ_EPLAN, "empty program");
  for (int i = 0; i < P->npasses; ++i) {
    int flags = F_STORE_PSI;
    if (i == 0 && !src) flags |= F_SYNTH;
    if (i == P->npasses - 1 && want_z) flags |= F_ZPART;
    const float2* in = (i == 0) ? src : dst;
    int rc = launch_pass(P, i, MODE_FWD, flags, batch, theta, x, x_stride, w, in ? in : dst, dst, nullptr, ws, st);
    if (rc) return rc;
  }
  if (want_z) {
    Geometry g = geometry(P, P->npasses - 1, MODE_FWD, batch);
    k_reduce_z<<<(batch + 127) / 128, 128, 0, st>>>(ws.zpart, g.cpr, P->n, w, zq, value, batch);
    g_call.launches++;
    CUDA_TRY(cudaGetLastError());
  }
  return LSQ_OK;
}

int lsq_fwd_bwd(const lsq_program* Pc, int batch, const double* theta, const double* x, int x_stride,
                const double* w, void* psi_v, void* lam_v, double* zq, double* value, double* grad_rows,
                double* grad_sum, double* egrad_rows, void* workspace, void* stream) {
  return lsq_fwd_bwd_ckpt(Pc, batch, theta, x, x_stride, w, psi_v, lam_v, nullptr, zq, value, grad_rows,
                          grad_sum, egrad_rows, workspace, stream);
}

int lsq_fwd_bwd_ckpt(const lsq_program* Pc, int batch, const double* theta, const double* x, int x_stride,
                     const double* w, void* psi_v, void* lam_v, void* ckpt_v, double* zq, double* value,
                     double* grad_rows, double* grad_sum, double* egrad_rows, void* workspace,
                     void* stream) {
  const lsq_program* P = Pc;
  if (!P || batch < 1 || !psi_v || !lam_v || !workspace) return fail(LSQ_EINVAL, "null argument");
  if (P->T && !theta) return fail(LSQ_EINVAL, "circuit has trainable parameters but none given");
  if (P->E && !x) return fail(LSQ_EINVAL, "circuit has encoding parameters but none given");
  if (P->npasses == 0) return fail(LSQ_EPLAN, "empty program");
  cudaStream_t st = (cudaStream_t)stream;
  WS ws = carve(P, batch, workspace);
  begin_call();
  float2* psi = (float2*)psi_v;
  float2* lam = (float2*)lam_v;
  k_group_table<<<std::max(1, (P->ngroups + 127) / 128), 128, 0, st>>>(P->d_words, P->d_fvals, theta, ws.gmats);
  g_call.launches++;
  if (P->nperrow && x) {
    const int64_t tot = (int64_t)batch * P->ngroups;
    k_row_table<<<(int)std::min<int64_t>((tot + 127) / 128, 8192), 128, 0, st>>>(P->d_words, P->d_fvals, theta, x, x_stride, batch, ws.rowtab);
    g_call.launches++;
  }
  if (P->prefix) {
    const int64_t tot = (int64_t)batch * P->n;
    k_prefix_table<<<(int)std::min<int64_t>((tot + 127) / 128, 8192), 128, 0, st>>>(P->d_words, P->d_fvals, theta, x, x_stride, batch, ws.ptab);
    g_call.launches++;
  }
  CUDA_TRY(cudaGetLastError());
  const int64_t mtot = (int64_t)batch * std::max(P->slot_total, 1);
  k_zero<<<(int)std::min<int64_t>((mtot + 255) / 256, 4096), 256, 0, st>>>(ws.macc, mtot);
  g_call.launches++;
  const int L = P->npasses;
  // checkpoint mode: pass i writes its output to ckpt[i] (i < L-1); the adjoint reads psi from
  // the checkpoints and writes lambda only. Otherwise psi is un-computed in place.
  float2* ck = (float2*)ckpt_v;
  const size_t vec = (size_t)batch << P->n;
  auto out_of = [&](int i) -> float2* { return ck ? ck + (size_t)i * vec : psi; };
  for (int i = 0; i < L - 1; ++i) {
    int flags = F_STORE_PSI | (i == 0 ? F_SYNTH : 0);
    const float2* in = i == 0 ? out_of(0) : out_of(i - 1);
    int rc = launch_pass(P, i, MODE_FWD, flags, batch, theta, x, x_stride, w, in, out_of(i), nullptr, ws, st);
    if (rc) return rc;
  }
  {
    int flags = (L == 1 ? F_SYNTH : 0) | (L > 1 ? F_STORE_LAM : 0);
    const float2* in = L > 1 ? out_of(L - 2) : psi;
    int rc = launch_pass(P, L - 1, MODE_TURN, flags, batch, theta, x, x_stride, w, in, psi, lam, ws, st);
    if (rc) return rc;
    Geometry g = geometry(P, L - 1, MODE_TURN, batch);
    k_reduce_z<<<(batch + 127) / 128, 128, 0, st>>>(ws.zpart, g.cpr, P->n, w, zq, value, batch);
    g_call.launches++;
    CUDA_TRY(cudaGetLastError());
  }
  for (int i = L - 2; i >= 0; --i) {
    int flags = i > 0 ? ((ck ? 0 : F_STORE_PSI) | F_STORE_LAM) : 0;
    float2* pin = out_of(i);
    int rc = launch_pass(P, i, MODE_BWD, flags, batch, theta, x, x_stride, w, pin, pin, lam, ws, st);
    if (rc) return rc;
  }
  return finish_grads(P, batch, theta, x, x_stride, ws, grad_rows, grad_sum, egrad_rows, st);
}

int lsq_bwd_from_state(const lsq_program* Pc, int batch, const double* theta, const double* x,
                       int x_stride, const double* w, const void* final_state, void* psi_v, void* lam_v,
                       double* zq, double* value, double* grad_rows, double* grad_sum,
                       double* egrad_rows, void* workspace, void* stream) {
  const lsq_program* P = Pc;
  if (!P || batch < 1 || !final_state || !psi_v || !lam_v || !workspace)
    return fail(LSQ_EINVAL, "null argument");
  if (P->T && !theta) return fail(LSQ_EINVAL, "circuit has trainable parameters but none given");
  if (P->E && !x) return fail(LSQ_EINVAL, "circuit has encoding parameters but none given");
  if (P->npasses == 0) return fail(LSQ_EPLAN, "empty program");
  cudaStream_t st = (cudaStream_t)stream;
  WS ws = carve(P, batch, workspace);
  begin_call();
  float2* psi = (float2*)psi_v;
  float2* lam = (float2*)lam_v;
  k_group_table<<<std::max(1, (P->ngroups + 127) / 128), 128, 0, st>>>(P->d_words, P->d_fvals, theta, ws.gmats);
  g_call.launches++;
  if (P->nperrow && x) {
    const int64_t tot = (int64_t)batch * P->ngroups;
    k_row_table<<<(int)std::min<int64_t>((tot + 127) / 128, 8192), 128, 0, st>>>(P->d_words, P->d_fvals, theta, x, x_stride, batch, ws.rowtab);
    g_call.launches++;
  }
  if (P->prefix) {
    const int64_t tot = (int64_t)batch * P->n;
    k_prefix_table<<<(int)std::min<int64_t>((tot + 127) / 128, 8192), 128, 0, st>>>(P->d_words, P->d_fvals, theta, x, x_stride, batch, ws.ptab);
    g_call.launches++;
  }
  CUDA_TRY(cudaGetLastError());
  const int64_t mtot = (int64_t)batch * std::max(P->slot_total, 1);
  k_zero<<<(int)std::min<int64_t>((mtot + 255) / 256, 4096), 256, 0, st>>>(ws.macc, mtot);
  g_call.launches++;
  const int L = P->npasses;
  {
    int flags = F_NOFWD | F_STORE_LAM | F_STORE_PSI;
    int rc = launch_pass(P, L - 1, MODE_TURN, flags, batch, theta, x, x_stride, w,
                         (const float2*)final_state, psi, lam, ws, st);
    if (rc) return rc;
    Geometry g = geometry(P, L - 1, MODE_TURN, batch);
    k_reduce_z<<<(batch + 127) / 128, 128, 0, st>>>(ws.zpart, g.cpr, P->n, w, zq, value, batch);
    g_call.launches++;
    CUDA_TRY(cudaGetLastError());
  }
  for (int i = L - 2; i >= 0; --i) {
    int flags = i > 0 ? (F_STORE_PSI | F_STORE_LAM) : 0;
    int rc = launch_pass(P, i, MODE_BWD, flags, batch, theta, x, x_stride, w, psi, psi, lam, ws, st);
    if (rc) return rc;
  }
  return finish_grads(P, batch, theta, x, x_stride, ws, grad_rows, grad_sum, egrad_rows, st);
}

}  // extern "C"
