// lsq_common.cuh -- shared definitions of the sm_100a engine: program layout (mirrors
// paper_2506_04891_b200/schedule.py), complex helpers, fp64 gate matrices and derivatives.
//
// Gate conventions restate the reference (pkg/src/layersim/gates.py:144-312): wire 0 is
// the most significant bit, 4x4 matrices index the first wire as the more significant
// local bit, rz/rzz/rx/ry/rot in radians, gpi/gpi2/ms in turns.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lsq {

// ---- program words (schedule.py) -------------------------------------------------------
constexpr int MAGIC = 0x4C535131;
// pass modes and flags (the specialised kernels' PassArgs contract, lsq_prims.cuh PMODE_/PF_)
constexpr int MODE_FWD = 0, MODE_TURN = 1, MODE_BWD = 2;
constexpr int F_SYNTH = 1,      // input psi is |0..0> (not read)
    F_STORE_PSI = 2,            // write psi at the end of the pass
    F_STORE_LAM = 4,            // write lambda at the end of the pass
    F_ZPART = 8,                // forward: accumulate <Z_q> partials of the output
    F_NOFWD = 16;               // turnaround on a given final state: skip the forward ops
constexpr int HDR_WORDS = 32, GATE_WORDS = 8, GROUP_WORDS = 16, PASS_WORDS = 24,
              PHASE_WORDS = 24, OP_WORDS = 8, SUB_WORDS = 8, PGROUP_WORDS = 4;
constexpr int SEC_GATES = 0, SEC_GROUPS = 1, SEC_PASSES = 2, SEC_PHASES = 3, SEC_OPS = 4,
              SEC_SUBS = 5, SEC_PGROUPS = 6, SEC_PREFIX = 7, SEC_OBS = 8, N_SECTIONS = 9;
constexpr int OP_U1 = 1, OP_U2 = 2, OP_DRUN = 3, OP_PX = 4, OP_PCX = 5;
constexpr int SRC_NONE = 0, SRC_REG = 1, SRC_THREAD = 2, SRC_NONLOCAL = 3;
constexpr int ENC_FLAG = 1 << 30;
constexpr int MAX_R = 5;
constexpr int MAX_GROUP_GATES = 64;

// pass word fields
enum { PW_M = 0, PW_R, PW_NPH, PW_PH0, PW_MASK, PW_NGRP, PW_PG0, PW_MATF, PW_SLOTF,
       PW_FIRSTSLOT, PW_OPLO, PW_OPN, PW_SUBLO, PW_SUBN };
// group word fields
enum { GW_ARITY = 0, GW_DIAG, GW_PERROW, GW_NG, GW_G0, GW_WA, GW_WB, GW_SLOT, GW_SLOTF,
       GW_MATF, GW_GRAD, GW_ROWIDX, GW_PREFIX };
constexpr int HDR_NPERROW = 28, HDR_PREFIX = 29, HDR_OBS = 30;
// phase words: [0,5) register local bits, [5,21) thread local bits, 21 op0, 22 nops
constexpr int PH_OP0 = 21, PH_NOPS = 22;

// gate codes = enumerate(GateKind) (gates.py)
enum GateCode { G_Z = 0, G_CZ, G_RZ, G_RZZ, G_GPI, G_S, G_CNOT, G_X, G_H, G_RY, G_RX, G_ROT,
                G_GPI2, G_MS, G_SX, G_ECR, G_SWAP };

__host__ __device__ inline int sec_off(const int* w, int s) { return w[8 + 2 * s]; }
__host__ __device__ inline int sec_cnt(const int* w, int s) { return w[9 + 2 * s]; }

// ---- complex helpers --------------------------------------------------------------------
struct cd {
  double r, i;
};
__device__ __forceinline__ cd mk(double r, double i) { return cd{r, i}; }
__device__ __forceinline__ cd cadd(cd a, cd b) { return cd{a.r + b.r, a.i + b.i}; }
__device__ __forceinline__ cd cmulx(cd a, cd b) {
  return cd{a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r};
}
__device__ __forceinline__ cd cconj(cd a) { return cd{a.r, -a.i}; }
__device__ __forceinline__ cd cscale(cd a, double s) { return cd{a.r * s, a.i * s}; }
__device__ __forceinline__ cd cexpi(double t) {
  double s, c;
  sincos(t, &s, &c);
  return cd{c, s};
}

// dense d x d (d = 2 or 4) row-major complex matrices
__device__ inline void mat_zero(cd* m, int d) {
  for (int i = 0; i < d * d; ++i) m[i] = cd{0, 0};
}
__device__ inline void mat_eye(cd* m, int d) {
  mat_zero(m, d);
  for (int i = 0; i < d; ++i) m[i * d + i] = cd{1, 0};
}
__device__ inline void mat_mul(const cd* a, const cd* b, cd* out, int d) {  // out = a b
  cd t[16];
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c) {
      cd s{0, 0};
      for (int k = 0; k < d; ++k) s = cadd(s, cmulx(a[r * d + k], b[k * d + c]));
      t[r * d + c] = s;
    }
  for (int i = 0; i < d * d; ++i) out[i] = t[i];
}
__device__ inline void mat_dag(const cd* a, cd* out, int d) {
  cd t[16];
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c) t[c * d + r] = cconj(a[r * d + c]);
  for (int i = 0; i < d * d; ++i) out[i] = t[i];
}
__device__ inline void mat_swap_wires(cd* m) {  // P m P, P = |ab> -> |ba> on 4x4
  const int p[4] = {0, 2, 1, 3};
  cd t[16];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) t[r * 4 + c] = m[p[r] * 4 + p[c]];
  for (int i = 0; i < 16; ++i) m[i] = t[i];
}

__device__ inline int gate_dim(int g) {
  return (g == G_CZ || g == G_RZZ || g == G_CNOT || g == G_MS || g == G_ECR || g == G_SWAP) ? 4 : 2;
}

// ---- gate matrices (reference gates.py:83-236) --------------------------------------
__device__ inline void rz2(double t, cd* m) {
  cd e = cexpi(-0.5 * t);
  m[0] = e; m[1] = cd{0, 0}; m[2] = cd{0, 0}; m[3] = cconj(e);
}
__device__ inline void ry2(double t, cd* m) {
  double s, c;
  sincos(0.5 * t, &s, &c);
  m[0] = cd{c, 0}; m[1] = cd{-s, 0}; m[2] = cd{s, 0}; m[3] = cd{c, 0};
}
__device__ inline void rx2(double t, cd* m) {
  double s, c;
  sincos(0.5 * t, &s, &c);
  m[0] = cd{c, 0}; m[1] = cd{0, -s}; m[2] = cd{0, -s}; m[3] = cd{c, 0};
}

__device__ inline void gate_matrix_dev(int g, const double* p, cd* m) {
  const double R2 = 0.70710678118654752440;
  const double TWO_PI = 6.28318530717958647692;
  int d = gate_dim(g);
  mat_zero(m, d);
  switch (g) {
    case G_Z: m[0] = cd{1, 0}; m[3] = cd{-1, 0}; break;
    case G_S: m[0] = cd{1, 0}; m[3] = cd{0, 1}; break;
    case G_X: m[1] = cd{1, 0}; m[2] = cd{1, 0}; break;
    case G_H: m[0] = cd{R2, 0}; m[1] = cd{R2, 0}; m[2] = cd{R2, 0}; m[3] = cd{-R2, 0}; break;
    case G_SX:
      m[0] = cd{0.5, 0.5}; m[1] = cd{0.5, -0.5}; m[2] = cd{0.5, -0.5}; m[3] = cd{0.5, 0.5};
      break;
    case G_RZ: rz2(p[0], m); break;
    case G_RY: ry2(p[0], m); break;
    case G_RX: rx2(p[0], m); break;
    case G_ROT: {
      cd a[4], b[4], c[4];
      rz2(p[0], a); ry2(p[1], b); rz2(p[2], c);
      mat_mul(b, a, m, 2);
      mat_mul(c, m, m, 2);
      break;
    }
    case G_GPI: {
      cd e = cexpi(TWO_PI * p[0]);
      m[1] = cconj(e); m[2] = e;
      break;
    }
    case G_GPI2: {
      cd e = cexpi(TWO_PI * p[0]);
      m[0] = cd{R2, 0}; m[3] = cd{R2, 0};
      m[1] = cmulx(cd{0, -R2}, cconj(e));
      m[2] = cmulx(cd{0, -R2}, e);
      break;
    }
    case G_CZ: m[0] = m[5] = m[10] = cd{1, 0}; m[15] = cd{-1, 0}; break;
    case G_CNOT: m[0] = m[5] = cd{1, 0}; m[11] = m[14] = cd{1, 0}; break;
    case G_SWAP: m[0] = m[6] = m[9] = m[15] = cd{1, 0}; break;
    case G_ECR:
      m[1] = cd{R2, 0}; m[3] = cd{0, R2};
      m[4] = cd{R2, 0}; m[6] = cd{0, -R2};
      m[9] = cd{0, R2}; m[11] = cd{R2, 0};
      m[12] = cd{0, -R2}; m[14] = cd{R2, 0};
      break;
    case G_RZZ: {
      cd e = cexpi(-0.5 * p[0]);
      m[0] = m[15] = e;
      m[5] = m[10] = cconj(e);
      break;
    }
    case G_MS: {
      double s, c;
      sincos(3.14159265358979323846 * p[2], &s, &c);
      cd es = cexpi(TWO_PI * (p[0] + p[1]));
      cd ed = cexpi(TWO_PI * (p[0] - p[1]));
      m[0] = m[5] = m[10] = m[15] = cd{c, 0};
      m[3] = cmulx(cd{0, -s}, cconj(es));
      m[12] = cmulx(cd{0, -s}, es);
      m[6] = cmulx(cd{0, -s}, ed);
      m[9] = cmulx(cd{0, -s}, cconj(ed));
      break;
    }
  }
}

__device__ inline void drz2(double t, cd* m) {
  cd e = cexpi(-0.5 * t);
  m[0] = cmulx(cd{0, -0.5}, e); m[1] = cd{0, 0}; m[2] = cd{0, 0}; m[3] = cmulx(cd{0, 0.5}, cconj(e));
}
__device__ inline void dry2(double t, cd* m) {
  double s, c;
  sincos(0.5 * t, &s, &c);
  m[0] = cd{-0.5 * s, 0}; m[1] = cd{-0.5 * c, 0}; m[2] = cd{0.5 * c, 0}; m[3] = cd{-0.5 * s, 0};
}

// d U / d p[k] (reference gates.py:239-312)
__device__ inline void gate_deriv_dev(int g, const double* p, int k, cd* m) {
  const double R2 = 0.70710678118654752440;
  const double TWO_PI = 6.28318530717958647692;
  const double PI = 3.14159265358979323846;
  int d = gate_dim(g);
  mat_zero(m, d);
  switch (g) {
    case G_RZ: drz2(p[0], m); break;
    case G_RY: dry2(p[0], m); break;
    case G_RX: {
      double s, c;
      sincos(0.5 * p[0], &s, &c);
      m[0] = cd{-0.5 * s, 0}; m[1] = cd{0, -0.5 * c}; m[2] = cd{0, -0.5 * c}; m[3] = cd{-0.5 * s, 0};
      break;
    }
    case G_RZZ: {
      cd e = cexpi(-0.5 * p[0]);
      m[0] = m[15] = cmulx(cd{0, -0.5}, e);
      m[5] = m[10] = cmulx(cd{0, 0.5}, cconj(e));
      break;
    }
    case G_GPI: {
      cd e = cexpi(TWO_PI * p[0]);
      m[1] = cmulx(cd{0, -TWO_PI}, cconj(e));
      m[2] = cmulx(cd{0, TWO_PI}, e);
      break;
    }
    case G_GPI2: {
      cd e = cexpi(TWO_PI * p[0]);
      m[1] = cscale(cconj(e), -TWO_PI * R2);
      m[2] = cscale(e, TWO_PI * R2);
      break;
    }
    case G_ROT: {
      cd a[4], b[4], c[4], t[4];
      rz2(p[0], a); ry2(p[1], b); rz2(p[2], c);
      if (k == 0) {
        drz2(p[0], t);
        mat_mul(b, t, m, 2); mat_mul(c, m, m, 2);
      } else if (k == 1) {
        dry2(p[1], t);
        mat_mul(t, a, m, 2); mat_mul(c, m, m, 2);
      } else {
        drz2(p[2], t);
        mat_mul(b, a, m, 2); mat_mul(t, m, m, 2);
      }
      break;
    }
    case G_MS: {
      double s, c;
      sincos(PI * p[2], &s, &c);
      cd es = cexpi(TWO_PI * (p[0] + p[1]));
      cd ed = cexpi(TWO_PI * (p[0] - p[1]));
      if (k == 2) {
        m[0] = m[5] = m[10] = m[15] = cd{-PI * s, 0};
        m[3] = cmulx(cd{0, -PI * c}, cconj(es));
        m[12] = cmulx(cd{0, -PI * c}, es);
        m[6] = cmulx(cd{0, -PI * c}, ed);
        m[9] = cmulx(cd{0, -PI * c}, cconj(ed));
      } else {
        double sg = (k == 0) ? 1.0 : -1.0;
        m[3] = cscale(cconj(es), -TWO_PI * s);
        m[12] = cscale(es, TWO_PI * s);
        m[6] = cscale(ed, sg * TWO_PI * s);
        m[9] = cscale(cconj(ed), -sg * TWO_PI * s);
      }
      break;
    }
    default: break;  // parameter-free gates
  }
}

// parameter value of gate `gw` slot j
__device__ inline double gate_param(const int* gw, int j, const double* fvals, const double* theta,
                                    const double* xrow) {
  int s = gw[2 + j];
  if (s == -1) return fvals[gw[5] + j];
  if (s & ENC_FLAG) return xrow[s & ~ENC_FLAG];
  return theta[s];
}

// group unitary U = G_s ... G_1 in the group basis; returns d
__device__ inline int group_unitary(const int* W, int gid, const double* fvals, const double* theta,
                                    const double* xrow, cd* U) {
  const int* grp = W + sec_off(W, SEC_GROUPS) + gid * GROUP_WORDS;
  const int* gates = W + sec_off(W, SEC_GATES);
  int d = 1 << grp[GW_ARITY];
  mat_eye(U, d);
  cd G[16];
  for (int j = 0; j < grp[GW_NG]; ++j) {
    const int* gw = gates + (grp[GW_G0] + j) * GATE_WORDS;
    double p[3] = {0, 0, 0};
    for (int k = 0; k < gw[7]; ++k) p[k] = gate_param(gw, k, fvals, theta, xrow);
    gate_matrix_dev(gw[0], p, G);
    if (d == 4 && gw[1]) mat_swap_wires(G);
    mat_mul(G, U, U, d);
  }
  return d;
}

// fp32 table entry of a group: 2x2 (8 floats) / 4x4 (32 floats) row-major re,im; diagonal
// groups store 2^arity phase angles as int32 fixed-point turns (2^32 = one turn).
__device__ inline void group_table_entry(const int* W, int gid, const double* fvals,
                                         const double* theta, const double* xrow, float* out) {
  const int* grp = W + sec_off(W, SEC_GROUPS) + gid * GROUP_WORDS;
  cd U[16];
  int d = group_unitary(W, gid, fvals, theta, xrow, U);
  if (grp[GW_DIAG]) {
    int* o = reinterpret_cast<int*>(out);
    for (int e = 0; e < d; ++e) {
      double t = atan2(U[e * d + e].i, U[e * d + e].r) * 0.15915494309189533577;  // turns
      long long v = llrint(t * 4294967296.0);
      o[e] = (int)(unsigned int)(v & 0xffffffffll);
    }
  } else {
    for (int e = 0; e < d * d; ++e) {
      out[2 * e] = (float)U[e].r;
      out[2 * e + 1] = (float)U[e].i;
    }
    if (d == 2) {
      // Euler / tangent form of the one-qubit kernels (codegen._emit_euler_tan): U = e^{i d}
      // diag(1, e^{ia}) [[c, -s], [s, c]] diag(1, e^{ig}) -> c = |U00|, t = s / c,
      // e^{ia} = U10 conj(U00) / |.|, e^{ig} = U11 conj(U00) e^{-ia} / c^2 (fp64 here, once)
      const double c2 = U[0].r * U[0].r + U[0].i * U[0].i, c = sqrt(c2);
      cd ea = mk(U[2].r * U[0].r + U[2].i * U[0].i, U[2].i * U[0].r - U[2].r * U[0].i);
      const double ns = sqrt(ea.r * ea.r + ea.i * ea.i);
      ea = ns > 1e-300 ? cscale(ea, 1.0 / ns) : mk(1.0, 0.0);
      cd dd = mk(U[3].r * U[0].r + U[3].i * U[0].i, U[3].i * U[0].r - U[3].r * U[0].i);
      dd = c2 > 1e-300 ? cscale(dd, 1.0 / c2) : mk(1.0, 0.0);
      const cd eg = cmulx(dd, cconj(ea));
      out[8] = (float)c;
      out[9] = c2 > 1e-300 ? (float)(ns / c2) : 0.f;  // |U10| |U00| / |U00|^2 = s / c
      out[10] = (float)ea.r;
      out[11] = (float)ea.i;
      out[12] = (float)eg.r;
      out[13] = (float)eg.i;
      out[14] = c2 > 1e-300 ? (float)(U[0].r / c) : 1.f;  // e^{i d} = U00 / |U00|
      out[15] = c2 > 1e-300 ? (float)(U[0].i / c) : 0.f;
    }
  }
}

}  // namespace lsq
