// lsq_pass.cuh -- the tile-pass kernel: one HBM round trip of a state batch through a
// group of fused gate layers (forward), the turnaround (<Z_q>, lambda = O psi), or the
// adjoint step (un-apply + per-group coupling matrices), on sm_100a.
//
// Replaces, for a whole block of layers at once, the reference's per-position passes
// (_fastops.pyx:93-125 apply_1q/apply_2q, kernels.py:579-637) and the per-position
// coupling einsums of the backward sweep (grad.py:40-73, 102-140).
//
// Execution model (see schedule.py for the host side):
//   * one CTA owns `tiles_per_cta` tiles of one batch row; a tile is 2^M amplitudes whose
//     index bits are the pass's M "local" physical bits;
//   * every thread holds 2^R amplitudes per state vector in registers; a "phase" fixes
//     which R local bits are register bits. Non-diagonal groups act only on register bits
//     (compile-time register indices via dispatch), diagonal groups on any bit;
//   * phases are separated by a transpose through XOR-swizzled shared memory;
//   * the first/last phase put local bits 0..3 (= physical bits 0..3) on lanes 0..15, so
//     every warp load/store touches whole 128-byte lines;
//   * coupling sums: per-thread fp32 -> warp shuffle tree -> per-warp shared slots
//     accumulated over the CTA's tiles -> fp64 per-CTA partials (deterministic order).
#pragma once
#include <type_traits>

#include "lsq_common.cuh"
#include "lsq_prims.cuh"

namespace lsq {

constexpr int MODE_FWD = 0, MODE_TURN = 1, MODE_BWD = 2;
constexpr int F_SYNTH = 1,      // input psi is |0..0> (not read)
    F_STORE_PSI = 2,            // write psi at the end of the pass
    F_STORE_LAM = 4,            // write lambda at the end of the pass
    F_ZPART = 8,                // forward: accumulate <Z_q> partials of the output
    F_NOFWD = 16;               // turnaround on a given final state: skip the forward ops


template <int R>
struct Layout {
  uint32_t tp;     // local index bits owned by the thread index
  uint32_t gt;     // physical offset of tp
  uint32_t st;     // swizzled shared index of tp
  uint32_t gr[R];  // physical offset of register bit k
  uint32_t sr[R];  // swizzled shared offset of register bit k
};

template <int M, int R>
__device__ __forceinline__ void make_layout(const int* ph, const int* pbit, int tid, Layout<R>& L) {
  uint32_t tp = 0, gt = 0;
#pragma unroll
  for (int j = 0; j < M - R; ++j) {
    if ((tid >> j) & 1) {
      int lb = ph[5 + j];
      tp |= 1u << lb;
      gt |= 1u << pbit[lb];
    }
  }
  L.tp = tp;
  L.gt = gt;
  L.st = swz(tp);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    int lb = ph[k];
    L.gr[k] = 1u << pbit[lb];
    L.sr[k] = swz(1u << lb);
  }
}

template <int R>
__device__ __forceinline__ uint32_t gofs(const Layout<R>& L, int i) {
  uint32_t r = L.gt;
#pragma unroll
  for (int k = 0; k < R; ++k)
    if ((i >> k) & 1) r |= L.gr[k];
  return r;
}
template <int R>
__device__ __forceinline__ uint32_t sofs(const Layout<R>& L, int i) {
  uint32_t r = L.st;
#pragma unroll
  for (int k = 0; k < R; ++k)
    if ((i >> k) & 1) r ^= L.sr[k];
  return r;
}

// ---- compile-time dispatch on register-bit indices ---------------------------------------
template <int R, int K = 0, typename F>
__device__ __forceinline__ void dispatch1(int k, F&& f) {
  if constexpr (K < R) {
    if (k == K)
      f(std::integral_constant<int, K>{});
    else
      dispatch1<R, K + 1>(k, f);
  }
}
template <int R, int A = 0, int B = 0, typename F>
__device__ __forceinline__ void dispatch2(int a, int b, F&& f) {
  if constexpr (A < R) {
    if constexpr (B < R) {
      if constexpr (A != B) {
        if (a == A && b == B) {
          f(std::integral_constant<int, A>{}, std::integral_constant<int, B>{});
          return;
        }
      }
      dispatch2<R, A, B + 1>(a, b, f);
    } else {
      dispatch2<R, A + 1, 0>(a, b, f);
    }
  }
}

// ---- diagonal runs ----------------------------------------------------------------------------
// Every diagonal group is a pure phase (unitary diagonal); a run of consecutive diagonal
// groups becomes one accumulated phase per amplitude in 32-bit fixed-point turns (exact
// modular addition), then one sincospi per amplitude.
template <int R>
struct DiagCtx {
  uint32_t tp;       // thread local bits
  uint64_t tbase;    // tile physical base (within the row)
};

__device__ __forceinline__ int src_const_bit(int s, uint32_t tp, uint64_t tbase) {
  int kind = s >> 8, v = s & 0xff;
  if (kind == SRC_THREAD) return (tp >> v) & 1;
  return (int)((tbase >> v) & 1);  // SRC_NONLOCAL
}

template <int R>
__device__ __forceinline__ void drun_angles(const int* subs, int nsub, const float* smat,
                                            uint32_t tp, uint64_t tbase, int32_t (&ph)[1 << R]) {
  int32_t c = 0;
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) ph[i] = 0;
  for (int s = 0; s < nsub; ++s) {
    const int* sw = subs + s * SUB_WORDS;
    const int* ang = reinterpret_cast<const int*>(smat + sw[3]);
    const int sa = sw[0], sb = sw[1], ar = sw[5];
    const int ka = sa >> 8, kb = sb >> 8;
    if (ar == 1) {
      if (ka == SRC_REG) {
        const int32_t lo = ang[0], hi = ang[1];
        dispatch1<R>(sa & 0xff, [&](auto K) {
#pragma unroll
          for (int i = 0; i < (1 << R); ++i) ph[i] += ((i >> K.value) & 1) ? hi : lo;
        });
      } else {
        c += ang[src_const_bit(sa, tp, tbase)];
      }
      continue;
    }
    if (ka != SRC_REG && kb != SRC_REG) {
      c += ang[2 * src_const_bit(sa, tp, tbase) + src_const_bit(sb, tp, tbase)];
    } else if (ka == SRC_REG && kb != SRC_REG) {
      const int bb = src_const_bit(sb, tp, tbase);
      const int32_t lo = ang[bb], hi = ang[2 + bb];
      dispatch1<R>(sa & 0xff, [&](auto K) {
#pragma unroll
        for (int i = 0; i < (1 << R); ++i) ph[i] += ((i >> K.value) & 1) ? hi : lo;
      });
    } else if (ka != SRC_REG && kb == SRC_REG) {
      const int ba = src_const_bit(sa, tp, tbase);
      const int32_t lo = ang[2 * ba], hi = ang[2 * ba + 1];
      dispatch1<R>(sb & 0xff, [&](auto K) {
#pragma unroll
        for (int i = 0; i < (1 << R); ++i) ph[i] += ((i >> K.value) & 1) ? hi : lo;
      });
    } else {
      int a = sa & 0xff, b = sb & 0xff;
      int32_t t0 = ang[0], t1 = ang[1], t2 = ang[2], t3 = ang[3];
      if (a > b) {  // swap roles: idx' = 2*b(B) + b(A)
        int tmp = a; a = b; b = tmp;
        int32_t u = t1; t1 = t2; t2 = u;
      }
      dispatch2<R>(a, b, [&](auto A, auto B) {
#pragma unroll
        for (int i = 0; i < (1 << R); ++i) {
          const int idx = 2 * ((i >> A.value) & 1) + ((i >> B.value) & 1);
          ph[i] += idx == 0 ? t0 : idx == 1 ? t1 : idx == 2 ? t2 : t3;
        }
      });
    }
  }
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) ph[i] += c;
}

template <int R, int NV>
__device__ __forceinline__ void apply_phases(const int32_t (&ph)[1 << R], float2 (*v)[1 << R], bool inverse) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) {
    float s, c;
    sincospif((float)ph[i] * 4.656612873077393e-10f, &s, &c);  // ph * 2^-31 half-turns
    if (inverse) s = -s;
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q][i] = cm(c, s, v[q][i]);
  }
}

// couplings of a diagonal run: M_e = sum conj(l) p over amplitudes with local index e.
// conj(l) p is recomputed per sub-op (no 2^R-entry temporary -> no register spills).

template <int NT, int R>
__device__ __forceinline__ void drun_couplings(const int* subs, int nsub, const float2* p, const float2* l,
                                               uint32_t tp, uint64_t tbase, float* wacc) {
  for (int s = 0; s < nsub; ++s) {
    const int* sw = subs + s * SUB_WORDS;
    const int slot = sw[4];
    if (slot < 0) continue;
    const int sa = sw[0], sb = sw[1], ar = sw[5];
    const int ka = sa >> 8, kb = sb >> 8;
    float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const bool ra = ka == SRC_REG, rb = (ar == 2) && kb == SRC_REG;
    if (!ra && !rb) {
      float tx = 0, ty = 0;
#pragma unroll
      for (int i = 0; i < (1 << R); ++i) { const float2 c = cjmul(l[i], p[i]); tx += c.x; ty += c.y; }
      const int e = ar == 1 ? src_const_bit(sa, tp, tbase)
                            : 2 * src_const_bit(sa, tp, tbase) + src_const_bit(sb, tp, tbase);
      v[2 * e] = tx;
      v[2 * e + 1] = ty;
    } else if (ra != rb) {
      // one register source: split by that register bit; the other index bit is constant
      const int k = ra ? (sa & 0xff) : (sb & 0xff);
      float a0x = 0, a0y = 0, a1x = 0, a1y = 0;
      dispatch1<R>(k, [&](auto K) {
#pragma unroll
        for (int i = 0; i < (1 << R); ++i) {
          const float2 c = cjmul(l[i], p[i]);
          if ((i >> K.value) & 1) { a1x += c.x; a1y += c.y; }
          else { a0x += c.x; a0y += c.y; }
        }
      });
      int e0, e1;
      if (ar == 1) { e0 = 0; e1 = 1; }
      else if (ra) { const int bb = src_const_bit(sb, tp, tbase); e0 = bb; e1 = 2 + bb; }
      else { const int ba = src_const_bit(sa, tp, tbase); e0 = 2 * ba; e1 = 2 * ba + 1; }
      v[2 * e0] = a0x; v[2 * e0 + 1] = a0y; v[2 * e1] = a1x; v[2 * e1 + 1] = a1y;
    } else {
      dispatch2<R>(sa & 0xff, sb & 0xff, [&](auto A, auto B) {
#pragma unroll
        for (int i = 0; i < (1 << R); ++i) {
          const float2 c = cjmul(l[i], p[i]);
          const int e = 2 * ((i >> A.value) & 1) + ((i >> B.value) & 1);
          v[2 * e] += c.x;
          v[2 * e + 1] += c.y;
        }
      });
    }
    warp_accumulate<NT, 8>(v, wacc + slot);
  }
}

// ---- the kernel ---------------------------------------------------------------------------------
template <int M, int R, int NV>
__global__ void __launch_bounds__(1 << (M - R), (NV == 1 && (1 << (M - R)) <= 256) ? 2 : 1)
    lsq_pass_kernel(PassArgs A) {
  constexpr int NT = 1 << (M - R);
  constexpr int NR = 1 << R;
  constexpr int NW = (NT + 31) / 32;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  const int* W = A.prog;
  const int* pw = W + sec_off(W, SEC_PASSES) + A.pass * PASS_WORDS;
  const int nph = pw[PW_NPH];
  const int matf = pw[PW_MATF];
  const int slotf = pw[PW_SLOTF];
  const int n = A.n;

  // ---- shared memory carve-up
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* s_x = reinterpret_cast<float2*>(smem_raw);
  int* s_ph = reinterpret_cast<int*>(s_x + (1 << M));
  int* s_ops = s_ph + nph * PHASE_WORDS;
  int* s_subs = s_ops + pw[PW_OPN] * OP_WORDS;
  int* s_pbit = s_subs + pw[PW_SUBN] * SUB_WORDS;  // 32 physical bits of local bits
  int* s_nbit = s_pbit + 32;                         // 32 nonlocal physical bits
  float* s_mat = reinterpret_cast<float*>(s_nbit + 32);
  float* s_acc = s_mat + ((matf + 3) & ~3);
  double* s_z = reinterpret_cast<double*>(s_acc + ((NW * slotf + 3) & ~3));
  float* s_red = reinterpret_cast<float*>(s_z + 34);

  // ---- stage the pass program, physical bit maps, group table
  {
    const int* gph = W + sec_off(W, SEC_PHASES) + pw[PW_PH0] * PHASE_WORDS;
    for (int i = tid; i < nph * PHASE_WORDS; i += NT) s_ph[i] = gph[i];
    const int* gop = W + sec_off(W, SEC_OPS) + pw[PW_OPLO] * OP_WORDS;
    for (int i = tid; i < pw[PW_OPN] * OP_WORDS; i += NT) s_ops[i] = gop[i];
    const int* gsub = W + sec_off(W, SEC_SUBS) + pw[PW_SUBLO] * SUB_WORDS;
    for (int i = tid; i < pw[PW_SUBN] * SUB_WORDS; i += NT) s_subs[i] = gsub[i];
    if (tid == 0) {
      const uint32_t mask = (uint32_t)pw[PW_MASK];
      int l = 0, q = 0;
      for (int p = 0; p < n; ++p) {
        if ((mask >> p) & 1) s_pbit[l++] = p;
        else s_nbit[q++] = p;
      }
    }
    const int row = blockIdx.x / A.ctas_per_row;
    const int* pg = W + sec_off(W, SEC_PGROUPS) + pw[PW_PG0] * PGROUP_WORDS;
    const int* groups = W + sec_off(W, SEC_GROUPS);
    for (int g = tid; g < pw[PW_NGRP]; g += NT) {
      const int gid = pg[g * PGROUP_WORDS], moff = pg[g * PGROUP_WORDS + 1];
      const int* grp = groups + gid * GROUP_WORDS;
      if (grp[GW_PERROW]) {
        const float* src = A.rowtab + ((size_t)row * A.nperrow + grp[GW_ROWIDX]) * 32;
        for (int e = 0; e < grp[GW_MATF]; ++e) s_mat[moff + e] = src[e];
      } else {
        const float* src = A.gmats + (size_t)gid * 32;
        for (int e = 0; e < grp[GW_MATF]; ++e) s_mat[moff + e] = src[e];
      }
    }
    for (int i = tid; i < NW * slotf; i += NT) s_acc[i] = 0.f;
    for (int i = tid; i < 34; i += NT) s_z[i] = 0.0;
  }
  __syncthreads();

  const int row = blockIdx.x / A.ctas_per_row;
  const int cslot = blockIdx.x % A.ctas_per_row;
  const size_t rowbase = (size_t)row << n;
  const int mode = A.mode, flags = A.flags;
  float* wacc = s_acc + warp * slotf;

  float2 v[NV][NR];  // v[0] = psi, v[1] = lambda

  auto exchange = [&](const Layout<R>& from, const Layout<R>& to) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      __syncthreads();
#pragma unroll
      for (int i = 0; i < NR; ++i) s_x[sofs<R>(from, i)] = v[q][i];
      __syncthreads();
#pragma unroll
      for (int i = 0; i < NR; ++i) v[q][i] = s_x[sofs<R>(to, i)];
    }
  };

  // forward ops of phase `ph`
  auto run_fwd = [&](int ph, const Layout<R>& L, uint64_t tbase) {
    const int* phw = s_ph + ph * PHASE_WORDS;
    const int o0 = phw[PH_OP0] - pw[PW_OPLO], no = phw[PH_NOPS];
    for (int o = o0; o < o0 + no; ++o) {
      const int* op = s_ops + o * OP_WORDS;
      const int kind = op[0];
      if (kind == OP_U1) {
        float m[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) m[e] = s_mat[op[5] + e];
        dispatch1<R>(op[1], [&](auto K) { u1_apply<R, K.value>(v[0], m); });
      } else if (kind == OP_PCX) {
        dispatch2<R>(op[1], op[2], [&](auto KC, auto KT) { perm_cx<R, KC.value, KT.value>(v[0]); });
      } else if (kind == OP_PX) {
        dispatch1<R>(op[1], [&](auto K) { perm_x<R, K.value>(v[0]); });
      } else if (kind == OP_U2) {
        float m[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) m[e] = s_mat[op[5] + e];
        dispatch2<R>(op[1], op[2], [&](auto KA, auto KB) { u2_apply<R, KA.value, KB.value>(v[0], m); });
      } else {
        int32_t ph_[NR];
        drun_angles<R>(s_subs + (op[6] - pw[PW_SUBLO]) * SUB_WORDS, op[7], s_mat, L.tp, tbase, ph_);
        apply_phases<R, 1>(ph_, v, false);
      }
    }
  };

  // adjoint ops of phase `ph` (reverse order): couplings at the post-group point, then U^dag
  auto run_bwd = [&](int ph, const Layout<R>& L, uint64_t tbase) {
    const int* phw = s_ph + ph * PHASE_WORDS;
    const int o0 = phw[PH_OP0] - pw[PW_OPLO], no = phw[PH_NOPS];
    for (int o = o0 + no - 1; o >= o0; --o) {
      const int* op = s_ops + o * OP_WORDS;
      const int kind = op[0];
      if (kind == OP_PCX) {
        dispatch2<R>(op[1], op[2], [&](auto KC, auto KT) {
#pragma unroll
          for (int q = 0; q < NV; ++q) perm_cx<R, KC.value, KT.value>(v[q]);
        });
      } else if (kind == OP_PX) {
        dispatch1<R>(op[1], [&](auto K) {
#pragma unroll
          for (int q = 0; q < NV; ++q) perm_x<R, K.value>(v[q]);
        });
      } else if (kind == OP_U1) {
        const float* g = s_mat + op[5];
        if constexpr (NV == 2) {
          if (op[4] >= 0) {
            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            dispatch1<R>(op[1], [&](auto K) { u1_coupling<R, K.value>(v[0], v[1], acc); });
            warp_accumulate<NT, 8>(acc, wacc + op[4]);
          }
        }
        // U^dag = conj transpose
        const float m[8] = {g[0], -g[1], g[4], -g[5], g[2], -g[3], g[6], -g[7]};
        dispatch1<R>(op[1], [&](auto K) {
#pragma unroll
          for (int q = 0; q < NV; ++q) u1_apply<R, K.value>(v[q], m);
        });
      } else if (kind == OP_U2) {
        const float* g = s_mat + op[5];
        if constexpr (NV == 2) {
          if (op[4] >= 0) {
            dispatch2<R>(op[1], op[2], [&](auto KA, auto KB) {
              auto row = [&](auto RRc) {
                float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                u2_coupling_row<R, KA.value, KB.value, RRc.value>(v[0], v[1], acc);
                warp_accumulate<NT, 8>(acc, wacc + op[4] + 8 * RRc.value);
              };
              row(std::integral_constant<int, 0>{});
              row(std::integral_constant<int, 1>{});
              row(std::integral_constant<int, 2>{});
              row(std::integral_constant<int, 3>{});
            });
          }
        }
        // U^dag straight from the shared table (conj transpose)
        dispatch2<R>(op[1], op[2], [&](auto KA, auto KB) {
#pragma unroll
          for (int q = 0; q < NV; ++q) u2_apply_dag<R, KA.value, KB.value>(v[q], g);
        });
      } else {
        const int* subs = s_subs + (op[6] - pw[PW_SUBLO]) * SUB_WORDS;
        if constexpr (NV == 2) drun_couplings<NT, R>(subs, op[7], v[0], v[1], L.tp, tbase, wacc);
        int32_t ph_[NR];
        drun_angles<R>(subs, op[7], s_mat, L.tp, tbase, ph_);
        apply_phases<R, NV>(ph_, v, true);
      }
    }
  };

  const int ntl = n - M;
  const int t0 = cslot * A.tiles_per_cta;
  for (int t = t0; t < t0 + A.tiles_per_cta; ++t) {
    uint64_t tbase = 0;
    for (int j = 0; j < ntl; ++j)
      if ((t >> j) & 1) tbase |= 1ull << s_nbit[j];
    const size_t base = rowbase + tbase;

    Layout<R> L;
    const bool nofwd = (mode == MODE_BWD) || (mode == MODE_TURN && (flags & F_NOFWD));
    const int first = nofwd ? nph - 1 : 0;
    make_layout<M, R>(s_ph + first * PHASE_WORDS, s_pbit, tid, L);

    // ---- load
    if (!nofwd && (flags & F_SYNTH)) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const bool one = (tbase | gofs<R>(L, i)) == 0;
        v[0][i] = make_float2(one ? 1.f : 0.f, 0.f);
      }
    } else {
#pragma unroll
      for (int i = 0; i < NR; ++i) v[0][i] = __ldcs(A.psi_in + base + gofs<R>(L, i));
    }
    if constexpr (NV == 2) {
      if (mode == MODE_BWD) {
#pragma unroll
        for (int i = 0; i < NR; ++i) v[1][i] = __ldcs(A.lam + base + gofs<R>(L, i));
      }
    }

    if (!nofwd) {
      for (int ph = 0; ph < nph; ++ph) {
        run_fwd(ph, L, tbase);
        if (ph + 1 < nph) {
          Layout<R> L2;
          make_layout<M, R>(s_ph + (ph + 1) * PHASE_WORDS, s_pbit, tid, L2);
          exchange(L, L2);
          L = L2;
        }
      }
    }

    if (mode == MODE_TURN || (flags & F_ZPART)) {
      // <Z> partials: per local bit D_l = sum (-1)^bit |psi|^2, S = sum |psi|^2
      float pz[M + 1];
#pragma unroll
      for (int e = 0; e <= M; ++e) pz[e] = 0.f;
      float S = 0.f;
      float Dk[R];
#pragma unroll
      for (int k = 0; k < R; ++k) Dk[k] = 0.f;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const float pr = v[0][i].x * v[0][i].x + v[0][i].y * v[0][i].y;
        S += pr;
#pragma unroll
        for (int k = 0; k < R; ++k) Dk[k] += ((i >> k) & 1) ? -pr : pr;
      }
      // scatter into local-bit order
      const int* phw = s_ph + ((mode == MODE_BWD) ? 0 : (nph - 1)) * PHASE_WORDS;
      pz[M] = S;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int lb = phw[k];
#pragma unroll
        for (int e = 0; e < M; ++e)
          if (e == lb) pz[e] += Dk[k];
      }
#pragma unroll
      for (int j = 0; j < M - R; ++j) {
        const int lb = phw[5 + j];
        const float sgn = ((L.tp >> lb) & 1) ? -S : S;
#pragma unroll
        for (int e = 0; e < M; ++e)
          if (e == lb) pz[e] += sgn;
      }
      warp_sum<NT, M + 1>(pz);
      if ((tid & 31) == 0) {
#pragma unroll
        for (int e = 0; e <= M; ++e) s_red[warp * (M + 1) + e] = pz[e];
      }
      __syncthreads();
      if (tid == 0) {
        double tot[M + 1];
        for (int e = 0; e <= M; ++e) {
          double s = 0.0;
          for (int w = 0; w < NW; ++w) s += (double)s_red[w * (M + 1) + e];
          tot[e] = s;
        }
        for (int e = 0; e < M; ++e) s_z[s_pbit[e]] += tot[e];
        for (int j = 0; j < ntl; ++j) {
          const int p = s_nbit[j];
          s_z[p] += ((tbase >> p) & 1) ? -tot[M] : tot[M];
        }
        s_z[n] += tot[M];
      }
      __syncthreads();
    }

    if constexpr (NV == 2) {
      if (mode == MODE_TURN) {
        // lambda = O psi, O = sum_q w_q Z_q (weights per wire q = n-1-p)
        const int* phw = s_ph + (nph - 1) * PHASE_WORDS;
        float base_o = 0.f;
        for (int j = 0; j < M - R; ++j) {
          const int lb = phw[5 + j];
          const int p = s_pbit[lb];
          const float w = A.wts ? (float)A.wts[n - 1 - p] : 1.f;
          base_o += ((L.tp >> lb) & 1) ? -w : w;
        }
        for (int j = 0; j < ntl; ++j) {
          const int p = s_nbit[j];
          const float w = A.wts ? (float)A.wts[n - 1 - p] : 1.f;
          base_o += ((tbase >> p) & 1) ? -w : w;
        }
        float wk[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const int p = s_pbit[phw[k]];
          wk[k] = A.wts ? (float)A.wts[n - 1 - p] : 1.f;
        }
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          float o = base_o;
#pragma unroll
          for (int k = 0; k < R; ++k) o += ((i >> k) & 1) ? -wk[k] : wk[k];
          v[1][i] = make_float2(o * v[0][i].x, o * v[0][i].y);
        }
      }
      if (mode == MODE_TURN || mode == MODE_BWD) {
        for (int ph = nph - 1; ph >= 0; --ph) {
          run_bwd(ph, L, tbase);
          if (ph > 0) {
            Layout<R> L2;
            make_layout<M, R>(s_ph + (ph - 1) * PHASE_WORDS, s_pbit, tid, L2);
            exchange(L, L2);
            L = L2;
          }
        }
      }
    }

    // ---- store
    if (flags & F_STORE_PSI) {
#pragma unroll
      for (int i = 0; i < NR; ++i) __stcs(A.psi_out + base + gofs<R>(L, i), v[0][i]);
    }
    if constexpr (NV == 2) {
      if (flags & F_STORE_LAM) {
#pragma unroll
        for (int i = 0; i < NR; ++i) __stcs(A.lam + base + gofs<R>(L, i), v[1][i]);
      }
    }
  }

  // ---- flush partials (fixed summation order -> deterministic)
  __syncthreads();
  if (slotf > 0 && A.part) {
    double* dst = A.part + (size_t)blockIdx.x * slotf;
    for (int f = tid; f < slotf; f += NT) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += (double)s_acc[w * slotf + f];
      dst[f] = s;
    }
  }
  if ((mode == MODE_TURN || (flags & F_ZPART)) && A.zpart) {
    double* dst = A.zpart + (size_t)blockIdx.x * (n + 1);
    for (int f = tid; f <= n; f += NT) dst[f] = s_z[f];
  }
}

}  // namespace lsq
