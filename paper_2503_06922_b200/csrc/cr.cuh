// Block cyclic reduction (CR) for the 6x6 block-tridiagonal SPD systems, on
// a whole-CTA team: the latency mode (one scenario per SM).
//
// Replaces the reference's per-solve SuperLU factorisations (solver.py:229-247
// ADMM KKT, _solve_active_subset 500-528, _solve_equality_direct 388-421)
// after the exact reduction of SURVEY §7.1, like the twisted LDL^T of
// linalg.cuh -- but with ceil(log2 N) dependent levels, each parallel over
// its blocks, instead of a chain of ~N/2 dependent 6x6 steps.  With a 16-warp
// CTA every level of an N = 101 system is a single pass.
//
// Elimination order: block i > 0 is eliminated at level l = ctz(i), against
// its level-l neighbours h = i - 2^l and j = i + 2^l (if j < N); block 0 is
// the root.  With M_{a,b} the current coupling block:
//   Dinv_i = D_i^{-1},  L_i = M_{h,i} Dinv_i,  R_i = M_{j,i} Dinv_i
//   D_h -= L_i M_{h,i}^T,  D_j -= R_i M_{i,j},  M_{h,j} = -L_i M_{i,j}
// Storage: D[N][kDiag] packed symmetric (D_i, then Dinv_i) and one array
// LR[2N][36]: L = LR (L[i] holds the coupling C(i) = M_{i-1,i} before the
// factorisation, so `HU = LR + 36` indexes U_k = M_{k,k+1} exactly as the
// twisted layout does) and R = LR + 36 N.  Every new coupling M_{h,j} is
// written to L[j].  A solve M x = v, in place (x overwrites v):
//   forward  (l = 0 ..)  v_j -= R_{j-2^l} v_{j-2^l} + L_{j+2^l} v_{j+2^l}  (survivors j)
//   root     x_0 = Dinv_0 v_0
//   backward (l = .. 0)  x_i = Dinv_i v_i - L_i^T x_h - R_i^T x_j          (eliminated i)
// Work is mapped on 6-lane groups (five per warp, lanes 30-31 idle): lane r
// of a group owns row r of its block, so the packed-row offsets of Dinv are
// fixed per thread.
#pragma once
#include "linalg.cuh"

namespace accfem {

DEV int cr_levels(int N) {
  int l = 0;
  while ((1 << l) < N) ++l;
  return l;
}
// blocks eliminated at level l
DEV int cr_elim_count(int N, int l) {
  const int s = 1 << l;
  return s <= N - 1 ? ((N - 1 - s) >> (l + 1)) + 1 : 0;
}
// survivors of level l (multiples of 2^(l+1) below N)
DEV int cr_surv_count(int N, int l) { return ((N - 1) >> (l + 1)) + 1; }

struct CrF {
  double* D;  // N x kDiag
  double* L;  // N x 36 (L[0] unused)
  double* R;  // N x 36 (R[0] unused)
};
// the CR factor behind a twisted-layout (D, U) pair: U = L + 36, R = L + 36 N
DEV CrF cr_of(int N, double* D, const double* U) {
  double* L = const_cast<double*>(U) - 36;
  return CrF{D, L, L + 36L * N};
}

#if defined(__CUDACC__)
#if defined(CR_TIMING)
__device__ long long g_cr_t[64];
__shared__ long long s_cr_t[32];
#define CR_T(k) do { if (threadIdx.x == 0) s_cr_t[k] = clock64(); } while (0)
#else
#define CR_T(k)
#endif
// A CTA team whose block-tridiagonal algebra is cyclic reduction.
struct TeamCR : TeamCta {
  DEV explicit TeamCR(const TeamCta& t) : TeamCta(t) {}
};

// returns the smallest failing block, or -1
static __device__ __noinline__ int cr_factor(const TeamCR& team, int N, CrF F) {
  const int Lv = cr_levels(N);
  const int lane = team.w.lane, grp = lane / 6, r = lane - 6 * grp;
  const bool glane = lane < 30;
  const int gid = 5 * team.warp + grp, ngr = 5 * team.nw;
  int fail = N;
  for (int l = 0; l < Lv; ++l) {
    const int s = 1 << l, ne = cr_elim_count(N, l);
    for (int q0 = 0; q0 < ne; q0 += ngr) {
      const int q = q0 + gid;
      const bool act = glane && q < ne;
      const int i = s + 2 * s * q, h = i - s, j = i + s;
      const bool hj = act && j < N;
      double dl[6] = {0, 0, 0, 0, 0, 0}, dr[6], nc[6], Lr[6], Rr[6], Di[36];
      if (act) {
        double Dm[36];
        unpack_sym(F.D + kDiag * i, Dm);
        if (!spd6_inv(Dm, Di)) fail = min(fail, i);
        const double* Cl = F.L + 36 * i;
        const double* Cr = F.L + 36 * (hj ? j : i);
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          double a = 0.0, b = 0.0;
#pragma unroll
          for (int t = 0; t < 6; ++t) {
            a += Cl[6 * r + t] * Di[6 * t + c];
            b += Cr[6 * t + r] * Di[6 * t + c];
          }
          Lr[c] = a;
          Rr[c] = hj ? b : 0.0;
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          double a = 0.0, b = 0.0, e = 0.0;
#pragma unroll
          for (int t = 0; t < 6; ++t) {
            a += Lr[t] * Cl[6 * c + t];
            b += Rr[t] * Cr[6 * t + c];
            e += Lr[t] * Cr[6 * t + c];
          }
          dl[c] = a;
          dr[c] = b;
          nc[c] = -e;
        }
      }
      __syncwarp();  // the group has read C(i) and C(j) before they are overwritten
      if (act) {
        if (r == 0) pack_sym(F.D + kDiag * i, Di);
        st6(F.L + 36 * i + 6 * r, Lr);
        st6(F.R + 36 * i + 6 * r, Rr);
        if (hj) {
          st6(F.L + 36 * j + 6 * r, nc);
          double* Dj = F.D + kDiag * j + r * (r + 1) / 2;
#pragma unroll
          for (int c = 0; c < 6; ++c)
            if (c <= r) Dj[c] -= dr[c];
        }
      }
      team.sync();  // D_h may also be D_j of the group to the left: two phases
      if (act) {
        double* Dh = F.D + kDiag * h + r * (r + 1) / 2;
#pragma unroll
        for (int c = 0; c < 6; ++c)
          if (c <= r) Dh[c] -= dl[c];
      }
      team.sync();
    }
  }
  if (team.rank() == 0) {
    double Dm[36], Di[36];
    unpack_sym(F.D, Dm);
    if (!spd6_inv(Dm, Di)) fail = min(fail, 0);
    pack_sym(F.D, Di);
  }
  fail = team.imin(fail);
  return fail < N ? fail : -1;
}

DEV double cr_fwd_row(int N, const CrF& F, const double* vg, int j, int s, int r) {
  double a = vg[6 * j + r], b = 0.0;
  if (j > 0) {
    const double* Rm = F.R + 36 * (j - s) + 6 * r;
    const double* w = vg + 6 * (j - s);
    a -= (Rm[0] * w[0] + Rm[2] * w[2] + Rm[4] * w[4]) + (Rm[1] * w[1] + Rm[3] * w[3] + Rm[5] * w[5]);
  }
  if (j + s < N) {
    const double* Lm = F.L + 36 * (j + s) + 6 * r;
    const double* w = vg + 6 * (j + s);
    b = (Lm[0] * w[0] + Lm[2] * w[2] + Lm[4] * w[4]) + (Lm[1] * w[1] + Lm[3] * w[3] + Lm[5] * w[5]);
  }
  return a - b;
}
DEV double cr_bwd_row(int N, const CrF& F, const double* vg, int i, int s, int r, const int* so) {
  const int h = i - s, j = i + s;
  const double* Dm = F.D + kDiag * i;
  const double* vi = vg + 6 * i;
  const double a0 = Dm[so[0]] * vi[0] + Dm[so[2]] * vi[2] + Dm[so[4]] * vi[4];
  const double a1 = Dm[so[1]] * vi[1] + Dm[so[3]] * vi[3] + Dm[so[5]] * vi[5];
  const double* Lm = F.L + 36 * i + r;
  const double* xh = vg + 6 * h;
  const double b0 = Lm[0] * xh[0] + Lm[12] * xh[2] + Lm[24] * xh[4];
  const double b1 = Lm[6] * xh[1] + Lm[18] * xh[3] + Lm[30] * xh[5];
  double c0 = 0.0, c1 = 0.0;
  if (j < N) {
    const double* Rm = F.R + 36 * i + r;
    const double* xj = vg + 6 * j;
    c0 = Rm[0] * xj[0] + Rm[12] * xj[2] + Rm[24] * xj[4];
    c1 = Rm[6] * xj[1] + Rm[18] * xj[3] + Rm[30] * xj[5];
  }
  return (a0 + a1) - ((b0 + b1) + (c0 + c1));
}
DEV double cr_root_row(const CrF& F, const double* vg, int r, const int* so) {
  const double* Dm = F.D;
  const double a0 = Dm[so[0]] * vg[0] + Dm[so[2]] * vg[2] + Dm[so[4]] * vg[4];
  const double a1 = Dm[so[1]] * vg[1] + Dm[so[3]] * vg[3] + Dm[so[5]] * vg[5];
  return a0 + a1;
}

// In-place solve of nrhs right-hand sides v_g = v + g*stride (x overwrites v).
// (rhs, block) items are spread over the groups; the top levels, whose items
// fit in the five groups of warp 0, run on warp 0 alone with warp barriers.
// In the backward sweep a group reads all of v_i before any lane writes x_i.
static __device__ __noinline__ void cr_solve_inplace(const TeamCR& team, int N, CrF F, double* v, int nrhs, long stride,
                                                     const int* rhs_block = nullptr) {
  const int Lv = cr_levels(N);
  const int lane = team.w.lane, grp = lane / 6, r = lane - 6 * grp;
  const bool glane = lane < 30;
  const int gid = 5 * team.warp + grp, ngr = 5 * team.nw;
  int so[6];
#pragma unroll
  for (int t = 0; t < 6; ++t) so[t] = sidx(r, t);
  // levels with at most kTail items run on warp 0 alone (warp barriers, up to
  // three passes of its five groups) instead of a CTA barrier each: measured
  // faster for N = 1001 (cfg5 -9 %), slower for N = 101 (+4 %)
  const int kTail = (nrhs == 1 && N > 256) ? 15 : 5;
  int ltop = 0;
  while (ltop < Lv && cr_surv_count(N, ltop) * nrhs > kTail) ++ltop;
  CR_T(0);
  for (int l = 0; l < ltop; ++l) {
    const int s = 1 << l, ns = cr_surv_count(N, l);
    // two items per group per pass: both rows' loads are in flight before
    // either store (items of one level never touch each other's rows)
    // rhs_block: right-hand side g is zero outside block rhs_block[g], so after
    // this level it is zero outside the (at most two) survivors j with
    // |j - rhs_block[g]| < 2s; the other survivors' rows are exact zeros and
    // are skipped (identical results, O(log N) forward items per right-hand side)
    const int items = rhs_block ? 2 * nrhs : nrhs * ns;
    if (glane)
      for (int u0 = gid; u0 < items; u0 += 2 * ngr) {
        double a[2];
        double* dst[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int u = u0 + k * ngr;
          dst[k] = nullptr;
          if (u < items) {
            int g, j;
            bool live = true;
            if (rhs_block) {
              g = u >> 1;
              const int kb = rhs_block[g], j0 = kb / (2 * s) * (2 * s);
              j = j0 + (u & 1) * 2 * s;
              live = (u & 1) == 0 || (kb > j0 && j / (2 * s) < ns);
            } else {
              const int q = nrhs == 1 ? u : u / nrhs;  // block-major: neighbouring groups share the factor rows
              g = u - q * nrhs;
              j = 2 * s * q;
            }
            if (live) {
              double* vg = v + g * stride;
              a[k] = cr_fwd_row(N, F, vg, j, s, r);
              dst[k] = vg + 6 * j + r;
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (dst[k]) *dst[k] = a[k];
      }
    team.sync();
    CR_T(1 + l);
  }
  if (nrhs == 1) {
    // single right-hand side: the top levels on warp 0, groups strided over the blocks
    if (team.warp == 0 && glane) {
      const unsigned m = 0x3fffffffu;
      for (int l = ltop; l < Lv; ++l) {
        const int s = 1 << l, ns = cr_surv_count(N, l);
        for (int q = grp; q < ns; q += 5) v[6 * (2 * s * q) + r] = cr_fwd_row(N, F, v, 2 * s * q, s, r);
        __syncwarp(m);
      }
      double a = 0.0;
      if (grp == 0) a = cr_root_row(F, v, r, so);
      __syncwarp(m);
      if (grp == 0) v[r] = a;
      __syncwarp(m);
      CR_T(20);
      for (int l = Lv - 1; l >= ltop; --l) {
        const int s = 1 << l, ne = cr_elim_count(N, l);
        for (int q0 = 0; q0 < ne; q0 += 5) {
          const int q = q0 + grp, i = s + 2 * s * q;
          if (q < ne) a = cr_bwd_row(N, F, v, i, s, r, so);
          __syncwarp(m);
          if (q < ne) v[6 * i + r] = a;
          __syncwarp(m);
        }
      }
    }
  } else if (ltop < Lv || nrhs <= 5) {
    // nrhs * blocks <= 5 from here on: warp 0 alone, group -> (rhs, block)
    if (team.warp == 0 && glane) {
      const unsigned m = 0x3fffffffu;
      const int g = grp;
      for (int l = ltop; l < Lv; ++l) {
        const int s = 1 << l, ns = cr_surv_count(N, l);
        const int gg = g / ns, q = g - gg * ns;
        if (gg < nrhs) {
          double* vg = v + gg * stride;
          vg[6 * (2 * s * q) + r] = cr_fwd_row(N, F, vg, 2 * s * q, s, r);
        }
        __syncwarp(m);
      }
      double a = 0.0;
      if (g < nrhs) a = cr_root_row(F, v + g * stride, r, so);
      __syncwarp(m);
      if (g < nrhs) v[g * stride + r] = a;
      __syncwarp(m);
      for (int l = Lv - 1; l >= ltop; --l) {
        const int s = 1 << l, ne = cr_elim_count(N, l);
        const int gg = ne > 0 ? g / ne : nrhs, q = g - gg * ne;
        const int i = s + 2 * s * q;
        if (gg < nrhs) a = cr_bwd_row(N, F, v + gg * stride, i, s, r, so);
        __syncwarp(m);
        if (gg < nrhs) v[gg * stride + 6 * i + r] = a;
        __syncwarp(m);
      }
    }
  } else {
    // every level had more than five items: the roots by group, warp-uniform trip counts
    for (int b = 5 * team.warp; b < nrhs; b += ngr) {
      const int g = b + grp;
      const bool act = glane && g < nrhs;
      double a = 0.0;
      if (act) a = cr_root_row(F, v + g * stride, r, so);
      __syncwarp();
      if (act) v[g * stride + r] = a;
    }
  }
  team.sync();
  CR_T(21);
  for (int l = ltop - 1; l >= 0; --l) {
    const int s = 1 << l, ne = cr_elim_count(N, l);
    const int items = nrhs * ne;
    for (int b = 5 * team.warp; b < items; b += 2 * ngr) {
      double a[2];
      double* dst[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int u = b + k * ngr + grp;
        dst[k] = nullptr;
        if (glane && u < items) {
          const int q = nrhs == 1 ? u : u / nrhs, g = u - q * nrhs;  // block-major
          const int i = s + 2 * s * q;
          a[k] = cr_bwd_row(N, F, v + g * stride, i, s, r, so);
          dst[k] = v + g * stride + 6 * i + r;
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 2; ++k)
        if (dst[k]) *dst[k] = a[k];
    }
    team.sync();
    CR_T(22 + l);
  }
}

// ---- the linear-algebra entry points of solve.cuh for a CR team ------------
DEV int twisted_factor(const TeamCR& t, int N, double* D, double* U, double* scratch, bool sh = false) {
  (void)scratch;
  (void)sh;
  return cr_factor(t, N, cr_of(N, D, U));
}
// out = M^{-1} rhs (out may alias rhs; tmp unused)
DEV void twisted_solve(const TeamCR& t, int N, const double* D, const double* U, const double* rhs, double* tmp,
                       double* out, int nrhs, long stride, bool sh = false, bool shv = false) {
  (void)tmp;
  (void)sh;
  (void)shv;
  if (out != rhs) {
    for (int g = 0; g < nrhs; ++g)
      for (int q = t.rank(); q < 6 * N; q += t.size()) out[g * stride + q] = rhs[g * stride + q];
    t.sync();
  }
  cr_solve_inplace(t, N, cr_of(N, const_cast<double*>(D), U), out, nrhs, stride);
}
DEV void twisted_solve_chunks(const TeamCR& t, int N, const double* D, const double* U, double* rhs, int nrhs,
                              long stride, const int* rhs_block = nullptr) {
  cr_solve_inplace(t, N, cr_of(N, const_cast<double*>(D), U), rhs, nrhs, stride, rhs_block);
}
DEV bool dense_chol(const TeamCR& team, int na, double* S, double* col);
#endif

}  // namespace accfem
