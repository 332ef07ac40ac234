// Block cyclic reduction (CR) factorisation and solves of the 6x6
// block-tridiagonal SPD systems, team-parallel.
//
// Replaces the reference's per-solve SuperLU factor of the quasi-definite
// KKT (solver.py:229-247, _solve_active_subset 500-528, _solve_equality_direct
// 388-421) after the exact reduction of SURVEY §7.1.  The twisted LDL^T in
// linalg.cuh is a chain of ~N/2 dependent 6x6 steps; CR needs ceil(log2 N)
// dependent levels, each fully parallel over its blocks.
//
// Elimination order: block i > 0 is eliminated at level l = ctz(i), against
// its level-l neighbours h = i - 2^l (always present) and j = i + 2^l (if
// j < N).  Block 0 is the root.  With M_{a,b} the current coupling block:
//   Dinv_i = D_i^{-1}
//   L_i    = M_{h,i} Dinv_i          R_i = M_{j,i} Dinv_i = M_{i,j}^T Dinv_i
//   D_h   -= L_i M_{h,i}^T           D_j -= R_i M_{i,j}
//   M_{h,j} = -L_i M_{i,j}           (the level-(l+1) coupling)
// Storage (struct CrF): D[N][kDiag] packed symmetric (D_i, then Dinv_i),
// L[N][36] and R[N][36].  Before the factorisation L[i] holds the level-0
// coupling C(i) = M_{i-1,i}, so `HU = L + 36` indexes the super-diagonal
// blocks U_k = M_{k,k+1} exactly as the twisted layout does; every new
// coupling M_{h,j} is written to L[j] (the left coupling of its right end).
// A solve M x = v is
//   forward  (l = 0 ..)  v_j -= R_{j-2^l} v_{j-2^l} + L_{j+2^l} v_{j+2^l}   (survivors j)
//   root     x_0 = Dinv_0 v_0
//   backward (l = .. 0)  x_i  = Dinv_i v_i - L_i^T x_h - R_i^T x_j         (eliminated i)
#pragma once
#include "../../../paper_2503_06922_b200/csrc/linalg.cuh"

namespace accfem {

struct CrF {
  double* D;  // N x kDiag
  double* L;  // N x 36 (L[0] unused)
  double* R;  // N x 36 (R[0] unused)
};

DEV int cr_levels(int N) {
  int l = 0;
  while ((1 << l) < N) ++l;
  return l;
}
// number of blocks eliminated at level l
DEV int cr_elim_count(int N, int l) {
  const int s = 1 << l;
  return s <= N - 1 ? ((N - 1 - s) >> (l + 1)) + 1 : 0;
}
// number of survivors of level l (multiples of 2^(l+1) below N)
DEV int cr_surv_count(int N, int l) { return ((N - 1) >> (l + 1)) + 1; }

// ---------------------------------------------------------------------------
// serial versions (emulation build and reference for the device code)
// ---------------------------------------------------------------------------
DEV int cr_factor(const TeamSerial&, int N, CrF F) {
  const int Lv = cr_levels(N);
  int fail = -1;
  for (int l = 0; l < Lv; ++l) {
    const int s = 1 << l, ne = cr_elim_count(N, l);
    // survivors are not read within a level, so both Schur updates apply at
    // once (in q order, as the device applies D_j in phase 1, D_h in phase 2)
    for (int q = 0; q < ne; ++q) {
      const int i = s + 2 * s * q, h = i - s, j = i + s;
      double Dm[36], Di[36], Cl[36], Cr[36], L[36], R[36];
      unpack_sym(F.D + kDiag * i, Dm);
      bool ok = spd6_inv(Dm, Di);
      if (!ok && fail < 0) fail = i;
      for (int e = 0; e < 36; ++e) Cl[e] = F.L[36 * i + e];
      const bool hj = j < N;
      for (int e = 0; e < 36; ++e) Cr[e] = hj ? F.L[36 * j + e] : 0.0;
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          double a = 0.0, b = 0.0;
          for (int t = 0; t < 6; ++t) {
            a += Cl[6 * r + t] * Di[6 * t + c];
            b += Cr[6 * t + r] * Di[6 * t + c];
          }
          L[6 * r + c] = a;
          R[6 * r + c] = b;
        }
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          double a = 0.0, b = 0.0, nc = 0.0;
          for (int t = 0; t < 6; ++t) {
            a += L[6 * r + t] * Cl[6 * c + t];
            b += R[6 * r + t] * Cr[6 * t + c];
            nc += L[6 * r + t] * Cr[6 * t + c];
          }
          if (c <= r) F.D[kDiag * h + r * (r + 1) / 2 + c] -= a;
          if (hj && c <= r) F.D[kDiag * j + r * (r + 1) / 2 + c] -= b;
          if (hj) F.L[36 * j + 6 * r + c] = -nc;
        }
      pack_sym(F.D + kDiag * i, Di);
      for (int e = 0; e < 36; ++e) {
        F.L[36 * i + e] = L[e];
        F.R[36 * i + e] = R[e];
      }
    }
  }
  double Dm[36], Di[36];
  unpack_sym(F.D, Dm);
  if (!spd6_inv(Dm, Di) && fail < 0) fail = 0;
  pack_sym(F.D, Di);
  return fail;
}

// Solve for nrhs right-hand sides v_g = v + g*stride (overwritten) into
// x_g = x + g*stride; x must not alias v.
DEV void cr_solve(const TeamSerial&, int N, CrF F, double* v, double* x, int nrhs, long stride) {
  const int Lv = cr_levels(N);
  for (int g = 0; g < nrhs; ++g) {
    double* vg = v + g * stride;
    double* xg = x + g * stride;
    for (int l = 0; l < Lv; ++l) {
      const int s = 1 << l, ns = cr_surv_count(N, l);
      for (int q = 0; q < ns; ++q) {
        const int j = 2 * s * q;
        for (int r = 0; r < 6; ++r) {
          double a = vg[6 * j + r];
          if (j > 0) {
            const double* Rm = F.R + 36 * (j - s) + 6 * r;
            const double* w = vg + 6 * (j - s);
            for (int t = 0; t < 6; ++t) a -= Rm[t] * w[t];
          }
          if (j + s < N) {
            const double* Lm = F.L + 36 * (j + s) + 6 * r;
            const double* w = vg + 6 * (j + s);
            for (int t = 0; t < 6; ++t) a -= Lm[t] * w[t];
          }
          vg[6 * j + r] = a;
        }
      }
    }
    for (int r = 0; r < 6; ++r) {
      double a = 0.0;
      for (int t = 0; t < 6; ++t) a += F.D[sidx(r, t)] * vg[t];
      xg[r] = a;
    }
    for (int l = Lv - 1; l >= 0; --l) {
      const int s = 1 << l, ne = cr_elim_count(N, l);
      for (int q = 0; q < ne; ++q) {
        const int i = s + 2 * s * q, h = i - s, j = i + s;
        for (int r = 0; r < 6; ++r) {
          double a = 0.0;
          for (int t = 0; t < 6; ++t) a += F.D[kDiag * i + sidx(r, t)] * vg[6 * i + t];
          for (int t = 0; t < 6; ++t) a -= F.L[36 * i + 6 * t + r] * xg[6 * h + t];
          if (j < N)
            for (int t = 0; t < 6; ++t) a -= F.R[36 * i + 6 * t + r] * xg[6 * j + t];
          xg[6 * i + r] = a;
        }
      }
    }
  }
}

#if defined(__CUDACC__)
// ---------------------------------------------------------------------------
// CTA-team versions.  The factorisation works on 6-lane groups (five per
// warp, lanes 30-31 idle): lane r of a group owns row r of the eliminated
// block's products; all six lanes invert D_i redundantly in registers.  The
// solve sweeps are flat loops over (rhs, block, row) items.
// ---------------------------------------------------------------------------
// levels l0 .. Lv-1 and the root; returns this thread's smallest failing
// block (N: none), not yet reduced over the team
DEV int cr_factor_levels(const TeamCta& team, int N, CrF F, int l0) {
  const int Lv = cr_levels(N);
  const int lane = team.w.lane, grp = lane / 6, r = lane - 6 * grp;
  const bool glane = lane < 30;
  const int gid = 5 * team.warp + grp, ngr = 5 * team.nw;
  int fail = N;  // smallest failing block (N: none)
  for (int l = l0; l < Lv; ++l) {
    const int s = 1 << l, ne = cr_elim_count(N, l);
    const int passes = (ne + ngr - 1) / ngr;
    for (int p = 0; p < passes; ++p) {
      const int q = p * ngr + gid;
      const bool act = glane && q < ne;
      const int i = s + 2 * s * q, h = i - s, j = i + s;
      const bool hj = act && j < N;
      double dl[6] = {0, 0, 0, 0, 0, 0}, dr[6], nc[6], Lr[6], Rr[6], Di[36];
      if (act) {
        double Dm[36];
        unpack_sym(F.D + kDiag * i, Dm);
        if (!spd6_inv(Dm, Di)) fail = min(fail, i);
        const double* Cl = F.L + 36 * i;
        const double* Cr = F.L + 36 * j;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          double a = 0.0, b = 0.0;
#pragma unroll
          for (int t = 0; t < 6; ++t) {
            a += Cl[6 * r + t] * Di[6 * t + c];
            if (hj) b += Cr[6 * t + r] * Di[6 * t + c];
          }
          Lr[c] = a;
          Rr[c] = b;
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          double a = 0.0, b = 0.0, e = 0.0;
#pragma unroll
          for (int t = 0; t < 6; ++t) {
            a += Lr[t] * Cl[6 * c + t];
            if (hj) {
              b += Rr[t] * Cr[6 * t + c];
              e += Lr[t] * Cr[6 * t + c];
            }
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
      team.sync();
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
  return fail;
}
DEVNI int cr_factor(const TeamCta& team, int N, CrF F) {
  const int fail = team.imin(cr_factor_levels(team, N, F, 0));
  return fail < N ? fail : -1;
}

// One forward step of survivor j (row r) and one backward step of eliminated
// block i (row r, packed-row offsets so[]) for right-hand side vg / xg.
DEV void cr_fwd_row(int N, const CrF& F, double* vg, int j, int s, int r) {
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
  vg[6 * j + r] = a - b;
}
DEV void cr_bwd_row(int N, const CrF& F, const double* vg, double* xg, int i, int s, int r, const int* so) {
  const int h = i - s, j = i + s;
  const double* Dm = F.D + kDiag * i;
  const double* vi = vg + 6 * i;
  double a0 = Dm[so[0]] * vi[0] + Dm[so[2]] * vi[2] + Dm[so[4]] * vi[4];
  double a1 = Dm[so[1]] * vi[1] + Dm[so[3]] * vi[3] + Dm[so[5]] * vi[5];
  const double* Lm = F.L + 36 * i + r;
  const double* xh = xg + 6 * h;
  double b0 = Lm[0] * xh[0] + Lm[12] * xh[2] + Lm[24] * xh[4];
  double b1 = Lm[6] * xh[1] + Lm[18] * xh[3] + Lm[30] * xh[5];
  double c0 = 0.0, c1 = 0.0;
  if (j < N) {
    const double* Rm = F.R + 36 * i + r;
    const double* xj = xg + 6 * j;
    c0 = Rm[0] * xj[0] + Rm[12] * xj[2] + Rm[24] * xj[4];
    c1 = Rm[6] * xj[1] + Rm[18] * xj[3] + Rm[30] * xj[5];
  }
  xg[6 * i + r] = (a0 + a1) - ((b0 + b1) + (c0 + c1));
}
DEV void cr_root_row(const CrF& F, const double* vg, double* xg, int r, const int* so) {
  const double* Dm = F.D;
  double a0 = Dm[so[0]] * vg[0] + Dm[so[2]] * vg[2] + Dm[so[4]] * vg[4];
  double a1 = Dm[so[1]] * vg[1] + Dm[so[3]] * vg[3] + Dm[so[5]] * vg[5];
  xg[r] = a0 + a1;
}

// Work is mapped on 6-lane groups (five per warp): lane r of a group always
// handles row r, so the packed-row offsets of Dinv are fixed per thread.
// The top levels, whose blocks fit in the five groups of warp 0, run on
// warp 0 alone with warp barriers (one CTA barrier for all of them).
// forward levels l0.., root, backward ..l0 (the leaves below l0 are the caller's)
DEV void cr_solve_levels(const TeamCta& team, int N, const CrF& F, int l0, double* v, double* x, int nrhs,
                         long stride) {
  const int Lv = cr_levels(N);
  const int lane = team.w.lane, grp = lane / 6, r = lane - 6 * grp;
  const bool glane = lane < 30;
  const int gid = 5 * team.warp + grp, ngr = 5 * team.nw;
  int so[6];
#pragma unroll
  for (int t = 0; t < 6; ++t) so[t] = sidx(r, t);
  // first level whose survivors (and so every later level's blocks) fit in warp 0 for all rhs
  int ltop = l0;
  while (ltop < Lv && cr_surv_count(N, ltop) * nrhs > 5) ++ltop;
  // (rhs, block) pairs are spread over the groups: u = g * count + q
  for (int l = l0; l < ltop; ++l) {
    const int s = 1 << l, ns = cr_surv_count(N, l);
    if (glane)
      for (int u = gid; u < nrhs * ns; u += ngr) {
        const int g = nrhs == 1 ? 0 : u / ns, q = u - g * ns;
        cr_fwd_row(N, F, v + g * stride, 2 * s * q, s, r);
      }
    team.sync();
  }
  if (ltop < Lv) {
    // nrhs * blocks <= 5 from here on: warp 0 alone, group -> (rhs, block)
    if (team.warp == 0 && glane) {
      const int g = grp;
      for (int l = ltop; l < Lv; ++l) {
        const int s = 1 << l, ns = cr_surv_count(N, l);
        const int gg = nrhs == 1 ? (g < ns ? 0 : 1) : g / ns, q = g - gg * ns;
        if (gg < nrhs) cr_fwd_row(N, F, v + gg * stride, 2 * s * q, s, r);
        __syncwarp(0x3fffffffu);
      }
      if (g < nrhs) cr_root_row(F, v + g * stride, x + g * stride, r, so);
      __syncwarp(0x3fffffffu);
      for (int l = Lv - 1; l >= ltop; --l) {
        const int s = 1 << l, ne = cr_elim_count(N, l);
        const int gg = nrhs == 1 ? (g < ne ? 0 : 1) : (ne > 0 ? g / ne : nrhs), q = g - gg * ne;
        if (gg < nrhs) cr_bwd_row(N, F, v + gg * stride, x + gg * stride, s + 2 * s * q, s, r, so);
        __syncwarp(0x3fffffffu);
      }
    }
  } else if (glane) {
    for (int g = gid; g < nrhs; g += ngr) cr_root_row(F, v + g * stride, x + g * stride, r, so);
  }
  team.sync();
  for (int l = ltop - 1; l >= l0; --l) {
    const int s = 1 << l, ne = cr_elim_count(N, l);
    if (glane)
      for (int u = gid; u < nrhs * ne; u += ngr) {
        const int g = nrhs == 1 ? 0 : u / ne, q = u - g * ne;
        cr_bwd_row(N, F, v + g * stride, x + g * stride, s + 2 * s * q, s, r, so);
      }
    team.sync();
  }
}
DEVNI void cr_solve(const TeamCta& team, int N, CrF F, double* v, double* x, int nrhs, long stride) {
  cr_solve_levels(team, N, F, 0, v, x, nrhs, stride);
}

#endif

}  // namespace accfem
