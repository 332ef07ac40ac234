// Segmented block-tridiagonal factor/solve for the ADMM loop: one factor,
// thousands of single-right-hand-side solves per QP (solver.py:298-311
// after the exact reduction of SURVEY §7.1).
//
// The N blocks are cut at the separators m*S (S = 2^a, m < nseg).  Every
// segment's interior blocks h+1 .. h+S-1 (h = m*S) are eliminated one after
// the other by one 6-lane group, with the cyclic-reduction formulas of
// cr.cuh applied against the fixed left separator h and the next block
// j = i+1 (Dinv_i in D[i], L_i = M_{h,i} Dinv_i in L[i], R_i = M_{i,i+1}^T
// Dinv_i in R[i], fill M_{h,i+1} in L[i+1]).  What is left is the
// block-tridiagonal system of the separators with couplings M_{p,q} in L[q];
// it is factored sequentially by group 0 (block LDL^T: D'_q^{-1} in D[q],
// X_q = M_{p,q}^T D'_p^{-1} in R[q]).
//
// A solve is four dependent chains: the segments forward (S-1 steps, all
// groups at once), the separators forward and backward (nseg-1 steps each,
// group 0), the segments backward (S-1 steps).  Each step is one 6x6 row
// mat-vec per lane plus a 6-lane shuffle broadcast of the new block; the
// parts that do not depend on the chain (the L_i v_i contributions to the
// separator, Dinv_i v_i, L_i^T x_h) are off the critical path.  With a = 3
// at N = 101 that is 38 short steps against 100 for the twisted LDL^T.
#pragma once
#include "cr.cuh"

namespace accfem {

DEV int seg_count(int N, int a) { return ((N - 1) >> a) + 1; }

// segment bits: the fewest chain steps (S-1) + (nseg-1) with nseg <= groups
DEV int seg_bits(int N, int groups) {
  int best = -1, cost = 1 << 30;
  for (int a = 1; a < 16; ++a) {
    const int ns = seg_count(N, a);
    if (ns > groups) continue;
    const int c = ((1 << a) - 1) + (ns - 1);
    if (c < cost) {
      cost = c;
      best = a;
    }
    if (ns == 1) break;
  }
  return best;
}

// one eliminated segment block (row r): the products of cr.cuh's formulas.
// Cl = M_{h,i}, Cr = M_{i,i+1} (hj: i+1 < N), Di = D_i^{-1}.
DEV void seg_block_rows(const double* Cl, const double* Cr, bool hj, const double* Di, int r, double* Lr,
                        double* Rr, double* dl, double* dr, double* nc) {
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double x0 = 0.0, x1 = 0.0;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      x0 += Cl[6 * r + t] * Di[6 * t + c];
      if (hj) x1 += Cr[6 * t + r] * Di[6 * t + c];
    }
    Lr[c] = x0;
    Rr[c] = x1;
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double x0 = 0.0, x1 = 0.0, x2 = 0.0;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      x0 += Lr[t] * Cl[6 * c + t];
      if (hj) {
        x1 += Rr[t] * Cr[6 * t + c];
        x2 += Lr[t] * Cr[6 * t + c];
      }
    }
    dl[c] = x0;
    dr[c] = x1;
    nc[c] = -x2;
  }
}

// separator step (row r): X = C^T P (P = D'^{-1}_p), D'_q row r = D_q row r - X_r C
DEV void seg_sep_rows(const double* C, const double* P, const double* Dq, int r, double* Xr, double* Dr) {
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double x0 = 0.0;
#pragma unroll
    for (int t = 0; t < 6; ++t) x0 += C[6 * t + r] * P[6 * t + c];
    Xr[c] = x0;
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double x0 = Dq[6 * r + c];
#pragma unroll
    for (int t = 0; t < 6; ++t) x0 -= Xr[t] * C[6 * t + c];
    Dr[c] = x0;
  }
}

DEV double dot6(const double* a, const double* w) {
  return (a[0] * w[0] + a[2] * w[2] + a[4] * w[4]) + (a[1] * w[1] + a[3] * w[3] + a[5] * w[5]);
}
// column r of a row-major 6x6 dotted with w
DEV double dot6c(const double* a, const double* w) {
  return (a[0] * w[0] + a[12] * w[2] + a[24] * w[4]) + (a[6] * w[1] + a[18] * w[3] + a[30] * w[5]);
}
// row r of a packed symmetric 6x6 dotted with w (so: packed offsets of row r)
DEV double dot6s(const double* p, const int* so, const double* w) {
  return (p[so[0]] * w[0] + p[so[2]] * w[2] + p[so[4]] * w[4]) + (p[so[1]] * w[1] + p[so[3]] * w[3] + p[so[5]] * w[5]);
}

// ---------------------------------------------------------------------------
// serial versions (emulation build); same arithmetic per row
// ---------------------------------------------------------------------------
DEV int seg_factor(const TeamSerial&, int N, CrF F, int a) {
  const int S = 1 << a, nseg = seg_count(N, a);
  int fail = -1;
  for (int m = 0; m < nseg; ++m) {
    const int h = m * S;
    double dlh[36];
    for (int e = 0; e < 36; ++e) dlh[e] = 0.0;
    for (int i = h + 1; i < h + S && i < N; ++i) {
      const int j = i + 1;
      const bool hj = j < N;
      double Dm[36], Di[36], Cl[36], Cr[36], L[36], R[36], dl[36], dr[36], nc[36];
      unpack_sym(F.D + kDiag * i, Dm);
      if (!spd6_inv(Dm, Di) && fail < 0) fail = i;
      for (int e = 0; e < 36; ++e) {
        Cl[e] = F.L[36 * i + e];
        Cr[e] = hj ? F.L[36 * j + e] : 0.0;
      }
      for (int r = 0; r < 6; ++r) seg_block_rows(Cl, Cr, hj, Di, r, L + 6 * r, R + 6 * r, dl + 6 * r, dr + 6 * r, nc + 6 * r);
      pack_sym(F.D + kDiag * i, Di);
      for (int e = 0; e < 36; ++e) {
        F.L[36 * i + e] = L[e];
        F.R[36 * i + e] = R[e];
        dlh[e] += dl[e];
      }
      if (hj) {
        for (int r = 0; r < 6; ++r)
          for (int c = 0; c <= r; ++c) F.D[kDiag * j + r * (r + 1) / 2 + c] -= dr[6 * r + c];
        for (int e = 0; e < 36; ++e) F.L[36 * j + e] = nc[e];
      }
    }
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c <= r; ++c) F.D[kDiag * h + r * (r + 1) / 2 + c] -= dlh[6 * r + c];
  }
  double Dm[36], Di[36];
  unpack_sym(F.D, Dm);
  if (!spd6_inv(Dm, Di) && fail < 0) fail = 0;
  pack_sym(F.D, Di);
  for (int m = 1; m < nseg; ++m) {
    const int p = (m - 1) * S, q = m * S;
    double P[36], Dq[36], X[36], Dn[36];
    unpack_sym(F.D + kDiag * p, P);
    unpack_sym(F.D + kDiag * q, Dq);
    for (int r = 0; r < 6; ++r) seg_sep_rows(F.L + 36 * q, P, Dq, r, X + 6 * r, Dn + 6 * r);
    for (int e = 0; e < 36; ++e) F.R[36 * q + e] = X[e];
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c <= r; ++c) Dm[6 * r + c] = Dm[6 * c + r] = Dn[6 * r + c];
    if (!spd6_inv(Dm, Di) && fail < 0) fail = q;
    pack_sym(F.D + kDiag * q, Di);
  }
  return fail;
}

DEV void seg_solve(const TeamSerial&, int N, const CrF& F, int a, double* v, double* x) {
  const int S = 1 << a, nseg = seg_count(N, a);
  int so[6][6];
  for (int r = 0; r < 6; ++r)
    for (int t = 0; t < 6; ++t) so[r][t] = sidx(r, t);
  // segments forward; the right separator is updated in the segment's pass,
  // the left one right after it (the device's phase 1 / phase 2 order)
  for (int m = 0; m < nseg; ++m) {
    const int h = m * S;
    if (h + 1 >= N) continue;
    double w[6], acc[6] = {0, 0, 0, 0, 0, 0};
    for (int t = 0; t < 6; ++t) w[t] = v[6 * (h + 1) + t];
    for (int i = h + 1; i < h + S && i < N; ++i) {
      double nv[6];
      for (int r = 0; r < 6; ++r) {
        acc[r] += dot6(F.L + 36 * i + 6 * r, w);
        nv[r] = i + 1 < N ? v[6 * (i + 1) + r] - dot6(F.R + 36 * i + 6 * r, w) : 0.0;
      }
      if (i + 1 < N)
        for (int r = 0; r < 6; ++r) v[6 * (i + 1) + r] = w[r] = nv[r];
    }
    for (int r = 0; r < 6; ++r) v[6 * h + r] -= acc[r];
  }
  // separators
  for (int r = 0; r < 6; ++r) x[r] = dot6s(F.D, so[r], v);
  for (int m = 1; m < nseg; ++m) {
    const int p = (m - 1) * S, q = m * S;
    double y[6];
    for (int r = 0; r < 6; ++r) y[r] = v[6 * q + r] - dot6(F.R + 36 * q + 6 * r, v + 6 * p);
    for (int r = 0; r < 6; ++r) v[6 * q + r] = y[r];
    for (int r = 0; r < 6; ++r) x[6 * q + r] = dot6s(F.D + kDiag * q, so[r], y);
  }
  for (int m = nseg - 2; m >= 0; --m) {
    const int p = m * S, q = (m + 1) * S;
    double xn[6];
    for (int r = 0; r < 6; ++r) xn[r] = x[6 * p + r] - dot6c(F.R + 36 * q + r, x + 6 * q);
    for (int r = 0; r < 6; ++r) x[6 * p + r] = xn[r];
  }
  // segments backward
  for (int m = 0; m < nseg; ++m) {
    const int h = m * S;
    for (int i = (h + S < N ? h + S : N) - 1; i > h; --i)
      for (int r = 0; r < 6; ++r) {
        double p = dot6s(F.D + kDiag * i, so[r], v + 6 * i) - dot6c(F.L + 36 * i + r, x + 6 * h);
        if (i + 1 < N) p -= dot6c(F.R + 36 * i + r, x + 6 * (i + 1));
        x[6 * i + r] = p;
      }
  }
}

#if defined(__CUDACC__)
// ---------------------------------------------------------------------------
// CTA-team versions: group g (lanes 6g' .. 6g'+5 of warp w, g = 5w + g')
// owns segment g; lane r of a group computes row r.  Loops run the same
// number of steps on every lane so the 6-lane broadcasts can be full-warp
// shuffles.
// ---------------------------------------------------------------------------
DEV int seg_factor(const TeamCta& team, int N, CrF F, int a) {
  const int lane = team.w.lane, grp = lane / 6, r = lane - 6 * grp;
  const unsigned gmask = 0x3fu << (6 * grp);
  const int gid = 5 * team.warp + grp;
  const int S = 1 << a, nseg = seg_count(N, a);
  const bool act = lane < 30 && gid < nseg;
  const int h = gid * S;
  int fail = N;
  double dlh[6] = {0, 0, 0, 0, 0, 0};
  if (act) {
    for (int i = h + 1; i < h + S && i < N; ++i) {
      const int j = i + 1;
      const bool hj = j < N;
      double Dm[36], Di[36], Lr[6], Rr[6], dl[6], dr[6], nc[6];
      unpack_sym(F.D + kDiag * i, Dm);
      if (!spd6_inv(Dm, Di)) fail = min(fail, i);
      seg_block_rows(F.L + 36 * i, F.L + 36 * (hj ? j : i), hj, Di, r, Lr, Rr, dl, dr, nc);
#pragma unroll
      for (int c = 0; c < 6; ++c) dlh[c] += dl[c];
      __syncwarp(gmask);  // the group has read C(i), C(i+1)
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
      __syncwarp(gmask);  // D_{i+1} and the fill are visible to the group
    }
  }
  team.sync();
  if (act) {  // the left separator's update (its left neighbour segment wrote in phase 1)
    double* Dh = F.D + kDiag * h + r * (r + 1) / 2;
#pragma unroll
    for (int c = 0; c < 6; ++c)
      if (c <= r) Dh[c] -= dlh[c];
  }
  team.sync();
  // separators: sequential block LDL^T on group 0
  if (team.warp == 0 && lane < 6) {
    double Dm[36], Di[36];
    unpack_sym(F.D, Dm);
    if (!spd6_inv(Dm, Di)) fail = min(fail, 0);
    __syncwarp(0x3fu);
    if (r == 0) pack_sym(F.D, Di);
    __syncwarp(0x3fu);
    for (int m = 1; m < nseg; ++m) {
      const int p = (m - 1) * S, q = m * S;
      double P[36], Dq[36], Xr[6], Dr[6];
      unpack_sym(F.D + kDiag * p, P);
      unpack_sym(F.D + kDiag * q, Dq);
      seg_sep_rows(F.L + 36 * q, P, Dq, r, Xr, Dr);
      __syncwarp(0x3fu);
      st6(F.R + 36 * q + 6 * r, Xr);
      double* Dp = F.D + kDiag * q + r * (r + 1) / 2;
#pragma unroll
      for (int c = 0; c < 6; ++c)
        if (c <= r) Dp[c] = Dr[c];
      __syncwarp(0x3fu);
      unpack_sym(F.D + kDiag * q, Dm);
      if (!spd6_inv(Dm, Di)) fail = min(fail, q);
      __syncwarp(0x3fu);
      if (r == 0) pack_sym(F.D + kDiag * q, Di);
      __syncwarp(0x3fu);
    }
  }
  fail = team.imin(fail);
  return fail < N ? fail : -1;
}

#if defined(SEG_TIMING)
__device__ unsigned long long g_seg_t[8];
#define SEG_T(k) do { if (threadIdx.x == 0 && blockIdx.x == 0) { long long _n = clock64(); g_seg_t[k] += _n - _seg_last; _seg_last = _n; } } while (0)
#else
#define SEG_T(k)
#endif
DEV void seg_solve(const TeamCta& team, int N, const CrF& F, int a, double* v, double* x) {
#if defined(SEG_TIMING)
  long long _seg_last = clock64();
#endif
  const int lane = team.w.lane, grp = lane / 6, r = lane - 6 * grp;
  const int gid = 5 * team.warp + grp, src = 6 * grp;
  const int S = 1 << a, nseg = seg_count(N, a);
  const bool act = lane < 30 && gid < nseg;
  const int h = act ? gid * S : 0;
  int so[6];
#pragma unroll
  for (int t = 0; t < 6; ++t) so[t] = sidx(r, t);
  // segments forward: v_{i+1} -= R_i v_i; L_i v_i accumulates for the separator
  double acc = 0.0;
  {
    double w[6];
    ld6(v + 6 * min(h + 1, N - 1), w);
#pragma unroll 2
    for (int t = 1; t < S; ++t) {
      const int i = h + t;
      const bool on = act && i < N;
      const int ic = min(i, N - 1), in = min(i + 1, N - 1);
      double Lr[6], Rr[6];
      ld6(F.L + 36 * ic + 6 * r, Lr);
      ld6(F.R + 36 * ic + 6 * r, Rr);
      const double vn = v[6 * in + r];
      const double l = dot6(Lr, w);
      const double nv = vn - dot6(Rr, w);
      if (on) acc += l;
      if (on && i + 1 < N) v[6 * (i + 1) + r] = nv;
#pragma unroll
      for (int q = 0; q < 6; ++q) w[q] = __shfl_sync(0xffffffffu, nv, src + q);
    }
  }
  SEG_T(0);
  team.sync();
  SEG_T(1);
  if (act && h + 1 < N) v[6 * h + r] -= acc;
  team.sync();
  SEG_T(2);
  // separators on warp 0 (group 0 carries the values; the whole warp steps)
  if (team.warp == 0) {
    const bool g0 = lane < 6;
    double y[6];
    ld6(v, y);
    if (g0) x[r] = dot6s(F.D, so, y);
    for (int m = 1; m < nseg; ++m) {
      const int p = (m - 1) * S, q = m * S;
      (void)p;
      double Xr[6];
      ld6(F.R + 36 * q + 6 * r, Xr);
      const double yr = v[6 * q + r] - dot6(Xr, y);
#pragma unroll
      for (int t = 0; t < 6; ++t) y[t] = __shfl_sync(0xffffffffu, yr, t);
      if (g0) {
        v[6 * q + r] = yr;
        x[6 * q + r] = dot6s(F.D + kDiag * q, so, y);
      }
    }
    __syncwarp();
    double xq[6];
    ld6(x + 6 * (nseg - 1) * S, xq);
    for (int m = nseg - 2; m >= 0; --m) {
      const int p = m * S, q = (m + 1) * S;
      const double xr = x[6 * p + r] - dot6c(F.R + 36 * q + r, xq);
#pragma unroll
      for (int t = 0; t < 6; ++t) xq[t] = __shfl_sync(0xffffffffu, xr, t);
      if (g0) x[6 * p + r] = xr;
    }
  }
  SEG_T(3);
  team.sync();
  SEG_T(4);
  // segments backward: x_i = Dinv_i v_i - L_i^T x_h - R_i^T x_{i+1}
  {
    double xh[6], xn[6];
    ld6(x + 6 * h, xh);
    const int j0 = h + S;
    if (act && j0 < N) {
      ld6(x + 6 * j0, xn);
    } else {
#pragma unroll
      for (int t = 0; t < 6; ++t) xn[t] = 0.0;
    }
#pragma unroll 2
    for (int t = S - 1; t >= 1; --t) {
      const int i = h + t;
      const bool on = act && i < N;
      const int ic = min(i, N - 1);
      double vi[6];
      ld6(v + 6 * ic, vi);
      const double base = dot6s(F.D + kDiag * ic, so, vi) - dot6c(F.L + 36 * ic + r, xh);
      const double p = on ? base - dot6c(F.R + 36 * ic + r, xn) : 0.0;
      if (on) x[6 * i + r] = p;
#pragma unroll
      for (int q = 0; q < 6; ++q) xn[q] = __shfl_sync(0xffffffffu, p, src + q);
    }
  }
  SEG_T(5);
  team.sync();
  SEG_T(6);
}
#endif

}  // namespace accfem
