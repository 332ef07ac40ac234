// 6x6 block-tridiagonal SPD factorisation and solves on one team.
//
// M = L L^T with L block lower-bidiagonal: diagonal blocks L_i (lower
// triangular), sub-diagonal blocks B_i = M_{i,i-1} L_{i-1}^{-T}.  We store
//   Li_i = L_i^{-1}           (lower, 6x6 row-major)
//   G_i  = Li_i B_i           (forward recurrence  w_i = Li_i r_i - G_i w_{i-1})
//   Hb_i = Li_i^T B_{i+1}^T   (backward recurrence x_i = Li_i^T w_i - Hb_i x_{i+1})
// so each step of either sweep is one dependent 6x6 mat-vec.  This replaces
// the reference's SuperLU factor of the quasi-definite KKT matrix
// (solver.py:229-247): the dual block is eliminated exactly.
#pragma once
#include "problem.cuh"

namespace accfem {

// in-register 6x6 Cholesky + triangular inverse; returns false on a
// non-positive pivot
DEV bool chol6_inv(const double* S, double* Li) {
  double L[36];
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
  for (int j = 0; j < 6; ++j) {
    double dj = S[6 * j + j];
    for (int k = 0; k < j; ++k) dj -= L[6 * j + k] * L[6 * j + k];
    if (!(dj > 0.0)) return false;
    double ljj = sqrt(dj);
    double inv = 1.0 / ljj;
    L[6 * j + j] = ljj;
    for (int i = j + 1; i < 6; ++i) {
      double s = S[6 * i + j];
      for (int k = 0; k < j; ++k) s -= L[6 * i + k] * L[6 * j + k];
      L[6 * i + j] = s * inv;
    }
  }
  // forward substitution for the inverse, column by column
  for (int i = 0; i < 36; ++i) Li[i] = 0.0;
  for (int c = 0; c < 6; ++c) {
    Li[6 * c + c] = 1.0 / L[6 * c + c];
    for (int r = c + 1; r < 6; ++r) {
      double s = 0.0;
      for (int k = c; k < r; ++k) s += L[6 * r + k] * Li[6 * k + c];
      Li[6 * r + c] = -s / L[6 * r + r];
    }
  }
  return true;
}

// Factor (Dm, Um) -> (Li, G, Hb).  scratch needs 72 doubles.  Returns the
// 0-based block of a failed pivot, or -1.
template <class Team>
DEV int block_factor(const Team& team, int N, const double* Dm, const double* Um, double* Li, double* G,
                     double* Hb, double* scratch) {
  double* B = scratch;
  double* S = scratch + 36;
  for (int i = 0; i < N; ++i) {
    if (i == 0) {
      PARFOR(t, 36) S[t] = Dm[t];
    } else {
      const double* U = Um + 36 * (i - 1);
      const double* Lp = Li + 36 * (i - 1);
      // B[r][c] = sum_k U[k][r] Lp[c][k]
      PARFOR(t, 36) {
        int r = t / 6, c = t % 6;
        double acc = 0.0;
        for (int k = 0; k <= c; ++k) acc += U[6 * k + r] * Lp[6 * c + k];
        B[t] = acc;
      }
      team.sync();
      PARFOR(t, 36) {
        int r = t / 6, c = t % 6;
        double acc = Dm[36 * i + t];
        for (int k = 0; k < 6; ++k) acc -= B[6 * r + k] * B[6 * c + k];
        S[t] = acc;
      }
    }
    team.sync();
    double L[36];
    double Sreg[36];
    for (int t = 0; t < 36; ++t) Sreg[t] = S[t];
    bool ok = chol6_inv(Sreg, L);  // every lane factors the same block redundantly
    if (!ok) return i;
    PARFOR(t, 36) Li[36 * i + t] = L[t];
    if (i > 0) {
      const double* Lp = Li + 36 * (i - 1);
      PARFOR(t, 36) {
        int r = t / 6, c = t % 6;
        double acc = 0.0;
        for (int k = 0; k <= r; ++k) acc += L[6 * r + k] * B[6 * k + c];
        G[36 * i + t] = acc;
        // Hb_{i-1}[r][c] = sum_k Lp[k][r] B[c][k]
        double acc2 = 0.0;
        for (int k = r; k < 6; ++k) acc2 += Lp[6 * k + r] * B[6 * c + k];
        Hb[36 * (i - 1) + t] = acc2;
      }
    }
    team.sync();
  }
  return -1;
}

// Solve M x = r for `nrhs` right-hand sides (r_g = rhs + g*stride, result to
// out + g*stride; out may alias rhs).
DEV void chain_solve(const TeamSerial&, int N, const double* Li, const double* G, const double* Hb,
                     const double* rhs, double* out, int nrhs, long stride) {
  for (int g = 0; g < nrhs; ++g) {
    const double* b = rhs + g * stride;
    double* o = out + g * stride;
    double wp[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < N; ++i) {
      double w[6];
      for (int r = 0; r < 6; ++r) {
        double c = 0.0;
        for (int j = 0; j <= r; ++j) c += Li[36 * i + 6 * r + j] * b[6 * i + j];
        if (i > 0)
          for (int j = 0; j < 6; ++j) c -= G[36 * i + 6 * r + j] * wp[j];
        w[r] = c;
      }
      for (int r = 0; r < 6; ++r) {
        o[6 * i + r] = w[r];
        wp[r] = w[r];
      }
    }
    double xn[6] = {0, 0, 0, 0, 0, 0};
    for (int i = N - 1; i >= 0; --i) {
      double xv[6];
      for (int r = 0; r < 6; ++r) {
        double c = 0.0;
        for (int j = r; j < 6; ++j) c += Li[36 * i + 6 * j + r] * o[6 * i + j];
        if (i < N - 1)
          for (int j = 0; j < 6; ++j) c -= Hb[36 * i + 6 * r + j] * xn[j];
        xv[r] = c;
      }
      for (int r = 0; r < 6; ++r) {
        o[6 * i + r] = xv[r];
        xn[r] = xv[r];
      }
    }
  }
}

#if defined(__CUDACC__)
// Warp version: lane = 6*g + r handles row r of right-hand side g (g < 5).
// Each recurrence step is one dependent 6-wide shuffle mat-vec; the
// independent Li_i r_i / Li_i^T w_i products and the next step's operands are
// loaded one step ahead.
DEV void chain_solve(const TeamWarp& team, int N, const double* __restrict__ Li, const double* __restrict__ G,
                     const double* __restrict__ Hb, const double* rhs, double* out, int nrhs, long stride) {
  const int lane = team.lane;
  const int g = lane / 6, r = lane % 6;
  const bool act = g < nrhs;
  const int gg = act ? g : 0;
  const double* b = rhs + gg * stride;
  double* o = out + gg * stride;
  const int src = 6 * (g < 5 ? g : 0);
  double wp = 0.0;
  for (int i = 0; i < N; ++i) {
    const double* li = Li + 36 * i + 6 * r;
    const double* gi = G + 36 * i + 6 * r;
    double c = 0.0;
#pragma unroll
    for (int j = 0; j < 6; ++j)
      if (j <= r) c += li[j] * b[6 * i + j];
    double acc0 = c, acc1 = 0.0;
    if (i > 0) {
      double w0 = __shfl_sync(0xffffffffu, wp, src + 0);
      double w1 = __shfl_sync(0xffffffffu, wp, src + 1);
      double w2 = __shfl_sync(0xffffffffu, wp, src + 2);
      double w3 = __shfl_sync(0xffffffffu, wp, src + 3);
      double w4 = __shfl_sync(0xffffffffu, wp, src + 4);
      double w5 = __shfl_sync(0xffffffffu, wp, src + 5);
      acc0 -= gi[0] * w0;
      acc1 -= gi[1] * w1;
      acc0 -= gi[2] * w2;
      acc1 -= gi[3] * w3;
      acc0 -= gi[4] * w4;
      acc1 -= gi[5] * w5;
    }
    wp = acc0 + acc1;
    __syncwarp();  // out may alias rhs: all lanes have read row block i
    if (act) o[6 * i + r] = wp;
  }
  __syncwarp();
  double xn = 0.0;
  for (int i = N - 1; i >= 0; --i) {
    const double* li = Li + 36 * i;
    const double* hi = Hb + 36 * i + 6 * r;
    double c = 0.0;
#pragma unroll
    for (int j = 0; j < 6; ++j)
      if (j >= r) c += li[6 * j + r] * o[6 * i + j];
    double acc0 = c, acc1 = 0.0;
    if (i < N - 1) {
      double x0 = __shfl_sync(0xffffffffu, xn, src + 0);
      double x1 = __shfl_sync(0xffffffffu, xn, src + 1);
      double x2 = __shfl_sync(0xffffffffu, xn, src + 2);
      double x3 = __shfl_sync(0xffffffffu, xn, src + 3);
      double x4 = __shfl_sync(0xffffffffu, xn, src + 4);
      double x5 = __shfl_sync(0xffffffffu, xn, src + 5);
      acc0 -= hi[0] * x0;
      acc1 -= hi[1] * x1;
      acc0 -= hi[2] * x2;
      acc1 -= hi[3] * x3;
      acc0 -= hi[4] * x4;
      acc1 -= hi[5] * x5;
    }
    xn = acc0 + acc1;
    __syncwarp();
    if (act) o[6 * i + r] = xn;
  }
  __syncwarp();
}
#endif

// y = M x for a symmetric block-tridiagonal (D, U) matrix; y must not alias x
template <class Team>
DEV void block_matvec(const Team& team, int N, const double* D, const double* U, const double* x, double* y) {
  PARFOR(j, 6 * N) {
    int k = j / 6, r = j % 6;
    const double* dr = D + 36 * k + 6 * r;
    const double* xk = x + 6 * k;
    double acc = 0.0;
    for (int c = 0; c < 6; ++c) acc += dr[c] * xk[c];
    if (k + 1 < N) {
      const double* ur = U + 36 * k + 6 * r;
      const double* xn = x + 6 * (k + 1);
      for (int c = 0; c < 6; ++c) acc += ur[c] * xn[c];
    }
    if (k > 0) {
      const double* up = U + 36 * (k - 1);
      const double* xp = x + 6 * (k - 1);
      for (int c = 0; c < 6; ++c) acc += up[6 * c + r] * xp[c];
    }
    y[j] = acc;
  }
  team.sync();
}

}  // namespace accfem
