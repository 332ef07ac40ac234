// 6x6 block-tridiagonal SPD factorisation and solves on one team, in place.
//
// Twisted ("burn at both ends") block LDL^T of M with diagonal blocks A_i and
// off-diagonal blocks C_i = M_{i,i+1}: the top half is eliminated downward,
// the bottom half upward, meeting at the middle block k = (N-1)/2:
//   top    S_0 = A_0,      X_i = C_{i-1}^T S_{i-1}^{-1},  S_i = A_i - X_i C_{i-1}   (i < k)
//   bottom T_{N-1} = A_{N-1}, Y_i = C_i T_{i+1}^{-1},    T_i = A_i - Y_i C_i^T     (i > k)
//   middle Z = A_k - X_k C_{k-1} - Y_k C_k^T
// Stored in place: D[i] <- S_i^{-1} / Z^{-1} / T_i^{-1};  U[i-1] <- X_i (i <= k),
// U[i] <- Y_i (i >= k).  A solve is two dependent sweeps of ~N/2 one-matvec
// steps each, run concurrently by two 6-lane groups of a warp.  This replaces
// the reference's SuperLU factor of the quasi-definite KKT (solver.py:229-247):
// the dual block is eliminated exactly.
#pragma once
#include "problem.cuh"

namespace accfem {

// symmetric positive definite 6x6 inverse (Cholesky); false on a non-positive pivot
DEV bool spd6_inv(const double* S, double* Inv) {
  double L[21];  // packed lower, row-major: (r, c) at r*(r+1)/2 + c
  for (int j = 0; j < 6; ++j) {
    double dj = S[6 * j + j];
    for (int k = 0; k < j; ++k) dj -= L[j * (j + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
    if (!(dj > 0.0)) return false;
    double ljj = sqrt(dj);
    L[j * (j + 1) / 2 + j] = ljj;
    double inv = 1.0 / ljj;
    for (int i = j + 1; i < 6; ++i) {
      double s = S[6 * i + j];
      for (int k = 0; k < j; ++k) s -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
      L[i * (i + 1) / 2 + j] = s * inv;
    }
  }
  // W = L^{-1} (lower), Inv = W^T W
  double W[21];
  for (int c = 0; c < 6; ++c) {
    W[c * (c + 1) / 2 + c] = 1.0 / L[c * (c + 1) / 2 + c];
    for (int r = c + 1; r < 6; ++r) {
      double s = 0.0;
      for (int k = c; k < r; ++k) s += L[r * (r + 1) / 2 + k] * W[k * (k + 1) / 2 + c];
      W[r * (r + 1) / 2 + c] = -s / L[r * (r + 1) / 2 + r];
    }
  }
  for (int r = 0; r < 6; ++r)
    for (int c = r; c < 6; ++c) {
      double s = 0.0;
      for (int k = c; k < 6; ++k) s += W[k * (k + 1) / 2 + r] * W[k * (k + 1) / 2 + c];
      Inv[6 * r + c] = s;
      Inv[6 * c + r] = s;
    }
  return true;
}

DEV int twist_split(int N) { return (N - 1) / 2; }

// In-place twisted factorisation.  scratch: 4 x 36 doubles per team.
// Returns the block of a failed pivot, or -1.
DEV int twisted_factor(const TeamSerial&, int N, double* D, double* U, double* scratch) {
  const int k = twist_split(N);
  double Sinv[36], X[36], Sn[36];
  // top: blocks 0..k-1
  for (int i = 0; i < k; ++i) {
    for (int t = 0; t < 36; ++t) Sn[t] = D[36 * i + t];
    if (i > 0) {
      const double* C = U + 36 * (i - 1);
      // X = C^T Sinv_{i-1};  S = A - X C
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          double a = 0.0;
          for (int q = 0; q < 6; ++q) a += C[6 * q + r] * Sinv[6 * q + c];
          X[6 * r + c] = a;
        }
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          double a = Sn[6 * r + c];
          for (int q = 0; q < 6; ++q) a -= X[6 * r + q] * C[6 * q + c];
          Sn[6 * r + c] = a;
        }
      for (int t = 0; t < 36; ++t) U[36 * (i - 1) + t] = X[t];
    }
    if (!spd6_inv(Sn, Sinv)) return i;
    for (int t = 0; t < 36; ++t) D[36 * i + t] = Sinv[t];
  }
  // bottom: blocks N-1 .. k+1
  for (int i = N - 1; i > k; --i) {
    for (int t = 0; t < 36; ++t) Sn[t] = D[36 * i + t];
    if (i < N - 1) {
      const double* C = U + 36 * i;
      const double* Tn = D + 36 * (i + 1);
      // Y = C Tinv_{i+1};  T = A - Y C^T
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          double a = 0.0;
          for (int q = 0; q < 6; ++q) a += C[6 * r + q] * Tn[6 * q + c];
          X[6 * r + c] = a;
        }
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          double a = Sn[6 * r + c];
          for (int q = 0; q < 6; ++q) a -= X[6 * r + q] * C[6 * c + q];
          Sn[6 * r + c] = a;
        }
      for (int t = 0; t < 36; ++t) U[36 * i + t] = X[t];
    }
    if (!spd6_inv(Sn, Sinv)) return i;
    for (int t = 0; t < 36; ++t) D[36 * i + t] = Sinv[t];
  }
  // middle
  for (int t = 0; t < 36; ++t) Sn[t] = D[36 * k + t];
  if (k > 0) {
    const double* C = U + 36 * (k - 1);
    const double* Sp = D + 36 * (k - 1);
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) {
        double a = 0.0;
        for (int q = 0; q < 6; ++q) a += C[6 * q + r] * Sp[6 * q + c];
        X[6 * r + c] = a;
      }
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) {
        double a = Sn[6 * r + c];
        for (int q = 0; q < 6; ++q) a -= X[6 * r + q] * C[6 * q + c];
        Sn[6 * r + c] = a;
      }
    for (int t = 0; t < 36; ++t) U[36 * (k - 1) + t] = X[t];
  }
  if (k < N - 1) {
    const double* C = U + 36 * k;
    const double* Tn = D + 36 * (k + 1);
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) {
        double a = 0.0;
        for (int q = 0; q < 6; ++q) a += C[6 * r + q] * Tn[6 * q + c];
        X[6 * r + c] = a;
      }
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) {
        double a = Sn[6 * r + c];
        for (int q = 0; q < 6; ++q) a -= X[6 * r + q] * C[6 * c + q];
        Sn[6 * r + c] = a;
      }
    for (int t = 0; t < 36; ++t) U[36 * k + t] = X[t];
  }
  if (!spd6_inv(Sn, Sinv)) return k;
  for (int t = 0; t < 36; ++t) D[36 * k + t] = Sinv[t];
  (void)scratch;
  return -1;
}

// Solve M x = r for `nrhs` right-hand sides: r_g = rhs + g*stride, result to
// out + g*stride (out may alias rhs); tmp (same layout) holds the sweep-1 values.
DEV void twisted_solve(const TeamSerial&, int N, const double* D, const double* U, const double* rhs, double* tmp,
                       double* out, int nrhs, long stride) {
  const int k = twist_split(N);
  for (int g = 0; g < nrhs; ++g) {
    const double* b = rhs + g * stride;
    double* v = tmp + g * stride;
    double* x = out + g * stride;
    for (int r = 0; r < 6; ++r) v[r] = b[r];
    for (int i = 1; i < k; ++i) {
      const double* X = U + 36 * (i - 1);
      for (int r = 0; r < 6; ++r) {
        double a = b[6 * i + r];
        for (int j = 0; j < 6; ++j) a -= X[6 * r + j] * v[6 * (i - 1) + j];
        v[6 * i + r] = a;
      }
    }
    for (int r = 0; r < 6; ++r) v[6 * (N - 1) + r] = b[6 * (N - 1) + r];
    for (int i = N - 2; i > k; --i) {
      const double* Y = U + 36 * i;
      for (int r = 0; r < 6; ++r) {
        double a = b[6 * i + r];
        for (int j = 0; j < 6; ++j) a -= Y[6 * r + j] * v[6 * (i + 1) + j];
        v[6 * i + r] = a;
      }
    }
    double t[6];
    for (int r = 0; r < 6; ++r) {
      double pt = 0.0, pb = 0.0;
      if (k > 0)
        for (int j = 0; j < 6; ++j) pt += U[36 * (k - 1) + 6 * r + j] * v[6 * (k - 1) + j];
      if (k < N - 1)
        for (int j = 0; j < 6; ++j) pb += U[36 * k + 6 * r + j] * v[6 * (k + 1) + j];
      t[r] = b[6 * k + r] - (pt + pb);
    }
    double xk[6];
    for (int r = 0; r < 6; ++r) {
      double a = 0.0;
      for (int j = 0; j < 6; ++j) a += D[36 * k + 6 * r + j] * t[j];
      xk[r] = a;
    }
    for (int r = 0; r < 6; ++r) x[6 * k + r] = xk[r];
    for (int i = k - 1; i >= 0; --i) {
      const double* X = U + 36 * i;  // X_{i+1}
      for (int r = 0; r < 6; ++r) {
        double a = 0.0;
        for (int j = 0; j < 6; ++j) a += D[36 * i + 6 * r + j] * v[6 * i + j];
        for (int j = 0; j < 6; ++j) a -= X[6 * j + r] * x[6 * (i + 1) + j];
        x[6 * i + r] = a;
      }
    }
    for (int i = k + 1; i < N; ++i) {
      const double* Y = U + 36 * (i - 1);  // Y_{i-1}
      for (int r = 0; r < 6; ++r) {
        double a = 0.0;
        for (int j = 0; j < 6; ++j) a += D[36 * i + 6 * r + j] * v[6 * i + j];
        for (int j = 0; j < 6; ++j) a -= Y[6 * j + r] * x[6 * (i - 1) + j];
        x[6 * i + r] = a;
      }
    }
  }
}

#if defined(__CUDACC__)
// Warp factorisation: lanes 0-15 run the top recursion, lanes 16-31 the
// bottom one; within a half, lane l owns entries l and l+16 of each 6x6
// product, and every lane of the half inverts the Schur block redundantly.
DEV int twisted_factor(const TeamWarp& team, int N, double* D, double* U, double* scratch) {
  const int lane = team.lane;
  const int half = lane >> 4, hl = lane & 15;
  const int k = twist_split(N);
  double* Xs = scratch + 72 * half;  // per-half product scratch
  double* Ss = Xs + 36;
  const int steps = k > (N - 1 - k) ? k : (N - 1 - k);
  int fail = -1;
  for (int t = 0; t < steps; ++t) {
    // top step i = t (< k); bottom step i = N-1-t (> k)
    int i = half == 0 ? t : N - 1 - t;
    bool act = half == 0 ? (t < k) : (N - 1 - t > k);
    bool first = (t == 0);
    const double* C = half == 0 ? U + 36 * (i - 1) : U + 36 * i;
    const double* Pn = half == 0 ? D + 36 * (i - 1) : D + 36 * (i + 1);  // previous inverse
    if (act && !first) {
      for (int e = hl; e < 36; e += 16) {
        int r = e / 6, c = e % 6;
        double a = 0.0;
        if (half == 0)
          for (int q = 0; q < 6; ++q) a += C[6 * q + r] * Pn[6 * q + c];
        else
          for (int q = 0; q < 6; ++q) a += C[6 * r + q] * Pn[6 * q + c];
        Xs[e] = a;
      }
    }
    __syncwarp();
    if (act) {
      for (int e = hl; e < 36; e += 16) {
        int r = e / 6, c = e % 6;
        double a = D[36 * i + e];
        if (!first) {
          if (half == 0)
            for (int q = 0; q < 6; ++q) a -= Xs[6 * r + q] * C[6 * q + c];
          else
            for (int q = 0; q < 6; ++q) a -= Xs[6 * r + q] * C[6 * c + q];
        }
        Ss[e] = a;
      }
    }
    __syncwarp();
    if (act) {
      double Sr[36], Inv[36];
      for (int e = 0; e < 36; ++e) Sr[e] = Ss[e];
      bool ok = spd6_inv(Sr, Inv);
      if (!ok && fail < 0) fail = i;
      for (int e = hl; e < 36; e += 16) {
        D[36 * i + e] = Inv[e];
        if (!first) {
          if (half == 0) U[36 * (i - 1) + e] = Xs[e];
          else U[36 * i + e] = Xs[e];
        }
      }
    }
    __syncwarp();
  }
  // middle block: lanes 0-15 form X_k C_{k-1}, lanes 16-31 Y_k C_k^T
  {
    const bool has = half == 0 ? (k > 0) : (k < N - 1);
    const double* C = half == 0 ? U + 36 * (k - 1) : U + 36 * k;
    const double* Pn = half == 0 ? D + 36 * (k - 1) : D + 36 * (k + 1);
    if (has) {
      for (int e = hl; e < 36; e += 16) {
        int r = e / 6, c = e % 6;
        double a = 0.0;
        if (half == 0)
          for (int q = 0; q < 6; ++q) a += C[6 * q + r] * Pn[6 * q + c];
        else
          for (int q = 0; q < 6; ++q) a += C[6 * r + q] * Pn[6 * q + c];
        Xs[e] = a;
      }
    }
    __syncwarp();
    if (has) {
      for (int e = hl; e < 36; e += 16) {
        int r = e / 6, c = e % 6;
        double a = 0.0;
        if (half == 0)
          for (int q = 0; q < 6; ++q) a += Xs[6 * r + q] * C[6 * q + c];
        else
          for (int q = 0; q < 6; ++q) a += Xs[6 * r + q] * C[6 * c + q];
        Ss[e] = a;
      }
    } else {
      for (int e = hl; e < 36; e += 16) Ss[e] = 0.0;
    }
    __syncwarp();
    double Sr[36], Inv[36];
    for (int e = 0; e < 36; ++e) Sr[e] = D[36 * k + e] - scratch[36 + e] - scratch[72 + 36 + e];
    bool ok = spd6_inv(Sr, Inv);
    if (!ok && fail < 0) fail = k;
    __syncwarp();
    if (lane < 16) {
      for (int e = hl; e < 36; e += 16) {
        D[36 * k + e] = Inv[e];
        if (k > 0) U[36 * (k - 1) + e] = scratch[e];
      }
    } else {
      for (int e = hl; e < 36; e += 16)
        if (k < N - 1) U[36 * k + e] = scratch[72 + e];
    }
    __syncwarp();
  }
  int worst = team.imin(fail < 0 ? (1 << 30) : fail);
  return worst == (1 << 30) ? -1 : worst;
}

// Warp solve: a group of 12 lanes per right-hand side (g < 2): lanes 0-5 sweep
// the top half, lanes 6-11 the bottom half; lane row r = lane % 6.  Both
// halves run the same trip count (the shorter one idles on its last step) so
// every shuffle is warp-uniform.  out must not alias tmp.
DEV void twisted_solve(const TeamWarp& team, int N, const double* __restrict__ D, const double* __restrict__ U,
                       const double* rhs, double* tmp, double* out, int nrhs, long stride) {
  const int lane = team.lane;
  const int g = lane / 12, sub = (lane % 12) / 6, r = lane % 6;
  const bool act = g < nrhs && lane < 24;
  const int gg = act ? g : 0;
  const double* b = rhs + gg * stride;
  double* v = tmp + gg * stride;
  double* x = out + gg * stride;
  const int k = twist_split(N);
  const int grp = 12 * (g < 2 ? g : 0);
  const int base = grp + 6 * sub;       // my half
  const int other = grp + 6 * (1 - sub);
  const int my_n = sub == 0 ? k : N - 1 - k;
  const int steps = (N - 1 - k) > k ? (N - 1 - k) : k;
  // sweep 1: top i = 0..k-1 (v_i = b_i - X_i v_{i-1}); bottom i = N-1..k+1 (u_i = b_i - Y_i u_{i+1})
  double prev = 0.0;
  for (int t = 0; t < steps; ++t) {
    const bool live = t < my_n;
    const int i = sub == 0 ? t : N - 1 - t;
    double a = live ? b[6 * i + r] : 0.0;
    if (t > 0) {
      double p0 = __shfl_sync(0xffffffffu, prev, base + 0), p1 = __shfl_sync(0xffffffffu, prev, base + 1);
      double p2 = __shfl_sync(0xffffffffu, prev, base + 2), p3 = __shfl_sync(0xffffffffu, prev, base + 3);
      double p4 = __shfl_sync(0xffffffffu, prev, base + 4), p5 = __shfl_sync(0xffffffffu, prev, base + 5);
      if (live) {
        const double* M = sub == 0 ? U + 36 * (i - 1) + 6 * r : U + 36 * i + 6 * r;
        double a1 = M[1] * p1 + M[3] * p3 + M[5] * p5;
        a -= M[0] * p0 + M[2] * p2 + M[4] * p4 + a1;
      }
    }
    if (live) {
      prev = a;
      if (act) v[6 * i + r] = a;
    }
  }
  // middle: x_k = Z^{-1} (b_k - (X_k v_{k-1} + Y_k u_{k+1}))
  double part = 0.0;
  {
    const bool has = my_n > 0;
    double p0 = __shfl_sync(0xffffffffu, prev, base + 0), p1 = __shfl_sync(0xffffffffu, prev, base + 1);
    double p2 = __shfl_sync(0xffffffffu, prev, base + 2), p3 = __shfl_sync(0xffffffffu, prev, base + 3);
    double p4 = __shfl_sync(0xffffffffu, prev, base + 4), p5 = __shfl_sync(0xffffffffu, prev, base + 5);
    if (has) {
      const double* M = sub == 0 ? U + 36 * (k - 1) + 6 * r : U + 36 * k + 6 * r;
      part = M[0] * p0 + M[1] * p1 + M[2] * p2 + M[3] * p3 + M[4] * p4 + M[5] * p5;
    }
  }
  const double opart = __shfl_sync(0xffffffffu, part, other + r);
  const double ptop = sub == 0 ? part : opart, pbot = sub == 0 ? opart : part;
  const double tk = b[6 * k + r] - (ptop + pbot);
  double xk;
  {
    const double* Dk = D + 36 * k + 6 * r;
    double q0 = __shfl_sync(0xffffffffu, tk, base + 0), q1 = __shfl_sync(0xffffffffu, tk, base + 1);
    double q2 = __shfl_sync(0xffffffffu, tk, base + 2), q3 = __shfl_sync(0xffffffffu, tk, base + 3);
    double q4 = __shfl_sync(0xffffffffu, tk, base + 4), q5 = __shfl_sync(0xffffffffu, tk, base + 5);
    xk = Dk[0] * q0 + Dk[1] * q1 + Dk[2] * q2 + Dk[3] * q3 + Dk[4] * q4 + Dk[5] * q5;
  }
  __syncwarp();  // sweep-1 values visible; b fully consumed (out may alias rhs)
  if (act && sub == 0) x[6 * k + r] = xk;
  // sweep 2: top i = k-1..0 (x_i = Sinv_i v_i - X_{i+1}^T x_{i+1}); bottom i = k+1..N-1
  double xp = xk;
  for (int t = 0; t < steps; ++t) {
    const bool live = t < my_n;
    const int i = sub == 0 ? k - 1 - t : k + 1 + t;
    double dv = 0.0;
    if (live) {
      const double* Di = D + 36 * i + 6 * r;
      const double* vi = v + 6 * i;
      dv = Di[0] * vi[0] + Di[1] * vi[1] + Di[2] * vi[2] + Di[3] * vi[3] + Di[4] * vi[4] + Di[5] * vi[5];
    }
    double p0 = __shfl_sync(0xffffffffu, xp, base + 0), p1 = __shfl_sync(0xffffffffu, xp, base + 1);
    double p2 = __shfl_sync(0xffffffffu, xp, base + 2), p3 = __shfl_sync(0xffffffffu, xp, base + 3);
    double p4 = __shfl_sync(0xffffffffu, xp, base + 4), p5 = __shfl_sync(0xffffffffu, xp, base + 5);
    if (live) {
      const double* Mc = sub == 0 ? U + 36 * i + r : U + 36 * (i - 1) + r;  // column r of X_{i+1} / Y_{i-1}
      double a1 = Mc[6] * p1 + Mc[18] * p3 + Mc[30] * p5;
      xp = dv - (Mc[0] * p0 + Mc[12] * p2 + Mc[24] * p4 + a1);
      if (act) x[6 * i + r] = xp;
    }
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
