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

// symmetric positive definite 6x6 inverse via LDL^T (six reciprocals, no
// square roots; fully unrolled so everything stays in registers).  Writes
// the full symmetric inverse; false on a non-positive pivot.
DEV bool spd6_inv(const double* S, double* Inv) {
  double L[15];  // strictly lower, packed: (i, j), j < i, at i*(i-1)/2 + j
  double d[6], di[6];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double a = S[6 * j + j];
#pragma unroll
    for (int q = 0; q < j; ++q) a -= L[j * (j - 1) / 2 + q] * (L[j * (j - 1) / 2 + q] * d[q]);
    ok = ok && (a > 0.0);
    d[j] = a;
#if defined(__CUDA_ARCH__)
    di[j] = __drcp_rn(a);  // correctly rounded: the same bits as 1.0 / a, ~half the latency
#else
    di[j] = 1.0 / a;
#endif
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      double t = S[6 * i + j];
#pragma unroll
      for (int q = 0; q < j; ++q) t -= L[i * (i - 1) / 2 + q] * (L[j * (j - 1) / 2 + q] * d[q]);
      L[i * (i - 1) / 2 + j] = t * di[j];
    }
  }
  // W = L^{-1} (unit lower): W_ij = -sum_{q=j}^{i-1} L_iq W_qj
  double W[15];
#pragma unroll
  for (int i = 1; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < i; ++j) {
      double t = -L[i * (i - 1) / 2 + j];
#pragma unroll
      for (int q = j + 1; q < i; ++q) t -= L[i * (i - 1) / 2 + q] * W[q * (q - 1) / 2 + j];
      W[i * (i - 1) / 2 + j] = t;
    }
  // Inv = W^T D^{-1} W: Inv_rc = sum_{q >= max(r, c)} W_qr W_qc / d_q
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = r; c < 6; ++c) {
      double t = (c == r) ? di[r] : W[c * (c - 1) / 2 + r] * di[c];
#pragma unroll
      for (int q = c + 1; q < 6; ++q) t += W[q * (q - 1) / 2 + r] * (W[q * (q - 1) / 2 + c] * di[q]);
      Inv[6 * r + c] = t;
      Inv[6 * c + r] = t;
    }
  return ok;
}

DEV int twist_split(int N) { return (N - 1) / 2; }

// Diagonal blocks are symmetric and stored packed: 21 lower entries padded to
// kDiag doubles so every block starts 16-byte aligned.
constexpr int kDiag = 22;
DEV int sidx(int r, int c) { return r >= c ? r * (r + 1) / 2 + c : c * (c + 1) / 2 + r; }
DEV void unpack_sym(const double* p, double* a) {
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c < 6; ++c) a[6 * r + c] = p[sidx(r, c)];
}
DEV void pack_sym(double* p, const double* a) {
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) p[r * (r + 1) / 2 + c] = a[6 * r + c];
}

// 6x6 / 6-vector register loads (16-byte aligned pointers)
DEV void ld36(const double* p, double* a) {
#if defined(__CUDA_ARCH__)
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int i = 0; i < 18; ++i) {
    double2 v = q[i];
    a[2 * i] = v.x;
    a[2 * i + 1] = v.y;
  }
#else
  for (int i = 0; i < 36; ++i) a[i] = p[i];
#endif
}
DEV void st36(double* p, const double* a) {
#if defined(__CUDA_ARCH__)
  double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
  for (int i = 0; i < 18; ++i) q[i] = make_double2(a[2 * i], a[2 * i + 1]);
#else
  for (int i = 0; i < 36; ++i) p[i] = a[i];
#endif
}
DEV void ld6(const double* p, double* a) {
#if defined(__CUDA_ARCH__)
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double2 v = q[i];
    a[2 * i] = v.x;
    a[2 * i + 1] = v.y;
  }
#else
  for (int i = 0; i < 6; ++i) a[i] = p[i];
#endif
}
DEV void st6(double* p, const double* a) {
#if defined(__CUDA_ARCH__)
  double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
  for (int i = 0; i < 3; ++i) q[i] = make_double2(a[2 * i], a[2 * i + 1]);
#else
  for (int i = 0; i < 6; ++i) p[i] = a[i];
#endif
}

// In-place twisted factorisation (D packed, kDiag per block; U full 6x6).
// Returns the block of a failed pivot, or -1.
DEV bool schur_block(bool top, const double* Ap, const double* C, const double* P, double* Xout, double* Dout) {
  double X[36], S[36];
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) a += (top ? C[6 * q + r] : C[6 * r + q]) * P[6 * q + c];
      X[6 * r + c] = a;
    }
  unpack_sym(Ap, S);
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      double a = S[6 * r + c];
#pragma unroll
      for (int q = 0; q < 6; ++q) a -= X[6 * r + q] * (top ? C[6 * q + c] : C[6 * c + q]);
      S[6 * r + c] = a;
    }
  st36(Xout, X);
  double Inv[36];
  bool ok = spd6_inv(S, Inv);
  pack_sym(Dout, Inv);
  return ok;
}

DEV int twisted_factor(const TeamSerial&, int N, double* D, double* U, double* scratch, bool sh = false) {
  (void)sh;
  const int k = twist_split(N);
  int fail = -1;
  for (int half = 0; half < 2; ++half) {
    const bool top = half == 0;
    const int cnt = top ? k : N - 1 - k;
    for (int t = 0; t < cnt; ++t) {
      const int i = top ? t : N - 1 - t;
      bool ok;
      if (t == 0) {
        double S[36], Inv[36];
        unpack_sym(D + kDiag * i, S);
        ok = spd6_inv(S, Inv);
        pack_sym(D + kDiag * i, Inv);
      } else {
        double C[36], P[36];
        double* Cp = top ? U + 36 * (i - 1) : U + 36 * i;
        for (int e = 0; e < 36; ++e) C[e] = Cp[e];
        unpack_sym(top ? D + kDiag * (i - 1) : D + kDiag * (i + 1), P);
        ok = schur_block(top, D + kDiag * i, C, P, Cp, D + kDiag * i);
      }
      if (!ok && fail < 0) fail = i;
    }
    // middle contribution of this half
    double part[36];
    for (int e = 0; e < 36; ++e) part[e] = 0.0;
    if (cnt > 0) {
      double C[36], P[36], X[36];
      double* Cp = top ? U + 36 * (k - 1) : U + 36 * k;
      for (int e = 0; e < 36; ++e) C[e] = Cp[e];
      unpack_sym(top ? D + kDiag * (k - 1) : D + kDiag * (k + 1), P);
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          double a = 0.0;
          for (int q = 0; q < 6; ++q) a += (top ? C[6 * q + r] : C[6 * r + q]) * P[6 * q + c];
          X[6 * r + c] = a;
        }
      for (int e = 0; e < 36; ++e) Cp[e] = X[e];
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          double a = 0.0;
          for (int q = 0; q < 6; ++q) a += X[6 * r + q] * (top ? C[6 * q + c] : C[6 * c + q]);
          part[6 * r + c] = a;
        }
    }
    for (int e = 0; e < 36; ++e) scratch[36 * half + e] = part[e];
  }
  double S[36], Inv[36];
  unpack_sym(D + kDiag * k, S);
  for (int e = 0; e < 36; ++e) S[e] = S[e] - (scratch[e] + scratch[36 + e]);
  bool ok = spd6_inv(S, Inv);
  pack_sym(D + kDiag * k, Inv);
  if (!ok && fail < 0) fail = k;
  return fail;
}

// Solve M x = r for `nrhs` right-hand sides: r_g = rhs + g*stride, result to
// out + g*stride; tmp (same layout) holds the sweep-1 values.  out may alias
// rhs or tmp.
DEV void twisted_solve(const TeamSerial&, int N, const double* D, const double* U, const double* rhs, double* tmp,
                       double* out, int nrhs, long stride, bool sh = false, bool shv = false) {
  (void)sh;
  (void)shv;
  const int k = twist_split(N);
  for (int g = 0; g < nrhs; ++g) {
    const double* b = rhs + g * stride;
    double* v = tmp + g * stride;
    double* x = out + g * stride;
    // sweep 1, top: v_i = b_i - X_i v_{i-1};  bottom: u_i = b_i - Y_i u_{i+1}
    for (int i = 0; i < k; ++i)
      for (int r = 0; r < 6; ++r) {
        double a = b[6 * i + r];
        if (i > 0)
          for (int j = 0; j < 6; ++j) a -= U[36 * (i - 1) + 6 * r + j] * v[6 * (i - 1) + j];
        v[6 * i + r] = a;
      }
    for (int i = N - 1; i > k; --i)
      for (int r = 0; r < 6; ++r) {
        double a = b[6 * i + r];
        if (i < N - 1)
          for (int j = 0; j < 6; ++j) a -= U[36 * i + 6 * r + j] * v[6 * (i + 1) + j];
        v[6 * i + r] = a;
      }
    double t[6], xk[6];
    for (int r = 0; r < 6; ++r) {
      double pt = 0.0, pb = 0.0;
      if (k > 0)
        for (int j = 0; j < 6; ++j) pt += U[36 * (k - 1) + 6 * r + j] * v[6 * (k - 1) + j];
      if (k < N - 1)
        for (int j = 0; j < 6; ++j) pb += U[36 * k + 6 * r + j] * v[6 * (k + 1) + j];
      t[r] = b[6 * k + r] - (pt + pb);
    }
    for (int r = 0; r < 6; ++r) {
      double a = 0.0;
      for (int j = 0; j < 6; ++j) a += D[kDiag * k + sidx(r, j)] * t[j];
      xk[r] = a;
    }
    // z_i = Dinv_i v_i (in place)
    for (int i = 0; i < N; ++i) {
      if (i == k) continue;
      double z[6];
      for (int r = 0; r < 6; ++r) {
        double a = 0.0;
        for (int j = 0; j < 6; ++j) a += D[kDiag * i + sidx(r, j)] * v[6 * i + j];
        z[r] = a;
      }
      for (int r = 0; r < 6; ++r) v[6 * i + r] = z[r];
    }
    for (int r = 0; r < 6; ++r) x[6 * k + r] = xk[r];
    // sweep 2, top: x_i = z_i - X_{i+1}^T x_{i+1};  bottom: x_i = z_i - Y_{i-1}^T x_{i-1}
    for (int i = k - 1; i >= 0; --i)
      for (int r = 0; r < 6; ++r) {
        double a = v[6 * i + r];
        for (int j = 0; j < 6; ++j) a -= U[36 * i + 6 * j + r] * x[6 * (i + 1) + j];
        x[6 * i + r] = a;
      }
    for (int i = k + 1; i < N; ++i)
      for (int r = 0; r < 6; ++r) {
        double a = v[6 * i + r];
        for (int j = 0; j < 6; ++j) a -= U[36 * (i - 1) + 6 * j + r] * x[6 * (i - 1) + j];
        x[6 * i + r] = a;
      }
  }
}

DEV void twisted_solve_multi(const TeamSerial& t, int N, const double* D, const double* U, const double* rhs,
                             double* tmp, double* out, int nrhs, long stride) {
  twisted_solve(t, N, D, U, rhs, tmp, out, nrhs, stride);
}
// in-place solve of nrhs right-hand sides (rhs + g*stride) in chunks of
// kMultiRhs.  The multi-RHS sweeps need no scratch: sweep 1 overwrites each
// block's right-hand side with its v (read first), the middle block's is
// read before anything is written to it, z and x replace v in place.
DEV void twisted_solve_chunks(const TeamSerial& t, int N, const double* D, const double* U, double* rhs, int nrhs,
                              long stride, const int* rhs_block = nullptr) {
  (void)rhs_block;  // support hint used by the cyclic-reduction team only
  for (int c0 = 0; c0 < nrhs; c0 += kMultiRhs) {
    const int nb = nrhs - c0 < kMultiRhs ? nrhs - c0 : kMultiRhs;
    double* b = rhs + (long)c0 * stride;
    twisted_solve(t, N, D, U, b, b, b, nb, stride);
  }
}

DEV int q_per_half(int N) {
  const int k = twist_split(N);
  const int K = k > N - 1 - k ? k : N - 1 - k;
  return (K + 1) / 2;
}

// Q(t) and Q(t)^T for odd t in [1, K-1] of both halves -> Qg[2][half][QH][36]
template <class Team>
DEV void twisted_q(const Team& team, int N, const double* U, double* Qg) {
  const int k = twist_split(N);
  const int QH = q_per_half(N);
  PARFOR(i, 2 * QH * 36) {
    const int h = i / (QH * 36), rem = i - h * QH * 36, qi = rem / 36, e = rem - 36 * qi;
    const int K = h == 0 ? k : N - 1 - k;
    const int t = 2 * qi + 1;
    if (t > K - 1) continue;
    const double* M1 = U + 36 * (h == 0 ? k - t - 1 : k + t);
    const double* M2 = U + 36 * (h == 0 ? k - t : k + t - 1);
    const int r = e / 6, c = e - 6 * r;
    double a = 0.0;
    for (int q = 0; q < 6; ++q) a += M2[6 * r + q] * M1[6 * q + c];
    Qg[(h * QH + qi) * 36 + e] = a;                      // Q
    Qg[(2 * QH + h * QH + qi) * 36 + 6 * c + r] = a;     // Q^T
  }
  team.sync();
}

DEV void twisted_solve_la(const TeamSerial& t, int N, const double* D, const double* U, const double* Qg, double* rhs,
                          double* tmp, double* out, bool sh) {
  (void)Qg;
  twisted_solve(t, N, D, U, rhs, tmp, out, 1, 0, sh);
}

#if defined(__CUDACC__)
// Warp factorisation: lane 0 runs the top recursion, lane 1 the bottom one,
// each 6x6 step entirely in registers; they meet at the middle block.
DEV int twisted_factor_impl(const TeamWarp& team, int N, double* D, double* U, double* scratch) {
  const int lane = team.lane;
  const int k = twist_split(N);
  int fail = 1 << 30;
  if (lane < 2) {
    const bool top = lane == 0;
    const int cnt = top ? k : N - 1 - k;
    for (int t = 0; t < cnt; ++t) {
      const int i = top ? t : N - 1 - t;
      bool ok;
      if (t == 0) {
        double S[36], Inv[36];
        unpack_sym(D + kDiag * i, S);
        ok = spd6_inv(S, Inv);
        pack_sym(D + kDiag * i, Inv);
      } else {
        double C[36], P[36];
        double* Cp = top ? U + 36 * (i - 1) : U + 36 * i;
        ld36(Cp, C);
        unpack_sym(top ? D + kDiag * (i - 1) : D + kDiag * (i + 1), P);
        ok = schur_block(top, D + kDiag * i, C, P, Cp, D + kDiag * i);
      }
      if (!ok && fail == (1 << 30)) fail = i;
    }
    double part[36];
#pragma unroll
    for (int e = 0; e < 36; ++e) part[e] = 0.0;
    if (cnt > 0) {
      double C[36], P[36], X[36];
      double* Cp = top ? U + 36 * (k - 1) : U + 36 * k;
      ld36(Cp, C);
      unpack_sym(top ? D + kDiag * (k - 1) : D + kDiag * (k + 1), P);
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          double a = 0.0;
#pragma unroll
          for (int q = 0; q < 6; ++q) a += (top ? C[6 * q + r] : C[6 * r + q]) * P[6 * q + c];
          X[6 * r + c] = a;
        }
      st36(Cp, X);
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          double a = 0.0;
#pragma unroll
          for (int q = 0; q < 6; ++q) a += X[6 * r + q] * (top ? C[6 * q + c] : C[6 * c + q]);
          part[6 * r + c] = a;
        }
    }
    st36(scratch + 36 * lane, part);
  }
  __syncwarp();
  if (lane == 0) {
    double S[36], Pt[36], Pb[36], Inv[36];
    unpack_sym(D + kDiag * k, S);
    ld36(scratch, Pt);
    ld36(scratch + 36, Pb);
#pragma unroll
    for (int e = 0; e < 36; ++e) S[e] = S[e] - (Pt[e] + Pb[e]);
    bool ok = spd6_inv(S, Inv);
    pack_sym(D + kDiag * k, Inv);
    if (!ok && fail == (1 << 30)) fail = k;
  }
  __syncwarp();
  int worst = team.imin(fail);
  return worst == (1 << 30) ? -1 : worst;
}

DEV int twisted_factor(const TeamWarp& team, int N, double* D, double* U, double* scratch, bool sh = false) {
  if (sh) {
    __builtin_assume(__isShared(D));
    __builtin_assume(__isShared(U));
    return twisted_factor_impl(team, N, D, U, scratch);
  }
  return twisted_factor_impl(team, N, D, U, scratch);
}

// Single-RHS warp solve: lanes 0-5 sweep the top half, lanes 6-11 the bottom
// half, lane row r = lane % 6; each step is one 6-wide shuffle mat-vec.  The
// loops are branch-free (clamped addresses, predicated stores) and walk
// incremental pointers; `sh` states that D and U live in shared memory.
// out may alias rhs, not tmp.
template <bool SH, bool SHV>
DEV void twisted_solve_impl(const TeamWarp& team, int N, const double* __restrict__ D,
                            const double* __restrict__ U, const double* rhs, double* tmp, double* out) {
  if (SH) {
    __builtin_assume(__isShared(D));
    __builtin_assume(__isShared(U));
  }
  if (SHV) {
    __builtin_assume(__isShared(rhs));
    __builtin_assume(__isShared(tmp));
    __builtin_assume(__isShared(out));
  }
  const int lane = team.lane;
  const int sub = lane < 6 ? 0 : (lane < 12 ? 1 : 2);  // lanes >= 12 shadow the top half
  const int r = lane % 6;
  const bool act = sub < 2;
  const bool top = sub != 1;
  const int base = top ? 0 : 6;
  const int k = twist_split(N);
  const int my_n = top ? k : N - 1 - k;
  const int n_common = k < N - 1 - k ? k : N - 1 - k;
  // ---- sweep 1: top v_t = b_t - X_t v_{t-1}; bottom u_i = b_i - Y_i u_{i+1}, i = N-1-t
  const int db = top ? 6 : -6;
  const int dM = top ? 36 : -36;
  const double* bp = rhs + (top ? 0 : 6 * (N - 1)) + r;
  double* vp = tmp + (top ? 0 : 6 * (N - 1)) + r;
  const double* Mp = (top ? U : U + 36 * (N - 2)) + 6 * r;
  double prev = 0.0;
  if (my_n > 0) {
    prev = *bp;
    if (act) *vp = prev;
  }
  auto step1 = [&](bool live) {
    bp += db;
    vp += db;
    const double a0 = *bp;
    const double m0 = Mp[0], m1 = Mp[1], m2 = Mp[2], m3 = Mp[3], m4 = Mp[4], m5 = Mp[5];
    Mp += dM;
    const double p0 = __shfl_sync(0xffffffffu, prev, base + 0), p1 = __shfl_sync(0xffffffffu, prev, base + 1);
    const double p2 = __shfl_sync(0xffffffffu, prev, base + 2), p3 = __shfl_sync(0xffffffffu, prev, base + 3);
    const double p4 = __shfl_sync(0xffffffffu, prev, base + 4), p5 = __shfl_sync(0xffffffffu, prev, base + 5);
    const double a = a0 - ((m0 * p0 + m2 * p2 + m4 * p4) + (m1 * p1 + m3 * p3 + m5 * p5));
    if (live) {
      prev = a;
      if (act) *vp = a;
    }
  };
  for (int t = 1; t < n_common; ++t) step1(true);
  const int te = n_common > 1 ? n_common : 1;
  if (k != N - 1 - k) step1(te < my_n);
  // ---- middle: x_k = Zinv (b_k - (X_k v_{k-1} + Y_k u_{k+1}))
  double part;
  {
    const double* M = (top ? U + 36 * (k > 0 ? k - 1 : 0) : U + 36 * (k < N - 1 ? k : 0)) + 6 * r;
    const double m0 = M[0], m1 = M[1], m2 = M[2], m3 = M[3], m4 = M[4], m5 = M[5];
    const double p0 = __shfl_sync(0xffffffffu, prev, base + 0), p1 = __shfl_sync(0xffffffffu, prev, base + 1);
    const double p2 = __shfl_sync(0xffffffffu, prev, base + 2), p3 = __shfl_sync(0xffffffffu, prev, base + 3);
    const double p4 = __shfl_sync(0xffffffffu, prev, base + 4), p5 = __shfl_sync(0xffffffffu, prev, base + 5);
    part = my_n > 0 ? (m0 * p0 + m1 * p1 + m2 * p2 + m3 * p3 + m4 * p4 + m5 * p5) : 0.0;
  }
  const double opart = __shfl_sync(0xffffffffu, part, (top ? 6 : 0) + r);
  const double tk = rhs[6 * k + r] - ((top ? part : opart) + (top ? opart : part));
  double xk;
  {
    const double* Dk = D + kDiag * k;
    const double d0 = Dk[sidx(r, 0)], d1 = Dk[sidx(r, 1)], d2 = Dk[sidx(r, 2)];
    const double d3 = Dk[sidx(r, 3)], d4 = Dk[sidx(r, 4)], d5 = Dk[sidx(r, 5)];
    const double q0 = __shfl_sync(0xffffffffu, tk, base + 0), q1 = __shfl_sync(0xffffffffu, tk, base + 1);
    const double q2 = __shfl_sync(0xffffffffu, tk, base + 2), q3 = __shfl_sync(0xffffffffu, tk, base + 3);
    const double q4 = __shfl_sync(0xffffffffu, tk, base + 4), q5 = __shfl_sync(0xffffffffu, tk, base + 5);
    xk = (d0 * q0 + d2 * q2 + d4 * q4) + (d1 * q1 + d3 * q3 + d5 * q5);
  }
  __syncwarp();  // sweep-1 values visible; rhs fully consumed (out may alias rhs)
  // ---- z_i = Dinv_i v_i for every block but k; lane handles (block, row) pairs
  parfor4(team, 6 * N, [&](int q) {
    const int i = q / 6, rr = q - 6 * i;
    if (i != k) {
      const double* Di = D + kDiag * i;
      const double* vi = tmp + 6 * i;
      const double z = (Di[sidx(rr, 0)] * vi[0] + Di[sidx(rr, 2)] * vi[2] + Di[sidx(rr, 4)] * vi[4]) +
                       (Di[sidx(rr, 1)] * vi[1] + Di[sidx(rr, 3)] * vi[3] + Di[sidx(rr, 5)] * vi[5]);
      out[q] = z;  // out != tmp: z parked in out, consumed below before x_i overwrites it
    }
  });
  __syncwarp();
  if (sub == 0) out[6 * k + r] = xk;
  // ---- sweep 2: top x_i = z_i - X_{i+1}^T x_{i+1}, i = k-1-t; bottom x_i = z_i - Y_{i-1}^T x_{i-1}, i = k+1+t
  double xp = xk;
  const int dx = top ? -6 : 6;
  double* xo = out + 6 * k + r;
  const int dC = top ? -36 : 36;
  const double* Cp = (top ? U + 36 * (k > 0 ? k - 1 : 0) : U + 36 * (k < N - 1 ? k : 0)) + r;
  auto step2 = [&](bool live) {
    xo += dx;
    const double z = *xo;
    const double m0 = Cp[0], m1 = Cp[6], m2 = Cp[12], m3 = Cp[18], m4 = Cp[24], m5 = Cp[30];
    Cp += dC;
    const double p0 = __shfl_sync(0xffffffffu, xp, base + 0), p1 = __shfl_sync(0xffffffffu, xp, base + 1);
    const double p2 = __shfl_sync(0xffffffffu, xp, base + 2), p3 = __shfl_sync(0xffffffffu, xp, base + 3);
    const double p4 = __shfl_sync(0xffffffffu, xp, base + 4), p5 = __shfl_sync(0xffffffffu, xp, base + 5);
    const double a = z - ((m0 * p0 + m2 * p2 + m4 * p4) + (m1 * p1 + m3 * p3 + m5 * p5));
    if (live) {
      xp = a;
      if (act) *xo = a;
    }
  };
  for (int t = 0; t < n_common; ++t) step2(true);
  if (k != N - 1 - k) step2(n_common < my_n);
  __syncwarp();
}

// Odd N (equal halves, no predicates): one block per dependent step, with
// z_i = Dinv_i v_i formed inside sweep 1 from the shuffled v_i the next step
// fetches anyway (off the critical path), so no separate z pass is needed.
template <bool SH, bool SHV>
DEV void twisted_solve_odd(const TeamWarp& team, int N, const double* __restrict__ D, const double* __restrict__ U,
                           const double* rhs, double* tmp, double* out) {
  if (SH) {
    __builtin_assume(__isShared(D));
    __builtin_assume(__isShared(U));
  }
  if (SHV) {
    __builtin_assume(__isShared(rhs));
    __builtin_assume(__isShared(tmp));
    __builtin_assume(__isShared(out));
  }
  const int lane = team.lane;
  const int sub = lane < 6 ? 0 : (lane < 12 ? 1 : 2);  // lanes >= 12 shadow the top half
  const int r = lane % 6;
  const bool act = sub < 2;
  const bool top = sub != 1;
  const int base = top ? 0 : 6;
  const int k = twist_split(N), K = k;
  const int o0 = sidx(r, 0), o1 = sidx(r, 1), o2 = sidx(r, 2), o3 = sidx(r, 3), o4 = sidx(r, 4), o5 = sidx(r, 5);
  (void)tmp;
  // sweep 1: v at distance K..1 (top blocks 0..k-1, bottom N-1..k+1)
  const int db = top ? 6 : -6, dM = top ? 36 : -36, dD = top ? kDiag : -kDiag;
  const double* bp = rhs + (top ? 0 : 6 * (N - 1)) + r;
  double* zp = out + (top ? 0 : 6 * (N - 1)) + r;
  const double* Dp = D + (top ? 0 : kDiag * (N - 1));
  const double* Mp = (top ? U : U + 36 * (N - 2)) + 6 * r;
  double prev = *bp;
  double p0, p1, p2, p3, p4, p5;
  // a factor in global memory (L2; the large-N mode) is software-pipelined:
  // the rows of step t+1 are requested while step t computes
  double nm0 = 0, nm1 = 0, nm2 = 0, nm3 = 0, nm4 = 0, nm5 = 0, nd0 = 0, nd1 = 0, nd2 = 0, nd3 = 0, nd4 = 0, nd5 = 0;
  if (!SH && K > 1) {
    nm0 = Mp[0]; nm1 = Mp[1]; nm2 = Mp[2]; nm3 = Mp[3]; nm4 = Mp[4]; nm5 = Mp[5];
    nd0 = Dp[o0]; nd1 = Dp[o1]; nd2 = Dp[o2]; nd3 = Dp[o3]; nd4 = Dp[o4]; nd5 = Dp[o5];
  }
  for (int t = 1; t < K; ++t) {
    bp += db;
    const double a0 = *bp;
    double m0, m1, m2, m3, m4, m5, d0, d1, d2, d3, d4, d5;
    if (!SH) {
      m0 = nm0; m1 = nm1; m2 = nm2; m3 = nm3; m4 = nm4; m5 = nm5;
      d0 = nd0; d1 = nd1; d2 = nd2; d3 = nd3; d4 = nd4; d5 = nd5;
      const double* Mn = t + 1 < K ? Mp + dM : Mp;
      const double* Dn = t + 1 < K ? Dp + dD : Dp;
      nm0 = Mn[0]; nm1 = Mn[1]; nm2 = Mn[2]; nm3 = Mn[3]; nm4 = Mn[4]; nm5 = Mn[5];
      nd0 = Dn[o0]; nd1 = Dn[o1]; nd2 = Dn[o2]; nd3 = Dn[o3]; nd4 = Dn[o4]; nd5 = Dn[o5];
    } else {
      m0 = Mp[0]; m1 = Mp[1]; m2 = Mp[2]; m3 = Mp[3]; m4 = Mp[4]; m5 = Mp[5];
      d0 = Dp[o0]; d1 = Dp[o1]; d2 = Dp[o2]; d3 = Dp[o3]; d4 = Dp[o4]; d5 = Dp[o5];
    }
    Mp += dM;
    p0 = __shfl_sync(0xffffffffu, prev, base + 0);
    p1 = __shfl_sync(0xffffffffu, prev, base + 1);
    p2 = __shfl_sync(0xffffffffu, prev, base + 2);
    p3 = __shfl_sync(0xffffffffu, prev, base + 3);
    p4 = __shfl_sync(0xffffffffu, prev, base + 4);
    p5 = __shfl_sync(0xffffffffu, prev, base + 5);
    prev = a0 - ((m0 * p0 + m2 * p2 + m4 * p4) + (m1 * p1 + m3 * p3 + m5 * p5));
    // z of the block just left behind: Dinv row r times its v
    const double z = (d0 * p0 + d2 * p2 + d4 * p4) + (d1 * p1 + d3 * p3 + d5 * p5);
    if (act) *zp = z;
    zp += db;
    Dp += dD;
  }
  // middle: fetch v at distance 1 once more: z of that block and the coupling part
  double part;
  {
    const double* M = (top ? U + 36 * (k > 0 ? k - 1 : 0) : U + 36 * k) + 6 * r;
    const double m0 = M[0], m1 = M[1], m2 = M[2], m3 = M[3], m4 = M[4], m5 = M[5];
    const double d0 = Dp[o0], d1 = Dp[o1], d2 = Dp[o2], d3 = Dp[o3], d4 = Dp[o4], d5 = Dp[o5];
    p0 = __shfl_sync(0xffffffffu, prev, base + 0);
    p1 = __shfl_sync(0xffffffffu, prev, base + 1);
    p2 = __shfl_sync(0xffffffffu, prev, base + 2);
    p3 = __shfl_sync(0xffffffffu, prev, base + 3);
    p4 = __shfl_sync(0xffffffffu, prev, base + 4);
    p5 = __shfl_sync(0xffffffffu, prev, base + 5);
    part = K > 0 ? (m0 * p0 + m1 * p1 + m2 * p2 + m3 * p3 + m4 * p4 + m5 * p5) : 0.0;
    const double z = (d0 * p0 + d2 * p2 + d4 * p4) + (d1 * p1 + d3 * p3 + d5 * p5);
    if (act && K > 0) *zp = z;
  }
  const double opart = __shfl_sync(0xffffffffu, part, (top ? 6 : 0) + r);
  const double tk = rhs[6 * k + r] - ((top ? part : opart) + (top ? opart : part));
  double xk;
  {
    const double* Dk = D + kDiag * k;
    const double d0 = Dk[o0], d1 = Dk[o1], d2 = Dk[o2], d3 = Dk[o3], d4 = Dk[o4], d5 = Dk[o5];
    const double q0 = __shfl_sync(0xffffffffu, tk, base + 0), q1 = __shfl_sync(0xffffffffu, tk, base + 1);
    const double q2 = __shfl_sync(0xffffffffu, tk, base + 2), q3 = __shfl_sync(0xffffffffu, tk, base + 3);
    const double q4 = __shfl_sync(0xffffffffu, tk, base + 4), q5 = __shfl_sync(0xffffffffu, tk, base + 5);
    xk = (d0 * q0 + d2 * q2 + d4 * q4) + (d1 * q1 + d3 * q3 + d5 * q5);
  }
  __syncwarp();  // z written; rhs fully consumed (out may alias rhs)
  if (sub == 0) out[6 * k + r] = xk;
  // sweep 2: x at distance 1..K: x = z - M2^T x_prev (column r of M2)
  double xp = xk;
  double* xo = out + 6 * k + r;
  const int dx = top ? -6 : 6;
  const double* Cp = (top ? U + 36 * (k > 0 ? k - 1 : 0) : U + 36 * k) + r;
  const int dC = top ? -36 : 36;
  double nc0 = 0, nc1 = 0, nc2 = 0, nc3 = 0, nc4 = 0, nc5 = 0;
  if (!SH && K > 0) {
    nc0 = Cp[0]; nc1 = Cp[6]; nc2 = Cp[12]; nc3 = Cp[18]; nc4 = Cp[24]; nc5 = Cp[30];
  }
  for (int t = 0; t < K; ++t) {
    xo += dx;
    const double z = *xo;
    double m0, m1, m2, m3, m4, m5;
    if (!SH) {
      m0 = nc0; m1 = nc1; m2 = nc2; m3 = nc3; m4 = nc4; m5 = nc5;
      const double* Cn = t + 1 < K ? Cp + dC : Cp;
      nc0 = Cn[0]; nc1 = Cn[6]; nc2 = Cn[12]; nc3 = Cn[18]; nc4 = Cn[24]; nc5 = Cn[30];
    } else {
      m0 = Cp[0]; m1 = Cp[6]; m2 = Cp[12]; m3 = Cp[18]; m4 = Cp[24]; m5 = Cp[30];
    }
    Cp += dC;
    p0 = __shfl_sync(0xffffffffu, xp, base + 0);
    p1 = __shfl_sync(0xffffffffu, xp, base + 1);
    p2 = __shfl_sync(0xffffffffu, xp, base + 2);
    p3 = __shfl_sync(0xffffffffu, xp, base + 3);
    p4 = __shfl_sync(0xffffffffu, xp, base + 4);
    p5 = __shfl_sync(0xffffffffu, xp, base + 5);
    xp = z - ((m0 * p0 + m2 * p2 + m4 * p4) + (m1 * p1 + m3 * p3 + m5 * p5));
    if (act) *xo = xp;
  }
  __syncwarp();
}

DEV void twisted_solve(const TeamWarp& team, int N, const double* D, const double* U, const double* rhs, double* tmp,
                       double* out, int nrhs, long stride, bool sh = false, bool shv = false) {
  (void)nrhs;
  (void)stride;
  if (N & 1) {
    if (sh && shv) twisted_solve_odd<true, true>(team, N, D, U, rhs, tmp, out);
    else if (sh) twisted_solve_odd<true, false>(team, N, D, U, rhs, tmp, out);
    else twisted_solve_odd<false, false>(team, N, D, U, rhs, tmp, out);
    return;
  }
  if (sh && shv) twisted_solve_impl<true, true>(team, N, D, U, rhs, tmp, out);
  else if (sh) twisted_solve_impl<true, false>(team, N, D, U, rhs, tmp, out);
  else twisted_solve_impl<false, false>(team, N, D, U, rhs, tmp, out);
}

// ---------------------------------------------------------------------------
// Two-blocks-per-step ("look-ahead") variant of the single-RHS solve.
//
// Per half, index blocks by their distance t from the middle block k (top:
// block k-t, bottom: block k+t; K = blocks in the half).  With
//   M1(t) = coupling of the sweep-1 step into distance t  (top X_{k-t}, bottom Y_{k+t}),
//   M2(t) = coupling of the sweep-2 step into distance t  (top X_{k-t+1}, bottom Y_{k+t-1}),
// and Q(t) = M2(t) M1(t) for odd t (stored by twisted_q, plus its transpose),
// sweep 1 computes two blocks from one source:   v(s-1) = b(s-1) - M1(s-1) v(s),
//   v(s-2) = c(s-2) + Q(s-1) v(s),  c(s-2) = b(s-2) - M1(s-2) b(s-1),
// and sweep 2 likewise outward:                  x(s+1) = z(s+1) - M2(s+1)^T x(s),
//   x(s+2) = c'(s+2) + Q(s+1)^T x(s),  c'(s+2) = z(s+2) - M2(s+2)^T z(s+1).
// The c / c' terms are independent of the recurrence and are formed for all
// blocks in parallel first, so each dependent step still costs one 6-wide
// shuffle mat-vec but advances two blocks.  Lanes 0-11 run the top half,
// 12-23 the bottom half; within a half lanes 0-5 produce the near block and
// lanes 6-11 the far block of a step.
// ---------------------------------------------------------------------------
DEV void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// Look-ahead solve for odd N (both halves have K = k blocks, so the two
// halves run identical schedules and the loops carry no predicates).
template <bool SH>
DEV void twisted_solve_la_impl(const TeamWarp& team, int N, const double* __restrict__ D,
                               const double* __restrict__ U, const double* __restrict__ Qg, double* rhs,
                               double* tmp, double* out) {
  if (SH) {
    __builtin_assume(__isShared(D));
    __builtin_assume(__isShared(U));
    __builtin_assume(__isShared(rhs));
    __builtin_assume(__isShared(tmp));
    __builtin_assume(__isShared(out));
  }
  const int lane = team.lane;
  const int h = (lane >= 12 && lane < 24) ? 1 : 0;  // lanes 24-31 shadow the top half
  const int g = (lane % 12) / 6, r = lane % 6;
  const bool act = lane < 24;
  const int k = twist_split(N), K = k;  // N odd: N - 1 - k == k
  const int QH = q_per_half(N);
  const int sg = h == 0 ? -1 : 1;       // block(t) = k + sg t
  const bool hasA = (K & 1) && K > 1;
  const int s0 = K - (hasA ? 1 : 0);
  const int P1 = s0 >= 4 ? (s0 - 2) / 2 : 0;
  const bool hasB = s0 >= 2;
  const int P2 = K / 2;
  const bool hasC = K & 1;
  // ---- c(t) = b(t) - M1(t) b(t+1), even t in [2, s0-2] of both halves (M1(t) = U[k-t-1] / U[k+t])
  for (int q = lane; q < 12 * P1; q += 32) {
    const int hh = q >= 6 * P1 ? 1 : 0;
    const int qq = q - 6 * P1 * hh;
    const int t = 2 + 2 * (qq / 6), rr = qq - 6 * (qq / 6);
    const int s2 = hh == 0 ? -1 : 1;
    const double* M = U + 36 * (hh == 0 ? k - t - 1 : k + t) + 6 * rr;
    const double* bn = rhs + 6 * (k + s2 * (t + 1));
    rhs[6 * (k + s2 * t) + rr] -=
        (M[0] * bn[0] + M[2] * bn[2] + M[4] * bn[4]) + (M[1] * bn[1] + M[3] * bn[3] + M[5] * bn[5]);
  }
  __syncwarp();
  // ---- sweep 1 (toward the middle); the source block is held by lane group gsrc
  int gsrc = 0;
  double cur = rhs[6 * (k + sg * K) + r];
  if (act && g == 0) tmp[6 * (k + sg * K) + r] = cur;
  double p[6];
  auto fetch = [&]() {
    const int b = 12 * h + 6 * gsrc;
#pragma unroll
    for (int j = 0; j < 6; ++j) p[j] = __shfl_sync(0xffffffffu, cur, b + j);
  };
  auto dot6 = [&](const double* M, int st) {
    return (M[0] * p[0] + M[2 * st] * p[2] + M[4 * st] * p[4]) + (M[st] * p[1] + M[3 * st] * p[3] + M[5 * st] * p[5]);
  };
  if (hasA) {  // distance K-1 from K: M1(K-1) = U[k-K] / U[k+K-1]
    const double* M = U + 36 * (h == 0 ? k - K : k + K - 1) + 6 * r;
    const double a0 = rhs[6 * (k + sg * (K - 1)) + r];
    fetch();
    const double a = a0 - dot6(M, 1);
    if (g == 0) {
      cur = a;
      if (act) tmp[6 * (k + sg * (K - 1)) + r] = a;
    }
  }
  if (P1 > 0) {
    // near block s-1 (group 0): M1(s-1) row; far block s-2 (group 1): Q(s-1) row
    const double* Mp = g == 0 ? U + 36 * (h == 0 ? k - s0 : k + s0 - 1) + 6 * r
                              : Qg + (h * QH + (s0 - 2) / 2) * 36 + 6 * r;
    const int dM = g == 0 ? (h == 0 ? 72 : -72) : -36;
    const int tb0 = g == 0 ? s0 - 1 : s0 - 2;
    const double* ap = rhs + 6 * (k + sg * tb0) + r;
    double* vp = tmp + 6 * (k + sg * tb0) + r;
    const int db = h == 0 ? 12 : -12;
    for (int pi = 0; pi < P1; ++pi) {
      const double m0 = Mp[0], m1 = Mp[1], m2 = Mp[2], m3 = Mp[3], m4 = Mp[4], m5 = Mp[5];
      const double a0 = *ap;
      fetch();
      const double d = (m0 * p[0] + m2 * p[2] + m4 * p[4]) + (m1 * p[1] + m3 * p[3] + m5 * p[5]);
      cur = g == 0 ? a0 - d : a0 + d;
      if (act) *vp = cur;
      gsrc = 1;
      Mp += dM;
      ap += db;
      vp += db;
    }
  }
  if (hasB) {  // distance 1 from 2: M1(1) = U[k-2] / U[k+1]
    const double* M = U + 36 * (h == 0 ? k - 2 : k + 1) + 6 * r;
    const double a0 = rhs[6 * (k + sg) + r];
    fetch();
    const double a = a0 - dot6(M, 1);
    if (g == 0) {
      cur = a;
      if (act) tmp[6 * (k + sg) + r] = a;
    }
    gsrc = 0;
  }
  // ---- middle: x_k = Zinv (b_k - (X_k v_{k-1} + Y_k u_{k+1})); M2(1) = U[k-1] / U[k]
  double part;
  {
    const double* M = U + 36 * (h == 0 ? k - 1 : k) + 6 * r;
    fetch();
    part = K >= 1 ? (M[0] * p[0] + M[1] * p[1] + M[2] * p[2] + M[3] * p[3] + M[4] * p[4] + M[5] * p[5]) : 0.0;
  }
  const double opart = __shfl_sync(0xffffffffu, part, (h == 0 ? 12 : 0) + 6 * g + r);
  const double tk = rhs[6 * k + r] - ((h == 0 ? part : opart) + (h == 0 ? opart : part));
  double xk;
  {
    const double* Dk = D + kDiag * k;
    const double d0 = Dk[sidx(r, 0)], d1 = Dk[sidx(r, 1)], d2 = Dk[sidx(r, 2)];
    const double d3 = Dk[sidx(r, 3)], d4 = Dk[sidx(r, 4)], d5 = Dk[sidx(r, 5)];
    const int b = 12 * h + 6 * g;
    double q[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) q[j] = __shfl_sync(0xffffffffu, tk, b + j);
    xk = (d0 * q[0] + d2 * q[2] + d4 * q[4]) + (d1 * q[1] + d3 * q[3] + d5 * q[5]);
  }
  __syncwarp();  // sweep-1 values visible
  // ---- z_i = Dinv_i v_i for every block but k (parked in out)
  parfor4(team, 6 * N, [&](int q) {
    const int i = q / 6, rr = q - 6 * i;
    if (i != k) {
      const double* Di = D + kDiag * i;
      const double* vi = tmp + 6 * i;
      out[q] = (Di[sidx(rr, 0)] * vi[0] + Di[sidx(rr, 2)] * vi[2] + Di[sidx(rr, 4)] * vi[4]) +
               (Di[sidx(rr, 1)] * vi[1] + Di[sidx(rr, 3)] * vi[3] + Di[sidx(rr, 5)] * vi[5]);
    }
  });
  __syncwarp();
  // ---- c'(t) = z(t) - M2(t)^T z(t-1), even t in [2, K] (M2(t) = U[k-t] / U[k+t-1])
  for (int q = lane; q < 12 * P2; q += 32) {
    const int hh = q >= 6 * P2 ? 1 : 0;
    const int qq = q - 6 * P2 * hh;
    const int t = 2 + 2 * (qq / 6), rr = qq - 6 * (qq / 6);
    const int s2 = hh == 0 ? -1 : 1;
    const double* Mc = U + 36 * (hh == 0 ? k - t : k + t - 1) + rr;
    const double* zn = out + 6 * (k + s2 * (t - 1));
    out[6 * (k + s2 * t) + rr] -=
        (Mc[0] * zn[0] + Mc[12] * zn[2] + Mc[24] * zn[4]) + (Mc[6] * zn[1] + Mc[18] * zn[3] + Mc[30] * zn[5]);
  }
  __syncwarp();
  if (h == 0 && g == 0 && act) out[6 * k + r] = xk;
  // ---- sweep 2 (outward): near s+1 (group 0): column r of M2(s+1); far s+2 (group 1): row r of Q(s+1)^T
  cur = xk;
  gsrc = 0;
  if (P2 > 0) {
    const double* Mp = g == 0 ? U + 36 * (h == 0 ? k - 1 : k) + r : Qg + (2 * QH + h * QH) * 36 + 6 * r;
    const int st = g == 0 ? 6 : 1;
    const int dM = g == 0 ? (h == 0 ? -72 : 72) : 36;
    const int tb0 = g == 0 ? 1 : 2;
    double* op = out + 6 * (k + sg * tb0) + r;
    const int db = h == 0 ? -12 : 12;
    for (int pi = 0; pi < P2; ++pi) {
      const double m0 = Mp[0], m1 = Mp[st], m2 = Mp[2 * st], m3 = Mp[3 * st], m4 = Mp[4 * st], m5 = Mp[5 * st];
      const double a0 = *op;
      fetch();
      const double d = (m0 * p[0] + m2 * p[2] + m4 * p[4]) + (m1 * p[1] + m3 * p[3] + m5 * p[5]);
      cur = g == 0 ? a0 - d : a0 + d;
      if (act) *op = cur;
      gsrc = 1;
      Mp += dM;
      op += db;
    }
  }
  if (hasC) {  // distance K (odd) from K-1: column r of M2(K) = U[k-K] / U[k+K-1]
    const double* Mc = U + 36 * (h == 0 ? k - K : k + K - 1) + r;
    const double a0 = out[6 * (k + sg * K) + r];
    fetch();
    const double a = a0 - dot6(Mc, 6);
    if (g == 0 && act) out[6 * (k + sg * K) + r] = a;
  }
  __syncwarp();
}

DEV void twisted_solve_la(const TeamWarp& team, int N, const double* D, const double* U, const double* Qg,
                          double* rhs, double* tmp, double* out, bool sh) {
  if (!(N & 1)) {  // even N: the halves differ by one block; use the one-block-per-step solve
    twisted_solve(team, N, D, U, rhs, tmp, out, 1, 0, sh, sh);
    return;
  }
  if (sh) twisted_solve_la_impl<true>(team, N, D, U, Qg, rhs, tmp, out);
  else twisted_solve_la_impl<false>(team, N, D, U, Qg, rhs, tmp, out);
}
// Many right-hand sides (g < 16): lanes 2g / 2g+1 sweep the top / bottom half
// of RHS g with the full 6x6 mat-vec in registers; the z_i = Dinv_i v_i
// products run across all lanes between the sweeps.  out may alias rhs.
DEV void twisted_solve_multi(const TeamWarp& team, int N, const double* __restrict__ D,
                             const double* __restrict__ U, const double* rhs, double* tmp, double* out, int nrhs,
                             long stride, const int* rhs_block = nullptr) {
  const int lane = team.lane;
  const int g = lane >> 1;
  const bool top = (lane & 1) == 0;
  const bool act = g < nrhs;
  const int k = twist_split(N);
  const int cnt = top ? k : N - 1 - k;
  const double* b = rhs + (act ? g : 0) * stride;
  double* v = tmp + (act ? g : 0) * stride;
  double* x = out + (act ? g : 0) * stride;
  double p[6] = {0, 0, 0, 0, 0, 0};
  // rhs_block (in-place solves only): right-hand side g is zero outside block
  // rhs_block[g], so each half's elimination is exactly zero (and v = b there)
  // until it reaches that block; the sweep starts there
  int t0 = 0;
  if (rhs_block && act) {
    const int kb = rhs_block[g];
    t0 = top ? kb : N - 1 - kb;
    t0 = t0 < 0 ? 0 : (t0 > cnt ? cnt : t0);
  }
  if (act) {
    for (int t = t0; t < cnt; ++t) {
      const int i = top ? t : N - 1 - t;
      double a[6];
      ld6(b + 6 * i, a);
      if (t > t0) {
        double M[36];
        ld36(top ? U + 36 * (i - 1) : U + 36 * i, M);
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          double s0 = M[6 * r] * p[0] + M[6 * r + 2] * p[2] + M[6 * r + 4] * p[4];
          double s1 = M[6 * r + 1] * p[1] + M[6 * r + 3] * p[3] + M[6 * r + 5] * p[5];
          a[r] -= s0 + s1;
        }
      }
#pragma unroll
      for (int r = 0; r < 6; ++r) p[r] = a[r];
      st6(v + 6 * i, a);
    }
  }
  double part[6] = {0, 0, 0, 0, 0, 0};
  if (act && cnt > 0) {
    double M[36];
    ld36(top ? U + 36 * (k - 1) : U + 36 * k, M);
#pragma unroll
    for (int r = 0; r < 6; ++r)
      part[r] = M[6 * r] * p[0] + M[6 * r + 1] * p[1] + M[6 * r + 2] * p[2] + M[6 * r + 3] * p[3] +
                M[6 * r + 4] * p[4] + M[6 * r + 5] * p[5];
  }
  double xk[6];
  {
    double t[6], bk[6], Dk[36];
    ld6(b + 6 * k, bk);
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      double o = __shfl_xor_sync(0xffffffffu, part[r], 1);
      double pt = top ? part[r] : o, pb = top ? o : part[r];
      t[r] = bk[r] - (pt + pb);
    }
    unpack_sym(D + kDiag * k, Dk);
#pragma unroll
    for (int r = 0; r < 6; ++r)
      xk[r] = Dk[6 * r] * t[0] + Dk[6 * r + 1] * t[1] + Dk[6 * r + 2] * t[2] + Dk[6 * r + 3] * t[3] +
              Dk[6 * r + 4] * t[4] + Dk[6 * r + 5] * t[5];
  }
  __syncwarp();
  const int nb = nrhs * N;
  for (int q = lane; q < nb; q += 32) {
    const int gg = q / N, i = q - gg * N;
    if (i == k) continue;
    double* vi = tmp + gg * stride + 6 * i;
    double vv[6], Dm[36], z[6];
    ld6(vi, vv);
    unpack_sym(D + kDiag * i, Dm);
#pragma unroll
    for (int r = 0; r < 6; ++r)
      z[r] = Dm[6 * r] * vv[0] + Dm[6 * r + 1] * vv[1] + Dm[6 * r + 2] * vv[2] + Dm[6 * r + 3] * vv[3] +
             Dm[6 * r + 4] * vv[4] + Dm[6 * r + 5] * vv[5];
    st6(vi, z);
  }
  __syncwarp();
  if (act) {
    if (top) st6(x + 6 * k, xk);
#pragma unroll
    for (int r = 0; r < 6; ++r) p[r] = xk[r];
    for (int t = 0; t < cnt; ++t) {
      const int i = top ? k - 1 - t : k + 1 + t;
      double a[6], M[36];
      ld6(v + 6 * i, a);
      ld36(top ? U + 36 * i : U + 36 * (i - 1), M);
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        double s0 = M[r] * p[0] + M[12 + r] * p[2] + M[24 + r] * p[4];
        double s1 = M[6 + r] * p[1] + M[18 + r] * p[3] + M[30 + r] * p[5];
        a[r] -= s0 + s1;
      }
#pragma unroll
      for (int r = 0; r < 6; ++r) p[r] = a[r];
      st6(x + 6 * i, a);
    }
  }
  __syncwarp();
}
// CTA teams: the block-tridiagonal recurrences are warp-cooperative; warp 0
// runs them while the other warps of the team wait at the barrier.
DEV int twisted_factor(const TeamCta& t, int N, double* D, double* U, double* scratch, bool sh = false) {
  return t.on_warp0([&](const TeamWarp& w) { return twisted_factor(w, N, D, U, scratch, sh); });
}
DEV void twisted_solve(const TeamCta& t, int N, const double* D, const double* U, const double* rhs, double* tmp,
                       double* out, int nrhs, long stride, bool sh = false, bool shv = false) {
  t.on_warp0([&](const TeamWarp& w) {
    twisted_solve(w, N, D, U, rhs, tmp, out, nrhs, stride, sh, shv);
    return 0;
  });
}
DEV void twisted_solve_multi(const TeamCta& t, int N, const double* D, const double* U, const double* rhs,
                             double* tmp, double* out, int nrhs, long stride) {
  t.on_warp0([&](const TeamWarp& w) {
    twisted_solve_multi(w, N, D, U, rhs, tmp, out, nrhs, stride);
    return 0;
  });
}
// every warp of the team solves its own chunks of kMultiRhs right-hand sides, in place
DEV void twisted_solve_chunks(const TeamCta& t, int N, const double* D, const double* U, double* rhs, int nrhs,
                              long stride, const int* rhs_block = nullptr) {
  for (int c0 = t.warp * kMultiRhs; c0 < nrhs; c0 += t.nw * kMultiRhs) {
    const int nb = nrhs - c0 < kMultiRhs ? nrhs - c0 : kMultiRhs;
    double* b = rhs + (long)c0 * stride;
    twisted_solve_multi(t.w, N, D, U, b, b, b, nb, stride, rhs_block ? rhs_block + c0 : nullptr);
  }
  t.sync();
}
DEV void twisted_solve_la(const TeamCta& t, int N, const double* D, const double* U, const double* Qg, double* rhs,
                          double* tmp, double* out, bool sh) {
  t.on_warp0([&](const TeamWarp& w) {
    twisted_solve_la(w, N, D, U, Qg, rhs, tmp, out, sh);
    return 0;
  });
}
#endif

// y = M x for a symmetric block-tridiagonal (D, U) matrix (full 6x6 diagonal
// blocks); y must not alias x.  Four rows per lane per pass keep four
// independent load streams in flight (the blocks live in L2).
DEV double bt_row(int N, const double* D, const double* U, const double* x, int j) {
  const int k = j / 6, r = j - 6 * k;
  const double* dr = D + 36 * k + 6 * r;
  const double* xk = x + 6 * k;
  double acc = dr[0] * xk[0] + dr[1] * xk[1] + dr[2] * xk[2] + dr[3] * xk[3] + dr[4] * xk[4] + dr[5] * xk[5];
  if (k + 1 < N) {
    const double* ur = U + 36 * k + 6 * r;
    const double* xn = x + 6 * (k + 1);
    acc += ur[0] * xn[0] + ur[1] * xn[1] + ur[2] * xn[2] + ur[3] * xn[3] + ur[4] * xn[4] + ur[5] * xn[5];
  }
  if (k > 0) {
    const double* up = U + 36 * (k - 1) + r;
    const double* xp = x + 6 * (k - 1);
    acc += up[0] * xp[0] + up[6] * xp[1] + up[12] * xp[2] + up[18] * xp[3] + up[24] * xp[4] + up[30] * xp[5];
  }
  return acc;
}

// One block row per thread: the three 6x6 blocks are loaded as 16-byte
// vectors (54 independent loads in flight from L2), each output row keeps
// bt_row's summation order.
template <class Team>
DEV void block_matvec(const Team& team, int N, const double* D, const double* U, const double* x, double* y) {
  PARFOR(k, N) {
    double xk[6], acc[6];
    ld6(x + 6 * k, xk);
    {
      double Dk[36];
      ld36(D + 36 * k, Dk);
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double* dr = Dk + 6 * r;
        acc[r] = dr[0] * xk[0] + dr[1] * xk[1] + dr[2] * xk[2] + dr[3] * xk[3] + dr[4] * xk[4] + dr[5] * xk[5];
      }
    }
    if (k + 1 < N) {
      double Uk[36], xn[6];
      ld36(U + 36 * k, Uk);
      ld6(x + 6 * (k + 1), xn);
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double* ur = Uk + 6 * r;
        acc[r] += ur[0] * xn[0] + ur[1] * xn[1] + ur[2] * xn[2] + ur[3] * xn[3] + ur[4] * xn[4] + ur[5] * xn[5];
      }
    }
    if (k > 0) {
      double Up[36], xp[6];
      ld36(U + 36 * (k - 1), Up);
      ld6(x + 6 * (k - 1), xp);
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double* up = Up + r;
        acc[r] += up[0] * xp[0] + up[6] * xp[1] + up[12] * xp[2] + up[18] * xp[3] + up[24] * xp[4] + up[30] * xp[5];
      }
    }
    st6(y + 6 * k, acc);
  }
  team.sync();
}

}  // namespace accfem
