// Multi-level nested dissection (ND) for the 6x6 block-tridiagonal SPD
// systems, on a whole-CTA team: the latency mode's linear algebra.
//
// Replaces the reference's per-solve SuperLU factorisations (solver.py:229-247
// ADMM KKT, _solve_active_subset 500-528, _solve_equality_direct 388-421)
// after the exact reduction of SURVEY §7.1.  A solve of the twisted LDL^T
// (linalg.cuh) is a chain of ~N/2 dependent 6x6 steps and one of cyclic
// reduction (cr.cuh) ~2 log2 N barrier-separated levels of ~700 cycles each
// (scripts/micro/cr16_bench.cu); here it is a few barrier-separated dense
// mat-vec stages: one warp per segment with the segment's dense inverse in
// shared memory.
//
// Level l holds a block-tridiagonal system of nb_l blocks (diagonal D_b,
// coupling U_b = M_{b,b+1}).  With period P = G + 1 (G = kNdG), block b is a
// separator iff b % P == G; the blocks between separators form segments of
// at most G blocks (<= 30 unknowns, one lane per unknown):
//   segment c = blocks [cP, min(cP + G, nb)),  separator c = block cP + G.
// Factor: every segment's dense inverse A_c^{-1} (Gauss-Jordan in registers,
// lane = row, pivot rows staged in shared memory), then the separators'
// Schur complement, again block tridiagonal:
//   S_ss  = D_s - U_{s-1}^T A_c^{-1}[L,L] U_{s-1} - U_s A_{c+1}^{-1}[F,F] U_s^T
//   S_ss' = -U_s A_{c+1}^{-1}[F,L] U_{s'-1}
// which is level l+1; a level of at most G blocks is one segment (the top).
// Solve M x = b, per level: y_c = A_c^{-1} b_c (every segment), separator
// right-hand sides r_s = b_s - U_{s-1}^T y_{s-1} - U_s y_{s+1}, solve level
// l+1 for x_S, then x_c = y_c - A_c^{-1} (U_{sL}^T x_{sL} @F + U_L x_{sR} @L).
// Symmetric positive definite input: the Gauss-Jordan pivots are the
// Schur-complement pivots of a Cholesky factorisation and stay positive.
#pragma once
#include "../../../paper_2503_06922_b200/csrc/linalg.cuh"

namespace accfem {

constexpr int kNdG = 5;               // blocks per segment (<= 30 unknowns per warp)
constexpr int kNdP = kNdG + 1;        // period of the separators
constexpr int kNdSeg = 6 * kNdG;      // unknowns of a full segment
constexpr int kNdSegSq = kNdSeg * kNdSeg;
constexpr int kNdMaxLevels = 6;

struct NdLevel {
  int nb;          // blocks of this level's system
  int nseg, nsep;  // segments (the last may be empty) and separators
  const double* D; // diagonal blocks: level 0 the caller's packed kDiag blocks, else nb x 36 full
  double* U;       // (nb - 1) x 36 couplings (level 0: a copy of the caller's)
  double* Ainv;    // nseg x kNdSegSq segment inverses, 30 x 30 row-major (identity-padded beyond the segment)
  double* x;       // 6 nb right-hand side / solution of levels > 0
};

struct NdPlan {
  int levels;
  NdLevel L[kNdMaxLevels];
};

HDEV int nd_nsep(int nb) { return nb > kNdG ? (nb - kNdG - 1) / kNdP + 1 : 0; }
HDEV int nd_seg_first(int c) { return c * kNdP; }
HDEV int nd_seg_blocks(int nb, int c) {
  const int f = c * kNdP;
  const int e = f + kNdG < nb ? f + kNdG : nb;
  return e > f ? e - f : 0;
}

// Carve the ND storage of an N-block system over `base` (or only measure it
// with base == nullptr: *used receives the doubles).  Level 0's diagonal
// blocks are the caller's packed D0 (read during the factorisation only).
HDEV NdPlan nd_plan(int N, double* base, const double* D0, long* used = nullptr) {
  NdPlan p;
  int nb = N, l = 0;
  long off = 64;  // the plan itself is stored in the first 64 doubles
  auto take = [&](long k) {
    double* r = base ? base + off : nullptr;
    off += (k + 1) & ~1L;
    return r;
  };
  while (true) {
    NdLevel& L = p.L[l];
    L.nb = nb;
    L.nsep = nd_nsep(nb);
    L.nseg = L.nsep + 1;
    L.Ainv = take((long)L.nseg * kNdSegSq);
    L.U = take(36L * (nb > 1 ? nb - 1 : 0));
    if (l == 0) {
      L.D = D0;
      L.x = nullptr;
    } else {
      L.D = take(36L * nb);
      L.x = take(6L * nb);
    }
    ++l;
    if (L.nsep == 0 || l == kNdMaxLevels) break;
    nb = L.nsep;
  }
  p.levels = l;
  if (used) *used = off;
  return p;
}
HDEV long nd_doubles(int N) {
  long used = 0;
  nd_plan(N, nullptr, nullptr, &used);
  return used;
}
HDEV bool nd_supported(int N) {
  int nb = N, l = 0;
  while (nd_nsep(nb) > 0) {
    nb = nd_nsep(nb);
    if (++l >= kNdMaxLevels - 1) return false;
  }
  return true;
}

#if defined(__CUDACC__)
// A CTA team whose block-tridiagonal algebra is nested dissection; `nd` is
// the team's ND storage (nd_doubles(N), shared memory), `piv` 32 doubles of
// pivot-row staging per warp.
struct TeamND : TeamCta {
  double* nd;
  double* piv;
  DEV TeamND(const TeamCta& t, double* nd_, double* piv_) : TeamCta(t), nd(nd_), piv(piv_) {}
};

#define ND_SH(p) ((void)0)

// the plan stored at the head of the ND storage by nd_factor
DEV const NdPlan& nd_stored(const TeamND& t) { return *reinterpret_cast<const NdPlan*>(t.nd); }

// entry (r, c) of diagonal block b of level l (level 0 is packed symmetric)
DEV double nd_dget(const NdLevel& L, bool packed, int b, int r, int c) {
  return packed ? L.D[kDiag * b + sidx(r, c)] : L.D[36 * b + 6 * r + c];
}

// Dense inverse of segment c of level L by one warp (lane = row), padded to
// 30 x 30 with identity rows.  Returns false on a non-positive pivot.
DEV bool nd_invert_segment(const TeamWarp& w, const NdLevel& L, bool packed, int c, double* piv) {
  const int f = nd_seg_first(c), nbk = nd_seg_blocks(L.nb, c), n = 6 * nbk;
  const int i = w.lane;
  const bool act = i < kNdSeg;
  double a[kNdSeg];
  const int bi = i / 6, ri = i - 6 * bi;
#pragma unroll
  for (int j = 0; j < kNdSeg; ++j) {
    const int bj = j / 6, rj = j - 6 * bj;
    double v = (i == j && i >= n) ? 1.0 : 0.0;
    if (i < n && j < n) {
      if (bj == bi) v = nd_dget(L, packed, f + bi, ri, rj);
      else if (bj == bi + 1) v = L.U[36 * (f + bi) + 6 * ri + rj];
      else if (bj + 1 == bi) v = L.U[36 * (f + bj) + 6 * rj + ri];
    }
    a[j] = v;
  }
  bool ok = true;
#pragma unroll
  for (int k = 0; k < kNdSeg; ++k) {
    if (k < n) {
      // pivot row k scaled by 1/a_kk, with the inverse's convention in column k
      const double akk = __shfl_sync(0xffffffffu, a[k], k);
      ok = ok && (akk > 0.0);
      const double p = __drcp_rn(akk);
      const double aik = a[k];
      // broadcast of row k: lane j < 30 publishes a_kj (its own column j of row k is in lane k only)
      if (i == k) {
#pragma unroll
        for (int j = 0; j < kNdSeg; ++j) piv[j] = a[j];
      }
      __syncwarp();
      if (i != k) {
#pragma unroll
        for (int j = 0; j < kNdSeg; ++j)
          if (j != k) a[j] -= aik * (piv[j] * p);
        a[k] = -aik * p;
      } else {
#pragma unroll
        for (int j = 0; j < kNdSeg; ++j) a[j] = (j == k) ? p : a[j] * p;
      }
      __syncwarp();
    }
  }
  if (act) {
    double* out = L.Ainv + (long)c * kNdSegSq + (long)i * kNdSeg;
#pragma unroll
    for (int j = 0; j < kNdSeg; j += 2) *reinterpret_cast<double2*>(out + j) = make_double2(a[j], a[j + 1]);
  }
  return ok;
}

// element (r, q) of the 6x6 sub-block (rb, cb) of segment c's inverse
DEV double nd_ainv(const NdLevel& L, int c, int rb, int cb, int r, int q) {
  return L.Ainv[(long)c * kNdSegSq + (long)(6 * rb + r) * kNdSeg + 6 * cb + q];
}

// Schur complement of level L onto its separators -> level Nx (= L + 1); one
// warp per separator, lanes over the 36 entries of S_ss and of S_ss'
DEV void nd_schur(const TeamND& team, const NdLevel& L, bool packed, NdLevel& Nx) {
  double* D = const_cast<double*>(Nx.D);
  for (int k = team.warp; k < L.nsep; k += team.nw) {
    const int s = k * kNdP + kNdG;          // separator block
    const int cl = k, cr = k + 1;           // segments on its left / right
    const int nl = nd_seg_blocks(L.nb, cl), nr = nd_seg_blocks(L.nb, cr);
    const double* Ul = L.U + 36 * (s - 1);  // M_{s-1, s}
    for (int e = team.w.lane; e < 36; e += 32) {
      const int r = e / 6, q = e - 6 * r;
      double v = nd_dget(L, packed, s, r, q);
      {  // - U_{s-1}^T Ainv_cl[L,L] U_{s-1}
        const int lb = nl - 1;
        double acc = 0.0;
        for (int t = 0; t < 6; ++t) {
          double inner = 0.0;
          for (int u = 0; u < 6; ++u) inner += nd_ainv(L, cl, lb, lb, t, u) * Ul[6 * u + q];
          acc += Ul[6 * t + r] * inner;
        }
        v -= acc;
      }
      if (nr > 0) {  // - U_s Ainv_cr[F,F] U_s^T
        const double* Us = L.U + 36 * s;
        double acc = 0.0;
        for (int t = 0; t < 6; ++t) {
          double inner = 0.0;
          for (int u = 0; u < 6; ++u) inner += nd_ainv(L, cr, 0, 0, t, u) * Us[6 * q + u];
          acc += Us[6 * r + t] * inner;
        }
        v -= acc;
      }
      D[36 * k + e] = v;
      if (k + 1 < L.nsep) {  // S_{s,s'} = - U_s Ainv_cr[F, L] U_{s'-1}
        const int s2 = s + kNdP;
        const double* Us = L.U + 36 * s;
        const double* Ur = L.U + 36 * (s2 - 1);
        double acc = 0.0;
        for (int t = 0; t < 6; ++t) {
          double inner = 0.0;
          for (int u = 0; u < 6; ++u) inner += nd_ainv(L, cr, 0, nr - 1, t, u) * Ur[6 * u + q];
          acc += Us[6 * r + t] * inner;
        }
        Nx.U[36 * k + e] = -acc;
      }
    }
  }
}

// Factor M (packed diagonal blocks D0, couplings U0): stores the plan and a
// copy of U0 in the ND storage; returns -1, or 0 if a pivot was not positive.
static __device__ __noinline__ int nd_factor(const TeamND& team, int N, const double* D0, const double* U0) {
  NdPlan p = nd_plan(N, team.nd, D0);
  if (team.rank() == 0) *reinterpret_cast<NdPlan*>(team.nd) = p;
  for (int q = team.rank(); q < 36 * (N - 1); q += team.size()) p.L[0].U[q] = U0[q];
  team.sync();
  int bad = 0;
  double* piv = team.piv + 32 * team.warp;
  for (int l = 0; l < p.levels; ++l) {
    const NdLevel& L = p.L[l];
    const bool packed = l == 0;
    for (int c = team.warp; c < L.nseg; c += team.nw)
      if (!nd_invert_segment(team.w, L, packed, c, piv)) bad = 1;
    team.sync();
    if (l + 1 < p.levels) {
      nd_schur(team, L, packed, p.L[l + 1]);
      team.sync();
    }
  }
  bad = team.isum(bad);
  return bad ? 0 : -1;
}

// y_c = Ainv_c b_c (lane = row), in place on v; unknowns beyond the segment
// read a clamped (finite) entry against a zero coefficient
DEV void nd_seg_apply(const TeamWarp& w, const double* A, double* vs, int n) {
  ND_SH(A);
  ND_SH(vs);
  const int i = w.lane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int j = 0; j < kNdSeg; j += 3) {
    const double* ar = A + j * kNdSeg + (i < kNdSeg ? i : 0);
    a0 += ar[0] * vs[j < n ? j : n - 1];
    a1 += ar[kNdSeg] * vs[j + 1 < n ? j + 1 : n - 1];
    a2 += ar[2 * kNdSeg] * vs[j + 2 < n ? j + 2 : n - 1];
  }
  __syncwarp();
  if (i < n) vs[i] = (a0 + a1) + a2;
  __syncwarp();
}

// separator right-hand side entry q of separator k of level L from its
// in-place y: r_k = b_s - U_{s-1}^T y_{s-1} - U_s y_{s+1}
DEV double nd_sep_rhs(const NdLevel& L, const double* v, int k, int q) {
  const int s = k * kNdP + kNdG;
  const double* Ul = L.U + 36 * (s - 1);
  const double* yl = v + 6 * (s - 1);
  ND_SH(Ul);
  ND_SH(yl);
  double t0 = Ul[q] * yl[0] + Ul[12 + q] * yl[2] + Ul[24 + q] * yl[4];
  double t1 = Ul[6 + q] * yl[1] + Ul[18 + q] * yl[3] + Ul[30 + q] * yl[5];
  if (s + 1 < L.nb) {
    const double* Us = L.U + 36 * s + 6 * q;
    const double* yr = v + 6 * (s + 1);
    ND_SH(Us);
    ND_SH(yr);
    t0 += Us[0] * yr[0] + Us[2] * yr[2] + Us[4] * yr[4];
    t1 += Us[1] * yr[1] + Us[3] * yr[3] + Us[5] * yr[5];
  }
  return v[6 * s + q] - (t0 + t1);
}

// x_c = y_c - Ainv_c w_c with w_c = U_{sL}^T x_{sL} on the first block and
// U_L x_{sR} on the last (zero elsewhere): only 12 columns of Ainv_c; the
// right separator's x is copied into v
DEV void nd_seg_back(const TeamWarp& w, const NdLevel& L, int c, double* v, const double* xs) {
  const int f = nd_seg_first(c), nbk = nd_seg_blocks(L.nb, c), n = 6 * nbk;
  if (n == 0) return;
  double* vs = v + 6 * f;
  const double* A = L.Ainv + (long)c * kNdSegSq;
  const int i = w.lane;
  // lanes 0-5: w on the first block, lanes 6-11: w on the last block
  double wv = 0.0;
  if (i < 6) {
    if (c > 0) {
      const double* U = L.U + 36 * (f - 1);  // M_{sL, F}
      const double* x = xs + 6 * (c - 1);
      for (int t = 0; t < 6; ++t) wv += U[6 * t + i] * x[t];
    }
  } else if (i < 12) {
    if (c < L.nsep) {
      const double* U = L.U + 36 * (f + nbk - 1) + 6 * (i - 6);  // M_{L, sR}
      const double* x = xs + 6 * c;
      for (int t = 0; t < 6; ++t) wv += U[t] * x[t];
    }
  }
  const int lb = 6 * (nbk - 1);
  const int ii = i < kNdSeg ? i : 0;
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    const double wf = __shfl_sync(0xffffffffu, wv, t);
    const double wl = __shfl_sync(0xffffffffu, wv, 6 + t);
    a0 += A[t * kNdSeg + ii] * wf;
    a1 += A[(lb + t) * kNdSeg + ii] * wl;
  }
  if (i < n) vs[i] -= (a0 + a1);
  if (c < L.nsep && i < 6) v[6 * (f + nbk) + i] = xs[6 * c + i];
  __syncwarp();
}

#if defined(ND_TIMING)
__shared__ long long s_nd_t[32];
#define ND_T(k) do { if (threadIdx.x == 0) s_nd_t[k] = clock64(); } while (0)
#else
#define ND_T(k)
#endif
// In-place solve of nrhs right-hand sides v + g*stride with the stored factor.
static __device__ __noinline__ void nd_solve(const TeamND& team, int N, double* v, int nrhs, long stride) {
  (void)N;
  ND_T(0);
  const NdPlan& p = nd_stored(team);
  const int levels = p.levels;
  ND_T(1);
  int st = 2;
  for (int g = 0; g < nrhs; ++g) {
    double* vg = v + g * stride;
    // downward: local solves, then the separators' right-hand sides into the next level
    for (int l = 0; l < levels; ++l) {
      const NdLevel& L = p.L[l];
      double* vl = l == 0 ? vg : L.x;
      const int nb = L.nb, nseg = L.nseg, nsep = L.nsep;
      const double* Ainv = L.Ainv;
      for (int c = team.warp; c < nseg; c += team.nw) {
        const int n = 6 * nd_seg_blocks(nb, c);
        if (n > 0) nd_seg_apply(team.w, Ainv + (long)c * kNdSegSq, vl + 6 * nd_seg_first(c), n);
      }
      team.sync();
      ND_T(st++);
      if (l + 1 < levels) {
        double* xn = p.L[l + 1].x;
        for (int it = team.rank(); it < 6 * nsep; it += team.size()) xn[it] = nd_sep_rhs(L, vl, it / 6, it % 6);
        team.sync();
        ND_T(st++);
      }
    }
    // upward: back-substitution with the separators' solution
    for (int l = levels - 2; l >= 0; --l) {
      const NdLevel& L = p.L[l];
      double* vl = l == 0 ? vg : L.x;
      const double* xs = p.L[l + 1].x;
      for (int c = team.warp; c < L.nseg; c += team.nw) nd_seg_back(team.w, L, c, vl, xs);
      team.sync();
      ND_T(st++);
    }
  }
}

// ---- the linear-algebra entry points of solve.cuh for an ND team ------------
DEV int twisted_factor(const TeamND& t, int N, double* D, double* U, double* scratch, bool sh = false) {
  (void)scratch;
  (void)sh;
  return nd_factor(t, N, D, U);
}
// out = M^{-1} rhs for the matrix last factored (out may alias rhs; tmp unused)
DEV void twisted_solve(const TeamND& t, int N, const double* D, const double* U, const double* rhs, double* tmp,
                       double* out, int nrhs, long stride, bool sh = false, bool shv = false) {
  (void)D;
  (void)U;
  (void)tmp;
  (void)sh;
  (void)shv;
  if (out != rhs) {
    for (int g = 0; g < nrhs; ++g)
      for (int q = t.rank(); q < 6 * N; q += t.size()) out[g * stride + q] = rhs[g * stride + q];
    t.sync();
  }
  nd_solve(t, N, out, nrhs, stride);
}
DEV void twisted_solve_chunks(const TeamND& t, int N, const double* D, const double* U, double* rhs, int nrhs,
                              long stride) {
  (void)D;
  (void)U;
  nd_solve(t, N, rhs, nrhs, stride);
}
DEV bool dense_chol(const TeamND& team, int na, double* S, double* col);
#endif

}  // namespace accfem
