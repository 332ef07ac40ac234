// Device-side problem description and per-scenario workspace layout.
//
// HBM layout (all FP64 unless noted; scenario-major, node-minor):
//   inputs   x0[S][6N], tensions[S][nc], applied[S][6N]
//   outputs  coords[S][6N], status/frames[S] (i32), per-frame trace, contacts
//   model    rest directors N x 9, per-element constants E x {len, offset 9,
//            Qa 9, Qb 9}, K_local 12x12 (kernel parameter)
//   mesh     corners T x 9, normals T x 3, AABB lo/hi T x 3, uniform grid CSR
//   workspace one slab per resident warp (team), see Ws below
#pragma once
#include "team.cuh"

namespace accfem {

constexpr int kMaxCables = 8;
constexpr double kRhoMin = 1e-6, kRhoMax = 1e6, kRhoEqFactor = 1e3, kBig = 1e30;  // solver.py:36-38
constexpr double kMinChord = 1e-9;                                                 // beam.py:23

struct Settings {
  double eps_abs, eps_rel, rho, sigma, alpha, beta0;
  double margin, radius;  // radius = max(margin + beta0, margin)   (engine.py:148-150, contact.py:65)
  int max_iterations, check_interval, adaptive_rho, scaling_iterations, polish;
  int backend;                // 0 accelerated_qp, 1 pgs_baseline (solver.py:717-741)
  double pgs_tol;             // solver.py:57
  int pgs_min_sweep_factor;   // solver.py:58
};

struct ModelDev {
  int N;                      // nodes
  double l0;                  // element rest length
  const double* rest_dir;     // N x 9
  const double* rest_len;     // E
  const double* offsets;      // E x 9   mean0^T E0          (beam.py:97)
  const double* rest_frames;  // E x 9   E0
  const double* qa;           // E x 9   T0_a^T E0
  const double* qb;           // E x 9   T0_b^T E0
  double kl[144];             // 12 x 12 local stiffness  (beam.py:215-253)
  int n_fixed;
  const int* fixed_node;      // n_fixed
  const int* fixed_dof;       // n_fixed
  const double* fixed_inc;    // n_fixed
  const int* fixed_row_of_dof;  // 6N: selector row index or -1
  int n_cables;
  double cable_off[3 * kMaxCables];
  double cable_dir[3 * kMaxCables];
  double axis[3];             // insertion axis (engine.py:97-99)
  int has_uniform;
  double uniform[3];
};

struct MeshDev {
  int T;                      // 0 = no mesh
  const double* corners;      // T x 9
  const double* normals;      // T x 3
  const double* lo;           // T x 3 triangle AABB
  const double* hi;           // T x 3
  const int* cell_start;      // ncell + 1
  const int* cell_tris;       // CSR: triangles whose AABB is within the query radius of the cell
  double origin[3];
  double inv_h;
  int dims[3];
};

struct Problem {
  Settings s;
  ModelDev m;
  MeshDev mesh;
};

// ---------------------------------------------------------------------------
// per-team workspace, carved from one slab of `ws_doubles(N)` doubles
// ---------------------------------------------------------------------------
struct Ws {
  // element pass
  double *R, *frames, *fe, *ke, *fint, *KD, *KU;
  // assembly
  double *fa, *g, *rres;
  // contacts (indexed by node during detection, by contact after compaction)
  double *cgap, *cpp, *cnrm;
  int *ctri, *cnode, *crow_of_node;
  // rows (fixed rows first, then contacts); unscaled bounds lo/up, scaled ls/us
  double *lo, *up, *ls, *us, *e, *rho, *as, *z, *y, *yprev, *tr, *yfull, *warm;
  // scaled system; HD/HU hold H_s, then M, then its twisted factor in place
  double *HD, *HU, *gs, *d, *colh, *xs, *xt, *rhs, *w, *v, *tmp;
  // solution / polish
  double *dx, *dxp, *yp, *S, *Sy, *wfix, *scr, *W, *Sf, *Cv, *Qg;
  int *act, *alist;
  unsigned long long* prof;  // PF_COUNT counters (profile builds) or null
  bool sh;                   // hot arrays live in shared memory
  // row-state storage (z, y, rho, ls, us: cap each; as: 3 cap): `rows_hot`
  // holds frames of at most `mh` rows, larger frames use `rows_cold` (full capacity)
  double *rows_hot, *rows_cold;
  int mh, mfull;
};

// point the row-state arrays at the block that holds a frame of m rows
HDEV void ws_rows(Ws& w, int m) {
  const bool hot = m <= w.mh;
  double* b = hot ? w.rows_hot : w.rows_cold;
  const long cap = hot ? w.mh : w.mfull;
  w.z = b; w.y = b + cap; w.rho = b + 2 * cap; w.ls = b + 3 * cap; w.us = b + 4 * cap; w.as = b + 5 * cap;
}

constexpr int kMultiRhs = 16;  // right-hand sides solved concurrently by one warp (2 lanes each)

// Carve a team's workspace.  Arrays touched by every ADMM iteration (the
// factor, the scaled iterate and the row state) come from `hot` (shared
// memory on the device) when given, else from the global slab `base`.
// Either base may be null to measure: *used / *hot_used receive the sizes.
// `cr`: the coupling blocks of the factor are the cyclic-reduction layout of
// cr.cuh (one 2N x 36 array LR, HU = LR + 36) instead of the twisted one.
// `mh` > 0 selects the lean hot set of the team kernels (four teams per SM):
// only the factor, the right-hand side and the row state of frames with at
// most mh rows are hot; the iterate x, g_s and the sweep scratch (unused by
// the odd-N solve) move to the slab.
HDEV Ws ws_carve(double* base, double* hot, int N, int nf, int cmax_polish, long* used = nullptr,
                 long* hot_used = nullptr, bool cr = false, int mh = 0) {
  long n = 6L * N, E = N - 1, m = (long)nf + N;  // rows: selector rows + at most one contact per node
  long cp = cmax_polish;
  Ws w;
  long off = 0, hoff = 0;
  auto take = [&](long k) { double* r = base ? base + off : nullptr; off += (k + 3) & ~3L; return r; };
  auto takeh = [&](long k) {
    if (!hot) return take(k);
    double* r = hot + hoff;
    hoff += (k + 1) & ~1L;
    return r;
  };
  // hot: the factor (packed symmetric diagonal blocks, full couplings) and the solve vectors
  w.HD = takeh(22L * N);
  if (cr) {
    double* lr = takeh(72L * N);
    w.HU = lr ? lr + 36 : nullptr;
  } else {
    w.HU = takeh(36 * E);
  }
  const bool lean = mh > 0 && !cr && mh < m;
  w.rhs = takeh(n);
  if (lean) {
    w.tmp = (N & 1) ? take(n) : takeh(n);
    w.xs = take(n);
    w.gs = take(n);
    w.rows_hot = takeh(8L * mh);
    w.rows_cold = take(8L * m);
    w.mh = mh;
  } else {
    w.tmp = takeh(n); w.xs = takeh(n); w.gs = takeh(n);
    w.rows_hot = takeh(8L * m);
    w.rows_cold = w.rows_hot;
    w.mh = (int)m;
  }
  w.mfull = (int)m;
  ws_rows(w, 0);
  w.xt = w.rhs;  // the solve writes its result over the right-hand side
  // cold
  w.yprev = take(m); w.tr = take(m);
  w.R = take(9L * N); w.frames = take(9 * E); w.fe = take(12 * E); w.ke = take(108 * E);
  w.fint = take(n); w.KD = take(36L * N); w.KU = take(36 * E);
  w.fa = take(n); w.g = take(n); w.rres = take(n);
  w.cgap = take(N); w.cpp = take(3L * N); w.cnrm = take(3L * N);
  w.lo = take(m); w.up = take(m); w.e = take(m); w.yfull = take(m); w.warm = take(N);
  w.d = take(n); w.colh = take(n); w.w = take(n); w.v = take(n);
  w.dx = take(n); w.dxp = take(n); w.yp = take(m); w.S = take(cp * cp); w.Sy = take(3 * cp);
  w.W = take(cp * n);      // polish: P^{-1} C~_c for every contact c
  w.Sf = take(cp * cp);    // polish: C P^{-1} C~^T over all contacts
  w.Cv = take(cp);
  w.Qg = take(4L * ((N + 1) / 2 + 1) * 36);  // look-ahead products Q and Q^T of both halves
  w.wfix = take(n);
  w.scr = take(160);
  double* ib = take((5L * N + m + 8) / 2 + 1);
  int* ip = reinterpret_cast<int*>(ib);
  w.ctri = ip; ip = ip ? ip + N : nullptr;
  w.cnode = ip; ip = ip ? ip + N : nullptr;
  w.crow_of_node = ip; ip = ip ? ip + N : nullptr;
  w.act = ip; ip = ip ? ip + m : nullptr;
  w.alist = ip;
  w.prof = nullptr;
  w.sh = hot != nullptr;
  if (used) *used = off;
  if (hot_used) *hot_used = hot ? hoff : 0;
  return w;
}

HDEV long ws_doubles(int N, int nf, int cmax_polish, bool cr = false, int mh = 0) {
  long used = 0;
  ws_carve(nullptr, nullptr, N, nf, cmax_polish, &used, nullptr, cr, mh);
  return used;
}

// hot-region size (doubles) of one team (ws_carve's takeh sequence)
HDEV long ws_hot_doubles(int N, int nf, bool cr = false, int mh = 0) {
  long n = 6L * N, m = (long)nf + N;
  auto r2 = [](long k) { return (k + 1) & ~1L; };
  const long fac = r2(22L * N) + (cr ? r2(72L * N) : r2(36L * (N - 1)));
  if (mh > 0 && !cr && mh < m) return fac + r2(n) + ((N & 1) ? 0 : r2(n)) + r2(8L * mh);
  return fac + 4 * r2(n) + r2(8L * m);
}

// ---------------------------------------------------------------------------
// frame / scenario results written by the solver
// ---------------------------------------------------------------------------
struct FrameStats {
  double dx_norm, actuation_scale, max_penetration, compl_worst, residual, pri, dua;
  int iterations, n_c, converged, retried, compl_ok;
  int pairs, polish_rounds;  // broad-phase pairs and polish rounds of the frame (measurement)
};

}  // namespace accfem
