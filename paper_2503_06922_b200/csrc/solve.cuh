// The accelerated quasi-static step on one team = one scenario:
//   rows / assembly        fixed selector rows + node contact rows (contact.py:148-178,
//                          constraints.py:40-63, engine.py:123-134)
//   ruiz                   modified Ruiz equilibration (solver.py:169-212)
//   admm                   relaxed ADMM with one cached factorisation per solve
//                          (solver.py:250-385), infeasibility test (424-446)
//   direct                 contact-free frames (solver.py:388-421)
//   polish                 active-set refinement (solver.py:449-528)
//   frame / run            Engine.step / run_static incl. retry, step limit,
//                          multiplicative rotation update, warm state
//                          (engine.py:136-283, solver.py:781-833)
//
// The KKT systems are reduced to the 6x6 block-tridiagonal normal matrix
// (SURVEY §7.1): ADMM solves (H_s + sigma I + A_s^T diag(rho) A_s) x = r;
// the direct and polish solves eliminate the selector rows exactly and
// handle the active contacts through a dense Schur complement.
#pragma once
#include "cr.cuh"
#include "linalg.cuh"
#include "mech.cuh"

namespace accfem {

enum Status {
  ST_OK = 0, ST_DOMAIN = 1, ST_DEGENERATE = 2, ST_MESH = 3, ST_NONCONV = 4, ST_INFEASIBLE = 5,
  ST_ENGINE_SOLVER = 6, ST_ENGINE_MAX_FRAMES = 7, ST_CAPACITY = 8, ST_LINALG = 9
};

struct QpResult {
  double pri, dua, rho_est;  // rho_est < 0: none reported
  int iterations, converged;
  int polish_rounds;         // active-set rounds run by the polish
};

struct Frame {  // per-frame problem sizes
  int nf, nc, m;
};

// ---------------------------------------------------------------------------
// rows
// ---------------------------------------------------------------------------
template <class Team>
DEV void build_rows(const Team& team, const Problem& P, const double* x, double insertion, double scale,
                    const Frame& F, Ws& ws) {
  const ModelDev& M = P.m;
  PARFOR(r, F.m) {
    if (r < F.nf) {
      double b = M.fixed_inc[r];
      int nd = M.fixed_node[r], dof = M.fixed_dof[r];
      if (insertion != 0.0 && nd == 0 && dof < 3) b += M.axis[dof] * insertion;
      b *= scale;
      ws.lo[r] = b;
      ws.up[r] = b;
    } else {
      int c = r - F.nf;
      int nd = ws.cnode[c];
      const double* nr = ws.cnrm + 3 * c;
      const double* pp = ws.cpp + 3 * c;
      const double* p = x + 6 * nd;
      ws.lo[r] = -kBig;
      ws.up[r] = (nr[0] * pp[0] + nr[1] * pp[1] + nr[2] * pp[2]) - (nr[0] * p[0] + nr[1] * p[1] + nr[2] * p[2]);
    }
  }
  team.sync();
}

// (A v)_r with unscaled rows
DEV double row_dot(const Problem& P, const Frame& F, const Ws& ws, int r, const double* v) {
  if (r < F.nf) return v[6 * P.m.fixed_node[r] + P.m.fixed_dof[r]];
  int c = r - F.nf;
  const double* nr = ws.cnrm + 3 * c;
  const double* vv = v + 6 * ws.cnode[c];
  return nr[0] * vv[0] + nr[1] * vv[1] + nr[2] * vv[2];
}

// (A^T y)_j with unscaled rows; y indexed by row
DEV double col_dot(const Problem& P, const Frame& F, const Ws& ws, int j, const double* y) {
  double acc = 0.0;
  int fr = P.m.fixed_row_of_dof[j];
  if (fr >= 0) acc += y[fr];
  int k = j / 6, cc = j % 6;
  if (cc < 3) {
    int c = ws.crow_of_node[k];
    if (c >= 0) acc += ws.cnrm[3 * c + cc] * y[F.nf + c];
  }
  return acc;
}

// out = A^T y with unscaled rows, as two conflict-free row passes (selector
// rows hit distinct DOFs, contact rows distinct nodes) instead of a per-DOF
// gather through the row-lookup tables
template <class Team>
DEV void at_y(const Team& team, const Problem& P, const Frame& F, const Ws& ws, const double* y, double* out) {
  const int n = 6 * P.m.N;
  parfor4(team, n, [&](int j) { out[j] = 0.0; });
  team.sync();
  PARFOR(r, F.nf) out[6 * P.m.fixed_node[r] + P.m.fixed_dof[r]] += y[r];
  team.sync();
  PARFOR(c, F.nc) {
    const double yc = y[F.nf + c];
    double* o = out + 6 * ws.cnode[c];
    const double* nr = ws.cnrm + 3 * c;
    o[0] += nr[0] * yc;
    o[1] += nr[1] * yc;
    o[2] += nr[2] * yc;
  }
  team.sync();
}

// ---------------------------------------------------------------------------
// modified Ruiz equilibration of [[H, A^T], [A, 0]] + cost scaling
// (solver.py:169-212).  Produces HD/HU (scaled H), as (scaled rows), gs, d,
// e and returns c.
// ---------------------------------------------------------------------------
// packed (r, c) of entry p < 21 of a symmetric 6x6 block
DEV void sym_rc(int p, int& r, int& c) {
  r = p < 1 ? 0 : p < 3 ? 1 : p < 6 ? 2 : p < 10 ? 3 : p < 15 ? 4 : 5;
  c = p - r * (r + 1) / 2;
}

// column infinity-norm of the block-tridiagonal H at DOF j (packed diagonal blocks)
DEV double hcol_max(const double* HD, const double* HU, int N, int j) {
  const int k = j / 6, cc = j % 6;
  double mx = 0.0;
  const double* dk = HD + kDiag * k;
#pragma unroll
  for (int r = 0; r < 6; ++r) mx = fmax(mx, fabs(dk[sidx(r, cc)]));
  if (k + 1 < N) {
    const double* u = HU + 36 * k + 6 * cc;
#pragma unroll
    for (int r = 0; r < 6; ++r) mx = fmax(mx, fabs(u[r]));
  }
  if (k > 0) {
    const double* u = HU + 36 * (k - 1) + cc;
#pragma unroll
    for (int r = 0; r < 6; ++r) mx = fmax(mx, fabs(u[6 * r]));
  }
  return mx;
}

// max_i |H_ij| d_i over the 18 stored entries of column j (unscaled H in HD/HU)
DEV double hcol_wmax(const double* HD, const double* HU, const double* d, int N, int j) {
  const int k = j / 6, cc = j % 6;
  double mx = 0.0;
  const double* dk = HD + kDiag * k;
  const double* wk = d + 6 * k;
#pragma unroll
  for (int r = 0; r < 6; ++r) mx = fmax(mx, fabs(dk[sidx(r, cc)]) * wk[r]);
  if (k + 1 < N) {
    const double* u = HU + 36 * k + 6 * cc;  // block (k+1, k) = U_k^T: column cc holds U_k row cc
    const double* wn = d + 6 * (k + 1);
#pragma unroll
    for (int r = 0; r < 6; ++r) mx = fmax(mx, fabs(u[r]) * wn[r]);
  }
  if (k > 0) {
    const double* u = HU + 36 * (k - 1) + cc;
    const double* wp = d + 6 * (k - 1);
#pragma unroll
    for (int r = 0; r < 6; ++r) mx = fmax(mx, fabs(u[6 * r]) * wp[r]);
  }
  return mx;
}

// Modified Ruiz equilibration of [[H, A^T], [A, 0]] + cost scaling
// (solver.py:169-212).  The reference rescales every stored entry each
// sweep; here H stays unscaled and the sweeps only carry the diagonal
// scalings d, e and the cost factor c (the scaled column maximum of column j
// is c d_j max_i |H_ij| d_i), so each sweep is one column pass; the scaled
// matrix H_s = c D H D and A_s = E A D are formed once at the end.  The
// result equals the reference's up to rounding.
template <class Team>
DEV double ruiz(const Team& team, const Problem& P, const Frame& F, Ws& ws) {
  const int N = P.m.N, n = 6 * N, E = N - 1;
  const int nf = F.nf, m = F.m;
  double* d = ws.tmp;   // hot scratch until the ADMM loop: the running column scaling
  double* hw = ws.colh; // per column: max_i |H_ij| d_i for the current d
  double* dd = ws.v;    // this sweep's column factors
  PARFOR(i, 21 * N) {
    int k = i / 21, p = i - 21 * k, r, c;
    sym_rc(p, r, c);
    ws.HD[kDiag * k + p] = ws.KD[36 * k + 6 * r + c];
  }
  parfor4(team, 36 * E, [&](int i) { ws.HU[i] = ws.KU[i]; });
  parfor4(team, n, [&](int j) {
    ws.gs[j] = ws.g[j];
    d[j] = 1.0;
  });
  PARFOR(r, m) {
    ws.e[r] = 1.0;
    if (r < nf) {
      ws.as[3 * r] = 1.0;
    } else {
      const double* nr = ws.cnrm + 3 * (r - nf);
      ws.as[3 * r] = nr[0];
      ws.as[3 * r + 1] = nr[1];
      ws.as[3 * r + 2] = nr[2];
    }
  }
  team.sync();
  parfor4(team, n, [&](int j) { hw[j] = hcol_wmax(ws.HD, ws.HU, d, N, j); });
  team.sync();
  double c = 1.0;
  double* ee = ws.tr;
  for (int sweep = 0; sweep < P.s.scaling_iterations; ++sweep) {
    // column factors from the scaled KKT column maxima: H part, then the A
    // part scattered row by row (selector rows, then contact rows)
    parfor4(team, n, [&](int j) { dd[j] = c * d[j] * hw[j]; });
    team.sync();
    PARFOR(r, nf) {
      const int j = 6 * P.m.fixed_node[r] + P.m.fixed_dof[r];
      dd[j] = fmax(dd[j], ws.e[r] * fabs(ws.as[3 * r]) * d[j]);
    }
    team.sync();
    PARFOR(ct, m - nf) {
      const int r = nf + ct, j0 = 6 * ws.cnode[ct];
      for (int q = 0; q < 3; ++q) dd[j0 + q] = fmax(dd[j0 + q], ws.e[r] * fabs(ws.as[3 * r + q]) * d[j0 + q]);
    }
    team.sync();
    parfor4(team, n, [&](int j) {
      const double mx = dd[j];
      dd[j] = 1.0 / sqrt(mx > 1e-12 ? mx : 1.0);
    });
    PARFOR(r, m) {
      double mx;
      if (r < nf) {
        mx = ws.e[r] * fabs(ws.as[3 * r]) * d[6 * P.m.fixed_node[r] + P.m.fixed_dof[r]];
      } else {
        const int nd = ws.cnode[r - nf];
        mx = fmax(fmax(fabs(ws.as[3 * r]) * d[6 * nd], fabs(ws.as[3 * r + 1]) * d[6 * nd + 1]),
                  fabs(ws.as[3 * r + 2]) * d[6 * nd + 2]) * ws.e[r];
      }
      ee[r] = 1.0 / sqrt(mx > 1e-12 ? mx : 1.0);
    }
    team.sync();
    parfor4(team, n, [&](int j) {
      d[j] *= dd[j];
      ws.gs[j] *= dd[j];
    });
    PARFOR(r, m) ws.e[r] *= ee[r];
    team.sync();
    // cost normalisation on the column maxima of the new scaled H
    double csum = 0.0, gmax = 0.0;
    PARFOR(j, n) {
      const double w = hcol_wmax(ws.HD, ws.HU, d, N, j);
      hw[j] = w;
      csum += c * d[j] * w;
      gmax = fmax(gmax, fabs(ws.gs[j]));
    }
    csum = team.sum(csum);
    gmax = team.max(gmax);
    const double gam = 1.0 / fmax(fmax(csum / n, gmax), 1e-12);
    parfor4(team, n, [&](int j) { ws.gs[j] *= gam; });
    c *= gam;
    team.sync();
  }
  // materialise H_s = c D H D, A_s = E A D; keep d for the unscaling
  parfor4(team, 21 * N, [&](int i) {
    int k = i / 21, p = i - 21 * k, r, cc;
    sym_rc(p, r, cc);
    ws.HD[kDiag * k + p] *= c * (d[6 * k + r] * d[6 * k + cc]);
  });
  parfor4(team, 36 * E, [&](int i) {
    int k = i / 36, t = i - 36 * k, r = t / 6, cc = t - 6 * r;
    ws.HU[i] *= c * (d[6 * k + r] * d[6 * (k + 1) + cc]);
  });
  PARFOR(r, m) {
    if (r < nf) {
      ws.as[3 * r] *= ws.e[r] * d[6 * P.m.fixed_node[r] + P.m.fixed_dof[r]];
    } else {
      const int nd = ws.cnode[r - nf];
      for (int q = 0; q < 3; ++q) ws.as[3 * r + q] *= ws.e[r] * d[6 * nd + q];
    }
  }
  parfor4(team, n, [&](int j) { ws.d[j] = d[j]; });
  team.sync();
  return c;
}

// ---------------------------------------------------------------------------
// residual norms of the unscaled problem at (dx = d o xs, y = e o ys / c)
// ---------------------------------------------------------------------------
struct Residuals {
  double pri, dua, ps, ds;
};

template <class Team>
DEV Residuals unscaled_residuals(const Team& team, const Problem& P, const Frame& F, Ws& ws, double c,
                                 double gnorm) {
  const int N = P.m.N, n = 6 * N;
  double* xu = ws.tmp;
  parfor4(team, n, [&](int j) { xu[j] = ws.d[j] * ws.xs[j]; });
  team.sync();
  double pri = 0.0, ps = 0.0;
  PARFOR(r, F.m) {
    double ax = row_dot(P, F, ws, r, xu);
    double zu = ws.z[r] / ws.e[r];
    ws.yfull[r] = ws.e[r] * ws.y[r] / c;
    pri = fmax(pri, fabs(ax - zu));
    ps = fmax(ps, fmax(fabs(ax), fabs(zu)));
  }
  block_matvec(team, N, ws.KD, ws.KU, xu, ws.v);  // includes sync
  at_y(team, P, F, ws, ws.yfull, ws.w);
  double dua = 0.0, ds = 0.0;
  parfor4(team, n, [&](int j) {
    const double hx = ws.v[j], aty = ws.w[j];
    dua = fmax(dua, fabs(hx + ws.g[j] + aty));
    ds = fmax(ds, fmax(fabs(hx), fabs(aty)));
  });
  Residuals R;
  R.pri = team.max(pri);
  R.ps = team.max(ps);
  R.dua = team.max(dua);
  R.ds = fmax(team.max(ds), gnorm);
  return R;
}

// OSQP-style primal infeasibility test on the dual increment (solver.py:424-446)
template <class Team>
DEV bool infeasible(const Team& team, const Problem& P, const Frame& F, Ws& ws, double c) {
  const int n = 6 * P.m.N;
  double nd = 0.0;
  PARFOR(r, F.m) {
    double v = ws.e[r] * (ws.y[r] - ws.yprev[r]) / c;
    ws.tr[r] = v;
    nd = fmax(nd, fabs(v));
  }
  nd = team.max(nd);
  double eps = fmax(P.s.eps_abs, 1e-10);
  if (nd <= eps) return false;
  team.sync();
  double sup_u = 0.0, sup_l = 0.0;
  PARFOR(r, F.m) {
    double v = ws.tr[r] / nd;
    ws.tr[r] = v;
    sup_u += ws.up[r] * fmax(v, 0.0);
    sup_l += ws.lo[r] * fmin(v, 0.0);
  }
  double support = team.sum(sup_u) + team.sum(sup_l);
  team.sync();
  if (!(support < -eps)) return false;
  at_y(team, P, F, ws, ws.tr, ws.w);
  double at = 0.0;
  parfor4(team, n, [&](int j) { at = fmax(at, fabs(ws.w[j])); });
  at = team.max(at);
  return at <= eps;
}

// ---------------------------------------------------------------------------
// reduced unscaled factor for the direct / polish solves: H (+ delta I on free
// DOFs) with selector DOFs replaced by identity rows/columns, factored in place
// in HD/HU
// ---------------------------------------------------------------------------
template <class Team>
DEV int reduced_factor(const Team& team, const Problem& P, double delta, Ws& ws) {
  const int N = P.m.N, E = N - 1;
  const int* frd = P.m.fixed_row_of_dof;
  PARFOR(i, 21 * N) {
    int k = i / 21, p = i - 21 * k, r, cc;
    sym_rc(p, r, cc);
    bool fr = frd[6 * k + r] >= 0, fc = frd[6 * k + cc] >= 0;
    double v = ws.KD[36 * k + 6 * r + cc];
    if (fr || fc) v = (r == cc) ? 1.0 : 0.0;
    else if (r == cc) v += delta;
    ws.HD[kDiag * k + p] = v;
  }
  PARFOR(i, 36 * E) {
    int k = i / 36, t = i - 36 * k, r = t / 6, cc = t - 6 * r;
    bool fr = frd[6 * k + r] >= 0, fc = frd[6 * (k + 1) + cc] >= 0;
    ws.HU[i] = (fr || fc) ? 0.0 : ws.KU[i];
  }
  team.sync();
  return twisted_factor(team, N, ws.HD, ws.HU, ws.scr, ws.sh);
}

// full-length rhs for the eliminated system: b at selector DOFs,
// -g - H_{:,F} b at free DOFs.  bvec (selector values by DOF) -> out
template <class Team>
DEV void eliminated_rhs(const Team& team, const Problem& P, const Frame& F, Ws& ws, double* out) {
  const int N = P.m.N, n = 6 * N;
  double* bvec = ws.w;
  PARFOR(j, n) {
    int fr = P.m.fixed_row_of_dof[j];
    bvec[j] = fr >= 0 ? ws.up[fr] : 0.0;
  }
  team.sync();
  block_matvec(team, N, ws.KD, ws.KU, bvec, ws.tmp);
  PARFOR(j, n) {
    int fr = P.m.fixed_row_of_dof[j];
    out[j] = fr >= 0 ? ws.up[fr] : -ws.g[j] - ws.tmp[j];
  }
  team.sync();
}

// selector multipliers from the exact KKT rows: y_r = -((H dx)_j + g_j + (C^T y_c)_j)
template <class Team>
DEV void selector_multipliers(const Team& team, const Problem& P, const Frame& F, Ws& ws, const double* dx,
                              double* yrow) {
  block_matvec(team, P.m.N, ws.KD, ws.KU, dx, ws.tmp);
  PARFOR(r, F.nf) {
    int j = 6 * P.m.fixed_node[r] + P.m.fixed_dof[r];
    double acc = ws.tmp[j] + ws.g[j];
    int k = j / 6, cc = j % 6;
    if (cc < 3) {
      int c = ws.crow_of_node[k];
      if (c >= 0) acc += ws.cnrm[3 * c + cc] * yrow[F.nf + c];
    }
    yrow[r] = -acc;
  }
  team.sync();
}

// contact-free frame: exact selector elimination + 3 refinement rounds
// (solver.py:388-421).  Writes ws.dx and ws.yfull[0..nf).
template <class Team>
DEV int direct_solve(const Team& team, const Problem& P, const Frame& F, Ws& ws, QpResult& res) {
  const int N = P.m.N, n = 6 * N;
  if (reduced_factor(team, P, 0.0, ws) >= 0) return ST_LINALG;
  eliminated_rhs(team, P, F, ws, ws.rhs);
  twisted_solve(team, N, ws.HD, ws.HU, ws.rhs, ws.tmp, ws.dx, 1, 0, ws.sh);
  team.sync();
  for (int it = 0; it < 3; ++it) {
    block_matvec(team, N, ws.KD, ws.KU, ws.dx, ws.tmp);
    PARFOR(j, n) {
      bool fx = P.m.fixed_row_of_dof[j] >= 0;
      ws.rhs[j] = fx ? 0.0 : -ws.g[j] - ws.tmp[j];
    }
    team.sync();
    twisted_solve(team, N, ws.HD, ws.HU, ws.rhs, ws.tmp, ws.w, 1, 0, ws.sh);
    team.sync();
    PARFOR(j, n) ws.dx[j] += ws.w[j];
    team.sync();
  }
  selector_multipliers(team, P, F, ws, ws.dx, ws.yfull);
  double dua = 0.0;
  block_matvec(team, N, ws.KD, ws.KU, ws.dx, ws.tmp);
  at_y(team, P, F, ws, ws.yfull, ws.w);
  parfor4(team, n, [&](int j) { dua = fmax(dua, fabs(ws.tmp[j] + ws.g[j] + ws.w[j])); });
  res.pri = 0.0;
  res.dua = team.max(dua);
  res.iterations = 0;
  res.converged = 1;
  res.rho_est = -1.0;
  return ST_OK;
}

// dense Cholesky + solve of the na x na Schur complement (row-major, ld = na)
template <class Team>
DEV bool dense_chol(const Team& team, int na, double* S) {
  for (int k = 0; k < na; ++k) {
    double piv = S[k * na + k];
    if (!(piv > 0.0)) return false;
    double l = sqrt(piv);
    team.sync();
    PARFOR(i, na - k) {
      int r = k + i;
      S[r * na + k] = (r == k) ? l : S[r * na + k] / l;
    }
    team.sync();
    int rem = na - k - 1;
    PARFOR(t, rem * rem) {
      int r = k + 1 + t / rem, cc = k + 1 + t % rem;
      if (cc <= r) S[r * na + cc] -= S[r * na + k] * S[cc * na + k];
    }
    team.sync();
  }
  return true;
}

#if defined(__CUDACC__)
// CTA teams: the small dense Schur factorisation and its solves run on warp 0
// with warp barriers only (a CTA barrier per pivot costs ~10x a pivot's work);
// every entry sees the same sequence of operations as the generic version.
DEV bool dense_chol_warp(const TeamWarp& w, int na, double* S) {
  for (int k = 0; k < na; ++k) {
    const double piv = S[k * na + k];
    if (!(piv > 0.0)) return false;
    const double l = sqrt(piv);
    __syncwarp();
    for (int r = k + w.lane; r < na; r += 32) S[r * na + k] = (r == k) ? l : S[r * na + k] / l;
    __syncwarp();
    for (int r = k + 1 + w.lane; r < na; r += 32) {
      const double srk = S[r * na + k];
      double* Sr = S + (long)r * na;
      for (int cc = k + 1; cc <= r; ++cc) Sr[cc] -= srk * S[cc * na + k];
    }
    __syncwarp();
  }
  return true;
}
DEV void dense_solve_warp(const TeamWarp& w, int na, const double* S, double* b) {
  for (int k = 0; k < na; ++k) {
    const double bk = b[k] / S[k * na + k];
    __syncwarp();
    if (w.lane == 0) b[k] = bk;
    for (int r = k + 1 + w.lane; r < na; r += 32) b[r] -= S[r * na + k] * bk;
    __syncwarp();
  }
  for (int k = na - 1; k >= 0; --k) {
    const double bk = b[k] / S[k * na + k];
    __syncwarp();
    if (w.lane == 0) b[k] = bk;
    for (int i = w.lane; i < k; i += 32) b[i] -= S[k * na + i] * bk;
    __syncwarp();
  }
}
// up to this many active contacts the Schur factor/solves run on one warp;
// larger systems (the 1000-node configs: 200-250 contacts) use the whole team,
// the scaled column copied to the contiguous `col`, the trailing lower triangle
// updated in panels with the lanes along a row (coalesced)
constexpr int kDenseWarpMax = 64;
DEV bool dense_chol(const TeamCta& team, int na, double* S, double* col) {
  team.sync();  // S assembled by the whole team
  if (na <= kDenseWarpMax)
    return team.on_warp0([&](const TeamWarp& w) { return dense_chol_warp(w, na, S) ? 1 : 0; }) != 0;
  // Right-looking, in panels of kPanel columns: inside a panel the columns are
  // factored one by one (a thread per row updates its panel entries); the
  // trailing matrix then takes the panel's kPanel updates in one pass per entry,
  // in column order -- every entry sees the same fused multiply-adds in the same
  // order as the column-by-column algorithm, with one L2 round trip per panel
  // instead of per column.
  constexpr int kPanel = 8;
  for (int k0 = 0; k0 < na; k0 += kPanel) {
    const int k1 = k0 + kPanel < na ? k0 + kPanel : na;
    for (int k = k0; k < k1; ++k) {
      const double piv = S[k * na + k];
      if (!(piv > 0.0)) return false;
      const double l = sqrt(piv);
      team.sync();
      PARFOR(i, na - k) {
        const int r = k + i;
        const double v = (r == k) ? l : S[r * na + k] / l;
        S[r * na + k] = v;
        col[r] = v;
      }
      team.sync();
      // panel columns c in (k, k1), rows r >= c
      PARFOR(i, na - k - 1) {
        const int r = k + 1 + i;
        const double cr = col[r];
        double* Sr = S + (long)r * na;
        double a[kPanel - 1], x[kPanel - 1];
#pragma unroll
        for (int j = 0; j < kPanel - 1; ++j) {
          const int c = k + 1 + j;
          const bool in = c < k1 && c <= r;
          a[j] = in ? Sr[c] : 0.0;
          x[j] = in ? col[c] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kPanel - 1; ++j) {
          const int c = k + 1 + j;
          if (c < k1 && c <= r) Sr[c] = a[j] - cr * x[j];
        }
      }
      team.sync();
    }
    // trailing entries (r, c), k1 <= c <= r: four rows per warp, lanes along c
    for (int r0 = k1 + team.warp; r0 < na; r0 += 4 * team.nw) {
      int rr[4];
      double lr[4][kPanel];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        rr[i] = r0 + i * team.nw;
#pragma unroll
        for (int t = 0; t < kPanel; ++t)
          lr[i][t] = rr[i] < na && k0 + t < k1 ? S[(long)rr[i] * na + k0 + t] : 0.0;
      }
      const int rmax = rr[3] < na ? rr[3] : na - 1;
      for (int cc = k1 + team.w.lane; cc <= rmax; cc += 32) {
        double lc[kPanel], a[4];
#pragma unroll
        for (int t = 0; t < kPanel; ++t) lc[t] = k0 + t < k1 ? S[(long)cc * na + k0 + t] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = rr[i] < na && cc <= rr[i] ? S[(long)rr[i] * na + cc] : 0.0;
#pragma unroll
        for (int t = 0; t < kPanel; ++t)
          if (k0 + t < k1) {
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = a[i] - lr[i][t] * lc[t];
          }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (rr[i] < na && cc <= rr[i]) S[(long)rr[i] * na + cc] = a[i];
      }
    }
    team.sync();
  }
  return true;
}
DEV void dense_solve(const TeamCta& team, int na, const double* S, double* b) {
  team.sync();
  if (na <= kDenseWarpMax) {
    team.on_warp0([&](const TeamWarp& w) {
      dense_solve_warp(w, na, S, b);
      return 0;
    });
    return;
  }
  for (int k = 0; k < na; ++k) {
    team.sync();
    double bk = b[k] / S[k * na + k];
    team.sync();
    if (team.rank() == 0) b[k] = bk;
    PARFOR(i, na - k - 1) {
      int r = k + 1 + i;
      b[r] -= S[r * na + k] * bk;
    }
  }
  for (int k = na - 1; k >= 0; --k) {
    team.sync();
    double bk = b[k] / S[k * na + k];
    team.sync();
    if (team.rank() == 0) b[k] = bk;
    PARFOR(i, k) b[i] -= S[k * na + i] * bk;
  }
  team.sync();
}
DEV bool dense_chol(const TeamCR& team, int na, double* S, double* col) {
  return dense_chol(static_cast<const TeamCta&>(team), na, S, col);
}
DEV void dense_solve(const TeamCR& team, int na, const double* S, double* b) {
  dense_solve(static_cast<const TeamCta&>(team), na, S, b);
}
#endif
template <class Team>
DEV bool dense_chol(const Team& team, int na, double* S, double* col) {
  (void)col;
  return dense_chol(team, na, S);
}

template <class Team>
DEV void dense_solve(const Team& team, int na, const double* S, double* b) {
  for (int k = 0; k < na; ++k) {
    team.sync();
    double bk = b[k] / S[k * na + k];
    team.sync();
    if (team.rank() == 0) b[k] = bk;
    PARFOR(i, na - k - 1) {
      int r = k + 1 + i;
      b[r] -= S[r * na + k] * bk;
    }
  }
  for (int k = na - 1; k >= 0; --k) {
    team.sync();
    double bk = b[k] / S[k * na + k];
    team.sync();
    if (team.rank() == 0) b[k] = bk;
    PARFOR(i, k) b[i] -= S[k * na + i] * bk;
  }
  team.sync();
}

// active-set polish (solver.py:449-528).  On entry ws.dx / ws.yfull hold the
// ADMM result (yfull unclipped); on acceptance they are replaced.
//
// Every round solves the regularised reduced KKT [[H+dI, C^T], [C, -dI]] of
// the active rows with the selector DOFs eliminated exactly, through a dense
// Schur complement over the active contacts.  P = H + dI (reduced) is factored
// once; W_c = P^{-1} C~_c for ALL contacts, S = C W and v = P^{-1} f are
// formed once per polish, so a round costs one block solve (the refinement
// round of _solve_active_subset) plus dense work on the active submatrix.
template <class Team>
DEV void dense_combine(const Team& team, int n, int na, const int* alist, const double* W, const double* y,
                       const double* base, double* out) {
  // four columns per thread, four contacts per pass: 16 independent W loads in
  // flight (the W panel is L2/HBM-resident for large N); each column still
  // accumulates in contact order
  const int s = team.size();
  for (int j0 = team.rank(); j0 < n; j0 += 4 * s) {
    int jj[4];
    double acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      jj[u] = j0 + u * s < n ? j0 + u * s : n - 1;
      acc[u] = base[jj[u]];
    }
    int q = 0;
    for (; q + 4 <= na; q += 4) {
      const double* w0 = W + (long)alist[q] * n;
      const double* w1 = W + (long)alist[q + 1] * n;
      const double* w2 = W + (long)alist[q + 2] * n;
      const double* w3 = W + (long)alist[q + 3] * n;
      const double y0 = y[q], y1 = y[q + 1], y2 = y[q + 2], y3 = y[q + 3];
      double e0[4], e1[4], e2[4], e3[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        e0[u] = w0[jj[u]];
        e1[u] = w1[jj[u]];
        e2[u] = w2[jj[u]];
        e3[u] = w3[jj[u]];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[u] -= y0 * e0[u];
        acc[u] -= y1 * e1[u];
        acc[u] -= y2 * e2[u];
        acc[u] -= y3 * e3[u];
      }
    }
    for (; q < na; ++q) {
      const double* wq = W + (long)alist[q] * n;
      const double yq = y[q];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] -= yq * wq[jj[u]];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u * s < n) out[j0 + u * s] = acc[u];
  }
  team.sync();
}

template <class Team>
DEV int polish(const Team& team, const Problem& P, const Frame& F, Ws& ws, QpResult& res, int cmax) {
  const int N = P.m.N, n = 6 * N, nf = F.nf, nc = F.nc;
  const double tol_act = fmax(10.0 * P.s.eps_abs, 1e-12);
  const double delta = 1e-9;
  if (nc > cmax) return ST_CAPACITY;
  PARFOR(c, nc) {
    int r = nf + c;
    double yc = fmax(ws.yfull[r], 0.0);
    double slack = ws.up[r] - row_dot(P, F, ws, r, ws.dx);
    ws.act[c] = (yc > tol_act) || (slack < tol_act);
  }
  team.sync();
  PROF_T0(t_pf);
  if (reduced_factor(team, P, delta, ws) >= 0) return ST_OK;  // splu failure -> no polish
  PROF_ADD(ws, PF_POL_FACTOR, t_pf);
  PROF_T0(t_pw);
  // W_c = P^{-1} C~_c (C~: contact row with selector DOFs zeroed); every warp
  // of the team solves its own chunks of 16 contacts
  parfor4(team, nc * n, [&](int t) { ws.W[t] = 0.0; });
  team.sync();
  PARFOR(c, nc) {
    const int nd = ws.cnode[c];
    for (int a = 0; a < 3; ++a) {
      const int j = 6 * nd + a;
      if (P.m.fixed_row_of_dof[j] < 0) ws.W[(long)c * n + j] = ws.cnrm[3 * c + a];
    }
  }
  team.sync();
  twisted_solve_chunks(team, N, ws.HD, ws.HU, ws.W, nc, n, ws.cnode);
  PARFOR(t, nc * nc) {
    const int p = t / nc, q = t - p * nc;
    const double* nr = ws.cnrm + 3 * p;
    const double* wq = ws.W + (long)q * n + 6 * ws.cnode[p];
    ws.Sf[t] = nr[0] * wq[0] + nr[1] * wq[1] + nr[2] * wq[2];
  }
  // v = P^{-1} f with f the eliminated right-hand side; Cv_c = C_c v
  eliminated_rhs(team, P, F, ws, ws.xt);
  twisted_solve(team, N, ws.HD, ws.HU, ws.xt, ws.tmp, ws.v, 1, 0, ws.sh);
  team.sync();
  PARFOR(c, nc) ws.Cv[c] = row_dot(P, F, ws, nf + c, ws.v);
  team.sync();
  bool found = false;
  double* dxp = ws.dxp;
  double* yp = ws.yp;
  double* yact = ws.Sy + cmax;      // na entries
  double* dyq = ws.Sy + 2 * cmax;   // na entries
  PROF_ADD(ws, PF_POL_W, t_pw);
  PROF_T0(t_pr);
  for (int round = 0; round < 6; ++round) {
    res.polish_rounds = round + 1;
    PROF_T0(t_r0);
    // active contact list in row order
    int na = 0;
    for (int base = 0; base < nc; base += team.size()) {
      int c = base + team.rank();
      bool a = c < nc && ws.act[c];
      int tot = 0;
      int pos = team.ballot_prefix(a, &tot);
      if (a) ws.alist[na + pos] = c;
      na += tot;
    }
    team.sync();
    PARFOR(q, na) ws.alist[N + ws.alist[q]] = q;
    team.sync();
    if (nf + na == 0) break;
    PROF_ADD(ws, PF_PR_LIST, t_r0);
    PROF_T0(t_r1);
    // S_a = S[act, act] + delta I, factored
    PARFOR(t, na * na) {
      const int p = t / na, q = t - p * na;
      const int cp = ws.alist[p], cq = ws.alist[q];
      // the two triangles of C P^{-1} C~^T agree to rounding; use the lower one
      double v = cp >= cq ? ws.Sf[cp * nc + cq] : ws.Sf[cq * nc + cp];
      ws.S[t] = v + (p == q ? delta : 0.0);
    }
    team.sync();
    if (na > 0 && !dense_chol(team, na, ws.S, ws.Sy)) return ST_OK;  // Sy[0, cmax): column scratch
    // y = S_a^{-1} (C v - b_C);  dx = v - W_act y
    PARFOR(q, na) yact[q] = ws.Cv[ws.alist[q]] - ws.up[nf + ws.alist[q]];
    team.sync();
    if (na > 0) dense_solve(team, na, ws.S, yact);
    PROF_ADD(ws, PF_PR_CHOL, t_r1);
    PROF_T0(t_r2);
    dense_combine(team, n, na, ws.alist, ws.W, yact, ws.v, dxp);
    PROF_ADD(ws, PF_PR_COMB, t_r2);
    PROF_T0(t_r3);
    // one refinement round against the exact KKT (solver.py:514-522)
    block_matvec(team, N, ws.KD, ws.KU, dxp, ws.xt);
    PARFOR(j, n) {
      const bool fx = P.m.fixed_row_of_dof[j] >= 0;
      double ct = 0.0;
      const int k = j / 6, a = j % 6;
      if (a < 3) {
        const int c = ws.crow_of_node[k];
        if (c >= 0 && ws.act[c]) ct = ws.cnrm[3 * c + a] * yact[ws.alist[N + c]];
      }
      ws.xt[j] = fx ? 0.0 : -ws.g[j] - ws.xt[j] - ct;
    }
    team.sync();
    twisted_solve(team, N, ws.HD, ws.HU, ws.xt, ws.tmp, ws.w, 1, 0, ws.sh);
    team.sync();
    PROF_ADD(ws, PF_PR_REFINE, t_r3);
    PROF_T0(t_r4);
    PARFOR(q, na) {
      const int c = ws.alist[q];
      const double r2 = ws.up[nf + c] - row_dot(P, F, ws, nf + c, dxp);
      dyq[q] = row_dot(P, F, ws, nf + c, ws.w) - r2;
    }
    team.sync();
    if (na > 0) dense_solve(team, na, ws.S, dyq);
    dense_combine(team, n, na, ws.alist, ws.W, dyq, ws.w, ws.colh);
    PARFOR(j, n) dxp[j] += ws.colh[j];
    PARFOR(q, na) yact[q] += dyq[q];
    team.sync();
    PROF_ADD(ws, PF_PR_CORR, t_r4);
    PROF_T0(t_r5);
    // multipliers by row: selectors from the exact KKT, active contacts, 0 otherwise
    PARFOR(c, nc) yp[nf + c] = 0.0;
    team.sync();
    PARFOR(q, na) yp[nf + ws.alist[q]] = yact[q];
    team.sync();
    selector_multipliers(team, P, F, ws, dxp, yp);
    int neg = 0, viol = 0;
    PARFOR(c, nc) {
      int r = nf + c;
      if (ws.act[c] && yp[r] < -1e-11) neg = 1;
      if (!ws.act[c] && row_dot(P, F, ws, r, dxp) - ws.up[r] > tol_act) viol = 1;
    }
    neg = team.any(neg);
    viol = team.any(viol);
    team.sync();
    PROF_ADD(ws, PF_PR_MULT, t_r5);
    if (!neg && !viol) {
      found = true;
      break;
    }
    PARFOR(c, nc) {
      int r = nf + c;
      bool a = ws.act[c];
      if (a && yp[r] < -1e-11) a = false;
      else if (!a && row_dot(P, F, ws, r, dxp) - ws.up[r] > tol_act) a = true;
      ws.act[c] = a;
    }
    team.sync();
  }
  PROF_ADD(ws, PF_POL_ROUNDS, t_pr);
  if (!found) return ST_OK;
  // acceptance (solver.py:483-497)
  double pri = 0.0, fin = 1.0;
  PARFOR(r, F.m) {
    double ax = row_dot(P, F, ws, r, dxp);
    pri = fmax(pri, fmax(ax - ws.up[r], 0.0));
    if (r < nf) pri = fmax(pri, fabs(ax - ws.up[r]));
  }
  block_matvec(team, N, ws.KD, ws.KU, dxp, ws.tmp);
  at_y(team, P, F, ws, yp, ws.w);
  double dua = 0.0;
  parfor4(team, n, [&](int j) {
    dua = fmax(dua, fabs(ws.tmp[j] + ws.g[j] + ws.w[j]));
    if (!isfinite(dxp[j])) fin = 0.0;
  });
  pri = team.max(pri);
  dua = team.max(dua);
  fin = team.min(fin);
  if (fin > 0.0 && pri <= fmax(res.pri, P.s.eps_abs) && dua <= fmax(res.dua, P.s.eps_abs)) {
    PARFOR(j, n) ws.dx[j] = dxp[j];
    PARFOR(r, F.m) ws.yfull[r] = yp[r];
    res.pri = pri;
    res.dua = dua;
  }
  team.sync();
  return ST_OK;
}


// ---------------------------------------------------------------------------
// projected Gauss-Seidel baseline (solve_pgs, solver.py:531-665) for the
// selector-only constraint sets of the engine (every fixed row is a plain
// DOF selector, so the reference's general equality rows are empty).  The
// selector DOFs are eliminated exactly (the reduced factor with identity
// rows), W = C~ K_ff^{-1} C~^T is formed from the multi-RHS solves
// W_c = K_ff^{-1} C~_c (C~: contact rows with the selector DOFs zeroed) and
// the sweeps run on one warp (lanes over the row's entries, a fixed-order
// butterfly sum): s_i = q0_i - W_i y, y_i += s_i / W_ii, y_i >= 0.
// ---------------------------------------------------------------------------
#if defined(__CUDACC__)
// one warp's fixed-order sum (every lane gets it)
DEV double pgs_wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
#endif

// s = q0 - W y over all rows; returns the reference's residual
// max(max(s, 0), |y o s|_inf / max(1, |y|_inf)) (solver.py:574-582)
template <class Team>
DEV double pgs_residual(const Team& team, int nc, const double* W, const double* q0, const double* y) {
  double pos = 0.0, ys = 0.0, ym = 0.0;
  PARFOR(i, nc) {
    double acc = 0.0;
    for (int j = 0; j < nc; ++j) acc += W[(long)i * nc + j] * y[j];
    const double si = q0[i] - acc;
    pos = fmax(pos, si);
    ys = fmax(ys, fabs(y[i] * si));
    ym = fmax(ym, fabs(y[i]));
  }
  pos = team.max(pos);
  ys = team.max(ys);
  ym = team.max(ym);
  return fmax(pos, ys / fmax(1.0, ym));
}

// the Gauss-Seidel sweeps; returns the sweeps run, *conv the convergence flag
template <class Team>
DEV int pgs_sweeps(const Team& team, int nc, const double* W, const double* q0, const double* diag, double* y,
                   double target, int min_sweeps, int max_sweeps, bool* conv) {
  int sweeps = 0;
  *conv = false;
  for (int sweep = 1; sweep <= max_sweeps; ++sweep) {
#if defined(__CUDA_ARCH__)
    if (team.rank() < 32) {
      const int lane = team.rank();
      for (int i = 0; i < nc; ++i) {
        const double* Wi = W + (long)i * nc;
        double acc = 0.0;
        for (int j = lane; j < nc; j += 32) acc += Wi[j] * y[j];
        acc = pgs_wsum(acc);
        const double di = diag[i];
        if (di > 0.0) {  // dead rows (W_ii <= 1e-30) keep their multiplier
          double yi = y[i] + (q0[i] - acc) / di;
          if (yi < 0.0) yi = 0.0;
          __syncwarp();
          if (lane == 0) y[i] = yi;
        }
        __syncwarp();
      }
    }
#else
    for (int i = 0; i < nc; ++i) {
      const double* Wi = W + (long)i * nc;
      double acc = 0.0;
      for (int j = 0; j < nc; ++j) acc += Wi[j] * y[j];
      if (diag[i] > 0.0) {
        double yi = y[i] + (q0[i] - acc) / diag[i];
        y[i] = yi < 0.0 ? 0.0 : yi;
      }
    }
#endif
    team.sync();
    sweeps = sweep;
    if (sweep >= min_sweeps && pgs_residual(team, nc, W, q0, y) <= target) {
      *conv = true;
      break;
    }
  }
  return sweeps;
}

// not inlined: the comparison backend keeps its registers out of the hot kernel's allocation
template <class Team>
DEV int solve_pgs(const Team& team, const Problem& P, const Frame& F, Ws& ws, QpResult& res, int cmax) {
  const int N = P.m.N, n = 6 * N, nf = F.nf, nc = F.nc;
  const int* frd = P.m.fixed_row_of_dof;
  if (nc > cmax) return ST_CAPACITY;
  // K_ff with the selector DOFs as identity rows; v = the eliminated free solution
  if (reduced_factor(team, P, 0.0, ws) >= 0) return ST_LINALG;
  eliminated_rhs(team, P, F, ws, ws.xt);
  twisted_solve(team, N, ws.HD, ws.HU, ws.xt, ws.tmp, ws.v, 1, 0, ws.sh);
  team.sync();
  int sweeps = 0;
  bool conv = true;
  double* y = ws.Sy + cmax;    // multipliers
  double* diag = ws.Sy;        // W_ii (dead rows: 0)
  double* q0 = ws.Cv;
  if (nc > 0) {
    // W_c = K_ff^{-1} C~_c for every contact (as the polish does)
    parfor4(team, nc * n, [&](int t) { ws.W[t] = 0.0; });
    team.sync();
    PARFOR(c, nc) {
      const int nd = ws.cnode[c];
      for (int a = 0; a < 3; ++a) {
        const int j = 6 * nd + a;
        if (frd[j] < 0) ws.W[(long)c * n + j] = ws.cnrm[3 * c + a];
      }
    }
    team.sync();
    twisted_solve_chunks(team, N, ws.HD, ws.HU, ws.W, nc, n, ws.cnode);
    // Delassus W_pq = C~_p W_q, q0 = C~ v - b_adj (b_adj removes the selector DOFs' prescribed part)
    PARFOR(t, nc * nc) {
      const int p = t / nc, q = t - p * nc;
      const int j0 = 6 * ws.cnode[p];
      const double* nr = ws.cnrm + 3 * p;
      const double* wq = ws.W + (long)q * n + j0;
      double acc = 0.0;
      for (int a = 0; a < 3; ++a)
        if (frd[j0 + a] < 0) acc += nr[a] * wq[a];
      ws.Sf[t] = acc;
    }
    PARFOR(c, nc) {
      const int j0 = 6 * ws.cnode[c];
      const double* nr = ws.cnrm + 3 * c;
      double cv = 0.0, adj = 0.0;
      for (int a = 0; a < 3; ++a) {
        const int fr = frd[j0 + a];
        if (fr < 0) cv += nr[a] * ws.v[j0 + a];
        else adj += nr[a] * ws.up[fr];
      }
      q0[c] = cv - (ws.up[nf + c] - adj);
      y[c] = fmax(ws.warm[ws.cnode[c]], 0.0);
      ws.alist[c] = c;  // dense_combine over every contact
    }
    team.sync();
    PARFOR(c, nc) {
      const double d = ws.Sf[(long)c * nc + c];
      diag[c] = d <= 1e-30 ? 0.0 : d;
    }
    double qmax = 0.0;
    PARFOR(c, nc) qmax = fmax(qmax, fabs(q0[c]));
    qmax = team.max(qmax);
    const double target = P.s.pgs_tol * fmax(qmax, 1e-12);
    const int min_sweeps = P.s.pgs_min_sweep_factor * (nc > 1 ? nc : 1);
    int max_sweeps = P.s.max_iterations > 250 * nc ? P.s.max_iterations : 250 * nc;
    if (min_sweeps > max_sweeps) max_sweeps = min_sweeps;
    sweeps = pgs_sweeps(team, nc, ws.Sf, q0, diag, y, target, min_sweeps, max_sweeps, &conv);
    // dx = v - K_ff^{-1} C~^T y = v - sum_c y_c W_c
    dense_combine(team, n, nc, ws.alist, ws.W, y, ws.v, ws.dx);
  } else {
    PARFOR(j, n) ws.dx[j] = ws.v[j];
    team.sync();
  }
  // multipliers by row: contacts clamped, selectors from the equilibrium residual
  PARFOR(c, nc) ws.yfull[nf + c] = fmax(y[c], 0.0);
  team.sync();
  selector_multipliers(team, P, F, ws, ws.dx, ws.yfull);
  double pri = 0.0;
  PARFOR(r, F.m) {
    const double v = row_dot(P, F, ws, r, ws.dx) - ws.up[r];
    pri = fmax(pri, r < nf ? fabs(v) : fmax(v, 0.0));
  }
  block_matvec(team, N, ws.KD, ws.KU, ws.dx, ws.tmp);
  at_y(team, P, F, ws, ws.yfull, ws.w);
  double dua = 0.0;
  parfor4(team, n, [&](int j) { dua = fmax(dua, fabs(ws.tmp[j] + ws.g[j] + ws.w[j])); });
  res.pri = team.max(pri);
  res.dua = team.max(dua);
  res.iterations = sweeps;
  res.converged = conv ? 1 : 0;
  res.rho_est = -1.0;
  return conv ? ST_OK : ST_NONCONV;
}

// ---------------------------------------------------------------------------
// one QP solve (solver.py:250-385 via solve_step 717-741).  Warm start y0 is
// taken from ws.warm (by node) and ws.wfix.  On return ws.dx, ws.yfull.
// ---------------------------------------------------------------------------
template <class Team>
DEV int solve_qp(const Team& team, const Problem& P, const Frame& F, Ws& ws, double rho_in, int has_wfix,
                 QpResult& res, int cmax) {
  const Settings& S = P.s;
  const int N = P.m.N, n = 6 * N, nf = F.nf, m = F.m;
  res.polish_rounds = 0;
  if (S.backend == 1) return solve_pgs(team, P, F, ws, res, cmax);  // solve_step dispatch (solver.py:729-731)
  if (F.nc == 0) {
    PROF_T0(t_dir);
    int st = direct_solve(team, P, F, ws, res);
    PROF_ADD(ws, PF_DIRECT, t_dir);
    return st;
  }
  double gnorm = 0.0;
  PARFOR(j, n) gnorm = fmax(gnorm, fabs(ws.g[j]));
  gnorm = team.max(gnorm);
  PROF_T0(t_ruiz);
  const double cost = ruiz(team, P, F, ws);  // Ruiz cost factor
  PROF_ADD(ws, PF_RUIZ, t_ruiz);
  double rho_bar = fmin(fmax(rho_in, kRhoMin), kRhoMax);
  double rho_eq = fmin(fmax(rho_bar * kRhoEqFactor, kRhoMin), kRhoMax);
  PARFOR(r, m) {
    ws.rho[r] = r < nf ? rho_eq : rho_bar;
    ws.ls[r] = ws.e[r] * ws.lo[r];
    ws.us[r] = ws.e[r] * ws.up[r];
  }
  team.sync();
  // M = H_s + sigma I + A_s^T diag(rho) A_s  (packed diagonal blocks; HU holds H_s off-diagonal):
  // sigma on the diagonal, then the selector and contact rank-one terms row by row
  parfor4(team, 6 * N, [&](int j) {
    const int k = j / 6, r = j - 6 * k;
    ws.HD[kDiag * k + r * (r + 1) / 2 + r] += S.sigma;
  });
  team.sync();
  PARFOR(r, nf) {
    const int k = P.m.fixed_node[r], c = P.m.fixed_dof[r];
    ws.HD[kDiag * k + c * (c + 1) / 2 + c] += ws.rho[r] * ws.as[3 * r] * ws.as[3 * r];
  }
  team.sync();
  PARFOR(t, 6 * (m - nf)) {
    const int ct = t / 6, e = t - 6 * ct;  // 6 packed entries of the 3x3 block
    const int rr = e < 1 ? 0 : (e < 3 ? 1 : 2), cc = e - rr * (rr + 1) / 2;
    const int row = nf + ct, k = ws.cnode[ct];
    ws.HD[kDiag * k + e] += ws.rho[row] * ws.as[3 * row + rr] * ws.as[3 * row + cc];
  }
  team.sync();
  PROF_T0(t_fac);
  int fbad = twisted_factor(team, N, ws.HD, ws.HU, ws.scr, ws.sh);
  PROF_ADD(ws, PF_FACTOR, t_fac);
  if (fbad >= 0) return ST_LINALG;
  // initial iterate (solver.py:287-289)
  PARFOR(j, n) ws.xs[j] = 0.0;
  PARFOR(r, m) {
    double y0;
    if (r < nf) y0 = has_wfix ? ws.wfix[r] : 0.0;
    else y0 = ws.warm[ws.cnode[r - nf]];
    ws.y[r] = cost * y0 / ws.e[r];
    ws.z[r] = fmin(fmax(0.0, ws.ls[r]), ws.us[r]);
  }
  team.sync();
  const double al = S.alpha, sg = S.sigma;
  parfor4(team, n, [&](int j) { ws.rhs[j] = sg * ws.xs[j] - ws.gs[j]; });
  team.sync();
  double rho_est = rho_bar;
  int k = 0;
  bool infeas = false;
  PROF_T0(t_iter);
  for (k = 1; k <= S.max_iterations; ++k) {
    // rhs = sigma x - g_s + A_s^T (rho o (z - y / rho)); the first term is
    // written by the previous iteration's x update (or before the loop);
    // selector rows touch distinct DOFs, contact rows distinct nodes: two
    // conflict-free passes
    PARFOR(r, nf) {
      double t = ws.rho[r] * (ws.z[r] - ws.y[r] / ws.rho[r]);
      ws.rhs[6 * P.m.fixed_node[r] + P.m.fixed_dof[r]] += ws.as[3 * r] * t;
    }
    team.sync();
    PARFOR(c, m - nf) {
      int r = nf + c;
      double t = ws.rho[r] * (ws.z[r] - ws.y[r] / ws.rho[r]);
      double* rr = ws.rhs + 6 * ws.cnode[c];
      rr[0] += ws.as[3 * r] * t;
      rr[1] += ws.as[3 * r + 1] * t;
      rr[2] += ws.as[3 * r + 2] * t;
    }
    team.sync();
    PROF_T0(t_ch);
    twisted_solve(team, N, ws.HD, ws.HU, ws.rhs, ws.tmp, ws.xt, 1, 0, ws.sh, ws.sh);
    team.sync();
    PROF_ADD(ws, PF_CHAIN, t_ch);
    PARFOR(r, m) {
      double zt;
      if (r < nf) {
        zt = ws.as[3 * r] * ws.xt[6 * P.m.fixed_node[r] + P.m.fixed_dof[r]];
      } else {
        const double* xx = ws.xt + 6 * ws.cnode[r - nf];
        zt = ws.as[3 * r] * xx[0] + ws.as[3 * r + 1] * xx[1] + ws.as[3 * r + 2] * xx[2];
      }
      double z = ws.z[r], y = ws.y[r], rh = ws.rho[r];
      double zr = al * zt + (1.0 - al) * z;
      double zn = fmin(fmax(zr + y / rh, ws.ls[r]), ws.us[r]);
      ws.yprev[r] = y;
      ws.y[r] = y + rh * (zr - zn);
      ws.z[r] = zn;
    }
    team.sync();  // every row has read x~ before the x update overwrites it
    // x update fused with the next iteration's rhs = sigma x - g_s (xt aliases rhs)
    parfor4(team, n, [&](int j) {
      const double xn = al * ws.xt[j] + (1.0 - al) * ws.xs[j];
      ws.xs[j] = xn;
      ws.rhs[j] = sg * xn - ws.gs[j];
    });
    team.sync();
    if (k <= 8 || k % S.check_interval == 0 || k == S.max_iterations) {
      PROF_T0(t_chk);
      Residuals R = unscaled_residuals(team, P, F, ws, cost, gnorm);
      team.sync();
      PROF_ADD(ws, PF_CHECK, t_chk);
      if (R.pri <= S.eps_abs + S.eps_rel * R.ps && R.dua <= S.eps_abs + S.eps_rel * R.ds) break;
      if (k % S.check_interval == 0) {
        infeas = infeasible(team, P, F, ws, cost);
        team.sync();
        if (infeas) break;
        if (k == S.check_interval) {
          double ratio = (R.pri / fmax(R.ps, 1e-12)) / fmax(R.dua / fmax(R.ds, 1e-12), 1e-12);
          rho_est = fmin(fmax(rho_bar * sqrt(ratio), kRhoMin), kRhoMax);
        }
      }
    }
  }
  PROF_ADD(ws, PF_ITER, t_iter);
#if defined(__CUDA_ARCH__) && defined(ACCFEM_PROFILE)
  if (ws.prof && team.rank() == 0) ws.prof[PF_ITERS] += (k > S.max_iterations ? S.max_iterations : k);
#endif
  if (k > S.max_iterations) k = S.max_iterations;
  if (infeas) return ST_INFEASIBLE;
  Residuals R = unscaled_residuals(team, P, F, ws, cost, gnorm);
  PARFOR(j, n) ws.dx[j] = ws.tmp[j];  // tmp holds d o xs
  team.sync();
  res.pri = R.pri;
  res.dua = R.dua;
  res.iterations = k;
  res.converged = (R.pri <= S.eps_abs + S.eps_rel * R.ps && R.dua <= S.eps_abs + S.eps_rel * R.ds) ? 1 : 0;
  res.rho_est = (S.adaptive_rho && k >= 3 * S.check_interval) ? rho_est : -1.0;
  if (S.polish && res.converged) {
    PROF_T0(t_pol);
    int st = polish(team, P, F, ws, res, cmax);
    PROF_ADD(ws, PF_POLISH, t_pol);
    if (st != ST_OK) return st;
  }
  return res.converged ? ST_OK : ST_NONCONV;
}

}  // namespace accfem
