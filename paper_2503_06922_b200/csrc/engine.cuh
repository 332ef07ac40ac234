// Engine.step / Engine.run_static on one team (engine.py:136-283).
#pragma once
#include "solve.cuh"

namespace accfem {

// per-launch batch I/O (device pointers; see include/accfem.h for meaning)
struct BatchDev {
  int S;
  const double* x0;          // S x 6N
  const double* tensions;    // S x n_cables or null
  const double* applied;     // S x 6N or null
  const double* insertion;   // S or null
  const double* warm_y_in;   // S x N or null
  const double* warm_fix_in; // S x nf or null
  const double* rho_in;      // S or null
  double* coords;            // S x 6N
  int* status;               // S
  int* frames;               // S
  int* converged;            // S
  double* residual;          // S
  int* n_contacts;           // S  (last frame)
  int* c_node;               // S x N
  int* c_tri;                // S x N
  double* c_gap;             // S x N
  double* c_y;               // S x N     limited multipliers
  double* c_force;           // S x N x 3 world force on the robot (-y n)
  double* c_normal;          // S x N x 3
  double* c_point;           // S x N x 3
  double* warm_y_out;        // S x N or null
  double* warm_fix_out;      // S x nf or null
  double* rho_out;           // S or null
  int trace_cap;             // frames recorded per scenario
  double* trace_stats;       // S x cap x kTraceStats or null
  double* trace_coords;      // S x cap x 6N or null
  int* trace_c_node;         // S x cap x N or null (with the fields below)
  int* trace_c_tri;
  double* trace_c_gap;
  double* trace_c_force;     // S x cap x N x 3
  double* trace_c_point;     // S x cap x N x 3
  int max_frames;
  int stop_on_tol;           // 1: run_static semantics; 0: exactly max_frames frames (step mode)
  double tol;
  int fail_on_limit;         // 1: exhausting max_frames is ST_ENGINE_MAX_FRAMES
  int cmax_polish;
  int hot_rows;              // lean hot set: row-state capacity in shared memory (0: full layout)
  long long* team_stats;     // 4 per team: scenarios, busy ns, start ns, end ns (or null)
  int team_stats_cap;
  int* work_counter;         // dynamic scenario queue
  unsigned long long* prof;  // per-team phase counters (profile builds)
};

constexpr int kTraceStats = 14;  // dx_norm, act_scale, max_pen, compl_worst, residual, iterations,
                                 // n_c, converged, retried, compl_ok, pri, dua, pairs, polish_rounds

// one frame.  x (6N) is advanced in place.  Returns a status.
template <class Team>
DEV int frame_step(const Team& team, const Problem& P, const BatchDev& B, int s, double* x, double insertion,
                   const double* tensions, const double* applied, Ws& ws, double& rho, int& has_wfix,
                   bool& pending, double& resid_prev, FrameStats& st, Frame& F) {
  const ModelDev& M = P.m;
  const int N = M.N, n = 6 * N;
  PROF_T0(t_el);
  int bad = element_pass(team, P, x, ws, true);
  PROF_ADD(ws, PF_ELEMENT, t_el);
  if (bad) return ST_DEGENERATE;
  if (pending) {
    double acc = 0.0;
    PARFOR(j, n) {
      double v = ws.fint[j] + ws.rres[j];
      acc += v * v;
    }
    resid_prev = sqrt(team.sum(acc));
    pending = false;
  }
  F.nf = M.n_fixed;
  PROF_T0(t_det);
  int pairs = 0;
  F.nc = P.mesh.T > 0 ? detect_pass(team, P, x, ws, &pairs) : 0;
  PROF_ADD(ws, PF_DETECT, t_det);
  if (P.mesh.T == 0) {
    PARFOR(k, N) ws.crow_of_node[k] = -1;
    team.sync();
  }
  F.m = F.nf + F.nc;
  ws_rows(ws, F.m);
  external_force(team, P, tensions, applied, ws);
  build_rows(team, P, x, insertion, 1.0, F, ws);
  QpResult res;
  int retried = 0;
  int code = solve_qp(team, P, F, ws, rho, has_wfix, res, B.cmax_polish);
  int rounds = res.polish_rounds;
  if (code == ST_NONCONV) {
    retried = 1;
    if (P.s.adaptive_rho && res.rho_est >= 0.0) rho = res.rho_est;
    build_rows(team, P, x, insertion * 0.5, 1.0, F, ws);
    code = solve_qp(team, P, F, ws, rho, has_wfix, res, B.cmax_polish);
    rounds += res.polish_rounds;
    if (code == ST_NONCONV) return ST_ENGINE_SOLVER;
  }
  if (code != ST_OK) return code;
  const int nf = F.nf, nc = F.nc;
  PROF_T0(t_post);
  // complementarity report on the unlimited result (solver.py:781-800)
  double mult_v = 0.0, gap_v = 0.0, prod_v = 0.0, eq_v = 0.0, ymax = 0.0, axmax = 0.0, nrm2 = 0.0;
  PARFOR(r, F.m) {
    double ax = row_dot(P, F, ws, r, ws.dx);
    double v = ax - ws.up[r];
    if (r < nf) {
      eq_v = fmax(eq_v, fabs(v));
    } else {
      double yc = fmax(ws.yfull[r], 0.0);
      mult_v = fmax(mult_v, -yc);
      gap_v = fmax(gap_v, fmax(v, 0.0));
      prod_v = fmax(prod_v, fabs(yc * v));
      ymax = fmax(ymax, fabs(yc));
      axmax = fmax(axmax, fabs(ax));
    }
  }
  PARFOR(j, n) nrm2 += ws.dx[j] * ws.dx[j];
  mult_v = team.max(mult_v);
  gap_v = team.max(gap_v);
  prod_v = team.max(prod_v);
  eq_v = team.max(eq_v);
  double scale = fmax(1.0, fmax(team.max(ymax), nc ? team.max(axmax) : 0.0));
  const double ctol = 1e-6;
  st.compl_ok = (mult_v <= ctol && gap_v <= ctol && prod_v <= ctol * scale && eq_v <= ctol) ? 1 : 0;
  st.compl_worst = fmax(fmax(gap_v, mult_v), fmax(prod_v, eq_v));
  // step limit (solver.py:803-823)
  double nrm = sqrt(team.sum(nrm2));
  double fac = (nrm <= P.s.beta0 || nrm == 0.0) ? 1.0 : P.s.beta0 / nrm;
  team.sync();
  // warm state from the unlimited result (engine.py:248-255)
  PARFOR(k, N) ws.warm[k] = 0.0;
  team.sync();
  PARFOR(c, nc) ws.warm[ws.cnode[c]] = fmax(ws.yfull[nf + c], 0.0);
  PARFOR(r, nf) ws.wfix[r] = ws.yfull[r];
  has_wfix = 1;
  if (P.s.adaptive_rho && res.rho_est >= 0.0 && (res.rho_est > 5.0 * rho || res.rho_est < rho / 5.0))
    rho = res.rho_est;
  // penetration before the step (engine.py:208)
  double pen0 = 0.0, pen1 = 0.0, dxn2 = 0.0;
  PARFOR(c, nc) pen0 = fmax(pen0, -ws.cgap[c]);
  // limited dx, end-of-frame plane gaps, advance (engine.py:195, 209-213, 291-297)
  PARFOR(j, n) {
    double v = ws.dx[j] * fac;
    ws.dx[j] = v;
    dxn2 += v * v;
  }
  team.sync();
  PARFOR(c, nc) pen1 = fmax(pen1, -(ws.up[nf + c] - row_dot(P, F, ws, nf + c, ws.dx)));
  PARFOR(k, N) {
    double* xk = x + 6 * k;
    const double* d = ws.dx + 6 * k;
    xk[0] += d[0];
    xk[1] += d[1];
    xk[2] += d[2];
    double out[3];
    rot_compose(d + 3, xk + 3, out);
    xk[3] = out[0];
    xk[4] = out[1];
    xk[5] = out[2];
  }
  // limited multipliers; deferred residual pieces A^T y - F_a (engine.py:199-203)
  PARFOR(r, F.m) {
    double y = r < nf ? ws.yfull[r] : fmax(ws.yfull[r], 0.0);
    ws.yp[r] = y * fac;
  }
  team.sync();
  at_y(team, P, F, ws, ws.yp, ws.rres);
  parfor4(team, n, [&](int j) { ws.rres[j] -= ws.fa[j]; });
  team.sync();
  pending = true;
  PROF_ADD(ws, PF_POST, t_post);
  st.dx_norm = sqrt(team.sum(dxn2));
  st.actuation_scale = fac;
  st.max_penetration = fmax(fmax(team.max(pen0), 0.0), fmax(team.max(pen1), 0.0));
  st.iterations = res.iterations;
  st.n_c = nc;
  st.converged = res.converged;
  st.retried = retried;
  st.residual = 0.0;
  st.pri = res.pri;
  st.dua = res.dua;
  st.pairs = pairs;
  st.polish_rounds = rounds;
  (void)B;
  (void)s;
  return ST_OK;
}

template <class Team>
DEV void write_contacts(const Team& team, const Problem& P, const Frame& F, const Ws& ws, int* node, int* tri,
                        double* gap, double* yv, double* force, double* normal, double* point) {
  PARFOR(c, F.nc) {
    double y = ws.yp[F.nf + c];
    if (node) node[c] = ws.cnode[c];
    if (tri) tri[c] = ws.ctri[c];
    if (gap) gap[c] = ws.cgap[c];
    if (yv) yv[c] = y;
    for (int a = 0; a < 3; ++a) {
      double nr = ws.cnrm[3 * c + a];
      if (force) force[3 * c + a] = -y * nr;
      if (normal) normal[3 * c + a] = nr;
      if (point) point[3 * c + a] = ws.cpp[3 * c + a];
    }
  }
}

template <class Team>
DEV void write_trace(const Team& team, const BatchDev& B, int s, int f, const FrameStats& st) {
  if (!B.trace_stats || f >= B.trace_cap) return;
  if (team.rank() == 0) {
    double* t = B.trace_stats + ((long)s * B.trace_cap + f) * kTraceStats;
    t[0] = st.dx_norm;
    t[1] = st.actuation_scale;
    t[2] = st.max_penetration;
    t[3] = st.compl_worst;
    t[4] = st.residual;
    t[5] = st.iterations;
    t[6] = st.n_c;
    t[7] = st.converged;
    t[8] = st.retried;
    t[9] = st.compl_ok;
    t[10] = st.pri;
    t[11] = st.dua;
    t[12] = st.pairs;
    t[13] = st.polish_rounds;
  }
}

// run_static (or a fixed number of frames) for scenario s
template <class Team>
DEV void run_scenario(const Team& team, const Problem& P, const BatchDev& B, int s, Ws& ws) {
  const ModelDev& M = P.m;
  const int N = M.N, n = 6 * N;
  double* x = B.coords + (long)s * n;
  PARFOR(j, n) x[j] = B.x0[(long)s * n + j];
  PARFOR(k, N) ws.warm[k] = B.warm_y_in ? B.warm_y_in[(long)s * N + k] : 0.0;
  PARFOR(r, M.n_fixed) ws.wfix[r] = B.warm_fix_in ? B.warm_fix_in[(long)s * M.n_fixed + r] : 0.0;
  team.sync();
  int has_wfix = B.warm_fix_in ? 1 : 0;
  double rho = B.rho_in ? B.rho_in[s] : P.s.rho;
  const double* tensions = B.tensions ? B.tensions + (long)s * M.n_cables : nullptr;
  const double* applied = B.applied ? B.applied + (long)s * n : nullptr;
  double insertion = B.insertion ? B.insertion[s] : 0.0;
  bool pending = false, have_last = false;
  int status = ST_OK, f = 0, conv = 0;
  FrameStats last;
  last.residual = 0.0;
  Frame F;
  F.nf = M.n_fixed;
  F.nc = 0;
  F.m = F.nf;
  PROF_T0(t_tot);
  for (f = 0; f < B.max_frames; ++f) {
    FrameStats cur;
    double resid_prev = 0.0;
    status = frame_step(team, P, B, s, x, insertion, tensions, applied, ws, rho, has_wfix, pending, resid_prev,
                        cur, F);
    if (have_last) {
      last.residual = resid_prev;  // the previous frame's residual needs F_int at this frame's start
      write_trace(team, B, s, f - 1, last);
    }
    if (status != ST_OK) break;
    if (B.trace_coords && f < B.trace_cap) {
      double* tc = B.trace_coords + ((long)s * B.trace_cap + f) * n;
      PARFOR(j, n) tc[j] = x[j];
    }
    if (B.trace_c_node && f < B.trace_cap) {
      long o = ((long)s * B.trace_cap + f) * N;
      write_contacts(team, P, F, ws, B.trace_c_node + o, B.trace_c_tri + o, B.trace_c_gap + o, nullptr,
                     B.trace_c_force + 3 * o, nullptr, B.trace_c_point + 3 * o);
      PARFOR(c, N - F.nc) B.trace_c_node[o + F.nc + c] = -1;
    }
    last = cur;
    have_last = true;
    if (B.stop_on_tol && cur.dx_norm <= B.tol) {
      conv = 1;
      ++f;
      break;
    }
  }
  int frames_done = f;
  PROF_ADD(ws, PF_TOTAL, t_tot);
#if defined(__CUDA_ARCH__) && defined(ACCFEM_PROFILE)
  if (ws.prof && team.rank() == 0) ws.prof[PF_FRAMES] += frames_done;
#endif
  if (status == ST_OK) {
    // last frame: contacts, and its residual from one more F_int pass
    long o = (long)s * N;
    write_contacts(team, P, F, ws, B.c_node + o, B.c_tri + o, B.c_gap + o, B.c_y + o, B.c_force + 3 * o,
                   B.c_normal + 3 * o, B.c_point + 3 * o);
    if (have_last) {
      int bad = element_pass(team, P, x, ws, false);
      if (!bad) {
        double acc = 0.0;
        PARFOR(j, n) {
          double v = ws.fint[j] + ws.rres[j];
          acc += v * v;
        }
        last.residual = sqrt(team.sum(acc));
      }
      write_trace(team, B, s, frames_done - 1, last);
    }
    if (!conv && B.stop_on_tol && B.fail_on_limit) status = ST_ENGINE_MAX_FRAMES;
  }
  if (B.warm_y_out) PARFOR(k, N) B.warm_y_out[(long)s * N + k] = ws.warm[k];
  if (B.warm_fix_out) PARFOR(r, M.n_fixed) B.warm_fix_out[(long)s * M.n_fixed + r] = ws.wfix[r];
  if (team.rank() == 0) {
    B.status[s] = status;
    B.frames[s] = frames_done;
    B.converged[s] = conv;
    B.residual[s] = last.residual;
    B.n_contacts[s] = status == ST_OK ? F.nc : 0;
    if (B.rho_out) B.rho_out[s] = rho;
  }
  team.sync();
}

}  // namespace accfem
