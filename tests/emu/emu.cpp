// TEST-ONLY serial emulation of the device solver.
//
// Compiles the exact team-generic source of paper_2503_06922_b200/csrc with
// g++ and runs every "team" on one CPU thread (TeamSerial), so the CPU test
// suite can check the device algorithm (block Cholesky reduction, exact
// selector elimination, grid broad phase, frame state machine) against the
// oracle without a GPU.  It is never loaded by the package: the product
// path is the sm_100a library, and it fails loudly when that is missing.
#include <vector>
#include <string>

#include "../../paper_2503_06922_b200/csrc/engine.cuh"
#include "../../paper_2503_06922_b200/csrc/host_build.hpp"

using namespace accfem;

struct EmuHandle {
  Problem P;
  int cmax = 0, n_cables = 0, n_fixed = 0, N = 0;
  std::vector<double> rest, rest_dir, rest_len, rest_frames, offsets, qa, qb, fixed_inc;
  std::vector<int> fixed_node, fixed_dof, frd;
  accfem_host::HostMesh mesh;
  std::vector<double> ws;
  std::string err;
};

extern "C" const char* emu_last_error(EmuHandle* h) { return h ? h->err.c_str() : ""; }

extern "C" EmuHandle* emu_create(const accfem_model_desc* md, const accfem_mesh_desc* mesh, const accfem_settings* sd) {
  EmuHandle* h = new EmuHandle();
  std::string v = accfem_host::validate(md, sd);
  if (!v.empty()) { h->err = v; return h; }
  const int N = md->node_count, E = N - 1;
  h->N = N;
  Problem& P = h->P;
  memset(&P, 0, sizeof(P));
  Settings& S = P.s;
  S.eps_abs = sd->eps_abs; S.eps_rel = sd->eps_rel; S.rho = sd->rho; S.sigma = sd->sigma;
  S.alpha = sd->alpha; S.beta0 = sd->beta0; S.margin = sd->margin;
  S.radius = std::max(sd->margin + sd->beta0, sd->margin);
  S.max_iterations = sd->max_iterations; S.check_interval = sd->check_interval;
  S.adaptive_rho = sd->adaptive_rho; S.scaling_iterations = sd->scaling_iterations; S.polish = sd->polish;
  S.backend = sd->backend; S.pgs_tol = sd->pgs_tol; S.pgs_min_sweep_factor = sd->pgs_min_sweep_factor;
  h->cmax = sd->polish_capacity > 0 ? sd->polish_capacity : std::min(N, 256);
  ModelDev& M = P.m;
  M.N = N; M.l0 = md->element_rest_length;
  accfem_host::local_stiffness(md, M.kl);
  M.n_cables = h->n_cables = sd->n_cables;
  for (int j = 0; j < sd->n_cables; ++j)
    for (int a = 0; a < 3; ++a) {
      M.cable_off[3 * j + a] = sd->cable_offset[3 * j + a];
      M.cable_dir[3 * j + a] = sd->cable_direction[3 * j + a];
    }
  const double* r = md->rest_coords;
  double ax[3] = {r[6] - r[0], r[7] - r[1], r[8] - r[2]};
  double nrm = sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
  for (int a = 0; a < 3; ++a) M.axis[a] = ax[a] / nrm;
  M.has_uniform = sd->has_uniform_load;
  for (int a = 0; a < 3; ++a) M.uniform[a] = sd->uniform_load[a];
  M.n_fixed = h->n_fixed = sd->n_fixed;
  h->fixed_node.assign(sd->fixed_node, sd->fixed_node + sd->n_fixed);
  h->fixed_dof.assign(sd->fixed_dof, sd->fixed_dof + sd->n_fixed);
  h->fixed_inc.assign(sd->fixed_increment, sd->fixed_increment + sd->n_fixed);
  h->frd.assign(6L * N, -1);
  for (int q = 0; q < sd->n_fixed; ++q) h->frd[6 * sd->fixed_node[q] + sd->fixed_dof[q]] = q;
  h->rest.assign(md->rest_coords, md->rest_coords + 6L * N);
  h->rest_dir.resize(9L * N); h->rest_len.resize(E); h->rest_frames.resize(9L * E);
  h->offsets.resize(9L * E); h->qa.resize(9L * E); h->qb.resize(9L * E);
  int bad = 0;
  model_setup(TeamSerial{}, N, h->rest.data(), h->rest_dir.data(), h->rest_len.data(), h->rest_frames.data(),
              h->offsets.data(), h->qa.data(), h->qb.data(), &bad);
  if (bad) { h->err = "rest configuration has coincident nodes"; return h; }
  std::string me = accfem_host::build_mesh(mesh, S.radius, h->mesh);
  if (!me.empty()) { h->err = me; return h; }
  M.rest_dir = h->rest_dir.data(); M.rest_len = h->rest_len.data(); M.rest_frames = h->rest_frames.data();
  M.offsets = h->offsets.data(); M.qa = h->qa.data(); M.qb = h->qb.data();
  M.fixed_node = h->fixed_node.data(); M.fixed_dof = h->fixed_dof.data(); M.fixed_inc = h->fixed_inc.data();
  M.fixed_row_of_dof = h->frd.data();
  MeshDev& G = P.mesh;
  G.T = h->mesh.T;
  if (G.T) {
    G.corners = h->mesh.corners.data(); G.normals = h->mesh.normals.data();
    G.lo = h->mesh.lo.data(); G.hi = h->mesh.hi.data();
    G.cell_start = h->mesh.cell_start.data();
    G.cell_tris = h->mesh.cell_tris.data();
    for (int a = 0; a < 3; ++a) { G.origin[a] = h->mesh.origin[a]; G.dims[a] = h->mesh.dims[a]; }
    G.inv_h = h->mesh.inv_h;
  }
  h->ws.assign(ws_doubles(N, sd->n_fixed, h->cmax) + 64, 0.0);
  return h;
}

extern "C" void emu_destroy(EmuHandle* h) { delete h; }

// the host grid build (checker for the device build, accfem_grid_download)
extern "C" int emu_grid_shape(EmuHandle* h, int32_t* dims, int64_t* n_cells, int64_t* n_entries) {
  for (int a = 0; a < 3; ++a) dims[a] = h->mesh.T ? h->mesh.dims[a] : 0;
  *n_cells = h->mesh.T ? h->mesh.ncell : 0;
  *n_entries = h->mesh.T ? h->mesh.cell_start.back() : 0;
  return 0;
}

extern "C" int emu_grid_download(EmuHandle* h, int32_t* cell_start, int32_t* cell_tris) {
  if (!h->mesh.T) return 0;
  memcpy(cell_start, h->mesh.cell_start.data(), h->mesh.cell_start.size() * sizeof(int32_t));
  memcpy(cell_tris, h->mesh.cell_tris.data(), h->mesh.cell_start.back() * sizeof(int32_t));
  return 0;
}

extern "C" int emu_element_pass(EmuHandle* h, int S, const double* x, double* fint, double* kd, double* ku, int* bad) {
  const int N = h->N, n = 6 * N, E = N - 1;
  Ws ws = ws_carve(h->ws.data(), nullptr, N, h->n_fixed, h->cmax);
  for (int s = 0; s < S; ++s) {
    int b = element_pass(TeamSerial{}, h->P, x + (long)s * n, ws, true);
    bad[s] = b;
    if (b) continue;
    memcpy(fint + (long)s * n, ws.fint, n * 8);
    memcpy(kd + (long)s * 36 * N, ws.KD, 36L * N * 8);
    memcpy(ku + (long)s * 36 * E, ws.KU, 36L * E * 8);
  }
  return 0;
}

extern "C" int emu_detect(EmuHandle* h, int S, const double* x, int* tri, double* gap, double* point) {
  const int N = h->N, n = 6 * N;
  Ws ws = ws_carve(h->ws.data(), nullptr, N, h->n_fixed, h->cmax);
  for (int s = 0; s < S; ++s) {
    int nc = detect_pass(TeamSerial{}, h->P, x + (long)s * n, ws);
    for (int k = 0; k < N; ++k) tri[(long)s * N + k] = -1;
    for (int c = 0; c < nc; ++c) {
      int k = ws.cnode[c];
      tri[(long)s * N + k] = ws.ctri[c];
      gap[(long)s * N + k] = ws.cgap[c];
      for (int a = 0; a < 3; ++a) point[((long)s * N + k) * 3 + a] = ws.cpp[3 * c + a];
    }
  }
  return 0;
}

extern "C" int emu_solve_batch(EmuHandle* h, const accfem_batch* io) {
  BatchDev B;
  memset(&B, 0, sizeof(B));
  B.S = io->S;
  B.x0 = io->x0; B.tensions = h->n_cables ? io->tensions : nullptr; B.applied = io->applied;
  B.insertion = io->insertion; B.warm_y_in = io->warm_y_in; B.warm_fix_in = io->warm_fixed_in; B.rho_in = io->rho_in;
  B.coords = io->coords; B.status = io->status; B.frames = io->frames; B.converged = io->converged;
  B.residual = io->residual; B.n_contacts = io->n_contacts; B.c_node = io->contact_node;
  B.c_tri = io->contact_triangle; B.c_gap = io->contact_gap; B.c_y = io->contact_multiplier;
  B.c_force = io->contact_force; B.c_normal = io->contact_normal; B.c_point = io->contact_point;
  B.warm_y_out = io->warm_y_out; B.warm_fix_out = io->warm_fixed_out; B.rho_out = io->rho_out;
  B.trace_cap = io->trace_cap; B.trace_stats = io->trace_stats; B.trace_coords = io->trace_coords;
  B.trace_c_node = io->trace_contact_node; B.trace_c_tri = io->trace_contact_triangle;
  B.trace_c_gap = io->trace_contact_gap; B.trace_c_force = io->trace_contact_force;
  B.trace_c_point = io->trace_contact_point;
  B.max_frames = io->max_frames; B.stop_on_tol = io->stop_on_tol; B.tol = io->tol;
  B.fail_on_limit = io->fail_on_limit; B.cmax_polish = h->cmax;
  Ws ws = ws_carve(h->ws.data(), nullptr, h->N, h->n_fixed, h->cmax);
  for (int s = 0; s < io->S; ++s) run_scenario(TeamSerial{}, h->P, B, s, ws);
  return 0;
}
