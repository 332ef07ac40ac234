// B200 (sm_100a) device library behind include/accfem.h.
//
// Kernels (all FP64; the solve kernels are persistent over a dynamic scenario
// queue, one CTA team = one scenario):
//   k_model_setup     per-model constants (once per handle)
//   k_solve<NW, CR>   run_static / step for a batch: element pass, detection,
//                     assembly, Ruiz, block-tridiagonal factorisation, ADMM or
//                     PGS, polish, update -- 2-warp teams (throughput), 4-warp
//                     teams, or 8-warp teams with cyclic reduction (latency)
//   k_element_pass    unit entry point: F_int + block-tridiagonal K
//   k_detect          unit entry point: per-node contact winner
//   k_grid_*          broad-phase grid build over the lumen mesh (grid.cuh; the
//                     cell lists are sorted with cub's segmented sort)
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/accfem.h"
#include "grid.cuh"
#include "host_build.hpp"
#include "ksolve.cuh"

using namespace accfem;

namespace {

constexpr int kWarpsPerBlock = 4;
// k_solve team widths: throughput mode (three 2-warp teams per SM share it)
// and latency mode (batches that leave SMs idle get 4-warp teams, whose
// parallel phases run twice as wide; measured p50 -15% at batch 1)
constexpr int kTeamWarps = 2;
constexpr int kLatencyTeamWarps = 4;
// latency mode with cyclic reduction: one CTA of kCrTeamWarps warps per scenario (ksolve_cr.cu)
constexpr int kCrTeamWarps = 8;

__global__ void k_model_setup(int N, const double* rest, double* rest_dir, double* rest_len, double* rest_frames,
                              double* offsets, double* qa, double* qb, int* bad) {
  TeamWarp team{(int)(threadIdx.x & 31)};
  if (threadIdx.x >= 32) return;
  model_setup(team, N, rest, rest_dir, rest_len, rest_frames, offsets, qa, qb, bad);
}

// k_solve<NW> lives in ksolve.cuh, one translation unit per team width
// (ksolve_<NW>.cu, compiled in parallel); this table reaches them.
static const KSolveEntry* solve_entry(int nw, bool cr = false) {
  static const KSolveEntry table[] = {ksolve_entry_2(), ksolve_entry_4(), ksolve_entry_cr()};
  for (const KSolveEntry& e : table)
    if (e.nw == nw && e.cr == cr) return &e;
  return nullptr;
}

__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    k_element_pass(Problem P, int S, const double* x, double* fint, double* kd, double* ku, double* frames, int* bad,
                   double* ws_base, long ws_stride, int* counter) {
  TeamWarp team{(int)(threadIdx.x & 31)};
  const long wid = (long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  Ws ws = ws_carve(ws_base + wid * ws_stride, nullptr, P.m.N, P.m.n_fixed, 1);
  const int N = P.m.N, n = 6 * N, E = N - 1;
  while (true) {
    int s = 0;
    if (team.lane == 0) s = atomicAdd(counter, 1);
    s = __shfl_sync(0xffffffffu, s, 0);
    if (s >= S) break;
    int b = element_pass(team, P, x + (long)s * n, ws, true);
    if (team.lane == 0 && bad) bad[s] = b;
    if (b) continue;
    for (int i = team.lane; i < n; i += 32) fint[(long)s * n + i] = ws.fint[i];
    if (kd)
      for (int i = team.lane; i < 36 * N; i += 32) kd[(long)s * 36 * N + i] = ws.KD[i];
    if (ku)
      for (int i = team.lane; i < 36 * E; i += 32) ku[(long)s * 36 * E + i] = ws.KU[i];
    if (frames)
      for (int i = team.lane; i < 9 * E; i += 32) frames[(long)s * 9 * E + i] = ws.frames[i];
    __syncwarp();
  }
}

__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    k_detect(Problem P, int S, const double* x, int* tri, double* gap, double* point, double* ws_base, long ws_stride,
             int* counter) {
  TeamWarp team{(int)(threadIdx.x & 31)};
  const long wid = (long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  Ws ws = ws_carve(ws_base + wid * ws_stride, nullptr, P.m.N, P.m.n_fixed, 1);
  const int N = P.m.N, n = 6 * N;
  while (true) {
    int s = 0;
    if (team.lane == 0) s = atomicAdd(counter, 1);
    s = __shfl_sync(0xffffffffu, s, 0);
    if (s >= S) break;
    int nc = detect_pass(team, P, x + (long)s * n, ws);
    // scatter back to node order: -1 for nodes without a contact
    for (int k = team.lane; k < N; k += 32) tri[(long)s * N + k] = -1;
    __syncwarp();
    for (int c = team.lane; c < nc; c += 32) {
      int k = ws.cnode[c];
      tri[(long)s * N + k] = ws.ctri[c];
      gap[(long)s * N + k] = ws.cgap[c];
      for (int a = 0; a < 3; ++a) point[((long)s * N + k) * 3 + a] = ws.cpp[3 * c + a];
    }
    __syncwarp();
  }
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  cudaError_t alloc(size_t count) {
    if (count <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess) n = count;
    return e;
  }
  cudaError_t upload(const T* h, size_t count) {
    cudaError_t e = alloc(count);
    if (e != cudaSuccess) return e;
    if (count) return cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice);
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

}  // namespace

struct accfem_handle {
  int device = 0;
  int sms = 0;
  int blocks_per_sm = 0;     // k_solve occupancy, throughput mode
  int solve_warps = 0;       // warps per k_solve block, throughput mode
  int lat_blocks_per_sm = 0; // the same for latency mode
  int lat_warps = 0;
  long hot_stride = 0;       // doubles of shared memory per warp (0: global mode)
  int cr_blocks_per_sm = 0;  // the cyclic-reduction latency kernel (0: disabled)
  long cr_hot_stride = 0;
  int force_mode = 0;        // test hook ACCFEM_MODE: 1 cr, 2 4-warp teams, 3 2-warp teams (0: by batch size)
  int hot_rows = 0;          // team kernels: lean hot set with this row capacity (0: full layout)
  int last_teams = 0;        // CTAs of the last solve launch
  int launches = 0;
  std::string err;
  Problem P;
  int n_cables = 0, n_fixed = 0, N = 0, cmax = 0;
  DevBuf<double> rest, rest_dir, rest_len, rest_frames, offsets, qa, qb, fixed_inc;
  DevBuf<int> fixed_node, fixed_dof, fixed_row_of_dof, bad;
  DevBuf<double> corners, normals, lo, hi;
  DevBuf<int> cell_start, cell_tris;
  long grid_cells = 0, grid_entries = 0;
  int grid_dims[3] = {0, 0, 0};
  DevBuf<double> ws;
  DevBuf<int> counter;
  long ws_stride = 0;
  long ws_teams = 0;         // per-team slabs preallocated at create
  int max_batch = 0;         // host-path staging capacity (scenarios per chunk)
  long trace_slots = 0;      // host-path trace staging (scenario-frames) for coords / contacts
  long stat_slots = 0;       // host-path trace staging (scenario-frames) for per-frame stats
  // ordering: every launch of this handle shares the work counter and the
  // workspace, so calls on different streams are chained through `done`
  cudaEvent_t done = nullptr;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  // host-path staging (accfem_solve_batch_host)
  DevBuf<double> h_x0, h_ten, h_app, h_ins, h_wy, h_wf, h_rho, o_coords, o_res, o_cd, o_wy, o_wf, o_rho, o_tr;
  DevBuf<int> o_ints;
  unsigned long long* prof = nullptr;  // development: per-team phase counters
};

// development hook (not part of include/accfem.h): per-team phase clock
// counters, PF_COUNT per resident team, in builds with -DACCFEM_PROFILE
extern "C" int accfem_dev_set_profile(accfem_handle* h, void* counters) {
  if (!h) return ACCFEM_E_ARG;
  h->prof = (unsigned long long*)counters;
#if defined(ACCFEM_PROFILE)
  return 0;
#else
  return 1;
#endif
}

static int fail(accfem_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}

#define CUDA_OK(h, expr)                                                                  \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) return fail((h), ACCFEM_E_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

static thread_local std::string g_create_error;

extern "C" int accfem_version(void) { return 1; }

extern "C" const char* accfem_last_error(const accfem_handle* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

// cell lists of the broad-phase grid on the device (grid.cuh); the host has
// sized the grid (hm.dims/h/rr) and uploaded the triangle AABBs
static cudaError_t build_grid(accfem_handle* h, const accfem_host::HostMesh& hm) {
  GridBuild g;
  g.lo = h->lo.p;
  g.hi = h->hi.p;
  g.T = hm.T;
  for (int a = 0; a < 3; ++a) {
    g.dims[a] = hm.dims[a];
    g.origin[a] = hm.origin[a];
    h->grid_dims[a] = hm.dims[a];
  }
  g.h = hm.h;
  g.inv_h = hm.inv_h;
  g.rr = hm.rr;
  const long ncell = hm.ncell;
  h->grid_cells = ncell;
  cudaError_t e;
#define GRID_OK(expr) \
  if ((e = (expr)) != cudaSuccess) return e
  DevBuf<int> count;  // released by its destructor on every path
  GRID_OK(count.alloc(ncell + 1));
  GRID_OK(h->cell_start.alloc(ncell + 1));
  GRID_OK(cudaMemset(count.p, 0, (ncell + 1) * sizeof(int)));
  const int tb = 128, tblocks = (int)std::min<long>((hm.T + 3) / 4, 148L * 16);  // 4 warps, 1 triangle each
  k_grid_count<<<tblocks, tb>>>(g, count.p);
  GRID_OK(cudaGetLastError());
  size_t tmp_bytes = 0;
  GRID_OK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, count.p, h->cell_start.p, (int)(ncell + 1)));
  DevBuf<char> tmp;
  GRID_OK(tmp.alloc(tmp_bytes));
  GRID_OK(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, count.p, h->cell_start.p, (int)(ncell + 1)));
  int entries = 0;
  GRID_OK(cudaMemcpy(&entries, h->cell_start.p + ncell, sizeof(int), cudaMemcpyDeviceToHost));
  h->grid_entries = entries;
  GRID_OK(h->cell_tris.alloc(std::max(entries, 1)));
  DevBuf<int> unsorted;
  GRID_OK(unsorted.alloc(std::max(entries, 1)));
  GRID_OK(cudaMemcpy(count.p, h->cell_start.p, (ncell + 1) * sizeof(int), cudaMemcpyDeviceToDevice));
  k_grid_fill<<<tblocks, tb>>>(g, count.p, unsorted.p);
  GRID_OK(cudaGetLastError());
  // order every cell's list by triangle id (the host build's order): a segmented
  // radix sort over the cell ranges (a per-cell rank sort is quadratic in the
  // list length, ~500 entries per cell on dense meshes)
  {
    size_t sort_bytes = 0;
    GRID_OK(cub::DeviceSegmentedSort::SortKeys(nullptr, sort_bytes, unsorted.p, h->cell_tris.p, entries, (int)ncell,
                                               h->cell_start.p, h->cell_start.p + 1));
    DevBuf<char> sort_tmp;
    GRID_OK(sort_tmp.alloc(std::max<size_t>(sort_bytes, 1)));
    GRID_OK(cub::DeviceSegmentedSort::SortKeys(sort_tmp.p, sort_bytes, unsorted.p, h->cell_tris.p, entries,
                                               (int)ncell, h->cell_start.p, h->cell_start.p + 1));
    GRID_OK(cudaDeviceSynchronize());
  }
  h->launches += 2;  // k_grid_count, k_grid_fill (the scan and the sort are cub's)
  GRID_OK(cudaDeviceSynchronize());
#undef GRID_OK
  return cudaSuccess;
}

extern "C" int accfem_create(const accfem_model_desc* md, const accfem_mesh_desc* mesh, const accfem_settings* sd,
                             int device, accfem_handle** out) {
  g_create_error.clear();
  if (!out) return ACCFEM_E_ARG;
  *out = nullptr;
  std::string v = accfem_host::validate(md, sd);
  if (!v.empty()) {
    g_create_error = v;
    return ACCFEM_E_DOMAIN;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    g_create_error = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    return ACCFEM_E_CUDA;
  }
  accfem_handle* h = new accfem_handle();
  h->device = device;
  const int N = md->node_count, E = N - 1;
  h->N = N;
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device);
  Problem& P = h->P;
  memset(&P, 0, sizeof(P));
  // settings
  Settings& S = P.s;
  S.eps_abs = sd->eps_abs; S.eps_rel = sd->eps_rel; S.rho = sd->rho; S.sigma = sd->sigma;
  S.alpha = sd->alpha; S.beta0 = sd->beta0; S.margin = sd->margin;
  S.radius = std::max(sd->margin + sd->beta0, sd->margin);
  S.max_iterations = sd->max_iterations; S.check_interval = sd->check_interval;
  S.adaptive_rho = sd->adaptive_rho; S.scaling_iterations = sd->scaling_iterations; S.polish = sd->polish;
  S.backend = sd->backend; S.pgs_tol = sd->pgs_tol; S.pgs_min_sweep_factor = sd->pgs_min_sweep_factor;
  h->cmax = sd->polish_capacity > 0 ? sd->polish_capacity : std::min(N, 256);
  // model
  ModelDev& M = P.m;
  M.N = N;
  M.l0 = md->element_rest_length;
  accfem_host::local_stiffness(md, M.kl);
  M.n_cables = sd->n_cables;
  h->n_cables = sd->n_cables;
  for (int j = 0; j < sd->n_cables; ++j)
    for (int a = 0; a < 3; ++a) {
      M.cable_off[3 * j + a] = sd->cable_offset[3 * j + a];
      M.cable_dir[3 * j + a] = sd->cable_direction[3 * j + a];
    }
  {
    const double* r = md->rest_coords;
    double ax[3] = {r[6] - r[0], r[7] - r[1], r[8] - r[2]};
    double nrm = sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
    for (int a = 0; a < 3; ++a) M.axis[a] = ax[a] / nrm;
  }
  M.has_uniform = sd->has_uniform_load;
  for (int a = 0; a < 3; ++a) M.uniform[a] = sd->uniform_load[a];
  M.n_fixed = sd->n_fixed;
  h->n_fixed = sd->n_fixed;
  std::vector<int> frd(6L * N, -1);
  for (int r = 0; r < sd->n_fixed; ++r) frd[6 * sd->fixed_node[r] + sd->fixed_dof[r]] = r;
  int rc = 0;
#define UP(buf, ptr, cnt) \
  if ((e = h->buf.upload((ptr), (cnt))) != cudaSuccess) { rc = 1; }
  UP(rest, md->rest_coords, 6L * N);
  UP(fixed_node, sd->fixed_node, sd->n_fixed);
  UP(fixed_dof, sd->fixed_dof, sd->n_fixed);
  UP(fixed_inc, sd->fixed_increment, sd->n_fixed);
  UP(fixed_row_of_dof, frd.data(), frd.size());
  if (!rc) {
    h->rest_dir.alloc(9L * N); h->rest_len.alloc(E); h->rest_frames.alloc(9L * E);
    h->offsets.alloc(9L * E); h->qa.alloc(9L * E); h->qb.alloc(9L * E); h->bad.alloc(1);
  }
  // mesh + grid
  accfem_host::HostMesh hm;
  std::string merr = accfem_host::build_mesh(mesh, S.radius, hm, /*with_lists=*/false);
  if (!merr.empty()) {
    g_create_error = merr;
    delete h;
    return ACCFEM_E_MESH;
  }
  if (hm.T > 0) {
    UP(corners, hm.corners.data(), hm.corners.size());
    UP(normals, hm.normals.data(), hm.normals.size());
    UP(lo, hm.lo.data(), hm.lo.size());
    UP(hi, hm.hi.data(), hm.hi.size());
    if (!rc && (e = build_grid(h, hm)) != cudaSuccess) rc = 1;
  }
#undef UP
  if (rc || h->counter.alloc(4) != cudaSuccess) {
    g_create_error = std::string("device allocation failed: ") + cudaGetErrorString(e);
    delete h;
    return ACCFEM_E_CUDA;
  }
  MeshDev& G = P.mesh;
  G.T = hm.T;
  G.corners = h->corners.p; G.normals = h->normals.p; G.lo = h->lo.p; G.hi = h->hi.p;
  G.cell_start = h->cell_start.p; G.cell_tris = h->cell_tris.p;
  for (int a = 0; a < 3; ++a) {
    G.origin[a] = hm.origin[a];
    G.dims[a] = hm.dims[a];
  }
  G.inv_h = hm.inv_h;
  M.rest_dir = h->rest_dir.p; M.rest_len = h->rest_len.p; M.rest_frames = h->rest_frames.p;
  M.offsets = h->offsets.p; M.qa = h->qa.p; M.qb = h->qb.p;
  M.fixed_node = h->fixed_node.p; M.fixed_dof = h->fixed_dof.p; M.fixed_inc = h->fixed_inc.p;
  M.fixed_row_of_dof = h->fixed_row_of_dof.p;
  // per-model constants on the device
  k_model_setup<<<1, 32>>>(N, h->rest.p, h->rest_dir.p, h->rest_len.p, h->rest_frames.p, h->offsets.p, h->qa.p,
                           h->qb.p, h->bad.p);
  h->launches++;
  int bad = 0;
  e = cudaMemcpy(&bad, h->bad.p, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    g_create_error = std::string("model setup: ") + cudaGetErrorString(e);
    delete h;
    return ACCFEM_E_CUDA;
  }
  if (bad) {
    g_create_error = "rest configuration has coincident nodes";
    delete h;
    return ACCFEM_E_DOMAIN;
  }
  // launch mode: hot arrays in shared memory when they fit; team width from
  // ACCFEM_TEAM_WARPS (development override) or the default
  {
    int max_smem = 0, smem_sm = 0, resv = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, device);
    const char* force_global = getenv("ACCFEM_GLOBAL_WORKSPACE");
    const char* tw = getenv("ACCFEM_TEAM_WARPS");
    const char* lean_env = getenv("ACCFEM_LEAN");
    h->solve_warps = kTeamWarps;
    h->lat_warps = kLatencyTeamWarps;
    if (tw && solve_entry(atoi(tw))) h->solve_warps = h->lat_warps = atoi(tw);
    // hot set of the team kernels: the full layout, or -- when it buys one more
    // team per SM -- the lean one (factor, rhs and the row state of frames of
    // up to `mh` rows in shared memory)
    long hot = (ws_hot_doubles(N, sd->n_fixed) + 15) & ~15L;
    {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, solve_entry(h->solve_warps)->kernel);
      auto per_sm = [&](long d) { return smem_sm / (long)(d * 8 + (long)fa.sharedSizeBytes + resv); };
      const int mfull = sd->n_fixed + N;
      if (lean_env && lean_env[0] == '1' && hot * 8 <= max_smem) {  // opt-in: measured slower
        const long want = per_sm(hot) + 1;
        int best = 0;
        for (int mh = mfull - 1; mh >= sd->n_fixed + 8 && mh > 0; --mh) {
          const long d = (ws_hot_doubles(N, sd->n_fixed, false, mh) + 15) & ~15L;
          if (per_sm(d) >= want) {
            best = mh;
            break;
          }
        }
        if (best > 0) {
          h->hot_rows = best;
          hot = (ws_hot_doubles(N, sd->n_fixed, false, best) + 15) & ~15L;
        }
      }
    }
    // development knob: ACCFEM_SMEM_PAD=<doubles> pads the hot set (fewer teams per SM)
    if (const char* pad = getenv("ACCFEM_SMEM_PAD")) hot = (hot + atol(pad) + 15) & ~15L;
    const bool in_smem = hot * 8 <= max_smem && !(force_global && force_global[0] == '1');
    if (!in_smem) h->hot_rows = 0;
    h->hot_stride = in_smem ? hot : 0;
    for (int mode = 0; mode < 2; ++mode) {
      const int nw = mode ? h->lat_warps : h->solve_warps;
      int* bps = mode ? &h->lat_blocks_per_sm : &h->blocks_per_sm;
      const void* kern = solve_entry(nw)->kernel;
      if (in_smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(hot * 8));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, kern, 32 * nw, in_smem ? hot * 8 : 0);
      if (*bps < 1) *bps = 1;
    }
    // latency mode: one 16-warp CTA per scenario, cyclic reduction, hot set in shared memory
    const char* no_cr = getenv("ACCFEM_NO_CR");
    const char* mode = getenv("ACCFEM_MODE");
    if (mode) h->force_mode = !strcmp(mode, "cr") ? 1 : !strcmp(mode, "team4") ? 2 : !strcmp(mode, "team2") ? 3 : 0;
    long hot_cr = (ws_hot_doubles(N, sd->n_fixed, true) + 15) & ~15L;
    const KSolveEntry* ce = solve_entry(kCrTeamWarps, true);
    h->cr_blocks_per_sm = 0;
    if (ce && !(no_cr && no_cr[0] == '1')) {
      const bool cr_smem = hot_cr * 8 <= max_smem && !(force_global && force_global[0] == '1');
      h->cr_hot_stride = cr_smem ? hot_cr : 0;
      if (cr_smem) cudaFuncSetAttribute(ce->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(hot_cr * 8));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h->cr_blocks_per_sm, ce->kernel, 32 * kCrTeamWarps,
                                                    cr_smem ? hot_cr * 8 : 0);
    }
  }
  // everything a solve call needs is allocated here, so solve calls never
  // cudaMalloc: one workspace slab per resident team of either team width,
  // and host-path staging for `max_batch` scenarios / trace slots
  {
    {
      // default: 16384 scenarios, at most ~2 GiB of staging for large models
      const long per = 8L * (3 * 6L * N + 2 + 13L * N) + 4L * (4 + 2L * N);
      h->max_batch = sd->max_batch > 0 ? sd->max_batch : (int)std::max(1L, std::min(16384L, (2L << 30) / per));
    }
    h->trace_slots = sd->trace_slots > 0 ? sd->trace_slots : 1024;
    h->stat_slots = std::max<long>(h->trace_slots, 65536);
    long stride = std::max(ws_doubles(N, sd->n_fixed, h->cmax, false, h->hot_rows),
                           ws_doubles(N, sd->n_fixed, h->cmax, true));
    stride = (stride + 31) & ~31L;
    h->ws_stride = stride;
    h->ws_teams = std::max<long>((long)h->sms * h->blocks_per_sm, (long)h->sms * h->lat_blocks_per_sm);
    h->ws_teams = std::max<long>(h->ws_teams, (long)h->sms * h->cr_blocks_per_sm);
    const long Sb = h->max_batch, n = 6L * N, nf = std::max(sd->n_fixed, 1), nc = std::max(sd->n_cables, 1);
    const long ts = h->trace_slots;
    rc = 0;
    if (h->ws.alloc((size_t)stride * h->ws_teams) != cudaSuccess) rc = 1;
    if (!rc && (h->h_x0.alloc(Sb * n) || h->h_ten.alloc(Sb * nc) || h->h_app.alloc(Sb * n) || h->h_ins.alloc(Sb) ||
                h->h_wy.alloc(Sb * N) || h->h_wf.alloc(Sb * nf) || h->h_rho.alloc(Sb)))
      rc = 1;
    if (!rc && (h->o_coords.alloc(Sb * n + Sb + Sb * N * 11) || h->o_ints.alloc(Sb * 4 + Sb * N * 2) ||
                h->o_wy.alloc(Sb * N) || h->o_wf.alloc(Sb * nf) || h->o_rho.alloc(Sb)))
      rc = 1;
    if (!rc && h->o_tr.alloc(h->stat_slots * ACCFEM_TRACE_STATS + ts * n + ts * N * 8) != cudaSuccess) rc = 1;
    if (!rc && cudaEventCreateWithFlags(&h->done, cudaEventDisableTiming) != cudaSuccess) rc = 1;
    if (rc) {
      g_create_error = std::string("device allocation failed: ") + cudaGetErrorString(cudaGetLastError());
      accfem_destroy(h);
      return ACCFEM_E_CUDA;
    }
  }
  *out = h;
  return 0;
}

extern "C" int accfem_destroy(accfem_handle* h) {
  if (!h) return 0;
  cudaSetDevice(h->device);
  if (h->done) cudaEventSynchronize(h->done);
  if (h->done) cudaEventDestroy(h->done);
  delete h;  // DevBuf members free themselves
  return 0;
}

// Calls on one handle share its work counter and workspace: a launch on a
// stream other than the previous call's waits for that call's completion
// event (same-stream calls are already ordered).
static int order_on(accfem_handle* h, cudaStream_t st) {
  if (h->has_last && h->last_stream != st) CUDA_OK(h, cudaStreamWaitEvent(st, h->done, 0));
  return 0;
}
static int mark_done(accfem_handle* h, cudaStream_t st) {
  CUDA_OK(h, cudaEventRecord(h->done, st));
  h->last_stream = st;
  h->has_last = true;
  return 0;
}

// teams the preallocated workspace can host for `cmax` and a team count
static long teams_cap(accfem_handle* h) { return h->ws_teams; }

extern "C" int accfem_grid_shape(const accfem_handle* h, int32_t* dims, int64_t* n_cells, int64_t* n_entries) {
  if (!h || !dims || !n_cells || !n_entries) return ACCFEM_E_ARG;
  for (int a = 0; a < 3; ++a) dims[a] = h->grid_dims[a];
  *n_cells = h->grid_cells;
  *n_entries = h->grid_entries;
  return 0;
}

extern "C" int accfem_grid_download(accfem_handle* h, int32_t* cell_start, int32_t* cell_tris) {
  if (!h || !cell_start || !cell_tris) return ACCFEM_E_ARG;
  if (h->grid_cells == 0) return 0;
  cudaSetDevice(h->device);
  CUDA_OK(h, cudaMemcpy(cell_start, h->cell_start.p, (h->grid_cells + 1) * sizeof(int), cudaMemcpyDeviceToHost));
  if (h->grid_entries)
    CUDA_OK(h, cudaMemcpy(cell_tris, h->cell_tris.p, h->grid_entries * sizeof(int), cudaMemcpyDeviceToHost));
  return 0;
}

extern "C" int accfem_teams_resident(accfem_handle* h) { return h ? h->sms * h->blocks_per_sm : 0; }
extern "C" long long accfem_workspace_bytes(accfem_handle* h) { return h ? (long long)h->ws.n * 8 : 0; }
extern "C" int accfem_launches(accfem_handle* h) { return h ? h->launches : 0; }
extern "C" int accfem_max_batch(accfem_handle* h) { return h ? h->max_batch : 0; }
extern "C" int accfem_last_launch_teams(accfem_handle* h) { return h ? h->last_teams : 0; }

extern "C" int accfem_solve_batch(accfem_handle* h, const accfem_batch* io, void* stream) {
  if (!h || !io) return ACCFEM_E_ARG;
  if (io->S <= 0) return 0;
  if (!io->x0 || !io->coords || !io->status || !io->frames || !io->converged || !io->residual || !io->n_contacts ||
      !io->contact_node || !io->contact_triangle || !io->contact_gap || !io->contact_multiplier ||
      !io->contact_force || !io->contact_normal || !io->contact_point)
    return fail(h, ACCFEM_E_ARG, "missing required batch buffer");
  if (io->max_frames < 1) return fail(h, ACCFEM_E_ARG, "max_frames must be >= 1");
  if (h->n_cables > 0 && io->tensions == nullptr) {
    // tensions None: no cable wrench (engine.py:111)
  }
  CUDA_OK(h, cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  // latency modes: one scenario per SM (cyclic reduction) when the batch fits
  // one wave of them, else 4-warp teams when it fits theirs; throughput mode otherwise
  bool cr = h->cr_blocks_per_sm > 0 && (long)io->S <= (long)h->sms * h->cr_blocks_per_sm;
  bool lat = !cr && (long)io->S <= (long)h->sms * h->lat_blocks_per_sm;
  if (h->force_mode) {
    cr = h->force_mode == 1 && h->cr_blocks_per_sm > 0;
    lat = h->force_mode == 2;
  }
  const int nw = cr ? kCrTeamWarps : lat ? h->lat_warps : h->solve_warps;
  const int bps = cr ? h->cr_blocks_per_sm : lat ? h->lat_blocks_per_sm : h->blocks_per_sm;
  long blocks = std::max(1L, std::min((long)io->S, (long)h->sms * bps));
  blocks = std::min(blocks, teams_cap(h));
  const long hot_stride = cr ? h->cr_hot_stride : h->hot_stride;
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
  if (B.trace_c_node && !(B.trace_c_tri && B.trace_c_gap && B.trace_c_force && B.trace_c_point))
    return fail(h, ACCFEM_E_ARG, "trace contact buffers must be given together");
  B.max_frames = io->max_frames; B.stop_on_tol = io->stop_on_tol; B.tol = io->tol;
  B.fail_on_limit = io->fail_on_limit; B.cmax_polish = h->cmax; B.work_counter = h->counter.p;
  B.hot_rows = cr ? 0 : h->hot_rows;
  B.team_stats = reinterpret_cast<long long*>(io->team_stats);
  B.team_stats_cap = io->team_stats ? io->team_stats_cap : 0;
  h->last_teams = (int)blocks;
  B.prof = h->prof;
  if (int rc = order_on(h, st)) return rc;
  CUDA_OK(h, cudaMemsetAsync(h->counter.p, 0, sizeof(int), st));
  CUDA_OK(h, solve_entry(nw, cr)->launch((unsigned)blocks, (size_t)(hot_stride * 8), st, h->P, B, h->ws.p,
                                         h->ws_stride, hot_stride));
  h->launches++;
  CUDA_OK(h, cudaGetLastError());
  return mark_done(h, st);
}

// unit kernels: one-warp teams, at most the preallocated team count
static long unit_blocks(accfem_handle* h, long S) {
  long want = (S + kWarpsPerBlock - 1) / kWarpsPerBlock;
  return std::max(1L, std::min(want, teams_cap(h) / kWarpsPerBlock));
}

extern "C" int accfem_element_pass(accfem_handle* h, int32_t S, const double* x, double* f_int, double* k_diag,
                                   double* k_off, double* frames, int32_t* degenerate, void* stream) {
  if (!h || !x || !f_int) return ACCFEM_E_ARG;
  if (S <= 0) return 0;
  CUDA_OK(h, cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  long blocks = unit_blocks(h, S);
  if (int rc = order_on(h, st)) return rc;
  CUDA_OK(h, cudaMemsetAsync(h->counter.p, 0, sizeof(int), st));
  k_element_pass<<<(unsigned)blocks, 32 * kWarpsPerBlock, 0, st>>>(h->P, S, x, f_int, k_diag, k_off, frames,
                                                                     degenerate, h->ws.p, h->ws_stride, h->counter.p);
  h->launches++;
  CUDA_OK(h, cudaGetLastError());
  return mark_done(h, st);
}

extern "C" int accfem_detect(accfem_handle* h, int32_t S, const double* x, int32_t* tri, double* gap, double* point,
                             void* stream) {
  if (!h || !x || !tri || !gap || !point) return ACCFEM_E_ARG;
  if (h->P.mesh.T == 0) return fail(h, ACCFEM_E_MESH, "contact detection needs a non-empty mesh");
  if (S <= 0) return 0;
  CUDA_OK(h, cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  long blocks = unit_blocks(h, S);
  if (int rc = order_on(h, st)) return rc;
  CUDA_OK(h, cudaMemsetAsync(h->counter.p, 0, sizeof(int), st));
  k_detect<<<(unsigned)blocks, 32 * kWarpsPerBlock, 0, st>>>(h->P, S, x, tri, gap, point, h->ws.p, h->ws_stride,
                                                               h->counter.p);
  h->launches++;
  CUDA_OK(h, cudaGetLastError());
  return mark_done(h, st);
}

// Host-pointer variant: stage inputs into the handle's preallocated device
// buffers, solve, copy results back -- in chunks of at most max_batch
// scenarios (and as many as the trace staging holds), all on one stream.
// This is the path the e2e measurement exercises.
extern "C" int accfem_solve_batch_host(accfem_handle* h, const accfem_batch* io, void* stream) {
  if (!h || !io) return ACCFEM_E_ARG;
  if (io->S <= 0) return 0;
  CUDA_OK(h, cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const long N = h->N, n = 6 * N, nf = h->n_fixed, nc = h->n_cables;
  const long tcap = io->trace_cap;
  const bool tr_stats = io->trace_stats && tcap > 0, tr_coords = io->trace_coords && tcap > 0,
             tr_c = io->trace_contact_node && tcap > 0;
  long chunk = h->max_batch;
  if (tr_stats) chunk = std::min(chunk, h->stat_slots / tcap);
  if (tr_coords || tr_c) chunk = std::min(chunk, h->trace_slots / tcap);
  if (chunk < 1) return fail(h, ACCFEM_E_ARG, "trace_cap exceeds the handle's trace staging (accfem_settings.trace_slots)");
  for (long s0 = 0; s0 < io->S; s0 += chunk) {
    const long S = std::min(chunk, (long)io->S - s0);
    accfem_batch d = *io;
    d.S = (int32_t)S;
    auto stage = [&](DevBuf<double>& b, const double* src, long per, const double** dst) -> int {
      if (!src) {
        *dst = nullptr;
        return 0;
      }
      CUDA_OK(h, cudaMemcpyAsync(b.p, src + s0 * per, S * per * sizeof(double), cudaMemcpyHostToDevice, st));
      *dst = b.p;
      return 0;
    };
    int rc = 0;
    if ((rc = stage(h->h_x0, io->x0, n, &d.x0))) return rc;
    if ((rc = stage(h->h_ten, nc ? io->tensions : nullptr, nc, &d.tensions))) return rc;
    if ((rc = stage(h->h_app, io->applied, n, &d.applied))) return rc;
    if ((rc = stage(h->h_ins, io->insertion, 1, &d.insertion))) return rc;
    if ((rc = stage(h->h_wy, io->warm_y_in, N, &d.warm_y_in))) return rc;
    if ((rc = stage(h->h_wf, io->warm_fixed_in, nf, &d.warm_fixed_in))) return rc;
    if ((rc = stage(h->h_rho, io->rho_in, 1, &d.rho_in))) return rc;
    // outputs: one double slab + one int slab
    double* p = h->o_coords.p;
    d.coords = p; p += S * n;
    d.residual = p; p += S;
    d.contact_gap = p; p += S * N;
    d.contact_multiplier = p; p += S * N;
    d.contact_force = p; p += S * N * 3;
    d.contact_normal = p; p += S * N * 3;
    d.contact_point = p; p += S * N * 3;
    int* q = h->o_ints.p;
    d.status = q; q += S;
    d.frames = q; q += S;
    d.converged = q; q += S;
    d.n_contacts = q; q += S;
    d.contact_node = q; q += S * N;
    d.contact_triangle = q; q += S * N;
    d.warm_y_out = io->warm_y_out ? h->o_wy.p : nullptr;
    d.warm_fixed_out = io->warm_fixed_out ? h->o_wf.p : nullptr;
    d.rho_out = io->rho_out ? h->o_rho.p : nullptr;
    d.trace_stats = nullptr;
    d.trace_coords = nullptr;
    d.team_stats = nullptr;  // device-pointer calls only
    d.team_stats_cap = 0;
    d.trace_contact_node = nullptr;
    d.trace_contact_triangle = nullptr;
    d.trace_contact_gap = d.trace_contact_force = d.trace_contact_point = nullptr;
    {
      double* t = h->o_tr.p;
      if (tr_stats) d.trace_stats = t;
      t += h->stat_slots * ACCFEM_TRACE_STATS;
      if (tr_coords) d.trace_coords = t;
      t += h->trace_slots * n;
      if (tr_c) {
        d.trace_contact_gap = t; t += S * tcap * N;
        d.trace_contact_force = t; t += S * tcap * N * 3;
        d.trace_contact_point = t; t += S * tcap * N * 3;
        int* ti = reinterpret_cast<int*>(t);
        d.trace_contact_node = ti; ti += S * tcap * N;
        d.trace_contact_triangle = ti;
      }
    }
    if ((rc = accfem_solve_batch(h, &d, stream))) return rc;
    auto back = [&](void* dst, const void* src, size_t elem, long per) -> int {
      if (dst && per) {
        char* o = static_cast<char*>(dst) + (size_t)s0 * per * elem;
        CUDA_OK(h, cudaMemcpyAsync(o, src, (size_t)S * per * elem, cudaMemcpyDeviceToHost, st));
      }
      return 0;
    };
    if ((rc = back(io->coords, d.coords, 8, n))) return rc;
    if ((rc = back(io->residual, d.residual, 8, 1))) return rc;
    if ((rc = back(io->status, d.status, 4, 1))) return rc;
    if ((rc = back(io->frames, d.frames, 4, 1))) return rc;
    if ((rc = back(io->converged, d.converged, 4, 1))) return rc;
    if ((rc = back(io->n_contacts, d.n_contacts, 4, 1))) return rc;
    if ((rc = back(io->contact_node, d.contact_node, 4, N))) return rc;
    if ((rc = back(io->contact_triangle, d.contact_triangle, 4, N))) return rc;
    if ((rc = back(io->contact_gap, d.contact_gap, 8, N))) return rc;
    if ((rc = back(io->contact_multiplier, d.contact_multiplier, 8, N))) return rc;
    if ((rc = back(io->contact_force, d.contact_force, 8, N * 3))) return rc;
    if ((rc = back(io->contact_normal, d.contact_normal, 8, N * 3))) return rc;
    if ((rc = back(io->contact_point, d.contact_point, 8, N * 3))) return rc;
    if (io->warm_y_out && (rc = back(io->warm_y_out, d.warm_y_out, 8, N))) return rc;
    if (io->warm_fixed_out && (rc = back(io->warm_fixed_out, d.warm_fixed_out, 8, nf))) return rc;
    if (io->rho_out && (rc = back(io->rho_out, d.rho_out, 8, 1))) return rc;
    if (tr_stats && (rc = back(io->trace_stats, d.trace_stats, 8, tcap * ACCFEM_TRACE_STATS))) return rc;
    if (tr_coords && (rc = back(io->trace_coords, d.trace_coords, 8, tcap * n))) return rc;
    if (tr_c) {
      if ((rc = back(io->trace_contact_node, d.trace_contact_node, 4, tcap * N))) return rc;
      if ((rc = back(io->trace_contact_triangle, d.trace_contact_triangle, 4, tcap * N))) return rc;
      if ((rc = back(io->trace_contact_gap, d.trace_contact_gap, 8, tcap * N))) return rc;
      if ((rc = back(io->trace_contact_force, d.trace_contact_force, 8, tcap * N * 3))) return rc;
      if ((rc = back(io->trace_contact_point, d.trace_contact_point, 8, tcap * N * 3))) return rc;
    }
  }
  CUDA_OK(h, cudaStreamSynchronize(st));
  return 0;
}
