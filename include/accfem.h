/*
 * accfem.h -- C ABI of the B200 quasi-static equilibrium solver.
 *
 * Drop-in boundary for the hot path of the reference package `cablefem`
 * (Acc-FEM, /root/reference/pkg/src/cablefem).  Every entry point replaces one
 * reference interface; the Python mirror `paper_2503_06922_b200.Engine` keeps
 * the reference's constructor / run_static / step signatures on top of it.
 *
 *   accfem_create            Engine.__init__            engine.py:87-103
 *                            (RobotModel.__post_init__  beam.py:71-99,
 *                             AabbTree(mesh)            mesh.py:204-243)
 *   accfem_solve_batch       Engine.run_static          engine.py:267-283
 *                            (frames of Engine.step     engine.py:136-240)
 *   accfem_element_pass      internal_force +           beam.py:311-325
 *                            assemble_tangent_stiffness beam.py:335-356
 *   accfem_detect            detect_contacts            contact.py:49-120
 *   accfem_destroy           (Engine garbage collection)
 *   accfem_last_error        exception message text     errors.py:4-44
 *
 * Conventions: plain pointers and sizes only; FP64 throughout, int32
 * indices.  Per-scenario arrays are scenario-major.  Pointers in
 * accfem_batch are DEVICE pointers unless passed to accfem_solve_batch_host,
 * which takes HOST pointers and performs the copies itself (timed e2e path).
 * A handle is bound to one device; calls on one handle are not thread-safe.
 * Calls on one handle are ordered even across streams: a launch on a stream
 * other than the previous call's waits for that call to finish (the handle's
 * work queue and workspace are shared), and the caller's stream sees the
 * results in stream order.
 * Return value: 0 on success, >= 100 on API/CUDA failure (message via
 * accfem_last_error); per-scenario outcomes are status codes below.
 */
#ifndef ACCFEM_H
#define ACCFEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* per-scenario status codes (mirrors the reference exception taxonomy, errors.py) */
#define ACCFEM_OK 0
#define ACCFEM_DOMAIN_ERROR 1        /* DomainError */
#define ACCFEM_DEGENERATE_ELEMENT 2  /* DegenerateElementError (beam.py:262-264) */
#define ACCFEM_MESH_ERROR 3          /* MeshError */
#define ACCFEM_NONCONVERGENCE 4      /* NonConvergenceError (only surfaces through retries) */
#define ACCFEM_INFEASIBLE 5          /* InfeasibleError (solver.py:346-348) */
#define ACCFEM_ENGINE_SOLVER 6       /* EngineError: solver failed twice (engine.py:184-188) */
#define ACCFEM_ENGINE_MAX_FRAMES 7   /* EngineError: run_static exhausted max_frames (engine.py:281) */
#define ACCFEM_CAPACITY 8            /* polish active set larger than the handle's capacity */
#define ACCFEM_LINALG 9              /* non-positive pivot in a factorisation */

/* API return codes */
#define ACCFEM_E_ARG 100
#define ACCFEM_E_CUDA 101
#define ACCFEM_E_MESH 102
#define ACCFEM_E_DOMAIN 103

#define ACCFEM_TRACE_STATS 14 /* dx_norm, actuation_scale, max_penetration, complementarity_worst,
                                 residual, iterations, n_c, converged, retried, complementarity_ok,
                                 primal_residual, dual_residual, broad-phase pairs, polish rounds */

typedef struct accfem_handle accfem_handle;

/* robot: RobotModel (beam.py:54-111) + MaterialParams (beam.py:26-51) */
typedef struct {
  int32_t node_count;
  double element_rest_length;
  const double* rest_coords; /* 6N host */
  double young_modulus, cross_section_area, bending_inertia, poisson_ratio, torsion_constant;
} accfem_model_desc;

/* lumen: TriangleMesh (mesh.py:19-61); normals as stored by the mesh (after orient/flip) */
typedef struct {
  int32_t vertex_count, triangle_count; /* triangle_count == 0: no mesh */
  const double* vertices;               /* V x 3 host */
  const int64_t* triangles;             /* T x 3 host */
  const double* normals;                /* T x 3 host */
} accfem_mesh_desc;

/* constraints, actuation and SolverSettings (solver.py:41-68) */
typedef struct {
  int32_t n_fixed;                /* selector rows, constraints.py:40-63 order */
  const int32_t* fixed_node;
  const int32_t* fixed_dof;
  const double* fixed_increment;
  int32_t n_cables;               /* CableSpec, constraints.py:71-103 (<= 8) */
  const double* cable_offset;     /* n_cables x 3 */
  const double* cable_direction;  /* n_cables x 3 */
  int32_t has_uniform_load;
  double uniform_load[3];
  double margin;                  /* Engine(margin=) */
  double eps_abs, eps_rel, rho, sigma, alpha, beta0;
  int32_t max_iterations, check_interval, adaptive_rho, scaling_iterations, polish;
  int32_t polish_capacity;        /* max contacts a polish can hold (0: min(N, 256)); a frame with more
                                     contacts than this reports ACCFEM_CAPACITY */
  /* capacities fixed at create: every device buffer a solve call uses is
     allocated by accfem_create, so solve calls never allocate */
  int32_t max_batch;              /* host-path staging, scenarios per chunk (0: 16384); larger host
                                     batches are processed in chunks */
  int32_t trace_slots;            /* host-path per-frame coords/contact trace staging, in
                                     scenario-frames (0: 1024) */
  /* frame solver (SolverSettings.backend, solver.py:717-741) */
  int32_t backend;                /* ACCFEM_BACKEND_QP or ACCFEM_BACKEND_PGS */
  double pgs_tol;                 /* solver.py:57 */
  int32_t pgs_min_sweep_factor;   /* solver.py:58 */
} accfem_settings;

#define ACCFEM_BACKEND_QP 0       /* accelerated_qp: Ruiz-scaled ADMM + polish (solver.py:250-528) */
#define ACCFEM_BACKEND_PGS 1      /* pgs_baseline: projected Gauss-Seidel on the Delassus operator (solver.py:531-665) */

typedef struct {
  int32_t S;                    /* scenarios in this call */
  /* inputs */
  const double* x0;             /* S x 6N                     (run_static x0) */
  const double* tensions;       /* S x n_cables or NULL        (StepInputs.tensions) */
  const double* applied;        /* S x 6N or NULL              (StepInputs.applied_force) */
  const double* insertion;      /* S or NULL                   (StepInputs.insertion_increment) */
  const double* warm_y_in;      /* S x N or NULL: per-node contact multipliers (engine.py:101) */
  const double* warm_fixed_in;  /* S x n_fixed or NULL: selector multipliers (engine.py:102) */
  const double* rho_in;         /* S or NULL: engine rho state (engine.py:103) */
  /* outputs */
  double* coords;               /* S x 6N final configuration */
  int32_t* status;              /* S */
  int32_t* frames;              /* S frames run */
  int32_t* converged;           /* S: reached |dx| <= tol */
  double* residual;             /* S equilibrium residual of the last frame */
  int32_t* n_contacts;          /* S contacts of the last frame */
  int32_t* contact_node;        /* S x N: the first n_contacts[s] entries are defined */
  int32_t* contact_triangle;    /* S x N */
  double* contact_gap;          /* S x N */
  double* contact_multiplier;   /* S x N (step-limited) */
  double* contact_force;        /* S x N x 3 */
  double* contact_normal;       /* S x N x 3 */
  double* contact_point;        /* S x N x 3 */
  double* warm_y_out;           /* S x N or NULL */
  double* warm_fixed_out;       /* S x n_fixed or NULL */
  double* rho_out;              /* S or NULL */
  /* optional per-frame trace (frames >= trace_cap are not recorded) */
  int32_t trace_cap;
  double* trace_stats;          /* S x cap x ACCFEM_TRACE_STATS */
  double* trace_coords;         /* S x cap x 6N */
  int32_t* trace_contact_node;  /* S x cap x N (-1 padded) */
  int32_t* trace_contact_triangle;
  double* trace_contact_gap;
  double* trace_contact_force;  /* S x cap x N x 3 */
  double* trace_contact_point;  /* S x cap x N x 3 */
  /* control */
  int32_t max_frames;
  int32_t stop_on_tol;          /* 1: run_static; 0: exactly max_frames frames (Engine.step) */
  double tol;
  int32_t fail_on_limit;        /* 1: exhausting max_frames -> ACCFEM_ENGINE_MAX_FRAMES */
  /* optional per-team (CTA) load-balance record of the launch: 4 int64 per
     team -- scenarios solved, busy ns, start ns, end ns (%globaltimer) --
     for up to team_stats_cap teams (accfem_last_launch_teams() were used) */
  int64_t* team_stats;
  int32_t team_stats_cap;
} accfem_batch;

int accfem_create(const accfem_model_desc* model, const accfem_mesh_desc* mesh, const accfem_settings* settings,
                  int device, accfem_handle** out);
int accfem_destroy(accfem_handle* h);
const char* accfem_last_error(const accfem_handle* h);
int accfem_version(void);

/* device-pointer batch; `stream` is a cudaStream_t (NULL = legacy default) */
int accfem_solve_batch(accfem_handle* h, const accfem_batch* io, void* stream);
/* same, host pointers: H2D of inputs, solve, D2H of outputs, synchronous */
int accfem_solve_batch_host(accfem_handle* h, const accfem_batch* io, void* stream);

/* unit entry points (device pointers) */
int accfem_element_pass(accfem_handle* h, int32_t S, const double* x, double* f_int, double* k_diag,
                        double* k_off, double* frames, int32_t* degenerate, void* stream);
int accfem_detect(accfem_handle* h, int32_t S, const double* x, int32_t* tri, double* gap, double* point,
                  void* stream);

/* introspection */
int accfem_teams_resident(accfem_handle* h);
long long accfem_workspace_bytes(accfem_handle* h);
int accfem_launches(accfem_handle* h); /* kernels launched by this handle so far */
int accfem_max_batch(accfem_handle* h); /* host-path chunk size (accfem_settings.max_batch) */
int accfem_last_launch_teams(accfem_handle* h); /* CTAs (teams) of the last solve launch */

/* broad-phase grid built on the device by accfem_create (replaces the
 * AabbTree build, mesh.py:204-243): dims[3], cell count, list entries; and a
 * copy of its CSR lists (cell_start[n_cells + 1], cell_tris[n_entries]) */
int accfem_grid_shape(const accfem_handle* h, int32_t* dims, int64_t* n_cells, int64_t* n_entries);
int accfem_grid_download(accfem_handle* h, int32_t* cell_start, int32_t* cell_tris);

#ifdef __cplusplus
}
#endif
#endif /* ACCFEM_H */
