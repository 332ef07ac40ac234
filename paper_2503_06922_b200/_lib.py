"""ctypes binding of include/accfem.h (the C ABI of the sm_100a library).

The library `libaccfem.so` is built in-tree by `paper_2503_06922_b200.build`
(nvcc -gencode arch=compute_100a,code=sm_100a).  There is no fallback: if the
library or a CUDA device is missing, `load()` raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ACCFEM_LIB") or os.path.join(HERE, "libaccfem.so")  # ACCFEM_LIB: development A/B builds

c_int32, c_double, c_void_p = ctypes.c_int32, ctypes.c_double, ctypes.c_void_p

TRACE_STATS = 14
BACKENDS = {"accelerated_qp": 0, "pgs_baseline": 1}  # include/accfem.h ACCFEM_BACKEND_*
E_CODES = {100: "bad argument", 101: "CUDA error", 102: "mesh error", 103: "domain error"}


class ModelDesc(ctypes.Structure):
    _fields_ = [("node_count", c_int32), ("element_rest_length", c_double), ("rest_coords", c_void_p),
                ("young_modulus", c_double), ("cross_section_area", c_double), ("bending_inertia", c_double),
                ("poisson_ratio", c_double), ("torsion_constant", c_double)]


class MeshDesc(ctypes.Structure):
    _fields_ = [("vertex_count", c_int32), ("triangle_count", c_int32), ("vertices", c_void_p),
                ("triangles", c_void_p), ("normals", c_void_p)]


class SettingsDesc(ctypes.Structure):
    _fields_ = [("n_fixed", c_int32), ("fixed_node", c_void_p), ("fixed_dof", c_void_p),
                ("fixed_increment", c_void_p), ("n_cables", c_int32), ("cable_offset", c_void_p),
                ("cable_direction", c_void_p), ("has_uniform_load", c_int32), ("uniform_load", c_double * 3),
                ("margin", c_double), ("eps_abs", c_double), ("eps_rel", c_double), ("rho", c_double),
                ("sigma", c_double), ("alpha", c_double), ("beta0", c_double), ("max_iterations", c_int32),
                ("check_interval", c_int32), ("adaptive_rho", c_int32), ("scaling_iterations", c_int32),
                ("polish", c_int32), ("polish_capacity", c_int32), ("max_batch", c_int32),
                ("trace_slots", c_int32), ("backend", c_int32), ("pgs_tol", c_double),
                ("pgs_min_sweep_factor", c_int32)]


BATCH_FIELDS = [
    ("S", c_int32),
    ("x0", c_void_p), ("tensions", c_void_p), ("applied", c_void_p), ("insertion", c_void_p),
    ("warm_y_in", c_void_p), ("warm_fixed_in", c_void_p), ("rho_in", c_void_p),
    ("coords", c_void_p), ("status", c_void_p), ("frames", c_void_p), ("converged", c_void_p),
    ("residual", c_void_p), ("n_contacts", c_void_p), ("contact_node", c_void_p),
    ("contact_triangle", c_void_p), ("contact_gap", c_void_p), ("contact_multiplier", c_void_p),
    ("contact_force", c_void_p), ("contact_normal", c_void_p), ("contact_point", c_void_p),
    ("warm_y_out", c_void_p), ("warm_fixed_out", c_void_p), ("rho_out", c_void_p),
    ("trace_cap", c_int32), ("trace_stats", c_void_p), ("trace_coords", c_void_p),
    ("trace_contact_node", c_void_p), ("trace_contact_triangle", c_void_p), ("trace_contact_gap", c_void_p),
    ("trace_contact_force", c_void_p), ("trace_contact_point", c_void_p),
    ("max_frames", c_int32), ("stop_on_tol", c_int32), ("tol", c_double), ("fail_on_limit", c_int32),
    ("team_stats", c_void_p), ("team_stats_cap", c_int32),
]


class BatchDesc(ctypes.Structure):
    _fields_ = BATCH_FIELDS


# exported symbols and their signatures (include/accfem.h)
SIGNATURES = {
    "accfem_create": (ctypes.c_int, [ctypes.POINTER(ModelDesc), ctypes.POINTER(MeshDesc),
                                     ctypes.POINTER(SettingsDesc), ctypes.c_int, ctypes.POINTER(c_void_p)]),
    "accfem_destroy": (ctypes.c_int, [c_void_p]),
    "accfem_last_error": (ctypes.c_char_p, [c_void_p]),
    "accfem_version": (ctypes.c_int, []),
    "accfem_solve_batch": (ctypes.c_int, [c_void_p, ctypes.POINTER(BatchDesc), c_void_p]),
    "accfem_solve_batch_host": (ctypes.c_int, [c_void_p, ctypes.POINTER(BatchDesc), c_void_p]),
    "accfem_element_pass": (ctypes.c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                           c_void_p, c_void_p]),
    "accfem_detect": (ctypes.c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "accfem_teams_resident": (ctypes.c_int, [c_void_p]),
    "accfem_workspace_bytes": (ctypes.c_longlong, [c_void_p]),
    "accfem_launches": (ctypes.c_int, [c_void_p]),
    "accfem_max_batch": (ctypes.c_int, [c_void_p]),
    "accfem_last_launch_teams": (ctypes.c_int, [c_void_p]),
    "accfem_grid_shape": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "accfem_grid_download": (ctypes.c_int, [c_void_p, c_void_p, c_void_p]),
}

_LIB = None


def bind(lib):
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def load(path=LIB_PATH):
    """Load the sm_100a library; raises if it is absent (no CPU fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(nvcc, sm_100a).  The device path has no CPU fallback.")
        _LIB = bind(ctypes.CDLL(path))
    return _LIB


def ptr(a):
    """Address of a numpy array / torch tensor (or None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


class Descriptors:
    """Keeps the numpy arrays behind the create-time descriptors alive."""

    def __init__(self, model, mesh, cables, fixed_rows, settings, margin, uniform_load, polish_capacity=0,
                 max_batch=0, trace_slots=0):
        self.keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(np.asarray(a, dtype=dt))
            self.keep.append(a)
            return a

        mat = model.material
        rest = arr(model.rest_configuration, np.float64)
        self.model = ModelDesc(model.node_count, model.element_rest_length, ptr(rest), mat.young_modulus,
                               mat.cross_section_area, mat.bending_inertia, mat.poisson_ratio, mat.torsion_constant)
        if mesh is not None:
            v = arr(mesh.vertices, np.float64)
            t = arr(mesh.triangles, np.int64)
            nr = arr(mesh.normals, np.float64)
            self.mesh = MeshDesc(len(v), len(t), ptr(v), ptr(t), ptr(nr))
        else:
            self.mesh = MeshDesc(0, 0, None, None, None)
        fn = arr([r[0] for r in fixed_rows] or [0], np.int32)
        fd = arr([r[1] for r in fixed_rows] or [0], np.int32)
        fi = arr([r[2] for r in fixed_rows] or [0.0], np.float64)
        co = arr([c.attachment_offset for c in cables] or [[0.0] * 3], np.float64)
        cd = arr([c.tension_direction for c in cables] or [[0.0] * 3], np.float64)
        s = settings
        uni = (c_double * 3)(*(uniform_load if uniform_load is not None else (0.0, 0.0, 0.0)))
        self.settings = SettingsDesc(len(fixed_rows), ptr(fn), ptr(fd), ptr(fi), len(cables), ptr(co), ptr(cd),
                                     1 if uniform_load is not None else 0, uni, float(margin), s.eps_abs, s.eps_rel,
                                     s.rho, s.sigma, s.alpha, s.beta0, s.max_iterations, s.check_interval,
                                     1 if s.adaptive_rho else 0, s.scaling_iterations, 1 if s.polish else 0,
                                     int(polish_capacity), int(max_batch), int(trace_slots),
                                     BACKENDS[s.backend], float(s.pgs_tol), int(s.pgs_min_sweep_factor))
