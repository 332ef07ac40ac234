"""TEST-ONLY binding of the serial emulation library (tests/emu/emu.cpp).

Same descriptors as the device C ABI; runs the team-generic device source on
one CPU thread so the CPU suite can check the device algorithm.
"""

import ctypes
import os
import subprocess

import numpy as np

from paper_2503_06922_b200 import _lib
from paper_2503_06922_b200.scene import fixed_rows

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libaccfem_emu.so")
SRC = [os.path.join(HERE, "emu.cpp")] + [
    os.path.join(HERE, "..", "..", "paper_2503_06922_b200", "csrc", f)
    for f in ("team.cuh", "so3.cuh", "problem.cuh", "mech.cuh", "linalg.cuh", "cr.cuh", "solve.cuh", "engine.cuh",
              "host_build.hpp")]


SO_ASAN = os.path.join(HERE, "libaccfem_emu_asan.so")


def build(force=False, sanitize=False):
    """The emulation library; sanitize=True builds the AddressSanitizer +
    UndefinedBehaviorSanitizer variant (load it with libasan preloaded)."""
    so = SO_ASAN if sanitize else SO
    newest = max(os.path.getmtime(p) for p in SRC)
    if force or not os.path.exists(so) or os.path.getmtime(so) < newest:
        flags = ["-O1", "-g", "-fsanitize=address,undefined", "-fno-omit-frame-pointer",
                 "-fno-sanitize-recover=undefined"] if sanitize else ["-O2"]
        subprocess.check_call(["g++", *flags, "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", "-o", so,
                               SRC[0]])
    return so


_EMU = None


def lib():
    global _EMU
    if _EMU is None:
        L = ctypes.CDLL(os.environ.get("ACCFEM_EMU_SO") or build())
        L.emu_create.restype = ctypes.c_void_p
        L.emu_create.argtypes = [ctypes.POINTER(_lib.ModelDesc), ctypes.POINTER(_lib.MeshDesc),
                                 ctypes.POINTER(_lib.SettingsDesc)]
        L.emu_last_error.restype = ctypes.c_char_p
        L.emu_last_error.argtypes = [ctypes.c_void_p]
        L.emu_destroy.argtypes = [ctypes.c_void_p]
        L.emu_solve_batch.argtypes = [ctypes.c_void_p, ctypes.POINTER(_lib.BatchDesc)]
        L.emu_element_pass.argtypes = [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 5
        L.emu_detect.argtypes = [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 4
        L.emu_grid_shape.argtypes = [ctypes.c_void_p] * 4
        L.emu_grid_download.argtypes = [ctypes.c_void_p] * 3
        _EMU = L
    return _EMU


class EmuEngine:
    def __init__(self, model, mesh=None, cables=(), fixed_specs=(), settings=None, margin=1e-4,
                 uniform_load=None):
        self.model, self.mesh, self.cables = model, mesh, list(cables)
        self.rows = fixed_rows(fixed_specs, model.node_count)
        self.desc = _lib.Descriptors(model, mesh, self.cables, self.rows, settings, margin, uniform_load)
        self.L = lib()
        self.h = self.L.emu_create(ctypes.byref(self.desc.model), ctypes.byref(self.desc.mesh),
                                   ctypes.byref(self.desc.settings))
        err = self.L.emu_last_error(self.h).decode()
        if err:
            raise RuntimeError(err)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.emu_destroy(self.h)

    def element_pass(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        S, N = x.shape[0], self.model.node_count
        f = np.zeros((S, 6 * N))
        kd = np.zeros((S, N, 6, 6))
        ku = np.zeros((S, N - 1, 6, 6))
        bad = np.zeros(S, np.int32)
        self.L.emu_element_pass(self.h, S, x.ctypes.data, f.ctypes.data, kd.ctypes.data, ku.ctypes.data,
                                bad.ctypes.data)
        return f, kd, ku, bad

    def broad_phase_grid(self):
        """Host build of the broad-phase grid (checker for Engine.broad_phase_grid)."""
        dims = np.zeros(3, np.int32)
        nc, ne = ctypes.c_int64(), ctypes.c_int64()
        self.L.emu_grid_shape(self.h, dims.ctypes.data, ctypes.addressof(nc), ctypes.addressof(ne))
        start = np.zeros(nc.value + 1, np.int32)
        tris = np.zeros(max(ne.value, 1), np.int32)
        self.L.emu_grid_download(self.h, start.ctypes.data, tris.ctypes.data)
        return dims, start, tris[:ne.value]

    def detect(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        S, N = x.shape[0], self.model.node_count
        tri = np.zeros((S, N), np.int32)
        gap = np.zeros((S, N))
        pt = np.zeros((S, N, 3))
        self.L.emu_detect(self.h, S, x.ctypes.data, tri.ctypes.data, gap.ctypes.data, pt.ctypes.data)
        return tri, gap, pt

    def solve(self, x0, tensions=None, applied=None, tol=1e-9, max_frames=5000, trace_cap=0, stop_on_tol=True,
              trace_coords=False):
        S, n = x0.shape
        N = n // 6
        H = dict(x0=np.ascontiguousarray(x0, np.float64),
                 tensions=None if tensions is None or not self.cables else np.ascontiguousarray(tensions, np.float64),
                 applied=None if applied is None else np.ascontiguousarray(applied, np.float64),
                 coords=np.zeros((S, n)), status=np.zeros(S, np.int32), frames=np.zeros(S, np.int32),
                 converged=np.zeros(S, np.int32), residual=np.zeros(S), n_contacts=np.zeros(S, np.int32),
                 contact_node=np.zeros((S, N), np.int32), contact_triangle=np.zeros((S, N), np.int32),
                 contact_gap=np.zeros((S, N)), contact_multiplier=np.zeros((S, N)),
                 contact_force=np.zeros((S, N, 3)), contact_normal=np.zeros((S, N, 3)),
                 contact_point=np.zeros((S, N, 3)))
        if trace_cap:
            H["trace_stats"] = np.zeros((S, trace_cap, _lib.TRACE_STATS))
            if trace_coords:
                H["trace_coords"] = np.zeros((S, trace_cap, n))
        d = _lib.BatchDesc()
        d.S = S
        for name, _ in _lib.BATCH_FIELDS:
            if name in H and H[name] is not None:
                setattr(d, name, H[name].ctypes.data)
        d.trace_cap = trace_cap
        d.max_frames = max_frames
        d.stop_on_tol = 1 if stop_on_tol else 0
        d.tol = tol
        d.fail_on_limit = 1 if stop_on_tol else 0
        self.L.emu_solve_batch(self.h, ctypes.byref(d))
        return H
