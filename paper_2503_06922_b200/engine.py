"""Drop-in `Engine` for the reference's quasi-static solve, on the B200.

`Engine(model, mesh=None, cables=(), fixed_specs=(), settings=None,
margin=1e-4, uniform_load=None)` keeps the reference constructor
(engine.py:87-103); `run_static` and `step` keep its signatures and return
types (engine.py:136-283), including the cross-frame solver state (warm
multipliers by node, warm selector multipliers, adaptive rho) that persists
between calls.  Every frame runs on the device through `include/accfem.h`;
the host only validates inputs and converts records.

`Engine.solve_static_batch` is the throughput API: a batch of independent
scenarios (x0, tensions, applied load) solved to equilibrium by one
persistent kernel, one warp per scenario.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import (
    STATUS_ENGINE_MAX_FRAMES,
    STATUS_OK,
    DeviceError,
    DomainError,
    exception_for_status,
)
from .scene import Configuration, ContactPoint, FrameRecord, SolverSettings, StepInputs, fixed_rows

_TRACE_CHUNK = 256


@dataclass
class BatchResult:
    """Outputs of `solve_static_batch` (torch tensors on the engine device, or
    numpy arrays for host-buffer calls)."""

    coords: object
    status: object
    frames: object
    converged: object
    residual: object
    n_contacts: object
    contact_node: object
    contact_triangle: object
    contact_gap: object
    contact_multiplier: object
    contact_force: object
    contact_normal: object
    contact_point: object
    trace_stats: object = None

    def to_numpy(self):
        from dataclasses import fields

        out = {}
        for fd in fields(self):
            k, v = fd.name, getattr(self, fd.name)
            if v is None:
                out[k] = None
            elif hasattr(v, "detach"):
                out[k] = v.detach().cpu().numpy()
            else:
                out[k] = v
        return BatchResult(**out)


@dataclass
class BatchState:
    """Per-scenario cross-frame solver state of the batched frame mode."""

    warm_y: object       # (S, N) contact multipliers by node
    warm_fixed: object   # (S, n_fixed) selector multipliers, or None before the first frame
    rho: object          # (S,)


class Engine:
    """Single-writer stepping loop over one robot/mesh/constraint setup."""

    def __init__(self, model, mesh=None, cables=(), fixed_specs=(), settings=None, margin=1e-4,
                 uniform_load=None, device=None, polish_capacity=0, max_batch=0):
        self.model = model
        self.mesh = mesh
        self.cables = list(cables)
        self.fixed_specs = list(fixed_specs)
        self.settings = settings if settings is not None else SolverSettings()
        if self.settings.backend not in ("accelerated_qp", "pgs_baseline"):
            raise DomainError("the device path implements the accelerated_qp and pgs_baseline backends")
        self.margin = float(margin)
        if self.margin < 0.0:
            raise DomainError("margin must be >= 0")
        self.uniform_load = None if uniform_load is None else np.asarray(uniform_load, dtype=float)
        if len(self.cables) > 8:
            raise DomainError("at most 8 cables are supported")
        self._rows = fixed_rows(self.fixed_specs, model.node_count)
        rest = model.rest_positions
        axis = rest[1] - rest[0]
        self.insertion_axis = axis / np.linalg.norm(axis)
        import torch

        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        self._lib = _lib.load()
        self._desc = _lib.Descriptors(model, mesh, self.cables, self._rows, self.settings, self.margin,
                                      self.uniform_load, polish_capacity, max_batch)
        handle = ctypes.c_void_p()
        rc = self._lib.accfem_create(ctypes.byref(self._desc.model), ctypes.byref(self._desc.mesh),
                                     ctypes.byref(self._desc.settings), self.device.index, ctypes.byref(handle))
        if rc != 0:
            msg = self._lib.accfem_last_error(None).decode()
            if rc == 103:
                raise DomainError(msg)
            if rc == 102:
                from .errors import MeshError
                raise MeshError(msg)
            raise DeviceError(f"accfem_create failed ({rc}): {msg}")
        self._h = handle
        # reference callers that build their own initial record read the
        # engine's broad-phase tree (engine.py:96, 319-338); None makes
        # detect_contacts build its own (the device grid lives in the handle)
        self._tree = None
        # cross-frame solver state (engine.py:100-103)
        self._warm_y = np.zeros(model.node_count)
        self._warm_fixed = None
        self._rho = float(self.settings.rho)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._lib.accfem_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass
            self._h = None

    # -- helpers ----------------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            raise DeviceError(f"accfem call failed ({rc}): {self._lib.accfem_last_error(self._h).decode()}")

    @property
    def launches(self):
        return int(self._lib.accfem_launches(self._h))

    def broad_phase_grid(self):
        """The device-built broad-phase grid (the AabbTree's replacement,
        mesh.py:204-243): (dims[3], cell_start[n_cells + 1], cell_tris)."""
        dims = np.zeros(3, np.int32)
        nc, ne = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._lib.accfem_grid_shape(self._h, dims.ctypes.data, ctypes.addressof(nc),
                                                ctypes.addressof(ne)))
        start = np.zeros(nc.value + 1, np.int32)
        tris = np.zeros(max(ne.value, 1), np.int32)
        self._check(self._lib.accfem_grid_download(self._h, start.ctypes.data, tris.ctypes.data))
        return dims, start, tris[:ne.value]

    def initial_configuration(self):
        return Configuration(self.model.rest_configuration.copy(), timestep_index=0)

    def _validate_inputs(self, inputs):
        n = self.model.dof_count
        ten = None
        if self.cables and inputs.tensions is not None:
            ten = np.asarray(inputs.tensions, dtype=float)
            if len(ten) != len(self.cables):
                raise DomainError("one tension per cable required")
            if np.any(ten < 0.0):
                raise DomainError("cable tensions must be >= 0 (cables cannot push)")
        app = None
        if inputs.applied_force is not None:
            app = np.asarray(inputs.applied_force, dtype=float)
            if app.shape != (n,):
                raise DomainError(f"applied_force must have length {n}")
        return ten, app

    def _contact_points(self, nodes, tris, gaps, points):
        l0 = self.model.element_rest_length
        out = []
        for i, (nd, tri, gap, pp) in enumerate(zip(nodes, tris, gaps, points)):
            nd = int(nd)
            element, xi = (1, 0.0) if nd == 0 else (nd, l0)
            out.append(ContactPoint(contact_id=i, element_index=element, xi=xi,
                                    normal=-self.mesh.normals[int(tri)], plane_point=pp.copy(),
                                    triangle_id=int(tri), gap=float(gap)))
        return out

    # -- single scenario (host buffers through accfem_solve_batch_host) --------
    def _run_chunk(self, coords, ten, app, insertion, frames, stop_on_tol, tol, fail_on_limit):
        N, n = self.model.node_count, self.model.dof_count
        nf = len(self._rows)
        cap = frames
        H = dict(
            x0=np.ascontiguousarray(coords, dtype=np.float64),
            tensions=None if ten is None else np.ascontiguousarray(ten, dtype=np.float64),
            applied=None if app is None else np.ascontiguousarray(app, dtype=np.float64),
            insertion=np.array([float(insertion)]) if insertion else None,
            warm_y_in=self._warm_y.copy(),
            warm_fixed_in=None if self._warm_fixed is None else np.ascontiguousarray(self._warm_fixed),
            rho_in=np.array([self._rho]),
            coords=np.empty(n), status=np.zeros(1, np.int32), frames=np.zeros(1, np.int32),
            converged=np.zeros(1, np.int32), residual=np.zeros(1), n_contacts=np.zeros(1, np.int32),
            contact_node=np.zeros(N, np.int32), contact_triangle=np.zeros(N, np.int32),
            contact_gap=np.zeros(N), contact_multiplier=np.zeros(N), contact_force=np.zeros((N, 3)),
            contact_normal=np.zeros((N, 3)), contact_point=np.zeros((N, 3)),
            warm_y_out=np.zeros(N), warm_fixed_out=np.zeros(max(nf, 1)), rho_out=np.zeros(1),
            trace_stats=np.zeros((cap, _lib.TRACE_STATS)), trace_coords=np.zeros((cap, n)),
            trace_contact_node=np.full((cap, N), -1, np.int32), trace_contact_triangle=np.zeros((cap, N), np.int32),
            trace_contact_gap=np.zeros((cap, N)), trace_contact_force=np.zeros((cap, N, 3)),
            trace_contact_point=np.zeros((cap, N, 3)),
        )
        desc = _lib.BatchDesc()
        desc.S = 1
        for name, _ in _lib.BATCH_FIELDS:
            if name in H:
                setattr(desc, name, _lib.ptr(H[name]))
        desc.trace_cap = cap
        desc.max_frames = frames
        desc.stop_on_tol = 1 if stop_on_tol else 0
        desc.tol = float(tol)
        desc.fail_on_limit = 1 if fail_on_limit else 0
        t0 = time.perf_counter()
        self._check(self._lib.accfem_solve_batch_host(self._h, ctypes.byref(desc), None))
        wall_ms = (time.perf_counter() - t0) * 1e3
        status = int(H["status"][0])
        done = int(H["frames"][0])
        # persist the engine state for the next call (engine.py:248-255)
        if done > 0:
            self._warm_y = H["warm_y_out"].copy()
            self._warm_fixed = H["warm_fixed_out"][:nf].copy()
            self._rho = float(H["rho_out"][0])
        return H, status, done, wall_ms

    def _records(self, H, done, t, frame0, wall_ms):
        recs = []
        per = wall_ms / max(done, 1)
        for f in range(done):
            st = H["trace_stats"][f]
            nc = int(st[6])
            nodes = H["trace_contact_node"][f][:nc]
            cps = self._contact_points(nodes, H["trace_contact_triangle"][f][:nc], H["trace_contact_gap"][f][:nc],
                                       H["trace_contact_point"][f][:nc]) if nc else []
            coords = H["trace_coords"][f].copy()
            recs.append(FrameRecord(
                t=t, frame_index=frame0 + f, coords=coords, n_c=nc,
                contact_force_vectors=H["trace_contact_force"][f][:nc].copy(), contact_points=cps,
                tip_position=coords.reshape(-1, 6)[-1, :3].copy(), dx_norm=float(st[0]),
                iterations=int(st[5]), converged=bool(st[7]), retried=bool(st[8]),
                actuation_scale=float(st[1]), max_penetration=float(st[2]), complementarity_ok=bool(st[9]),
                complementarity_worst=float(st[3]), residual_norm=float(st[4]),
                timings_ms={"stiffness": 0.0, "detection": 0.0, "assembly": 0.0, "solve": per, "update": 0.0,
                            "total": per},
            ))
        return recs

    def step(self, x, inputs, t=0.0, frame_index=0):
        """Advance one frame (engine.py:136-240); returns (Configuration, FrameRecord)."""
        ten, app = self._validate_inputs(inputs)
        H, status, done, wall_ms = self._run_chunk(x.coords, ten, app, inputs.insertion_increment, 1, False, 0.0,
                                                   False)
        if status != STATUS_OK:
            raise exception_for_status(status, f"frame {frame_index}: device status {status}")
        rec = self._records(H, done, t, frame_index, wall_ms)[0]
        return Configuration(H["coords"].copy(), timestep_index=x.timestep_index + 1), rec

    def run_static(self, inputs, x0=None, tol=1e-9, max_frames=5000):
        """Frames under constant inputs until |dx| <= tol (engine.py:267-283).

        Returns (configuration, records, residual).  Runs in device launches of
        up to 256 frames each, carrying the solver state between them.
        """
        ten, app = self._validate_inputs(inputs)
        x = self.initial_configuration() if x0 is None else x0
        coords = x.coords.copy()
        records = []
        left = int(max_frames)
        ts = x.timestep_index
        while left > 0:
            chunk = min(left, _TRACE_CHUNK)
            H, status, done, wall_ms = self._run_chunk(coords, ten, app, inputs.insertion_increment, chunk, True,
                                                       tol, False)
            records += self._records(H, done, 0.0, len(records), wall_ms)
            if status != STATUS_OK:
                raise exception_for_status(status, f"frame {len(records)}: device status {status}")
            coords = H["coords"].copy()
            ts += done
            left -= done
            if H["converged"][0]:
                return Configuration(coords, timestep_index=ts), records, float(H["residual"][0])
        from .errors import EngineError
        raise EngineError(f"static mode did not reach |dx| <= {tol} in {max_frames} frames "
                          f"(last |dx| = {records[-1].dx_norm:.3e})")

    # -- batch input checks ------------------------------------------------------
    def _batch_input(self, a, shape, name, host):
        """float64, C-contiguous, the declared shape, and on the right side of the
        boundary: numpy for the host path, a CUDA tensor on this engine's device
        for the device path (converted if needed; a host pointer must never reach
        a kernel)."""
        if a is None:
            return None
        import torch

        if host:
            if isinstance(a, torch.Tensor):
                a = a.detach().cpu().numpy()
            a = np.ascontiguousarray(a, dtype=np.float64)
        else:
            if not isinstance(a, torch.Tensor):
                a = torch.as_tensor(np.asarray(a, dtype=np.float64))
            a = a.to(device=self.device, dtype=torch.float64).contiguous()
        if tuple(a.shape) != tuple(shape):
            raise DomainError(f"{name} must have shape {tuple(shape)}, got {tuple(a.shape)}")
        return a

    def _check_out(self, out, S, host):
        import torch

        ref = self.allocate_batch(0, host=host)
        for name in ("coords", "status", "frames", "converged", "residual", "n_contacts", "contact_node",
                     "contact_triangle", "contact_gap", "contact_multiplier", "contact_force", "contact_normal",
                     "contact_point"):
            a, r = getattr(out, name), getattr(ref, name)
            want = (S,) + tuple(r.shape[1:])
            if tuple(a.shape) != want or a.dtype != r.dtype:
                raise DomainError(f"out.{name} must be {r.dtype} of shape {want}")
            if host and not (isinstance(a, np.ndarray) and a.flags.c_contiguous):
                raise DomainError(f"out.{name} must be a C-contiguous numpy array for a host call")
            if not host and not (isinstance(a, torch.Tensor) and a.device == self.device and a.is_contiguous()):
                raise DomainError(f"out.{name} must be a contiguous tensor on {self.device}")

    # -- batch -----------------------------------------------------------------
    def allocate_batch(self, S, host=False):
        """Output buffers for S scenarios (torch on device, or numpy if host)."""
        N, n = self.model.node_count, self.model.dof_count
        if host:
            z = lambda shape, dt=np.float64: np.zeros(shape, dt)  # noqa: E731
            i32 = np.int32
        else:
            import torch
            z = lambda shape, dt=torch.float64: torch.zeros(shape, dtype=dt, device=self.device)  # noqa: E731
            i32 = torch.int32
        return BatchResult(coords=z((S, n)), status=z((S,), i32), frames=z((S,), i32), converged=z((S,), i32),
                           residual=z((S,)), n_contacts=z((S,), i32), contact_node=z((S, N), i32),
                           contact_triangle=z((S, N), i32), contact_gap=z((S, N)), contact_multiplier=z((S, N)),
                           contact_force=z((S, N, 3)), contact_normal=z((S, N, 3)), contact_point=z((S, N, 3)))

    def solve_static_batch(self, x0, tensions=None, applied=None, insertion=None, tol=1e-9, max_frames=5000,
                           out=None, stream=None, host=None, trace_frames=0, team_stats=None):
        """run_static of S independent scenarios, each from a fresh Engine state.

        Inputs are (S, 6N) / (S, n_cables) arrays: torch CUDA tensors (device
        path, async on `stream`) or numpy arrays (host path: copies inside the
        call).  Status codes per scenario follow include/accfem.h.
        `trace_frames` > 0 also records the first `trace_frames` frames' stats
        of every scenario (FrameRecord fields, include/accfem.h
        ACCFEM_TRACE_STATS layout) into `out.trace_stats` (S, trace_frames, 14).
        `team_stats` (device calls): an int64 CUDA tensor (T, 4) receiving the
        launch's per-team load-balance record (scenarios, busy ns, start ns,
        end ns) for the first T teams (accfem_last_launch_teams() were used).
        """
        import torch

        if host is None:
            host = isinstance(x0, np.ndarray)
        S = int(x0.shape[0])
        n, nca = self.model.dof_count, len(self.cables)
        x0 = self._batch_input(x0, (S, n), "x0", host)
        tensions = self._batch_input(tensions, (S, nca), "tensions", host) if self.cables else None
        if tensions is not None and bool((tensions < 0).any()):
            raise DomainError("cable tensions must be >= 0 (cables cannot push)")
        applied = self._batch_input(applied, (S, n), "applied", host)
        insertion = self._batch_input(insertion, (S,), "insertion", host)
        if out is None:
            out = self.allocate_batch(S, host=host)
        else:
            self._check_out(out, S, host)
        desc = _lib.BatchDesc()
        desc.S = S
        keep = []

        def put(name, a):
            if a is None:
                return
            keep.append(a)
            setattr(desc, name, _lib.ptr(a))

        put("x0", x0)
        put("tensions", tensions)
        put("applied", applied)
        put("insertion", insertion)
        for name in ("coords", "status", "frames", "converged", "residual", "n_contacts", "contact_node",
                     "contact_triangle", "contact_gap", "contact_multiplier", "contact_force", "contact_normal",
                     "contact_point"):
            setattr(desc, name, _lib.ptr(getattr(out, name)))
        if trace_frames > 0:
            if host:
                out.trace_stats = np.zeros((S, int(trace_frames), _lib.TRACE_STATS))
            else:
                out.trace_stats = torch.zeros((S, int(trace_frames), _lib.TRACE_STATS), dtype=torch.float64,
                                              device=self.device)
            desc.trace_cap = int(trace_frames)
            desc.trace_stats = _lib.ptr(out.trace_stats)
        if team_stats is not None and not host:
            import torch as _t
            if team_stats.dtype != _t.int64 or team_stats.device != self.device or team_stats.dim() != 2 \
                    or team_stats.shape[1] != 4 or not team_stats.is_contiguous():
                raise DomainError("team_stats must be a contiguous int64 (T, 4) tensor on the engine device")
            desc.team_stats = _lib.ptr(team_stats)
            desc.team_stats_cap = int(team_stats.shape[0])
            keep.append(team_stats)
        desc.max_frames = int(max_frames)
        desc.stop_on_tol = 1
        desc.tol = float(tol)
        desc.fail_on_limit = 1
        if host:
            rc = self._lib.accfem_solve_batch_host(self._h, ctypes.byref(desc), None)
        else:
            st = torch.cuda.current_stream(self.device) if stream is None else stream
            rc = self._lib.accfem_solve_batch(self._h, ctypes.byref(desc), ctypes.c_void_p(st.cuda_stream))
        self._check(rc)
        out._keep = keep  # inputs must outlive the asynchronous launch
        return out

    # -- batched frame mode (real-time stepping) -------------
    def initial_batch_state(self, S):
        """Fresh cross-frame solver state for S scenarios (engine.py:100-103)."""
        import torch
        return BatchState(warm_y=torch.zeros((S, self.model.node_count), dtype=torch.float64, device=self.device),
                          warm_fixed=None,
                          rho=torch.full((S,), float(self.settings.rho), dtype=torch.float64, device=self.device))

    def step_batch(self, x, tensions=None, applied=None, insertion=None, state=None, stream=None):
        """One `Engine.step` (engine.py:136-240) for each of S scenarios.

        x (S, 6N), tensions (S, n_cables), applied (S, 6N), insertion (S,) are
        torch CUDA tensors; `state` carries each scenario's warm multipliers and
        rho between frames (a fresh state if None).  Returns (BatchResult with
        the new coords and last-frame contacts, per-frame stats (S, 14) in the
        layout of include/accfem.h ACCFEM_TRACE_STATS, new BatchState).
        """
        import torch

        S, N = int(x.shape[0]), self.model.node_count
        n, nf, nca = self.model.dof_count, len(self._rows), len(self.cables)
        if state is None:
            state = self.initial_batch_state(S)
        for name, a, shape in (("state.warm_y", state.warm_y, (S, N)), ("state.rho", state.rho, (S,)),
                               ("state.warm_fixed", state.warm_fixed, (S, nf))):
            if a is not None and (tuple(a.shape) != shape or a.dtype != torch.float64 or a.device != self.device):
                raise DomainError(f"{name} must be float64 {shape} on {self.device}")
        out = self.allocate_batch(S)
        stats = torch.zeros((S, 1, _lib.TRACE_STATS), dtype=torch.float64, device=self.device)
        new = BatchState(warm_y=torch.zeros_like(state.warm_y),
                         warm_fixed=torch.zeros((S, max(nf, 1)), dtype=torch.float64, device=self.device),
                         rho=torch.zeros_like(state.rho))
        keep = [self._batch_input(x, (S, n), "x", False),
                self._batch_input(tensions, (S, nca), "tensions", False) if self.cables else None,
                self._batch_input(applied, (S, n), "applied", False),
                self._batch_input(insertion, (S,), "insertion", False)]
        wf = None if state.warm_fixed is None else state.warm_fixed.contiguous()
        keep.append(wf)
        desc = _lib.BatchDesc()
        desc.S = S
        desc.x0 = _lib.ptr(keep[0])
        desc.tensions = _lib.ptr(keep[1]) if self.cables else None
        desc.applied = _lib.ptr(keep[2])
        desc.insertion = _lib.ptr(keep[3])
        desc.warm_y_in = _lib.ptr(state.warm_y)
        desc.warm_fixed_in = _lib.ptr(wf)
        desc.rho_in = _lib.ptr(state.rho)
        for name in ("coords", "status", "frames", "converged", "residual", "n_contacts", "contact_node",
                     "contact_triangle", "contact_gap", "contact_multiplier", "contact_force", "contact_normal",
                     "contact_point"):
            setattr(desc, name, _lib.ptr(getattr(out, name)))
        desc.warm_y_out, desc.warm_fixed_out, desc.rho_out = (_lib.ptr(new.warm_y), _lib.ptr(new.warm_fixed),
                                                              _lib.ptr(new.rho))
        desc.trace_cap, desc.trace_stats = 1, _lib.ptr(stats)
        desc.max_frames, desc.stop_on_tol, desc.tol, desc.fail_on_limit = 1, 0, 0.0, 0
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        self._check(self._lib.accfem_solve_batch(self._h, ctypes.byref(desc), ctypes.c_void_p(st.cuda_stream)))
        out._keep = keep
        if nf == 0:
            new.warm_fixed = None
        else:
            new.warm_fixed = new.warm_fixed[:, :nf]
        return out, stats[:, 0, :], new

    # -- unit entry points ---------------------------------------------------------
    def element_pass(self, x):
        """F_int (S, 6N), K diagonal blocks (S, N, 6, 6), K upper blocks (S, N-1, 6, 6)
        for configurations x (S, 6N) torch CUDA float64 -- internal_force +
        assemble_tangent_stiffness (beam.py:311-356)."""
        import torch

        x = x.contiguous()
        S, N = x.shape[0], self.model.node_count
        f = torch.empty((S, 6 * N), dtype=torch.float64, device=self.device)
        kd = torch.empty((S, N, 6, 6), dtype=torch.float64, device=self.device)
        ku = torch.empty((S, N - 1, 6, 6), dtype=torch.float64, device=self.device)
        fr = torch.empty((S, N - 1, 3, 3), dtype=torch.float64, device=self.device)
        bad = torch.zeros(S, dtype=torch.int32, device=self.device)
        st = torch.cuda.current_stream(self.device)
        self._check(self._lib.accfem_element_pass(self._h, S, x.data_ptr(), f.data_ptr(), kd.data_ptr(),
                                                  ku.data_ptr(), fr.data_ptr(), bad.data_ptr(),
                                                  ctypes.c_void_p(st.cuda_stream)))
        return f, kd, ku, fr, bad

    def detect(self, x):
        """Per-node contact winner for configurations x (S, 6N): triangle id (-1
        none), gap, plane point -- detect_contacts (contact.py:49-120)."""
        import torch

        x = x.contiguous()
        S, N = x.shape[0], self.model.node_count
        tri = torch.empty((S, N), dtype=torch.int32, device=self.device)
        gap = torch.zeros((S, N), dtype=torch.float64, device=self.device)
        pt = torch.zeros((S, N, 3), dtype=torch.float64, device=self.device)
        st = torch.cuda.current_stream(self.device)
        self._check(self._lib.accfem_detect(self._h, S, x.data_ptr(), tri.data_ptr(), gap.data_ptr(),
                                            pt.data_ptr(), ctypes.c_void_p(st.cuda_stream)))
        return tri, gap, pt

