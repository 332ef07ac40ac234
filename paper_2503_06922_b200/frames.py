"""Real-time frame mode on the device.

The reference's frame mode is `run_scenario` (engine.py:300-316): one initial
record (`_initial_record`, engine.py:319-338) and then one `Engine.step` per
frame period with the inputs a `Scenario` samples from its timelines
(`Timeline`, scenario.py:61-77; `Scenario.inputs_at`, scenario.py:143-149):
cable tensions clamped at zero and an insertion increment of
rate(t) * frame_period that the engine applies to the base clamp rows
(engine.py:123-134).

Here:
  Timeline, Trajectory.inputs_at   the same sampling rules
  initial_record(engine, x)        device contact detection at t = 0
  run_scenario(engine, traj)       one trajectory, one Engine.step (device
                                   launch) per frame -- the reference's records
  run_trajectories(engine, trajs)  S trajectories of one scene in lockstep:
                                   one Engine.step_batch launch per frame for
                                   all of them, per-scenario warm state on the
                                   device
  Trajectory.from_dict(raw)        the scenario-file subset that defines a
                                   trajectory (robot, tube mesh, fixed nodes,
                                   tensions, insertion_rate, frame_period,
                                   duration, margin, uniform_load, solver)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ScenarioError, exception_for_status
from .scene import (
    MATERIAL_PRESETS,
    ContactPoint,
    FixedNodeSpec,
    FrameRecord,
    MaterialParams,
    SolverSettings,
    StepInputs,
    default_cables,
    make_tube,
    orient_normals,
    straight_model,
)

_ZERO_TIMINGS = {"stiffness": 0.0, "detection": 0.0, "assembly": 0.0, "solve": 0.0, "update": 0.0, "total": 0.0}


@dataclass
class Timeline:
    """Piecewise-linear samples (times strictly increasing), clamped ends (scenario.py:61-77)."""

    samples: np.ndarray  # (k, 2)

    def __post_init__(self):
        self.samples = np.asarray(self.samples, dtype=float).reshape(-1, 2)
        times = self.samples[:, 0]
        if len(times) == 0:
            raise ScenarioError("timeline needs at least one sample")
        if np.any(np.diff(times) <= 0.0):
            raise ScenarioError("timeline sample times must be strictly increasing")

    def value(self, t):
        return float(np.interp(t, self.samples[:, 0], self.samples[:, 1]))


@dataclass
class Trajectory:
    """Inputs of one frame-mode run: tension timelines of cables 1..3, an
    insertion-rate timeline, the frame period and the duration
    (the input half of the reference's Scenario, scenario.py:80-149)."""

    tensions: dict = field(default_factory=dict)   # cable index (1..3) -> Timeline
    insertion_rate: Timeline = field(default_factory=lambda: Timeline([[0.0, 0.0]]))
    frame_period: float = 1.0 / 30.0
    duration: float = 0.0
    engine_kwargs: dict = field(default_factory=dict)  # scene of Trajectory.from_dict (else the caller's engine)

    def __post_init__(self):
        if self.frame_period <= 0.0:
            raise ScenarioError("frame_period must be positive")
        if self.duration < 0.0:
            raise ScenarioError("duration must be >= 0")
        for j in self.tensions:
            if int(j) not in (1, 2, 3):
                raise ScenarioError(f"cable index {j} out of range 1..3")

    @property
    def n_frames(self):
        """Frames after the initial record (engine.py:309-310)."""
        return int(round(self.duration / self.frame_period)) if self.duration > 0 else 0

    def inputs_at(self, t):
        """StepInputs at time t (scenario.py:143-149)."""
        tensions = np.array([max(self.tensions[j].value(t), 0.0) if j in self.tensions else 0.0
                             for j in (1, 2, 3)])
        rate = self.insertion_rate.value(t)
        return StepInputs(tensions=tensions, insertion_increment=rate * self.frame_period)

    @classmethod
    def from_dict(cls, raw):
        """A trajectory and its scene from the scenario-file subset (scenario.py:35-59,
        96-141, 186-228); unknown top-level keys are rejected like the reference's schema."""
        allowed = {"name", "robot", "mesh", "margin", "fixed_nodes", "insertion_rate", "tensions", "uniform_load",
                   "solver", "frame_period", "duration"}
        extra = set(raw) - allowed
        if extra:
            raise ScenarioError(f"unknown scenario keys {sorted(extra)}")
        try:
            robot = dict(raw["robot"])
        except KeyError as exc:
            raise ScenarioError(f"scenario missing required key: {exc}") from exc
        mat_cfg = robot.get("material", "a")
        if isinstance(mat_cfg, str):
            if mat_cfg not in MATERIAL_PRESETS:
                raise ScenarioError(f"unknown material preset {mat_cfg!r}; presets are {sorted(MATERIAL_PRESETS)}")
            mat_kwargs = dict(MATERIAL_PRESETS[mat_cfg])
        else:
            mat_kwargs = dict(mat_cfg)
        for opt in ("poisson_ratio", "torsion_constant"):
            if robot.get(opt) is not None:
                mat_kwargs[opt] = robot[opt]
        model = straight_model(int(robot["node_count"]), float(robot["length"]), MaterialParams(**mat_kwargs),
                               base=robot.get("base", (0.0, 0.0, 0.0)), axis=robot.get("axis", (1.0, 0.0, 0.0)))
        mesh = None
        mcfg = dict(raw.get("mesh") or {})
        if mcfg:
            if "tube" not in mcfg:
                raise ScenarioError("trajectory meshes are tubes ({'tube': {...}}); load STL/OBJ files with "
                                    "scene.load_mesh and pass engine_kwargs")
            tube = mcfg["tube"]
            mesh = make_tube(tube["path_points"], tube["radii"], segments=int(tube.get("segments", 16)))
            orient_normals(mesh, model.rest_positions)
        specs = [FixedNodeSpec(int(item["node"]), tuple(item.get("dofs", (0, 1, 2, 3, 4, 5))))
                 for item in raw.get("fixed_nodes", [{"node": 0}])]
        try:
            solver = SolverSettings(**dict(raw.get("solver", {})))
        except TypeError as exc:
            raise ScenarioError(f"bad solver settings: {exc}") from exc
        uniform = raw.get("uniform_load")
        kwargs = dict(model=model, mesh=mesh, cables=default_cables(radius=float(robot.get("cable_radius", 0.004))),
                      fixed_specs=specs, settings=solver, margin=float(raw.get("margin", 1e-4)),
                      uniform_load=None if uniform is None else np.asarray(uniform, dtype=float))
        tensions = {int(k): Timeline(v) for k, v in dict(raw.get("tensions", {})).items()}
        return cls(tensions=tensions, insertion_rate=Timeline(raw.get("insertion_rate", [[0.0, 0.0]])),
                   frame_period=float(raw.get("frame_period", 1.0 / 30.0)), duration=float(raw.get("duration", 0.0)),
                   engine_kwargs=kwargs)

    def build_engine(self, device=None):
        from .engine import Engine
        if not self.engine_kwargs:
            raise ScenarioError("this trajectory carries no scene (construct it with from_dict)")
        return Engine(**self.engine_kwargs, device=device)


def initial_record(engine, x):
    """The t = 0 record (engine.py:319-338): contacts detected on the device with
    query radius margin + beta0, no solve."""
    contacts = []
    if engine.mesh is not None:
        import torch
        tri, gap, pt = engine.detect(torch.tensor(x.coords.reshape(1, -1), device=engine.device))
        tri, gap, pt = tri.cpu().numpy()[0], gap.cpu().numpy()[0], pt.cpu().numpy()[0]
        nodes = np.flatnonzero(tri >= 0)
        contacts = engine._contact_points(nodes, tri[nodes], gap[nodes], pt[nodes])
    return FrameRecord(
        t=0.0, frame_index=0, coords=x.coords.copy(), n_c=len(contacts),
        contact_force_vectors=np.zeros((len(contacts), 3)), contact_points=contacts,
        tip_position=x.positions()[-1].copy(), dx_norm=0.0, iterations=0, converged=True, retried=False,
        actuation_scale=1.0, max_penetration=max(0.0, -min((c.gap for c in contacts), default=0.0)),
        complementarity_ok=True, complementarity_worst=0.0, residual_norm=0.0, timings_ms=dict(_ZERO_TIMINGS))


def run_scenario(engine, traj):
    """Frame mode (engine.py:300-316): the initial record plus one Engine.step
    per frame period; raises the reference's exception class on a device failure."""
    x = engine.initial_configuration()
    records = [initial_record(engine, x)]
    for k in range(1, traj.n_frames + 1):
        t = k * traj.frame_period
        x, rec = engine.step(x, traj.inputs_at(t), t=t, frame_index=k)
        records.append(rec)
    return records


@dataclass
class TrajectoryBatch:
    """Outputs of run_trajectories for S trajectories of F = max frames:
    per-frame stats (S, F, 14) in the ACCFEM_TRACE_STATS layout, coords
    (S, F, 6N), contact triangle per node (S, F, N; -1 none), status (S) and the
    number of frames each trajectory completed (S)."""

    stats: np.ndarray
    coords: np.ndarray
    contact_triangle: np.ndarray
    status: np.ndarray
    frames: np.ndarray
    records: list = None  # per trajectory: [FrameRecord] (initial record first), if requested


def run_trajectories(engine, trajs, records=False):
    """S trajectories of the engine's scene in lockstep (the batched real-time
    mode): frame k of every trajectory is one Engine.step_batch launch with
    per-trajectory tensions and insertion increments sampled from its
    timelines; warm multipliers and rho persist per trajectory on the device.
    A trajectory whose step fails keeps its status and stops advancing (the
    reference's run_scenario would raise there)."""
    import torch

    S = len(trajs)
    N, n = engine.model.node_count, engine.model.dof_count
    F = max(t.n_frames for t in trajs) if S else 0
    dev = engine.device
    x = torch.tensor(np.tile(engine.model.rest_configuration, (S, 1)), device=dev)
    state = None
    stats = np.zeros((S, F, _lib.TRACE_STATS))
    coords = np.zeros((S, F, n))
    ctri = np.full((S, F, N), -1, np.int32)
    status = np.zeros(S, np.int32)
    done = np.zeros(S, np.int32)
    recs = [[initial_record(engine, engine.initial_configuration())] for _ in range(S)] if records else None
    for k in range(1, F + 1):
        inp = [t.inputs_at(k * t.frame_period) for t in trajs]
        ten = torch.tensor(np.array([i.tensions for i in inp]), device=dev) if engine.cables else None
        ins = torch.tensor([i.insertion_increment for i in inp], dtype=torch.float64, device=dev)
        out, st, new_state = engine.step_batch(x, ten, None, ins, state)
        r = out.to_numpy()
        st = st.cpu().numpy()
        live = (status == 0) & (np.array([k <= t.n_frames for t in trajs]))
        ok = live & (r.status == 0)
        status[live & (r.status != 0)] = r.status[live & (r.status != 0)]
        # trajectories that failed or finished keep their last state
        keep = torch.tensor(~ok, device=dev)
        x = torch.where(keep[:, None], x, out.coords)
        if state is None:
            state = new_state
        else:
            state.warm_y = torch.where(keep[:, None], state.warm_y, new_state.warm_y)
            state.rho = torch.where(keep, state.rho, new_state.rho)
            if new_state.warm_fixed is not None:
                state.warm_fixed = new_state.warm_fixed if state.warm_fixed is None else \
                    torch.where(keep[:, None], state.warm_fixed, new_state.warm_fixed)
        for s in np.flatnonzero(ok):
            stats[s, k - 1] = st[s]
            coords[s, k - 1] = r.coords[s]
            nc = int(r.n_contacts[s])
            ctri[s, k - 1, r.contact_node[s, :nc]] = r.contact_triangle[s, :nc]
            done[s] = k
            if records:
                cps = engine._contact_points(r.contact_node[s, :nc], r.contact_triangle[s, :nc],
                                             r.contact_gap[s, :nc], r.contact_point[s, :nc]) if nc else []
                t = k * trajs[s].frame_period
                recs[s].append(FrameRecord(
                    t=t, frame_index=k, coords=r.coords[s].copy(), n_c=nc,
                    contact_force_vectors=r.contact_force[s, :nc].copy(), contact_points=cps,
                    tip_position=r.coords[s].reshape(-1, 6)[-1, :3].copy(), dx_norm=float(st[s, 0]),
                    iterations=int(st[s, 5]), converged=bool(st[s, 7]), retried=bool(st[s, 8]),
                    actuation_scale=float(st[s, 1]), max_penetration=float(st[s, 2]),
                    complementarity_ok=bool(st[s, 9]), complementarity_worst=float(st[s, 3]),
                    residual_norm=float(st[s, 4]), timings_ms=dict(_ZERO_TIMINGS)))
    return TrajectoryBatch(stats=stats, coords=coords, contact_triangle=ctri, status=status, frames=done,
                           records=recs)


def raise_for(batch, s):
    """The reference's exception for trajectory s of a TrajectoryBatch (None if it completed)."""
    st = int(batch.status[s])
    if st == 0:
        return None
    return exception_for_status(st, f"trajectory {s}: frame {int(batch.frames[s]) + 1} failed (status {st})")


__all__ = ["Timeline", "Trajectory", "TrajectoryBatch", "initial_record", "run_scenario", "run_trajectories",
           "raise_for", "ContactPoint"]
