"""Workload generators for the BASELINE.json configs.

Every config is one shared scene (robot model, lumen mesh, clamps, cables,
settings) plus per-scenario inputs (x0, cable tensions, applied nodal load).
The batch path (`Engine.solve_static_batch`) consumes exactly these arrays;
the CPU oracle consumes the same arrays scenario by scenario.

  cfg1  cantilever, 20 elements, cable tip wrench, no contact
  cfg2  50 elements in a straight tube (18-segment flat-bottom lumen)
  cfg3  100 elements in the lumen mesh, ~20 contacts            (headline)
  cfg3p 100 elements on the constriction floor (reference bench.py:51-71)
  cfg4  batch of cfg3 samples: tensions, load scale, insertion offset
  cfg5  1000 elements on the constriction floor, 200 contacts
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from .scene import (
    FixedNodeSpec,
    MATERIAL_PRESETS,
    MaterialParams,
    SolverSettings,
    default_cables,
    make_rectangle,
    make_tube,
    orient_normals,
    straight_model,
)

CFG4_SEED = 20261018
CFG4_TOTAL = 65536


@dataclass
class Workload:
    """A shared scene plus a batch of per-scenario inputs."""

    name: str
    model: object
    mesh: object
    fixed_specs: list
    cables: list
    settings: SolverSettings
    margin: float
    x0: np.ndarray            # (S, 6N)
    tensions: np.ndarray      # (S, n_cables) or None
    applied: np.ndarray       # (S, 6N) or None
    max_frames: int = 5000
    tol: float = 1e-9
    uniform_load: np.ndarray = None
    meta: dict = field(default_factory=dict)

    @property
    def size(self):
        return self.x0.shape[0]

    def engine_kwargs(self):
        return dict(model=self.model, mesh=self.mesh, cables=self.cables,
                    fixed_specs=self.fixed_specs, settings=self.settings,
                    margin=self.margin, uniform_load=self.uniform_load)

    def subset(self, idx):
        idx = np.atleast_1d(np.asarray(idx))
        return Workload(self.name, self.model, self.mesh, self.fixed_specs, self.cables,
                        self.settings, self.margin, self.x0[idx],
                        None if self.tensions is None else self.tensions[idx],
                        None if self.applied is None else self.applied[idx],
                        self.max_frames, self.tol, self.uniform_load, dict(self.meta))


def material_a():
    return MaterialParams(**MATERIAL_PRESETS["a"])


def lumen_mesh(model, constriction_node, segments=18, radius=3.6e-3, floor_drop=4e-5,
               extra_length=0.0):
    """Straight tube whose flat bottom facet sits `floor_drop` below the rest
    line, widening and falling away beyond the constriction node."""
    length = model.total_length
    l0 = model.element_rest_length
    xs = np.arange(-0.01, length + 0.05 + extra_length, 0.005)
    xc = (constriction_node + 0.49) * l0
    past = np.maximum(xs - xc, 0.0)
    r = radius + 0.1 * past
    z = -floor_drop - 0.05 * past + r * np.cos(np.pi / segments)
    path = np.stack([xs, np.zeros_like(xs), z], axis=1)
    mesh = make_tube(path, r, segments=segments)
    orient_normals(mesh, model.rest_positions)
    return mesh


def _press_load(model, nodes, per_node):
    f = np.zeros(model.dof_count)
    f.reshape(-1, 6)[nodes, 2] = -per_node
    return f


def cfg1(n_scenarios=1, seed=1):
    """Cantilever, 20 elements, tensions T_j ~ U[0, 1] N, no contact."""
    model = straight_model(21, 0.07, material_a())
    rng = np.random.default_rng(seed)
    tensions = rng.uniform(0.0, 1.0, size=(n_scenarios, 3))
    x0 = np.tile(model.rest_configuration, (n_scenarios, 1))
    return Workload("cfg1", model, None, [FixedNodeSpec(0)], default_cables(0.004),
                    SolverSettings(), 1e-4, x0, tensions, None, max_frames=5000)


def cfg_tube(node_count, length, loaded, name, n_scenarios=1, max_frames=400):
    model = straight_model(node_count, length, material_a())
    mesh = lumen_mesh(model, loaded)
    applied = np.tile(_press_load(model, np.arange(1, loaded + 1), 0.02), (n_scenarios, 1))
    tensions = np.tile([0.01, 0.0, 0.0], (n_scenarios, 1))
    x0 = np.tile(model.rest_configuration, (n_scenarios, 1))
    return Workload(name, model, mesh, [FixedNodeSpec(0)], default_cables(0.004),
                    SolverSettings(), 1e-4, x0, tensions, applied, max_frames=max_frames)


def cfg2(n_scenarios=1):
    """50 elements in a straight tube, load on nodes 1..8."""
    return cfg_tube(51, 0.235, 8, "cfg2", n_scenarios)


def cfg3(n_scenarios=1):
    """100 elements in the lumen mesh, load on nodes 1..20 (~20 contacts)."""
    return cfg_tube(101, 0.47, 20, "cfg3", n_scenarios)


def constriction(node_count, target, name, n_scenarios=1, load_per_node=0.02, margin=1e-4, length=None):
    """Floor strip under the loaded nodes (reference bench.py:51-71).
    `length` overrides the bench's constant-l0 length (0.47 m per 100 nodes)."""
    total = 0.47 * node_count / 100.0 if length is None else float(length)
    model = straight_model(node_count, total, material_a())
    l0 = model.element_rest_length
    loaded = np.arange(1, target + 1)
    x_lo = loaded[0] * l0 - 0.49 * l0
    x_hi = loaded[-1] * l0 + 0.49 * l0
    floor = make_rectangle(((x_lo + x_hi) / 2.0, 0.0, -0.4 * margin), x_hi - x_lo, 1.0, normal_axis="z")
    applied = np.tile(_press_load(model, loaded, load_per_node), (n_scenarios, 1))
    x0 = np.tile(model.rest_configuration, (n_scenarios, 1))
    return Workload(name, model, floor, [FixedNodeSpec(0)], [], SolverSettings(), margin,
                    x0, None, applied, max_frames=5000)


def cfg3p(n_scenarios=1):
    return constriction(101, 20, "cfg3p", n_scenarios)


def cfg5(n_scenarios=1, target=200):
    return constriction(1001, target, "cfg5", n_scenarios)


@lru_cache(maxsize=4)
def _cfg4_table(seed, table):
    """(tensions, load scale, insertion offset) of every scenario of the batch."""
    l0 = 0.47 / 100
    rng = np.random.default_rng(seed)
    tensions = rng.uniform(0.0, 0.02, size=(table, 3))
    scale = rng.uniform(1.0, 1.5, size=table)
    offset = rng.uniform(0.0, 2.0 * l0, size=table)
    return tensions, scale, offset


@lru_cache(maxsize=1)
def _cfg3_scene():
    return cfg3(1)


def cfg4(n_scenarios=65536, seed=CFG4_SEED, start=0):
    """Batch of cfg3 samples: T_j ~ U[0, 0.02] N, load scale ~ U[1, 1.5],
    insertion offset ~ U[0, 2 l0] along the lumen axis (encoded in x0).

    Samples are drawn for indices [0, start + n_scenarios) and sliced, so any
    shard [start, start + n) of the 65,536-scenario batch is reproducible on
    its own rank.
    """
    base = _cfg3_scene()
    model = base.model
    # one fixed table for the whole 65,536-scenario batch, so any shard
    # [start, start + n) is identical on every rank and in every call
    table = CFG4_TOTAL if start + n_scenarios <= CFG4_TOTAL else start + n_scenarios
    t_all, s_all, o_all = _cfg4_table(seed, table)
    tensions = t_all[start:start + n_scenarios].copy()
    scale = s_all[start:start + n_scenarios]
    offset = o_all[start:start + n_scenarios]
    unit = _press_load(model, np.arange(1, 21), 0.02)
    applied = scale[:, None] * unit[None, :]
    x0 = np.tile(model.rest_configuration, (n_scenarios, 1))
    x0.reshape(n_scenarios, -1, 6)[:, :, 0] += offset[:, None]
    return Workload("cfg4", model, base.mesh, base.fixed_specs, base.cables, base.settings,
                    base.margin, x0, tensions, applied, max_frames=400,
                    meta={"seed": seed, "start": start})


def cfg5_fine(n_scenarios=1):
    """cfg5's fine discretisation (L = 0.47 m, l0 = 0.47 mm): the reference's
    ADMM stalls and the frame fails twice -> EngineError at frame 0
    (SURVEY Appendix C).  A parity case of failure, not a throughput config."""
    return constriction(1001, 200, "cfg5_fine", n_scenarios, length=0.47)


def infeasible_press(n_scenarios=1, push=1e-3):
    """Base node clamped with a prescribed increment `push` m INTO a floor it
    already touches: the selector row contradicts the node's contact row, so
    ADMM's certificate test (solver.py:424-446) raises InfeasibleError."""
    model = straight_model(21, 0.07, material_a())
    l0 = model.element_rest_length
    margin = 1e-4
    floor = make_rectangle((0.0, 0.0, -0.4 * margin), 0.98 * l0, 1.0, normal_axis="z")
    applied = None
    x0 = np.tile(model.rest_configuration, (n_scenarios, 1))
    fixed = [FixedNodeSpec(0, prescribed_increment=(0.0, 0.0, -push, 0.0, 0.0, 0.0))]
    return Workload("infeasible", model, floor, fixed, [], SolverSettings(), margin, x0, None, applied,
                    max_frames=50)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg3p": cfg3p, "cfg4": cfg4, "cfg5": cfg5}
