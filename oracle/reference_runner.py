"""CPU REFERENCE RUNNER -- measurement infrastructure only, never on the product path.

Runs the UNMODIFIED reference package (`cablefem`, pip-installed into
`baseline/_ref` by `python -m pip install --no-index --no-build-isolation
--find-links /opt/wheelhouse --target baseline/_ref --no-deps <copy of
/root/reference/pkg>`; git-ignored, shipped to the GPU box with the repo
snapshot) through its own public API: `Engine(...).run_static(...)`
(engine.py:267-283).  Only `bench.py`'s cpu_baseline / `--impl reference` legs
and tests use it.  When baseline/_ref is absent the callers fall back to the
numpy restatement (`oracle/accfem_oracle.py`, kind "port").
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def available():
    return os.path.isdir(os.path.join(REF, "cablefem"))


def _import():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from cablefem import beam, constraints, engine, mesh, solver  # noqa: F401
    return beam, constraints, engine, mesh, solver


def reference_engine(w):
    """The reference Engine of a repo Workload's scene (same data, reference classes)."""
    beam, constraints, engine, mesh_mod, solver = _import()
    m = w.model
    mat = beam.MaterialParams(m.material.young_modulus, m.material.cross_section_area, m.material.bending_inertia,
                              m.material.poisson_ratio, m.material.torsion_constant)
    model = beam.RobotModel(m.node_count, m.element_rest_length, m.rest_configuration.copy(), mat)
    ref_mesh = None
    if w.mesh is not None:
        ref_mesh = mesh_mod.TriangleMesh(w.mesh.vertices.copy(), w.mesh.triangles.copy())
        ref_mesh.normals = w.mesh.normals.copy()
    cables = [constraints.CableSpec(c.cable_index, c.attachment_offset.copy(), c.tension_direction.copy())
              for c in w.cables]
    fixed = [constraints.FixedNodeSpec(f.node_index, tuple(f.fixed_dofs), tuple(f.prescribed_increment))
             for f in w.fixed_specs]
    s = w.settings
    settings = solver.SolverSettings(eps_abs=s.eps_abs, eps_rel=s.eps_rel, max_iterations=s.max_iterations,
                                     rho=s.rho, sigma=s.sigma, alpha=s.alpha, beta0=s.beta0,
                                     check_interval=s.check_interval, adaptive_rho=s.adaptive_rho,
                                     scaling_iterations=s.scaling_iterations, polish=s.polish, backend=s.backend,
                                     pgs_tol=s.pgs_tol, pgs_min_sweep_factor=s.pgs_min_sweep_factor)
    return engine.Engine(model, mesh=ref_mesh, cables=cables, fixed_specs=fixed, settings=settings,
                         margin=w.margin, uniform_load=w.uniform_load)


def run_static(w, i, eng=None):
    """One reference run_static of scenario i of w; returns a status code
    (0 ok, else the errors.py class mapped as in include/accfem.h)."""
    beam, _, engine, _, _ = _import()
    eng = reference_engine(w) if eng is None else eng
    x0 = beam.Configuration(w.x0[i].copy())
    inputs = engine.StepInputs(tensions=None if w.tensions is None else w.tensions[i].copy(),
                               applied_force=None if w.applied is None else w.applied[i].copy())
    try:
        eng.run_static(inputs, x0=x0, tol=w.tol, max_frames=w.max_frames)
    except Exception as exc:  # noqa: BLE001 - the status is the measurement
        name = type(exc).__name__
        if name == "EngineError":
            return 7 if "static mode" in str(exc) else 6
        return {"DomainError": 1, "DegenerateElementError": 2, "MeshError": 3, "NonConvergenceError": 4,
                "InfeasibleError": 5}.get(name, -1)
    return 0
