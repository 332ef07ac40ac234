"""Build reference (`cablefem`) objects from a repo Workload.

Only used in THIS container to generate golden fixtures from the real
reference (/root/reference is absent on the GPU box).  The reference is
imported in place, read-only.
"""

import os
import sys

import numpy as np

REF_SRC = os.environ.get("ACCFEM_REFERENCE_SRC", "/root/reference/pkg/src")


def import_reference():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import cablefem  # noqa: F401
    from cablefem import beam, constraints, engine, mesh, solver
    return beam, constraints, engine, mesh, solver


def reference_engine(w):
    beam, constraints, engine, mesh_mod, solver = import_reference()
    m = w.model
    mat = beam.MaterialParams(m.material.young_modulus, m.material.cross_section_area,
                              m.material.bending_inertia, m.material.poisson_ratio,
                              m.material.torsion_constant)
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
                                     scaling_iterations=s.scaling_iterations, polish=s.polish,
                                     backend=s.backend, pgs_tol=s.pgs_tol,
                                     pgs_min_sweep_factor=s.pgs_min_sweep_factor)
    return engine.Engine(model, mesh=ref_mesh, cables=cables, fixed_specs=fixed, settings=settings,
                         margin=w.margin, uniform_load=w.uniform_load)


def reference_inputs(w, i):
    _, _, engine, _, _ = import_reference()
    return engine.StepInputs(tensions=None if w.tensions is None else w.tensions[i].copy(),
                             applied_force=None if w.applied is None else w.applied[i].copy())


def run_reference(w, i, engine=None):
    """run_static of scenario i; returns a dict of outputs (status included)."""
    beam, _, eng_mod, _, _ = import_reference()
    eng = reference_engine(w) if engine is None else engine
    x0 = beam.Configuration(w.x0[i].copy())
    out = {"status_exc": None}
    try:
        x, recs, resid = eng.run_static(reference_inputs(w, i), x0=x0, tol=w.tol, max_frames=w.max_frames)
    except Exception as exc:  # noqa: BLE001 - status is part of parity
        out["status_exc"] = exc
        return out
    last = recs[-1]
    out.update(
        coords=x.coords.copy(), frames=len(recs),
        iterations=np.array([r.iterations for r in recs], dtype=np.int32),
        n_c=np.array([r.n_c for r in recs], dtype=np.int32),
        dx_norm=np.array([r.dx_norm for r in recs]),
        retried=np.array([r.retried for r in recs]),
        residual=float(resid),
        contact_nodes=np.array([eng_mod.contact_node(c) for c in last.contact_points], dtype=np.int32),
        contact_tris=np.array([c.triangle_id for c in last.contact_points], dtype=np.int32),
        contact_gaps=np.array([c.gap for c in last.contact_points]),
        contact_forces=np.asarray(last.contact_force_vectors).reshape(-1, 3),
        records=recs,
    )
    return out
