"""Dump golden fixtures from the REAL reference (run in the build container).

    python tests/golden/make_golden.py

/root/reference is read-only and absent on the GPU box, so everything the
parity tests need from the reference is frozen here into small .npz files:

  so3.npz        exp/log/compose of scipy Rotation on edge-case rotation vectors
  beam.npz       F_int and block-tridiagonal K of the reference on perturbed chains
  detect.npz     contact detection on 50 random triangle soups (test_contact.py:113-130
                 recipe, seed 42) and on cfg3 lumen states -- bit-exact fields
  solves.npz     run_static outputs of cfg1/cfg2/cfg3/cfg3p/cfg5 and 16 cfg4 samples
  meshes.npz     the lumen meshes the reference saw (checks the repo's generators)
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from ref_bridge import import_reference, reference_engine, run_reference  # noqa: E402

from paper_2503_06922_b200 import scenarios  # noqa: E402
from paper_2503_06922_b200.scene import MaterialParams, straight_model  # noqa: E402


def so3_cases():
    _, _, _, _, _ = import_reference()
    from cablefem import so3
    rng = np.random.default_rng(3)
    vecs = [np.zeros(3), np.array([1e-9, 0, 0]), np.array([0, 5e-4, 0]), np.array([0, 0, 1e-3]),
            np.array([0, 0, 1.0000001e-3]), np.array([np.pi, 0, 0]), np.array([0, np.pi - 1e-9, 0]),
            np.array([1.0, 2.0, -0.5])]
    vecs += list(rng.normal(size=(40, 3)) * rng.choice([1e-5, 1e-2, 0.5, 2.0], size=(40, 1)))
    v = np.array(vecs)
    mats = so3.exp_so3(v)
    inc = rng.normal(size=v.shape) * 1e-3
    return dict(rotvec=v, exp=mats, log=so3.log_so3(mats), inc=inc, compose=so3.compose_rotvec(inc, v))


def beam_cases():
    beam, _, _, _, _ = import_reference()
    rng = np.random.default_rng(11)
    out = {}
    for tag, nodes, length in (("a", 21, 0.07), ("b", 12, 0.55)):
        mat = beam.MaterialParams(510e6, 5.551e-6, 5.041e-12)
        model = beam.straight_model(nodes, length, mat)
        coords = []
        for k in range(6):
            c = model.rest_configuration.reshape(-1, 6).copy()
            amp = [0.0, 1e-4, 1e-3, 1e-2, 5e-2, 0.3][k]
            c[:, :3] += rng.normal(size=(nodes, 3)) * amp * model.element_rest_length
            c[:, 3:] += rng.normal(size=(nodes, 3)) * amp
            coords.append(c.ravel())
        coords = np.array(coords)
        fint, kd, ku = [], [], []
        for c in coords:
            x = beam.Configuration(c)
            fint.append(beam.internal_force(x, model))
            dense = beam.assemble_tangent_stiffness(x, model).matrix.toarray().reshape(nodes, 6, nodes, 6)
            i = np.arange(nodes)
            kd.append(dense[i, :, i, :])
            ku.append(dense[i[:-1], :, i[:-1] + 1, :])
        out[f"{tag}_nodes"] = nodes
        out[f"{tag}_length"] = length
        out[f"{tag}_coords"] = coords
        out[f"{tag}_fint"] = np.array(fint)
        out[f"{tag}_kd"] = np.array(kd)
        out[f"{tag}_ku"] = np.array(ku)
    return out


def detect_cases():
    beam, _, _, mesh_mod, _ = import_reference()
    from cablefem.contact import detect_contacts
    mat = beam.MaterialParams(510e6, 5.551e-6, 5.041e-12)
    model = beam.straight_model(12, 0.55, mat)
    rng = np.random.default_rng(42)
    verts_all, tri_counts, pos_all, margins = [], [], [], []
    res = []
    for _scene in range(50):
        n_tri = rng.integers(40, 500)
        verts = rng.uniform(-0.4, 0.9, size=(n_tri * 3, 3))
        mesh = mesh_mod.TriangleMesh(verts, np.arange(n_tri * 3).reshape(-1, 3))
        coords = model.rest_configuration.reshape(-1, 6).copy()
        coords[:, :3] += rng.uniform(-0.05, 0.05, size=3)
        x = beam.Configuration(coords.ravel())
        margin = float(rng.uniform(1e-3, 2e-2))
        cs = detect_contacts(x, model, mesh, margin)
        verts_all.append(verts)
        tri_counts.append(n_tri)
        pos_all.append(coords[:, :3])
        margins.append(margin)
        res.append([(c.element_index - 1 if c.xi == 0.0 else c.element_index, c.triangle_id, c.gap,
                     *c.plane_point, *c.normal) for c in cs])
    flat = [(s, *r) for s, rows in enumerate(res) for r in rows]
    arr = np.array(flat, dtype=float)
    return dict(rand_verts=np.concatenate(verts_all), rand_tri_counts=np.array(tri_counts),
                rand_positions=np.array(pos_all), rand_margins=np.array(margins), rand_contacts=arr)


def solve_cases():
    out = {}
    meshes = {}
    for name in ("cfg1", "cfg3p", "cfg3", "cfg2", "cfg5"):
        w = scenarios.CONFIGS[name](1)
        ws = [w]
        if name == "cfg1":
            ws = [scenarios.cfg1(3, seed=1)]
        for w in ws:
            eng = None
            for i in range(w.size):
                t = time.time()
                o = run_reference(w, i, reference_engine(w))
                tag = f"{name}_{i}"
                print(tag, "status", o["status_exc"], "frames", o.get("frames"), "its",
                      o.get("iterations", np.zeros(1)).sum(), "t", round(time.time() - t, 2), flush=True)
                _store(out, tag, o)
            if w.mesh is not None:
                meshes[f"{name}_vertices"] = w.mesh.vertices
                meshes[f"{name}_triangles"] = w.mesh.triangles
                meshes[f"{name}_normals"] = w.mesh.normals
            del eng
    w = scenarios.cfg4(16)
    meshes["cfg4_x0"] = w.x0
    meshes["cfg4_tensions"] = w.tensions
    meshes["cfg4_applied"] = w.applied
    for i in range(w.size):
        o = run_reference(w, i)
        print("cfg4", i, "frames", o.get("frames"), flush=True)
        _store(out, f"cfg4_{i}", o)
    return out, meshes


def _store(out, tag, o):
    if o["status_exc"] is not None:
        from paper_2503_06922_b200.errors import status_from_exception
        out[f"{tag}_status"] = status_from_exception(o["status_exc"])
        return
    out[f"{tag}_status"] = 0
    for key in ("coords", "frames", "iterations", "n_c", "dx_norm", "retried", "residual", "contact_nodes",
                "contact_tris", "contact_gaps", "contact_forces"):
        out[f"{tag}_{key}"] = o[key]
    recs = o["records"]
    out[f"{tag}_frame_coords"] = np.array([r.coords for r in recs[:16]])
    out[f"{tag}_frame_residual"] = np.array([r.residual_norm for r in recs])
    out[f"{tag}_frame_compl_worst"] = np.array([r.complementarity_worst for r in recs])
    out[f"{tag}_frame_max_pen"] = np.array([r.max_penetration for r in recs])
    out[f"{tag}_frame_scale"] = np.array([r.actuation_scale for r in recs])


def main():
    np.savez_compressed(os.path.join(HERE, "so3.npz"), **so3_cases())
    np.savez_compressed(os.path.join(HERE, "beam.npz"), **beam_cases())
    np.savez_compressed(os.path.join(HERE, "detect.npz"), **detect_cases())
    solves, meshes = solve_cases()
    np.savez_compressed(os.path.join(HERE, "solves.npz"), **solves)
    np.savez_compressed(os.path.join(HERE, "meshes.npz"), **meshes)


if __name__ == "__main__":
    main()
