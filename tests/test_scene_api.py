"""Host-side scene API: validation rules mirror the reference, generators
match it, trajectory CSV format."""

import numpy as np
import pytest

from paper_2503_06922_b200 import (
    DomainError,
    FixedNodeSpec,
    MaterialParams,
    MeshError,
    SolverSettings,
    TriangleMesh,
    default_cables,
    make_rectangle,
    straight_model,
)
from paper_2503_06922_b200.outputs import write_trajectory_csv
from paper_2503_06922_b200.scene import FrameRecord, fixed_rows, rotvec_to_matrix


def test_material_and_model_validation():
    with pytest.raises(DomainError):
        MaterialParams(-1.0, 1.0, 1.0)
    m = MaterialParams(510e6, 5.551e-6, 5.041e-12)
    assert m.torsion_constant == 2 * m.bending_inertia
    with pytest.raises(DomainError):
        straight_model(1, 0.1, m)
    model = straight_model(21, 0.07, m)
    assert model.dof_count == 126 and abs(model.element_rest_length - 0.0035) < 1e-15


def test_fixed_rows_and_duplicates():
    rows = fixed_rows([FixedNodeSpec(0), FixedNodeSpec(3, (0, 2), (1e-3, 0.0))], 5)
    assert len(rows) == 8 and rows[6] == (3, 0, 1e-3)
    with pytest.raises(DomainError):
        fixed_rows([FixedNodeSpec(0), FixedNodeSpec(0, (1,))], 5)
    with pytest.raises(DomainError):
        fixed_rows([FixedNodeSpec(7)], 5)


def test_settings_backend_and_mesh_validation():
    assert SolverSettings(backend="pgs_baseline").backend == "pgs_baseline"  # device PGS (§8(f) rank 3)
    with pytest.raises(DomainError):
        SolverSettings(backend="active_set_oracle")  # CPU test oracle only
    with pytest.raises(DomainError):
        SolverSettings(alpha=2.5)
    with pytest.raises(MeshError):
        TriangleMesh(np.zeros((3, 3)), np.array([[0, 1, 2]]))
    r = make_rectangle((0, 0, 0), 1.0, 1.0)
    assert np.allclose(r.normals, [[0, 0, 1], [0, 0, 1]])


def test_cables_and_rotvec():
    cab = default_cables(0.004)
    assert len(cab) == 3 and np.allclose(cab[0].attachment_offset, [0, 0.004, 0])
    R = rotvec_to_matrix(np.array([0.0, 0.0, np.pi / 2]))
    assert np.allclose(R @ [1, 0, 0], [0, 1, 0], atol=1e-15)


def test_trajectory_csv(tmp_path):
    coords = np.zeros(12)
    rec = FrameRecord(t=0.1, frame_index=1, coords=coords, n_c=0, contact_force_vectors=np.zeros((0, 3)),
                      contact_points=[], tip_position=np.zeros(3), dx_norm=0.0, iterations=7, converged=True,
                      retried=False, actuation_scale=1.0, max_penetration=0.0, complementarity_ok=True,
                      complementarity_worst=0.0, residual_norm=0.0, timings_ms={"solve": 1.0, "total": 1.0})
    p = write_trajectory_csv(tmp_path / "t.csv", "demo", [rec, rec], node_count=2)
    lines = p.read_text().splitlines()
    assert lines[7].startswith("t,node0_x") and lines[8].endswith(",0.0,7")
    assert p.read_text() == write_trajectory_csv(tmp_path / "u.csv", "demo", [rec, rec], 2).read_text()


def test_load_mesh_matches_reference_loader(tmp_path):
    """Binary STL, ASCII STL and OBJ give the reference loader's indexed mesh
    (vertex order, triangles, normals) -- the reference from baseline/_ref."""
    import os
    import sys
    ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "cablefem")):
        pytest.skip("baseline/_ref not installed")
    sys.path.insert(0, ref_dir)
    from cablefem import mesh as rm

    from paper_2503_06922_b200.scene import load_mesh, make_tube
    x = np.linspace(0.0, 0.1, 15)
    m = make_tube(np.stack([x, 0 * x, 0.001 * np.sin(30 * x)], 1), 0.003 + 0 * x, segments=10)
    rm.save_stl(rm.TriangleMesh(m.vertices.copy(), m.triangles.copy()), tmp_path / "b.stl")
    with open(tmp_path / "a.stl", "w") as f:
        f.write("solid s\n")
        for t in m.triangles:
            f.write(" facet normal 0 0 1\n  outer loop\n")
            for v in m.vertices[t]:
                f.write(f"   vertex {v[0]:.9e} {v[1]:.9e} {v[2]:.9e}\n")
            f.write("  endloop\n endfacet\n")
        f.write("endsolid s\n")
    with open(tmp_path / "c.obj", "w") as f:
        for v in m.vertices:
            f.write(f"v {float(v[0])!r} {float(v[1])!r} {float(v[2])!r}\n")
        for t in m.triangles:
            f.write(f"f {t[0] + 1}/1 {t[1] + 1} {t[2] + 1}\n")
    for name in ("b.stl", "a.stl", "c.obj"):
        r, o = rm.load_mesh(tmp_path / name), load_mesh(tmp_path / name)
        assert np.array_equal(r.vertices, o.vertices) and np.array_equal(r.triangles, o.triangles), name
        assert np.allclose(r.normals, o.normals), name
    (tmp_path / "q.obj").write_text("v 0 0 0\nf 1 2 3 4\n")
    with pytest.raises(MeshError):
        load_mesh(tmp_path / "q.obj")
    with pytest.raises(MeshError):
        load_mesh(tmp_path / "missing.stl")
