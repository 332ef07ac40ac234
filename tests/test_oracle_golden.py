"""Pin the CPU oracle (oracle/accfem_oracle.py) against fixtures dumped from
the real reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import accfem_oracle as O
from paper_2503_06922_b200 import scenarios
from paper_2503_06922_b200.scene import MaterialParams, TriangleMesh, straight_model


def test_so3_matches_reference(golden):
    g = golden("so3.npz")
    assert np.array_equal(O.rot_exp(g["rotvec"]), g["exp"])
    assert np.array_equal(O.rot_log(g["exp"]), g["log"])
    assert np.array_equal(O.rot_compose(g["inc"], g["rotvec"]), g["compose"])


@pytest.mark.parametrize("tag", ["a", "b"])
def test_element_pass_matches_reference(golden, tag):
    g = golden("beam.npz")
    model = straight_model(int(g[f"{tag}_nodes"]), float(g[f"{tag}_length"]),
                           MaterialParams(510e6, 5.551e-6, 5.041e-12))
    cm = O.ChainModel(model)
    for c, f_ref, kd_ref, ku_ref in zip(g[f"{tag}_coords"], g[f"{tag}_fint"], g[f"{tag}_kd"], g[f"{tag}_ku"]):
        assert np.array_equal(O.internal_force(cm, c), f_ref)
        kd, ku = O.block_tridiagonal(O.tangent_matrix(cm, O.chain_state(cm, c)[2]), cm.N)
        assert np.array_equal(kd, kd_ref) and np.array_equal(ku, ku_ref)


def test_detection_matches_reference_bit_exact(golden):
    g = golden("detect.npz")
    verts = g["rand_verts"]
    counts = g["rand_tri_counts"]
    ref = g["rand_contacts"]
    start = 0
    for s, n_tri in enumerate(counts):
        v = verts[start:start + 3 * n_tri]
        start += 3 * n_tri
        lum = O.Lumen(TriangleMesh(v, np.arange(3 * n_tri).reshape(-1, 3)))
        m = float(g["rand_margins"][s])
        got = O.detect(lum, g["rand_positions"][s], m, m)
        want = ref[ref[:, 0] == s]
        assert len(got) == len(want)
        for c, r in zip(got, want):
            assert c[0] == r[1] and c[1] == r[2] and c[2] == r[3]
            assert np.array_equal(c[3], r[4:7]) and np.array_equal(c[4], r[7:10])


def test_generators_match_reference_meshes(golden):
    g = golden("meshes.npz")
    for name in ("cfg2", "cfg3", "cfg3p", "cfg5"):
        w = scenarios.CONFIGS[name](1)
        assert np.array_equal(w.mesh.vertices, g[f"{name}_vertices"]), name
        assert np.array_equal(w.mesh.triangles, g[f"{name}_triangles"]), name
        assert np.array_equal(w.mesh.normals, g[f"{name}_normals"]), name
    w = scenarios.cfg4(16)
    assert np.array_equal(w.x0, g["cfg4_x0"])
    assert np.array_equal(w.tensions, g["cfg4_tensions"])
    assert np.array_equal(w.applied, g["cfg4_applied"])


def compare_solve(g, tag, got):
    assert got["status"] == int(g[f"{tag}_status"]), tag
    if got["status"] != 0:
        return
    assert got["frames"] == int(g[f"{tag}_frames"]), tag
    assert np.array_equal(got["iterations"], g[f"{tag}_iterations"]), tag
    assert np.array_equal(got["n_c"], g[f"{tag}_n_c"]), tag
    assert np.array_equal(got["contact_nodes"], g[f"{tag}_contact_nodes"]), tag
    assert np.array_equal(got["contact_tris"], g[f"{tag}_contact_tris"]), tag
    ref = g[f"{tag}_coords"]
    assert np.max(np.abs(got["coords"] - ref)) <= 1e-6 * np.max(np.abs(ref)), tag
    fr = g[f"{tag}_contact_forces"]
    if fr.size:
        assert np.max(np.abs(got["contact_forces"] - fr)) <= 1e-5 * max(np.max(np.abs(fr)), 1e-12), tag


@pytest.mark.parametrize("name", ["cfg1", "cfg3p", "cfg3", "cfg5"])
def test_oracle_solves_match_reference(golden, name):
    g = golden("solves.npz")
    w = scenarios.cfg1(3, seed=1) if name == "cfg1" else scenarios.CONFIGS[name](1)
    for i, got in enumerate(O.solve_workload(w)):
        compare_solve(g, f"{name}_{i}", got)


@pytest.mark.slow
def test_oracle_cfg2_matches_reference(golden):
    g = golden("solves.npz")
    compare_solve(g, "cfg2_0", O.solve_workload(scenarios.cfg2(1))[0])


def test_oracle_cfg4_samples_match_reference(golden):
    g = golden("solves.npz")
    w = scenarios.cfg4(16)
    for i, got in enumerate(O.solve_workload(w, indices=range(0, 16, 3))):
        compare_solve(g, f"cfg4_{3 * i}", got)


def test_reference_runner_matches_reference_status_and_frames(golden):
    """oracle/reference_runner.py (the bench's CPU arm) drives the unmodified reference
    from baseline/_ref: cfg3p solves (status 0) and the infeasible press reports status 5."""
    import pytest
    from oracle import reference_runner
    from paper_2503_06922_b200 import scenarios
    if not reference_runner.available():
        pytest.skip("baseline/_ref not installed")
    assert reference_runner.run_static(scenarios.cfg3p(1), 0) == 0
    assert reference_runner.run_static(scenarios.infeasible_press(1), 0) == 5
