"""Frame mode: Timeline / Trajectory.inputs_at sampling
rules on the CPU (scenario.py:61-77, 143-149), and on the GPU the device
run_scenario (one Engine.step per frame) and the batched lockstep
run_trajectories (one step_batch launch per frame for all trajectories)
against the reference's run_scenario records (tests/golden/make_golden_frames.py)."""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from make_golden_frames import FRAME_SCENES  # noqa: E402

from paper_2503_06922_b200.errors import ScenarioError  # noqa: E402
from paper_2503_06922_b200.frames import Timeline, Trajectory  # noqa: E402


def test_timeline_and_inputs_at_follow_the_reference():
    tl = Timeline([[0.0, 1.0], [1.0, 3.0]])
    assert tl.value(-1.0) == 1.0 and tl.value(0.5) == 2.0 and tl.value(5.0) == 3.0  # clamped ends
    with pytest.raises(ScenarioError):
        Timeline([[0.0, 1.0], [0.0, 2.0]])
    with pytest.raises(ScenarioError):
        Timeline(np.zeros((0, 2)))
    tr = Trajectory(tensions={1: Timeline([[0.0, -0.5], [1.0, 0.5]]), 3: Timeline([[0.0, 0.2]])},
                    insertion_rate=Timeline([[0.0, 0.01], [1.0, 0.03]]), frame_period=0.1, duration=1.0)
    assert tr.n_frames == 10
    inp = tr.inputs_at(0.25)
    assert np.allclose(inp.tensions, [0.0, 0.0, 0.2])  # negative tension clamped, cable 2 absent -> 0
    assert inp.insertion_increment == pytest.approx(0.015 * 0.1)
    with pytest.raises(ScenarioError):
        Trajectory(frame_period=0.0)
    with pytest.raises(ScenarioError):
        Trajectory.from_dict({"robot": {"node_count": 5, "length": 0.1}, "bogus": 1})
    t = Trajectory.from_dict(FRAME_SCENES["tube_a"])
    assert t.engine_kwargs["mesh"].triangle_count > 0 and t.n_frames == 10


def _check(g, tag, coords, n_c, its, retried, dx, tri, force, rows):
    """Frame records vs the reference: counts exact, coords 1e-6, forces 1e-5 (per contact)."""
    assert np.array_equal(n_c[rows], g[f"{tag}_n_c"][rows]), tag
    assert np.array_equal(its[rows], g[f"{tag}_iterations"][rows]), tag
    assert np.array_equal(retried[rows].astype(bool), g[f"{tag}_retried"][rows].astype(bool)), tag
    assert np.array_equal(tri[rows], g[f"{tag}_tri"][rows]), tag
    ref = g[f"{tag}_coords"][rows]
    assert np.abs(coords[rows] - ref).max() <= 1e-6 * np.abs(ref).max(), tag
    gd = g[f"{tag}_dx_norm"][rows]
    assert np.all(np.abs(dx[rows] - gd) <= 1e-6 * gd + 1e-10), tag
    fr = g[f"{tag}_force"][rows]
    err = np.linalg.norm(force[rows] - fr, axis=-1)
    assert np.all(err <= 1e-5 * np.linalg.norm(fr, axis=-1) + 1e-10 * max(np.abs(fr).max(), 1e-30)), tag


def _arrays(recs, N):
    F = len(recs)
    tri = np.full((F, N), -1, np.int32)
    force = np.zeros((F, N, 3))
    for f, r in enumerate(recs):
        for c, fv in zip(r.contact_points, np.asarray(r.contact_force_vectors).reshape(-1, 3)):
            node = c.element_index - 1 if c.xi == 0.0 else c.element_index
            tri[f, node] = c.triangle_id
            force[f, node] = fv
    return (np.array([r.coords for r in recs]), np.array([r.n_c for r in recs]),
            np.array([r.iterations for r in recs]), np.array([r.retried for r in recs]),
            np.array([r.dx_norm for r in recs]), tri, force)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted(FRAME_SCENES))
def test_device_run_scenario_matches_reference(golden, tag):
    from paper_2503_06922_b200.frames import run_scenario
    g = golden("frames.npz")
    traj = Trajectory.from_dict(FRAME_SCENES[tag])
    eng = traj.build_engine(device=0)
    recs = run_scenario(eng, traj)
    assert len(recs) == int(g[f"{tag}_records"])
    N = eng.model.node_count
    _check(g, tag, *_arrays(recs, N), rows=slice(None))


@pytest.mark.gpu
def test_batched_trajectories_match_reference(golden):
    """tube_a and tube_b (one scene, different tension / insertion timelines),
    plus 6 more copies of them, in one lockstep batch."""
    from paper_2503_06922_b200.frames import run_trajectories
    g = golden("frames.npz")
    tags = ["tube_a", "tube_b"] * 4
    trajs = [Trajectory.from_dict(FRAME_SCENES[t]) for t in tags]
    eng = trajs[0].build_engine(device=0)
    out = run_trajectories(eng, trajs, records=True)
    assert np.all(out.status == 0) and np.all(out.frames == 10)
    N = eng.model.node_count
    for s, tag in enumerate(tags):
        _check(g, tag, *_arrays(out.records[s], N), rows=slice(None))


def test_bench_report_writer_matches_reference_format(tmp_path, golden):
    """write_benchmark_outputs produces the reference's JSON and CSV byte for byte
    (bench.py:140-153) on the same result dict."""
    from make_golden_frames import FAKE_RESULT
    from paper_2503_06922_b200.benchreport import BenchmarkConfig, write_benchmark_outputs
    g = golden("frames.npz")
    write_benchmark_outputs(FAKE_RESULT, tmp_path / "r.json")
    assert (tmp_path / "r.csv").read_text() == str(g["writer_csv"])
    assert (tmp_path / "r.json").read_text() == str(g["writer_json"])
    with pytest.raises(Exception):
        BenchmarkConfig(repetitions=0)


@pytest.mark.gpu
def test_device_bench_cells_match_reference(golden, tmp_path):
    """run_cell through the device Engine: achieved contacts, mean ADMM iterations /
    PGS sweeps and max penetration equal the reference's run_cell (bench.py:74-107)."""
    from make_golden_frames import BENCH_CELLS
    from paper_2503_06922_b200.benchreport import (BenchmarkConfig, run_benchmark, run_cell,
                                                   write_benchmark_outputs)
    g = golden("frames.npz")
    for nodes, target, backend in BENCH_CELLS:
        cfg = BenchmarkConfig(node_counts=[nodes], contact_targets=[target], backends=[backend], repetitions=4,
                              warmup_frames=2)
        row = run_cell(nodes, target, backend, cfg, device=0)
        tag = f"cell_{nodes}_{target}_{backend}"
        assert row["achieved_contacts"] == float(g[f"{tag}_achieved"]), tag
        assert row["iters"] == float(g[f"{tag}_iters"]), (tag, row["iters"], float(g[f"{tag}_iters"]))
        assert abs(row["max_penetration"] - float(g[f"{tag}_max_pen"])) <= 1e-6 * float(g[f"{tag}_max_pen"]) + 1e-12
    res = run_benchmark(BenchmarkConfig(node_counts=[41], contact_targets=[8], backends=["accelerated_qp"],
                                        repetitions=2, warmup_frames=1), device=0)
    csv = write_benchmark_outputs(res, tmp_path / "b.json")
    assert csv.read_text().splitlines()[0].startswith("backend,nodes,dof")
