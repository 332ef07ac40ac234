"""Dump frame-mode golden fixtures from the REAL reference: `run_scenario`
(engine.py:300-316) on scenario dicts parsed by the reference's own
`parse_scenario` (scenario.py:186-228).

    python tests/golden/make_golden_frames.py      (build container only)

Writes tests/golden/frames.npz: per scenario the record count, and per record
coords, n_c, iterations, retried, dx_norm, contact triangles (-1 padded),
contact forces.  The scenario dicts are FRAME_SCENES below (also imported by
the GPU tests, which build the same scenes with Trajectory.from_dict).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def _tube(n_pts=24, r=0.0036):
    xs = np.linspace(-0.02, 0.11, n_pts)
    return {"path_points": [[float(x), 0.0, 0.00005 + r * np.cos(np.pi / 18)] for x in xs],
            "radii": [r] * n_pts, "segments": 18}


_TUBE_SCENE = {"robot": {"node_count": 21, "length": 0.07, "material": "a"}, "mesh": {"tube": _tube()},
               "uniform_load": [0.0, 0.0, -0.002], "frame_period": 0.03, "duration": 0.3}

FRAME_SCENES = {
    "ramp": {"name": "ramp", "robot": {"node_count": 21, "length": 0.07, "material": "a"},
             "tensions": {"1": [[0.0, 0.0], [0.2, 0.3]], "2": [[0.0, 0.0], [0.2, 0.1]]},
             "insertion_rate": [[0.0, 0.0], [0.1, 0.01]], "frame_period": 0.02, "duration": 0.2},
    "tube_a": dict(_TUBE_SCENE, name="tube_a", tensions={"1": [[0.0, 0.0], [0.3, 0.05]]},
                   insertion_rate=[[0.0, 0.01], [0.3, 0.0]]),
    "tube_b": dict(_TUBE_SCENE, name="tube_b", tensions={"2": [[0.0, 0.02], [0.15, 0.0], [0.3, 0.04]],
                                                         "3": [[0.0, 0.0], [0.3, 0.02]]},
                   insertion_rate=[[0.0, 0.0], [0.1, 0.02], [0.3, 0.005]]),
}


BENCH_CELLS = [(41, 8, "accelerated_qp"), (61, 4, "accelerated_qp"), (41, 8, "pgs_baseline")]
FAKE_RESULT = {"environment": {"cablefem_version": "0.1.0", "cpu": "x", "platform": "p", "python": "3", "threads": 1},
               "config": {"node_counts": [10], "contact_targets": [2]}, "config_hash": "abc",
               "rows": [{"backend": "accelerated_qp", "nodes": 10, "dof": 60, "target_contacts": 2,
                         "achieved_contacts": 2.0, "mean_ms": 1.5, "p50_ms": 1.25, "solve_mean_ms": 1.0,
                         "solve_p50_ms": 0.75, "iters": 25.0, "flagged": False}]}


def main():
    from ref_bridge import import_reference
    import_reference()
    from cablefem import engine as ce, scenario as sc
    out = {}
    for tag, raw in FRAME_SCENES.items():
        recs = ce.run_scenario(sc.parse_scenario(raw))
        N = len(recs[0].coords) // 6
        out[f"{tag}_records"] = len(recs)
        out[f"{tag}_coords"] = np.array([r.coords for r in recs])
        out[f"{tag}_n_c"] = np.array([r.n_c for r in recs])
        out[f"{tag}_iterations"] = np.array([r.iterations for r in recs])
        out[f"{tag}_retried"] = np.array([r.retried for r in recs])
        out[f"{tag}_dx_norm"] = np.array([r.dx_norm for r in recs])
        tri = np.full((len(recs), N), -1, np.int32)
        frc = np.zeros((len(recs), N, 3))
        for f, r in enumerate(recs):
            for c, fv in zip(r.contact_points, np.asarray(r.contact_force_vectors).reshape(-1, 3)):
                node = ce.contact_node(c)
                tri[f, node] = c.triangle_id
                frc[f, node] = fv
        out[f"{tag}_tri"] = tri
        out[f"{tag}_force"] = frc
        print(tag, len(recs), "records; n_c", [r.n_c for r in recs], "its", [r.iterations for r in recs], flush=True)
    # bench cells (bench.py:74-107) and the report writer's CSV (bench.py:140-153)
    from cablefem import bench as cb
    import tempfile
    for nodes, target, backend in BENCH_CELLS:
        cfg = cb.BenchmarkConfig(node_counts=[nodes], contact_targets=[target], backends=[backend],
                                 repetitions=4, warmup_frames=2)
        row = cb.run_cell(nodes, target, backend, cfg)
        tag = f"cell_{nodes}_{target}_{backend}"
        out[f"{tag}_iters"] = row["iters"]
        out[f"{tag}_achieved"] = row["achieved_contacts"]
        out[f"{tag}_max_pen"] = row["max_penetration"]
        print(tag, row["iters"], row["achieved_contacts"], flush=True)
    with tempfile.TemporaryDirectory() as tmp:
        cb.write_benchmark_outputs(FAKE_RESULT, os.path.join(tmp, "r.json"))
        out["writer_csv"] = np.array(open(os.path.join(tmp, "r.csv")).read())
        out["writer_json"] = np.array(open(os.path.join(tmp, "r.json")).read())
    np.savez_compressed(os.path.join(HERE, "frames.npz"), **out)


if __name__ == "__main__":
    main()
