"""Trajectory CSV in the reference's format (scenario.py:245-279), for runs
driven through the device Engine (`run_scenario`, `step_batch`)."""

from __future__ import annotations

from pathlib import Path

from . import __version__


def write_trajectory_csv(path, name, records, node_count, solver="accelerated_qp", config_hash="", overrides=(),
                         threads=1, include_timings=False):
    """One row per FrameRecord plus the reproducibility header; timing columns
    are zeroed unless include_timings, so identical runs give identical files."""
    cols = ["t"]
    for n in range(node_count):
        cols += [f"node{n}_x", f"node{n}_y", f"node{n}_z"]
    cols += ["n_c", "tip_x", "tip_y", "tip_z", "solve_ms", "iters"]
    lines = [
        f"# paper_2503_06922_b200 {__version__} trajectory",
        f"# scenario: {name}",
        f"# config_hash: {config_hash}",
        f"# threads: {threads}",
        f"# solver: {solver}",
        f"# overrides: {' '.join(overrides) if overrides else '(none)'}",
        f"# timings: {'wall-clock' if include_timings else 'zeroed for reproducibility'}",
        ",".join(cols),
    ]
    for rec in records:
        pos = rec.coords.reshape(-1, 6)[:, :3].ravel()
        solve_ms = rec.solve_ms if include_timings else 0.0
        row = [repr(float(rec.t))] + [repr(float(v)) for v in pos] + [str(rec.n_c)]
        row += [repr(float(v)) for v in rec.tip_position] + [repr(float(solve_ms)), str(rec.iterations)]
        lines.append(",".join(row))
    Path(path).write_text("\n".join(lines) + "\n")
    return Path(path)
