"""Dump failure-mode and solver-state golden fixtures from the REAL reference.

    python tests/golden/make_golden_status.py      (build container only)

Writes tests/golden/status.npz.  Each case is a Workload variant run through
the reference's `Engine.run_static` (engine.py:267-283); the fixture holds the
status class (errors.py taxonomy -> include/accfem.h codes), the frame index
named in an EngineError message, and for successful runs the same per-frame
records as solves.npz (iterations, n_c, dx_norm, retried, residual).

  retry_ok      cfg4[0] with max_iterations=300: frame retried once with the
                adopted rho estimate, then succeeds (engine.py:168-188)
  retry_fail0   cfg3 with max_iterations=30: solver fails twice at frame 0 -> EngineError
  retry_fail9   cfg3 with max_iterations=200: fails twice at frame 9 -> EngineError
  infeasible    base clamp pushed into a floor it touches -> InfeasibleError
                (certificate test, solver.py:424-446)
  cfg5_fine     1001 nodes at l0 = 0.47 mm -> EngineError at frame 0
  cfg5_250      1001 nodes, 250 pressed contacts (bench.py:51-71 with target 250)
  cfg4_984      cfg4 scenarios whose reference run exhausts max_frames = 400
  cfg4_5450       (EngineError "static mode did not reach ...")
  maxframes3    cfg3 with max_frames = 3 -> EngineError
"""

import dataclasses
import os
import re
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from ref_bridge import run_reference  # noqa: E402

from paper_2503_06922_b200 import scenarios  # noqa: E402
from paper_2503_06922_b200.errors import status_from_exception  # noqa: E402


def _settings(w, **kw):
    w.settings = dataclasses.replace(w.settings, **kw)
    return w


def _frames(w, k):
    w.max_frames = k
    return w


CASES = {
    "retry_ok": lambda: _settings(scenarios.cfg4(1), max_iterations=300),
    "retry_fail0": lambda: _settings(scenarios.cfg3(1), max_iterations=30),
    "retry_fail9": lambda: _settings(scenarios.cfg3(1), max_iterations=200),
    "infeasible": lambda: scenarios.infeasible_press(1),
    "cfg5_fine": lambda: scenarios.cfg5_fine(1),
    "cfg5_250": lambda: scenarios.cfg5(1, target=250),
    "cfg4_984": lambda: scenarios.cfg4(1, start=984),
    "cfg4_5450": lambda: scenarios.cfg4(1, start=5450),
    "maxframes3": lambda: _frames(scenarios.cfg3(1), 3),
}


def main():
    out = {}
    for tag, make in CASES.items():
        w = make()
        t = time.time()
        o = run_reference(w, 0)
        exc = o["status_exc"]
        if exc is not None:
            out[f"{tag}_status"] = status_from_exception(exc)
            m = re.search(r"frame (\d+)", str(exc))
            out[f"{tag}_fail_frame"] = int(m.group(1)) if m else -1
            print(tag, type(exc).__name__, str(exc)[:80], round(time.time() - t, 1), flush=True)
            continue
        out[f"{tag}_status"] = 0
        for key in ("coords", "frames", "iterations", "n_c", "dx_norm", "retried", "residual", "contact_nodes",
                    "contact_tris", "contact_gaps", "contact_forces"):
            out[f"{tag}_{key}"] = o[key]
        out[f"{tag}_frame_residual"] = np.array([r.residual_norm for r in o["records"]])
        out[f"{tag}_frame_scale"] = np.array([r.actuation_scale for r in o["records"]])
        print(tag, "ok frames", o["frames"], "retried", int(np.sum(o["retried"])), round(time.time() - t, 1),
              flush=True)
    np.savez_compressed(os.path.join(HERE, "status.npz"), **out)


if __name__ == "__main__":
    main()
