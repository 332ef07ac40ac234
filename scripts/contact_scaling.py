"""Criterion 6 of the reference (test_acceptance.py:159-196) on the device:
mean frame time at 5 vs 50 active contacts on the 400-node constriction scene
(bench.build_constriction_engine(400, target)), accelerated QP vs the PGS
baseline, frames alternated between the two scenes like the reference.

    python scripts/contact_scaling.py [--reps 20] [--warmup 8]

One frame = Engine.step_batch of one scenario (one k_solve launch with
max_frames = 1), wall clock around the launch + synchronize."""
import argparse
import dataclasses
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_06922_b200 import scenarios  # noqa: E402
from paper_2503_06922_b200.engine import Engine  # noqa: E402


def growth(backend, reps, warmup):
    dev = torch.device("cuda", 0)
    scenes = {}
    for target in (5, 50):
        w = scenarios.constriction(400, target, f"c400_{target}")
        w.settings = dataclasses.replace(w.settings, backend=backend)
        eng = Engine(**w.engine_kwargs(), device=0)
        scenes[target] = [eng, torch.tensor(w.x0, device=dev), torch.tensor(w.applied, device=dev), None]
    times, contacts, iters = {5: [], 50: []}, {5: [], 50: []}, {5: [], 50: []}
    for k in range(warmup + reps):
        for target in (5, 50):
            eng, x, app, state = scenes[target]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out, stats, state = eng.step_batch(x, None, app, None, state)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) * 1e3
            scenes[target][1], scenes[target][3] = out.coords, state
            if k >= warmup:
                st = stats.cpu().numpy()[0]
                times[target].append(dt)
                contacts[target].append(int(st[6]))
                iters[target].append(int(st[5]))
    return {t: {"mean_ms": statistics.mean(times[t]), "contacts": statistics.mean(contacts[t]),
                "iterations": statistics.mean(iters[t])} for t in (5, 50)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=8)
    a = ap.parse_args()
    res = {}
    for backend in ("accelerated_qp", "pgs_baseline"):
        r = growth(backend, a.reps, a.warmup)
        res[backend] = {**r, "growth": r[50]["mean_ms"] / r[5]["mean_ms"]}
    res["criterion_6"] = {"qp_growth_le_1.30": res["accelerated_qp"]["growth"] <= 1.30,
                          "pgs_growth_ge_2": res["pgs_baseline"]["growth"] >= 2.0}
    print(json.dumps(res, indent=1))
