"""Batch-1 latency probe: p50 wall-clock of Engine.solve_static_batch (device
tensors, synchronize) per config, in the mode ACCFEM_MODE selects."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_06922_b200 import scenarios  # noqa: E402
from paper_2503_06922_b200.engine import Engine  # noqa: E402


def probe(tag, w, reps=12):
    eng = Engine(**w.engine_kwargs(), device=0)
    dev = torch.device("cuda", 0)
    a = [None if v is None else torch.tensor(v, device=dev) for v in (w.x0, w.tensions, w.applied)]
    o = eng.allocate_batch(w.size)
    ts = []
    for rep in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.solve_static_batch(a[0], a[1], a[2], tol=w.tol, max_frames=w.max_frames, out=o)
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append((time.perf_counter() - t0) * 1e3)
    st = o.status.cpu().numpy()
    p50 = statistics.median(ts)
    print(f"{os.environ.get('ACCFEM_MODE', 'auto'):6s} {tag:10s} S={w.size:4d} p50 {p50:8.3f} ms "
          f"min {min(ts):8.3f} -> {w.size / (p50 * 1e-3):9.1f} solves/s frames {o.frames.cpu().numpy()[:4]} "
          f"status {np.unique(st)}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg3p", "cfg4_s0", "cfg1", "cfg5"]
    for tag in which:
        if tag == "cfg4_s0":
            w = scenarios.cfg4(1)
        elif tag == "cfg1":
            w = scenarios.cfg1(1)
        elif tag == "cfg4_148":
            w = scenarios.cfg4(148)
        elif tag.startswith("cfg5_"):
            w = scenarios.cfg5(int(tag.split("_")[1]))
        else:
            w = scenarios.CONFIGS[tag](1)
        probe(tag, w, reps=6 if tag.startswith("cfg5") else 12)
