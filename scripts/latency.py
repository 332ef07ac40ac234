"""Single-solve latency probe (development helper): p50 wall clock of a
batch-1 solve_static_batch + synchronize for cfg3p and cfg4 scenario 0."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2503_06922_b200 import scenarios
from paper_2503_06922_b200.engine import Engine

for tag, wl in (("cfg3p", scenarios.cfg3p(1)), ("cfg4_s0", scenarios.cfg4(1)), ("cfg1", scenarios.cfg1(1))):
    eng = Engine(**wl.engine_kwargs(), device=0)
    a = [None if v is None else torch.tensor(v, device="cuda:0") for v in (wl.x0, wl.tensions, wl.applied)]
    o = eng.allocate_batch(1)
    ts = []
    for rep in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.solve_static_batch(a[0], a[1], a[2], tol=wl.tol, max_frames=wl.max_frames, out=o)
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{tag}: p50 {statistics.median(ts):.3f} ms  frames {int(o.frames[0].item())}  "
          f"status {int(o.status[0].item())}", flush=True)
