"""cfg5 (1001 nodes, 200 contacts) device timing probe (development helper):
batch-1 wall clock and a small batch throughput."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2503_06922_b200 import scenarios
from paper_2503_06922_b200.engine import Engine

for S in (1, 148):
    w = scenarios.cfg5(S)
    eng = Engine(**w.engine_kwargs(), device=0)
    a = [None if v is None else torch.tensor(v, device="cuda:0") for v in (w.x0, w.tensions, w.applied)]
    o = eng.allocate_batch(S)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        eng.solve_static_batch(a[0], a[1], a[2], tol=w.tol, max_frames=w.max_frames, out=o)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"cfg5 S={S}: {dt*1e3:.1f} ms -> {S/dt:.1f} solves/s, frames {o.frames[:4].tolist()}, status {o.status[:4].tolist()}",
          flush=True)
