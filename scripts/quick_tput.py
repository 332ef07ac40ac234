"""Quick device throughput probe for cfg4 batches (development helper)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2503_06922_b200 import scenarios
from paper_2503_06922_b200.engine import Engine
S = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
w = scenarios.cfg4(S)
eng = Engine(**w.engine_kwargs(), device=0)
t = lambda a: torch.tensor(a, device="cuda:0")
x0, ten, app = t(w.x0), t(w.tensions), t(w.applied)
print("teams resident", eng._lib.accfem_teams_resident(eng._h))
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for rep in range(REPS):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = eng.solve_static_batch(x0, ten, app, tol=w.tol, max_frames=w.max_frames)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    st = r.status.cpu().numpy()
    print(f"S={S} {dt*1e3:.1f} ms  {S/dt:.0f} solves/s  status counts {np.bincount(st)}  frames mean {r.frames.float().mean().item():.2f}")
bad = np.flatnonzero(st != 0)
print("non-ok scenarios", bad.tolist(), "status", st[bad].tolist())
