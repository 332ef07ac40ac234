"""Small launches of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): k_solve in the three modes (2-warp, 4-warp, 8-warp
cyclic reduction), the PGS backend, the unit element-pass / detection
kernels and the device grid build.  Prints one line per case."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_06922_b200 import scenarios  # noqa: E402
from paper_2503_06922_b200.engine import Engine  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda a: None if a is None else torch.tensor(a, device=dev)  # noqa: E731
which = sys.argv[1:] or ["team2", "team4", "cr", "pgs", "units"]
for mode in which:
    if mode in ("team2", "team4", "cr"):
        os.environ["ACCFEM_MODE"] = mode
        for w in (scenarios.cfg3p(2), scenarios.cfg1(2)):
            w.max_frames = 2
            eng = Engine(**w.engine_kwargs(), device=0)
            r = eng.solve_static_batch(t(w.x0), t(w.tensions), t(w.applied), tol=w.tol, max_frames=w.max_frames,
                                       trace_frames=2)
            torch.cuda.synchronize()
            print(mode, w.name, "status", r.status.cpu().tolist(), "frames", r.frames.cpu().tolist(), flush=True)
        os.environ.pop("ACCFEM_MODE")
    elif mode == "pgs":
        w = scenarios.cfg3p(1)
        w.settings = dataclasses.replace(w.settings, backend="pgs_baseline")
        w.max_frames = 2
        eng = Engine(**w.engine_kwargs(), device=0)
        r = eng.solve_static_batch(t(w.x0), None, t(w.applied), tol=w.tol, max_frames=2)
        torch.cuda.synchronize()
        print("pgs status", r.status.cpu().tolist(), flush=True)
    elif mode == "units":
        w = scenarios.cfg3(1)
        eng = Engine(**w.engine_kwargs(), device=0)  # includes the grid build kernels
        x = t(w.x0)
        f, kd, ku, fr, bad = eng.element_pass(x)
        tri, gap, pt = eng.detect(x)
        torch.cuda.synchronize()
        print("units contacts", int((tri >= 0).sum()), flush=True)
