"""Per-phase device time breakdown (development): loads libaccfem_prof.so
(built with -DACCFEM_PROFILE) and reports clock cycles per solve by phase."""
import ctypes, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2503_06922_b200 import _lib, build, scenarios
import os
so = os.environ.get("ACCFEM_PROF_SO") or build.build(profile=True)
_lib._LIB = _lib.bind(ctypes.CDLL(so))
_lib._LIB.accfem_dev_set_profile.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
from paper_2503_06922_b200.engine import Engine
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1776
if name.startswith("c400_"):  # criterion-6 constriction scenes (400 nodes, 5 or 50 contacts)
    w = scenarios.constriction(400, int(name[5:]), name, n_scenarios=S)
else:
    w = scenarios.cfg4(S) if name == "cfg4" else scenarios.CONFIGS[name](S)
eng = Engine(**w.engine_kwargs(), device=0)
teams = eng._lib.accfem_teams_resident(eng._h)
prof = torch.zeros((teams, 24), dtype=torch.int64, device="cuda:0")
assert eng._lib.accfem_dev_set_profile(eng._h, prof.data_ptr()) == 0
t = lambda a: None if a is None else torch.tensor(a, device="cuda:0")
torch.cuda.synchronize(); t0 = time.perf_counter()
r = eng.solve_static_batch(t(w.x0), t(w.tensions), t(w.applied), tol=w.tol, max_frames=w.max_frames)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
p = prof.sum(0).cpu().numpy().astype(float)
names = ["element", "detect", "ruiz", "factor", "admm_iter", "chain", "check", "polish", "direct", "post", "total",
         "iters", "frames"]
print(f"{name} S={S} wall {dt*1e3:.1f} ms -> {S/dt:.0f} solves/s; frames/solve {p[12]/S:.2f} iters/solve {p[11]/S:.1f}")
for i, nm in enumerate(names[:11]):
    print(f"  {nm:10s} {p[i]/S/1e6:9.3f} Mcycles/solve  {100*p[i]/max(p[10],1):5.1f}%")
print(f"  per ADMM iteration: {p[4]/max(p[11],1):.0f} cycles (chain {p[5]/max(p[11],1):.0f})")
print(f"  polish: factor {p[13]/S/1e6:.3f} W+S+v {p[14]/S/1e6:.3f} rounds {p[15]/S/1e6:.3f} Mcycles/solve")
print(f"  per frame: element {p[0]/max(p[12],1):.0f} detect {p[1]/max(p[12],1):.0f} ruiz {p[2]/max(p[12],1):.0f} factor {p[3]/max(p[12],1):.0f} polish {p[7]/max(p[12],1):.0f}")
print(f"  polish round parts (Mcycles/solve): list {p[16]/S/1e6:.3f} chol+solve {p[17]/S/1e6:.3f} combine {p[18]/S/1e6:.3f} "
      f"refine {p[19]/S/1e6:.3f} correction {p[20]/S/1e6:.3f} multipliers {p[21]/S/1e6:.3f}")
