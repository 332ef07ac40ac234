"""One k_solve launch of the bench workload (cfg4, 8192 scenarios) for ncu;
prints the library sha the capture belongs to."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_06922_b200 import _lib, scenarios  # noqa: E402
from paper_2503_06922_b200.engine import Engine  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
w = scenarios.cfg4(S)
eng = Engine(**w.engine_kwargs(), device=0)
dev = torch.device("cuda", 0)
r = eng.solve_static_batch(torch.tensor(w.x0, device=dev), torch.tensor(w.tensions, device=dev),
                           torch.tensor(w.applied, device=dev), tol=w.tol, max_frames=w.max_frames)
torch.cuda.synchronize()
sys.argv = sys.argv[:1]
import bench  # noqa: E402

print("solved", S, "status0", int((r.status == 0).sum()), "library_source_sha256_16", bench.library_sha())
