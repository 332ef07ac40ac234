"""Device broad-phase grid build on a 10^5-triangle tube: Engine creation time
(host sizing + device count/scan/fill/sort) vs the host build (emulation)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_2503_06922_b200 import scenarios  # noqa: E402
from paper_2503_06922_b200.engine import Engine  # noqa: E402
from paper_2503_06922_b200.scene import FixedNodeSpec, make_tube  # noqa: E402

w = scenarios.cfg3(1)
x = np.linspace(-0.01, 0.52, 400)
path = np.stack([x, 0.002 * np.sin(40 * x), 0.001 * np.cos(25 * x)], axis=1)
tube = make_tube(path, 0.0036 + 0.0004 * np.sin(30 * x), segments=128)
kw = dict(model=w.model, mesh=tube, fixed_specs=[FixedNodeSpec(0)], margin=w.margin, settings=w.settings)
torch.zeros(1, device="cuda:0")
Engine(**kw, device=0)  # warm (context, module load)
ts = []
for _ in range(5):
    t = time.perf_counter()
    eng = Engine(**kw, device=0)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t)
dims, start, tris = eng.broad_phase_grid()
print(f"triangles {tube.triangle_count} grid {dims.tolist()} entries {tris.size} "
      f"device create median {1e3 * float(np.median(ts)):.1f} ms")
try:
    from emu.emu_binding import EmuEngine
    t = time.perf_counter()
    EmuEngine(**kw)
    print(f"host (emulation) create {1e3 * (time.perf_counter() - t):.1f} ms")
except Exception as e:  # noqa: BLE001
    print("emu unavailable:", e)
