"""An UNMODIFIED reference caller through the device Engine.

The reference package is the pip install under baseline/_ref (git-ignored,
shipped to the GPU box with the repo snapshot; never /root/reference at run
time).  A subprocess imports it, runs the reference's own `run_scenario`
(engine.py:300-316) and `bench.run_cell` (bench.py:74-107) on the CPU, then
`paper_2503_06922_b200.dropin.install()` and the very same calls again on the
device, and compares the FrameRecords: frame count, per-frame n_c and ADMM
iterations, retried flags, contact triangles, coords (1e-6 rel) and forces.
Also checks that `except cablefem.errors.EngineError` catches a device failure.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
import cablefem.scenario as sc, cablefem.engine as ce, cablefem.bench as cb, cablefem.errors as cerr
from cablefem.solver import SolverSettings

def tube(n_pts=24, r=0.0036):
    xs = np.linspace(-0.02, 0.11, n_pts)
    return {"path_points": [[float(x), 0.0, 0.00005 + r * np.cos(np.pi / 18)] for x in xs],
            "radii": [r] * n_pts, "segments": 18}

SCEN = [
    {"name": "ramp", "robot": {"node_count": 21, "length": 0.07, "material": "a"},
     "tensions": {"1": [[0.0, 0.0], [0.2, 0.3]], "2": [[0.0, 0.0], [0.2, 0.1]]},
     "insertion_rate": [[0.0, 0.0], [0.1, 0.01]], "frame_period": 0.02, "duration": 0.2},
    {"name": "tube", "robot": {"node_count": 21, "length": 0.07, "material": "a"},
     "mesh": {"tube": tube()}, "uniform_load": [0.0, 0.0, -0.002],
     "tensions": {"1": [[0.0, 0.0], [0.3, 0.05]]},
     "insertion_rate": [[0.0, 0.01], [0.3, 0.0]], "frame_period": 0.03, "duration": 0.3},
]

def recs_of(raw):
    return ce.run_scenario(sc.parse_scenario(raw))

def compare(a, b, tag):
    assert len(a) == len(b), (tag, len(a), len(b))
    for ra, rb in zip(a, b):
        assert ra.frame_index == rb.frame_index and ra.n_c == rb.n_c, tag
        assert ra.iterations == rb.iterations, (tag, ra.frame_index, ra.iterations, rb.iterations)
        assert bool(ra.retried) == bool(rb.retried), tag
        assert [c.triangle_id for c in ra.contact_points] == [c.triangle_id for c in rb.contact_points], tag
        sc_ = max(np.abs(rb.coords).max(), 1e-12)
        assert np.abs(ra.coords - rb.coords).max() <= 1e-6 * sc_, (tag, ra.frame_index)
        fa, fb = np.asarray(ra.contact_force_vectors), np.asarray(rb.contact_force_vectors)
        if fb.size:
            assert np.abs(fa - fb).max() <= 1e-5 * np.abs(fb).max() + 1e-12, tag
        assert abs(ra.dx_norm - rb.dx_norm) <= 1e-6 * rb.dx_norm + 1e-12, tag

ref = [recs_of(r) for r in SCEN]
cfg = cb.BenchmarkConfig(node_counts=[41], contact_targets=[8], backends=["accelerated_qp"], repetitions=4,
                         warmup_frames=1)
row_ref = cb.run_cell(41, 8, "accelerated_qp", cfg)

from paper_2503_06922_b200 import dropin
from paper_2503_06922_b200.engine import Engine as Dev
dropin.install(device=0)
assert sc.Engine is not ce.__dict__.get("_orig", None)
dev = [recs_of(r) for r in SCEN]
for r, d, raw in zip(ref, dev, SCEN):
    compare(d, r, raw["name"])
row_dev = cb.run_cell(41, 8, "accelerated_qp", cfg)
assert row_dev["achieved_contacts"] == row_ref["achieved_contacts"], (row_dev, row_ref)
assert row_dev["iters"] == row_ref["iters"], (row_dev["iters"], row_ref["iters"])
assert row_dev["max_penetration"] == pytest_approx(row_ref["max_penetration"])
# a device failure is caught by the reference's own exception class
raw = dict(SCEN[0]); raw["solver"] = {"max_iterations": 2}
eng = sc.parse_scenario(raw).build_engine()
assert isinstance(eng, Dev)
try:
    x = eng.initial_configuration()
    from cablefem.engine import StepInputs
    eng.run_static(StepInputs(tensions=np.array([0.5, 0.0, 0.0])), x0=x, tol=1e-9, max_frames=3)
    raise SystemExit("expected EngineError")
except cerr.EngineError:
    pass
dropin.uninstall()
print("DROPIN_OK")
'''


def test_unmodified_reference_callers_run_on_the_device():
    if not os.path.isdir(os.path.join(REF, "cablefem")):
        pytest.skip("reference install baseline/_ref absent (pip install --target baseline/_ref)")
    pre = (f"REF = {REF!r}\nROOT = {ROOT!r}\n"
           "def pytest_approx(v):\n"
           "    class A:\n"
           "        def __eq__(s, o): return abs(o - v) <= 1e-6 * max(abs(v), 1e-9) + 1e-12\n"
           "    return A()\n")
    res = subprocess.run([sys.executable, "-c", pre + SCRIPT], capture_output=True, text=True, timeout=900)
    assert res.returncode == 0 and "DROPIN_OK" in res.stdout, res.stdout[-3000:] + res.stderr[-3000:]
