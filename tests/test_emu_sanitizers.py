"""AddressSanitizer + UndefinedBehaviorSanitizer over the device algorithm.

compute-sanitizer is closed on this GPU pool (gpurun answers "compute-sanitizer
is closed on this pool", exit 86), so the memory-safety evidence for the solver
is this: the same team-generic device source, compiled by g++ with
-fsanitize=address,undefined (tests/emu), runs element passes, detection on
random soups and a 1e5-triangle tube, run_static of cfg1/cfg3p/cfg2 (ADMM,
polish, direct path), the PGS backend and a failure case, in a subprocess with
libasan preloaded; any report fails the test."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, dataclasses, numpy as np
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
from emu.emu_binding import EmuEngine
from paper_2503_06922_b200 import scenarios
from paper_2503_06922_b200.scene import TriangleMesh, straight_model, MaterialParams, FixedNodeSpec, SolverSettings
for w in (scenarios.cfg1(2, seed=1), scenarios.cfg3p(1), scenarios.cfg2(1), scenarios.infeasible_press(1)):
    w.max_frames = min(w.max_frames, 30)
    e = EmuEngine(**w.engine_kwargs())
    H = e.solve(w.x0, w.tensions, w.applied, w.tol, w.max_frames, trace_cap=w.max_frames)
    e.element_pass(w.x0)
    if w.mesh is not None:
        e.detect(w.x0)
    print(w.name, H["status"].tolist(), H["frames"].tolist(), flush=True)
w = scenarios.cfg3p(1)
w.settings = dataclasses.replace(w.settings, backend="pgs_baseline")
w.max_frames = 3
H = EmuEngine(**w.engine_kwargs()).solve(w.x0, None, w.applied, w.tol, 3, trace_cap=3)
print("pgs", H["status"].tolist(), flush=True)
rng = np.random.default_rng(42)
model = straight_model(12, 0.55, MaterialParams(510e6, 5.551e-6, 5.041e-12))
for _ in range(5):
    n_tri = int(rng.integers(40, 500))
    v = rng.uniform(-0.4, 0.9, size=(n_tri * 3, 3))
    mesh = TriangleMesh(v, np.arange(n_tri * 3).reshape(-1, 3))
    e = EmuEngine(model, mesh=mesh, fixed_specs=[FixedNodeSpec(0)], margin=float(rng.uniform(1e-3, 2e-2)),
                  settings=SolverSettings(beta0=1e-300))
    x = model.rest_configuration.reshape(-1, 6).copy()
    x[:, :3] += rng.uniform(-0.05, 0.05, size=3)
    e.detect(x.reshape(1, -1))
print("SANITIZED_OK")
'''


def test_device_source_under_asan_and_ubsan():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from emu import emu_binding
    try:
        so = emu_binding.build(sanitize=True)
    except subprocess.CalledProcessError:
        pytest.skip("g++ sanitizer runtime unavailable")
    libasan = subprocess.run(["g++", "-print-file-name=libasan.so"], capture_output=True, text=True).stdout.strip()
    if not os.path.exists(libasan):
        pytest.skip("libasan not found")
    env = dict(os.environ, LD_PRELOAD=libasan, ASAN_OPTIONS="detect_leaks=0:abort_on_error=1",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1", ACCFEM_EMU_SO=so)
    res = subprocess.run([sys.executable, "-c", f"ROOT = {ROOT!r}\n" + SCRIPT], env=env, capture_output=True,
                         text=True, timeout=900)
    bad = [ln for ln in res.stderr.splitlines() if "AddressSanitizer" in ln or "runtime error" in ln]
    assert res.returncode == 0 and "SANITIZED_OK" in res.stdout and not bad, (res.stdout[-2000:], res.stderr[-4000:])
