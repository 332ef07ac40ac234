"""Dump golden fixtures of the reference's PGS backend (solve_pgs,
solver.py:531-665) through its Engine (backend="pgs_baseline").

    python tests/golden/make_golden_pgs.py      (build container only)

Writes tests/golden/pgs.npz:
  cfg3p_*        run_static of cfg3p (101 nodes, 20 floor contacts) with PGS
  c400_{5,50}_*  the criterion-6 scenes (bench.build_constriction_engine(400,
                 5|50), test_acceptance.py:159-196): 4 Engine.step frames each --
                 coords, sweeps, n_c, contact forces per frame
"""

import dataclasses
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from ref_bridge import import_reference, reference_engine, reference_inputs, run_reference  # noqa: E402

from paper_2503_06922_b200 import scenarios  # noqa: E402


def pgs(w):
    w.settings = dataclasses.replace(w.settings, backend="pgs_baseline")
    return w


def main():
    out = {}
    t = time.time()
    w = pgs(scenarios.cfg3p(1))
    o = run_reference(w, 0)
    assert o["status_exc"] is None, o["status_exc"]
    for key in ("coords", "frames", "iterations", "n_c", "dx_norm", "residual", "contact_nodes", "contact_tris",
                "contact_forces"):
        out[f"cfg3p_{key}"] = o[key]
    print("cfg3p pgs frames", o["frames"], "sweeps", o["iterations"], round(time.time() - t, 1), flush=True)
    beam, _, engine_mod, _, _ = import_reference()
    for target in (5, 50):
        t = time.time()
        w = pgs(scenarios.constriction(400, target, f"c400_{target}"))
        eng = reference_engine(w)
        x = beam.Configuration(w.x0[0].copy())
        coords, sweeps, ncs, forces = [], [], [], []
        for k in range(4):
            x, rec = eng.step(x, reference_inputs(w, 0), t=0.0, frame_index=k)
            coords.append(x.coords.copy())
            sweeps.append(rec.iterations)
            ncs.append(rec.n_c)
            forces.append(np.asarray(rec.contact_force_vectors).reshape(-1, 3))
        tag = f"c400_{target}"
        out[f"{tag}_coords"] = np.array(coords)
        out[f"{tag}_sweeps"] = np.array(sweeps)
        out[f"{tag}_n_c"] = np.array(ncs)
        for k, f in enumerate(forces):
            out[f"{tag}_forces_{k}"] = f
        print(tag, "sweeps", sweeps, "n_c", ncs, round(time.time() - t, 1), flush=True)
    np.savez_compressed(os.path.join(HERE, "pgs.npz"), **out)


if __name__ == "__main__":
    main()
