"""A/B bit-identity check of two library builds (development).

usage: python scripts/ab_bitexact.py OLD.so NEW.so
Runs the same workloads in every kernel mode with each build (ACCFEM_LIB selects
the library, one subprocess per build) and compares every output array bit for
bit; contact slots beyond n_contacts are undefined and masked.
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("cfg5", 8, "cr"), ("cfg5", 8, "team2"), ("cfg5", 8, "team4"), ("cfg4", 64, "team2"),
         ("cfg4", 16, "cr"), ("cfg3p", 4, "cr"), ("cfg3p", 4, "team2")]


def run(out):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2503_06922_b200 import scenarios
    from paper_2503_06922_b200.engine import Engine
    res = {}
    for name, S, mode in CASES:
        os.environ["ACCFEM_MODE"] = mode
        w = scenarios.cfg4(S) if name == "cfg4" else scenarios.CONFIGS[name](S)
        eng = Engine(**w.engine_kwargs(), device=0)
        t = lambda a: None if a is None else torch.tensor(a, device="cuda:0")
        r = eng.solve_static_batch(t(w.x0), t(w.tensions), t(w.applied), tol=w.tol, max_frames=w.max_frames)
        from dataclasses import fields
        rn = r.to_numpy()
        for fd in fields(rn):
            v = getattr(rn, fd.name)
            if v is not None:
                res[f"{name}_{S}_{mode}_{fd.name}"] = np.asarray(v)
    np.savez(out, **res)


def main():
    if sys.argv[1] == "--run":
        run(sys.argv[2])
        return
    outs = []
    for i, so in enumerate(os.path.abspath(p) for p in sys.argv[1:3]):  # dlopen needs a path, not a bare name
        out = f"/tmp/ab_{i}.npz"
        subprocess.run([sys.executable, __file__, "--run", out], check=True, env={**os.environ, "ACCFEM_LIB": so})
        outs.append(np.load(out))
    a, b = outs
    bad = 0
    for name, S, mode in CASES:
        p = f"{name}_{S}_{mode}_"
        nc = a[p + "n_contacts"]
        diffs = []
        for k in sorted(x for x in a.files if x.startswith(p)):
            x, y = a[k], b[k]
            if k.endswith(("contact_node", "contact_triangle", "contact_gap", "contact_multiplier", "contact_force",
                           "contact_normal", "contact_point")):
                m = np.arange(x.shape[1])[None, :] < nc[:, None]
                x, y = x[m], y[m]
            if x.shape != y.shape or x.tobytes() != y.tobytes():
                diffs.append(k[len(p):])
        bad += bool(diffs)
        print(f"{name} S={S} {mode:6s} status {np.unique(a[p + 'status'])} frames {a[p + 'frames'][:4]}: "
              f"{'bit-identical' if not diffs else 'DIFFERS in ' + ', '.join(diffs)}")
    print("ALL BIT-IDENTICAL" if not bad else f"{bad} cases differ")


if __name__ == "__main__":
    main()
