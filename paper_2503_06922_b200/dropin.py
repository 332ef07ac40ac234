"""Route an unmodified `cablefem` program through the B200 Engine.

The reference binds `Engine` by name in four modules (engine.py:84,
scenario.py:18, bench.py:23, validate.py:21); `install()` rebinds each of them
to `paper_2503_06922_b200.engine.Engine`, so `run_scenario` (engine.py:300-316),
`Scenario.build_engine` (scenario.py:132-141), `bench.run_cell`
(bench.py:74-107) and the validation suites construct the device engine and
step it through the C ABI.  This is the one-line integration INTEGRATION.md
describes; `uninstall()` restores the reference classes.

Only the accelerated_qp backend exists on the device: a caller that asks for
another backend gets the DomainError the Engine constructor raises.
"""

from __future__ import annotations

_MODULES = ("cablefem.engine", "cablefem.scenario", "cablefem.bench", "cablefem.validate")
_saved = {}


def install(device=None):
    """Rebind `Engine` in every reference module that imported it by name."""
    import importlib

    from .engine import Engine as DeviceEngine

    cls = DeviceEngine
    if device is not None:
        class _Bound(DeviceEngine):  # noqa: D401 - same class, device pinned
            def __init__(self, *a, **kw):
                kw.setdefault("device", device)
                super().__init__(*a, **kw)
        cls = _Bound
    for name in _MODULES:
        mod = importlib.import_module(name)
        if name not in _saved:
            _saved[name] = mod.Engine
        mod.Engine = cls
    return cls


def uninstall():
    import importlib

    for name, orig in list(_saved.items()):
        importlib.import_module(name).Engine = orig
        del _saved[name]
