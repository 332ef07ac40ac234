"""Exception taxonomy of the reference, kept verbatim in meaning.

Mirrors `cablefem/errors.py:4-44` so callers that catch the reference's
exceptions keep working.  When the reference package `cablefem` is importable
(installed, or on sys.path) every class here also SUBCLASSES the reference
class of the same name, so `except cablefem.errors.EngineError` catches a
device failure raised by this package.  The device path reports a
per-scenario status code (`STATUS_*` below, identical to `include/accfem.h`)
and the host wrapper turns it back into the matching exception for
single-scenario calls.
"""

try:  # the reference's own classes, when present (drop-in for callers that catch them)
    from cablefem import errors as _ref
except Exception:  # noqa: BLE001 - reference not installed: standalone taxonomy
    _ref = None


def _bases(name, *own):
    ref = getattr(_ref, name, None) if _ref is not None else None
    return (ref, *own) if ref is not None else own


class CableFemError(*_bases("CableFemError", Exception)):
    """Root of every simulator error (reference `errors.py:4`)."""


class DomainError(*_bases("DomainError", CableFemError, ValueError)):
    """Argument outside its mathematical domain (reference `errors.py:8`)."""


class DegenerateElementError(*_bases("DegenerateElementError", CableFemError)):
    """Coincident element end nodes (reference `errors.py:12`)."""


class MeshError(*_bases("MeshError", CableFemError)):
    """Empty / malformed mesh (reference `errors.py:16`)."""


class ScenarioError(*_bases("ScenarioError", CableFemError)):
    """Scenario description invalid (reference `errors.py:20`)."""


class NonConvergenceError(*_bases("NonConvergenceError", CableFemError)):
    """ADMM ran out of iterations; carries the last iterate (reference `errors.py:24-32`)."""

    def __init__(self, message, result=None):
        Exception.__init__(self, message)
        self.result = result


class InfeasibleError(*_bases("InfeasibleError", CableFemError)):
    """Primal infeasibility certificate found (reference `errors.py:35-41`)."""

    def __init__(self, message, certificate=None):
        Exception.__init__(self, message)
        self.certificate = certificate


class EngineError(*_bases("EngineError", CableFemError)):
    """A frame failed after the retry, or static mode ran out of frames (reference `errors.py:44`)."""


class DeviceError(CableFemError):
    """CUDA / C-ABI failure (no reference counterpart: the reference has no device)."""


# per-scenario status codes written by the device path (same values as include/accfem.h)
STATUS_OK = 0
STATUS_DOMAIN = 1
STATUS_DEGENERATE = 2
STATUS_MESH = 3
STATUS_NONCONVERGENCE = 4
STATUS_INFEASIBLE = 5
STATUS_ENGINE_SOLVER = 6      # solver failed twice in one frame (engine.py:184-188)
STATUS_ENGINE_MAX_FRAMES = 7  # run_static exhausted max_frames (engine.py:281-283)
STATUS_CAPACITY = 8           # more contacts than the handle's contact capacity
STATUS_LINALG = 9             # a factorization hit a non-positive pivot

STATUS_NAMES = {
    STATUS_OK: "ok",
    STATUS_DOMAIN: "DomainError",
    STATUS_DEGENERATE: "DegenerateElementError",
    STATUS_MESH: "MeshError",
    STATUS_NONCONVERGENCE: "NonConvergenceError",
    STATUS_INFEASIBLE: "InfeasibleError",
    STATUS_ENGINE_SOLVER: "EngineError",
    STATUS_ENGINE_MAX_FRAMES: "EngineError",
    STATUS_CAPACITY: "DeviceError",
    STATUS_LINALG: "DeviceError",
}

_STATUS_CLASS = {
    STATUS_DOMAIN: DomainError,
    STATUS_DEGENERATE: DegenerateElementError,
    STATUS_MESH: MeshError,
    STATUS_NONCONVERGENCE: NonConvergenceError,
    STATUS_INFEASIBLE: InfeasibleError,
    STATUS_ENGINE_SOLVER: EngineError,
    STATUS_ENGINE_MAX_FRAMES: EngineError,
    STATUS_CAPACITY: DeviceError,
    STATUS_LINALG: DeviceError,
}


def exception_for_status(status, message):
    """Exception instance matching a device status code (None for STATUS_OK)."""
    if status == STATUS_OK:
        return None
    return _STATUS_CLASS.get(int(status), DeviceError)(message)


def status_from_exception(exc):
    """Status code for a reference exception instance (used by parity tests)."""
    name = type(exc).__name__
    table = {
        "DomainError": STATUS_DOMAIN,
        "DegenerateElementError": STATUS_DEGENERATE,
        "MeshError": STATUS_MESH,
        "NonConvergenceError": STATUS_NONCONVERGENCE,
        "InfeasibleError": STATUS_INFEASIBLE,
    }
    if name == "EngineError":
        return STATUS_ENGINE_MAX_FRAMES if "static mode" in str(exc) else STATUS_ENGINE_SOLVER
    return table.get(name, -1)
