"""B200-native quasi-static equilibrium solver for cable-driven continuum
robots in contact (the hot path of Acc-FEM, arXiv 2503.06922).

Reference-compatible scene API (`scene`), the device-backed `Engine`
(`engine`), workload generators (`scenarios`) and the C ABI binding
(`_lib`, include/accfem.h).  Importing the package does not touch the GPU;
constructing an `Engine` loads the sm_100a library and fails loudly if it or
a CUDA device is missing.
"""

from .errors import (  # noqa: F401
    CableFemError,
    DegenerateElementError,
    DeviceError,
    DomainError,
    EngineError,
    InfeasibleError,
    MeshError,
    NonConvergenceError,
    ScenarioError,
)
from .scene import (  # noqa: F401
    CableSpec,
    Configuration,
    ContactPoint,
    FixedNodeSpec,
    FrameRecord,
    MATERIAL_PRESETS,
    MaterialParams,
    RobotModel,
    SolverSettings,
    StepInputs,
    TriangleMesh,
    contact_node,
    default_cables,
    load_mesh,
    make_rectangle,
    make_tube,
    orient_normals,
    straight_model,
)

__version__ = "0.1.0"


def __getattr__(name):
    if name in ("Engine", "BatchResult"):
        from . import engine
        return getattr(engine, name)
    if name in ("Timeline", "Trajectory", "run_scenario", "run_trajectories", "initial_record"):
        from . import frames
        return getattr(frames, name)
    raise AttributeError(name)
