"""Scene description types with the reference's constructor signatures.

These are plain host-side value objects (robot discretisation, material,
fixed DOFs, cables, lumen mesh, solver settings, per-frame inputs and the
per-frame record).  They carry no hot-path arithmetic: everything that the
reference computes per frame (element frames, stiffness, forces, contact
detection, the QP solve) happens on the device behind `include/accfem.h`.
Mesh generators (`make_tube`, `make_rectangle`, `orient_normals`) are scene
construction, listed as configuration plumbing in SURVEY.md §2 rows 4/9.

Reference anchors (all under /root/reference/pkg/src/cablefem/):
  MaterialParams      beam.py:26-51        RobotModel / straight_model beam.py:54-133
  Configuration       beam.py:136-161      FixedNodeSpec constraints.py:20-37
  CableSpec / default_cables constraints.py:71-103
  TriangleMesh        mesh.py:19-61        make_rectangle / make_tube mesh.py:332-401
  orient_normals      mesh.py:150-170      SolverSettings solver.py:41-68
  StepInputs / FrameRecord engine.py:40-81 ContactPoint contact.py:22-30
  MATERIAL_PRESETS    scenario.py:24-33
"""

from __future__ import annotations

import re
import struct
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from .errors import DegenerateElementError, DomainError, MeshError

MIN_CHORD_LENGTH = 1e-9
_DEGENERATE_TWICE_AREA_SQ = 1e-20

MATERIAL_PRESETS = {
    "a": dict(young_modulus=510e6, cross_section_area=5.551e-6, bending_inertia=5.041e-12),
    "b": dict(young_modulus=307e6, cross_section_area=9.03e-6, bending_inertia=19.233e-12),
    "c": dict(young_modulus=510e6, cross_section_area=5.551e-6, bending_inertia=5.041e-12),
    "d": dict(young_modulus=510e6, cross_section_area=5.551e-6, bending_inertia=5.041e-12),
}


# ----------------------------------------------------------------------------
# small host rotation helpers (scene setup / convenience accessors only)
# ----------------------------------------------------------------------------

def rotvec_to_matrix(v):
    """exp map of rotation vectors, scipy `from_rotvec().as_matrix()` formulas."""
    v = np.asarray(v, dtype=float)
    flat = v.reshape(-1, 3)
    th = np.sqrt((flat ** 2).sum(axis=1))
    small = th <= 1e-3
    th2 = th * th
    with np.errstate(divide="ignore", invalid="ignore"):
        scale = np.where(small, 0.5 - th2 / 48 + th2 * th2 / 3840, np.sin(th / 2) / np.where(small, 1.0, th))
    qx, qy, qz = (flat * scale[:, None]).T
    qw = np.cos(th / 2)
    m = np.empty((len(flat), 3, 3))
    m[:, 0, 0] = qx * qx - qy * qy - qz * qz + qw * qw
    m[:, 0, 1] = 2 * (qx * qy - qz * qw)
    m[:, 0, 2] = 2 * (qx * qz + qy * qw)
    m[:, 1, 0] = 2 * (qx * qy + qz * qw)
    m[:, 1, 1] = -qx * qx + qy * qy - qz * qz + qw * qw
    m[:, 1, 2] = 2 * (qy * qz - qx * qw)
    m[:, 2, 0] = 2 * (qx * qz - qy * qw)
    m[:, 2, 1] = 2 * (qy * qz + qx * qw)
    m[:, 2, 2] = -qx * qx - qy * qy + qz * qz + qw * qw
    return m.reshape(v.shape[:-1] + (3, 3))


def _axis_rotvec(axis):
    """Rotation vector of the minimal rotation taking +X onto unit `axis`."""
    ex = np.array([1.0, 0.0, 0.0])
    cr = np.cross(ex, axis)
    s = np.linalg.norm(cr)
    c = float(ex @ axis)
    if s > 1e-12:
        return cr / s * np.arctan2(s, c)
    if c > 0.0:
        return np.zeros(3)
    ref = np.array([1.0, 0.0, 0.0]) if abs(ex[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    ax = np.cross(ex, ref)
    return ax / np.linalg.norm(ax) * np.pi


# ----------------------------------------------------------------------------
# robot
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class MaterialParams:
    """Beam section properties, SI units (reference beam.py:26-51)."""

    young_modulus: float
    cross_section_area: float
    bending_inertia: float
    poisson_ratio: float = 0.3
    torsion_constant: float | None = None

    def __post_init__(self):
        if self.torsion_constant is None:
            object.__setattr__(self, "torsion_constant", 2.0 * self.bending_inertia)
        for name in ("young_modulus", "cross_section_area", "bending_inertia",
                     "poisson_ratio", "torsion_constant"):
            if not getattr(self, name) > 0.0:
                raise DomainError(f"MaterialParams.{name} must be strictly positive")

    @property
    def shear_modulus(self):
        return self.young_modulus / (2.0 * (1.0 + self.poisson_ratio))


@dataclass
class RobotModel:
    """Serial chain of `node_count` nodes, 6 DOF each (reference beam.py:54-111).

    The derived per-element constants (rest element frames, director offsets,
    the 12x12 local stiffness) are computed on the device by `accfem_create`.
    """

    node_count: int
    element_rest_length: float
    rest_configuration: np.ndarray
    material: MaterialParams

    def __post_init__(self):
        m = int(self.node_count)
        if m < 2:
            raise DomainError("node_count must be >= 2")
        if not self.element_rest_length > 0.0:
            raise DomainError("element_rest_length must be positive")
        self.rest_configuration = np.asarray(self.rest_configuration, dtype=float)
        if self.rest_configuration.shape != (6 * m,):
            raise DomainError(f"rest_configuration must have length {6 * m}")
        if not np.all(np.isfinite(self.rest_configuration)):
            raise DomainError("rest_configuration must be finite")
        pos = self.rest_positions
        chords = np.linalg.norm(np.diff(pos, axis=0), axis=1)
        if np.any(chords < MIN_CHORD_LENGTH):
            raise DegenerateElementError("rest configuration has coincident nodes")
        if not np.allclose(chords, self.element_rest_length, rtol=1e-6, atol=1e-12):
            raise DomainError("rest node spacing does not match element_rest_length")

    @property
    def rest_positions(self):
        return self.rest_configuration.reshape(-1, 6)[:, :3].copy()

    @property
    def dof_count(self):
        return 6 * self.node_count

    @property
    def element_count(self):
        return self.node_count - 1

    @property
    def total_length(self):
        return self.element_count * self.element_rest_length


def straight_model(node_count, length, material, base=(0.0, 0.0, 0.0), axis=(1.0, 0.0, 0.0)):
    """Straight rest line from `base` along `axis` (reference beam.py:114-133)."""
    if node_count < 2:
        raise DomainError("node_count must be >= 2")
    axis = np.asarray(axis, dtype=float)
    axis = axis / np.linalg.norm(axis)
    l0 = length / (node_count - 1)
    coords = np.zeros((node_count, 6))
    coords[:, :3] = np.asarray(base, dtype=float) + np.outer(np.arange(node_count) * l0, axis)
    coords[:, 3:] = _axis_rotvec(axis)
    return RobotModel(node_count, l0, coords.ravel(), material)


@dataclass
class Configuration:
    """Generalised coordinates [tx ty tz rx ry rz] per node (reference beam.py:136-161)."""

    coords: np.ndarray
    timestep_index: int = 0

    def __post_init__(self):
        self.coords = np.asarray(self.coords, dtype=float)
        if self.coords.ndim != 1 or self.coords.size % 6 != 0:
            raise DomainError("coords must be a flat vector of length 6M")
        if not np.all(np.isfinite(self.coords)):
            raise DomainError("coords must be finite")

    @property
    def node_count(self):
        return self.coords.size // 6

    def positions(self):
        return self.coords.reshape(-1, 6)[:, :3]

    def rotation_vectors(self):
        return self.coords.reshape(-1, 6)[:, 3:]

    def director_frames(self):
        return rotvec_to_matrix(self.rotation_vectors())


# ----------------------------------------------------------------------------
# boundary conditions and actuation
# ----------------------------------------------------------------------------

ALL_DOFS = (0, 1, 2, 3, 4, 5)
TRANSLATION_DOFS = (0, 1, 2)


@dataclass(frozen=True)
class FixedNodeSpec:
    """Fixed DOFs of one node with optional prescribed increments (constraints.py:20-37)."""

    node_index: int
    fixed_dofs: tuple = ALL_DOFS
    prescribed_increment: tuple = None

    def __post_init__(self):
        if self.prescribed_increment is None:
            object.__setattr__(self, "prescribed_increment", tuple(0.0 for _ in self.fixed_dofs))
        if len(self.prescribed_increment) != len(self.fixed_dofs):
            raise DomainError("prescribed_increment length must match fixed_dofs")
        if any(d not in ALL_DOFS for d in self.fixed_dofs):
            raise DomainError("fixed_dofs entries must be in 0..5")
        if not all(np.isfinite(v) for v in self.prescribed_increment):
            raise DomainError("prescribed_increment must be finite")


def fixed_rows(specs, node_count):
    """Selector rows as (node, dof, increment) triples, validated like
    `assemble_fixed_constraints` (constraints.py:40-63)."""
    out, seen = [], set()
    for spec in specs:
        if not 0 <= spec.node_index < node_count:
            raise DomainError(f"fixed node {spec.node_index} out of range")
        for dof, inc in zip(spec.fixed_dofs, spec.prescribed_increment):
            key = (spec.node_index, dof)
            if key in seen:
                raise DomainError(f"duplicate fixed DOF {key}")
            seen.add(key)
            out.append((int(spec.node_index), int(dof), float(inc)))
    return out


@dataclass(frozen=True)
class CableSpec:
    """Cable attachment offset and pull direction in the tip frame (constraints.py:71-87)."""

    cable_index: int
    attachment_offset: np.ndarray = field(default=None)
    tension_direction: np.ndarray = field(default=None)

    def __post_init__(self):
        off = np.asarray(self.attachment_offset, dtype=float)
        d = np.asarray(self.tension_direction, dtype=float)
        nrm = np.linalg.norm(d)
        if not np.isfinite(nrm) or abs(nrm - 1.0) > 1e-9:
            raise DomainError("tension_direction must be a unit vector")
        object.__setattr__(self, "attachment_offset", off)
        object.__setattr__(self, "tension_direction", d)


def default_cables(radius=0.004):
    """Three cables, 120 deg apart on a circle in the tip section (constraints.py:90-103)."""
    out = []
    for j in range(3):
        phi = 2.0 * np.pi * j / 3.0
        out.append(CableSpec(j + 1, np.array([0.0, radius * np.cos(phi), radius * np.sin(phi)]),
                             np.array([-1.0, 0.0, 0.0])))
    return out


# ----------------------------------------------------------------------------
# lumen mesh
# ----------------------------------------------------------------------------

@dataclass
class TriangleMesh:
    """Triangle soup with winding normals facing the free cavity (mesh.py:19-61)."""

    vertices: np.ndarray
    triangles: np.ndarray
    normals: np.ndarray = field(init=False)

    def __post_init__(self):
        self.vertices = np.asarray(self.vertices, dtype=float).reshape(-1, 3)
        self.triangles = np.asarray(self.triangles, dtype=np.int64).reshape(-1, 3)
        if self.triangles.size == 0:
            raise MeshError("mesh has no triangles")
        if not np.all(np.isfinite(self.vertices)):
            raise MeshError("mesh vertices contain non-finite values")
        if self.triangles.min() < 0 or self.triangles.max() >= len(self.vertices):
            raise MeshError("triangle indices out of range")
        a, b, c = (self.vertices[self.triangles[:, k]] for k in range(3))
        cr = np.cross(b - a, c - a)
        nrm = np.linalg.norm(cr, axis=1)
        bad = np.flatnonzero(nrm * nrm < _DEGENERATE_TWICE_AREA_SQ)
        if bad.size:
            raise MeshError(f"degenerate (zero-area) triangles at indices {bad[:10].tolist()}")
        self.normals = cr / nrm[:, None]

    @property
    def triangle_count(self):
        return len(self.triangles)

    def corners(self):
        return self.vertices[self.triangles]

    def bounds(self):
        used = self.vertices[np.unique(self.triangles)]
        return used.min(axis=0), used.max(axis=0)

    def flip(self, which):
        which = np.asarray(which, dtype=np.int64)
        self.triangles[which] = self.triangles[which][:, [0, 2, 1]]
        self.normals[which] = -self.normals[which]


def orient_normals(mesh, reference_points):
    """Global winding vote toward `reference_points` (mesh.py:150-170)."""
    pts = np.asarray(reference_points, dtype=float).reshape(-1, 3)
    cen = mesh.corners().mean(axis=1)
    d2 = ((cen[:, None, :] - pts[None, :, :]) ** 2).sum(axis=2)
    off = pts[np.argmin(d2, axis=1)] - cen
    side = np.einsum("ij,ij->i", mesh.normals, off)
    w = 1.0 / np.maximum(np.einsum("ij,ij->i", off, off), 1e-18)
    if float(np.sign(side) @ w) < 0.0:
        mesh.flip(np.arange(mesh.triangle_count))
        return int(mesh.triangle_count)
    return 0


def make_rectangle(center, u_span, v_span, normal_axis="z"):
    """Two-triangle rectangle with +axis winding normal (mesh.py:332-345)."""
    spans = {"z": ((1, 0, 0), (0, 1, 0)), "y": ((0, 0, 1), (1, 0, 0)), "x": ((0, 1, 0), (0, 0, 1))}
    u, v = (np.asarray(a, dtype=float) for a in spans[normal_axis])
    c = np.asarray(center, dtype=float)
    hu, hv = u * u_span / 2, v * v_span / 2
    verts = np.array([c - hu - hv, c + hu - hv, c + hu + hv, c - hu + hv])
    return TriangleMesh(verts, np.array([[0, 1, 2], [0, 2, 3]]))


def make_tube(path_points, radii, segments=16):
    """Tube around a polyline, parallel-transported rings, normals inward (mesh.py:348-401)."""
    path = np.asarray(path_points, dtype=float)
    radii = np.broadcast_to(np.asarray(radii, dtype=float), (len(path),))
    if len(path) < 2:
        raise MeshError("tube path needs at least two points")
    tang = np.gradient(path, axis=0)
    tang /= np.linalg.norm(tang, axis=1, keepdims=True)
    ref = np.array([0.0, 0.0, 1.0])
    if abs(tang[0] @ ref) > 0.9:
        ref = np.array([0.0, 1.0, 0.0])
    n0 = np.cross(tang[0], ref)
    transported = [n0 / np.linalg.norm(n0)]
    for t in tang[1:]:
        prev = transported[-1]
        nn = prev - (prev @ t) * t
        ln = np.linalg.norm(nn)
        if ln < 1e-12:
            nn = np.cross(t, ref)
            ln = np.linalg.norm(nn)
        transported.append(nn / ln)
    ang = np.linspace(0.0, 2 * np.pi, segments, endpoint=False)
    cos_a, sin_a = np.cos(ang)[:, None], np.sin(ang)[:, None]
    rings = [p[None, :] + r * (cos_a * f[None, :] + sin_a * np.cross(t, f)[None, :])
             for p, r, f, t in zip(path, radii, transported, tang)]
    verts = np.vstack(rings)
    i = np.arange(len(path) - 1)[:, None]
    j = np.arange(segments)[None, :]
    j2 = (j + 1) % segments
    a0, a1 = i * segments + j, i * segments + j2
    b0, b1 = (i + 1) * segments + j, (i + 1) * segments + j2
    tris = np.stack([np.stack([a0, b0, a1], -1), np.stack([a1, b0, b1], -1)], axis=2).reshape(-1, 3)
    mesh = TriangleMesh(verts, tris)
    orient_normals(mesh, path)
    return mesh


_STL_RECORD = np.dtype([("normal", "<f4", (3,)), ("corners", "<f4", (3, 3)), ("attr", "<u2")])
_FLOAT = r"[-+]?(?:\d+\.?\d*|\.\d+)(?:[eE][-+]?\d+)?"


def _mesh_from_corner_list(corners, where):
    """Triangle soup (3k x 3 corner rows) -> indexed mesh: identical corners are
    merged; vertices come out in lexicographic order (numpy unique), triangles in
    file order -- the indexing the reference's loader produces (mesh.py:64-133)."""
    corners = np.asarray(corners, dtype=float).reshape(-1, 3)
    if corners.shape[0] == 0 or corners.shape[0] % 3:
        raise MeshError(f"{where}: corner count {corners.shape[0]} is not a positive multiple of 3")
    vertices, index = np.unique(corners, axis=0, return_inverse=True)
    return TriangleMesh(vertices, np.asarray(index).reshape(-1, 3))


def _read_stl(path):
    raw = path.read_bytes()
    if len(raw) >= 84:
        count = int(np.frombuffer(raw, dtype="<u4", count=1, offset=80)[0])
        if len(raw) == 84 + _STL_RECORD.itemsize * count:  # binary: header, count, 50-byte records
            rec = np.frombuffer(raw, dtype=_STL_RECORD, count=count, offset=84)
            return _mesh_from_corner_list(rec["corners"].astype(float), path)
    text = raw.decode("ascii", errors="replace")
    if not text.lstrip().lower().startswith("solid"):
        raise MeshError(f"{path}: neither a binary STL (size/count mismatch) nor an ASCII one ('solid' header)")
    rows = []
    for line in text.splitlines():
        tokens = line.split()
        if tokens[:1] != ["vertex"]:
            continue
        values = re.findall(_FLOAT, line[line.index("vertex") + 6:])
        if len(tokens) != 4 or len(values) != 3:
            raise MeshError(f"{path}: bad vertex record {line.strip()!r}")
        rows.append([float(v) for v in values])
    return _mesh_from_corner_list(rows, path)


def _read_obj(path):
    vertices, faces = [], []
    for number, line in enumerate(path.read_text().splitlines(), start=1):
        tokens = line.split()
        if not tokens or tokens[0][0] == "#":
            continue
        if tokens[0] == "v":
            vertices.append([float(t) for t in tokens[1:4]])
        elif tokens[0] == "f":
            corners = [int(t.partition("/")[0]) - 1 for t in tokens[1:]]
            if len(corners) != 3:
                raise MeshError(f"{path}:{number}: {len(corners)}-gon face; only triangles are supported "
                                "(export the OBJ triangulated)")
            faces.append(corners)
    if not faces:
        raise MeshError(f"{path}: the OBJ file has no faces")
    return TriangleMesh(np.asarray(vertices, dtype=float), np.asarray(faces))


_READERS = {".stl": _read_stl, ".obj": _read_obj}


def load_mesh(path):
    """Triangle mesh from an STL (binary or ASCII) or a triangulated OBJ file, in
    meters -- the loader contract of the reference (mesh.py:64-133; MeshError on
    missing / malformed files)."""
    path = Path(path)
    if not path.exists():
        raise MeshError(f"mesh file not found: {path}")
    reader = _READERS.get(path.suffix.lower())
    if reader is None:
        raise MeshError(f"unsupported mesh format {path.suffix!r} (.stl or .obj): {path}")
    return reader(path)


# ----------------------------------------------------------------------------
# solver settings, per-frame inputs and records
# ----------------------------------------------------------------------------

BACKENDS = ("accelerated_qp", "pgs_baseline")  # the reference's active_set_oracle stays a CPU test oracle


@dataclass
class SolverSettings:
    """ADMM / step settings (reference solver.py:41-68).

    The device path implements the `accelerated_qp` backend (the hot path) and
    the `pgs_baseline` comparison backend; the reference's
    exhaustive `active_set_oracle` remains a CPU test oracle.
    """

    eps_abs: float = 1e-6
    eps_rel: float = 1e-6
    max_iterations: int = 4000
    rho: float = 0.1
    sigma: float = 1e-6
    alpha: float = 1.6
    beta0: float = 0.005
    backend: str = "accelerated_qp"
    check_interval: int = 25
    adaptive_rho: bool = True
    scaling_iterations: int = 10
    polish: bool = True
    pgs_tol: float = 1e-6
    pgs_min_sweep_factor: int = 10

    def __post_init__(self):
        if self.eps_abs <= 0.0 or self.eps_rel <= 0.0 or self.pgs_tol <= 0.0:
            raise DomainError("tolerances must be positive")
        if not 0.0 < self.alpha < 2.0:
            raise DomainError("alpha must lie in (0, 2)")
        if self.beta0 <= 0.0:
            raise DomainError("beta0 must be positive")
        if self.backend not in BACKENDS:
            raise DomainError(f"unknown backend {self.backend!r}; the device path implements {BACKENDS}")
        if self.max_iterations < 1:
            raise DomainError("max_iterations must be >= 1")
        if self.check_interval < 1:
            raise DomainError("check_interval must be >= 1")


@dataclass
class StepInputs:
    """Per-frame control inputs (reference engine.py:40-49)."""

    tensions: np.ndarray = None
    insertion_increment: float = 0.0
    applied_force: np.ndarray = None

    def scaled(self, factor):
        return replace(self, insertion_increment=self.insertion_increment * factor)


@dataclass(frozen=True)
class ContactPoint:
    """One node contact (reference contact.py:22-30)."""

    contact_id: int
    element_index: int
    xi: float
    normal: np.ndarray
    plane_point: np.ndarray
    triangle_id: int
    gap: float


@dataclass
class FrameRecord:
    """Per-frame measurements (reference engine.py:52-81)."""

    t: float
    frame_index: int
    coords: np.ndarray
    n_c: int
    contact_force_vectors: np.ndarray
    contact_points: list
    tip_position: np.ndarray
    dx_norm: float
    iterations: int
    converged: bool
    retried: bool
    actuation_scale: float
    max_penetration: float
    complementarity_ok: bool
    complementarity_worst: float
    residual_norm: float
    timings_ms: dict
    factorization_count: int = 1

    @property
    def solve_ms(self):
        return self.timings_ms["solve"]

    @property
    def total_ms(self):
        return self.timings_ms["total"]


def contact_node(contact):
    """0-based node of a node contact (reference engine.py:286-288)."""
    return contact.element_index - 1 if contact.xi == 0.0 else contact.element_index
