"""CPU ORACLE -- test infrastructure only, never on the product path.

A numpy/scipy restatement of the reference's quasi-static solve
(`Engine.run_static`, /root/reference/pkg/src/cablefem/engine.py:267-283) for
the device path to be checked against.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
leg may import this module.

Parity pinning: `tests/test_oracle_golden.py` checks this restatement against
fixtures dumped from the real reference (`tests/golden/make_golden.py`, run in
the build container where /root/reference exists): element forces and
stiffness, rotation maps, contact detection (bit-exact), and full run_static
solves of cfg1/cfg2/cfg3/cfg3p/cfg4 samples (frame counts, per-frame ADMM
iteration counts, contact sets, coordinates, forces).

Third-party arithmetic the reference relies on, used identically here:
scipy 1.18.1 `Rotation` (so3.py:24-46) and SuperLU `splu` (solver.py:242).
Each function cites the reference lines it restates.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from scipy.spatial.transform import Rotation

RHO_MIN, RHO_MAX = 1e-6, 1e6          # solver.py:36
RHO_EQ_FACTOR = 1e3                    # solver.py:37
BIG = 1e30                             # solver.py:38
MIN_CHORD = 1e-9                       # beam.py:23

# status codes (same values as paper_2503_06922_b200.errors / include/accfem.h)
OK, DOMAIN, DEGENERATE, MESH, NONCONV, INFEASIBLE, ENGINE_SOLVER, ENGINE_MAX_FRAMES = range(8)


class OracleFailure(Exception):
    def __init__(self, status, message, payload=None):
        super().__init__(message)
        self.status = status
        self.payload = payload


# ----------------------------------------------------------------------------
# SO(3) -- so3.py:24-91 (scipy Rotation semantics)
# ----------------------------------------------------------------------------

def rot_exp(v):
    v = np.asarray(v, dtype=float)
    return Rotation.from_rotvec(v.reshape(-1, 3)).as_matrix().reshape(v.shape[:-1] + (3, 3))


def rot_log(m):
    m = np.asarray(m, dtype=float)
    return Rotation.from_matrix(m.reshape(-1, 3, 3)).as_rotvec().reshape(m.shape[:-2] + (3,))


def rot_compose(inc, base):
    """rotvec of exp(inc) @ exp(base) -- so3.py:40-46."""
    return (Rotation.from_rotvec(np.atleast_2d(inc)) * Rotation.from_rotvec(np.atleast_2d(base))).as_rotvec()


def min_rotation(a, b):
    """Minimal rotation a -> b, batched -- so3.py:49-82."""
    axis = np.cross(a, b)
    s = np.linalg.norm(axis, axis=1)
    c = np.einsum("ij,ij->i", a, b)
    out = np.empty((len(a), 3, 3))
    reg = s > 1e-12
    if reg.any():
        out[reg] = rot_exp(axis[reg] / s[reg, None] * np.arctan2(s[reg], c[reg])[:, None])
    out[~reg & (c > 0.0)] = np.eye(3)
    flip = ~reg & (c <= 0.0)
    if flip.any():
        ref = np.where(np.abs(a[flip, 0:1]) < 0.9, [[1.0, 0.0, 0.0]], [[0.0, 1.0, 0.0]])
        ax = np.cross(a[flip], ref)
        ax /= np.linalg.norm(ax, axis=1, keepdims=True)
        out[flip] = rot_exp(ax * np.pi)
    return out


def mid_rotation(ra, rb):
    """Geodesic midpoint ra exp(log(ra^T rb)/2) -- so3.py:85-91."""
    return ra @ rot_exp(0.5 * rot_log(np.swapaxes(ra, -1, -2) @ rb))


# ----------------------------------------------------------------------------
# beam chain -- beam.py
# ----------------------------------------------------------------------------

def local_stiffness(mat, l0):
    """12x12 Euler-Bernoulli element matrix -- beam.py:215-253."""
    E, A, I = mat.young_modulus, mat.cross_section_area, mat.bending_inertia
    GJ = mat.shear_modulus * mat.torsion_constant
    k = np.zeros((12, 12))

    def put(i, j, v):
        k[i, j] = k[j, i] = v

    ax, t = E * A / l0, GJ / l0
    b12, b6, b4, b2 = 12 * E * I / l0 ** 3, 6 * E * I / l0 ** 2, 4 * E * I / l0, 2 * E * I / l0
    for (i, j, v) in [(0, 0, ax), (6, 6, ax), (0, 6, -ax), (3, 3, t), (9, 9, t), (3, 9, -t),
                      (1, 1, b12), (7, 7, b12), (1, 7, -b12), (2, 2, b12), (8, 8, b12), (2, 8, -b12),
                      (4, 4, b4), (10, 10, b4), (4, 10, b2), (5, 5, b4), (11, 11, b4), (5, 11, b2),
                      (1, 5, b6), (1, 11, b6), (7, 5, -b6), (7, 11, -b6),
                      (2, 4, -b6), (2, 10, -b6), (8, 4, b6), (8, 10, b6)]:
        put(i, j, v)
    return k


class ChainModel:
    """Per-model constants -- RobotModel.__post_init__, beam.py:71-99."""

    def __init__(self, model):
        self.N = model.node_count
        self.l0 = model.element_rest_length
        rest = model.rest_configuration.reshape(-1, 6)
        self.rest_pos = rest[:, :3].copy()
        self.rest_dir = rot_exp(rest[:, 3:])
        self.rest_len = np.linalg.norm(np.diff(self.rest_pos, axis=0), axis=1)
        self.rest_frames = element_frames(self.rest_pos, self.rest_dir, np.eye(3)[None].repeat(self.N - 1, 0))
        mean0 = mid_rotation(self.rest_dir[:-1], self.rest_dir[1:])
        self.offsets = np.swapaxes(mean0, -1, -2) @ self.rest_frames
        self.k_local = local_stiffness(model.material, self.l0)
        self.dof = 6 * self.N


def element_frames(pos, dirs, offsets):
    """Co-rotational frames -- beam.py:256-271."""
    chords = pos[1:] - pos[:-1]
    lens = np.linalg.norm(chords, axis=1)
    if np.any(lens < MIN_CHORD):
        bad = int(np.argmax(lens < MIN_CHORD)) + 1
        raise OracleFailure(DEGENERATE, f"element {bad} has coincident nodes")
    pred = mid_rotation(dirs[:-1], dirs[1:]) @ offsets
    return min_rotation(pred[:, :, 0], chords / lens[:, None]) @ pred


def chain_state(cm, coords):
    c = coords.reshape(-1, 6)
    pos, dirs = c[:, :3], rot_exp(c[:, 3:])
    return pos, dirs, element_frames(pos, dirs, cm.offsets)


def internal_force(cm, coords, state=None):
    """F_int -- beam.py:283-325."""
    pos, dirs, frames = chain_state(cm, coords) if state is None else state
    et = np.swapaxes(frames, -1, -2)
    t0t = np.swapaxes(cm.rest_dir, -1, -2)
    d = np.zeros((cm.N - 1, 12))
    d[:, 3:6] = rot_log(et @ dirs[:-1] @ t0t[:-1] @ cm.rest_frames)
    d[:, 6] = np.linalg.norm(pos[1:] - pos[:-1], axis=1) - cm.rest_len
    d[:, 9:12] = rot_log(et @ dirs[1:] @ t0t[1:] @ cm.rest_frames)
    f_glob = np.einsum("eij,ekj->eki", frames, (d @ cm.k_local.T).reshape(-1, 4, 3)).reshape(-1, 12)
    out = np.zeros(cm.dof)
    idx = 6 * np.arange(cm.N - 1)[:, None] + np.arange(12)[None, :]
    np.add.at(out, idx.ravel(), f_glob.ravel())
    return out


def tangent_blocks(cm, frames):
    """Per-element global 12x12 blocks E kl E^T, symmetrised -- beam.py:335-347."""
    kl = cm.k_local.reshape(4, 3, 4, 3)
    blk = np.einsum("eij,pjqk,elk->epiql", frames, kl, frames, optimize=True).reshape(-1, 12, 12)
    return 0.5 * (blk + np.swapaxes(blk, -1, -2))


def tangent_matrix(cm, frames):
    """Assembled CSR tangent -- beam.py:347-356."""
    ke = tangent_blocks(cm, frames)
    idx = 6 * np.arange(cm.N - 1)[:, None] + np.arange(12)[None, :]
    rows = np.repeat(idx, 12, axis=1).ravel()
    cols = np.tile(idx, (1, 12)).ravel()
    mat = sp.coo_matrix((ke.ravel(), (rows, cols)), shape=(cm.dof, cm.dof)).tocsr()
    return (0.5 * (mat + mat.T)).tocsr()


def block_tridiagonal(csr, n_nodes):
    """(D[N,6,6], U[N-1,6,6]) view of a 6x6 block-tridiagonal CSR matrix."""
    dense = csr.toarray().reshape(n_nodes, 6, n_nodes, 6)
    i = np.arange(n_nodes)
    return dense[i, :, i, :].copy(), dense[i[:-1], :, i[:-1] + 1, :].copy()


# ----------------------------------------------------------------------------
# contact detection -- contact.py:49-120, mesh.py:199-329
# ----------------------------------------------------------------------------

def closest_points(p, a, b, c):
    """Ericson region classification, first match wins -- mesh.py:271-329."""
    ab, ac, ap = b - a, c - a, p - a
    dot = lambda u, v: np.einsum("ij,ij->i", u, v)  # noqa: E731
    d1, d2 = dot(ab, ap), dot(ac, ap)
    bp = p - b
    d3, d4 = dot(ab, bp), dot(ac, bp)
    cp = p - c
    d5, d6 = dot(ab, cp), dot(ac, cp)
    out = np.empty_like(a)
    done = np.zeros(len(a), dtype=bool)

    def take(mask, val):
        mask = mask & ~done
        out[mask] = val[mask]
        done[mask] = True

    take((d1 <= 0) & (d2 <= 0), a)
    take((d3 >= 0) & (d4 <= d3), b)
    take((d6 >= 0) & (d5 <= d6), c)
    with np.errstate(divide="ignore", invalid="ignore"):
        vc = d1 * d4 - d3 * d2
        v_ab = np.where(d1 - d3 != 0.0, d1 / (d1 - d3), 0.0)
        take((vc <= 0) & (d1 >= 0) & (d3 <= 0), a + v_ab[:, None] * ab)
        vb = d5 * d2 - d1 * d6
        w_ac = np.where(d2 - d6 != 0.0, d2 / (d2 - d6), 0.0)
        take((vb <= 0) & (d2 >= 0) & (d6 <= 0), a + w_ac[:, None] * ac)
        va = d3 * d6 - d5 * d4
        den_bc = (d4 - d3) + (d5 - d6)
        w_bc = np.where(den_bc != 0.0, (d4 - d3) / den_bc, 0.0)
        take((va <= 0) & (d4 - d3 >= 0) & (d5 - d6 >= 0), b + w_bc[:, None] * (c - b))
        den = va + vb + vc
        v = np.where(den != 0.0, vb / den, 0.0)
        w = np.where(den != 0.0, vc / den, 0.0)
    rest = ~done
    out[rest] = (a + v[:, None] * ab + w[:, None] * ac)[rest]
    return out


class Lumen:
    """Mesh arrays plus the per-triangle AABBs the reference filters on (mesh.py:204-207)."""

    def __init__(self, mesh):
        self.corners = mesh.corners()
        self.normals = mesh.normals
        self.lo = self.corners.min(axis=1)
        self.hi = self.corners.max(axis=1)

    def candidates(self, p, radius):
        """Triangles whose AABB meets the sphere, ascending -- mesh.py:245-268 (leaf test)."""
        g = np.maximum(self.lo - p, np.maximum(0.0, p - self.hi))
        return np.flatnonzero(np.einsum("ij,ij->i", g, g) <= radius * radius)


def detect(lumen, positions, margin, radius):
    """Node contacts: list of (node, tri, gap, plane_point, normal) -- contact.py:49-120."""
    radius = max(radius, margin)
    nodes, cands = [], []
    for k in range(len(positions)):
        cc = lumen.candidates(positions[k], radius)
        if cc.size:
            nodes.append(np.full(cc.size, k))
            cands.append(cc)
    if not nodes:
        return []
    nodes = np.concatenate(nodes)
    cands = np.concatenate(cands)
    cor = lumen.corners[cands]
    p = positions[nodes]
    cl = closest_points(p, cor[:, 0], cor[:, 1], cor[:, 2])
    off = p - cl
    eu = np.linalg.norm(off, axis=1)
    pg = np.einsum("ij,ij->i", lumen.normals[cands], off)
    signed = np.where(pg >= 0.0, eu, -eu)
    ok = (signed <= margin) & (eu <= radius) & (np.abs(pg) >= 0.9 * eu - 1e-12)
    if not ok.any():
        return []
    ne = nodes[ok]
    order = np.lexsort((cands[ok], signed[ok], ne))
    _, first = np.unique(ne[order], return_index=True)
    win = np.flatnonzero(ok)[order[first]]
    return [(int(nodes[b]), int(cands[b]), float(pg[b]), cl[b].copy(), -lumen.normals[cands[b]])
            for b in win]


# ----------------------------------------------------------------------------
# QP solve -- solver.py
# ----------------------------------------------------------------------------

def _ninf(v):
    return float(np.abs(v).max()) if np.size(v) else 0.0


class QP:
    """Stacked interval form l <= A dx <= u, equalities first -- solver.py:144-162."""

    def __init__(self, h, g, a_fn, b_fn, a_c, b_c):
        self.h = sp.csc_matrix(h)
        self.g = g
        self.n = h.shape[0]
        self.n_eq = a_fn.shape[0]
        self.n_c = a_c.shape[0]
        self.a_fn, self.b_fn, self.a_c, self.b_c = a_fn.tocsr(), b_fn, a_c.tocsr(), b_c
        if self.n_eq + self.n_c:
            self.a = sp.vstack([self.a_fn, self.a_c], format="csr")
        else:
            self.a = sp.csr_matrix((0, self.n))
        self.lower = np.concatenate([b_fn, np.full(self.n_c, -BIG)])
        self.upper = np.concatenate([b_fn, b_c])


class Result:
    def __init__(self, dx, y_c, y_fn, pri, dua, iterations, converged, rho_estimate=None):
        self.dx, self.y_c, self.y_fn = dx, y_c, y_fn
        self.primal_residual, self.dual_residual = pri, dua
        self.iterations, self.converged, self.rho_estimate = iterations, converged, rho_estimate
        self.polish_applied = False


def ruiz(h, a, g, sweeps):
    """Modified Ruiz equilibration + cost scaling -- solver.py:169-212."""
    n, m = h.shape[0], a.shape[0]
    hc_ = sp.coo_matrix(h)
    ac_ = sp.coo_matrix(a)
    hr, hcol, hv = hc_.row, hc_.col, hc_.data.copy()
    ar, acol, av = ac_.row, ac_.col, ac_.data.copy()
    g = g.copy()
    d, e, c = np.ones(n), np.ones(m), 1.0
    for _ in range(sweeps):
        colh = np.zeros(n)
        np.maximum.at(colh, hcol, np.abs(hv))
        cola = np.zeros(m)
        if m:
            np.maximum.at(colh, acol, np.abs(av))
            np.maximum.at(cola, ar, np.abs(av))
        dd = 1.0 / np.sqrt(np.where(colh > 1e-12, colh, 1.0))
        ee = 1.0 / np.sqrt(np.where(cola > 1e-12, cola, 1.0)) if m else cola
        hv *= dd[hr] * dd[hcol]
        if m:
            av *= ee[ar] * dd[acol]
        g *= dd
        d *= dd
        if m:
            e *= ee
        colh = np.zeros(n)
        np.maximum.at(colh, hcol, np.abs(hv))
        gam = 1.0 / max(colh.mean() if n else 0.0, _ninf(g), 1e-12)
        hv *= gam
        g *= gam
        c *= gam
    return (sp.csc_matrix((hv, (hr, hcol)), shape=(n, n)), sp.csr_matrix((av, (ar, acol)), shape=(m, n)),
            g, d, e, c)


def certificate(qp, d, e, c, dy_scaled, s):
    """OSQP primal-infeasibility test -- solver.py:424-446."""
    if qp.a.shape[0] == 0:
        return None
    dy = e * dy_scaled / c
    nd = _ninf(dy)
    eps = max(s.eps_abs, 1e-10)
    if nd <= eps:
        return None
    dy = dy / nd
    support = float(qp.upper @ np.maximum(dy, 0.0) + qp.lower @ np.minimum(dy, 0.0))
    if support < -eps and _ninf(qp.a.T @ dy) <= eps:
        return dy
    return None


def admm(qp, s, y0=None, rho=None):
    """Relaxed ADMM with one cached factorization -- solver.py:250-385."""
    if qp.n_c == 0:
        return equality_direct(qp, s)
    n, m, n_eq = qp.n, qp.a.shape[0], qp.n_eq
    hs, as_, gs, d, e, c = ruiz(qp.h, qp.a, qp.g, s.scaling_iterations)
    ls = np.where(np.isfinite(qp.lower), e * qp.lower, qp.lower)
    us = np.where(np.isfinite(qp.upper), e * qp.upper, qp.upper)
    rho_bar = float(np.clip(s.rho if rho is None else rho, RHO_MIN, RHO_MAX))
    rv = np.full(m, rho_bar)
    rv[:n_eq] = np.clip(rho_bar * RHO_EQ_FACTOR, RHO_MIN, RHO_MAX)
    kkt = sp.bmat([[hs + s.sigma * sp.eye(n), as_.T], [as_, -sp.diags(1.0 / rv)]], format="csc")
    lu = spla.splu(kkt)
    x = np.zeros(n)
    y = np.zeros(m) if y0 is None else c * np.asarray(y0, dtype=float) / e
    z = np.clip(as_ @ x, ls, us)
    al, sg = s.alpha, s.sigma
    pri = dua = np.inf
    infeasible = None
    rho_est = rho_bar
    k = 0
    for k in range(1, s.max_iterations + 1):
        sol = lu.solve(np.concatenate([sg * x - gs, z - y / rv]))
        xt = sol[:n]
        zt = z + (sol[n:] - y) / rv
        x_prev, y_prev = x, y
        x = al * xt + (1.0 - al) * x_prev
        zr = al * zt + (1.0 - al) * z
        zn = np.clip(zr + y / rv, ls, us)
        y = y + rv * (zr - zn)
        z = zn
        if k <= 8 or k % s.check_interval == 0 or k == s.max_iterations:
            xu, yu, zu = d * x, e * y / c, z / e
            ax_ = qp.a @ xu
            hx = qp.h @ xu
            aty = qp.a.T @ yu
            pri, dua = _ninf(ax_ - zu), _ninf(hx + qp.g + aty)
            ps = max(_ninf(ax_), _ninf(zu))
            ds = max(_ninf(hx), _ninf(aty), _ninf(qp.g))
            if pri <= s.eps_abs + s.eps_rel * ps and dua <= s.eps_abs + s.eps_rel * ds:
                break
            if k % s.check_interval == 0:
                infeasible = certificate(qp, d, e, c, y - y_prev, s)
                if infeasible is not None:
                    break
                if k == s.check_interval:
                    ratio = (pri / max(ps, 1e-12)) / max(dua / max(ds, 1e-12), 1e-12)
                    rho_est = float(np.clip(rho_bar * np.sqrt(ratio), RHO_MIN, RHO_MAX))
    if infeasible is not None:
        raise OracleFailure(INFEASIBLE, "constraints are primal infeasible", infeasible)
    dx, yf, zu = d * x, e * y / c, z / e
    ax_ = qp.a @ dx
    hx = qp.h @ dx
    aty = qp.a.T @ yf
    pri, dua = _ninf(ax_ - zu), _ninf(hx + qp.g + aty)
    conv = pri <= s.eps_abs + s.eps_rel * max(_ninf(ax_), _ninf(zu)) and \
        dua <= s.eps_abs + s.eps_rel * max(_ninf(hx), _ninf(aty), _ninf(qp.g))
    res = Result(dx, np.maximum(yf[n_eq:], 0.0), yf[:n_eq], pri, dua, k, bool(conv),
                 rho_est if (s.adaptive_rho and k >= 3 * s.check_interval) else None)
    if s.polish and res.converged:
        polish(qp, res, s)
    if not res.converged:
        raise OracleFailure(NONCONV, f"ADMM did not converge in {s.max_iterations} iterations", res)
    return res


def equality_direct(qp, s):
    """Contact-free frame: regularised KKT + 3 refinements -- solver.py:388-421."""
    n, m = qp.n, qp.n_eq
    if m == 0:
        dx = spla.splu(sp.csc_matrix(qp.h)).solve(-qp.g)
        yfn = np.zeros(0)
    else:
        exact = sp.bmat([[qp.h, qp.a_fn.T], [qp.a_fn, None]], format="csc")
        reg = sp.bmat([[qp.h + s.sigma * sp.eye(n), qp.a_fn.T], [qp.a_fn, -s.sigma * sp.eye(m)]], format="csc")
        lu = spla.splu(reg)
        rhs = np.concatenate([-qp.g, qp.b_fn])
        sol = lu.solve(rhs)
        for _ in range(3):
            sol = sol + lu.solve(rhs - exact @ sol)
        dx, yfn = sol[:n], sol[n:]
    pri = _ninf(qp.a_fn @ dx - qp.b_fn) if m else 0.0
    dua = _ninf(qp.h @ dx + qp.g + (qp.a_fn.T @ yfn if m else 0.0))
    if pri > max(s.eps_abs, 1e-8 * max(1.0, _ninf(qp.b_fn) if m else 0.0)):
        raise OracleFailure(INFEASIBLE, f"equality constraints inconsistent (residual {pri:.3e})")
    return Result(dx, np.zeros(0), yfn, pri, dua, 0, True)


def polish(qp, res, s):
    """Active-set refinement, <= 6 rounds -- solver.py:449-497."""
    m, n_eq = qp.a.shape[0], qp.n_eq
    slack = qp.upper - qp.a @ res.dx
    tol_act = max(10 * s.eps_abs, 1e-12)
    act = np.zeros(m, dtype=bool)
    act[:n_eq] = True
    act[n_eq:] = (res.y_c > tol_act) | (slack[n_eq:] < tol_act)
    best = None
    for _ in range(6):
        idx = np.flatnonzero(act)
        if idx.size == 0:
            break
        pt = active_subset(qp, idx)
        if pt is None:
            return
        dxp, yp = pt
        neg = (yp[n_eq:] < -1e-11) & act[n_eq:]
        viol = ((qp.a[n_eq:] @ dxp - qp.upper[n_eq:] > tol_act) & ~act[n_eq:]) if m > n_eq \
            else np.zeros(0, dtype=bool)
        if not neg.any() and not viol.any():
            best = pt
            break
        act[n_eq:][neg] = False
        act[n_eq:][viol] = True
    if best is None:
        return
    dxp, yp = best
    feas = qp.a @ dxp - qp.upper
    pri = max(_ninf(np.maximum(feas, 0.0)), _ninf(qp.a[:n_eq] @ dxp - qp.upper[:n_eq]) if n_eq else 0.0)
    dua = _ninf(qp.h @ dxp + qp.g + qp.a.T @ yp)
    if not np.all(np.isfinite(dxp)):
        return
    if pri <= max(res.primal_residual, s.eps_abs) and dua <= max(res.dual_residual, s.eps_abs):
        res.dx, res.y_fn, res.y_c = dxp, yp[:n_eq], np.maximum(yp[n_eq:], 0.0)
        res.primal_residual, res.dual_residual = pri, dua
        res.polish_applied = True


def active_subset(qp, idx):
    """Regularised reduced KKT + one refinement -- solver.py:500-528."""
    n, m = qp.n, qp.a.shape[0]
    aa = qp.a[idx].tocsr()
    ba = qp.upper[idx]
    delta = 1e-9
    reg = sp.bmat([[qp.h + delta * sp.eye(n), aa.T], [aa, -delta * sp.eye(idx.size)]], format="csc")
    try:
        lu = spla.splu(reg)
    except RuntimeError:
        return None
    rhs = np.concatenate([-qp.g, ba])
    sol = lu.solve(rhs)
    dxp, mu = sol[:n], sol[n:]
    sol = sol + lu.solve(np.concatenate([-qp.g - qp.h @ dxp - aa.T @ mu, ba - aa @ dxp]))
    if not np.all(np.isfinite(sol)):
        return None
    yp = np.zeros(m)
    yp[idx] = sol[n:]
    return sol[:n], yp


# ----------------------------------------------------------------------------
# engine -- engine.py:84-297
# ----------------------------------------------------------------------------

class FrameOut:
    __slots__ = ("coords", "n_c", "contacts", "forces", "dx_norm", "iterations", "converged", "retried",
                 "actuation_scale", "max_penetration", "compl_ok", "compl_worst", "residual", "y_c")


class OracleEngine:
    """run_static / step of one scene, with the reference's cross-frame state."""

    def __init__(self, model, mesh=None, cables=(), fixed_specs=(), settings=None, margin=1e-4,
                 uniform_load=None):
        self.cm = ChainModel(model)
        self.lumen = Lumen(mesh) if mesh is not None else None
        self.cables = list(cables)
        self.settings = settings
        self.margin = float(margin)
        self.uniform = None if uniform_load is None else np.asarray(uniform_load, dtype=float)
        self.fixed = []
        seen = set()
        for spec in fixed_specs:
            for dof, inc in zip(spec.fixed_dofs, spec.prescribed_increment):
                key = (spec.node_index, dof)
                if key in seen:
                    raise OracleFailure(DOMAIN, f"duplicate fixed DOF {key}")
                seen.add(key)
                self.fixed.append((spec.node_index, dof, float(inc)))
        rp = self.cm.rest_pos
        self.axis = (rp[1] - rp[0]) / np.linalg.norm(rp[1] - rp[0])
        self.warm = {}
        self.warm_fixed = None
        self.rho = settings.rho

    # -- assembly pieces ----------------------------------------------------
    def fixed_system(self, insertion, scale=1.0):
        """Selector rows + insertion on node-0 translations -- engine.py:123-134."""
        nf, n = len(self.fixed), self.cm.dof
        a = sp.csr_matrix((np.ones(nf), (np.arange(nf), [6 * nd + dof for nd, dof, _ in self.fixed])),
                          shape=(nf, n))
        b = np.array([inc for _, _, inc in self.fixed], dtype=float)
        if insertion:
            inc = self.axis * insertion
            for r, (nd, dof, _) in enumerate(self.fixed):
                if nd == 0 and dof < 3:
                    b[r] += inc[dof]
        return a, b * scale

    def external_force(self, frames, tensions, applied):
        """Cable tip wrench + applied + uniform -- engine.py:108-121, constraints.py:111-136."""
        f = np.zeros(self.cm.dof)
        if self.cables and tensions is not None:
            tm = frames[-1]
            tensions = np.asarray(tensions, dtype=float)
            if np.any(tensions < 0.0):
                raise OracleFailure(DOMAIN, "cable tensions must be >= 0 (cables cannot push)")
            force, moment = np.zeros(3), np.zeros(3)
            for cab, t in zip(self.cables, tensions):
                fl = t * cab.tension_direction
                force += tm @ fl
                moment += tm @ np.cross(cab.attachment_offset, fl)
            f[-6:-3] += force
            f[-3:] += moment
        if applied is not None:
            f += applied
        if self.uniform is not None:
            f.reshape(-1, 6)[:, :3] += self.uniform
        return f

    def contact_rows(self, contacts, coords):
        """Node-contact rows n^T at the node translations, b = n.X - n.p -- contact.py:148-178."""
        nc, n = len(contacts), self.cm.dof
        rows, cols, vals = [], [], []
        b = np.zeros(nc)
        for i, (node, _, _, pp, nrm) in enumerate(contacts):
            # node 0 -> element 1, xi = 0 (weights on node a); node k -> element k, xi = l0 (node b)
            elem = 1 if node == 0 else node
            a_node, b_node = elem - 1, elem
            wa, wb = (1.0, 0.0) if node == 0 else (0.0, 1.0)
            for dof in range(3):
                rows += [i, i]
                cols += [6 * a_node + dof, 6 * b_node + dof]
                vals += [nrm[dof] * wa, nrm[dof] * wb]
            p = wa * coords[6 * a_node:6 * a_node + 3] + wb * coords[6 * b_node:6 * b_node + 3]
            b[i] = nrm @ pp - nrm @ p
        return sp.csr_matrix((vals, (rows, cols)), shape=(nc, n)), b

    # -- one frame ------------------------------------------------------------
    def step(self, coords, tensions=None, applied=None, insertion=0.0):
        cm, s = self.cm, self.settings
        state = chain_state(cm, coords)
        frames = state[2]
        k = tangent_matrix(cm, frames)
        fint = internal_force(cm, coords, state)
        contacts = []
        if self.lumen is not None:
            contacts = detect(self.lumen, state[0], self.margin, self.margin + s.beta0)
        a_c, b_c = self.contact_rows(contacts, coords) if contacts else (sp.csr_matrix((0, cm.dof)), np.zeros(0))
        a_fn, b_fn = self.fixed_system(insertion)
        f_a = self.external_force(frames, tensions, applied)
        y0 = np.array([self.warm.get(c[0], 0.0) for c in contacts]) if contacts else None
        yfix = np.zeros(a_fn.shape[0]) if self.warm_fixed is None or len(self.warm_fixed) != a_fn.shape[0] \
            else self.warm_fixed
        ystack = np.concatenate([yfix, y0]) if y0 is not None else None
        qp = QP(k, fint - f_a, a_fn, b_fn, a_c, b_c)
        retried = False
        try:
            res = admm(qp, s, y0=ystack, rho=self.rho)
        except OracleFailure as first:
            if first.status != NONCONV:
                raise
            retried = True
            if s.adaptive_rho and first.payload is not None and first.payload.rho_estimate is not None:
                self.rho = first.payload.rho_estimate
            a2, b2 = self.fixed_system(insertion * 0.5)
            qp = QP(k, fint - f_a, a2, b2, a_c, b_c)
            try:
                res = admm(qp, s, y0=ystack, rho=self.rho)
            except OracleFailure as second:
                if second.status != NONCONV:
                    raise
                raise OracleFailure(ENGINE_SOLVER, "solver failed twice", second.payload) from None
        # complementarity report (solver.py:781-800) on the unlimited result
        vc = a_c @ res.dx - b_c
        vf = a_fn @ res.dx - b_fn
        scale = max(1.0, _ninf(res.y_c), _ninf(a_c @ res.dx) if len(contacts) else 0.0)
        mult_v = max(0.0, -(res.y_c.min() if res.y_c.size else 0.0))
        gap_v = float(np.maximum(vc, 0.0).max()) if vc.size else 0.0
        prod_v = float(np.abs(res.y_c * vc).max()) if vc.size else 0.0
        eq_v = _ninf(vf)
        tol = 1e-6
        ok = mult_v <= tol and gap_v <= tol and prod_v <= tol * scale and eq_v <= tol
        # step limit (solver.py:803-823)
        nrm = float(np.linalg.norm(res.dx))
        fac = 1.0 if (nrm <= s.beta0 or nrm == 0.0) else s.beta0 / nrm
        dx, yc, yfn = res.dx * fac, res.y_c * fac, res.y_fn * fac
        # advance (engine.py:291-297)
        c6 = coords.reshape(-1, 6).copy()
        d6 = dx.reshape(-1, 6)
        c6[:, :3] += d6[:, :3]
        c6[:, 3:] = rot_compose(d6[:, 3:], c6[:, 3:])
        new = c6.ravel()
        # warm state (engine.py:248-255)
        self.warm = {c[0]: float(y) for c, y in zip(contacts, res.y_c)}
        self.warm_fixed = res.y_fn.copy()
        est = res.rho_estimate
        if s.adaptive_rho and est is not None and (est > 5.0 * self.rho or est < self.rho / 5.0):
            self.rho = est
        out = FrameOut()
        out.coords = new
        out.n_c = len(contacts)
        out.contacts = contacts
        out.y_c = yc
        out.forces = (-yc[:, None] * np.array([c[4] for c in contacts])) if contacts else np.zeros((0, 3))
        out.residual = float(np.linalg.norm(internal_force(cm, new) + a_c.T @ yc + a_fn.T @ yfn - f_a))
        pen0 = max(0.0, -min((c[2] for c in contacts), default=0.0))
        pen1 = max(0.0, float(-(b_c - a_c @ dx).min())) if contacts else 0.0
        out.max_penetration = max(pen0, pen1)
        out.dx_norm = float(np.linalg.norm(dx))
        out.iterations = res.iterations
        out.converged = res.converged
        out.retried = retried
        out.actuation_scale = fac
        out.compl_ok = bool(ok)
        out.compl_worst = max(gap_v, mult_v, prod_v, eq_v)
        return out

    def run_static(self, x0, tensions=None, applied=None, tol=1e-9, max_frames=5000):
        """Frames until |dx| <= tol -- engine.py:267-283.  Returns (coords, [FrameOut])."""
        x = np.asarray(x0, dtype=float).copy()
        recs = []
        for _ in range(max_frames):
            fr = self.step(x, tensions, applied)
            x = fr.coords
            recs.append(fr)
            if fr.dx_norm <= tol:
                return x, recs
        raise OracleFailure(ENGINE_MAX_FRAMES, f"static mode did not reach |dx| <= {tol} in {max_frames} frames",
                            recs)


def solve_workload(w, indices=None):
    """Oracle run_static over scenarios of a Workload; one fresh engine each
    (the batch semantics of `accfem_solve_batch`).  Returns a list of dicts."""
    idx = range(w.size) if indices is None else indices
    out = []
    for i in idx:
        eng = OracleEngine(**w.engine_kwargs())
        rec = {"status": OK}
        try:
            x, recs = eng.run_static(w.x0[i], None if w.tensions is None else w.tensions[i],
                                     None if w.applied is None else w.applied[i], tol=w.tol,
                                     max_frames=w.max_frames)
        except OracleFailure as exc:
            rec["status"] = exc.status
            out.append(rec)
            continue
        last = recs[-1]
        rec.update(coords=x, frames=len(recs), iterations=np.array([r.iterations for r in recs], np.int32),
                   n_c=np.array([r.n_c for r in recs], np.int32), residual=last.residual,
                   contact_nodes=np.array([c[0] for c in last.contacts], np.int32),
                   contact_tris=np.array([c[1] for c in last.contacts], np.int32),
                   contact_gaps=np.array([c[2] for c in last.contacts]),
                   contact_forces=last.forces.reshape(-1, 3), records=recs)
        out.append(rec)
    return out
