"""CPU ORACLE for the citywind RANS step path -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference algorithm
(/root/reference/pkg/src/citywind/, "the reference" below) used as the parity
checker for the CUDA path in ``paper_2204_01117_b200``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline / reference arm
may import it.  The product never routes through this module.

Layout.  Unlike the reference (C-order (nx, ny, nz) arrays) every field here
is stored x-fastest, shaped (nz, ny, nx[+1]) -- the device layout -- so the
oracle and the GPU fields compare element for element.  Pressure unknowns are
numbered in C order of that layout, which *is* the reference's x-fastest
numbering (linalg.py:53-54,71-72), so the PCG vectors coincide too.

Arithmetic.  Every expression keeps the reference's operation order, so on
the same inputs the oracle reproduces the reference's float64 results (checked
against fixtures generated from the reference by scripts/make_golden.py; see
tests/test_oracle_golden.py).  A and W are assembled as scipy CSR exactly as
the reference does (linalg.py:57-126, 201-232), so A.p and W.r are the same
csr_matvec calls.

Pinned: yes -- against tests/golden/*.npz produced by importing the reference.
"""
from __future__ import annotations

import hashlib
import math
import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

AIR, BUILDING, TREE, INLET, OUTLET, SOLID_WALL = range(6)
_LABEL_NAMES = {"inlet": INLET, "outlet": OUTLET, "solid_wall": SOLID_WALL}
_FACES = ("x_min", "x_max", "y_min", "y_max", "z_min", "z_max")
VON_KARMAN = 0.41
DIV_REDUCTION_TARGET = 10.0 ** -4.5          # solver.py:232
K_FLOOR, OMEGA_FLOOR = 1e-12, 1e-8           # turbulence.py:14-15


# ---------------------------------------------------------------------------
# grid, parameters, state  (grid.py:33-84, solver.py:26-97, grid.py:492-571)

@dataclass(frozen=True)
class Grid:
    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    origin: tuple = (0.0, 0.0, 0.0)

    @property
    def is_2d(self):
        return self.nz == 1

    @property
    def cshape(self):                       # device/oracle array shape of a cell field
        return (self.nz, self.ny, self.nx)

    def h(self, axis):
        return (self.dx, self.dy, self.dz)[axis]

    def n(self, axis):
        return (self.nx, self.ny, self.nz)[axis]


def aax(axis):
    """physical axis (0=x,1=y,2=z) -> array axis in the x-fastest layout."""
    return 2 - axis


def _sl(axis, s):
    t = [slice(None)] * 3
    t[aax(axis)] = s
    return tuple(t)


@dataclass
class Params:
    dt: float = 0.1
    nu: float = 1.57e-5
    cd_tree: float = 0.2
    cd_building: float = 1.0
    drag_a: float = 0.62
    drag_b: float = 2.5
    drag_eps: float = 1e-10
    c_mu: float = 0.09
    alpha: float = 0.52
    beta: float = 0.0708
    sigma: float = 0.5
    sigma_star: float = 0.6
    c_lim: float = 7.0 / 8.0
    turb_intensity: float = 0.05
    u_ref: float = 1.0
    length_scale: float = 10.0
    turbulence: bool = True

    def inlet_k_omega(self):
        return inlet_turbulence(self.turb_intensity, self.u_ref, self.length_scale, self.c_mu)


def inlet_turbulence(intensity, u_ref, length_scale, c_mu=0.09):
    """turbulence.py:26-33"""
    k = 1.5 * (intensity * u_ref) ** 2
    k = max(k, K_FLOOR)
    om = c_mu ** (-0.25) * np.sqrt(k) / length_scale
    return k, max(om, OMEGA_FLOOR)


def nu_stable(grid, dt):
    """turbulence.py:18-23"""
    s = 1.0 / grid.dx ** 2 + 1.0 / grid.dy ** 2
    if not grid.is_2d:
        s += 1.0 / grid.dz ** 2
    return 1.0 / (2.0 * dt * s)


@dataclass
class Inlet:
    kind: str = "uniform"
    speed: float = 1.0
    u_star: float = 0.5
    z0: float = 0.5
    kappa: float = VON_KARMAN
    direction: tuple = (1.0, 0.0)

    def __post_init__(self):
        d = np.asarray(self.direction, dtype=float)[:2]
        nrm = np.linalg.norm(d)
        self.direction = (float(d[0] / nrm), float(d[1] / nrm))

    def speed_at(self, z):
        """solver.py:75-82"""
        z = np.asarray(z, dtype=float)
        if self.kind == "uniform":
            return np.full_like(z, self.speed)
        out = np.zeros_like(z)
        m = z > self.z0
        out[m] = self.u_star / self.kappa * np.log(z[m] / self.z0)
        return out

    def rotated(self, degrees):
        a = np.deg2rad(degrees)
        dx, dy = self.direction
        return Inlet(self.kind, self.speed, self.u_star, self.z0, self.kappa,
                     (dx * np.cos(a) - dy * np.sin(a), dx * np.sin(a) + dy * np.cos(a)))


@dataclass
class State:
    grid: Grid
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    p: np.ndarray
    k: np.ndarray
    omega: np.ndarray
    nu_t: np.ndarray
    labels: np.ndarray
    phi: np.ndarray
    lad: np.ndarray
    time: float = 0.0
    step_count: int = 0

    @classmethod
    def zeros(cls, grid, labels=None, phi=None, lad=None, k0=1e-6, omega0=1.0):
        nz, ny, nx = grid.cshape
        c = grid.cshape
        return cls(grid,
                   np.zeros((nz, ny, nx + 1)), np.zeros((nz, ny + 1, nx)),
                   np.zeros((nz + 1, ny, nx)), np.zeros(c), np.full(c, k0),
                   np.full(c, omega0), np.full(c, k0 / omega0),
                   np.zeros(c, np.int8) if labels is None else labels,
                   np.ones(c) if phi is None else phi,
                   np.zeros(c) if lad is None else lad)

    def copy(self):
        return State(self.grid, *(getattr(self, n).copy() for n in
                                  ("u", "v", "w", "p", "k", "omega", "nu_t",
                                   "labels", "phi", "lad")),
                     time=self.time, step_count=self.step_count)

    def comp(self, axis):
        return (self.u, self.v, self.w)[axis]

    def set_comp(self, axis, arr):
        setattr(self, "uvw"[axis], arr)

    def cell_velocity(self):
        """grid.py:561-566 -> list [uc, vc, wc]"""
        return [0.5 * (a[_sl(ax, slice(None, -1))] + a[_sl(ax, slice(1, None))])
                for ax, a in enumerate((self.u, self.v, self.w))]

    def speed(self):
        uc, vc, wc = self.cell_velocity()
        return np.sqrt(uc * uc + vc * vc + wc * wc)


def interior_mask(labels):
    """grid.py:481-484"""
    return (labels == AIR) | (labels == BUILDING) | (labels == TREE)


def classify_boundary(grid, faces):
    """grid.py:439-470: later writes win, ascending priority Outlet<Wall<Inlet."""
    req = _FACES[:4] if grid.is_2d else _FACES
    lab = np.zeros(grid.cshape, np.int8)
    slab = {"x_min": _sl(0, slice(0, 1)), "x_max": _sl(0, slice(grid.nx - 1, grid.nx)),
            "y_min": _sl(1, slice(0, 1)), "y_max": _sl(1, slice(grid.ny - 1, grid.ny)),
            "z_min": _sl(2, slice(0, 1)), "z_max": _sl(2, slice(grid.nz - 1, grid.nz))}
    for want in (OUTLET, SOLID_WALL, INLET):
        for f in req:
            if faces[f] == want:
                lab[slab[f]] = want
    return lab


def merge_labels(boundary, interior):
    """grid.py:473-478"""
    out = boundary.copy()
    m = (boundary == AIR) & (interior != AIR)
    out[m] = interior[m]
    return out


# ---------------------------------------------------------------------------
# pressure operator, AI preconditioner, PCG  (linalg.py)

class SingularSystemError(ValueError):
    pass


@dataclass
class PressureSystem:
    A: sp.csr_matrix
    index: np.ndarray
    unknown: np.ndarray

    @property
    def n(self):
        return self.A.shape[0]


def build_pressure_matrix(grid, labels):
    """linalg.py:57-126 (7-point, outlet Dirichlet, inlet/wall Neumann)."""
    unk = interior_mask(labels)
    n = int(unk.sum())
    if n == 0:
        raise ValueError("no flow cells to solve for")
    index = np.full(grid.cshape, -1, np.int64)
    index[unk] = np.arange(n)
    diag = np.zeros(grid.cshape)
    rows, cols, vals = [], [], []
    n_dir = 0
    for axis, step in ((0, 1), (0, -1), (1, 1), (1, -1), (2, 1), (2, -1)):
        if grid.is_2d and axis == 2:
            continue
        w = 1.0 / grid.h(axis) ** 2
        N = grid.n(axis)
        src = _sl(axis, slice(0, N - 1) if step > 0 else slice(1, N))
        dst = _sl(axis, slice(1, N) if step > 0 else slice(0, N - 1))
        a_unk = unk[src]
        pair = a_unk & unk[dst]
        rows.append(index[src][pair])
        cols.append(index[dst][pair])
        vals.append(np.full(int(pair.sum()), -w))
        outl = a_unk & (labels[dst] == OUTLET)
        n_dir += int(outl.sum())
        d = diag[src]                       # view: accumulate in offset order
        d[pair] += w
        d[outl] += w
    if n_dir == 0:
        raise SingularSystemError("no outlet cells: pressure defined only up to a constant")
    dvec = diag[unk]
    r = np.concatenate(rows + [np.arange(n)])
    c = np.concatenate(cols + [np.arange(n)])
    v = np.concatenate(vals + [dvec])
    A = sp.csr_matrix((v, (r, c)), shape=(n, n))
    A.sum_duplicates()
    A.sort_indices()
    return PressureSystem(A, index, unk)


def build_ai_preconditioner(A, omega=1.65):
    """linalg.py:201-232, order 1, untruncated: W = K^T K with
    K = sqrt(2-omega) Dbar^-1/2 (I - L Dbar^-1), Dbar = D/omega."""
    d = A.diagonal()
    dbar_inv = omega / d
    L = sp.tril(A, k=-1, format="csr")
    inner = sp.identity(A.shape[0], format="csr") - L @ sp.diags(dbar_inv)
    K = sp.diags(np.sqrt((2.0 - omega) * dbar_inv)) @ inner
    W = (K.T @ K).tocsr()
    return ((W + W.T) * 0.5).tocsr()


def default_projection_tol(W):
    """solver.py:235-243"""
    return 1e-8 * max(float(np.mean(W.diagonal())), 1e-300)


@dataclass
class PcgReport:
    iterations: int
    converged: bool
    criterion: float


def pcg_solve(A, b, W, tol, x0=None, res_inf_target=None, max_iter=10_000):
    """linalg.py:310-368 -- identical iterate sequence and stopping rule."""
    b2 = float(b @ b)
    if b2 == 0.0:
        return np.zeros_like(b), PcgReport(0, True, 0.0)

    def done(r, crit):
        if not 0.0 <= crit < tol:
            return False
        return res_inf_target is None or float(np.max(np.abs(r))) <= res_inf_target

    x = np.zeros_like(b) if x0 is None else x0.astype(float).copy()
    r = b - A @ x if x0 is not None else b.copy()
    z = W @ r
    rz = float(r @ z)
    crit = rz / b2
    if done(r, crit):
        return x, PcgReport(0, True, crit)
    if rz < 0.0:
        return x, PcgReport(0, False, crit)
    p = z.copy()
    for it in range(1, max_iter + 1):
        Ap = A @ p
        pAp = float(p @ Ap)
        if pAp <= 0:
            return x, PcgReport(it - 1, False, crit)
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        z = W @ r
        rz_new = float(r @ z)
        crit = rz_new / b2
        if done(r, crit):
            return x, PcgReport(it, True, crit)
        if rz_new < 0.0:
            return x, PcgReport(it, False, crit)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, PcgReport(max_iter, False, crit)


class ProjectionError(RuntimeError):
    def __init__(self, report):
        super().__init__(f"pressure solve did not converge: {report}")
        self.report = report


# ---------------------------------------------------------------------------
# stage helpers

def _edge_pad(a, axis):
    pw = [(0, 0)] * 3
    pw[aax(axis)] = (1, 1)
    return np.pad(a, pw, mode="edge")


def avg_to_faces(c, axis):
    """solver.py:138-147"""
    p = _edge_pad(c, axis)
    return 0.5 * (p[_sl(axis, slice(0, -1))] + p[_sl(axis, slice(1, None))])


def face_adjacent(cells, axis):
    """solver.py:311-320"""
    p = _edge_pad(cells, axis)
    return p[_sl(axis, slice(0, -1))] | p[_sl(axis, slice(1, None))]


def component_laplacian(arr, grid):
    """solver.py:175-190 (edge-replicated, axes accumulated x, y, z)."""
    out = np.zeros_like(arr)
    for axis in range(3):
        if arr.shape[aax(axis)] == 1 or (grid.is_2d and axis == 2):
            continue
        h = grid.h(axis)
        p = _edge_pad(arr, axis)
        out += (p[_sl(axis, slice(0, -2))] - 2.0 * p[_sl(axis, slice(1, -1))]
                + p[_sl(axis, slice(2, None))]) / h ** 2
    return out


def drag_factor_cells(state, params):
    """solver.py:123-135"""
    g = np.zeros_like(state.phi)
    b = state.labels == BUILDING
    if b.any():
        ratio = (1.0 - state.phi[b]) / (state.phi[b] + params.drag_eps)
        g[b] = params.cd_building * params.drag_a * ratio ** params.drag_b
    t = state.labels == TREE
    if t.any():
        g[t] = params.cd_tree * state.lad[t]
    return g


def apply_drag(state, params, dt):
    """solver.py:150-168"""
    cdg = drag_factor_cells(state, params)
    if not cdg.any():
        return state
    speed = state.speed()
    for axis in range(3):
        if state.grid.is_2d and axis == 2:
            continue
        arr = state.comp(axis)
        arr *= np.maximum(0.0, 1.0 - dt * avg_to_faces(cdg, axis) * avg_to_faces(speed, axis))
    return state


def diffuse(state, params, dt):
    """solver.py:193-208"""
    cap = nu_stable(state.grid, dt) - params.nu
    if cap <= 0:
        warnings.warn(f"time step {dt} exceeds the molecular-diffusion stability bound",
                      stacklevel=2)
        cap = 0.0
    nu_eff = params.nu + np.clip(state.nu_t, 0.0, cap)
    for axis in range(3):
        if state.grid.is_2d and axis == 2:
            continue
        arr = state.comp(axis)
        arr += dt * avg_to_faces(nu_eff, axis) * component_laplacian(arr, state.grid)
    return state


def divergence(state):
    """solver.py:215-221"""
    g = state.grid
    u, v, w = state.u, state.v, state.w
    div = (u[:, :, 1:] - u[:, :, :-1]) / g.dx + (v[:, 1:, :] - v[:, :-1, :]) / g.dy
    if not g.is_2d:
        div = div + (w[1:] - w[:-1]) / g.dz
    return div


def max_interior_divergence(state):
    """solver.py:224-229"""
    m = interior_mask(state.labels)
    if not m.any():
        return 0.0
    return float(np.max(np.abs(divergence(state)[m])))


def project(state, psys, dt, W, tol=None, max_iter=10_000):
    """solver.py:246-304"""
    g = state.grid
    unk = psys.unknown
    div = divergence(state)
    b = -div[unk] / dt
    if tol is None:
        tol = default_projection_tol(W)
    res_target = DIV_REDUCTION_TARGET * float(np.max(np.abs(b))) if b.any() else None
    x0 = state.p[unk].copy()
    if not x0.any():
        x0 = None
    x, rep = pcg_solve(psys.A, b, W, tol, x0, res_target, max_iter)
    if not rep.converged:
        raise ProjectionError(rep)
    p = np.zeros(g.cshape)
    p[unk] = x
    state.p = p
    outlet = state.labels == OUTLET
    for axis in range(3):
        if g.is_2d and axis == 2:
            continue
        h = g.h(axis)
        lo, hi = _sl(axis, slice(0, -1)), _sl(axis, slice(1, None))
        a_unk, b_unk = unk[lo], unk[hi]
        plo, phi_ = p[lo], p[hi]
        grad = np.zeros_like(plo)
        both = a_unk & b_unk
        grad[both] = (phi_[both] - plo[both]) / h
        to_out = a_unk & outlet[hi]
        grad[to_out] = -plo[to_out] / h
        from_out = b_unk & outlet[lo]
        grad[from_out] = phi_[from_out] / h
        state.comp(axis)[_sl(axis, slice(1, -1))] -= dt * grad
    return state, rep


def apply_boundary_conditions(state, profile, params):
    """solver.py:330-400: ordered outlet copies per side, inlet scalars,
    inlet faces, then walls zero every touching face."""
    g = state.grid
    lab = state.labels
    k_in, om_in = params.inlet_k_omega()
    dir_x, dir_y = profile.direction
    inlet, wall, outlet = lab == INLET, lab == SOLID_WALL, lab == OUTLET
    sides = [(0, 0), (0, g.nx - 1), (1, 0), (1, g.ny - 1)]
    if not g.is_2d:
        sides += [(2, 0), (2, g.nz - 1)]
    for axis, pos in sides:
        cs = _sl(axis, pos)
        inner = _sl(axis, pos + 1 if pos == 0 else pos - 1)
        m2 = outlet[cs]
        if not m2.any():
            continue
        for name in ("k", "omega", "nu_t", "p"):
            a = getattr(state, name)
            a[cs][m2] = a[inner][m2]
        for caxis in range(3):
            if g.is_2d and caxis == 2:
                continue
            a = state.comp(caxis)
            if caxis == axis:
                outer = pos + 1 if pos > 0 else 0
                src = pos if pos > 0 else 1
                a[_sl(axis, outer)][m2] = a[_sl(axis, src)][m2]
            else:
                m = face_adjacent(outlet, caxis)[cs]
                a[cs][m] = a[inner][m]
    if inlet.any():
        state.k[inlet] = k_in
        state.omega[inlet] = om_in
        state.nu_t[inlet] = k_in / om_in
    uz = profile.speed_at(g.origin[2] + (np.arange(g.nz) + 0.5) * g.dz)
    if inlet.any():
        mu = face_adjacent(inlet, 0)
        state.u[mu] = (np.ones(state.u.shape) * uz[:, None, None] * dir_x)[mu]
        mv = face_adjacent(inlet, 1)
        state.v[mv] = (np.ones(state.v.shape) * uz[:, None, None] * dir_y)[mv]
        if not g.is_2d:
            state.w[face_adjacent(inlet, 2)] = 0.0
    if wall.any():
        state.u[face_adjacent(wall, 0)] = 0.0
        state.v[face_adjacent(wall, 1)] = 0.0
        if not g.is_2d:
            state.w[face_adjacent(wall, 2)] = 0.0
    return state


# ---------------------------------------------------------------------------
# advection  (advection.py:16-173, _kernels.py:25-58)

_OFF = {0: (0.0, 0.5, 0.5), 1: (0.5, 0.0, 0.5), 2: (0.5, 0.5, 0.0), 3: (0.5, 0.5, 0.5)}


def _positions(grid, comp):
    """Sample positions (cell units) of a component's array, broadcastable
    over the x-fastest array: returns (X, Y, Z)."""
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    shp = {0: (nx + 1, ny, nz), 1: (nx, ny + 1, nz), 2: (nx, ny, nz + 1), 3: (nx, ny, nz)}[comp]
    off = _OFF[comp]
    X = (np.arange(shp[0]) + off[0])[None, None, :]
    Y = (np.arange(shp[1]) + off[1])[None, :, None]
    Z = (np.arange(shp[2]) + off[2])[:, None, None]
    return X, Y, Z


def gather(arr, fx, fy, fz, minmax=False):
    """Trilinear sample of an x-fastest array at fractional coordinates
    (advection.py:49-101): indices clamped to [0, n-2], weights to [0, 1],
    size-1 axes use stride 0."""
    fx, fy, fz = np.broadcast_arrays(fx, fy, fz)
    nz, ny, nx = arr.shape
    i0 = np.clip(np.floor(fx).astype(np.int64), 0, max(nx - 2, 0))
    j0 = np.clip(np.floor(fy).astype(np.int64), 0, max(ny - 2, 0))
    k0 = np.clip(np.floor(fz).astype(np.int64), 0, max(nz - 2, 0))
    tx = np.clip(fx - i0, 0.0, 1.0)
    ty = np.clip(fy - j0, 0.0, 1.0)
    tz = np.clip(fz - k0, 0.0, 1.0)
    flat = np.ascontiguousarray(arr).ravel()
    base = k0 * (ny * nx) + j0 * nx + i0
    sx = 1 if nx > 1 else 0
    sy = nx if ny > 1 else 0
    sz = ny * nx if nz > 1 else 0

    def at(o):
        return flat.take(base + o if o else base)

    c000, c100, c010, c110 = at(0), at(sx), at(sy), at(sx + sy)
    c001, c101, c011, c111 = at(sz), at(sx + sz), at(sy + sz), at(sx + sy + sz)
    c00 = c000 * (1 - tx) + c100 * tx
    c10 = c010 * (1 - tx) + c110 * tx
    c01 = c001 * (1 - tx) + c101 * tx
    c11 = c011 * (1 - tx) + c111 * tx
    c0 = c00 * (1 - ty) + c10 * ty
    c1 = c01 * (1 - ty) + c11 * ty
    val = c0 * (1 - tz) + c1 * tz
    if not minmax:
        return val
    st = (c000, c100, c010, c110, c001, c101, c011, c111)
    return val, np.minimum.reduce(st), np.maximum.reduce(st)


def sample(arr, comp, X, Y, Z, minmax=False):
    o = _OFF[comp]
    return gather(arr, X - o[0], Y - o[1], Z - o[2], minmax)


def velocity_at(state, X, Y, Z):
    return (sample(state.u, 0, X, Y, Z), sample(state.v, 1, X, Y, Z),
            sample(state.w, 2, X, Y, Z))


def maccormack(state, arr, comp, dt):
    """advection.py:125-142"""
    g = state.grid
    X, Y, Z = _positions(g, comp)
    us, vs, ws = velocity_at(state, X, Y, Z)
    ahead, mn, mx = sample(arr, comp, X - dt * us / g.dx, Y - dt * vs / g.dy,
                           Z - dt * ws / g.dz, minmax=True)
    back = sample(ahead, comp, X + dt * us / g.dx, Y + dt * vs / g.dy, Z + dt * ws / g.dz)
    return np.clip(ahead + 0.5 * (arr - back), mn, mx)


def advect_velocity(state, dt):
    u = maccormack(state, state.u, 0, dt)
    v = maccormack(state, state.v, 1, dt)
    w = state.w.copy() if state.grid.is_2d else maccormack(state, state.w, 2, dt)
    return u, v, w


def upwind_scalar(state, f, dt):
    """advection.py:154-173 (axes applied sequentially x, y, z)."""
    g = state.grid
    vel = state.cell_velocity()
    out = f.copy()
    for axis in range(3):
        if g.n(axis) == 1:
            continue
        a = vel[axis]
        h = g.h(axis)
        fwd = np.zeros_like(f)
        bwd = np.zeros_like(f)
        lo, hi = _sl(axis, slice(0, -1)), _sl(axis, slice(1, None))
        diff = (f[hi] - f[lo]) / h
        bwd[hi] = diff
        fwd[lo] = diff
        out -= dt * (np.maximum(a, 0.0) * bwd + np.minimum(a, 0.0) * fwd)
    return out


# ---------------------------------------------------------------------------
# turbulence  (turbulence.py:36-132)

def pad_laplacian(f, grid):
    out = np.zeros_like(f)
    for axis in range(3):
        n = grid.n(axis)
        if n == 1:
            continue
        h = grid.h(axis)
        core = (f[_sl(axis, slice(0, -2))] - 2.0 * f[_sl(axis, slice(1, -1))]
                + f[_sl(axis, slice(2, None))]) / h ** 2
        out[_sl(axis, slice(1, -1))] += core
        out[_sl(axis, slice(0, 1))] += (f[_sl(axis, slice(1, 2))] - f[_sl(axis, slice(0, 1))]) / h ** 2
        out[_sl(axis, slice(n - 1, n))] += (f[_sl(axis, slice(n - 2, n - 1))]
                                            - f[_sl(axis, slice(n - 1, n))]) / h ** 2
    return out


def strain_rate_sq(state):
    g = state.grid
    u, v, w = state.u, state.v, state.w
    dudx = (u[:, :, 1:] - u[:, :, :-1]) / g.dx
    dvdy = (v[:, 1:, :] - v[:, :-1, :]) / g.dy
    dwdz = (w[1:] - w[:-1]) / g.dz
    uc, vc, wc = state.cell_velocity()

    def grad(fc, axis):
        if fc.shape[aax(axis)] == 1:
            return np.zeros_like(fc)
        return np.gradient(fc, g.h(axis), axis=aax(axis))

    dudy, dudz = grad(uc, 1), grad(uc, 2)
    dvdx, dvdz = grad(vc, 0), grad(vc, 2)
    dwdx, dwdy = grad(wc, 0), grad(wc, 1)
    s2 = dudx ** 2 + dvdy ** 2 + dwdz ** 2
    return s2 + 0.5 * ((dudy + dvdx) ** 2 + (dudz + dwdx) ** 2 + (dvdz + dwdy) ** 2)


def eddy_viscosity(k, omega, s2, c_mu, c_lim):
    om_t = np.maximum(omega, c_lim * np.sqrt(s2) / (c_mu / 2.0))
    return k / np.maximum(om_t, OMEGA_FLOOR)


def update_turbulence(state, params, dt):
    g = state.grid
    s2 = strain_rate_sq(state)
    cap = max(nu_stable(g, dt) - params.nu, 0.0)
    p_k = 2.0 * state.nu_t * s2
    dk = params.nu + np.minimum(params.sigma_star * state.nu_t, cap)
    dw = params.nu + np.minimum(params.sigma * state.nu_t, cap)
    k_new = (state.k + dt * (p_k + dk * pad_laplacian(state.k, g))) \
        / (1.0 + dt * params.c_mu * state.omega)
    w_new = (state.omega + dt * (2.0 * params.alpha * s2 + dw * pad_laplacian(state.omega, g))) \
        / (1.0 + dt * params.beta * state.omega)
    for name, arr in (("k", k_new), ("omega", w_new)):
        if not np.all(np.isfinite(arr)):
            kk, jj, ii = np.nonzero(~np.isfinite(arr))
            first = min(zip(ii.tolist(), jj.tolist(), kk.tolist()))
            raise FloatingPointError(
                f"turbulence update produced non-finite {name} at cell {first}")
    state.k = np.maximum(k_new, K_FLOOR)
    state.omega = np.maximum(w_new, OMEGA_FLOOR)
    state.nu_t = eddy_viscosity(state.k, state.omega, s2, params.c_mu, params.c_lim)
    return state


# ---------------------------------------------------------------------------
# full step (solver.py:407-461), initial state (:464-481), regions (:535-549)

@dataclass
class StepReport:
    pcg: PcgReport | None = None
    cfl: float = 0.0
    div_before: float = 0.0
    div_after: float = 0.0


def step(state, params, psys, W, profile, pcg_tol=None):
    rep = StepReport()
    dt = params.dt
    if dt == 0.0:
        return rep
    if params.turbulence:
        k_new = upwind_scalar(state, state.k, dt)
        om_new = upwind_scalar(state, state.omega, dt)
    state.u, state.v, state.w = advect_velocity(state, dt)
    if params.turbulence:
        state.k, state.omega = k_new, om_new
    diffuse(state, params, dt)
    apply_drag(state, params, dt)
    apply_boundary_conditions(state, profile, params)
    rep.div_before = max_interior_divergence(state)
    _, rep.pcg = project(state, psys, dt, W, tol=pcg_tol)
    rep.div_after = max_interior_divergence(state)
    if params.turbulence:
        update_turbulence(state, params, dt)
    apply_boundary_conditions(state, profile, params)
    smax = max(float(np.max(np.abs(state.u))), float(np.max(np.abs(state.v))),
               float(np.max(np.abs(state.w))), 1e-300)
    rep.cfl = smax * dt / min(state.grid.dx, state.grid.dy, state.grid.dz)
    state.time += dt
    state.step_count += 1
    return rep


def make_initial_state(grid, labels, phi, lad, params, profile, mode="inflow"):
    k_in, om_in = params.inlet_k_omega()
    st = State.zeros(grid, labels, phi, lad, k0=k_in, omega0=om_in)
    if not params.turbulence:
        st.nu_t[:] = 0.0
    if mode == "inflow":
        uz = profile.speed_at(grid.origin[2] + (np.arange(grid.nz) + 0.5) * grid.dz)
        st.u[:] = uz[:, None, None] * profile.direction[0]
        st.v[:] = uz[:, None, None] * profile.direction[1]
    elif mode != "rest":
        raise ValueError(f"unknown init mode {mode!r}")
    apply_boundary_conditions(st, profile, params)
    return st


def cell_centers(grid, axis):
    return grid.origin[axis] + (np.arange(grid.n(axis)) + 0.5) * grid.h(axis)


def region_average_speed(state, lo, hi):
    g = state.grid
    x, y, z = (cell_centers(g, a) for a in range(3))
    mx = (x >= lo[0]) & (x <= hi[0])
    my = (y >= lo[1]) & (y <= hi[1])
    mz = (z >= lo[2]) & (z <= hi[2])
    m = mz[:, None, None] & my[None, :, None] & mx[None, None, :] & (state.labels == AIR)
    if not m.any():
        raise ValueError("region contains no air cells")
    return float(np.mean(state.speed()[m]))


# ---------------------------------------------------------------------------
# scenario glue (schema v1, scenario.py:132-301; only what the path needs)

@dataclass
class Scene:
    grid: Grid
    faces: dict
    inlet: Inlet
    params: Params
    objects: list
    design: list = field(default_factory=list)
    objective: dict | None = None
    subdiv: int = 4
    ai_omega: float = 1.65
    pcg_tol: float | None = None
    init_mode: str = "inflow"
    paint: dict | None = None
    base_dir: str = "."


def scene_from_dict(doc, base_dir="."):
    gd = doc["grid"]
    grid = Grid(int(gd["nx"]), int(gd["ny"]), int(gd.get("nz", 1)), float(gd["dx"]),
                float(gd["dy"]), float(gd.get("dz", gd["dx"])),
                tuple(gd.get("origin", (0.0, 0.0, 0.0))))
    faces = {f: _LABEL_NAMES[v] for f, v in doc["boundaries"].items()}
    i = doc.get("inlet", {})
    inlet = Inlet(i.get("kind", "uniform"), float(i.get("speed", 1.0)),
                  float(i.get("u_star", 0.5)), float(i.get("z0", 0.5)),
                  direction=tuple(i.get("direction", (1.0, 0.0))))
    params = Params(**doc.get("solver", {}))
    num = doc.get("numerics", {})
    return Scene(grid, faces, inlet, params, list(doc.get("objects", [])),
                 list(doc.get("design", [])), doc.get("objective"),
                 int(num.get("subdiv", 4)), float(num.get("ai_omega", 1.65)),
                 num.get("pcg_tol"), num.get("init", "inflow"), doc.get("paint"), base_dir)


class Compiled:
    """CompiledScenario.compile (scenario.py:375-381) + voxelize_design."""

    def __init__(self, scene):
        self.scene = scene
        self.boundary = classify_boundary(scene.grid, scene.faces)
        self.psys = build_pressure_matrix(scene.grid, self.boundary)
        self.W = build_ai_preconditioner(self.psys.A, scene.ai_omega)

    def voxelize_design(self, theta=None):
        from oracle import voxel_oracle
        return voxel_oracle.voxelize_scene(self.scene, self.boundary, theta)

    def make_state(self, theta=None):
        labels, phi, lad = self.voxelize_design(theta)
        sc = self.scene
        return make_initial_state(sc.grid, labels, phi, lad, sc.params, sc.inlet, sc.init_mode)

    def step_state(self, state):
        sc = self.scene
        return step(state, sc.params, self.psys, self.W, sc.inlet, sc.pcg_tol)


def evaluate_objective(compiled, theta, profile=None):
    """optimize.py:77-104: loss and trailing-window region speeds."""
    sc = compiled.scene
    ob = sc.objective
    settle, frac = int(ob.get("settle_steps", 300)), float(ob.get("avg_fraction", 0.25))
    target = float(ob.get("target_speed", 0.55))
    profile = profile or sc.inlet
    labels, phi, lad = compiled.voxelize_design(theta)
    st = make_initial_state(sc.grid, labels, phi, lad, sc.params, profile, sc.init_mode)
    window = max(1, int(round(settle * frac)))
    regs = ob["regions"]
    sums = np.zeros(len(regs))
    count = 0
    for n in range(settle):
        step(st, sc.params, compiled.psys, compiled.W, profile, sc.pcg_tol)
        if n >= settle - window:
            for ri, r in enumerate(regs):
                sums[ri] += region_average_speed(st, r["lo"], r["hi"])
            count += 1
    speeds = sums / count
    loss = float(np.sum((speeds - target) ** 2))
    if not math.isfinite(loss):
        raise FloatingPointError(f"objective evaluation produced {loss}")
    return loss, speeds


def to_ref_layout(a):
    """x-fastest (nz, ny, nx) -> reference C-order (nx, ny, nz)."""
    return np.ascontiguousarray(np.asarray(a).transpose(2, 1, 0))


def from_ref_layout(a):
    return np.ascontiguousarray(np.asarray(a).transpose(2, 1, 0))


def field_digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def trace_streamlines(state, seeds, step_len, max_steps=2000, min_speed=1e-6):
    """solver.py:488-532: RK2 midpoint streamlines of the staggered velocity."""
    g = state.grid
    origin = np.asarray(g.origin, float)
    spacing = np.array([g.dx, g.dy, g.dz])
    lo = origin
    hi = origin + spacing * np.array([g.nx, g.ny, g.nz])

    def vel(p):
        c = (p - origin) / spacing
        us, vs, ws = velocity_at(state, np.array([c[0]]), np.array([c[1]]), np.array([c[2]]))
        return np.array([us[0], vs[0], ws[0]])

    out = []
    for seed in np.atleast_2d(np.asarray(seeds, float)):
        if np.any(seed < lo) or np.any(seed > hi):
            out.append(np.empty((0, 3)))
            continue
        pts, p = [seed.copy()], seed.copy()
        for _ in range(max_steps):
            v1 = vel(p)
            s1 = np.linalg.norm(v1)
            if s1 < min_speed:
                break
            mid = p + 0.5 * step_len * v1 / s1
            if np.any(mid < lo) or np.any(mid > hi):
                break
            v2 = vel(mid)
            s2 = np.linalg.norm(v2)
            if s2 < min_speed:
                break
            p = p + step_len * v2 / s2
            if np.any(p < lo) or np.any(p > hi):
                break
            pts.append(p.copy())
        out.append(np.array(pts))
    return out


def gradient_descent(compiled, theta0, lo, hi, lam=1.0, eps=0.1, max_iter=30, rel_tol=1e-3):
    """optimize.py:112-192: forward differences (+eps, or -eps past the upper
    bound), theta <- clamp(theta - lam * grad), stop after 3 consecutive
    relative loss changes below rel_tol.  Returns (thetas, losses)."""
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    theta = np.clip(np.asarray(theta0, float), lo, hi)
    base = evaluate_objective(compiled, theta)[0]
    history, thetas = [base], [theta.copy()]
    stable = 0
    for _ in range(max_iter):
        grad = np.zeros_like(theta)
        for i in range(len(theta)):
            h = eps if theta[i] + eps <= hi[i] else -eps
            t = theta.copy()
            t[i] += h
            grad[i] = (evaluate_objective(compiled, t)[0] - base) / h
        theta = np.clip(theta - lam * grad, lo, hi)
        base = evaluate_objective(compiled, theta)[0]
        if not math.isfinite(base):
            break
        rel = abs(history[-1] - base) / max(history[-1], 1e-12)
        history.append(base)
        thetas.append(theta.copy())
        if rel < rel_tol:
            stable += 1
            if stable >= 3:
                break
        else:
            stable = 0
    return thetas, history
