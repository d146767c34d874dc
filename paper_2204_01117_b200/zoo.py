"""The preconditioner benchmark of the paper's appendix,
host side.

The reference compares its approximate-inverse preconditioner with CG,
Jacobi, SSOR, IC(0) and modified IC on a 2-D Poisson benchmark system:
condition numbers by Lanczos and PCG iteration counts
(reference ``citywind.linalg`` :178-303, 375-462 and ``citywind.validate``
:243-313).  SSOR / IC / MIC need two sparse triangular solves per
application -- serial by construction -- and the system is small
(128 x 193 x 2), so, as the survey prescribes, this module runs on the host
with scipy.  It is NOT on the step path: the device step uses the matrix-free
AI1 stencil inside ``k_pcg`` (``linalg.build_ai_preconditioner``).

Names and arguments follow the reference: ``benchmark_matrix``,
``build_reference_preconditioner``, ``estimate_condition_number``,
``pcg_solve``, ``bench_preconditioners``, ``omega_sweep``; the explicit
Jacobi / AI matrices the benchmark needs are ``jacobi_matrix`` and
``ai_matrix`` (the device-side ``linalg`` builders return stencil tags).
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from scipy.linalg import eigh_tridiagonal

from .grid import CellLabel, GridSpec
from .linalg import PcgReport, build_pressure_matrix

__all__ = ["assemble_pressure_matrix", "benchmark_matrix", "ExplicitPreconditioner", "TriangularPreconditioner",
           "jacobi_matrix", "ai_matrix", "build_reference_preconditioner", "estimate_condition_number",
           "pcg_solve", "BenchRow", "bench_preconditioners", "omega_sweep", "MIC_RELAXATION",
           "SSOR_BENCH_OMEGA"]

MIC_RELAXATION = 0.93     # share of the dropped fill moved onto the diagonal (linalg.py:235-239)
SSOR_BENCH_OMEGA = 1.45   # SSOR relaxation of the published benchmark (validate.py:28-29)


def assemble_pressure_matrix(psys) -> sp.csr_matrix:
    """The pressure operator of a ``linalg.PressureSystem`` as an explicit
    CSR matrix (linalg.py:57-126): per unknown, -1/h^2 to every unknown
    neighbour, +1/h^2 on the diagonal for every unknown or outlet neighbour;
    inlet / wall neighbours are Neumann ghosts.  Unknowns numbered x-fastest
    (``psys.index``)."""
    g, lab, idx = psys.grid, psys.labels, psys.index
    n = psys.n
    h = (g.dx, g.dy, g.dz)
    diag = np.zeros(n)
    rows, cols, vals = [], [], []
    for axis in range(2 if g.is_2d else 3):
        w = 1.0 / h[axis] ** 2
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[axis], hi[axis] = slice(0, -1), slice(1, None)
        ia, ib = idx[tuple(lo)], idx[tuple(hi)]          # cell and its +axis neighbour
        la, lb = lab[tuple(lo)], lab[tuple(hi)]
        both = (ia >= 0) & (ib >= 0)
        for a, b in ((ia, ib), (ib, ia)):                # the coupling both ways
            rows.append(a[both])
            cols.append(b[both])
            vals.append(np.full(int(both.sum()), -w))
        # diagonal: unknown or outlet neighbour on either side
        out = int(CellLabel.OUTLET)
        cnt = np.zeros(n)
        np.add.at(cnt, ia[(ia >= 0) & ((ib >= 0) | (lb == out))], 1.0)
        np.add.at(cnt, ib[(ib >= 0) & ((ia >= 0) | (la == out))], 1.0)
        diag += cnt * w
    r = np.concatenate(rows + [np.arange(n)])
    c = np.concatenate(cols + [np.arange(n)])
    v = np.concatenate(vals + [diag])
    A = sp.csr_matrix((v, (r, c)), shape=(n, n))
    A.sum_duplicates()
    A.sort_indices()
    return A


def benchmark_matrix(size: str = "small") -> sp.csr_matrix:
    """The benchmark Poisson system of validate.py:251-268: an nx x (ny+1) x 2
    grid of unknowns with a ghost outlet row on top and Neumann elsewhere."""
    dims = {"small": (128, 192, 8e-3), "large": (512, 768, 2e-3)}
    if size not in dims:
        raise ValueError(f"unknown benchmark size {size!r}")
    nx, ny, h = dims[size]
    grid = GridSpec(nx, ny + 1, 2, h, h, h)
    labels = np.full(grid.shape, int(CellLabel.AIR), np.int8)
    labels[:, -1, :] = int(CellLabel.OUTLET)
    return assemble_pressure_matrix(build_pressure_matrix(grid, labels))


# ---------------------------------------------------------------------------
# preconditioners with explicit matrices

class ExplicitPreconditioner:
    """M^-1 given as a sparse matrix W (Jacobi, AI): apply = W r."""

    def __init__(self, W, name: str):
        self.W = sp.csr_matrix(W)
        self.name = name
        self._fact = None

    def apply(self, r):
        return self.W @ r

    def apply_m(self, x):                      # M x = W^-1 x (Lanczos inner product)
        if self._fact is None:
            self._fact = spla.splu(self.W.tocsc())
        return self._fact.solve(x)


class TriangularPreconditioner:
    """M = G G^T with lower-triangular G: apply = two triangular solves."""

    def __init__(self, G, name: str):
        self.G = sp.csr_matrix(G)
        self.name = name
        self._fact = spla.splu(self.G.tocsc(), permc_spec="NATURAL")

    def apply(self, r):
        return self._fact.solve(self._fact.solve(r), trans="T")

    def apply_m(self, x):
        return self.G @ (self.G.T @ x)


class _Identity:
    name = "cg"

    def apply(self, r):
        return r

    def apply_m(self, x):
        return x


def jacobi_matrix(A) -> ExplicitPreconditioner:
    d = A.diagonal()
    if np.any(d == 0):
        raise ValueError("zero diagonal entry")
    return ExplicitPreconditioner(sp.diags(1.0 / d), "jacobi")


def ai_matrix(A, omega: float = 1.65, order: int = 1, truncate: bool = True) -> ExplicitPreconditioner:
    """Explicit W = K^T K of the approximate inverse (linalg.py:201-232):
    K = sqrt((2 - w) w / d) (I - L w/d [+ (L w/d)^2])."""
    if not 0.0 < omega < 2.0:
        raise ValueError(f"omega must lie in (0, 2), got {omega}")
    if order not in (1, 2):
        raise ValueError("order must be 1 or 2")
    A = sp.csr_matrix(A)
    d = A.diagonal()
    if np.any(d <= 0):
        raise ValueError("AI preconditioner requires a positive diagonal")
    s = omega / d
    N = sp.tril(A, k=-1, format="csr") @ sp.diags(s)
    T = sp.identity(A.shape[0], format="csr") - N
    if order == 2:
        T = T + N @ N
    K = sp.diags(np.sqrt((2.0 - omega) * s)) @ T
    W = (K.T @ K).tocsr()
    if truncate:
        mask = A.copy()
        mask.data[:] = 1.0
        W = W.multiply(mask).tocsr()
    return ExplicitPreconditioner(((W + W.T) * 0.5).tocsr(), f"ai{order}")


def _incomplete_cholesky(A, tau: float) -> sp.csr_matrix:
    """G of an incomplete LDL^T on A's lower pattern (linalg.py:241-281),
    left-looking over columns; fill outside the pattern goes onto the two
    diagonals it would couple, scaled by tau (0: IC(0), 1: MIC)."""
    L = sp.tril(A, k=-1, format="csc")
    n = A.shape[0]
    d = A.diagonal().astype(float).copy()
    col = []
    for k in range(n):
        a, b = L.indptr[k], L.indptr[k + 1]
        col.append(dict(zip(L.indices[a:b].tolist(), L.data[a:b].tolist())))
    for k in range(n):
        piv = d[k]
        if piv <= 0:
            raise ValueError(f"incomplete Cholesky breakdown at row {k}: pivot {piv:.3e}")
        below = sorted(col[k].items())
        for m, (r, lr) in enumerate(below):
            d[r] -= lr * lr / piv
            target = col[r]
            for s, ls in below[m + 1:]:
                f = lr * ls / piv
                if s in target:
                    target[s] -= f
                elif tau:
                    d[r] -= tau * f
                    d[s] -= tau * f
    sq = np.sqrt(d)
    rr, cc, vv = [np.arange(n)], [np.arange(n)], [sq]
    for k in range(n):
        if col[k]:
            rows = np.fromiter(col[k].keys(), np.int64, len(col[k]))
            rr.append(rows)
            cc.append(np.full(len(rows), k))
            vv.append(np.fromiter(col[k].values(), float, len(col[k])) / sq[k])
    return sp.csr_matrix((np.concatenate(vv), (np.concatenate(rr), np.concatenate(cc))), shape=A.shape)


def build_reference_preconditioner(A, kind: str, omega: float = 1.0, mic_tau: float = MIC_RELAXATION):
    """SSOR / IC / MIC (linalg.py:284-303), benchmark scale only (n <= 1e5)."""
    kind = kind.lower()
    if A.shape[0] > 100_000:
        raise ValueError("reference preconditioners are benchmark-only (n <= 1e5)")
    A = sp.csr_matrix(A)
    if kind == "ssor":
        d = A.diagonal()
        # M = (D/w + L) ((2 - w) D/w)^-1 (D/w + L)^T = G G^T
        G = (sp.diags(d / omega) + sp.tril(A, k=-1)) @ sp.diags(np.sqrt(omega / ((2.0 - omega) * d)))
        return TriangularPreconditioner(G, "ssor")
    if kind in ("ic", "mic"):
        return TriangularPreconditioner(_incomplete_cholesky(A, 0.0 if kind == "ic" else mic_tau), kind)
    raise ValueError(f"unknown reference preconditioner kind {kind!r}")


# ---------------------------------------------------------------------------
# condition numbers and PCG

def _lanczos_top(op, inner, n: int, seed: int, max_iter: int, rtol: float = 1e-9):
    """Largest eigenvalue of `op`, self-adjoint in <x, y> = x . inner(y):
    Lanczos with full re-orthogonalisation (linalg.py:374-421).  Returns
    (value, converged)."""
    v = np.random.default_rng(seed).standard_normal(n)
    mv = inner(v)
    nrm = float(np.sqrt(v @ mv))
    Q, MQ = [v / nrm], [mv / nrm]
    alpha, beta = [], []
    last, same = None, 0
    for j in range(max_iter):
        w = op(Q[-1])
        a = float(w @ MQ[-1])
        alpha.append(a)
        w = w - a * Q[-1] - (beta[-1] * Q[-2] if j else 0.0)
        for q, mq in zip(Q, MQ):
            w = w - float(w @ mq) * q
        mw = inner(w)
        b = float(np.sqrt(max(float(w @ mw), 0.0)))
        ev = eigh_tridiagonal(np.array(alpha), np.array(beta), eigvals_only=True) if beta else np.array(alpha)
        top = float(ev[-1])
        if last is not None and abs(top - last) <= rtol * max(abs(top), 1e-300):
            same += 1
            if same >= 3:
                return top, True
        else:
            same = 0
        last = top
        if b <= 1e-14 * max(abs(a), 1.0) or j == max_iter - 1:
            return top, j < max_iter - 1
        beta.append(b)
        Q.append(w / b)
        MQ.append(mw / b)
    return (last if last is not None else 0.0), False


def estimate_condition_number(A, preconditioner=None, norm: str = "eig", max_iter: int = 200) -> float:
    """kappa(M^-1 A) (linalg.py:424-462): "eig" -- extreme eigenvalues of the
    M-self-adjoint operator, the smallest from Lanczos on the inverse;
    "2" -- sigma_max / sigma_min of the product via the normal operators."""
    M = preconditioner or _Identity()
    A = sp.csr_matrix(A)
    n = A.shape[0]
    lu = spla.splu(A.tocsc())
    if norm == "eig":
        hi, ok1 = _lanczos_top(lambda x: M.apply(A @ x), M.apply_m, n, 1, max_iter)
        inv_lo, ok2 = _lanczos_top(lambda x: lu.solve(M.apply_m(x)), M.apply_m, n, 2, max_iter)
    elif norm == "2":
        plain = lambda x: x  # noqa: E731
        hi, ok1 = _lanczos_top(lambda x: A @ M.apply(M.apply(A @ x)), plain, n, 1, max_iter)
        inv_lo, ok2 = _lanczos_top(lambda x: lu.solve(M.apply_m(M.apply_m(lu.solve(x)))), plain, n, 2, max_iter)
        hi, inv_lo = np.sqrt(hi), np.sqrt(inv_lo)
    else:
        raise ValueError(f"unknown norm {norm!r}")
    if not (ok1 and ok2):
        import warnings
        warnings.warn("condition-number Lanczos hit the iteration budget; estimate may be outside the 5% target",
                      stacklevel=2)
    return float(max(hi * inv_lo, 1.0))


def pcg_solve(A, b, preconditioner=None, tol: float = 1e-5, max_iter: int = 10_000, x0=None,
              res_inf_target: float | None = None):
    """Host PCG with the reference's stopping rule (linalg.py:310-368):
    (M^-1 r).r / |b|^2 < tol (and max|r| <= res_inf_target when given);
    a negative criterion or non-positive curvature ends it unconverged.
    The device projection runs the same rule inside ``k_pcg``."""
    M = preconditioner or _Identity()
    b = np.asarray(b, float)
    if not np.all(np.isfinite(b)):
        raise ValueError("right-hand side contains non-finite entries")
    bb = float(b @ b)
    if bb == 0.0:
        return np.zeros_like(b), PcgReport(0, True, 0.0)
    A = sp.csr_matrix(A)
    ok = lambda r, c: 0.0 <= c < tol and (res_inf_target is None or float(np.abs(r).max()) <= res_inf_target)  # noqa: E731
    x = np.zeros_like(b) if x0 is None else np.array(x0, float)
    r = b.copy() if x0 is None else b - A @ x
    z = M.apply(r)
    rz = float(r @ z)
    crit = rz / bb
    if ok(r, crit):
        return x, PcgReport(0, True, crit)
    if rz < 0.0:
        return x, PcgReport(0, False, crit)
    p = z.copy()
    for it in range(1, max_iter + 1):
        q = A @ p
        pq = float(p @ q)
        if pq <= 0:
            return x, PcgReport(it - 1, False, crit)
        a = rz / pq
        x += a * p
        r -= a * q
        z = M.apply(r)
        rz1 = float(r @ z)
        crit = rz1 / bb
        if ok(r, crit):
            return x, PcgReport(it, True, crit)
        if rz1 < 0.0:
            return x, PcgReport(it, False, crit)
        p = z + (rz1 / rz) * p
        rz = rz1
    return x, PcgReport(max_iter, False, crit)


# ---------------------------------------------------------------------------
# the benchmark (validate.py:243-313)

@dataclass
class BenchRow:
    preconditioner: str
    omega: float
    kappa: float
    iterations: int
    wall_ms: float


def bench_preconditioners(size: str = "small", omega: float = 1.65, tol: float = 1e-5,
                          norm: str = "2") -> list:
    """kappa and PCG iterations of every preconditioner on the benchmark
    system, right-hand side N(0, 1) with seed 0 (validate.py:271-300)."""
    A = benchmark_matrix(size)
    b = np.random.default_rng(0).standard_normal(A.shape[0])
    zoo = [("cg", None, 0.0), ("jacobi", jacobi_matrix(A), 0.0),
           ("ai1", ai_matrix(A, omega, 1, truncate=False), omega),
           ("ai2", ai_matrix(A, omega, 2, truncate=False), omega)]
    if size == "small":
        zoo += [("ssor", build_reference_preconditioner(A, "ssor", omega=SSOR_BENCH_OMEGA), SSOR_BENCH_OMEGA),
                ("ic", build_reference_preconditioner(A, "ic"), 0.0),
                ("mic", build_reference_preconditioner(A, "mic"), 0.0)]
    out = []
    for name, pre, om in zoo:
        kappa = estimate_condition_number(A, pre, norm=norm, max_iter=400)
        t0 = time.perf_counter()
        _, rep = pcg_solve(A, b, pre, tol=tol, max_iter=20_000)
        out.append(BenchRow(name, om, kappa, rep.iterations, (time.perf_counter() - t0) * 1e3))
    return out


def omega_sweep(size: str = "small", omegas=None, order: int = 1, norm: str = "2") -> list:
    """kappa(omega) of the approximate inverse (validate.py:303-313)."""
    omegas = [round(1.0 + 0.1 * i, 2) for i in range(10)] if omegas is None else omegas
    A = benchmark_matrix(size)
    return [(om, estimate_condition_number(A, ai_matrix(A, om, order, truncate=False), norm=norm)) for om in omegas]
