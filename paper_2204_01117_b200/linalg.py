"""Pressure operator and preconditioner objects (reference ``citywind.linalg``).

The reference assembles A (7-point Laplacian) and W = K^T K (untruncated AI1)
as scipy CSR matrices (linalg.py:57-126, 201-232).  Here both stay
matrix-free on the device: ``PressureSystem`` carries the labels the operator
was built from and lends out native contexts whose per-cell code field and
64-entry coefficient table encode A and W exactly (see csrc/cw_pcg.cuh).
``pcg_solve`` is not a separate host function: the whole warm-started PCG
runs inside one persistent device kernel per projection.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import SingularSystemError
from .grid import CellLabel, GridSpec, interior_mask, to_device_layout
from .runtime import ContextPool

__all__ = ["PcgReport", "PressureSystem", "build_pressure_matrix", "Preconditioner",
           "IdentityPreconditioner", "MatrixPreconditioner", "build_ai_preconditioner",
           "build_jacobi", "SingularSystemError"]


@dataclass
class PcgReport:
    iterations: int
    converged: bool
    criterion: float


class PressureSystem:
    """The pressure operator of one grid + label set (linalg.py:34-50)."""

    def __init__(self, grid: GridSpec, labels: np.ndarray):
        self.grid = grid
        self.labels = np.asarray(labels, np.int8).copy()
        self._unknown = interior_mask(self.labels)
        self.n = int(self._unknown.sum())
        self._index = None
        self._labels_dev = {}
        self.pool = ContextPool()

    @property
    def index(self) -> np.ndarray:
        """Grid-shaped unknown number (x-fastest), -1 elsewhere (linalg.py:71-72)."""
        if self._index is None:
            idx = np.full(self.grid.shape, -1, np.int64)
            flat_f = np.arange(self.grid.n_cells).reshape(self.grid.shape, order="F")
            order = np.argsort(flat_f[self._unknown], kind="stable")
            ranks = np.empty_like(order)
            ranks[order] = np.arange(len(order))
            idx[self._unknown] = ranks
            self._index = idx
        return self._index

    def labels_on(self, device) -> torch.Tensor:
        key = str(device)
        if key not in self._labels_dev:
            self._labels_dev[key] = torch.from_numpy(to_device_layout(self.labels)).to(device)
        return self._labels_dev[key]

    @property
    def A(self):
        raise AttributeError("the device pressure operator is matrix-free (no CSR); "
                             "see csrc/cw_pcg.cuh for its stencil")


def build_pressure_matrix(grid: GridSpec, labels: np.ndarray,
                          pin_if_singular: bool = False) -> PressureSystem:
    """linalg.py:57-126.  Validates like the reference (no flow cells ->
    ValueError; no unknown next to an outlet -> SingularSystemError)."""
    labels = np.asarray(labels, np.int8)
    unk = interior_mask(labels)
    if not unk.any():
        raise ValueError("no flow cells to solve for")
    outlet = labels == int(CellLabel.OUTLET)
    touches = False
    for axis in range(3):
        if grid.is_2d and axis == 2:
            continue
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[axis] = slice(0, -1)
        hi[axis] = slice(1, None)
        lo, hi = tuple(lo), tuple(hi)
        if np.any(unk[lo] & outlet[hi]) or np.any(unk[hi] & outlet[lo]):
            touches = True
            break
    if not touches:
        if pin_if_singular:
            raise NotImplementedError("pin_if_singular is only used by the 2D appendix benchmarks")
        raise SingularSystemError("no outlet cells: pressure defined only up to a constant")
    return PressureSystem(grid, labels)


class Preconditioner:
    name = "identity"
    kind = 0


class IdentityPreconditioner(Preconditioner):
    pass


class MatrixPreconditioner(Preconditioner):
    """Explicit sparse M^-1 in the reference; here a kind + omega tag that
    selects the device stencil (linalg.py:160-175)."""

    def __init__(self, kind: int, omega: float = 1.65, name: str = "matrix"):
        self.kind = kind
        self.omega = float(omega)
        self.name = name


def build_jacobi(psys) -> MatrixPreconditioner:
    return MatrixPreconditioner(1, name="jacobi")


def build_ai_preconditioner(psys, omega: float = 1.65, order: int = 1,
                            truncate: bool = True) -> MatrixPreconditioner:
    """linalg.py:201-232.  The scenario pipeline uses order 1 untruncated
    (scenario.py:111-113,377-379); that is the variant the device applies."""
    if not 0.0 < omega < 2.0:
        raise ValueError(f"omega must lie in (0, 2), got {omega}")
    if order not in (1, 2):
        raise ValueError("order must be 1 or 2")
    if order != 1 or truncate:
        raise NotImplementedError("the device preconditioner is the untruncated AI1 "
                                  "(ai_order=1, ai_truncate=False) used by the scenario pipeline")
    return MatrixPreconditioner(2, omega=omega, name="ai1")
