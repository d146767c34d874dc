"""Native context management: one ``cw_ctx`` per (operator, device, precision).

A context owns the device workspace of one step in flight (advection and PCG
temporaries, the report ring, the grid-barrier words).  ``ContextPool`` hands
out contexts so concurrent design evaluations (the reference's thread pool,
optimize.py:137-142) never share a workspace.
"""
from __future__ import annotations

import ctypes as C
import threading

import torch

from . import _native as N

_DT = {torch.float32: 4, torch.float64: 8}


class Context:
    def __init__(self, grid, dtype=torch.float32, device=None):
        self.grid = grid
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if self.device.type != "cuda":
            raise RuntimeError("citywind_b200 contexts live on CUDA devices only")
        self._lib = N.lib()
        g = N.cw_grid(grid.nx, grid.ny, grid.nz, float(grid.dx), float(grid.dy), float(grid.dz),
                      N.dbl3(grid.origin))
        h = C.c_void_p()
        N.check(self._lib.cw_ctx_create(C.byref(g), _DT[dtype], self.device.index or 0, C.byref(h)))
        self.h = h
        self.n_unknown = None
        self.tol_default = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self._lib.cw_ctx_destroy(h)
            except Exception:
                pass
            self.h = None

    @property
    def stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def set_operator(self, labels_dev: torch.Tensor, omega: float, precond: int = 2):
        n = C.c_longlong()
        tol = C.c_double()
        N.check(self._lib.cw_set_operator(self.h, N.ptr(labels_dev), float(omega), C.byref(n),
                                          C.byref(tol), self.stream))
        tk = C.c_double()
        N.check(self._lib.cw_set_preconditioner(self.h, int(precond), C.byref(tk)))
        self.n_unknown = int(n.value)
        self.tol_default = float(tk.value)

    # -- field marshalling -------------------------------------------------
    @staticmethod
    def fields(state, g=None, has_drag=False):
        f = state.fields
        return N.cw_fields(N.ptr(f["u"]), N.ptr(f["v"]), N.ptr(f["w"]), N.ptr(f["p"]), N.ptr(f["k"]),
                           N.ptr(f["omega"]), N.ptr(f["nu_t"]), N.ptr(state.labels_dev),
                           N.ptr(g), int(bool(has_drag)), N.labels_version(state.labels_dev))

    def read_reports(self, n):
        out = (N.cw_report * max(n, 1))()
        got = C.c_int()
        rc = self._lib.cw_read_reports(self.h, out, n, C.byref(got), self.stream)
        return rc, [out[i] for i in range(got.value)]


class ContextPool:
    """Free-list of contexts for one operator (labels + omega)."""

    def __init__(self):
        self._free: dict = {}
        self._lock = threading.Lock()

    def acquire(self, grid, labels_dev, omega, precond, dtype, device):
        key = (str(device), dtype, float(omega), int(precond))
        with self._lock:
            lst = self._free.setdefault(key, [])
            if lst:
                return lst.pop()
        ctx = Context(grid, dtype, device)
        ctx.set_operator(labels_dev, omega, precond)
        ctx.key = key
        return ctx

    def release(self, ctx):
        with self._lock:
            self._free.setdefault(ctx.key, []).append(ctx)
