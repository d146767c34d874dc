"""Drop-in backend for the reference's ``citywind.solver.step`` on
reference-layout states.

A reference caller holds a ``citywind.grid.FlowState`` (grid.py:492-571):
float64 numpy arrays in C order with x slowest -- u (nx+1, ny, nz),
v (nx, ny+1, nz), w (nx, ny, nz+1), p / k / omega / nu_t (nx, ny, nz) --
plus int8 labels and a PorosityField.  ``RefStepper.step`` takes exactly the
reference's ``step(state, params, psys, preconditioner, profile, advector,
pcg_tol)`` arguments (solver.py:407-410), duck-typed so the reference's own
objects work unchanged, and per call:

1. uploads the seven float64 arrays (pinned staging; arrays this binding
   returned last step are already pinned), converting each to the device's
   x-fastest precision on the device (``cw_ref_layout``, a tiled transpose),
   in the order the step first uses them: the step starts once u, v, w are
   up, waits for nu_t before the diffusion and for p before the first
   boundary pass (``cw_step_defer``), and k / omega arrive while the
   projection runs (``cw_step_defer_kw``: their upwind step and boundary
   writes move behind it);
2. runs one device step (``cw_step``);
3. converts the seven fields back to float64 C order on the device and
   downloads them into pinned arrays, which it assigns to the state's
   attributes -- the reference's step reassigns them too (solver.py:423-425);
4. advances ``state.time`` / ``state.step_count`` and returns a StepReport
   with the reference's fields.

The pressure operator and the AI1 preconditioner are rebuilt on the device
from the state's labels (the reference builds them from the same labels,
scenario.py:375-381); ``psys`` / ``preconditioner`` only select the kind:
a reference ``MatrixPreconditioner`` named "ai1" (untruncated, as the
scenario pipeline builds it), "jacobi", or None / identity.  The AI weight
omega is not stored by the reference's preconditioner (linalg.py:160-167),
so it is a constructor argument (the scenario's ``numerics.ai_omega``).
Labels and porosity are re-uploaded when the state holds different array
objects than at the previous call (in-place edits of the same label /
porosity arrays between steps are not detected).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .grid import FlowState, GridSpec, PorosityField, to_device_layout
from .linalg import MatrixPreconditioner as _DevPre
from .linalg import build_pressure_matrix
from .solver import InletProfile, SolverParams, StepReport, step as _dev_step

# upload order, the order of first use in the step: u, v, w (advection),
# nu_t (diffusion), p (first boundary pass, projection), then k and omega,
# whose first readers run after the projection (cw_step_defer_kw)
ORDER = ("u", "v", "w", "nu_t", "p", "k", "omega")
LATE = ("nu_t", "p", "k", "omega")
KIND = {"u": 0, "v": 1, "w": 2, "p": 3, "k": 3, "omega": 3, "nu_t": 3}
_PARAM_FIELDS = tuple(SolverParams.__dataclass_fields__)


def _shape(grid, name):
    nx, ny, nz = int(grid.nx), int(grid.ny), int(grid.nz)
    return {"u": (nx + 1, ny, nz), "v": (nx, ny + 1, nz), "w": (nx, ny, nz + 1)}.get(name, (nx, ny, nz))


def _params(params) -> SolverParams:
    if isinstance(params, SolverParams):
        return params
    return SolverParams(**{f: getattr(params, f) for f in _PARAM_FIELDS if hasattr(params, f)})


def _profile(profile) -> InletProfile:
    if isinstance(profile, InletProfile):
        return profile
    return InletProfile(kind=profile.kind, speed=profile.speed, u_star=profile.u_star, z0=profile.z0,
                        kappa=profile.kappa, direction=tuple(profile.direction))


def _pre_kind(preconditioner, psys, ai_omega):
    """Device preconditioner for the reference's object (linalg.py:150-232)."""
    if preconditioner is None:
        return _DevPre(0, ai_omega, "identity")
    if isinstance(preconditioner, _DevPre):
        return preconditioner
    name = getattr(preconditioner, "name", None)
    if name == "jacobi":
        return _DevPre(1, ai_omega, "jacobi")
    if name == "ai1":
        W, A = getattr(preconditioner, "W", None), getattr(psys, "A", None)
        if W is not None and A is not None and W.nnz == A.nnz:
            raise NotImplementedError("truncated AI1 (W on A's sparsity pattern) is not on the device path; "
                                      "the scenario pipeline builds it untruncated (scenario.py:377-379)")
        return _DevPre(2, ai_omega, "ai1")
    if type(preconditioner).__name__ == "IdentityPreconditioner":
        return _DevPre(0, ai_omega, "identity")
    raise NotImplementedError(f"preconditioner {name or type(preconditioner).__name__!r} is not on the device path")


class _Slot:
    """Device state, operator and staging buffers of one grid."""

    def __init__(self, grid: GridSpec, dtype, device):
        self.grid = grid
        self.dev = FlowState.zeros(grid, dtype=dtype, device=device)
        self.d64 = {n: torch.empty(int(np.prod(_shape(grid, n))), dtype=torch.float64, device=device)
                    for n in ORDER}
        self.pin_in = {n: torch.empty(_shape(grid, n), dtype=torch.float64, pin_memory=True) for n in ORDER}
        # two sets of returned arrays, alternated per step (a caller's array
        # from two steps back is reused)
        self.pin_out = [{n: torch.empty(_shape(grid, n), dtype=torch.float64, pin_memory=True) for n in ORDER}
                        for _ in range(2)]
        self.np_out = [{n: t.numpy() for n, t in s.items()} for s in self.pin_out]
        self.ours = {}            # field -> id of the array we returned last
        self.out_set = 0
        self.lab_obj = None
        self.lab_host = None
        self.psys = None
        self.por_obj = None
        self.up = torch.cuda.Stream(device)
        self.down = torch.cuda.Stream(device)


class RefStepper:
    """``step(state, params, psys, preconditioner, profile, advector, pcg_tol)``
    on a reference-layout float64 state, computed on the B200."""

    def __init__(self, dtype=torch.float32, device=None, ai_omega: float = 1.65):
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ai_omega = float(ai_omega)
        self._slots = {}
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    # -- state plumbing ------------------------------------------------------
    def _slot(self, g) -> _Slot:
        key = (int(g.nx), int(g.ny), int(g.nz), float(g.dx), float(g.dy), float(g.dz),
               tuple(float(o) for o in getattr(g, "origin", (0.0, 0.0, 0.0))))
        s = self._slots.get(key)
        if s is None:
            grid = GridSpec(key[0], key[1], key[2], key[3], key[4], key[5], key[6])
            s = self._slots[key] = _Slot(grid, self.dtype, self.device)
        return s

    def _sync_static(self, s: _Slot, state):
        lab = state.labels
        if lab is not s.lab_obj:
            lab = np.asarray(lab, dtype=np.int8)
            if lab.shape != _shape(s.grid, "p"):
                raise ValueError(f"labels has shape {lab.shape}, expected {_shape(s.grid, 'p')}")
            if s.lab_host is None or not np.array_equal(lab, s.lab_host):
                s.dev.labels_dev.copy_(torch.from_numpy(to_device_layout(lab)))
                s.dev._drag_key = None
                s.psys = build_pressure_matrix(s.grid, lab)
                s.lab_host = lab.copy()
            s.lab_obj = state.labels
        por = state.porosity
        key = (id(por), id(por.phi), id(por.lad))
        if key != s.por_obj:
            s.dev.porosity = PorosityField(np.asarray(por.phi, np.float64), np.asarray(por.lad, np.float64))
            s.por_obj = key

    def prepare(self, state, preconditioner=None, psys=None):
        """One-time setup for a state's grid, outside any timed loop: device
        buffers, pinned staging, the labels' pressure operator and a context
        (what CompiledScenario.compile does once per scenario)."""
        s = self._slot(state.grid)
        self._sync_static(s, state)
        pre = _pre_kind(preconditioner, psys, self.ai_omega)
        ctx = s.psys.pool.acquire(s.grid, s.psys.labels_on(self.device), pre.omega, pre.kind, self.dtype,
                                  self.device)
        s.psys.pool.release(ctx)
        torch.cuda.synchronize(self.device)

    # -- the step --------------------------------------------------------------
    def step(self, state, params, psys=None, preconditioner=None, profile=None, advector=None,
             pcg_tol: float | None = None) -> StepReport:
        prm = _params(params)
        if prm.dt == 0.0:
            return StepReport()        # solver.py:413-414: dt == 0 leaves the state untouched
        s = self._slot(state.grid)
        self._sync_static(s, state)
        pre = _pre_kind(preconditioner, psys, self.ai_omega)
        lib = N.lib()
        ctx = s.psys.pool.acquire(s.grid, s.psys.labels_on(self.device), pre.omega, pre.kind, self.dtype,
                                  self.device)
        try:
            cur = torch.cuda.current_stream(self.device)
            late = {}
            # 1. host arrays -> device float64 staging -> device layout
            for n in ORDER:
                a = getattr(state, n)
                if a.shape != _shape(s.grid, n):
                    raise ValueError(f"{n} has shape {a.shape}, expected {_shape(s.grid, n)}")
                if s.ours.get(n) == id(a):
                    host = s.pin_out[1 - s.out_set][n]       # returned by the previous call: pinned already
                else:
                    np.copyto(s.pin_in[n].numpy(), a, casting="same_kind")
                    host = s.pin_in[n]
                with torch.cuda.stream(s.up):
                    s.d64[n].copy_(host.view(-1), non_blocking=True)
                    self.h2d_bytes += s.d64[n].numel() * 8
                    if n in LATE:     # converted on the copy stream: the step waits late
                        N.check(lib.cw_ref_layout(ctx.h, 0, KIND[n], N.ptr(s.d64[n]), N.ptr(s.dev.fields[n]),
                                                  N.c_stream(s.up)))
                        ev = torch.cuda.Event()
                        ev.record(s.up)
                        late[n] = ev
                    else:
                        ev = torch.cuda.Event()
                        ev.record(s.up)
                if n not in late:
                    cur.wait_event(ev)
                    N.check(lib.cw_ref_layout(ctx.h, 0, KIND[n], N.ptr(s.d64[n]), N.ptr(s.dev.fields[n]),
                                              N.c_stream(cur)))
        finally:
            s.psys.pool.release(ctx)
        s.dev.touch()
        # 2. one device step.  If it raises, the reference's step has already
        # reassigned the state's arrays (solver.py:423-425 onwards) and left
        # them as they are at the raise; the device state is rolled back to
        # exactly that (solver._rollback), so it is downloaded before the
        # exception propagates, without advancing time / step_count
        try:
            rep = _dev_step(s.dev, prm, s.psys, pre, _profile(profile), pcg_tol=pcg_tol,
                            _defer=(late["nu_t"], late["p"], late["omega"]))
        except Exception:
            try:
                self._download(s, state, pre)
            except Exception:   # a failed download must not mask the step's exception
                pass
            raise
        self._download(s, state, pre)
        state.time += prm.dt
        state.step_count += 1
        return rep

    def _download(self, s: _Slot, state, pre) -> None:
        """device layout -> float64 C order -> pinned host arrays assigned to
        the state's attributes."""
        lib = N.lib()
        out, out_np = s.pin_out[s.out_set], s.np_out[s.out_set]
        ctx = s.psys.pool.acquire(s.grid, s.psys.labels_on(self.device), pre.omega, pre.kind, self.dtype,
                                  self.device)
        try:
            cur = torch.cuda.current_stream(self.device)
            for n in ORDER:
                N.check(lib.cw_ref_layout(ctx.h, 1, KIND[n], N.ptr(s.dev.fields[n]), N.ptr(s.d64[n]),
                                          N.c_stream(cur)))
                ev = torch.cuda.Event()
                ev.record(cur)
                with torch.cuda.stream(s.down):
                    s.down.wait_event(ev)
                    out[n].view(-1).copy_(s.d64[n], non_blocking=True)
                    self.d2h_bytes += s.d64[n].numel() * 8
            s.down.synchronize()
        finally:
            s.psys.pool.release(ctx)
        for n in ORDER:
            setattr(state, n, out_np[n])
            s.ours[n] = id(out_np[n])
        s.out_set ^= 1


_default = None


def step(state, params, psys=None, preconditioner=None, profile=None, advector=None, pcg_tol=None,
         ai_omega: float = 1.65) -> StepReport:
    """Module-level drop-in for ``citywind.solver.step`` (solver.py:407-461)."""
    global _default
    if _default is None or _default.ai_omega != float(ai_omega):
        _default = RefStepper(ai_omega=ai_omega)
    return _default.step(state, params, psys, preconditioner, profile, advector, pcg_tol)
