"""Time-split RANS step on the B200 (reference ``citywind.solver``).

Same public names, argument meanings, defaults and exceptions as the
reference module (solver.py:26-549); every compute call lands in the CUDA
kernels of ``libcitywind_b200.so`` through the C ABI (include/citywind_b200.h).
``step`` runs one whole step per call (synchronising once to return its
StepReport, like the reference); ``step_many`` enqueues many steps with no
host synchronisation between them.
"""
from __future__ import annotations

import ctypes as C
import threading
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import ProjectionError
from .grid import CellLabel, FlowState, GridSpec, PorosityField, default_device
from .linalg import MatrixPreconditioner, PcgReport, PressureSystem
from .runtime import Context

VON_KARMAN = 0.41
DIV_REDUCTION_TARGET = 10.0 ** -4.5
STAGE_KEYS = ("advect", "diffuse", "drag", "boundary", "project", "turbulence", "boundary2")
K_FLOOR, OMEGA_FLOOR = 1e-12, 1e-8


def inlet_turbulence(intensity, u_ref, length_scale, c_mu=0.09):
    """k = 1.5 (I U)^2, omega = C_mu^-1/4 sqrt(k) / L (turbulence.py:26-33)."""
    k = max(1.5 * (intensity * u_ref) ** 2, K_FLOOR)
    om = c_mu ** (-0.25) * np.sqrt(k) / length_scale
    return k, max(om, OMEGA_FLOOR)


def nu_stable(grid: GridSpec, dt: float) -> float:
    """turbulence.py:18-23"""
    s = 1.0 / grid.dx ** 2 + 1.0 / grid.dy ** 2
    if not grid.is_2d:
        s += 1.0 / grid.dz ** 2
    return 1.0 / (2.0 * dt * s)


@dataclass
class SolverParams:
    """solver.py:26-50 (same fields and defaults)."""

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

    def native(self, dt=None) -> N.cw_params:
        k_in, om_in = self.inlet_k_omega()
        return N.cw_params(float(self.dt if dt is None else dt), self.nu, self.cd_tree,
                           self.cd_building, self.drag_a, self.drag_b, self.drag_eps, self.c_mu,
                           self.alpha, self.beta, self.sigma, self.sigma_star, self.c_lim,
                           float(k_in), float(om_in), int(bool(self.turbulence)))


@dataclass
class InletProfile:
    """solver.py:54-97: uniform or logarithmic inlet wind along a direction."""

    kind: str = "uniform"
    speed: float = 1.0
    u_star: float = 0.5
    z0: float = 0.5
    kappa: float = VON_KARMAN
    direction: tuple = (1.0, 0.0)

    def __post_init__(self):
        d = np.asarray(self.direction, dtype=float)[:2]
        n = np.linalg.norm(d)
        if n == 0:
            raise ValueError("inlet direction must be non-zero")
        self.direction = (float(d[0] / n), float(d[1] / n))
        if self.kind not in ("uniform", "logarithmic"):
            raise ValueError(f"unknown inlet profile kind {self.kind!r}")

    def speed_at(self, z) -> np.ndarray:
        z = np.asarray(z, dtype=float)
        if self.kind == "uniform":
            return np.full_like(z, self.speed)
        out = np.zeros_like(z)
        above = z > self.z0
        out[above] = self.u_star / self.kappa * np.log(z[above] / self.z0)
        return out

    def reference_speed(self, grid: GridSpec) -> float:
        if self.kind == "uniform":
            return self.speed
        z_top = grid.origin[2] + grid.nz * grid.dz
        return float(self.speed_at(np.array([max(z_top, self.z0 * np.e)]))[0])

    def rotated(self, degrees: float) -> "InletProfile":
        a = np.deg2rad(degrees)
        dx, dy = self.direction
        return InletProfile(kind=self.kind, speed=self.speed, u_star=self.u_star, z0=self.z0,
                            kappa=self.kappa,
                            direction=(dx * np.cos(a) - dy * np.sin(a), dx * np.sin(a) + dy * np.cos(a)))

    def native(self) -> N.cw_inlet:
        return N.cw_inlet(0 if self.kind == "uniform" else 1, float(self.speed), float(self.u_star),
                          float(self.z0), float(self.kappa), float(self.direction[0]),
                          float(self.direction[1]))


@dataclass
class StepReport:
    """solver.py:101-110"""

    timings: dict = field(default_factory=dict)
    pcg: PcgReport | None = None
    cfl: float = 0.0
    div_before: float = 0.0
    div_after: float = 0.0

    @property
    def wall_time(self) -> float:
        return sum(self.timings.values())


# ---------------------------------------------------------------------------
# context plumbing

_scratch = {}
_scratch_lock = threading.Lock()


def _scratch_ctx(state: FlowState) -> Context:
    """A context without a pressure operator, for the non-projection stages."""
    key = (state.grid, state.dtype, str(state.device))
    with _scratch_lock:
        ctx = _scratch.get(key)
        if ctx is None:
            ctx = _scratch[key] = Context(state.grid, state.dtype, state.device)
    return ctx


def _pre_kind(preconditioner):
    if preconditioner is None:
        return 0, 1.65
    if isinstance(preconditioner, MatrixPreconditioner):
        return preconditioner.kind, preconditioner.omega
    kind = getattr(preconditioner, "kind", None)
    if kind is None:
        raise TypeError("preconditioner must come from paper_2204_01117_b200.linalg")
    return int(kind), float(getattr(preconditioner, "omega", 1.65))


def _acquire(psys: PressureSystem, preconditioner, state: FlowState) -> Context:
    if not isinstance(psys, PressureSystem):
        raise TypeError("psys must be a paper_2204_01117_b200.linalg.PressureSystem")
    if psys.grid != state.grid:
        raise ValueError("pressure system and state are on different grids")
    kind, omega = _pre_kind(preconditioner)
    return psys.pool.acquire(psys.grid, psys.labels_on(state.device), omega, kind, state.dtype,
                             state.device)


def drag_coefficient(state: FlowState, params: SolverParams):
    """Per-cell C_d * G on the device (drag_factor_cells, solver.py:123-135),
    cached on the state until its labels/porosity or the drag constants change."""
    key = (params.cd_tree, params.cd_building, params.drag_a, params.drag_b, params.drag_eps,
           state.dtype)
    if state._drag_key != key:
        ctx = _scratch_ctx(state)
        if state._g is None or state._g.dtype != state.dtype:
            state._g = torch.empty(state.grid.dshape("p"), dtype=state.dtype, device=state.device)
        prm = params.native()
        has = C.c_int()
        N.check(N.lib().cw_drag_coefficient(ctx.h, N.ptr(state.phi_dev), N.ptr(state.lad_dev),
                                            N.ptr(state.labels_dev), C.byref(prm), N.ptr(state._g),
                                            C.byref(has), ctx.stream))
        state._has_drag = bool(has.value)
        state._drag_key = key
    return state._g, state._has_drag


def drag_factor_cells(state: FlowState, params: SolverParams) -> np.ndarray:
    g, _ = drag_coefficient(state, params)
    return np.ascontiguousarray(g.cpu().numpy().astype(np.float64).transpose(2, 1, 0))


def _raise_for(rc: int, rep, grid: GridSpec):
    if rc == N.CW_OK:
        return
    if rc == N.CW_ERR_PCG:
        raise ProjectionError(PcgReport(rep.iterations, bool(rep.converged), rep.criterion))
    if rc == N.CW_ERR_HALO:
        raise ValueError(f"z-slab halo too shallow: max|w| dt/dz = {rep.criterion:.3f} this step reaches "
                         f"{rep.bad_cell} planes across a slab face (2 floor(S) + 4); rebuild the slabs "
                         f"with halo >= {rep.bad_cell} or take a smaller dt")
    if rc == N.CW_ERR_NONFINITE:
        ijk = tuple(int(x) for x in np.unravel_index(rep.bad_cell, grid.shape))
        name = "k" if rep.bad_field == 0 else "omega"
        raise FloatingPointError(f"turbulence update produced non-finite {name} at cell {ijk}")
    N.check(rc)


def _rollback(ctx, f, rep, step_turbulence=None):
    """Leave the state as the reference does when a step raises.
    * A non-finite turbulence update (turbulence.py:121-131, raised before it
      assigns): advected k and omega, the previous nu_t (``cw_turb_rollback``).
    * A failed projection inside a full step (solver.py:272-276, ProjectionError
      or the non-finite right-hand side's ValueError): p untouched by the
      solve, and with turbulence on the step's advected k and omega
      (``cw_proj_rollback``); ``step_turbulence`` is None for a stand-alone
      project(), which touches neither."""
    if rep.status == N.CW_ERR_NONFINITE:
        N.check(N.lib().cw_turb_rollback(ctx.h, C.byref(f), ctx.stream))
    elif rep.status in (N.CW_ERR_PCG, N.CW_ERR_RHS) and step_turbulence is not None:
        N.check(N.lib().cw_proj_rollback(ctx.h, C.byref(f), int(bool(step_turbulence)), ctx.stream))


def _report_of(r, timings) -> StepReport:
    return StepReport(timings=timings, pcg=PcgReport(int(r.iterations), bool(r.converged), float(r.criterion)),
                      cfl=float(r.cfl), div_before=float(r.div_before), div_after=float(r.div_after))


def _warn_cap(state, params, dt):
    if nu_stable(state.grid, dt) - params.nu <= 0:
        warnings.warn(f"time step {dt} exceeds the molecular-diffusion stability bound; "
                      "eddy viscosity fully suppressed this step", stacklevel=3)


# ---------------------------------------------------------------------------
# the step

def step(state: FlowState, params: SolverParams, psys: PressureSystem, preconditioner,
         profile: InletProfile, advector=None, pcg_tol: float | None = None, _defer=None) -> StepReport:
    """One time-split step (solver.py:407-461); returns per-stage device
    timings (seconds) and the solver statistics.  ``_defer`` (internal):
    (nu_t_ready, p_ready[, k_omega_ready]) CUDA events the step waits for
    before the first stage that uses that field (``cw_step_defer``,
    ``cw_step_defer_kw``)."""
    reps = step_many(state, params, psys, preconditioner, profile, 1, pcg_tol, stage_timings=True, _defer=_defer)
    return reps[0] if reps else StepReport()


class HostStepper:
    """Steps a host-resident state: the reference's drop-in for callers whose
    ``FlowState`` lives in host memory (solver.py:407-461 on numpy arrays).

    ``host`` maps the seven field names to pinned CPU tensors in the device
    layout; ``state`` is the device ``FlowState`` the steps run on.  Every
    ``step`` uploads all seven fields, runs one step and downloads all seven
    fields again.  The copies run on their own streams, in pieces (CHUNKS per
    field), and overlap across the two copy directions: a piece of step s+1
    starts uploading as soon as the same piece of step s is back in host
    memory, while the later pieces are still coming down.  The step starts
    once u, v, w are up; nu_t, p, k and omega travel later and the step
    waits for each only before its first stage that uses it (the diffusion,
    the first boundary pass, and for k / omega the upwind step moved behind
    the projection: ``cw_step_defer``, ``cw_step_defer_kw``), so their copies
    overlap the step.  ``synchronize()`` waits for the last download.
    """

    CHUNKS = 1   # pieces per field (4 measured the same at C3: the duplex link is the limit)
    LATE = ("nu_t", "p", "k", "omega")   # fields whose upload may overlap the step, in use order

    def __init__(self, state: FlowState, host: dict):
        from .grid import FIELDS
        assert self.LATE in ((), ("nu_t", "p"), ("nu_t", "p", "k", "omega")), \
            "cw_step_defer knows nu_t and p, cw_step_defer_kw k and omega"
        self.names = tuple(n for n in FIELDS if n not in self.LATE) + tuple(self.LATE)
        self._n_early = len(self.names) - len(self.LATE)
        self.state = state
        self.host = host
        dev = state.fields[self.names[0]].device
        self._up = torch.cuda.Stream(dev)
        self._down = torch.cuda.Stream(dev)
        # (device piece, host piece) views, and the events marking each piece back on the host
        self._pieces = []
        for n in self.names:
            d, h = state.fields[n].view(-1), host[n].view(-1)
            b = np.linspace(0, d.numel(), self.CHUNKS + 1).astype(int)
            self._pieces += [(d[b[q]:b[q + 1]], h[b[q]:b[q + 1]]) for q in range(self.CHUNKS)]
        self._back = [None] * len(self._pieces)

    def step(self, params: SolverParams, psys: PressureSystem, preconditioner, profile: InletProfile,
             pcg_tol: float | None = None) -> StepReport:
        cur = torch.cuda.current_stream()
        ready = {}   # field name (None: all early fields) -> upload-complete event
        with torch.cuda.stream(self._up):
            for q, (d, h) in enumerate(self._pieces):
                if self._back[q] is not None:
                    self._up.wait_event(self._back[q])
                d.copy_(h, non_blocking=True)
                nf = (q + 1) // self.CHUNKS          # fields complete after this piece
                if (q + 1) % self.CHUNKS == 0 and nf >= self._n_early:
                    ev = torch.cuda.Event()
                    ev.record(self._up)
                    ready[None if nf == self._n_early else self.names[nf - 1]] = ev
        cur.wait_event(ready[None])
        defer = (ready["nu_t"], ready["p"], ready.get("omega")) if "nu_t" in ready and "p" in ready else None
        rep = step(self.state, params, psys, preconditioner, profile, pcg_tol=pcg_tol, _defer=defer)
        done = torch.cuda.Event()
        done.record(cur)
        with torch.cuda.stream(self._down):
            self._down.wait_event(done)
            for q, (d, h) in enumerate(self._pieces):
                h.copy_(d, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self._down)
                self._back[q] = ev
        return rep

    def synchronize(self):
        self._down.synchronize()


def step_many(state: FlowState, params: SolverParams, psys: PressureSystem, preconditioner,
              profile: InletProfile, nsteps: int, pcg_tol: float | None = None,
              stage_timings: bool = False, read_back: bool = True, _defer=None, regions=None) -> list:
    """``nsteps`` calls of ``step`` enqueued back to back on the device (no
    host synchronisation between steps).  If a step fails, the following
    steps of the batch are skipped on the device and the exception of the
    failing step is raised with the state as it was at the failure.

    ``regions=(lo, hi, sums, counts)``: after every step the mean speeds of
    the boxes (rows of lo / hi) are added on the device to the float64
    tensor ``sums`` and the air-cell counts written to ``counts`` (int64) --
    the trailing window of evaluate_objective (optimize.py:93-99) without a
    host round trip per step (``cw_step_regions``)."""
    dt = params.dt
    if dt == 0.0 or nsteps <= 0:
        return [StepReport() for _ in range(max(nsteps, 0))]
    _warn_cap(state, params, dt)
    state._turbulence = bool(params.turbulence)   # for finish(): the failed step's rollback
    ctx = _acquire(psys, preconditioner, state)
    state.touch()
    try:
        g, has_drag = drag_coefficient(state, params)
        f = ctx.fields(state, g, has_drag)
        prm = params.native()
        inl = profile.native()
        tol = -1.0 if pcg_tol is None else float(pcg_tol)
        lib = N.lib()
        if stage_timings:
            lib.cw_set_stage_timing(ctx.h, 1)
        if _defer is not None:
            N.check(lib.cw_step_defer(ctx.h, C.c_void_p(_defer[0].cuda_event), C.c_void_p(_defer[1].cuda_event)))
            if len(_defer) > 2 and _defer[2] is not None:
                N.check(lib.cw_step_defer_kw(ctx.h, C.c_void_p(_defer[2].cuda_event)))
        if regions is not None:
            rlo, rhi, rsums, rcounts = regions
            rlo = np.ascontiguousarray(np.atleast_2d(rlo), dtype=np.float64)
            rhi = np.ascontiguousarray(np.atleast_2d(rhi), dtype=np.float64)
            if rsums.dtype != torch.float64 or rcounts.dtype != torch.int64 or rsums.numel() < len(rlo):
                raise ValueError("regions: sums must be float64 and counts int64 device tensors of n entries")
            N.check(lib.cw_step_regions(ctx.h, len(rlo), rlo.ctypes.data_as(C.POINTER(C.c_double)),
                                        rhi.ctypes.data_as(C.POINTER(C.c_double)), N.ptr(rsums),
                                        N.ptr(rcounts)))
        t0 = time.perf_counter()
        done = 0
        reports = []
        while done < nsteps:
            chunk = min(nsteps - done, 2048)
            N.check(lib.cw_step(ctx.h, C.byref(f), C.byref(prm), C.byref(inl), tol, chunk, ctx.stream))
            if not read_back:
                done += chunk
                continue
            rc, reps = ctx.read_reports(chunk)
            if rc != N.CW_OK and not reps:
                N.check(rc)
            wall = (time.perf_counter() - t0) / chunk
            timings = {"step": wall}
            if stage_timings:
                ms = (C.c_float * 7)()
                lib.cw_read_stage_timings(ctx.h, ms)
                lib.cw_set_stage_timing(ctx.h, 0)
                timings = {k: float(ms[i]) * 1e-3 for i, k in enumerate(STAGE_KEYS)}
            for r in reps:
                if r.status != N.CW_OK:
                    _rollback(ctx, f, r, params.turbulence)
                    _raise_for(r.status, r, state.grid)
                reports.append(_report_of(r, dict(timings)))
                state.time += dt
                state.step_count += 1
            done += chunk
            t0 = time.perf_counter()
        if not read_back:
            state.time += dt * nsteps
            state.step_count += nsteps
        return reports
    finally:
        if regions is not None:
            N.lib().cw_step_regions(ctx.h, 0, None, None, None, None)
        psys.pool.release(ctx)


def finish(state: FlowState, psys: PressureSystem, preconditioner, nsteps: int):
    """Read back the reports of steps enqueued with ``read_back=False``."""
    ctx = _acquire(psys, preconditioner, state)
    try:
        rc, reps = ctx.read_reports(nsteps)
        for r in reps:
            if r.status != N.CW_OK:
                _rollback(ctx, ctx.fields(state, state._g, state._has_drag), r, getattr(state, "_turbulence", True))
                _raise_for(r.status, r, state.grid)
        return [_report_of(r, {}) for r in reps]
    finally:
        psys.pool.release(ctx)


# ---------------------------------------------------------------------------
# stage functions (same names as the reference; each runs its device kernels)

def _stage(state, params, profile, stage, dt, psys=None, preconditioner=None, tol=None, max_iter=None):
    if psys is not None:
        ctx = _acquire(psys, preconditioner, state)
    else:
        ctx = _scratch_ctx(state)
    state.touch()
    try:
        if max_iter is not None:
            N.check(N.lib().cw_set_max_iter(ctx.h, int(max_iter)))
        g, has_drag = drag_coefficient(state, params) if stage == N.STAGE_DRAG else (None, False)
        f = ctx.fields(state, g, has_drag)
        prm = params.native(dt)
        inl = (profile or InletProfile()).native()
        N.check(N.lib().cw_run_stage(ctx.h, C.byref(f), C.byref(prm), C.byref(inl), stage,
                                     -1.0 if tol is None else float(tol), ctx.stream))
        rc, reps = ctx.read_reports(1)
        if rc != N.CW_OK:
            if not reps:
                N.check(rc)
            _rollback(ctx, f, reps[0])
            _raise_for(rc, reps[0], state.grid)
        return reps[0]
    finally:
        if max_iter is not None:
            N.lib().cw_set_max_iter(ctx.h, 10_000)
        if psys is not None:
            psys.pool.release(ctx)


def advect(state: FlowState, params: SolverParams, dt: float) -> FlowState:
    """Advection stage of step (solver.py:418-425): upwind k/omega
    (advection.py:154-173) and MacCormack u, v, w (advection.py:125-152)."""
    _stage(state, params, None, N.STAGE_ADVECT, dt)
    return state


def diffuse(state: FlowState, params: SolverParams, dt: float) -> FlowState:
    """solver.py:193-208"""
    _warn_cap(state, params, dt)
    _stage(state, params, None, N.STAGE_DIFFUSE, dt)
    return state


def apply_drag(state: FlowState, params: SolverParams, dt: float) -> FlowState:
    """solver.py:150-168"""
    _stage(state, params, None, N.STAGE_DRAG, dt)
    return state


def apply_boundary_conditions(state: FlowState, profile: InletProfile,
                              params: SolverParams) -> FlowState:
    """solver.py:330-400"""
    _stage(state, params, profile, N.STAGE_BOUNDARY, params.dt)
    return state


def update_turbulence(state: FlowState, params: SolverParams, dt: float) -> FlowState:
    """turbulence.py:100-132"""
    _stage(state, params, None, N.STAGE_TURBULENCE, dt)
    return state


def project(state: FlowState, psys: PressureSystem, dt: float, preconditioner=None,
            tol: float | None = None, max_iter: int = 10_000):
    """solver.py:246-304: warm-started PCG + gradient update, on the device.
    A solve that has not converged after ``max_iter`` iterations raises
    ProjectionError (pcg_solve(max_iter), linalg.py:310-368)."""
    if max_iter < 0:
        raise ValueError("max_iter must be >= 0")
    r = _stage(state, SolverParams(dt=dt), None, N.STAGE_PROJECT, dt, psys, preconditioner, tol,
               max_iter=None if max_iter == 10_000 else max_iter)
    return state, PcgReport(int(r.iterations), bool(r.converged), float(r.criterion))


def divergence(state: FlowState) -> torch.Tensor:
    """Cell divergence (solver.py:215-221) as a device tensor (nz, ny, nx)."""
    g = state.grid
    f = state.fields
    div = (f["u"][:, :, 1:] - f["u"][:, :, :-1]) / g.dx + (f["v"][:, 1:, :] - f["v"][:, :-1, :]) / g.dy
    if not g.is_2d:
        div = div + (f["w"][1:] - f["w"][:-1]) / g.dz
    return div


def max_interior_divergence(state: FlowState) -> float:
    """solver.py:224-229 (diagnostic helper; the step computes it in-kernel)."""
    lab = state.labels_dev
    m = (lab == 0) | (lab == 1) | (lab == 2)
    if not bool(m.any()):
        return 0.0
    return float(divergence(state).abs()[m].max())


def make_initial_state(grid: GridSpec, labels, porosity, params: SolverParams,
                       profile: InletProfile, mode: str = "inflow", dtype=torch.float32,
                       device=None) -> FlowState:
    """solver.py:464-481.  ``labels``/``porosity`` may be host arrays in the
    reference layout or a (labels_dev, phi_dev, lad_dev) device triple."""
    device = device or default_device()
    k_in, om_in = params.inlet_k_omega()
    if isinstance(labels, tuple):
        state = FlowState.zeros(grid, k0=k_in, omega0=om_in, dtype=dtype, device=device, static_dev=labels)
    else:
        state = FlowState.zeros(grid, labels, porosity, k0=k_in, omega0=om_in, dtype=dtype,
                                device=device)
    if not params.turbulence:
        state.fields["nu_t"].zero_()
    if mode == "inflow":
        uz = profile.speed_at(grid.origin[2] + (np.arange(grid.nz) + 0.5) * grid.dz)
        dx_, dy_ = profile.direction
        ux = torch.from_numpy(uz * dx_).to(device=device, dtype=dtype)
        uy = torch.from_numpy(uz * dy_).to(device=device, dtype=dtype)
        state.fields["u"].copy_(ux[:, None, None].expand_as(state.fields["u"]))
        state.fields["v"].copy_(uy[:, None, None].expand_as(state.fields["v"]))
    elif mode != "rest":
        raise ValueError(f"unknown init mode {mode!r}")
    apply_boundary_conditions(state, profile, params)
    return state


def region_average_speeds(state: FlowState, los, his) -> tuple:
    """Several region_average_speed boxes in one device pass; returns
    (means, counts)."""
    los = np.atleast_2d(np.asarray(los, float))
    his = np.atleast_2d(np.asarray(his, float))
    n = len(los)
    ctx = _scratch_ctx(state)
    f = ctx.fields(state)
    lo_a, lo_p = N.as_cdouble_array(los.ravel())
    hi_a, hi_p = N.as_cdouble_array(his.ravel())
    means = (C.c_double * n)()
    counts = (C.c_longlong * n)()
    N.check(N.lib().cw_region_speed(ctx.h, C.byref(f), n, lo_p, hi_p, means, counts, ctx.stream))
    return np.array(means[:]), np.array(counts[:])


def region_average_speed(state: FlowState, box_lo, box_hi,
                         z_band: tuple | None = None) -> float:
    """Mean |u| over centres of Air cells inside a box (solver.py:535-549)."""
    lo = np.asarray(box_lo, dtype=float).copy()
    hi = np.asarray(box_hi, dtype=float).copy()
    if z_band is not None:
        lo[2] = max(lo[2], z_band[0])
        hi[2] = min(hi[2], z_band[1])
    means, counts = region_average_speeds(state, lo[None], hi[None])
    if counts[0] == 0:
        raise ValueError("region contains no air cells")
    return float(means[0])


def probe_velocities(state: FlowState, points, out: torch.Tensor | None = None) -> torch.Tensor:
    """Velocities at physical points on the device (``cw_probe``): float64
    staggered trilinear samples of u, v, w (run_simulation's probes,
    scenario.py:473-478, through Advector.velocity_at, advection.py:107-111).
    Returns (or fills) a (n, 3) float64 device tensor; no host synchronisation."""
    pts = torch.as_tensor(np.asarray(points, dtype=np.float64).reshape(-1, 3), device=state.device)
    if out is None:
        out = torch.empty((pts.shape[0], 3), dtype=torch.float64, device=state.device)
    ctx = _scratch_ctx(state)
    f = ctx.fields(state)
    N.check(N.lib().cw_probe(ctx.h, C.byref(f), int(pts.shape[0]), N.ptr(pts), N.ptr(out), ctx.stream))
    # pts is freed only after the kernel ran: torch's caching allocator reuses
    # the block on this same stream, after the kernel in stream order
    return out


def probe_velocity(state: FlowState, pos) -> tuple:
    """Velocity at a physical point (the probes of run_simulation,
    scenario.py:473-478): staggered trilinear samples of u, v, w."""
    v = probe_velocities(state, [pos])[0].cpu().numpy()
    return float(v[0]), float(v[1]), float(v[2])


def trace_streamlines(state: FlowState, seeds, step_len: float, max_steps: int = 2000,
                      min_speed: float = 1e-6) -> list:
    """Midpoint (RK2) streamlines of the instantaneous velocity (solver.py:488-532),
    one device thread per seed (``cw_streamlines``).  A polyline ends on domain
    exit, after max_steps, or where the speed drops below min_speed; seeds
    outside the domain give empty polylines."""
    sd = np.atleast_2d(np.asarray(seeds, dtype=np.float64))
    n = sd.shape[0]
    dev = state.device
    seeds_d = torch.as_tensor(np.ascontiguousarray(sd), device=dev)
    paths = torch.empty((n, int(max_steps) + 1, 3), dtype=torch.float64, device=dev)
    lens = torch.empty(n, dtype=torch.int32, device=dev)
    ctx = _scratch_ctx(state)
    f = ctx.fields(state)
    N.check(N.lib().cw_streamlines(ctx.h, C.byref(f), n, N.ptr(seeds_d), float(step_len), int(max_steps),
                                   float(min_speed), N.ptr(paths), N.ptr(lens), ctx.stream))
    p, m = paths.cpu().numpy(), lens.cpu().numpy()
    return [p[i, :m[i]].copy() if m[i] > 0 else np.empty((0, 3)) for i in range(n)]
