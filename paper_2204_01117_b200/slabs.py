"""z-slab decomposition of one simulation.

The reference steps one grid in one process (solver.py:407-461).  Here the
grid splits into z-slabs: slab r owns cell planes [k_lo, k_hi) (and the
w-faces with the same indices, the last slab also face nz) and keeps a window
of ``halo`` extra planes on each side.  x-fastest storage makes every plane
one contiguous run of memory, so a halo exchange is a plane copy.

A step on the slabs (``SlabDomain.step``):

1. refresh every window's halo planes of the state from the owners;
2. ``CW_STAGE_PRE`` on each window (advect, diffuse, drag, boundary).  Each
   stage reads at most a few planes around a cell, so the owned planes come
   out exactly as in the whole-grid step while the outer halo planes (whose
   neighbours lie outside the window) go stale; ``halo`` covers the reach of
   the whole chain;
3. the projection on all slabs at once: one cooperative launch per device
   whose blocks push their boundary planes into the neighbours' halo planes
   while they compute them, and whose dot products are folded per slab and
   combined in slab order (``cw_slab_group_pcg`` on one device,
   ``cw_slab_attach`` across devices);
4. refresh the halo planes of p (the gradient update reads across the slab
   faces);
5. ``CW_STAGE_POST`` on each window (gradient, div after, turbulence,
   boundary, CFL).

Reductions (div before/after, CFL, region sums, the default PCG tolerance)
cover owned planes only and are combined over slabs.

Backends of the halo refresh: ``LocalExchange`` (every slab in this process,
plane copies) and ``DistExchange`` (one slab per rank, torch.distributed
point-to-point: NCCL over NVLink on the GPU, gloo on the CPU for tests).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .grid import FIELDS, FlowState, GridSpec
from .linalg import PcgReport
from .solver import SolverParams, InletProfile, StepReport, drag_coefficient

DEFAULT_HALO = 4
_DT = {torch.float32: 4, torch.float64: 8}


def plan_slabs(nz: int, n: int, align: int = 1) -> list:
    """Balanced contiguous plane ranges [(k_lo, k_hi), ...] in z order.  With
    ``align`` > 1 the inner boundaries fall on multiples of ``align`` when
    the planes allow it (the PCG's chunk size: the slab split then sums the
    dot products exactly as the whole grid does, bit for bit)."""
    if not 1 <= n <= nz:
        raise ValueError(f"cannot split {nz} planes into {n} slabs")
    nblk = -(-nz // align) if align > 1 else nz
    if align > 1 and nblk >= n:
        base, extra = divmod(nblk, n)
        out, k = [], 0
        for r in range(n):
            t = (base + (1 if r < extra else 0)) * align
            out.append((k, min(k + t, nz)))
            k = min(k + t, nz)
        if all(b > a for a, b in out):
            return out
    base, extra = divmod(nz, n)
    out, k = [], 0
    for r in range(n):
        t = base + (1 if r < extra else 0)
        out.append((k, k + t))
        k += t
    return out


def whole_grid_chunk(grid: GridSpec, dtype, device) -> int:
    """The z-chunk a whole-grid context's PCG uses (``cw_pcg_chunk_of``)."""
    g = N.cw_grid(grid.nx, grid.ny, grid.nz, float(grid.dx), float(grid.dy), float(grid.dz), N.dbl3(grid.origin))
    zc = C.c_int()
    N.check(N.lib().cw_pcg_chunk_of(C.byref(g), _DT[dtype], torch.device(device).index or 0, C.byref(zc)))
    return int(zc.value)


def whole_grid_tol(state: FlowState, omega: float, precond: int) -> float:
    """default_projection_tol of the whole grid (solver.py:235-243), computed
    exactly as the single-context step computes it."""
    from .runtime import Context
    ctx = Context(state.grid, state.dtype, state.device)
    ctx.set_operator(state.labels_dev, omega, precond)
    return ctx.tol_default


@dataclass(frozen=True)
class SlabWindow:
    """Planes of one slab: owned [k_lo, k_hi), stored window [kb, ke)."""
    k_lo: int
    k_hi: int
    kb: int
    ke: int
    nz: int                     # global plane count

    @classmethod
    def of(cls, k_lo, k_hi, halo, nz):
        return cls(k_lo, k_hi, max(k_lo - halo, 0), min(k_hi + halo, nz), nz)

    @property
    def nz_local(self) -> int:
        return self.ke - self.kb

    def planes(self, name: str) -> tuple:
        """Global index range of the window's stored planes of a field."""
        return (self.kb, self.ke + (1 if name == "w" else 0))

    def owned(self, name: str) -> tuple:
        """Global index range of the planes this slab owns (w: faces k_lo..k_hi-1, plus nz on the top slab)."""
        top = 1 if (name == "w" and self.k_hi == self.nz) else 0
        return (self.k_lo, self.k_hi + top)


def window_of(t: torch.Tensor, win: SlabWindow, name: str) -> torch.Tensor:
    """The window of a whole-grid device field (planes are the leading dim)."""
    a, b = win.planes(name)
    return t[a:b]


# ---------------------------------------------------------------------------
# halo exchange backends

class LocalExchange:
    """Every slab in this process: copy each halo plane from its owner."""

    def __init__(self, windows: list):
        self.windows = windows

    def owner(self, g: int, name: str) -> int:
        for r, w in enumerate(self.windows):
            a, b = w.owned(name)
            if a <= g < b:
                return r
        raise IndexError(g)

    def exchange(self, fields: list, names=FIELDS):
        """fields[r][name]: slab r's window tensors."""
        for r, w in enumerate(self.windows):
            for name in names:
                a, b = w.planes(name)
                oa, ob = w.owned(name)
                for lo, hi in ((a, oa), (ob, b)):
                    g = lo
                    while g < hi:     # runs of planes with one owner
                        s = self.owner(g, name)
                        sa, sb = self.windows[s].owned(name)
                        e = min(hi, sb)
                        src = fields[s][name][g - self.windows[s].kb:e - self.windows[s].kb]
                        fields[r][name][g - w.kb:e - w.kb].copy_(src)
                        g = e


class DistExchange:
    """One slab per rank (torch.distributed point-to-point: NCCL over NVLink
    on the GPU, gloo on the CPU).  The halo depth must not exceed a
    neighbour's owned thickness, so only adjacent ranks talk."""

    def __init__(self, windows: list, rank: int, group=None):
        self.windows = windows
        self.rank = rank
        self.group = group

    def exchange(self, fields: dict, names=FIELDS):
        """fields[name]: this rank's window tensors (planes are the leading dim)."""
        import torch.distributed as dist
        r, w = self.rank, self.windows[self.rank]
        ops, keep = [], []
        for name in names:
            t = fields[name]
            a, b = w.planes(name)
            oa, ob = w.owned(name)
            for nb in (r - 1, r + 1):
                if not 0 <= nb < len(self.windows):
                    continue
                v = self.windows[nb]
                va, vb = v.planes(name)
                voa, vob = v.owned(name)
                # what I hold of theirs: my window minus my owned part, on their side
                ra, rb = (a, oa) if nb < r else (ob, b)
                # what they hold of mine: their window minus their owned part, on my side
                sa, sb = (vob, vb) if nb < r else (va, voa)
                if not (voa <= ra and rb <= vob) or not (oa <= sa and sb <= ob):
                    raise ValueError("halo deeper than a neighbour slab")
                if rb > ra:
                    recv = t[ra - w.kb:rb - w.kb]
                    keep.append(recv)
                    ops.append(dist.P2POp(dist.irecv, recv, nb, self.group))
                if sb > sa:
                    send = t[sa - w.kb:sb - w.kb].contiguous()
                    keep.append(send)
                    ops.append(dist.P2POp(dist.isend, send, nb, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


# ---------------------------------------------------------------------------
# one slab on the device

class SlabPart:
    """A slab context (``cw_ctx_create_slab``) with its window of the state."""

    def __init__(self, grid: GridSpec, win: SlabWindow, halo: int, dtype, device):
        self.grid = grid
        self.win = win
        self.device = torch.device(device)
        self.dtype = dtype
        self._lib = N.lib()
        g = N.cw_grid(grid.nx, grid.ny, grid.nz, float(grid.dx), float(grid.dy), float(grid.dz),
                      N.dbl3(grid.origin))
        h = C.c_void_p()
        N.check(self._lib.cw_ctx_create_slab(C.byref(g), win.k_lo, win.k_hi, int(halo), _DT[dtype],
                                             self.device.index or 0, C.byref(h)))
        self.h = h
        self.fields = None
        self.labels = None
        self.g = None
        self.has_drag = False

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

    def load(self, state: FlowState, params: SolverParams):
        """Copy this slab's window out of a whole-grid state."""
        self.fields = {n: window_of(state.fields[n], self.win, n).clone() for n in FIELDS}
        self.labels = window_of(state.labels_dev, self.win, "p").contiguous()
        g, has = drag_coefficient(state, params)
        self.g = window_of(g, self.win, "p").contiguous()
        self.has_drag = has

    def set_chunk(self, zc: int):
        N.check(self._lib.cw_set_pcg_chunk(self.h, int(zc)))
        z, nch = C.c_int(), C.c_int()
        N.check(self._lib.cw_pcg_chunks(self.h, C.byref(z), C.byref(nch)))
        return int(nch.value)

    def set_operator(self, omega: float, precond: int = 2):
        n, tol = C.c_longlong(), C.c_double()
        N.check(self._lib.cw_set_operator(self.h, N.ptr(self.labels), float(omega), C.byref(n), C.byref(tol),
                                          self.stream))
        tk = C.c_double()
        N.check(self._lib.cw_set_preconditioner(self.h, int(precond), C.byref(tk)))
        s, js, m, outl = C.c_double(), C.c_double(), C.c_longlong(), C.c_int()
        N.check(self._lib.cw_operator_partials(self.h, C.byref(s), C.byref(js), C.byref(m), C.byref(outl)))
        return float(s.value), float(js.value), int(m.value), bool(outl.value)

    def native_fields(self):
        f = self.fields
        return N.cw_fields(N.ptr(f["u"]), N.ptr(f["v"]), N.ptr(f["w"]), N.ptr(f["p"]), N.ptr(f["k"]),
                           N.ptr(f["omega"]), N.ptr(f["nu_t"]), N.ptr(self.labels), N.ptr(self.g),
                           int(bool(self.has_drag)), N.labels_version(self.labels))

    def run(self, stage: int, prm, inl, tol=-1.0):
        f = self.native_fields()
        N.check(self._lib.cw_run_stage(self.h, C.byref(f), C.byref(prm), C.byref(inl), int(stage), float(tol),
                                       self.stream))

    def reports(self, n):
        out = (N.cw_report * max(n, 1))()
        got = C.c_int()
        rc = self._lib.cw_read_reports(self.h, out, n, C.byref(got), self.stream)
        return rc, [out[i] for i in range(got.value)]

    def buffers(self) -> N.cw_slab_buffers:
        b = N.cw_slab_buffers()
        N.check(self._lib.cw_slab_buffers_get(self.h, C.byref(b)))
        return b

    def owned_view(self, name: str) -> torch.Tensor:
        a, b = self.win.owned(name)
        return self.fields[name][a - self.win.kb:b - self.win.kb]


def _combine(parts_reports, tol):
    """Merge the per-slab reports of one step (PRE, SOLVE, POST slots)."""
    its = {int(r[1].iterations) for r in parts_reports}
    if len(its) != 1:
        raise RuntimeError(f"slabs disagree on the PCG iteration count: {sorted(its)}")
    sol = parts_reports[0][1]
    div_before = max(float(r[1].div_before) for r in parts_reports)
    div_after = max(float(r[2].div_after) for r in parts_reports)
    cfl = max(float(r[2].cfl) for r in parts_reports)
    return StepReport(timings={}, pcg=PcgReport(int(sol.iterations), bool(sol.converged), float(sol.criterion)),
                      cfl=cfl, div_before=div_before, div_after=div_after)


class SlabDomain:
    """Every slab of one grid in this process, on one device (the emulated
    decomposition: the same kernels and exchange plan as one slab per GPU)."""

    def __init__(self, state: FlowState, params: SolverParams, profile: InletProfile, nslab: int,
                 omega: float = 1.65, precond: int = 2, halo: int = DEFAULT_HALO, pcg_tol=None):
        grid = state.grid
        self.grid = grid
        self.params = params
        self.profile = profile
        self.zc = whole_grid_chunk(grid, state.dtype, state.device)
        ranges = plan_slabs(grid.nz, nslab, self.zc)
        if min(b - a for a, b in ranges) < halo:
            raise ValueError(f"slabs of {min(b - a for a, b in ranges)} planes cannot feed a {halo}-plane halo")
        self.windows = [SlabWindow.of(a, b, halo, grid.nz) for a, b in ranges]
        self.halo = halo
        self.parts = [SlabPart(grid, w, halo, state.dtype, state.device) for w in self.windows]
        for p in self.parts:
            p.load(state, params)
            if p.win.k_lo % self.zc == 0:
                p.set_chunk(self.zc)      # the whole grid's chunks: bitwise the whole grid's dot products
        sums = [p.set_operator(omega, precond) for p in self.parts]
        n = sum(s[2] for s in sums)
        if n == 0:
            raise ValueError("no flow cells to solve for")
        if not any(s[3] for s in sums):
            from .errors import SingularSystemError
            raise SingularSystemError("no outlet cells: pressure defined only up to a constant")
        self.tol = float(pcg_tol) if pcg_tol is not None else whole_grid_tol(state, omega, precond)
        self.exchange = LocalExchange(self.windows)
        self.time = state.time
        self.step_count = state.step_count

    def step(self) -> StepReport:
        prm = self.params.native()
        inl = self.profile.native()
        self.exchange.exchange([p.fields for p in self.parts])
        for p in self.parts:
            p.run(N.CW_STAGE_PRE, prm, inl)
        ctxs = (C.c_void_p * len(self.parts))(*[p.h.value for p in self.parts])
        fs = (N.cw_fields * len(self.parts))(*[p.native_fields() for p in self.parts])
        N.check(N.lib().cw_slab_group_pcg(ctxs, fs, len(self.parts), C.byref(prm), self.tol,
                                          self.parts[0].stream))
        self.exchange.exchange([p.fields for p in self.parts], names=("p",))
        for p in self.parts:
            p.run(N.CW_STAGE_POST, prm, inl)
        reps = []
        for p in self.parts:
            rc, r = p.reports(3)
            if rc != N.CW_OK:
                from .solver import _raise_for
                bad = next((x for x in r if x.status != N.CW_OK), r[-1] if r else None)
                _raise_for(rc, bad, self.grid)
            reps.append(r)
        self.time += self.params.dt
        self.step_count += 1
        return _combine(reps, self.tol)

    def gather(self) -> dict:
        """Whole-grid device copies of the owned planes of every field."""
        out = {}
        for name in FIELDS:
            out[name] = torch.cat([p.owned_view(name) for p in self.parts], dim=0)
        return out


# ---------------------------------------------------------------------------
# one slab per device (one process per GPU)

class DistSlabSolver:
    """This rank's slab of a grid split over the ranks of a torch.distributed
    group (one GPU each).  Halos move with NCCL point-to-point over NVLink;
    the projection is one cooperative launch per GPU whose blocks store their
    boundary planes straight into the neighbours' halo planes (CUDA IPC
    mappings) and meet the other GPUs at rank 0's barrier."""

    def __init__(self, state: FlowState, params: SolverParams, profile: InletProfile, group=None,
                 omega: float = 1.65, precond: int = 2, halo: int = DEFAULT_HALO, pcg_tol=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.n = dist.get_world_size(group)
        grid = state.grid
        self.grid = grid
        self.params = params
        self.profile = profile
        self.zc = whole_grid_chunk(grid, state.dtype, state.device)
        ranges = plan_slabs(grid.nz, self.n, self.zc)
        if min(b - a for a, b in ranges) < halo:
            raise ValueError(f"slabs of {min(b - a for a, b in ranges)} planes cannot feed a {halo}-plane halo")
        self.windows = [SlabWindow.of(a, b, halo, grid.nz) for a, b in ranges]
        self.halo = halo
        self.part = SlabPart(grid, self.windows[self.rank], halo, state.dtype, state.device)
        self.part.load(state, params)
        aligned = all(a % self.zc == 0 for a, _ in ranges)
        nch = self.part.set_chunk(self.zc) if aligned else None
        s, js, m, outl = self.part.set_operator(omega, precond)
        if nch is None:
            z, c = C.c_int(), C.c_int()
            N.check(N.lib().cw_pcg_chunks(self.part.h, C.byref(z), C.byref(c)))
            nch = int(c.value)
        t = torch.tensor([s, js, float(m), float(outl)], dtype=torch.float64, device=state.device)
        dist.all_reduce(t, group=group)
        if t[2].item() == 0:
            raise ValueError("no flow cells to solve for")
        if t[3].item() == 0:
            from .errors import SingularSystemError
            raise SingularSystemError("no outlet cells: pressure defined only up to a constant")
        # this slab's place in the solve's chunk order (dot products folded per chunk, in order)
        counts = [None] * self.n
        dist.all_gather_object(counts, nch, group=group)
        N.check(N.lib().cw_slab_chunks(self.part.h, sum(counts[:self.rank]), sum(counts)))
        self.tol = float(pcg_tol) if pcg_tol is not None else whole_grid_tol(state, omega, precond)
        self.exchange = DistExchange(self.windows, self.rank, group)
        self._attach()
        self.time = state.time
        self.step_count = state.step_count

    def _attach(self):
        """Open the neighbours' (and rank 0's) PCG buffers through CUDA IPC."""
        if self.n == 1:
            return
        lib = N.lib()
        mine = self.part.buffers()
        handles = {}
        for name in N.cw_slab_buffers.BUFFERS:
            h = (C.c_ubyte * 64)()
            N.check(lib.cw_ipc_get(C.c_void_p(getattr(mine, name)), h))
            handles[name] = bytes(h)
        allh = [None] * self.n
        self.dist.all_gather_object(allh, (handles, mine.o0, mine.o1), group=self.group)
        dev = self.part.device.index or 0
        self._opened = []

        def open_peer(r):
            if r == self.rank:
                return mine
            hs, o0, o1 = allh[r]
            b = N.cw_slab_buffers()
            for name in N.cw_slab_buffers.BUFFERS:
                p = C.c_void_p()
                N.check(lib.cw_ipc_open((C.c_ubyte * 64)(*hs[name]), dev, C.byref(p)))
                self._opened.append(p)
                setattr(b, name, p.value)
            b.o0, b.o1 = o0, o1
            return b

        lower = open_peer(self.rank - 1) if self.rank > 0 else None
        upper = open_peer(self.rank + 1) if self.rank + 1 < self.n else None
        root = open_peer(0) if self.rank not in (0, 1) else (mine if self.rank == 0 else lower)
        N.check(lib.cw_slab_attach(self.part.h, self.rank, self.n, C.byref(lower) if lower else None,
                                   C.byref(upper) if upper else None, C.byref(root)))
        self.dist.barrier(group=self.group)

    def step(self) -> StepReport:
        return self.step_many(1)[0]

    def step_many(self, n: int) -> list:
        """n steps enqueued back to back (halo exchanges are NCCL calls on the
        same stream), then one read of the 3n stage reports and one max
        all-reduce of the per-step diagnostics."""
        prm = self.params.native()
        inl = self.profile.native()
        p = self.part
        done = 0
        out = []
        while done < n:
            chunk = min(n - done, 1000)       # 3 report slots per step (ring of 4096)
            for _ in range(chunk):
                self.exchange.exchange(p.fields)
                p.run(N.CW_STAGE_PRE, prm, inl)
                p.run(N.CW_STAGE_SOLVE, prm, inl, self.tol)
                self.exchange.exchange(p.fields, names=("p",))
                p.run(N.CW_STAGE_POST, prm, inl)
            rc, r = p.reports(3 * chunk)
            if rc != N.CW_OK:
                from .solver import _raise_for
                bad = next((x for x in r if x.status != N.CW_OK), r[-1] if r else None)
                _raise_for(rc, bad, self.grid)
            t = torch.tensor([[r[3 * q + 1].div_before, r[3 * q + 2].div_after, r[3 * q + 2].cfl]
                              for q in range(chunk)], dtype=torch.float64, device=p.device)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
            for q in range(chunk):
                sr = r[3 * q + 1]
                out.append(StepReport(timings={}, pcg=PcgReport(int(sr.iterations), bool(sr.converged),
                                                                float(sr.criterion)),
                                      cfl=float(t[q, 2]), div_before=float(t[q, 0]), div_after=float(t[q, 1])))
            self.time += self.params.dt * chunk
            self.step_count += chunk
            done += chunk
        return out
