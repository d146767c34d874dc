"""Benchmark: RANS cell-steps/s on the C3 block city (256x256x64), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N=1 runs one C3 simulation on cuda:0.  N>1 (torchrun, one process per GPU)
runs one independent C3 design per GPU -- the optimizer's design-per-GPU
axis (no data-path collective), weak scaling; the timed region is bracketed
by barriers and the max over ranks is reported.  ``--impl reference`` times
the reference algorithm's CPU path (the oracle port, oracle/) on the host
cores over bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

_argv = sys.argv[1:]
# BLAS threads of the CPU legs, set before numpy loads OpenBLAS: all host
# cores for the reference arm, one for the B200 arm's cpu_baseline sample
if "--impl" in _argv and "reference" in _argv:
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
else:
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "RANS cell-steps/sec at 256x256x64 (C3 block city)"
UNIT = "cell-steps/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# algorithmic bytes: per step 164*N + 44*I*Nu (+8*Nu); the PCG
# launch moves 20*N (divergence -> r0) + 8*Nu (z0 = W r0) + 44*I*Nu
PCG_B_PER_UNKNOWN_ITER = 44
ADV_PREDICT_B_PER_CELL = 40   # SURVEY.md 8d phase P1: 5 fields in, 5 out, fp32
ADV_CORRECT_B_PER_CELL = 36   # 6 fields in (velocity, predictor), 3 out, fp32


def c3_doc(dt):
    from paper_2204_01117_b200 import scenes
    return scenes.block_city(256, 256, 64, 2.0, 0, 6, dt)


def hbm_peak():
    try:
        with open(PEAKS_FILE) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    """SM clock and clock-event reasons sampled during the timed region: NVML
    every 10 ms on a thread (falls back to `nvidia-smi -lms 100`)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")
    NAMES = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
    BITS = (0x4, 0x8, 0x40, 0x20)      # nvmlClocksEventReason* (nvml.h)

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.sm, self.mx, self.reasons = [], None, set()
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.nvml = (pynvml, h)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            t0 = time.perf_counter()   # the poll loop is warm before the timed region starts
            while len(self.sm) < 2 and time.perf_counter() - t0 < 2.0:
                time.sleep(0.002)
            self.sm.clear()
            self.reasons.clear()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = int(get_reasons(h))
                for n, b in zip(self.NAMES, self.BITS):
                    if r & b:
                        self.reasons.add(n)
            except Exception:
                pass
            self.stop.wait(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = list(self.sm), self.mx, set(self.reasons)
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml 10 ms" if self.nvml is not None else "nvidia-smi 100 ms"}


# ---------------------------------------------------------------------------
# CPU reference: the reference algorithm (the oracle port, oracle/, pinned to
# the reference's goldens) stepping the C3 city on the host cores

def blas_threads():
    return int(os.environ.get("OPENBLAS_NUM_THREADS", "0") or 0) or (os.cpu_count() or 1)


def oracle_state_from_device(co, comp, dev):
    """The device state after its warm-up steps as an oracle State (the
    oracle keeps the same x-fastest layout, float64)."""
    f = {n: dev.fields[n].double().cpu().numpy() for n in ("u", "v", "w", "p", "k", "omega", "nu_t")}
    return co.State(comp.scene.grid, f["u"], f["v"], f["w"], f["p"], f["k"], f["omega"], f["nu_t"],
                    dev.labels_dev.cpu().numpy(), dev.phi_dev.cpu().numpy(), dev.lad_dev.cpu().numpy(),
                    time=dev.time, step_count=dev.step_count)


def bench_config(args):
    """The `config` dict of both arms (identical by construction)."""
    return {"workload": "C3 block city 256x256x64 (seed 0: 36 buildings + 16 trees), dt %.2f; timed steps "
                        "%d-%d of a simulation from the inflow initial state" % (args.dt, args.warmup + 1,
                                                                                  args.warmup + args.steps),
            "cells": 256 * 256 * 64, "unknowns": 3999992, "dt": args.dt,
            "l2": "inputs larger than L2: ~250 MB state+workspace per step > 126 MB L2",
            "parallelism": "one simulation per process" if int(os.environ.get("WORLD_SIZE", "1")) == 1
            else "design-per-GPU (one C3 simulation per rank)"}


def run_reference(args):
    """`--impl reference`: the reference algorithm's full steps on the host
    cores, same scene, same steps as the B200 arm (warm-up steps W untimed,
    then K timed steps); prints its own per-step PCG iteration counts."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import citywind_oracle as co
    doc = c3_doc(args.dt)
    t0 = time.perf_counter()
    comp = co.Compiled(co.scene_from_dict(doc))
    st = comp.make_state()
    setup = time.perf_counter() - t0
    warm = [comp.step_state(st).pcg.iterations for _ in range(args.warmup)]
    iters, secs = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ts = time.perf_counter()
        iters.append(comp.step_state(st).pcg.iterations)
        secs.append(time.perf_counter() - ts)
    wall = time.perf_counter() - t0
    ncell = doc_cells(doc)
    value = ncell * args.steps / wall
    cores = blas_threads()
    sample = (f"{args.steps} full C3 steps (steps {args.warmup + 1}-{args.warmup + args.steps}) of the oracle "
              f"port (numpy + scipy CSR, the reference's algorithm; pinned to reference goldens), after "
              f"{args.warmup} untimed steps and {setup:.0f} s of voxelize + operator setup; scipy CSR matvec "
              f"and numpy single-threaded, OpenBLAS ddot on {cores} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": bench_config(args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "pcg_iterations": iters, "pcg_iterations_warmup": warm,
            "seconds_per_step": [round(x, 2) for x in secs], "wall_s": wall, "setup_s": setup}
    print(json.dumps(line), flush=True)


def doc_cells(doc):
    g = doc["grid"]
    return g["nx"] * g["ny"] * g["nz"]


def golden_iterations():
    """Per-step PCG counts of the unmodified reference on this scene
    (tests/golden/cfg_c3_city_256.npz, scripts/make_golden_configs.py)."""
    path = os.path.join(ROOT, "tests", "golden", "cfg_c3_city_256.npz")
    if not os.path.exists(path):
        return None
    return np.load(path)["pcg_iterations"].tolist()


# ---------------------------------------------------------------------------
# the B200 arm

def zslab_child(args):
    """Child-process body of the z-slab leg (one per rank, its own process
    group): prints one JSON line on rank 0.  Kept out of the parent so that a
    failure on the multi-GPU path cannot take the bench line down with it."""
    import torch
    import torch.distributed as dist
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    from paper_2204_01117_b200.slabs import DEFAULT_HALO, DistSlabSolver
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    doc = c3_doc(args.dt)
    ncell = doc_cells(doc)
    sc = scenario_from_dict(doc)
    comp = CompiledScenario.compile(sc, dtype=torch.float32)
    state = comp.make_state()
    # a 6-plane halo covers the step's reach for max|w| dt/dz < 2 (2 floor(S) + 4,
    # DESIGN.md 5) when the slabs are deep enough to feed it, else the default 4
    halo = 6 if sc.grid.nz // world >= 6 else DEFAULT_HALO
    sol = DistSlabSolver(state, sc.solver, sc.inlet, omega=sc.ai_omega, pcg_tol=sc.pcg_tol, halo=halo)
    del state
    sol.step_many(args.warmup)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    reps = sol.step_many(args.steps)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        print("ZSLAB " + json.dumps({
            "value": ncell * args.steps / (ms * 1e-3), "ms_per_step": ms / args.steps,
            "pcg_iterations": [r.pcg.iterations for r in reps], "slabs": world,
            "planes_per_slab": [w.k_hi - w.k_lo for w in sol.windows], "halo": halo,
            "path": "slabs.DistSlabSolver: NCCL halo exchange, one cooperative PCG launch per GPU with "
                    "boundary planes stored into the neighbours over NVLink (CUDA IPC) and a cross-GPU barrier"}),
              flush=True)
    dist.destroy_process_group()


def zslab_leg(args, dist, rank):
    """One C3 simulation split into z-slabs, one per GPU, timed in
    a child process per rank (device events, max over ranks).  Returns
    (ok on every rank, result dict)."""
    import subprocess
    import torch
    env = dict(os.environ)
    env["MASTER_PORT"] = str(int(os.environ.get("MASTER_PORT", "29500")) + 11)
    cmd = [sys.executable, os.path.abspath(__file__), "--zslab-child", "--steps", str(args.steps),
           "--warmup", str(args.warmup), "--dt", str(args.dt)]
    res, ok = {}, 1.0
    try:
        out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
        line = next((ln[6:] for ln in out.stdout.splitlines() if ln.startswith("ZSLAB ")), None)
        if out.returncode != 0:
            ok = 0.0
            res = {"error": f"child exit {out.returncode}: {out.stderr.strip().splitlines()[-1] if out.stderr.strip() else ''}"[:300]}
        elif rank == 0:
            res = json.loads(line)
    except Exception as e:   # reported, and the design-per-GPU number stands
        ok = 0.0
        res = {"error": f"{type(e).__name__}: {e}"[:300]}
    flag = torch.tensor([ok], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return bool(flag.item() > 0), res


def run_b200(args):
    import ctypes as C

    import torch

    from paper_2204_01117_b200 import _native as N
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.refbind import RefStepper
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    doc = c3_doc(args.dt)
    ncell = doc_cells(doc)
    sc = scenario_from_dict(doc)
    comp = CompiledScenario.compile(sc, dtype=torch.float32)
    t0 = time.perf_counter()
    state = comp.make_state()
    torch.cuda.synchronize()
    voxelize_s = time.perf_counter() - t0
    nu = comp.psys.n

    # warm-up (untimed): steps 1..W
    warm = [r.pcg.iterations for r in comp.step_states(state, args.warmup)]
    snap = state.copy()                      # the state the timed steps start from
    lib = N.lib()
    ctx = solver._acquire(comp.psys, comp.preconditioner, state)
    comp.psys.pool.release(ctx)

    def timed_steps(st, k, roofline):
        if roofline:
            N.check(lib.cw_pcg_timing(ctx.h, k))
        lib.cw_launch_count(ctx.h, 1)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clocks:
            ev0.record()
            solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, k, sc.pcg_tol,
                             read_back=False)
            ev1.record()
            torch.cuda.synchronize()
        barrier()
        launches = int(lib.cw_launch_count(ctx.h, 1))
        reps = solver.finish(st, comp.psys, comp.preconditioner, k)
        return ev0.elapsed_time(ev1), [r.pcg.iterations for r in reps], launches, clocks

    # the timed steps W+1 .. W+K, device-resident state
    ms, iters, launches, clocks = timed_steps(state, args.steps, True)
    pcg_ms = (C.c_float * args.steps)()
    got = C.c_int()
    N.check(lib.cw_read_pcg_timing(ctx.h, pcg_ms, args.steps, C.byref(got)))
    pcg_ms = np.array(pcg_ms[:got.value], float)
    pred_ms, corr_ms = (C.c_float * args.steps)(), (C.c_float * args.steps)()
    got_a = C.c_int()
    N.check(lib.cw_read_adv_timing(ctx.h, pred_ms, corr_ms, args.steps, C.byref(got_a)))
    pred_ms = np.array(pred_ms[:got_a.value], float)
    corr_ms = np.array(corr_ms[:got_a.value], float)
    ms_max = max_over_ranks(ms)
    value = world * ncell * args.steps / (ms_max * 1e-3)

    # steady state: the K steps after those (PCG counts have settled)
    ms_s, iters_s, _, _ = timed_steps(state, args.steps, False)
    ms_s = max_over_ranks(ms_s)
    steady = {"value": world * ncell * args.steps / (ms_s * 1e-3), "ms_per_step": ms_s / args.steps,
              "steps": f"{args.warmup + args.steps + 1}-{args.warmup + 2 * args.steps}",
              "pcg_iterations": iters_s}

    # roofline of the dominant kernel (k_pcg)
    peak, peak_kind = hbm_peak()
    bytes_per_launch = [20.0 * ncell + 8.0 * nu + PCG_B_PER_UNKNOWN_ITER * i * nu for i in iters[:len(pcg_ms)]]
    achieved = float(np.sum(bytes_per_launch) / (np.sum(pcg_ms) * 1e-3) / 1e9) if len(pcg_ms) else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "pcg_dram_bytes.json")
    if os.path.exists(prof) and bytes_per_launch:
        # measured DRAM bytes of one captured launch (ncu --set full), scaled
        # by its ratio to the algorithmic bytes onto this run's mean launch
        with open(prof) as fh:
            ratio = json.load(fh).get("traffic_over_algorithmic")
        if ratio:
            traffic = float(ratio * np.mean(bytes_per_launch))
    roofline = {"kernel": "k_pcg<float> (whole warm-started PCG, one cooperative launch per step)",
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                "peak_source": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                "bytes_model": "20*N + 8*Nu + 44*I*Nu per launch (SURVEY.md 8d, fp32 vectors)",
                "pcg_ms_per_launch": float(np.mean(pcg_ms)) if len(pcg_ms) else None,
                "pcg_share_of_step": float(np.sum(pcg_ms) / ms) if len(pcg_ms) else None}
    adv = {}
    for name, t_ms, bpc, what in (
            ("k_mac_predict", pred_ms, ADV_PREDICT_B_PER_CELL, "u,v,w,k,omega in; u~,v~,w~,k',omega' out"),
            ("k_mac_correct", corr_ms, ADV_CORRECT_B_PER_CELL, "u,v,w and u~,v~,w~ in; u',v',w' out")):
        if len(t_ms):
            ach = bpc * ncell / (np.mean(t_ms) * 1e-3) / 1e9
            adv[name] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "us_per_launch": float(np.mean(t_ms) * 1e3),
                         "bytes_model": f"{bpc} B/cell ({what}), fp32"}
    roofline["advection"] = adv

    # end to end through the reference-facing drop-in (refbind.RefStepper):
    # the SAME steps W+1 .. W+K from the same state, held the way a reference
    # caller holds it -- float64 C-order (nx, ny, nz) numpy arrays (reference
    # grid.py:492-571); every step uploads the seven arrays, converts them to
    # the device layout, steps, converts back and downloads them
    import types
    ref = lambda t: np.ascontiguousarray(t.double().cpu().numpy().transpose(2, 1, 0))  # noqa: E731
    g = sc.grid
    host = types.SimpleNamespace(grid=types.SimpleNamespace(nx=g.nx, ny=g.ny, nz=g.nz, dx=g.dx, dy=g.dy, dz=g.dz,
                                                            origin=tuple(g.origin)),
                                 labels=ref(snap.labels_dev).astype(np.int8), time=snap.time,
                                 step_count=snap.step_count,
                                 porosity=types.SimpleNamespace(phi=ref(snap.phi_dev), lad=ref(snap.lad_dev)))
    for n in ("u", "v", "w", "p", "k", "omega", "nu_t"):
        setattr(host, n, ref(snap.fields[n]))
    state_for_cpu = snap
    stepper = RefStepper(ai_omega=sc.ai_omega)
    pre = types.SimpleNamespace(name="ai1")
    stepper.prepare(host, pre)               # buffers + operator, once per grid (untimed, like compile)
    e2e_iters = []
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_iters.append(stepper.step(host, sc.solver, None, pre, sc.inlet, None, sc.pcg_tol).pcg.iterations)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": world * ncell * args.steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": stepper.h2d_bytes // args.steps, "d2h_bytes_per_step": stepper.d2h_bytes // args.steps,
           "steps": f"{args.warmup + 1}-{args.warmup + args.steps}", "pcg_iterations": e2e_iters,
           "same_iterations_as_device_leg": e2e_iters == iters,
           "path": "refbind.RefStepper.step(state, params, psys, preconditioner, profile) on a reference-layout "
                   "float64 state (host numpy arrays, C order): per step 7 float64 arrays up, device-side layout "
                   "conversion, one device step, conversion back, 7 float64 arrays down; first call copies the "
                   "caller's pageable arrays into pinned staging, later calls reuse the pinned arrays it returned"}

    kmax = float(state.fields["k"].max())

    # N > 1: the same C3 simulation split into z-slabs over the GPUs
    zslab = None
    if dist is not None and not args.no_zslab:
        zok, zslab = zslab_leg(args, dist, rank)
        zslab["ok"] = zok

    # seconds per design evaluation (C4 recipe on the C3 city: 16 extent
    # parameters, 6 street regions), one design per GPU, voxelize + settle +
    # trailing-window region sums through optimize.evaluate_objective
    design = None
    if not args.no_design:
        from paper_2204_01117_b200 import scenes as _sc
        from paper_2204_01117_b200.optimize import evaluate_objective
        ddoc = _sc.block_city_design(256, 256, 64, 2.0, 0, 6, args.dt, settle_steps=args.settle)
        dcomp = CompiledScenario.compile(scenario_from_dict(ddoc), dtype=torch.float32)
        theta = np.array([d["initial"] for d in ddoc["design"]])
        theta[rank % len(theta)] += 0.1 * (ddoc["design"][rank % len(theta)]["hi"]
                                           - ddoc["design"][rank % len(theta)]["initial"])
        evaluate_objective(dcomp, theta)     # first call: operator + context setup
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev = evaluate_objective(dcomp, theta)
        torch.cuda.synchronize()
        t_eval = max_over_ranks(time.perf_counter() - t0)
        # the two recipes the CPU baseline times (profiles/cpu_baselines_r2.json,
        # scripts/cpu_baselines.py): channel_opt.json at its own settle 260 and
        # C4 at 96x96x24 (settle 120), initial designs
        small = {}
        # channel_opt.json as recorded with the reference goldens (tests/golden)
        chopt_doc = json.loads(str(np.load(os.path.join(ROOT, "tests", "golden", "cfg_chopt_sim_120.npz"))["doc"]))
        for tag, sc_small in (("channel_opt_settle260", scenario_from_dict(chopt_doc)),
                              ("c4_96x96x24_settle120", scenario_from_dict(
                                  _sc.block_city_design(96, 96, 24, 2.0, seed=0, nb=6, dt=0.2, settle_steps=120)))):
            c_small = CompiledScenario.compile(sc_small, dtype=torch.float32)
            th = np.array([p.initial for p in sc_small.design])
            evaluate_objective(c_small, th)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            e_small = evaluate_objective(c_small, th)
            torch.cuda.synchronize()
            small[tag] = {"seconds_per_evaluation": time.perf_counter() - t1, "loss": e_small.loss}
        # the reference's default settle of 300 steps (optimize.py:46-48), timed
        # only: the C3 city at dt 0.2 leaves the reference model's stable window
        # after ~30 steps, so no parity claim rides on it
        from paper_2204_01117_b200.optimize import ObjectiveSpec
        spec300 = ObjectiveSpec.from_scenario(dcomp.scenario)
        spec300.settle_steps = 300
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        evaluate_objective(dcomp, theta, spec300)
        torch.cuda.synchronize()
        t300 = max_over_ranks(time.perf_counter() - t1)
        design = {"seconds_per_evaluation": t_eval, "evaluations_per_hour": 3600.0 * world / t_eval,
                  "seconds_per_evaluation_settle300": t300,
                  "cpu_baseline_recipes": small,
                  "settle_steps": args.settle, "n_params": len(theta), "designs_in_parallel": world,
                  "loss": ev.loss,
                  "note": "C4 recipe (16 params, 6 regions) on the C3 city, dt %.2f; voxelize + settle steps + "
                          "trailing-window region sums (summed on the device)" % args.dt}
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        # one full oracle step (the reference's algorithm, 1 BLAS thread) from
        # the state the timed steps start at: step W+1 of the same simulation
        from oracle import citywind_oracle as co
        t0 = time.perf_counter()
        ocomp = co.Compiled(co.scene_from_dict(doc))
        setup = time.perf_counter() - t0
        ost = oracle_state_from_device(co, ocomp, state_for_cpu)
        t0 = time.perf_counter()
        orep = ocomp.step_state(ost)
        t_step = time.perf_counter() - t0
        cpu = {"value": ncell / t_step, "unit": UNIT, "cores": blas_threads(), "kind": "port",
               "sample": (f"one full C3 step (step {args.warmup + 1}, {orep.pcg.iterations} PCG iterations, "
                          f"{t_step:.1f} s) of the oracle port from the same state the timed steps start at; "
                          f"OPENBLAS_NUM_THREADS={blas_threads()}; operator setup {setup:.1f} s untimed")}
    gold = golden_iterations()
    seq = warm + iters
    golden_check = None
    if gold is not None:
        n = min(len(gold), len(seq))
        golden_check = {"reference_steps": f"1-{n}", "pcg_iterations_equal": seq[:n] == gold[:n],
                        "source": "tests/golden/cfg_c3_city_256.npz (the unmodified reference, 1 BLAS thread)"}
    cfg = bench_config(args)
    # N > 1: the headline is the design-per-GPU axis (one independent C3
    # simulation per GPU, weak scaling, no data-path collective); one C3 grid
    # split into z-slabs over the GPUs (strong scaling, NCCL halos + IPC
    # PCG barriers) is reported beside it in "zslab" -- at C3 a slab of
    # 64 / N planes leaves each GPU too few PCG units to amortise the per-phase
    # barrier and fold
    scaling, ms_step = "weak", ms_max / args.steps
    per_gpu = None
    if world > 1:
        per_gpu = {"value": value, "ms_per_step": ms_step, "scaling": "weak",
                   "note": "one independent C3 simulation per GPU (the headline)"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": cfg, "precision": "fp32 fields; PCG residual and dot products in fp64",
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clocks.summary(), "pcg_iterations": iters, "pcg_iterations_warmup": warm,
            "golden_check": golden_check, "steady": steady, "voxelize_s": voxelize_s,
            "design_eval": design, "zslab": zslab, "design_per_gpu": per_gpu, "k_max_end": kmax}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--dt", type=float, default=0.2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-design", action="store_true")
    ap.add_argument("--no-zslab", action="store_true", help="N > 1: skip the z-slab leg (design-per-GPU only)")
    ap.add_argument("--zslab-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--settle", type=int, default=120)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.zslab_child:
        zslab_child(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
