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
if "--impl" in _argv and "reference" in _argv:
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
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
# PCG iterations of C3 steps 1..60 at dt 0.2 (device run; the parity gates
# hold the device's per-step counts equal to the reference's) -- used only to
# extrapolate the CPU reference's bounded samples to the same steps the B200
# arm times (steps warmup+1 .. warmup+steps)
C3_ITERS = [264, 265, 249, 231, 202, 183, 170, 147, 132, 115, 106, 100, 96, 91, 87, 85, 83, 84, 83, 84,
            83, 84, 84, 85, 84, 85, 84, 85, 84, 85, 84, 85, 84, 85, 84, 85, 84, 85, 85, 85,
            85, 86, 85, 85, 85, 86, 85, 86, 85, 86, 86, 85, 86, 85, 86, 85, 86, 86, 85, 85]


def ref_iters_per_step(warmup, steps):
    seq = C3_ITERS + [C3_ITERS[-1]] * max(0, warmup + steps - len(C3_ITERS))
    return float(np.mean(seq[warmup:warmup + steps]))


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
# CPU baseline: the oracle port on bounded samples of the C3 step

class OracleSampler:
    """Times the reference algorithm (oracle/ port, numpy+scipy CSR) on the
    full C3 grid: the non-projection stages of one step, and M PCG
    iterations (A.p, W.r, dots, axpys exactly as pcg_solve).  A full step
    is extrapolated as t_stages + t_iter * I."""

    def __init__(self, doc):
        from oracle import citywind_oracle as co
        self.co = co
        t0 = time.perf_counter()
        self.comp = co.Compiled(co.scene_from_dict(doc))
        self.state = self.comp.make_state()
        self.setup_s = time.perf_counter() - t0
        self.n = self.state.labels.size
        self.nu = self.comp.psys.n

    def stages(self):
        co, st, sc = self.co, self.state, self.comp.scene
        dt = sc.params.dt
        t0 = time.perf_counter()
        k_new = co.upwind_scalar(st, st.k, dt)
        om_new = co.upwind_scalar(st, st.omega, dt)
        st.u, st.v, st.w = co.advect_velocity(st, dt)
        st.k, st.omega = k_new, om_new
        co.diffuse(st, sc.params, dt)
        co.apply_drag(st, sc.params, dt)
        co.apply_boundary_conditions(st, sc.inlet, sc.params)
        b = -co.divergence(st)[self.comp.psys.unknown] / dt
        co.update_turbulence(st, sc.params, dt)
        co.apply_boundary_conditions(st, sc.inlet, sc.params)
        self.b = b
        return time.perf_counter() - t0

    def pcg_iters(self, m):
        A, W, b = self.comp.psys.A, self.comp.W, self.b
        x = np.zeros_like(b)
        r = b.copy()
        z = W @ r
        rz = float(r @ z)
        p = z.copy()
        t0 = time.perf_counter()
        for _ in range(m):
            Ap = A @ p
            alpha = rz / float(p @ Ap)
            x += alpha * p
            r -= alpha * Ap
            z = W @ r
            rz_new = float(r @ z)
            p = z + (rz_new / rz) * p
            rz = rz_new
        return (time.perf_counter() - t0) / m

    def sample(self, m=8, iters_per_step=None):
        ts = self.stages()
        ti = self.pcg_iters(m)
        step_s = ts + ti * (iters_per_step if iters_per_step is not None else float(np.mean(C3_ITERS[3:23])))
        return self.n / step_s, ts, ti


def cpu_threads():
    return int(os.environ.get("OPENBLAS_NUM_THREADS", "0") or 0) or (os.cpu_count() or 1)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    doc = c3_doc(args.dt)
    smp = OracleSampler(doc)
    ips = ref_iters_per_step(args.warmup, args.steps)
    for _ in range(args.warmup):
        smp.sample(4, ips)
    vals, tstage, titer = [], [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, ts, ti = smp.sample(4, ips)
        vals.append(v)
        tstage.append(ts)
        titer.append(ti)
    wall = time.perf_counter() - t0
    value = float(np.mean(vals))
    cores = cpu_threads()
    sample = (f"per step: the C3 step's non-projection stages on the full 256x256x64 grid "
              f"(mean {np.mean(tstage):.2f} s) + 4 PCG iterations (mean {np.mean(titer):.3f} s/iteration), "
              f"extrapolated to {ips:.1f} iterations/step (the mean of C3 steps {args.warmup + 1}-"
              f"{args.warmup + args.steps}, the steps the B200 arm times); oracle/ numpy+scipy port, "
              f"OpenBLAS ddot on {cores} threads, CSR matvec single-threaded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * doc_cells(doc) / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "C3 block city 256x256x64, seed 0, 52 objects",
                                            "dt": args.dt},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


def doc_cells(doc):
    g = doc["grid"]
    return g["nx"] * g["ny"] * g["nz"]


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
    sol = DistSlabSolver(state, sc.solver, sc.inlet, omega=sc.ai_omega, pcg_tol=sc.pcg_tol)
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
            "planes_per_slab": [w.k_hi - w.k_lo for w in sol.windows], "halo": DEFAULT_HALO,
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
        out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
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

    doc = c3_doc(args.dt)
    ncell = doc_cells(doc)
    sc = scenario_from_dict(doc)
    comp = CompiledScenario.compile(sc, dtype=torch.float32)
    t0 = time.perf_counter()
    state = comp.make_state()
    torch.cuda.synchronize()
    voxelize_s = time.perf_counter() - t0
    nu = comp.psys.n

    # warm-up (untimed)
    comp.step_states(state, args.warmup)
    lib = N.lib()
    ctx = solver._acquire(comp.psys, comp.preconditioner, state)
    comp.psys.pool.release(ctx)
    N.check(lib.cw_pcg_timing(ctx.h, args.steps))
    lib.cw_launch_count(ctx.h, 1)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ev0.record()
        solver.step_many(state, sc.solver, comp.psys, comp.preconditioner, sc.inlet, args.steps,
                         sc.pcg_tol, read_back=False)
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = int(lib.cw_launch_count(ctx.h, 1))
    reps = solver.finish(state, comp.psys, comp.preconditioner, args.steps)
    iters = [r.pcg.iterations for r in reps]
    pcg_ms = (C.c_float * args.steps)()
    got = C.c_int()
    N.check(lib.cw_read_pcg_timing(ctx.h, pcg_ms, args.steps, C.byref(got)))
    pcg_ms = np.array(pcg_ms[:got.value], float)
    pred_ms, corr_ms = (C.c_float * args.steps)(), (C.c_float * args.steps)()
    got_a = C.c_int()
    N.check(lib.cw_read_adv_timing(ctx.h, pred_ms, corr_ms, args.steps, C.byref(got_a)))
    pred_ms = np.array(pred_ms[:got_a.value], float)
    corr_ms = np.array(corr_ms[:got_a.value], float)
    ms_max = ms
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = world * ncell * args.steps / (ms_max * 1e-3)

    # roofline of the dominant kernel (k_pcg)
    peak, peak_kind = hbm_peak()
    bytes_per_launch = [20.0 * ncell + 8.0 * nu + PCG_B_PER_UNKNOWN_ITER * i * nu for i in iters[:len(pcg_ms)]]
    achieved = float(np.sum(bytes_per_launch) / (np.sum(pcg_ms) * 1e-3) / 1e9) if len(pcg_ms) else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "pcg_dram_bytes.json")
    if os.path.exists(prof) and bytes_per_launch:
        # measured DRAM bytes of one captured launch, scaled by the ratio to
        # its algorithmic bytes onto this run's mean launch
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
    # the advection kernels (MacCormack predictor with the k/omega upwind, corrector)
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

    # end to end through the reference-facing API: host state in, host state out
    names = ("u", "v", "w", "p", "k", "omega", "nu_t")
    host = {n: torch.empty(state.fields[n].shape, dtype=state.fields[n].dtype, pin_memory=True) for n in names}
    for n in names:
        host[n].copy_(state.fields[n])
    k_e2e = max(1, min(args.steps, 5))
    stepper = solver.HostStepper(state, host)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    e2e_iters = []
    for _ in range(k_e2e):
        e2e_iters.append(stepper.step(sc.solver, comp.psys, comp.preconditioner, sc.inlet,
                                      pcg_tol=sc.pcg_tol).pcg.iterations)
    stepper.synchronize()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    xfer = sum(int(host[n].numel() * host[n].element_size()) for n in names)
    e2e = {"value": world * ncell * k_e2e / e2e_s, "unit": UNIT, "h2d_bytes_per_step": xfer,
           "d2h_bytes_per_step": xfer, "steps": k_e2e, "pcg_iterations": e2e_iters,
           "path": "solver.HostStepper.step() on a host-resident state: every step uploads the 7 fields from "
                   "pinned host memory, steps, and downloads the 7 fields; the two copy directions overlap "
                   "field by field across consecutive steps, and nu_t and p upload while the advection runs"}

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
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev = evaluate_objective(dcomp, theta)
        torch.cuda.synchronize()
        t_eval = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([t_eval], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_eval = float(t.item())
        design = {"seconds_per_evaluation": t_eval, "evaluations_per_hour": 3600.0 * world / t_eval,
                  "settle_steps": args.settle, "n_params": len(theta), "designs_in_parallel": world,
                  "loss": ev.loss,
                  "note": "C4 recipe (16 params, 6 regions) on the C3 city; settle kept inside the "
                          "reference model's stable window at dt 0.2"}
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        smp = OracleSampler(doc)
        v, ts, ti = smp.sample(4)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": (f"oracle/ numpy+scipy port on the full C3 grid: non-projection stages of one step "
                          f"({ts:.2f} s) + 4 PCG iterations ({ti:.3f} s each), extrapolated to "
                          f"{np.mean(iters):.1f} iterations/step (this run's mean); setup {smp.setup_s:.1f} s")}
        cpu["value"] = smp.n / (ts + ti * float(np.mean(iters)))
    scaling, parallelism, ms_step = "weak", f"design-per-GPU x{world}", ms_max / args.steps
    per_gpu = None
    if zslab is not None and zslab.get("ok"):
        # headline at N > 1: one grid z-slab sharded over the GPUs (strong
        # scaling); the independent-design throughput is kept beside it
        per_gpu = {"value": value, "ms_per_step": ms_step, "scaling": "weak",
                   "note": "one independent C3 simulation per GPU"}
        value, ms_step = zslab["value"], zslab["ms_per_step"]
        scaling, parallelism = "strong", f"z-slab x{world}"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C3 block city 256x256x64, seed 0, 36 buildings + 16 trees, dt %.2f" % args.dt,
                       "cells": ncell, "unknowns": nu, "parallelism": parallelism,
                       "l2": "inputs larger than L2: ~250 MB state+workspace per step > 126 MB L2",
                       "precision": "fp32 fields; PCG residual and dot products in fp64"},
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clocks.summary(), "pcg_iterations": iters, "voxelize_s": voxelize_s,
            "design_eval": design, "zslab": zslab, "design_per_gpu": per_gpu,
            "k_max_end": kmax}
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
