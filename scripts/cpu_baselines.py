"""CPU baselines of BASELINE.md section 3, timed on the UNMODIFIED reference
(citywind, imported from /root/reference/pkg/src in the build container):

* C1 cuboid 64x64x32, dt 0.3, all 200 steps;
* C2 street canyon 128x128x64, dt 0.2, first 20 steps;
  each with OPENBLAS_NUM_THREADS=1 and with one BLAS thread per core;
* design evaluations: P = core-count concurrent processes (1 BLAS thread
  each), one evaluate_objective each, on channel_opt.json (its own settle 260)
  and on the C4 recipe at 96x96x24 (settle 120).

    python scripts/cpu_baselines.py            -> profiles/cpu_baselines_r2.json

Each measurement runs in its own process (the BLAS thread count is fixed at
import).  Reference runs never write into the read-only reference tree.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "profiles", "cpu_baselines_r2.json")

CHILD = r'''
import json, os, sys, time, tempfile
sys.dont_write_bytecode = True
sys.path.insert(0, {ref!r}); sys.path.insert(0, {root!r})
os.chdir(tempfile.mkdtemp())
import numpy as np
from paper_2204_01117_b200 import scenes
from citywind.scenario import CompiledScenario, scenario_from_dict
kind, arg = sys.argv[1], sys.argv[2]
if kind == "traj":
    doc = {{"c1": lambda: scenes.cuboid(64, 64, 32, 2.0, 0.3),
           "c2": lambda: scenes.canyon(128, 128, 64, 1.0, 0.2)}}[arg]()
    steps = {{"c1": 200, "c2": 20}}[arg]
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    st = comp.make_state()
    its = []
    t0 = time.perf_counter()
    for _ in range(steps):
        its.append(comp.step_state(st).pcg.iterations)
    dt = time.perf_counter() - t0
    n = doc["grid"]["nx"] * doc["grid"]["ny"] * doc["grid"]["nz"]
    print(json.dumps({{"steps": steps, "seconds": dt, "s_per_step": dt / steps,
                      "cell_steps_per_s": n * steps / dt, "pcg_mean": float(np.mean(its))}}))
else:
    import citywind.optimize as opt
    if arg == "chopt":
        with open(os.path.join({ref!r}, "citywind", "scenarios", "channel_opt.json")) as fh:
            doc = json.load(fh)
    else:
        doc = scenes.block_city_design(96, 96, 24, 2.0, seed=0, nb=6, dt=0.2, settle_steps=120)
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    theta = np.array([p.initial for p in comp.scenario.design])
    t0 = time.perf_counter()
    ev = opt.evaluate_objective(comp, theta)
    print(json.dumps({{"seconds": time.perf_counter() - t0, "loss": ev.loss,
                      "settle": doc["objective"]["settle_steps"]}}))
'''


def run(kind, arg, threads, n_proc=1):
    env = dict(os.environ, OPENBLAS_NUM_THREADS=str(threads),
               NUMBA_CACHE_DIR=os.path.join(tempfile.gettempdir(), "numba_cache_golden"),
               PYTHONDONTWRITEBYTECODE="1")
    code = CHILD.format(ref=REF, root=ROOT)
    t0 = time.perf_counter()
    procs = [subprocess.Popen([sys.executable, "-c", code, kind, arg], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.DEVNULL, text=True) for _ in range(n_proc)]
    outs = [json.loads(p.communicate()[0].strip().splitlines()[-1]) for p in procs]
    return outs, time.perf_counter() - t0


def main():
    cores = os.cpu_count() or 1
    try:
        model = next(ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name"))
    except Exception:
        model = "unknown"
    res = {"host": {"cpu": model, "cores": cores}, "source": "unmodified reference (citywind) from /root/reference",
           "trajectories": {}, "design_evaluations": {}}
    for cfg in ("c1", "c2"):
        for thr in (1, cores):
            outs, _ = run("traj", cfg, thr)
            res["trajectories"][f"{cfg}_blas{thr}"] = outs[0]
            print(cfg, thr, outs[0], flush=True)
    for rec in ("chopt", "c4_96"):
        outs, wall = run("eval", rec, 1, cores)
        secs = [o["seconds"] for o in outs]
        res["design_evaluations"][rec] = {
            "processes": cores, "blas_threads": 1, "seconds_per_evaluation_mean": sum(secs) / len(secs),
            "wall_seconds": wall, "evaluations_per_hour": 3600.0 * cores / wall, "settle": outs[0]["settle"],
            "loss": outs[0]["loss"]}
        print(rec, res["design_evaluations"][rec], flush=True)
    with open(OUT, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
