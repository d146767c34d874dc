"""Golden fixtures on BASELINE.json's configs and the reference's bundled
scenes, made by running the UNMODIFIED reference (citywind) here.

    python scripts/make_golden_configs.py --only NAME     (one fixture per process)

Fixtures (tests/golden/cfg_<name>.npz; arrays x-fastest, (nz, ny, nx[+1])):

* trajectories -- per-step PCG iterations / converged / criterion, cfl,
  div_before, div_after, per-field L2 norms, k and nu_t maxima; the end
  fields in float32, either whole or as a fixed stride subsample (``sub_*``,
  every STRIDE-th element of the flattened x-fastest array) plus the
  float64 field's SHA-256:
    c1_cuboid_64    C1 64x64x32 cuboid, dt 0.3, 200 steps (whole fields)
    c2_canyon_128   C2 128x128x64 canyon, dt 0.2, 20 steps (stride 16)
    c2_canyon_128_500  the same over BASELINE.json's full 500 steps
    c3_city_256     C3 256x256x64 block city, dt 0.2, 25 steps (stride 64) --
                    the bench scene and horizon (bench.py times steps 6-25)
    bielefeld_120   src/scenarios/bielefeld_like.json, 120 steps (stride 4)
    chopt_sim_120   src/scenarios/channel_opt.json, initial design (its
                    translate_x / translate_y bindings applied), 120 steps
* optimizer runs through the reference's own optimize.py:
    chopt_opt_120   channel_opt.json with settle_steps 120 (inside the
                    scene's stable window): gradient_descent
                    max_iter 2 (eps 0.1, lam 1), every FD gradient recorded
    c4_city_96      C4 recipe (16 extent parameters, 6 regions) at 96x96x24,
                    dt 0.2, settle 120: gradient_descent max_iter 1
* one evaluate_objective of the C4 recipe at 256x256x64 (c4_city_256_eval):
  loss, region speeds and the per-step PCG counts at the initial design

Reference runs use OPENBLAS_NUM_THREADS=1 and never write into
the read-only reference tree.
"""
from __future__ import annotations

import argparse
import copy
import hashlib
import json
import os
import sys
import tempfile
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_cache_golden"))
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2204_01117_b200 import scenes  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
FIELDS = ("u", "v", "w", "p", "k", "omega", "nu_t")
BUNDLED = os.path.join(REF, "citywind", "scenarios")


def xf(a):
    return np.ascontiguousarray(np.asarray(a).transpose(2, 1, 0))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def bundled(name):
    with open(os.path.join(BUNDLED, name)) as fh:
        return json.load(fh)


def chopt(settle=None):
    doc = bundled("channel_opt.json")
    if settle is not None:
        doc = copy.deepcopy(doc)
        doc["objective"]["settle_steps"] = settle
    return doc


def c4_96():
    return scenes.block_city_design(96, 96, 24, 2.0, seed=0, nb=6, dt=0.2, settle_steps=120)


# name -> (doc factory, steps, stride (0 = whole fields), theta: "initial" or None)
TRAJ = {
    "c1_cuboid_64": (lambda: scenes.cuboid(64, 64, 32, 2.0, 0.3), 200, 0, None),
    "c2_canyon_128": (lambda: scenes.canyon(128, 128, 64, 1.0, 0.2), 20, 16, None),
    "c2_canyon_128_500": (lambda: scenes.canyon(128, 128, 64, 1.0, 0.2), 500, 16, None),
    "c3_city_256": (lambda: scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2), 25, 64, None),
    "bielefeld_120": (lambda: bundled("bielefeld_like.json"), 120, 4, None),
    "chopt_sim_120": (lambda: chopt(), 120, 0, "initial"),
}
OPT = {
    "chopt_opt_120": (lambda: chopt(120), 2),
    "c4_city_96": (c4_96, 1),
}
# one design evaluation through the reference's own optimize.evaluate_objective
# at the initial design (per-step PCG counts recorded):
#   c4_city_256_eval  the C4 recipe at BASELINE.json's 256x256x64 (bench.py's
#                     design_eval scene), settle 120
EVAL = {
    "c4_city_256_eval": lambda: scenes.block_city_design(256, 256, 64, 2.0, 0, 6, 0.2, settle_steps=120),
}


def run_traj(name):
    from citywind.scenario import CompiledScenario, scenario_from_dict
    make, steps, stride, theta = TRAJ[name]
    doc = make()
    sc = scenario_from_dict(doc, base_dir=".")
    t0 = time.perf_counter()
    comp = CompiledScenario.compile(sc)
    th = None
    if theta == "initial":
        th = np.array([p.initial for p in sc.design])
    st = comp.make_state(th)
    rec = {k: [] for k in ("pcg_iterations", "pcg_converged", "pcg_criterion", "cfl", "div_before",
                           "div_after", "k_max", "nut_max", "step_seconds")}
    norms = {n: [] for n in FIELDS}
    for s in range(steps):
        ts = time.perf_counter()
        rep = comp.step_state(st)
        rec["step_seconds"].append(time.perf_counter() - ts)
        rec["pcg_iterations"].append(rep.pcg.iterations)
        rec["pcg_converged"].append(rep.pcg.converged)
        rec["pcg_criterion"].append(rep.pcg.criterion)
        rec["cfl"].append(rep.cfl)
        rec["div_before"].append(rep.div_before)
        rec["div_after"].append(rep.div_after)
        rec["k_max"].append(float(st.k.max()))
        rec["nut_max"].append(float(st.nu_t.max()))
        for n in FIELDS:
            norms[n].append(float(np.linalg.norm(getattr(st, n))))
        print(f"{name} step {s + 1}: it={rep.pcg.iterations} {rec['step_seconds'][-1]:.1f}s "
              f"kmax={rec['k_max'][-1]:.3g}", flush=True)
    out = {k: np.array(v) for k, v in rec.items()}
    out.update({f"norm_{n}": np.array(v) for n, v in norms.items()})
    for n in FIELDS:
        a = xf(getattr(st, n))
        out[f"sha_{n}"] = np.array(sha(a))
        out[f"shape_{n}"] = np.array(a.shape)
        if stride:
            out[f"sub_{n}"] = a.ravel()[::stride].astype(np.float32)
        else:
            out[n] = a.astype(np.float32)
    out.update(steps=np.array(steps), stride=np.array(stride), doc=np.array(json.dumps(doc)),
               theta=np.array(th if th is not None else []),
               wall_seconds=np.array(time.perf_counter() - t0),
               blas_threads=np.array(os.environ.get("OPENBLAS_NUM_THREADS", "")))
    np.savez_compressed(os.path.join(OUT, f"cfg_{name}.npz"), **out)
    print(f"{name}: {steps} steps in {time.perf_counter() - t0:.1f}s, iters={rec['pcg_iterations']}")


def run_opt(name):
    import citywind.optimize as opt
    from citywind.scenario import CompiledScenario, scenario_from_dict
    make, max_iter = OPT[name]
    doc = make()
    sc = scenario_from_dict(doc, base_dir=".")
    comp = CompiledScenario.compile(sc)
    grads, bases = [], []
    orig = opt.finite_diff_gradient

    def recording(*a, **k):
        g, b = orig(*a, **k)
        grads.append(np.array(g))
        bases.append(b.loss)
        return g, b

    opt.finite_diff_gradient = recording
    t0 = time.perf_counter()
    try:
        res = opt.gradient_descent(comp, max_iter=max_iter)
    finally:
        opt.finite_diff_gradient = orig
    wall = time.perf_counter() - t0
    out = dict(doc=np.array(json.dumps(doc)), max_iter=np.array(max_iter),
               theta_history=np.array(res.theta_history), history=np.array(res.history),
               grads=np.array(grads), grad_base_loss=np.array(bases),
               region_speeds=np.array(res.region_speeds), iterations=np.array(res.iterations),
               wall_seconds=np.array(wall), workers=np.array(opt._n_workers()))
    np.savez_compressed(os.path.join(OUT, f"cfg_{name}.npz"), **out)
    print(f"{name}: {wall:.1f}s history={res.history} grads={grads} thetas={res.theta_history}")


def run_eval(name):
    import citywind.optimize as opt
    from citywind.scenario import CompiledScenario, scenario_from_dict
    doc = EVAL[name]()
    sc = scenario_from_dict(doc, base_dir=".")
    comp = CompiledScenario.compile(sc)
    theta = np.array([p.initial for p in sc.design])
    its = []
    orig = opt.step

    def recording(state, *a, **k):
        rep = orig(state, *a, **k)
        its.append(rep.pcg.iterations)
        print(f"{name} step {len(its)}: it={rep.pcg.iterations} kmax={float(state.k.max()):.3g}", flush=True)
        return rep

    opt.step = recording
    t0 = time.perf_counter()
    try:
        ev = opt.evaluate_objective(comp, theta)
    finally:
        opt.step = orig
    wall = time.perf_counter() - t0
    np.savez_compressed(os.path.join(OUT, f"cfg_{name}.npz"), doc=np.array(json.dumps(doc)), theta=theta,
                        loss=np.array(ev.loss), region_speeds=np.array(ev.region_speeds),
                        pcg_iterations=np.array(its), wall_seconds=np.array(wall))
    print(f"{name}: {wall:.1f}s loss={ev.loss} speeds={ev.region_speeds} iters={its}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", required=True, choices=sorted(TRAJ) + sorted(OPT) + sorted(EVAL))
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    os.chdir(tempfile.mkdtemp())
    if a.only in TRAJ:
        run_traj(a.only)
    elif a.only in EVAL:
        run_eval(a.only)
    else:
        run_opt(a.only)


if __name__ == "__main__":
    main()
