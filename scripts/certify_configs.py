"""Certify the config goldens (SURVEY.md 8c protocol): does the REFERENCE
algorithm itself keep its per-step PCG iteration counts when its state is
perturbed at the level of float32 arithmetic (relative noise 1e-6 on the
velocity and turbulence fields after every step)?  A scene whose counts
survive is certified for exact iteration-count parity in fp32.

Runs the oracle (pinned to the reference by tests/test_oracle_golden.py) and
compares with the reference goldens (tests/golden/cfg_<name>.npz).  Results
go to tests/golden/cert_<name>.json (one file per scene, so several scenes
can be certified in parallel processes).

    python scripts/certify_configs.py NAME [NAME ...]
"""
from __future__ import annotations

import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import citywind_oracle as co  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def _scene(name):
    """(doc, steps, theta) of a config golden: from the golden when it exists,
    else from the generator table (the golden may still be running)."""
    path = os.path.join(GOLD, f"cfg_{name}.npz")
    if os.path.exists(path):
        g = np.load(path)
        return json.loads(str(g["doc"])), int(g["steps"]), (g["theta"] if g["theta"].size else None)
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    import make_golden_configs as mg
    make, steps, _, theta = mg.TRAJ[name]
    doc = make()
    th = np.array([p["initial"] for p in doc.get("design", [])]) if theta == "initial" else None
    return doc, steps, th


def certify(name, amp=1e-6, seed=0):
    doc, steps, theta = _scene(name)
    comp = co.Compiled(co.scene_from_dict(doc))
    st = comp.make_state(theta)
    rng = np.random.default_rng(seed)
    its = []
    t0 = time.perf_counter()
    for _ in range(steps):
        its.append(comp.step_state(st).pcg.iterations)
        for f in ("u", "v", "w", "k", "omega", "nu_t"):
            a = getattr(st, f)
            setattr(st, f, a * (1 + amp * rng.standard_normal(a.shape)))
    path = os.path.join(GOLD, f"cfg_{name}.npz")
    while not os.path.exists(path):   # the reference's own run may still be going
        time.sleep(30)
    time.sleep(5)
    g = np.load(path)
    gold = g["pcg_iterations"].tolist()
    off = [i + 1 for i, (a, b) in enumerate(zip(its, gold)) if a != b]
    # the field noise floor: the perturbed reference algorithm's end fields
    # against the reference's own (whole fields or the golden's subsample)
    stride = int(g["stride"])
    floor = {}
    for n in ("u", "v", "w", "p", "k", "omega", "nu_t"):
        a = np.asarray(getattr(st, n)).ravel()
        b = g[f"sub_{n}"] if stride else g[n].ravel()
        if stride:
            a = a[::stride]
        floor[n] = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    return {"steps": len(gold), "noise": amp, "mismatched_steps": off, "certified": not off,
            "field_floor_rel_l2": floor, "oracle_seconds": round(time.perf_counter() - t0, 1)}


def certify_objective(name, amp=1e-6, seed=0):
    """The objective's noise floor: the reference algorithm's loss at the
    golden's design vectors with fp32-level noise on the state after every
    step, against the reference's own losses (cfg_<name>.npz history)."""
    g = np.load(os.path.join(GOLD, f"cfg_{name}.npz"))
    doc = json.loads(str(g["doc"]))
    comp = co.Compiled(co.scene_from_dict(doc))
    rng = np.random.default_rng(seed)
    orig = co.step

    def noisy(st, *a, **k):
        rep = orig(st, *a, **k)
        for f in ("u", "v", "w", "k", "omega", "nu_t"):
            x = getattr(st, f)
            setattr(st, f, x * (1 + amp * rng.standard_normal(x.shape)))
        return rep

    co.step = noisy
    t0 = time.perf_counter()
    try:
        losses = [co.evaluate_objective(comp, th)[0] for th in g["theta_history"]]
    finally:
        co.step = orig
    gold = g["history"].tolist()
    rel = [abs(a - b) / abs(b) for a, b in zip(losses, gold)]
    return {"noise": amp, "losses": losses, "golden_losses": gold, "loss_floor_rel": rel,
            "oracle_seconds": round(time.perf_counter() - t0, 1)}


def certify_eval(name, amp=1e-6, seed=0):
    """One design evaluation's noise floor: the reference algorithm's loss and
    region speeds at the golden's design with fp32-level noise on the state
    after every step, and the per-step PCG counts, against the reference's
    own evaluate_objective (cfg_<name>.npz from make_golden_configs EVAL)."""
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    import make_golden_configs as mg
    doc = mg.EVAL[name]()
    comp = co.Compiled(co.scene_from_dict(doc))
    theta = np.array([p["initial"] for p in doc["design"]])
    rng = np.random.default_rng(seed)
    orig = co.step
    its = []

    def noisy(st, *a, **k):
        rep = orig(st, *a, **k)
        its.append(rep.pcg.iterations)
        for f in ("u", "v", "w", "k", "omega", "nu_t"):
            x = getattr(st, f)
            setattr(st, f, x * (1 + amp * rng.standard_normal(x.shape)))
        return rep

    co.step = noisy
    t0 = time.perf_counter()
    try:
        res = co.evaluate_objective(comp, theta)
    finally:
        co.step = orig
    loss, speeds = res[0], np.asarray(res[1], float)
    path = os.path.join(GOLD, f"cfg_{name}.npz")
    while not os.path.exists(path):   # the reference's own run may still be going
        time.sleep(60)
    time.sleep(5)
    g = np.load(path)
    gold_its = g["pcg_iterations"].tolist()
    moved = [i + 1 for i, (a, b) in enumerate(zip(its, gold_its)) if a != b]
    return {"noise": amp, "loss": loss, "golden_loss": float(g["loss"]),
            "loss_floor_rel": [abs(loss - float(g["loss"])) / abs(float(g["loss"]))],
            "speed_floor_rel": (np.abs(speeds - g["region_speeds"]) / np.abs(g["region_speeds"])).tolist(),
            "mismatched_steps": moved, "certified": not moved,
            "oracle_seconds": round(time.perf_counter() - t0, 1)}


def main():
    for name in sys.argv[1:]:
        if name.endswith("_eval"):
            res = certify_eval(name)
        elif name in ("chopt_opt_120", "c4_city_96"):
            res = certify_objective(name)
        else:
            res = certify(name)
        print(name, res, flush=True)
        with open(os.path.join(GOLD, f"cert_{name}.json"), "w") as fh:
            json.dump(res, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
