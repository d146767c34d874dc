"""Developer experiment (CPU): do PCG recurrence variants keep the
reference's per-step iteration counts?

The oracle's step loop runs unchanged (its own fp64 pcg_solve decides every
step); at every projection the same (A, b, W, tol, x0, res_target) is also
solved by emulations of device-precision variants, whose iteration counts
are recorded next to the reference's:

  std  the device's standard PCG: p, z, Ap, x float32; r float64; fp64 dots
  cg1  Chronopoulos-Gear single-reduction PCG (one grid barrier per
       iteration): u = W r, w = A u, s = w + beta s, r -= alpha s; same
       storage precisions (u, w, s, p, x float32; r float64)

    python scripts/dev_cg_variants.py cuboid64 200
"""
from __future__ import annotations

import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import citywind_oracle as co  # noqa: E402
from paper_2204_01117_b200 import scenes  # noqa: E402

f32 = np.float32


def _done(r, crit, tol, res_t):
    if not 0.0 <= crit < tol:
        return False
    return res_t is None or float(np.max(np.abs(r))) <= res_t


def pcg_std(A, b, W, tol, x0, res_t, max_iter=10000):
    b2 = float(b @ b)
    x = np.zeros(b.shape, f32) if x0 is None else x0.astype(f32)
    r = b - A @ x.astype(float) if x0 is not None else b.copy()
    z = (W @ r).astype(f32)
    rz = float(r @ z.astype(float))
    crit = rz / b2
    if _done(r, crit, tol, res_t):
        return 0
    p = z.copy()
    for it in range(1, max_iter + 1):
        Ap = (A @ p.astype(float)).astype(f32)
        pAp = float(p.astype(float) @ Ap.astype(float))
        alpha = rz / pAp
        x = (x + f32(alpha) * p).astype(f32)
        r = r - alpha * Ap.astype(float)
        z = (W @ r).astype(f32)
        rzn = float(r @ z.astype(float))
        crit = rzn / b2
        if _done(r, crit, tol, res_t):
            return it
        p = (z + f32(rzn / rz) * p).astype(f32)
        rz = rzn
    return -1


def pcg_cg1(A, b, W, tol, x0, res_t, max_iter=10000):
    b2 = float(b @ b)
    x = np.zeros(b.shape, f32) if x0 is None else x0.astype(f32)
    r = b - A @ x.astype(float) if x0 is not None else b.copy()
    u = (W @ r).astype(f32)
    w = (A @ u.astype(float)).astype(f32)
    g = float(r @ u.astype(float))
    dl = float(w.astype(float) @ u.astype(float))
    crit = g / b2
    if _done(r, crit, tol, res_t):
        return 0
    alpha = g / dl
    beta = 0.0
    p = np.zeros_like(u)
    s = np.zeros_like(w)
    for it in range(1, max_iter + 1):
        p = (u + f32(beta) * p).astype(f32)
        s = (w + f32(beta) * s).astype(f32)
        x = (x + f32(alpha) * p).astype(f32)
        r = r - alpha * s.astype(float)
        u = (W @ r).astype(f32)
        w = (A @ u.astype(float)).astype(f32)
        gn = float(r @ u.astype(float))
        dl = float(w.astype(float) @ u.astype(float))
        crit = gn / b2
        if _done(r, crit, tol, res_t):
            return it
        beta = gn / g
        alpha = gn / (dl - beta * gn / alpha)
        g = gn
    return -1


def pcg_cg2(A, b, W, tol, x0, res_t, max_iter=10000):
    """Standard PCG vectors (p = z + beta p, Ap = A p, r -= alpha Ap), but
    alpha from the single-reduction identity (p, Ap) = (z, Az) - beta rz / alpha_prev
    (Chronopoulos-Gear), with (z, Az) reduced in the same pass as r.z: one
    grid barrier per iteration."""
    b2 = float(b @ b)
    x = np.zeros(b.shape, f32) if x0 is None else x0.astype(f32)
    r = b - A @ x.astype(float) if x0 is not None else b.copy()
    z = (W @ r).astype(f32)
    rz = float(r @ z.astype(float))
    zaz = float(z.astype(float) @ (A @ z.astype(float)).astype(f32).astype(float))
    crit = rz / b2
    if _done(r, crit, tol, res_t):
        return 0
    p = z.copy()
    pap = zaz
    for it in range(1, max_iter + 1):
        alpha = rz / pap
        Ap = (A @ p.astype(float)).astype(f32)
        x = (x + f32(alpha) * p).astype(f32)
        r = r - alpha * Ap.astype(float)
        z = (W @ r).astype(f32)
        rzn = float(r @ z.astype(float))
        zaz = float(z.astype(float) @ (A @ z.astype(float)).astype(f32).astype(float))
        crit = rzn / b2
        if _done(r, crit, tol, res_t):
            return it
        beta = rzn / rz
        p = (z + f32(beta) * p).astype(f32)
        pap = zaz - beta * rzn / alpha
        rz = rzn
    return -1


def main():
    name = sys.argv[1]
    steps = int(sys.argv[2])
    docs = {
        "cuboid64": lambda: scenes.cuboid(64, 64, 32, 2.0, 0.3),
        "cuboid32": lambda: scenes.cuboid(32, 32, 16, 2.0, 0.3),
        "city64": lambda: scenes.block_city(64, 64, 24, 2.0, seed=3, nb=3, dt=0.25),
        "canyon128": lambda: scenes.canyon(128, 128, 64, 1.0, 0.2),
        "city256": lambda: scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2),
        "city96": lambda: scenes.block_city(96, 96, 24, 2.0, 0, 6, 0.2),
        "bielefeld": lambda: json.load(open("/root/reference/pkg/src/citywind/scenarios/bielefeld_like.json")),
    }
    comp = co.Compiled(co.scene_from_dict(docs[name]()))
    st = comp.make_state()
    rows = []
    orig = co.pcg_solve

    def hooked(A, b, W, tol, x0=None, res_inf_target=None, max_iter=10_000):
        x, rep = orig(A, b, W, tol, x0, res_inf_target, max_iter)
        rows.append((rep.iterations, pcg_std(A, b, W, tol, x0, res_inf_target),
                     pcg_cg2(A, b, W, tol, x0, res_inf_target)))
        return x, rep

    co.pcg_solve = hooked
    for s in range(steps):
        comp.step_state(st)
        ref, a, c = rows[-1]
        print(f"step {s + 1}: ref {ref} std {a} cg2 {c}", flush=True)
    arr = np.array(rows)
    print("std mismatches", int(np.sum(arr[:, 1] != arr[:, 0])), "cg2 mismatches",
          int(np.sum(arr[:, 2] != arr[:, 0])), "of", len(rows))


if __name__ == "__main__":
    main()
