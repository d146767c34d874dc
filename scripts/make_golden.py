"""Generate golden fixtures by running the UNMODIFIED reference (citywind).

Run here (the reference is importable only in the build container):
    python scripts/make_golden.py [--only NAME]
Writes tests/golden/<name>.npz.  Arrays are stored x-fastest, shaped
(nz, ny, nx[+1]), i.e. in the device/oracle layout.  Reference runs use
OPENBLAS_NUM_THREADS=1 (SURVEY.md 8c protocol) and never write into the
read-only reference tree (bytecode and numba caches are redirected).
"""
from __future__ import annotations

import argparse
import hashlib
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


def xf(a):
    return np.ascontiguousarray(np.asarray(a).transpose(2, 1, 0))


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# name -> (scene dict, steps, store full voxel arrays?)
SCENES = {
    "cuboid_32": (scenes.cuboid(32, 32, 16, 2.0, 0.3), 40),
    "canyon_48": (scenes.canyon(48, 48, 24, 1.0, 0.2, n_trees=4), 25),
    "city_64": (scenes.block_city(64, 64, 24, 2.0, seed=3, nb=3, dt=0.25), 30),
    "channel2d": (scenes.channel_2d(24, 16, 0.1, 2.0), 60),
    "paint_city_48": (scenes.painted_city(), 15),
}
VOXEL_ONLY = {
    "vox_canyon_128": scenes.canyon(128, 128, 64, 1.0, 0.2),
    "vox_city_256": scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.5),
}


def run_scene(name, doc, steps):
    from citywind.scenario import CompiledScenario, scenario_from_dict

    sc = scenario_from_dict(doc, base_dir=".")
    t0 = time.perf_counter()
    comp = CompiledScenario.compile(sc)
    labels, poros = comp.voxelize_design()
    st = comp.make_state()
    init = {f"init_{n}": xf(getattr(st, n)) for n in ("u", "v", "w", "p", "k", "omega", "nu_t")}
    iters, conv, crit, cfl, dvb, dva = [], [], [], [], [], []
    for _ in range(steps):
        rep = comp.step_state(st)
        iters.append(rep.pcg.iterations)
        conv.append(rep.pcg.converged)
        crit.append(rep.pcg.criterion)
        cfl.append(rep.cfl)
        dvb.append(rep.div_before)
        dva.append(rep.div_after)
    W = comp.preconditioner.W
    out = dict(init)
    out.update({n: xf(getattr(st, n)) for n in ("u", "v", "w", "p", "k", "omega", "nu_t")})
    out.update(labels=xf(labels), phi=xf(poros.phi), lad=xf(poros.lad),
               index=xf(comp.psys.index), pcg_iterations=np.array(iters),
               pcg_converged=np.array(conv), pcg_criterion=np.array(crit),
               cfl=np.array(cfl), div_before=np.array(dvb), div_after=np.array(dva),
               w_diag_mean=np.array(float(np.mean(W.diagonal()))),
               a_nnz=np.array(comp.psys.A.nnz), w_nnz=np.array(W.nnz),
               steps=np.array(steps))
    if doc.get("paint"):
        img, mask = scenes.paint_rasters()
        out.update(paint_image=img, paint_mask=mask)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"{name}: {steps} steps in {time.perf_counter() - t0:.1f}s, iters={iters}")


def voxel_only(name, doc):
    from citywind.scenario import CompiledScenario, scenario_from_dict
    import citywind.grid as cg

    calls = {"n": 0}
    orig = cg.points_in_mesh

    def counting(pts, mesh, *a, **k):
        calls["n"] += 1
        return orig(pts, mesh, *a, **k)

    cg.points_in_mesh = counting
    try:
        sc = scenario_from_dict(doc, base_dir=".")
        comp = CompiledScenario.compile(sc)
        t0 = time.perf_counter()
        labels, poros = comp.voxelize_design()
        dt = time.perf_counter() - t0
    finally:
        cg.points_in_mesh = orig
    lab, phi, lad = xf(labels), xf(poros.phi), xf(poros.lad)
    cut = np.nonzero((phi < 1.0) | (lad > 0))
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        labels_sha=np.array(digest(lab)), phi_sha=np.array(digest(phi)),
        lad_sha=np.array(digest(lad)), index_sha=np.array(digest(xf(comp.psys.index))),
        cut_idx=np.stack(cut).astype(np.int32), cut_phi=phi[cut], cut_lad=lad[cut],
        label_counts=np.bincount(lab.ravel(), minlength=6),
        fallback_calls=np.array(calls["n"]), voxelize_seconds=np.array(dt))
    print(f"{name}: voxelized in {dt:.2f}s, fallback calls {calls['n']}, cut cells {len(cut[0])}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    cwd = tempfile.mkdtemp()
    os.chdir(cwd)
    scenes.write_paint_files(cwd)
    for name, (doc, steps) in SCENES.items():
        if a.only in (None, name):
            run_scene(name, doc, steps)
    for name, doc in VOXEL_ONLY.items():
        if a.only in (None, name):
            voxel_only(name, doc)


if __name__ == "__main__":
    main()
