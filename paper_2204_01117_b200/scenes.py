"""Synthetic scene generators in the reference's scenario-JSON schema v1.

The reference's schema is parsed by ``citywind.scenario.scenario_from_dict``
(/root/reference/pkg/src/citywind/scenario.py:132-301); these builders emit
plain dicts in that schema so the oracle, the reference itself (when it is
importable) and this package all consume byte-identical inputs.  The recipes
follow SURVEY.md Appendix D (C1 cuboid, C2 street canyon, C3/C5 block city,
C4 16-parameter design on the block-city generator).
"""
from __future__ import annotations

import copy

import numpy as np

_NUMERICS = {"subdiv": 4, "ai_omega": 1.65, "ai_order": 1, "init": "inflow"}


def cuboid(nx: int = 64, ny: int = 64, nz: int = 32, h: float = 2.0,
           dt: float = 0.3, steps: int = 200) -> dict:
    """C1: one opaque box building in uniform 3 m/s inflow along +x."""
    return {
        "version": 1, "name": f"cuboid-{nx}x{ny}x{nz}",
        "grid": {"nx": nx, "ny": ny, "nz": nz, "dx": h, "dy": h, "dz": h},
        "boundaries": {"x_min": "inlet", "x_max": "outlet", "y_min": "outlet",
                       "y_max": "outlet", "z_min": "solid_wall", "z_max": "outlet"},
        "inlet": {"kind": "uniform", "speed": 3.0, "direction": [1, 0]},
        "solver": {"dt": dt, "turbulence": True, "turb_intensity": 0.1,
                   "u_ref": 3.0, "length_scale": 20.0},
        "objects": [{"name": "building", "kind": "building", "shape": "box",
                     "lo": [0.35 * nx * h, 0.40 * ny * h, 0.0],
                     "hi": [0.45 * nx * h, 0.60 * ny * h, 0.5 * nz * h], "phi": 0.0}],
        "run": {"steps": steps, "snapshot_every": 0},
        "numerics": dict(_NUMERICS),
    }


def canyon(nx: int = 128, ny: int = 128, nz: int = 64, h: float = 1.0,
           dt: float = 0.2, steps: int = 500, n_trees: int = 8) -> dict:
    """C2: two opaque slabs with a row of porous tree cylinders between them."""
    L, W = nx * h, ny * h
    objs = [
        {"name": "slab_s", "kind": "building", "shape": "box",
         "lo": [0.2 * L, 0.30 * W, 0.0], "hi": [0.8 * L, 0.42 * W, 18.0 * h], "phi": 0.0},
        {"name": "slab_n", "kind": "building", "shape": "box",
         "lo": [0.2 * L, 0.58 * W, 0.0], "hi": [0.8 * L, 0.70 * W, 18.0 * h], "phi": 0.0},
    ]
    for i in range(n_trees):
        objs.append({"name": f"tree{i}", "kind": "tree", "shape": "cylinder",
                     "center": [0.25 * L + 0.075 * L * i, 0.5 * W], "radius": 3.0 * h,
                     "z0": 3.0 * h, "z1": 11.0 * h, "lad": 1.0})
    return {
        "version": 1, "name": f"canyon-{nx}x{ny}x{nz}",
        "grid": {"nx": nx, "ny": ny, "nz": nz, "dx": h, "dy": h, "dz": h},
        "boundaries": {"x_min": "inlet", "x_max": "outlet", "y_min": "outlet",
                       "y_max": "outlet", "z_min": "solid_wall", "z_max": "outlet"},
        "inlet": {"kind": "logarithmic", "u_star": 0.4, "z0": 0.5, "direction": [0.8, 0.6]},
        "solver": {"dt": dt, "turbulence": True, "turb_intensity": 0.1,
                   "u_ref": 4.0, "length_scale": 20.0},
        "objects": objs,
        "run": {"steps": steps, "snapshot_every": 0},
        "numerics": dict(_NUMERICS),
    }


def block_city(nx: int = 256, ny: int = 256, nz: int = 64, h: float = 2.0,
               seed: int = 0, nb: int = 6, dt: float = 0.5, steps: int = 100,
               trees: bool = True) -> dict:
    """C3 (and C5 at 512x512x128): an nb x nb lattice of random blocks.

    RNG call order follows SURVEY.md Appendix D exactly so seed 0 at
    256x256x64 yields the survey's 52-object city (36 buildings, 16 trees).
    """
    rng = np.random.default_rng(seed)
    px = 0.7 * nx * h / nb
    py = 0.7 * ny * h / nb
    objs = []
    for i in range(nb):
        for j in range(nb):
            x0 = 0.15 * nx * h + i * px
            y0 = 0.15 * ny * h + j * py
            fx, fy = rng.uniform(0.45, 0.75, 2)
            ht = rng.uniform(8.0, 0.6 * nz * h)
            phi = float(rng.choice([0.0, 0.0, 0.0, 0.3]))
            objs.append({"name": f"b{i}_{j}", "kind": "building", "shape": "box",
                         "lo": [x0, y0, 0.0],
                         "hi": [x0 + fx * px, y0 + fy * py, float(ht)], "phi": phi})
            if rng.random() < 0.5 and trees:
                objs.append({"name": f"t{i}_{j}", "kind": "tree", "shape": "cylinder",
                             "center": [x0 + 0.9 * px, y0 + 0.9 * py],
                             "radius": 0.08 * px, "z0": 2.0, "z1": 12.0, "lad": 1.2})
    return {
        "version": 1, "name": f"block-city-{nx}x{ny}x{nz}-s{seed}",
        "grid": {"nx": nx, "ny": ny, "nz": nz, "dx": h, "dy": h, "dz": h},
        "boundaries": {"x_min": "inlet", "y_min": "inlet", "x_max": "outlet",
                       "y_max": "outlet", "z_min": "solid_wall", "z_max": "outlet"},
        "inlet": {"kind": "logarithmic", "u_star": 0.53, "z0": 0.5, "direction": [1, 1]},
        "solver": {"dt": dt, "turbulence": True, "turb_intensity": 0.1,
                   "u_ref": 5.0, "length_scale": 35.0},
        "objects": objs,
        "run": {"steps": steps, "snapshot_every": 0},
        "numerics": dict(_NUMERICS),
    }


def block_city_design(nx: int = 256, ny: int = 256, nz: int = 64, h: float = 2.0,
                      seed: int = 0, nb: int = 6, dt: float = 0.5,
                      settle_steps: int = 300) -> dict:
    """C4: block city plus 16 design parameters (extent_z of 8 blocks and
    extent_x of 8 blocks, scenario.py:394-398 bindings) and 6 objective
    regions (3 courtyards, 3 corner gaps)."""
    doc = block_city(nx, ny, nz, h, seed, nb, dt)
    blocks = [o for o in doc["objects"] if o["kind"] == "building"]
    design = []
    for n, o in enumerate(blocks[:8]):
        span = 0.25 * (o["hi"][2] - o["lo"][2])
        design.append({"name": f"h_{o['name']}", "lo": -span, "hi": span, "initial": 0.0,
                       "object": o["name"], "transform": "extent_z"})
    for n, o in enumerate(blocks[8:16]):
        span = 0.2 * (o["hi"][0] - o["lo"][0])
        design.append({"name": f"w_{o['name']}", "lo": -span, "hi": span, "initial": 0.0,
                       "object": o["name"], "transform": "extent_x"})
    Lx, Ly = nx * h, ny * h
    px, py = 0.7 * Lx / nb, 0.7 * Ly / nb
    x0, y0 = 0.15 * Lx, 0.15 * Ly
    zt = max(6.0, 3.0 * h)
    regions = []
    # pedestrian-level street slabs between block columns / rows: a block
    # covers at most 0.75 of its pitch (0.9 with the extent design range) and
    # trees start at 0.82, so [0.76, 0.81] of a pitch is open street for most
    # of the slab's length
    for r in range(3):  # streets along y, behind block column r (sheltered: heat pockets)
        c = r % nb
        regions.append({"name": f"street_y{r}",
                        "lo": [x0 + c * px + 0.76 * px, y0, 0.0],
                        "hi": [x0 + c * px + 0.81 * px + h, y0 + nb * py, zt]})
    for r in range(3):  # streets along x (wind comfort)
        c = r % nb
        regions.append({"name": f"street_x{r}",
                        "lo": [x0, y0 + c * py + 0.76 * py, 0.0],
                        "hi": [x0 + nb * px, y0 + c * py + 0.81 * py + h, zt]})
    doc["design"] = design
    doc["objective"] = {"regions": regions, "target_speed": 0.55,
                        "settle_steps": settle_steps, "avg_fraction": 0.25}
    doc["name"] = doc["name"].replace("block-city", "block-city-design")
    return doc


def channel_2d(nx: int = 24, ny: int = 16, dt: float = 0.1, speed: float = 2.0) -> dict:
    """2D walled channel (the reference tests' `channel()` helper geometry)."""
    return {
        "version": 1, "name": f"channel2d-{nx}x{ny}",
        "grid": {"nx": nx, "ny": ny, "nz": 1, "dx": 1.0, "dy": 1.0, "dz": 1.0},
        "boundaries": {"x_min": "inlet", "x_max": "outlet",
                       "y_min": "solid_wall", "y_max": "solid_wall"},
        "inlet": {"kind": "uniform", "speed": speed, "direction": [1, 0]},
        "solver": {"dt": dt, "turbulence": True, "u_ref": speed},
        "objects": [],
        "run": {"steps": 50},
        "numerics": dict(_NUMERICS),
    }


def karman(resolution: str = "desk", speed: float = 10.0) -> dict:
    """The 2-D cylinder wake of the paper's validation (the reference's
    scenarios/karman_desk.json and karman.json): a 46 mm cylinder in a
    channel, inlet at y = 0, outlet at the top, side walls, seeded initial
    perturbation 2% of the inlet speed."""
    n, h, dt, steps = ((256, 384), 0.004, 2e-4, 4000) if resolution == "desk" else ((512, 768), 0.002, 1e-4, 20000)
    return {
        "version": 1, "name": "karman-desk" if resolution == "desk" else "karman-full",
        "grid": {"nx": n[0], "ny": n[1], "nz": 1, "dx": h, "dy": h, "dz": h},
        "boundaries": {"y_min": "inlet", "y_max": "outlet", "x_min": "solid_wall", "x_max": "solid_wall"},
        "inlet": {"kind": "uniform", "speed": speed, "direction": [0, 1]},
        "solver": {"dt": dt, "nu": 1.57e-5, "turbulence": True, "turb_intensity": 0.01, "u_ref": speed,
                   "length_scale": 0.046},
        "objects": [{"name": "cylinder", "kind": "building", "shape": "cylinder", "center": [0.512, 0.384],
                     "radius": 0.023, "phi": 0.0}],
        "run": {"steps": steps, "snapshot_every": 0 if resolution == "desk" else 4000},
        "numerics": dict(_NUMERICS, perturb=0.02),
    }


def paint_rasters():
    """Raster and tree mask (ny=40, nx=48) of ``painted_city``: opaque, porous
    and noisy patches, a tree patch over a porous one (non-zero mask = tree)."""
    rng = np.random.default_rng(11)
    img = np.full((40, 48), 255, np.uint8)
    img[5:15, 6:20] = 0
    img[20:32, 10:18] = 76
    img[8:30, 28:40] = 180
    img[33:38, 2:46] = rng.integers(0, 256, (5, 44))
    mask = np.zeros_like(img)
    mask[22:30, 30:38] = 255
    mask[2:6, 40:46] = 1
    return img, mask


def write_paint_files(directory: str) -> None:
    """Write paint.pgm / trees.pgm (binary PGM, grid.py:412-416) for ``painted_city``."""
    import os
    from .grid import write_pgm
    img, mask = paint_rasters()
    write_pgm(os.path.join(directory, "paint.pgm"), img)
    write_pgm(os.path.join(directory, "trees.pgm"), mask)


def painted_city(dt: float = 0.3) -> dict:
    """48x40x16 scene on a painted base layer extruded to 9 m (grid.py:337-377)
    plus a box building crossing the paint and a tree cylinder; the rasters
    come from ``write_paint_files`` in the scenario's base directory."""
    doc = cuboid(48, 40, 16, 2.0, dt)
    doc["name"] = "paint-city-48x40x16"
    doc["paint"] = {"path": "paint.pgm", "extrude_height": 9.0, "tree_mask": "trees.pgm", "tree_lad": 0.8}
    doc["objects"] = [
        {"name": "b0", "kind": "building", "shape": "box", "lo": [30.0, 14.0, 0.0], "hi": [50.0, 30.0, 14.0],
         "phi": 0.2},
        {"name": "t0", "kind": "tree", "shape": "cylinder", "center": [70.0, 60.0], "radius": 5.0,
         "z0": 2.0, "z1": 12.0, "lad": 1.5},
    ]
    return doc


def scaled(doc: dict, **grid) -> dict:
    """Copy of ``doc`` with grid entries replaced (used to shrink scenes)."""
    out = copy.deepcopy(doc)
    out["grid"].update(grid)
    return out


CONFIGS = {
    "C1": lambda: cuboid(64, 64, 32, 2.0, 0.3, 200),
    "C2": lambda: canyon(128, 128, 64, 1.0, 0.2, 500),
    "C3": lambda: block_city(256, 256, 64, 2.0, 0, 6, 0.2),
    "C4": lambda: block_city_design(256, 256, 64, 2.0, 0, 6, 0.2),
    "C5": lambda: block_city(512, 512, 128, 2.0, 0, 6, 0.2),
}
