"""Pin the CPU oracle against fixtures produced by the unmodified reference
(scripts/make_golden.py).  CPU-only: no GPU, no product code on the compute
path -- this is what makes the oracle trustworthy as the parity checker."""
import hashlib
import os

import numpy as np
import pytest

from oracle import citywind_oracle as co
from oracle import voxel_oracle as vo
from paper_2204_01117_b200 import scenes
from helpers import golden, oracle_compiled

GOLD = os.path.join(os.path.dirname(__file__), "golden")

STEP_SCENES = {
    "cuboid_32": lambda: scenes.cuboid(32, 32, 16, 2.0, 0.3),
    "canyon_48": lambda: scenes.canyon(48, 48, 24, 1.0, 0.2, n_trees=4),
    "city_64": lambda: scenes.block_city(64, 64, 24, 2.0, seed=3, nb=3, dt=0.25),
    "channel2d": lambda: scenes.channel_2d(24, 16, 0.1, 2.0),
    "paint_city_48": scenes.painted_city,
}


@pytest.fixture(scope="module")
def base_dir(tmp_path_factory):
    """Rasters of the painted scene, as the golden script wrote them."""
    d = tmp_path_factory.mktemp("paint")
    scenes.write_paint_files(str(d))
    return str(d)


def test_paint_rasters_match_fixture(base_dir):
    g = load("paint_city_48")
    img = vo.read_raster(os.path.join(base_dir, "paint.pgm"))
    mask = vo.read_raster(os.path.join(base_dir, "trees.pgm"))
    assert np.array_equal(img, g["paint_image"]) and np.array_equal(mask, g["paint_mask"])
    assert (g["labels"] == 1).sum() > 0 and ((g["phi"] > 0) & (g["phi"] < 1)).sum() > 0


def load(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def rel_l2(a, b):
    d = np.linalg.norm((np.asarray(a, float) - np.asarray(b, float)).ravel())
    n = np.linalg.norm(np.asarray(b, float).ravel())
    return d / max(n, 1e-300)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(STEP_SCENES))
def test_oracle_voxelizer_and_index_bitexact(name, base_dir):
    g = load(name)
    comp = co.Compiled(co.scene_from_dict(STEP_SCENES[name](), base_dir))
    labels, phi, lad = comp.voxelize_design()
    assert np.array_equal(labels, g["labels"])
    assert np.array_equal(phi, g["phi"])
    assert np.array_equal(lad, g["lad"])
    assert np.array_equal(comp.psys.index, g["index"])
    assert comp.psys.A.nnz == int(g["a_nnz"]) and comp.W.nnz == int(g["w_nnz"])
    assert float(np.mean(comp.W.diagonal())) == float(g["w_diag_mean"])


@pytest.mark.parametrize("name", sorted(STEP_SCENES))
def test_oracle_steps_match_reference(name, base_dir):
    g = load(name)
    comp = co.Compiled(co.scene_from_dict(STEP_SCENES[name](), base_dir))
    st = comp.make_state()
    for f in ("u", "v", "w", "p", "k", "omega", "nu_t"):
        assert np.array_equal(getattr(st, f), g[f"init_{f}"]), f
    iters = []
    for _ in range(int(g["steps"])):
        rep = comp.step_state(st)
        iters.append(rep.pcg.iterations)
    assert iters == g["pcg_iterations"].tolist()
    for f in ("u", "v", "w", "p", "k", "omega", "nu_t"):
        assert rel_l2(getattr(st, f), g[f]) <= 1e-11, f


@pytest.mark.parametrize("name", ["vox_canyon_128", "vox_city_256"])
def test_oracle_voxelizer_full_size_bitexact(name):
    g = load(name)
    doc = {"vox_canyon_128": lambda: scenes.canyon(128, 128, 64, 1.0, 0.2),
           "vox_city_256": lambda: scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.5)}[name]()
    comp = co.Compiled(co.scene_from_dict(doc))
    labels, phi, lad = comp.voxelize_design()
    cut = tuple(g["cut_idx"].astype(np.int64))
    assert np.array_equal(phi[cut], g["cut_phi"])
    assert np.array_equal(lad[cut], g["cut_lad"])
    assert sha(labels) == str(g["labels_sha"])
    assert sha(phi) == str(g["phi_sha"])
    assert sha(lad) == str(g["lad_sha"])
    assert sha(comp.psys.index) == str(g["index_sha"])


@pytest.mark.parametrize("name,steps", [("c1_cuboid_64", 15), ("chopt_sim_120", 15), ("bielefeld_120", 4)])
def test_oracle_matches_config_golden_prefix(name, steps):
    """The oracle against the reference's config goldens
    (scripts/make_golden_configs.py): the first steps' PCG counts and per-step
    field L2 norms."""
    import json
    g = golden(f"cfg_{name}")
    comp = oracle_compiled(json.loads(str(g["doc"])))
    theta = g["theta"] if g["theta"].size else None
    st = comp.make_state(theta)
    for s in range(steps):
        assert comp.step_state(st).pcg.iterations == g["pcg_iterations"][s]
        for n in ("u", "v", "w", "p", "k", "omega", "nu_t"):
            a = float(np.linalg.norm(getattr(st, n)))
            assert abs(a - g[f"norm_{n}"][s]) <= 1e-11 * abs(g[f"norm_{n}"][s]), (s, n)
