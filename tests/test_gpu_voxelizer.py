"""Device voxelizer: bit-exact against fixtures produced by the reference
(labels, phi, LAD) -- box exact-coverage path, cylinder column casts and
the primary-direction point-cast fallback."""
import hashlib

import numpy as np
import pytest

from helpers import golden
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SMALL = {
    "cuboid_32": lambda: scenes.cuboid(32, 32, 16, 2.0, 0.3),
    "canyon_48": lambda: scenes.canyon(48, 48, 24, 1.0, 0.2, n_trees=4),
    "city_64": lambda: scenes.block_city(64, 64, 24, 2.0, seed=3, nb=3, dt=0.25),
    "channel2d": lambda: scenes.channel_2d(24, 16, 0.1, 2.0),
}
FULL = {
    "vox_canyon_128": lambda: scenes.canyon(128, 128, 64, 1.0, 0.2),
    "vox_city_256": lambda: scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.5),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _device_vox(doc):
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    lab, phi, lad = comp.voxelize_design_device()
    return comp, lab.cpu().numpy(), phi.cpu().numpy(), lad.cpu().numpy()


@pytest.mark.parametrize("name", sorted(SMALL))
def test_voxelizer_bitexact_small(name):
    g = golden(name)
    _, lab, phi, lad = _device_vox(SMALL[name]())
    assert np.array_equal(lab, g["labels"])
    assert np.array_equal(phi, g["phi"]), np.max(np.abs(phi - g["phi"]))
    assert np.array_equal(lad, g["lad"]), np.max(np.abs(lad - g["lad"]))


@pytest.mark.parametrize("name", sorted(FULL))
def test_voxelizer_bitexact_full_size(name):
    """C2 canyon (8 point-cast fallbacks) and the C3 block city (16)."""
    g = golden(name)
    comp, lab, phi, lad = _device_vox(FULL[name]())
    cut = tuple(g["cut_idx"].astype(np.int64))
    bad = np.nonzero(phi[cut] != g["cut_phi"])[0]
    assert len(bad) == 0, f"{len(bad)} cut cells differ, first {[c[bad[0]] for c in cut]}"
    assert np.array_equal(lad[cut], g["cut_lad"])
    assert sha(lab) == str(g["labels_sha"])
    assert sha(phi) == str(g["phi_sha"])
    assert sha(lad) == str(g["lad_sha"])
    assert sha(np.ascontiguousarray(comp.psys.index.transpose(2, 1, 0))) == str(g["index_sha"])


def test_design_offsets_move_objects():
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    doc = scenes.block_city_design(64, 64, 24, 2.0, seed=3, nb=3, dt=0.25, settle_steps=4)
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    lab0, phi0, _ = comp.voxelize_design_device()
    theta = np.array([d["hi"] for d in doc["design"]])
    lab1, phi1, _ = comp.voxelize_design_device(theta)
    assert float((phi1 < 1).sum()) > float((phi0 < 1).sum())   # blocks grew
