"""GPU: the painted-porosity base layer (decode_painted_porosity, ref
grid.py:337-377, combined with the objects, scenario.py:402-412) against the
reference's fixture: labels, phi and LAD bit for bit through the device
voxelizer, then 15 steps with identical PCG iteration counts."""
import numpy as np
import pytest

from helpers import FIELDS, fields_of, golden, rel_l2
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def compiled(tmp_path_factory):
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    d = tmp_path_factory.mktemp("paint")
    scenes.write_paint_files(str(d))
    return CompiledScenario.compile(scenario_from_dict(scenes.painted_city(), base_dir=str(d)))


def test_painted_voxelizer_bitexact(compiled):
    g = golden("paint_city_48")
    lab, phi, lad = (t.cpu().numpy() for t in compiled.voxelize_design_device())
    assert np.array_equal(lab, g["labels"])
    assert np.array_equal(phi, g["phi"])
    assert np.array_equal(lad, g["lad"])


def test_painted_steps_match_reference(compiled):
    g = golden("paint_city_48")
    st = compiled.make_state()
    for n in FIELDS:
        assert rel_l2(fields_of(st)[n], g[f"init_{n}"]) <= 1e-6, n
    reps = compiled.step_states(st, int(g["steps"]))
    assert [r.pcg.iterations for r in reps] == g["pcg_iterations"].tolist()
    got = fields_of(st)
    for n in FIELDS:
        assert rel_l2(got[n], g[n]) <= 1e-4, n


def test_host_decode_matches_device_layer(compiled):
    """grid.decode_painted_porosity (host API) equals the device base layer
    where no object covers the cell."""
    from paper_2204_01117_b200.grid import decode_painted_porosity, to_device_layout
    img, mask = scenes.paint_rasters()
    lab, por = decode_painted_porosity(img, compiled.scenario.grid, mask, 9.0, 0.8)
    g = golden("paint_city_48")
    free = (g["lad"] == to_device_layout(por.lad)) & (g["phi"] == to_device_layout(por.phi))
    assert free.mean() > 0.9
    assert np.array_equal(np.where(free, g["phi"], 0), np.where(free, to_device_layout(por.phi), 0))
