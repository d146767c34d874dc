"""GPU: ragged grids -- no extent a multiple of the 32x32 PCG tile, the 16-element
row pitch or the 32x8 stage block -- against the oracle: iteration counts equal,
fields within 1e-4 (fp32), and the voxelizer bit-exact against the oracle."""
import numpy as np
import pytest

from helpers import FIELDS, device_params, device_state, device_system, fields_of, oracle_compiled, rel_l2
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("shape", [(37, 29, 11), (33, 17, 5), (50, 9, 7)])
def test_ragged_grid_steps_match_oracle(shape):
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    nx, ny, nz = shape
    doc = scenes.cuboid(nx, ny, nz, 2.0, 0.3)
    comp = oracle_compiled(doc)
    labels, phi, lad = comp.voxelize_design()
    dl, dp, da = (t.cpu().numpy() for t in
                  CompiledScenario.compile(scenario_from_dict(doc)).voxelize_design_device())
    assert np.array_equal(dl, labels) and np.array_equal(dp, phi) and np.array_equal(da, lad)
    ost = comp.make_state()
    dst = device_state(ost, torch.float32)
    psys, pre = device_system(comp)
    p, prof = device_params(comp.scene)
    reps = solver.step_many(dst, p, psys, pre, prof, 12)
    want = [comp.step_state(ost).pcg.iterations for _ in range(12)]
    assert [r.pcg.iterations for r in reps] == want
    got = fields_of(dst)
    for n in FIELDS:
        assert rel_l2(got[n], getattr(ost, n)) <= 1e-4, n
