"""GPU: velocity probes and streamlines on the device
against the oracle's restatement of Advector.velocity_at (advection.py:49-111)
and trace_streamlines (solver.py:488-532) on the same state values."""
import numpy as np
import pytest

from helpers import device_state, oracle_compiled, round_state
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def states():
    """A stepped oracle state, rounded to fp32, and its device copy."""
    from oracle import citywind_oracle as co
    comp = oracle_compiled(scenes.canyon(48, 48, 24, 1.0, 0.2, n_trees=4))
    ost = comp.make_state()
    for _ in range(5):
        comp.step_state(ost)
    round_state(ost, np.float32)
    return co, ost, device_state(ost, torch.float32)


def test_probe_velocities_match_oracle(states):
    from paper_2204_01117_b200.solver import probe_velocities, probe_velocity
    co, ost, dst = states
    rng = np.random.default_rng(4)
    g = dst.grid
    pts = rng.uniform([-2.0, -2.0, -1.0], [g.nx * g.dx + 2, g.ny * g.dy + 2, g.nz * g.dz + 1], (200, 3))
    got = probe_velocities(dst, pts).cpu().numpy()
    c = (pts - np.asarray(g.origin)) / np.array([g.dx, g.dy, g.dz])
    want = np.stack(co.velocity_at(ost, c[:, 0], c[:, 1], c[:, 2]), axis=1)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-14)
    assert np.allclose(probe_velocity(dst, pts[3]), want[3], rtol=1e-12, atol=1e-14)


def test_streamlines_match_oracle(states):
    from paper_2204_01117_b200.solver import trace_streamlines
    co, ost, dst = states
    seeds = [[2.0, 10.0, 5.0], [5.0, 30.0, 8.0], [1.0, 24.0, 14.0], [-5.0, 0.0, 0.0], [20.0, 20.0, 1.5]]
    got = trace_streamlines(dst, seeds, 0.5, max_steps=300)
    want = co.trace_streamlines(ost, seeds, 0.5, max_steps=300)
    assert len(got) == len(want)
    assert got[3].shape == (0, 3) and want[3].shape == (0, 3)
    for a, b in zip(got, want):
        n = min(len(a), len(b))
        assert abs(len(a) - len(b)) <= 1, (len(a), len(b))
        if n:
            np.testing.assert_allclose(a[:n], b[:n], rtol=1e-9, atol=1e-9)
    assert max(len(a) for a in got) > 20


def test_run_simulation_probes_on_device():
    """run_simulation(probes=...) records one sample per step without a host
    sync per step; the last row equals a probe of the final state."""
    from paper_2204_01117_b200.scenario import run_simulation, scenario_from_dict
    from paper_2204_01117_b200.solver import probe_velocity
    pts = [(20.0, 30.0, 6.0), (40.0, 12.0, 3.0)]
    out = run_simulation(scenario_from_dict(scenes.cuboid(32, 32, 16, 2.0, 0.3)), steps=6, probes=pts)
    assert len(out["probes"]) == 2 and out["probes"][0].shape == (6, 3)
    for pi, p in enumerate(pts):
        assert np.allclose(out["probes"][pi][-1], probe_velocity(out["state"], p), rtol=0, atol=0)
    assert len(out["pcg_iterations"]) == 6


def test_probed_run_longer_than_the_report_ring():
    """run_simulation with probes enqueues steps without reading their reports;
    a run longer than the device's report ring (4096) is read in batches."""
    from paper_2204_01117_b200 import scenes
    from paper_2204_01117_b200.scenario import run_simulation, scenario_from_dict
    sc = scenario_from_dict(scenes.channel_2d(24, 16, 0.05, 1.0))
    out = run_simulation(sc, steps=4200, snapshot_every=0, probes=[(10.0, 8.0, 0.5)])
    assert out["probes"][0].shape == (4200, 3) and len(out["pcg_iterations"]) == 4200
    assert abs(out["time"] - 4200 * 0.05) < 1e-9
