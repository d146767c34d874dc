"""Host post-processing of the appendix validations (validate.py:32-67):
the Strouhal relation and the FFT peak estimate, on known answers."""
import numpy as np
import pytest

from paper_2204_01117_b200 import scenes
from paper_2204_01117_b200.validate import shedding_frequency, strouhal_theory


def test_strouhal_theory():
    re, st, f = strouhal_theory(10.0)
    assert re == pytest.approx(10.0 * 0.046 / 1.57e-5)
    assert st == pytest.approx(0.198 * (1 - 19.7 / re))
    assert f == pytest.approx(st * 10.0 / 0.046)


@pytest.mark.parametrize("f0", [20.0, 43.0, 120.5])
def test_shedding_frequency_of_a_noisy_sinusoid(f0):
    dt = 3.6e-4
    t = np.arange(4000) * dt
    rng = np.random.default_rng(0)
    s = 0.3 * np.sin(2 * np.pi * f0 * t + 0.4) + 0.02 * rng.standard_normal(t.size) + 1.5
    f, quality = shedding_frequency(s, dt)
    assert f == pytest.approx(f0, rel=5e-3) and quality > 5.0
    assert shedding_frequency(s[:20], dt) == (0.0, 0.0)      # too short after halving


def test_karman_scene_is_the_reference_fixture():
    d = scenes.karman("desk")
    assert d["grid"] == {"nx": 256, "ny": 384, "nz": 1, "dx": 0.004, "dy": 0.004, "dz": 0.004}
    assert d["numerics"]["perturb"] == 0.02 and d["objects"][0]["radius"] == 0.023
    assert scenes.karman("full")["run"] == {"steps": 20000, "snapshot_every": 4000}
