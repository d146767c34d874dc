"""GPU: the paper's appendix validations on the device path (SURVEY 8f-2,
paper_2204_01117_b200/validate.py) against the unmodified reference's
citywind.validate (tests/golden/validate_desk.json,
scripts/make_golden_validate.py):
* the 2-D cylinder wake at 10 m/s (desk resolution, 2066 steps): the shedding
  frequency of the device run (fp32) within 1% of the reference's own
  measurement and within the reference's distance of the Strouhal law + 1%;
* the porosity model against no-slip walls (phi 0.2 and 0.6 at 2 m/s, 700
  steps each): the top-outlet mean speeds of both modes within 1e-4 relative
  (absolute 1e-6 where the walls block the channel) of the reference's."""
import json
import os

import pytest

from helpers import GOLD

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _gold():
    path = os.path.join(GOLD, "validate_desk.json")
    if not os.path.exists(path):
        pytest.skip("golden not generated")
    with open(path) as fh:
        return json.load(fh)


def test_karman_shedding_frequency_matches_reference():
    from paper_2204_01117_b200 import validate
    g = _gold()["karman"][0]
    row = validate.validate_karman(speeds=(g["speed"],), resolution="desk")[0]
    assert row.steps == g["steps"]
    assert abs(row.f_theory - g["f_theory"]) <= 1e-12 * g["f_theory"]
    assert not row.flagged and not g["flagged"]
    assert abs(row.f_measured - g["f_measured"]) <= 0.01 * g["f_measured"], (row, g)
    assert row.rel_err <= g["rel_err"] + 0.01


def test_porosity_model_matches_reference():
    from paper_2204_01117_b200 import validate
    gold = _gold()["porosity"]
    rows = validate.validate_porosity(speeds=(2.0,), phis=tuple(r["phi"] for r in gold), resolution="desk")
    for row, g in zip(rows, gold):
        assert row.phi == g["phi"] and row.speed == g["speed"]
        for key in ("v_out_drag", "v_out_truth"):
            want, got = g[key], getattr(row, key)
            assert abs(got - want) <= max(1e-4 * abs(want), 1e-6), (key, row, g)
