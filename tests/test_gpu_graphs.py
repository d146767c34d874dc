"""GPU: whole steps replayed as CUDA graphs (cw_step with CW_GRAPHS=1) give the
directly launched steps bit for bit -- including a batch that mixes captured
and direct steps (reports stay in step order) and the trailing-window region
sums baked into the captured step."""
import os

import numpy as np
import pytest

from helpers import FIELDS
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run(graphs, steps=8):
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    os.environ["CW_GRAPHS"] = "1" if graphs else "0"
    try:
        doc = scenes.block_city(48, 48, 16, 2.0, seed=5, nb=3, dt=0.25)
        comp = CompiledScenario.compile(scenario_from_dict(doc))
        sc = comp.scenario
        st = comp.make_state()
        reps = solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, steps // 2, sc.pcg_tol)
        reps += [solver.step(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet)]   # timed: direct launch
        lo = np.array([[10.0, 10.0, 0.0]])
        hi = np.array([[60.0, 60.0, 8.0]])
        sums = torch.zeros(1, dtype=torch.float64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        reps += solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, steps // 2 - 1, sc.pcg_tol,
                                 regions=(lo, hi, sums, cnt))
        return st, [r.pcg.iterations for r in reps], [r.cfl for r in reps], float(sums.item())
    finally:
        os.environ.pop("CW_GRAPHS", None)


def test_graph_steps_equal_direct_steps():
    a, ia, ca, sa = _run(True)
    b, ib, cb, sb = _run(False)
    assert ia == ib and ca == cb and sa == sb
    for n in FIELDS:
        assert torch.equal(a.fields[n], b.fields[n]), n
