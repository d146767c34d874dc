"""GPU: whole steps with one k_bc_replay launch per boundary pass (the
composition of the ordered per-side write lists, cw_step.cuh
k_bc_compose_*) equal the steps that launch the ordered lists one side at a
time (CW_BC_COMPOSE=0), solver.py:330-400, bit for bit: a street canyon with
outlets on four sides, an inlet, a ground wall and porous trees, fp32 and
fp64.  tests/test_gpu_walls.py checks single passes against the oracle.
Also: a step with k / omega deferred behind the projection
(cw_step_defer_kw, refbind's upload order) equals the plain step bitwise."""
import os

import pytest

from helpers import FIELDS
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run(env, dtype, steps=10):
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        doc = scenes.canyon(48, 40, 24, 1.0, 0.2, n_trees=4)
        comp = CompiledScenario.compile(scenario_from_dict(doc), dtype=dtype)
        sc = comp.scenario
        st = comp.make_state()
        reps = solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, steps, sc.pcg_tol)
        assert st._has_drag
        return st, [r.pcg.iterations for r in reps], [r.cfl for r in reps]
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_composed_boundary_steps_equal_ordered_lists(dtype):
    dt = getattr(torch, dtype)
    a, ia, ca = _run({"CW_BC_COMPOSE": "1"}, dt)
    b, ib, cb = _run({"CW_BC_COMPOSE": "0"}, dt)
    assert ia == ib and ca == cb
    for n in FIELDS:
        assert torch.equal(a.fields[n], b.fields[n]), n


@pytest.mark.parametrize("turbulence", [True, False])
def test_deferred_k_omega_step_equals_plain_step(turbulence):
    """cw_step_defer_kw (refbind's upload order): the predictor saves the old
    cell-centred velocity, the projection runs before the upwind k / omega
    step and before the k / omega / nu_t writes of the first boundary pass --
    the same writes as the plain step, so the fields are bit-identical."""
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    doc = scenes.canyon(48, 40, 24, 1.0, 0.2, n_trees=4)
    doc["solver"]["turbulence"] = turbulence
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    sc = comp.scenario
    a = comp.make_state()
    comp.step_states(a, 3)
    b = a.copy()
    for _ in range(6):
        ev = [torch.cuda.Event() for _ in range(3)]
        for e in ev:
            e.record()
        ra = solver.step(a, sc.solver, comp.psys, comp.preconditioner, sc.inlet, pcg_tol=sc.pcg_tol, _defer=tuple(ev))
        rb = solver.step(b, sc.solver, comp.psys, comp.preconditioner, sc.inlet, pcg_tol=sc.pcg_tol)
        assert ra.pcg.iterations == rb.pcg.iterations and ra.cfl == rb.cfl
    for n in FIELDS:
        assert torch.equal(a.fields[n], b.fields[n]), n
