"""GPU: the reference-facing drop-in pieces.

* refbind.RefStepper steps a REFERENCE-LAYOUT float64 state (C order,
  x slowest, grid.py:492-571) through the reference's step signature
  (solver.py:407-410) -- checked against goldens made by the unmodified
  reference;
* FlowState field views write through (reference code mutates the arrays it
  fetches, solver.py:164-167);
* project(max_iter=...) (solver.py:246-249);
* the device trailing-window region sums of evaluate_objective equal the
  host loop of the reference (optimize.py:93-99).
"""
import types

import numpy as np
import pytest

from helpers import FIELDS, golden, oracle_compiled, rel_l2
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def ref(a):
    """device / oracle x-fastest (nz, ny, nx) -> reference C order (nx, ny, nz)"""
    return np.ascontiguousarray(np.asarray(a).transpose(2, 1, 0))


def _ref_state(g, comp):
    """A reference-layout FlowState stand-in (the attributes the reference's
    step reads and reassigns) holding the golden's initial fields."""
    og = comp.scene.grid
    grid = types.SimpleNamespace(nx=og.nx, ny=og.ny, nz=og.nz, dx=og.dx, dy=og.dy, dz=og.dz,
                                 origin=tuple(og.origin))
    st = types.SimpleNamespace(grid=grid, time=0.0, step_count=0, labels=ref(g["labels"]).astype(np.int8),
                               porosity=types.SimpleNamespace(phi=ref(g["phi"]), lad=ref(g["lad"])))
    for n in FIELDS:
        setattr(st, n, ref(g[f"init_{n}"]).astype(np.float64))
    return st


@pytest.mark.parametrize("name,doc", [
    ("city_64", lambda: scenes.block_city(64, 64, 24, 2.0, seed=3, nb=3, dt=0.25)),
    ("canyon_48", lambda: scenes.canyon(48, 48, 24, 1.0, 0.2, n_trees=4)),
])
def test_refbind_steps_reference_layout_state(name, doc):
    from paper_2204_01117_b200.refbind import RefStepper
    g = golden(name)
    comp = oracle_compiled(doc())
    st = _ref_state(g, comp)
    stepper = RefStepper(ai_omega=comp.scene.ai_omega)
    pre = types.SimpleNamespace(name="ai1")            # the reference's MatrixPreconditioner duck
    its = []
    for _ in range(int(g["steps"])):
        rep = stepper.step(st, comp.scene.params, None, pre, comp.scene.inlet, None, None)
        its.append(rep.pcg.iterations)
    assert its == g["pcg_iterations"].tolist()
    assert st.step_count == int(g["steps"])
    assert abs(st.time - int(g["steps"]) * comp.scene.params.dt) < 1e-12
    for n in FIELDS:
        a = getattr(st, n)
        assert a.dtype == np.float64 and a.shape == ref(g[n]).shape
        e = rel_l2(a, ref(g[n]))
        assert e <= 1e-4, f"{n}: rel-L2 {e:.3e}"


def test_refbind_dt_zero_is_identity_and_pageable_inputs_are_copied():
    from paper_2204_01117_b200.refbind import RefStepper
    g = golden("cuboid_32")
    comp = oracle_compiled(scenes.cuboid(32, 32, 16, 2.0, 0.3))
    st = _ref_state(g, comp)
    before = {n: getattr(st, n).copy() for n in FIELDS}
    stepper = RefStepper()
    p0 = comp.scene.params
    p0.dt, dt = 0.0, p0.dt
    rep = stepper.step(st, p0, None, types.SimpleNamespace(name="ai1"), comp.scene.inlet)
    assert rep.pcg is None and st.step_count == 0
    for n in FIELDS:
        assert getattr(st, n) is not None and np.array_equal(getattr(st, n), before[n])
    p0.dt = dt
    # a caller edit of a returned (pinned) array is seen by the next step
    stepper.step(st, p0, None, types.SimpleNamespace(name="ai1"), comp.scene.inlet)
    st.k = st.k * 1.0          # a new pageable array: copied into the staging buffer
    rep = stepper.step(st, p0, None, types.SimpleNamespace(name="ai1"), comp.scene.inlet)
    assert rep.pcg.iterations == g["pcg_iterations"][1]


def test_field_views_write_through():
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    comp = CompiledScenario.compile(scenario_from_dict(scenes.cuboid(16, 12, 8, 2.0, 0.3)))
    st = comp.make_state()
    u = st.u
    assert st.u is u                                  # two reads alias, like the reference's arrays
    u *= 2.0                                          # in-place ufunc
    assert np.array_equal(st.fields["u"].cpu().numpy().transpose(2, 1, 0), u.astype(np.float32))
    st.k[1, 2, 3] = 7.5                               # item assignment through a fresh view
    assert float(st.fields["k"][3, 2, 1]) == 7.5
    sub = st.v[:, 1:-1, :]                           # a slice writes through its parent
    sub += 1.0
    assert np.allclose(st.fields["v"].cpu().numpy().transpose(2, 1, 0)[:, 1:-1, :], st.v[:, 1:-1, :])
    old = st.w
    comp.step_states(st, 1)                           # the step reassigns: the old view is detached
    snap = st.fields["w"].clone()
    old[...] = 123.0
    assert torch.equal(st.fields["w"], snap)


def test_project_max_iter():
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.errors import ProjectionError
    from helpers import device_state, device_system
    comp = oracle_compiled(scenes.cuboid(32, 32, 16, 2.0, 0.3))
    ost = comp.make_state()
    comp.step_state(ost)
    ost.u = ost.u + 0.05 * np.random.default_rng(0).standard_normal(ost.u.shape)
    dst = device_state(ost, torch.float32)
    psys, pre = device_system(comp)
    with pytest.raises(ProjectionError) as ei:
        solver.project(dst, psys, comp.scene.params.dt, pre, max_iter=5)
    assert ei.value.report.iterations == 5 and not ei.value.report.converged
    with pytest.raises(co.ProjectionError) as eo:
        co.project(ost.copy(), comp.psys, comp.scene.params.dt, comp.W, max_iter=5)
    assert eo.value.report.iterations == 5
    # the default cap is back in force afterwards
    _, rep = solver.project(dst, psys, comp.scene.params.dt, pre)
    assert rep.converged


def test_trailing_window_device_sums_equal_host_loop():
    """evaluate_objective's window sums on the device (cw_step_regions) are
    the reference's host loop `sums += region_average_speed(...)`, bit for bit."""
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.optimize import evaluate_objective
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    doc = scenes.block_city_design(48, 48, 16, 2.0, seed=5, nb=3, dt=0.25, settle_steps=12)
    sc = scenario_from_dict(doc)
    comp = CompiledScenario.compile(sc)
    theta = np.array([d["initial"] for d in doc["design"]])
    ev = evaluate_objective(comp, theta)
    regs = sc.objective.regions
    lo = np.array([r.lo for r in regs], float)
    hi = np.array([r.hi for r in regs], float)
    st = solver.make_initial_state(sc.grid, comp.voxelize_design_device(theta), None, sc.solver, sc.inlet,
                                   mode=sc.init_mode)
    window = max(1, int(round(12 * sc.objective.avg_fraction)))
    solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, 12 - window, sc.pcg_tol)
    sums = np.zeros(len(regs))
    for _ in range(window):
        solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, 1, sc.pcg_tol)
        means, _ = solver.region_average_speeds(st, lo, hi)
        sums += means
    np.testing.assert_array_equal(ev.region_speeds, sums / window)
