"""GPU: the reference-facing pipeline (CompiledScenario, run_simulation,
evaluate_objective, finite-difference gradients, snapshots) against the
oracle on the same scenario JSON -- device voxelizer included."""
import os

import numpy as np
import pytest

from helpers import FIELDS, fields_of, oracle_compiled, rel_l2
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _design_doc():
    doc = scenes.block_city_design(48, 48, 16, 2.0, seed=5, nb=3, dt=0.25, settle_steps=12)
    doc["design"] = doc["design"][:2]        # two parameters keep the oracle's N+1 runs short
    return doc


def test_design_regions_contain_air():
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    from paper_2204_01117_b200.solver import region_average_speeds
    doc = _design_doc()
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    st = comp.make_state()
    regs = doc["objective"]["regions"]
    _, counts = region_average_speeds(st, [r["lo"] for r in regs], [r["hi"] for r in regs])
    assert np.all(counts > 0), counts


def test_run_simulation_matches_oracle():
    from paper_2204_01117_b200.scenario import run_simulation, scenario_from_dict
    doc = scenes.cuboid(24, 24, 12, 2.0, 0.3, steps=20)
    out = run_simulation(scenario_from_dict(doc), steps=20)
    comp = oracle_compiled(doc)
    ost = comp.make_state()
    iters = [comp.step_state(ost).pcg.iterations for _ in range(20)]
    assert out["pcg_iterations"] == iters
    got = fields_of(out["state"])
    for n in FIELDS:
        assert rel_l2(got[n], getattr(ost, n)) <= 1e-4, n
    assert set(out["timings"]) >= {"advect", "project", "turbulence"}


def test_evaluate_objective_matches_oracle():
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200.optimize import evaluate_objective
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    doc = _design_doc()
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    theta = np.array([d["initial"] + 0.5 * (d["hi"] - d["initial"]) for d in doc["design"]])
    ev = evaluate_objective(comp, theta)
    oloss, ospeeds = co.evaluate_objective(oracle_compiled(doc), theta)
    assert abs(ev.loss - oloss) <= 1e-4 * abs(oloss)
    np.testing.assert_allclose(ev.region_speeds, ospeeds, rtol=1e-4)


def test_fd_gradient_matches_oracle():
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200.optimize import DesignVector, ObjectiveSpec, finite_diff_gradient
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    doc = _design_doc()
    sc = scenario_from_dict(doc)
    comp = CompiledScenario.compile(sc)
    theta = np.array([d["initial"] for d in doc["design"]])
    grad, base = finite_diff_gradient(comp, theta, ObjectiveSpec.from_scenario(sc), eps=0.5)
    oc = oracle_compiled(doc)
    design = DesignVector.from_scenario(sc)
    l0, _ = co.evaluate_objective(oc, theta)
    og = []
    for i in range(len(theta)):
        h = 0.5 if theta[i] + 0.5 <= design.hi[i] else -0.5
        t = theta.copy()
        t[i] += h
        og.append((co.evaluate_objective(oc, t)[0] - l0) / h)
    assert abs(base.loss - l0) <= 1e-4 * abs(l0)
    np.testing.assert_allclose(grad, og, rtol=2e-2, atol=1e-4 * abs(l0))


def test_snapshot_roundtrip(tmp_path):
    from paper_2204_01117_b200.io import read_snapshot, snapshot_to_state, write_snapshot
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    comp = CompiledScenario.compile(scenario_from_dict(scenes.cuboid(16, 12, 8, 2.0, 0.3)))
    st = comp.make_state()
    comp.step_states(st, 3)
    path = os.path.join(tmp_path, "s.bin")
    write_snapshot(path, st)
    snap = read_snapshot(path)
    assert snap.step == 3 and snap.arrays["u"].shape == (17, 12, 8)
    back = snapshot_to_state(snap)
    a, b = fields_of(st), fields_of(back)
    for n in FIELDS:
        np.testing.assert_array_equal(a[n], b[n])
    assert torch.equal(back.labels_dev.cpu(), st.labels_dev.cpu())


def test_snapshot_format_matches_oracle_layout(tmp_path):
    """Payload is x-fastest float32 (io.py:30-31): the reference layout
    transposed -- compare against the oracle's own field arrays."""
    from paper_2204_01117_b200.io import read_snapshot, write_snapshot
    from helpers import device_state
    comp = oracle_compiled(scenes.cuboid(16, 12, 8, 2.0, 0.3))
    ost = comp.make_state()
    path = os.path.join(tmp_path, "s.bin")
    write_snapshot(path, device_state(ost, torch.float32))
    snap = read_snapshot(path)
    for n in ("u", "v", "w", "k"):
        np.testing.assert_array_equal(snap.arrays[n], getattr(ost, n).astype(np.float32).transpose(2, 1, 0))


def test_gradient_descent_trajectory_matches_oracle():
    """optimize.gradient_descent on the device against the oracle's
    restatement (optimize.py:112-192): the same theta after two iterations
    (north_star: optimized design parameters within 1e-4)."""
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200.optimize import DesignVector, gradient_descent
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    doc = _design_doc()
    sc = scenario_from_dict(doc)
    comp = CompiledScenario.compile(sc)
    res = gradient_descent(comp, eps=0.5, max_iter=2, lam=2.0)
    design = DesignVector.from_scenario(sc)
    thetas, losses = co.gradient_descent(oracle_compiled(doc), design.values, design.lo, design.hi,
                                         lam=2.0, eps=0.5, max_iter=2)
    assert len(res.theta_history) == len(thetas) == 3
    for a, b in zip(res.theta_history, thetas):
        np.testing.assert_allclose(a, b, rtol=1e-4, atol=1e-4 * max(1.0, float(np.abs(b).max())))
    np.testing.assert_allclose(res.history, losses, rtol=1e-4)
    assert not np.allclose(thetas[0], thetas[-1])      # the design moved


def test_host_stepper_equals_device_steps():
    """HostStepper (host-resident state, overlapped upload/download per field)
    gives bit for bit the fields of the same steps on a device-resident state."""
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.grid import FIELDS as NAMES
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    comp = CompiledScenario.compile(scenario_from_dict(scenes.cuboid(24, 24, 12, 2.0, 0.3, steps=6)))
    sc = comp.scenario
    ref = comp.make_state()
    work = ref.copy()
    host = {n: torch.empty(ref.fields[n].shape, dtype=ref.fields[n].dtype, pin_memory=True) for n in NAMES}
    for n in NAMES:
        host[n].copy_(ref.fields[n])
        work.fields[n].zero_()                      # the device copy is overwritten by every upload
    stepper = solver.HostStepper(work, host)
    its = [stepper.step(sc.solver, comp.psys, comp.preconditioner, sc.inlet).pcg.iterations for _ in range(6)]
    stepper.synchronize()
    want = solver.step_many(ref, sc.solver, comp.psys, comp.preconditioner, sc.inlet, 6)
    assert its == [r.pcg.iterations for r in want]
    for n in NAMES:
        assert torch.equal(host[n], ref.fields[n].cpu()), n


def test_step_defer_waits_for_late_fields():
    """cw_step_defer: a step started before nu_t and p are on the device waits
    for their events before the first stage that uses them.  The true values
    land on a side stream only after a long sleep, the device copies hold
    poison until then, and the step still equals the ordinary step bit for bit."""
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.grid import FIELDS as NAMES
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    comp = CompiledScenario.compile(scenario_from_dict(scenes.cuboid(24, 24, 12, 2.0, 0.3, steps=6)))
    sc = comp.scenario
    ref = comp.make_state()
    solver.step_many(ref, sc.solver, comp.psys, comp.preconditioner, sc.inlet, 2)   # non-zero p, nu_t
    work = ref.copy()
    solver.step_many(ref, sc.solver, comp.psys, comp.preconditioner, sc.inlet, 1)
    true_nut, true_p = work.fields["nu_t"].clone(), work.fields["p"].clone()
    work.fields["nu_t"].fill_(1e3)
    work.fields["p"].fill_(1e3)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(40_000_000)                 # ~20 ms: the step reaches its waits first
        work.fields["nu_t"].copy_(true_nut)
        ev_nut = torch.cuda.Event()
        ev_nut.record(side)
        work.fields["p"].copy_(true_p)
        ev_p = torch.cuda.Event()
        ev_p.record(side)
    rep = solver.step(work, sc.solver, comp.psys, comp.preconditioner, sc.inlet, _defer=(ev_nut, ev_p))
    torch.cuda.synchronize()
    assert rep.pcg.iterations > 0
    for n in NAMES:
        assert torch.equal(work.fields[n], ref.fields[n]), n


def test_robustness_check_matches_oracle():
    """optimize.robustness_check (optimize.py:195-207): one evaluation per
    wind-direction offset, against the oracle's evaluate_objective with the
    rotated inlet profile."""
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200.optimize import robustness_check
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    doc = _design_doc()
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    theta = np.array([d["initial"] for d in doc["design"]])
    rows = robustness_check(comp, theta, offsets_deg=(-10.0, 0.0, 10.0))
    oc = oracle_compiled(doc)
    for row in rows:
        oloss, ospeeds = co.evaluate_objective(oc, theta, profile=oc.scene.inlet.rotated(row["offset_deg"]))
        assert abs(row["loss"] - oloss) <= 1e-4 * abs(oloss), (row, oloss)
        np.testing.assert_allclose(row["region_speeds"], ospeeds, rtol=1e-4)
