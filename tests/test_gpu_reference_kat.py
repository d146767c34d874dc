"""The reference's own known-answer tests (pkg/tests/test_solver.py,
test_turbulence.py), restated against the device API.  Each test cites the
reference test it ports."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2204_01117_b200.grid import CellLabel, FlowState, GridSpec, classify_boundary  # noqa: E402
from paper_2204_01117_b200 import solver  # noqa: E402
from paper_2204_01117_b200.linalg import build_ai_preconditioner, build_pressure_matrix  # noqa: E402
from paper_2204_01117_b200.solver import InletProfile, SolverParams  # noqa: E402

CHANNEL = {"x_min": CellLabel.INLET, "x_max": CellLabel.OUTLET,
           "y_min": CellLabel.SOLID_WALL, "y_max": CellLabel.SOLID_WALL}


def channel(nx=24, ny=16, nz=1, h=1.0):
    g = GridSpec(nx, ny, nz, h, h, h)
    f = dict(CHANNEL)
    if nz > 1:
        f["z_min"] = CellLabel.SOLID_WALL
        f["z_max"] = CellLabel.SOLID_WALL
    return g, classify_boundary(g, f)


def system(g, labels):
    psys = build_pressure_matrix(g, labels)
    return psys, build_ai_preconditioner(psys, 1.65, 1, truncate=False)


# --- drag (test_solver.py:41-78) --------------------------------------------
def test_drag_air_unchanged():
    st = FlowState.zeros(GridSpec(8, 8, 1, 1, 1, 1))
    st.u = np.full(st.u.shape, 3.0)
    solver.apply_drag(st, SolverParams(), 0.1)
    np.testing.assert_allclose(st.u, 3.0)


def test_drag_opaque_zeroes_in_one_step():
    g = GridSpec(8, 8, 1, 1, 1, 1)
    st = FlowState.zeros(g)
    st.labels = np.full(g.shape, int(CellLabel.BUILDING), np.int8)
    por = st.porosity
    por.phi[:] = 0.0
    st.porosity = por
    st.u = np.full(st.u.shape, 5.0)
    solver.apply_drag(st, SolverParams(), 0.1)
    np.testing.assert_allclose(st.u, 0.0)


def test_drag_tree_factor():
    g = GridSpec(4, 4, 1, 1, 1, 1)
    st = FlowState.zeros(g, dtype=torch.float64)
    st.labels = np.full(g.shape, int(CellLabel.TREE), np.int8)
    por = st.porosity
    por.lad[:] = 1.0
    st.porosity = por
    st.u = np.full(st.u.shape, 2.0)
    solver.apply_drag(st, SolverParams(cd_tree=0.2), 0.1)
    np.testing.assert_allclose(st.u, 1.92, rtol=1e-12)


@pytest.mark.parametrize("speed,dt,phi", [(0.0, 1.0, 0.5), (50.0, 10.0, 0.0), (3.0, 0.001, 1.0),
                                          (12.0, 0.3, 0.37)])
def test_drag_never_increases(speed, dt, phi):
    g = GridSpec(4, 4, 1, 1, 1, 1)
    st = FlowState.zeros(g)
    st.labels = np.full(g.shape, int(CellLabel.BUILDING), np.int8)
    por = st.porosity
    por.phi[:] = phi
    st.porosity = por
    st.u = np.full(st.u.shape, speed)
    solver.apply_drag(st, SolverParams(), dt)
    assert np.all(st.u <= speed + 1e-6) and np.all(st.u >= 0.0)


# --- diffusion (test_solver.py:82-112) ----------------------------------------
def test_diffuse_identity_at_zero_viscosity():
    st = FlowState.zeros(GridSpec(16, 16, 1, 1, 1, 1))
    st.nu_t = np.zeros(st.nu_t.shape)
    u0 = np.random.default_rng(0).standard_normal(st.u.shape)
    st.u = u0
    solver.diffuse(st, SolverParams(nu=0.0), 0.1)
    np.testing.assert_allclose(st.u, u0, atol=1e-6)


def test_diffuse_heat_equation_decay():
    n, L = 64, 1.0
    g = GridSpec(n, 4, 1, L / n, L / n, L / n)
    st = FlowState.zeros(g, dtype=torch.float64)
    x = np.arange(n + 1) * (L / n)
    st.u = np.sin(2 * np.pi * x / L)[:, None, None] * np.ones((n + 1, 4, 1))
    nu, dt = 1e-3, 1e-3
    for _ in range(100):
        solver.diffuse(st, SolverParams(nu=nu, dt=dt), dt)
    expected = np.exp(-nu * (2 * np.pi / L) ** 2 * 100 * dt)
    mid = st.u[:, 2, 0]
    amp = np.max(np.abs(mid[8:-8] / np.sin(2 * np.pi * x[8:-8] / L)))
    assert amp == pytest.approx(expected, rel=0.02)


# --- projection (test_solver.py:116-169) --------------------------------------
def test_divergence_free_input_unchanged():
    g, lab = channel(32, 32)
    psys, pre = system(g, lab)
    st = FlowState.zeros(g, lab)
    st.u = np.full(st.u.shape, 2.0)
    u0 = st.u
    _, rep = solver.project(st, psys, 0.1, pre)
    assert rep.iterations == 0 or np.allclose(st.p, 0, atol=1e-8)
    np.testing.assert_allclose(st.u, u0, atol=1e-6)


@pytest.mark.parametrize("shape", [(32, 32, 1), (32, 32, 16)])
def test_random_field_divergence_drops_4_orders(shape):
    g, lab = channel(*shape)
    psys, pre = system(g, lab)
    st = FlowState.zeros(g, lab)
    rng = np.random.default_rng(7)
    st.u = rng.standard_normal(st.u.shape)
    st.v = rng.standard_normal(st.v.shape)
    if shape[2] > 1:
        st.w = rng.standard_normal(st.w.shape)
    solver.apply_boundary_conditions(st, InletProfile(speed=1.0), SolverParams())
    before = solver.max_interior_divergence(st)
    solver.project(st, psys, 0.1, pre)
    assert solver.max_interior_divergence(st) <= 1e-4 * before


def test_global_mass_balance():
    g, lab = channel(24, 12)
    psys, pre = system(g, lab)
    params, prof = SolverParams(dt=0.1), InletProfile(speed=2.0)
    st = solver.make_initial_state(g, lab, None, params, prof, mode="rest", dtype=torch.float64)
    solver.apply_boundary_conditions(st, prof, params)
    solver.project(st, psys, params.dt, pre)
    u = st.u
    influx = float(np.sum(u[1, 1:-1, :])) * g.dy * g.dz
    outflux = float(np.sum(u[-2, 1:-1, :])) * g.dy * g.dz
    assert outflux == pytest.approx(influx, rel=1e-6)


# --- boundaries (test_solver.py:173-224) --------------------------------------
def test_uniform_inlet_faces():
    g, lab = channel(12, 8)
    st = FlowState.zeros(g, lab)
    solver.apply_boundary_conditions(st, InletProfile(speed=2.0), SolverParams())
    u = st.u
    np.testing.assert_allclose(u[0, :, :], 2.0)
    np.testing.assert_allclose(u[1, 1:-1, :], 2.0)


def test_outlet_copies_interior():
    g, lab = channel(12, 8)
    st = FlowState.zeros(g, lab)
    st.u = np.random.default_rng(2).standard_normal(st.u.shape)
    solver.apply_boundary_conditions(st, InletProfile(speed=1.0), SolverParams())
    u = st.u
    np.testing.assert_allclose(u[-1, :, :], u[-2, :, :])


def test_walls_zeroed_including_interior_wall_cells():
    g, lab = channel(12, 8)
    lab[6, 4, 0] = int(CellLabel.SOLID_WALL)
    st = FlowState.zeros(g, lab)
    st.u = np.ones(st.u.shape)
    st.v = np.ones(st.v.shape)
    solver.apply_boundary_conditions(st, InletProfile(speed=1.0), SolverParams())
    u, v = st.u, st.v
    np.testing.assert_allclose(v[:, 0, :], 0.0)
    np.testing.assert_allclose(v[:, 1, :], 0.0)
    np.testing.assert_allclose(v[:, -1, :], 0.0)
    assert u[6, 4, 0] == 0.0 and u[7, 4, 0] == 0.0 and v[6, 4, 0] == 0.0 and v[6, 5, 0] == 0.0


# --- step (test_solver.py:228-311) --------------------------------------------
def test_dt_zero_is_identity():
    g, lab = channel()
    psys = build_pressure_matrix(g, lab)
    params, prof = SolverParams(dt=0.0), InletProfile(speed=1.5)
    st = solver.make_initial_state(g, lab, None, params, prof)
    u0, k0 = st.u, st.k
    solver.step(st, params, psys, None, prof)
    np.testing.assert_array_equal(st.u, u0)
    np.testing.assert_array_equal(st.k, k0)


def test_empty_domain_reaches_uniform_inflow():
    g = GridSpec(24, 16, 1, 1, 1, 1)
    lab = classify_boundary(g, {"x_min": CellLabel.INLET, "x_max": CellLabel.OUTLET,
                                "y_min": CellLabel.OUTLET, "y_max": CellLabel.OUTLET})
    psys, pre = system(g, lab)
    params, prof = SolverParams(dt=0.1, u_ref=2.0), InletProfile(speed=2.0)
    st = solver.make_initial_state(g, lab, None, params, prof, mode="rest")
    solver.step_many(st, params, psys, pre, prof, 500)
    np.testing.assert_allclose(st.u[2:-2, 2:-2, :], 2.0, atol=1e-3)


def test_walled_channel_core_near_inflow():
    g, lab = channel(24, 16)
    psys, pre = system(g, lab)
    params, prof = SolverParams(dt=0.1, u_ref=2.0), InletProfile(speed=2.0)
    st = solver.make_initial_state(g, lab, None, params, prof, mode="rest")
    solver.step_many(st, params, psys, pre, prof, 500)
    np.testing.assert_allclose(st.u[2:-2, 4:-4, :], 2.0, atol=1e-2)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_divergence_reduced_every_step_and_invariants(dtype):
    """test_solver.py:273-283 (fp64: the reference's 1e-4 drop).  A float32
    field of O(2 m/s) velocities resolves divergence only to ~eps32*|u|/h,
    so the fp32 run gates on max(1e-4 * before, 100 * eps32 * |u|max / h)."""
    g, lab = channel(24, 16)
    psys, pre = system(g, lab)
    params, prof = SolverParams(dt=0.1, u_ref=2.0), InletProfile(speed=2.0)
    st = solver.make_initial_state(g, lab, None, params, prof, mode="rest", dtype=dtype)
    floor = 0.0 if dtype == torch.float64 else 100 * np.finfo(np.float32).eps * 2.5 / g.dx
    for rep in solver.step_many(st, params, psys, pre, prof, 50):
        if rep.div_before > 1e-12:
            assert rep.div_after <= max(1e-4 * rep.div_before, floor)
    st.validate()


# --- region averages (test_solver.py:357-404) ---------------------------------
def test_region_average_uniform_and_mixed():
    st = FlowState.zeros(GridSpec(10, 10, 1, 1, 1, 1))
    st.u = np.full(st.u.shape, 3.0)
    assert solver.region_average_speed(st, (2, 2, 0), (8, 8, 1)) == pytest.approx(3.0)
    st2 = FlowState.zeros(GridSpec(2, 1, 1, 1, 1, 1))
    st2.u = np.array([2.0, 2.0, 6.0]).reshape(3, 1, 1)
    assert solver.region_average_speed(st2, (0, 0, 0), (2, 1, 1)) == pytest.approx(3.0)


def test_region_average_matches_bruteforce():
    g = GridSpec(9, 7, 3, 0.5, 0.5, 0.5)
    st = FlowState.zeros(g, dtype=torch.float64)
    rng = np.random.default_rng(10)
    st.u = rng.standard_normal(st.u.shape)
    st.v = rng.standard_normal(st.v.shape)
    st.w = rng.standard_normal(st.w.shape)
    lab = np.zeros(g.shape, np.int8)
    lab[0, :, :] = int(CellLabel.SOLID_WALL)
    st.labels = lab
    lo, hi = (0.6, 0.4, 0.0), (3.4, 2.9, 1.5)
    got = solver.region_average_speed(st, lo, hi)
    u, v, w = st.u, st.v, st.w
    speeds = []
    for i in range(9):
        for j in range(7):
            for k in range(3):
                c = ((i + 0.5) * 0.5, (j + 0.5) * 0.5, (k + 0.5) * 0.5)
                if not all(lo[a] <= c[a] <= hi[a] for a in range(3)) or lab[i, j, k] != 0:
                    continue
                uu = 0.5 * (u[i, j, k] + u[i + 1, j, k])
                vv = 0.5 * (v[i, j, k] + v[i, j + 1, k])
                ww = 0.5 * (w[i, j, k] + w[i, j, k + 1])
                speeds.append(np.sqrt(uu ** 2 + vv ** 2 + ww ** 2))
    assert got == pytest.approx(np.mean(speeds), rel=1e-12)


def test_region_without_air_raises():
    g = GridSpec(4, 4, 1, 1, 1, 1)
    st = FlowState.zeros(g)
    st.labels = np.full(g.shape, int(CellLabel.BUILDING), np.int8)
    with pytest.raises(ValueError):
        solver.region_average_speed(st, (0, 0, 0), (4, 4, 1))


# --- turbulence (test_turbulence.py:31-125) ------------------------------------
def test_turbulence_positivity_at_huge_dt():
    g = GridSpec(8, 8, 4, 1, 1, 1)
    st = FlowState.zeros(g, k0=1.0, omega0=1.0)
    st.u = np.random.default_rng(1).standard_normal(st.u.shape)
    solver.update_turbulence(st, SolverParams(), 50.0)
    assert np.all(st.k > 0) and np.all(st.omega > 0) and np.all(st.nu_t >= 0)


def test_turbulence_nan_names_the_cell():
    """test_turbulence.py:118-125; the named cell is the first non-finite one
    in the reference's C order, as the oracle reports it."""
    from oracle import citywind_oracle as co
    g = GridSpec(4, 4, 1, 1, 1, 1)
    st = FlowState.zeros(g)
    k = st.k
    k[1, 2, 0] = np.inf
    st.k = k
    st.omega = np.ones(g.shape)
    st.nu_t = np.full(g.shape, 0.25)
    before = {n: np.array(getattr(st, n)) for n in ("k", "omega", "nu_t")}
    with pytest.raises(FloatingPointError, match=r"at cell \(\d+, \d+, \d+\)") as ei:
        solver.update_turbulence(st, SolverParams(dt=0.1), 1e30)
    # the reference raises before it assigns (turbulence.py:121-131): the
    # state keeps its k, omega and nu_t (cw_turb_rollback)
    for n, a in before.items():
        np.testing.assert_array_equal(np.array(getattr(st, n)), a, err_msg=n)
    og = co.Grid(4, 4, 1, 1.0, 1.0, 1.0)
    ost = co.State.zeros(og)
    ost.k[0, 2, 1] = np.inf
    ost.omega[:] = 1.0
    with pytest.raises(FloatingPointError) as eo:
        co.update_turbulence(ost, co.Params(dt=0.1), 1e30)
    assert str(ei.value).split("at cell")[1] == str(eo.value).split("at cell")[1]


def test_huge_nu_t_capped_no_nan():
    """test_turbulence.py:105-116"""
    st = FlowState.zeros(GridSpec(8, 8, 1, 1.0, 1.0, 1.0))
    st.u = np.random.default_rng(6).standard_normal(st.u.shape)
    st.nu_t = np.full(st.nu_t.shape, 1e6)
    solver.diffuse(st, SolverParams(dt=0.1, nu=0.0), 0.1)
    assert np.all(np.isfinite(st.u)) and np.max(np.abs(st.u)) < 10.0


def test_singular_system_raises():
    from paper_2204_01117_b200.errors import SingularSystemError
    g = GridSpec(8, 8, 1, 1, 1, 1)
    lab = classify_boundary(g, {"x_min": CellLabel.INLET, "x_max": CellLabel.SOLID_WALL,
                                "y_min": CellLabel.SOLID_WALL, "y_max": CellLabel.SOLID_WALL})
    with pytest.raises(SingularSystemError):
        build_pressure_matrix(g, lab)


@pytest.mark.parametrize("turbulence", [True, False])
def test_failed_projection_leaves_the_reference_state(turbulence):
    """A step whose projection does not converge (pcg_tol 0: no criterion is
    below it, so 10000 iterations, solver.py:272-276) raises ProjectionError
    with the state as the
    reference leaves it: u, v, w, nu_t and p after the first boundary pass
    (the failed solve does not replace p) and k, omega as advected this step
    (cw_proj_rollback); float64 against the oracle, directly and through the
    reference-layout binding (refbind, where k / omega are uploaded behind the
    projection, cw_step_defer_kw)."""
    import types

    from oracle import citywind_oracle as co
    from helpers import FIELDS, device_params, device_state, device_system, oracle_compiled
    from paper_2204_01117_b200 import scenes
    from paper_2204_01117_b200.errors import ProjectionError
    from paper_2204_01117_b200.refbind import RefStepper
    doc = scenes.cuboid(24, 20, 12, 2.0, 0.3)
    doc["solver"]["turbulence"] = turbulence
    comp = oracle_compiled(doc)
    sc = comp.scene
    ost = comp.make_state()
    comp.step_state(ost)                                  # a state with a pressure field
    dst = device_state(ost, torch.float64)
    ref = lambda a: np.ascontiguousarray(np.asarray(a).transpose(2, 1, 0))   # noqa: E731
    og = sc.grid
    rst = types.SimpleNamespace(
        grid=types.SimpleNamespace(nx=og.nx, ny=og.ny, nz=og.nz, dx=og.dx, dy=og.dy, dz=og.dz, origin=tuple(og.origin)),
        time=1.0, step_count=1, labels=ref(ost.labels).astype(np.int8),
        porosity=types.SimpleNamespace(phi=ref(ost.phi), lad=ref(ost.lad)))
    for n in FIELDS:
        setattr(rst, n, ref(getattr(ost, n)).astype(np.float64))
    with pytest.raises(co.ProjectionError):
        co.step(ost, sc.params, comp.psys, comp.W, sc.inlet, 0.0)
    psys, pre = device_system(comp)
    p, prof = device_params(sc)
    with pytest.raises(ProjectionError):
        solver.step(dst, p, psys, pre, prof, pcg_tol=0.0)
    stepper = RefStepper(dtype=torch.float64, ai_omega=sc.ai_omega)
    with pytest.raises(ProjectionError):
        stepper.step(rst, p, None, types.SimpleNamespace(name="ai1"), prof, None, 0.0)
    assert rst.step_count == 1 and rst.time == 1.0
    for n in FIELDS:
        want = getattr(ost, n)
        got = dst.fields[n].cpu().numpy()
        scale = max(float(np.abs(want).max()), 1e-30)
        assert float(np.abs(got - want).max()) <= 1e-9 * scale, n
        assert float(np.abs(ref(getattr(rst, n)) - want).max()) <= 1e-9 * scale, n
