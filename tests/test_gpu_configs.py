"""GPU parity on BASELINE.json's configs and the reference's bundled scenes,
against goldens made by the UNMODIFIED reference
(scripts/make_golden_configs.py, OPENBLAS_NUM_THREADS=1):

* C1 64x64x32 cuboid, dt 0.3, 200 steps (whole end fields);
* C2 128x128x64 street canyon, 20 steps;
* C3 256x256x64 block city, dt 0.2, steps 1-25 -- the bench scene; bench.py
  times steps 6-25;
* src/scenarios/bielefeld_like.json, 120 steps;
* src/scenarios/channel_opt.json's initial design (translate_x / translate_y
  bindings, scenario.py:394-398), 120 steps;
* gradient_descent on channel_opt (settle 120) and the C4 16-parameter
  recipe at 96x96x24 (FD gradient + one update).

Gates (north_star): identical per-step PCG iteration counts on every scene
the oracle certifies (tests/golden/cert_<name>.json: the reference's counts
survive fp32-level noise), per-step field L2 norms and end fields within
1e-4 relative (whole fields, or the golden's fixed stride subsample for the
large grids), per-step CFL within 1e-4.
"""
import json
import os

import numpy as np
import pytest

from helpers import FIELDS, GOLD, rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")

TRAJ = ["c1_cuboid_64", "c2_canyon_128", "c3_city_256", "bielefeld_120", "chopt_sim_120"]


def _gold(name):
    return np.load(os.path.join(GOLD, f"cfg_{name}.npz"))


def _certified(name):
    path = os.path.join(GOLD, f"cert_{name}.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", TRAJ)
def test_config_trajectory_matches_reference(name):
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    g = _gold(name)
    doc = json.loads(str(g["doc"]))
    sc = scenario_from_dict(doc)
    comp = CompiledScenario.compile(sc)
    theta = g["theta"] if g["theta"].size else None
    st = comp.make_state(theta)
    steps = int(g["steps"])
    iters, cfl, divb, norms = [], [], [], {n: [] for n in FIELDS}
    for _ in range(steps):
        rep = solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, 1, sc.pcg_tol)[0]
        iters.append(rep.pcg.iterations)
        cfl.append(rep.cfl)
        divb.append(rep.div_before)
        for n in FIELDS:
            norms[n].append(float(torch.linalg.vector_norm(st.fields[n].double())))
    gold_it = g["pcg_iterations"].tolist()
    cert = _certified(name)
    if cert is not None and not cert["certified"]:
        # the reference itself moves on these steps under fp32-level noise:
        # gate the others exactly, these within one iteration
        soft = set(cert["mismatched_steps"])
        for s, (a, b) in enumerate(zip(iters, gold_it), start=1):
            assert a == b or (s in soft and abs(a - b) <= 1), (s, a, b)
    else:
        assert iters == gold_it
    np.testing.assert_allclose(cfl, g["cfl"], rtol=1e-4)
    np.testing.assert_allclose(divb, g["div_before"], rtol=1e-3)
    for n in FIELDS:
        np.testing.assert_allclose(norms[n], g[f"norm_{n}"], rtol=1e-4, err_msg=n)
    stride = int(g["stride"])
    for n in FIELDS:
        got = st.fields[n].double().cpu().numpy()
        if stride:
            e = rel_l2(got.ravel()[::stride], g[f"sub_{n}"])
        else:
            e = rel_l2(got, g[n])
        assert e <= 1e-4, f"{n}: rel-L2 {e:.3e}"


def test_channel_opt_gradient_descent_matches_reference():
    """channel_opt.json (settle 120, its stable window): the reference's
    gradient_descent(max_iter=2) -- FD gradients, theta trajectory, losses."""
    from paper_2204_01117_b200.optimize import ObjectiveSpec, finite_diff_gradient, gradient_descent
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    g = _gold("chopt_opt_120")
    sc = scenario_from_dict(json.loads(str(g["doc"])))
    comp = CompiledScenario.compile(sc)
    res = gradient_descent(comp, max_iter=int(g["max_iter"]))
    np.testing.assert_allclose(res.history, g["history"], rtol=1e-4)
    assert len(res.theta_history) == len(g["theta_history"])
    for a, b in zip(res.theta_history, g["theta_history"]):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-4 * max(1.0, float(np.abs(b).max())))
    grad, base = finite_diff_gradient(comp, g["theta_history"][0], ObjectiveSpec.from_scenario(sc))
    assert abs(base.loss - g["grad_base_loss"][0]) <= 1e-4 * abs(g["grad_base_loss"][0])
    # a forward difference over eps = 0.1 amplifies the losses' relative
    # error 1e-4 by L / eps
    np.testing.assert_allclose(grad, g["grads"][0], rtol=0, atol=2e-4 * abs(base.loss) / 0.1)


def test_c4_recipe_fd_gradient_and_update_match_reference():
    """C4 (16 extent parameters, 6 regions) at 96x96x24, settle 120: the
    reference's gradient_descent(max_iter=1) = one base evaluation, the
    16-job FD gradient and the updated design's evaluation."""
    from paper_2204_01117_b200.optimize import gradient_descent
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    g = _gold("c4_city_96")
    sc = scenario_from_dict(json.loads(str(g["doc"])))
    comp = CompiledScenario.compile(sc)
    res = gradient_descent(comp, max_iter=1)
    np.testing.assert_allclose(res.history, g["history"], rtol=1e-4)
    L = float(g["history"][0])
    for a, b in zip(res.theta_history, g["theta_history"]):
        np.testing.assert_allclose(a, b, rtol=0, atol=2e-4 * L / 0.1)
