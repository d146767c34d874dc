"""Developer profile of one design evaluation (bench.py's design_eval leg):
wall time of make_state and evaluate_objective, and a cProfile of the
second evaluation (host-side hot spots).  Usage: python scripts/dev_design_profile.py"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_01117_b200 import scenes  # noqa: E402
from paper_2204_01117_b200.optimize import evaluate_objective  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402


def timed(f, *a):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = f(*a)
    torch.cuda.synchronize()
    return r, time.perf_counter() - t


def main():
    doc = scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2)
    comp = CompiledScenario.compile(scenario_from_dict(doc), dtype=torch.float32)
    for i in range(3):
        _, t = timed(comp.make_state)
        print(f"make_state call {i}: {t * 1e3:.1f} ms", flush=True)
    ddoc = scenes.block_city_design(256, 256, 64, 2.0, 0, 6, 0.2, settle_steps=120)
    dcomp = CompiledScenario.compile(scenario_from_dict(ddoc), dtype=torch.float32)
    theta = np.array([d["initial"] for d in ddoc["design"]])
    for i in range(5):
        _, t = timed(evaluate_objective, dcomp, theta)
        print(f"evaluate_objective call {i}: {t:.3f} s", flush=True)
    # phases of one evaluation, each synchronised
    from paper_2204_01117_b200.solver import make_initial_state, step_many
    sc = dcomp.scenario
    for i in range(3):
        lab, t_vox = timed(dcomp.voxelize_design_device, theta)
        st, t_init = timed(make_initial_state, sc.grid, lab, None, sc.solver, sc.inlet, sc.init_mode, dcomp.dtype,
                           dcomp.device)
        _, t_head = timed(step_many, st, sc.solver, dcomp.psys, dcomp.preconditioner, sc.inlet, 60, sc.pcg_tol)
        _, t_tail = timed(step_many, st, sc.solver, dcomp.psys, dcomp.preconditioner, sc.inlet, 60, sc.pcg_tol)
        print(f"phases {i}: voxelize {t_vox * 1e3:.1f} ms, initial state {t_init * 1e3:.1f} ms, "
              f"steps 1-60 {t_head * 1e3:.1f} ms, steps 61-120 {t_tail * 1e3:.1f} ms", flush=True)
    # make_initial_state's pieces
    from paper_2204_01117_b200.grid import FlowState
    from paper_2204_01117_b200.solver import apply_boundary_conditions
    k_in, om_in = sc.solver.inlet_k_omega()
    for i in range(4):
        lab = dcomp.voxelize_design_device(theta)
        st, t_z = timed(lambda: FlowState.zeros(sc.grid, k0=k_in, omega0=om_in, dtype=dcomp.dtype,
                                                device=dcomp.device, static_dev=lab))
        _, t_bc = timed(apply_boundary_conditions, st, sc.inlet, sc.solver)
        _, t_bc2 = timed(apply_boundary_conditions, st, sc.inlet, sc.solver)
        print(f"initial pieces {i}: zeros {t_z * 1e3:.1f} ms, first boundary pass {t_bc * 1e3:.1f} ms, "
              f"second {t_bc2 * 1e3:.1f} ms", flush=True)
    pr = cProfile.Profile()
    torch.cuda.synchronize()
    pr.enable()
    evaluate_objective(dcomp, theta)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(30)


if __name__ == "__main__":
    main()
