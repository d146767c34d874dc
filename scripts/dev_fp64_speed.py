"""Developer check: C3 steady-state step time in fp32 and fp64 (steps 26-45
after 25 warm-up steps, device events).  Usage: python scripts/dev_fp64_speed.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_01117_b200 import scenes, solver  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

for dtype in (torch.float32, torch.float64):
    sc = scenario_from_dict(scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2))
    comp = CompiledScenario.compile(sc, dtype=dtype)
    st = comp.make_state()
    comp.step_states(st, 25)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    reps = comp.step_states(st, 20)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    its = [r.pcg.iterations for r in reps]
    print(f"{dtype}: {ms:.2f} ms/step, {256 * 256 * 64 / ms / 1e-3:.3g} cell-steps/s, iterations {its[:4]}...")
