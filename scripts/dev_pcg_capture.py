"""Developer tool: run C3 for a few steps so that one k_pcg launch can be captured
under ncu (`ncu -k regex:k_pcg --launch-skip 3 --launch-count 1 ...`), and
print the per-step device time without ncu.  Usage: python scripts/dev_pcg_capture.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2204_01117_b200 import scenes, solver  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
comp = CompiledScenario.compile(scenario_from_dict(scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2)))
st = comp.make_state()
comp.step_states(st, 3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = solver.step_many(st, comp.scenario.solver, comp.psys, comp.preconditioner, comp.scenario.inlet, n)
e1.record()
torch.cuda.synchronize()
its = [r.pcg.iterations for r in reps]
ms = e0.elapsed_time(e1)
print(f"{n} steps {ms:.2f} ms, {ms / n:.3f} ms/step, iterations {its}, {ms / sum(its) * 1e3:.2f} us/iteration (whole step)")
