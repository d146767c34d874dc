"""Developer probe: time one PCG phase in isolation at C3 (CW_PCG_PROBE)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01117_b200 import scenes, solver
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
comp = CompiledScenario.compile(scenario_from_dict(scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2)))
st = comp.make_state()
comp.step_states(st, 2)
n = 200
for mode in (1, 2, 3):
    os.environ["CW_PCG_PROBE"] = f"{mode},{n}"
    s = st.copy()
    solver.step_many(s, comp.scenario.solver, comp.psys, comp.preconditioner, comp.scenario.inlet, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    solver.step_many(s, comp.scenario.solver, comp.psys, comp.preconditioner, comp.scenario.inlet, 1)
    e1.record(); torch.cuda.synchronize()
    print(f"mode {mode}: {e0.elapsed_time(e1) * 1e3 / n:.2f} us per phase+barrier (incl. rest of step /{n})", flush=True)
os.environ.pop("CW_PCG_PROBE")
