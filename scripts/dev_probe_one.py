"""Developer probe for ncu: one C3 projection whose PCG loop is replaced by
N repetitions of one phase (CW_PCG_PROBE=mode,N set by the caller)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01117_b200 import scenes, solver
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
probe = os.environ.pop("CW_PCG_PROBE", "2,50")
comp = CompiledScenario.compile(scenario_from_dict(scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2)))
st = comp.make_state()
comp.step_states(st, 2)
os.environ["CW_PCG_PROBE"] = probe
solver.step_many(st, comp.scenario.solver, comp.psys, comp.preconditioner, comp.scenario.inlet, 1)
torch.cuda.synchronize()
print("done", probe)
