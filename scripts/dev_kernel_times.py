"""Developer tool: warm per-kernel device times of C3 steps (CUPTI via torch.profiler).
Usage: python scripts/dev_kernel_times.py [steps]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402
from paper_2204_01117_b200 import scenes, solver  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
comp = CompiledScenario.compile(scenario_from_dict(scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2)))
st = comp.make_state()
comp.step_states(st, 15)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    reps = solver.step_many(st, comp.scenario.solver, comp.psys, comp.preconditioner, comp.scenario.inlet, n)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.split("(")[0].replace("void ", "").replace("cw::", "")
        agg[name][0] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        agg[name][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"{n} steps, iterations {[r.pcg.iterations for r in reps]}; per step:")
for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k[:60]:60s} {c / n:5.1f} launches {t / n:9.1f} us  {100 * t / tot:5.1f}%")
print(f"  total {tot / n:.1f} us per step")
