"""Developer timing: where the C3 design voxelization spends its time."""
import cProfile
import os
import pstats
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2204_01117_b200 import scenes  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

comp = CompiledScenario.compile(scenario_from_dict(scenes.block_city_design(256, 256, 64, 2.0, 0, 6, 0.2)))
comp.voxelize_design_device()
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    comp.voxelize_design_device()
    torch.cuda.synchronize()
    print(f"voxelize_design_device: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
comp.voxelize_design_device()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
