"""Developer probe: one projection on a small scene with verbose errors."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from helpers import device_params, device_state, device_system, oracle_compiled
from paper_2204_01117_b200 import scenes, solver, _native as N
comp = oracle_compiled(scenes.cuboid(int(sys.argv[1]) if len(sys.argv) > 1 else 32, 32, 16, 2.0, 0.3))
from helpers import perturbed
ost = perturbed(comp.make_state(), 1)
dst = device_state(ost, torch.float32)
psys, pre = device_system(comp)
p, prof = device_params(comp.scene)
try:
    _, rep = solver.project(dst, psys, 0.3, pre)
    print("ok", rep)
except Exception as e:
    print("EXC", type(e).__name__, e, "| last_error:", N.last_error())
