"""Developer check: one C4 design evaluation at 256x256x64 against the
reference golden (loss, region speeds, per-step counts); argument fp64 runs
the device in float64.  Usage: python scripts/dev_c4_eval.py [fp64]"""
import json, os, sys
import torch
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2204_01117_b200.optimize import evaluate_objective
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
from paper_2204_01117_b200.solver import make_initial_state, step_many
g = np.load("tests/golden/cfg_c4_city_256_eval.npz")
sc = scenario_from_dict(json.loads(str(g["doc"])))
comp = CompiledScenario.compile(sc, dtype=torch.float64 if "fp64" in sys.argv else torch.float32)
theta = np.asarray(g["theta"], float)
ev = evaluate_objective(comp, theta)
print("loss", ev.loss, float(g["loss"]), "rel", abs(ev.loss - float(g["loss"])) / float(g["loss"]))
print("speeds rel", (np.abs(ev.region_speeds - g["region_speeds"]) / g["region_speeds"]).tolist())
st = make_initial_state(sc.grid, comp.voxelize_design_device(theta), None, sc.solver, sc.inlet, mode=sc.init_mode, dtype=comp.dtype, device=comp.device)
its = [r.pcg.iterations for r in step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, 120, sc.pcg_tol)]
gold = g["pcg_iterations"].tolist()
print("count mismatches", [(i+1, a, b) for i, (a, b) in enumerate(zip(its, gold)) if a != b])
