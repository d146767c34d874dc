"""Developer probe: time one PCG phase in isolation at C3 (CW_PCG_PROBE)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01117_b200 import scenes, solver
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
comp = CompiledScenario.compile(scenario_from_dict(scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2)))
st = comp.make_state()
try:
    comp.step_states(st, 2)
except Exception as exc:   # ablation builds (CW_ABL) solve wrongly; time them from the initial state
    print("warm-up steps failed:", type(exc).__name__, flush=True)
    st = comp.make_state()
NAMES = {1: "phase A + barrier", 2: "phase B + barrier", 3: "barrier", 4: "phase A TMA stream only + barrier",
         5: "barrier + 2 folds", 6: "A,B alternating (per phase)", 7: "A,B alternating, stream only (per phase)",
         8: "A,B alternating, barrier wait reported (per phase)",
         9: "A,B alternating, no global stores (per phase)",
         10: "A,B alternating, no loads: compute on stale stages (per phase)",
         12: "A,B alternating, TMA wait reported (per phase)",
         13: "A,B alternating, mean first-stage latency reported", 14: "A,B alternating, mean job time reported",
         15: "A,B alternating, max over blocks of job time", 16: "A,B alternating, min over blocks of job time",
         17: "barrier + chunk-structured fold (2 values)", 18: "barrier + fold_multi (2 values)"}


def timed(mode, n):
    os.environ["CW_PCG_PROBE"] = f"{mode},{n}"
    s = st.copy()
    try:
        solver.step_many(s, comp.scenario.solver, comp.psys, comp.preconditioner, comp.scenario.inlet, 1)
    except Exception:
        s = st.copy()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    try:
        rep = solver.step_many(s, comp.scenario.solver, comp.psys, comp.preconditioner, comp.scenario.inlet, 1)
    except Exception as exc:   # ablation builds: the state after a probe may be non-finite
        rep = None
        print("  step raised", type(exc).__name__, flush=True)
    e1.record(); torch.cuda.synchronize()
    if rep is not None and mode >= 13:
        print(f"  {NAMES[mode]}: {rep[0].pcg.criterion:.2f} us", flush=True)
    if rep is not None and mode in (8, 12):
        what = "grid-barrier" if mode == 8 else "TMA stage (thread 0)"
        print(f"  mean {what} wait per block and phase: {rep[0].pcg.criterion:.2f} us", flush=True)
    return e0.elapsed_time(e1) * 1e3


modes = [int(m) for m in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 3, 4, 5, 6, 7]
for mode in modes:
    a, b = timed(mode, 100), timed(mode, 400)
    print(f"mode {mode} ({NAMES.get(mode, '?')}): {(b - a) / 300:.2f} us per iteration", flush=True)
os.environ.pop("CW_PCG_PROBE")
