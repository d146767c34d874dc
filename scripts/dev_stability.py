"""Developer probe: stability of a scene on the device (k, nu_t, CFL over time)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2204_01117_b200 import scenes
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
cfg = sys.argv[1]; n = int(sys.argv[2]); dts = [float(x) for x in sys.argv[3:]]
for dt in dts:
    doc = {"C3": lambda: scenes.block_city(256, 256, 64, 2.0, 0, 6, dt),
           "C2": lambda: scenes.canyon(128, 128, 64, 1.0, dt, 500),
           "C1": lambda: scenes.cuboid(64, 64, 32, 2.0, dt, 200)}[cfg]()
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    st = comp.make_state()
    out = []
    for chunk in range(n // 20):
        try:
            reps = comp.step_states(st, 20)
        except Exception as e:
            out.append(f"FAIL at chunk {chunk}: {type(e).__name__}"); break
        f = st.fields
        out.append("s%d k%.3g nut%.3g cfl%.2f it%.0f" % ((chunk + 1) * 20, float(f["k"].max()), float(f["nu_t"].max()),
                   reps[-1].cfl, np.mean([r.pcg.iterations for r in reps])))
    print(cfg, dt, " | ".join(out), flush=True)
