"""Developer check: k / nu_t maxima and PCG counts over a long C3 run at a
given dt (is the reference model's outlet runaway, reached
within the design-evaluation horizon?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_01117_b200 import scenes  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

dt = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
nx = int(sys.argv[3]) if len(sys.argv) > 3 else 256
nz = int(sys.argv[4]) if len(sys.argv) > 4 else 64
comp = CompiledScenario.compile(scenario_from_dict(scenes.block_city(nx, nx, nz, 2.0, 0, 6, dt)))
st = comp.make_state()
for s in range(0, n, 10):
    reps = comp.step_states(st, 10)
    k = st.fields["k"]
    print(f"step {s + 10}: it {[r.pcg.iterations for r in reps]} kmax {float(k.max()):.4g} "
          f"nut_max {float(st.fields['nu_t'].max()):.4g} cfl {reps[-1].cfl:.3f}", flush=True)
