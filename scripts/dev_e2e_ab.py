"""Developer A/B: HostStepper with nu_t / p uploads deferred into the step
(default) against all seven fields up before the step starts (LATE = ())."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2204_01117_b200 import scenes, solver  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

comp = CompiledScenario.compile(scenario_from_dict(scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2)))
sc = comp.scenario
state = comp.make_state()
comp.step_states(state, 20)
names = ("u", "v", "w", "p", "k", "omega", "nu_t")
host = {n: torch.empty(state.fields[n].shape, dtype=state.fields[n].dtype, pin_memory=True) for n in names}
for n in names:
    host[n].copy_(state.fields[n])
for rep in range(3):
    for late in (("nu_t", "p"), ()):
        solver.HostStepper.LATE = late
        st = solver.HostStepper(state, host)
        st.step(sc.solver, comp.psys, comp.preconditioner, sc.inlet)
        st.synchronize()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        its = []
        for _ in range(5):
            its.append(st.step(sc.solver, comp.psys, comp.preconditioner, sc.inlet).pcg.iterations)
        st.synchronize()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 5 * 1e3
        print(f"LATE={late!s:16s} {ms:7.3f} ms/step  iterations {its}", flush=True)
