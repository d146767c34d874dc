"""Developer timeline of one refbind.RefStepper.step at C3 (CUPTI through
torch.profiler): every copy and kernel with its start offset and duration,
so the gaps between the upload, the device step and the download show."""
import os
import sys
import time
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2204_01117_b200 import refbind, scenes  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

sc = scenario_from_dict(scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2))
comp = CompiledScenario.compile(sc)
st = comp.make_state()
comp.step_states(st, 30)
ref = lambda t: np.ascontiguousarray(t.double().cpu().numpy().transpose(2, 1, 0))  # noqa: E731
g = sc.grid
host = types.SimpleNamespace(grid=types.SimpleNamespace(nx=g.nx, ny=g.ny, nz=g.nz, dx=g.dx, dy=g.dy, dz=g.dz,
                                                        origin=tuple(g.origin)),
                             labels=ref(st.labels_dev).astype(np.int8), time=0.0, step_count=0,
                             porosity=types.SimpleNamespace(phi=ref(st.phi_dev), lad=ref(st.lad_dev)))
for n in ("u", "v", "w", "p", "k", "omega", "nu_t"):
    setattr(host, n, ref(st.fields[n]))
stepper = refbind.RefStepper(ai_omega=sc.ai_omega)
pre = types.SimpleNamespace(name="ai1")
for _ in range(3):
    stepper.step(host, sc.solver, None, pre, sc.inlet, None, sc.pcg_tol)
torch.cuda.synchronize()
walls = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        t0 = time.perf_counter()
        stepper.step(host, sc.solver, None, pre, sc.inlet, None, sc.pcg_tol)
        walls.append(time.perf_counter() - t0)
print("wall per call (ms):", [round(w * 1e3, 2) for w in walls])
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
half = ev[len(ev) // 2:]          # the second call
t0 = half[0].time_range.start
last_end = t0
for e in half:
    s, d = e.time_range.start - t0, e.time_range.end - e.time_range.start
    gap = e.time_range.start - last_end
    print(f"{s / 1e3:8.3f} ms  +{d / 1e3:7.3f} ms  gap {gap / 1e3:7.3f}  {e.name[:70]}")
    last_end = max(last_end, e.time_range.end)
