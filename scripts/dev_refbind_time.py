"""Developer timing of refbind.RefStepper at C3: per-call wall time and the
split between upload + conversion, the device step and conversion + download."""
import os
import sys
import time
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2204_01117_b200 import refbind, scenes, solver  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

sc = scenario_from_dict(scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2))
comp = CompiledScenario.compile(sc)
st = comp.make_state()
comp.step_states(st, 5)
ref = lambda t: np.ascontiguousarray(t.double().cpu().numpy().transpose(2, 1, 0))  # noqa: E731
g = sc.grid
host = types.SimpleNamespace(grid=types.SimpleNamespace(nx=g.nx, ny=g.ny, nz=g.nz, dx=g.dx, dy=g.dy, dz=g.dz,
                                                        origin=tuple(g.origin)),
                             labels=ref(st.labels_dev).astype(np.int8), time=0.0, step_count=0,
                             porosity=types.SimpleNamespace(phi=ref(st.phi_dev), lad=ref(st.lad_dev)))
for n in ("u", "v", "w", "p", "k", "omega", "nu_t"):
    setattr(host, n, ref(st.fields[n]))
orig_step = refbind._dev_step
tsplit = {}


def timed_step(*a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig_step(*a, **k)
    torch.cuda.synchronize()
    tsplit["step"] = time.perf_counter() - t0
    return r


refbind._dev_step = timed_step
t0 = time.perf_counter()
stepper = refbind.RefStepper(ai_omega=sc.ai_omega)
pre = types.SimpleNamespace(name="ai1")
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = stepper.step(host, sc.solver, None, pre, sc.inlet, None, sc.pcg_tol)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"call {i}: {dt * 1e3:.1f} ms, device step {tsplit['step'] * 1e3:.1f} ms, it {rep.pcg.iterations}",
          flush=True)
# raw copy bandwidth
a = torch.empty(235667456 // 8, dtype=torch.float64, pin_memory=True)
d = torch.empty_like(a, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(a, non_blocking=True); torch.cuda.synchronize()
    h2d = time.perf_counter() - t0
    t0 = time.perf_counter(); a.copy_(d, non_blocking=True); torch.cuda.synchronize()
    d2h = time.perf_counter() - t0
print(f"pinned 235.7 MB: H2D {h2d * 1e3:.1f} ms ({0.2357 / h2d:.1f} GB/s), D2H {d2h * 1e3:.1f} ms ({0.2357 / d2h:.1f} GB/s)")
