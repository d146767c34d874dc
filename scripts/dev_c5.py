"""Developer check: the C5 grid (512x512x128, 33.5 M cells) on one GPU -- compile,
voxelize, a few timed steps, PCG iteration counts and device time per step.
Usage: python scripts/dev_c5.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2204_01117_b200 import scenes, solver  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
t0 = time.perf_counter()
comp = CompiledScenario.compile(scenario_from_dict(scenes.CONFIGS["C5"]()))
st = comp.make_state()
torch.cuda.synchronize()
print(f"C5 compile + voxelize + initial state: {time.perf_counter() - t0:.1f} s", flush=True)
comp.step_states(st, 3)
torch.cuda.synchronize()
import ctypes as C  # noqa: E402
import json  # noqa: E402
from paper_2204_01117_b200 import _native as N  # noqa: E402
ctx = solver._acquire(comp.psys, comp.preconditioner, st)
comp.psys.pool.release(ctx)
N.check(N.lib().cw_pcg_timing(ctx.h, n))
zc, nch = C.c_int(), C.c_int()
N.check(N.lib().cw_pcg_chunks(ctx.h, C.byref(zc), C.byref(nch)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = solver.step_many(st, comp.scenario.solver, comp.psys, comp.preconditioner, comp.scenario.inlet, n)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
ncell = 512 * 512 * 128
its = [r.pcg.iterations for r in reps]
print(f"C5: {n} steps {ms / n:.2f} ms/step, {ncell * n / ms * 1e3:.3e} cell-steps/s, iterations {its}, "
      f"cfl {[round(r.cfl, 3) for r in reps]}, k max {float(st.fields['k'].max()):.3g}, "
      f"GPU memory {torch.cuda.max_memory_allocated() / 1e9:.2f} GB", flush=True)
pcg = (C.c_float * n)()
got = C.c_int()
N.check(N.lib().cw_read_pcg_timing(ctx.h, pcg, n, C.byref(got)))
pcg = [pcg[q] for q in range(got.value)]
nu = comp.psys.n
byt = [20.0 * ncell + 8.0 * nu + 44.0 * i * nu for i in its]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
ach = sum(byt) / (sum(pcg) * 1e-3) / 1e9
print(f"C5 k_pcg: zc {zc.value}, {nch.value} chunks, {sum(pcg) / len(pcg):.2f} ms per launch "
      f"({100 * sum(pcg) / ms:.1f}% of the steps), {ach:.0f} GB/s algorithmic = {ach / peak:.3f} of {peak:.0f} GB/s",
      flush=True)
