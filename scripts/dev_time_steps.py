"""Developer timing probe (not the bench): time device steps of a scene whose
voxelization is supplied by the oracle, print per-stage device times and
PCG iteration counts.  Usage: python scripts/dev_time_steps.py C3 20"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import device_params, device_state, device_system, oracle_compiled  # noqa: E402
from paper_2204_01117_b200 import scenes, solver  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    prec = torch.float64 if "fp64" in sys.argv else torch.float32
    doc = scenes.CONFIGS[cfg]()
    t0 = time.time()
    comp = oracle_compiled(doc)
    ost = comp.make_state()
    print(f"oracle compile+voxelize {time.time() - t0:.1f}s", flush=True)
    dst = device_state(ost, prec)
    psys, pre = device_system(comp)
    p, prof = device_params(comp.scene)
    r = solver.step(dst, p, psys, pre, prof)
    print("first step timings (ms):", {k: round(v * 1e3, 3) for k, v in r.timings.items()},
          "iters", r.pcg.iterations, flush=True)
    for _ in range(2):
        r = solver.step(dst, p, psys, pre, prof)
        print("step timings (ms):", {k: round(v * 1e3, 3) for k, v in r.timings.items()},
              "iters", r.pcg.iterations, "cfl %.3f" % r.cfl, flush=True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = solver.step_many(dst, p, psys, pre, prof, n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    its = [x.pcg.iterations for x in reps]
    ncell = doc["grid"]["nx"] * doc["grid"]["ny"] * doc["grid"]["nz"]
    print(f"{cfg}: {n} steps {ms:.1f} ms -> {ms / n:.3f} ms/step, {ncell * n / ms * 1e3:.3e} cell-steps/s, "
          f"iters {its}, mean {np.mean(its):.1f}, ms/iter {ms / sum(its):.4f}")


if __name__ == "__main__":
    main()
