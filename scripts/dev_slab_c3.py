"""Developer check: the C3 scene split into N z-slabs in one process
(SlabDomain, the slab contexts and kernels of one slab per GPU) against the
whole-grid step: PCG counts, bitwise equality or the largest difference,
and the per-step time.  Usage: python scripts/dev_slab_c3.py [N ...]"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import FIELDS  # noqa: E402
from paper_2204_01117_b200 import scenes  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402
from paper_2204_01117_b200.slabs import SlabDomain, plan_slabs, whole_grid_chunk  # noqa: E402


def main():
    doc = scenes.block_city(256, 256, 64, 2.0, 0, 6, 0.2)
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    sc = comp.scenario
    zc = whole_grid_chunk(sc.grid, torch.float32, "cuda:0")
    for n in [int(a) for a in sys.argv[1:]] or [2, 4, 8]:
        ref = comp.make_state()
        print(f"nslab {n}: whole-grid chunk {zc}, plan {plan_slabs(sc.grid.nz, n, zc)}", flush=True)
        dom = SlabDomain(ref.copy(), sc.solver, sc.inlet, n, omega=sc.ai_omega, halo=6, pcg_tol=sc.pcg_tol)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got = [dom.step().pcg.iterations for _ in range(5)]
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        want = [r.pcg.iterations for r in comp.step_states(ref, 5)]
        out = dom.gather()
        diff = {f: float((out[f] - ref.fields[f]).abs().max()) for f in FIELDS}
        print(f"   counts {got} vs {want}; bitwise {all(v == 0.0 for v in diff.values())}; "
              f"max |diff| {max(diff.values()):.3g}; {1e3 * (t1 - t0) / 5:.1f} ms/step", flush=True)


if __name__ == "__main__":
    main()
