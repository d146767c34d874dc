"""Developer check: does a z-slab split reproduce the whole-grid step bit for
bit, and how deep must the halo be?  Prints per-field max |difference| for
several halo depths and slab counts, and the steps' max|w| dt / dz."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_01117_b200 import scenes  # noqa: E402
from paper_2204_01117_b200.grid import FIELDS  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402
from paper_2204_01117_b200.slabs import SlabDomain  # noqa: E402

cases = {
    "cuboid32": scenes.cuboid(32, 32, 16, 2.0, 0.3, steps=12),
    "city48": scenes.block_city(48, 48, 24, 2.0, seed=3, nb=3, dt=0.25, steps=8),
    "city48_dt1": scenes.block_city(48, 48, 24, 2.0, seed=3, nb=3, dt=1.0, steps=8),
}
for name, doc in cases.items():
    comp = CompiledScenario.compile(scenario_from_dict(doc))
    sc = comp.scenario
    base = comp.make_state()
    ref = base.copy()
    steps = doc["run"]["steps"]
    reps = comp.step_states(ref, steps)
    wmax = float(ref.fields["w"].abs().max()) * sc.solver.dt / sc.grid.dz
    print(f"{name}: ref iterations {[r.pcg.iterations for r in reps]}, end max|w| dt/dz {wmax:.3f}", flush=True)
    for nslab in (2, 3, 4):
        for halo in (3, 4, 5, 6, 7):
            try:
                dom = SlabDomain(base.copy(), sc.solver, sc.inlet, nslab, omega=sc.ai_omega, halo=halo,
                                 pcg_tol=sc.pcg_tol)
                its = [dom.step().pcg.iterations for _ in range(steps)]
                out = dom.gather()
                diffs = {n: float((out[n].double() - ref.fields[n].double()).abs().max()) for n in FIELDS}
                print(f"  nslab {nslab} halo {halo} zc {dom.zc} windows {[(w.k_lo, w.k_hi) for w in dom.windows]}: "
                      f"iters equal {its == [r.pcg.iterations for r in reps]}, "
                      f"bitwise {all(v == 0 for v in diffs.values())}, max|diff| "
                      + " ".join(f"{n}={v:.1e}" for n, v in diffs.items()), flush=True)
            except Exception as exc:
                print(f"  nslab {nslab} halo {halo}: {type(exc).__name__}: {exc}", flush=True)
