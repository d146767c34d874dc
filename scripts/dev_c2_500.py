"""Developer check: BASELINE.json config 2 over its full 500 steps on the
device (fp32 and fp64) against the reference golden cfg_c2_canyon_128_500:
first step whose PCG count differs, k_max next to the reference's, where (if
anywhere) the device raises, end-field rel-L2.  Usage:
python scripts/dev_c2_500.py [fp32|fp64 ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_01117_b200 import solver  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    g = np.load(os.path.join(ROOT, "tests", "golden", "cfg_c2_canyon_128_500.npz"))
    gold = g["pcg_iterations"].tolist()
    kref = g["k_max"]
    for prec in sys.argv[1:] or ["fp32", "fp64"]:
        dtype = torch.float32 if prec == "fp32" else torch.float64
        sc = scenario_from_dict(json.loads(str(g["doc"])))
        comp = CompiledScenario.compile(sc, dtype=dtype)
        st = comp.make_state()
        its, km, err = [], [], None
        for s in range(int(g["steps"])):
            try:
                r = solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, 1, sc.pcg_tol)[0]
            except Exception as e:  # noqa: BLE001
                err = f"step {s + 1}: {type(e).__name__}: {e}"[:300]
                break
            its.append(r.pcg.iterations)
            km.append(float(st.fields["k"].max()))
        first = next((i + 1 for i, (a, b) in enumerate(zip(its, gold)) if a != b), None)
        print(f"{prec}: {len(its)} steps, first count mismatch at step {first}, "
              f"mismatches {sum(a != b for a, b in zip(its, gold))}, error: {err}")
        for s in (25, 50, 75, 100, 125, 150, 200, 300, 400, 500):
            if s <= len(km):
                print(f"   step {s}: it {its[s - 1]} / ref {gold[s - 1]}, k_max {km[s - 1]:.3g} / ref {kref[s - 1]:.3g}")
        if err is None:
            stride = int(g["stride"])
            out = {n: rel(st.fields[n].double().cpu().numpy().ravel()[::stride], g[f"sub_{n}"])
                   for n in ("u", "v", "w", "p", "k", "omega", "nu_t")}
            print("   end rel-L2:", {k: f"{v:.2e}" for k, v in out.items()})


if __name__ == "__main__":
    main()
