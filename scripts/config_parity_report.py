"""Parity report on the config goldens (the numbers behind
tests/test_gpu_configs.py): per scene, whether the per-step PCG counts equal
the reference's, and each end field's relative L2 error next to the
reference's own noise floor (scripts/certify_configs.py).

    python scripts/config_parity_report.py      -> profiles/r2_config_parity.md
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import FIELDS, GOLD, rel_l2  # noqa: E402
from paper_2204_01117_b200 import solver  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

TRAJ = ["c1_cuboid_64", "c2_canyon_128", "c3_city_256", "bielefeld_120", "chopt_sim_120"]


def main():
    rows = []
    for name in TRAJ:
        g = np.load(os.path.join(GOLD, f"cfg_{name}.npz"))
        with open(os.path.join(GOLD, f"cert_{name}.json")) as fh:
            cert = json.load(fh)
        doc = json.loads(str(g["doc"]))
        sc = scenario_from_dict(doc)
        comp = CompiledScenario.compile(sc)
        theta = g["theta"] if g["theta"].size else None
        st = comp.make_state(theta)
        reps = solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, int(g["steps"]), sc.pcg_tol)
        its = [r.pcg.iterations for r in reps]
        stride = int(g["stride"])
        err = {}
        for n in FIELDS:
            got = st.fields[n].double().cpu().numpy()
            err[n] = rel_l2(got.ravel()[::stride], g[f"sub_{n}"]) if stride else rel_l2(got, g[n])
        rows.append((name, int(g["steps"]), its == g["pcg_iterations"].tolist(),
                     sum(a != b for a, b in zip(its, g["pcg_iterations"])), cert, err))
    out = ["| scene | steps | PCG counts = reference | reference's own count moves under fp32-level noise | "
           + " | ".join(f"{n} err / floor" for n in FIELDS) + " |",
           "|---|---|---|---|" + "---|" * len(FIELDS)]
    for name, steps, same, nbad, cert, err in rows:
        fl = cert["field_floor_rel_l2"]
        out.append(f"| {name} | {steps} | {'yes' if same else f'no ({nbad} steps)'} | "
                   f"{cert['mismatched_steps'] or 'none'} | "
                   + " | ".join(f"{err[n]:.1e} / {fl[n]:.1e}" for n in FIELDS) + " |")
    text = ("Config parity (GPU fp32 vs the unmodified reference's goldens; floor = the reference "
            "algorithm's own end-field deviation under 1e-6 relative noise per step)\n\n" + "\n".join(out) + "\n")
    with open(os.path.join(ROOT, "profiles", "r2_config_parity.md"), "w") as fh:
        fh.write(text)
    print(text)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    main()
