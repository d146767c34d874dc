"""Developer check: the device step in float64 against a config golden's
per-step field norms (fp64): the largest relative deviation per field.
Usage: python scripts/dev_fp64_norms.py NAME"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_01117_b200 import solver  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402

FIELDS = ("u", "v", "w", "p", "k", "omega", "nu_t")
for name in sys.argv[1:]:
    g = np.load(os.path.join(ROOT, "tests", "golden", f"cfg_{name}.npz"))
    sc = scenario_from_dict(json.loads(str(g["doc"])))
    comp = CompiledScenario.compile(sc, dtype=torch.float64)
    theta = g["theta"] if g["theta"].size else None
    st = comp.make_state(theta)
    its, norms = [], {n: [] for n in FIELDS}
    for _ in range(int(g["steps"])):
        its.append(solver.step_many(st, sc.solver, comp.psys, comp.preconditioner, sc.inlet, 1, sc.pcg_tol)[0]
                   .pcg.iterations)
        for n in FIELDS:
            norms[n].append(float(torch.linalg.vector_norm(st.fields[n])))
    dev = {n: float(np.max(np.abs(np.array(norms[n]) - g[f"norm_{n}"]) / np.maximum(np.abs(g[f"norm_{n}"]), 1e-300)))
           for n in FIELDS}
    print(name, "counts identical:", its == g["pcg_iterations"].tolist(),
          "max rel norm deviation:", {n: f"{v:.1e}" for n, v in dev.items()})
