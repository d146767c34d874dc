"""Golden fixture of the reference's preconditioner benchmark:
validate.bench_preconditioners("small") -- condition number (2-norm,
Lanczos) and PCG iteration count per preconditioner on the 128 x 193 x 2
benchmark system -- and validate.omega_sweep("small"), by importing the
UNMODIFIED reference here.  Writes tests/golden/zoo_small.json.

    python scripts/make_golden_zoo.py
"""
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from citywind import validate  # noqa: E402

t0 = time.perf_counter()
rows = validate.bench_preconditioners("small")
t1 = time.perf_counter()
sweep = validate.omega_sweep("small")
t2 = time.perf_counter()
out = {"bench": [{"preconditioner": r.preconditioner, "omega": r.omega, "kappa": r.kappa,
                  "iterations": r.iterations, "wall_ms": r.wall_ms} for r in rows],
       "omega_sweep": [[om, k] for om, k in sweep],
       "seconds": {"bench": round(t1 - t0, 1), "sweep": round(t2 - t1, 1)},
       "source": "citywind.validate.bench_preconditioners('small') and omega_sweep('small'), unmodified reference"}
with open(os.path.join(ROOT, "tests", "golden", "zoo_small.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out, indent=1))
