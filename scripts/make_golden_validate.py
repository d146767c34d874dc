"""Golden fixtures of the reference's appendix validations, by
importing the UNMODIFIED reference here:
  validate_karman(speeds=(10.0,), resolution="desk")  -- shedding frequency
  validate_porosity(speeds=(2.0,), phis=(0.2, 0.6), resolution="desk")
Writes tests/golden/validate_desk.json.

    python scripts/make_golden_validate.py
"""
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import tempfile  # noqa: E402

os.chdir(tempfile.mkdtemp())
from citywind import validate  # noqa: E402

out = {"source": "citywind.validate, unmodified reference"}
t0 = time.perf_counter()
rows = validate.validate_karman(speeds=(10.0,), resolution="desk")
out["karman"] = [vars(r) for r in rows]
out["karman_seconds"] = round(time.perf_counter() - t0, 1)
print(out["karman"], flush=True)
t0 = time.perf_counter()
rows = validate.validate_porosity(speeds=(2.0,), phis=(0.2, 0.6), resolution="desk")
out["porosity"] = [vars(r) for r in rows]
out["porosity_seconds"] = round(time.perf_counter() - t0, 1)
print(out["porosity"], flush=True)
with open(os.path.join(ROOT, "tests", "golden", "validate_desk.json"), "w") as fh:
    json.dump(out, fh, indent=1, default=float)
