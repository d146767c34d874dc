"""Developer run: validate_karman at its default speeds (desk and full
resolution) and validate_porosity at its default grid of cases, on the
device.  Usage: python scripts/dev_validate_all.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_01117_b200 import validate  # noqa: E402

for res in ("desk", "full"):
    t = time.perf_counter()
    for r in validate.validate_karman(resolution=res):
        print(f"karman {res}: U {r.speed:4.1f} Re {r.re:8.0f} f {r.f_measured:7.3f} Hz (theory {r.f_theory:7.3f}) "
              f"err {100 * r.rel_err:5.2f}% flagged {r.flagged} steps {r.steps} wall {r.wall_s:.1f} s", flush=True)
    print(f"karman {res} total {time.perf_counter() - t:.1f} s", flush=True)
t = time.perf_counter()
for r in validate.validate_porosity():
    print(f"porosity: U {r.speed} phi {r.phi:.1f} drag {r.v_out_drag:.4f} truth {r.v_out_truth:.4f} "
          f"rel_err {r.rel_err:.3g}", flush=True)
print(f"porosity total {time.perf_counter() - t:.1f} s")
