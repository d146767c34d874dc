"""Developer run: validate_karman at full resolution (512x768) in float64 at
the default speeds.  Usage: python scripts/dev_karman_full64.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_01117_b200 import validate  # noqa: E402

for r in validate.validate_karman(resolution="full", dtype=torch.float64):
    print(f"karman full fp64: U {r.speed:4.1f} f {r.f_measured:7.3f} Hz (theory {r.f_theory:7.3f}) "
          f"err {100 * r.rel_err:5.2f}% flagged {r.flagged} steps {r.steps} wall {r.wall_s:.1f} s", flush=True)
