import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2204_01117_b200 import validate
for dt in (torch.float64, torch.float32):
    try:
        t = time.perf_counter()
        r = validate.validate_karman(speeds=(2.0,), resolution="full", dtype=dt)[0]
        print(dt, r, time.perf_counter() - t, flush=True)
    except Exception as e:
        print(dt, "raised", type(e).__name__, str(e)[:200], flush=True)
