import sys, time
sys.path.insert(0, "/root/repo")
from paper_2204_01117_b200 import validate
t = time.perf_counter()
for r in validate.validate_porosity():
    print(f"U {r.speed} phi {r.phi:.1f} drag {r.v_out_drag:.5f} truth {r.v_out_truth:.5f} rel_err {r.rel_err:.3g}", flush=True)
print("total", time.perf_counter() - t)
