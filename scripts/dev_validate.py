import sys, time
sys.path.insert(0, "/root/repo")
from paper_2204_01117_b200 import validate
t=time.perf_counter()
rows = validate.validate_porosity(speeds=(2.0,), phis=(0.2, 0.6), resolution="desk")
print(rows, time.perf_counter()-t)
t=time.perf_counter()
rows = validate.validate_karman(speeds=(10.0,), resolution="desk")
print(rows, time.perf_counter()-t)
