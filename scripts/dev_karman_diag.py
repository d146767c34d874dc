import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2204_01117_b200 import validate
from paper_2204_01117_b200.scenario import CompiledScenario
sc = validate.karman_scenario(2.0, "full")
for dt in (torch.float64, torch.float32):
    comp = CompiledScenario.compile(sc, dtype=dt)
    st = comp.make_state()
    try:
        for blk in range(21):
            comp.step_states(st, 200)
            f = st.fields
            print(dt, (blk + 1) * 200, "kmax %.3g omax %.3g omin %.3g numax %.3g umax %.3g" % (
                float(f["k"].max()), float(f["omega"].max()), float(f["omega"].min()), float(f["nu_t"].max()),
                float(f["v"].abs().max())), flush=True)
    except Exception as e:
        print(dt, "raised at block", blk, str(e)[:150], flush=True)
