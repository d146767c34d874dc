"""Developer diagnostic: where does a z-slab step first differ from the
whole-grid step?  One step, stage by stage (PRE, SOLVE, POST) on the whole
grid (one context, the same stage entry points) and on SlabDomain's parts;
per field: max |difference| over the owned planes and the planes it sits on."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2204_01117_b200 import _native as N  # noqa: E402
from paper_2204_01117_b200 import scenes, solver  # noqa: E402
from paper_2204_01117_b200.grid import FIELDS  # noqa: E402
from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict  # noqa: E402
from paper_2204_01117_b200.slabs import SlabDomain  # noqa: E402

nslab = int(sys.argv[1]) if len(sys.argv) > 1 else 2
halo = int(sys.argv[2]) if len(sys.argv) > 2 else 4
doc = scenes.cuboid(32, 32, 16, 2.0, 0.3, steps=3)
comp = CompiledScenario.compile(scenario_from_dict(doc))
sc = comp.scenario
st = comp.make_state()
comp.step_states(st, 2)
ref = st.copy()
dom = SlabDomain(st.copy(), sc.solver, sc.inlet, nslab, omega=sc.ai_omega, halo=halo, pcg_tol=sc.pcg_tol)
prm, inl = sc.solver.native(), sc.inlet.native()
ctx = solver._acquire(comp.psys, comp.preconditioner, ref)
g, has = solver.drag_coefficient(ref, sc.solver)
f = ctx.fields(ref, g, has)
lib = N.lib()


def whole(stage):
    N.check(lib.cw_run_stage(ctx.h, C.byref(f), C.byref(prm), C.byref(inl), stage, float(dom.tol), ctx.stream))
    rc, _ = ctx.read_reports(1)


def compare(tag):
    out = dom.gather()
    for n in FIELDS:
        d = (out[n].double() - ref.fields[n].double()).abs()
        m = float(d.max())
        planes = sorted(set(int(k) for k in torch.nonzero(d.amax(dim=(1, 2)) > 0).flatten().tolist()))
        print(f"  {tag} {n}: max|diff| {m:.2e} on planes {planes[:12]}", flush=True)


dom.exchange.exchange([p.fields for p in dom.parts])
for p in dom.parts:
    p.run(N.CW_STAGE_PRE, prm, inl)
whole(N.CW_STAGE_PRE)
print(f"nslab {nslab} halo {halo} windows {[(w.k_lo, w.k_hi, w.kb, w.ke) for w in dom.windows]}")
compare("PRE")
ctxs = (C.c_void_p * len(dom.parts))(*[p.h.value for p in dom.parts])
fs = (N.cw_fields * len(dom.parts))(*[p.native_fields() for p in dom.parts])
N.check(lib.cw_slab_group_pcg(ctxs, fs, len(dom.parts), C.byref(prm), dom.tol, dom.parts[0].stream))
whole(N.CW_STAGE_SOLVE)
compare("SOLVE")
dom.exchange.exchange([p.fields for p in dom.parts], names=("p",))
for p in dom.parts:
    p.run(N.CW_STAGE_POST, prm, inl)
whole(N.CW_STAGE_POST)
compare("POST")
for p in dom.parts:
    print("  reports", [(r.iterations, r.criterion) for r in p.reports(3)[1]])
