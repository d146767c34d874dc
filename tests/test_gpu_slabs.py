"""GPU: the z-slab decomposition against the whole-grid step.

Every slab of one grid runs in this process on one device (``SlabDomain``):
the same slab contexts, halo plan and projection kernel as one slab per GPU,
with the slabs' PCG blocks in one cooperative launch.  The dot products are
folded per slab and combined in slab order, so the bits differ from the
whole-grid fold by rounding only: iteration counts must be identical and the
fields equal to fp32 rounding."""
import numpy as np
import pytest

from helpers import FIELDS, rel_l2
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _compiled(doc):
    from paper_2204_01117_b200.scenario import CompiledScenario, scenario_from_dict
    return CompiledScenario.compile(scenario_from_dict(doc))


def _run_pair(doc, nslab, steps, halo=4):
    from paper_2204_01117_b200.slabs import SlabDomain
    comp = _compiled(doc)
    sc = comp.scenario
    ref = comp.make_state()
    dom = SlabDomain(ref.copy(), sc.solver, sc.inlet, nslab, omega=sc.ai_omega, halo=halo, pcg_tol=sc.pcg_tol)
    got_it, ref_it = [], []
    for _ in range(steps):
        got_it.append(dom.step().pcg.iterations)
    ref_it = [r.pcg.iterations for r in comp.step_states(ref, steps)]
    return dom, ref, got_it, ref_it


@pytest.mark.parametrize("nslab", [2, 3])
def test_slabs_match_whole_grid_cuboid(nslab):
    doc = scenes.cuboid(32, 32, 16, 2.0, 0.3, steps=12)
    dom, ref, got_it, ref_it = _run_pair(doc, nslab, 12)
    assert got_it == ref_it
    out = dom.gather()
    for n in FIELDS:
        a = out[n].double().cpu().numpy()
        b = ref.fields[n].double().cpu().numpy()
        assert a.shape == b.shape, n
        assert rel_l2(a, b) <= 1e-5, (n, rel_l2(a, b))


def test_slabs_match_whole_grid_city():
    doc = scenes.block_city(48, 48, 24, 2.0, seed=3, nb=3, dt=0.25, steps=8)
    dom, ref, got_it, ref_it = _run_pair(doc, 4, 8)
    assert got_it == ref_it
    out = dom.gather()
    for n in FIELDS:
        assert rel_l2(out[n].double().cpu().numpy(), ref.fields[n].double().cpu().numpy()) <= 1e-5, n


def test_single_slab_is_the_whole_grid():
    """One slab: the slab path reduces to the whole-grid kernels bit for bit."""
    doc = scenes.cuboid(24, 24, 12, 2.0, 0.3, steps=6)
    dom, ref, got_it, ref_it = _run_pair(doc, 1, 6)
    assert got_it == ref_it
    out = dom.gather()
    for n in FIELDS:
        assert torch.equal(out[n], ref.fields[n]), n


def test_halo_too_deep_is_rejected():
    from paper_2204_01117_b200.slabs import SlabDomain
    comp = _compiled(scenes.cuboid(16, 16, 8, 2.0, 0.3))
    st = comp.make_state()
    with pytest.raises(ValueError):
        SlabDomain(st, comp.scenario.solver, comp.scenario.inlet, 4, halo=4)


def test_dist_slab_solver_single_rank():
    """The one-slab-per-GPU driver with a one-rank NCCL group equals the
    whole-grid step bit for bit (the multi-GPU attach path needs >1 GPU)."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2204_01117_b200.slabs import DistSlabSolver
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comp = _compiled(scenes.cuboid(24, 24, 12, 2.0, 0.3, steps=5))
        sc = comp.scenario
        ref = comp.make_state()
        sol = DistSlabSolver(ref.copy(), sc.solver, sc.inlet, omega=sc.ai_omega, pcg_tol=sc.pcg_tol)
        got = [r.pcg.iterations for r in sol.step_many(5)]
        want = [r.pcg.iterations for r in comp.step_states(ref, 5)]
        assert got == want
        for n in FIELDS:
            assert torch.equal(sol.part.owned_view(n), ref.fields[n]), n
    finally:
        dist.destroy_process_group()
