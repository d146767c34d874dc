"""GPU: the z-slab decomposition against the whole-grid step.

Every slab of one grid runs in this process on one device (``SlabDomain``):
the same slab contexts, halo plan and projection kernel as one slab per GPU,
with the slabs' PCG blocks in one cooperative launch.  The dot products are
folded per z-chunk in a fixed tree and summed in global chunk order, the
slab contexts use the whole grid's chunks, and the MacCormack traces work in
global plane coordinates, so 1, 2, 3 and 4 slabs give the whole-grid step
BIT FOR BIT (torch.equal).  A halo shallower than the step's reach
(2 floor(max|w| dt/dz) + 4 planes) fails the step loudly."""
import pytest

from helpers import FIELDS
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
    got_it = [dom.step().pcg.iterations for _ in range(steps)]
    ref_it = [r.pcg.iterations for r in comp.step_states(ref, steps)]
    return dom, ref, got_it, ref_it


def _assert_bitwise(dom, ref):
    out = dom.gather()
    for n in FIELDS:
        assert out[n].shape == ref.fields[n].shape, n
        assert torch.equal(out[n], ref.fields[n]), (n, float((out[n] - ref.fields[n]).abs().max()))


@pytest.mark.parametrize("nslab", [1, 2, 3, 4])
def test_slabs_equal_whole_grid_cuboid(nslab):
    doc = scenes.cuboid(32, 32, 16, 2.0, 0.3, steps=12)
    dom, ref, got_it, ref_it = _run_pair(doc, nslab, 12)
    assert got_it == ref_it
    _assert_bitwise(dom, ref)


@pytest.mark.parametrize("nslab,halo", [(2, 4), (3, 5), (4, 4)])
def test_slabs_equal_whole_grid_city(nslab, halo):
    doc = scenes.block_city(48, 48, 24, 2.0, seed=3, nb=3, dt=0.25, steps=8)
    dom, ref, got_it, ref_it = _run_pair(doc, nslab, 8, halo)
    assert got_it == ref_it
    _assert_bitwise(dom, ref)


def test_slabs_equal_whole_grid_multi_chunk():
    """A grid whose whole-grid PCG takes z-chunks of several planes (the
    slab boundaries fall on chunk boundaries: plan_slabs aligns them)."""
    import os
    os.environ["CW_PCG_ZC"] = "4"
    try:
        doc = scenes.block_city(64, 64, 32, 2.0, seed=1, nb=3, dt=0.25, steps=5)
        dom, ref, got_it, ref_it = _run_pair(doc, 2, 5)
        assert dom.zc == 4 and all(w.k_lo % 4 == 0 for w in dom.windows)
        assert got_it == ref_it
        _assert_bitwise(dom, ref)
    finally:
        os.environ.pop("CW_PCG_ZC")


def test_halo_shallower_than_the_reach_fails_loudly():
    """At dt 1 the block city's max|w| dt/dz exceeds 1: the backtrace can
    reach 2 floor(S) + 4 = 6 planes across a slab face, so a 4-plane halo
    must raise (the reference's backtrace is unbounded, advection.py:125-142),
    and a 6-plane halo steps bit for bit like the whole grid."""
    doc = scenes.block_city(48, 48, 24, 2.0, seed=3, nb=3, dt=1.0, steps=8)
    with pytest.raises(ValueError, match="halo too shallow"):
        _run_pair(doc, 2, 8, halo=4)
    dom, ref, got_it, ref_it = _run_pair(doc, 2, 8, halo=6)
    assert got_it == ref_it
    _assert_bitwise(dom, ref)


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


def _ipc_child(handle, n, q):
    """Second process on the same GPU: open the exporter's buffer through
    cw_ipc_open, check the pattern, write the reply, close."""
    import ctypes as C
    import numpy as np
    import torch as T
    from cuda.bindings import runtime as rt
    from paper_2204_01117_b200 import _native as N
    try:
        T.cuda.set_device(0)
        p = C.c_void_p()
        N.check(N.lib().cw_ipc_open((C.c_ubyte * 64)(*handle), 0, C.byref(p)))
        host = np.empty(n, np.float32)
        err, = rt.cudaMemcpy(host.ctypes.data, p.value, 4 * n, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        ok = bool(np.array_equal(host, np.arange(n, dtype=np.float32)))
        reply = np.full(n, -2.5, np.float32)
        err2, = rt.cudaMemcpy(p.value, reply.ctypes.data, 4 * n, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
        rt.cudaDeviceSynchronize()
        N.check(N.lib().cw_ipc_close(p))
        q.put((ok, int(err), int(err2)))
    except Exception as exc:   # reported to the parent
        q.put(("error", repr(exc)))


def test_ipc_round_trip_two_processes_one_gpu():
    """The cross-GPU slab attach rests on cw_ipc_get / cw_ipc_open: export a
    device buffer (a cudaMalloc base pointer, as the slab contexts' buffers
    are) from this process, open it in another process on the same device,
    read it there and write back; this process sees the write."""
    import ctypes as C
    import numpy as np
    import torch.multiprocessing as mp
    from cuda.bindings import runtime as rt
    from paper_2204_01117_b200 import _native as N
    n = 4096
    torch.cuda.init()
    err, dptr = rt.cudaMalloc(4 * n)
    assert int(err) == 0
    try:
        src = np.arange(n, dtype=np.float32)
        rt.cudaMemcpy(dptr, src.ctypes.data, 4 * n, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
        h = (C.c_ubyte * 64)()
        N.check(N.lib().cw_ipc_get(C.c_void_p(int(dptr)), h))
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        p = ctx.Process(target=_ipc_child, args=(bytes(h), n, q))
        p.start()
        res = q.get(timeout=120)
        p.join(timeout=60)
        assert res[0] is True and res[1:] == (0, 0), res
        back = np.empty(n, np.float32)
        rt.cudaMemcpy(back.ctypes.data, dptr, 4 * n, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        assert np.array_equal(back, np.full(n, -2.5, np.float32))
    finally:
        rt.cudaFree(dptr)
