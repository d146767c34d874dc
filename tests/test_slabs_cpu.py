"""z-slab host logic on the CPU: the plane plan, the window geometry, and the
halo refresh with one slab per rank (``DistExchange`` over gloo, world sizes
2 and 3) against the in-process ``LocalExchange``."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_01117_b200.slabs import DistExchange, LocalExchange, SlabWindow, plan_slabs

SHAPES = {"u": (9, 6), "v": (8, 7), "w": (8, 6), "p": (8, 6), "k": (8, 6), "omega": (8, 6), "nu_t": (8, 6)}


def _global(nz, seed=0):
    g = torch.Generator().manual_seed(seed)
    return {n: torch.rand((nz + (1 if n == "w" else 0),) + SHAPES[n][::-1], generator=g, dtype=torch.float64)
            for n in SHAPES}


def _windows(nz, n, halo):
    return [SlabWindow.of(a, b, halo, nz) for a, b in plan_slabs(nz, n)]


def _local_fields(glob, w):
    """The window with its owned planes from the global field and garbage halos."""
    out = {}
    for n, t in glob.items():
        a, b = w.planes(n)
        loc = torch.full((b - a,) + t.shape[1:], -777.0, dtype=t.dtype)
        oa, ob = w.owned(n)
        loc[oa - a:ob - a] = t[oa:ob]
        out[n] = loc
    return out


def _check(glob, w, loc):
    for n, t in glob.items():
        a, b = w.planes(n)
        assert torch.equal(loc[n], t[a:b]), n


def test_plan_slabs_balanced_and_contiguous():
    for nz, n in ((64, 8), (64, 3), (10, 4), (7, 7)):
        r = plan_slabs(nz, n)
        assert r[0][0] == 0 and r[-1][1] == nz
        assert all(r[i][1] == r[i + 1][0] for i in range(n - 1))
        sizes = [b - a for a, b in r]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        plan_slabs(4, 5)


def test_windows_cover_faces_once():
    ws = _windows(20, 4, 3)
    for name in ("p", "w"):
        owned = [w.owned(name) for w in ws]
        assert owned[0][0] == 0 and owned[-1][1] == (21 if name == "w" else 20)
        assert all(owned[i][1] == owned[i + 1][0] for i in range(3))


@pytest.mark.parametrize("nz,n,halo", [(16, 2, 4), (20, 4, 3), (12, 3, 2)])
def test_local_exchange_fills_halos(nz, n, halo):
    glob = _global(nz)
    ws = _windows(nz, n, halo)
    locs = [_local_fields(glob, w) for w in ws]
    LocalExchange(ws).exchange(locs)
    for w, loc in zip(ws, locs):
        _check(glob, w, loc)


def _worker(rank, world, port, nz, halo, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        glob = _global(nz)
        ws = _windows(nz, world, halo)
        loc = _local_fields(glob, ws[rank])
        DistExchange(ws, rank).exchange(loc)
        _check(glob, ws[rank], loc)
        # a second refresh of p only leaves the others untouched
        loc["p"].fill_(-1.0)
        a, b = ws[rank].planes("p")
        oa, ob = ws[rank].owned("p")
        loc["p"][oa - a:ob - a] = glob["p"][oa:ob]
        DistExchange(ws, rank).exchange(loc, names=("p",))
        _check(glob, ws[rank], loc)
        out[rank] = True
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,nz,halo", [(2, 12, 4), (3, 15, 3)])
def test_dist_exchange_gloo(world, nz, halo):
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), nz, halo, out), nprocs=world, join=True)
    assert all(out.get(r) for r in range(world))
