"""Design-per-rank sharding of the optimizer (world size 2, gloo, CPU).

The forward evaluation is replaced by an analytic CPU objective so the test
checks the host logic only: job construction (forward/backward steps at the
bounds, optimize.py:124-135), round-robin sharding over ranks, the single
all-reduce of the losses, and equality with the serial gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class _Sc:
    def __init__(self):
        from paper_2204_01117_b200.scenario import DesignParam
        self.design = [DesignParam(f"p{i}", -1.0, 1.0 if i != 2 else 0.05, 0.0, "o", "extent_z")
                       for i in range(5)]

    def design_bounds(self):
        return (np.array([p.initial for p in self.design]), np.array([p.lo for p in self.design]),
                np.array([p.hi for p in self.design]))


class _Comp:
    scenario = _Sc()


def _fake_eval(compiled, theta, spec=None, profile=None):
    from paper_2204_01117_b200.optimize import Evaluation
    t = np.asarray(theta, float)
    loss = float(np.sum((t - 0.3) ** 2) + np.sin(t).sum())
    return Evaluation(loss=loss, region_speeds=np.zeros(1), theta=t)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_01117_b200.optimize import DesignVector, finite_diff_gradient
    comp = _Comp()
    design = DesignVector.from_scenario(comp.scenario)
    theta = np.array([0.1, -0.2, 0.0, 0.5, 0.9])
    grad, _ = finite_diff_gradient(comp, theta, None, eps=0.1, design=design, group=dist.group.WORLD,
                                   evaluate=_fake_eval)
    out[rank] = grad.tolist()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_fd_gradient_sharded_equals_serial():
    from paper_2204_01117_b200.optimize import DesignVector, finite_diff_gradient, shard
    assert shard(5, 0, 2) == [0, 2, 4] and shard(5, 1, 2) == [1, 3]
    comp = _Comp()
    design = DesignVector.from_scenario(comp.scenario)
    theta = np.array([0.1, -0.2, 0.0, 0.5, 0.9])
    serial, _ = finite_diff_gradient(comp, theta, None, eps=0.1, design=design, evaluate=_fake_eval)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        np.testing.assert_array_equal(np.array(out[r]), serial)
    # p2 (0 + 0.1 > 0.05) takes a backward difference; p4 lands exactly on
    # its bound (0.9 + 0.1 == 1.0) and stays forward (the reference uses <=)
    from paper_2204_01117_b200.optimize import fd_jobs
    steps, _ = fd_jobs(theta, design, 0.1)
    assert steps == [0.1, 0.1, -0.1, 0.1, 0.1]


def _failing_eval(compiled, theta, spec=None, profile=None):
    t = np.asarray(theta, float)
    if t[3] > 0.55:      # the job perturbing p3, owned by rank 1 (round robin)
        raise FloatingPointError("objective evaluation produced nan")
    return _fake_eval(compiled, theta, spec, profile)


def _failing_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_01117_b200.optimize import DesignVector, finite_diff_gradient
    comp = _Comp()
    design = DesignVector.from_scenario(comp.scenario)
    theta = np.array([0.1, -0.2, 0.0, 0.5, 0.9])
    try:
        finite_diff_gradient(comp, theta, None, eps=0.1, design=design, group=dist.group.WORLD,
                             evaluate=_failing_eval)
        out[rank] = "returned"
    except FloatingPointError as exc:
        out[rank] = f"FloatingPointError: {exc}"
    dist.destroy_process_group()


def test_fd_gradient_sharded_job_error_raises_on_every_rank():
    """a job that raises on one rank must not leave the others
    waiting in the all-reduce; every rank raises the same exception type."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_failing_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        assert out[r].startswith("FloatingPointError"), out[r]
        assert "job 3" in out[r]
