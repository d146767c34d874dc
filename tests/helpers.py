"""Shared test helpers: moving states between the oracle (numpy, x-fastest)
and the device FlowState, and the relative-L2 metric used by every parity
gate (north_star: 1e-4 in fp32)."""
from __future__ import annotations

import os

import numpy as np

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIELDS = ("u", "v", "w", "p", "k", "omega", "nu_t")


def rel_l2(a, b):
    a = np.asarray(a, float).ravel()
    b = np.asarray(b, float).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def golden(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def ref_grid(og):
    from paper_2204_01117_b200.grid import GridSpec
    return GridSpec(og.nx, og.ny, og.nz, og.dx, og.dy, og.dz, tuple(og.origin))


def device_state(ost, dtype):
    """oracle State -> device FlowState (same x-fastest layout, no transposes)."""
    import torch
    from paper_2204_01117_b200.grid import FlowState
    dev = torch.device("cuda", 0)
    f = {n: torch.from_numpy(np.ascontiguousarray(getattr(ost, n))).to(dev, dtype) for n in FIELDS}
    return FlowState(ref_grid(ost.grid), f,
                     torch.from_numpy(np.ascontiguousarray(ost.labels)).to(dev),
                     torch.from_numpy(np.ascontiguousarray(ost.phi, dtype=np.float64)).to(dev),
                     torch.from_numpy(np.ascontiguousarray(ost.lad, dtype=np.float64)).to(dev),
                     ost.time, ost.step_count)


def fields_of(dst):
    return {n: dst.fields[n].double().cpu().numpy() for n in FIELDS}


def round_state(ost, np_dtype):
    """Round an oracle state's fields to the device precision (in place)."""
    for n in FIELDS:
        setattr(ost, n, getattr(ost, n).astype(np_dtype).astype(np.float64))
    return ost


def oracle_compiled(doc):
    from oracle import citywind_oracle as co
    return co.Compiled(co.scene_from_dict(doc))


def device_system(comp):
    """Device pressure system + AI1 preconditioner for an oracle Compiled."""
    from paper_2204_01117_b200.grid import to_ref_layout
    from paper_2204_01117_b200.linalg import build_ai_preconditioner, build_pressure_matrix
    g = ref_grid(comp.scene.grid)
    psys = build_pressure_matrix(g, to_ref_layout(comp.boundary))
    pre = build_ai_preconditioner(psys, comp.scene.ai_omega, 1, truncate=False)
    return psys, pre


def device_params(sc):
    from paper_2204_01117_b200.solver import InletProfile, SolverParams
    p = SolverParams(**vars(sc.params))
    i = sc.inlet
    prof = InletProfile(i.kind, i.speed, i.u_star, i.z0, i.kappa, i.direction)
    return p, prof


def perturbed(ost, seed=0, amp=0.3):
    """Smooth + noisy perturbation of an oracle state's velocity and turbulence."""
    rng = np.random.default_rng(seed)
    for n in ("u", "v", "w"):
        a = getattr(ost, n)
        setattr(ost, n, a + amp * rng.standard_normal(a.shape))
    ost.k = ost.k * (1.0 + 0.5 * rng.random(ost.k.shape))
    ost.omega = ost.omega * (1.0 + 0.5 * rng.random(ost.omega.shape))
    ost.nu_t = ost.nu_t * (1.0 + 5.0 * rng.random(ost.nu_t.shape))
    ost.p = 0.1 * rng.standard_normal(ost.p.shape)
    return ost
