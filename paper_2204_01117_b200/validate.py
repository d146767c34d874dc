"""The paper's appendix validations on the device path (
reference ``citywind.validate`` :32-235): the cylinder wake's shedding
frequency against the empirical Strouhal law, and the porosity-drag model
against no-slip walls on the same geometry.  Every simulation runs through
this package's device step (2-D mode, interior SOLID_WALL cells, probes on
the device); only the post-processing -- an FFT of one probe series, means
of a few numbers -- runs on the host.  The preconditioner benchmark of the
same reference module is ``paper_2204_01117_b200.zoo``.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import scenes
from .geometry import cylinder_mesh
from .grid import CellLabel, GridSpec, PorosityField, classify_boundary, merge_labels
from .linalg import build_ai_preconditioner, build_pressure_matrix
from .scenario import run_simulation, scenario_from_dict
from .solver import InletProfile, SolverParams, make_initial_state, step_many
from .voxelize import GridObject, voxelize

__all__ = ["AIR_NU", "CYLINDER_D", "strouhal_theory", "shedding_frequency", "KarmanRow", "karman_scenario",
           "validate_karman", "PorosityRow", "validate_porosity"]

AIR_NU = 1.57e-5
CYLINDER_D = 0.046


def strouhal_theory(speed: float, diameter: float = CYLINDER_D, nu: float = AIR_NU) -> tuple:
    """(Re, St, f) of the empirical St = 0.198 (1 - 19.7 / Re), 250 < Re < 2.5e5
    (validate.py:32-37)."""
    re = speed * diameter / nu
    st = 0.198 * (1.0 - 19.7 / re)
    return re, st, st * speed / diameter


def shedding_frequency(series, dt: float) -> tuple:
    """Dominant frequency of a probe series (validate.py:40-67): the second
    half, mean removed, Hann window, power spectrum, the peak refined by a
    parabola through the log powers of its neighbours.  Returns (f, quality)
    with quality = peak power / median power."""
    s = np.asarray(series, float)
    s = s[len(s) // 2:]
    s = s - s.mean()
    if len(s) < 16:
        return 0.0, 0.0
    power = np.abs(np.fft.rfft(s * np.hanning(len(s)))) ** 2
    df = np.fft.rfftfreq(len(s), dt)[1]
    power[0] = 0.0
    k = int(np.argmax(power))
    if power[k] <= 0:
        return 0.0, 0.0
    shift = 0.0
    if 0 < k < len(power) - 1:
        lm, l0, lp = (np.log(power[q] + 1e-300) for q in (k - 1, k, k + 1))
        curv = lm - 2.0 * l0 + lp
        if curv != 0:
            shift = float(np.clip(0.5 * (lm - lp) / curv, -0.5, 0.5))
    return float((k + shift) * df), float(power[k] / max(np.median(power[1:]), 1e-300))


@dataclass
class KarmanRow:
    speed: float
    re: float
    f_measured: float
    f_theory: float
    rel_err: float
    flagged: bool
    steps: int
    wall_s: float


def karman_scenario(speed: float, resolution: str = "desk"):
    """The bundled wake scene at `speed`, dt keeping the advective CFL at 0.9
    (validate.py:82-89)."""
    sc = scenario_from_dict(scenes.karman(resolution))
    dt = 0.9 * sc.grid.dx / speed
    return replace(sc, inlet=replace(sc.inlet, speed=speed), solver=replace(sc.solver, dt=dt, u_ref=speed))


def validate_karman(speeds=(2.0, 10.0, 20.0), resolution: str = "desk", settle_periods: float = 8.0,
                    measure_periods: float = 24.0, progress=None, dtype=torch.float32) -> list:
    """Per speed: settle, then measure the cross-stream velocity at a probe a
    diameter behind and 2.5 diameters beside the cylinder, and compare its
    shedding frequency with the Strouhal relation (validate.py:92-118)."""
    rows = []
    for speed in speeds:
        sc = karman_scenario(speed, resolution)
        re, _, f_th = strouhal_theory(speed)
        period = 1.0 / (f_th * sc.solver.dt)          # steps per shedding period
        n = int((settle_periods + measure_periods) * period)
        probe = (0.512 + CYLINDER_D, 0.384 + 2.5 * CYLINDER_D, sc.grid.dz / 2)
        t0 = time.perf_counter()
        out = run_simulation(sc, steps=n, snapshot_every=0, probes=[probe], on_step=progress, dtype=dtype)
        wall = time.perf_counter() - t0
        cross = out["probes"][0][:, 0]                 # the flow is +y: x is cross-stream
        keep = int(measure_periods * period)
        f, quality = shedding_frequency(cross[-2 * keep:], sc.solver.dt)
        rows.append(KarmanRow(speed=speed, re=re, f_measured=f, f_theory=f_th, rel_err=abs(f - f_th) / f_th,
                              flagged=quality < 5.0, steps=n, wall_s=wall))
    return rows


@dataclass
class PorosityRow:
    phi: float
    speed: float
    v_out_drag: float
    v_out_truth: float
    rel_err: float


def _porosity_setup(resolution: str):
    """Grid and base time step (validate.py:136-139), and the labels: a
    bottom-centre inlet flanked by outlets, side walls, top outlet
    (validate.py:142-150)."""
    grid, dt = (GridSpec(512, 640, 1, 1.0, 1.0, 1.0), 0.1) if resolution == "full" else \
        (GridSpec(128, 160, 1, 4.0, 4.0, 4.0), 0.4)
    labels = classify_boundary(grid, {"y_min": CellLabel.OUTLET, "y_max": CellLabel.OUTLET,
                                      "x_min": CellLabel.SOLID_WALL, "x_max": CellLabel.SOLID_WALL})
    third = grid.nx // 3
    labels[third:grid.nx - third, 0, :] = int(CellLabel.INLET)
    return grid, dt, labels


def _circle_row(grid: GridSpec, phi: float, n: int = 8) -> list:
    """n solid disks across the channel at mid-height whose packing leaves
    porosity phi (phi = 0: disks cover their squares, validate.py:153-174)."""
    if phi >= 1.0:
        return []
    lo, hi = grid.extent()
    pitch = (hi[0] - lo[0]) / n
    r = 0.5 * pitch * np.sqrt(2.0) * 1.02 if phi <= 0.0 else pitch * np.sqrt((1.0 - phi) / np.pi)
    y = lo[1] + 0.5 * (hi[1] - lo[1])
    return [GridObject(kind=CellLabel.BUILDING,
                       mesh=cylinder_mesh((lo[0] + (q + 0.5) * pitch, y), r, -grid.dz, 2 * grid.dz, segments=48),
                       phi=0.0, name=f"circle{q}") for q in range(n)]


def _top_outlet_mean_speed(state, top_outlet: torch.Tensor) -> torch.Tensor:
    """Mean cell speed over the top row's outlet cells (validate.py:177-181),
    on the device (2-D: one plane)."""
    f = state.fields
    ny = state.grid.ny
    uc = 0.5 * (f["u"][0, ny - 1, :-1] + f["u"][0, ny - 1, 1:])
    vc = 0.5 * (f["v"][0, ny - 1, :] + f["v"][0, ny, :])
    wc = 0.5 * (f["w"][0, ny - 1, :] + f["w"][1, ny - 1, :])
    sp = torch.sqrt((uc * uc + vc * vc) + wc * wc)
    return sp[top_outlet].double().mean()


def validate_porosity(speeds=(2.0, 5.0), phis=(0.0, 0.2, 0.4, 0.6, 0.8, 1.0), resolution: str = "desk",
                      steps: int = 700, avg_steps: int = 150, dtype=torch.float32) -> list:
    """Each (speed, phi) twice: the disks as porous building cells with drag,
    and as no-slip SOLID_WALL cells (pressure operator rebuilt), compared by
    the top-outlet mean speed over the last avg_steps steps
    (validate.py:184-235)."""
    grid, dt0, base = _porosity_setup(resolution)
    top = torch.from_numpy(base[:, -1, 0] == int(CellLabel.OUTLET))
    rows = []
    for speed in speeds:
        profile = InletProfile(kind="uniform", speed=speed, direction=(0, 1))
        params = SolverParams(dt=dt0 * 2.0 / max(speed, 2.0), nu=AIR_NU, cd_building=1.0, turbulence=True,
                              turb_intensity=0.05, u_ref=speed, length_scale=grid.dx * 10)
        for phi in phis:
            objs = _circle_row(grid, phi)

            def run(mode: str) -> float:
                if objs:
                    obj_labels, poros = voxelize(objs, grid, subdiv=4)
                else:
                    obj_labels, poros = np.full(grid.shape, int(CellLabel.AIR), np.int8), PorosityField.open_air(grid)
                if mode == "truth":
                    labels = base.copy()
                    labels[poros.phi < 0.5] = int(CellLabel.SOLID_WALL)
                    poros = PorosityField.open_air(grid)
                else:
                    labels = merge_labels(base, obj_labels)
                psys = build_pressure_matrix(grid, labels)
                pre = build_ai_preconditioner(psys, 1.65, 1, truncate=False)
                st = make_initial_state(grid, labels, poros, params, profile, mode="rest", dtype=dtype)
                mask = top.to(st.device)
                step_many(st, params, psys, pre, profile, steps - avg_steps)
                acc = torch.zeros((), dtype=torch.float64, device=st.device)
                for _ in range(avg_steps):                 # no host sync until the end
                    step_many(st, params, psys, pre, profile, 1, read_back=False)
                    acc += _top_outlet_mean_speed(st, mask)
                from .solver import finish
                finish(st, psys, pre, avg_steps)
                return float(acc) / avg_steps

            v_drag = run("drag")
            v_truth = v_drag if phi >= 1.0 else run("truth")
            rows.append(PorosityRow(phi=phi, speed=speed, v_out_drag=v_drag, v_out_truth=v_truth,
                                    rel_err=abs(v_drag - v_truth) / max(abs(v_truth), 1e-12)))
    return rows
