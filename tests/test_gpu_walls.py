"""GPU: non-box unknown sets -- interior SOLID_WALL cells
inside the flow, as validate_porosity's no-slip "truth" runs build them
(ref validate.py:210-217), started from rest (solver.py:464-481 mode "rest").
Per-step PCG iteration counts must equal the oracle's; fields within 1e-4."""
import numpy as np
import pytest

from helpers import FIELDS, device_params, device_state, fields_of, ref_grid, rel_l2
from paper_2204_01117_b200 import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_interior_walls_match_oracle(prec):
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    from paper_2204_01117_b200.grid import to_ref_layout
    from paper_2204_01117_b200.linalg import build_ai_preconditioner, build_pressure_matrix
    doc = scenes.cuboid(32, 20, 8, 1.0, 0.1)
    doc["objects"] = []
    doc["solver"]["u_ref"] = 2.0
    doc["inlet"]["speed"] = 2.0
    sc = co.scene_from_dict(doc)
    g = sc.grid
    labels = co.classify_boundary(g, sc.faces)          # x-fastest (nz, ny, nx)
    labels[1:6, 7:13, 10:14] = 5                          # an interior no-slip block
    labels[1:3, 2:4, 20:26] = 5                           # and a low wall near the side
    phi, lad = np.ones(g.cshape), np.zeros(g.cshape)
    psys = co.build_pressure_matrix(g, labels)
    W = co.build_ai_preconditioner(psys.A, sc.ai_omega)
    ost = co.make_initial_state(g, labels, phi, lad, sc.params, sc.inlet, mode="rest")
    dtype = torch.float32 if prec == "fp32" else torch.float64
    dst = device_state(ost, dtype)
    dpsys = build_pressure_matrix(ref_grid(g), to_ref_layout(labels))
    dpre = build_ai_preconditioner(dpsys, sc.ai_omega, 1, truncate=False)
    p, prof = device_params(sc)
    want = []
    for _ in range(20):
        want.append(co.step(ost, sc.params, psys, W, sc.inlet).pcg.iterations)
    reps = solver.step_many(dst, p, dpsys, dpre, prof, 20)
    assert [r.pcg.iterations for r in reps] == want
    got = fields_of(dst)
    tol = 1e-4 if prec == "fp32" else 1e-9
    for n in FIELDS:
        assert rel_l2(got[n], getattr(ost, n)) <= tol, n
    # no-slip: every face touching a wall cell is zero
    u = got["u"]
    assert np.all(u[1:6, 7:13, 10:15] == 0.0)


def test_boundary_lists_follow_labels_changed_in_place():
    """The boundary writes replay per-labels lists (cw_capi.cu build_bc_lists):
    changing the labels of a state in place (same device tensor) must rebuild
    them -- the result equals the oracle's apply_boundary_conditions
    (solver.py:330-400) on the new labels, bit for bit in float64."""
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    doc = scenes.cuboid(24, 16, 8, 1.0, 0.1)
    doc["objects"] = []
    sc = co.scene_from_dict(doc)
    g = sc.grid
    labels = co.classify_boundary(g, sc.faces)
    phi, lad = np.ones(g.cshape), np.zeros(g.cshape)
    ost = co.make_initial_state(g, labels, phi, lad, sc.params, sc.inlet, mode="rest")
    rng = np.random.default_rng(5)
    for n in FIELDS:
        setattr(ost, n, rng.standard_normal(getattr(ost, n).shape))
    dst = device_state(ost, torch.float64)
    p, prof = device_params(sc)
    solver.apply_boundary_conditions(dst, prof, p)        # builds the lists for the first labels
    co.apply_boundary_conditions(ost, sc.inlet, sc.params)
    got = fields_of(dst)
    for n in FIELDS:
        np.testing.assert_array_equal(got[n], getattr(ost, n), err_msg=n)
    # new labels, written into the same device tensor: an interior wall block
    # and an outlet patch turned into wall
    lab2 = labels.copy()
    lab2[2:5, 5:9, 8:12] = 5
    lab2[-1, :, :4] = 5
    dst.labels_dev.copy_(torch.from_numpy(np.ascontiguousarray(lab2)).to(dst.labels_dev.device))
    ost.labels = lab2
    for n in FIELDS:
        a = rng.standard_normal(getattr(ost, n).shape)
        setattr(ost, n, a)
        dst.fields[n].copy_(torch.from_numpy(np.ascontiguousarray(a)))
    solver.apply_boundary_conditions(dst, prof, p)
    co.apply_boundary_conditions(ost, sc.inlet, sc.params)
    got = fields_of(dst)
    for n in FIELDS:
        np.testing.assert_array_equal(got[n], getattr(ost, n), err_msg=n)


def test_boundary_full_volume_path_without_labels_version(monkeypatch):
    """labels_version 0 (a C caller that does not version its labels) keeps
    the full-volume boundary kernels: same result as the oracle."""
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import _native as N
    from paper_2204_01117_b200 import solver
    monkeypatch.setattr(N, "labels_version", lambda t: 0)
    doc = scenes.cuboid(20, 12, 6, 1.0, 0.1)
    sc = co.scene_from_dict(doc)
    g = sc.grid
    labels = co.classify_boundary(g, sc.faces)
    labels[1:3, 3:6, 5:9] = 5
    ost = co.make_initial_state(g, labels, np.ones(g.cshape), np.zeros(g.cshape), sc.params, sc.inlet, mode="rest")
    rng = np.random.default_rng(9)
    for n in FIELDS:
        setattr(ost, n, rng.standard_normal(getattr(ost, n).shape))
    dst = device_state(ost, torch.float64)
    p, prof = device_params(sc)
    solver.apply_boundary_conditions(dst, prof, p)
    co.apply_boundary_conditions(ost, sc.inlet, sc.params)
    got = fields_of(dst)
    for n in FIELDS:
        np.testing.assert_array_equal(got[n], getattr(ost, n), err_msg=n)


@pytest.mark.parametrize("layout", ["all_outlets", "mixed", "random", "random_large"])
def test_composed_boundary_pass_equals_ordered_lists(layout, monkeypatch, capfd):
    """One boundary pass is ONE k_bc_replay launch of the lists' composition
    (cw_step.cuh k_bc_compose_*): with outlets on every side (every edge and
    corner where a later side reads or overwrites an earlier side's write),
    an inlet face, walls and a wall touching the outlets, the result equals
    the oracle's ordered apply_boundary_conditions (solver.py:330-400) and
    the ordered per-side launches (CW_BC_COMPOSE=0) bit for bit in float64,
    and bit for bit between the two paths in float32 -- also on a box whose
    edge lines carry more ordered writes than the replay's block 0 holds."""
    from oracle import citywind_oracle as co
    from paper_2204_01117_b200 import solver
    doc = scenes.cuboid(160, 160, 96, 1.0, 0.1) if layout == "random_large" else scenes.cuboid(22, 14, 9, 1.0, 0.1)
    sc = co.scene_from_dict(doc)
    g = sc.grid
    labels = co.classify_boundary(g, sc.faces)           # x-fastest (nz, ny, nx)
    monkeypatch.setenv("CW_BC_DEBUG", "1")
    if layout.startswith("random"):
        # random outlet / wall / inlet / air cells on every boundary layer:
        # edges where a later side's write does not cover an earlier side's
        # read, i.e. ordered writes in the composition
        rng = np.random.default_rng(7)
        lab = rng.choice(np.array([4, 4, 4, 5, 3, 0], np.int8), size=labels.shape)
        inner = (slice(1, -1),) * 3
        lab[inner] = labels[inner]
        labels = lab
    elif layout == "all_outlets":
        labels[:, :, 0] = 4
        labels[:, :, -1] = 4
        labels[:, 0, :] = 4
        labels[:, -1, :] = 4
        labels[0, :, :] = 4
        labels[-1, :, :] = 4
        labels[3:6, 4:8, 6:10] = 5
    else:
        labels[0, :, :] = 5
        labels[:, 0, 3:9] = 5                            # a wall strip on an outlet side
        labels[2:7, 5:9, 8:12] = 5
        labels[-1, :, :] = 4
    vals = {}
    for prec in ("fp64", "fp32"):
        for compose in ("1", "0"):
            monkeypatch.setenv("CW_BC_COMPOSE", compose)
            ost = co.make_initial_state(g, labels, np.ones(g.cshape), np.zeros(g.cshape), sc.params, sc.inlet,
                                        mode="rest")
            r2 = np.random.default_rng(11)
            for n in FIELDS:
                setattr(ost, n, r2.standard_normal(getattr(ost, n).shape))
            dst = device_state(ost, torch.float64 if prec == "fp64" else torch.float32)   # new labels tensor: lists rebuilt
            p, prof = device_params(sc)
            solver.apply_boundary_conditions(dst, prof, p)
            vals[prec, compose] = fields_of(dst)
            if prec == "fp64":
                co.apply_boundary_conditions(ost, sc.inlet, sc.params)
                for n in FIELDS:
                    np.testing.assert_array_equal(vals[prec, compose][n], getattr(ost, n), err_msg=f"{compose} {n}")
        for n in FIELDS:
            np.testing.assert_array_equal(vals[prec, "1"][n], vals[prec, "0"][n], err_msg=f"{prec} {n}")
    # random boundary labels make ordered writes (box-shaped outlet sides
    # make none: a later side always overwrites what it reads from an
    # earlier one); block 0 of the replay holds up to 2048 of them, the large
    # random box has more (a gather launch first)
    err = capfd.readouterr().err
    print(err)
    if layout.startswith("random"):
        assert "ordered" in err and " 0 ordered" not in err, err[-500:]
    if layout == "random_large":
        assert "gather launch" in err, err[-500:]
