"""The appendix preconditioner benchmark on the host (SURVEY 8f-4,
paper_2204_01117_b200/zoo.py): the reference's own unit tests for these
functions (reference tests/test_linalg.py TestJacobiAndReferences, TestPcg,
TestConditionNumber) restated, the benchmark matrix against the oracle's
assembly, and the benchmark's condition numbers and iteration counts
against the unmodified reference's (tests/golden/zoo_small.json,
scripts/make_golden_zoo.py)."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
from threadpoolctl import threadpool_limits

from helpers import GOLD
from paper_2204_01117_b200 import zoo
from paper_2204_01117_b200.grid import CellLabel, GridSpec
from paper_2204_01117_b200.linalg import build_pressure_matrix


def _karman(nx, ny):
    """A 2-D channel: inlet at x = 0, outlet at x = nx - 1, walls at y = 0, ny - 1."""
    g = GridSpec(nx, ny, 1, 1.0, 1.0, 1.0)
    lab = np.zeros(g.shape, np.int8)
    lab[0, :, :] = int(CellLabel.INLET)
    lab[-1, :, :] = int(CellLabel.OUTLET)
    lab[:, 0, :] = int(CellLabel.SOLID_WALL)
    lab[:, -1, :] = int(CellLabel.SOLID_WALL)
    lab[3:5, ny // 2 - 1:ny // 2 + 1, :] = int(CellLabel.SOLID_WALL)   # an obstacle
    return zoo.assemble_pressure_matrix(build_pressure_matrix(g, lab))


def test_assembly_matches_oracle():
    from oracle import citywind_oracle as co
    g = GridSpec(9, 7, 5, 1.0, 0.5, 2.0)
    rng = np.random.default_rng(1)
    lab = rng.choice(np.array([0, 0, 0, 1, 2, 3, 4, 5], np.int8), size=g.shape)
    lab[-1, :, :] = int(CellLabel.OUTLET)
    A = zoo.assemble_pressure_matrix(build_pressure_matrix(g, lab))
    og = co.Grid(9, 7, 5, 1.0, 0.5, 2.0)
    B = co.build_pressure_matrix(og, np.ascontiguousarray(lab.transpose(2, 1, 0))).A
    assert A.shape == B.shape
    assert abs(A - B).max() == 0.0


def test_ssor_apply_matches_dense():
    A = _karman(16, 16)
    omega = 1.3
    pre = zoo.build_reference_preconditioner(A, "ssor", omega=omega)
    Ad = A.toarray()
    D = np.diag(np.diag(Ad))
    L = np.tril(Ad, -1)
    M = (D / omega + L) @ np.linalg.inv(D / omega) @ (D / omega + L).T / (2 - omega)
    r = np.random.default_rng(3).standard_normal(A.shape[0])
    np.testing.assert_allclose(pre.apply(r), np.linalg.solve(M, r), rtol=1e-10)


def test_ic_factor_reproduces_a_on_its_pattern():
    A = _karman(10, 10)
    G = zoo.build_reference_preconditioner(A, "ic").G.toarray()
    mask = A.toarray() != 0
    np.testing.assert_allclose((G @ G.T)[mask], A.toarray()[mask], atol=1e-10)


def test_mic_moves_dropped_fill_to_the_diagonal():
    A = _karman(10, 10)
    ic = zoo.build_reference_preconditioner(A, "ic").G.toarray()
    mic = zoo.build_reference_preconditioner(A, "mic", mic_tau=1.0).G.toarray()
    # full modification preserves the row sums of A (the dropped fill is lumped)
    np.testing.assert_allclose((mic @ mic.T).sum(axis=1), A.toarray().sum(axis=1), atol=1e-9)
    assert not np.allclose(ic, mic)


def test_ic_breakdown_names_row_and_size_guard():
    with pytest.raises(ValueError, match="row"):
        zoo.build_reference_preconditioner(sp.csr_matrix(np.array([[1.0, 2.0], [2.0, 1.0]])), "ic")
    with pytest.raises(ValueError):
        zoo.build_reference_preconditioner(sp.identity(200_000, format="csr"), "ssor")
    with pytest.raises(ValueError):
        zoo.build_reference_preconditioner(sp.identity(4, format="csr"), "ilut")


def test_pcg_cases():
    A = sp.identity(10, format="csr")
    x, rep = zoo.pcg_solve(A, np.arange(10.0), tol=1e-12)
    assert rep.iterations <= 1 and rep.converged
    np.testing.assert_allclose(x, np.arange(10.0))
    x, rep = zoo.pcg_solve(sp.identity(5, format="csr"), np.zeros(5))
    assert rep.iterations == 0 and rep.converged
    rng = np.random.default_rng(8)
    B = rng.standard_normal((50, 50))
    A = sp.csr_matrix(B @ B.T + 50 * np.eye(50))
    b = rng.standard_normal(50)
    x, rep = zoo.pcg_solve(A, b, tol=1e-16, max_iter=500)
    assert rep.converged
    np.testing.assert_allclose(x, np.linalg.solve(A.toarray(), b), rtol=1e-6)
    _, rep = zoo.pcg_solve(_karman(16, 24), np.ones(_karman(16, 24).shape[0]), tol=1e-30, max_iter=3)
    assert not rep.converged and rep.iterations == 3


def test_condition_numbers_against_dense():
    A = sp.diags([1.0, 100.0]).tocsr()
    assert zoo.estimate_condition_number(A) == pytest.approx(100.0, rel=1e-6)
    A = _karman(12, 16)
    ev = np.linalg.eigvalsh(A.toarray())
    assert zoo.estimate_condition_number(A) == pytest.approx(ev[-1] / ev[0], rel=0.05)
    pre = zoo.jacobi_matrix(A)
    Dh = np.diag(1.0 / np.sqrt(A.diagonal()))
    ev = np.linalg.eigvalsh(Dh @ A.toarray() @ Dh)
    assert zoo.estimate_condition_number(A, pre) == pytest.approx(ev[-1] / ev[0], rel=0.05)
    A = _karman(8, 10)
    pre = zoo.ai_matrix(A, 1.65, 1, truncate=False)
    sv = np.linalg.svd(pre.W.toarray() @ A.toarray(), compute_uv=False)
    assert zoo.estimate_condition_number(A, pre, norm="2") == pytest.approx(sv[0] / sv[-1], rel=0.05)


def test_benchmark_matches_reference():
    """validate.bench_preconditioners("small") and omega_sweep("small") of
    the unmodified reference: the same benchmark matrix and preconditioner
    matrices (bitwise, scripts/make_golden_zoo.py checked them), so the
    iteration counts agree exactly and the condition numbers (AI1, MIC and
    one omega-sweep point here; ~10 s each) to 1e-6."""
    path = os.path.join(GOLD, "zoo_small.json")
    if not os.path.exists(path):
        pytest.skip("golden not generated")
    with open(path) as fh:
        gold = json.load(fh)
    with threadpool_limits(limits=1):   # numpy may have loaded OpenBLAS before conftest pinned its threads
        A = zoo.benchmark_matrix("small")
        b = np.random.default_rng(0).standard_normal(A.shape[0])
        pres = {"cg": None, "jacobi": zoo.jacobi_matrix(A), "ai1": zoo.ai_matrix(A, 1.65, 1, truncate=False),
                "ai2": zoo.ai_matrix(A, 1.65, 2, truncate=False),
                "ssor": zoo.build_reference_preconditioner(A, "ssor", omega=zoo.SSOR_BENCH_OMEGA),
                "ic": zoo.build_reference_preconditioner(A, "ic"),
                "mic": zoo.build_reference_preconditioner(A, "mic")}
        for row in gold["bench"]:
            _, rep = zoo.pcg_solve(A, b, pres[row["preconditioner"]], tol=1e-5, max_iter=20_000)
            assert rep.iterations == row["iterations"], row
        for row in gold["bench"]:
            if row["preconditioner"] in ("ai1", "mic"):
                k = zoo.estimate_condition_number(A, pres[row["preconditioner"]], norm="2", max_iter=400)
                assert k == pytest.approx(row["kappa"], rel=1e-6), row
        om, kg = gold["omega_sweep"][5]
        k = zoo.estimate_condition_number(A, zoo.ai_matrix(A, om, 1, truncate=False), norm="2")
        assert k == pytest.approx(kg, rel=1e-6)
