"""Host logic of the reference-layout binding (paper_2204_01117_b200.refbind)
that needs no GPU: the reference objects it accepts (duck-typed) and how it
maps them -- preconditioner kinds, parameter and inlet conversion, the
reference-layout array shapes (grid.py:492-571)."""
import types

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2204_01117_b200 import refbind
from paper_2204_01117_b200.solver import InletProfile, SolverParams


def test_preconditioner_kinds():
    assert refbind._pre_kind(None, None, 1.65).kind == 0
    assert refbind._pre_kind(types.SimpleNamespace(name="jacobi"), None, 1.65).kind == 1
    A = sp.identity(4, format="csr") * 2.0
    W_full = sp.csr_matrix(np.ones((4, 4)))
    pre = refbind._pre_kind(types.SimpleNamespace(name="ai1", W=W_full), types.SimpleNamespace(A=A), 1.5)
    assert pre.kind == 2 and pre.omega == 1.5
    # a truncated AI1 (W on A's pattern) is not the device stencil: refused loudly
    with pytest.raises(NotImplementedError):
        refbind._pre_kind(types.SimpleNamespace(name="ai1", W=A.copy()), types.SimpleNamespace(A=A), 1.65)
    with pytest.raises(NotImplementedError):
        refbind._pre_kind(types.SimpleNamespace(name="ssor"), None, 1.65)
    IdentityPreconditioner = type("IdentityPreconditioner", (), {})
    assert refbind._pre_kind(IdentityPreconditioner(), None, 1.65).kind == 0


def test_params_and_profile_conversion():
    ref_params = types.SimpleNamespace(**{f: getattr(SolverParams(), f) for f in SolverParams.__dataclass_fields__})
    ref_params.dt = 0.123
    p = refbind._params(ref_params)
    assert isinstance(p, SolverParams) and p.dt == 0.123
    prof = types.SimpleNamespace(kind="logarithmic", speed=3.0, u_star=0.4, z0=0.5, kappa=0.41, direction=[0.8, 0.6])
    q = refbind._profile(prof)
    assert isinstance(q, InletProfile) and q.direction == (0.8, 0.6) and q.u_star == 0.4


def test_reference_layout_shapes():
    g = types.SimpleNamespace(nx=5, ny=4, nz=3)
    assert refbind._shape(g, "u") == (6, 4, 3)
    assert refbind._shape(g, "v") == (5, 5, 3)
    assert refbind._shape(g, "w") == (5, 4, 4)
    for n in ("p", "k", "omega", "nu_t"):
        assert refbind._shape(g, n) == (5, 4, 3)
    assert refbind.ORDER[:3] == ("u", "v", "w") and set(refbind.LATE) == {"nu_t", "p", "k", "omega"}
