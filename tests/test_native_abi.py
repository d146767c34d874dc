"""CPU-side checks of the C ABI: the library builds, loads without a GPU and
exports exactly the functions include/citywind_b200.h declares, and the
ctypes signature table covers each of them."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "citywind_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(cw_[a-z_0-9]+)\s*\(", src))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2204_01117_b200 import build, _native
    build.build()
    return _native.lib()


def test_header_declares_expected_entry_points():
    names = declared()
    for n in ("cw_ctx_create", "cw_set_operator", "cw_step", "cw_read_reports", "cw_voxelize",
              "cw_run_stage", "cw_region_speed", "cw_drag_coefficient"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for n in declared():
        assert hasattr(lib, n), n


def test_ctypes_table_matches_header():
    from paper_2204_01117_b200 import _native
    assert set(_native.SIGNATURES) == declared()


def test_abi_version(lib):
    assert lib.cw_abi_version() == 2


def test_context_creation_fails_loudly_without_gpu(lib):
    import ctypes as C
    import torch
    from paper_2204_01117_b200 import _native as N
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = N.cw_grid(8, 8, 8, 1.0, 1.0, 1.0, N.dbl3((0, 0, 0)))
    h = C.c_void_p()
    rc = lib.cw_ctx_create(C.byref(g), 4, 0, C.byref(h))
    assert rc != N.CW_OK
    assert "cuda" in N.last_error().lower() or "device" in N.last_error().lower()


def test_bad_arguments_are_rejected(lib):
    import ctypes as C
    from paper_2204_01117_b200 import _native as N
    h = C.c_void_p()
    g = N.cw_grid(0, 8, 8, 1.0, 1.0, 1.0, N.dbl3((0, 0, 0)))
    assert lib.cw_ctx_create(C.byref(g), 4, 0, C.byref(h)) == N.CW_ERR_INVALID
    g = N.cw_grid(8, 8, 8, 1.0, 1.0, 1.0, N.dbl3((0, 0, 0)))
    assert lib.cw_ctx_create(C.byref(g), 3, 0, C.byref(h)) == N.CW_ERR_INVALID
