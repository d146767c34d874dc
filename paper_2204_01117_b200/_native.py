"""ctypes binding of the C ABI in include/citywind_b200.h.

The shared library is built in-tree by ``paper_2204_01117_b200.build``.  There
is no CPU fallback: if the library is missing or no CUDA device is present,
every compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
import itertools
import os
import threading

import numpy as np

from .errors import (ClassificationError, NativeError, ProjectionError,
                     SingularSystemError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CW_LIB") or os.path.join(HERE, "libcitywind_b200.so")   # CW_LIB: developer variant builds

CW_OK, CW_ERR_INVALID, CW_ERR_CUDA, CW_ERR_SINGULAR, CW_ERR_PCG = 0, 1, 2, 3, 4
CW_ERR_NONFINITE, CW_ERR_TIMEOUT, CW_ERR_RHS, CW_ERR_GEOMETRY, CW_ERR_HALO = 5, 6, 7, 8, 9
STAGE_ADVECT, STAGE_DIFFUSE, STAGE_DRAG, STAGE_BOUNDARY, STAGE_PROJECT, STAGE_TURBULENCE = range(1, 7)


class cw_grid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("dx", C.c_double),
                ("dy", C.c_double), ("dz", C.c_double), ("origin", C.c_double * 3)]


class cw_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("dt", "nu", "cd_tree", "cd_building", "drag_a", "drag_b",
                                          "drag_eps", "c_mu", "alpha", "beta", "sigma",
                                          "sigma_star", "c_lim", "k_in", "omega_in")] + \
               [("turbulence", C.c_int)]


class cw_inlet(C.Structure):
    _fields_ = [("kind", C.c_int), ("speed", C.c_double), ("u_star", C.c_double),
                ("z0", C.c_double), ("kappa", C.c_double), ("dir_x", C.c_double),
                ("dir_y", C.c_double)]


class cw_fields(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("u", "v", "w", "p", "k", "omega", "nu_t", "labels", "g")] + \
               [("has_drag", C.c_int), ("labels_version", C.c_longlong)]


_LABEL_UIDS = itertools.count(1)


def labels_version(t) -> int:
    """A key that changes whenever the content of the labels tensor ``t`` may
    have changed: a process-unique id stamped on the tensor object (a new
    tensor at a recycled address gets a new id) and torch's in-place version
    counter.  The context keys its boundary-write lists on it."""
    if t is None:
        return 0
    uid = getattr(t, "_cw_uid", None)
    if uid is None:
        uid = next(_LABEL_UIDS)
        t._cw_uid = uid
    return (uid << 24) | (int(t._version) & 0xFFFFFF)


class cw_report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("status", C.c_int),
                ("bad_field", C.c_int), ("criterion", C.c_double), ("cfl", C.c_double),
                ("div_before", C.c_double), ("div_after", C.c_double),
                ("bad_cell", C.c_longlong), ("ms_total", C.c_float)]


class cw_object(C.Structure):
    _fields_ = [("kind", C.c_int), ("shape", C.c_int), ("phi", C.c_double), ("lad", C.c_double),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("vert_offset", C.c_int),
                ("n_verts", C.c_int), ("tri_offset", C.c_int), ("n_tris", C.c_int)]


class cw_slab_buffers(C.Structure):
    _fields_ = [("r0", C.c_void_p), ("r1", C.c_void_p), ("p0", C.c_void_p), ("p1", C.c_void_p),
                ("z", C.c_void_p), ("Ap", C.c_void_p), ("xbar", C.c_void_p), ("xval", C.c_void_p),
                ("o0", C.c_int), ("o1", C.c_int)]

    BUFFERS = ("r0", "r1", "p0", "p1", "z", "Ap", "xbar", "xval")


CW_STAGE_PRE, CW_STAGE_POST, CW_STAGE_SOLVE = 7, 8, 9
CW_MAX_SLABS = 64

# exported symbol -> (restype, argtypes); must match include/citywind_b200.h
_P = C.c_void_p
SIGNATURES = {
    "cw_abi_version": (C.c_int, []),
    "cw_last_error": (C.c_char_p, []),
    "cw_ctx_create": (C.c_int, [C.POINTER(cw_grid), C.c_int, C.c_int, C.POINTER(_P)]),
    "cw_ctx_destroy": (None, [_P]),
    "cw_ctx_create_slab": (C.c_int, [C.POINTER(cw_grid), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(_P)]),
    "cw_slab_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.POINTER(C.c_int)]),
    "cw_operator_partials": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_longlong), C.POINTER(C.c_int)]),
    "cw_slab_buffers_get": (C.c_int, [_P, C.POINTER(cw_slab_buffers)]),
    "cw_slab_attach": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(cw_slab_buffers),
                                 C.POINTER(cw_slab_buffers), C.POINTER(cw_slab_buffers)]),
    "cw_slab_group_pcg": (C.c_int, [C.POINTER(_P), C.POINTER(cw_fields), C.c_int, C.POINTER(cw_params),
                                    C.c_double, _P]),
    "cw_ipc_get": (C.c_int, [_P, C.POINTER(C.c_ubyte)]),
    "cw_ipc_open": (C.c_int, [C.POINTER(C.c_ubyte), C.c_int, C.POINTER(_P)]),
    "cw_ipc_close": (C.c_int, [_P]),
    "cw_set_paint": (C.c_int, [_P, _P, _P, C.c_int, C.c_double]),
    "cw_probe": (C.c_int, [_P, C.POINTER(cw_fields), C.c_int, _P, _P, _P]),
    "cw_streamlines": (C.c_int, [_P, C.POINTER(cw_fields), C.c_int, _P, C.c_double, C.c_int, C.c_double,
                                 _P, _P, _P]),
    "cw_set_operator": (C.c_int, [_P, _P, C.c_double, C.POINTER(C.c_longlong),
                                  C.POINTER(C.c_double), _P]),
    "cw_set_preconditioner": (C.c_int, [_P, C.c_int, C.POINTER(C.c_double)]),
    "cw_drag_coefficient": (C.c_int, [_P, _P, _P, _P, C.POINTER(cw_params), _P,
                                      C.POINTER(C.c_int), _P]),
    "cw_apply_boundary": (C.c_int, [_P, C.POINTER(cw_fields), C.POINTER(cw_params),
                                    C.POINTER(cw_inlet), _P]),
    "cw_step": (C.c_int, [_P, C.POINTER(cw_fields), C.POINTER(cw_params), C.POINTER(cw_inlet),
                          C.c_double, C.c_int, _P]),
    "cw_run_stage": (C.c_int, [_P, C.POINTER(cw_fields), C.POINTER(cw_params), C.POINTER(cw_inlet),
                               C.c_int, C.c_double, _P]),
    "cw_read_reports": (C.c_int, [_P, C.POINTER(cw_report), C.c_int, C.POINTER(C.c_int), _P]),
    "cw_step_defer": (C.c_int, [_P, _P, _P]),
    "cw_step_defer_kw": (C.c_int, [_P, _P]),
    "cw_set_max_iter": (C.c_int, [_P, C.c_int]),
    "cw_pcg_chunk_of": (C.c_int, [C.POINTER(cw_grid), C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "cw_set_pcg_chunk": (C.c_int, [_P, C.c_int]),
    "cw_slab_chunks": (C.c_int, [_P, C.c_int, C.c_int]),
    "cw_pcg_chunks": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "cw_ref_layout": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, _P]),
    "cw_turb_rollback": (C.c_int, [_P, C.POINTER(cw_fields), _P]),
    "cw_proj_rollback": (C.c_int, [_P, C.POINTER(cw_fields), C.c_int, _P]),
    "cw_set_stage_timing": (C.c_int, [_P, C.c_int]),
    "cw_read_stage_timings": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "cw_pcg_timing": (C.c_int, [_P, C.c_int]),
    "cw_read_pcg_timing": (C.c_int, [_P, C.POINTER(C.c_float), C.c_int, C.POINTER(C.c_int)]),
    "cw_read_adv_timing": (C.c_int, [_P, C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int,
                                     C.POINTER(C.c_int)]),
    "cw_launch_count": (C.c_longlong, [_P, C.c_int]),
    "cw_region_speed": (C.c_int, [_P, C.POINTER(cw_fields), C.c_int, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_longlong), _P]),
    "cw_step_regions": (C.c_int, [_P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), _P, _P]),
    "cw_voxelize": (C.c_int, [_P, C.POINTER(cw_object), C.c_int, C.POINTER(C.c_double),
                              C.POINTER(C.c_int), C.c_int, _P, _P, _P, _P, C.POINTER(C.c_int), _P]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load the extension (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                        "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
                h = C.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(h, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = h
    return _lib


def last_error() -> str:
    return lib().cw_last_error().decode(errors="replace")


def check(rc: int, report=None):
    if rc == CW_OK:
        return
    msg = last_error()
    if rc == CW_ERR_SINGULAR:
        raise SingularSystemError(msg)
    if rc == CW_ERR_PCG:
        raise ProjectionError(report)
    if rc == CW_ERR_NONFINITE:
        raise FloatingPointError(msg)
    if rc in (CW_ERR_INVALID, CW_ERR_RHS, CW_ERR_HALO):
        raise ValueError(msg)
    if rc == CW_ERR_GEOMETRY:
        raise ClassificationError(msg)
    raise NativeError(f"citywind_b200 error {rc}: {msg}")


def ptr(t) -> int:
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else t.data_ptr()


def dbl3(a) -> C.Array:
    return (C.c_double * 3)(*[float(x) for x in a])


def as_cdouble_array(a: np.ndarray):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def c_stream(stream) -> C.c_void_p:
    """The cudaStream_t of a torch stream, for the C ABI's `void *stream`."""
    return C.c_void_p(stream.cuda_stream)
