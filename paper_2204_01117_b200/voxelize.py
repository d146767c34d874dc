"""Device voxelizer entry (reference ``citywind.grid.voxelize``, grid.py:233-325).

``voxelize_device`` packs the objects (boxes as exact (lo, hi); cylinders and
OBJ meshes as triangle lists) and calls ``cw_voxelize``, which computes the
per-cell porosity phi, LAD and labels on the GPU bit-exactly, combines them
with the open-air layer (scenario.py:351-360) and overlays them under the
boundary frame (grid.py:473-478).
"""
from __future__ import annotations

import ctypes as C
import threading
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .geometry import TriangleMesh
from .grid import CellLabel, GridSpec, to_device_layout


@dataclass
class GridObject:
    """One building or tree: a closed mesh or an exact axis box (grid.py:108-130)."""

    kind: CellLabel
    mesh: TriangleMesh | None = None
    box: tuple | None = None
    phi: float = 0.0
    lad: float = 0.0
    name: str = ""

    def __post_init__(self):
        if (self.mesh is None) == (self.box is None):
            raise ValueError("GridObject needs exactly one of mesh or box")
        if self.kind not in (CellLabel.BUILDING, CellLabel.TREE):
            raise ValueError("object kind must be Building or Tree")
        if not 0.0 <= self.phi <= 1.0:
            raise ValueError("object phi must be in [0, 1]")
        if self.lad < 0:
            raise ValueError("object LAD must be >= 0")


_paint_lock = threading.Lock()


def voxelize_device(ctx, objects, grid: GridSpec, subdiv: int, boundary_dev: torch.Tensor, paint=None):
    """Returns (labels_dev int8, phi_dev float64, lad_dev float64) in the
    x-fastest layout; labels already merged with the boundary labels.
    ``paint``: optional base layer (image uint8 (ny, nx) device tensor, tree
    mask or None, kmax, tree_lad) under the objects (scenario.py:402-412)."""
    if paint is not None:
        img, mask, kmax, tree_lad = paint
        with _paint_lock:   # the paint lives in the shared voxelizer context for this call only
            N.check(N.lib().cw_set_paint(ctx.h, N.ptr(img), N.ptr(mask), int(kmax), float(tree_lad)))
            try:
                return voxelize_device(ctx, objects, grid, subdiv, boundary_dev)
            finally:
                torch.cuda.current_stream(boundary_dev.device).synchronize()
                N.check(N.lib().cw_set_paint(ctx.h, None, None, 0, 1.0))
    if not 1 <= subdiv <= 8:
        raise ValueError("subdiv must be in [1, 8]")
    device = boundary_dev.device
    objs = (N.cw_object * max(len(objects), 1))()
    verts, tris = [], []
    nv = nt = 0
    for n, ob in enumerate(objects):
        o = objs[n]
        o.kind = int(ob.kind)
        o.phi = float(ob.phi)
        o.lad = float(ob.lad)
        if ob.mesh is not None:
            ob.mesh.validate_closed()
            o.shape = 1
            o.vert_offset, o.n_verts = nv, len(ob.mesh.vertices)
            o.tri_offset, o.n_tris = nt, len(ob.mesh.triangles)
            verts.append(np.asarray(ob.mesh.vertices, np.float64))
            tris.append(np.asarray(ob.mesh.triangles, np.int32))
            nv += o.n_verts
            nt += o.n_tris
        else:
            o.shape = 0
            lo, hi = ob.box
            o.lo = N.dbl3(lo)
            o.hi = N.dbl3(hi)
    vbuf = np.ascontiguousarray(np.concatenate(verts) if verts else np.zeros((1, 3)), np.float64)
    tbuf = np.ascontiguousarray(np.concatenate(tris) if tris else np.zeros((1, 3), np.int32), np.int32)
    shape = grid.dshape("p")
    labels = torch.empty(shape, dtype=torch.int8, device=device)
    phi = torch.empty(shape, dtype=torch.float64, device=device)
    lad = torch.empty(shape, dtype=torch.float64, device=device)
    nwarn = C.c_int()
    N.check(N.lib().cw_voxelize(ctx.h, objs, len(objects), vbuf.ctypes.data_as(C.POINTER(C.c_double)),
                                tbuf.ctypes.data_as(C.POINTER(C.c_int)), int(subdiv), N.ptr(boundary_dev),
                                N.ptr(labels), N.ptr(phi), N.ptr(lad), C.byref(nwarn), ctx.stream))
    if nwarn.value:
        warnings.warn(f"overlapping Building/Tree objects in {nwarn.value} cell(s); "
                      "keeping the lower-phi kind", stacklevel=3)
    return labels, phi, lad


def voxelize(objects, grid: GridSpec, subdiv: int = 4, device=None):
    """Reference-shaped convenience API: host (labels, PorosityField) in the
    reference layout, computed on the device (no boundary frame)."""
    from .grid import PorosityField, default_device, to_ref_layout
    from .runtime import Context
    device = device or default_device()
    ctx = Context(grid, torch.float32, device)
    bnd = torch.zeros(grid.dshape("p"), dtype=torch.int8, device=device)
    lab, phi, lad = voxelize_device(ctx, objects, grid, subdiv, bnd)
    return (to_ref_layout(lab.cpu().numpy()),
            PorosityField(to_ref_layout(phi.cpu().numpy()), to_ref_layout(lad.cpu().numpy())))


__all__ = ["GridObject", "voxelize", "voxelize_device", "to_device_layout"]
