"""Grid, labels, porosity and the device-resident flow state.

Mirrors the reference's ``citywind.grid`` interface (grid.py:19-130,
439-571): ``GridSpec``, ``CellLabel``, ``PorosityField``, ``classify_boundary``,
``merge_labels``, ``interior_mask`` and ``FlowState``.  The difference is
where the fields live: ``FlowState`` keeps u, v, w, p, k, omega, nu_t as
CUDA tensors in the x-fastest layout (torch shapes (nz, ny, nx[+1])); its
``u``/``v``/... attributes return host copies in the reference's C-order
(nx[+1], ny, nz) float64 layout and accept assignment of such arrays.
In-place edits of a returned host copy do not reach the device -- assign
the array back (``state.u = arr``) or edit ``state.fields['u']`` directly.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

import numpy as np
import torch


class CellLabel(IntEnum):
    AIR = 0
    BUILDING = 1
    TREE = 2
    INLET = 3
    OUTLET = 4
    SOLID_WALL = 5


INTERIOR_LABELS = (CellLabel.AIR, CellLabel.BUILDING, CellLabel.TREE)
BOUNDARY_LABELS = (CellLabel.INLET, CellLabel.OUTLET, CellLabel.SOLID_WALL)
FIELDS = ("u", "v", "w", "p", "k", "omega", "nu_t")


@dataclass(frozen=True)
class GridSpec:
    """Uniform staggered Cartesian grid; nz = 1 selects 2D mode (grid.py:33-84)."""

    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    origin: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise ValueError("cell counts must be >= 1")
        if min(self.dx, self.dy, self.dz) <= 0:
            raise ValueError("cell spacings must be > 0")

    @property
    def shape(self):
        return (self.nx, self.ny, self.nz)

    @property
    def n_cells(self):
        return self.nx * self.ny * self.nz

    @property
    def is_2d(self):
        return self.nz == 1

    @property
    def cell_volume(self):
        return self.dx * self.dy * self.dz

    @property
    def spacing(self):
        return np.array([self.dx, self.dy, self.dz])

    def axis_centers(self, axis):
        return self.origin[axis] + (np.arange(self.shape[axis]) + 0.5) * self.spacing[axis]

    def cell_centers(self):
        x, y, z = (self.axis_centers(a) for a in range(3))
        return np.stack(np.meshgrid(x, y, z, indexing="ij"), axis=-1)

    def extent(self):
        lo = np.asarray(self.origin, dtype=float)
        return lo, lo + self.spacing * np.array(self.shape)

    # device layout helpers -------------------------------------------------
    def dshape(self, name: str):
        nx, ny, nz = self.shape
        return {"u": (nz, ny, nx + 1), "v": (nz, ny + 1, nx), "w": (nz + 1, ny, nx)}.get(
            name, (nz, ny, nx))


@dataclass
class PorosityField:
    """phi in [0, 1] per cell (1 = open air) and LAD >= 0 (grid.py:87-105),
    host float64 in the reference layout (nx, ny, nz)."""

    phi: np.ndarray
    lad: np.ndarray

    @classmethod
    def open_air(cls, grid: GridSpec):
        return cls(np.ones(grid.shape), np.zeros(grid.shape))

    def validate(self):
        if np.any(self.phi < 0) or np.any(self.phi > 1):
            raise ValueError("phi outside [0, 1]")
        if np.any(self.lad < 0):
            raise ValueError("LAD must be >= 0")

    def copy(self):
        return PorosityField(self.phi.copy(), self.lad.copy())


def to_device_layout(a: np.ndarray) -> np.ndarray:
    """reference C-order (nx, ny, nz) -> x-fastest (nz, ny, nx)."""
    return np.ascontiguousarray(np.asarray(a).transpose(2, 1, 0))


def to_ref_layout(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).transpose(2, 1, 0))


_FACE_KEYS = ("x_min", "x_max", "y_min", "y_max", "z_min", "z_max")


def classify_boundary(grid: GridSpec, faces: dict) -> np.ndarray:
    """One-cell boundary layer from per-face assignments; edge/corner cells
    take the priority Inlet > SolidWall > Outlet (grid.py:439-470).  Host
    int8 labels in the reference layout."""
    required = _FACE_KEYS[:4] if grid.is_2d else _FACE_KEYS
    missing = [k for k in required if k not in faces]
    if missing:
        raise ValueError(f"missing boundary face assignment(s): {missing}")
    for key, lab in faces.items():
        if key not in _FACE_KEYS:
            raise ValueError(f"unknown face {key!r}")
        if CellLabel(lab) not in BOUNDARY_LABELS:
            raise ValueError(f"face {key} must be Inlet/Outlet/SolidWall, got {lab}")
    labels = np.zeros(grid.shape, dtype=np.int8)
    sel = {"x_min": np.s_[0:1, :, :], "x_max": np.s_[grid.nx - 1:, :, :],
           "y_min": np.s_[:, 0:1, :], "y_max": np.s_[:, grid.ny - 1:, :],
           "z_min": np.s_[:, :, 0:1], "z_max": np.s_[:, :, grid.nz - 1:]}
    for want in (CellLabel.OUTLET, CellLabel.SOLID_WALL, CellLabel.INLET):
        for key in required:
            if CellLabel(faces[key]) == want:
                labels[sel[key]] = int(want)
    return labels


def merge_labels(boundary: np.ndarray, interior: np.ndarray) -> np.ndarray:
    """Interior object labels under the boundary frame (grid.py:473-478)."""
    out = boundary.copy()
    m = (boundary == int(CellLabel.AIR)) & (interior != int(CellLabel.AIR))
    out[m] = interior[m]
    return out


def interior_mask(labels: np.ndarray) -> np.ndarray:
    """Cells that take part in the pressure solve (grid.py:481-484)."""
    return (labels == 0) | (labels == 1) | (labels == 2)


# ---------------------------------------------------------------------------
# painted porosity (grid.py:337-429): host raster I/O and the host decode; the
# device path feeds the raster to cw_set_paint + cw_voxelize instead

def read_pgm(path) -> np.ndarray:
    """Binary 8-bit PGM (P5) as a (rows, cols) uint8 array; row 0 = min-y row."""
    data = open(path, "rb").read()
    fields, pos = [], 0
    while len(fields) < 4:
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        if data[pos:pos + 1] == b"#":              # comment to end of line
            pos = data.find(b"\n", pos)
            pos = len(data) if pos < 0 else pos
            continue
        end = pos
        while end < len(data) and not data[end:end + 1].isspace():
            end += 1
        fields.append(data[pos:end])
        pos = end
    if fields[0] != b"P5":
        raise ValueError(f"not a binary PGM: magic {fields[0]!r}")
    w, h, maxval = (int(f) for f in fields[1:])
    if maxval != 255:
        raise ValueError(f"PGM depth must be 8-bit (maxval 255), got {maxval}")
    return np.frombuffer(data, dtype=np.uint8, count=w * h, offset=pos + 1).reshape(h, w)


def write_pgm(path, image: np.ndarray) -> None:
    image = np.asarray(image, dtype=np.uint8)
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n255\n" % (image.shape[1], image.shape[0]))
        fh.write(np.ascontiguousarray(image).tobytes())


def load_raster(path) -> np.ndarray:
    """PGM or 8-bit grayscale PNG (grid.py:419-429)."""
    if str(path).lower().endswith(".pgm"):
        return read_pgm(path)
    from PIL import Image
    img = Image.open(path)
    return np.asarray(img if img.mode == "L" else img.convert("L"), dtype=np.uint8)


def paint_planes(grid: "GridSpec", extrude_height) -> int:
    """Planes [0, kmax) that carry the paint (grid.py:365-369)."""
    if grid.is_2d or extrude_height is None:
        return grid.nz
    zc = grid.axis_centers(2) - grid.origin[2]
    return int(np.sum(zc <= extrude_height))


def decode_painted_porosity(image: np.ndarray, grid: "GridSpec", tree_mask=None, extrude_height=None,
                            tree_lad: float = 1.0):
    """Raster -> (labels, PorosityField) in the reference layout (grid.py:337-377):
    phi = pixel / 255 extruded over the painted planes; dark pixels BUILDING,
    tree-mask pixels TREE with LAD tree_lad."""
    image = np.asarray(image)
    if image.dtype != np.uint8:
        raise ValueError(f"painted porosity must be 8-bit, got {image.dtype}")
    if image.shape != (grid.ny, grid.nx):
        raise ValueError(f"raster shape {image.shape} != (ny, nx) = {(grid.ny, grid.nx)}")
    tree = np.zeros(image.shape, bool) if tree_mask is None else np.asarray(tree_mask) != 0
    if tree.shape != image.shape:
        raise ValueError("tree mask shape differs from image")
    phi2 = image.astype(np.float64).T / 255.0
    t2 = tree.T
    lab2 = np.where(t2, int(CellLabel.TREE), np.where((phi2 < 1.0) | t2, int(CellLabel.BUILDING),
                                                       int(CellLabel.AIR))).astype(np.int8)
    labels = np.full(grid.shape, int(CellLabel.AIR), np.int8)
    poros = PorosityField.open_air(grid)
    km = paint_planes(grid, extrude_height)
    labels[:, :, :km] = lab2[:, :, None]
    poros.phi[:, :, :km] = phi2[:, :, None]
    poros.lad[:, :, :km] = np.where(t2, float(tree_lad), 0.0)[:, :, None]
    return labels, poros


def encode_porosity_raster(poros: PorosityField, k: int = 0) -> np.ndarray:
    """One z-slice of phi as a (ny, nx) uint8 raster (grid.py:380-382)."""
    return np.round(poros.phi[:, :, k].T * 255.0).astype(np.uint8)


def default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2204_01117_b200 needs a CUDA device (B200); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


class FieldView(np.ndarray):
    """Reference-layout float64 host copy of one device field that writes
    through.  ``state.u`` in the reference is the live array: code such as
    ``arr = state.u; arr *= fac`` or ``state.k[i, j, k] = x`` mutates the
    state (reference solver.py:164-167).  Item assignment and in-place
    ufuncs on a FieldView (or any slice of it) therefore copy the whole
    field back to the device.  A view taken before the state was stepped is
    detached, as the reference's arrays are once ``step`` reassigns them
    (solver.py:423-425): writing to it no longer touches the state."""

    def _wt(self):
        return getattr(self, "_cw", None)

    def __array_finalize__(self, obj):
        if obj is not None and type(obj) is FieldView:
            self._cw = getattr(obj, "_cw", None)

    def _push(self):
        cw = self._wt()
        if cw is None:
            return
        state, name, root = cw
        if state._views.get(name, (None, None))[1] is root:   # still the state's live view
            state._set(name, root.view(np.ndarray), _touch=False)
            state._views[name] = (state._view_key(name), root)

    def __setitem__(self, key, value):
        np.ndarray.__setitem__(self.view(np.ndarray), key, value)
        self._push()

    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kwargs):
        plain = lambda a: a.view(np.ndarray) if isinstance(a, FieldView) else a  # noqa: E731
        args = [plain(a) for a in inputs]
        if out is not None:
            kwargs["out"] = tuple(plain(o) for o in out)
        res = getattr(ufunc, method)(*args, **kwargs)
        if out is not None:
            for o in out:
                if isinstance(o, FieldView):
                    o._push()
            return out[0] if len(out) == 1 else out
        return res


class FlowState:
    """Device-resident simulation state (grid.py:492-571).

    ``fields[name]`` are CUDA tensors in the x-fastest layout; ``labels_dev``
    is int8, ``phi_dev``/``lad_dev`` float64 (bit-exact voxelizer output).
    Attribute access ``state.u`` etc. returns a write-through reference-layout
    float64 copy (``FieldView``).
    """

    def __init__(self, grid: GridSpec, fields: dict, labels_dev, phi_dev, lad_dev,
                 time: float = 0.0, step_count: int = 0):
        self.grid = grid
        self.fields = fields
        self.labels_dev = labels_dev
        self.phi_dev = phi_dev
        self.lad_dev = lad_dev
        self.time = time
        self.step_count = step_count
        self._drag_key = None
        self._g = None
        self._has_drag = False
        self._version = 0
        self._views = {}

    def touch(self):
        """Mark the device fields as changed (a step or stage ran): field
        views taken before are detached from the state."""
        self._version += 1
        self._views.clear()

    def _view_key(self, name):
        return (self._version, self.fields[name]._version, self.fields[name].data_ptr())

    # construction ----------------------------------------------------------
    @classmethod
    def zeros(cls, grid: GridSpec, labels=None, porosity=None, k0: float = 1e-6,
              omega0: float = 1.0, dtype=torch.float32, device=None, static_dev=None):
        """Zero velocity and pressure, k0 / omega0 turbulence.  ``static_dev``:
        a (labels, phi, lad) device triple in the x-fastest layout (a device
        voxelizer's output), taken as is instead of ``labels`` / ``porosity``."""
        device = device or default_device()
        f = {}
        for n in FIELDS:
            t = torch.zeros(grid.dshape(n), dtype=dtype, device=device)
            f[n] = t
        f["k"].fill_(k0)
        f["omega"].fill_(omega0)
        f["nu_t"].fill_(k0 / omega0)
        if static_dev is not None:
            return cls(grid, f, *static_dev)
        lab = np.zeros(grid.shape, np.int8) if labels is None else np.asarray(labels, np.int8)
        por = PorosityField.open_air(grid) if porosity is None else porosity
        return cls(grid, f,
                   torch.from_numpy(to_device_layout(lab)).to(device),
                   torch.from_numpy(to_device_layout(np.asarray(por.phi, np.float64))).to(device),
                   torch.from_numpy(to_device_layout(np.asarray(por.lad, np.float64))).to(device))

    @property
    def device(self):
        return self.fields["u"].device

    @property
    def dtype(self):
        return self.fields["u"].dtype

    # reference-layout host views ---------------------------------------------
    def _get(self, name):
        return to_ref_layout(self.fields[name].detach().cpu().numpy().astype(np.float64))

    def _set(self, name, value, _touch=True):
        value = np.asarray(value, dtype=np.float64)
        shp = self.grid.dshape(name)[::-1]
        if value.shape != shp:
            value = np.broadcast_to(value, shp)
        self.fields[name].copy_(torch.from_numpy(to_device_layout(value)).to(self.dtype))
        if _touch:
            self.touch()

    def __getattr__(self, name):
        if name in FIELDS and "fields" in self.__dict__:
            # one live view per field while the device copy is unchanged, so
            # two reads alias like the reference's arrays
            key, arr = self._views.get(name, (None, None))
            if arr is None or key != self._view_key(name):
                arr = np.ascontiguousarray(self._get(name)).view(FieldView)
                arr._cw = (self, name, arr)
                self._views[name] = (self._view_key(name), arr)
            return arr
        raise AttributeError(name)

    def __setattr__(self, name, value):
        if name in FIELDS and "fields" in self.__dict__:
            self._set(name, value)
        else:
            object.__setattr__(self, name, value)

    @property
    def labels(self) -> np.ndarray:
        return to_ref_layout(self.labels_dev.cpu().numpy())

    @labels.setter
    def labels(self, value):
        self.labels_dev.copy_(torch.from_numpy(to_device_layout(np.asarray(value, np.int8))))
        self._drag_key = None

    @property
    def porosity(self) -> PorosityField:
        return PorosityField(to_ref_layout(self.phi_dev.cpu().numpy()),
                             to_ref_layout(self.lad_dev.cpu().numpy()))

    @porosity.setter
    def porosity(self, por: PorosityField):
        self.phi_dev.copy_(torch.from_numpy(to_device_layout(np.asarray(por.phi, np.float64))))
        self.lad_dev.copy_(torch.from_numpy(to_device_layout(np.asarray(por.lad, np.float64))))
        self._drag_key = None

    def __getstate__(self):
        d = dict(self.__dict__)
        d["_views"] = {}
        return d

    def copy(self) -> "FlowState":
        return FlowState(self.grid, {n: t.clone() for n, t in self.fields.items()},
                         self.labels_dev.clone(), self.phi_dev.clone(), self.lad_dev.clone(),
                         self.time, self.step_count)

    def validate(self):
        f = self.fields
        if bool((f["k"] < 0).any()):
            raise ValueError("negative turbulent kinetic energy")
        if bool((f["omega"] <= 0).any()):
            raise ValueError("non-positive specific dissipation")
        if bool((f["nu_t"] < 0).any()):
            raise ValueError("negative eddy viscosity")
        self.porosity.validate()

    def cell_velocity(self) -> np.ndarray:
        u, v, w = self.u, self.v, self.w
        return np.stack([0.5 * (u[:-1] + u[1:]), 0.5 * (v[:, :-1] + v[:, 1:]),
                         0.5 * (w[:, :, :-1] + w[:, :, 1:])], axis=-1)

    def speed(self) -> np.ndarray:
        vel = self.cell_velocity()
        return np.sqrt(np.sum(vel * vel, axis=-1))

    def to_host(self) -> dict:
        """All fields as reference-layout float64 arrays (one D2H per field)."""
        return {n: self._get(n) for n in FIELDS}
