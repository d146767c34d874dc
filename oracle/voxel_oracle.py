"""CPU ORACLE for the porosity voxelizer -- TEST INFRASTRUCTURE ONLY.

numpy restatement of the reference voxelizer path:
  scenario.py:327-360,383-417 (design bindings, object instantiation, layer merge)
  grid.py:337-377,385-429 (painted-porosity base layer, PGM/PNG rasters)
  grid.py:133-141,144-211,214-230,233-325,473-478 (candidates, column casts,
      exact box coverage, sample merge, labels)
  geometry.py:145-241,301-316 (batch ray casts, point queries, cylinder mesh)
Outputs are x-fastest (nz, ny, nx) arrays: int8 labels, float64 phi and LAD.
Every floating-point expression keeps the reference's operation order, and
the per-cell sample mean uses np.mean exactly as the reference does
(grid.py:316,319), so the result is bit-identical to the reference (pinned by
tests/test_oracle_golden.py against fixtures made from the reference).
The painted-porosity layer is pinned by the paint_city golden
(scripts/make_golden.py writes its raster into the fixture).
"""
from __future__ import annotations

import hashlib
import warnings

import numpy as np

from oracle.citywind_oracle import AIR, BUILDING, TREE, merge_labels

EPS_PARALLEL = 1e-10
EPS_BARY = 1e-10
EPS_T = 1e-9
_PRIMARY = np.array([0.285601, 0.571808, 0.769137])
_PRIMARY = _PRIMARY / np.linalg.norm(_PRIMARY)


class ClassificationError(RuntimeError):
    pass


# --- meshes (geometry.py:276-316) ------------------------------------------

def cylinder_mesh(center, radius, z0, z1, segments=48):
    cx, cy = center
    ang = np.linspace(0.0, 2 * np.pi, segments, endpoint=False)
    rx = cx + radius * np.cos(ang)
    ry = cy + radius * np.sin(ang)
    verts = np.concatenate([np.stack([rx, ry, np.full(segments, float(z0))], 1),
                            np.stack([rx, ry, np.full(segments, float(z1))], 1),
                            np.array([[cx, cy, z0], [cx, cy, z1]], dtype=float)])
    i = np.arange(segments)
    j = (i + 1) % segments
    cb, ct = 2 * segments, 2 * segments + 1
    tris = np.stack([np.stack([i, j, segments + j], 1),
                     np.stack([i, segments + j, segments + i], 1),
                     np.stack([np.full(segments, cb), j, i], 1),
                     np.stack([np.full(segments, ct), segments + i, segments + j], 1)],
                    1).reshape(-1, 3)
    return verts, tris


def box_mesh(lo, hi):
    (x0, y0, z0), (x1, y1, z1) = np.asarray(lo, float), np.asarray(hi, float)
    v = np.array([[x0, y0, z0], [x1, y0, z0], [x1, y1, z0], [x0, y1, z0],
                  [x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]])
    quads = [(0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (2, 3, 7, 6), (0, 4, 7, 3), (1, 2, 6, 5)]
    t = []
    for a, b, c, d in quads:
        t += [[a, b, c], [a, c, d]]
    return v, np.array(t)


def _corners(verts, tris):
    return verts[tris[:, 0]], verts[tris[:, 1]], verts[tris[:, 2]]


# --- point queries (geometry.py:145-241) -----------------------------------

def cast_batch(points, direction, verts, tris):
    v0, v1, v2 = _corners(verts, tris)
    e1, e2 = v1 - v0, v2 - v0
    nrm = np.cross(e1, e2)
    area2 = np.linalg.norm(nrm, axis=1)
    ok = area2 * 0.5 > 1e-12
    v0, e1, e2, nrm, area2 = v0[ok], e1[ok], e2[ok], nrm[ok], area2[ok]
    counts = np.zeros(len(points), np.int64)
    amb = np.zeros(len(points), bool)
    if len(v0) == 0:
        return counts, amb
    pvec = np.cross(direction, e2)
    det = np.einsum("tj,tj->t", e1, pvec)
    par = np.abs(det) <= EPS_PARALLEL * area2
    sdet = np.where(par, 1.0, det)
    chunk = max(1, int(4_000_000 // len(v0)))
    for lo in range(0, len(points), chunk):
        p = points[lo:lo + chunk]
        tv = p[:, None, :] - v0[None, :, :]
        u = np.einsum("ntj,tj->nt", tv, pvec) / sdet
        q = np.cross(tv, e1[None, :, :])
        v = np.einsum("ntj,j->nt", q, direction) / sdet
        t = np.einsum("ntj,tj->nt", q, e2) / sdet
        w = 1.0 - u - v
        loose = (u >= -EPS_BARY) & (v >= -EPS_BARY) & (w >= -EPS_BARY)
        hit = ~par[None, :] & loose & (t > EPS_T)
        gr = ~par[None, :] & loose & ((u <= EPS_BARY) | (v <= EPS_BARY) | (w <= EPS_BARY)
                                      | (np.abs(t) <= EPS_T))
        pd = np.abs(np.einsum("ntj,tj->nt", tv, nrm)) / area2
        gr |= par[None, :] & (pd <= EPS_T)
        counts[lo:lo + chunk] = hit.sum(axis=1)
        amb[lo:lo + chunk] = gr.any(axis=1)
    return counts, amb


def retry_direction(point, attempt):
    key = np.asarray(point, dtype=np.float64).tobytes() + attempt.to_bytes(4, "little")
    seed = int.from_bytes(hashlib.blake2b(key, digest_size=8).digest(), "little")
    d = np.random.default_rng(seed).normal(size=3)
    return d / np.linalg.norm(d)


def points_in_mesh(points, verts, tris, max_retries=8, stats=None):
    points = np.atleast_2d(np.asarray(points, float))
    res = np.zeros(len(points), bool)
    lo, hi = verts.min(axis=0) - EPS_T, verts.max(axis=0) + EPS_T
    act = np.all((points >= lo) & (points <= hi), axis=1)
    if not act.any():
        return res
    idx = np.nonzero(act)[0]
    c, amb = cast_batch(points[idx], _PRIMARY, verts, tris)
    res[idx] = c % 2 == 1
    for attempt in range(1, max_retries + 1):
        bad = idx[amb]
        if len(bad) == 0:
            return res
        if stats is not None:
            stats["recasts"] = stats.get("recasts", 0) + len(bad)
        still = np.zeros(len(bad), bool)
        for n, i in enumerate(bad):
            cc, aa = cast_batch(points[i:i + 1], retry_direction(points[i], attempt), verts, tris)
            res[i] = cc[0] % 2 == 1
            still[n] = aa[0]
        idx, amb = bad, still
    if amb.any():
        raise ClassificationError(f"{int(amb.sum())} point(s) unclassifiable")
    return res


# --- column classification (grid.py:144-211) -------------------------------

def classify_columns(verts, tris, xs, ys, zs, stats=None):
    """inside flags (len(xs), len(ys), len(zs)) by +z column casts."""
    v0, v1, v2 = _corners(verts, tris)
    e1, e2 = v1 - v0, v2 - v0
    det = e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]
    scale = np.maximum(np.abs(e1[:, 0] * e2[:, 1]) + np.abs(e1[:, 1] * e2[:, 0]), 1e-300)
    vert = np.abs(det) <= 1e-12 * scale
    sdet = np.where(vert, 1.0, det)
    xy = np.stack([v0[:, :2], v1[:, :2], v2[:, :2]])
    tlo, thi = xy.min(axis=0), xy.max(axis=0)
    ncx, ncy, nz = len(xs), len(ys), len(zs)
    cols = np.stack(np.meshgrid(xs, ys, indexing="ij"), axis=-1).reshape(-1, 2)
    inside = np.zeros((len(cols), nz), bool)
    ambiguous = np.zeros(len(cols), bool)
    chunk = max(1, int(4_000_000 // max(len(v0), 1)))
    for lo in range(0, len(cols), chunk):
        p = cols[lo:lo + chunk]
        px, py = p[:, 0:1], p[:, 1:2]
        rx = px - v0[None, :, 0]
        ry = py - v0[None, :, 1]
        u = (rx * e2[None, :, 1] - ry * e2[None, :, 0]) / sdet
        v = (ry * e1[None, :, 0] - rx * e1[None, :, 1]) / sdet
        w = 1.0 - u - v
        loose = (u >= -EPS_BARY) & (v >= -EPS_BARY) & (w >= -EPS_BARY) & ~vert[None, :]
        graze = loose & ((u <= EPS_BARY) | (v <= EPS_BARY) | (w <= EPS_BARY))
        near = vert[None, :] & (px >= tlo[None, :, 0] - EPS_T) & (px <= thi[None, :, 0] + EPS_T) \
            & (py >= tlo[None, :, 1] - EPS_T) & (py <= thi[None, :, 1] + EPS_T)
        amb = graze.any(axis=1) | near.any(axis=1)
        zc = v0[None, :, 2] + u * e1[None, :, 2] + v * e2[None, :, 2]
        for n in range(len(p)):
            row = lo + n
            if amb[n]:
                ambiguous[row] = True
                continue
            cr = np.sort(zc[n][loose[n]])
            if cr.size and np.min(np.abs(cr[None, :] - zs[:, None])) <= EPS_T:
                ambiguous[row] = True
                continue
            inside[row] = ((cr.size - np.searchsorted(cr, zs)) % 2) == 1
    if ambiguous.any():
        rows = np.nonzero(ambiguous)[0]
        if stats is not None:
            stats["fallback_columns"] = stats.get("fallback_columns", 0) + len(rows)
        pts = np.empty((len(rows) * nz, 3))
        pts[:, 0] = np.repeat(cols[rows, 0], nz)
        pts[:, 1] = np.repeat(cols[rows, 1], nz)
        pts[:, 2] = np.tile(zs, len(rows))
        inside[rows] = points_in_mesh(pts, verts, tris, stats=stats).reshape(len(rows), nz)
    return inside.reshape(ncx, ncy, nz)


# --- voxelize (grid.py:214-325) --------------------------------------------

def _centers(grid, axis):
    return grid.origin[axis] + (np.arange(grid.n(axis)) + 0.5) * grid.h(axis)


def box_coverage_axes(grid, lo, hi):
    """per-axis clipped overlap fractions (grid.py:221-227)."""
    fr = []
    for a in range(3):
        h = grid.h(a)
        cell_lo = _centers(grid, a) - 0.5 * h
        ov = np.minimum(hi[a], cell_lo + h) - np.maximum(lo[a], cell_lo)
        fr.append(np.clip(ov / h, 0.0, 1.0))
    return fr


def voxelize(objects, grid, subdiv=4, stats=None):
    """objects: list of dicts {kind: BUILDING|TREE, phi, lad, box:(lo,hi)} or
    {kind, phi, lad, mesh:(verts, tris)}.  Returns labels, phi, lad in the
    x-fastest layout."""
    if not 1 <= subdiv <= 8:
        raise ValueError("subdiv must be in [1, 8]")
    nsamp = subdiv ** 3
    sphi, slad, kind_of = {}, {}, {}
    shape_ref = (grid.nx, grid.ny, grid.nz)

    def note(flat, ophi, kind):
        prev = kind_of.get(flat)
        if prev is None or ophi < prev[0]:
            if prev is not None and prev[1] != kind:
                warnings.warn(f"overlapping objects in cell {flat}", stacklevel=3)
            kind_of[flat] = (ophi, kind)

    def subs(axis, cells):
        h = grid.h(axis)
        base = grid.origin[axis] + cells * h
        offs = (np.arange(subdiv) + 0.5) * h / subdiv
        return (base[:, None] + offs[None, :]).ravel()

    for ob in objects:
        eff = 1.0 if ob["kind"] == TREE else ob["phi"]
        lad_on = ob["kind"] == TREE and ob["lad"] > 0
        if "mesh" in ob:
            verts, tris = ob["mesh"]
            blo, bhi = verts.min(axis=0), verts.max(axis=0)
            cand = []
            for a in range(3):
                c = _centers(grid, a)
                pad = 0.5 * grid.h(a)
                cand.append(np.nonzero((c >= blo[a] - pad) & (c <= bhi[a] + pad))[0])
            if any(len(r) == 0 for r in cand):
                continue
            ins = classify_columns(verts, tris, subs(0, cand[0]), subs(1, cand[1]),
                                   subs(2, cand[2]), stats)
            ncx, ncy, ncz = (len(r) for r in cand)
            blocks = ins.reshape(ncx, subdiv, ncy, subdiv, ncz, subdiv) \
                .transpose(0, 2, 4, 1, 3, 5).reshape(ncx, ncy, ncz, nsamp)
            for cx, cy, cz in zip(*np.nonzero(blocks.any(axis=-1))):
                flat = int(np.ravel_multi_index((cand[0][cx], cand[1][cy], cand[2][cz]),
                                                shape_ref))
                b = blocks[cx, cy, cz]
                s = sphi.setdefault(flat, np.ones(nsamp))
                np.minimum(s, np.where(b, eff, 1.0), out=s)
                if lad_on:
                    l_ = slad.setdefault(flat, np.zeros(nsamp))
                    np.maximum(l_, np.where(b, ob["lad"], 0.0), out=l_)
                note(flat, eff, ob["kind"])
        else:
            lo = np.asarray(ob["box"][0], float)
            hi = np.asarray(ob["box"][1], float)
            fx, fy, fz = box_coverage_axes(grid, lo, hi)
            cov = (fx[:, None, None] * fy[None, :, None] * fz[None, None, :]).ravel()
            for flat in np.nonzero(cov > 0.0)[0]:
                c = cov[flat]
                flat = int(flat)
                s = sphi.setdefault(flat, np.ones(nsamp))
                s *= 1.0 - c * (1.0 - eff)
                if lad_on:
                    l_ = slad.setdefault(flat, np.zeros(nsamp))
                    l_ += ob["lad"] * c
                note(flat, eff, ob["kind"])

    phi_r = np.ones(shape_ref)
    lad_r = np.zeros(shape_ref)
    lab_r = np.zeros(shape_ref, np.int8)
    for flat, s in sphi.items():
        phi_r[np.unravel_index(flat, shape_ref)] = s.mean()
    for flat, s in slad.items():
        lad_r[np.unravel_index(flat, shape_ref)] = s.mean()
    for flat, (_, kind) in kind_of.items():
        ijk = np.unravel_index(flat, shape_ref)
        if phi_r[ijk] < 1.0 - 1e-12 or lad_r[ijk] > 0.0:
            lab_r[ijk] = kind
    t = lambda a: np.ascontiguousarray(a.transpose(2, 1, 0))  # noqa: E731
    return t(lab_r), t(phi_r), t(lad_r)


# --- scenario layer (scenario.py:327-360, 383-417) --------------------------

def scene_objects(scene, theta=None):
    """Instantiate objects with the design offsets/extents applied."""
    grid = scene.grid
    off = {o["name"]: np.zeros(3) for o in scene.objects}
    ext = {o["name"]: np.zeros(3) for o in scene.objects}
    if scene.design:
        vals = np.array([float(d["initial"]) for d in scene.design]) if theta is None \
            else np.asarray(theta, float)
        for d, val in zip(scene.design, vals):
            ax = "xyz".index(d["transform"][-1])
            (off if d["transform"].startswith("translate") else ext)[d["object"]][ax] += val
    out = []
    zlo = grid.origin[2]
    zhi = zlo + grid.h(2) * grid.nz
    for o in scene.objects:
        kind = BUILDING if o.get("kind", "building") == "building" else TREE
        of, ex = off[o["name"]], ext[o["name"]]
        base = {"kind": kind, "phi": float(o.get("phi", 0.0)), "lad": float(o.get("lad", 0.0))}
        if o["shape"] == "box":
            base["box"] = (np.asarray(o["lo"], float) + of, np.asarray(o["hi"], float) + of + ex)
        elif o["shape"] == "cylinder":
            z0 = o.get("z0")
            z1 = o.get("z1")
            z0 = zlo - grid.dz if z0 is None else z0
            z1 = zhi + grid.dz if z1 is None else z1
            base["mesh"] = cylinder_mesh((o["center"][0] + of[0], o["center"][1] + of[1]),
                                         float(o.get("radius", 0.0)) + ex[0],
                                         z0 + of[2], z1 + of[2] + ex[2])
        else:
            raise NotImplementedError("mesh-file objects are not used by the parity scenes")
        out.append(base)
    return out


def read_raster(path):
    """grid.py:385-429: binary PGM (P5, maxval 255) or 8-bit PNG, (rows, cols)."""
    if not str(path).lower().endswith(".pgm"):
        from PIL import Image
        img = Image.open(path)
        return np.asarray(img if img.mode == "L" else img.convert("L"), dtype=np.uint8)
    data = open(path, "rb").read()
    toks, pos = [], 0
    while len(toks) < 4:
        while data[pos:pos + 1].isspace():
            pos += 1
        if data[pos:pos + 1] == b"#":
            while pos < len(data) and data[pos] != 0x0A:
                pos += 1
            continue
        st = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        toks.append(data[st:pos])
    w, h = int(toks[1]), int(toks[2])
    return np.frombuffer(data, np.uint8, count=w * h, offset=pos + 1).reshape(h, w)


def painted_layer(grid, image, tree_mask, extrude_height, tree_lad):
    """decode_painted_porosity (grid.py:337-377) in the x-fastest layout:
    planes k < kmax take phi = pixel / 255, TREE where the mask is set (LAD
    tree_lad), BUILDING where phi < 1, else AIR."""
    labels = np.zeros(grid.cshape, np.int8)
    phi = np.ones(grid.cshape)
    lad = np.zeros(grid.cshape)
    img = np.asarray(image, np.uint8)
    tree = np.zeros(img.shape, bool) if tree_mask is None else np.asarray(tree_mask) != 0
    if grid.nz == 1 or extrude_height is None:
        kmax = grid.nz
    else:
        zc = grid.origin[2] + (np.arange(grid.nz) + 0.5) * grid.dz - grid.origin[2]
        kmax = int(np.sum(zc <= extrude_height))
    p2 = img.astype(float) / 255.0                      # (ny, nx): x fastest already
    l2 = np.where(tree, TREE, np.where((p2 < 1.0) | tree, BUILDING, AIR)).astype(np.int8)
    for k in range(kmax):
        phi[k] = p2
        labels[k] = l2
        lad[k] = np.where(tree, tree_lad, 0.0)
    return labels, phi, lad


def combine_layers(bl, bp, ba, al, ap, aa):
    """combine_porosity (scenario.py:351-360): lower phi wins, LAD by max,
    object TREE labels over AIR."""
    phi = np.minimum(bp, ap)
    lad = np.maximum(ba, aa)
    labels = bl.copy()
    take = ap < bp
    labels[take] = al[take]
    labels[(al == TREE) & (labels == AIR)] = TREE
    return labels, phi, lad


def combine_with_open_air(labels, phi, lad):
    """combine_porosity (scenario.py:351-360) against an open-air base layer."""
    phi_c = np.minimum(np.ones_like(phi), phi)
    lad_c = np.maximum(np.zeros_like(lad), lad)
    lab = np.zeros_like(labels)
    take = phi < 1.0
    lab[take] = labels[take]
    lab[(labels == TREE) & (lab == AIR)] = TREE
    return lab, phi_c, lad_c


def voxelize_scene(scene, boundary_labels, theta=None, stats=None):
    """CompiledScenario.voxelize_design (scenario.py:383-417)."""
    import os
    labels, phi, lad = (np.zeros(scene.grid.cshape, np.int8), np.ones(scene.grid.cshape),
                        np.zeros(scene.grid.cshape))
    paint = getattr(scene, "paint", None)
    if paint is not None:
        base = getattr(scene, "base_dir", ".")
        img = read_raster(os.path.join(base, paint["path"]))
        mask = read_raster(os.path.join(base, paint["tree_mask"])) if paint.get("tree_mask") else None
        labels, phi, lad = painted_layer(scene.grid, img, mask, paint.get("extrude_height"),
                                         float(paint.get("tree_lad", 1.0)))
    if scene.objects:
        ol, op, oa = voxelize(scene_objects(scene, theta), scene.grid, scene.subdiv, stats)
        if paint is not None:
            labels, phi, lad = combine_layers(labels, phi, lad, ol, op, oa)
        else:
            labels, phi, lad = combine_with_open_air(ol, op, oa)
    return merge_labels(boundary_labels, labels), phi, lad
