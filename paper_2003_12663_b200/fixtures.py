"""Benchmark geometries.

* Icosphere shells (reference ``src/fixtures.py``): vertices are reproduced
  bit for bit -- the same vertex creation order and the same rounding of
  the edge-midpoint normalisation (``p / ||p||`` with the ddot norm) -- so
  configs 1-3 are identical inputs on both sides.  Built level by level with
  array operations instead of per-edge dictionaries.
* ``rod_plane_mesh``: the synthetic disconnector-like config 4:
  a capsule rod electrode above a grounded slab electrode, with a closed
  dielectric post insulator standing just above the slab (a sub-panel gap,
  so the deferred near-singular pass is exercised).  Deterministic, no RNG;
  structured "cube-capsule" grids, so vertex numbering is spatially local.
* ``close_gap_mesh``: two concentric shells 2 % apart (deferred pairs on
  every row) for near-pass parity.
"""

from __future__ import annotations

import numpy as np

from . import _fp
from .mesh import EPS0, PatchSpec, SurfaceMesh, _parse_patch, build_mesh

__all__ = [
    "icosphere",
    "sphere_levels",
    "sphere_mesh_parts",
    "sphere_mesh",
    "concentric_mesh",
    "mesh_text",
    "mesh_from_parts",
    "rod_plane_parts",
    "rod_plane_mesh",
    "close_gap_mesh",
]

_PHI = (1.0 + np.sqrt(5.0)) / 2.0
_ICO_V = np.array(
    [[-1, _PHI, 0], [1, _PHI, 0], [-1, -_PHI, 0], [1, -_PHI, 0],
     [0, -1, _PHI], [0, 1, _PHI], [0, -1, -_PHI], [0, 1, -_PHI],
     [_PHI, 0, -1], [_PHI, 0, 1], [-_PHI, 0, -1], [-_PHI, 0, 1]],
    dtype=np.float64,
)
_ICO_F = np.array(
    [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
     [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
     [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
     [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]],
    dtype=np.intp,
)


def _edge_midpoints(verts, faces):
    """Projected midpoints of the face edges (ab, bc, ca per face, faces in
    order), numbered in first-creation order.  Returns (new_vertices,
    mid_index (nf, 3))."""
    e = np.stack([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]], axis=1).reshape(-1, 2)
    key = np.minimum(e[:, 0], e[:, 1]) * (len(verts) + 1) + np.maximum(e[:, 0], e[:, 1])
    uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")  # creation order
    rank = np.empty(len(uniq), dtype=np.intp)
    rank[order] = np.arange(len(uniq))
    src = e[first[order]]  # (i, j) as first encountered
    p = verts[src[:, 0]] + verts[src[:, 1]]
    p = p / _fp.norm3_fused(p)[:, None]
    mid = len(verts) + rank[inv].reshape(-1, 3)
    return p, mid


def icosphere(level: int):
    """Unit icosphere (vertices, faces), outward winding (src/fixtures.py:26-50)."""
    verts = _ICO_V / _fp.norm3_axis(_ICO_V)[:, None]
    faces = _ICO_F.copy()
    for _ in range(level):
        newv, mid = _edge_midpoints(verts, faces)
        a, b, c = faces[:, 0], faces[:, 1], faces[:, 2]
        ab, bc, ca = mid[:, 0], mid[:, 1], mid[:, 2]
        faces = np.stack([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                          np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], axis=1).reshape(-1, 3)
        verts = np.vstack([verts, newv])
    return verts, faces


def sphere_levels() -> dict:
    return {lev: 10 * 4 ** lev + 2 for lev in range(7)}


def sphere_mesh_parts(level: int, radius: float = 1.0, tag: int = 0,
                      center=(0.0, 0.0, 0.0), flip: bool = False, id_offset: int = 0):
    """One curved sphere shell: corners = level-L icosphere, midside nodes =
    projected edge midpoints (src/fixtures.py:80-118)."""
    verts, faces = icosphere(level)
    if flip:
        faces = faces[:, [0, 2, 1]]
    newv, mid = _edge_midpoints(verts, faces)
    allv = np.vstack([verts, newv]) * radius + np.asarray(center, dtype=np.float64)
    ids = np.concatenate([faces, mid], axis=1) + id_offset
    tris = [(tuple(int(k) for k in row), tag) for row in ids.tolist()]
    return allv, tris


def mesh_text(vertices, tris, patch_lines) -> str:
    out = ["bemesh 1"]
    out += [f"vertex {i} {float(p[0])!r} {float(p[1])!r} {float(p[2])!r}"
            for i, p in enumerate(np.asarray(vertices).tolist())]
    out += ["triangle " + " ".join(str(k) for k in ids) + f" {tag}" for ids, tag in tris]
    out += list(patch_lines)
    return "\n".join(out) + "\n"


def mesh_from_parts(vertices, tri_ids, tri_tags, patch_lines, name="<fixture>") -> SurfaceMesh:
    """Build a mesh straight from arrays (same result as text + parse_mesh,
    since repr() round-trips float64 exactly)."""
    patches = {}
    scale = 1.0
    for ln in patch_lines:
        parts = ln.split()
        if parts[0] == "permittivity":
            scale = EPS0 if parts[1] == "relative" else 1.0
            continue

        def err(_l, msg):
            raise ValueError(msg)

        p = _parse_patch(parts, err, 0)
        patches[p.tag] = p
    if scale != 1.0:
        patches = {t: PatchSpec(p.tag, p.kind, v0=p.v0, index=p.index,
                                eps_plus=p.eps_plus * scale, eps_minus=p.eps_minus * scale)
                   for t, p in patches.items()}
    return build_mesh(vertices, tri_ids, tri_tags, patches, name=name)


def _parts_arrays(tris):
    ids = np.array([t[0] for t in tris], dtype=np.intp)
    tags = np.array([t[1] for t in tris], dtype=np.intp)
    return ids, tags


def sphere_mesh(level: int, radius: float = 1.0, v0: float = 1.0) -> SurfaceMesh:
    verts, tris = sphere_mesh_parts(level, radius=radius, tag=0)
    ids, tags = _parts_arrays(tris)
    return mesh_from_parts(verts, ids, tags, [f"patch 0 electrode {v0!r}"],
                           name=f"<sphere L{level} R{radius}>")


def concentric_mesh(level: int, shells) -> SurfaceMesh:
    """Concentric outward-wound shells; `shells` = [(radius, patch tail)]."""
    vs, ids, tags, lines = [], [], [], []
    off = 0
    for tag, (radius, tail) in enumerate(shells):
        v, tris = sphere_mesh_parts(level, radius=radius, tag=tag, id_offset=off)
        i, t = _parts_arrays(tris)
        vs.append(v)
        ids.append(i)
        tags.append(t)
        lines.append(f"patch {tag} {tail}")
        off += len(v)
    return mesh_from_parts(np.vstack(vs), np.vstack(ids), np.concatenate(tags), lines,
                           name=f"<concentric L{level}>")


def close_gap_mesh(level: int = 3, gap: float = 0.02) -> SurfaceMesh:
    """Electrode shells at r=1 (1 V) and r=1+gap (0 V): every collocation
    row has deferred near-singular pairs on the opposite shell."""
    return concentric_mesh(level, [(1.0, "electrode 1.0"), (1.0 + gap, "electrode 0.0")])


# ---------------------------------------------------------------------------
# config 4: rod-plane + insulator
# ---------------------------------------------------------------------------


def _box_grid(ext, counts):
    """Closed, outward-wound quadratic triangle grid on the box
    [-X,X] x [-Y,Y] x [-Z,Z] with (nx, ny, nz) cells per axis.  Returns
    (points (m,3), tri node ids (nt,6)); midside nodes are the straight edge
    midpoints (curved later by a projection).  Vertices are numbered face by
    face in grid order (first occurrence), so numbering is spatially local."""
    X, Y, Z = (float(e) for e in ext)
    nx, ny, nz = (int(c) for c in counts)
    faces = (  # origin, u axis (length), v axis (length), cells u, cells v
        ((-X, -Y, Z), (2 * X, 0, 0), (0, 2 * Y, 0), nx, ny),
        ((-X, Y, -Z), (2 * X, 0, 0), (0, -2 * Y, 0), nx, ny),
        ((-X, -Y, -Z), (2 * X, 0, 0), (0, 0, 2 * Z), nx, nz),
        ((X, Y, -Z), (-2 * X, 0, 0), (0, 0, 2 * Z), nx, nz),
        ((X, -Y, -Z), (0, 2 * Y, 0), (0, 0, 2 * Z), ny, nz),
        ((-X, Y, -Z), (0, -2 * Y, 0), (0, 0, 2 * Z), ny, nz),
    )
    half = np.array([X / nx, Y / ny, Z / nz])  # half-cell sizes (lattice unit)
    all_pts, all_tris = [], []
    base = 0
    for o, du, dv, mu, mv in faces:
        o, du, dv = (np.array(a, dtype=np.float64) for a in (o, du, dv))
        iu, iv = np.meshgrid(np.arange(2 * mu + 1), np.arange(2 * mv + 1), indexing="xy")
        lat = o + (iu.ravel()[:, None] / (2 * mu)) * du + (iv.ravel()[:, None] / (2 * mv)) * dv
        W = 2 * mu + 1

        def L(a, b):
            return b * W + a

        j, i = np.meshgrid(np.arange(mv), np.arange(mu), indexing="ij")
        i = i.ravel()
        j = j.ravel()
        a0, b0 = 2 * i, 2 * j
        c00, c10, c01, c11 = L(a0, b0), L(a0 + 2, b0), L(a0, b0 + 2), L(a0 + 2, b0 + 2)
        even = (i + j) % 2 == 0
        # even cells: (c00,c10,c11),(c00,c11,c01); odd: (c00,c10,c01),(c10,c11,c01)
        t1 = np.where(even[:, None], np.stack([c00, c10, c11], 1), np.stack([c00, c10, c01], 1))
        t2 = np.where(even[:, None], np.stack([c00, c11, c01], 1), np.stack([c10, c11, c01], 1))
        tri = np.stack([t1, t2], axis=1).reshape(-1, 3)
        ua, va = tri % W, tri // W
        mids = [L((ua[:, k] + ua[:, (k + 1) % 3]) // 2, (va[:, k] + va[:, (k + 1) % 3]) // 2) for k in range(3)]
        tri6 = np.column_stack([tri, np.stack(mids, 1)])
        all_pts.append(lat)
        all_tris.append(tri6 + base)
        base += len(lat)
    pts = np.vstack(all_pts)
    tris = np.vstack(all_tris)
    key = np.rint((pts + np.array([X, Y, Z])) / half).astype(np.int64)
    kk = (key[:, 0] * (2 * ny + 1) + key[:, 1]) * (2 * nz + 1) + key[:, 2]
    used = np.zeros(len(pts), dtype=bool)
    used[tris.ravel()] = True
    kk = np.where(used, kk, -1 - np.arange(len(pts)))
    uniq, first, inv = np.unique(kk, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty(len(uniq), dtype=np.intp)
    rank[order] = np.arange(len(uniq))
    gid = rank[inv]
    keep = np.zeros(len(uniq), dtype=bool)
    keep[gid[tris.ravel()]] = True
    # renumber the used lattice points densely in first-use order
    live = np.cumsum(keep[order]) - 1
    dense = np.full(len(uniq), -1, dtype=np.intp)
    dense[order] = np.where(keep[order], live, -1)
    out_pts = np.empty((int(keep.sum()), 3))
    out_pts[dense[gid[used]]] = pts[used]
    return out_pts, dense[gid[tris]]


def _capsule(n_round, radius, half_len, center):
    """Capsule (cylinder of half length `half_len` with hemispherical ends)
    meshed by projecting the elongated box [-1,1]^2 x [-1-h, 1+h], h =
    half_len/radius, with uniform box cells, so panels stay near-isotropic."""
    h = half_len / radius
    nz = int(round(n_round * (1.0 + h)))
    pts, tris = _box_grid((1.0, 1.0, 1.0 + h), (n_round, n_round, nz))
    zc = np.clip(pts[:, 2], -h, h)
    q = np.column_stack([pts[:, 0], pts[:, 1], pts[:, 2] - zc])
    q = q / np.linalg.norm(q, axis=1)[:, None]
    xyz = radius * q
    xyz[:, 2] += radius * zc
    return xyz + np.asarray(center, dtype=np.float64), tris


def _slab(counts, half_ext, center):
    pts, tris = _box_grid(half_ext, counts)
    return pts + np.asarray(center, dtype=np.float64), tris


def rod_plane_parts(scale: float = 1.0, v0: float = 0.0, v_plane: float = -1.0e5):
    """Vertices, triangle ids, tags and patch lines of config 4.

    `scale` multiplies the mesh resolution (panel count ~ scale^2 * 2e5).
    The grounded rod sits above the energised plane (-100 kV): with the
    driven electrode being the coarse one, the reference's GMRES (row
    equilibration + true-residual gate, src/solver.py:98-146) converges at
    its default 1e-8 (74 iterations at scale 1); with the fine rod driven
    instead it stalls at a true residual of 1.1e-8."""
    s = float(scale)
    parts = []
    # rod electrode: capsule r=2 cm, cylinder 0.5 m, tip 10 cm above the slab
    n_r = max(2, int(round(16 * s)))
    parts.append(_capsule(n_r, 0.02, 0.25, (0.0, 0.0, 0.02 + 0.25 + 0.10)) + (0,))
    # post insulator: closed capsule r=6 cm, half length 0.15 m, standing 4 mm
    # above the slab, 0.3 m beside the rod
    n_ir = max(2, int(round(24 * s)))
    parts.append(_capsule(n_ir, 0.06, 0.15, (0.30, 0.0, 0.06 + 0.15 + 0.004)) + (1,))
    # grounded slab: 2 m x 2 m x 0.1 m, top face at z = 0
    n_g = max(2, int(round(190 * s)))
    parts.append(_slab((n_g, n_g, max(1, int(round(5 * s)))), (1.0, 1.0, 0.05), (0.0, 0.0, -0.05)) + (2,))
    vs, ids, tags = [], [], []
    off = 0
    for xyz, tri, tag in parts:
        vs.append(xyz)
        ids.append(tri + off)
        tags.append(np.full(len(tri), tag, dtype=np.intp))
        off += len(xyz)
    lines = [
        "permittivity relative",
        f"patch 0 electrode {float(v0)!r}",
        "patch 1 dielectric 1.0 4.0",
        f"patch 2 electrode {float(v_plane)!r}",
    ]
    return np.vstack(vs), np.vstack(ids), np.concatenate(tags), lines


def rod_plane_mesh(scale: float = 1.0, v0: float = 0.0, v_plane: float = -1.0e5) -> SurfaceMesh:
    v, ids, tags, lines = rod_plane_parts(scale, v0, v_plane)
    return mesh_from_parts(v, ids, tags, lines, name=f"<rod-plane x{scale}>")
