"""Curved six-node triangle meshes and the derived per-vertex arrays that form
the device input contract.

Mirrors ``hvbem.mesh`` (reference ``src/mesh.py``): same record format, same
validation messages, same row-kind priority (electrode > floating >
dielectric, ``src/mesh.py:360-392``).  Unlike the reference, every derived
array is built with whole-mesh NumPy operations instead of per-triangle
Python loops: a 200k-panel mesh is processed in a
couple of seconds.  Circumcentres/radii are reproduced bit for bit (they feed
the pair classification); the FMA-chained dot products of the reference's
``_flat_circumcircle`` (``src/mesh.py:188-200``) are emulated by
:mod:`._fp`.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import _fp
from .quadrature import regular_rule

__all__ = [
    "EPS0",
    "MeshError",
    "Vertex",
    "CurvedTriangle",
    "PatchSpec",
    "SurfaceMesh",
    "Dirichlet",
    "FloatingDirichlet",
    "DielectricJump",
    "load_mesh",
    "parse_mesh",
    "save_mesh",
    "map_reference",
    "surface_frame",
    "classify_vertex",
    "shape_functions",
    "shape_gradients",
    "KIND_DIRICHLET",
    "KIND_FLOATING",
    "KIND_DIELECTRIC",
]

EPS0 = 8.8541878128e-12  # F/m, reference src/mesh.py:37
MIN_CIRCUMRADIUS = 1e-12  # src/mesh.py:39
MIN_JACOBIAN = 1e-14  # src/mesh.py:40

# integer row-kind codes used by the device kernels
KIND_DIRICHLET = 0
KIND_FLOATING = 1
KIND_DIELECTRIC = 2


class MeshError(ValueError):
    """Invalid mesh file or mesh geometry (reference src/mesh.py:43)."""


@dataclass(frozen=True)
class Dirichlet:
    v0: float


@dataclass(frozen=True)
class FloatingDirichlet:
    index: int


@dataclass(frozen=True)
class DielectricJump:
    eps_plus: float
    eps_minus: float


@dataclass(frozen=True)
class Vertex:
    id: int
    position: np.ndarray


@dataclass(frozen=True)
class PatchSpec:
    """Boundary condition of a patch tag (reference src/mesh.py:79-98)."""

    tag: int
    kind: str
    v0: float = 0.0
    index: int = -1
    eps_plus: float = 0.0
    eps_minus: float = 0.0

    @property
    def is_floating(self) -> bool:
        return self.kind in ("floating", "sheet")


@dataclass
class CurvedTriangle:
    """Six-node triangle view (node order c0 c1 c2 m01 m12 m20)."""

    index: int
    corner_ids: tuple
    midside_ids: tuple
    patch_tag: int
    nodes: np.ndarray = field(repr=False)
    circumcenter: np.ndarray = field(repr=False)
    circumradius: float = 0.0

    @property
    def node_ids(self) -> tuple:
        return tuple(self.corner_ids) + tuple(self.midside_ids)


# ---------------------------------------------------------------------------
# quadratic Lagrange basis on the reference triangle (src/mesh.py:124-158)
# ---------------------------------------------------------------------------


def shape_functions(uv) -> np.ndarray:
    """(m, 6) values of the six quadratic shape functions."""
    uv = np.atleast_2d(np.asarray(uv, dtype=np.float64))
    u = uv[:, 0]
    v = uv[:, 1]
    w = 1.0 - u - v
    return np.stack(
        [w * (2.0 * w - 1.0), u * (2.0 * u - 1.0), v * (2.0 * v - 1.0),
         4.0 * w * u, 4.0 * u * v, 4.0 * v * w],
        axis=1,
    )


def shape_gradients(uv):
    """(dN/du, dN/dv), each (m, 6)."""
    uv = np.atleast_2d(np.asarray(uv, dtype=np.float64))
    u = uv[:, 0]
    v = uv[:, 1]
    w = 1.0 - u - v
    z = np.zeros_like(u)
    gu = np.stack([1.0 - 4.0 * w, 4.0 * u - 1.0, z, 4.0 * (w - u), 4.0 * v, -4.0 * v], axis=1)
    gv = np.stack([1.0 - 4.0 * w, z, 4.0 * v - 1.0, -4.0 * u, 4.0 * u, 4.0 * (w - v)], axis=1)
    return gu, gv


def map_reference(tri, uv) -> np.ndarray:
    """Surface point(s) of the quadratic map at reference uv."""
    pts = shape_functions(uv) @ np.asarray(tri.nodes)
    return pts[0] if np.ndim(uv) == 1 else pts


def surface_frame(tri, uv):
    """Unit normal and area element at uv (src/mesh.py:168-185)."""
    single = np.ndim(uv) == 1
    gu, gv = shape_gradients(uv)
    nodes = np.asarray(tri.nodes)
    cr = _fp.cross3(gu @ nodes, gv @ nodes)
    jac = _fp.norm3_axis(cr)
    if np.any(jac < MIN_JACOBIAN):
        raise MeshError(
            f"degenerate surface Jacobian on triangle {tri.index} "
            f"(|J| = {jac.min():.3e})"
        )
    nrm = cr / jac[:, None]
    if single:
        return nrm[0], float(jac[0])
    return nrm, jac


def flat_circumcircles(corners: np.ndarray):
    """Circumcentre and radius of the flat corner triangles, (nt,3,3) in.

    Bit-identical to reference ``_flat_circumcircle`` (src/mesh.py:188-200):
    unfused cross products, FMA-chained 3-dots, radius = sqrt(ddot)."""
    a = corners[:, 0]
    ab = corners[:, 1] - a
    ac = corners[:, 2] - a
    nrm = _fp.cross3(ab, ac)
    nn = _fp.dot3(nrm, nrm)
    num = _fp.dot3(ac, ac)[:, None] * _fp.cross3(nrm, ab) + _fp.dot3(ab, ab)[:, None] * _fp.cross3(ac, nrm)
    with np.errstate(divide="ignore", invalid="ignore"):
        center = a + num / (2.0 * nn)[:, None]
    degenerate = ~(nn > 0.0)
    center = np.where(degenerate[:, None], a, center)
    radius = _fp.norm3_fused(center - a)
    radius = np.where(degenerate, 0.0, radius)
    return center, radius


def _flat_circumcircle(corners):
    """Single-triangle form used by the reference tests (tests/conftest.py:72)."""
    c, r = flat_circumcircles(np.asarray(corners, dtype=np.float64)[None])
    return c[0], float(r[0])


# ---------------------------------------------------------------------------
# SurfaceMesh
# ---------------------------------------------------------------------------


class SurfaceMesh:
    """Validated surface mesh with precomputed collocation data.

    Attribute names follow reference ``SurfaceMesh`` (src/mesh.py:208-352).
    Extra array attributes (``row_kind_code``, ``row_v0``, ``row_float``,
    ``row_eps_plus``, ``row_eps_minus``, ``vc_ptr``/``vc_tri``/``vc_corner``)
    are the flat forms the device kernels consume.
    """

    def __init__(self, vertices, triangles=None, patches=None, *,
                 tri_node_ids=None, tri_tags=None):
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64)
        self.patches = dict(patches or {})
        if triangles is not None:
            tri_node_ids = np.array([t.node_ids for t in triangles], dtype=np.intp)
            tri_tags = np.array([t.patch_tag for t in triangles], dtype=np.intp)
            self._triangles = list(triangles)
        else:
            self._triangles = None
        self.tri_node_ids = np.ascontiguousarray(tri_node_ids, dtype=np.intp).reshape(-1, 6)
        self.tri_tags = np.ascontiguousarray(tri_tags, dtype=np.intp).reshape(-1)
        self.tri_nodes = np.ascontiguousarray(self.vertices[self.tri_node_ids])  # (nt,6,3)
        if triangles is not None:
            self.circumcenters = np.stack([np.asarray(t.circumcenter, dtype=float) for t in triangles])
            self.circumradii = np.array([float(t.circumradius) for t in triangles])
        else:
            self.circumcenters, self.circumradii = flat_circumcircles(self.tri_nodes[:, :3])
        self._vertex_corners = None
        self._vertex_triangles = None
        self._build_collocation()
        self._cache_lock = threading.Lock()
        self._table_cache: dict = {}
        self._device_cache: dict = {}

    # -- construction ---------------------------------------------------------

    def _build_collocation(self):
        nv = len(self.vertices)
        nt = len(self.tri_node_ids)
        used = np.zeros(nv, dtype=bool)
        used[self.tri_node_ids.ravel()] = True
        if not used.all():
            raise MeshError(f"vertex {int(np.argmin(used))} belongs to no triangle")
        is_corner = np.zeros(nv, dtype=bool)
        is_corner[self.tri_node_ids[:, :3].ravel()] = True
        ids = np.nonzero(is_corner)[0]
        index = np.full(nv, -1, dtype=np.intp)
        index[ids] = np.arange(len(ids))
        self.colloc_vertex_ids = ids
        self.colloc_index = index
        self.colloc_points = self.vertices[ids]
        self.tri_corner_cols = index[self.tri_node_ids[:, :3]]

        # star of each collocation vertex: (triangle, corner) in triangle order
        cols = self.tri_corner_cols.ravel()
        order = np.argsort(cols, kind="stable")  # stable: triangle order kept
        counts = np.bincount(cols, minlength=len(ids))
        self.vc_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.intp)
        self.vc_tri = (order // 3).astype(np.intp)
        self.vc_corner = (order % 3).astype(np.intp)

        self._classify_rows(nt)
        self._compute_weights_and_normals()

    def _classify_rows(self, nt):
        """Row kinds by junction priority (reference classify_vertex,
        src/mesh.py:360-392), vectorised over all incidences.  When several
        electrode (floating) triangles meet, the reference keeps the last one
        in triangle order; so do we."""
        n = len(self.colloc_vertex_ids)
        tags = sorted(self.patches)
        kind_of = np.array([
            0 if self.patches[t].kind == "electrode" else (1 if self.patches[t].is_floating else 2)
            for t in tags
        ], dtype=np.int64)
        if not tags:
            raise MeshError(f"unknown patch tag {int(self.tri_tags[0])}")
        tag_arr = np.array(tags, dtype=np.intp)
        pos = np.clip(np.searchsorted(tag_arr, self.tri_tags), 0, len(tags) - 1)
        tri_patch = np.where(tag_arr[pos] == self.tri_tags, pos, -1).astype(np.int64)
        if np.any(tri_patch < 0):
            raise MeshError(f"unknown patch tag {int(self.tri_tags[np.argmin(tri_patch)])}")
        tri_kind = kind_of[tri_patch]

        # incidences (vertex, triangle) over all six nodes, restricted to corners
        vid = self.tri_node_ids.ravel()
        tri = np.repeat(np.arange(nt), 6)
        col = self.colloc_index[vid]
        m = col >= 0
        col, tri = col[m], tri[m]
        kind = tri_kind[tri]

        last_elec = np.full(n, -1, dtype=np.int64)
        last_float = np.full(n, -1, dtype=np.int64)
        em = kind == 0
        np.maximum.at(last_elec, col[em], tri[em])
        fm = kind == 1
        np.maximum.at(last_float, col[fm], tri[fm])

        code = np.full(n, KIND_DIELECTRIC, dtype=np.int32)
        code[last_float >= 0] = KIND_FLOATING
        code[last_elec >= 0] = KIND_DIRICHLET
        v0 = np.zeros(n)
        fidx = np.full(n, -1, dtype=np.int64)
        eps_p = np.zeros(n)
        eps_m = np.zeros(n)
        patch_list = [self.patches[t] for t in tags]
        pv0 = np.array([p.v0 for p in patch_list])
        pidx = np.array([p.index for p in patch_list], dtype=np.int64)
        pep = np.array([p.eps_plus for p in patch_list])
        pem = np.array([p.eps_minus for p in patch_list])
        sel = code == KIND_DIRICHLET
        v0[sel] = pv0[tri_patch[last_elec[sel]]]
        sel = code == KIND_FLOATING
        fidx[sel] = pidx[tri_patch[last_float[sel]]]

        # dielectric-only vertices must see exactly one (eps+, eps-) pair
        diel_rows = np.nonzero(code == KIND_DIELECTRIC)[0]
        if len(diel_rows):
            dm = (code[col] == KIND_DIELECTRIC) & (kind == 2)
            dc, dtri = col[dm], tri[dm]
            ep = pep[tri_patch[dtri]]
            em_ = pem[tri_patch[dtri]]
            first_p = np.full(n, np.nan)
            first_m = np.full(n, np.nan)
            # any incidence that disagrees with the vertex's first pair is a conflict
            o = np.argsort(dc, kind="stable")
            dc_s, ep_s, em_s = dc[o], ep[o], em_[o]
            starts = np.concatenate([[True], dc_s[1:] != dc_s[:-1]])
            first_p[dc_s[starts]] = ep_s[starts]
            first_m[dc_s[starts]] = em_s[starts]
            bad = (ep_s != first_p[dc_s]) | (em_s != first_m[dc_s])
            if np.any(bad):
                bad_rows = np.unique(dc_s[bad])
                r = int(bad_rows[0])
                vsel = dc_s == r
                pairs = sorted({(float(a), float(b)) for a, b in zip(ep_s[vsel], em_s[vsel])})
                raise MeshError(
                    f"vertex {int(self.colloc_vertex_ids[r])} joins dielectric interfaces "
                    f"with different permittivity pairs {pairs}; triple junctions are not "
                    "supported"
                )
            eps_p[diel_rows] = first_p[diel_rows]
            eps_m[diel_rows] = first_m[diel_rows]

        self.row_kind_code = code
        self.row_v0 = v0
        self.row_float = fidx
        self.row_eps_plus = eps_p
        self.row_eps_minus = eps_m
        self._row_kinds = None

        floats = sorted({p.index for p in self.patches.values() if p.is_floating})
        if floats and floats != list(range(len(floats))):
            raise MeshError(f"floating indices must be contiguous from 0, got {floats}")
        self.n_floating = len(floats)

    def _compute_weights_and_normals(self):
        """Lumped weights and averaged vertex normals with the degree-4 rule
        (reference src/mesh.py:277-313), all triangles at once; per-vertex
        accumulation keeps the reference's triangle order (np.add.at)."""
        rule = regular_rule(4)
        gu, gv = shape_gradients(rule.nodes)
        lam = np.column_stack([1.0 - rule.nodes[:, 0] - rule.nodes[:, 1],
                               rule.nodes[:, 0], rule.nodes[:, 1]])
        tu = np.matmul(gu, self.tri_nodes)  # (nt, q, 3); batched BLAS (einsum is ~5x slower here)
        tv = np.matmul(gv, self.tri_nodes)
        cr = _fp.cross3(tu, tv)
        jac = _fp.norm3_axis(cr)
        low = np.nonzero((jac < MIN_JACOBIAN).any(axis=1))[0]
        if len(low):
            raise MeshError(f"degenerate Jacobian in triangle {int(low[0])}")
        unit = cr / jac[..., None]
        wj = rule.weights[None, :] * jac  # (nt, q)
        contrib = wj @ lam  # (nt, 3)
        n_avg = np.matmul(lam.T, wj[:, :, None] * unit)  # (nt, 3, 3)
        n = len(self.colloc_points)
        cols = self.tri_corner_cols.ravel()
        w = np.zeros(n)
        np.add.at(w, cols, contrib.ravel())
        normals = np.zeros((n, 3))
        np.add.at(normals, cols, n_avg.reshape(-1, 3))
        norms = _fp.norm3_axis(normals)
        if np.any(norms < MIN_JACOBIAN):
            bad = int(np.argmin(norms))
            raise MeshError(
                f"vertex {self.colloc_vertex_ids[bad]} has a vanishing averaged normal "
                "(folded surface?)"
            )
        self.lumped_weights = w
        self.colloc_normals = normals / norms[:, None]

    # -- lazily built object views (the reference exposes them eagerly) ------

    @property
    def triangles(self):
        if self._triangles is None:
            ids = self.tri_node_ids
            self._triangles = [
                CurvedTriangle(
                    index=i,
                    corner_ids=tuple(int(k) for k in ids[i, :3]),
                    midside_ids=tuple(int(k) for k in ids[i, 3:]),
                    patch_tag=int(self.tri_tags[i]),
                    nodes=self.tri_nodes[i],
                    circumcenter=self.circumcenters[i],
                    circumradius=float(self.circumradii[i]),
                )
                for i in range(len(ids))
            ]
        return self._triangles

    @property
    def vertex_corners(self):
        """vertex id -> [(triangle, corner), ...] in triangle order."""
        if self._vertex_corners is None:
            out = [[] for _ in range(len(self.vertices))]
            for i, vid in enumerate(self.colloc_vertex_ids):
                a, b = self.vc_ptr[i], self.vc_ptr[i + 1]
                out[int(vid)] = list(zip(self.vc_tri[a:b].tolist(), self.vc_corner[a:b].tolist()))
            self._vertex_corners = out
        return self._vertex_corners

    @property
    def vertex_triangles(self):
        if self._vertex_triangles is None:
            out = [[] for _ in range(len(self.vertices))]
            for t, ids in enumerate(self.tri_node_ids.tolist()):
                for vid in ids:
                    out[vid].append(t)
            self._vertex_triangles = out
        return self._vertex_triangles

    @property
    def row_kinds(self):
        if self._row_kinds is None:
            out = []
            for c, v0, k, ep, em in zip(self.row_kind_code.tolist(), self.row_v0.tolist(),
                                        self.row_float.tolist(), self.row_eps_plus.tolist(),
                                        self.row_eps_minus.tolist()):
                if c == KIND_DIRICHLET:
                    out.append(Dirichlet(v0))
                elif c == KIND_FLOATING:
                    out.append(FloatingDirichlet(int(k)))
                else:
                    out.append(DielectricJump(ep, em))
            self._row_kinds = out
        return self._row_kinds

    # -- queries --------------------------------------------------------------

    @property
    def n_collocation(self) -> int:
        return len(self.colloc_points)

    @property
    def n_triangles(self) -> int:
        return len(self.tri_node_ids)

    def patch_of(self, tri_index: int) -> PatchSpec:
        return self.patches[int(self.tri_tags[tri_index])]

    def bounding_box(self):
        return self.vertices.min(axis=0), self.vertices.max(axis=0)

    def floating_collocation(self, k: int) -> np.ndarray:
        return np.nonzero((self.row_kind_code == KIND_FLOATING) & (self.row_float == k))[0].astype(np.intp)

    def total_area(self) -> float:
        return float(self.lumped_weights.sum())

    def tables(self, order: int):
        """Per-order host quadrature tables (reference src/mesh.py:343-352)."""
        from .assembly import TriangleTables

        with self._cache_lock:
            tab = self._table_cache.get(order)
            if tab is None:
                tab = TriangleTables(self, order)
                self._table_cache[order] = tab
            return tab


def classify_vertex(mesh: SurfaceMesh, vertex_id: int):
    """Row kind of a collocation vertex (reference src/mesh.py:360-392)."""
    col = int(mesh.colloc_index[vertex_id]) if 0 <= vertex_id < len(mesh.colloc_index) else -1
    if col < 0:
        tris = mesh.vertex_triangles[vertex_id]
        if not tris:
            raise MeshError(f"vertex {vertex_id} belongs to no triangle")
        raise MeshError(f"vertex {vertex_id} is not a corner vertex")
    return mesh.row_kinds[col]


# ---------------------------------------------------------------------------
# text format (reference src/mesh.py:400-577)
# ---------------------------------------------------------------------------


def _parse_patch(parts, err, lineno):
    tag = int(parts[1])
    ptype = parts[2]
    if ptype == "electrode":
        return PatchSpec(tag, "electrode", v0=float(parts[3]))
    if ptype == "floating":
        return PatchSpec(tag, "floating", index=int(parts[3]))
    if ptype == "sheet":
        return PatchSpec(tag, "sheet", index=int(parts[3]),
                         eps_plus=float(parts[4]), eps_minus=float(parts[5]))
    if ptype == "dielectric":
        return PatchSpec(tag, "dielectric", eps_plus=float(parts[3]), eps_minus=float(parts[4]))
    err(lineno, f"unknown patch kind {ptype!r}")


def parse_mesh(text: str, name: str = "<string>") -> SurfaceMesh:
    """Parse the ``bemesh 1`` text format into a validated SurfaceMesh."""
    vert_pos: dict = {}
    tri_lines: list = []
    tri_ids: list = []
    tri_tag: list = []
    patches: dict = {}
    scale = 1.0
    header = False

    def err(lineno, msg):
        raise MeshError(f"{name}:{lineno}: {msg}")

    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        parts = line.split()
        if not header:
            if parts != ["bemesh", "1"]:
                err(lineno, f"expected header 'bemesh 1', got {line!r}")
            header = True
            continue
        rec = parts[0]
        try:
            if rec == "vertex":
                if len(parts) != 5:
                    err(lineno, "vertex needs: vertex <id> <x> <y> <z>")
                vid = int(parts[1])
                pos = (float(parts[2]), float(parts[3]), float(parts[4]))
                if not all(np.isfinite(pos)):
                    err(lineno, f"non-finite vertex position {parts[2:5]}")
                if vid in vert_pos:
                    err(lineno, f"duplicate vertex id {vid}")
                vert_pos[vid] = pos
            elif rec == "triangle":
                if len(parts) != 8:
                    err(lineno, "triangle needs 6 node ids and a patch tag")
                tri_ids.append([int(p) for p in parts[1:7]])
                tri_tag.append(int(parts[7]))
                tri_lines.append(lineno)
            elif rec == "patch":
                p = _parse_patch(parts, err, lineno)
                if p.tag in patches:
                    err(lineno, f"duplicate patch tag {p.tag}")
                patches[p.tag] = p
            elif rec == "permittivity":
                if parts[1] == "relative":
                    scale = EPS0
                elif parts[1] == "absolute":
                    scale = 1.0
                else:
                    err(lineno, "permittivity must be 'relative' or 'absolute'")
            else:
                err(lineno, f"unknown record {rec!r}")
        except MeshError:
            raise
        except (ValueError, IndexError) as exc:
            err(lineno, f"malformed record: {exc}")

    if not header:
        raise MeshError(f"{name}: empty file (missing 'bemesh 1' header)")
    if not vert_pos:
        raise MeshError(f"{name}: no vertices")
    if not tri_ids:
        raise MeshError(f"{name}: no triangles")
    nv = len(vert_pos)
    if sorted(vert_pos) != list(range(nv)):
        raise MeshError(f"{name}: vertex ids must be contiguous 0..{nv - 1}")
    vertices = np.array([vert_pos[i] for i in range(nv)], dtype=np.float64)
    if scale != 1.0:
        patches = {
            t: PatchSpec(p.tag, p.kind, v0=p.v0, index=p.index,
                         eps_plus=p.eps_plus * scale, eps_minus=p.eps_minus * scale)
            for t, p in patches.items()
        }
    for p in patches.values():
        if p.kind in ("sheet", "dielectric") and (p.eps_plus <= 0 or p.eps_minus <= 0):
            raise MeshError(f"{name}: patch {p.tag}: permittivities must be > 0")
    return build_mesh(vertices, np.array(tri_ids, dtype=np.intp), np.array(tri_tag, dtype=np.intp),
                      patches, name=name, linenos=tri_lines)


def build_mesh(vertices, tri_ids, tri_tags, patches, name="<arrays>", linenos=None) -> SurfaceMesh:
    """Validate triangle records in file order (first failure wins, with the
    reference's message for that check) and build the SurfaceMesh."""
    vertices = np.asarray(vertices, dtype=np.float64)
    tri_ids = np.asarray(tri_ids, dtype=np.intp).reshape(-1, 6)
    tri_tags = np.asarray(tri_tags, dtype=np.intp).reshape(-1)
    nt = len(tri_ids)
    nv = len(vertices)
    if linenos is None:
        linenos = list(range(1, nt + 1))
    linenos = np.asarray(linenos)

    bad_range = ((tri_ids < 0) | (tri_ids >= nv)).any(axis=1)
    s = np.sort(tri_ids, axis=1)
    bad_distinct = (s[:, 1:] == s[:, :-1]).any(axis=1) & ~bad_range
    known = np.isin(tri_tags, np.array(sorted(patches), dtype=np.intp))
    bad_tag = ~known
    safe_ids = np.where(bad_range[:, None], 0, tri_ids)
    nodes = vertices[safe_ids]
    cc, cr = flat_circumcircles(nodes[:, :3])
    bad_radius = cr < MIN_CIRCUMRADIUS
    probe = regular_rule(6)
    gu, gv = shape_gradients(probe.nodes)
    jac = _fp.norm3_axis(_fp.cross3(np.matmul(gu, nodes), np.matmul(gv, nodes)))
    bad_jac = (jac < MIN_JACOBIAN).any(axis=1)
    anybad = bad_range | bad_distinct | bad_tag | bad_radius | bad_jac
    if np.any(anybad):
        i = int(np.argmax(anybad))
        ln = int(linenos[i])
        if bad_range[i]:
            vid = int(tri_ids[i][np.argmax((tri_ids[i] < 0) | (tri_ids[i] >= nv))])
            raise MeshError(f"{name}:{ln}: triangle references vertex {vid} of {nv}")
        if bad_distinct[i]:
            raise MeshError(f"{name}:{ln}: triangle node ids must be distinct")
        if bad_tag[i]:
            raise MeshError(f"{name}:{ln}: unknown patch tag {int(tri_tags[i])}")
        if bad_radius[i]:
            raise MeshError(f"{name}:{ln}: degenerate triangle (circumradius {cr[i]:.3e} m)")
        raise MeshError(
            f"degenerate surface Jacobian on triangle {i} (|J| = {jac[i].min():.3e})"
        )
    mesh = SurfaceMesh.__new__(SurfaceMesh)
    mesh.vertices = np.ascontiguousarray(vertices)
    mesh.patches = dict(patches)
    mesh._triangles = None
    mesh.tri_node_ids = np.ascontiguousarray(tri_ids)
    mesh.tri_tags = np.ascontiguousarray(tri_tags)
    mesh.tri_nodes = np.ascontiguousarray(nodes)
    mesh.circumcenters = cc
    mesh.circumradii = cr
    mesh._vertex_corners = None
    mesh._vertex_triangles = None
    mesh._build_collocation()
    mesh._cache_lock = threading.Lock()
    mesh._table_cache = {}
    mesh._device_cache = {}
    return mesh


def load_mesh(path) -> SurfaceMesh:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_mesh(fh.read(), name=str(path))


def _patch_line(tag, p: PatchSpec) -> str:
    if p.kind == "electrode":
        return f"patch {tag} electrode {p.v0!r}"
    if p.kind == "floating":
        return f"patch {tag} floating {p.index}"
    if p.kind == "sheet":
        return f"patch {tag} sheet {p.index} {p.eps_plus!r} {p.eps_minus!r}"
    return f"patch {tag} dielectric {p.eps_plus!r} {p.eps_minus!r}"


def save_mesh(mesh_or_parts, path) -> None:
    """Write the ``bemesh 1`` format (reference src/mesh.py:542-577)."""
    if isinstance(mesh_or_parts, SurfaceMesh):
        vertices = mesh_or_parts.vertices
        tris = list(zip(mesh_or_parts.tri_node_ids.tolist(), mesh_or_parts.tri_tags.tolist()))
        patches = mesh_or_parts.patches
    else:
        vertices, tris, patches = mesh_or_parts
    lines = ["bemesh 1"]
    lines += [f"vertex {i} {float(p[0])!r} {float(p[1])!r} {float(p[2])!r}"
              for i, p in enumerate(np.asarray(vertices).tolist())]
    lines += ["triangle " + " ".join(str(int(k)) for k in ids) + f" {int(tag)}" for ids, tag in tris]
    lines += [_patch_line(t, patches[t]) for t in sorted(patches)]
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(lines) + "\n")
