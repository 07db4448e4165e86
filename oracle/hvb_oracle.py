"""CPU ORACLE -- test infrastructure only.

An independent NumPy restatement of the reference hvbem hot path
(reference pkg/src/hvbem/*.py), used ONLY by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg as the checker and the
CPU baseline.  The product path (paper_2003_12663_b200) never imports it.

Pinned against the live reference: tests/golden/make_golden.py imports the
reference in the build container and records matrices, solutions, fields
and traced lines; tests/test_oracle_golden.py checks this module against
those fixtures (parity pinned).

It restates (file:line of the reference):
  * rules: Dunavant (quadrature.py:97-146), Gauss-Legendre / collapsed
    square / split-corner Duffy (149-199), graded composite (343-406);
  * decisions: classification (assembly.py:155-168), flat closest point
    (quadrature.py:236-277), subdivision (296-332), grading trigger (430);
  * rows: regular sweep (assembly.py:173-200), singular Duffy batch
    (202-235), deferred near pass (245-292), row equations (408-468),
    charge functional (540-569);
  * GMRES (solver.py:86-225), fields (postprocess.py:104-170), surface
    distance (198-218), Dormand-Prince tracer (229-357), streamer (365-374).

Vectorisation differs from the reference (whole row blocks at once); the
discrete decisions use the reference's rounding: unfused axis norms and the
ddot FMA chain fma(a2,b2,fma(a1,b1,a0*b0)) measured in the reference
container (exact FMA via rational arithmetic here).
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

FOUR_PI = 4.0 * np.pi
EPS0 = 8.8541878128e-12

# ---------------------------------------------------------------------------
# exact-rounding helpers
# ---------------------------------------------------------------------------


def fma_exact(a: float, b: float, c: float) -> float:
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def ddot3(a, b) -> float:
    """OpenBLAS ddot chain for length-3 vectors (reference container)."""
    return fma_exact(float(a[2]), float(b[2]), fma_exact(float(a[1]), float(b[1]), float(a[0]) * float(b[0])))


def axis_norm(d):
    d = np.asarray(d, dtype=float)
    return np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])


# ---------------------------------------------------------------------------
# rules (reference quadrature.py)
# ---------------------------------------------------------------------------

_DUN = {
    2: [("s", 1.0 / 6.0, 1.0 / 3.0)],
    4: [("s", 0.445948490915965, 0.223381589678011), ("s", 0.091576213509771, 0.109951743655322)],
    6: [("s", 0.249286745170910, 0.116786275726379), ("s", 0.063089014491502, 0.050844906370207),
        ("r", 0.310352451033785, 0.053145049844816, 0.082851075618374)],
    8: [("c", 0.14431560767771356), ("s", 0.45929258829267405, 0.0950916342673329),
        ("s", 0.1705693077517035, 0.10321737053473093), ("s", 0.05054722831703301, 0.032458497623204935),
        ("r", 0.26311282963480714, 0.00839477740988042, 0.027230314174413347)],
}


def dunavant(order):
    uv, w = [], []
    for g in _DUN[order]:
        if g[0] == "c":
            pts, wt = [(1 / 3, 1 / 3)], g[1]
        elif g[0] == "s":
            a, wt = g[1], g[2]
            b = 1.0 - 2.0 * a
            pts = [(a, a), (b, a), (a, b)]  # (l1, l2) of (b,a,a), (a,b,a), (a,a,b)
        else:
            a, b, wt = g[1], g[2], g[3]
            c = 1.0 - a - b
            pts = [(b, c), (c, b), (a, c), (c, a), (a, b), (b, a)]
        uv += pts
        w += [0.5 * wt] * len(pts)
    return np.array(uv), np.array(w)


def _gl01(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def _map(nodes, weights, corners):
    a = corners[0]
    e1 = corners[1] - a
    e2 = corners[2] - a
    out = a + np.outer(nodes[:, 0], e1) + np.outer(nodes[:, 1], e2)
    det = abs(e1[0] * e2[1] - e1[1] * e2[0])
    return out, weights * (2.0 * det) * 0.5


def duffy(corner, n1d):
    s, ws = _gl01(n1d)
    S, T = np.meshgrid(s, s, indexing="ij")
    WS, WT = np.meshgrid(ws, ws, indexing="ij")
    sq = np.column_stack([(S * (1.0 - T)).ravel(), (S * T).ravel()])
    wsq = (WS * WT * S).ravel()
    halves = [np.array([[0.0, 0.0], [1.0, 0.0], [0.5, 0.5]]), np.array([[0.0, 0.0], [0.5, 0.5], [0.0, 1.0]])]
    parts = [_map(sq, wsq, h) for h in halves]
    uv = np.vstack([p[0] for p in parts])
    w = np.concatenate([p[1] for p in parts])
    u, v = uv[:, 0], uv[:, 1]
    l0 = 1.0 - u - v
    if corner == 1:
        u, v = l0, u
    elif corner == 2:
        u, v = v, l0
    return np.column_stack([u, v]), w


def graded(depth, n1d, outer):
    if depth == 0:
        return duffy(0, n1d)
    on, ow = dunavant(outer)
    uvs, ws = [], []
    for lev in range(depth):
        s = 0.5 ** lev
        h = 0.5 * s
        for cell in (np.array([[h, 0.0], [s, 0.0], [0.0, s]]), np.array([[h, 0.0], [0.0, s], [0.0, h]])):
            m01 = 0.5 * (cell[0] + cell[1])
            m12 = 0.5 * (cell[1] + cell[2])
            m20 = 0.5 * (cell[2] + cell[0])
            for ch in (np.array([cell[0], m01, m20]), np.array([m01, cell[1], m12]),
                       np.array([m20, m12, cell[2]]), np.array([m01, m12, m20])):
                n_, w_ = _map(on, ow, ch)
                uvs.append(n_)
                ws.append(w_)
    dn, dw = duffy(0, n1d)
    sc = 0.5 ** depth
    uvs.append(dn * sc)
    ws.append(dw * sc * sc)
    return np.vstack(uvs), np.concatenate(ws)


def shape6(uv):
    u, v = uv[:, 0], uv[:, 1]
    w = 1.0 - u - v
    N = np.stack([w * (2 * w - 1), u * (2 * u - 1), v * (2 * v - 1), 4 * w * u, 4 * u * v, 4 * v * w], 1)
    Nu = np.stack([1 - 4 * w, 4 * u - 1, 0 * u, 4 * (w - u), 4 * v, -4 * v], 1)
    Nv = np.stack([1 - 4 * w, 0 * u, 4 * v - 1, -4 * u, 4 * u, 4 * (w - v)], 1)
    return N, Nu, Nv


def curved(nodes6, uv):
    """points and area elements of one curved triangle at uv (m,2)."""
    N, Nu, Nv = shape6(uv)
    p = N @ nodes6
    cr = np.cross(Nu @ nodes6, Nv @ nodes6)
    return p, np.sqrt(np.sum(cr * cr, axis=1))


# ---------------------------------------------------------------------------
# per-pair decisions
# ---------------------------------------------------------------------------


def closest_point_flat(x, a, b, c):
    ab, ac = b - a, c - a
    d1, d2 = ddot3(ab, x - a), ddot3(ac, x - a)
    if d1 <= 0.0 and d2 <= 0.0:
        return 0.0, 0.0
    d3, d4 = ddot3(ab, x - b), ddot3(ac, x - b)
    if d3 >= 0.0 and d4 <= d3:
        return 1.0, 0.0
    d5, d6 = ddot3(ab, x - c), ddot3(ac, x - c)
    if d6 >= 0.0 and d5 <= d6:
        return 0.0, 1.0
    vc = d1 * d4 - d3 * d2
    if vc <= 0.0 and d1 >= 0.0 and d3 <= 0.0:
        return d1 / (d1 - d3), 0.0
    vb = d5 * d2 - d1 * d6
    if vb <= 0.0 and d2 >= 0.0 and d6 <= 0.0:
        return 0.0, d2 / (d2 - d6)
    va = d3 * d6 - d5 * d4
    if va <= 0.0 and (d4 - d3) >= 0.0 and (d5 - d6) >= 0.0:
        t = (d4 - d3) / ((d4 - d3) + (d5 - d6))
        return 1.0 - t, t
    den = 1.0 / (va + vb + vc)
    return vb * den, vc * den


_REF = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])


def near_rule(x, nodes6, R, cfg):
    """(uv, w) of the near-singular composite rule (quadrature.py:409-450)."""
    a, b, c = nodes6[0], nodes6[1], nodes6[2]
    us, vs = closest_point_flat(x, a, b, c)
    nearest = a + us * (b - a) + vs * (c - a)
    dd = x - nearest
    dist = math.sqrt(ddot3(dd, dd))
    depth = cfg["bisect_depth"] if dist < cfg["bisect_trigger"] * R else 0
    bn, bw = graded(depth, cfg["near_duffy_points"], cfg["near_outer_order"])
    bary = np.array([1.0 - us - vs, us, vs])
    p = np.array([us, vs])
    one = np.nonzero(bary > 1.0 - 1e-9)[0]
    if one.size:
        k = int(one[0])
        subs = [np.roll(_REF, -k, axis=0)]
    else:
        zero = np.nonzero(bary < 1e-9)[0]
        c0, c1, c2 = _REF
        if zero.size and zero[0] == 0:
            subs = [np.array([p, c2, c0]), np.array([p, c0, c1])]
        elif zero.size and zero[0] == 1:
            subs = [np.array([p, c0, c1]), np.array([p, c1, c2])]
        elif zero.size:
            subs = [np.array([p, c1, c2]), np.array([p, c2, c0])]
        else:
            subs = [np.array([p, c0, c1]), np.array([p, c1, c2]), np.array([p, c2, c0])]
    uvs, ws = [], []
    for cc in subs:
        pieces = [cc] if depth == 0 else [np.array([cc[0], cc[1], 0.5 * (cc[1] + cc[2])]),
                                          np.array([cc[0], 0.5 * (cc[1] + cc[2]), cc[2]])]
        for pc in pieces:
            n_, w_ = _map(bn, bw, pc)
            uvs.append(n_)
            ws.append(w_)
    return np.vstack(uvs), np.concatenate(ws)


DEFAULT_CFG = dict(regular_order=6, duffy_points=6, near_duffy_points=8, near_outer_order=8, eta=1.2,
                   bisect_depth=3, bisect_trigger=0.3)


# ---------------------------------------------------------------------------
# kernel rows
# ---------------------------------------------------------------------------


class Tables:
    def __init__(self, mesh, order):
        uv, w = dunavant(order)
        N, Nu, Nv = shape6(uv)
        X = mesh.tri_nodes
        self.pts = np.einsum("qk,tkd->tqd", N, X)
        cr = np.cross(np.einsum("qk,tkd->tqd", Nu, X), np.einsum("qk,tkd->tqd", Nv, X))
        self.jw = w[None, :] * np.sqrt(np.sum(cr * cr, axis=2))
        self.hats = np.column_stack([1.0 - uv[:, 0] - uv[:, 1], uv[:, 0], uv[:, 1]])


def _kernel(kind, d, n_x):
    r = np.sqrt(np.sum(d * d, axis=-1))
    if kind == "sl":
        return 1.0 / (FOUR_PI * r)
    if kind == "adl":
        return (d @ n_x) / (FOUR_PI * r ** 3)
    return d / (FOUR_PI * r ** 3)[..., None]


def kernel_rows(mesh, X, own_cols, kind, normals=None, cfg=None, tables=None):
    """Full kernel rows (regular + singular + near) for points X (R,3).
    kind 'sl' / 'adl' -> (R, n); 'efield' -> (R, n, 3).  Returns (rows,
    near_pairs list of (r, t))."""
    cfg = {**DEFAULT_CFG, **(cfg or {})}
    tab = tables or Tables(mesh, cfg["regular_order"])
    n = mesh.n_collocation
    nt = mesh.n_triangles
    X = np.asarray(X, dtype=float).reshape(-1, 3)
    R = len(X)
    vec = kind == "efield"
    out = np.zeros((R, n, 3) if vec else (R, n))
    cols = mesh.tri_corner_cols
    thr = cfg["eta"] * mesh.circumradii
    near_pairs = []
    for r in range(R):
        x = X[r]
        own = own_cols[r] if own_cols is not None else -1
        n_x = normals[r] if normals is not None else None
        regular = axis_norm(x[None, :] - mesh.circumcenters) > thr
        sing = np.zeros(nt, dtype=bool)
        if own >= 0:
            star = np.nonzero((cols == own).any(axis=1))[0]
            sing[star] = True
        regular &= ~sing
        d = x[None, None, :] - tab.pts
        k = _kernel(kind, d, n_x)
        if vec:
            k = k * tab.jw[..., None]
            k[~regular] = 0.0
            con = np.einsum("tqd,qc->tcd", k, tab.hats)
            for ax in range(3):
                out[r, :, ax] = np.bincount(cols.ravel(), con[:, :, ax].ravel(), minlength=n)
        else:
            k = k * tab.jw
            k[~regular] = 0.0
            out[r] = np.bincount(cols.ravel(), (k @ tab.hats).ravel(), minlength=n)
        # singular (assembly.py:202-235)
        if own >= 0:
            for t, c in zip(mesh.vc_tri[mesh.vc_ptr[own]:mesh.vc_ptr[own + 1]],
                            mesh.vc_corner[mesh.vc_ptr[own]:mesh.vc_ptr[own + 1]]):
                uv, w = duffy(int(c), cfg["duffy_points"])
                _add_pair(out[r], mesh.tri_nodes[t], uv, w, x, kind, n_x, cols[t])
        # near (assembly.py:245-292)
        for t in np.nonzero(~regular & ~sing)[0]:
            near_pairs.append((r, int(t)))
            uv, w = near_rule(x, mesh.tri_nodes[t], mesh.circumradii[t], cfg)
            _add_pair(out[r], mesh.tri_nodes[t], uv, w, x, kind, n_x, cols[t])
    return out, near_pairs


def _add_pair(row, nodes6, uv, w, x, kind, n_x, cols):
    p, jac = curved(nodes6, uv)
    k = _kernel(kind, x[None, :] - p, n_x)
    hats = np.column_stack([1.0 - uv[:, 0] - uv[:, 1], uv[:, 0], uv[:, 1]])
    wj = w * jac
    for c in range(3):
        if k.ndim == 2:
            row[cols[c]] += np.sum(k * (wj * hats[:, c])[:, None], axis=0)
        else:
            row[cols[c]] += np.sum(k * wj * hats[:, c])


# ---------------------------------------------------------------------------
# system
# ---------------------------------------------------------------------------


def row_equations(mesh, rows, cfg=None, tables=None):
    """Dense rows of the system (assembly.py:408-468) for the given indices."""
    cfg = {**DEFAULT_CFG, **(cfg or {})}
    tab = tables or Tables(mesh, cfg["regular_order"])
    n = mesh.n_collocation
    size = n + mesh.n_floating
    out = np.zeros((len(rows), size))
    for k, row in enumerate(rows):
        if row < n:
            code = mesh.row_kind_code[row]
            if code in (0, 1):
                r, _ = kernel_rows(mesh, mesh.colloc_points[row:row + 1], [row], "sl", cfg=cfg, tables=tab)
                out[k, :n] = r[0]
                if code == 1:
                    out[k, n + mesh.row_float[row]] = -1.0
            else:
                r, _ = kernel_rows(mesh, mesh.colloc_points[row:row + 1], [row], "adl",
                                   normals=mesh.colloc_normals[row:row + 1], cfg=cfg, tables=tab)
                ep, em = mesh.row_eps_plus[row], mesh.row_eps_minus[row]
                out[k, :n] = (ep - em) * r[0]
                out[k, row] += 0.5 * (ep + em)
        else:
            kk = row - n
            members = np.nonzero((mesh.row_kind_code == 1) & (mesh.row_float == kk))[0]
            adl, ids = neutrality_scales(mesh, kk)
            out[k, :n] = charge_vector(mesh, members, adl, ids, cfg, tab)
    return out


def neutrality_scales(mesh, k):
    for p in mesh.patches.values():
        if p.kind == "sheet" and p.index == k:
            return p.eps_plus - p.eps_minus, 0.5 * (p.eps_plus + p.eps_minus)
    return EPS0, 0.5 * EPS0


def charge_vector(mesh, members, adl, ids, cfg=None, tables=None):
    n = mesh.n_collocation
    q = np.zeros(n)
    for i in members:
        r, _ = kernel_rows(mesh, mesh.colloc_points[i:i + 1], [i], "adl", normals=mesh.colloc_normals[i:i + 1],
                           cfg=cfg, tables=tables)
        w = mesh.lumped_weights[i]
        q += w * adl * r[0]
        q[i] += w * ids
    return q


def assemble_dense(mesh, cfg=None):
    size = mesh.n_collocation + mesh.n_floating
    return row_equations(mesh, range(size), cfg)


def rhs(mesh):
    r = np.where(mesh.row_kind_code == 0, mesh.row_v0, 0.0)
    return np.concatenate([r, np.zeros(mesh.n_floating)])


def entry_error(a, b, floor=1e-4):
    """max_ij |a-b| / max(|b_ij|, floor*||b_i||_inf): <= 1e-10 means every
    entry matches to 1e-10 relative or 1e-14 of its row's max."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    rowmax = np.max(np.abs(b), axis=1, keepdims=True)
    den = np.maximum(np.abs(b), floor * rowmax)
    den = np.where(den > 0, den, 1.0)
    return float(np.max(np.abs(a - b) / den))


# ---------------------------------------------------------------------------
# GMRES (solver.py:86-225) -- restated for semantics tests
# ---------------------------------------------------------------------------


def gmres(A, b, restart=100, rel_tol=1e-8, max_iters=2000, row_equilibrate=True, matvec=None):
    """``matvec`` (optional) replaces A @ z in the operator and the true
    residual -- e.g. the reference's float32 row dots for single storage
    (assembly.py:386-392); row scales and the diagonal come from A."""
    mv = matvec or (lambda z: np.asarray(A, dtype=float) @ z)
    A = np.asarray(A, dtype=float)
    b = np.asarray(b, dtype=float)
    N = len(b)
    left = 1.0 / np.where(np.abs(A).max(axis=1) > 0, np.abs(A).max(axis=1), 1.0) if row_equilibrate else np.ones(N)
    d = np.diag(A) * left
    right = np.where(np.abs(d) < 1e-30, 1.0, d)
    bs = left * b
    nbs, nb = np.linalg.norm(bs), np.linalg.norm(b)
    if nb == 0:
        return np.zeros(N), 0, 0.0

    def op(z):
        return left * mv(z / right)

    def tres(x):
        return np.linalg.norm(b - mv(x)) / nb

    x = np.zeros(N)
    it = 0
    best = np.inf
    while it < max_iters:
        r = bs - op(x)
        beta = np.linalg.norm(r)
        if beta / nbs <= rel_tol and tres(x / right) <= rel_tol:
            return x / right, it, tres(x / right)
        md = min(restart, max_iters - it)
        V = np.zeros((md + 1, N))
        H = np.zeros((md + 1, md))
        cs, sn, g = np.zeros(md), np.zeros(md), np.zeros(md + 1)
        g[0] = beta
        V[0] = r / beta
        used, conv = 0, False
        for j in range(md):
            w = op(V[j])
            n0 = np.linalg.norm(w)
            for i in range(j + 1):
                H[i, j] = V[i] @ w
                w = w - H[i, j] * V[i]
            n1 = np.linalg.norm(w)
            if n1 < n0 / np.sqrt(2.0):
                for i in range(j + 1):
                    c_ = V[i] @ w
                    H[i, j] += c_
                    w = w - c_ * V[i]
                n1 = np.linalg.norm(w)
            H[j + 1, j] = n1
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            if den == 0.0:
                used, conv = j, True
                break
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            used = j + 1
            if n1 == 0.0:
                conv = True
                break
            V[j + 1] = w / n1
            if abs(g[j + 1]) <= rel_tol * nbs:
                conv = True
                break
        if used:
            y = np.linalg.solve(np.triu(H[:used, :used]), g[:used])
            x = x + V[:used].T @ y
        it += used
        tr = tres(x / right)
        best = min(best, tr)
        if conv and tr <= rel_tol:
            return x / right, it, tr
    raise RuntimeError(f"oracle GMRES did not converge (best {best:.3e})")


# ---------------------------------------------------------------------------
# fields (postprocess.py:104-170)
# ---------------------------------------------------------------------------


def efield_points(mesh, u, X, cfg=None, tables=None):
    rows, _ = kernel_rows(mesh, X, None, "efield", cfg=cfg, tables=tables)
    return np.einsum("j,rjd->rd", np.asarray(u), rows)


def potential_points(mesh, u, X, cfg=None):
    rows, _ = kernel_rows(mesh, X, None, "sl", cfg=cfg)
    return rows @ np.asarray(u)


def surface_field(mesh, u, side=1.0, cfg=None, indices=None):
    idx = np.arange(mesh.n_collocation) if indices is None else np.asarray(indices)
    out = np.empty(len(idx))
    tab = Tables(mesh, {**DEFAULT_CFG, **(cfg or {})}["regular_order"])
    for k, i in enumerate(idx):
        rows, _ = kernel_rows(mesh, mesh.colloc_points[i:i + 1], [i], "efield", cfg=cfg, tables=tab)
        e = np.asarray(u) @ rows[0] + side * 0.5 * u[i] * mesh.colloc_normals[i]
        out[k] = np.linalg.norm(e)
    return out


def streamer(arcs, mags, e_tab, a_tab, k_str):
    a = np.interp(mags, e_tab, a_tab)
    v = float(np.sum(0.5 * (a[1:] + a[:-1]) * np.diff(arcs)))
    return v, v > k_str


# ---------------------------------------------------------------------------
# surface distance and field-line tracer (postprocess.py:198-357)
# ---------------------------------------------------------------------------


def surface_distance(mesh, x, candidates=12):
    """(d_surf, local R): 12 circumcircle candidates by ||x-cc||-R, flat
    closest point mapped through the quadratic patch (postprocess.py:198-218)."""
    x = np.asarray(x, dtype=float)
    lower = axis_norm(mesh.circumcenters - x[None, :]) - mesh.circumradii
    order = np.argsort(lower, kind="stable")[:candidates]
    best, local = np.inf, mesh.circumradii[order[0]]
    for t in order:
        X6 = mesh.tri_nodes[t]
        u, v = closest_point_flat(x, X6[0], X6[1], X6[2])
        p, _ = curved(X6, np.array([[u, v]]))
        dd = x - p[0]
        d = math.sqrt(ddot3(dd, dd))
        if d < best:
            best, local = d, mesh.circumradii[t]
    return float(best), float(local)


_DPA = ((), (1 / 5,), (3 / 40, 9 / 40), (44 / 45, -56 / 15, 32 / 9),
        (19372 / 6561, -25360 / 2187, 64448 / 6561, -212 / 729),
        (9017 / 3168, -355 / 33, 46732 / 5247, 49 / 176, -5103 / 18656),
        (35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84))
_DPB5 = np.array([35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84, 0.0])
_DPB4 = np.array([5179 / 57600, 0.0, 7571 / 16695, 393 / 640, -92097 / 339200, 187 / 2100, 1 / 40])


def trace_line(mesh, u, start, orientation=1, rel_tol=1e-6, h_min_frac=1e-6, h_max_frac=0.05, surface_tol_frac=0.1,
               e_floor=0.0, max_length_frac=4.0, bbox_factor=1.5, cfg=None, efield=None, tables=None):
    """Dormand-Prince 5(4) on the unit tangent (postprocess.py:244-357).
    Returns (points (m,3), |E| (m,), arcs (m,), termination).  ``efield``
    overrides the field evaluator (default: oracle kernel rows)."""
    tab = tables or Tables(mesh, {**DEFAULT_CFG, **(cfg or {})}["regular_order"])
    ev = efield or (lambda p: efield_points(mesh, u, p[None], cfg, tab)[0])
    lo, hi = mesh.vertices.min(axis=0), mesh.vertices.max(axis=0)
    center, half = 0.5 * (lo + hi), 0.5 * (hi - lo) * bbox_factor
    diag = math.sqrt(ddot3(hi - lo, hi - lo))
    h_min, h_max, l_max = h_min_frac * diag, h_max_frac * diag, max_length_frac * diag
    sign = 1.0 if orientation >= 0 else -1.0

    def tangent(p):
        e = ev(p)
        mag = math.sqrt(ddot3(e, e))
        if mag <= e_floor or mag == 0.0:
            return None, mag
        return sign * e / mag, mag

    x = np.asarray(start, dtype=float)
    t0, mag0 = tangent(x)
    if t0 is None:
        raise ValueError("weak field at the start point")
    pts, mags, arcs = [x.copy()], [mag0], [0.0]
    term, h, s, k1, armed = "MaxLength", h_max, 0.0, t0, False
    while True:
        d_surf, local_r = surface_distance(mesh, x)
        hit = surface_tol_frac * local_r
        if d_surf > 2.0 * hit:
            armed = True
        if armed and d_surf < hit:
            term = "SurfaceHit"
            xe = x + k1 * d_surf
            pts[-1] = xe
            arcs[-1] += d_surf
            e = ev(xe)
            mags[-1] = math.sqrt(ddot3(e, e))
            break
        if s >= l_max:
            break
        if np.any(np.abs(x - center) > half):
            term = "LeftDomain"
            break
        h_cap = h_max if d_surf > 4.0 * h_max else max(h_min, 0.45 * d_surf)
        h = min(h, h_cap, l_max - s + h_min)
        ks, failed = [k1], False
        for stage in range(1, 7):
            acc = 0
            for a, k in zip(_DPA[stage], ks):
                acc = acc + a * k
            ti, _ = tangent(x + h * acc)
            if ti is None:
                term, failed = "WeakField", True
                break
            ks.append(ti)
        if failed:
            break
        K = np.array(ks)
        x5, x4 = x + h * (_DPB5 @ K), x + h * (_DPB4 @ K)
        dd = x5 - x4
        err = math.sqrt(ddot3(dd, dd))
        tol = rel_tol * max(1.0, math.sqrt(ddot3(x5, x5)) / diag) * diag
        if err <= tol or h <= h_min * 1.0000001:
            x, s = x5, s + h
            t_new, mag_new = tangent(x)
            pts.append(x.copy())
            mags.append(mag_new)
            arcs.append(s)
            if t_new is None:
                term = "WeakField"
                break
            k1 = t_new
        factor = 0.9 * (tol / err) ** 0.2 if err > 0.0 else 2.0
        h = float(np.clip(h * np.clip(factor, 0.2, 2.0), h_min, h_max))
    return np.array(pts), np.array(mags), np.array(arcs), term
