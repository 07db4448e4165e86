"""Bit-faithful floating-point helpers for the host-side geometry.

The reference's discrete decisions (pair classification, flat closest point,
subdivision, grading trigger, circumcircles) are computed by NumPy whose 1-d
``a @ b`` on length-3 float64 vectors goes through OpenBLAS ``ddot``; in the
reference container that kernel evaluates the fused chain
``fma(a2, b2, fma(a1, b1, a0*b0))`` (measured: 0 mismatches in 2e5 random
triples).  Axis reductions
(``np.linalg.norm(d, axis=1)``) are unfused ``(d0*d0 + d1*d1) + d2*d2``.

The CUDA kernels reproduce the same chains with ``fma`` and ``__dmul_rn`` /
``__dadd_rn``.  On the host we need a vectorised correctly rounded FMA, which
NumPy lacks; :func:`fma` emulates it exactly with the Boldo-Melquiond
round-to-odd construction (error-free TwoProd/TwoSum + one odd rounding).
"""

from __future__ import annotations

import numpy as np

_SPLIT = 134217729.0  # 2**27 + 1 (Veltkamp splitter for binary64)


def _two_sum(a, b):
    s = a + b
    bb = s - a
    err = (a - (s - bb)) + (b - bb)
    return s, err


def _split(a):
    c = _SPLIT * a
    hi = c - (c - a)
    return hi, a - hi


def _two_prod(a, b):
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    err = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return p, err


def _add_round_odd(a, b):
    """a + b rounded to odd (exact sum, then force an odd last bit when the
    nearest rounding was inexact)."""
    s, e = _two_sum(a, b)
    s = np.asarray(s, dtype=np.float64)
    e = np.asarray(e, dtype=np.float64)
    bits = s.view(np.int64)
    even = (bits & 1) == 0
    fix = (e != 0.0) & even
    if np.any(fix):
        toward = np.where(e > 0.0, np.inf, -np.inf)
        s = np.where(fix, np.nextafter(s, toward), s)
    return s


def fma(a, b, c):
    """Correctly rounded a*b + c, elementwise (no overflow/underflow handling
    beyond what the mesh coordinates need)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    ph, pl = _two_prod(a, b)
    uh, ul = _two_sum(c, pl)
    th, tl = _two_sum(ph, uh)
    v = _add_round_odd(tl, ul)
    out = th + v
    # exact zero products / non-finite inputs: fall back to plain arithmetic
    bad = ~np.isfinite(out) | ~np.isfinite(ph)
    if np.any(bad):
        out = np.where(bad, a * b + c, out)
    return out


def dot3(a, b):
    """Length-3 dot product along the last axis with the reference's
    ddot rounding: fma(a2, b2, fma(a1, b1, a0*b0))."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    acc = a[..., 0] * b[..., 0]
    acc = fma(a[..., 1], b[..., 1], acc)
    return fma(a[..., 2], b[..., 2], acc)


def norm3_fused(d):
    """np.linalg.norm of a single 3-vector (sqrt of the ddot chain)."""
    return np.sqrt(dot3(d, d))


def norm3_axis(d):
    """np.linalg.norm(d, axis=-1) for 3-vectors: unfused (x*x + y*y) + z*z."""
    d = np.asarray(d, dtype=np.float64)
    return np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])


def cross3(a, b):
    """np.cross for 3-vectors (unfused products and differences)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    out = np.empty(np.broadcast_shapes(a.shape, b.shape))
    out[..., 0] = a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1]
    out[..., 1] = a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2]
    out[..., 2] = a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]
    return out
