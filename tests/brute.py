"""Brute-force evaluators used to pin the oracle (test code only, independent of oracle/).

* `strip_polygon_area`: exact area of an intersection of strips |alpha.s + beta.u - gamma| <= h/2
  in the (s,u) plane by half-plane clipping of a large box -- the inner product of
  eqn,xport,ip for rect spatial and pillbox angular bases is exactly
  such an area (each factor is an indicator of a strip).
* `interval_overlap`: 1D overlap length (for the Dirac angular basis).
"""
import numpy as np


def _clip(poly, a, b, c):
    """Keep the part of convex polygon `poly` with a*s + b*u <= c."""
    out = []
    n = len(poly)
    for k in range(n):
        p, q = poly[k], poly[(k + 1) % n]
        fp = a * p[0] + b * p[1] - c
        fq = a * q[0] + b * q[1] - c
        if fp <= 0:
            out.append(p)
        if (fp < 0 < fq) or (fq < 0 < fp):
            t = fp / (fp - fq)
            out.append((p[0] + t * (q[0] - p[0]), p[1] + t * (q[1] - p[1])))
    return out


def _area(poly):
    if len(poly) < 3:
        return 0.0
    s = 0.0
    for k in range(len(poly)):
        x0, y0 = poly[k]
        x1, y1 = poly[(k + 1) % len(poly)]
        s += x0 * y1 - x1 * y0
    return abs(s) / 2.0


def strip_polygon_area(strips, box):
    """strips: list of (alpha, beta, centre, width) meaning |alpha*s + beta*u - centre| <= width/2."""
    s0, s1, u0, u1 = box
    poly = [(s0, u0), (s1, u0), (s1, u1), (s0, u1)]
    for a, b, c, w in strips:
        poly = _clip(poly, a, b, c + 0.5 * w)
        poly = _clip(poly, -a, -b, -(c - 0.5 * w))
        if not poly:
            return 0.0
    return _area(poly)


def interval_overlap(a0, a1, b0, b1):
    return max(0.0, min(a1, b1) - max(a0, b0))


def quad2(f, x0, x1, y0, y1, n=400):
    """Midpoint-rule 2D quadrature."""
    xs = x0 + (np.arange(n) + 0.5) * (x1 - x0) / n
    ys = y0 + (np.arange(n) + 0.5) * (y1 - y0) / n
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    return f(X, Y).sum() * (x1 - x0) * (y1 - y0) / (n * n)
