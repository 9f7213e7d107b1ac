"""Paraxial ray optics, one separable axis at a time (paper §2.1).

A ray at a plane is theta = (s, u, t, v); transforms are separable
affine maps with a 2x2 block per axis plus offsets (display P:685-709).  The
missing tab,optics is replaced by the standard ray-transfer matrices
(reading Z1):

  propagation  T_d : s' = s + d u,  u' = u
  thin lens    R_f(c): s' = s,      u' = u - (s - c)/f

`Affine1D` is the (s,u) block [[m00, m01], [m10, m11]] with offsets (o0, o1).
Expression order is fixed (written out, no BLAS) because the plan's integer band
tables must agree bit-for-bit with an independent implementation (reading Z21).
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class Affine1D:
    m00: float
    m01: float
    m10: float
    m11: float
    o0: float = 0.0
    o1: float = 0.0

    def apply(self, s, u):
        return self.m00 * s + self.m01 * u + self.o0, self.m10 * s + self.m11 * u + self.o1

    def det(self):
        return self.m00 * self.m11 - self.m01 * self.m10


IDENTITY = Affine1D(1.0, 0.0, 0.0, 1.0, 0.0, 0.0)


def translate(d):
    """T_d: free-space propagation by distance d along the optical axis."""
    return Affine1D(1.0, d, 0.0, 1.0, 0.0, 0.0)


def lens(f, c=0.0):
    """R_f(c): ideal thin lens of focal length f centred at c (u' = u - (s - c)/f)."""
    if f == 0.0:
        raise ValueError("zero focal length")
    return Affine1D(1.0, 0.0, -1.0 / f, 1.0, 0.0, c / f)


def compose(a, b):
    """(a o b): apply b first, then a (P:677 'o denotes function composition')."""
    return Affine1D(
        a.m00 * b.m00 + a.m01 * b.m10,
        a.m00 * b.m01 + a.m01 * b.m11,
        a.m10 * b.m00 + a.m11 * b.m10,
        a.m10 * b.m01 + a.m11 * b.m11,
        a.m00 * b.o0 + a.m01 * b.o1 + a.o0,
        a.m10 * b.o0 + a.m11 * b.o1 + a.o1,
    )


def invert(a):
    """Inverse map; a singular block is an error naming the block."""
    det = a.m00 * a.m11 - a.m01 * a.m10
    if abs(det) <= 1e-12:
        raise ValueError("singular (s,u) block, det=%g" % det)
    i00 = a.m11 / det
    i01 = -a.m01 / det
    i10 = -a.m10 / det
    i11 = a.m00 / det
    return Affine1D(i00, i01, i10, i11,
                    -(i00 * a.o0 + i01 * a.o1),
                    -(i10 * a.o0 + i11 * a.o1))
