"""Seeded synthetic volumes and vectors (restated in DESIGN.md).

* `flame_volume`: flame-like emission -- a conical sheet plus the paper's
  "four-pronged phantom" as four tilted Gaussian prongs, multiplied by
  smooth multiplicative noise, clipped at 0, max-normalised to 1, rasterised with
  2x supersampling per axis (the paper generates data on a finer grid).
  Its support stays inside the central 50% of the box (reading Z14).
* parity inputs: U[0,1) and N(0,1) from numpy PCG64 with fixed seeds.

Layout of every volume: float32 array of shape (nz, ny, nx) -- x fastest in memory
(P:1033-1045).
"""
import numpy as np
from scipy.ndimage import gaussian_filter


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def uniform_volume(vol, seed=0):
    return _rng(seed).random((vol["nz"], vol["ny"], vol["nx"])).astype(np.float32)


def uniform_vector(n, seed=1):
    return _rng(seed).random(n).astype(np.float32)


def normal_vector(n, seed=2):
    return _rng(seed).standard_normal(n).astype(np.float32)


def _segment_dist2(X, Y, Z, a, b):
    ax, ay, az = a
    bx, by, bz = b
    dx, dy, dz = bx - ax, by - ay, bz - az
    t = ((X - ax) * dx + (Y - ay) * dy + (Z - az) * dz) / (dx * dx + dy * dy + dz * dz)
    t = np.clip(t, 0.0, 1.0)
    return (X - ax - t * dx) ** 2 + (Y - ay - t * dy) ** 2 + (Z - az - t * dz) ** 2


def _flame_density(X, Y, Z, L):
    sig = 0.025 * L
    inside = np.abs(Y) <= 0.25 * L
    h = np.clip((Y + 0.25 * L) / (0.5 * L), 0.0, 1.0)
    rho = np.sqrt(X * X + Z * Z)
    r0 = 0.15 * L * (1.0 - h) ** 0.6
    amp = np.where(inside, np.sqrt(np.maximum(np.sin(np.pi * h), 0.0)), 0.0)
    out = amp * np.exp(-(rho - r0) ** 2 / (2.0 * sig * sig))
    base = (0.0, -0.18 * L, 0.0)
    for sx in (-1.0, 1.0):
        for sz in (-1.0, 1.0):
            tip = (sx * 0.15 * L, 0.18 * L, sz * 0.15 * L)
            out = out + np.exp(-_segment_dist2(X, Y, Z, base, tip) / (2.0 * sig * sig))
    return out


def flame_volume(vol, seed=1234, supersample=2):
    """Flame-like phantom on the voxel grid of `vol` (nz, ny, nx) float32, max 1."""
    nx, ny, nz = vol["nx"], vol["ny"], vol["nz"]
    dx, dy, dz = vol["dx"], vol["dy"], vol["dz"]
    L = max(nx * dx, ny * dy, nz * dz)
    ss = supersample
    fx = (np.arange(nx * ss) - (nx * ss - 1) / 2.0) * (dx / ss)
    fy = (np.arange(ny * ss) - (ny * ss - 1) / 2.0) * (dy / ss)
    out = np.zeros((nz, ny, nx), np.float64)
    Yg, Xg = np.meshgrid(fy, fx, indexing="ij")
    for iz in range(nz):
        acc = np.zeros((ny * ss, nx * ss))
        for sub in range(ss):
            z = (iz * ss + sub - (nz * ss - 1) / 2.0) * (dz / ss)
            acc += _flame_density(Xg, Yg, z, L)
        out[iz] = acc.reshape(ny, ss, nx, ss).mean(axis=(1, 3)) / ss
    noise = gaussian_filter(_rng(seed).standard_normal((nz, ny, nx)), sigma=2.0)
    noise /= noise.std()
    out = np.clip(out * (1.0 + 0.3 * noise), 0.0, None)
    out /= out.max()
    return out.astype(np.float32)
