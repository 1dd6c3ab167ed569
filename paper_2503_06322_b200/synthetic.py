"""Seeded, SIMD-invariant synthetic fields for the benchmark configurations.

Only elementwise + - * / and uniform draws are used (no libm transcendental,
FFT, normal draws or data reductions), so the same seed gives bit-identical
arrays on every x86 host regardless of the SIMD path numpy dispatches to
(SURVEY §8d).  Recipes:

* ``grf``       -- Gaussian-like random field: uniform noise on a grid padded
                   by m per side, m passes of the 3-point box filter per axis,
                   centre crop, analytic unit-variance scale.            (C1, C3)
* ``smooth_noise`` -- polynomial field 4x(1-x)(1-2y)^2 + 4z(1-z)(2z-1) plus
                   1e-3 uniform noise.                                 (C2, C4, C5)
* ``nyx_like``  -- densities e(1.5 g), temperature 1e4 e(1.15 g), velocities
                   1e7 g with e(x) = (1 + x/1024)^1024 by 10 squarings.   (C3)
"""
from __future__ import annotations

import hashlib
import math
from fractions import Fraction

import numpy as np


def _box_weights_sq_sum(m: int) -> Fraction:
    w = [Fraction(1)]
    for _ in range(m):
        nw = [Fraction(0)] * (len(w) + 2)
        for i, v in enumerate(w):
            for j in range(3):
                nw[i + j] += v / 3
        w = nw
    return sum(v * v for v in w)


def grf(shape, m: int = 8, seed: int = 0, dtype=np.float32) -> np.ndarray:
    shape = tuple(int(s) for s in shape)
    d = len(shape)
    rng = np.random.default_rng(seed)
    a = rng.random(tuple(s + 2 * m for s in shape))
    a *= 2.0
    a -= 1.0
    for axis in range(d):
        for _ in range(m):
            lo = [slice(None)] * d
            mid = [slice(None)] * d
            hi = [slice(None)] * d
            lo[axis] = slice(0, -2)
            mid[axis] = slice(1, -1)
            hi[axis] = slice(2, None)
            t = a[tuple(lo)] + a[tuple(mid)]
            t += a[tuple(hi)]
            t /= 3.0
            a[tuple(mid)] = t
    crop = tuple(slice(m, m + s) for s in shape)
    out = np.ascontiguousarray(a[crop])
    var = Fraction(1, 3) * _box_weights_sq_sum(m) ** d
    scale = 1.0 / math.sqrt(float(var))
    out *= scale
    return out.astype(dtype)


def smooth_noise(shape, seed: int = 0, noise: float = 1e-3, dtype=np.float32, planes=None) -> np.ndarray:
    """f = 4x(1-x)(1-2y)^2 + 4z(1-z)(2z-1) + noise*(2u-1) on the unit cube
    (the last three axes; leading axes repeat the pattern).

    ``planes=(lo, hi)`` (3-D only) returns exactly ``smooth_noise(shape)[lo:hi]`` without
    generating the rest: the uniform stream is advanced past the first lo planes' draws (one
    64-bit draw per value), so a rank can build its own dim-0 block of a field that does not fit
    one host (C4 / C5 block partitions)."""
    orig = tuple(int(s) for s in shape)
    shape = orig
    while len(shape) < 3:
        shape = (1,) + shape
    n0, n1, n2 = shape[-3:]
    lo, hi = 0, n0
    if planes is not None:
        if len(orig) != 3:
            raise ValueError("planes= needs a 3-D shape")
        lo, hi = int(planes[0]), int(planes[1])
        if not 0 <= lo <= hi <= n0:
            raise ValueError("planes out of range")

    def coord(n):
        return np.arange(n, dtype=np.float64) / float(max(n - 1, 1))

    x, y, z = coord(n0), coord(n1), coord(n2)
    px = 4.0 * x * (1.0 - x)
    qy = (1.0 - 2.0 * y) * (1.0 - 2.0 * y)
    rz = 4.0 * z * (1.0 - z) * (2.0 * z - 1.0)
    rng = np.random.default_rng(seed)
    if lo:
        rng.bit_generator.advance(lo * n1 * n2)
    out = np.empty(shape[:-3] + (hi - lo, n1, n2), dtype=dtype)
    flat = out.reshape((-1, hi - lo, n1, n2))
    slab = max(1, (1 << 24) // max(1, n1 * n2))   # consecutive draws: same stream as one call
    for i in range(flat.shape[0]):
        for a in range(lo, hi, slab):
            b = min(hi, a + slab)
            f = px[a:b, None, None] * qy[None, :, None]
            f = f + rz[None, None, :]
            u = rng.random((b - a, n1, n2))
            u *= 2.0
            u -= 1.0
            u *= noise
            f += u
            flat[i, a - lo:b - lo] = f
    return out.reshape(orig if planes is None else (hi - lo, n1, n2))


def _e(x: np.ndarray) -> np.ndarray:
    y = 1.0 + x / 1024.0
    for _ in range(10):
        y = y * y
    return y


NYX_FIELDS = ("baryon_density", "dark_matter_density", "temperature",
              "velocity_x", "velocity_y", "velocity_z")


def nyx_like(shape, field: str, seed: int | None = None, dtype=np.float32) -> np.ndarray:
    idx = NYX_FIELDS.index(field)
    g = grf(shape, m=8, seed=idx if seed is None else seed, dtype=np.float64)
    if field in ("baryon_density", "dark_matter_density"):
        out = _e(1.5 * g)
    elif field == "temperature":
        out = 1e4 * _e(1.15 * g)
    else:
        out = 1e7 * g
    return out.astype(dtype)


def sha256(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).view(np.uint8).reshape(-1)).hexdigest()
