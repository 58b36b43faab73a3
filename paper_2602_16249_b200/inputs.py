"""Synthetic workload generation for the hot path (host side, numpy).

* Perlin patch masks with exact masked counts, restating ``perlin_field`` +
  ``mask_from_field`` (proj/src/masking.cpp:21-92; constants
  proj/include/affmae/masking.hpp:36-38), vectorised.
* Visible patch-centre coordinates ``c*patch + patch/2`` in ascending patch
  index (proj/src/geometry.cpp:44-50, proj/src/pipeline.cpp:412-427).
* The op-sweep tensors of SURVEY.md §8(d): q/k/v/blanks ~ 0.5 N(0,1), a BiasNet
  drawn like ``BiasNet::init`` (proj/src/attention.cpp:16-31), dO ~ N(0,1),
  merge scores ~ U(0.1, 0.9).
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def mix64(z):
    """splitmix64 finaliser (proj/include/affmae/rng.hpp:8-13), vectorised on uint64."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLD
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _corner_gradient(seed, ix, iy):
    # proj/src/masking.cpp:21-26
    with np.errstate(over="ignore"):
        k = mix64(mix64(ix.astype(np.uint64) * _GOLD ^ iy.astype(np.uint64)) ^ np.uint64(seed))
    ang = (k >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 6.283185307179586476925287
    return np.cos(ang), np.sin(ang)


def _fade(t):
    return t * t * t * (t * (t * 6.0 - 15.0) + 10.0)


def _octave(x, y, seed):
    # perlin_octave_at, proj/src/masking.cpp:34-49
    fx0, fy0 = np.floor(x), np.floor(y)
    x0, y0 = fx0.astype(np.int64), fy0.astype(np.int64)
    tx, ty = x - fx0, y - fy0
    gx, gy = _corner_gradient(seed, x0, y0)
    n00 = gx * tx + gy * ty
    gx, gy = _corner_gradient(seed, x0 + 1, y0)
    n10 = gx * (tx - 1.0) + gy * ty
    gx, gy = _corner_gradient(seed, x0, y0 + 1)
    n01 = gx * tx + gy * (ty - 1.0)
    gx, gy = _corner_gradient(seed, x0 + 1, y0 + 1)
    n11 = gx * (tx - 1.0) + gy * (ty - 1.0)
    u, v = _fade(tx), _fade(ty)
    a = n00 + (n10 - n00) * u
    b = n01 + (n11 - n01) * u
    return a + (b - a) * v


def perlin_field(h, w, octaves=2, base_freq=4.0, persistence=0.5, seed=1):
    """proj/src/masking.cpp:51-69."""
    field = np.zeros((h, w))
    ii, jj = np.meshgrid(np.arange(h, dtype=np.float64), np.arange(w, dtype=np.float64),
                         indexing="ij")
    for o in range(octaves):
        freq = base_freq * float(1 << o)
        amp = persistence ** o
        with np.errstate(over="ignore"):
            os_ = int(mix64(np.uint64(seed) + _GOLD * np.uint64(o + 1)))
        py = ii * freq / float(h)
        px = jj * freq / float(w)
        field = field + amp * _octave(px, py, os_)
    return field


def mask_from_field(field, ratio):
    """Exactly round(ratio*cells) masked cells, largest field first, ties by
    index (proj/src/masking.cpp:71-92).  Returns bool [h, w], True = hidden."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("mask_from_field: ratio must be in [0, 1]")
    flat = field.reshape(-1)
    want = int(np.floor(ratio * flat.size + 0.5))  # llround of a non-negative value
    order = np.lexsort((np.arange(flat.size), -flat))
    masked = np.zeros(flat.size, bool)
    masked[order[:want]] = True
    return masked.reshape(field.shape)


def perlin_mask(grid, ratio, seed):
    return mask_from_field(perlin_field(grid, grid, seed=seed), ratio)


def visible_coords(mask, patch=8):
    """Pixel centres of the visible cells in ascending patch index, float32 [V, 2]."""
    ys, xs = np.nonzero(~mask)
    return np.stack([xs * patch + patch * 0.5, ys * patch + patch * 0.5], 1).astype(np.float32)


def lattice_batch(batch, grid, ratio=0.75, patch=8, seed0=1000):
    """[B, V, 2] visible coordinates of B Perlin masks (seeds seed0 + b).
    Exact mask counts make V identical for every image."""
    out = [visible_coords(perlin_mask(grid, ratio, seed0 + b), patch) for b in range(batch)]
    return np.stack(out)


def bias_params(heads, hidden, rng):
    """BiasNet-shaped parameters (proj/src/attention.cpp:16-31 scales; b1, b2 and
    the blank scalar get small random values so every parameter is exercised)."""
    return dict(
        w1=(rng.standard_normal((heads, 2 * hidden)) / np.sqrt(2.0)).astype(np.float32),
        b1=(0.3 * rng.standard_normal((heads, hidden))).astype(np.float32),
        w2=(rng.standard_normal((heads, hidden)) / np.sqrt(hidden)).astype(np.float32),
        b2=(0.3 * rng.standard_normal((heads, 1))).astype(np.float32),
        blank=(0.3 * rng.standard_normal((heads, 1))).astype(np.float32),
    )


def bf16_round(x):
    """Round-to-nearest-even float32 -> bfloat16 -> float32 (host)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)
