"""Seeded test problems shared by the parity tests (host side, numpy).

Inputs follow SURVEY.md §8(c)/(d): the GPU gets bf16 tensors, the oracle gets
the SAME bf16-rounded values as float32 (b32 tensors).
"""
from __future__ import annotations

import numpy as np

from paper_2602_16249_b200 import inputs


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / max(den, 1e-30))


def lattice_coords(batch, grid, ratio=0.75, seed0=1000):
    return inputs.lattice_batch(batch, grid, ratio, 8, seed0)


def random_coords(batch, n, extent, rng):
    return rng.uniform(0.0, extent, (batch, n, 2)).astype(np.float32)


def attn_problem(coords, heads, head_dim, hidden, rng, scale=0.5):
    """q/k/v/blanks ~ scale*N(0,1) rounded to bf16; BiasNet fp32."""
    B, N, _ = coords.shape
    hd = heads * head_dim
    r = lambda *s: inputs.bf16_round(scale * rng.standard_normal(s).astype(np.float32))
    return dict(coords=coords, q=r(B, N, hd), k=r(B, N, hd), v=r(B, N, hd),
                bk=r(heads, head_dim), bv=r(heads, head_dim),
                bias=inputs.bias_params(heads, hidden, rng),
                dout=inputs.bf16_round(rng.standard_normal((B, N, hd)).astype(np.float32)),
                heads=heads, head_dim=head_dim, hidden=hidden)
