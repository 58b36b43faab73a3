"""CPU: synthetic-input generation (paper_2602_16249_b200/inputs.py) against the
reference's Perlin masks (tests/golden) and basic invariants."""
import os

import numpy as np

from paper_2602_16249_b200 import inputs

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def test_perlin_mask_matches_reference_bit_for_bit():
    m = inputs.perlin_mask(64, 0.75, 3)
    np.testing.assert_array_equal(m.astype(np.uint8), G["perlin64_r075_s3"])


def test_exact_mask_count_gives_static_shapes():
    # proj/src/masking.cpp:79: exactly round(r * cells) cells masked -> identical N per image
    c = inputs.lattice_batch(3, 128, 0.75, 8, seed0=5)
    assert c.shape == (3, 128 * 128 - 12288, 2)
    assert (c % 8 == 4).all()


def test_bf16_round():
    x = np.array([1.0, 1.0 + 2 ** -9, 1.0 + 3 * 2 ** -9, -2.5], np.float32)
    np.testing.assert_array_equal(inputs.bf16_round(x), [1.0, 1.0, 1.0 + 2 ** -7, -2.5])
