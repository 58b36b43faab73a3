"""CPU: the oracle restatement against the reference's own installed Python API
(baseline/_ref, `pip install --no-deps` of /root/reference/proj; the functions
exposed by proj/bindings/module.cpp:111-136,221-227)."""
import os
import sys

import numpy as np
import pytest

from oracle import port

REF = os.path.join(os.path.dirname(os.path.dirname(__file__)), "baseline", "_ref")
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "affmae")),
                                reason="reference package not installed in baseline/_ref")


@pytest.fixture(scope="module")
def affmae():
    sys.path.insert(0, REF)
    try:
        import affmae as m
    finally:
        sys.path.remove(REF)
    return m


def test_hilbert_and_sfc_order(affmae):
    for x in range(8):
        for y in range(8):
            assert affmae.hilbert_index(8, x, y) == port.hilbert_index(8, x, y)
    rng = np.random.default_rng(1)
    c = rng.uniform(0, 100, (300, 2)).astype(np.float32)
    np.testing.assert_array_equal(np.asarray(affmae.sfc_order(c.astype(np.float64))), port.sfc_order(c))


def test_knn(affmae):
    rng = np.random.default_rng(2)
    q = rng.uniform(0, 20, (15, 2)).astype(np.float32)
    k = np.floor(rng.uniform(0, 20, (40, 2))).astype(np.float32)
    i1, v1 = affmae.knn(q.astype(np.float64), k.astype(np.float64), 7)
    i2, v2 = port.knn(q, k, 7)
    np.testing.assert_array_equal(v1, v2.astype(bool))
    np.testing.assert_array_equal(np.where(v1, i1, 0), i2)


def test_select_retained_and_count(affmae):
    rng = np.random.default_rng(3)
    for n in (1, 7, 100, 4096):
        s = rng.uniform(0, 1, n)
        s[::5] = np.round(s[::5], 1)
        np.testing.assert_array_equal(np.asarray(affmae.select_retained(s.reshape(-1, 1), 0.4)),
                                      port.select_retained(s, 0.4))
        assert affmae.retained_count(n, 0.4) == port.retained_count(n, 0.4)
