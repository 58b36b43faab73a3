"""Index builder parity: sfc_order / balanced_clusters / cluster_neighborhood / knn
on the GPU (through the C ABI) against the oracle restatement, BIT-EXACT
(proj/src/geometry.cpp:57-216; proj/tests/test_geometry.cpp)."""
import zlib

import numpy as np
import pytest

from oracle import port
from tests.problems import lattice_coords, random_coords


def _dev(a, dt):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


CASES = [
    ("lattice256", lambda rng: lattice_coords(4, 256), 16, 3),
    ("lattice128", lambda rng: lattice_coords(3, 128, seed0=11), 16, 3),
    ("lattice64_c8", lambda rng: lattice_coords(2, 64, seed0=3), 8, 3),
    ("random", lambda rng: random_coords(3, 1000, 100.0, rng), 16, 3),
    ("random_g5", lambda rng: random_coords(2, 777, 50.0, rng), 8, 5),
    ("duplicates", lambda rng: np.tile(np.array([[[3.0, 7.0]]], np.float32), (2, 5, 1)), 2, 3),
    ("single", lambda rng: np.array([[[1.0, 2.0]]], np.float32), 16, 3),
    ("tiny_fewer_clusters", lambda rng: random_coords(2, 10, 10.0, rng), 8, 3),
    ("coarse_grid_ties", lambda rng: (np.floor(random_coords(2, 500, 20.0, rng)) * 2.0).astype(np.float32), 16, 3),
    ("negative_coords", lambda rng: random_coords(2, 300, 100.0, rng) - 50.0, 16, 3),
    # large segments: the sort splits each image over a CTA cluster; constant
    # keys run no radix pass at all (a CTA must not leave while peers read it)
    ("constant_large", lambda rng: np.full((2, 8192, 2), 5.0, np.float32), 16, 3),
    ("random_large", lambda rng: random_coords(2, 12000, 300.0, rng), 16, 3),
    # 20 images: clusters of 4 CTAs for the Hilbert sort, of 2 for the axis sorts
    ("batch20", lambda rng: random_coords(20, 5000, 200.0, rng), 16, 3),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_cluster_index_bit_exact(case):
    import torch
    from paper_2602_16249_b200 import ops
    name, mk, cluster, groups = case
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    coords = np.ascontiguousarray(mk(rng), dtype=np.float32)
    B, N, _ = coords.shape
    index = ops.cluster_index(_dev(coords, torch.float32), cluster, groups)
    idx, valid = ops.neighbor_expand(index)
    torch.cuda.synchronize()
    perm, cof, nbr = (t.cpu().numpy() for t in (index.perm, index.cluster_of, index.nbr_cl))
    roff, rcl = index.rev_off.cpu().numpy(), index.rev_cl.cpu().numpy()
    idx, valid = idx.cpu().numpy(), valid.cpu().numpy()
    for b in range(B):
        want = port.cluster_index(coords[b], cluster, groups)
        np.testing.assert_array_equal(perm[b], want["members"], err_msg=f"perm image {b}")
        np.testing.assert_array_equal(cof[b], want["cluster_of"], err_msg=f"cluster_of image {b}")
        np.testing.assert_array_equal(nbr[b], want["nbr_cl"], err_msg=f"nbr_cl image {b}")
        np.testing.assert_array_equal(valid[b], want["valid"], err_msg=f"valid image {b}")
        np.testing.assert_array_equal(np.where(want["valid"] > 0, idx[b], 0), want["idx"],
                                      err_msg=f"idx image {b}")
        # reverse CSR: c' lists exactly the clusters whose neighbourhood holds c', ascending
        Cn, G = want["nbr_cl"].shape
        for c2 in range(Cn):
            lst = rcl[b, roff[b, c2]:roff[b, c2 + 1]]
            exp = [c for c in range(Cn) if c2 in want["nbr_cl"][c]]
            np.testing.assert_array_equal(lst, exp)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 37, 5000])
def test_sfc_order_bit_exact(n):
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(n)
    coords = random_coords(2, n, 1000.0, rng)
    perm = ops.sfc_order(_dev(coords, torch.float32)).cpu().numpy()
    for b in range(2):
        np.testing.assert_array_equal(perm[b], port.sfc_order(coords[b]))


@pytest.mark.gpu
def test_knn_far_and_clumped_queries():
    """Grid path safety net: keys clumped in a corner, queries far away (ring budget
    exhausted -> exact scan), plus many identical keys (index tie-break)."""
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(77)
    keys = np.concatenate([rng.uniform(0, 3, (1, 900, 2)), np.full((1, 300, 2), 1.5)], 1).astype(np.float32)
    q = rng.uniform(500, 2000, (1, 1200, 2)).astype(np.float32)
    q[0, :200] = rng.uniform(0, 3, (200, 2))
    idx, valid = ops.knn(_dev(q, torch.float32), _dev(keys, torch.float32), 8)
    wi, wv = port.knn(q[0], keys[0], 8)
    np.testing.assert_array_equal(valid.cpu().numpy()[0], wv)
    np.testing.assert_array_equal(idx.cpu().numpy()[0], wi)


@pytest.mark.gpu
@pytest.mark.parametrize("nq,nk,k", [(10, 40, 12), (50, 7, 10), (64, 300, 32), (5, 5, 3),
                                     # grid-accelerated path (nk >= 512, nq*nk >= 2^20, k <= 16)
                                     (3000, 2000, 8), (1500, 1000, 16), (2100, 600, 5), (2000, 4000, 1),
                                     (1200, 1500, 32), (1100, 1000, 24)])
def test_knn_bit_exact(nq, nk, k):
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(nq * 1000 + nk)
    q = random_coords(2, nq, 20.0, rng)
    keys = random_coords(2, nk, 20.0, rng)
    keys[:, : nk // 3] = np.floor(keys[:, : nk // 3])  # ties
    idx, valid = ops.knn(_dev(q, torch.float32), _dev(keys, torch.float32), k)
    idx, valid = idx.cpu().numpy(), valid.cpu().numpy()
    for b in range(2):
        wi, wv = port.knn(q[b], keys[b], k)
        np.testing.assert_array_equal(valid[b], wv)
        np.testing.assert_array_equal(np.where(wv > 0, idx[b], 0), wi)
