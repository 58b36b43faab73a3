"""Device-side Perlin masks and stage-0 coordinates (perlin_field +
mask_from_field, proj/src/masking.cpp:34-92; the visible lattice, proj/src/geometry.cpp:44-50)
against the reference's golden mask and the numpy restatement pinned to it
(tests/test_inputs.py): bit-exact masks and coordinates."""
import os

import numpy as np
import pytest

from paper_2602_16249_b200 import inputs

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


@pytest.mark.gpu
def test_device_mask_matches_reference_golden():
    from paper_2602_16249_b200 import ops
    m = ops.perlin_masks([3], 64, 0.75)
    np.testing.assert_array_equal(m[0].cpu().numpy(), G["perlin64_r075_s3"])


@pytest.mark.gpu
@pytest.mark.parametrize("grid,ratio,seed0,batch", [(256, 0.75, 1000, 4), (128, 0.5, 7, 3), (37, 0.4, 123, 2), (37, 0.3, 5, 1),
                                                    (64, 0.0, 1, 1), (64, 1.0, 2, 1), (2, 0.5, 9, 2)])
def test_device_masks_bit_exact(grid, ratio, seed0, batch):
    from paper_2602_16249_b200 import ops
    seeds = [seed0 + b for b in range(batch)]
    m = ops.perlin_masks(seeds, grid, ratio).cpu().numpy()
    for b, s in enumerate(seeds):
        want = inputs.perlin_mask(grid, ratio, s).astype(np.uint8)
        np.testing.assert_array_equal(m[b], want)
        assert m[b].sum() == int(np.floor(ratio * grid * grid + 0.5))


@pytest.mark.gpu
def test_device_masks_match_compiled_reference():
    """Directly against the compiled reference's perlin_field + mask_from_field (oracle/_ref)."""
    from oracle import ref
    from paper_2602_16249_b200 import ops
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    seeds = [5, 77, 1234]
    m = ops.perlin_masks(seeds, 96, 0.6).cpu().numpy()
    for b, s in enumerate(seeds):
        np.testing.assert_array_equal(m[b], ref.perlin_mask(96, 0.6, s))


@pytest.mark.gpu
def test_device_visible_coords_match_lattice_batch():
    from paper_2602_16249_b200 import ops
    seeds = [1000 + b for b in range(5)]
    m = ops.perlin_masks(seeds, 256, 0.75)
    coords, count = ops.visible_coords(m, patch=8)
    want = inputs.lattice_batch(5, 256, 0.75, 8, seed0=1000)
    np.testing.assert_array_equal(coords.cpu().numpy(), want)
    assert (count.cpu().numpy() == want.shape[1]).all()


@pytest.mark.gpu
def test_device_mask_rejects_bad_args():
    from paper_2602_16249_b200 import ops
    with pytest.raises(ValueError, match="ratio"):
        ops.perlin_masks([1], 64, 1.5)
    with pytest.raises(ValueError, match="2x2"):
        ops.perlin_masks([1], 1, 0.5)


@pytest.mark.gpu
@pytest.mark.parametrize("size,seeds", [(64, [3, 4, 5]), (224, [11, 12]), (2, [7]), (37, [99])])
def test_device_synth_images_match_reference(size, seeds):
    """synth_image (proj/src/pipeline.cpp:169-227) on the device against the compiled reference:
    the RNG draws and the Perlin base are exact, exp() is within 1 ulp -> |diff| <= 1e-12."""
    from oracle import ref
    from paper_2602_16249_b200 import ops
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    img = ops.synth_images(seeds, size).cpu().numpy()
    for b, s in enumerate(seeds):
        want = ref.synth_image(size, s)
        assert np.abs(img[b] - want).max() <= 1e-12, (s, np.abs(img[b] - want).max())


@pytest.mark.gpu
def test_device_targets_patchify_masked_rows_and_loss():
    """The step's reconstruction targets built on the device: synth_image -> patchify
    (proj/src/pipeline.cpp:131-150) -> masked rows (Model::loss_parts, :588-596) -> masked MSE,
    against a numpy restatement of patchify on the same images."""
    import torch
    from paper_2602_16249_b200 import ops
    seeds, size, patch, ratio = [21, 22], 64, 8, 0.75
    img = ops.synth_images(seeds, size)
    vec = ops.patchify(img, patch)
    g = size // patch
    want = img.cpu().numpy().reshape(2, g, patch, g, patch).transpose(0, 1, 3, 2, 4).reshape(2, g * g, patch * patch)
    np.testing.assert_array_equal(vec.cpu().numpy(), want.astype(np.float32))
    m = ops.perlin_masks(seeds, g, ratio)
    rows = ops.masked_rows(m)
    mm = m.cpu().numpy().reshape(2, -1)
    for b in range(2):
        np.testing.assert_array_equal(rows[b].cpu().numpy(), b * g * g + np.nonzero(mm[b])[0])
    r = rows.reshape(-1)
    pred = torch.zeros((r.numel(), patch * patch), dtype=torch.bfloat16, device="cuda")
    loss, _ = ops.masked_mse(pred, vec.reshape(-1, patch * patch), r)
    tgt = want.reshape(-1, patch * patch)[r.cpu().numpy()]
    assert abs(float(loss.item()) - float((tgt.astype(np.float32) ** 2).mean())) <= 1e-5
