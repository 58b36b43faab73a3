"""Device inputs at the step's size (32 images, 256 x 256 cells): Perlin masks, stage-0
coordinates, masked rows; synth_image of 8 images at 256 x 256 pixels and their patchify --
for ncu captures of the §8(f) #4 kernels."""
import torch

from paper_2602_16249_b200 import ops

seeds = [1000 + b for b in range(32)]
for _ in range(3):
    m = ops.perlin_masks(seeds, 256, 0.75)
    ops.visible_coords(m, nvis=16384)
    img = ops.synth_images(seeds[:8], 256)
    ops.patchify(img, 8)
    ops.masked_rows(m)
torch.cuda.synchronize()
print("ok")
