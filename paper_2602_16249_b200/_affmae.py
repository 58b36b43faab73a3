"""`_affmae` -- the reference's Python module surface (proj/bindings/module.cpp:88-336) for the
functions on the hot path, on the B200 library.  numpy in, numpy / lists out, no torch; the
reference's exceptions map the same way (ConfigError -> ValueError, NumericError ->
ArithmeticError, module.cpp:91-92).

    from paper_2602_16249_b200 import _affmae as affmae
    affmae.sfc_order(coords); affmae.knn(q, keys, k); affmae.select_retained(scores, d_s)

Covered (same names, arguments and results): round_b16, hilbert_index, sfc_order, knn,
make_mask / Mask, retained_count, select_retained, synth_image, Model (make_mask, train,
masked_mse, stage_tokens, save, load, n_params).  Not covered -- outside the hot path
(diagnostics, PSD, single-query interpolation probes): perlin_field,
upsample_nearest, radial_psd, psd_slope, interp_softmax, interp_invpow, singular_values,
effective_rank, pca_project, flop_scaling.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import capi, devmem
from . import model as _model


class ConfigError(ValueError):
    """affmae::ConfigError (include/affmae/errors.hpp:8-11)."""


class NumericError(ArithmeticError):
    """affmae::NumericError (include/affmae/errors.hpp:12-15)."""


def _check(rc, what):
    try:
        capi.check(rc, what)
    except ValueError as e:
        raise ConfigError(str(e)) from None
    except ArithmeticError as e:
        raise NumericError(str(e)) from None


def _lib():
    return capi.lib()


def _dev(a: np.ndarray) -> devmem.DeviceBuffer:
    a = np.ascontiguousarray(a)
    d = devmem.DeviceBuffer(a.nbytes)
    devmem.h2d(d.ptr, a)
    return d


def _coords2d(a, what) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 2:
        raise ConfigError(f"{what}: expected a 2-d array")  # tensor_2d, module.cpp:32-38
    return a.astype(np.float32)  # the b32 tensors the reference builds from them


# ------------------------------------------------------------------ numerics
def round_b16(values):
    """round each value to the nearest IEEE binary16 (through fp32, as a b16emu Tensor::set)."""
    a = np.asarray(values, dtype=np.float64)
    return a.astype(np.float32).astype(np.float16).astype(np.float64)


# ------------------------------------------------------------------ geometry
def hilbert_index(n: int, x: int, y: int) -> int:
    return int(_lib().affmae_hilbert_index(n, x, y))


def sfc_order(coords) -> list:
    """space-filling-curve token order for N x 2 coordinates (src/geometry.cpp:69-106)."""
    c = _coords2d(coords, "sfc_order")
    n = c.shape[0]
    if n < 1:
        raise ConfigError("sfc_order: empty point set")
    L = _lib()
    dc = _dev(c)
    perm = devmem.DeviceBuffer(4 * n)
    wsb = L.affmae_sfc_order_workspace(C.c_int64(1), C.c_int64(n))
    ws = devmem.DeviceBuffer(wsb)
    _check(L.affmae_sfc_order(C.c_void_p(dc.ptr), C.c_int64(1), C.c_int64(n), C.c_void_p(perm.ptr),
                              C.c_void_p(ws.ptr), C.c_size_t(wsb), None), "sfc_order")
    return [int(v) for v in devmem.d2h(perm.ptr, (n,), np.int32)]


def knn(queries, keys, k: int):
    """exact brute-force KNN; returns (indices, valid) of shape Q x k (src/geometry.cpp:188-216)."""
    kk = _coords2d(keys, "knn keys")
    q = _coords2d(queries, "knn queries")
    nq, nk = q.shape[0], kk.shape[0]
    if nk < 1:
        raise ConfigError("knn: empty key set")
    if k < 1:
        raise ConfigError("knn: k must be >= 1")
    if nq == 0:
        return np.zeros((0, k), np.int64), np.zeros((0, k), bool)
    dq, dk = _dev(q), _dev(kk)
    idx, val = devmem.DeviceBuffer(4 * nq * k), devmem.DeviceBuffer(nq * k)
    _check(_lib().affmae_knn(C.c_void_p(dq.ptr), C.c_void_p(dk.ptr), C.c_int64(1), C.c_int64(nq), C.c_int64(nk),
                             C.c_int64(k), C.c_void_p(idx.ptr), C.c_void_p(val.ptr), None), "knn")
    return (devmem.d2h(idx.ptr, (nq, k), np.int32).astype(np.int64),
            devmem.d2h(val.ptr, (nq, k), np.uint8).astype(bool))


# ------------------------------------------------------------------- masking
@dataclass
class Mask:
    """MaskSpec (include/affmae/masking.hpp:12-22)."""
    hp: int
    wp: int
    patch: int
    ratio: float
    seed: int
    _masked: np.ndarray

    @property
    def masked(self) -> np.ndarray:
        return self._masked.astype(bool)

    def masked_count(self) -> int:
        return int(self._masked.sum())

    def __repr__(self):
        return f"Mask({self.hp}x{self.wp}, masked {self.masked_count()})"


_M64 = (1 << 64) - 1


def _random_mask(hp, wp, ratio, seed):
    """random_mask (src/masking.cpp:94-110): splitmix64 Fisher-Yates of the cells, first
    llround(ratio * cells) masked."""
    cells = hp * wp
    want = int(np.floor(ratio * cells + 0.5)) if ratio * cells >= 0 else 0
    state = [_model.mix64(seed) ^ 0x6d61736b]

    def nxt():
        state[0] = (state[0] + 0x9E3779B97F4A7C15) & _M64
        z = state[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)
    order = list(range(cells))
    for i in range(cells, 1, -1):
        j = nxt() % i
        order[i - 1], order[j] = order[j], order[i - 1]
    m = np.zeros(cells, np.uint8)
    m[order[:want]] = 1
    return m.reshape(hp, wp)


def make_mask(strategy: str, grid: int, ratio: float, seed: int = 1, patch: int = 8) -> Mask:
    """perlin or random mask with an exact masked-cell count (module.cpp:154-156)."""
    if not (0.0 <= ratio <= 1.0):
        raise ConfigError("mask_from_field: ratio must be in [0, 1]")
    if strategy == "perlin":
        L = _lib()
        wsb = L.affmae_perlin_mask_workspace(C.c_int64(1), C.c_int64(grid), C.c_int64(grid), C.c_int(2),
                                             C.c_double(4.0))
        ws, out = devmem.DeviceBuffer(wsb), devmem.DeviceBuffer(grid * grid)
        seeds = np.array([seed], np.uint64)
        _check(L.affmae_perlin_mask(seeds.ctypes.data_as(C.c_void_p), C.c_int64(1), C.c_int64(grid),
                                    C.c_int64(grid), C.c_int(2), C.c_double(4.0), C.c_double(0.5),
                                    C.c_double(ratio), C.c_void_p(out.ptr), C.c_void_p(ws.ptr), C.c_size_t(wsb),
                                    None), "perlin_mask")
        m = devmem.d2h(out.ptr, (grid, grid), np.uint8)
    elif strategy == "random":
        m = _random_mask(grid, grid, ratio, seed)
    else:
        raise ConfigError(f"mask strategy must be perlin or random, got {strategy}")
    return Mask(grid, grid, patch, ratio, seed, m)


# ------------------------------------------------------------------- merging
def retained_count(n: int, d_s: float) -> int:
    r = _lib().affmae_retained_count(n, d_s)
    if r < 0:
        raise ConfigError("retained_count: d_s must be in (0, 1]")
    return int(r)


def select_retained(scores, d_s: float) -> list:
    """indices of the top round(d_s * N) scores, ascending (src/merging.cpp:56-69)."""
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 2:
        raise ConfigError("select_retained: expected a 2-d array")
    n = s.shape[0]
    r = retained_count(n, d_s)
    L = _lib()
    ds = _dev(s.reshape(-1).astype(np.float32))  # the b32 score tensor of the tape
    out = devmem.DeviceBuffer(4 * r)
    wsb = L.affmae_select_retained_workspace(C.c_int64(1), C.c_int64(n))
    ws = devmem.DeviceBuffer(wsb)
    _check(L.affmae_select_retained(C.c_void_p(ds.ptr), C.c_int64(1), C.c_int64(n), C.c_double(d_s),
                                    C.c_void_p(out.ptr), C.c_void_p(ws.ptr), C.c_size_t(wsb), None),
           "select_retained")
    return [int(v) for v in devmem.d2h(out.ptr, (r,), np.int32)]


# ------------------------------------------------------------------ pipeline
def synth_image(size: int, seed: int = 1) -> np.ndarray:
    """procedural grayscale test image in [0, 1] (src/pipeline.cpp:169-227)."""
    if size < 2:
        raise ConfigError("synth_image: size must be >= 2")
    L = _lib()
    wsb = L.affmae_synth_images_workspace(C.c_int64(1), C.c_int64(size))
    ws, img = devmem.DeviceBuffer(wsb), devmem.DeviceBuffer(size * size * 8)
    seeds = np.array([seed], np.uint64)
    _check(L.affmae_synth_images(seeds.ctypes.data_as(C.c_void_p), C.c_int64(1), C.c_int64(size),
                                 C.c_void_p(img.ptr), C.c_void_p(ws.ptr), C.c_size_t(wsb), None), "synth_image")
    return devmem.d2h(img.ptr, (size, size), np.float64)


class Model:
    """Model (module.cpp:268-335) on the device training step.  The reference builds its model
    from PipelineConfig::toy() (head_dim 12, widths 48) -- sizes the device kernels are not
    compiled for -- so `config` (a paper_2602_16249_b200.model.PipelineConfig) is required;
    the remaining keywords override it like the reference's toy_config (module.cpp:72-84)."""

    def __init__(self, image=64, lambda_aux=0.5, lr=1e-3, warmup=100, mask_ratio=0.5, strategy="perlin", seed=1,
                 precision="b32", config=None):
        if config is None:
            raise ConfigError("Model: the reference's toy() widths (head_dim 12) are not compiled on the device; "
                              "pass config=PipelineConfig(...)")
        if precision != "b32":
            raise ConfigError("Model: the device step keeps b32 master values (bf16 compute)")
        from dataclasses import replace
        self.cfg = replace(config, image=image, lambda_aux=lambda_aux, lr=lr, warmup=warmup, mask_ratio=mask_ratio,
                           mask_strategy=strategy, seed=seed, batch=1)
        try:
            self._m = _model.Model(self.cfg)
        except ValueError as e:
            raise ConfigError(str(e)) from None

    @property
    def n_params(self) -> int:
        return int(self._m.n_values)

    def make_mask(self, seed: int) -> Mask:
        return make_mask(self.cfg.mask_strategy, self.cfg.grid(), self.cfg.mask_ratio, seed, self.cfg.patch)

    def _load(self, image, mask: Mask):
        img = np.asarray(image, dtype=np.float64)
        if img.shape != (self.cfg.image, self.cfg.image):
            raise ConfigError("encode: image does not match the model's image size")
        self._m.set_images(img[None])
        self._m.set_masks(np.asarray(mask._masked, np.uint8)[None])

    def train(self, steps: int, images, rank_every: int = 0) -> dict:
        """train() (src/pipeline.cpp:682-746): a fresh AdamW over `steps` steps, image
        images[step % n], mask Model::make_mask(mix64(seed * phi + step))."""
        if steps < 1:
            raise ConfigError("train: steps must be >= 1")
        if len(images) == 0:
            raise ConfigError("train: need at least one image")
        self._m.reset_optimizer(steps)
        first = last = None
        for step in range(steps):
            img = images[step % len(images)]
            self._load(img, self.make_mask(_model.step_mask_seed(self.cfg.seed, step)))
            loss = self._m.train_step()[0]
            if not np.isfinite(loss):
                raise NumericError(f"train: non-finite loss at step {step}")
            first = loss if first is None else first
            last = loss
        return {"first_loss": first, "last_loss": last, "final_r_hat": []}

    def masked_mse(self, image, mask: Mask) -> float:
        self._load(image, mask)
        return float(self._m.forward()[1])

    def stage_tokens(self, image, mask: Mask) -> list:
        self._load(image, mask)
        self._m.forward()
        return [self._m.stage_output(s)[0][0].astype(np.float64) for s in range(len(self.cfg.stages))]

    def save(self, d: str):
        self._m.save(d)

    def load(self, d: str):
        self._m.load(d)
