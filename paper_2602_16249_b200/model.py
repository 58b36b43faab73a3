"""Host side of the device-resident training step (no torch): the reference's
``PipelineConfig`` / ``Model`` / ``train`` surface (proj/include/affmae/config.hpp:9-52,
proj/include/affmae/pipeline.hpp:70-149) over the C ABI's ``affmae_model_*`` entry points.

Arrays cross as numpy; device buffers belong to the library.  Every compute call goes
through ``libaffmae_b200.so`` -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace
from typing import List

import numpy as np

from . import capi

MAX_STAGES = 8


class _StageCfg(C.Structure):
    _fields_ = [("dim", C.c_int64), ("heads", C.c_int), ("blocks", C.c_int), ("cluster", C.c_int64),
                ("groups", C.c_int), ("d_s", C.c_double), ("interp_k", C.c_int)]


class ModelCfg(C.Structure):
    """affmae_model_cfg (include/affmae_b200.h)."""
    _fields_ = [("image", C.c_int64), ("patch", C.c_int64), ("n_stages", C.c_int),
                ("stages", _StageCfg * MAX_STAGES), ("dec_dim", C.c_int64), ("dec_depth", C.c_int),
                ("dec_heads", C.c_int), ("gather_k", C.c_int), ("self_k", C.c_int), ("lambda_aux", C.c_double),
                ("mask_strategy", C.c_int), ("mask_ratio", C.c_double), ("optim", capi.AdamwCfg),
                ("seed", C.c_uint64), ("bias_hidden", C.c_int), ("scorer_hidden", C.c_int), ("merge_k", C.c_int),
                ("batch", C.c_int64)]


class ModelInfo(C.Structure):
    _fields_ = [("n_params", C.c_int), ("n_values", C.c_int64), ("tokens", C.c_int64 * MAX_STAGES),
                ("masked", C.c_int64), ("device_bytes", C.c_int64), ("steps_taken", C.c_int64)]


@dataclass
class StageConfig:
    """StageConfig (proj/include/affmae/config.hpp:9-17)."""
    dim: int = 64
    heads: int = 4
    blocks: int = 2
    cluster: int = 16
    groups: int = 3
    d_s: float = 0.4
    interp_k: int = 8


@dataclass
class PipelineConfig:
    """PipelineConfig (proj/include/affmae/config.hpp:35-52) + the trainer's step count and
    the per-device batch of the data-parallel step."""
    image: int = 64
    patch: int = 8
    stages: List[StageConfig] = field(default_factory=list)
    dec_dim: int = 64
    dec_depth: int = 1
    dec_heads: int = 4
    gather_k: int = 8
    self_k: int = 8
    lambda_aux: float = 0.5
    mask_strategy: str = "perlin"
    mask_ratio: float = 0.5
    lr: float = 1e-3
    warmup: int = 100
    weight_decay: float = 0.05
    beta1: float = 0.883
    beta2: float = 0.935
    total_steps: int = 1000
    seed: int = 1
    bias_hidden: int = 8
    scorer_hidden: int = 16
    merge_k: int = 8
    batch: int = 1

    def c_struct(self) -> ModelCfg:
        c = ModelCfg()
        c.image, c.patch, c.n_stages = self.image, self.patch, len(self.stages)
        for i, s in enumerate(self.stages):
            c.stages[i] = _StageCfg(s.dim, s.heads, s.blocks, s.cluster, s.groups, s.d_s, s.interp_k)
        c.dec_dim, c.dec_depth, c.dec_heads = self.dec_dim, self.dec_depth, self.dec_heads
        c.gather_k, c.self_k, c.lambda_aux = self.gather_k, self.self_k, self.lambda_aux
        c.mask_strategy = {"perlin": 0, "random": 1}[self.mask_strategy]
        c.mask_ratio = self.mask_ratio
        c.optim = capi.AdamwCfg(self.lr, self.warmup, self.weight_decay, self.beta1, self.beta2, self.total_steps)
        c.seed, c.bias_hidden, c.scorer_hidden, c.merge_k = self.seed, self.bias_hidden, self.scorer_hidden, self.merge_k
        c.batch = self.batch
        return c

    def grid(self) -> int:
        return self.image // self.patch


def aff_tiny(image=224, batch=2, **kw) -> PipelineConfig:
    """BASELINE configs[0]: AFF-tiny-like encoder, dims 64/128/256/512,
    heads 2/4/8/16, blocks 3/4/18/5, cluster 16, groups 3, d_s 0.4, 75% mask."""
    st = [StageConfig(d, h, b, 16, 3, 0.4, 8) for d, h, b in ((64, 2, 3), (128, 4, 4), (256, 8, 18), (512, 16, 5))]
    return PipelineConfig(image=image, patch=8, stages=st, dec_dim=64, dec_heads=2, mask_ratio=0.75, batch=batch, **kw)


def affmae_b(image=1024, batch=16, **kw) -> PipelineConfig:
    """AFFMAE-B as pinned by this repo (the reference has no AFF-B preset):
    AutoFocusFormer-Base stage shape, dims 128/256/512/1024, heads 4/8/16/32, blocks
    3/4/18/2, cluster 16, groups 3, d_s 0.4, interp_k 8; decoder 256 wide, 8 heads, depth 1;
    patch 8, 75% Perlin mask, deep supervision lambda 0.5 (BASELINE configs[2])."""
    st = [StageConfig(d, h, b, 16, 3, 0.4, 8) for d, h, b in ((128, 4, 3), (256, 8, 4), (512, 16, 18), (1024, 32, 2))]
    return PipelineConfig(image=image, patch=8, stages=st, dec_dim=256, dec_heads=8, mask_ratio=0.75, batch=batch,
                          **kw)


def affmae_l(image=1024, batch=8, **kw) -> PipelineConfig:
    """AFFMAE-L (BASELINE configs[4]): dims 192/384/768/1536 do not fit the compiled LayerNorm
    widths at the last stage; kept for reference (create() raises EUNSUPPORTED)."""
    st = [StageConfig(d, h, b, 16, 3, 0.4, 8) for d, h, b in ((192, 6, 3), (384, 12, 4), (768, 24, 18), (1536, 48, 2))]
    return PipelineConfig(image=image, patch=8, stages=st, dec_dim=256, dec_heads=8, mask_ratio=0.75, batch=batch,
                          **kw)


def mix64(z: int) -> int:
    """proj/include/affmae/rng.hpp:8-13."""
    m = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def step_mask_seed(seed: int, step: int) -> int:
    """train()'s mask seed of step `step` (proj/src/pipeline.cpp:700-701)."""
    return mix64((seed * 0x9E3779B97F4A7C15 + step) & ((1 << 64) - 1))


def _lib():
    L = capi.lib()
    if not getattr(L, "_model_bound", False):
        L.affmae_model_param_name.restype = C.c_char_p
        L.affmae_model_create.argtypes = [C.POINTER(ModelCfg), C.POINTER(C.c_void_p)]
        for f in ("affmae_model_destroy", "affmae_model_get_info", "affmae_model_param_name",
                  "affmae_model_param_dims", "affmae_model_get_params", "affmae_model_set_params",
                  "affmae_model_get_grads", "affmae_model_inputs", "affmae_model_make_masks",
                  "affmae_model_forward_backward", "affmae_model_apply_step", "affmae_model_train_step",
                  "affmae_model_grad_buffer", "affmae_model_save", "affmae_model_load",
                  "affmae_model_stage_output", "affmae_model_force_retained", "affmae_model_forward",
                  "affmae_model_reset_optimizer", "affmae_nccl_unique_id", "affmae_model_set_world"):
            getattr(L, f).argtypes = None
        L._model_bound = True
    return L


class Model:
    """Model + AdamW + train() of the reference (proj/src/pipeline.cpp:255-746) on the device."""

    def __init__(self, cfg: PipelineConfig):
        self.cfg = cfg
        L = _lib()
        h = C.c_void_p()
        self._cs = cfg.c_struct()
        capi.check(L.affmae_model_create(C.byref(self._cs), C.byref(h)), "model_create")
        self._h = h
        info = ModelInfo()
        capi.check(L.affmae_model_get_info(h, C.byref(info)), "model_info")
        self.n_params, self.n_values = info.n_params, info.n_values
        self.tokens = [info.tokens[i] for i in range(len(cfg.stages))]
        self.masked = info.masked
        self.device_bytes = info.device_bytes
        self.names, self.dims = [], []
        for i in range(self.n_params):
            self.names.append(L.affmae_model_param_name(h, C.c_int(i)).decode())
            r, c = C.c_int64(), C.c_int64()
            capi.check(L.affmae_model_param_dims(h, C.c_int(i), C.byref(r), C.byref(c)))
            self.dims.append((r.value, c.value))
        img, msk = C.c_void_p(), C.c_void_p()
        capi.check(L.affmae_model_inputs(h, C.byref(img), C.byref(msk)))
        self.images_ptr, self.masked_ptr = img.value, msk.value
        self._loss = None

    def close(self):
        if getattr(self, "_h", None):
            _lib().affmae_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- params
    def _split(self, flat):
        out, o = {}, 0
        for n, (r, c) in zip(self.names, self.dims):
            out[n] = flat[o:o + r * c].reshape(r, c)
            o += r * c
        return out

    def params(self) -> dict:
        flat = np.empty(self.n_values, np.float32)
        capi.check(_lib().affmae_model_get_params(self._h, flat.ctypes.data_as(C.c_void_p)), "model_get_params")
        return self._split(flat)

    def grads(self) -> dict:
        flat = np.empty(self.n_values, np.float32)
        capi.check(_lib().affmae_model_get_grads(self._h, flat.ctypes.data_as(C.c_void_p)), "model_get_grads")
        return self._split(flat)

    def set_params(self, values: dict):
        flat = np.concatenate([np.asarray(values[n], np.float32).ravel() for n in self.names])
        capi.check(_lib().affmae_model_set_params(self._h, flat.ctypes.data_as(C.c_void_p)), "model_set_params")

    # -------------------------------------------------------------- inputs
    def set_images(self, images: np.ndarray, stream=None):
        """images [B, S, S] float64 (synth_image) -> the model's device input buffer."""
        from . import devmem
        a = np.ascontiguousarray(images, np.float64)
        assert a.shape == (self.cfg.batch, self.cfg.image, self.cfg.image), a.shape
        devmem.h2d(self.images_ptr, a, stream)

    def set_masks(self, masked: np.ndarray, stream=None):
        from . import devmem
        a = np.ascontiguousarray(masked, np.uint8)
        assert a.shape == (self.cfg.batch, self.cfg.grid(), self.cfg.grid()), a.shape
        devmem.h2d(self.masked_ptr, a, stream)

    def make_masks(self, seeds, stream=None):
        """Model::make_mask (proj/src/pipeline.cpp:625-637) of every image of the batch."""
        s = np.ascontiguousarray(np.asarray(seeds, np.uint64))
        assert s.shape == (self.cfg.batch,)
        capi.check(_lib().affmae_model_make_masks(self._h, s.ctypes.data_as(C.c_void_p), C.c_void_p(stream)),
                   "model_make_masks")

    def get_masks(self) -> np.ndarray:
        from . import devmem
        g = self.cfg.grid()
        return devmem.d2h(self.masked_ptr, (self.cfg.batch, g, g), np.uint8)

    # ---------------------------------------------------------------- steps
    def _loss_buf(self):
        from . import devmem
        if self._loss is None:
            self._loss = devmem.DeviceBuffer(16)
        return self._loss

    def forward_backward(self, stream=None):
        """-> (total, main, aux) of the batch-mean loss; gradients left on the device."""
        from . import devmem
        lb = self._loss_buf()
        capi.check(_lib().affmae_model_forward_backward(self._h, C.c_void_p(lb.ptr), C.c_void_p(stream)),
                   "model_forward_backward")
        return tuple(float(x) for x in devmem.d2h(lb.ptr, (3,), np.float32, stream))

    def forward(self, stream=None):
        """encode + decode + deep_sup + loss_parts without the backward -> (total, main, aux)."""
        from . import devmem
        lb = self._loss_buf()
        capi.check(_lib().affmae_model_forward(self._h, C.c_void_p(lb.ptr), C.c_void_p(stream)), "model_forward")
        return tuple(float(x) for x in devmem.d2h(lb.ptr, (3,), np.float32, stream))

    def reset_optimizer(self, total_steps):
        """A fresh AdamW(cfg.optim, total_steps), as the reference's train() builds per call."""
        capi.check(_lib().affmae_model_reset_optimizer(self._h, C.c_int64(total_steps)), "model_reset_optimizer")

    def apply_step(self, stream=None):
        capi.check(_lib().affmae_model_apply_step(self._h, C.c_void_p(stream)), "model_apply_step")

    def train_step(self, use_graph=False, stream=None, read_loss=True):
        from . import devmem
        lb = self._loss_buf()
        capi.check(_lib().affmae_model_train_step(self._h, C.c_void_p(lb.ptr), C.c_int(int(use_graph)),
                                                  C.c_void_p(stream)), "model_train_step")
        if read_loss:
            return tuple(float(x) for x in devmem.d2h(lb.ptr, (3,), np.float32, stream))
        return None

    def stage_output(self, s):
        """-> (coords [B, N_s, 2], features [B, N_s, D_s], merge scores [B, N_s] or None) of the
        last forward."""
        n, d = self.tokens[s], self.cfg.stages[s].dim
        co = np.empty((self.cfg.batch, n, 2), np.float32)
        fe = np.empty((self.cfg.batch, n, d), np.float32)
        sc = np.empty((self.cfg.batch, n), np.float32) if s + 1 < len(self.cfg.stages) else None
        capi.check(_lib().affmae_model_stage_output(
            self._h, C.c_int(s), co.ctypes.data_as(C.c_void_p), fe.ctypes.data_as(C.c_void_p),
            sc.ctypes.data_as(C.c_void_p) if sc is not None else None), "model_stage_output")
        return co, fe, sc

    def force_retained(self, stage, retained=None):
        """Parity-test teacher forcing: merge `stage` keeps `retained` [B, R] (ascending)
        instead of its own selection; None restores the model's selection."""
        if retained is None:
            capi.check(_lib().affmae_model_force_retained(self._h, C.c_int(stage), None), "model_force_retained")
            return
        r = np.ascontiguousarray(retained, np.int32)
        capi.check(_lib().affmae_model_force_retained(self._h, C.c_int(stage), r.ctypes.data_as(C.c_void_p)),
                   "model_force_retained")

    def set_world(self, world, rank, nccl_id=None):
        """Data-parallel rank `rank` of `world`: the loss gradient is seeded with 1/world;
        with nccl_id (bytes of nccl_unique_id() from rank 0) every forward_backward ends with
        an NCCL all-reduce of the gradients, without it the caller sums them."""
        idb = None
        if nccl_id is not None:
            idb = (C.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
        capi.check(_lib().affmae_model_set_world(self._h, C.c_int(world), C.c_int(rank), idb), "model_set_world")

    def grads_device_to_host(self):
        """the flat gradient arena (device layout) as a host fp32 array"""
        from . import devmem
        p, n = self.grad_buffer()
        return devmem.d2h(p, (n,), np.float32)

    def grads_host_to_device(self, flat):
        from . import devmem
        p, n = self.grad_buffer()
        assert flat.size == n
        devmem.h2d(p, np.ascontiguousarray(flat, np.float32))

    def grad_buffer(self):
        p, n = C.c_void_p(), C.c_int64()
        capi.check(_lib().affmae_model_grad_buffer(self._h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def save(self, directory):
        capi.check(_lib().affmae_model_save(self._h, str(directory).encode()), "model_save")

    def load(self, directory):
        capi.check(_lib().affmae_model_load(self._h, str(directory).encode()), "model_load")


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0; broadcast it to the other ranks)."""
    buf = (C.c_uint8 * 128)()
    capi.check(_lib().affmae_nccl_unique_id(buf), "nccl_unique_id")
    return bytes(buf)


def with_batch(cfg: PipelineConfig, batch: int) -> PipelineConfig:
    return replace(cfg, batch=batch)
