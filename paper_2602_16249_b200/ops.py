"""Torch-facing wrappers of the C ABI (device-resident hot path).

Every function here takes CUDA torch tensors, allocates outputs/workspace with
torch, and launches through :mod:`paper_2602_16249_b200.capi` on the current
torch stream.  No computation happens in Python or torch; if the CUDA library
is absent the first call raises (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import capi

BF16 = torch.bfloat16


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _req(t, dtype, name):
    if t is None:
        raise ValueError(f"{name} is required")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


@dataclass
class ClusterIndex:
    """Device-resident cluster index (include/affmae_b200.h: affmae_cluster_index)."""
    geom: capi.ClusterGeom
    perm: torch.Tensor        # [B, N] int32
    cluster_of: torch.Tensor  # [B, N] int32
    nbr_cl: torch.Tensor      # [B, C, G] int32
    rev_off: torch.Tensor     # [B, C+1] int32
    rev_cl: torch.Tensor      # [B, C*G] int32

    def c_struct(self):
        return capi.ClusterIndex(*(capi.ptr(t) for t in (self.perm, self.cluster_of, self.nbr_cl,
                                                          self.rev_off, self.rev_cl)))


def geometry(batch, tokens, cluster, groups):
    return capi.geometry(batch, tokens, cluster, groups)


def empty_index(geom, device="cuda"):
    B, N, Cn, G = geom.batch, geom.tokens, geom.n_clusters, geom.groups_eff
    i32 = dict(dtype=torch.int32, device=device)
    return ClusterIndex(geom, torch.empty((B, N), **i32), torch.empty((B, N), **i32),
                        torch.empty((B, Cn, G), **i32), torch.empty((B, Cn + 1), **i32),
                        torch.empty((B, Cn * G), **i32))


@dataclass
class BiasNet:
    """BiasNet parameters (proj/include/affmae/attention.hpp:16-29) as fp32 device tensors."""
    w1: torch.Tensor     # [h, 2H]
    b1: torch.Tensor     # [h, H]
    w2: torch.Tensor     # [h, H]
    b2: torch.Tensor     # [h] or [h, 1]
    blank: torch.Tensor  # [h] or [h, 1]
    patch: float = 8.0

    @property
    def hidden(self):
        return self.w1.shape[1] // 2

    @staticmethod
    def from_numpy(d, device="cuda", patch=8.0):
        t = {k: torch.as_tensor(d[k], dtype=torch.float32, device=device).contiguous()
             for k in ("w1", "b1", "w2", "b2", "blank")}
        return BiasNet(patch=patch, **t)


def _attn_structs(q, k, v, blank_k, blank_v, coords, bias, heads, head_dim):
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (blank_k, "blank_k"), (blank_v, "blank_v")):
        _req(t, BF16, n)
    _req(coords, torch.float32, "coords")
    for n in ("w1", "b1", "w2", "b2", "blank"):
        _req(getattr(bias, n), torch.float32, f"bias.{n}")
    desc = capi.AttnDesc(heads, head_dim, bias.hidden, float(bias.patch))
    ins = capi.AttnInputs(*(capi.ptr(t) for t in (q, k, v, blank_k, blank_v, coords, bias.w1,
                                                   bias.b1, bias.w2, bias.b2, bias.blank)))
    return desc, ins


def _workspace(nbytes, device):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


@dataclass
class AttnPlan:
    """Geometry plan of the attention op (affmae_attn_plan): built once per cluster index,
    reused by forward and backward (the reference's AttnOp freezes coords + NeighborIndex at
    construction, proj/src/attention.cpp:374-383)."""
    c: capi.AttnPlan
    buf: torch.Tensor


def attn_plan(geom, coords, index: ClusterIndex, heads, head_dim, hidden, patch=8.0,
              with_reverse=True, buf=None, stream=None) -> AttnPlan:
    _req(coords, torch.float32, "coords")
    L = capi.lib()
    desc = capi.AttnDesc(heads, head_dim, hidden, float(patch))
    nbytes = L.affmae_attn_plan_workspace(C.byref(geom), C.c_int(int(with_reverse)))
    if buf is None or buf.numel() < nbytes:
        buf = _workspace(nbytes, coords.device)
    pl = capi.AttnPlan()
    pl.buf = C.c_void_p(buf.data_ptr())
    pl.bytes = C.c_size_t(buf.numel())
    idx = index.c_struct()
    capi.check(L.affmae_attn_plan_build(C.byref(geom), C.byref(desc), C.c_void_p(coords.data_ptr()),
                                        C.byref(idx), C.c_int(int(with_reverse)), C.byref(pl),
                                        _stream(stream)), "attn_plan_build")
    return AttnPlan(pl, buf)


def attn_fwd(geom, q, k, v, blank_k, blank_v, coords, perm, nbr_cl, bias: BiasNet, heads,
             head_dim, out=None, lse=None, workspace=None, stream=None, plan: AttnPlan | None = None):
    """Cluster attention forward (nbhd_attn_streaming, proj/src/attention.cpp:199).
    q/k/v [B, N, h*d] bf16 -> (out [B, N, h*d] bf16, lse [B, N, h] fp32).  With `plan`
    the geometry records come from the plan (perm / nbr_cl are then not read)."""
    desc, ins = _attn_structs(q, k, v, blank_k, blank_v, coords, bias, heads, head_dim)
    B, N = geom.batch, geom.tokens
    if out is None:
        out = torch.empty((B, N, heads * head_dim), dtype=BF16, device=q.device)
    if lse is None:
        lse = torch.empty((B, N, heads), dtype=torch.float32, device=q.device)
    L = capi.lib()
    if plan is not None:
        nbytes = L.affmae_attn_fwd_planned_workspace(C.byref(geom), C.byref(desc))
        if workspace is None or workspace.numel() < nbytes:
            workspace = _workspace(nbytes, q.device)
        capi.check(L.affmae_attn_fwd_planned(C.byref(geom), C.byref(desc), C.byref(ins), C.byref(plan.c),
                                             C.c_void_p(out.data_ptr()), C.c_void_p(lse.data_ptr()),
                                             C.c_void_p(workspace.data_ptr()),
                                             C.c_size_t(workspace.numel()), _stream(stream)),
                   "attn_fwd_planned")
        return out, lse
    _req(perm, torch.int32, "perm")
    _req(nbr_cl, torch.int32, "nbr_cl")
    nbytes = L.affmae_attn_fwd_workspace(C.byref(geom), C.byref(desc))
    if workspace is None or workspace.numel() < nbytes:
        workspace = _workspace(nbytes, q.device)
    capi.check(L.affmae_attn_fwd(C.byref(geom), C.byref(desc), C.byref(ins),
                                 C.c_void_p(perm.data_ptr()), C.c_void_p(nbr_cl.data_ptr()),
                                 C.c_void_p(out.data_ptr()), C.c_void_p(lse.data_ptr()),
                                 C.c_void_p(workspace.data_ptr()), C.c_size_t(workspace.numel()),
                                 _stream(stream)), "attn_fwd")
    return out, lse


@dataclass
class AttnGrads:
    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor
    dblank_k: torch.Tensor
    dblank_v: torch.Tensor
    dw1: torch.Tensor
    db1: torch.Tensor
    dw2: torch.Tensor
    db2: torch.Tensor
    dblank: torch.Tensor

    @staticmethod
    def zeros_like(q, blank_k, bias: BiasNet):
        f32 = dict(dtype=torch.float32, device=q.device)
        h = bias.w1.shape[0]
        return AttnGrads(torch.empty_like(q), torch.empty_like(q), torch.empty_like(q),
                         torch.zeros(blank_k.shape, **f32), torch.zeros(blank_k.shape, **f32),
                         torch.zeros(bias.w1.shape, **f32), torch.zeros(bias.b1.shape, **f32),
                         torch.zeros(bias.w2.shape, **f32), torch.zeros(h, **f32),
                         torch.zeros(h, **f32))


def attn_bwd(geom, q, k, v, blank_k, blank_v, coords, index: ClusterIndex, bias: BiasNet, heads,
             head_dim, out, lse, dout, grads: AttnGrads | None = None, workspace=None,
             stream=None, plan: AttnPlan | None = None):
    """Cluster attention backward (nbhd_attn_backward, proj/src/attention.cpp:241-358).
    dq/dk/dv are overwritten; BiasNet and blank gradients accumulate (+=), like
    CustomOp::backward (proj/include/affmae/tape.hpp:29-31)."""
    desc, ins = _attn_structs(q, k, v, blank_k, blank_v, coords, bias, heads, head_dim)
    for t, n in ((out, "out"), (dout, "dout")):
        _req(t, BF16, n)
    _req(lse, torch.float32, "lse")
    if grads is None:
        grads = AttnGrads.zeros_like(q, blank_k, bias)
    L = capi.lib()
    g = capi.AttnGrads(*(capi.ptr(getattr(grads, n)) for n in (
        "dq", "dk", "dv", "dblank_k", "dblank_v", "dw1", "db1", "dw2", "db2", "dblank")))
    if plan is not None:
        nbytes = L.affmae_attn_bwd_planned_workspace(C.byref(geom), C.byref(desc))
        if workspace is None or workspace.numel() < nbytes:
            workspace = _workspace(nbytes, q.device)
        capi.check(L.affmae_attn_bwd_planned(C.byref(geom), C.byref(desc), C.byref(ins), C.byref(plan.c),
                                             C.c_void_p(out.data_ptr()), C.c_void_p(lse.data_ptr()),
                                             C.c_void_p(dout.data_ptr()), C.byref(g),
                                             C.c_void_p(workspace.data_ptr()),
                                             C.c_size_t(workspace.numel()), _stream(stream)),
                   "attn_bwd_planned")
        return grads
    nbytes = L.affmae_attn_bwd_workspace(C.byref(geom), C.byref(desc))
    if workspace is None or workspace.numel() < nbytes:
        workspace = _workspace(nbytes, q.device)
    idx = index.c_struct()
    capi.check(L.affmae_attn_bwd(C.byref(geom), C.byref(desc), C.byref(ins), C.byref(idx),
                                 C.c_void_p(out.data_ptr()), C.c_void_p(lse.data_ptr()),
                                 C.c_void_p(dout.data_ptr()), C.byref(g),
                                 C.c_void_p(workspace.data_ptr()), C.c_size_t(workspace.numel()),
                                 _stream(stream)), "attn_bwd")
    return grads


def gattn_fwd(q, k, v, blank_k, blank_v, coords, idx, valid, bias: BiasNet, heads, head_dim,
              stream=None):
    """Attention over general neighbour rows (the decoder's cross / self attention,
    proj/src/pipeline.cpp:495-535 over nbhd_attn_streaming): q/k/v [B, N, h*d] bf16,
    coords [B, N, 2], idx/valid [B, N, W] (W <= 31) -> (out [B, N, h*d] bf16, lse [B, N, h])."""
    desc, ins = _attn_structs(q, k, v, blank_k, blank_v, coords, bias, heads, head_dim)
    _req(idx, torch.int32, "idx")
    _req(valid, torch.uint8, "valid")
    B, N, W = idx.shape
    out = torch.empty_like(q)
    lse = torch.empty((B, N, heads), dtype=torch.float32, device=q.device)
    capi.check(capi.lib().affmae_gattn_fwd(C.byref(desc), C.byref(ins), C.c_void_p(idx.data_ptr()),
                                           C.c_void_p(valid.data_ptr()), C.c_int64(B), C.c_int64(N),
                                           C.c_int64(W), C.c_void_p(out.data_ptr()),
                                           C.c_void_p(lse.data_ptr()), _stream(stream)), "gattn_fwd")
    return out, lse


def gattn_bwd(q, k, v, blank_k, blank_v, coords, idx, valid, bias: BiasNet, heads, head_dim, dout,
              grads: AttnGrads | None = None, stream=None, gather=False, workspace=None):
    """Backward of gattn_fwd (nbhd_attn_backward, proj/src/attention.cpp:241-358): dq bf16
    overwritten; dk / dv fp32 and the blank / BiasNet gradients accumulate (+=).  gather:
    dk / dv through a per-call reverse CSR (when heads*head_dim allows), else scattered (the
    default: at the decoder's shape the CSR build costs what the reductions save)."""
    desc, ins = _attn_structs(q, k, v, blank_k, blank_v, coords, bias, heads, head_dim)
    _req(idx, torch.int32, "idx")
    _req(valid, torch.uint8, "valid")
    _req(dout, BF16, "dout")
    B, N, W = idx.shape
    if grads is None:
        grads = AttnGrads.zeros_like(q, blank_k, bias)
        grads.dk = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
        grads.dv = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
    _req(grads.dk, torch.float32, "dk")
    _req(grads.dv, torch.float32, "dv")
    L = capi.lib()
    nbytes = L.affmae_gattn_bwd_workspace(C.byref(desc), C.c_int64(B), C.c_int64(N), C.c_int64(W)) if gather else 0
    if nbytes and (workspace is None or workspace.numel() < nbytes):
        workspace = _workspace(nbytes, q.device)
    ws = (C.c_void_p(workspace.data_ptr()), C.c_size_t(workspace.numel())) if nbytes else (None, C.c_size_t(0))
    capi.check(L.affmae_gattn_bwd(
        C.byref(desc), C.byref(ins), C.c_void_p(idx.data_ptr()), C.c_void_p(valid.data_ptr()), C.c_int64(B),
        C.c_int64(N), C.c_int64(W), C.c_void_p(dout.data_ptr()),
        *[C.c_void_p(getattr(grads, n).data_ptr()) for n in (
            "dq", "dk", "dv", "dblank_k", "dblank_v", "dw1", "db1", "dw2", "db2", "dblank")],
        *ws, _stream(stream)), "gattn_bwd")
    return grads


# --------------------------------------------------------------- index build
def cluster_index(coords, cluster, groups, workspace=None, stream=None) -> ClusterIndex:
    """balanced_clusters + cluster_neighborhood on device, batched
    (proj/src/geometry.cpp:108-186).  coords [B, N, 2] fp32 -> ClusterIndex."""
    _req(coords, torch.float32, "coords")
    B, N, two = coords.shape
    if two != 2:
        raise ValueError("coords must be [B, N, 2]")
    geom = geometry(B, N, cluster, groups)
    idx = empty_index(geom, coords.device)
    L = capi.lib()
    nbytes = L.affmae_cluster_index_workspace(C.byref(geom))
    if workspace is None or workspace.numel() < nbytes:
        workspace = _workspace(nbytes, coords.device)
    cs = idx.c_struct()
    capi.check(L.affmae_cluster_index_build(C.byref(geom), C.c_void_p(coords.data_ptr()),
                                            C.byref(cs), C.c_void_p(workspace.data_ptr()),
                                            C.c_size_t(workspace.numel()), _stream(stream)),
               "cluster_index_build")
    return idx


def neighbor_expand(index: ClusterIndex, stream=None):
    """The reference's per-token NeighborIndex (idx [B, N, M] int32, valid uint8)."""
    g = index.geom
    idx = torch.empty((g.batch, g.tokens, g.width), dtype=torch.int32, device=index.perm.device)
    valid = torch.empty((g.batch, g.tokens, g.width), dtype=torch.uint8, device=index.perm.device)
    capi.check(capi.lib().affmae_neighbor_expand(C.byref(g), C.c_void_p(index.perm.data_ptr()),
                                                 C.c_void_p(index.nbr_cl.data_ptr()),
                                                 C.c_void_p(idx.data_ptr()),
                                                 C.c_void_p(valid.data_ptr()), _stream(stream)),
               "neighbor_expand")
    return idx, valid


def sfc_order(coords, stream=None):
    """sfc_order (proj/src/geometry.cpp:69-106), batched: [B, N, 2] -> perm [B, N] int32."""
    _req(coords, torch.float32, "coords")
    B, N, _ = coords.shape
    L = capi.lib()
    nbytes = L.affmae_sfc_order_workspace(C.c_int64(B), C.c_int64(N))
    ws = _workspace(nbytes, coords.device)
    perm = torch.empty((B, N), dtype=torch.int32, device=coords.device)
    capi.check(L.affmae_sfc_order(C.c_void_p(coords.data_ptr()), C.c_int64(B), C.c_int64(N),
                                  C.c_void_p(perm.data_ptr()), C.c_void_p(ws.data_ptr()),
                                  C.c_size_t(ws.numel()), _stream(stream)), "sfc_order")
    return perm


def knn(queries, keys, k, stream=None):
    """Exact brute-force KNN (proj/src/geometry.cpp:188-216), batched:
    queries [B, Q, 2], keys [B, K, 2] -> (idx [B, Q, k] int32, valid [B, Q, k] uint8)."""
    _req(queries, torch.float32, "queries")
    _req(keys, torch.float32, "keys")
    B, Q, _ = queries.shape
    K = keys.shape[1]
    idx = torch.empty((B, Q, k), dtype=torch.int32, device=queries.device)
    valid = torch.empty((B, Q, k), dtype=torch.uint8, device=queries.device)
    capi.check(capi.lib().affmae_knn(C.c_void_p(queries.data_ptr()), C.c_void_p(keys.data_ptr()),
                                     C.c_int64(B), C.c_int64(Q), C.c_int64(K), C.c_int64(k),
                                     C.c_void_p(idx.data_ptr()), C.c_void_p(valid.data_ptr()),
                                     _stream(stream)), "knn")
    return idx, valid


# ------------------------------------------------------------ device inputs
def perlin_masks(seeds, grid, ratio, octaves=2, base_freq=4.0, persistence=0.5, device="cuda", stream=None):
    """perlin_field + mask_from_field (proj/src/masking.cpp:34-92) for len(seeds) images on the
    device: -> masked [B, grid, grid] uint8 (1 = hidden), bit-exact with the reference."""
    B = len(seeds)
    sd = (C.c_uint64 * max(B, 1))(*[int(s) for s in seeds])
    L = capi.lib()
    nbytes = L.affmae_perlin_mask_workspace(C.c_int64(B), C.c_int64(grid), C.c_int64(grid), C.c_int(octaves),
                                            C.c_double(base_freq))
    ws = _workspace(nbytes, device)
    masked = torch.empty((B, grid, grid), dtype=torch.uint8, device=device)
    capi.check(L.affmae_perlin_mask(sd, C.c_int64(B), C.c_int64(grid), C.c_int64(grid), C.c_int(octaves),
                                    C.c_double(base_freq), C.c_double(persistence), C.c_double(ratio),
                                    C.c_void_p(masked.data_ptr()), C.c_void_p(ws.data_ptr()),
                                    C.c_size_t(ws.numel()), _stream(stream)), "perlin_mask")
    return masked


def synth_images(seeds, size, device="cuda", stream=None):
    """synth_image (proj/src/pipeline.cpp:169-227) for len(seeds) images on the device:
    -> [B, size, size] float64."""
    B = len(seeds)
    sd = (C.c_uint64 * max(B, 1))(*[int(s) for s in seeds])
    L = capi.lib()
    ws = _workspace(L.affmae_synth_images_workspace(C.c_int64(B), C.c_int64(size)), device)
    img = torch.empty((B, size, size), dtype=torch.float64, device=device)
    capi.check(L.affmae_synth_images(sd, C.c_int64(B), C.c_int64(size), C.c_void_p(img.data_ptr()),
                                     C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel()), _stream(stream)),
               "synth_images")
    return img


def patchify(img, patch=8, stream=None):
    """patchify (proj/src/pipeline.cpp:131-150): [B, H, W] float64 -> [B, T, patch^2] float32."""
    _req(img, torch.float64, "img")
    B, H, W = img.shape
    out = torch.empty((B, (H // patch) * (W // patch), patch * patch), dtype=torch.float32, device=img.device)
    capi.check(capi.lib().affmae_patchify(C.c_void_p(img.data_ptr()), C.c_int64(B), C.c_int64(H), C.c_int64(W),
                                          C.c_int64(patch), C.c_void_p(out.data_ptr()), _stream(stream)),
               "patchify")
    return out


def masked_rows(masked, nmask=None, stream=None):
    """Global target rows b*T + cell of the masked cells, ascending per image -> [B, nmask] int32."""
    _req(masked, torch.uint8, "masked")
    B = masked.shape[0]
    cells = masked[0].numel()
    if nmask is None:
        nmask = int(masked[0].sum().item())
    rows = torch.empty((B, nmask), dtype=torch.int32, device=masked.device)
    capi.check(capi.lib().affmae_masked_rows(C.c_void_p(masked.data_ptr()), C.c_int64(B), C.c_int64(cells),
                                             C.c_int64(nmask), C.c_void_p(rows.data_ptr()), _stream(stream)),
               "masked_rows")
    return rows


def visible_coords(masked, patch=8, nvis=None, stream=None):
    """Visible patch centres in ascending cell index (proj/src/geometry.cpp:44-50):
    masked [B, h, w] uint8 -> (coords [B, nvis, 2] fp32, count [B] int32)."""
    _req(masked, torch.uint8, "masked")
    B, h, w = masked.shape
    if nvis is None:
        nvis = h * w - int(masked[0].sum().item())
    coords = torch.empty((B, nvis, 2), dtype=torch.float32, device=masked.device)
    count = torch.empty(B, dtype=torch.int32, device=masked.device)
    capi.check(capi.lib().affmae_visible_coords(C.c_void_p(masked.data_ptr()), C.c_int64(B), C.c_int64(h),
                                                C.c_int64(w), C.c_double(patch), C.c_int64(nvis),
                                                C.c_void_p(coords.data_ptr()), C.c_void_p(count.data_ptr()),
                                                _stream(stream)), "visible_coords")
    return coords, count


# ------------------------------------------------------------ AFT1 files / checkpoints
def aft_write(path, t, dtype=0, stream=None):
    """write_aft (proj/src/tensor_io.cpp:60-66) from a device tensor: fp32 (dtype 0 b32 /
    1 b16emu) or uint8 (dtype 2, write_aft_u8)."""
    _req(t, torch.uint8 if dtype == 2 else torch.float32, "t")
    dims = (C.c_int64 * max(t.dim(), 1))(*t.shape)
    capi.check(capi.lib().affmae_aft_write(str(path).encode(), C.c_void_p(t.data_ptr()), dims, C.c_int(t.dim()),
                                           C.c_int(dtype), _stream(stream)), "aft_write")


def aft_read(path, device="cuda", stream=None):
    """read_aft (proj/src/tensor_io.cpp:78-105) into a device fp32 tensor -> (tensor, dtype code)."""
    L = capi.lib()
    dt, nd = C.c_int(), C.c_int()
    dims = (C.c_int64 * 8)()
    capi.check(L.affmae_aft_read_header(str(path).encode(), C.byref(dt), C.byref(nd), dims), "aft_read")
    shape = tuple(dims[i] for i in range(nd.value))
    out = torch.empty(shape, dtype=torch.float32, device=device)
    capi.check(L.affmae_aft_read(str(path).encode(), C.c_void_p(out.data_ptr()), C.c_int64(out.numel()), None,
                                 _stream(stream)), "aft_read")
    return out, dt.value


_PREC = {"b32": 0, "b16emu": 1, "b64": 2}


def save_checkpoint(directory, params, stream=None):
    """save_checkpoint (proj/src/pipeline.cpp:757-770): params = {name: (fp32 device tensor,
    precision name)} in ParamStore order."""
    names = list(params)
    n = len(names)
    ts = [params[k][0] for k in names]
    for t, k in zip(ts, names):
        _req(t, torch.float32, k)
    dim_arrs = [(C.c_int64 * max(t.dim(), 1))(*t.shape) for t in ts]
    capi.check(capi.lib().affmae_checkpoint_save(
        str(directory).encode(), C.c_int(n), (C.c_char_p * max(n, 1))(*[k.encode() for k in names]),
        (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in ts]),
        (C.POINTER(C.c_int64) * max(n, 1))(*[C.cast(d, C.POINTER(C.c_int64)) for d in dim_arrs]),
        (C.c_int * max(n, 1))(*[t.dim() for t in ts]), (C.c_int * max(n, 1))(*[_PREC[params[k][1]] for k in names]),
        _stream(stream)), "checkpoint_save")


def load_checkpoint(directory, params, stream=None):
    """load_checkpoint (proj/src/pipeline.cpp:772-797) into {name: fp32 device tensor}."""
    names = list(params)
    n = len(names)
    ts = [params[k] for k in names]
    for t, k in zip(ts, names):
        _req(t, torch.float32, k)
    capi.check(capi.lib().affmae_checkpoint_load(
        str(directory).encode(), C.c_int(n), (C.c_char_p * max(n, 1))(*[k.encode() for k in names]),
        (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in ts]), (C.c_int64 * max(n, 1))(*[t.numel() for t in ts]),
        _stream(stream)), "checkpoint_load")


# ------------------------------------------------------------ interpolation
def interp_fwd(queries, key_coords, feats, idx, valid, p, eps=1e-6, stream=None):
    """make_interp_op forward (proj/src/interpolation.cpp:192-222), batched:
    queries [B, Q, 2] fp32, key_coords [B, N, 2] fp32, feats [B, N, D] bf16, idx/valid
    [B, Q, K] (e.g. from knn), p [1] fp32 -> out [B, Q, D] bf16."""
    _req(queries, torch.float32, "queries")
    _req(key_coords, torch.float32, "key_coords")
    _req(feats, torch.bfloat16, "feats")
    _req(idx, torch.int32, "idx")
    _req(valid, torch.uint8, "valid")
    _req(p, torch.float32, "p")
    B, Q, _ = queries.shape
    N, D = feats.shape[1], feats.shape[2]
    K = idx.shape[2]
    out = torch.empty((B, Q, D), dtype=torch.bfloat16, device=feats.device)
    capi.check(capi.lib().affmae_interp_fwd(
        C.c_void_p(queries.data_ptr()), C.c_void_p(key_coords.data_ptr()), C.c_void_p(feats.data_ptr()),
        C.c_void_p(idx.data_ptr()), C.c_void_p(valid.data_ptr()), C.c_int64(B), C.c_int64(Q), C.c_int64(N),
        C.c_int64(D), C.c_int64(K), C.c_void_p(p.data_ptr()), C.c_double(eps), C.c_void_p(out.data_ptr()),
        _stream(stream)), "interp_fwd")
    return out


def interp_bwd(queries, key_coords, feats, idx, valid, p, dout, eps=1e-6, dfeats=None, dp=None, dqueries=None,
               stream=None, gather=True, workspace=None):
    """make_interp_op backward (proj/src/interpolation.cpp:224-251): accumulates into
    dfeats [B, N, D] fp32, dp [1] fp32 and dqueries [B, Q, 2] fp32 (zeros if not given).
    gather=True (default): dfeats through a per-call reverse CSR (affmae_interp_bwd_gather);
    gather=False: scattered fp32 reductions (affmae_interp_bwd, no workspace)."""
    _req(dout, torch.bfloat16, "dout")
    B, Q, _ = queries.shape
    N, D = feats.shape[1], feats.shape[2]
    K = idx.shape[2]
    dev = feats.device
    if dfeats is None:
        dfeats = torch.zeros((B, N, D), dtype=torch.float32, device=dev)
    if dp is None:
        dp = torch.zeros(1, dtype=torch.float32, device=dev)
    if dqueries is None:
        dqueries = torch.zeros((B, Q, 2), dtype=torch.float32, device=dev)
    args = (C.c_void_p(queries.data_ptr()), C.c_void_p(key_coords.data_ptr()), C.c_void_p(feats.data_ptr()),
            C.c_void_p(idx.data_ptr()), C.c_void_p(valid.data_ptr()), C.c_int64(B), C.c_int64(Q), C.c_int64(N),
            C.c_int64(D), C.c_int64(K), C.c_void_p(p.data_ptr()), C.c_double(eps), C.c_void_p(dout.data_ptr()),
            C.c_void_p(dfeats.data_ptr()), C.c_void_p(dp.data_ptr()), C.c_void_p(dqueries.data_ptr()))
    L = capi.lib()
    if gather:
        nbytes = L.affmae_interp_bwd_gather_workspace(C.c_int64(B), C.c_int64(Q), C.c_int64(N), C.c_int64(K))
        if workspace is None or workspace.numel() < nbytes:
            workspace = _workspace(nbytes, dev)
        capi.check(L.affmae_interp_bwd_gather(*args, C.c_void_p(workspace.data_ptr()), C.c_size_t(workspace.numel()),
                                              _stream(stream)), "interp_bwd_gather")
    else:
        capi.check(L.affmae_interp_bwd(*args, _stream(stream)), "interp_bwd")
    return dfeats, dp, dqueries


# ----------------------------------------------------------- dense linear
def linear(x, w, bias=None, act="none", stream=None):
    """y = act(x W^T + b) on the tcgen05 tensor cores (Tape matmul + bias + gelu_erf):
    x [M, K] bf16, w [N, K] bf16, bias [N] fp32 (zeros if None), act 'none' | 'gelu'."""
    _req(x, torch.bfloat16, "x")
    _req(w, torch.bfloat16, "w")
    M, K = x.shape
    N = w.shape[0]
    if bias is None:
        bias = torch.zeros(N, dtype=torch.float32, device=x.device)
    _req(bias, torch.float32, "bias")
    y = torch.empty((M, N), dtype=torch.bfloat16, device=x.device)
    wsb = int(capi.lib().affmae_linear_workspace(C.c_int64(M), C.c_int64(N), C.c_int64(K)))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    capi.check(capi.lib().affmae_linear_fwd(
        C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(bias.data_ptr()), C.c_int64(M), C.c_int64(N),
        C.c_int64(K), C.c_int({"none": 0, "gelu": 1}[act]), C.c_void_p(y.data_ptr()), C.c_void_p(ws.data_ptr()),
        C.c_size_t(ws.numel()), _stream(stream)), "linear")
    return y


def linear_gelu_save(x, w, bias=None, stream=None):
    """y = GELU(x W^T + b) and the pre-activation (for gelu_bwd), one tcgen05 launch."""
    _req(x, torch.bfloat16, "x")
    _req(w, torch.bfloat16, "w")
    M, K = x.shape
    N = w.shape[0]
    if bias is None:
        bias = torch.zeros(N, dtype=torch.float32, device=x.device)
    y = torch.empty((M, N), dtype=torch.bfloat16, device=x.device)
    pre = torch.empty((M, N), dtype=torch.bfloat16, device=x.device)
    wsb = int(capi.lib().affmae_linear_workspace(C.c_int64(M), C.c_int64(N), C.c_int64(K)))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    capi.check(capi.lib().affmae_linear_fwd_gelu_aux(
        C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(bias.data_ptr()), C.c_int64(M), C.c_int64(N),
        C.c_int64(K), C.c_void_p(y.data_ptr()), C.c_void_p(pre.data_ptr()), C.c_void_p(ws.data_ptr()),
        C.c_size_t(ws.numel()), _stream(stream)), "linear_gelu_save")
    return y, pre


def gelu_bwd(pre, dy, stream=None):
    """dpre = dy * gelu'(pre) (the Tape's gelu VJP, erf form)."""
    _req(pre, torch.bfloat16, "pre")
    _req(dy, torch.bfloat16, "dy")
    dpre = torch.empty_like(pre)
    capi.check(capi.lib().affmae_gelu_bwd(C.c_void_p(pre.data_ptr()), C.c_void_p(dy.data_ptr()),
                                          C.c_int64(pre.numel()), C.c_void_p(dpre.data_ptr()), _stream(stream)),
               "gelu_bwd")
    return dpre


def linear_add(x, w, bias, c, stream=None):
    """y = x W^T + b + c (the residual c bf16 [M, N] added in fp32 before the one rounding)."""
    for t, n in ((x, "x"), (w, "w"), (c, "c")):
        _req(t, torch.bfloat16, n)
    _req(bias, torch.float32, "bias")
    M, K = x.shape
    N = w.shape[0]
    y = torch.empty((M, N), dtype=torch.bfloat16, device=x.device)
    capi.check(capi.lib().affmae_linear_fwd_add(
        C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(bias.data_ptr()), C.c_int64(M), C.c_int64(N),
        C.c_int64(K), C.c_void_p(c.data_ptr()), C.c_void_p(y.data_ptr()), _stream(stream)), "linear_add")
    return y


def linear_dx_gelu(dy, w, pre, stream=None):
    """dh = (dy W) * gelu'(pre): the input gradient of y = GELU(pre) W^T + b, one tcgen05 pass."""
    for t, n in ((dy, "dy"), (w, "w"), (pre, "pre")):
        _req(t, torch.bfloat16, n)
    M, N = dy.shape
    K = w.shape[1]
    dh = torch.empty((M, K), dtype=torch.bfloat16, device=dy.device)
    capi.check(capi.lib().affmae_linear_dx_gelu(
        C.c_void_p(dy.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(pre.data_ptr()), C.c_int64(M), C.c_int64(N),
        C.c_int64(K), C.c_void_p(dh.data_ptr()), _stream(stream)), "linear_dx_gelu")
    return dh


def linear_dx_f32(dy, w, dx=None, beta=0.0, stream=None):
    """dx = dy W + beta dx in fp32 (dx [M, K] fp32; a new zero buffer if None)."""
    _req(dy, torch.bfloat16, "dy")
    _req(w, torch.bfloat16, "w")
    M, N = dy.shape
    K = w.shape[1]
    if dx is None:
        dx = torch.zeros((M, K), dtype=torch.float32, device=dy.device)
    capi.check(capi.lib().affmae_linear_dx_f32(
        C.c_void_p(dy.data_ptr()), C.c_void_p(w.data_ptr()), C.c_int64(M), C.c_int64(N), C.c_int64(K),
        C.c_void_p(dx.data_ptr()), C.c_float(beta), _stream(stream)), "linear_dx_f32")
    return dx


def linear_bwd(x, w, dy, dw=None, db=None, need_dx=True, stream=None):
    """Backward of y = x W^T + b (dy already through the activation) on tcgen05: returns
    (dx bf16 [M, K], dw fp32 [N, K] +=, db fp32 [N] +=); dw/db are zeros if not given."""
    _req(x, torch.bfloat16, "x")
    _req(w, torch.bfloat16, "w")
    _req(dy, torch.bfloat16, "dy")
    M, K = x.shape
    N = w.shape[0]
    dev = x.device
    dx = torch.empty((M, K), dtype=torch.bfloat16, device=dev) if need_dx else None
    if dw is None:
        dw = torch.zeros((N, K), dtype=torch.float32, device=dev)
    if db is None:
        db = torch.zeros(N, dtype=torch.float32, device=dev)
    wsb = int(capi.lib().affmae_linear_bwd_workspace(C.c_int64(M), C.c_int64(N), C.c_int64(K)))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    capi.check(capi.lib().affmae_linear_bwd(
        C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(dy.data_ptr()), C.c_int64(M), C.c_int64(N),
        C.c_int64(K), C.c_void_p(dx.data_ptr() if dx is not None else 0), C.c_void_p(dw.data_ptr()),
        C.c_void_p(db.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel()), _stream(stream)),
        "linear_bwd")
    return dx, dw, db


def layer_norm(x, gamma, beta, stream=None):
    """Tape::layer_norm (proj/src/tape.cpp:84-100, eps 1e-5): x [R, C] bf16 -> (y bf16, stats)."""
    _req(x, torch.bfloat16, "x")
    R, Cc = x.shape
    y = torch.empty_like(x)
    stats = torch.empty((R, 2), dtype=torch.float32, device=x.device)
    capi.check(capi.lib().affmae_layernorm_fwd(
        C.c_void_p(x.data_ptr()), C.c_void_p(gamma.data_ptr()), C.c_void_p(beta.data_ptr()), C.c_int64(R),
        C.c_int64(Cc), C.c_void_p(y.data_ptr()), C.c_void_p(stats.data_ptr()), _stream(stream)), "layer_norm")
    return y, stats


def layer_norm_bwd(x, gamma, stats, dy, dgamma=None, dbeta=None, stream=None):
    """VJP of layer_norm (proj/src/tape.cpp:581-617): returns (dx bf16, dgamma +=, dbeta +=)."""
    _req(dy, torch.bfloat16, "dy")
    R, Cc = x.shape
    dx = torch.empty_like(x)
    if dgamma is None:
        dgamma = torch.zeros(Cc, dtype=torch.float32, device=x.device)
    if dbeta is None:
        dbeta = torch.zeros(Cc, dtype=torch.float32, device=x.device)
    wsb = int(capi.lib().affmae_layernorm_bwd_workspace(C.c_int64(R), C.c_int64(Cc)))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    capi.check(capi.lib().affmae_layernorm_bwd(
        C.c_void_p(x.data_ptr()), C.c_void_p(gamma.data_ptr()), C.c_void_p(stats.data_ptr()),
        C.c_void_p(dy.data_ptr()), C.c_int64(R), C.c_int64(Cc), C.c_void_p(dx.data_ptr()),
        C.c_void_p(dgamma.data_ptr()), C.c_void_p(dbeta.data_ptr()), C.c_void_p(ws.data_ptr()),
        C.c_size_t(ws.numel()), _stream(stream)), "layer_norm_bwd")
    return dx, dgamma, dbeta


def norm_clamp(x, limit, stream=None):
    """NormClampOp forward (proj/src/pipeline.cpp:75-97): rows of x [R, d] bf16 to norm <= limit."""
    _req(x, torch.bfloat16, "x")
    y = torch.empty_like(x)
    capi.check(capi.lib().affmae_norm_clamp_fwd(C.c_void_p(x.data_ptr()), C.c_int64(x.shape[0]),
                                                C.c_int64(x.shape[1]), C.c_double(limit), C.c_void_p(y.data_ptr()),
                                                _stream(stream)), "norm_clamp")
    return y


def norm_clamp_bwd(x, g, limit, dx=None, stream=None):
    """NormClampOp VJP (proj/src/pipeline.cpp:99-125): dx (bf16) += J^T g; a new zero dx
    unless one is given to accumulate into."""
    _req(g, torch.bfloat16, "g")
    dx = torch.zeros_like(x) if dx is None else dx
    capi.check(capi.lib().affmae_norm_clamp_bwd(C.c_void_p(x.data_ptr()), C.c_void_p(g.data_ptr()),
                                                C.c_int64(x.shape[0]), C.c_int64(x.shape[1]), C.c_double(limit),
                                                C.c_void_p(dx.data_ptr()), _stream(stream)), "norm_clamp_bwd")
    return dx


def masked_mse(pred, patches, cells, dloss=1.0, need_grad=True, stream=None):
    """Reconstruction loss (Tape::mse, proj/src/tape.cpp:431-446) of pred [R, p] bf16 against
    patches[cells] (patches [n_cells, p] fp32, cells [R] int32): (loss [1] fp32, dpred bf16 or None)."""
    _req(pred, torch.bfloat16, "pred")
    _req(patches, torch.float32, "patches")
    _req(cells, torch.int32, "cells")
    R, P = pred.shape
    loss = torch.empty(1, dtype=torch.float32, device=pred.device)
    dpred = torch.empty_like(pred) if need_grad else None
    wsb = int(capi.lib().affmae_masked_mse_workspace(C.c_int64(R)))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=pred.device)
    capi.check(capi.lib().affmae_masked_mse(
        C.c_void_p(pred.data_ptr()), C.c_void_p(patches.data_ptr()), C.c_void_p(cells.data_ptr()), C.c_int64(R),
        C.c_int64(P), C.c_void_p(loss.data_ptr()), C.c_void_p(dpred.data_ptr() if dpred is not None else 0),
        C.c_float(dloss), C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel()), _stream(stream)), "masked_mse")
    return loss, dpred


# ---------------------------------------------------------------- optimizer
class AdamW:
    """AdamW (proj/include/affmae/pipeline.hpp:112-127; src/pipeline.cpp:639-680) over a list of
    fp32 CUDA parameter tensors: they are packed back to back in one flat buffer (the tensors
    become views into it), with flat grad / moment buffers, and every step is one fused launch."""

    def __init__(self, shapes, lr=1e-3, warmup=100, weight_decay=0.05, beta1=0.883, beta2=0.935,
                 total_steps=1000, device="cuda"):
        self.cfg = capi.AdamwCfg(lr, warmup, weight_decay, beta1, beta2, total_steps)
        sizes = [int(np.prod(s)) for s in shapes]
        offs = np.concatenate([[0], np.cumsum([(z + 3) // 4 * 4 for z in sizes])]).astype(np.int64)
        n = int(offs[-1])
        f32 = dict(dtype=torch.float32, device=device)
        self.value, self.grad = torch.zeros(n, **f32), torch.zeros(n, **f32)
        self.m, self.v = torch.zeros(n, **f32), torch.zeros(n, **f32)
        self.params = [self.value[o:o + z].view(*s) for o, z, s in zip(offs[:-1], sizes, shapes)]
        self.grads = [self.grad[o:o + z].view(*s) for o, z, s in zip(offs[:-1], sizes, shapes)]
        self.seg_off = torch.as_tensor(offs[:-1], device=device)
        self.seg_decay = torch.as_tensor(np.array([1 if s[0] > 1 else 0 for s in shapes], np.uint8),
                                         device=device)
        self.t = 0

    def lr_at(self, step):
        return capi.lib().affmae_adamw_lr(C.byref(self.cfg), C.c_int64(step))

    def step(self, stream=None):
        capi.check(capi.lib().affmae_adamw_step(
            C.byref(self.cfg), C.c_int64(self.t), C.c_int64(len(self.params)), C.c_void_p(self.seg_off.data_ptr()),
            C.c_void_p(self.seg_decay.data_ptr()), C.c_int64(self.value.numel()), C.c_void_p(self.value.data_ptr()),
            C.c_void_p(self.grad.data_ptr()), C.c_void_p(self.m.data_ptr()), C.c_void_p(self.v.data_ptr()),
            _stream(stream)), "adamw_step")
        self.t += 1

    def _state_views(self, names):
        offs, out = 0, []
        for nm, p in zip(names, self.params):
            out.append((nm, p, self.m[offs:offs + p.numel()].view(p.shape), self.v[offs:offs + p.numel()].view(p.shape)))
            offs += (p.numel() + 3) // 4 * 4
        return out

    def save(self, directory, names, precs=None, stream=None):
        """save_checkpoint (proj/src/pipeline.cpp:757-770) of the parameters under `names`
        (precision names per parameter, default "b32"): <dir>/manifest.tsv holds ONLY the
        parameters, so the reference's load_checkpoint reads the directory unchanged.  The
        state the reference omits goes to its own checkpoint in <dir>/optim/: the moments as
        "<name>.m" / "<name>.v" and the step count as "step" (AFT1 b32)."""
        precs = precs or ["b32"] * len(names)
        entries, state = {}, {}
        for (nm, p, m, v), pr in zip(self._state_views(names), precs):
            entries[nm] = (p, pr)
            state[nm + ".m"] = (m, "b32")
            state[nm + ".v"] = (v, "b32")
        state["step"] = (torch.tensor([float(self.t)], device=self.value.device), "b32")
        save_checkpoint(directory, entries, stream=stream)
        save_checkpoint(os.path.join(str(directory), "optim"), state, stream=stream)

    def load(self, directory, names, stream=None):
        """load_checkpoint into the parameters; the moments and step count come from
        <dir>/optim/ when present (written by save()), else the optimizer restarts from zero
        moments at step 0 -- a plain reference checkpoint loads too."""
        entries, state = {}, {}
        for nm, p, m, v in self._state_views(names):
            entries[nm] = p
            state[nm + ".m"] = m
            state[nm + ".v"] = v
        load_checkpoint(directory, entries, stream=stream)
        optim_dir = os.path.join(str(directory), "optim")
        if os.path.exists(os.path.join(optim_dir, "manifest.tsv")):
            step = torch.zeros(1, device=self.value.device)
            state["step"] = step
            load_checkpoint(optim_dir, state, stream=stream)
            self.t = int(step.item())
        else:
            self.m.zero_()
            self.v.zero_()
            self.t = 0


# -------------------------------------------------------------------- merge
def retained_count(n, d_s):
    """retained_count (proj/src/merging.cpp:50-54): clamp(floor(d_s*n + 0.5), 1, n)."""
    r = capi.lib().affmae_retained_count(n, d_s)
    if r < 0:
        raise ValueError("retained_count: d_s must be in (0, 1]")
    return int(r)


def select_retained(scores, d_s, stream=None):
    """select_retained (proj/src/merging.cpp:56-69), batched: scores [B, N] fp32 ->
    retained [B, R] int32 ascending (top round(d_s N) scores, ties to lower index)."""
    _req(scores, torch.float32, "scores")
    B, N = scores.shape
    R = retained_count(N, d_s)
    L = capi.lib()
    ws = _workspace(L.affmae_select_retained_workspace(C.c_int64(B), C.c_int64(N)), scores.device)
    out = torch.empty((B, R), dtype=torch.int32, device=scores.device)
    capi.check(L.affmae_select_retained(C.c_void_p(scores.data_ptr()), C.c_int64(B), C.c_int64(N),
                                        C.c_double(d_s), C.c_void_p(out.data_ptr()),
                                        C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel()),
                                        _stream(stream)), "select_retained")
    return out


@dataclass
class MergePlan:
    """Device merge plan (include/affmae_b200.h: affmae_merge_plan)."""
    retained: torch.Tensor   # [B, R] int32
    target: torch.Tensor     # [B, N] int32
    pool_idx: torch.Tensor   # [B, R, k_m] int32
    pool_dist: torch.Tensor  # [B, R, k_m] float64
    pool_cnt: torch.Tensor   # [B, R] int32
    row_of: torch.Tensor     # [B, N] int32
    k_m: int

    def c_struct(self):
        return capi.MergePlan(*(capi.ptr(t) for t in (self.target, self.pool_idx, self.pool_dist,
                                                       self.pool_cnt, self.row_of)))


def merge_plan(coords, retained, k_m, workspace=None, stream=None) -> MergePlan:
    """merge_plan (proj/src/merging.cpp:71-116), batched, bit-exact."""
    _req(coords, torch.float32, "coords")
    _req(retained, torch.int32, "retained")
    B, N, _ = coords.shape
    R = retained.shape[1]
    dev = coords.device
    i32 = dict(dtype=torch.int32, device=dev)
    plan = MergePlan(retained, torch.empty((B, N), **i32), torch.empty((B, R, k_m), **i32),
                     torch.empty((B, R, k_m), dtype=torch.float64, device=dev),
                     torch.empty((B, R), **i32), torch.empty((B, N), **i32), k_m)
    L = capi.lib()
    nbytes = L.affmae_merge_plan_workspace(C.c_int64(B), C.c_int64(N), C.c_int64(R))
    if workspace is None or workspace.numel() < nbytes:
        workspace = _workspace(nbytes, dev)
    ps = plan.c_struct()
    capi.check(L.affmae_merge_plan_build(C.c_void_p(coords.data_ptr()),
                                         C.c_void_p(retained.data_ptr()), C.c_int64(B),
                                         C.c_int64(N), C.c_int64(R), C.c_int(k_m), C.byref(ps),
                                         C.c_void_p(workspace.data_ptr()),
                                         C.c_size_t(workspace.numel()), _stream(stream)),
               "merge_plan")
    return plan


def merge_pool_fwd(feats, scores, p_merge, plan: MergePlan, out=None, stream=None):
    """MergePoolOp::forward (proj/src/merging.cpp:121-166): [B, R, 2D] bf16."""
    _req(feats, BF16, "feats")
    _req(scores, torch.float32, "scores")
    _req(p_merge, torch.float32, "p_merge")
    B, N, D = feats.shape
    R = plan.retained.shape[1]
    if out is None:
        out = torch.empty((B, R, 2 * D), dtype=BF16, device=feats.device)
    ps = plan.c_struct()
    capi.check(capi.lib().affmae_merge_pool_fwd(
        C.c_void_p(feats.data_ptr()), C.c_void_p(scores.data_ptr()), C.c_void_p(p_merge.data_ptr()),
        C.c_void_p(plan.retained.data_ptr()), C.byref(ps), C.c_int64(B), C.c_int64(N), C.c_int64(R),
        C.c_int64(D), C.c_int(plan.k_m), C.c_void_p(out.data_ptr()), _stream(stream)),
        "merge_pool_fwd")
    return out


def importance_scores(feats, w1, b1, w2, b2, stream=None):
    """importance_scores (proj/src/merging.cpp:31-48): feats [..., D] fp32, w1 [D, H], b1 [H],
    w2 [H], b2 [1] fp32 (MergeParams layout) -> scores [...] fp32 (binary64 inside)."""
    _req(feats, torch.float32, "feats")
    for t, n in ((w1, "w1"), (b1, "b1"), (w2, "w2"), (b2, "b2")):
        _req(t, torch.float32, n)
    D, H = w1.shape
    if feats.shape[-1] != D:
        raise ValueError("importance_scores: feature width does not match the scorer")
    rows = feats.numel() // D
    out = torch.empty(feats.shape[:-1], dtype=torch.float32, device=feats.device)
    capi.check(capi.lib().affmae_importance_scores(
        C.c_void_p(feats.data_ptr()), C.c_int64(rows), C.c_int64(D), C.c_void_p(w1.data_ptr()),
        C.c_void_p(b1.data_ptr()), C.c_void_p(w2.data_ptr()), C.c_void_p(b2.data_ptr()), C.c_int(H),
        C.c_void_p(out.data_ptr()), _stream(stream)), "importance_scores")
    return out


def merge_tokens(coords, feats, scores, retained, k_m, p_merge, proj_wt, ln_gamma, ln_beta, stream=None):
    """merge_tokens (proj/src/merging.cpp:242-273), batched: coords [B, N, 2] fp32, feats
    [B, N, D] bf16, scores [B, N] fp32, retained [B, R] int32 ascending, p_merge [1] fp32,
    proj_wt [D, 2D] bf16 (the reference's proj_w transposed), ln_gamma / ln_beta [D] fp32 ->
    (retained coords [B, R, 2] fp32, merged feats [B, R, D] bf16)."""
    _req(coords, torch.float32, "coords")
    _req(feats, BF16, "feats")
    _req(scores, torch.float32, "scores")
    _req(retained, torch.int32, "retained")
    _req(proj_wt, BF16, "proj_wt")
    B, N, D = feats.shape
    R = retained.shape[1]
    dev = feats.device
    out_f = torch.empty((B, R, D), dtype=BF16, device=dev)
    out_c = torch.empty((B, R, 2), dtype=torch.float32, device=dev)
    L = capi.lib()
    nbytes = L.affmae_merge_tokens_workspace(C.c_int64(B), C.c_int64(N), C.c_int64(R), C.c_int64(D), C.c_int(k_m))
    ws = _workspace(nbytes, dev)
    capi.check(L.affmae_merge_tokens(
        C.c_void_p(coords.data_ptr()), C.c_void_p(feats.data_ptr()), C.c_void_p(scores.data_ptr()),
        C.c_void_p(retained.data_ptr()), C.c_int64(B), C.c_int64(N), C.c_int64(R), C.c_int64(D), C.c_int(k_m),
        C.c_void_p(p_merge.data_ptr()), C.c_void_p(proj_wt.data_ptr()), C.c_void_p(ln_gamma.data_ptr()),
        C.c_void_p(ln_beta.data_ptr()), C.c_void_p(out_f.data_ptr()), C.c_void_p(out_c.data_ptr()),
        C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel()), _stream(stream)), "merge_tokens")
    return out_c, out_f


def merge_pool_bwd(feats, scores, p_merge, plan: MergePlan, dout, dfeats=None, dscores=None,
                   dp=None, workspace=None, stream=None):
    """MergePoolOp::backward (proj/src/merging.cpp:169-219): dfeats [B, N, D] bf16 and
    dscores [B, N] are overwritten, dp [1] accumulates (+=)."""
    _req(dout, BF16, "dout")
    B, N, D = feats.shape
    R = plan.retained.shape[1]
    dev = feats.device
    if dfeats is None:
        dfeats = torch.empty_like(feats)
    if dscores is None:
        dscores = torch.empty((B, N), dtype=torch.float32, device=dev)
    if dp is None:
        dp = torch.zeros(1, dtype=torch.float32, device=dev)
    L = capi.lib()
    nbytes = L.affmae_merge_pool_bwd_workspace(C.c_int64(B), C.c_int64(R))
    if workspace is None or workspace.numel() < nbytes:
        workspace = _workspace(nbytes, dev)
    ps = plan.c_struct()
    capi.check(L.affmae_merge_pool_bwd(
        C.c_void_p(feats.data_ptr()), C.c_void_p(scores.data_ptr()), C.c_void_p(p_merge.data_ptr()),
        C.c_void_p(plan.retained.data_ptr()), C.byref(ps), C.c_int64(B), C.c_int64(N), C.c_int64(R),
        C.c_int64(D), C.c_int(plan.k_m), C.c_void_p(dout.data_ptr()), C.c_void_p(dfeats.data_ptr()),
        C.c_void_p(dscores.data_ptr()), C.c_void_p(dp.data_ptr()), C.c_void_p(workspace.data_ptr()),
        C.c_size_t(workspace.numel()), _stream(stream)), "merge_pool_bwd")
    return dfeats, dscores, dp
