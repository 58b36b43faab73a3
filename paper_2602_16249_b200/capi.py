"""ctypes binding of the C ABI in ``include/affmae_b200.h`` (libaffmae_b200.so).

This is the thin layer the Python side (tests, bench, the torch-facing op
wrappers in :mod:`paper_2602_16249_b200.ops`) uses to reach the CUDA kernels.
Device memory comes from torch tensors (``data_ptr()``) and streams from
``torch.cuda.current_stream()`` -- torch is plumbing here, every compute call
goes through the C ABI.  There is no fallback: if the shared library is
missing, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libaffmae_b200.so")

OK, ECONFIG, ENUMERIC, EUNSUPPORTED, ECUDA = 0, 2, 3, 4, 5

# Every symbol include/affmae_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "affmae_last_error", "affmae_version", "affmae_cluster_geometry",
    "affmae_cluster_index_workspace", "affmae_cluster_index_build", "affmae_neighbor_expand",
    "affmae_sfc_order_workspace", "affmae_sfc_order", "affmae_knn",
    "affmae_attn_fwd_workspace", "affmae_attn_fwd", "affmae_attn_bwd_workspace", "affmae_attn_bwd",
    "affmae_attn_plan_workspace", "affmae_attn_plan_build", "affmae_attn_fwd_planned_workspace",
    "affmae_attn_fwd_planned", "affmae_attn_bwd_planned_workspace", "affmae_attn_bwd_planned",
    "affmae_retained_count", "affmae_select_retained_workspace", "affmae_select_retained",
    "affmae_merge_plan_workspace", "affmae_merge_plan_build", "affmae_merge_pool_fwd",
    "affmae_importance_scores", "affmae_merge_tokens_workspace", "affmae_merge_tokens",
    "affmae_merge_pool_bwd_workspace", "affmae_merge_pool_bwd", "affmae_interp_fwd", "affmae_interp_bwd",
    "affmae_adamw_lr", "affmae_adamw_step", "affmae_linear_workspace", "affmae_linear_fwd",
    "affmae_linear_bwd_workspace", "affmae_linear_bwd", "affmae_linear_fwd_gelu_aux", "affmae_gelu_bwd", "affmae_linear_fwd_add", "affmae_linear_dx_gelu", "affmae_linear_dx_f32", "affmae_layernorm_fwd", "affmae_layernorm_bwd_workspace",
    "affmae_layernorm_bwd", "affmae_norm_clamp_fwd", "affmae_norm_clamp_bwd", "affmae_masked_mse_workspace",
    "affmae_masked_mse", "affmae_gattn_fwd", "affmae_gattn_bwd", "affmae_gattn_bwd_workspace",
    "affmae_interp_bwd_gather_workspace", "affmae_interp_bwd_gather", "affmae_perlin_mask_workspace",
    "affmae_perlin_mask", "affmae_visible_coords", "affmae_synth_images_workspace", "affmae_synth_images",
    "affmae_patchify", "affmae_masked_rows", "affmae_aft_write", "affmae_aft_read_header",
    "affmae_aft_read", "affmae_checkpoint_save", "affmae_checkpoint_load",
    "affmae_flop_count_attn", "affmae_flop_count_attn_dense",
    "affmae_model_create", "affmae_model_destroy", "affmae_model_get_info", "affmae_model_param_name",
    "affmae_model_param_dims", "affmae_model_get_params", "affmae_model_set_params", "affmae_model_get_grads",
    "affmae_model_inputs", "affmae_model_make_masks", "affmae_model_forward_backward", "affmae_model_apply_step",
    "affmae_model_train_step", "affmae_model_grad_buffer", "affmae_model_save", "affmae_model_load",
    "affmae_model_stage_output", "affmae_model_force_retained", "affmae_model_forward",
    "affmae_model_reset_optimizer", "affmae_hilbert_index", "affmae_nccl_unique_id", "affmae_model_set_world",
)


class AffmaeError(RuntimeError):
    pass


class ClusterGeom(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("batch", "tokens", "cluster", "groups", "n_clusters",
                                         "groups_eff", "max_size", "width")]


class ClusterIndex(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("perm", "cluster_of", "nbr_cl", "rev_off", "rev_cl")]


class AttnDesc(C.Structure):
    _fields_ = [("heads", C.c_int), ("head_dim", C.c_int), ("bias_hidden", C.c_int),
                ("patch", C.c_double)]


class AttnInputs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("q", "k", "v", "blank_k", "blank_v", "coords", "w1",
                                          "b1", "w2", "b2", "blank")]


class AdamwCfg(C.Structure):
    _fields_ = [("lr", C.c_double), ("warmup", C.c_int64), ("weight_decay", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("total_steps", C.c_int64)]


class AttnGrads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("dq", "dk", "dv", "dblank_k", "dblank_v", "dw1", "db1",
                                          "dw2", "db2", "dblank")]


class AttnPlan(C.Structure):
    _fields_ = [("buf", C.c_void_p), ("bytes", C.c_size_t)] + \
        [(n, C.c_int64) for n in ("batch", "tokens", "n_clusters", "groups_eff", "width")] + \
        [("patch", C.c_double), ("has_reverse", C.c_int)]


class MergePlan(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("target", "pool_idx", "pool_dist", "pool_cnt", "row_of")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise AffmaeError(
                f"CUDA extension missing: {LIB_PATH}; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.affmae_last_error.restype = C.c_char_p
        L.affmae_retained_count.restype = C.c_int64
        L.affmae_retained_count.argtypes = [C.c_int64, C.c_double]
        if hasattr(L, "affmae_hilbert_index"):
            L.affmae_hilbert_index.restype = C.c_uint64
            L.affmae_hilbert_index.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        for f in ("affmae_flop_count_attn", "affmae_flop_count_attn_dense"):
            if hasattr(L, f):
                getattr(L, f).restype = C.c_uint64
        if hasattr(L, "affmae_adamw_lr"):
            L.affmae_adamw_lr.restype = C.c_double
        # every size query returns size_t: without the restype ctypes would truncate it to a
        # 32-bit int (a >= 2 GiB workspace would come back wrong)
        for f in EXPORTS:
            if f.endswith("_workspace") and hasattr(L, f):
                getattr(L, f).restype = C.c_size_t
        _lib = L
    return _lib


def check(rc: int, what: str = ""):
    """Maps status codes onto the reference's exception taxonomy (ConfigError ->
    ValueError, NumericError -> ArithmeticError; proj/bindings/module.cpp:91-92)."""
    if rc == OK:
        return
    msg = lib().affmae_last_error().decode()
    if what:
        msg = f"{what}: {msg}"
    if rc in (ECONFIG, EUNSUPPORTED):
        raise ValueError(msg)
    if rc == ENUMERIC:
        raise ArithmeticError(msg)
    raise AffmaeError(msg)


def ptr(t) -> int | None:
    """Device address of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def geometry(batch: int, tokens: int, cluster: int, groups: int) -> ClusterGeom:
    g = ClusterGeom(batch, tokens, cluster, groups, 0, 0, 0, 0)
    check(lib().affmae_cluster_geometry(C.byref(g)), "cluster_geometry")
    return g


def flop_count_attn(n: int, m: int, h: int, d: int) -> int:
    """flop_count_attn (proj/src/attention.cpp:360-364); ValueError on non-positive args."""
    r = lib().affmae_flop_count_attn(C.c_int64(n), C.c_int64(m), C.c_int64(h), C.c_int64(d))
    if r == 0:
        check(ECONFIG, "flop_count_attn")
    return int(r)


def flop_count_attn_dense(n: int, h: int, d: int) -> int:
    """flop_count_attn_dense (proj/src/attention.cpp:366-370)."""
    r = lib().affmae_flop_count_attn_dense(C.c_int64(n), C.c_int64(h), C.c_int64(d))
    if r == 0:
        check(ECONFIG, "flop_count_attn_dense")
    return int(r)
