"""CPU: the C-ABI library loads and exports every symbol include/affmae_b200.h declares,
and its host-only entry points behave like the reference (no GPU compute here)."""
import ctypes as C
import os
import re

import pytest

from oracle import port
from paper_2602_16249_b200 import capi

HDR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "affmae_b200.h")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"\b(affmae_[a-z0-9_]+)\s*\(", src)))


def test_header_and_exports_agree():
    assert declared() == sorted(capi.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = capi.lib()
    missing = [s for s in declared() if not hasattr(L, s)]
    assert not missing, missing


def test_geometry_closed_forms():
    for n, s, g in ((16384, 16, 3), (8281, 16, 3), (10, 8, 3), (1, 16, 3), (77, 8, 3)):
        geo = capi.geometry(2, n, s, g)
        assert (geo.n_clusters, geo.groups_eff, geo.max_size, geo.width) == port.cluster_shape(n, s, g)


def test_errors_map_to_reference_taxonomy():
    with pytest.raises(ValueError, match="empty point set"):
        capi.geometry(1, 0, 16, 3)
    with pytest.raises(ValueError, match="size must be"):
        capi.geometry(1, 10, 0, 3)


def test_retained_count_matches_oracle():
    L = capi.lib()
    for n in (1, 2, 7, 100, 4096, 16384):
        for ds in (0.25, 0.35, 0.4, 0.5, 1.0):
            assert L.affmae_retained_count(n, ds) == port.retained_count(n, ds)
    assert L.affmae_retained_count(10, 0.0) == -2


def test_workspace_queries_are_host_side():
    L = capi.lib()
    geo = capi.geometry(4, 16384, 16, 3)
    assert L.affmae_cluster_index_workspace(C.byref(geo)) > 0
    d = capi.AttnDesc(4, 32, 8, 8.0)
    assert L.affmae_attn_bwd_workspace(C.byref(geo), C.byref(d)) > L.affmae_attn_fwd_workspace(C.byref(geo), C.byref(d))
    d_bad = capi.AttnDesc(4, 24, 8, 8.0)
    assert L.affmae_attn_fwd_workspace(C.byref(geo), C.byref(d_bad)) == 0


def test_aft_header_parsing_is_host_only(tmp_path):
    """affmae_aft_read_header (write_aft's header, proj/src/tensor_io.cpp:51-57,78-92) on files
    written by the compiled reference, and the ConfigError cases -- no device needed."""
    import numpy as np
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    L = capi.lib()
    p = str(tmp_path / "t.aft")
    ref.write_aft(p, np.zeros((3, 4, 5)), 1)
    dt, nd, dims = C.c_int(), C.c_int(), (C.c_int64 * 8)()
    capi.check(L.affmae_aft_read_header(p.encode(), C.byref(dt), C.byref(nd), dims))
    assert (dt.value, nd.value, list(dims[:3])) == (1, 3, [3, 4, 5])
    (tmp_path / "bad.aft").write_bytes(b"AFT1" + bytes([7]) + bytes(4))
    with pytest.raises(ValueError, match="bad AFT1 dtype"):
        capi.check(L.affmae_aft_read_header(str(tmp_path / "bad.aft").encode(), C.byref(dt), C.byref(nd), dims))
    (tmp_path / "nd.aft").write_bytes(b"AFT1" + bytes([0]) + (9).to_bytes(4, "little"))
    with pytest.raises(ValueError, match="implausible AFT1 ndim"):
        capi.check(L.affmae_aft_read_header(str(tmp_path / "nd.aft").encode(), C.byref(dt), C.byref(nd), dims))
    with pytest.raises(ValueError, match="no checkpoint index"):
        capi.check(L.affmae_checkpoint_load(str(tmp_path / "none").encode(), 0, None, None, None, None))


def test_flop_count_attn_golden():
    """Golden values of proj/tests/test_attention.cpp:193-198."""
    assert capi.flop_count_attn(4096, 192, 6, 64) == 1242710016
    assert capi.flop_count_attn(1, 1, 1, 1) == 4 * 2 + 6 * 2
    assert capi.flop_count_attn_dense(256, 2, 8) == 4 * 256 * 256 * 2 * 8 + 6 * 256 * 256 * 2
    with pytest.raises(ValueError, match="positive"):
        capi.flop_count_attn(0, 48, 4, 32)


def test_malformed_aft1_is_a_config_error(tmp_path):
    """Extents whose product overflows int64 (or exceeds INT64_MAX) are rejected with
    ConfigError before any allocation, instead of aborting the host process."""
    import struct
    L = capi.lib()
    for dims in ([1 << 62, 4], [1 << 63, 1], [3, 5]):
        p = tmp_path / "bad.aft"
        p.write_bytes(b"AFT1" + bytes([0]) + struct.pack("<I", len(dims)) +
                      b"".join(struct.pack("<Q", d) for d in dims))
        rc = L.affmae_aft_read(str(p).encode(), None, C.c_int64(1 << 40), None, None)
        assert rc == capi.ECONFIG, dims
        msg = L.affmae_last_error().decode()
        if dims[0] > 3:
            assert "implausible" in msg, msg
