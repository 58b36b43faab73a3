"""AFT1 files and checkpoints from / into device memory against the
reference's own write_aft / write_aft_u8 / read_aft (proj/src/tensor_io.cpp:60-105, compiled
into oracle/_ref): byte-identical files, exact values back, and load_checkpoint's ConfigError
cases (proj/src/pipeline.cpp:772-797)."""
import os

import numpy as np
import pytest

from oracle import ref

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _dev(a, dt=None):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda", dtype=dt)


@pytest.mark.parametrize("shape,prec", [((3, 5), 0), ((7,), 0), ((2, 3, 4), 1), ((1, 1), 0), ((4, 2), 2)])
def test_aft_write_is_byte_identical_to_reference(tmp_path, shape, prec):
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(sum(shape) + prec)
    v = rng.standard_normal(shape).astype(np.float32)
    if prec == 1:  # b16emu tensors hold binary16 values
        v = v.astype(np.float16).astype(np.float32)
    ours, theirs = str(tmp_path / "ours.aft"), str(tmp_path / "ref.aft")
    # a b64 tensor is stored as b32 (include/affmae/tensor_io.hpp:14): write it with code 0
    ops.aft_write(ours, _dev(v), dtype=0 if prec == 2 else prec)
    ref.write_aft(theirs, v.astype(np.float64), prec)
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_aft_u8_and_read_back(tmp_path):
    import torch
    from paper_2602_16249_b200 import ops
    b = np.arange(24, dtype=np.uint8).reshape(4, 6) * 7
    ours, theirs = str(tmp_path / "m.aft"), str(tmp_path / "m_ref.aft")
    ops.aft_write(ours, _dev(b, torch.uint8), dtype=2)
    ref.write_aft_u8(theirs, b)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    t, dt = ops.aft_read(theirs)
    assert dt == 2 and tuple(t.shape) == (4, 6)
    np.testing.assert_array_equal(t.cpu().numpy(), b.astype(np.float32))


def test_aft_read_reference_file_exact(tmp_path):
    from paper_2602_16249_b200 import ops
    v = np.random.default_rng(1).standard_normal((5, 9)).astype(np.float32)
    p = str(tmp_path / "r.aft")
    ref.write_aft(p, v.astype(np.float64), 0)
    t, dt = ops.aft_read(p)
    assert dt == 0
    np.testing.assert_array_equal(t.cpu().numpy(), v)
    vals, rdt = ref.read_aft(p)  # and the reference reads our write of it back identically
    ops.aft_write(str(tmp_path / "w.aft"), t)
    vals2, _ = ref.read_aft(str(tmp_path / "w.aft"))
    np.testing.assert_array_equal(vals, vals2)


def test_aft_rejects_bad_files(tmp_path):
    from paper_2602_16249_b200 import ops
    p = tmp_path / "bad.aft"
    p.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(ValueError, match="not an AFT1"):
        ops.aft_read(str(p))
    ref.write_aft(str(tmp_path / "t.aft"), np.ones((4, 4)), 0)
    raw = (tmp_path / "t.aft").read_bytes()
    (tmp_path / "trunc.aft").write_bytes(raw[:-5])
    with pytest.raises(ValueError, match="truncated"):
        ops.aft_read(str(tmp_path / "trunc.aft"))


def test_checkpoint_round_trip_and_reference_format(tmp_path):
    import torch
    from paper_2602_16249_b200 import ops
    rng = np.random.default_rng(4)
    params = {"enc.s0.wq": (_dev(rng.standard_normal((8, 4)).astype(np.float32)), "b32"),
              "enc.s0.ln1.g": (_dev(np.ones(8, np.float32)), "b32"),
              "dec.mask_token": (_dev(rng.standard_normal((1, 8)).astype(np.float16).astype(np.float32)), "b16emu")}
    d = tmp_path / "ckpt"
    ops.save_checkpoint(str(d), params)
    manifest = (d / "manifest.tsv").read_text()
    assert manifest == ("enc.s0.wq\t8x4\tb32\tenc.s0.wq.aft\n" "enc.s0.ln1.g\t8\tb32\tenc.s0.ln1.g.aft\n"
                        "dec.mask_token\t1x8\tb16emu\tdec.mask_token.aft\n")
    for k, (t, prec) in params.items():  # the reference reads every file back exactly
        vals, dt = ref.read_aft(str(d / f"{k}.aft"))
        assert dt == (1 if prec == "b16emu" else 0)
        np.testing.assert_array_equal(vals, t.cpu().numpy().reshape(-1).astype(np.float64))
    dst = {k: torch.zeros_like(t) for k, (t, _) in params.items()}
    ops.load_checkpoint(str(d), dst)
    for k in params:
        assert torch.equal(dst[k], params[k][0])
    with pytest.raises(ValueError, match="missing parameter"):
        ops.load_checkpoint(str(d), {**dst, "extra": torch.zeros(3, device="cuda")})
    with pytest.raises(ValueError, match="unknown parameter"):
        ops.load_checkpoint(str(d), {k: dst[k] for k in list(dst)[:2]})
    with pytest.raises(ValueError, match="size mismatch|too small"):
        ops.load_checkpoint(str(d), {**dst, "enc.s0.ln1.g": torch.zeros(4, device="cuda")})


def test_adamw_checkpoint_resumes_bit_identically(tmp_path):
    """Parameters + AdamW moments + step through the AFT1 checkpoint: a resumed optimizer takes
    the same next step as the uninterrupted one (the reference saves values only)."""
    import torch
    from paper_2602_16249_b200 import ops
    shapes, names = [(16, 8), (8,), (3, 5)], ["w", "b", "u"]
    rng = np.random.default_rng(8)

    def run(opt, steps):
        for _ in range(steps):
            for g in opt.grads:
                g.copy_(torch.as_tensor(rng.standard_normal(tuple(g.shape)), dtype=torch.float32))
            opt.step()

    a = ops.AdamW(shapes, warmup=2, total_steps=10)
    for p in a.params:
        p.copy_(torch.as_tensor(rng.standard_normal(tuple(p.shape)), dtype=torch.float32))
    run(a, 3)
    a.save(str(tmp_path / "ck"), names)
    # the parameter manifest stays loadable by the reference (optimizer state lives in optim/)
    if ref.available():
        got = ref.load_checkpoint(str(tmp_path / "ck"), names, [p.numel() for p in a.params])
        for nm, p in zip(names, a.params):
            np.testing.assert_array_equal(got[nm], p.cpu().numpy().ravel().astype(np.float64))
    b = ops.AdamW(shapes, warmup=2, total_steps=10)
    b.load(str(tmp_path / "ck"), names)
    assert b.t == 3 and torch.equal(b.value, a.value) and torch.equal(b.m, a.m) and torch.equal(b.v, a.v)
    g = [torch.as_tensor(rng.standard_normal(tuple(x.shape)), dtype=torch.float32) for x in a.grads]
    for opt in (a, b):
        for dst, src in zip(opt.grads, g):
            dst.copy_(src)
        opt.step()
    torch.cuda.synchronize()
    assert torch.equal(a.value, b.value)


def test_adamw_loads_plain_reference_checkpoint(tmp_path):
    """A checkpoint without optimizer state (the reference's save_checkpoint layout) loads
    into AdamW: parameters restored, moments zero, step 0."""
    import torch
    from paper_2602_16249_b200 import ops
    shapes, names = [(4, 3), (3,)], ["w", "b"]
    vals = [np.arange(12, dtype=np.float64).reshape(4, 3) / 7, np.array([0.5, -1.0, 2.0])]
    d = tmp_path / "plain"
    d.mkdir()
    with open(d / "manifest.tsv", "w") as f:
        for nm, v in zip(names, vals):
            ref.write_aft(str(d / f"{nm}.aft"), v)
            f.write(f"{nm}\t{'x'.join(map(str, v.shape))}\tb32\t{nm}.aft\n")
    a = ops.AdamW(shapes)
    a.m.fill_(3.0)
    a.t = 5
    a.load(str(d), names)
    assert a.t == 0 and float(a.m.abs().sum()) == 0.0
    for p, v in zip(a.params, vals):
        np.testing.assert_array_equal(p.cpu().numpy(), v.astype(np.float32))
