"""Model files: save_model / load_model (format :373).

Pins: the product's writer (csrc/model_io.cu) emits exactly the bytes the reference's own
BinaryWriter (proj/core/src/binary_io.cpp, compiled by oracle/make_ref_golden.sh) emits for the
same record — tests/golden/ref_infra.json model_*_hex; the product reader and the oracle's
streaming reader both accept those files and reject truncated / corrupted / wrong-version /
wrong-magic files with IoError; on the GPU, load -> predict equals predict of the operator built
from the same parameters bit for bit, and save -> load -> predict is bit-identical.
"""
import json
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2509_01416_b200 import operators as OPS, snop
from paper_2509_01416_b200.errors import InvalidArgument, IoError
from tests import oracle_lib as O

GOLD = json.loads((Path(__file__).parent / "golden" / "ref_infra.json").read_text())


def _fnv1a(b: bytes) -> int:
    h = 0xcbf29ce484222325
    for x in b:
        h = ((h ^ x) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


# The tiny architectures of oracle/ref_golden_main.cpp (parameters exact in fp32).
def tiny_deeponet():
    bs, ts = [4, 3, 2], [1, 3, 2]
    nbp = 4 * 3 + 3 + 3 * 2 + 2
    ntp = 1 * 3 + 3 + 3 * 2 + 2
    bp = np.array([((i % 7) - 3) * 0.125 for i in range(nbp)], np.float32)
    tp = np.array([((i % 5) - 2) * 0.25 for i in range(ntp)], np.float32)
    prm = OPS.DeepONetParams(OPS.dense_from_packed(bs, bp), OPS.dense_from_packed(ts, tp), OPS.TANH, 0.125)
    return snop.Grid1D(10.0, 4), prm, (1.0, 0.5)


def tiny_fno():
    n = 3 * 2 + 1 * (2 * 2 * 2 * 2 + 2 * 2 + 2) + 3 * 2 + 2 * 3 + 1
    flat = np.array([float((((i * 3) % 11) - 5)) / 16.0 for i in range(n)], np.float32)
    return snop.Grid1D(10.0, 8), OPS.fno_from_packed(2, 2, 1, 3, OPS.GELU, flat), (1.0, 0.8)


def _write_golden(tmp_path, key):
    p = tmp_path / f"{key}.bin"
    p.write_bytes(bytes.fromhex(GOLD[key]))
    return p


def _oracle_load(path):
    import ctypes as C
    h = C.c_void_p()
    code = O.lib().oracle_model_load(str(path).encode(), C.byref(h))
    if code != 0:
        raise O.OracleError(code, O.lib().oracle_last_error().decode())
    return O.OracleOperator(h.value, 0)


def test_golden_digest_is_fnv1a():
    for key in ("model_deeponet_hex", "model_fno_hex"):
        b = bytes.fromhex(GOLD[key])
        assert struct.unpack("<Q", b[-8:])[0] == _fnv1a(b[:-8])


def test_writer_matches_reference_bytes(tmp_path):
    g, prm, ref = tiny_deeponet()
    p = tmp_path / "d.bin"
    snop.write_deeponet_file(p, g, prm, ref)
    assert p.read_bytes().hex() == GOLD["model_deeponet_hex"]
    g, prm, ref = tiny_fno()
    p = tmp_path / "f.bin"
    snop.write_fno_file(p, g, prm, ref)
    assert p.read_bytes().hex() == GOLD["model_fno_hex"]


def test_inspect_golden(tmp_path):
    info = snop.inspect_model(_write_golden(tmp_path, "model_deeponet_hex"))
    assert (info.arch, info.grid.n_cells, info.grid.length_cm) == (0, 4, 10.0)
    assert (info.sigma_t_star, info.sigma_s0_star, info.activation) == (1.0, 0.5, OPS.TANH)
    assert (info.n_branch, info.n_trunk, info.latent, info.has_bias0, info.bias0) == (3, 3, 2, 1, 0.125)
    assert info.n_params == 23 + 14
    info = snop.inspect_model(_write_golden(tmp_path, "model_fno_hex"))
    assert (info.arch, info.grid.n_cells, info.sigma_s0_star, info.activation) == (1, 8, 0.8, OPS.GELU)
    assert (info.width, info.modes, info.layers, info.hidden, info.n_params) == (2, 2, 1, 3, 41)


def test_oracle_loader_reads_golden(tmp_path):
    g, prm, ref = tiny_deeponet()
    op = _oracle_load(_write_golden(tmp_path, "model_deeponet_hex"))
    direct = O.OracleOperator.deeponet(10.0, 4, ref, OPS.TANH, prm.branch.sizes, prm.branch.packed(),
                                       prm.trunk.sizes, prm.trunk.packed(), 0.125)
    s = np.random.default_rng(0).uniform(0, 1, (3, 4))
    assert np.array_equal(op.predict(s), direct.predict(s))
    g, prm, ref = tiny_fno()
    op = _oracle_load(_write_golden(tmp_path, "model_fno_hex"))
    direct = O.OracleOperator.fno(10.0, 8, ref, OPS.GELU, 2, 2, 1, 3, prm.packed())
    s = np.random.default_rng(1).uniform(0, 1, (3, 8))
    assert np.array_equal(op.predict(s), direct.predict(s))


def _corruptions(b: bytes):
    yield "truncated-digest", b[:-3]
    yield "truncated-body", b[: len(b) // 2]
    yield "empty", b""
    flipped = bytearray(b)
    flipped[len(b) // 2] ^= 0x01
    yield "bit-flip", bytes(flipped)
    yield "trailing", b + b"\x00"
    ver = bytearray(b[:-8])
    ver[14] = 2  # u32 version right after the 4+10-byte magic string
    yield "version-2", bytes(ver) + struct.pack("<Q", _fnv1a(bytes(ver)))
    mag = bytearray(b[:-8])
    mag[4] = ord("X")
    yield "bad-magic", bytes(mag) + struct.pack("<Q", _fnv1a(bytes(mag)))


@pytest.mark.parametrize("key", ["model_deeponet_hex", "model_fno_hex"])
def test_corrupt_files_rejected(tmp_path, key):
    good = bytes.fromhex(GOLD[key])
    for name, data in _corruptions(good):
        p = tmp_path / f"{name}.bin"
        p.write_bytes(data)
        with pytest.raises(IoError):
            snop.inspect_model(p)
        with pytest.raises(O.OracleError) as e:
            _oracle_load(p)
        assert e.value.code == 4, name
    with pytest.raises(IoError):
        snop.inspect_model(tmp_path / "missing.bin")


def test_c2_size_roundtrip_header(tmp_path):
    prm = OPS.deeponet_init(2000, width=128, activation=OPS.TANH)
    p = tmp_path / "c2.bin"
    snop.write_deeponet_file(p, snop.Grid1D(10.0, 2000), prm)
    info = snop.inspect_model(p)
    assert info.n_params == prm.branch.packed().size + prm.trunk.packed().size
    assert p.stat().st_size == 8 * info.n_params + 8 + 4 + 10 + 4 + 4 + 8 + 8 + 8 + 8 + 8 + 4 + 4 + 8 * 5 + 4 + 8 * 5 + 1 + 8 + 8
    o = _oracle_load(p)
    d = O.OracleOperator.deeponet(10.0, 2000, (1.0, 0.5), OPS.TANH, prm.branch.sizes, prm.branch.packed(),
                                  prm.trunk.sizes, prm.trunk.packed())
    s = np.random.default_rng(2).uniform(0, 1, (2, 2000))
    assert np.array_equal(o.predict(s), d.predict(s))


# ---------------------------------------------------------------- device --------------------------
@pytest.mark.gpu
def test_gpu_load_golden_equals_create(tmp_path):
    for make, key, factory in ((tiny_deeponet, "model_deeponet_hex", snop.SolutionOperator.deeponet),
                               (tiny_fno, "model_fno_hex", snop.SolutionOperator.fno)):
        g, prm, ref = make()
        loaded = snop.SolutionOperator.load(_write_golden(tmp_path, key))
        assert loaded.grid == g and loaded.reference_params == ref
        direct = factory(g, prm, ref)
        s = np.random.default_rng(3).uniform(0, 1, (5, g.n_cells))
        a, b = loaded.predict(s), direct.predict(s)
        assert np.array_equal(a, b)
        o = _oracle_load(tmp_path / f"{key}.bin").predict(s)
        assert np.max(np.abs(a - o)) / np.max(np.abs(o)) < 1e-5


@pytest.mark.gpu
def test_gpu_save_load_predict_bit_identical(tmp_path):
    g = snop.Grid1D(10.0, 2000)
    op = snop.SolutionOperator.deeponet(g, OPS.deeponet_init(2000, width=128, activation=OPS.TANH))
    s = np.random.default_rng(4).uniform(0, 1, (8, 2000))
    before = op.predict(s)
    op.save(tmp_path / "don.bin")
    again = snop.SolutionOperator.load(tmp_path / "don.bin")
    assert np.array_equal(again.predict(s), before)
    gf = snop.Grid1D(10.0, 1024)
    fop = snop.SolutionOperator.fno(gf, OPS.fno_init(64, 16, 4, 128, OPS.GELU))
    sf = np.random.default_rng(5).uniform(0, 1, (8, 1024))
    before = fop.predict(sf)
    fop.save(tmp_path / "fno.bin")
    assert np.array_equal(snop.SolutionOperator.load(tmp_path / "fno.bin").predict(sf), before)
    ex = snop.SolutionOperator.exact(gf, 8)
    with pytest.raises(InvalidArgument):
        ex.save(tmp_path / "exact.bin")
