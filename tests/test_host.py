"""Host-side logic and the C ABI surface (CPU only, no GPU compute)."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_1502_00324_b200 as fc
from paper_1502_00324_b200 import _native, stream as st
import oracle as O
from paper_1502_00324_b200.codec import _quadtree
from conftest import ROOT, load_golden, oracle_collage_ssd, oracle_encoding


def _header_symbols():
    text = Path(ROOT, "include", "fracodec_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|void|const char\*)\s+(fc_\w+)\(", text, re.M)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _native.load_library()
    syms = _header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_native.exported_symbols())
    assert lib.fc_version() == 1


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_native.DeviceUnavailableError):
        _native.Context()
    with pytest.raises(_native.DeviceUnavailableError):
        fc.encode(fc.GrayImage.full(32, 32, 1), fc.EncoderConfig(pool=fc.PoolParams(pool_cap=2)))


def test_entropy_lut_matches_numpy_entropy_terms():
    for n in (16, 64, 256, 1024):
        lut = _native.entropy_lut(n)
        counts = np.arange(1, n + 1).reshape(1, -1)
        p = counts / n
        assert (p * np.log(p)).ravel().tobytes() == lut.tobytes()


@pytest.mark.parametrize("golden,tag", [
    ("encode_cases.npz", "tiled_proposed"), ("encode_cases.npz", "tiled_baseline"),
    ("encode_cases.npz", "noise"), ("encode_cases.npz", "flat"), ("encode_cases.npz", "c1"),
    ("encode_lena.npz", "lena256")])
def test_stream_roundtrip_and_decoder_on_golden(golden, tag):
    g = load_golden(golden)
    data = g[f"bytes_{tag}"].tobytes()
    s = fc.deserialize(data)
    assert fc.serialize(s) == data
    recs = np.array([(r.step, r.offset, r.isometry, r.domain_address, r.s_index) for r in s.records])
    assert np.array_equal(recs, g[f"records_{tag}"])
    # leaf origins (Z-order decode) == the oracle's depth-first walk
    enc = oracle_encoding(s)
    walk = O.iter_leaves(enc.width, enc.height, enc.records)
    x, y, side = fc.leaf_origins(s)
    assert list(zip(x.tolist(), y.tolist(), side.tolist())) == [(a, b, c) for _, a, b, c in walk]
    if tag != "lena256":
        dec, deltas = O.decode(enc)
        assert np.array_equal(dec, g[f"decoded_{tag}"])
        assert deltas == list(g[f"deltas_{tag}"])
    # encoder bookkeeping == one decoder pass on the original (test_codec.py:77-86)
    assert oracle_collage_ssd(s, g[f"image_{tag}"]) == int(g[f"collage_{tag}"])


def test_stream_error_taxonomy():
    good = st.CompressedStream(16, 16, "proposed", (8, 4, 2, 2), ((0.1,), (0.2, 0.4), (0.3, 0.8), (0.5, 0.9)),
                               (((0, 0), (4, 0), (8, 0)),) * 4, (st.MatchRecord(1, 128, 0, 0, 0),))
    data = fc.serialize(good)
    assert fc.deserialize(data) == good
    with pytest.raises(st.BadMagicError):
        fc.deserialize(b"JUNK" + data[4:])
    with pytest.raises(st.VersionMismatchError):
        fc.deserialize(data[:4] + bytes([9]) + data[5:])
    with pytest.raises(st.TruncatedStreamError):
        fc.deserialize(data[:-1])
    bad = st.CompressedStream(16, 16, "proposed", good.strides, good.s_sets, good.pools,
                              (st.MatchRecord(1, 128, 0, 3, 0),))
    with pytest.raises(ValueError):
        fc.serialize(bad)
    # address 3 in a 3-entry pool, packed by hand: step 0, off 128, iso 0, addr 3 (2 bits)
    hand = bytearray(data)
    payload_at = len(data) - 2
    bits = "00" + format(128, "08b") + "000" + "11"
    hand[payload_at:] = int(bits.ljust(16, "0"), 2).to_bytes(2, "big")
    with pytest.raises(st.AddressRangeError):
        fc.deserialize(bytes(hand))


def test_quadtree_child_order_and_dfs():
    calls = {}

    def match(level, origins):
        calls[level] = [tuple(o) for o in origins]
        errs = np.zeros(len(origins))
        if level < 4:
            errs[0] = 1e18
        return errs

    leaves = fc.run_quadtree(16, 16, (1.0, 1.0, 1.0), match)
    assert calls[2] == [(0, 0), (8, 0), (0, 8), (8, 8)]
    assert calls[3] == [(0, 0), (4, 0), (0, 4), (4, 4)]
    assert calls[4] == [(0, 0), (2, 0), (0, 2), (2, 2)]
    assert [lv for lv, _, _, _ in leaves] == [4, 4, 4, 4, 3, 3, 3, 2, 2, 2]


def test_quadtree_matches_oracle_driver_on_random_splits():
    import oracle as O

    rng = np.random.default_rng(5)
    draws = {}

    def errs_for(level, n):
        key = (level, n)
        if key not in draws:
            draws[key] = rng.integers(0, 3, n) * 1e9
        return draws[key]

    ref = O.run_quadtree(64, 48, (1.0, 1.0, 1.0), lambda lv, o: errs_for(lv, len(o)))
    got = fc.run_quadtree(64, 48, (1.0, 1.0, 1.0), lambda lv, o: errs_for(lv, len(o)))
    assert got == ref


def test_coord_table_equality():
    t = fc.CoordTable(np.array([[1, 2], [3, 4]]))
    assert t == ((1, 2), (3, 4))
    assert t[1] == (3, 4) and len(t) == 2
    assert t != ((1, 2),)


def test_workload_generators_are_deterministic():
    from paper_1502_00324_b200 import workloads as W

    a = W.make_image("c1")
    assert a.shape == (128, 128) and a.dtype == np.uint8
    assert np.array_equal(a, W.make_image("c1"))
    assert set(W.WORKLOADS) == {"c1", "c2", "c3", "c4", "c5"}


def test_native_record_packer_matches_numpy_packer():
    """fc_pack_records (host C, used by serialize for the device encoder's int32
    records) produces the bytes of the numpy word packer, and rejects records
    outside their level's pool / s set."""
    rng = np.random.default_rng(7)
    abits = np.array([0, 5, 17, 23], dtype=np.int64)
    sbits = np.array([0, 1, 1, 3], dtype=np.int64)
    plen = np.array([1, 20, 100000, 5000000], dtype=np.int64)
    slen = np.array([1, 2, 2, 7], dtype=np.int64)
    for n in (1, 2, 7, 1000, 4099):
        steps = rng.integers(1, 5, n)
        rec = np.stack([steps, rng.integers(0, 256, n), rng.integers(0, 8, n),
                        rng.integers(0, plen[steps - 1]), rng.integers(0, slen[steps - 1]),
                        rng.integers(0, 1 << 20, n)], axis=1).astype(np.int32)
        r = rec[:, :5]  # strided int32 view, as codec.encode hands it over
        got, nbits = _native.pack_records(r, abits, sbits, plen, slen)
        lv = steps - 1
        u = r.astype(np.uint64)
        val = (lv.astype(np.uint64) << np.uint64(8)) | u[:, 1]
        val = (val << np.uint64(3)) | u[:, 2]
        val = (val << abits[lv].astype(np.uint64)) | u[:, 3]
        val = (val << sbits[lv].astype(np.uint64)) | u[:, 4]
        widths = 13 + abits[lv] + sbits[lv]
        assert nbits == int(widths.sum())
        assert got == st._pack_words(val, widths)
    bad = rec.copy()
    bad[3, 3] = plen[bad[3, 0] - 1]
    with pytest.raises(IndexError):
        _native.pack_records(bad[:, :5], abits, sbits, plen, slen)
