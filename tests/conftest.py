import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running case")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)


def oracle_encoding(stream):
    """The oracle's OracleEncoding for a product CompressedStream (checker
    side only: lets oracle.collage_pass / oracle.decode evaluate a stream the
    device produced)."""
    import oracle as O

    recs = [(int(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4])) for r in stream.records.array]
    return O.OracleEncoding(width=stream.width, height=stream.height, mode=stream.mode,
                            strides=tuple(stream.strides), s_sets=tuple(stream.s_sets),
                            pools=tuple(tuple(map(tuple, p)) if not hasattr(p, "array") else
                                        tuple(map(tuple, p.array.tolist())) for p in stream.pools),
                            records=recs, errors=[], scans={})


def oracle_collage_ssd(stream, pixels):
    """One collage pass of the stream applied to ``pixels`` (oracle), squared
    error against ``pixels``: the encoder's collage SSD (test_codec.py:77-86)."""
    import oracle as O

    enc = oracle_encoding(stream)
    out = O.collage_pass(pixels, enc, O.iter_leaves(enc.width, enc.height, enc.records))
    d = out.astype(np.int64) - pixels.astype(np.int64)
    return int((d * d).sum())
