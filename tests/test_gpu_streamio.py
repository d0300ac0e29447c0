"""F2 wire formats: write_stream output is byte-identical to the reference
CLI `gen` (digests in tests/golden/streamio.json, made by running it)."""

import hashlib
import io
import json
import os

import pytest

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import streamio

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("case", ["raw64_small", "f64le_small", "text_small",
                                  "raw64_multi_chunk", "f64le_multi_chunk"])
def test_write_stream_matches_reference_cli(case):
    g = json.load(open(os.path.join(HERE, "golden", "streamio.json")))["cases"][case]
    p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, g["stream"]))
    st = R.init_vector(p, mv=g["lanes"])
    buf = io.BytesIO()
    n = streamio.write_stream(st, g["count"], buf, case.split("_")[0], chunk=1 << 22)
    data = buf.getvalue()
    assert n == len(data) == g["bytes"]
    assert hashlib.sha256(data).hexdigest() == g["sha256"]


def test_write_stream_errors():
    p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
    st = R.init_vector(p, mv=4)
    with pytest.raises(ValueError):
        streamio.write_stream(st, 10, io.BytesIO(), "csv")
    assert streamio.write_stream(st, 0, io.BytesIO(), "raw64") == 0
