"""F3 interleaved BitSource on the device against the reference's own
stats.BitSource output (tests/golden/bitsource.npz)."""

import json
import os

import numpy as np
import pytest

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("sel", bitsource.SELECTORS)
@pytest.mark.parametrize("k", [1, 3])
def test_bitsource_matches_reference(sel, k):
    meta = json.load(open(os.path.join(HERE, "golden", "bitsource.json")))
    with np.load(os.path.join(HERE, "golden", "bitsource.npz")) as z:
        want = z[f"bitsource_{sel}_{k}"]
    src = bitsource.interstream_source(R.DEFAULT_MASTER_SEED, meta["streams"][0], k, meta["lanes"], sel)
    got = np.concatenate([src.take(n).cpu().numpy() for n in meta["takes"]])
    assert got.dtype == want.dtype
    assert np.array_equal(got, want)


def test_bitsource_errors():
    with pytest.raises(ValueError):
        bitsource.BitSource([], "float_leading")
    p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
    with pytest.raises(ValueError):
        bitsource.BitSource([R.init_vector(p, mv=2)], "nope")
