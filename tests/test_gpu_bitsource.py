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


@pytest.mark.parametrize("sel", bitsource.SELECTORS)
@pytest.mark.parametrize("k,mv", [(2, 64), (3, 1 << 16)])
def test_one_launch_interleave_equals_per_stream(sel, k, mv):
    """The one-launch interleaved fill (RSA_FLAG_INTERLEAVE / RSA_FLAG_LOW32)
    equals the per-stream fill + device transpose, through pending draws,
    whole blocks and partial tails, and leaves identical lane states."""
    plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 4, k)
    srcs = []
    for fused in (True, False):
        src = bitsource.BitSource([R.init_vector(p, m0=7, s0=3, mv=mv) for p in plist], sel)
        if not fused:
            src._fused = None
        else:
            assert src._fused is not None
        srcs.append(src)
    takes = [5, mv * k * 3 + 1, mv * 5, 3 * mv * k, 17, mv * k * 40 + 3]
    for n in takes:
        a, b = (s.take(n).cpu().numpy() for s in srcs)
        assert np.array_equal(a, b), n
    for x, y in zip(srcs[0].streams, srcs[1].streams):
        assert x.draws == y.draws
        for name in ("m1", "m2", "s", "_pending"):
            assert np.array_equal(getattr(x, name).cpu().numpy(), getattr(y, name).cpu().numpy()), name
