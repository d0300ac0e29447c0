"""F1 fused battery consumers (csrc/battery_fused.cu) against the
materialised path and a numpy restatement, on awkward layouts: a source
already part-consumed (buffered surplus + pending draws), tails that end
mid-block, tuple lengths that do not divide the tile, 1 / 2 / 4 streams, both
selectors.  The fused path must count exactly what the materialised variates
give and leave the source in exactly the same state."""

import numpy as np
import pytest
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import _lib, bitsource, stats

pytestmark = pytest.mark.gpu


class Proxy:
    """Hides the BitSource type: forces the materialised path."""

    def __init__(self, src):
        self.src = src

    def take(self, n):
        return self.src.take(n)


def make(k, mv, sel, first=11):
    plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, first, k) if k > 1 else \
        [R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, first))]
    return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=mv) for p in plist], sel)


CASES = [  # streams, lanes, selector, variates consumed before the test
    (2, 1024, "float_leading", 0),
    (2, 1024, "float_leading", 555),
    (1, 512, "raw_low_bits", 77),
    (4, 256, "float_leading", 1001),
    (2, 128, "raw_low_bits", 3),
]
KINDS = [  # (kind, d, p1, p2, cells)
    (_lib.RSA_BT_HIST, 1, 1 << 20, 0, 1 << 20),
    (_lib.RSA_BT_SERIAL, 2, 2, 1024, 1 << 20),
    (_lib.RSA_BT_SERIAL, 3, 3, 100, 10 ** 6),
    (_lib.RSA_BT_SERIAL, 6, 6, 10, 10 ** 6),
    (_lib.RSA_BT_POKER, 5, 0, 0, 5),
    (_lib.RSA_BT_MAX_OF_T, 32, 32, 128, 128),
    (_lib.RSA_BT_MAX_OF_T, 7, 7, 100, 100),
    (_lib.RSA_BT_PERMUTATION, 9, 9, 0, 362880),
    (_lib.RSA_BT_PERMUTATION, 3, 3, 0, 6),
]


@pytest.mark.parametrize("k,mv,sel,pre", CASES)
@pytest.mark.parametrize("kind,d,p1,p2,cells", KINDS)
def test_fused_counts_equal_materialised(k, mv, sel, pre, kind, d, p1, p2, cells):
    a, b = make(k, mv, sel), make(k, mv, sel)
    if pre:
        a.take(pre)
        b.take(pre)
    n_tuples = (7 * k * mv + 333) // d + 5  # several whole blocks and a ragged tail
    assert stats._fused_plan(a, n_tuples * d) is not None
    ta, tb = stats._Tally(cells), stats._Tally(cells)
    stats._count_tuples(a, kind, d, p1, p2, n_tuples, ta)
    stats._count_tuples(Proxy(b), kind, d, p1, p2, n_tuples, tb)
    assert torch.equal(ta.cells, tb.cells)
    assert int(ta.cells.sum().item()) == n_tuples
    assert int(ta.tie.item()) == int(tb.tie.item()) == 0
    # the source advanced exactly as the materialised take did
    assert torch.equal(a.take(2 * k * mv + 17), b.take(2 * k * mv + 17))


def _gaps_numpy(v: np.ndarray) -> np.ndarray:
    side = v > 0.5
    flips = np.flatnonzero(side[1:] != side[:-1]) + 1
    runs = np.diff(np.concatenate([[0], flips]))  # closed runs; the final open run is dropped
    return np.bincount(np.minimum(runs, 64) - 1, minlength=64)


@pytest.mark.parametrize("k,mv,sel,pre", CASES)
def test_fused_gaps_equal_numpy(k, mv, sel, pre):
    a, b = make(k, mv, sel), make(k, mv, sel)
    if pre:
        a.take(pre)
        b.take(pre)
    n = 9 * k * mv + 4321
    want = _gaps_numpy(b.take(n).cpu().numpy())
    assert stats._fused_plan(a, n) is not None
    rep = stats.gaps_test(a, n)
    # the statistic is a function of the counts: recompute it from the numpy counts
    runs = int(want.sum())
    law = np.ldexp(1.0, -np.arange(1, 65))
    law[-1] = np.ldexp(1.0, -63)
    ref = stats._against_law("gaps", {}, n, want, law * runs)
    assert rep.result == ref.result
    assert torch.equal(a.take(k * mv + 5), b.take(k * mv + 5))


def test_gaps_array_path_degenerate_runs():
    """The materialised gaps path across several sweeps, with long runs that
    span many tiles (a stream of constant stretches) and runs of length >= 64."""
    rng = np.random.default_rng(3)
    lengths = np.concatenate([rng.integers(1, 5, 3000), [700, 5000, 64, 65, 63, 1]])
    rng.shuffle(lengths)
    sides = np.arange(lengths.size) % 2
    v = np.repeat(np.where(sides == 1, 0.75, 0.25), lengths)

    class Src:
        def __init__(self):
            self.at = 0

        def take(self, n):
            out = v[self.at:self.at + n]
            self.at += n
            return out

    old = stats._CHUNK
    stats._CHUNK = 4096  # several sweeps
    try:
        rep = stats.gaps_test(Src(), v.size)
    finally:
        stats._CHUNK = old
    want = _gaps_numpy(v)
    runs = int(want.sum())
    law = np.ldexp(1.0, -np.arange(1, 65))
    law[-1] = np.ldexp(1.0, -63)
    assert rep.result == stats._against_law("gaps", {}, v.size, want, law * runs).result


def test_fourier_binning_kernel_equals_searchsorted():
    """rsa_battery_fourier_bin = numpy searchsorted(side='left') + bincount,
    including values exactly on an edge."""
    from paper_1811_11629_b200 import _device
    edges = stats._normal_edges()
    rng = np.random.default_rng(8)
    z = rng.normal(0, np.sqrt(1 / 12), size=(1 << 16, 2))
    z[:63, 0] = edges
    z[63:126, 1] = np.nextafter(edges, 1.0)
    dz = torch.as_tensor(z, device="cuda").contiguous()
    de = torch.as_tensor(edges, device="cuda")
    cells = torch.zeros(128, dtype=torch.int64, device="cuda")
    _lib.call("rsa_battery_fourier_bin", dz.data_ptr(), z.shape[0], de.data_ptr(), cells.data_ptr(),
              _device.stream(dz.device))
    want = np.concatenate([np.bincount(np.searchsorted(edges, z[:, 0]), minlength=64),
                           np.bincount(np.searchsorted(edges, z[:, 1]), minlength=64)])
    assert np.array_equal(cells.cpu().numpy(), want)


def test_fused_rejects_unsupported_layouts():
    """Stream counts that do not divide the CTA, or blocks that are not whole
    tiles, take the materialised path (fused_target None); the C ABI rejects
    them outright."""
    assert make(3, 256, "float_leading").fused_target() is None
    assert make(2, 100, "float_leading").fused_target() is None
    assert make(2, 256, "raw_word").fused_target() is None
    spec = _lib.BatterySpec(test=_lib.RSA_BT_SERIAL, d=2, p1=2, p2=1024, pos0=0, seg0=0)
    assert _lib.load().rsa_battery_fused(None, 3, 256, 1, 9, 1, None, None, None, spec, None, None, None, None,
                                         None) == _lib.RSA_EINVAL


@pytest.mark.parametrize("n", [1, 5, 8, 64, 127, 128, 129, 1000, 4095, 362880, 10 ** 6, 1 << 20, 3628800])
def test_device_chi2_sum_is_numpys(n):
    """rsa_battery_chi2_sum restates numpy's pairwise summation of
    np.square(counts - e): bit-identical for every tree shape."""
    rng = np.random.default_rng(n)
    counts = rng.poisson(95.4, n).astype(np.int64)
    e = 1e8 / n
    want = np.square(counts - e).sum()
    got = stats._chi2_sum_device(torch.as_tensor(counts, device="cuda"), e)
    assert got == float(want)


@pytest.mark.parametrize("variant,trials", [("top20bits", 64), ("msb_of_20", 64)])
@pytest.mark.parametrize("k,mv,sel,pre", CASES)
def test_fused_collisions_equal_materialised(variant, trials, k, mv, sel, pre):
    """Collision balls fed in registers (per-trial bitmaps in device memory,
    20-variate balls across tiles through the boundary slots) give the
    materialised path's exact per-trial collision histogram."""
    a, b = make(k, mv, sel), make(k, mv, sel)
    if pre:
        a.take(pre)
        b.take(pre)
    d = 20 if variant == "msb_of_20" else 1
    assert stats._fused_plan(a, trials * stats.COLLISION_BALLS * d) is not None
    ra = stats.collision_test(a, variant, trials)
    rb = stats.collision_test(Proxy(b), variant, trials)
    assert ra.result == rb.result and ra.samples == rb.samples
    assert torch.equal(a.take(3 * k * mv + 1), b.take(3 * k * mv + 1))
