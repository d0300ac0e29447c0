"""F1 chi-square battery on the GPU against the reference's own
stats.run_battery output on the same interleaved streams
(tests/golden/battery.json, produced by running the reference)."""

import json
import math
import os

import numpy as np
import pytest

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    return json.load(open(os.path.join(HERE, "golden", "battery.json")))


def test_battery_matches_reference():
    g = _golden()
    plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, g["streams"][0], len(g["streams"]))

    def make(sel):
        return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=g["lanes"]) for p in plist], sel)

    rep = stats.run_battery(make, budget=g["budget"])
    got = {r.name: r.record() for r in rep.reports}
    assert [list(e) for e in rep.errors] == [list(e) for e in g["errors"]]
    assert list(got) == [r["name"] for r in g["reports"]]
    for want in g["reports"]:
        r = got[want["name"]]
        assert (r["samples"], r["dof"], r["params"]) == (want["samples"], want["dof"], want["params"]), want["name"]
        # every statistic and p-value bit-equal, Fourier included: on these
        # variates cuFFT and pocketfft agree to 1.3e-15 and no coefficient
        # changes cell (test_fourier_cells_vs_pocketfft bounds the general case)
        assert r["statistic"] == want["statistic"], want["name"]
        assert r["p"] == want["p"], want["name"]


def test_degenerate_sources_fail_and_floors():
    class Const:
        def take(self, n):
            return np.full(n, 0.25)

    assert not stats.freq_test(Const(), 1 << 20).pass_1e6
    with pytest.raises(stats.InsufficientSamples):
        stats.freq_test(Const(), 1000)
    with pytest.raises(stats.TieDetected):
        stats.permutation_test(Const(), 3, 1000)
    with pytest.raises(ValueError):
        stats.serial_test(Const(), 7, 1 << 22)
    # perfectly uniform counter sweep scores chi2 = 0 (stats test_freq, test_serial)
    sweep = (np.arange(1 << 20) + 0.5) / (1 << 20)

    class Sweep:
        def take(self, n):
            return sweep[:n]

    r = stats.freq_test(Sweep(), 1 << 20)
    assert r.result.statistic == 0.0 and r.result.p_value == 1.0


def test_poker_and_collision_tables():
    assert abs(stats.poker_probabilities().sum() - 1.0) < 1e-15
    d = stats.collision_distribution(4, 8)
    assert abs(d.sum() - 1.0) < 1e-12


def test_weakened_modes():
    """Reference acceptance c11 (test_acceptance.py:234-253): the unit skip with
    e=9 passes the battery at budget 1e7; the identity cipher (e=1, test mode)
    on a counter fails frequency / serial_d2 / max_of_t."""
    from paper_1811_11629_b200 import rsacore
    p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))

    def factory(params):
        return lambda sel: bitsource.BitSource([R.init_vector(params, m0=0, s0=1, mv=65536)], sel)

    unit9 = rsacore.make_params(p.p1, p.p2, 9, p.skip, skip_mode=rsacore.SKIP_UNIT)
    rep = stats.run_battery(factory(unit9), budget=10_000_000)
    assert not rep.errors, rep.errors
    assert [r.name for r in rep.reports if not r.pass_1e6] == []
    unit1 = rsacore.make_params(p.p1, p.p2, 1, p.skip, skip_mode=rsacore.SKIP_UNIT, test_mode=True)
    weak = stats.run_battery(factory(unit1), budget=10_000_000, tests=["frequency", "serial_d2", "max_of_t"])
    assert not weak.all_pass


def test_calibration_sources():
    """stats.UniformSource passes, stats.ArraySource of a constant fails
    (the reference's calibration helpers, stats.py:138-160)."""
    assert stats.freq_test(stats.UniformSource(9), 1 << 21).pass_1e6
    assert not stats.freq_test(stats.ArraySource([0.25]), 1 << 21).pass_1e6
    src = stats.ArraySource([0.1, 0.2, 0.3])
    assert src.take(4).tolist() == [0.1, 0.2, 0.3, 0.1] and src.take(2).tolist() == [0.2, 0.3]


def test_fourier_cells_vs_pocketfft():
    """The Fourier test against the reference's own computation on the same
    variates (numpy's pocketfft + searchsorted, stats.py:440-465): cuFFT and
    pocketfft coefficients agree to < 1e-12; every coefficient the two bin
    differently lies within that distance of a cell edge; the device cells
    equal a host bincount of the device coefficients (the binning kernel);
    and the statistic formed from the pocketfft cells equals the reference's
    golden value exactly."""
    import torch
    g = _golden()
    plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, g["streams"][0], len(g["streams"]))

    def make():
        return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=g["lanes"]) for p in plist], "float_leading")

    m = stats.FOURIER_M
    blocks = g["budget"] // (2 * m)
    cells = stats._fourier_cells(make(), blocks, m).cpu().numpy()
    zt = make().take(blocks * 2 * m).view(blocks, 2 * m)
    cg = (torch.fft.fft(torch.complex(zt[:, 0::2] - 0.5, zt[:, 1::2] - 0.5), dim=-1) / math.sqrt(m)).cpu().numpy()
    z = zt.cpu().numpy()
    cn = np.fft.fft((z[:, 0::2] - 0.5) + 1j * (z[:, 1::2] - 0.5), axis=-1) / math.sqrt(m)
    diff = float(np.abs(cg - cn).max())
    assert diff < 1e-12, diff
    edges = stats._normal_edges()
    moved = 0
    for a, b in ((cg.real, cn.real), (cg.imag, cn.imag)):
        a, b = a.reshape(-1), b.reshape(-1)
        ia, ib = np.searchsorted(edges, a), np.searchsorted(edges, b)
        bad = np.flatnonzero(ia != ib)
        moved += bad.size
        for k in bad:  # a coefficient that changed cells sits within the transform error of an edge
            assert np.min(np.abs(edges - b[k])) <= diff
    gpu_bins = np.concatenate([np.bincount(np.searchsorted(edges, x.reshape(-1)), minlength=64)
                               for x in (cg.real, cg.imag)])
    assert np.array_equal(cells, gpu_bins)
    host = np.concatenate([np.bincount(np.searchsorted(edges, x.reshape(-1)), minlength=64)
                           for x in (cn.real, cn.imag)])
    assert int(np.abs(cells - host).sum()) <= 2 * moved
    used = blocks * 2 * m
    e = used / 128
    want = next(r for r in g["reports"] if r["name"] == "fourier")
    assert float(np.square(host - e).sum() / e) == want["statistic"]
