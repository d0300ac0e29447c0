"""K2 fused consumer (config 4) against the numpy restatement of the A13
definitions applied to the C oracle's draws: histograms exact, moments
rel 1e-9, correlations abs 1e-11 (SURVEY.md §8(c) tolerances)."""

import numpy as np
import pytest
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import vecgen
from oracle import coracle
from oracle import rsa_oracle as O

pytestmark = pytest.mark.gpu

SEED = 0x243F6A8885A308D3


def oracle_draws(table, first, count, N):
    rec = table.records()
    out = np.empty((count, N), dtype=np.float64)
    one = lambda v: np.array([v], dtype=np.uint64)
    for j in range(count):
        r = rec[first + j]
        cp = coracle.params(int(r["p1"]), int(r["p2"]), int(r["e"]), int(r["a"]))
        _, f = coracle.fill(cp, one(0), one(0), one(1), N, raw=False)
        out[j] = f.reshape(-1)
    return out


@pytest.mark.parametrize("n_inst,N", [(256, 1 << 16), (34, 70001)])
def test_fused_matches_oracle(n_inst, N):
    t = R.derive_params_table(SEED, 0, n_inst)
    fc = R.FusedConsumer(t)
    res = fc.run(N)
    r = oracle_draws(t, 0, n_inst, N)
    ref = O.fused_reference(r)
    hist = res.hist.cpu().numpy().astype(np.int64)
    assert np.array_equal(hist, ref["hist"])
    assert np.array_equal(res.pooled_hist.cpu().numpy(), ref["pooled_hist"])
    m = {k: v.cpu().numpy() for k, v in res.moments().items()}
    np.testing.assert_allclose(m["mean"], ref["mean"], rtol=1e-9, atol=0)
    np.testing.assert_allclose(m["var"], ref["var"], rtol=1e-9, atol=0)
    np.testing.assert_allclose(m["lag1"], ref["lag1"], rtol=0, atol=1e-11)
    assert abs(res.pooled_correlation() - ref["corr"]) < 1e-11
    st = res.stats.cpu().numpy()
    assert np.array_equal(st[:, 3], r[:, 0]) and np.array_equal(st[:, 4], r[:, -1])


def test_fused_state_advances_like_fill():
    t = R.derive_params_table(SEED, 100, 8)
    fc = R.FusedConsumer(t)
    fc.run(1000)
    fc.run(24)
    # the same instances through the fill kernel, Mv = 1 each
    for j in range(8):
        st = R.init_vector(t.params(j), mv=1)
        R.take_raw(st, 1024)
        assert int(st.s[0].item()) == int(fc.s[j].item())
        assert int(st.m1[0].item()) == int(fc.m1[j].item())
        assert int(st.m2[0].item()) == int(fc.m2[j].item())


def test_fused_rejects_odd_count():
    t = R.derive_params_table(SEED, 0, 3)
    with pytest.raises(ValueError):
        R.FusedConsumer(t)
    with pytest.raises(ValueError):
        R.FusedConsumer(R.derive_params_table(SEED, 0, 2)).run(1)


def test_many_instance_fill_config3(golden_meta):
    """Config 3 layout: instance-major take_floats of Mv=64 streams via one
    multi-instance rsa_fill launch, against the reference digests."""
    ids = golden_meta["c3_ids"]
    lo = 0
    t = R.derive_params_table(SEED, lo, max(ids) + 1)
    from paper_1811_11629_b200 import _device, _lib
    d = t.device
    sel = torch.tensor(ids, device=d)
    inst = t.inst[sel].contiguous()
    n, mv, blocks = len(ids), 64, 1024
    m1, m2, s = vecgen._init_lanes(inst, n, mv, 0, 1, d)
    out = torch.empty((n, blocks * mv), dtype=torch.float64, device=d)
    _lib.call("rsa_fill", inst.data_ptr(), n, mv, blocks, 9, _lib.RSA_FLAG_FAST, m1.data_ptr(),
              m2.data_ptr(), s.data_ptr(), None, out.data_ptr(), blocks * mv, _device.stream(d))
    from conftest import sha
    for j, sid in enumerate(ids):
        assert sha(out[j].cpu().numpy().astype("<f8")) == golden_meta[f"c3_id{sid}_f64_sha256"], sid


def test_fused_stays_inside_its_buffers():
    """Guard bands around the per-instance statistics, histograms and lane
    state (compute-sanitizer is closed on this pool); an instance count that
    leaves idle lanes in the last CTA."""
    from paper_1811_11629_b200 import _device, _lib
    n, G = 130, 256
    t = R.derive_params_table(SEED, 7, n)
    fc = R.FusedConsumer(t)
    d = t.device
    stats = torch.full((n + 2 * G, 6), -3.0, dtype=torch.float64, device=d)
    hist = torch.full((n + 2 * G, 64), -5, dtype=torch.int32, device=d)
    _lib.call("rsa_fused_stats", t.inst.data_ptr(), n, 300, 9, fc.m1.data_ptr(), fc.m2.data_ptr(),
              fc.s.data_ptr(), stats[G:].data_ptr(), hist[G:].data_ptr(), _device.stream(d))
    torch.cuda.synchronize()
    assert bool((stats[:G] == -3.0).all()) and bool((stats[G + n:] == -3.0).all())
    assert bool((hist[:G] == -5).all()) and bool((hist[G + n:] == -5).all())
    assert bool((hist[G:G + n].sum(dim=1) == 300).all())
