"""Config 2 at its full BASELINE size, bit-exact: all 2^30 doubles of the
bench's fill (stream 0 of the default master seed, the bench's seeded m0,
Mv = 2^22, 256 blocks) for every bench exponent, compared with the numpy
oracle through a position-weighted checksum of the float64 bit patterns,
sum_i bits(r_i) * (2 i + 1) mod 2^64.  The oracle side runs the lane range in
one chunk per host core (lanes are independent, test_vecgen.py:156-171).
"""

import dataclasses
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import vecgen
from oracle import rsa_oracle as O

pytestmark = pytest.mark.gpu

MV, BLOCKS = 1 << 22, 256


def _oracle_chunk(args):
    """Checksum of lanes [lo, hi) over all blocks (numpy, wrapping uint64)."""
    P, m0, lo, hi = args
    st = O.init(P, m0=m0, mv=MV, lanes=range(lo, hi))
    w = np.arange(lo, hi, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    step = np.uint64(2 * MV)
    acc = np.uint64(0)
    with np.errstate(over="ignore"):
        for _ in range(BLOCKS):
            f = O.floats_from_raw(O.next_block_raw(st), P).view(np.uint64)
            acc += np.sum(f * w, dtype=np.uint64)
            w += step
    return int(acc)


def _device_checksum(out: torch.Tensor) -> int:
    acc = 0
    bits = out.view(torch.int64)
    chunk = 1 << 26
    for a in range(0, bits.numel(), chunk):
        idx = torch.arange(a, a + chunk, dtype=torch.int64, device=out.device)
        acc += int((bits[a:a + chunk] * (2 * idx + 1)).sum().item())
    return acc % (1 << 64)


# the oracle workers are forked after CUDA init; they only run numpy
@pytest.mark.filterwarnings("ignore:This process .* is multi-threaded:DeprecationWarning")
@pytest.mark.parametrize("e", [3, 5, 17, 65537])
def test_config2_full_fill_checksum(e):
    import bench
    base = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
    m0 = bench.seeded_m0(base.n)
    st0 = R.init_vector(base, m0=m0, mv=MV)
    pe = dataclasses.replace(base, e=e)
    st = vecgen.VectorState(params=pe, mv=MV, m1=st0.m1, m2=st0.m2, s=st0.s)
    out = R.take_floats(st, MV * BLOCKS)
    got = _device_checksum(out)
    del out
    P = O.Params(pe.p1, pe.p2, e, pe.skip.a)
    procs = max(1, min(32, os.cpu_count() or 1))
    edges = [MV * k // procs for k in range(procs + 1)]
    with mp.get_context("fork").Pool(procs) as pool:
        parts = pool.map(_oracle_chunk, [(P, m0, edges[k], edges[k + 1]) for k in range(procs)])
    assert got == sum(parts) % (1 << 64)


# ---------------------------------------------------------------------------
# configs 3 and 4 checked inside the bench's own full-size launches
# (bench_configs.Config3 / Config4 are the objects bench.py times)

def _c3_oracle_row(rec):
    """One config-3 instance from the C oracle: Mv = 64 lanes seeded like
    init_vector(m0=0, s0=1) (vecgen.py:44-69), 1024 blocks -> (f64 row, state)."""
    from oracle import coracle
    P = O.Params(int(rec["p1"]), int(rec["p2"]), 9, int(rec["a"]))
    s = O.lane_seeds(P, 1, 64)
    m1 = np.zeros(64, dtype=np.uint64)
    m2 = np.zeros(64, dtype=np.uint64)
    _, f = coracle.fill(coracle.params(P.p1, P.p2, 9, P.a), m1, m2, s, 1024, raw=False)
    return f.reshape(-1), (m1, m2, s)


def test_config3_bench_launch_parity(golden_meta):
    """BASELINE config 3 exactly as bench.py times it: ids 0..65535, Mv 64,
    1024 blocks, ONE rsa_fill launch into the 32 GiB instance-major output.
    256 random instances + the reference-digest ids: full 2^16-double rows and
    the final lane state bit-exact against the C oracle, and the reference's
    own sha256 digests of those rows (vectors.json c3_id*_f64_sha256)."""
    import bench_configs as C
    from conftest import sha
    w = C.Config3(torch.device("cuda", 0))
    assert w.n == 1 << 16 and w.numbers_per_step == 1 << 32
    w.step()
    torch.cuda.synchronize()
    rng = np.random.default_rng(0xC3C3)
    pick = sorted(set(rng.choice(w.n, 256, replace=False).tolist()) | set(golden_meta["c3_ids"]))
    idx = torch.tensor(pick, device=w.out.device)
    rows = w.out.index_select(0, idx).cpu().numpy()
    lanes = (idx[:, None] * 64 + torch.arange(64, device=idx.device)).reshape(-1)
    st = [t.index_select(0, lanes).cpu().numpy().reshape(len(pick), 64) for t in (w.m1, w.m2, w.s)]
    del w
    torch.cuda.empty_cache()
    rec = R.derive_params_table(R.DEFAULT_MASTER_SEED, 0, 1 << 16).records()
    for j, i in enumerate(pick):
        f, (m1, m2, s) = _c3_oracle_row(rec[i])
        assert np.array_equal(rows[j], f), f"config-3 instance {i}: f64 row differs from the oracle"
        assert np.array_equal(st[0][j], m1) and np.array_equal(st[1][j], m2) and np.array_equal(st[2][j], s), i
    for sid in golden_meta["c3_ids"]:
        assert sha(rows[pick.index(sid)].astype("<f8")) == golden_meta[f"c3_id{sid}_f64_sha256"], sid


def test_config4_bench_launch_parity(golden_meta, golden_vectors):
    """BASELINE config 4 exactly as bench.py times it: 2^20 instances x 2^16
    draws in one k_fused launch (+ the pool kernels).  256 random instances
    (128 whole pairs) + the reference-digest ids: per-instance histograms
    exact, moments rel 1e-9, lag-1 and pair cross sums abs 1e-11 against the
    numpy A13 restatement on C-oracle draws (and, for the digest ids, on the
    reference's own draws, vectors.npz c4_id*_f64); the pooled outputs equal
    the per-instance sums of the same launch."""
    import bench_configs as C
    from oracle import coracle
    w = C.Config4(torch.device("cuda", 0))
    assert w.n == 1 << 20 and w.numbers_per_step == 1 << 36
    res = w.step()
    torch.cuda.synchronize()
    N = w.DRAWS
    rng = np.random.default_rng(0xC4C4)
    pairs = set(rng.choice(w.n // 2, 128, replace=False).tolist()) | {i // 2 for i in golden_meta["c4_ids"]}
    pick = sorted(2 * p + k for p in pairs for k in (0, 1))
    idx = torch.tensor(pick, device=res.stats.device)
    stats = res.stats.index_select(0, idx).cpu().numpy()
    hist = res.hist.index_select(0, idx).cpu().numpy().astype(np.int64)
    mom = {k: v.index_select(0, idx).cpu().numpy() for k, v in res.moments().items()}
    rec = w.table.records()
    one = lambda v: np.array([v], dtype=np.uint64)
    draws = np.empty((len(pick), N))
    for j, i in enumerate(pick):
        r = rec[i]
        _, f = coracle.fill(coracle.params(int(r["p1"]), int(r["p2"]), 9, int(r["a"])), one(0), one(0), one(1),
                            N, raw=False)
        draws[j] = f.reshape(-1)
    for sid in golden_meta["c4_ids"]:  # the oracle draws ARE the reference's on these ids
        assert np.array_equal(draws[pick.index(sid)], golden_vectors[f"c4_id{sid}_f64"]), sid
    ref = O.fused_reference(draws)
    assert np.array_equal(hist, ref["hist"])
    np.testing.assert_allclose(mom["mean"], ref["mean"], rtol=1e-9, atol=0)
    np.testing.assert_allclose(mom["var"], ref["var"], rtol=1e-9, atol=0)
    np.testing.assert_allclose(mom["lag1"], ref["lag1"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(stats[0::2, 5], ref["xy_even"], rtol=1e-9, atol=0)
    assert np.array_equal(stats[:, 3], draws[:, 0]) and np.array_equal(stats[:, 4], draws[:, -1])
    # pooled outputs of the same launch = sums of its per-instance rows
    allst = res.stats
    assert torch.equal(res.pooled_hist, res.hist.to(torch.int64).sum(dim=0))
    assert int(res.pooled_hist.sum().item()) == w.n * N
    want = [allst[:, 0].sum(), allst[:, 1].sum(), allst[0::2, 5].sum(), allst[0::2, 0].sum(),
            allst[1::2, 0].sum(), allst[0::2, 1].sum(), allst[1::2, 1].sum()]
    got = res.pooled.cpu().numpy()
    np.testing.assert_allclose(got, [float(x) for x in want], rtol=1e-12, atol=0)
    assert abs(res.pooled_correlation()) < 1e-4  # 2^35 pairs of independent streams: sd ~ 5e-6
