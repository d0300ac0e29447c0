"""K3 safe-prime scan and K4 instance setup on the B200 against the
reference's census / derivation fixtures and the C oracle (config 5)."""

import numpy as np
import pytest
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import _lib, paramfactory, rsacore, skipgen
from conftest import sha
from oracle import coracle
from oracle import rsa_oracle as O

pytestmark = pytest.mark.gpu


def test_full_census(golden_census):
    sp = paramfactory.safe_primes_u32(1 << 31, 1 << 32).cpu().numpy().view(np.uint32)
    assert len(sp) == golden_census["safe_primes"] == 3_060_794
    assert sha(sp.astype("<u4")) == golden_census["sha256_u32le"]
    tab = paramfactory.safe_prime_table()
    assert tab.n_sp == 3_060_794 and tab.n_p1 == golden_census["p1_window_count"]


@pytest.mark.parametrize("lo,hi", [(2, 5000), (0, 12), (5, 8), (11, 12), ((1 << 31) + 1, (1 << 31) + 100_001),
                                   ((1 << 32) - 1_000_000, 1 << 32), (3037000000, 3037100000),
                                   (1_000_000, 1_200_000), (10_000, 400_000), (10_190, 10_230),
                                   ((1 << 31) - 5, (1 << 31) + 5), (3_000_000_011, 3_000_000_012)])
def test_scan_windows(lo, hi):
    got = R.safe_primes_in(lo, hi).cpu().numpy().tolist()
    want = [p for p in range(max(lo, 2), min(hi, 11)) if O.is_safe_prime(p)]
    if hi > 11:
        sp, _ = coracle.census(max(lo, 11), hi)
        want += sp.tolist()
    assert got == want


def test_literal_mr_census(golden_census):
    """BASELINE config 5 verbatim: MR (2, 7, 61) on every odd n in
    [2^31, 2^32) and on (n-1)/2 gives the reference's census exactly."""
    sp = paramfactory.safe_primes_u32(1 << 31, 1 << 32, literal_mr=True).cpu().numpy().view(np.uint32)
    assert len(sp) == golden_census["safe_primes"]
    assert sha(sp.astype("<u4")) == golden_census["sha256_u32le"]


@pytest.mark.parametrize("lo,hi", [(2, 5000), (0, 12), (5, 8), (10_190, 10_230), (10_000, 400_000),
                                   ((1 << 31) - 5, (1 << 31) + 5), ((1 << 32) - 1_000_000, 1 << 32),
                                   (3037000000, 3037100000)])
def test_literal_mr_windows(lo, hi):
    a = paramfactory.safe_primes_u32(lo, hi, literal_mr=True).cpu().numpy().tolist()
    b = paramfactory.safe_primes_u32(lo, hi).cpu().numpy().tolist() if hi > max(lo, 2) else []
    assert a == b
    want = [p for p in range(max(lo, 2), min(hi, 11)) if O.is_safe_prime(p)]
    if hi > 11:
        sp, _ = coracle.census(max(lo, 11), hi)
        want += sp.tolist()
    assert a == want


def test_literal_mr_pseudoprime_neighbourhoods():
    """Base-2 strong pseudoprimes (and their safe-prime partners) decided by
    bases 7 / 61 in the literal scan, equal to the table-based scan."""
    from test_spsp2_table import load_table
    _, _, vals = load_table()
    for t in vals[::23]:
        lo, hi = max(11, t - 300), min(1 << 32, t + 300)
        assert paramfactory.safe_primes_u32(lo, hi, literal_mr=True).cpu().numpy().tolist() == \
            paramfactory.safe_primes_u32(lo, hi).cpu().numpy().tolist(), t


def test_scan_pseudoprime_neighbourhoods():
    """Every candidate whose verdict the base-2 pseudoprime table decides (p or
    (p-1)/2 is a base-2 strong pseudoprime and the other half passes base 2)
    is scanned in a small window and compared with the C oracle."""
    from test_spsp2_table import load_table, sprp2
    _, _, vals = load_table()
    decided = []
    for t in vals:
        if t % 12 == 11 and sprp2((t - 1) // 2):
            decided.append(t)
        if t % 6 == 5 and 2 * t + 1 < 1 << 32 and sprp2(2 * t + 1):
            decided.append(2 * t + 1)
    assert len(decided) == 55
    for p in decided:
        lo, hi = max(11, p - 600), min(1 << 32, p + 600)
        got = R.safe_primes_in(lo, hi).cpu().numpy().tolist()
        want, _ = coracle.census(lo, hi)
        assert got == want.tolist(), p
        assert p not in got


def test_segment_stitching():
    a = R.safe_primes_in(2_000_000, 2_500_000).cpu().numpy()
    b = R.safe_primes_in(2_500_000, 3_000_000).cpu().numpy()
    assert np.concatenate([a, b]).tolist() == R.safe_primes_in(2_000_000, 3_000_000).cpu().numpy().tolist()


def test_nth_safe_prime():
    assert R.nth_safe_prime_in(11, 100, 0) == 11
    assert R.nth_safe_prime_in(11, 100, 1) == 23
    assert R.nth_safe_prime_in(5, 100, 1) == 7
    with pytest.raises(R.NotFound):
        R.nth_safe_prime_in(11, 100, 8)
    with pytest.raises(ValueError):
        R.nth_safe_prime_in(100, 100, 0)


def test_batched_predicates():
    rng = np.random.default_rng(3)
    n = np.concatenate([np.arange(0, 20000, dtype=np.uint32),
                        rng.integers(1 << 31, 1 << 32, size=200_000, dtype=np.uint64).astype(np.uint32),
                        np.array([2147483783, 3037000943, 4294967087, 4294967291], dtype=np.uint32)])
    t = torch.from_numpy(n.view(np.int32)).cuda()
    isp = torch.empty(len(n), dtype=torch.uint8, device="cuda")
    iss = torch.empty(len(n), dtype=torch.uint8, device="cuda")
    _lib.call("rsa_is_safe_prime32", t.data_ptr(), len(n), isp.data_ptr(), iss.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    isp, iss = isp.cpu().numpy().astype(bool), iss.cpu().numpy().astype(bool)
    sample = list(range(0, len(n), 7))
    assert [bool(isp[i]) for i in sample] == [O.is_prime(int(n[i])) for i in sample]
    assert [bool(iss[i]) for i in sample] == [O.is_safe_prime(int(n[i])) for i in sample]
    assert iss[-4:].tolist() == [True, True, True, False]


def test_find_pair(golden_streams):
    assert list(R.find_pair(3037000943)) == golden_streams["find_pair_anchor"]
    assert list(R.find_pair(2147483783)) == golden_streams["find_pair_first"]
    with pytest.raises(R.NotFound):
        R.find_pair(2147483783, tol=0.0)
    with pytest.raises(ValueError):
        R.find_pair((1 << 31) + 1)


def test_derive_stream_params_matches_reference(golden_streams):
    seed = golden_streams["master_seed"]
    for sid in [0, 1, 2, 3, 7, 100, 511, 61644, 63194, 65535, (1 << 20) - 1]:
        p = R.derive_stream_params(R.StreamKey(seed, sid))
        g = golden_streams["streams"][str(sid)]
        assert (p.p1, p.p2, p.n, p.e, p.skip.a, p.p2inv, p.b) == \
            (g["p1"], g["p2"], g["n"], g["e"], g["a"], g["p2inv"], g["b"]), sid
    ex = golden_streams["extra"]
    p = R.derive_stream_params(R.StreamKey(7, 8), e=17)
    assert (p.p1, p.p2, p.e) == (ex["e17_id7_seed7"]["p1"], ex["e17_id7_seed7"]["p2"], 17)
    p = R.derive_stream_params(R.StreamKey(0xBEEF, 3))
    assert (p.p1, p.p2, p.skip.a) == (ex["seed_beef_id3"]["p1"], ex["seed_beef_id3"]["p2"], ex["seed_beef_id3"]["a"])
    p = R.derive_stream_params(R.StreamKey(1, 2), multiplier=skipgen.MULTIPLIER_TABLE[5])
    assert (p.p1, p.p2, p.skip.a) == (ex["mult5_seed1_id2"]["p1"], ex["mult5_seed1_id2"]["p2"],
                                      skipgen.MULTIPLIER_TABLE[5])
    p = R.derive_stream_params(R.StreamKey((1 << 64) - 3, 5))
    assert (p.p1, p.p2) == (ex["seed_big_id5"]["p1"], ex["seed_big_id5"]["p2"])
    with pytest.raises(ValueError):
        R.derive_stream_params(R.StreamKey(1, 2), multiplier_table=())
    with pytest.raises(R.DerivationExhausted):
        R.derive_stream_params(R.StreamKey(1, 2), e=4)


def test_derive_negative_keys_like_reference():
    """Negative stream ids / master seeds reduce mod S exactly as the
    reference's Python % does (paramfactory.py:249); values computed with the
    reference in the build container."""
    want = {(R.DEFAULT_MASTER_SEED, -5): (2669237027, 3455433887, 3003776879),
            (-12345, 77): (2975481599, 3099791447, 3027930091),
            (-1, -1): (2229924539, 4136181143, 2966714411)}
    for (seed, sid), (p1, p2, a) in want.items():
        p = R.derive_stream_params(R.StreamKey(seed, sid))
        assert (p.p1, p.p2, p.skip.a) == (p1, p2, a), (seed, sid)


def test_derive_all_2e20(golden_derive_all, golden_streams):
    """Config 5: 2^20 instance tuples built on the device, packed like the
    golden digest (computed by the reference), plus device-only constants
    checked by identity."""
    n = golden_derive_all["ids"]
    t = R.derive_params_table(golden_streams["master_seed"], 0, n)
    rec = t.records()
    rows = np.zeros(n, dtype=coracle.TUPLE_DTYPE)
    for f in ("p1", "p2", "a", "p2inv", "n", "b"):
        rows[f] = rec[f]
    assert sha(rows[:65536]) == golden_derive_all["sha256_first_65536"]
    assert sha(rows) == golden_derive_all["sha256"]
    steps = t.steps.cpu().numpy()
    assert {str(i): int(steps[i]) for i in np.nonzero(steps)[0]} == golden_derive_all["advanced_ids"]
    R32 = np.uint64(1 << 32)
    p1 = rec["p1"].astype(np.uint64)
    assert ((p1 * rec["p1_inv"].astype(np.uint64)) % R32 == 1).all()
    assert (rec["n_float"] == rec["n"].astype(np.float64)).all()
    assert (rec["n_recip"] == 1.0 / rec["n_float"]).all()
    assert (rec["flags"] == _lib.RSA_FLAG_FAST).all()
    # a sample against the host packer
    for j in (0, 1, 61644, 1000, n - 1):
        host = rsacore._instance_record(t.params(j))[0]
        for f in ("k1", "k2", "r2_1", "r2_2", "garner", "q1", "q2", "p2_inv"):
            assert host[f] == rec[j][f], (j, f)


def test_table_e_and_errors(golden_streams):
    t = R.derive_params_table(golden_streams["master_seed"], 0, 64, e=17)
    assert (t.records()["e"] == 17).all()
    with pytest.raises(R.DerivationExhausted):
        R.derive_params_table(0, 0, 4, e=259)


def test_safe_prime_index_and_unindexed_search(golden_streams):
    """The bucket index matches searchsorted, and the indexed search returns
    byte-identical instances / pairs to the plain binary search (NULL index)."""
    tab = paramfactory.safe_prime_table()
    keys = torch.arange(paramfactory.SP_INDEX_LEN, dtype=torch.int64, device=tab.sp.device) << paramfactory.SP_INDEX_SHIFT
    want = torch.searchsorted(tab.sp.to(torch.int64), keys)
    assert torch.equal(tab.index.to(torch.int64), want)
    n = 1 << 16
    cfg = paramfactory._setup_config(golden_streams["master_seed"], 12345, 9,
                                     len(paramfactory.MULTIPLIER_TABLE), 0)
    mult = tab.mult_table(tuple(paramfactory.MULTIPLIER_TABLE))
    outs = []
    for idx in (tab.index.data_ptr(), None):
        inst = torch.empty((n, 128), dtype=torch.uint8, device=tab.sp.device)
        st = torch.empty(n, dtype=torch.int32, device=tab.sp.device)
        steps = torch.empty(n, dtype=torch.int32, device=tab.sp.device)
        _lib.call("rsa_setup_instances", cfg, n, mult.data_ptr(), tab.sp.data_ptr(), tab.n_sp, idx,
                  tab.sp.data_ptr(), tab.n_p1, inst.data_ptr(), st.data_ptr(), steps.data_ptr(), None)
        outs.append((inst.cpu(), st.cpu(), steps.cpu()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    p1 = tab.sp[:: max(1, tab.n_p1 // 4096)][:4096].contiguous()
    res = []
    for idx in (tab.index.data_ptr(), None):
        p2 = torch.zeros(p1.numel(), dtype=torch.int32, device=p1.device)
        st = torch.zeros(p1.numel(), dtype=torch.int32, device=p1.device)
        _lib.call("rsa_find_pair", p1.data_ptr(), p1.numel(), paramfactory.Q_DEFAULT,
                  paramfactory.tolerance_int(paramfactory.DEFAULT_TOLERANCE, paramfactory.Q_DEFAULT),
                  tab.sp.data_ptr(), tab.n_sp, idx, p2.data_ptr(), st.data_ptr(), None)
        res.append((p2.cpu(), st.cpu()))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
    assert (res[0][1] == 0).sum() > 0


@pytest.mark.parametrize("n_a", [len(paramfactory.MULTIPLIER_TABLE), 494])
def test_stream_indices_both_index_space_paths(n_a, golden_streams):
    """S = K_P1*K_P2*n_a below 2^50 takes the FP64-quotient mulmod, above it
    the 128-bit path; both must reproduce the host's exact stream_indices."""
    table = tuple(paramfactory.MULTIPLIER_TABLE[i % len(paramfactory.MULTIPLIER_TABLE)] for i in range(n_a))
    assert (paramfactory._index_space(n_a) >= 1 << 50) == (n_a == 494)
    seed, first, n = golden_streams["master_seed"], (1 << 40) + 7, 512
    t = R.derive_params_table(seed, first, n, multiplier_table=table)
    rec = t.records()
    steps = t.steps.cpu().numpy()
    sp = paramfactory.safe_prime_table().sp.cpu().numpy().view(np.uint32)
    for j in range(n):
        ordinal, ai = paramfactory.stream_indices(paramfactory.StreamKey(seed, first + j), n_a)
        assert int(rec[j]["a"]) == table[ai]
        assert int(rec[j]["p1"]) == int(sp[(ordinal + int(steps[j])) % paramfactory.K_P1])


@pytest.mark.parametrize("fn", ["rsa_safe_prime_scan", "rsa_safe_prime_scan_mr"])
@pytest.mark.parametrize("lo,hi", [(2, 70_000), ((1 << 31) + 1, (1 << 31) + (1 << 26) + 7)])
def test_scans_stay_inside_their_buffers(fn, lo, hi):
    """Guard bands around scratch and output (no compute-sanitizer on this
    pool): each scan writes only its outputs and declared scratch."""
    from paper_1811_11629_b200 import _device
    L = _lib.load()
    d = torch.device("cuda")
    nb = int(getattr(L, fn + "_scratch_bytes")(lo, hi))
    G = 4096
    sc = torch.full((nb + 2 * G,), 0x5A, dtype=torch.uint8, device=d)
    want, _ = coracle.census(max(lo, 11), hi)
    want = [p for p in range(max(lo, 2), min(hi, 11)) if O.is_safe_prime(p)] + want.tolist()
    cap = len(want)
    out = torch.full((cap + 2 * G,), 7, dtype=torch.int32, device=d)
    cnt = torch.zeros(1, dtype=torch.int64, device=d)
    rc = getattr(L, fn)(lo, hi, out[G:].data_ptr(), cap, cnt.data_ptr(), sc[G:].data_ptr(), nb, _device.stream(d))
    assert rc == 0
    torch.cuda.synchronize()
    assert int(cnt.item()) == cap
    assert out[G:G + cap].cpu().numpy().view(np.uint32).tolist() == want
    assert bool((out[:G] == 7).all()) and bool((out[G + cap:] == 7).all())
    assert bool((sc[:G] == 0x5A).all()) and bool((sc[G + nb:] == 0x5A).all())


def test_setup_writes_only_found_records():
    """k_setup stages records in shared memory and writes them as 16-byte
    words: records of ids it did not derive, and bytes past the table, stay
    untouched."""
    from paper_1811_11629_b200 import _device
    tab = paramfactory.safe_prime_table()
    d = tab.sp.device
    n = 1000
    cfg = paramfactory._setup_config(paramfactory.DEFAULT_MASTER_SEED, 61640, 9,
                                     len(paramfactory.MULTIPLIER_TABLE), 0)
    cfg.max_steps = 1  # ids whose first p1 has no partner stay NotFound (e.g. 61644)
    mult = tab.mult_table(tuple(paramfactory.MULTIPLIER_TABLE))
    G = 64
    inst = torch.full(((n + 2 * G), 128), 0xC3, dtype=torch.uint8, device=d)
    st = torch.empty(n, dtype=torch.int32, device=d)
    _lib.call("rsa_setup_instances", cfg, n, mult.data_ptr(), tab.sp.data_ptr(), tab.n_sp,
              tab.index.data_ptr(), tab.sp.data_ptr(), tab.n_p1, inst[G:].data_ptr(), st.data_ptr(), None,
              _device.stream(d))
    torch.cuda.synchronize()
    s = st.cpu().numpy()
    rec = inst[G:G + n].cpu().numpy()
    assert (s != 0).any() and (s == 0).any()
    assert (rec[s != 0] == 0xC3).all()
    assert not (rec[s == 0] == 0xC3).all(axis=1).any()
    assert bool((inst[:G] == 0xC3).all()) and bool((inst[G + n:] == 0xC3).all())
