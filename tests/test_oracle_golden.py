"""Pin the CPU oracles (oracle/) to the reference's own outputs.

The golden fixtures were produced by tests/golden/make_golden.py importing the
reference package; these tests prove the numpy and C restatements reproduce
them exactly before either is trusted as the checker of the CUDA path.
"""

import dataclasses

import numpy as np
import pytest

from conftest import sha
from oracle import coracle
from oracle import rsa_oracle as O


def test_scalar_regression(golden_regression, oracle_stream0):
    raws = O.scalar_raws(oracle_stream0, 16)
    assert raws == golden_regression["raw"]
    f = [min(c / oracle_stream0.n_float, O.MAX_BELOW_ONE) for c in raws]
    assert [x.hex() for x in f] == golden_regression["f64_hex"]
    # the acceptance suite's pinned 4-value vectors (test_acceptance.py:22-29)
    assert raws[:4] == [3198687466090183645, 1783912959308574348,
                        8527461190466845143, 7967842367115529255]


@pytest.mark.parametrize("mv", [1, 2, 8, 64])
def test_vector_streams(golden_vectors, oracle_stream0, mv):
    st = O.init(oracle_stream0, mv=mv)
    raw = O.take_raw(st, 4096)
    assert np.array_equal(raw, golden_vectors[f"c1_mv{mv}_raw"])
    assert np.array_equal(O.floats_from_raw(raw, oracle_stream0), golden_vectors[f"c1_mv{mv}_f64"])


def test_seeded_and_wide(golden_vectors, golden_meta, oracle_stream0):
    st = O.init(oracle_stream0, m0=golden_meta["seeded_m0"], mv=64)
    assert np.array_equal(O.take_raw(st, 4096), golden_vectors["c1_seeded_mv64_raw"])
    st = O.init(oracle_stream0, mv=65536)
    raw = O.take_raw(st, 2 * 65536)
    assert sha(raw.astype("<u8")) == golden_meta["c1_mv65536"]["raw_sha256"]
    assert sha(O.floats_from_raw(raw, oracle_stream0).astype("<f8")) == golden_meta["c1_mv65536"]["f64_sha256"]


def test_partial_takes(golden_vectors, golden_meta, oracle_stream0):
    st = O.init(oracle_stream0, mv=8)
    got = np.concatenate([O.take_raw(st, k) for k in golden_meta["take_parts_sizes"]])
    assert np.array_equal(got, golden_vectors["take_parts_mv8"])


@pytest.mark.parametrize("e", [3, 5, 9, 17, 257, 65537])
def test_exponent_lane_subsets(golden_vectors, golden_meta, oracle_stream0, e):
    P = dataclasses.replace(oracle_stream0, e=e)
    lanes = golden_vectors["c2_lanes"].tolist()
    st = O.init(P, m0=golden_meta["seeded_m0"], mv=golden_meta["c2"]["mv"], lanes=lanes)
    blocks = O.blocks_raw(st, 16)
    assert np.array_equal(blocks, golden_vectors[f"c2_e{e}_raw"])
    assert np.array_equal(O.floats_from_raw(blocks, P), golden_vectors[f"c2_e{e}_f64"])


def test_c_oracle_matches_numpy_lanes(golden_vectors, golden_meta, oracle_stream0):
    P = oracle_stream0
    lanes = golden_vectors["c2_lanes"].tolist()
    st = O.init(P, m0=golden_meta["seeded_m0"], mv=golden_meta["c2"]["mv"], lanes=lanes)
    for e in (3, 9, 65537):
        cp = coracle.params(P.p1, P.p2, e, P.a)
        m1, m2, s = st.m1.copy(), st.m2.copy(), st.s.copy()
        raw, f = coracle.fill(cp, m1, m2, s, 16)
        assert np.array_equal(raw, golden_vectors[f"c2_e{e}_raw"])
        assert np.array_equal(f, golden_vectors[f"c2_e{e}_f64"])


def test_many_instances(golden_streams, golden_vectors, golden_meta):
    for sid in golden_meta["c3_ids"]:
        P = O.from_fields(golden_streams["streams"][str(sid)])
        st = O.init(P, mv=64)
        f = O.take_floats(st, 1 << 16)
        assert sha(f.astype("<f8")) == golden_meta[f"c3_id{sid}_f64_sha256"], sid


def test_scalar_streams_c(golden_streams, golden_vectors, golden_meta, oracle_stream0):
    P = oracle_stream0
    one = lambda v: np.array([v], dtype=np.uint64)
    raw, _ = coracle.fill(coracle.params(P.p1, P.p2, P.e, P.a), one(0), one(0), one(1), 1 << 16, f64=False)
    assert sha(raw.reshape(-1).astype("<u8")) == golden_meta["c1_scalar_65536_raw_sha256"]
    for sid in golden_meta["c4_ids"]:
        Q = O.from_fields(golden_streams["streams"][str(sid)])
        raw, f = coracle.fill(coracle.params(Q.p1, Q.p2, Q.e, Q.a), one(0), one(0), one(1), 1 << 16)
        assert sha(raw.reshape(-1).astype("<u8")) == golden_meta[f"c4_id{sid}_raw_sha256"]
        assert np.array_equal(f.reshape(-1), golden_vectors[f"c4_id{sid}_f64"])


def test_miniature_and_counter_modes(golden_vectors, golden_meta, oracle_stream0):
    mini = O.from_fields(golden_meta["miniature"])
    assert O.scalar_raws(mini, 3036 * 2) == golden_vectors["mini_scalar_raw"].tolist()
    # full period: each ciphertext exactly q-1 = 12 times (test_acceptance.py:45-61)
    counts = np.bincount(golden_vectors["mini_scalar_raw"][:3036].astype(np.int64), minlength=253)
    assert (counts == 12).all()
    st = O.init(mini, mv=3)
    assert np.array_equal(O.take_raw(st, 3036 * 3), golden_vectors["mini_mv3_raw"])
    assert O.init(mini, mv=4).s.tolist() == golden_vectors["mini_mv4_seeds"].tolist() == [1, 8, 12, 5]
    tiny = O.from_fields(golden_meta["tiny"])
    assert O.scalar_raws(tiny, 200) == golden_vectors["tiny_unit_raw"].tolist()
    P = oracle_stream0
    unit = dataclasses.replace(P, mode="unit")
    for mv in (1, 3, 8):
        st = O.init(unit, m0=5, mv=mv)
        assert np.array_equal(O.take_raw(st, 64), golden_vectors[f"unit_m05_mv{mv}_raw"])
    const = dataclasses.replace(P, mode="const", skip_const=golden_meta["const_skip"])
    st = O.init(const, mv=7)
    assert np.array_equal(O.take_raw(st, 50), golden_vectors["const_mv7_raw"])


def test_clamp_and_lane_seeds(golden_vectors, oracle_stream0):
    P = oracle_stream0
    f = O.floats_from_raw(golden_vectors["clamp_raw"], P)
    assert np.array_equal(f, golden_vectors["clamp_f64"])
    assert f[1] == O.MAX_BELOW_ONE
    assert np.array_equal(O.lane_seeds(P, 1, 64), golden_vectors["lane_seeds_mv64"])
    assert np.array_equal(O.lane_seeds(P, 777, 64), golden_vectors["lane_seeds_mv64_s0_777"])


def test_stream_indices(golden_streams):
    for sid, (ordinal, ai) in golden_streams["stream_indices"].items():
        assert O.stream_indices(golden_streams["master_seed"], int(sid)) == (ordinal, ai)


def test_census_c(golden_census, census_c):
    sp, nprimes = census_c
    assert nprimes == golden_census["primes"] == 98_182_656
    assert len(sp) == golden_census["safe_primes"] == 3_060_794
    assert sha(sp.astype("<u4")) == golden_census["sha256_u32le"]
    assert sp[:64].tolist() == golden_census["head"]
    lo, hi = golden_census["p1_window"]
    assert int(((sp >= lo) & (sp < hi)).sum()) == golden_census["p1_window_count"] == 1_291_847


def test_census_small_windows():
    # safe_primes_in(2, 5000) equals the predicate (test_paramfactory.py:15-19)
    sp, _ = coracle.census(11, 5000)
    want = [p for p in range(11, 5000) if O.is_safe_prime(p)]
    assert sp.tolist() == want
    lo = (1 << 31) + 1
    sp, _ = coracle.census(lo, lo + 100_000)
    assert sp.tolist() == [p for p in range(lo, lo + 100_000) if O.is_safe_prime(p)]
    assert sp[0] == 2147483783


def test_find_pair_and_streams(golden_streams, census_c):
    sp, _ = census_c
    assert O.find_pair_sorted(3037000943, sp) == golden_streams["find_pair_anchor"][1]
    assert O.find_pair_sorted(2147483783, sp) == golden_streams["find_pair_first"][1]
    for sid in list(range(64)) + [61644, 63194, 65535, (1 << 20) - 1]:
        row = golden_streams["streams"][str(sid)]
        p1, p2, a, _ = O.derive(golden_streams["master_seed"], sid, sp, 0)
        assert (p1, p2, a) == (row["p1"], row["p2"], row["a"]), sid


def test_derive_all_c(golden_derive_all, golden_streams, census_c):
    sp, _ = census_c
    n = golden_derive_all["ids"]
    rows, steps = coracle.derive(golden_streams["master_seed"], 0, n, sp, O.MULTIPLIER_TABLE)
    assert sha(rows[:65536]) == golden_derive_all["sha256_first_65536"]
    assert sha(rows) == golden_derive_all["sha256"]
    adv = {str(i): int(steps[i]) for i in np.nonzero(steps)[0]}
    assert adv == golden_derive_all["advanced_ids"]
    assert len(set(zip(rows["p1"].tolist(), rows["p2"].tolist()))) == golden_derive_all["distinct_pairs"]


def test_fused_reference_definitions():
    # the A13 estimators on a stream with a known answer: r_k = k/N
    N = 1024
    r = np.tile(np.arange(N, dtype=np.float64) / N, (2, 1))
    out = O.fused_reference(r)
    assert np.allclose(out["mean"], (N - 1) / (2 * N))
    assert out["hist"].sum() == 2 * N and (out["hist"] == N // 64).all()
    assert abs(out["corr"] - 1.0) < 1e-12
