"""Host-side logic of the drop-in API (no GPU): parameter construction and
validation, seeds, snapshot text, instance packing, derivation constants.
Mirrors the reference's host-only tests (test_rsacore.py:17-86,
test_paramfactory.py, test_skipgen.py)."""

import dataclasses

import numpy as np
import pytest

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import _lib, paramfactory, rsacore, skipgen
from paper_1811_11629_b200.rsacore import InvalidParams, InvalidSeed, MalformedSnapshot
from paper_1811_11629_b200.shard import shard_range


def q13():
    return skipgen.SkipParams.create(2, q=13, allow_weak=True)


def mini():
    return rsacore.make_params(11, 23, e=3, skip=q13(), test_mode=True)


def tiny():
    return rsacore.make_params(7, 11, e=3, skip=q13(), skip_mode=rsacore.SKIP_UNIT, test_mode=True)


def prod(golden_regression):
    g = golden_regression["params"]
    skip = skipgen.SkipParams.create(g["a"])
    return rsacore.make_params(g["p1"], g["p2"], g["e"], skip)


def test_constants_equal_reference(golden_streams):
    assert skipgen.Q_DEFAULT == (1 << 63) - 25
    # the table order is pinned by the reference's (ordinal, multiplier index) picks
    for sid, (_, ai) in golden_streams["stream_indices"].items():
        assert skipgen.MULTIPLIER_TABLE[ai] == golden_streams["streams"][sid]["a"]
    assert paramfactory.tolerance_int(1e-6, skipgen.Q_DEFAULT) == 9223372036854
    assert paramfactory._index_space(16) == 1_291_831 * 1_768_937 * 16


def test_stream_indices_match_golden(golden_streams):
    for sid, want in golden_streams["stream_indices"].items():
        key = R.StreamKey(golden_streams["master_seed"], int(sid))
        assert list(paramfactory.stream_indices(key)) == want


def test_make_params_errors():
    with pytest.raises(InvalidParams, match="odd"):
        rsacore.make_params(7, 11, e=2, skip=q13(), skip_mode=rsacore.SKIP_UNIT, test_mode=True)
    with pytest.raises(InvalidParams, match="p1 == p2"):
        rsacore.make_params(11, 11, e=3, skip=q13(), test_mode=True)
    with pytest.raises(InvalidParams, match="safe prime"):
        rsacore.make_params(13, 23, e=3, skip=q13(), test_mode=True)
    with pytest.raises(InvalidParams, match="outside"):
        rsacore.make_params(11, 47, e=3, skip=skipgen.default_skip_params())


def test_production_params(golden_regression):
    p = prod(golden_regression)
    g = golden_regression["params"]
    assert (p.n, p.p2inv, p.b, p.skip.q1, p.skip.q2) == (g["n"], g["p2inv"], g["b"], g["q1"], g["q2"])
    assert p.n_float.hex() == g["n_float_hex"]
    assert mini().b == 78
    assert tiny().p2inv == 2


def test_init_semantics():
    st = rsacore.init(mini())
    assert (st.m1, st.m2, st.s, st.draws) == (0, 0, 1, 0)
    assert (rsacore.init(tiny(), m0=38).m1, rsacore.init(tiny(), m0=38).m2) == (3, 5)
    with pytest.raises(InvalidSeed):
        rsacore.init(mini(), s0=13)
    with pytest.raises(InvalidSeed):
        rsacore.init(mini(), m0=-1)


def test_vector_init_argument_errors(golden_regression):
    p = prod(golden_regression)
    # raised before any device work, so they hold without a GPU
    with pytest.raises(ValueError):
        R.init_vector(p, mv=0)
    with pytest.raises(InvalidSeed):
        R.init_vector(p, s0=p.skip.q, mv=2)
    with pytest.raises(InvalidSeed):
        R.init_vector(p, m0=-5)


def test_snapshot_roundtrip(golden_regression):
    p = prod(golden_regression)
    st = rsacore.GeneratorState(m1=5, m2=7, s=11, draws=99)
    text = rsacore.snapshot(st, p).to_text()
    p2, st2 = rsacore.restore(text)
    assert p2 == p and (st2.m1, st2.m2, st2.s, st2.draws) == (5, 7, 11, 99)
    assert rsacore.params_from_text(rsacore.params_to_text(p)) == p
    with pytest.raises(MalformedSnapshot):
        rsacore.restore(text.replace("m1=5", "m1=zz"))
    with pytest.raises(MalformedSnapshot):
        rsacore.restore(text.replace("rsarand-snapshot-v1", "nope"))


def test_jump_and_decrypt():
    p = mini()
    st = rsacore.init(p)
    rsacore.jump_periods(st, p, 3)
    assert (st.m1, st.m2, st.draws) == (3 * 78 % 11, 3 * 78 % 23, 36)
    with pytest.raises(R.NotInvertible):
        rsacore.decrypt(5, tiny())
    with pytest.raises(R.UnsupportedSkipMode):
        rsacore.jump_periods(rsacore.init(tiny()), tiny(), 1)


def test_instance_record_constants(golden_regression):
    for p in (prod(golden_regression), mini(), tiny(),
              dataclasses.replace(prod(golden_regression), e=65537)):
        r = rsacore._instance_record(p)[0]
        R32 = 1 << 32
        for pp, inv, k, r2 in ((p.p1, "p1_inv", "k1", "r2_1"), (p.p2, "p2_inv", "k2", "r2_2")):
            assert pp * int(r[inv]) % R32 == 1
            assert int(r[k]) == pow(R32, 2 * p.e, pp)
            assert int(r[r2]) == R32 * R32 % pp
        assert int(r["garner"]) == p.p2inv * R32 % p.p1
        assert float(r["n_recip"]) == 1.0 / p.n_float
        assert int(r["n"]) == p.n and int(r["e"]) == p.e
    assert rsacore._instance_record(prod(golden_regression))[0]["flags"] == _lib.RSA_FLAG_FAST
    assert rsacore._instance_record(mini())[0]["flags"] == 0
    assert rsacore._instance_record(tiny())[0]["flags"] == _lib.RSA_FLAG_FIXED


def test_numtheory_host():
    assert R.modinv(3, 220) == 147
    assert R.powmod(2, 10, 1000) == 24
    assert R.mulmod((1 << 63) - 26, (1 << 63) - 26, (1 << 63) - 25) == 1
    sieve = np.ones(20000, dtype=bool)
    sieve[:2] = False
    for i in range(2, 142):
        if sieve[i]:
            sieve[i * i::i] = False
    assert [n for n in range(20000) if R.is_prime64(n)] == np.flatnonzero(sieve).tolist()
    assert R.is_prime64((1 << 63) - 25) and not R.is_prime64(3215031751)
    assert R.factor64((1 << 63) - 26).distinct_primes() == skipgen.Q_DEFAULT_FACTORS
    assert R.is_safe_prime(2147483783) and R.is_safe_prime(5) and not R.is_safe_prime(13)


def test_skip_params():
    sk = q13()
    assert (sk.q1, sk.q2) == (6, 1)
    with pytest.raises(ValueError):
        skipgen.SkipParams.create(3)          # weak multiplier at the default q
    with pytest.raises(ValueError):
        skipgen.SkipParams.create(1 << 40)    # a*a > q
    st = skipgen.SkipState(1)
    for _ in range(1000):
        skipgen.next_skip(st, skipgen.default_skip_params())
    assert st.s == skipgen.skip_power(skipgen.default_skip_params(), 1000)


def test_shard_range():
    for total, world, align in ((1 << 20, 8, 2), (65536, 3, 1), (10, 4, 2)):
        spans = [shard_range(total, world, r, align) for r in range(world)]
        assert spans[0][0] == 0
        for (s0, c0), (s1, _) in zip(spans, spans[1:]):
            assert s0 + c0 == s1
        assert sum(c for _, c in spans) == total
        assert all(s % align == 0 and c % align == 0 for s, c in spans)


def test_fused_garner_bound():
    """csrc/draw.cuh draw_fast_hc<E, true>: h = REDC(y1*A + c2r*B) mod p1 with
    A = k1*p2inv, B = -p2inv*R (mod p1) equals the two-product Garner
    (c1 - c2)*p2inv mod p1 (rsacore.py:207-210), the 64-bit sum never
    overflows and one conditional add/subtract makes h canonical, for p1 up to
    floor(sqrt q) (the largest p1 paramfactory.py:27-30 can produce) — checked
    with Python ints at the extremes of every operand."""
    import random
    R32, M32 = 1 << 32, (1 << 32) - 1
    q = (1 << 63) - 25
    gf_max = 3037000499
    assert gf_max * gf_max <= q < (gf_max + 1) ** 2
    rng = random.Random(7)
    for p1 in (gf_max, gf_max - 2, (1 << 31) + 11, 2663418827):
        p1inv = pow(p1, -1, R32)
        for _ in range(300):
            p2 = rng.randrange(1 << 31, 1 << 32) | 1
            try:
                p2inv = pow(p2, -1, p1)
            except ValueError:
                continue
            e = 9
            k1 = pow(R32, 2 * e, p1)
            garner = p2inv * R32 % p1
            A = k1 * garner * pow(R32, -1, p1) % p1
            B = p1 - garner
            for y1, c2 in ((p1 - 1, p2 - 1), (p1 - 1, p1 - 1), (0, 0),
                           (rng.randrange(p1), rng.randrange(p2))):
                c2r = c2 - p1 if c2 >= p1 else c2
                t = y1 * A + c2r * B
                assert t < 1 << 64
                m = (t & M32) * p1inv & M32
                u = m * p1 >> 32
                th = t >> 32
                r = (th - u) & M32
                r = (r + p1) & M32 if th < u else r
                h = r - p1 if r >= p1 else r
                c1 = y1 * k1 * pow(R32, -1, p1) % p1
                assert h == (c1 - c2) * p2inv % p1


def test_identity_caches_follow_the_params_object(golden_regression):
    """rsacore's per-take front caches are keyed by object identity and never
    return another params object's entry."""
    g = golden_regression["params"]
    p = rsacore.make_params(g["p1"], g["p2"], g["e"], skipgen.SkipParams.create(g["a"]))
    f1 = rsacore.instance_flags(p)
    assert f1 == rsacore.instance_flags(p)
    assert f1 == int(rsacore._instance_record(p)[0]["flags"])
    # an equal-valued but distinct object gets its own (equal) entry
    q = rsacore.make_params(g["p1"], g["p2"], g["e"], skipgen.SkipParams.create(g["a"]))
    assert q is not p and rsacore.instance_flags(q) == f1


def test_call_cache_follows_the_loaded_library(monkeypatch):
    """_lib.call caches typed entry points per library object: replacing the
    library (a reload) is honoured on the next call."""
    from paper_1811_11629_b200 import _lib

    class FakeLib:
        def __init__(self, rc):
            self.rc = rc
            self.calls = 0

        def rsa_fake(self, *a):
            self.calls += 1
            return self.rc

    a, b = FakeLib(_lib.RSA_OK), FakeLib(_lib.RSA_OK)
    monkeypatch.setattr(_lib, "_LIB", a)
    _lib.call("rsa_fake", 1)
    monkeypatch.setattr(_lib, "_LIB", b)
    _lib.call("rsa_fake", 2)
    assert (a.calls, b.calls) == (1, 1)
    _lib._FN.pop("rsa_fake", None)
