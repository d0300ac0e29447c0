"""K1 bulk fill parity on the B200: the CUDA path through the drop-in API /
C ABI against the reference's golden vectors and the CPU oracles, bit-exact
(integer ciphertexts and float64 outputs alike)."""

import dataclasses

import numpy as np
import pytest
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import _lib, rsacore, skipgen, vecgen
from conftest import sha
from oracle import coracle
from oracle import rsa_oracle as O

pytestmark = pytest.mark.gpu


def u64np(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


@pytest.fixture(scope="module")
def p0(golden_regression):
    g = golden_regression["params"]
    return rsacore.make_params(g["p1"], g["p2"], g["e"], skipgen.SkipParams.create(g["a"]))


def test_regression_vectors_scalar(p0, golden_regression):
    st = rsacore.init(p0)
    assert rsacore.take_raws(st, p0, 16) == golden_regression["raw"]
    assert st.draws == 16
    assert (st.m1, st.m2, st.s) == tuple(golden_regression["state_after_16"][k] for k in ("m1", "m2", "s"))
    st = rsacore.init(p0)
    assert [x.hex() for x in rsacore.take_floats(st, p0, 16)] == golden_regression["f64_hex"]
    st = rsacore.init(p0)
    assert [rsacore.next_raw(st, p0) for _ in range(4)] == golden_regression["raw"][:4]


def test_scalar_stream_2e16(p0, golden_meta):
    st = rsacore.init(p0)
    raw = np.array(rsacore.take_raws(st, p0, 1 << 16), dtype=np.uint64)
    assert sha(raw.astype("<u8")) == golden_meta["c1_scalar_65536_raw_sha256"]


def test_scalar_stream_2e20_vs_c_oracle(p0):
    """Config 1 at full size: 2^20 sequential draws of one lane."""
    st = R.init_vector(p0, mv=1)
    raw = u64np(R.take_raw(st, 1 << 20))
    one = lambda v: np.array([v], dtype=np.uint64)
    want, wf = coracle.fill(coracle.params(p0.p1, p0.p2, p0.e, p0.skip.a), one(0), one(0), one(1), 1 << 20)
    assert np.array_equal(raw, want.reshape(-1))
    st = R.init_vector(p0, mv=1)
    assert np.array_equal(u64np(R.take_floats(st, 1 << 20)), wf.reshape(-1))


@pytest.mark.parametrize("mv", [1, 2, 8, 64])
def test_vector_streams(p0, golden_vectors, mv):
    st = R.init_vector(p0, mv=mv)
    raw = R.take_raw(st, 4096)
    assert np.array_equal(u64np(raw), golden_vectors[f"c1_mv{mv}_raw"])
    st = R.init_vector(p0, mv=mv)
    assert np.array_equal(u64np(R.take_floats(st, 4096)), golden_vectors[f"c1_mv{mv}_f64"])
    assert np.array_equal(u64np(R.floats_from_raw(raw, p0)), golden_vectors[f"c1_mv{mv}_f64"])


def test_seeded_and_wide(p0, golden_vectors, golden_meta):
    st = R.init_vector(p0, m0=golden_meta["seeded_m0"], mv=64)
    assert np.array_equal(u64np(R.take_raw(st, 4096)), golden_vectors["c1_seeded_mv64_raw"])
    st = R.init_vector(p0, mv=65536)
    raw = u64np(R.take_raw(st, 2 * 65536))
    assert sha(raw.astype("<u8")) == golden_meta["c1_mv65536"]["raw_sha256"]
    st = R.init_vector(p0, mv=65536)
    f = u64np(R.take_floats(st, 2 * 65536))
    assert sha(f.astype("<f8")) == golden_meta["c1_mv65536"]["f64_sha256"]


def test_partial_takes_and_pending(p0, golden_vectors, golden_meta):
    st = R.init_vector(p0, mv=8)
    got = np.concatenate([u64np(R.take_raw(st, k)) for k in golden_meta["take_parts_sizes"]])
    assert np.array_equal(got, golden_vectors["take_parts_mv8"])
    # floats drain the same raw pending buffer (vecgen.py:142-144)
    a, b = R.init_vector(p0, mv=8), R.init_vector(p0, mv=8)
    parts = [u64np(R.take_floats(a, k)) for k in (3, 13, 0, 5)]
    assert np.array_equal(np.concatenate(parts), u64np(R.take_floats(b, 21)))
    assert a.draws == b.draws == 24
    assert len(R.take_raw(R.init_vector(p0, mv=4), 0)) == 0
    with pytest.raises(ValueError):
        R.take_raw(a, -1)


def test_chained_calls_equal_one_call(p0):
    a, b = R.init_vector(p0, mv=256), R.init_vector(p0, mv=256)
    one = u64np(R.take_raw(a, 256 * 40))
    parts = np.concatenate([u64np(R.next_block_raw(b)) for _ in range(8)] +
                           [u64np(R.take_raw(b, 256 * 32))])
    assert np.array_equal(one, parts)
    for name in ("m1", "m2", "s"):
        assert torch.equal(getattr(a, name), getattr(b, name))


def test_next_block_matches_floats_of_raw(p0):
    a, b = R.init_vector(p0, mv=96), R.init_vector(p0, mv=96)
    for _ in range(5):
        f = R.next_block(a)
        r = R.next_block_raw(b)
        assert torch.equal(f, R.floats_from_raw(r, p0))


def _lane_subset_check(p0, golden_vectors, golden_meta, e, blocks=16):
    pe = dataclasses.replace(p0, e=e)  # e=65537 bypasses validation like the reference recipe
    mv = golden_meta["c2"]["mv"]
    d = torch.device("cuda")
    inst = rsacore.device_instance(pe, d)
    m1, m2, s = vecgen._init_lanes(inst, 1, mv, golden_meta["seeded_m0"] % pe.n, 1, d)
    st = vecgen.VectorState(params=pe, mv=mv, m1=m1, m2=m2, s=s)
    raw = torch.empty(blocks * mv, dtype=torch.uint64, device=d)
    f64 = torch.empty(blocks * mv, dtype=torch.float64, device=d)
    vecgen._fill(st, blocks, raw, f64)
    lanes = golden_vectors["c2_lanes"]
    raw = u64np(raw).reshape(blocks, mv)[:, lanes]
    f64 = u64np(f64).reshape(blocks, mv)[:, lanes]
    assert np.array_equal(raw, golden_vectors[f"c2_e{e}_raw"][:blocks])
    assert np.array_equal(f64, golden_vectors[f"c2_e{e}_f64"][:blocks])


@pytest.mark.parametrize("e", [3, 5, 9, 17, 257, 65537])
def test_config2_exponents_lane_subset(p0, golden_vectors, golden_meta, e):
    """Config 2 (Mv = 2^22, seeded m0) for every exponent, against the
    reference's own lane-subset draws."""
    _lane_subset_check(p0, golden_vectors, golden_meta, e)


def test_config2_full_fill_properties(p0, golden_meta):
    """2^30 doubles at Mv=2^22 (256 blocks): random lanes bit-exact against
    the C oracle over all blocks; size-independent properties on the whole."""
    mv, blocks = 1 << 22, 256
    st = R.init_vector(p0, m0=golden_meta["seeded_m0"], mv=mv)
    s_init = u64np(st.s)
    out = R.take_floats(st, mv * blocks)
    assert float(out.min()) >= 0.0 and float(out.max()) < 1.0
    assert abs(float(out.mean()) - 0.5) < 1e-4
    rng = np.random.default_rng(7)
    lanes = np.unique(rng.integers(0, mv, size=1024))
    m0 = golden_meta["seeded_m0"]
    cp = coracle.params(p0.p1, p0.p2, p0.e, p0.skip.a)
    m1 = np.full(len(lanes), m0 % p0.p1, dtype=np.uint64)
    m2 = np.full(len(lanes), m0 % p0.p2, dtype=np.uint64)
    s = np.ascontiguousarray(s_init[lanes])
    _, want = coracle.fill(cp, m1, m2, s, blocks, raw=False)
    got = out.view(blocks, mv)[:, torch.from_numpy(lanes).cuda()].cpu().numpy()
    assert np.array_equal(got, want)
    assert np.array_equal(u64np(st.s)[lanes], s)


def test_e65537_full_vector(p0, golden_vectors, golden_meta):
    pe = dataclasses.replace(p0, e=65537)
    d = torch.device("cuda")
    inst = rsacore.device_instance(pe, d)
    m1, m2, s = vecgen._init_lanes(inst, 1, 256, golden_meta["seeded_m0"] % pe.n, 1, d)
    st = vecgen.VectorState(params=pe, mv=256, m1=m1, m2=m2, s=s)
    got = np.stack([u64np(R.next_block_raw(st)) for _ in range(8)])
    assert np.array_equal(got, golden_vectors["c2_e65537_mv256_raw"])


def test_miniature_test_mode(golden_vectors, golden_meta):
    g = golden_meta["miniature"]
    mini = rsacore.make_params(g["p1"], g["p2"], g["e"],
                               skipgen.SkipParams.create(g["a"], q=g["q"], allow_weak=True),
                               test_mode=True)
    st = rsacore.init(mini)
    raws = rsacore.take_raws(st, mini, 3036 * 2)
    assert raws == golden_vectors["mini_scalar_raw"].tolist()
    assert (st.m1, st.m2, st.s) == (0, 0, 1)  # full period recurs (test_acceptance.py:45-61)
    v = R.init_vector(mini, mv=3)
    assert np.array_equal(u64np(R.take_raw(v, 3036 * 3)), golden_vectors["mini_mv3_raw"])
    assert u64np(R.init_vector(mini, mv=4).s).tolist() == [1, 8, 12, 5]


def test_counter_modes(p0, golden_vectors, golden_meta):
    g = golden_meta["tiny"]
    tiny = rsacore.make_params(g["p1"], g["p2"], g["e"],
                               skipgen.SkipParams.create(g["a"], q=g["q"], allow_weak=True),
                               skip_mode="unit", test_mode=True)
    st = rsacore.init(tiny)
    assert rsacore.take_raws(st, tiny, 200) == golden_vectors["tiny_unit_raw"].tolist()
    assert golden_vectors["tiny_unit_raw"][37] == 48  # the worked Garner example
    unit9 = rsacore.make_params(p0.p1, p0.p2, 9, p0.skip, skip_mode="unit")
    for mv in (1, 3, 8):
        v = R.init_vector(unit9, m0=5, mv=mv)
        assert np.array_equal(u64np(R.take_raw(v, 64)), golden_vectors[f"unit_m05_mv{mv}_raw"])
    const9 = rsacore.make_params(p0.p1, p0.p2, 9, p0.skip, skip_mode="const",
                                 skip_const=golden_meta["const_skip"])
    v = R.init_vector(const9, mv=7)
    assert np.array_equal(u64np(R.take_raw(v, 50)), golden_vectors["const_mv7_raw"])
    st = rsacore.init(const9)
    assert rsacore.take_raws(st, const9, 50) == golden_vectors["const_mv7_raw"].tolist()


def test_clamp_and_float_map(p0, golden_vectors):
    raw = torch.from_numpy(golden_vectors["clamp_raw"]).cuda()
    f = u64np(R.floats_from_raw(raw, p0))
    assert np.array_equal(f, golden_vectors["clamp_f64"])
    assert f[1] == rsacore.MAX_BELOW_ONE
    # reciprocal + two Markstein steps == IEEE fl(c)/fl(n), on random and edge ciphertexts
    rng = np.random.default_rng(11)
    for n in (p0.n, (1 << 63) - 25 - 4_600_000_000_000 | 1, (1 << 63) + 4_200_000_000_001, 77, 253):
        c = rng.integers(0, n, size=1 << 22, dtype=np.uint64)
        c[:8] = [0, 1, n - 1, n - 2, n // 2, n // 3, 1 << 52, (1 << 53) + 1]
        edges = np.array([1 << k for k in range(64) if (1 << k) < n], dtype=np.uint64)
        c = np.concatenate([c, edges, edges - np.uint64(1)])
        want = np.minimum(c.astype(np.float64) / float(n), rsacore.MAX_BELOW_ONE)
        got = np.empty_like(want)
        ct = torch.from_numpy(c).cuda()
        out = torch.empty(len(c), dtype=torch.float64, device="cuda")
        for fn in ("rsa_floats_from_raw", "rsa_floats_from_raw_dd"):  # 5-op and 4-op quotients
            _lib.call(fn, ct.data_ptr(), len(c), n, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
            assert np.array_equal(u64np(out), want), (fn, n)


def test_lane_seeds(p0, golden_vectors):
    assert np.array_equal(np.array(skipgen.lane_offset_seeds(p0.skip, 1, 64), dtype=np.uint64), golden_vectors["lane_seeds_mv64"])
    assert np.array_equal(np.array(skipgen.lane_offset_seeds(p0.skip, 777, 64), dtype=np.uint64),
                          golden_vectors["lane_seeds_mv64_s0_777"])
    v = R.init_vector(p0, mv=64)
    assert np.array_equal(u64np(v.s), golden_vectors["lane_seeds_mv64"])


def test_lane_partition_matches_whole(p0):
    """Halves of the lane vector advanced separately equal the fused update
    (test_vecgen.py:156-171) — what licenses sharding lanes across GPUs."""
    whole = R.init_vector(p0, mv=8)
    halves = []
    for sl in (slice(0, 4), slice(4, 8)):
        h = R.init_vector(p0, mv=8)
        h.m1, h.m2, h.s, h.mv = h.m1[sl].clone(), h.m2[sl].clone(), h.s[sl].clone(), 4
        halves.append(h)
    for _ in range(50):
        blk = u64np(R.next_block(whole))
        assert np.array_equal(blk, np.concatenate([u64np(R.next_block(h)) for h in halves]))


def test_lane_states_distinct(p0):
    v = R.init_vector(p0, mv=64)
    R.take_raw(v, 64 * 10_000)
    assert len(np.unique(u64np(v.s))) == 64


def test_take_into_host_buffer(p0):
    a, b = R.init_vector(p0, mv=1 << 12), R.init_vector(p0, mv=1 << 12)
    n = (1 << 26) + 12345
    host = torch.empty(n, dtype=torch.float64).pin_memory()
    R.take_floats(a, n, out=host)
    dev = R.take_floats(b, n)
    assert torch.equal(host, dev.cpu())
    assert torch.equal(a._pending, b._pending) and a.draws == b.draws


def _fill_with(pe, flags, mv, blocks, m0, raw=True, f64=True):
    from paper_1811_11629_b200 import _device
    d = torch.device("cuda")
    inst = rsacore.device_instance(pe, d)
    m1, m2, s = vecgen._init_lanes(inst, 1, mv, m0 % pe.n, 1, d)
    s0 = u64np(s).copy()
    r = torch.empty(blocks * mv, dtype=torch.uint64, device=d) if raw else None
    f = torch.empty(blocks * mv, dtype=torch.float64, device=d) if f64 else None
    _lib.call("rsa_fill", inst.data_ptr(), 1, mv, blocks, pe.e, flags, m1.data_ptr(), m2.data_ptr(),
              s.data_ptr(), r.data_ptr() if raw else None, f.data_ptr() if f64 else None, blocks * mv,
              _device.stream(d))
    return (u64np(r) if raw else None, u64np(f) if f64 else None,
            (u64np(m1), u64np(m2), u64np(s)), s0)


@pytest.mark.parametrize("e", [3, 5, 7, 9, 17, 257, 65537])
def test_fast_equals_general_path(p0, golden_meta, e):
    """The specialised fast kernel (lazy Montgomery, FMA float map, 2 or 1 lanes
    per thread) and the general kernel (plain %-reductions) agree bit-for-bit
    on every raw value, double and final lane state, and both match the C
    oracle on sampled lanes (specialised and runtime exponents)."""
    pe = dataclasses.replace(p0, e=e)
    mv, blocks, m0 = 1 << 16, 64, golden_meta["seeded_m0"]
    rh, fh, sh, s0 = _fill_with(pe, _lib.RSA_FLAG_FAST, mv, blocks, m0)
    for extra in (_lib.RSA_FLAG_GENERAL_PATH, _lib.RSA_FLAG_ONE_LANE):
        ri, fi, si, _ = _fill_with(pe, _lib.RSA_FLAG_FAST | extra, mv, blocks, m0)
        assert np.array_equal(rh, ri) and np.array_equal(fh, fi)
        for a, b in zip(sh, si):
            assert np.array_equal(a, b)
    # f64-only and raw-only variants take different code paths
    _, f_only, _, _ = _fill_with(pe, _lib.RSA_FLAG_FAST, mv, blocks, m0, raw=False)
    r_only, _, _, _ = _fill_with(pe, _lib.RSA_FLAG_FAST, mv, blocks, m0, f64=False)
    assert np.array_equal(f_only, fh) and np.array_equal(r_only, rh)
    lanes = np.unique(np.random.default_rng(e).integers(0, mv, size=200))
    cp = coracle.params(pe.p1, pe.p2, e, pe.skip.a)
    k = len(lanes)
    want_r, want_f = coracle.fill(cp, np.full(k, m0 % pe.p1, dtype=np.uint64),
                                  np.full(k, m0 % pe.p2, dtype=np.uint64), s0[lanes].copy(), blocks)
    assert np.array_equal(rh.reshape(blocks, mv)[:, lanes], want_r)
    assert np.array_equal(fh.reshape(blocks, mv)[:, lanes], want_f)


def test_odd_lane_counts_take_the_scalar_store_path(p0):
    for mv in (1, 3, 33, 65):
        a = R.init_vector(p0, mv=mv)
        got = u64np(R.take_floats(a, mv * 50))
        st = O.init(O.Params(p0.p1, p0.p2, p0.e, p0.skip.a), mv=mv)
        assert np.array_equal(got, O.take_floats(st, mv * 50))


@pytest.mark.parametrize("mv,stride_pad", [(64, 0), (3, 0), (8, 5), (1, 0)])
def test_multi_instance_layout(golden_streams, mv, stride_pad):
    """n_inst > 1 in one launch: instance-major rows out[i*stride + k*mv + g],
    each row the instance's own stream (odd mv / padded strides take the
    one-lane path)."""
    from paper_1811_11629_b200 import _device
    t = R.derive_params_table(golden_streams["master_seed"], 10, 6)
    d = t.device
    blocks = 37
    stride = blocks * mv + stride_pad
    m1, m2, s = vecgen._init_lanes(t.inst, 6, mv, 12345, 1, d)
    out = torch.full((6 * stride,), -1.0, dtype=torch.float64, device=d)
    raw = torch.zeros(6 * stride, dtype=torch.uint64, device=d)
    _lib.call("rsa_fill", t.inst.data_ptr(), 6, mv, blocks, 9, _lib.RSA_FLAG_FAST, m1.data_ptr(),
              m2.data_ptr(), s.data_ptr(), raw.data_ptr(), out.data_ptr(), stride, _device.stream(d))
    out, raw = u64np(out).reshape(6, stride), u64np(raw).reshape(6, stride)
    for i in range(6):
        P = O.from_fields(golden_streams["streams"][str(10 + i)])
        st = O.init(P, m0=12345, mv=mv)
        want = O.take_raw(st, blocks * mv)
        assert np.array_equal(raw[i, :blocks * mv], want)
        assert np.array_equal(out[i, :blocks * mv], O.floats_from_raw(want, P))
        assert (out[i, blocks * mv:] == -1.0).all()


def test_capi_argument_errors(p0):
    from paper_1811_11629_b200 import _device
    lib = _lib.load()
    d = torch.device("cuda")
    inst = rsacore.device_instance(p0, d)
    st = torch.zeros(3 * 8, dtype=torch.uint64, device=d)
    o = torch.empty(64, dtype=torch.float64, device=d)
    sp = _device.stream(d)
    # inst_stride smaller than a row of output for n_inst > 1
    assert lib.rsa_fill(inst.data_ptr(), 2, 4, 4, 9, 1, st.data_ptr(), st.data_ptr(), st.data_ptr(),
                        None, o.data_ptr(), 8, sp) == _lib.RSA_EINVAL
    assert lib.rsa_fill(inst.data_ptr(), 1, 0, 4, 9, 1, st.data_ptr(), st.data_ptr(), st.data_ptr(),
                        None, o.data_ptr(), 8, sp) == _lib.RSA_EINVAL
    assert lib.rsa_fused_stats(inst.data_ptr(), 3, 4, 9, st.data_ptr(), st.data_ptr(), st.data_ptr(),
                               o.data_ptr(), o.data_ptr(), sp) == _lib.RSA_EINVAL
    # zero blocks is a no-op
    assert lib.rsa_fill(inst.data_ptr(), 1, 4, 0, 9, 1, st.data_ptr(), st.data_ptr(), st.data_ptr(),
                        None, o.data_ptr(), 0, sp) == _lib.RSA_OK
    with pytest.raises(_lib.RsaCudaError):
        _lib.call("rsa_safe_prime_scan", 0, (1 << 32) + 1, None, 0, st.data_ptr(), None, 0, sp)
    # the interleaved / low-32 layouts exist on the fast kernel only
    for extra in (_lib.RSA_FLAG_INTERLEAVE, _lib.RSA_FLAG_LOW32):
        assert lib.rsa_fill(inst.data_ptr(), 1, 4, 2, 9, _lib.RSA_FLAG_GENERAL_PATH | extra, st.data_ptr(),
                            st.data_ptr(), st.data_ptr(), None, o.data_ptr(), 8, sp) == _lib.RSA_EPARAMS
    # segmented fill: no output is an error, a non-fast instance is rejected
    assert lib.rsa_fill_segmented(inst.data_ptr(), 1, 1, 4096, 9, 1, st.data_ptr(), st.data_ptr(),
                                  st.data_ptr(), None, None, 4096, st.data_ptr(), 8, sp) == _lib.RSA_EINVAL
    assert lib.rsa_fill_segmented(inst.data_ptr(), 1, 1, 4096, 9, 0, st.data_ptr(), st.data_ptr(),
                                  st.data_ptr(), None, o.data_ptr(), 4096, st.data_ptr(), 8, sp) == _lib.RSA_EPARAMS


def test_float_map_many_moduli_and_near_midpoints(golden_streams):
    """The reciprocal + Markstein float maps (5-op, and the 4-op double-double
    form of the fused kernels) against IEEE division for 512 derived moduli: random ciphertexts and ciphertexts whose quotient sits
    next to a rounding midpoint (the hardest inputs for a correctly rounded
    divide)."""
    from paper_1811_11629_b200 import _device
    t = R.derive_params_table(golden_streams["master_seed"], 5000, 512)
    ns = t.records()["n"].astype(np.uint64)
    rng = np.random.default_rng(99)
    d = torch.device("cuda")
    for n in ns[:: 8].tolist() + ns[1:: 8][:8].tolist():
        c = rng.integers(0, n, size=1 << 16, dtype=np.uint64)
        # near-midpoints: c ~ (j + 1/2) 2^-53 n for random j in [2^51, 2^53)
        j = rng.integers(1 << 51, 1 << 53, size=1 << 14, dtype=np.uint64)
        from fractions import Fraction
        mids = [int((Fraction(int(k)) + Fraction(1, 2)) * n / (1 << 53)) for k in j[:2048]]
        c = np.concatenate([c, np.array([m + dd for m in mids for dd in (-1, 0, 1) if 0 <= m + dd < n],
                                        dtype=np.uint64)])
        want = np.minimum(c.astype(np.float64) / float(n), rsacore.MAX_BELOW_ONE)
        ct = torch.from_numpy(c).to(d)
        out = torch.empty(len(c), dtype=torch.float64, device=d)
        for fn in ("rsa_floats_from_raw", "rsa_floats_from_raw_dd"):  # 5-op and 4-op quotients
            _lib.call(fn, ct.data_ptr(), len(c), int(n), out.data_ptr(), _device.stream(d))
            assert np.array_equal(u64np(out), want), (fn, n)


# lanes x blocks <= 2^23 take K1p (one thread per draw), larger ones K1s (segments)
@pytest.mark.parametrize("mv,blocks,e", [(1, 1 << 18, 9), (1, 1 << 20, 3), (3, 40000, 5), (64, 20000, 65537),
                                         (100, 3000, 7), (2048, 100, 9), (1, 70, 17),
                                         (64, (1 << 17) + 5, 9), (8, (1 << 20) + 3, 5), (1, (1 << 23) + 7, 3),
                                         # K1p at its largest segment indices (19- and 18-bit jump tables)
                                         (1, 1 << 23, 9), (3, (1 << 21) + 1, 17)])
def test_segmented_fill_equals_lane_fill(p0, mv, blocks, e):
    """rsa_fill_segmented (lanes split across threads: jump-ahead skip + scanned
    message sums) is bit-identical to the one-thread-per-lane rsa_fill, outputs
    and final lane state alike."""
    from paper_1811_11629_b200 import _device
    pe = dataclasses.replace(p0, e=e)
    d = torch.device("cuda")
    inst = rsacore.device_instance(pe, d)
    lib = _lib.load()
    assert lib.rsa_fill_segments(mv, blocks) > 1
    res = []
    for seg in (False, True):
        m1, m2, s = vecgen._init_lanes(inst, 1, mv, 987654321, 1, d)
        r = torch.empty(blocks * mv, dtype=torch.uint64, device=d)
        f = torch.empty(blocks * mv, dtype=torch.float64, device=d)
        if seg:
            nb = int(lib.rsa_fill_segmented_scratch_bytes(mv, blocks))
            sc = torch.empty(nb, dtype=torch.uint8, device=d)
            _lib.call("rsa_fill_segmented", inst.data_ptr(), 1, mv, blocks, e, _lib.RSA_FLAG_FAST,
                      m1.data_ptr(), m2.data_ptr(), s.data_ptr(), r.data_ptr(), f.data_ptr(),
                      blocks * mv, sc.data_ptr(), nb, _device.stream(d))
        else:
            _lib.call("rsa_fill", inst.data_ptr(), 1, mv, blocks, e, _lib.RSA_FLAG_FAST, m1.data_ptr(),
                      m2.data_ptr(), s.data_ptr(), r.data_ptr(), f.data_ptr(), blocks * mv, _device.stream(d))
        res.append([u64np(x) for x in (r, f, m1, m2, s)])
    for a, b in zip(*res):
        assert np.array_equal(a, b)


def test_vector_snapshot_restore_and_jump(p0):
    a = R.init_vector(p0, mv=16)
    R.take_raw(a, 16 * 10 + 5)
    snap = vecgen.snapshot(a)
    want = u64np(R.take_raw(a, 1000))
    b = vecgen.restore(snap)
    assert np.array_equal(u64np(R.take_raw(b, 1000)), want)
    assert b.draws == a.draws
    # one period jump = u*b added to every lane message (rsacore.jump_periods per lane)
    c = R.init_vector(p0, mv=4)
    seeds = u64np(c.s)
    vecgen.jump_periods(c, 3)
    for g in range(4):
        st = rsacore.GeneratorState(m1=0, m2=0, s=int(seeds[g]))
        rsacore.jump_periods(st, p0, 3)
        assert (int(c.m1[g].item()), int(c.m2[g].item())) == (st.m1, st.m2)
    got = u64np(R.take_raw(c, 4 * 8)).reshape(8, 4)
    for g in range(4):
        st = rsacore.GeneratorState(m1=3 * p0.b % p0.p1, m2=3 * p0.b % p0.p2, s=int(seeds[g]))
        assert got[:, g].tolist() == rsacore.take_raws(st, p0, 8)


@pytest.mark.parametrize("mv", [1, 2, 8, 64])
def test_vector_equals_interleaved_scalar_streams(p0, mv):
    """Reference acceptance c09 (test_acceptance.py:192-206): take_floats at Mv
    equals the block-major interleave of Mv scalar streams seeded with the lane
    offsets, 10^5 blocks, bit-exact.  The scalar side is independent of this
    package: lane seeds from the oracle's skip_power restatement
    (skipgen.py:124-138), every lane's scalar stream from the C oracle, and up
    to 4 lanes also from the pure-Python-int scalar recurrence
    (oracle.scalar_raws, rsacore.py:236-258) mapped by floats_from_raw."""
    from oracle import coracle
    blocks = 100_000
    got = R.take_floats(R.init_vector(p0, mv=mv), blocks * mv).cpu().numpy().reshape(blocks, mv)
    P = O.Params(p0.p1, p0.p2, p0.e, p0.skip.a)
    seeds = O.lane_seeds(P, 1, mv)
    assert skipgen.lane_offset_seeds(p0.skip, 1, mv) == [int(x) for x in seeds]
    z = np.zeros(1, dtype=np.uint64)
    for g in range(mv):
        _, f = coracle.fill(coracle.params(P.p1, P.p2, P.e, P.a), z.copy(), z.copy(), seeds[g:g + 1].copy(),
                            blocks, raw=False)
        assert np.array_equal(got[:, g], f.reshape(-1)), f"lane {g} differs from the C-oracle scalar stream"
    for g in sorted({0, mv // 3, (2 * mv) // 3, mv - 1}):
        raws = np.array(O.scalar_raws(P, blocks, m0=0, s0=int(seeds[g])), dtype=np.uint64)
        assert np.array_equal(got[:, g], O.floats_from_raw(raws, P)), f"lane {g} vs Python-int scalar stream"


@pytest.mark.parametrize("mv,blocks,stride_pad", [(1, 20000, 0), (5, 4000, 3), (64, 9000, 16), (64, 40000, 2)])
def test_segmented_multi_instance(golden_streams, mv, blocks, stride_pad):
    """rsa_fill_segmented with n_inst > 1 (instance-major rows, padded
    strides) equals rsa_fill on the same lanes, outputs and final state."""
    from paper_1811_11629_b200 import _device
    t = R.derive_params_table(golden_streams["master_seed"], 3, 4)
    d = t.device
    lib = _lib.load()
    lanes = 4 * mv
    assert lib.rsa_fill_segments(lanes, blocks) > 1
    stride = blocks * mv + stride_pad
    res = []
    for seg in (False, True):
        m1, m2, s = vecgen._init_lanes(t.inst, 4, mv, 424242, 7, d)
        raw = torch.zeros(4 * stride, dtype=torch.uint64, device=d)
        f = torch.full((4 * stride,), -1.0, dtype=torch.float64, device=d)
        args = (t.inst.data_ptr(), 4, mv, blocks, 9, _lib.RSA_FLAG_FAST, m1.data_ptr(), m2.data_ptr(),
                s.data_ptr(), raw.data_ptr(), f.data_ptr(), stride)
        if seg:
            nb = int(lib.rsa_fill_segmented_scratch_bytes(lanes, blocks))
            sc = torch.empty(nb, dtype=torch.uint8, device=d)
            _lib.call("rsa_fill_segmented", *args, sc.data_ptr(), nb, _device.stream(d))
        else:
            _lib.call("rsa_fill", *args, _device.stream(d))
        res.append([u64np(x) for x in (raw, f, m1, m2, s)])
    for a, b in zip(*res):
        assert np.array_equal(a, b)
    f = res[1][1].reshape(4, stride)
    assert (f[:, blocks * mv:] == -1.0).all()


def test_next_skip_array():
    """skipgen.next_skip_array (skipgen.py:108-116) = a*s mod q elementwise,
    for the production modulus and a generic prime, numpy in -> numpy out and
    CUDA tensor in -> tensor out."""
    rng = np.random.default_rng(11)
    for a, q in ((2983799827, skipgen.Q_DEFAULT), (2, 13), (3, (1 << 61) - 1)):
        sp = skipgen.SkipParams(q=q, a=a, q1=q // a, q2=q % a)
        s = rng.integers(1, min(q, 1 << 63), size=4099, dtype=np.uint64)
        want = np.array([a * int(x) % q for x in s], dtype=np.uint64)
        got = skipgen.next_skip_array(s, sp)
        assert isinstance(got, np.ndarray) and np.array_equal(got, want)
        t = torch.from_numpy(s.view(np.int64)).cuda().view(torch.uint64)
        assert np.array_equal(u64np(skipgen.next_skip_array(t, sp)), want)
    assert skipgen.next_skip_array(np.zeros(0, dtype=np.uint64), sp).size == 0


def test_distinct_states_on_concurrent_streams(p0):
    """Distinct states advanced concurrently on distinct CUDA streams (the
    reentrancy promise of include/rsarand_b200.h) give the
    same draws as one after the other: lane fill, segmented fill and host out."""
    cases = [(4096, 64 * 4096), (1, 1 << 16), (64, 64 * 3000)]
    want = []
    for mv, n in cases:
        st = R.init_vector(p0, m0=777, mv=mv)
        want.append(u64np(R.take_floats(st, n)))
    streams = [torch.cuda.Stream() for _ in cases]
    outs = []
    for (mv, n), s in zip(cases, streams):
        with torch.cuda.stream(s):
            st = R.init_vector(p0, m0=777, mv=mv)
            outs.append(R.take_floats(st, n))
    torch.cuda.synchronize()
    for w, o in zip(want, outs):
        assert np.array_equal(w, u64np(o))
    # host-out takes on two streams at once
    hosts = [torch.empty(n, dtype=torch.float64).pin_memory() for _, n in cases[:2]]
    for (mv, n), s, h in zip(cases[:2], streams, hosts):
        with torch.cuda.stream(s):
            R.take_floats(R.init_vector(p0, m0=777, mv=mv), n, out=h)
    torch.cuda.synchronize()
    for w, h in zip(want, hosts):
        assert np.array_equal(w, h.numpy())


@pytest.mark.parametrize("mv,blocks", [(1, 70), (1, 4099), (3, 1000), (64, 1 << 13), (1, (1 << 23) + 9)])
def test_segmented_fill_stays_inside_its_buffers(p0, mv, blocks):
    """Guard bands around the scratch and the output (compute-sanitizer is
    not available on this pool): rsa_fill_segmented writes exactly its
    outputs and at most rsa_fill_segmented_scratch_bytes of scratch, in both
    the per-draw (K1p) and the segment (K1s) regimes."""
    from paper_1811_11629_b200 import _device
    d = torch.device("cuda")
    lib = _lib.load()
    inst = rsacore.device_instance(p0, d)
    m1, m2, s = vecgen._init_lanes(inst, 1, mv, 31337, 1, d)
    nb = int(lib.rsa_fill_segmented_scratch_bytes(mv, blocks))
    G = 4096
    sc = torch.full((nb + 2 * G,), 0xA5, dtype=torch.uint8, device=d)
    n = blocks * mv
    f = torch.full((n + 2 * G,), -7.0, dtype=torch.float64, device=d)
    _lib.call("rsa_fill_segmented", inst.data_ptr(), 1, mv, blocks, p0.e, _lib.RSA_FLAG_FAST,
              m1.data_ptr(), m2.data_ptr(), s.data_ptr(), None, f[G:].data_ptr(), n,
              sc[G:].data_ptr(), nb, _device.stream(d))
    torch.cuda.synchronize()
    assert bool((sc[:G] == 0xA5).all()) and bool((sc[G + nb:] == 0xA5).all())
    assert bool((f[:G] == -7.0).all()) and bool((f[G + n:] == -7.0).all())
    assert bool((f[G:G + n] >= 0).all()) and bool((f[G:G + n] < 1).all())


@pytest.mark.parametrize("mv,blocks,flags", [(4096, 33, 0), (4095, 33, 0), (4096, 5, 8), (7, 9, 0)])
def test_lane_fill_stays_inside_its_buffers(p0, mv, blocks, flags):
    """Guard bands around rsa_fill's outputs (two-lane, one-lane and odd-Mv
    paths)."""
    from paper_1811_11629_b200 import _device
    d = torch.device("cuda")
    inst = rsacore.device_instance(p0, d)
    m1, m2, s = vecgen._init_lanes(inst, 1, mv, 99, 1, d)
    n, G = blocks * mv, 1024
    r = torch.full((n + 2 * G,), 11, dtype=torch.int64, device=d)
    f = torch.full((n + 2 * G,), -9.0, dtype=torch.float64, device=d)
    _lib.call("rsa_fill", inst.data_ptr(), 1, mv, blocks, p0.e, _lib.RSA_FLAG_FAST | flags, m1.data_ptr(),
              m2.data_ptr(), s.data_ptr(), r[G:].data_ptr(), f[G:].data_ptr(), n, _device.stream(d))
    torch.cuda.synchronize()
    assert bool((r[:G] == 11).all()) and bool((r[G + n:] == 11).all())
    assert bool((f[:G] == -9.0).all()) and bool((f[G + n:] == -9.0).all())


@pytest.mark.parametrize("mv,n", [(1, 4096), (1, 1 << 16), (64, 64 * 600)])
def test_repeated_takes_replay_graph_equal_stream(p0, mv, n):
    """Identical segmented takes into a reused buffer are captured into a CUDA
    graph on the second call and replayed after (vecgen._segmented_launch);
    the concatenated outputs and the final state equal one long take."""
    st = R.init_vector(p0, m0=5, mv=mv)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    got = []
    for _ in range(5):
        R.take_floats(st, n, out=out)
        got.append(u64np(out).copy())
    assert any(k[5] == mv and k[6] == n // mv for k in vecgen._GRAPHS)
    ref = R.init_vector(p0, m0=5, mv=mv)
    want = u64np(R.take_floats(ref, 5 * n))
    assert np.array_equal(np.concatenate(got), want)
    for a, b in ((st.m1, ref.m1), (st.m2, ref.m2), (st.s, ref.s)):
        assert torch.equal(a, b)
    assert st.draws == ref.draws
    vecgen.clear_graph_cache()
    assert not vecgen._GRAPHS


def test_segmented_take_inside_user_capture(p0):
    """A repeated identical segmented take inside the caller's own CUDA-graph
    capture joins that graph instead of nesting a capture."""
    vecgen.clear_graph_cache()
    st = R.init_vector(p0, m0=9, mv=64)
    out = torch.empty(64 * 4096, dtype=torch.float64, device="cuda")
    R.take_floats(st, out.numel(), out=out)  # first call: direct launch
    ref = R.init_vector(p0, m0=9, mv=64)
    want = u64np(R.take_floats(ref, 3 * out.numel()))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.capture_begin()
        R.take_floats(st, out.numel(), out=out)  # the second identical call, under capture
        g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(u64np(out), want[out.numel():2 * out.numel()])
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(u64np(out), want[2 * out.numel():])
    vecgen.clear_graph_cache()


def test_lookahead_stays_out_of_state_image(p0):
    """The scalar look-ahead buffer is kept beside the state: vars(state) is
    the reference's four fields, and copies / pickles continue the stream."""
    import copy
    import pickle
    st = rsacore.init(p0, m0=31337)
    rsacore.next_raw(st, p0)
    assert set(vars(st)) == {"m1", "m2", "s", "draws"}
    a, b = copy.deepcopy(st), pickle.loads(pickle.dumps(st))
    want = [rsacore.next_raw(st, p0) for _ in range(5)]
    assert [rsacore.next_raw(a, p0) for _ in range(5)] == want
    assert [rsacore.next_raw(b, p0) for _ in range(5)] == want
    n = len(rsacore._LOOKAHEADS)
    del a, b
    assert len(rsacore._LOOKAHEADS) == n - 2


def test_scalar_lookahead_matches_reference_steps(p0):
    """rsacore.next_raw / next_f64 served from the GPU look-ahead buffer: every
    value and the state fields after every draw equal a Python-int walk of
    the reference recurrence (rsacore.py:213-233), across refills, mixed with
    take_raws, jump_periods and direct state edits (which invalidate the
    buffer)."""
    P = O.Params(p0.p1, p0.p2, p0.e, p0.skip.a)

    def walk(m1, m2, s, k):
        out = []
        for _ in range(k):
            s = P.a * s % P.q
            m1, m2 = (m1 + s) % P.p1, (m2 + s) % P.p2
            c2 = pow(m2, P.e, P.p2)
            out.append(((pow(m1, P.e, P.p1) + P.p1 - c2 % P.p1) % P.p1 * P.p2inv % P.p1 * P.p2 + c2, m1, m2, s))
        return out

    st = rsacore.init(p0, m0=424242)
    m1, m2, s = st.m1, st.m2, st.s
    steps = walk(m1, m2, s, rsacore.LOOKAHEAD + 300)
    for i, (c, a1, a2, sk) in enumerate(steps[:rsacore.LOOKAHEAD + 100]):
        if i % 3 == 2:
            r = rsacore.next_f64(st, p0)
            assert r == min(float(c) / float(p0.n), O.MAX_BELOW_ONE), i
        else:
            assert rsacore.next_raw(st, p0) == c, i
        assert (st.m1, st.m2, st.s, st.draws) == (a1, a2, sk, i + 1), i
    # a bulk take in between, then single draws again (the buffer is stale)
    k = rsacore.LOOKAHEAD + 100
    assert rsacore.take_raws(st, p0, 50) == [x[0] for x in steps[k:k + 50]]
    for c, a1, a2, sk in steps[k + 50:k + 80]:
        assert rsacore.next_raw(st, p0) == c
        assert (st.m1, st.m2, st.s) == (a1, a2, sk)
    # direct edit of the state: the next draw follows the edited state
    st.m1 = (st.m1 + 1) % p0.p1
    want = walk(st.m1, st.m2, st.s, 2)
    assert [rsacore.next_raw(st, p0) for _ in range(2)] == [w[0] for w in want]
    # period jump (state fields change): still consistent
    rsacore.jump_periods(st, p0, 3)
    want = walk(st.m1, st.m2, st.s, 3)
    assert [rsacore.next_raw(st, p0) for _ in range(3)] == [w[0] for w in want]


def test_launch_counter_counts_executed_kernels(p0):
    """rsa_launch_count (+ vecgen's graph-replay correction) — the evidence
    behind bench.py's gpu_launches: one bulk fill = 1 kernel; a repeated
    segmented take = its kernels once per call whether launched directly,
    captured or replayed."""
    vecgen.clear_graph_cache()
    st = R.init_vector(p0, mv=1 << 18)
    c0 = vecgen.launch_count()
    R.take_floats(st, (1 << 18) * 4)
    assert vecgen.launch_count() - c0 == 1
    s1 = R.init_vector(p0, mv=64)
    out = torch.empty(64 * 4096, dtype=torch.float64, device="cuda")
    c0 = vecgen.launch_count()
    R.take_floats(s1, out.numel(), out=out)  # direct
    per_call = vecgen.launch_count() - c0
    assert per_call >= 2
    for _ in range(3):  # capture + replay, then replays
        c0 = vecgen.launch_count()
        R.take_floats(s1, out.numel(), out=out)
        assert vecgen.launch_count() - c0 == per_call
    vecgen.clear_graph_cache()
