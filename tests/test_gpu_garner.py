"""Both Garner forms of the fast draw (csrc/draw.cuh draw_fast_hc).

Derived streams have p1 <= floor(sqrt q) and take the fused form
h = REDC(y1*A + c2r*B); make_params with the primes given in the other order
(p1 > sqrt q, still a valid production instance, rsacore.py:166-181) takes the
two-product form.  Both are checked bit-exact against the C oracle — through
the lane fill (two lanes per thread), the segmented scalar fill and the fused
consumer — and a table mixing the two forms in one launch / one warp.
"""

import numpy as np
import pytest
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import _device, _lib, paramfactory, rsacore, skipgen, vecgen
from oracle import coracle
from oracle import rsa_oracle as O

pytestmark = pytest.mark.gpu

GF_P1_MAX = 3037000499


@pytest.fixture(scope="module")
def pair(golden_regression):
    g = golden_regression["params"]
    sk = skipgen.SkipParams.create(g["a"])
    small = rsacore.make_params(g["p1"], g["p2"], 9, sk)
    big = rsacore.make_params(g["p2"], g["p1"], 9, sk)
    assert small.p1 <= GF_P1_MAX < big.p1
    return small, big


def _oracle(p, m1, m2, s, blocks):
    return coracle.fill(coracle.params(p.p1, p.p2, p.e, p.skip.a), m1, m2, s, blocks)


@pytest.mark.parametrize("e", [3, 9, 65537, 7])
def test_swapped_primes_lane_fill(pair, e):
    import dataclasses
    for p in pair:
        pe = dataclasses.replace(p, e=e)
        mv, blocks = 4096, 40
        # e = 65537 is above MAX_EXPONENT: seed at e = 9, then swap the params
        # in (the reference's own recipe, test_cli.py:183)
        st0 = R.init_vector(p, m0=987654321987, mv=mv)
        fresh = lambda: vecgen.VectorState(params=pe, mv=mv, m1=st0.m1.clone(), m2=st0.m2.clone(),
                                           s=st0.s.clone())
        m1, m2, s = (x.cpu().numpy().copy() for x in (st0.m1, st0.m2, st0.s))
        raw = R.take_raw(fresh(), mv * blocks).cpu().numpy()
        want, wf = _oracle(pe, m1, m2, s, blocks)
        assert np.array_equal(raw, want.reshape(-1)), (pe.p1, e)
        assert np.array_equal(R.take_floats(fresh(), mv * blocks).cpu().numpy(), wf.reshape(-1))


def test_swapped_primes_segmented_scalar(pair):
    """Mv = 1 with 2^18 draws runs the segmented fill (K1s)."""
    n = 1 << 18
    for p in pair:
        assert _lib.load().rsa_fill_segments(1, n) > 1
        st = R.init_vector(p, mv=1)
        got = R.take_raw(st, n).cpu().numpy()
        one = lambda v: np.array([v], dtype=np.uint64)
        want, _ = _oracle(p, one(0), one(0), one(1), n)
        assert np.array_equal(got, want.reshape(-1))


def _mixed_table(pair, count):
    recs = [rsacore._instance_record(pair[j % 2] if j % 3 else pair[0]) for j in range(count)]
    inst = torch.from_numpy(np.concatenate(recs).view(np.uint8).reshape(count, 128).copy()).cuda()
    z = torch.zeros(count, dtype=torch.int32, device=inst.device)
    return paramfactory.InstanceTable(inst, z, z.clone(), 0, 0, 9)


def test_mixed_table_fill(pair):
    """One multi-instance launch whose threads take different Garner forms."""
    n_inst, mv, blocks = 10, 64, 33
    t = _mixed_table(pair, n_inst)
    d = t.device
    m1, m2, s = vecgen._init_lanes(t.inst, n_inst, mv, 4242, 1, d)
    s0 = s.cpu().numpy().copy()
    raw = torch.zeros(n_inst * blocks * mv, dtype=torch.uint64, device=d)
    _lib.call("rsa_fill", t.inst.data_ptr(), n_inst, mv, blocks, 9, _lib.RSA_FLAG_FAST, m1.data_ptr(),
              m2.data_ptr(), s.data_ptr(), raw.data_ptr(), None, blocks * mv, _device.stream(d))
    raw = raw.cpu().numpy().reshape(n_inst, blocks, mv)
    for i in range(n_inst):
        p = t.params(i)
        lanes = slice(i * mv, (i + 1) * mv)
        want, _ = _oracle(p, np.full(mv, 4242 % p.p1, dtype=np.uint64),
                          np.full(mv, 4242 % p.p2, dtype=np.uint64), s0[lanes].copy(), blocks)
        assert np.array_equal(raw[i], want), i


def test_mixed_table_fused(pair):
    """Fused consumer over a table whose warps mix the two forms (the warp
    takes the two-product form together, so the partner shuffles stay
    converged)."""
    n_inst, N = 64, 3000
    t = _mixed_table(pair, n_inst)
    res = R.FusedConsumer(t).run(N)
    r = np.empty((n_inst, N))
    one = lambda v: np.array([v], dtype=np.uint64)
    for j in range(n_inst):
        _, f = _oracle(t.params(j), one(0), one(0), one(1), N)
        r[j] = f.reshape(-1)
    ref = O.fused_reference(r)
    assert np.array_equal(res.hist.cpu().numpy().astype(np.int64), ref["hist"])
    st = res.stats.cpu().numpy()
    assert np.array_equal(st[:, 3], r[:, 0]) and np.array_equal(st[:, 4], r[:, -1])
