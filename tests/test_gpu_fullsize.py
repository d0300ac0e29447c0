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
