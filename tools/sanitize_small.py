"""Small end-to-end run for compute-sanitizer (memcheck): every kernel family once."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import paramfactory, stats, bitsource

p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
st = R.init_vector(p, mv=6)
R.take_raw(st, 37)
R.take_floats(st, 41)
st = R.init_vector(p, mv=64)
R.take_floats(st, 64 * 5 + 3)
sc = R.init(p)
R.rsacore.take_raws(sc, p, 5)
t = R.derive_params_table(R.DEFAULT_MASTER_SEED, 0, 6)
R.FusedConsumer(t).run(100)
paramfactory.safe_primes_u32(2, 200000)
paramfactory.safe_primes_u32(2, 200000, literal_mr=True)
st = R.init_vector(p, mv=1)
R.take_floats(st, 4096 + 5)          # one thread per draw (K1p)
st = R.init_vector(p, mv=64)
R.take_raw(st, 64 * 200)             # K1p across 64 lanes
src = bitsource.interstream_source(R.DEFAULT_MASTER_SEED, 0, 2, 8)
stats.poker_test(src, 5000)
stats.max_of_t_test(src, 8, 5000, 16)
stats.permutation_test(src, 3, 6000)
stats.collision_test(src, "top20bits", 64)
torch.cuda.synchronize()
print("sanitize run ok")
