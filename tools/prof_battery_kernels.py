"""ncu target: one fused battery launch per kind at budget 1e8 (2 interleaved
streams, Mv = 2^16): frequency, serial d2, poker, max-of-t, permutation, gaps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats

plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2)


def make(sel="float_leading"):
    return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=1 << 16) for p in plist], sel)


n = 100_000_000
stats.freq_test(make(), n)
stats.serial_test(make(), 2, n)
stats.poker_test(make(), n)
stats.max_of_t_test(make(), samples=n)
stats.permutation_test(make(), stats.permutation_t_for_budget(n), n)
stats.gaps_test(make(), n)
torch.cuda.synchronize()
print("ok")
