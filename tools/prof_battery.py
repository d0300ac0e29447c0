"""Per-test wall time of the GPU battery at budget 1e8 (2 interleaved streams)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats

plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2)


def make(sel):
    return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=1 << 16) for p in plist], sel)


stats.run_battery(make, budget=1 << 23)
for name in list(stats.CORE_TESTS) + [f"{t}_low" for t in stats.LOW_BIT_TESTS]:
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = stats.run_battery(make, budget=100_000_000, tests=[name])
    torch.cuda.synchronize()
    print(f"{name:22s} {1e3 * (time.perf_counter() - t):8.1f} ms  samples={rep.reports[0].samples}")
