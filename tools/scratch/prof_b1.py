import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats
plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2)
def make(sel):
    return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=1 << 16) for p in plist], sel)
stats.run_battery(make, budget=1 << 23, tests=["serial_d2"])
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    rep = stats.run_battery(make, budget=100_000_000, tests=["serial_d2"])
    torch.cuda.synchronize(); print("wall ms", 1e3 * (time.perf_counter() - t))
