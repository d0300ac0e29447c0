import cProfile, pstats, io, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats
plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2)
def make(sel):
    return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=1 << 16) for p in plist], sel)
stats.run_battery(make, budget=1 << 23)
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
stats.run_battery(make, budget=100_000_000)
torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t)
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue())
