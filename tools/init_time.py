"""init_vector(mv=2^22) wall time (K1 lane seeding)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
R.init_vector(p, mv=1 << 22); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    R.init_vector(p, mv=1 << 22)
torch.cuda.synchronize()
print("init_vector(2^22) ms", (time.perf_counter() - t) / 10 * 1e3)
