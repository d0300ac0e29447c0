"""Battery kernel vs source width: frequency / serial d2 / max-of-t at budget 1e8 on a
2-stream BitSource of Mv = 2^16 (run_battery's) vs 2^17, 2^18 lanes per stream."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats
dev = torch.device("cuda", 0)
plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2, dev=dev)
for mv in (1 << 16, 1 << 17, 1 << 18):
    for name in ("frequency", "serial_d2", "max_of_t", "permutation"):
        ts = []
        for rep in range(4):
            src = bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=mv, device=dev) for p in plist], "float_leading")
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fin = stats._runner(name)(src, 100_000_000)
            e1.record(); torch.cuda.synchronize(); fin()
            ts.append(e0.elapsed_time(e1))
        print(f"mv={mv} {name:12s} {min(ts[1:]):.3f} ms", flush=True)
