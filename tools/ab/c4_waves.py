"""Config-4 tail probe: fused-consumer throughput per draw at whole vs fractional waves
(9 CTAs of 128 threads per SM -> 1332 CTAs per wave; 2^20 instances = 6.15 waves)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
dev = torch.device("cuda", 0)
tab = R.derive_params_table(R.DEFAULT_MASTER_SEED, 0, 1 << 20, dev=dev)
from paper_1811_11629_b200.paramfactory import InstanceTable
DRAWS = 1 << 14
for n in (1332 * 128 * 5, 1332 * 128 * 6, 1 << 20, 1332 * 128 * 7 // 2 * 2):
    n = min(n, 1 << 20)
    sub = R.derive_params_table(R.DEFAULT_MASTER_SEED, 0, n, dev=dev)
    fc = R.FusedConsumer(sub)
    fc.run(DRAWS); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fc.run(DRAWS); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"n={n} waves={n/128/1332:.2f} ms={ms:.2f} G draws/s={n*DRAWS/ms/1e6:.1f}", flush=True)
