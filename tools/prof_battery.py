"""Per-test wall time of the GPU battery at budget 1e8 (2 interleaved streams),
and the device time of its kernels (CUPTI via torch.profiler): what the
test spends on the GPU vs on the host (count-vector read-back and the
chi-square statistic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats

plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2)


def make(sel):
    return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=1 << 16) for p in plist], sel)


stats.run_battery(make, budget=1 << 23)
tot_wall = tot_dev = 0.0
for name in list(stats.CORE_TESTS) + [f"{t}_low" for t in stats.LOW_BIT_TESTS]:
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = stats.run_battery(make, budget=100_000_000, tests=[name])
    torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        stats.run_battery(make, budget=100_000_000, tests=[name])
        torch.cuda.synchronize()
    kern = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = (ev.name or "?").split("(")[0].replace("void ", "")[:40]
            kern[k] = kern.get(k, 0.0) + ev.device_time_total / 1e3
    dev = sum(kern.values())
    tot_wall += wall
    tot_dev += dev
    top = ", ".join(f"{k} {v:.2f}" for k, v in sorted(kern.items(), key=lambda x: -x[1])[:3])
    print(f"{name:22s} wall {wall:7.2f} ms  device {dev:7.2f} ms  samples={rep.reports[0].samples}  [{top}]")
print(f"total wall {tot_wall:.1f} ms, device {tot_dev:.1f} ms")
