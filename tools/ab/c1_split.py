"""Config-1 take: host time per call vs device time per call vs graph replay alone."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import vecgen
p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
out = torch.empty(1 << 20, dtype=torch.float64, device="cuda")
for mv in (1, 64, 65536):
    v = R.init_vector(p, mv=mv)
    for _ in range(3):
        R.take_floats(v, 1 << 20, out=out)
    torch.cuda.synchronize()
    N = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter(); e0.record()
    for i in range(N):
        R.take_floats(v, 1 << 20, out=out)
    e1.record(); th = (time.perf_counter() - t) / N * 1e6
    torch.cuda.synchronize(); td = e0.elapsed_time(e1) / N * 1e3
    g = list(vecgen._GRAPHS.values())[-1][0] if mv < 65536 and vecgen._GRAPHS else None
    tg = None
    if g is not None:
        torch.cuda.synchronize()
        e0.record()
        for i in range(N):
            g.replay()
        e1.record(); torch.cuda.synchronize(); tg = e0.elapsed_time(e1) / N * 1e3
        # device-only: one graph replay bracketed by events after a sync
        ts = []
        for i in range(20):
            torch.cuda.synchronize(); e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
    print(f"mv={mv}: host {th:.1f} us/call, device loop {td:.1f} us/call, graph replay loop {tg}, single replay us (min/med) {ts[0] if g else None} {ts[10] if g else None}", flush=True)
    vecgen.clear_graph_cache()
