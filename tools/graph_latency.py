"""Per-call latency of repeated identical segmented takes (CUDA-graph replay
after the second call): first, second (capture) and steady-state calls."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
for mv in (1, 64):
    st = R.init_vector(p, mv=mv)
    out = torch.empty(1 << 20, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ts = []
    for i in range(40):
        t = time.perf_counter()
        R.take_floats(st, 1 << 20, out=out)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"mv={mv}: call1 {ts[0]:.3f} ms  call2 (capture) {ts[1]:.3f} ms  steady median {sorted(ts[5:])[len(ts[5:]) // 2]:.4f} ms")
