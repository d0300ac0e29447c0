"""e2e D2H pipeline: take_floats(out=pinned host) throughput per staging-chunk size,
against one plain 8 GiB device->host copy (B200 box: 55.3 GB/s pipelined vs 50.9 GB/s plain)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import vecgen
p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
st = R.init_vector(p, m0=5, mv=1 << 22)
host = torch.empty(1 << 30, dtype=torch.float64, pin_memory=True)
for chunk in (1 << 24, 1 << 25, 1 << 26, 1 << 27):
    vecgen._HOST_CHUNK_VALUES = chunk
    R.take_floats(st, 1 << 30, out=host)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(2):
        R.take_floats(st, 1 << 30, out=host)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    print(chunk, f"{2 * 8 * (1 << 30) / el / 1e9:.1f} GB/s", f"{2 * (1 << 30) / el / 1e9:.2f} G/s")
# raw copy engine rate
dev = torch.empty(1 << 30, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(2):
    host.copy_(dev, non_blocking=True)
torch.cuda.synchronize(); el = time.perf_counter() - t
print("plain D2H", f"{2 * 8 * (1 << 30) / el / 1e9:.1f} GB/s")
