"""run_battery at budget 1e8: host time to queue all tests vs total wall (is the battery host-bound?)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats
dev = torch.device("cuda", 0)
plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2, dev=dev)
def make(sel):
    return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=1 << 16, device=dev) for p in plist], sel)
orig = stats._runner
marks = {}
def timed_runner(core):
    f = orig(core)
    def g(src, budget):
        t = time.perf_counter(); r = f(src, budget); marks.setdefault(core, []).append(time.perf_counter() - t); return r
    return g
for _ in range(2):
    stats.run_battery(make, budget=100_000_000)
torch.cuda.synchronize()
stats._runner = timed_runner
t0 = time.perf_counter()
rep = stats.run_battery(make, budget=100_000_000)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
q = sum(sum(v) for v in marks.values())
print(f"wall {wall*1e3:.1f} ms, host time inside the 23 queue calls {q*1e3:.1f} ms")
for k, v in marks.items():
    print(f"  {k:16s} " + " ".join(f"{x*1e3:.2f}" for x in v))
t = time.perf_counter(); src = make("float_leading"); torch.cuda.synchronize(); print(f"make_source {1e3*(time.perf_counter()-t):.2f} ms")
# inside run_battery: time the Fourier steps on its side stream
import math
from paper_1811_11629_b200 import _lib, _device
orig_fc = stats._fourier_cells
def fc(source, n_blocks, m):
    dev = stats._dev()
    T = []
    t = time.perf_counter()
    edges = torch.as_tensor(stats._normal_edges(), device=dev); T.append(("edges", time.perf_counter() - t)); t = time.perf_counter()
    cells = torch.zeros(128, dtype=torch.int64, device=dev); T.append(("zeros", time.perf_counter() - t)); t = time.perf_counter()
    per_call = max(1, (1 << 26) // (2 * m)); left = n_blocks
    while left:
        k = min(per_call, left)
        z = stats._on_device(source.take(2 * m * k)).view(k, 2 * m); T.append(("take", time.perf_counter() - t)); t = time.perf_counter()
        c = torch.complex(z[:, 0::2] - 0.5, z[:, 1::2] - 0.5); T.append(("complex", time.perf_counter() - t)); t = time.perf_counter()
        coeff = (torch.fft.fft(c, dim=-1) / math.sqrt(m)).contiguous(); T.append(("fft", time.perf_counter() - t)); t = time.perf_counter()
        _lib.call("rsa_battery_fourier_bin", torch.view_as_real(coeff).data_ptr(), coeff.numel(), edges.data_ptr(), cells.data_ptr(), _device.stream(dev))
        T.append(("bin", time.perf_counter() - t)); t = time.perf_counter()
        left -= k
    print("fourier steps: " + " ".join(f"{a}={b*1e3:.2f}" for a, b in T))
    return cells
stats._fourier_cells = fc
stats._runner = orig
for i in range(3):
    t0 = time.perf_counter(); rep = stats.run_battery(make, budget=100_000_000); torch.cuda.synchronize(); print(f"wall {1e3*(time.perf_counter()-t0):.1f} ms")
