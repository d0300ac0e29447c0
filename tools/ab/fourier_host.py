"""Host time of each step of the Fourier test's queueing (no syncs)."""
import os, sys, time, math
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats, _lib, _device
dev = torch.device("cuda", 0)
plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2, dev=dev)
def make(sel):
    return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=1 << 16, device=dev) for p in plist], sel)
m = 1 << 20
for rep in range(3):
    src = make("float_leading")
    torch.cuda.synchronize()
    T = []
    t = time.perf_counter()
    z = stats._on_device(src.take(2 * m * 32)).view(32, 2 * m); T.append(("take", time.perf_counter() - t)); t = time.perf_counter()
    c = torch.complex(z[:, 0::2] - 0.5, z[:, 1::2] - 0.5); T.append(("complex", time.perf_counter() - t)); t = time.perf_counter()
    f = torch.fft.fft(c, dim=-1); T.append(("fft", time.perf_counter() - t)); t = time.perf_counter()
    f = (f / math.sqrt(m)).contiguous(); T.append(("scale", time.perf_counter() - t)); t = time.perf_counter()
    torch.cuda.synchronize(); T.append(("sync", time.perf_counter() - t))
    print(" ".join(f"{k}={v*1e3:.2f}ms" for k, v in T), flush=True)
t = time.perf_counter(); src = make("float_leading"); print(f"make_source host {1e3*(time.perf_counter()-t):.2f} ms")
t = time.perf_counter(); st = R.init_vector(plist[0], m0=0, s0=1, mv=1 << 16, device=dev); print(f"init_vector host {1e3*(time.perf_counter()-t):.2f} ms")
