"""Host-API latency of single-stream calls (B200 box: derive_stream_params 0.32 ms/stream vs the
reference's ~1 ms; init_vector(mv=64) 0.056 ms; rsacore.take_raws(16) 0.12 ms)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
t = time.perf_counter()
for i in range(1, 201):
    R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, i))
print("derive_stream_params ms/stream", (time.perf_counter() - t) / 200 * 1e3)
p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
t = time.perf_counter()
for i in range(200):
    st = R.init_vector(p, mv=64)
torch.cuda.synchronize()
print("init_vector(mv=64) ms", (time.perf_counter() - t) / 200 * 1e3)
st = R.init(p)
t = time.perf_counter()
for i in range(200):
    R.rsacore.take_raws(st, p, 16)
print("take_raws(16) ms", (time.perf_counter() - t) / 200 * 1e3)
t = time.perf_counter()
for i in range(4096):
    R.rsacore.next_raw(st, p)
print("next_raw ms (4096 calls, look-ahead refills included)", (time.perf_counter() - t) / 4096 * 1e3)
t = time.perf_counter()
for i in range(50):
    R.rsacore.take_floats(st, p, 1 << 16)
print("rsacore.take_floats(2^16) ms", (time.perf_counter() - t) / 50 * 1e3)
for mv in (1, 64, 65536):
    v = R.init_vector(p, mv=mv)
    out = torch.empty(1 << 20, dtype=torch.float64, device="cuda")
    R.take_floats(v, 1 << 20, out=out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(50):
        R.take_floats(v, 1 << 20, out=out)
    t_host = (time.perf_counter() - t) / 50 * 1e3
    torch.cuda.synchronize()
    t_all = (time.perf_counter() - t) / 50 * 1e3
    print(f"vecgen.take_floats(2^20, mv={mv}) host-call ms {t_host:.4f}  incl. sync ms {t_all:.4f}")
