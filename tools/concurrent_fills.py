"""A/B: the bench step's four fills (e = 3, 5, 17, 65537; 2^30 doubles each)
issued back to back on one stream vs on four streams at once (the hardware
then co-schedules CTAs of different exponents on each SM).  Same outputs."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import vecgen

E = (3, 5, 17, 65537)
MV, BLOCKS = 1 << 22, 256
base = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
st0 = R.init_vector(base, m0=bench.seeded_m0(base.n), mv=MV)
states = {e: vecgen.VectorState(params=dataclasses.replace(base, e=e), mv=MV, m1=st0.m1.clone(),
                                m2=st0.m2.clone(), s=st0.s.clone()) for e in E}
outs = {e: torch.empty(MV * BLOCKS, dtype=torch.float64, device="cuda") for e in E}
streams = {e: torch.cuda.Stream() for e in E}
main = torch.cuda.current_stream()


def serial():
    for e in E:
        R.take_floats(states[e], MV * BLOCKS, out=outs[e])


def concurrent():
    for e in E:
        streams[e].wait_stream(main)
    for e in sorted(E, key=lambda x: -x):  # the long e = 65537 fill first
        with torch.cuda.stream(streams[e]):
            R.take_floats(states[e], MV * BLOCKS, out=outs[e])
    for e in E:
        main.wait_stream(streams[e])


for name, fn in (("serial", serial), ("concurrent", concurrent), ("serial", serial), ("concurrent", concurrent)):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(3):
        fn()
    b.record(main)
    b.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"{name:10s} {ms:7.3f} ms/step  {4 * MV * BLOCKS / ms / 1e6:7.2f} Gnumbers/s")
