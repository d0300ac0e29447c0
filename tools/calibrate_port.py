"""Speed calibration of the CPU baseline: the reference's own vecgen (imported
from /root/reference in the build container; it cannot travel to the GPU box)
against oracle/rsa_oracle.py's lockstep port, one process, Mv = 65536, 3 s per
measurement.  Output: profiles/r01_port_calibration.txt.

    PYTHONPATH=/root/reference/pkg/src python tools/calibrate_port.py
"""
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rsarand import paramfactory, vecgen  # noqa: E402  (the reference)

from oracle import rsa_oracle as O  # noqa: E402

p = paramfactory.derive_stream_params(paramfactory.StreamKey(paramfactory.DEFAULT_MASTER_SEED, 0))
for e in (3, 5, 9, 17, 65537):
    pe = dataclasses.replace(p, e=e)
    st0 = vecgen.init_vector(p, m0=12345, mv=65536)
    st = vecgen.VectorState(params=pe, mv=65536, m1=st0.m1, m2=st0.m2, s=st0.s)
    vecgen.take_floats(st, 65536)
    t, n = time.perf_counter(), 0
    while time.perf_counter() - t < 3:
        vecgen.take_floats(st, 1 << 20)
        n += 1 << 20
    ref = n / (time.perf_counter() - t)
    P = O.Params(p.p1, p.p2, e, p.skip.a)
    ost = O.init(P, m0=12345, mv=65536)
    m1, m2, s = ost.m1.copy(), ost.m2.copy(), ost.s.copy()
    t, n = time.perf_counter(), 0
    while time.perf_counter() - t < 3:
        raw, m1, m2, s = O.block_raw(m1, m2, s, P)
        O.floats_from_raw(raw, P)
        n += 65536
    port = n / (time.perf_counter() - t)
    print(f"e={e:<6d} reference vecgen.take_floats {ref / 1e6:6.2f} M/s   oracle port {port / 1e6:6.2f} M/s"
          f"   port/reference {port / ref:.2f}", flush=True)
