"""Time the one-instance fill kernel at config-2 size in each output mode
(state advance only / raw / f64 / raw+f64) for e = 3, 9, 65537: what the
float map and the stores cost on top of the draw.  A/B probe, not product."""
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1811_11629_b200 as R  # noqa: E402
from paper_1811_11629_b200 import _lib, _device  # noqa: E402
from paper_1811_11629_b200.rsacore import instance_flags  # noqa: E402
from paper_1811_11629_b200.vecgen import device_instance  # noqa: E402

MV, BLOCKS = 1 << 22, 256
dev = torch.device("cuda:0")
base = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0), dev=dev)
raw = torch.empty(MV * BLOCKS, dtype=torch.uint64, device=dev)
f64 = torch.empty(MV * BLOCKS, dtype=torch.float64, device=dev)
for e in (3, 9, 65537):
    p = dataclasses.replace(base, e=e)
    st = R.init_vector(base, m0=12345, mv=MV, device=dev)
    inst = device_instance(p, dev)
    flags = instance_flags(p)
    res = {}
    for mode, (r, f) in {"none": (None, None), "raw": (raw, None), "f64": (None, f64),
                         "raw+f64": (raw, f64)}.items():
        def go():
            _lib.call("rsa_fill", inst.data_ptr(), 1, MV, BLOCKS, e, flags, st.m1.data_ptr(), st.m2.data_ptr(),
                      st.s.data_ptr(), r.data_ptr() if r is not None else None,
                      f.data_ptr() if f is not None else None, BLOCKS * MV, _device.stream(dev))
        for _ in range(2):
            go()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record()
        for _ in range(5):
            go()
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / 5
        res[mode] = (round(ms, 3), round(MV * BLOCKS / ms / 1e6, 1))
    print("e=%d" % e, res, flush=True)
