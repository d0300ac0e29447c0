"""One bulk fill (2^30 f64, Mv=2^22) per exponent — the ncu target.

    python tools/prof_fill.py [e ...]
"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import vecgen

es = [int(x) for x in sys.argv[1:]] or [3, 5, 17, 65537]
base = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
st0 = R.init_vector(base, m0=12345, mv=1 << 22)
out = torch.empty(1 << 30, dtype=torch.float64, device="cuda")
for e in es:
    p = dataclasses.replace(base, e=e)
    st = vecgen.VectorState(params=p, mv=1 << 22, m1=st0.m1.clone(), m2=st0.m2.clone(), s=st0.s.clone())
    R.take_floats(st, 1 << 30, out=out)
torch.cuda.synchronize()
print("ok", es)
