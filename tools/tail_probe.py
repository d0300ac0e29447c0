"""Wave quantisation of the bulk fill: draws/s of one 256-block fill at
Mv = 2^22 (16384 CTAs = 11.07 waves of 148 x 10 resident CTAs) against lane
counts that are whole waves."""
import dataclasses, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import vecgen

base = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
wave = 148 * 10 * 128 * 2
for e in (3, 9, 65537):
    p = dataclasses.replace(base, e=e)
    for mv in (1 << 22, 11 * wave, 12 * wave, 10 * wave, 11 * wave + wave // 10):
        st0 = R.init_vector(base, m0=1234, mv=mv)
        st = vecgen.VectorState(params=p, mv=mv, m1=st0.m1, m2=st0.m2, s=st0.s)
        out = torch.empty(mv * 256, dtype=torch.float64, device="cuda")
        for _ in range(2):
            R.take_floats(st, mv * 256, out=out)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            R.take_floats(st, mv * 256, out=out)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / 5
        print(f"e={e:<6} mv={mv:>8} waves={mv / wave:6.2f}  {ms:8.3f} ms  {mv * 256 / ms / 1e6:7.2f} G/s")
        del out
