"""One full safe-prime scan of [2^31, 2^32) — the ncu target."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1811_11629_b200 import paramfactory

for _ in range(2):
    sp = paramfactory.safe_primes_u32(1 << 31, 1 << 32)
torch.cuda.synchronize()
print("ok", sp.numel())
