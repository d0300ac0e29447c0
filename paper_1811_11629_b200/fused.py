"""Fused consumer (config 4): generate in registers, reduce in-kernel.

No reference function exists; the estimator
definitions below are this framework's, fixed here and mirrored by the numpy
oracle (oracle/rsa_oracle.py: fused_reference).  Per instance over draws
r_0..r_{N-1} of one Mv = 1 stream (rsacore.take_floats order):

    mean = S1/N,  var = (S2 - S1^2/N)/(N-1)
    lag1 = [L - mean*(2 S1 - r_0 - r_{N-1}) + (N-1) mean^2] / (S2 - S1^2/N),
           L = sum_{k<N-1} r_k r_{k+1}
    hist[b] = #{k : floor(64 r_k) = b}      (stats._bin_uniform, stats.py:178-180)

Pooled over instances: the histogram sum and the Pearson correlation of
X = r^(2j), Y = r^(2j+1) at equal k over all pairs j (pairs never straddle a
shard, so multi-GPU needs only one all-reduce of 7 doubles + 64 counts).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _device, _lib
from .paramfactory import InstanceTable
from .vecgen import _init_lanes

POOLED_FIELDS = ("s1", "s2", "xy_even", "s1_even", "s1_odd", "s2_even", "s2_odd")


@dataclass
class FusedStats:
    draws: int
    stats: torch.Tensor        # float64 [n, 6]: s1, s2, lag, first, last, xy
    hist: torch.Tensor         # int32 [n, 64] (uint32 counts)
    pooled: torch.Tensor       # float64 [7] (POOLED_FIELDS)
    pooled_hist: torch.Tensor  # int64 [64]

    @property
    def n_inst(self) -> int:
        return int(self.stats.shape[0])

    def moments(self) -> dict:
        N = float(self.draws)
        s1, s2, lag, r0, rl = (self.stats[:, i] for i in range(5))
        mean = s1 / N
        css = s2 - s1 * s1 / N
        var = css / (N - 1.0)
        lag1 = (lag - mean * (2.0 * s1 - r0 - rl) + (N - 1.0) * mean * mean) / css
        return {"mean": mean, "var": var, "lag1": lag1}

    def pooled_correlation(self, n_pairs_total: int | None = None) -> float:
        p = self.pooled.cpu().numpy().tolist()
        pairs = n_pairs_total if n_pairs_total is not None else self.n_inst // 2
        M = float(pairs) * self.draws
        mx, my = p[3] / M, p[4] / M
        cov = p[2] / M - mx * my
        vx, vy = p[5] / M - mx * mx, p[6] / M - my * my
        return cov / math.sqrt(vx * vy)


class FusedConsumer:
    """Mv = 1 streams for every instance of a device InstanceTable."""

    def __init__(self, table: InstanceTable, m0: int = 0, s0: int = 1):
        if table.count % 2:
            raise ValueError("the fused consumer pairs instances (2j, 2j+1): count must be even")
        if not 0 <= m0 < 1 << 128 or not 1 <= s0 < (1 << 63) - 25:
            raise ValueError("seeds out of range")
        self.table = table
        self.e = table.e
        self.m1, self.m2, self.s = _init_lanes(table.inst, table.count, 1, m0, s0, None)
        self.draws = 0

    def run(self, draws: int) -> FusedStats:
        if draws < 2:
            raise ValueError("the fused statistics need at least 2 draws per instance (var uses N-1)")
        d = self.table.device
        n = self.table.count
        stats = torch.empty((n, 6), dtype=torch.float64, device=d)
        hist = torch.empty((n, 64), dtype=torch.int32, device=d)
        pooled = torch.empty(7, dtype=torch.float64, device=d)
        pooled_hist = torch.empty(64, dtype=torch.int64, device=d)
        st = _device.stream(d)
        _lib.call("rsa_fused_stats", self.table.inst.data_ptr(), n, draws, self.e,
                  self.m1.data_ptr(), self.m2.data_ptr(), self.s.data_ptr(), stats.data_ptr(),
                  hist.data_ptr(), st)
        _lib.call("rsa_fused_pool", stats.data_ptr(), hist.data_ptr(), n, pooled.data_ptr(),
                  pooled_hist.data_ptr(), st)
        self.draws += draws
        return FusedStats(draws, stats, hist, pooled, pooled_hist)


def all_reduce_pooled(res: FusedStats, group=None) -> FusedStats:
    """Sum the pooled statistics over the ranks of `group` (one NCCL all-reduce
    each for the 7 doubles and the 64 counts; gloo on CPU tensors works too)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl" or res.pooled.device.type == "cpu":
        dist.all_reduce(res.pooled, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(res.pooled_hist, op=dist.ReduceOp.SUM, group=group)
        return res
    # gloo with device tensors: reduce through host copies
    p, h = res.pooled.cpu(), res.pooled_hist.cpu()
    dist.all_reduce(p, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    res.pooled.copy_(p)
    res.pooled_hist.copy_(h)
    return res
