"""Interleaved variate source: the device twin of
rsarand.stats.BitSource (stats.py:89-136) over the interstream protocol of
the reference CLI (cli.py:162-176).

Selectors: 'float_leading' (the stream doubles), 'raw_low_bits' (low 32 bits
of the raw ciphertexts scaled to [0, 1)), 'raw_word' (the raw uint64 words).
Several streams are interleaved round-robin by draw index, stream 0 first,
with the same surplus buffering as the reference.  Everything stays on the
device: each stream's block fill runs in K1, the views and the round-robin
transpose are device tensor ops.
"""

from __future__ import annotations

from typing import Sequence

import torch

from . import paramfactory, vecgen
from .vecgen import VectorState

SELECTORS = ("float_leading", "raw_low_bits", "raw_word")


class BitSource:
    """Single-consumer variate source over one or more VectorStates."""

    SELECTORS = SELECTORS

    def __init__(self, streams: Sequence[VectorState], selector: str = "float_leading") -> None:
        if selector not in SELECTORS:
            raise ValueError(f"unknown selector {selector!r}")
        if not streams:
            raise ValueError("need at least one stream")
        self.streams = list(streams)
        self.selector = selector
        self._buffer: torch.Tensor | None = None

    def _view(self, raw: torch.Tensor, state: VectorState) -> torch.Tensor:
        if self.selector == "float_leading":
            return vecgen.floats_from_raw(raw, state.params)
        if self.selector == "raw_low_bits":
            low = (raw.view(torch.int64) & 0xFFFFFFFF).to(torch.float64)
            return low / float(1 << 32)
        return raw

    def take(self, count: int) -> torch.Tensor:
        if count < 0:
            raise ValueError("count must be >= 0")
        k = len(self.streams)
        if k == 1:
            return self._view(vecgen.take_raw(self.streams[0], count), self.streams[0])
        parts = []
        have = 0
        if self._buffer is not None and self._buffer.numel():
            head = self._buffer[:count]
            self._buffer = self._buffer[head.numel():]
            parts.append(head)
            have = head.numel()
        if have < count:
            rounds = -(-(count - have) // k)
            views = [self._view(vecgen.take_raw(st, rounds), st) for st in self.streams]
            flat = torch.stack(views).T.reshape(-1)
            need = count - have
            parts.append(flat[:need])
            self._buffer = flat[need:]
        return parts[0] if len(parts) == 1 else torch.cat(parts)


def interstream_params(master_seed: int, first_stream: int, m_p: int, e: int = 9, dev=None):
    """cli.cmd_test's interstream protocol: distinct prime pairs for streams
    first..first+m_p-1, one common multiplier (the first stream's)."""
    first = paramfactory.derive_stream_params(paramfactory.StreamKey(master_seed, first_stream), e=e, dev=dev)
    out = [first]
    for j in range(1, m_p):
        out.append(paramfactory.derive_stream_params(paramfactory.StreamKey(master_seed, first_stream + j),
                                                     e=e, multiplier=first.skip.a, dev=dev))
    return out


def interstream_source(master_seed: int, first_stream: int, m_p: int, lanes: int,
                       selector: str = "float_leading", e: int = 9, dev=None) -> BitSource:
    plist = interstream_params(master_seed, first_stream, m_p, e, dev)
    return BitSource([vecgen.init_vector(p, m0=0, s0=1, mv=lanes, device=dev) for p in plist], selector)
