"""Interleaved variate source: the device twin of
rsarand.stats.BitSource (stats.py:89-136) over the interstream protocol of
the reference CLI (cli.py:162-176).

Selectors: 'float_leading' (the stream doubles), 'raw_low_bits' (low 32 bits
of the raw ciphertexts scaled to [0, 1)), 'raw_word' (the raw uint64 words).
Several streams are interleaved round-robin by draw index, stream 0 first,
with the same surplus buffering as the reference.  Everything stays on the
device.  When the streams share Mv, exponent and the fast kernel, whole
blocks come from ONE K1 launch that writes the round-robin order and the
selector's view directly (RSA_FLAG_INTERLEAVE / RSA_FLAG_LOW32; the streams'
lane arrays become views of one combined array); partial blocks and pending
draws take the per-stream path (take_raw, view, device transpose).
"""

from __future__ import annotations

from typing import Sequence

import torch

from . import _device, _lib, paramfactory, vecgen
from .rsacore import device_instance, instance_flags
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
        self._fused = self._setup_fused()

    def _setup_fused(self) -> tuple | None:
        """(instance table, m1, m2, s) for the one-launch interleaved fill, or
        None when the streams do not share one fast kernel configuration."""
        st = self.streams
        if len(st) < 2 or len({id(x) for x in st}) != len(st):
            return None
        p0 = st[0].params
        if any(x.mv != st[0].mv or x.params.e != p0.e or x.device != st[0].device for x in st):
            return None
        if not all(instance_flags(x.params) & _lib.RSA_FLAG_FAST for x in st):
            return None
        d = st[0].device
        inst = torch.cat([device_instance(x.params, d) for x in st]).contiguous()
        comb = []
        for name in ("m1", "m2", "s"):
            t = torch.cat([getattr(x, name) for x in st]).contiguous()
            for i, x in enumerate(st):  # the streams keep working on views of the combined lanes
                setattr(x, name, t[i * x.mv:(i + 1) * x.mv])
            comb.append(t)
        return (inst, *comb)

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
            flat = self._rounds(rounds)
            need = count - have
            parts.append(flat[:need])
            self._buffer = flat[need:]
        return parts[0] if len(parts) == 1 else torch.cat(parts)


    # ---- fused counting (stats.py: the battery consumers fed in registers) ----

    def fused_target(self) -> tuple | None:
        """(instance table, m1, m2, s) when whole blocks of this source can be
        generated and counted in one rsa_battery_fused launch (the selector's
        variates, same Mv / exponent / fast kernel for every stream, the
        stream count dividing the CTA, a block a whole number of tiles, and
        the streams in lockstep); None otherwise."""
        if self.selector not in ("float_leading", "raw_low_bits"):
            return None
        st = self.streams
        k, mv = len(st), st[0].mv
        if 256 % k or (mv * k) % _lib.RSA_BT_TILE or len({x._pending.numel() for x in st}) != 1:
            return None
        if k == 1:
            x = st[0]
            if not instance_flags(x.params) & _lib.RSA_FLAG_FAST:
                return None
            return device_instance(x.params, x.device), x.m1, x.m2, x.s
        return self._fused

    def buffered(self) -> int:
        """Variates available without generating a new block (the surplus
        buffer plus every stream's pending draws)."""
        buf = 0 if self._buffer is None else self._buffer.numel()
        return buf + len(self.streams) * self.streams[0]._pending.numel()

    def count_fused(self, blocks: int, spec, counts: torch.Tensor, flag: torch.Tensor | None,
                    slots: torch.Tensor | None, records: torch.Tensor | None) -> None:
        """Generate `blocks` whole blocks of every stream and count them with
        rsa_battery_fused (nothing is materialised); the streams advance
        exactly as take(blocks * Mv * k) would advance them.  Call only when
        buffered() == 0."""
        target = self.fused_target()
        if target is None or self.buffered():
            raise ValueError("this source cannot be counted by the fused kernel")
        inst, m1, m2, s = target
        st = self.streams
        flags = _lib.RSA_FLAG_FAST | (_lib.RSA_FLAG_LOW32 if self.selector == "raw_low_bits" else 0)
        ptr = lambda t: None if t is None else t.data_ptr()
        _lib.call("rsa_battery_fused", inst.data_ptr(), len(st), st[0].mv, blocks, st[0].params.e, flags,
                  m1.data_ptr(), m2.data_ptr(), s.data_ptr(), spec, counts.data_ptr(), ptr(flag), ptr(slots),
                  ptr(records), _device.stream(st[0].device))
        for x in st:
            x.draws += blocks * x.mv

    def _per_stream(self, rounds: int) -> torch.Tensor:
        views = [self._view(vecgen.take_raw(st, rounds), st) for st in self.streams]
        return torch.stack(views).T.reshape(-1)

    def _rounds(self, rounds: int) -> torch.Tensor:
        """`rounds` draws of every stream, interleaved (rounds * k values)."""
        st = self.streams
        k = len(st)
        pend = [x._pending.numel() for x in st]
        mv = st[0].mv
        if self._fused is None or len(set(pend)) != 1 or (rounds - min(pend[0], rounds)) < mv:
            return self._per_stream(rounds)
        dev = st[0].device
        dtype = torch.uint64 if self.selector == "raw_word" else torch.float64
        res = torch.empty(rounds * k, dtype=dtype, device=dev)
        pos = min(pend[0], rounds)  # pending draws first (equal across the streams)
        if pos:
            res[:pos * k] = self._per_stream(pos)
        nb = (rounds - pos) // mv
        L = _lib.load()
        if int(L.rsa_fill_segments(k * mv, nb)) > 1:  # too few lanes: per-stream segmented fills
            res[pos * k:(pos + nb * mv) * k] = self._per_stream(nb * mv)
        else:
            inst, m1, m2, s = self._fused
            seg = res[pos * k:(pos + nb * mv) * k]
            flags = _lib.RSA_FLAG_FAST | _lib.RSA_FLAG_INTERLEAVE
            raw = f64 = None
            if self.selector == "raw_word":
                raw = seg.data_ptr()
            else:
                f64 = seg.data_ptr()
                if self.selector == "raw_low_bits":
                    flags |= _lib.RSA_FLAG_LOW32
            _lib.call("rsa_fill", inst.data_ptr(), k, mv, nb, st[0].params.e, flags, m1.data_ptr(),
                      m2.data_ptr(), s.data_ptr(), raw, f64, 0, _device.stream(dev))
            for x in st:
                x.draws += nb * mv
        pos += nb * mv
        if rounds > pos:
            res[pos * k:] = self._per_stream(rounds - pos)
        return res


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
