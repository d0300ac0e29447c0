"""Lane-vectorised bulk draws — the drop-in for rsarand.vecgen.

Mirrors /root/reference/pkg/src/rsarand/vecgen.py (names, arguments, stream
order, the `_pending` partial-block buffer and error behaviour), with the lane
arrays held as uint64 CUDA tensors and every step run by the K1 kernel
(csrc/fill.cu) through the C ABI.  Results are torch tensors on the state's
device; `out=` may name a preallocated device tensor, or a (pinned) host tensor,
in which case blocks are generated in chunks and copied back while the next
chunk computes.
"""

from __future__ import annotations

import functools

import os
import threading
from collections import OrderedDict
from dataclasses import dataclass, field

import torch

from . import _device, _lib, skipgen  # noqa: F401  (skipgen: the reference module's namespace, vecgen.py:1-20)
from .rsacore import (SKIP_LCG, GeneratorParams, InvalidSeed, device_instance,
                      instance_flags, validate_params,
                      MAX_BELOW_ONE, SKIP_CONST, SKIP_UNIT)  # noqa: F401


def _empty_u64(dev) -> torch.Tensor:
    return torch.empty(0, dtype=torch.uint64, device=dev)


@dataclass
class VectorState:
    """Mv lanes of (m1, m2, s) sharing one GeneratorParams (vecgen.py:31-41)."""

    params: GeneratorParams
    mv: int
    m1: torch.Tensor
    m2: torch.Tensor
    s: torch.Tensor
    draws: int = 0
    _pending: torch.Tensor | None = field(default=None)

    def __post_init__(self):
        if self._pending is None:
            self._pending = _empty_u64(self.m1.device)

    @property
    def device(self) -> torch.device:
        return self.m1.device


def _split_m0(m0: int) -> tuple[int, int]:
    return m0 & 0xFFFFFFFFFFFFFFFF, m0 >> 64


def _init_lanes(inst: torch.Tensor, n_inst: int, mv: int, m0: int, s0: int, dev):
    d = inst.device if dev is None else _device.device(dev)
    lanes = n_inst * mv
    m1 = torch.empty(lanes, dtype=torch.uint64, device=d)
    m2 = torch.empty(lanes, dtype=torch.uint64, device=d)
    s = torch.empty(lanes, dtype=torch.uint64, device=d)
    lo, hi = _split_m0(m0)
    if hi >> 64:
        raise ValueError("m0 must be below 2^128 here (reduce it mod n first)")
    _lib.call("rsa_init_lanes", inst.data_ptr(), n_inst, mv, lo, hi, s0,
              m1.data_ptr(), m2.data_ptr(), s.data_ptr(), _device.stream(d))
    return m1, m2, s


def init_vector(params: GeneratorParams, m0: int = 0, s0: int = 1, mv: int = 1,
                device=None) -> VectorState:
    """VectorState seeded like the scalar init, with lane offsets (vecgen.py:44-69)."""
    validate_params(params)
    if mv < 1:
        raise ValueError("lane count must be >= 1")
    if m0 < 0 or s0 < 0:
        raise InvalidSeed("seeds must be nonnegative")
    if params.skip_mode == SKIP_LCG:
        s0 = s0 % params.skip.q
        if s0 == 0:
            raise InvalidSeed(f"s0={s0} is divisible by q")
    d = _device.device(device)
    inst = device_instance(params, d)
    m1, m2, s = _init_lanes(inst, 1, mv, m0 % params.n, s0, d)
    return VectorState(params=params, mv=mv, m1=m1, m2=m2, s=s)


@functools.lru_cache(maxsize=1024)
def _segment_plan(lanes: int, blocks: int) -> tuple[int, int]:
    """(segments per lane, scratch bytes) of rsa_fill_segmented for this shape."""
    L = _lib.load()
    nseg = int(L.rsa_fill_segments(lanes, blocks))
    return nseg, int(L.rsa_fill_segmented_scratch_bytes(lanes, blocks)) if nseg > 1 else 0


def _fill(state: VectorState, blocks: int, raw: torch.Tensor | None, f64: torch.Tensor | None) -> None:
    """Advance all lanes `blocks` steps, writing block-major outputs.  Few
    lanes x many blocks (the scalar stream, Mv = 64) take the segmented kernel
    (rsa_fill_segmented: jump-ahead skip + scanned message sums), which splits
    every lane across many threads with bit-identical results."""
    if blocks <= 0:
        return
    p = state.params
    d = state.device
    inst = device_instance(p, d)
    flags = instance_flags(p)
    out_r = raw.data_ptr() if raw is not None else None
    out_f = f64.data_ptr() if f64 is not None else None
    nseg, nbytes = _segment_plan(state.mv, blocks)
    if nseg > 1 and flags & _lib.RSA_FLAG_FAST and (raw is not None or f64 is not None):

        def launch():
            scratch = torch.empty(nbytes, dtype=torch.uint8, device=d)
            _lib.call("rsa_fill_segmented", inst.data_ptr(), 1, state.mv, blocks, p.e, flags,
                      state.m1.data_ptr(), state.m2.data_ptr(), state.s.data_ptr(), out_r, out_f,
                      blocks * state.mv, scratch.data_ptr(), nbytes, _device.stream(d))
            return scratch

        key = (d.index, inst.data_ptr(), state.m1.data_ptr(), state.m2.data_ptr(), state.s.data_ptr(),
               state.mv, blocks, p.e, flags, out_r, out_f)
        _segmented_launch(key, launch, inst)
    else:
        _lib.call("rsa_fill", inst.data_ptr(), 1, state.mv, blocks, p.e, flags,
                  state.m1.data_ptr(), state.m2.data_ptr(), state.s.data_ptr(), out_r, out_f,
                  blocks * state.mv, _device.stream(d))
    state.draws += blocks * state.mv


# Repeated segmented fills of one shape (the scalar stream / Mv = 64 takes of
# a fixed size into a reused buffer) are launch-bound: the second identical
# call captures the launches into a CUDA graph and later calls replay it
# (kernel arguments are device pointers, so a replay reads the lane state as
# it is then).  Bounded LRU; the entry keeps the instance record and the
# graph's scratch alive.
_GRAPHS: "OrderedDict[tuple, tuple]" = OrderedDict()
_SEEN: "OrderedDict[tuple, None]" = OrderedDict()
_GRAPH_MAX = 8
_GRAPH_LOCK = threading.Lock()
# RSARAND_GRAPH_REPLAY=0 turns the replay off (every call launches directly)
_GRAPH_REPLAY = os.environ.get("RSARAND_GRAPH_REPLAY", "1") != "0"


_GRAPH_NET = 0  # kernels executed by graph replays minus the launches recorded at capture


def launch_count() -> int:
    """Kernels of the library executed so far in this process: the C ABI's
    launch counter corrected for CUDA-graph capture / replay of segmented
    takes (bench.py's gpu_launches)."""
    return int(_lib.load().rsa_launch_count()) + _GRAPH_NET


def clear_graph_cache() -> None:
    """Drop the captured segmented-fill graphs (and the scratch they hold)."""
    with _GRAPH_LOCK:
        _GRAPHS.clear()
        _SEEN.clear()


def _segmented_launch(key: tuple, launch, keep: torch.Tensor) -> None:
    d = keep.device
    # inside a caller's own capture the launches simply join that graph
    if not _GRAPH_REPLAY or torch.cuda.is_current_stream_capturing():
        launch()
        return
    with _GRAPH_LOCK:
        hit = _GRAPHS.get(key)
        if hit is not None:
            _GRAPHS.move_to_end(key)
            action = "replay"
        elif key not in _SEEN:
            _SEEN[key] = None
            if len(_SEEN) > 4 * _GRAPH_MAX:
                _SEEN.popitem(last=False)
            action = "direct"
        else:
            del _SEEN[key]  # second identical call: capture it
            action = "capture"
    if action == "direct":
        launch()
        return
    global _GRAPH_NET
    if action == "replay":
        if torch.cuda.current_device() == d.index:
            hit[0].replay()
        else:
            with torch.cuda.device(d):
                hit[0].replay()
        _GRAPH_NET += hit[3]
        return
    # capture on a side stream without torch.cuda.graph's synchronize /
    # gc / empty_cache (only our own kernels are recorded); thread-local
    # capture mode, so other threads' CUDA calls (allocator) stay legal
    cur = torch.cuda.current_stream(d)
    side = torch.cuda.Stream(device=d)
    side.wait_stream(cur)
    g = torch.cuda.CUDAGraph()
    c0 = int(_lib.load().rsa_launch_count())
    with torch.cuda.device(d), torch.cuda.stream(side):
        g.capture_begin(capture_error_mode="thread_local")
        try:
            scratch = launch()
        finally:
            g.capture_end()
    captured = int(_lib.load().rsa_launch_count()) - c0
    _GRAPH_NET -= captured  # recorded, not executed; the replays below execute them
    cur.wait_stream(side)
    with _GRAPH_LOCK:
        _GRAPHS[key] = (g, keep, scratch, captured)
        if len(_GRAPHS) > _GRAPH_MAX:
            _GRAPHS.popitem(last=False)
    with torch.cuda.device(d):
        g.replay()
    _GRAPH_NET += captured


def next_block_raw(state: VectorState) -> torch.Tensor:
    """Advance every lane one step; the Mv raw ciphertexts (vecgen.py:87-100)."""
    out = torch.empty(state.mv, dtype=torch.uint64, device=state.device)
    _fill(state, 1, out, None)
    return out


def floats_from_raw(raw: torch.Tensor, params: GeneratorParams, out: torch.Tensor | None = None) -> torch.Tensor:
    """r = min(fl(c)/fl(n), 1-2^-53) elementwise (vecgen.py:103-107)."""
    if raw.device.type != "cuda":
        raise _lib.RsaCudaError("floats_from_raw expects a CUDA uint64 tensor")
    raw = raw.contiguous()
    if out is None:
        out = torch.empty(raw.shape, dtype=torch.float64, device=raw.device)
    _lib.call("rsa_floats_from_raw", raw.data_ptr(), raw.numel(), params.n, out.data_ptr(),
              _device.stream(raw.device))
    return out


def next_block(state: VectorState) -> torch.Tensor:
    """Advance one step; the Mv doubles in lane order (vecgen.py:110-112)."""
    out = torch.empty(state.mv, dtype=torch.float64, device=state.device)
    _fill(state, 1, None, out)
    return out


def _take_device(state: VectorState, count: int, out: torch.Tensor, floats: bool) -> None:
    """Exactly `count` values in stream order into the device tensor `out`,
    honouring and refilling the partial-block buffer (vecgen.py:115-139)."""
    have = 0
    pend = state._pending
    if pend.numel():
        k = min(count, pend.numel())
        if floats:
            floats_from_raw(pend[:k], state.params, out[:k])
        else:
            out[:k].copy_(pend[:k])
        state._pending = pend[k:]
        have = k
    need = count - have
    full = need // state.mv
    if full:
        seg = out[have:have + full * state.mv]
        _fill(state, full, None if floats else seg, seg if floats else None)
        have += full * state.mv
    tail = count - have
    if tail:
        block = next_block_raw(state)
        if floats:
            floats_from_raw(block[:tail], state.params, out[have:])
        else:
            out[have:].copy_(block[:tail])
        state._pending = block[tail:]


# chunk of whole blocks generated per D2H hop when `out` is on the host
_HOST_CHUNK_VALUES = 1 << 25


def _take(state: VectorState, count: int, out, floats: bool) -> torch.Tensor:
    if count < 0:
        raise ValueError("count must be >= 0")
    dtype = torch.float64 if floats else torch.uint64
    if out is None:
        out = torch.empty(count, dtype=dtype, device=state.device)
    if out.dtype != dtype or out.numel() < count or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous {dtype} tensor with >= {count} elements")
    out = out[:count]
    if out.device.type == "cuda":
        _take_device(state, count, out, floats)
        return out
    _take_to_host(state, count, out, floats)
    return out


def _take_to_host(state: VectorState, count: int, out: torch.Tensor, floats: bool) -> None:
    """Generate on the device in whole-block chunks and stream them to the host
    buffer; chunk i+1 computes while chunk i copies (two staging buffers, a
    copy stream, events)."""
    d = state.device
    dtype = out.dtype
    chunk = max(state.mv, (_HOST_CHUNK_VALUES // state.mv) * state.mv)
    stage = [torch.empty(min(chunk, count), dtype=dtype, device=d) for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    comp = torch.cuda.current_stream(d)
    copy = torch.cuda.Stream(d)
    pos, k = 0, 0
    while pos < count:
        n = min(chunk, count - pos)
        buf = stage[k & 1]
        if k >= 2:
            comp.wait_event(done[k & 1])  # staging buffer free again
        _take_device(state, n, buf[:n], floats)
        ready = torch.cuda.Event()
        ready.record(comp)
        copy.wait_event(ready)
        with torch.cuda.stream(copy):
            out[pos:pos + n].copy_(buf[:n], non_blocking=True)
            done[k & 1].record(copy)
        pos += n
        k += 1
    copy.synchronize()


def take_raw(state: VectorState, count: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Exactly count raw values in stream order (vecgen.py:115-139)."""
    return _take(state, count, out, floats=False)


def take_floats(state: VectorState, count: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Exactly count doubles in stream order (vecgen.py:142-144)."""
    return _take(state, count, out, floats=True)


# ---------------------------------------------------------------------------
# checkpoint / resume and period jumps for lane vectors (
# the reference has these for the scalar state only, rsacore.py:276-417)

def jump_periods(state: VectorState, u: int) -> VectorState:
    """Advance every lane u full skip periods (u*(q-1) draws each) in O(1):
    one period leaves the skip unchanged and adds b to the message
    (rsacore.py:276-289), so the jump is m += u*b on every lane."""
    from .rsacore import UnsupportedSkipMode
    p = state.params
    if p.skip_mode != SKIP_LCG:
        raise UnsupportedSkipMode(f"jump_periods undefined for {p.skip_mode} mode")
    if u < 0:
        raise ValueError("u must be >= 0")
    if state._pending.numel():
        raise ValueError("jump_periods needs a block-aligned state (drain the pending values first)")
    ub1, ub2 = u * p.b % p.p1, u * p.b % p.p2
    for arr, add, mod in ((state.m1, ub1, p.p1), (state.m2, ub2, p.p2)):
        v = arr.view(torch.int64)  # residues < 2^32: exact in int64
        v.add_(add).remainder_(mod)
    state.draws += state.mv * u * (p.skip.q - 1)
    return state


def snapshot(state: VectorState) -> dict:
    """Host image of a VectorState: the reference's params text
    (rsacore.params_to_text) plus the lane arrays, draw count and pending raws."""
    from .rsacore import params_to_text
    return {"params": params_to_text(state.params), "mv": state.mv, "draws": state.draws,
            "m1": state.m1.cpu().numpy().copy(), "m2": state.m2.cpu().numpy().copy(),
            "s": state.s.cpu().numpy().copy(), "pending": state._pending.cpu().numpy().copy()}


def restore(snap: dict, device=None) -> VectorState:
    """Rebuild a VectorState from snapshot(); re-validates the parameters and
    the lane residue ranges like rsacore.restore (rsacore.py:393-417)."""
    import numpy as np
    from .rsacore import MalformedSnapshot, params_from_text
    p = params_from_text(snap["params"])
    mv = int(snap["mv"])
    arrs = [np.asarray(snap[k], dtype=np.uint64) for k in ("m1", "m2", "s")]
    if any(a.shape != (mv,) for a in arrs):
        raise MalformedSnapshot("lane arrays must have mv entries")
    if (arrs[0] >= p.p1).any() or (arrs[1] >= p.p2).any():
        raise MalformedSnapshot("message residue outside [0, p)")
    if p.skip_mode == SKIP_LCG and ((arrs[2] == 0) | (arrs[2] >= p.skip.q)).any():
        raise MalformedSnapshot("skip outside [1, q)")
    d = _device.device(device)
    m1, m2, s = (torch.from_numpy(a.copy()).to(d) for a in arrs)
    pend = torch.from_numpy(np.asarray(snap["pending"], dtype=np.uint64).copy()).to(d)
    return VectorState(params=p, mv=mv, m1=m1, m2=m2, s=s, draws=int(snap["draws"]), _pending=pend)
