"""Stream wire formats: the reference CLI's `gen` output
(cli.py:131-151; little-endian, test_cli.py:60-131) fed by the device.

    write_stream(state, count, fh, fmt="f64le" | "raw64" | "text", chunk=1 << 22)

Chunks of `chunk` values are generated on the GPU straight into one of two
pinned host buffers (vecgen.take_raw/take_floats(out=pinned)), and a writer
thread drains the previous chunk to the file while the next one computes.
"raw64" writes the uint64 ciphertexts, "f64le" the doubles, "text" one
`repr(float)` per line (Python's shortest round-trip form, identical to the
reference's f"{v!r}\\n").  Byte-for-byte equal to `rsarand gen` for the same
state and count (tests/test_gpu_streamio.py).
"""

from __future__ import annotations

import queue
import threading

import numpy as np
import torch

from . import vecgen

FORMATS = ("raw64", "f64le", "text")


def _encode(buf: torch.Tensor, n: int, fmt: str) -> bytes:
    arr = buf[:n].numpy()
    if fmt == "raw64":
        return arr.astype("<u8", copy=False).tobytes()
    if fmt == "f64le":
        return arr.astype("<f8", copy=False).tobytes()
    return "".join(f"{v!r}\n" for v in arr.tolist()).encode("ascii")


def write_stream(state: vecgen.VectorState, count: int, fh, fmt: str = "f64le",
                 chunk: int = 1 << 22) -> int:
    """Write `count` values of the stream to the binary file object `fh`;
    returns the number of bytes written."""
    if fmt not in FORMATS:
        raise ValueError(f"format must be one of {FORMATS}")
    if count < 0 or chunk < 1:
        raise ValueError("count must be >= 0 and chunk >= 1")
    dtype = torch.uint64 if fmt == "raw64" else torch.float64
    bufs = [torch.empty(min(chunk, max(count, 1)), dtype=dtype).pin_memory() for _ in range(2)]
    free = [threading.Event(), threading.Event()]
    for ev in free:
        ev.set()
    q: queue.Queue = queue.Queue(maxsize=2)
    written = [0]
    err: list = []

    def writer():
        while True:
            item = q.get()
            if item is None:
                return
            k, n = item
            try:
                data = _encode(bufs[k], n, fmt)
                fh.write(data)
                written[0] += len(data)
            except Exception as exc:  # surface on the caller's thread
                err.append(exc)
            finally:
                free[k].set()

    th = threading.Thread(target=writer, daemon=True)
    th.start()
    try:
        pos, k = 0, 0
        while pos < count and not err:
            n = min(chunk, count - pos)
            free[k].wait()
            free[k].clear()
            if fmt == "raw64":
                vecgen.take_raw(state, n, out=bufs[k])
            else:
                vecgen.take_floats(state, n, out=bufs[k])
            q.put((k, n))
            pos += n
            k ^= 1
    finally:
        q.put(None)
        th.join()
    if err:
        raise err[0]
    return written[0]
