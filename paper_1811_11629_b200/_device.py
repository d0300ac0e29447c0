"""Device plumbing: torch supplies device memory and the current stream; the
kernels behind the C ABI do the work.  No GPU means no generation (loud error)."""

from __future__ import annotations

import torch

from ._lib import RsaCudaError


_CUDA_OK = False  # set once a CUDA device was found (the check costs ~1 us per call)


def device(dev=None) -> torch.device:
    global _CUDA_OK
    if _CUDA_OK and type(dev) is torch.device and dev.type == "cuda" and dev.index is not None:
        return dev  # the hot path: a VectorState's own tensor device
    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RsaCudaError("rsarand_b200 needs a CUDA device (sm_100a); none is available")
        _CUDA_OK = True
    if dev is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(dev)
    if d.type != "cuda":
        raise RsaCudaError(f"rsarand_b200 computes on CUDA devices only, got {d}")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream(dev: torch.device) -> int:
    """cudaStream_t of torch's current stream on `dev` (no Stream object built)."""
    if _raw_stream is not None and dev.index is not None:
        return _raw_stream(dev.index)
    return torch.cuda.current_stream(dev).cuda_stream


def u64(values, dev: torch.device) -> torch.Tensor:
    """uint64 device tensor from Python ints (exact for all of [0, 2^64))."""
    import numpy as np
    arr = np.asarray(values, dtype=np.uint64)
    return torch.from_numpy(arr).to(dev)


def to_ints(t: torch.Tensor) -> list[int]:
    return t.cpu().numpy().tolist()
