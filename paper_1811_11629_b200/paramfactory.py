"""Deterministic per-stream parameters — the drop-in for rsarand.paramfactory.

Mirrors /root/reference/pkg/src/rsarand/paramfactory.py (constants, StreamKey,
safe_primes_in, nth_safe_prime_in, find_pair, stream_indices,
derive_stream_params, exceptions).  The reference's lazily sieved p1 table
(paramfactory.py:160-189) becomes one device-resident list of all 3,060,794
safe primes in [2^31, 2^32), built once per device by the K3 Miller-Rabin scan
(csrc/primes.cu); pair search and instance construction run in K4
(csrc/setup.cu), one thread per stream id.  `derive_params_table` is the batch
form the many-instance and fused configurations use.
"""

from __future__ import annotations

import functools
import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib, numtheory, rsacore
from .skipgen import MULTIPLIER_TABLE, Q_DEFAULT, SkipParams

DEFAULT_MASTER_SEED = 0x243F6A8885A308D3   # paramfactory.py:24
DEFAULT_TOLERANCE = 1e-6                   # paramfactory.py:25
SQRT_Q = 3037000499                        # paramfactory.py:27
P1_WINDOW = ((1 << 31) + 1, SQRT_Q + 1)    # paramfactory.py:30
N_P1_WINDOW = 1_291_847                    # paramfactory.py:35-36
N_P2_WINDOW = 1_768_947
K_P1 = 1_291_831                           # paramfactory.py:41-42
K_P2 = 1_768_937
SIGMA = 35_705_744_587                     # paramfactory.py:47-48
EPSILON = 7
MAX_STEPS = 256                            # paramfactory.py:270

SAFE_PRIME_CENSUS = 3_060_794              # [2^31, 2^32) (test_acceptance.py:152-153)


class NotFound(LookupError):
    """No qualifying safe prime in the requested range/window (paramfactory.py:51-52)."""


class DerivationExhausted(RuntimeError):
    """No valid parameter set within the bounded ordinal advance (paramfactory.py:55-56)."""


@dataclass(frozen=True)
class StreamKey:
    master_seed: int
    stream_id: int


# ---------------------------------------------------------------------------
# safe primes on the device

def safe_primes_u32(lo: int, hi: int, dev=None) -> torch.Tensor:
    """Ascending safe primes in [lo, hi) (hi <= 2^32) as a uint32 device tensor."""
    if hi > 1 << 32:
        raise ValueError("sieve windows are limited to 2^32")
    d = _device.device(dev)
    lo = max(lo, 2)
    if lo >= hi:
        return torch.empty(0, dtype=torch.uint32, device=d)
    L = _lib.load()
    scratch_bytes = int(L.rsa_safe_prime_scan_scratch_bytes(lo, hi))
    scratch = torch.empty(max(scratch_bytes, 16), dtype=torch.uint8, device=d)
    count = torch.zeros(1, dtype=torch.uint64, device=d)
    # capacity: the density of safe primes never exceeds 1 per 12 candidates
    # (+2 for 5 and 7); the 2^31..2^32 census is far below that
    cap = (hi - lo) // 12 + 4 if hi - lo < (1 << 26) else int(1.1 * SAFE_PRIME_CENSUS * (hi - lo) / (1 << 31)) + 4096
    out = torch.empty(cap, dtype=torch.uint32, device=d)
    rc = L.rsa_safe_prime_scan(lo, hi, out.data_ptr(), cap, count.data_ptr(), scratch.data_ptr(),
                               scratch_bytes, _device.stream(d))
    _lib.check(rc, "rsa_safe_prime_scan")
    n = int(count.cpu().numpy()[0])
    if n > cap:
        raise _lib.RsaCudaError(f"safe-prime scan overflow ({n} > {cap})")
    return out[:n]


def safe_primes_in(lo: int, hi: int, dev=None) -> torch.Tensor:
    """Sorted safe primes in [lo, hi) as uint64 (paramfactory.py:105-130)."""
    lo = max(lo, 2)
    if hi > 1 << 32:
        raise ValueError("sieve windows are limited to 2^32")
    sp = safe_primes_u32(lo, hi, dev)
    return sp.to(torch.int64).to(torch.uint64)


def nth_safe_prime_in(lo: int, hi: int, k: int, dev=None) -> int:
    """The k-th (0-based) safe prime >= lo, below hi (paramfactory.py:133-157)."""
    if lo >= hi:
        raise ValueError("empty range")
    if k < 0:
        raise ValueError("ordinal must be >= 0")
    if hi > 1 << 32:
        raise NotImplementedError("the device scan covers [0, 2^32)")
    # widen in 2^24 segments like the reference, scanning only what is needed
    seen = 0
    for start in range(lo, hi, 1 << 24):
        arr = safe_primes_u32(start, min(start + (1 << 24), hi), dev)
        if seen + arr.numel() > k:
            return int(arr[k - seen].item())
        seen += arr.numel()
    raise NotFound(f"fewer than {k + 1} safe primes in [{lo}, {hi})")


def safe_prime_index(sp: torch.Tensor) -> torch.Tensor:
    """Bucket index of a sorted device u32 table (rsa_safe_prime_index):
    index[b] = number of entries below b*2^16, b = 0..65536."""
    idx = torch.empty(SP_INDEX_LEN, dtype=torch.int32, device=sp.device)
    _lib.call("rsa_safe_prime_index", sp.data_ptr(), int(sp.numel()), idx.data_ptr(), _device.stream(sp.device))
    return idx


SP_INDEX_LEN = 65537


class SafePrimeTable:
    """All safe primes of [2^31, 2^32) on one device (the p1 table is its
    prefix inside P1_WINDOW)."""

    def __init__(self, dev):
        self.device = dev
        self.sp = safe_primes_u32(1 << 31, 1 << 32, dev)
        self.n_sp = int(self.sp.numel())
        as64 = self.sp.to(torch.int64)
        self.n_p1 = int(torch.searchsorted(as64, torch.tensor([P1_WINDOW[1]], device=dev)).item())
        self.index = safe_prime_index(self.sp)
        self.mult_cache: dict = {}

    def mult_table(self, table: tuple) -> torch.Tensor:
        t = self.mult_cache.get(table)
        if t is None:
            t = torch.tensor(np.asarray(table, dtype=np.uint32).view(np.int32), device=self.device)
            self.mult_cache[table] = t
        return t


_TABLES: dict = {}
_TABLES_LOCK = threading.Lock()


def safe_prime_table(dev=None) -> SafePrimeTable:
    d = _device.device(dev)
    with _TABLES_LOCK:
        t = _TABLES.get(d.index)
        if t is None:
            t = _TABLES[d.index] = SafePrimeTable(d)
        return t


# ---------------------------------------------------------------------------
# pair search

def tolerance_int(tol: float, q: int) -> int:
    """Largest integer d with d <= tol*q as Python evaluates it (int vs float
    comparison is exact), so |p1 p2 - q| <= tol*q  <=>  |.| <= tolerance_int."""
    bound = tol * q
    if bound < 0:
        return -1
    return math.floor(bound)


def find_pair(p1: int, q: int = Q_DEFAULT, tol: float = DEFAULT_TOLERANCE, dev=None) -> tuple[int, int]:
    """(p1, p2): the safe prime nearest floor(q/p1), ties to the smaller, p2 != p1,
    2^31 < p2 < 2^32, |p1 p2 - q| <= tol q (paramfactory.py:195-219)."""
    if not (1 << 31) < p1 < (1 << 32) or not numtheory.is_safe_prime(p1):
        raise ValueError(f"p1={p1} is not a 32-bit safe prime")
    t = tolerance_int(tol, q)
    if t < 0:
        raise NotFound(f"no safe-prime partner for p1={p1} within {tol} of q")
    if not 0 < q < 1 << 64:
        raise NotImplementedError("q must fit in 64 bits")
    tab = safe_prime_table(dev)
    d = tab.device
    p1t = torch.tensor([p1], dtype=torch.int64, device=d).to(torch.uint32)
    p2 = torch.zeros(1, dtype=torch.uint32, device=d)
    st = torch.zeros(1, dtype=torch.int32, device=d)
    _lib.call("rsa_find_pair", p1t.data_ptr(), 1, q, min(t, (1 << 64) - 1), tab.sp.data_ptr(),
              tab.n_sp, tab.index.data_ptr(), p2.data_ptr(), st.data_ptr(), _device.stream(d))
    if int(st.item()) != 0:
        raise NotFound(f"no safe-prime partner for p1={p1} within {tol} of q")
    return p1, int(p2.to(torch.int64).item())


# ---------------------------------------------------------------------------
# derivation

@functools.lru_cache(maxsize=8)
def _index_space(n_a: int) -> int:
    """K_P1*K_P2*n_a, with the published constants re-checked (paramfactory.py:225-239)."""
    space = K_P1 * K_P2 * n_a
    if not numtheory.is_prime64(K_P1) or not numtheory.is_prime64(K_P2):
        raise RuntimeError("index radices must be prime")
    if math.gcd(SIGMA, space) != 1:
        raise RuntimeError("SIGMA shares a factor with the index space")
    phi = 1
    for p, k in numtheory.factor64(space).factors:
        phi *= (p - 1) * p ** (k - 1)
    if math.gcd(EPSILON, phi) != 1:
        raise RuntimeError("EPSILON shares a factor with phi(index space)")
    return space


def stream_indices(key: StreamKey, n_a: int = len(MULTIPLIER_TABLE)) -> tuple[int, int]:
    """(p1 ordinal, multiplier index) (paramfactory.py:242-250); host scalar, exact."""
    space = _index_space(n_a)
    beta = pow((key.master_seed + key.stream_id * SIGMA) % space, EPSILON, space)
    return beta % K_P1, beta // (K_P1 * K_P2) % n_a


@functools.lru_cache(maxsize=64)
def _checked_skip(a: int) -> SkipParams:
    """SkipParams.create(a) (primality of q, a*a <= q, primitive root), once per a."""
    return SkipParams.create(a)


def _exponent_usable(e: int) -> bool:
    """make_params accepts e for production pairs iff e is odd and 3 <= e <= 257
    (gcd(e, (p1-1)(p2-1)) = 1 always holds: (p-1)/2 is a prime > 2^30)."""
    return e % 2 == 1 and 3 <= e <= rsacore.MAX_EXPONENT


def _setup_config(master_seed: int, first_id: int, e: int, n_a: int, multiplier: int,
                  start_step: int = 0) -> _lib.SetupConfig:
    space = _index_space(n_a)
    cfg = _lib.SetupConfig()
    cfg.seed_mod_S = master_seed % space
    cfg.first_id = first_id
    cfg.sigma = SIGMA
    cfg.k_p1, cfg.k_p2 = K_P1, K_P2
    cfg.q = Q_DEFAULT
    cfg.tol = tolerance_int(DEFAULT_TOLERANCE, Q_DEFAULT)
    cfg.epsilon = EPSILON
    cfg.e = e
    cfg.n_mult = n_a
    cfg.multiplier = multiplier
    cfg.max_steps = MAX_STEPS
    cfg.start_step = start_step
    return cfg


@dataclass
class InstanceTable:
    """Device table of rsa_instance records for a contiguous range of stream ids."""

    inst: torch.Tensor      # uint8 [count, 128]
    status: torch.Tensor    # int32 [count]
    steps: torch.Tensor     # int32 [count] (uint32 values)
    master_seed: int
    first_id: int
    e: int

    @property
    def count(self) -> int:
        return int(self.status.numel())

    @property
    def device(self) -> torch.device:
        return self.inst.device

    def records(self) -> np.ndarray:
        return self.inst.cpu().numpy().reshape(-1).view(_lib.INSTANCE_DTYPE)

    def params(self, j: int) -> rsacore.GeneratorParams:
        r = self.records()[j]
        skip = SkipParams(q=int(r["q"]), a=int(r["a"]), q1=int(r["q1"]), q2=int(r["q2"]))
        return rsacore.GeneratorParams(p1=int(r["p1"]), p2=int(r["p2"]), n=int(r["n"]), e=int(r["e"]),
                                       skip=skip, p2inv=int(r["p2inv"]), b=int(r["b"]),
                                       n_float=float(r["n_float"]))


def _run_setup(cfg: _lib.SetupConfig, count: int, table: tuple, dev) -> InstanceTable:
    tab = safe_prime_table(dev)
    d = tab.device
    inst = torch.empty((count, 128), dtype=torch.uint8, device=d)
    status = torch.empty(count, dtype=torch.int32, device=d)
    steps = torch.empty(count, dtype=torch.int32, device=d)
    mult = tab.mult_table(table)
    _lib.call("rsa_setup_instances", cfg, count, mult.data_ptr(), tab.sp.data_ptr(), tab.n_sp,
              tab.index.data_ptr(), tab.sp.data_ptr(), tab.n_p1, inst.data_ptr(), status.data_ptr(), steps.data_ptr(),
              _device.stream(d))
    return InstanceTable(inst, status, steps, 0, cfg.first_id, cfg.e)


def derive_params_table(master_seed: int, first_id: int, count: int, e: int = rsacore.DEFAULT_EXPONENT,
                        multiplier_table: tuple = MULTIPLIER_TABLE, multiplier: int | None = None,
                        dev=None) -> InstanceTable:
    """Batch derive_stream_params for ids first_id .. first_id+count-1 (lcg mode),
    entirely on the device; raises DerivationExhausted naming the first id that
    has no valid pair within the bounded ordinal advance."""
    if not multiplier_table:
        raise ValueError("multiplier table must be non-empty")
    if count < 1:
        raise ValueError("count must be >= 1")
    if master_seed < 0 or first_id < 0 or first_id + count > 1 << 64:
        raise ValueError("seed and stream ids must be nonnegative 64-bit values")
    if multiplier is not None:
        _checked_skip(multiplier)
    else:
        for a in set(multiplier_table):
            _checked_skip(a)
    if not _exponent_usable(e):
        raise DerivationExhausted(f"no valid parameters for exponent e={e}")
    cfg = _setup_config(master_seed, first_id, e, len(multiplier_table), multiplier or 0)
    t = _run_setup(cfg, count, tuple(multiplier_table), dev)
    t.master_seed = master_seed
    if int(torch.count_nonzero(t.status).item()):
        j = int(torch.nonzero(t.status != 0)[0].item())
        raise DerivationExhausted(f"no valid parameters for stream id {first_id + j}")
    return t


def derive_stream_params(key: StreamKey, e: int = rsacore.DEFAULT_EXPONENT,
                         multiplier_table: tuple = MULTIPLIER_TABLE,
                         skip_mode: str = rsacore.SKIP_LCG, skip_const: int = 0,
                         multiplier: int | None = None, dev=None) -> rsacore.GeneratorParams:
    """GeneratorParams for a stream key (paramfactory.py:253-278): the device
    search picks (p1, p2); the host re-validates with make_params and, should it
    reject the pair, resumes the search at the next ordinal step."""
    if not multiplier_table:
        raise ValueError("multiplier table must be non-empty")
    ordinal, a_index = stream_indices(key, len(multiplier_table))
    a = multiplier if multiplier is not None else multiplier_table[a_index]
    skip = SkipParams.create(a)
    if not _exponent_usable(e) or key.stream_id < 0 or key.master_seed < 0:
        raise DerivationExhausted(f"no valid parameters near ordinal {ordinal}")
    start = 0
    while start < MAX_STEPS:
        cfg = _setup_config(key.master_seed, key.stream_id % (1 << 64), e, len(multiplier_table),
                            a, start)
        # stream_id enters only through id*SIGMA mod S, so reduce it mod S exactly
        cfg.first_id = key.stream_id % _index_space(len(multiplier_table))
        t = _run_setup(cfg, 1, tuple(multiplier_table), dev)
        if int(t.status[0].item()) != 0:
            break
        rec = t.records()[0]
        step = int(t.steps[0].item())
        try:
            return rsacore.make_params(int(rec["p1"]), int(rec["p2"]), e, skip,
                                       skip_mode=skip_mode, skip_const=skip_const)
        except rsacore.InvalidParams:
            start = step + 1
    raise DerivationExhausted(f"no valid parameters near ordinal {ordinal}")
