"""Per-stream parameters from (master seed, stream id) — drop-in for
`rsarand.paramfactory` (same names, constants and exceptions;
paramfactory.py:24-278).

Where the reference sieves the p1 window lazily and searches partners with
per-candidate Miller-Rabin calls, this module keeps ONE device-resident sorted
list of all 3,060,794 safe primes of [2^31, 2^32) (built once per device by
the K3 scan, csrc/primes.cu) plus its 2^12-bucket index; the pair search and
the instance constants run in K4 (csrc/setup.cu), one thread per stream id.
`derive_params_table` is the batch form (configs 3-5).
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

# published constants of the reference (paramfactory.py:24-48, 270)
DEFAULT_MASTER_SEED = 0x243F6A8885A308D3   # the hex digits of pi
DEFAULT_TOLERANCE = 1e-6                   # |p1 p2 - q| <= tolerance * q
SQRT_Q = math.isqrt(Q_DEFAULT)             # 3037000499
P1_WINDOW = (2 ** 31 + 1, SQRT_Q + 1)      # p1 in (2^31, sqrt(q)], p2 above it
N_P1_WINDOW = 1_291_847                    # safe primes in the p1 window
N_P2_WINDOW = 1_768_947                    # ... and in (sqrt(q), 2^32)
K_P1, K_P2 = 1_291_831, 1_768_937          # prime radices of the index space (<= the window counts)
SIGMA = 35_705_744_587                     # stream-id stride, coprime to the index space
EPSILON = 7                                # the index permutation x -> x^7 mod S
MAX_STEPS = 256                            # bounded ordinal advance

SAFE_PRIME_CENSUS = 3_060_794              # safe primes in [2^31, 2^32) (test_acceptance.py:152-153)


class NotFound(LookupError):
    """The requested safe prime or partner does not exist in the range."""


class DerivationExhausted(RuntimeError):
    """MAX_STEPS ordinal advances found no valid prime pair."""


@dataclass(frozen=True)
class StreamKey:
    master_seed: int
    stream_id: int


# ---------------------------------------------------------------------------
# safe primes on the device

def safe_primes_u32(lo: int, hi: int, dev=None, literal_mr: bool = False) -> torch.Tensor:
    """Ascending safe primes in [lo, hi) (hi <= 2^32) as a uint32 device tensor.
    literal_mr: run the census as BASELINE config 5 words it (Miller-Rabin
    2, 7, 61 on every odd n and on (n-1)/2, rsa_safe_prime_scan_mr) instead of
    the sieve + base-2 SPRP + pseudoprime-table scan; the list is the same."""
    if hi > 1 << 32:
        raise ValueError("sieve windows are limited to 2^32")
    d = _device.device(dev)
    lo = max(lo, 2)
    if lo >= hi:
        return torch.empty(0, dtype=torch.uint32, device=d)
    L = _lib.load()
    fn = "rsa_safe_prime_scan_mr" if literal_mr else "rsa_safe_prime_scan"
    scratch_bytes = int(getattr(L, fn + "_scratch_bytes")(lo, hi))
    scratch = torch.empty(max(scratch_bytes, 16), dtype=torch.uint8, device=d)
    count = torch.zeros(1, dtype=torch.uint64, device=d)
    # capacity: the density of safe primes never exceeds 1 per 12 candidates
    # (+2 for 5 and 7); the 2^31..2^32 census is far below that
    cap = (hi - lo) // 12 + 4 if hi - lo < (1 << 26) else int(1.1 * SAFE_PRIME_CENSUS * (hi - lo) / (1 << 31)) + 4096
    out = torch.empty(cap, dtype=torch.uint32, device=d)
    rc = getattr(L, fn)(lo, hi, out.data_ptr(), cap, count.data_ptr(), scratch.data_ptr(),
                        scratch_bytes, _device.stream(d))
    _lib.check(rc, fn)
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
    """The safe prime of ordinal k (0-based) among those in [lo, hi)."""
    if hi <= lo:
        raise ValueError("empty range: need lo < hi")
    if k < 0:
        raise ValueError("ordinal must be >= 0")
    if hi > 2 ** 32:
        raise NotImplementedError("the device scan covers [0, 2^32)")
    step = 1 << 24      # scan only as far as the ordinal needs
    before = 0
    for a in range(lo, hi, step):
        chunk = safe_primes_u32(a, min(a + step, hi), dev)
        if k < before + chunk.numel():
            return int(chunk[k - before].item())
        before += chunk.numel()
    raise NotFound(f"only {before} safe primes in [{lo}, {hi}), no ordinal {k}")


def safe_prime_index(sp: torch.Tensor) -> torch.Tensor:
    """Bucket index of a sorted device u32 table (rsa_safe_prime_index):
    index[b] = number of entries below b*2^SP_INDEX_SHIFT, b = 0..2^(32-SP_INDEX_SHIFT)."""
    idx = torch.empty(SP_INDEX_LEN, dtype=torch.int32, device=sp.device)
    _lib.call("rsa_safe_prime_index", sp.data_ptr(), int(sp.numel()), idx.data_ptr(), _device.stream(sp.device))
    return idx


SP_INDEX_SHIFT = 12                          # include/rsarand_b200.h RSA_SP_INDEX_SHIFT
SP_INDEX_LEN = (1 << (32 - SP_INDEX_SHIFT)) + 1


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
    """(p1, p2) with p2 the 32-bit safe prime closest to floor(q / p1) (the
    smaller on a tie), p2 != p1 and |p1 p2 - q| <= tol q."""
    if p1 <= 2 ** 31 or p1 >= 2 ** 32 or not numtheory.is_safe_prime(p1):
        raise ValueError(f"p1={p1} is not a 32-bit safe prime")
    if not 0 < q < 2 ** 64:
        raise NotImplementedError("q must fit in 64 bits")
    limit = tolerance_int(tol, q)
    missing = NotFound(f"no safe prime p2 with |p1*p2 - q| <= {tol}*q for p1={p1}")
    if limit < 0:
        raise missing
    tab = safe_prime_table(dev)
    d = tab.device
    p1_dev = torch.tensor([p1], dtype=torch.int64, device=d).to(torch.uint32)
    p2_dev = torch.zeros(1, dtype=torch.uint32, device=d)
    status = torch.zeros(1, dtype=torch.int32, device=d)
    _lib.call("rsa_find_pair", p1_dev.data_ptr(), 1, q, min(limit, 2 ** 64 - 1), tab.sp.data_ptr(),
              tab.n_sp, tab.index.data_ptr(), p2_dev.data_ptr(), status.data_ptr(), _device.stream(d))
    if int(status.item()):
        raise missing
    return p1, int(p2_dev.to(torch.int64).item())


# ---------------------------------------------------------------------------
# derivation

def _phi(n: int) -> int:
    phi = n
    for p in numtheory.factor64(n).distinct_primes():
        phi = phi // p * (p - 1)
    return phi


@functools.lru_cache(maxsize=8)
def _index_space(n_a: int) -> int:
    """S = K_P1 K_P2 n_a, after checking that id -> (t + id SIGMA)^EPSILON
    mod S is a permutation: SIGMA a unit and EPSILON coprime to phi(S)."""
    S = K_P1 * K_P2 * n_a
    radices_prime = numtheory.is_prime64(K_P1) and numtheory.is_prime64(K_P2)
    if not radices_prime:
        raise RuntimeError("K_P1 and K_P2 must be prime")
    if math.gcd(S, SIGMA) > 1:
        raise RuntimeError(f"SIGMA is not a unit modulo the index space {S}")
    if math.gcd(_phi(S), EPSILON) > 1:
        raise RuntimeError(f"x -> x^{EPSILON} does not permute Z_{S}")
    return S


def stream_indices(key: StreamKey, n_a: int = len(MULTIPLIER_TABLE)) -> tuple[int, int]:
    """(p1 ordinal, multiplier index) of a stream: beta = (t + id SIGMA)^EPSILON
    mod S, ordinal = beta mod K_P1, index = floor(beta / (K_P1 K_P2)) mod n_a."""
    S = _index_space(n_a)
    beta = pow((key.master_seed + key.stream_id * SIGMA) % S, EPSILON, S)
    upper, ordinal = divmod(beta, K_P1)
    return ordinal, (upper // K_P2) % n_a


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
    """GeneratorParams of one stream.  The device picks (p1, p2) from the
    stream's ordinal (advancing at most MAX_STEPS ordinals); the host then
    builds and validates the params with make_params and, if that rejects the
    pair, resumes the device search one ordinal further."""
    if len(multiplier_table) == 0:
        raise ValueError("multiplier table must be non-empty")
    n_a = len(multiplier_table)
    ordinal, a_index = stream_indices(key, n_a)
    skip = SkipParams.create(multiplier_table[a_index] if multiplier is None else multiplier)
    exhausted = DerivationExhausted(f"no valid parameters within {MAX_STEPS} ordinals of {ordinal}")
    if not _exponent_usable(e):  # negative keys reduce mod S like the reference's (paramfactory.py:249)
        raise exhausted
    step = 0
    while step < MAX_STEPS:
        cfg = _setup_config(key.master_seed, 0, e, n_a, skip.a, step)
        cfg.first_id = key.stream_id % _index_space(n_a)   # ids enter only through id*SIGMA mod S
        found = _run_setup(cfg, 1, tuple(multiplier_table), dev)
        if int(found.status[0].item()):
            break
        rec = found.records()[0]
        try:
            return rsacore.make_params(int(rec["p1"]), int(rec["p2"]), e, skip,
                                       skip_mode=skip_mode, skip_const=skip_const)
        except rsacore.InvalidParams:
            step = int(found.steps[0].item()) + 1
    raise exhausted
