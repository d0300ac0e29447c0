"""Generator parameters, validation and the scalar stream API.

Mirrors /root/reference/pkg/src/rsarand/rsacore.py: same names, fields,
exceptions and error messages.  Parameter construction and validation are
host-side (exact Python ints, once per stream, as in the reference); every
draw runs on the GPU through the C ABI (rsa_fill with one lane), so the
scalar API is the Mv = 1 case of the lane kernels.
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib, numtheory
from .skipgen import Q_DEFAULT, SkipParams, default_skip_params

DEFAULT_EXPONENT = 9          # rsacore.py:21
MAX_EXPONENT = 257            # rsacore.py:22

SKIP_LCG = "lcg"              # rsacore.py:24-27
SKIP_UNIT = "unit"
SKIP_CONST = "const"
SKIP_MODES = (SKIP_LCG, SKIP_UNIT, SKIP_CONST)

MAX_BELOW_ONE = math.nextafter(1.0, 0.0)   # rsacore.py:30

SNAPSHOT_HEADER = "rsarand-snapshot-v1"
PARAMS_HEADER = "rsarand-params-v1"
_PARAM_FIELDS = ("p1", "p2", "n", "e", "q", "a", "q1", "q2", "p2inv", "b",
                 "skip_mode", "skip_const", "test_mode")
_STATE_FIELDS = ("m1", "m2", "s", "draws")

_MODE_CODE = {SKIP_LCG: _lib.RSA_SKIP_LCG, SKIP_UNIT: _lib.RSA_SKIP_UNIT,
              SKIP_CONST: _lib.RSA_SKIP_CONST}


class InvalidParams(ValueError):
    """A generator-parameter invariant is violated (rsacore.py:40-41)."""


class InvalidSeed(ValueError):
    """Seed skip s0 is congruent to 0 mod q (rsacore.py:44-45)."""


class UnsupportedSkipMode(RuntimeError):
    """Operation defined only for the lcg skip mode (rsacore.py:48-49)."""


class MalformedSnapshot(ValueError):
    """Snapshot text is missing fields or violates an invariant (rsacore.py:52-53)."""


@dataclass(frozen=True)
class GeneratorParams:
    """Per-stream constants (rsacore.py:56-76)."""

    p1: int
    p2: int
    n: int
    e: int
    skip: SkipParams
    p2inv: int
    b: int
    skip_mode: str = SKIP_LCG
    skip_const: int = 0
    test_mode: bool = False
    n_float: float = 0.0


@dataclass
class GeneratorState:
    """Scalar stream state (rsacore.py:79-86)."""

    m1: int
    m2: int
    s: int
    draws: int = 0


def make_params(p1: int, p2: int, e: int = DEFAULT_EXPONENT, skip: SkipParams | None = None,
                skip_mode: str = SKIP_LCG, skip_const: int = 0,
                test_mode: bool = False) -> GeneratorParams:
    """Build and validate GeneratorParams (rsacore.py:89-107)."""
    if skip is None:
        skip = default_skip_params()
    if p1 == p2:
        raise InvalidParams("p1 == p2")
    n = p1 * p2
    try:
        p2inv = numtheory.modinv(p2, p1)
    except numtheory.NotInvertible as exc:
        raise InvalidParams(f"p2 not invertible mod p1: {exc}") from exc
    params = GeneratorParams(p1=p1, p2=p2, n=n, e=e, skip=skip, p2inv=p2inv,
                             b=skip.q * (skip.q - 1) // 2 % n, skip_mode=skip_mode,
                             skip_const=skip_const, test_mode=test_mode, n_float=float(n))
    validate_params(params)
    return params


def _root_factors(q: int):
    from .skipgen import Q_DEFAULT_FACTORS
    return Q_DEFAULT_FACTORS if q == Q_DEFAULT else None


# The number-theoretic checks are pure functions of their integers; streams are
# re-validated on every init / init_vector, so they are memoised.
@functools.lru_cache(maxsize=1 << 14)
def _is_safe_prime(p: int) -> bool:
    return numtheory.is_safe_prime(p)


@functools.lru_cache(maxsize=1 << 10)
def _is_prime64(q: int) -> bool:
    return numtheory.is_prime64(q)


@functools.lru_cache(maxsize=1 << 12)
def _is_primitive_root(a: int, q: int) -> bool:
    return numtheory.is_primitive_root(a, q, _root_factors(q))


def validate_params(params: GeneratorParams) -> None:
    """Raise InvalidParams naming the first violated invariant (rsacore.py:117-181)."""
    p1, p2, n, e, sk = params.p1, params.p2, params.n, params.e, params.skip
    checks = (
        (p1 == p2, "p1 == p2"),
        (n != p1 * p2, "n != p1*p2"),
        (lambda: not _is_safe_prime(p1), f"p1={p1} is not a safe prime"),
        (lambda: not _is_safe_prime(p2), f"p2={p2} is not a safe prime"),
        (e < 1 or e % 2 == 0, f"exponent e={e} must be odd and positive"),
        (e > MAX_EXPONENT, f"exponent e={e} above {MAX_EXPONENT}"),
        (lambda: not _is_prime64(sk.q), f"q={sk.q} is not prime"),
        (sk.a * sk.a > sk.q, "multiplier violates a*a <= q"),
        (sk.q1 != sk.q // sk.a or sk.q2 != sk.q % sk.a, "inconsistent Schrage constants q1/q2"),
        (lambda: not _is_primitive_root(sk.a, sk.q), f"a={sk.a} is not a primitive root mod q"),
        (math.gcd(n, sk.q) != 1, "gcd(n, q) != 1"),
        (math.gcd(n, sk.q - 1) != 1, "gcd(n, q-1) != 1"),
        (params.b != sk.q * (sk.q - 1) // 2 % n, "inconsistent period offset b"),
        (params.b == 0, "period offset b is zero"),
        (params.p2inv <= 0 or params.p2inv >= p1 or p2 * params.p2inv % p1 != 1,
         "p2inv is not the inverse of p2 mod p1"),
        (params.skip_mode not in SKIP_MODES, f"unknown skip mode {params.skip_mode!r}"),
    )
    for bad, msg in checks:
        if bad() if callable(bad) else bad:
            raise InvalidParams(msg)
    if params.skip_mode == SKIP_CONST:
        if not 0 <= params.skip_const < n:
            raise InvalidParams("constant skip outside [0, n)")
    elif params.skip_const != 0:
        raise InvalidParams("skip_const must be 0 outside const mode")
    if params.n_float != float(n):
        raise InvalidParams("inconsistent cached n_float")
    if params.test_mode:
        return
    prod = (
        (not (1 << 31) < p1 < (1 << 32), f"p1={p1} outside (2^31, 2^32)"),
        (not (1 << 31) < p2 < (1 << 32), f"p2={p2} outside (2^31, 2^32)"),
        (e < 3, "production exponent must be >= 3"),
        (math.gcd(e, (p1 - 1) * (p2 - 1)) != 1, f"gcd(e, (p1-1)(p2-1)) != 1 for e={e}"),
        (sk.a < (1 << 31), f"weak multiplier a={sk.a} requires test_mode"),
        (abs(n - sk.q) > 1e-6 * sk.q, "|n - q| exceeds one part in 10^6"),
    )
    for bad, msg in prod:
        if bad:
            raise InvalidParams(msg)


# ---------------------------------------------------------------------------
# device instance packing (the host twin of csrc/setup.cu:build_instance)

def _instance_record(params: GeneratorParams) -> np.ndarray:
    p1, p2, e, sk = params.p1, params.p2, params.e, params.skip
    if not (2 < p1 < 1 << 32 and 2 < p2 < 1 << 32) or p1 % 2 == 0 or p2 % 2 == 0:
        raise InvalidParams("the CUDA kernels need odd primes below 2^32")
    if not 0 < e < 1 << 31 or sk.q >= 1 << 64 or sk.a >= 1 << 32:
        raise InvalidParams("parameters exceed the CUDA kernels' 64-bit ranges")
    R = 1 << 32
    rec = np.zeros(1, dtype=_lib.INSTANCE_DTYPE)
    r = rec[0]
    r["p1"], r["p2"] = p1, p2
    r["p1_inv"], r["p2_inv"] = pow(p1, -1, R), pow(p2, -1, R)
    r["a"], r["e"] = sk.a, e
    r["k1"], r["k2"] = pow(R, 2 * e, p1), pow(R, 2 * e, p2)
    r["r2_1"], r["r2_2"] = R * R % p1, R * R % p2
    r["garner"], r["p2inv"] = params.p2inv * R % p1, params.p2inv
    r["q1"], r["q2"] = sk.q1 & 0xFFFFFFFF, sk.q2 & 0xFFFFFFFF
    fast = (sk.q == Q_DEFAULT and params.skip_mode == SKIP_LCG
            and (1 << 31) < p1 < R and (1 << 31) < p2 < R)
    r["flags"] = (_lib.RSA_FLAG_FAST if fast else 0) | (
        _lib.RSA_FLAG_FIXED if params.skip_mode != SKIP_LCG else 0)
    r["skip_mode"] = _MODE_CODE[params.skip_mode]
    r["n"], r["q"], r["b"] = params.n, sk.q, params.b
    r["n_float"] = float(params.n)
    r["n_recip"] = 1.0 / float(params.n)
    r["n_recip_lo"] = recip_lo(r["n_float"], r["n_recip"])
    r["skip_const"] = params.skip_const
    return rec


def recip_lo(nf: float, y: float) -> float:
    """RN(RN(1 - nf*y) * y) with the inner residual exact (as the device's
    fma(-nf, y, 1) computes it): the low half of 1/nf ~ y + y_lo."""
    from fractions import Fraction
    e = float(1 - Fraction(nf) * Fraction(y))       # exactly representable
    return float(Fraction(e) * Fraction(y))          # single rounding


@functools.lru_cache(maxsize=256)
def _device_instance_cached(params: GeneratorParams, dev_index: int) -> torch.Tensor:
    rec = _instance_record(params)
    return torch.from_numpy(rec.view(np.uint8).copy()).to(torch.device("cuda", dev_index))


def device_instance(params: GeneratorParams, dev=None) -> torch.Tensor:
    """128-byte rsa_instance on the device for one stream."""
    d = _device.device(dev)
    return _device_instance_cached(params, d.index)


def instance_flags(params: GeneratorParams) -> int:
    return int(_instance_record(params)[0]["flags"])


def skip_only_instance(skip: SkipParams, dev=None) -> torch.Tensor:
    """An rsa_instance carrying only (q, a) — for lane-seed computation."""
    rec = np.zeros(1, dtype=_lib.INSTANCE_DTYPE)
    rec[0]["p1"], rec[0]["p2"], rec[0]["a"], rec[0]["q"] = 3, 5, skip.a, skip.q
    rec[0]["skip_mode"] = _lib.RSA_SKIP_LCG
    d = _device.device(dev)
    return torch.from_numpy(rec.view(np.uint8).copy()).to(d)


# ---------------------------------------------------------------------------
# scalar stream (rsacore.py:189-264) — the Mv = 1 lane on the GPU

def init(params: GeneratorParams, m0: int = 0, s0: int = 1) -> GeneratorState:
    """Fresh stream state (rsacore.py:189-204)."""
    validate_params(params)
    if m0 < 0 or s0 < 0:
        raise InvalidSeed("seeds must be nonnegative")
    if params.skip_mode == SKIP_CONST:
        s = params.skip_const
    else:
        s = s0 % params.skip.q
        if s == 0:
            raise InvalidSeed(f"s0={s0} is divisible by q")
    return GeneratorState(m1=m0 % params.p1, m2=m0 % params.p2, s=s)


def _scalar_run(state: GeneratorState, params: GeneratorParams, count: int, raw: bool, f64: bool,
                dev=None):
    d = _device.device(dev)
    inst = device_instance(params, d)
    s_in = 1 if params.skip_mode == SKIP_UNIT else state.s
    st = _device.u64([state.m1, state.m2, s_in], d)
    m1, m2, s = st[0:1], st[1:2], st[2:3]
    out_raw = torch.empty(count, dtype=torch.uint64, device=d) if raw else None
    out_f64 = torch.empty(count, dtype=torch.float64, device=d) if f64 else None
    if count:
        flags = instance_flags(params)
        args = (inst.data_ptr(), 1, 1, count, params.e, flags, m1.data_ptr(), m2.data_ptr(), s.data_ptr(),
                out_raw.data_ptr() if raw else None, out_f64.data_ptr() if f64 else None, count)
        L = _lib.load()
        if flags & _lib.RSA_FLAG_FAST and (raw or f64) and int(L.rsa_fill_segments(1, count)) > 1:
            # one lane, many draws: split it across threads (K1s, bit-identical)
            nb = int(L.rsa_fill_segmented_scratch_bytes(1, count))
            scratch = torch.empty(nb, dtype=torch.uint8, device=d)
            _lib.call("rsa_fill_segmented", *args, scratch.data_ptr(), nb, _device.stream(d))
        else:
            _lib.call("rsa_fill", *args, _device.stream(d))
    new = _device.to_ints(st)
    state.m1, state.m2 = new[0], new[1]
    if params.skip_mode == SKIP_LCG or (params.skip_mode == SKIP_UNIT and count):
        state.s = new[2]
    state.draws += count
    return out_raw, out_f64


def next_raw(state: GeneratorState, params: GeneratorParams) -> int:
    """Advance one step; the raw ciphertext c in [0, n) (rsacore.py:213-226)."""
    return take_raws(state, params, 1)[0]


def next_f64(state: GeneratorState, params: GeneratorParams) -> float:
    """Next double in [0, 1) (rsacore.py:229-233)."""
    return take_floats(state, params, 1)[0]


def take_raws(state: GeneratorState, params: GeneratorParams, count: int) -> list[int]:
    """count sequential raw draws (rsacore.py:236-258)."""
    raw, _ = _scalar_run(state, params, count, True, False)
    return _device.to_ints(raw)


def take_floats(state: GeneratorState, params: GeneratorParams, count: int) -> list[float]:
    """count sequential next_f64 draws (rsacore.py:261-264)."""
    _, f = _scalar_run(state, params, count, False, True)
    return f.cpu().numpy().tolist()


def decrypt(c: int, params: GeneratorParams) -> int:
    """c^d mod n, d = e^-1 mod (p1-1)(p2-1): validation hook (rsacore.py:267-273)."""
    d = numtheory.modinv(params.e, (params.p1 - 1) * (params.p2 - 1))
    return pow(c, d, params.n)


def jump_periods(state: GeneratorState, params: GeneratorParams, u: int) -> GeneratorState:
    """Advance u full skip periods (u*(q-1) draws) in O(1) (rsacore.py:276-289)."""
    if params.skip_mode != SKIP_LCG:
        raise UnsupportedSkipMode(f"jump_periods undefined for {params.skip_mode} mode")
    ub = u * params.b
    state.m1 = (state.m1 + ub) % params.p1
    state.m2 = (state.m2 + ub) % params.p2
    state.draws += u * (params.skip.q - 1)
    return state


# ---------------------------------------------------------------------------
# snapshot text format (rsacore.py:292-417)

@dataclass(frozen=True)
class StreamSnapshot:
    params: GeneratorParams
    m1: int
    m2: int
    s: int
    draws: int

    def to_text(self) -> str:
        body = [SNAPSHOT_HEADER, *params_lines(self.params)]
        body += [f"{k}={getattr(self, k):x}" for k in _STATE_FIELDS]
        return "\n".join(body) + "\n"

    @classmethod
    def from_text(cls, text: str) -> "StreamSnapshot":
        f = _parse_kv(text, SNAPSHOT_HEADER, set(_PARAM_FIELDS) | set(_STATE_FIELDS))
        return cls(params=_params_from_fields(f), m1=_hex(f, "m1"), m2=_hex(f, "m2"),
                   s=_hex(f, "s"), draws=_hex(f, "draws"))


def _parse_kv(text: str, header: str, expected: set) -> dict:
    lines = [ln.strip() for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != header:
        raise MalformedSnapshot(f"missing or unknown header (want {header!r})")
    out: dict = {}
    for ln in lines[1:]:
        key, sep, val = ln.partition("=")
        if not sep or key in out:
            raise MalformedSnapshot(f"bad line {ln!r}")
        out[key] = val
    if set(out) != expected:
        raise MalformedSnapshot(f"missing={sorted(expected - set(out))} "
                                f"unknown={sorted(set(out) - expected)}")
    return out


def _hex(f: dict, key: str) -> int:
    try:
        return int(f[key], 16)
    except ValueError as exc:
        raise MalformedSnapshot(f"field {key} is not hex: {f[key]!r}") from exc


def _params_from_fields(f: dict) -> GeneratorParams:
    skip = SkipParams(q=_hex(f, "q"), a=_hex(f, "a"), q1=_hex(f, "q1"), q2=_hex(f, "q2"))
    n = _hex(f, "n")
    return GeneratorParams(p1=_hex(f, "p1"), p2=_hex(f, "p2"), n=n, e=_hex(f, "e"), skip=skip,
                           p2inv=_hex(f, "p2inv"), b=_hex(f, "b"), skip_mode=f["skip_mode"],
                           skip_const=_hex(f, "skip_const"), test_mode=bool(_hex(f, "test_mode")),
                           n_float=float(n))


def params_lines(params: GeneratorParams) -> list[str]:
    vals = {"p1": params.p1, "p2": params.p2, "n": params.n, "e": params.e, "q": params.skip.q,
            "a": params.skip.a, "q1": params.skip.q1, "q2": params.skip.q2, "p2inv": params.p2inv,
            "b": params.b, "skip_const": params.skip_const, "test_mode": int(params.test_mode)}
    return [f"skip_mode={params.skip_mode}" if k == "skip_mode" else f"{k}={vals[k]:x}"
            for k in _PARAM_FIELDS]


def params_to_text(params: GeneratorParams) -> str:
    return "\n".join([PARAMS_HEADER, *params_lines(params)]) + "\n"


def params_from_text(text: str) -> GeneratorParams:
    params = _params_from_fields(_parse_kv(text, PARAMS_HEADER, set(_PARAM_FIELDS)))
    try:
        validate_params(params)
    except InvalidParams as exc:
        raise MalformedSnapshot(f"exported params invalid: {exc}") from exc
    return params


def snapshot(state: GeneratorState, params: GeneratorParams) -> StreamSnapshot:
    return StreamSnapshot(params=params, m1=state.m1, m2=state.m2, s=state.s, draws=state.draws)


def restore(snap) -> tuple[GeneratorParams, GeneratorState]:
    """Rebuild (params, state), re-validating everything (rsacore.py:393-417)."""
    if isinstance(snap, str):
        snap = StreamSnapshot.from_text(snap)
    params = snap.params
    try:
        validate_params(params)
    except InvalidParams as exc:
        raise MalformedSnapshot(f"snapshot params invalid: {exc}") from exc
    if not 0 <= snap.m1 < params.p1:
        raise MalformedSnapshot("m1 outside [0, p1)")
    if not 0 <= snap.m2 < params.p2:
        raise MalformedSnapshot("m2 outside [0, p2)")
    if params.skip_mode == SKIP_CONST:
        if snap.s != params.skip_const:
            raise MalformedSnapshot("const-mode skip register mismatch")
    elif not 1 <= snap.s < params.skip.q:
        raise MalformedSnapshot("skip outside [1, q)")
    if snap.draws < 0:
        raise MalformedSnapshot("negative draw count")
    return params, GeneratorState(m1=snap.m1, m2=snap.m2, s=snap.s, draws=snap.draws)
