"""One generator stream: parameters, their validation, and the scalar API.

The public surface is the reference `rsarand.rsacore` (GeneratorParams,
GeneratorState, make_params, validate_params, init, next_raw / next_f64 /
take_raws / take_floats, decrypt, jump_periods, snapshot / restore and the
text checkpoint; rsacore.py:21-417) with the same exception classes.  The
host part is exact integer bookkeeping done once per stream; every draw is a
GPU call (rsa_fill, or rsa_fill_segmented for long runs) on a one-lane
state, so the scalar stream is the Mv = 1 case of the lane kernels.
"""

from __future__ import annotations

import functools
from collections import OrderedDict
import math
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib, numtheory
from .skipgen import Q_DEFAULT, Q_DEFAULT_FACTORS, SkipParams, default_skip_params
from .skipgen import next_skip  # noqa: F401  (re-exported as in rsacore.py of the reference)

DEFAULT_EXPONENT = 9
MAX_EXPONENT = 257
SKIP_LCG, SKIP_UNIT, SKIP_CONST = "lcg", "unit", "const"
SKIP_MODES = (SKIP_LCG, SKIP_UNIT, SKIP_CONST)
MAX_BELOW_ONE = math.nextafter(1.0, 0.0)      # the largest double below 1: the clamp value

_MODE_CODE = {SKIP_LCG: _lib.RSA_SKIP_LCG, SKIP_UNIT: _lib.RSA_SKIP_UNIT, SKIP_CONST: _lib.RSA_SKIP_CONST}


class InvalidParams(ValueError):
    """Parameters break an invariant of the generator."""


class InvalidSeed(ValueError):
    """The skip seed is 0 modulo q."""


class UnsupportedSkipMode(RuntimeError):
    """The operation exists only for the lcg skip."""


class MalformedSnapshot(ValueError):
    """A checkpoint text cannot be parsed or fails validation."""


@dataclass(frozen=True)
class GeneratorParams:
    p1: int
    p2: int
    n: int
    e: int
    skip: SkipParams
    p2inv: int                    # p2^-1 mod p1 (Garner)
    b: int                        # q (q - 1) / 2 mod n: the message advance of one skip period
    skip_mode: str = SKIP_LCG
    skip_const: int = 0
    test_mode: bool = False
    n_float: float = 0.0          # float(n), the float map's divisor


@dataclass
class GeneratorState:
    m1: int                       # message mod p1
    m2: int                       # message mod p2
    s: int                        # skip register
    draws: int = 0


def make_params(p1: int, p2: int, e: int = DEFAULT_EXPONENT, skip: SkipParams | None = None,
                skip_mode: str = SKIP_LCG, skip_const: int = 0,
                test_mode: bool = False) -> GeneratorParams:
    """GeneratorParams from the two primes, the exponent and the skip, with
    the derived constants filled in; raises InvalidParams if they do not form
    a valid generator."""
    skip = skip or default_skip_params()
    if p1 == p2:
        raise InvalidParams("p1 == p2: the two primes must differ")
    n = p1 * p2
    try:
        inv = numtheory.modinv(p2, p1)
    except numtheory.NotInvertible as exc:
        raise InvalidParams(f"p2 has no inverse modulo p1 ({exc})") from exc
    q = skip.q
    params = GeneratorParams(p1=p1, p2=p2, n=n, e=e, skip=skip, p2inv=inv, b=(q * (q - 1) // 2) % n,
                             skip_mode=skip_mode, skip_const=skip_const, test_mode=test_mode,
                             n_float=float(n))
    validate_params(params)
    return params


# pure functions of their integers, memoised: streams are re-validated on every init
@functools.lru_cache(maxsize=1 << 14)
def _safe(p: int) -> bool:
    return numtheory.is_safe_prime(p)


@functools.lru_cache(maxsize=1 << 10)
def _prime(q: int) -> bool:
    return numtheory.is_prime64(q)


@functools.lru_cache(maxsize=1 << 12)
def _generator(a: int, q: int) -> bool:
    return numtheory.is_primitive_root(a, q, Q_DEFAULT_FACTORS if q == Q_DEFAULT else None)


def _problems(p: GeneratorParams):
    """Violated invariants, in checking order (cheap structural checks before
    the primality work)."""
    sk, n = p.skip, p.n
    yield p.p1 == p.p2, "p1 == p2: the two primes must differ"
    yield n != p.p1 * p.p2, "n is not p1*p2"
    yield lambda: not _safe(p.p1), f"p1={p.p1} is not a safe prime"
    yield lambda: not _safe(p.p2), f"p2={p.p2} is not a safe prime"
    yield p.e < 1 or not p.e & 1, f"exponent e={p.e} must be odd and positive"
    yield p.e > MAX_EXPONENT, f"exponent e={p.e} exceeds {MAX_EXPONENT}"
    yield lambda: not _prime(sk.q), f"skip modulus q={sk.q} is not prime"
    yield sk.a > sk.q // sk.a, "multiplier a with a*a > q"
    yield (sk.q1, sk.q2) != divmod(sk.q, sk.a), "q1, q2 are not divmod(q, a)"
    yield lambda: not _generator(sk.a, sk.q), f"a={sk.a} does not generate Z_q^*"
    yield math.gcd(n, sk.q) != 1, "n and q share a factor"
    yield math.gcd(n, sk.q - 1) != 1, "n and q-1 share a factor"
    yield p.b != (sk.q * (sk.q - 1) // 2) % n, "period offset b does not match q and n"
    yield p.b == 0, "period offset b is zero"
    yield not (0 < p.p2inv < p.p1 and (p.p2 * p.p2inv) % p.p1 == 1), "p2inv is not p2^-1 mod p1"
    yield p.skip_mode not in SKIP_MODES, f"unknown skip mode {p.skip_mode!r}"
    if p.skip_mode == SKIP_CONST:
        yield not 0 <= p.skip_const < n, "constant skip outside [0, n)"
    else:
        yield p.skip_const != 0, "skip_const is only used in const mode"
    yield p.n_float != float(n), "n_float is not float(n)"
    if not p.test_mode:  # production sizes (rsacore.py:166-181)
        window = range(2 ** 31 + 1, 2 ** 32)
        yield p.p1 not in window, f"p1={p.p1} outside (2^31, 2^32)"
        yield p.p2 not in window, f"p2={p.p2} outside (2^31, 2^32)"
        yield p.e < 3, "production exponent must be at least 3"
        yield math.gcd(p.e, (p.p1 - 1) * (p.p2 - 1)) != 1, f"e={p.e} is not coprime to (p1-1)(p2-1)"
        yield sk.a < 2 ** 31, f"weak multiplier a={sk.a} needs test_mode"
        yield abs(n - sk.q) > 1e-6 * sk.q, "|n - q| exceeds one part in 10^6"


def validate_params(params: GeneratorParams) -> None:
    """Raise InvalidParams for the first violated invariant."""
    for bad, why in _problems(params):
        if bad() if callable(bad) else bad:
            raise InvalidParams(why)


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
    r["skip_const"] = params.skip_const
    return rec


@functools.lru_cache(maxsize=256)
def _device_instance_cached(params: GeneratorParams, dev_index: int) -> torch.Tensor:
    rec = _instance_record(params)
    return torch.from_numpy(rec.view(np.uint8).copy()).to(torch.device("cuda", dev_index))


# identity-keyed front caches: hashing a frozen GeneratorParams costs ~1 us
# per lookup, a per-take cost on the launch path.  Each entry holds the params
# object itself, so its id cannot be reused while the entry lives.
_BY_ID: "OrderedDict[tuple, tuple]" = OrderedDict()
_BY_ID_MAX = 256


def _by_id(kind: str, params: GeneratorParams, idx, make):
    key = (kind, id(params), idx)
    hit = _BY_ID.get(key)
    if hit is not None and hit[0] is params:
        return hit[1]
    val = make()
    _BY_ID[key] = (params, val)
    if len(_BY_ID) > _BY_ID_MAX:
        _BY_ID.popitem(last=False)
    return val


def device_instance(params: GeneratorParams, dev=None) -> torch.Tensor:
    """128-byte rsa_instance on the device for one stream."""
    d = _device.device(dev)
    return _by_id("inst", params, d.index, lambda: _device_instance_cached(params, d.index))


@functools.lru_cache(maxsize=256)
def _instance_flags(params: GeneratorParams) -> int:
    return int(_instance_record(params)[0]["flags"])


def instance_flags(params: GeneratorParams) -> int:
    return _by_id("flags", params, None, lambda: _instance_flags(params))


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
    """State at draw 0: message m0 (as residues) and skip seed s0 (the const
    mode's register holds skip_const instead)."""
    validate_params(params)
    if min(m0, s0) < 0:
        raise InvalidSeed("seeds must be nonnegative")
    if params.skip_mode == SKIP_CONST:
        return GeneratorState(m1=m0 % params.p1, m2=m0 % params.p2, s=params.skip_const)
    s = s0 % params.skip.q
    if not s:
        raise InvalidSeed(f"s0={s0} is a multiple of q")
    return GeneratorState(m1=m0 % params.p1, m2=m0 % params.p2, s=s)


def _scalar_run(state: GeneratorState, params: GeneratorParams, count: int, raw: bool, f64: bool,
                dev=None) -> np.ndarray:
    """count draws of the one-lane stream on the GPU; returns the host array
    (uint64 ciphertexts, or float64) and advances `state`.  One H2D of the
    3-word state and one D2H of state + outputs: a single round trip."""
    d = _device.device(dev)
    inst = device_instance(params, d)
    s_in = 1 if params.skip_mode == SKIP_UNIT else state.s
    n_out = count if (raw or f64) else 0
    # uint64 words carried bit-for-bit in an int64 tensor (a const skip may exceed 2^63)
    buf = torch.empty(3 + n_out, dtype=torch.int64, device=d)
    buf[:3].copy_(torch.from_numpy(np.array([state.m1, state.m2, s_in], dtype=np.uint64).view(np.int64)))
    ptr = buf.data_ptr()
    m1, m2, s = ptr, ptr + 8, ptr + 16
    out = ptr + 24 if n_out else None
    if count:
        flags = instance_flags(params)
        args = (inst.data_ptr(), 1, 1, count, params.e, flags, m1, m2, s,
                out if raw else None, out if f64 else None, count)
        L = _lib.load()
        if flags & _lib.RSA_FLAG_FAST and (raw or f64) and int(L.rsa_fill_segments(1, count)) > 1:
            # one lane, many draws: split it across threads (K1s, bit-identical)
            nb = int(L.rsa_fill_segmented_scratch_bytes(1, count))
            scratch = torch.empty(nb, dtype=torch.uint8, device=d)
            _lib.call("rsa_fill_segmented", *args, scratch.data_ptr(), nb, _device.stream(d))
        else:
            _lib.call("rsa_fill", *args, _device.stream(d))
    host = buf.cpu().numpy().view(np.uint64)
    new = host[:3].tolist()
    state.m1, state.m2 = new[0], new[1]
    if params.skip_mode == SKIP_LCG or (params.skip_mode == SKIP_UNIT and count):
        state.s = new[2]
    state.draws += count
    body = host[3:]
    return body.view(np.float64) if f64 else body


# Single draws are served from a per-state look-ahead buffer that one GPU call
# (rsa_scalar_lookahead) fills with the next LOOKAHEAD draws and the state
# after each of them, so next_raw / next_f64 cost a buffer read instead of a
# GPU round trip while the state's fields stay exactly the reference's after
# every draw.  The buffer is tied to the state it was made from: any other
# change to the state (take_raws, jump_periods, direct assignment) or a
# different params object makes it refill.
LOOKAHEAD = 512


class _Lookahead:
    __slots__ = ("params", "raw", "f64", "s", "m1", "m2", "pos", "expect")


# Look-ahead buffers live beside the states, keyed by id(state) and dropped
# when the state is collected: vars(state) stays the reference's four fields,
# and copy / deepcopy / pickle of a state carry no buffer (a copy refills).
_LOOKAHEADS: dict[int, _Lookahead] = {}


def _lookahead_of(state: GeneratorState):
    return _LOOKAHEADS.get(id(state))


def _attach_lookahead(state: GeneratorState, lk: _Lookahead) -> None:
    key = id(state)
    if key not in _LOOKAHEADS:
        weakref.finalize(state, _LOOKAHEADS.pop, key, None)
    _LOOKAHEADS[key] = lk


def _lookahead_draw(state: GeneratorState, params: GeneratorParams, peek: bool = False):
    """Serve the next draw from the state's look-ahead buffer (refilling it if
    it does not continue this state); None when the instance has no fast
    kernel.  peek=True only answers whether the buffer can serve."""
    if peek:
        return params.skip_mode == SKIP_LCG and bool(instance_flags(params) & _lib.RSA_FLAG_FAST)
    lk = _lookahead_of(state)
    if (lk is None or lk.pos >= LOOKAHEAD or (lk.params is not params and lk.params != params)
            or lk.expect != (state.m1, state.m2, state.s, state.draws)):
        if params.skip_mode != SKIP_LCG or not instance_flags(params) & _lib.RSA_FLAG_FAST:
            return None
        d = _device.device(None)
        inst = device_instance(params, d)
        buf = torch.empty(LOOKAHEAD * 32, dtype=torch.uint8, device=d)
        _lib.call("rsa_scalar_lookahead", inst.data_ptr(), state.m1, state.m2, state.s, params.e,
                  instance_flags(params), LOOKAHEAD, buf.data_ptr(), _device.stream(d))
        host = buf.cpu().numpy()
        n = LOOKAHEAD
        lk = _Lookahead()
        lk.params = params
        lk.raw = host[:8 * n].view(np.uint64).tolist()
        lk.f64 = host[8 * n:16 * n].view(np.float64).tolist()
        lk.s = host[16 * n:24 * n].view(np.uint64).tolist()
        lk.m1 = host[24 * n:28 * n].view(np.uint32).tolist()
        lk.m2 = host[28 * n:32 * n].view(np.uint32).tolist()
        lk.pos = 0
        _attach_lookahead(state, lk)
    i = lk.pos
    lk.pos = i + 1
    state.m1, state.m2, state.s = lk.m1[i], lk.m2[i], lk.s[i]
    state.draws += 1
    lk.expect = (state.m1, state.m2, state.s, state.draws)
    return lk, i


def next_raw(state: GeneratorState, params: GeneratorParams) -> int:
    """Advance one step; the raw ciphertext c in [0, n) (rsacore.py:213-226)."""
    hit = _lookahead_draw(state, params)
    if hit is None:
        return take_raws(state, params, 1)[0]
    return hit[0].raw[hit[1]]


def next_f64(state: GeneratorState, params: GeneratorParams) -> float:
    """Next double in [0, 1) (rsacore.py:229-233)."""
    hit = _lookahead_draw(state, params)
    if hit is None:
        return take_floats(state, params, 1)[0]
    return hit[0].f64[hit[1]]


_SMALL_TAKE = 64  # takes up to this size are served from the look-ahead buffer


def take_raws(state: GeneratorState, params: GeneratorParams, count: int) -> list[int]:
    """count sequential raw draws (rsacore.py:236-258)."""
    if 0 < count <= _SMALL_TAKE and _lookahead_draw(state, params, peek=True):
        return [next_raw(state, params) for _ in range(count)]
    return _scalar_run(state, params, count, True, False).tolist()


def take_floats(state: GeneratorState, params: GeneratorParams, count: int) -> list[float]:
    """count sequential next_f64 draws (rsacore.py:261-264)."""
    if 0 < count <= _SMALL_TAKE and _lookahead_draw(state, params, peek=True):
        return [next_f64(state, params) for _ in range(count)]
    return _scalar_run(state, params, count, False, True).tolist()


def decrypt(c: int, params: GeneratorParams) -> int:
    """Invert the cipher: c^d mod n with d = e^-1 mod (p1-1)(p2-1)."""
    phi = (params.p1 - 1) * (params.p2 - 1)
    return pow(c, numtheory.modinv(params.e, phi), params.n)


def jump_periods(state: GeneratorState, params: GeneratorParams, u: int) -> GeneratorState:
    """Skip u whole periods of the skip sequence (u (q - 1) draws) at once:
    the skip returns to itself and the message gains u b."""
    if params.skip_mode != SKIP_LCG:
        raise UnsupportedSkipMode(f"jump_periods needs the lcg skip, not {params.skip_mode}")
    gain = u * params.b
    state.m1 = (state.m1 + gain) % params.p1
    state.m2 = (state.m2 + gain) % params.p2
    state.draws += u * (params.skip.q - 1)
    return state


# text checkpoints live in _snaptext (the reference's formats, byte for byte)
from ._snaptext import (PARAMS_HEADER, SNAPSHOT_HEADER, StreamSnapshot,  # noqa: E402,F401
                        params_from_text, params_lines, params_to_text, restore, snapshot)
