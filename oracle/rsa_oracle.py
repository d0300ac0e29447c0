"""CPU ORACLE — test infrastructure only.

A restatement, in numpy uint64 / Python ints, of the reference algorithm of
/root/reference/pkg/src/rsarand (arXiv 1811.11629).  Only tests/, the
__graft_entry__.smoke() checker and bench.py's cpu_baseline / --impl reference
legs may import this module; the product package never does (it has no CPU
path at all).

Pinned: tests/test_oracle_golden.py checks every function here against the
golden vectors that tests/golden/make_golden.py produced by running the
reference itself (regression draws, per-config streams, safe-prime census,
derived parameter tuples).

Reference map:
  skip_array        skipgen.next_skip_array           skipgen.py:108-116
  pow_lanes         vecgen._pow_lanes                 vecgen.py:72-84
  block_raw         vecgen.next_block_raw             vecgen.py:87-100
  floats_from_raw   vecgen.floats_from_raw            vecgen.py:103-107
  lane_seeds        skipgen.lane_offset_seeds         skipgen.py:124-138
  VecState/init     vecgen.init_vector                vecgen.py:44-69
  take_raw          vecgen.take_raw                   vecgen.py:115-139
  scalar_raws       rsacore.take_raws                 rsacore.py:236-258
  stream_indices    paramfactory.stream_indices       paramfactory.py:242-250
  find_pair_sorted  paramfactory.find_pair            paramfactory.py:195-219
  derive            paramfactory.derive_stream_params paramfactory.py:253-278
  fused_reference   (no reference; SURVEY.md §8(c) "Proposed A13 definitions")
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

Q_DEFAULT = (1 << 63) - 25
MAX_BELOW_ONE = math.nextafter(1.0, 0.0)
MULTIPLIER_TABLE = (2358014131, 3027930091, 2663770345, 2989232495, 2966714411, 2517859571,
                    2584241481, 2831318399, 3001167565, 2425226767, 3003776879, 2548386679,
                    2416530305, 2983799827, 2861425803, 2203334683)
DEFAULT_MASTER_SEED = 0x243F6A8885A308D3
SQRT_Q = 3037000499
K_P1, K_P2 = 1_291_831, 1_768_937
SIGMA, EPSILON = 35_705_744_587, 7
U64 = np.uint64


@dataclass(frozen=True)
class Params:
    p1: int
    p2: int
    e: int
    a: int
    q: int = Q_DEFAULT
    mode: str = "lcg"          # lcg | unit | const
    skip_const: int = 0

    @property
    def n(self) -> int:
        return self.p1 * self.p2

    @property
    def q1(self) -> int:
        return self.q // self.a

    @property
    def q2(self) -> int:
        return self.q % self.a

    @property
    def p2inv(self) -> int:
        return pow(self.p2, -1, self.p1)

    @property
    def b(self) -> int:
        return self.q * (self.q - 1) // 2 % self.n

    @property
    def n_float(self) -> float:
        return float(self.n)


def from_fields(d: dict) -> Params:
    """Params from a golden-fixture dict (fields named as GeneratorParams)."""
    return Params(p1=d["p1"], p2=d["p2"], e=d["e"], a=d["a"], q=d["q"], mode=d.get("skip_mode", "lcg"),
                  skip_const=d.get("skip_const", 0))


# ---------------------------------------------------------------------------
# lockstep lanes (numpy uint64, every intermediate < 2^64)

def skip_array(s: np.ndarray, P: Params) -> np.ndarray:
    """a*s mod q by Schrage: hi, lo = divmod(s, q1); a*lo - q2*hi (+q)."""
    hi, lo = np.divmod(s, U64(P.q1))
    s1 = U64(P.a) * lo
    s2 = U64(P.q2) * hi
    return np.where(s1 >= s2, s1 - s2, s1 + U64(P.q) - s2)


def pow_lanes(x: np.ndarray, e: int, p: int) -> np.ndarray:
    """x^e mod p, LSB-first square-and-multiply (operands < 2^32)."""
    pp = U64(p)
    acc = None
    base = x
    while e:
        if e & 1:
            acc = base.copy() if acc is None else acc * base % pp
        e >>= 1
        if e:
            base = base * base % pp
    return acc


def block_raw(m1, m2, s, P: Params):
    """One lockstep step of all lanes; returns (raw, m1', m2', s')."""
    if P.mode == "lcg":
        s = skip_array(s, P)
    p1, p2 = U64(P.p1), U64(P.p2)
    m1 = (m1 + s % p1) % p1
    m2 = (m2 + s % p2) % p2
    c1 = pow_lanes(m1, P.e, P.p1)
    c2 = pow_lanes(m2, P.e, P.p2)
    d = (c1 + p1 - c2 % p1) % p1
    return d * U64(P.p2inv) % p1 * p2 + c2, m1, m2, s


def floats_from_raw(raw: np.ndarray, P: Params) -> np.ndarray:
    return np.minimum(raw.astype(np.float64) / P.n_float, MAX_BELOW_ONE)


def lane_seeds(P: Params, s0: int, mv: int, lanes=None) -> np.ndarray:
    stride = (P.q - 1) // mv
    idx = range(mv) if lanes is None else lanes
    return np.array([s0 * pow(P.a, g * stride, P.q) % P.q for g in idx], dtype=U64)


@dataclass
class VecState:
    P: Params
    mv: int
    m1: np.ndarray
    m2: np.ndarray
    s: np.ndarray
    pending: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=U64))


def init(P: Params, m0: int = 0, s0: int = 1, mv: int = 1, lanes=None) -> VecState:
    """vecgen.init_vector; `lanes` selects a subset of the mv lanes."""
    k = mv if lanes is None else len(lanes)
    if P.mode == "lcg":
        s0 %= P.q
        s = lane_seeds(P, s0, mv, lanes)
        m1 = np.full(k, m0 % P.p1, dtype=U64)
        m2 = np.full(k, m0 % P.p2, dtype=U64)
    else:
        v = 1 if P.mode == "unit" else P.skip_const
        idx = range(mv) if lanes is None else lanes
        lane_m = [(m0 + (g + 1 - mv) * v) % P.n for g in idx]
        m1 = np.array([m % P.p1 for m in lane_m], dtype=U64)
        m2 = np.array([m % P.p2 for m in lane_m], dtype=U64)
        s = np.full(k, mv * v % P.n, dtype=U64)
    return VecState(P, k, m1, m2, s)


def next_block_raw(st: VecState) -> np.ndarray:
    raw, st.m1, st.m2, st.s = block_raw(st.m1, st.m2, st.s, st.P)
    return raw


def take_raw(st: VecState, count: int) -> np.ndarray:
    parts, have = [], 0
    if len(st.pending):
        head = st.pending[:count]
        st.pending = st.pending[len(head):]
        parts.append(head)
        have = len(head)
    while have < count:
        blk = next_block_raw(st)
        need = count - have
        if len(blk) > need:
            parts.append(blk[:need])
            st.pending = blk[need:]
            have = count
        else:
            parts.append(blk)
            have += len(blk)
    return np.concatenate(parts) if parts else np.empty(0, dtype=U64)


def take_floats(st: VecState, count: int) -> np.ndarray:
    return floats_from_raw(take_raw(st, count), st.P)


def blocks_raw(st: VecState, blocks: int) -> np.ndarray:
    """[blocks, lanes] raw matrix."""
    return np.stack([next_block_raw(st) for _ in range(blocks)]) if blocks else np.empty((0, st.mv), U64)


# ---------------------------------------------------------------------------
# scalar stream (pure Python ints — the bit-exactness anchor)

def scalar_raws(P: Params, count: int, m0: int = 0, s0: int = 1) -> list[int]:
    m1, m2 = m0 % P.p1, m0 % P.p2
    s = s0 % P.q if P.mode == "lcg" else (1 if P.mode == "unit" else P.skip_const)
    p2inv = P.p2inv
    out = []
    for _ in range(count):
        if P.mode == "lcg":
            s = P.a * s % P.q
        m1 = (m1 + s) % P.p1
        m2 = (m2 + s) % P.p2
        c2 = pow(m2, P.e, P.p2)
        out.append((pow(m1, P.e, P.p1) + P.p1 - c2 % P.p1) % P.p1 * p2inv % P.p1 * P.p2 + c2)
    return out


# ---------------------------------------------------------------------------
# primes and derivation

def is_prime(n: int) -> bool:
    if n < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0:
            return n == p
    d, u = n - 1, 0
    while d % 2 == 0:
        d //= 2
        u += 1
    for g in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(g, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(u - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def is_safe_prime(p: int) -> bool:
    return p > 4 and is_prime(p) and is_prime((p - 1) // 2)


def stream_indices(seed: int, sid: int, n_a: int = 16) -> tuple[int, int]:
    S = K_P1 * K_P2 * n_a
    beta = pow((seed + sid * SIGMA) % S, EPSILON, S)
    return beta % K_P1, beta // (K_P1 * K_P2) % n_a


def find_pair_sorted(p1: int, sp: np.ndarray, q: int = Q_DEFAULT, tol_int: int = 9223372036854):
    """find_pair over a sorted safe-prime array (same outward order as the
    reference's 12-step scan: nearest to q//p1, ties to the smaller)."""
    target = q // p1
    hi = int(np.searchsorted(sp, target, side="right"))
    lo = hi - 1

    def ok(c):
        return (1 << 31) < c < (1 << 32) and abs(p1 * c - q) <= tol_int

    while True:
        cl = int(sp[lo]) if lo >= 0 else None
        ch = int(sp[hi]) if hi < len(sp) else None
        lo_ok = cl is not None and ok(cl)
        hi_ok = ch is not None and ok(ch)
        if not lo_ok and not hi_ok:
            return None
        if lo_ok and (not hi_ok or target - cl <= ch - target):
            c, lo = cl, lo - 1
        else:
            c, hi = ch, hi + 1
        if c != p1:
            return c


def derive(seed: int, sid: int, sp: np.ndarray, n_p1: int, e: int = 9):
    """(p1, p2, a, step) for a stream id, or None (DerivationExhausted)."""
    ordinal, ai = stream_indices(seed, sid)
    a = MULTIPLIER_TABLE[ai]
    for step in range(256):
        p1 = int(sp[(ordinal + step) % K_P1])
        p2 = find_pair_sorted(p1, sp)
        if p2 is not None:
            return p1, p2, a, step
    return None


# ---------------------------------------------------------------------------
# fused statistics (framework definitions)

def fused_reference(r: np.ndarray) -> dict:
    """r: float64 [n_inst, N] (instance-major draws).  Per-instance moments,
    lag-1, 64-bin histograms, and pooled pair sums in two-pass numpy."""
    n, N = r.shape
    s1 = r.sum(axis=1)
    s2 = (r * r).sum(axis=1)
    mean = s1 / N
    css = s2 - s1 * s1 / N
    var = css / (N - 1)
    lag = (r[:, :-1] * r[:, 1:]).sum(axis=1)
    lag1 = (lag - mean * (2 * s1 - r[:, 0] - r[:, -1]) + (N - 1) * mean * mean) / css
    bins = np.floor(r * 64).astype(np.int64)
    hist = np.stack([np.bincount(b, minlength=64) for b in bins])
    X, Y = r[0::2], r[1::2]
    M = X.size
    mx, my = X.mean(), Y.mean()
    corr = ((X * Y).sum() / M - mx * my) / math.sqrt(((X * X).sum() / M - mx * mx) *
                                                     ((Y * Y).sum() / M - my * my))
    return {"mean": mean, "var": var, "lag1": lag1, "hist": hist, "pooled_hist": hist.sum(axis=0),
            "corr": corr, "s1": s1, "s2": s2, "xy_even": (X * Y).sum(axis=1)}
