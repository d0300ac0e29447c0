"""Text checkpoints of one stream: the "rsarand-snapshot-v1" and
"rsarand-params-v1" formats of the reference (rsacore.py:292-417).

A checkpoint is a header line followed by `key=value` lines in a fixed order:
thirteen parameter keys, then (snapshot only) the state keys m1, m2, s,
draws.  Values are lower-case hex without prefix except `skip_mode`, which is
the mode word.  Output is byte-identical to the reference's; tests pin it
(tests/test_snapshot_text.py against tests/golden/snapshot.json).

Re-exported by rsacore (StreamSnapshot, snapshot, restore, params_to_text,
params_from_text, params_lines).
"""

from __future__ import annotations

from dataclasses import dataclass

SNAPSHOT_HEADER = "rsarand-snapshot-v1"
PARAMS_HEADER = "rsarand-params-v1"

# (key, how to read it off a GeneratorParams)
_PARAM_KEYS = (
    ("p1", lambda p: p.p1), ("p2", lambda p: p.p2), ("n", lambda p: p.n), ("e", lambda p: p.e),
    ("q", lambda p: p.skip.q), ("a", lambda p: p.skip.a), ("q1", lambda p: p.skip.q1),
    ("q2", lambda p: p.skip.q2), ("p2inv", lambda p: p.p2inv), ("b", lambda p: p.b),
    ("skip_mode", lambda p: p.skip_mode), ("skip_const", lambda p: p.skip_const),
    ("test_mode", lambda p: int(p.test_mode)),
)
_STATE_KEYS = ("m1", "m2", "s", "draws")


def _err(msg: str):
    from .rsacore import MalformedSnapshot
    return MalformedSnapshot(msg)


def params_lines(params) -> list:
    """The parameter block of either format, one `key=value` string per key."""
    out = []
    for key, get in _PARAM_KEYS:
        v = get(params)
        out.append(f"{key}={v}" if key == "skip_mode" else f"{key}={v:x}")
    return out


def _render(header: str, lines: list) -> str:
    return header + "\n" + "".join(ln + "\n" for ln in lines)


def _fields(text: str, header: str, keys: tuple) -> dict:
    """key -> raw value string; exactly `keys`, each once, under `header`."""
    rows = [r.strip() for r in text.splitlines()]
    rows = [r for r in rows if r]
    if not rows or rows[0] != header:
        raise _err(f"missing or unknown header (want {header!r})")
    got: dict = {}
    for row in rows[1:]:
        if "=" not in row:
            raise _err(f"bad line {row!r}")
        key, val = row.split("=", 1)
        if key in got:
            raise _err(f"bad line {row!r}")
        got[key] = val
    missing, extra = set(keys) - set(got), set(got) - set(keys)
    if missing or extra:
        raise _err(f"missing={sorted(missing)} unknown={sorted(extra)}")
    return got


def _int16(got: dict, key: str) -> int:
    try:
        return int(got[key], 16)
    except ValueError:
        raise _err(f"field {key} is not hex: {got[key]!r}") from None


def _params_of(got: dict):
    from .rsacore import GeneratorParams
    from .skipgen import SkipParams
    h = {k: _int16(got, k) for k, _ in _PARAM_KEYS if k != "skip_mode"}
    return GeneratorParams(p1=h["p1"], p2=h["p2"], n=h["n"], e=h["e"],
                           skip=SkipParams(q=h["q"], a=h["a"], q1=h["q1"], q2=h["q2"]),
                           p2inv=h["p2inv"], b=h["b"], skip_mode=got["skip_mode"],
                           skip_const=h["skip_const"], test_mode=bool(h["test_mode"]),
                           n_float=float(h["n"]))


@dataclass(frozen=True)
class StreamSnapshot:
    params: object   # GeneratorParams
    m1: int
    m2: int
    s: int
    draws: int

    def to_text(self) -> str:
        state = [f"{k}={getattr(self, k):x}" for k in _STATE_KEYS]
        return _render(SNAPSHOT_HEADER, params_lines(self.params) + state)

    @classmethod
    def from_text(cls, text: str) -> "StreamSnapshot":
        keys = tuple(k for k, _ in _PARAM_KEYS) + _STATE_KEYS
        got = _fields(text, SNAPSHOT_HEADER, keys)
        return cls(_params_of(got), *(_int16(got, k) for k in _STATE_KEYS))


def params_to_text(params) -> str:
    return _render(PARAMS_HEADER, params_lines(params))


def params_from_text(text: str):
    from .rsacore import InvalidParams, validate_params
    p = _params_of(_fields(text, PARAMS_HEADER, tuple(k for k, _ in _PARAM_KEYS)))
    try:
        validate_params(p)
    except InvalidParams as exc:
        raise _err(f"exported params invalid: {exc}") from exc
    return p


def snapshot(state, params) -> StreamSnapshot:
    return StreamSnapshot(params, state.m1, state.m2, state.s, state.draws)


def _state_problem(snap: StreamSnapshot):
    from .rsacore import SKIP_CONST
    p = snap.params
    if not 0 <= snap.m1 < p.p1:
        return "m1 outside [0, p1)"
    if not 0 <= snap.m2 < p.p2:
        return "m2 outside [0, p2)"
    if p.skip_mode == SKIP_CONST and snap.s != p.skip_const:
        return "const-mode skip register mismatch"
    if p.skip_mode != SKIP_CONST and not 0 < snap.s < p.skip.q:
        return "skip outside [1, q)"
    if snap.draws < 0:
        return "negative draw count"
    return None


def restore(snap):
    """(params, state) from a StreamSnapshot or its text, re-validating the
    parameters and the state against them."""
    from .rsacore import GeneratorState, InvalidParams, validate_params
    if isinstance(snap, str):
        snap = StreamSnapshot.from_text(snap)
    try:
        validate_params(snap.params)
    except InvalidParams as exc:
        raise _err(f"snapshot params invalid: {exc}") from exc
    problem = _state_problem(snap)
    if problem:
        raise _err(problem)
    return snap.params, GeneratorState(m1=snap.m1, m2=snap.m2, s=snap.s, draws=snap.draws)
