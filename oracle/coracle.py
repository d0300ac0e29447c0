"""ctypes wrapper of the C oracle (oracle/rsa_oracle.c) — test infrastructure only.

Builds oracle/liboracle.so with gcc on first use (oracle/Makefile recipe).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "rsa_oracle.c")

_lib = None


class OracleParams(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("p1", "p2", "e", "a", "q", "p2inv", "mode", "n")]


TUPLE_DTYPE = np.dtype([("p1", "<u4"), ("p2", "<u4"), ("a", "<u4"), ("p2inv", "<u4"),
                        ("n", "<u8"), ("b", "<u8")])


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["make", "-C", HERE, "-s", "liboracle.so"], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        u64 = ctypes.c_uint64
        lib.oracle_fill.argtypes = [ctypes.POINTER(OracleParams), u64, u64, P, P, P, P, P, u64]
        lib.oracle_fill.restype = None
        lib.oracle_census.argtypes = [u64, u64, P, u64, ctypes.POINTER(u64)]
        lib.oracle_census.restype = u64
        lib.oracle_derive.argtypes = [u64, u64, u64, P, u64, P, u64, u64, u64, P, P]
        lib.oracle_derive.restype = None
        _lib = lib
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def params(p1, p2, e, a, q=(1 << 63) - 25, mode=0) -> OracleParams:
    return OracleParams(p1=p1, p2=p2, e=e, a=a, q=q, p2inv=pow(p2, -1, p1), mode=mode, n=p1 * p2)


def fill(P: OracleParams, m1: np.ndarray, m2: np.ndarray, s: np.ndarray, blocks: int,
         raw: bool = True, f64: bool = True):
    """Advance lanes in place; returns ([blocks, lanes] raw, [blocks, lanes] f64)."""
    lanes = len(s)
    for arr in (m1, m2, s):
        assert arr.dtype == np.uint64 and arr.flags.c_contiguous
    r = np.empty((blocks, lanes), dtype=np.uint64) if raw else None
    f = np.empty((blocks, lanes), dtype=np.float64) if f64 else None
    load().oracle_fill(ctypes.byref(P), lanes, blocks, _ptr(m1), _ptr(m2), _ptr(s), _ptr(r), _ptr(f),
                       lanes)
    return r, f


def census(lo: int = 1 << 31, hi: int = 1 << 32):
    """(sorted uint32 safe primes in [lo, hi), number of primes in [lo, hi))."""
    cap = max(1024, (hi - lo) // 100)
    out = np.empty(cap, dtype=np.uint32)
    npr = ctypes.c_uint64(0)
    n = load().oracle_census(lo, hi, _ptr(out), cap, ctypes.byref(npr))
    assert n <= cap
    return out[:n].copy(), int(npr.value)


def derive(seed: int, first: int, count: int, sp: np.ndarray, mult, q=(1 << 63) - 25,
           tol=9223372036854):
    S = 1291831 * 1768937 * len(mult)
    out = np.zeros(count, dtype=TUPLE_DTYPE)
    steps = np.zeros(count, dtype=np.uint32)
    m = np.asarray(mult, dtype=np.uint32)
    sp = np.ascontiguousarray(sp, dtype=np.uint32)
    load().oracle_derive(seed % S, first, count, _ptr(sp), len(sp), _ptr(m), len(m), q, tol,
                         _ptr(out), _ptr(steps))
    return out, steps
