"""ctypes binding of librsarand_b200.so (include/rsarand_b200.h).

The product path has exactly one implementation: these CUDA kernels.  If the
library is missing or cannot be loaded, every operation raises — there is no
CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _build

_LIB = None
_LOCK = threading.Lock()

c_u32, c_u64, c_i32, c_vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p

RSA_OK = 0
RSA_EINVAL = -1
RSA_ECUDA = -2
RSA_EPARAMS = -3
RSA_ECAPACITY = -4
RSA_EALIGN = -5

RSA_SKIP_LCG, RSA_SKIP_UNIT, RSA_SKIP_CONST = 0, 1, 2
RSA_BT_HIST, RSA_BT_SERIAL, RSA_BT_POKER, RSA_BT_MAX_OF_T, RSA_BT_PERMUTATION, RSA_BT_COLLISION = 1, 2, 3, 4, 5, 6
RSA_BT_GAPS = 7
RSA_BT_TILE = 256
RSA_FLAG_FAST, RSA_FLAG_FIXED, RSA_FLAG_GENERAL_PATH, RSA_FLAG_ONE_LANE = 1, 2, 4, 8
RSA_FLAG_INTERLEAVE, RSA_FLAG_LOW32 = 16, 32

# rsa_instance (128 bytes) — field order and offsets mirror the C struct.
INSTANCE_DTYPE = np.dtype({
    "names": ["p1", "p2", "p1_inv", "p2_inv", "a", "e", "k1", "k2", "r2_1", "r2_2",
              "garner", "p2inv", "q1", "q2", "flags", "skip_mode", "n", "q", "b",
              "n_float", "n_recip", "skip_const", "reserved1", "reserved2"],
    "formats": ["<u4"] * 16 + ["<u8"] * 3 + ["<f8", "<f8", "<u8", "<f8", "<u8"],
    "offsets": [0, 4, 8, 12, 16, 20, 24, 28, 32, 36, 40, 44, 48, 52, 56, 60,
                64, 72, 80, 88, 96, 104, 112, 120],
    "itemsize": 128,
})

FUSED_STAT_DTYPE = np.dtype([("s1", "<f8"), ("s2", "<f8"), ("lag", "<f8"), ("first", "<f8"),
                             ("last", "<f8"), ("xy", "<f8")])


class BatterySpec(ctypes.Structure):
    _fields_ = [("test", c_i32), ("d", c_u32), ("p1", c_u32), ("p2", c_u32), ("pos0", c_u64), ("seg0", c_u64),
                ("aux", c_u64)]


GAP_RECORD_BYTES = 16  # rsa_gap_record: head, tail, len, bits (uint32 each)


class SetupConfig(ctypes.Structure):
    _fields_ = [("seed_mod_S", c_u64), ("first_id", c_u64), ("sigma", c_u64),
                ("k_p1", c_u64), ("k_p2", c_u64), ("q", c_u64), ("tol", c_u64),
                ("epsilon", c_u32), ("e", c_u32), ("n_mult", c_u32), ("multiplier", c_u32),
                ("max_steps", c_u32), ("start_step", c_u32)]


ABI_VERSION = 4  # include/rsarand_b200.h RSA_ABI_VERSION

# name -> (restype, argtypes); the CPU test checks this list against include/*.h
PROTOTYPES = {
    "rsa_fill": (ctypes.c_int, [c_vp, c_u32, c_u32, c_u64, c_u32, c_u32, c_vp, c_vp, c_vp,
                                c_vp, c_vp, c_u64, c_vp]),
    "rsa_floats_from_raw": (ctypes.c_int, [c_vp, c_u64, c_u64, c_vp, c_vp]),
    "rsa_floats_from_raw_dd": (ctypes.c_int, [c_vp, c_u64, c_u64, c_vp, c_vp]),
    "rsa_skip_array": (ctypes.c_int, [c_vp, c_u64, c_u64, c_u64, c_vp, c_vp]),
    "rsa_fill_segments": (c_u64, [c_u64, c_u64]),
    "rsa_scalar_lookahead": (ctypes.c_int, [c_vp, c_u64, c_u64, c_u64, c_u32, c_u32, c_u32, c_vp, c_vp]),
    "rsa_fill_segmented_scratch_bytes": (c_u64, [c_u64, c_u64]),
    "rsa_fill_segmented": (ctypes.c_int, [c_vp, c_u32, c_u32, c_u64, c_u32, c_u32, c_vp, c_vp, c_vp,
                                          c_vp, c_vp, c_u64, c_vp, c_u64, c_vp]),
    "rsa_init_lanes": (ctypes.c_int, [c_vp, c_u32, c_u32, c_u64, c_u64, c_u64, c_vp, c_vp,
                                      c_vp, c_vp]),
    "rsa_fused_stats": (ctypes.c_int, [c_vp, c_u32, c_u64, c_u32, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_vp]),
    "rsa_fused_pool": (ctypes.c_int, [c_vp, c_vp, c_u32, c_vp, c_vp, c_vp]),
    "rsa_safe_prime_scan_scratch_bytes": (c_u64, [c_u64, c_u64]),
    "rsa_safe_prime_scan": (ctypes.c_int, [c_u64, c_u64, c_vp, c_u64, c_vp, c_vp, c_u64, c_vp]),
    "rsa_safe_prime_scan_mr_scratch_bytes": (c_u64, [c_u64, c_u64]),
    "rsa_safe_prime_scan_mr": (ctypes.c_int, [c_u64, c_u64, c_vp, c_u64, c_vp, c_vp, c_u64, c_vp]),
    "rsa_is_safe_prime32": (ctypes.c_int, [c_vp, c_u64, c_vp, c_vp, c_vp]),
    "rsa_safe_prime_index": (ctypes.c_int, [c_vp, c_u64, c_vp, c_vp]),
    "rsa_find_pair": (ctypes.c_int, [c_vp, c_u64, c_u64, c_u64, c_vp, c_u64, c_vp, c_vp, c_vp, c_vp]),
    "rsa_setup_instances": (ctypes.c_int, [ctypes.POINTER(SetupConfig), c_u64, c_vp, c_vp, c_u64,
                                           c_vp, c_vp, c_u64, c_vp, c_vp, c_vp, c_vp]),
    "rsa_probe_imad": (ctypes.c_int, [c_u32, c_u32, c_vp, ctypes.POINTER(ctypes.c_double), c_vp]),
    "rsa_battery_count": (ctypes.c_int, [ctypes.c_int, c_vp, c_u64, c_u32, c_u32, c_vp, c_vp, c_vp]),
    "rsa_battery_fused": (ctypes.c_int, [c_vp, c_u32, c_u32, c_u64, c_u32, c_u32, c_vp, c_vp, c_vp,
                                         ctypes.POINTER(BatterySpec), c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rsa_battery_gaps_array": (ctypes.c_int, [c_vp, c_u64, ctypes.POINTER(BatterySpec), c_vp, c_vp, c_vp]),
    "rsa_battery_stitch": (ctypes.c_int, [ctypes.POINTER(BatterySpec), c_vp, c_u64, c_u64, c_vp, c_vp, c_vp]),
    "rsa_battery_gaps_stitch": (ctypes.c_int, [c_vp, c_u64, c_vp, c_vp]),
    "rsa_battery_collision_array": (ctypes.c_int, [c_vp, c_u64, ctypes.POINTER(BatterySpec), c_vp, c_vp]),
    "rsa_battery_collision_hist": (ctypes.c_int, [c_vp, c_u64, c_vp, c_vp]),
    "rsa_battery_fourier_bin": (ctypes.c_int, [c_vp, c_u64, c_vp, c_vp, c_vp]),
    "rsa_battery_chi2_scratch_bytes": (c_u64, [c_u64]),
    "rsa_battery_chi2_sum": (ctypes.c_int, [c_vp, c_u64, ctypes.c_double, c_vp, c_vp, c_u64, c_vp]),
    "rsa_abi_version": (ctypes.c_int, []),
    "rsa_built_arch": (ctypes.c_int, []),
    "rsa_last_error": (ctypes.c_char_p, []),
    "rsa_launch_count": (c_u64, []),
}


class RsaCudaError(RuntimeError):
    """A C-ABI call failed (status code and CUDA error text attached)."""


def lib_path() -> str:
    """The in-tree library; RSARAND_B200_LIB overrides it (A/B runs only)."""
    return os.environ.get("RSARAND_B200_LIB", _build.LIB)


def load(build_if_missing: bool = True):
    """Load (building in-tree first if needed) and type the shared library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        path = lib_path()
        if not os.path.exists(path):
            if not build_if_missing:
                raise RsaCudaError(f"CUDA library not built: {path}")
            _build.build()
        lib = ctypes.CDLL(path)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.rsa_abi_version() != ABI_VERSION:
            raise RsaCudaError("librsarand_b200 ABI mismatch")
        _LIB = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != RSA_OK:
        err = load().rsa_last_error().decode(errors="replace")
        raise RsaCudaError(f"{what} failed with status {rc}: {err}")


_FN: dict = {}  # name -> (library, typed entry point): skips a getattr per call


def call(name: str, *args) -> None:
    lib = _LIB if _LIB is not None else load()
    hit = _FN.get(name)
    if hit is None or hit[0] is not lib:
        hit = _FN[name] = (lib, getattr(lib, name))
    rc = hit[1](*args)
    if rc != RSA_OK:
        check(rc, name)
