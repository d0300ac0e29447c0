"""C ABI surface (no GPU needed): the library builds for sm_100a, loads, and
exports exactly what include/rsarand_b200.h declares, with struct layouts that
match the Python views."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1811_11629_b200 import _build, _lib

HEADER = os.path.join(_build.INCLUDE, "rsarand_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return re.findall(r"^(?:int|uint64_t|const char\*)\s+(rsa_\w+)\(", text, flags=re.M)


def test_library_builds_and_loads():
    path = _build.build()
    assert os.path.exists(path)
    lib = _lib.load()
    assert lib.rsa_abi_version() == _lib.ABI_VERSION == 4
    assert lib.rsa_built_arch() == 100


def test_every_declared_symbol_exported_and_typed():
    names = declared_functions()
    assert len(names) >= 14
    lib = ctypes.CDLL(_build.LIB)
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.PROTOTYPES, n
    assert set(_lib.PROTOTYPES) == set(names)


def test_cubin_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_struct_layouts_match(tmp_path):
    fields = list(_lib.INSTANCE_DTYPE.names)
    cfg_fields = [f for f, _ in _lib.SetupConfig._fields_]
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    src.append('printf("%zu %zu %zu\\n", sizeof(rsa_instance), sizeof(rsa_setup_config), sizeof(rsa_fused_stat));')
    for f in fields:
        src.append(f'printf("%zu\\n", offsetof(rsa_instance, {f}));')
    for f in cfg_fields:
        src.append(f'printf("%zu\\n", offsetof(rsa_setup_config, {f}));')
    src.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(c)], check=True)
    vals = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    sizes = list(map(int, vals[:3]))
    offs = list(map(int, vals[3:]))
    assert sizes == [128, ctypes.sizeof(_lib.SetupConfig), _lib.FUSED_STAT_DTYPE.itemsize]
    assert offs[:len(fields)] == [_lib.INSTANCE_DTYPE.fields[f][1] for f in fields]
    assert offs[len(fields):] == [getattr(_lib.SetupConfig, f).offset for f in cfg_fields]


def test_battery_struct_layouts_match(tmp_path):
    spec_fields = [f for f, _ in _lib.BatterySpec._fields_]
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    src.append('printf("%zu %zu %d %d\\n", sizeof(rsa_battery_spec), sizeof(rsa_gap_record), RSA_BT_TILE, RSA_BT_GAPS);')
    for f in spec_fields:
        src.append(f'printf("%zu\\n", offsetof(rsa_battery_spec, {f}));')
    src.append("return 0;}")
    c = tmp_path / "bt.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "bt"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(c)], check=True)
    vals = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()))
    assert vals[:4] == [ctypes.sizeof(_lib.BatterySpec), _lib.GAP_RECORD_BYTES, _lib.RSA_BT_TILE, _lib.RSA_BT_GAPS]
    assert vals[4:] == [getattr(_lib.BatterySpec, f).offset for f in spec_fields]


def test_argument_errors_need_no_gpu():
    lib = _lib.load()
    # invalid arguments are rejected before any launch (status, not a crash)
    assert lib.rsa_fill(None, 1, 1, 1, 9, 1, None, None, None, None, None, 1, None) == _lib.RSA_EINVAL
    assert lib.rsa_fused_stats(None, 3, 1, 9, None, None, None, None, None, None) == _lib.RSA_EINVAL
    assert lib.rsa_safe_prime_scan_scratch_bytes(0, (1 << 32) + 1) == 0
    assert lib.rsa_safe_prime_scan_scratch_bytes(1 << 31, 1 << 32) > 0


def test_segmented_sizing_needs_no_gpu():
    """rsa_fill_segments / rsa_fill_segmented_scratch_bytes (host-only): no
    split for lane counts that fill the chip or runs too short to split; the
    one-thread-per-draw regime (K1p, up to 2^23 draws) needs 8 bytes per draw
    plus small per-segment tables; beyond it the segment regime (K1s) needs
    only per-segment sums."""
    lib = _lib.load()
    assert lib.rsa_fill_segments(1 << 17, 1 << 20) == 1      # lanes fill the chip
    assert lib.rsa_fill_segments(1, 31) == 1                 # too short to split
    assert lib.rsa_fill_segments(1, 1 << 20) > 1
    k1p = lib.rsa_fill_segmented_scratch_bytes(1, 1 << 20)
    assert 8 << 20 <= k1p < (9 << 20)
    k1s = lib.rsa_fill_segmented_scratch_bytes(1, 1 << 24)   # > 2^23 draws: K1s
    assert 0 < k1s < (1 << 22)
    assert lib.rsa_fill_segmented_scratch_bytes(64, 1 << 17) >= 8 << 23  # 2^23 draws: still K1p
    assert lib.rsa_safe_prime_scan_mr_scratch_bytes(0, (1 << 32) + 1) == 0
    assert lib.rsa_safe_prime_scan_mr_scratch_bytes(1 << 31, 1 << 32) > lib.rsa_safe_prime_scan_scratch_bytes(1 << 31, 1 << 32) // 8


def test_c_abi_example_compiles(tmp_path):
    """examples/c_abi_stream0.c (the hot path through the C ABI alone) builds
    against include/rsarand_b200.h and links against the library."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None or not os.path.exists("/usr/local/cuda/include/cuda_runtime.h"):
        pytest.skip("gcc / CUDA headers not available")
    from paper_1811_11629_b200 import _lib
    libdir = os.path.dirname(_lib.lib_path())
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["gcc", "-O2", f"-I{root}/include", "-I/usr/local/cuda/include",
                    os.path.join(root, "examples", "c_abi_stream0.c"), "-o", str(tmp_path / "ex"),
                    f"-L{libdir}", "-lrsarand_b200", "-L/usr/local/cuda/lib64", "-lcudart"], check=True)


def test_no_cpu_fallback(monkeypatch):
    """The product path never computes on the host: without a CUDA device
    every draw / scan entry point raises RsaCudaError, and a missing library
    is an error rather than a fallback."""
    import torch
    import paper_1811_11629_b200 as R
    if torch.cuda.is_available():
        pytest.skip("needs a host without a GPU")
    p = R.make_params(2663418827, 3462982283, 9, R.SkipParams.create(2983799827))
    for call in (lambda: R.init_vector(p, mv=4), lambda: R.rsacore.take_raws(R.init(p), p, 4),
                 lambda: R.safe_primes_in(11, 1000),
                 lambda: R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))):
        with pytest.raises(_lib.RsaCudaError):
            call()
    monkeypatch.setenv("RSARAND_B200_LIB", "/nonexistent/librsarand_b200.so")
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(_lib.RsaCudaError):
        _lib.load(build_if_missing=False)
