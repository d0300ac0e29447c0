"""The base-2 strong-pseudoprime table that finishes the scan's safe-prime
verdicts (paper_1811_11629_b200/csrc/spsp2_table.inc, tools/gen_spsp2.c).

CPU checks: the table is sorted, has the published size (2314 below 2^32),
every entry is an odd composite that passes the base-2 SPRP test, and the
generator reproduces the table exactly on a prefix range.  The GPU check that
the scan decides every table-relevant candidate like the oracle lives in
tests/test_gpu_setup.py (test_scan_pseudoprime_neighbourhoods)."""

import os
import re
import shutil
import subprocess

import pytest

from oracle import rsa_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "paper_1811_11629_b200", "csrc", "spsp2_table.inc")
GEN = os.path.join(ROOT, "tools", "gen_spsp2.c")


def load_table():
    txt = open(INC).read()
    count = int(re.search(r"#define RSA_SPSP2_COUNT (\d+)u", txt).group(1))
    fnv = int(re.search(r"#define RSA_SPSP2_FNV (0x[0-9a-f]+)ull", txt).group(1), 16)
    body = txt.split("#define RSA_SPSP2_TABLE", 1)[1]
    vals = [int(v) for v in re.findall(r"(\d+)u", body)]
    return count, fnv, vals


def sprp2(n):
    d, u = n - 1, 0
    while d % 2 == 0:
        d //= 2
        u += 1
    x = pow(2, d, n)
    if x in (1, n - 1):
        return True
    for _ in range(u - 1):
        x = x * x % n
        if x == n - 1:
            return True
    return False


def smallest_factor(n):
    f = 3
    while f * f <= n:
        if n % f == 0:
            return f
        f += 2
    return n


def test_table_shape_and_checksum():
    count, fnv, vals = load_table()
    assert count == len(vals) == 2314  # spsp(2) below 2^32
    assert vals == sorted(set(vals)) and vals[0] == 2047 and vals[-1] < 1 << 32
    h = 1469598103934665603
    for v in vals:
        for b in v.to_bytes(4, "little"):
            h = ((h ^ b) * 1099511628211) % (1 << 64)
    assert h == fnv


def test_entries_are_composite_base2_sprps():
    _, _, vals = load_table()
    for v in vals:
        assert v % 2 == 1 and sprp2(v)
        assert not O.is_prime(v)
    # spot-check true factors on a spread of entries (trial division is slow
    # for the largest ones, so every 16th)
    for v in vals[::16]:
        assert smallest_factor(v) < v


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_generator_reproduces_prefix(tmp_path):
    exe = tmp_path / "gen_spsp2"
    subprocess.run(["gcc", "-O2", "-fopenmp", GEN, "-o", str(exe)], check=True)
    hi = 1 << 25
    out = subprocess.run([str(exe), "0", str(hi)], check=True, capture_output=True, text=True).stdout
    got = [int(v) for v in out.split()]
    _, _, vals = load_table()
    assert got == [v for v in vals if v < hi]
    assert len(got) > 100
