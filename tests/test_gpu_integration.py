"""The reference-side ctypes shim printed in INTEGRATION.md runs against the
built library and reproduces vecgen.next_block_raw (the binding a maintainer
would add to rsarand is executable, not just illustrative)."""

import os
import re

import numpy as np
import pytest
import torch

import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import _lib, vecgen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _shim_namespace():
    txt = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# rsarand/_b200\.py.*?)```", txt, re.S).group(1)
    code = code.replace('ctypes.CDLL("librsarand_b200.so")', f'ctypes.CDLL({_lib.lib_path()!r})')
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def test_integration_shim_matches_vecgen():
    ns = _shim_namespace()
    p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
    a = R.init_vector(p, m0=99, mv=256)
    b = R.init_vector(p, m0=99, mv=256)
    for _ in range(3):
        got = ns["next_block_raw"](a).cpu().numpy()
        want = vecgen.next_block_raw(b).cpu().numpy()
        assert np.array_equal(got, want)
    rec = ns["pack"](p)
    host = np.frombuffer(R.rsacore._instance_record(p).tobytes(), dtype=ns["INSTANCE"])[0]
    for f in ns["INSTANCE"].names:
        assert rec[f] == host[f], f


def _build_c_example(tmp_path):
    import subprocess
    exe = tmp_path / "c_abi_stream0"
    libdir = os.path.dirname(_lib.lib_path())
    subprocess.run(["gcc", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "examples", "c_abi_stream0.c"), "-o", str(exe), f"-L{libdir}",
                    "-lrsarand_b200", "-L/usr/local/cuda/lib64", "-lcudart",
                    f"-Wl,-rpath,{libdir}:/usr/local/cuda/lib64"], check=True)
    return exe


def test_c_abi_example_reproduces_regression_vector(tmp_path, golden_regression):
    """examples/c_abi_stream0.c: scan -> index -> derive stream 0 -> seed ->
    four draws, all through the C ABI, equals the reference's pinned vector."""
    import subprocess
    out = subprocess.run([str(_build_c_example(tmp_path))], check=True, capture_output=True,
                         text=True).stdout.split()
    g = golden_regression
    assert int(out[0]) == 3_060_794
    assert [int(x) for x in out[1:4]] == [g["params"]["p1"], g["params"]["p2"], g["params"]["a"]]
    assert [int(x) for x in out[4:8]] == g["raw"][:4]
