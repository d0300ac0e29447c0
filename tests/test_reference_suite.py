"""The reference's own unit tests for the host-side modules, run unchanged
against this package (CPU, build container only: /root/reference is absent
on the GPU box, and the reference's tests are executed from there, never
copied).  A module alias makes `import rsarand.<m>` resolve to
paper_1811_11629_b200.<m>; the selection is the reference tests that need no
CUDA device here (their draw / sieve / derivation tests need the GPU in this
package and are covered by the -m gpu parity suite against the reference's
golden vectors instead).
"""

import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RUNNER = r"""
import importlib, sys, types
sys.path.insert(0, {root!r})
import paper_1811_11629_b200  # noqa: F401
pkg = types.ModuleType("rsarand")
pkg.__path__ = []
sys.modules["rsarand"] = pkg
for k in ("numtheory", "skipgen", "rsacore", "paramfactory", "vecgen", "stats"):
    m = importlib.import_module("paper_1811_11629_b200." + k)
    sys.modules["rsarand." + k] = m
    setattr(pkg, k, m)
import pytest
sys.exit(pytest.main(["-q", "-p", "no:cacheprovider", "--tb=short", "-k", {sel!r}] + {files!r}))
"""

SELECTIONS = [
    # every numtheory test except the 110 s full-volume factoring sweep
    (["test_numtheory.py"], "not full_volume"),
    # skip parameters, single-register skips, skip powers, the multiplier table
    (["test_skipgen.py"], "TestCreate or TestNextSkip and not Array or TestSkipPower or TestMultiplierTable"),
    # init, parameter construction / validation, bijectivity, decryption, period jumps on miniatures
    (["test_rsacore.py"], "TestInit or (TestMakeParams and not production) or TestBijectivity or "
                          "(TestDecrypt and not stream) or (TestJumpPeriods and not twelve and not continue)"),
]


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="the reference is only present in the build container")
@pytest.mark.parametrize("files,sel", SELECTIONS, ids=[s[0][0] for s in SELECTIONS])
def test_reference_unit_tests_pass_against_the_package(files, sel, tmp_path):
    code = RUNNER.format(root=ROOT, sel=sel, files=[os.path.join(REF_TESTS, f) for f in files])
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    res = subprocess.run([sys.executable, "-c", code], cwd=str(tmp_path), env=env,
                         capture_output=True, text=True, timeout=600)
    tail = "\n".join(res.stdout.splitlines()[-15:])
    assert res.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail and "error" not in tail.lower(), tail


NAMESPACE = r"""
import importlib, sys
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, {root!r})
out = {{}}
for m in ("numtheory", "skipgen", "rsacore", "paramfactory", "vecgen", "stats", ""):
    ref = importlib.import_module("rsarand" + ("." + m if m else ""))
    ours = importlib.import_module("paper_1811_11629_b200" + ("." + m if m else ""))
    names = {{n for n in dir(ref) if not n.startswith("_") and not isinstance(getattr(ref, n), type(sys))
             or n in ("skipgen", "vecgen", "rsacore", "numtheory", "paramfactory", "stats")}}
    std = {{"np", "math", "dataclass", "field", "annotations", "Sequence", "Callable", "functools", "special"}}
    out[m or "rsarand"] = sorted(n for n in names - std if not hasattr(ours, n))
print(out)
"""


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="the reference is only present in the build container")
def test_public_names_of_every_reference_module_exist():
    """Every public name of rsarand and its host-side modules (functions,
    classes, constants, re-exported modules) exists under the same name in the
    drop-in package."""
    res = subprocess.run([sys.executable, "-c", NAMESPACE.format(root=ROOT)], capture_output=True, text=True,
                         timeout=300, env=dict(os.environ, PYTHONDONTWRITEBYTECODE="1"))
    assert res.returncode == 0, res.stderr[-2000:]
    missing = eval(res.stdout.strip().splitlines()[-1])
    assert all(not v for v in missing.values()), missing
