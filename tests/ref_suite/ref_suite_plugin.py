"""pytest plugin for the reference's own tests run through the `fasthog`
shim (compat/) on the GPU (tests/test_gpu_ref_suite.py).

* Checks that `import fasthog` resolves to the shim, i.e. to this package.
* Two names the reference tests import lie outside the hot path:
  the CLI (`fasthog.cli`) and the naive-vs-integral bench harness
  (`fasthog.run_bench` / `fasthog.bench`).  They are provided here as test-only
  stubs that SKIP the test using them, so the modules that import them at the
  top still run every other test.
* DIFFERS lists the reference tests whose assertion does not hold for a
  correct GPU implementation, each with the reason; they are reported as
  xfail (strict: they must actually fail, so the list cannot go stale).
"""
import sys
import types

import pytest

import fasthog

if "compat" not in fasthog.__file__:
    raise RuntimeError(f"fasthog resolves to {fasthog.__file__}, not the compat shim")

OUT_OF_SCOPE = "out of scope (SURVEY §2): {}"


def _skip(what):
    def f(*a, **k):
        pytest.skip(OUT_OF_SCOPE.format(what))
    return f


_cli = types.ModuleType("fasthog.cli")
_cli.main = _skip("the fasthog command-line interface")
sys.modules["fasthog.cli"] = _cli
fasthog.cli = _cli
_bench = types.ModuleType("fasthog.bench")
_bench.run_bench = _skip("the naive-vs-integral bench harness")
sys.modules["fasthog.bench"] = _bench
fasthog.bench = _bench
fasthog.run_bench = _bench.run_bench

# nodeid suffix -> why the reference's assertion does not apply
DIFFERS = {
    # detector.py:148 compares scan's score with np.dot(w, d) + b for EXACT equality;
    # np.dot is OpenBLAS ddot, whose summation order is library- and CPU-defined
    # (DYNAMIC_ARCH kernels), so no other summation reproduces it bit for bit.  The
    # device sums the same products in fp64 in its own order: measured |diff| 7e-15
    # on a score of 3.97 (relative 2e-15); the north star's bar is 1e-5 relative,
    # which test_gpu_parity.py and test_gpu_c5_full.py check against the oracle.
    "test_detector.py::test_scan_matches_naive_recompute":
        "fp64 summation order differs from OpenBLAS ddot (relative error ~1e-15)",
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        for key, why in DIFFERS.items():
            if item.nodeid.endswith(key):
                item.add_marker(pytest.mark.xfail(reason=why, strict=True))
