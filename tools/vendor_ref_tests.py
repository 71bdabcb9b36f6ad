#!/usr/bin/env python
"""Copy the reference's own test modules (the hot-path ones) from
/root/reference/pkg/tests into baseline/_ref_tests/ so that
tests/test_gpu_ref_suite.py can run them, unchanged, against this package
through the `fasthog` shim (compat/).  Like baseline/_ref (the pip-installed
reference), the copy is git-ignored -- it is test infrastructure, not part
of the product or of the repository's history -- and it travels to the GPU
box with the working tree.  No-op when /root/reference is absent.
"""
import os
import shutil
import sys

SRC = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "baseline", "_ref_tests")
# the hot-path modules; test_cli.py / test_bench.py cover the
# out-of-scope CLI and naive-vs-integral bench harness
MODULES = ["conftest.py", "test_gradient.py", "test_integral.py", "test_descriptor.py",
           "test_detector.py", "test_image_io.py", "test_acceptance.py"]


def main() -> int:
    if not os.path.isdir(SRC):
        print(f"vendor_ref_tests: {SRC} absent, keeping {DST} as is")
        return 0
    os.makedirs(DST, exist_ok=True)
    for m in MODULES:
        shutil.copy2(os.path.join(SRC, m), os.path.join(DST, m))
    print(f"vendor_ref_tests: {len(MODULES)} modules -> {DST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
