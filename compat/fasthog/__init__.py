"""`fasthog` compatibility shim (SURVEY §4 re-targeting plan).

Put `compat/` first on PYTHONPATH and `import fasthog` resolves to the B200
package: the flat API (reference __init__.py:4-65) and the submodules
`fasthog.gradient`, `.integral`, `.descriptor`, `.detector`, `.image_io`,
`.errors` expose the same names, backed by libhogb200.so (no CPU fallback).
Names outside the hot path (the CPU bench harness, the CLI) are not provided.
"""
import os
import sys

_ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_1703_06256_b200 import *  # noqa: E402,F401,F403
from paper_1703_06256_b200 import __version__  # noqa: E402,F401

from . import descriptor, detector, errors, gradient, image_io, integral  # noqa: E402,F401
