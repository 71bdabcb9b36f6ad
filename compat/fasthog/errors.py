"""`fasthog.errors` -> the B200 package (drop-in shim; see compat/fasthog/__init__.py)."""
from paper_1703_06256_b200.errors import *  # noqa: F401,F403
from paper_1703_06256_b200 import errors as _impl

globals().update({k: getattr(_impl, k) for k in dir(_impl) if not k.startswith("__")})
