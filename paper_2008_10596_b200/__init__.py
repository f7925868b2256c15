"""B200-native checkpoint drain / restart refill (CRAC hot path).

The product is libcrac_b200.so (C++ host engine + sm_100a kernels) behind
include/crac_engine.h; this package holds its sources (csrc/), the build
(build.py) and the Python mirror of the reference engine API (engine.py).
"""
from . import engine  # noqa: F401
from .engine import (CracError, Image, Session, decode_check, hash_chunks, restart,  # noqa: F401
                     restart_from_address, summarize_image)
