"""B200-native RailS hot path (arXiv 2510.19262): LPT spraying scheduler + rail pack.

The product is the C-ABI library ``librails.so`` (include/rails.h) built from the
sm_100a kernels in ``csrc/``; ``rails`` is its ctypes binding, ``pipeline`` chains
the calls into one pass of the path, ``dist`` shards it over ranks.
"""
from . import rails  # noqa: F401

__all__ = ["rails"]
