"""B200-native (sm_100a) non-Hermitian FEAST quadrature projector (arXiv 1404.2891).

The hot path lives in libfeast_b200.so (C ABI: include/feast.h); `feast` is its thin binding.
"""
from .feast import (BI, RIGHT, RULE_GAUSS_LEGENDRE, RULE_TRAPEZOID, RULE_TRAPEZOID_ENDPOINT, Feast, FeastError,
                    colmajor, empty_colmajor, load_library)

__all__ = ["Feast", "FeastError", "load_library", "colmajor", "empty_colmajor", "RIGHT", "BI", "RULE_TRAPEZOID",
           "RULE_TRAPEZOID_ENDPOINT", "RULE_GAUSS_LEGENDRE"]
