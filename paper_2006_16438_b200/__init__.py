"""B200-native CP-ARLS-LEV hot path (arXiv 2006.16438).

The product is libcparls.so (csrc/, C ABI in include/cparls.h); this package
is its ctypes binding.  There is no CPU fallback.
"""
from .cparls import (Comm, Cparls, CparlsError, EXPORTED, LIB_PATH, lib, plan_rows, route_nonzeros,  # noqa: F401
                     version)
