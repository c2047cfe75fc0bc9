"""B200-native shifted Krylov (COCG / BiCG) hot path of the Komega paper (arxiv 2001.08707).

The product is libshiftk.so (C-ABI: include/shiftk.h; kernels: csrc/).  ``shiftk`` is the thin
ctypes binding; ``device`` holds the torch plumbing (device memory for inputs).  Nothing here
imports the CPU oracle (oracle/), which is test infrastructure only.
"""
from . import shiftk  # noqa: F401
from .shiftk import Solver, load, make_operator, apply_operator  # noqa: F401
