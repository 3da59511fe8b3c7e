"""B200-native (sm_100a) Polylla core (GPolylla, arXiv 2403.14723).

The product is ``libpolylla.so`` (CUDA kernels behind the C ABI of include/polylla.h);
``polylla`` is its thin ctypes binding.  See DESIGN.md.
"""
from . import polylla  # noqa: F401

__all__ = ["polylla"]
