"""B200-native hot path of Saturating Coordinate Descent (arXiv 2003.03572).

The product is libsacd.so (CUDA, sm_100a) behind the C ABI in include/sacd.h;
`sacd.Sacd` is its thin ctypes binding.
"""
from .sacd import Sacd, SacdError, load_library  # noqa: F401
