"""B200-native Random Batch Method step library (arXiv:1812.10575).

The product is librbm.so (C ABI in include/rbm.h, CUDA for sm_100a under
csrc/); ``rbm`` is its thin ctypes binding.
"""
from . import rbm  # noqa: F401
from .rbm import RBM, Direct, RbmError, make_config  # noqa: F401
