"""B200-native LOBPCG hot path of arXiv 2109.00485 (MFDn) behind the C ABI of
include/blockeig_b200.h. The product is libblockeig_b200.so (C++ host code +
sm_100a CUDA kernels); the C++ mirror of the reference API lives in cpp/;
abi.py is the ctypes binding used by the tests and bench.py."""
from .abi import lib  # noqa: F401
