"""B200-native hybrid-parallel 3D-ResAttNet training step (arXiv 2104.05035).

The product is librn.so (C ABI in include/rn.h, CUDA kernels for sm_100a in
csrc/); `rn` is its thin ctypes binding."""
from . import rn  # noqa: F401
