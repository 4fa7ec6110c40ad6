"""B200-native data-parallel volume rendering: per-rank DVR of a brick + sort-last compositing.

The data path is libdprt_cuda.so (sm_100a kernels behind the C ABI in include/dprt_cuda.h); this package
is the host side, shaped like the reference's `dprt` API (engine / api / transport).  See DESIGN.md.
"""

__version__ = "0.1.0"
