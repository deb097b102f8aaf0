"""B200-native (sm_100a) exact hypercube convolution (Serang, arXiv:1608.00206).

The compute path is libhc.so (csrc/, C ABI in include/hc.h); ``paper_1608_00206_b200.hc``
is a thin ctypes binding (argument marshalling only).  There is no CPU fallback: if the
extension is missing, importing ``paper_1608_00206_b200.hc`` raises ImportError.
Build with ``python paper_1608_00206_b200/build.py``.
"""
