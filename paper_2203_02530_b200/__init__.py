"""B200-native distributed SpMV hot path of arXiv 2203.02530.

The product is the C-ABI shared library ``lib/libdspmv.so`` (declared in
``include/dspmv.h``); ``paper_2203_02530_b200.dspmv`` is a thin ctypes
binding with the same names (argument marshalling only -- every step of the
path runs in the library's sm_100a kernels and C++ executor).  There is no
CPU fallback: importing the binding raises if the library is missing.
"""
from . import dspmv  # noqa: F401
