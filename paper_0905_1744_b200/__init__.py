"""B200-native hot path of Sample-Align-D (arXiv 0905.1744).

``libsa`` (include/sa.h, csrc/) holds every step as sm_100a CUDA kernels; this
package is its thin ctypes binding (``binding``), the per-rank step driver
(``pipeline``) and the in-tree build (``build``).  Importing the package does
not load the library; the first binding call does, and fails loudly if it is
missing -- there is no CPU fallback.
"""
__version__ = "0.1.0"
