"""B200-native shadow-page synchronisation (CRUM, arXiv 1808.00117).

The product is libcrum.so (C ABI: include/crum.h) built from csrc/ for
sm_100a; ``paper_1808_00117_b200.crum`` is its thin ctypes binding.  Importing
``paper_1808_00117_b200.crum`` fails loudly if the library has not been built
-- there is no CPU fallback.
"""
