"""B200-native MACE symmetric tensor contraction (arXiv 2504.10700), product package.

libsymcon.so (C ABI, include/symcon.h) holds every step of the hot path; this package only
marshals arguments (`_lib`), manages device memory / streams / autograd (`ops`) and the
sharded data-parallel step (`dist`).
"""
