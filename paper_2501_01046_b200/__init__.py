"""neardup_b200: B200-native MinHash-LSH near-duplicate detection hot path.

A drop-in for the hot path of the reference CPU library (neardup,
/root/reference/proj): signatures, band keys, bucket grouping, candidate
comparison and union-find clustering run as hand-written sm_100a kernels in
libneardup_b200.so behind the C-ABI of include/neardup_b200.h.  The Python
modules mirror the reference's C++ headers (minhash.hpp, lsh.hpp,
compare.hpp, dedup_graph.hpp, pipeline.hpp).
"""
from . import _lib  # noqa: F401

__version__ = "0.1.0"
