"""B200-native (sm_100a) Arc Blanc ocean hot path (arXiv 2503.03326).

Native library: paper_2503_03326_b200/lib/libocean_b200.so (C-ABI in
include/ocean_b200.h). Python mirror of the reference API: `ocean`.
"""
__all__ = ["ocean", "build"]
