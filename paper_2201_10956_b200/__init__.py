"""B200-native exhaustive third-order (SNP-triple) K2 epistasis search.

The compute path is native: libepi3cu.so (sm_100a CUDA + C ABI,
include/epi3cu.h). `epi3` is the Python mirror of the reference API over that
ABI; `partition` holds the multi-GPU partition/merge plumbing.
"""
