"""B200-native GraphPy sparse hot path (arxiv 2402.03548): gSpMMv with fused
degree normalisation, gSDDMM, edge softmax and weighted gSpMM over an
edge-ID-carrying CSR/CSC kernel-graph, behind the C ABI of include/gsp.h.

``Graph`` is the ctypes binding of libgsp.so (sm_100a kernels); there is no CPU
fallback.
"""
from .gsp import (BUILD_L2_PERSIST, BUILD_REVERSE, BUILD_SHARE_SYMMETRIC, NORM_BOTH, NORM_NONE, NORM_RIGHT, OP_ADD, OP_DIV,  # noqa: F401
                  OP_MUL, OP_SUB, PART_REVERSE, REDUCE_MAX, REDUCE_MIN, REDUCE_SUM, SIDE_DST, SIDE_SRC, Graph,
                  GspError, gsp_tensor, lib, version)
