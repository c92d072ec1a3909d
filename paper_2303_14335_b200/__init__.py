"""B200-native MPLD hot path (arxiv 2303.14335): exact-cover layout decomposition
in CUDA for sm_100a behind the C ABI of include/mpld.h.  See DESIGN.md."""
from .mpld import (MPLDError, Context, lib, version, mpld_decompose, mpld_decompose_batch, decompose_graph,
                   EXPORTS, STAT_NAMES, MPLD_FLAG_VALIDATE, MPLD_FLAG_TILES, MPLD_MAX_COMPONENT, MPLD_MAX_K)

__all__ = ["MPLDError", "Context", "lib", "version", "mpld_decompose", "mpld_decompose_batch", "decompose_graph",
           "EXPORTS", "STAT_NAMES", "MPLD_FLAG_VALIDATE", "MPLD_FLAG_TILES", "MPLD_MAX_COMPONENT", "MPLD_MAX_K"]
