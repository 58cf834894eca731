"""B200-native R-Sparse rank-aware sparse linear operator (arXiv 2504.19449).

The product is librsparse_b200.so (C ABI in include/rsparse_b200.h,
hand-written sm_100a kernels in csrc/).  This package is the host-side
mirror of the reference's operator API over that ABI.
"""
from ._lib import (CudaError, IoError, NumericError, RspError, UsageError,  # noqa: F401
                   lib)
from . import model, offline  # noqa: F401  (mlp_forward / apply_linear; decompose / scores on the GPU)
from .layer import (BatchedStack, DecomposedLayer, IoReport, Recipe, SparsityPlan, Stack,  # noqa: F401
                    TokenParallelStack,
                    forward, gather_matvec, io_cost, keep_count, read_decomposed_layer, read_rspl,
                    read_rspl_header, shard_rows, threshold_sparsify, top_k_by_magnitude,
                    write_decomposed_layer)

__all__ = [
    "DecomposedLayer", "SparsityPlan", "IoReport", "Recipe", "Stack", "TokenParallelStack", "BatchedStack",
    "forward", "io_cost",
    "gather_matvec", "threshold_sparsify", "top_k_by_magnitude", "keep_count", "shard_rows", "lib",
    "read_decomposed_layer", "write_decomposed_layer", "read_rspl", "read_rspl_header",
    "RspError", "UsageError", "NumericError", "IoError", "CudaError", "offline", "model",
]
