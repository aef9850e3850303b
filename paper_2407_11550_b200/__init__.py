"""B200-native Ada-KV (arXiv 2407.11550) compression + compressed-decode path.

The product is the C-ABI CUDA library lib/libadakv_b200.so (include/adakv_b200.h)
and its C++ drop-in header (include/adakv_b200/adakv.hpp).  This package is the
Python host side: ctypes bindings (_lib), torch-tensor ops (ops), the model-level
pipeline (pipeline) and multi-GPU sharding (sharding).
"""
from ._lib import AdaKVError, InvalidArgument, OutOfRange, lib  # noqa: F401
from .ops import (CompressedCache, append_kv, append_rows, apportion, compress, decode,  # noqa: F401
                  pyramid_layer_budgets, repair_zero_budgets, safeguard_blend, segmented_select,
                  uniform_allocation, window_scores, workspace_status)

__all__ = ["AdaKVError", "InvalidArgument", "OutOfRange", "CompressedCache", "compress", "decode",
           "append_kv", "append_rows", "window_scores", "segmented_select", "apportion", "uniform_allocation",
           "safeguard_blend", "repair_zero_budgets", "pyramid_layer_budgets", "workspace_status", "lib"]
