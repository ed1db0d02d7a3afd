"""B200-native Apophenia repeat-finding hot path (arXiv 2406.18111).

The product is libapo.so (C ABI in include/apo.h, sm_100a CUDA kernels in
csrc/); this package is its thin Python binding.  No CPU fallback.
"""
from .apo import (ApoError, Context, History, Trie, default_context, exported_symbols, load_library,  # noqa: F401
                  candidates, find_repeats, find_repeats_batched, suffix_array, suffix_array_batched)

__all__ = ["ApoError", "Context", "History", "Trie", "default_context", "exported_symbols", "load_library", "candidates",
           "find_repeats", "find_repeats_batched", "suffix_array", "suffix_array_batched"]
