"""tcreduce on B200: the chained tensor-core arithmetic reduction of arXiv 2001.05585, sm_100a-native.

The reduction runs in hand-written sm_100a kernels (libtcreduce_b200.so) behind a C ABI
(include/tcreduce_b200.h); this package is the Python mirror of the reference's
``tcreduce`` API (reduction.hpp) over that ABI.  There is no CPU fallback.
"""
from .reduction import (AtomicOrder, DistKind, Engine, Finalize, ReductionConfig, ReductionOutcome, Variant,
                        block_count, block_results, counters, exact_sum, generate, reduce, single_pass_async,
                        single_pass_reduce, variant_name)

__all__ = ["AtomicOrder", "DistKind", "Engine", "Finalize", "ReductionConfig", "ReductionOutcome", "Variant",
           "block_count", "block_results", "counters", "exact_sum", "generate", "reduce", "single_pass_async",
           "single_pass_reduce", "variant_name"]
