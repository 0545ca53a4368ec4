"""ctypes binding of the C ABI declared in include/tcreduce_b200.h.

This is the same binding a maintainer would add to a Python caller of the reference
(INTEGRATION.md).  The library is loaded from the package directory only; when it is
missing the import fails loudly -- there is no CPU fallback anywhere in the package.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libtcreduce_b200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "tcreduce_b200.h")

TCR_OK = 0
TCR_INVALID_ARGUMENT = -1
TCR_OUT_OF_RANGE = -2
TCR_CUDA_ERROR = -3
TCR_NCCL_ERROR = -4
TCR_NOT_SUPPORTED = -5


class tcr_config(C.Structure):
    _fields_ = [("variant", C.c_int32), ("m", C.c_uint32), ("R", C.c_uint32), ("B", C.c_uint32),
                ("f", C.c_double), ("atomic_order", C.c_int32), ("atomic_seed", C.c_uint64),
                ("finalize", C.c_int32), ("engine", C.c_int32)]


class tcr_outcome(C.Structure):
    _fields_ = [("value", C.c_double), ("overflow", C.c_int32), ("level_count", C.c_uint64),
                ("sim_steps", C.c_uint64), ("mma_count", C.c_uint64), ("atomic_count", C.c_uint64),
                ("shuffle_count", C.c_uint64)]


_P = C.c_void_p
_SZ = C.c_size_t
_CFG = C.POINTER(tcr_config)
_OUT = C.POINTER(tcr_outcome)

SIGNATURES = {
    "tcr_config_init": (None, [_CFG]),
    "tcr_validate": (C.c_int, [_CFG]),
    "tcr_reduce_f32_host": (C.c_int, [_P, _SZ, _CFG, _OUT]),
    "tcr_reduce_f16_host": (C.c_int, [_P, _SZ, _CFG, _OUT]),
    "tcr_reduce_f32_device": (C.c_int, [_P, _SZ, _CFG, _OUT, _P]),
    "tcr_reduce_f16_device": (C.c_int, [_P, _SZ, _CFG, _OUT, _P]),
    "tcr_single_pass_f16_async": (C.c_int, [_P, _SZ, _CFG, _P, _P, _P]),
    "tcr_single_pass_f32_async": (C.c_int, [_P, _SZ, _CFG, _P, _P, _P]),
    "tcr_block_results_f16_device": (C.c_int, [_P, _SZ, _CFG, _P, _P]),
    "tcr_block_results_f32_device": (C.c_int, [_P, _SZ, _CFG, _P, _P]),
    "tcr_reduce_f16_sharded": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.POINTER(C.c_int32), C.c_int32,
                                         _CFG, _OUT]),
    "tcr_block_count": (_SZ, [_SZ, _CFG]),
    "tcr_single_pass_counters": (C.c_int, [_SZ, _CFG, _OUT]),
    "tcr_group_elems": (_SZ, [_CFG]),
    "tcr_generate_f16_device": (C.c_int, [_P, _SZ, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_double,
                                          _SZ, _P]),
    "tcr_generate_f32_device": (C.c_int, [_P, _SZ, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_double,
                                          _SZ, _P]),
    "tcr_exact_sum_f16_device": (C.c_int, [_P, _SZ, C.POINTER(C.c_double), C.POINTER(C.c_double), _P]),
    "tcr_shuffle_f16_async": (C.c_int, [_P, _SZ, _P, _P]),
    "tcr_cub_sum_f16_async": (C.c_int, [_P, _SZ, C.c_int, _P, _P]),
    "tcr_read_probe_async": (C.c_int, [_P, _SZ, _P]),
    "tcr_last_launch_count": (C.c_int, []),
    "tcr_release_stream": (C.c_int, [_P]),
    "tcr_release_all": (C.c_int, []),
    "tcr_last_engine": (C.c_int, []),
    "tcr_last_error": (C.c_char_p, []),
    "tcr_version": (C.c_char_p, []),
    "tcr_enable_profiling_knobs": (C.c_int, []),
    "tcr_reset_profiling_knobs": (None, []),
    "tcr_debug_timestamps": (C.c_int, [_P, _SZ]),
    "tcr_ordered_stats": (C.c_int, [_P]),
}

_lib = None


class TcrError(RuntimeError):
    pass


def load():
    """Load libtcreduce_b200.so (build it first with __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`. "
                              "The package has no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a tcr_status to the Python analogue of the reference's exception types."""
    if rc == TCR_OK:
        return
    msg = load().tcr_last_error().decode(errors="replace")
    if rc == TCR_INVALID_ARGUMENT:
        raise ValueError(msg)          # std::invalid_argument
    if rc == TCR_OUT_OF_RANGE:
        raise IndexError(msg)          # std::out_of_range
    if rc == TCR_NOT_SUPPORTED:
        raise NotImplementedError(msg)
    raise TcrError(f"tcreduce error {rc}: {msg}")


@contextlib.contextmanager
def profiling_knobs(env: dict):
    """Profiling / A-B only: apply TCR_* knobs (e.g. {"TCR_SPLIT": "4"}) for the duration of the
    block.  The library never reads the environment by itself (tcr_enable_profiling_knobs reads
    it once, here); on exit the variables and the production defaults are restored."""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        load().tcr_enable_profiling_knobs()
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        load().tcr_reset_profiling_knobs()


def header_symbols() -> list[str]:
    """Function names declared in include/tcreduce_b200.h."""
    import re
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(tcr_\w+)\s*\(", text, re.M)))
