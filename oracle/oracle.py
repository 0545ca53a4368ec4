"""ctypes view of the CPU oracle (liboracle.so) and the compiled reference (_ref/libtcreduce_ref.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg as the *checker* and the CPU baseline -- never by
the product package ``paper_2001_05585_b200``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtcreduce_ref.so")

VARIANTS = {"oracle64": 0, "shuffle32": 1, "half_tree": 2, "recurrence": 3, "single_pass": 4, "split": 5}
DISTS = {"normal": 0, "uniform": 1, "integers": 2, "constant": 3}


class Config(C.Structure):
    """orc_config / ref_config: mirrors ReductionConfig (reduction.hpp:39-57)."""

    _fields_ = [("variant", C.c_int32), ("m", C.c_uint32), ("R", C.c_uint32), ("B", C.c_uint32),
                ("f", C.c_double), ("atomic_order", C.c_int32), ("atomic_seed", C.c_uint64)]


class Outcome(C.Structure):
    """orc_outcome / ref_outcome: mirrors ReductionOutcome (reduction.hpp:59-67)."""

    _fields_ = [("value", C.c_double), ("overflow", C.c_int32), ("level_count", C.c_uint64),
                ("sim_steps", C.c_uint64), ("mma_count", C.c_uint64), ("atomic_count", C.c_uint64),
                ("shuffle_count", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def make_config(variant="single_pass", m=4, R=1, B=128, f=0.5, atomic_order=0, atomic_seed=0):
    if isinstance(variant, str):
        variant = VARIANTS[variant]
    return Config(variant, m, R, B, f, atomic_order, atomic_seed)


def build(force: bool = False) -> None:
    """Build liboracle.so (and _ref when /root/reference exists) with oracle/Makefile."""
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


_orc = None
_ref = None

_F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_U16P = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")


def lib():
    global _orc
    if _orc is None:
        build()
        L = C.CDLL(ORACLE_SO)
        L.orc_from_single.argtypes = [C.c_float]
        L.orc_from_single.restype = C.c_uint16
        L.orc_to_single.argtypes = [C.c_uint16]
        L.orc_to_single.restype = C.c_float
        L.orc_splitmix_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_splitmix_draw.restype = C.c_uint64
        L.orc_generate.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_size_t, _F32P]
        L.orc_generate_range.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_size_t,
                                         C.c_size_t, _F32P]
        L.orc_generate_range_f16.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_double,
                                             C.c_size_t, C.c_size_t, _U16P]
        L.orc_oracle64.argtypes = [_F32P, C.c_size_t]
        L.orc_oracle64.restype = C.c_double
        L.orc_exact_sum_f16.argtypes = [_U16P, C.c_size_t, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_validate.argtypes = [C.POINTER(Config)]
        L.orc_block_count.argtypes = [C.c_size_t, C.POINTER(Config)]
        L.orc_block_count.restype = C.c_size_t
        L.orc_warp_offset.argtypes = [C.c_size_t, C.c_size_t, C.POINTER(Config)]
        L.orc_warp_offset.restype = C.c_size_t
        L.orc_chained_warp_reduce.argtypes = [_F32P, C.c_size_t, C.c_size_t, C.POINTER(Config),
                                              C.POINTER(C.c_float), C.POINTER(C.c_int), C.POINTER(C.c_uint64)]
        for name in ("orc_shuffle32", "orc_half_tree"):
            getattr(L, name).argtypes = [_F32P, C.c_size_t, C.POINTER(Outcome)]
        for name in ("orc_recurrence", "orc_split", "orc_reduce"):
            getattr(L, name).argtypes = [_F32P, C.c_size_t, C.POINTER(Config), C.POINTER(Outcome)]
        L.orc_single_pass.argtypes = [_F32P, C.c_size_t, C.POINTER(Config), C.c_int, C.POINTER(Outcome),
                                      C.c_void_p]
        L.orc_single_pass_f16.argtypes = [_U16P, C.c_size_t, C.POINTER(Config), C.c_int, C.POINTER(Outcome),
                                          C.c_void_p]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference headers compiled as-is (oracle/_ref).  Raises if it was never built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(REF_SO)
        L.ref_from_single.argtypes = [C.c_float]
        L.ref_from_single.restype = C.c_uint16
        L.ref_to_single.argtypes = [C.c_uint16]
        L.ref_to_single.restype = C.c_float
        L.ref_generate.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_size_t, _F32P]
        L.ref_oracle64.argtypes = [_F32P, C.c_size_t]
        L.ref_oracle64.restype = C.c_double
        for name in ("ref_reduce", "ref_single_pass_reduce"):
            getattr(L, name).argtypes = [_F32P, C.c_size_t, C.POINTER(Config), C.POINTER(Outcome)]
        L.ref_validate.argtypes = [C.POINTER(Config)]
        L.ref_chained_warp_reduce.argtypes = [_F32P, C.c_size_t, C.c_size_t, C.POINTER(Config),
                                              C.POINTER(C.c_float), C.POINTER(C.c_uint64)]
        L.ref_warp_offset.argtypes = [C.c_size_t, C.c_size_t, C.POINTER(Config)]
        L.ref_warp_offset.restype = C.c_size_t
        L.ref_single_pass_parallel.argtypes = [_F32P, C.c_size_t, C.POINTER(Config), C.c_int,
                                               C.POINTER(Outcome), C.c_void_p]
        L.ref_csv_header.restype = C.c_char_p
        L.ref_csv_row.argtypes = [C.POINTER(Config), C.c_uint64, C.c_uint64, C.c_char_p, C.c_double, C.c_int,
                                  C.c_double, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_char_p, C.c_size_t]
        L.ref_run_point_csv.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_size_t,
                                        C.POINTER(Config), C.c_char_p, C.c_size_t]
        _ref = L
    return _ref


class OracleError(Exception):
    pass


def _check(rc):
    if rc == -1:
        raise ValueError("invalid_argument")
    if rc == -2:
        raise IndexError("out_of_range")
    if rc:
        raise OracleError(rc)


# ----------------------------------------------------------------------------- oracle API

def generate(dist="uniform", seed=0, n=1, lo=0, hi=9, c=1.0, first=0) -> np.ndarray:
    kind = DISTS[dist] if isinstance(dist, str) else dist
    out = np.empty(n, np.float32)
    if first == 0:
        _check(lib().orc_generate(kind, seed, lo, hi, c, n, out))
    else:
        _check(lib().orc_generate_range(kind, seed, lo, hi, c, first, n, out))
    return out


def generate_f16(dist="uniform", seed=0, n=1, lo=0, hi=9, c=1.0, first=0) -> np.ndarray:
    kind = DISTS[dist] if isinstance(dist, str) else dist
    out = np.empty(n, np.uint16)
    _check(lib().orc_generate_range_f16(kind, seed, lo, hi, c, first, n, out))
    return out


def from_single(x: float) -> int:
    return lib().orc_from_single(x)


def to_single(h: int) -> float:
    return lib().orc_to_single(h)


def oracle64(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, np.float32)
    return lib().orc_oracle64(x, x.size)


def exact_sum_f16(h: np.ndarray):
    h = np.ascontiguousarray(h, np.uint16)
    s, a = C.c_double(), C.c_double()
    lib().orc_exact_sum_f16(h, h.size, C.byref(s), C.byref(a))
    return s.value, a.value


def single_pass(x: np.ndarray, threads: int = 1, want_blocks: bool = False, **cfg):
    """orc_single_pass on fp32 (or binary16 bits if x.dtype == uint16)."""
    c = make_config(**cfg)
    n = x.size
    blocks = lib().orc_block_count(max(n, 1), C.byref(c))
    bo = np.empty(blocks, np.float32) if want_blocks else None
    out = Outcome()
    bp = bo.ctypes.data_as(C.c_void_p) if bo is not None else None
    if x.dtype == np.uint16:
        _check(lib().orc_single_pass_f16(np.ascontiguousarray(x), n, C.byref(c), threads, C.byref(out), bp))
    else:
        _check(lib().orc_single_pass(np.ascontiguousarray(x, np.float32), n, C.byref(c), threads,
                                     C.byref(out), bp))
    return (out, bo) if want_blocks else out


def reduce(x: np.ndarray, **cfg) -> Outcome:
    c = make_config(**cfg)
    out = Outcome()
    x = np.ascontiguousarray(x, np.float32)
    _check(lib().orc_reduce(x, x.size, C.byref(c), C.byref(out)))
    return out


def chained_warp_reduce(x: np.ndarray, base: int, **cfg):
    c = make_config(**cfg)
    x = np.ascontiguousarray(x, np.float32)
    v, ov, mc = C.c_float(), C.c_int(0), C.c_uint64(0)
    _check(lib().orc_chained_warp_reduce(x, x.size, base, C.byref(c), C.byref(v), C.byref(ov), C.byref(mc)))
    return v.value, bool(ov.value), mc.value


# -------------------------------------------------------------------------- reference API

def ref_generate(dist="uniform", seed=0, n=1, lo=0, hi=9, c=1.0) -> np.ndarray:
    kind = DISTS[dist] if isinstance(dist, str) else dist
    out = np.empty(n, np.float32)
    _check(ref().ref_generate(kind, seed, lo, hi, c, n, out))
    return out


def ref_reduce(x: np.ndarray, **cfg) -> Outcome:
    c = make_config(**cfg)
    out = Outcome()
    x = np.ascontiguousarray(x, np.float32)
    _check(ref().ref_reduce(x, x.size, C.byref(c), C.byref(out)))
    return out


def ref_csv_header() -> str:
    """csv.hpp:14-15 kCsvHeader, from the compiled reference."""
    return ref().ref_csv_header().decode()


def ref_csv_row(n, seed, dist, value, error_pct, overflow, sim_steps, mma_count, atomic_count, **cfg) -> str:
    """csv.hpp:19-48 csv_row of a SweepRecord with these fields (error_pct None = nullopt)."""
    c = make_config(**cfg)
    buf = C.create_string_buffer(1024)
    _check(ref().ref_csv_row(C.byref(c), n, seed, dist.encode(), value, 0 if error_pct is None else 1,
                             0.0 if error_pct is None else error_pct, int(bool(overflow)), sim_steps, mma_count,
                             atomic_count, buf, len(buf)))
    return buf.value.decode()


def ref_run_point_csv(dist="uniform", seed=0, n=1, lo=0, hi=9, c=1.0, **cfg) -> str:
    """harness.hpp:103-117 run_point on the CPU reference, as its csv.hpp row."""
    kind = DISTS[dist] if isinstance(dist, str) else dist
    cf = make_config(**cfg)
    buf = C.create_string_buffer(1024)
    _check(ref().ref_run_point_csv(kind, seed, lo, hi, c, n, C.byref(cf), buf, len(buf)))
    return buf.value.decode()


def ref_single_pass_parallel(x: np.ndarray, threads: int, want_blocks: bool = False, **cfg):
    c = make_config(**cfg)
    x = np.ascontiguousarray(x, np.float32)
    blocks = lib().orc_block_count(max(x.size, 1), C.byref(c))
    bo = np.empty(blocks, np.float32) if want_blocks else None
    out = Outcome()
    _check(ref().ref_single_pass_parallel(x, x.size, C.byref(c), threads, C.byref(out),
                                          bo.ctypes.data_as(C.c_void_p) if bo is not None else None))
    return (out, bo) if want_blocks else out
