"""Python mirror of the reference's reduction API (/root/reference/proj/include/tcreduce/reduction.hpp).

Same names, same argument meaning, same error behaviour (std::invalid_argument -> ValueError,
std::out_of_range -> IndexError).  Every call goes through the C ABI into the sm_100a
kernels; nothing here computes a sum on the host.

    reduce(x, cfg)               reduction.hpp:344   (x: host float32 array or CUDA tensor)
    single_pass_reduce(x, cfg)   reduction.hpp:281
    ReductionConfig / validate   reduction.hpp:39-57
    ReductionOutcome             reduction.hpp:59-67
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum

import numpy as np

from . import _capi


class Variant(enum.IntEnum):          # reduction.hpp:23
    oracle64 = 0
    shuffle32 = 1
    half_tree = 2
    recurrence = 3
    single_pass = 4
    split = 5


class AtomicOrder(enum.IntEnum):      # reduction.hpp:25
    ascending = 0
    seeded_permutation = 1


class Finalize(enum.IntEnum):         # device-side combine of block results (tcreduce_b200.h)
    tree = 0
    ordered = 1
    atomic = 2


class Engine(enum.IntEnum):          # tcreduce_b200.h tcr_engine
    auto = 0
    mma_sync = 1          # TMA bulk ring + ldmatrix.trans + HMMA
    tcgen05 = 2           # tensor-map TMA (SW32) + tcgen05.mma into TMEM
    mma_sync_regs = 3     # 128-bit loads into registers + MOVM + HMMA (tails, fp32 input)
    mma_sync_async = 4    # per-warp cp.async ring + ldmatrix.trans + HMMA


class DistKind(enum.IntEnum):         # harness.hpp:20
    normal = 0
    uniform = 1
    integers = 2
    constant = 3


def variant_name(v: Variant) -> str:  # reduction.hpp:27-37
    return Variant(v).name


@dataclasses.dataclass
class ReductionConfig:
    variant: Variant = Variant.single_pass
    m: int = 4
    R: int = 1
    B: int = 128
    f: float = 0.5
    atomic_order: AtomicOrder = AtomicOrder.ascending
    atomic_seed: int = 0
    finalize: Finalize = Finalize.ordered   # the reference's serial combine (reduction.hpp:257-268)
    engine: Engine = Engine.auto

    def warps_per_block(self) -> int:
        return self.B // 32

    def to_c(self) -> _capi.tcr_config:
        return _capi.tcr_config(int(self.variant), self.m, self.R, self.B, float(self.f), int(self.atomic_order),
                                self.atomic_seed, int(self.finalize), int(self.engine))

    def validate(self) -> None:
        """ReductionConfig::validate (reduction.hpp:50-56); raises ValueError."""
        c = self.to_c()
        _capi.check(_capi.load().tcr_validate(C.byref(c)))


@dataclasses.dataclass
class ReductionOutcome:
    value: float = 0.0
    overflow: bool = False
    level_count: int = 0
    sim_steps: int = 0
    mma_count: int = 0
    atomic_count: int = 0
    shuffle_count: int = 0

    @classmethod
    def from_c(cls, o: _capi.tcr_outcome) -> "ReductionOutcome":
        return cls(o.value, bool(o.overflow), o.level_count, o.sim_steps, o.mma_count, o.atomic_count,
                   o.shuffle_count)


def _stream_ptr(t) -> int:
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def reduce(x, cfg: ReductionConfig) -> ReductionOutcome:
    """reduce() (reduction.hpp:344-358).

    x may be a host float32 array (the reference's std::span<const float>: copied to the
    device, converted to binary16 with round-to-nearest-even inside the kernel), a host float16
    array (binary16 values, half the copy bytes; same result as its float32 widening), a CPU
    tensor of either dtype, or a CUDA tensor of dtype float16 / float32 (device resident, no copy)."""
    lib = _capi.load()
    c = cfg.to_c()
    out = _capi.tcr_outcome()
    import torch
    if isinstance(x, torch.Tensor) and not x.is_cuda:
        x = x.contiguous().numpy()
    if isinstance(x, np.ndarray) or isinstance(x, (list, tuple)):
        if isinstance(x, np.ndarray) and x.dtype == np.float16:
            a = np.ascontiguousarray(x)
            _capi.check(lib.tcr_reduce_f16_host(a.ctypes.data_as(C.c_void_p), a.size, C.byref(c), C.byref(out)))
        else:
            a = np.ascontiguousarray(x, dtype=np.float32)
            _capi.check(lib.tcr_reduce_f32_host(a.ctypes.data_as(C.c_void_p), a.size, C.byref(c), C.byref(out)))
        return ReductionOutcome.from_c(out)
    if not isinstance(x, torch.Tensor):
        raise TypeError("x must be a host float16/float32 array or a tensor")
    x = x.contiguous()
    if x.dtype == torch.float16:
        fn = lib.tcr_reduce_f16_device
    elif x.dtype == torch.float32:
        fn = lib.tcr_reduce_f32_device
    else:
        raise TypeError(f"unsupported dtype {x.dtype}")
    with torch.cuda.device(x.device):
        _capi.check(fn(C.c_void_p(x.data_ptr()), x.numel(), C.byref(c), C.byref(out), C.c_void_p(_stream_ptr(x))))
    return ReductionOutcome.from_c(out)


def single_pass_reduce(x, cfg: ReductionConfig) -> ReductionOutcome:
    """single_pass_reduce (reduction.hpp:281-293): cfg taken by value, variant forced."""
    cfg = dataclasses.replace(cfg, variant=Variant.single_pass)
    return reduce(x, cfg)


def block_count(n: int, cfg: ReductionConfig) -> int:
    c = cfg.to_c()
    return _capi.load().tcr_block_count(n, C.byref(c))


def block_results(x, cfg: ReductionConfig):
    """Per-block fp32 results of single_pass (reduction.hpp:248-255) as a CUDA float32 tensor.
    x: binary16 CUDA tensor, or float32 (the reference's format: from_single applied by the fp32
    paths, fused into the load where the engine has it)."""
    import torch
    if x.dtype not in (torch.float16, torch.float32):
        raise TypeError(f"block_results takes a float16 or float32 tensor, got {x.dtype}")
    x = x.contiguous()
    c = cfg.to_c()
    nb = block_count(x.numel(), cfg)
    out = torch.empty(nb, dtype=torch.float32, device=x.device)
    lib = _capi.load()
    fn = lib.tcr_block_results_f16_device if x.dtype == torch.float16 else lib.tcr_block_results_f32_device
    with torch.cuda.device(x.device):
        _capi.check(fn(C.c_void_p(x.data_ptr()), x.numel(), C.byref(c), C.c_void_p(out.data_ptr()),
                       C.c_void_p(_stream_ptr(x))))
    return out


def single_pass_async(x, cfg: ReductionConfig, result, overflow) -> None:
    """Enqueue single_pass on the current stream; result (float32[1]) and overflow (int32[1]) stay on device."""
    import torch
    if x.dtype not in (torch.float16, torch.float32):
        raise TypeError(f"single_pass_async takes float16 or float32, got {x.dtype}")
    x = x.contiguous()
    lib = _capi.load()
    c = cfg.to_c()
    fn = lib.tcr_single_pass_f16_async if x.dtype == torch.float16 else lib.tcr_single_pass_f32_async
    _capi.check(fn(C.c_void_p(x.data_ptr()), x.numel(), C.byref(c), C.c_void_p(result.data_ptr()),
                   C.c_void_p(overflow.data_ptr()), C.c_void_p(_stream_ptr(x))))


def generate(dist, seed: int, n: int, device="cuda", dtype="float16", lo: int = 0, hi: int = 9, c: float = 1.0,
             first: int = 0, out=None):
    """harness.hpp:47-80 on the device: elements [first, first+n) of generate(dist, N)."""
    import torch
    kind = int(DistKind[dist]) if isinstance(dist, str) else int(dist)
    tdt = torch.float16 if dtype in ("float16", torch.float16) else torch.float32
    if out is None:
        out = torch.empty(n, dtype=tdt, device=device)
    lib = _capi.load()
    fn = lib.tcr_generate_f16_device if out.dtype == torch.float16 else lib.tcr_generate_f32_device
    with torch.cuda.device(out.device):
        _capi.check(fn(C.c_void_p(out.data_ptr()), n, kind, seed, lo, hi, float(c), first,
                       C.c_void_p(_stream_ptr(out))))
    return out


def exact_sum(x) -> tuple[float, float]:
    """Exact sum and sum |x| of a CUDA float16 tensor (fixed point on the device)."""
    s, a = C.c_double(), C.c_double()
    with __import__("torch").cuda.device(x.device):
        _capi.check(_capi.load().tcr_exact_sum_f16_device(C.c_void_p(x.data_ptr()), x.numel(), C.byref(s),
                                                          C.byref(a), C.c_void_p(_stream_ptr(x))))
    return s.value, a.value


def counters(n: int, cfg: ReductionConfig) -> ReductionOutcome:
    c = cfg.to_c()
    out = _capi.tcr_outcome()
    _capi.check(_capi.load().tcr_single_pass_counters(n, C.byref(c), C.byref(out)))
    return ReductionOutcome.from_c(out)


def last_launch_count() -> int:
    return _capi.load().tcr_last_launch_count()


def last_engine() -> Engine:
    return Engine(_capi.load().tcr_last_engine())
