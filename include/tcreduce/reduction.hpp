// tcreduce/reduction.hpp -- drop-in replacement for the reference header of the same name
// (/root/reference/proj/include/tcreduce/reduction.hpp), backed by the B200 kernels.
//
// Same namespace, types, function names, argument meaning and exception types.  A caller of
// the reference switches by putting this include/ directory first on the include path and
// linking paper_2001_05585_b200/libtcreduce_b200.so.  The reduction itself runs on the GPU
// through the C ABI in tcreduce_b200.h; nothing in this header sums on the host.
//
//   reference                                     here
//   reduce(span<const float>, cfg)   :344        -> tcr_reduce_f32_host
//   single_pass_reduce(span, cfg)    :281        -> tcr_reduce_f32_host (variant forced)
//   ReductionConfig{...}.validate()  :39-57      -> tcr_validate
//   ReductionOutcome                 :59-67      -> tcr_outcome
//   warp_offset                      :154-158    (pure index arithmetic, kept inline)
//
//   oracle64 / shuffle32_reduce /
//   half_tree_reduce / recurrence_reduce /
//   split_reduce                     :106-341    -> tcr_reduce_f32_host (variant set)
//   chained_warp_reduce              :164-184    -> one warp chunk as a one-block single_pass
//   detail::SimCounters, MmaStats    :71-82, fragment.hpp:16-20 (counter structs)
//
// Additions (B200-only): ReductionConfig::finalize / engine, and device-pointer overloads
// reduce_device_f16 / reduce_device_f32 for data already resident in HBM.
//
// The reference's own unit tests (proj/tests/test_reduction.cpp, test_harness.cpp) compile
// against this header unchanged (oracle/Makefile target ref_tests) and pass on the B200.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>

#include "tcreduce_b200.h"

// The reference's reduction.hpp includes its fragment/half emulator headers; when they are on
// the include path (a caller that keeps the reference tree behind this directory), pull them in
// the same way so code using Half / HalfFragment / MmaStats keeps compiling.
#if __has_include("tcreduce/fragment.hpp")
#include "tcreduce/fragment.hpp"
#define TCREDUCE_B200_REFERENCE_FRAGMENT 1
#endif

namespace tcreduce {

enum class Variant { oracle64, shuffle32, half_tree, recurrence, single_pass, split };

enum class AtomicOrder { ascending, seeded_permutation };

// How the GPU combines block results (the reference serialises them, reduction.hpp:257-268).
enum class Finalize { tree, ordered, atomic };

// Kernel family (tcr_engine): automatic = measured best (mma_sync_async for m = 16).
enum class Engine { automatic, mma_sync, tcgen05, mma_sync_regs, mma_sync_async };

inline const char* variant_name(Variant v) {
    switch (v) {
        case Variant::oracle64: return "oracle64";
        case Variant::shuffle32: return "shuffle32";
        case Variant::half_tree: return "half_tree";
        case Variant::recurrence: return "recurrence";
        case Variant::single_pass: return "single_pass";
        case Variant::split: return "split";
    }
    return "?";
}

namespace detail {

[[noreturn]] inline void raise(int rc) {
    const std::string msg = tcr_last_error();
    if (rc == TCR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == TCR_OUT_OF_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error("tcreduce-b200 error " + std::to_string(rc) + ": " + msg);
}

inline void check(int rc) {
    if (rc != TCR_OK) raise(rc);
}

}  // namespace detail

struct ReductionConfig {
    Variant variant = Variant::single_pass;
    std::size_t m = 4;        // fragment side
    unsigned R = 1;           // MMA chain length per warp
    unsigned B = 128;         // block size in threads, multiple of 32
    double f = 0.5;           // tensor fraction, split variant only
    AtomicOrder atomic_order = AtomicOrder::ascending;
    std::uint64_t atomic_seed = 0;
    Finalize finalize = Finalize::ordered;   // the reference's serial combine (reduction.hpp:257-268)
    Engine engine = Engine::automatic;

    unsigned warps_per_block() const { return B / 32; }

    tcr_config to_c() const {
        tcr_config c;
        tcr_config_init(&c);
        c.variant = static_cast<int32_t>(variant);
        c.m = m > 0xFFFFFFFFu ? 0u : static_cast<uint32_t>(m);
        c.R = R;
        c.B = B;
        c.f = f;
        c.atomic_order = static_cast<int32_t>(atomic_order);
        c.atomic_seed = atomic_seed;
        c.finalize = static_cast<int32_t>(finalize);
        c.engine = static_cast<int32_t>(engine);
        return c;
    }

    void validate() const {
        const tcr_config c = to_c();
        detail::check(tcr_validate(&c));
    }
};

#ifndef TCREDUCE_B200_REFERENCE_FRAGMENT
// fragment.hpp:16-20 (the counter struct the reference's MMA emulation fills).
struct MmaStats {
    std::uint64_t mma_count = 0;
    std::uint64_t loads = 0;
    std::uint64_t stores = 0;
};
#endif

struct ReductionOutcome {
    double value = 0.0;       // binary32 result (binary64 for the oracle)
    bool overflow = false;    // some Half produced during the run was non-finite
    std::uint64_t level_count = 0;
    std::uint64_t sim_steps = 0;
    std::uint64_t mma_count = 0;
    std::uint64_t atomic_count = 0;
    std::uint64_t shuffle_count = 0;
};

namespace detail {

// reduction.hpp:71-82: running counters of one reduction.
struct SimCounters {
    MmaStats mma;
    std::uint64_t atomic_count = 0;
    std::uint64_t shuffle_count = 0;
    std::uint64_t sim_steps = 0;
    bool overflow = false;
};

inline ReductionOutcome from_c(const tcr_outcome& o) {
    ReductionOutcome r;
    r.value = o.value;
    r.overflow = o.overflow != 0;
    r.level_count = o.level_count;
    r.sim_steps = o.sim_steps;
    r.mma_count = o.mma_count;
    r.atomic_count = o.atomic_count;
    r.shuffle_count = o.shuffle_count;
    return r;
}

}  // namespace detail

// Base index of a warp's contiguous chunk of R*m^2 elements (reduction.hpp:154-158).
inline std::size_t warp_offset(std::size_t block_id, std::size_t warp_in_block, const ReductionConfig& cfg) {
    return static_cast<std::size_t>(cfg.R) * cfg.m * cfg.m * (block_id * cfg.warps_per_block() + warp_in_block);
}

// Dispatch on cfg.variant (reduction.hpp:344-358), host fp32 input.
inline ReductionOutcome reduce(std::span<const float> x, const ReductionConfig& cfg) {
    const tcr_config c = cfg.to_c();
    tcr_outcome o;
    detail::check(tcr_reduce_f32_host(x.data(), x.size(), &c, &o));
    return detail::from_c(o);
}

// reduction.hpp:281-293 (cfg by value, variant forced).
inline ReductionOutcome single_pass_reduce(std::span<const float> x, ReductionConfig cfg) {
    cfg.variant = Variant::single_pass;
    return reduce(x, cfg);
}

// reduction.hpp:106-110: binary64 sum (0 for an empty span, as the reference).
inline double oracle64(std::span<const float> x) {
    ReductionConfig cfg;
    cfg.variant = Variant::oracle64;
    return reduce(x, cfg).value;
}

// reduction.hpp:113-122 / :126-151: bit-exact strided pairwise trees (fp32 / binary16 partials).
inline ReductionOutcome shuffle32_reduce(std::span<const float> x) {
    ReductionConfig cfg;
    cfg.variant = Variant::shuffle32;
    return reduce(x, cfg);
}

inline ReductionOutcome half_tree_reduce(std::span<const float> x) {
    ReductionConfig cfg;
    cfg.variant = Variant::half_tree;
    return reduce(x, cfg);
}

// reduction.hpp:189-231 and :298-341 (cfg by value, variant forced).
inline ReductionOutcome recurrence_reduce(std::span<const float> x, ReductionConfig cfg) {
    cfg.variant = Variant::recurrence;
    return reduce(x, cfg);
}

inline ReductionOutcome split_reduce(std::span<const float> x, ReductionConfig cfg) {
    cfg.variant = Variant::split;
    return reduce(x, cfg);
}

// reduction.hpp:164-184: the warp chunk x[base, base + R m^2) through the tensor-core chain and
// the finishing MMA -- on the device, as a single_pass over that chunk with one warp per block
// (its one block result IS the chunk result).  Same out_of_range contract and counter updates.
inline float chained_warp_reduce(std::span<const float> x, std::size_t base, const ReductionConfig& cfg,
                                 detail::SimCounters& sc) {
    const std::size_t chunk = static_cast<std::size_t>(cfg.R) * cfg.m * cfg.m;
    if (base + chunk > x.size()) throw std::out_of_range("chained_warp_reduce: chunk exceeds input");
    if (cfg.R == 0) {   // no chain: the finishing MMA of a zero accumulator
        ++sc.mma.mma_count;
        return 0.0f;
    }
    ReductionConfig one = cfg;
    one.variant = Variant::single_pass;
    one.B = 32;
    const ReductionOutcome o = reduce(x.subspan(base, chunk), one);
    sc.mma.mma_count += cfg.R + 1ull;
    sc.mma.loads += cfg.R;
    sc.overflow = sc.overflow || o.overflow;
    return static_cast<float>(o.value);
}

// Device-resident input (binary16 bits or fp32), result synchronously on the host.
inline ReductionOutcome reduce_device_f16(const std::uint16_t* d_x, std::size_t n, const ReductionConfig& cfg,
                                          void* cuda_stream = nullptr) {
    const tcr_config c = cfg.to_c();
    tcr_outcome o;
    detail::check(tcr_reduce_f16_device(d_x, n, &c, &o, cuda_stream));
    return detail::from_c(o);
}

inline ReductionOutcome reduce_device_f32(const float* d_x, std::size_t n, const ReductionConfig& cfg,
                                          void* cuda_stream = nullptr) {
    const tcr_config c = cfg.to_c();
    tcr_outcome o;
    detail::check(tcr_reduce_f32_device(d_x, n, &c, &o, cuda_stream));
    return detail::from_c(o);
}

}  // namespace tcreduce
