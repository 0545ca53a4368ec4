// tcr_pipeline.cuh -- shared sm_100a pipeline pieces: mbarriers, TMA / bulk copies, named
// barriers, the canonical pairwise trees and the last-CTA finaliser.
#pragma once
#include <type_traits>

#include <cuda.h>
#include <cstdint>

#include "tcr_device.cuh"
#include "tcr_kernels.h"

namespace tcr {
namespace pipe {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Watchdog: a pipeline bug must surface as a kernel error, never as a hung GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins == (1u << 28)) __trap();
    }
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ float warp_tree_xor(float v) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const float o = __shfl_xor_sync(kFull, v, off);
        v = (lane_id() & off) ? (o + v) : (v + o);
    }
    return v;
}

// Adjacent pairwise tree ((v0 + v1) + (v2 + v3)) ... over the `seg` (power of two) values
// ld(base), ..., ld(base + seg - 1): compile-time register trees up to 128 values (no
// local-memory stack), a binary-counter stack beyond.
template <int SEG, typename LD>
__device__ __forceinline__ float static_segment_tree(LD ld, uint32_t base) {
    float v[SEG];
#pragma unroll
    for (int i = 0; i < SEG; ++i) v[i] = ld(base + i);
#pragma unroll
    for (int len = SEG; len > 1; len >>= 1)
#pragma unroll
        for (int i = 0; i < len / 2; ++i) v[i] = v[2 * i] + v[2 * i + 1];
    return v[0];
}

template <typename LD>
__device__ __forceinline__ float lane_segment_tree(LD ld, uint32_t base, uint32_t seg) {
    switch (seg) {
    case 1: return ld(base);
    case 2: return static_segment_tree<2>(ld, base);
    case 4: return static_segment_tree<4>(ld, base);
    case 8: return static_segment_tree<8>(ld, base);
    case 16: return static_segment_tree<16>(ld, base);
    case 32: return static_segment_tree<32>(ld, base);
    case 64: return static_segment_tree<32>(ld, base) + static_segment_tree<32>(ld, base + 32);
    case 128: {
        const float a = static_segment_tree<32>(ld, base) + static_segment_tree<32>(ld, base + 32);
        const float b = static_segment_tree<32>(ld, base + 64) + static_segment_tree<32>(ld, base + 96);
        return a + b;
    }
    default: {
        float stk[24];
        int top = 0;
        for (uint32_t i = 0; i < seg; ++i) {
            float v = ld(base + i);
            for (uint32_t b = i; b & 1; b >>= 1) v = stk[--top] + v;
            stk[top++] = v;
        }
        return stk[0];
    }
    }
}

// Adjacent tree over seg (power of two, 4..128) consecutive values at a 16-byte aligned address,
// read with 16-byte L2 loads (__ldcg), all in flight.
template <int SEG>
__device__ __forceinline__ float vec_tree(const float* v) {
    float x[SEG];
#pragma unroll
    for (int i = 0; i < SEG / 4; ++i) {
        const float4 q = __ldcg(reinterpret_cast<const float4*>(v) + i);
        x[4 * i] = q.x;
        x[4 * i + 1] = q.y;
        x[4 * i + 2] = q.z;
        x[4 * i + 3] = q.w;
    }
#pragma unroll
    for (int len = SEG; len > 1; len >>= 1)
#pragma unroll
        for (int i = 0; i < len / 2; ++i) x[i] = x[2 * i] + x[2 * i + 1];
    return x[0];
}

__device__ __forceinline__ float vec_segment_tree(const float* v, uint32_t seg) {
    switch (seg) {
    case 4: return vec_tree<4>(v);
    case 8: return vec_tree<8>(v);
    case 16: return vec_tree<16>(v);
    case 32: return vec_tree<32>(v);
    case 64: return vec_tree<32>(v) + vec_tree<32>(v + 32);
    default: return (vec_tree<32>(v) + vec_tree<32>(v + 32)) + (vec_tree<32>(v + 64) + vec_tree<32>(v + 96));
    }
}

// Canonical adjacent tree over vals[0,count) (zero padded to a power of two) by the first
// `nthr` threads (power of two, multiple of 32); every thread of the CTA must call it.
// REG: per-thread segments of <= 128 values as compile-time register trees with all loads in
// flight at once (the last CTA's finalise of the cp.async engine: ~1 L2 round trip instead of a
// local-memory stack walk); same tree, same result.
template <bool REG = false>
__device__ __forceinline__ float cta_tree(const float* vals, uint64_t count, float* s_scratch, unsigned nthr) {
    uint64_t P = 1;
    while (P < count) P <<= 1;
    uint64_t seg = P / nthr;
    if (seg == 0) seg = 1;
    float acc = 0.0f;
    const uint64_t lo = uint64_t(threadIdx.x) * seg;
    if (REG && seg >= 4 && seg <= 128 && lo + seg <= count) {
        // whole segment inside: 16-byte L2 loads, all in flight, compact code (this path runs
        // once per launch, cold in the instruction cache: fewer instructions = fewer misses)
        if (threadIdx.x < nthr) acc = vec_segment_tree(vals + lo, uint32_t(seg));
    } else if (REG && seg <= 128) {
        if (threadIdx.x < nthr && lo < P)
            acc = lane_segment_tree([&](uint32_t i) { return i < count ? __ldcg(vals + i) : 0.0f; }, uint32_t(lo),
                                    uint32_t(seg));
    } else if (threadIdx.x < nthr && lo < P) {
        float stk[40];
        int top = 0;
        // batches of 8 independent L2 loads in flight, then the same streaming stack order
        for (uint64_t i0 = 0; i0 < seg; i0 += 8) {
            float v8[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t idx = lo + i0 + k;
                v8[k] = (i0 + k < seg && idx < count) ? __ldcg(vals + idx) : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (i0 + k < seg) {
                    float v = v8[k];
                    for (uint64_t b = i0 + k; b & 1; b >>= 1) v = stk[--top] + v;
                    stk[top++] = v;
                }
            }
        }
        acc = stk[0];
    }
    if (threadIdx.x < nthr) {
        acc = warp_tree_xor(acc);
        if (lane_id() == 0) s_scratch[threadIdx.x >> 5] = acc;
    }
    __syncthreads();
    float r = 0.0f;
    if (threadIdx.x < 32) {
        r = lane_id() < (nthr >> 5) ? s_scratch[lane_id()] : 0.0f;
        r = warp_tree_xor(r);
    }
    __syncthreads();
    return r;
}


// reduction.hpp:257-268: serial binary32 accumulation of the block results, ascending or in the
// seeded Fisher-Yates permutation (SplitMix64, rng.hpp).  One thread.
__device__ __forceinline__ float ordered_sum(const SpParams& p) {
    float acc = 0.0f;
    if (p.atomic_order == 1) {
        uint32_t* order = p.order_scratch;
        for (uint64_t i = 0; i < p.n_blocks; ++i) order[i] = uint32_t(i);
        uint64_t st = p.atomic_seed;
        for (uint64_t i = p.n_blocks; i > 1; --i) {
            st += 0x9E3779B97F4A7C15ull;
            uint64_t z = st;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            const uint64_t r = z % i;
            const uint32_t tt = order[i - 1];
            order[i - 1] = order[r];
            order[r] = tt;
        }
        for (uint64_t i = 0; i < p.n_blocks; ++i) acc += __ldcg(p.block_partials + order[i]);
    } else {
        for (uint64_t b = 0; b < p.n_blocks; ++b) acc += __ldcg(p.block_partials + b);
    }
    return acc;
}

// Last-CTA-done finaliser shared by the persistent engines: every thread of the CTA calls it
// after publishing its partials (__threadfence + __syncthreads done by the caller).
// The caller's __syncthreads() after its last global writes makes them visible to thread 0, whose
// fence before the ticket then releases them grid-wide (cumulativity; the cooperative-groups grid
// barrier pattern): no fence by every thread.  stamps (profiling, may be null): %globaltimer
// after the ticket and after the tree, last CTA only.
__device__ __forceinline__ unsigned long long fin_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <bool REG = false>
__device__ __forceinline__ void finalize_last_cta(const SpParams& p, float* s_scratch, int* s_last, unsigned nthr,
                                                  unsigned long long* stamps = nullptr) {
    if (!(p.finalize == kFinTree || p.finalize == kFinOrdered)) return;
    if (threadIdx.x == 0) {
        // one acquire-release RMW: releases the CTA's writes (made visible to thread 0 by the
        // caller's barrier) and, for the last CTA, acquires everybody else's
        unsigned tk;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(tk) : "l"(p.ticket) : "memory");
        *s_last = (tk == gridDim.x - 1);
    }
    __syncthreads();
    if (!*s_last) return;
    if (stamps && threadIdx.x == 0) stamps[0] = fin_gtimer();
    if (p.finalize == kFinTree) {
        const float r = cta_tree<REG>(p.group_partials, p.n_groups, s_scratch, nthr);
        if (threadIdx.x == 0) *p.result = r;
    } else if (threadIdx.x == 0) {
        *p.result = ordered_sum(p);
    }
    if (threadIdx.x == 0) {
        *p.ticket = 0u;
        if (stamps) stamps[1] = fin_gtimer();
    }
}

// Block stage (reference pairwise tree over W chunk results, reduction.hpp:253, :90-101) for the
// nblk logical blocks starting at global block block0, by `nwarps` warps (w = caller's index in
// that set): chunk results chunks[b*W + j] -> blocks[b].
//   W <= 16: one block per LANE (the tree in registers, v[i] += v[i + len/2] over pow2(W));
//   W > 16:  32 blocks per warp pass (transpose-reduce), or one block per warp (shfl_down offsets
//            pow2(W)/2 .. 1 pair the same operands).
__device__ __forceinline__ void publish_block(const SpParams& p, uint64_t gb, float x) {
    if (gb < p.n_blocks) {
        if (p.block_partials) p.block_partials[gb] = x;
        if (p.finalize == kFinAtomic) atomicAdd(p.result, x);
    }
}

template <int PW>   // pow2(W) <= 16
__device__ __forceinline__ float lane_block_tree(const float* chunks, uint32_t W, uint32_t b) {
    float v[PW];
    const float* src = chunks + b * W;
    if (W == uint32_t(PW) && PW == 16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 a = reinterpret_cast<const float4*>(src)[q];
            v[(4 * q) % PW] = a.x; v[(4 * q + 1) % PW] = a.y; v[(4 * q + 2) % PW] = a.z; v[(4 * q + 3) % PW] = a.w;
        }
    } else if (W == uint32_t(PW) && PW == 8) {
        const float4 a = reinterpret_cast<const float4*>(src)[0], c = reinterpret_cast<const float4*>(src)[1];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4 % PW] = c.x; v[5 % PW] = c.y; v[6 % PW] = c.z; v[7 % PW] = c.w;
    } else if (W == uint32_t(PW) && PW == 4) {
        const float4 a = reinterpret_cast<const float4*>(src)[0];
        v[0] = a.x; v[1 % PW] = a.y; v[2 % PW] = a.z; v[3 % PW] = a.w;
    } else if (W == uint32_t(PW) && PW == 2) {
        const float2 a = reinterpret_cast<const float2*>(src)[0];
        v[0] = a.x; v[1 % PW] = a.y;
    } else {
#pragma unroll
        for (int j = 0; j < PW; ++j) v[j] = uint32_t(j) < W ? src[j] : 0.0f;
    }
#pragma unroll
    for (int len = PW; len > 1; len >>= 1)
#pragma unroll
        for (int i = 0; i < len / 2; ++i) v[i] += v[i + len / 2];
    return v[0];
}

__device__ __forceinline__ void range_trees_blocks(const SpParams& p, uint64_t block0, uint32_t nblk,
                                                   const float* chunks, float* blocks, uint32_t w, uint32_t nwarps) {
    const uint32_t W = p.W;
    const unsigned lane = lane_id();
    if (W <= 16) {
        // the W dispatch hoisted out of the block loop (one loop per tree width); W in 9..16
        // (B = 512: one block per lane, 4 vector loads) measured faster than a warp per block
        auto run = [&](auto pw) {
            constexpr int PW = decltype(pw)::value;
            for (uint32_t b = w * 32u + lane; b < nblk; b += nwarps * 32u) {
                const float x = PW == 1 ? chunks[b] : lane_block_tree<PW>(chunks, W, b);
                blocks[b] = x;
                publish_block(p, block0 + b, x);
            }
        };
        if (W == 1) run(std::integral_constant<int, 1>{});
        else if (W == 2) run(std::integral_constant<int, 2>{});
        else if (W <= 4) run(std::integral_constant<int, 4>{});
        else if (W <= 8) run(std::integral_constant<int, 8>{});
        else run(std::integral_constant<int, 16>{});
        return;
    }
    uint32_t P = 1;
    while (P < W) P <<= 1;
    if (P == 32) {
        // 32 blocks per warp pass: lane l loads chunk l of each of the 32 blocks (conflict free),
        // then a transpose-reduce: the step with offset o performs level len = 2o of the
        // reference tree (v[i] += v[i + o]) for half of the blocks a lane still holds, the lane
        // pair l, l^o exchanging the other half; lane l ends with block l.  31 shuffles per 32
        // blocks instead of 5 per block, the same operand pairs.
        for (uint32_t b0 = w * 32u; b0 < nblk; b0 += nwarps * 32u) {
            float v[32];
#pragma unroll
            for (uint32_t r = 0; r < 32; ++r) v[r] = (b0 + r < nblk && lane < W) ? chunks[(b0 + r) * W + lane] : 0.0f;
#pragma unroll
            for (uint32_t o = 16; o >= 1; o >>= 1) {
                const bool up = lane & o;
#pragma unroll
                for (uint32_t r = 0; r < o; ++r) {
                    const float recv = __shfl_xor_sync(kFull, up ? v[r] : v[r + o], o);
                    v[r] = up ? recv + v[r + o] : v[r] + recv;
                }
            }
            if (b0 + lane < nblk) {
                blocks[b0 + lane] = v[0];
                publish_block(p, block0 + b0 + lane, v[0]);
            }
        }
        return;
    }
    for (uint32_t b = w; b < nblk; b += nwarps) {
        float x = lane < W ? chunks[b * W + lane] : 0.0f;
        for (uint32_t off = P >> 1; off >= 1; off >>= 1) x += __shfl_down_sync(kFull, x, off);
        if (lane == 0) {
            blocks[b] = x;
            publish_block(p, block0 + b, x);
        }
    }
}

// Block stage for one whole group (tile) of G blocks.
__device__ __forceinline__ void tile_trees_blocks(const SpParams& p, uint64_t tile, const float* chunks,
                                                  float* blocks, uint32_t w, uint32_t nwarps) {
    range_trees_blocks(p, tile * p.G, p.G, chunks, blocks, w, nwarps);
}

// Group stage: adjacent tree over the G (power of two) block results of group `tile`, by one
// warp: each lane a contiguous segment (streaming binary-counter stack), then the xor tree
// across lanes.  GLOBAL: `blocks` lives in global memory written by other CTAs (L2 loads).
template <bool GLOBAL = false>
__device__ __forceinline__ void tile_tree_group(const SpParams& p, uint64_t tile, const float* blocks) {
    const uint32_t G = p.G;
    const unsigned lane = lane_id();
    if (!p.group_partials) return;
    const uint32_t seg = G >= 32 ? G / 32 : 1;
    auto ld = [&](uint32_t i) -> float {
        if constexpr (GLOBAL) return __ldcg(blocks + i);
        else return blocks[i];
    };
    float x = 0.0f;
    if (lane * seg < G) x = lane_segment_tree(ld, lane * seg, seg);
    x = warp_tree_xor(x);
    if (lane == 0) p.group_partials[tile] = x;
}

// The same group tree by a whole 8-warp CTA (every thread calls): thread t reduces blocks
// [t seg, (t+1) seg) with the register segment tree, the warps' xor trees pair adjacent lanes,
// thread 0 pairs the 8 warp results.  One eighth of the serial work per thread of the one-warp
// version, which matters when G is large (B = 32: G = 1024 blocks per group).
template <bool GLOBAL = false>
__device__ __forceinline__ void tile_tree_group_cta(const SpParams& p, uint64_t tile, const float* blocks) {
    __shared__ float s_w[8];
    const uint32_t G = p.G;
    const uint32_t seg = G >= 256u ? G / 256u : 1u;
    const uint32_t lo = threadIdx.x * seg;
    auto ld = [&](uint32_t i) -> float {
        if constexpr (GLOBAL) return __ldcg(blocks + i);
        else return blocks[i];
    };
    float x = lo < G ? lane_segment_tree(ld, lo, seg) : 0.0f;
    x = warp_tree_xor(x);
    if (lane_id() == 0) s_w[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0 && p.group_partials) {
        const float a = (s_w[0] + s_w[1]) + (s_w[2] + s_w[3]);
        const float b = (s_w[4] + s_w[5]) + (s_w[6] + s_w[7]);
        p.group_partials[tile] = a + b;
    }
}

}  // namespace pipe
}  // namespace tcr
