// tcr_sp_async.cu -- single-pass chained reduction, m = 16: per-warp cp.async pipeline engine.
//
// Same element partition, block stage and group stage as the other engines (reference
// reduction.hpp:164-184, :238-275).  Every warp owns a private ring of D fragment stages
// (512 B each) in shared memory and streams its own warp-chunks through it:
//
//   cp.async.cg 16 B per lane (LDGSTS, L1 bypass) -> stage (f + D-1) % D, one commit group per
//   fragment; cp.async.wait_group(D-1) retires fragment f; ONE ldmatrix.x4.trans hands every
//   lane the A fragment whose row j is column j of the 16x16 fragment (all 16 k), ONE
//   HMMA.16816 against ones accumulates C_r = ones x M_r + C_{r-1} (reduction.hpp:177).
//   C_R -> binary16 and the finishing HMMA run once per two chunks.
//
// No CTA-wide synchronisation inside the stream: D-1 fragments per warp are always in flight
// without holding registers, and the zero-fill form of cp.async gives the reference's zero
// padding (reduction.hpp:244-245) for the ragged tail for free.  The destination of each
// 16-byte line is XOR-swizzled on row bit 2 so the transposing ldmatrix is bank-conflict free.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <cuda_runtime.h>

#include "tcr_device.cuh"
#include "tcr_kernels.h"
#include "tcr_pipeline.cuh"

namespace tcr {

namespace {

using namespace pipe;

constexpr int kAsWarps = 8;
constexpr int kAsThreads = 32 * kAsWarps;
constexpr int kAsStageBytes = 512;

// L2 prefetch granularity of the 16-byte copies (PF: 0 none, 128, 256 bytes)
template <int PF = 256>
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, uint32_t src_bytes) {
    if constexpr (PF == 256)
        asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes)
                     : "memory");
    else if constexpr (PF == 128)
        asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes)
                     : "memory");
    else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes) : "memory");
}
// Same copy with an L2 eviction-priority policy (the streamed input is read exactly once).
__device__ __forceinline__ void cp_async16_pol(uint32_t saddr, const void* g, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint.L2::256B [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& d0, uint32_t& d1, uint32_t& d2, uint32_t& d3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3)
                 : "r"(addr));
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// byte offset of line (k, half) of a fragment stage, swizzled: half ^= bit 2 of k
__device__ __forceinline__ uint32_t swz(uint32_t k, uint32_t half) { return 32u * k + 16u * (half ^ ((k >> 2) & 1u)); }

// One work unit = Cu consecutive chunks starting at global chunk c0 (a whole group or a piece of
// whole blocks of it): warp w takes the unit's chunks w, w + 8, w + 16, ...; chunk results to
// s_chunk[unit-local chunk].  Any R, any tail (zero-fill copies past n).
template <int RT, int D>
__device__ __forceinline__ void as_unit(const SpParams& p, uint64_t c0, uint32_t Cu, uint32_t ring_saddr,
                                        float* s_chunk, bool& ovf) {
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned c = lane & 3u;
    const uint32_t R = RT > 0 ? uint32_t(RT) : p.R;
    const uint32_t nch = Cu > warp ? (Cu - warp + kAsWarps - 1) / kAsWarps : 0;
    const uint32_t F = nch * R;
    const uint64_t ce = uint64_t(R) * 256u;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    const uint64_t n = p.n;
    // copy side: lane copies bytes [16*lane, 16*lane+16) of the fragment = line (k = lane/2, half = lane&1)
    const uint32_t cp_dst = swz(lane >> 1, lane & 1u);
    // ldmatrix side: matrix mi = lane>>3 supplies line (k = (lane&7) + 8*(mi>>1), half = mi&1)
    const uint32_t mi = lane >> 3;
    const uint32_t ld_off = swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);

    // issue cursor (called with f = 0, 1, 2, ... in order): element of fragment f for this warp,
    // advanced by increments instead of a division by the runtime R
    uint64_t ie = (c0 + warp) * ce + 8u * lane;
    uint32_t ir = 0;
    const uint64_t chunk_step = uint64_t(kAsWarps) * ce - uint64_t(R - 1) * 256u;
    auto issue = [&](uint32_t f) {
        if (f < F) {
            const uint64_t e = ie;
            const uint32_t bytes = e + 8 <= n ? 16u : (e < n ? uint32_t(n - e) * 2u : 0u);
            cp_async16(ring_saddr + (f % D) * kAsStageBytes + cp_dst, x + (e < n ? e : 0), bytes);
            if (++ir == R) {
                ir = 0;
                ie += chunk_step;
            } else {
                ie += 256u;
            }
        }
        cp_async_commit();
    };

#pragma unroll
    for (int f = 0; f < D - 1; ++f) issue(uint32_t(f));

    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t r = 0, ci = 0, pend = 0;
    uint32_t a01p = 0, a23p = 0;   // packed binary16 partials of the pending (even) chunk
    for (uint32_t f = 0; f < F; ++f) {
        issue(f + D - 1);
        cp_async_wait<D - 1>();
        __syncwarp();
        uint32_t d0, d1, d2, d3;
        ldsm_x4_trans(ring_saddr + (f % D) * kAsStageBytes + ld_off, d0, d1, d2, d3);
        __syncwarp();  // every lane has its registers before the stage is refilled
        mma_16816(acc, d0, d1, d2, d3, kOnesF16x2, kOnesF16x2);
        if (++r == R) {
            // thread (g, c): acc[0] = C_R[j = g], acc[2] = C_R[j = g + 8] -> binary16 (:179-181)
            const uint32_t pk = uint32_t(f32_to_h(acc[0])) | (uint32_t(f32_to_h(acc[2])) << 16);
            const uint32_t vA = __shfl_sync(kFull, pk, 8 * c);        // (h_2c,   h_2c+8)
            const uint32_t vB = __shfl_sync(kFull, pk, 8 * c + 4);    // (h_2c+1, h_2c+9)
            const uint32_t a01 = prmt(vA, vB, 0x5410), a23 = prmt(vA, vB, 0x7632);
            if (pend) {
                float fin[4] = {0.f, 0.f, 0.f, 0.f};
                // finishing MMA (reduction.hpp:182): rows 0-7 chunk ci-1, rows 8-15 chunk ci
                mma_16816(fin, a01p, a01, a23p, a23, kOnesF16x2, kOnesF16x2);
                ovf |= !isfinite(fin[0]) || !isfinite(fin[2]);
                if (lane == 0) {
                    s_chunk[warp + (ci - 1) * kAsWarps] = fin[0];
                    s_chunk[warp + ci * kAsWarps] = fin[2];
                }
                pend = 0;
            } else {
                a01p = a01;
                a23p = a23;
                pend = 1;
            }
            acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
            r = 0;
            ++ci;
        }
    }
    if (pend) {
        float fin[4] = {0.f, 0.f, 0.f, 0.f};
        mma_16816(fin, a01p, a01p, a23p, a23p, kOnesF16x2, kOnesF16x2);
        ovf |= !isfinite(fin[0]);
        if (lane == 0) s_chunk[warp + (ci - 1) * kAsWarps] = fin[0];
    }
    cp_async_wait<0>();
}


// Static fast path: a unit entirely inside n, RT in 1..5 with 2*RT | D, every warp's fragment
// count a multiple of D and its chunk count a multiple of 8.  Stage indices and chunk
// boundaries are compile-time.
//
// Column-sum form: with A = ones (16x16) and B = M split into its column halves, the two
// HMMA.16816 give every lane (g, c) C[2c], C[2c+1] and C[2c+8], C[2c+9] -- exactly the B
// fragment of column g of the finishing MMA.  The same k positions are summed as in the
// M^T x ones form of as_unit (bit-identical results), but no shuffles are needed: lane group g
// keeps chunk (8i + g)'s binary16 partials and ONE finishing HMMA (A = ones) per 8 chunks
// returns their 8 results (lane c: chunks 2c, 2c+1).
template <int RT, int D>
__device__ __forceinline__ void as_unit_static(const SpParams& p, uint64_t c0, uint32_t Cu, uint32_t ring_saddr,
                                               float* s_chunk, bool& ovf) {
    static_assert(D % (2 * RT) == 0, "static path needs 2*RT | depth");
    constexpr uint32_t CPI = D / RT;                 // chunks per outer iteration
    constexpr uint64_t CE = uint64_t(RT) * 256u;     // chunk elements
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t iters = Cu / kAsWarps / CPI;
    const uint16_t* gp = static_cast<const uint16_t*>(p.x) + (c0 + warp) * CE + 8u * lane;
    const uint32_t cp_dst = ring_saddr + swz(lane >> 1, lane & 1u);
    const uint32_t mi = lane >> 3;
    const uint32_t ld_base = ring_saddr + swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);
    // global element offset of warp-local fragment f (chunk f/RT, fragment f%RT)
#define TCR_FRAG_OFF(f) (uint64_t((f) / RT) * kAsWarps * CE + uint64_t((f) % RT) * 256u)
    constexpr uint64_t ITB = uint64_t(CPI) * kAsWarps * CE;     // elements per outer iteration
    uint64_t pol = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
    for (int u = 0; u < D - 1; ++u) {
        cp_async16_pol(cp_dst + u * kAsStageBytes, gp + TCR_FRAG_OFF(u), pol);
        cp_async_commit();
    }
    float* out = s_chunk + warp;
    uint32_t bb0 = 0, bb1 = 0;   // finishing-MMA B fragment: column g = chunk 8i + g
    for (uint32_t it = 0; it < iters; ++it) {
        const uint16_t* gq = gp + uint64_t(it) * ITB;
        float lo[4], hi[4];
#pragma unroll
        for (int u = 0; u < D; ++u) {
            // refill the stage consumed one step ago with fragment it*D + u + D-1
            if (it + 1 < iters || u == 0)
                cp_async16_pol(cp_dst + ((u + D - 1) % D) * kAsStageBytes, gq + TCR_FRAG_OFF(u + D - 1), pol);
            cp_async_commit();
            cp_async_wait<D - 1>();
            __syncwarp();
            uint32_t d0, d1, d2, d3;
            ldsm_x4_trans(ld_base + u * kAsStageBytes, d0, d1, d2, d3);
            if (u % RT == 0) lo[0] = lo[1] = lo[2] = lo[3] = hi[0] = hi[1] = hi[2] = hi[3] = 0.f;
            // C_r = ones x M_r + C_{r-1} (reduction.hpp:177): columns 0-7 and 8-15
            mma_16816(lo, kOnesF16x2, kOnesF16x2, kOnesF16x2, kOnesF16x2, d0, d2);
            mma_16816(hi, kOnesF16x2, kOnesF16x2, kOnesF16x2, kOnesF16x2, d1, d3);
            if (u % RT == RT - 1) {
                const uint32_t ci = it * CPI + u / RT;          // warp-local chunk
                const uint32_t k = ci & 7u;
                // C_R -> binary16 (:179-181), kept by the lanes of group g = k
                const uint32_t b0 = pack_h2(lo[0], lo[1]), b1 = pack_h2(hi[0], hi[1]);
                if (g == k) {
                    bb0 = b0;
                    bb1 = b1;
                }
                if (k == 7) {
                    // finishing MMA (:182) for chunks ci-7 .. ci
                    float fin[4] = {0.f, 0.f, 0.f, 0.f};
                    mma_16816(fin, kOnesF16x2, kOnesF16x2, kOnesF16x2, kOnesF16x2, bb0, bb1);
                    ovf |= !isfinite(fin[0]) || !isfinite(fin[1]);
                    if (g == 0) {
                        out[(ci - 7 + 2 * c) * kAsWarps] = fin[0];
                        out[(ci - 6 + 2 * c) * kAsWarps] = fin[1];
                    }
                }
            }
        }
    }
#undef TCR_FRAG_OFF
    cp_async_wait<0>();
}

// Ring depth per chain length: 2*R | D keeps every stage index and chunk pair compile-time.
template <int RT> struct AsDepth { static constexpr int value = 16; };
template <> struct AsDepth<1> { static constexpr int value = 16; };
template <> struct AsDepth<2> { static constexpr int value = 16; };
template <> struct AsDepth<3> { static constexpr int value = 24; };   // 12: -0..3 % (mode 11)
template <> struct AsDepth<4> { static constexpr int value = 16; };
template <> struct AsDepth<5> { static constexpr int value = 20; };   // 10: -3..5 % (mode 11)
template <> struct AsDepth<6> { static constexpr int value = 24; };
template <> struct AsDepth<7> { static constexpr int value = 14; };   // 28 would not fit 2 CTAs/SM
template <> struct AsDepth<8> { static constexpr int value = 16; };

int as_depth(uint32_t R) {
    switch (R) {
    case 1: return AsDepth<1>::value;
    case 2: return AsDepth<2>::value;
    case 3: return AsDepth<3>::value;
    case 4: return AsDepth<4>::value;
    case 5: return AsDepth<5>::value;
    case 6: return AsDepth<6>::value;
    case 7: return AsDepth<7>::value;
    case 8: return AsDepth<8>::value;
    default: return AsDepth<0>::value;
    }
}

__host__ __device__ inline bool static_unit(uint32_t Cu, uint32_t R, int D) {
    return R >= 1 && R <= 8 && Cu % (8 * kAsWarps) == 0 && (Cu / kAsWarps) * R >= uint32_t(D) &&
           ((Cu / kAsWarps) * R) % uint32_t(D) == 0;
}

template <int RT, int D = AsDepth<RT>::value>
constexpr uint32_t as_smem_bytes() {
    return uint32_t(kAsWarps) * D * kAsStageBytes;
}

// Persistent CTAs over work units u = group_begin*S .. group_end*S (strided by the grid, so
// concurrent CTAs read neighbouring units).  Per unit: stream -> chunk results -> block trees
// (reduction.hpp:253) -> group tree, either in place (S = 1) or by the CTA that completes the
// group (S > 1).
// Profiling (debug_mode 20, never set in production): %globaltimer stamps per CTA (start,
// streaming done) and of the last CTA's finalise, read back by tcr_debug_timestamps.
__device__ unsigned long long g_dbg_ts[4 * 1024 + 4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int RT, int D = AsDepth<RT>::value>
__global__ void __launch_bounds__(kAsThreads) sp_async_kernel(const SpParams p) {
    pdl_wait();      // launched early (programmatic serialization): the previous grid first
    pdl_release();
    extern __shared__ __align__(128) unsigned char s_ring[];
    __shared__ __align__(16) float s_chunk[kMaxChunksPerGroup];
    __shared__ __align__(16) float s_block[kMaxChunksPerGroup];
    __shared__ float s_scratch[32];
    __shared__ int s_last, s_glast;
    __shared__ unsigned long long s_next;
    const unsigned warp = threadIdx.x >> 5;
    const uint32_t ring = smem_u32(s_ring) + warp * D * kAsStageBytes;
    bool ovf = false;
    const uint32_t G = p.G, Cg = G * p.W;
    const bool stamp = p.debug_mode == 20 && threadIdx.x == 0 && blockIdx.x < 1024;
    if (stamp) g_dbg_ts[4 * blockIdx.x] = gtimer();
    // unit space: groups [group_begin, tail_group) in `split` pieces, then the tail groups
    // [tail_group, group_end) in `split_tail` smaller pieces
    const uint64_t u_main = (p.tail_group - p.group_begin) * p.split;
    const uint64_t u_total = u_main + (p.group_end - p.tail_group) * p.split_tail;
    const bool dyn = p.work_counter != nullptr;
    uint64_t u;
    if (dyn) {
        if (threadIdx.x == 0) s_next = atomicAdd(p.work_counter, 1ull);
        __syncthreads();
        u = s_next;
    } else {
        u = blockIdx.x;
    }
    while (u < u_total) {
        // thread 0 claims the next unit now; the atomic's latency hides behind this unit's stream
        unsigned long long nxt = u + gridDim.x;
        if (dyn && threadIdx.x == 0) nxt = atomicAdd(p.work_counter, 1ull);
        uint64_t gi;
        uint32_t S, piece;
        if (u < u_main) {
            S = p.split;
            gi = p.group_begin + u / S;
            piece = uint32_t(u % S);
        } else {
            S = p.split_tail;
            gi = p.tail_group + (u - u_main) / S;
            piece = uint32_t((u - u_main) % S);
        }
        const uint32_t Cu = Cg / S, Gu = G / S;
        const uint64_t c0 = gi * Cg + uint64_t(piece) * Cu;
        const uint64_t b0 = gi * G + uint64_t(piece) * Gu;
        bool done = false;
        if constexpr (RT > 0) {
            if (static_unit(Cu, RT, D) && (c0 + Cu) * p.chunk_elems <= p.n) {
                as_unit_static<RT, D>(p, c0, Cu, ring, s_chunk, ovf);
                done = true;
            }
        }
        if (!done) as_unit<RT, D>(p, c0, Cu, ring, s_chunk, ovf);
        __syncthreads();
        if (dyn && threadIdx.x == 0) {
            s_next = nxt;
            if (nxt == u_total + gridDim.x - 1) *p.work_counter = 0ull;   // the last claim: reset
        }
        range_trees_blocks(p, b0, Gu, s_chunk, s_block, warp, kAsWarps);
        __syncthreads();
        if (S == 1) {
            // large groups (B = 32: G = 1024) by the whole CTA, small ones by one warp (no barrier)
            if (G >= 256) tile_tree_group_cta(p, gi, s_block);
            else if (warp == 0) tile_tree_group(p, gi, s_block);
        } else {
            for (uint32_t b = threadIdx.x; b < Gu; b += kAsThreads) p.block_scratch[b0 + b] = s_block[b];
            __syncthreads();
            if (threadIdx.x == 0) {
                // one acquire-release RMW releases the CTA's block results (visible to thread 0
                // through the barrier) and, for the piece that completes the group, acquires
                // the other pieces' (the cooperative-groups grid-barrier pattern)
                unsigned t;
                asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(p.group_count + gi) : "memory");
                s_glast = t == S - 1;
            }
            __syncthreads();
            if (s_glast) {
                if (G >= 256) {
                    tile_tree_group_cta<true>(p, gi, p.block_scratch + gi * G);
                } else if (warp == 0) {
                    tile_tree_group<true>(p, gi, p.block_scratch + gi * G);
                }
                if (threadIdx.x == 0) p.group_count[gi] = 0u;
            }
        }
        __syncthreads();
        u = dyn ? s_next : nxt;
    }
    if (__any_sync(kFull, ovf) && lane_id() == 0) atomicOr(p.overflow, 1u);
    if (stamp) g_dbg_ts[4 * blockIdx.x + 1] = gtimer();
    __syncthreads();
    finalize_last_cta<true>(p, s_scratch, &s_last, kAsThreads, p.debug_mode == 20 ? g_dbg_ts + 4 * 1024 : nullptr);
    if (stamp) {
        g_dbg_ts[4 * blockIdx.x + 2] = gtimer();
        g_dbg_ts[4 * blockIdx.x + 3] = s_last;
    }
}

using AsKernel = void (*)(SpParams);

struct AsPick {
    AsKernel fn;
    uint32_t smem;
};

AsPick pick(uint32_t R, int mode = 0) {
    // profiling modes 9 / 10: ring depth 8 / 32 for R = 1 (default 16)
    if (R == 1 && mode == 9) return {sp_async_kernel<1, 8>, as_smem_bytes<1, 8>()};
    if (R == 1 && mode == 10) return {sp_async_kernel<1, 32>, as_smem_bytes<1, 32>()};
    // profiling mode 11: the shallower rings of the odd chain lengths
    if (R == 3 && mode == 11) return {sp_async_kernel<3, 12>, as_smem_bytes<3, 12>()};
    if (R == 5 && mode == 11) return {sp_async_kernel<5, 10>, as_smem_bytes<5, 10>()};
    switch (R) {
    case 1: return {sp_async_kernel<1>, as_smem_bytes<1>()};
    case 2: return {sp_async_kernel<2>, as_smem_bytes<2>()};
    case 3: return {sp_async_kernel<3>, as_smem_bytes<3>()};
    case 4: return {sp_async_kernel<4>, as_smem_bytes<4>()};
    case 5: return {sp_async_kernel<5>, as_smem_bytes<5>()};
    case 6: return {sp_async_kernel<6>, as_smem_bytes<6>()};
    case 7: return {sp_async_kernel<7>, as_smem_bytes<7>()};
    case 8: return {sp_async_kernel<8>, as_smem_bytes<8>()};
    default: return {sp_async_kernel<0>, as_smem_bytes<0>()};
    }
}

bool as_attr_once() {
    static PerDeviceOnce once;
    return once([] {
        for (int mode : {0, 9, 10, 11})
            for (uint32_t R = 0; R <= 8; ++R) {
                const AsPick k = pick(R, mode);
                cudaFuncAttributes fa{};
                cudaError_t e = cudaFuncGetAttributes(&fa, k.fn);
                if (e == cudaSuccess)
                    e = cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024 - int(fa.sharedSizeBytes));
                if (e != cudaSuccess) return e;
            }
        return cudaSuccess;
    }) == cudaSuccess;
}

// Work units per CTA below which the grid's tail (the last CTAs still streaming) starves HBM:
// measured at n = 2^28 (R = 3: 2.3 groups per CTA, 5.22 -> 5.66 TB/s with S = 2; R = 1: 3.5
// groups per CTA, S = 2 neutral) and n = 2^30 (>= 9 groups per CTA: splitting costs 1-3 %).
constexpr double kMinUnitsPerCta = 3.0;
// The last kTailUnitsPerCta x grid units are pieces of 1/kTailSplit group, handed out
// dynamically (first come, first served), so the grid finishes within a small piece.
constexpr uint32_t kTailSplit = 4;   // measured: 8 costs 1-4 % (small pieces drain), 2 gains less
constexpr uint32_t kTailUnitsPerCta = 2;
constexpr bool kDynamicSchedule = true;

}  // namespace

bool async_plan(const SpGeometry& g, SpParams* p, int grid) {
    const uint64_t groups = p->group_end - p->group_begin;
    p->split = p->split_tail = 1;
    p->tail_group = p->group_end;
    if (groups == 0 || grid < 1) return false;
    const uint32_t Cg = g.G * g.W;
    const int D = as_depth(g.R);
    const bool st1 = static_unit(Cg, g.R, D);
    auto ok = [&](uint32_t S) {   // S pieces of whole blocks that keep the static path
        return S <= g.G && S <= 64 && (!st1 || static_unit(Cg / S, g.R, D));
    };
    auto knob_pow2 = [&](uint32_t want, uint32_t dflt) {   // profiling override (knobs())
        if (!want) return dflt;
        uint32_t S = 1;
        while (S * 2 <= want && S * 2 <= g.G) S *= 2;
        return S;
    };
    const Knobs& k = knobs();
    uint32_t S = 1;
    while (double(groups) * S < kMinUnitsPerCta * grid && ok(S * 2)) S *= 2;
    S = knob_pow2(k.split, S);
    uint32_t St = S;
    while (St < kTailSplit && ok(St * 2)) St *= 2;
    St = std::max(S, knob_pow2(k.tail_split, St));
    p->split = S;
    p->split_tail = St;
    if (St > S) {
        const uint64_t tail = std::min<uint64_t>(groups, (uint64_t(kTailUnitsPerCta) * grid + St - 1) / St);
        p->tail_group = p->group_end - tail;
        if (p->tail_group == p->group_begin) p->split = St;
    }
    return k.sched >= 0 ? k.sched != 0 : kDynamicSchedule;
}

namespace {

// CTAs per SM: two 64 KiB rings per SM measured best (n = 2^30, R = 1: 2/SM 312.8 us, 3/SM
// 332.5 us, 1/SM 540 us); the launch pads dynamic shared memory so that no SM takes a third
// CTA.  Knob ctas_per_sm overrides (profiling).
int as_ctas_per_sm() {
    return knobs().ctas_per_sm > 0 ? knobs().ctas_per_sm : 2;
}

uint32_t as_launch_smem_uncached(const AsPick& k, int cps) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k.fn);
    int dev = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    // the largest footprint that still lets cps CTAs (each with 1 KiB reserved) share the SM
    const long fit = long(per_sm) / cps - 1024 - long(fa.sharedSizeBytes);
    const long cap = 227 * 1024 - long(fa.sharedSizeBytes);
    long want = std::min(fit, cap);
    want -= want % 128;
    return uint32_t(std::max<long>(long(k.smem), want));
}

// (kernel, CTAs per SM) -> launch smem and resident CTAs per SM, queried once (the runtime
// queries cost microseconds of host time per call otherwise)
struct AsLaunch {
    AsKernel fn;
    int dev;
    int cps;
    uint32_t smem;
    int per_sm;
};

AsLaunch as_launch(const AsPick& k, int cps) {
    static std::mutex mu;
    static std::vector<AsLaunch> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    for (const AsLaunch& a : cache)
        if (a.fn == k.fn && a.dev == dev && a.cps == cps) return a;
    AsLaunch a{k.fn, dev, cps, as_launch_smem_uncached(k, cps), 0};
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a.per_sm, k.fn, kAsThreads, a.smem);
    if (a.per_sm < 1) a.per_sm = 1;
    cache.push_back(a);
    return a;
}

}  // namespace

int debug_timestamps(unsigned long long* host, size_t count) {
    if (count > 4 * 1024 + 4) count = 4 * 1024 + 4;
    return cudaMemcpyFromSymbol(host, g_dbg_ts, count * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
}

int async_max_grid(uint32_t R, int mode) {
    as_attr_once();
    const int cps = as_ctas_per_sm();
    const AsLaunch a = as_launch(pick(R, mode), cps);
    return std::min(a.per_sm, cps) * sm_count();
}

cudaError_t launch_async(const SpParams& p, int grid, cudaStream_t s) {
    if (!as_attr_once()) return cudaErrorInvalidValue;
    const AsPick k = pick(p.R, p.debug_mode);
    // programmatic dependent launch: back-to-back reductions on a stream overlap this grid's launch
    // with the previous grid's tail (the kernel waits for it before its first global access)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kAsThreads);
    cfg.dynamicSmemBytes = as_launch(k, as_ctas_per_sm()).smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k.fn, p);
}

}  // namespace tcr
