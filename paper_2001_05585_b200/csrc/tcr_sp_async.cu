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

template <int RT, int D>
__device__ __forceinline__ void as_group(const SpParams& p, uint64_t gi, uint32_t ring_saddr, float* s_chunk,
                                         bool& ovf) {
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned c = lane & 3u;
    const uint32_t R = RT > 0 ? uint32_t(RT) : p.R;
    const uint32_t Cg = p.G * p.W;
    const uint32_t nch = Cg > warp ? (Cg - warp + kAsWarps - 1) / kAsWarps : 0;
    const uint32_t F = nch * R;
    const uint64_t ce = uint64_t(R) * 256u;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    const uint64_t n = p.n;
    // copy side: lane copies bytes [16*lane, 16*lane+16) of the fragment = line (k = lane/2, half = lane&1)
    const uint32_t cp_dst = swz(lane >> 1, lane & 1u);
    // ldmatrix side: matrix mi = lane>>3 supplies line (k = (lane&7) + 8*(mi>>1), half = mi&1)
    const uint32_t mi = lane >> 3;
    const uint32_t ld_off = swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);

    // element index of fragment f's first element for this warp
    auto frag_elem = [&](uint32_t f) -> uint64_t {
        const uint32_t ci = f / R, r = f - ci * R;
        return (gi * uint64_t(Cg) + warp + uint64_t(ci) * kAsWarps) * ce + uint64_t(r) * 256u;
    };
    auto issue = [&](uint32_t f) {
        if (f < F) {
            const uint64_t e = frag_elem(f) + 8u * lane;
            const uint32_t bytes = e + 8 <= n ? 16u : (e < n ? uint32_t(n - e) * 2u : 0u);
            cp_async16(ring_saddr + (f % D) * kAsStageBytes + cp_dst, x + (e < n ? e : 0), bytes);
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


// Static fast path: full group, RT in {1, 2, 4} (RT | D), and every warp's fragment count a
// multiple of D.  Stage indices, chunk boundaries and finishing pairs are compile-time.
// The stream never drains between two static groups of the same CTA: the last D-1 refills of a
// group fetch the first D-1 fragments of the next one (same stages, same commit-group count),
// so memory stays busy through the block/group trees and the CTA barrier.
template <int RT, int D>
__device__ __forceinline__ void as_group_static(const SpParams& p, uint64_t gi, uint32_t ring_saddr, float* s_chunk,
                                                bool& ovf, bool prologue, bool prefetch_next, uint64_t gnext) {
    static_assert(D % (2 * RT) == 0, "static path needs 2*RT | depth");
    constexpr uint32_t CPI = D / RT;                 // chunks per outer iteration
    constexpr uint64_t CE = uint64_t(RT) * 256u;            // chunk elements
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned c = lane & 3u;
    const uint32_t Cg = p.G * p.W;
    const uint32_t nch = Cg / kAsWarps;
    const uint32_t iters = nch / CPI;
    const uint16_t* gp = static_cast<const uint16_t*>(p.x) + (gi * uint64_t(Cg) + warp) * CE + 8u * lane;
    const uint32_t cp_dst = ring_saddr + swz(lane >> 1, lane & 1u);
    const uint32_t mi = lane >> 3;
    const uint32_t ld_base = ring_saddr + swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);
    // global element offset of warp-local fragment g (chunk g/RT, fragment g%RT)
#define TCR_FRAG_OFF(g) (uint64_t((g) / RT) * kAsWarps * CE + uint64_t((g) % RT) * 256u)
    // iteration rotation: CTAs start their sweep of the group at different offsets so that
    // concurrent CTAs do not hit the same DRAM channel phase (profiling mode 14)
    const uint32_t rot = p.debug_mode == 14 ? uint32_t(blockIdx.x % iters) : 0u;
    const uint64_t ITB = uint64_t(CPI) * kAsWarps * CE;     // elements per outer iteration
    if (prologue) {
        const uint16_t* g0 = gp + uint64_t(rot) * ITB;
#pragma unroll
        for (int u = 0; u < D - 1; ++u) {
            cp_async16(cp_dst + u * kAsStageBytes, g0 + TCR_FRAG_OFF(u), 16u);
            cp_async_commit();
        }
    }
    const uint16_t* gn = static_cast<const uint16_t*>(p.x) + (gnext * uint64_t(Cg) + warp) * CE + 8u * lane;
    float* out = s_chunk + warp;
    uint32_t ip = rot;                                         // physical iteration
    for (uint32_t it = 0; it < iters; ++it) {
        const uint32_t ipn = ip + 1 == iters ? 0u : ip + 1;
        const uint16_t* gq = gp + uint64_t(ip) * ITB;
        const uint16_t* gqn = gp + uint64_t(ipn) * ITB;
        uint32_t a01p = 0, a23p = 0;
        float acc[4];
#pragma unroll
        for (int u = 0; u < D; ++u) {
            // refill the stage consumed one step ago with fragment it*D + u + D-1
            if (it + 1 < iters || u == 0)
                cp_async16(cp_dst + ((u + D - 1) % D) * kAsStageBytes,
                           u == 0 ? gq + TCR_FRAG_OFF(D - 1) : gqn + TCR_FRAG_OFF(u - 1), 16u);
            else if (prefetch_next)   // stage u-1 <- fragment u-1 of the next group
                cp_async16(cp_dst + ((u + D - 1) % D) * kAsStageBytes, gn + TCR_FRAG_OFF(u - 1), 16u);
            cp_async_commit();
            cp_async_wait<D - 1>();
            __syncwarp();
            uint32_t d0, d1, d2, d3;
            ldsm_x4_trans(ld_base + u * kAsStageBytes, d0, d1, d2, d3);
            if (u % RT == 0) acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
            mma_16816(acc, d0, d1, d2, d3, kOnesF16x2, kOnesF16x2);
            if (u % RT == RT - 1) {
                const uint32_t pk = uint32_t(f32_to_h(acc[0])) | (uint32_t(f32_to_h(acc[2])) << 16);
                const uint32_t vA = __shfl_sync(kFull, pk, 8 * c);
                const uint32_t vB = __shfl_sync(kFull, pk, 8 * c + 4);
                const uint32_t a01 = prmt(vA, vB, 0x5410), a23 = prmt(vA, vB, 0x7632);
                if ((u / RT) % 2 == 0) {
                    a01p = a01;
                    a23p = a23;
                } else {
                    float fin[4] = {0.f, 0.f, 0.f, 0.f};
                    mma_16816(fin, a01p, a01, a23p, a23, kOnesF16x2, kOnesF16x2);
                    ovf |= !isfinite(fin[0]) || !isfinite(fin[2]);
                    if (lane == 0) {
                        const uint32_t ci = ip * CPI + u / RT;     // odd chunk of the pair
                        out[(ci - 1) * kAsWarps] = fin[0];
                        out[ci * kAsWarps] = fin[2];
                    }
                }
            }
        }
        ip = ipn;
    }
#undef TCR_FRAG_OFF
    if (!prefetch_next) cp_async_wait<0>();
}


constexpr int kAsBufs = 4;   // per-group block tables in flight (warp-blocks mode)
constexpr int kWbMaxBlocks = 256;

// Warp-blocks mode: warp w owns the contiguous chunks [w*Cpw, (w+1)*Cpw) of the group, where
// Cpw = Cg/8 is a whole number of logical blocks, so the reference's block tree (:253) runs in
// registers (shfl_down over pow2(W)-lane segments) and no CTA barrier is needed: the warp that
// completes a group last (shared counter) runs the group tree.  Fragments stream contiguously.
template <int RT, int D>
__device__ __forceinline__ void as_group_warpblocks(const SpParams& p, uint64_t gi, uint32_t k_iter, uint32_t ring_saddr,
                                                    float* s_blocks, uint32_t* s_done, volatile uint32_t* s_gen,
                                                    bool& ovf) {
    static_assert(D % (2 * RT) == 0, "static path needs 2*RT | depth");
    constexpr uint32_t CPI = D / RT;
    constexpr uint64_t CE = uint64_t(RT) * 256u;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned c = lane & 3u;
    const uint32_t W = p.W, G = p.G;
    const uint32_t Cg = G * W;
    const uint32_t Cpw = Cg / kAsWarps;
    const uint32_t iters = Cpw / CPI;
    uint32_t P = 1;
    while (P < W) P <<= 1;
    const uint32_t bpb = 32u / P;                 // blocks per 32-lane batch
    const uint32_t b0 = warp * (Cpw / W);         // first group-local block of this warp
    const uint32_t buf = k_iter % kAsBufs;
    float* blocks = s_blocks + buf * kWbMaxBlocks;
    // the buffer must have been released by the tree of iteration k_iter - kAsBufs
    if (lane == 0)
        while (s_gen[buf] != k_iter - kAsBufs) { }
    __syncwarp();
    const uint16_t* gp = static_cast<const uint16_t*>(p.x) + (gi * uint64_t(Cg) + uint64_t(warp) * Cpw) * CE + 8u * lane;
    const uint32_t cp_dst = ring_saddr + swz(lane >> 1, lane & 1u);
    const uint32_t mi = lane >> 3;
    const uint32_t ld_base = ring_saddr + swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);
#pragma unroll
    for (int u = 0; u < D - 1; ++u) {
        cp_async16(cp_dst + u * kAsStageBytes, gp + uint64_t(u) * 256u, 16u);
        cp_async_commit();
    }
    float held = 0.0f;
    for (uint32_t it = 0; it < iters; ++it) {
        const uint16_t* gq = gp + uint64_t(it) * D * 256u;
        uint32_t a01p = 0, a23p = 0;
        float acc[4];
#pragma unroll
        for (int u = 0; u < D; ++u) {
            if (it + 1 < iters || u == 0)
                cp_async16(cp_dst + ((u + D - 1) % D) * kAsStageBytes, gq + uint64_t(u + D - 1) * 256u, 16u);
            cp_async_commit();
            cp_async_wait<D - 1>();
            __syncwarp();
            uint32_t d0, d1, d2, d3;
            ldsm_x4_trans(ld_base + u * kAsStageBytes, d0, d1, d2, d3);
            if (u % RT == 0) acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
            mma_16816(acc, d0, d1, d2, d3, kOnesF16x2, kOnesF16x2);
            if (u % RT == RT - 1) {
                const uint32_t pk = uint32_t(f32_to_h(acc[0])) | (uint32_t(f32_to_h(acc[2])) << 16);
                const uint32_t vA = __shfl_sync(kFull, pk, 8 * c);
                const uint32_t vB = __shfl_sync(kFull, pk, 8 * c + 4);
                const uint32_t a01 = prmt(vA, vB, 0x5410), a23 = prmt(vA, vB, 0x7632);
                if ((u / RT) % 2 == 0) {
                    a01p = a01;
                    a23p = a23;
                } else {
                    float fin[4] = {0.f, 0.f, 0.f, 0.f};
                    mma_16816(fin, a01p, a01, a23p, a23, kOnesF16x2, kOnesF16x2);
                    ovf |= !isfinite(fin[0]) || !isfinite(fin[2]);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t ci = it * CPI + u / RT - 1 + h;      // warp-local chunk
                        const uint32_t bl = ci / W, j = ci - bl * W;
                        if (lane == (bl % bpb) * P + j) held = h ? fin[2] : fin[0];
                        if (j == W - 1 && (bl % bpb == bpb - 1 || ci == Cpw - 1)) {
                            // flush: pairwise trees over the P-lane segments (reduction.hpp:90-101)
                            float v = held;
                            for (uint32_t off = P >> 1; off >= 1; off >>= 1) v += __shfl_down_sync(kFull, v, off);
                            const uint32_t seg = lane / P;
                            const uint32_t blk = bl - (bl % bpb) + seg;
                            if (lane % P == 0 && seg <= bl % bpb) {
                                blocks[b0 + blk] = v;
                                const uint64_t gb = gi * G + b0 + blk;
                                if (gb < p.n_blocks) {
                                    if (p.block_partials) p.block_partials[gb] = v;
                                    if (p.finalize == kFinAtomic) atomicAdd(p.result, v);
                                }
                            }
                            held = 0.0f;
                        }
                    }
                }
            }
        }
    }
    cp_async_wait<0>();
    // group stage: the last warp to finish runs the adjacent tree over the G block results
    __syncwarp();
    uint32_t last = 0;
    if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&s_done[buf], 1u) == kAsWarps - 1;
    }
    last = __shfl_sync(kFull, last, 0);
    if (last) {
        __threadfence_block();
        tile_tree_group(p, gi, blocks);
        __syncwarp();
        if (lane == 0) {
            s_done[buf] = 0;
            __threadfence_block();
            s_gen[buf] = k_iter;
        }
    }
}


// ===================================================================== interleaved stream engine
// Two launches.  (1) sp_stream_kernel: every warp of the GPU takes global chunks gw, gw + TW,
// gw + 2 TW, ... (TW = all warps of the grid), so at each step the whole GPU reads one
// contiguous window of TW fragments -- the same DRAM-friendly sweep as a grid-stride read --
// and writes one fp32 chunk result per chunk.  (2) sp_tree_kernel: per group, the reference's
// block trees and the group tree over those chunk results, then the last-CTA finaliser.
// The extra traffic is 8 bytes per chunk (1.6 % at R = 1).
template <int RT, int D>
__global__ void __launch_bounds__(kAsThreads) sp_stream_kernel(const SpParams p, float* chunk_res, uint64_t n_chunks) {
    extern __shared__ __align__(128) unsigned char s_ring[];
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned c = lane & 3u;
    const uint64_t TW = uint64_t(gridDim.x) * kAsWarps;
    const uint64_t gw = uint64_t(blockIdx.x) * kAsWarps + warp;
    const uint32_t ring = smem_u32(s_ring) + warp * D * kAsStageBytes;
    constexpr uint64_t CE = uint64_t(RT) * 256u;
    const uint64_t my_chunks = gw < n_chunks ? (n_chunks - gw + TW - 1) / TW : 0;
    const uint64_t F = my_chunks * RT;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    const uint64_t n = p.n;
    const uint32_t cp_dst = swz(lane >> 1, lane & 1u);
    const uint32_t mi = lane >> 3;
    const uint32_t ld_off = swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);
    bool ovf = false;
    auto issue = [&](uint64_t f) {
        if (f < F) {
            const uint64_t k = f / RT, r = f - k * RT;
            const uint64_t e = (gw + k * TW) * CE + r * 256u + 8u * lane;
            const uint32_t bytes = e + 8 <= n ? 16u : (e < n ? uint32_t(n - e) * 2u : 0u);
            cp_async16(ring + uint32_t(f % D) * kAsStageBytes + cp_dst, x + (e < n ? e : 0), bytes);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int f = 0; f < D - 1; ++f) issue(uint64_t(f));
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t r = 0, pend = 0;
    uint64_t ci = 0;
    uint32_t a01p = 0, a23p = 0;
    for (uint64_t f = 0; f < F; ++f) {
        issue(f + D - 1);
        cp_async_wait<D - 1>();
        __syncwarp();
        uint32_t d0, d1, d2, d3;
        ldsm_x4_trans(ring + uint32_t(f % D) * kAsStageBytes + ld_off, d0, d1, d2, d3);
        mma_16816(acc, d0, d1, d2, d3, kOnesF16x2, kOnesF16x2);
        if (++r == RT) {
            const uint32_t pk = uint32_t(f32_to_h(acc[0])) | (uint32_t(f32_to_h(acc[2])) << 16);
            const uint32_t vA = __shfl_sync(kFull, pk, 8 * c);
            const uint32_t vB = __shfl_sync(kFull, pk, 8 * c + 4);
            const uint32_t a01 = prmt(vA, vB, 0x5410), a23 = prmt(vA, vB, 0x7632);
            if (pend) {
                float fin[4] = {0.f, 0.f, 0.f, 0.f};
                mma_16816(fin, a01p, a01, a23p, a23, kOnesF16x2, kOnesF16x2);
                ovf |= !isfinite(fin[0]) || !isfinite(fin[2]);
                if (lane == 0) {
                    chunk_res[gw + (ci - 1) * TW] = fin[0];
                    chunk_res[gw + ci * TW] = fin[2];
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
        if (lane == 0) chunk_res[gw + (ci - 1) * TW] = fin[0];
    }
    cp_async_wait<0>();
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
}

__global__ void __launch_bounds__(kAsThreads) sp_tree_kernel(const SpParams p, const float* chunk_res) {
    __shared__ float s_chunk[kMaxChunksPerGroup];
    __shared__ float s_block[kMaxChunksPerGroup];
    __shared__ float s_scratch[32];
    __shared__ int s_last;
    const unsigned warp = threadIdx.x >> 5;
    const uint32_t Cg = p.G * p.W;
    for (uint64_t gi = p.group_begin + blockIdx.x; gi < p.group_end; gi += gridDim.x) {
        for (uint32_t i = threadIdx.x; i < Cg; i += blockDim.x) s_chunk[i] = __ldcg(chunk_res + gi * Cg + i);
        __syncthreads();
        tile_trees_blocks(p, gi, s_chunk, s_block, warp, kAsWarps);
        __syncthreads();
        if (warp == 0) tile_tree_group(p, gi, s_block);
        __syncthreads();
    }
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kAsThreads);
}

// Ring depth per chain length: 2*R | D keeps every stage index and chunk pair compile-time.
template <int RT> struct AsDepth { static constexpr int value = 8; };
template <> struct AsDepth<1> { static constexpr int value = 16; };
template <> struct AsDepth<2> { static constexpr int value = 16; };
template <> struct AsDepth<3> { static constexpr int value = 12; };
template <> struct AsDepth<4> { static constexpr int value = 16; };
template <> struct AsDepth<5> { static constexpr int value = 10; };

template <int RT, int D = AsDepth<RT>::value>
constexpr uint32_t as_smem_bytes() {
    return uint32_t(kAsWarps) * D * kAsStageBytes;
}

template <int RT, int D = AsDepth<RT>::value>
__global__ void __launch_bounds__(kAsThreads) sp_async_kernel(const SpParams p) {
    extern __shared__ __align__(128) unsigned char s_ring[];
    __shared__ float s_chunk[kMaxChunksPerGroup];
    __shared__ float s_block[kMaxChunksPerGroup];
    __shared__ float s_wblocks[kAsBufs * kWbMaxBlocks];
    __shared__ uint32_t s_done[kAsBufs];
    __shared__ uint32_t s_gen[kAsBufs];
    __shared__ float s_scratch[32];
    __shared__ int s_last;
    const unsigned warp = threadIdx.x >> 5;
    const uint32_t ring = smem_u32(s_ring) + warp * D * kAsStageBytes;
    bool ovf = false;
    const uint64_t full_groups = p.n / (uint64_t(p.G) * p.W * p.chunk_elems);
    const uint32_t Cg = p.G * p.W;
    bool static_ok = false, warp_blocks = false;
    if constexpr (RT > 0) {
        static_ok = (Cg % kAsWarps == 0) && ((Cg / kAsWarps) * RT) % D == 0;
        warp_blocks = static_ok && ((Cg / kAsWarps) % p.W == 0) && p.G <= uint32_t(kWbMaxBlocks) && p.debug_mode == 12;
    }
    if (threadIdx.x < kAsBufs) {
        s_done[threadIdx.x] = 0;
        s_gen[threadIdx.x] = uint32_t(threadIdx.x) - kAsBufs;   // "iteration buf - kAsBufs completed"
    }
    __syncthreads();
    bool prefetched = false;   // this group's first D-1 fragments are already in flight
    uint32_t k_iter = 0;
    // group order: strided over CTAs (default) or, in profiling mode 15, one contiguous range of
    // groups per CTA with the stream prefetching across group boundaries
    const bool contiguous = p.debug_mode == 15;
    const uint64_t ngr = p.group_end - p.group_begin;
    const uint64_t per = (ngr + gridDim.x - 1) / gridDim.x;
    const uint64_t g_first = contiguous ? p.group_begin + blockIdx.x * per : p.group_begin + blockIdx.x;
    const uint64_t g_last = contiguous ? (p.group_begin + (blockIdx.x + 1) * per < p.group_end
                                              ? p.group_begin + (blockIdx.x + 1) * per : p.group_end)
                                       : p.group_end;
    const uint64_t g_step = contiguous ? 1 : gridDim.x;
    for (uint64_t gi = g_first; gi < g_last; gi += g_step, ++k_iter) {
        if constexpr (RT > 0) {
            if (warp_blocks && gi < full_groups) {
                as_group_warpblocks<RT, D>(p, gi, k_iter, ring, s_wblocks, s_done, s_gen, ovf);
                continue;
            }
        }
        if constexpr (RT > 0) {
            if (static_ok && gi < full_groups) {
                const uint64_t gn = gi + g_step;
                const bool next_static = gn < g_last && gn < full_groups && (p.debug_mode == 8 || contiguous);
                as_group_static<RT, D>(p, gi, ring, s_chunk, ovf, !prefetched, next_static, gn);
                prefetched = next_static;
            } else {
                as_group<RT, D>(p, gi, ring, s_chunk, ovf);
                prefetched = false;
            }
        } else {
            as_group<RT, D>(p, gi, ring, s_chunk, ovf);
        }
        __syncthreads();
        tile_trees_blocks(p, gi, s_chunk, s_block, warp, kAsWarps);
        __syncthreads();
        if (warp == 0) tile_tree_group(p, gi, s_block);
        __syncthreads();
    }
    if (__any_sync(kFull, ovf) && lane_id() == 0) atomicOr(p.overflow, 1u);
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kAsThreads);
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
    switch (R) {
    case 1: return {sp_async_kernel<1>, as_smem_bytes<1>()};
    case 2: return {sp_async_kernel<2>, as_smem_bytes<2>()};
    case 3: return {sp_async_kernel<3>, as_smem_bytes<3>()};
    case 4: return {sp_async_kernel<4>, as_smem_bytes<4>()};
    case 5: return {sp_async_kernel<5>, as_smem_bytes<5>()};
    default: return {sp_async_kernel<0>, as_smem_bytes<0>()};
    }
}

bool as_attr_once() {
    static bool done = false;
    if (!done) {
        for (int mode : {0, 9, 10})
        for (uint32_t R = 0; R <= 5; ++R) {
            const AsPick k = pick(R, mode);
            if (cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(k.smem)) != cudaSuccess)
                return false;
        }
        done = true;
    }
    return true;
}

using StreamKernel = void (*)(SpParams, float*, uint64_t);

StreamKernel pick_stream(uint32_t R) {
    switch (R) {
    case 1: return sp_stream_kernel<1, AsDepth<1>::value>;
    case 2: return sp_stream_kernel<2, AsDepth<2>::value>;
    case 3: return sp_stream_kernel<3, AsDepth<3>::value>;
    case 4: return sp_stream_kernel<4, AsDepth<4>::value>;
    case 5: return sp_stream_kernel<5, AsDepth<5>::value>;
    default: return nullptr;
    }
}

uint32_t stream_smem(uint32_t R) {
    switch (R) {
    case 1: return as_smem_bytes<1>();
    case 2: return as_smem_bytes<2>();
    case 3: return as_smem_bytes<3>();
    case 4: return as_smem_bytes<4>();
    default: return as_smem_bytes<5>();
    }
}

}  // namespace

bool stream_supported(uint32_t R) { return pick_stream(R) != nullptr; }

cudaError_t launch_stream(const SpParams& p, float* chunk_res, uint64_t n_chunks, cudaStream_t s) {
    StreamKernel fn = pick_stream(p.R);
    if (!fn) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        for (uint32_t R = 1; R <= 5; ++R) {
            const cudaError_t e =
                cudaFuncSetAttribute(pick_stream(R), cudaFuncAttributeMaxDynamicSharedMemorySize, int(stream_smem(R)));
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kAsThreads, stream_smem(p.R));
    if (per_sm < 1) per_sm = 1;
    const uint64_t want = (n_chunks + kAsWarps - 1) / kAsWarps;
    const int grid = int(std::min<uint64_t>(want, uint64_t(per_sm) * sm_count()));
    fn<<<grid, kAsThreads, stream_smem(p.R), s>>>(p, chunk_res, n_chunks);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    int per_sm_t = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_t, sp_tree_kernel, kAsThreads, 0);
    const uint64_t groups = p.group_end - p.group_begin;
    const int grid_t = int(std::min<uint64_t>(groups, uint64_t(per_sm_t < 1 ? 1 : per_sm_t) * sm_count()));
    sp_tree_kernel<<<grid_t, kAsThreads, 0, s>>>(p, chunk_res);
    return cudaGetLastError();
}

int async_max_grid(uint32_t R, int mode) {
    as_attr_once();
    const AsPick k = pick(R, mode);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.fn, kAsThreads, k.smem);
    if (per_sm < 1) per_sm = 1;
    return per_sm * sm_count();
}

cudaError_t launch_async(const SpParams& p, int grid, cudaStream_t s) {
    if (!as_attr_once()) return cudaErrorInvalidValue;
    const AsPick k = pick(p.R, p.debug_mode);
    k.fn<<<grid, kAsThreads, k.smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace tcr
