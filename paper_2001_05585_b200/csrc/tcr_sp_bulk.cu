// tcr_sp_bulk.cu -- single-pass chained reduction, m = 16: the TMA-fed mma.sync engine.
//
// Same element partition, block stage and group stage as the other engines (reference
// reduction.hpp:164-184, :238-275).  Warp-specialised persistent CTA, 8 streaming warps + 1
// manager warp:
//
//   streaming warp w   owns a ring of NS 2 KiB stages (4 fragments) and its own full-mbarriers;
//                      lane 0 refills the stage it has just consumed with ONE cp.async.bulk
//                      (1-D TMA, L2 evict-first) of the next 2 KiB of the warp's stream, so NS
//                      stages are always in flight with no per-lane copy instructions.  The
//                      warp's stream is its contiguous share (1/8) of every work unit, unit
//                      after unit: the issue cursor runs into the NEXT unit before the current
//                      one is consumed, so a unit boundary never drains the pipeline.
//                      Per fragment: ldmatrix.x4.trans + two HMMA.16816 in the column-sum form
//                      (A = ones, B = the fragment's column halves: C_r = ones x M_r + C_{r-1},
//                      reduction.hpp:177); C_R -> binary16 (:179-181) stays in the lanes of
//                      group g = chunk mod 8, one finishing HMMA per 8 chunks (:182).
//   manager warp       claims work units QD ahead (atomic counter) into a shared queue, and per
//                      unit -- off the streaming warps' critical path, double-buffered chunk
//                      tables -- runs the block trees (:253), the group tree or, for a piece of
//                      a group, publishes its block results and takes the group ticket (the
//                      piece that completes the group runs the group tree).
//
// Units: whole groups, then the last ~2 x grid units as pieces of a few blocks, so every CTA
// finishes within one small piece of the others.  Full groups only (the ragged tail group, if
// any, runs on the register engine in a second launch that finalises).
#include <algorithm>
#include <cuda_runtime.h>

#include "tcr_device.cuh"
#include "tcr_kernels.h"
#include "tcr_pipeline.cuh"

namespace tcr {

namespace {

using namespace pipe;

constexpr int kBkWarps = 8;                        // streaming warps
constexpr int kBkThreads = 32 * (kBkWarps + 1);    // + the manager warp
constexpr int kBkQ = 8;                            // unit queue slots
constexpr int kBkQD = 6;                           // units claimed ahead
constexpr uint32_t kBkTailPieceBytes = 64 * 1024;  // target size of the tail pieces
constexpr uint32_t kBkTailUnitsPerCta = 2;

__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& d0, uint32_t& d1, uint32_t& d2, uint32_t& d3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3)
                 : "r"(addr));
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__host__ __device__ constexpr uint32_t bk_gcd(uint32_t a, uint32_t b) { return b ? bk_gcd(b, a % b) : a; }
__host__ __device__ constexpr uint32_t bk_lcm(uint32_t a, uint32_t b) { return a / bk_gcd(a, b) * b; }

struct BkShared {
    uint64_t full[kBkWarps][8];        // per-warp stage barriers (NS <= 8)
    uint64_t qfull[kBkQ];              // unit queue slot written
    uint64_t done[2];                  // chunk table b complete (8 streaming warps)
    uint64_t freed[2];                 // chunk table b consumed by the manager
    unsigned long long q[kBkQ];        // unit queue
    float chunk[2][kMaxChunksPerGroup];
    float block[kMaxChunksPerGroup];
    float scratch[32];
    int last;
};

// unit u -> (group, pieces of that group, piece)
struct Unit {
    uint64_t gi;
    uint32_t S, piece;
};
__device__ __forceinline__ Unit unit_of(const SpParams& p, uint64_t u) {
    const uint64_t u_main = (p.tail_group - p.group_begin) * p.split;
    Unit r;
    if (u < u_main) {
        r.S = p.split;
        r.gi = p.group_begin + u / r.S;
        r.piece = uint32_t(u % r.S);
    } else {
        r.S = p.split_tail;
        r.gi = p.tail_group + (u - u_main) / r.S;
        r.piece = uint32_t((u - u_main) % r.S);
    }
    return r;
}

template <int RT, int NS, uint32_t kBkStage, bool IL, int XM = 0>
__global__ void __launch_bounds__(kBkThreads) sp_bulk_kernel(const SpParams p) {
    extern __shared__ __align__(1024) unsigned char s_ring_raw[];
    __shared__ BkShared sh;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const uint32_t G = p.G, Cg = G * p.W;
    const uint64_t u_total = (p.tail_group - p.group_begin) * p.split + (p.group_end - p.tail_group) * p.split_tail;
    const unsigned long long last_claim = u_total + uint64_t(kBkQD) * gridDim.x - 1;

    if (threadIdx.x == 0) {
        for (int w = 0; w < kBkWarps; ++w)
            for (int s = 0; s < NS; ++s) mbar_init(&sh.full[w][s], 1);
        for (int i = 0; i < kBkQ; ++i) mbar_init(&sh.qfull[i], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sh.done[b], kBkWarps);
            mbar_init(&sh.freed[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    bool ovf = false;

    if (warp < kBkWarps) {
        // ------------------------------------------------------------------ streaming warp
        const uint32_t ring = smem_u32(s_ring_raw) + warp * NS * kBkStage;
        const char* x = static_cast<const char*>(p.x);
        const uint64_t policy = evict_first_policy();
        // issue cursor (warp-uniform): queue index, next fragment of the warp's share, fragments
        // in the share, the share's first chunk
        uint32_t ik = 0, ifr = 0, infr = 0;
        uint64_t ic0 = 0;
        bool idone = false;
        uint32_t t_issue = 0;
        constexpr uint32_t GR = bk_lcm(kBkStage / 512u, uint32_t(RT));   // granule: lcm(stage, chunk) fragments
        constexpr uint32_t GC = GR / RT;                                   // chunks per granule
        auto open_issue_unit = [&]() {   // the share of unit ik (waits for the claim)
            mbar_wait(&sh.qfull[ik % kBkQ], (ik / kBkQ) & 1u);
            const unsigned long long u = sh.q[ik % kBkQ];
            if (u >= u_total) {
                idone = true;
                return;
            }
            const Unit un = unit_of(p, u);
            const uint32_t Cu = Cg / un.S, nc = Cu / kBkWarps;
            ic0 = un.gi * Cg + uint64_t(un.piece) * Cu + (IL ? 0 : uint64_t(warp) * nc);
            infr = nc * uint32_t(RT);
            ifr = 0;
        };
        auto issue = [&]() {   // every lane: the next stage of the stream into slot t_issue % NS
            if (idone) return;
            if (ifr == infr) {
                ++ik;
                open_issue_unit();
                if (idone) return;
            }
            constexpr uint32_t FPS = kBkStage / 512u;
            const uint32_t nf = min(FPS, infr - ifr);
            const uint32_t slot = t_issue % NS;
            const uint32_t bar = smem_u32(&sh.full[warp][slot]);
            if (lane == 0) mbar_expect_tx(&sh.full[warp][slot], nf * 512u);
            // IL: the share is granules w, w + 8, w + 16, ... of GR = lcm(stage, R) fragments (whole
            // chunks, whole stages) of the unit, so the CTA reads one compact region at a time
            // with one copy per stage; else the contiguous w-th eighth of the unit
            const uint64_t gfrag = IL ? ic0 * uint64_t(RT) + (uint64_t(warp) + uint64_t(kBkWarps) * (ifr / GR)) * GR + ifr % GR
                                      : ic0 * uint64_t(RT) + ifr;
            if (lane == 0) {
                if constexpr (XM == 2)   // profiling: no L2 eviction hint
                    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     ring + slot * kBkStage),
                                 "l"(reinterpret_cast<uint64_t>(x + gfrag * 512u)), "r"(nf * 512u), "r"(bar)
                                 : "memory");
                else
                    asm volatile(
                        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
                        "[%3], %4;" ::"r"(ring + slot * kBkStage),
                        "l"(reinterpret_cast<uint64_t>(x + gfrag * 512u)), "r"(nf * 512u), "r"(bar), "l"(policy)
                        : "memory");
            }
            ifr += nf;
            ++t_issue;
        };
        open_issue_unit();
#pragma unroll 1
        for (int s = 0; s < NS; ++s) issue();
        // ldmatrix row address of this lane inside a fragment: matrix mi = lane>>3 supplies line
        // (k = (lane&7) + 8*(mi>>1), half = mi&1): d0 = (k 0-7, j 0-7), d1 = (k 0-7, j 8-15),
        // d2 = (k 8-15, j 0-7), d3 = (k 8-15, j 8-15)
        const uint32_t mi = lane >> 3;
        const uint32_t ld_off = 32u * ((lane & 7u) + 8u * (mi >> 1)) + 16u * (mi & 1u);
        const unsigned g = lane >> 2, c = lane & 3u;
        uint32_t t_cons = 0;
#pragma unroll 1
        for (uint32_t k = 0;; ++k) {
            mbar_wait(&sh.qfull[k % kBkQ], (k / kBkQ) & 1u);
            const unsigned long long u = sh.q[k % kBkQ];
            if (u >= u_total) break;
            const Unit un = unit_of(p, u);
            const uint32_t Cu = Cg / un.S, nc = Cu / kBkWarps;
            const uint32_t buf = k & 1u;
            mbar_wait(&sh.freed[buf], ((k >> 1) & 1u) ^ 1u);   // the manager is done with this table
            // chunk ci of the share is unit-local chunk (w + 8 (ci / GC)) GC + ci % GC (IL) or w nc + ci
            float* out = sh.chunk[buf] + (IL ? warp * GC : warp * nc);
            auto oidx = [&](uint32_t i) { return IL ? (i / GC) * (kBkWarps * GC) + i % GC : i; };
            const uint32_t nfrag = nc * uint32_t(RT);
            float lo[4] = {0.f, 0.f, 0.f, 0.f}, hi[4] = {0.f, 0.f, 0.f, 0.f};
            uint32_t bb0 = 0, bb1 = 0;
            uint32_t r = 0, ci = 0;
            constexpr uint32_t FPS = kBkStage / 512u;   // fragments per stage
#pragma unroll 1
            for (uint32_t f0 = 0; f0 < nfrag; f0 += FPS) {
                const uint32_t slot = t_cons % NS;
                mbar_wait(&sh.full[warp][slot], (t_cons / NS) & 1u);
                const uint32_t sb = ring + slot * kBkStage + ld_off;
                const uint32_t nf = min(FPS, nfrag - f0);
#pragma unroll
                for (uint32_t q = 0; q < FPS; ++q) {
                    if (XM != 1 && q < nf) {   // XM 1 (profiling): stream only, no MMA
                        uint32_t d0, d1, d2, d3;
                        ldsm_x4_trans(sb + q * 512u, d0, d1, d2, d3);
                        // C_r = ones x M_r + C_{r-1} (reduction.hpp:177): columns 0-7 and 8-15
                        mma_16816(lo, kOnesF16x2, kOnesF16x2, kOnesF16x2, kOnesF16x2, d0, d2);
                        mma_16816(hi, kOnesF16x2, kOnesF16x2, kOnesF16x2, kOnesF16x2, d1, d3);
                        if (++r == uint32_t(RT)) {
                            r = 0;
                            // C_R -> binary16 (:179-181), kept by the lanes of group g = ci mod 8
                            const uint32_t b0 = pack_h2(lo[0], lo[1]), b1 = pack_h2(hi[0], hi[1]);
                            const uint32_t kk = ci & 7u;
                            if (g == kk) {
                                bb0 = b0;
                                bb1 = b1;
                            }
                            lo[0] = lo[1] = lo[2] = lo[3] = hi[0] = hi[1] = hi[2] = hi[3] = 0.f;
                            if (kk == 7u || ci + 1 == nc) {
                                // finishing MMA (:182) for chunks ci-kk .. ci (missing ones are zero)
                                float fin[4] = {0.f, 0.f, 0.f, 0.f};
                                mma_16816(fin, kOnesF16x2, kOnesF16x2, kOnesF16x2, kOnesF16x2, bb0, bb1);
                                ovf |= !isfinite(fin[0]) || !isfinite(fin[1]);
                                if (g == 0) {
                                    if (2 * c <= kk) out[oidx(ci - kk + 2 * c)] = fin[0];
                                    if (2 * c + 1 <= kk) out[oidx(ci - kk + 2 * c + 1)] = fin[1];
                                }
                                bb0 = bb1 = 0;
                            }
                            ++ci;
                        }
                    }
                }
                // the MMAs consumed this lane's fragments: order its generic reads of the slot
                // before the async-proxy refill, then lane 0 refills it
                fence_proxy_async();
                __syncwarp();
                issue();
                ++t_cons;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.done[buf]);
        }
    } else {
        // -------------------------------------------------------------------- manager warp
        unsigned long long* ctr = p.work_counter;
        if (lane == 0) {
            for (int i = 0; i < kBkQD; ++i) {
                const unsigned long long u = atomicAdd(ctr, 1ull);
                if (u == last_claim) *ctr = 0ull;
                sh.q[i] = u;
                mbar_arrive(&sh.qfull[i]);
            }
        }
        __syncwarp();
#pragma unroll 1
        for (uint32_t k = 0;; ++k) {
            const unsigned long long u = sh.q[k % kBkQ];   // written by this warp's lane 0
            if (u >= u_total) break;
            unsigned long long nxt = 0;
            if (lane == 0) nxt = atomicAdd(ctr, 1ull);   // its latency hides behind this unit
            const Unit un = unit_of(p, u);
            const uint32_t Gu = G / un.S;
            const uint64_t b0 = un.gi * G + uint64_t(un.piece) * Gu;
            const uint32_t buf = k & 1u;
            mbar_wait(&sh.done[buf], (k >> 1) & 1u);
            range_trees_blocks(p, b0, Gu, sh.chunk[buf], sh.block, 0, 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.freed[buf]);
            if (un.S == 1) {
                tile_tree_group(p, un.gi, sh.block);
            } else {
                for (uint32_t b = lane; b < Gu; b += 32) p.block_scratch[b0 + b] = sh.block[b];
                __syncwarp();
                unsigned t = 0;
                if (lane == 0)
                    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(p.group_count + un.gi) : "memory");
                t = __shfl_sync(kFull, t, 0);
                __syncwarp();   // lane 0's acquire orders the other lanes' reads of the pieces
                if (t == un.S - 1) {
                    tile_tree_group<true>(p, un.gi, p.block_scratch + un.gi * G);
                    if (lane == 0) p.group_count[un.gi] = 0u;
                }
            }
            if (lane == 0) {
                if (nxt == last_claim) *ctr = 0ull;
                const uint32_t slot = (k + kBkQD) % kBkQ;
                sh.q[slot] = nxt;
                mbar_arrive(&sh.qfull[slot]);
            }
            __syncwarp();
        }
    }
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    __syncthreads();
    finalize_last_cta<true>(p, sh.scratch, &sh.last, 32 * kBkWarps);
}

using BkKernel = void (*)(SpParams);

struct BkPick {
    BkKernel fn;
    uint32_t ring;   // dynamic shared memory: 8 warps x NS stages
};

template <int RT, int NS, uint32_t SB, bool IL = false, int XM = 0>
constexpr BkPick bk_make() {
    return {sp_bulk_kernel<RT, NS, SB, IL, XM>, uint32_t(kBkWarps) * NS * SB};
}

// Ring shape per chain length: NS stages of SB bytes per warp (default 4 x 2 KiB), each warp
// streaming the contiguous eighth of a unit.  Profiling modes (debug_mode, R = 1; measured in
// DESIGN.md section 3): 30 = 6 x 2 KiB, 31 = 3 x 4 KiB, 32 = 8 x 1 KiB, 33 / 37 = shares
// interleaved in granules of lcm(stage, chunk), 34 / 36 / 38 = stream only (no MMA; timing),
// 35 = no L2 eviction hint.
BkPick bk_pick(uint32_t R, int mode = 0) {
    if (R == 1 && mode == 30) return bk_make<1, 6, 2048>();
    if (R == 1 && mode == 31) return bk_make<1, 3, 4096>();
    if (R == 1 && mode == 32) return bk_make<1, 8, 1024>();
    if (R == 1 && mode == 33) return bk_make<1, 4, 2048, true>();       // granule-interleaved shares
    if (R == 1 && mode == 34) return bk_make<1, 4, 2048, false, 1>();   // stream only (timing)
    if (R == 1 && mode == 35) return bk_make<1, 4, 2048, false, 2>();   // no L2 hint
    if (R == 1 && mode == 36) return bk_make<1, 4, 2048, true, 1>();    // stream only, interleaved
    if (R == 1 && mode == 37) return bk_make<1, 3, 4096, true>();       // 3 x 4 KiB interleaved
    if (R == 1 && mode == 38) return bk_make<1, 3, 4096, true, 1>();    // the same, stream only
    switch (R) {
    case 1: return bk_make<1, 4, 2048>();
    case 2: return bk_make<2, 4, 2048>();
    case 3: return bk_make<3, 4, 2048>();
    case 4: return bk_make<4, 4, 2048>();
    case 5: return bk_make<5, 4, 2048>();
    case 6: return bk_make<6, 4, 2048>();
    case 7: return bk_make<7, 4, 2048>();
    case 8: return bk_make<8, 4, 2048>();
    default: return {nullptr, 0};
    }
}

}  // namespace

// chunks per interleave granule (lcm(8, R) fragments: covers the 2 and 4 KiB stage shapes)
static uint32_t bk_granule_chunks(uint32_t R) { return bk_lcm(8, R) / R; }

bool bulk_supported(const SpGeometry& g) {
    // R <= 8 (compile-time chain), the group a whole number of granules per warp, at least one
    // full group
    return g.m == 16 && g.R >= 1 && g.R <= 8 && (uint64_t(g.G) * g.W) % (kBkWarps * bk_granule_chunks(g.R)) == 0 &&
           uint64_t(g.G) * g.W <= uint64_t(kMaxChunksPerGroup) && g.n / g.group_elems > 0;
}

int bulk_max_grid(uint32_t R, int mode) {
    static PerDeviceOnce once;
    const cudaError_t e = once([] {
        for (int md : {0, 30, 31, 32, 33, 34, 35, 36, 37, 38})
            for (uint32_t r = 1; r <= 8; ++r) {
                const BkPick k = bk_pick(r, md);
                const cudaError_t a = cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           int(k.ring));
                if (a != cudaSuccess) return a;
            }
        return cudaSuccess;
    });
    if (e != cudaSuccess) return 0;
    const BkPick k = bk_pick(R, mode);
    if (!k.fn) return 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.fn, kBkThreads, k.ring);
    return std::max(1, std::min(per_sm, 2)) * sm_count();
}

void bulk_plan(const SpGeometry& g, SpParams* p, int grid) {
    const uint64_t groups = p->group_end - p->group_begin;
    const uint32_t Cg = g.G * g.W;
    // pieces of S whole blocks, each warp share a whole number of chunks
    auto ok = [&](uint32_t S) {
        return S <= g.G && g.G % S == 0 && (Cg / S) % (kBkWarps * bk_granule_chunks(g.R)) == 0;
    };
    uint32_t S = 1;
    while (double(groups) * S < 3.0 * grid && ok(S * 2)) S *= 2;
    uint32_t St = S;
    const uint64_t group_bytes = g.group_elems * 2;
    while (group_bytes / St > kBkTailPieceBytes && ok(St * 2)) St *= 2;
    p->split = S;
    p->split_tail = St;
    p->tail_group = p->group_end;
    if (St > S) {
        const uint64_t tail = std::min<uint64_t>(groups, (uint64_t(kBkTailUnitsPerCta) * grid + St - 1) / St);
        p->tail_group = p->group_end - tail;
        if (p->tail_group == p->group_begin) p->split = St;
    }
}

cudaError_t launch_bulk(const SpParams& p, int grid, cudaStream_t s) {
    const BkPick k = bk_pick(p.R, p.debug_mode);
    if (!k.fn || bulk_max_grid(p.R, p.debug_mode) == 0) return cudaErrorInvalidValue;
    k.fn<<<grid, kBkThreads, k.ring, s>>>(p);
    return cudaGetLastError();
}

}  // namespace tcr
