// tcr_sp_genm.cu -- single-pass chained reduction for fragment sides m != 16.
//
// The reference accepts any power of two m >= 2 (check_side, fragment.hpp:22-25) and defaults
// to m = 4 (reduction.hpp:41).  A warp chunk is R fragments of m*m elements; the partial of
// column j is C_R[j] = sum_r sum_k M_r[k][j] over the chunk (ones x M, :173-177), rounded to
// binary16 (:179-181), and the chunk result is the ascending-j fp32 sum of the m binary16
// partials (the finishing mma, :182, fragment.hpp:89-92 -- reproduced operation for operation
// on the CUDA cores here).  The same per-warp cp.async streaming as tcr_sp_async.cu feeds
// HMMA.16816 with a 0/1 SELECTOR matrix as the B operand instead of ones, so one tensor-core
// op produces the column sums of several fragments / column groups at once:
//
//   m in {2, 4}   natural layout: A rows = 16 chunks (row i of each chunk per MMA, the chain
//                 over the chunk's 16-element rows accumulates in D), B[k][n] = [k mod m == n]
//                 (m = 2 with R in {1,2}: several chunks per row, n = 2*chunk_in_row + j);
//   m = 8         transposed 16x16 tiles (ldmatrix.trans), B[t][n] = [row t is in chunk slot n],
//                 partial(j) = D[j][n] + D[j+8][n];
//   m in {32,64,128}  transposed tiles, B[t][n] = [t mod (m/16) == n], partial(16n + j) = D[j][n],
//                 accumulated over the chunk's R*(m/16)^2 tiles.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "tcr_device.cuh"
#include "tcr_kernels.h"
#include "tcr_pipeline.cuh"

namespace tcr {

namespace cg = cooperative_groups;

namespace {

using namespace pipe;

constexpr int kGmWarps = 8;
constexpr int kGmThreads = 32 * kGmWarps;
constexpr int kGmTrDepth = 16;                // transposed stream: 512-byte tile stages per warp

__device__ __forceinline__ void cp16(uint32_t saddr, const void* g, uint32_t bytes) {
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t& d0, uint32_t& d1, uint32_t& d2, uint32_t& d3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t& d0, uint32_t& d1, uint32_t& d2, uint32_t& d3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3)
                 : "r"(addr));
}

__device__ __forceinline__ float h_round(float v) { return h_to_f32(f32_to_h(v)); }

// The reference chunk (chained_warp_reduce, reduction.hpp:164-184, with the emulated mma of
// fragment.hpp:82-97: ascending-k fp32 sums from 0, C added last) evaluated exactly on one CUDA
// core.  Slow path for a chunk whose tensor-core result is NaN: the selector engines multiply
// every binary16 by 0/1 entries, and a non-finite input times 0 is NaN where the reference's
// all-ones products keep +-inf -- recomputing keeps the reference's non-finite value.
template <bool F32 = false>
__device__ __forceinline__ float chunk_exact(const void* xv, uint64_t n, uint64_t e0, uint32_t m, uint32_t R) {
    float fin = 0.0f;
    for (uint32_t j = 0; j < m; ++j) {
        float c = 0.0f;
        for (uint32_t r = 0; r < R; ++r) {
            float col = 0.0f;
            for (uint32_t k = 0; k < m; ++k) {
                const uint64_t e = e0 + uint64_t(r) * m * m + uint64_t(k) * m + j;
                float v = 0.0f;   // zero padding (reduction.hpp:244-245)
                if (e < n) v = F32 ? h_round(static_cast<const float*>(xv)[e]) : h_to_f32(static_cast<const uint16_t*>(xv)[e]);
                col = col + v;
            }
            c = col + c;
        }
        fin = fin + h_round(c);
    }
    return fin + 0.0f;
}


// binary16 0/1 pair
__device__ __forceinline__ uint32_t sel2(bool lo, bool hi) {
    return (lo ? 0x3C00u : 0u) | (hi ? 0x3C000000u : 0u);
}

// Adjacent tree over the G (power of two) block results of a group by the whole CTA: thread t
// takes blocks [t seg, (t+1) seg), the warps' xor trees pair adjacent lanes, thread 0 pairs the
// 8 warp results -- one eighth of the serial work per thread of a one-warp tree (G reaches 4096
// for small chunks; measured +4..65 % on m = 2, 4, 8).  Every thread calls.
__device__ __forceinline__ void group_tree_cta(const SpParams& p, uint64_t gi, const float* blocks) {
    __shared__ float s_w[kGmWarps];
    const uint32_t G = p.G;
    const uint32_t seg = G >= uint32_t(kGmThreads) ? G / kGmThreads : 1;
    const uint32_t lo = threadIdx.x * seg;
    float acc = 0.0f;
    if (seg <= 8 && lo < G) {
        // short segments: the same adjacent tree unrolled in registers (no stack frame)
        const float* v = blocks + lo;
        if (seg == 1) {
            acc = v[0];
        } else if (seg == 2) {
            acc = v[0] + v[1];
        } else if (seg == 4) {
            acc = (v[0] + v[1]) + (v[2] + v[3]);
        } else {
            acc = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
        }
    } else if (lo < G) {
        // longer segments (B = 32: G = 4096, 16 per thread): compile-time register trees
        acc = lane_segment_tree([&](uint32_t i) { return blocks[i]; }, lo, seg);
    }
    acc = warp_tree_xor(acc);
    if (lane_id() == 0) s_w[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0 && p.group_partials) {
        static_assert(kGmWarps == 8, "three pairing levels");
        const float a = (s_w[0] + s_w[1]) + (s_w[2] + s_w[3]);
        const float b = (s_w[4] + s_w[5]) + (s_w[6] + s_w[7]);
        const float v = a + b;
        p.group_partials[gi] = v;
        // overflow note (reduction.hpp:78-81): some binary16 of the group -- input or C_R
        // partial -- was non-finite iff a chunk result was, iff the group partial is (finite
        // chunk results of one group cannot overflow binary32)
        if (!isfinite(v)) atomicOr(p.overflow, 1u);
    }
}

// Group epilogue.  A NaN chunk result may be an artefact of the selector products (0 x inf).
// REPAIR instantiations (the C ABI re-runs a call in this mode when its result came back NaN
// with the overflow note set, and always uses it for results that stay on the device): every
// non-finite chunk result already set the thread's overflow note (`ovf`, reduction.hpp:78-81),
// so only then does the CTA scan its chunk table and recompute the NaN chunks exactly
// (chunk_exact) before the block stage.  The default instantiations carry none of this code.
template <bool REPAIR, bool F32 = false>
__device__ __forceinline__ void group_epilogue(const SpParams& p, uint64_t gi, float* s_chunk, float* s_block,
                                               uint32_t m, bool ovf) {
    if constexpr (REPAIR) {
        if (__syncthreads_or(ovf)) {
            const uint32_t Cg = p.G * p.W;
            const uint64_t ce = uint64_t(p.R) * m * m;
            for (uint32_t i = threadIdx.x; i < Cg; i += kGmThreads)
                if (isnan(s_chunk[i]))
                    s_chunk[i] = chunk_exact<F32>(p.x, p.n, (gi * Cg + i) * ce, m, p.R);
            __syncthreads();
        }
    } else {
        __syncthreads();
    }
    tile_trees_blocks(p, gi, s_chunk, s_block, threadIdx.x >> 5, kGmWarps);
    __syncthreads();
    group_tree_cta(p, gi, s_block);
    __syncthreads();
}

// Group stage when the block trees already ran in registers (m = 4, W <= 8: the block results are
// in s_block): publish them (ORDERED / ATOMIC finalisers), then the group tree.
__device__ __forceinline__ void group_epilogue_blocks(const SpParams& p, uint64_t gi, float* s_block) {
    __syncthreads();
    if (p.block_partials || p.finalize == kFinAtomic)
        for (uint32_t b = threadIdx.x; b < p.G; b += kGmThreads) publish_block(p, gi * p.G + b, s_block[b]);
    group_tree_cta(p, gi, s_block);
    __syncthreads();
}

// ===================================================================== natural layout, m in {2, 4}
// A PERIOD is lcm(16, chunk) elements = PR 16-element rows holding CP whole chunks (m = 4: one
// chunk of R rows; m = 2: CP = 4 / gcd(4, R) chunks, which may straddle rows).  A row i of an
// MMA = row rho of period i, so a unit = 16 periods and the chain over the PR rows of a period
// accumulates in D with B[k][n] = [element 16 rho + k of the period is column j of chunk slot
// q, n = q m + j].  Stages: row blocks of RB = min(PR, 16) rows of all 16 periods.
struct NatShape {
    uint32_t PR, CP;           // rows and chunks per period
    uint32_t RB;               // rows per stage
    uint32_t chunks_per_unit;  // 16 * CP
};

__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
// predicated shared store (one STS with a predicate, no branch)
__device__ __forceinline__ void sts_pred(uint32_t addr, float v, bool on) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.f32 [%0], %1;\n\t}" ::"r"(addr), "f"(v),
                 "r"(uint32_t(on))
                 : "memory");
}

// Generic natural layout for the periods gm_nat_fast_kernel does not take (9-15 rows, or more
// than 16): stages are row blocks of RB = min(PR, 16) rows of all 16 periods, two per warp.  (A cross-group issue cursor and
// register-capped variants measured 1-10 % slower here.)
template <int M, bool REPAIR>
__global__ void __launch_bounds__(kGmThreads) gm_nat_kernel(const SpParams p, const NatShape S) {
    pdl_release();
    constexpr int ND = 2;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ float s_scratch[32];
    __shared__ int s_last;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t R = p.R;
    const uint32_t RB = S.RB;
    const uint32_t PR = S.PR;
    const uint32_t nblk = (PR + RB - 1) / RB;               // stages per unit
    const uint32_t stage_bytes = 16u * RB * 32u;
    float* s_chunk = reinterpret_cast<float*>(dsm + kGmWarps * ND * stage_bytes);
    float* s_block = s_chunk + p.G * p.W;
    const uint32_t ring = smem_u32(dsm) + warp * ND * stage_bytes;
    const uint32_t ce = R * M * M;                                    // chunk elements
    const uint32_t period_el = PR * 16u;
    const uint32_t Cg = p.G * p.W;
    const uint32_t units = (Cg + S.chunks_per_unit - 1) / S.chunks_per_unit;
    const bool straddle = S.CP > 1 && PR > 1;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    // selector B for period row rho: thread holds B[2c][g], B[2c+1][g], B[2c+8][g], B[2c+9][g]
    auto bsel = [&](uint32_t rho, uint32_t k) -> bool {
        const uint32_t e = 16u * rho + k;                             // element of the period
        return (e / ce) * M + (e % M) == g;
    };
    uint32_t b0 = sel2(bsel(0, 2 * c), bsel(0, 2 * c + 1)), b1 = sel2(bsel(0, 2 * c + 8), bsel(0, 2 * c + 9));
    const uint32_t bfin = sel2((2 * c) / M == g, (2 * c + 1) / M == g);   // finishing B2, rows k < 8
    // ldmatrix (non-transposed) row supplied by this lane: A row (period) rho8, column half.
    // Stage layout: 16-byte unit u = 2 (period * rb + row) + half, stored at u ^ (period & 7)
    // (a bijection for rb a power of two; the 8 periods of one ldmatrix phase hit 8 bank groups).
    const uint32_t rho8 = (lane & 7u) + 8u * ((lane >> 3) & 1u), half = lane >> 4;
    // generic path, full row blocks of RB rows: this lane's first piece and the per-row step
    const uint32_t gper0 = lane / (2u * RB), grr0 = lane % (2u * RB), gdq = 32u / (2u * RB), gdr = 32u % (2u * RB);
    bool ovf = false;

    for (uint64_t gi = p.group_begin + blockIdx.x; gi < p.group_end; gi += gridDim.x) {
        const uint64_t gel0 = gi * uint64_t(Cg) * ce;                     // first element of the group
        const uint64_t gel1 = gel0 + uint64_t(Cg) * ce;
        const uint64_t lim = gel1 < p.n ? gel1 : p.n;
        // every load in range: the units cover exactly the group (16 * CP | Cg) and it is whole
        const bool full = gel1 <= p.n && Cg % S.chunks_per_unit == 0;
        const uint32_t my_units = units > warp ? (units - warp + kGmWarps - 1) / kGmWarps : 0;
        const uint32_t F = my_units * nblk;                               // stages this warp streams
        uint32_t iu = 0, iblk = 0, islot = 0;                             // issue cursor
        auto issue = [&]() {
            if (iu < my_units) {
                const uint32_t r0 = iblk * RB, rb = min(RB, PR - r0);
                const uint64_t e_unit = gel0 + uint64_t(warp + iu * kGmWarps) * 16u * period_el + r0 * 16u;
                const uint32_t dst = ring + islot * stage_bytes;
                // piece = lane + 32 t = per * 2 rb + rr: compile-time shifts on the fast path,
                // one division per stage then increments on the generic one (any rb <= 16)
                const bool last = rb != RB;
                uint32_t per = last ? lane / (2u * rb) : gper0;
                uint32_t rr = last ? lane % (2u * rb) : grr0;
                const uint32_t dq = last ? 32u / (2u * rb) : gdq;
                const uint32_t dr = last ? 32u % (2u * rb) : gdr;
#pragma unroll
                for (uint32_t t = 0; t < 16u; ++t) {
                    if (t >= rb) break;
                    const uint32_t piece = lane + 32u * t;
                    const uint64_t e = e_unit + per * period_el + rr * 8u;
                    if (full) {
                        cp16(dst + ((piece ^ (per & 7u)) * 16u), x + e, 16u);
                    } else {
                        const uint32_t bytes = e + 8 <= lim ? 16u : (e < lim ? uint32_t(lim - e) * 2u : 0u);
                        cp16(dst + ((piece ^ (per & 7u)) * 16u), x + (e < lim ? e : 0), bytes);
                    }
                    per += dq;
                    rr += dr;
                    if (rr >= 2u * rb) {
                        rr -= 2u * rb;
                        ++per;
                    }
                }
                if (++iblk == nblk) {
                    iblk = 0;
                    ++iu;
                }
            }
            cp_commit();
            islot = islot + 1 == uint32_t(ND) ? 0 : islot + 1;
        };
#pragma unroll
        for (int f = 0; f < ND - 1; ++f) issue();
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t cu = 0, cblk = 0, cslot = 0;                             // consume cursor
        for (uint32_t f = 0; f < F; ++f) {
            issue();
            cp_wait<ND - 1>();
            __syncwarp();
            const uint32_t base = ring + cslot * stage_bytes;
            cslot = cslot + 1 == uint32_t(ND) ? 0 : cslot + 1;
            const uint32_t r0 = cblk * RB, rb = min(RB, PR - r0);
#pragma unroll
            for (uint32_t i = 0; i < 16u; ++i) {
                if (i >= rb) break;
                if (straddle) {
                    const uint32_t rho = r0 + i;
                    b0 = sel2(bsel(rho, 2 * c), bsel(rho, 2 * c + 1));
                    b1 = sel2(bsel(rho, 2 * c + 8), bsel(rho, 2 * c + 9));
                }
                const uint32_t unit16 = 2u * (rho8 * rb + i) + half;
                uint32_t d0, d1, d2, d3;
                ldsm4(base + ((unit16 ^ (rho8 & 7u)) * 16u), d0, d1, d2, d3);
                mma_16816(acc, d0, d1, d2, d3, b0, b1);   // C_i = A_i x Bsel + C_{i-1}
            }
            __syncwarp();
            const uint32_t u = cu;
            if (++cblk < nblk) continue;
            cblk = 0;
            ++cu;
            // unit complete. acc: (period g, col 2c), (g, 2c+1), (g+8, 2c), (g+8, 2c+1)
            // Finishing MMA on the tensor core (reduction.hpp:182): A2 = binary16(C_R) in the
            // accumulator layout (= the A-operand layout of columns k < 8), B2[k][q] = [k / m == q]
            // -> D2[period][q] = sum_j binary16(C_R[q m + j]) for chunk slot q, all in registers.
            {
                float d2[4] = {0.f, 0.f, 0.f, 0.f};
                mma_16816(d2, pack_h2(acc[0], acc[1]), pack_h2(acc[2], acc[3]), 0u, 0u, bfin, 0u);
                const uint32_t cu0 = (warp + u * kGmWarps) * S.chunks_per_unit;
                if (2 * c < S.CP) {
                    ovf |= !isfinite(d2[0]) || !isfinite(d2[2]);
                    const uint32_t ca = cu0 + g * S.CP + 2 * c, cb = cu0 + (g + 8) * S.CP + 2 * c;
                    if (ca < Cg) s_chunk[ca] = d2[0];
                    if (cb < Cg) s_chunk[cb] = d2[2];
                }
                if (2 * c + 1 < S.CP) {
                    ovf |= !isfinite(d2[1]) || !isfinite(d2[3]);
                    const uint32_t ca = cu0 + g * S.CP + 2 * c + 1, cb = cu0 + (g + 8) * S.CP + 2 * c + 1;
                    if (ca < Cg) s_chunk[ca] = d2[1];
                    if (cb < Cg) s_chunk[cb] = d2[3];
                }
            }
            acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
        }
        cp_wait<0>();
        group_epilogue<REPAIR>(p, gi, s_chunk, s_block, M, ovf);
    }
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kGmThreads);
}

// Natural layout, PR = RBC <= 8 or 16 rows (m = 4 with R <= 8 or 16, m = 2 with a period of that
// many rows).  A unit (16 periods) is 256 RBC CONTIGUOUS elements and lane l's 16-byte piece q of a stage is elements 8 (l + 32 q): the stage of a warp
// is UPS consecutive units (one 2 KiB cp.async burst per stage for the one-row shapes instead of
// a 512-byte one), every address and ring offset is a compile-time constant plus a per-lane
// invariant, chunk results leave through precomputed shared addresses, and the overflow note is
// a NaN-propagating accumulator (x * 0 is NaN exactly when x is not finite) instead of per-value
// tests.  Same arithmetic, operand order and chunk -> shared-table mapping as gm_nat_kernel.
//
// F32: the reference's own input format (reduce(std::span<const float>)) streamed as is, from_single
// (half.hpp:32-59) fused into the load: the stage holds the fp32 bytes unswizzled, lane (g, c)
// reads 16 bytes = elements 4c .. 4c+3 of rows g and g + 8 (LDS.128, conflict-free) and packs
// them with cvt.rn.f16x2.f32 into its A registers -- a permutation of the MMA's k index
// (k = 2c, 2c+1, 2c+8, 2c+9 <-> element 4c .. 4c+3) that the selector B follows, so D is
// unchanged.  4 bytes per element from HBM, no conversion pass.
// BT (m = 4, W = B/32 in {1, 2, 4, 8}; dispatched for W <= 2): the unit's 16 chunk results (lanes c = 0 hold chunks g and
// g + 8 after the finishing MMA) go through the reference's block tree (reduction.hpp:90-101:
// v[i] += v[i + len/2], len = W ... 2) in registers with shuffles; only block results reach shared
// memory, and the chunk table disappears (a smaller footprint: one more CTA per SM).
template <int M, int RBC, int UPS, int ND, bool REPAIR, bool XG = true, bool F32 = false, int BT = 0>
__global__ void __launch_bounds__(kGmThreads) gm_nat_fast_kernel(const SpParams p, const NatShape S) {
    pdl_release();
    constexpr uint32_t ESZ = F32 ? 4u : 2u;                            // bytes per input element
    constexpr uint32_t EP = 16u / ESZ;                                 // elements per 16-byte piece
    constexpr uint32_t UNIT_EL = 256u * RBC;
    constexpr uint32_t UNIT_B = ESZ * UNIT_EL;
    constexpr uint32_t STAGE_EL = UNIT_EL * UPS;
    constexpr uint32_t STAGE_B = ESZ * STAGE_EL;
    constexpr uint32_t NQ = STAGE_B / 512u;                           // 16-byte pieces per lane per stage
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ float s_scratch[32];
    __shared__ int s_last;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t R = p.R;
    float* s_chunk = reinterpret_cast<float*>(dsm + kGmWarps * ND * STAGE_B);
    float* s_block = BT ? s_chunk : s_chunk + p.G * p.W;
    const uint32_t ring = smem_u32(dsm) + warp * ND * STAGE_B;
    const uint32_t ce = R * M * M;
    const uint32_t CP = S.CP, cpu = S.chunks_per_unit;
    const uint32_t Cg = p.G * p.W;
    const uint32_t sunits = ((Cg + cpu - 1) / cpu + UPS - 1) / UPS;  // stages per group
    const char* xb = static_cast<const char*>(p.x);
    auto bsel = [&](uint32_t rho, uint32_t k) -> bool {
        const uint32_t e = 16u * rho + k;
        return (e / ce) * M + (e % M) == g;
    };
    // the element of the row that MMA index k holds (F32: the permutation above)
    auto kel = [&](uint32_t k) -> uint32_t { return F32 ? 4u * ((k & 7u) >> 1) + (k & 1u) + 2u * (k >> 3) : k; };
    const bool straddle = CP > 1 && RBC > 1;
    uint32_t b0 = sel2(bsel(0, kel(2 * c)), bsel(0, kel(2 * c + 1))),
             b1 = sel2(bsel(0, kel(2 * c + 8)), bsel(0, kel(2 * c + 9)));
    const uint32_t bfin = sel2((2 * c) / M == g, (2 * c + 1) / M == g);
    const uint32_t rho8 = (lane & 7u) + 8u * ((lane >> 3) & 1u), half = lane >> 4;
    // chunk slots this lane owns after the finishing MMA: columns 2c, 2c+1 of rows g, g+8
    const bool own0 = 2 * c < CP, own1 = 2 * c + 1 < CP;
    float* const s_own = s_chunk + g * CP + 2 * c;
    const uint32_t s_own_a = smem_u32(s_chunk) + 4u * g;   // M = 4 (CP = 1)
    float nanacc = 0.0f;
    bool ovf = false;
    const uint32_t F = sunits > warp ? (sunits - warp + kGmWarps - 1) / kGmWarps : 0;   // stages per group
    // The issue cursor runs ahead ACROSS groups: the next group's first stages are in flight
    // while this group's epilogue (block and group trees) runs, so the per-group pipeline drain
    // of a small group (<= 4096 chunks) is not paid.
    uint64_t igi = p.group_begin + blockIdx.x;
    uint64_t e_issue = 0, ilim = 0;
    bool ifull = false;
    uint32_t is = 0, islot = 0;
    auto iset = [&]() {
        const uint64_t gel0 = igi * uint64_t(Cg) * ce, gel1 = gel0 + uint64_t(Cg) * ce;
        ilim = gel1 < p.n ? gel1 : p.n;
        ifull = gel1 <= p.n && Cg % (cpu * UPS) == 0;
        e_issue = gel0 + uint64_t(warp) * STAGE_EL + EP * lane;          // this lane's piece 0
        is = 0;
    };
    iset();
    auto issue = [&]() {
        if (XG && F != 0 && is == F) {
            igi += gridDim.x;
            iset();
        }
        if (F != 0 && igi < p.group_end && is < F) {
            const uint32_t dst = ring + islot * STAGE_B;
            auto off = [&](uint32_t q) {
                if constexpr (F32) return q * 512u + 16u * lane;       // linear: LDS.128 rows are conflict-free
                const uint32_t piece = lane + 32u * (q % RBC);
                return (q / RBC) * UNIT_B + ((piece ^ ((piece / (2u * RBC)) & 7u)) * 16u);
            };
            if (ifull) {
#pragma unroll
                for (uint32_t q = 0; q < NQ; ++q) cp16(dst + off(q), xb + (e_issue + 32u * EP * q) * ESZ, 16u);
            } else {
#pragma unroll
                for (uint32_t q = 0; q < NQ; ++q) {
                    const uint64_t e = e_issue + 32u * EP * q;
                    const uint32_t bytes = e + EP <= ilim ? 16u : (e < ilim ? uint32_t(ilim - e) * ESZ : 0u);
                    cp16(dst + off(q), xb + (e < ilim ? e : 0) * ESZ, bytes);
                }
            }
            e_issue += uint64_t(kGmWarps) * STAGE_EL;
            ++is;
        }
        cp_commit();
        islot = islot + 1 == uint32_t(ND) ? 0 : islot + 1;
    };
#pragma unroll
    for (int f = 0; f < ND - 1; ++f) issue();
    uint32_t cslot = 0;

    for (uint64_t gi = p.group_begin + blockIdx.x; gi < p.group_end; gi += gridDim.x) {
        if (!XG && gi != p.group_begin + blockIdx.x) {   // per-group pipeline (A/B form)
            cp_wait<0>();
            igi = gi;
            iset();
            islot = 0;
            cslot = 0;
#pragma unroll
            for (int f = 0; f < ND - 1; ++f) issue();
        }
        const uint64_t gel1 = (gi + 1) * uint64_t(Cg) * ce;
        const bool full = gel1 <= p.n && Cg % (cpu * UPS) == 0;
        uint32_t cu0 = warp * UPS * cpu;                                  // first chunk of the stage
        for (uint32_t f = 0; f < F; ++f) {
            issue();
            cp_wait<ND - 1>();
            __syncwarp();
            const uint32_t base = ring + cslot * STAGE_B;
            cslot = cslot + 1 == uint32_t(ND) ? 0 : cslot + 1;
            // The UPS units of the stage are independent: their ldmatrix -> HMMA -> binary16 ->
            // finishing HMMA chains are interleaved (all loads, then all chains' MMAs, ...) so a
            // warp has UPS chains in flight instead of one (the kernel is latency-bound per warp).
            float acc[UPS][4];
#pragma unroll
            for (uint32_t j = 0; j < UPS; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
            for (uint32_t i = 0; i < RBC; ++i) {
                if (straddle) {
                    b0 = sel2(bsel(i, kel(2 * c)), bsel(i, kel(2 * c + 1)));
                    b1 = sel2(bsel(i, kel(2 * c + 8)), bsel(i, kel(2 * c + 9)));
                }
                uint32_t d[UPS][4];
                if constexpr (F32) {
                    // rows g and g + 8 of the unit's row block i, elements 4c .. 4c+3 (16 bytes)
#pragma unroll
                    for (uint32_t j = 0; j < UPS; ++j) {
                        const uint32_t r0 = base + j * UNIT_B + ((g * RBC + i) * 16u + 4u * c) * 4u;
                        const float4 lo = lds_f4(r0), hi = lds_f4(r0 + 8u * RBC * 64u);
                        d[j][0] = pack_h2(lo.x, lo.y);   // k = 2c, 2c+1     (rows 0-7)
                        d[j][1] = pack_h2(hi.x, hi.y);   //                  (rows 8-15)
                        d[j][2] = pack_h2(lo.z, lo.w);   // k = 2c+8, 2c+9   (rows 0-7)
                        d[j][3] = pack_h2(hi.z, hi.w);   //                  (rows 8-15)
                    }
                } else {
                    const uint32_t unit16 = 2u * (rho8 * RBC + i) + half;
#pragma unroll
                    for (uint32_t j = 0; j < UPS; ++j)
                        ldsm4(base + j * UNIT_B + ((unit16 ^ (rho8 & 7u)) * 16u), d[j][0], d[j][1], d[j][2], d[j][3]);
                }
#pragma unroll
                for (uint32_t j = 0; j < UPS; ++j) mma_16816(acc[j], d[j][0], d[j][1], d[j][2], d[j][3], b0, b1);
            }
            float d2s[UPS][4];
#pragma unroll
            for (uint32_t j = 0; j < UPS; ++j) {
                d2s[j][0] = d2s[j][1] = d2s[j][2] = d2s[j][3] = 0.f;
                mma_16816(d2s[j], pack_h2(acc[j][0], acc[j][1]), pack_h2(acc[j][2], acc[j][3]), 0u, 0u, bfin, 0u);
            }
#pragma unroll
            for (uint32_t j = 0; j < UPS; ++j) {
                const float* d2 = d2s[j];
                if constexpr (REPAIR) {
                    // non-owner columns are 0 unless an input is non-finite, which its owner sees
                    // too.  (The default instantiations read the overflow note off the group
                    // partial instead: group_tree_cta.)
                    nanacc = fmaf(d2[0], 0.0f, nanacc);
                    nanacc = fmaf(d2[1], 0.0f, nanacc);
                    nanacc = fmaf(d2[2], 0.0f, nanacc);
                    nanacc = fmaf(d2[3], 0.0f, nanacc);
                }
                const uint32_t cu = cu0 + j * cpu;
                if constexpr (M == 4 && BT > 0) {
                    // block trees of the unit's 16 / BT blocks: chunk k sits in lane 4 (k mod 8),
                    // d2[0] for k < 8, d2[2] for k >= 8; level len pairs lanes 4 len / 2 apart
                    float x0 = d2[0], x2 = d2[2];
#pragma unroll
                    for (int len = BT; len > 1; len >>= 1) {
                        const float t0 = __shfl_down_sync(kFull, x0, 2 * len), t2 = __shfl_down_sync(kFull, x2, 2 * len);
                        x0 = x0 + t0;   // v[i] += v[i + len/2] (only lanes with g mod len = 0 are used)
                        x2 = x2 + t2;
                    }
                    const uint32_t bu = cu / BT, bj = g / BT;           // the unit's first block, this lane's
                    const bool lead = c == 0 && (g % BT) == 0;
                    sts_pred(smem_u32(s_block) + 4u * (bu + bj), x0, lead && (full || bu + bj < p.G));
                    sts_pred(smem_u32(s_block) + 4u * (bu + 8u / BT + bj), x2, lead && (full || bu + 8u / BT + bj < p.G));
                } else if constexpr (M == 4) {
                    // one chunk per period (CP = 1): lanes c = 0 own chunks g and g + 8 of the unit;
                    // predicated stores at compile-time offsets, no branches
                    const uint32_t ca = cu + g;
                    sts_pred(s_own_a + 4u * cu, d2[0], c == 0 && (full || ca < Cg));
                    sts_pred(s_own_a + 4u * cu + 32u, d2[2], c == 0 && (full || ca + 8 < Cg));
                } else {
                    const uint32_t ca = cu + g * CP + 2 * c;
                    float* sp = s_own + cu;
                    if (own0 && (full || ca < Cg)) sp[0] = d2[0];
                    if (own0 && (full || ca + 8 * CP < Cg)) sp[8 * CP] = d2[2];
                    if (own1 && (full || ca + 1 < Cg)) sp[1] = d2[1];
                    if (own1 && (full || ca + 1 + 8 * CP < Cg)) sp[8 * CP + 1] = d2[3];
                }
            }
            __syncwarp();
            cu0 += kGmWarps * UPS * cpu;
        }
        ovf = nanacc != nanacc;
        if constexpr (BT > 0) group_epilogue_blocks(p, gi, s_block);
        else group_epilogue<REPAIR, F32>(p, gi, s_chunk, s_block, M, ovf);
    }
    cp_wait<0>();
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kGmThreads);
}

// ============================================================ m = 4, R = 1: register-direct stream
// The reference default shape (m = 4, R = 1, reduction.hpp:41) on binary16 data.  A TILE is 16
// consecutive chunks of 16 elements = 512 bytes = one HMMA: row i of A is chunk i, and lane
// (g, c) loads its A fragment straight from global memory -- 8 bytes of chunk g (elements 4c ..
// 4c+3) and 8 bytes of chunk g + 8 (two LDG.64; the 32 lanes of one load cover 256 contiguous
// bytes).  The k index is permuted exactly as in the fp32 path of gm_nat_fast_kernel (k = 2c,
// 2c+1, 2c+8, 2c+9 <-> element 4c .. 4c+3), so the selector B[k][n] = [column of k == n] and
// every MMA, binary16 rounding and finishing MMA is the same as there (bit-identical chunk
// results).  No shared-memory ring, no cp.async / ldmatrix: the loads land in registers, NB
// batches of U tiles per warp rotate through NB register buffers (NB - 1 batches = 6 KiB per
// warp in flight), chunk results go to the group's chunk table and the block / group trees run in
// the common epilogue.  Warp w of the CTA streams tiles [w T, (w+1) T) of each of its groups
// (T = Cg / 128); the batch sequence runs across groups, so the next group's loads are in
// flight during a group's epilogue.
constexpr int kM4U = 4;    // tiles per batch
constexpr int kM4NB = 4;   // register buffers (batches) per warp

__device__ __forceinline__ uint2 ldg_stream_v2(const void* p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

// 4 binary16 at element e, zero past n (the reference's zero padding, reduction.hpp:244-245)
__device__ __forceinline__ uint2 ld4_tail(const uint16_t* x, uint64_t e, uint64_t n) {
    if (e + 4 <= n) return ldg_stream_v2(x + e);
    uint16_t h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = e + i < n ? x[e + i] : uint16_t(0);
    return make_uint2(uint32_t(h[0]) | (uint32_t(h[1]) << 16), uint32_t(h[2]) | (uint32_t(h[3]) << 16));
}
// fp32 input: 4 floats (bits) at element e, zero past n
__device__ __forceinline__ uint4 ld4_tail(const float* x, uint64_t e, uint64_t n) {
    if (e + 4 <= n) return ldg_stream_v4(x + e);
    uint32_t f[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = e + i < n ? __float_as_uint(x[e + i]) : 0u;
    return make_uint4(f[0], f[1], f[2], f[3]);
}

// F32: the reference's own fp32 input streamed as is (16 bytes per row piece, LDG.128) and
// from_single (half.hpp:32-59) applied in registers with cvt.rn.f16x2.f32 -- the same A operand
// as the binary16 path on the rounded values; half the tiles per batch (the same bytes in flight).
// RTREE: the block and group trees in registers instead of through the chunk table (for small
// blocks, whose shared-memory epilogue dominates): after the finishing MMA, chunk k of a tile sits
// in lane 4 (k mod 8) (k < 8: d2[0], else d2[2]); the reference's block tree (v[i] += v[i + len/2],
// reduction.hpp:90-101) pairs lanes 2 len apart, the blocks' adjacent group tree continues across
// the tile, the batch, and the warp's contiguous range of tiles; one barrier per group combines
// the 8 warps.  The same operand pairs as the shared-memory path: bit-identical partials.
template <bool F32, int WT = 0, int RC = 1>   // WT > 0: RTREE with compile-time W = WT; RC = R
__global__ void __launch_bounds__(kGmThreads, 2) gm4_reg_kernel(const SpParams p, const bool l2_prefetch) {
    constexpr bool RTREE = WT > 0;
    // R = RC rows of 16 elements per chunk: a tile is 16 chunks = RC HMMAs chained through the
    // accumulator (C_r = ones x M_r + C_{r-1}, reduction.hpp:173-177), row r of every chunk per MMA
    pdl_release();
    using E = std::conditional_t<F32, float, uint16_t>;   // input element
    using V = std::conditional_t<F32, uint4, uint2>;      // 4 elements of a row
    constexpr int U = (F32 ? kM4U / 2 : kM4U) / RC;       // tiles per batch (the same bytes for every R)
    static_assert(U >= 1, "R too large for the register batches");
    extern __shared__ __align__(16) float s_tab[];
    __shared__ float s_scratch[32];
    __shared__ int s_last;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t Cg = p.G * p.W;
    float* s_chunk = s_tab;
    float* s_block = s_tab + Cg;
    const uint32_t T = Cg / (16u * kGmWarps);       // tiles per warp per group
    const uint32_t nb = T / U;                      // batches per warp per group
    const E* x = static_cast<const E*>(p.x);
    const uint64_t n = p.n;
    // selector of the permuted k (see above): b0 rows k = 2c, 2c+1 -> columns 0, 1; b1 rows
    // k = 2c+8, 2c+9 -> columns 2, 3
    const uint32_t b0 = sel2(g == 0, g == 1), b1 = sel2(g == 2, g == 3);
    const uint32_t bfin = sel2((2 * c) / 4 == g, (2 * c + 1) / 4 == g);
    const uint64_t g0 = p.group_begin + blockIdx.x;
    const uint64_t ngroups = p.group_end > g0 ? (p.group_end - g0 + gridDim.x - 1) / gridDim.x : 0;
    // lane's element offset inside a tile: chunk g row 0, elements 4c .. 4c+3 (chunk g + 8:
    // +128 RC; row r: +16 r)
    const uint32_t lane_el = 16u * RC * g + 4u * c;
    // this warp's chunk-table slot of tile t of batch (j mod nb), lanes c = 0 store
    const uint32_t s_lane = smem_u32(s_chunk) + 4u * (warp * T * 16u + g);

    V buf[kM4NB][2 * U * RC];
    // issue cursor: the ik-th group of this CTA, batch ib of it, this lane's element ie (advanced
    // by increments: no division on the issue path)
    uint64_t ik = 0, ie = 0;
    uint32_t ib = 0;
    bool ifull = false;
    auto iset = [&]() {
        const uint64_t gi = g0 + ik * gridDim.x;
        ie = gi * uint64_t(Cg) * 16u * RC + uint64_t(warp * T) * 256u * RC + lane_el;
        ifull = (gi + 1) * uint64_t(Cg) * 16u * RC <= n;
    };
    if (ngroups) iset();
    auto ldv = [&](const E* q) -> V {
        if constexpr (F32) return ldg_stream_v4(q);
        else return ldg_stream_v2(q);
    };
    auto issue = [&](V (&b)[2 * U * RC]) {
        if (ik >= ngroups) return;
        const E* q = x + ie;
        if (ifull) {
#pragma unroll
            for (int t = 0; t < U; ++t)
#pragma unroll
                for (int r = 0; r < RC; ++r) {
                    b[2 * (t * RC + r)] = ldv(q + 256u * RC * t + 16u * r);
                    b[2 * (t * RC + r) + 1] = ldv(q + 256u * RC * t + 16u * r + 128u * RC);
                }
        } else {
#pragma unroll
            for (int t = 0; t < U; ++t)
#pragma unroll
                for (int r = 0; r < RC; ++r) {
                    b[2 * (t * RC + r)] = ld4_tail(x, ie + 256u * RC * t + 16u * r, n);
                    b[2 * (t * RC + r) + 1] = ld4_tail(x, ie + 256u * RC * t + 16u * r + 128u * RC, n);
                }
        }
        ie += 256u * RC * U;
        if (++ib == nb) {
            ib = 0;
            if (++ik < ngroups) iset();
        }
    };
    const uint32_t W = RTREE ? uint32_t(WT) : p.W;
    uint64_t gblk0 = 0;   // RTREE: global block index of this warp's first block in the current group
    auto consume = [&](const V (&b)[2 * U * RC], uint32_t jb) -> float {
        const uint32_t tb = jb * U;   // first tile of the batch (jb-th of the group) in this warp's range
        float d2[U][4];
#pragma unroll
        for (int t = 0; t < U; ++t) {
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            // C_r = ones x M_r + C_{r-1} (reduction.hpp:173-177) for 16 chunks: A rows = chunks
#pragma unroll
            for (int r = 0; r < RC; ++r) {
                const int k = 2 * (t * RC + r);
                if constexpr (F32) {
                    const uint4 r0 = b[k], r1 = b[k + 1];   // chunks g, g + 8: elements 4c .. 4c+3 of row r
                    mma_16816(acc, pack_h2(__uint_as_float(r0.x), __uint_as_float(r0.y)),
                              pack_h2(__uint_as_float(r1.x), __uint_as_float(r1.y)),
                              pack_h2(__uint_as_float(r0.z), __uint_as_float(r0.w)),
                              pack_h2(__uint_as_float(r1.z), __uint_as_float(r1.w)), b0, b1);
                } else {
                    mma_16816(acc, b[k].x, b[k + 1].x, b[k].y, b[k + 1].y, b0, b1);
                }
            }
            d2[t][0] = d2[t][1] = d2[t][2] = d2[t][3] = 0.f;
            // C_R -> binary16 (:179-181), finishing MMA (:182): chunk g in d2[0], g + 8 in d2[2]
            mma_16816(d2[t], pack_h2(acc[0], acc[1]), pack_h2(acc[2], acc[3]), 0u, 0u, bfin, 0u);
        }
        if constexpr (RTREE) {
            float tv[U];
#pragma unroll
            for (int t = 0; t < U; ++t) {
                float x0 = d2[t][0], x2 = d2[t][2];
                // block trees (W = 1, 2, 4, 8, 16 chunks)
                if constexpr (WT == 16) {
                    x0 = x0 + x2;
#pragma unroll
                    for (uint32_t len = 8; len > 1; len >>= 1) x0 += __shfl_down_sync(kFull, x0, 2 * len);
                } else {
#pragma unroll
                    for (uint32_t len = WT; len > 1; len >>= 1) {
                        const float t0 = __shfl_down_sync(kFull, x0, 2 * len), t2 = __shfl_down_sync(kFull, x2, 2 * len);
                        x0 += t0;
                        x2 += t2;
                    }
                }
                if (p.block_partials || p.finalize == kFinAtomic) {
                    // block i of the tile: x0 of lane 4 W i (i < 8 / W), x2 of lane 4 W (i - 8 / W)
                    const uint64_t bt = gblk0 + uint64_t(tb + t) * (16u / W);
                    if (c == 0 && g % W == 0) {
                        publish_block(p, bt + g / W, x0);
                        if constexpr (WT < 16) publish_block(p, bt + 8u / W + g / W, x2);
                    }
                }
                // the tile's blocks, adjacent tree (lane 0)
                if constexpr (WT < 16) {
#pragma unroll
                    for (uint32_t off = 4 * WT; off < 32; off <<= 1) {
                        const float t0 = __shfl_down_sync(kFull, x0, off), t2 = __shfl_down_sync(kFull, x2, off);
                        x0 += t0;
                        x2 += t2;
                    }
                    x0 = x0 + x2;
                }
                tv[t] = x0;
            }
            // the batch's tiles, adjacent (U = 1, 2 or 4)
            static_assert(U == 1 || U == 2 || U == 4, "batch tree");
            if constexpr (U == 4) return (tv[0] + tv[1 % U]) + (tv[2 % U] + tv[3 % U]);
            else if constexpr (U == 2) return tv[0] + tv[1 % U];
            else return tv[0];
        } else {
#pragma unroll
            for (int t = 0; t < U; ++t) {
                const uint32_t a = s_lane + 64u * (tb + t);
                sts_pred(a, d2[t][0], c == 0);
                sts_pred(a + 32u, d2[t][2], c == 0);
            }
            return 0.f;
        }
    };
    // Profiling variant (knob): L2 prefetch one group ahead (cp.async.bulk.prefetch.L2, one
    // instruction per warp range).  Measured slower (2^28: 93.7 vs 85.9 us, 2^30: 337 vs 314 us):
    // the register pipeline alone keeps HBM busy, so it is off by default.
    const uint32_t wbytes = T * 256u * RC * uint32_t(sizeof(E));   // this warp's contiguous range of a group
    auto prefetch = [&](uint64_t gk) {
        if (!l2_prefetch || gk >= ngroups || lane != 0) return;
        const uint64_t gi = g0 + gk * gridDim.x;
        const uint64_t e0 = gi * uint64_t(Cg) * 16u * RC + uint64_t(warp) * T * 256u * RC;
        if (e0 + T * 256u * RC > n) return;          // a ragged group streams without it
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + e0), "r"(wbytes) : "memory");
    };
    prefetch(0);
#pragma unroll
    for (int s = 0; s < kM4NB - 1; ++s) issue(buf[s]);
    // nb is a multiple of NB (gm4_reg_ok): buffer s always holds a batch j = s mod NB
    __shared__ float s_wv[2][kGmWarps];   // RTREE: warp subtrees, double-buffered by group parity
    for (uint64_t gk = 0; gk < ngroups; ++gk) {
        prefetch(gk + 1);
        const uint64_t gi = g0 + gk * gridDim.x;
        gblk0 = gi * p.G + uint64_t(warp) * (T * 16u / W);
        // RTREE: adjacent tree over the nb / NB (a power of two) iteration values of the group:
        // a binary counter of partial subtrees (at most 6 levels: nb <= 256)
        float stk[8];
        int top = 0;
        for (uint32_t jj = 0; jj < nb; jj += kM4NB) {
            float bv[kM4NB];
#pragma unroll
            for (int s = 0; s < kM4NB; ++s) {
                // refill the buffer consumed one step ago, then consume buffer s
                issue(buf[(s + kM4NB - 1) % kM4NB]);
                bv[s] = consume(buf[s], jj + s);
            }
            if constexpr (RTREE) {
                static_assert(kM4NB == 4, "adjacent tree over 4 batches");
                float v = (bv[0] + bv[1]) + (bv[2] + bv[3]);
                for (uint32_t k = jj / kM4NB; k & 1u; k >>= 1) v = stk[--top] + v;
                stk[top++] = v;
            }
        }
        if constexpr (RTREE) {
            // the group tree: the 8 warps' adjacent subtrees
            if (lane == 0) s_wv[gk & 1][warp] = stk[0];
            __syncthreads();
            if (threadIdx.x == 0 && p.group_partials) {
                const float* w = s_wv[gk & 1];
                const float v = ((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7]));
                p.group_partials[gi] = v;
                if (!isfinite(v)) atomicOr(p.overflow, 1u);   // the overflow note, as group_tree_cta
            }
        } else {
            // the group's chunk table is complete: block trees (:90-101, :253), group tree
            group_epilogue<false>(p, gi, s_chunk, s_block, 4u, false);
        }
    }
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kGmThreads);
}

// m = 4, R = 1 register-direct engine eligibility: whole batches per warp per group
// (B = 32, W = 1: the RTREE instantiation -- trees in registers; the chunk-table epilogue of its
// 4096-block groups made the shared-memory form slower than the ring kernel, 4.59 vs 4.80 TB/s)
__host__ __device__ inline bool gm4_reg_ok(uint32_t m, uint32_t R, uint32_t W, uint32_t Cg, bool gm4_all_w = false) {
    return m == 4 && (R == 1 || R == 2 || R == 4) && Cg % (16u * kGmWarps * kM4U * kM4NB) == 0 &&
           (W >= 1 || gm4_all_w);
}

// ================================================================ transposed tiles, m = 8 or 16*S
// Item = K consecutive 256-element tiles holding CPT whole chunks: m = 8 -> lcm(16, 4R) segments
// (CPT = 4 / gcd(4, R); a chunk may straddle tiles, so the selector follows the tile), m >= 32
// -> one chunk.
struct TrShape {
    uint32_t K;      // tiles per item
    uint32_t CPT;    // chunks per item
};

// Chunk results leave the MMA accumulators through a per-warp staging area instead of
// warp shuffles: each lane stores its binary16-rounded partials (row = chunk, column = j), and
// once a batch of chunks is staged each lane sums ONE chunk's row in ascending j (fragment.hpp:
// 89-92).  Row strides (12 floats for m = 8, m + 4 otherwise) keep the 128-bit row reads
// conflict free.
template <int MM>
struct TrStage {
    static constexpr uint32_t SW = MM == 8 ? 12u : uint32_t(MM) + 4u;           // row stride
    static constexpr uint32_t ROWS = MM == 8 ? 32u : (1024u / MM < 32u ? 1024u / MM : 32u);
    static constexpr uint32_t FLOATS = ROWS * SW;                                 // per warp
};

template <int MM, int SI, int KC, bool REPAIR>   // MM = 8, 32, 64, 128
__global__ void __launch_bounds__(kGmThreads) gm_tr_kernel(const SpParams p, const TrShape S) {
    pdl_release();
    // stages of T tiles: m >= 32 items are K = R (m/16)^2 (a multiple of 4) contiguous tiles, so a
    // 2 KiB stage of 4 tiles stays inside one item (one issue / wait / sync per 4 tiles); m = 8
    // with one-tile items (K = 1: R = 1, 2, 4) is dealt to the warps in runs of SI = 4 adjacent
    // items, a stage = one run (SI = 1: items dealt one by one, one tile per stage).  KC > 1:
    // m = 8 items of exactly KC tiles (R = 3, 5, 7, 8, ...), one whole item per stage, the
    // straddling selectors precomputed per tile.
    static_assert(SI == 1 || MM == 8, "item runs only for one-tile items");
    static_assert(KC == 1 || (MM == 8 && SI == 1), "whole-item stages only for m = 8");
    constexpr uint32_t T = MM >= 32 ? 4u : (SI > 1 ? uint32_t(SI) : uint32_t(KC));
    constexpr int D = kGmTrDepth / int(T);
    constexpr uint32_t SG = MM >= 32 ? MM / 16 : 1;    // column groups per chunk (m >= 32)
    using ST = TrStage<MM>;
    extern __shared__ __align__(128) unsigned char s_ring[];   // [kGmWarps][D][512], staging, tables
    __shared__ float s_scratch[32];
    __shared__ int s_last;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t ring = smem_u32(s_ring) + warp * kGmTrDepth * 512u;
    float* s_stage = reinterpret_cast<float*>(s_ring + kGmWarps * kGmTrDepth * 512) + warp * ST::FLOATS;
    float* s_chunk = reinterpret_cast<float*>(s_ring + kGmWarps * kGmTrDepth * 512) + kGmWarps * ST::FLOATS;
    const uint32_t Cg = p.G * p.W;
    float* s_block = s_chunk + Cg;
    const uint32_t items = Cg / S.CPT;
    const uint32_t R = p.R;
    // staged rows per batch: chunks (m = 8: CPT per item) or items (m >= 32, one chunk each)
    const uint32_t batch_items = MM == 8 ? 32u / S.CPT : ST::ROWS;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    // selector rows kappa in {2c, 2c+1, 2c+8, 2c+9} of tile kt of the item, column n = g
    auto bsel = [&](uint32_t kt, uint32_t k) -> bool {
        if (MM >= 32) return (k % SG) == g;
        if (S.CPT > 1) return ((16u * kt + k) / (4u * R)) == g;   // m = 8: chunk slot of segment
        return g == 0;
    };
    uint32_t b0 = sel2(bsel(0, 2 * c), bsel(0, 2 * c + 1)), b1 = sel2(bsel(0, 2 * c + 8), bsel(0, 2 * c + 9));
    const bool straddle = MM == 8 && S.CPT > 1 && S.K > 1;      // m = 8, R odd or R = 2 mod 4
    uint32_t bk0[KC], bk1[KC];                                   // KC > 1: selectors of tile t
#pragma unroll
    for (int kt = 0; kt < KC; ++kt) {
        bk0[kt] = sel2(bsel(kt, 2 * c), bsel(kt, 2 * c + 1));
        bk1[kt] = sel2(bsel(kt, 2 * c + 8), bsel(kt, 2 * c + 9));
    }
    // swizzled 16-byte lines (conflict-free transposing ldmatrix), as in tcr_sp_async.cu
    auto swz = [](uint32_t k, uint32_t h) { return 32u * k + 16u * (h ^ ((k >> 2) & 1u)); };
    const uint32_t cp_dst = swz(lane >> 1, lane & 1u);
    const uint32_t mi = lane >> 3;
    const uint32_t ld_off = swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);
    bool ovf = false;

    for (uint64_t gi = p.group_begin + blockIdx.x; gi < p.group_end; gi += gridDim.x) {
        const uint64_t tile0 = gi * uint64_t(items) * S.K;          // first tile of the group
        const uint64_t gend = (tile0 + uint64_t(items) * S.K) * 256u;
        const uint64_t glim = gend < p.n ? gend : p.n;
        const bool full = gend <= p.n && items % uint32_t(SI) == 0;
        const uint32_t runs = (items + SI - 1) / SI;
        const uint32_t my_runs = runs > warp ? (runs - warp + kGmWarps - 1) / kGmWarps : 0;
        const uint32_t my_items = my_runs * SI;
        uint32_t iit = 0, ik = 0, islot = 0;                          // issue cursor
        auto issue = [&]() {
            if (iit < my_runs) {
                const uint64_t e0 = (tile0 + uint64_t(warp + iit * kGmWarps) * SI * S.K + ik) * 256u + 8u * lane;
                const uint32_t dst = ring + islot * (512u * T) + cp_dst;
                if (full) {
#pragma unroll
                    for (uint32_t t = 0; t < T; ++t) cp16(dst + 512u * t, x + e0 + 256u * t, 16u);
                } else {
#pragma unroll
                    for (uint32_t t = 0; t < T; ++t) {
                        const uint64_t e = e0 + 256u * t;
                        const uint32_t bytes = e + 8 <= glim ? 16u : (e < glim ? uint32_t(glim - e) * 2u : 0u);
                        cp16(dst + 512u * t, x + (e < glim ? e : 0), bytes);
                    }
                }
                if (SI > 1 || (ik += T) == S.K) {
                    ik = 0;
                    ++iit;
                }
            }
            cp_commit();
            islot = islot + 1 == uint32_t(D) ? 0 : islot + 1;
        };
        // finish a staged batch of `nb` items starting at item-of-warp index it0
        auto flush = [&](uint32_t it0, uint32_t nb) {
            __syncwarp();
            const uint32_t rows = MM == 8 ? nb * S.CPT : nb;
            if (lane < rows) {
                const float* row = s_stage + lane * ST::SW;
                float r = 0.0f;
#pragma unroll
                for (uint32_t j = 0; j < (MM == 8 ? 8u : uint32_t(MM)); j += 4) {
                    const float4 v = *reinterpret_cast<const float4*>(row + j);
                    r = r + v.x; r = r + v.y; r = r + v.z; r = r + v.w;
                }
                r = r + 0.0f;
                ovf |= !isfinite(r);
                const uint32_t b = MM == 8 ? lane / S.CPT : lane;
                const uint32_t wi = it0 + b;                            // item of this warp
                const uint32_t item = SI == 1 ? warp + wi * kGmWarps : (warp + wi / SI * kGmWarps) * SI + wi % SI;
                const uint32_t ch = MM == 8 ? item * S.CPT + lane % S.CPT : item;
                if (SI == 1 || ch < Cg) s_chunk[ch] = r;
            }
            __syncwarp();
        };
#pragma unroll 1
        for (int f = 0; f < D - 1; ++f) issue();
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t ck = 0, it = 0, cslot = 0, nb = 0;
        while (it < my_items) {
            issue();
            cp_wait<D - 1>();
            __syncwarp();
            if constexpr (SI > 1) {
                // a run of SI one-tile items: each tile completes an item
#pragma unroll
                for (uint32_t t = 0; t < T; ++t) {
                    uint32_t d0, d1, d2, d3;
                    ldsm4t(ring + cslot * (512u * T) + 512u * t + ld_off, d0, d1, d2, d3);
                    float a4[4] = {0.f, 0.f, 0.f, 0.f};
                    mma_16816(a4, d0, d1, d2, d3, b0, b1);
                    const uint32_t r0 = nb * S.CPT;
                    if (2 * c < S.CPT) s_stage[(r0 + 2 * c) * ST::SW + g] = h_round(a4[0] + a4[2]);
                    if (2 * c + 1 < S.CPT) s_stage[(r0 + 2 * c + 1) * ST::SW + g] = h_round(a4[1] + a4[3]);
                    ++it;
                    if (++nb == batch_items) {
                        flush(it - nb, nb);
                        nb = 0;
                    }
                }
                __syncwarp();
                cslot = cslot + 1 == uint32_t(D) ? 0 : cslot + 1;
            } else {
#pragma unroll
                for (uint32_t t = 0; t < T; ++t) {
                    uint32_t d0, d1, d2, d3;
                    ldsm4t(ring + cslot * (512u * T) + 512u * t + ld_off, d0, d1, d2, d3);
                    if (KC > 1) {
                        b0 = bk0[t % KC];
                        b1 = bk1[t % KC];
                    } else if (straddle) {
                        b0 = sel2(bsel(ck + t, 2 * c), bsel(ck + t, 2 * c + 1));
                        b1 = sel2(bsel(ck + t, 2 * c + 8), bsel(ck + t, 2 * c + 9));
                    }
                    mma_16816(acc, d0, d1, d2, d3, b0, b1);
                }
                __syncwarp();
                cslot = cslot + 1 == uint32_t(D) ? 0 : cslot + 1;
                if ((ck += T) < S.K) continue;
                ck = 0;
                // ---- item complete: acc = (j16 = g, n = 2c), (g, 2c+1), (g+8, 2c), (g+8, 2c+1)
                if (MM == 8) {
                    // partial(chunk slot n, j8 = g) = D[g][n] + D[g+8][n]  -> staged row (nb CPT + n)
                    const uint32_t r0 = nb * S.CPT;
                    if (2 * c < S.CPT) s_stage[(r0 + 2 * c) * ST::SW + g] = h_round(acc[0] + acc[2]);
                    if (2 * c + 1 < S.CPT) s_stage[(r0 + 2 * c + 1) * ST::SW + g] = h_round(acc[1] + acc[3]);
                } else {
                    // partial(j = 16 n + j16) = D[j16][n]
                    float* row = s_stage + nb * ST::SW;
                    if (2 * c < SG) {
                        row[16 * (2 * c) + g] = h_round(acc[0]);
                        row[16 * (2 * c) + g + 8] = h_round(acc[2]);
                    }
                    if (2 * c + 1 < SG) {
                        row[16 * (2 * c + 1) + g] = h_round(acc[1]);
                        row[16 * (2 * c + 1) + g + 8] = h_round(acc[3]);
                    }
                }
                acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
                ++it;
                if (++nb == batch_items) {
                    flush(it - nb, nb);
                    nb = 0;
                }
            }
        }
        if (nb) flush(it - nb, nb);
        cp_wait<0>();
        group_epilogue<REPAIR>(p, gi, s_chunk, s_block, MM, ovf);
    }
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kGmThreads);
}

// =============================================================== wide fragments, m >= 256
// A chunk (R fragments of m x m) is streamed in column SLABS of 256 columns: for slab s, the R*m
// rows of the chunk contribute one 256-element tile each (elements [256 s, 256 s + 256) of the
// row, 512 contiguous bytes).  A tile's 16 segments are 16 different column groups, so two
// HMMA.16816 per tile with identity selectors (B_lo[k][n] = [k == n], B_hi[k][n] = [k == n + 8])
// accumulate the slab's 256 column sums over the chain of rows in D_lo / D_hi; at the end of a
// slab the partials are rounded to binary16 (reduction.hpp:179-181) and added to the running
// ascending-j finishing sum (:182, fragment.hpp:89-92), carried across the m / 256 slabs.
template <bool REPAIR>
__global__ void __launch_bounds__(kGmThreads) gm_wide_kernel(const SpParams p, const uint32_t m) {
    pdl_release();
    // 2 KiB stages: tiles of 4 consecutive rows of one slab (R m rows, a multiple of 4)
    constexpr uint32_t T = 4;
    constexpr int D = kGmTrDepth / int(T);
    extern __shared__ __align__(128) unsigned char s_ring[];   // [kGmWarps][D][512] + tables
    __shared__ float s_scratch[32];
    __shared__ int s_last;
    float* s_chunk = reinterpret_cast<float*>(s_ring + kGmWarps * kGmTrDepth * 512);
    float* s_block = s_chunk + p.G * p.W;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t ring = smem_u32(s_ring) + warp * kGmTrDepth * 512u;
    const uint32_t Cg = p.G * p.W;
    const uint32_t rows = p.R * m;                  // rows of a chunk (R fragments)
    const uint32_t slabs = m / 256u;
    const uint64_t chunk_el = uint64_t(rows) * m;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    const uint32_t blo0 = sel2(2 * c == g, 2 * c + 1 == g), blo1 = sel2(2 * c + 8 == g, 2 * c + 9 == g);
    const uint32_t bhi0 = sel2(2 * c == g + 8, 2 * c + 1 == g + 8), bhi1 = sel2(2 * c + 8 == g + 8, 2 * c + 9 == g + 8);
    auto swz = [](uint32_t k, uint32_t h) { return 32u * k + 16u * (h ^ ((k >> 2) & 1u)); };
    const uint32_t cp_dst = swz(lane >> 1, lane & 1u);
    const uint32_t mi = lane >> 3;
    const uint32_t ld_off = swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);
    bool ovf = false;

    // stream cursor: item (chunk of this warp), slab, row
    struct Cur {
        uint32_t it, s, i;
    };
    auto advance = [&](Cur& q) {
        if ((q.i += T) == rows) {
            q.i = 0;
            if (++q.s == slabs) {
                q.s = 0;
                ++q.it;
            }
        }
    };
    for (uint64_t gi = p.group_begin + blockIdx.x; gi < p.group_end; gi += gridDim.x) {
        const uint64_t gel0 = gi * uint64_t(Cg) * chunk_el;
        const uint32_t my_items = Cg > warp ? (Cg - warp + kGmWarps - 1) / kGmWarps : 0;
        Cur iq{0, 0, 0}, cq{0, 0, 0};
        uint32_t slot_i = 0, slot_c = 0;
        auto issue = [&]() {
            if (iq.it < my_items) {
                const uint64_t e0 = gel0 + uint64_t(warp + iq.it * kGmWarps) * chunk_el + uint64_t(iq.i) * m +
                                    256u * iq.s + 8u * lane;
#pragma unroll
                for (uint32_t q = 0; q < T; ++q) {
                    const uint64_t e = e0 + uint64_t(q) * m;
                    const uint32_t bytes = e + 8 <= p.n ? 16u : (e < p.n ? uint32_t(p.n - e) * 2u : 0u);
                    cp16(ring + slot_i * (512u * T) + 512u * q + cp_dst, x + (e < p.n ? e : 0), bytes);
                }
                advance(iq);
            }
            cp_commit();
            slot_i = slot_i + 1 == D ? 0 : slot_i + 1;
        };
#pragma unroll 1
        for (int f = 0; f < D - 1; ++f) issue();
        float lo[4] = {0.f, 0.f, 0.f, 0.f}, hi[4] = {0.f, 0.f, 0.f, 0.f};
        float r = 0.0f;
        while (cq.it < my_items) {
            issue();
            cp_wait<D - 1>();
            __syncwarp();
#pragma unroll
            for (uint32_t q = 0; q < T; ++q) {
                uint32_t d0, d1, d2, d3;
                ldsm4t(ring + slot_c * (512u * T) + 512u * q + ld_off, d0, d1, d2, d3);
                mma_16816(lo, d0, d1, d2, d3, blo0, blo1);
                mma_16816(hi, d0, d1, d2, d3, bhi0, bhi1);
            }
            __syncwarp();
            slot_c = slot_c + 1 == D ? 0 : slot_c + 1;
            const Cur done = cq;
            advance(cq);
            if (done.i + T < rows) continue;
            // ---- slab complete: D[j16][n] = partial of column 256 s + 16 n + j16 (n < 8 in lo)
            const float hl[4] = {h_round(lo[0]), h_round(lo[1]), h_round(lo[2]), h_round(lo[3])};
            const float hh[4] = {h_round(hi[0]), h_round(hi[1]), h_round(hi[2]), h_round(hi[3])};
#pragma unroll
            for (uint32_t j = 0; j < 256u; ++j) {   // ascending j = 16 n + j16
                const uint32_t n = (j >> 4) & 7u, j16 = j & 15u;
                const uint32_t reg = 2u * (j16 >> 3) + (n & 1u);
                const float v = j < 128u ? hl[reg] : hh[reg];
                r = r + __shfl_sync(kFull, v, 4 * (j16 & 7u) + (n >> 1));
            }
            lo[0] = lo[1] = lo[2] = lo[3] = 0.f;
            hi[0] = hi[1] = hi[2] = hi[3] = 0.f;
            if (done.s + 1 < slabs) continue;
            r = r + 0.0f;
            ovf |= !isfinite(r);
            if (lane == 0) s_chunk[warp + done.it * kGmWarps] = r;
            r = 0.0f;
        }
        cp_wait<0>();
        group_epilogue<REPAIR>(p, gi, s_chunk, s_block, m, ovf);
    }
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kGmThreads);
}

// ============================================ wide fragments, m = 256 SL (SL <= 8): CTA per chunk
// The whole CTA reduces one chunk at a time: warp w streams the contiguous rows
// [w R m / 8, (w + 1) R m / 8) of the chunk (each row = SL 512-byte tiles, one HMMA pair per tile
// into the slab's accumulators -- 8 SL registers), so every chunk keeps 8 warps busy and every
// warp reads one contiguous range.  At the chunk end the 8 warp partials of each column are added
// in warp order (fixed), rounded to binary16 (reduction.hpp:179-181) and summed by a fixed
// lane-then-warp tree into the chunk result (the finishing MMA's sum, :182; binary16 partials of
// similar magnitude add exactly in fp32, so the order rarely matters).
template <int SL, bool REPAIR>
__global__ void __launch_bounds__(kGmThreads) gm_wide_cta_kernel(const SpParams p, const uint32_t m) {
    pdl_release();
    // 2 KiB stages of 4 consecutive tiles of the warp's stream (rows / 8 * SL tiles per chunk,
    // a multiple of 4): one issue / wait / sync per 4 tiles
    constexpr uint32_t T = 4;
    constexpr int D = kGmTrDepth / int(T);
    constexpr uint32_t QS = SL > 4 ? uint32_t(SL) : 4u;         // tiles per consumer iteration
    extern __shared__ __align__(128) unsigned char s_ring[];   // ring | part[8][m] | tables
    __shared__ float s_scratch[32];
    __shared__ float s_wsum[kGmWarps];
    __shared__ int s_last;
    float* s_part = reinterpret_cast<float*>(s_ring + kGmWarps * kGmTrDepth * 512);
    float* s_chunk = s_part + kGmWarps * m;
    const uint32_t Cg = p.G * p.W;
    float* s_block = s_chunk + Cg;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t ring = smem_u32(s_ring) + warp * kGmTrDepth * 512u;
    const uint64_t rows = uint64_t(p.R) * m;
    const uint64_t chunk_el = rows * m;
    const uint64_t span = rows / kGmWarps * m;                  // elements of this warp per chunk
    const uint64_t w_off = uint64_t(warp) * span;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    const uint32_t blo0 = sel2(2 * c == g, 2 * c + 1 == g), blo1 = sel2(2 * c + 8 == g, 2 * c + 9 == g);
    const uint32_t bhi0 = sel2(2 * c == g + 8, 2 * c + 1 == g + 8), bhi1 = sel2(2 * c + 8 == g + 8, 2 * c + 9 == g + 8);
    auto swz = [](uint32_t k, uint32_t h) { return 32u * k + 16u * (h ^ ((k >> 2) & 1u)); };
    const uint32_t cp_dst = swz(lane >> 1, lane & 1u);
    const uint32_t mi = lane >> 3;
    const uint32_t ld_off = swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);
    bool ovf = false;

    for (uint64_t gi = p.group_begin + blockIdx.x; gi < p.group_end; gi += gridDim.x) {
        const uint64_t gel0 = gi * uint64_t(Cg) * chunk_el;
        uint32_t iit = 0, islot = 0;
        uint64_t ioff = 0;                                         // issue cursor (chunk, offset)
        auto issue = [&]() {
            if (iit < Cg) {
                const uint64_t e0 = gel0 + uint64_t(iit) * chunk_el + w_off + ioff + 8u * lane;
                const uint32_t dst = ring + islot * (512u * T) + cp_dst;
                if (e0 + 256u * T <= p.n) {
#pragma unroll
                    for (uint32_t q = 0; q < T; ++q) cp16(dst + 512u * q, x + e0 + 256u * q, 16u);
                } else {
#pragma unroll
                    for (uint32_t q = 0; q < T; ++q) {
                        const uint64_t e = e0 + 256u * q;
                        const uint32_t bytes = e + 8 <= p.n ? 16u : (e < p.n ? uint32_t(p.n - e) * 2u : 0u);
                        cp16(dst + 512u * q, x + (e < p.n ? e : 0), bytes);
                    }
                }
                ioff += 256u * T;
                if (ioff == span) {
                    ioff = 0;
                    ++iit;
                }
            }
            cp_commit();
            islot = islot + 1 == uint32_t(D) ? 0 : islot + 1;
        };
#pragma unroll 1
        for (int f = 0; f < D - 1; ++f) issue();
        uint32_t cslot = 0;
        for (uint32_t it = 0; it < Cg; ++it) {
            float acc[SL][2][4];
#pragma unroll
            for (int sl = 0; sl < SL; ++sl)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[sl][0][q] = acc[sl][1][q] = 0.f;
            for (uint64_t q0 = 0; q0 < rows / kGmWarps * SL; q0 += QS) {
#pragma unroll
                for (uint32_t h = 0; h < QS / T; ++h) {
                    issue();
                    cp_wait<D - 1>();
                    __syncwarp();
#pragma unroll
                    for (uint32_t q = 0; q < T; ++q) {
                        const int sl = int((h * T + q) % uint32_t(SL));   // tile (row, slab) order
                        uint32_t d0, d1, d2, d3;
                        ldsm4t(ring + cslot * (512u * T) + 512u * q + ld_off, d0, d1, d2, d3);
                        mma_16816(acc[sl][0], d0, d1, d2, d3, blo0, blo1);
                        mma_16816(acc[sl][1], d0, d1, d2, d3, bhi0, bhi1);
                    }
                    __syncwarp();
                    cslot = cslot + 1 == uint32_t(D) ? 0 : cslot + 1;
                }
            }
            // warp partials: D[j16][n] = column 256 sl + 16 n + j16 (n + 8 for the hi half)
            float* part = s_part + warp * m;
#pragma unroll
            for (int sl = 0; sl < SL; ++sl)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint32_t col0 = 256u * sl + 128u * hh;
                    part[col0 + 16 * (2 * c) + g] = acc[sl][hh][0];
                    part[col0 + 16 * (2 * c + 1) + g] = acc[sl][hh][1];
                    part[col0 + 16 * (2 * c) + g + 8] = acc[sl][hh][2];
                    part[col0 + 16 * (2 * c + 1) + g + 8] = acc[sl][hh][3];
                }
            __syncthreads();
            float t = 0.0f;
            for (uint32_t col = threadIdx.x; col < m; col += kGmThreads) {
                float cs = 0.0f;
#pragma unroll
                for (int w = 0; w < kGmWarps; ++w) cs = cs + s_part[w * m + col];
                t = t + h_round(cs);
            }
            t = warp_tree_xor(t);
            if (lane == 0) s_wsum[warp] = t;
            __syncthreads();
            if (threadIdx.x == 0) {
                float r = 0.0f;
#pragma unroll
                for (int w = 0; w < kGmWarps; ++w) r = r + s_wsum[w];
                r = r + 0.0f;
                ovf |= !isfinite(r);
                s_chunk[it] = r;
            }
        }
        cp_wait<0>();
        group_epilogue<REPAIR>(p, gi, s_chunk, s_block, m, ovf);
    }
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kGmThreads);
}

// ======================================= wide fragments, m >= 1024: a CLUSTER of CS CTAs per chunk
// As gm_wide_cta_kernel, but the chunk's rows are split over the CS CTAs of a thread-block
// cluster (CS x 8 warps, each a contiguous row range): every CTA adds its 8 warp partials per
// column, and the cluster's rank 0 adds the CS CTA column sums in rank order through distributed
// shared memory (cluster.map_shared_rank), then rounds and sums as before.  2^28 elements are
// only 256 chunks at m = 1024: one CTA per chunk left most SMs idle.
template <int SL, bool REPAIR>
__global__ void __launch_bounds__(kGmThreads) gm_wide_cluster_kernel(const SpParams p, const uint32_t m) {
    pdl_release();
    constexpr uint32_t T = 4;                                    // tiles per stage (as gm_wide_cta_kernel)
    constexpr int D = kGmTrDepth / int(T);
    constexpr uint32_t QS = SL > 4 ? uint32_t(SL) : 4u;
    extern __shared__ __align__(128) unsigned char s_ring[];   // ring | part[8][m] | cta[m] | tables
    __shared__ float s_scratch[32];
    __shared__ float s_wsum[kGmWarps];
    __shared__ int s_last;
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t CS = cluster.num_blocks();
    const uint32_t rank = cluster.block_rank();
    const uint64_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
    float* s_part = reinterpret_cast<float*>(s_ring + kGmWarps * kGmTrDepth * 512);
    float* s_cta = s_part + kGmWarps * m;                       // this CTA's column sums
    float* s_chunk = s_cta + m;
    const uint32_t Cg = p.G * p.W;
    float* s_block = s_chunk + Cg;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t ring = smem_u32(s_ring) + warp * kGmTrDepth * 512u;
    const uint64_t rows = uint64_t(p.R) * m;
    const uint64_t chunk_el = rows * m;
    const uint64_t rpw = rows / (uint64_t(kGmWarps) * CS);     // rows of this warp per chunk
    const uint64_t span = rpw * m;
    const uint64_t w_off = (uint64_t(rank) * kGmWarps + warp) * span;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    const uint32_t blo0 = sel2(2 * c == g, 2 * c + 1 == g), blo1 = sel2(2 * c + 8 == g, 2 * c + 9 == g);
    const uint32_t bhi0 = sel2(2 * c == g + 8, 2 * c + 1 == g + 8), bhi1 = sel2(2 * c + 8 == g + 8, 2 * c + 9 == g + 8);
    auto swz = [](uint32_t k, uint32_t h) { return 32u * k + 16u * (h ^ ((k >> 2) & 1u)); };
    const uint32_t cp_dst = swz(lane >> 1, lane & 1u);
    const uint32_t mi = lane >> 3;
    const uint32_t ld_off = swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);
    bool ovf = false;

    for (uint64_t gi = p.group_begin + cid; gi < p.group_end; gi += ncl) {
        const uint64_t gel0 = gi * uint64_t(Cg) * chunk_el;
        uint32_t iit = 0, islot = 0;
        uint64_t ioff = 0;                                         // issue cursor (chunk, offset)
        auto issue = [&]() {
            if (iit < Cg) {
                const uint64_t e0 = gel0 + uint64_t(iit) * chunk_el + w_off + ioff + 8u * lane;
                const uint32_t dst = ring + islot * (512u * T) + cp_dst;
                if (e0 + 256u * T <= p.n) {
#pragma unroll
                    for (uint32_t q = 0; q < T; ++q) cp16(dst + 512u * q, x + e0 + 256u * q, 16u);
                } else {
#pragma unroll
                    for (uint32_t q = 0; q < T; ++q) {
                        const uint64_t e = e0 + 256u * q;
                        const uint32_t bytes = e + 8 <= p.n ? 16u : (e < p.n ? uint32_t(p.n - e) * 2u : 0u);
                        cp16(dst + 512u * q, x + (e < p.n ? e : 0), bytes);
                    }
                }
                ioff += 256u * T;
                if (ioff == span) {
                    ioff = 0;
                    ++iit;
                }
            }
            cp_commit();
            islot = islot + 1 == uint32_t(D) ? 0 : islot + 1;
        };
#pragma unroll 1
        for (int f = 0; f < D - 1; ++f) issue();
        uint32_t cslot = 0;
        for (uint32_t it = 0; it < Cg; ++it) {
            float acc[SL][2][4];
#pragma unroll
            for (int sl = 0; sl < SL; ++sl)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[sl][0][q] = acc[sl][1][q] = 0.f;
            for (uint64_t q0 = 0; q0 < rpw * SL; q0 += QS) {
#pragma unroll
                for (uint32_t h = 0; h < QS / T; ++h) {
                    issue();
                    cp_wait<D - 1>();
                    __syncwarp();
#pragma unroll
                    for (uint32_t q = 0; q < T; ++q) {
                        const int sl = int((h * T + q) % uint32_t(SL));   // tile (row, slab) order
                        uint32_t d0, d1, d2, d3;
                        ldsm4t(ring + cslot * (512u * T) + 512u * q + ld_off, d0, d1, d2, d3);
                        mma_16816(acc[sl][0], d0, d1, d2, d3, blo0, blo1);
                        mma_16816(acc[sl][1], d0, d1, d2, d3, bhi0, bhi1);
                    }
                    __syncwarp();
                    cslot = cslot + 1 == uint32_t(D) ? 0 : cslot + 1;
                }
            }
            // warp partials: D[j16][n] = column 256 sl + 16 n + j16 (n + 8 for the hi half)
            float* part = s_part + warp * m;
#pragma unroll
            for (int sl = 0; sl < SL; ++sl)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint32_t col0 = 256u * sl + 128u * hh;
                    part[col0 + 16 * (2 * c) + g] = acc[sl][hh][0];
                    part[col0 + 16 * (2 * c + 1) + g] = acc[sl][hh][1];
                    part[col0 + 16 * (2 * c) + g + 8] = acc[sl][hh][2];
                    part[col0 + 16 * (2 * c + 1) + g + 8] = acc[sl][hh][3];
                }
            __syncthreads();
            // this CTA's column sums (8 warp partials in warp order) -> s_cta, visible cluster-wide
            for (uint32_t col = threadIdx.x; col < m; col += kGmThreads) {
                float cs = 0.0f;
#pragma unroll
                for (int w = 0; w < kGmWarps; ++w) cs = cs + s_part[w * m + col];
                s_cta[col] = cs;
            }
            cluster.sync();
            if (rank == 0) {
                // the cluster's CTAs in rank order through distributed shared memory
                float t = 0.0f;
                for (uint32_t col = threadIdx.x; col < m; col += kGmThreads) {
                    float cs = 0.0f;
                    for (uint32_t q = 0; q < CS; ++q) cs = cs + cluster.map_shared_rank(s_cta, q)[col];
                    t = t + h_round(cs);
                }
                t = warp_tree_xor(t);
                if (lane == 0) s_wsum[warp] = t;
                __syncthreads();
                if (threadIdx.x == 0) {
                    float r = 0.0f;
#pragma unroll
                    for (int w = 0; w < kGmWarps; ++w) r = r + s_wsum[w];
                    r = r + 0.0f;
                    ovf |= !isfinite(r);
                    s_chunk[it] = r;
                }
            }
            cluster.sync();                     // s_cta is reused by the next chunk
        }
        cp_wait<0>();
        if (rank == 0) group_epilogue<REPAIR>(p, gi, s_chunk, s_block, m, ovf);
    }
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kGmThreads);
}


uint32_t gcd32(uint32_t a, uint32_t b) {
    while (b) {
        const uint32_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

bool nat_shape(uint32_t m, uint32_t R, uint32_t Cg, NatShape* S) {
    const uint64_t ce = uint64_t(R) * m * m;             // chunk elements (m in {2, 4}: 4R or 16R)
    if (ce > 0xFFFFFFFFull / 32) return false;
    // period = lcm(16, ce) elements
    const uint64_t g16 = gcd32(16, uint32_t(ce % 16));  // gcd(16, ce)
    const uint64_t period = ce / g16 * 16;
    S->PR = uint32_t(period / 16);
    S->CP = uint32_t(period / ce);
    if (S->CP * m > 8) return false;                     // N = 8 selector columns
    S->RB = S->PR < 16 ? S->PR : 16;                    // rows per stage (any count <= 16)
    S->chunks_per_unit = 16 * S->CP;
    if (Cg % S->CP) return false;                        // groups start on a period
    return true;
}

bool tr_shape(uint32_t m, uint32_t R, uint32_t Cg, TrShape* S) {
    if (m == 8) {
        // chunk = 4R segments; item = lcm(16, 4R) segments = K tiles holding CPT (<= 4) chunks
        const uint64_t cs = 4ull * R;
        const uint64_t item = cs / gcd32(16, uint32_t(cs % 16)) * 16;
        if (item / 16 > 0xFFFFFFFFull) return false;
        S->K = uint32_t(item / 16);
        S->CPT = uint32_t(item / cs);
    } else if (m == 32 || m == 64 || m == 128) {
        S->K = R * (m / 16) * (m / 16);
        S->CPT = 1;
    } else {
        return false;
    }
    return Cg % S->CPT == 0;
}

}  // namespace

bool wide_ok(const SpGeometry& g) {
    // m >= 256: rows = R m and the per-chunk cursor fit 32 bits
    return g.m >= 256 && uint64_t(g.R) * g.m < (1ull << 31) && g.G * g.W <= uint32_t(kMaxChunksGenm);
}

bool genm_supported(const SpGeometry& g) {
    const uint32_t Cg = g.G * g.W;
    if (g.m >= 256) return wide_ok(g);
    if (g.m == 2 || g.m == 4) {
        NatShape S;
        return nat_shape(g.m, g.R, Cg, &S);
    }
    TrShape S;
    return tr_shape(g.m, g.R, Cg, &S);
}

namespace {
template <typename K, typename S>
cudaError_t launch_gm(K fn, uint32_t dyn, uint64_t groups, const SpParams& p, const S& shape, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGmThreads, dyn);
    if (per_sm < 1) per_sm = 1;
    const int grid = int(groups < uint64_t(per_sm) * sm_count() ? groups : uint64_t(per_sm) * sm_count());
    fn<<<grid, kGmThreads, dyn, s>>>(p, shape);
    return cudaGetLastError();
}

// Engines with a flag instead of a shape argument (gm4_reg_kernel)
cudaError_t launch_gm(void (*fn)(SpParams, bool), uint32_t dyn, uint64_t groups, const SpParams& p, bool flag,
                      cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGmThreads, dyn);
    if (per_sm < 1) per_sm = 1;
    const int grid = int(groups < uint64_t(per_sm) * sm_count() ? groups : uint64_t(per_sm) * sm_count());
    fn<<<grid, kGmThreads, dyn, s>>>(p, flag);
    return cudaGetLastError();
}

// Thread-block-cluster launch (CS CTAs per cluster, one group of chunks per cluster at a time).
template <typename K>
cudaError_t launch_cluster(K fn, uint32_t dyn, uint64_t groups, uint32_t CS, const SpParams& p, uint32_t m,
                           cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kGmThreads, 1, 1);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(CS, 1, 1);
    int max_clusters = 0;
    e = cudaOccupancyMaxActiveClusters(&max_clusters, fn, &cfg);
    if (e != cudaSuccess) return e;
    if (max_clusters < 1) max_clusters = 1;
    const uint64_t ncl = groups < uint64_t(max_clusters) ? groups : uint64_t(max_clusters);
    cfg.gridDim = dim3(unsigned(ncl * CS), 1, 1);
    e = cudaLaunchKernelEx(&cfg, fn, p, m);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}
}  // namespace

template <bool REPAIR>
cudaError_t launch_genm_t(const SpParams& p, const SpGeometry& g, cudaStream_t s) {
    const uint32_t Cg = g.G * g.W;
    const uint64_t groups = p.group_end - p.group_begin;
    const uint32_t tables = (Cg + g.G + 3u) / 4u * 16u;   // chunk results [Cg] + block results [G]
    if (g.m == 2 || g.m == 4) {
        NatShape S;
        if (!nat_shape(g.m, g.R, Cg, &S)) return cudaErrorInvalidValue;
        // PR <= 8 or 16: a unit of 16 periods is one contiguous stage of 512 PR bytes
        const bool fast = S.PR == S.RB && (S.PR <= 8 || S.PR == 16) && !knobs().gm_nat_generic;
        if (!REPAIR && g.R <= 2 && gm4_reg_ok(g.m, g.R, g.W, Cg, knobs().gm_nat_alt == 10) && knobs().gm_nat_alt != 8) {
            // m = 4, R = 1: register-direct stream (knob values: 8 the ring kernels, 9 with the
            // L2 prefetch; A/B)
            const bool pf = knobs().gm_nat_alt == 9;
            if (g.R == 2) {
                if (g.W == 1) return launch_gm(gm4_reg_kernel<false, 1, 2>, 16u, groups, p, pf, s);
                return launch_gm(gm4_reg_kernel<false, 0, 2>, tables * 1u, groups, p, pf, s);
            }
            if (g.R == 4) {
                if (g.W == 1) return launch_gm(gm4_reg_kernel<false, 1, 4>, 16u, groups, p, pf, s);
                return launch_gm(gm4_reg_kernel<false, 0, 4>, tables * 1u, groups, p, pf, s);
            }
            if (g.W == 1) return launch_gm(gm4_reg_kernel<false, 1>, 16u, groups, p, pf, s);
            if (g.W == 4 && knobs().gm_nat_alt == 11)   // profiling A/B
                return launch_gm(gm4_reg_kernel<false, 4>, 16u, groups, p, false, s);
            return launch_gm(gm4_reg_kernel<false>, tables * 1u, groups, p, pf, s);
        }
        if (fast && !REPAIR && g.m == 4 && S.RB == 1 && g.W <= 2 && knobs().gm_nat_alt == 0) {
            // m = 4, R = 1, B = 32 / 64: block trees in registers, no chunk table (tables: block
            // results only).  Measured at 2^28: B = 32 4.07 -> 4.89 TB/s, B = 64 4.75 -> 4.79;
            // B = 128 / 256 neutral / -4 % (the shuffle tree costs what the table saved), not used
            void (*fb)(SpParams, NatShape) = nullptr;
            switch (g.W) {
            case 1: fb = gm_nat_fast_kernel<4, 1, 4, 3, false, true, false, 1>; break;
            default: fb = gm_nat_fast_kernel<4, 1, 4, 3, false, true, false, 2>; break;
            }
            return launch_gm(fb, kGmWarps * 3u * (512u * 4u) + (g.G + 3u) / 4u * 16u, groups, p, S, s);
        }
        if (fast) {
            const int a = knobs().gm_nat_alt;                           // knob: ring shape A/B (7: no register block trees)
            void (*ff)(SpParams, NatShape) = nullptr;
            uint32_t stage = 0, nd = 0;
            // (units per stage, stages): 2 KiB stages; one-row periods 3 stages -> 3 CTAs per SM
            // (+7..38 % over 4 stages / 2 CTAs, A/B on m = 2, 4).  Cross-group prefetch (XG) for
            // one-row periods (m = 2 R = 1: +9 %), per-group pipelines for 2- and 4-row periods
            // (+1..3 %); knob value 3 flips both for A/B.
#define TCR_NATF(MV, RBV, UPSV, NDV) \
    { ff = gm_nat_fast_kernel<MV, RBV, UPSV, NDV, REPAIR>; stage = 512u * RBV * UPSV; nd = NDV; }
#define TCR_NATFX(MV, RBV, UPSV, NDV) \
    { ff = gm_nat_fast_kernel<MV, RBV, UPSV, NDV, REPAIR, false>; stage = 512u * RBV * UPSV; nd = NDV; }
#define TCR_NATF_M(MV)                                                        \
    switch (S.RB) {                                                           \
    case 1:                                                                   \
        if (a == 1) TCR_NATF(MV, 1, 4, 4) else if (a == 2) TCR_NATF(MV, 1, 2, 6) \
        else if (a == 3) TCR_NATFX(MV, 1, 4, 3) else if (a == 4) TCR_NATF(MV, 1, 4, 5) \
        else if (a == 5) TCR_NATF(MV, 1, 2, 8) else if (a == 6) TCR_NATF(MV, 1, 2, 5) \
        else TCR_NATF(MV, 1, 4, 3)   \
        break;                                                                \
    case 2: if (a == 3) TCR_NATF(MV, 2, 2, 4) else TCR_NATFX(MV, 2, 2, 4) break; \
    case 4: if (a == 3) TCR_NATF(MV, 4, 1, 4) else TCR_NATFX(MV, 4, 1, 4) break; \
    case 3: TCR_NATFX(MV, 3, 1, 4) break;                                     \
    case 5: TCR_NATFX(MV, 5, 1, 3) break;                                     \
    case 6: TCR_NATFX(MV, 6, 1, 3) break;                                     \
    case 7: TCR_NATFX(MV, 7, 1, 3) break;                                     \
    case 8: TCR_NATF(MV, 8, 1, 2) break;                                      \
    default: TCR_NATF(MV, 16, 1, 2) break;                                    \
    }
            if (g.m == 2) {
                TCR_NATF_M(2)
            } else {
                TCR_NATF_M(4)
            }
#undef TCR_NATF_M
#undef TCR_NATFX
#undef TCR_NATF
            return launch_gm(ff, kGmWarps * nd * stage + tables, groups, p, S, s);
        }
        // any other period (rows not a power of two, or more than 16): row blocks of <= 16 rows
        void (*fn)(SpParams, NatShape) = g.m == 2 ? gm_nat_kernel<2, REPAIR> : gm_nat_kernel<4, REPAIR>;
        return launch_gm(fn, kGmWarps * 2u * (16u * S.RB * 32u) + tables, groups, p, S, s);
    }
    if (g.m >= 256) {
        if (!wide_ok(g)) return cudaErrorInvalidValue;
        const uint32_t ring = kGmWarps * kGmTrDepth * 512u;
        if (g.m <= 2048 && !knobs().gm_wide_warp) {   // knob: profiling A/B
            const uint32_t dyn = ring + kGmWarps * g.m * 4u + tables;
            switch (g.m) {
            case 256: return launch_gm(gm_wide_cta_kernel<1, REPAIR>, dyn, groups, p, g.m, s);
            case 512: return launch_gm(gm_wide_cta_kernel<2, REPAIR>, dyn, groups, p, g.m, s);
            case 1024:
                if (!knobs().gm_no_cluster)   // knob: profiling A/B
                    return launch_cluster(gm_wide_cluster_kernel<4, REPAIR>, dyn + g.m * 4u, groups, 4, p, g.m, s);
                return launch_gm(gm_wide_cta_kernel<4, REPAIR>, dyn, groups, p, g.m, s);
            default:
                if (!knobs().gm_no_cluster)
                    return launch_cluster(gm_wide_cluster_kernel<8, REPAIR>, dyn + g.m * 4u, groups, 8, p, g.m, s);
                return launch_gm(gm_wide_cta_kernel<8, REPAIR>, dyn, groups, p, g.m, s);
            }
        }
        return launch_gm(gm_wide_kernel<REPAIR>, ring + tables, groups, p, g.m, s);
    }
    TrShape S;
    if (!tr_shape(g.m, g.R, Cg, &S)) return cudaErrorInvalidValue;
    void (*fn)(SpParams, TrShape) = nullptr;
    uint32_t stage = 0;
    switch (g.m) {
    case 8:
        if (knobs().gm_tr8_single) fn = gm_tr_kernel<8, 1, 1, REPAIR>;   // knob: A/B
        else if (S.K == 1) fn = gm_tr_kernel<8, 4, 1, REPAIR>;
        else if (S.K == 2) fn = gm_tr_kernel<8, 1, 2, REPAIR>;
        else if (S.K == 3) fn = gm_tr_kernel<8, 1, 3, REPAIR>;
        else if (S.K == 5) fn = gm_tr_kernel<8, 1, 5, REPAIR>;
        else if (S.K == 7) fn = gm_tr_kernel<8, 1, 7, REPAIR>;
        else fn = gm_tr_kernel<8, 1, 1, REPAIR>;
        stage = TrStage<8>::FLOATS;
        break;
    case 32: fn = gm_tr_kernel<32, 1, 1, REPAIR>; stage = TrStage<32>::FLOATS; break;
    case 64: fn = gm_tr_kernel<64, 1, 1, REPAIR>; stage = TrStage<64>::FLOATS; break;
    case 128: fn = gm_tr_kernel<128, 1, 1, REPAIR>; stage = TrStage<128>::FLOATS; break;
    default: return cudaErrorInvalidValue;
    }
    return launch_gm(fn, kGmWarps * (kGmTrDepth * 512u + stage * 4u) + tables, groups, p, S, s);
}

// fp32 input straight into the natural-layout kernel (m in {2, 4}, periods of <= 8 rows that
// the fast kernel takes): from_single fused into the load.
bool genm_f32_supported(const SpGeometry& g) {
    if (!(g.m == 2 || g.m == 4) || knobs().gm_nat_generic) return false;
    NatShape S;
    if (!nat_shape(g.m, g.R, g.G * g.W, &S)) return false;
    return S.PR == S.RB && S.PR <= 8;
}

template <bool REPAIR>
cudaError_t launch_genm_f32_t(const SpParams& p, const SpGeometry& g, cudaStream_t s) {
    const uint32_t Cg = g.G * g.W;
    const uint64_t groups = p.group_end - p.group_begin;
    const uint32_t tables = (Cg + g.G + 3u) / 4u * 16u;
    NatShape S;
    if (!genm_f32_supported(g) || !nat_shape(g.m, g.R, Cg, &S)) return cudaErrorInvalidValue;
    if (!REPAIR && g.R <= 2 && gm4_reg_ok(g.m, g.R, g.W, Cg, knobs().gm_nat_alt == 10) && knobs().gm_nat_alt != 8) {
        // fp32, m = 4, R = 1: the register-direct engine with from_single in registers
        const bool pf = knobs().gm_nat_alt == 9;
        if (g.R == 2) {
            if (g.W == 1) return launch_gm(gm4_reg_kernel<true, 1, 2>, 16u, groups, p, pf, s);
            return launch_gm(gm4_reg_kernel<true, 0, 2>, tables * 1u, groups, p, pf, s);
        }
        if (g.W == 1) return launch_gm(gm4_reg_kernel<true, 1>, 16u, groups, p, pf, s);
        return launch_gm(gm4_reg_kernel<true>, tables * 1u, groups, p, pf, s);
    }
    if (!REPAIR && g.m == 4 && S.RB == 1 && g.W <= 2 && knobs().gm_nat_alt == 0) {
        // fp32, m = 4, R = 1, B = 32 / 64: register block trees (as the binary16 path)
        void (*fb)(SpParams, NatShape) = nullptr;
        switch (g.W) {
        case 1: fb = gm_nat_fast_kernel<4, 1, 2, 3, false, true, true, 1>; break;
        default: fb = gm_nat_fast_kernel<4, 1, 2, 3, false, true, true, 2>; break;
        }
        return launch_gm(fb, kGmWarps * 3u * (1024u * 2u) + (g.G + 3u) / 4u * 16u, groups, p, S, s);
    }
    void (*ff)(SpParams, NatShape) = nullptr;
    uint32_t stage = 0, nd = 0;
    // 2-4 KiB stages of fp32 (twice the bytes of the binary16 unit)
#define TCR_NATF32(MV, RBV, UPSV, NDV, XGV) \
    { ff = gm_nat_fast_kernel<MV, RBV, UPSV, NDV, REPAIR, XGV, true>; stage = 1024u * RBV * UPSV; nd = NDV; }
#define TCR_NATF32_M(MV)                          \
    switch (S.RB) {                               \
    case 1: TCR_NATF32(MV, 1, 2, 3, true) break;  \
    case 2: TCR_NATF32(MV, 2, 1, 4, false) break; \
    case 3: TCR_NATF32(MV, 3, 1, 3, false) break; \
    case 4: TCR_NATF32(MV, 4, 1, 3, false) break; \
    case 5: TCR_NATF32(MV, 5, 1, 2, false) break; \
    case 6: TCR_NATF32(MV, 6, 1, 2, false) break; \
    case 7: TCR_NATF32(MV, 7, 1, 2, false) break; \
    default: TCR_NATF32(MV, 8, 1, 2, false) break; \
    }
    if (g.m == 2) {
        TCR_NATF32_M(2)
    } else {
        TCR_NATF32_M(4)
    }
#undef TCR_NATF32_M
#undef TCR_NATF32
    return launch_gm(ff, kGmWarps * nd * stage + tables, groups, p, S, s);
}

cudaError_t launch_genm(const SpParams& p, const SpGeometry& g, cudaStream_t s, bool repair, bool f32) {
    if (f32) return repair ? launch_genm_f32_t<true>(p, g, s) : launch_genm_f32_t<false>(p, g, s);
    return repair ? launch_genm_t<true>(p, g, s) : launch_genm_t<false>(p, g, s);
}

}  // namespace tcr
