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
#include <cuda_runtime.h>

#include "tcr_device.cuh"
#include "tcr_kernels.h"
#include "tcr_pipeline.cuh"

namespace tcr {

namespace {

using namespace pipe;

constexpr int kGmWarps = 8;
constexpr int kGmThreads = 32 * kGmWarps;
constexpr int kGmTrDepth = 8;                 // transposed stream: 512-byte tile stages per warp

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

// binary16 0/1 pair
__device__ __forceinline__ uint32_t sel2(bool lo, bool hi) {
    return (lo ? 0x3C00u : 0u) | (hi ? 0x3C000000u : 0u);
}

// Adjacent tree over G (power of two) block results by one warp; any G.
__device__ __forceinline__ void group_tree_any(const SpParams& p, uint64_t gi, const float* blocks) {
    const uint32_t G = p.G;
    const unsigned lane = lane_id();
    if (!p.group_partials) return;
    const uint32_t seg = G >= 32 ? G / 32 : 1;
    float acc = 0.0f;
    if (lane * seg < G) {
        float stk[16];
        int top = 0;
        for (uint32_t i = 0; i < seg; ++i) {
            float v = blocks[lane * seg + i];
            for (uint32_t b = i; b & 1; b >>= 1) v = stk[--top] + v;
            stk[top++] = v;
        }
        acc = stk[0];
    }
    acc = warp_tree_xor(acc);
    if (lane == 0) p.group_partials[gi] = acc;
}

__device__ __forceinline__ void group_epilogue(const SpParams& p, uint64_t gi, float* s_chunk, float* s_block) {
    __syncthreads();
    tile_trees_blocks(p, gi, s_chunk, s_block, threadIdx.x >> 5, kGmWarps);
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) group_tree_any(p, gi, s_block);
    __syncthreads();
}

// ===================================================================== natural layout, m in {2, 4}
// Unit = 16 A-rows.  L >= 1: rows per chunk (unit = 16 chunks); L == 0: CR chunks per row.
struct NatShape {
    uint32_t L, CR, unit_rows, chunks_per_unit;
};

template <int M>
__global__ void __launch_bounds__(kGmThreads) gm_nat_kernel(const SpParams p, const NatShape S) {
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ float s_scratch[32];
    __shared__ int s_last;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t R = p.R;
    const uint32_t unit_bytes = S.unit_rows * 32u;
    float* s_chunk = reinterpret_cast<float*>(dsm + kGmWarps * 2u * unit_bytes);
    float* s_block = s_chunk + kMaxChunksGenm;
    const uint32_t buf0 = smem_u32(dsm) + warp * 2u * unit_bytes;
    const uint64_t chunk_el = uint64_t(R) * M * M;
    const uint32_t Cg = p.G * p.W;
    const uint32_t units = (Cg + S.chunks_per_unit - 1) / S.chunks_per_unit;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    // selector B: thread holds B[2c][g], B[2c+1][g], B[2c+8][g], B[2c+9][g]
    auto bsel = [&](uint32_t k) -> bool {
        if (S.L > 0) return (k % M) == g && g < M;
        const uint32_t q = k / uint32_t(R * M * M);
        return q * M + (k % M) == g;
    };
    const uint32_t b0 = sel2(bsel(2 * c), bsel(2 * c + 1)), b1 = sel2(bsel(2 * c + 8), bsel(2 * c + 9));
    // ldmatrix (non-transposed) row supplied by this lane: A row rho, column half
    const uint32_t rho = (lane & 7u) + 8u * ((lane >> 3) & 1u), half = lane >> 4;
    bool ovf = false;

    for (uint64_t gi = p.group_begin + blockIdx.x; gi < p.group_end; gi += gridDim.x) {
        const uint64_t gel0 = gi * uint64_t(Cg) * chunk_el;               // first element of the group
        const uint64_t gel1 = gel0 + uint64_t(Cg) * chunk_el;
        const uint64_t lim = gel1 < p.n ? gel1 : p.n;
        auto issue = [&](uint32_t u, uint32_t b) {
            if (u < units) {
                const uint64_t e_unit = gel0 + uint64_t(u) * S.chunks_per_unit * chunk_el;
                for (uint32_t piece = lane; piece < S.unit_rows * 2u; piece += 32) {
                    const uint64_t e = e_unit + uint64_t(piece) * 8u;
                    const uint32_t bytes = e + 8 <= lim ? 16u : (e < lim ? uint32_t(lim - e) * 2u : 0u);
                    cp16(buf0 + b * unit_bytes + piece * 16u, x + (e < lim ? e : 0), bytes);
                }
            }
            cp_commit();
        };
        uint32_t b = 0;
        uint32_t u = warp;
        issue(u, 0);
        for (; u < units; u += kGmWarps, b ^= 1u) {
            issue(u + kGmWarps, b ^ 1u);
            cp_wait<1>();
            __syncwarp();
            const uint32_t base = buf0 + b * unit_bytes;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            const uint32_t steps = S.L > 0 ? S.L : 1u;
            for (uint32_t i = 0; i < steps; ++i) {
                const uint32_t row = S.L > 0 ? rho * S.L + i : rho;
                uint32_t d0, d1, d2, d3;
                ldsm4(base + row * 32u + half * 16u, d0, d1, d2, d3);
                mma_16816(acc, d0, d1, d2, d3, b0, b1);   // C_i = A_i x Bsel + C_{i-1}
            }
            __syncwarp();
            // acc: (row g, col 2c), (g, 2c+1), (g+8, 2c), (g+8, 2c+1)
            const uint32_t cu0 = u * S.chunks_per_unit;
            if (S.L > 0) {
                // chunk = A row; partial j in column j (j < M): lanes c = 0 (j 0,1) and c = 1 (j 2,3)
                const float h0 = h_round(acc[0]), h1 = h_round(acc[1]), h2 = h_round(acc[2]), h3 = h_round(acc[3]);
                const float n0 = __shfl_down_sync(kFull, h0, 1), n1 = __shfl_down_sync(kFull, h1, 1);
                const float n2 = __shfl_down_sync(kFull, h2, 1), n3 = __shfl_down_sync(kFull, h3, 1);
                if (c == 0) {
                    // ascending-j fp32 sum from 0.0f, then + 0 (fragment.hpp:89-92)
                    float ra = 0.0f, rb = 0.0f;
                    ra = ra + h0; ra = ra + h1;
                    rb = rb + h2; rb = rb + h3;
                    if (M == 4) {
                        ra = ra + n0; ra = ra + n1;
                        rb = rb + n2; rb = rb + n3;
                    }
                    ra = ra + 0.0f;
                    rb = rb + 0.0f;
                    ovf |= !isfinite(ra) || !isfinite(rb);
                    if (cu0 + g < Cg) s_chunk[cu0 + g] = ra;
                    if (cu0 + g + 8 < Cg) s_chunk[cu0 + g + 8] = rb;
                }
            } else {
                // M == 2, CR chunks per row: lane (g, q) owns chunk q of rows g and g+8
                if (c < S.CR) {
                    float ra = 0.0f, rb = 0.0f;
                    ra = ra + h_round(acc[0]); ra = ra + h_round(acc[1]); ra = ra + 0.0f;
                    rb = rb + h_round(acc[2]); rb = rb + h_round(acc[3]); rb = rb + 0.0f;
                    ovf |= !isfinite(ra) || !isfinite(rb);
                    const uint32_t ca = cu0 + g * S.CR + c, cb = cu0 + (g + 8) * S.CR + c;
                    if (ca < Cg) s_chunk[ca] = ra;
                    if (cb < Cg) s_chunk[cb] = rb;
                }
            }
        }
        cp_wait<0>();
        group_epilogue(p, gi, s_chunk, s_block);
    }
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kGmThreads);
}

// ================================================================ transposed tiles, m = 8 or 16*S
// Item = K consecutive 256-element tiles holding CPT whole chunks (m = 8, R in {1,2,4}) or one
// chunk (m = 8 with 4 | R, and m >= 32).
struct TrShape {
    uint32_t K;      // tiles per item
    uint32_t CPT;    // chunks per item
};

template <int MM>   // 8, 32, 64, 128
__global__ void __launch_bounds__(kGmThreads) gm_tr_kernel(const SpParams p, const TrShape S) {
    constexpr int D = kGmTrDepth;
    constexpr uint32_t SG = MM >= 32 ? MM / 16 : 1;    // column groups per chunk (m >= 32)
    extern __shared__ __align__(128) unsigned char s_ring[];   // [kGmWarps][D][512] + tables
    __shared__ float s_scratch[32];
    __shared__ int s_last;
    float* s_chunk = reinterpret_cast<float*>(s_ring + kGmWarps * D * 512);
    float* s_block = s_chunk + kMaxChunksGenm;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const unsigned g = lane >> 2, c = lane & 3u;
    const uint32_t ring = smem_u32(s_ring) + warp * D * 512u;
    const uint32_t Cg = p.G * p.W;
    const uint32_t items = Cg / S.CPT;
    const uint32_t R = p.R;
    const uint16_t* x = static_cast<const uint16_t*>(p.x);
    // selector rows kappa in {2c, 2c+1, 2c+8, 2c+9}, column n = g
    auto bsel = [&](uint32_t k) -> bool {
        if (MM >= 32) return (k % SG) == g;
        if (S.CPT > 1) return (k / (4u * R)) == g;   // m = 8: chunk slot of tile row k
        return g == 0;
    };
    const uint32_t b0 = sel2(bsel(2 * c), bsel(2 * c + 1)), b1 = sel2(bsel(2 * c + 8), bsel(2 * c + 9));
    // swizzled 16-byte lines (conflict-free transposing ldmatrix), as in tcr_sp_async.cu
    auto swz = [](uint32_t k, uint32_t h) { return 32u * k + 16u * (h ^ ((k >> 2) & 1u)); };
    const uint32_t cp_dst = swz(lane >> 1, lane & 1u);
    const uint32_t mi = lane >> 3;
    const uint32_t ld_off = swz((lane & 7u) + 8u * (mi >> 1), mi & 1u);
    bool ovf = false;

    for (uint64_t gi = p.group_begin + blockIdx.x; gi < p.group_end; gi += gridDim.x) {
        const uint64_t tile0 = gi * uint64_t(items) * S.K;          // first tile of the group
        const uint32_t my_items = items > warp ? (items - warp + kGmWarps - 1) / kGmWarps : 0;
        const uint32_t F = my_items * S.K;                            // tiles this warp streams
        auto tile_of = [&](uint32_t f) -> uint64_t {                  // warp-local stream -> tile
            const uint32_t it = f / S.K, k = f - it * S.K;
            return tile0 + uint64_t(warp + it * kGmWarps) * S.K + k;
        };
        auto issue = [&](uint32_t f) {
            if (f < F) {
                const uint64_t e = tile_of(f) * 256u + 8u * lane;
                const uint32_t bytes = e + 8 <= p.n ? 16u : (e < p.n ? uint32_t(p.n - e) * 2u : 0u);
                cp16(ring + (f % D) * 512u + cp_dst, x + (e < p.n ? e : 0), bytes);
            }
            cp_commit();
        };
#pragma unroll
        for (int f = 0; f < D - 1; ++f) issue(uint32_t(f));
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t k_in_item = 0, it = 0;
        for (uint32_t f = 0; f < F; ++f) {
            issue(f + D - 1);
            cp_wait<D - 1>();
            __syncwarp();
            uint32_t d0, d1, d2, d3;
            ldsm4t(ring + (f % D) * 512u + ld_off, d0, d1, d2, d3);
            __syncwarp();
            mma_16816(acc, d0, d1, d2, d3, b0, b1);
            if (++k_in_item < S.K) continue;
            // ---- item complete: acc = (j16 = g, n = 2c), (g, 2c+1), (g+8, 2c), (g+8, 2c+1)
            const uint32_t item = warp + it * kGmWarps;
            if (MM == 8) {
                // partial(chunk slot n, j8 = g) = D[g][n] + D[g+8][n]
                const float pe = h_round(acc[0] + acc[2]), po = h_round(acc[1] + acc[3]);
                for (uint32_t sl = 0; sl < S.CPT; ++sl) {
                    const float src = (sl & 1u) ? po : pe;
                    float r = 0.0f;
                    for (uint32_t j = 0; j < 8; ++j) r = r + __shfl_sync(kFull, src, 4 * j + (sl >> 1));
                    r = r + 0.0f;
                    ovf |= !isfinite(r);
                    if (lane == 0) s_chunk[item * S.CPT + sl] = r;
                }
            } else {
                const float h[4] = {h_round(acc[0]), h_round(acc[1]), h_round(acc[2]), h_round(acc[3])};
                float r = 0.0f;
#pragma unroll
                for (uint32_t j = 0; j < uint32_t(MM); ++j) {   // ascending j = 16 n + j16
                    const uint32_t n = j >> 4, j16 = j & 15u;
                    const uint32_t reg = 2u * (j16 >> 3) + (n & 1u);
                    r = r + __shfl_sync(kFull, h[reg], 4 * (j16 & 7u) + (n >> 1));
                }
                r = r + 0.0f;
                ovf |= !isfinite(r);
                if (lane == 0) s_chunk[item] = r;
            }
            acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
            k_in_item = 0;
            ++it;
        }
        cp_wait<0>();
        group_epilogue(p, gi, s_chunk, s_block);
    }
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, &s_last, kGmThreads);
}

bool nat_shape(uint32_t m, uint32_t R, uint32_t Cg, NatShape* S) {
    const uint32_t ce = R * m * m;            // chunk elements
    if (ce >= 16) {
        if (ce % 16) return false;            // chunk must be whole 16-element rows
        S->L = ce / 16;
        if (S->L > 16) return false;          // unit = 16 chunks <= 8 KB per stage
        S->CR = 1;
        S->unit_rows = 16 * S->L;
        S->chunks_per_unit = 16;
    } else {
        if (16 % ce) return false;            // whole chunks per row
        S->L = 0;
        S->CR = 16 / ce;
        if (S->CR * m > 8) return false;      // N = 8 selector columns
        S->unit_rows = 16;
        S->chunks_per_unit = 16 * S->CR;
    }
    if ((uint64_t(Cg) * ce) % 8) return false;  // 16-byte copies never straddle a group
    return true;
}

bool tr_shape(uint32_t m, uint32_t R, uint32_t Cg, TrShape* S) {
    if (m == 8) {
        if (R == 1 || R == 2 || R == 4) {
            S->K = 1;
            S->CPT = 4 / R;
        } else if (R % 4 == 0) {
            S->K = R / 4;
            S->CPT = 1;
        } else {
            return false;
        }
    } else if (m == 32 || m == 64 || m == 128) {
        S->K = R * (m / 16) * (m / 16);
        S->CPT = 1;
    } else {
        return false;
    }
    return Cg % S->CPT == 0;
}

}  // namespace

bool genm_supported(const SpGeometry& g) {
    const uint32_t Cg = g.G * g.W;
    if (g.m == 2 || g.m == 4) {
        NatShape S;
        return nat_shape(g.m, g.R, Cg, &S);
    }
    TrShape S;
    return tr_shape(g.m, g.R, Cg, &S);
}

cudaError_t launch_genm(const SpParams& p, const SpGeometry& g, cudaStream_t s) {
    const uint32_t Cg = g.G * g.W;
    const uint64_t groups = p.group_end - p.group_begin;
    int per_sm = 0;
    if (g.m == 2 || g.m == 4) {
        NatShape S;
        if (!nat_shape(g.m, g.R, Cg, &S)) return cudaErrorInvalidValue;
        const uint32_t dyn = kGmWarps * 2u * S.unit_rows * 32u + 2u * kMaxChunksGenm * 4u;
        auto fn = g.m == 2 ? gm_nat_kernel<2> : gm_nat_kernel<4>;
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
        if (e != cudaSuccess) return e;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGmThreads, dyn);
        if (per_sm < 1) per_sm = 1;
        const int grid = int(groups < uint64_t(per_sm) * sm_count() ? groups : uint64_t(per_sm) * sm_count());
        fn<<<grid, kGmThreads, dyn, s>>>(p, S);
        return cudaGetLastError();
    }
    TrShape S;
    if (!tr_shape(g.m, g.R, Cg, &S)) return cudaErrorInvalidValue;
    void (*fn)(SpParams, TrShape) = nullptr;
    switch (g.m) {
    case 8: fn = gm_tr_kernel<8>; break;
    case 32: fn = gm_tr_kernel<32>; break;
    case 64: fn = gm_tr_kernel<64>; break;
    case 128: fn = gm_tr_kernel<128>; break;
    default: return cudaErrorInvalidValue;
    }
    const uint32_t dyn = kGmWarps * kGmTrDepth * 512u + 2u * kMaxChunksGenm * 4u;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGmThreads, dyn);
    if (per_sm < 1) per_sm = 1;
    const int grid = int(groups < uint64_t(per_sm) * sm_count() ? groups : uint64_t(per_sm) * sm_count());
    fn<<<grid, kGmThreads, dyn, s>>>(p, S);
    return cudaGetLastError();
}

}  // namespace tcr
