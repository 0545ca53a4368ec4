// tcr_sp_bulk.cu -- single-pass chained reduction, m = 16, TMA-staged mma.sync engine.
//
// Same element partition / block stage / group stage as tcr_single_pass.cu and tcr_tc05.cu
// (reference reduction.hpp:164-184, :238-275).  Data path:
//
//   warp 0 (one thread)  cp.async.bulk (1-D TMA) of whole slots -- SC consecutive warp-chunks,
//                        16-32 KB -- into a shared-memory ring, completion on an mbarrier.
//   warps 1..8           per fragment ONE ldmatrix.x4.trans + ONE HMMA.16816: the transposing
//                        matrix load hands every lane the A fragment whose row j is column j of
//                        the 16x16 fragment (all 16 k), so D[j][*] = ones x M_r + C exactly as
//                        reduction.hpp:177; C_R -> binary16, finishing HMMA per two chunks;
//                        chunk results into the tile table, then block and group trees.
//
// No data passes through registers before it is consumed, so memory-level parallelism is the
// ring depth (~190 KB per SM), not a register budget.
#include <cuda_runtime.h>

#include "tcr_device.cuh"
#include "tcr_kernels.h"
#include "tcr_pipeline.cuh"

namespace tcr {

namespace {

using namespace pipe;

constexpr int kBkConsumers = 16;                      // consumer warps
constexpr int kBkThreads = 32 * (1 + kBkConsumers);
constexpr uint32_t kBkRingBytes = 192 * 1024;
constexpr int kBkTileBufs = 2;

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

struct BkLayout {
    uint32_t bar_off, misc_off, total;
};

__host__ __device__ inline BkLayout bk_layout(uint32_t slot_bytes, uint32_t ns) {
    BkLayout L;
    L.bar_off = slot_bytes * ns;
    L.misc_off = L.bar_off + 16 * ns + 16;
    L.total = L.misc_off + 4 * (2 * kBkTileBufs * kMaxChunksPerGroup + 32 + 8) + 128;
    return L;
}

// Reduce SCW chunks of one warp in a slot.  Returns nothing; writes chunk results.
template <int RT>
__device__ __forceinline__ void bk_warp_chunks(uint32_t slot_saddr, uint32_t lane_off, uint32_t R, uint32_t scw,
                                               uint32_t cw, float* chunks, uint32_t chunk_base, bool& ovf) {
    const unsigned lane = lane_id();
    const unsigned c = lane & 3u;
    const uint32_t Rr = RT > 0 ? uint32_t(RT) : R;
    const uint32_t chunk_bytes = Rr * 512u;
    // two chunks per finishing MMA
    for (uint32_t i = 0; i < scw; i += 2) {
        uint32_t a01[2], a23[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t ci = cw + (i + h) * kBkConsumers;   // chunk index within the slot
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            if (i + h < scw) {
                const uint32_t base = slot_saddr + ci * chunk_bytes + lane_off;
                if constexpr (RT > 0) {
#pragma unroll
                    for (int r = 0; r < RT; ++r) {
                        uint32_t d0, d1, d2, d3;
                        ldsm_x4_trans(base + r * 512u, d0, d1, d2, d3);
                        mma_16816(acc, d0, d1, d2, d3, kOnesF16x2, kOnesF16x2);
                    }
                } else {
                    for (uint32_t r = 0; r < Rr; ++r) {
                        uint32_t d0, d1, d2, d3;
                        ldsm_x4_trans(base + r * 512u, d0, d1, d2, d3);
                        mma_16816(acc, d0, d1, d2, d3, kOnesF16x2, kOnesF16x2);
                    }
                }
            }
            // thread (g, c): acc[0] = C_R[j = g], acc[2] = C_R[j = g + 8]  -> binary16 (:179-181)
            const uint32_t pk = uint32_t(f32_to_h(acc[0])) | (uint32_t(f32_to_h(acc[2])) << 16);
            const uint32_t vA = __shfl_sync(kFull, pk, 8 * c);       // (h_2c,   h_2c+8)
            const uint32_t vB = __shfl_sync(kFull, pk, 8 * c + 4);   // (h_2c+1, h_2c+9)
            a01[h] = prmt(vA, vB, 0x5410);                           // (h_2c,   h_2c+1)
            a23[h] = prmt(vA, vB, 0x7632);                           // (h_2c+8, h_2c+9)
        }
        float fin[4] = {0.f, 0.f, 0.f, 0.f};
        // finishing MMA (reduction.hpp:182): rows 0-7 chunk i, rows 8-15 chunk i+1
        mma_16816(fin, a01[0], a01[1], a23[0], a23[1], kOnesF16x2, kOnesF16x2);
        ovf |= !isfinite(fin[0]) || (i + 1 < scw && !isfinite(fin[2]));
        if (lane == 0) {
            chunks[chunk_base + cw + i * kBkConsumers] = fin[0];
            if (i + 1 < scw) chunks[chunk_base + cw + (i + 1) * kBkConsumers] = fin[2];
        }
    }
}

template <int RT>
__global__ void __launch_bounds__(kBkThreads, 1)
sp_bulk_kernel(const SpParams p, const uint32_t SC, const uint32_t ns, const uint64_t n_tiles) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    const uint32_t R = RT > 0 ? uint32_t(RT) : p.R;
    const uint32_t slot_bytes = SC * R * 512u;
    const BkLayout L = bk_layout(slot_bytes, ns);
    unsigned char* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + ns;
    float* s_chunk = reinterpret_cast<float*>(smem + L.misc_off);          // [kBkTileBufs][256]
    float* s_block = s_chunk + kBkTileBufs * kMaxChunksPerGroup;           // [kBkTileBufs][256]
    float* s_scratch = s_block + kBkTileBufs * kMaxChunksPerGroup;
    int* s_last = reinterpret_cast<int*>(s_scratch + 32);

    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const uint32_t Cg = p.G * p.W;
    const uint32_t slots_per_tile = Cg / SC;

    if (warp == 0 && lane == 0) {
        for (uint32_t i = 0; i < ns; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kBkConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    bool ovf = false;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t policy = evict_first_policy();
            const char* x = static_cast<const char*>(p.x);
            uint32_t t = 0;
            for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const uint64_t tile_byte0 = tile * uint64_t(Cg) * R * 512u;
                for (uint32_t s = 0; s < slots_per_tile; ++s, ++t) {
                    const uint32_t rs = t % ns, ph = (t / ns) & 1;
                    mbar_wait(&empty[rs], ph ^ 1);
                    mbar_expect_tx(&full[rs], slot_bytes);
                    bulk_load_1d(ring + size_t(rs) * slot_bytes, x + tile_byte0 + uint64_t(s) * slot_bytes, slot_bytes,
                                 &full[rs], policy);
                }
            }
        }
    } else {
        const uint32_t cw = warp - 1;   // consumer index
        // ldmatrix row address of this lane inside a fragment: matrix mi = lane>>3 supplies
        // line (k = (lane&7) + 8*(mi>>1), half = mi&1)  -> byte 32k + 16*half
        const uint32_t mi = lane >> 3;
        const uint32_t lane_off = 32u * ((lane & 7u) + 8u * (mi >> 1)) + 16u * (mi & 1u);
        const uint32_t scw = SC / kBkConsumers;  // chunks per consumer warp per slot
        uint32_t t = 0, k = 0;
        for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
            const uint32_t buf = k % kBkTileBufs;
            float* chunks = s_chunk + buf * kMaxChunksPerGroup;
            for (uint32_t s = 0; s < slots_per_tile; ++s, ++t) {
                const uint32_t rs = t % ns, ph = (t / ns) & 1;
                mbar_wait(&full[rs], ph);
                const uint32_t sa = smem_u32(ring + size_t(rs) * slot_bytes);
                if (p.debug_mode != 1) bk_warp_chunks<RT>(sa, lane_off, R, scw, cw, chunks, s * SC, ovf);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[rs]);
            }
            named_bar(1, 32 * kBkConsumers);
            float* blocks = s_block + buf * kMaxChunksPerGroup;
            tile_trees_blocks(p, tile, chunks, blocks, cw, kBkConsumers);
            named_bar(1, 32 * kBkConsumers);
            if (cw == 0) tile_tree_group(p, tile, blocks);
        }
        if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    }
    __threadfence();
    __syncthreads();
    finalize_last_cta(p, s_scratch, s_last, 512);
}

}  // namespace

bool bulk_plan(const SpGeometry& g, uint32_t* SC_out, uint32_t* ns_out) {
    if (g.m != 16) return false;
    const uint64_t cg = uint64_t(g.G) * g.W;
    // slot = SC chunks (a multiple of the consumer count), ~32 KB, dividing the tile
    uint32_t SC = 0;
    for (uint32_t cand = 256; cand >= uint32_t(kBkConsumers); cand -= kBkConsumers) {
        if (cand % kBkConsumers == 0 && cg % cand == 0 && uint64_t(cand) * g.R * 512u <= 49152u) {
            SC = cand;
            break;
        }
    }
    if (!SC) return false;
    const uint32_t slot = SC * g.R * 512u;
    uint32_t ns = kBkRingBytes / slot;
    if (ns > 16) ns = 16;
    if (ns < 3) return false;
    if (bk_layout(slot, ns).total > 227u * 1024u) return false;
    *SC_out = SC;
    *ns_out = ns;
    return true;
}

cudaError_t launch_bulk(const SpParams& p, const SpGeometry& g, uint64_t n_tiles, int grid, cudaStream_t s) {
    uint32_t SC, ns;
    if (!bulk_plan(g, &SC, &ns)) return cudaErrorInvalidValue;
    const BkLayout L = bk_layout(SC * g.R * 512u, ns);
    static PerDeviceOnce once;
    const cudaError_t ea = once([] {
        for (auto fn : {sp_bulk_kernel<0>, sp_bulk_kernel<1>, sp_bulk_kernel<2>, sp_bulk_kernel<3>,
                        sp_bulk_kernel<4>, sp_bulk_kernel<5>}) {
            const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    });
    if (ea != cudaSuccess) return ea;
    switch (g.R) {
    case 1: sp_bulk_kernel<1><<<grid, kBkThreads, L.total, s>>>(p, SC, ns, n_tiles); break;
    case 2: sp_bulk_kernel<2><<<grid, kBkThreads, L.total, s>>>(p, SC, ns, n_tiles); break;
    case 3: sp_bulk_kernel<3><<<grid, kBkThreads, L.total, s>>>(p, SC, ns, n_tiles); break;
    case 4: sp_bulk_kernel<4><<<grid, kBkThreads, L.total, s>>>(p, SC, ns, n_tiles); break;
    case 5: sp_bulk_kernel<5><<<grid, kBkThreads, L.total, s>>>(p, SC, ns, n_tiles); break;
    default: sp_bulk_kernel<0><<<grid, kBkThreads, L.total, s>>>(p, SC, ns, n_tiles); break;
    }
    return cudaGetLastError();
}

}  // namespace tcr
