// tcr_tc05.cu -- single-pass chained reduction on the 5th-gen tensor cores (tcgen05 + TMA + TMEM).
//
// Same element partition, block stage and group stage as tcr_single_pass.cu (reference
// reduction.hpp:164-184, :238-275); different machinery:
//
//   warp 0  TMA producer  -- cp.async.bulk.tensor.3d (SWIZZLE_32B) streams whole slots of the
//                            input (Q MMA-groups of 8 warp-chunks) into a smem ring; mbarrier tx.
//   warp 1  MMA issuer    -- one thread issues tcgen05.mma.kind::f16, M=128 N=16 K=16:
//                            A = 8 chunks' fragment r viewed MN-major (row m = 16*chunk + j,
//                            K = fragment row k), B = ones.  The 32-byte swizzle the TMA applies
//                            is exactly the UMMA SWIZZLE_32B MN-major atom, so TMEM lane
//                            16*chunk + j accumulates column j of the chunk: the reference's
//                            C_r = ones x M_r + C_{r-1}, chained R times in TMEM.
//   warps 2-5 epilogue    -- tcgen05.ld (32x32b) of the accumulators, C_R -> binary16 (RNE) with
//                            the overflow note, the finishing MMA (HMMA.16816: sum of the 16
//                            binary16 partials, two chunks per warp), block pairwise tree, group
//                            tree -> group partial.  Last CTA finalises.
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>

#include "tcr_device.cuh"
#include "tcr_kernels.h"
#include "tcr_pipeline.cuh"

namespace tcr {

namespace {

using namespace pipe;

constexpr int kEpiWarp0 = 2;
constexpr int kAccBufs = 8;         // TMEM accumulator ring depth
constexpr uint32_t kRingBytes = 160 * 1024;

// UMMA shared-memory matrix descriptor (sm_100: version 1 at bits 46-47).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout & 7) << 61;
    return d;
}

constexpr uint32_t kLayoutNone = 0, kLayoutSw32 = 6;

// kind::f16 instruction descriptor: D f32, A/B f16, A MN-major, B K-major, N=16, M=128.
constexpr uint32_t kIdesc = (1u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | (0u << 16) | ((16u >> 3) << 17) |
                            ((128u >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate,
                                         uint32_t idesc = kIdesc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Profiling-only instruction descriptors (debug modes 4/5): A K-major; N = 64.
constexpr uint32_t kIdescKmajor = (1u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescN64 = (1u << 4) | (1u << 15) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
    return v;
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

constexpr int kEpiGroups = 3;                         // epilogue warpgroups, round-robin over slots
constexpr int kTileBufs = 4;                            // per-tile chunk/block tables in flight

__host__ __device__ constexpr int tc_threads(int eg) { return 64 + 128 * eg; }  // TMA warp + MMA warp + epilogue

struct SmemLayout {
    uint32_t ring_off, ones_off, bar_off, misc_off, total;
};

__host__ __device__ inline SmemLayout smem_layout(uint32_t slot_bytes, uint32_t ns, uint32_t acc = kAccBufs) {
    SmemLayout L;
    L.ring_off = 0;
    L.ones_off = slot_bytes * ns;
    L.bar_off = L.ones_off + 1024;
    L.misc_off = L.bar_off + 8 * (2 * ns + 2 * acc) + 16;
    // s_chunk[kTileBufs][256] + s_block[kTileBufs][256] + s_scratch[32] + s_done[kTileBufs] + s_own[4] + s_last
    L.total = L.misc_off + 4 * (2 * kTileBufs * kMaxChunksPerGroup + 32 + kTileBufs + 8) + 1024;  // +1024 align slack
    return L;
}

// Q MMA-groups per slot, EG epilogue warpgroups, ACC TMEM accumulator buffers, CPS CTAs per SM.
template <int Q, int EG = kEpiGroups, int ACC = kAccBufs, int CPS = 1>
__global__ void __launch_bounds__(tc_threads(EG), CPS)
tc05_kernel(const __grid_constant__ CUtensorMap tmap, const SpParams p, const uint32_t ns, const uint64_t n_tiles) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t R = p.R, W = p.W, G = p.G;
    const uint32_t slot_bytes = 4096u * Q * R;
    const SmemLayout L = smem_layout(slot_bytes, ns, ACC);
    unsigned char* ring = smem + L.ring_off;
    uint16_t* ones = reinterpret_cast<uint16_t*>(smem + L.ones_off);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + ns;
    uint64_t* tfull = empty + ns;
    uint64_t* tempty = tfull + ACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC);
    float* s_chunk = reinterpret_cast<float*>(smem + L.misc_off);             // [kTileBufs][256]
    float* s_block = s_chunk + kTileBufs * kMaxChunksPerGroup;                 // [kTileBufs][256]
    float* s_scratch = s_block + kTileBufs * kMaxChunksPerGroup;               // [32]
    uint32_t* s_done = reinterpret_cast<uint32_t*>(s_scratch + 32);            // [kTileBufs]
    uint32_t* s_own = s_done + kTileBufs;                                      // [4]
    int* s_last = reinterpret_cast<int*>(s_own + 4);

    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const uint32_t Cg = G * W;                        // chunks per tile (group)
    const uint32_t slots_per_tile = Cg / (8u * Q);
    constexpr uint32_t acc_cols = 16u * Q;            // TMEM columns per accumulator buffer

    // ---- setup
    for (uint32_t i = threadIdx.x; i < 512; i += blockDim.x) ones[i] = 0x3C00u;
    if (threadIdx.x < kTileBufs) s_done[threadIdx.x] = 0;
    if (warp == 0 && lane == 0) {
        for (uint32_t i = 0; i < ns; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < ACC; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    constexpr uint32_t ncols = acc_cols * ACC <= 32 ? 32 : acc_cols * ACC <= 64 ? 64
                             : acc_cols * ACC <= 128 ? 128 : acc_cols * ACC <= 256 ? 256 : 512;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // ones[] visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    bool ovf = false;

    if (warp == 0) {
        // ================= TMA producer
        if (lane == 0) {
            const uint64_t policy = evict_first_policy();
            uint32_t t = 0;
            const uint64_t slabs_per_slot = 16ull * Q * R;   // 8-row slabs (128 elements)
            for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const uint64_t slab0 = tile * (uint64_t(Cg) * R * 2);  // chunk = R*256 el = 2R slabs
                for (uint32_t s = 0; s < slots_per_tile; ++s, ++t) {
                    const uint32_t rs = t % ns, ph = (t / ns) & 1;
                    mbar_wait(&empty[rs], ph ^ 1);
                    mbar_expect_tx(&full[rs], slot_bytes);
                    if (p.debug_mode == 2)
                        bulk_load_1d(ring + size_t(rs) * slot_bytes,
                                     static_cast<const char*>(p.x) + (slab0 + uint64_t(s) * slabs_per_slot) * 256,
                                     slot_bytes, &full[rs], policy);
                    else
                        tma_load_3d(ring + size_t(rs) * slot_bytes, &tmap, &full[rs], 0, 0,
                                    int(slab0 + uint64_t(s) * slabs_per_slot), policy);
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (single thread)
        if (lane == 0) {
            const uint64_t bdesc = umma_desc(smem_u32(ones), 128, 256, kLayoutNone);
            uint32_t t = 0;
            for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                for (uint32_t s = 0; s < slots_per_tile; ++s, ++t) {
                    const uint32_t rs = t % ns, ph = (t / ns) & 1;
                    const uint32_t ab = t % ACC, aph = (t / ACC) & 1;
                    mbar_wait(&full[rs], ph);
                    if (p.debug_mode == 1) {
                        mbar_arrive(&empty[rs]);
                        continue;
                    }
                    if (!(p.debug_mode >= 3 && p.debug_mode <= 5)) mbar_wait(&tempty[ab], aph ^ 1);
                    tc_fence_after();
                    const uint32_t sbase = smem_u32(ring + size_t(rs) * slot_bytes);
#pragma unroll
                    for (uint32_t q = 0; q < uint32_t(Q); ++q) {
                        const uint32_t d = tmem_base + ab * acc_cols + 16u * q;
                        for (uint32_t r = 0; r < R; ++r) {
                            // 8 chunks of this MMA-group, fragment r: MN atoms (chunks) R*512 B apart,
                            // K groups of 8 rows 256 B apart
                            const uint32_t a = sbase + (8u * q * R + r) * 512u;
                            if (p.debug_mode == 4)        // timing only: A read K-major (wrong partition)
                                umma_f16(tmem_base, umma_desc(a, 256u, R * 512u, kLayoutSw32), bdesc, r > 0 ? 1u : 0u,
                                         kIdescKmajor);
                            else if (p.debug_mode == 5)   // timing only: N = 64 into one accumulator
                                umma_f16(tmem_base, umma_desc(a, R * 512u, 256u, kLayoutSw32), bdesc, r > 0 ? 1u : 0u,
                                         kIdescN64);
                            else
                                umma_f16(d, umma_desc(a, R * 512u, 256u, kLayoutSw32), bdesc, r > 0 ? 1u : 0u);
                        }
                    }
                    umma_commit(&empty[rs]);   // smem slot reusable once these MMAs retire
                    umma_commit(&tfull[ab]);   // accumulators ready for the epilogue
                }
            }
        }
    } else {
        // ================= epilogue: warpgroup eg takes slots t = eg (mod EG)
        uint64_t n_tiles_epi = n_tiles;
        const uint32_t ew = warp - kEpiWarp0;         // 0 .. 4*EG-1
        const uint32_t eg = ew >> 2, w4 = ew & 3u;    // warpgroup, warp within it
        const uint32_t qw = warp & 3u;                // TMEM lane quarter this warp may access
        const uint32_t c = lane & 3u;
        const int bar_id = 1 + int(eg);
        uint32_t t = 0, k = 0;
        if (p.debug_mode == 1 || (p.debug_mode >= 3 && p.debug_mode <= 5)) n_tiles_epi = 0;
        uint32_t P = 1;
        while (P < W) P <<= 1;
        for (uint64_t tile = blockIdx.x; tile < n_tiles_epi; tile += gridDim.x, ++k) {
            const uint32_t buf = k % kTileBufs;
            float* chunks = s_chunk + buf * kMaxChunksPerGroup;
            for (uint32_t s = 0; s < slots_per_tile; ++s, ++t) {
                if (t % EG != eg) continue;
                const uint32_t ab = t % ACC, aph = (t / ACC) & 1;
                mbar_wait(&tfull[ab], aph);
                tc_fence_after();
                uint32_t v[Q];
                const uint32_t taddr = tmem_base + ((32u * qw) << 16) + ab * acc_cols;
#pragma unroll
                for (int q = 0; q < Q; ++q) v[q] = tmem_ld1(taddr + 16u * q);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[ab]);
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    // lane l holds C_R[j = l & 15] of chunk 2*qw + (l >> 4) of MMA-group q
                    const uint32_t h = f32_to_h(__uint_as_float(v[q]));
                    const uint32_t hp = h | (__shfl_down_sync(kFull, h, 1) << 16);  // even lanes: (h_2i, h_2i+1)
                    const uint32_t a0 = __shfl_sync(kFull, hp, 2 * c);
                    const uint32_t a2 = __shfl_sync(kFull, hp, 2 * c + 8);
                    const uint32_t a1 = __shfl_sync(kFull, hp, 16 + 2 * c);
                    const uint32_t a3 = __shfl_sync(kFull, hp, 16 + 2 * c + 8);
                    float fin[4] = {0.f, 0.f, 0.f, 0.f};
                    // finishing MMA (reduction.hpp:182): rows 0-7 chunk A, rows 8-15 chunk B
                    mma_16816(fin, a0, a1, a2, a3, kOnesF16x2, kOnesF16x2);
                    // a non-finite binary16 partial makes its finishing sum non-finite
                    ovf |= !isfinite(fin[0]) || !isfinite(fin[2]);
                    if (lane == 0) {
                        const uint32_t ch = s * 8u * Q + 8u * q + 2u * qw;
                        chunks[ch] = fin[0];
                        chunks[ch + 1] = fin[2];
                    }
                }
                // slot bookkeeping: the warpgroup that completes a tile runs its trees
                named_bar(bar_id, 128);
                if (w4 == 0 && lane == 0) {
                    __threadfence_block();
                    const uint32_t old = atomicAdd(&s_done[buf], 1u);
                    s_own[eg] = (old + 1 == slots_per_tile);
                    __threadfence_block();
                }
                named_bar(bar_id, 128);
                if (s_own[eg]) {
                    float* blocks = s_block + buf * kMaxChunksPerGroup;
                    tile_trees_blocks(p, tile, chunks, blocks, w4, 4);
                    named_bar(bar_id, 128);
                    if (w4 == 0) {
                        tile_tree_group(p, tile, blocks);
                        if (lane == 0) s_done[buf] = 0;
                    }
                    named_bar(bar_id, 128);
                }
            }
        }
        if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);
    }

    // ---- teardown
    tc_fence_before();
    __threadfence();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));

    finalize_last_cta(p, s_scratch, s_last, EG >= 2 ? 256 : 128);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

}  // namespace

bool tc05_plan(const SpGeometry& g, uint32_t* Q_out, uint32_t* ns_out) {
    if (g.m != 16 || g.R > 12) return false;
    const uint64_t cg = uint64_t(g.G) * g.W;
    if (cg % 8 != 0 || cg > uint64_t(kMaxChunksPerGroup)) return false;
    uint32_t Q = 4;
    while (Q > 1 && (cg % (8ull * Q) != 0 || Q * g.R > 8)) Q >>= 1;
    const uint32_t slot = 4096u * Q * g.R;
    uint32_t ns = kRingBytes / slot;
    if (ns > 16) ns = 16;
    if (smem_layout(slot, ns).total > 227u * 1024u) return false;
    if (ns < 2) return false;
    *Q_out = Q;
    *ns_out = ns;
    return true;
}

cudaError_t launch_tc05(const SpParams& p, const SpGeometry& g, uint64_t n_tiles, int grid, cudaStream_t s) {
    uint32_t Q, ns;
    if (!tc05_plan(g, &Q, &ns)) return cudaErrorInvalidValue;
    EncodeTiledFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap map;
    const cuuint64_t dims[3] = {16, 8, cuuint64_t(n_tiles * g.group_elems / 128)};
    const cuuint64_t strides[2] = {32, 256};
    const cuuint32_t box[3] = {16, 8, cuuint32_t(16u * Q * g.R)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(p.x), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    static PerDeviceOnce once;
    const cudaError_t ea = once([] {
        for (auto fn : {tc05_kernel<1>, tc05_kernel<2>, tc05_kernel<4>, tc05_kernel<1, 1, 4, 2>, tc05_kernel<2, 1, 4, 2>,
                        tc05_kernel<4, 1, 4, 2>}) {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    });
    if (ea != cudaSuccess) return ea;
    if (p.debug_mode == 11) {
        // profiling: two CTAs per SM (half ring, one epilogue warpgroup, 4 accumulators each)
        const uint32_t ns2 = ns / 2 < 2 ? 2 : ns / 2;
        const SmemLayout L2 = smem_layout(4096u * Q * g.R, ns2, 4);
        const int grid2 = int(std::min<uint64_t>(n_tiles, 2ull * sm_count()));
        if (Q == 4) tc05_kernel<4, 1, 4, 2><<<grid2, tc_threads(1), L2.total, s>>>(map, p, ns2, n_tiles);
        else if (Q == 2) tc05_kernel<2, 1, 4, 2><<<grid2, tc_threads(1), L2.total, s>>>(map, p, ns2, n_tiles);
        else tc05_kernel<1, 1, 4, 2><<<grid2, tc_threads(1), L2.total, s>>>(map, p, ns2, n_tiles);
        return cudaGetLastError();
    }
    const SmemLayout L = smem_layout(4096u * Q * g.R, ns);
    if (Q == 4) tc05_kernel<4><<<grid, tc_threads(kEpiGroups), L.total, s>>>(map, p, ns, n_tiles);
    else if (Q == 2) tc05_kernel<2><<<grid, tc_threads(kEpiGroups), L.total, s>>>(map, p, ns, n_tiles);
    else tc05_kernel<1><<<grid, tc_threads(kEpiGroups), L.total, s>>>(map, p, ns, n_tiles);
    return cudaGetLastError();
}

}  // namespace tcr
