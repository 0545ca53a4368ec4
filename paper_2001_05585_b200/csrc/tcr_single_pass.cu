// tcr_single_pass.cu -- single-pass chained tensor-core reduction, m = 16 (mma.sync path).
//
// Replaces tcreduce::single_pass_reduce / detail::single_pass_core
// (reference reduction.hpp:238-293) and chained_warp_reduce (:164-184).
//
// Element partition (identical to the reference): a warp chunk is R consecutive
// 256-element fragments; fragment r viewed row-major as M_r[k][j] (16x16); the
// chain computes C_R[j] = sum_r sum_k M_r[k][j] (ones x M_r + C, fp32 accumulate),
// rounds C_R to binary16, and a finishing MMA sums the 16 binary16 partials.
//
// Register layout: every lane loads ONE 16-byte line (8 consecutive j of one k)
// per fragment with a streaming 128-bit load; four MOVM (movmatrix .trans) turn
// rows into columns, so lane (g, c) ends up holding k-pairs of a single column j.
// A shuffle with lane^16 brings the other k-half, which makes each A row of
// HMMA.16816 one full column j of the fragment:  D[j][*] = sum_k M_r[k][j] + C.
//
// Block stage (reference :249-255): the W chunk results of a logical block are
// combined with the reference's pairwise tree (offsets pow2(W)/2 .. 1); group /
// grid stage: deterministic pairwise tree (default), reference-ordered serial
// sum, or the paper's atomicAdd.
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>
#include <type_traits>

#include "tcr_device.cuh"
#include "tcr_kernels.h"
#include "tcr_pipeline.cuh"

namespace tcr {

namespace {

constexpr int U = 4;  // fragments in flight per warp (rolling prefetch depth)

struct Frag {
    uint32_t r0, r1, r2, r3;
};

template <bool F32IN, bool CHECKED>
__device__ __forceinline__ Frag load_line(const void* x, uint64_t e, uint64_t n) {
    // e = element index of this lane's 8-element line
    Frag f;
    if (!CHECKED || e + 8 <= n) {
        if constexpr (F32IN) {
            const float* p = static_cast<const float*>(x) + e;
            const float4 lo = ldg_stream_f4(p);
            const float4 hi = ldg_stream_f4(p + 4);
            f.r0 = pack_h2(lo.x, lo.y);
            f.r1 = pack_h2(lo.z, lo.w);
            f.r2 = pack_h2(hi.x, hi.y);
            f.r3 = pack_h2(hi.z, hi.w);
        } else {
            const uint4 v = ldg_stream_v4(static_cast<const uint16_t*>(x) + e);
            f.r0 = v.x;
            f.r1 = v.y;
            f.r2 = v.z;
            f.r3 = v.w;
        }
    } else {
        // ragged tail: zero padding exactly like reduction.hpp:244-245
        uint16_t h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (e + i < n) {
                if constexpr (F32IN) h[i] = f32_to_h(static_cast<const float*>(x)[e + i]);
                else h[i] = static_cast<const uint16_t*>(x)[e + i];
            } else {
                h[i] = 0;
            }
        }
        f.r0 = h[0] | (uint32_t(h[1]) << 16);
        f.r1 = h[2] | (uint32_t(h[3]) << 16);
        f.r2 = h[4] | (uint32_t(h[5]) << 16);
        f.r3 = h[6] | (uint32_t(h[7]) << 16);
    }
    return f;
}

// Adjacent pairwise tree over 32 lanes (lane 2i pairs with 2i+1, then groups of 2, ...).
__device__ __forceinline__ float warp_tree_xor(float v) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const float o = __shfl_xor_sync(kFull, v, off);
        // keep the left operand on the left: (lower index) + (higher index)
        v = (lane_id() & off) ? (o + v) : (v + o);
    }
    return v;
}

// Canonical adjacent tree over vals[0, count) padded with zeros to a power of two,
// computed by one CTA (blockDim.x threads, power of two, <= 1024).
__device__ float cta_tree(const float* vals, uint64_t count, float* s_scratch) {
    uint64_t P = 1;
    while (P < count) P <<= 1;
    const unsigned T = blockDim.x;
    uint64_t seg = P / T;
    if (seg == 0) seg = 1;
    float acc = 0.0f;
    const uint64_t lo = uint64_t(threadIdx.x) * seg;
    if (lo < P) {
        // streaming adjacent tree over [lo, lo + seg) (seg is a power of two)
        float stk[40];
        int top = 0;
        for (uint64_t i = 0; i < seg; ++i) {
            const uint64_t idx = lo + i;
            float v = idx < count ? __ldcg(vals + idx) : 0.0f;
            for (uint64_t b = i; b & 1; b >>= 1) v = stk[--top] + v;
            stk[top++] = v;
        }
        acc = stk[0];
    }
    acc = warp_tree_xor(acc);
    const unsigned w = threadIdx.x >> 5;
    if (lane_id() == 0) s_scratch[w] = acc;
    __syncthreads();
    float r = 0.0f;
    if (w == 0) {
        const unsigned nw = T >> 5;
        r = lane_id() < nw ? s_scratch[lane_id()] : 0.0f;
        r = warp_tree_xor(r);
    }
    __syncthreads();
    return r;  // valid in thread 0
}

__device__ void finalize_cta(const SpParams& p, float* s_scratch) {
    if (p.finalize == kFinTree) {
        const float r = cta_tree(p.group_partials, p.n_groups, s_scratch);
        if (threadIdx.x == 0) *p.result = r;
    } else if (p.finalize == kFinOrdered) {
        // reduction.hpp:257-268: serial binary32 accumulation in ascending block order or
        // the seeded Fisher-Yates order of SplitMix64(atomic_seed).
        if (threadIdx.x == 0) {
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
                    const uint32_t t = order[i - 1];
                    order[i - 1] = order[r];
                    order[r] = t;
                }
                for (uint64_t i = 0; i < p.n_blocks; ++i) acc += __ldcg(p.block_partials + order[i]);
            } else {
                for (uint64_t b = 0; b < p.n_blocks; ++b) acc += __ldcg(p.block_partials + b);
            }
            *p.result = acc;
        }
    }
}

template <bool F32IN, bool CHECKED>
__device__ __noinline__ void sp16_group(const SpParams& p, uint64_t gi, float* s_chunk, bool& ovf) {
    const unsigned warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const unsigned c = lane & 3;
    // load mapping: lane L = 8a + 4b + d reads line (k = 2a + b + 8(d>>1), half h = d&1)
    const unsigned la = lane >> 3, lb = (lane >> 2) & 1, ld = lane & 3;
    const uint32_t line_off = 16u * (2u * la + lb + 8u * (ld >> 1)) + 8u * (ld & 1u);
    const uint32_t R = p.R, W = p.W, G = p.G;
    const uint32_t Cg = G * W;                      // chunks per group
    const uint64_t ce = p.chunk_elems;              // R*256
    const uint64_t jump = 256ull + uint64_t(kSpWarps - 1) * ce;  // next fragment at chunk wrap
    const uint64_t chunk0 = gi * uint64_t(Cg);
    const uint32_t nch = Cg > warp ? (Cg - warp + kSpWarps - 1) / kSpWarps : 0;
    const uint32_t F = nch * R;
    uint64_t l_elem = (chunk0 + warp) * ce + line_off;
    uint32_t l_r = 0;
    Frag buf[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (uint32_t(u) < F) {
            buf[u] = load_line<F32IN, CHECKED>(p.x, l_elem, p.n);
            if (++l_r == R) { l_r = 0; l_elem += jump; } else { l_elem += 256; }
        } else {
            buf[u] = Frag{0, 0, 0, 0};
        }
    }
    float acc1[4] = {0.f, 0.f, 0.f, 0.f}, acc2[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t c_r = 0, c_ch = warp;
    for (uint32_t f0 = 0; f0 < F; f0 += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const Frag v = buf[u];
            if (f0 + U + u < F) {
                buf[u] = load_line<F32IN, CHECKED>(p.x, l_elem, p.n);
                if (++l_r == R) { l_r = 0; l_elem += jump; } else { l_elem += 256; }
            }
            if (f0 + u < F) {
                const uint32_t t0 = movmatrix_trans(v.r0), t1 = movmatrix_trans(v.r1);
                const uint32_t t2 = movmatrix_trans(v.r2), t3 = movmatrix_trans(v.r3);
                const uint32_t q0 = __shfl_xor_sync(kFull, t0, 16), q1 = __shfl_xor_sync(kFull, t1, 16);
                const uint32_t q2 = __shfl_xor_sync(kFull, t2, 16), q3 = __shfl_xor_sync(kFull, t3, 16);
                if (c_r == 0) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) { acc1[i] = 0.f; acc2[i] = 0.f; }
                }
                mma_16816(acc1, t0, t1, q0, q1, kOnesF16x2, kOnesF16x2);
                mma_16816(acc2, t2, t3, q2, q3, kOnesF16x2, kOnesF16x2);
                if (++c_r == R) {
                    const uint32_t h0 = f32_to_h(acc1[0]), h1 = f32_to_h(acc1[2]);
                    const uint32_t h2 = f32_to_h(acc2[0]), h3 = f32_to_h(acc2[2]);
                    const uint32_t sel = c == 0 ? h0 : c == 1 ? h1 : c == 2 ? h2 : h3;
                    const uint32_t v0 = __shfl_sync(kFull, sel, c);
                    const uint32_t v1 = __shfl_sync(kFull, sel, 4 + c);
                    const uint32_t v2 = __shfl_sync(kFull, sel, 8 + c);
                    const uint32_t v3 = __shfl_sync(kFull, sel, 12 + c);
                    const uint32_t a01 = v0 | (v1 << 16), a23 = v2 | (v3 << 16);
                    float fin[4] = {0.f, 0.f, 0.f, 0.f};
                    mma_16816(fin, a01, a01, a23, a23, kOnesF16x2, kOnesF16x2);
                    // any non-finite binary16 partial makes the finishing sum non-finite (and no
                    // sum of 16 finite binary16 values overflows fp32): one check per chunk
                    ovf |= !isfinite(fin[0]);
                    if (lane == 0) s_chunk[c_ch] = fin[0];
                    c_r = 0;
                    c_ch += kSpWarps;
                }
            }
        }
    }
}


// Fast path for full groups with a compile-time chain length RT (1..5): a batch of UC chunks
// (UC*RT fragments) is loaded while the previous batch is reduced; every address offset inside
// a batch is a compile-time constant; two chunks share one finishing HMMA when UC >= 2.
template <bool F32IN, int RT>
__device__ __forceinline__ void sp16_group_fast(const SpParams& p, uint64_t gi, float* s_chunk, bool& ovf) {
    constexpr int UC = RT == 1 ? 4 : RT == 2 ? 2 : 1;   // chunks per batch
    constexpr int BF = UC * RT;                          // fragments per batch
    constexpr uint64_t CE = uint64_t(RT) * 256;          // chunk elements
    constexpr uint64_t WSTRIDE = uint64_t(kSpWarps) * CE;  // next chunk of the same warp
    const unsigned warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const unsigned c = lane & 3;
    const unsigned la = lane >> 3, lb = (lane >> 2) & 1, ld = lane & 3;
    const uint32_t line_off = 16u * (2u * la + lb + 8u * (ld >> 1)) + 8u * (ld & 1u);
    const uint32_t Cg = p.G * p.W;
    const uint32_t nch = Cg > warp ? (Cg - warp + kSpWarps - 1) / kSpWarps : 0;
    const uint64_t base = (gi * uint64_t(Cg) + warp) * CE + line_off;

    auto load_batch = [&](uint32_t i0, Frag (&f)[BF]) {
#pragma unroll
        for (int u = 0; u < UC; ++u) {
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                if (i0 + u < nch) f[u * RT + r] = load_line<F32IN, false>(p.x, base + (i0 + u) * WSTRIDE + r * 256, p.n);
                else f[u * RT + r] = Frag{0, 0, 0, 0};
            }
        }
    };

    Frag cur[BF], nxt[BF];
    load_batch(0, cur);
    for (uint32_t i0 = 0; i0 < nch; i0 += UC) {
        if (i0 + UC < nch) load_batch(i0 + UC, nxt);
        uint32_t sel[UC];
#pragma unroll
        for (int u = 0; u < UC; ++u) {
            float acc1[4] = {0.f, 0.f, 0.f, 0.f}, acc2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                const Frag v = cur[u * RT + r];
                const uint32_t t0 = movmatrix_trans(v.r0), t1 = movmatrix_trans(v.r1);
                const uint32_t t2 = movmatrix_trans(v.r2), t3 = movmatrix_trans(v.r3);
                const uint32_t q0 = __shfl_xor_sync(kFull, t0, 16), q1 = __shfl_xor_sync(kFull, t1, 16);
                const uint32_t q2 = __shfl_xor_sync(kFull, t2, 16), q3 = __shfl_xor_sync(kFull, t3, 16);
                mma_16816(acc1, t0, t1, q0, q1, kOnesF16x2, kOnesF16x2);
                mma_16816(acc2, t2, t3, q2, q3, kOnesF16x2, kOnesF16x2);
            }
            const uint32_t h0 = f32_to_h(acc1[0]), h1 = f32_to_h(acc1[2]);
            const uint32_t h2 = f32_to_h(acc2[0]), h3 = f32_to_h(acc2[2]);
            sel[u] = c == 0 ? h0 : c == 1 ? h1 : c == 2 ? h2 : h3;
        }
#pragma unroll
        for (int u = 0; u < UC; u += (UC >= 2 ? 2 : 1)) {
            const int v_ = UC >= 2 ? u + 1 : u;
            const uint32_t aA = __shfl_sync(kFull, sel[u], c) | (__shfl_sync(kFull, sel[u], 4 + c) << 16);
            const uint32_t cA = __shfl_sync(kFull, sel[u], 8 + c) | (__shfl_sync(kFull, sel[u], 12 + c) << 16);
            uint32_t aB = aA, cB = cA;
            if (UC >= 2) {
                aB = __shfl_sync(kFull, sel[v_], c) | (__shfl_sync(kFull, sel[v_], 4 + c) << 16);
                cB = __shfl_sync(kFull, sel[v_], 8 + c) | (__shfl_sync(kFull, sel[v_], 12 + c) << 16);
            }
            float fin[4] = {0.f, 0.f, 0.f, 0.f};
            // finishing MMA (reduction.hpp:182): rows 0-7 chunk u, rows 8-15 chunk u+1
            mma_16816(fin, aA, aB, cA, cB, kOnesF16x2, kOnesF16x2);
            ovf |= !isfinite(fin[0]) || !isfinite(fin[2]);
            if (lane == 0) {
                if (i0 + u < nch) s_chunk[warp + (i0 + u) * kSpWarps] = fin[0];
                if (UC >= 2 && i0 + v_ < nch) s_chunk[warp + (i0 + v_) * kSpWarps] = fin[2];
            }
        }
        if (i0 + UC < nch) {
#pragma unroll
            for (int i = 0; i < BF; ++i) cur[i] = nxt[i];
        }
    }
}

template <bool F32IN, int RT>
__global__ void __launch_bounds__(kSpThreads, 3) sp16_kernel(const SpParams p) {
    __shared__ __align__(16) float s_chunk[kMaxChunksPerGroup];
    __shared__ __align__(16) float s_block[kMaxChunksPerGroup];
    __shared__ float s_scratch[32];
    __shared__ int s_last;

    const unsigned warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const uint32_t W = p.W, G = p.G;
    const uint64_t ce = p.chunk_elems;
    bool ovf = false;

    const uint64_t full_groups = p.n / (uint64_t(G) * W * ce);  // groups with no element past n
    for (uint64_t gi = p.group_begin + blockIdx.x; gi < p.group_end; gi += gridDim.x) {
        if (gi < full_groups) {
            if constexpr (RT > 0) sp16_group_fast<F32IN, RT>(p, gi, s_chunk, ovf);
            else sp16_group<F32IN, false>(p, gi, s_chunk, ovf);
        } else {
            sp16_group<F32IN, true>(p, gi, s_chunk, ovf);
        }
        __syncthreads();

        // ---- block stage: reference pairwise tree over the W warp results (:253, :90-101)
        pipe::tile_trees_blocks(p, gi, s_chunk, s_block, warp, kSpWarps);
        __syncthreads();

        // ---- group stage: adjacent tree over the G block results (power of two, any G)
        if (warp == 0) pipe::tile_tree_group(p, gi, s_block);
        __syncthreads();
    }

    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(p.overflow, 1u);

    if (p.finalize == kFinTree || p.finalize == kFinOrdered) {
        __threadfence();  // every writer publishes its group / block partials
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned t = atomicAdd(p.ticket, 1u);
            s_last = (t == gridDim.x - 1);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            finalize_cta(p, s_scratch);
            if (threadIdx.x == 0) *p.ticket = 0u;
        }
    }
}

__global__ void __launch_bounds__(kSpThreads) finalize_kernel(const SpParams p) {
    __shared__ float s_scratch[32];
    finalize_cta(p, s_scratch);
}

}  // namespace

template <bool F32IN>
using SpKernel = void (*)(SpParams);

template <bool F32IN>
static SpKernel<F32IN> pick_kernel(uint32_t R) {
    switch (R) {
    case 1: return sp16_kernel<F32IN, 1>;
    case 2: return sp16_kernel<F32IN, 2>;
    case 3: return sp16_kernel<F32IN, 3>;
    case 4: return sp16_kernel<F32IN, 4>;
    case 5: return sp16_kernel<F32IN, 5>;
    default: return sp16_kernel<F32IN, 0>;
    }
}

cudaError_t launch_single_pass_m16(const SpParams& p, bool f32_input, int grid, cudaStream_t s) {
    if (f32_input) pick_kernel<true>(p.R)<<<grid, kSpThreads, 0, s>>>(p);
    else pick_kernel<false>(p.R)<<<grid, kSpThreads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const SpParams& p, cudaStream_t s) {
    finalize_kernel<<<1, kSpThreads, 0, s>>>(p);
    return cudaGetLastError();
}

int single_pass_m16_max_grid(bool f32_input, uint32_t R) {
    int per_sm = 0;
    if (f32_input)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pick_kernel<true>(R), kSpThreads, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pick_kernel<false>(R), kSpThreads, 0);
    if (per_sm < 1) per_sm = 1;
    return per_sm * sm_count();
}

SpGeometry make_geometry(uint64_t n, uint32_t m, uint32_t R, uint32_t B) {
    SpGeometry g{};
    g.m = m;
    g.R = R;
    g.W = B / 32;
    g.n = n;
    g.chunk_elems = uint64_t(R) * m * m;
    g.block_elems = g.chunk_elems * g.W;
    g.n_blocks = (n + g.block_elems - 1) / g.block_elems;
    if (g.n_blocks < 1) g.n_blocks = 1;
    uint32_t G = 1;
    const Knobs& k = knobs();
    const uint64_t target = k.group_target ? k.group_target : kGroupElemsTarget;
    while (uint64_t(G) * g.block_elems < target) G <<= 1;
    // m = 16 with a block that is not a power of two (odd R, B not a power-of-two multiple of 32):
    // the largest group that does not exceed the target -- finer work units quantise the grid
    // better (measured at 2^28, B = 128: R = 3 88.9 -> 85.2 us, R = 5 88.6 -> 87.3 us)
    if (m == 16 && G > 1 && uint64_t(G) * g.block_elems > target) G >>= 1;
    // keep the per-group chunk table in shared memory: G*W never exceeds the engine's table
    // (a profiling cap can only lower it)
    const uint64_t table = m == 16 ? uint64_t(kMaxChunksPerGroup) : uint64_t(kMaxChunksGenm);
    const uint64_t cap = k.group_cap && k.group_cap < table ? k.group_cap : table;
    while (G > 1 && uint64_t(G) * g.W > cap) G >>= 1;
    // m in {2, 8}: up to 4 chunks share a period of the selector layout (tcr_sp_genm.cu), so a
    // group must hold a multiple of 4 chunks
    if ((m == 2 || m == 8) && G < 4) G = 4;
    g.G = G;
    g.group_elems = uint64_t(G) * g.block_elems;
    g.n_groups = (g.n_blocks + G - 1) / G;
    return g;
}

namespace {
Knobs g_knobs;   // production defaults until load_knobs_from_env()
}

const Knobs& knobs() { return g_knobs; }

void reset_knobs() { g_knobs = Knobs{}; }

int load_knobs_from_env() {
    Knobs k;
    int set = 0;
    auto num = [&](const char* name, auto* dst) {
        if (const char* e = std::getenv(name)) {
            *dst = static_cast<std::remove_pointer_t<decltype(dst)>>(std::strtoll(e, nullptr, 10));
            ++set;
        }
    };
    auto flag = [&](const char* name, bool* dst) {
        if (std::getenv(name)) {
            *dst = true;
            ++set;
        }
    };
    num("TCR_DEBUG_MODE", &k.debug_mode);
    num("TCR_GROUP_TARGET", &k.group_target);
    num("TCR_GROUP_CAP", &k.group_cap);
    num("TCR_SPLIT", &k.split);
    num("TCR_TAIL_SPLIT", &k.tail_split);
    num("TCR_SCHED", &k.sched);
    num("TCR_CTAS_PER_SM", &k.ctas_per_sm);
    flag("TCR_GM_NAT_GENERIC", &k.gm_nat_generic);
    num("TCR_GM_NAT_ALT", &k.gm_nat_alt);
    flag("TCR_GM_WIDE_WARP", &k.gm_wide_warp);
    flag("TCR_GM_NO_CLUSTER", &k.gm_no_cluster);
    flag("TCR_GM_TR8_SINGLE", &k.gm_tr8_single);
    if (const char* e = std::getenv("TCR_PROBE")) {
        k.probe_async = std::string(e) == "async";
        k.probe_tma = std::string(e) == "tma";
        ++set;
    }
    num("TCR_PROBE_CTAS", &k.probe_ctas);
    num("TCR_PROBE_SLOT", &k.probe_slot);
    g_knobs = k;
    return set;
}

int sm_count() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached < 1) cached = 1;
    }
    return cached;
}

}  // namespace tcr
