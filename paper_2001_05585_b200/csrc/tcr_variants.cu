// tcr_variants.cu -- the other Variants of the reference's reduce() dispatcher on the device.
//
//   shuffle32  reduction.hpp:113-122  whole-array fp32 pairwise tree, v[i] += v[i + len/2]
//   half_tree  reduction.hpp:126-151  same tree, every partial stored through binary16
//   (recurrence and split are composed on the host side of the C ABI from the single_pass
//    kernels and these.)
//
// The strided pairwise tree is reproduced BIT-FOR-BIT.  Viewing the P = pow2(n) zero-padded
// values as K rows of S = P / K columns (x[i + k S]), the first log2(K) levels of the tree
// (len = P ... 2S) pair rows k and k + len/(2S) of the SAME column, so they are a strided tree
// over the K rows of every column; what is left is the same problem on the S column results.
// Row phases (tree_rows_kernel): each thread owns 16 bytes of adjacent columns, streams its K rows
// with cp.async (coalesced rows) and runs the K-row strided tree in registers;
// phases repeat (K = 16: P -> P/16) until <= 64 Ki values remain, which one CTA finishes
// (per-thread binary-counter stacks in bit-reversed row order, then the in-shared-memory
// strided levels).  Zero padding is implicit (loads beyond n read 0).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tcr_device.cuh"
#include "tcr_kernels.h"

namespace tcr {

namespace {

constexpr int kTreeThreads = 1024;

template <bool HALF>
__device__ __forceinline__ float tree_add(float a, float b, bool& ovf) {
    if constexpr (HALF) {
        const uint16_t h = f32_to_h(a + b);   // from_single(v[i] + v[i + len/2]) (:140)
        ovf |= h_overflowed(h);
        return h_to_f32(h);                   // to_single (:142)
    } else {
        return a + b;
    }
}

template <typename T, bool HALF>
__device__ __forceinline__ float tree_load(const T* x, uint64_t idx, uint64_t n, bool& ovf) {
    if (idx >= n) return 0.0f;
    float v;
    if constexpr (sizeof(T) == 2) v = h_to_f32(x[idx]);
    else v = x[idx];
    if constexpr (HALF) {
        const uint16_t h = f32_to_h(v);       // inputs pass through binary16 (:131-134)
        ovf |= h_overflowed(h);
        v = h_to_f32(h);
    }
    return v;
}

__device__ __forceinline__ uint64_t bitrev(uint64_t j, int bits) {
    return bits == 0 ? 0 : (__brevll(j) >> (64 - bits));
}

// Strided subtree over `count` (power of two) values vals(i + k*stride), k = 0..count-1, for column i.
template <typename T, bool HALF>
__device__ float column_tree(const T* x, uint64_t n, uint64_t col, uint64_t stride, uint64_t count, bool& ovf) {
    int bits = 0;
    while ((1ull << bits) < count) ++bits;
    float stk[48];
    int top = 0;
    for (uint64_t j = 0; j < count; ++j) {
        float v = tree_load<T, HALF>(x, col + bitrev(j, bits) * stride, n, ovf);
        for (uint64_t b = j; b & 1; b >>= 1) v = tree_add<HALF>(stk[--top], v, ovf);
        stk[top++] = v;
    }
    return stk[0];
}

template <typename T, bool HALF>
__global__ void __launch_bounds__(256) tree_phase1(const T* x, uint64_t n, uint64_t S, uint64_t K, float* cols,
                                                   uint32_t* ovf_flag) {
    bool ovf = false;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < S; i += uint64_t(gridDim.x) * blockDim.x)
        cols[i] = column_tree<T, HALF>(x, n, i, S, K, ovf);
    if (__any_sync(kFull, ovf) && lane_id() == 0) atomicOr(ovf_flag, 1u);
}

// One CTA: strided tree over vals[0, S) (S a power of two, entries beyond `valid` are zero).
template <typename T, bool HALF>
__global__ void __launch_bounds__(kTreeThreads) tree_phase2(const T* vals, uint64_t valid, uint64_t S, float* out,
                                                            uint32_t* ovf_flag) {
    __shared__ float v[kTreeThreads];
    bool ovf = false;
    const uint64_t T_ = S < kTreeThreads ? S : kTreeThreads;
    if (threadIdx.x < T_) v[threadIdx.x] = column_tree<T, HALF>(vals, valid, threadIdx.x, T_, S / T_, ovf);
    __syncthreads();
    for (uint64_t len = T_; len > 1; len >>= 1) {
        float r = 0.0f;
        if (threadIdx.x < len / 2) r = tree_add<HALF>(v[threadIdx.x], v[threadIdx.x + len / 2], ovf);
        __syncthreads();
        if (threadIdx.x < len / 2) v[threadIdx.x] = r;
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = v[0];
    if (__any_sync(kFull, ovf) && lane_id() == 0) atomicOr(ovf_flag, 1u);
}

// One row phase: K rows x S columns of `x` (entries >= valid are zero) -> out[S].  A thread
// tile = 16 bytes of columns (CW = 8 binary16 or 4 fp32) x K rows, streamed by cp.async into a
// per-thread slot of a 3-deep shared-memory ring (no register cost for loads in flight, zero
// fill past `valid`), then reduced column by column in registers.
constexpr int kRowK = 16, kRowThreads = 128, kRowDepth = 3;

__device__ __forceinline__ void cp16_zfill(uint32_t saddr, const void* g, uint32_t bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(bytes) : "memory");
}

template <typename T, bool HALF>
__global__ void __launch_bounds__(kRowThreads) tree_rows_kernel(const T* x, uint64_t valid, uint64_t S, float* out,
                                                                uint32_t* ovf_flag) {
    constexpr int CW = 16 / sizeof(T);
    extern __shared__ __align__(16) unsigned char s_rows[];   // [kRowDepth][kRowK][kRowThreads][16 B]
    bool ovf = false;
    const uint64_t tiles = S / CW;
    const uint64_t step = uint64_t(gridDim.x) * kRowThreads;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(s_rows)) + threadIdx.x * 16u;
    auto issue = [&](uint64_t t, int slot) {
        if (t < tiles) {
            const uint64_t c0 = t * CW;
#pragma unroll
            for (int k = 0; k < kRowK; ++k) {
                const uint64_t e = c0 + uint64_t(k) * S;
                const uint32_t bytes = e + CW <= valid ? 16u : (e < valid ? uint32_t(valid - e) * sizeof(T) : 0u);
                cp16_zfill(base + uint32_t((slot * kRowK + k) * kRowThreads) * 16u, x + (e < valid ? e : 0), bytes);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    uint64_t t = uint64_t(blockIdx.x) * kRowThreads + threadIdx.x;
#pragma unroll
    for (int d = 0; d < kRowDepth - 1; ++d) issue(t + uint64_t(d) * step, d);
    int slot = 0;
    for (; t < tiles; t += step) {
        issue(t + uint64_t(kRowDepth - 1) * step, (slot + kRowDepth - 1) % kRowDepth);
        asm volatile("cp.async.wait_group %0;" ::"n"(kRowDepth - 1) : "memory");
        const uint4* row = reinterpret_cast<const uint4*>(s_rows) + (slot * kRowK) * kRowThreads + threadIdx.x;
        uint4 r[kRowK];
#pragma unroll
        for (int k = 0; k < kRowK; ++k) r[k] = row[k * kRowThreads];
        float res[CW];
        if constexpr (sizeof(T) == 2 && HALF) {
            // half_tree on binary16 input: from_single(a + b) of two binary16 values equals the
            // native round-to-nearest binary16 add (an fp32 intermediate has 24 >= 2*11 + 2
            // significand bits, so the double rounding is innocuous), and inf / NaN propagate to
            // the column result, so packed HADD2 trees reproduce the reference bit for bit and a
            // non-finite column result is exactly "some partial overflowed" (:136-146).
            __half2 hv[kRowK][4];
#pragma unroll
            for (int k = 0; k < kRowK; ++k) {
                hv[k][0] = *reinterpret_cast<const __half2*>(&r[k].x);
                hv[k][1] = *reinterpret_cast<const __half2*>(&r[k].y);
                hv[k][2] = *reinterpret_cast<const __half2*>(&r[k].z);
                hv[k][3] = *reinterpret_cast<const __half2*>(&r[k].w);
            }
#pragma unroll
            for (int h = kRowK / 2; h >= 1; h >>= 1)
#pragma unroll
                for (int k = 0; k < h; ++k)
#pragma unroll
                    for (int q = 0; q < 4; ++q) hv[k][q] = __hadd2(hv[k][q], hv[k + h][q]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 f = __half22float2(hv[0][q]);
                res[2 * q] = f.x;
                res[2 * q + 1] = f.y;
                ovf |= !isfinite(f.x) || !isfinite(f.y);
            }
        } else
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            float v[kRowK];
#pragma unroll
            for (int k = 0; k < kRowK; ++k) {
                const uint32_t w = (&r[k].x)[sizeof(T) == 2 ? c / 2 : c];
                if constexpr (sizeof(T) == 2) {
                    const uint16_t h = uint16_t((c & 1) ? (w >> 16) : (w & 0xFFFFu));
                    if constexpr (HALF) ovf |= h_overflowed(h);
                    v[k] = h_to_f32(h);
                } else {
                    v[k] = __uint_as_float(w);
                    if constexpr (HALF) {
                        const uint16_t h = f32_to_h(v[k]);   // inputs through binary16 (:131-134)
                        ovf |= h_overflowed(h);
                        v[k] = h_to_f32(h);
                    }
                }
            }
#pragma unroll
            for (int h = kRowK / 2; h >= 1; h >>= 1)
#pragma unroll
                for (int k = 0; k < h; ++k) v[k] = tree_add<HALF>(v[k], v[k + h], ovf);
            res[c] = v[0];
        }
        float4* o = reinterpret_cast<float4*>(out + t * CW);
#pragma unroll
        for (int q = 0; q < CW / 4; ++q) o[q] = make_float4(res[4 * q], res[4 * q + 1], res[4 * q + 2], res[4 * q + 3]);
        slot = slot + 1 == kRowDepth ? 0 : slot + 1;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (__any_sync(kFull, ovf) && lane_id() == 0) atomicOr(ovf_flag, 1u);
}

// fp32 level results -> binary16 next-level input with the overflow note (reduction.hpp:205-207)
__global__ void round_level_kernel(const float* in, uint16_t* out, uint64_t count, uint32_t* ovf_flag) {
    bool ovf = false;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint16_t h = f32_to_h(in[i]);
        ovf |= h_overflowed(h);
        out[i] = h;
    }
    if (__any_sync(kFull, ovf) && lane_id() == 0) atomicOr(ovf_flag, 1u);
}

template <typename T, bool HALF>
cudaError_t launch_rows(const T* x, uint64_t valid, uint64_t S, float* out, uint32_t* ovf, cudaStream_t s) {
    constexpr uint32_t dyn = kRowDepth * kRowK * kRowThreads * 16u;
    static PerDeviceOnce once;   // per instantiation
    const cudaError_t ea = once([] {
        return cudaFuncSetAttribute(tree_rows_kernel<T, HALF>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
    });
    if (ea != cudaSuccess) return ea;
    const uint64_t tiles = S / (16 / sizeof(T));
    const uint64_t b = (tiles + kRowThreads - 1) / kRowThreads, cap = uint64_t(sm_count()) * 2;
    tree_rows_kernel<T, HALF><<<unsigned(b < cap ? b : cap), kRowThreads, dyn, s>>>(x, valid, S, out, ovf);
    return cudaGetLastError();
}

template <typename T, bool HALF>
cudaError_t tree_impl(const T* x, uint64_t n, float* cols, float* out, uint32_t* ovf, cudaStream_t s) {
    uint64_t P = 1;
    while (P < n) P <<= 1;
    if (P <= kTreeThreads * 64ull) {
        tree_phase2<T, HALF><<<1, kTreeThreads, 0, s>>>(x, n, P, out, ovf);
        return cudaGetLastError();
    }
    // first row phase reads the input (binary16 or fp32); later phases read fp32 column results
    uint64_t S = P / kRowK;
    float* buf[2] = {cols, cols + S};
    cudaError_t e = launch_rows<T, HALF>(x, n, S, buf[0], ovf, s);
    if (e != cudaSuccess) return e;
    int b = 0;
    while (S > kTreeThreads * 64ull) {
        const uint64_t S2 = S / kRowK;
        e = launch_rows<float, HALF>(buf[b], S, S2, buf[b ^ 1], ovf, s);
        if (e != cudaSuccess) return e;
        b ^= 1;
        S = S2;
    }
    tree_phase2<float, HALF><<<1, kTreeThreads, 0, s>>>(buf[b], S, S, out, ovf);
    return cudaGetLastError();
}

}  // namespace

int tree_launches(uint64_t n) {
    uint64_t P = 1;
    while (P < n) P <<= 1;
    if (P <= kTreeThreads * 64ull) return 1;
    int k = 2;   // first row phase + the one-CTA finish
    for (uint64_t S = P / kRowK; S > kTreeThreads * 64ull; S /= kRowK) ++k;
    return k;
}

uint64_t tree_cols_needed(uint64_t n) {
    uint64_t P = 1;
    while (P < n) P <<= 1;
    return P / kRowK + P / (kRowK * kRowK) + 64;   // ping-pong column buffers of the row phases
}

cudaError_t launch_pairwise_tree(const void* x, bool f32, uint64_t n, bool half, float* cols, float* out,
                                 uint32_t* ovf, cudaStream_t s) {
    if (f32) {
        return half ? tree_impl<float, true>(static_cast<const float*>(x), n, cols, out, ovf, s)
                    : tree_impl<float, false>(static_cast<const float*>(x), n, cols, out, ovf, s);
    }
    return half ? tree_impl<uint16_t, true>(static_cast<const uint16_t*>(x), n, cols, out, ovf, s)
                : tree_impl<uint16_t, false>(static_cast<const uint16_t*>(x), n, cols, out, ovf, s);
}


cudaError_t launch_round_level(const float* in, uint16_t* out, uint64_t count, uint32_t* ovf, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    uint64_t blocks = (count + 255) / 256;
    if (blocks > uint64_t(sm_count()) * 8) blocks = uint64_t(sm_count()) * 8;
    round_level_kernel<<<unsigned(blocks), 256, 0, s>>>(in, out, count, ovf);
    return cudaGetLastError();
}

}  // namespace tcr
