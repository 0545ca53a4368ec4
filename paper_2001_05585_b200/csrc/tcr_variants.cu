// tcr_variants.cu -- the other Variants of the reference's reduce() dispatcher on the device.
//
//   shuffle32  reduction.hpp:113-122  whole-array fp32 pairwise tree, v[i] += v[i + len/2]
//   half_tree  reduction.hpp:126-151  same tree, every partial stored through binary16
//   oracle64   reduction.hpp:106-110  binary64 sum
//   (recurrence and split are composed on the host side of the C ABI from the single_pass
//    kernels and these.)
//
// The strided pairwise tree is reproduced BIT-FOR-BIT: after s levels, slot i holds the strided
// subtree over x[i + k*S] (S = P / 2^s), and a strided tree over k is the adjacent tree over the
// bit-reversed k.  Phase 1 lets every thread stream one column i through a binary-counter stack
// in bit-reversed row order (each step reads one contiguous row of S values: coalesced), phase 2
// repeats the construction over the S column results inside one CTA and finishes with the
// classic in-shared-memory strided levels.  Zero padding to P = pow2(n) is implicit.
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

// binary64 sum (oracle64): fixed thread -> element assignment, fixed-order trees: deterministic.
template <typename T>
__global__ void __launch_bounds__(256) dsum_kernel(const T* x, uint64_t n, double* partials, uint32_t* ticket,
                                                   double* out) {
    double acc = 0.0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        if constexpr (sizeof(T) == 2) acc += double(h_to_f32(x[i]));
        else acc += double(x[i]);
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(kFull, acc, off);
    __shared__ double sw[8];
    __shared__ int s_last;
    if (lane_id() == 0) sw[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < 8; ++w) b += sw[w];
        partials[blockIdx.x] = b;
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        double t = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) t += __ldcg(partials + b);
        *out = t;
        *ticket = 0u;
    }
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
cudaError_t tree_impl(const T* x, uint64_t n, float* cols, uint64_t cols_cap, float* out, uint32_t* ovf,
                      cudaStream_t s) {
    uint64_t P = 1;
    while (P < n) P <<= 1;
    const uint64_t S = P < cols_cap ? P : cols_cap;   // columns of phase 1 (power of two)
    if (P <= kTreeThreads * 64ull) {
        tree_phase2<T, HALF><<<1, kTreeThreads, 0, s>>>(x, n, P, out, ovf);
        return cudaGetLastError();
    }
    const uint64_t blocks = (S + 255) / 256;
    tree_phase1<T, HALF><<<unsigned(blocks), 256, 0, s>>>(x, n, S, P / S, cols, ovf);
    tree_phase2<float, HALF><<<1, kTreeThreads, 0, s>>>(cols, S, S, out, ovf);
    return cudaGetLastError();
}

}  // namespace

uint64_t tree_cols_needed() { return 1ull << 18; }

cudaError_t launch_pairwise_tree(const void* x, bool f32, uint64_t n, bool half, float* cols, float* out,
                                 uint32_t* ovf, cudaStream_t s) {
    const uint64_t cap = tree_cols_needed();
    if (f32) {
        return half ? tree_impl<float, true>(static_cast<const float*>(x), n, cols, cap, out, ovf, s)
                    : tree_impl<float, false>(static_cast<const float*>(x), n, cols, cap, out, ovf, s);
    }
    return half ? tree_impl<uint16_t, true>(static_cast<const uint16_t*>(x), n, cols, cap, out, ovf, s)
                : tree_impl<uint16_t, false>(static_cast<const uint16_t*>(x), n, cols, cap, out, ovf, s);
}

cudaError_t launch_dsum(const void* x, bool f32, uint64_t n, double* partials, uint32_t* ticket, double* out,
                        cudaStream_t s) {
    const int grid = sm_count() * 4;
    if (f32) dsum_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), n, partials, ticket, out);
    else dsum_kernel<uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(x), n, partials, ticket, out);
    return cudaGetLastError();
}

cudaError_t launch_round_level(const float* in, uint16_t* out, uint64_t count, uint32_t* ovf, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    uint64_t blocks = (count + 255) / 256;
    if (blocks > uint64_t(sm_count()) * 8) blocks = uint64_t(sm_count()) * 8;
    round_level_kernel<<<unsigned(blocks), 256, 0, s>>>(in, out, count, ovf);
    return cudaGetLastError();
}

}  // namespace tcr
