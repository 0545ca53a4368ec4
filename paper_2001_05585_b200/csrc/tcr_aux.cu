// tcr_aux.cu -- input generation, exact sums and the GPU comparison points.
//
//  * generate: harness.hpp:47-80 (SplitMix64 rng.hpp:9-26) with jump-ahead, so every
//    thread produces its own elements; binary16 output is the reference's from_single.
//  * exact sum: fixed-point (2^-24 units) 128-bit sum of binary16 values -- the error
//    reference at any n, computed on the device.
//  * shuffle: the paper's CUDA-core baseline -- fp32 warp-shuffle reduction.
//  * read probe: streaming-read ceiling used for the roofline.
//  * CUB DeviceReduce::Sum (half -> float) and (half -> half): the library comparators.
#include <cub/device/device_reduce.cuh>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tcr_device.cuh"
#include "tcr_kernels.h"
#include "tcr_pipeline.cuh"

namespace tcr {

namespace {

// --------------------------------------------------------------------------- generate

__device__ __forceinline__ float gen_value(int kind, uint64_t seed, int64_t lo, uint64_t span,
                                           double c, uint64_t g) {
    switch (kind) {
    case 3:  // constant
        return float(c);
    case 1:  // uniform: (float)((next() >> 11) * 2^-53), element g uses draw g+1
        return float(double(splitmix_draw(seed, g + 1) >> 11) * 0x1.0p-53);
    case 2:  // integers: lo + next() % span
        return float(lo + (long long)(splitmix_draw(seed, g + 1) % span));
    default: {  // normal: Box-Muller on draws 2p+1 (open unit) and 2p+2
        const uint64_t pr = g >> 1;
        const double u1 = double((splitmix_draw(seed, 2 * pr + 1) >> 11) + 1) * 0x1.0p-53;
        const double u2 = double(splitmix_draw(seed, 2 * pr + 2) >> 11) * 0x1.0p-53;
        const double r = sqrt(-2.0 * log(u1));
        const double t = 2.0 * 3.141592653589793 * u2;
        return float((g & 1) ? r * sin(t) : r * cos(t));
    }
    }
}

template <bool F16OUT>
__global__ void gen_kernel(void* out, uint64_t count, int kind, uint64_t seed, int64_t lo,
                           uint64_t span, double c, uint64_t first) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const float v = gen_value(kind, seed, lo, span, c, first + i);
        if constexpr (F16OUT) static_cast<uint16_t*>(out)[i] = f32_to_h(v);
        else static_cast<float*>(out)[i] = v;
    }
}

// -------------------------------------------------------------------------- exact sum

struct I128 {
    unsigned long long lo;
    long long hi;
};

__device__ __forceinline__ void add128(I128& a, long long v) {
    const unsigned long long old = a.lo;
    a.lo += (unsigned long long)v;
    a.hi += (v < 0 ? -1 : 0) + (a.lo < old ? 1 : 0);
}

__device__ __forceinline__ void add128(I128& a, const I128& b) {
    const unsigned long long old = a.lo;
    a.lo += b.lo;
    a.hi += b.hi + (a.lo < old ? 1 : 0);
}

// binary16 -> signed multiple of 2^-24 (exact; |v| < 2^40)
__device__ __forceinline__ long long h_fixed(uint16_t h) {
    const uint32_t e = (h >> 10) & 31u, m = h & 1023u;
    const long long mag = e == 0 ? (long long)m : (long long)(1024u + m) << (e - 1);
    return (h & 0x8000u) ? -mag : mag;
}

constexpr int kExactThreads = 256;
constexpr int kExactGrid = 1184;  // 8 per SM on 148 SMs

struct ExactWs {
    I128 sum[kExactGrid];
    I128 abs[kExactGrid];
    unsigned long long nonfinite[kExactGrid];
    double nf_sum[kExactGrid];
};

__global__ void __launch_bounds__(kExactThreads) exact_kernel(const uint16_t* x, uint64_t n, ExactWs* ws) {
    I128 s{0, 0}, a{0, 0};
    unsigned long long nf = 0;
    double nfs = 0.0;
    // 64-bit per-thread accumulators, flushed to 128-bit every 2^20 elements (< 2^60)
    long long ls = 0, la = 0;
    uint32_t cnt = 0;
    const uint64_t n8 = n / 8;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += stride) {
        const uint4 v = ldg_stream_v4(x + 8 * i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const uint16_t h = uint16_t(w[q] >> (16 * hh));
                if (h_overflowed(h)) {
                    ++nf;
                    nfs += double(h_to_f32(h));
                } else {
                    const long long f = h_fixed(h);
                    ls += f;
                    la += f < 0 ? -f : f;
                }
            }
        }
        if (++cnt == (1u << 17)) {
            add128(s, ls);
            add128(a, la);
            ls = la = 0;
            cnt = 0;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 7)) {
        const uint16_t h = x[8 * n8 + threadIdx.x];
        if (h_overflowed(h)) {
            ++nf;
            nfs += double(h_to_f32(h));
        } else {
            const long long f = h_fixed(h);
            ls += f;
            la += f < 0 ? -f : f;
        }
    }
    add128(s, ls);
    add128(a, la);
    // block reduction (128-bit)
    __shared__ I128 ss[kExactThreads], sa[kExactThreads];
    __shared__ unsigned long long snf[kExactThreads];
    __shared__ double snfs[kExactThreads];
    ss[threadIdx.x] = s;
    sa[threadIdx.x] = a;
    snf[threadIdx.x] = nf;
    snfs[threadIdx.x] = nfs;
    __syncthreads();
    for (int off = kExactThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < unsigned(off)) {
            add128(ss[threadIdx.x], ss[threadIdx.x + off]);
            add128(sa[threadIdx.x], sa[threadIdx.x + off]);
            snf[threadIdx.x] += snf[threadIdx.x + off];
            snfs[threadIdx.x] += snfs[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ws->sum[blockIdx.x] = ss[0];
        ws->abs[blockIdx.x] = sa[0];
        ws->nonfinite[blockIdx.x] = snf[0];
        ws->nf_sum[blockIdx.x] = snfs[0];
    }
}

__device__ double i128_to_double_scaled(I128 v) {
    // value * 2^-24, one final rounding is enough for reporting purposes
    const bool neg = v.hi < 0;
    if (neg) {
        v.lo = ~v.lo + 1ull;
        v.hi = ~v.hi + (v.lo == 0 ? 1 : 0);
    }
    const double d = ldexp(double((unsigned long long)v.hi), 64) + double(v.lo);
    return (neg ? -d : d) * 0x1.0p-24;
}

__global__ void exact_finish_kernel(const ExactWs* ws, int grid, double* out3) {
    if (threadIdx.x != 0) return;
    I128 s{0, 0}, a{0, 0};
    unsigned long long nf = 0;
    double nfs = 0.0;
    for (int b = 0; b < grid; ++b) {
        add128(s, ws->sum[b]);
        add128(a, ws->abs[b]);
        nf += ws->nonfinite[b];
        nfs += ws->nf_sum[b];
    }
    if (nf) {
        out3[0] = nfs;
        out3[1] = __longlong_as_double(0x7FF0000000000000ll);
        out3[2] = double(nf);
    } else {
        out3[0] = i128_to_double_scaled(s);
        out3[1] = i128_to_double_scaled(a);
        out3[2] = 0.0;
    }
}

// -------------------------------------------------------------------- shuffle baseline

constexpr int kShThreads = 256;

__global__ void __launch_bounds__(kShThreads) shuffle_kernel(const uint16_t* x, uint64_t n, float* partials,
                                                             uint32_t* ticket, float* result) {
    // classic CUDA-core reduction: per-thread fp32 sums of binary16 loads (4 x 16 B in flight),
    // __shfl_down warp tree, shared-memory block tree, last-block-done grid finaliser.
    float acc = 0.0f;
    const uint64_t n8 = n / 8;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n8; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ldg_stream_v4(x + 8 * (i + u * stride));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const __half2* h = reinterpret_cast<const __half2*>(&v[u]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 f = __half22float2(h[q]);
                acc += f.x;
                acc += f.y;
            }
        }
    }
    for (; i < n8; i += stride) {
        const uint4 v = ldg_stream_v4(x + 8 * i);
        const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 f = __half22float2(h[q]);
            acc += f.x;
            acc += f.y;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 7)) acc += h_to_f32(x[8 * n8 + threadIdx.x]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(kFull, acc, off);
    __shared__ float sw[kShThreads / 32];
    __shared__ int s_last;
    if (lane_id() == 0) sw[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < kShThreads / 32 ? sw[threadIdx.x] : 0.0f;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(kFull, v, off);
        if (threadIdx.x == 0) {
            partials[blockIdx.x] = v;
            __threadfence();
            s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (s_last && threadIdx.x < 32) {
        __threadfence();
        float v = 0.0f;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) v += __ldcg(partials + b);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(kFull, v, off);
        if (threadIdx.x == 0) {
            *result = v;
            *ticket = 0u;
        }
    }
}

// ------------------------------------------------------------------------- read probe

__global__ void __launch_bounds__(256) read_probe_kernel(const uint4* x, uint64_t n16, uint32_t* sink) {
    uint32_t acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ldg_stream_v4(x + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) {
        const uint4 v = ldg_stream_v4(x + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9E3779B9u) sink[0] = acc;  // practically never taken; keeps the loads live
}

__global__ void convert_kernel(const float* in, uint16_t* out, uint64_t count) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) out[i] = f32_to_h(in[i]);
}

// Streaming-read probe through cp.async (LDGSTS) instead of LDG: same grid-stride 512-byte
// warp rows, a per-warp 8-stage shared-memory ring (profiling: the LDGSTS path's ceiling).
__global__ void __launch_bounds__(256) read_probe_async_kernel(const uint4* x, uint64_t n16, uint32_t* sink) {
    __shared__ __align__(128) uint4 ring[8][8][32];
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const uint64_t TW = uint64_t(gridDim.x) * 8;
    const uint64_t gw = uint64_t(blockIdx.x) * 8 + warp;
    const uint64_t rows = n16 / 32;
    uint32_t acc = 0;
    auto issue = [&](uint64_t k) {
        const uint64_t row = gw + k * TW;
        if (row < rows) {
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&ring[warp][k & 7][lane]));
            asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(dst), "l"(x + row * 32 + lane) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int k = 0; k < 7; ++k) issue(uint64_t(k));
    for (uint64_t k = 0; gw + k * TW < rows; ++k) {
        issue(k + 7);
        asm volatile("cp.async.wait_group 7;" ::: "memory");
        const uint4 v = ring[warp][k & 7][lane];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (acc == 0x9E3779B9u) sink[0] = acc;
}

// Streaming-read probe through 1-D TMA (cp.async.bulk): each CTA streams one contiguous range
// in `slot`-byte copies through an NSLOT ring, one producer thread, one consumer warp touching
// one word per slot (profiling: the bulk-copy path's ceiling with large copies).
template <int NSLOT>
__global__ void __launch_bounds__(64) read_probe_tma_kernel(const char* x, uint64_t bytes, uint32_t slot, uint32_t* sink) {
    extern __shared__ __align__(128) unsigned char pring[];
    __shared__ uint64_t full[NSLOT], empty[NSLOT];
    const uint64_t per = (bytes / gridDim.x) & ~uint64_t(15);
    const uint64_t b0 = per * blockIdx.x, b1 = blockIdx.x + 1 == gridDim.x ? (bytes & ~uint64_t(15)) : b0 + per;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSLOT; ++i) {
            pipe::mbar_init(&full[i], 1);
            pipe::mbar_init(&empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    uint32_t acc = 0;
    uint32_t t = 0;
    for (uint64_t off = b0; off < b1; off += slot, ++t) {
        const uint32_t si = t % NSLOT, ph = (t / NSLOT) & 1u;
        const uint32_t sz = uint32_t(min(uint64_t(slot), b1 - off));
        if (warp == 0) {
            if (lane == 0) {
                pipe::mbar_wait(&empty[si], ph ^ 1u);
                pipe::mbar_expect_tx(&full[si], sz);
                pipe::bulk_load_1d(pring + size_t(si) * slot, x + off, sz, &full[si], pipe::evict_first_policy());
            }
        } else {
            pipe::mbar_wait(&full[si], ph);
            if (lane == 0) {
                acc ^= *reinterpret_cast<const uint32_t*>(pring + size_t(si) * slot);
                pipe::mbar_arrive(&empty[si]);
            }
        }
    }
    if (acc == 0x9E3779B9u) sink[0] = acc;
}

}  // namespace

cudaError_t launch_read_probe_tma(const void* x, uint64_t bytes, uint32_t* sink, int grid, uint32_t slot, cudaStream_t s) {
    const uint32_t nslot = 4;
    const uint32_t smem = nslot * slot;
    cudaFuncSetAttribute(read_probe_tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    read_probe_tma_kernel<4><<<grid, 64, smem, s>>>(static_cast<const char*>(x), bytes, slot, sink);
    return cudaGetLastError();
}

cudaError_t launch_read_probe_async(const void* x, uint64_t bytes, uint32_t* sink, int grid, cudaStream_t s) {
    read_probe_async_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(x), bytes / 16, sink);
    return cudaGetLastError();
}

cudaError_t launch_convert_f32_f16(const float* in, uint16_t* out, uint64_t count, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    uint64_t blocks = (count + 255) / 256;
    const uint64_t cap = uint64_t(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    convert_kernel<<<unsigned(blocks), 256, 0, s>>>(in, out, count);
    return cudaGetLastError();
}

cudaError_t launch_generate(void* out, bool f16_out, uint64_t count, int kind, uint64_t seed, int64_t lo,
                            int64_t hi, double c, uint64_t first, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    const uint64_t span = uint64_t(hi - lo) + 1;
    uint64_t blocks = (count + 255) / 256;
    const uint64_t cap = uint64_t(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    if (f16_out) gen_kernel<true><<<unsigned(blocks), 256, 0, s>>>(out, count, kind, seed, lo, span, c, first);
    else gen_kernel<false><<<unsigned(blocks), 256, 0, s>>>(out, count, kind, seed, lo, span, c, first);
    return cudaGetLastError();
}

size_t exact_ws_bytes() { return sizeof(ExactWs); }

cudaError_t launch_exact_sum_f16(const uint16_t* x, uint64_t n, void* ws, double* d_out3, cudaStream_t s) {
    exact_kernel<<<kExactGrid, kExactThreads, 0, s>>>(x, n, static_cast<ExactWs*>(ws));
    exact_finish_kernel<<<1, 32, 0, s>>>(static_cast<const ExactWs*>(ws), kExactGrid, d_out3);
    return cudaGetLastError();
}

int shuffle_max_grid() {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, shuffle_kernel, kShThreads, 0);
    if (per_sm < 1) per_sm = 1;
    return per_sm * sm_count();
}

cudaError_t launch_shuffle_f16(const uint16_t* x, uint64_t n, float* partials, uint32_t* ticket, float* result,
                               int grid, cudaStream_t s) {
    shuffle_kernel<<<grid, kShThreads, 0, s>>>(x, n, partials, ticket, result);
    return cudaGetLastError();
}

cudaError_t launch_read_probe(const void* x, uint64_t bytes, uint32_t* sink, int grid, cudaStream_t s) {
    read_probe_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(x), bytes / 16, sink);
    return cudaGetLastError();
}

// fp32 accumulation of binary16 input: CUB's Sum(const __half*, float*) semantics
// (device_reduce.cuh: the accumulator is the output type).
struct HalfToFloatSum {
    __device__ __forceinline__ float operator()(float a, float b) const { return a + b; }
    __device__ __forceinline__ float operator()(float a, __half b) const { return a + __half2float(b); }
    __device__ __forceinline__ float operator()(__half a, float b) const { return __half2float(a) + b; }
    __device__ __forceinline__ float operator()(__half a, __half b) const { return __half2float(a) + __half2float(b); }
};

size_t cub_temp_bytes(uint64_t n, bool half_out) {
    size_t bytes = 0;
    const __half* in = nullptr;
    if (half_out) {
        __half* out = nullptr;
        cub::DeviceReduce::Sum(nullptr, bytes, in, out, (int64_t)n);
    } else {
        float* out = nullptr;
        cub::DeviceReduce::Reduce(nullptr, bytes, in, out, (int64_t)n, HalfToFloatSum{}, 0.0f);
    }
    return bytes;
}

cudaError_t cub_sum_f16(const uint16_t* x, uint64_t n, void* out, bool half_out, void* temp, size_t temp_bytes,
                        cudaStream_t s) {
    const __half* in = reinterpret_cast<const __half*>(x);
    if (half_out)
        return cub::DeviceReduce::Sum(temp, temp_bytes, in, static_cast<__half*>(out), (int64_t)n, s);
    return cub::DeviceReduce::Reduce(temp, temp_bytes, in, static_cast<float*>(out), (int64_t)n, HalfToFloatSum{},
                                     0.0f, s);
}

}  // namespace tcr
