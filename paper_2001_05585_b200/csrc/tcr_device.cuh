// tcr_device.cuh -- sm_100a device primitives shared by the tcreduce kernels.
//
// Everything here is inline PTX for the B200 (compute_100a): warp-level
// movmatrix / mma.sync, binary16 conversion, cache-hinted vector loads.
#pragma once

#include <cstdint>
#include <cuda_fp16.h>

namespace tcr {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kOnesF16x2 = 0x3C003C00u;  // two binary16 1.0

// 16-byte streaming load: read-only path, do not allocate in L1 (every byte is read once).
__device__ __forceinline__ uint4 ldg_stream_v4(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ float4 ldg_stream_f4(const void* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

// In-register 8x8 transpose of binary16 elements across the warp (SASS: MOVM).
// Thread l supplies M[l/4][2(l%4)..+1] and receives M^T[l/4][2(l%4)..+1].
__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}

// D = A(16x16 f16) * B(16x8 f16) + C(16x8 f32)   (SASS: HMMA.16816.F32)
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// fp32 -> binary16 round-to-nearest-even (cvt.rn.f16.f32): bit-identical to the
// reference from_single (half.hpp:32-59) for every non-NaN input, subnormals included.
__device__ __forceinline__ uint16_t f32_to_h(float x) {
    return __half_as_ushort(__float2half_rn(x));
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ float h_to_f32(uint16_t h) { return __half2float(__ushort_as_half(h)); }

__device__ __forceinline__ bool h_overflowed(uint16_t h) { return (h & 0x7C00u) == 0x7C00u; }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch: let a successor launched with programmatic stream serialization
// (the ORDERED finaliser chain) be scheduled now; it waits for this grid in-kernel
// (griddepcontrol.wait).  A no-op for ordinary successors.
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// ... and, launched that way itself, wait for the predecessor grid's completion and memory flush
// before the first global access (a no-op for an ordinary launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// SplitMix64 k-th draw, k >= 1 (rng.hpp:13-18 with the state jumped ahead by k*gamma).
__device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace tcr
