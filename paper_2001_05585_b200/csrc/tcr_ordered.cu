// tcr_ordered.cu -- the ORDERED finaliser: the reference's serial binary32 accumulation of the
// block results, ascending or in the seeded Fisher-Yates order (reduction.hpp:257-268).
//
// s_0 = +0, s_{k+1} = fl(s_k + b_{pi(k)}) is one dependent chain of fp32 adds; its latency
// (4 cycles per add) is the floor of any literal evaluation.  One CTA: warps 1..7 stage the
// block results IN ORDER into a double-buffered shared-memory window (gathering through the
// order for a permutation), thread 0 runs the chain out of shared memory, so the chain never
// waits on an L2 load.  (The order itself is computed once on the host per (blocks, seed) and
// cached in the workspace -- tcr_capi.cpp.)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "tcr_device.cuh"
#include "tcr_kernels.h"

namespace tcr {

namespace {

constexpr int kOrdThreads = 256;
constexpr uint32_t kOrdBatch = 4096;   // values per staged window

__global__ void __launch_bounds__(kOrdThreads) ordered_serial_kernel(const float* __restrict__ blocks,
                                                                     const uint32_t* __restrict__ order, uint64_t nb,
                                                                     float* result) {
    __shared__ __align__(16) float buf[2][kOrdBatch];
    const unsigned tid = threadIdx.x;
    const uint64_t nbatch = (nb + kOrdBatch - 1) / kOrdBatch;
    // producers: threads 32..255 (warps 1-7); consumer: thread 0
    auto stage = [&](uint64_t k) {
        if (tid < 32 || k >= nbatch) return;
        float* dst = buf[k & 1];
        const uint64_t base = k * kOrdBatch;
        for (uint32_t i = tid - 32; i < kOrdBatch; i += kOrdThreads - 32) {
            const uint64_t j = base + i;
            float v = 0.0f;
            if (j < nb) v = __ldcg(blocks + (order ? order[j] : j));
            dst[i] = v;
        }
    };
    stage(0);
    __syncthreads();
    float acc = 0.0f;
    for (uint64_t k = 0; k < nbatch; ++k) {
        stage(k + 1);   // the next window loads while thread 0 runs this one
        if (tid == 0) {
            const float4* src = reinterpret_cast<const float4*>(buf[k & 1]);
            const uint32_t cnt = uint32_t(nb - k * kOrdBatch < kOrdBatch ? nb - k * kOrdBatch : kOrdBatch);
            const uint32_t c4 = cnt / 4;
#pragma unroll 8
            for (uint32_t i = 0; i < c4; ++i) {
                const float4 v = src[i];
                acc += v.x;
                acc += v.y;
                acc += v.z;
                acc += v.w;
            }
            for (uint32_t i = 4 * c4; i < cnt; ++i) acc += buf[k & 1][i];
        }
        __syncthreads();
    }
    if (tid == 0) *result = acc;
}

// ------------------------------------------------------------------ any order, in parallel
//
// The chain can be evaluated exactly without doing it add by add.  While the running sum stays in
// one binade [2^e, 2^(e+1)) (sign sigma), the fp32 values there are the integer multiples T u of
// u = 2^(e-23) with T in [2^23, 2^24), and fl(s + b) = sigma u round(T + sigma b / u), rounding to
// the nearest integer, ties to the EVEN integer (= even mantissa).  So over a segment of blocks:
//   q_k = sigma b_k / u (exact in binary64),  r_k = its rounding,  T_{k+1} = T_k + r_k,
// where r_k depends on T_k only through the parity of T_k and only when q_k is an exact tie.
// A segment's RECORD for a guessed (sigma, e) holds, for both start parities p0, the total
// sum_k r_k and the min / max of the partial sums; it applies to an actual running sum s iff s is
// normal with that sign and exponent and every partial T stays in [2^23 + 1, 2^24 - 1] (then
// every real T_k + q_k lies strictly inside the binade and the rounding above IS fl's).
// Records with the same guess compose associatively.
//
//   0. ordered_agg / ordered_scan: binary64 sums of every 2048 positions of the order, and their
//      exclusive prefix (one CTA).
//   1. every CTA (2048 positions = 64 segments of 32, one warp per 8 segments): binary64 segment
//      sums -> the approximate running sum before each segment -> its guess; the segment records
//      (one value per lane: tie-parity maps and partial sums by warp scans); a segment predicted
//      to leave its binade is marked for block-by-block addition; lane 0 of warp 0 composes runs
//      of equal guesses into the CTA's run list.
//   2. the last CTA (ticket): per chunk of 256 CTAs, a binary tree of compositions over the CTA
//      composites in shared memory (a node is valid when all its CTAs are one run with one
//      guess); the CTAs' run lists and the blocks of segments without a usable guess are staged
//      in shared memory; one warp walks the tree with the actual running sum -- apply a node when
//      its record holds, else descend; at a CTA: its runs, else their segments' records, else the
//      segment's blocks add by add (a warp-wide chain).  The result is the serial sum, bit for bit.
//
// Guesses only steer the speed: a wrong one fails its check and the walk descends.

__device__ __forceinline__ uint64_t u64min(uint64_t a, uint64_t b) { return a < b ? a : b; }

// The two serial chains evaluated this way: binary32 (the reference's combine of block results,
// reduction.hpp:264-268) and binary64 (oracle64, reduction.hpp:106-110).  In a binade the values
// are T u with T in [2^MANT, 2^(MANT+1)).
template <typename A> struct OxFmt;
template <> struct OxFmt<float> {
    using I = int32_t;
    using U = uint32_t;
    static constexpr int kMant = 23, kBias = 127, kEmax = 254;
    static constexpr U kExpMask = 0xFFu;
    static constexpr double kQMax = 33554432.0;            // 2^25: 32 roundings stay below 2^30
    static constexpr int64_t kClamp = 1ll << 30;
    static constexpr double kMargin = 512.0;               // ulps (the binary64 prefix vs the chain)
    __device__ static U bits(float s) { return __float_as_uint(s); }
    __device__ static float from(U b) { return __uint_as_float(b); }
};
template <> struct OxFmt<double> {
    using I = int64_t;
    using U = uint64_t;
    static constexpr int kMant = 52, kBias = 1023, kEmax = 2046;
    static constexpr U kExpMask = 0x7FFu;
    static constexpr double kQMax = 144115188075855872.0;  // 2^57: 32 roundings stay below 2^62
    static constexpr int64_t kClamp = 1ll << 60;
    static constexpr double kMargin = 1048576.0;           // 2^20 ulps
    __device__ static U bits(double s) { return uint64_t(__double_as_longlong(s)); }
    __device__ static double from(U b) { return __longlong_as_double((long long)b); }
};

template <typename A>
struct __align__(16) OxRec {    // binary32: 32 bytes; binary64: 64
    int32_t hdr;                // bit 0 valid, bit 1 negative, bits 2.. biased exponent of s
    int32_t pad;
    typename OxFmt<A>::I dT[2];  // sum of the roundings r_k for start parity 0 / 1
    typename OxFmt<A>::I mn[2];  // min / max partial sum (relative to T_0) for start parity 0 / 1
    typename OxFmt<A>::I mx[2];
};
static_assert(sizeof(OxRec<float>) == 32, "record layout");
// |dT|, |mn|, |mx| are clamped to kClamp: a record that can apply keeps every partial sum inside
// one binade (|.| < 2^(MANT+1)), so a clamped record never passes rec_applies.
template <typename A>
__device__ __forceinline__ typename OxFmt<A>::I ox_clamp(int64_t v) {
    constexpr int64_t C = OxFmt<A>::kClamp;
    return typename OxFmt<A>::I(v < -C ? -C : (v > C ? C : v));
}

constexpr uint32_t kOxSeg = 32;                             // positions per segment (one per lane)
constexpr uint32_t kOxSegPerWarp = 8;
constexpr uint32_t kOxSegPerCta = kOxSegPerWarp * (kOrdThreads / 32);   // 64
constexpr uint32_t kOxPerCta = kOxSeg * kOxSegPerCta;                  // 2048 positions
constexpr uint32_t kOxSegPool = 256;                        // staged serial segments per chunk
constexpr uint32_t kOxNoPool = 0xFFFFFFFFu;
// walk CTA = record CTAs per walk tree (leaves) = staged runs per chunk
// (512 threads for binary32 too: the 1024-thread walk CTA is capped at 64 registers and the walker
// warp spilled; measured cfg2 uniform 335.7 -> 333.2 us, normal 549 -> 530, m = 4 normal 2^28
// 7678 -> 7153, m = 4 uniform 207.5 -> 212.0)
template <typename A> struct OxWalk { static constexpr int kThreads = 512; };

// walk counters of the last launch (profiling): tree nodes applied, CTA runs applied, segment
// records applied, segments added block by block
__device__ unsigned long long g_ord_stats[4];
// profiling: %globaltimer of the first record CTA start, the last prefix, the last record end,
// the walk start and end
__device__ unsigned long long g_ord_times[5];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct OxParams {
    const float* blocks;        // the sequence (block results, reduction.hpp:248-255; or fp32 input)
    const uint16_t* halves;     // ... or binary16 input (oracle64 over binary16), when non-null
    const uint32_t* order;      // position -> index (seeded permutation) or null (ascending)
    uint64_t nb;
    uint32_t grid;              // record CTAs
    void* segrec;               // [grid * 64] OxRec<A> segment records
    void* runrec;               // [grid * 64] OxRec<A> run composites
    uint32_t* runinfo;          // [grid * 64] first local segment << 8 | segment count
    uint32_t* nrun;             // [grid]
    const double* pre;          // [grid] binary64 sum of the positions before each record CTA
    void* result;               // A
    int dbg;                    // profiling (debug_mode 41): per-chunk phase times via printf
};

__device__ __forceinline__ float ox_load(const OxParams& P, uint64_t k) {
    if (k >= P.nb) return 0.0f;   // trailing positions: + 0 is the identity of the chain (s is never -0)
    const uint64_t i = P.order ? __ldg(P.order + k) : k;
    return P.halves ? h_to_f32(__ldg(P.halves + i)) : __ldcg(P.blocks + i);
}

// (parity-indexed fields are selected, never indexed: a runtime index would put the record in
// local memory)
template <typename A>
__device__ __forceinline__ bool rec_applies(const OxRec<A>& r, A s) {
    using F = OxFmt<A>;
    using I = typename F::I;
    if (!(r.hdr & 1)) return false;
    const typename F::U bits = F::bits(s);
    const int ex = int((bits >> F::kMant) & F::kExpMask);
    if (ex == 0 || ex == int(F::kExpMask)) return false;       // zero, subnormal, inf, NaN
    if (ex != (r.hdr >> 2) || int(bits >> (8 * sizeof(A) - 1)) != ((r.hdr >> 1) & 1)) return false;
    const I T0 = I((bits & ((typename F::U(1) << F::kMant) - 1)) | (typename F::U(1) << F::kMant));
    const bool p1 = T0 & 1;
    const I mn = p1 ? r.mn[1] : r.mn[0], mx = p1 ? r.mx[1] : r.mx[0];
    return T0 + mn >= (I(1) << F::kMant) + 1 && T0 + mx <= (I(1) << (F::kMant + 1)) - 1;
}

template <typename A>
__device__ __forceinline__ A rec_apply(const OxRec<A>& r, A s) {
    using F = OxFmt<A>;
    using I = typename F::I;
    const typename F::U bits = F::bits(s);
    constexpr typename F::U kM = (typename F::U(1) << F::kMant) - 1;
    const I T0 = I((bits & kM) | (typename F::U(1) << F::kMant));
    const I T1 = T0 + ((T0 & 1) ? r.dT[1] : r.dT[0]);
    return F::from((bits & ~kM) | typename F::U(T1 - (I(1) << F::kMant)));
}

template <typename A>
__device__ __forceinline__ OxRec<A> rec_invalid() {
    OxRec<A> r;
    r.hdr = 0;
    r.pad = 0;
    r.dT[0] = r.dT[1] = 0;
    r.mn[0] = r.mn[1] = r.mx[0] = r.mx[1] = 0;
    return r;
}

template <typename A>
__device__ __forceinline__ bool rec_joinable(const OxRec<A>& a, const OxRec<A>& b) {
    return (a.hdr & 1) && a.hdr == b.hdr;
}

// Compose b after a (same guess, both valid).
template <typename A>
__device__ __forceinline__ OxRec<A> rec_compose(const OxRec<A>& a, const OxRec<A>& b) {
    OxRec<A> c;
    c.hdr = a.hdr;
    c.pad = 0;
#pragma unroll
    for (int p0 = 0; p0 < 2; ++p0) {
        const int64_t d = a.dT[p0];
        const bool pm = (p0 + a.dT[p0]) & 1;
        const int64_t bdT = pm ? b.dT[1] : b.dT[0], bmn = pm ? b.mn[1] : b.mn[0], bmx = pm ? b.mx[1] : b.mx[0];
        c.dT[p0] = ox_clamp<A>(d + bdT);
        c.mn[p0] = ox_clamp<A>(a.mn[p0] < d + bmn ? int64_t(a.mn[p0]) : d + bmn);
        c.mx[p0] = ox_clamp<A>(a.mx[p0] > d + bmx ? int64_t(a.mx[p0]) : d + bmx);
    }
    return c;
}

// guess for an approximate running sum S: its binade in A (normal range only)
template <typename A>
__device__ __forceinline__ bool ox_guess(double S, bool* neg, int* e) {
    const uint64_t bits = uint64_t(__double_as_longlong(S));
    const int de = int((bits >> 52) & 0x7FF);            // biased binary64 exponent
    *neg = (bits >> 63) != 0;
    *e = de - 1023 + OxFmt<A>::kBias;                    // biased exponent in A
    return de != 0 && *e >= 1 && *e <= OxFmt<A>::kEmax;
}

// 2^k as a binary64 built from its bits (k in the normal range)
__device__ __forceinline__ double pow2d(int k) { return __longlong_as_double((long long)(uint64_t(1023 + k) << 52)); }

template <typename I>
__device__ __forceinline__ I warp_min(I v) {
    if constexpr (sizeof(I) == 4) {
        return __reduce_min_sync(kFull, v);
    } else {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const I o = __shfl_xor_sync(kFull, v, off);
            v = o < v ? o : v;
        }
        return v;
    }
}
template <typename I>
__device__ __forceinline__ I warp_max(I v) {
    if constexpr (sizeof(I) == 4) {
        return __reduce_max_sync(kFull, v);
    } else {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const I o = __shfl_xor_sync(kFull, v, off);
            v = o > v ? o : v;
        }
        return v;
    }
}

// One warp, one value per lane: the record of the 32 values in lane order for the guess (neg, e).
// The rounding of q_k = sigma b_k / u depends on the running T only for an exact tie: with no tie
// in the warp one scan gives both parities' record.
template <typename A>
__device__ __forceinline__ OxRec<A> warp_record1(float b, bool neg, int e) {
    using F = OxFmt<A>;
    using I = typename F::I;
    const unsigned lane = threadIdx.x & 31u;
    const int sh = F::kBias + F::kMant - e;              // sigma / u = sigma 2^sh
    if (sh > 1023 || sh < -1022) return rec_invalid<A>();   // warp-uniform: the guess is
    const double q = double(b) * (neg ? -pow2d(sh) : pow2d(sh));
    const bool fin = isfinite(b) && fabs(q) < F::kQMax;
    const bool ok = __all_sync(kFull, fin);
    const double f = fin ? floor(q) : 0.0, ph = fin ? q - f : 0.0;
    const I fi = I(f);
    OxRec<A> rec;
    rec.pad = 0;
    if (!__any_sync(kFull, ph == 0.5)) {
        I inc = fi + (ph > 0.5 ? 1 : 0);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const I a = __shfl_up_sync(kFull, inc, off);
            if (lane >= uint32_t(off)) inc += a;
        }
        const I mn = ox_clamp<A>(warp_min(inc)), mx = ox_clamp<A>(warp_max(inc));
        const I tot = ox_clamp<A>(__shfl_sync(kFull, inc, 31));
        rec.dT[0] = rec.dT[1] = tot;
        rec.mn[0] = rec.mn[1] = mn;
        rec.mx[0] = rec.mx[1] = mx;
    } else {
        auto rr = [&](uint32_t p) -> I { return ph < 0.5 ? fi : (ph > 0.5 ? fi + 1 : fi + I((p + fi) & 1)); };
        // the lane's parity map p -> (p + r(p)) & 1, composed in lane order (inclusive scan)
        uint32_t m0 = uint32_t(rr(0) & 1), m1 = uint32_t((1 + rr(1)) & 1);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t a0 = __shfl_up_sync(kFull, m0, off), a1 = __shfl_up_sync(kFull, m1, off);
            if (lane >= uint32_t(off)) {
                const uint32_t n0 = a0 ? m1 : m0, n1 = a1 ? m1 : m0;   // mine(earlier(p))
                m0 = n0;
                m1 = n1;
            }
        }
        uint32_t s0 = __shfl_up_sync(kFull, m0, 1), s1 = __shfl_up_sync(kFull, m1, 1);
        if (lane == 0) {
            s0 = 0u;
            s1 = 1u;
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            I inc = rr(t ? s1 : s0);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const I a = __shfl_up_sync(kFull, inc, off);
                if (lane >= uint32_t(off)) inc += a;
            }
            rec.mn[t] = ox_clamp<A>(warp_min(inc));
            rec.mx[t] = ox_clamp<A>(warp_max(inc));
            rec.dT[t] = ox_clamp<A>(__shfl_sync(kFull, inc, 31));
        }
    }
    rec.hdr = (ok ? 1 : 0) | (neg ? 2 : 0) | (e << 2);
    return rec;
}

// One warp: s + v_0 + v_1 + ... + v_31 (lane l holds v_l), one add at a time in A (the reference's
// loop); every lane runs the same chain, so s stays warp-uniform.  All 32 shuffles are issued
// before the dependent adds, so the chain costs the adds' latency, not the shuffles'.
template <typename A>
__device__ __forceinline__ A warp_chain32(float v, A s) {
    float a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = __shfl_sync(kFull, v, i);
#pragma unroll
    for (int i = 0; i < 32; ++i) s += A(a[i]);
    return s;
}

// The same chain over 32 values staged in shared memory (16-byte aligned): broadcast vector loads.
template <typename A>
__device__ __forceinline__ A smem_chain32(const float* v, A s) {
    float4 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = reinterpret_cast<const float4*>(v)[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        s += A(a[i].x);
        s += A(a[i].y);
        s += A(a[i].z);
        s += A(a[i].w);
    }
    return s;
}

// Programmatic dependent launch: each kernel of the chain lets the next one launch at once and
// waits for its predecessor's results (griddepcontrol; no-ops without the launch attribute).
__device__ __forceinline__ void pdl_wait_and_release() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// binary64 sum of the positions [2048 b, 2048 b + 2048) of the order -> agg[b]
__global__ void __launch_bounds__(kOrdThreads) ordered_agg_kernel(const OxParams P, double* agg) {
    __shared__ double s_w[kOrdThreads / 32];
    pdl_wait_and_release();
    const uint64_t base = uint64_t(blockIdx.x) * kOxPerCta;
    double d = 0.0;
    if (!P.order && !P.halves && base + kOxPerCta <= P.nb && (reinterpret_cast<uintptr_t>(P.blocks) & 15u) == 0) {
        // ascending fp32 block results, a whole window: 16-byte L2 loads, all in flight (the
        // generic per-position loads below serialise on their branches: 14 -> ~4 us at m = 4 2^28)
        static_assert(kOxPerCta % (4 * kOrdThreads) == 0, "whole float4 per thread");
        constexpr uint32_t NV = kOxPerCta / (4 * kOrdThreads);
        const float4* v = reinterpret_cast<const float4*>(P.blocks + base) + threadIdx.x;
        float4 q[NV];
#pragma unroll
        for (uint32_t i = 0; i < NV; ++i) q[i] = __ldcg(v + i * kOrdThreads);
#pragma unroll
        for (uint32_t i = 0; i < NV; ++i) d += (double(q[i].x) + double(q[i].y)) + (double(q[i].z) + double(q[i].w));
    } else if (P.order && !P.halves && base + kOxPerCta <= P.nb) {
        // seeded permutation, a whole window: the order indices, then the gathers, all in flight
        constexpr uint32_t NP = kOxPerCta / kOrdThreads;
        uint32_t ix[NP];
#pragma unroll
        for (uint32_t i = 0; i < NP; ++i) ix[i] = __ldg(P.order + base + i * kOrdThreads + threadIdx.x);
        float q[NP];
#pragma unroll
        for (uint32_t i = 0; i < NP; ++i) q[i] = __ldcg(P.blocks + ix[i]);
#pragma unroll
        for (uint32_t i = 0; i < NP; ++i) d += double(q[i]);
    } else {
#pragma unroll
        for (uint32_t i = 0; i < kOxPerCta / kOrdThreads; ++i) d += double(ox_load(P, base + i * kOrdThreads + threadIdx.x));
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) d += __shfl_xor_sync(kFull, d, off);
    if ((threadIdx.x & 31u) == 0) s_w[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < kOrdThreads / 32; ++w) a += s_w[w];
        agg[blockIdx.x] = a;
    }
}

// exclusive prefix of agg[0, grid) in binary64, one CTA of 1024 threads: pre[b]
__global__ void __launch_bounds__(1024) ordered_scan_kernel(const double* agg, double* pre, uint32_t grid) {
    __shared__ double s_t[1024];
    pdl_wait_and_release();
    const uint32_t t = threadIdx.x;
    const uint32_t per = (grid + 1023) / 1024, lo = t * per, hi = min(grid, lo + per);
    double sum = 0.0;
    for (uint32_t i = lo; i < hi; ++i) sum += __ldcg(agg + i);
    s_t[t] = sum;
    __syncthreads();
    for (uint32_t off = 1; off < 1024; off <<= 1) {   // inclusive Hillis-Steele scan of the thread sums
        const double v = t >= off ? s_t[t - off] : 0.0;
        __syncthreads();
        s_t[t] += v;
        __syncthreads();
    }
    double run = t ? s_t[t - 1] : 0.0;
    for (uint32_t i = lo; i < hi; ++i) {
        pre[i] = run;
        run += __ldcg(agg + i);
    }
}

// Records: CTA b = positions [2048 b, 2048 b + 2048) = 64 segments; warp w segments 8w .. 8w+7.
template <typename A>
__global__ void __launch_bounds__(kOrdThreads, 4) ordered_records_kernel(const OxParams P) {
    using F = OxFmt<A>;
    using Rec = OxRec<A>;
    __shared__ double s_ss[kOxSegPerCta];
    __shared__ double s_S[kOxSegPerCta];
    __shared__ Rec s_run[kOxSegPerCta];        // per warp: its runs at [8 w, 8 w + count)
    __shared__ uint32_t s_info[kOxSegPerCta];
    __shared__ uint32_t s_wn[kOrdThreads / 32];
    Rec* segrec = static_cast<Rec*>(P.segrec);
    Rec* runrec = static_cast<Rec*>(P.runrec);
    const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint64_t b = blockIdx.x;
    const uint64_t base = b * kOxPerCta;
    pdl_wait_and_release();
    if (tid == 0) atomicMin(&g_ord_times[0], gtimer());
    float v[kOxSegPerWarp];
#pragma unroll
    for (uint32_t i = 0; i < kOxSegPerWarp; ++i) v[i] = 0.0f;
    if (!P.order && !P.halves && base + kOxPerCta <= P.nb) {
        // ascending block results, a whole window: plain coalesced L2 loads, all in flight
#pragma unroll
        for (uint32_t i = 0; i < kOxSegPerWarp; ++i) v[i] = __ldcg(P.blocks + base + (warp * kOxSegPerWarp + i) * kOxSeg + lane);
    } else if (P.order && !P.halves && base + kOxPerCta <= P.nb) {
        // seeded permutation, a whole window: all 8 order indices, then all 8 gathers in flight
        uint32_t ix[kOxSegPerWarp];
#pragma unroll
        for (uint32_t i = 0; i < kOxSegPerWarp; ++i) ix[i] = __ldg(P.order + base + (warp * kOxSegPerWarp + i) * kOxSeg + lane);
#pragma unroll
        for (uint32_t i = 0; i < kOxSegPerWarp; ++i) v[i] = __ldcg(P.blocks + ix[i]);
    } else {
#pragma unroll
        for (uint32_t i = 0; i < kOxSegPerWarp; ++i) v[i] = ox_load(P, base + (warp * kOxSegPerWarp + i) * kOxSeg + lane);
    }
#pragma unroll
    for (uint32_t i = 0; i < kOxSegPerWarp; ++i) {
        double d = double(v[i]);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) d += __shfl_xor_sync(kFull, d, off);
        if (lane == 0) s_ss[warp * kOxSegPerWarp + i] = d;
    }
    __syncthreads();
    if (warp == 0) {
        // exclusive prefix of the 64 segment sums (two per lane), from the CTA's prefix
        const double a0 = s_ss[2 * lane], a1 = s_ss[2 * lane + 1];
        double inc = a0 + a1;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double t = __shfl_up_sync(kFull, inc, off);
            if (lane >= uint32_t(off)) inc += t;
        }
        const double ex = __ldcg(P.pre + b) + (inc - (a0 + a1));
        s_S[2 * lane] = ex;
        s_S[2 * lane + 1] = ex + a0;
        if (lane == 0) atomicMax(&g_ord_times[1], gtimer());
    }
    __syncthreads();
    Rec r[kOxSegPerWarp];
#pragma unroll
    for (uint32_t i = 0; i < kOxSegPerWarp; ++i) {
        const uint32_t si = warp * kOxSegPerWarp + i;
        const double S = s_S[si];
        bool neg;
        int e;
        r[i] = ox_guess<A>(S, &neg, &e) ? warp_record1<A>(v[i], neg, e) : rec_invalid<A>();
        if (r[i].hdr & 1) {
            // predicted to leave its binade (the estimated start plus the record's partial sums
            // within kMargin ulps of an edge): the segment will be added block by block -- a run
            // break.  The margin covers the distance between the binary64 prefix and the actual
            // chain (binary32: measured <= 84 ulps at 2^30 uniform, m = 4); a wrong prediction
            // only costs speed (the walk descends)
            const double T0 = fabs(S) * pow2d(F::kBias + F::kMant - e);
            const double lo = pow2d(F::kMant) + F::kMargin, hi = pow2d(F::kMant + 1) - F::kMargin;
            if (T0 + double(min(r[i].mn[0], r[i].mn[1])) < lo || T0 + double(max(r[i].mx[0], r[i].mx[1])) > hi)
                r[i].hdr &= ~1;
        }
        if (lane == 0) segrec[b * kOxSegPerCta + si] = r[i];
    }
    // the warp's runs (lane 0), then thread 0 joins the warps' run lists
    if (lane == 0) {
        uint32_t nr = 0, first = 0;
        Rec c = r[0];
#pragma unroll
        for (uint32_t i = 1; i <= kOxSegPerWarp; ++i) {
            if (i < kOxSegPerWarp && rec_joinable(c, r[i])) {
                c = rec_compose(c, r[i]);
                continue;
            }
            s_run[warp * kOxSegPerWarp + nr] = c;
            s_info[warp * kOxSegPerWarp + nr] = ((warp * kOxSegPerWarp + first) << 8) | (i - first);
            ++nr;
            if (i < kOxSegPerWarp) {
                c = r[i];
                first = i;
            }
        }
        s_wn[warp] = nr;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t nr = 0;
        Rec c = s_run[0];
        uint32_t ci = s_info[0];
        for (uint32_t w = 0; w < kOrdThreads / 32; ++w) {
            for (uint32_t j = (w == 0 ? 1 : 0); j < s_wn[w]; ++j) {
                const Rec& x = s_run[w * kOxSegPerWarp + j];
                const uint32_t xi = s_info[w * kOxSegPerWarp + j];
                if (rec_joinable(c, x)) {
                    c = rec_compose(c, x);
                    ci += xi & 0xFFu;
                    continue;
                }
                runrec[b * kOxSegPerCta + nr] = c;
                P.runinfo[b * kOxSegPerCta + nr] = ci;
                ++nr;
                c = x;
                ci = xi;
            }
        }
        runrec[b * kOxSegPerCta + nr] = c;
        P.runinfo[b * kOxSegPerCta + nr] = ci;
        P.nrun[b] = nr + 1;
        atomicMax(&g_ord_times[2], gtimer());
    }
}

template <typename A>
struct OxWalkSmem {
    static constexpr uint32_t CH = OxWalk<A>::kThreads;    // leaves per chunk = staged runs
    OxRec<A> node[2 * CH - 1];      // tree over the chunk's CTA composites (heap order)
    OxRec<A> run[CH];               // staged run lists
    uint32_t runinfo[CH];           // first << 8 | count
    uint32_t runseg[CH];            // segment pool slot of an invalid one-segment run, or kOxNoPool
    uint32_t owner[CH];             // leaf that owns the staged run
    uint32_t runbase[CH];           // first staged run of each leaf, or kOxNoPool
    uint32_t leafnr[CH];            // runs of each leaf
    uint32_t segid[kOxSegPool];     // global segment of each staged serial segment
    __align__(16) float seg[kOxSegPool][kOxSeg];  // staged values of serial segments
    uint8_t kind[2 * CH];           // 0 empty, 1 valid composite, 2 descend
    uint8_t pred[2 * CH];           // the node's composite is predicted to apply (estimated start)
    uint32_t items[CH];             // the walk plan: topmost predicted nodes and uncovered leaves
    uint32_t wsum[CH / 32];
    uint32_t nruns, nsegs, nitems;
};

// The walk (one CTA): per chunk of CH record CTAs, stage, build the tree, walk it with warp 0.
template <typename A>
__global__ void __launch_bounds__(OxWalk<A>::kThreads) ordered_walk_kernel(const OxParams P) {
    using Rec = OxRec<A>;
    constexpr uint32_t CH = OxWalk<A>::kThreads;
    extern __shared__ __align__(16) unsigned char ox_smem[];
    OxWalkSmem<A>& W = *reinterpret_cast<OxWalkSmem<A>*>(ox_smem);
    const Rec* segrec = static_cast<const Rec*>(P.segrec);
    const Rec* runrec = static_cast<const Rec*>(P.runrec);
    const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    pdl_wait_and_release();
    if (tid == 0) g_ord_times[3] = gtimer();
    A s = A(0);
    unsigned long long st[4] = {0, 0, 0, 0};
    for (uint64_t c0 = 0; c0 < P.grid; c0 += CH) {
        const unsigned long long tc0 = gtimer();
        const uint32_t cn = uint32_t(u64min(CH, P.grid - c0));
        uint32_t L = 2;   // leaves of this chunk's tree: a power of two >= cn (shallow trees for small grids)
        while (L < cn) L <<= 1;
        if (tid == 0) W.nruns = W.nsegs = 0;
        __syncthreads();
        // leaves: the CTA composite when the CTA is one valid run; reserve pool space for the others
        const uint32_t li = L - 1 + tid;
        uint8_t kd = 0;
        uint32_t nr = 0, rb = kOxNoPool;
        if (tid < cn) {
            const uint64_t cb = c0 + tid;
            nr = __ldcg(P.nrun + cb);
            const Rec r0 = runrec[cb * kOxSegPerCta];
            if (nr == 1 && (r0.hdr & 1)) {
                W.node[li] = r0;
                kd = 1;
            } else {
                kd = 2;
                const uint32_t at = atomicAdd(&W.nruns, nr);
                if (at + nr <= CH) {
                    rb = at;
                    for (uint32_t r = 0; r < nr; ++r) W.owner[at + r] = tid;
                } else {
                    // does not fit: walked from global memory; mark its share of the pool unused
                    for (uint32_t r = at; r < at + nr && r < CH; ++r) W.owner[r] = kOxNoPool;
                }
            }
        }
        if (tid < L) W.kind[li] = kd;
        W.runbase[tid] = rb;
        W.leafnr[tid] = nr;
        __syncthreads();
        const unsigned long long tc1 = gtimer();
        // stage the runs (one per thread), and reserve a pool slot for each serial segment
        const uint32_t staged = min(W.nruns, CH);
        for (uint32_t j = tid; j < staged; j += CH) {
            const uint32_t t = W.owner[j];
            if (t == kOxNoPool) continue;
            const uint64_t cb = c0 + t;
            const uint32_t r = j - W.runbase[t];
            const Rec rr = runrec[cb * kOxSegPerCta + r];
            const uint32_t ri = __ldcg(P.runinfo + cb * kOxSegPerCta + r);
            W.run[j] = rr;
            W.runinfo[j] = ri;
            uint32_t sl = kOxNoPool;
            if (!(rr.hdr & 1) && (ri & 0xFFu) == 1u) {
                const uint32_t ss = atomicAdd(&W.nsegs, 1u);
                if (ss < kOxSegPool) {
                    sl = ss;
                    W.segid[ss] = uint32_t(cb * kOxSegPerCta + (ri >> 8));
                }
            }
            W.runseg[j] = sl;
        }
        __syncthreads();
        const unsigned long long tc2 = gtimer();
        // stage the serial segments' values, all threads at once
        const uint32_t nseg = min(W.nsegs, kOxSegPool);
        for (uint32_t e2 = tid; e2 < nseg * kOxSeg; e2 += CH)
            W.seg[e2 / kOxSeg][e2 % kOxSeg] = ox_load(P, uint64_t(W.segid[e2 / kOxSeg]) * kOxSeg + e2 % kOxSeg);
        // internal nodes, level by level (heap order: children 2i+1, 2i+2)
        for (uint32_t cnt = L / 2, lo = L / 2 - 1;; cnt >>= 1, lo = (lo - 1) / 2) {
            __syncthreads();
            if (tid < cnt) {
                const uint32_t i = lo + tid, l = 2 * i + 1, r = 2 * i + 2;
                const uint8_t kl = W.kind[l], kr = W.kind[r];
                uint8_t k;
                if (kl == 0) {
                    k = kr;
                    if (kr == 1) W.node[i] = W.node[r];
                } else if (kr == 0) {
                    k = kl;
                    if (kl == 1) W.node[i] = W.node[l];
                } else if (kl == 1 && kr == 1 && rec_joinable(W.node[l], W.node[r])) {
                    W.node[i] = rec_compose(W.node[l], W.node[r]);
                    k = 1;
                } else {
                    k = 2;
                }
                W.kind[i] = k;
            }
            if (cnt == 1) break;
        }
        __syncthreads();
        const unsigned long long tc3 = gtimer();
        // the plan: a node's composite is predicted to apply at the binary64 prefix before its
        // first record CTA; the walk visits the topmost predicted nodes and the uncovered leaves
        // in order, and descends only where a prediction fails
        for (uint32_t i = tid; i < 2 * L - 1; i += CH) {
            uint32_t f = i;
            while (f < L - 1) f = 2 * f + 1;   // leftmost leaf
            const uint32_t t = f - (L - 1);
            bool pr = false;
            if (W.kind[i] == 1 && t < cn) pr = rec_applies(W.node[i], A(__ldcg(P.pre + c0 + t)));
            W.pred[i] = pr ? 1 : 0;
        }
        __syncthreads();
        uint32_t item = 0, emit = 0;
        if (tid < cn && W.kind[L - 1 + tid] != 0) {
            uint32_t i = L - 1 + tid, cover = W.pred[i] ? i : kOxNoPool;
            while (i > 0) {
                i = (i - 1) / 2;
                if (W.pred[i]) cover = i;
            }
            if (cover == kOxNoPool) {
                item = L - 1 + tid;
                emit = 1;
            } else {
                uint32_t f = cover;
                while (f < L - 1) f = 2 * f + 1;
                item = cover;
                emit = f == L - 1 + tid;
            }
        }
        // block-wide exclusive scan of the emit flags -> the plan in leaf order
        const unsigned bal = __ballot_sync(kFull, emit);
        if (lane == 0) W.wsum[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {
            const uint32_t v = lane < CH / 32 ? W.wsum[lane] : 0u;
            uint32_t inc = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t t2 = __shfl_up_sync(kFull, inc, off);
                if (lane >= uint32_t(off)) inc += t2;
            }
            if (lane < CH / 32) W.wsum[lane] = inc - v;
            if (lane == 31) W.nitems = inc;
        }
        __syncthreads();
        if (emit) W.items[W.wsum[warp] + __popc(bal & ((1u << lane) - 1u))] = item;
        __syncthreads();
        const unsigned long long tc4 = gtimer();
        // the walk: warp 0 -- each plan item applied when its record holds, else depth-first
        // below it with an explicit stack
        if (warp == 0) {
            const uint32_t nit = W.nitems;
            long long cy[6] = {0, 0, 0, 0, 0, 0};   // profiling (mode 41): cycles per step kind
            int cn6[6] = {0, 0, 0, 0, 0, 0};
            long long c_prev = clock64();
            auto tick = [&](int k) {
                if (P.dbg) {
                    const long long c = clock64();
                    cy[k] += c - c_prev;
                    ++cn6[k];
                    c_prev = c;
                }
            };
            for (uint32_t j = 0; j < nit; ++j) {
                const uint32_t root = W.items[j];
                tick(5);
                if (W.pred[root] && rec_applies(W.node[root], s)) {
                    s = rec_apply(W.node[root], s);
                    ++st[0];
                    tick(0);
                    continue;
                }
                uint32_t stk[24];
                int top = 0;
                stk[top++] = root;
                while (top > 0) {
                    const uint32_t i = stk[--top];
                    const uint8_t k = W.kind[i];
                    if (k == 0) continue;
                    if (k == 1 && rec_applies(W.node[i], s)) {
                        s = rec_apply(W.node[i], s);
                        ++st[0];
                        continue;
                    }
                    if (i < L - 1) {                   // internal: right pushed first, left walked first
                        stk[top++] = 2 * i + 2;
                        stk[top++] = 2 * i + 1;
                        tick(1);
                        continue;
                    }
                    // leaf: record CTA cb, its runs (staged or from global)
                    const uint32_t t = i - (L - 1);
                    const uint64_t cb = c0 + t;
                    const uint32_t rb2 = W.runbase[t];
                    const uint32_t nr2 = k == 1 ? 1u : W.leafnr[t];
                    for (uint32_t r = 0; r < nr2; ++r) {
                        Rec rr;
                        uint32_t ri, sl = kOxNoPool;
                        if (k == 1) {
                            rr = W.node[i];
                            ri = kOxSegPerCta;   // segments 0 .. 63
                        } else if (rb2 != kOxNoPool) {
                            rr = W.run[rb2 + r];
                            ri = W.runinfo[rb2 + r];
                            sl = W.runseg[rb2 + r];
                        } else {
                            rr = runrec[cb * kOxSegPerCta + r];
                            ri = __ldcg(P.runinfo + cb * kOxSegPerCta + r);
                        }
                        if (rec_applies(rr, s)) {
                            s = rec_apply(rr, s);
                            ++st[1];
                            tick(2);
                            continue;
                        }
                        const uint32_t sf = ri >> 8, sc = ri & 0xFFu;
                        for (uint32_t q = sf; q < sf + sc; ++q) {
                            const uint64_t gs = cb * kOxSegPerCta + q;
                            if (sc > 1 || (rr.hdr & 1)) {
                                const Rec sr = segrec[gs];
                                if (rec_applies(sr, s)) {
                                    s = rec_apply(sr, s);
                                    ++st[2];
                                    tick(3);
                                    continue;
                                }
                                tick(3);
                            }
                            if (sl != kOxNoPool) s = smem_chain32<A>(W.seg[sl], s);
                            else s = warp_chain32<A>(ox_load(P, gs * kOxSeg + lane), s);
                            ++st[3];
                            tick(4);
                        }
                    }
                }
            }
            if (P.dbg && lane == 0)
                printf("  walk cycles: roots %lld (%d), nodes %lld (%d), runs %lld (%d), segrec %lld (%d), serial %lld (%d), item starts %lld (%d)\n",
                       cy[0], cn6[0], cy[1], cn6[1], cy[2], cn6[2], cy[3], cn6[3], cy[4], cn6[4], cy[5], cn6[5]);
        }
        if (P.dbg && tid == 0)
            printf("ordered walk chunk %llu: leaves %.2f us, runs staged %.2f us (%u), segments staged + tree %.2f us (%u), "
                   "plan %.2f us (%u items), walk %.2f us\n", (unsigned long long)c0, (tc1 - tc0) * 1e-3, (tc2 - tc1) * 1e-3,
                   W.nruns, (tc3 - tc2) * 1e-3, W.nsegs, (tc4 - tc3) * 1e-3, W.nitems, (gtimer() - tc4) * 1e-3);
        __syncthreads();
    }
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) g_ord_stats[i] = st[i];
        g_ord_times[4] = gtimer();
        *static_cast<A*>(P.result) = s;
    }
}

}  // namespace

cudaError_t launch_ordered(const float* blocks, const uint32_t* order, uint64_t nb, float* result, cudaStream_t s) {
    ordered_serial_kernel<<<1, kOrdThreads, 0, s>>>(blocks, order, nb, result);
    return cudaGetLastError();
}

int ordered_stats(unsigned long long* host) {
    if (cudaMemcpyFromSymbol(host, g_ord_stats, sizeof(g_ord_stats)) != cudaSuccess) return -1;
    if (cudaMemcpyFromSymbol(host + 4, g_ord_times, sizeof(g_ord_times)) != cudaSuccess) return -1;
    const unsigned long long init[5] = {~0ull, 0, 0, 0, 0};   // re-arm min / max for the next launch
    return cudaMemcpyToSymbol(g_ord_times, init, sizeof(init)) == cudaSuccess ? 0 : -1;
}

int ordered_grid(uint64_t nb) { return int((nb + kOxPerCta - 1) / kOxPerCta); }

size_t ordered_ws_bytes(uint64_t nb, bool binary64) {
    const size_t grid = size_t(ordered_grid(nb));
    const size_t rec = binary64 ? sizeof(OxRec<double>) : sizeof(OxRec<float>);
    return grid * kOxSegPerCta * (2 * rec + sizeof(uint32_t)) + grid * (2 * sizeof(double) + sizeof(uint32_t)) + 256;
}

namespace {

template <typename A>
cudaError_t launch_chain(const float* blocks, const uint16_t* halves, const uint32_t* order, uint64_t nb, void* ws,
                         A* result, cudaStream_t s) {
    const int grid = ordered_grid(nb);
    constexpr size_t smem = sizeof(OxWalkSmem<A>);
    static PerDeviceOnce once;
    const cudaError_t ea = once([] {
        return cudaFuncSetAttribute(ordered_walk_kernel<A>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    });
    if (ea != cudaSuccess) return ea;
    OxParams P{};
    P.blocks = blocks;
    P.halves = halves;
    P.order = order;
    P.nb = nb;
    P.grid = uint32_t(grid);
    P.dbg = knobs().debug_mode == 41;
    char* w = static_cast<char*>(ws);
    const size_t ns = size_t(grid) * kOxSegPerCta;
    // 16-byte aligned members first
    OxRec<A>* segrec = reinterpret_cast<OxRec<A>*>(w);
    OxRec<A>* runrec = segrec + ns;
    double* agg = reinterpret_cast<double*>(runrec + ns);
    double* pre = agg + grid;
    P.segrec = segrec;
    P.runrec = runrec;
    P.pre = pre;
    P.runinfo = reinterpret_cast<uint32_t*>(pre + grid);
    P.nrun = P.runinfo + ns;
    P.result = result;
    // four stream-ordered launches with programmatic dependent launch: each grid is scheduled while
    // its predecessor runs and waits on it in-kernel (the launch latencies overlap)
    auto pdl = [&](auto kernel, unsigned g, unsigned t, size_t dyn, auto... args) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(g);
        cfg.blockDim = dim3(t);
        cfg.dynamicSmemBytes = dyn;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kernel, args...);
    };
    cudaError_t e = pdl(ordered_agg_kernel, unsigned(grid), unsigned(kOrdThreads), 0, P, agg);
    if (e == cudaSuccess) e = pdl(ordered_scan_kernel, 1u, 1024u, 0, static_cast<const double*>(agg), pre, uint32_t(grid));
    if (e == cudaSuccess) e = pdl(ordered_records_kernel<A>, unsigned(grid), unsigned(kOrdThreads), 0, P);
    if (e == cudaSuccess) e = pdl(ordered_walk_kernel<A>, 1u, unsigned(OxWalk<A>::kThreads), smem, P);
    return e;
}

}  // namespace

cudaError_t launch_ordered_parallel(const float* blocks, const uint32_t* order, uint64_t nb, void* ws, uint32_t* ticket,
                                    float* result, cudaStream_t s) {
    (void)ticket;
    return launch_chain<float>(blocks, nullptr, order, nb, ws, result, s);
}

cudaError_t launch_serial_sum64(const void* x, bool f32, uint64_t n, void* ws, double* result, cudaStream_t s) {
    return f32 ? launch_chain<double>(static_cast<const float*>(x), nullptr, nullptr, n, ws, result, s)
               : launch_chain<double>(nullptr, static_cast<const uint16_t*>(x), nullptr, n, ws, result, s);
}

}  // namespace tcr
