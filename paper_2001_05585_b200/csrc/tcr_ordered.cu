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

__device__ __forceinline__ int32_t clamp30(int64_t v) {
    return int32_t(v < -(1ll << 30) ? -(1ll << 30) : (v > (1ll << 30) ? (1ll << 30) : v));
}
__device__ __forceinline__ uint64_t u64min(uint64_t a, uint64_t b) { return a < b ? a : b; }

struct __align__(16) OrdRec {   // 32 bytes, two 16-byte accesses
    int32_t hdr;                // bit 0 valid, bit 1 negative, bits 2.. biased exponent of s
    int32_t dT[2];              // sum of the roundings r_k for start parity 0 / 1
    int32_t mn[2], mx[2];       // min / max partial sum (relative to T_0) for start parity 0 / 1
    int32_t pad;
};
static_assert(sizeof(OrdRec) == 32, "record layout");
// |dT|, |mn|, |mx| are clamped to 2^30: a record that can apply keeps every partial sum inside
// one binade (|.| < 2^24), so a clamped record never passes rec_applies.

constexpr uint32_t kOxSeg = 32;                             // positions per segment (one per lane)
constexpr uint32_t kOxSegPerWarp = 8;
constexpr uint32_t kOxSegPerCta = kOxSegPerWarp * (kOrdThreads / 32);   // 64
constexpr uint32_t kOxPerCta = kOxSeg * kOxSegPerCta;                  // 2048 positions
constexpr int kOxWalkThreads = 1024;
constexpr uint32_t kOxChunk = kOxWalkThreads;               // record CTAs per walk tree (leaves)
constexpr uint32_t kOxNodes = 2 * kOxChunk - 1;
constexpr uint32_t kOxRunPool = 1024;                       // staged runs per chunk
constexpr uint32_t kOxSegPool = 256;                        // staged serial segments per chunk
constexpr uint32_t kOxNoPool = 0xFFFFFFFFu;
constexpr double kOxMargin = 512.0;                         // units of the binade's ulp

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
    const float* blocks;        // block results (reduction.hpp:248-255)
    const uint32_t* order;      // position -> block (seeded permutation) or null (ascending)
    uint64_t nb;
    uint32_t grid;              // record CTAs
    OrdRec* segrec;             // [grid * 64] segment records
    OrdRec* runrec;             // [grid * 64] run composites
    uint32_t* runinfo;          // [grid * 64] first local segment << 8 | segment count
    uint32_t* nrun;             // [grid]
    const double* pre;          // [grid] binary64 sum of the positions before each record CTA
    float* result;
    int dbg;                    // profiling (debug_mode 41): per-chunk phase times via printf
};

__device__ __forceinline__ float ox_load(const OxParams& P, uint64_t k) {
    if (k >= P.nb) return 0.0f;   // trailing positions: + 0 is the identity of the chain (s is never -0)
    return __ldcg(P.blocks + (P.order ? __ldg(P.order + k) : k));
}

// (parity-indexed fields are selected, never indexed: a runtime index would put the record in
// local memory)
__device__ __forceinline__ bool rec_applies(const OrdRec& r, float s) {
    if (!(r.hdr & 1)) return false;
    const uint32_t bits = __float_as_uint(s);
    const uint32_t ex = (bits >> 23) & 0xFFu;
    if (ex == 0 || ex == 0xFFu) return false;                  // zero, subnormal, inf, NaN
    if (int32_t(ex) != (r.hdr >> 2) || int32_t(bits >> 31) != ((r.hdr >> 1) & 1)) return false;
    const int32_t T0 = int32_t((bits & 0x7FFFFFu) | 0x800000u);
    const bool p1 = T0 & 1;
    const int32_t mn = p1 ? r.mn[1] : r.mn[0], mx = p1 ? r.mx[1] : r.mx[0];
    return T0 + mn >= (1 << 23) + 1 && T0 + mx <= (1 << 24) - 1;
}

__device__ __forceinline__ float rec_apply(const OrdRec& r, float s) {
    const uint32_t bits = __float_as_uint(s);
    const int32_t T0 = int32_t((bits & 0x7FFFFFu) | 0x800000u);
    const int32_t T1 = T0 + ((T0 & 1) ? r.dT[1] : r.dT[0]);
    return __uint_as_float((bits & 0xFF800000u) | uint32_t(T1 - (1 << 23)));
}

__device__ __forceinline__ OrdRec rec_invalid() {
    OrdRec r;
    r.hdr = 0;
    r.dT[0] = r.dT[1] = 0;
    r.mn[0] = r.mn[1] = r.mx[0] = r.mx[1] = 0;
    r.pad = 0;
    return r;
}

__device__ __forceinline__ bool rec_joinable(const OrdRec& a, const OrdRec& b) { return (a.hdr & 1) && a.hdr == b.hdr; }

// Compose b after a (same guess, both valid).
__device__ __forceinline__ OrdRec rec_compose(const OrdRec& a, const OrdRec& b) {
    OrdRec c;
    c.hdr = a.hdr;
    c.pad = 0;
#pragma unroll
    for (int p0 = 0; p0 < 2; ++p0) {
        const int64_t d = a.dT[p0];
        const bool pm = (p0 + a.dT[p0]) & 1;
        const int64_t bdT = pm ? b.dT[1] : b.dT[0], bmn = pm ? b.mn[1] : b.mn[0], bmx = pm ? b.mx[1] : b.mx[0];
        c.dT[p0] = clamp30(d + bdT);
        c.mn[p0] = clamp30(a.mn[p0] < d + bmn ? int64_t(a.mn[p0]) : d + bmn);
        c.mx[p0] = clamp30(a.mx[p0] > d + bmx ? int64_t(a.mx[p0]) : d + bmx);
    }
    return c;
}

// guess for an approximate running sum S: its binade (normal binary32 range only)
__device__ __forceinline__ bool ox_guess(double S, bool* neg, int* e) {
    const uint64_t bits = uint64_t(__double_as_longlong(S));
    const int de = int((bits >> 52) & 0x7FF);            // biased binary64 exponent
    *neg = (bits >> 63) != 0;
    *e = de - 1023 + 127;                                // biased binary32 exponent
    return de != 0 && *e >= 1 && *e <= 254;
}

// One warp, one value per lane: the record of the 32 values in lane order for the guess (neg, e).
// The rounding of q_k = sigma b_k / u depends on the running T only for an exact tie: with no tie
// in the warp one scan gives both parities' record.
__device__ __forceinline__ OrdRec warp_record1(float b, bool neg, int e) {
    const unsigned lane = threadIdx.x & 31u;
    // sigma / u = sigma 2^(150 - e), built from its bits
    const double scale = __longlong_as_double((long long)(uint64_t(1023 + 150 - e) << 52) | (neg ? (1ll << 63) : 0ll));
    const double q = double(b) * scale;
    const bool fin = isfinite(b) && fabs(q) < 33554432.0;   // 2^25
    const bool ok = __all_sync(kFull, fin);
    const double f = fin ? floor(q) : 0.0, ph = fin ? q - f : 0.0;
    const int32_t fi = int32_t(f);
    OrdRec rec;
    rec.pad = 0;
    if (!__any_sync(kFull, ph == 0.5)) {
        int32_t inc = fi + (ph > 0.5 ? 1 : 0);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int32_t a = __shfl_up_sync(kFull, inc, off);
            if (lane >= uint32_t(off)) inc += a;
        }
        const int32_t mn = __reduce_min_sync(kFull, inc), mx = __reduce_max_sync(kFull, inc);
        const int32_t tot = __shfl_sync(kFull, inc, 31);
        rec.dT[0] = rec.dT[1] = tot;
        rec.mn[0] = rec.mn[1] = mn;
        rec.mx[0] = rec.mx[1] = mx;
    } else {
        auto rr = [&](uint32_t p) -> int32_t { return ph < 0.5 ? fi : (ph > 0.5 ? fi + 1 : fi + int32_t((p + fi) & 1)); };
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
            int32_t inc = rr(t ? s1 : s0);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int32_t a = __shfl_up_sync(kFull, inc, off);
                if (lane >= uint32_t(off)) inc += a;
            }
            rec.mn[t] = __reduce_min_sync(kFull, inc);
            rec.mx[t] = __reduce_max_sync(kFull, inc);
            rec.dT[t] = __shfl_sync(kFull, inc, 31);
        }
    }
    rec.hdr = (ok ? 1 : 0) | (neg ? 2 : 0) | (e << 2);
    return rec;
}

// One warp: s + v_0 + v_1 + ... + v_31 (lane l holds v_l), one fp32 add at a time (the reference's
// loop); every lane runs the same chain, so s stays warp-uniform.  All 32 shuffles are issued
// before the dependent adds, so the chain costs the adds' latency, not the shuffles'.
__device__ __forceinline__ float warp_chain32(float v, float s) {
    float a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = __shfl_sync(kFull, v, i);
#pragma unroll
    for (int i = 0; i < 32; ++i) s += a[i];
    return s;
}

// The same chain over 32 values staged in shared memory (16-byte aligned): broadcast vector loads.
__device__ __forceinline__ float smem_chain32(const float* v, float s) {
    float4 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = reinterpret_cast<const float4*>(v)[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        s += a[i].x;
        s += a[i].y;
        s += a[i].z;
        s += a[i].w;
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
#pragma unroll
    for (uint32_t i = 0; i < kOxPerCta / kOrdThreads; ++i) d += double(ox_load(P, base + i * kOrdThreads + threadIdx.x));
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
__global__ void __launch_bounds__(kOrdThreads, 4) ordered_records_kernel(const OxParams P) {
    __shared__ double s_ss[kOxSegPerCta];
    __shared__ double s_S[kOxSegPerCta];
    __shared__ OrdRec s_run[kOxSegPerCta];     // per warp: its runs at [8 w, 8 w + count)
    __shared__ uint32_t s_info[kOxSegPerCta];
    __shared__ uint32_t s_wn[kOrdThreads / 32];
    const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint64_t b = blockIdx.x;
    const uint64_t base = b * kOxPerCta;
    pdl_wait_and_release();
    if (tid == 0) atomicMin(&g_ord_times[0], gtimer());
    float v[kOxSegPerWarp];
#pragma unroll
    for (uint32_t i = 0; i < kOxSegPerWarp; ++i) v[i] = ox_load(P, base + (warp * kOxSegPerWarp + i) * kOxSeg + lane);
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
    OrdRec r[kOxSegPerWarp];
#pragma unroll
    for (uint32_t i = 0; i < kOxSegPerWarp; ++i) {
        const uint32_t si = warp * kOxSegPerWarp + i;
        const double S = s_S[si];
        bool neg;
        int e;
        r[i] = ox_guess(S, &neg, &e) ? warp_record1(v[i], neg, e) : rec_invalid();
        if (r[i].hdr & 1) {
            // predicted to leave its binade (the estimated start plus the record's partial sums
            // within kOxMargin units of an edge): the segment will be added block by block -- a
            // run break.  The margin covers the distance between the binary64 prefix and the
            // actual binary32 chain (measured <= 84 units at 2^30 uniform, m = 4); a wrong
            // prediction only costs speed (the walk descends)
            const double T0 = fabs(S) * __longlong_as_double((long long)(uint64_t(1023 + 150 - e) << 52));
            const double mg = kOxMargin;
            if (T0 + double(min(r[i].mn[0], r[i].mn[1])) < 8388608.0 + mg ||
                T0 + double(max(r[i].mx[0], r[i].mx[1])) > 16777216.0 - mg)
                r[i].hdr &= ~1;
        }
        if (lane == 0) P.segrec[b * kOxSegPerCta + si] = r[i];
    }
    // the warp's runs (lane 0), then thread 0 joins the warps' run lists
    if (lane == 0) {
        uint32_t nr = 0, first = 0;
        OrdRec c = r[0];
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
        OrdRec c = s_run[0];
        uint32_t ci = s_info[0];
        for (uint32_t w = 0; w < kOrdThreads / 32; ++w) {
            for (uint32_t j = (w == 0 ? 1 : 0); j < s_wn[w]; ++j) {
                const OrdRec& x = s_run[w * kOxSegPerWarp + j];
                const uint32_t xi = s_info[w * kOxSegPerWarp + j];
                if (rec_joinable(c, x)) {
                    c = rec_compose(c, x);
                    ci += xi & 0xFFu;
                    continue;
                }
                P.runrec[b * kOxSegPerCta + nr] = c;
                P.runinfo[b * kOxSegPerCta + nr] = ci;
                ++nr;
                c = x;
                ci = xi;
            }
        }
        P.runrec[b * kOxSegPerCta + nr] = c;
        P.runinfo[b * kOxSegPerCta + nr] = ci;
        P.nrun[b] = nr + 1;
        atomicMax(&g_ord_times[2], gtimer());
    }
}

struct OxWalkSmem {
    OrdRec node[kOxNodes];          // tree over the chunk's CTA composites (heap order)
    OrdRec run[kOxRunPool];         // staged run lists
    uint32_t runinfo[kOxRunPool];   // first << 8 | count
    uint32_t runseg[kOxRunPool];    // segment pool slot of an invalid one-segment run, or kOxNoPool
    uint32_t owner[kOxRunPool];     // leaf that owns the staged run
    uint32_t runbase[kOxChunk];     // first staged run of each leaf, or kOxNoPool
    uint32_t leafnr[kOxChunk];      // runs of each leaf
    uint32_t segid[kOxSegPool];     // global segment of each staged serial segment
    __align__(16) float seg[kOxSegPool][kOxSeg];  // staged blocks of serial segments
    uint8_t kind[kOxNodes + 1];     // 0 empty, 1 valid composite, 2 descend
    uint8_t pred[kOxNodes + 1];     // the node's composite is predicted to apply (estimated start)
    uint32_t items[kOxChunk];       // the walk plan: topmost predicted nodes and uncovered leaves
    uint32_t wsum[kOxWalkThreads / 32];
    uint32_t nruns, nsegs, nitems;
};

// The walk (one CTA): per chunk of 1024 record CTAs, stage, build the tree, walk it with warp 0.
__global__ void __launch_bounds__(kOxWalkThreads) ordered_walk_kernel(const OxParams P) {
    extern __shared__ __align__(16) unsigned char ox_smem[];
    OxWalkSmem& W = *reinterpret_cast<OxWalkSmem*>(ox_smem);
    const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    pdl_wait_and_release();
    if (tid == 0) g_ord_times[3] = gtimer();
    float s = 0.0f;
    unsigned long long st[4] = {0, 0, 0, 0};
    for (uint64_t c0 = 0; c0 < P.grid; c0 += kOxChunk) {
        const unsigned long long tc0 = gtimer();
        const uint32_t cn = uint32_t(u64min(kOxChunk, P.grid - c0));
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
            const OrdRec r0 = P.runrec[cb * kOxSegPerCta];
            if (nr == 1 && (r0.hdr & 1)) {
                W.node[li] = r0;
                kd = 1;
            } else {
                kd = 2;
                const uint32_t at = atomicAdd(&W.nruns, nr);
                if (at + nr <= kOxRunPool) {
                    rb = at;
                    for (uint32_t r = 0; r < nr; ++r) W.owner[at + r] = tid;
                } else {
                    // does not fit: walked from global memory; mark its share of the pool unused
                    for (uint32_t r = at; r < at + nr && r < kOxRunPool; ++r) W.owner[r] = kOxNoPool;
                }
            }
        }
        if (tid < L) W.kind[li] = kd;
        W.runbase[tid] = rb;
        W.leafnr[tid] = nr;
        __syncthreads();
        const unsigned long long tc1 = gtimer();
        // stage the runs (one per thread), and reserve a pool slot for each serial segment
        const uint32_t staged = min(W.nruns, kOxRunPool);
        for (uint32_t j = tid; j < staged; j += kOxWalkThreads) {
            const uint32_t t = W.owner[j];
            if (t == kOxNoPool) continue;
            const uint64_t cb = c0 + t;
            const uint32_t r = j - W.runbase[t];
            const OrdRec rr = P.runrec[cb * kOxSegPerCta + r];
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
        // stage the serial segments' blocks, all threads at once
        const uint32_t nseg = min(W.nsegs, kOxSegPool);
        for (uint32_t e2 = tid; e2 < nseg * kOxSeg; e2 += kOxWalkThreads)
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
        for (uint32_t i = tid; i < 2 * L - 1; i += kOxWalkThreads) {
            uint32_t f = i;
            while (f < L - 1) f = 2 * f + 1;   // leftmost leaf
            const uint32_t t = f - (L - 1);
            bool pr = false;
            if (W.kind[i] == 1 && t < cn) pr = rec_applies(W.node[i], float(__ldcg(P.pre + c0 + t)));
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
            const uint32_t v = W.wsum[lane];
            uint32_t inc = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t t2 = __shfl_up_sync(kFull, inc, off);
                if (lane >= uint32_t(off)) inc += t2;
            }
            W.wsum[lane] = inc - v;
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
            for (uint32_t j = 0; j < nit; ++j) {
            const uint32_t root = W.items[j];
            if (W.pred[root] && rec_applies(W.node[root], s)) {
                s = rec_apply(W.node[root], s);
                ++st[0];
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
                    continue;
                }
                // leaf: record CTA cb, its runs (staged or from global)
                const uint32_t t = i - (L - 1);
                const uint64_t cb = c0 + t;
                const uint32_t rb2 = W.runbase[t];
                const uint32_t nr2 = k == 1 ? 1u : W.leafnr[t];
                for (uint32_t r = 0; r < nr2; ++r) {
                    OrdRec rr;
                    uint32_t ri, sl = kOxNoPool;
                    if (k == 1) {
                        rr = W.node[i];
                        ri = kOxSegPerCta;   // segments 0 .. 63
                    } else if (rb2 != kOxNoPool) {
                        rr = W.run[rb2 + r];
                        ri = W.runinfo[rb2 + r];
                        sl = W.runseg[rb2 + r];
                    } else {
                        rr = P.runrec[cb * kOxSegPerCta + r];
                        ri = __ldcg(P.runinfo + cb * kOxSegPerCta + r);
                    }
                    if (rec_applies(rr, s)) {
                        s = rec_apply(rr, s);
                        ++st[1];
                        continue;
                    }
                    const uint32_t sf = ri >> 8, sc = ri & 0xFFu;
                    for (uint32_t q = sf; q < sf + sc; ++q) {
                        const uint64_t gs = cb * kOxSegPerCta + q;
                        if (sc > 1 || (rr.hdr & 1)) {
                            const OrdRec sr = P.segrec[gs];
                            if (rec_applies(sr, s)) {
                                s = rec_apply(sr, s);
                                ++st[2];
                                continue;
                            }
                        }
                        if (sl != kOxNoPool) s = smem_chain32(W.seg[sl], s);
                        else s = warp_chain32(ox_load(P, gs * kOxSeg + lane), s);
                        ++st[3];
                    }
                }
            }
            }
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
        *P.result = s;
    }
}

constexpr size_t kOxSmem = sizeof(OxWalkSmem);

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

size_t ordered_ws_bytes(uint64_t nb) {
    const size_t grid = size_t(ordered_grid(nb));
    return grid * kOxSegPerCta * (2 * sizeof(OrdRec) + sizeof(uint32_t)) + grid * (2 * sizeof(double) + sizeof(uint32_t)) +
           256;
}

cudaError_t launch_ordered_parallel(const float* blocks, const uint32_t* order, uint64_t nb, void* ws, uint32_t* ticket,
                                    float* result, cudaStream_t s) {
    (void)ticket;
    const int dbg = knobs().debug_mode == 41;
    const int grid = ordered_grid(nb);
    static PerDeviceOnce once;
    const cudaError_t ea = once([] {
        return cudaFuncSetAttribute(ordered_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kOxSmem));
    });
    if (ea != cudaSuccess) return ea;
    OxParams P{};
    P.blocks = blocks;
    P.order = order;
    P.nb = nb;
    P.grid = uint32_t(grid);
    char* w = static_cast<char*>(ws);
    const size_t ns = size_t(grid) * kOxSegPerCta;
    // 8-byte members first
    double* agg = reinterpret_cast<double*>(w);
    double* pre = agg + grid;
    P.pre = pre;
    P.segrec = reinterpret_cast<OrdRec*>(pre + grid);
    P.runrec = P.segrec + ns;
    P.runinfo = reinterpret_cast<uint32_t*>(P.runrec + ns);
    P.nrun = P.runinfo + ns;
    P.result = result;
    P.dbg = dbg;
    // four stream-ordered launches with programmatic dependent launch: each grid is scheduled while
    // its predecessor runs and waits on it in-kernel (the launch latencies overlap)
    auto pdl = [&](auto kernel, unsigned g, unsigned t, size_t smem, auto... args) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(g);
        cfg.blockDim = dim3(t);
        cfg.dynamicSmemBytes = smem;
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
    if (e == cudaSuccess) e = pdl(ordered_records_kernel, unsigned(grid), unsigned(kOrdThreads), 0, P);
    if (e == cudaSuccess) e = pdl(ordered_walk_kernel, 1u, unsigned(kOxWalkThreads), kOxSmem, P);
    return e;
}

}  // namespace tcr
