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

// ------------------------------------------------------------------ ascending order, in parallel
//
// The chain can be evaluated exactly without doing it add by add.  While the running sum stays in
// one binade [2^e, 2^(e+1)) (sign sigma), the fp32 values there are the integer multiples T u of
// u = 2^(e-23) with T in [2^23, 2^24), and fl(s + b) = sigma u round(T + sigma b / u), rounding to
// the nearest integer, ties to the EVEN integer (= even mantissa).  So over a group of blocks:
//   q_k = sigma b_k / u (exact in binary64),  r_k = its rounding,  T_{k+1} = T_k + r_k,
// where r_k depends on T_k only through the parity of T_k and only when q_k is an exact tie.
// A group's RECORD for a guessed (sigma, e) holds, for both start parities p0, the total
// sum_k r_k and the min / max of the partial sums; it applies to an actual running sum s iff s is
// normal with that sign and exponent and every partial T stays in [2^23 + 1, 2^24 - 1] (then
// every real T_k + q_k lies strictly inside the binade and the rounding above IS fl's).
// Records of consecutive groups with the same guess compose associatively into runs.
//
//   1. every CTA: approximate prefix of the group partials (binary64) -> a guess per group;
//      one warp per group builds its record (two passes: tie-parity maps, warp scan, sums);
//      thread 0 composes the CTA's groups into runs.
//   2. the last CTA (ticket): one warp walks the runs in order with the actual running sum --
//      apply when the record holds, else the group's records one by one, else the group's
//      blocks add by add (a warp-wide chain).  The result is the serial sum, bit for bit.
//
// Guesses only steer the speed: a wrong one fails its check and the walk falls back.

__device__ __forceinline__ int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ uint64_t u64min(uint64_t a, uint64_t b) { return a < b ? a : b; }

struct OrdRec {                 // 40 bytes
    int32_t hdr;                // bit 0 valid, bit 1 negative, bits 2.. biased exponent of s
    int32_t pad;
    int64_t dT[2];              // sum of r_k for start parity 0 / 1 (|.| < 2^25 when valid)
    int32_t mn[2], mx[2];       // min / max partial sum (relative to T_0) for start parity 0 / 1
};
static_assert(sizeof(OrdRec) == 40, "record layout");

constexpr uint32_t kOrdPer = 64;   // groups per CTA (records and composition in shared memory)

// profiling counters of the last walk: CTA composites applied, group records applied, groups
// added block by block, groups whose record was invalid / unsafe
__device__ unsigned long long g_ord_stats[4];
// profiling: %globaltimer of the first CTA start, the last look-back end, the last record end,
// the walk start and end (min / max over CTAs)
__device__ unsigned long long g_ord_times[5];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct OrdParams {
    const float* blocks;        // block results, ascending
    const float* group_partials;
    uint64_t nb, n_groups;
    uint32_t G;                 // blocks per group
    OrdRec* grec;               // [n_groups] group records
    OrdRec* crec;               // [grid] the CTA's composite (when all its groups are one run)
    uint32_t* cone;             // [grid] 1 iff crec is usable
    double* agg;                // [grid] sum of the CTA's group partials (binary64)
    double* incl;               // [grid] inclusive prefix of agg
    uint32_t* flag;             // [grid] 0 / 1 aggregate / 2 inclusive published; zero on entry, exit
    uint32_t* ticket;           // zero on entry / exit
    float* result;
};

__device__ __forceinline__ bool rec_applies(const OrdRec& r, float s, int64_t* T0out, int* p0out) {
    if (!(r.hdr & 1)) return false;
    const uint32_t bits = __float_as_uint(s);
    const uint32_t ex = (bits >> 23) & 0xFFu;
    if (ex == 0 || ex == 0xFFu) return false;                  // zero, subnormal, inf, NaN
    if (int32_t(ex) != (r.hdr >> 2) || int32_t(bits >> 31) != ((r.hdr >> 1) & 1)) return false;
    const int64_t T0 = int64_t((bits & 0x7FFFFFu) | 0x800000u);
    const int p0 = int(T0 & 1);
    if (T0 + r.mn[p0] < (1 << 23) + 1 || T0 + r.mx[p0] > (1 << 24) - 1) return false;
    *T0out = T0;
    *p0out = p0;
    return true;
}

__device__ __forceinline__ float rec_apply(const OrdRec& r, float s) {
    const uint32_t bits = __float_as_uint(s);
    const int64_t T0 = int64_t((bits & 0x7FFFFFu) | 0x800000u);
    const int64_t T1 = T0 + r.dT[T0 & 1];
    return __uint_as_float((bits & 0xFF800000u) | uint32_t(T1 - (1 << 23)));
}

// Compose b after a (same guess, both valid).
__device__ __forceinline__ OrdRec rec_compose(const OrdRec& a, const OrdRec& b) {
    OrdRec c;
    c.hdr = a.hdr;
    c.pad = 0;
#pragma unroll
    for (int p0 = 0; p0 < 2; ++p0) {
        const int pm = int((p0 + a.dT[p0]) & 1);
        const int64_t d = a.dT[p0];
        c.dT[p0] = d + b.dT[pm];
        const int64_t mn = d + b.mn[pm], mx = d + b.mx[pm];
        // the partial sums stay < 2^25 in magnitude whenever the run can apply; clamp the rest
        // so the check fails instead of overflowing
        c.mn[p0] = int32_t(i64max(-(1ll << 30), i64min(a.mn[p0], mn)));
        c.mx[p0] = int32_t(i64min(1ll << 30, i64max(a.mx[p0], mx)));
    }
    return c;
}

// One warp: the record of blocks [b0, b0 + cnt) for the guess (neg, e); lanes take consecutive
// slices of J = ceil(cnt / 32).
__device__ OrdRec warp_record(const float* blocks, uint64_t b0, uint32_t cnt, bool neg, int e) {
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t J = (cnt + 31) / 32;
    const uint32_t lo = lane * J, hi = min(cnt, lo + J);
    const double scale = ldexp(neg ? -1.0 : 1.0, 23 - (e - 127));   // sigma / u
    bool ok = true;
    // pass 1: the lane's tie-parity map, as its end parity for start parity 0 and 1
    uint32_t pe[2] = {0u, 1u};
    for (uint32_t k = lo; k < hi; ++k) {
        const float b = __ldg(blocks + b0 + k);
        const double q = double(b) * scale;
        ok &= isfinite(b) && fabs(q) < 33554432.0;   // 2^25
        const double f = floor(q), ph = q - f;
        const int64_t fi = int64_t(f);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int64_t r = ph < 0.5 ? fi : (ph > 0.5 ? fi + 1 : fi + ((pe[t] + fi) & 1));
            pe[t] = uint32_t((pe[t] + r) & 1);
        }
    }
    // inclusive warp scan of the maps (compose in lane order), then the lane's start parities
    uint32_t m0 = pe[0], m1 = pe[1];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t a0 = __shfl_up_sync(kFull, m0, off), a1 = __shfl_up_sync(kFull, m1, off);
        if (lane >= uint32_t(off)) {
            // (this after earlier): p -> mine(earlier(p))
            const uint32_t n0 = a0 ? m1 : m0, n1 = a1 ? m1 : m0;
            m0 = n0;
            m1 = n1;
        }
    }
    uint32_t s0 = __shfl_up_sync(kFull, m0, 1), s1 = __shfl_up_sync(kFull, m1, 1);
    if (lane == 0) {
        s0 = 0u;
        s1 = 1u;
    }
    // pass 2: partial sums from the lane's start parities
    int64_t acc[2] = {0, 0}, mn[2] = {INT64_MAX, INT64_MAX}, mx[2] = {INT64_MIN, INT64_MIN};
    uint32_t pp[2] = {s0, s1};
    for (uint32_t k = lo; k < hi; ++k) {
        const float b = __ldg(blocks + b0 + k);
        const double q = double(b) * scale;
        const double f = floor(q), ph = q - f;
        const int64_t fi = int64_t(f);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int64_t r = ph < 0.5 ? fi : (ph > 0.5 ? fi + 1 : fi + ((pp[t] + fi) & 1));
            pp[t] = uint32_t((pp[t] + r) & 1);
            acc[t] += r;
            mn[t] = i64min(mn[t], acc[t]);
            mx[t] = i64max(mx[t], acc[t]);
        }
    }
    // exclusive scan of the lane sums, then the warp's min / max of all partial sums
    OrdRec rec;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        int64_t inc = acc[t];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t a = __shfl_up_sync(kFull, inc, off);
            if (lane >= uint32_t(off)) inc += a;
        }
        const int64_t excl = inc - acc[t];
        int64_t lmn = hi > lo ? excl + mn[t] : INT64_MAX, lmx = hi > lo ? excl + mx[t] : INT64_MIN;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            lmn = i64min(lmn, __shfl_xor_sync(kFull, lmn, off));
            lmx = i64max(lmx, __shfl_xor_sync(kFull, lmx, off));
        }
        rec.dT[t] = __shfl_sync(kFull, inc, 31);
        rec.mn[t] = int32_t(i64max(-(1ll << 30), i64min(lmn, 1ll << 30)));
        rec.mx[t] = int32_t(i64max(-(1ll << 30), i64min(lmx, 1ll << 30)));
    }
    ok = __all_sync(kFull, ok);
    rec.hdr = (ok ? 1 : 0) | (neg ? 2 : 0) | (e << 2);
    rec.pad = 0;
    return rec;
}

// One warp: s + blocks[b0], + blocks[b0 + 1], ... one fp32 add at a time (the reference's loop);
// every lane runs the same chain on broadcast values, so s stays warp-uniform.
__device__ float warp_serial(const float* blocks, uint64_t b0, uint32_t cnt, float s) {
    const unsigned lane = threadIdx.x & 31u;
    for (uint32_t base = 0; base < cnt; base += 32) {
        const uint32_t k = base + lane;
        const float v = k < cnt ? __ldcg(blocks + b0 + k) : 0.0f;
        const uint32_t m = min(32u, cnt - base);
        for (uint32_t i = 0; i < m; ++i) s += __shfl_sync(kFull, v, i);
    }
    return s;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// CTA b owns groups [64 b, 64 b + 64).  The approximate running sum before them comes from a
// decoupled look-back over the CTAs' published aggregates (each CTA publishes its aggregate at
// once and its inclusive prefix as soon as it knows it; a CTA only waits on lower-numbered ones,
// which were scheduled before it), so no separate scan launch is needed.
__global__ void __launch_bounds__(kOrdThreads) ordered_ascending_kernel(const OrdParams P) {
    __shared__ double s_gp[kOrdPer];
    __shared__ double s_S[kOrdPer];
    __shared__ OrdRec s_rec[kOrdPer];
    __shared__ double s_pre;
    __shared__ int s_last;
    __shared__ OrdRec s_wrec[kOrdThreads];
    __shared__ OrdRec s_grp[kOrdPer];
    __shared__ uint32_t s_wone[kOrdThreads];
    const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint64_t b = blockIdx.x;
    const uint64_t ga = b * kOrdPer, gb = u64min(P.n_groups, ga + kOrdPer);
    const uint32_t ng = uint32_t(gb - ga);
    if (tid == 0) atomicMin(&g_ord_times[0], gtimer());
    if (tid < kOrdPer) s_gp[tid] = tid < ng ? double(__ldcg(P.group_partials + ga + tid)) : 0.0;
    __syncthreads();
    if (warp == 0) {
        double a = s_gp[lane] + s_gp[lane + 32];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) a += __shfl_xor_sync(kFull, a, off);
        if (lane == 0) {
            P.agg[b] = a;
            if (b == 0) P.incl[b] = a;
            __threadfence();
            st_release(P.flag + b, b == 0 ? 2u : 1u);
        }
        // look-back: windows of 32 predecessors, nearest first
        double pre = 0.0;
        int64_t j = int64_t(b) - 1;
        while (j >= 0) {
            const int64_t idx = j - int64_t(lane);
            uint32_t f = idx >= 0 ? ld_acquire(P.flag + idx) : 2u;
            const unsigned ready2 = __ballot_sync(kFull, f == 2u);
            const unsigned stop = ready2 ? (__ffs(ready2) - 1) : 31u;      // nearest inclusive (or window end)
            const unsigned zero = __ballot_sync(kFull, f == 0u) & ((stop == 31u && !ready2) ? kFull : ((2u << stop) - 1u));
            if (zero) continue;                                            // a predecessor has not published yet
            double v = 0.0;
            if (idx >= 0 && lane <= stop) v = (ready2 && lane == stop) ? __ldcg(P.incl + idx) : __ldcg(P.agg + idx);
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
            pre += v;
            if (ready2) break;
            j -= 32;
        }
        if (lane == 0) {
            s_pre = pre;
            if (b != 0) {
                P.incl[b] = pre + a;
                __threadfence();
                st_release(P.flag + b, 2u);
            }
        }
    }
    __syncthreads();
    if (tid == 0) atomicMax(&g_ord_times[1], gtimer());
    if (tid == 0) {
        double S = s_pre;
        for (uint32_t i = 0; i < ng; ++i) {
            s_S[i] = S;
            S += s_gp[i];
        }
    }
    __syncthreads();
    // records: warp w takes groups w, w + 8, ... of the CTA
    for (uint32_t i = warp; i < ng; i += kOrdThreads / 32) {
        const double S = s_S[i];
        const uint64_t g = ga + i;
        const uint64_t b0 = g * P.G;
        const uint32_t cnt = uint32_t(u64min(P.G, P.nb - b0));
        // guess: the binade of the approximate sum, unless it is within 1e-3 of a boundary
        int ex = 0;
        const double fr = frexp(fabs(S), &ex);   // |S| = fr 2^ex, fr in [0.5, 1)
        const bool safe = S != 0.0 && fr > 0.5005 && fr < 0.9995 && ex - 1 + 127 >= 1 && ex - 1 + 127 <= 254;
        OrdRec r;
        if (safe) {
            r = warp_record(P.blocks, b0, cnt, S < 0.0, ex - 1 + 127);
        } else {
            r.hdr = 0;
            r.pad = 0;
            r.dT[0] = r.dT[1] = 0;
            r.mn[0] = r.mn[1] = r.mx[0] = r.mx[1] = 0;
        }
        if (lane == 0) {
            s_rec[i] = r;
            P.grec[g] = r;
        }
    }
    __syncthreads();
    if (tid == 0) {
        // the CTA's composite, when all its groups are one run (valid, same guess)
        OrdRec c = s_rec[0];
        bool one = (c.hdr & 1) != 0;
        for (uint32_t i = 1; one && i < ng; ++i) {
            one = s_rec[i].hdr == c.hdr;
            if (one) c = rec_compose(c, s_rec[i]);
        }
        P.crec[b] = c;
        P.cone[b] = one ? 1u : 0u;
        atomicMax(&g_ord_times[2], gtimer());
        unsigned t;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(P.ticket) : "memory");
        s_last = t == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    if (tid == 0) g_ord_times[3] = gtimer();
    // the walk, in block order: chunks of 256 CTAs staged in shared memory by the whole CTA,
    // walked by warp 0 with the actual running sum
    float s = 0.0f;
    unsigned long long st[4] = {0, 0, 0, 0};
    for (uint32_t c0 = 0; c0 < gridDim.x; c0 += kOrdThreads) {
        const uint32_t cn = min(uint32_t(kOrdThreads), gridDim.x - c0);
        if (tid < cn) {
            s_wone[tid] = __ldcg(P.cone + c0 + tid);
            s_wrec[tid] = P.crec[c0 + tid];
        }
        __syncthreads();
        if (warp == 0) {
            for (uint32_t k = 0; k < cn; ++k) {
                int64_t T0;
                int p0;
                if (s_wone[k] && rec_applies(s_wrec[k], s, &T0, &p0)) {
                    s = rec_apply(s_wrec[k], s);
                    if (lane == 0) ++st[0];
                    continue;
                }
                const uint64_t jg0 = uint64_t(c0 + k) * kOrdPer, jg1 = u64min(P.n_groups, jg0 + kOrdPer);
                // the CTA's group records, all at once (one round trip, not one per group)
                for (uint64_t g = jg0 + lane; g < jg1; g += 32) s_grp[g - jg0] = P.grec[g];
                __syncwarp();
                for (uint64_t g = jg0; g < jg1; ++g) {
                    const OrdRec gr = s_grp[g - jg0];
                    if (rec_applies(gr, s, &T0, &p0)) {
                        s = rec_apply(gr, s);
                        if (lane == 0) ++st[1];
                    } else {
                        if (lane == 0) {
                            ++st[2];
                            if (!(gr.hdr & 1)) ++st[3];
                        }
                        const uint64_t b0 = g * P.G;
                        s = warp_serial(P.blocks, b0, uint32_t(u64min(P.G, P.nb - b0)), s);
                    }
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }
    for (uint32_t j = tid; j < gridDim.x; j += kOrdThreads) P.flag[j] = 0u;
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) g_ord_stats[i] = st[i];
        g_ord_times[4] = gtimer();
        *P.result = s;
        *P.ticket = 0u;
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

size_t ordered_ws_bytes(uint64_t n_groups, int grid) {
    return n_groups * sizeof(OrdRec) + size_t(grid) * (sizeof(OrdRec) + 2 * sizeof(double) + 2 * sizeof(uint32_t)) + 256;
}

int ordered_grid(uint64_t n_groups) { return int((n_groups + kOrdPer - 1) / kOrdPer); }

cudaError_t launch_ordered_ascending(const float* blocks, const float* group_partials, uint64_t nb, uint64_t n_groups,
                                     uint32_t G, void* ws, uint32_t* ticket, float* result, cudaStream_t s) {
    const int grid = ordered_grid(n_groups);
    OrdParams P{};
    P.blocks = blocks;
    P.group_partials = group_partials;
    P.nb = nb;
    P.n_groups = n_groups;
    P.G = G;
    char* w = static_cast<char*>(ws);
    P.grec = reinterpret_cast<OrdRec*>(w);
    P.crec = P.grec + n_groups;
    P.agg = reinterpret_cast<double*>(P.crec + grid);
    P.incl = P.agg + grid;
    P.cone = reinterpret_cast<uint32_t*>(P.incl + grid);
    P.flag = P.cone + grid;
    P.ticket = ticket;
    P.result = result;
    ordered_ascending_kernel<<<grid, kOrdThreads, 0, s>>>(P);
    return cudaGetLastError();
}

}  // namespace tcr
