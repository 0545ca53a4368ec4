// tcr_capi.cpp -- the extern "C" boundary (include/tcreduce_b200.h).
//
// Host-side responsibilities only: config validation mirroring the reference
// (reduction.hpp:50-56, fragment.hpp:22-25), per-(device, stream) workspace,
// launch geometry, the pipelined host->device drop-in path, and the reference
// counter formulas.  All arithmetic runs in the sm_100a kernels; there is no
// CPU fallback: a missing device or kernel is an error, never a host loop.
#include "tcreduce_b200.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <utility>

#include "tcr_kernels.h"

#include <dlfcn.h>
#include <nccl.h>

#include <vector>

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;
thread_local int g_engine = 0;  // engine that ran the full groups of the last call
// m != 16 engines: use the NaN-repairing instantiations (tcr_sp_genm.cu, group_epilogue)
thread_local bool g_repair = false;

// NVTX range around each public entry point (visible in nsys / ncu range filters; no cost when
// no tool is attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct RepairScope {
    bool prev;
    explicit RepairScope(bool on) : prev(g_repair) { g_repair = g_repair || on; }
    ~RepairScope() { g_repair = prev; }
};

// Synchronous entry points: a result that comes back NaN with the overflow note set on a
// selector engine (m != 16) may be a 0 x inf artefact -- run the call again with the repairing
// kernels, which reproduce the reference's +-inf / NaN exactly.  Finite data never pays.
template <class F>
int with_nan_retry(const tcr_config* c, tcr_outcome* out, F&& call) {
    int rc = call();
    if (rc == TCR_OK && c && out && c->m != 16 && !g_repair && out->overflow && std::isnan(out->value) &&
        (c->variant == TCR_SINGLE_PASS || c->variant == TCR_RECURRENCE || c->variant == TCR_SPLIT)) {
        RepairScope rs(true);
        rc = call();
    }
    return rc;
}

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define TCR_CUDA(expr)                                                                          \
    do {                                                                                        \
        const cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                                  \
            return fail(TCR_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_));   \
    } while (0)

struct Workspace {
    float* group_partials = nullptr;
    size_t gp_cap = 0;
    float* block_partials = nullptr;
    size_t bp_cap = 0;
    uint32_t* order = nullptr;   // seeded-permutation block order (host-computed, cached)
    size_t order_cap = 0;
    uint64_t order_nb = 0, order_seed = 0;
    bool order_ok = false;
    uint32_t* ord_ws = nullptr;   // ascending ORDERED: group records, runs (tcr_ordered.cu)
    size_t ord_cap = 0;
    // small fixed area: result(float), overflow(u32), ticket(u32), shuffle ticket, exact out[3]
    unsigned char* fixed = nullptr;
    void* exact_ws = nullptr;
    float* shuffle_partials = nullptr;
    void* cub_temp = nullptr;
    size_t cub_cap = 0;
    void* host_pinned = nullptr;  // 64 bytes of result readback
    uint16_t* conv = nullptr;  // fp32 -> binary16 staging for m != 16
    size_t conv_cap = 0;
    // variants: tree columns, double partials, recurrence level buffers, whole-input staging
    float* tree_cols = nullptr;
    size_t tree_cap = 0;
    double* dpart = nullptr;
    size_t dpart_cap = 0;
    float* lvl_f32 = nullptr;
    size_t lvl_f32_cap = 0;
    uint16_t* lvl16[2] = {nullptr, nullptr};
    size_t lvl16_cap[2] = {0, 0};
    float* block_scratch = nullptr;  // split work units of the cp.async engine
    size_t bs_cap = 0;
    uint32_t* group_count = nullptr;  // kept zero between launches
    size_t gc_cap = 0;
    unsigned long long* work_counter = nullptr;  // kept zero between launches
    size_t wc_cap = 0;
    float* stage = nullptr;  // host path of the non-single_pass variants
    size_t stage_cap = 0;
    float* unaligned = nullptr;  // aligned copy of a device input that is not 16-byte aligned
    size_t unaligned_cap = 0;
    // pipelined host path
    float* ring[2] = {nullptr, nullptr};
    uint16_t* ring16[2] = {nullptr, nullptr};
    size_t ring_cap = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
    // pageable host input: a pinned staging ring filled by parallel host copies (kStageSlots
    // slots of kStageBytes), each slot's H2D tracked by an event
    void* pin_stage = nullptr;
    cudaEvent_t pin_free[4] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t pin_seq = 0;
    // split variant: the shuffle32 share on an auxiliary stream
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;

    // Free every device / pinned buffer, stream and event (the owner guarantees no work in flight).
    void release() {
        auto f = [](auto*& ptr) {
            if (ptr) cudaFree(ptr);
            ptr = nullptr;
        };
        f(group_partials); f(block_partials); f(order); f(fixed); f(exact_ws); f(shuffle_partials); f(cub_temp);
        f(conv); f(tree_cols); f(dpart); f(lvl_f32); f(lvl16[0]); f(lvl16[1]); f(block_scratch); f(group_count);
        f(work_counter); f(ord_ws); f(stage); f(unaligned); f(ring[0]); f(ring[1]); f(ring16[0]); f(ring16[1]);
        if (host_pinned) cudaFreeHost(host_pinned);
        host_pinned = nullptr;
        if (pin_stage) cudaFreeHost(pin_stage);
        pin_stage = nullptr;
        for (cudaEvent_t* e : {&pin_free[0], &pin_free[1], &pin_free[2], &pin_free[3]})
            if (*e) cudaEventDestroy(*e), *e = nullptr;
        for (cudaEvent_t* e : {&copied[0], &copied[1], &consumed[0], &consumed[1], &fork, &join})
            if (*e) cudaEventDestroy(*e), *e = nullptr;
        for (cudaStream_t* st : {&copy_stream, &aux_stream})
            if (*st) cudaStreamDestroy(*st), *st = nullptr;
    }

    float* result() { return reinterpret_cast<float*>(fixed); }
    uint32_t* overflow() { return reinterpret_cast<uint32_t*>(fixed + 4); }
    uint32_t* ticket() { return reinterpret_cast<uint32_t*>(fixed + 8); }
    uint32_t* sh_ticket() { return reinterpret_cast<uint32_t*>(fixed + 12); }
    uint32_t* sink() { return reinterpret_cast<uint32_t*>(fixed + 16); }
    uint32_t* var_ticket() { return reinterpret_cast<uint32_t*>(fixed + 20); }
    float* var_result() { return reinterpret_cast<float*>(fixed + 24); }
    double* exact_out() { return reinterpret_cast<double*>(fixed + 32); }
    double* dsum_out() { return reinterpret_cast<double*>(fixed + 64); }
};

std::mutex g_mu;
std::map<std::pair<int, cudaStream_t>, Workspace*> g_ws;
std::vector<std::pair<int, cudaStream_t>> g_reap;   // host streams of exited threads

// Release the workspace bound to (device, stream), if any (no work may be in flight on it).
void release_ws(int dev, cudaStream_t s) {
    Workspace* w = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_ws.find({dev, s});
        if (it == g_ws.end()) return;
        w = it->second;
        g_ws.erase(it);
    }
    if (w) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(dev);
        cudaStreamSynchronize(s);
        w->release();
        delete w;
        cudaSetDevice(cur);
    }
}

void reap_exited_threads() {
    std::vector<std::pair<int, cudaStream_t>> todo;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (g_reap.empty()) return;
        todo.swap(g_reap);
    }
    for (auto& [dev, st] : todo) {
        release_ws(dev, st);
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(dev);
        cudaStreamDestroy(st);
        cudaSetDevice(cur);
    }
}

void reap_exited_threads();

int get_ws(cudaStream_t s, Workspace** out) {
    reap_exited_threads();
    int dev = 0;
    TCR_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_ws.find({dev, s});
    if (it != g_ws.end()) {
        *out = it->second;
        return TCR_OK;
    }
    // built completely before it is published: a failed allocation (OOM) leaves no half-made
    // workspace behind for later calls to write through
    std::unique_ptr<Workspace> w(new Workspace());
    cudaError_t e = cudaMalloc(&w->fixed, 256);
    if (e == cudaSuccess) e = cudaMemset(w->fixed, 0, 256);
    if (e == cudaSuccess) e = cudaMalloc(&w->exact_ws, tcr::exact_ws_bytes());
    if (e == cudaSuccess) e = cudaMalloc(&w->shuffle_partials, sizeof(float) * 8192);
    if (e == cudaSuccess) e = cudaMallocHost(&w->host_pinned, 64);
    if (e != cudaSuccess) {
        w->release();
        return fail(TCR_CUDA_ERROR, std::string("workspace allocation: ") + cudaGetErrorString(e));
    }
    *out = w.get();
    g_ws[{dev, s}] = w.release();
    return TCR_OK;
}

template <class T>
int ensure(T** p, size_t* cap, size_t count, cudaStream_t s) {
    if (*cap >= count) return TCR_OK;
    TCR_CUDA(cudaStreamSynchronize(s));
    if (*p) TCR_CUDA(cudaFree(*p));
    *p = nullptr;
    const size_t want = std::max<size_t>(count, 1024);
    // +16 bytes: a ragged tail's last 16-byte copy line (partial, zero-filled past n) stays
    // inside the allocation even when it starts at the last element
    TCR_CUDA(cudaMalloc(reinterpret_cast<void**>(p), want * sizeof(T) + 16));
    *cap = want;
    return TCR_OK;
}

template <typename T>
int ensure_zero(T** p, size_t* cap, size_t count, cudaStream_t s) {
    if (*cap >= count) return TCR_OK;
    const int rc = ensure(p, cap, count, s);
    if (rc) return rc;
    TCR_CUDA(cudaMemsetAsync(*p, 0, *cap * sizeof(T), s));
    return TCR_OK;
}

int validate_cfg(const tcr_config* c) {
    if (!c) return fail(TCR_INVALID_ARGUMENT, "null config");
    // fragment.hpp:22-25
    if (c->m < 2 || (c->m & (c->m - 1)) != 0)
        return fail(TCR_INVALID_ARGUMENT, "fragment side must be a power of two >= 2");
    // reduction.hpp:52-55
    if (c->R < 1) return fail(TCR_INVALID_ARGUMENT, "R must be >= 1");
    if (c->B < 32 || c->B > 1024 || c->B % 32 != 0)
        return fail(TCR_INVALID_ARGUMENT, "B must be a multiple of 32 in [32, 1024]");
    if (c->f < 0.0 || c->f > 1.0) return fail(TCR_INVALID_ARGUMENT, "f must be in [0, 1]");
    if (c->finalize < TCR_FINALIZE_TREE || c->finalize > TCR_FINALIZE_ATOMIC)
        return fail(TCR_INVALID_ARGUMENT, "unknown finalize mode");
    if (c->atomic_order != TCR_ASCENDING && c->atomic_order != TCR_SEEDED_PERMUTATION)
        return fail(TCR_INVALID_ARGUMENT, "unknown atomic order");
    return TCR_OK;
}

int check_supported(const tcr_config* c) {
    if (c->m != 16) {
        const tcr::SpGeometry g = tcr::make_geometry(1u << 20, c->m, c->R, c->B);
        if (!tcr::genm_supported(g))
            return fail(TCR_NOT_SUPPORTED, "fragment side m=" + std::to_string(c->m) + " with R=" + std::to_string(c->R) +
                                               " exceeds the B200 path's index limits (R*m^2 too large for the "
                                               "32-bit per-chunk cursors)");
    }
    if (c->engine < TCR_ENGINE_AUTO || c->engine > TCR_ENGINE_MMA_SYNC_ASYNC)
        return fail(TCR_INVALID_ARGUMENT, "unknown engine");
    return TCR_OK;
}

// Engine choice for the full groups: explicit, or AUTO = the measured winner when the geometry
// allows it.  The register engine always takes the ragged tail and the fp32 input path.
int pick_engine(const tcr_config* c, const tcr::SpGeometry& g, bool f32) {
    if (f32) return TCR_ENGINE_MMA_SYNC_REGS;
    uint32_t a, b;
    const bool full = g.n / g.group_elems > 0;
    switch (c->engine) {
    case TCR_ENGINE_TCGEN05: return full && tcr::tc05_plan(g, &a, &b) ? TCR_ENGINE_TCGEN05 : TCR_ENGINE_MMA_SYNC_REGS;
    case TCR_ENGINE_MMA_SYNC: return tcr::bulk_supported(g) ? TCR_ENGINE_MMA_SYNC : TCR_ENGINE_MMA_SYNC_REGS;
    case TCR_ENGINE_MMA_SYNC_REGS: return TCR_ENGINE_MMA_SYNC_REGS;
    case TCR_ENGINE_MMA_SYNC_ASYNC: return TCR_ENGINE_MMA_SYNC_ASYNC;
    default:
        // AUTO: the measured winner on B200 for binary16 input (DESIGN.md §3 table):
        // per-warp cp.async pipeline 6.1 TB/s > TMA-bulk mma.sync 4.5 > register mma.sync 3.6 >
        // tcgen05 2.8 (n = 2^30, R = 1, B = 1024)
        return TCR_ENGINE_MMA_SYNC_ASYNC;
    }
}

uint64_t next_pow2(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

void counters(uint64_t n, const tcr_config* c, tcr_outcome* o) {
    // reduction.hpp:240-242 and :270-273, :95-96, :177, :182, :267
    const tcr::SpGeometry g = tcr::make_geometry(n, c->m, c->R, c->B);
    const uint64_t P = next_pow2(g.W);
    uint64_t lv = 0;
    for (uint64_t len = P; len > 1; len /= 2) ++lv;
    o->level_count = 1;
    o->sim_steps = 2ull * c->R + 2 + lv + g.n_blocks;
    o->mma_count = g.n_blocks * g.W * (c->R + 1ull);
    o->atomic_count = g.n_blocks;
    o->shuffle_count = g.n_blocks * (P - 1);
}

// A seeded-permutation atomic order asks for the reference's serial combine in that order
// (reduction.hpp:257-268): honour it even when finalize was left at TREE, which has no order to
// permute (otherwise the seed would be silently ignored).
tcr_config normalized(const tcr_config* c) {
    tcr_config n = *c;
    if (n.atomic_order == TCR_SEEDED_PERMUTATION && n.finalize == TCR_FINALIZE_TREE) n.finalize = TCR_FINALIZE_ORDERED;
    return n;
}

// Enqueue single_pass over groups [g0, g1) of a (possibly chunked) input: the streaming kernel
// (block results, group partials, TREE / ATOMIC finalise in its last CTA).
int enqueue_sp_main(const void* x, uint64_t x_offset, uint64_t n, const tcr_config* c_in, bool f32, float* d_result,
                    uint32_t* d_overflow, float* d_blocks, Workspace* w, cudaStream_t s, uint64_t g0, uint64_t g1,
                    bool finalize_here) {
    const tcr_config cn = normalized(c_in);
    const tcr_config* c = &cn;
    const tcr::SpGeometry g = tcr::make_geometry(n, c->m, c->R, c->B);
    tcr::SpParams p{};
    p.x = static_cast<const char*>(x) - x_offset * (f32 ? 4 : 2);
    p.n = n;
    p.R = c->R;
    p.W = g.W;
    p.G = g.G;
    p.chunk_elems = g.chunk_elems;
    p.n_blocks = g.n_blocks;
    p.n_groups = g.n_groups;
    p.group_begin = g0;
    p.group_end = g1;
    int rc = ensure(&w->group_partials, &w->gp_cap, g.n_groups, s);
    if (rc) return rc;
    p.group_partials = w->group_partials;
    p.block_partials = d_blocks;
    if (c->finalize == TCR_FINALIZE_ORDERED && !d_blocks) {
        rc = ensure(&w->block_partials, &w->bp_cap, g.n_blocks, s);
        if (rc) return rc;
        p.block_partials = w->block_partials;
        if (c->atomic_order == TCR_SEEDED_PERMUTATION) {
            rc = ensure(&w->order, &w->order_cap, g.n_blocks, s);
            if (rc) return rc;
        }
    }
    p.order_scratch = w->order;
    p.result = d_result;
    p.overflow = d_overflow;
    p.ticket = w->ticket();
    p.finalize = finalize_here ? c->finalize : tcr::kFinNone;
    if (c->finalize == TCR_FINALIZE_ATOMIC) p.finalize = tcr::kFinAtomic;
    p.atomic_order = c->atomic_order;
    p.atomic_seed = c->atomic_seed;
    p.debug_mode = tcr::knobs().debug_mode;   // 0 unless tcr_enable_profiling_knobs()
    p.split = 1;
    if (c->finalize == TCR_FINALIZE_ATOMIC && g0 == 0) {
        TCR_CUDA(cudaMemsetAsync(d_result, 0, sizeof(float), s));
        ++g_launches;
    }
    if (c->m != 16) {
        // m != 16: the selector-matrix engine; fp32 input straight in where the natural layout
        // takes it (from_single fused into the load), else callers convert first
        if (f32 && !tcr::genm_f32_supported(g)) return fail(TCR_NOT_SUPPORTED, "internal: this m needs binary16 input");
        g_engine = TCR_ENGINE_MMA_SYNC_ASYNC;
        TCR_CUDA(tcr::launch_genm(p, g, s, g_repair, f32));
        ++g_launches;
        return TCR_OK;
    }
    int engine = pick_engine(c, g, f32);
    // a partial group range (pipelined host path) can only run on engines that take any range
    if ((g0 != 0 || g1 != g.n_groups) && (engine == TCR_ENGINE_TCGEN05 || engine == TCR_ENGINE_MMA_SYNC))
        engine = TCR_ENGINE_MMA_SYNC_REGS;
    g_engine = engine;
    if (engine == TCR_ENGINE_MMA_SYNC_ASYNC) {
        const uint64_t maxg = uint64_t(tcr::async_max_grid(c->R, p.debug_mode));
        const bool dyn = tcr::async_plan(g, &p, int(maxg));
        if (p.split > 1 || p.split_tail > 1) {
            rc = ensure(&w->block_scratch, &w->bs_cap, g.n_groups * g.G, s);
            if (rc) return rc;
            rc = ensure_zero(&w->group_count, &w->gc_cap, g.n_groups, s);
            if (rc) return rc;
            p.block_scratch = w->block_scratch;
            p.group_count = w->group_count;
        }
        if (dyn) {
            rc = ensure_zero(&w->work_counter, &w->wc_cap, 1, s);
            if (rc) return rc;
            p.work_counter = w->work_counter;
        }
        const uint64_t units = (p.tail_group - p.group_begin) * p.split + (p.group_end - p.tail_group) * p.split_tail;
        const int grid = int(std::min<uint64_t>(units, maxg));
        TCR_CUDA(tcr::launch_async(p, grid, s));
        ++g_launches;
        return TCR_OK;
    }
    if (engine == TCR_ENGINE_MMA_SYNC) {
        // full groups on the TMA-fed engine, the ragged tail group (if any) on the register
        // engine in a second launch that finalises
        const uint64_t n_tiles = n / g.group_elems;
        tcr::SpParams pt = p;
        pt.group_begin = 0;
        pt.group_end = n_tiles;
        if (n_tiles < g.n_groups) pt.finalize = tcr::kFinNone;
        if (c->finalize == TCR_FINALIZE_ATOMIC) pt.finalize = tcr::kFinAtomic;
        const int maxg = tcr::bulk_max_grid(c->R, p.debug_mode);
        if (maxg <= 0) return fail(TCR_CUDA_ERROR, "TMA engine: shared-memory opt-in failed");
        tcr::bulk_plan(g, &pt, maxg);
        if (pt.split > 1 || pt.split_tail > 1) {
            rc = ensure(&w->block_scratch, &w->bs_cap, g.n_groups * g.G, s);
            if (rc) return rc;
            rc = ensure_zero(&w->group_count, &w->gc_cap, g.n_groups, s);
            if (rc) return rc;
            pt.block_scratch = w->block_scratch;
            pt.group_count = w->group_count;
        }
        rc = ensure_zero(&w->work_counter, &w->wc_cap, 1, s);
        if (rc) return rc;
        pt.work_counter = w->work_counter;
        const uint64_t units = (pt.tail_group - pt.group_begin) * pt.split + (pt.group_end - pt.tail_group) * pt.split_tail;
        TCR_CUDA(tcr::launch_bulk(pt, int(std::min<uint64_t>(units, uint64_t(maxg))), s));
        ++g_launches;
        if (n_tiles == g.n_groups) return TCR_OK;
        p.group_begin = n_tiles;
    }
    if (engine == TCR_ENGINE_TCGEN05) {
        // full groups on the tcgen05 engine (one CTA per SM), the ragged tail (< 1 group) on the
        // register engine; the last launch finalises
        const uint64_t n_tiles = n / g.group_elems;
        tcr::SpParams pt = p;
        pt.group_begin = 0;
        pt.group_end = n_tiles;
        if (n_tiles < g.n_groups) pt.finalize = tcr::kFinNone;
        if (c->finalize == TCR_FINALIZE_ATOMIC) pt.finalize = tcr::kFinAtomic;
        const int grid = int(std::min<uint64_t>(n_tiles, uint64_t(tcr::sm_count())));
        TCR_CUDA(tcr::launch_tc05(pt, g, n_tiles, grid, s));
        ++g_launches;
        if (n_tiles == g.n_groups) return TCR_OK;
        p.group_begin = n_tiles;
    }
    const uint64_t groups = p.group_end - p.group_begin;
    const int maxg = tcr::single_pass_m16_max_grid(f32, c->R);
    const int grid = int(std::min<uint64_t>(groups, uint64_t(maxg)));
    TCR_CUDA(tcr::launch_single_pass_m16(p, f32, grid, s));
    ++g_launches;
    return TCR_OK;
}

// The reference's block order for a seeded permutation (reduction.hpp:257-268: Fisher-Yates driven
// by SplitMix64(atomic_seed), rng.hpp), computed once on the host per (blocks, seed) and kept in
// the workspace.
int ensure_order(Workspace* w, uint64_t nb, uint64_t seed, cudaStream_t s) {
    if (w->order_nb == nb && w->order_seed == seed && w->order_ok) return TCR_OK;
    std::vector<uint32_t> ord(nb);
    for (uint64_t i = 0; i < nb; ++i) ord[i] = uint32_t(i);
    uint64_t st = seed;
    for (uint64_t i = nb; i > 1; --i) {
        st += 0x9E3779B97F4A7C15ull;
        uint64_t z = st;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        std::swap(ord[i - 1], ord[z % i]);
    }
    w->order_ok = false;
    int rc = ensure(&w->order, &w->order_cap, nb, s);
    if (rc) return rc;
    TCR_CUDA(cudaMemcpyAsync(w->order, ord.data(), nb * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    TCR_CUDA(cudaStreamSynchronize(s));   // the host vector goes out of scope
    w->order_nb = nb;
    w->order_seed = seed;
    w->order_ok = true;
    return TCR_OK;
}

// ORDERED finalise: the reference's serial fp32 chain over the published block results, in
// ascending or seeded-permutation order, evaluated in parallel and bit for bit (tcr_ordered.cu).
int enqueue_ordered(uint64_t n, const tcr_config* c, const float* blocks, float* d_result, Workspace* w, cudaStream_t s) {
    const tcr::SpGeometry g = tcr::make_geometry(n, c->m, c->R, c->B);
    const uint32_t* order = nullptr;
    if (c->atomic_order == TCR_SEEDED_PERMUTATION) {
        int rc = ensure_order(w, g.n_blocks, c->atomic_seed, s);
        if (rc) return rc;
        order = w->order;
    }
    if (tcr::knobs().debug_mode == 40) {   // profiling only: the literal serial chain
        TCR_CUDA(tcr::launch_ordered(blocks, order, g.n_blocks, d_result, s));
        ++g_launches;
        return TCR_OK;
    }
    const size_t bytes = tcr::ordered_ws_bytes(g.n_blocks);
    int rc = ensure_zero(&w->ord_ws, &w->ord_cap, (bytes + 3) / 4, s);   // look-back flags start at 0
    if (rc) return rc;
    TCR_CUDA(tcr::launch_ordered_parallel(blocks, order, g.n_blocks, w->ord_ws, w->ticket(), d_result, s));
    ++g_launches;
    return TCR_OK;
}

int enqueue_sp(const void* x, uint64_t x_offset, uint64_t n, const tcr_config* c_in, bool f32, float* d_result,
               uint32_t* d_overflow, float* d_blocks, Workspace* w, cudaStream_t s, uint64_t g0, uint64_t g1,
               bool finalize_here) {
    const tcr_config cn = normalized(c_in);
    if (cn.finalize != TCR_FINALIZE_ORDERED || !finalize_here)
        return enqueue_sp_main(x, x_offset, n, &cn, f32, d_result, d_overflow, d_blocks, w, s, g0, g1, finalize_here);
    // ORDERED: the streaming kernel publishes the block results, then the ordered chain
    int rc = enqueue_sp_main(x, x_offset, n, &cn, f32, d_result, d_overflow, d_blocks, w, s, g0, g1, false);
    if (rc) return rc;
    return enqueue_ordered(n, &cn, d_blocks ? d_blocks : w->block_partials, d_result, w, s);
}

int enqueue_finalize(uint64_t n, const tcr_config* c_in, float* d_result, Workspace* w, cudaStream_t s) {
    const tcr_config cn = normalized(c_in);
    const tcr_config* c = &cn;
    if (c->finalize == TCR_FINALIZE_ATOMIC) return TCR_OK;
    if (c->finalize == TCR_FINALIZE_ORDERED) return enqueue_ordered(n, c, w->block_partials, d_result, w, s);
    const tcr::SpGeometry g = tcr::make_geometry(n, c->m, c->R, c->B);
    tcr::SpParams p{};
    p.n = n;
    p.R = c->R;
    p.W = g.W;
    p.G = g.G;
    p.n_blocks = g.n_blocks;
    p.n_groups = g.n_groups;
    p.group_partials = w->group_partials;
    p.block_partials = w->block_partials;
    p.order_scratch = w->order;
    p.result = d_result;
    p.finalize = c->finalize;
    p.atomic_order = c->atomic_order;
    p.atomic_seed = c->atomic_seed;
    TCR_CUDA(tcr::launch_finalize(p, s));
    ++g_launches;
    return TCR_OK;
}

// The kernels stream 16-byte lines: an input that does not start on a 16-byte boundary (e.g. a
// tensor slice; the reference takes any span) is first copied into an aligned workspace buffer.
int aligned_input(const void** d_x, size_t n, bool f32, Workspace* w, cudaStream_t s) {
    if (reinterpret_cast<uintptr_t>(*d_x) % 16 == 0) return TCR_OK;
    const size_t bytes = n * (f32 ? 4 : 2);
    int rc = ensure(&w->unaligned, &w->unaligned_cap, (bytes + 3) / 4, s);
    if (rc) return rc;
    TCR_CUDA(cudaMemcpyAsync(w->unaligned, *d_x, bytes, cudaMemcpyDeviceToDevice, s));
    *d_x = w->unaligned;
    return TCR_OK;
}

int sp_async(const void* d_x, size_t n, const tcr_config* c, bool f32, float* d_result, uint32_t* d_overflow,
             cudaStream_t s) {
    g_launches = 0;
    if (n == 0) return fail(TCR_INVALID_ARGUMENT, "input must be non-empty");  // reduction.hpp:282
    int rc = validate_cfg(c);
    if (rc) return rc;
    rc = check_supported(c);
    if (rc) return rc;
    if (!d_x || !d_result || !d_overflow) return fail(TCR_INVALID_ARGUMENT, "null device pointer");
    Workspace* w = nullptr;
    rc = get_ws(s, &w);
    if (rc) return rc;
    rc = aligned_input(&d_x, n, f32, w, s);
    if (rc) return rc;
    const tcr::SpGeometry g = tcr::make_geometry(n, c->m, c->R, c->B);
    if (f32 && c->m != 16 && !tcr::genm_f32_supported(g)) {
        // from_single (fragment.hpp:68) applied up front, then the binary16 engine
        rc = ensure(&w->conv, &w->conv_cap, n, s);
        if (rc) return rc;
        TCR_CUDA(tcr::launch_convert_f32_f16(static_cast<const float*>(d_x), w->conv, n, s));
        ++g_launches;
        return enqueue_sp(w->conv, 0, n, c, false, d_result, d_overflow, nullptr, w, s, 0, g.n_groups, true);
    }
    return enqueue_sp(d_x, 0, n, c, f32, d_result, d_overflow, nullptr, w, s, 0, g.n_groups, true);
}

int read_result(Workspace* w, cudaStream_t s, float* value, uint32_t* ovf) {
    TCR_CUDA(cudaMemcpyAsync(w->host_pinned, w->fixed, 8, cudaMemcpyDeviceToHost, s));
    TCR_CUDA(cudaStreamSynchronize(s));
    std::memcpy(value, w->host_pinned, 4);
    std::memcpy(ovf, static_cast<char*>(w->host_pinned) + 4, 4);
    return TCR_OK;
}


// ------------------------------------------------------------------ the other variants (:344-358)

int sync_read(void* host, const void* dev, size_t bytes, Workspace* w, cudaStream_t s) {
    TCR_CUDA(cudaMemcpyAsync(w->host_pinned, dev, bytes, cudaMemcpyDeviceToHost, s));
    TCR_CUDA(cudaStreamSynchronize(s));
    std::memcpy(host, w->host_pinned, bytes);
    return TCR_OK;
}

uint64_t levels_of(uint64_t n) {  // pairwise_tree levels of a pow2-padded length (reduction.hpp:90-101)
    uint64_t P = 1, lv = 0;
    while (P < n) {
        P <<= 1;
        ++lv;
    }
    return lv;
}

// shuffle32 (:113-122) / half_tree (:126-151): bit-exact strided pairwise tree.
int run_tree(const void* d_x, bool f32, uint64_t n, bool half, tcr_outcome* out, Workspace* w, cudaStream_t s) {
    if (n == 0) return fail(TCR_INVALID_ARGUMENT, "input must be non-empty");
    int rc = ensure(&w->tree_cols, &w->tree_cap, tcr::tree_cols_needed(n), s);
    if (rc) return rc;
    TCR_CUDA(cudaMemsetAsync(w->overflow(), 0, 4, s));
    TCR_CUDA(tcr::launch_pairwise_tree(d_x, f32, n, half, w->tree_cols, w->var_result(), w->overflow(), s));
    g_launches += tcr::tree_launches(n);
    float v;
    uint32_t o;
    rc = sync_read(&v, w->var_result(), 4, w, s);
    if (rc) return rc;
    rc = sync_read(&o, w->overflow(), 4, w, s);
    if (rc) return rc;
    const uint64_t lv = levels_of(n);
    out->value = v;
    out->overflow = half && o ? 1 : 0;
    out->level_count = lv;
    out->sim_steps = 4 * lv;
    out->shuffle_count = (1ull << lv) - 1;
    return TCR_OK;
}

// oracle64 (:106-110): the reference's left-to-right binary64 sum, bit for bit -- the serial
// chain evaluated in parallel (tcr_ordered.cu, binary64 records).
int run_oracle64(const void* d_x, bool f32, uint64_t n, tcr_outcome* out, Workspace* w, cudaStream_t s) {
    out->value = 0.0;
    if (n == 0) return TCR_OK;   // the reference's oracle64 of an empty span is 0
    const size_t bytes = tcr::ordered_ws_bytes(n, true);
    int rc = ensure_zero(&w->ord_ws, &w->ord_cap, (bytes + 3) / 4, s);
    if (rc) return rc;
    TCR_CUDA(tcr::launch_serial_sum64(d_x, f32, n, w->ord_ws, w->dsum_out(), s));
    g_launches += 4;
    return sync_read(&out->value, w->dsum_out(), 8, w, s);
}

// single_pass with the result read back (used by recurrence / split)
int run_single_pass(const void* d_x, bool f32, uint64_t n, const tcr_config* c, tcr_outcome* out, Workspace* w,
                    cudaStream_t s) {
    TCR_CUDA(cudaMemsetAsync(w->overflow(), 0, 4, s));
    const int before = g_launches;
    int rc = sp_async(d_x, n, c, f32, w->result(), w->overflow(), s);
    if (rc) return rc;
    g_launches += before + 1;
    float v;
    uint32_t o;
    rc = read_result(w, s, &v, &o);
    if (rc) return rc;
    std::memset(out, 0, sizeof *out);
    out->value = v;
    out->overflow = o ? 1 : 0;
    counters(n, c, out);
    return TCR_OK;
}

// recurrence (:189-231): levels of chained_warp_reduce with binary16 inter-level partials.  A
// level's chunk results are single_pass block results at B = 32 (one warp chunk per block).
int run_recurrence(const void* d_x, bool f32, uint64_t n0, const tcr_config* c, tcr_outcome* out, Workspace* w,
                   cudaStream_t s) {
    if (n0 == 0) return fail(TCR_INVALID_ARGUMENT, "input must be non-empty");
    const uint64_t group = uint64_t(c->m) * c->m, chunk = group * c->R;
    std::memset(out, 0, sizeof *out);
    tcr_config cb = *c;
    cb.variant = TCR_SINGLE_PASS;
    cb.B = 32;
    cb.finalize = TCR_FINALIZE_TREE;
    uint32_t ovf_any = 0;
    const void* cur = d_x;
    bool cur_f32 = f32;
    uint64_t n = n0;
    int nb = 0;
    // the overflow flag accumulates (OR) over the levels on the device: one read at the end
    TCR_CUDA(cudaMemsetAsync(w->overflow(), 0, 4, s));
    while (n >= group) {
        const uint64_t count = (n + chunk - 1) / chunk;
        int rc = ensure(&w->lvl_f32, &w->lvl_f32_cap, count, s);
        if (rc) return rc;
        rc = ensure(&w->lvl16[nb], &w->lvl16_cap[nb], count, s);
        if (rc) return rc;
        const tcr::SpGeometry g = tcr::make_geometry(n, cb.m, cb.R, cb.B);
        if (cur_f32 && cb.m != 16 && !tcr::genm_f32_supported(g)) {
            rc = ensure(&w->conv, &w->conv_cap, n, s);
            if (rc) return rc;
            TCR_CUDA(tcr::launch_convert_f32_f16(static_cast<const float*>(cur), w->conv, n, s));
            cur = w->conv;
            cur_f32 = false;
        }
        rc = enqueue_sp(cur, 0, n, &cb, cur_f32, w->result(), w->overflow(), w->lvl_f32, w, s, 0, g.n_groups, true);
        if (rc) return rc;
        TCR_CUDA(tcr::launch_round_level(w->lvl_f32, w->lvl16[nb], count, w->overflow(), s));
        ++g_launches;
        cur = w->lvl16[nb];
        cur_f32 = false;
        nb ^= 1;
        n = count;
        ++out->level_count;
        out->sim_steps += 2ull * c->R + 3;
        out->mma_count += count * (c->R + 1ull);
    }
    {
        uint32_t o;
        int rc = sync_read(&o, w->overflow(), 4, w, s);
        if (rc) return rc;
        ovf_any |= o;
    }
    if (n == 1) {
        if (cur_f32) {
            float v;
            int rc = sync_read(&v, cur, 4, w, s);
            if (rc) return rc;
            out->value = v;
        } else {
            uint16_t h;
            int rc = sync_read(&h, cur, 2, w, s);
            if (rc) return rc;
            uint32_t u = uint32_t(h & 0x8000u) << 16;
            const uint32_t e = (h >> 10) & 31u, mnt = h & 1023u;
            float f;
            if (e == 0) {
                f = float(mnt) * 0x1.0p-24f;
                std::memcpy(&u, &f, 4);
                u |= uint32_t(h & 0x8000u) << 16;
            } else if (e == 31) {
                u |= 0x7F800000u | (mnt << 13);
            } else {
                u |= ((e + 112) << 23) | (mnt << 13);
            }
            std::memcpy(&f, &u, 4);
            out->value = f;
        }
    } else {
        // leftover shorter than one group: zero-padded two-step reduce with R = 1 (:218-223)
        tcr_config c1 = cb;
        c1.R = 1;
        tcr_outcome o1;
        int rc = run_single_pass(cur, cur_f32, n, &c1, &o1, w, s);
        if (rc) return rc;
        out->value = o1.value;
        ovf_any |= uint32_t(o1.overflow);
        out->sim_steps += 5;
        out->mma_count += 2;
    }
    out->overflow = ovf_any ? 1 : 0;
    return TCR_OK;
}

// split (:298-341): tensor share at R = 1 through single_pass, the rest through shuffle32 --
// the two shares run CONCURRENTLY (the tree on an auxiliary stream forked from and joined back
// into the caller's), as the paper's variant #3 intends; one host read.
int run_split(const void* d_x, bool f32, uint64_t n, const tcr_config* c, tcr_outcome* out, Workspace* w,
              cudaStream_t s) {
    if (n == 0) return fail(TCR_INVALID_ARGUMENT, "input must be non-empty");
    std::memset(out, 0, sizeof *out);
    tcr_config tc = *c;
    tc.variant = TCR_SINGLE_PASS;
    tc.R = 1;
    const uint64_t chunk_block = uint64_t(c->m) * c->m * (c->B / 32);
    uint64_t tensor_len = uint64_t(c->f * double(n));
    tensor_len = tensor_len / chunk_block * chunk_block;
    const uint64_t tree_len = n - tensor_len;
    int launches = 0;
    if (tree_len > 0) {
        int rc = ensure(&w->tree_cols, &w->tree_cap, tcr::tree_cols_needed(tree_len), s);
        if (rc) return rc;
        if (!w->aux_stream) {
            TCR_CUDA(cudaStreamCreateWithFlags(&w->aux_stream, cudaStreamNonBlocking));
            TCR_CUDA(cudaEventCreateWithFlags(&w->fork, cudaEventDisableTiming));
            TCR_CUDA(cudaEventCreateWithFlags(&w->join, cudaEventDisableTiming));
        }
    }
    TCR_CUDA(cudaMemsetAsync(w->overflow(), 0, 4, s));
    if (tensor_len > 0) {
        int rc = sp_async(d_x, tensor_len, &tc, f32, w->result(), w->overflow(), s);
        if (rc) return rc;
        launches += g_launches;
    }
    if (tree_len > 0) {
        TCR_CUDA(cudaEventRecord(w->fork, s));
        TCR_CUDA(cudaStreamWaitEvent(w->aux_stream, w->fork, 0));
        const char* base = static_cast<const char*>(d_x) + tensor_len * (f32 ? 4 : 2);
        TCR_CUDA(tcr::launch_pairwise_tree(base, f32, tree_len, false, w->tree_cols, w->var_result(), w->sink(),
                                           w->aux_stream));
        launches += tcr::tree_launches(tree_len);
        TCR_CUDA(cudaEventRecord(w->join, w->aux_stream));
        TCR_CUDA(cudaStreamWaitEvent(s, w->join, 0));
    }
    g_launches = launches;
    unsigned char h[32];
    int rc = sync_read(h, w->fixed, 32, w, s);
    if (rc) return rc;
    float tensor_part = 0.0f, shuffle_part = 0.0f;
    uint32_t ovf = 0;
    std::memcpy(&tensor_part, h, 4);
    std::memcpy(&ovf, h + 4, 4);
    std::memcpy(&shuffle_part, h + 24, 4);
    tcr_outcome t{}, sh{};
    if (tensor_len > 0) {
        counters(tensor_len, &tc, &t);
        t.overflow = ovf ? 1 : 0;
        out->level_count = 1;
    }
    if (tree_len > 0) {
        const uint64_t lv = levels_of(tree_len);
        sh.level_count = lv;
        sh.sim_steps = 4 * lv;
        sh.shuffle_count = (1ull << lv) - 1;
        out->shuffle_count = sh.shuffle_count;
        out->level_count = std::max<uint64_t>(out->level_count, sh.level_count);
    }
    if (tensor_len == 0) out->value = shuffle_part;
    else if (tree_len == 0) out->value = tensor_part;
    else out->value = tensor_part + shuffle_part;
    out->overflow = t.overflow;
    out->sim_steps = std::max(t.sim_steps, sh.sim_steps) + ((tensor_len > 0 && tree_len > 0) ? 1 : 0);
    out->mma_count = t.mma_count;
    out->atomic_count = t.atomic_count;
    out->shuffle_count += t.shuffle_count;
    return TCR_OK;
}

int run_variant(const void* d_x, bool f32, uint64_t n, const tcr_config* c, tcr_outcome* out, Workspace* w,
                cudaStream_t s) {
    switch (c->variant) {
    case TCR_ORACLE64: return run_oracle64(d_x, f32, n, out, w, s);
    case TCR_SHUFFLE32: return run_tree(d_x, f32, n, false, out, w, s);
    case TCR_HALF_TREE: return run_tree(d_x, f32, n, true, out, w, s);
    case TCR_RECURRENCE: {
        int rc = validate_cfg(c);
        if (rc) return rc;
        rc = check_supported(c);
        if (rc) return rc;
        return run_recurrence(d_x, f32, n, c, out, w, s);
    }
    case TCR_SPLIT: {
        if (n == 0) return fail(TCR_INVALID_ARGUMENT, "input must be non-empty");
        int rc = validate_cfg(c);
        if (rc) return rc;
        rc = check_supported(c);
        if (rc) return rc;
        return run_split(d_x, f32, n, c, out, w, s);
    }
    default: return fail(TCR_INVALID_ARGUMENT, "unknown variant");
    }
}

int reduce_device(const void* d_x, size_t n, const tcr_config* c, tcr_outcome* out, bool f32, cudaStream_t s) {
    if (!out) return fail(TCR_INVALID_ARGUMENT, "null outcome");
    std::memset(out, 0, sizeof *out);
    if (!c) return fail(TCR_INVALID_ARGUMENT, "null config");
    Workspace* w = nullptr;
    int rc = get_ws(s, &w);
    if (rc) return rc;
    if (c->variant != TCR_SINGLE_PASS) {
        g_launches = 0;
        if (n > 0 && d_x) {
            rc = aligned_input(&d_x, n, f32, w, s);
            if (rc) return rc;
        }
        return run_variant(d_x, f32, n, c, out, w, s);
    }
    TCR_CUDA(cudaMemsetAsync(w->overflow(), 0, 4, s));
    rc = sp_async(d_x, n, c, f32, w->result(), w->overflow(), s);
    if (rc) return rc;
    ++g_launches;  // memset
    float v;
    uint32_t o;
    rc = read_result(w, s, &v, &o);
    if (rc) return rc;
    out->value = v;
    out->overflow = o ? 1 : 0;
    counters(n, c, out);
    return TCR_OK;
}

}  // namespace

extern "C" {

void tcr_config_init(tcr_config* c) {
    std::memset(c, 0, sizeof *c);
    c->variant = TCR_SINGLE_PASS;
    c->m = 4;
    c->R = 1;
    c->B = 128;
    c->f = 0.5;
    c->atomic_order = TCR_ASCENDING;
    c->atomic_seed = 0;
    c->finalize = TCR_FINALIZE_ORDERED;   // the reference's combine: drop-in callers get its value
    c->engine = TCR_ENGINE_AUTO;
}

int tcr_validate(const tcr_config* c) { return validate_cfg(c); }

const char* tcr_last_error(void) { return g_err.c_str(); }
const char* tcr_version(void) { return "tcreduce-b200 0.1 (sm_100a)"; }
int tcr_last_launch_count(void) { return g_launches; }

int tcr_release_stream(void* stream) {
    int dev = 0;
    TCR_CUDA(cudaGetDevice(&dev));
    release_ws(dev, static_cast<cudaStream_t>(stream));
    return TCR_OK;
}

int tcr_release_all(void) {
    reap_exited_threads();
    std::vector<std::pair<int, cudaStream_t>> keys;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (auto& kv : g_ws) keys.push_back(kv.first);
    }
    for (auto& k : keys) release_ws(k.first, k.second);
    return TCR_OK;
}
int tcr_last_engine(void) { return g_engine; }
// Profiling hook (not in the public header): timestamps of the last TCR_DEBUG_MODE=20 launch of
// the cp.async engine, 4 per CTA (start, streaming done, after finalise, is-last).
int tcr_debug_timestamps(unsigned long long* host, size_t count) { return tcr::debug_timestamps(host, count); }

size_t tcr_block_count(size_t n, const tcr_config* c) {
    if (!c || validate_cfg(c)) return 0;
    return tcr::make_geometry(n, c->m, c->R, c->B).n_blocks;
}

size_t tcr_group_elems(const tcr_config* c) {
    if (!c || validate_cfg(c)) return 0;
    return tcr::make_geometry(1, c->m, c->R, c->B).group_elems;
}

int tcr_single_pass_counters(size_t n, const tcr_config* c, tcr_outcome* out) {
    int rc = validate_cfg(c);
    if (rc) return rc;
    std::memset(out, 0, sizeof *out);
    counters(n, c, out);
    return TCR_OK;
}

int tcr_single_pass_f16_async(const uint16_t* d_x, size_t n, const tcr_config* c, float* d_result,
                              uint32_t* d_overflow, void* stream) {
    NvtxRange nvtx_("tcr_single_pass_f16_async");
    // The result stays on the device, so there is no retry: on a selector engine (m != 16) a
    // non-finite input can surface as NaN where the reference has +-inf (the overflow flag is
    // exact either way).  The synchronous entry points re-run such calls with the repairing
    // kernels; this one keeps the fast instantiations.
    return sp_async(d_x, n, c, false, d_result, d_overflow, static_cast<cudaStream_t>(stream));
}

int tcr_single_pass_f32_async(const float* d_x, size_t n, const tcr_config* c, float* d_result,
                              uint32_t* d_overflow, void* stream) {
    NvtxRange nvtx_("tcr_single_pass_f32_async");
    return sp_async(d_x, n, c, true, d_result, d_overflow, static_cast<cudaStream_t>(stream));
}

int tcr_reduce_f16_device(const uint16_t* d_x, size_t n, const tcr_config* c, tcr_outcome* out, void* stream) {
    NvtxRange nvtx_("tcr_reduce_f16_device");
    return with_nan_retry(c, out, [&] { return reduce_device(d_x, n, c, out, false, static_cast<cudaStream_t>(stream)); });
}

int tcr_reduce_f32_device(const float* d_x, size_t n, const tcr_config* c, tcr_outcome* out, void* stream) {
    NvtxRange nvtx_("tcr_reduce_f32_device");
    return with_nan_retry(c, out, [&] { return reduce_device(d_x, n, c, out, true, static_cast<cudaStream_t>(stream)); });
}

}  // extern "C"

namespace {

// NCCL is resolved lazily with dlopen: no link-time dependency, and inside a PyTorch process the
// already-loaded libnccl.so.2 is reused instead of a second copy.
struct Nccl {
    decltype(&ncclCommInitAll) comm_init_all = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl r;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return r;
        r.comm_init_all = reinterpret_cast<decltype(&ncclCommInitAll)>(dlsym(h, "ncclCommInitAll"));
        r.group_start = reinterpret_cast<decltype(&ncclGroupStart)>(dlsym(h, "ncclGroupStart"));
        r.group_end = reinterpret_cast<decltype(&ncclGroupEnd)>(dlsym(h, "ncclGroupEnd"));
        r.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
        r.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
        r.ok = r.comm_init_all && r.group_start && r.group_end && r.all_reduce && r.error_string;
        return r;
    }();
    return n;
}

}  // namespace

extern "C" {

int tcr_reduce_f16_sharded(const uint16_t* const* d_x, const size_t* n, const int32_t* devices, int32_t ngpu,
                           const tcr_config* c, tcr_outcome* out) {
    NvtxRange nvtx_("tcr_reduce_f16_sharded");
    RepairScope rs(c && c->m != 16);   // one combined result: repair up front
    g_launches = 0;
    if (!out) return fail(TCR_INVALID_ARGUMENT, "null outcome");
    std::memset(out, 0, sizeof *out);
    if (!d_x || !n || !devices || ngpu < 1) return fail(TCR_INVALID_ARGUMENT, "bad shard description");
    int rc = validate_cfg(c);
    if (rc) return rc;
    if (c->variant != TCR_SINGLE_PASS) return fail(TCR_NOT_SUPPORTED, "sharded reduce implements single_pass");
    rc = check_supported(c);
    if (rc) return rc;
    uint64_t total = 0;
    const uint64_t ge = tcr::make_geometry(1, c->m, c->R, c->B).group_elems;
    for (int i = 0; i < ngpu; ++i) {
        if (n[i] == 0 || !d_x[i]) return fail(TCR_INVALID_ARGUMENT, "empty shard");
        if (i + 1 < ngpu && n[i] % ge != 0)
            return fail(TCR_INVALID_ARGUMENT, "shards must be multiples of tcr_group_elems except the last");
        total += n[i];
    }
    const Nccl& N = nccl();
    if (!N.ok) return fail(TCR_NCCL_ERROR, "libnccl.so.2 not found");
    int dev0 = 0;
    TCR_CUDA(cudaGetDevice(&dev0));
    // communicator cache keyed by the device list
    static std::mutex mu;
    static std::map<std::vector<int>, std::vector<ncclComm_t>> comms;
    std::vector<int> key(devices, devices + ngpu);
    std::vector<ncclComm_t>* cm = nullptr;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = comms.find(key);
        if (it == comms.end()) {
            std::vector<ncclComm_t> v(static_cast<size_t>(ngpu));
            const ncclResult_t r = N.comm_init_all(v.data(), ngpu, key.data());
            if (r != ncclSuccess) return fail(TCR_NCCL_ERROR, std::string("ncclCommInitAll: ") + N.error_string(r));
            it = comms.emplace(key, std::move(v)).first;
        }
        cm = &it->second;
    }
    tcr_config cc = *c;
    if (cc.finalize == TCR_FINALIZE_ORDERED) cc.finalize = TCR_FINALIZE_TREE;  // per shard; combine below
    std::vector<Workspace*> ws(static_cast<size_t>(ngpu));
    int launches = 0;
    for (int i = 0; i < ngpu; ++i) {
        TCR_CUDA(cudaSetDevice(devices[i]));
        rc = get_ws(nullptr, &ws[size_t(i)]);
        if (rc) return rc;
        TCR_CUDA(cudaMemsetAsync(ws[size_t(i)]->overflow(), 0, 4, nullptr));
        rc = sp_async(d_x[i], n[i], &cc, false, ws[size_t(i)]->result(), ws[size_t(i)]->overflow(), nullptr);
        if (rc) return rc;
        launches += g_launches;
    }
    ncclResult_t r = N.group_start();
    for (int i = 0; r == ncclSuccess && i < ngpu; ++i) {
        float* v = ws[size_t(i)]->result();
        r = N.all_reduce(v, v, 1, ncclFloat, ncclSum, (*cm)[size_t(i)], nullptr);
    }
    const ncclResult_t r2 = N.group_end();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(TCR_NCCL_ERROR, std::string("ncclAllReduce: ") + N.error_string(r != ncclSuccess ? r : r2));
    uint32_t ovf = 0;
    float value = 0.0f;
    for (int i = ngpu - 1; i >= 0; --i) {
        TCR_CUDA(cudaSetDevice(devices[i]));
        float v;
        uint32_t o;
        rc = read_result(ws[size_t(i)], nullptr, &v, &o);
        if (rc) return rc;
        ovf |= o;
        value = v;  // identical on every rank after the all-reduce; keep device 0's
    }
    TCR_CUDA(cudaSetDevice(dev0));
    g_launches = launches;
    out->value = value;
    out->overflow = ovf ? 1 : 0;
    counters(total, c, out);
    return TCR_OK;
}

}  // extern "C"

namespace {

// Per-block results of single_pass into d_blocks[n_blocks] (parity hook): binary16 or fp32 input
// through the same kernels the reductions use (fp32: from_single fused into the load where the
// engine has it, else one conversion pass first).
int block_results(const void* d_x, size_t n, const tcr_config* c, bool f32, float* d_blocks, cudaStream_t s) {
    RepairScope rs(c && c->m != 16);   // parity hook: per-block values exact for non-finite data too
    g_launches = 0;
    if (n == 0) return fail(TCR_INVALID_ARGUMENT, "input must be non-empty");
    int rc = validate_cfg(c);
    if (rc) return rc;
    rc = check_supported(c);
    if (rc) return rc;
    Workspace* w = nullptr;
    rc = get_ws(s, &w);
    if (rc) return rc;
    if (!d_x || !d_blocks) return fail(TCR_INVALID_ARGUMENT, "null device pointer");
    const void* xa = d_x;   // 16-byte lines: an unaligned slice is copied first
    rc = aligned_input(&xa, n, f32, w, s);
    if (rc) return rc;
    tcr_config cc = *c;
    cc.finalize = TCR_FINALIZE_TREE;
    cc.atomic_order = TCR_ASCENDING;
    const tcr::SpGeometry g = tcr::make_geometry(n, c->m, c->R, c->B);
    if (f32 && c->m != 16 && !tcr::genm_f32_supported(g)) {
        rc = ensure(&w->conv, &w->conv_cap, n, s);
        if (rc) return rc;
        TCR_CUDA(tcr::launch_convert_f32_f16(static_cast<const float*>(xa), w->conv, n, s));
        ++g_launches;
        xa = w->conv;
        f32 = false;
    }
    return enqueue_sp(xa, 0, n, &cc, f32, w->result(), w->overflow(), d_blocks, w, s, 0, g.n_groups, true);
}

}  // namespace

extern "C" {

int tcr_block_results_f16_device(const uint16_t* d_x, size_t n, const tcr_config* c, float* d_blocks,
                                 void* stream) {
    NvtxRange nvtx_("tcr_block_results_f16_device");
    return block_results(d_x, n, c, false, d_blocks, static_cast<cudaStream_t>(stream));
}

int tcr_block_results_f32_device(const float* d_x, size_t n, const tcr_config* c, float* d_blocks, void* stream) {
    NvtxRange nvtx_("tcr_block_results_f32_device");
    return block_results(d_x, n, c, true, d_blocks, static_cast<cudaStream_t>(stream));
}

namespace {
// Host-input calls run on a per-thread, per-device stream, so concurrent callers on different
// host threads get separate workspaces (the reference's reduce() is reentrant,
// reduction.hpp:19-21).
struct HostStreams {
    std::map<int, cudaStream_t> m;
    // A host thread's streams and their workspaces (ring buffers of ~384 MiB) go with the
    // thread: at thread exit they are queued (no CUDA call from a thread-exit handler, where the
    // runtime's own per-thread state may already be gone) and the next API call frees them.
    ~HostStreams() {
        std::lock_guard<std::mutex> lk(g_mu);
        for (auto& kv : m) g_reap.push_back(kv);
    }
};

int host_stream(cudaStream_t* out) {
    thread_local HostStreams hs;
    auto& streams = hs.m;
    int dev = 0;
    TCR_CUDA(cudaGetDevice(&dev));
    auto& st = streams[dev];
    if (!st) TCR_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    *out = st;
    return TCR_OK;
}

// H2D of a pageable host range (the reference's caller passes a std::vector, reduction.hpp:344):
// through the workspace's pinned staging ring, each slot filled by parallel host copies while
// the previous slots' DMAs run on the copy stream.  Pinned (or registered) sources go straight.
constexpr size_t kStageBytes = 16u << 20;
constexpr int kStageSlots = 4;

bool is_pageable(const void* x) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, x) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return pa.type == cudaMemoryTypeUnregistered;
}

void parallel_copy(char* dst, const char* src, size_t bytes) {
    static const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = unsigned(std::min<size_t>(std::min(16u, hw), std::max<size_t>(1, bytes >> 20)));
    if (nt <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> pool;
    const size_t per = (bytes / nt + 63) & ~size_t(63);
    for (unsigned t = 1; t < nt; ++t) {
        const size_t b0 = std::min(bytes, per * t), b1 = std::min(bytes, per * (t + 1));
        if (b1 > b0) pool.emplace_back([=] { std::memcpy(dst + b0, src + b0, b1 - b0); });
    }
    std::memcpy(dst, src, std::min(bytes, per));
    for (auto& th : pool) th.join();
}

int h2d(void* dst, const char* src, size_t bytes, bool pageable, Workspace* w) {
    if (!pageable) {
        TCR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, w->copy_stream));
        return TCR_OK;
    }
    if (!w->pin_stage) {
        TCR_CUDA(cudaMallocHost(&w->pin_stage, kStageBytes * kStageSlots));
        for (auto& e : w->pin_free) TCR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (size_t off = 0; off < bytes; off += kStageBytes) {
        const int slot = int(w->pin_seq++ % kStageSlots);
        char* pin = static_cast<char*>(w->pin_stage) + size_t(slot) * kStageBytes;
        TCR_CUDA(cudaEventSynchronize(w->pin_free[slot]));   // its previous DMA is done
        const size_t b = std::min(kStageBytes, bytes - off);
        parallel_copy(pin, src + off, b);
        TCR_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, pin, b, cudaMemcpyHostToDevice, w->copy_stream));
        TCR_CUDA(cudaEventRecord(w->pin_free[slot], w->copy_stream));
    }
    return TCR_OK;
}

// Host-input reduce(): pipelined H2D of group-aligned chunks on a copy stream (2-slot ring,
// pinned source, or pageable through the pinned staging ring), reduce kernel per chunk on the compute stream, one finaliser.
// f32: fp32 values converted to binary16 on the device (fused into the m = 16 kernel);
// otherwise binary16 bit patterns (half the bytes over PCIe).
int reduce_host(const void* x, bool f32, size_t n, const tcr_config* c, tcr_outcome* out) {
    g_launches = 0;
    if (!out) return fail(TCR_INVALID_ARGUMENT, "null outcome");
    std::memset(out, 0, sizeof *out);
    if (!c) return fail(TCR_INVALID_ARGUMENT, "null config");
    const size_t esz = f32 ? sizeof(float) : sizeof(uint16_t);
    if (c->variant != TCR_SINGLE_PASS) {
        // the other variants take the whole input on the device, then the same dispatcher
        if (c->variant < TCR_ORACLE64 || c->variant > TCR_SPLIT) return fail(TCR_INVALID_ARGUMENT, "unknown variant");
        cudaStream_t s0 = nullptr;
        int rc0 = host_stream(&s0);
        if (rc0) return rc0;
        Workspace* w0 = nullptr;
        rc0 = get_ws(s0, &w0);
        if (rc0) return rc0;
        if (n == 0) {
            if (c->variant == TCR_ORACLE64) return TCR_OK;
            return fail(TCR_INVALID_ARGUMENT, "input must be non-empty");
        }
        if (!x) return fail(TCR_INVALID_ARGUMENT, "null input");
        rc0 = ensure(&w0->stage, &w0->stage_cap, f32 ? n : (n + 1) / 2, s0);
        if (rc0) return rc0;
        TCR_CUDA(cudaMemcpyAsync(w0->stage, x, n * esz, cudaMemcpyHostToDevice, s0));
        return run_variant(w0->stage, f32, n, c, out, w0, s0);
    }
    if (n == 0) return fail(TCR_INVALID_ARGUMENT, "input must be non-empty");
    if (!x) return fail(TCR_INVALID_ARGUMENT, "null input");
    int rc = validate_cfg(c);
    if (rc) return rc;
    rc = check_supported(c);
    if (rc) return rc;
    cudaStream_t s = nullptr;
    rc = host_stream(&s);
    if (rc) return rc;
    Workspace* w = nullptr;
    rc = get_ws(s, &w);
    if (rc) return rc;
    const tcr::SpGeometry g = tcr::make_geometry(n, c->m, c->R, c->B);
    // chunk: whole groups, ~32 Mi elements (128 MiB of fp32 / 64 MiB of binary16)
    const uint64_t groups_per_chunk = std::max<uint64_t>(1, (32ull << 20) / g.group_elems);
    const uint64_t chunk_elems = groups_per_chunk * g.group_elems;
    const uint64_t n_chunks = (g.n_groups + groups_per_chunk - 1) / groups_per_chunk;
    const uint64_t ring_elems = std::min<uint64_t>(chunk_elems, n);
    if (w->ring_cap < ring_elems) {
        TCR_CUDA(cudaStreamSynchronize(s));
        if (w->copy_stream) TCR_CUDA(cudaStreamSynchronize(w->copy_stream));
        for (auto& r : w->ring)
            if (r) TCR_CUDA(cudaFree(r));
        for (auto& r : w->ring) TCR_CUDA(cudaMalloc(&r, ring_elems * sizeof(float) + 16));
        for (auto& r : w->ring16)
            if (r) TCR_CUDA(cudaFree(r));
        for (auto& r : w->ring16) TCR_CUDA(cudaMalloc(&r, ring_elems * sizeof(uint16_t) + 16));
        w->ring_cap = ring_elems;
    }
    if (!w->copy_stream) {
        TCR_CUDA(cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            TCR_CUDA(cudaEventCreateWithFlags(&w->copied[i], cudaEventDisableTiming));
            TCR_CUDA(cudaEventCreateWithFlags(&w->consumed[i], cudaEventDisableTiming));
        }
    }
    tcr_config cc = *c;
    TCR_CUDA(cudaMemsetAsync(w->overflow(), 0, 4, s));
    const char* xb = static_cast<const char*>(x);
    const bool f32_direct = f32 && cc.m != 16 && tcr::genm_f32_supported(g);
    const bool pageable = n * esz >= (1u << 20) && is_pageable(x);
    for (uint64_t k = 0; k < n_chunks; ++k) {
        const int slot = int(k & 1);
        const uint64_t e0 = k * chunk_elems;
        const uint64_t e1 = std::min<uint64_t>(n, e0 + chunk_elems);
        const uint64_t g0 = k * groups_per_chunk;
        const uint64_t g1 = std::min<uint64_t>(g.n_groups, g0 + groups_per_chunk);
        void* dst = f32 ? static_cast<void*>(w->ring[slot]) : static_cast<void*>(w->ring16[slot]);
        if (k >= 2) TCR_CUDA(cudaStreamWaitEvent(w->copy_stream, w->consumed[slot], 0));
        rc = h2d(dst, xb + e0 * esz, (e1 - e0) * esz, pageable, w);
        if (rc) return rc;
        TCR_CUDA(cudaEventRecord(w->copied[slot], w->copy_stream));
        TCR_CUDA(cudaStreamWaitEvent(s, w->copied[slot], 0));
        const bool last = (k + 1 == n_chunks);
        // single chunk: finalise in the same launch; otherwise one finaliser at the end
        if (!f32 || cc.m == 16 || f32_direct) {
            rc = enqueue_sp(dst, e0, n, &cc, f32, w->result(), w->overflow(), nullptr, w, s, g0, g1,
                            last && n_chunks == 1);
        } else {
            TCR_CUDA(tcr::launch_convert_f32_f16(w->ring[slot], w->ring16[slot], e1 - e0, s));
            ++g_launches;
            rc = enqueue_sp(w->ring16[slot], e0, n, &cc, false, w->result(), w->overflow(), nullptr, w, s, g0, g1,
                            last && n_chunks == 1);
        }
        if (rc) return rc;
        TCR_CUDA(cudaEventRecord(w->consumed[slot], s));
    }
    if (n_chunks > 1) {
        rc = enqueue_finalize(n, &cc, w->result(), w, s);
        if (rc) return rc;
    }
    float v;
    uint32_t o;
    rc = read_result(w, s, &v, &o);
    if (rc) return rc;
    out->value = v;
    out->overflow = o ? 1 : 0;
    counters(n, c, out);
    return TCR_OK;
}
}  // namespace

int tcr_reduce_f32_host(const float* x, size_t n, const tcr_config* c, tcr_outcome* out) {
    NvtxRange nvtx_("tcr_reduce_f32_host");
    // Drop-in for reduce(std::span<const float>, cfg)
    return with_nan_retry(c, out, [&] { return reduce_host(x, true, n, c, out); });
}

int tcr_reduce_f16_host(const uint16_t* x, size_t n, const tcr_config* c, tcr_outcome* out) {
    NvtxRange nvtx_("tcr_reduce_f16_host");
    return with_nan_retry(c, out, [&] { return reduce_host(x, false, n, c, out); });
}

int tcr_generate_f16_device(uint16_t* d_x, size_t n, int32_t dist, uint64_t seed, int64_t lo, int64_t hi,
                            double cval, size_t first, void* stream) {
    if (dist < 0 || dist > 3) return fail(TCR_INVALID_ARGUMENT, "unknown distribution");
    if (dist == TCR_DIST_INTEGERS && hi < lo) return fail(TCR_INVALID_ARGUMENT, "integers: hi < lo");
    TCR_CUDA(tcr::launch_generate(d_x, true, n, dist, seed, lo, hi, cval, first, static_cast<cudaStream_t>(stream)));
    return TCR_OK;
}

int tcr_generate_f32_device(float* d_x, size_t n, int32_t dist, uint64_t seed, int64_t lo, int64_t hi,
                            double cval, size_t first, void* stream) {
    if (dist < 0 || dist > 3) return fail(TCR_INVALID_ARGUMENT, "unknown distribution");
    if (dist == TCR_DIST_INTEGERS && hi < lo) return fail(TCR_INVALID_ARGUMENT, "integers: hi < lo");
    TCR_CUDA(tcr::launch_generate(d_x, false, n, dist, seed, lo, hi, cval, first, static_cast<cudaStream_t>(stream)));
    return TCR_OK;
}

int tcr_exact_sum_f16_device(const uint16_t* d_x, size_t n, double* sum, double* abs_sum, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (reinterpret_cast<uintptr_t>(d_x) % 16) return fail(TCR_INVALID_ARGUMENT, "input must be 16-byte aligned");
    Workspace* w = nullptr;
    int rc = get_ws(s, &w);
    if (rc) return rc;
    TCR_CUDA(tcr::launch_exact_sum_f16(d_x, n, w->exact_ws, w->exact_out(), s));
    double h[3];
    TCR_CUDA(cudaMemcpyAsync(h, w->exact_out(), sizeof h, cudaMemcpyDeviceToHost, s));
    TCR_CUDA(cudaStreamSynchronize(s));
    *sum = h[0];
    *abs_sum = h[1];
    return TCR_OK;
}

int tcr_shuffle_f16_async(const uint16_t* d_x, size_t n, float* d_result, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) return fail(TCR_INVALID_ARGUMENT, "input must be non-empty");
    if (reinterpret_cast<uintptr_t>(d_x) % 16) return fail(TCR_INVALID_ARGUMENT, "input must be 16-byte aligned");
    Workspace* w = nullptr;
    int rc = get_ws(s, &w);
    if (rc) return rc;
    const int grid = std::min(tcr::shuffle_max_grid(), 8192);
    TCR_CUDA(tcr::launch_shuffle_f16(d_x, n, w->shuffle_partials, w->sh_ticket(), d_result, grid, s));
    g_launches = 1;
    return TCR_OK;
}

int tcr_cub_sum_f16_async(const uint16_t* d_x, size_t n, int half_acc, void* d_result, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Workspace* w = nullptr;
    int rc = get_ws(s, &w);
    if (rc) return rc;
    const size_t need = tcr::cub_temp_bytes(n, half_acc != 0);
    rc = ensure(reinterpret_cast<unsigned char**>(&w->cub_temp), &w->cub_cap, need, s);
    if (rc) return rc;
    TCR_CUDA(tcr::cub_sum_f16(d_x, n, d_result, half_acc != 0, w->cub_temp, w->cub_cap, s));
    return TCR_OK;
}

int tcr_enable_profiling_knobs(void) { return tcr::load_knobs_from_env(); }

int tcr_ordered_stats(unsigned long long* host4) { return tcr::ordered_stats(host4); }

void tcr_reset_profiling_knobs(void) { tcr::reset_knobs(); }

int tcr_read_probe_async(const void* d_x, size_t bytes, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Workspace* w = nullptr;
    int rc = get_ws(s, &w);
    if (rc) return rc;
    const tcr::Knobs& k = tcr::knobs();   // profiling: cp.async probe / CTAs per SM
    const int per_sm = k.probe_ctas > 0 ? k.probe_ctas : 8;
    if (k.probe_tma)
        TCR_CUDA(tcr::launch_read_probe_tma(d_x, bytes, w->sink(), tcr::sm_count() * (k.probe_ctas > 0 ? k.probe_ctas : 2),
                                            k.probe_slot > 0 ? uint32_t(k.probe_slot) : 16384u, s));
    else if (k.probe_async)
        TCR_CUDA(tcr::launch_read_probe_async(d_x, bytes, w->sink(), tcr::sm_count() * per_sm, s));
    else
        TCR_CUDA(tcr::launch_read_probe(d_x, bytes, w->sink(), tcr::sm_count() * per_sm, s));
    return TCR_OK;
}

}  // extern "C"
