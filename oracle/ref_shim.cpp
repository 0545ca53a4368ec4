// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file against the
// reference's own headers where they lie (/root/reference/proj/include) into
// oracle/_ref/libtcreduce_ref.so.  Nothing here restates an algorithm: every
// call goes straight into tcreduce:: as shipped.  The one composite function,
// ref_single_pass_parallel, is the survey's bit-identical parallel form of
// detail::single_pass_core: the reference's own
// chained_warp_reduce + detail::pairwise_tree per block on worker threads,
// then the reference's serial ascending accumulation.  It exists so the CPU
// baseline can use every host core.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "tcreduce/csv.hpp"
#include "tcreduce/harness.hpp"
#include "tcreduce/reduction.hpp"

using namespace tcreduce;

extern "C" {
typedef struct {
    int32_t variant;
    uint32_t m, R, B;
    double f;
    int32_t atomic_order;
    uint64_t atomic_seed;
} ref_config;

typedef struct {
    double value;
    int32_t overflow;
    uint64_t level_count, sim_steps, mma_count, atomic_count, shuffle_count;
} ref_outcome;
}  // extern "C"

static ReductionConfig to_cfg(const ref_config* c) {
    ReductionConfig cfg;
    cfg.variant = static_cast<Variant>(c->variant);
    cfg.m = c->m;
    cfg.R = c->R;
    cfg.B = c->B;
    cfg.f = c->f;
    cfg.atomic_order = static_cast<AtomicOrder>(c->atomic_order);
    cfg.atomic_seed = c->atomic_seed;
    return cfg;
}

static void to_out(const ReductionOutcome& o, ref_outcome* out) {
    out->value = o.value;
    out->overflow = o.overflow ? 1 : 0;
    out->level_count = o.level_count;
    out->sim_steps = o.sim_steps;
    out->mma_count = o.mma_count;
    out->atomic_count = o.atomic_count;
    out->shuffle_count = o.shuffle_count;
}

// 0 ok, -1 invalid_argument, -2 out_of_range, -3 other
template <class F>
static int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::out_of_range&) {
        return -2;
    } catch (...) {
        return -3;
    }
}

extern "C" {

uint16_t ref_from_single(float x) { return from_single(x).bits; }
float ref_to_single(uint16_t h) { return to_single(Half{h}); }

int ref_generate(int kind, uint64_t seed, int64_t lo, int64_t hi, double c, size_t n, float* out) {
    return guard([&] {
        Distribution d;
        d.kind = static_cast<DistKind>(kind);
        d.seed = seed;
        d.lo = lo;
        d.hi = hi;
        d.c = c;
        const std::vector<float> v = generate(d, n);
        std::memcpy(out, v.data(), n * sizeof(float));
    });
}

double ref_oracle64(const float* x, size_t n) { return oracle64(std::span<const float>(x, n)); }

int ref_reduce(const float* x, size_t n, const ref_config* c, ref_outcome* out) {
    return guard([&] { to_out(reduce(std::span<const float>(x, n), to_cfg(c)), out); });
}

int ref_single_pass_reduce(const float* x, size_t n, const ref_config* c, ref_outcome* out) {
    return guard([&] { to_out(single_pass_reduce(std::span<const float>(x, n), to_cfg(c)), out); });
}

int ref_validate(const ref_config* c) {
    return guard([&] { to_cfg(c).validate(); });
}

int ref_chained_warp_reduce(const float* x, size_t n, size_t base, const ref_config* c, float* out,
                            uint64_t* mma_count) {
    return guard([&] {
        detail::SimCounters sc;
        *out = chained_warp_reduce(std::span<const float>(x, n), base, to_cfg(c), sc);
        *mma_count = sc.mma.mma_count;
    });
}

size_t ref_warp_offset(size_t b, size_t w, const ref_config* c) { return warp_offset(b, w, to_cfg(c)); }

// Parallel single_pass: per-block work with the reference's own functions; serial ascending
// accumulation exactly as reduction.hpp:264-268.  block_out (optional) gets block results.
int ref_single_pass_parallel(const float* x, size_t n, const ref_config* c, int threads,
                             ref_outcome* out, float* block_out) {
    return guard([&] {
        if (n == 0) throw std::invalid_argument("input must be non-empty");
        const ReductionConfig cfg = to_cfg(c);
        cfg.validate();
        const std::size_t chunk_block = static_cast<std::size_t>(cfg.R) * cfg.m * cfg.m * cfg.warps_per_block();
        const std::size_t blocks = std::max<std::size_t>(1, (n + chunk_block - 1) / chunk_block);
        std::vector<float> br(blocks);
        std::vector<int> ovf(static_cast<std::size_t>(threads > 0 ? threads : 1), 0);
        const int T = threads > 0 ? threads : 1;
        auto work = [&](int t) {
            std::vector<float> chunk(chunk_block);
            detail::SimCounters sc;
            for (std::size_t b = static_cast<std::size_t>(t); b < blocks; b += static_cast<std::size_t>(T)) {
                const std::size_t lo = b * chunk_block;
                const std::size_t cnt = lo < n ? std::min(chunk_block, n - lo) : 0;
                std::fill(chunk.begin(), chunk.end(), 0.0f);
                if (cnt) std::memcpy(chunk.data(), x + lo, cnt * sizeof(float));
                std::vector<float> wr(cfg.warps_per_block());
                for (std::size_t w = 0; w < wr.size(); ++w)
                    wr[w] = chained_warp_reduce(chunk, warp_offset(0, w, cfg), cfg, sc);
                std::uint64_t ops = 0;
                detail::pairwise_tree(wr, ops);
                br[b] = wr[0];
            }
            ovf[static_cast<std::size_t>(t)] = sc.overflow ? 1 : 0;
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
        float acc = 0.0f;
        for (std::size_t b = 0; b < blocks; ++b) acc += br[b];
        if (block_out) std::memcpy(block_out, br.data(), blocks * sizeof(float));
        out->value = acc;
        out->overflow = 0;
        for (int v : ovf) out->overflow |= v;
        const std::size_t W = cfg.warps_per_block();
        const std::size_t P = detail::next_pow2(W);
        unsigned lv = 0;
        for (std::size_t len = P; len > 1; len /= 2) ++lv;
        out->level_count = 1;
        out->sim_steps = 2ull * cfg.R + 2 + lv + blocks;
        out->mma_count = blocks * W * (cfg.R + 1);
        out->atomic_count = blocks;
        out->shuffle_count = blocks * (P - 1);
    });
}

// csv.hpp:14-15 as shipped.
const char* ref_csv_header() { return kCsvHeader; }

static int put(const std::string& s, char* buf, size_t cap) {
    if (s.size() + 1 > cap) return -3;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

// csv.hpp:19-48 as shipped, on a SweepRecord built from explicit fields (has_err = 0: nullopt).
int ref_csv_row(const ref_config* c, uint64_t n, uint64_t seed, const char* dist, double value, int has_err,
                double err, int overflow, uint64_t sim_steps, uint64_t mma_count, uint64_t atomic_count, char* buf,
                size_t cap) {
    int rc = 0;
    const int g = guard([&] {
        SweepRecord rec;
        rec.config = to_cfg(c);
        rec.n = n;
        rec.seed = seed;
        rec.dist = dist;
        rec.value = value;
        if (has_err) rec.error_pct = err;
        rec.overflow = overflow != 0;
        rec.sim_steps = sim_steps;
        rec.mma_count = mma_count;
        rec.atomic_count = atomic_count;
        rc = put(csv_row(rec), buf, cap);
    });
    return g ? g : rc;
}

// harness.hpp:103-117 (run_point: generate, reduce, oracle64 error) as shipped, returned as its
// csv.hpp row.
int ref_run_point_csv(int kind, uint64_t seed, int64_t lo, int64_t hi, double cc, size_t n, const ref_config* c,
                      char* buf, size_t cap) {
    int rc = 0;
    const int g = guard([&] {
        Distribution d;
        d.kind = static_cast<DistKind>(kind);
        d.seed = seed;
        d.lo = lo;
        d.hi = hi;
        d.c = cc;
        rc = put(csv_row(run_point(d, n, to_cfg(c))), buf, cap);
    });
    return g ? g : rc;
}

}  // extern "C"
