// tcr_kernels.h -- host-visible launch interface of the tcreduce sm_100a kernels.
// Internal to libtcreduce_b200.so; the public surface is include/tcreduce_b200.h.
#pragma once

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

namespace tcr {

enum Finalize : int32_t {
    kFinNone = -1,     // leave group partials for a later finalize launch
    kFinTree = 0,      // deterministic pairwise tree over block results (default)
    kFinOrdered = 1,   // reference order: serial fp32 sum, ascending or seeded permutation
    kFinAtomic = 2,    // paper's atomicAdd per block (non-deterministic order)
};

// Group-size target: a CTA reduces G logical blocks (G a power of two) of at least this many
// elements, so the deterministic tree is a fixed function of (n, m, R, B) only.
constexpr uint64_t kGroupElemsTarget = 1ull << 18;   // 512 KiB of binary16 (measured: fewer pipeline drains)
constexpr int kSpWarps = 8;            // warps per CTA of the single-pass kernel
constexpr int kSpThreads = kSpWarps * 32;
constexpr int kMaxChunksPerGroup = 1024;
constexpr int kMaxChunksGenm = 4096;     // chunk table of the m != 16 engine (small chunks)

struct SpGeometry {
    uint32_t m, R, W;          // fragment side, chain length, warps per logical block (B/32)
    uint64_t n;                // elements
    uint64_t chunk_elems;      // R*m*m            (a warp's chunk, reduction.hpp:240)
    uint64_t block_elems;      // chunk_elems*W    (a logical block's chunk, :241)
    uint64_t n_blocks;         // max(1, ceil(n / block_elems))  (:242)
    uint32_t G;                // logical blocks per group (power of two)
    uint64_t group_elems;      // G*block_elems
    uint64_t n_groups;         // ceil(n_blocks / G)
};

SpGeometry make_geometry(uint64_t n, uint32_t m, uint32_t R, uint32_t B);

struct SpParams {
    const void* x;
    uint64_t n;
    uint32_t R, W, G;
    uint64_t chunk_elems, n_blocks, n_groups;
    uint64_t group_begin, group_end;   // groups covered by this launch
    float* group_partials;             // [n_groups]   (tree finaliser input)
    float* block_partials;             // [n_blocks] or null (ordered finaliser / parity tests)
    float* result;                     // device scalar
    uint32_t* overflow;                // device flag (OR)
    uint32_t* ticket;                  // last-CTA-done counter, returns to 0
    uint32_t* order_scratch;           // [n_blocks] for the seeded-permutation finaliser
    int32_t finalize;
    int32_t atomic_order;
    uint64_t atomic_seed;
    // Work units of the cp.async engine.  Groups [group_begin, tail_group) are split into
    // `split` pieces of G/split whole blocks, the tail groups [tail_group, group_end) into
    // `split_tail` pieces (small units at the end balance the grid).  Pieces of one group put
    // their block results in block_scratch[n_groups*G] and the CTA completing the group
    // (group_count[n_groups], zero on entry and exit) runs its group tree: the tree -- and so
    // the TREE result -- does not depend on the split.  work_counter (zero on entry and exit)
    // hands units out dynamically; null = grid-stride order.
    uint32_t split, split_tail;
    uint64_t tail_group;
    float* block_scratch;
    uint32_t* group_count;
    unsigned long long* work_counter;
    // Profiling hook (env TCR_DEBUG_MODE, never set in production): tcgen05 engine only --
    // 1 = TMA stream only (no MMA / epilogue), 2 = 1-D bulk copies instead of the tensor map,
    // 3 = TMA + MMA without the epilogue (accumulators overwritten unread), 4 = as 3 with A read
    // K-major, 5 = as 3 with N = 64 (timing only; results are not meaningful in modes 1-5).
    // cp.async engine: 9 / 10 = ring depth 8 / 32 for R = 1, 11 = depth 12 / 10 for R = 3 / 5
    // (results identical).
    int32_t debug_mode;
};

// Single-pass chained-MMA reduction, m = 16, binary16 (or fp32 convert-on-load) input.
cudaError_t launch_single_pass_m16(const SpParams& p, bool f32_input, int grid, cudaStream_t s);
cudaError_t launch_finalize(const SpParams& p, cudaStream_t s);

// tcgen05 + TMA engine over the first n_tiles FULL groups (binary16 input).  tc05_plan says
// whether the geometry is supported (m = 16, R <= 12, G*W a multiple of 8) and picks the slot
// size (Q MMA-groups of 8 chunks) and ring depth.
bool tc05_plan(const SpGeometry& g, uint32_t* Q, uint32_t* ring_slots);
cudaError_t launch_tc05(const SpParams& p, const SpGeometry& g, uint64_t n_tiles, int grid, cudaStream_t s);

// TMA-fed mma.sync engine (tcr_sp_bulk.cu): per-warp rings refilled by 1-D bulk copies, a manager
// warp claiming work units ahead (p.work_counter, zero on entry and exit) and running the trees.
// FULL groups [p.group_begin, p.group_end) only.  bulk_plan sets split / split_tail / tail_group
// (pieces need p.block_scratch and p.group_count, zero on entry and exit).
bool bulk_supported(const SpGeometry& g);
int bulk_max_grid(uint32_t R, int debug_mode = 0);
void bulk_plan(const SpGeometry& g, SpParams* p, int grid);
cudaError_t launch_bulk(const SpParams& p, int grid, cudaStream_t s);

// Per-warp cp.async pipeline engine (LDGSTS ring per warp, ldmatrix.trans + HMMA); handles any
// group range including the ragged tail (zero-fill copies).  binary16 input.
int async_max_grid(uint32_t R, int debug_mode = 0);
// profiling: per-CTA %globaltimer stamps of the last debug_mode-20 launch
int debug_timestamps(unsigned long long* host, size_t count);
cudaError_t launch_async(const SpParams& p, int grid, cudaStream_t s);
// Work-unit plan of the cp.async engine over groups [p.group_begin, p.group_end) on `grid`
// CTAs: sets split, split_tail, tail_group; returns whether units are handed out dynamically.
// Env TCR_SPLIT / TCR_TAIL_SPLIT / TCR_SCHED override (profiling).
bool async_plan(const SpGeometry& g, SpParams* p, int grid);

// ORDERED finaliser (tcr_ordered.cu): serial binary32 sum of blocks[order[k]] (order null:
// ascending), the reference's accumulation (reduction.hpp:257-268).
cudaError_t launch_ordered(const float* blocks, const uint32_t* order, uint64_t nb, float* result, cudaStream_t s);
// Any order in parallel, bit-identical to the serial chain (tcr_ordered.cu): per-segment
// records of the binade-local integer arithmetic, composed into runs and a tree, walked by one
// warp.  order: position -> block, or null (ascending).  ws: >= ordered_ws_bytes(nb), zero on
// first use (look-back flags return to zero); ticket zero on entry and exit.
size_t ordered_ws_bytes(uint64_t nb, bool binary64 = false);
int ordered_stats(unsigned long long* host);   // profiling: counters and phase stamps of the last walk
int ordered_grid(uint64_t nb);
cudaError_t launch_ordered_parallel(const float* blocks, const uint32_t* order, uint64_t nb, void* ws, uint32_t* ticket,
                                    float* result, cudaStream_t s);
// oracle64 (reduction.hpp:106-110): the reference's serial binary64 sum of n fp32 (f32) or
// binary16 values, by the same parallel evaluation in binary64 -- bit for bit the left-to-right
// loop.  ws: >= ordered_ws_bytes(n, true).
cudaError_t launch_serial_sum64(const void* x, bool f32, uint64_t n, void* ws, double* result, cudaStream_t s);

// Fragment sides m != 16 (tcr_sp_genm.cu): binary16 input, any group range.
bool genm_supported(const SpGeometry& g);
// repair: instantiations that recompute NaN chunk results exactly (non-finite inputs; see
// group_epilogue in tcr_sp_genm.cu).
// f32: fp32 input with from_single fused into the load (genm_f32_supported shapes only).
bool genm_f32_supported(const SpGeometry& g);
cudaError_t launch_genm(const SpParams& p, const SpGeometry& g, cudaStream_t s, bool repair, bool f32 = false);

// Variants (tcr_variants.cu): bit-exact strided pairwise trees (shuffle32 / half_tree) and the
// recurrence level rounding (oracle64 is the binary64 serial chain of tcr_ordered.cu).
uint64_t tree_cols_needed(uint64_t n);
int tree_launches(uint64_t n);
cudaError_t launch_pairwise_tree(const void* x, bool f32, uint64_t n, bool half, float* cols, float* out,
                                 uint32_t* ovf, cudaStream_t s);
cudaError_t launch_round_level(const float* in, uint16_t* out, uint64_t count, uint32_t* ovf, cudaStream_t s);

// fp32 -> binary16 (RNE, from_single) conversion of count elements.
cudaError_t launch_convert_f32_f16(const float* in, uint16_t* out, uint64_t count, cudaStream_t s);
int single_pass_m16_max_grid(bool f32_input, uint32_t R);

// Input generation (harness.hpp:47-80 with SplitMix64 jump-ahead), binary16 or fp32 output.
cudaError_t launch_generate(void* out, bool f16_out, uint64_t count, int kind, uint64_t seed,
                            int64_t lo, int64_t hi, double c, uint64_t first, cudaStream_t s);

// Exact fixed-point sum of binary16 values (+ sum |x|, non-finite count).  ws: >= exact_ws_bytes().
size_t exact_ws_bytes();
cudaError_t launch_exact_sum_f16(const uint16_t* x, uint64_t n, void* ws, double* d_out3,
                                 cudaStream_t s);

// CUDA-core fp32 warp-shuffle reduction of binary16 input (the paper's baseline).
cudaError_t launch_shuffle_f16(const uint16_t* x, uint64_t n, float* partials, uint32_t* ticket,
                               float* result, int grid, cudaStream_t s);
int shuffle_max_grid();

// Pure streaming-read probe: the achievable read bandwidth ceiling.
cudaError_t launch_read_probe(const void* x, uint64_t bytes, uint32_t* sink, int grid, cudaStream_t s);
cudaError_t launch_read_probe_tma(const void* x, uint64_t bytes, uint32_t* sink, int grid, uint32_t slot, cudaStream_t s);
cudaError_t launch_read_probe_async(const void* x, uint64_t bytes, uint32_t* sink, int grid, cudaStream_t s);

// CUB DeviceReduce::Sum comparators.
size_t cub_temp_bytes(uint64_t n, bool half_out);
cudaError_t cub_sum_f16(const uint16_t* x, uint64_t n, void* out, bool half_out, void* temp,
                        size_t temp_bytes, cudaStream_t s);

int sm_count();

// Runs set() once per CUDA device for one call site: function attributes such as the dynamic
// shared-memory opt-in live in each device's context, so a per-process flag would leave every
// device after the first without them.  Thread-safe; device ordinals < 64.
class PerDeviceOnce {
  public:
    template <typename F>
    cudaError_t operator()(F set) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        std::lock_guard<std::mutex> lock(mu_);
        const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
        if (done_ & bit) return cudaSuccess;
        e = set();
        if (e == cudaSuccess) done_ |= bit;
        return e;
    }

  private:
    std::mutex mu_;
    uint64_t done_ = 0;
};

// Profiling knobs (A/B experiments only).  Every field holds its production default unless the
// process called tcr_enable_profiling_knobs(), which reads the TCR_* environment variables ONCE;
// nothing on a reduce() path calls getenv.  Some knobs change the group size G -- and so the
// TREE result -- which is why they are never read implicitly (the reference is a pure function
// of input and config, reduction.hpp:19-21).
struct Knobs {
    int debug_mode = 0;                // TCR_DEBUG_MODE: engine-specific profiling modes (SpParams)
    uint64_t group_target = 0;         // TCR_GROUP_TARGET: elements per group (0 = kGroupElemsTarget)
    uint64_t group_cap = 0;            // TCR_GROUP_CAP: chunk-table entries (0 = engine table; clamped to it)
    uint32_t split = 0, tail_split = 0;   // TCR_SPLIT / TCR_TAIL_SPLIT: work-unit pieces (0 = planner)
    int sched = -1;                    // TCR_SCHED: 0 static grid-stride, 1 dynamic (-1 = planner)
    int ctas_per_sm = 0;               // TCR_CTAS_PER_SM (0 = 2)
    bool gm_nat_generic = false;       // TCR_GM_NAT_GENERIC
    int gm_nat_alt = 0;                // TCR_GM_NAT_ALT
    bool gm_wide_warp = false;         // TCR_GM_WIDE_WARP
    bool gm_no_cluster = false;        // TCR_GM_NO_CLUSTER
    bool gm_tr8_single = false;        // TCR_GM_TR8_SINGLE
    bool probe_async = false;          // TCR_PROBE=async
    bool probe_tma = false;            // TCR_PROBE=tma (TCR_PROBE_SLOT bytes per copy, default 16384)
    int probe_slot = 0;
    int probe_ctas = 0;                // TCR_PROBE_CTAS (0 = 8)
};
const Knobs& knobs();
int load_knobs_from_env();   // returns how many TCR_* knobs were set
void reset_knobs();

}  // namespace tcr
