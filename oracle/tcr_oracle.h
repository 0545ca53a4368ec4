/*
 * tcr_oracle.h -- CPU restatement of the reference tcreduce algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 product
 * path (paper_2001_05585_b200/csrc), never part of it: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load liboracle.so.  The product library never links or calls it.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj/include/tcreduce/) in plain C.  Parity of this
 * restatement is pinned two ways (see tests/test_oracle.py):
 *   1. bit-for-bit against the reference headers themselves, compiled by
 *      oracle/Makefile into oracle/_ref/libtcreduce_ref.so;
 *   2. against the known-answer values in the reference's own tests
 *      (test_half.cpp, test_fragment.cpp, test_reduction.cpp, acceptance.cpp)
 *      and the committed golden fixtures in tests/golden/.
 */
#ifndef TCR_ORACLE_H
#define TCR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Variant / AtomicOrder / DistKind mirror reduction.hpp:23,25 and harness.hpp:20. */
enum { ORC_ORACLE64 = 0, ORC_SHUFFLE32 = 1, ORC_HALF_TREE = 2, ORC_RECURRENCE = 3,
       ORC_SINGLE_PASS = 4, ORC_SPLIT = 5 };
enum { ORC_ASCENDING = 0, ORC_SEEDED_PERMUTATION = 1 };
enum { ORC_NORMAL = 0, ORC_UNIFORM = 1, ORC_INTEGERS = 2, ORC_CONSTANT = 3 };

/* ReductionConfig (reduction.hpp:39-57). */
typedef struct {
    int32_t variant;
    uint32_t m, R, B;
    double f;
    int32_t atomic_order;
    uint64_t atomic_seed;
} orc_config;

/* ReductionOutcome (reduction.hpp:59-67). */
typedef struct {
    double value;
    int32_t overflow;
    uint64_t level_count, sim_steps, mma_count, atomic_count, shuffle_count;
} orc_outcome;

/* Error codes: 0 ok, -1 invalid_argument, -2 out_of_range. */

/* half.hpp:32-59 / :61-79 / :82 */
uint16_t orc_from_single(float x);
float orc_to_single(uint16_t h);
int orc_is_overflowed(uint16_t h);

/* rng.hpp:14-19 (one step) and the jump-ahead form used by the GPU generator. */
uint64_t orc_splitmix_next(uint64_t *state);
uint64_t orc_splitmix_draw(uint64_t seed, uint64_t k); /* k-th draw, k >= 1 */

/* harness.hpp:47-80: sequential generator (exactly the reference's loop). */
int orc_generate(int kind, uint64_t seed, int64_t lo, int64_t hi, double c, size_t n, float *out);
/* Jump-ahead generator: elements [first, first+count) of generate(dist, N) for any N > first+count. */
int orc_generate_range(int kind, uint64_t seed, int64_t lo, int64_t hi, double c, size_t first,
                       size_t count, float *out);
/* Same, rounded to binary16 bits with orc_from_single (what the GPU stores). */
int orc_generate_range_f16(int kind, uint64_t seed, int64_t lo, int64_t hi, double c, size_t first,
                           size_t count, uint16_t *out);

/* reduction.hpp:106-110 */
double orc_oracle64(const float *x, size_t n);
/* Exact sum of the binary16-rounded inputs (fixed point, 2^-24 units, 128-bit);
 * also returns sum |x|.  Used for error-vs-exact reporting. */
void orc_exact_sum_f16(const uint16_t *h, size_t n, double *sum, double *abs_sum);

int orc_validate(const orc_config *cfg);                        /* reduction.hpp:50-56 */
size_t orc_warp_offset(size_t block, size_t warp, const orc_config *cfg); /* :154-158 */
/* reduction.hpp:164-184; returns 0/-2; *out = D'[0][0]; counters updated. */
int orc_chained_warp_reduce(const float *x, size_t n, size_t base, const orc_config *cfg,
                            float *out, int *overflow, uint64_t *mma_count);

/* reduction.hpp:113-122, :126-151, :189-231, :281-293, :298-341, :344-358 */
int orc_shuffle32(const float *x, size_t n, orc_outcome *out);
int orc_half_tree(const float *x, size_t n, orc_outcome *out);
int orc_recurrence(const float *x, size_t n, const orc_config *cfg, orc_outcome *out);
/* single_pass with `threads` worker threads over blocks (bit-identical for any thread
 * count: blocks are independent, the atomic stage stays serial).  block_out, if non-NULL,
 * receives the per-block results (blocks = max(1, ceil(n / (R*m*m*B/32)))). */
int orc_single_pass(const float *x, size_t n, const orc_config *cfg, int threads, orc_outcome *out,
                    float *block_out);
/* Same but the input is binary16 bits (already rounded): identical semantics. */
int orc_single_pass_f16(const uint16_t *h, size_t n, const orc_config *cfg, int threads,
                        orc_outcome *out, float *block_out);
int orc_split(const float *x, size_t n, const orc_config *cfg, orc_outcome *out);
int orc_reduce(const float *x, size_t n, const orc_config *cfg, orc_outcome *out);

size_t orc_block_count(size_t n, const orc_config *cfg);

#ifdef __cplusplus
}
#endif
#endif
