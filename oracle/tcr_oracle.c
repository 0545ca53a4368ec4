/*
 * tcr_oracle.c -- CPU restatement of the reference tcreduce algorithms.
 *
 * TEST INFRASTRUCTURE ONLY (see tcr_oracle.h).  The B200 product path never
 * links this file; it exists so tests/ and bench.py can check the GPU results.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no -march: every float
 * operation must round exactly like the reference's g++ -O2 build).
 *
 * Citations are /root/reference/proj/include/tcreduce/<file>:<line>.
 */
#include "tcr_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ half.hpp */

static uint32_t round_shift_even(uint32_t v, unsigned s) { /* half.hpp:22-28 */
    const uint32_t halfway = 1u << (s - 1);
    const uint32_t rem = v & ((1u << s) - 1);
    uint32_t r = v >> s;
    if (rem > halfway || (rem == halfway && (r & 1u))) ++r;
    return r;
}

uint16_t orc_from_single(float x) { /* half.hpp:32-59 */
    uint32_t u;
    memcpy(&u, &x, sizeof u);
    const uint32_t sign = (u >> 16) & 0x8000u;
    u &= 0x7FFFFFFFu;
    if (u >= 0x7F800000u) {
        if (u > 0x7F800000u) return 0x7E00u;
        return (uint16_t)(sign | 0x7C00u);
    }
    const uint32_t e = u >> 23;
    const uint32_t m = u & 0x7FFFFFu;
    if (e < 113) {
        if (e < 102) return (uint16_t)sign;
        const uint32_t sig = round_shift_even(m | 0x800000u, 126 - e);
        return (uint16_t)(sign | sig);
    }
    if (e >= 143) return (uint16_t)(sign | 0x7C00u);
    uint32_t v = ((e - 112) << 10) | (m >> 13);
    const uint32_t rem = m & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (v & 1u))) ++v;
    if (v >= 0x7C00u) return (uint16_t)(sign | 0x7C00u);
    return (uint16_t)(sign | v);
}

float orc_to_single(uint16_t h) { /* half.hpp:61-79 */
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t e = (h >> 10) & 0x1Fu;
    const uint32_t m = h & 0x3FFu;
    uint32_t u;
    if (e == 0) {
        float f = (float)m * 0x1.0p-24f;
        memcpy(&u, &f, sizeof u);
        u |= sign;
    } else if (e == 31) {
        u = sign | 0x7F800000u | (m << 13);
    } else {
        u = sign | ((e + 112) << 23) | (m << 13);
    }
    float out;
    memcpy(&out, &u, sizeof out);
    return out;
}

int orc_is_overflowed(uint16_t h) { return (h & 0x7C00u) == 0x7C00u; } /* half.hpp:82 */

/* ------------------------------------------------------------------- rng.hpp */

#define SM_GAMMA 0x9E3779B97F4A7C15ull

static inline uint64_t sm_mix(uint64_t z) { /* rng.hpp:15-17 */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t orc_splitmix_next(uint64_t *state) { return sm_mix(*state += SM_GAMMA); } /* rng.hpp:13-18 */

/* After k calls of next() the state is seed + k*gamma (mod 2^64), so the k-th draw is
 * mix(seed + k*gamma).  This is what lets every GPU thread generate its own elements. */
uint64_t orc_splitmix_draw(uint64_t seed, uint64_t k) { return sm_mix(seed + k * SM_GAMMA); }

static inline double unit_of(uint64_t d) { return (double)(d >> 11) * 0x1.0p-53; }          /* rng.hpp:22 */
static inline double unit_open_of(uint64_t d) { return (double)((d >> 11) + 1) * 0x1.0p-53; } /* rng.hpp:25 */

/* --------------------------------------------------------------- harness.hpp */

int orc_generate(int kind, uint64_t seed, int64_t lo, int64_t hi, double c, size_t n, float *out) {
    /* harness.hpp:47-80, the reference's sequential loop verbatim in C */
    if (n < 1) return -1;
    uint64_t st = seed;
    switch (kind) {
    case ORC_CONSTANT:
        for (size_t i = 0; i < n; ++i) out[i] = (float)c;
        return 0;
    case ORC_UNIFORM:
        for (size_t i = 0; i < n; ++i) out[i] = (float)unit_of(orc_splitmix_next(&st));
        return 0;
    case ORC_INTEGERS: {
        if (hi < lo) return -1;
        const uint64_t span = (uint64_t)(hi - lo) + 1;
        for (size_t i = 0; i < n; ++i)
            out[i] = (float)(lo + (long long)(orc_splitmix_next(&st) % span));
        return 0;
    }
    case ORC_NORMAL:
        for (size_t i = 0; i < n; i += 2) {
            const double u1 = unit_open_of(orc_splitmix_next(&st));
            const double u2 = unit_of(orc_splitmix_next(&st));
            const double r = sqrt(-2.0 * log(u1));
            const double t = 2.0 * 3.141592653589793238462643383279502884 * u2;
            out[i] = (float)(r * cos(t));
            if (i + 1 < n) out[i + 1] = (float)(r * sin(t));
        }
        return 0;
    }
    return -1;
}

int orc_generate_range(int kind, uint64_t seed, int64_t lo, int64_t hi, double c, size_t first,
                       size_t count, float *out) {
    /* Jump-ahead restatement of harness.hpp:47-80: element i of uniform/integers uses draw
     * i+1; normal pair p = i/2 uses draws 2p+1 (u1, open) and 2p+2 (u2); even i -> cos. */
    switch (kind) {
    case ORC_CONSTANT:
        for (size_t i = 0; i < count; ++i) out[i] = (float)c;
        return 0;
    case ORC_UNIFORM:
        for (size_t i = 0; i < count; ++i) out[i] = (float)unit_of(orc_splitmix_draw(seed, first + i + 1));
        return 0;
    case ORC_INTEGERS: {
        if (hi < lo) return -1;
        const uint64_t span = (uint64_t)(hi - lo) + 1;
        for (size_t i = 0; i < count; ++i)
            out[i] = (float)(lo + (long long)(orc_splitmix_draw(seed, first + i + 1) % span));
        return 0;
    }
    case ORC_NORMAL:
        for (size_t i = 0; i < count; ++i) {
            const size_t g = first + i, p = g >> 1;
            const double u1 = unit_open_of(orc_splitmix_draw(seed, 2 * p + 1));
            const double u2 = unit_of(orc_splitmix_draw(seed, 2 * p + 2));
            const double r = sqrt(-2.0 * log(u1));
            const double t = 2.0 * 3.141592653589793238462643383279502884 * u2;
            out[i] = (float)((g & 1) ? r * sin(t) : r * cos(t));
        }
        return 0;
    }
    return -1;
}

int orc_generate_range_f16(int kind, uint64_t seed, int64_t lo, int64_t hi, double c, size_t first,
                           size_t count, uint16_t *out) {
    const size_t CH = 4096;
    float buf[4096];
    for (size_t s = 0; s < count; s += CH) {
        const size_t k = count - s < CH ? count - s : CH;
        int rc = orc_generate_range(kind, seed, lo, hi, c, first + s, k, buf);
        if (rc) return rc;
        for (size_t i = 0; i < k; ++i) out[s + i] = orc_from_single(buf[i]);
    }
    return 0;
}

/* ------------------------------------------------------------- reduction.hpp */

double orc_oracle64(const float *x, size_t n) { /* reduction.hpp:106-110 */
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) acc += (double)x[i];
    return acc;
}

void orc_exact_sum_f16(const uint16_t *h, size_t n, double *sum, double *abs_sum) {
    /* Every finite binary16 is an integer multiple of 2^-24 below 2^40 in those units,
     * so a 128-bit fixed-point sum is exact for any n < 2^87. */
    __int128 s = 0, a = 0;
    int nonfinite = 0;
    double nf = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const uint16_t b = h[i];
        if ((b & 0x7C00u) == 0x7C00u) {
            nonfinite = 1;
            nf += (double)orc_to_single(b);
            continue;
        }
        const int64_t mag = (int64_t)ldexp((double)fabsf(orc_to_single(b)), 24);
        s += (b & 0x8000u) ? -mag : mag;
        a += mag;
    }
    if (nonfinite) {
        *sum = nf;
        *abs_sum = INFINITY;
        return;
    }
    *sum = ldexp((double)s, -24); /* one rounding: __floattidf is round-to-nearest */
    *abs_sum = ldexp((double)a, -24);
}

static int check_side(size_t m) { return (m < 2 || (m & (m - 1)) != 0) ? -1 : 0; } /* fragment.hpp:22-25 */

int orc_validate(const orc_config *cfg) { /* reduction.hpp:50-56 */
    if (check_side(cfg->m)) return -1;
    if (cfg->R < 1) return -1;
    if (cfg->B < 32 || cfg->B > 1024 || cfg->B % 32 != 0) return -1;
    if (cfg->f < 0.0 || cfg->f > 1.0) return -1;
    return 0;
}

size_t orc_warp_offset(size_t block, size_t warp, const orc_config *cfg) { /* :154-158 */
    return (size_t)cfg->R * cfg->m * cfg->m * (block * (cfg->B / 32) + warp);
}

static size_t next_pow2(size_t n) { /* reduction.hpp:86 */
    size_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

/* reduction.hpp:90-101 on a caller-provided buffer already padded to pow2 with zeros */
static unsigned pairwise_tree(float *v, size_t p, uint64_t *ops) {
    unsigned levels = 0;
    for (size_t len = p; len > 1; len /= 2) {
        for (size_t i = 0; i < len / 2; ++i) {
            v[i] = v[i] + v[i + len / 2];
            ++*ops;
        }
        ++levels;
    }
    return levels;
}

/* Element source: fp32 input (converted with from_single at load, fragment.hpp:68) or
 * binary16 bits.  Elements at index >= n read as +0 (the zero padding of :244-245). */
typedef struct {
    const float *f32;
    const uint16_t *f16;
    size_t n;
} src_t;

static inline uint16_t src_half(const src_t *s, size_t i) {
    if (i >= s->n) return 0;
    return s->f16 ? s->f16[i] : orc_from_single(s->f32[i]);
}

/* chained_warp_reduce (reduction.hpp:164-184) with the emulated mma (fragment.hpp:82-97).
 * ones x M has identical rows, so row 0 of every product is computed (bit-identical to
 * computing all m rows); the overflow note over all m^2 entries of the C_R copy equals the
 * note over row 0 for the same reason.  Caller guarantees base + R*m^2 <= padded size. */
static float chained_core(const src_t *s, size_t base, unsigned m, unsigned R, int *overflow,
                          float *c /* scratch, m floats */, float *col /* scratch */) {
    const size_t group = (size_t)m * m;
    for (unsigned j = 0; j < m; ++j) c[j] = 0.0f;                        /* :172 */
    for (unsigned r = 0; r < R; ++r) {
        const size_t off = base + (size_t)r * group;
        for (unsigned j = 0; j < m; ++j) col[j] = 0.0f;                  /* acc = 0.0f */
        for (unsigned k = 0; k < m; ++k) {                               /* ascending k */
            for (unsigned j = 0; j < m; ++j) {
                const uint16_t h = src_half(s, off + (size_t)k * m + j); /* load_fragment */
                if (orc_is_overflowed(h)) *overflow = 1;                 /* sc.note(mr) */
                col[j] += 1.0f * orc_to_single(h);                       /* to_single(1)*to_single(b) */
            }
        }
        for (unsigned j = 0; j < m; ++j) c[j] = col[j] + c[j];           /* + c.at(i,j), C last */
    }
    float d = 0.0f;                                                      /* second mma, row 0 */
    for (unsigned j = 0; j < m; ++j) {
        const uint16_t a = orc_from_single(c[j]);                        /* :180 */
        if (orc_is_overflowed(a)) *overflow = 1;                         /* :181 */
        d += orc_to_single(a) * 1.0f;
    }
    return d + 0.0f;                                                     /* + fill_accum(0) */
}

int orc_chained_warp_reduce(const float *x, size_t n, size_t base, const orc_config *cfg,
                            float *out, int *overflow, uint64_t *mma_count) {
    if (check_side(cfg->m)) return -1;
    const size_t group = (size_t)cfg->m * cfg->m;
    if (base + cfg->R * group > n) return -2; /* :168-169 */
    src_t s = {x, NULL, n};
    float *c = malloc(2 * sizeof(float) * cfg->m);
    *out = chained_core(&s, base, cfg->m, cfg->R, overflow, c, c + cfg->m);
    free(c);
    *mma_count += cfg->R + 1;
    return 0;
}

size_t orc_block_count(size_t n, const orc_config *cfg) { /* :240-242 */
    const size_t chunk_block = (size_t)cfg->R * cfg->m * cfg->m * (cfg->B / 32);
    size_t b = (n + chunk_block - 1) / chunk_block;
    return b < 1 ? 1 : b;
}

typedef struct {
    const src_t *s;
    const orc_config *cfg;
    size_t blocks, t, T;
    float *block_results;
    int overflow;
} sp_job;

static void *sp_worker(void *arg) {
    sp_job *j = (sp_job *)arg;
    const unsigned W = j->cfg->B / 32, m = j->cfg->m, R = j->cfg->R;
    const size_t P = next_pow2(W);
    float *v = malloc(sizeof(float) * (P + 2 * m));
    float *c = v + P;
    for (size_t b = j->t; b < j->blocks; b += j->T) {
        for (size_t w = 0; w < P; ++w) v[w] = 0.0f;
        for (unsigned w = 0; w < W; ++w)                                /* :251-252 */
            v[w] = chained_core(j->s, orc_warp_offset(b, w, j->cfg), m, R, &j->overflow, c, c + m);
        uint64_t ops = 0;
        pairwise_tree(v, P, &ops);                                      /* :253 */
        j->block_results[b] = v[0];                                     /* :254 */
    }
    free(v);
    return NULL;
}

/* detail::single_pass_core + single_pass_reduce (reduction.hpp:238-293) */
static int single_pass_src(const src_t *s, const orc_config *cfg, int threads, orc_outcome *out,
                           float *block_out) {
    if (s->n == 0) return -1;  /* :282 */
    if (orc_validate(cfg)) return -1; /* :283 */
    const size_t blocks = orc_block_count(s->n, cfg);
    float *br = block_out ? block_out : malloc(sizeof(float) * blocks);
    if (threads < 1) threads = 1;
    if ((size_t)threads > blocks) threads = (int)blocks;
    sp_job *jobs = calloc((size_t)threads, sizeof(sp_job));
    pthread_t *tid = calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (sp_job){s, cfg, blocks, (size_t)t, (size_t)threads, br, 0};
        if (threads == 1) sp_worker(&jobs[t]);
        else pthread_create(&tid[t], NULL, sp_worker, &jobs[t]);
    }
    int overflow = 0;
    for (int t = 0; t < threads; ++t) {
        if (threads > 1) pthread_join(tid[t], NULL);
        overflow |= jobs[t].overflow;
    }
    free(jobs);
    free(tid);

    /* :257-268 -- serial "atomic" accumulation, ascending or seeded Fisher-Yates order */
    float acc = 0.0f;
    if (cfg->atomic_order == ORC_SEEDED_PERMUTATION) {
        size_t *order = malloc(sizeof(size_t) * blocks);
        for (size_t i = 0; i < blocks; ++i) order[i] = i;
        uint64_t st = cfg->atomic_seed;
        for (size_t i = blocks; i > 1; --i) {
            const size_t r = (size_t)(orc_splitmix_next(&st) % i);
            const size_t tmp = order[i - 1];
            order[i - 1] = order[r];
            order[r] = tmp;
        }
        for (size_t i = 0; i < blocks; ++i) acc += br[order[i]];
        free(order);
    } else {
        for (size_t b = 0; b < blocks; ++b) acc += br[b];
    }
    if (!block_out) free(br);

    const unsigned W = cfg->B / 32;
    const size_t P = next_pow2(W);
    unsigned tree_levels = 0;
    for (size_t len = P; len > 1; len /= 2) ++tree_levels;
    memset(out, 0, sizeof *out);
    out->value = acc;
    out->overflow = overflow;
    out->level_count = 1;
    out->sim_steps = 2ull * cfg->R + 2 + tree_levels + blocks;          /* :271-273 */
    out->mma_count = (uint64_t)blocks * W * (cfg->R + 1);
    out->atomic_count = blocks;
    out->shuffle_count = (uint64_t)blocks * (P - 1);
    return 0;
}

int orc_single_pass(const float *x, size_t n, const orc_config *cfg, int threads, orc_outcome *out,
                    float *block_out) {
    src_t s = {x, NULL, n};
    return single_pass_src(&s, cfg, threads, out, block_out);
}

int orc_single_pass_f16(const uint16_t *h, size_t n, const orc_config *cfg, int threads,
                        orc_outcome *out, float *block_out) {
    src_t s = {NULL, h, n};
    return single_pass_src(&s, cfg, threads, out, block_out);
}

int orc_shuffle32(const float *x, size_t n, orc_outcome *out) { /* reduction.hpp:113-122 */
    if (n == 0) return -1;
    const size_t P = next_pow2(n);
    float *v = calloc(P, sizeof(float));
    memcpy(v, x, n * sizeof(float));
    memset(out, 0, sizeof *out);
    const unsigned levels = pairwise_tree(v, P, &out->shuffle_count);
    out->value = v[0];
    out->level_count = levels;
    out->sim_steps = 4ull * levels;
    free(v);
    return 0;
}

int orc_half_tree(const float *x, size_t n, orc_outcome *out) { /* reduction.hpp:126-151 */
    if (n == 0) return -1;
    memset(out, 0, sizeof *out);
    const size_t P = next_pow2(n);
    float *v = calloc(P, sizeof(float));
    for (size_t i = 0; i < n; ++i) {
        const uint16_t h = orc_from_single(x[i]);
        if (orc_is_overflowed(h)) out->overflow = 1;
        v[i] = orc_to_single(h);
    }
    unsigned levels = 0;
    for (size_t len = P; len > 1; len /= 2) {
        for (size_t i = 0; i < len / 2; ++i) {
            const uint16_t h = orc_from_single(v[i] + v[i + len / 2]);
            if (orc_is_overflowed(h)) out->overflow = 1;
            v[i] = orc_to_single(h);
            ++out->shuffle_count;
        }
        ++levels;
    }
    out->value = v[0];
    out->level_count = levels;
    out->sim_steps = 4ull * levels;
    free(v);
    return 0;
}

int orc_recurrence(const float *x, size_t n0, const orc_config *cfg, orc_outcome *out) {
    /* reduction.hpp:189-231 */
    if (n0 == 0) return -1;
    if (orc_validate(cfg)) return -1;
    memset(out, 0, sizeof *out);
    const unsigned m = cfg->m, R = cfg->R;
    const size_t group = (size_t)m * m, chunk = (size_t)R * group;
    float *work = malloc(sizeof(float) * n0);
    memcpy(work, x, sizeof(float) * n0);
    float *c = malloc(2 * sizeof(float) * m);
    int overflow = 0;
    uint64_t mma = 0, steps = 0;
    size_t n = n0;
    while (n >= group) {
        const size_t count = (n + chunk - 1) / chunk;
        src_t s = {work, NULL, n}; /* work.resize(count*chunk, 0): reads past n are zero */
        float *next = malloc(sizeof(float) * count);
        for (size_t i = 0; i < count; ++i) {
            const float r = chained_core(&s, i * chunk, m, R, &overflow, c, c + m);
            mma += R + 1;
            const uint16_t h = orc_from_single(r);
            if (orc_is_overflowed(h)) overflow = 1;
            next[i] = orc_to_single(h);
        }
        free(work);
        work = next;
        n = count;
        ++out->level_count;
        steps += 2ull * R + 3;
    }
    if (n == 1) {
        out->value = work[0];
    } else {
        src_t s = {work, NULL, n}; /* resize(group, 0) */
        out->value = chained_core(&s, 0, m, 1, &overflow, c, c + m);
        mma += 2;
        steps += 5;
    }
    free(work);
    free(c);
    out->overflow = overflow;
    out->sim_steps = steps;
    out->mma_count = mma;
    return 0;
}

int orc_split(const float *x, size_t n, const orc_config *cfg, orc_outcome *out) {
    /* reduction.hpp:298-341 */
    if (n == 0) return -1;
    if (orc_validate(cfg)) return -1;
    orc_config tcfg = *cfg;
    tcfg.R = 1;
    const size_t chunk_block = (size_t)cfg->m * cfg->m * (cfg->B / 32);
    size_t tensor_len = (size_t)(cfg->f * (double)n);
    tensor_len = tensor_len / chunk_block * chunk_block;
    memset(out, 0, sizeof *out);
    orc_outcome t = {0}, sh = {0};
    float tensor_part = 0.0f, shuffle_part = 0.0f;
    uint64_t tensor_steps = 0, shuffle_steps = 0;
    if (tensor_len > 0) {
        src_t s = {x, NULL, tensor_len};
        single_pass_src(&s, &tcfg, 1, &t, NULL);
        tensor_part = (float)t.value;
        tensor_steps = t.sim_steps;
        out->level_count = 1;
    }
    if (tensor_len < n) {
        orc_shuffle32(x + tensor_len, n - tensor_len, &sh);
        shuffle_part = (float)sh.value;
        shuffle_steps = sh.sim_steps;
        out->shuffle_count = sh.shuffle_count;
        if (sh.level_count > out->level_count) out->level_count = sh.level_count;
    }
    if (tensor_len == 0) out->value = shuffle_part;
    else if (tensor_len == n) out->value = tensor_part;
    else out->value = tensor_part + shuffle_part;
    out->overflow = t.overflow;
    out->sim_steps = (tensor_steps > shuffle_steps ? tensor_steps : shuffle_steps) +
                     ((tensor_len > 0 && tensor_len < n) ? 1 : 0);
    out->mma_count = t.mma_count;
    out->atomic_count = t.atomic_count;
    out->shuffle_count += t.shuffle_count;
    return 0;
}

int orc_reduce(const float *x, size_t n, const orc_config *cfg, orc_outcome *out) {
    switch (cfg->variant) { /* reduction.hpp:344-358 */
    case ORC_ORACLE64:
        memset(out, 0, sizeof *out);
        out->value = orc_oracle64(x, n);
        return 0;
    case ORC_SHUFFLE32: return orc_shuffle32(x, n, out);
    case ORC_HALF_TREE: return orc_half_tree(x, n, out);
    case ORC_RECURRENCE: return orc_recurrence(x, n, cfg, out);
    case ORC_SINGLE_PASS: return orc_single_pass(x, n, cfg, 1, out, NULL);
    case ORC_SPLIT: return orc_split(x, n, cfg, out);
    }
    return -1;
}
