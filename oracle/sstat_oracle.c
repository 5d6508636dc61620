/*
 * sstat_oracle.c — CPU restatement of the reference sufficient-statistics path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or the CPU baseline — never as the product path.  The product path is
 * the CUDA library under paper_2604_23826_b200/ and fails loudly without it.
 *
 * Parity pinning: every function here is checked bit-for-bit against the
 * reference library itself (oracle/_ref, built from /root/reference/proj/src by
 * oracle/Makefile) and against the reference tests' known-answer vectors
 * (tests/golden/, tests/test_oracle.py).
 *
 * Reference anchors (paths relative to /root/reference/proj):
 *   check_chunk            src/suffstats.cpp:33-45
 *   accumulate_into<Acc>   src/suffstats.cpp:50-70   (row-major, ascending pairs,
 *                                                    separate mul + add: the
 *                                                    reference builds with
 *                                                    -ffp-contract=off, CMakeLists.txt:12-14)
 *   accumulate_chunk       src/suffstats.cpp:74-84
 *   merge_suffstats        src/suffstats.cpp:86-105
 *   accumulate_comoments   src/suffstats.cpp:107-132
 *   merge_comoments        src/suffstats.cpp:134-159
 *   plan_partitions        src/reduce.cpp:8-16
 *   run_reduction fold     include/sstat/reduce.hpp:70-146 (ascending range fold,
 *                                                    lowest failing range reported)
 *   column_sum             src/reduce.cpp:32-88
 *   RowRng / rand_between  include/sstat/rng.hpp:14-48
 *   make_record (Table1)   src/datagen.cpp:13-34
 *
 * Must be compiled with -ffp-contract=off (oracle/Makefile does).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_NONFINITE 1
#define ORC_INVALID 3

/* ---------------- RowRng (rng.hpp:14-48) ---------------- */
static const uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

static uint64_t mix64(uint64_t z) {
    z += kGolden;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

typedef struct { uint64_t base, pos; } row_rng;

static void rng_init(row_rng* r, uint64_t seed, uint64_t row_index) {
    r->base = mix64(mix64(seed) ^ mix64(row_index + kGolden));
    r->pos = 0;
}
static uint64_t rng_next(row_rng* r) { return mix64(r->base + (++r->pos) * kGolden); }
static double rng_unit(row_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static int64_t rng_between(int64_t lo, int64_t hi, row_rng* r) {
    uint64_t span = (uint64_t)(hi - lo) + 1;
    if (span == 0) return (int64_t)rng_next(r);
    return lo + (int64_t)(rng_next(r) % span);
}

uint64_t oracle_rowrng_u64(uint64_t seed, uint64_t row_index, uint64_t position) {
    row_rng r;
    rng_init(&r, seed, row_index);
    uint64_t v = 0;
    for (uint64_t i = 0; i < position; ++i) v = rng_next(&r);
    return v;
}

/* ---------------- synthetic generators ----------------
 * Measurement inputs; bit-portable to the CUDA generator
 * (paper_2604_23826_b200/csrc/generate.cu): integer SplitMix64 plus IEEE + - x in
 * a fixed order, no FMA.  Row index fed to RowRng is the 1-based row number,
 * as generate_row does (datagen.cpp:36-49).
 *   kind 0 (MIXED16): columns [0, n_int) integer rand_between(1,100), the rest
 *          Irwin-Hall Gaussians z (12 uniforms - 6) mixed x_j = mu + z_j + 0.5 z_{j-1}
 *          inside the Gaussian block;
 *   kind 1 (ID_GAUSS): column 0 = the 1-based row number, the rest Gaussian as above;
 *   kind 2 (GAUSS): every column Gaussian. */
#define GEN_MIXED 0
#define GEN_ID_GAUSS 1
#define GEN_GAUSS 2

static double irwin_hall(row_rng* r) {
    double s = 0.0;
    for (int i = 0; i < 12; ++i) s = s + rng_unit(r);
    return s - 6.0;
}

void oracle_generate(uint32_t kind, uint64_t seed, double mu, uint32_t n_int, uint64_t first_row,
                     uint64_t n_rows, uint32_t p, double* out) {
    for (uint64_t i = 0; i < n_rows; ++i) {
        const uint64_t index = first_row + i + 1;
        row_rng r;
        rng_init(&r, seed, index);
        double* row = out + i * p;
        uint32_t j = 0;
        if (kind == GEN_MIXED) {
            for (; j < n_int && j < p; ++j) row[j] = (double)rng_between(1, 100, &r);
        } else if (kind == GEN_ID_GAUSS) {
            row[0] = (double)index;
            j = 1;
        }
        double zprev = 0.0;
        for (; j < p; ++j) {
            const double z = irwin_hall(&r);
            row[j] = (mu + z) + 0.5 * zprev;
            zprev = z;
        }
    }
}

/* Table1 record (datagen.cpp:13-34): identifier A, B,C,D uniform ints, E..K derived. */
void oracle_table1_row(uint64_t seed, uint64_t index, double* out11) {
    row_rng r;
    rng_init(&r, seed, index);
    const int64_t ib = rng_between(3, 8, &r);
    const int64_t ic = rng_between(1, 10, &r);
    const int64_t id = rng_between(1, 100, &r);
    const double b = (double)ib, c = (double)ic, d = (double)id;
    out11[0] = (double)index;
    out11[1] = b;
    out11[2] = c;
    out11[3] = d;
    out11[4] = trunc(log(c) / log(b) * 100.0);
    out11[5] = round(log(d) / log(b) * 10000.0);
    out11[6] = trunc(fabs(cos(c)) * 100.0);
    out11[7] = trunc(fabs(sin(d)) * 100.0);
    const double cot_c = 1.0 / tan(c);
    out11[8] = round(fabs(cot_c) * 1000.0);
    out11[9] = fabs(tan(d));
    out11[10] = (double)(id / ic);
}

void oracle_table1_chunk(uint64_t seed, uint64_t first_index, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i) oracle_table1_row(seed, first_index + i, out + i * 11);
}

/* IidUniform rows (datagen.cpp:42-48): identifier then p uniforms lo + u*span. */
void oracle_iid_row(uint64_t seed, uint64_t index, uint32_t p, double lo, double hi, double* out) {
    row_rng r;
    rng_init(&r, seed, index);
    out[0] = (double)index;
    const double span = hi - lo;
    for (uint32_t j = 0; j < p; ++j) out[j + 1] = lo + rng_unit(&r) * span;
}

/* ---------------- accumulate_chunk (suffstats.cpp:33-84) ---------------- */

/* check_chunk: first non-finite in row-major order. */
static int check_chunk(const double* v, uint64_t rows, uint32_t p, uint64_t start_row,
                       uint64_t* err_row, uint32_t* err_col) {
    for (uint64_t r = 0; r < rows; ++r)
        for (uint32_t c = 0; c < p; ++c)
            if (!isfinite(v[r * p + c])) {
                if (err_row) *err_row = start_row + r;
                if (err_col) *err_col = c;
                return ORC_NONFINITE;
            }
    return ORC_OK;
}

static void accumulate_f64(const double* v, uint64_t rows, uint32_t p, double* sums, double* cross) {
    const size_t np = (size_t)p * (p + 1) / 2;
    double* s = calloc(p, sizeof(double));
    double* S = calloc(np, sizeof(double));
    for (uint64_t r = 0; r < rows; ++r) {
        const double* x = v + r * p;
        for (uint32_t j = 0; j < p; ++j) s[j] += x[j];
        double* out = S;
        for (uint32_t j = 0; j < p; ++j) {
            const double xj = x[j];
            for (uint32_t k = j; k < p; ++k) *out++ += xj * x[k];
        }
    }
    memcpy(sums, s, p * sizeof(double));
    memcpy(cross, S, np * sizeof(double));
    free(s);
    free(S);
}

static void accumulate_f32(const double* v, uint64_t rows, uint32_t p, double* sums, double* cross) {
    const size_t np = (size_t)p * (p + 1) / 2;
    float* s = calloc(p, sizeof(float));
    float* S = calloc(np, sizeof(float));
    float* x = calloc(p, sizeof(float));
    for (uint64_t r = 0; r < rows; ++r) {
        const double* row = v + r * p;
        for (uint32_t j = 0; j < p; ++j) {
            x[j] = (float)row[j];
            s[j] += x[j];
        }
        float* out = S;
        for (uint32_t j = 0; j < p; ++j) {
            const float xj = x[j];
            for (uint32_t k = j; k < p; ++k) *out++ += xj * x[k];
        }
    }
    for (uint32_t j = 0; j < p; ++j) sums[j] = (double)s[j];
    for (size_t i = 0; i < np; ++i) cross[i] = (double)S[i];
    free(s);
    free(S);
    free(x);
}

/* Returns ORC_OK or ORC_NONFINITE (err_row absolute, err_col). n_out = rows. */
int oracle_accumulate_chunk(const double* values, uint64_t rows, uint32_t p, uint64_t start_row,
                            uint32_t precision, uint64_t* n_out, double* sums, double* cross,
                            uint64_t* err_row, uint32_t* err_col) {
    if (p == 0) return ORC_INVALID;
    int st = check_chunk(values, rows, p, start_row, err_row, err_col);
    if (st != ORC_OK) return st;
    *n_out = rows;
    if (precision == 1) accumulate_f32(values, rows, p, sums, cross);
    else accumulate_f64(values, rows, p, sums, cross);
    return ORC_OK;
}

/* merge_suffstats (suffstats.cpp:86-105): a += b elementwise, binary32 path rounds each add. */
void oracle_merge(uint32_t p, uint32_t precision, uint64_t* n_a, double* sums_a, double* cross_a,
                  uint64_t n_b, const double* sums_b, const double* cross_b) {
    const size_t np = (size_t)p * (p + 1) / 2;
    *n_a += n_b;
    if (precision == 1) {
        for (uint32_t j = 0; j < p; ++j) sums_a[j] = (double)((float)sums_a[j] + (float)sums_b[j]);
        for (size_t i = 0; i < np; ++i) cross_a[i] = (double)((float)cross_a[i] + (float)cross_b[i]);
    } else {
        for (uint32_t j = 0; j < p; ++j) sums_a[j] += sums_b[j];
        for (size_t i = 0; i < np; ++i) cross_a[i] += cross_b[i];
    }
}

/* plan_partitions (reduce.cpp:8-16).  Returns the range count, or 0 on invalid input.
 * starts/counts may be NULL to query the count. */
uint64_t oracle_plan_partitions(uint64_t n_rows, uint64_t chunk_rows, uint64_t* starts, uint64_t* counts) {
    if (chunk_rows == 0 || n_rows == 0) return 0;
    uint64_t i = 0;
    for (uint64_t s = 0; s < n_rows; s += chunk_rows, ++i) {
        if (starts) starts[i] = s;
        if (counts) counts[i] = (chunk_rows < n_rows - s) ? chunk_rows : n_rows - s;
    }
    return i;
}

/* ---------------- run_reduction over in-memory rows (reduce.hpp:70-146) ----------------
 * A thread pool pulls ranges from an atomic counter, each range accumulates into its
 * own slot, then the slots fold in ascending range order from the empty identity.
 * The lowest failing range is reported.  rows points at the dataset's row 0. */
typedef struct {
    const double* rows;
    uint32_t p, precision;
    const uint64_t* starts;
    const uint64_t* counts;
    uint64_t n_ranges;
    double* slot_sums;   /* n_ranges * p */
    double* slot_cross;  /* n_ranges * np */
    uint64_t* slot_n;
    int* slot_status;
    uint64_t* slot_err_row;
    uint32_t* slot_err_col;
    volatile uint64_t next;
    volatile int failed;
} pool_job;

static void* pool_worker(void* arg) {
    pool_job* job = (pool_job*)arg;
    const size_t np = (size_t)job->p * (job->p + 1) / 2;
    while (!job->failed) {
        const uint64_t i = __atomic_fetch_add(&job->next, 1, __ATOMIC_RELAXED);
        if (i >= job->n_ranges) break;
        const double* chunk = job->rows + job->starts[i] * job->p;
        int st = oracle_accumulate_chunk(chunk, job->counts[i], job->p, job->starts[i], job->precision,
                                         &job->slot_n[i], job->slot_sums + i * job->p,
                                         job->slot_cross + i * np, &job->slot_err_row[i],
                                         &job->slot_err_col[i]);
        job->slot_status[i] = st;
        if (st != ORC_OK) job->failed = 1;
    }
    return NULL;
}

/* Returns ORC_OK, or ORC_NONFINITE with *err_range = lowest failing range index that
 * was processed (ranges never started after the failure are not examined, exactly as
 * the reference's workers stop pulling once `failed` is set). */
int oracle_run_reduction(const double* rows, uint32_t p, uint32_t precision, const uint64_t* starts,
                         const uint64_t* counts, uint64_t n_ranges, uint32_t workers, uint64_t* n_out,
                         double* sums, double* cross, uint64_t* err_range, uint64_t* err_row,
                         uint32_t* err_col) {
    if (p == 0 || workers == 0) return ORC_INVALID;
    const size_t np = (size_t)p * (p + 1) / 2;
    pool_job job;
    memset(&job, 0, sizeof job);
    job.rows = rows;
    job.p = p;
    job.precision = precision;
    job.starts = starts;
    job.counts = counts;
    job.n_ranges = n_ranges;
    job.slot_sums = calloc(n_ranges * p + 1, sizeof(double));
    job.slot_cross = calloc(n_ranges * np + 1, sizeof(double));
    job.slot_n = calloc(n_ranges + 1, sizeof(uint64_t));
    job.slot_status = calloc(n_ranges + 1, sizeof(int));
    job.slot_err_row = calloc(n_ranges + 1, sizeof(uint64_t));
    job.slot_err_col = calloc(n_ranges + 1, sizeof(uint32_t));
    for (uint64_t i = 0; i < n_ranges; ++i) job.slot_status[i] = -1;

    uint32_t pool = workers;
    if (pool > n_ranges) pool = n_ranges ? (uint32_t)n_ranges : 1;
    if (pool <= 1) {
        pool_worker(&job);
    } else {
        pthread_t* th = malloc(sizeof(pthread_t) * pool);
        for (uint32_t t = 0; t < pool; ++t) pthread_create(&th[t], NULL, pool_worker, &job);
        for (uint32_t t = 0; t < pool; ++t) pthread_join(th[t], NULL);
        free(th);
    }
    int st = ORC_OK;
    if (job.failed) {
        for (uint64_t i = 0; i < n_ranges; ++i)
            if (job.slot_status[i] > 0) {
                st = job.slot_status[i];
                if (err_range) *err_range = i;
                if (err_row) *err_row = job.slot_err_row[i];
                if (err_col) *err_col = job.slot_err_col[i];
                break;
            }
    } else {
        *n_out = 0;
        memset(sums, 0, p * sizeof(double));
        memset(cross, 0, np * sizeof(double));
        for (uint64_t i = 0; i < n_ranges; ++i)
            oracle_merge(p, precision, n_out, sums, cross, job.slot_n[i], job.slot_sums + i * p,
                         job.slot_cross + i * np);
    }
    free(job.slot_sums);
    free(job.slot_cross);
    free(job.slot_n);
    free(job.slot_status);
    free(job.slot_err_row);
    free(job.slot_err_col);
    return st;
}

/* Generator-fed run_reduction for the CPU baseline at sizes with no file: each worker
 * generates its range with oracle_generate into a private buffer, then accumulates it. */
typedef struct {
    uint32_t kind, n_int, p;
    uint64_t seed;
    double mu;
    const uint64_t* starts;
    const uint64_t* counts;
    uint64_t n_ranges;
    double* slot_sums;
    double* slot_cross;
    volatile uint64_t next;
} gen_job;

static void* gen_worker(void* arg) {
    gen_job* job = (gen_job*)arg;
    const size_t np = (size_t)job->p * (job->p + 1) / 2;
    double* buf = NULL;
    uint64_t cap = 0;
    for (;;) {
        const uint64_t i = __atomic_fetch_add(&job->next, 1, __ATOMIC_RELAXED);
        if (i >= job->n_ranges) break;
        if (job->counts[i] > cap) {
            free(buf);
            cap = job->counts[i];
            buf = malloc(cap * job->p * sizeof(double));
        }
        oracle_generate(job->kind, job->seed, job->mu, job->n_int, job->starts[i], job->counts[i], job->p, buf);
        uint64_t n;
        oracle_accumulate_chunk(buf, job->counts[i], job->p, job->starts[i], 0, &n, job->slot_sums + i * job->p,
                                job->slot_cross + i * np, NULL, NULL);
    }
    free(buf);
    return NULL;
}

void oracle_generated_reduction(uint32_t kind, uint64_t seed, double mu, uint32_t n_int, uint32_t p,
                                const uint64_t* starts, const uint64_t* counts, uint64_t n_ranges,
                                uint32_t workers, uint64_t* n_out, double* sums, double* cross) {
    const size_t np = (size_t)p * (p + 1) / 2;
    gen_job job;
    memset(&job, 0, sizeof job);
    job.kind = kind;
    job.n_int = n_int;
    job.p = p;
    job.seed = seed;
    job.mu = mu;
    job.starts = starts;
    job.counts = counts;
    job.n_ranges = n_ranges;
    job.slot_sums = calloc(n_ranges * p + 1, sizeof(double));
    job.slot_cross = calloc(n_ranges * np + 1, sizeof(double));
    uint32_t pool = workers ? workers : 1;
    pthread_t* th = malloc(sizeof(pthread_t) * pool);
    for (uint32_t t = 0; t < pool; ++t) pthread_create(&th[t], NULL, gen_worker, &job);
    for (uint32_t t = 0; t < pool; ++t) pthread_join(th[t], NULL);
    free(th);
    *n_out = 0;
    memset(sums, 0, p * sizeof(double));
    memset(cross, 0, np * sizeof(double));
    for (uint64_t i = 0; i < n_ranges; ++i)
        oracle_merge(p, 0, n_out, sums, cross, counts[i], job.slot_sums + i * p, job.slot_cross + i * np);
    free(job.slot_sums);
    free(job.slot_cross);
}

/* ---------------- column_sum (reduce.cpp:32-88) ----------------
 * f64 (or f32) sum plus an int128 exact sum while every value is integral and
 * |v| < 2^63.  Per range, then merged in ascending range order; the note names the
 * first non-integral row of the first failing range in fold order.
 * Outputs: float_sum; exact_ok; exact sum as (hi, lo) two's-complement 128-bit;
 * note_row = absolute row of the first non-integral value (when !exact_ok). */
int oracle_column_sum(const double* rows, uint32_t p, uint32_t column, uint32_t precision,
                      const uint64_t* starts, const uint64_t* counts, uint64_t n_ranges,
                      double* float_sum, int* exact_ok, int64_t* exact_hi, uint64_t* exact_lo,
                      uint64_t* note_row) {
    if (column >= p) return ORC_INVALID;
    const double kInt63 = 9223372036854775808.0;
    double f64 = 0.0;
    float f32 = 0.0f;
    __int128 exact = 0;
    int ok = 1;
    uint64_t nrow = 0;
    for (uint64_t i = 0; i < n_ranges; ++i) {
        double pf64 = 0.0;
        float pf32 = 0.0f;
        __int128 pex = 0;
        int pok = 1;
        uint64_t prow = 0;
        for (uint64_t r = 0; r < counts[i]; ++r) {
            const double v = rows[(starts[i] + r) * p + column];
            if (precision == 1) pf32 += (float)v;
            else pf64 += v;
            if (pok) {
                if (v == trunc(v) && fabs(v) < kInt63) pex += (__int128)v;
                else {
                    pok = 0;
                    prow = starts[i] + r;
                }
            }
        }
        if (precision == 1) f32 += pf32;
        else f64 += pf64;
        exact += pex;
        if (!pok && ok) {
            ok = 0;
            nrow = prow;
        }
    }
    *float_sum = precision == 1 ? (double)f32 : f64;
    *exact_ok = ok;
    *exact_hi = (int64_t)(exact >> 64);
    *exact_lo = (uint64_t)exact;
    *note_row = nrow;
    return ORC_OK;
}

/* ---------------- co-moments (suffstats.cpp:107-159) ---------------- */
int oracle_accumulate_comoments(const double* values, uint64_t rows, uint32_t p, uint64_t start_row,
                                uint64_t* n_out, double* mean, double* m2, uint64_t* err_row,
                                uint32_t* err_col) {
    int st = check_chunk(values, rows, p, start_row, err_row, err_col);
    if (st != ORC_OK) return st;
    const size_t np = (size_t)p * (p + 1) / 2;
    memset(mean, 0, p * sizeof(double));
    memset(m2, 0, np * sizeof(double));
    *n_out = rows;
    if (rows == 0) return ORC_OK;
    for (uint64_t r = 0; r < rows; ++r)
        for (uint32_t j = 0; j < p; ++j) mean[j] += values[r * p + j];
    for (uint32_t j = 0; j < p; ++j) mean[j] /= (double)rows;
    double* delta = malloc(p * sizeof(double));
    for (uint64_t r = 0; r < rows; ++r) {
        for (uint32_t j = 0; j < p; ++j) delta[j] = values[r * p + j] - mean[j];
        double* out = m2;
        for (uint32_t j = 0; j < p; ++j) {
            const double dj = delta[j];
            for (uint32_t k = j; k < p; ++k) *out++ += dj * delta[k];
        }
    }
    free(delta);
    return ORC_OK;
}

void oracle_merge_comoments(uint32_t p, uint64_t* n_a, double* mean_a, double* m2_a, uint64_t n_b,
                            const double* mean_b, const double* m2_b) {
    const size_t np = (size_t)p * (p + 1) / 2;
    if (n_b == 0) return;
    if (*n_a == 0) {
        *n_a = n_b;
        memcpy(mean_a, mean_b, p * sizeof(double));
        memcpy(m2_a, m2_b, np * sizeof(double));
        return;
    }
    const double na = (double)*n_a, nb = (double)n_b, n = na + nb;
    double* delta = malloc(p * sizeof(double));
    for (uint32_t j = 0; j < p; ++j) delta[j] = mean_b[j] - mean_a[j];
    const double scale = na * nb / n;
    size_t e = 0;
    for (uint32_t j = 0; j < p; ++j)
        for (uint32_t k = j; k < p; ++k, ++e) m2_a[e] = m2_a[e] + m2_b[e] + delta[j] * delta[k] * scale;
    for (uint32_t j = 0; j < p; ++j) mean_a[j] += delta[j] * (nb / n);
    *n_a += n_b;
    free(delta);
}

/* SymPacked index (linalg.hpp:58-61). */
uint64_t oracle_packed_index(uint64_t p, uint64_t j, uint64_t k) {
    if (j > k) {
        uint64_t t = j;
        j = k;
        k = t;
    }
    return j * p - j * (j - 1) / 2 + (k - j);
}
