/*
 * sstat_cuda.h — C ABI of the B200 sufficient-statistics engine (libsstat_b200.so).
 *
 * Drop-in boundary for the reference's single-pass sufficient-statistics path
 * (paths relative to /root/reference/proj):
 *
 *   reference symbol                                   replaced by
 *   -------------------------------------------------  ------------------------------
 *   accumulate_chunk(Chunk, DatasetSchema, Precision)  sstat_cuda_accumulate
 *     include/sstat/suffstats.hpp:50-51, src/suffstats.cpp:74-84
 *   dataset_suffstats(path, schema, plan, timings)     sstat_cuda_dataset
 *     include/sstat/suffstats.hpp:71-72, src/suffstats.cpp:279-288
 *     = run_reduction<SuffStats>(accumulate_chunk, merge_suffstats)
 *       include/sstat/reduce.hpp:70-146
 *   merge_suffstats(SuffStats, SuffStats)              sstat_merge (host, tiny)
 *     include/sstat/suffstats.hpp:54, src/suffstats.cpp:86-105
 *   plan_partitions(n, chunk_rows)                     sstat_plan_partitions (host)
 *     include/sstat/reduce.hpp:36, src/reduce.cpp:8-16
 *   column_sum(path, column, plan)                     sstat_cuda_column_sum
 *     include/sstat/reduce.hpp:148-162, src/reduce.cpp:32-88
 *   accumulate_comoments / merge_comoments             sstat_cuda_comoments
 *     include/sstat/suffstats.hpp:56-57, src/suffstats.cpp:107-159
 *
 * Conventions.  Plain pointers and sizes only.  Every pointer is caller-owned and
 * borrowed for the duration of the call; nothing allocated by the library crosses
 * the ABI.  Row data is row-major little-endian binary64, exactly the Chunk layout
 * (chunk.hpp:13-24) and the SSTATBIN payload (binfile.hpp:17-29).  Outputs follow
 * SuffStats (suffstats.hpp:19-30): n, sums[p], cross[p(p+1)/2] as the packed upper
 * triangle in SymPacked order (linalg.hpp:50-61), index(j,k) = j*p - j*(j-1)/2 + (k-j).
 *
 * Errors.  Functions return an sstat_status.  The reference throws; the C++ glue
 * (integration/sstat_cuda_glue.hpp) maps codes back to its exception types:
 *   SSTAT_ERR_NONFINITE  accumulate: NonFiniteError(row, col)            errors.hpp:59-72
 *                        dataset:    ReductionError(range_index, "range i failed:
 *                                    non-finite value at row R, column C")
 *                                    (reduce.hpp:132-134, suffstats.cpp:41-44)
 *   SSTAT_ERR_SCHEMA     SchemaMismatchError                             errors.hpp:52-56
 *   SSTAT_ERR_INVALID    std::invalid_argument / std::out_of_range
 *   SSTAT_ERR_IO / _FORMAT  IoError / FormatError (file sources)         errors.hpp:18-30
 *   SSTAT_ERR_UNSUPPORTED  also: p > 2048 columns outside reference-order mode (the fast
 *                        path stages whole rows in shared memory)
 *   SSTAT_ERR_PEER       another rank of the communicator failed
 *   SSTAT_ERR_CUDA / _NCCL / _OOM / _UNSUPPORTED  device-side failures (no reference
 *                        equivalent; the glue throws sstat::Error).
 *
 * Threading.  A context is bound to one CUDA device and serialises its own calls
 * (internal mutex); distinct contexts are independent.  The only process-wide state is
 * K2's write-once, mutex-guarded launch-geometry cache per (device, p).
 */
#ifndef SSTAT_CUDA_H
#define SSTAT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSTAT_CUDA_ABI_VERSION 2

typedef enum {
    SSTAT_OK = 0,
    SSTAT_ERR_NONFINITE = 1,
    SSTAT_ERR_SCHEMA = 2,
    SSTAT_ERR_INVALID = 3,
    SSTAT_ERR_CUDA = 4,
    SSTAT_ERR_NCCL = 5,
    SSTAT_ERR_OOM = 6,
    SSTAT_ERR_UNSUPPORTED = 7,
    SSTAT_ERR_IO = 8,
    SSTAT_ERR_FORMAT = 9,
    SSTAT_ERR_PEER = 10 /* another rank of the communicator failed (its status is in msg)  */
} sstat_status;

/* PrecisionMode (reduce.hpp:40-45). */
#define SSTAT_PRECISION_BINARY64 0u
#define SSTAT_PRECISION_BINARY32_DIAGNOSTIC 1u

/* Accumulation flags.
 *   SSTAT_FLAG_NO_SHIFT  accumulate raw x instead of x - c, c = first row of each
 *                        range (the default per-range shift; results are mapped back
 *                        to raw sums / X^T X, exactly for integer data).
 *   SSTAT_FLAG_REFEXACT  reference-order mode: one sequential multiply-then-add chain
 *                        per (range, entry) in the order of accumulate_into
 *                        (suffstats.cpp:56-67) and the ascending range fold
 *                        (reduce.hpp:142-145): bit-identical to the reference for any
 *                        data.  Required for Binary32Diagnostic.
 */
#define SSTAT_FLAG_NO_SHIFT (1u << 0)
#define SSTAT_FLAG_REFEXACT (1u << 1)

typedef struct sstat_cuda_ctx sstat_cuda_ctx;

typedef struct {
    uint64_t row;         /* absolute 0-based row of the first non-finite value   */
    uint32_t col;         /* its 0-based column                                   */
    uint32_t status;      /* sstat_status of the failing call                     */
    uint64_t range_index; /* dataset calls: lowest failing range (ReductionError) */
    char msg[256];        /* reference-format message                             */
} sstat_cuda_error;

/* ReductionTimings (reduce.hpp:56-60), device-side breakdown. */
typedef struct {
    double h2d_seconds;      /* host->device copies, first start to last end (host / file sources) */
    double kernel_seconds;   /* accumulate kernels, device events                   */
    double exchange_seconds; /* NCCL all-gather of per-range partials               */
    double fold_seconds;     /* per-range + ascending range folds                   */
    double total_seconds;    /* whole call, host wall clock                         */
    uint64_t bytes_read;     /* payload bytes this rank consumed (rows * p * 8)     */
    uint64_t h2d_bytes;      /* bytes copied host->device                           */
    uint32_t kernel_launches;/* kernels launched by the call                        */
    uint32_t n_local_ranges; /* ranges this rank accumulated                        */
    char kernel[96];         /* the accumulate kernel that ran, e.g. "k_smallp<2, true>" */
} sstat_cuda_timings;

typedef enum {
    SSTAT_SRC_DEVICE = 0, /* ptr is device memory on the context's device          */
    SSTAT_SRC_HOST = 1,   /* ptr is host memory (pinned: direct DMA; else staged)  */
    SSTAT_SRC_FILE = 2,   /* path names an SSTATBIN file (binfile.hpp:17-29)        */
    SSTAT_SRC_READER = 3  /* rows come from read_rows (below)                       */
} sstat_source_kind;

/* The reader of an SSTAT_SRC_READER source: BinaryReader::read_rows (reference
 * src/binfile.cpp:140-161) as a C callback.  The engine asks for rows [first_row, first_row +
 * n_rows) (whole staging slots, ascending, one call at a time per device) and the callback
 * either copies them into `scratch` (pinned staging memory of n_rows * p * 8 bytes) and returns
 * scratch, or returns a pointer to host memory already holding them (pinned memory is copied to
 * the device by DMA directly) that stays valid until the pass returns.  NULL = the read failed
 * (SSTAT_ERR_IO).  Lets a dataset larger than host memory stream through the pinned ring. */
typedef const void* (*sstat_read_rows_fn)(void* user, uint64_t first_row, uint64_t n_rows, void* scratch);

typedef struct {
    uint32_t kind;        /* sstat_source_kind                                       */
    uint32_t reserved;
    const void* ptr;      /* DEVICE/HOST: rows [first_row, first_row + n_rows)       */
    uint64_t first_row;   /* absolute dataset row held at ptr[0] (READER: first row  */
    uint64_t n_rows;      /* rows addressable (READER: rows read_rows can serve);    */
                          /* 0 with ptr NULL: an empty shard (a rank or group member */
                          /* holding no ranges)                                      */
    const char* path;     /* FILE                                                    */
    sstat_read_rows_fn read_rows; /* READER                                          */
    void* user;           /* READER: passed to read_rows                             */
} sstat_cuda_source;

/* ---- library / context ---- */
int sstat_cuda_abi_version(void);
const char* sstat_status_string(int status);

/* One context per process per device.  device < 0 selects the current device. */
int sstat_cuda_init(sstat_cuda_ctx** ctx, int device);

/* A device group: one process driving n_gpus devices (SURVEY.md §8(b) Export 1; the paper's
 * single host process over all GPUs).  Member i is rank i of n_gpus: the plan's
 * ranges are sharded contiguously exactly as in the multi-process path (sstat_shard_ranges),
 * every member accumulates its share in parallel on its own host thread, and the rank buffers
 * meet on devices[0] for the same ascending fold — results are bit-identical to one device and
 * to n_gpus processes.  Exchange: fused by default — when every member reaches devices[0]'s memory
 * (the same device, or peer access over NVLink) each member's fold kernel writes its range
 * partials straight into devices[0]'s gather buffer; otherwise NCCL communicators from
 * ncclCommInitAll (distinct devices) or peer copies.  SSTAT_GROUP_EXCHANGE=fused|copy|nccl
 * overrides.  Group calls:
 *   sstat_cuda_dataset / _comoments / _column_sum: a FILE or HOST source is read by every member
 *     (each its own ranges); a DEVICE source is an ARRAY of n_gpus sources, element i = member
 *     i's shard on devices[i] (first_row / n_rows as in the multi-process call);
 *   sstat_cuda_accumulate: the member whose device holds the chunk (host chunks: member 0);
 *   sstat_cuda_range_partials: member 0;
 *   sstat_cuda_generate: the member whose device holds dst;
 *   sstat_cuda_set_staging / _set_host_threads: every member (host threads default to
 *     min(16, cores) / n_gpus per member);
 *   sstat_cuda_set_stream (non-NULL) and sstat_cuda_comm_init: rejected.
 * n_gpus = 0 (devices NULL): every visible device. */
int sstat_cuda_init_devices(sstat_cuda_ctx** ctx, int n_gpus, const int* devices);
/* Devices a context drives: 1, or the group's n_gpus. */
int sstat_cuda_device_count(const sstat_cuda_ctx* ctx);
int sstat_cuda_destroy(sstat_cuda_ctx* ctx);

/* Launch work on an external cudaStream_t (e.g. the host framework's current stream);
 * NULL restores the context's own stream.  The own stream is a blocking stream: it is ordered
 * after work on the legacy default stream, so device sources written there need no sync. */
int sstat_cuda_set_stream(sstat_cuda_ctx* ctx, void* cuda_stream);

/* Host staging for HOST/FILE sources: `slots` device buffers of `slot_bytes` each. */
int sstat_cuda_set_staging(sstat_cuda_ctx* ctx, uint32_t slots, uint64_t slot_bytes);

/* Host feeder threads for PAGEABLE/FILE sources (the loader of reference
 * src/binfile.cpp:140-161 BinaryReader::read_rows): each staging slot is filled by
 * `threads` parallel pread/memcpy workers, so the pass runs at the H2D link rate rather than
 * one core's copy rate.  0 = min(16, hardware threads).  Does not change any result. */
int sstat_cuda_set_host_threads(sstat_cuda_ctx* ctx, uint32_t threads);

/* ---- multi-GPU (one process per GPU, rows sharded contiguously by range) ----
 * A rank whose local phase fails still joins the exchange with its status in its header: every
 * rank returns an error (the failing one its own, the others SSTAT_ERR_PEER), none hangs —
 * except after a sticky CUDA error, which leaves the device unable to take part. */
/* 128-byte ncclUniqueId, created on rank 0 and broadcast by the host framework. */
int sstat_cuda_nccl_unique_id(void* id_out, size_t id_bytes);
int sstat_cuda_comm_init(sstat_cuda_ctx* ctx, int rank, int world, const void* id, size_t id_bytes);
/* Ranges [first, last) owned by `rank`: first = floor(rank * n_ranges / world). */
int sstat_shard_ranges(uint64_t n_ranges, int rank, int world, uint64_t* first, uint64_t* last);

/* ---- the hot path ---- */

/* accumulate_chunk: rows is a host or device pointer to n_rows x p binary64. */
int sstat_cuda_accumulate(sstat_cuda_ctx* ctx, const double* rows, uint64_t n_rows, uint32_t p,
                          uint64_t start_row, uint32_t precision, uint32_t flags, uint64_t* n_out,
                          double* sums_out, double* cross_out, sstat_cuda_error* err);

/* dataset_suffstats: the plan's ranges (ascending, contiguous, covering the dataset),
 * accumulated per range, folded in ascending range order.  With a communicator of
 * world W, every rank passes the full plan and a source holding at least its shard
 * (sstat_shard_ranges); every rank returns the same result.  Output pointers are host. */
int sstat_cuda_dataset(sstat_cuda_ctx* ctx, const sstat_cuda_source* src, uint32_t p,
                       const uint64_t* range_start, const uint64_t* range_count, uint64_t n_ranges,
                       uint32_t precision, uint32_t flags, uint64_t* n_out, double* sums_out,
                       double* cross_out, sstat_cuda_timings* timings, sstat_cuda_error* err);

/* Per-range partials of ranges [first_range, last_range) of the plan, without the fold:
 * (last_range - first_range) x (p + p(p+1)/2) doubles into host memory, each
 * [sums | packed cross] in raw (unshifted) space — what one rank contributes to the
 * exchange.  For persisting partials (resume) and for checking the multi-GPU layout. */
int sstat_cuda_range_partials(sstat_cuda_ctx* ctx, const sstat_cuda_source* src, uint32_t p,
                              const uint64_t* range_start, const uint64_t* range_count, uint64_t n_ranges,
                              uint64_t first_range, uint64_t last_range, uint32_t precision, uint32_t flags,
                              double* partials_out, sstat_cuda_error* err);

/* ---- the passes next to the path ---- */

/* ColumnSumResult (reduce.hpp:148-158). */
typedef struct {
    double float_sum;            /* binary64 (or binary32 widened) sum of the column          */
    int32_t exact_ok;            /* every value integral and |v| < 2^63: exact sum present    */
    int32_t float_matches_exact; /* double_equals_int128(float_sum, exact)  (util.cpp:47-52)  */
    int64_t exact_hi;            /* exact sum, two's-complement 128-bit: hi:lo                */
    uint64_t exact_lo;
    uint64_t note_row;           /* !exact_ok: absolute row of the first non-integral value   */
} sstat_column_sum_result;

/* column_sum (reduce.cpp:32-88): the column's float sum plus the exact 128-bit integer sum,
 * per range then merged in ascending range order — the identifier check against n(n+1)/2.
 * SSTAT_FLAG_REFEXACT (always for binary32): each range summed sequentially, bit-identical
 * float_sum.  Column out of range: SSTAT_ERR_INVALID (std::out_of_range). */
int sstat_cuda_column_sum(sstat_cuda_ctx* ctx, const sstat_cuda_source* src, uint32_t p, uint32_t column,
                          const uint64_t* range_start, const uint64_t* range_count, uint64_t n_ranges,
                          uint32_t precision, uint32_t flags, sstat_column_sum_result* out, sstat_cuda_error* err);

/* Centered co-moments over the plan (accumulate_comoments + merge_comoments,
 * suffstats.cpp:107-159): n, mean[p] and M2 = sum (x - mean)(x - mean)^T packed, per range
 * from the shifted single-pass moments (c = the range's first row), merged in ascending
 * range order with the pairwise update. */
int sstat_cuda_comoments(sstat_cuda_ctx* ctx, const sstat_cuda_source* src, uint32_t p, const uint64_t* range_start,
                         const uint64_t* range_count, uint64_t n_ranges, uint32_t flags, uint64_t* n_out,
                         double* mean_out, double* m2_out, sstat_cuda_error* err);

/* ---- host helpers (no device work) ---- */

/* The range fold over gathered per-rank buffers (host memory), the same code the device
 * runs after the all-gather: rank q's buffer starts at buf + q*rank_stride with a
 * 4-double header ({lowest failing range, first non-finite row*p+col, status, 0}), then its ranges [floor(qR/W), floor((q+1)R/W)) of p + p(p+1)/2
 * doubles each.  flags & SSTAT_FLAG_REFEXACT (or Binary32Diagnostic): the reference's
 * ascending fold from +0.0; otherwise the 32-lane fast fold of the default mode.
 * out receives p + p(p+1)/2 doubles. */
int sstat_fold_ranges_host(const double* buf, uint64_t rank_stride, uint64_t n_ranges, int world, uint32_t p,
                           uint32_t precision, uint32_t flags, double* out);

/* plan_partitions: returns the range count (0 on invalid input, like the reference's
 * invalid_argument); fills starts/counts when non-NULL. */
uint64_t sstat_plan_partitions(uint64_t n_rows, uint64_t chunk_rows, uint64_t* starts, uint64_t* counts);

/* merge_suffstats: a <- a + b elementwise (binary32 mode rounds each add through float). */
int sstat_merge(uint32_t p, uint32_t precision, uint64_t* n_a, double* sums_a, double* cross_a, uint64_t n_b,
                const double* sums_b, const double* cross_b);

/* ---- measurement-side generator (bit-identical to oracle/sstat_oracle.c) ---- */
#define SSTAT_GEN_MIXED 0u    /* n_int integer columns rand_between(1,100), rest Gaussian */
#define SSTAT_GEN_ID_GAUSS 1u /* column 0 = 1-based row number, rest Gaussian            */
#define SSTAT_GEN_GAUSS 2u    /* all Gaussian                                            */
int sstat_cuda_generate(sstat_cuda_ctx* ctx, double* dst_device, uint32_t kind, uint64_t seed, double mu,
                        uint32_t n_int, uint64_t first_row, uint64_t n_rows, uint32_t p);

#ifdef __cplusplus
}
#endif
#endif /* SSTAT_CUDA_H */
