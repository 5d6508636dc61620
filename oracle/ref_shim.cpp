// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/sstat_oracle.c header).  oracle/Makefile
// compiles /root/reference/proj/src/*.cpp where they lie (no copies) together with
// this file into oracle/_ref/libsstat_ref.so.  Python tests and bench.py's
// reference arm load it with ctypes to:
//   * pin the C restatement (oracle/sstat_oracle.c) bit-for-bit against the
//     reference's own accumulate_chunk / merge_suffstats / dataset_suffstats;
//   * time the reference's own dataset_suffstats on the host cores (bench.py
//     --impl reference);
//   * run the reference's unchanged host finalisation (analyze, run_pca) on a
//     SuffStats produced by either engine, for the cov/corr/eigenvalue parity.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sstat/analysis.hpp"
#include "sstat/binfile.hpp"
#include "sstat/datagen.hpp"
#include "sstat/errors.hpp"
#include "sstat/pca.hpp"
#include "sstat/reduce.hpp"
#include "sstat/suffstats.hpp"

using namespace sstat;

namespace {

enum : int {
    REF_OK = 0,
    REF_NONFINITE = 1,
    REF_SCHEMA = 2,
    REF_INVALID = 3,
    REF_REDUCTION = 4,
    REF_IO = 5,
    REF_FORMAT = 6,
    REF_CANCELLATION = 7,
    REF_OTHER = 9,
};

struct RefError {
    std::uint64_t row;
    std::uint32_t col;
    std::uint64_t range_index;
    char msg[256];
};

void set_msg(RefError* err, const std::string& s) {
    if (!err) return;
    std::strncpy(err->msg, s.c_str(), sizeof err->msg - 1);
    err->msg[sizeof err->msg - 1] = 0;
}

DatasetSchema schema_of(std::uint32_t p, std::uint32_t n_ids, const std::uint32_t* ids) {
    DatasetSchema s = DatasetSchema::generic(p, false);
    for (std::uint32_t i = 0; i < n_ids; ++i) s.identifier_columns.push_back(ids[i]);
    return s;
}

Chunk chunk_of(const double* values, std::uint64_t rows, std::uint32_t p, std::uint64_t start_row) {
    Chunk c;
    c.start_row = start_row;
    c.row_count = rows;
    c.column_count = p;
    c.values.assign(values, values + rows * p);
    return c;
}

void export_stats(const SuffStats& ss, std::uint64_t* n, double* sums, double* cross) {
    *n = ss.n;
    std::memcpy(sums, ss.sums.data(), ss.sums.size() * sizeof(double));
    std::memcpy(cross, ss.cross.data(), ss.cross.packed_size() * sizeof(double));
}

SuffStats import_stats(std::uint32_t p, std::uint32_t n_ids, const std::uint32_t* ids, std::uint32_t precision,
                       std::uint64_t n, const double* sums, const double* cross) {
    SuffStats ss = SuffStats::empty(schema_of(p, n_ids, ids), static_cast<PrecisionMode>(precision));
    ss.n = n;
    std::memcpy(ss.sums.data(), sums, p * sizeof(double));
    std::memcpy(ss.cross.data(), cross, ss.cross.packed_size() * sizeof(double));
    return ss;
}

template <class F>
int guarded(RefError* err, F&& f) {
    try {
        f();
        return REF_OK;
    } catch (const NonFiniteError& e) {
        if (err) {
            err->row = e.row();
            err->col = static_cast<std::uint32_t>(e.column());
        }
        set_msg(err, e.what());
        return REF_NONFINITE;
    } catch (const ReductionError& e) {
        if (err) err->range_index = e.range_index();
        set_msg(err, e.what());
        return REF_REDUCTION;
    } catch (const SchemaMismatchError& e) {
        set_msg(err, e.what());
        return REF_SCHEMA;
    } catch (const CancellationError& e) {
        set_msg(err, e.what());
        return REF_CANCELLATION;
    } catch (const IoError& e) {
        set_msg(err, e.what());
        return REF_IO;
    } catch (const FormatError& e) {
        set_msg(err, e.what());
        return REF_FORMAT;
    } catch (const std::invalid_argument& e) {
        set_msg(err, e.what());
        return REF_INVALID;
    } catch (const std::out_of_range& e) {
        set_msg(err, e.what());
        return REF_INVALID;
    } catch (const std::exception& e) {
        set_msg(err, e.what());
        return REF_OTHER;
    }
}

} // namespace

extern "C" {

// accumulate_chunk (suffstats.cpp:74-84) on one in-memory chunk.
int ref_accumulate_chunk(const double* values, std::uint64_t rows, std::uint32_t p, std::uint64_t start_row,
                         std::uint32_t precision, std::uint64_t* n, double* sums, double* cross, RefError* err) {
    return guarded(err, [&] {
        auto ss = accumulate_chunk(chunk_of(values, rows, p, start_row), DatasetSchema::generic(p, false),
                                   static_cast<PrecisionMode>(precision));
        export_stats(ss, n, sums, cross);
    });
}

// merge_suffstats (suffstats.cpp:86-105): a <- merge(a, b).
int ref_merge(std::uint32_t p, std::uint32_t precision, std::uint64_t* n_a, double* sums_a, double* cross_a,
              std::uint64_t n_b, const double* sums_b, const double* cross_b) {
    return guarded(nullptr, [&] {
        auto a = import_stats(p, 0, nullptr, precision, *n_a, sums_a, cross_a);
        auto b = import_stats(p, 0, nullptr, precision, n_b, sums_b, cross_b);
        export_stats(merge_suffstats(std::move(a), b), n_a, sums_a, cross_a);
    });
}

// BinaryWriter (binfile.cpp:49-120): writes an SSTATBIN file of rows x p values.
int ref_write_binary(const char* path, const double* values, std::uint64_t rows, std::uint32_t p,
                     int with_checksum, RefError* err) {
    return guarded(err, [&] {
        BinaryWriter w(path, p, with_checksum != 0);
        const std::uint64_t block = 1u << 16;
        for (std::uint64_t s = 0; s < rows; s += block) {
            Chunk c = chunk_of(values + s * p, std::min<std::uint64_t>(block, rows - s), p, s);
            w.append(c);
        }
        w.finish();
    });
}

// dataset_suffstats (suffstats.cpp:279-288) over an SSTATBIN file with
// plan_partitions(n, chunk_rows) (reduce.cpp:8-16) and `workers` threads.
int ref_dataset_suffstats(const char* path, std::uint32_t p, std::uint64_t chunk_rows, std::uint32_t workers,
                          std::uint32_t precision, std::uint64_t* n, double* sums, double* cross,
                          double* read_seconds, double* work_seconds, RefError* err) {
    return guarded(err, [&] {
        BinaryReader probe(path);
        ReductionPlan plan;
        plan.partition = plan_partitions(probe.rows(), chunk_rows);
        plan.worker_count = workers;
        plan.precision = static_cast<PrecisionMode>(precision);
        ReductionTimings t;
        auto ss = dataset_suffstats(path, DatasetSchema::generic(p, false), plan, &t);
        export_stats(ss, n, sums, cross);
        if (read_seconds) *read_seconds = t.read_seconds;
        if (work_seconds) *work_seconds = t.work_seconds;
    });
}

// dataset_suffstats with an explicit partition (any ranges covering [0, n)).
int ref_dataset_suffstats_ranges(const char* path, std::uint32_t p, const std::uint64_t* starts,
                                 const std::uint64_t* counts, std::uint64_t n_ranges, std::uint32_t workers,
                                 std::uint64_t* n, double* sums, double* cross, RefError* err) {
    return guarded(err, [&] {
        ReductionPlan plan;
        for (std::uint64_t i = 0; i < n_ranges; ++i) plan.partition.ranges.push_back({starts[i], counts[i]});
        plan.worker_count = workers;
        auto ss = dataset_suffstats(path, DatasetSchema::generic(p, false), plan);
        export_stats(ss, n, sums, cross);
    });
}

// plan_partitions (reduce.cpp:8-16).
std::uint64_t ref_plan_partitions(std::uint64_t n_rows, std::uint64_t chunk_rows, std::uint64_t* starts,
                                  std::uint64_t* counts, RefError* err) {
    std::uint64_t count = 0;
    int st = guarded(err, [&] {
        auto part = plan_partitions(n_rows, chunk_rows);
        count = part.ranges.size();
        if (starts && counts)
            for (std::size_t i = 0; i < part.ranges.size(); ++i) {
                starts[i] = part.ranges[i].start_row;
                counts[i] = part.ranges[i].row_count;
            }
    });
    return st == REF_OK ? count : 0;
}

// generate_row (datagen.cpp:36-49): Table1 (kind 0, 11 columns) or IidUniform (kind 1).
void ref_generate_row(int kind, std::uint64_t iid_columns, double lo, double hi, std::uint64_t seed,
                      std::uint64_t index, double* out) {
    GeneratorKind k = kind == 0 ? GeneratorKind::table1() : GeneratorKind::iid_uniform(iid_columns, lo, hi);
    auto row = generate_row(k, seed, index);
    std::memcpy(out, row.data(), row.size() * sizeof(double));
}

// column_sum (reduce.cpp:32-88) over an SSTATBIN file.
int ref_column_sum(const char* path, std::uint32_t column, std::uint64_t chunk_rows, std::uint32_t workers,
                   std::uint32_t precision, double* float_sum, int* exact_ok, std::int64_t* exact_hi,
                   std::uint64_t* exact_lo, int* float_matches, char* note, RefError* err) {
    return guarded(err, [&] {
        BinaryReader probe(path);
        ReductionPlan plan;
        plan.partition = plan_partitions(probe.rows(), chunk_rows);
        plan.worker_count = workers;
        plan.precision = static_cast<PrecisionMode>(precision);
        auto r = column_sum(path, column, plan);
        *float_sum = r.float_sum;
        *exact_ok = r.exact_sum.has_value();
        *float_matches = r.float_matches_exact;
        if (r.exact_sum) {
            *exact_hi = static_cast<std::int64_t>(*r.exact_sum >> 64);
            *exact_lo = static_cast<std::uint64_t>(*r.exact_sum);
        }
        if (note) {
            note[0] = 0;
            if (r.exact_note) std::strncpy(note, r.exact_note->c_str(), 255);
        }
    });
}

// accumulate_comoments / merge_comoments (suffstats.cpp:107-159).
int ref_accumulate_comoments(const double* values, std::uint64_t rows, std::uint32_t p, std::uint64_t start_row,
                             std::uint64_t* n, double* mean, double* m2, RefError* err) {
    return guarded(err, [&] {
        auto cm = accumulate_comoments(chunk_of(values, rows, p, start_row), DatasetSchema::generic(p, false));
        *n = cm.n;
        std::memcpy(mean, cm.mean.data(), p * sizeof(double));
        std::memcpy(m2, cm.m2.data(), cm.m2.packed_size() * sizeof(double));
    });
}

int ref_merge_comoments(std::uint32_t p, std::uint64_t* n_a, double* mean_a, double* m2_a, std::uint64_t n_b,
                        const double* mean_b, const double* m2_b) {
    return guarded(nullptr, [&] {
        CoMoments a = CoMoments::empty(DatasetSchema::generic(p, false));
        CoMoments b = CoMoments::empty(DatasetSchema::generic(p, false));
        a.n = *n_a;
        b.n = n_b;
        std::memcpy(a.mean.data(), mean_a, p * sizeof(double));
        std::memcpy(b.mean.data(), mean_b, p * sizeof(double));
        std::memcpy(a.m2.data(), m2_a, a.m2.packed_size() * sizeof(double));
        std::memcpy(b.m2.data(), m2_b, b.m2.packed_size() * sizeof(double));
        auto m = merge_comoments(std::move(a), b);
        *n_a = m.n;
        std::memcpy(mean_a, m.mean.data(), p * sizeof(double));
        std::memcpy(m2_a, m.m2.data(), m.m2.packed_size() * sizeof(double));
    });
}

// analyze (analysis.cpp:108-137): identifiers excluded by default; outputs the kept
// column count q, means[q], cov[q*q], corr[q*q] (corr_ok=0 when undefined).
int ref_analyze(std::uint32_t p, std::uint32_t n_ids, const std::uint32_t* ids, std::uint64_t n,
                const double* sums, const double* cross, int ddof, std::uint32_t* q, double* mean, double* cov,
                double* corr, int* corr_ok, RefError* err) {
    return guarded(err, [&] {
        auto ss = import_stats(p, n_ids, ids, 0, n, sums, cross);
        AnalysisOptions opt;
        opt.ddof = ddof;
        auto r = analyze(ss, opt);
        const std::size_t m = r.included_columns.size();
        *q = static_cast<std::uint32_t>(m);
        std::memcpy(mean, r.mean.data(), m * sizeof(double));
        std::memcpy(cov, r.covariance.data(), m * m * sizeof(double));
        *corr_ok = r.correlation.has_value();
        if (r.correlation) std::memcpy(corr, r.correlation->data(), m * m * sizeof(double));
    });
}

// run_pca (pca.cpp:114-154), basis 0 = covariance, 1 = correlation; eigenvalues descending.
int ref_run_pca(std::uint32_t p, std::uint32_t n_ids, const std::uint32_t* ids, std::uint64_t n,
                const double* sums, const double* cross, int basis, std::uint32_t* q, double* eigenvalues,
                RefError* err) {
    return guarded(err, [&] {
        auto ss = import_stats(p, n_ids, ids, 0, n, sums, cross);
        auto r = run_pca(ss, basis == 0 ? PcaBasis::Covariance : PcaBasis::Correlation);
        *q = static_cast<std::uint32_t>(r.eigenvalues.size());
        std::memcpy(eigenvalues, r.eigenvalues.data(), r.eigenvalues.size() * sizeof(double));
    });
}

// save_suffstats / load_suffstats (suffstats.cpp:190-277) — sidecar round trip.
int ref_save_suffstats(const char* path, std::uint32_t p, std::uint32_t n_ids, const std::uint32_t* ids,
                       std::uint32_t precision, std::uint64_t n, const double* sums, const double* cross,
                       RefError* err) {
    return guarded(err, [&] { save_suffstats(import_stats(p, n_ids, ids, precision, n, sums, cross), path); });
}

} // extern "C"
