// sstat_cuda_glue.hpp — the reference-side binding of the B200 engine.
//
// Header-only C++20 glue a maintainer of the reference (arxiv/paper_2604_23826, the
// sstat C++ library under proj/) adds to route its sufficient-statistics pass through
// libsstat_b200.so.  It speaks the reference's own types (SuffStats, Chunk,
// DatasetSchema, ReductionPlan, ReductionTimings) and rethrows the reference's own
// exception classes, so every caller of dataset_suffstats / accumulate_chunk —
// cmd_suffstats, cmd_pipeline stage 6 (tools/sstat_main.cpp:265-298, 509-534) — keeps
// its code and its finalisation (analyze, run_pca, save_suffstats) unchanged.
//
//   reference (proj/)                               glue
//   accumulate_chunk   src/suffstats.cpp:74-84      sstat::cuda::accumulate_chunk
//   dataset_suffstats  src/suffstats.cpp:279-288    sstat::cuda::dataset_suffstats
//   run_reduction's per_chunk callable              sstat::cuda::per_chunk(engine, schema, precision)
//     include/sstat/reduce.hpp:70-146
//   column_sum         src/reduce.cpp:32-88         sstat::cuda::column_sum
//   accumulate_comoments + merge_comoments          sstat::cuda::dataset_comoments
//     src/suffstats.cpp:107-159
//
// Requires the reference headers (include/sstat) and include/sstat_cuda.h; link with
// -lsstat_b200.  See INTEGRATION.md.
#pragma once

#include <cstdint>
#include <filesystem>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sstat/binfile.hpp"
#include "sstat/chunk.hpp"
#include "sstat/errors.hpp"
#include "sstat/reduce.hpp"
#include "sstat/schema.hpp"
#include "sstat/suffstats.hpp"
#include "sstat_cuda.h"

namespace sstat::cuda {

/// Device-side failure with no reference equivalent (CUDA, NCCL, OOM, unsupported).
class DeviceError : public sstat::Error {
public:
    DeviceError(int status, const std::string& what) : Error(what), status_(status) {}
    int status() const { return status_; }

private:
    int status_;
};

namespace detail {
[[noreturn]] inline void rethrow(int st, const sstat_cuda_error& e, bool in_dataset) {
    const std::string msg(e.msg);
    switch (st) {
        case SSTAT_ERR_NONFINITE:
            if (in_dataset) throw sstat::ReductionError(e.range_index, msg);  // reduce.hpp:132-134
            throw sstat::NonFiniteError(e.row, e.col, msg);                   // suffstats.cpp:41-44
        case SSTAT_ERR_SCHEMA:
            if (in_dataset) throw sstat::ReductionError(e.range_index, msg);
            throw sstat::SchemaMismatchError(msg);
        case SSTAT_ERR_INVALID: throw std::invalid_argument(msg);
        case SSTAT_ERR_IO: throw sstat::IoError(msg);
        case SSTAT_ERR_FORMAT: throw sstat::FormatError(msg);
        default: throw DeviceError(st, std::string(sstat_status_string(st)) + ": " + msg);
    }
}

inline SuffStats make_result(const DatasetSchema& schema, PrecisionMode precision, std::uint64_t n,
                             const std::vector<double>& sums, const std::vector<double>& cross) {
    SuffStats ss = SuffStats::empty(schema, precision);
    ss.n = n;
    ss.sums = sums;
    std::copy(cross.begin(), cross.end(), ss.cross.data());
    return ss;
}
}  // namespace detail

/// One libsstat_b200 context: one CUDA device, or a device group — every GPU of the box
/// driven from this one process (sstat_cuda_init_devices; the paper's single host process,
/// PAPER.md:70).  Thread-safe: calls serialise per engine.
class Engine {
public:
    explicit Engine(int device = -1) {
        sstat_cuda_ctx* c = nullptr;
        const int st = sstat_cuda_init(&c, device);
        if (st != SSTAT_OK) throw DeviceError(st, std::string("sstat_cuda_init: ") + sstat_status_string(st));
        ctx_.reset(c);
    }
    /// A device group over `devices`: the plan's ranges are sharded contiguously over them and
    /// folded in the same order — bit-identical to one device.
    explicit Engine(const std::vector<int>& devices) {
        sstat_cuda_ctx* c = nullptr;
        const int st = sstat_cuda_init_devices(&c, static_cast<int>(devices.size()),
                                               devices.empty() ? nullptr : devices.data());
        if (st != SSTAT_OK) throw DeviceError(st, std::string("sstat_cuda_init_devices: ") + sstat_status_string(st));
        ctx_.reset(c);
    }
    /// Every visible GPU as one group (an empty list: sstat_cuda_init_devices(ctx, 0, NULL)).
    static Engine all_devices() { return Engine(std::vector<int>{}); }
    int device_count() const { return sstat_cuda_device_count(get()); }
    sstat_cuda_ctx* get() const { return ctx_.get(); }

    /// Multi-GPU: one process per GPU; `id` from sstat_cuda_nccl_unique_id on rank 0,
    /// broadcast by the host (MPI, a file, a socket ...).
    void attach_communicator(int rank, int world, const void* id, std::size_t id_bytes) {
        const int st = sstat_cuda_comm_init(get(), rank, world, id, id_bytes);
        if (st != SSTAT_OK) throw DeviceError(st, "sstat_cuda_comm_init failed");
    }

private:
    struct Free {
        void operator()(sstat_cuda_ctx* c) const { sstat_cuda_destroy(c); }
    };
    std::unique_ptr<sstat_cuda_ctx, Free> ctx_;
};

/// accumulate_chunk on the GPU (host chunk; the library copies it to HBM).
inline SuffStats accumulate_chunk(Engine& eng, const Chunk& chunk, const DatasetSchema& schema,
                                  PrecisionMode precision = PrecisionMode::Binary64, std::uint32_t flags = 0) {
    schema.validate();
    if (chunk.column_count != schema.column_count())  // check_chunk, suffstats.cpp:34-37
        throw SchemaMismatchError("chunk has " + std::to_string(chunk.column_count) + " columns, schema has " +
                                  std::to_string(schema.column_count()));
    const std::uint32_t p = static_cast<std::uint32_t>(schema.column_count());
    std::vector<double> sums(p), cross(static_cast<std::size_t>(p) * (p + 1) / 2);
    std::uint64_t n = 0;
    sstat_cuda_error err{};
    const int st = sstat_cuda_accumulate(eng.get(), chunk.values.data(), chunk.row_count, p, chunk.start_row,
                                         static_cast<std::uint32_t>(precision), flags, &n, sums.data(), cross.data(),
                                         &err);
    if (st != SSTAT_OK) detail::rethrow(st, err, false);
    return detail::make_result(schema, precision, n, sums, cross);
}

/// A per_chunk callable for the reference's own run_reduction (reduce.hpp:70-146):
///   run_reduction(path, plan, sstat::cuda::per_chunk(eng, schema), merge, identity)
inline auto per_chunk(Engine& eng, const DatasetSchema& schema, PrecisionMode precision = PrecisionMode::Binary64,
                      std::uint32_t flags = 0) {
    return [&eng, schema, precision, flags](const Chunk& chunk) {
        return accumulate_chunk(eng, chunk, schema, precision, flags);
    };
}

inline void fill_timings(ReductionTimings* timings, const sstat_cuda_timings& t) {
    if (!timings) return;
    timings->read_seconds = t.h2d_seconds;
    timings->work_seconds = t.kernel_seconds + t.fold_seconds;
    timings->bytes_read = t.bytes_read;
}

/// dataset_suffstats on the GPU: the SSTATBIN file is streamed through pinned staging
/// buffers into HBM; ranges and the ascending range fold follow the plan.
inline SuffStats dataset_suffstats(Engine& eng, const std::filesystem::path& dataset, const DatasetSchema& schema,
                                   const ReductionPlan& plan, ReductionTimings* timings = nullptr,
                                   std::uint32_t flags = 0) {
    if (plan.worker_count < 1) throw std::invalid_argument("run_reduction: worker_count must be >= 1");
    schema.validate();
    const std::uint32_t p = static_cast<std::uint32_t>(schema.column_count());
    std::vector<std::uint64_t> starts, counts;
    for (const auto& r : plan.partition.ranges) {
        starts.push_back(r.start_row);
        counts.push_back(r.row_count);
    }
    const std::string path = dataset.string();
    sstat_cuda_source src{};
    src.kind = SSTAT_SRC_FILE;
    src.path = path.c_str();
    std::vector<double> sums(p), cross(static_cast<std::size_t>(p) * (p + 1) / 2);
    std::uint64_t n = 0;
    sstat_cuda_timings t{};
    sstat_cuda_error err{};
    const int st = sstat_cuda_dataset(eng.get(), &src, p, starts.data(), counts.data(), starts.size(),
                                      static_cast<std::uint32_t>(plan.precision), flags, &n, sums.data(), cross.data(),
                                      timings ? &t : nullptr, &err);
    if (st != SSTAT_OK) detail::rethrow(st, err, true);
    fill_timings(timings, t);
    return detail::make_result(schema, plan.precision, n, sums, cross);
}

/// dataset_suffstats over rows already in memory: `rows` is a host pointer (pinned
/// memory is DMA'd directly) or a device pointer to this rank's rows, starting at
/// absolute row `first_row`.
inline SuffStats dataset_suffstats(Engine& eng, const double* rows, std::uint64_t first_row, std::uint64_t n_rows,
                                   bool on_device, const DatasetSchema& schema, const ReductionPlan& plan,
                                   ReductionTimings* timings = nullptr, std::uint32_t flags = 0) {
    schema.validate();
    const std::uint32_t p = static_cast<std::uint32_t>(schema.column_count());
    std::vector<std::uint64_t> starts, counts;
    for (const auto& r : plan.partition.ranges) {
        starts.push_back(r.start_row);
        counts.push_back(r.row_count);
    }
    sstat_cuda_source src{};
    src.kind = on_device ? SSTAT_SRC_DEVICE : SSTAT_SRC_HOST;
    src.ptr = rows;
    src.first_row = first_row;
    src.n_rows = n_rows;
    std::vector<double> sums(p), cross(static_cast<std::size_t>(p) * (p + 1) / 2);
    std::uint64_t n = 0;
    sstat_cuda_timings t{};
    sstat_cuda_error err{};
    const int st = sstat_cuda_dataset(eng.get(), &src, p, starts.data(), counts.data(), starts.size(),
                                      static_cast<std::uint32_t>(plan.precision), flags, &n, sums.data(), cross.data(),
                                      timings ? &t : nullptr, &err);
    if (st != SSTAT_OK) detail::rethrow(st, err, true);
    fill_timings(timings, t);
    return detail::make_result(schema, plan.precision, n, sums, cross);
}

namespace detail {
inline std::vector<std::uint64_t> starts_of(const ReductionPlan& plan) {
    std::vector<std::uint64_t> v;
    for (const auto& r : plan.partition.ranges) v.push_back(r.start_row);
    return v;
}
inline std::vector<std::uint64_t> counts_of(const ReductionPlan& plan) {
    std::vector<std::uint64_t> v;
    for (const auto& r : plan.partition.ranges) v.push_back(r.row_count);
    return v;
}
}  // namespace detail

/// column_sum over an SSTATBIN file (reduce.cpp:32-88), same result type.
inline ColumnSumResult column_sum(Engine& eng, const std::filesystem::path& dataset, std::size_t column,
                                  const ReductionPlan& plan, std::uint32_t flags = 0) {
    const std::string path = dataset.string();
    // the column count comes from the file header (binfile.hpp:17-29)
    BinaryReader probe(dataset);
    if (column >= probe.columns())
        throw std::out_of_range("column_sum: column " + std::to_string(column) + " out of range, dataset has " +
                                std::to_string(probe.columns()) + " columns");
    const auto starts = detail::starts_of(plan), counts = detail::counts_of(plan);
    sstat_cuda_source src{};
    src.kind = SSTAT_SRC_FILE;
    src.path = path.c_str();
    sstat_column_sum_result r{};
    sstat_cuda_error err{};
    const int st = sstat_cuda_column_sum(eng.get(), &src, probe.columns(), static_cast<std::uint32_t>(column),
                                         starts.data(), counts.data(), starts.size(),
                                         static_cast<std::uint32_t>(plan.precision), flags, &r, &err);
    if (st != SSTAT_OK) detail::rethrow(st, err, true);
    ColumnSumResult out;
    out.float_sum = r.float_sum;
    if (r.exact_ok) {
        out.exact_sum = static_cast<int128>((static_cast<unsigned __int128>(static_cast<std::uint64_t>(r.exact_hi)) << 64) |
                                            r.exact_lo);
        out.float_matches_exact = r.float_matches_exact != 0;
    } else {
        out.exact_note = "non-integral value at row " + std::to_string(r.note_row) + "; exact sum unavailable";
    }
    return out;
}

/// run_reduction(accumulate_comoments, merge_comoments) over an SSTATBIN file.
inline CoMoments dataset_comoments(Engine& eng, const std::filesystem::path& dataset, const DatasetSchema& schema,
                                   const ReductionPlan& plan) {
    schema.validate();
    const std::uint32_t p = static_cast<std::uint32_t>(schema.column_count());
    const std::string path = dataset.string();
    const auto starts = detail::starts_of(plan), counts = detail::counts_of(plan);
    sstat_cuda_source src{};
    src.kind = SSTAT_SRC_FILE;
    src.path = path.c_str();
    CoMoments cm = CoMoments::empty(schema);
    std::uint64_t n = 0;
    sstat_cuda_error err{};
    const int st = sstat_cuda_comoments(eng.get(), &src, p, starts.data(), counts.data(), starts.size(), 0, &n,
                                        cm.mean.data(), cm.m2.data(), &err);
    if (st != SSTAT_OK) detail::rethrow(st, err, true);
    cm.n = n;
    return cm;
}

}  // namespace sstat::cuda
