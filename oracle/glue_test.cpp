// glue_test.cpp — TEST INFRASTRUCTURE: drives the reference's own library through
// integration/sstat_cuda_glue.hpp on a GPU, the way a maintainer of the reference would
// use it.  Built by `make -C oracle glue` against the reference objects in oracle/_ref
// (compiled from /root/reference/proj/src) and libsstat_b200.so; run by
// tests/test_gpu_glue.py.  Exit code 0 = every check passed.
//
// Checks (reference anchors under /root/reference/proj):
//   1. pipeline stage 6 (tools/sstat_main.cpp:509-534): binary-path dataset_suffstats
//      equals the sequential CSV-path result bit-exactly (operator==) — here the GPU
//      pass in reference-order mode against the reference's own CPU pass;
//   2. the fast GPU pass within the Cauchy-Schwarz tolerance, and analyze / run_pca
//      (src/analysis.cpp:108-137, src/pca.cpp:114-154) on it within 1e-12 / 1e-10;
//   3. the GPU as run_reduction's per_chunk (include/sstat/reduce.hpp:70-146);
//   4. error mapping: non-finite -> ReductionError(range, message), bad file -> FormatError,
//      partition mismatch -> std::invalid_argument, accumulate_chunk -> NonFiniteError;
//   5. sidecar round trip (src/suffstats.cpp:190-277) of a GPU result;
//   8. the device-group engine (one process, several devices) through the same glue call.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "sstat/analysis.hpp"
#include "sstat/binfile.hpp"
#include "sstat/datagen.hpp"
#include "sstat/pca.hpp"
#include "sstat/suffstats.hpp"
#include "sstat_cuda_glue.hpp"

using namespace sstat;

static int failures = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        if (!(cond)) {                                                               \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
            ++failures;                                                              \
        }                                                                            \
    } while (0)

static double cs_err(const SuffStats& a, const SuffStats& b) {
    const std::size_t p = a.sums.size();
    double worst = 0;
    for (std::size_t j = 0; j < p; ++j)
        for (std::size_t k = j; k < p; ++k) {
            const double scale = std::sqrt(std::fabs(b.cross.at(j, j) * b.cross.at(k, k)));
            worst = std::max(worst, std::fabs(a.cross.at(j, k) - b.cross.at(j, k)) / (scale > 0 ? scale : 1));
        }
    return worst;
}

static std::filesystem::path write_table1(const std::filesystem::path& dir, std::uint64_t n, std::uint64_t seed,
                                          std::uint64_t poison_row = 0) {
    auto path = dir / ("t1_" + std::to_string(n) + "_" + std::to_string(poison_row) + ".bin");
    BinaryWriter w(path, 11);
    for (std::uint64_t i = 1; i <= n; ++i) {
        auto row = generate_row(GeneratorKind::table1(), seed, i);
        if (poison_row && i - 1 == poison_row) row[9] = std::numeric_limits<double>::infinity();
        w.append_row(row.data(), row.size());
    }
    w.finish();
    return path;
}

int main() {
    const auto dir = std::filesystem::temp_directory_path() / ("sstat_glue_" + std::to_string(::getpid()));
    std::filesystem::create_directories(dir);
    cuda::Engine eng(0);
    const auto schema = DatasetSchema::table1();

    // 1. stage-6 bit-exactness through the GPU (reference-order mode)
    const std::uint64_t n = 200000;
    auto bin = write_table1(dir, n, 5);
    ReductionPlan plan;
    plan.partition = plan_partitions(n, 1 << 14);
    plan.worker_count = 8;
    const SuffStats cpu = dataset_suffstats(bin, schema, plan);
    const SuffStats gpu_exact = cuda::dataset_suffstats(eng, bin, schema, plan, nullptr, SSTAT_FLAG_REFEXACT);
    CHECK(gpu_exact == cpu);

    // 2. fast pass + the reference's own finalisation on it
    ReductionTimings t;
    const SuffStats gpu = cuda::dataset_suffstats(eng, bin, schema, plan, &t);
    CHECK(gpu.n == cpu.n);
    CHECK(cs_err(gpu, cpu) <= 1e-12);
    CHECK(t.bytes_read == n * 11 * 8);
    for (std::size_t j : {0u, 1u, 2u, 3u, 10u}) CHECK(gpu.sums[j] == cpu.sums[j]);  // integer columns exact
    const auto a_cpu = analyze(cpu), a_gpu = analyze(gpu);
    double cov_err = 0, corr_err = 0;
    for (std::size_t j = 0; j < a_cpu.covariance.rows(); ++j)
        for (std::size_t k = 0; k < a_cpu.covariance.cols(); ++k) {
            const double s = std::sqrt(a_cpu.covariance(j, j) * a_cpu.covariance(k, k));
            cov_err = std::max(cov_err, std::fabs(a_gpu.covariance(j, k) - a_cpu.covariance(j, k)) / s);
            corr_err = std::max(corr_err, std::fabs((*a_gpu.correlation)(j, k) - (*a_cpu.correlation)(j, k)));
        }
    CHECK(cov_err <= 1e-12);
    CHECK(corr_err <= 1e-12);
    const auto pc = run_pca(cpu, PcaBasis::Correlation), pg = run_pca(gpu, PcaBasis::Correlation);
    double ev_err = 0;
    for (std::size_t i = 0; i < pc.eigenvalues.size(); ++i)
        ev_err = std::max(ev_err, std::fabs(pg.eigenvalues[i] - pc.eigenvalues[i]) / std::fabs(pc.eigenvalues[i]));
    CHECK(ev_err <= 1e-10);

    // 3. GPU as the per_chunk of the reference's run_reduction (its thread pool, its fold)
    auto merge = [](SuffStats a, SuffStats b) { return merge_suffstats(std::move(a), b); };
    const SuffStats via_pool = run_reduction(bin, plan, cuda::per_chunk(eng, schema, PrecisionMode::Binary64,
                                                                        SSTAT_FLAG_REFEXACT),
                                             merge, SuffStats::empty(schema));
    CHECK(via_pool == cpu);

    // 4. error mapping
    auto bad = write_table1(dir, 50000, 5, 40000);
    ReductionPlan bplan;
    bplan.partition = plan_partitions(50000, 4096);
    std::string cpu_msg, gpu_msg;
    std::size_t cpu_range = 0, gpu_range = 1;
    try {
        dataset_suffstats(bad, schema, bplan);
    } catch (const ReductionError& e) {
        cpu_msg = e.what();
        cpu_range = e.range_index();
    }
    try {
        cuda::dataset_suffstats(eng, bad, schema, bplan);
    } catch (const ReductionError& e) {
        gpu_msg = e.what();
        gpu_range = e.range_index();
    }
    CHECK(!cpu_msg.empty() && cpu_msg == gpu_msg);
    CHECK(cpu_range == gpu_range);
    bool threw = false;
    try {
        ReductionPlan wrong;
        wrong.partition = plan_partitions(n - 1, 1 << 14);
        cuda::dataset_suffstats(eng, bin, schema, wrong);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    {
        auto junk = dir / "junk.bin";
        std::ofstream(junk) << "not a dataset at all, definitely not SSTATBIN";
        threw = false;
        try {
            cuda::dataset_suffstats(eng, junk, schema, plan);
        } catch (const FormatError&) {
            threw = true;
        }
        CHECK(threw);
    }
    {
        Chunk c;
        c.start_row = 40;
        c.row_count = 2;
        c.column_count = 2;
        c.values = {1.0, 2.0, 3.0, std::numeric_limits<double>::infinity()};
        threw = false;
        try {
            cuda::accumulate_chunk(eng, c, DatasetSchema::generic(2));
        } catch (const NonFiniteError& e) {
            threw = e.row() == 41 && e.column() == 1;
        }
        CHECK(threw);
    }

    // 6. column_sum through the glue (reduce.cpp:32-88): identifier column of Table1
    {
        const auto cs_cpu = column_sum(bin, 0, plan);
        const auto cs_gpu = cuda::column_sum(eng, bin, 0, plan, SSTAT_FLAG_REFEXACT);
        CHECK(cs_cpu.exact_sum.has_value() && cs_gpu.exact_sum.has_value());
        CHECK(*cs_gpu.exact_sum == *cs_cpu.exact_sum);
        CHECK(*cs_gpu.exact_sum == static_cast<int128>(n) * (n + 1) / 2);
        CHECK(cs_gpu.float_sum == cs_cpu.float_sum && cs_gpu.float_matches_exact == cs_cpu.float_matches_exact);
        const auto frac_cpu = column_sum(bin, 9, plan);  // J = |tan(d)| is not integral
        const auto frac_gpu = cuda::column_sum(eng, bin, 9, plan);
        CHECK(!frac_gpu.exact_sum && frac_gpu.exact_note == frac_cpu.exact_note);
    }

    // 7. co-moments (run_reduction of accumulate_comoments / merge_comoments) vs the CPU
    {
        auto per = [&](const Chunk& ch) { return accumulate_comoments(ch, schema); };
        auto mrg = [](CoMoments a, CoMoments b) { return merge_comoments(std::move(a), b); };
        const CoMoments cm_cpu = run_reduction(bin, plan, per, mrg, CoMoments::empty(schema));
        const CoMoments cm_gpu = cuda::dataset_comoments(eng, bin, schema, plan);
        CHECK(cm_gpu.n == cm_cpu.n);
        double worst = 0;
        for (std::size_t j = 0; j < 11; ++j)
            for (std::size_t k = j; k < 11; ++k) {
                const double sc = std::sqrt(cm_cpu.m2.at(j, j) * cm_cpu.m2.at(k, k));
                worst = std::max(worst, std::fabs(cm_gpu.m2.at(j, k) - cm_cpu.m2.at(j, k)) / sc);
            }
        CHECK(worst <= 1e-12);
    }

    // 8. the device-group engine (sstat_cuda_init_devices): the reference's single-process
    //    dataset_suffstats(path, schema, plan) over every member — {0} and {0, 0, 0} (three
    //    members on one GPU: per-member file feeders, peer-copy exchange, device fold over three
    //    rank buffers) give the single-device bits, in both modes
    {
        for (const std::vector<int>& devs : {std::vector<int>{0}, std::vector<int>{0, 0, 0}}) {
            cuda::Engine group(devs);
            CHECK(group.device_count() == static_cast<int>(devs.size()));
            const SuffStats g_exact = cuda::dataset_suffstats(group, bin, schema, plan, nullptr, SSTAT_FLAG_REFEXACT);
            CHECK(g_exact == cpu);
            const SuffStats g_fast = cuda::dataset_suffstats(group, bin, schema, plan);
            CHECK(g_fast == gpu);
        }
    }

    // 9. seeded random plans through the unmodified reference: row counts from one row to 300k,
    //    chunks from one row to the whole file, 1-16 workers — reference-order mode equal to the
    //    reference's dataset_suffstats, the fast pass within the Cauchy-Schwarz bar with the
    //    integer columns exact, a three-member group equal to one GPU
    {
        std::mt19937_64 rng(20261019);
        cuda::Engine group(std::vector<int>{0, 0, 0});
        for (int c = 0; c < 8; ++c) {
            const std::uint64_t nr = 1 + rng() % 300000;
            const std::uint64_t chunk = c % 3 == 0 ? 1 + rng() % 64 : 1 + rng() % nr;
            auto f = write_table1(dir, nr, 100 + c);
            ReductionPlan pl;
            pl.partition = plan_partitions(nr, chunk < nr / 20000 ? nr / 20000 + 1 : chunk);
            pl.worker_count = 1 + rng() % 16;
            const SuffStats ref = dataset_suffstats(f, schema, pl);
            CHECK(cuda::dataset_suffstats(eng, f, schema, pl, nullptr, SSTAT_FLAG_REFEXACT) == ref);
            const SuffStats fast = cuda::dataset_suffstats(eng, f, schema, pl);
            CHECK(fast.n == ref.n && cs_err(fast, ref) <= 1e-12);
            for (std::size_t j : {0u, 1u, 2u, 3u, 10u}) CHECK(fast.sums[j] == ref.sums[j]);
            CHECK(cuda::dataset_suffstats(group, f, schema, pl) == fast);
            // column_sum (reference order: the reference's float sum; exact sums either way) and
            // the co-moments on the same plan
            for (std::size_t col : {std::size_t(0), std::size_t(9)}) {
                const auto cs_ref = column_sum(f, col, pl);
                const auto cs_ex = cuda::column_sum(eng, f, col, pl, SSTAT_FLAG_REFEXACT);
                const auto cs_fast = cuda::column_sum(eng, f, col, pl);
                CHECK(cs_ex.float_sum == cs_ref.float_sum && cs_ex.exact_sum == cs_ref.exact_sum);
                CHECK(cs_fast.exact_sum == cs_ref.exact_sum && cs_fast.exact_note == cs_ref.exact_note);
            }
            auto per = [&](const Chunk& ch) { return accumulate_comoments(ch, schema); };
            auto mrg = [](CoMoments a, CoMoments b) { return merge_comoments(std::move(a), b); };
            const CoMoments cm_ref = run_reduction(f, pl, per, mrg, CoMoments::empty(schema));
            const CoMoments cm_gpu = cuda::dataset_comoments(eng, f, schema, pl);
            CHECK(cm_gpu.n == cm_ref.n);
            if (nr > 1)
                for (std::size_t j = 0; j < 11; ++j)
                    for (std::size_t k = j; k < 11; ++k) {
                        const double sc = std::sqrt(cm_ref.m2.at(j, j) * cm_ref.m2.at(k, k));
                        if (sc > 0) CHECK(std::fabs(cm_gpu.m2.at(j, k) - cm_ref.m2.at(j, k)) <= 1e-12 * sc);
                    }
            std::filesystem::remove(f);
        }
    }

    // 5. sidecar round trip of the GPU result
    auto side = dir / "gpu.ssf";
    save_suffstats(gpu, side);
    CHECK(load_suffstats(side) == gpu);

    std::filesystem::remove_all(dir);
    std::printf("glue_test: %s (%d failures); stage-6 exact=%d cs_err=%.2e cov_err=%.2e corr_err=%.2e ev_err=%.2e\n",
                failures ? "FAILED" : "OK", failures, int(gpu_exact == cpu), cs_err(gpu, cpu), cov_err, corr_err,
                ev_err);
    return failures ? 1 : 0;
}
