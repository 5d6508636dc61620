// engine.cu — host runtime and C ABI of the B200 sufficient-statistics engine.
//
// Replaces the reference's parallel reduction engine for the sufficient-statistics
// path (reference include/sstat/reduce.hpp:70-146 run_reduction, src/suffstats.cpp:279-288
// dataset_suffstats):  the std::thread pool pulling ranges becomes HBM-resident (or
// streamed) row shards accumulated tile by tile by K1/K2, the per-range partial slots
// become a device buffer of per-range partials (K3a), and the ascending range fold
// becomes K3b — run after the exchange when rows are sharded over GPUs: an NCCL all-gather
// between processes (one per GPU), or, for a device group driven by one process, K3a writing
// each member's partials straight into member 0's gather buffer.  Results are a fixed
// function of (data, plan): bit-identical for any GPU count, grid size or staging layout.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cxxabi.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/sstat_cuda.h"
#include "common.cuh"
#include "fold.cuh"
#include "kernels.h"

using namespace sstat_b200;

namespace {

constexpr uint64_t kNone = ~0ull;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    uint64_t gen = 0;  // bumped by every (re)allocation: a new allocation may reuse the old address
    cudaError_t reserve(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        ++gen;
        const size_t want = std::max<size_t>(n, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        ++gen;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(n, 256);
        cudaError_t e = cudaMallocHost(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// NVTX ranges around each ABI call and its phases (host-side enqueue timeline for nsys / ncu
// range replay; header-only NVTX3, no cost without an attached tool).
struct Trace {
    explicit Trace(const char* name) { nvtxRangePushA(name); }
    ~Trace() { nvtxRangePop(); }
    Trace(const Trace&) = delete;
    Trace& operator=(const Trace&) = delete;
};

// Host feeder threads (the loader half of reference src/binfile.cpp:140-161 read_rows): a
// staging slot is filled by parallel page-cache reads / memcpys of disjoint row blocks, so
// the pageable and file sources run at the H2D link rate instead of one core's copy rate.
// The calling thread takes tasks too; run() returns when every task is done and rethrows
// the first task exception.
class FillPool {
public:
    explicit FillPool(unsigned threads) {
        for (unsigned i = 1; i < threads; ++i) th_.emplace_back([this] { loop(); });
    }
    ~FillPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    unsigned size() const { return (unsigned)th_.size() + 1; }
    void run(size_t n, const std::function<void(size_t)>& fn) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            next_ = 0;
            n_ = n;
            pending_ = n;
            err_ = nullptr;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
        fn_ = nullptr;
        if (err_) std::rethrow_exception(err_);
    }

private:
    void work() {
        for (;;) {
            size_t i;
            const std::function<void(size_t)>* fn;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (!fn_ || next_ >= n_) return;
                i = next_++;
                fn = fn_;
            }
            std::exception_ptr e;
            try {
                (*fn)(i);
            } catch (...) {
                e = std::current_exception();
            }
            std::lock_guard<std::mutex> lk(mu_);
            if (e && !err_) err_ = e;
            if (--pending_ == 0) done_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || (gen_ != seen && fn_ && next_ < n_); });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    const std::function<void(size_t)>* fn_ = nullptr;
    size_t next_ = 0, n_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
    std::exception_ptr err_;
};

unsigned default_host_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return std::max(1u, std::min(16u, hw ? hw : 1u));
}

}  // namespace

struct sstat_cuda_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t own = nullptr, stream = nullptr, copy = nullptr;
    // K2's idle-slot launch runs on this context's own side stream (TileJob::side)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::mutex mu;
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    DevBuf d_meta, d_tiles, d_rank, d_gather, d_shift, d_result, d_flags, d_counts, d_aux, d_claim, d_pieces;
    HostBuf h_meta, h_result, h_shift, h_flags, h_counts, h_pieces;
    uint32_t n_slots = 4;
    uint64_t slot_bytes = 256ull << 20;  // requested slot size
    uint64_t slot_cap = 0;               // allocated: >= slot_bytes, grown to the largest unsplittable unit
    std::vector<DevBuf> slots;
    std::vector<HostBuf> bounce;
    std::vector<cudaEvent_t> ev_copied, ev_free;
    // ev[0..4]: K1 / fold / exchange brackets; ev[5], ev[6]: the H2D span of a streamed call;
    // ev[7]: a group member's end of local work, joined by member 0's stream
    cudaEvent_t ev[8] = {};
    bool h2d_timed = false;  // ev[5] / ev[6] recorded by this call's stream_chunks
    // per-call state kept across calls: the last uploaded plan (skip identical re-uploads)
    // and whether the rank header / range flags are still in their reset state
    std::vector<uint64_t> meta_last;
    uint64_t meta_gen = 0;  // d_meta.gen holding meta_last (0 = none)
    bool flags_clean = false;
    uint64_t clean_rank = 0;   // DevBuf::gen of d_rank / d_flags when last reset
    uint64_t clean_flags = 0;
    uint64_t clean_len = 0;
    // host feeder for pageable / file sources (created on first use)
    unsigned host_threads = 0;  // 0 = default_host_threads()
    std::unique_ptr<FillPool> pool;
    // CUDA graph of the last device-resident K1 pass (gather, K1, K3a, K3b, read-back), replayed
    // while every input of the captured launches is unchanged (graph_key)
    cudaStream_t cap = nullptr;  // private capture stream (the caller's stream is never captured)
    cudaGraphExec_t graph = nullptr;
    std::vector<uint64_t> graph_key;
    const void* last_kernel = nullptr;  // the accumulate kernel the last pass launched (timings)
    // ---- device group (sstat_cuda_init_devices): one process driving G devices ----
    // members[g] is a full per-device context with rank g of world G; the group context itself
    // owns no device state.  Exchange: NCCL (ncclCommInitAll over distinct devices) or peer
    // copies into member 0 (`peer`: a device listed twice, or SSTAT_PEER_EXCHANGE=1).
    std::vector<sstat_cuda_ctx*> members;
    bool peer = false;   // exchange by peer copies into member 0
    bool fused = false;  // exchange fused into the local phase: members write member 0's gather buffer
    double* ext_rank = nullptr;  // (member of a fused group, during a call) its slot of member 0's gather buffer
    std::unique_ptr<FillPool> gpool;  // one host thread per member for the local phase
    bool is_group() const { return !members.empty(); }
};

namespace {

// ---- error plumbing ----
struct Fail {
    int status;
    std::string msg;
    uint64_t row = 0, range = 0;
    uint32_t col = 0;
};

int report(sstat_cuda_error* err, const Fail& f) {
    if (err) {
        err->status = (uint32_t)f.status;
        err->row = f.row;
        err->col = f.col;
        err->range_index = f.range;
        std::snprintf(err->msg, sizeof err->msg, "%s", f.msg.c_str());
    }
    return f.status;
}

Fail cuda_fail(cudaError_t e, const char* what) {
    Fail f;
    f.status = (e == cudaErrorMemoryAllocation) ? SSTAT_ERR_OOM : SSTAT_ERR_CUDA;
    f.msg = std::string(what) + ": " + cudaGetErrorString(e);
    return f;
}

#define CUDA_TRY(expr)                                       \
    do {                                                     \
        cudaError_t e_ = (expr);                             \
        if (e_ != cudaSuccess) throw cuda_fail(e_, #expr);   \
    } while (0)

// ---- SSTATBIN (reference include/sstat/binfile.hpp:17-29): 64-byte header, payload at 64 ----
struct BinFile {
    int fd = -1;
    uint64_t rows = 0;
    uint32_t cols = 0;
    ~BinFile() {
        if (fd >= 0) ::close(fd);
    }
};

uint64_t le64(const unsigned char* b) {
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
    return v;
}
uint32_t le32(const unsigned char* b) { return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24); }

// Header and size validation, with the reference's error classes (binfile.cpp:24-47,122-138).
void open_bin(const char* path, BinFile& f) {
    Fail io{SSTAT_ERR_IO, ""}, fmt{SSTAT_ERR_FORMAT, ""};
    struct stat st;
    if (!path || ::stat(path, &st) != 0) {
        io.msg = std::string("no such file: ") + (path ? path : "(null)");
        throw io;
    }
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0) {
        io.msg = std::string("cannot open ") + path;
        throw io;
    }
    unsigned char h[64];
    if (::pread(f.fd, h, 64, 0) != 64) {
        fmt.msg = std::string("file too small for header: ") + path;
        throw fmt;
    }
    if (std::memcmp(h, "SSTATBIN", 8) != 0) {
        fmt.msg = "bad magic: not a binary dataset file";
        throw fmt;
    }
    const uint32_t version = le32(h + 8);
    if (version != 1) {
        fmt.msg = "unsupported format version " + std::to_string(version);
        throw fmt;
    }
    f.rows = le64(h + 12);
    f.cols = le32(h + 20);
    const uint64_t checksum = le64(h + 24);
    const uint32_t flags = le32(h + 32);
    if (flags & ~1u) {
        fmt.msg = "unknown header flags";
        throw fmt;
    }
    if (!(flags & 1u) && checksum != 0) {
        fmt.msg = "checksum field set without checksum flag";
        throw fmt;
    }
    for (int i = 36; i < 64; ++i)
        if (h[i] != 0) {
            fmt.msg = "reserved header bytes are not zero";
            throw fmt;
        }
    if (f.cols == 0) {
        fmt.msg = "column count is zero";
        throw fmt;
    }
    const uint64_t expect = 64 + f.rows * (uint64_t)f.cols * 8;
    if ((uint64_t)st.st_size != expect) {
        fmt.msg = std::string("file size mismatch in ") + path + ": header implies " + std::to_string(expect) +
                  " bytes, file has " + std::to_string((uint64_t)st.st_size);
        throw fmt;
    }
}

void read_exact(int fd, void* dst, uint64_t bytes, uint64_t offset) {
    char* d = static_cast<char*>(dst);
    while (bytes) {
        const ssize_t got = ::pread(fd, d, bytes > (1ull << 30) ? (1ull << 30) : bytes, (off_t)offset);
        if (got <= 0) throw Fail{SSTAT_ERR_FORMAT, "truncated read"};
        d += got;
        bytes -= (uint64_t)got;
        offset += (uint64_t)got;
    }
}

// Row source abstraction for host-side staging.
struct HostRows {
    const sstat_cuda_source* src;
    BinFile* file;
    uint32_t p;
    bool pinned;
    const double* host_row(uint64_t row) const {
        return static_cast<const double*>(src->ptr) + (row - src->first_row) * p;
    }
    bool reader() const { return src->kind == SSTAT_SRC_READER; }
    // copy rows [row, row + n) into dst (pageable ptr / file)
    void fill(void* dst, uint64_t row, uint64_t n) const {
        if (file) read_exact(file->fd, dst, n * p * 8, 64 + row * p * 8);
        else std::memcpy(dst, host_row(row), n * p * 8);
    }
    // rows [row, row + n) in host memory: the reader's own pointer, or `scratch` once filled
    const void* get(void* scratch, uint64_t row, uint64_t n) const {
        if (!reader()) {
            fill(scratch, row, n);
            return scratch;
        }
        const void* q = src->read_rows(src->user, row, n, scratch);
        if (!q)
            throw Fail{SSTAT_ERR_IO, "read_rows failed for rows [" + std::to_string(row) + ", " +
                                         std::to_string(row + n) + ")"};
        return q;
    }
    // the same, as row blocks of >= 4 MiB spread over the feeder threads
    void fill_parallel(FillPool& pool, void* dst, uint64_t row, uint64_t n) const {
        const uint64_t row_bytes = (uint64_t)p * 8;
        const uint64_t min_rows = std::max<uint64_t>(1, (4ull << 20) / row_bytes);
        const uint64_t parts = std::max<uint64_t>(1, std::min<uint64_t>(pool.size(), n / min_rows));
        if (parts == 1) return fill(dst, row, n);
        const uint64_t per = (n + parts - 1) / parts;
        pool.run(parts, [&](size_t i) {
            const uint64_t r0 = i * per, r1 = std::min(n, r0 + per);
            if (r0 < r1) fill(static_cast<char*>(dst) + r0 * row_bytes, row + r0, r1 - r0);
        });
    }
};

// Staging ring of n_slots device slots (+ pinned bounce buffers for pageable / file sources).
// Slots are at least the requested slot_bytes and at least `min_bytes`: the largest unit the
// call cannot split (a fast-path tile; reference-order ranges are split into pieces instead).
void ensure_slots(sstat_cuda_ctx* c, bool need_bounce, uint64_t min_bytes) {
    const uint64_t cap = std::max<uint64_t>(c->slot_bytes, (min_bytes + 127) & ~(uint64_t)127);
    if (c->slots.size() != c->n_slots) {
        for (auto& s : c->slots) s.release();
        for (auto& b : c->bounce) b.release();
        for (auto e : c->ev_copied) cudaEventDestroy(e);
        for (auto e : c->ev_free) cudaEventDestroy(e);
        c->slots.assign(c->n_slots, DevBuf{});
        c->bounce.assign(c->n_slots, HostBuf{});
        c->ev_copied.assign(c->n_slots, nullptr);
        c->ev_free.assign(c->n_slots, nullptr);
        for (uint32_t i = 0; i < c->n_slots; ++i) {
            CUDA_TRY(cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming));
        }
    }
    for (uint32_t i = 0; i < c->n_slots; ++i) {
        CUDA_TRY(c->slots[i].reserve(cap));
        if (need_bounce) CUDA_TRY(c->bounce[i].reserve(cap));
    }
    c->slot_cap = cap;
}

enum class Mode { Dataset, Chunk, Partials, Comoments };

struct Plan {
    Mode mode = Mode::Dataset;
    uint64_t want_r0 = 0, want_r1 = 0;  // Mode::Partials: ranges to accumulate
    double* partials_host = nullptr;    // Mode::Partials: [(want_r1 - want_r0) * E]
    uint32_t p, precision, flags;
    uint64_t R, r0, r1, L, lmax, E, n_tiles, total, span_begin, span_end;
    const uint64_t* starts;
    const uint64_t* counts;
    std::vector<uint64_t> tile_row, tile_rows;  // host view of local tiles (streaming)
};

// K1's tile height for a plan: kBigTileRows when the whole plan (every rank's ranges) has at
// least kBigTileMin such tiles (C2: 6104) and p > 8 (p <= 8 measured 3 % slower with them);
// kTileRows when it has at least kFillTiles of those; else — a plan too small to fill two waves
// of K1's CTA slots with 4096-row tiles (C1: 245 tiles for 592 slots) — the shortest height (a
// multiple of 32, at least kMinTileRows) whose tiles fit as many whole waves as 4096-row tiles
// would start: one (C1: 1696 rows, 590 tiles) or two (2.5e6 x 16: 2144 rows, 1168 tiles).
// Measured with L2 flushed before every call (profiles/r02_small_plans_cold.log): C1 57.5 -> 48.8
// us per call, 2e6 x 16 82 -> 73, 2.5e6 x 16 106 -> 85; the previous rule, powers of two down to
// at least two waves, gave C1 512-row tiles.  A function of the global plan alone: every rank and
// GPU count cuts the same tiles.
uint64_t smallp_tile_rows(const Plan& P) {
    if (const char* env = getenv("SSTAT_K1_TILE_ROWS")) {  // experiment knob: a fixed height (multiple of 32)
        const uint64_t tr = strtoull(env, nullptr, 10);
        if (tr >= 32 && tr <= kBigTileRows && tr % 32 == 0) return tr;
    }
    if (P.p > 8 && P.total / kBigTileRows >= kBigTileMin) return kBigTileRows;
    if (P.total / kTileRows >= kFillTiles) return kTileRows;  // sum of ceil(count / TR) >= total / TR
    auto tiles_of = [&](uint64_t tr) {
        uint64_t t = 0;
        for (uint64_t i = 0; i < P.R; ++i) t += (P.counts[i] + tr - 1) / tr;
        return t;
    };
    // as many whole waves as 4096-row tiles would start (one or two), each as short as they fit; a
    // wave is kWaveSMs x the CTAs per SM of the kernel this width runs (4 up to p = 16, 3 at
    // p = 24-32, 2 at p = 40-64: C1 592 slots, p = 32 444)
    const uint64_t wave = kWaveSMs * smallp_rt_ctas_per_sm(P.p);
    if (tiles_of(kTileRows) > 2 * wave) return kTileRows;
    const uint64_t target = tiles_of(kTileRows) > wave ? 2 * wave : wave;
    if (P.R > target) return kTileRows;  // a tile per range at least
    // tiles_of falls as the height grows: the smallest multiple of 32 in [lo, kTileRows] that fits
    uint64_t lo = std::max<uint64_t>(kMinTileRows, ((P.total + target - 1) / target + 31) / 32 * 32);
    if (lo >= kTileRows) return kTileRows;
    uint64_t hi = kTileRows;  // fits: tiles_of(kTileRows) <= target here
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2 / 32 * 32;
        if (tiles_of(mid) <= target) hi = mid;
        else lo = mid + 32;
    }
    return hi;
}

uint64_t tile_rows_for(const Plan& P) { return P.p > 64 ? widep_tile_rows(P.p) : smallp_tile_rows(P); }

struct Outcome {
    uint64_t bad_lin = kNone;  // lowest first-non-finite linear index over all ranks
    int failed_rank = -1;      // first rank whose header reports a failure (multi-process)
    int failed_status = 0;
};

// Streams units of rows (tiles, or reference-order range pieces) through the staging ring.
// `launch(base, base_row, first_unit, last_unit)` enqueues the kernel for one chunk: a maximal
// run of row-contiguous units fitting one slot.  A unit with chained[u] != 0 (a later piece of a
// range streamed in pieces) always starts a new chunk, so only a chunk's first unit continues
// an earlier one.
template <class Launch>
void stream_chunks(sstat_cuda_ctx* c, const HostRows& hr, const std::vector<uint64_t>& unit_row,
                   const std::vector<uint64_t>& unit_rows, Launch&& launch, sstat_cuda_timings* tm,
                   const std::vector<uint8_t>* chained = nullptr) {
    const uint64_t row_bytes = (uint64_t)hr.p * 8;
    const uint64_t n_units = unit_row.size();
    uint64_t u = 0, chunk = 0;
    while (u < n_units) {
        // maximal run of row-contiguous units fitting one slot
        uint64_t v = u, bytes = 0;
        while (v < n_units) {
            const uint64_t b = unit_rows[v] * row_bytes;
            if (v > u && (bytes + b > c->slot_cap || unit_row[v] != unit_row[v - 1] + unit_rows[v - 1] ||
                          (chained && (*chained)[v])))
                break;
            if (b > c->slot_cap) throw Fail{SSTAT_ERR_UNSUPPORTED, "staging slot smaller than one work unit"};
            bytes += b;
            ++v;
        }
        const uint32_t slot = (uint32_t)(chunk % c->n_slots);
        const uint64_t row0 = unit_row[u], nrows = bytes / row_bytes;
        CUDA_TRY(cudaStreamWaitEvent(c->copy, c->ev_free[slot], 0));
        if (tm && chunk == 0) CUDA_TRY(cudaEventRecord(c->ev[5], c->copy));
        const void* host_src;
        if (hr.pinned) {
            host_src = hr.host_row(row0);
        } else {
            // the bounce buffer of this slot is reused: its previous copy must be done
            if (chunk >= c->n_slots) CUDA_TRY(cudaEventSynchronize(c->ev_copied[slot]));
            if (hr.reader()) {
                host_src = hr.get(c->bounce[slot].p, row0, nrows);
            } else {
                if (!c->pool) c->pool.reset(new FillPool(c->host_threads ? c->host_threads : default_host_threads()));
                hr.fill_parallel(*c->pool, c->bounce[slot].p, row0, nrows);
                host_src = c->bounce[slot].p;
            }
        }
        CUDA_TRY(cudaMemcpyAsync(c->slots[slot].p, host_src, bytes, cudaMemcpyHostToDevice, c->copy));
        CUDA_TRY(cudaEventRecord(c->ev_copied[slot], c->copy));
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_copied[slot], 0));
        launch(static_cast<const double*>(c->slots[slot].p), row0, u, v);
        CUDA_TRY(cudaEventRecord(c->ev_free[slot], c->stream));
        if (tm) {
            tm->h2d_bytes += bytes;
            tm->kernel_launches += 1;
        }
        u = v;
        ++chunk;
    }
    if (tm && chunk > 0) {  // h2d_seconds: first copy start to last copy end on the copy stream
        CUDA_TRY(cudaEventRecord(c->ev[6], c->copy));
        c->h2d_timed = true;
    }
}

void check_plan(sstat_cuda_ctx* c, const sstat_cuda_source* src, Plan& P, BinFile& file) {
    const bool whole = P.mode == Mode::Dataset || P.mode == Mode::Comoments;  // dataset-level calls
    const bool single_chunk = !whole;
    Fail inv{SSTAT_ERR_INVALID, ""};
    if (P.p == 0) {
        inv.msg = "schema: column count must be >= 1";
        throw inv;
    }
    if (P.precision > 1) {
        inv.msg = "unknown precision mode";
        throw inv;
    }
    if (P.R > 0 && (!P.starts || !P.counts)) {
        inv.msg = "null range arrays";
        throw inv;
    }
    P.total = 0;
    for (uint64_t i = 0; i < P.R; ++i) {
        if (i > 0 && P.starts[i] < P.starts[i - 1] + P.counts[i - 1]) {
            inv.msg = "partition ranges must be ascending and disjoint";
            throw inv;
        }
        P.total += P.counts[i];
    }
    const int world = single_chunk ? 1 : c->world;
    if (src->kind == SSTAT_SRC_FILE) {
        open_bin(src->path, file);
        if (file.rows != P.total) {
            inv.msg = "run_reduction: partition covers " + std::to_string(P.total) + " rows but dataset has " +
                      std::to_string(file.rows);
            throw inv;
        }
        if (file.cols != P.p) {
            Fail f{SSTAT_ERR_SCHEMA, "range 0 failed: chunk has " + std::to_string(file.cols) + " columns, schema has " +
                                         std::to_string(P.p)};
            f.range = 0;
            throw f;
        }
    } else if (src->kind == SSTAT_SRC_DEVICE || src->kind == SSTAT_SRC_HOST || src->kind == SSTAT_SRC_READER) {
        // (a rank or group member without ranges may pass an empty source: no rows, no pointer)
        if (src->kind == SSTAT_SRC_READER ? !src->read_rows : (!src->ptr && src->n_rows > 0)) {
            inv.msg = src->kind == SSTAT_SRC_READER ? "null read_rows callback" : "null row pointer";
            throw inv;
        }
        if (world == 1 && whole) {
            const uint64_t ds = src->first_row + src->n_rows;
            if (src->first_row != 0 || ds != P.total) {
                inv.msg = "run_reduction: partition covers " + std::to_string(P.total) + " rows but dataset has " +
                          std::to_string(src->n_rows) + " rows";
                throw inv;
            }
        }
    } else {
        inv.msg = "unknown source kind";
        throw inv;
    }
    uint64_t ds_rows = kNone;  // dataset rows when known to this rank
    if (src->kind == SSTAT_SRC_FILE) ds_rows = file.rows;
    else if (world == 1 && whole) ds_rows = src->first_row + src->n_rows;
    if (P.R > 0 && ds_rows != kNone && P.starts[P.R - 1] + P.counts[P.R - 1] > ds_rows) {
        inv.msg = "partition exceeds the dataset";
        throw inv;
    }
    P.r0 = (uint64_t)c->rank * P.R / world;
    P.r1 = (uint64_t)(c->rank + 1) * P.R / world;
    if (world == 1) {
        P.r0 = 0;
        P.r1 = P.R;
    }
    if (P.mode == Mode::Partials) {
        if (P.want_r0 > P.want_r1 || P.want_r1 > P.R) {
            inv.msg = "range window out of bounds";
            throw inv;
        }
        P.r0 = P.want_r0;
        P.r1 = P.want_r1;
    }
    P.L = P.r1 - P.r0;
    P.lmax = (P.R + world - 1) / world;
    P.E = partial_len(P.p);
    P.span_begin = P.L ? P.starts[P.r0] : 0;
    P.span_end = P.L ? P.starts[P.r1 - 1] + P.counts[P.r1 - 1] : 0;
    if (src->kind != SSTAT_SRC_FILE && P.L > 0 &&
        (P.span_begin < src->first_row || P.span_end > src->first_row + src->n_rows)) {
        inv.msg = "source rows [" + std::to_string(src->first_row) + ", " + std::to_string(src->first_row + src->n_rows) +
                  ") do not cover this rank's ranges [" + std::to_string(P.span_begin) + ", " +
                  std::to_string(P.span_end) + ")";
        throw inv;
    }
    const bool reference_order = P.mode != Mode::Comoments && ((P.flags & SSTAT_FLAG_REFEXACT) || P.precision == 1);
    if (P.L > 65535 && reference_order) {
        inv.msg = "reference-order mode supports at most 65535 ranges per device";
        throw inv;
    }
}

// Local ranges [starts | counts | tile prefix] to the device (skipped when identical to the
// previous call's upload).  Sets P.n_tiles.
uint64_t* upload_meta(sstat_cuda_ctx* c, Plan& P, uint64_t TR, cudaStream_t s) {
    const uint64_t L = P.L;
    CUDA_TRY(c->h_meta.reserve((3 * L + 1) * 8));
    uint64_t* hm = c->h_meta.as<uint64_t>();
    uint64_t nt = 0;
    for (uint64_t i = 0; i < L; ++i) {
        hm[i] = P.starts[P.r0 + i];
        hm[L + i] = P.counts[P.r0 + i];
        hm[2 * L + i] = nt;
        nt += (P.counts[P.r0 + i] + TR - 1) / TR;
    }
    hm[3 * L] = nt;
    P.n_tiles = nt;
    CUDA_TRY(c->d_meta.reserve((3 * L + 1) * 8));
    uint64_t* d_starts = c->d_meta.as<uint64_t>();
    const bool same_plan = c->meta_gen == c->d_meta.gen && c->meta_last.size() == 3 * L + 1 &&
                           std::equal(hm, hm + 3 * L + 1, c->meta_last.begin());
    c->meta_gen = 0;  // re-validated below once the upload is enqueued
    if (!same_plan) {
        CUDA_TRY(cudaMemcpyAsync(d_starts, hm, (3 * L + 1) * 8, cudaMemcpyHostToDevice, s));
        c->meta_last.assign(hm, hm + 3 * L + 1);
    }
    c->meta_gen = c->d_meta.gen;
    return d_starts;
}

// Every range of [starts, starts + n) begins on a 16-byte boundary of the rows at `base`.
bool rows_aligned16(const double* base, uint64_t base_row, const uint64_t* starts, uint64_t n, uint32_t p) {
    if (reinterpret_cast<uintptr_t>(base) % 16) return false;
    for (uint64_t i = 0; i < n; ++i)
        if (((starts[i] - base_row) * p) % 2) return false;
    return true;
}

// What the local phase hands to the exchange and fold.  refexact / comoments are pure functions
// of the arguments (classify), so a rank that failed early still knows its layout.
struct Local {
    bool refexact = false, comoments = false, shift = false;
    bool graphable = false;  // one GPU, resident K1 pass: folds and read-back are in the graph
    bool hdr_first = false;  // graph read-back laid out [header | result] (one-range plans)
    bool scanned = false;    // the non-finite scan already ran for this rank
    double* rank_buf = nullptr;
    uint64_t rank_stride = 0;  // kHdr + lmax * E doubles
    bool ext = false;          // rank_buf is a slot of a group's gather buffer (not this context's d_rank)
};

void classify(const Plan& P, Local& st) {
    st.comoments = P.mode == Mode::Comoments;  // co-moments always take the shifted fast path
    st.refexact = !st.comoments && ((P.flags & SSTAT_FLAG_REFEXACT) || P.precision == 1);
    st.shift = !(P.flags & SSTAT_FLAG_NO_SHIFT) && !st.refexact;
}

int call_world(const sstat_cuda_ctx* c, const Plan& P) {
    return (P.mode == Mode::Dataset || P.mode == Mode::Comoments) ? c->world : 1;
}

// Reference-order pieces: each local range split into pieces of at most `max_rows` rows (an
// even number, so a piece keeps its range's 16-byte alignment); piece_range = its local range,
// chained = a later piece (its chains continue the earlier pieces').
struct Pieces {
    std::vector<uint64_t> row, rows, range;
    std::vector<uint8_t> chained;
};
Pieces split_ranges(const Plan& P, uint64_t max_rows) {
    Pieces pc;
    max_rows = std::max<uint64_t>(2, max_rows & ~(uint64_t)1);
    for (uint64_t i = 0; i < P.L; ++i) {
        const uint64_t rs = P.starts[P.r0 + i], rc = P.counts[P.r0 + i];
        uint64_t off = 0;
        do {
            const uint64_t k = std::min(max_rows, rc - off);
            pc.row.push_back(rs + off);
            pc.rows.push_back(k);
            pc.range.push_back(i);
            pc.chained.push_back(off > 0);
            off += k;
        } while (off < rc);
    }
    return pc;
}

// Pieces' (start, count) to the device: [starts | counts] of n pieces.
uint64_t* upload_pieces(sstat_cuda_ctx* c, const Pieces& pc, cudaStream_t s) {
    const uint64_t n = pc.row.size();
    CUDA_TRY(c->h_pieces.reserve(2 * n * 8));
    CUDA_TRY(c->d_pieces.reserve(2 * n * 8));
    uint64_t* h = c->h_pieces.as<uint64_t>();
    std::copy(pc.row.begin(), pc.row.end(), h);
    std::copy(pc.rows.begin(), pc.rows.end(), h + n);
    CUDA_TRY(cudaMemcpyAsync(c->d_pieces.p, h, 2 * n * 8, cudaMemcpyHostToDevice, s));
    return c->d_pieces.as<uint64_t>();
}

bool host_pinned(const sstat_cuda_source* src) {
    if (src->kind != SSTAT_SRC_HOST) return false;
    cudaPointerAttributes attr{};
    bool pinned = false;
    if (cudaPointerGetAttributes(&attr, src->ptr) == cudaSuccess) pinned = attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return pinned;
}

// Phase 1: this device's ranges — accumulate (K1/K1w/K2 or reference order), fold per range
// (K3a) into the rank buffer [header | lmax x E], and (world > 1) locate the first non-finite
// value so every rank knows it before the exchange.  One GPU, resident K1: the whole pass
// including the folds and the read-back is one replayed CUDA graph.
void run_local(sstat_cuda_ctx* c, const sstat_cuda_source* src, Plan& P, BinFile& file, Local& st,
               sstat_cuda_timings* tm) {
    check_plan(c, src, P, file);
    c->h2d_timed = false;
    const int world = call_world(c, P);
    const bool comoments = st.comoments, refexact = st.refexact, shift = st.shift;
    // K2 stages at least one k-step (4 rows) of every column in shared memory, double-buffered
    if (P.p > kMaxWideP && !refexact)
        throw Fail{SSTAT_ERR_UNSUPPORTED, "p = " + std::to_string(P.p) + " exceeds the " + std::to_string(kMaxWideP) +
                                              "-column limit of the fast path (reference-order mode has none)"};
    const uint32_t p = P.p;
    const uint64_t E = P.E, L = P.L;
    cudaStream_t s = c->stream;

    // ---- local plan → device ----
    const uint64_t TR = tile_rows_for(P);
    auto tiles_of = [TR](uint64_t count) { return (count + TR - 1) / TR; };
    uint64_t* d_starts = upload_meta(c, P, TR, s);
    uint64_t* d_counts = d_starts + L;
    uint64_t* d_prefix = d_starts + 2 * L;
    const uint64_t nt = P.n_tiles;
    uint32_t fold_k = 1;  // K3a's cluster size: the most chunks any local range folds in
    for (uint64_t i = 0; i < L; ++i) fold_k = std::max(fold_k, fold_chunks(tiles_of(P.counts[P.r0 + i])));

    const uint64_t rank_stride = kHdr + P.lmax * E;
    CUDA_TRY(c->d_flags.reserve(std::max<uint64_t>(L, 1) * 4));
    st.rank_stride = rank_stride;
    // the header ([0] lowest failing range, [1] first non-finite index: all-ones = none;
    // [2] the rank's status, [3] spare: 0) and the range flags are only written when something
    // is flagged or failed: reset them only after such a call or a realloc
    if (c->ext_rank) {
        // a member of a fused device group: K3a and the scan write this member's slot of member
        // 0's gather buffer directly (peer stores / atomics over NVLink): the exchange is the fold
        st.rank_buf = c->ext_rank;
        st.ext = true;
        CUDA_TRY(cudaMemsetAsync(st.rank_buf, 0xff, 2 * 8, s));
        CUDA_TRY(cudaMemsetAsync(st.rank_buf + 2, 0, (kHdr - 2) * 8, s));
        CUDA_TRY(cudaMemsetAsync(c->d_flags.p, 0, std::max<uint64_t>(L, 1) * 4, s));
    } else {
        CUDA_TRY(c->d_rank.reserve(rank_stride * 8));
        st.rank_buf = c->d_rank.as<double>();
        if (!(c->flags_clean && c->clean_rank == c->d_rank.gen && c->clean_flags == c->d_flags.gen &&
              L <= c->clean_len)) {
            CUDA_TRY(cudaMemsetAsync(c->d_rank.p, 0xff, 2 * 8, s));
            CUDA_TRY(cudaMemsetAsync(c->d_rank.as<double>() + 2, 0, (kHdr - 2) * 8, s));
            CUDA_TRY(cudaMemsetAsync(c->d_flags.p, 0, std::max<uint64_t>(L, 1) * 4, s));
            c->clean_rank = c->d_rank.gen;
            c->clean_flags = c->d_flags.gen;
            c->clean_len = std::max<uint64_t>(L, 1);
        }
    }
    c->flags_clean = false;  // until this call ends with nothing flagged
    double* rank_buf = st.rank_buf;
    uint32_t* d_flags = c->d_flags.as<uint32_t>();
    if (!refexact) {
        CUDA_TRY(c->d_tiles.reserve(std::max<uint64_t>(nt, 1) * E * 8));
        if (shift) CUDA_TRY(c->d_shift.reserve(std::max<uint64_t>(L, 1) * p * 8));
    }
    const double* d_shift = shift ? c->d_shift.as<double>() : nullptr;
    const bool wide = p > 64;
    // Folding ranges inside K1 (last CTA of a range folds it) was measured and rejected: the
    // folds' L2/HBM round trips under the streaming load stretch K1's tail by ~0.5 ms, far
    // more than the ~40 us the separate K3a/K3b launches cost.
    CUDA_TRY(c->d_result.reserve(E * 8));

    auto tile_job = [&](const double* base, uint64_t base_row, uint64_t t0, uint64_t t1) {
        TileJob j{};
        j.base = base;
        j.base_row = base_row;
        j.range_start = d_starts;
        j.range_count = d_counts;
        j.tile_prefix = d_prefix;
        j.shift = d_shift;
        j.n_ranges = (uint32_t)L;
        j.p = p;
        j.tile_begin = t0;
        j.tile_end = t1;
        j.tile_partials = c->d_tiles.as<double>();
        j.launched = &c->last_kernel;
        j.tile_rows = (uint32_t)TR;
        if (wide) {
            CUDA_TRY(c->d_claim.reserve(sizeof(unsigned long long)));
            j.claim = c->d_claim.as<unsigned long long>();
            j.side = c->side;
            j.fork = c->ev_fork;
            j.join = c->ev_join;
        }
        uint32_t kernels = 1;
        CUDA_TRY(wide ? (splitp_handles(p) ? launch_splitp(j, c->sms, s) : launch_widep(j, c->sms, s, &kernels))
                      : launch_smallp(j, c->sms, s));
        if (tm) tm->kernel_launches += kernels - 1;  // the callers count one accumulate kernel
    };

    // ---- K1 on a resident shard, one GPU: the whole pass as one replayed CUDA graph ----
    // (launch-bound for small shards: four kernels, three events and the read-back become one
    // cudaGraphLaunch; captured on a private stream, keyed by every input the launches bake in.
    // Each external event node costs ~5-7 us of replay: the graph times K1 and the two folds
    // together — five events measured 14 us slower per call at C1 and C2)
    const bool graphable = src->kind == SSTAT_SRC_DEVICE && world == 1 && P.mode == Mode::Dataset && !refexact &&
                           !wide && L > 0 && nt > 0 && !getenv("SSTAT_NO_GRAPH");
    st.graphable = graphable;
    if (graphable) {
        CUDA_TRY(c->h_result.reserve(E * 8 + kHdr * 8));
        CUDA_TRY(c->d_result.reserve((E + kHdr) * 8));  // K3b appends the rank header
        const double* base = static_cast<const double*>(src->ptr);
        // timed = the graph records the K1 / fold events (each external event node costs ~5 us of
        // replay, so calls without timings replay a graph without them).  small = a plan cut into
        // short tiles (smallp_tile_rows): K1 and K3a read each range's shift row in place, so the
        // gather kernel drops out; one_range: K3b (a copy of one partial) drops out too.
        const bool timed = tm != nullptr;
        const bool small = TR < kTileRows;
        const bool one_range = P.R == 1;
        st.hdr_first = one_range;
        const std::vector<uint64_t> key = {
            (uint64_t)(uintptr_t)base, src->first_row, p, L, nt, E, P.r0, shift, (uint64_t)(uintptr_t)s, timed, TR,
            one_range,
            c->d_meta.gen, c->d_tiles.gen, c->d_rank.gen, c->d_flags.gen, c->d_shift.gen, c->d_result.gen,
            (uint64_t)(uintptr_t)c->h_result.p, (uint64_t)(uintptr_t)c->d_meta.p, (uint64_t)(uintptr_t)c->d_tiles.p,
            (uint64_t)(uintptr_t)c->d_rank.p, (uint64_t)(uintptr_t)c->d_shift.p, (uint64_t)(uintptr_t)c->d_result.p};
        if (!(c->graph && c->graph_key == key)) {
            if (c->graph) cudaGraphExecDestroy(c->graph);
            c->graph = nullptr;
            c->graph_key.clear();
            CUDA_TRY(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeRelaxed));
            cudaGraph_t g = nullptr;
            try {
                const cudaStream_t cs = c->cap;
                if (shift && !small)
                    CUDA_TRY(launch_gather_shift(base, src->first_row, d_starts, d_counts, (uint32_t)L, p,
                                                 c->d_shift.as<double>(), cs));
                if (timed) CUDA_TRY(cudaEventRecordWithFlags(c->ev[0], cs, cudaEventRecordExternal));
                TileJob j{};
                j.base = base;
                j.base_row = src->first_row;
                j.range_start = d_starts;
                j.range_count = d_counts;
                j.tile_prefix = d_prefix;
                j.shift = small ? nullptr : d_shift;
                j.shift_in_place = small && shift;
                j.n_ranges = (uint32_t)L;
                j.p = p;
                j.tile_begin = 0;
                j.tile_end = nt;
                j.tile_partials = c->d_tiles.as<double>();
                j.launched = &c->last_kernel;
                j.tile_rows = (uint32_t)TR;
                CUDA_TRY(launch_smallp(j, c->sms, cs));
                if (timed) CUDA_TRY(cudaEventRecordWithFlags(c->ev[1], cs, cudaEventRecordExternal));
                CUDA_TRY(launch_range_fold(c->d_tiles.as<double>(), d_prefix, d_counts, small ? nullptr : d_shift,
                                           small && shift ? base : nullptr, src->first_row, d_starts, (uint32_t)L, p,
                                           P.r0, rank_buf, d_flags, fold_k, cs));
                if (one_range) {
                    // one range: the fold of one partial is the partial itself (K3a adds + 0.0 like the
                    // fold would), so the read-back takes the rank buffer [header | partial] directly
                    if (timed) CUDA_TRY(cudaEventRecordWithFlags(c->ev[4], cs, cudaEventRecordExternal));
                    CUDA_TRY(cudaMemcpyAsync(c->h_result.p, rank_buf, (E + kHdr) * 8, cudaMemcpyDeviceToHost, cs));
                } else {
                    CUDA_TRY(launch_final_fold(rank_buf, rank_stride, P.R, 1, p, 0u, false, c->d_result.as<double>(), cs));
                    if (timed) CUDA_TRY(cudaEventRecordWithFlags(c->ev[4], cs, cudaEventRecordExternal));
                    CUDA_TRY(cudaMemcpyAsync(c->h_result.p, c->d_result.p, (E + kHdr) * 8, cudaMemcpyDeviceToHost, cs));
                }
            } catch (...) {
                cudaStreamEndCapture(c->cap, &g);
                if (g) cudaGraphDestroy(g);
                cudaGetLastError();
                throw;
            }
            CUDA_TRY(cudaStreamEndCapture(c->cap, &g));
            const cudaError_t ie = cudaGraphInstantiate(&c->graph, g, 0);
            cudaGraphDestroy(g);
            CUDA_TRY(ie);
            c->graph_key = key;
        }
        CUDA_TRY(cudaGraphLaunch(c->graph, s));
        if (tm) {
            tm->bytes_read += (P.span_end - P.span_begin) * p * 8;
            tm->kernel_launches += (shift && !small ? 1 : 0) + 2 + (one_range ? 0 : 1);  // [gather] K1 K3a [K3b]
        }
        return;  // everything up to the read-back is in the graph
    }

    CUDA_TRY(cudaEventRecord(c->ev[0], s));
    if (tm) tm->bytes_read += (P.span_end - P.span_begin) * p * 8;
    if (L > 0 && src->kind == SSTAT_SRC_DEVICE) {
        const double* base = static_cast<const double*>(src->ptr);
        const uint64_t base_row = src->first_row;
        if (refexact) {
            CUDA_TRY(launch_refexact(base, base_row, d_starts, d_counts, (uint32_t)L, p, P.precision, P.r0, rank_buf,
                                     rank_buf + kHdr, d_flags, rows_aligned16(base, base_row, P.starts + P.r0, L, p),
                                     false, s));
            CUDA_TRY(cudaEventRecord(c->ev[1], s));
            if (tm) tm->kernel_launches += 1;
        } else {
            // the shift table: each range's first row, gathered from the resident shard
            if (shift) {
                CUDA_TRY(launch_gather_shift(base, base_row, d_starts, d_counts, (uint32_t)L, p, c->d_shift.as<double>(), s));
                if (tm) tm->kernel_launches += 1;
            }
            CUDA_TRY(cudaEventRecord(c->ev[0], s));  // kernel_seconds brackets K1/K2 alone
            if (nt > 0) tile_job(base, base_row, 0, nt);
            CUDA_TRY(cudaEventRecord(c->ev[1], s));
            if (comoments)
                CUDA_TRY(launch_comoment_range(c->d_tiles.as<double>(), d_prefix, d_counts, d_shift, (uint32_t)L, p,
                                               rank_buf + kHdr, P.r0, rank_buf, d_flags, s));
            else
                CUDA_TRY(launch_range_fold(c->d_tiles.as<double>(), d_prefix, d_counts, d_shift, nullptr, 0, d_starts,
                                           (uint32_t)L, p, P.r0, rank_buf, d_flags, fold_k, s));
            if (tm) tm->kernel_launches += 2;
        }
        if (world > 1 || P.mode == Mode::Partials) {
            // every rank must know its first non-finite before the exchange; on one GPU the
            // scan runs only when a range was flagged (after the result read-back)
            CUDA_TRY(launch_find_nonfinite(base, base_row, d_starts, d_counts, (uint32_t)L, p, d_flags, rank_buf,
                                           c->sms * 2, s));
            if (tm) tm->kernel_launches += 1;
            st.scanned = true;
        }
        CUDA_TRY(cudaEventRecord(c->ev[2], s));
    } else if (L > 0) {
        // ---- host / file source: pinned staging ring, copy stream || compute stream ----
        const bool pinned = host_pinned(src);
        HostRows hr{src, src->kind == SSTAT_SRC_FILE ? &file : nullptr, p, pinned};
        // reference-order ranges stream as slot-sized pieces; fast-path tiles are whole units
        ensure_slots(c, !pinned, refexact ? 2ull * p * 8 : TR * p * 8);  // (readers: bounce = scratch)
        if (shift) {
            CUDA_TRY(c->h_shift.reserve(L * p * 8));
            double* hs = c->h_shift.as<double>();
            for (uint64_t i = 0; i < L; ++i) {
                if (P.counts[P.r0 + i] == 0) std::fill(hs + i * p, hs + (i + 1) * p, 0.0);
                else if (file.fd >= 0) hr.fill(hs + i * p, P.starts[P.r0 + i], 1);
                else if (hr.reader()) {
                    const void* q = hr.get(hs + i * p, P.starts[P.r0 + i], 1);
                    if (q != hs + i * p) std::memcpy(hs + i * p, q, p * 8);
                } else std::memcpy(hs + i * p, hr.host_row(P.starts[P.r0 + i]), p * 8);
            }
            CUDA_TRY(cudaMemcpyAsync(c->d_shift.p, hs, L * p * 8, cudaMemcpyHostToDevice, s));
        }
        CUDA_TRY(cudaEventRecord(c->ev[0], s));
        CUDA_TRY(cudaStreamWaitEvent(c->copy, c->ev[0], 0));
        if (refexact) {
            // units = range pieces of at most one slot; a range longer than a slot continues its
            // chains across launches (resume_first), so the order of operations is unchanged
            const Pieces pc = split_ranges(P, c->slot_cap / ((uint64_t)p * 8));
            const uint64_t* d_pc = upload_pieces(c, pc, s);
            const uint64_t npc = pc.row.size();
            stream_chunks(c, hr, pc.row, pc.rows,
                          [&](const double* base, uint64_t base_row, uint64_t u0, uint64_t u1) {
                              // pieces [u0, u1) belong to consecutive local ranges from pc.range[u0]
                              const uint64_t lr = pc.range[u0];
                              CUDA_TRY(launch_refexact(base, base_row, d_pc + u0, d_pc + npc + u0, (uint32_t)(u1 - u0),
                                                       p, P.precision, P.r0 + lr, rank_buf, rank_buf + kHdr + lr * E,
                                                       d_flags + lr,
                                                       rows_aligned16(base, base_row, pc.row.data() + u0, u1 - u0, p),
                                                       pc.chained[u0] != 0, s));
                          },
                          tm, &pc.chained);
            CUDA_TRY(cudaEventRecord(c->ev[1], s));
        } else {
            std::vector<uint64_t> trow(nt), trows(nt);
            for (uint64_t i = 0, t = 0; i < L; ++i) {
                const uint64_t rs = P.starts[P.r0 + i], rc = P.counts[P.r0 + i];
                for (uint64_t q = 0; q < tiles_of(rc); ++q, ++t) {
                    trow[t] = rs + q * TR;
                    trows[t] = std::min<uint64_t>(TR, rs + rc - trow[t]);
                }
            }
            stream_chunks(c, hr, trow, trows,
                          [&](const double* base, uint64_t base_row, uint64_t t0, uint64_t t1) {
                              tile_job(base, base_row, t0, t1);
                          },
                          tm);
            CUDA_TRY(cudaEventRecord(c->ev[1], s));
            if (comoments)
                CUDA_TRY(launch_comoment_range(c->d_tiles.as<double>(), d_prefix, d_counts, d_shift, (uint32_t)L, p,
                                               rank_buf + kHdr, P.r0, rank_buf, d_flags, s));
            else
                CUDA_TRY(launch_range_fold(c->d_tiles.as<double>(), d_prefix, d_counts, d_shift, nullptr, 0, d_starts,
                                           (uint32_t)L, p, P.r0, rank_buf, d_flags, fold_k, s));
            if (tm) tm->kernel_launches += 1;
        }
        // Non-finite localisation: re-stream only the flagged ranges (error path).
        CUDA_TRY(c->h_flags.reserve(L * 4));
        CUDA_TRY(cudaMemcpyAsync(c->h_flags.p, d_flags, L * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        const uint32_t* hf = c->h_flags.as<uint32_t>();
        bool any = false;
        for (uint64_t i = 0; i < L; ++i) any |= hf[i] != 0;
        if (any) {
            // header[0] flags the rank for the scan kernel
            uint64_t lowest = kNone;
            for (uint64_t i = 0; i < L && lowest == kNone; ++i)
                if (hf[i]) lowest = P.r0 + i;
            CUDA_TRY(cudaMemcpyAsync(rank_buf, &lowest, 8, cudaMemcpyHostToDevice, s));
            for (uint64_t i = 0; i < L; ++i) {
                if (!hf[i]) continue;
                std::vector<uint64_t> urow{P.starts[P.r0 + i]}, urows{P.counts[P.r0 + i]};
                // split the range into slot-sized pieces of whole rows
                std::vector<uint64_t> prow, prows;
                const uint64_t per = std::max<uint64_t>(1, c->slot_cap / (p * 8));
                for (uint64_t r = 0; r < urows[0]; r += per) {
                    prow.push_back(urow[0] + r);
                    prows.push_back(std::min(per, urows[0] - r));
                }
                uint32_t one = 1;
                CUDA_TRY(cudaMemcpyAsync(d_flags, &one, 4, cudaMemcpyHostToDevice, s));
                stream_chunks(c, hr, prow, prows,
                              [&](const double* base, uint64_t base_row, uint64_t u0, uint64_t u1) {
                                  // scan rows [prow[u0], prow[u1-1]+prows[u1-1]) as a one-range job
                                  uint64_t hmeta[2] = {prow[u0], 0};
                                  for (uint64_t k = u0; k < u1; ++k) hmeta[1] += prows[k];
                                  c->meta_gen = 0;  // d_meta overwritten: re-upload next call
                                  CUDA_TRY(cudaMemcpyAsync(d_starts, hmeta, 16, cudaMemcpyHostToDevice, s));
                                  CUDA_TRY(launch_find_nonfinite(base, base_row, d_starts, d_starts + 1, 1, p, d_flags,
                                                                 rank_buf, c->sms * 2, s));
                                  CUDA_TRY(cudaStreamSynchronize(s));
                              },
                              nullptr);
            }
        }
        st.scanned = true;
        CUDA_TRY(cudaEventRecord(c->ev[2], s));
    } else {
        CUDA_TRY(cudaEventRecord(c->ev[1], s));
        CUDA_TRY(cudaEventRecord(c->ev[2], s));
    }
}

// A rank whose local phase failed still joins the exchange: its header carries the status so
// every rank fails together instead of waiting in the collective (reduce.hpp:111-134 never
// deadlocks either).  The layout is a function of the arguments alone.
void publish_status(sstat_cuda_ctx* c, const Plan& P, Local& st, int status) {
    const uint64_t E = partial_len(P.p), lmax = (P.R + c->world - 1) / c->world;
    st.rank_stride = kHdr + lmax * E;
    if (c->ext_rank) {
        st.rank_buf = c->ext_rank;
        st.ext = true;
    } else {
        CUDA_TRY(c->d_rank.reserve(st.rank_stride * 8));
        st.rank_buf = c->d_rank.as<double>();
    }
    st.graphable = false;
    const uint64_t hdr[kHdr] = {kNone, kNone, (uint64_t)status, 0};
    CUDA_TRY(cudaMemcpyAsync(st.rank_buf, hdr, sizeof hdr, cudaMemcpyHostToDevice, c->stream));
    c->flags_clean = false;
}

// Rank-ordered all-gather of the per-range partials (multi-process: one communicator rank per
// process).  Returns the buffer the fold reads.
const double* exchange(sstat_cuda_ctx* c, const Local& st, int world) {
    if (world == 1) return st.rank_buf;
    CUDA_TRY(c->d_gather.reserve(st.rank_stride * world * 8));
    ncclResult_t r = ncclAllGather(st.rank_buf, c->d_gather.p, st.rank_stride, ncclDouble, c->comm, c->stream);
    if (r != ncclSuccess) throw Fail{SSTAT_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r)};
    return c->d_gather.as<double>();
}

// "k_smallp<2, true>" for a kernel's host stub (cudaFuncGetName + demangle, namespaces and the
// parameter list dropped): which accumulate kernel a pass actually ran, for the timings.
void kernel_name(const void* fn, char* out, size_t cap) {
    out[0] = 0;
    if (!fn) return;
    const char* mangled = nullptr;
    if (cudaFuncGetName(&mangled, fn) != cudaSuccess || !mangled) {
        cudaGetLastError();
        return;
    }
    int status = 0;
    char* dem = abi::__cxa_demangle(mangled, nullptr, nullptr, &status);
    std::string name = status == 0 && dem ? dem : mangled;
    std::free(dem);
    // drop the parameter list (the last top-level '('), then the namespace qualifiers before the
    // kernel's own name (the last top-level "::")
    int depth = 0;
    size_t cut = name.size(), start = 0;
    for (size_t i = 0; i < name.size(); ++i) {  // the parameter list: the last top-level '('
        const char ch = name[i];
        if (ch == '<') ++depth;
        else if (ch == '>') --depth;
        else if (ch == '(' && depth == 0 && name.compare(i, 12, "(anonymous n") != 0) cut = i;
    }
    depth = 0;
    for (size_t i = 0; i < cut; ++i) {  // the kernel's own name: after the last top-level "::" or ' '
        const char ch = name[i];
        if (ch == '<') ++depth;
        else if (ch == '>') --depth;
        else if (depth == 0 && ch == ':' && i + 1 < cut && name[i + 1] == ':') start = i + 2;
        else if (depth == 0 && ch == ' ' && name.compare(i, 10, " namespace") != 0) start = i + 1;
    }
    std::snprintf(out, cap, "%s", name.substr(start, cut - start).c_str());
}

// Phase 2: the ascending range fold (K3b) or the co-moment merge over the gathered rank
// buffers, one read-back of the result and every rank header, then the headers: lowest failing
// range / first non-finite index over all ranks, and the first rank that reported a failure.
void run_fold(sstat_cuda_ctx* c, const sstat_cuda_source* src, const Plan& P, const Local& st, const double* fold_buf,
              int world, double* result_host, Outcome& out, sstat_cuda_timings* tm) {
    Trace trace_tail("sstat.fold+readback");
    const uint32_t p = P.p;
    const uint64_t E = P.E ? P.E : partial_len(p), L = P.L;
    cudaStream_t s = c->stream;
    if (!st.graphable) {
        CUDA_TRY(cudaEventRecord(c->ev[3], s));
        CUDA_TRY(c->d_result.reserve((E + world * kHdr) * 8));
        if (st.comoments) {
            // every range's count (the merge weights), for all ranks' ranges
            CUDA_TRY(c->h_counts.reserve(std::max<uint64_t>(P.R, 1) * 8));
            CUDA_TRY(c->d_counts.reserve(std::max<uint64_t>(P.R, 1) * 8));
            std::memcpy(c->h_counts.p, P.counts, P.R * 8);
            CUDA_TRY(cudaMemcpyAsync(c->d_counts.p, c->h_counts.p, P.R * 8, cudaMemcpyHostToDevice, s));
            CUDA_TRY(launch_comoment_merge(fold_buf, st.rank_stride, P.R, world, c->d_counts.as<uint64_t>(), p,
                                           c->d_result.as<double>(), s));
        } else {
            CUDA_TRY(launch_final_fold(fold_buf, st.rank_stride, P.R, world, p, st.refexact ? P.precision : 0u,
                                       st.refexact, c->d_result.as<double>(), s));
        }
        if (tm) tm->kernel_launches += 1;
        CUDA_TRY(cudaEventRecord(c->ev[4], s));
        CUDA_TRY(c->h_result.reserve(E * 8 + world * kHdr * 8));
        // result and every rank's header in one read-back (K3b appends the headers)
        CUDA_TRY(cudaMemcpyAsync(c->h_result.p, c->d_result.p, (E + world * kHdr) * 8, cudaMemcpyDeviceToHost, s));
    }
    double* hres = c->h_result.as<double>();
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaGetLastError());
    if (st.graphable && st.hdr_first) {  // [header | result] -> [result | header]
        double hdr[kHdr];
        std::memcpy(hdr, hres, sizeof hdr);
        std::memmove(hres, hres + kHdr, E * 8);
        std::memcpy(hres + E, hdr, sizeof hdr);
    }
    if (!st.scanned && world == 1 && L > 0) {
        uint64_t flagged;
        std::memcpy(&flagged, hres + E, 8);
        if (flagged != kNone) {  // error path: locate the first non-finite value of the flagged ranges
            uint64_t* d_starts = c->d_meta.as<uint64_t>();
            CUDA_TRY(launch_find_nonfinite(static_cast<const double*>(src->ptr), src->first_row, d_starts, d_starts + L,
                                           (uint32_t)L, p, c->d_flags.as<uint32_t>(), st.rank_buf, c->sms * 2, s));
            CUDA_TRY(cudaMemcpyAsync(hres + E, st.rank_buf, kHdr * 8, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
        }
    }
    bool any_flag = false;
    for (int q = 0; q < world; ++q) {
        uint64_t lin, range, status;
        std::memcpy(&range, hres + E + q * kHdr, 8);
        std::memcpy(&lin, hres + E + q * kHdr + 1, 8);
        std::memcpy(&status, hres + E + q * kHdr + 2, 8);
        out.bad_lin = std::min(out.bad_lin, lin);
        any_flag |= range != kNone || status != 0;
        if (status != 0 && out.failed_rank < 0) {
            out.failed_rank = q;
            out.failed_status = (int)status;
        }
    }
    if (!st.ext) c->flags_clean = !any_flag;  // (a fused group's fold reads the gather buffer)
    if (result_host) std::memcpy(result_host, hres, E * 8);
    if (tm) kernel_name(c->last_kernel, tm->kernel, sizeof tm->kernel);
    if (tm && st.graphable) {  // the graph records three events: K1, then both folds together
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
        tm->kernel_seconds += ms * 1e-3;
        cudaEventElapsedTime(&ms, c->ev[1], c->ev[4]);
        tm->fold_seconds += ms * 1e-3;
        tm->n_local_ranges = (uint32_t)L;
    } else if (tm) {
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
        tm->kernel_seconds += ms * 1e-3;
        cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]);
        tm->fold_seconds += ms * 1e-3;
        cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]);
        tm->fold_seconds += ms * 1e-3;
        cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
        tm->exchange_seconds += ms * 1e-3;
        if (c->h2d_timed && cudaEventElapsedTime(&ms, c->ev[5], c->ev[6]) == cudaSuccess) tm->h2d_seconds += ms * 1e-3;
        tm->n_local_ranges = (uint32_t)L;
    }
}

Fail peer_failure(const Outcome& o) {
    return Fail{SSTAT_ERR_PEER, "rank " + std::to_string(o.failed_rank) + " failed: " +
                                    sstat_status_string(o.failed_status)};
}

// The engine proper on one context (one GPU, or one rank of a multi-process communicator).
// Returns the all-rank outcome; throws Fail.
void run(sstat_cuda_ctx* c, const sstat_cuda_source* src, Plan& P, double* result_host, Outcome& out,
         sstat_cuda_timings* tm) {
    BinFile file;
    Trace trace_run(P.mode == Mode::Comoments ? "sstat.comoments" : P.mode == Mode::Partials ? "sstat.range_partials"
                    : P.mode == Mode::Chunk ? "sstat.accumulate_chunk" : "sstat.dataset");
    Local st;
    classify(P, st);
    const int world = call_world(c, P);
    if (world == 1) {
        run_local(c, src, P, file, st, tm);
        if (P.mode == Mode::Partials) {
            const uint64_t E = P.E, L = P.L;
            CUDA_TRY(c->h_result.reserve((L * E + kHdr) * 8));
            double* hres = c->h_result.as<double>();
            CUDA_TRY(cudaMemcpyAsync(hres, st.rank_buf, (kHdr + L * E) * 8, cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            std::memcpy(&out.bad_lin, hres + 1, 8);
            if (L) std::memcpy(P.partials_host, hres + kHdr, L * E * 8);
            return;
        }
        run_fold(c, src, P, st, st.rank_buf, 1, result_host, out, tm);
        return;
    }
    // multi-process: a local failure is published in the rank header, the exchange still runs
    Fail local;
    bool failed = false;
    try {
        run_local(c, src, P, file, st, tm);
    } catch (const Fail& f) {
        local = f;
        failed = true;
    }
    if (failed) {
        try {
            publish_status(c, P, st, local.status);
        } catch (const Fail&) {
            throw local;  // the device cannot even publish (sticky CUDA error): peers are not told
        }
    }
    const double* fold_buf = exchange(c, st, world);
    run_fold(c, src, P, st, fold_buf, world, result_host, out, tm);
    if (failed) throw local;
    if (out.failed_rank >= 0) throw peer_failure(out);
}

// column_sum (reference src/reduce.cpp:32-88) over the plan's ranges; 32-byte partials
// {float sum, exact lo, exact hi, first non-integral row} per tile / range.  The rank buffer is
// [header part {0, status, 0, 0} | lmax range parts].
struct ColResult {
    double f;
    uint64_t lo, hi, bad_row;
};

struct ColLocal {
    char* rank_buf = nullptr;
    uint64_t stride = 0;  // in 32-byte parts: header + lmax
};

void colsum_local(sstat_cuda_ctx* c, const sstat_cuda_source* src, Plan& P, uint32_t column, BinFile& file,
                  ColLocal& cl) {
    check_plan(c, src, P, file);
    if (column >= P.p)
        throw Fail{SSTAT_ERR_INVALID, "column_sum: column " + std::to_string(column) + " out of range, dataset has " +
                                          std::to_string(P.p) + " columns"};
    const uint32_t p = P.p;
    const uint64_t L = P.L;
    const bool sequential = (P.flags & SSTAT_FLAG_REFEXACT) || P.precision == 1;
    cudaStream_t s = c->stream;
    uint64_t* d_starts = upload_meta(c, P, kTileRows, s);
    uint64_t* d_counts = d_starts + L;
    uint64_t* d_prefix = d_starts + 2 * L;
    const uint64_t nt = P.n_tiles;
    cl.stride = 1 + P.lmax;
    CUDA_TRY(c->d_rank.reserve(cl.stride * 32));
    CUDA_TRY(c->d_aux.reserve(std::max<uint64_t>(nt, 1) * 32));
    cl.rank_buf = static_cast<char*>(c->d_rank.p);
    c->flags_clean = false;  // d_rank is shared with the sufficient-statistics header: reset it next time
    CUDA_TRY(cudaMemsetAsync(cl.rank_buf, 0, 32, s));  // header part: status 0
    void* range_parts = cl.rank_buf + 32;
    if (L > 0 && src->kind == SSTAT_SRC_DEVICE) {
        const double* base = static_cast<const double*>(src->ptr);
        CUDA_TRY(launch_colsum(base, src->first_row, p, column, d_starts, d_counts, d_prefix, (uint32_t)L, 0, nt,
                               sequential, P.precision, c->d_aux.p, range_parts, c->sms, false, s));
        if (!sequential) CUDA_TRY(launch_colsum_range_fold(c->d_aux.p, d_prefix, (uint32_t)L, range_parts, s));
    } else if (L > 0) {
        const bool pinned = host_pinned(src);
        HostRows hr{src, src->kind == SSTAT_SRC_FILE ? &file : nullptr, p, pinned};
        ensure_slots(c, !pinned, sequential ? 2ull * p * 8 : (uint64_t)kTileRows * p * 8);
        cudaEvent_t e0 = c->ev[0];
        CUDA_TRY(cudaEventRecord(e0, s));
        CUDA_TRY(cudaStreamWaitEvent(c->copy, e0, 0));
        if (sequential) {  // units = range pieces; a piece after the first continues its range's sums
            const Pieces pc = split_ranges(P, c->slot_cap / ((uint64_t)p * 8));
            const uint64_t* d_pc = upload_pieces(c, pc, s);
            const uint64_t npc = pc.row.size();
            stream_chunks(c, hr, pc.row, pc.rows,
                          [&](const double* base, uint64_t base_row, uint64_t u0, uint64_t u1) {
                              const uint64_t lr = pc.range[u0];
                              CUDA_TRY(launch_colsum(base, base_row, p, column, d_pc + u0, d_pc + npc + u0, nullptr,
                                                     (uint32_t)(u1 - u0), 0, 0, true, P.precision, nullptr,
                                                     static_cast<char*>(range_parts) + 32 * lr, c->sms,
                                                     pc.chained[u0] != 0, s));
                          },
                          nullptr, &pc.chained);
        } else {  // units = tiles
            std::vector<uint64_t> urow, urows;
            for (uint64_t i = 0; i < L; ++i) {
                const uint64_t rs = P.starts[P.r0 + i], rc = P.counts[P.r0 + i];
                for (uint64_t q = 0; q * kTileRows < rc; ++q) {
                    urow.push_back(rs + q * kTileRows);
                    urows.push_back(std::min<uint64_t>(kTileRows, rc - q * kTileRows));
                }
            }
            stream_chunks(c, hr, urow, urows,
                          [&](const double* base, uint64_t base_row, uint64_t t0, uint64_t t1) {
                              CUDA_TRY(launch_colsum(base, base_row, p, column, d_starts, d_counts, d_prefix,
                                                     (uint32_t)L, t0, t1, false, P.precision, c->d_aux.p, nullptr,
                                                     c->sms, false, s));
                          },
                          nullptr);
            CUDA_TRY(launch_colsum_range_fold(c->d_aux.p, d_prefix, (uint32_t)L, range_parts, s));
        }
    }
}

void colsum_publish(sstat_cuda_ctx* c, const Plan& P, ColLocal& cl, int status) {
    cl.stride = 1 + (P.R + c->world - 1) / c->world;
    CUDA_TRY(c->d_rank.reserve(cl.stride * 32));
    cl.rank_buf = static_cast<char*>(c->d_rank.p);
    c->flags_clean = false;
    const uint64_t hdr[4] = {0, (uint64_t)status, 0, 0};
    CUDA_TRY(cudaMemcpyAsync(cl.rank_buf, hdr, sizeof hdr, cudaMemcpyHostToDevice, c->stream));
}

// The final ascending fold over the gathered rank buffers, and every rank's header part.
void colsum_fold(sstat_cuda_ctx* c, const Plan& P, const void* fold_buf, uint64_t stride, int world, ColResult& res,
                 Outcome& out) {
    cudaStream_t s = c->stream;
    CUDA_TRY(c->d_result.reserve((1 + world) * 32));
    CUDA_TRY(launch_colsum_final(fold_buf, stride, P.R, world, P.precision, c->d_result.p, s));
    CUDA_TRY(c->h_result.reserve((1 + world) * 32));
    CUDA_TRY(cudaMemcpyAsync(c->h_result.p, c->d_result.p, (1 + world) * 32, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const uint64_t* h = c->h_result.as<uint64_t>();
    std::memcpy(&res, h, 32);
    for (int q = 0; q < world; ++q)
        if (h[4 * (1 + q) + 1] != 0 && out.failed_rank < 0) {
            out.failed_rank = q;
            out.failed_status = (int)h[4 * (1 + q) + 1];
        }
}

void run_colsum(sstat_cuda_ctx* c, const sstat_cuda_source* src, Plan& P, uint32_t column, ColResult& res) {
    Trace trace_run("sstat.column_sum");
    BinFile file;
    ColLocal cl;
    Outcome out;
    const int world = c->world;
    if (world == 1) {
        colsum_local(c, src, P, column, file, cl);
        colsum_fold(c, P, cl.rank_buf, cl.stride, 1, res, out);
        return;
    }
    Fail local;
    bool failed = false;
    try {
        colsum_local(c, src, P, column, file, cl);
    } catch (const Fail& f) {
        local = f;
        failed = true;
    }
    if (failed) {
        try {
            colsum_publish(c, P, cl, local.status);
        } catch (const Fail&) {
            throw local;
        }
    }
    CUDA_TRY(c->d_gather.reserve(cl.stride * 32 * world));
    ncclResult_t r = ncclAllGather(cl.rank_buf, c->d_gather.p, cl.stride * 4, ncclDouble, c->comm, c->stream);
    if (r != ncclSuccess) throw Fail{SSTAT_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r)};
    colsum_fold(c, P, c->d_gather.p, cl.stride, world, res, out);
    if (failed) throw local;
    if (out.failed_rank >= 0) throw peer_failure(out);
}

// ---- device groups (one process, G devices) ----

// Runs fn(i) for every member on the group's host threads (one per member), each bound to its
// member's device and holding its lock.  Returns each member's failure (failed[i] != 0).
template <class Fn>
void group_each(sstat_cuda_ctx* g, std::vector<Fail>& fails, std::vector<char>& failed, Fn&& fn) {
    const size_t G = g->members.size();
    fails.assign(G, Fail{});
    failed.assign(G, 0);
    g->gpool->run(G, [&](size_t i) {
        sstat_cuda_ctx* m = g->members[i];
        std::lock_guard<std::mutex> lk(m->mu);
        cudaSetDevice(m->device);
        try {
            fn(i, m);
        } catch (const Fail& f) {
            fails[i] = f;
            failed[i] = 1;
        } catch (const std::bad_alloc&) {
            fails[i] = Fail{SSTAT_ERR_OOM, "host allocation failed"};
            failed[i] = 1;
        } catch (const std::exception& e) {
            fails[i] = Fail{SSTAT_ERR_INVALID, e.what()};
            failed[i] = 1;
        }
    });
}

// A member that failed publishes its status in its rank header exactly like a failing rank of
// a multi-process communicator, and the exchange and fold still run, so the group exercises
// the same failure path on one GPU.  Members whose device cannot publish end the call here
// (after every member's queued work drained).  Returns the lowest failed member or -1.
int group_publish(sstat_cuda_ctx* g, const std::vector<Fail>& fails, const std::vector<char>& failed,
                  const std::function<void(size_t, sstat_cuda_ctx*, int)>& publish) {
    int first = -1;
    bool stuck = false;
    for (size_t i = 0; i < g->members.size(); ++i) {
        if (!failed[i]) continue;
        if (first < 0) first = (int)i;
        sstat_cuda_ctx* m = g->members[i];
        std::lock_guard<std::mutex> lk(m->mu);
        cudaSetDevice(m->device);
        try {
            publish(i, m, fails[i].status);
        } catch (const Fail&) {
            stuck = true;
        }
    }
    if (stuck) {
        for (sstat_cuda_ctx* m : g->members) {
            std::lock_guard<std::mutex> lk(m->mu);
            cudaSetDevice(m->device);
            cudaStreamSynchronize(m->stream);
            cudaStreamSynchronize(m->copy);
            cudaGetLastError();
        }
        throw fails[first];
    }
    return first;
}

// Moves every member's rank buffer (stride_doubles each, at bufs[i]) into member 0's gather
// buffer in rank order: grouped ncclAllGather over the ncclCommInitAll communicators, or (no
// communicators: peer-copy and fused groups — column_sum is not fused) peer copies
// (cudaMemcpyPeerAsync over NVLink) ordered after each member's stream.  Returns member
// 0's gathered buffer; member 0's stream is ordered after every contribution.
void* group_gather(sstat_cuda_ctx* g, const std::vector<const void*>& bufs, uint64_t stride_doubles) {
    const int G = (int)g->members.size();
    sstat_cuda_ctx* m0 = g->members[0];
    if (G == 1) return const_cast<void*>(bufs[0]);  // one member: its own rank buffer
    std::vector<std::unique_lock<std::mutex>> locks;
    for (sstat_cuda_ctx* m : g->members) locks.emplace_back(m->mu);
    const uint64_t bytes = stride_doubles * 8;
    if (!m0->comm) {  // peer copies (the peer-copy groups, and the calls a fused group does not fuse)
        CUDA_TRY(cudaSetDevice(m0->device));
        CUDA_TRY(m0->d_gather.reserve(bytes * G));
        for (int i = 0; i < G; ++i) {
            sstat_cuda_ctx* m = g->members[i];
            if (i > 0) {
                CUDA_TRY(cudaSetDevice(m->device));
                CUDA_TRY(cudaEventRecord(m->ev[7], m->stream));
                CUDA_TRY(cudaSetDevice(m0->device));
                CUDA_TRY(cudaStreamWaitEvent(m0->stream, m->ev[7], 0));
            }
            CUDA_TRY(cudaMemcpyPeerAsync(m0->d_gather.as<char>() + i * bytes, m0->device, bufs[i], m->device, bytes,
                                         m0->stream));
        }
        return m0->d_gather.p;
    }
    for (sstat_cuda_ctx* m : g->members) {
        CUDA_TRY(cudaSetDevice(m->device));
        CUDA_TRY(m->d_gather.reserve(bytes * G));
    }
    ncclResult_t r = ncclGroupStart();
    for (int i = 0; i < G && r == ncclSuccess; ++i) {
        sstat_cuda_ctx* m = g->members[i];
        r = ncclAllGather(bufs[i], m->d_gather.p, stride_doubles, ncclDouble, m->comm, m->stream);
    }
    const ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        throw Fail{SSTAT_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r != ncclSuccess ? r : r2)};
    CUDA_TRY(cudaSetDevice(m0->device));
    return m0->d_gather.p;
}

// Sources of a group call: DEVICE = one source per member (its shard, on its device);
// HOST / FILE = one source every member reads its own ranges from.
const sstat_cuda_source* member_src(const sstat_cuda_source* src, size_t i) {
    return src->kind == SSTAT_SRC_DEVICE ? src + i : src;
}

void sum_timings(sstat_cuda_timings* tm, const std::vector<sstat_cuda_timings>& tms) {
    if (!tm) return;
    for (const auto& t : tms) {
        tm->h2d_seconds = std::max(tm->h2d_seconds, t.h2d_seconds);
        tm->kernel_seconds = std::max(tm->kernel_seconds, t.kernel_seconds);
        tm->fold_seconds = std::max(tm->fold_seconds, t.fold_seconds);
        tm->bytes_read += t.bytes_read;
        tm->h2d_bytes += t.h2d_bytes;
        tm->kernel_launches += t.kernel_launches;
        tm->n_local_ranges += t.n_local_ranges;
    }
}

// dataset_suffstats / co-moments over a device group: every member accumulates its contiguous
// share of the ranges in parallel (rank i of G, the same shard rule as the multi-process path),
// the rank buffers meet in member 0, and member 0 runs the same fold — bit-identical to one GPU
// and to G processes.
void run_group(sstat_cuda_ctx* g, const sstat_cuda_source* src, const Plan& P0, double* result_host, Outcome& out,
               sstat_cuda_timings* tm) {
    Trace trace_run(P0.mode == Mode::Comoments ? "sstat.group.comoments" : "sstat.group.dataset");
    const size_t G = g->members.size();
    std::vector<Plan> Ps(G, P0);
    std::vector<Local> sts(G);
    std::vector<BinFile> files(G);
    std::vector<sstat_cuda_timings> tms(G);
    std::vector<Fail> fails;
    std::vector<char> failed;
    for (size_t i = 0; i < G; ++i) classify(Ps[i], sts[i]);
    sstat_cuda_ctx* m0 = g->members[0];
    const bool fused = g->fused && G > 1;
    if (fused) {
        // every member's rank buffer is its slot of member 0's gather buffer (the layout of the
        // exchange, a function of the plan alone): K3a's stores are the all-gather
        const uint64_t E = partial_len(P0.p), lmax = (P0.R + G - 1) / G, stride = kHdr + lmax * E;
        {
            std::lock_guard<std::mutex> lk(m0->mu);
            CUDA_TRY(cudaSetDevice(m0->device));
            CUDA_TRY(m0->d_gather.reserve(G * stride * 8));
        }
        for (size_t i = 0; i < G; ++i) g->members[i]->ext_rank = m0->d_gather.as<double>() + i * stride;
    }
    struct ClearExt {  // members return to their own rank buffers whatever happens
        sstat_cuda_ctx* g;
        ~ClearExt() {
            for (auto* m : g->members) m->ext_rank = nullptr;
        }
    } clear_ext{g};
    group_each(g, fails, failed, [&](size_t i, sstat_cuda_ctx* m) {
        run_local(m, member_src(src, i), Ps[i], files[i], sts[i], tm ? &tms[i] : nullptr);
    });
    const int first_failed = group_publish(g, fails, failed, [&](size_t i, sstat_cuda_ctx* m, int status) {
        publish_status(m, Ps[i], sts[i], status);
    });
    const double* fold_buf;
    if (fused) {  // member 0's stream waits for every member's local phase
        std::lock_guard<std::mutex> lk0(m0->mu);
        for (size_t i = 1; i < G; ++i) {
            sstat_cuda_ctx* m = g->members[i];
            std::lock_guard<std::mutex> lk(m->mu);
            CUDA_TRY(cudaSetDevice(m->device));
            CUDA_TRY(cudaEventRecord(m->ev[7], m->stream));
            CUDA_TRY(cudaSetDevice(m0->device));
            CUDA_TRY(cudaStreamWaitEvent(m0->stream, m->ev[7], 0));
        }
        CUDA_TRY(cudaSetDevice(m0->device));
        fold_buf = m0->d_gather.as<double>();
    } else {
        std::vector<const void*> bufs(G);
        for (size_t i = 0; i < G; ++i) bufs[i] = sts[i].rank_buf;
        fold_buf = static_cast<const double*>(group_gather(g, bufs, sts[0].rank_stride));
    }
    std::lock_guard<std::mutex> lk(m0->mu);
    sstat_cuda_timings t0{};
    run_fold(m0, member_src(src, 0), Ps[0], sts[0], fold_buf, (int)G, result_host, out, tm ? &t0 : nullptr);
    if (first_failed >= 0) {
        if (out.failed_rank != first_failed)
            throw Fail{SSTAT_ERR_CUDA, "group: rank headers disagree with the members' failures"};
        throw fails[first_failed];
    }
    if (tm) {
        // every member's copy span (member 0's stream has waited for all of them: complete)
        for (size_t i = 0; i < G; ++i) {
            sstat_cuda_ctx* m = g->members[i];
            float ms = 0;
            if (m->h2d_timed && cudaEventElapsedTime(&ms, m->ev[5], m->ev[6]) == cudaSuccess)
                tms[i].h2d_seconds = ms * 1e-3;
        }
        tms[0].fold_seconds += t0.fold_seconds;
        tms[0].exchange_seconds += t0.exchange_seconds;
        tms[0].kernel_launches += t0.kernel_launches;
        sum_timings(tm, tms);
        tm->exchange_seconds = t0.exchange_seconds;
        std::memcpy(tm->kernel, t0.kernel, sizeof tm->kernel);
    }
}

void run_group_colsum(sstat_cuda_ctx* g, const sstat_cuda_source* src, const Plan& P0, uint32_t column,
                      ColResult& res) {
    Trace trace_run("sstat.group.column_sum");
    const size_t G = g->members.size();
    std::vector<Plan> Ps(G, P0);
    std::vector<ColLocal> cls(G);
    std::vector<BinFile> files(G);
    std::vector<Fail> fails;
    std::vector<char> failed;
    group_each(g, fails, failed,
               [&](size_t i, sstat_cuda_ctx* m) { colsum_local(m, member_src(src, i), Ps[i], column, files[i], cls[i]); });
    const int first_failed = group_publish(g, fails, failed, [&](size_t i, sstat_cuda_ctx* m, int status) {
        colsum_publish(m, Ps[i], cls[i], status);
    });
    std::vector<const void*> bufs(G);
    for (size_t i = 0; i < G; ++i) bufs[i] = cls[i].rank_buf;
    const void* fold_buf = group_gather(g, bufs, cls[0].stride * 4);
    sstat_cuda_ctx* m0 = g->members[0];
    std::lock_guard<std::mutex> lk(m0->mu);
    Outcome out;
    colsum_fold(m0, Ps[0], fold_buf, cls[0].stride, (int)G, res, out);
    if (first_failed >= 0) {
        if (out.failed_rank != first_failed)
            throw Fail{SSTAT_ERR_CUDA, "group: rank headers disagree with the members' failures"};
        throw fails[first_failed];
    }
}

// double_equals_int128 (reference src/util.cpp:47-52).
bool double_equals_i128(double d, __int128 v) {
    if (!std::isfinite(d) || d != std::trunc(d)) return false;
    if (std::fabs(d) >= 0x1p127) return false;
    return static_cast<__int128>(d) == v;
}

uint64_t range_of_row(const Plan& P, uint64_t row) {
    uint64_t lo = 0, hi = P.R;  // last range with start <= row
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) / 2;
        if (P.starts[mid] <= row) lo = mid;
        else hi = mid;
    }
    return lo;
}

struct Guard {
    sstat_cuda_ctx* c;
    std::lock_guard<std::mutex> lk;
    explicit Guard(sstat_cuda_ctx* ctx) : c(ctx), lk(ctx->mu) { cudaSetDevice(ctx->device); }
};

}  // namespace

extern "C" {

int sstat_cuda_abi_version(void) { return SSTAT_CUDA_ABI_VERSION; }

const char* sstat_status_string(int status) {
    switch (status) {
        case SSTAT_OK: return "ok";
        case SSTAT_ERR_NONFINITE: return "non-finite value";
        case SSTAT_ERR_SCHEMA: return "schema mismatch";
        case SSTAT_ERR_INVALID: return "invalid argument";
        case SSTAT_ERR_CUDA: return "CUDA error";
        case SSTAT_ERR_NCCL: return "NCCL error";
        case SSTAT_ERR_OOM: return "out of device memory";
        case SSTAT_ERR_UNSUPPORTED: return "unsupported";
        case SSTAT_ERR_IO: return "I/O error";
        case SSTAT_ERR_FORMAT: return "format error";
        case SSTAT_ERR_PEER: return "another rank failed";
        default: return "unknown status";
    }
}

}  // extern "C"

namespace {

void free_device_state(sstat_cuda_ctx* c) {
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->copy) cudaStreamSynchronize(c->copy);
    if (c->side) cudaStreamSynchronize(c->side);
    if (c->comm) ncclCommDestroy(c->comm);
    c->comm = nullptr;
    for (DevBuf* b : {&c->d_meta, &c->d_tiles, &c->d_rank, &c->d_gather, &c->d_shift, &c->d_result, &c->d_flags,
                      &c->d_counts, &c->d_aux, &c->d_claim, &c->d_pieces})
        b->release();
    for (HostBuf* b : {&c->h_meta, &c->h_result, &c->h_shift, &c->h_flags, &c->h_counts, &c->h_pieces}) b->release();
    for (auto& s : c->slots) s.release();
    for (auto& b : c->bounce) b.release();
    for (auto e : c->ev_copied) cudaEventDestroy(e);
    for (auto e : c->ev_free) cudaEventDestroy(e);
    for (auto e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->graph) cudaGraphExecDestroy(c->graph);
    for (cudaStream_t s : {c->own, c->copy, c->cap, c->side})
        if (s) cudaStreamDestroy(s);
}

// One device's context.  The context's own stream is a blocking stream: work on it is ordered
// after the legacy default stream, so a device source written by a default-stream producer
// (e.g. a torch kernel with no explicit stream) is complete before it is read.
int init_device(sstat_cuda_ctx* c, int device) {
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess) return SSTAT_ERR_CUDA;
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&c->own, cudaStreamDefault) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return SSTAT_ERR_CUDA;
    c->stream = c->own;
    for (auto& e : c->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return SSTAT_ERR_CUDA;
    return SSTAT_OK;
}

int device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

template <class Body>
int guarded(sstat_cuda_error* err, Body&& body) {
    try {
        body();
        return SSTAT_OK;
    } catch (const Fail& f) {
        cudaGetLastError();
        return report(err, f);
    } catch (const std::bad_alloc&) {
        return report(err, Fail{SSTAT_ERR_OOM, "host allocation failed"});
    } catch (const std::exception& e) {
        return report(err, Fail{SSTAT_ERR_INVALID, e.what()});
    }
}

Fail nonfinite_failure(const Plan& P, const Outcome& o, bool in_dataset) {
    Fail f{SSTAT_ERR_NONFINITE, ""};
    f.row = o.bad_lin / P.p;
    f.col = (uint32_t)(o.bad_lin % P.p);
    if (in_dataset) {
        f.range = range_of_row(P, f.row);
        f.msg = "range " + std::to_string(f.range) + " failed: non-finite value at row " + std::to_string(f.row) +
                ", column " + std::to_string(f.col);
    } else {
        f.range = 0;
        f.msg = "non-finite value at row " + std::to_string(f.row) + ", column " + std::to_string(f.col);
    }
    return f;
}

}  // namespace

extern "C" {

int sstat_cuda_init(sstat_cuda_ctx** out, int device) {
    if (!out) return SSTAT_ERR_INVALID;
    *out = nullptr;
    const int n = device_count();
    if (n == 0) return SSTAT_ERR_CUDA;
    if (device < 0) cudaGetDevice(&device);
    if (device >= n) return SSTAT_ERR_INVALID;
    auto* c = new sstat_cuda_ctx;
    const int st = init_device(c, device);
    if (st != SSTAT_OK) {
        free_device_state(c);
        delete c;
        return st;
    }
    *out = c;
    return SSTAT_OK;
}

int sstat_cuda_init_devices(sstat_cuda_ctx** out, int n_gpus, const int* devices) {
    if (!out || n_gpus < 0 || (n_gpus > 0 && !devices)) return SSTAT_ERR_INVALID;
    *out = nullptr;
    const int n = device_count();
    if (n == 0) return SSTAT_ERR_CUDA;
    std::vector<int> all;
    if (n_gpus == 0) {  // every visible device
        for (int i = 0; i < n; ++i) all.push_back(i);
        n_gpus = n;
        devices = all.data();
    }
    bool distinct = true;
    for (int i = 0; i < n_gpus; ++i) {
        if (devices[i] < 0 || devices[i] >= n) return SSTAT_ERR_INVALID;
        for (int j = 0; j < i; ++j) distinct = distinct && devices[j] != devices[i];
    }
    auto* g = new sstat_cuda_ctx;
    g->device = devices[0];
    int st = SSTAT_OK;
    for (int i = 0; i < n_gpus && st == SSTAT_OK; ++i) {
        auto* m = new sstat_cuda_ctx;
        g->members.push_back(m);
        st = init_device(m, devices[i]);
        m->rank = i;
        m->world = n_gpus;
        // the members share the host: feeder threads split between them
        m->host_threads = std::max(1u, default_host_threads() / (unsigned)n_gpus);
    }
    // Exchange: fused (every member reaches member 0's memory: the same device, or peer access
    // over NVLink) unless SSTAT_GROUP_EXCHANGE picks "copy" (peer copies) or "nccl"
    // (ncclCommInitAll + grouped all-gather; also the default when a member cannot reach member 0)
    bool reach = true;
    for (int i = 1; i < n_gpus && st == SSTAT_OK; ++i) {
        if (devices[i] == devices[0]) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devices[i], devices[0]);
        if (can) {
            cudaSetDevice(devices[i]);
            const cudaError_t pe = cudaDeviceEnablePeerAccess(devices[0], 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) can = 0;
            cudaGetLastError();
        }
        reach = reach && can;
    }
    const char* xenv = getenv("SSTAT_GROUP_EXCHANGE");
    const std::string xmode = xenv ? xenv : "";
    if (n_gpus > 1) {
        if (xmode == "copy") g->peer = true;
        else if (xmode == "nccl") g->peer = !distinct;  // NCCL needs distinct devices
        else if (reach) g->fused = true;
        else g->peer = !distinct;
        if (getenv("SSTAT_PEER_EXCHANGE") && atoi(getenv("SSTAT_PEER_EXCHANGE")) != 0) g->peer = true, g->fused = false;
    }
    if (st == SSTAT_OK && n_gpus > 1 && !g->peer && !g->fused) {
        std::vector<ncclComm_t> comms(n_gpus);
        if (ncclCommInitAll(comms.data(), n_gpus, devices) != ncclSuccess) st = SSTAT_ERR_NCCL;
        else
            for (int i = 0; i < n_gpus; ++i) g->members[i]->comm = comms[i];
    }
    if (st == SSTAT_OK && g->peer && distinct)  // direct NVLink copies between member 0 and the rest
        for (int i = 1; i < n_gpus; ++i) {
            cudaSetDevice(devices[0]);
            cudaDeviceEnablePeerAccess(devices[i], 0);
            cudaSetDevice(devices[i]);
            cudaDeviceEnablePeerAccess(devices[0], 0);
            cudaGetLastError();  // already enabled / no P2P: cudaMemcpyPeerAsync still works
        }
    if (st == SSTAT_OK && g->fused && getenv("SSTAT_DEBUG")) fprintf(stderr, "sstat: device group of %d, fused exchange\n", n_gpus);
    if (st != SSTAT_OK) {
        for (auto* m : g->members) {
            free_device_state(m);
            delete m;
        }
        delete g;
        return st;
    }
    g->gpool.reset(new FillPool((unsigned)n_gpus));
    cudaSetDevice(devices[0]);
    *out = g;
    return SSTAT_OK;
}

int sstat_cuda_device_count(const sstat_cuda_ctx* c) {
    if (!c) return 0;
    return c->is_group() ? (int)c->members.size() : 1;
}

int sstat_cuda_destroy(sstat_cuda_ctx* c) {
    if (!c) return SSTAT_OK;
    if (c->is_group()) {
        {
            std::lock_guard<std::mutex> lk(c->mu);
            c->gpool.reset();
            for (auto* m : c->members) {
                std::lock_guard<std::mutex> lm(m->mu);
                free_device_state(m);
            }
        }
        for (auto* m : c->members) delete m;
        delete c;
        return SSTAT_OK;
    }
    {
        Guard g(c);
        free_device_state(c);
    }
    delete c;
    return SSTAT_OK;
}

int sstat_cuda_set_stream(sstat_cuda_ctx* c, void* stream) {
    if (!c) return SSTAT_ERR_INVALID;
    if (c->is_group()) return stream ? SSTAT_ERR_UNSUPPORTED : SSTAT_OK;  // members keep their own streams
    Guard g(c);
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own;
    return SSTAT_OK;
}

int sstat_cuda_set_staging(sstat_cuda_ctx* c, uint32_t slots, uint64_t slot_bytes) {
    if (!c || slots < 2 || slot_bytes < (1u << 20)) return SSTAT_ERR_INVALID;
    if (c->is_group()) {
        for (auto* m : c->members)
            if (int st = sstat_cuda_set_staging(m, slots, slot_bytes)) return st;
        return SSTAT_OK;
    }
    Guard g(c);
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->copy);
    for (auto& s : c->slots) s.release();
    for (auto& b : c->bounce) b.release();
    for (auto e : c->ev_copied) cudaEventDestroy(e);
    for (auto e : c->ev_free) cudaEventDestroy(e);
    c->slots.clear();
    c->bounce.clear();
    c->ev_copied.clear();
    c->ev_free.clear();
    c->n_slots = slots;
    c->slot_bytes = slot_bytes & ~(uint64_t)127;
    c->slot_cap = 0;
    return SSTAT_OK;
}

int sstat_cuda_set_host_threads(sstat_cuda_ctx* c, uint32_t threads) {
    if (!c || threads > 1024) return SSTAT_ERR_INVALID;
    if (c->is_group()) {
        for (auto* m : c->members)
            if (int st = sstat_cuda_set_host_threads(m, threads)) return st;
        return SSTAT_OK;
    }
    Guard g(c);
    c->host_threads = threads;
    c->pool.reset();
    return SSTAT_OK;
}

int sstat_cuda_nccl_unique_id(void* id_out, size_t id_bytes) {
    if (!id_out || id_bytes < sizeof(ncclUniqueId)) return SSTAT_ERR_INVALID;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return SSTAT_ERR_NCCL;
    std::memcpy(id_out, &id, sizeof id);
    return SSTAT_OK;
}

int sstat_cuda_comm_init(sstat_cuda_ctx* c, int rank, int world, const void* id, size_t id_bytes) {
    if (!c || c->is_group() || world < 1 || rank < 0 || rank >= world) return SSTAT_ERR_INVALID;
    Guard g(c);
    if (c->comm) {
        ncclCommDestroy(c->comm);
        c->comm = nullptr;
    }
    c->rank = rank;
    c->world = world;
    if (world == 1 && !id) return SSTAT_OK;
    if (!id || id_bytes < sizeof(ncclUniqueId)) return SSTAT_ERR_INVALID;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    if (ncclCommInitRank(&c->comm, world, uid, rank) != ncclSuccess) {
        c->comm = nullptr;
        c->rank = 0;
        c->world = 1;
        return SSTAT_ERR_NCCL;
    }
    return SSTAT_OK;
}

int sstat_shard_ranges(uint64_t n_ranges, int rank, int world, uint64_t* first, uint64_t* last) {
    if (world < 1 || rank < 0 || rank >= world || !first || !last) return SSTAT_ERR_INVALID;
    *first = (uint64_t)rank * n_ranges / world;
    *last = (uint64_t)(rank + 1) * n_ranges / world;
    return SSTAT_OK;
}

int sstat_cuda_dataset(sstat_cuda_ctx* c, const sstat_cuda_source* src, uint32_t p, const uint64_t* range_start,
                       const uint64_t* range_count, uint64_t n_ranges, uint32_t precision, uint32_t flags,
                       uint64_t* n_out, double* sums_out, double* cross_out, sstat_cuda_timings* tm,
                       sstat_cuda_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!c || !src || !n_out || !sums_out || !cross_out)
        return report(err, Fail{SSTAT_ERR_INVALID, "null argument"});
    const double t0 = now_s();
    if (tm) std::memset(tm, 0, sizeof *tm);
    return guarded(err, [&] {
        Guard g(c);
        if (!c->is_group() && c->world > 1 && !c->comm) throw Fail{SSTAT_ERR_INVALID, "communicator not initialised"};
        Plan P{};
        P.p = p;
        P.precision = precision;
        P.flags = flags;
        P.R = n_ranges;
        P.starts = range_start;
        P.counts = range_count;
        std::vector<double> result(partial_len(p ? p : 1));
        Outcome o;
        if (c->is_group()) run_group(c, src, P, result.data(), o, tm);
        else run(c, src, P, result.data(), o, tm);
        if (o.bad_lin != kNone) throw nonfinite_failure(P, o, true);
        if (o.failed_rank >= 0) throw peer_failure(o);
        uint64_t total = 0;
        for (uint64_t i = 0; i < n_ranges; ++i) total += range_count[i];
        *n_out = total;
        std::memcpy(sums_out, result.data(), p * 8);
        std::memcpy(cross_out, result.data() + p, (partial_len(p) - p) * 8);
        if (tm) tm->total_seconds = now_s() - t0;
    });
}

int sstat_cuda_accumulate(sstat_cuda_ctx* c, const double* rows, uint64_t n_rows, uint32_t p, uint64_t start_row,
                          uint32_t precision, uint32_t flags, uint64_t* n_out, double* sums_out, double* cross_out,
                          sstat_cuda_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!c || !n_out || !sums_out || !cross_out) return report(err, Fail{SSTAT_ERR_INVALID, "null argument"});
    if (p == 0) return report(err, Fail{SSTAT_ERR_INVALID, "schema: column count must be >= 1"});
    if (precision > 1) return report(err, Fail{SSTAT_ERR_INVALID, "unknown precision mode"});
    if (c->is_group()) {  // one chunk: the member whose device holds it (host chunks: member 0)
        cudaPointerAttributes attr{};
        sstat_cuda_ctx* m = c->members[0];
        if (rows && cudaPointerGetAttributes(&attr, rows) == cudaSuccess && attr.type == cudaMemoryTypeDevice)
            for (auto* q : c->members)
                if (q->device == attr.device) {
                    m = q;
                    break;
                }
        cudaGetLastError();
        return sstat_cuda_accumulate(m, rows, n_rows, p, start_row, precision, flags, n_out, sums_out, cross_out, err);
    }
    return guarded(err, [&] {
        Guard g(c);
        const uint64_t E = partial_len(p);
        if (n_rows == 0) {
            *n_out = 0;
            std::memset(sums_out, 0, p * 8);
            std::memset(cross_out, 0, (E - p) * 8);
            return;
        }
        if (!rows) throw Fail{SSTAT_ERR_INVALID, "null row pointer"};
        cudaPointerAttributes attr{};
        sstat_cuda_source src{};
        src.kind = SSTAT_SRC_HOST;
        if (cudaPointerGetAttributes(&attr, rows) == cudaSuccess &&
            (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged))
            src.kind = SSTAT_SRC_DEVICE;
        cudaGetLastError();
        src.ptr = rows;
        src.first_row = start_row;
        src.n_rows = n_rows;
        uint64_t rs = start_row, rc = n_rows;
        Plan P{};
        P.mode = Mode::Chunk;
        P.p = p;
        P.precision = precision;
        P.flags = flags;
        P.R = 1;
        P.starts = &rs;
        P.counts = &rc;
        std::vector<double> result(E);
        Outcome o;
        run(c, &src, P, result.data(), o, nullptr);
        if (o.bad_lin != kNone) throw nonfinite_failure(P, o, false);
        *n_out = n_rows;
        std::memcpy(sums_out, result.data(), p * 8);
        std::memcpy(cross_out, result.data() + p, (E - p) * 8);
    });
}

int sstat_cuda_range_partials(sstat_cuda_ctx* c, const sstat_cuda_source* src, uint32_t p,
                              const uint64_t* range_start, const uint64_t* range_count, uint64_t n_ranges,
                              uint64_t first_range, uint64_t last_range, uint32_t precision, uint32_t flags,
                              double* partials_out, sstat_cuda_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!c || !src || (!partials_out && last_range > first_range))
        return report(err, Fail{SSTAT_ERR_INVALID, "null argument"});
    if (c->is_group())  // the window on member 0 (its source: the first of a DEVICE source array)
        return sstat_cuda_range_partials(c->members[0], src, p, range_start, range_count, n_ranges, first_range,
                                         last_range, precision, flags, partials_out, err);
    return guarded(err, [&] {
        Guard g(c);
        Plan P{};
        P.mode = Mode::Partials;
        P.want_r0 = first_range;
        P.want_r1 = last_range;
        P.partials_host = partials_out;
        P.p = p;
        P.precision = precision;
        P.flags = flags;
        P.R = n_ranges;
        P.starts = range_start;
        P.counts = range_count;
        Outcome o;
        run(c, src, P, nullptr, o, nullptr);
        if (o.bad_lin != kNone) throw nonfinite_failure(P, o, true);
    });
}

int sstat_fold_ranges_host(const double* buf, uint64_t rank_stride, uint64_t n_ranges, int world, uint32_t p,
                           uint32_t precision, uint32_t flags, double* out) {
    if (!buf || !out || world < 1 || p == 0 || precision > 1) return SSTAT_ERR_INVALID;
    const uint64_t E = partial_len(p);
    const bool reference_order = (flags & SSTAT_FLAG_REFEXACT) || precision == 1;
    for (uint64_t e = 0; e < E; ++e)
        out[e] = reference_order ? fold_entry(buf, rank_stride, n_ranges, world, p, precision, e)
                                 : fold_fast(buf, rank_stride, n_ranges, world, E, e);
    return SSTAT_OK;
}

int sstat_cuda_column_sum(sstat_cuda_ctx* c, const sstat_cuda_source* src, uint32_t p, uint32_t column,
                          const uint64_t* range_start, const uint64_t* range_count, uint64_t n_ranges,
                          uint32_t precision, uint32_t flags, sstat_column_sum_result* out, sstat_cuda_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!c || !src || !out) return report(err, Fail{SSTAT_ERR_INVALID, "null argument"});
    return guarded(err, [&] {
        Guard g(c);
        if (!c->is_group() && c->world > 1 && !c->comm) throw Fail{SSTAT_ERR_INVALID, "communicator not initialised"};
        Plan P{};
        P.p = p;
        P.precision = precision;
        P.flags = flags;
        P.R = n_ranges;
        P.starts = range_start;
        P.counts = range_count;
        ColResult r{};
        if (c->is_group()) run_group_colsum(c, src, P, column, r);
        else run_colsum(c, src, P, column, r);
        const __int128 exact = (__int128)(((unsigned __int128)r.hi << 64) | r.lo);
        out->float_sum = r.f;
        out->exact_ok = r.bad_row == kNone;
        out->exact_hi = (int64_t)r.hi;
        out->exact_lo = r.lo;
        out->note_row = r.bad_row;
        out->float_matches_exact = out->exact_ok && double_equals_i128(r.f, exact);
    });
}

int sstat_cuda_comoments(sstat_cuda_ctx* c, const sstat_cuda_source* src, uint32_t p, const uint64_t* range_start,
                         const uint64_t* range_count, uint64_t n_ranges, uint32_t flags, uint64_t* n_out,
                         double* mean_out, double* m2_out, sstat_cuda_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    if (!c || !src || !n_out || !mean_out || !m2_out) return report(err, Fail{SSTAT_ERR_INVALID, "null argument"});
    return guarded(err, [&] {
        Guard g(c);
        if (!c->is_group() && c->world > 1 && !c->comm) throw Fail{SSTAT_ERR_INVALID, "communicator not initialised"};
        Plan P{};
        P.mode = Mode::Comoments;
        P.p = p;
        P.precision = 0;
        P.flags = flags & ~SSTAT_FLAG_REFEXACT;
        P.R = n_ranges;
        P.starts = range_start;
        P.counts = range_count;
        std::vector<double> result(partial_len(p ? p : 1));
        Outcome o;
        if (c->is_group()) run_group(c, src, P, result.data(), o, nullptr);
        else run(c, src, P, result.data(), o, nullptr);
        if (o.bad_lin != kNone) throw nonfinite_failure(P, o, true);
        if (o.failed_rank >= 0) throw peer_failure(o);
        uint64_t total = 0;
        for (uint64_t i = 0; i < n_ranges; ++i) total += range_count[i];
        *n_out = total;
        std::memcpy(mean_out, result.data(), p * 8);
        std::memcpy(m2_out, result.data() + p, (partial_len(p) - p) * 8);
    });
}

uint64_t sstat_plan_partitions(uint64_t n_rows, uint64_t chunk_rows, uint64_t* starts, uint64_t* counts) {
    if (chunk_rows == 0 || n_rows == 0) return 0;
    const uint64_t R = (n_rows + chunk_rows - 1) / chunk_rows;
    if (starts && counts)
        for (uint64_t i = 0; i < R; ++i) {
            starts[i] = i * chunk_rows;
            counts[i] = std::min(chunk_rows, n_rows - starts[i]);
        }
    return R;
}

int sstat_merge(uint32_t p, uint32_t precision, uint64_t* n_a, double* sums_a, double* cross_a, uint64_t n_b,
                const double* sums_b, const double* cross_b) {
    if (!n_a || !sums_a || !cross_a || !sums_b || !cross_b || p == 0 || precision > 1) return SSTAT_ERR_INVALID;
    const uint64_t np = (uint64_t)p * (p + 1) / 2;
    *n_a += n_b;
    if (precision == 1) {
        for (uint32_t j = 0; j < p; ++j) sums_a[j] = (double)((float)sums_a[j] + (float)sums_b[j]);
        for (uint64_t i = 0; i < np; ++i) cross_a[i] = (double)((float)cross_a[i] + (float)cross_b[i]);
    } else {
        for (uint32_t j = 0; j < p; ++j) sums_a[j] += sums_b[j];
        for (uint64_t i = 0; i < np; ++i) cross_a[i] += cross_b[i];
    }
    return SSTAT_OK;
}

int sstat_cuda_generate(sstat_cuda_ctx* c, double* dst, uint32_t kind, uint64_t seed, double mu, uint32_t n_int,
                        uint64_t first_row, uint64_t n_rows, uint32_t p) {
    if (!c || (!dst && n_rows) || p == 0 || kind > 2) return SSTAT_ERR_INVALID;
    if (c->is_group()) {  // on the member whose device holds dst
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, dst) != cudaSuccess || attr.type != cudaMemoryTypeDevice) {
            cudaGetLastError();
            return SSTAT_ERR_INVALID;
        }
        for (auto* m : c->members)
            if (m->device == attr.device) return sstat_cuda_generate(m, dst, kind, seed, mu, n_int, first_row, n_rows, p);
        return SSTAT_ERR_INVALID;
    }
    Guard g(c);
    cudaError_t e = launch_generate(dst, kind, seed, mu, n_int, first_row, n_rows, p, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    return e == cudaSuccess ? SSTAT_OK : SSTAT_ERR_CUDA;
}

}  // extern "C"
