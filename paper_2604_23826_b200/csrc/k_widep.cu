// k_widep.cu — K2: wide-p (p > 64) sufficient statistics, a SYRK on the FP64 DMMA pipe.
//
// Replaces accumulate_into<double> (reference src/suffstats.cpp:50-70) where X^T X is
// compute-bound (p(p+2) flops per 8p bytes).  Column blocks of 8 form an nb x nb grid of
// 8x8 output blocks; its upper triangle is cut into 4x4-block rectangles (I <= J).  A
// consumer warp owns one rectangle and runs the same straight-line program for every
// rectangle — 16 DMMA per k-step over 8 operand fragments, no per-block predicates (blocks
// past p multiply zero fragments; a diagonal rectangle's 6 mirrored blocks are computed and
// dropped), so the warp-synchronous DMMAs are never guarded.  C consumer warps (4 or 8)
// form a group = one CTA; G = ceil(items / C) groups cover the triangle.
//
// The G groups of a tile form one thread-block CLUSTER (split into m equal clusters when
// G > 16) that streams the tile through shared memory once:
//   * producer warp of cluster rank k: one elected lane waits until every consumer warp
//     of the cluster has released the ring slot (`empty`, K x C arrivals), then issues the
//     stage's rows rr = k (mod K) as TMA bulk copies multicast to all K CTAs
//     (cp.async.bulk ... .multicast::cluster), each completing on the receiving CTA's
//     `full` mbarrier, which expects the whole stage's bytes (expect_tx by its own
//     producer).  The tile leaves HBM once and L2 once per cluster instead of once per
//     group; rows are padded to pitch = 4 mod 16 doubles so the 4-row fragment reads are
//     conflict-free.  Odd p (8-byte-aligned rows) falls back to per-CTA 8-byte cp.async
//     with cp.async.mbarrier.arrive;
//   * consumer warps: wait `full`, read fragments (next k-step's loads in flight while the
//     current DMMAs issue), subtract the range shift held in registers, DMMA, then arrive on
//     the slot's `empty` mbarrier of every CTA of the cluster (mapa + remote arrive).
// Column sums of rectangle J ride on the warp that owns rectangle (0, J).  Each (tile, group)
// writes disjoint entries of the tile's canonical partial, so the result is a fixed
// function of the tile (independent of C, clusters, grid, ring depth and work split).
//
// Launch geometry is chosen once per (device, p) from the occupancy calculator (make_plan).
// When cluster placement leaves CTA slots idle, a second, cluster-less launch fills them on a
// side stream and both claim work dynamically from one CAS-updated word (claim_unit).
// k_widep_wg is the same body in one 512-thread CTA per SM: 12 consumer warps (three consumer
// warpgroups) and a producer warpgroup that hands them registers (setmaxnreg); the plan for
// each p builds both geometries and keeps the one wasting fewer DMMA blocks (launch_widep).
// SSTAT_WIDEP_* environment variables override the choices for experiments and tests:
// CONSUMERS (4 | 8), CLUSTER / MAXCLUSTER (K), NOCLUSTER, RING, SROWS (4 | 8 | 16), PERSM
// (CTAs per SM), R (rectangle side), WG (0 | 1: the kernel), SPARE=0 (no side launch); and
// SSTAT_DEBUG prints the plans.
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <utility>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace sstat_b200 {
namespace {

int sms_of(int device) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n;
}

constexpr uint32_t kIdle = 1u << 28;
// Fragment reads of the padded rectangle columns (up to 32 nr - 1 >= p) run past a row's
// pitch into the next row (harmless: those blocks are dropped) and, on a slot's last row,
// past the ring: kSlack doubles of shared memory keep them inside the allocation.
constexpr uint32_t kSlack = 32;

struct WideGeom {
    uint32_t p, nb, nr, pitch, n_groups, consumers, ring;
    uint32_t R;              // rectangle side in 8-column blocks (nr = ceil(nb / R))
    uint32_t csize;          // CTAs per cluster (K)
    uint32_t cpt;            // clusters per tile (m); n_groups == K * m
    const uint32_t* items;   // device [n_groups][consumers]: item words (item_word)
    // dynamic split with a concurrent second launch (nullptr = static unit order): both
    // launches claim work from one 64-bit word — role 0 (clustered, cpt == 1) whole tiles
    // from the bottom, role 1 (cluster-less) (tile, group) units from the top
    unsigned long long* claim;
    uint32_t role;
};

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on the barrier at the same smem offset in cluster CTA `cta`
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
    asm volatile(
        "{\n"
        ".reg .b32 ra;\n"
        "mapa.shared::cluster.u32 ra, %0, %1;\n"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// producer side of `empty`: the arrivals come from other CTAs' consumers
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}

// Canonical writes of one 8x8 block (column blocks A <= B) from lane (g, kk).
__device__ __forceinline__ void write_block(double* out, uint32_t p, uint32_t A, uint32_t B, int g, int kk,
                                            const double (&c)[2]) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t a = A * 8 + g, b = B * 8 + 2 * kk + i;
        if (a >= p || b >= p) continue;
        if (A == B && a > b) continue;
        out[p + packed_index(p, a < b ? a : b, a < b ? b : a)] = c[i];
    }
}

struct UnitInfo {
    uint64_t t;
    uint32_t r, rows;
    const double* tile;
};

__device__ __forceinline__ UnitInfo unit_info(const TileJob& job, const WideGeom& geo, uint32_t tile_rows,
                                              uint64_t t) {
    UnitInfo ui;
    ui.t = t;
    ui.r = range_of_tile(job.tile_prefix, job.n_ranges, t);
    const uint64_t rs = __ldg(job.range_start + ui.r), rc = __ldg(job.range_count + ui.r);
    const uint64_t row0 = rs + (t - __ldg(job.tile_prefix + ui.r)) * tile_rows;
    const uint64_t left = rs + rc - row0;
    ui.rows = left < tile_rows ? (uint32_t)left : tile_rows;
    ui.tile = job.base + (row0 - job.base_row) * geo.p;
    return ui;
}

// One k-step: 4 rows of the stage at `st` (lane kk reads row kk) for the 2R fragments.
template <int R>
__device__ __forceinline__ void load_frags(double (&r)[2 * R], const double* st, int colI, int colJ) {
#pragma unroll
    for (int a = 0; a < 2 * R; ++a) r[a] = st[a < R ? colI + 8 * a : colJ + 8 * (a - R)];
}
// DADD shares the FP64 pipe with DMMA (profiles/r01_fp64_mix_probe.log): only the warps that
// own a rectangle (0, J) add the column sums (SUMS), the others issue 2R DADD per R*R DMMA.
template <bool SUMS, int R>
__device__ __forceinline__ void kprep(double (&sums)[R], double (&r)[2 * R], const double (&cw)[2 * R]) {
#pragma unroll
    for (int a = 0; a < 2 * R; ++a) r[a] -= cw[a];
    if (SUMS) {
#pragma unroll
        for (int a = 0; a < R; ++a) sums[a] += r[R + a];
    }
}
template <int R>
__device__ __forceinline__ void kmma(double (&acc)[R * R][2], const double (&r)[2 * R]) {
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
        for (int b = 0; b < R; ++b) dmma_8x8x4(acc[a * R + b][0], acc[a * R + b][1], r[a], r[R + b]);
}

// ---- work items ----
// An item is one consumer warp's share of a tile: which 8-column blocks its fragments hold and
// which block products it accumulates, as one straight-line program per KIND:
//   kRect      R x R rectangle of the R-block groups I < J (I == J: a diagonal rectangle whose
//              mirrored blocks are computed and dropped)
//   kRectCol3  R x (R-1): groups I x J without J's last block
//   kRectRow3  (R-1) x R: groups I x J without I's last block
//   kDiagCol   diagonal group I's upper blocks (a <= b) + the column strip (I's blocks x block J)
//   kDiagRow   diagonal group I's upper blocks + the row strip (block J x I's blocks)
// Word: idle << 28 | kind << 24 | sums << 23 | I << 11 | J (J: a group for the rectangle
// kinds, an absolute block for the strips).  `sums`: the item adds the column sums of its
// J fragments (rectangles) or of all its fragments (diagonal kinds).
enum : uint32_t { kRect = 0, kRectCol3 = 1, kRectRow3 = 2, kDiagCol = 3, kDiagRow = 4 };
constexpr uint32_t kSumsBit = 1u << 23;
__host__ __device__ constexpr uint32_t item_word(uint32_t kind, uint32_t I, uint32_t J, bool sums) {
    return (kind << 24) | (sums ? kSumsBit : 0u) | (I << 11) | J;
}

template <int R, uint32_t KIND>
struct Prog {
    static constexpr bool DIAG = KIND == kDiagCol || KIND == kDiagRow;
    static constexpr int NI = KIND == kRectRow3 ? R - 1 : R;      // fragments of group I
    static constexpr int NJ = DIAG ? 1 : (KIND == kRectCol3 ? R - 1 : R);
    static constexpr int NF = NI + NJ;
    static constexpr int NDIAG = R * (R + 1) / 2;
    static constexpr int NACC = DIAG ? NDIAG + R : NI * NJ;
    static constexpr int NSUM = DIAG ? NF : NJ;                    // fragments whose sums it adds
    static constexpr int SUM0 = DIAG ? 0 : NI;                     // ... starting at this one
    // product i: fragment fa(i) as the A operand (rows of the block pair), fb(i) as B
    __host__ __device__ static constexpr int fa(int i) {
        if (!DIAG) return i / NJ;
        if (i < NDIAG) {
            int a = 0, left = i;
            while (left >= R - a) left -= R - a, ++a;
            return a;
        }
        return KIND == kDiagCol ? i - NDIAG : NI;
    }
    __host__ __device__ static constexpr int fb(int i) {
        if (!DIAG) return NI + i % NJ;
        if (i < NDIAG) {
            int a = 0, left = i;
            while (left >= R - a) left -= R - a, ++a;
            return a + left;
        }
        return KIND == kDiagCol ? NI : i - NDIAG;
    }
};

constexpr uint64_t kNoUnit = ~0ull;

// The claim word: low 32 bits = tiles taken by role 0 from the bottom (a prefix [0, a)),
// high 32 bits = units taken by role 1 from the top (tile T-1-b/G, group b%G).  Updated by
// CAS only when the claim is valid, so a <= T - ceil(b/G) always holds: every tile is
// processed once, wholly by one role.  Returns the unit (role 0: tile; role 1: tile*G+group).
__device__ uint64_t claim_unit(unsigned long long* W, uint32_t role, uint64_t T, uint32_t G) {
    unsigned long long old = atomicAdd(W, 0ull);
    for (;;) {
        const uint64_t a = old & 0xffffffffull, b = old >> 32;
        unsigned long long nw;
        uint64_t result;
        if (role == 0) {
            if (a + (b + G - 1) / G >= T) return kNoUnit;
            nw = old + 1;
            result = a;
        } else {
            const uint64_t tb = b / G;
            if (tb >= T || T - 1 - tb < a) return kNoUnit;  // a started tile is always >= a
            nw = old + (1ull << 32);
            result = (T - 1 - tb) * G + b % G;
        }
        const unsigned long long seen = atomicCAS(W, old, nw);
        if (seen == old) return result;
        old = seen;
    }
}

// Collective over the CTA (K = 1) or the cluster: one thread claims, everyone gets the unit.
// Producer and consumer warps call it at the same unit boundaries from different code paths
// (barrier.sync 1 / barrier.cluster count arrivals, not call sites).
__device__ __forceinline__ uint64_t acquire_unit(const TileJob& job, const WideGeom& geo, uint32_t K, uint32_t it,
                                                 uint64_t* s_claim) {
    uint64_t* slot = &s_claim[it & 1];
    const uint32_t rank = K > 1 ? cluster_rank() : 0;
    if (threadIdx.x == 0 && rank == 0)
        *slot = claim_unit(geo.claim, geo.role, job.tile_end - job.tile_begin, geo.n_groups);
    if (K > 1) {
        cluster_sync_all();
        uint64_t v;
        asm volatile(
            "{\n"
            ".reg .b32 ra;\n"
            "mapa.shared::cluster.u32 ra, %1, 0;\n"
            "ld.shared::cluster.u64 %0, [ra];\n"
            "}\n"
            : "=l"(v)
            : "r"(smem_u32(slot))
            : "memory");
        return v;
    }
    asm volatile("barrier.sync 1;\n" ::: "memory");
    return *(volatile uint64_t*)slot;
}

// One ring stage of SROWS rows of an R x R rectangle (the plain plans): a straight-line program with the next k-step's fragment
// loads issued under the current k-step's DMMAs.  The slot is released (release()) as soon as
// the last k-step's fragments have been consumed by its shift subtraction — before that
// k-step's DMMAs — so the producers can refill it a k-step earlier.
template <int SROWS, int R, bool SUMS, class Release>
__device__ __forceinline__ void consume_stage_rect(double (&acc)[R * R][2], double (&sums)[R], const double* st,
                                              uint32_t pitch, int colI, int colJ, const double (&cw)[2 * R],
                                              Release&& release) {
    constexpr int Q = SROWS / 4;
    double ra[2 * R], rb[2 * R];
    load_frags<R>(ra, st, colI, colJ);
#pragma unroll
    for (int q = 0; q < Q; q += 2) {
        if (q + 1 < Q) load_frags<R>(rb, st + 4 * (q + 1) * pitch, colI, colJ);
        kprep<SUMS, R>(sums, ra, cw);
        if (q + 1 == Q) release();
        kmma<R>(acc, ra);
        if (q + 2 < Q) load_frags<R>(ra, st + 4 * (q + 2) * pitch, colI, colJ);
        if (q + 1 < Q) {
            kprep<SUMS, R>(sums, rb, cw);
            if (q + 2 == Q) release();
            kmma<R>(acc, rb);
        }
    }
}

// One ring stage of SROWS rows of item program P: a straight-line program with the next
// k-step's fragment loads issued under the current k-step's DMMAs.  The slot is released
// (release()) as soon as the last k-step's fragments have been consumed by its shift subtraction
// — before that k-step's DMMAs — so the producers can refill it a k-step earlier.
// Fragment f reads column colI + 8f (f < NI) or colJ + 8(f - NI); DADD shares the FP64 pipe with
// DMMA (profiles/r01_fp64_mix_probe.log), so only the items marked `sums` add column sums.
template <class P>
__device__ __forceinline__ void load_frags_p(double (&r)[P::NF], const double* st, int colI, int colJ) {
#pragma unroll
    for (int f = 0; f < P::NF; ++f) r[f] = st[f < P::NI ? colI + 8 * f : colJ + 8 * (f - P::NI)];
}
template <class P, bool SUMS>
__device__ __forceinline__ void kprep_p(double (&sums)[P::NSUM], double (&r)[P::NF], const double (&cw)[P::NF]) {
#pragma unroll
    for (int f = 0; f < P::NF; ++f) r[f] -= cw[f];
    if (SUMS) {
#pragma unroll
        for (int k = 0; k < P::NSUM; ++k) sums[k] += r[P::SUM0 + k];
    }
}
// (the operand indices are forced to compile-time constants: a runtime index into the
// fragment registers would put them in local memory)
template <class P, int... Is>
__device__ __forceinline__ void kmma_seq(double (&acc)[P::NACC][2], const double (&r)[P::NF],
                                         std::integer_sequence<int, Is...>) {
    (dmma_8x8x4(acc[Is][0], acc[Is][1], r[std::integral_constant<int, P::fa(Is)>::value],
                r[std::integral_constant<int, P::fb(Is)>::value]),
     ...);
}
template <class P>
__device__ __forceinline__ void kmma_p(double (&acc)[P::NACC][2], const double (&r)[P::NF]) {
    kmma_seq<P>(acc, r, std::make_integer_sequence<int, P::NACC>{});
}
template <class P, class Blk, int... Is>
__device__ __forceinline__ void write_items_seq(double* out, uint32_t p, uint32_t nb, int g, int kk,
                                                const double (&acc)[P::NACC][2], Blk&& blk,
                                                std::integer_sequence<int, Is...>) {
    auto one = [&](auto ic) {
        constexpr int i = decltype(ic)::value;
        const uint32_t A = blk(P::fa(i)), B = blk(P::fb(i));
        if (A <= B && B < nb) write_block(out, p, A, B, g, kk, acc[i]);
    };
    (one(std::integral_constant<int, Is>{}), ...);
}
template <int SROWS, class P, bool SUMS, class Release>
__device__ __forceinline__ void consume_stage_p(double (&acc)[P::NACC][2], double (&sums)[P::NSUM], const double* st,
                                              uint32_t pitch, int colI, int colJ, const double (&cw)[P::NF],
                                              Release&& release) {
    constexpr int Q = SROWS / 4;
    double ra[P::NF], rb[P::NF];
    load_frags_p<P>(ra, st, colI, colJ);
#pragma unroll
    for (int q = 0; q < Q; q += 2) {
        if (q + 1 < Q) load_frags_p<P>(rb, st + 4 * (q + 1) * pitch, colI, colJ);
        kprep_p<P, SUMS>(sums, ra, cw);
        if (q + 1 == Q) release();
        kmma_p<P>(acc, ra);
        if (q + 2 < Q) load_frags_p<P>(ra, st + 4 * (q + 2) * pitch, colI, colJ);
        if (q + 1 < Q) {
            kprep_p<P, SUMS>(sums, rb, cw);
            if (q + 2 == Q) release();
            kmma_p<P>(acc, rb);
        }
    }
}

// One unit (tile, group) of item program P for this warp: the stages, then the epilogue — the
// item's disjoint canonical entries of the tile partial.  Advances the ring position.
template <int SROWS, int R, class P, bool SUMS, class Wait, class Release>
__device__ __forceinline__ void run_item(const TileJob& job, const WideGeom& geo, const UnitInfo& ui, uint32_t I,
                                         uint32_t J, int g, int kk, const double* sm, uint32_t slot_elems,
                                         uint32_t& slot, uint32_t& ph, Wait&& wait, Release&& release) {
    const uint32_t p = geo.p, pitch = geo.pitch, nb = geo.nb;
    // the 8-column block of fragment f
    auto blk = [&](int f) -> uint32_t {
        return f < P::NI ? R * I + f : (P::DIAG ? J : R * J + (f - P::NI));
    };
    const int colI = (int)(8 * R * I) + g, colJ = (int)(8 * (P::DIAG ? J : R * J)) + g;
    double cw[P::NF];
#pragma unroll
    for (int f = 0; f < P::NF; ++f) {
        const int col = (int)(8 * blk(f)) + g;
        cw[f] = (col < (int)p && job.shift != nullptr) ? job.shift[(uint64_t)ui.r * p + col] : 0.0;
    }
    double acc[P::NACC][2], sums[P::NSUM];
#pragma unroll
    for (int i = 0; i < P::NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
    for (int i = 0; i < P::NSUM; ++i) sums[i] = 0.0;
    const uint32_t n_stages = (ui.rows + SROWS - 1) / SROWS;
    for (uint32_t sidx = 0; sidx < n_stages; ++sidx) {
        wait(slot, ph);
        const double* st = sm + slot * slot_elems + kk * pitch;
        const uint32_t s0 = slot;
        consume_stage_p<SROWS, P, SUMS>(acc, sums, st, pitch, colI, colJ, cw, [&]() { release(s0); });
        if (++slot == geo.ring) slot = 0, ph ^= 1;
    }
    double* out = job.tile_partials + ui.t * partial_len(p);
    write_items_seq<P>(out, p, nb, g, kk, acc, blk, std::make_integer_sequence<int, P::NACC>{});
    if (SUMS) {
#pragma unroll
        for (int k = 0; k < P::NSUM; ++k) {
            sums[k] += __shfl_xor_sync(0xffffffffu, sums[k], 1);
            sums[k] += __shfl_xor_sync(0xffffffffu, sums[k], 2);
        }
        if (kk == 0) {
#pragma unroll
            for (int k = 0; k < P::NSUM; ++k) {
                const int col = (int)(8 * blk(P::SUM0 + k)) + g;
                if (col < (int)p) out[col] = sums[k];
            }
        }
    }
}

// SROWS = rows per ring stage (compile-time, so a stage is one straight-line program with
// the next k-step's fragment loads issued under the current k-step's DMMAs).  Launched with
// cluster dimension geo.csize (1 = no cluster).
// Warps [0, consumers) consume; warp `consumers` is the producer; any further warps (the
// rest of the producer warpgroup of k_widep_wg) follow the producer's unit sequence without
// issuing anything, so every collective (barrier.sync 1, barrier.cluster) sees all threads.
template <int SROWS, int R, bool WG, bool BAL = false>
__device__ __forceinline__ void widep_body(const TileJob& job, const WideGeom& geo, uint32_t tile_rows, double* sm) {
    // ring x (SROWS x pitch) | kSlack doubles | full[ring] | empty[ring]
    const uint32_t p = geo.p, pitch = geo.pitch, nb = geo.nb, ring = geo.ring, K = geo.csize;
    const uint32_t slot_elems = SROWS * pitch;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + ring * slot_elems + kSlack);
    uint64_t* empty = full + ring;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t consumers = geo.consumers;
    // even p: one TMA bulk copy per row (rows 16-byte aligned when the base is); odd p: rows
    // are 8 (mod 16) bytes long, so row PAIRS are copied (pitch = p, unpadded) and an odd last
    // row goes as p - 1 doubles + 1 plain store; otherwise (base not 16-byte aligned, or an
    // odd p stage starting on an odd row) 8-byte cp.async from all lanes, waited on by the
    // producer itself.  `full` always expects one arrival (the producer's lane 0).
    const bool even_p = (p % 2 == 0);
    // unit u = (tile u / m, cluster part u % m) covers groups [(u % m) K, (u % m + 1) K) of
    // the tile; cluster c (K consecutive CTAs) runs units c, c + n_clusters, ... so the m
    // parts of a tile start side by side
    const uint32_t rank = K > 1 ? cluster_rank() : 0;
    const uint32_t m = geo.cpt;
    const uint64_t units = (job.tile_end - job.tile_begin) * m;
    const uint64_t u_first = blockIdx.x / K, u_step = gridDim.x / K;
    __shared__ uint64_t s_claim[2];
    // unit -> (tile, group): static order (u / m, (u % m) K + rank), or claimed (role 0: the
    // tile, group = rank; role 1: tile * n_groups + group)
    auto next_unit = [&](uint64_t& u, uint32_t it) -> bool {
        if (geo.claim) {
            u = acquire_unit(job, geo, K, it, s_claim);
            return u != kNoUnit;
        }
        if (it > 0) u += u_step;
        return u < units;
    };
    auto unit_tile = [&](uint64_t u) -> uint64_t {
        return job.tile_begin + (geo.claim ? (geo.role == 0 ? u : u / geo.n_groups) : u / m);
    };
    auto unit_group = [&](uint64_t u) -> uint32_t {
        return geo.claim ? (geo.role == 0 ? rank : (uint32_t)(u % geo.n_groups)) : (uint32_t)(u % m) * K + rank;
    };

    // the column pad [p, pitch) of every slot is never written by the copies: zero it once
    for (uint32_t i = threadIdx.x; i < ring * SROWS * (pitch - p); i += blockDim.x) {
        const uint32_t row = i / (pitch - p), col = p + i % (pitch - p);
        sm[row * pitch + col] = 0.0;
    }
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < ring; ++s) {
            mbar_init(&full[s], 1u);
            mbar_init(&empty[s], consumers * K);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // every CTA's barriers are initialised before any peer multicasts into it or arrives on it
    if (K > 1) cluster_sync_all(); else __syncthreads();

    uint32_t slot = 0, ph = 0;  // ring position, advanced once per stage
    if (warp >= (int)consumers) {
        // ---------------- producer ----------------
        if (WG) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
        const uint16_t mask = (uint16_t)((1u << K) - 1);
        uint64_t u = u_first;
        for (uint32_t it = 0; next_unit(u, it); ++it) {
            if (warp != (int)consumers) continue;  // idle warps of the producer warpgroup
            const UnitInfo ui = unit_info(job, geo, tile_rows, unit_tile(u));
            const uint32_t n_stages = (ui.rows + SROWS - 1) / SROWS;
            const double* crow = job.shift != nullptr ? job.shift + (uint64_t)ui.r * p : nullptr;
            for (uint32_t sidx = 0; sidx < n_stages; ++sidx) {
                // all K x C consumer warps of the cluster are done with this slot everywhere
                mbar_wait_cluster(&empty[slot], ph ^ 1);
                const uint32_t r0 = sidx * SROWS;
                const uint32_t vrows = ui.rows - r0 < SROWS ? ui.rows - r0 : SROWS;
                double* dst = sm + slot * slot_elems;
                const double* src = ui.tile + (uint64_t)r0 * p;
                // rows past the tile end hold the shift row, so x - c = 0 there (plain local
                // stores, ordered before the release of this lane's arrive below)
                for (uint32_t rr = vrows; rr < SROWS; ++rr)
                    for (uint32_t j = lane; j < p; j += 32) dst[rr * pitch + j] = crow ? crow[j] : 0.0;
                const bool aligned = (reinterpret_cast<uintptr_t>(src) % 16) == 0;
                if (!even_p && aligned && (vrows & 1) && lane == 0)  // odd last row: its last double
                    dst[(vrows - 1) * pitch + p - 1] = src[(uint64_t)(vrows - 1) * p + p - 1];
                __syncwarp();
                if (aligned && even_p) {
                    if (lane == 0) {
                        // this CTA receives every valid row of the stage, from all K producers
                        mbar_arrive_expect_tx(&full[slot], vrows * p * 8);
                        if (K > 1) {
                            for (uint32_t rr = rank; rr < vrows; rr += K)
                                bulk_g2s_mc(dst + rr * pitch, src + (uint64_t)rr * p, p * 8, &full[slot], mask);
                        } else {
                            for (uint32_t rr = 0; rr < vrows; ++rr)
                                bulk_g2s(dst + rr * pitch, src + (uint64_t)rr * p, p * 8, &full[slot]);
                        }
                    }
                } else if (aligned) {  // odd p, pitch == p: pairs of rows are 16-byte multiples
                    if (lane == 0) {
                        const uint32_t npairs = vrows / 2;
                        const bool odd_last = vrows & 1;
                        mbar_arrive_expect_tx(&full[slot], npairs * 16 * p + (odd_last ? 8 * (p - 1) : 0));
                        for (uint32_t i = rank; i < npairs; i += K) {
                            if (K > 1)
                                bulk_g2s_mc(dst + 2 * i * pitch, src + (uint64_t)2 * i * p, p * 16, &full[slot], mask);
                            else
                                bulk_g2s(dst + 2 * i * pitch, src + (uint64_t)2 * i * p, p * 16, &full[slot]);
                        }
                        if (odd_last && npairs % K == rank) {
                            double* d = dst + (vrows - 1) * pitch;
                            const double* g = src + (uint64_t)(vrows - 1) * p;
                            if (K > 1) bulk_g2s_mc(d, g, (p - 1) * 8, &full[slot], mask);
                            else bulk_g2s(d, g, (p - 1) * 8, &full[slot]);
                        }
                    }
                } else {
                    // every CTA stages its own copy (no multicast), then arrives once complete
                    for (uint32_t rr = 0; rr < vrows; ++rr)
                        for (uint32_t j = lane; j < p; j += 32) cp_async8(dst + rr * pitch + j, src + (uint64_t)rr * p + j);
                    asm volatile("cp.async.wait_all;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_local(&full[slot]);
                }
                if (++slot == ring) slot = 0, ph ^= 1;
            }
        }
    } else {
        // ---------------- consumers ----------------
        if (WG) asm volatile("setmaxnreg.inc.sync.aligned.u32 152;\n" ::: "memory");
        const int g = lane >> 2, kk = lane & 3;
        const uint64_t E = partial_len(p);
        uint64_t u = u_first;
        for (uint32_t it = 0; next_unit(u, it); ++it) {
            const UnitInfo ui = unit_info(job, geo, tile_rows, unit_tile(u));
            const uint32_t grp = unit_group(u);
            if constexpr (BAL) {
            const uint32_t item = __ldg(geo.items + grp * consumers + warp);
            const uint32_t I = (item >> 11) & 0xfff, J = item & 0x7ff, kind = (item >> 24) & 7;
            const bool sums = item & kSumsBit;
            auto wait = [&](uint32_t s, uint32_t phase) { mbar_wait(&full[s], phase); };
            auto release = [&](uint32_t s) {
                __syncwarp();
                if ((uint32_t)lane < K) mbar_arrive_cluster(&empty[s], lane);
            };
            // warp-uniform dispatch to the item's straight-line program; an idle (padding) warp of
            // the last group keeps the ring protocol only
            if (item & kIdle) {
                const uint32_t n_stages = (ui.rows + SROWS - 1) / SROWS;
                for (uint32_t sidx = 0; sidx < n_stages; ++sidx) {
                    wait(slot, ph);
                    release(slot);
                    if (++slot == ring) slot = 0, ph ^= 1;
                }
            } else if (kind == kRect) {
                if (sums) run_item<SROWS, R, Prog<R, kRect>, true>(job, geo, ui, I, J, g, kk, sm, slot_elems, slot, ph, wait, release);
                else run_item<SROWS, R, Prog<R, kRect>, false>(job, geo, ui, I, J, g, kk, sm, slot_elems, slot, ph, wait, release);
            } else if constexpr (BAL && R == 4) {  // the balanced decomposition's kinds (make_items_balanced8)
                if (kind == kRectCol3) {
                    if (sums) run_item<SROWS, R, Prog<R, kRectCol3>, true>(job, geo, ui, I, J, g, kk, sm, slot_elems, slot, ph, wait, release);
                    else run_item<SROWS, R, Prog<R, kRectCol3>, false>(job, geo, ui, I, J, g, kk, sm, slot_elems, slot, ph, wait, release);
                } else if (kind == kRectRow3) {
                    run_item<SROWS, R, Prog<R, kRectRow3>, false>(job, geo, ui, I, J, g, kk, sm, slot_elems, slot, ph, wait, release);
                } else if (kind == kDiagCol) {
                    if (sums) run_item<SROWS, R, Prog<R, kDiagCol>, true>(job, geo, ui, I, J, g, kk, sm, slot_elems, slot, ph, wait, release);
                    else run_item<SROWS, R, Prog<R, kDiagCol>, false>(job, geo, ui, I, J, g, kk, sm, slot_elems, slot, ph, wait, release);
                } else {
                    run_item<SROWS, R, Prog<R, kDiagRow>, false>(job, geo, ui, I, J, g, kk, sm, slot_elems, slot, ph, wait, release);
                }
            }
            } else {
            const uint32_t item = __ldg(geo.items + grp * consumers + warp);
            const bool idle = item & kIdle;
            const uint32_t I = (item >> 11) & 0xfff, J = item & 0x7ff;
            // fragment a reads column colI + 8a (a < R, rectangle I) or colJ + 8(a-R) (rectangle
            // J); columns past p read the zero pad with c = 0, rows past the tile end read c
            const int colI = (int)(8 * R * I) + g, colJ = (int)(8 * R * J) + g;
            const bool sums_here = !idle && I == 0;  // rectangle (0, J) sums rectangle J's columns
            double cw[2 * R];
#pragma unroll
            for (int a = 0; a < 2 * R; ++a) {
                const int col = a < R ? colI + 8 * a : colJ + 8 * (a - R);
                cw[a] = (!idle && col < (int)p && job.shift != nullptr) ? job.shift[(uint64_t)ui.r * p + col] : 0.0;
            }
            double acc[R * R][2], sums[R];
#pragma unroll
            for (int i = 0; i < R * R; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
            for (int i = 0; i < R; ++i) sums[i] = 0.0;

            const uint32_t n_stages = (ui.rows + SROWS - 1) / SROWS;
            for (uint32_t sidx = 0; sidx < n_stages; ++sidx) {
                mbar_wait(&full[slot], ph);
                // an idle (padding) warp of the last group keeps the ring protocol only
                const double* st = sm + slot * slot_elems + kk * pitch;
                auto release = [&]() {
                    __syncwarp();
                    if ((uint32_t)lane < K) mbar_arrive_cluster(&empty[slot], lane);
                };
                if (sums_here)
                    consume_stage_rect<SROWS, R, true>(acc, sums, st, pitch, colI, colJ, cw, release);
                else if (!idle)
                    consume_stage_rect<SROWS, R, false>(acc, sums, st, pitch, colI, colJ, cw, release);
                else
                    release();
                if (++slot == ring) slot = 0, ph ^= 1;
            }

            // ---- epilogue: disjoint canonical entries of the tile partial ----
            double* out = job.tile_partials + ui.t * E;
            if (!idle) {
#pragma unroll
                for (int a = 0; a < R; ++a)
#pragma unroll
                    for (int b = 0; b < R; ++b) {
                        const uint32_t A = R * I + a, B = R * J + b;
                        if (A <= B && B < nb) write_block(out, p, A, B, g, kk, acc[a * R + b]);
                    }
            }
            if (sums_here) {
#pragma unroll
                for (int a = 0; a < R; ++a) {
                    sums[a] += __shfl_xor_sync(0xffffffffu, sums[a], 1);
                    sums[a] += __shfl_xor_sync(0xffffffffu, sums[a], 2);
                }
                if (kk == 0) {
#pragma unroll
                    for (int a = 0; a < R; ++a)
                        if (colJ + 8 * a < (int)p) out[colJ + 8 * a] = sums[a];
                }
            }
            }
        }
    }
    // no CTA leaves while a peer may still multicast into it or arrive on its barriers
    if (K > 1) cluster_sync_all();
}

template <int SROWS, int R>
__global__ void __maxnreg__(168) k_widep(TileJob job, WideGeom geo, uint32_t tile_rows) {
    extern __shared__ __align__(128) double sm[];
    widep_body<SROWS, R, false>(job, geo, tile_rows, sm);
}

// Three consumer warpgroups (12 warps, three per SM sub-partition) + one producer warpgroup
// in a 512-thread CTA, one CTA per SM: launched at 128 registers per thread, the producer
// warpgroup hands registers to the consumers (setmaxnreg: 3 x 152 + 56 = 512 per
// sub-partition lane), which a dedicated producer warp could not do (a 13th warp would put
// four warps on one sub-partition and cap every warp at 128 registers).
constexpr uint32_t kWgConsumers = 12;
template <int SROWS, int R>
__global__ void __launch_bounds__(512, 1) k_widep_wg(TileJob job, WideGeom geo, uint32_t tile_rows) {
    extern __shared__ __align__(128) double sm[];
    widep_body<SROWS, R, true>(job, geo, tile_rows, sm);
}
// k_widep_wg with the item kinds of the balanced decomposition (make_items_balanced8; R = 4).
// A kernel of its own: compiling the extra programs into k_widep_wg cost its plain-rectangle
// plans 1-5 % (p = 256 / 512 / 1024).
template <int SROWS>
__global__ void __launch_bounds__(512, 1) k_widep_wgb(TileJob job, WideGeom geo, uint32_t tile_rows) {
    extern __shared__ __align__(128) double sm[];
    widep_body<SROWS, 4, true, true>(job, geo, tile_rows, sm);
}

// Rectangles (I <= J) of the nr x nr rectangle grid, dealt to n_groups groups of
// `consumers` warps (the last groups padded with idle warps).
std::vector<uint32_t> make_items(uint32_t nr, uint32_t consumers, uint32_t n_groups) {
    std::vector<uint32_t> items;
    for (uint32_t I = 0; I < nr; ++I)
        for (uint32_t J = I; J < nr; ++J) items.push_back(item_word(kRect, I, J, I == 0));
    while (items.size() < (size_t)n_groups * consumers) items.push_back(kIdle);
    return items;
}

// The balanced decomposition for 8 x 8 groups of 4 blocks (p = 249..256, C5's width) in three
// 12-warp groups: the plain plan gives every SM sub-partition three 16-DMMA rectangles (48 DMMA
// per k-step) although only 528 of the 576 blocks are upper-triangle blocks (44 per
// sub-partition).  Here the 8 diagonal groups take their 10 upper blocks plus one 4-block strip
// each (14 DMMA), cut from the rectangles (I, I+1) (column strips, leaving 4 x 3 rectangles)
// and (5, 7) (a row strip, leaving a 3 x 4): 20 rectangles of 16, 8 trimmed ones of 12 and 8
// diagonal items of 14, dealt {16, 16, 12} to 8 sub-partitions and {16, 14, 14} to 4 — 44 DMMA
// per k-step on every sub-partition, no mirrored block, every column summed once.
std::vector<uint32_t> make_items_balanced8() {
    const uint32_t nr = 8, R = 4;
    std::vector<uint32_t> t16, t12, d14;
    auto split = [](uint32_t I, uint32_t J) { return J == I + 1 || (I == 5 && J == 7); };
    for (uint32_t I = 0; I < nr; ++I)
        for (uint32_t J = I + 1; J < nr; ++J)
            if (!split(I, J)) t16.push_back(item_word(kRect, I, J, I == 0));
    for (uint32_t I = 0; I + 1 < nr; ++I) {
        t12.push_back(item_word(kRectCol3, I, I + 1, I == 0));            // blocks 4(I+1) .. 4(I+1)+2
        d14.push_back(item_word(kDiagCol, I, R * (I + 1) + R - 1, I == 0));  // + column block 4(I+1)+3
    }
    t12.push_back(item_word(kRectRow3, 5, 7, false));            // rows 20..22 x group 7
    d14.push_back(item_word(kDiagRow, 7, R * 5 + R - 1, false));  // group 7 + row block 23
    // the items that add column sums first, so they land on distinct sub-partitions
    std::stable_partition(t16.begin(), t16.end(), [](uint32_t w) { return (w & kSumsBit) != 0; });
    std::vector<std::vector<uint32_t>> sub(12);  // sub-partition k: group k / 4, warps k % 4 + 4m
    for (uint32_t k = 0; k < 12; ++k) sub[k].push_back(t16[k]);
    for (uint32_t k = 0; k < 8; ++k) sub[k].push_back(t16[12 + k]);
    // t12[0] (sums) away from the sub-partitions holding a summing rectangle (0..5)
    for (uint32_t k = 0; k < 8; ++k) sub[k].push_back(t12[(k + 2) % 8]);
    for (uint32_t k = 8; k < 12; ++k) {
        sub[k].push_back(d14[2 * (k - 8)]);
        sub[k].push_back(d14[2 * (k - 8) + 1]);
    }
    std::vector<uint32_t> tab(3 * 12, kIdle);
    for (uint32_t k = 0; k < 12; ++k)
        for (uint32_t m = 0; m < 3; ++m) tab[(k / 4) * 12 + m * 4 + k % 4] = sub[k][m];
    return tab;
}

uint32_t env_u32(const char* name, uint32_t dflt) {
    const char* v = getenv(name);
    return v ? (uint32_t)atoi(v) : dflt;
}

// One launch geometry per (device, p): chosen once from the occupancy calculator, its
// rectangle table kept on the device for the life of the process.
struct Plan {
    int device = -1;
    bool wg = false;  // k_widep_wg (12 consumer warps) instead of k_widep
    bool bal = false;  // k_widep_wgb: the balanced decomposition (8 x 8 groups of 4 blocks)
    uint32_t p = 0, srows = 0, R = 0, grid_cap = 0;  // grid_cap = clusters in flight
    size_t smem = 0;
    WideGeom geo{};
    uint32_t resident = 0;  // CTAs per SM the plan targets
    // CTA slots the clustered plan leaves idle (cluster placement) run a cluster-less plan on
    // a side stream over a proportional share of the tiles
    bool has_spare = false;
    uint32_t spare_ctas = 0;
    size_t spare_smem = 0;
    WideGeom spare_geo{};
};
std::mutex g_plan_mu;
std::vector<Plan> g_plans;

bool balanced_applies(bool wg, uint32_t R, uint32_t nr) {
    return wg && R == 4 && nr == 8 && !env_u32("SSTAT_WIDEP_NOBALANCE", 0);
}
template <int SROWS, int R>
void (*kernel_of(bool wg, bool bal))(TileJob, WideGeom, uint32_t) {
    if constexpr (R == 4)
        if (bal) return k_widep_wgb<SROWS>;
    return wg ? k_widep_wg<SROWS, R> : k_widep<SROWS, R>;
}

template <int SROWS, int R>
cudaError_t make_plan(int device, WideGeom geo, Plan& out, bool force_nocluster, bool wg) {
    const bool bal = balanced_applies(wg, R, geo.nr);
    auto kern = kernel_of<SROWS, R>(wg, bal);
    if (wg) geo.consumers = kWgConsumers;
    const int threads = wg ? 512 : (int)(geo.consumers + 1) * 32;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    // the opt-in limit only caps what a launch may request; set it once to the maximum so
    // plans with different rings never invalidate each other
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    const size_t max_dyn = 227 * 1024 - fa.sharedSizeBytes;  // the claim slots are static
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_dyn);
    if (e != cudaSuccess) return e;
    // deepest ring (2..4 stages) that keeps the target CTAs per SM (2 for 4-warp groups, so
    // two groups share an SM's four DMMA units; 1 for 8-warp groups)
    // smaller rectangles need fewer registers: three 4-warp CTAs per SM
    const int want = wg ? 1 : (int)env_u32("SSTAT_WIDEP_PERSM", geo.consumers == 4 ? (R == 4 ? 2 : 3) : 1);
    size_t smem = 0;
    int per_sm = 0;
    for (uint32_t ring = env_u32("SSTAT_WIDEP_RING", wg ? 12 : 4); ring >= 2; --ring) {
        geo.ring = ring;
        smem = sizeof(double) * (ring * SROWS * geo.pitch + kSlack) + 2 * ring * sizeof(uint64_t);
        if (smem > max_dyn) continue;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
        if (e != cudaSuccess) return e;
        if (per_sm >= want) break;
    }
    if (per_sm < 1) return cudaErrorInvalidConfiguration;

    // Cluster size K: every candidate K >= 2 (a tile's groups share its stream through the
    // multicast; K = 1 only when the tile has one group or SSTAT_WIDEP_NOCLUSTER), scored by
    // the useful consumer warps it keeps resident = clusters in flight x K x C x the real
    // share of the groups.  The calculator's cluster placement (GPC sizes) and the idle
    // padding of K * m groups are what separate the candidates.
    const uint32_t items = geo.nr * (geo.nr + 1) / 2;
    const uint32_t groups = (items + geo.consumers - 1) / geo.consumers;
    const uint32_t kmax = std::min<uint32_t>(env_u32("SSTAT_WIDEP_MAXCLUSTER", 16), groups);
    const bool nocluster = force_nocluster || env_u32("SSTAT_WIDEP_NOCLUSTER", 0) != 0 || groups == 1;
    struct Cand {
        WideGeom g;
        int clusters;
        double value;  // useful consumer warps resident: clusters x K x C x items / (n_groups C)
    };
    std::vector<Cand> cands;
    const uint32_t kforce = env_u32("SSTAT_WIDEP_CLUSTER", 0);
    for (uint32_t K = nocluster ? 1 : 2; K <= (nocluster ? 1 : kmax); ++K) {
        if (kforce && K != kforce) continue;
        WideGeom g = geo;
        g.csize = K;
        g.cpt = (groups + K - 1) / K;
        g.n_groups = g.csize * g.cpt;
        int clusters = 0;
        if (K == 1) {
            clusters = sms_of(device) * std::min(per_sm, want);
        } else {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = K;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.blockDim = dim3(threads);
            cfg.dynamicSmemBytes = smem;
            cfg.gridDim = dim3(K * 64);
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess) {
                (void)cudaGetLastError();
                continue;
            }
        }
        if (clusters > 0) cands.push_back({g, clusters, (double)clusters * K * items / g.n_groups});
    }
    if (cands.empty()) return cudaErrorInvalidConfiguration;
    // the largest cluster within 4% of the best value: fewer clusters per tile means fewer
    // HBM / L2 re-reads of the tile (one cluster per tile reads it from HBM exactly once)
    double top = 0;
    for (const Cand& c : cands) top = std::max(top, c.value);
    const Cand* pick = nullptr;
    for (const Cand& c : cands)
        if (c.value >= 0.96 * top && (!pick || c.g.cpt < pick->g.cpt ||
                                      (c.g.cpt == pick->g.cpt && c.value > pick->value)))
            pick = &c;
    WideGeom best = pick->g;
    const uint32_t best_clusters = (uint32_t)pick->clusters;

    std::vector<uint32_t> tab = make_items(best.nr, best.consumers, best.n_groups);
    if (bal && best.n_groups == 3) tab = make_items_balanced8();
    uint32_t* d_items = nullptr;
    e = cudaMalloc(&d_items, tab.size() * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
    e = cudaMemcpy(d_items, tab.data(), tab.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    best.items = d_items;
    out.device = device;
    out.wg = wg;
    out.bal = bal;
    out.p = geo.p;
    out.srows = SROWS;
    out.R = R;
    out.grid_cap = best_clusters;
    out.resident = (uint32_t)std::min(per_sm, want);
    out.smem = smem;
    out.geo = best;
    if (getenv("SSTAT_DEBUG"))
        fprintf(stderr, "k_widep%s<%d,%d>: p=%u C=%u groups=%u/%u cluster=%u x %u ring=%u smem=%zu per_sm=%d clusters=%u\n",
                wg ? "_wg" : "", SROWS, R, geo.p, best.consumers, groups, best.n_groups, best.csize, best.cpt, best.ring, smem, per_sm,
                best_clusters);
    return cudaSuccess;
}

template <int SROWS, int R>
cudaError_t launch_plan(const TileJob& job, const Plan& pl, cudaStream_t stream) {
    const uint64_t tiles = job.tile_end - job.tile_begin;
    if (tiles == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = pl.geo.csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(pl.wg ? 512 : (pl.geo.consumers + 1) * 32);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const uint64_t units = tiles * pl.geo.cpt;
    cfg.gridDim = dim3((unsigned)(std::min<uint64_t>(units, pl.grid_cap) * pl.geo.csize));
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel_of<SROWS, R>(pl.wg, pl.bal), job, pl.geo,
                                       widep_tile_rows(pl.geo.p));
    if (e != cudaSuccess) return e;
    if (job.launched && pl.geo.role == 0)  // the clustered launch (the spare one is its helper)
        *job.launched = (const void*)kernel_of<SROWS, R>(pl.wg, pl.bal);
    return cudaGetLastError();
}

template <int SROWS>
cudaError_t make_plan_r(int device, const WideGeom& geo, Plan& out, bool force_nocluster, bool wg) {
    return geo.R == 2 ? make_plan<SROWS, 2>(device, geo, out, force_nocluster, wg)
           : geo.R == 3 ? make_plan<SROWS, 3>(device, geo, out, force_nocluster, wg)
                        : make_plan<SROWS, 4>(device, geo, out, force_nocluster, wg);
}
cudaError_t make_plan_any(int device, const WideGeom& geo, uint32_t srows, Plan& out, bool force_nocluster,
                          bool wg) {
    return srows == 16 ? make_plan_r<16>(device, geo, out, force_nocluster, wg)
           : srows == 8 ? make_plan_r<8>(device, geo, out, force_nocluster, wg)
                        : make_plan_r<4>(device, geo, out, force_nocluster, wg);
}
template <int SROWS>
cudaError_t launch_plan_r(const TileJob& job, const Plan& pl, cudaStream_t stream) {
    return pl.R == 2 ? launch_plan<SROWS, 2>(job, pl, stream)
           : pl.R == 3 ? launch_plan<SROWS, 3>(job, pl, stream)
                       : launch_plan<SROWS, 4>(job, pl, stream);
}
cudaError_t launch_plan_any(const TileJob& job, const Plan& pl, cudaStream_t stream) {
    return pl.srows == 16 ? launch_plan_r<16>(job, pl, stream)
           : pl.srows == 8 ? launch_plan_r<8>(job, pl, stream)
                           : launch_plan_r<4>(job, pl, stream);
}

// Rectangle side R (8-column blocks): the fewest DMMA-equivalents per useful block over the
// warp slots of a tile (idle padding included), R*R DMMA + R/4 for the 2R shift DADDs per
// warp k-step; ties go to the larger R (fewer groups re-reading the tile).
uint32_t choose_r(uint32_t nb, uint32_t consumers) {
    uint32_t best = 4;
    double best_cost = 0;
    for (uint32_t R : {4u, 3u, 2u}) {
        const uint32_t nr = (nb + R - 1) / R, items = nr * (nr + 1) / 2;
        const uint32_t slots = (items + consumers - 1) / consumers * consumers;
        // 2x2 rectangles load one fragment per DMMA and need twice the groups per tile: measured
        // 15-25 % below this model from p = 136 on (profiles/r01_p_sweep.log), hence the 1.25
        // (not at nb <= 12, where they measured best)
        // 3x3 rectangles: 9 DMMA per 6 fragments, measured ~15 % below the model in 4-warp
        // groups where the costs are close (p = 200, 296, 352) and ~5 % in 12-warp groups
        // (p = 352 vs 296: profiles/r01_k2_wg_sweep.log)
        const double pen = R == 2 && nb > 12 ? 1.25 : R == 3 ? (consumers >= 12 ? 1.05 : 1.15) : 1.0;
        const double cost = slots * (R * R + R / 4.0) / (nb * (nb + 1) / 2.0) * pen;
        if (best_cost == 0 || cost < 0.97 * best_cost) best = R, best_cost = cost;
    }
    return best;
}

// Share of the DMMA blocks a tile's warp slots compute (groups x warps x R^2, idle padding,
// blocks past p and mirrored diagonal blocks included) that are upper-triangle blocks.
double plan_efficiency(const Plan& pl) {
    const double useful = pl.geo.nb * (pl.geo.nb + 1) / 2.0;
    return useful / ((double)pl.geo.n_groups * pl.geo.consumers * pl.geo.R * pl.geo.R);
}
void free_plan(const Plan& pl) {
    cudaFree(const_cast<uint32_t*>(pl.geo.items));
    if (pl.has_spare) cudaFree(const_cast<uint32_t*>(pl.spare_geo.items));
}

// The launch geometry for width p with the 4/8-warp kernel (wg = false) or k_widep_wg, plus the
// cluster-less side plan for the CTA slots its cluster placement leaves idle.
cudaError_t build_plan(int device, uint32_t p, uint32_t srows, bool wg, Plan& pl, uint32_t force_r = 0) {
    WideGeom geo{};
    geo.p = p;
    geo.nb = (p + 7) / 8;
    geo.R = env_u32("SSTAT_WIDEP_R", force_r ? force_r : choose_r(geo.nb, wg ? kWgConsumers : 4));
    if (geo.R < 2 || geo.R > 4) geo.R = 4;
    geo.nr = (geo.nb + geo.R - 1) / geo.R;
    // pitch = 4 (mod 16) doubles puts the 4 rows of a k-step in distinct 32-byte bank
    // groups, so each half-warp fragment read is one conflict-free wavefront
    // (odd p: unpadded, the stage is copied as row pairs; see k_widep)
    geo.pitch = p % 2 ? p : ((p + 15) / 16) * 16 + 4;
    // 4-warp groups (two CTAs per SM) leave at most 3 idle rectangles per tile, 8-warp
    // groups up to 7 but re-read less; the multicast makes the extra groups cheap
    // (measured: 4-warp groups win up to p = 512, +5 % at 384 and +14 % at 512; even at 1024)
    const uint32_t items = geo.nr * (geo.nr + 1) / 2;
    geo.consumers = std::min<uint32_t>(12, std::max<uint32_t>(1, env_u32("SSTAT_WIDEP_CONSUMERS", items <= 300 ? 4 : 8)));
    // 12-consumer-warp CTAs: registers cap them at 8-row stages for 4x4 rectangles
    if (wg && geo.R == 4 && srows > 8 && !getenv("SSTAT_WIDEP_SROWS")) srows = 8;
    cudaError_t e = make_plan_any(device, geo, srows, pl, false, wg);
    if (e != cudaSuccess) return e;
    const uint64_t slots = (uint64_t)sms_of(device) * pl.resident;
    const uint64_t used = (uint64_t)pl.grid_cap * pl.geo.csize;
    // CTA slots the cluster placement leaves idle get a cluster-less launch (>= 4 % of
    // the slots, whole-tile clusters only)
    if (pl.geo.csize > 1 && pl.geo.cpt == 1 && slots > used && 25 * (slots - used) >= slots) {
        Plan ps;
        WideGeom g2 = geo;
        g2.consumers = pl.geo.consumers;
        e = make_plan_any(device, g2, srows, ps, true, wg);
        if (e != cudaSuccess) return e;
        pl.has_spare = true;
        pl.spare_ctas = (uint32_t)(slots - used);
        pl.spare_smem = ps.smem;
        pl.spare_geo = ps.geo;
    }
    return cudaSuccess;
}

}  // namespace

uint32_t widep_tile_rows(uint32_t) { return 32768; }

namespace {
cudaError_t launch_forked(const TileJob& job, const Plan& pl, cudaStream_t stream, uint32_t* kernels);
}

cudaError_t launch_widep(const TileJob& job, int, cudaStream_t stream, uint32_t* kernels) {
    if (kernels) *kernels = 1;
    const uint32_t p = job.p;
    if (p > kMaxWideP || p < 2) return cudaErrorInvalidValue;
    int device = 0;
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return e;
    // stage height: 16 rows up to p = 256, then 8, then 4 (a stage stays ~33 KB)
    uint32_t srows = p <= 256 ? 16 : p <= 512 ? 8 : 4;
    if (const uint32_t e = env_u32("SSTAT_WIDEP_SROWS", 0)) srows = e >= 16 ? 16 : e >= 8 ? 8 : 4;
    // any experiment override: the plan is built for this call only (not cached)
    bool tuned = false;
    for (const char* knob : {"SSTAT_WIDEP_CONSUMERS", "SSTAT_WIDEP_NOCLUSTER", "SSTAT_WIDEP_MAXCLUSTER",
                             "SSTAT_WIDEP_CLUSTER", "SSTAT_WIDEP_RING", "SSTAT_WIDEP_SROWS", "SSTAT_WIDEP_PERSM",
                             "SSTAT_WIDEP_R", "SSTAT_WIDEP_WG"})
        tuned = tuned || getenv(knob) != nullptr;
    Plan pl;
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        bool found = false;
        if (!tuned)
            for (const Plan& q : g_plans)
                if (q.device == device && q.p == p) pl = q, found = true;
        if (!found) {
            // the 12-consumer-warp kernel (three warps per SM sub-partition instead of two)
            // unless its useful share of the computed DMMA blocks is more than 5 % below the
            // 4-warp kernel's (measured, profiles/r01_k2_wg_sweep.log: +8-17 % at p = 136-144,
            // +4 % at 256, +8 % at 416-448, +18-22 % at 640-1024; worse at p <= 128, at p = 168
            // (its 4x4 rectangles: 60 % useful blocks against 92 % for 3x3 in 4-warp groups),
            // 296 and 384)
            const char* wg_env = getenv("SSTAT_WIDEP_WG");
            const uint32_t nb = (p + 7) / 8;
            if (wg_env) {
                e = build_plan(device, p, srows, atoi(wg_env) != 0, pl);
            } else if (nb <= 16) {
                e = build_plan(device, p, srows, false, pl);
            } else if ((nb <= 25 && nb != 18) || nb == 29 || nb == 30) {
                // p = 129-200 except 137-144, and p = 225-240: the 4-warp kernel with 3x3
                // rectangles beats the efficiency model's pick (measured,
                // profiles/r01_k2_r_window.log: p = 130 / 136 / 152 / 160 / 176 / 184 / 192 / 200
                // +12 / +11 / +26 / +24 / +26 / +8 / +8 / +8 %, p = 232 / 240 +11 / +12 %;
                // p = 144, 216, 264-320 keep the model's plan)
                e = build_plan(device, p, srows, false, pl, 3);
            } else {
                Plan pc, pw;
                e = build_plan(device, p, srows, false, pc);
                if (e == cudaSuccess) e = build_plan(device, p, srows, true, pw);
                if (e == cudaSuccess) {
                    const bool use_wg = plan_efficiency(pw) >= 0.95 * plan_efficiency(pc);
                    pl = use_wg ? pw : pc;
                    free_plan(use_wg ? pc : pw);
                    if (getenv("SSTAT_DEBUG"))
                        fprintf(stderr, "k_widep: p=%u efficiency 4-warp %.3f, 12-warp %.3f -> %s\n", p,
                                plan_efficiency(pc), plan_efficiency(pw), use_wg ? "k_widep_wg" : "k_widep");
                }
            }
            if (e != cudaSuccess) return e;
            if (!tuned) g_plans.push_back(pl);
        }
    }
    e = launch_forked(job, pl, stream, kernels);
    if (tuned) free_plan(pl);  // experiment plans are not cached (cudaFree waits for the launches)
    return e;
}

namespace {
cudaError_t launch_forked(const TileJob& job, const Plan& pl, cudaStream_t stream, uint32_t* kernels) {
    if (!pl.has_spare || !job.claim || !job.side || job.tile_end - job.tile_begin < 2 ||
        env_u32("SSTAT_WIDEP_SPARE", 1) == 0)
        return launch_plan_any(job, pl, stream);
    cudaError_t e;
    // fork: the clustered plan on `stream` and the cluster-less plan on the caller's side
    // stream claim tiles / units dynamically from one word (claim_unit); if the side launch
    // cannot run alongside, the clustered one simply takes every tile.  Join before returning.
    unsigned long long* W = job.claim;  // the caller's scratch word (one launch at a time per caller)
    if ((e = cudaMemsetAsync(W, 0, sizeof *W, stream)) != cudaSuccess) return e;
    Plan pa = pl, pb = pl;
    pa.geo.claim = W;
    pa.geo.role = 0;
    pb.geo = pl.spare_geo;
    pb.geo.claim = W;
    pb.geo.role = 1;
    pb.grid_cap = pl.spare_ctas;
    pb.smem = pl.spare_smem;
    if ((e = cudaEventRecord(job.fork, stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(job.side, job.fork, 0)) != cudaSuccess) return e;
    e = launch_plan_any(job, pa, stream);
    cudaError_t e2 = launch_plan_any(job, pb, job.side);
    cudaError_t e3 = cudaEventRecord(job.join, job.side);
    if (e3 == cudaSuccess) e3 = cudaStreamWaitEvent(stream, job.join, 0);
    if (kernels) *kernels = 2;
    return e != cudaSuccess ? e : e2 != cudaSuccess ? e2 : e3;
}
}  // namespace

}  // namespace sstat_b200
