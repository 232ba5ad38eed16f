// power_sums.cuh — the hot path: one persistent streaming reduction per fit.
//
// Replaces accumulate_into / accumulate / accumulate_parallel / require_finite
// (reference proj/src/power_sums.cpp:13-90) and, fused into the same launch,
// build_normal_system + solve_gaussian (normal_backend.cpp:13-74).
//
// Data path (per CTA, one CTA per SM; shapes per degree in PsCfg):
//   feed           : one lane streams the CTA's tiles HBM -> SMEM with
//                    cp.async.bulk (TMA engine, L2 evict-first) into a
//                    STAGES-deep ring guarded by mbarriers — a producer warp
//                    (m <= 5, plus a dynamically claimed tail), or the last
//                    consumer warp to release a stage refills it (SELF_FEED,
//                    m >= 6).
//   consumers      : 7 or 8 warps; each thread takes P = 16 points of the
//                    tile (x, y via LDS.128, conflict-free) and forms its
//                    terms: for m <= 2 exactly the reference's (power *= x,
//                    rounded power * y); from m = 3 the PRODUCTS terms (the
//                    reference's powers up to x^m, exact fused-multiply-add
//                    products pw_j * y and pw_a * pw_b above x^m). Each term
//                    column is summed over the P points by a balanced tree or
//                    DFMA chains, the next tiles' sums are added, and that
//                    partial is folded into a per-thread compensated (hi, lo)
//                    pair with magnitude-ordered Fast2Sum. SPLIT (m >= 6):
//                    lane pairs exchange column sums by shuffle and each
//                    keeps half the columns' state.
//   epilogue       : warp reduce-scatter -> CTA (fixed warp order) -> global
//                    slot per CTA (and per dynamic chunk) -> the last CTA to
//                    finish (atomic ticket) reduces all slots in a fixed
//                    order, checks finiteness, writes the PowerSums image and
//                    runs the one-warp solve.
// Every reduction order is a fixed function of (n, degree, grid), so results
// are deterministic run to run; accumulate and accumulate_parallel(…, 1) are
// the same launch and therefore bit-identical (power_sums.hpp:25-31).
//
// Error bound (vs the exact sum of the kernel's own terms T_i): each fold
// adds a plain partial — the per-thread column sum over P points (tree depth
// log2 P; CL + log2(P/CL) for DFMA chains of CL products), +1 for the lane
// pair exchange, then FOLD_TILES - 1 sequential adds of further tiles' sums
// — into an error-free (Fast2Sum) compensated pair, so
//   |S_gpu - S_exact| <= gamma_L * sum|T_i| + ulp(S_exact) + O(n u^2 sum|T_i|),
//   L = PsCfg<M>::ERR_LEVELS: 5 for m <= 2, 10 for m = 3, 4, 16 for m = 5
//   (8 tiles per fold), 17 for m >= 6,
// u = 2^-53. Queryable through lsqfit_cuda_sum_error_levels() (and the terms
// through lsqfit_cuda_sum_terms()).
#pragma once

#include "common.cuh"
#include "solve.cuh"

namespace lsq {

#ifndef LSQ_PRODUCER_SLEEP
// The suspend-hint wait compiles to NANOSLEEP.SYNCS with the hint as its
// bound; A/B showed no gain, so the producer spins on try_wait by default.
#define LSQ_PRODUCER_SLEEP 0
#endif
#ifndef LSQ_PAIR_UNROLL_MIN
#define LSQ_PAIR_UNROLL_MIN 4
#endif
#ifndef LSQ_PAIR_UNROLL_MAX
#define LSQ_PAIR_UNROLL_MAX 4
#endif

#ifndef LSQ_WS_MIN
// Warp-specialised split shape from this degree (99: the self-fed shape).
// A/B against self-feed (profiles/r02_ab_warp_specialised.txt), same bits:
// n = 1e9 m = 6 / 8 / 9 / 10 3.8-5.3 / 1.3-4.5 / 3.6-3.9 / 1.5-1.8% faster,
// m = 7 and 12 within 0.7%; sustained m = 6 / 8 1.3-3.2 / 1.5-2.1%; at
// n = 1e8 m = 8 2-3% faster but m = 6 3.5-10% slower.
#define LSQ_WS_MIN 6
#endif
#ifndef LSQ_WS_CONSUMER_REGS
#define LSQ_WS_CONSUMER_REGS 240
#endif
#ifndef LSQ_WS_PRODUCER_REGS
#define LSQ_WS_PRODUCER_REGS 24  // 24 + 2 x 240 = 3 x 168: setmaxnreg moves registers within the launch allocation
#endif
#ifndef LSQ_SELF_FEED_MIN
#define LSQ_SELF_FEED_MIN 6  // A/B: self-feed 2-13% faster for m >= 5 with the reference's terms; with product terms m = 5 is 4% faster producer-fed (+ dynamic tail)
#endif
#ifndef LSQ_PS_GRIDSTRIDE_MAX
// Tiles dealt round-robin (the grid sweeps HBM together) up to this degree,
// contiguous per-CTA ranges above. Sustained A/B (50-launch blocks, n = 4e9):
// round-robin 1.2-1.7% faster for m = 1..3, neutral beyond (m = 4 with the
// reference's terms 1.7% slower; with product terms and the dynamic tail
// m = 4, 5 are 0.5-1% faster than with the contiguous deal).
#define LSQ_PS_GRIDSTRIDE_MAX 5
#endif
#ifndef LSQ_P16_MAX
#define LSQ_P16_MAX 12  // round 2 (product terms): P = 16 everywhere; the split degrees 8-11% faster than P = 8 x 12 warps
#endif

#ifndef LSQ_DYN_MAX
// Probe (tools/stream_balance.cu, 32 GiB): a static deal of the TMA-ring
// stream leaves the CTAs finishing 0.6-0.9 ms apart over 4.7 ms (per-SM
// bandwidth is not fair); a dynamic tail of 20-30% in 8-tile chunks
// recovers 3% (7.35 -> 7.58 TB/s).
#define LSQ_DYN_MAX 5  // with product terms: m = 4 7-8% (burst) / 1.3-1.8% (sustained) faster at 1e9, 4% at 1e8; m = 5 (producer-fed) 4% / 6.5% at 1e9 / 1e8
#endif
#ifndef LSQ_DYN_DEN
#define LSQ_DYN_DEN 2  // dynamic tail = tiles / LSQ_DYN_DEN
#endif
#ifndef LSQ_DYN_CHUNK
#define LSQ_DYN_CHUNK 8  // smallest chunk, tiles
#endif
#ifndef LSQ_DYN_MIN_TILES_PER_CTA
// A/B (sustained): from 128 tiles per CTA (n >= 6.8e7 points) the balance
// gains 1-4% for m <= 2; the heavier m = 3 consumer loses 6% at 1e8-1.5e8
// points to the chunk reductions and gains from ~2.5e8, hence 512 there.
#define LSQ_DYN_MIN_TILES_PER_CTA(m) ((m) <= 2 ? 128 : 512)
#endif
#ifndef LSQ_DYN_MID_TILES_PER_CTA
#define LSQ_DYN_MID_TILES_PER_CTA 1024  // below: the mid-size plan
#endif
#ifndef LSQ_DYN_MID_DEN
#define LSQ_DYN_MID_DEN 8
#endif
#ifndef LSQ_DYN_MID_CHUNK
#define LSQ_DYN_MID_CHUNK 16
#endif
#ifndef LSQ_DYN_MID_MIN_TILES
#define LSQ_DYN_MID_MIN_TILES 32
#endif
constexpr uint32_t kDynMaxChunks = 4096;    // chunk records (scratch and final-reduction bound)
constexpr uint32_t kDynEnd = 0xffffffffu;   // ring-stage tag: no more chunks

// Consumer warps of the record-combine kernel.
constexpr int kConsumerWarps = 7;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr uint32_t kPieceBytes = 16384;  // bulk-copy granule

#ifndef LSQ_CONSUMER_SLEEP
#define LSQ_CONSUMER_SLEEP 0
#endif
// Consumers waiting for a tile: spin on try_wait, or (A/B knob) try_wait with
// a suspend-time hint so the warp sleeps in hardware until the phase flips.
__device__ __forceinline__ void consumer_wait(uint64_t* bar, uint32_t parity) {
#if LSQ_CONSUMER_SLEEP
    if (mbar_try_wait(bar, parity)) return;
    const uint64_t t0 = globaltimer_ns();
    while (!mbar_try_wait_sleep(bar, parity, LSQ_CONSUMER_SLEEP)) {
        if (globaltimer_ns() - t0 > 20000000000ull) {
            printf("lsqfit: mbarrier wait timed out (block %d thread %d)\n", blockIdx.x, threadIdx.x);
            __trap();
        }
    }
#else
    mbar_wait(bar, parity);
#endif
}

// Reductions for the column-split degrees: with round 1's 12-warp shape the
// reduce-scatter versions spilled (the NV-wide register arrays met the
// 168-register cap of a 384-thread CTA) and cost 2.5% at n = 1e9; in the
// 8-warp P = 16 shape (255 registers) they do not spill, are neutral at
// n = 1e9 and 6-8.5% faster at n = 1e6 (profiles/r02_ab_reduce_scatter.txt).
#ifndef LSQ_RS_SPLIT
#define LSQ_RS_SPLIT 1  // SPLIT CTA reduction by lane reduce-scatter (else per-column trees)
#endif
#ifndef LSQ_RS_FINAL
#define LSQ_RS_FINAL 1  // SPLIT degrees' last-CTA reduction: wide + reduce-scatter (else per-column warps)
#endif
#ifndef LSQ_PRODUCT_MIN
#define LSQ_PRODUCT_MIN 3  // fused multiply-add terms from this degree (sustained A/B: m = 3 5%, m = 4 12% faster, m = 2 neutral)
#endif
#ifndef LSQ_PRODUCT_CHAIN
#define LSQ_PRODUCT_CHAIN 8  // DFMA chain length of a product column (A/B: 8 beats 4 by 1-7% for m >= 6, 2 is slower)
#endif

template <int M>
struct PsCfg {
    static constexpr int NS = 2 * M;             // s[1..2M]
    static constexpr int NT = M + 1;             // t[0..M]
    static constexpr int NV = NS + NT;           // compensated sums
#ifndef LSQ_P16_MIN
#define LSQ_P16_MIN 0
#endif
    static constexpr int P = (M >= LSQ_P16_MIN && M <= LSQ_P16_MAX) ? 16 : 8;  // points per thread per tile
    // Warp w issues on SM sub-partition w % 4 and the register file is split
    // per sub-partition, so 8 warps give every sub-partition two consumers
    // and 255 registers/thread. SELF_FEED: all 8 warps consume and the last
    // warp to release a ring stage refills it (no producer warp). Otherwise:
    // 7 consumers + a producer warp (one sub-partition's FP64 pipe half used).
    // WS (warp-specialised, split degrees): 8 consumer warps at
    // LSQ_WS_CONSUMER_REGS registers and a 4-warp producer group shrunk to
    // LSQ_WS_PRODUCER_REGS by setmaxnreg (a 384-thread CTA launches at 168);
    // consumers release a stage by a plain mbarrier arrive, the producer
    // lane refills it as soon as its round completes.
    static constexpr bool WS = M >= LSQ_WS_MIN;
    static constexpr bool SELF_FEED = !WS && M >= LSQ_SELF_FEED_MIN;
    static constexpr bool GRIDSTRIDE = M <= LSQ_PS_GRIDSTRIDE_MAX;
    // DYN (producer-fed degrees): the last ~1/4 of the tiles are dealt in
    // chunks claimed from a global counter, each chunk summed into its own
    // record (see PsArgs), so per-SM bandwidth unfairness no longer sets the
    // finish time while the result stays independent of which CTA took which
    // chunk.
    static constexpr bool DYN = !SELF_FEED && M <= LSQ_DYN_MAX;
    // WS register split (per sub-partition: producer + 2 consumers = 3 x 168):
    // the dynamic-tail producer needs more than 24 registers
    static constexpr int WS_PROD_REGS = DYN ? 40 : LSQ_WS_PRODUCER_REGS;
    static constexpr int WS_CONS_REGS = DYN ? 232 : LSQ_WS_CONSUMER_REGS;
#ifndef LSQ_PROD_CW
#define LSQ_PROD_CW 7
#endif
#ifndef LSQ_SPLIT_MIN
#define LSQ_SPLIT_MIN 6  // round 2: m = 6..12 6-11% faster split (P = 16, 8 warps); m = 5 is producer-fed
#endif
#ifndef LSQ_SPLIT_CW
#define LSQ_SPLIT_CW 12
#endif
    // SPLIT (FP64-bound high degrees): the two lanes of a pair exchange their
    // tree sums by shuffle so each keeps the compensated state of only half
    // the columns (even lane: even columns, odd lane: odd columns). Halving
    // the per-thread state fits P = 16 points per thread in 8 warps' 255
    // registers (round 2, with product terms: 8-11% faster than round 1's
    // P = 8 x 12 warps, which the split also allowed: 168 registers).
    static constexpr bool SPLIT = (SELF_FEED || WS) && M >= LSQ_SPLIT_MIN;
#ifndef LSQ_SPLIT16_CW
#define LSQ_SPLIT16_CW 8
#endif
    static constexpr int CW =
        (SELF_FEED || WS) ? (SPLIT ? (P == 8 ? LSQ_SPLIT_CW : LSQ_SPLIT16_CW) : 8) : LSQ_PROD_CW;
    static constexpr int CONSUMERS = CW * 32;
    static constexpr int THREADS = CONSUMERS + (SELF_FEED ? 0 : (WS ? 128 : 32));
    static constexpr int TILE = CONSUMERS * P;      // points per tile
    // From m = 6 the per-thread lo words, and from m = 10 the carried pair
    // partials too, live in shared memory ([v][thread] columns, conflict-free,
    // touched once per tile) to keep the hot loop spill-free.
#ifndef LSQ_LO_SMEM_MIN
#define LSQ_LO_SMEM_MIN 6
#endif
    static constexpr bool LO_SMEM = (M >= LSQ_LO_SMEM_MIN);
#ifndef LSQ_PEND_SMEM_MIN
#define LSQ_PEND_SMEM_MIN 10  // A/B (self-feed): registers +1.6% at m=9; m=10..12 within noise
#endif
    static constexpr bool PEND_SMEM = !SPLIT && (M >= LSQ_PEND_SMEM_MIN);
    // compensated columns per thread
    static constexpr int NW = SPLIT ? (NV + 1) / 2 : NV;
    // Degrees whose consumer loop unrolls the tile pair (A/B-measured: faster
    // for m = 4..6, slower for m <= 3 and for the register-bound m >= 7).
    static constexpr bool PAIR_UNROLL = (M >= LSQ_PAIR_UNROLL_MIN && M <= LSQ_PAIR_UNROLL_MAX);
#ifndef LSQ_FOLD_TILES_HI
#define LSQ_FOLD_TILES_HI 8  // A/B: 4 vs 2 tiles 6-9% faster for m >= 7 (1-3% slower for m <= 3); 8 vs 4 a further 3-5%
#endif
#ifndef LSQ_FOLD_HI_MIN
#define LSQ_FOLD_HI_MIN 5
#endif
    // Tiles per fold: 2 when the pair is unrolled or HBM-bound, more for the
    // FP64-bound degrees (fewer compensation steps per point).
    static constexpr int FOLD_TILES = PAIR_UNROLL ? 2 : (M >= LSQ_FOLD_HI_MIN ? LSQ_FOLD_TILES_HI : 2);
    // PRODUCTS (the FP64-bound degrees): fused multiply-add terms. The
    // moments t[j] sum the exact products pw_j * y, and s[k] for k > M the
    // exact products pw_{k/2} * pw_{k-k/2} of two powers <= M (the powers
    // themselves keep the reference's repeated multiplication), so a point
    // costs (M-1) DMUL for the powers plus ~1 op per column instead of
    // (2M-1) DMUL + a DMUL per moment. Product columns are summed as P/CL
    // DFMA chains of CL terms, then a tree (csrc: prod_sum).
    static constexpr bool PRODUCTS = M >= LSQ_PRODUCT_MIN;
    static constexpr int CL = PRODUCTS ? (LSQ_PRODUCT_CHAIN < P ? LSQ_PRODUCT_CHAIN : P) : 1;
    static constexpr int LOG2P = P == 16 ? 4 : 3;
    static constexpr int TILE_LEVELS =
        PRODUCTS && (CL + LOG2P - (CL >= 8 ? 3 : CL >= 4 ? 2 : CL >= 2 ? 1 : 0)) > LOG2P
            ? CL + LOG2P - (CL >= 8 ? 3 : CL >= 4 ? 2 : CL >= 2 ? 1 : 0)
            : LOG2P;
    // Rounding depth of each folded plain partial: the tile tree (depth
    // log2 P; CL + log2(P/CL) for product chains), then FOLD_TILES - 1
    // sequential adds. The stated sum bound, against the exact sum of the
    // kernel's own terms (the reference's rounded terms, or the exact
    // products in PRODUCTS mode), is
    // |S - S_exact| <= ERR_LEVELS * u * sum|T| + ulp(S_exact) (+ O(u^2)).
    static constexpr int ERR_LEVELS = TILE_LEVELS + (SPLIT ? 1 : 0) + FOLD_TILES - 1;
    // DYN: two [warps][NV] dd buffers, alternated per chunk (no barrier
    // between one chunk's cross-warp read and the next chunk's writes)
    static constexpr size_t RED_BYTES = size_t(CW) * NV * 2 * sizeof(double) * (DYN ? 2 : 1);
    static constexpr size_t LO_BYTES = LO_SMEM ? size_t(NW) * CONSUMERS * sizeof(double) : 0;
    static constexpr size_t PEND_BYTES = PEND_SMEM ? size_t(NV) * CONSUMERS * sizeof(double) : 0;
    // Ring depth: the A/B-preferred depth, capped by what fits next to the
    // smem-resident words (227 KB per CTA, ~2 KB of it static).
    static constexpr int PREF_STAGES = (P == 16) ? 3 : (M >= 10 ? 3 : (PEND_SMEM ? 4 : 5));
    static constexpr int FIT_STAGES =
        int((232448 - 2048 - 64 - RED_BYTES - LO_BYTES - PEND_BYTES) / (size_t(TILE) * 16 + 16));
    static constexpr int STAGES = PREF_STAGES < FIT_STAGES ? PREF_STAGES : FIT_STAGES;
    static_assert(STAGES >= 2, "ring needs two stages");
    static constexpr size_t RING_BYTES = size_t(STAGES) * TILE * 16;
    static constexpr size_t SMEM_BYTES =
        RING_BYTES + 2 * STAGES * sizeof(uint64_t) + RED_BYTES + LO_BYTES + PEND_BYTES + 64;
    // the `empty` barrier words double as the SELF_FEED release counters
};

// The 3M+1 column sums of one thread's P points of a tile, each a balanced
// tree (depth log2 P) over exactly the reference's terms.
// Slot map: s[k] (k = 1..2M) -> k-1, t[j] (j = 0..M) -> 2M + j.
template <int M, int P>
__device__ __forceinline__ void tile_sums(const double (&x)[P], const double (&y)[P], double (&ts)[3 * M + 1]) {
    double tmp[P];
    // t[0] += 1.0 * y  (power_sums.cpp:22 with power == 1: the term is y exactly)
#pragma unroll
    for (int j = 0; j < P; ++j) tmp[j] = y[j];
    ts[2 * M] = tree_sum<P>(tmp);
    if constexpr (M >= 1) {
        double pw[P];
#pragma unroll
        for (int j = 0; j < P; ++j) pw[j] = x[j];  // power = 1.0 * x == x exactly
#pragma unroll
        for (int k = 1; k <= 2 * M; ++k) {
            if (k > 1) {
#pragma unroll
                for (int j = 0; j < P; ++j) pw[j] = __dmul_rn(pw[j], x[j]);  // power *= x
            }
#pragma unroll
            for (int j = 0; j < P; ++j) tmp[j] = pw[j];
            ts[k - 1] = tree_sum<P>(tmp);
            if (k <= M) {
#pragma unroll
                for (int j = 0; j < P; ++j) tmp[j] = __dmul_rn(pw[j], y[j]);  // power * y
                ts[2 * M + k] = tree_sum<P>(tmp);
            }
        }
    }
}

// SPLIT mode: the same column trees, handed to `put(v, tree_sum)` one
// column at a time (so they need not all stay live).
template <int M, int P, class Put>
__device__ __forceinline__ void tile_sums_put(const double (&x)[P], const double (&y)[P], Put&& put) {
    double tmp[P];
#pragma unroll
    for (int j = 0; j < P; ++j) tmp[j] = y[j];  // t[0] term: 1.0 * y == y
    put(2 * M, tree_sum<P>(tmp));
    double pw[P];
#pragma unroll
    for (int j = 0; j < P; ++j) pw[j] = x[j];  // power = 1.0 * x == x exactly
#pragma unroll
    for (int k = 1; k <= 2 * M; ++k) {
        if (k > 1) {
#pragma unroll
            for (int j = 0; j < P; ++j) pw[j] = __dmul_rn(pw[j], x[j]);  // power *= x
        }
#pragma unroll
        for (int j = 0; j < P; ++j) tmp[j] = pw[j];
        put(k - 1, tree_sum<P>(tmp));
        if (k <= M) {
#pragma unroll
            for (int j = 0; j < P; ++j) tmp[j] = __dmul_rn(pw[j], y[j]);  // power * y
            put(2 * M + k, tree_sum<P>(tmp));
        }
    }
}

// PRODUCTS mode: sum of the exact products a[j] * b[j] over P points as
// P/CL fused multiply-add chains of CL terms (chain c takes points c, c + C,
// ...), then a balanced tree over the chains. Each exact product suffers at
// most CL + log2(P/CL) roundings.
template <int P, int CL>
__device__ __forceinline__ double prod_sum(const double (&a)[P], const double (&b)[P]) {
    constexpr int C = P / CL;
    static_assert(C * CL == P, "chain length must divide P");
    double acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        acc[c] = __dmul_rn(a[c], b[c]);
#pragma unroll
        for (int r = 1; r < CL; ++r) acc[c] = __fma_rn(a[c + r * C], b[c + r * C], acc[c]);
    }
    return tree_sum<C>(acc);
}

// Emission order of the PRODUCTS columns (ProdOrder<M>::slot[i] = record slot
// of the i-th column tile_sums_prod emits): t0, then per power k = 1..M:
// s_k, t_k, and the product columns it completes, s_{2k-1} = pw_{k-1} pw_k
// and s_{2k} = pw_k pw_k when above M. Slot map as tile_sums: s[k] -> k-1,
// t[j] -> 2M + j.
template <int M>
struct ProdOrder {
    int slot[3 * M + 1];
    constexpr ProdOrder() : slot() {
        int i = 0;
        slot[i++] = 2 * M;
        for (int k = 1; k <= M; ++k) {
            slot[i++] = k - 1;
            slot[i++] = 2 * M + k;
            if (2 * k - 1 > M) slot[i++] = 2 * k - 2;
            if (2 * k > M) slot[i++] = 2 * k - 1;
        }
    }
};

// PRODUCTS mode: the 3M+1 column sums of one thread's P points, handed to
// put(i, slot, sum) in ProdOrder<M> order. Powers by the reference's
// repeated multiplication (power *= x) up to M only; two consecutive powers
// are live at a time.
template <int M, int P, int CL, class Put>
__device__ __forceinline__ void tile_sums_prod(const double (&x)[P], const double (&y)[P], Put&& put) {
    double tmp[P];
#pragma unroll
    for (int j = 0; j < P; ++j) tmp[j] = y[j];  // t[0] term: 1.0 * y == y
    int i = 0;
    put(i++, 2 * M, tree_sum<P>(tmp));
    double pp[P], pw[P];
#pragma unroll
    for (int j = 0; j < P; ++j) pw[j] = x[j];  // power = 1.0 * x == x exactly
#pragma unroll
    for (int k = 1; k <= M; ++k) {
        if (k > 1) {
#pragma unroll
            for (int j = 0; j < P; ++j) {
                pp[j] = pw[j];
                pw[j] = __dmul_rn(pw[j], x[j]);  // power *= x
            }
        }
#pragma unroll
        for (int j = 0; j < P; ++j) tmp[j] = pw[j];
        put(i++, k - 1, tree_sum<P>(tmp));                                  // s_k
        put(i++, 2 * M + k, prod_sum<P, CL>(pw, y));                        // t_k = sum pw_k * y
        if (2 * k - 1 > M) put(i++, 2 * k - 2, prod_sum<P, CL>(pp, pw));    // s_{2k-1}
        if (2 * k > M) put(i++, 2 * k - 1, prod_sum<P, CL>(pw, pw));        // s_{2k}
    }
}

// Per-thread low words of the compensated sums: registers, or a [v][thread]
// shared-memory column.
template <int NV, bool SMEM, int STRIDE>
struct LoWords {
    double v[NV];
    __device__ __forceinline__ void init(double*, int) {
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = 0.0;
    }
    __device__ __forceinline__ double& operator[](int i) { return v[i]; }
};
template <int NV, int STRIDE>
struct LoWords<NV, true, STRIDE> {
    double* p;
    __device__ __forceinline__ void init(double* base, int tid) {
        p = base + tid;
#pragma unroll
        for (int i = 0; i < NV; ++i) p[i * STRIDE] = 0.0;
    }
    __device__ __forceinline__ double& operator[](int i) { return p[i * STRIDE]; }
};

struct PsArgs {
    const double2* xy;
    uint64_t n;           // points in this launch (this shard)
    double2* cta_slots;   // [gridDim.x][NV] dd partials
    unsigned* ticket;     // zero between launches (the last CTA resets it)
    lsqfit_result* out;   // device result
    unsigned flags;
    // Dynamic tail (PsCfg::DYN): tiles [static_tiles, n_tiles) form n_chunks
    // chunks of shrinking size (guided self-scheduling, sizes a fixed
    // function of the chunk index, dyn_chunk()). Chunk c's dd sums go to
    // chunk_slots[c], whichever CTA claimed it; the final reduction takes the
    // CTA slots then the chunk records (reduce_records_wide: a fixed order).
    // dyn_counters[0] = chunk claims (zero between launches, re-armed by the
    // last CTA).
    uint64_t static_tiles;
    uint64_t chunk_s0;    // size of the first G chunks; halves every G chunks
    uint32_t chunk_min;   // ... down to this size (the last chunk may be short)
    uint32_t n_chunks;
    double2* chunk_slots;
    unsigned* dyn_counters;
};

// Tiles first + j * stride (j < count) of dynamic chunk c: levels of `grid`
// chunks of size s0, s0/2, ... while above chunk_min, then blocks of `grid`
// chunks of chunk_min. Within a level (block) chunk i takes every grid-th
// tile from i, so the CTAs working through one level sweep HBM together,
// like the static round-robin deal. Shared by the producer, the consumers
// and (through the same loop) the host sizing.
__host__ __device__ inline void dyn_chunk(uint64_t c, uint64_t grid, uint64_t static_tiles, uint64_t s0,
                                          uint64_t chunk_min, uint64_t n_tiles, uint64_t& first,
                                          uint64_t& count) {
    uint64_t off = static_tiles, size = s0;
    while (size > chunk_min && c >= grid) {
        off += grid * size;
        c -= grid;
        size >>= 1;
    }
    if (size > chunk_min) {
        first = off + c;
        count = size;
        return;
    }
    first = off + (c / grid) * grid * chunk_min + c % grid;
    count = first >= n_tiles ? 0 : (n_tiles - first + grid - 1) / grid;
    if (count > chunk_min) count = chunk_min;
}

// Host: the dynamic-tail plan for `tiles` tiles over `grid` CTAs — the last
// tiles / den in chunks of halving size (first level: half the tail over the
// grid) down to `chunk` tiles, the floor doubled until at most max_chunks
// records. dyn_chunk() over c < n_chunks partitions [static_tiles, tiles)
// exactly (tests/test_dyn_schedule.py checks it on many shapes).
struct DynPlan {
    uint64_t static_tiles, s0;
    uint32_t chunk_min, n_chunks;
};
inline DynPlan dyn_plan(uint64_t tiles, uint64_t grid, uint64_t den, uint64_t chunk, uint64_t max_chunks) {
    const uint64_t dyn = tiles / den;
    const uint64_t s0 = dyn / (2 * grid);
    for (uint64_t kmin = chunk;; kmin *= 2) {
        // the levels (sizes > kmin) sum to < 2 * grid * s0 <= dyn, so they fit
        uint64_t off = tiles - dyn, size = s0, chunks = 0;
        while (size > kmin) {
            off += grid * size;
            chunks += grid;
            size >>= 1;
        }
        // then blocks of grid chunks of kmin (strided; no empty chunk)
        const uint64_t rem = tiles - off, block = grid * kmin;
        chunks += (rem / block) * grid + (rem % block < grid ? rem % block : grid);
        if (chunks <= max_chunks)
            return DynPlan{tiles - dyn, s0, static_cast<uint32_t>(kmin), static_cast<uint32_t>(chunks)};
    }
}

// Warp 0 of a CTA: given the final dd sums in smem (vals_hi/lo[NV]) and the
// point count, write the PowerSums image, check finiteness (require_finite,
// power_sums.cpp:28-35) and optionally solve. `scratch` holds >= dim*dim +
// 2*dim + 3M + 2 doubles of shared memory.
template <int M>
__device__ void finalize_fit(const double* vals_hi, const double* vals_lo, uint64_t n, unsigned flags,
                             lsqfit_result* out, double* scratch) {
    constexpr int NS = 2 * M, NV = 3 * M + 1, DIM = M + 1;
    const int lane = threadIdx.x & 31;
    double* s = scratch;            // 2M+1
    double* t = s + (2 * M + 1);    // M+1
    double* A = t + (M + 1);        // DIM*DIM
    double* b = A + DIM * DIM;      // DIM
    double* x = b + DIM;            // DIM
    int bad = 0;
    for (int v = lane; v < NV; v += 32) {
        const double h = vals_hi[v], l = vals_lo[v];
        const double val = __dadd_rn(h, l);
        out->part_hi[v] = h;
        out->part_lo[v] = l;
        if (v < NS) {
            s[v + 1] = val;
            out->s[v + 1] = val;
        } else {
            t[v - NS] = val;
            out->t[v - NS] = val;
        }
        bad |= !isfinite(val);
    }
    if (lane == 0) {
        s[0] = static_cast<double>(n);  // s[0] counts points exactly (power_sums.hpp:11-12)
        out->s[0] = s[0];
        out->n = n;
        out->degree = M;
    }
    bad = __any_sync(0xffffffffu, bad);
    __syncwarp();
    int status = bad ? LSQFIT_EOVERFLOW : LSQFIT_OK;
    if (status == LSQFIT_OK && (flags & LSQFIT_SOLVE)) {
        warp_build_normal_system(s, t, M, A, b);
        status = warp_solve<DIM>(A, b, x);
        if (status == LSQFIT_OK)
            for (int k = lane; k < DIM; k += 32) out->coeffs[k] = x[k];
    }
    if (lane == 0) out->status = status;
}

// Reduce `count` dd records src[i*NV + v] (i ascending) for every v, using
// WARPS warps: warp w owns v = w, w+WARPS, ...; lane l sums records
// l, l+32, ... then a shfl-down tree. Fixed order => deterministic.
template <int NV, int WARPS, class Load>
__device__ __forceinline__ void reduce_records(int count, Load load, double* vals_hi, double* vals_lo) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int v = warp; v < NV; v += WARPS) {
        double h = 0.0, l = 0.0;
        // records i = lane, lane+32, ... in ascending order; loads issued in
        // batches of 8 ahead of the dependent dd chain (latency-bound tail)
        for (int base = lane; base < count; base += 8 * 32) {
            double2 r[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int i = base + q * 32;
                r[q] = i < count ? load(i, v) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (base + q * 32 < count) dd_add(h, l, r[q].x, r[q].y);
        }
        warp_reduce_dd_down(h, l);
        if (lane == 0) {
            vals_hi[v] = h;
            vals_lo[v] = l;
        }
    }
}

#ifndef LSQ_SF_L2_PREFETCH
// Self-fed degrees up to LSQ_SF_L2_PREFETCH_MAX_M: each refill also
// prefetches the next tile into L2 (A/B, profiles/r02_ab_sf_l2_prefetch.txt:
// m = 6 7.5% / m = 7 3-5% / m = 8 1.2% faster in alternating launches,
// 1.6% / +0.6% sustained; m = 12 2.7% slower; 2 or 4 tiles ahead no better).
#define LSQ_SF_L2_PREFETCH 1
#endif
#ifndef LSQ_SF_L2_PREFETCH_MAX_M
#define LSQ_SF_L2_PREFETCH_MAX_M 8
#endif
#ifndef LSQ_PS_PROBE
#define LSQ_PS_PROBE 0  // dev probe of the self-fed consumers (profiles/r02_ab_warp_ring.txt)
#endif
#ifdef LSQ_PS_TRACE
// Dev probe only (tools/ps_trace.py): per-CTA globaltimer stamps.
__device__ unsigned long long g_ps_trace[1024][8];
#define LSQ_TRACE(slot)                                                     \
    do {                                                                    \
        if (threadIdx.x == 0 && blockIdx.x < 1024) g_ps_trace[blockIdx.x][slot] = globaltimer_ns(); \
    } while (0)
#else
#define LSQ_TRACE(slot) \
    do {                \
    } while (0)
#endif

// Reduce `count` dd records (record i, column v = load(i, v)) with WARPS
// warps for many records: warp w takes the contiguous records
// [count*w/WARPS, count*(w+1)/WARPS), its lanes every 32nd of them for all
// NV columns at once (NV independent loads in flight per record), then a
// shfl-down tree per column, then the warps in ascending order (thread
// v < NV). A fixed function of count: deterministic. red_hi/red_lo:
// [WARPS][NV] shared scratch; named barrier 1 over `threads` threads.
template <int NV, int WARPS, class Load>
__device__ __forceinline__ void reduce_records_wide(int count, Load load, double* red_hi, double* red_lo,
                                                    double* vals_hi, double* vals_lo, int threads) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double h[NV], l[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) h[v] = l[v] = 0.0;
    if (warp < WARPS) {
        const int lo = static_cast<int>(int64_t(count) * warp / WARPS);
        const int hi = static_cast<int>(int64_t(count) * (warp + 1) / WARPS);
        for (int i = lo + lane; i < hi; i += 32) {
            double2 r[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) r[v] = load(i, v);
#pragma unroll
            for (int v = 0; v < NV; ++v) dd_add(h[v], l[v], r[v].x, r[v].y);
        }
        int c0 = 0, cnt = NV;
        reduce_scatter_level<NV, 16, 1>(h, l, lane, c0, cnt);
        constexpr int CF = reduce_scatter_count<NV, 16, 1>();
#pragma unroll
        for (int i = 0; i < CF; ++i) {
            const int v = c0 + i;
            if (i < cnt) {
                red_hi[warp * NV + v] = h[i];
                red_lo[warp * NV + v] = l[i];
            }
        }
    }
    named_bar_sync(1, threads);
    if (threadIdx.x < NV) {
        const int v = threadIdx.x;
        double sh = red_hi[v], sl = red_lo[v];
        for (int w = 1; w < WARPS; ++w) dd_add(sh, sl, red_hi[w * NV + v], red_lo[w * NV + v]);
        vals_hi[v] = sh;
        vals_lo[v] = sl;
    }
}

template <int M>
__global__ void __launch_bounds__(PsCfg<M>::THREADS, 1) power_sums_kernel(PsArgs a) {
    using C = PsCfg<M>;
    constexpr int NV = C::NV, P = C::P, TILE = C::TILE, STAGES = C::STAGES;
    constexpr int CW = C::CW, CONSUMERS = C::CONSUMERS;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2* ring = reinterpret_cast<double2*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + C::RING_BYTES);
    uint64_t* empty = full + STAGES;
    double* red_hi = reinterpret_cast<double*>(empty + STAGES);  // [warps][NV]
    double* red_lo = red_hi + CW * NV;
    double* lo_smem = red_hi + C::RED_BYTES / sizeof(double);  // [NV][CONSUMERS] when C::LO_SMEM
    __shared__ int s_is_last;
    __shared__ double s_vals[2 * NV];
    __shared__ double s_scratch[(2 * M + 1) + (M + 1) + (M + 1) * (M + 1) + 2 * (M + 1) + 8];

    LSQ_TRACE(0);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    const uint64_t n = a.n;
    const uint64_t n_tiles = (n + TILE - 1) / TILE;
    const uint64_t G = gridDim.x, bid = blockIdx.x;
    // DYN: only tiles [0, n_static) are dealt statically (the rest are
    // claimed in chunks, below).
    const uint64_t n_static = C::DYN ? a.static_tiles : n_tiles;
    // GRIDSTRIDE: tiles dealt round-robin, CTA b takes tiles b, b + G, ...
    // (the grid sweeps the array together); else CTA b owns the contiguous
    // tile range [T*b/G, T*(b+1)/G)
    constexpr bool GS = C::GRIDSTRIDE;
    const uint64_t t_begin = GS ? bid : n_static * bid / G;
    const uint64_t t_end = GS ? 0 : n_static * (bid + 1) / G;
    const uint64_t my_tiles = GS ? (n_static > bid ? (n_static - 1 - bid) / G + 1 : 0) : t_end - t_begin;
    auto tile_index = [&](uint64_t it) { return GS ? bid + it * G : t_begin + it; };
    const bool owns_last = n_static == n_tiles && (GS ? (n_tiles > 0 && (n_tiles - 1) % G == bid) : (t_end == n_tiles));

    // Only the globally last tile can be ragged; it belongs to the last CTA.
    const int last_valid = static_cast<int>(n - (n_tiles ? (n_tiles - 1) * TILE : 0));
    const bool cta_ragged = owns_last && my_tiles > 0 && last_valid < TILE;

    // Stream this CTA's tile `it` into ring stage `stage` (one thread): the
    // full barrier expects its bytes, the bulk-copy engine completes them.
    auto issue_global = [&](uint64_t g, bool ragged, int stage, uint64_t pol) {
        const uint32_t bytes = ragged ? uint32_t(last_valid) * 16u : uint32_t(TILE) * 16u;
        mbar_arrive_expect_tx(&full[stage], bytes);
        const unsigned char* src = reinterpret_cast<const unsigned char*>(a.xy + g * TILE);
        unsigned char* dst = reinterpret_cast<unsigned char*>(ring + stage * TILE);
        for (uint32_t off = 0; off < bytes; off += kPieceBytes) {
            const uint32_t len = (bytes - off < kPieceBytes) ? (bytes - off) : kPieceBytes;
            bulk_g2s(dst + off, src + off, len, &full[stage], pol);
        }
    };
    auto issue_tile = [&](uint64_t it, int stage, uint64_t pol) {
        issue_global(tile_index(it), cta_ragged && it + 1 == my_tiles, stage, pol);
        if constexpr ((C::SELF_FEED || C::WS) && LSQ_SF_L2_PREFETCH > 0 && M <= LSQ_SF_L2_PREFETCH_MAX_M) {
            // the tile LSQ_SF_L2_PREFETCH further on into L2 (never the CTA's
            // last, possibly partial, tile)
            if (it + LSQ_SF_L2_PREFETCH + 1 < my_tiles) {
                const unsigned char* src =
                    reinterpret_cast<const unsigned char*>(a.xy + tile_index(it + LSQ_SF_L2_PREFETCH) * TILE);
                for (uint32_t off = 0; off < uint32_t(TILE) * 16u; off += kPieceBytes)
                    bulk_prefetch_l2(src + off, kPieceBytes);
            }
        }
    };
    // DYN: chunk id (or kDynEnd) of the chunk whose first tile is in a stage.
    __shared__ unsigned s_info[STAGES];
    // SELF_FEED: per-stage release counters (monotonic; the warp whose
    // increment completes a round of CW is the stage's last reader).
    uint32_t* released = reinterpret_cast<uint32_t*>(empty);

    // PDL: everything above touches only registers and shared memory; from
    // here on the kernel reads the points and the scratch (slots, ticket,
    // chunk counters) a previous launch may still be using, so wait for it.
    // The next launch may be scheduled right away: its CTAs wait the same way.
    grid_dependency_wait();
    allow_dependent_launch();
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            if constexpr (C::SELF_FEED) released[2 * s] = 0u;
            else mbar_init(&empty[s], CW);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if constexpr (C::SELF_FEED) {
        if (tid == 0) {
            const uint64_t pol = l2_evict_first_policy();
            for (uint64_t it = 0; it < my_tiles && it < uint64_t(STAGES); ++it) issue_tile(it, int(it), pol);
        }
    }

    // hi/lo: per-thread compensated sums. Tiles are consumed in pairs whose
    // tree sums are added (one more tree level) before folding, so one fold
    // covers 2P points.
    constexpr int NW = C::NW;
    double hi[NW];
    LoWords<NW, C::LO_SMEM, CONSUMERS> lo;
#pragma unroll
    for (int v = 0; v < NW; ++v) hi[v] = 0.0;
    if (warp < CW) lo.init(lo_smem, tid);

    if constexpr (C::WS) {
        if (warp >= CW) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::WS_PROD_REGS));
        else asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::WS_CONS_REGS));
    }
    if (!C::SELF_FEED && warp >= CW) {
        // ---------------- producer warp: HBM -> SMEM ring via the bulk-copy engine
        if (warp == CW && lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int stage = 0;
            uint32_t round = 0;  // how many times the ring has wrapped
            auto wait_free = [&]() {
                if (round > 0) {
                    if constexpr (LSQ_PRODUCER_SLEEP) mbar_wait_sleep(&empty[stage], (round - 1) & 1, LSQ_PRODUCER_SLEEP);
                    else mbar_wait(&empty[stage], (round - 1) & 1);
                }
            };
            auto advance = [&]() {
                if (++stage == STAGES) {
                    stage = 0;
                    ++round;
                }
            };
            for (uint64_t it = 0; it < my_tiles; ++it) {
                wait_free();
                issue_tile(it, stage, pol);
                advance();
            }
            if constexpr (C::DYN) {
                // Dynamic tail: claim chunks until none are left, then tag
                // one stage kDynEnd (completed by a plain arrive, no bytes).
                if (a.n_chunks > 0) {
                    for (;;) {
                        const unsigned c = atomicAdd(&a.dyn_counters[0], 1u);
                        wait_free();
                        if (c >= a.n_chunks) {
                            s_info[stage] = kDynEnd;
                            mbar_arrive(&full[stage]);
                            break;
                        }
                        s_info[stage] = c;
                        uint64_t first, cnt;
                        dyn_chunk(c, G, a.static_tiles, a.chunk_s0, a.chunk_min, n_tiles, first, cnt);
                        for (uint64_t j = 0; j < cnt; ++j) {
                            if (j > 0) wait_free();
                            const uint64_t g = first + j * G;
                            issue_global(g, g + 1 == n_tiles && last_valid < TILE, stage, pol);
                            advance();
                        }
                    }
                }
            }
        }
    } else {
        // ---------------- consumers
        int stage = 0;
        uint32_t phase = 0;
        uint64_t it_c = 0;  // tiles consumed by this warp
#ifdef LSQ_PS_TRACE
        uint64_t it_trace = 0;
#endif
        // Wait for the next tile, pull this thread's P points into registers,
        // release the slot, and return the tile's 3M+1 tree sums.
        auto consume = [&](bool ragged, double (&ts)[NV]) {
            consumer_wait(&full[stage], phase);
#ifdef LSQ_PS_TRACE
            if (it_trace++ == 0) LSQ_TRACE(6);
#endif
            const double2* tile = ring + stage * TILE;
            double x[P], y[P];
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const double2 v = tile[j * CONSUMERS + tid];
                x[j] = v.x;
                y[j] = v.y;
            }
            __syncwarp();
            if constexpr (C::SELF_FEED) {
                // The last of the CW warps to finish reading the stage refills
                // it with the tile STAGES ahead (no thread ever waits to issue).
                if (lane == 0) {
                    const uint32_t prev = atom_add_acq_rel_cta(&released[2 * stage], 1u);
                    if (prev % CW == CW - 1 && it_c + STAGES < my_tiles) {
                        fence_proxy_async_smem();
                        issue_tile(it_c + STAGES, stage, l2_evict_first_policy());
                    }
                }
                ++it_c;
            } else {
                if (lane == 0) mbar_arrive(&empty[stage]);
            }
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1u;
            }
            if (ragged) {
                // Points past n are (0, 0): their terms are exactly zero for
                // s[k>=1] and t[j] (s[0] is the integer n).
#pragma unroll
                for (int j = 0; j < P; ++j)
                    if (j * CONSUMERS + tid >= last_valid) x[j] = y[j] = 0.0;
            }
            if constexpr (C::PRODUCTS)
                tile_sums_prod<M, P, C::CL>(x, y, [&](int, int slot, double v) { ts[slot] = v; });
            else
                tile_sums<M, P>(x, y, ts);
        };
        // SPLIT: the same pipeline step, column sums handed to `put`.
        auto consume_with = [&](bool ragged, auto&& put) {
#if LSQ_PS_PROBE
            // Dev probe (tools/ab.py timing only, wrong sums): after the first
            // STAGES tiles the ring is re-read without waiting; PROBE 1 also
            // skips the release, PROBE 2 keeps its atomic (no refill).
            if (it_c < uint64_t(STAGES)) consumer_wait(&full[stage], phase);
#else
            consumer_wait(&full[stage], phase);
#endif
            const double2* tile = ring + stage * TILE;
            double x[P], y[P];
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const double2 v = tile[j * CONSUMERS + tid];
                x[j] = v.x;
                y[j] = v.y;
            }
            __syncwarp();
#if LSQ_PS_PROBE == 1
            if (false) {
#else
            if (C::WS && lane == 0) {
                mbar_arrive(&empty[stage]);
            } else if (lane == 0) {
#endif
                const uint32_t prev = atom_add_acq_rel_cta(&released[2 * stage], 1u);
                if (prev % CW == CW - 1 && it_c + STAGES < my_tiles && !LSQ_PS_PROBE) {
                    fence_proxy_async_smem();
                    issue_tile(it_c + STAGES, stage, l2_evict_first_policy());
                }
            }
            ++it_c;
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1u;
            }
            if (ragged) {
#pragma unroll
                for (int j = 0; j < P; ++j)
                    if (j * CONSUMERS + tid >= last_valid) x[j] = y[j] = 0.0;
            }
            if constexpr (C::PRODUCTS)
                tile_sums_prod<M, P, C::CL>(x, y, [&](int i, int, double v) { put(i, v); });  // paired by emission index
            else
                tile_sums_put<M, P>(x, y, put);
        };
        // `count` tiles from the ring into hi/lo (all but SPLIT);
        // `ragged_last`: the last of them is the globally last, partial tile.
        auto run_tiles = [&](uint64_t count, bool ragged_last) {
            if constexpr (C::PAIR_UNROLL) {
                const uint64_t pairs = count / 2;
                for (uint64_t pr = 0; pr < pairs; ++pr) {
                    double ta[NV], tb[NV];
                    consume(false, ta);
                    consume(ragged_last && !(count & 1) && pr + 1 == pairs, tb);
#pragma unroll
                    for (int v = 0; v < NV; ++v) fold_sorted(hi[v], lo[v], __dadd_rn(ta[v], tb[v]));
                }
                if (count & 1) {
                    double ta[NV];
                    consume(ragged_last, ta);
#pragma unroll
                    for (int v = 0; v < NV; ++v) fold_sorted(hi[v], lo[v], ta[v]);
                }
            } else {
                // High degree: a carried partial — the tree sums of FOLD_TILES
                // consecutive tiles are added in sequence, then folded once
                // (keeps the register footprint of one tile; the unrolled pair
                // spills, and fewer folds cut the compensation cost per point).
                constexpr int K = C::FOLD_TILES;
                LoWords<NV, C::PEND_SMEM, CONSUMERS> pend;
                if constexpr (C::PEND_SMEM) pend.init(lo_smem + (C::LO_SMEM ? NV * CONSUMERS : 0), tid);
                int k = 0;  // tiles in the carried partial
                for (uint64_t it = 0; it < count; ++it) {
                    double ts[NV];
                    consume(ragged_last && it + 1 == count, ts);
                    if (k == K - 1) {
#pragma unroll
                        for (int v = 0; v < NV; ++v) fold_sorted(hi[v], lo[v], __dadd_rn(pend[v], ts[v]));
                        k = 0;
                    } else if (k == 0) {
#pragma unroll
                        for (int v = 0; v < NV; ++v) pend[v] = ts[v];
                        k = 1;
                    } else {
#pragma unroll
                        for (int v = 0; v < NV; ++v) pend[v] = __dadd_rn(pend[v], ts[v]);
                        ++k;
                    }
                }
                if (k != 0) {
#pragma unroll
                    for (int v = 0; v < NV; ++v) fold_sorted(hi[v], lo[v], pend[v]);
                }
            }
        };
        // hi/lo of every consumer -> dst[0..NV) (fixed order: lanes by a
        // shuffle-down tree, then warps ascending). All but SPLIT.
        auto reduce_store = [&](double2* dst, int buf) {
            double* rh = red_hi + buf * (2 * CW * NV);
            double* rl = rh + CW * NV;
            // lanes: reduce-scatter (each column's warp sum lands in one lane)
            double h[NV], l[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                h[v] = hi[v];
                l[v] = lo[v];
            }
            int c0 = 0, cnt = NV;
            reduce_scatter_level<NV, 16, 1>(h, l, lane, c0, cnt);
            constexpr int CF = reduce_scatter_count<NV, 16, 1>();
#pragma unroll
            for (int i = 0; i < CF; ++i) {
                const int v = c0 + i;
                if (i < cnt) {
                    rh[warp * NV + v] = h[i];
                    rl[warp * NV + v] = l[i];
                }
            }
            named_bar_sync(1, CONSUMERS);
            if (tid < NV) {
                double h = rh[tid], l = rl[tid];
                for (int w = 1; w < CW; ++w) dd_add(h, l, rh[w * NV + tid], rl[w * NV + tid]);
                dst[tid] = make_double2(h, l);
            }
        };
        // Tiles are consumed in pairs: one more tree level, then one fold.
        if constexpr (C::SPLIT) {
            // Column-split carried partials: per tile, every column's tree
            // sum is paired with the partner lane's by one shuffle (one more
            // tree level: 2P points), and the owner adds it to its carried
            // partial; FOLD_TILES tiles per fold as below.
            constexpr int K = C::FOLD_TILES;
            const bool odd = (lane & 1) != 0;
            double pend[NW];
#pragma unroll
            for (int j = 0; j < NW; ++j) pend[j] = 0.0;
            int k = 0;
            for (uint64_t it = 0; it < my_tiles; ++it) {
                double stash[NV];
                // pend restarts at 0 after each fold (0 + val == val exactly):
                // a plain add, no per-column select
                auto own = [&](int j, double val) { pend[j] = __dadd_rn(pend[j], val); };
                consume_with(cta_ragged && it + 1 == my_tiles, [&](int v, double t) {
                    if ((v & 1) == 0) {
                        if (v + 1 < NV) {
                            stash[v] = t;  // wait for the odd partner column
                        } else {           // last column (NV odd): the even lane owns it
                            const double r = __shfl_xor_sync(0xffffffffu, t, 1);
                            if (!odd) own(v >> 1, __dadd_rn(t, r));
                        }
                        return;
                    }
                    const double a = stash[v - 1], b = t;  // my sums of columns v-1, v
                    const double r = __shfl_xor_sync(0xffffffffu, odd ? a : b, 1);
                    own(v >> 1, __dadd_rn(odd ? b : a, r));  // even: column v-1, odd: column v
                });
                if (++k == K) {
#pragma unroll
                    for (int j = 0; j < NW; ++j) {
                        fold_sorted(hi[j], lo[j], pend[j]);
                        pend[j] = 0.0;
                    }
                    k = 0;
                }
            }
            if (k != 0) {
#pragma unroll
                for (int j = 0; j < NW; ++j) fold_sorted(hi[j], lo[j], pend[j]);
            }
        } else {
          run_tiles(my_tiles, cta_ragged);
        }

        LSQ_TRACE(1);
        // ---------------- CTA reduction (consumers only; fixed order)
        if constexpr (C::SPLIT) {
            // reduce over the lanes of one parity: lane 0 ends with the even
            // columns, lane 1 with the odd ones
#if LSQ_RS_SPLIT
            // reduce-scatter over the 16 lanes of one parity (offsets 16..2):
            // owned column j of parity p is emission index 2j + p
            double h[NW], l[NW];
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                h[j] = hi[j];
                l[j] = lo[j];
            }
            int c0 = 0, cnt = NW;
            reduce_scatter_level<NW, 16, 2>(h, l, lane, c0, cnt);
            constexpr int CF = reduce_scatter_count<NW, 16, 2>();
#pragma unroll
            for (int i = 0; i < CF; ++i) {
                const int e = 2 * (c0 + i) + (lane & 1);
                if (i < cnt && e < NV) {
                    red_hi[warp * NV + e] = h[i];
                    red_lo[warp * NV + e] = l[i];
                }
            }
#else
            // per column: shuffle-down tree over the lanes of one parity;
            // lane p ends with owned column j of parity p (emission 2j + p)
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                double h = hi[j], l = lo[j];
#pragma unroll
                for (int off = 16; off >= 2; off >>= 1) {
                    const double oh = __shfl_down_sync(0xffffffffu, h, off);
                    const double ol = __shfl_down_sync(0xffffffffu, l, off);
                    dd_add(h, l, oh, ol);
                }
                const int e = 2 * j + lane;
                if (lane < 2 && e < NV) {
                    red_hi[warp * NV + e] = h;
                    red_lo[warp * NV + e] = l;
                }
            }
#endif
            named_bar_sync(1, CONSUMERS);
            if (tid < NV) {
                double h0 = red_hi[tid], l0 = red_lo[tid];
                for (int w = 1; w < CW; ++w) dd_add(h0, l0, red_hi[w * NV + tid], red_lo[w * NV + tid]);
                // emission index -> record slot (PRODUCTS: ProdOrder<M>)
                constexpr ProdOrder<M> order{};
                const int v = C::PRODUCTS ? order.slot[tid] : tid;
                a.cta_slots[bid * NV + v] = make_double2(h0, l0);
            }
        } else {
            reduce_store(a.cta_slots + bid * NV, 0);
        }

        if constexpr (C::DYN) {
            // ---------------- dynamic tail: one record per chunk, whichever
            // CTA claimed it (the static reduction used red_ buffer 0)
            if (a.n_chunks > 0) {
                int buf = 1;
                for (;;) {
                    consumer_wait(&full[stage], phase);
                    const unsigned c = reinterpret_cast<volatile unsigned*>(s_info)[stage];
                    if (c == kDynEnd) break;
                    uint64_t first, cnt;
                    dyn_chunk(c, G, a.static_tiles, a.chunk_s0, a.chunk_min, n_tiles, first, cnt);
#pragma unroll
                    for (int v = 0; v < NV; ++v) hi[v] = lo[v] = 0.0;
                    run_tiles(cnt, first + (cnt - 1) * G + 1 == n_tiles && last_valid < TILE);
                    reduce_store(a.chunk_slots + size_t(c) * NV, buf);
                    buf ^= 1;
                }
            }
        }
        LSQ_TRACE(4);
        __threadfence();
        named_bar_sync(1, CONSUMERS);
        if (tid == 0) {
            const unsigned prev = atomicAdd(a.ticket, 1u);
            s_is_last = (prev == gridDim.x - 1);
        }
        named_bar_sync(1, CONSUMERS);
        LSQ_TRACE(2);
        if (s_is_last) {
            __threadfence();
            const double2* slots = a.cta_slots;
            if (C::DYN && a.n_chunks > 0) {
                // CTA slots, then the chunk records, in index order
                const double2* chunks = a.chunk_slots;
                named_bar_sync(1, CONSUMERS);  // red_ buffers free
                reduce_records_wide<NV, CW>(
                    static_cast<int>(G + a.n_chunks),
                    [&](int i, int v) {
                        return i < static_cast<int>(G) ? __ldcg(&slots[size_t(i) * NV + v])
                                                       : __ldcg(&chunks[size_t(i - static_cast<int>(G)) * NV + v]);
                    },
                    red_hi, red_lo, s_vals, s_vals + NV, CONSUMERS);
            } else if (LSQ_RS_FINAL || !C::SPLIT) {
                named_bar_sync(1, CONSUMERS);  // red_ buffers free
                reduce_records_wide<NV, CW>(
                    static_cast<int>(G), [&](int i, int v) { return __ldcg(&slots[size_t(i) * NV + v]); }, red_hi,
                    red_lo, s_vals, s_vals + NV, CONSUMERS);
            } else {
                reduce_records<NV, CW>(
                    static_cast<int>(G), [&](int i, int v) { return __ldcg(&slots[size_t(i) * NV + v]); }, s_vals,
                    s_vals + NV);
            }
            named_bar_sync(1, CONSUMERS);
            LSQ_TRACE(5);
            if (tid == 0) {
                *a.ticket = 0u;  // re-arm for the next launch
                if (C::DYN && a.n_chunks > 0) a.dyn_counters[0] = 0u;
            }
            if (warp == 0) finalize_fit<M>(s_vals, s_vals + NV, n, a.flags, a.out, s_scratch);
            __syncwarp();
            LSQ_TRACE(3);
        }
    }
}

// Combine per-shard results (ascending shard order) and finish the fit.
template <int M>
__global__ void __launch_bounds__(kConsumers, 1) combine_kernel(const lsqfit_result* parts, int n_parts,
                                                                unsigned flags, lsqfit_result* out) {
    constexpr int NV = 3 * M + 1;
    __shared__ double s_vals[2 * NV];
    __shared__ double s_scratch[(2 * M + 1) + (M + 1) + (M + 1) * (M + 1) + 2 * (M + 1) + 8];
    __shared__ unsigned long long s_n;
    if (threadIdx.x == 0) {
        unsigned long long n = 0;
        for (int i = 0; i < n_parts; ++i) n += parts[i].n;
        s_n = n;
    }
    reduce_records<NV, kConsumerWarps>(
        n_parts, [&](int i, int v) { return make_double2(parts[i].part_hi[v], parts[i].part_lo[v]); }, s_vals,
        s_vals + NV);
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) finalize_fit<M>(s_vals, s_vals + NV, s_n, flags, out, s_scratch);
}

}  // namespace lsq
