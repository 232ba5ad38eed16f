// common.cuh — device helpers shared by the sm_100a kernels: double-double
// arithmetic (compensated sums), mbarrier + bulk-copy (TMA engine) PTX
// wrappers, warp reductions.
//
// Everything is compiled with --fmad=false and uses explicit _rn intrinsics
// where rounding matters, so the arithmetic is the IEEE binary64 the reference
// performs on x86-64 SSE2 (no FMA contraction, no extended precision).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>
#include <cstdio>

#include "lsqfit_cuda.h"

namespace lsq {

// ---------------------------------------------------------------------------
// Double-double (unevaluated hi + lo) arithmetic.
// ---------------------------------------------------------------------------

// Knuth TwoSum: s = fl(a + b), e = exact error, (a + b == s + e exactly).
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// Fold a plain partial v into the running compensated pair (hi, lo): order
// the operands by magnitude, then Dekker's Fast2Sum (exact error term when
// |a| >= |b|) — 1 compare + 3 adds + the lo update, vs TwoSum's 6 + 1.
__device__ __forceinline__ void fold_sorted(double& hi, double& lo, double v) {
    const bool swap = fabs(v) > fabs(hi);
    const double a = swap ? v : hi;
    const double b = swap ? hi : v;
    const double s = __dadd_rn(a, b);
    const double e = __dsub_rn(b, __dsub_rn(s, a));
    hi = s;
    lo = __dadd_rn(lo, e);
}

// (ahi, alo) += (bhi, blo), renormalised so that hi == fl(hi + lo).
__device__ __forceinline__ void dd_add(double& ahi, double& alo, double bhi, double blo) {
    double s, e;
    two_sum(ahi, bhi, s, e);
    e = __dadd_rn(e, __dadd_rn(alo, blo));
    const double h = __dadd_rn(s, e);
    alo = __dsub_rn(e, __dsub_rn(h, s));
    ahi = h;
}

// Lane 0 receives the dd sum over the warp, combined in a fixed tree order.
__device__ __forceinline__ void warp_reduce_dd_down(double& hi, double& lo) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const double oh = __shfl_down_sync(0xffffffffu, hi, off);
        const double ol = __shfl_down_sync(0xffffffffu, lo, off);
        dd_add(hi, lo, oh, ol);
    }
}

// Warp reduce-scatter of N double-double columns by recursive halving: at
// the level with lane offset OFF every lane hands the partner the half of its
// current columns it does not keep and adds the partner's copy of the half it
// keeps (lanes with the OFF bit clear keep the lower half; odd counts are
// padded with a zero column). After the levels OFF = FIRST .. LAST, a lane
// holds the sums over its lane group of columns [c0, c0 + cnt) in h[0..),
// l[0..): c0 and cnt (its real columns; the rest of its
// reduce_scatter_count() slots are padding, which may alias another lane's
// columns) are returned through the references (start with c0 = 0, cnt = N). Each column costs ~N/16 dd additions per lane instead of the
// 5 levels x N of a shuffle-down tree per column, and every column's order
// is a fixed function of the lane bits: deterministic.
template <int C, int OFF, int LAST, int N>
__device__ __forceinline__ void reduce_scatter_level(double (&h)[N], double (&l)[N], int lane, int& c0, int& cnt) {
    if constexpr (OFF >= LAST && OFF >= 1) {
        constexpr int H = (C + 1) / 2;
        const bool up = (lane & OFF) != 0;
#pragma unroll
        for (int i = 0; i < H; ++i) {
            const bool real = H + i < C;
            const int j = real ? H + i : 0;
            const double uh = real ? h[j] : 0.0, ul = real ? l[j] : 0.0;
            double kh = up ? uh : h[i], kl = up ? ul : l[i];
            const double gh = up ? h[i] : uh, gl = up ? l[i] : ul;
            const double rh = __shfl_xor_sync(0xffffffffu, gh, OFF);
            const double rl = __shfl_xor_sync(0xffffffffu, gl, OFF);
            dd_add(kh, kl, rh, rl);
            h[i] = kh;
            l[i] = kl;
        }
        if (up) {
            c0 += H;
            cnt = cnt > H ? cnt - H : 0;
        } else {
            cnt = cnt < H ? cnt : H;
        }
        reduce_scatter_level<H, OFF / 2, LAST>(h, l, lane, c0, cnt);
    }
}
// Columns per lane left after reduce_scatter_level<C, FIRST, LAST>.
template <int C, int FIRST, int LAST>
__host__ __device__ constexpr int reduce_scatter_count() {
    int c = C;
    for (int off = FIRST; off >= LAST && off >= 1; off /= 2) c = (c + 1) / 2;
    return c;
}

__device__ __forceinline__ double warp_reduce_sum_down(double v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
    return v;
}

// ---------------------------------------------------------------------------
// mbarrier / bulk async copy (cp.async.bulk -> SASS UBLKCP) wrappers.
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// try_wait with a suspend-time hint: the waiting thread sleeps in hardware
// until the phase completes or ~hint_ns elapse (no issue-slot spinning).
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t hint_ns) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity), "r"(hint_ns)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Bounded wait: a pipeline that stalls for > 20 s is a bug, so fail loudly
// (trap -> launch error on the host) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const uint64_t t0 = globaltimer_ns();
    while (!mbar_try_wait(bar, parity)) {
        if (globaltimer_ns() - t0 > 20000000000ull) {
            printf("lsqfit: mbarrier wait timed out (block %d thread %d parity %u)\n", blockIdx.x, threadIdx.x,
                   parity);
            __trap();
        }
    }
}

// Same bounded wait, sleeping in hardware between probes (for a thread that
// is usually far ahead, e.g. the producer waiting for a free ring slot).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t hint_ns = 1000000u) {
    if (mbar_try_wait(bar, parity)) return;
    const uint64_t t0 = globaltimer_ns();
    while (!mbar_try_wait_sleep(bar, parity, hint_ns)) {
        if (globaltimer_ns() - t0 > 20000000000ull) {
            printf("lsqfit: mbarrier wait timed out (block %d thread %d parity %u)\n", blockIdx.x, threadIdx.x,
                   parity);
            __trap();
        }
    }
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Bulk global -> shared copy completed on `bar` (tx bytes). bytes % 16 == 0,
// both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}

// Bulk prefetch of global memory into L2 (a hint: no completion, no smem).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src_gmem, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src_gmem), "r"(bytes) : "memory");
}

// Shared-memory counter increment with acquire-release semantics at CTA
// scope: the caller's (and, through a preceding __syncwarp, its warp's)
// earlier reads are ordered before it, and later work after every earlier
// increment. Returns the previous value.
__device__ __forceinline__ uint32_t atom_add_acq_rel_cta(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_addr(p)), "r"(v)
                 : "memory");
    return old;
}

// Order this thread's generic-proxy shared-memory accesses before its
// subsequent async-proxy (bulk copy) accesses.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Programmatic dependent launch (PDL). A kernel launched with the
// programmatic-stream-serialization attribute may start while the previous
// kernel in the stream is still running; grid_dependency_wait() blocks until
// that kernel has completed and its memory is visible (a no-op when there is
// no such prerequisite), and allow_dependent_launch() lets the NEXT kernel's
// CTAs be scheduled (they, in turn, wait for this grid before touching memory).
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void allow_dependent_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Named barrier over the first `threads` threads of the CTA (id 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// 256-bit global load of two AoS points (sm_100: LDG.E.ENL2.256), no L1 allocation.
__device__ __forceinline__ void ldg_2pts(const double* p, double& x0, double& y0, double& x1, double& y1) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(x0), "=d"(y0), "=d"(x1), "=d"(y1)
                 : "l"(p));
}

// In-place balanced tree sum of P values (P a power of two): depth log2 P.
template <int P>
__device__ __forceinline__ double tree_sum(double (&v)[P]) {
#pragma unroll
    for (int w = P / 2; w >= 1; w >>= 1) {
#pragma unroll
        for (int i = 0; i < w; ++i) v[i] = __dadd_rn(v[i], v[i + w]);
    }
    return v[0];
}


}  // namespace lsq
