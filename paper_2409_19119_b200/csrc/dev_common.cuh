// dev_common.cuh -- device helpers shared by the kernel translation units (ax.cu, gs.cu, vec.cu):
// Dirichlet/owner bit access, fixed-order block reductions, the last-CTA finish, and the NVLink
// peer-memory primitives (release/acquire epochs, mailbox push/pull).
//
// All reductions are two-level and fixed-order (no floating-point atomics), so results are bitwise
// repeatable run to run (reading 7/8).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cassert>
#include <cstdint>

#include "ax_tma.cuh"
#include "nek_ctx.h"

namespace nekb200 {

// Device-side invariant checks of the index-driven kernels (gather-scatter maps, halo slots): active in
// the checked build (build.py --checked -> libnek_checked.so, -DNEK_CHECKED), a failed check is a device
// assert (cudaErrorAssert, the call returns NEK_ECUDA).  compute-sanitizer is not available on the
// GPU pool, so this build plus the parity suite is the memory-safety evidence.
#ifdef NEK_CHECKED
#define NEK_CHECK(c) assert(c)
#else
#define NEK_CHECK(c) ((void)0)
#endif

__device__ __forceinline__ bool bit_of(const uint32_t *__restrict__ bits, int64_t l)
{
    return (__ldg(bits + (l >> 5)) >> (l & 31)) & 1u;
}

// Fixed-order block sum of v (blockDim.x a multiple of 32, <= 1024): a
// butterfly within each warp, then warp 0 folds the per-warp sums in warp
// order.  Deterministic; result valid in thread 0.  sred needs 32 entries.
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double block_sum(double v, double *sred)
{
    const int t = threadIdx.x, nw = (int)(blockDim.x >> 5);
    v = warp_sum(v);
    if ((t & 31) == 0) sred[t >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (t < 32) {
        r = t < nw ? sred[t] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

// Fixed-order block sum for any blockDim.x <= 1024 (smem tree); sred needs blockDim.x entries.
__device__ __forceinline__ double block_sum_any(double v, double *sred)
{
    const int t = threadIdx.x;
    sred[t] = v;
    __syncthreads();
    for (int s = 512; s > 0; s >>= 1) {
        if (s < (int)blockDim.x && t < s && t + s < (int)blockDim.x) sred[t] += sred[t + s];
        __syncthreads();
    }
    double r = sred[0];
    __syncthreads();
    return r;
}

// ------------------------------------------------------- accurate dot products
// Inner products are accumulated as unevaluated double-double sums (hi, lo): every product is split
// exactly (TwoProduct via fma) and every addition carries its exact rounding error (TwoSum) -- the
// Dot2 scheme of Ogita, Rump and Oishi that the oracle uses (oracle/nek_oracle.c), so the GPU's
// reductions, in whatever tree order, agree with the oracle's to about an ulp (reading 17).
// The cost is a few extra FP64 operations per point in bandwidth-bound kernels.
__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e)
{
    const double x = __dadd_rn(a, b), z = __dsub_rn(x, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(x, z)), __dsub_rn(b, z));
    s = x;
}
// (hi, lo) += x y
__device__ __forceinline__ void dd_add_prod(double &hi, double &lo, double x, double y)
{
    const double h = __dmul_rn(x, y), r = fma(x, y, -h);
    double e;
    two_sum(hi, h, hi, e);
    lo = __dadd_rn(lo, __dadd_rn(e, r));
}
// (hi, lo) += (bhi, blo)
__device__ __forceinline__ void dd_add(double &hi, double &lo, double bhi, double blo)
{
    double e;
    two_sum(hi, bhi, hi, e);
    lo = __dadd_rn(__dadd_rn(lo, blo), e);
}
__device__ __forceinline__ void warp_sum_dd(double &hi, double &lo)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double bh = __shfl_xor_sync(0xffffffffu, hi, o), bl = __shfl_xor_sync(0xffffffffu, lo, o);
        dd_add(hi, lo, bh, bl);
    }
}
// fixed-order block sum of (hi, lo) pairs (blockDim.x a multiple of 32, <= 1024); result valid in
// thread 0; sred needs 64 entries
__device__ __forceinline__ void block_sum_dd(double &hi, double &lo, double *sred)
{
    const int t = threadIdx.x, nw = (int)(blockDim.x >> 5);
    warp_sum_dd(hi, lo);
    if ((t & 31) == 0) { sred[2 * (t >> 5)] = hi; sred[2 * (t >> 5) + 1] = lo; }
    __syncthreads();
    if (t < 32) {
        hi = t < nw ? sred[2 * t] : 0.0;
        lo = t < nw ? sred[2 * t + 1] : 0.0;
        warp_sum_dd(hi, lo);
    }
    __syncthreads();
}

// ------------------------------------------------------------ peer memory
// One process per GPU (or one context per virtual rank in the loopback group); every rank maps its
// peers' mailbox / halo buffers and writes into them directly (NVLink, or the same device).  A value
// block is followed by a system-scope release store of a monotonically increasing epoch; the reader
// acquires the epoch and then reads.  All ranks run the same sequence of exchanges, so epochs agree.
// A spin gives up after timeout_ns of %globaltimer and raises *err (a volatile store into mapped host
// memory, visible to the host without a synchronisation): error, never a hang.
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// relaxed system-scope accesses: no fence of their own (one fence.acq_rel.sys orders a batch)
__device__ __forceinline__ void st_relaxed_sys(uint64_t *p, uint64_t v)
{
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// the release / acquire halves of the last-CTA reductions (cheaper than __threadfence's fence.sc.gpu)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint64_t globaltimer_ns()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ bool wait_epoch(const uint64_t *flag, uint64_t e, int *err, uint64_t timeout_ns)
{
    if (ld_acquire_sys(flag) >= e) return true;
    const uint64_t t0 = globaltimer_ns();
    for (int it = 0;; ++it) {   // poll relaxed (no L1 invalidation per poll), acquire once it is there
        if (ld_relaxed_sys(flag) >= e) return ld_acquire_sys(flag) >= e;
        if (it > 64) __nanosleep(64);
        if ((it & 255) == 0 && globaltimer_ns() - t0 > timeout_ns) break;
    }
    *(volatile int *)err = 1;
    __threadfence_system();
    return false;
}

// single thread: publish up to 3 values on `channel` to every rank (self included)
__device__ __forceinline__ void mail_push(const P2PMail &M, int channel, double v0, double v1, double v2)
{
    const uint64_t e = ++M.epochs[channel];
    const size_t base = ((size_t)channel * 2 + (e & 1)) * M.nranks;
    for (int q = 0; q < M.nranks; ++q) {
        double *dst = (q == M.me ? M.mbox : M.peer_mbox[q]) + (base + M.me) * 4;
        dst[0] = v0; dst[1] = v1; dst[2] = v2;
    }
    // one system-scope release fence orders the values above (every peer's) before all the flags
    fence_acq_rel_sys();
    for (int q = 0; q < M.nranks; ++q) {
        double *dst = (q == M.me ? M.mbox : M.peer_mbox[q]) + (base + M.me) * 4;
        st_relaxed_sys(reinterpret_cast<uint64_t *>(dst + 3), e);
    }
}

// single thread: wait for the current epoch of `channel` from every rank and
// return the rank-ordered sums of the value slots (NaN after a timeout)
__device__ __forceinline__ void mail_pull(const P2PMail &M, int channel, double *sum3)
{
    const uint64_t e = *(volatile uint64_t *)&M.epochs[channel];
    const size_t base = ((size_t)channel * 2 + (e & 1)) * M.nranks;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    bool ok = true;
    for (int q = 0; q < M.nranks; ++q) {
        const double *src = M.mbox + (base + q) * 4;
        ok &= wait_epoch(reinterpret_cast<const uint64_t *>(src + 3), e, M.err, M.timeout_ns);
        const double b0 = ((volatile const double *)src)[0], b1 = ((volatile const double *)src)[1],
                     b2 = ((volatile const double *)src)[2];
        if (q == 0) { a0 = b0; a1 = b1; a2 = b2; }
        else { a0 += b0; a1 += b1; a2 += b2; }
    }
    if (!ok) a0 = a1 = a2 = __longlong_as_double(0x7ff8000000000000ll);
    sum3[0] = a0; sum3[1] = a1; sum3[2] = a2;
}

// The same with the per-rank waits in parallel: called by all 32 lanes of one warp; lane q < nranks
// acquires rank q's slot, lane 0 folds the values in rank order (the bits of mail_pull).  nranks <= 32.
__device__ __forceinline__ void mail_pull_warp(const P2PMail &M, int channel, double *sum3)
{
    const int lane = threadIdx.x & 31;
    if (M.nranks > 32) {
        if (lane == 0) mail_pull(M, channel, sum3);
        return;
    }
    const uint64_t e = *(volatile uint64_t *)&M.epochs[channel];
    const size_t base = ((size_t)channel * 2 + (e & 1)) * M.nranks;
    double b0 = 0.0, b1 = 0.0, b2 = 0.0;
    bool ok = true;
    if (lane < M.nranks) {
        const double *src = M.mbox + (base + lane) * 4;
        ok = wait_epoch(reinterpret_cast<const uint64_t *>(src + 3), e, M.err, M.timeout_ns);
        b0 = ((volatile const double *)src)[0];
        b1 = ((volatile const double *)src)[1];
        b2 = ((volatile const double *)src)[2];
    }
    const bool all_ok = __all_sync(0xffffffffu, ok);
    double a0 = __shfl_sync(0xffffffffu, b0, 0), a1 = __shfl_sync(0xffffffffu, b1, 0),
           a2 = __shfl_sync(0xffffffffu, b2, 0);
    for (int q = 1; q < M.nranks; ++q) {
        const double c0 = __shfl_sync(0xffffffffu, b0, q), c1 = __shfl_sync(0xffffffffu, b1, q),
                     c2 = __shfl_sync(0xffffffffu, b2, q);
        a0 += c0; a1 += c1; a2 += c2;
    }
    if (!all_ok) a0 = a1 = a2 = __longlong_as_double(0x7ff8000000000000ll);
    if (lane == 0) { sum3[0] = a0; sum3[1] = a1; sum3[2] = a2; }
}

// Last CTA to finish folds the (hi, lo) partials part[2c], part[2c+1], c < count (fixed order),
// into dst[0] = hi + lo and resets the counter.  ctas_total: CTAs (over one or several concurrent
// launches) that share `counter`.  sred: 64 entries.
__device__ __forceinline__ void last_block_finish(double *part, int64_t count, double *dst, unsigned int *counter,
                                                  double *sred, int *s_last, const P2PMail *mail = nullptr,
                                                  unsigned int ctas_total = 0)
{
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        *s_last = atomicAdd(counter, 1u) == (ctas_total ? ctas_total : gridDim.x) - 1;
    }
    __syncthreads();
    if (*s_last) {
        fence_acq_rel_gpu();
        double hi = 0.0, lo = 0.0;
        for (int64_t c = threadIdx.x; c < count; c += blockDim.x)
            dd_add(hi, lo, ((volatile double *)part)[2 * c], ((volatile double *)part)[2 * c + 1]);
        block_sum_dd(hi, lo, sred);
        const double a = __dadd_rn(hi, lo);
        if (threadIdx.x == 0) {
            dst[0] = a;
            *counter = 0u;
            if (mail) mail_push(*mail, 0, a, 0.0, 0.0);   // sigma straight to every rank (channel 0)
        }
    }
}

// grid of a grid-stride kernel: enough CTAs for n items at `per` items per CTA, at most `waves` CTAs
// per SM of the current device
inline int stride_grid(int64_t n, int per, int waves)
{
    const int64_t want = (n + per - 1) / per;
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)waves * device_sms()));
}

}  // namespace nekb200
