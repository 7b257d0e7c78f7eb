// vec.cu -- the vector kernels of the hot path: Jacobi inverse, the fused Jacobi-PCG updates with
// deterministic last-CTA reductions (reading 8 owner-copy inner products), the NVLink
// mailbox exchange of the reduction slots, the projection space (NEXT #2) and, via
// pmg_kernels.cuh, the p-multigrid transfers and Chebyshev smoother (NEXT #1).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "dev_common.cuh"

namespace nekb200 {

__global__ void dinv_kernel(int64_t n, const uint32_t *__restrict__ mbits, const double *__restrict__ d,
                            double *__restrict__ dinv)
{
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x)
        dinv[l] = bit_of(mbits, l) ? 0.0 : 1.0 / d[l];
}

cudaError_t launch_dinv(int64_t n, const uint32_t *mbits, const double *d, double *dinv, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    dinv_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 16 * device_sms()), 256, 0, s>>>(n, mbits, d, dinv);
    return cudaGetLastError();
}

template <class T>
__global__ void copy_mask_kernel(int64_t n, const uint32_t *__restrict__ mbits, const T *__restrict__ src,
                                 T *__restrict__ dst)
{
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x)
        dst[l] = bit_of(mbits, l) ? T(0) : src[l];
}

template <class T>
cudaError_t launch_copy_mask(int64_t n, const uint32_t *mbits, const T *src, T *dst, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    copy_mask_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 16 * device_sms()), 256, 0, s>>>(n, mbits, src, dst);
    return cudaGetLastError();
}

// --------------------------------------------------------------------- PCG
constexpr int VEC_THREADS = 256;
constexpr int VEC_UNROLL = 4;
int device_sms()
{
    static int cache[64] = {};
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) { cudaGetLastError(); d = 0; }
    if (!cache[d]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) {
            cudaGetLastError();
            return 1;
        }
        cache[d] = v;
    }
    return cache[d];
}

int vec_blocks() { return 4 * device_sms(); }
// residual update: 2 CTAs per SM with 4 double2 per thread per tile (NEK_UPD_CTAS = 4 or 8: that many CTAs
// per SM with 2 double2 per thread per tile; measurement switch)
// the single-rank deferred update (no last CTA, 3 double2 per thread): 3 CTAs per SM (measured: config 2
// 5.87-5.89 vs 5.92 ms at 2 per SM, 16x16x128 0.82 vs 0.78 of the copy peak); NEK_UPD_CTAS overrides
int upd_blocks_deferred()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NEK_UPD_CTAS");
        v = e ? atoi(e) : 3;
        if (v != 2 && v != 3 && v != 4) v = 3;
    }
    return v * device_sms();
}

int upd_blocks()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NEK_UPD_CTAS");
        v = e ? atoi(e) : 2;
        if (v != 2 && v != 3 && v != 4 && v != 8) v = 2;
    }
    return v * device_sms();
}

// red_all holds [nranks][RED_N]; sums are taken in rank order.
__device__ __forceinline__ double rank_sum(const double *red_all, int nranks, int slot)
{
    double s = red_all[slot];
    for (int q = 1; q < nranks; ++q) s += red_all[q * RED_N + slot];
    return s;
}

// r = M b, p = Dinv r, x = 0; [<r, Dinv r>_o, <r, r>_o] reduced by the last CTA into dst[0..1].
// two double-double dots per CTA: part[4c .. 4c+3] = (hi0, lo0, hi1, lo1)
__device__ __forceinline__ void store_part2(double *part, double h0, double l0, double h1, double l1, double *sred)
{
    block_sum_dd(h0, l0, sred);
    block_sum_dd(h1, l1, sred);
    if (threadIdx.x == 0) {
        part[4 * blockIdx.x] = h0; part[4 * blockIdx.x + 1] = l0;
        part[4 * blockIdx.x + 2] = h1; part[4 * blockIdx.x + 3] = l1;
    }
}
// the fixed-order fold of the nblk CTA pairs (valid in thread 0)
__device__ __forceinline__ void fold_part2(const double *part, int nblk, double *sred, double &a0, double &a1)
{
    double h0 = 0.0, l0 = 0.0, h1 = 0.0, l1 = 0.0;
    for (int c = threadIdx.x; c < nblk; c += blockDim.x) {
        dd_add(h0, l0, ((volatile const double *)part)[4 * c], ((volatile const double *)part)[4 * c + 1]);
        dd_add(h1, l1, ((volatile const double *)part)[4 * c + 2], ((volatile const double *)part)[4 * c + 3]);
    }
    block_sum_dd(h0, l0, sred);
    block_sum_dd(h1, l1, sred);
    a0 = __dadd_rn(h0, l0);
    a1 = __dadd_rn(h1, l1);
}
__device__ __forceinline__ void last_block_finish2(double *part, int nblk, double *dst, unsigned int *counter,
                                                   double *sred, int *s_last)
{
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        *s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (*s_last) {
        fence_acq_rel_gpu();
        double a0, a1;
        fold_part2(part, nblk, sred, a0, a1);
        if (threadIdx.x == 0) { dst[0] = a0; dst[1] = a1; *counter = 0u; }
    }
}

__global__ void __launch_bounds__(VEC_THREADS)
    pcg_init_kernel(int64_t n, const uint32_t *__restrict__ mbits, const uint32_t *__restrict__ obits,
                    const double *__restrict__ b, const double *__restrict__ dinv, double *__restrict__ r,
                    double *__restrict__ p, double *__restrict__ x, double *__restrict__ part, double *dst,
                    unsigned int *counter, bool p_zero)
{
    __shared__ double sred[VEC_THREADS];
    __shared__ int s_last;
    double h0 = 0.0, l0 = 0.0, h1 = 0.0, l1 = 0.0;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x) {
        const double rv = bit_of(mbits, l) ? 0.0 : b[l];
        const double z = __dmul_rn(dinv[l], rv);
        r[l] = rv;
        p[l] = p_zero ? 0.0 : z;
        x[l] = 0.0;
        if (bit_of(obits, l)) { dd_add_prod(h0, l0, rv, z); dd_add_prod(h1, l1, rv, rv); }
    }
    store_part2(part, h0, l0, h1, l1, sred);
    last_block_finish2(part, gridDim.x, dst, counter, sred, &s_last);
}

cudaError_t launch_pcg_init(int64_t n, const uint32_t *mbits, const uint32_t *obits, const double *b,
                            const double *dinv, double *r, double *p, double *x, double *part, int nblk,
                            double *dst, unsigned int *counter, bool p_zero, cudaStream_t s)
{
    pcg_init_kernel<<<nblk, VEC_THREADS, 0, s>>>(n, mbits, obits, b, dinv, r, p, x, part, dst, counter, p_zero);
    return cudaGetLastError();
}


__global__ void pcg_init_fin_kernel(PcgScalars *sc, const double *red_all, int nranks, double *hist)
{
    const double rho = rank_sum(red_all, nranks, RED_RHO), rr = rank_sum(red_all, nranks, RED_RR);
    sc->rho = rho;
    sc->rr = rr;
    sc->bb = sqrt(rr);
    sc->iter = 0;
    sc->status = NEK_MAXIT;
    sc->done = 0;
    sc->alpha = 0.0;
    sc->beta = 0.0;
    sc->rho_next = rho;
    sc->fold_ready = 0;
    sc->booked = 0;
    if (hist) hist[0] = rr > 0.0 ? 1.0 : 0.0;
    if (!(rr > 0.0)) { sc->done = 1; sc->status = NEK_OK; }              // b = 0 -> x = 0, 0 iterations
    else if (sc->tol >= 1.0) { sc->done = 1; sc->status = NEK_OK; }      // ||r0|| <= tol ||b||
    else if (sc->maxit <= 0) { sc->done = 1; sc->status = NEK_MAXIT; }
}

cudaError_t launch_pcg_init_fin(PcgScalars *sc, const double *red_all, int nranks, double *hist, cudaStream_t s)
{
    pcg_init_fin_kernel<<<1, 1, 0, s>>>(sc, red_all, nranks, hist);
    return cudaGetLastError();
}

// alpha = rho / sigma; x += alpha p; r -= alpha w; [<r, Dinv r>_o, <r, r>_o]
// reduced by the last CTA into dst[0..1].  Two points per thread (16-byte loads).
__global__ void __launch_bounds__(VEC_THREADS, 2)
    pcg_update_kernel(int64_t n, const uint32_t *__restrict__ obits, const double *__restrict__ dinv,
                      const double *__restrict__ p, const double *__restrict__ w, double *__restrict__ x,
                      double *__restrict__ r, const double *__restrict__ red_all, int nranks, PcgScalars *sc,
                      double *__restrict__ part, double *dst, unsigned int *counter)
{
    __shared__ double sred[VEC_THREADS];
    __shared__ int s_last;
    if (*(volatile int *)&sc->done) return;
    const double sigma = rank_sum(red_all, nranks, RED_SIGMA);
    if (!(sigma > 0.0)) {                       // breakdown: <p, A p> <= 0
        if (blockIdx.x == 0 && threadIdx.x == 0) sc->status = NEK_ENOTSPD;
        return;
    }
    const double alpha = sc->rho / sigma;
    double h0 = 0.0, l0 = 0.0, h1 = 0.0, l1 = 0.0;
    const int64_t n2 = n >> 1;
    const double2 *p2 = reinterpret_cast<const double2 *>(p), *w2 = reinterpret_cast<const double2 *>(w);
    const double2 *d2 = reinterpret_cast<const double2 *>(dinv);
    double2 *x2 = reinterpret_cast<double2 *>(x), *r2 = reinterpret_cast<double2 *>(r);
    // VEC_UNROLL double2 per thread per tile, strided by blockDim (coalesced), all loads issued first
    const int64_t tile = (int64_t)VEC_UNROLL * blockDim.x;
    for (int64_t base = blockIdx.x * tile + threadIdx.x; base < n2; base += (int64_t)gridDim.x * tile) {
        double2 pv[VEC_UNROLL], wv[VEC_UNROLL], dv[VEC_UNROLL], xv[VEC_UNROLL], rv[VEC_UNROLL];
        uint32_t ow[VEC_UNROLL];
#pragma unroll
        for (int q = 0; q < VEC_UNROLL; ++q) {
            const int64_t h = base + (int64_t)q * blockDim.x;
            if (h < n2) {
                pv[q] = p2[h]; wv[q] = w2[h]; dv[q] = d2[h]; xv[q] = x2[h]; rv[q] = r2[h];
                ow[q] = __ldg(obits + ((2 * h) >> 5)) >> ((2 * h) & 31);
            }
        }
#pragma unroll
        for (int q = 0; q < VEC_UNROLL; ++q) {
            const int64_t h = base + (int64_t)q * blockDim.x;
            if (h < n2) {
                xv[q].x = fma(alpha, pv[q].x, xv[q].x); xv[q].y = fma(alpha, pv[q].y, xv[q].y);
                rv[q].x = fma(-alpha, wv[q].x, rv[q].x); rv[q].y = fma(-alpha, wv[q].y, rv[q].y);
                x2[h] = xv[q]; r2[h] = rv[q];
                if (ow[q] & 1u) { dd_add_prod(h0, l0, rv[q].x, __dmul_rn(dv[q].x, rv[q].x)); dd_add_prod(h1, l1, rv[q].x, rv[q].x); }
                if (ow[q] & 2u) { dd_add_prod(h0, l0, rv[q].y, __dmul_rn(dv[q].y, rv[q].y)); dd_add_prod(h1, l1, rv[q].y, rv[q].y); }
            }
        }
    }
    if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const int64_t l = n - 1;
        x[l] = fma(alpha, p[l], x[l]);
        const double rv = fma(-alpha, w[l], r[l]);
        r[l] = rv;
        if (bit_of(obits, l)) { dd_add_prod(h0, l0, rv, __dmul_rn(dinv[l], rv)); dd_add_prod(h1, l1, rv, rv); }
    }
    store_part2(part, h0, l0, h1, l1, sred);
    last_block_finish2(part, gridDim.x, dst, counter, sred, &s_last);
}

cudaError_t launch_pcg_update(int64_t n, const uint32_t *obits, const double *dinv, const double *p,
                              const double *w, double *x, double *r, const double *red_all, int nranks,
                              PcgScalars *sc, double *part, int nblk, double *dst, unsigned int *counter,
                              cudaStream_t s)
{
    pcg_update_kernel<<<nblk, VEC_THREADS, 0, s>>>(n, obits, dinv, p, w, x, r, red_all, nranks, sc, part, dst, counter);
    return cudaGetLastError();
}

// beta = rho'/rho; p = Dinv r + beta p.  The last block to finish updates the
// scalars (rho <- rho', iteration count, history, convergence, breakdown).
__global__ void __launch_bounds__(VEC_THREADS, 4)
    pcg_pupdate_kernel(int64_t n, const double *__restrict__ dinv, const double *__restrict__ r,
                       double *__restrict__ p, const double *__restrict__ red_all, int nranks, PcgScalars *sc,
                       double *__restrict__ hist, unsigned int *counter)
{
    __shared__ bool last;
    if (*(volatile int *)&sc->done) return;
    const bool breakdown = *(volatile int *)&sc->status == NEK_ENOTSPD;
    const double rho1 = rank_sum(red_all, nranks, RED_RHO), rr = rank_sum(red_all, nranks, RED_RR);
    const double rho = sc->rho, bb = sc->bb, tol = sc->tol;
    const bool conv = sqrt(rr) <= tol * bb;
    if (!breakdown && !conv) {
        const double beta = rho1 / rho;
        const int64_t n2 = n >> 1;
        const double2 *d2 = reinterpret_cast<const double2 *>(dinv), *r2 = reinterpret_cast<const double2 *>(r);
        double2 *p2 = reinterpret_cast<double2 *>(p);
        const int64_t tile = (int64_t)VEC_UNROLL * blockDim.x;
        for (int64_t base = blockIdx.x * tile + threadIdx.x; base < n2; base += (int64_t)gridDim.x * tile) {
            double2 dv[VEC_UNROLL], rv[VEC_UNROLL], pv[VEC_UNROLL];
#pragma unroll
            for (int q = 0; q < VEC_UNROLL; ++q) {
                const int64_t h = base + (int64_t)q * blockDim.x;
                if (h < n2) { dv[q] = d2[h]; rv[q] = r2[h]; pv[q] = p2[h]; }
            }
#pragma unroll
            for (int q = 0; q < VEC_UNROLL; ++q) {
                const int64_t h = base + (int64_t)q * blockDim.x;
                if (h < n2) {
                    pv[q].x = fma(beta, pv[q].x, dv[q].x * rv[q].x);
                    pv[q].y = fma(beta, pv[q].y, dv[q].y * rv[q].y);
                    p2[h] = pv[q];
                }
            }
        }
        if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) p[n - 1] = fma(beta, p[n - 1], dinv[n - 1] * r[n - 1]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        *counter = 0u;
        if (breakdown) { sc->done = 1; return; }
        const int it = sc->iter + 1;
        sc->iter = it;
        sc->rho = rho1;
        sc->rr = rr;
        if (hist) hist[it] = sqrt(rr) / bb;
        if (conv) { sc->done = 1; sc->status = NEK_OK; }
        else if (it >= sc->maxit) { sc->done = 1; sc->status = NEK_MAXIT; }
        __threadfence();
    }
}

cudaError_t launch_pcg_pupdate(int64_t n, const double *dinv, const double *r, double *p, const double *red_all,
                               int nranks, PcgScalars *sc, double *hist, unsigned int *counter, int nblk,
                               cudaStream_t s)
{
    pcg_pupdate_kernel<<<nblk, VEC_THREADS, 0, s>>>(n, dinv, r, p, red_all, nranks, sc, hist, counter);
    return cudaGetLastError();
}

// ---------------------------------------------------------- fused PCG path
// Iteration bookkeeping after <r, Dinv r> and <r, r> of the new residual are
// known: history, convergence / maxit, the pending alpha for the deferred x
// update and beta for the next direction.
__device__ __forceinline__ void pcg_bookkeep(PcgScalars *sc, double rho1, double rr, double alpha, double *hist)
{
    const int it = sc->iter + 1;
    sc->iter = it;
    sc->rr = rr;
    sc->alpha = alpha;
    if (hist) hist[it] = sqrt(rr) / sc->bb;
    sc->beta = rho1 / sc->rho;
    sc->rho = rho1;
    if (sqrt(rr) <= sc->tol * sc->bb) { sc->done = 1; sc->status = NEK_OK; }
    else if (it >= sc->maxit) { sc->done = 1; sc->status = NEK_MAXIT; }
    __threadfence();
}

template <int UNR, int MINB>
__global__ void __launch_bounds__(VEC_THREADS, MINB)
    pcg_update_fused_kernel(int64_t n, const uint32_t *__restrict__ obits, const double *__restrict__ dinv,
                            const double *__restrict__ w, double *__restrict__ r, const double *__restrict__ red_all,
                            int nranks, PcgScalars *sc, double *hist, double *__restrict__ part, double *dst,
                            unsigned int *counter, P2PMail mail, int keep, int defer, int pf)
{
    __shared__ double sred[VEC_THREADS];
    __shared__ int s_last;
    __shared__ double s_sig[3];
    const uint64_t pol = tma::policy_keep(keep & 1);
    const int64_t n2 = n >> 1;
    const int64_t tile = (int64_t)UNR * blockDim.x;
    int64_t base = blockIdx.x * tile + threadIdx.x;
    double2 wv[UNR], dv[UNR], rv[UNR];
    uint32_t ow[UNR];
    auto load = [&](int64_t b0) {
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
            const int64_t h = b0 + (int64_t)q * blockDim.x;
            if (h < n2) {
                wv[q] = tma::ld2(w + 2 * h, pol); dv[q] = tma::ld2(dinv + 2 * h, pol); rv[q] = tma::ld2(r + 2 * h, pol);
                ow[q] = tma::ldu(obits + ((2 * h) >> 5), pol) >> ((2 * h) & 31);
            }
        }
    };
    // the first tile's streams are issued before the dependent scalar reads (done, sigma, rho), so
    // their latencies overlap; w, r, Dinv are complete (stream order) whatever the scalars say
    load(base);
    // the scalars are final when the kernel starts (stream order): their loads are issued together
    // with the convergence flag's instead of after it
    // defer (P2P): rho of this iteration is rho_next (the Ax that pulled (rho', rr) set it); CTA 0
    // counts the iteration and the next Ax records it (ax.cu, DEFER_MAIL)
    const double rho0 = defer ? sc->rho_next : sc->rho;
    double sigma = (mail.nranks > 1) ? 0.0 : rank_sum(red_all, nranks, RED_SIGMA);
    if (*(volatile int *)&sc->done) return;
    if (mail.nranks > 1) {                       // sigma of every rank from the mailbox (channel 0)
        if (threadIdx.x < 32) mail_pull_warp(mail, 0, s_sig);
        __syncthreads();
        sigma = s_sig[0];
        if (blockIdx.x == 0 && threadIdx.x == 0) sc->sigma = sigma;
    }
    if (!(sigma > 0.0)) {                       // breakdown: <p, A p> <= 0, or a peer timed out (NaN)
        if (blockIdx.x == 0 && threadIdx.x == 0) { sc->status = NEK_ENOTSPD; sc->alpha = 0.0; sc->done = 1; }
        return;
    }
    const double alpha = rho0 / sigma;
    if (defer && blockIdx.x == 0 && threadIdx.x == 0) {
        sc->iter = sc->iter + 1;
        sc->rho = rho0;
        sc->alpha = alpha;
        sc->fold_ready = 1;
    }
    double h0 = 0.0, l0 = 0.0, h1 = 0.0, l1 = 0.0;
    double g0 = 0.0, k0 = 0.0, g1 = 0.0, k1 = 0.0;   // the .y points: two independent Dot2 chains per dot
    for (bool first = true; base < n2; base += (int64_t)gridDim.x * tile, first = false) {
        if (pf && threadIdx.x == 0) {   // vectors beyond L2: this CTA's next tile of w, r, Dinv toward L2
            const int64_t nb = base - threadIdx.x + (int64_t)gridDim.x * tile;
            if (nb < n2) {
                const uint32_t bytes = (uint32_t)(16 * (nb + tile <= n2 ? tile : n2 - nb));
                tma::prefetch_l2(w + 2 * nb, bytes);
                tma::prefetch_l2(r + 2 * nb, bytes);
                tma::prefetch_l2(dinv + 2 * nb, bytes);
            }
        }
        if (!first) load(base);
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
            const int64_t h = base + (int64_t)q * blockDim.x;
            if (h < n2) {
                rv[q].x = fma(-alpha, wv[q].x, rv[q].x); rv[q].y = fma(-alpha, wv[q].y, rv[q].y);
                tma::st2(r + 2 * h, rv[q], pol);
                if (ow[q] & 1u) { dd_add_prod(h0, l0, rv[q].x, __dmul_rn(dv[q].x, rv[q].x)); dd_add_prod(h1, l1, rv[q].x, rv[q].x); }
                if (ow[q] & 2u) { dd_add_prod(g0, k0, rv[q].y, __dmul_rn(dv[q].y, rv[q].y)); dd_add_prod(g1, k1, rv[q].y, rv[q].y); }
            }
        }
    }
    if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const int64_t l = n - 1;
        const double rl = fma(-alpha, w[l], r[l]);
        r[l] = rl;
        if (bit_of(obits, l)) { dd_add_prod(h0, l0, rl, __dmul_rn(dinv[l], rl)); dd_add_prod(h1, l1, rl, rl); }
    }
    dd_add(h0, l0, g0, k0);
    dd_add(h1, l1, g1, k1);
    store_part2(part, h0, l0, h1, l1, sred);
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        fence_acq_rel_gpu();
        double b0, b1;
        fold_part2(part, (int)gridDim.x, sred, b0, b1);
        if (threadIdx.x == 0) {
            *counter = 0u;
            if (nranks == 1) pcg_bookkeep(sc, b0, b1, alpha, hist);
            else if (mail.nranks > 1) mail_push(mail, 1, b0, b1, 0.0);   // to every rank (channel 1)
            else { dst[0] = b0; dst[1] = b1; }
        }
    }
}

cudaError_t launch_pcg_update_fused(int64_t n, const uint32_t *obits, const double *dinv, const double *w, double *r,
                                    const double *red_all, int nranks, PcgScalars *sc, double *hist, double *part,
                                    int nblk, double *dst, unsigned int *counter, cudaStream_t s,
                                    const P2PMail *mail, int keep, int defer, bool pf)
{
    P2PMail m;
    if (mail) m = *mail;
    const int per_sm = nblk / device_sms();
    if (per_sm == 3)
        pcg_update_fused_kernel<3, 3><<<nblk, VEC_THREADS, 0, s>>>(n, obits, dinv, w, r, red_all, nranks, sc, hist,
                                                                   part, dst, counter, m, keep, defer, pf ? 1 : 0);
    else if (per_sm >= 8)
        pcg_update_fused_kernel<2, 8><<<nblk, VEC_THREADS, 0, s>>>(n, obits, dinv, w, r, red_all, nranks, sc, hist,
                                                                   part, dst, counter, m, keep, defer, pf ? 1 : 0);
    else if (per_sm >= 4)
        pcg_update_fused_kernel<2, 4><<<nblk, VEC_THREADS, 0, s>>>(n, obits, dinv, w, r, red_all, nranks, sc, hist,
                                                                   part, dst, counter, m, keep, defer, pf ? 1 : 0);
    else
        pcg_update_fused_kernel<4, 2><<<nblk, VEC_THREADS, 0, s>>>(n, obits, dinv, w, r, red_all, nranks, sc, hist,
                                                                   part, dst, counter, m, keep, defer, pf ? 1 : 0);
    return cudaGetLastError();
}

// ------------------------------------------------ deferred reductions (single rank)
// The residual update of the single-rank N = 7 path without last-CTA work: every CTA folds the Ax
// launch's sigma partials itself (the same fixed order in every CTA, while its first tile of w, r, Dinv
// is in flight), and leaves its own (rho', rr) partials; the next Ax launch folds those at entry and does
// the bookkeeping (ax.cu), or pcg_defer_finish does after the last update of a solve.  Every value is
// computed as on the last-CTA path; only the grouping of the double-double folds differs (within an ulp).
// No kernel writes a scalar that another CTA of the same launch reads at entry: the update counts the
// iteration (sc->iter), the Ax that folds its partials records them (sc->booked, history, convergence).
__device__ __forceinline__ double fold_pairs(const double *part, int count, double *sred)
{
    double hi = 0.0, lo = 0.0;
    for (int c = threadIdx.x; c < count; c += blockDim.x) dd_add(hi, lo, part[2 * c], part[2 * c + 1]);
    block_sum_dd(hi, lo, sred);
    return __dadd_rn(hi, lo);
}

template <int UNR, int MINB>
__global__ void __launch_bounds__(VEC_THREADS, MINB)
    pcg_update_deferred_kernel(int64_t n, const uint32_t *__restrict__ obits, const double *__restrict__ dinv,
                               const double *__restrict__ w, double *__restrict__ r, const double *__restrict__ axpart,
                               int nax, PcgScalars *sc, double *__restrict__ upart, int keep, int pf)
{
    __shared__ double sred[VEC_THREADS];
    __shared__ double s_sig;
    const uint64_t pol = tma::policy_keep(keep & 1);
    const int64_t n2 = n >> 1;
    const int64_t tile = (int64_t)UNR * blockDim.x;
    int64_t base = blockIdx.x * tile + threadIdx.x;
    double2 wv[UNR], dv[UNR], rv[UNR];
    uint32_t ow[UNR];
    auto load = [&](int64_t b0) {
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
            const int64_t h = b0 + (int64_t)q * blockDim.x;
            if (h < n2) {
                wv[q] = tma::ld2(w + 2 * h, pol); dv[q] = tma::ld2(dinv + 2 * h, pol); rv[q] = tma::ld2(r + 2 * h, pol);
                ow[q] = tma::ldu(obits + ((2 * h) >> 5), pol) >> ((2 * h) & 31);
            }
        }
    };
    load(base);
    const double rho = sc->rho_next;
    if (*(volatile int *)&sc->done) return;
    const double sg = fold_pairs(axpart, nax, sred);   // sigma of the Ax launch, folded in every CTA
    if (threadIdx.x == 0) s_sig = sg;
    __syncthreads();
    const double sigma = s_sig;
    if (!(sigma > 0.0)) {                       // breakdown: <p, A p> <= 0
        if (blockIdx.x == 0 && threadIdx.x == 0) { sc->status = NEK_ENOTSPD; sc->alpha = 0.0; sc->done = 1; }
        return;
    }
    const double alpha = rho / sigma;
    if (blockIdx.x == 0 && threadIdx.x == 0) {   // the Ax launch is complete: rho moves on, alpha is pending
        sc->iter = sc->iter + 1;
        sc->rho = rho;
        sc->alpha = alpha;
        sc->sigma = sigma;
        sc->fold_ready = 1;
    }
    double h0 = 0.0, l0 = 0.0, h1 = 0.0, l1 = 0.0, g0 = 0.0, k0 = 0.0, g1 = 0.0, k1 = 0.0;
    for (bool first = true; base < n2; base += (int64_t)gridDim.x * tile, first = false) {
        if (pf && threadIdx.x == 0) {   // vectors beyond L2: this CTA's next tile of w, r, Dinv toward L2
            const int64_t nb = base - threadIdx.x + (int64_t)gridDim.x * tile;
            if (nb < n2) {
                const uint32_t bytes = (uint32_t)(16 * (nb + tile <= n2 ? tile : n2 - nb));
                tma::prefetch_l2(w + 2 * nb, bytes);
                tma::prefetch_l2(r + 2 * nb, bytes);
                tma::prefetch_l2(dinv + 2 * nb, bytes);
            }
        }
        if (!first) load(base);
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
            const int64_t h = base + (int64_t)q * blockDim.x;
            if (h < n2) {
                rv[q].x = fma(-alpha, wv[q].x, rv[q].x); rv[q].y = fma(-alpha, wv[q].y, rv[q].y);
                tma::st2(r + 2 * h, rv[q], pol);
                if (ow[q] & 1u) { dd_add_prod(h0, l0, rv[q].x, __dmul_rn(dv[q].x, rv[q].x)); dd_add_prod(h1, l1, rv[q].x, rv[q].x); }
                if (ow[q] & 2u) { dd_add_prod(g0, k0, rv[q].y, __dmul_rn(dv[q].y, rv[q].y)); dd_add_prod(g1, k1, rv[q].y, rv[q].y); }
            }
        }
    }
    if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const int64_t l = n - 1;
        const double rl = fma(-alpha, w[l], r[l]);
        r[l] = rl;
        if (bit_of(obits, l)) { dd_add_prod(h0, l0, rl, __dmul_rn(dinv[l], rl)); dd_add_prod(h1, l1, rl, rl); }
    }
    dd_add(h0, l0, g0, k0);
    dd_add(h1, l1, g1, k1);
    store_part2(upart, h0, l0, h1, l1, sred);
}

cudaError_t launch_pcg_update_deferred(int64_t n, const uint32_t *obits, const double *dinv, const double *w,
                                       double *r, const double *axpart, int nax, PcgScalars *sc, double *upart,
                                       int nblk, int keep, cudaStream_t s, bool pf)
{
    const int per_sm = nblk / device_sms();
    if (per_sm >= 4)
        pcg_update_deferred_kernel<2, 4><<<nblk, VEC_THREADS, 0, s>>>(n, obits, dinv, w, r, axpart, nax, sc, upart,
                                                                     keep, pf ? 1 : 0);
    else if (per_sm == 3)
        pcg_update_deferred_kernel<3, 3><<<nblk, VEC_THREADS, 0, s>>>(n, obits, dinv, w, r, axpart, nax, sc, upart,
                                                                     keep, pf ? 1 : 0);
    else
        pcg_update_deferred_kernel<4, 2><<<nblk, VEC_THREADS, 0, s>>>(n, obits, dinv, w, r, axpart, nax, sc, upart,
                                                                     keep, pf ? 1 : 0);
    return cudaGetLastError();
}

// after the last update of a solve when no Ax followed it: fold its partials and book the iteration
__global__ void __launch_bounds__(VEC_THREADS) pcg_defer_finish_kernel(PcgScalars *sc, const double *upart,
                                                                      int nupd, double *hist, P2PMail mail)
{
    __shared__ double sred[VEC_THREADS];
    if (*(volatile int *)&sc->done || !*(volatile int *)&sc->fold_ready || sc->booked >= sc->iter) return;
    double a0, a1;
    if (mail.nranks > 1) {   // P2P: every rank's (rho', rr) from the mailbox (channel 1)
        if (threadIdx.x < 32) mail_pull_warp(mail, 1, sred);
        __syncthreads();
        a0 = sred[0]; a1 = sred[1];
    } else {
        fold_part2(upart, nupd, sred, a0, a1);
    }
    if (threadIdx.x == 0) {
        const int it = sc->iter;
        sc->booked = it;
        sc->rr = a1;
        if (hist) hist[it] = sqrt(a1) / sc->bb;
        sc->beta = a0 / sc->rho;
        sc->rho_next = a0;
        if (sqrt(a1) <= sc->tol * sc->bb) { sc->done = 1; sc->status = NEK_OK; }
        else if (it >= sc->maxit) { sc->done = 1; sc->status = NEK_MAXIT; }
        __threadfence();
    }
}

cudaError_t launch_pcg_defer_finish(PcgScalars *sc, const double *upart, int nupd, double *hist, cudaStream_t s,
                                    const P2PMail *mail)
{
    P2PMail m;
    if (mail) m = *mail;
    pcg_defer_finish_kernel<<<1, VEC_THREADS, 0, s>>>(sc, upart, nupd, hist, m);
    return cudaGetLastError();
}

// P2P: pull <r, Dinv r> and <r, r> of every rank (channel 1) and do the bookkeeping
__global__ void pcg_fin_p2p_kernel(PcgScalars *sc, P2PMail mail, double *hist)
{
    __shared__ double v[3];
    if (sc->done) return;
    mail_pull_warp(mail, 1, v);
    __syncwarp();
    if (threadIdx.x == 0) pcg_bookkeep(sc, v[0], v[1], sc->rho / sc->sigma, hist);
}

cudaError_t launch_pcg_fin_p2p(PcgScalars *sc, const P2PMail &mail, double *hist, cudaStream_t s)
{
    pcg_fin_p2p_kernel<<<1, 32, 0, s>>>(sc, mail, hist);
    return cudaGetLastError();
}

__global__ void pcg_iter_fin_kernel(PcgScalars *sc, const double *red_all, int nranks, double *hist)
{
    if (sc->done) return;
    const double sigma = rank_sum(red_all, nranks, RED_SIGMA);
    const double alpha = sc->rho / sigma;
    pcg_bookkeep(sc, rank_sum(red_all, nranks, RED_RHO), rank_sum(red_all, nranks, RED_RR), alpha, hist);
}

cudaError_t launch_pcg_iter_fin(PcgScalars *sc, const double *red_all, int nranks, double *hist, cudaStream_t s)
{
    pcg_iter_fin_kernel<<<1, 1, 0, s>>>(sc, red_all, nranks, hist);
    return cudaGetLastError();
}

// the deferred x += alpha p of the last iteration
__global__ void pcg_xfinal_kernel(int64_t n, const PcgScalars *sc, const double *__restrict__ p, double *__restrict__ x)
{
    const double alpha = sc->alpha;
    if (alpha == 0.0 || sc->status == NEK_ENOTSPD) return;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x)
        x[l] = fma(alpha, p[l], x[l]);
}

cudaError_t launch_pcg_xfinal(int64_t n, const PcgScalars *sc, const double *p, double *x, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    pcg_xfinal_kernel<<<vec_blocks(), VEC_THREADS, 0, s>>>(n, sc, p, x);
    return cudaGetLastError();
}

// ------------------------------------------------------- L2 residency release
// After an L2-resident solve the kept lines would stay evict_last (persisting) and squeeze every
// later kernel into the rest of the L2: demote them to evict_normal, one 128-byte line per step.
__global__ void l2_demote_kernel(L2Ranges R)
{
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int q = 0; q < R.count; ++q) {
        const char *base = reinterpret_cast<const char *>(R.ptr[q]);
        const int64_t lines = (R.bytes[q] + 127) / 128;
        for (int64_t k = tid; k < lines; k += nth)
            asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(
                             reinterpret_cast<uintptr_t>(base + k * 128) & ~(uintptr_t)127)
                         : "memory");
    }
}

cudaError_t launch_l2_demote(const L2Ranges &R, cudaStream_t s)
{
    if (R.count <= 0) return cudaSuccess;
    l2_demote_kernel<<<4 * device_sms(), 256, 0, s>>>(R);
    return cudaGetLastError();
}

// ------------------------------------------------ NVLink peer-memory exchange
// Every rank's reduction slots to every rank over peer memory (mailbox layout: [channel][epoch
// parity][rank][4] doubles, slot 3 holds the epoch as u64; the parity split means a slot is rewritten
// only two exchanges later, by which time its reader has provably consumed it).  phase: 3 = push and
// pull in one launch (one process per GPU, all ranks' launches run concurrently); 1 = push only,
// 2 = pull only (the loopback group runs the pushes of every rank before any pull).
__global__ void red_exchange_kernel(int channel, int me, int nranks, const double *__restrict__ red_loc,
                                    double *__restrict__ red_all, double *mbox, double *const *peer_mbox,
                                    uint64_t *epochs, int *err, uint64_t timeout_ns, int phase)
{
    __shared__ uint64_t s_e;
    const int q = threadIdx.x;
    if (q == 0) s_e = (phase & 1) ? ++epochs[channel] : epochs[channel];
    __syncthreads();
    const uint64_t e = s_e;
    const size_t base = ((size_t)channel * 2 + (e & 1)) * nranks;
    if ((phase & 1) && q < nranks) {
        double *dst = (q == me ? mbox : peer_mbox[q]) + (base + me) * 4;
        dst[0] = red_loc[0]; dst[1] = red_loc[1]; dst[2] = red_loc[2];
        st_release_sys(reinterpret_cast<uint64_t *>(dst + 3), e);   // release: orders the values before it
    }
    if ((phase & 2) && q < nranks) {
        const double *src = mbox + (base + q) * 4;
        const double nan = __longlong_as_double(0x7ff8000000000000ll);
        const bool ok = wait_epoch(reinterpret_cast<const uint64_t *>(src + 3), e, err, timeout_ns);
        red_all[q * RED_N + 0] = ok ? ((volatile const double *)src)[0] : nan;
        red_all[q * RED_N + 1] = ok ? ((volatile const double *)src)[1] : nan;
        red_all[q * RED_N + 2] = ok ? ((volatile const double *)src)[2] : nan;
    }
}

cudaError_t launch_red_exchange(int channel, const P2PMail &M, const double *red_loc, double *red_all, int phase,
                                cudaStream_t s)
{
    red_exchange_kernel<<<1, 32, 0, s>>>(channel, M.me, M.nranks, red_loc, red_all, M.mbox, M.peer_mbox, M.epochs,
                                         M.err, M.timeout_ns, phase);
    return cudaGetLastError();
}

// ------------------------------------------------ projection (NEXT #2)
// out_part[block][i] = block partial of <V_i, y>_owner for i < l (V is [l][n] row-major);
// the caller reduces the partials in block order.  l <= PROJ_MAXV.
constexpr int PROJ_MAXV = 32;

__global__ void __launch_bounds__(256)
    multidot_kernel(int64_t n, int l, const double *__restrict__ V, const double *__restrict__ y,
                    const uint32_t *__restrict__ obits, double *__restrict__ out_part)
{
    __shared__ double sred[32];
    double acc[PROJ_MAXV];
#pragma unroll
    for (int i = 0; i < PROJ_MAXV; ++i) acc[i] = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        if (!bit_of(obits, p)) continue;
        const double yv = y[p];
#pragma unroll
        for (int i = 0; i < PROJ_MAXV; ++i)
            if (i < l) acc[i] = fma(V[(int64_t)i * n + p], yv, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < PROJ_MAXV; ++i) {
        if (i >= l) break;
        const double s2 = block_sum(acc[i], sred);
        if (threadIdx.x == 0) out_part[(int64_t)blockIdx.x * l + i] = s2;
    }
}

cudaError_t launch_multidot(int64_t n, int l, const double *V, const double *y, const uint32_t *obits,
                            double *out_part, int nblk, cudaStream_t s)
{
    if (l <= 0) return cudaSuccess;
    multidot_kernel<<<nblk, 256, 0, s>>>(n, l, V, y, obits, out_part);
    return cudaGetLastError();
}

// y = a * y + sum_{i<l} c[i] * V_i  (c on the device)
__global__ void multiaxpy_kernel(int64_t n, int l, double a, double *__restrict__ y, const double *__restrict__ V,
                                 const double *__restrict__ c)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        double v = a == 0.0 ? 0.0 : a * y[p];
        for (int i = 0; i < l; ++i) v = fma(c[i], V[(int64_t)i * n + p], v);
        y[p] = v;
    }
}

cudaError_t launch_multiaxpy(int64_t n, int l, double a, double *y, const double *V, const double *c, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    multiaxpy_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 8 * device_sms()), 256, 0, s>>>(n, l, a, y, V, c);
    return cudaGetLastError();
}

// z = alpha * x + beta * y
__global__ void axpby_kernel(int64_t n, double alpha, const double *__restrict__ x, double beta,
                             const double *__restrict__ y, double *__restrict__ z)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        z[p] = fma(alpha, x[p], beta * y[p]);
}

cudaError_t launch_axpby(int64_t n, double alpha, const double *x, double beta, const double *y, double *z,
                         cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    axpby_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 8 * device_sms()), 256, 0, s>>>(n, alpha, x, beta, y, z);
    return cudaGetLastError();
}


#include "pmg_kernels.cuh"

template cudaError_t launch_copy_mask<double>(int64_t, const uint32_t *, const double *, double *, cudaStream_t);
template cudaError_t launch_copy_mask<float>(int64_t, const uint32_t *, const float *, float *, cudaStream_t);

}  // namespace nekb200
