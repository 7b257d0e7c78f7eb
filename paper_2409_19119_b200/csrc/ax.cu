// ax.cu -- the local operator of the hot path: geometric factors, the Ax
// kernels and the Jacobi diagonal.
//
//   geom      geometric factors of the isoparametric map
//   ax        local Helmholtz apply w = h1 D^T G D u + h2 wJ u with the Dirichlet mask on input and
//             output and an optional <u, w> partial (sum factorisation, O(N^4) work,
//             O(N^3) memory): v5 (N = 7, FP64 tensor cores), v6 (N <= 9, TMA metric ring), v0 (any N)
//   diag      exact diagonal of h1 K_L + h2 B_L (reading 10)
// D lives in constant memory, so every kernel that reads it is in this translation unit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "dev_common.cuh"

namespace nekb200 {

__constant__ double c_D[16][256];   // D for every order N (row-major, (N+1)^2 used)
__constant__ float c_Df[16][256];   // the same in FP32 (reduced-precision pMG levels, NEXT #3)

cudaError_t upload_D(int N, const double *D)
{
    cudaError_t e = cudaMemcpyToSymbol(c_D, D, sizeof(double) * (N + 1) * (N + 1), sizeof(double) * 256 * N,
                                       cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    float Df[256];
    for (int i = 0; i < (N + 1) * (N + 1); ++i) Df[i] = (float)D[i];
    return cudaMemcpyToSymbol(c_Df, Df, sizeof(float) * (N + 1) * (N + 1), sizeof(float) * 256 * N,
                              cudaMemcpyHostToDevice);
}

// ------------------------------------------------------------------ geometry
// One thread per local point; D from constant memory.  G_ab = w_q J grad r_a .
// grad r_b (a <= b: rr rs rt ss st tt), wJ = w_q J.  J <= 0 -> smallest bad l in *bad.
__global__ void geom_kernel(int N, int64_t n, const double *__restrict__ xyz, const double *__restrict__ wq,
                            double *__restrict__ G, double *__restrict__ wJ, unsigned long long *bad)
{
    const int Nq = N + 1, P2 = Nq * Nq, P3 = P2 * Nq;
    const double *D = c_D[N];
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / P3;
        const int q = (int)(l - e * P3), i = q % Nq, j = (q / Nq) % Nq, k = q / P2;
        const double *X = xyz + e * P3, *Y = xyz + n + e * P3, *Z = xyz + 2 * n + e * P3;
        double xr = 0, xs = 0, xt = 0, yr = 0, ys = 0, yt = 0, zr = 0, zs = 0, zt = 0;
        for (int m = 0; m < Nq; ++m) {
            const double dr = D[i * Nq + m], ds = D[j * Nq + m], dt = D[k * Nq + m];
            const int a = m + Nq * j + P2 * k, b = i + Nq * m + P2 * k, c = i + Nq * j + P2 * m;
            xr = fma(dr, X[a], xr); yr = fma(dr, Y[a], yr); zr = fma(dr, Z[a], zr);
            xs = fma(ds, X[b], xs); ys = fma(ds, Y[b], ys); zs = fma(ds, Z[b], zs);
            xt = fma(dt, X[c], xt); yt = fma(dt, Y[c], yt); zt = fma(dt, Z[c], zt);
        }
        // cofactors of dx/dr: rows of J * (dx/dr)^{-1}
        const double c_rx = ys * zt - yt * zs, c_ry = xt * zs - xs * zt, c_rz = xs * yt - xt * ys;
        const double c_sx = yt * zr - yr * zt, c_sy = xr * zt - xt * zr, c_sz = xt * yr - xr * yt;
        const double c_tx = yr * zs - ys * zr, c_ty = xs * zr - xr * zs, c_tz = xr * ys - xs * yr;
        const double J = xr * c_rx + yr * c_ry + zr * c_rz;
        if (!(J > 0.0)) atomicMin(bad, (unsigned long long)l);
        const double w = wq[i] * wq[j] * wq[k];
        const double f = w / J;   // w J * (1/J)^2
        double *Ge = G + e * 6 * (int64_t)P3 + q;
        Ge[0 * P3] = f * (c_rx * c_rx + c_ry * c_ry + c_rz * c_rz);
        Ge[1 * P3] = f * (c_rx * c_sx + c_ry * c_sy + c_rz * c_sz);
        Ge[2 * P3] = f * (c_rx * c_tx + c_ry * c_ty + c_rz * c_tz);
        Ge[3 * P3] = f * (c_sx * c_sx + c_sy * c_sy + c_sz * c_sz);
        Ge[4 * P3] = f * (c_sx * c_tx + c_sy * c_ty + c_sz * c_tz);
        Ge[5 * P3] = f * (c_tx * c_tx + c_ty * c_ty + c_tz * c_tz);
        wJ[l] = w * J;
    }
}

cudaError_t launch_geom(int N, int64_t E, const double *xyz, double *G, double *wJ, const double *wq,
                        unsigned long long *bad, cudaStream_t s)
{
    const int64_t n = E * (N + 1) * (N + 1) * (N + 1);
    if (n == 0) return cudaSuccess;
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 16 * device_sms());
    geom_kernel<<<blocks, 256, 0, s>>>(N, n, xyz, wq, G, wJ, bad);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- Ax v0
// Any order N.  EPB elements per CTA (threadIdx.y), (N+1)^2 threads per element
// (threadIdx.x, i fastest), the k-column of u and of the result in registers,
// one (i,j) slice per element in shared memory at a time.  One <u, w> partial
// per CTA.
constexpr int v0_epb(int NQ) { return NQ * NQ >= 128 ? 1 : 128 / (NQ * NQ); }

template <int NQ>
__global__ void __launch_bounds__(NQ *NQ *v0_epb(NQ))
    ax_v0_kernel(int64_t nelem, int64_t eoff, const int32_t *__restrict__ elist, const double *__restrict__ u,
                 const double *__restrict__ G, const double *__restrict__ wJ, const uint32_t *__restrict__ mbits,
                 double h1, double h2, double *__restrict__ w, double *__restrict__ part, const int *__restrict__ done)
{
    constexpr int P2 = NQ * NQ, P3 = P2 * NQ, N = NQ - 1, EPB = v0_epb(NQ);
    if (done && *(volatile const int *)done) return;
    __shared__ double sD[NQ * NQ];
    __shared__ double sa[EPB][P2], sb[EPB][P2];
    __shared__ double sred[2][P2 * EPB];
    const int t = threadIdx.x, g = threadIdx.y, i = t % NQ, j = t / NQ;
    const int64_t rel = (int64_t)blockIdx.x * EPB + g;
    const bool valid = rel < nelem;
    const int64_t pos = eoff + (valid ? rel : 0);
    const int64_t e = elist ? (int64_t)elist[pos] : pos;
    for (int q = t + P2 * g; q < NQ * NQ; q += P2 * EPB) sD[q] = c_D[N][q];
    const double *ue = u + e * P3;
    const double *Ge = G + e * 6 * (int64_t)P3;
    double ru[NQ], rw[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
        const int64_t l = e * P3 + k * P2 + t;
        double v = valid ? ue[k * P2 + t] : 0.0;
        if (valid && mbits && bit_of(mbits, l)) v = 0.0;
        ru[k] = v;
        rw[k] = 0.0;
    }
    __syncthreads();
    double *sag = sa[g], *sbg = sb[g];
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
        sag[t] = ru[k];
        __syncthreads();
        double ur = 0, us = 0, ut = 0;
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
            ur = fma(sD[i * NQ + m], sag[j * NQ + m], ur);
            us = fma(sD[j * NQ + m], sag[m * NQ + i], us);
            ut = fma(sD[k * NQ + m], ru[m], ut);
        }
        const int q = k * P2 + t;
        double Grr = 0, Grs = 0, Grt = 0, Gss = 0, Gst = 0, Gtt = 0;
        if (valid) {
            Grr = Ge[q]; Grs = Ge[P3 + q]; Grt = Ge[2 * P3 + q];
            Gss = Ge[3 * P3 + q]; Gst = Ge[4 * P3 + q]; Gtt = Ge[5 * P3 + q];
        }
        const double gr = Grr * ur + Grs * us + Grt * ut;
        const double gs = Grs * ur + Gss * us + Gst * ut;
        const double gt = Grt * ur + Gst * us + Gtt * ut;
        __syncthreads();
        sag[t] = gr;
        sbg[t] = gs;
        __syncthreads();
        double acc = 0;
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
            acc = fma(sD[m * NQ + i], sag[j * NQ + m], acc);
            acc = fma(sD[m * NQ + j], sbg[m * NQ + i], acc);
        }
        rw[k] += acc;
#pragma unroll
        for (int m = 0; m < NQ; ++m) rw[m] = fma(sD[k * NQ + m], gt, rw[m]);
        __syncthreads();
    }
    double dhi = 0.0, dlo = 0.0;
    if (valid) {
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            const int64_t l = e * P3 + k * P2 + t;
            double v = h1 * rw[k];
            if (h2 != 0.0) v = fma(h2 * wJ[l], ru[k], v);
            if (mbits && bit_of(mbits, l)) v = 0.0;
            w[l] = v;
            dd_add_prod(dhi, dlo, ru[k], v);
        }
    }
    if (part) {
        // fixed-order CTA sum (double-double) over the linear thread index
        const int lt = t + P2 * g, nt = P2 * EPB;
        sred[0][lt] = dhi;
        sred[1][lt] = dlo;
        __syncthreads();
        for (int s2 = 512; s2 > 0; s2 >>= 1) {
            if (s2 < nt && lt < s2 && lt + s2 < nt) {
                double h = sred[0][lt], lo = sred[1][lt];
                dd_add(h, lo, sred[0][lt + s2], sred[1][lt + s2]);
                sred[0][lt] = h;
                sred[1][lt] = lo;
            }
            __syncthreads();
        }
        if (lt == 0) { part[2 * blockIdx.x] = sred[0][0]; part[2 * blockIdx.x + 1] = sred[1][0]; }
    }
}

// Fixed-order reduction of count (hi, lo) partials (part[2c], part[2c+1]) into dst[0] = hi + lo.
__global__ void reduce_kernel(const double *__restrict__ part, int64_t count, int nd, double *__restrict__ dst,
                              const int *done)
{
    __shared__ double sred[64];
    if (done && *(volatile const int *)done) return;
    double hi = 0.0, lo = 0.0;
    for (int64_t c = threadIdx.x; c < count; c += blockDim.x) dd_add(hi, lo, part[2 * c], part[2 * c + 1]);
    block_sum_dd(hi, lo, sred);
    if (threadIdx.x == 0) dst[0] = __dadd_rn(hi, lo);
}

cudaError_t launch_reduce(const double *part, int64_t count, int nd, double *dst, const int *done, cudaStream_t s)
{
    reduce_kernel<<<1, 1024, 0, s>>>(part, count, nd, dst, done);
    return cudaGetLastError();
}

__device__ __forceinline__ void dmma8x8x4(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}


// ------------------------------------------------------------------- Ax v5
// v4 with the roles of j and k exchanged: a warp owns the k-slabs {2w, 2w+1},
// lane (q, r) the points (i = 2q + v, j = r, k).  Every per-slab load or store
// of a warp is then one contiguous 512-byte (j, i) plane (4 L1 wavefronts
// instead of 8), the t contraction runs on the thread's own k-line in
// registers, and DMMA does the r (over i) and s (over j) contractions.
struct AxV5Smem {
    alignas(16) double sD[64];
    alignas(16) double sU[2][8][8][8];     // [parity][k][j][i] new p (fused PCG prologue)
    alignas(16) double sGT[2][8][8][8];    // [parity][k][j][i] g_t exchange (CTA-wide)
    alignas(16) double sGS[4][2][8][8];    // [warp][slab][j][i] g_s transpose (per warp)
    double sred[128];
    int last;
};

// TMAG: the 24 KB metric block of the element two ahead is brought into a 2-stage
// shared-memory ring by one TMA bulk copy while this element computes (dynamic smem).
template <bool HELM, bool FUSED, int MINB, bool TMAG = false, bool PF = false>
__global__ void __launch_bounds__(128, MINB)
    ax_v5_kernel(int64_t nelem, int64_t eoff, const int32_t *__restrict__ elist, const double *u,
                 const double *__restrict__ G, const double *__restrict__ wJ, const uint32_t *__restrict__ mbits,
                 double h1, double h2, double *__restrict__ w, double *__restrict__ part, int64_t part_off,
                 int64_t fin_total, double *__restrict__ dst, unsigned int *counter, const int *__restrict__ done,
                 double *pvec, double *__restrict__ xvec, const double *__restrict__ rvec,
                 const double *__restrict__ dvec, PcgScalars *sc, P2PMail mail, unsigned int ctas_total,
                 int keep, const double *__restrict__ upart, int nupd, double *hist, int defer)
{
    constexpr int P3 = 512, N = 7;
    __shared__ AxV5Smem S;
    extern __shared__ __align__(128) double gstage[];          // TMAG: [2][6 * 512]
    __shared__ uint64_t gfull[2];
    double beta = 0.0, alpha = 0.0;
    const uint64_t polv = tma::policy_keep(keep & 1), polx = tma::policy_keep(keep & 2);
    const int t = threadIdx.x, lane = t & 31, wq = t >> 5, q = lane & 3, r = lane >> 2;
    const int64_t nit = (int64_t)blockIdx.x < nelem ? (nelem - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (t < 64) S.sD[t] = c_D[N][t];
    __syncthreads();
    double Br[2], As[2], Bt[2], Ast[2];
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
        Br[s2] = S.sD[r * 8 + 2 * q + s2];       // r fwd   B(K=(s,q), n=r) = D(i_out=r, m=2q+s)
        As[s2] = S.sD[r * 8 + 4 * s2 + q];       // s fwd   A(r, K=(s,q))   = D(j_out=r, m=4s+q)
        Bt[s2] = S.sD[(2 * q + s2) * 8 + r];     // r trans B(K=(s,q), n=r) = D(i=2q+s, i'=r)
        Ast[s2] = S.sD[(4 * s2 + q) * 8 + r];    // s trans A(r, K=(s,q))   = D(j=4s+q, j'=r)
    }
    auto elem_at = [&](int64_t it) -> int64_t {
        const int64_t pos = eoff + blockIdx.x + it * (int64_t)gridDim.x;
        return elist ? (int64_t)elist[pos] : pos;
    };
    auto g_issue = [&](int64_t it, int st) {
        tma::fence_proxy_async();
        tma::mbar_arrive_expect_tx(&gfull[st], 6 * P3 * 8);
        tma::bulk_g2s(gstage + st * 6 * P3, G + elem_at(it) * 6 * (int64_t)P3, 6 * P3 * 8, &gfull[st],
                      tma::policy_evict_first());
    };
    if (TMAG) {
        if (t == 0) {
            tma::mbar_init(&gfull[0], 1);
            tma::mbar_init(&gfull[1], 1);
            tma::fence_mbar_init();
        }
        __syncthreads();
        if (t == 0) {
            if (nit > 0) g_issue(0, 0);
            if (nit > 1) g_issue(1, 1);
        }
    }
    if (FUSED) { beta = sc->beta; alpha = sc->alpha; }   // issued beside the done load, not after it
    bool stop = done && *(volatile const int *)done;
    if (FUSED && defer && !stop && *(volatile const int *)&sc->fold_ready) {
        // deferred reductions: the previous update's (rho', rr) -- folded from its CTA partials in the
        // same fixed order in every CTA (single rank, DEFER_FOLD), or every rank's pushed totals pulled
        // from the mailbox in rank order (P2P, DEFER_MAIL) -- give beta and the convergence decision
        // here; CTA 0 of the booking launch records the iteration (vec.cu, the deferred updates)
        const double rho_old = sc->rho, bb = sc->bb, tol = sc->tol;
        const int it = sc->iter, maxit = sc->maxit;
        if (defer & DEFER_MAIL) {
            if (t < 32) mail_pull_warp(mail, 1, &S.sred[64]);
        } else {
            double h0 = 0.0, l0 = 0.0, h1 = 0.0, l1 = 0.0;
            for (int c = t; c < nupd; c += blockDim.x) {
                dd_add(h0, l0, upart[4 * c], upart[4 * c + 1]);
                dd_add(h1, l1, upart[4 * c + 2], upart[4 * c + 3]);
            }
            block_sum_dd(h0, l0, S.sred);
            block_sum_dd(h1, l1, S.sred);
            if (t == 0) { S.sred[64] = __dadd_rn(h0, l0); S.sred[65] = __dadd_rn(h1, l1); }
        }
        __syncthreads();
        const double rho1 = S.sred[64], rr = S.sred[65];
        const bool conv = sqrt(rr) <= tol * bb;
        stop = conv || it >= maxit;
        if ((defer & DEFER_BOOK) && blockIdx.x == 0 && t == 0) {
            sc->booked = it;
            sc->rr = rr;
            if (hist) hist[it] = sqrt(rr) / bb;
            sc->beta = rho1 / rho_old;
            sc->rho_next = rho1;
            if (conv) { sc->status = NEK_OK; sc->done = 1; }
            else if (stop) { sc->status = NEK_MAXIT; sc->done = 1; }
            __threadfence();
        }
        beta = rho1 / rho_old;
    }
    if (stop) {
        if (TMAG) {                              // drain the metric copies already in flight
            if (nit > 0) tma::mbar_wait(&gfull[0], 0);
            if (nit > 1) tma::mbar_wait(&gfull[1], 0);
        }
        return;
    }
    const int kb = 2 * wq;                       // this warp's first k-slab
    double dhi = 0.0, dlo = 0.0;
    int64_t e_next = nit > 0 ? elem_at(0) : 0;
    for (int64_t it = 0; it < nit; ++it) {
        const int64_t e = e_next;                // element list read one iteration ahead
        if (it + 1 < nit) e_next = elem_at(it + 1);
        if (PF && !TMAG && t == 0 && it + 1 < nit)   // the next element's metric block toward L2 (large launches)
            tma::prefetch_l2(G + e_next * 6 * (int64_t)P3, 6 * P3 * 8);
        const double *ue = u + e * P3;
        const double *Ge = G + e * 6 * (int64_t)P3;
        const int par = (int)(it & 1);
        uint32_t mword = 0u;
        if (mbits && lane < 16) mword = __ldg(mbits + e * 16 + lane);
        double2 uc[8];                           // own k-line
        double2 uk[2];                           // own slabs
        double ub[2][2];                         // s-fwd B operand: u(i = r, j = 4s+q, k)
        double2 Gv[2][6];
        if (FUSED) {
            // p <- Dinv r + beta p and x <- x + alpha p on the own slabs, then share p
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                const int64_t l = e * P3 + 64 * (kb + kk) + 8 * r + 2 * q;
                const double2 po = tma::ld2(pvec + l, polv);
                const double2 rv = tma::ld2(rvec + l, polv);
                const double2 dv = tma::ld2(dvec + l, polv);
                double2 xv = tma::ld2(xvec + l, polx);
                double2 pn;
                pn.x = fma(beta, po.x, dv.x * rv.x);
                pn.y = fma(beta, po.y, dv.y * rv.y);
                xv.x = fma(alpha, po.x, xv.x);
                xv.y = fma(alpha, po.y, xv.y);
                tma::st2(pvec + l, pn, polv);
                tma::st2(xvec + l, xv, polx);
                *reinterpret_cast<double2 *>(&S.sU[par][kb + kk][r][2 * q]) = pn;
                uk[kk] = pn;
                if (!TMAG) {
#pragma unroll
                    for (int a = 0; a < 6; ++a)
                        Gv[kk][a] = *reinterpret_cast<const double2 *>(Ge + a * P3 + 64 * (kb + kk) + 8 * r + 2 * q);
                }
            }
            __syncthreads();
#pragma unroll
            for (int m = 0; m < 8; ++m) uc[m] = *reinterpret_cast<const double2 *>(&S.sU[par][m][r][2 * q]);
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) ub[kk][s2] = S.sU[par][kb + kk][4 * s2 + q][r];
        } else {
#pragma unroll
        for (int m = 0; m < 8; ++m) uc[m] = *reinterpret_cast<const double2 *>(ue + 64 * m + 8 * r + 2 * q);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const int k = kb + kk;
            uk[kk] = *reinterpret_cast<const double2 *>(ue + 64 * k + 8 * r + 2 * q);
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) ub[kk][s2] = ue[64 * k + 8 * (4 * s2 + q) + r];
            if (!TMAG) {
#pragma unroll
                for (int a = 0; a < 6; ++a)
                    Gv[kk][a] = *reinterpret_cast<const double2 *>(Ge + a * P3 + 64 * k + 8 * r + 2 * q);
            }
        }
        if (mbits) {
            // own point (i=2q+v, j=r, k): word 2k + (r >> 2), bit 8 (r & 3) + 2q + v
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const uint32_t wd = __shfl_sync(0xffffffffu, mword, 2 * m + (r >> 2)) >> (8 * (r & 3) + 2 * q);
                if (wd & 1u) uc[m].x = 0.0;
                if (wd & 2u) uc[m].y = 0.0;
            }
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                const int k = kb + kk;
                const uint32_t wd = __shfl_sync(0xffffffffu, mword, 2 * k + (r >> 2)) >> (8 * (r & 3) + 2 * q);
                if (wd & 1u) uk[kk].x = 0.0;
                if (wd & 2u) uk[kk].y = 0.0;
                // (i = r, j = 4s+q, k): word 2k + (j >> 2) = 2k + s, bit 8 (q) + r
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    const uint32_t wb = __shfl_sync(0xffffffffu, mword, 2 * k + s2);
                    if ((wb >> (8 * q + r)) & 1u) ub[kk][s2] = 0.0;
                }
            }
        }
        }
        if (TMAG) {
            const int st = (int)(it & 1);
            tma::mbar_wait(&gfull[st], (uint32_t)((it >> 1) & 1));
            const double *sg = gstage + st * 6 * P3;
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int a = 0; a < 6; ++a)
                    Gv[kk][a] = *reinterpret_cast<const double2 *>(sg + a * P3 + 64 * (kb + kk) + 8 * r + 2 * q);
        }
        double2 acc[2];
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const int k = kb + kk;
            double ur0 = 0.0, ur1 = 0.0, us0 = 0.0, us1 = 0.0;
            dmma8x8x4(ur0, ur1, uk[kk].x, Br[0]);
            dmma8x8x4(ur0, ur1, uk[kk].y, Br[1]);
            dmma8x8x4(us0, us1, As[0], ub[kk][0]);
            dmma8x8x4(us0, us1, As[1], ub[kk][1]);
            double ut0a = 0.0, ut0b = 0.0, ut1a = 0.0, ut1b = 0.0;
#pragma unroll
            for (int m = 0; m < 8; m += 2) {
                const double2 d = *reinterpret_cast<const double2 *>(S.sD + k * 8 + m);
                ut0a = fma(d.x, uc[m].x, ut0a); ut0b = fma(d.y, uc[m + 1].x, ut0b);
                ut1a = fma(d.x, uc[m].y, ut1a); ut1b = fma(d.y, uc[m + 1].y, ut1b);
            }
            const double ut0 = ut0a + ut0b, ut1 = ut1a + ut1b;
            const double2 *Gk = Gv[kk];
            const double gr0 = Gk[0].x * ur0 + Gk[1].x * us0 + Gk[2].x * ut0;
            const double gr1 = Gk[0].y * ur1 + Gk[1].y * us1 + Gk[2].y * ut1;
            const double gs0 = Gk[1].x * ur0 + Gk[3].x * us0 + Gk[4].x * ut0;
            const double gs1 = Gk[1].y * ur1 + Gk[3].y * us1 + Gk[4].y * ut1;
            const double gt0 = Gk[2].x * ur0 + Gk[4].x * us0 + Gk[5].x * ut0;
            const double gt1 = Gk[2].y * ur1 + Gk[4].y * us1 + Gk[5].y * ut1;
            double wr0 = 0.0, wr1 = 0.0;
            dmma8x8x4(wr0, wr1, gr0, Bt[0]);
            dmma8x8x4(wr0, wr1, gr1, Bt[1]);
            acc[kk] = make_double2(wr0, wr1);
            *reinterpret_cast<double2 *>(&S.sGS[wq][kk][r][2 * q]) = make_double2(gs0, gs1);
            *reinterpret_cast<double2 *>(&S.sGT[par][k][r][2 * q]) = make_double2(gt0, gt1);
        }
        __syncwarp();
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {         // s transposed (DMMA)
            double ws0 = 0.0, ws1 = 0.0;
            dmma8x8x4(ws0, ws1, Ast[0], S.sGS[wq][kk][q][r]);
            dmma8x8x4(ws0, ws1, Ast[1], S.sGS[wq][kk][4 + q][r]);
            acc[kk].x += ws0;
            acc[kk].y += ws1;
        }
        __syncthreads();                         // sGT[par] complete (and every G read of this element done)
        if (TMAG && t == 0 && it + 2 < nit) g_issue(it + 2, (int)(it & 1));
        double2 gtl[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) gtl[m] = *reinterpret_cast<const double2 *>(&S.sGT[par][m][r][2 * q]);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const int k = kb + kk;
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
            for (int m = 0; m < 8; m += 2) {
                const double d0 = S.sD[m * 8 + k], d1 = S.sD[(m + 1) * 8 + k];
                a0 = fma(d0, gtl[m].x, a0); b0 = fma(d1, gtl[m + 1].x, b0);
                a1 = fma(d0, gtl[m].y, a1); b1 = fma(d1, gtl[m + 1].y, b1);
            }
            const int64_t l = e * P3 + 64 * k + 8 * r + 2 * q;
            double v0 = h1 * (acc[kk].x + (a0 + b0)), v1 = h1 * (acc[kk].y + (a1 + b1));
            if (HELM) {
                const double2 wj = *reinterpret_cast<const double2 *>(wJ + l);
                v0 = fma(h2 * wj.x, uk[kk].x, v0);
                v1 = fma(h2 * wj.y, uk[kk].y, v1);
            }
            if (mbits) {
                const uint32_t wd = __shfl_sync(0xffffffffu, mword, 2 * k + (r >> 2)) >> (8 * (r & 3) + 2 * q);
                if (wd & 1u) v0 = 0.0;
                if (wd & 2u) v1 = 0.0;
            }
            tma::st2(w + l, make_double2(v0, v1), polv);
            dd_add_prod(dhi, dlo, uk[kk].x, v0);
            dd_add_prod(dhi, dlo, uk[kk].y, v1);
        }
    }
    if (part) {
        block_sum_dd(dhi, dlo, S.sred);
        if (t == 0) { part[2 * (part_off + blockIdx.x)] = dhi; part[2 * (part_off + blockIdx.x) + 1] = dlo; }
        if (fin_total > 0)
            last_block_finish(part, fin_total, dst, counter, S.sred, &S.last, mail.nranks > 1 ? &mail : nullptr,
                              ctas_total);
    }
}

template <bool HELM, int MINB, bool TMAG = false>
static cudaError_t ax_v5_launch(const AxLaunch &L, const double *u, const double *G, const double *wJ,
                                const uint32_t *mbits, double h1, double h2, double *w, int64_t grid, cudaStream_t s)
{
    const size_t dsm = TMAG ? 2 * 6 * 512 * sizeof(double) : 0;
    if (TMAG) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(ax_v5_kernel<HELM, true, MINB, TMAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dsm);
            cudaFuncSetAttribute(ax_v5_kernel<HELM, false, MINB, TMAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dsm);
            attr = true;
        }
    }
    const unsigned ctas = L.ctas_total ? L.ctas_total : (unsigned)grid;
    // large launches (vectors beyond L2): a bulk L2 prefetch of the next element's metric block, worth its
    // register-pressure spills there; small ones keep the spill-free kernel
    const bool pf = !TMAG && L.nelem >= L.pf_min;
    if (L.fused) {
        auto k = pf ? ax_v5_kernel<HELM, true, MINB, TMAG, !TMAG> : ax_v5_kernel<HELM, true, MINB, TMAG, false>;
        k<<<(unsigned)grid, 128, dsm, s>>>(
            L.nelem, L.eoff, L.elist, (const double *)L.p, G, wJ, mbits, h1, h2, w, L.part, L.part_off, L.fin_total,
            L.dst, L.counter, L.done, L.p, L.x, L.r, L.dinv, const_cast<PcgScalars *>(L.sc), L.mail, ctas, L.keep,
            L.upart, L.nupd, L.hist, L.defer);
    } else {
        auto k = pf ? ax_v5_kernel<HELM, false, MINB, TMAG, !TMAG> : ax_v5_kernel<HELM, false, MINB, TMAG, false>;
        k<<<(unsigned)grid, 128, dsm, s>>>(
            L.nelem, L.eoff, L.elist, u, G, wJ, mbits, h1, h2, w, L.part, L.part_off, L.fin_total, L.dst, L.counter,
            L.done, nullptr, nullptr, nullptr, nullptr, nullptr, L.mail, ctas, L.keep, nullptr, 0, nullptr, 0);
    }
    return cudaGetLastError();
}

#include "ax_v6.cuh"

// v6 (any N <= 9): the default for N != 7, variant 11 at any N <= 9
static bool use_v6(int variant, int N) { return N <= 9 && ((variant == 0 && N != 7) || variant == 11); }
static int v6_minb(int N)
{
    switch (N + 1) {
#define NEK_CASE(NQ) case NQ: return V6<NQ>::MINB;
        NEK_CASE(2) NEK_CASE(3) NEK_CASE(4) NEK_CASE(5) NEK_CASE(6) NEK_CASE(7) NEK_CASE(8) NEK_CASE(9) NEK_CASE(10)
#undef NEK_CASE
    }
    return 1;
}
static int v6_epb(int N)
{
    switch (N + 1) {
#define NEK_CASE(NQ) case NQ: return V6<NQ>::EPB;
        NEK_CASE(2) NEK_CASE(3) NEK_CASE(4) NEK_CASE(5) NEK_CASE(6) NEK_CASE(7) NEK_CASE(8) NEK_CASE(9) NEK_CASE(10)
#undef NEK_CASE
    }
    return 1;
}

bool ax_variant_valid(int variant) { return variant == 0 || variant == 1 || variant == 8 || variant == 10 || variant == 11 || variant == 12; }

// Few elements per CTA (the pipeline never fills, e.g. config 2: 4096 elements on 148 SMs): the v5
// configuration with the TMA-staged metric ring at 3 CTAs/SM; otherwise register streaming at 4 CTAs/SM
// (98% of the copy peak at scale).
constexpr int V5_SMALL_ELEMS_PER_CTA = 16;
static bool v5_small(int64_t nelem) { return nelem <= (int64_t)V5_SMALL_ELEMS_PER_CTA * 4 * device_sms(); }

// The fused PCG launch with L2-resident vectors: register streaming at 4 CTAs/SM (variant 12) beats the
// TMA metric ring at any size (config 2: 23.8 vs 22.6 GDOF/s, Ax 89% vs 83% of the copy peak by
// algorithmic bytes); nek_ax and the unfused launches keep the default (TMA ring: 32.4 vs 27.7).
int ax_effective_variant(int variant, int N, bool fused, int keep)
{
    return (variant == 0 && N == 7 && fused && keep) ? 12 : variant;
}

int ax_concrete_variant(int variant, int N, int64_t nelem)
{
    return (N == 7 && variant == 0) ? (v5_small(nelem) ? 10 : 12) : variant;
}

static bool is_v5(int variant, int N) { return N == 7 && (variant == 0 || variant == 8 || variant == 10 || variant == 12); }

bool ax_has_fused(int variant, int N) { return is_v5(variant, N) || use_v6(variant, N); }
bool ax_is_v5(int variant, int N) { return is_v5(variant, N); }

// v5 CTAs per SM of a variant (0: the launch decides by size)
static int v5_per_sm(int variant, int64_t nelem)
{
    switch (variant) {
    case 0: return v5_small(nelem) ? 3 : 4;
    case 8: return 3;
    case 10: return 3;
    case 12: return 4;
    default: return 0;
    }
}

// variant (N = 7): 0 = default (v5: TMA metric ring at 3 CTAs/SM for small launches, register streaming at
// 4 CTAs/SM otherwise), 8 = v5 register streaming at 3 CTAs/SM, 10 = v5 + TMA metric ring (3 CTAs/SM),
// 12 = v5 register streaming at 4 CTAs/SM (any size), 11 = v6, 1 = v0 (any N)
int64_t ax_grid(int variant, int N, int64_t nelem)
{
    if (nelem <= 0) return 0;
    if (is_v5(variant, N)) return std::min<int64_t>(nelem, (int64_t)v5_per_sm(variant, nelem) * device_sms());
    if (use_v6(variant, N)) {
        const int64_t nbat = (nelem + v6_epb(N) - 1) / v6_epb(N);
        return std::min<int64_t>(nbat, (int64_t)v6_minb(N) * device_sms());
    }
    const int epb = v0_epb(N + 1);
    return (nelem + epb - 1) / epb;
}

// FP32 Ax (v6) on all elements, for the reduced-precision pMG levels; N <= 9
cudaError_t launch_ax_f(int N, int64_t E, const float *u, const float *Gf, const float *wJf, const uint32_t *mbits,
                        double h1, double h2, float *w, cudaStream_t s)
{
    if (E <= 0) return cudaSuccess;
    switch (N + 1) {
#define NEK_CASE(NQ)                                                                         \
    case NQ:                                                                                 \
        return h2 != 0.0 ? ax_v6_launch_f<NQ, true>(E, u, Gf, wJf, mbits, h1, h2, w, s)   \
                         : ax_v6_launch_f<NQ, false>(E, u, Gf, wJf, mbits, h1, h2, w, s);
        NEK_CASE(2) NEK_CASE(3) NEK_CASE(4) NEK_CASE(5) NEK_CASE(6) NEK_CASE(7) NEK_CASE(8) NEK_CASE(9) NEK_CASE(10)
#undef NEK_CASE
    }
    return cudaErrorInvalidValue;
}

int ax_gstride_f(int N) { return ((6 * (N + 1) * (N + 1) * (N + 1) + 3) / 4) * 4; }

// enough partial slots for any variant (two concurrent launches of up to 4 CTAs per SM each)
int ax_partials_needed(int variant, int N, int64_t E)
{
    return (int)std::max<int64_t>(std::max<int64_t>(2 * ax_grid(variant, N, E), E), 2 * 4 * (int64_t)device_sms());
    // (partial slots; each slot holds a (hi, lo) pair of doubles)
}

template <int NQ>
static void ax_v0_launch(int64_t nelem, int64_t eoff, const int32_t *elist, const double *u, const double *G,
                         const double *wJ, const uint32_t *mbits, double h1, double h2, double *w, double *part,
                         const int *done, cudaStream_t s)
{
    constexpr int EPB = v0_epb(NQ);
    ax_v0_kernel<NQ><<<(unsigned)((nelem + EPB - 1) / EPB), dim3(NQ * NQ, EPB), 0, s>>>(
        nelem, eoff, elist, u, G, wJ, mbits, h1, h2, w, part, done);
}

cudaError_t launch_ax(int variant, int N, const AxLaunch &L, const double *u, const double *G, const double *wJ,
                      const uint32_t *mbits, double h1, double h2, double *w, cudaStream_t s, int *nlaunch)
{
    if (L.nelem <= 0) {
        if (L.fin_total > 0 && L.part) {   // nothing to compute here, but the reduction must still happen
            if (nlaunch) ++*nlaunch;
            return launch_reduce(L.part, L.fin_total, 1, L.dst, L.done, s);
        }
        return cudaSuccess;
    }
    if (is_v5(variant, N)) {
        if (nlaunch) ++*nlaunch;
        const int64_t grid = L.grid > 0 ? std::min<int64_t>(L.grid, L.nelem) : ax_grid(variant, N, L.nelem);
        const bool tmag = variant == 10 || (variant == 0 && v5_small(L.nelem));
        const int per_sm = v5_per_sm(variant, L.nelem);
        if (tmag)
            return h2 != 0.0 ? ax_v5_launch<true, 3, true>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                             : ax_v5_launch<false, 3, true>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
        if (per_sm == 4)
            return h2 != 0.0 ? ax_v5_launch<true, 4>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                             : ax_v5_launch<false, 4>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
        return h2 != 0.0 ? ax_v5_launch<true, 3>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                         : ax_v5_launch<false, 3>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
    }
    if (use_v6(variant, N)) {
        if (nlaunch) ++*nlaunch;
        const int64_t grid = ax_grid(variant, N, L.nelem);
        switch (N + 1) {
#define NEK_CASE(NQ)                                                                        \
    case NQ:                                                                                \
        return h2 != 0.0 ? ax_v6_launch<NQ, true>(L, u, G, wJ, mbits, h1, h2, w, grid, s) \
                         : ax_v6_launch<NQ, false>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
            NEK_CASE(2) NEK_CASE(3) NEK_CASE(4) NEK_CASE(5) NEK_CASE(6) NEK_CASE(7) NEK_CASE(8) NEK_CASE(9)
            NEK_CASE(10)
#undef NEK_CASE
        }
        return cudaErrorInvalidValue;
    }
    double *part = L.part ? L.part + 2 * L.part_off : nullptr;   // v0: one (hi, lo) partial per CTA
    switch (N) {
#define NEK_CASE(NN) \
    case NN: ax_v0_launch<NN + 1>(L.nelem, L.eoff, L.elist, u, G, wJ, mbits, h1, h2, w, part, L.done, s); break;
        NEK_CASE(1) NEK_CASE(2) NEK_CASE(3) NEK_CASE(4) NEK_CASE(5) NEK_CASE(6) NEK_CASE(7) NEK_CASE(8)
        NEK_CASE(9) NEK_CASE(10) NEK_CASE(11) NEK_CASE(12) NEK_CASE(13) NEK_CASE(14) NEK_CASE(15)
#undef NEK_CASE
    default: return cudaErrorInvalidValue;
    }
    if (nlaunch) ++*nlaunch;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (L.fin_total > 0 && L.part) {
        if (nlaunch) ++*nlaunch;
        return launch_reduce(L.part, L.fin_total, 1, L.dst, L.done, s);
    }
    return cudaSuccess;
}

// ----------------------------------------------------------------- Jacobi
__global__ void diag_kernel(int N, int64_t n, const double *__restrict__ G, const double *__restrict__ wJ, double h1,
                            double h2, double *__restrict__ d)
{
    const int Nq = N + 1, P2 = Nq * Nq, P3 = P2 * Nq;
    const double *D = c_D[N];
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / P3;
        const int q = (int)(l - e * P3), i = q % Nq, j = (q / Nq) % Nq, k = q / P2;
        const double *Ge = G + e * 6 * (int64_t)P3;
        double s = 0.0;
        for (int m = 0; m < Nq; ++m) {
            const double a = D[m * Nq + i], b = D[m * Nq + j], c = D[m * Nq + k];
            s = fma(a * a, Ge[0 * P3 + m + Nq * j + P2 * k], s);
            s = fma(b * b, Ge[3 * P3 + i + Nq * m + P2 * k], s);
            s = fma(c * c, Ge[5 * P3 + i + Nq * j + P2 * m], s);
        }
        const double Dii = D[i * Nq + i], Djj = D[j * Nq + j], Dkk = D[k * Nq + k];
        s += 2.0 * (Dii * Djj * Ge[1 * P3 + q] + Dii * Dkk * Ge[2 * P3 + q] + Djj * Dkk * Ge[4 * P3 + q]);
        d[l] = h1 * s + h2 * wJ[l];
    }
}

cudaError_t launch_diag(int N, int64_t E, const double *G, const double *wJ, double h1, double h2, double *d,
                        cudaStream_t s)
{
    const int64_t n = E * (N + 1) * (N + 1) * (N + 1);
    if (n == 0) return cudaSuccess;
    diag_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 16 * device_sms()), 256, 0, s>>>(N, n, G, wJ, h1, h2, d);
    return cudaGetLastError();
}

}  // namespace nekb200
