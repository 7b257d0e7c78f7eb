// kernels.cu -- sm_100a FP64 kernels of the hot path.
//
//   geom      geometric factors of the isoparametric map
//   ax        local Helmholtz apply w = h1 D^T G D u + h2 wJ u with the Dirichlet
//             mask on input and output and an optional <u, w> partial
//             (sum factorisation, O(N^4) work, O(N^3) memory)
//   gs_*      gather-scatter QQ^T: local runs, interface partial + pack,
//             unpack + scatter (reading 7)
//   diag      exact diagonal of h1 K_L + h2 B_L (reading 10)
//   pcg_*     fused Jacobi-PCG vector updates with deterministic block
//             reductions (reading 8 owner-copy inner products)
// All reductions are two-level and fixed-order (no floating-point atomics), so
// results are bitwise repeatable run to run.
#include <cuda_runtime.h>

#include <cstdint>

#include "nek_ctx.h"

namespace nekb200 {

__constant__ double c_D[16][256];   // D for every order N (row-major, (N+1)^2 used)

cudaError_t upload_D(int N, const double *D)
{
    return cudaMemcpyToSymbol(c_D, D, sizeof(double) * (N + 1) * (N + 1), sizeof(double) * 256 * N,
                              cudaMemcpyHostToDevice);
}

__device__ __forceinline__ bool bit_of(const uint32_t *__restrict__ bits, int64_t l)
{
    return (__ldg(bits + (l >> 5)) >> (l & 31)) & 1u;
}

// Fixed-order block sum of v (blockDim.x <= 1024); result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double *sred)
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
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    geom_kernel<<<blocks, 256, 0, s>>>(N, n, xyz, wq, G, wJ, bad);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- Ax v0
// One element per CTA, (N+1)^2 threads (i fastest), the k-column of u and of
// the result in registers, one (i,j) slice in shared memory at a time.
template <int NQ>
__global__ void __launch_bounds__(NQ *NQ)
    ax_v0_kernel(int64_t eoff, const int32_t *__restrict__ elist, const double *__restrict__ u,
                 const double *__restrict__ G, const double *__restrict__ wJ, const uint32_t *__restrict__ mbits,
                 double h1, double h2, double *__restrict__ w, double *__restrict__ part, const int *__restrict__ done)
{
    constexpr int P2 = NQ * NQ, P3 = P2 * NQ, N = NQ - 1;
    if (done && *(volatile const int *)done) return;
    __shared__ double sD[NQ * NQ];
    __shared__ double sa[P2], sb[P2];
    __shared__ double sred[P2];
    const int t = threadIdx.x, i = t % NQ, j = t / NQ;
    const int64_t pos = eoff + blockIdx.x;
    const int64_t e = elist ? (int64_t)elist[pos] : pos;
    for (int q = t; q < NQ * NQ; q += P2) sD[q] = c_D[N][q];
    const double *ue = u + e * P3;
    const double *Ge = G + e * 6 * (int64_t)P3;
    double ru[NQ], rw[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
        const int64_t l = e * P3 + k * P2 + t;
        double v = ue[k * P2 + t];
        if (mbits && bit_of(mbits, l)) v = 0.0;
        ru[k] = v;
        rw[k] = 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
        sa[t] = ru[k];
        __syncthreads();
        double ur = 0, us = 0, ut = 0;
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
            ur = fma(sD[i * NQ + m], sa[j * NQ + m], ur);
            us = fma(sD[j * NQ + m], sa[m * NQ + i], us);
            ut = fma(sD[k * NQ + m], ru[m], ut);
        }
        const int q = k * P2 + t;
        const double Grr = Ge[q], Grs = Ge[P3 + q], Grt = Ge[2 * P3 + q];
        const double Gss = Ge[3 * P3 + q], Gst = Ge[4 * P3 + q], Gtt = Ge[5 * P3 + q];
        const double gr = Grr * ur + Grs * us + Grt * ut;
        const double gs = Grs * ur + Gss * us + Gst * ut;
        const double gt = Grt * ur + Gst * us + Gtt * ut;
        __syncthreads();
        sa[t] = gr;
        sb[t] = gs;
        __syncthreads();
        double acc = 0;
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
            acc = fma(sD[m * NQ + i], sa[j * NQ + m], acc);
            acc = fma(sD[m * NQ + j], sb[m * NQ + i], acc);
        }
        rw[k] += acc;
#pragma unroll
        for (int m = 0; m < NQ; ++m) rw[m] = fma(sD[k * NQ + m], gt, rw[m]);
        __syncthreads();
    }
    double dot = 0.0;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
        const int64_t l = e * P3 + k * P2 + t;
        double v = h1 * rw[k];
        if (h2 != 0.0) v = fma(h2 * wJ[l], ru[k], v);
        if (mbits && bit_of(mbits, l)) v = 0.0;
        w[l] = v;
        dot = fma(ru[k], v, dot);
    }
    if (part) {
        double s = block_sum(dot, sred);
        if (t == 0) part[pos] = s;
    }
}

int ax_partials_needed(int variant, int N, int64_t E) { (void)variant; (void)N; return (int)E; }

template <int NQ>
static void ax_v0_launch(int64_t nelem, int64_t eoff, const int32_t *elist, const double *u, const double *G,
                         const double *wJ, const uint32_t *mbits, double h1, double h2, double *w, double *part,
                         const int *done, cudaStream_t s)
{
    ax_v0_kernel<NQ><<<(unsigned)nelem, NQ * NQ, 0, s>>>(eoff, elist, u, G, wJ, mbits, h1, h2, w, part, done);
}

cudaError_t launch_ax(int variant, int N, int64_t nelem, int64_t eoff, const int32_t *elist, const double *u,
                      const double *G, const double *wJ, const uint32_t *mbits, double h1, double h2, double *w,
                      double *part, const int *done, cudaStream_t s, int *nlaunch)
{
    (void)variant;
    if (nelem <= 0) return cudaSuccess;
    switch (N) {
#define NEK_CASE(NN) \
    case NN: ax_v0_launch<NN + 1>(nelem, eoff, elist, u, G, wJ, mbits, h1, h2, w, part, done, s); break;
        NEK_CASE(1) NEK_CASE(2) NEK_CASE(3) NEK_CASE(4) NEK_CASE(5) NEK_CASE(6) NEK_CASE(7) NEK_CASE(8)
        NEK_CASE(9) NEK_CASE(10) NEK_CASE(11) NEK_CASE(12) NEK_CASE(13) NEK_CASE(14) NEK_CASE(15)
#undef NEK_CASE
    default: return cudaErrorInvalidValue;
    }
    if (nlaunch) ++*nlaunch;
    return cudaGetLastError();
}

// Fixed-order reduction of count x nd partials (row-major [count][nd]) into dst[nd].
__global__ void reduce_kernel(const double *__restrict__ part, int64_t count, int nd, double *__restrict__ dst,
                              const int *done)
{
    __shared__ double sred[1024];
    if (done && *(volatile const int *)done) return;
    for (int d = 0; d < nd; ++d) {
        double s = 0.0;
        for (int64_t c = threadIdx.x; c < count; c += blockDim.x) s += part[c * nd + d];
        s = block_sum(s, sred);
        if (threadIdx.x == 0) dst[d] = s;
    }
}

cudaError_t launch_reduce(const double *part, int64_t count, int nd, double *dst, const int *done, cudaStream_t s)
{
    reduce_kernel<<<1, 1024, 0, s>>>(part, count, nd, dst, done);
    return cudaGetLastError();
}

// ---------------------------------------------------------- gather-scatter
// One thread per run: left fold in canonical order, then broadcast.
__global__ void gs_local_kernel(int64_t nruns, const int32_t *__restrict__ perm, const int32_t *__restrict__ offs,
                                double *__restrict__ v, const int *done)
{
    if (done && *(volatile const int *)done) return;
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    const int o0 = offs[r], o1 = offs[r + 1];
    double s = v[perm[o0]];
    for (int c = o0 + 1; c < o1; ++c) s += v[perm[c]];
    for (int c = o0; c < o1; ++c) v[perm[c]] = s;
}

cudaError_t launch_gs_local(int64_t nruns, const int32_t *perm, const int32_t *offs, double *v, const int *done,
                            cudaStream_t s)
{
    if (nruns <= 0) return cudaSuccess;
    gs_local_kernel<<<(unsigned)((nruns + 255) / 256), 256, 0, s>>>(nruns, perm, offs, v, done);
    return cudaGetLastError();
}

__global__ void gs_ifc_partial_kernel(int64_t nifc, const int32_t *__restrict__ perm, const int32_t *__restrict__ offs,
                                      const double *__restrict__ v, double *__restrict__ partial, const int *done)
{
    if (done && *(volatile const int *)done) return;
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nifc) return;
    const int o0 = offs[r], o1 = offs[r + 1];
    double s = v[perm[o0]];
    for (int c = o0 + 1; c < o1; ++c) s += v[perm[c]];
    partial[r] = s;
}

__global__ void gs_pack_kernel(int64_t nslots, const int32_t *__restrict__ send_run, const double *__restrict__ partial,
                               double *__restrict__ sendbuf, const int *done)
{
    if (done && *(volatile const int *)done) return;
    const int64_t sidx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sidx < nslots) sendbuf[sidx] = partial[send_run[sidx]];
}

cudaError_t launch_gs_ifc_pack(int64_t nifc, const int32_t *perm, const int32_t *offs, const double *v,
                               double *partial, int64_t nslots, const int32_t *send_run, double *sendbuf,
                               const int *done, cudaStream_t s)
{
    if (nifc > 0) gs_ifc_partial_kernel<<<(unsigned)((nifc + 255) / 256), 256, 0, s>>>(nifc, perm, offs, v, partial, done);
    if (nslots > 0) gs_pack_kernel<<<(unsigned)((nslots + 255) / 256), 256, 0, s>>>(nslots, send_run, partial, sendbuf, done);
    return cudaGetLastError();
}

// total = fold of contributions in ascending rank order (own partial or a
// received slot), then written to every local copy.
__global__ void gs_unpack_kernel(int64_t nifc, const int32_t *__restrict__ perm, const int32_t *__restrict__ offs,
                                 const int32_t *__restrict__ coffs, const int32_t *__restrict__ contrib,
                                 const double *__restrict__ partial, const double *__restrict__ recvbuf,
                                 double *__restrict__ v, const int *done)
{
    if (done && *(volatile const int *)done) return;
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nifc) return;
    const int c0 = coffs[r], c1 = coffs[r + 1];
    int src = contrib[c0];
    double s = src < 0 ? partial[r] : recvbuf[src];
    for (int c = c0 + 1; c < c1; ++c) {
        src = contrib[c];
        s += src < 0 ? partial[r] : recvbuf[src];
    }
    for (int c = offs[r]; c < offs[r + 1]; ++c) v[perm[c]] = s;
}

cudaError_t launch_gs_ifc_unpack(int64_t nifc, const int32_t *perm, const int32_t *offs, const int32_t *coffs,
                                 const int32_t *contrib, const double *partial, const double *recvbuf, double *v,
                                 const int *done, cudaStream_t s)
{
    if (nifc <= 0) return cudaSuccess;
    gs_unpack_kernel<<<(unsigned)((nifc + 255) / 256), 256, 0, s>>>(nifc, perm, offs, coffs, contrib, partial,
                                                                    recvbuf, v, done);
    return cudaGetLastError();
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
    diag_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(N, n, G, wJ, h1, h2, d);
    return cudaGetLastError();
}

__global__ void dinv_kernel(int64_t n, const uint32_t *__restrict__ mbits, const double *__restrict__ d,
                            double *__restrict__ dinv)
{
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x)
        dinv[l] = bit_of(mbits, l) ? 0.0 : 1.0 / d[l];
}

cudaError_t launch_dinv(int64_t n, const uint32_t *mbits, const double *d, double *dinv, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    dinv_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(n, mbits, d, dinv);
    return cudaGetLastError();
}

__global__ void copy_mask_kernel(int64_t n, const uint32_t *__restrict__ mbits, const double *__restrict__ src,
                                 double *__restrict__ dst)
{
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x)
        dst[l] = bit_of(mbits, l) ? 0.0 : src[l];
}

cudaError_t launch_copy_mask(int64_t n, const uint32_t *mbits, const double *src, double *dst, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    copy_mask_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(n, mbits, src, dst);
    return cudaGetLastError();
}

// --------------------------------------------------------------------- PCG
constexpr int VEC_THREADS = 256;
int vec_blocks() { return 148 * 8; }

// r = M b, p = Dinv r, x = 0; partials [<r, Dinv r>_o, <r, r>_o] per block.
__global__ void __launch_bounds__(VEC_THREADS)
    pcg_init_kernel(int64_t n, const uint32_t *__restrict__ mbits, const uint32_t *__restrict__ obits,
                    const double *__restrict__ b, const double *__restrict__ dinv, double *__restrict__ r,
                    double *__restrict__ p, double *__restrict__ x, double *__restrict__ part)
{
    __shared__ double sred[VEC_THREADS];
    double a0 = 0.0, a1 = 0.0;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x) {
        const double rv = bit_of(mbits, l) ? 0.0 : b[l];
        const double z = dinv[l] * rv;
        r[l] = rv;
        p[l] = z;
        x[l] = 0.0;
        if (bit_of(obits, l)) { a0 = fma(rv, z, a0); a1 = fma(rv, rv, a1); }
    }
    a0 = block_sum(a0, sred);
    a1 = block_sum(a1, sred);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = a0; part[2 * blockIdx.x + 1] = a1; }
}

cudaError_t launch_pcg_init(int64_t n, const uint32_t *mbits, const uint32_t *obits, const double *b,
                            const double *dinv, double *r, double *p, double *x, double *part, int nblk,
                            cudaStream_t s)
{
    pcg_init_kernel<<<nblk, VEC_THREADS, 0, s>>>(n, mbits, obits, b, dinv, r, p, x, part);
    return cudaGetLastError();
}

// red_all holds [nranks][RED_N]; sums are taken in rank order.
__device__ __forceinline__ double rank_sum(const double *red_all, int nranks, int slot)
{
    double s = red_all[slot];
    for (int q = 1; q < nranks; ++q) s += red_all[q * RED_N + slot];
    return s;
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

// alpha = rho / sigma; x += alpha p; r -= alpha w; partials [<r, Dinv r>_o, <r, r>_o].
__global__ void __launch_bounds__(VEC_THREADS)
    pcg_update_kernel(int64_t n, const uint32_t *__restrict__ obits, const double *__restrict__ dinv,
                      const double *__restrict__ p, const double *__restrict__ w, double *__restrict__ x,
                      double *__restrict__ r, const double *__restrict__ red_all, int nranks, PcgScalars *sc,
                      double *__restrict__ part)
{
    __shared__ double sred[VEC_THREADS];
    if (*(volatile int *)&sc->done) return;
    const double sigma = rank_sum(red_all, nranks, RED_SIGMA);
    if (!(sigma > 0.0)) {                       // breakdown: <p, A p> <= 0
        if (blockIdx.x == 0 && threadIdx.x == 0) { sc->status = NEK_ENOTSPD; }
        return;
    }
    const double alpha = sc->rho / sigma;
    double a0 = 0.0, a1 = 0.0;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x) {
        x[l] = fma(alpha, p[l], x[l]);
        const double rv = fma(-alpha, w[l], r[l]);
        r[l] = rv;
        if (bit_of(obits, l)) {
            a0 = fma(rv, dinv[l] * rv, a0);
            a1 = fma(rv, rv, a1);
        }
    }
    a0 = block_sum(a0, sred);
    a1 = block_sum(a1, sred);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = a0; part[2 * blockIdx.x + 1] = a1; }
}

cudaError_t launch_pcg_update(int64_t n, const uint32_t *obits, const double *dinv, const double *p,
                              const double *w, double *x, double *r, const double *red_all, int nranks,
                              PcgScalars *sc, double *part, int nblk, cudaStream_t s)
{
    pcg_update_kernel<<<nblk, VEC_THREADS, 0, s>>>(n, obits, dinv, p, w, x, r, red_all, nranks, sc, part);
    return cudaGetLastError();
}

// beta = rho'/rho; p = Dinv r + beta p.  The last block to finish updates the
// scalars (rho <- rho', iteration count, history, convergence, breakdown).
__global__ void __launch_bounds__(VEC_THREADS)
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
        for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x)
            p[l] = fma(beta, p[l], dinv[l] * r[l]);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
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

}  // namespace nekb200
