// ax_v6.cuh -- Ax for any order N = 1..9 (included by kernels.cu after c_D and the helpers).
//
// The operator of P:188-192 by sum factorisation, w = h1 D^T G D u + h2 wJ u:
//   u_r = (I x I x D) u, u_s = (I x D x I) u, u_t = (D x I x I) u     3 (N+1)^4 FMA per element
//   (g_r, g_s, g_t) = G (u_r, u_s, u_t)                               15 flop per point
//   w = D_r^T g_r + D_s^T g_s + D_t^T g_t                              3 (N+1)^4 FMA per element
//
// Design (sm_100a, FP64, HBM-bound at 72 B per point):
//  * persistent CTAs over batches of EPB elements; the six metric planes of each element (the
//    bulk of the traffic, 48 B per point) arrive by TMA bulk copy into a STAGES-deep shared-memory
//    ring (mbarrier completion), the batch after next in flight while this one computes;
//  * u (or, fused into PCG, p, r, Dinv, x), wJ and the mask words of the next batch are
//    prefetched column-wise into registers (coalesced: the (i,j) column index is the fast one);
//  * every 1-D contraction is done by a thread that owns a whole line of the element (r-lines
//    (j,k), s-lines (i,k), t-columns (i,j)): one shared-memory access per point and direction,
//    and D enters as compile-time constant-bank operands (cdv<T>(N, ..) with unrolled indices), so
//    the inner products are pure DFMA chains with no loads;
//  * line buffers are padded to an odd row stride so r-lines (lanes a row apart) hit distinct
//    banks; g_r / g_s overwrite u_r / u_s in place, and the transposed results overwrite them again;
//  * fused PCG prologue (as in v5): p <- Dinv r + beta p, x <- x + alpha p, then w = A p;
//  * one fixed-order <u, w> partial per CTA, finished by the last CTA (deterministic).
#pragma once

template <class T> __device__ __forceinline__ T cdv(int N, int i);
template <> __device__ __forceinline__ double cdv<double>(int N, int i) { return c_D[N][i]; }
template <> __device__ __forceinline__ float cdv<float>(int N, int i) { return c_Df[N][i]; }

// per-element metric block stride (elements of T): 6 planes, padded to 16 bytes for the TMA copy
template <int NQ, class T>
constexpr int v6_gstride() { return sizeof(T) == 8 ? 6 * NQ * NQ * NQ : ((6 * NQ * NQ * NQ + 3) / 4) * 4; }

template <int NQ, class T = double>
struct V6 {
    static constexpr int P2 = NQ * NQ, P3 = P2 * NQ;
    static constexpr int GS = v6_gstride<NQ, T>();
    static constexpr int PP = (NQ % 2 == 0) ? NQ + 1 : NQ;     // padded row stride of the line buffers
    // FP32 (reduced-precision pMG levels) halves the shared-memory stage: two elements per CTA at N = 7
    static constexpr int EPB = NQ == 2 ? 32 : NQ == 3 ? 14 : NQ == 4 ? 8 : NQ == 5 ? 5 : NQ == 6 ? 3 : NQ == 7 ? 2
                             : (NQ == 8 && sizeof(T) == 4) ? 2 : 1;
    static constexpr int NT = ((EPB * P2 + 31) / 32) * 32;
    static constexpr int STAGES = NQ == 10 ? 1 : 2;
    static constexpr int MINB = sizeof(T) == 4 ? (NQ <= 7 ? 4 : NQ == 8 ? 3 : 2) : (NQ <= 3 ? 4 : NQ == 4 ? 3 : 2);
    static constexpr int WB = NQ * NQ * PP;                       // one element's padded line buffer
    static constexpr size_t STAGE_D = (size_t)EPB * GS;           // elements of T per TMA stage
    static constexpr size_t SMEM = sizeof(T) * (STAGES * STAGE_D + 3 * (size_t)EPB * WB);
};

template <int NQ, bool HELM, bool FUSED, class T = double>
__global__ void __launch_bounds__(V6<NQ, T>::NT, V6<NQ, T>::MINB)
    ax_v6_kernel(int64_t nelem, int64_t eoff, const int32_t *__restrict__ elist, const T *u,
                 const T *__restrict__ G, const T *__restrict__ wJ, const uint32_t *__restrict__ mbits,
                 double h1d, double h2d, T *__restrict__ w, double *__restrict__ part, int64_t part_off,
                 int64_t fin_total, double *__restrict__ dst, unsigned int *counter, const int *__restrict__ done,
                 T *pvec, T *__restrict__ xvec, const T *__restrict__ rvec,
                 const T *__restrict__ dvec, const PcgScalars *sc, P2PMail mail, unsigned int ctas_total)
{
    using C = V6<NQ, T>;
    constexpr int N = NQ - 1, P2 = C::P2, P3 = C::P3, PP = C::PP, EPB = C::EPB, ST = C::STAGES, WB = C::WB;
    constexpr int GS = C::GS;
    if (done && *(volatile const int *)done) return;
    extern __shared__ __align__(128) unsigned char dsm_raw[];
    T *dsm = reinterpret_cast<T *>(dsm_raw);
    const T h1 = (T)h1d, h2 = (T)h2d;
    T *stage = dsm;                                       // [ST][EPB][GS]
    T *UP = dsm + ST * C::STAGE_D;                        // [EPB][WB]  u, then D_r^T g_r
    T *UR = UP + EPB * WB;                                // [EPB][WB]  u_r, then g_r, then D_r^T g_r
    T *US = UR + EPB * WB;                                // [EPB][WB]  u_s, then g_s, then D_s^T g_s
    __shared__ uint64_t full[ST];
    __shared__ double sred[64];
    __shared__ int s_last;
    const int t = threadIdx.x;
    const int b = t / P2, ij = t % P2, a = ij % NQ, c = ij / NQ;
    const bool lane_ok = t < EPB * P2;
    const int64_t nbat = (nelem + EPB - 1) / EPB;
    const int64_t nit = (int64_t)blockIdx.x < nbat ? (nbat - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    T beta = 0, alpha = 0;
    if (FUSED) { beta = (T)sc->beta; alpha = (T)sc->alpha; }

    auto elem_of = [&](int64_t it, int bb, int64_t *e) -> bool {
        const int64_t rel = (blockIdx.x + it * (int64_t)gridDim.x) * EPB + bb;
        if (rel >= nelem) return false;
        *e = elist ? (int64_t)elist[eoff + rel] : eoff + rel;
        return true;
    };
    auto issue = [&](int64_t it, int st) {                // lanes 0..EPB-1 of warp 0
        int64_t e;
        uint64_t *bar = &full[st];
        if (elem_of(it, t, &e)) {
            tma::mbar_arrive_expect_tx(bar, GS * (uint32_t)sizeof(T));
            tma::bulk_g2s(stage + st * C::STAGE_D + (size_t)t * GS, G + e * (int64_t)GS, GS * (uint32_t)sizeof(T), bar,
                          tma::policy_evict_first());
        } else {
            tma::mbar_arrive_expect_tx(bar, 0);
        }
    };
    if (t == 0) {
        for (int s = 0; s < ST; ++s) tma::mbar_init(&full[s], EPB);
        tma::fence_mbar_init();
    }
    __syncthreads();
    if (t < EPB) {
        tma::fence_proxy_async();
        for (int s = 0; s < ST && s < nit; ++s) issue(s, s);
    }

    // column-wise register prefetch of the next batch: point (i = a, j = c, k) of element slot b
    T nu[NQ], nr[FUSED ? NQ : 1], nd[FUSED ? NQ : 1], nx[FUSED ? NQ : 1], nw[HELM ? NQ : 1];
    uint32_t nm[NQ];
    int64_t ne = 0;
    bool nvalid = false;
    auto prefetch = [&](int64_t it) {
        nvalid = lane_ok && elem_of(it, b, &ne);
        if (!nvalid) return;
        const int64_t l0 = ne * P3 + ij;
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            const int64_t l = l0 + k * P2;
            nu[k] = u[l];
            if (FUSED) { nr[k] = rvec[l]; nd[k] = dvec[l]; nx[k] = xvec[l]; }
            if (HELM) nw[k] = wJ[l];
            nm[k] = mbits ? __ldg(mbits + (l >> 5)) : 0u;
        }
    };
    if (nit > 0) prefetch(0);

    double dhi = 0.0, dlo = 0.0;
    for (int64_t it = 0; it < nit; ++it) {
        const int st = (int)(it % ST);
        // ---- prologue: this batch's column into registers and into UP (padded)
        const bool valid = nvalid;
        const int64_t e = ne;
        T uc[NQ], hterm[HELM ? NQ : 1];
        uint32_t cmask = 0u;                                           // bit k: point k of the column is Dirichlet
        if (valid) {
            const int64_t l0 = e * P3 + ij;
#pragma unroll
            for (int k = 0; k < NQ; ++k) cmask |= ((nm[k] >> ((l0 + k * P2) & 31)) & 1u) << k;
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
                T v;
                if (FUSED) {
                    v = fma(beta, nu[k], nd[k] * nr[k]);          // p = Dinv r + beta p (Dinv masked)
                    const int64_t l = l0 + k * P2;
                    pvec[l] = v;
                    xvec[l] = fma(alpha, nu[k], nx[k]);           // deferred x += alpha p_old
                } else {
                    v = ((cmask >> k) & 1u) ? T(0) : nu[k];
                }
                uc[k] = v;
                if (HELM) hterm[k] = h2 * nw[k] * v;
                UP[b * WB + (k * NQ + c) * PP + a] = v;
            }
        }
        __syncthreads();                                               // (1) UP complete
        // ---- r-lines (j = a, k = c) and s-lines (i = a, k = c)
        if (valid) {
            T x[NQ];
            const T *row = UP + b * WB + (c * NQ + a) * PP;
#pragma unroll
            for (int m = 0; m < NQ; ++m) x[m] = row[m];
            T *orow = UR + b * WB + (c * NQ + a) * PP;
#pragma unroll
            for (int i = 0; i < NQ; ++i) {
                T s = 0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) s = fma(cdv<T>(N, i * NQ + m), x[m], s);
                orow[i] = s;
            }
            const T *col = UP + b * WB + (c * NQ) * PP + a;
#pragma unroll
            for (int m = 0; m < NQ; ++m) x[m] = col[m * PP];
            T *ocol = US + b * WB + (c * NQ) * PP + a;
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
                T s = 0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) s = fma(cdv<T>(N, j * NQ + m), x[m], s);
                ocol[j * PP] = s;
            }
        }
        if (t == 0) tma::mbar_wait(&full[st], (uint32_t)((it / ST) & 1));
        __syncthreads();                                               // (2) u_r, u_s complete; G landed
        // ---- t-columns (i = a, j = c): u_t, metric, g_t and D_t^T g_t in registers
        T wt[NQ];
        if (valid) {
            const T *Ge = stage + st * C::STAGE_D + (size_t)b * GS + c * NQ + a;
            T gt[NQ];
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
                T ut = 0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) ut = fma(cdv<T>(N, k * NQ + m), uc[m], ut);
                const int pk = b * WB + (k * NQ + c) * PP + a;
                const T ur = UR[pk], us = US[pk];
                const T *g = Ge + k * P2;
                const T Grr = g[0], Grs = g[P3], Grt = g[2 * P3], Gss = g[3 * P3], Gst = g[4 * P3], Gtt = g[5 * P3];
                UR[pk] = Grr * ur + Grs * us + Grt * ut;
                US[pk] = Grs * ur + Gss * us + Gst * ut;
                gt[k] = Grt * ur + Gst * us + Gtt * ut;
            }
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
                T s = 0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) s = fma(cdv<T>(N, m * NQ + k), gt[m], s);
                wt[k] = s;
            }
        }
        __syncthreads();                                               // (3) g_r, g_s complete; stage free
        if (t < EPB && it + ST < nit) {
            tma::fence_proxy_async();
            issue(it + ST, st);
        }
        if (it + 1 < nit) prefetch(it + 1);                            // lands during the rest of this batch
        // ---- transposed r-lines and s-lines, in place
        if (valid) {
            T x[NQ];
            T *row = UR + b * WB + (c * NQ + a) * PP;
#pragma unroll
            for (int m = 0; m < NQ; ++m) x[m] = row[m];
#pragma unroll
            for (int i = 0; i < NQ; ++i) {
                T s = 0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) s = fma(cdv<T>(N, m * NQ + i), x[m], s);
                row[i] = s;
            }
            T *col = US + b * WB + (c * NQ) * PP + a;
#pragma unroll
            for (int m = 0; m < NQ; ++m) x[m] = col[m * PP];
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
                T s = 0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) s = fma(cdv<T>(N, m * NQ + j), x[m], s);
                col[j * PP] = s;
            }
        }
        __syncthreads();                                               // (4) transposed terms complete
        // ---- epilogue on the own column
        if (valid) {
            const int64_t l0 = e * P3 + ij;
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
                const int pk = b * WB + (k * NQ + c) * PP + a;
                T v = h1 * (UR[pk] + US[pk] + wt[k]);
                if (HELM) v += hterm[k];
                const int64_t l = l0 + k * P2;
                if ((cmask >> k) & 1u) v = T(0);
                w[l] = v;
                dd_add_prod(dhi, dlo, (double)uc[k], (double)v);
            }
        }
    }
    if (part) {
        block_sum_dd(dhi, dlo, sred);
        if (t == 0) { part[2 * (part_off + blockIdx.x)] = dhi; part[2 * (part_off + blockIdx.x) + 1] = dlo; }
        if (fin_total > 0)
            last_block_finish(part, fin_total, dst, counter, sred, &s_last, mail.nranks > 1 ? &mail : nullptr,
                              ctas_total);
    }
}

template <int NQ, bool HELM>
static cudaError_t ax_v6_launch(const AxLaunch &L, const double *u, const double *G, const double *wJ,
                                const uint32_t *mbits, double h1, double h2, double *w, int64_t grid, cudaStream_t s)
{
    using C = V6<NQ>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e1 = cudaFuncSetAttribute(ax_v6_kernel<NQ, HELM, true, double>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        cudaError_t e2 = cudaFuncSetAttribute(ax_v6_kernel<NQ, HELM, false, double>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e1 != cudaSuccess) return e1;
        if (e2 != cudaSuccess) return e2;
        attr = true;
    }
    const unsigned tot = L.ctas_total ? L.ctas_total : (unsigned)grid;
    if (L.fused)
        ax_v6_kernel<NQ, HELM, true, double><<<(unsigned)grid, C::NT, C::SMEM, s>>>(
            L.nelem, L.eoff, L.elist, L.p, G, wJ, mbits, h1, h2, w, L.part, L.part_off, L.fin_total, L.dst,
            L.counter, L.done, L.p, L.x, L.r, L.dinv, L.sc, L.mail, tot);
    else
        ax_v6_kernel<NQ, HELM, false, double><<<(unsigned)grid, C::NT, C::SMEM, s>>>(
            L.nelem, L.eoff, L.elist, u, G, wJ, mbits, h1, h2, w, L.part, L.part_off, L.fin_total, L.dst,
            L.counter, L.done, nullptr, nullptr, nullptr, nullptr, nullptr, L.mail, tot);
    return cudaGetLastError();
}

// FP32 operator for the reduced-precision pMG levels (NEXT #3): no PCG fusion, no dot
template <int NQ, bool HELM>
static cudaError_t ax_v6_launch_f(int64_t nelem, const float *u, const float *G, const float *wJ,
                                  const uint32_t *mbits, double h1, double h2, float *w, cudaStream_t s)
{
    using C = V6<NQ, float>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(ax_v6_kernel<NQ, HELM, false, float>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int64_t nbat = (nelem + C::EPB - 1) / C::EPB;
    const int64_t grid = std::min<int64_t>(nbat, (int64_t)C::MINB * device_sms());
    if (grid <= 0) return cudaSuccess;
    ax_v6_kernel<NQ, HELM, false, float><<<(unsigned)grid, C::NT, C::SMEM, s>>>(
        nelem, 0, nullptr, u, G, wJ, mbits, h1, h2, w, nullptr, 0, 0, nullptr, nullptr, nullptr, nullptr, nullptr,
        nullptr, nullptr, nullptr, P2PMail(), (unsigned)grid);
    return cudaGetLastError();
}
