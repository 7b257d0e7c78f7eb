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
#include <cstdlib>
#include <utility>

#include "ax_tma.cuh"
#include "nek_ctx.h"

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

__device__ __forceinline__ bool bit_of(const uint32_t *__restrict__ bits, int64_t l)
{
    return (__ldg(bits + (l >> 5)) >> (l & 31)) & 1u;
}

// Programmatic dependent launch (PDL): a kernel launched with the programmatic-serialisation
// attribute may start while its predecessor in the stream drains; it does its predecessor-independent
// prologue (index lists, metric-factor TMA), then waits here for the predecessor's completion and
// memory flush.  Without the attribute both are no-ops.  Measured at config 2 (CUDA graph of the
// fused PCG iteration): 19.8 vs 22.3 GDOF/s with PDL on Ax -> gs -> update, and nek_ax 24.3 vs 27.9,
// so it is off by default (NEK_PDL=1 turns it on).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NEK_PDL");
        v = e ? atoi(e) != 0 : 0;
    }
    return v;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? at : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
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
__device__ __forceinline__ bool wait_epoch(const uint64_t *flag, uint64_t e, int *err)
{
    for (long it = 0; it < (1l << 22); ++it) {   // ~0.5 s
        if (ld_acquire_sys(flag) >= e) return true;
        if (it > 64) __nanosleep(64);
    }
    atomicExch(err, 1);
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
    __threadfence_system();
    for (int q = 0; q < M.nranks; ++q) {
        double *dst = (q == M.me ? M.mbox : M.peer_mbox[q]) + (base + M.me) * 4;
        st_release_sys(reinterpret_cast<uint64_t *>(dst + 3), e);
    }
}

// single thread: wait for the current epoch of `channel` from every rank and
// return the rank-ordered sums of the value slots
__device__ __forceinline__ void mail_pull(const P2PMail &M, int channel, double *sum3)
{
    const uint64_t e = *(volatile uint64_t *)&M.epochs[channel];
    const size_t base = ((size_t)channel * 2 + (e & 1)) * M.nranks;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int q = 0; q < M.nranks; ++q) {
        const double *src = M.mbox + (base + q) * 4;
        wait_epoch(reinterpret_cast<const uint64_t *>(src + 3), e, M.err);
        const double b0 = ((volatile const double *)src)[0], b1 = ((volatile const double *)src)[1],
                     b2 = ((volatile const double *)src)[2];
        if (q == 0) { a0 = b0; a1 = b1; a2 = b2; }
        else { a0 += b0; a1 += b1; a2 += b2; }
    }
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
    if (lane < M.nranks) {
        const double *src = M.mbox + (base + lane) * 4;
        wait_epoch(reinterpret_cast<const uint64_t *>(src + 3), e, M.err);
        b0 = ((volatile const double *)src)[0];
        b1 = ((volatile const double *)src)[1];
        b2 = ((volatile const double *)src)[2];
    }
    double a0 = __shfl_sync(0xffffffffu, b0, 0), a1 = __shfl_sync(0xffffffffu, b1, 0),
           a2 = __shfl_sync(0xffffffffu, b2, 0);
    for (int q = 1; q < M.nranks; ++q) {
        const double c0 = __shfl_sync(0xffffffffu, b0, q), c1 = __shfl_sync(0xffffffffu, b1, q),
                     c2 = __shfl_sync(0xffffffffu, b2, q);
        a0 += c0; a1 += c1; a2 += c2;
    }
    if (lane == 0) { sum3[0] = a0; sum3[1] = a1; sum3[2] = a2; }
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
    __shared__ double sred[P2 * EPB];
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
    double dot = 0.0;
    if (valid) {
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            const int64_t l = e * P3 + k * P2 + t;
            double v = h1 * rw[k];
            if (h2 != 0.0) v = fma(h2 * wJ[l], ru[k], v);
            if (mbits && bit_of(mbits, l)) v = 0.0;
            w[l] = v;
            dot = fma(ru[k], v, dot);
        }
    }
    if (part) {
        // fixed-order CTA sum over the linear thread index
        const int lt = t + P2 * g, nt = P2 * EPB;
        sred[lt] = dot;
        __syncthreads();
        for (int s2 = 512; s2 > 0; s2 >>= 1) {
            if (s2 < nt && lt < s2 && lt + s2 < nt) sred[lt] += sred[lt + s2];
            __syncthreads();
        }
        if (lt == 0) part[blockIdx.x] = sred[0];
    }
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

// Last CTA to finish sums part[0..count) (fixed order) into dst[0] and resets the counter.
// ctas_total: CTAs (over one or several concurrent launches) that share `counter`.
__device__ __forceinline__ void last_block_finish(double *part, int64_t count, double *dst, unsigned int *counter,
                                                  double *sred, int *s_last, const P2PMail *mail = nullptr,
                                                  unsigned int ctas_total = 0)
{
    if (threadIdx.x == 0) {
        __threadfence();
        *s_last = atomicAdd(counter, 1u) == (ctas_total ? ctas_total : gridDim.x) - 1;
    }
    __syncthreads();
    if (*s_last) {
        __threadfence();
        double a = 0.0;
        for (int64_t c = threadIdx.x; c < count; c += blockDim.x) a += ((volatile double *)part)[c];
        a = block_sum(a, sred);
        if (threadIdx.x == 0) {
            dst[0] = a;
            *counter = 0u;
            if (mail) mail_push(*mail, 0, a, 0.0, 0.0);   // sigma straight to every rank (channel 0)
        }
    }
}

// ------------------------------------------------------------------- Ax v1
template <bool HELM>
__global__ void __launch_bounds__(AXV1_THREADS, AXV1_CTAS_PER_SM)
    ax_v1_kernel(int64_t nelem, int64_t eoff, const int32_t *__restrict__ elist, const double *__restrict__ u,
                 const double *__restrict__ G, const double *__restrict__ wJ, const uint32_t *__restrict__ mbits,
                 double h1, double h2, double *__restrict__ w, double *__restrict__ part, int64_t part_off,
                 int64_t fin_total, double *__restrict__ dst, unsigned int *counter, const int *__restrict__ done)
{
    constexpr int NQ = AXV1_NQ, P3 = 512, N = NQ - 1;
    constexpr uint32_t BYTES = (7 + (HELM ? 1 : 0)) * P3 * 8;
    if (done && *(volatile const int *)done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    AxV1Smem<HELM> &S = *reinterpret_cast<AxV1Smem<HELM> *>(smem_raw);
    const int t = threadIdx.x, i = t & 7, j = t >> 3;
    const int64_t nit = (int64_t)blockIdx.x < nelem ? (nelem - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint64_t pol = tma::policy_evict_first();

    auto elem_of = [&](int64_t it) -> int64_t {
        const int64_t pos = eoff + blockIdx.x + it * (int64_t)gridDim.x;
        return elist ? (int64_t)elist[pos] : pos;
    };
    auto issue = [&](int64_t it, int st) {
        const int64_t e = elem_of(it);
        tma::fence_proxy_async();
        tma::mbar_arrive_expect_tx(&S.full[st], BYTES);
        tma::bulk_g2s(S.stage[st], u + e * P3, P3 * 8, &S.full[st], pol);
        tma::bulk_g2s(S.stage[st] + P3, G + e * 6 * P3, 6 * P3 * 8, &S.full[st], pol);
        if (HELM) tma::bulk_g2s(S.stage[st] + 7 * P3, wJ + e * P3, P3 * 8, &S.full[st], pol);
    };
    if (t == 0) {
        tma::mbar_init(&S.full[0], 1);
        tma::mbar_init(&S.full[1], 1);
        tma::fence_mbar_init();
    }
    __syncthreads();
    if (t == 0) {
        if (nit > 0) issue(0, 0);
        if (nit > 1) issue(1, 1);
    }
    double Dri[NQ], Drj[NQ], Dci[NQ], Dcj[NQ];
#pragma unroll
    for (int m = 0; m < NQ; ++m) {
        Dri[m] = c_D[N][i * NQ + m]; Drj[m] = c_D[N][j * NQ + m];
        Dci[m] = c_D[N][m * NQ + i]; Dcj[m] = c_D[N][m * NQ + j];
    }
    S.sD[t] = c_D[N][t];                 // D row-major, read warp-uniformly for the t direction
    double dot = 0.0;
    for (int64_t it = 0; it < nit; ++it) {
        const int st = (int)(it & 1);
        const int64_t e = elem_of(it);
        tma::mbar_wait(&S.full[st], (uint32_t)((it >> 1) & 1));
        const double *su = S.stage[st];
        const double *sG = su + P3;
        double ru[NQ], ut[NQ], gt[NQ], rw[NQ];
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            double v = su[k * 64 + t];
            if (mbits && bit_of(mbits, e * P3 + k * 64 + t)) v = 0.0;
            ru[k] = v;
        }
        // t direction on the thread's own k-column: ut = D ru
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            double a = 0.0;
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 d = *reinterpret_cast<const double2 *>(&S.sD[k * NQ + m]);
                a = fma(d.x, ru[m], a);
                a = fma(d.y, ru[m + 1], a);
            }
            ut[k] = a;
        }
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            S.sa[t] = ru[k];
            __syncthreads();
            double ur = 0.0, us = 0.0;
#pragma unroll
            for (int m = 0; m < NQ; ++m) {
                ur = fma(Dri[m], S.sa[j * NQ + m], ur);
                us = fma(Drj[m], S.sa[m * NQ + i], us);
            }
            const int q = k * 64 + t;
            const double Grr = sG[q], Grs = sG[P3 + q], Grt = sG[2 * P3 + q];
            const double Gss = sG[3 * P3 + q], Gst = sG[4 * P3 + q], Gtt = sG[5 * P3 + q];
            const double gr = Grr * ur + Grs * us + Grt * ut[k];
            const double gs = Grs * ur + Gss * us + Gst * ut[k];
            gt[k] = Grt * ur + Gst * us + Gtt * ut[k];
            S.sb[t] = gr;
            S.sc[t] = gs;
            __syncthreads();
            double acc = 0.0;
#pragma unroll
            for (int m = 0; m < NQ; ++m) {
                acc = fma(Dci[m], S.sb[j * NQ + m], acc);
                acc = fma(Dcj[m], S.sc[m * NQ + i], acc);
            }
            rw[k] = acc;
        }
        // transposed t direction: rw += D^T gt on the k-column
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 d = *reinterpret_cast<const double2 *>(&S.sD[k * NQ + m]);
                rw[m] = fma(d.x, gt[k], rw[m]);
                rw[m + 1] = fma(d.y, gt[k], rw[m + 1]);
            }
        }
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            const int64_t l = e * P3 + k * 64 + t;
            double v = h1 * rw[k];
            if (HELM) v = fma(h2 * su[7 * P3 + k * 64 + t], ru[k], v);
            if (mbits && bit_of(mbits, l)) v = 0.0;
            w[l] = v;
            dot = fma(ru[k], v, dot);
        }
        __syncthreads();   // stage `st` fully consumed by all threads
        if (t == 0 && it + 2 < nit) issue(it + 2, st);
    }
    if (part) {
        const double s = block_sum(dot, S.sred);
        if (t == 0) part[part_off + blockIdx.x] = s;
        if (fin_total > 0) last_block_finish(part, fin_total, dst, counter, S.sred, &S.last);
    }
}

// ------------------------------------------------------------------- Ax v2
// Same staging as v1 (2-stage TMA ring per CTA), but KS k-groups of 64 threads
// share each element: 64*KS threads per CTA.  Accumulations are split into
// independent partial sums (ILP) and the Dirichlet words ride along in the TMA
// transaction.
template <bool HELM, int KS>
__global__ void __launch_bounds__(64 * KS, KS == 2 ? 3 : 2)
    ax_v2_kernel(int64_t nelem, int64_t eoff, const int32_t *__restrict__ elist, const double *__restrict__ u,
                 const double *__restrict__ G, const double *__restrict__ wJ, const uint32_t *__restrict__ mbits,
                 double h1, double h2, double *__restrict__ w, double *__restrict__ part, int64_t part_off,
                 int64_t fin_total, double *__restrict__ dst, unsigned int *counter, const int *__restrict__ done)
{
    constexpr int NQ = 8, P3 = 512, N = 7, KPG = NQ / KS;
    const uint32_t BYTES = (7 + (HELM ? 1 : 0)) * P3 * 8 + (mbits ? 64 : 0);
    if (done && *(volatile const int *)done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    AxV2Smem<HELM, KS> &S = *reinterpret_cast<AxV2Smem<HELM, KS> *>(smem_raw);
    const int t = threadIdx.x, c = t & 63, g = t >> 6, i = c & 7, j = c >> 3;
    const int k0 = g * KPG;
    const int64_t nit = (int64_t)blockIdx.x < nelem ? (nelem - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint64_t pol = tma::policy_evict_first();

    auto elem_of = [&](int64_t it) -> int64_t {
        const int64_t pos = eoff + blockIdx.x + it * (int64_t)gridDim.x;
        return elist ? (int64_t)elist[pos] : pos;
    };
    auto issue = [&](int64_t it, int st) {
        const int64_t e = elem_of(it);
        tma::fence_proxy_async();
        tma::mbar_arrive_expect_tx(&S.full[st], BYTES);
        tma::bulk_g2s(S.stage[st], u + e * P3, P3 * 8, &S.full[st], pol);
        tma::bulk_g2s(S.stage[st] + P3, G + e * 6 * P3, 6 * P3 * 8, &S.full[st], pol);
        if (HELM) tma::bulk_g2s(S.stage[st] + 7 * P3, wJ + e * P3, P3 * 8, &S.full[st], pol);
        if (mbits) tma::bulk_g2s(S.mstage[st], mbits + e * 16, 64, &S.full[st], pol);
    };
    if (t == 0) {
        tma::mbar_init(&S.full[0], 1);
        tma::mbar_init(&S.full[1], 1);
        tma::fence_mbar_init();
    }
    if (t < 64) S.sD[t] = c_D[N][t];
    __syncthreads();
    if (t == 0) {
        if (nit > 0) issue(0, 0);
        if (nit > 1) issue(1, 1);
    }
    double Dri[NQ], Drj[NQ], Dci[NQ], Dcj[NQ];
#pragma unroll
    for (int m = 0; m < NQ; ++m) {
        Dri[m] = S.sD[i * NQ + m]; Drj[m] = S.sD[j * NQ + m];
        Dci[m] = S.sD[m * NQ + i]; Dcj[m] = S.sD[m * NQ + j];
    }
    double dot = 0.0;
    double *sa = S.sa[g], *sb = S.sb[g], *sc = S.sc[g];
    for (int64_t it = 0; it < nit; ++it) {
        const int st = (int)(it & 1);
        const int64_t e = elem_of(it);
        tma::mbar_wait(&S.full[st], (uint32_t)((it >> 1) & 1));
        const double *su = S.stage[st];
        const double *sG = su + P3;
        const uint32_t *mw = S.mstage[st];
        // the whole k-column of u (masked): needed by the t contraction
        double ru[NQ];
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            double v = su[k * 64 + c];
            if (mbits && ((mw[2 * k + (c >> 5)] >> (c & 31)) & 1u)) v = 0.0;
            ru[k] = v;
        }
        double ut[KPG], gt[KPG], rw[KPG];
#pragma unroll
        for (int kk = 0; kk < KPG; ++kk) {
            const double *Dk = S.sD + (k0 + kk) * NQ;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 d = *reinterpret_cast<const double2 *>(Dk + m);
                a0 = fma(d.x, ru[m], a0);
                a1 = fma(d.y, ru[m + 1], a1);
            }
            ut[kk] = a0 + a1;
        }
#pragma unroll
        for (int kk = 0; kk < KPG; ++kk) {
            const int k = k0 + kk;
            double uk = su[k * 64 + c];
            if (mbits && ((mw[2 * k + (c >> 5)] >> (c & 31)) & 1u)) uk = 0.0;
            sa[c] = uk;
            __syncthreads();
            double ur0 = 0.0, ur1 = 0.0, us0 = 0.0, us1 = 0.0;
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 a = *reinterpret_cast<const double2 *>(sa + j * NQ + m);
                ur0 = fma(Dri[m], a.x, ur0);
                ur1 = fma(Dri[m + 1], a.y, ur1);
                us0 = fma(Drj[m], sa[m * NQ + i], us0);
                us1 = fma(Drj[m + 1], sa[(m + 1) * NQ + i], us1);
            }
            const double ur = ur0 + ur1, us = us0 + us1;
            const int q = k * 64 + c;
            const double Grr = sG[q], Grs = sG[P3 + q], Grt = sG[2 * P3 + q];
            const double Gss = sG[3 * P3 + q], Gst = sG[4 * P3 + q], Gtt = sG[5 * P3 + q];
            sb[c] = Grr * ur + Grs * us + Grt * ut[kk];
            sc[c] = Grs * ur + Gss * us + Gst * ut[kk];
            gt[kk] = Grt * ur + Gst * us + Gtt * ut[kk];
            __syncthreads();
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 x = *reinterpret_cast<const double2 *>(sb + j * NQ + m);
                a0 = fma(Dci[m], x.x, a0);
                a1 = fma(Dci[m + 1], x.y, a1);
                b0 = fma(Dcj[m], sc[m * NQ + i], b0);
                b1 = fma(Dcj[m + 1], sc[(m + 1) * NQ + i], b1);
            }
            rw[kk] = (a0 + a1) + (b0 + b1);
        }
        // transposed t contraction: this group's slices contribute to every k
        double pt[NQ];
#pragma unroll
        for (int m = 0; m < NQ; ++m) pt[m] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KPG; ++kk) {
            const double *Dk = S.sD + (k0 + kk) * NQ;
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 d = *reinterpret_cast<const double2 *>(Dk + m);
                pt[m] = fma(d.x, gt[kk], pt[m]);
                pt[m + 1] = fma(d.y, gt[kk], pt[m + 1]);
            }
        }
        if (KS > 1) {
#pragma unroll
            for (int m = 0; m < NQ; ++m) S.spart[g][m][c] = pt[m];
            __syncthreads();
        }
#pragma unroll
        for (int kk = 0; kk < KPG; ++kk) {
            const int k = k0 + kk;
            double tt;
            if (KS > 1) {
                tt = S.spart[0][k][c];
#pragma unroll
                for (int gg = 1; gg < KS; ++gg) tt += S.spart[gg][k][c];
            } else {
                tt = pt[kk];
            }
            const int64_t l = e * P3 + k * 64 + c;
            const bool masked = mbits && ((mw[2 * k + (c >> 5)] >> (c & 31)) & 1u);
            const double uk = masked ? 0.0 : su[k * 64 + c];
            double v = h1 * (rw[kk] + tt);
            if (HELM) v = fma(h2 * su[7 * P3 + k * 64 + c], uk, v);
            if (masked) v = 0.0;
            w[l] = v;
            dot = fma(uk, v, dot);
        }
        __syncthreads();   // stage `st` fully consumed
        if (t == 0 && it + 2 < nit) issue(it + 2, st);
    }
    if (part) {
        const double sum = block_sum(dot, S.sred);
        if (t == 0) part[part_off + blockIdx.x] = sum;
        if (fin_total > 0) last_block_finish(part, fin_total, dst, counter, S.sred, &S.last);
    }
}

template <bool HELM, int KS>
static cudaError_t ax_v2_launch(const AxLaunch &L, const double *u, const double *G, const double *wJ,
                                const uint32_t *mbits, double h1, double h2, double *w, int64_t grid, cudaStream_t s)
{
    static bool attr = false;
    const size_t smem = sizeof(AxV2Smem<HELM, KS>);
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(ax_v2_kernel<HELM, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    ax_v2_kernel<HELM, KS><<<(unsigned)grid, 64 * KS, smem, s>>>(L.nelem, L.eoff, L.elist, u, G, wJ, mbits, h1, h2,
                                                                w, L.part, L.part_off, L.fin_total, L.dst,
                                                                L.counter, L.done);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- Ax v3
template <bool HELM, int KS>
__global__ void __launch_bounds__(64 * KS, KS == 1 ? 6 : 3)
    ax_v3_kernel(int64_t nelem, int64_t eoff, const int32_t *__restrict__ elist, const double *__restrict__ u,
                 const double *__restrict__ G, const double *__restrict__ wJ, const uint32_t *__restrict__ mbits,
                 double h1, double h2, double *__restrict__ w, double *__restrict__ part, int64_t part_off,
                 int64_t fin_total, double *__restrict__ dst, unsigned int *counter, const int *__restrict__ done)
{
    constexpr int NQ = 8, P3 = 512, N = 7, KPG = NQ / KS, PF = 2;
    if (done && *(volatile const int *)done) return;
    __shared__ AxV3Smem<KS> S;
    const int t = threadIdx.x, c = t & 63, g = t >> 6, i = c & 7, j = c >> 3;
    const int k0 = g * KPG;
    const int64_t nit = (int64_t)blockIdx.x < nelem ? (nelem - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint64_t pol = tma::policy_evict_first();
    auto elem_of = [&](int64_t it) -> int64_t {
        const int64_t pos = eoff + blockIdx.x + it * (int64_t)gridDim.x;
        return elist ? (int64_t)elist[pos] : pos;
    };
    auto prefetch = [&](int64_t it) {
        const int64_t e = elem_of(it);
        tma::prefetch_l2(u + e * P3, P3 * 8);
        tma::prefetch_l2(G + e * 6 * P3, 6 * P3 * 8);
        if (HELM) tma::prefetch_l2(wJ + e * P3, P3 * 8);
        if (mbits) tma::prefetch_l2(mbits + e * 16, 64);
    };
    if (t == 0)
        for (int a = 0; a < PF && a < nit; ++a) prefetch(a);
    if (t < 64) S.sD[t] = c_D[N][t];
    __syncthreads();
    double Dri[NQ], Drj[NQ], Dci[NQ], Dcj[NQ];
#pragma unroll
    for (int m = 0; m < NQ; ++m) {
        Dri[m] = S.sD[i * NQ + m]; Drj[m] = S.sD[j * NQ + m];
        Dci[m] = S.sD[m * NQ + i]; Dcj[m] = S.sD[m * NQ + j];
    }
    double dot = 0.0;
    double *sa = S.sa[g], *sb = S.sb[g], *sc = S.sc[g];
    for (int64_t it = 0; it < nit; ++it) {
        const int64_t e = elem_of(it);
        if (t == 0 && it + PF < nit) prefetch(it + PF);
        const double *ue = u + e * P3;
        const double *Ge = G + e * 6 * (int64_t)P3;
        uint32_t mw[2 * NQ];
        if (mbits) {
#pragma unroll
            for (int k = 0; k < NQ; ++k) mw[2 * k] = __ldg(mbits + e * 16 + 2 * k + (c >> 5)) >> (c & 31);
        }
        double ru[NQ];
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            double v = tma::ldg_ef(ue + k * 64 + c, pol);
            if (mbits && (mw[2 * k] & 1u)) v = 0.0;
            ru[k] = v;
        }
        double ut[KPG], gt[KPG], rw[KPG];
#pragma unroll
        for (int kk = 0; kk < KPG; ++kk) {
            const double *Dk = S.sD + (k0 + kk) * NQ;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 d = *reinterpret_cast<const double2 *>(Dk + m);
                a0 = fma(d.x, ru[m], a0);
                a1 = fma(d.y, ru[m + 1], a1);
            }
            ut[kk] = a0 + a1;
        }
        double Gn[6];
#pragma unroll
        for (int a = 0; a < 6; ++a) Gn[a] = tma::ldg_ef(Ge + a * P3 + k0 * 64 + c, pol);
#pragma unroll
        for (int kk = 0; kk < KPG; ++kk) {
            const int k = k0 + kk;
            double Gc[6];
#pragma unroll
            for (int a = 0; a < 6; ++a) Gc[a] = Gn[a];
            if (kk + 1 < KPG) {
#pragma unroll
                for (int a = 0; a < 6; ++a) Gn[a] = tma::ldg_ef(Ge + a * P3 + (k + 1) * 64 + c, pol);
            }
            if (KS == 1) {
                sa[c] = ru[kk];
            } else {
                double uk = ue[k * 64 + c];
                if (mbits && ((__ldg(mbits + e * 16 + 2 * k + (c >> 5)) >> (c & 31)) & 1u)) uk = 0.0;
                sa[c] = uk;
            }
            __syncthreads();
            double ur0 = 0.0, ur1 = 0.0, us0 = 0.0, us1 = 0.0;
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 a = *reinterpret_cast<const double2 *>(sa + j * NQ + m);
                ur0 = fma(Dri[m], a.x, ur0);
                ur1 = fma(Dri[m + 1], a.y, ur1);
                us0 = fma(Drj[m], sa[m * NQ + i], us0);
                us1 = fma(Drj[m + 1], sa[(m + 1) * NQ + i], us1);
            }
            const double ur = ur0 + ur1, us = us0 + us1;
            sb[c] = Gc[0] * ur + Gc[1] * us + Gc[2] * ut[kk];
            sc[c] = Gc[1] * ur + Gc[3] * us + Gc[4] * ut[kk];
            gt[kk] = Gc[2] * ur + Gc[4] * us + Gc[5] * ut[kk];
            __syncthreads();
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 x = *reinterpret_cast<const double2 *>(sb + j * NQ + m);
                a0 = fma(Dci[m], x.x, a0);
                a1 = fma(Dci[m + 1], x.y, a1);
                b0 = fma(Dcj[m], sc[m * NQ + i], b0);
                b1 = fma(Dcj[m + 1], sc[(m + 1) * NQ + i], b1);
            }
            rw[kk] = (a0 + a1) + (b0 + b1);
        }
        double pt[NQ];
#pragma unroll
        for (int m = 0; m < NQ; ++m) pt[m] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KPG; ++kk) {
            const double *Dk = S.sD + (k0 + kk) * NQ;
#pragma unroll
            for (int m = 0; m < NQ; m += 2) {
                const double2 d = *reinterpret_cast<const double2 *>(Dk + m);
                pt[m] = fma(d.x, gt[kk], pt[m]);
                pt[m + 1] = fma(d.y, gt[kk], pt[m + 1]);
            }
        }
        if (KS > 1) {
#pragma unroll
            for (int m = 0; m < NQ; ++m) S.spart[g][m][c] = pt[m];
            __syncthreads();
        }
#pragma unroll
        for (int kk = 0; kk < KPG; ++kk) {
            const int k = k0 + kk;
            double tt;
            if (KS > 1) {
                tt = S.spart[0][k][c];
#pragma unroll
                for (int gg = 1; gg < KS; ++gg) tt += S.spart[gg][k][c];
            } else {
                tt = pt[kk];
            }
            const int64_t l = e * P3 + k * 64 + c;
            bool masked;
            double uk;
            if (KS == 1) { uk = ru[kk]; masked = mbits && (mw[2 * kk] & 1u); }
            else {
                masked = mbits && ((__ldg(mbits + e * 16 + 2 * k + (c >> 5)) >> (c & 31)) & 1u);
                uk = masked ? 0.0 : ue[k * 64 + c];
            }
            double v = h1 * (rw[kk] + tt);
            if (HELM) v = fma(h2 * wJ[l], uk, v);
            if (masked) v = 0.0;
            w[l] = v;
            dot = fma(uk, v, dot);
        }
        if (KS > 1) __syncthreads();   // spart reuse
    }
    if (part) {
        const double sum = block_sum(dot, S.sred);
        if (t == 0) part[part_off + blockIdx.x] = sum;
        if (fin_total > 0) last_block_finish(part, fin_total, dst, counter, S.sred, &S.last);
    }
}

template <bool HELM, int KS>
static cudaError_t ax_v3_launch(const AxLaunch &L, const double *u, const double *G, const double *wJ,
                                const uint32_t *mbits, double h1, double h2, double *w, int64_t grid, cudaStream_t s)
{
    ax_v3_kernel<HELM, KS><<<(unsigned)grid, 64 * KS, 0, s>>>(L.nelem, L.eoff, L.elist, u, G, wJ, mbits, h1, h2, w,
                                                             L.part, L.part_off, L.fin_total, L.dst, L.counter,
                                                             L.done);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- Ax v4
// FP64 tensor cores (DMMA, mma.sync m8n8k4 f64) for the r and t contractions,
// registers for the s contraction, no shared-memory staging of the streams.
// One CTA = 4 warps per element; warp w owns the j-slabs {2w, 2w+1}; lane
// (q = lane & 3, r = lane >> 2) owns the points (i = 2q + v, j, k = r),
// v in {0,1}, which is exactly the m8n8 accumulator layout of an 8x8 (k, i)
// slab.  Contractions over i use a permuted K order (K = 2q + s) so the
// accumulator of one product feeds the A operand of the next without shuffles;
// the contraction over k needs k in the K position, so u is also loaded in
// the transposed layout (an L1 hit) and g_t goes through a per-warp shared
// transpose.  The j contraction stays inside each thread's j-line (u) or goes
// through one CTA-wide exchange (g_s).
__device__ __forceinline__ void dmma8x8x4(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

struct AxV4Smem {
    alignas(16) double sD[64];
    alignas(16) double sGS[2][8][8][8];    // [parity][k][j][i] g_s exchange
    alignas(16) double sGT[4][2][8][8];    // [warp][slab][k][i] g_t transpose
    double sred[128];
    int last;
};

template <bool HELM>
__global__ void __launch_bounds__(128, 3)
    ax_v4_kernel(int64_t nelem, int64_t eoff, const int32_t *__restrict__ elist, const double *__restrict__ u,
                 const double *__restrict__ G, const double *__restrict__ wJ, const uint32_t *__restrict__ mbits,
                 double h1, double h2, double *__restrict__ w, double *__restrict__ part, int64_t part_off,
                 int64_t fin_total, double *__restrict__ dst, unsigned int *counter, const int *__restrict__ done)
{
    constexpr int P3 = 512, N = 7;
    if (done && *(volatile const int *)done) return;
    __shared__ AxV4Smem S;
    const int t = threadIdx.x, lane = t & 31, wq = t >> 5, q = lane & 3, r = lane >> 2;
    const int64_t nit = (int64_t)blockIdx.x < nelem ? (nelem - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint64_t pol = tma::policy_evict_first();
    if (t < 64) S.sD[t] = c_D[N][t];
    __syncthreads();
    // D fragments
    double Br[2], At[2], Bt[2], Atr[2];
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
        Br[s2] = S.sD[r * 8 + 2 * q + s2];       // r fwd   B(K=(s,q), n=r) = D(i_out=r, m=2q+s)
        At[s2] = S.sD[r * 8 + 4 * s2 + q];       // t fwd   A(r, K=(s,q))   = D(k_out=r, m=4s+q)
        Bt[s2] = S.sD[(2 * q + s2) * 8 + r];     // r trans B(K=(s,q), n=r) = D(i=2q+s, i'=r)
        Atr[s2] = S.sD[(4 * s2 + q) * 8 + r];    // t trans A(r, K=(s,q))   = D(k=4s+q, k'=r)
    }
    const int jb = 2 * wq;                       // this warp's first slab
    double dot = 0.0;
    auto elem_at = [&](int64_t it) -> int64_t {
        const int64_t pos = eoff + blockIdx.x + it * (int64_t)gridDim.x;
        return elist ? (int64_t)elist[pos] : pos;
    };
    int64_t e_next = nit > 0 ? elem_at(0) : 0;
    for (int64_t it = 0; it < nit; ++it) {
        const int64_t e = e_next;                // element list read one iteration ahead
        if (it + 1 < nit) e_next = elem_at(it + 1);
        const double *ue = u + e * P3;
        const double *Ge = G + e * 6 * (int64_t)P3;
        const int par = (int)(it & 1);
        // Dirichlet words of the element: lanes 0..15 hold one each
        uint32_t mword = 0u;
        if (mbits && lane < 16) mword = __ldg(mbits + e * 16 + lane);
        // ---- loads: own j-lines of u, transposed u for the t-fwd B operand, own metric factors
        double2 uo[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) uo[m] = *reinterpret_cast<const double2 *>(ue + 64 * r + 8 * m + 2 * q);
        double ub[2][2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) ub[jj][s2] = ue[64 * (4 * s2 + q) + 8 * (jb + jj) + r];
        double2 Gv[2][6];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int a = 0; a < 6; ++a)
                Gv[jj][a] = *reinterpret_cast<const double2 *>(Ge + a * P3 + 64 * r + 8 * (jb + jj) + 2 * q);
        if (mbits) {
            const uint32_t w0 = __shfl_sync(0xffffffffu, mword, 2 * r), w1 = __shfl_sync(0xffffffffu, mword, 2 * r + 1);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const uint32_t wd = (m < 4 ? w0 : w1) >> (8 * (m & 3) + 2 * q);
                if (wd & 1u) uo[m].x = 0.0;
                if (wd & 2u) uo[m].y = 0.0;
            }
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const uint32_t wd = __shfl_sync(0xffffffffu, mword, 2 * (4 * s2 + q) + (wq >> 1));
#pragma unroll
                for (int jj = 0; jj < 2; ++jj)
                    if ((wd >> (8 * ((jb + jj) & 3) + r)) & 1u) ub[jj][s2] = 0.0;
            }
        }
        // ---- per own slab: r and t forward (DMMA), s forward (registers), metric, r transposed (DMMA)
        double2 acc[2], uj[2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {   // this warp's two slabs of u again (L1 hit; a runtime index
            const int j = jb + jj;         // into uo[] would go to local memory)
            uj[jj] = *reinterpret_cast<const double2 *>(ue + 64 * r + 8 * j + 2 * q);
            if (mbits) {
                const uint32_t wd = __shfl_sync(0xffffffffu, mword, 2 * r + (j >> 2)) >> (8 * (j & 3) + 2 * q);
                if (wd & 1u) uj[jj].x = 0.0;
                if (wd & 2u) uj[jj].y = 0.0;
            }
        }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = jb + jj;
            double ur0 = 0.0, ur1 = 0.0, ut0 = 0.0, ut1 = 0.0;
            dmma8x8x4(ur0, ur1, uj[jj].x, Br[0]);
            dmma8x8x4(ur0, ur1, uj[jj].y, Br[1]);
            dmma8x8x4(ut0, ut1, At[0], ub[jj][0]);
            dmma8x8x4(ut0, ut1, At[1], ub[jj][1]);
            double us0a = 0.0, us0b = 0.0, us1a = 0.0, us1b = 0.0;
#pragma unroll
            for (int m = 0; m < 8; m += 2) {
                const double2 d = *reinterpret_cast<const double2 *>(S.sD + j * 8 + m);
                us0a = fma(d.x, uo[m].x, us0a); us0b = fma(d.y, uo[m + 1].x, us0b);
                us1a = fma(d.x, uo[m].y, us1a); us1b = fma(d.y, uo[m + 1].y, us1b);
            }
            const double us0 = us0a + us0b, us1 = us1a + us1b;
            const double2 *Gj = Gv[jj];
            const double gr0 = Gj[0].x * ur0 + Gj[1].x * us0 + Gj[2].x * ut0;
            const double gr1 = Gj[0].y * ur1 + Gj[1].y * us1 + Gj[2].y * ut1;
            const double gs0 = Gj[1].x * ur0 + Gj[3].x * us0 + Gj[4].x * ut0;
            const double gs1 = Gj[1].y * ur1 + Gj[3].y * us1 + Gj[4].y * ut1;
            const double gt0 = Gj[2].x * ur0 + Gj[4].x * us0 + Gj[5].x * ut0;
            const double gt1 = Gj[2].y * ur1 + Gj[4].y * us1 + Gj[5].y * ut1;
            double wr0 = 0.0, wr1 = 0.0;
            dmma8x8x4(wr0, wr1, gr0, Bt[0]);
            dmma8x8x4(wr0, wr1, gr1, Bt[1]);
            acc[jj] = make_double2(wr0, wr1);
            *reinterpret_cast<double2 *>(&S.sGS[par][r][j][2 * q]) = make_double2(gs0, gs1);
            *reinterpret_cast<double2 *>(&S.sGT[wq][jj][r][2 * q]) = make_double2(gt0, gt1);
        }
        __syncwarp();
        // ---- t transposed (DMMA) from the per-warp transpose buffer
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            double wt0 = 0.0, wt1 = 0.0;
            dmma8x8x4(wt0, wt1, Atr[0], S.sGT[wq][jj][q][r]);
            dmma8x8x4(wt0, wt1, Atr[1], S.sGT[wq][jj][4 + q][r]);
            acc[jj].x += wt0;
            acc[jj].y += wt1;
        }
        __syncthreads();                                  // sGS[par] complete
        // ---- s transposed: w_s(i, j', k) = sum_j D(j, j') g_s(i, j, k)
        double2 gsl[8];
#pragma unroll
        for (int jx = 0; jx < 8; ++jx) gsl[jx] = *reinterpret_cast<const double2 *>(&S.sGS[par][r][jx][2 * q]);
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = jb + jj;
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
            for (int jx = 0; jx < 8; jx += 2) {
                const double d0 = S.sD[jx * 8 + j], d1 = S.sD[(jx + 1) * 8 + j];
                a0 = fma(d0, gsl[jx].x, a0); b0 = fma(d1, gsl[jx + 1].x, b0);
                a1 = fma(d0, gsl[jx].y, a1); b1 = fma(d1, gsl[jx + 1].y, b1);
            }
            const int64_t l = e * P3 + 64 * r + 8 * j + 2 * q;
            double v0 = h1 * (acc[jj].x + (a0 + b0)), v1 = h1 * (acc[jj].y + (a1 + b1));
            if (HELM) {
                const double2 wj = *reinterpret_cast<const double2 *>(wJ + l);
                v0 = fma(h2 * wj.x, uj[jj].x, v0);
                v1 = fma(h2 * wj.y, uj[jj].y, v1);
            }
            if (mbits) {
                const uint32_t wd = __shfl_sync(0xffffffffu, mword, 2 * r + (j >> 2)) >> (8 * (j & 3) + 2 * q);
                if (wd & 1u) v0 = 0.0;
                if (wd & 2u) v1 = 0.0;
            }
            *reinterpret_cast<double2 *>(w + l) = make_double2(v0, v1);
            dot = fma(uj[jj].x, v0, dot);
            dot = fma(uj[jj].y, v1, dot);
        }
    }
    if (part) {
        const double sum = block_sum(dot, S.sred);
        if (t == 0) part[part_off + blockIdx.x] = sum;
        if (fin_total > 0) last_block_finish(part, fin_total, dst, counter, S.sred, &S.last);
    }
    (void)pol;
}

template <bool HELM>
static cudaError_t ax_v4_launch(const AxLaunch &L, const double *u, const double *G, const double *wJ,
                                const uint32_t *mbits, double h1, double h2, double *w, int64_t grid, cudaStream_t s)
{
    ax_v4_kernel<HELM><<<(unsigned)grid, 128, 0, s>>>(L.nelem, L.eoff, L.elist, u, G, wJ, mbits, h1, h2, w, L.part,
                                                       L.part_off, L.fin_total, L.dst, L.counter, L.done);
    return cudaGetLastError();
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
template <bool HELM, bool FUSED, int MINB, bool L2PF = false, bool TMAG = false>
__global__ void __launch_bounds__(128, MINB)
    ax_v5_kernel(int64_t nelem, int64_t eoff, const int32_t *__restrict__ elist, const double *u,
                 const double *__restrict__ G, const double *__restrict__ wJ, const uint32_t *__restrict__ mbits,
                 double h1, double h2, double *__restrict__ w, double *__restrict__ part, int64_t part_off,
                 int64_t fin_total, double *__restrict__ dst, unsigned int *counter, const int *__restrict__ done,
                 double *pvec, double *__restrict__ xvec, const double *__restrict__ rvec,
                 const double *__restrict__ dvec, PcgScalars *sc, P2PMail mail, unsigned int ctas_total,
                 int keep, int fold, double *hist)
{
    constexpr int P3 = 512, N = 7;
    pdl_trigger();
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
    pdl_wait();                                  // predecessor's outputs (p, r, scalars) complete
    if (FUSED) { beta = sc->beta; alpha = sc->alpha; }   // issued beside the done load, not after it
    if (done && *(volatile const int *)done) {
        if (TMAG) {                              // drain the metric copies already in flight
            if (nit > 0) tma::mbar_wait(&gfull[0], 0);
            if (nit > 1) tma::mbar_wait(&gfull[1], 0);
        }
        return;
    }
    if (FUSED) {
        if ((fold & 1) && *(volatile const int *)&sc->fold_ready) {
            // folded bookkeeping: (rho', rr) of the last update from every rank (mailbox channel 1),
            // beta = rho' / rho, convergence / maxit; one CTA records it (no separate fin kernel)
            __shared__ double s_m[3];
            __shared__ int s_stop;
            if (t == 0) {
                mail_pull(mail, 1, s_m);
                const double rho1 = s_m[0], rr = s_m[1], rho = sc->rho, bb = sc->bb;
                const int it = sc->iter;
                const bool conv = sqrt(rr) <= sc->tol * bb, stop = conv || it >= sc->maxit;
                if ((fold & 2) && blockIdx.x == 0) {
                    sc->rr = rr;
                    if (hist) hist[it] = sqrt(rr) / bb;
                    sc->beta = rho1 / rho;
                    sc->rho_next = rho1;
                    if (conv) { sc->status = NEK_OK; sc->done = 1; }
                    else if (stop) { sc->status = NEK_MAXIT; sc->done = 1; }
                    __threadfence();
                }
                s_m[2] = rho1 / rho;
                s_stop = stop;
            }
            __syncthreads();
            if (s_stop) {
                if (TMAG) {
                    if (nit > 0) tma::mbar_wait(&gfull[0], 0);
                    if (nit > 1) tma::mbar_wait(&gfull[1], 0);
                }
                return;
            }
            beta = s_m[2];
        }
    }
    const int kb = 2 * wq;                       // this warp's first k-slab
    double dot = 0.0;
    int64_t e_next = nit > 0 ? elem_at(0) : 0;
    for (int64_t it = 0; it < nit; ++it) {
        const int64_t e = e_next;                // element list read one iteration ahead
        if (it + 1 < nit) e_next = elem_at(it + 1);
        const double *ue = u + e * P3;
        const double *Ge = G + e * 6 * (int64_t)P3;
        const int par = (int)(it & 1);
        if (L2PF && t == 0 && it + 1 < nit) {    // next element's streams into L2 while this one computes
            const int64_t pn = eoff + blockIdx.x + (it + 1) * (int64_t)gridDim.x;
            const int64_t en = elist ? (int64_t)elist[pn] : pn;
            tma::prefetch_l2(G + en * 6 * (int64_t)P3, 6 * P3 * 8);
            if (FUSED) {
                tma::prefetch_l2(pvec + en * P3, P3 * 8);
                tma::prefetch_l2(rvec + en * P3, P3 * 8);
                tma::prefetch_l2(dvec + en * P3, P3 * 8);
                tma::prefetch_l2(xvec + en * P3, P3 * 8);
            } else {
                tma::prefetch_l2(u + en * P3, P3 * 8);
            }
        }
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
            dot = fma(uk[kk].x, v0, dot);
            dot = fma(uk[kk].y, v1, dot);
        }
    }
    if (part) {
        const double sum = block_sum(dot, S.sred);
        if (t == 0) part[part_off + blockIdx.x] = sum;
        if (fin_total > 0)
            last_block_finish(part, fin_total, dst, counter, S.sred, &S.last, mail.nranks > 1 ? &mail : nullptr,
                              ctas_total);
    }
}

template <bool HELM, int MINB, bool L2PF = false, bool TMAG = false>
static cudaError_t ax_v5_launch(const AxLaunch &L, const double *u, const double *G, const double *wJ,
                                const uint32_t *mbits, double h1, double h2, double *w, int64_t grid, cudaStream_t s)
{
    const size_t dsm = TMAG ? 2 * 6 * 512 * sizeof(double) : 0;
    if (TMAG) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(ax_v5_kernel<HELM, true, MINB, L2PF, TMAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dsm);
            cudaFuncSetAttribute(ax_v5_kernel<HELM, false, MINB, L2PF, TMAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dsm);
            attr = true;
        }
    }
    if (L.fused)
        return launch_k(pdl_enabled(), ax_v5_kernel<HELM, true, MINB, L2PF, TMAG>, (unsigned)grid, 128, dsm, s, L.nelem,
                        L.eoff, L.elist, (const double *)L.p, G, wJ, mbits, h1, h2, w, L.part, L.part_off, L.fin_total,
                        L.dst, L.counter, L.done, L.p, L.x, L.r, L.dinv, const_cast<PcgScalars *>(L.sc), L.mail,
                        L.ctas_total ? L.ctas_total : (unsigned)grid, L.keep, L.fold, L.hist);
    else
        ax_v5_kernel<HELM, false, MINB, L2PF, TMAG><<<(unsigned)grid, 128, dsm, s>>>(L.nelem, L.eoff, L.elist, u, G, wJ, mbits, h1, h2, w,
                                                                  L.part, L.part_off, L.fin_total, L.dst, L.counter,
                                                                  L.done, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                                  L.mail, L.ctas_total ? L.ctas_total : (unsigned)grid, L.keep,
                                                                  0, nullptr);
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

// The fused PCG launch with L2-resident vectors: register streaming at 4 CTAs/SM (variant 12) beats the
// TMA metric ring at any size (config 2: 23.8 vs 22.6 GDOF/s, Ax 89% vs 83% of the copy peak by
// algorithmic bytes); nek_ax and the unfused launches keep the default (TMA ring: 32.4 vs 27.7).
int ax_effective_variant(int variant, int N, bool fused, int keep)
{
    return (variant == 0 && N == 7 && fused && keep) ? 12 : variant;
}

// the folded P2P bookkeeping (AxLaunch::fold) is implemented by the N = 7 kernel v5
bool ax_has_fold(int variant, int N)
{
    return N == 7 && (variant == 0 || variant == 8 || variant == 9 || variant == 10 || variant == 12);
}

bool ax_has_fused(int variant, int N)
{
    return ((variant == 0 || variant == 8 || variant == 9 || variant == 10 || variant == 12) && N == 7) ||
           use_v6(variant, N);
}

// variant (N = 7): 0 = default (v5, DMMA, k-slabs, 4 CTAs/SM), 8 = v5 at 3 CTAs/SM,
// 9 = v5 + L2 bulk prefetch of the next element, 10 = v5 + TMA ring for G (3 CTAs/SM), 12 = v5 at 4 CTAs/SM
// (the large-problem default, at any size), 1 = v0 (any N), 2 = v1, 3 = v2 with 2 k-groups,
// 4 = v2 with 4 k-groups, 5 = v3 with 2 k-groups, 6 = v3 with 1 k-group, 7 = v4 (DMMA, j-slabs)
constexpr int V5_SMALL_ELEMS_PER_CTA = 16;
static int per_sm_of(int variant)
{
    switch (variant) {
    case 0: return 4;
    case 8: return 3;
    case 9: return 4;
    case 10: return 3;
    case 12: return 4;
    case 7: return 3;
    case 6: return 6;
    case 2: return 3;
    case 3: return 3;
    case 4: return 2;
    case 5: return 3;
    default: return 0;
    }
}
int64_t ax_grid(int variant, int N, int64_t nelem)
{
    if (nelem <= 0) return 0;
    if (N == 7 && variant == 0 && nelem <= (int64_t)V5_SMALL_ELEMS_PER_CTA * 4 * 148)
        return std::min<int64_t>(nelem, 3 * 148);   // auto: the TMA-staged configuration (see launch_ax)
    if (N == 7 && per_sm_of(variant) > 0) return std::min<int64_t>(nelem, (int64_t)per_sm_of(variant) * 148);
    if (use_v6(variant, N)) {
        const int64_t nbat = (nelem + v6_epb(N) - 1) / v6_epb(N);
        return std::min<int64_t>(nbat, (int64_t)v6_minb(N) * 148);
    }
    const int epb = v0_epb(N + 1);
    return (nelem + epb - 1) / epb;
}

// enough partial slots for any variant (two concurrent launches of up to 4 CTAs per SM each)
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

int ax_partials_needed(int variant, int N, int64_t E)
{
    return (int)std::max<int64_t>(std::max<int64_t>(2 * ax_grid(variant, N, E), E), 2 * 4 * 148);
}

template <bool HELM>
static cudaError_t ax_v1_launch(const AxLaunch &L, const double *u, const double *G, const double *wJ,
                                const uint32_t *mbits, double h1, double h2, double *w, cudaStream_t s)
{
    static bool attr = false;
    const size_t smem = sizeof(AxV1Smem<HELM>);
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(ax_v1_kernel<HELM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int64_t grid = ax_grid(2, 7, L.nelem);
    ax_v1_kernel<HELM><<<(unsigned)grid, AXV1_THREADS, smem, s>>>(L.nelem, L.eoff, L.elist, u, G, wJ, mbits, h1, h2, w,
                                                                  L.part, L.part_off, L.fin_total, L.dst, L.counter,
                                                                  L.done);
    return cudaGetLastError();
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
    if (N == 7 && variant == 2) {
        if (nlaunch) ++*nlaunch;
        return h2 != 0.0 ? ax_v1_launch<true>(L, u, G, wJ, mbits, h1, h2, w, s)
                         : ax_v1_launch<false>(L, u, G, wJ, mbits, h1, h2, w, s);
    }
    if (N == 7 && (variant == 3 || variant == 4)) {
        if (nlaunch) ++*nlaunch;
        const int64_t grid = ax_grid(variant, N, L.nelem);
        if (variant == 4)
            return h2 != 0.0 ? ax_v2_launch<true, 4>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                             : ax_v2_launch<false, 4>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
        return h2 != 0.0 ? ax_v2_launch<true, 2>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                         : ax_v2_launch<false, 2>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
    }
    if (N == 7 && (variant == 0 || variant == 8 || variant == 9 || variant == 10 || variant == 12)) {
        if (nlaunch) ++*nlaunch;
        const int64_t grid = L.grid > 0 ? std::min<int64_t>(L.grid, L.nelem) : ax_grid(variant, N, L.nelem);
        if (variant == 12)
            return h2 != 0.0 ? ax_v5_launch<true, 4>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                             : ax_v5_launch<false, 4>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
        if (variant == 9)
            return h2 != 0.0 ? ax_v5_launch<true, 4, true>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                             : ax_v5_launch<false, 4, true>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
        if (variant == 10)
            return h2 != 0.0 ? ax_v5_launch<true, 3, false, true>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                             : ax_v5_launch<false, 3, false, true>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
        if (variant == 0) {
            // few elements per CTA (the pipeline never fills): TMA-staged metric prefetch at 3 CTAs/SM
            // (the fused PCG launch with L2-resident vectors runs variant 12 instead, see
            // ax_effective_variant); otherwise register streaming at 4 CTAs/SM (98% of the copy peak at scale)
            if (L.nelem <= (int64_t)V5_SMALL_ELEMS_PER_CTA * 4 * 148)
                return h2 != 0.0 ? ax_v5_launch<true, 3, false, true>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                                 : ax_v5_launch<false, 3, false, true>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
            return h2 != 0.0 ? ax_v5_launch<true, 4>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                             : ax_v5_launch<false, 4>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
        }
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
    if (N == 7 && variant == 7) {
        if (nlaunch) ++*nlaunch;
        const int64_t grid = ax_grid(variant, N, L.nelem);
        return h2 != 0.0 ? ax_v4_launch<true>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                         : ax_v4_launch<false>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
    }
    if (N == 7 && (variant == 6 || variant == 5)) {
        if (nlaunch) ++*nlaunch;
        const int64_t grid = ax_grid(variant, N, L.nelem);
        if (variant == 6)
            return h2 != 0.0 ? ax_v3_launch<true, 1>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                             : ax_v3_launch<false, 1>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
        return h2 != 0.0 ? ax_v3_launch<true, 2>(L, u, G, wJ, mbits, h1, h2, w, grid, s)
                         : ax_v3_launch<false, 2>(L, u, G, wJ, mbits, h1, h2, w, grid, s);
    }
    double *part = L.part ? L.part + L.part_off : nullptr;   // v0: one partial per CTA
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

// ---------------------------------------------------------- gather-scatter
constexpr int GS_PPT_DEFAULT = 8;
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

// Runs grouped by length (2: face, 4: edge, 8: vertex nodes of a box; anything
// else generic), each class kept in canonical first-touch order, copies
// ascending: the sum order of every run is unchanged (bit-exact with the
// oracle) but fixed-length runs need no offsets and load their indices as one
// vector (one dependent load level fewer).
// pairs / quads per thread: NEK_GS_PPT = 8 (8 pairs, 4 quads), 4 (4, 2), 2 (2, 1) or 1 (1, 1)
static int gs_ppt()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NEK_GS_PPT");
        v = e ? atoi(e) : GS_PPT_DEFAULT;
        if (v != 1 && v != 2 && v != 4 && v != 8) v = GS_PPT_DEFAULT;
    }
    return v;
}

// Each warp takes a contiguous block of runs of one class and lane l handles
// runs l, l+32, ... of it, so every warp-wide load touches consecutive runs
// (first-touch order keeps their copies close in memory).
template <class T, int GS_PAIRS_PER_THREAD, int GS_QUADS_PER_THREAD, bool PDLW = false>
__device__ __forceinline__ void gs_classes_body(int64_t wid, int lane, int64_t n2, const int2 *__restrict__ p2,
                                                int64_t n4, const int4 *__restrict__ p4, int64_t n8,
                                                const int4 *__restrict__ p8, int64_t ng,
                                                const int32_t *__restrict__ pg, const int32_t *__restrict__ og,
                                                T *__restrict__ v, uint64_t pol, const int *done = nullptr)
{
    const int64_t w2 = (n2 + 32 * GS_PAIRS_PER_THREAD - 1) / (32 * GS_PAIRS_PER_THREAD);
    const int64_t w4 = (n4 + 32 * GS_QUADS_PER_THREAD - 1) / (32 * GS_QUADS_PER_THREAD);
    const int64_t w8 = (n8 + 31) / 32;
    if (wid < w2) {
        const int64_t r0 = wid * 32 * GS_PAIRS_PER_THREAD + lane;
        int2 c[GS_PAIRS_PER_THREAD];
        T a[GS_PAIRS_PER_THREAD], b[GS_PAIRS_PER_THREAD];
#pragma unroll
        for (int q = 0; q < GS_PAIRS_PER_THREAD; ++q) if (r0 + 32 * q < n2) c[q] = tma::ldi2(p2 + r0 + 32 * q, pol);
        if (PDLW) {
            pdl_wait();
            if (done && *(volatile const int *)done) return;
        }
#pragma unroll
        for (int q = 0; q < GS_PAIRS_PER_THREAD; ++q)
            if (r0 + 32 * q < n2) { a[q] = tma::ld1(v + c[q].x, pol); b[q] = tma::ld1(v + c[q].y, pol); }
#pragma unroll
        for (int q = 0; q < GS_PAIRS_PER_THREAD; ++q)
            if (r0 + 32 * q < n2) { const T s = a[q] + b[q]; tma::st1(v + c[q].x, s, pol); tma::st1(v + c[q].y, s, pol); }
        return;
    }
    wid -= w2;
    if (wid < w4) {
        const int64_t r0 = wid * 32 * GS_QUADS_PER_THREAD + lane;
        int4 c[GS_QUADS_PER_THREAD];
        T a[GS_QUADS_PER_THREAD][4];
#pragma unroll
        for (int q = 0; q < GS_QUADS_PER_THREAD; ++q) if (r0 + 32 * q < n4) c[q] = tma::ldi4(p4 + r0 + 32 * q, pol);
        if (PDLW) {
            pdl_wait();
            if (done && *(volatile const int *)done) return;
        }
#pragma unroll
        for (int q = 0; q < GS_QUADS_PER_THREAD; ++q)
            if (r0 + 32 * q < n4) {
                a[q][0] = tma::ld1(v + c[q].x, pol); a[q][1] = tma::ld1(v + c[q].y, pol);
                a[q][2] = tma::ld1(v + c[q].z, pol); a[q][3] = tma::ld1(v + c[q].w, pol);
            }
#pragma unroll
        for (int q = 0; q < GS_QUADS_PER_THREAD; ++q)
            if (r0 + 32 * q < n4) {
                const T s = ((a[q][0] + a[q][1]) + a[q][2]) + a[q][3];
                tma::st1(v + c[q].x, s, pol); tma::st1(v + c[q].y, s, pol);
                tma::st1(v + c[q].z, s, pol); tma::st1(v + c[q].w, s, pol);
            }
        return;
    }
    wid -= w4;
    if (PDLW) {
        pdl_wait();
        if (done && *(volatile const int *)done) return;
    }
    if (wid < w8) {
        const int64_t r = wid * 32 + lane;
        if (r >= n8) return;
        const int4 a = p8[2 * r], b = p8[2 * r + 1];
        const T s = ((((((v[a.x] + v[a.y]) + v[a.z]) + v[a.w]) + v[b.x]) + v[b.y]) + v[b.z]) + v[b.w];
        v[a.x] = s; v[a.y] = s; v[a.z] = s; v[a.w] = s;
        v[b.x] = s; v[b.y] = s; v[b.z] = s; v[b.w] = s;
        return;
    }
    wid -= w8;
    const int64_t r = wid * 32 + lane;
    if (r < ng) {
        const int o0 = og[r], o1 = og[r + 1];
        T s = v[pg[o0]];
        for (int c = o0 + 1; c < o1; ++c) s += v[pg[c]];
        for (int c = o0; c < o1; ++c) v[pg[c]] = s;
    }
}

template <class T, int PPT>
__global__ void __launch_bounds__(256)
    gs_classes_kernel(int64_t n2, const int2 *__restrict__ p2, int64_t n4, const int4 *__restrict__ p4, int64_t n8,
                      const int4 *__restrict__ p8, int64_t ng, const int32_t *__restrict__ pg,
                      const int32_t *__restrict__ og, T *__restrict__ v, const int *done, int keep)
{
    pdl_trigger();
    gs_classes_body<T, PPT, (PPT > 1 ? PPT / 2 : 1), true>((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5,
                                                            threadIdx.x & 31, n2, p2, n4, p4, n8, p8, ng, pg, og, v,
                                                            tma::policy_keep(keep), done);
}

static int64_t gs_class_warps(const GsClasses &C, int ppt)
{
    const int qpt = ppt > 1 ? ppt / 2 : 1;
    return (C.n2 + 32 * ppt - 1) / (32 * ppt) + (C.n4 + 32 * qpt - 1) / (32 * qpt) + (C.n8 + 31) / 32 +
           (C.ng + 31) / 32;
}

// local runs (warps [0, cw)) and, after them, the halo unpack (warps [cw, ...)):
// one lane per interface run waits for this epoch's halo of every neighbour,
// folds the contributions in rank order and writes the total to the local copies.
template <class T, int PPT>
__global__ void __launch_bounds__(256)
    gs_classes_unpack_kernel(int64_t n2, const int2 *__restrict__ p2, int64_t n4, const int4 *__restrict__ p4,
                             int64_t n8, const int4 *__restrict__ p8, int64_t ng, const int32_t *__restrict__ pg,
                             const int32_t *__restrict__ og, int64_t cw, HaloUnpack U, T *__restrict__ v,
                             const int *done, int C_keep)
{
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const bool skip = done && *(volatile const int *)done;
    if (wid < cw) {
        if (!skip) gs_classes_body<T, PPT, (PPT > 1 ? PPT / 2 : 1)>(wid, lane, n2, p2, n4, p4, n8, p8, ng, pg, og, v, tma::policy_keep(C_keep));
        return;
    }
    const uint64_t e = *(volatile const uint64_t *)(U.epochs + 2);
    if (lane == 0)
        for (int k = 0; k < U.nnbr; ++k) wait_epoch(U.hflags + U.nbr[k], e, U.err);
    __syncwarp();
    if (skip) return;
    const int64_t r = (wid - cw) * 32 + lane;
    if (r >= U.nifc) return;
    const T *recv = reinterpret_cast<const T *>(U.recv) + (int64_t)(e & 1) * U.half;
    const T *partial = reinterpret_cast<const T *>(U.partial);
    const int c0 = U.coffs[r], c1 = U.coffs[r + 1];
    int src = U.contrib[c0];
    T s = src < 0 ? partial[r] : ((volatile const T *)recv)[src];
    for (int c = c0 + 1; c < c1; ++c) {
        src = U.contrib[c];
        s += src < 0 ? partial[r] : ((volatile const T *)recv)[src];
    }
    for (int c = U.offs[r]; c < U.offs[r + 1]; ++c) v[U.perm[c]] = s;
}

template <class T>
cudaError_t launch_gs_classes_unpack(const GsClasses &C, const HaloUnpack &U, T *v, const int *done,
                                     cudaStream_t s)
{
    const int ppt = gs_ppt();
    const int64_t cw = gs_class_warps(C, ppt), uw = (U.nifc + 31) / 32;
    const int64_t warps = cw + std::max<int64_t>(uw, 1);   // at least one waiting warp keeps epochs in step
    const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
#define NEK_GSU(PP)                                                                                                   \
    gs_classes_unpack_kernel<T, PP><<<grid, 256, 0, s>>>(C.n2, (const int2 *)C.p2, C.n4, (const int4 *)C.p4, C.n8,     \
                                                        (const int4 *)C.p8, C.ng, C.pg, C.og, cw, U, v, done, C.keep)
    if (ppt == 1) NEK_GSU(1); else if (ppt == 2) NEK_GSU(2); else if (ppt == 4) NEK_GSU(4); else NEK_GSU(8);
#undef NEK_GSU
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_gs_classes(const GsClasses &C, T *v, const int *done, cudaStream_t s)
{
    const int ppt = gs_ppt();
    const int64_t warps = gs_class_warps(C, ppt);
    if (warps <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
#define NEK_GSC(PP)                                                                                                   \
    return launch_k(pdl_enabled(), gs_classes_kernel<T, PP>, grid, 256, 0, s, C.n2, (const int2 *)C.p2, C.n4,          \
                    (const int4 *)C.p4, C.n8, (const int4 *)C.p8, C.ng, (const int32_t *)C.pg,                        \
                    (const int32_t *)C.og, v, done, C.keep)
    if (ppt == 1) NEK_GSC(1); else if (ppt == 2) NEK_GSC(2); else if (ppt == 4) NEK_GSC(4); else NEK_GSC(8);
#undef NEK_GSC
    return cudaGetLastError();
}

template <class T>
__global__ void gs_ifc_partial_kernel(int64_t nifc, const int32_t *__restrict__ perm, const int32_t *__restrict__ offs,
                                      const T *__restrict__ v, T *__restrict__ partial, const int *done)
{
    if (done && *(volatile const int *)done) return;
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nifc) return;
    const int o0 = offs[r], o1 = offs[r + 1];
    T s = v[perm[o0]];
    for (int c = o0 + 1; c < o1; ++c) s += v[perm[c]];
    partial[r] = s;
}

template <class T>
__global__ void gs_pack_kernel(int64_t nslots, const int32_t *__restrict__ send_run, const T *__restrict__ partial,
                               T *__restrict__ sendbuf, const int *done)
{
    if (done && *(volatile const int *)done) return;
    const int64_t sidx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sidx < nslots) sendbuf[sidx] = partial[send_run[sidx]];
}

template <class T>
cudaError_t launch_gs_ifc_pack(int64_t nifc, const int32_t *perm, const int32_t *offs, const T *v,
                               T *partial, int64_t nslots, const int32_t *send_run, T *sendbuf,
                               const int *done, cudaStream_t s)
{
    if (nifc > 0) gs_ifc_partial_kernel<<<(unsigned)((nifc + 255) / 256), 256, 0, s>>>(nifc, perm, offs, v, partial, done);
    if (nslots > 0) gs_pack_kernel<<<(unsigned)((nslots + 255) / 256), 256, 0, s>>>(nslots, send_run, partial, sendbuf, done);
    return cudaGetLastError();
}

// total = fold of contributions in ascending rank order (own partial or a
// received slot), then written to every local copy.
template <class T>
__global__ void gs_unpack_kernel(int64_t nifc, const int32_t *__restrict__ perm, const int32_t *__restrict__ offs,
                                 const int32_t *__restrict__ coffs, const int32_t *__restrict__ contrib,
                                 const T *__restrict__ partial, const T *__restrict__ recvbuf,
                                 T *__restrict__ v, const int *done, const uint64_t *epoch, int64_t half)
{
    if (done && *(volatile const int *)done) return;
    if (epoch) recvbuf += (int64_t)(*epoch & 1) * half;   // P2P: double-buffered by epoch parity
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nifc) return;
    const int c0 = coffs[r], c1 = coffs[r + 1];
    int src = contrib[c0];
    T s = src < 0 ? partial[r] : recvbuf[src];
    for (int c = c0 + 1; c < c1; ++c) {
        src = contrib[c];
        s += src < 0 ? partial[r] : recvbuf[src];
    }
    for (int c = offs[r]; c < offs[r + 1]; ++c) v[perm[c]] = s;
}

template <class T>
cudaError_t launch_gs_ifc_unpack(int64_t nifc, const int32_t *perm, const int32_t *offs, const int32_t *coffs,
                                 const int32_t *contrib, const T *partial, const T *recvbuf, T *v,
                                 const int *done, cudaStream_t s, const uint64_t *epoch, int64_t half)
{
    if (nifc <= 0) return cudaSuccess;
    gs_unpack_kernel<<<(unsigned)((nifc + 255) / 256), 256, 0, s>>>(nifc, perm, offs, coffs, contrib, partial,
                                                                    recvbuf, v, done, epoch, half);
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
    copy_mask_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(n, mbits, src, dst);
    return cudaGetLastError();
}

// --------------------------------------------------------------------- PCG
constexpr int VEC_THREADS = 256;
constexpr int VEC_UNROLL = 4;
constexpr int UPD_CFG_DEFAULT = 2;
int vec_blocks() { return 148 * 4; }
// residual-update CTAs per SM: NEK_UPD_CFG = 2 (4 double2 per thread per tile), 4 (4) or 8 (2)
static int upd_cfg()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NEK_UPD_CFG");
        v = e ? atoi(e) : UPD_CFG_DEFAULT;
        if (v != 2 && v != 4 && v != 8) v = UPD_CFG_DEFAULT;
    }
    return v;
}
int upd_blocks() { return 148 * upd_cfg(); }

// red_all holds [nranks][RED_N]; sums are taken in rank order.
__device__ __forceinline__ double rank_sum(const double *red_all, int nranks, int slot)
{
    double s = red_all[slot];
    for (int q = 1; q < nranks; ++q) s += red_all[q * RED_N + slot];
    return s;
}

// r = M b, p = Dinv r, x = 0; [<r, Dinv r>_o, <r, r>_o] reduced by the last CTA into dst[0..1].
__device__ __forceinline__ void last_block_finish2(double *part, int nblk, double *dst, unsigned int *counter,
                                                   double *sred, int *s_last)
{
    if (threadIdx.x == 0) {
        __threadfence();
        *s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (*s_last) {
        __threadfence();
        double a0 = 0.0, a1 = 0.0;
        for (int c = threadIdx.x; c < nblk; c += blockDim.x) {
            a0 += ((volatile double *)part)[2 * c];
            a1 += ((volatile double *)part)[2 * c + 1];
        }
        a0 = block_sum(a0, sred);
        a1 = block_sum(a1, sred);
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
    double a0 = 0.0, a1 = 0.0;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x) {
        const double rv = bit_of(mbits, l) ? 0.0 : b[l];
        const double z = dinv[l] * rv;
        r[l] = rv;
        p[l] = p_zero ? 0.0 : z;
        x[l] = 0.0;
        if (bit_of(obits, l)) { a0 = fma(rv, z, a0); a1 = fma(rv, rv, a1); }
    }
    a0 = block_sum(a0, sred);
    a1 = block_sum(a1, sred);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = a0; part[2 * blockIdx.x + 1] = a1; }
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
    double a0 = 0.0, a1 = 0.0;
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
                if (ow[q] & 1u) { a0 = fma(rv[q].x, dv[q].x * rv[q].x, a0); a1 = fma(rv[q].x, rv[q].x, a1); }
                if (ow[q] & 2u) { a0 = fma(rv[q].y, dv[q].y * rv[q].y, a0); a1 = fma(rv[q].y, rv[q].y, a1); }
            }
        }
    }
    if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const int64_t l = n - 1;
        x[l] = fma(alpha, p[l], x[l]);
        const double rv = fma(-alpha, w[l], r[l]);
        r[l] = rv;
        if (bit_of(obits, l)) { a0 = fma(rv, dinv[l] * rv, a0); a1 = fma(rv, rv, a1); }
    }
    a0 = block_sum(a0, sred);
    a1 = block_sum(a1, sred);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = a0; part[2 * blockIdx.x + 1] = a1; }
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
// QQ^T w at one local point from the unassembled w (gather-scatter folded into the
// residual update).  id = -1: not in a local run (unshared, or an interface copy
// whose total the halo unpack already wrote); id >= 0: the other copy of a pair
// run (a + b == b + a exactly, so both copies get the canonical bits); id <= -2:
// run -(id+2) of the generic list, folded in canonical order.
__device__ __forceinline__ double w_assembled(int32_t id, double wl, const double *__restrict__ w, const GsInline &gi)
{
    if (id == -1) return wl;
    if (id >= 0) return wl + __ldg(w + id);
    const int run = -id - 2;
    const int o0 = gi.offs[run], o1 = gi.offs[run + 1];
    double s = __ldg(w + gi.perm[o0]);
    for (int c = o0 + 1; c < o1; ++c) s += __ldg(w + gi.perm[c]);
    return s;
}

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
                            unsigned int *counter, P2PMail mail, GsInline gi, int keep, int fold)
{
    __shared__ double sred[VEC_THREADS];
    __shared__ int s_last;
    __shared__ double s_sig[3];
    pdl_trigger();
    pdl_wait();
    const uint64_t pol = tma::policy_keep(keep & 1);
    const int64_t n2 = n >> 1;
    const int2 *i2 = reinterpret_cast<const int2 *>(gi.idx);
    const int64_t tile = (int64_t)UNR * blockDim.x;
    int64_t base = blockIdx.x * tile + threadIdx.x;
    double2 wv[UNR], dv[UNR], rv[UNR];
    uint32_t ow[UNR];
    int2 id[UNR];
    auto load = [&](int64_t b0) {
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
            const int64_t h = b0 + (int64_t)q * blockDim.x;
            if (h < n2) {
                wv[q] = tma::ld2(w + 2 * h, pol); dv[q] = tma::ld2(dinv + 2 * h, pol); rv[q] = tma::ld2(r + 2 * h, pol);
                ow[q] = tma::ldu(obits + ((2 * h) >> 5), pol) >> ((2 * h) & 31);
                if (gi.idx) id[q] = i2[h];
            }
        }
    };
    // the first tile's streams are issued before the dependent scalar reads (done, sigma, rho), so
    // their latencies overlap; w, r, Dinv are complete (stream order) whatever the scalars say
    load(base);
    if (*(volatile int *)&sc->done) return;
    double sigma;
    if (mail.nranks > 1) {                       // sigma of every rank from the mailbox (channel 0)
        if (threadIdx.x < 32) mail_pull_warp(mail, 0, s_sig);
        __syncthreads();
        sigma = s_sig[0];
        if (blockIdx.x == 0 && threadIdx.x == 0) sc->sigma = sigma;
    } else {
        sigma = rank_sum(red_all, nranks, RED_SIGMA);
    }
    if (!(sigma > 0.0)) {                       // breakdown: <p, A p> <= 0
        if (blockIdx.x == 0 && threadIdx.x == 0) { sc->status = NEK_ENOTSPD; sc->alpha = 0.0; sc->done = 1; }
        return;
    }
    const double alpha = (fold ? sc->rho_next : sc->rho) / sigma;
    double a0 = 0.0, a1 = 0.0;
    for (bool first = true; base < n2; base += (int64_t)gridDim.x * tile, first = false) {
        if (!first) load(base);
        if (gi.idx) {   // the gather-scatter QQ^T of w, on the fly (canonical order, bit-exact)
#pragma unroll
            for (int q = 0; q < UNR; ++q) {
                const int64_t h = base + (int64_t)q * blockDim.x;
                if (h < n2) {
                    wv[q].x = w_assembled(id[q].x, wv[q].x, w, gi);
                    wv[q].y = w_assembled(id[q].y, wv[q].y, w, gi);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
            const int64_t h = base + (int64_t)q * blockDim.x;
            if (h < n2) {
                rv[q].x = fma(-alpha, wv[q].x, rv[q].x); rv[q].y = fma(-alpha, wv[q].y, rv[q].y);
                tma::st2(r + 2 * h, rv[q], pol);
                if (ow[q] & 1u) { a0 = fma(rv[q].x, dv[q].x * rv[q].x, a0); a1 = fma(rv[q].x, rv[q].x, a1); }
                if (ow[q] & 2u) { a0 = fma(rv[q].y, dv[q].y * rv[q].y, a0); a1 = fma(rv[q].y, rv[q].y, a1); }
            }
        }
    }
    if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const int64_t l = n - 1;
        const double wl = gi.idx ? w_assembled(gi.idx[l], w[l], w, gi) : w[l];
        const double rv = fma(-alpha, wl, r[l]);
        r[l] = rv;
        if (bit_of(obits, l)) { a0 = fma(rv, dinv[l] * rv, a0); a1 = fma(rv, rv, a1); }
    }
    a0 = block_sum(a0, sred);
    a1 = block_sum(a1, sred);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = a0; part[2 * blockIdx.x + 1] = a1; }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        double b0 = 0.0, b1 = 0.0;
        for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) {
            b0 += ((volatile double *)part)[2 * c];
            b1 += ((volatile double *)part)[2 * c + 1];
        }
        b0 = block_sum(b0, sred);
        b1 = block_sum(b1, sred);
        if (threadIdx.x == 0) {
            *counter = 0u;
            if (nranks == 1) pcg_bookkeep(sc, b0, b1, alpha, hist);
            else if (mail.nranks > 1) {
                if (fold) {                      // the next Ax pulls (rho', rr) and does the bookkeeping
                    sc->alpha = alpha;
                    sc->iter += 1;
                    sc->rho = sc->rho_next;
                    sc->fold_ready = 1;
                    __threadfence();
                }
                mail_push(mail, 1, b0, b1, 0.0);   // to every rank (channel 1)
            }
            else { dst[0] = b0; dst[1] = b1; }
        }
    }
}

// The same residual update with the three streams (w, r, Dinv) staged through shared memory by TMA
// bulk copies: a 4-stage ring of 1024-point chunks per CTA, the chunk three ahead in flight while
// this one is consumed, so the bytes in flight do not depend on registers.  Measured at config 2:
// 21.9 vs 20.1 us per launch for the register-streamed kernel above (whose time is dominated by the
// dependent scalar reads at entry and the last-CTA finish, not by memory-level parallelism), so it
// is off by default; NEK_UPD_TMA=1 selects it.
constexpr int UPT_CH = 1024, UPT_ST = 4, UPT_THREADS = 256;
constexpr size_t UPT_SMEM = (size_t)UPT_ST * 3 * UPT_CH * sizeof(double);

__global__ void __launch_bounds__(UPT_THREADS, 2)
    pcg_update_tma_kernel(int64_t n, const uint32_t *__restrict__ obits, const double *__restrict__ dinv,
                          const double *__restrict__ w, double *__restrict__ r, const double *__restrict__ red_all,
                          int nranks, PcgScalars *sc, double *hist, double *__restrict__ part, double *dst,
                          unsigned int *counter, P2PMail mail, int keep)
{
    extern __shared__ __align__(128) double ring[];    // [stage][w | r | Dinv][UPT_CH]
    __shared__ uint64_t full[UPT_ST];
    __shared__ double sred[32];
    __shared__ int s_last;
    __shared__ double s_sig[3];
    if (*(volatile int *)&sc->done) return;
    const int t = threadIdx.x;
    double sigma;
    if (mail.nranks > 1) {                       // sigma of every rank from the mailbox (channel 0)
        if (t == 0) mail_pull(mail, 0, s_sig);
        __syncthreads();
        sigma = s_sig[0];
        if (blockIdx.x == 0 && t == 0) sc->sigma = sigma;
    } else {
        sigma = rank_sum(red_all, nranks, RED_SIGMA);
    }
    if (!(sigma > 0.0)) {                        // breakdown: <p, A p> <= 0
        if (blockIdx.x == 0 && t == 0) { sc->status = NEK_ENOTSPD; sc->alpha = 0.0; sc->done = 1; }
        return;
    }
    const double alpha = sc->rho / sigma;
    const uint64_t pol = tma::policy_keep(keep & 1);
    const int64_t nch = (n + UPT_CH - 1) / UPT_CH;
    const int64_t nk = (int64_t)blockIdx.x < nch ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (t == 0) {
        for (int q = 0; q < UPT_ST; ++q) tma::mbar_init(&full[q], 1);
        tma::fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t k, int st) {
        const int64_t c0 = (blockIdx.x + k * (int64_t)gridDim.x) * UPT_CH;
        const int64_t cnt = n - c0 < UPT_CH ? n - c0 : UPT_CH;
        const uint32_t bytes = (uint32_t)((cnt * 8) & ~(int64_t)15);
        tma::fence_proxy_async();
        tma::mbar_arrive_expect_tx(&full[st], 3 * bytes);
        if (bytes) {
            double *sb = ring + (size_t)st * 3 * UPT_CH;
            tma::bulk_g2s(sb, w + c0, bytes, &full[st], pol);
            tma::bulk_g2s(sb + UPT_CH, r + c0, bytes, &full[st], pol);
            tma::bulk_g2s(sb + 2 * UPT_CH, dinv + c0, bytes, &full[st], pol);
        }
    };
    if (t == 0)
        for (int q = 0; q < UPT_ST && q < nk; ++q) issue(q, q);
    double a0 = 0.0, a1 = 0.0;
    for (int64_t k = 0; k < nk; ++k) {
        const int st = (int)(k % UPT_ST);
        tma::mbar_wait(&full[st], (uint32_t)((k / UPT_ST) & 1));
        const int64_t c0 = (blockIdx.x + k * (int64_t)gridDim.x) * UPT_CH;
        const int cnt = (int)(n - c0 < UPT_CH ? n - c0 : UPT_CH);
        const int covered = (int)(((int64_t)cnt * 8 & ~(int64_t)15) / 8);
        const double *sb = ring + (size_t)st * 3 * UPT_CH;
#pragma unroll
        for (int q = 0; q < UPT_CH / (2 * UPT_THREADS); ++q) {
            const int p = 2 * (t + q * UPT_THREADS);
            if (p >= cnt) continue;
            const uint32_t ow = tma::ldu(obits + ((c0 + p) >> 5), pol) >> ((c0 + p) & 31);
            if (p + 2 <= covered) {
                const double2 wv = *reinterpret_cast<const double2 *>(sb + p);
                double2 rv = *reinterpret_cast<const double2 *>(sb + UPT_CH + p);
                const double2 dv = *reinterpret_cast<const double2 *>(sb + 2 * UPT_CH + p);
                rv.x = fma(-alpha, wv.x, rv.x);
                rv.y = fma(-alpha, wv.y, rv.y);
                tma::st2(r + c0 + p, rv, pol);
                if (ow & 1u) { a0 = fma(rv.x, dv.x * rv.x, a0); a1 = fma(rv.x, rv.x, a1); }
                if (ow & 2u) { a0 = fma(rv.y, dv.y * rv.y, a0); a1 = fma(rv.y, rv.y, a1); }
            } else {                             // odd tail point (n odd), read directly
                const int64_t l = c0 + p;
                const double rv = fma(-alpha, w[l], r[l]);
                r[l] = rv;
                if (ow & 1u) { a0 = fma(rv, dinv[l] * rv, a0); a1 = fma(rv, rv, a1); }
            }
        }
        __syncthreads();                         // stage st consumed by every thread
        if (t == 0 && k + UPT_ST < nk) issue(k + UPT_ST, st);
    }
    a0 = block_sum(a0, sred);
    a1 = block_sum(a1, sred);
    if (t == 0) { part[2 * blockIdx.x] = a0; part[2 * blockIdx.x + 1] = a1; }
    if (t == 0) {
        __threadfence();
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        double b0 = 0.0, b1 = 0.0;
        for (int c = t; c < (int)gridDim.x; c += blockDim.x) {
            b0 += ((volatile double *)part)[2 * c];
            b1 += ((volatile double *)part)[2 * c + 1];
        }
        b0 = block_sum(b0, sred);
        b1 = block_sum(b1, sred);
        if (t == 0) {
            *counter = 0u;
            if (nranks == 1) pcg_bookkeep(sc, b0, b1, alpha, hist);
            else if (mail.nranks > 1) mail_push(mail, 1, b0, b1, 0.0);   // to every rank (channel 1)
            else { dst[0] = b0; dst[1] = b1; }
        }
    }
}

static bool upd_tma()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NEK_UPD_TMA");
        v = e ? atoi(e) != 0 : 0;
    }
    return v;
}

cudaError_t launch_pcg_update_fused(int64_t n, const uint32_t *obits, const double *dinv, const double *w, double *r,
                                    const double *red_all, int nranks, PcgScalars *sc, double *hist, double *part,
                                    int nblk, double *dst, unsigned int *counter, cudaStream_t s,
                                    const P2PMail *mail, const GsInline *gi, int keep, int fold)
{
    P2PMail m;
    if (mail) m = *mail;
    GsInline g;
    if (gi) g = *gi;
    if (!g.idx && upd_tma() && !fold) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(pcg_update_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)UPT_SMEM);
            attr = true;
        }
        pcg_update_tma_kernel<<<148 * 2, UPT_THREADS, UPT_SMEM, s>>>(n, obits, dinv, w, r, red_all, nranks, sc, hist,
                                                                     part, dst, counter, m, keep);
        return cudaGetLastError();
    }
    switch (nblk / 148) {
    case 8:
        return launch_k(pdl_enabled(), pcg_update_fused_kernel<2, 8>, nblk, VEC_THREADS, 0, s, n, obits, dinv, w, r,
                        red_all, nranks, sc, hist, part, dst, counter, m, g, keep, fold);
        break;
    case 4:
        return launch_k(pdl_enabled(), pcg_update_fused_kernel<4, 4>, nblk, VEC_THREADS, 0, s, n, obits, dinv, w, r,
                        red_all, nranks, sc, hist, part, dst, counter, m, g, keep, fold);
        break;
    default:
        return launch_k(pdl_enabled(), pcg_update_fused_kernel<4, 2>, nblk, VEC_THREADS, 0, s, n, obits, dinv, w, r,
                        red_all, nranks, sc, hist, part, dst, counter, m, g, keep, fold);
    }
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

// folded path, after the last update of a solve: the bookkeeping its (rho', rr) would get from the next Ax
__global__ void pcg_fold_finish_kernel(PcgScalars *sc, P2PMail mail, double *hist)
{
    if (sc->done || !sc->fold_ready) return;
    double v[3];
    mail_pull(mail, 1, v);
    const double rr = v[1], bb = sc->bb;
    const int it = sc->iter;
    sc->rr = rr;
    if (hist) hist[it] = sqrt(rr) / bb;
    sc->beta = v[0] / sc->rho;
    sc->rho_next = v[0];
    if (sqrt(rr) <= sc->tol * bb) { sc->status = NEK_OK; sc->done = 1; }
    else if (it >= sc->maxit) { sc->status = NEK_MAXIT; sc->done = 1; }
}

cudaError_t launch_pcg_fold_finish(PcgScalars *sc, const P2PMail &mail, double *hist, cudaStream_t s)
{
    pcg_fold_finish_kernel<<<1, 1, 0, s>>>(sc, mail, hist);
    return cudaGetLastError();
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
    l2_demote_kernel<<<148 * 4, 256, 0, s>>>(R);
    return cudaGetLastError();
}

// ------------------------------------------------ NVLink peer-memory exchange
// One process per GPU; every rank maps its peers' mailbox / halo buffers
// (CUDA IPC) and writes into them directly over NVLink.  A value block is
// followed by a system-scope release store of a monotonically increasing
// epoch; the reader acquires the epoch and then reads.  All ranks run the same
// sequence of exchanges, so epochs agree.  Spins give up after ~2^26 polls and
// raise *err (no hang if a peer died).
// mailbox layout: [channel][epoch parity][rank][4] doubles; slot 3 holds the epoch
// (as u64).  The parity split means a slot is rewritten only two exchanges later,
// by which time its reader has provably consumed it.
__global__ void red_exchange_kernel(int channel, int me, int nranks, const double *__restrict__ red_loc,
                                    double *__restrict__ red_all, double *mbox, double *const *peer_mbox,
                                    uint64_t *epochs, int *err)
{
    __shared__ uint64_t s_e;
    const int q = threadIdx.x;
    if (q == 0) s_e = ++epochs[channel];
    __syncthreads();
    const uint64_t e = s_e;
    const size_t base = ((size_t)channel * 2 + (e & 1)) * nranks;
    if (q < nranks) {
        double *dst = (q == me ? mbox : peer_mbox[q]) + (base + me) * 4;
        dst[0] = red_loc[0]; dst[1] = red_loc[1]; dst[2] = red_loc[2];
        __threadfence_system();
        st_release_sys(reinterpret_cast<uint64_t *>(dst + 3), e);
    }
    if (q < nranks) {
        const double *src = mbox + (base + q) * 4;
        if (wait_epoch(reinterpret_cast<const uint64_t *>(src + 3), e, err)) {
            red_all[q * RED_N + 0] = ((volatile const double *)src)[0];
            red_all[q * RED_N + 1] = ((volatile const double *)src)[1];
            red_all[q * RED_N + 2] = ((volatile const double *)src)[2];
        }
    }
}

cudaError_t launch_red_exchange(int channel, int me, int nranks, const double *red_loc, double *red_all, double *mbox,
                                double *const *peer_mbox, uint64_t *epochs, int *err, cudaStream_t s)
{
    red_exchange_kernel<<<1, 32, 0, s>>>(channel, me, nranks, red_loc, red_all, mbox, peer_mbox, epochs, err);
    return cudaGetLastError();
}

// pack with the interface partials folded in (one thread per send slot; a run
// shared with several neighbours is folded once per slot, same bits)
template <class T>
__global__ void gs_pack_p2p_fused_kernel(int64_t nslots, const int32_t *__restrict__ perm,
                                         const int32_t *__restrict__ offs, const T *__restrict__ v,
                                         T *__restrict__ partial, const int32_t *__restrict__ send_run,
                                         const int32_t *__restrict__ slot_nbr, double *const *peer_recv,
                                         const int64_t *__restrict__ remote_off, const int64_t *__restrict__ send_offs,
                                         const int64_t *__restrict__ remote_half, int nnbr, int me,
                                         uint64_t *const *peer_hflags, uint64_t *epochs, unsigned int *counter,
                                         const int *done, const int4 *__restrict__ pack4)
{
    __shared__ int s_last;
    const uint64_t e = epochs[2] + 1;
    const int64_t par = (int64_t)(e & 1);   // receive half by epoch parity, in units of the NEIGHBOUR's half size
    if (!(done && *(volatile const int *)done)) {
        for (int64_t sidx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sidx < nslots;
             sidx += (int64_t)gridDim.x * blockDim.x) {
            const int run = send_run[sidx];
            T s;
            const int4 c4 = pack4 ? pack4[sidx] : make_int4(-2, -1, -1, -1);
            if (c4.x >= 0) {                     // <= 4 local copies, listed per slot (one dependent level)
                s = v[c4.x];
                if (c4.y >= 0) s += v[c4.y];
                if (c4.z >= 0) s += v[c4.z];
                if (c4.w >= 0) s += v[c4.w];
            } else {
                const int o0 = offs[run], o1 = offs[run + 1];
                s = v[perm[o0]];
                for (int c = o0 + 1; c < o1; ++c) s += v[perm[c]];
            }
            partial[run] = s;
            const int k = slot_nbr[sidx];
            reinterpret_cast<T *>(peer_recv[k])[par * remote_half[k] + remote_off[k] + (sidx - send_offs[k])] = s;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        *counter = 0u;
        epochs[2] = e;
        __threadfence_system();
        for (int k = 0; k < nnbr; ++k) st_release_sys(peer_hflags[k] + me, e);
    }
}

template <class T>
cudaError_t launch_gs_pack_p2p_fused(const int32_t *perm, const int32_t *offs, const T *v, T *partial,
                                     int64_t nslots, const int32_t *send_run, const int32_t *slot_nbr,
                                     double *const *peer_recv, const int64_t *remote_off, const int64_t *send_offs,
                                     const int64_t *remote_half, int nnbr, int me, uint64_t *const *peer_hflags,
                                     uint64_t *epochs, unsigned int *counter, const int *done, cudaStream_t s,
                                     const int4 *pack4)
{
    // latency-bound gathers (slot -> copies -> values with pack4, else slot -> run -> copies -> values)
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((nslots + 127) / 128, 148 * 16));
    gs_pack_p2p_fused_kernel<<<blocks, 128, 0, s>>>(nslots, perm, offs, v, partial, send_run, slot_nbr, peer_recv,
                                                    remote_off, send_offs, remote_half, nnbr, me, peer_hflags, epochs,
                                                    counter, done, pack4);
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
    multiaxpy_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(n, l, a, y, V, c);
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
    axpby_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(n, alpha, x, beta, y, z);
    return cudaGetLastError();
}


// the gather-scatter family for the FP64 path and the FP32 pMG levels (NEXT #3)
#define NEK_GS_INST(T)                                                                                          \
    template cudaError_t launch_gs_classes<T>(const GsClasses &, T *, const int *, cudaStream_t);                \
    template cudaError_t launch_gs_classes_unpack<T>(const GsClasses &, const HaloUnpack &, T *, const int *,   \
                                                     cudaStream_t);                                             \
    template cudaError_t launch_gs_ifc_pack<T>(int64_t, const int32_t *, const int32_t *, const T *, T *, int64_t, \
                                               const int32_t *, T *, const int *, cudaStream_t);                \
    template cudaError_t launch_gs_ifc_unpack<T>(int64_t, const int32_t *, const int32_t *, const int32_t *,    \
                                                 const int32_t *, const T *, const T *, T *, const int *,       \
                                                 cudaStream_t, const uint64_t *, int64_t);                      \
    template cudaError_t launch_copy_mask<T>(int64_t, const uint32_t *, const T *, T *, cudaStream_t);           \
    template cudaError_t launch_gs_pack_p2p_fused<T>(const int32_t *, const int32_t *, const T *, T *, int64_t,  \
                                                     const int32_t *, const int32_t *, double *const *,         \
                                                     const int64_t *, const int64_t *, const int64_t *, int, int, \
                                                     uint64_t *const *, uint64_t *, unsigned int *, const int *, \
                                                     cudaStream_t, const int4 *);
NEK_GS_INST(double)
NEK_GS_INST(float)
#undef NEK_GS_INST

#include "pmg_kernels.cuh"

}  // namespace nekb200
