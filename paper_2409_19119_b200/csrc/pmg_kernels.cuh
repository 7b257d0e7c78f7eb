// pmg_kernels.cuh -- device kernels of the p-multigrid preconditioner (included by kernels.cu).
//
// Transfers between orders (reading P4), per element by sum factorisation with the 1-D
// interpolation matrix J[I][i] = h_i^{N_c}(xi^{N_f}_I) in shared memory:
//   prolong   u_f += (J x J x J) e_c                    (fine points; the coarse field is continuous)
//   restrict  f_c  = (J^T x J^T x J^T)(O_f * r_f)        (owner-copy injection; QQ^T and the mask
//                                                         of the coarse level follow in api)
// Chebyshev iteration (Saad Alg. 12.1; reading P5) as fused pointwise kernels:
//   first     d = (Dinv f) / theta;  x = d;  r = f        (x0 = 0)
//   restart   r = f - w;  d = (Dinv r) / theta;  x += d   (w = A x0)
//   step      r -= w;  d = c1 d + c2 (Dinv r);  x += d    (w = A d)
//   resid     r = f - w
// plus an owner-copy dot with a deterministic last-CTA finish, and the PCG direction update
// p = z + beta p for a general preconditioner.  Every kernel returns at once when *done is set
// (a converged solve inside a replayed graph).
#pragma once

constexpr int XF_THREADS = 128;

// one CTA per element; IN points per direction a, OUT points b; TRANS: J^T (b < a) with owner weights
template <bool TRANS, bool ADD, class T>
__global__ void __launch_bounds__(XF_THREADS)
    xfer_kernel(int64_t E, int a, int b, const T *__restrict__ J, const T *__restrict__ in,
                const uint32_t *__restrict__ obits, T *__restrict__ out, const int *__restrict__ done)
{
    if (done && *(volatile const int *)done) return;
    extern __shared__ __align__(16) unsigned char xs_raw[];
    T *xs = reinterpret_cast<T *>(xs_raw);
    // J as stored: TRANS=false -> [b][a] (rows: output points), TRANS=true -> [a][b] (rows: input points)
    T *sJ = xs;                                   // 256
    T *s0 = xs + 256;                             // a^3
    T *s1 = s0 + a * a * a;                       // a^2 b
    T *s2 = s1 + a * a * b;                       // a b^2
    const int t = threadIdx.x;
    const int a3 = a * a * a, b3 = b * b * b;
    for (int q = t; q < a * b; q += blockDim.x) sJ[q] = J[q];
    for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
        const T *ue = in + e * a3;
        for (int q = t; q < a3; q += blockDim.x) {
            T v = ue[q];
            if (TRANS) {
                const int64_t l = e * a3 + q;
                if (!((__ldg(obits + (l >> 5)) >> (l & 31)) & 1u)) v = T(0);
            }
            s0[q] = v;
        }
        __syncthreads();
        // i direction: s1[k][j][I] = sum_i M[I][i] s0[k][j][i]
        for (int q = t; q < a * a * b; q += blockDim.x) {
            const int I = q % b, kj = q / b;
            T s = 0;
            for (int i = 0; i < a; ++i) s += (TRANS ? sJ[i * b + I] : sJ[I * a + i]) * s0[kj * a + i];
            s1[q] = s;
        }
        __syncthreads();
        // j direction: s2[k][J][I] = sum_j M[J][j] s1[k][j][I]
        for (int q = t; q < a * b * b; q += blockDim.x) {
            const int I = q % b, Jj = (q / b) % b, k = q / (b * b);
            T s = 0;
            for (int j = 0; j < a; ++j) s += (TRANS ? sJ[j * b + Jj] : sJ[Jj * a + j]) * s1[(k * a + j) * b + I];
            s2[q] = s;
        }
        __syncthreads();
        // k direction: out[K][J][I] = sum_k M[K][k] s2[k][J][I]
        T *oe = out + e * b3;
        for (int q = t; q < b3; q += blockDim.x) {
            const int IJ = q % (b * b), K = q / (b * b);
            T s = 0;
            for (int k = 0; k < a; ++k) s += (TRANS ? sJ[k * b + K] : sJ[K * a + k]) * s2[k * b * b + IJ];
            if (ADD) oe[q] += s;
            else oe[q] = s;
        }
        __syncthreads();
    }
}

template <class T>
static void xfer_attr()
{
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(xfer_kernel<true, false, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        cudaFuncSetAttribute(xfer_kernel<false, true, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        attr = true;
    }
}

template <class T>
cudaError_t launch_prolong_add(int64_t E, int Nc, int Nf, const T *J, const T *ec, T *uf, const int *done,
                               cudaStream_t s)
{
    if (E <= 0) return cudaSuccess;
    const int a = Nc + 1, b = Nf + 1;
    const size_t smem = sizeof(T) * (256 + a * a * a + a * a * b + a * b * b);
    xfer_attr<T>();
    const int grid = (int)std::min<int64_t>(E, 16 * device_sms());
    xfer_kernel<false, true, T><<<grid, XF_THREADS, smem, s>>>(E, a, b, J, ec, nullptr, uf, done);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_restrict(int64_t E, int Nf, int Nc, const T *J, const T *rf, const uint32_t *obits, T *fc,
                            const int *done, cudaStream_t s)
{
    if (E <= 0) return cudaSuccess;
    const int a = Nf + 1, b = Nc + 1;
    const size_t smem = sizeof(T) * (256 + a * a * a + a * a * b + a * b * b);
    xfer_attr<T>();
    const int grid = (int)std::min<int64_t>(E, 16 * device_sms());
    xfer_kernel<true, false, T><<<grid, XF_THREADS, smem, s>>>(E, a, b, J, rf, obits, fc, done);
    return cudaGetLastError();
}

// mode 0: first (x0 = 0), 1: restart (w = A x0), 2: step (w = A d), 3: resid r = f - w only
template <class T>
__global__ void __launch_bounds__(256)
    cheb_kernel(int mode, int64_t n, const T *__restrict__ dinv, const T *__restrict__ f,
                const T *__restrict__ w, T theta, T c1, T c2, T *__restrict__ d,
                T *__restrict__ x, T *__restrict__ r, const int *__restrict__ done)
{
    if (done && *(volatile const int *)done) return;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x) {
        if (mode == 0) {
            const T fv = f[l];
            const T dv = dinv[l] * fv / theta;
            d[l] = dv; x[l] = dv; r[l] = fv;
        } else if (mode == 1) {
            const T rv = f[l] - w[l];
            const T dv = dinv[l] * rv / theta;
            r[l] = rv; d[l] = dv; x[l] = x[l] + dv;
        } else if (mode == 2) {
            const T rv = r[l] - w[l];
            const T dv = c1 * d[l] + c2 * (dinv[l] * rv);
            r[l] = rv; d[l] = dv; x[l] = x[l] + dv;
        } else {
            r[l] = f[l] - w[l];
        }
    }
}

template <class T>
cudaError_t launch_cheb(int mode, int64_t n, const T *dinv, const T *f, const T *w, double theta, double c1,
                        double c2, T *d, T *x, T *r, const int *done, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * device_sms()));
    cheb_kernel<T><<<grid, 256, 0, s>>>(mode, n, dinv, f, w, (T)theta, (T)c1, (T)c2, d, x, r, done);
    return cudaGetLastError();
}

// precision conversion (FP32 preconditioner, NEXT #3): out[l] = (To) in[l]
template <class Ti, class To>
__global__ void convert_kernel(int64_t n, const Ti *__restrict__ in, To *__restrict__ out, const int *__restrict__ done)
{
    if (done && *(volatile const int *)done) return;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x)
        out[l] = (To)in[l];
}

template <class Ti, class To>
cudaError_t launch_convert(int64_t n, const Ti *in, To *out, const int *done, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * device_sms()));
    convert_kernel<Ti, To><<<grid, 256, 0, s>>>(n, in, out, done);
    return cudaGetLastError();
}

// metric factors [E][6][P3] (FP64) -> [E][gs] (FP32, per-element stride padded to 16 bytes)
__global__ void geom_to_f32_kernel(int64_t E, int P3, int gs, const double *__restrict__ G, float *__restrict__ Gf)
{
    const int64_t tot = E * (int64_t)gs;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < tot; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = q / gs;
        const int o = (int)(q - e * gs);
        Gf[q] = o < 6 * P3 ? (float)G[e * 6 * (int64_t)P3 + o] : 0.0f;
    }
}

cudaError_t launch_geom_to_f32(int64_t E, int N, const double *G, float *Gf, cudaStream_t s)
{
    const int P3 = (N + 1) * (N + 1) * (N + 1), gs = ax_gstride_f(N);
    const int64_t tot = E * (int64_t)gs;
    if (tot <= 0) return cudaSuccess;
    geom_to_f32_kernel<<<(int)std::min<int64_t>((tot + 255) / 256, 8 * device_sms()), 256, 0, s>>>(E, P3, gs, G, Gf);
    return cudaGetLastError();
}

#define NEK_PMG_INST(T)                                                                                         \
    template cudaError_t launch_prolong_add<T>(int64_t, int, int, const T *, const T *, T *, const int *,        \
                                               cudaStream_t);                                                   \
    template cudaError_t launch_restrict<T>(int64_t, int, int, const T *, const T *, const uint32_t *, T *,      \
                                            const int *, cudaStream_t);                                         \
    template cudaError_t launch_cheb<T>(int, int64_t, const T *, const T *, const T *, double, double, double, T *, \
                                        T *, T *, const int *, cudaStream_t);
NEK_PMG_INST(double)
NEK_PMG_INST(float)
#undef NEK_PMG_INST
template cudaError_t launch_convert<double, float>(int64_t, const double *, float *, const int *, cudaStream_t);
template cudaError_t launch_convert<float, double>(int64_t, const float *, double *, const int *, cudaStream_t);

// dst[0] = sum over owner copies of a[l] b[l] (double-double: per-thread strided sums, block sums,
// CTA (hi, lo) partials folded by the last CTA)
__global__ void __launch_bounds__(256)
    dot_owner_kernel(int64_t n, const uint32_t *__restrict__ obits, const double *__restrict__ a,
                     const double *__restrict__ b, double *__restrict__ part, double *dst, unsigned int *counter,
                     const int *__restrict__ done)
{
    __shared__ double sred[64];
    __shared__ int s_last;
    if (done && *(volatile const int *)done) return;
    double hi = 0.0, lo = 0.0;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x)
        if (bit_of(obits, l)) dd_add_prod(hi, lo, a[l], b[l]);
    block_sum_dd(hi, lo, sred);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = hi; part[2 * blockIdx.x + 1] = lo; }
    last_block_finish(part, gridDim.x, dst, counter, sred, &s_last);
}

cudaError_t launch_dot_owner(int64_t n, const uint32_t *obits, const double *a, const double *b, double *part,
                             int nblk, double *dst, unsigned int *counter, const int *done, cudaStream_t s)
{
    dot_owner_kernel<<<nblk, 256, 0, s>>>(n, obits, a, b, part, dst, counter, done);
    return cudaGetLastError();
}

// beta = rho'/rho (rho' = rank-ordered sum of red_all[RED_RHO]); p = z + beta p; last CTA does the
// bookkeeping of pcg_pupdate_kernel (iteration, history, convergence on ||r||, breakdown)
__global__ void __launch_bounds__(256)
    pcg_pupdate_z_kernel(int64_t n, const double *__restrict__ z, double *__restrict__ p,
                         const double *__restrict__ red_all, int nranks, PcgScalars *sc, double *__restrict__ hist,
                         unsigned int *counter)
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
            p[l] = z[l] + beta * p[l];
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

cudaError_t launch_pcg_pupdate_z(int64_t n, const double *z, double *p, const double *red_all, int nranks,
                                 PcgScalars *sc, double *hist, unsigned int *counter, int nblk, cudaStream_t s)
{
    pcg_pupdate_z_kernel<<<nblk, 256, 0, s>>>(n, z, p, red_all, nranks, sc, hist, counter);
    return cudaGetLastError();
}

// Lanczos / Jacobi-PCG helpers at setup: r -= alpha w; z = Dinv r   and   p = z + beta p
__global__ void lanczos_rz_kernel(int64_t n, double alpha, const double *__restrict__ w, const double *__restrict__ dinv,
                                  double *__restrict__ r, double *__restrict__ z)
{
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n; l += (int64_t)gridDim.x * blockDim.x) {
        const double rv = w ? r[l] - alpha * w[l] : r[l];
        r[l] = rv;
        z[l] = dinv[l] * rv;
    }
}

cudaError_t launch_lanczos_rz(int64_t n, double alpha, const double *w, const double *dinv, double *r, double *z,
                              cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * device_sms()));
    lanczos_rz_kernel<<<grid, 256, 0, s>>>(n, alpha, w, dinv, r, z);
    return cudaGetLastError();
}
