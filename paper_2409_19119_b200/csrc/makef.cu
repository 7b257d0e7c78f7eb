// makef.cu -- dealiased advection (readings M1-M4).
//
// For each element, component c and GLL test node l (reading M1):
//   F_c(l) = - sum_q rho_q J_q phi_l(xi_q) (u . grad u_c)(xi_q)
//          = - [(J^T x J^T x J^T) ( sum_a Ut_a  d_a u_c )](l),   Ut_a = sum_b G_ab u_b   (reading M3)
// on the M^3 Gauss-Legendre lattice (3/2 rule, N = 7 -> M = 12: the paper's "12^3 working set").
// G_ab = rho J d r_a / d x_b at the fine points is computed once by makef_geom_kernel and streamed
// (9 M^3 values per element); the velocity stays in HBM at GLL resolution.
//
// Kernel design (sm_100a, FP64): one element per CTA iteration, persistent CTAs, every tensor
// contraction done by a thread owning a whole line of the current stage (i-lines, j-lines or
// k-columns), the 1-D matrices J (interpolation) and Dq = J D (derivative at the fine points) as
// compile-time constant-bank operands, line buffers padded to an odd stride.  Per element and
// component: value/derivative interpolation in 3 stages (2 / 3 / 3 contractions), the pointwise
// product with the contravariant velocity, and the transposed interpolation back in 3 stages.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "ax_tma.cuh"
#include "nek_ctx.h"

namespace nekb200 {

constexpr int MK_MAXN = 9;
__constant__ double c_Jq[MK_MAXN + 1][16 * 10];   // [N][I * (N+1) + i] = h_i(xi^GL_I), default M of N
__constant__ double c_Dq[MK_MAXN + 1][16 * 10];   // derivative of the interpolant at the GL points
__constant__ double c_wq[MK_MAXN + 1][16];        // GL weights

#ifndef MK_PF_G
#define MK_PF_G 1   // bulk L2 prefetch of the next element's lattice factors
#endif
constexpr int mk_m(int NQ) { return (3 * NQ + 1) / 2; }   // ceil(3 (N+1) / 2)
constexpr int odd(int n) { return n | 1; }

template <int NQ>
struct MK {
    static constexpr int N = NQ - 1, MQ = mk_m(NQ), P3 = NQ * NQ * NQ, M3 = MQ * MQ * MQ;
    static constexpr int PN = odd(NQ), PM = odd(MQ);            // padded i strides
    // buffers (doubles): U3 [3][NQ][NQ][PN]; UT [3][M3] (Ut, then F); A/B [NQ][NQ][PM];
    // AA/AD/BA [NQ][MQ][PM]; F [M3]; back-projection reuses A/B and AA
    static constexpr int SZ_U = NQ * NQ * PN, SZ_A = NQ * NQ * PM, SZ_AA = NQ * MQ * PM;
    static constexpr int SMEM_D = 3 * SZ_U + 3 * M3 + 2 * SZ_A + 3 * SZ_AA + M3;
    static constexpr int NT = 256;
    static constexpr int MINB = (SMEM_D * 8 + 1024) * 2 <= 227 * 1024 ? 2 : 1;   // two CTAs per SM when they fit
};

template <int NQ> __device__ __forceinline__ double Jm(int I, int i) { return c_Jq[NQ - 1][I * NQ + i]; }
template <int NQ> __device__ __forceinline__ double Dm(int I, int i) { return c_Dq[NQ - 1][I * NQ + i]; }

// Work items of a contraction stage: `lines` lines of `outs` outputs each, split into `ch` chunks of
// `w` outputs so that lines * ch covers the CTA (a stage with fewer lines than threads would leave most
// threads waiting at the next barrier).  Each output is the same fixed-order FMA chain whatever the
// split, so the results do not depend on it.
__host__ __device__ constexpr int mk_chunks(int lines, int outs, int nt)
{
    return (nt + lines - 1) / lines < outs ? (nt + lines - 1) / lines : outs;
}
__host__ __device__ constexpr int mk_width(int lines, int outs, int nt)
{
    return (outs + mk_chunks(lines, outs, nt) - 1) / mk_chunks(lines, outs, nt);
}

template <int NQ>
__global__ void __launch_bounds__(MK<NQ>::NT, MK<NQ>::MINB)
    makef_kernel(int64_t E, const double *__restrict__ G9, const double *__restrict__ u0,
                 const double *__restrict__ u1, const double *__restrict__ u2, double *__restrict__ f0,
                 double *__restrict__ f1, double *__restrict__ f2)
{
    using C = MK<NQ>;
    constexpr int MQ = C::MQ, P3 = C::P3, M3 = C::M3, PN = C::PN, PM = C::PM, NT = C::NT;
    constexpr int SZ_U = C::SZ_U, SZ_A = C::SZ_A, SZ_AA = C::SZ_AA;
    extern __shared__ __align__(16) double sm[];
    double *U3 = sm;                       // [3][NQ][NQ][PN]
    double *UT = U3 + 3 * SZ_U;            // [3][M3]  (k, j, i) fine-point order, unpadded
    double *SA = UT + 3 * M3;              // [NQ][NQ][PM]
    double *SB = SA + SZ_A;
    double *AA = SB + SZ_A;                // [NQ][MQ][PM]
    double *AD = AA + SZ_AA;
    double *BA = AD + SZ_AA;
    double *F = BA + SZ_AA;                // [M3]
    const int t = threadIdx.x, nt = blockDim.x;
    // stage shapes (lines, outputs per line) and their splits
    constexpr int L_UI = 3 * NQ * NQ, CH_UI = mk_chunks(L_UI, MQ, NT), W_UI = mk_width(L_UI, MQ, NT);
    constexpr int L_UJ = 3 * NQ * MQ, CH_UJ = mk_chunks(L_UJ, MQ, NT), W_UJ = mk_width(L_UJ, MQ, NT);
    constexpr int L_UK = 3 * MQ * MQ, CH_UK = mk_chunks(L_UK, MQ, NT), W_UK = mk_width(L_UK, MQ, NT);
    constexpr int L_I = NQ * NQ, CH_I = mk_chunks(L_I, MQ, NT), W_I = mk_width(L_I, MQ, NT);
    constexpr int L_J = 2 * NQ * MQ, CH_J = mk_chunks(L_J, MQ, NT), W_J = mk_width(L_J, MQ, NT);
    constexpr int L_K = MQ * MQ, CH_K = mk_chunks(L_K, MQ, NT), W_K = mk_width(L_K, MQ, NT);
    constexpr int L_KT = MQ * MQ, CH_KT = mk_chunks(L_KT, NQ, NT), W_KT = mk_width(L_KT, NQ, NT);
    constexpr int L_JT = NQ * MQ, CH_JT = mk_chunks(L_JT, NQ, NT), W_JT = mk_width(L_JT, NQ, NT);
    constexpr int L_IT = NQ * NQ, CH_IT = mk_chunks(L_IT, NQ, NT), W_IT = mk_width(L_IT, NQ, NT);
    for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
        // the next element's lattice factors into L2 while this one computes (read in the Ut stage)
        if (MK_PF_G && t == 0 && e + gridDim.x < E && (9 * M3 * 8) % 16 == 0)
            tma::prefetch_l2(G9 + (e + gridDim.x) * 9 * (int64_t)M3, 9 * M3 * 8);
        // ---- velocity into shared memory (padded i stride)
        for (int q = t; q < 3 * P3; q += nt) {
            const int c = q / P3, p = q - c * P3, i = p % NQ, kj = p / NQ;
            const double *src = c == 0 ? u0 : c == 1 ? u1 : u2;
            U3[c * SZ_U + kj * PN + i] = src[e * P3 + p];
        }
        __syncthreads();
        // ---- U at the fine points, 3 components together: i-lines, j-lines, k-columns
        for (int it = t; it < L_UI * CH_UI; it += nt) {              // i: [c][k][j] lines
            const int L = it % L_UI, ch = it / L_UI;
            const int c = L / (NQ * NQ), kj = L % (NQ * NQ);
            double x[NQ];
#pragma unroll
            for (int m = 0; m < NQ; ++m) x[m] = U3[c * SZ_U + kj * PN + m];
            double *o = (c == 0 ? SA : c == 1 ? SB : AA) + kj * PM;  // scratch per component
#pragma unroll
            for (int ii = 0; ii < W_UI; ++ii) {
                const int I = ch * W_UI + ii;
                if (I >= MQ) break;
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) s = fma(Jm<NQ>(I, m), x[m], s);
                o[I] = s;
            }
        }
        __syncthreads();
        for (int it = t; it < L_UJ * CH_UJ; it += nt) {              // j: [c][k][I] lines
            const int L = it % L_UJ, ch = it / L_UJ;
            const int c = L / (NQ * MQ), r = L % (NQ * MQ), k = r / MQ, I = r % MQ;
            const double *in = (c == 0 ? SA : c == 1 ? SB : AA);
            double x[NQ];
#pragma unroll
            for (int m = 0; m < NQ; ++m) x[m] = in[(k * NQ + m) * PM + I];
            double *o = (c == 0 ? AD : c == 1 ? BA : F);              // [k][J][I] stride PM (F: own layout)
#pragma unroll
            for (int jj = 0; jj < W_UJ; ++jj) {
                const int J = ch * W_UJ + jj;
                if (J >= MQ) break;
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) s = fma(Jm<NQ>(J, m), x[m], s);
                if (c < 2) o[(k * MQ + J) * PM + I] = s;
                else o[(k * MQ + J) * MQ + I] = s;                     // F holds NQ*MQ*MQ <= M3 values
            }
        }
        __syncthreads();
        for (int it = t; it < L_UK * CH_UK; it += nt) {              // k: [c][J][I] columns -> U
            const int L = it % L_UK, ch = it / L_UK;
            const int c = L / (MQ * MQ), JI = L % (MQ * MQ);
            double x[NQ];
            if (c < 2) {
                const double *in = c == 0 ? AD : BA;
                const int J = JI / MQ, I = JI % MQ;
#pragma unroll
                for (int m = 0; m < NQ; ++m) x[m] = in[(m * MQ + J) * PM + I];
            } else {
#pragma unroll
                for (int m = 0; m < NQ; ++m) x[m] = F[m * MQ * MQ + JI];
            }
#pragma unroll
            for (int kk = 0; kk < W_UK; ++kk) {
                const int K = ch * W_UK + kk;
                if (K >= MQ) break;
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) s = fma(Jm<NQ>(K, m), x[m], s);
                UT[c * M3 + K * MQ * MQ + JI] = s;
            }
        }
        __syncthreads();
        // ---- contravariant velocity Ut_a = sum_b G_ab U_b (G streamed from HBM), in place
        const double *Ge = G9 + e * 9 * (int64_t)M3;
        for (int q = t; q < M3; q += nt) {
            const double ux = UT[q], uy = UT[M3 + q], uz = UT[2 * M3 + q];
            double g[9];
#pragma unroll
            for (int a = 0; a < 9; ++a) g[a] = __ldcs(Ge + a * M3 + q);
            UT[q] = g[0] * ux + g[1] * uy + g[2] * uz;
            UT[M3 + q] = g[3] * ux + g[4] * uy + g[5] * uz;
            UT[2 * M3 + q] = g[6] * ux + g[7] * uy + g[8] * uz;
        }
        __syncthreads();
        // ---- per component: gradient at the fine points, F = Ut . grad u_c, project back
        for (int c = 0; c < 3; ++c) {
            const double *uc = U3 + c * SZ_U;
            for (int it = t; it < L_I * CH_I; it += nt) {            // i: A = J u, B = Dq u
                const int L = it % L_I, ch = it / L_I;
                double x[NQ];
#pragma unroll
                for (int m = 0; m < NQ; ++m) x[m] = uc[L * PN + m];
#pragma unroll
                for (int ii = 0; ii < W_I; ++ii) {
                    const int I = ch * W_I + ii;
                    if (I >= MQ) break;
                    double a = 0.0, b = 0.0;
#pragma unroll
                    for (int m = 0; m < NQ; ++m) { a = fma(Jm<NQ>(I, m), x[m], a); b = fma(Dm<NQ>(I, m), x[m], b); }
                    SA[L * PM + I] = a;
                    SB[L * PM + I] = b;
                }
            }
            __syncthreads();
            for (int it = t; it < L_J * CH_J; it += nt) {            // j: AA, AD from A; BA from B
                const int L = it % L_J, ch = it / L_J;
                const int which = L / (NQ * MQ), r = L % (NQ * MQ), k = r / MQ, I = r % MQ;
                const double *in = which == 0 ? SA : SB;
                double x[NQ];
#pragma unroll
                for (int m = 0; m < NQ; ++m) x[m] = in[(k * NQ + m) * PM + I];
#pragma unroll
                for (int jj = 0; jj < W_J; ++jj) {
                    const int J = ch * W_J + jj;
                    if (J >= MQ) break;
                    if (which == 0) {
                        double a = 0.0, d = 0.0;
#pragma unroll
                        for (int m = 0; m < NQ; ++m) { a = fma(Jm<NQ>(J, m), x[m], a); d = fma(Dm<NQ>(J, m), x[m], d); }
                        AA[(k * MQ + J) * PM + I] = a;
                        AD[(k * MQ + J) * PM + I] = d;
                    } else {
                        double a = 0.0;
#pragma unroll
                        for (int m = 0; m < NQ; ++m) a = fma(Jm<NQ>(J, m), x[m], a);
                        BA[(k * MQ + J) * PM + I] = a;
                    }
                }
            }
            __syncthreads();
            for (int it = t; it < L_K * CH_K; it += nt) {            // k: d_r, d_s, d_t and F
                const int L = it % L_K, ch = it / L_K;
                const int J = L / MQ, I = L % MQ;
                double xa[NQ], xd[NQ], xb[NQ];
#pragma unroll
                for (int m = 0; m < NQ; ++m) {
                    xa[m] = AA[(m * MQ + J) * PM + I];
                    xd[m] = AD[(m * MQ + J) * PM + I];
                    xb[m] = BA[(m * MQ + J) * PM + I];
                }
#pragma unroll
                for (int kk = 0; kk < W_K; ++kk) {
                    const int K = ch * W_K + kk;
                    if (K >= MQ) break;
                    double dr = 0.0, ds = 0.0, dt = 0.0;
#pragma unroll
                    for (int m = 0; m < NQ; ++m) {
                        dr = fma(Jm<NQ>(K, m), xb[m], dr);
                        ds = fma(Jm<NQ>(K, m), xd[m], ds);
                        dt = fma(Dm<NQ>(K, m), xa[m], dt);
                    }
                    const int q = K * MQ * MQ + L;
                    F[q] = UT[q] * dr + UT[M3 + q] * ds + UT[2 * M3 + q] * dt;
                }
            }
            __syncthreads();
            for (int it = t; it < L_KT * CH_KT; it += nt) {          // k^T: P1[k][J][I] into AA
                const int L = it % L_KT, ch = it / L_KT;
                double x[MQ];
#pragma unroll
                for (int K = 0; K < MQ; ++K) x[K] = F[K * MQ * MQ + L];
                const int J = L / MQ, I = L % MQ;
#pragma unroll
                for (int kk = 0; kk < W_KT; ++kk) {
                    const int k = ch * W_KT + kk;
                    if (k >= NQ) break;
                    double s = 0.0;
#pragma unroll
                    for (int K = 0; K < MQ; ++K) s = fma(Jm<NQ>(K, k), x[K], s);
                    AA[(k * MQ + J) * PM + I] = s;
                }
            }
            __syncthreads();
            for (int it = t; it < L_JT * CH_JT; it += nt) {          // j^T: P2[k][j][I] into SA
                const int L = it % L_JT, ch = it / L_JT;
                const int k = L / MQ, I = L % MQ;
                double x[MQ];
#pragma unroll
                for (int J = 0; J < MQ; ++J) x[J] = AA[(k * MQ + J) * PM + I];
#pragma unroll
                for (int jj = 0; jj < W_JT; ++jj) {
                    const int j = ch * W_JT + jj;
                    if (j >= NQ) break;
                    double s = 0.0;
#pragma unroll
                    for (int J = 0; J < MQ; ++J) s = fma(Jm<NQ>(J, j), x[J], s);
                    SA[(k * NQ + j) * PM + I] = s;
                }
            }
            __syncthreads();
            double *fo = (c == 0 ? f0 : c == 1 ? f1 : f2) + e * P3;
            for (int it = t; it < L_IT * CH_IT; it += nt) {          // i^T: out[k][j][i] = -sum_I J[I][i] P2
                const int L = it % L_IT, ch = it / L_IT;
                double x[MQ];
#pragma unroll
                for (int I = 0; I < MQ; ++I) x[I] = SA[L * PM + I];
#pragma unroll
                for (int ii = 0; ii < W_IT; ++ii) {
                    const int i = ch * W_IT + ii;
                    if (i >= NQ) break;
                    double s = 0.0;
#pragma unroll
                    for (int I = 0; I < MQ; ++I) s = fma(Jm<NQ>(I, i), x[I], s);
                    fo[L * NQ + i] = -s;
                }
            }
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------ FP64 tensor cores (N = 7)
// The same stages as makef_kernel with every 1-D contraction done as 8x8x4 FP64 tensor-core products
// (mma.sync.m8n8k4.f64, DMMA): a stage is a small GEMM, rows = the lines of the stage, columns = the
// outputs of a line (12 fine points padded to 16, or 8 GLL nodes), K = the points contracted (8 or 12);
// the 1-D matrices J and Dq = J D sit in registers as B fragments, A fragments come from the shared
// line buffers, and each warp takes 8-row x 8-column tiles.  One DMMA does 256 FMAs for one
// instruction, so the stages are no longer bound by instruction issue and FMA latency.
__device__ __forceinline__ void mk_dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int NQ>
__global__ void __launch_bounds__(MK<NQ>::NT, MK<NQ>::MINB)
    makef_mma_kernel(int64_t E, const double *__restrict__ G9, const double *__restrict__ u0,
                     const double *__restrict__ u1, const double *__restrict__ u2, double *__restrict__ f0,
                     double *__restrict__ f1, double *__restrict__ f2)
{
    static_assert(NQ == 8, "the DMMA tiling is written for N = 7 (8 GLL nodes, 12 fine points)");
    using C = MK<NQ>;
    constexpr int MQ = C::MQ, P3 = C::P3, M3 = C::M3, PN = C::PN, PM = C::PM, NW = C::NT / 32;
    constexpr int SZ_U = C::SZ_U, SZ_A = C::SZ_A, SZ_AA = C::SZ_AA;
    extern __shared__ __align__(16) double sm[];
    double *U3 = sm;
    double *UT = U3 + 3 * SZ_U;
    double *SA = UT + 3 * M3;
    double *SB = SA + SZ_A;
    double *AA = SB + SZ_A;
    double *AD = AA + SZ_AA;
    double *BA = AD + SZ_AA;
    double *F = BA + SZ_AA;
    const int t = threadIdx.x, nt = blockDim.x, warp = t >> 5, lane = t & 31;
    const int ar = lane >> 2, ac = lane & 3;     // A (row ar, col ac), B (row ac, col ar), D (row ar, cols 2ac, 2ac+1)
    // forward B fragments: B(k = m, n = I) = J[I][m] (K = 8 GLL nodes, 2 k-steps; N = 12 -> 2 tiles of 8)
    double BJ[2][2], BDq[2][2];
#pragma unroll
    for (int n2 = 0; n2 < 2; ++n2)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const int I = n2 * 8 + ar, m = ks * 4 + ac;
            BJ[n2][ks] = I < MQ ? Jm<NQ>(I, m) : 0.0;
            BDq[n2][ks] = I < MQ ? Dm<NQ>(I, m) : 0.0;
        }
    // transposed B fragments: B(k = K, n = i) = J[K][i] (K = 12 fine points, 3 k-steps; N = 8)
    double BT[3];
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) BT[ks] = Jm<NQ>(ks * 4 + ac, ar);
    for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
        if (MK_PF_G && t == 0 && e + gridDim.x < E && (9 * M3 * 8) % 16 == 0)
            tma::prefetch_l2(G9 + (e + gridDim.x) * 9 * (int64_t)M3, 9 * M3 * 8);
        for (int q = t; q < 3 * P3; q += nt) {
            const int c = q / P3, p = q - c * P3, i = p % NQ, kj = p / NQ;
            const double *src = c == 0 ? u0 : c == 1 ? u1 : u2;
            U3[c * SZ_U + kj * PN + i] = src[e * P3 + p];
        }
        __syncthreads();
        // ---- U at the fine points, 3 components: i (rows c,k,j; 192), j (rows c,k,I; 288), k (rows c,J,I; 432)
        for (int tile = warp; tile < 24 * 2; tile += NW) {
            const int mt = tile >> 1, n2 = tile & 1;
            const int row = mt * 8 + ar, c = row / 64, kj = row % 64;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) mk_dmma(d0, d1, U3[c * SZ_U + kj * PN + ks * 4 + ac], (n2 ? BJ[1][ks] : BJ[0][ks]));
            const int orow = mt * 8 + ar, oc = orow / 64, okj = orow % 64, I0 = n2 * 8 + 2 * ac;
            double *o = (oc == 0 ? SA : oc == 1 ? SB : AA) + okj * PM;
            if (I0 < MQ) o[I0] = d0;
            if (I0 + 1 < MQ) o[I0 + 1] = d1;
        }
        __syncthreads();
        for (int tile = warp; tile < 36 * 2; tile += NW) {
            const int mt = tile >> 1, n2 = tile & 1;
            const int row = mt * 8 + ar, c = row / (NQ * MQ), r = row % (NQ * MQ), k = r / MQ, I = r % MQ;
            const double *in = (c == 0 ? SA : c == 1 ? SB : AA);
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) mk_dmma(d0, d1, in[(k * NQ + ks * 4 + ac) * PM + I], (n2 ? BJ[1][ks] : BJ[0][ks]));
            const int J0 = n2 * 8 + 2 * ac;
            if (c < 2) {
                double *o = c == 0 ? AD : BA;
                if (J0 < MQ) o[(k * MQ + J0) * PM + I] = d0;
                if (J0 + 1 < MQ) o[(k * MQ + J0 + 1) * PM + I] = d1;
            } else {
                if (J0 < MQ) F[(k * MQ + J0) * MQ + I] = d0;
                if (J0 + 1 < MQ) F[(k * MQ + J0 + 1) * MQ + I] = d1;
            }
        }
        __syncthreads();
        for (int tile = warp; tile < 54 * 2; tile += NW) {
            const int mt = tile >> 1, n2 = tile & 1;
            const int row = mt * 8 + ar, c = row / (MQ * MQ), JI = row % (MQ * MQ), J = JI / MQ, I = JI % MQ;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const int m = ks * 4 + ac;
                const double a = c == 0 ? AD[(m * MQ + J) * PM + I] : c == 1 ? BA[(m * MQ + J) * PM + I]
                                                                            : F[m * MQ * MQ + JI];
                mk_dmma(d0, d1, a, (n2 ? BJ[1][ks] : BJ[0][ks]));
            }
            const int K0 = n2 * 8 + 2 * ac;
            if (K0 < MQ) UT[c * M3 + K0 * MQ * MQ + JI] = d0;
            if (K0 + 1 < MQ) UT[c * M3 + (K0 + 1) * MQ * MQ + JI] = d1;
        }
        __syncthreads();
        // ---- contravariant velocity Ut_a = sum_b G_ab U_b (G streamed from HBM), in place
        const double *Ge = G9 + e * 9 * (int64_t)M3;
        for (int q = t; q < M3; q += nt) {
            const double ux = UT[q], uy = UT[M3 + q], uz = UT[2 * M3 + q];
            double g[9];
#pragma unroll
            for (int a = 0; a < 9; ++a) g[a] = __ldcs(Ge + a * M3 + q);
            UT[q] = g[0] * ux + g[1] * uy + g[2] * uz;
            UT[M3 + q] = g[3] * ux + g[4] * uy + g[5] * uz;
            UT[2 * M3 + q] = g[6] * ux + g[7] * uy + g[8] * uz;
        }
        __syncthreads();
        for (int c = 0; c < 3; ++c) {
            const double *uc = U3 + c * SZ_U;
            for (int tile = warp; tile < 8 * 2; tile += NW) {           // i: A = J u, B = Dq u (rows k,j)
                const int mt = tile >> 1, n2 = tile & 1, L = mt * 8 + ar;
                double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const double x = uc[L * PN + ks * 4 + ac];
                    mk_dmma(a0, a1, x, (n2 ? BJ[1][ks] : BJ[0][ks]));
                    mk_dmma(b0, b1, x, (n2 ? BDq[1][ks] : BDq[0][ks]));
                }
                const int I0 = n2 * 8 + 2 * ac;
                if (I0 < MQ) { SA[L * PM + I0] = a0; SB[L * PM + I0] = b0; }
                if (I0 + 1 < MQ) { SA[L * PM + I0 + 1] = a1; SB[L * PM + I0 + 1] = b1; }
            }
            __syncthreads();
            for (int tile = warp; tile < 24 * 2; tile += NW) {          // j: AA, AD from A; BA from B
                const int mt = tile >> 1, n2 = tile & 1;
                const int row = mt * 8 + ar, which = row / (NQ * MQ), r = row % (NQ * MQ), k = r / MQ, I = r % MQ;
                const double *in = which == 0 ? SA : SB;
                double a0 = 0.0, a1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const double x = in[(k * NQ + ks * 4 + ac) * PM + I];
                    mk_dmma(a0, a1, x, (n2 ? BJ[1][ks] : BJ[0][ks]));
                    if (which == 0) mk_dmma(d0, d1, x, (n2 ? BDq[1][ks] : BDq[0][ks]));
                }
                const int J0 = n2 * 8 + 2 * ac;
                double *oa = which == 0 ? AA : BA;
                if (J0 < MQ) {
                    oa[(k * MQ + J0) * PM + I] = a0;
                    if (which == 0) AD[(k * MQ + J0) * PM + I] = d0;
                }
                if (J0 + 1 < MQ) {
                    oa[(k * MQ + J0 + 1) * PM + I] = a1;
                    if (which == 0) AD[(k * MQ + J0 + 1) * PM + I] = d1;
                }
            }
            __syncthreads();
            for (int tile = warp; tile < 18 * 2; tile += NW) {          // k: d_r, d_s, d_t and F (rows J,I)
                const int mt = tile >> 1, n2 = tile & 1, L = mt * 8 + ar, J = L / MQ, I = L % MQ;
                double r0 = 0.0, r1 = 0.0, s0 = 0.0, s1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const int m = ks * 4 + ac, ix = (m * MQ + J) * PM + I;
                    mk_dmma(r0, r1, BA[ix], (n2 ? BJ[1][ks] : BJ[0][ks]));
                    mk_dmma(s0, s1, AD[ix], (n2 ? BJ[1][ks] : BJ[0][ks]));
                    mk_dmma(q0, q1, AA[ix], (n2 ? BDq[1][ks] : BDq[0][ks]));
                }
                const int K0 = n2 * 8 + 2 * ac;
                if (K0 < MQ) {
                    const int qq = K0 * MQ * MQ + L;
                    F[qq] = UT[qq] * r0 + UT[M3 + qq] * s0 + UT[2 * M3 + qq] * q0;
                }
                if (K0 + 1 < MQ) {
                    const int qq = (K0 + 1) * MQ * MQ + L;
                    F[qq] = UT[qq] * r1 + UT[M3 + qq] * s1 + UT[2 * M3 + qq] * q1;
                }
            }
            __syncthreads();
            for (int tile = warp; tile < 18; tile += NW) {              // k^T: P1[k][J][I] into AA (rows J,I)
                const int L = tile * 8 + ar, J = L / MQ, I = L % MQ;
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 3; ++ks) mk_dmma(d0, d1, F[(ks * 4 + ac) * MQ * MQ + L], BT[ks]);
                const int k0 = 2 * ac;
                AA[(k0 * MQ + J) * PM + I] = d0;
                AA[((k0 + 1) * MQ + J) * PM + I] = d1;
            }
            __syncthreads();
            for (int tile = warp; tile < 12; tile += NW) {              // j^T: P2[k][j][I] into SA (rows k,I)
                const int row = tile * 8 + ar, k = row / MQ, I = row % MQ;
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 3; ++ks) mk_dmma(d0, d1, AA[(k * MQ + ks * 4 + ac) * PM + I], BT[ks]);
                const int j0 = 2 * ac;
                SA[(k * NQ + j0) * PM + I] = d0;
                SA[(k * NQ + j0 + 1) * PM + I] = d1;
            }
            __syncthreads();
            double *fo = (c == 0 ? f0 : c == 1 ? f1 : f2) + e * P3;
            for (int tile = warp; tile < 8; tile += NW) {               // i^T: out[k][j][i] = -sum_I J[I][i] P2
                const int L = tile * 8 + ar;
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 3; ++ks) mk_dmma(d0, d1, SA[L * PM + ks * 4 + ac], BT[ks]);
                const int i0 = 2 * ac;
                fo[L * NQ + i0] = -d0;
                fo[L * NQ + i0 + 1] = -d1;
            }
            __syncthreads();
        }
    }
}

// Variant with the three velocity components merged in every stage (9 barriers per element instead
// of 26, 192..576 lines per stage): one CTA per SM, the whole 12^3 working set of an element (values,
// contravariant velocity and the three integrands) resident in shared memory (226 KB at N = 7).
template <int NQ>
struct MK3 {
    using B = MK<NQ>;
    static constexpr int MQ = B::MQ, M3 = B::M3, SZ_U = B::SZ_U, SZ_A = B::SZ_A, SZ_AA = B::SZ_AA;
    static constexpr int SMEM_D = 3 * SZ_U + 6 * SZ_A + 9 * SZ_AA + 6 * M3;
    static constexpr bool FITS = SMEM_D * 8 <= 227 * 1024;
};

template <int NQ, int NT>
__global__ void __launch_bounds__(NT, 1)
    makef3_kernel(int64_t E, const double *__restrict__ G9, const double *__restrict__ u0,
                  const double *__restrict__ u1, const double *__restrict__ u2, double *__restrict__ f0,
                  double *__restrict__ f1, double *__restrict__ f2)
{
    using C = MK<NQ>;
    constexpr int MQ = C::MQ, P3 = C::P3, M3 = C::M3, PN = C::PN, PM = C::PM;
    constexpr int SZ_U = C::SZ_U, SZ_A = C::SZ_A, SZ_AA = C::SZ_AA;
    extern __shared__ __align__(16) double sm[];
    double *U3 = sm;                       // [3][NQ][NQ][PN]
    double *SA = U3 + 3 * SZ_U;            // [3][NQ][NQ][PM]   A, later P2
    double *SB = SA + 3 * SZ_A;            // [3][NQ][NQ][PM]   B
    double *AA = SB + 3 * SZ_A;            // [3][NQ][MQ][PM]   AA, later P1
    double *AD = AA + 3 * SZ_AA;
    double *BA = AD + 3 * SZ_AA;
    double *UT = BA + 3 * SZ_AA;           // [3][M3]  U, then Ut
    double *F = UT + 3 * M3;               // [3][M3]
    const int t = threadIdx.x;
    for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
        if (MK_PF_G && t == 0 && e + gridDim.x < E && (9 * M3 * 8) % 16 == 0)
            tma::prefetch_l2(G9 + (e + gridDim.x) * 9 * (int64_t)M3, 9 * M3 * 8);
        for (int q = t; q < 3 * P3; q += NT) {
            const int c = q / P3, p = q - c * P3;
            const double *src = c == 0 ? u0 : c == 1 ? u1 : u2;
            U3[c * SZ_U + (p / NQ) * PN + p % NQ] = src[e * P3 + p];
        }
        __syncthreads();
        for (int L = t; L < 3 * NQ * NQ; L += NT) {                  // i: A = J u, B = Dq u
            const int c = L / (NQ * NQ), kj = L % (NQ * NQ);
            double x[NQ];
#pragma unroll
            for (int m = 0; m < NQ; ++m) x[m] = U3[c * SZ_U + kj * PN + m];
            double *oa = SA + c * SZ_A + kj * PM, *ob = SB + c * SZ_A + kj * PM;
#pragma unroll 2
            for (int I = 0; I < MQ; ++I) {
                double a = 0.0, b = 0.0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) { a = fma(Jm<NQ>(I, m), x[m], a); b = fma(Dm<NQ>(I, m), x[m], b); }
                oa[I] = a;
                ob[I] = b;
            }
        }
        __syncthreads();
        for (int L = t; L < 6 * NQ * MQ; L += NT) {                  // j: AA, AD from A; BA from B
            const int cw = L / (NQ * MQ), r = L % (NQ * MQ), k = r / MQ, I = r % MQ;
            const int c = cw >> 1, which = cw & 1;
            const double *in = (which == 0 ? SA : SB) + c * SZ_A;
            double x[NQ];
#pragma unroll
            for (int m = 0; m < NQ; ++m) x[m] = in[(k * NQ + m) * PM + I];
            if (which == 0) {
#pragma unroll 2
                for (int J = 0; J < MQ; ++J) {
                    double a = 0.0, d = 0.0;
#pragma unroll
                    for (int m = 0; m < NQ; ++m) { a = fma(Jm<NQ>(J, m), x[m], a); d = fma(Dm<NQ>(J, m), x[m], d); }
                    AA[c * SZ_AA + (k * MQ + J) * PM + I] = a;
                    AD[c * SZ_AA + (k * MQ + J) * PM + I] = d;
                }
            } else {
#pragma unroll 2
                for (int J = 0; J < MQ; ++J) {
                    double a = 0.0;
#pragma unroll
                    for (int m = 0; m < NQ; ++m) a = fma(Jm<NQ>(J, m), x[m], a);
                    BA[c * SZ_AA + (k * MQ + J) * PM + I] = a;
                }
            }
        }
        __syncthreads();
        for (int L = t; L < 3 * MQ * MQ; L += NT) {                  // k: U = J AA
            const int c = L / (MQ * MQ), JI = L % (MQ * MQ), J = JI / MQ, I = JI % MQ;
            double x[NQ];
#pragma unroll
            for (int m = 0; m < NQ; ++m) x[m] = AA[c * SZ_AA + (m * MQ + J) * PM + I];
#pragma unroll 2
            for (int K = 0; K < MQ; ++K) {
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) s = fma(Jm<NQ>(K, m), x[m], s);
                UT[c * M3 + K * MQ * MQ + JI] = s;
            }
        }
        __syncthreads();
        const double *Ge = G9 + e * 9 * (int64_t)M3;                 // Ut = G U, in place
        for (int q0 = t; q0 < M3; q0 += 4 * NT) {
            double g[4][9];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int q = q0 + h * NT;
                if (q < M3) {
#pragma unroll
                    for (int a = 0; a < 9; ++a) g[h][a] = __ldcs(Ge + a * M3 + q);
                }
            }
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int q = q0 + h * NT;
                if (q < M3) {
                    const double ux = UT[q], uy = UT[M3 + q], uz = UT[2 * M3 + q];
                    UT[q] = g[h][0] * ux + g[h][1] * uy + g[h][2] * uz;
                    UT[M3 + q] = g[h][3] * ux + g[h][4] * uy + g[h][5] * uz;
                    UT[2 * M3 + q] = g[h][6] * ux + g[h][7] * uy + g[h][8] * uz;
                }
            }
        }
        __syncthreads();
        for (int L = t; L < 3 * MQ * MQ; L += NT) {                  // k: d_r, d_s, d_t and F_c
            const int c = L / (MQ * MQ), JI = L % (MQ * MQ), J = JI / MQ, I = JI % MQ;
            double xa[NQ], xd[NQ], xb[NQ];
#pragma unroll
            for (int m = 0; m < NQ; ++m) {
                const int o = c * SZ_AA + (m * MQ + J) * PM + I;
                xa[m] = AA[o]; xd[m] = AD[o]; xb[m] = BA[o];
            }
#pragma unroll 2
            for (int K = 0; K < MQ; ++K) {
                double dr = 0.0, ds = 0.0, dt = 0.0;
#pragma unroll
                for (int m = 0; m < NQ; ++m) {
                    dr = fma(Jm<NQ>(K, m), xb[m], dr);
                    ds = fma(Jm<NQ>(K, m), xd[m], ds);
                    dt = fma(Dm<NQ>(K, m), xa[m], dt);
                }
                const int q = K * MQ * MQ + JI;
                F[c * M3 + q] = UT[q] * dr + UT[M3 + q] * ds + UT[2 * M3 + q] * dt;
            }
        }
        __syncthreads();
        for (int L = t; L < 3 * MQ * MQ; L += NT) {                  // k^T: P1 into AA
            const int c = L / (MQ * MQ), JI = L % (MQ * MQ), J = JI / MQ, I = JI % MQ;
            double x[MQ];
#pragma unroll
            for (int K = 0; K < MQ; ++K) x[K] = F[c * M3 + K * MQ * MQ + JI];
#pragma unroll 2
            for (int k = 0; k < NQ; ++k) {
                double s = 0.0;
#pragma unroll
                for (int K = 0; K < MQ; ++K) s = fma(Jm<NQ>(K, k), x[K], s);
                AA[c * SZ_AA + (k * MQ + J) * PM + I] = s;
            }
        }
        __syncthreads();
        for (int L = t; L < 3 * NQ * MQ; L += NT) {                  // j^T: P2 into SA
            const int c = L / (NQ * MQ), r = L % (NQ * MQ), k = r / MQ, I = r % MQ;
            double x[MQ];
#pragma unroll
            for (int J = 0; J < MQ; ++J) x[J] = AA[c * SZ_AA + (k * MQ + J) * PM + I];
#pragma unroll 2
            for (int j = 0; j < NQ; ++j) {
                double s = 0.0;
#pragma unroll
                for (int J = 0; J < MQ; ++J) s = fma(Jm<NQ>(J, j), x[J], s);
                SA[c * SZ_A + (k * NQ + j) * PM + I] = s;
            }
        }
        __syncthreads();
        for (int L = t; L < 3 * NQ * NQ; L += NT) {                  // i^T: out = -J^T P2
            const int c = L / (NQ * NQ), kj = L % (NQ * NQ);
            double x[MQ];
#pragma unroll
            for (int I = 0; I < MQ; ++I) x[I] = SA[c * SZ_A + kj * PM + I];
            double *fo = (c == 0 ? f0 : c == 1 ? f1 : f2) + e * P3 + kj * NQ;
#pragma unroll 2
            for (int i = 0; i < NQ; ++i) {
                double s = 0.0;
#pragma unroll
                for (int I = 0; I < MQ; ++I) s = fma(Jm<NQ>(I, i), x[I], s);
                fo[i] = -s;
            }
        }
        __syncthreads();
    }
}

// G_ab = rho J d r_a / d x_b at the fine points (setup; reading M1).  One element per CTA
// iteration, the same line-owned sum factorisation as the apply: for each coordinate x_d the three
// reference derivatives at the fine points (stored as Jacobian entries [3d + a] in G9), then per
// point the cofactor inverse, rho J and the 9 factors in place.
template <int NQ>
__global__ void __launch_bounds__(MK<NQ>::NT)
    makef_geom_kernel(int64_t E, const double *__restrict__ xyz, int64_t n, double *__restrict__ G9,
                      unsigned long long *bad)
{
    using C = MK<NQ>;
    constexpr int MQ = C::MQ, P3 = C::P3, M3 = C::M3, PN = C::PN, PM = C::PM;
    constexpr int SZ_U = C::SZ_U, SZ_A = C::SZ_A, SZ_AA = C::SZ_AA;
    extern __shared__ __align__(16) double sm[];
    double *X = sm;                        // [3][NQ][NQ][PN]
    double *SA = X + 3 * SZ_U, *SB = SA + SZ_A, *AA = SB + SZ_A, *AD = AA + SZ_AA, *BA = AD + SZ_AA;
    const int t = threadIdx.x, nt = blockDim.x;
    for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
        double *Ge = G9 + e * 9 * (int64_t)M3;
        for (int q = t; q < 3 * P3; q += nt) {
            const int d = q / P3, p = q - d * P3;
            X[d * SZ_U + (p / NQ) * PN + p % NQ] = xyz[d * n + e * P3 + p];
        }
        __syncthreads();
        for (int d = 0; d < 3; ++d) {
            const double *xd = X + d * SZ_U;
            for (int L = t; L < NQ * NQ; L += nt) {
                double x[NQ];
#pragma unroll
                for (int m = 0; m < NQ; ++m) x[m] = xd[L * PN + m];
#pragma unroll 2
                for (int I = 0; I < MQ; ++I) {
                    double a = 0.0, b = 0.0;
#pragma unroll
                    for (int m = 0; m < NQ; ++m) { a = fma(Jm<NQ>(I, m), x[m], a); b = fma(Dm<NQ>(I, m), x[m], b); }
                    SA[L * PM + I] = a;
                    SB[L * PM + I] = b;
                }
            }
            __syncthreads();
            for (int L = t; L < 2 * NQ * MQ; L += nt) {
                const int which = L / (NQ * MQ), r = L % (NQ * MQ), k = r / MQ, I = r % MQ;
                const double *in = which == 0 ? SA : SB;
                double x[NQ];
#pragma unroll
                for (int m = 0; m < NQ; ++m) x[m] = in[(k * NQ + m) * PM + I];
#pragma unroll 2
                for (int J = 0; J < MQ; ++J) {
                    double a = 0.0, dd = 0.0;
#pragma unroll
                    for (int m = 0; m < NQ; ++m) { a = fma(Jm<NQ>(J, m), x[m], a); dd = fma(Dm<NQ>(J, m), x[m], dd); }
                    if (which == 0) { AA[(k * MQ + J) * PM + I] = a; AD[(k * MQ + J) * PM + I] = dd; }
                    else BA[(k * MQ + J) * PM + I] = a;
                }
            }
            __syncthreads();
            for (int L = t; L < MQ * MQ; L += nt) {
                const int J = L / MQ, I = L % MQ;
                double xa[NQ], xd2[NQ], xb[NQ];
#pragma unroll
                for (int m = 0; m < NQ; ++m) {
                    xa[m] = AA[(m * MQ + J) * PM + I];
                    xd2[m] = AD[(m * MQ + J) * PM + I];
                    xb[m] = BA[(m * MQ + J) * PM + I];
                }
#pragma unroll 2
                for (int K = 0; K < MQ; ++K) {
                    double dr = 0.0, ds = 0.0, dt = 0.0;
#pragma unroll
                    for (int m = 0; m < NQ; ++m) {
                        dr = fma(Jm<NQ>(K, m), xb[m], dr);
                        ds = fma(Jm<NQ>(K, m), xd2[m], ds);
                        dt = fma(Dm<NQ>(K, m), xa[m], dt);
                    }
                    const int q = K * MQ * MQ + L;
                    Ge[(3 * d + 0) * M3 + q] = dr;
                    Ge[(3 * d + 1) * M3 + q] = ds;
                    Ge[(3 * d + 2) * M3 + q] = dt;
                }
            }
            __syncthreads();
        }
        for (int q = t; q < M3; q += nt) {
            const int I = q % MQ, J = (q / MQ) % MQ, K = q / (MQ * MQ);
            double Jd[3][3];                                         // [d][a] = d x_d / d r_a
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int a = 0; a < 3; ++a) Jd[d][a] = Ge[(3 * d + a) * M3 + q];
            const double c00 = Jd[1][1] * Jd[2][2] - Jd[1][2] * Jd[2][1];
            const double c01 = Jd[1][2] * Jd[2][0] - Jd[1][0] * Jd[2][2];
            const double c02 = Jd[1][0] * Jd[2][1] - Jd[1][1] * Jd[2][0];
            const double c10 = Jd[0][2] * Jd[2][1] - Jd[0][1] * Jd[2][2];
            const double c11 = Jd[0][0] * Jd[2][2] - Jd[0][2] * Jd[2][0];
            const double c12 = Jd[0][1] * Jd[2][0] - Jd[0][0] * Jd[2][1];
            const double c20 = Jd[0][1] * Jd[1][2] - Jd[0][2] * Jd[1][1];
            const double c21 = Jd[0][2] * Jd[1][0] - Jd[0][0] * Jd[1][2];
            const double c22 = Jd[0][0] * Jd[1][1] - Jd[0][1] * Jd[1][0];
            const double det = Jd[0][0] * c00 + Jd[0][1] * c01 + Jd[0][2] * c02;
            if (!(det > 0.0)) atomicMin(bad, (unsigned long long)(e * M3 + q));
            // rho J (d r_a / d x_b) = rho cof[b][a]   (inverse = cof^T / J)
            const double rho = c_wq[NQ - 1][I] * c_wq[NQ - 1][J] * c_wq[NQ - 1][K];
            const double cof[3][3] = {{c00, c01, c02}, {c10, c11, c12}, {c20, c21, c22}};
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) Ge[(3 * a + b) * M3 + q] = rho * cof[b][a];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ host side
// Gauss-Legendre nodes/weights by Newton on P_M (Legendre recurrence), Chebyshev initial guesses
static void gauss_legendre(int M, double *x, double *w)
{
    for (int i = 0; i < M; ++i) {
        double z = -std::cos(M_PI * (i + 0.75) / (M + 0.5));
        double dp = 1.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = z;
            for (int k = 2; k <= M; ++k) {
                const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
                p0 = p1; p1 = p2;
            }
            dp = M * (z * p1 - p0) / (z * z - 1.0);
            const double dz = p1 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-16) break;
        }
        x[i] = z;
        w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
}

int makef_lattice(int N) { return (3 * (N + 1) + 1) / 2; }

cudaError_t makef_upload(int N)
{
    const int NQ = N + 1, MQ = makef_lattice(N);
    std::vector<double> xg(NQ), wg(NQ), D(NQ * NQ), xq(MQ), wq(MQ), J(MQ * NQ), Dq(MQ * NQ), lam(NQ);
    gll_rule(N, xg.data(), wg.data());
    deriv_matrix(N, xg.data(), D.data());
    gauss_legendre(MQ, xq.data(), wq.data());
    for (int i = 0; i < NQ; ++i) {
        double p = 1.0;
        for (int k = 0; k < NQ; ++k)
            if (k != i) p *= xg[i] - xg[k];
        lam[i] = 1.0 / p;
    }
    for (int I = 0; I < MQ; ++I) {              // barycentric interpolation GLL -> GL (no shared nodes)
        double den = 0.0;
        for (int i = 0; i < NQ; ++i) den += lam[i] / (xq[I] - xg[i]);
        for (int i = 0; i < NQ; ++i) J[I * NQ + i] = lam[i] / (xq[I] - xg[i]) / den;
    }
    for (int I = 0; I < MQ; ++I)
        for (int i = 0; i < NQ; ++i) {
            double s = 0.0;
            for (int m = 0; m < NQ; ++m) s += J[I * NQ + m] * D[m * NQ + i];
            Dq[I * NQ + i] = s;
        }
    cudaError_t e;
    if ((e = cudaMemcpyToSymbol(c_Jq, J.data(), sizeof(double) * J.size(), sizeof(double) * 160 * N)) != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_Dq, Dq.data(), sizeof(double) * Dq.size(), sizeof(double) * 160 * N)) != cudaSuccess) return e;
    return cudaMemcpyToSymbol(c_wq, wq.data(), sizeof(double) * MQ, sizeof(double) * 16 * N);
}

template <int NQ>
static cudaError_t geom_launch(int64_t E, const double *xyz, double *G9, unsigned long long *bad, cudaStream_t s)
{
    using C = MK<NQ>;
    const size_t smem = sizeof(double) * (3 * C::SZ_U + 2 * C::SZ_A + 3 * C::SZ_AA);
    cudaError_t e = cudaFuncSetAttribute(makef_geom_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<int64_t>(E, 2 * (int64_t)device_sms());
    makef_geom_kernel<NQ><<<grid, C::NT, smem, s>>>(E, xyz, E * C::P3, G9, bad);
    return cudaGetLastError();
}

template <int NQ, int NT>
static cudaError_t apply3_launch(int64_t E, const double *G9, const double *u0, const double *u1, const double *u2,
                                 double *f0, double *f1, double *f2, cudaStream_t s)
{
    const size_t smem = sizeof(double) * MK3<NQ>::SMEM_D;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(makef3_kernel<NQ, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int per_sm = std::max(1, std::min((int)((227 * 1024) / (smem + 1024)), 2048 / NT));
    const int grid = (int)std::min<int64_t>(E, (int64_t)device_sms() * per_sm);
    makef3_kernel<NQ, NT><<<grid, NT, smem, s>>>(E, G9, u0, u1, u2, f0, f1, f2);
    return cudaGetLastError();
}

static int makef_variant()
{
    static int v = -1;
    if (v < 0) {
        // 0: per-component stages, two CTAs per SM (default; N = 7 on the FP64 tensor cores); 1 / 2:
        // components merged in every stage, one CTA per SM with 256 / 384 threads; 3: the FMA stages at
        // N = 7 too
        const char *env = getenv("NEK_MAKEF_VARIANT");
        v = env ? atoi(env) : 0;
    }
    return v;
}

template <int NQ>
static cudaError_t apply_launch(int64_t E, const double *G9, const double *u0, const double *u1, const double *u2,
                                double *f0, double *f1, double *f2, cudaStream_t s)
{
    if constexpr (MK3<NQ>::FITS) {
        const int v = makef_variant();
        if (v == 1) return apply3_launch<NQ, 256>(E, G9, u0, u1, u2, f0, f1, f2, s);
        if (v == 2) return apply3_launch<NQ, 384>(E, G9, u0, u1, u2, f0, f1, f2, s);
    }
    using C = MK<NQ>;
    const size_t smem = sizeof(double) * C::SMEM_D;
    int per_sm = (int)((227 * 1024) / (smem + 1024));
    per_sm = std::max(1, std::min(per_sm, 2048 / C::NT));
    const int grid = (int)std::min<int64_t>(E, (int64_t)device_sms() * per_sm);
    if constexpr (NQ == 8) {
        if (makef_variant() != 3) {   // N = 7: FP64 tensor cores (NEK_MAKEF_VARIANT = 3: the FMA kernel)
            static bool attr_m = false;
            if (!attr_m) {
                cudaError_t e = cudaFuncSetAttribute(makef_mma_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem);
                if (e != cudaSuccess) return e;
                attr_m = true;
            }
            makef_mma_kernel<NQ><<<grid, C::NT, smem, s>>>(E, G9, u0, u1, u2, f0, f1, f2);
            return cudaGetLastError();
        }
    }
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(makef_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    makef_kernel<NQ><<<grid, C::NT, smem, s>>>(E, G9, u0, u1, u2, f0, f1, f2);
    return cudaGetLastError();
}

cudaError_t launch_makef_geom(int N, int64_t E, const double *xyz, double *G9, unsigned long long *bad, cudaStream_t s)
{
    if (E <= 0) return cudaSuccess;
    switch (N + 1) {
#define NEK_CASE(NQ) case NQ: return geom_launch<NQ>(E, xyz, G9, bad, s);
        NEK_CASE(2) NEK_CASE(3) NEK_CASE(4) NEK_CASE(5) NEK_CASE(6) NEK_CASE(7) NEK_CASE(8) NEK_CASE(9) NEK_CASE(10)
#undef NEK_CASE
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_makef(int N, int64_t E, const double *G9, const double *u0, const double *u1, const double *u2,
                         double *f0, double *f1, double *f2, cudaStream_t s)
{
    if (E <= 0) return cudaSuccess;
    switch (N + 1) {
#define NEK_CASE(NQ) case NQ: return apply_launch<NQ>(E, G9, u0, u1, u2, f0, f1, f2, s);
        NEK_CASE(2) NEK_CASE(3) NEK_CASE(4) NEK_CASE(5) NEK_CASE(6) NEK_CASE(7) NEK_CASE(8) NEK_CASE(9) NEK_CASE(10)
#undef NEK_CASE
    }
    return cudaErrorInvalidValue;
}

}  // namespace nekb200

namespace nekb200 {

// FP64 FMA throughput probe (SURVEY 8(d) "FP64 DFMA peak: an unrolled register-only FMA chain"):
// 8 independent chains per thread, 1184 CTAs x 256 threads; the roofline denominator of makef.
__global__ void __launch_bounds__(256) dfma_probe_kernel(int iters, double seed, double *out)
{
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-9 + k;
    const double m = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678) out[0] = s;   // keep the chains alive
}

}  // namespace nekb200

extern "C" int nek_probe_dfma_tflops(int device, double *tflops)
{
    using namespace nekb200;
    if (!tflops) return NEK_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return NEK_ENODEV;
    double *out = nullptr;
    if (cudaMalloc((void **)&out, sizeof(double)) != cudaSuccess) return NEK_ENOMEM;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int grid = 8 * device_sms(), iters = 4096;
    dfma_probe_kernel<<<grid, 256>>>(64, 1.0, out);          // warm-up
    cudaEventRecord(a);
    dfma_probe_kernel<<<grid, 256>>>(iters, 1.0, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a); cudaEventDestroy(b);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess || ms <= 0.f) return NEK_ECUDA;
    *tflops = 2.0 * (double)grid * 256 * iters * 16 * 8 / (ms * 1e-3) / 1e12;
    return NEK_OK;
}
