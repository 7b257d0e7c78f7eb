// gs.cu -- the gather-scatter QQ^T of the hot path ("C0 continuity implies ... unit-depth
// stencils"; reading 7): local runs, the interface partials and the halo pack/unpack of
// the cross-GPU exchange (NCCL-staged and NVLink peer-memory forms).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "dev_common.cuh"
#include "gs_body.cuh"
#include "pack_body.cuh"

namespace nekb200 {

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

template <class T, int PPT>
__global__ void __launch_bounds__(256)
    gs_classes_kernel(int64_t n2, const int2 *__restrict__ p2, int64_t n4, const int4 *__restrict__ p4, int64_t n8,
                      const int4 *__restrict__ p8, int64_t ng, const int32_t *__restrict__ pg,
                      const int32_t *__restrict__ og, T *__restrict__ v, const int *done, int keep, int64_t nv)
{
    gs_classes_body<T, PPT, PPT / 2>((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, threadIdx.x & 31, n2, p2,
                                     n4, p4, n8, p8, ng, pg, og, v, tma::policy_keep(keep), done, nv);
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
    if (wid < cw) {
        gs_classes_body<T, PPT, PPT / 2>(wid, lane, n2, p2, n4, p4, n8, p8, ng, pg, og, v, tma::policy_keep(C_keep), done,
                                         U.nv);
        return;
    }
    const uint64_t e = *(volatile const uint64_t *)(U.epochs + 2);
    bool ok = true;
    if (lane == 0)
        for (int k = 0; k < U.nnbr; ++k) ok &= wait_epoch(U.hflags + U.nbr[k], e, U.err, U.timeout_ns);
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (done && *(volatile const int *)done) return;
    const int64_t r = (wid - cw) * 32 + lane;
    if (r >= U.nifc) return;
    const T *recv = reinterpret_cast<const T *>(U.recv) + (int64_t)(e & 1) * U.half;
    const T *partial = reinterpret_cast<const T *>(U.partial);
    const int c0 = U.coffs[r], c1 = U.coffs[r + 1];
    NEK_CHECK(c0 < c1);
    int src = U.contrib[c0];
    NEK_CHECK(src < U.half);
    T s = src < 0 ? partial[r] : ((volatile const T *)recv)[src];
    for (int c = c0 + 1; c < c1; ++c) {
        src = U.contrib[c];
        NEK_CHECK(src < U.half);
        s += src < 0 ? partial[r] : ((volatile const T *)recv)[src];
    }
    for (int c = U.offs[r]; c < U.offs[r + 1]; ++c) NEK_CHECK(U.perm[c] >= 0 && U.perm[c] < U.nv);
    if (!ok) s = T(__longlong_as_double(0x7ff8000000000000ll));   // a neighbour timed out: NaN, not stale data
    for (int c = U.offs[r]; c < U.offs[r + 1]; ++c) v[U.perm[c]] = s;
}

template <class T>
cudaError_t launch_gs_classes_unpack(const GsClasses &C, const HaloUnpack &U, T *v, const int *done,
                                     cudaStream_t s)
{
    const int64_t cw = gs_class_warps(C, GS_PPT), uw = (U.nifc + 31) / 32;
    const int64_t warps = cw + std::max<int64_t>(uw, 1);   // at least one waiting warp keeps epochs in step
    const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
    gs_classes_unpack_kernel<T, GS_PPT><<<grid, 256, 0, s>>>(C.n2, (const int2 *)C.p2, C.n4, (const int4 *)C.p4, C.n8,
                                                             (const int4 *)C.p8, C.ng, C.pg, C.og, cw, U, v, done, C.keep);
    return cudaGetLastError();
}

// Element-chunk order: CTA c takes the runs of every class whose first copy lies in element chunk c
// (GS_CHUNK elements), so the pairs, quads and octets around the same elements are gathered and
// scattered together and the CTAs of one wave sweep a contiguous window of w -- each sector is read
// and written once while it is in L2, instead of once per class pass over the whole vector.  Same
// runs, same canonical sums: bit-identical to the class-major kernel.  Per thread and round: up to
// CH_PR pairs, CH_QR quads and one octet (one round per chunk for box meshes), then the other runs.
constexpr int GS_CHUNK = 7, CH_PR = 3, CH_QR = 1;

int gs_chunk_elems() { return GS_CHUNK; }
static int gs_chunk_ctas_per_sm()
{
    static int v = [] {
        const char *e = getenv("NEK_GS_CTAS");
        return e ? std::max(1, atoi(e)) : 3;
    }();
    return v;
}

template <class T>
__global__ void __launch_bounds__(256, 3)
    gs_chunk_kernel(int64_t nchunk, const int32_t *__restrict__ coff, const int2 *__restrict__ p2,
                    const int4 *__restrict__ p4, const int4 *__restrict__ p8, const int32_t *__restrict__ pg,
                    const int32_t *__restrict__ og, T *__restrict__ v, const int *done, int keep, int64_t nv)
{
    const uint64_t pol = tma::policy_keep(keep & 1);
    const int t = threadIdx.x;
    const int64_t S = nchunk + 1;
    bool checked = false;
    // persistent CTAs, chunk c = blockIdx.x + j * gridDim.x: the CTAs of one step sweep a contiguous
    // window; the index block of the next chunk is prefetched to L2 while this one is gathered
    for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
        const int32_t a2 = coff[c], b2 = coff[c + 1], a4 = coff[S + c], b4 = coff[S + c + 1];
        const int32_t a8 = coff[2 * S + c], b8 = coff[2 * S + c + 1], ag = coff[3 * S + c], bg = coff[3 * S + c + 1];
        if (c + gridDim.x < nchunk) {
            const int64_t cn = c + gridDim.x;
            const char *q2 = reinterpret_cast<const char *>(p2 + coff[cn]);
            const int64_t n2b = 8 * (int64_t)(coff[cn + 1] - coff[cn]);
            const char *q4 = reinterpret_cast<const char *>(p4 + coff[S + cn]);
            const int64_t n4b = 16 * (int64_t)(coff[S + cn + 1] - coff[S + cn]);
            if (128 * (int64_t)t < n2b) asm volatile("prefetch.global.L2 [%0];" ::"l"(q2 + 128 * t));
            if (t < 64 && 128 * (int64_t)t < n4b) asm volatile("prefetch.global.L2 [%0];" ::"l"(q4 + 128 * t));
        }
        for (int32_t o2 = a2, o4 = a4, o8 = a8; o2 < b2 || o4 < b4 || o8 < b8;
             o2 += 256 * CH_PR, o4 += 256 * CH_QR, o8 += 256) {
            int2 i2[CH_PR];
            int4 i4[CH_QR], i8a, i8b;
            T x2[CH_PR], y2[CH_PR], q[CH_QR][4], e[8];
#pragma unroll
            for (int k = 0; k < CH_PR; ++k) if (o2 + t + 256 * k < b2) i2[k] = tma::ldi2(p2 + o2 + t + 256 * k, pol);
#pragma unroll
            for (int k = 0; k < CH_QR; ++k) if (o4 + t + 256 * k < b4) i4[k] = tma::ldi4(p4 + o4 + t + 256 * k, pol);
            const bool h8 = o8 + t < b8;
            if (h8) { i8a = p8[2 * (o8 + t)]; i8b = p8[2 * (o8 + t) + 1]; }
#pragma unroll
            for (int k = 0; k < CH_PR; ++k)
                if (o2 + t + 256 * k < b2) {
                    NEK_CHECK(i2[k].x >= 0 && i2[k].x < i2[k].y && i2[k].y < nv);
                    x2[k] = tma::ld1(v + i2[k].x, pol); y2[k] = tma::ld1(v + i2[k].y, pol);
                }
#pragma unroll
            for (int k = 0; k < CH_QR; ++k)
                if (o4 + t + 256 * k < b4) {
                    NEK_CHECK(i4[k].x >= 0 && i4[k].x < i4[k].y && i4[k].y < i4[k].z && i4[k].z < i4[k].w &&
                              i4[k].w < nv);
                    q[k][0] = tma::ld1(v + i4[k].x, pol); q[k][1] = tma::ld1(v + i4[k].y, pol);
                    q[k][2] = tma::ld1(v + i4[k].z, pol); q[k][3] = tma::ld1(v + i4[k].w, pol);
                }
            if (h8) {
                NEK_CHECK(i8a.x >= 0 && i8a.x < i8a.y && i8a.y < i8a.z && i8a.z < i8a.w && i8a.w < i8b.x &&
                          i8b.x < i8b.y && i8b.y < i8b.z && i8b.z < i8b.w && i8b.w < nv);
                e[0] = tma::ld1(v + i8a.x, pol); e[1] = tma::ld1(v + i8a.y, pol);
                e[2] = tma::ld1(v + i8a.z, pol); e[3] = tma::ld1(v + i8a.w, pol);
                e[4] = tma::ld1(v + i8b.x, pol); e[5] = tma::ld1(v + i8b.y, pol);
                e[6] = tma::ld1(v + i8b.z, pol); e[7] = tma::ld1(v + i8b.w, pol);
            }
            if (!checked) {   // the flag's latency overlaps the loads above; nothing is stored once it is set
                if (done && *(volatile const int *)done) return;
                checked = true;
            }
#pragma unroll
            for (int k = 0; k < CH_PR; ++k)
                if (o2 + t + 256 * k < b2) {
                    const T s = x2[k] + y2[k];
                    tma::st1(v + i2[k].x, s, pol); tma::st1(v + i2[k].y, s, pol);
                }
#pragma unroll
            for (int k = 0; k < CH_QR; ++k)
                if (o4 + t + 256 * k < b4) {
                    const T s = ((q[k][0] + q[k][1]) + q[k][2]) + q[k][3];
                    tma::st1(v + i4[k].x, s, pol); tma::st1(v + i4[k].y, s, pol);
                    tma::st1(v + i4[k].z, s, pol); tma::st1(v + i4[k].w, s, pol);
                }
            if (h8) {
                const T s = ((((((e[0] + e[1]) + e[2]) + e[3]) + e[4]) + e[5]) + e[6]) + e[7];
                v[i8a.x] = s; v[i8a.y] = s; v[i8a.z] = s; v[i8a.w] = s;
                v[i8b.x] = s; v[i8b.y] = s; v[i8b.z] = s; v[i8b.w] = s;
            }
        }
        if (ag < bg && !checked) {
            if (done && *(volatile const int *)done) return;
            checked = true;
        }
        for (int32_t r = ag + t; r < bg; r += 256) {
            const int o0 = og[r], o1 = og[r + 1];
            NEK_CHECK(o0 < o1 && pg[o0] >= 0 && pg[o1 - 1] < nv);
            T s = tma::ld1(v + pg[o0], pol);
            for (int k = o0 + 1; k < o1; ++k) s += tma::ld1(v + pg[k], pol);
            for (int k = o0; k < o1; ++k) v[pg[k]] = s;
        }
    }
}

template <class T>
cudaError_t launch_gs_classes(const GsClasses &C, T *v, const int *done, cudaStream_t s)
{
    if (C.coff) {
        if (C.nchunk <= 0) return cudaSuccess;
        const int64_t grid = std::min<int64_t>(C.nchunk, gs_chunk_ctas_per_sm() * (int64_t)device_sms());
        gs_chunk_kernel<T><<<(unsigned)grid, 256, 0, s>>>(C.nchunk, C.coff, (const int2 *)C.p2,
                                                             (const int4 *)C.p4, (const int4 *)C.p8, C.pg, C.og, v,
                                                             done, C.keep, C.nv);
        return cudaGetLastError();
    }
    const int64_t warps = gs_class_warps(C, GS_PPT);
    if (warps <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
    gs_classes_kernel<T, GS_PPT><<<grid, 256, 0, s>>>(C.n2, (const int2 *)C.p2, C.n4, (const int4 *)C.p4, C.n8,
                                                      (const int4 *)C.p8, C.ng, C.pg, C.og, v, done, C.keep, C.nv);
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
             sidx += (int64_t)gridDim.x * blockDim.x)
            pack_slot<T>(sidx, perm, offs, v, partial, send_run, slot_nbr, peer_recv, remote_off, send_offs,
                         remote_half, nnbr, par, pack4);
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
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((nslots + 127) / 128, 16 * device_sms()));
    gs_pack_p2p_fused_kernel<<<blocks, 128, 0, s>>>(nslots, perm, offs, v, partial, send_run, slot_nbr, peer_recv,
                                                    remote_off, send_offs, remote_half, nnbr, me, peer_hflags, epochs,
                                                    counter, done, pack4);
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
    template cudaError_t launch_gs_pack_p2p_fused<T>(const int32_t *, const int32_t *, const T *, T *, int64_t,  \
                                                     const int32_t *, const int32_t *, double *const *,         \
                                                     const int64_t *, const int64_t *, const int64_t *, int, int, \
                                                     uint64_t *const *, uint64_t *, unsigned int *, const int *, \
                                                     cudaStream_t, const int4 *);
NEK_GS_INST(double)
NEK_GS_INST(float)
#undef NEK_GS_INST

}  // namespace nekb200
