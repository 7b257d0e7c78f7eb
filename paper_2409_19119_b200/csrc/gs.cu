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
    // persistent CTAs, chunk c = blockIdx.x + j * gridDim.x: the CTAs of one step sweep a contiguous
    // window; the index block of the next chunk is prefetched to L2 while this one is gathered
    const uint64_t pol = tma::policy_keep(keep & 1);
    bool checked = false;
    for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x)
        if (!gs_chunk_runs<T>(c, nchunk, coff, p2, p4, p8, pg, og, v, done, checked, pol, nv)) return;
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
    if (threadIdx.x == 0) {   // release (GPU scope): the CTA's peer stores, ordered by the barrier, before
        fence_acq_rel_gpu();  // the count; the last CTA's system-scope fence below is cumulative over them
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        *counter = 0u;
        epochs[2] = e;
        fence_acq_rel_sys();   // acquire the other CTAs' releases, release everything before the flags
        for (int k = 0; k < nnbr; ++k) st_relaxed_sys(peer_hflags[k] + me, e);
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
