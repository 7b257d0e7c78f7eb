// gs_body.cuh -- the local gather-scatter of one warp's share of the runs (device code shared by
// the gs kernels of gs.cu and the fused single-rank PCG kernel of ax.cu).
#pragma once

namespace nekb200 {

// Runs grouped by length (2: face, 4: edge, 8: vertex nodes of a box; anything
// else generic), each class kept in canonical first-touch order, copies
// ascending: the sum order of every run is unchanged (bit-exact with the
// oracle) but fixed-length runs need no offsets and load their indices as one
// vector (one dependent load level fewer).
constexpr int GS_PPT = 8;   // pairs per thread (quads: GS_PPT / 2)

// Each warp takes a contiguous block of runs of one class and lane l handles
// runs l, l+32, ... of it, so every warp-wide load touches consecutive runs
// (first-touch order keeps their copies close in memory).
template <class T, int GS_PAIRS_PER_THREAD, int GS_QUADS_PER_THREAD>
__device__ __forceinline__ void gs_classes_body(int64_t wid, int lane, int64_t n2, const int2 *__restrict__ p2,
                                                int64_t n4, const int4 *__restrict__ p4, int64_t n8,
                                                const int4 *__restrict__ p8, int64_t ng,
                                                const int32_t *__restrict__ pg, const int32_t *__restrict__ og,
                                                T *__restrict__ v, uint64_t pol, const int *done = nullptr,
                                                int64_t nv = 0)
{
    // the index and value loads are issued before the (dependent) read of the convergence flag, so
    // the two latencies overlap; nothing is stored once `done` is set
    const int64_t w2 = (n2 + 32 * GS_PAIRS_PER_THREAD - 1) / (32 * GS_PAIRS_PER_THREAD);
    const int64_t w4 = (n4 + 32 * GS_QUADS_PER_THREAD - 1) / (32 * GS_QUADS_PER_THREAD);
    const int64_t w8 = (n8 + 31) / 32;
    if (wid < w2) {
        const int64_t r0 = wid * 32 * GS_PAIRS_PER_THREAD + lane;
        int2 c[GS_PAIRS_PER_THREAD];
        T a[GS_PAIRS_PER_THREAD], b[GS_PAIRS_PER_THREAD];
#pragma unroll
        for (int q = 0; q < GS_PAIRS_PER_THREAD; ++q) if (r0 + 32 * q < n2) c[q] = tma::ldi2(p2 + r0 + 32 * q, pol);
#pragma unroll
        for (int q = 0; q < GS_PAIRS_PER_THREAD; ++q)   // canonical: copies ascending, inside the vector
            if (r0 + 32 * q < n2) NEK_CHECK(c[q].x >= 0 && c[q].x < c[q].y && c[q].y < nv);
#pragma unroll
        for (int q = 0; q < GS_PAIRS_PER_THREAD; ++q)
            if (r0 + 32 * q < n2) { a[q] = tma::ld1(v + c[q].x, pol); b[q] = tma::ld1(v + c[q].y, pol); }
        if (done && *(volatile const int *)done) return;
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
#pragma unroll
        for (int q = 0; q < GS_QUADS_PER_THREAD; ++q)
            if (r0 + 32 * q < n4)
                NEK_CHECK(c[q].x >= 0 && c[q].x < c[q].y && c[q].y < c[q].z && c[q].z < c[q].w && c[q].w < nv);
#pragma unroll
        for (int q = 0; q < GS_QUADS_PER_THREAD; ++q)
            if (r0 + 32 * q < n4) {
                a[q][0] = tma::ld1(v + c[q].x, pol); a[q][1] = tma::ld1(v + c[q].y, pol);
                a[q][2] = tma::ld1(v + c[q].z, pol); a[q][3] = tma::ld1(v + c[q].w, pol);
            }
        if (done && *(volatile const int *)done) return;
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
    if (done && *(volatile const int *)done) return;
    if (wid < w8) {
        const int64_t r = wid * 32 + lane;
        if (r >= n8) return;
        const int4 a = p8[2 * r], b = p8[2 * r + 1];
        NEK_CHECK(a.x >= 0 && a.x < a.y && a.y < a.z && a.z < a.w && a.w < b.x && b.x < b.y && b.y < b.z &&
                  b.z < b.w && b.w < nv);
        const T s = ((((((tma::ld1(v + a.x, pol) + tma::ld1(v + a.y, pol)) + tma::ld1(v + a.z, pol)) +
                        tma::ld1(v + a.w, pol)) + tma::ld1(v + b.x, pol)) + tma::ld1(v + b.y, pol)) +
                     tma::ld1(v + b.z, pol)) + tma::ld1(v + b.w, pol);
        v[a.x] = s; v[a.y] = s; v[a.z] = s; v[a.w] = s;
        v[b.x] = s; v[b.y] = s; v[b.z] = s; v[b.w] = s;
        return;
    }
    wid -= w8;
    const int64_t r = wid * 32 + lane;
    if (r < ng) {
        const int o0 = og[r], o1 = og[r + 1];
        NEK_CHECK(o0 < o1 && pg[o0] >= 0 && pg[o1 - 1] < nv);
        for (int c = o0 + 1; c < o1; ++c) NEK_CHECK(pg[c - 1] < pg[c]);
        T s = tma::ld1(v + pg[o0], pol);
        for (int c = o0 + 1; c < o1; ++c) s += tma::ld1(v + pg[c], pol);
        for (int c = o0; c < o1; ++c) v[pg[c]] = s;
    }
}


__host__ __device__ inline int64_t gs_class_warps_of(const GsClasses &C, int ppt)
{
    const int qpt = ppt > 1 ? ppt / 2 : 1;
    return (C.n2 + 32 * ppt - 1) / (32 * ppt) + (C.n4 + 32 * qpt - 1) / (32 * qpt) + (C.n8 + 31) / 32 +
           (C.ng + 31) / 32;
}

// element-chunk gs (gs.cu gs_chunk_kernel, vec.cu pcg_gs_update_kernel): chunk size and per-round runs
constexpr int GS_CHUNK = 7, CH_PR = 3, CH_QR = 1;

// The runs of element chunk c (all classes), in place on v: the first CH_PR x 256 pairs, CH_QR x 256
// quads and 256 octets per round (one round for a box-mesh chunk), then the runs of other lengths.
// `done` is read once per kernel (checked), after the first loads are in flight.  Returns false when
// the solve is done (nothing stored).
template <class T>
__device__ __forceinline__ bool gs_chunk_runs(int64_t c, int64_t nchunk, const int32_t *__restrict__ coff,
                                              const int2 *__restrict__ p2, const int4 *__restrict__ p4,
                                              const int4 *__restrict__ p8, const int32_t *__restrict__ pg,
                                              const int32_t *__restrict__ og, T *__restrict__ v, const int *done,
                                              bool &checked, uint64_t pol, int64_t nv)
{
    const int t = threadIdx.x;
    const int64_t S = nchunk + 1;
    const int32_t a2 = coff[c], b2 = coff[c + 1], a4 = coff[S + c], b4 = coff[S + c + 1];
    const int32_t a8 = coff[2 * S + c], b8 = coff[2 * S + c + 1], ag = coff[3 * S + c], bg = coff[3 * S + c + 1];
    if (c + gridDim.x < nchunk) {   // the next chunk's index block toward L2 meanwhile
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
            if (done && *(volatile const int *)done) return false;
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
        if (done && *(volatile const int *)done) return false;
        checked = true;
    }
    for (int32_t r = ag + t; r < bg; r += 256) {
        const int o0 = og[r], o1 = og[r + 1];
        NEK_CHECK(o0 < o1 && pg[o0] >= 0 && pg[o1 - 1] < nv);
        T s = tma::ld1(v + pg[o0], pol);
        for (int k = o0 + 1; k < o1; ++k) s += tma::ld1(v + pg[k], pol);
        for (int k = o0; k < o1; ++k) v[pg[k]] = s;
    }
    return true;
}

}  // namespace nekb200
