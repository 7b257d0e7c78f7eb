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

}  // namespace nekb200
