// ax_tma.cuh -- Ax v1 for N = 7: persistent CTAs, TMA bulk copies of each
// element's u / G / wJ into a 2-stage shared-memory ring (mbarrier
// completion), BK5-style k-slice sum factorisation with the D rows/columns a
// thread needs held in registers and the t-direction D taken from constant
// memory (warp-uniform), and a fused, deterministic <u, w> reduction finished
// by the last CTA.
//
// Work per element: u_r, u_s, u_t by one 8-term contraction per
// point and direction; g = G u_grad (6 factors); w = D^T g in the three
// directions; w = h1 w + h2 wJ u; Dirichlet mask on input and output.
// HBM traffic per local point: u 8 B + G 48 B (+ wJ 8 B) in, w 8 B out.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace nekb200 {
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ double ldg_ef(const double *p, uint64_t policy)
{
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(policy));
    return v;
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// L2-resident PCG vectors (small problems whose vectors fit in the 126 MB L2 next to
// the streamed metric factors): keep = evict_last for the vectors every kernel of the
// iteration touches, evict_normal otherwise.
__device__ __forceinline__ uint64_t policy_keep(bool keep) { return keep ? policy_evict_last() : policy_evict_normal(); }
__device__ __forceinline__ double2 ld2(const double *p, uint64_t pol)
{
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld1(const double *p, uint64_t pol)
{
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld1(const float *p, uint64_t pol)
{
    float v;
    asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st2(double *p, double2 v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st1(double *p, double v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st1(float *p, float v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ int2 ldi2(const int2 *p, uint64_t pol)
{
    int2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int4 ldi4(const int4 *p, uint64_t pol)
{
    int4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ldu(const uint32_t *p, uint64_t pol)
{
    uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

}  // namespace tma

constexpr int AXV1_NQ = 8;
constexpr int AXV1_THREADS = 64;       // one (i, j) column per thread
constexpr int AXV1_CTAS_PER_SM = 3;

template <bool HELM>
struct AxV1Smem {
    static constexpr int P3 = 512;
    static constexpr int PLANES = 7 + (HELM ? 1 : 0);     // u, 6 G factors, (wJ)
    double stage[2][PLANES * P3];
    alignas(16) double sD[64];
    alignas(16) double sa[64], sb[64], sc[64];
    double sred[64];
    uint64_t full[2];
    int last;
};

// Ax v2: each element is shared by KS "k-groups" of 64 threads; group g owns
// the k-slices [g*8/KS, (g+1)*8/KS) of every (i, j) column, so a CTA has 64*KS
// threads (more warps per SM for the same shared-memory staging per element).
template <bool HELM, int KS>
struct AxV2Smem {
    static constexpr int P3 = 512;
    static constexpr int PLANES = 7 + (HELM ? 1 : 0);
    double stage[2][PLANES * P3];          // u | G (6 planes) | wJ
    alignas(16) uint32_t mstage[2][16];    // the element's Dirichlet bits (TMA'd with the stage)
    alignas(16) double sD[64];
    alignas(16) double sa[KS][64];
    alignas(16) double sb[KS][64];
    alignas(16) double sc[KS][64];
    alignas(16) double spart[KS][8][64];   // per-group partial of the transposed t contraction
    double sred[64 * KS];
    uint64_t full[2];
    int last;
};

// Ax v3: no shared-memory staging of the streams.  Each CTA prefetches the
// u / G / wJ / mask blocks of the element PF ahead into L2 with
// cp.async.bulk.prefetch.L2 and its threads then load their k-column of u and,
// one k-slice ahead, their 6 metric factors straight into registers.  Shared
// memory only carries the k-slices exchanged by the r and s contractions.
template <int KS>
struct AxV3Smem {
    alignas(16) double sD[64];
    alignas(16) double sa[KS][64];
    alignas(16) double sb[KS][64];
    alignas(16) double sc[KS][64];
    alignas(16) double spart[KS > 1 ? KS : 1][8][64];
    double sred[64 * KS];
    int last;
};

}  // namespace nekb200
