// api.cu -- the C ABI (include/nek.h): setup, operator, gather-scatter, PCG.
//
// Orchestration only: every step of the path runs in the kernels of
// kernels.cu (and NCCL for the cross-GPU exchange).  One internal stream
// s_main carries the work of a call (forked from / joined to the caller's
// stream with events); a second stream s_comm carries the NCCL halo so it
// overlaps the Ax of interior elements.  PCG iterations are
// captured once into a CUDA graph and replayed (no host synchronisation
// inside the loop except the periodic convergence poll).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nek.h"
#include "nek_ctx.h"

using namespace nekb200;

static thread_local std::string g_last_error;

static int fail(nek_ctx *ctx, int code, const std::string &msg)
{
    if (ctx) ctx->err = msg;
    g_last_error = msg;
    return code;
}

#define CK(call)                                                                                        \
    do {                                                                                                \
        cudaError_t _e = (call);                                                                        \
        if (_e != cudaSuccess)                                                                          \
            return fail(ctx, _e == cudaErrorMemoryAllocation ? NEK_ENOMEM : NEK_ECUDA,                  \
                        std::string(#call) + ": " + cudaGetErrorString(_e));                            \
    } while (0)
#define NK(call)                                                                                        \
    do {                                                                                                \
        ncclResult_t _r = (call);                                                                       \
        if (_r != ncclSuccess) return fail(ctx, NEK_ENCCL, std::string(#call) + ": " + ncclGetErrorString(_r)); \
    } while (0)

template <class T>
static cudaError_t dalloc(nek_ctx *ctx, T **p, int64_t count)
{
    *p = nullptr;
    if (count <= 0) count = 1;
    cudaError_t e = cudaMalloc((void **)p, sizeof(T) * (size_t)count);
    if (e == cudaSuccess) ctx->device_bytes += sizeof(T) * count;
    return e;
}

template <class T>
static cudaError_t upload(nek_ctx *ctx, T **p, const std::vector<T> &v)
{
    cudaError_t e = dalloc(ctx, p, (int64_t)v.size());
    if (e != cudaSuccess || v.empty()) return e;
    return cudaMemcpy(*p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
}

static bool is_device_ptr(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static std::vector<uint32_t> pack_bits(const std::vector<uint8_t> &v)
{
    std::vector<uint32_t> b((v.size() + 31) / 32 + 1, 0u);
    for (size_t l = 0; l < v.size(); ++l)
        if (v[l]) b[l >> 5] |= 1u << (l & 31);
    return b;
}

// ------------------------------------------------------------ timing pool
namespace {
using nekb200::TimedLaunch;
struct TimerPool {
    std::vector<cudaEvent_t> free_ev;
    std::vector<TimedLaunch> pending;
};
}  // namespace
static TimerPool &pool_of(nek_ctx *ctx)
{
    static thread_local std::vector<std::pair<nek_ctx *, TimerPool>> pools;
    for (auto &p : pools) if (p.first == ctx) return p.second;
    pools.push_back({ctx, TimerPool()});
    return pools.back().second;
}
static cudaEvent_t take_event(nek_ctx *ctx)
{
    TimerPool &P = pool_of(ctx);
    if (!P.free_ev.empty()) { cudaEvent_t e = P.free_ev.back(); P.free_ev.pop_back(); return e; }
    cudaEvent_t e; cudaEventCreate(&e); return e;
}
enum { CLS_AX = 0, CLS_GS = 1, CLS_HALO = 2, CLS_VEC = 3, CLS_AXU = 4 };
struct Scope {
    nek_ctx *ctx; int cls; cudaStream_t s; cudaEvent_t a = nullptr;
    // inside a stream capture the records must be EXTERNAL event nodes (a plain record only
    // becomes a dependency edge of the graph)
    static void rec(nek_ctx *c, cudaEvent_t e, cudaStream_t st)
    {
        if (c->capturing) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
        else cudaEventRecord(e, st);
    }
    Scope(nek_ctx *c, int k, cudaStream_t st = nullptr) : ctx(c), cls(k), s(st ? st : c->s_main) {
        if (ctx->timing) { a = take_event(ctx); rec(ctx, a, s); }
    }
    ~Scope() {
        if (ctx->timing) {
            cudaEvent_t b = take_event(ctx);
            rec(ctx, b, s);
            // inside a stream capture the pair becomes two event-record nodes of the graph; their
            // elapsed time is read after every replay
            if (ctx->capturing) ctx->graph_timers.push_back({cls, a, b});
            else pool_of(ctx).pending.push_back({cls, a, b});
        }
    }
};

static double *cls_slot(nek_ctx *ctx, int cls)
{
    return cls == CLS_AX ? &ctx->stats.ax_ms : cls == CLS_GS ? &ctx->stats.gs_ms
         : cls == CLS_HALO ? &ctx->stats.halo_ms : cls == CLS_AXU ? &ctx->stats.axu_ms : &ctx->stats.vec_ms;
}

// after a replay of a graph captured in timing mode (the caller synchronised the stream)
static void harvest_graph_timers(nek_ctx *ctx)
{
    for (auto &t : ctx->graph_timers) {
        float ms = 0.f;
        cudaError_t e = cudaEventElapsedTime(&ms, t.a, t.b);
        if (e != cudaSuccess) {
            cudaGetLastError();
            ms = 0.f;
            if (getenv("NEK_DEBUG")) fprintf(stderr, "nek: graph timer: %s\n", cudaGetErrorString(e));
        }
        *cls_slot(ctx, t.cls) += ms;
    }
}

static void harvest_timers(nek_ctx *ctx)
{
    TimerPool &P = pool_of(ctx);
    for (auto &t : P.pending) {
        float ms = 0.f;
        cudaEventSynchronize(t.b);
        if (cudaEventElapsedTime(&ms, t.a, t.b) != cudaSuccess) { cudaGetLastError(); ms = 0.f; }
        *cls_slot(ctx, t.cls) += ms;
        P.free_ev.push_back(t.a); P.free_ev.push_back(t.b);
    }
    P.pending.clear();
}

// ------------------------------------------------------------ collectives
// One process per GPU: NCCL at setup and for the staged (NCCL) transport; peer memory (CUDA IPC) for
// the NVLink transport.  Loopback group (P virtual ranks on one GPU, loopback.h): host allgathers
// through the group, stage-serialised device copies, sibling pointers instead of IPC handles.
static int lb_fail(nek_ctx *ctx)
{
    return fail(ctx, NEK_ENCCL, "loopback group barrier failed (a rank stopped or timed out)");
}

// every rank's `bytes` host bytes into all[nranks * bytes] (rank order); synchronous
static int coll_allgather_host(nek_ctx *ctx, const void *mine, size_t bytes, void *all)
{
    if (ctx->nranks == 1) { std::memcpy(all, mine, bytes); return NEK_OK; }
    if (ctx->lb) return ctx->lb->allgather(ctx->rank, mine, bytes, all) ? NEK_OK : lb_fail(ctx);
    const size_t b = std::max<size_t>(bytes, 1);
    unsigned char *d = nullptr;
    CK(cudaMalloc(&d, b * (ctx->nranks + 1)));
    if (bytes) CK(cudaMemcpy(d + b * ctx->nranks, mine, bytes, cudaMemcpyHostToDevice));
    NK(ncclAllGather(d + b * ctx->nranks, d, b, ncclUint8, ctx->nccl, ctx->s_main));
    CK(cudaStreamSynchronize(ctx->s_main));
    for (int q = 0; q < ctx->nranks && bytes; ++q)
        CK(cudaMemcpy(static_cast<char *>(all) + q * bytes, d + q * b, bytes, cudaMemcpyDeviceToHost));
    cudaFree(d);
    return NEK_OK;
}

// loopback only: `strm` waits for the work every other rank issued before this point (each rank
// records an event, the ranks swap events through the group; two events alternate so a fast rank's
// next record never replaces one a slow rank has still to wait on)
static int lb_stage_sync(nek_ctx *ctx, cudaStream_t strm)
{
    if (!ctx->lb || ctx->nranks == 1) return NEK_OK;
    cudaEvent_t mine = ctx->ev_lb[ctx->lb_seq++ & 1];
    CK(cudaEventRecord(mine, strm));
    std::vector<cudaEvent_t> ev(ctx->nranks);
    if (!ctx->lb->allgather(ctx->rank, &mine, sizeof(mine), ev.data())) return lb_fail(ctx);
    for (int q = 0; q < ctx->nranks; ++q)
        if (q != ctx->rank) CK(cudaStreamWaitEvent(strm, ev[q], 0));
    return NEK_OK;
}

// every rank's `bytes` device bytes at `send` into recv[nranks * bytes] (rank order), stream-ordered
static int coll_allgather_dev(nek_ctx *ctx, const void *send, void *recv, size_t bytes, cudaStream_t strm)
{
    if (ctx->nranks == 1) {
        CK(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, strm));
        return NEK_OK;
    }
    if (!ctx->lb) {
        NK(ncclAllGather(send, recv, bytes, ncclUint8, ctx->nccl, strm));
        return NEK_OK;
    }
    std::vector<const void *> src(ctx->nranks);
    if (!ctx->lb->allgather(ctx->rank, &send, sizeof(send), src.data())) return lb_fail(ctx);
    int st;
    if ((st = lb_stage_sync(ctx, strm)) != NEK_OK) return st;   // every sender's producer has run
    for (int q = 0; q < ctx->nranks; ++q)
        CK(cudaMemcpyAsync(static_cast<char *>(recv) + q * bytes, src[q], bytes, cudaMemcpyDeviceToDevice, strm));
    return lb_stage_sync(ctx, strm);   // no rank rewrites its send buffer before every rank has copied it
}

// a peer wait timed out earlier in this context (sticky: the exchange epochs are out of step)
static int check_peer(nek_ctx *ctx)
{
    if (ctx->p2p_err_host && *(volatile int *)ctx->p2p_err_host)
        return fail(ctx, NEK_ENCCL, "peer exchange timed out (a rank stopped participating); rebuild the context");
    return NEK_OK;
}

// ------------------------------------------------------------ building blocks
static int do_ax(nek_ctx *ctx, double h1, double h2, const double *u, double *w, const AxLaunch &L,
                 cudaStream_t strm = nullptr)
{
    if (!strm) strm = ctx->s_main;
    Scope sc(ctx, CLS_AX, strm);
    int nl = 0;
    const int var = L.variant >= 0 ? L.variant : ax_effective_variant(ctx->variant, ctx->N, L.fused, L.keep);
    CK(launch_ax(var, ctx->N, L, u, ctx->G, ctx->wJ, ctx->mbits, h1, h2, w, strm, &nl));
    ctx->stats.ax_launches += L.nelem > 0;
    ctx->stats.launches += nl;
    ctx->stats.ax_elements += L.nelem;
    // algorithmic HBM bytes: u, 6 metric factors, w (+ wJ for Helmholtz),
    // + r, Dinv, x, p in and p, x out when the PCG direction update is fused into the prologue
    const double per_pt = 8.0 * (1 + 6 + 1 + (h2 != 0.0 ? 1 : 0) + (L.fused ? 5 : 0));
    ctx->stats.ax_bytes += per_pt * (double)ctx->P3 * (double)L.nelem;
    return NEK_OK;
}

static P2PMail mail_of(const nek_ctx *ctx)
{
    P2PMail m;
    m.mbox = ctx->mbox; m.peer_mbox = ctx->d_peer_mbox; m.epochs = ctx->epochs; m.err = ctx->p2p_err;
    m.me = ctx->rank; m.nranks = ctx->nranks; m.timeout_ns = ctx->p2p_timeout_ns;
    return m;
}

template <class T> static ncclDataType_t nccl_type();
template <> ncclDataType_t nccl_type<double>() { return ncclDouble; }
template <> ncclDataType_t nccl_type<float>() { return ncclFloat; }

// halo buffers are allocated as doubles; FP32 levels (NEXT #3) use them as floats (same slot counts)
template <class T> static T *as(double *p) { return reinterpret_cast<T *>(p); }

template <class T>
static int halo_start(nek_ctx *ctx, const T *v, const int *done, cudaStream_t strm = nullptr)
{
    if (!strm) strm = ctx->s_main;
    if (ctx->p2p) {   // interface partials written straight into the neighbours' buffers over NVLink
        Scope sc(ctx, CLS_HALO, strm);
        CK(launch_gs_pack_p2p_fused<T>(ctx->ifc_perm, ctx->ifc_offs, v, as<T>(ctx->ifc_partial), ctx->nslots,
                                       ctx->send_run, ctx->d_slot_nbr, ctx->d_peer_recv, ctx->d_remote_off,
                                       ctx->d_send_offs, ctx->d_remote_half, (int)ctx->neighbors.size(), ctx->rank,
                                       ctx->d_peer_hflags, ctx->epochs, ctx->counter + 3, done, strm,
                                       reinterpret_cast<const int4 *>(ctx->pack4)));
        ctx->stats.launches += 1;
        ctx->stats.halo_launches += 1;
        return NEK_OK;
    }
    {
        Scope sc(ctx, CLS_HALO, strm);
        CK(launch_gs_ifc_pack<T>(ctx->nifc, ctx->ifc_perm, ctx->ifc_offs, v, as<T>(ctx->ifc_partial), ctx->nslots,
                                 ctx->send_run, as<T>(ctx->sendbuf), done, strm));
        ctx->stats.launches += (ctx->nifc > 0) + (ctx->nslots > 0);
        ctx->stats.halo_launches += 1;
    }
    if (ctx->lb) {   // staged loopback: the NCCL send/recv pairs become device copies from the neighbours
        int st;
        if ((st = lb_stage_sync(ctx, strm)) != NEK_OK) return st;
        for (size_t k = 0; k < ctx->neighbors.size(); ++k) {
            const size_t cnt = (size_t)(ctx->send_offs[k + 1] - ctx->send_offs[k]);
            if (cnt)
                CK(cudaMemcpyAsync(as<T>(ctx->recvbuf) + ctx->send_offs[k],
                                   reinterpret_cast<const T *>(ctx->lb_halo_src[k]), cnt * sizeof(T),
                                   cudaMemcpyDeviceToDevice, strm));
        }
        if ((st = lb_stage_sync(ctx, strm)) != NEK_OK) return st;
        CK(cudaEventRecord(ctx->ev_join, strm));
        return NEK_OK;
    }
    CK(cudaEventRecord(ctx->ev_fork, strm));
    CK(cudaStreamWaitEvent(ctx->s_comm, ctx->ev_fork, 0));
    NK(ncclGroupStart());
    for (size_t k = 0; k < ctx->neighbors.size(); ++k) {
        size_t cnt = (size_t)(ctx->send_offs[k + 1] - ctx->send_offs[k]);
        NK(ncclSend(as<T>(ctx->sendbuf) + ctx->send_offs[k], cnt, nccl_type<T>(), ctx->neighbors[k], ctx->nccl,
                    ctx->s_comm));
        NK(ncclRecv(as<T>(ctx->recvbuf) + ctx->send_offs[k], cnt, nccl_type<T>(), ctx->neighbors[k], ctx->nccl,
                    ctx->s_comm));
    }
    NK(ncclGroupEnd());
    CK(cudaEventRecord(ctx->ev_join, ctx->s_comm));
    return NEK_OK;
}

template <class T>
static int halo_finish(nek_ctx *ctx, T *v, const int *done)
{
    CK(cudaStreamWaitEvent(ctx->s_main, ctx->ev_join, 0));
    Scope sc(ctx, CLS_HALO);
    CK(launch_gs_ifc_unpack<T>(ctx->nifc, ctx->ifc_perm, ctx->ifc_offs, ctx->coffs, ctx->contrib,
                               as<T>(ctx->ifc_partial), as<T>(ctx->recvbuf), v, done, ctx->s_main));
    ctx->stats.launches += (ctx->nifc > 0);
    return NEK_OK;
}

template <class T>
static int do_gs_local(nek_ctx *ctx, T *v, const int *done)
{
    Scope sc(ctx, CLS_GS);
    CK(launch_gs_classes<T>(ctx->gsc, v, done, ctx->s_main));
    ctx->stats.gs_launches += 1;
    ctx->stats.launches += (ctx->nruns > 0);
    return NEK_OK;
}

// P2P: the local runs and the halo unpack (which waits for the neighbours' data) in one launch
template <class T>
static int gs_local_and_unpack_p2p(nek_ctx *ctx, T *v, const int *done, bool skip_local = false)
{
    int st;
    if ((st = lb_stage_sync(ctx, ctx->s_main)) != NEK_OK) return st;   // loopback: the neighbours' packs ran
    Scope sc(ctx, CLS_GS);
    HaloUnpack U;
    U.nifc = ctx->nifc; U.perm = ctx->ifc_perm; U.offs = ctx->ifc_offs; U.coffs = ctx->coffs;
    U.contrib = ctx->contrib; U.nbr = ctx->d_nbr; U.partial = ctx->ifc_partial; U.recv = ctx->recv2;
    U.half = std::max<int64_t>(ctx->nslots, 1); U.hflags = ctx->hflags; U.epochs = ctx->epochs; U.nnbr = (int)ctx->neighbors.size();
    U.err = ctx->p2p_err; U.timeout_ns = ctx->p2p_timeout_ns; U.nv = ctx->n;
    CK(launch_gs_classes_unpack<T>(skip_local ? GsClasses() : ctx->gsc, U, v, done, ctx->s_main));
    ctx->stats.gs_launches += 1;
    ctx->stats.launches += 1;
    return NEK_OK;
}

// v <- QQ^T v (global)
template <class T>
static int gs_full(nek_ctx *ctx, T *v, const int *done)
{
    int st;
    if (ctx->nranks > 1 && (st = halo_start<T>(ctx, v, done)) != NEK_OK) return st;
    if (ctx->p2p) return gs_local_and_unpack_p2p<T>(ctx, v, done);
    if ((st = do_gs_local<T>(ctx, v, done)) != NEK_OK) return st;
    if (ctx->nranks > 1 && (st = halo_finish<T>(ctx, v, done)) != NEK_OK) return st;
    return NEK_OK;
}

// w = M QQ^T (h1 K_L + h2 B_L) M u.  With dot: this rank's <M u, A_L M u> into
// red_loc[RED_SIGMA] (then allgathered across ranks into red_all).  fused: the
// PCG direction / deferred x update is applied in the Ax prologue (u == vp).
static bool use_fused(const nek_ctx *ctx) { return ax_has_fused(ctx->variant, ctx->N); }

// deferred reductions: one rank, the fused v5 kernel.  The Ax leaves its sigma partials for the update
// (no last-CTA fold) and folds the update's (rho', rr) partials at entry (no last-CTA bookkeeping).
static bool use_defer(const nek_ctx *ctx)
{
    return ctx->defer && ctx->nranks == 1 && ctx->E > 0 && use_fused(ctx) &&
           ax_is_v5(ax_effective_variant(ctx->variant, ctx->N, true, ctx->l2keep), ctx->N);
}

// the same at P > 1 over peer memory: the update pushes this rank's (rho', rr) as before, and the next
// Ax pulls every rank's from the mailbox at entry instead of a separate bookkeeping kernel
static bool use_defer_p2p(const nek_ctx *ctx)
{
    return ctx->defer && ctx->nranks > 1 && ctx->p2p && use_fused(ctx) && ctx->N == 7 &&
           ax_is_v5(ax_effective_variant(ctx->variant, ctx->N, true, ctx->l2keep), ctx->N);
}

static int apply_op(nek_ctx *ctx, double h1, double h2, const double *u, double *w, bool dot, const int *done,
                    bool fused = false)
{
    int st;
    AxLaunch L;
    L.done = done;
    L.keep = ctx->l2keep;
    L.pf_min = ctx->v5_pf_min;
    int var = ax_effective_variant(ctx->variant, ctx->N, fused, ctx->l2keep);   // the kernel do_ax launches
    if (fused) {
        L.fused = true;
        L.p = ctx->vp; L.x = ctx->vx; L.r = ctx->vr; L.dinv = ctx->vdinv; L.sc = ctx->sc;
    }
    L.counter = ctx->counter + 1;
    L.dst = ctx->red_loc + RED_SIGMA;
    if (ctx->nranks == 1) {
        L.nelem = ctx->E;
        if (dot) { L.part = ctx->part; L.fin_total = ax_grid(var, ctx->N, ctx->E); }
        if (dot && fused && use_defer(ctx)) {
            L.fin_total = 0; L.upart = ctx->upart; L.nupd = upd_blocks_deferred(); L.hist = ctx->hist;
            L.defer = DEFER_FOLD | DEFER_BOOK;
        }
        if ((st = do_ax(ctx, h1, h2, u, w, L)) != NEK_OK) return st;
        return do_gs_local(ctx, w, done);
    }
    const int64_t nb = ctx->n_boundary, ni = ctx->E - ctx->n_boundary;
    // concurrent boundary / interior launches of the N = 7 kernel: split one wave of CTAs between them
    // (the boundary CTAs take ~4 elements each) so no interior CTA starts late and the halo pack finds
    // the slots the boundary CTAs free (NEK_BND_SPLIT=0: each launch sized on its own).  Both launches
    // run the v5 configuration the whole partition would get, so the wave is the one they occupy.
    const bool split = ctx->concurrent_bnd && ctx->bnd_split && ctx->N == 7 &&
                       (var == 0 || var == 8 || var == 10 || var == 12) && nb > 0 && ni > 0;
    if (split) {
        var = ax_concrete_variant(var, ctx->N, ctx->E);
        L.variant = var;
    }
    int64_t g1 = ax_grid(var, ctx->N, nb), g2 = ax_grid(var, ctx->N, ni);
    if (split) {
        const int64_t wave = ax_grid(var, ctx->N, ctx->E);
        if (ctx->bnd_epc > 0) {   // NEK_BND_EPC: boundary elements per boundary CTA
            const int64_t epc = ctx->bnd_epc;
            g1 = std::min<int64_t>(nb, std::max<int64_t>(1, std::min<int64_t>((nb + epc - 1) / epc, wave / 4)));
        } else {
            // the split that finishes first: the interior launch takes ceil(ni / g2) element rounds, the
            // halo is ready after ceil(nb / g1) rounds plus the pack (~1.7 rounds, measured); the gs waits
            // for both.  Ties: the larger boundary share (the halo earlier).
            double best = 1e30;
            for (int64_t c1 = 1; c1 < wave && c1 <= nb; ++c1) {
                const int64_t c2 = wave - c1;
                const double T = std::max<double>((double)((ni + c2 - 1) / c2), (double)((nb + c1 - 1) / c1) + 1.7);
                if (T <= best) { best = T; g1 = c1; }
            }
        }
        g2 = std::min<int64_t>(ni, std::max<int64_t>(1, wave - g1));
    }
    const bool push = fused && dot && ctx->p2p;   // the finalising CTA sends sigma to every rank itself
    L.elist = ctx->elist;
    // deferred bookkeeping (P2P): every CTA of both launches pulls (rho', rr); the first launch that has
    // elements records the iteration
    const int dbase = (fused && dot && use_defer_p2p(ctx)) ? DEFER_MAIL : 0;
    if (dbase) { L.mail = mail_of(ctx); L.hist = ctx->hist; }
    auto set_defer = [&](bool first) { L.defer = dbase ? (dbase | (first ? DEFER_BOOK : 0)) : 0; };
    const bool book_bnd = nb > 0;
    {
    Scope span(ctx, CLS_AXU);   // the whole Ax phase (both launches and the send), for the union time
    ctx->stats.axu_spans += 1;
    if (ax_has_fused(ctx->variant, ctx->N) && ctx->p2p && !ctx->concurrent_bnd) {
        // Boundary elements, then the halo send, then the interior elements, in stream order: the
        // NVLink transfer overlaps the interior work and the send never waits for SM
        // slots held by the persistent interior grid; the last CTA of either launch finalises sigma.
        if (dot) { L.part = ctx->part; L.fin_total = g1 + g2; L.ctas_total = (unsigned)(g1 + g2); }
        if (push) L.mail = mail_of(ctx);
        L.nelem = nb; L.eoff = 0; L.part_off = 0;
        set_defer(book_bnd);
        if ((st = do_ax(ctx, h1, h2, u, w, L)) != NEK_OK) return st;
        if ((st = halo_start(ctx, w, done)) != NEK_OK) return st;
        L.nelem = ni; L.eoff = nb; L.part_off = g1;
        set_defer(!book_bnd);
        if ((st = do_ax(ctx, h1, h2, u, w, L)) != NEK_OK) return st;
    } else if (ax_has_fused(ctx->variant, ctx->N)) {
        // Boundary elements and the halo send on the high-priority stream, interior elements on
        // the main stream, concurrently; the last CTA of either launch finalises sigma.
        CK(cudaEventRecord(ctx->ev_fork2, ctx->s_main));
        CK(cudaStreamWaitEvent(ctx->s_hi, ctx->ev_fork2, 0));
        if (dot) { L.part = ctx->part; L.fin_total = g1 + g2; L.ctas_total = (unsigned)(g1 + g2); }
        if (push) L.mail = mail_of(ctx);
        L.nelem = nb; L.eoff = 0; L.part_off = 0;
        if (split) L.grid = g1;
        set_defer(book_bnd);
        if ((st = do_ax(ctx, h1, h2, u, w, L, ctx->s_hi)) != NEK_OK) return st;
        if ((st = halo_start(ctx, w, done, ctx->s_hi)) != NEK_OK) return st;
        CK(cudaEventRecord(ctx->ev_bnd, ctx->s_hi));
        L.nelem = ni; L.eoff = nb; L.part_off = g1;
        if (split) L.grid = g2;
        set_defer(!book_bnd);
        if ((st = do_ax(ctx, h1, h2, u, w, L)) != NEK_OK) return st;
        CK(cudaStreamWaitEvent(ctx->s_main, ctx->ev_bnd, 0));
    } else {
        L.nelem = nb;
        if (dot) { L.part = ctx->part; L.part_off = 0; L.fin_total = ni > 0 ? 0 : g1; }
        if (push && ni == 0) L.mail = mail_of(ctx);
        set_defer(book_bnd);
        if ((st = do_ax(ctx, h1, h2, u, w, L)) != NEK_OK) return st;
        if ((st = halo_start(ctx, w, done)) != NEK_OK) return st;
        if (ni > 0) {
            L.nelem = ni;
            L.eoff = nb;
            if (dot) { L.part_off = g1; L.fin_total = g1 + g2; }
            if (push) L.mail = mail_of(ctx);
            set_defer(!book_bnd);
            if ((st = do_ax(ctx, h1, h2, u, w, L)) != NEK_OK) return st;
        }
    }
    }
    if (ctx->p2p) return gs_local_and_unpack_p2p(ctx, w, done);
    if ((st = do_gs_local(ctx, w, done)) != NEK_OK) return st;
    return halo_finish(ctx, w, done);
}

// share this rank's reduction slots with every rank (rank-ordered; red_all == red_loc at one rank).
// channel: 0 = after Ax (sigma), 1 = after the residual update (rho', rr)
static int exchange_slots(nek_ctx *ctx, int channel)
{
    if (ctx->nranks == 1) return NEK_OK;
    if (ctx->p2p) {
        const P2PMail m = mail_of(ctx);
        if (ctx->lb) {   // loopback: every rank's push before any rank's pull
            int st;
            CK(launch_red_exchange(channel, m, ctx->red_loc, ctx->red_all, 1, ctx->s_main));
            if ((st = lb_stage_sync(ctx, ctx->s_main)) != NEK_OK) return st;
            CK(launch_red_exchange(channel, m, ctx->red_loc, ctx->red_all, 2, ctx->s_main));
            ctx->stats.launches += 2;
            return NEK_OK;
        }
        CK(launch_red_exchange(channel, m, ctx->red_loc, ctx->red_all, 3, ctx->s_main));
        ctx->stats.launches += 1;
        return NEK_OK;
    }
    return coll_allgather_dev(ctx, ctx->red_loc, ctx->red_all, sizeof(double) * RED_N, ctx->s_main);
}

// The persisting-L2 carve-out of an L2-resident solve, raised on entry and restored when the solve
// returns (after its final stream synchronisation).  It is a device-wide limit (include/nek.h).
struct L2SetAside {
    size_t prev = 0;
    bool on = false;
    explicit L2SetAside(nek_ctx *ctx)
    {
        if (!ctx->l2keep || ctx->l2_setaside <= 0) return;
        if (cudaDeviceGetLimit(&prev, cudaLimitPersistingL2CacheSize) != cudaSuccess) { cudaGetLastError(); return; }
        if ((size_t)ctx->l2_setaside <= prev) return;
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)ctx->l2_setaside) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        on = true;
    }
    ~L2SetAside()
    {
        if (on && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prev) != cudaSuccess) cudaGetLastError();
    }
};

// Single-GPU nek_ax / nek_gs run straight on the caller's stream (no event hand-off to s_main
// and back, which costs a few microseconds per call); restored on scope exit.
struct OnCallerStream {
    nek_ctx *ctx;
    cudaStream_t saved;
    bool on;
    OnCallerStream(nek_ctx *c, void *stream) : ctx(c), saved(c->s_main), on(c->nranks == 1 && !c->timing)
    {
        if (on) ctx->s_main = (cudaStream_t)stream;
    }
    ~OnCallerStream()
    {
        if (on) ctx->s_main = saved;
    }
};

static void enter(nek_ctx *ctx, void *stream)
{
    cudaEventRecord(ctx->ev_in, (cudaStream_t)stream);
    cudaStreamWaitEvent(ctx->s_main, ctx->ev_in, 0);
}
static void leave(nek_ctx *ctx, void *stream)
{
    cudaEventRecord(ctx->ev_out, ctx->s_main);
    cudaStreamWaitEvent((cudaStream_t)stream, ctx->ev_out, 0);
}

static int ensure_stage(nek_ctx *ctx)
{
    if (!ctx->stage_in) CK(dalloc(ctx, &ctx->stage_in, ctx->n));
    if (!ctx->stage_out) CK(dalloc(ctx, &ctx->stage_out, ctx->n));
    return NEK_OK;
}

static int ensure_dinv(nek_ctx *ctx, double h1, double h2)
{
    if (ctx->dinv_valid && ctx->dinv_h1 == h1 && ctx->dinv_h2 == h2) return NEK_OK;
    CK(launch_diag(ctx->N, ctx->E, ctx->G, ctx->wJ, h1, h2, ctx->vtmp, ctx->s_main));
    int st = gs_full(ctx, ctx->vtmp, nullptr);
    if (st != NEK_OK) return st;
    CK(launch_dinv(ctx->n, ctx->mbits, ctx->vtmp, ctx->vdinv, ctx->s_main));
    ctx->stats.launches += 2;
    ctx->dinv_valid = true; ctx->dinv_h1 = h1; ctx->dinv_h2 = h2;
    if (ctx->graph && (ctx->graph_h1 != h1 || ctx->graph_h2 != h2)) {
        cudaGraphExecDestroy(ctx->graph);
        ctx->graph = nullptr;
    }
    return NEK_OK;
}

// Peer mappings of the mailbox, the halo receive buffer and the halo flags.  Each rank publishes one
// record -- CUDA IPC handles (one process per GPU) or raw device pointers (loopback group) of those
// buffers and of its staged send buffer, where each rank's data lands in its receive buffer, and its
// receive-buffer half size -- then opens its peers' allocations.  Any IPC failure leaves ctx->p2p
// false on every rank (the NCCL transport stays in use).
struct PeerRec {
    cudaIpcMemHandle_t h[3];
    void *raw[4];   // mbox, recv2, hflags, sendbuf (loopback)
    int64_t half;
};

static int setup_p2p(nek_ctx *ctx, bool want_p2p)
{
    const int P = ctx->nranks, me = ctx->rank;
    const int nn = (int)ctx->neighbors.size();
    CK(cudaHostAlloc((void **)&ctx->p2p_err_host, sizeof(int), cudaHostAllocMapped));
    *ctx->p2p_err_host = 0;
    CK(cudaHostGetDevicePointer((void **)&ctx->p2p_err, ctx->p2p_err_host, 0));
    if (const char *e = getenv("NEK_P2P_TIMEOUT_MS")) ctx->p2p_timeout_ns = (uint64_t)std::max(1.0, atof(e)) * 1000000ull;
    if (want_p2p) {
        CK(dalloc(ctx, &ctx->mbox, (int64_t)2 * 2 * P * 4));
        CK(cudaMemset(ctx->mbox, 0, sizeof(double) * 2 * 2 * P * 4));
        CK(dalloc(ctx, &ctx->hflags, P));
        CK(cudaMemset(ctx->hflags, 0, sizeof(uint64_t) * P));
        CK(dalloc(ctx, &ctx->recv2, 2 * std::max<int64_t>(ctx->nslots, 1)));
        CK(dalloc(ctx, &ctx->epochs, 4));
        CK(cudaMemset(ctx->epochs, 0, sizeof(uint64_t) * 4));
    }
    // record: PeerRec, then the offsets of every rank's data in MY receive buffer (-1: not a neighbour)
    const size_t rec_bytes = sizeof(PeerRec) + sizeof(int64_t) * P;
    std::vector<unsigned char> mine(rec_bytes, 0), all(rec_bytes * P, 0);
    PeerRec R;
    std::memset(&R, 0, sizeof(R));
    R.raw[0] = ctx->mbox; R.raw[1] = ctx->recv2; R.raw[2] = ctx->hflags; R.raw[3] = ctx->sendbuf;
    R.half = std::max<int64_t>(ctx->nslots, 1);
    bool ok = true;
    if (want_p2p && !ctx->lb &&
        (cudaIpcGetMemHandle(&R.h[0], ctx->mbox) != cudaSuccess || cudaIpcGetMemHandle(&R.h[1], ctx->recv2) != cudaSuccess ||
         cudaIpcGetMemHandle(&R.h[2], ctx->hflags) != cudaSuccess)) {
        cudaGetLastError();
        ok = false;   // no IPC: stay on NCCL (every rank must agree, below)
    }
    std::memcpy(mine.data(), &R, sizeof(R));
    std::vector<int64_t> offs(P, -1);   // where neighbour q's data lands in MY receive buffer
    for (int k = 0; k < nn; ++k) offs[ctx->neighbors[k]] = ctx->send_offs[k];
    std::memcpy(mine.data() + sizeof(R), offs.data(), sizeof(int64_t) * P);
    int st;
    if ((st = coll_allgather_host(ctx, mine.data(), rec_bytes, all.data())) != NEK_OK) return st;
    auto rec = [&](int q) { PeerRec r; std::memcpy(&r, all.data() + rec_bytes * q, sizeof(r)); return r; };
    auto off_of = [&](int q, int p) {
        int64_t o;
        std::memcpy(&o, all.data() + rec_bytes * q + sizeof(PeerRec) + sizeof(int64_t) * p, sizeof(o));
        return o;
    };
    if (!want_p2p) {   // staged loopback: where each neighbour keeps the slots it sends to this rank
        ctx->lb_halo_src.assign(nn, nullptr);
        for (int k = 0; k < nn; ++k) {
            const int q = ctx->neighbors[k];
            ctx->lb_halo_src[k] = static_cast<const double *>(rec(q).raw[3]) + off_of(q, me);
        }
        return NEK_OK;
    }
    std::vector<double *> pm(P, nullptr), pr(P, nullptr);
    std::vector<uint64_t *> pf(P, nullptr);
    for (int q = 0; q < P && ok; ++q) {
        if (q == me) { pm[q] = ctx->mbox; continue; }
        const PeerRec r = rec(q);
        const bool nbr = std::find(ctx->neighbors.begin(), ctx->neighbors.end(), q) != ctx->neighbors.end();
        if (ctx->lb) {   // same process, same device: the sibling's pointers as they are
            pm[q] = (double *)r.raw[0];
            if (nbr) { pr[q] = (double *)r.raw[1]; pf[q] = (uint64_t *)r.raw[2]; }
            continue;
        }
        void *p = nullptr;
        if (cudaIpcOpenMemHandle(&p, r.h[0], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) { ok = false; break; }
        ctx->ipc_opened.push_back(p); pm[q] = (double *)p;
        if (!nbr) continue;
        if (cudaIpcOpenMemHandle(&p, r.h[1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) { ok = false; break; }
        ctx->ipc_opened.push_back(p); pr[q] = (double *)p;
        if (cudaIpcOpenMemHandle(&p, r.h[2], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) { ok = false; break; }
        ctx->ipc_opened.push_back(p); pf[q] = (uint64_t *)p;
    }
    // every rank must agree on the transport
    int okv = ok ? 1 : 0;
    std::vector<int> oks(P);
    if ((st = coll_allgather_host(ctx, &okv, sizeof(int), oks.data())) != NEK_OK) return st;
    for (int q = 0; q < P; ++q) okv &= oks[q];
    if (!okv) {
        cudaGetLastError();
        for (void *p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
        ctx->ipc_opened.clear();
        return NEK_OK;
    }
    // device-side tables
    std::vector<double *> nrecv(nn);
    std::vector<uint64_t *> nflag(nn);
    std::vector<int64_t> roff(nn), rhalf(nn);
    for (int k = 0; k < nn; ++k) {
        const int q = ctx->neighbors[k];
        nrecv[k] = pr[q];
        nflag[k] = pf[q];
        roff[k] = off_of(q, me);
        rhalf[k] = rec(q).half;   // the neighbour's half size, not ours
    }
    std::vector<int32_t> slot_nbr(ctx->nslots), nbr32(ctx->neighbors.begin(), ctx->neighbors.end());
    for (int k = 0; k < nn; ++k)
        for (int64_t s = ctx->send_offs[k]; s < ctx->send_offs[k + 1]; ++s) slot_nbr[s] = k;
    CK(upload(ctx, &ctx->d_peer_mbox, pm));
    CK(upload(ctx, &ctx->d_peer_recv, nrecv));
    CK(upload(ctx, &ctx->d_peer_hflags, nflag));
    CK(upload(ctx, &ctx->d_remote_off, roff));
    CK(upload(ctx, &ctx->d_remote_half, rhalf));
    CK(upload(ctx, &ctx->d_send_offs, ctx->send_offs));
    CK(upload(ctx, &ctx->d_slot_nbr, slot_nbr));
    CK(upload(ctx, &ctx->d_nbr, nbr32));
    ctx->p2p = true;
    return NEK_OK;
}

// ------------------------------------------------------------------- ABI
extern "C" {

int nek_version(void) { return NEK_ABI_VERSION; }
const char *nek_last_error(void) { return g_last_error.c_str(); }
const char *nek_errmsg(const nek_ctx *ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

int nek_comm_unique_id(unsigned char id[128])
{
    nek_ctx *ctx = nullptr;
    if (!id) return fail(ctx, NEK_EINVAL, "null id");
    ncclUniqueId u;
    NK(ncclGetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
    return NEK_OK;
}

// parent != NULL: an internal pMG level context on the parent's streams and NCCL communicator
static int setup_impl(nek_ctx *ctx, int64_t E, int N, const double *xyz, const int64_t *gid,
                      const uint8_t *dirichlet, const nek_comm *comm, void *stream, nek_ctx *parent = nullptr)
{
    if (N < 1 || N > 15) return fail(ctx, NEK_EORDER, "order N=" + std::to_string(N) + " outside [1,15]");
    if (E < 0 || (E > 0 && (!xyz || !gid))) return fail(ctx, NEK_EINVAL, "E < 0 or null xyz/gid");
    if (comm && comm->nranks > 1 && (comm->rank < 0 || comm->rank >= comm->nranks))
        return fail(ctx, NEK_EINVAL, "bad rank");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { cudaGetLastError(); return fail(ctx, NEK_ENODEV, "no CUDA device"); }
    if (ctx->device < 0 || ctx->device >= ndev) return fail(ctx, NEK_EINVAL, "bad device ordinal");
    CK(cudaSetDevice(ctx->device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, ctx->device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(ctx, NEK_ENODEV, std::string("library built for sm_100a only; device is ") + prop.name);

    ctx->E = E; ctx->N = N; ctx->Nq = N + 1; ctx->P3 = ctx->Nq * ctx->Nq * ctx->Nq; ctx->n = E * ctx->P3;
    ctx->rank = comm && comm->nranks > 1 ? comm->rank : 0;
    ctx->nranks = comm && comm->nranks > 1 ? comm->nranks : 1;
    if (ctx->nranks > 1 && !parent) {
        ctx->lb = loop_group_of(comm->nccl_id);
        if (ctx->lb && ctx->lb->nranks != ctx->nranks) return fail(ctx, NEK_EINVAL, "loopback group size != nranks");
    }
    if (parent) { ctx->rank = parent->rank; ctx->nranks = parent->nranks; ctx->lb = parent->lb; }

    // host planning (local maps + validation)
    nek_plan *p = nullptr;
    int st = nek_plan_create(&p, E, N, gid, dirichlet, xyz);
    ctx->plan = p;
    if (st != NEK_OK) return fail(ctx, st, p ? p->err : "plan allocation failed");

    if (parent) {
        ctx->s_main = parent->s_main; ctx->s_comm = parent->s_comm; ctx->s_hi = parent->s_hi;
        ctx->owns_streams = false;
    } else {
        CK(cudaStreamCreateWithFlags(&ctx->s_main, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->s_comm, cudaStreamNonBlocking));
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&ctx->s_hi, cudaStreamNonBlocking, hi));
    }
    for (cudaEvent_t *e : {&ctx->ev_in, &ctx->ev_out, &ctx->ev_fork, &ctx->ev_join, &ctx->ev_fork2, &ctx->ev_bnd,
                           &ctx->ev_lb[0], &ctx->ev_lb[1]})
        CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    enter(ctx, stream);

    if (ctx->nranks > 1) {
        if (parent) {
            ctx->nccl = parent->nccl;
            ctx->owns_nccl = false;
        } else if (!ctx->lb) {
            ncclUniqueId uid;
            std::memcpy(&uid, comm->nccl_id, 128);
            NK(ncclCommInitRank(&ctx->nccl, ctx->nranks, uid, ctx->rank));
        }
        // setup collective: allgather of element-surface gids (sorted) of every rank
        int64_t ns = nek_plan_surface_gids(p, nullptr);
        std::vector<int64_t> mine(ns);
        nek_plan_surface_gids(p, mine.data());
        std::vector<int64_t> counts(ctx->nranks);
        if ((st = coll_allgather_host(ctx, &ns, sizeof(int64_t), counts.data())) != NEK_OK) return st;
        int64_t mx = 1;
        for (auto c : counts) mx = std::max(mx, c);
        mine.resize(mx, -1);
        std::vector<int64_t> all((size_t)mx * ctx->nranks);
        if ((st = coll_allgather_host(ctx, mine.data(), sizeof(int64_t) * mx, all.data())) != NEK_OK) return st;
        std::vector<const int64_t *> lists(ctx->nranks);
        for (int q = 0; q < ctx->nranks; ++q) lists[q] = all.data() + (size_t)q * mx;
        st = nek_plan_set_ranks(p, ctx->rank, ctx->nranks, counts.data(), lists.data());
        if (st != NEK_OK) return fail(ctx, st, p->err);
    }

    // reference element
    std::vector<double> x(N + 1), w(N + 1), D((N + 1) * (N + 1));
    gll_rule(N, x.data(), w.data());
    deriv_matrix(N, x.data(), D.data());
    CK(upload_D(N, D.data()));

    // maps -> device (int32 offsets: n_local < 2^31 is enforced by the plan)
    auto to32 = [](const std::vector<int64_t> &v) { return std::vector<int32_t>(v.begin(), v.end()); };
    ctx->nruns = (int64_t)p->offs.size() - 1; ctx->nperm = (int64_t)p->perm.size();
    CK(upload(ctx, &ctx->perm, p->perm));
    CK(upload(ctx, &ctx->offs, to32(p->offs)));
    {   // length classes of the local runs (same runs, same order within a class)
        std::vector<int32_t> c2, c4, c8, cg, og(1, 0);
        for (int64_t r = 0; r < ctx->nruns; ++r) {
            const int64_t a = p->offs[r], len = p->offs[r + 1] - a;
            std::vector<int32_t> &dst = len == 2 ? c2 : len == 4 ? c4 : len == 8 ? c8 : cg;
            for (int64_t c = 0; c < len; ++c) dst.push_back(p->perm[a + c]);
            if (len != 2 && len != 4 && len != 8) og.push_back((int32_t)cg.size());
        }
        CK(upload(ctx, &ctx->gs_p2, c2)); CK(upload(ctx, &ctx->gs_p4, c4)); CK(upload(ctx, &ctx->gs_p8, c8));
        CK(upload(ctx, &ctx->gs_pg, cg)); CK(upload(ctx, &ctx->gs_og, og));
        ctx->gsc.n2 = (int64_t)c2.size() / 2; ctx->gsc.n4 = (int64_t)c4.size() / 4; ctx->gsc.n8 = (int64_t)c8.size() / 8;
        ctx->gsc.ng = (int64_t)og.size() - 1;
        ctx->gsc.nv = ctx->n;
        ctx->gsc.p2 = ctx->gs_p2; ctx->gsc.p4 = ctx->gs_p4; ctx->gsc.p8 = ctx->gs_p8;
        ctx->gsc.pg = ctx->gs_pg; ctx->gsc.og = ctx->gs_og;
        {   // element-chunk offsets of the four classes (runs are in first-copy order within a class)
            const char *genv = getenv("NEK_GS_CHUNK");
            if (!(genv && std::strcmp(genv, "0") == 0) && E > 0) {
                const int64_t K = gs_chunk_elems(), nch = (E + K - 1) / K, S = nch + 1, span = K * ctx->P3;
                std::vector<int32_t> coff((size_t)(4 * S), 0);
                auto fill = [&](int k, const std::vector<int32_t> &first) {
                    int64_t r = 0;
                    for (int64_t c = 0; c <= nch; ++c) {
                        while (r < (int64_t)first.size() && first[r] < c * span) ++r;
                        coff[(size_t)(k * S + c)] = (int32_t)r;
                    }
                    coff[(size_t)(k * S + nch)] = (int32_t)first.size();
                };
                std::vector<int32_t> f2, f4, f8, fg;
                for (size_t r = 0; r < c2.size(); r += 2) f2.push_back(c2[r]);
                for (size_t r = 0; r < c4.size(); r += 4) f4.push_back(c4[r]);
                for (size_t r = 0; r < c8.size(); r += 8) f8.push_back(c8[r]);
                for (size_t r = 0; r + 1 < og.size(); ++r) fg.push_back(cg[og[r]]);
                fill(0, f2); fill(1, f4); fill(2, f8); fill(3, fg);
                CK(upload(ctx, &ctx->gs_coff, coff));
                ctx->gsc.coff = ctx->gs_coff; ctx->gsc.nchunk = nch;
            }
        }
        // boundary Ax + halo send beside the interior Ax (concurrent streams) pays off for small
        // per-rank problems, where the boundary launch alone would leave most SMs idle; for large
        // ones the send must not queue behind the persistent interior grid (measured)
        const char *cenv = getenv("NEK_CONCURRENT_BND");
        ctx->concurrent_bnd = cenv ? std::strcmp(cenv, "1") == 0 : E < 16384;
        const char *senv = getenv("NEK_BND_SPLIT");
        ctx->bnd_split = !(senv && std::strcmp(senv, "0") == 0);
        const char *eenv = getenv("NEK_BND_EPC");
        ctx->bnd_epc = eenv ? std::max(0, atoi(eenv)) : 0;
    }
    ctx->nifc = (int64_t)p->ifc_offs.size() - 1; ctx->nifc_perm = (int64_t)p->ifc_perm.size();
    CK(upload(ctx, &ctx->ifc_perm, p->ifc_perm));
    CK(upload(ctx, &ctx->ifc_offs, to32(p->ifc_offs)));
    CK(upload(ctx, &ctx->send_run, p->send_run));
    {   // per send slot, the local copies of its run in canonical order (the P2P pack's gather list)
        std::vector<int32_t> p4(4 * p->send_run.size(), -1);
        for (size_t q = 0; q < p->send_run.size(); ++q) {
            const int64_t r = p->send_run[q], a = p->ifc_offs[r], b = p->ifc_offs[r + 1];
            if (b - a > 4) { p4[4 * q] = -2; continue; }
            for (int64_t c = a; c < b; ++c) p4[4 * q + (c - a)] = p->ifc_perm[c];
        }
        CK(upload(ctx, &ctx->pack4, p4));
    }
    CK(upload(ctx, &ctx->coffs, to32(p->contrib_offs)));
    CK(upload(ctx, &ctx->contrib, p->contrib));
    ctx->nslots = (int64_t)p->send_run.size();
    ctx->neighbors = p->neighbors;
    ctx->send_offs = p->send_offs;
    CK(dalloc(ctx, &ctx->ifc_partial, ctx->nifc));
    CK(dalloc(ctx, &ctx->sendbuf, ctx->nslots));
    CK(dalloc(ctx, &ctx->recvbuf, ctx->nslots));
    CK(upload(ctx, &ctx->elist, p->elem_order));
    ctx->n_boundary = p->n_boundary;
    CK(upload(ctx, &ctx->mbits, pack_bits(p->mask)));
    CK(upload(ctx, &ctx->obits, pack_bits(p->owner)));
    ctx->n_masked = 0;
    for (auto m : p->mask) ctx->n_masked += m;

    // NVLink peer-memory path: map the peers' mailbox / halo buffers (CUDA IPC, or the siblings' own
    // pointers in a loopback group); NEK_P2P=0 or a staged loopback group keeps the NCCL-path kernels
    if (ctx->nranks > 1) {
        const char *env = getenv("NEK_P2P");
        const bool want = !(env && std::strcmp(env, "0") == 0) && !(ctx->lb && ctx->lb->transport == 1);
        if ((st = setup_p2p(ctx, want)) != NEK_OK) return st;
    }

    // geometry
    const int64_t n = ctx->n;
    CK(dalloc(ctx, &ctx->G, 6 * n));
    CK(dalloc(ctx, &ctx->wJ, n));
    {
        double *dxyz = nullptr, *dwq = nullptr;
        unsigned long long *dbad = nullptr, hbad = ~0ull;
        CK(cudaMalloc(&dxyz, sizeof(double) * 3 * std::max<int64_t>(n, 1)));
        CK(cudaMalloc(&dwq, sizeof(double) * (N + 1)));
        CK(cudaMalloc(&dbad, sizeof(unsigned long long)));
        if (n) CK(cudaMemcpy(dxyz, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dwq, w.data(), sizeof(double) * (N + 1), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dbad, &hbad, sizeof(hbad), cudaMemcpyHostToDevice));
        CK(launch_geom(N, E, dxyz, ctx->G, ctx->wJ, dwq, dbad, ctx->s_main));
        CK(cudaMemcpyAsync(&hbad, dbad, sizeof(hbad), cudaMemcpyDeviceToHost, ctx->s_main));
        CK(cudaStreamSynchronize(ctx->s_main));
        cudaFree(dxyz); cudaFree(dwq); cudaFree(dbad);
        if (hbad != ~0ull) {
            int64_t l = (int64_t)hbad;
            return fail(ctx, NEK_EGEOM, "non-positive Jacobian at element " + std::to_string(l / ctx->P3) +
                                           ", node " + std::to_string(l % ctx->P3));
        }
    }
    // work vectors, reductions, scalars
    for (double **v : {&ctx->vr, &ctx->vp, &ctx->vw, &ctx->vx, &ctx->vdinv, &ctx->vtmp}) CK(dalloc(ctx, v, n));
    // partial slots of (hi, lo) pairs: Ax one per CTA, the vector kernels two dots per CTA
    ctx->npart = std::max<int64_t>(2 * (int64_t)ax_partials_needed(1, N, E), std::max(4 * vec_blocks(), 4 * upd_blocks()));
    {
        // L2-resident PCG vectors: when p, r, Dinv, w (and x) plus the gather-scatter lists fit in the
        // L2 next to the streamed metric factors (evict_first), keep them there (evict_last) across
        // the kernels of an iteration; NEK_L2KEEP = 0 / 1 / 3 overrides the size rule
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device);
        const double vec = 8.0 * (double)n, idx = 4.0 * (double)ctx->nperm;
        int keep = 0;
        if (4 * vec + idx <= 0.6 * l2) keep = 1;
        if (5 * vec + idx <= 0.6 * l2) keep = 3;
        const char *kenv = getenv("NEK_L2KEEP");
        if (kenv) keep = atoi(kenv);
        ctx->l2keep = keep;
        ctx->gsc.keep = keep & 1;
        // evict_last lines live in the persisting L2 set-aside: sized for the kept vectors (clamped to
        // cudaDevAttrMaxPersistingL2CacheSize; NEK_L2SETASIDE = MiB) and granted only for the duration
        // of a solve -- the carve-out halves the write bandwidth of everything else (measured: 3.0 vs
        // 5.9 TB/s for a streaming write, nek_ax and the pMG V-cycle 11-15% slower)
        if (keep) {
            int maxp = 0;
            cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
            double want = ((keep & 2) ? 5 : 4) * vec + idx;
            const char *senv = getenv("NEK_L2SETASIDE");
            if (senv) want = (double)atoll(senv) * (1 << 20);
            ctx->l2_setaside = (int64_t)std::min<double>(want, (double)maxp);
            ctx->l2_setaside_max = maxp;
        }
    }
    CK(dalloc(ctx, &ctx->part, ctx->npart));
    CK(dalloc(ctx, &ctx->upart, 4 * (int64_t)std::max(upd_blocks(), upd_blocks_deferred())));
    {
        const char *denv = getenv("NEK_DEFER");
        ctx->defer = !(denv && std::strcmp(denv, "0") == 0);
        const char *penv = getenv("NEK_V5_PF_MIN");
        if (penv) ctx->v5_pf_min = (int64_t)atoll(penv);
    }
    CK(dalloc(ctx, &ctx->red_loc, RED_N));
    if (ctx->nranks > 1) CK(dalloc(ctx, &ctx->red_all, RED_N * ctx->nranks));
    else ctx->red_all = ctx->red_loc;
    CK(dalloc(ctx, &ctx->sc, 1));
    CK(cudaMallocHost(&ctx->sc_host, sizeof(PcgScalars)));
    CK(dalloc(ctx, &ctx->counter, 4));
    CK(cudaMemset(ctx->counter, 0, 4 * sizeof(unsigned int)));
    CK(cudaMemset(ctx->red_loc, 0, sizeof(double) * RED_N));
    CK(cudaStreamSynchronize(ctx->s_main));
    leave(ctx, stream);
    return NEK_OK;
}

int nek_setup(nek_ctx **out, int64_t E, int N, const double *xyz, const int64_t *gid, const uint8_t *dirichlet,
              const nek_comm *comm, int device, void *stream)
{
    if (!out) return fail(nullptr, NEK_EINVAL, "null out");
    *out = nullptr;
    nek_ctx *ctx = new (std::nothrow) nek_ctx();
    if (!ctx) return fail(nullptr, NEK_ENOMEM, "host allocation failed");
    ctx->device = device;
    int st;
    try {
        st = setup_impl(ctx, E, N, xyz, gid, dirichlet, comm, stream);
    } catch (const std::bad_alloc &) {
        st = fail(ctx, NEK_ENOMEM, "host allocation failed");
    }
    if (st != NEK_OK) {
        g_last_error = ctx->err;
        if (ctx->lb) ctx->lb->abort();   // the other ranks' collectives fail instead of waiting
        nek_free(ctx);
        return st;
    }
    *out = ctx;
    return NEK_OK;
}

int nek_free(nek_ctx *ctx)
{
    if (!ctx) return NEK_OK;
    cudaSetDevice(ctx->device);
    for (cudaStream_t st : {ctx->s_main, ctx->s_hi, ctx->s_comm})
        if (st) cudaStreamSynchronize(st);
    // loopback: no rank releases buffers its siblings may still write into (their kernels are done once
    // every rank has synchronised; a failed setup aborted the group first, so this returns at once)
    if (ctx->lb) ctx->lb->barrier();
    if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
    for (auto &t : ctx->graph_timers) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
    for (void *p : {(void *)ctx->G, (void *)ctx->wJ, (void *)ctx->perm, (void *)ctx->offs, (void *)ctx->ifc_perm,
                    (void *)ctx->ifc_offs, (void *)ctx->send_run, (void *)ctx->pack4, (void *)ctx->coffs,
                    (void *)ctx->contrib,
                    (void *)ctx->ifc_partial, (void *)ctx->sendbuf, (void *)ctx->recvbuf, (void *)ctx->elist,
                    (void *)ctx->mbits, (void *)ctx->obits, (void *)ctx->vr, (void *)ctx->vp, (void *)ctx->vw,
                    (void *)ctx->vx, (void *)ctx->vdinv, (void *)ctx->vtmp, (void *)ctx->stage_in,
                    (void *)ctx->stage_out, (void *)ctx->part, (void *)ctx->red_loc, (void *)ctx->sc,
                    (void *)ctx->counter, (void *)ctx->hist, (void *)ctx->gs_p2, (void *)ctx->gs_p4,
                    (void *)ctx->gs_p8, (void *)ctx->gs_pg, (void *)ctx->gs_og, (void *)ctx->gs_coff,
                    (void *)ctx->upart})
        if (p) cudaFree(p);
    if (ctx->red_all && ctx->red_all != ctx->red_loc) cudaFree(ctx->red_all);
    for (void *p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
    if (ctx->p2p_err_host) cudaFreeHost(ctx->p2p_err_host);
    for (void *p : {(void *)ctx->mbox, (void *)ctx->d_peer_mbox, (void *)ctx->epochs,
                    (void *)ctx->recv2, (void *)ctx->d_peer_recv, (void *)ctx->d_remote_off, (void *)ctx->d_send_offs,
                    (void *)ctx->d_remote_half,
                    (void *)ctx->d_slot_nbr, (void *)ctx->d_nbr, (void *)ctx->hflags, (void *)ctx->d_peer_hflags})
        if (p) cudaFree(p);
    if (ctx->sc_host) cudaFreeHost(ctx->sc_host);
    TimerPool &P = pool_of(ctx);
    for (auto &t : P.pending) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
    for (auto e : P.free_ev) cudaEventDestroy(e);
    P.pending.clear(); P.free_ev.clear();
    for (cudaEvent_t e : {ctx->ev_in, ctx->ev_out, ctx->ev_fork, ctx->ev_join, ctx->ev_fork2, ctx->ev_bnd,
                          ctx->ev_lb[0], ctx->ev_lb[1]})
        if (e) cudaEventDestroy(e);
    if (ctx->nccl && ctx->owns_nccl) ncclCommDestroy(ctx->nccl);
    if (ctx->owns_streams) {
        if (ctx->s_main) cudaStreamDestroy(ctx->s_main);
        if (ctx->s_comm) cudaStreamDestroy(ctx->s_comm);
        if (ctx->s_hi) cudaStreamDestroy(ctx->s_hi);
    }
    nek_plan_free(ctx->plan);
    delete ctx;
    return NEK_OK;
}

int nek_ax(nek_ctx *ctx, double h1, double h2, const double *u, double *w, void *stream)
{
    if (!ctx) return fail(nullptr, NEK_EINVAL, "null ctx");
    if (!u || !w || (const void *)u == (void *)w) return fail(ctx, NEK_EINVAL, "null or aliasing u/w");
    CK(cudaSetDevice(ctx->device));
    const bool du = is_device_ptr(u), dw = is_device_ptr(w);
    int st;
    if ((st = check_peer(ctx)) != NEK_OK) return st;
    OnCallerStream on_caller(ctx, stream);
    if (!on_caller.on) enter(ctx, stream);
    const double *ud = u;
    double *wd = w;
    if (!du || !dw) { if ((st = ensure_stage(ctx)) != NEK_OK) return st; }
    if (!du) { CK(cudaMemcpyAsync(ctx->stage_in, u, sizeof(double) * ctx->n, cudaMemcpyHostToDevice, ctx->s_main)); ud = ctx->stage_in; }
    if (!dw) wd = ctx->stage_out;
    if ((st = apply_op(ctx, h1, h2, ud, wd, false, nullptr)) != NEK_OK) return st;
    if (!dw) {
        CK(cudaMemcpyAsync(w, wd, sizeof(double) * ctx->n, cudaMemcpyDeviceToHost, ctx->s_main));
        CK(cudaStreamSynchronize(ctx->s_main));
        if ((st = check_peer(ctx)) != NEK_OK) return st;   // device-pointer calls report it at the next call
    }
    if (!on_caller.on) leave(ctx, stream);
    return NEK_OK;
}

int nek_gs(nek_ctx *ctx, double *v, void *stream)
{
    if (!ctx) return fail(nullptr, NEK_EINVAL, "null ctx");
    if (!v) return fail(ctx, NEK_EINVAL, "null v");
    CK(cudaSetDevice(ctx->device));
    const bool dv = is_device_ptr(v);
    int st;
    if ((st = check_peer(ctx)) != NEK_OK) return st;
    OnCallerStream on_caller(ctx, stream);
    if (!on_caller.on) enter(ctx, stream);
    double *vd = v;
    if (!dv) {
        if ((st = ensure_stage(ctx)) != NEK_OK) return st;
        CK(cudaMemcpyAsync(ctx->stage_in, v, sizeof(double) * ctx->n, cudaMemcpyHostToDevice, ctx->s_main));
        vd = ctx->stage_in;
    }
    if ((st = gs_full(ctx, vd, nullptr)) != NEK_OK) return st;
    if (!dv) {
        CK(cudaMemcpyAsync(v, vd, sizeof(double) * ctx->n, cudaMemcpyDeviceToHost, ctx->s_main));
        CK(cudaStreamSynchronize(ctx->s_main));
        if ((st = check_peer(ctx)) != NEK_OK) return st;
    }
    if (!on_caller.on) leave(ctx, stream);
    return NEK_OK;
}

// one PCG iteration (device-resident, skipped once sc->done is set)
static int pcg_iteration(nek_ctx *ctx, double h1, double h2)
{
    int st;
    const int *done = &ctx->sc->done;
    const int nb = vec_blocks();
    if (use_fused(ctx) && ctx->p2p) {
        // sigma pushed by the Ax kernel, pulled by the update kernel; (rho', rr) pushed by the
        // update kernel, pulled by the bookkeeping kernel (or, deferred, by the next Ax): no
        // separate exchange launches
        const bool dp = use_defer_p2p(ctx);
        if (dp && (st = lb_stage_sync(ctx, ctx->s_main)) != NEK_OK) return st;   // loopback: (rho', rr) pushed
        if ((st = apply_op(ctx, h1, h2, ctx->vp, ctx->vw, true, done, true)) != NEK_OK) return st;
        const P2PMail m = mail_of(ctx);
        if ((st = lb_stage_sync(ctx, ctx->s_main)) != NEK_OK) return st;   // loopback: every rank pushed sigma
        {
            Scope sc(ctx, CLS_VEC);
            CK(launch_pcg_update_fused(ctx->n, ctx->obits, ctx->vdinv, ctx->vw, ctx->vr, ctx->red_all, ctx->nranks,
                                       ctx->sc, ctx->hist, ctx->part, upd_blocks(), ctx->red_loc + RED_RHO,
                                       ctx->counter + 2, ctx->s_main, &m, ctx->l2keep, dp ? 1 : 0,
                                       ctx->E >= ctx->v5_pf_min));
            ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
        }
        if (dp) return NEK_OK;
        if ((st = lb_stage_sync(ctx, ctx->s_main)) != NEK_OK) return st;   // loopback: every rank pushed (rho', rr)
        {
            Scope sc(ctx, CLS_VEC);
            CK(launch_pcg_fin_p2p(ctx->sc, m, ctx->hist, ctx->s_main));
            ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
        }
        return NEK_OK;
    }
    if (use_defer(ctx)) {
        // Ax: fold the last update's (rho', rr), bookkeeping, p and deferred x, w = A p, sigma partials;
        // update: fold sigma, r -= alpha w, (rho', rr) partials -- no last-CTA work in either
        if ((st = apply_op(ctx, h1, h2, ctx->vp, ctx->vw, true, done, true)) != NEK_OK) return st;
        const int var = ax_effective_variant(ctx->variant, ctx->N, true, ctx->l2keep);
        Scope sc(ctx, CLS_VEC);
        CK(launch_pcg_update_deferred(ctx->n, ctx->obits, ctx->vdinv, ctx->vw, ctx->vr, ctx->part,
                                      (int)ax_grid(var, ctx->N, ctx->E), ctx->sc, ctx->upart, upd_blocks_deferred(),
                                      ctx->l2keep, ctx->s_main, ctx->E >= ctx->v5_pf_min));
        ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
        return NEK_OK;
    }
    if (use_fused(ctx)) {
        // Ax prologue: p = Dinv r + beta p, x += alpha p (deferred); then w = A p, sigma
        if ((st = apply_op(ctx, h1, h2, ctx->vp, ctx->vw, true, done, true)) != NEK_OK) return st;
        if ((st = exchange_slots(ctx, 0)) != NEK_OK) return st;
        {
            Scope sc(ctx, CLS_VEC);
            CK(launch_pcg_update_fused(ctx->n, ctx->obits, ctx->vdinv, ctx->vw, ctx->vr, ctx->red_all, ctx->nranks,
                                       ctx->sc, ctx->hist, ctx->part, upd_blocks(), ctx->red_loc + RED_RHO,
                                       ctx->counter + 2, ctx->s_main, nullptr, ctx->l2keep, 0,
                                       ctx->E >= ctx->v5_pf_min));
            ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
        }
        if (ctx->nranks > 1) {
            if ((st = exchange_slots(ctx, 1)) != NEK_OK) return st;
            CK(launch_pcg_iter_fin(ctx->sc, ctx->red_all, ctx->nranks, ctx->hist, ctx->s_main));
            ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
        }
        return NEK_OK;
    }
    if ((st = apply_op(ctx, h1, h2, ctx->vp, ctx->vw, true, done)) != NEK_OK) return st;
    if ((st = exchange_slots(ctx, 0)) != NEK_OK) return st;
    {
        Scope sc(ctx, CLS_VEC);
        CK(launch_pcg_update(ctx->n, ctx->obits, ctx->vdinv, ctx->vp, ctx->vw, ctx->vx, ctx->vr, ctx->red_all,
                             ctx->nranks, ctx->sc, ctx->part, upd_blocks(), ctx->red_loc + RED_RHO, ctx->counter + 2,
                             ctx->s_main));
        ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
    }
    if ((st = exchange_slots(ctx, 1)) != NEK_OK) return st;
    {
        Scope sc(ctx, CLS_VEC);
        CK(launch_pcg_pupdate(ctx->n, ctx->vdinv, ctx->vr, ctx->vp, ctx->red_all, ctx->nranks, ctx->sc, ctx->hist,
                              ctx->counter, nb, ctx->s_main));
        ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
    }
    return NEK_OK;
}

int nek_pcg_solve(nek_ctx *ctx, double h1, double h2, const double *b, double *x, double tol, int maxit, int *iters,
                  double *relres, double *hist, void *stream)
{
    if (!ctx) return fail(nullptr, NEK_EINVAL, "null ctx");
    if (!b || !x || maxit < 0 || !(tol >= 0.0)) return fail(ctx, NEK_EINVAL, "bad b/x/maxit/tol");
    CK(cudaSetDevice(ctx->device));
    int st;
    if ((st = check_peer(ctx)) != NEK_OK) return st;
    enter(ctx, stream);
    if ((st = ensure_dinv(ctx, h1, h2)) != NEK_OK) return st;
    if (ctx->hist_cap < maxit + 1) {
        if (ctx->hist) cudaFree(ctx->hist);
        ctx->hist = nullptr;
        const int cap = std::max<int>(maxit + 1, std::max<int>(1024, 2 * (int)ctx->hist_cap));   // grow rarely: graphs hold it
        CK(dalloc(ctx, &ctx->hist, cap));
        ctx->hist_cap = cap;
        if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
    }
    const bool db = is_device_ptr(b), dx = is_device_ptr(x);
    const double *bd = b;
    if (!db) {
        if ((st = ensure_stage(ctx)) != NEK_OK) return st;
        CK(cudaMemcpyAsync(ctx->stage_in, b, sizeof(double) * ctx->n, cudaMemcpyHostToDevice, ctx->s_main));
        bd = ctx->stage_in;
    }
    L2SetAside l2scope(ctx);
    PcgScalars *H = ctx->sc_host;
    std::memset(H, 0, sizeof(*H));
    H->tol = tol; H->maxit = maxit;
    CK(cudaMemcpyAsync(ctx->sc, H, sizeof(PcgScalars), cudaMemcpyHostToDevice, ctx->s_main));
    const int nb = vec_blocks();
    {
        Scope sc(ctx, CLS_VEC);
        CK(launch_pcg_init(ctx->n, ctx->mbits, ctx->obits, bd, ctx->vdinv, ctx->vr, ctx->vp, ctx->vx, ctx->part, nb,
                           ctx->red_loc + RED_RHO, ctx->counter + 2, use_fused(ctx), ctx->s_main));
        ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
    }
    if ((st = exchange_slots(ctx, 1)) != NEK_OK) return st;
    CK(launch_pcg_init_fin(ctx->sc, ctx->red_all, ctx->nranks, ctx->hist, ctx->s_main));
    ctx->stats.launches += 1;

    // iterations per graph replay: a replay boundary costs ~6 us on the device; a converged solve
    // overshoots by < C iterations whose kernels return at entry
    const int C = std::max(1, std::min(maxit, 20));
    const char *genv = getenv("NEK_NO_GRAPH");
    // loopback: the stage syncs swap events between host threads at every exchange, so the iterations
    // are launched directly (a captured graph would freeze one set of cross-rank waits)
    const bool use_graph = !(genv && std::strcmp(genv, "0") != 0) && !ctx->lb;
    if (use_graph && (!ctx->graph || ctx->graph_iters != C || ctx->graph_h1 != h1 || ctx->graph_h2 != h2 ||
                      ctx->graph_timing != ctx->timing)) {
        if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
        for (auto &t : ctx->graph_timers) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
        ctx->graph_timers.clear();
        ctx->capturing = true;
        cudaGraph_t g;
        nek_stats_t saved = ctx->stats;
        CK(cudaStreamBeginCapture(ctx->s_main, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < C; ++k) {
            if ((st = pcg_iteration(ctx, h1, h2)) != NEK_OK) {
                cudaStreamEndCapture(ctx->s_main, &g);
                ctx->capturing = false;
                return st;
            }
        }
        ctx->capturing = false;
        CK(cudaStreamEndCapture(ctx->s_main, &g));
        ctx->graph_timing = ctx->timing;
        // launches recorded in one replay of the graph
        ctx->graph_stats = ctx->stats;
        ctx->graph_stats.launches -= saved.launches;
        ctx->graph_stats.ax_launches -= saved.ax_launches;
        ctx->graph_stats.ax_elements -= saved.ax_elements;
        ctx->graph_stats.gs_launches -= saved.gs_launches;
        ctx->graph_stats.halo_launches -= saved.halo_launches;
        ctx->graph_stats.vec_launches -= saved.vec_launches;
        ctx->graph_stats.ax_bytes -= saved.ax_bytes;
        ctx->graph_stats.axu_spans -= saved.axu_spans;
        ctx->stats = saved;
        CK(cudaGraphInstantiate(&ctx->graph, g, 0));
        cudaGraphDestroy(g);
        ctx->graph_iters = C; ctx->graph_h1 = h1; ctx->graph_h2 = h2;
    }
    int launched = 0;
    while (launched < maxit) {
        if (use_graph) {
            CK(cudaGraphLaunch(ctx->graph, ctx->s_main));
            const nek_stats_t &g = ctx->graph_stats;
            ctx->stats.ax_bytes += g.ax_bytes;
            ctx->stats.launches += g.launches; ctx->stats.ax_launches += g.ax_launches;
            ctx->stats.ax_elements += g.ax_elements; ctx->stats.gs_launches += g.gs_launches;
            ctx->stats.halo_launches += g.halo_launches; ctx->stats.vec_launches += g.vec_launches;
            ctx->stats.axu_spans += g.axu_spans;
            launched += C;
            if (ctx->timing) {   // per-kernel device time of this replay (event-record nodes)
                CK(cudaStreamSynchronize(ctx->s_main));
                harvest_graph_timers(ctx);
            }
        } else {
            if ((st = pcg_iteration(ctx, h1, h2)) != NEK_OK) return st;
            launched += 1;
        }
        if (tol > 0.0 && (launched % (use_graph ? C : 10)) == 0) {
            CK(cudaMemcpyAsync(H, ctx->sc, sizeof(PcgScalars), cudaMemcpyDeviceToHost, ctx->s_main));
            CK(cudaStreamSynchronize(ctx->s_main));
            if (H->done) break;
        }
    }
    if (use_defer(ctx)) {   // the last update's (rho', rr) when no Ax followed it
        CK(launch_pcg_defer_finish(ctx->sc, ctx->upart, upd_blocks_deferred(), ctx->hist, ctx->s_main));
        ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
    } else if (use_defer_p2p(ctx)) {
        if ((st = lb_stage_sync(ctx, ctx->s_main)) != NEK_OK) return st;   // loopback: (rho', rr) pushed
        const P2PMail m = mail_of(ctx);
        CK(launch_pcg_defer_finish(ctx->sc, nullptr, 0, ctx->hist, ctx->s_main, &m));
        ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
    }
    if (use_fused(ctx)) {   // the deferred x += alpha p of the last iteration
        CK(launch_pcg_xfinal(ctx->n, ctx->sc, ctx->vp, ctx->vx, ctx->s_main));
        ctx->stats.launches += 1; ctx->stats.vec_launches += 1;
    }
    if (ctx->l2keep) {      // release the L2-resident vectors (evict_last -> evict_normal)
        L2Ranges R;
        const int64_t vb = 8 * ctx->n;
        R.add(ctx->vp, vb); R.add(ctx->vr, vb); R.add(ctx->vw, vb); R.add(ctx->vdinv, vb);
        if (ctx->l2keep & 2) R.add(ctx->vx, vb);
        R.add(ctx->gsc.p2, 8 * ctx->gsc.n2); R.add(ctx->gsc.p4, 16 * ctx->gsc.n4);
        R.add(ctx->obits, 4 * ((ctx->n + 31) / 32));
        CK(launch_l2_demote(R, ctx->s_main));
        ctx->stats.launches += 1;
    }
    CK(cudaMemcpyAsync(H, ctx->sc, sizeof(PcgScalars), cudaMemcpyDeviceToHost, ctx->s_main));
    if (dx) CK(cudaMemcpyAsync(x, ctx->vx, sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice, ctx->s_main));
    else CK(cudaMemcpyAsync(x, ctx->vx, sizeof(double) * ctx->n, cudaMemcpyDeviceToHost, ctx->s_main));
    CK(cudaStreamSynchronize(ctx->s_main));
    if (hist && H->iter >= 0)
        CK(cudaMemcpy(hist, ctx->hist, sizeof(double) * (H->iter + 1), cudaMemcpyDeviceToHost));
    if (ctx->timing) harvest_timers(ctx);
    if ((st = check_peer(ctx)) != NEK_OK) return st;
    if (iters) *iters = H->iter;
    if (relres) *relres = H->bb > 0 ? std::sqrt(H->rr) / H->bb : 0.0;
    leave(ctx, stream);
    if (H->status == NEK_ENOTSPD) return fail(ctx, NEK_ENOTSPD, "PCG breakdown: <p, A p> <= 0 at iteration " + std::to_string(H->iter));
    return H->status;
}

int nek_get_info(const nek_ctx *ctx, nek_info_t *info)
{
    if (!ctx || !info) return NEK_EINVAL;
    std::memset(info, 0, sizeof(*info));
    info->E = ctx->E; info->N = ctx->N; info->rank = ctx->rank; info->nranks = ctx->nranks;
    info->n_local = ctx->n; info->n_dof = ctx->E * ctx->N * ctx->N * ctx->N; info->n_masked = ctx->n_masked;
    info->n_runs = ctx->nruns; info->n_perm = ctx->nperm; info->n_ifc_runs = ctx->nifc; info->n_ifc_perm = ctx->nifc_perm;
    info->n_neighbors = (int64_t)ctx->neighbors.size(); info->halo_doubles = ctx->nslots;
    info->n_boundary_elems = ctx->n_boundary; info->device_bytes = ctx->device_bytes; info->geom_min_jac = ctx->min_jac;
    info->transport = ctx->nranks == 1 ? 0 : (ctx->p2p ? 2 : 1);
    info->l2_keep = ctx->l2keep; info->l2_setaside = ctx->l2_setaside; info->l2_setaside_max = ctx->l2_setaside_max;
    return NEK_OK;
}

int nek_get_gs_map(const nek_ctx *ctx, int32_t *perm, int64_t *offs)
{
    if (!ctx || !ctx->plan) return NEK_EINVAL;
    if (perm) nek_plan_get(ctx->plan, NEK_PLAN_PERM, perm);
    if (offs) nek_plan_get(ctx->plan, NEK_PLAN_OFFS, offs);
    return NEK_OK;
}

int nek_get_geom(const nek_ctx *ctx_c, double *G, double *wJ)
{
    nek_ctx *ctx = const_cast<nek_ctx *>(ctx_c);
    if (!ctx) return NEK_EINVAL;
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->s_main));
    if (G) CK(cudaMemcpy(G, ctx->G, sizeof(double) * 6 * ctx->n, cudaMemcpyDeviceToHost));
    if (wJ) CK(cudaMemcpy(wJ, ctx->wJ, sizeof(double) * ctx->n, cudaMemcpyDeviceToHost));
    return NEK_OK;
}

int nek_get_dinv(nek_ctx *ctx, double h1, double h2, double *dinv, void *stream)
{
    if (!ctx || !dinv) return fail(ctx, NEK_EINVAL, "null");
    CK(cudaSetDevice(ctx->device));
    enter(ctx, stream);
    int st = ensure_dinv(ctx, h1, h2);
    if (st != NEK_OK) return st;
    if (is_device_ptr(dinv)) {
        CK(cudaMemcpyAsync(dinv, ctx->vdinv, sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice, ctx->s_main));
    } else {
        CK(cudaMemcpyAsync(dinv, ctx->vdinv, sizeof(double) * ctx->n, cudaMemcpyDeviceToHost, ctx->s_main));
        CK(cudaStreamSynchronize(ctx->s_main));
    }
    leave(ctx, stream);
    return NEK_OK;
}

int nek_set_timing(nek_ctx *ctx, int on)
{
    if (!ctx) return NEK_EINVAL;
    ctx->timing = on != 0;
    return NEK_OK;
}

int nek_get_stats(nek_ctx *ctx, nek_stats_t *stats, int reset)
{
    if (!ctx || !stats) return NEK_EINVAL;
    cudaSetDevice(ctx->device);
    harvest_timers(ctx);
    *stats = ctx->stats;
    if (reset) std::memset(&ctx->stats, 0, sizeof(ctx->stats));
    return NEK_OK;
}

int nek_set_variant(nek_ctx *ctx, int v)
{
    if (!ctx || !ax_variant_valid(v)) return fail(ctx, NEK_EINVAL, "unknown Ax variant " + std::to_string(v));
    ctx->variant = v;
    if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
    return NEK_OK;
}

}  // extern "C"

// ------------------------------------------------------------ projection
struct nek_proj {
    nek_ctx *ctx = nullptr;
    int L = 0, l = 0;
    bool hvalid = false;
    double h1 = 0, h2 = 0;
    double *X = nullptr, *B = nullptr;          // [L][n]
    double *xbar = nullptr, *db = nullptr, *dx = nullptr, *v = nullptr, *av = nullptr, *bm = nullptr;
    double *coef = nullptr, *part = nullptr, *gath = nullptr;
    int nblk = 0;
};

// global owner-copy dot products <V_i, y> for i < l, returned on the host (rank-ordered across ranks)
static int proj_dots(nek_proj *P, int l, const double *V, const double *y, double *out)
{
    nek_ctx *ctx = P->ctx;
    if (l <= 0) return NEK_OK;
    CK(launch_multidot(ctx->n, l, V, y, ctx->obits, P->part, P->nblk, ctx->s_main));
    ctx->stats.launches += 1;
    std::vector<double> hp((size_t)P->nblk * l);
    CK(cudaMemcpyAsync(hp.data(), P->part, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, ctx->s_main));
    CK(cudaStreamSynchronize(ctx->s_main));
    for (int i = 0; i < l; ++i) {
        double s = 0.0;
        for (int b = 0; b < P->nblk; ++b) s += hp[(size_t)b * l + i];
        out[i] = s;
    }
    if (ctx->nranks > 1) {
        CK(cudaMemcpyAsync(P->gath + (size_t)ctx->nranks * PROJ_MAX_VECTORS, out, sizeof(double) * l,
                           cudaMemcpyHostToDevice, ctx->s_main));
        int st;
        if ((st = coll_allgather_dev(ctx, P->gath + (size_t)ctx->nranks * PROJ_MAX_VECTORS, P->gath,
                                     sizeof(double) * l, ctx->s_main)) != NEK_OK)
            return st;
        std::vector<double> all((size_t)ctx->nranks * l);
        CK(cudaMemcpyAsync(all.data(), P->gath, sizeof(double) * all.size(), cudaMemcpyDeviceToHost, ctx->s_main));
        CK(cudaStreamSynchronize(ctx->s_main));
        for (int i = 0; i < l; ++i) {
            double s = all[i];
            for (int q = 1; q < ctx->nranks; ++q) s += all[(size_t)q * l + i];
            out[i] = s;
        }
    }
    return NEK_OK;
}

extern "C" int nek_proj_create(nek_ctx *ctx, int max_vectors, nek_proj **out)
{
    if (!ctx || !out || max_vectors < 0 || max_vectors > PROJ_MAX_VECTORS)
        return fail(ctx, NEK_EINVAL, "max_vectors must be in [0, 32]");
    *out = nullptr;
    CK(cudaSetDevice(ctx->device));
    nek_proj *P = new (std::nothrow) nek_proj();
    if (!P) return fail(ctx, NEK_ENOMEM, "host allocation failed");
    P->ctx = ctx; P->L = max_vectors;
    P->nblk = 2 * device_sms();
    const int64_t n = std::max<int64_t>(ctx->n, 1);
    int st = NEK_OK;
    auto al = [&](double **p, int64_t cnt) {
        if (st != NEK_OK) return;
        if (cudaMalloc(p, sizeof(double) * std::max<int64_t>(cnt, 1)) != cudaSuccess) {
            cudaGetLastError();
            st = fail(ctx, NEK_ENOMEM, "projection space allocation failed");
        }
    };
    al(&P->X, (int64_t)P->L * n); al(&P->B, (int64_t)P->L * n);
    for (double **p : {&P->xbar, &P->db, &P->dx, &P->v, &P->av, &P->bm}) al(p, n);
    al(&P->coef, PROJ_MAX_VECTORS); al(&P->part, (int64_t)P->nblk * PROJ_MAX_VECTORS);
    al(&P->gath, (int64_t)(ctx->nranks + 1) * PROJ_MAX_VECTORS);
    if (st != NEK_OK) { nek_proj_free(P); return st; }
    *out = P;
    return NEK_OK;
}

extern "C" int nek_proj_free(nek_proj *P)
{
    if (!P) return NEK_OK;
    cudaSetDevice(P->ctx->device);
    cudaStreamSynchronize(P->ctx->s_main);
    for (double *p : {P->X, P->B, P->xbar, P->db, P->dx, P->v, P->av, P->bm, P->coef, P->part, P->gath})
        if (p) cudaFree(p);
    delete P;
    return NEK_OK;
}

extern "C" int nek_proj_size(const nek_proj *P) { return P ? P->l : -1; }

extern "C" int nek_proj_reset(nek_proj *P)
{
    if (!P) return NEK_EINVAL;
    P->l = 0;
    return NEK_OK;
}

extern "C" int nek_proj_solve(nek_proj *P, double h1, double h2, const double *b, double *x, double tol, int maxit,
                              int *iters, double *relres, void *stream)
{
    if (!P) return fail(nullptr, NEK_EINVAL, "null projection");
    nek_ctx *ctx = P->ctx;
    if (!b || !x || maxit < 0 || !(tol >= 0.0)) return fail(ctx, NEK_EINVAL, "bad b/x/maxit/tol");
    CK(cudaSetDevice(ctx->device));
    const int64_t n = ctx->n;
    int st;
    enter(ctx, stream);
    if (!P->hvalid || P->h1 != h1 || P->h2 != h2) { P->l = 0; P->hvalid = true; P->h1 = h1; P->h2 = h2; }
    // M b (b may live on the host)
    const double *bsrc = b;
    if (!is_device_ptr(b)) {
        if ((st = ensure_stage(ctx)) != NEK_OK) return st;
        CK(cudaMemcpyAsync(ctx->stage_in, b, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->s_main));
        bsrc = ctx->stage_in;
    }
    CK(launch_copy_mask(n, ctx->mbits, bsrc, P->bm, ctx->s_main));
    double alpha[PROJ_MAX_VECTORS];
    if (P->l > 0) {
        if ((st = proj_dots(P, P->l, P->X, P->bm, alpha)) != NEK_OK) return st;
        CK(cudaMemcpyAsync(P->coef, alpha, sizeof(double) * P->l, cudaMemcpyHostToDevice, ctx->s_main));
        CK(launch_multiaxpy(n, P->l, 0.0, P->xbar, P->X, P->coef, ctx->s_main));
        CK(launch_multiaxpy(n, P->l, 0.0, P->v, P->B, P->coef, ctx->s_main));
        CK(launch_axpby(n, 1.0, P->bm, -1.0, P->v, P->db, ctx->s_main));
        ctx->stats.launches += 3;
    } else {
        CK(cudaMemsetAsync(P->xbar, 0, sizeof(double) * n, ctx->s_main));
        CK(cudaMemcpyAsync(P->db, P->bm, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s_main));
    }
    double bn2 = 0.0, dn2 = 0.0;
    if ((st = proj_dots(P, 1, P->bm, P->bm, &bn2)) != NEK_OK) return st;
    if ((st = proj_dots(P, 1, P->db, P->db, &dn2)) != NEK_OK) return st;
    const double bn = std::sqrt(bn2), dn = std::sqrt(dn2);
    double rel = 1.0;
    if (bn > 0.0 && dn > 0.0) rel = std::min(1.0, tol * bn / dn);
    int it = 0;
    double rr = 0.0;
    int pst = nek_pcg_solve(ctx, h1, h2, P->db, P->dx, rel, maxit, &it, &rr, nullptr, ctx->s_main);
    if (pst < 0) return pst;
    CK(launch_axpby(n, 1.0, P->xbar, 1.0, P->dx, P->v, ctx->s_main));   // x = xbar + dx (in v)
    ctx->stats.launches += 1;
    if (is_device_ptr(x)) CK(cudaMemcpyAsync(x, P->v, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s_main));
    else CK(cudaMemcpyAsync(x, P->v, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->s_main));
    // update the space
    if (P->L > 0 && bn > 0.0) {
        if (P->l < P->L) {
            CK(cudaMemcpyAsync(P->v, P->dx, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s_main));
            if ((st = apply_op(ctx, h1, h2, P->v, P->av, false, nullptr)) != NEK_OK) return st;
            double c[PROJ_MAX_VECTORS];
            for (int pass = 0; pass < 2 && P->l > 0; ++pass) {
                if ((st = proj_dots(P, P->l, P->B, P->v, c)) != NEK_OK) return st;
                for (int i = 0; i < P->l; ++i) c[i] = -c[i];
                CK(cudaMemcpyAsync(P->coef, c, sizeof(double) * P->l, cudaMemcpyHostToDevice, ctx->s_main));
                CK(launch_multiaxpy(n, P->l, 1.0, P->v, P->X, P->coef, ctx->s_main));
                CK(launch_multiaxpy(n, P->l, 1.0, P->av, P->B, P->coef, ctx->s_main));
                ctx->stats.launches += 2;
            }
            double nrm2 = 0.0;
            if ((st = proj_dots(P, 1, P->v, P->av, &nrm2)) != NEK_OK) return st;
            if (nrm2 > 0.0) {
                const double inv = 1.0 / std::sqrt(nrm2);
                CK(launch_axpby(n, inv, P->v, 0.0, P->v, P->X + (int64_t)P->l * n, ctx->s_main));
                CK(launch_axpby(n, inv, P->av, 0.0, P->av, P->B + (int64_t)P->l * n, ctx->s_main));
                ctx->stats.launches += 2;
                P->l += 1;
            }
        } else {   // full: restart from the current solution
            if ((st = apply_op(ctx, h1, h2, P->v, P->av, false, nullptr)) != NEK_OK) return st;
            double nrm2 = 0.0;
            if ((st = proj_dots(P, 1, P->v, P->av, &nrm2)) != NEK_OK) return st;
            if (nrm2 > 0.0) {
                const double inv = 1.0 / std::sqrt(nrm2);
                CK(launch_axpby(n, inv, P->v, 0.0, P->v, P->X, ctx->s_main));
                CK(launch_axpby(n, inv, P->av, 0.0, P->av, P->B, ctx->s_main));
                ctx->stats.launches += 2;
                P->l = 1;
            } else {
                P->l = 0;
            }
        }
    }
    CK(cudaStreamSynchronize(ctx->s_main));
    if (iters) *iters = it;
    if (relres) *relres = bn > 0.0 ? rr * dn / bn : 0.0;
    leave(ctx, stream);
    return pst;
}

#include "pmg.inc"
#include "makef.inc"
