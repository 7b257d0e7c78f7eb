// nek_ctx.h -- internal state of a context (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

#include "loopback.h"
#include "nek.h"
#include "nek_plan_impl.h"

namespace nekb200 {

// Device-side scalars of one PCG solve (one struct, device memory).
struct PcgScalars {
    double rho;        // <r, z> of the current iterate
    double bb;         // ||M b||
    double tol;        // relative tolerance
    double rr;         // ||r||^2 of the current iterate
    int iter;          // iterations completed
    int maxit;
    int done;          // 1 once converged / maxit / breakdown
    int status;        // NEK_OK, NEK_MAXIT, NEK_ENOTSPD
    double sigma;      // global <p, A p> of the current iteration (P2P path)
    double alpha;      // alpha of the last update whose x += alpha p is still pending (fused path)
    double beta;       // beta for the next direction update (fused path)
    // deferred reductions (single rank, N = 7): the update leaves its dot partials, the next Ax folds them
    double rho_next;   // rho for the next update's alpha (written by the Ax that folded the partials)
    int fold_ready;    // 1 once an update has left partials (the next Ax folds them)
    int booked;        // iterations whose (rho', rr) the bookkeeping has recorded
};

// NVLink peer mailbox of a rank: [channel][epoch parity][rank][4] doubles, slot 3 = epoch.
struct P2PMail {
    double *mbox = nullptr;               // local mailbox
    double *const *peer_mbox = nullptr;   // [nranks] (own entry = local)
    uint64_t *epochs = nullptr;
    int *err = nullptr;                   // mapped host memory: raised on a timed-out wait
    int me = 0, nranks = 1;
    uint64_t timeout_ns = 0;
};

// Reduction slots (device): red_loc = this rank's partial sums, red_all = the
// nranks partials gathered in rank order (equal to red_loc at nranks == 1).
enum { RED_SIGMA = 0, RED_RHO = 1, RED_RR = 2, RED_N = 3 };

struct KernelArgsCommon {
    int64_t n;            // local points
    const uint32_t *mbits;  // Dirichlet bit per local point
    const uint32_t *obits;  // owner bit per local point
};

// a pair of timing events around one kernel class
struct TimedLaunch { int cls; cudaEvent_t a, b; };

// GLL rule (ascending nodes, weights) and D[i][j] = h_j'(x_i), host.
void gll_rule(int N, double *x, double *w);
void deriv_matrix(int N, const double *x, double *D);

// pmg_topo.cpp: p-multigrid level construction (host)
void interp_matrix(int Nfrom, int Nto, double *J);
void interp_elements_host(int64_t E, int Nin, int Nout, const double *J, const double *in, double *out);
int pmg_coarse_ids(int64_t E, int Nf, const int64_t *gid, const uint8_t *mask, int Nc, int64_t *gid_c,
                   uint8_t *mask_c, std::string &err);

// kernels.cu entry points (all launched on `s`)
cudaError_t upload_D(int N, const double *D);
cudaError_t launch_geom(int N, int64_t E, const double *xyz, double *G, double *wJ, const double *wq,
                        unsigned long long *bad, cudaStream_t s);
// One Ax launch over elements [eoff, eoff + nelem) of `elist` (or of 0..E-1 when
// elist is NULL).  part/part_off: where its per-CTA <u, w> partials go; when
// fin_total > 0 the launch also reduces part[0..fin_total) into dst[0].
// deferred-reduction modes of the fused v5 Ax (AxLaunch::defer): where the previous update's (rho', rr)
// come from, and whether this launch's CTA 0 records the iteration (one launch per operator application)
enum { DEFER_FOLD = 1, DEFER_MAIL = 2, DEFER_BOOK = 4 };

struct AxLaunch {
    int64_t nelem = 0, eoff = 0;
    const int32_t *elist = nullptr;
    double *part = nullptr;
    int64_t part_off = 0, fin_total = 0;
    double *dst = nullptr;
    unsigned int *counter = nullptr;
    const int *done = nullptr;
    // fused PCG prologue (Ax v5 only): p <- Dinv r + beta p, x <- x + alpha p on the
    // element's points before the operator is applied to the new p (u == p then)
    bool fused = false;
    P2PMail mail;                        // mail.nranks > 1: the finalising CTA pushes sigma to every rank
    unsigned int ctas_total = 0;         // > 0: CTAs of all concurrent launches sharing the finalise counter
    double *p = nullptr, *x = nullptr;
    const double *r = nullptr, *dinv = nullptr;
    const PcgScalars *sc = nullptr;
    int keep = 0;                        // L2-resident mode: bit 0 p, r, Dinv, w; bit 1 also x
    int64_t grid = 0;                    // > 0: CTAs of this launch (v5), else ax_grid
    // deferred reductions (single rank, fused v5): fold the previous update's nupd dot partials at entry
    // (upart: [nupd][4] = (hi, lo) of <r, Dinv r> and <r, r>) and leave this launch's sigma partials
    // unfolded for the update
    const double *upart = nullptr;
    int nupd = 0;
    int defer = 0;   // DEFER_* bits
    // v5 launches of at least pf_min elements bulk-prefetch the next element's metric block to L2
    int64_t pf_min = 16384;
    double *hist = nullptr;
    int variant = -1;                    // >= 0: the Ax variant of this launch (overrides the context's)
};
cudaError_t launch_ax(int variant, int N, const AxLaunch &L, const double *u, const double *G, const double *wJ,
                      const uint32_t *mbits, double h1, double h2, double *w, cudaStream_t s, int *nlaunch);
int64_t ax_grid(int variant, int N, int64_t nelem);      // partial slots one launch writes
bool ax_variant_valid(int variant);
int ax_concrete_variant(int variant, int N, int64_t nelem);   // the configuration variant 0 picks for nelem
int ax_effective_variant(int variant, int N, bool fused, int keep);
int ax_partials_needed(int variant, int N, int64_t E);
// FP32 operator (v6, N <= 9): Gf is [E][ax_gstride_f(N)] (6 planes, padded to 16 bytes per element)
cudaError_t launch_ax_f(int N, int64_t E, const float *u, const float *Gf, const float *wJf, const uint32_t *mbits,
                        double h1, double h2, float *w, cudaStream_t s);
int ax_gstride_f(int N);

// gather-scatter runs grouped by length (see kernels.cu)
struct GsClasses {
    int64_t n2 = 0, n4 = 0, n8 = 0, ng = 0;
    int64_t nv = 0;                      // length of the vector the runs index (checked build)
    const int32_t *p2 = nullptr, *p4 = nullptr, *p8 = nullptr, *pg = nullptr, *og = nullptr;
    int keep = 0;                        // L2 evict_last on the index lists and values (L2-resident mode)
    // element-chunk order (gs_chunk_kernel): coff[k * (nchunk + 1) + c] = first run of class k (pairs,
    // quads, octets, other) whose first copy lies in element chunk c; nullptr: class-major kernel
    const int32_t *coff = nullptr;
    int64_t nchunk = 0;
};
template <class T> cudaError_t launch_gs_classes(const GsClasses &C, T *v, const int *done, cudaStream_t s);
int gs_chunk_elems();   // elements per chunk of the element-chunk gs kernel
cudaError_t launch_reduce(const double *part, int64_t count, int nd, double *dst, const int *done, cudaStream_t s);
cudaError_t launch_gs_local(int64_t nruns, const int32_t *perm, const int32_t *offs, double *v, const int *done,
                            cudaStream_t s);
template <class T>
cudaError_t launch_gs_ifc_pack(int64_t nifc, const int32_t *perm, const int32_t *offs, const T *v,
                               T *partial, int64_t nslots, const int32_t *send_run, T *sendbuf,
                               const int *done, cudaStream_t s);
template <class T>
cudaError_t launch_gs_ifc_unpack(int64_t nifc, const int32_t *perm, const int32_t *offs, const int32_t *coffs,
                                 const int32_t *contrib, const T *partial, const T *recvbuf, T *v,
                                 const int *done, cudaStream_t s, const uint64_t *epoch = nullptr,
                                 int64_t half = 0);
cudaError_t launch_diag(int N, int64_t E, const double *G, const double *wJ, double h1, double h2, double *d,
                        cudaStream_t s);
cudaError_t launch_dinv(int64_t n, const uint32_t *mbits, const double *d, double *dinv, cudaStream_t s);
template <class T> cudaError_t launch_copy_mask(int64_t n, const uint32_t *mbits, const T *src, T *dst, cudaStream_t s);
cudaError_t launch_pcg_init(int64_t n, const uint32_t *mbits, const uint32_t *obits, const double *b,
                            const double *dinv, double *r, double *p, double *x, double *part, int nblk,
                            double *dst, unsigned int *counter, bool p_zero, cudaStream_t s);
// fused path: r -= alpha w and the two dots; at nranks == 1 the last CTA also
// does the iteration bookkeeping, at nranks > 1 pcg_iter_fin does it after the allgather
cudaError_t launch_pcg_update_fused(int64_t n, const uint32_t *obits, const double *dinv, const double *w, double *r,
                                    const double *red_all, int nranks, PcgScalars *sc, double *hist, double *part,
                                    int nblk, double *dst, unsigned int *counter, cudaStream_t s,
                                    const P2PMail *mail = nullptr, int keep = 0, int defer = 0, bool pf = false);
// deferred reductions (single rank, N = 7): sigma folded from the Ax's nax partials at entry, (rho', rr)
// partials left in upart ([nblk][4]) for the next Ax or for pcg_defer_finish
cudaError_t launch_pcg_update_deferred(int64_t n, const uint32_t *obits, const double *dinv, const double *w,
                                       double *r, const double *axpart, int nax, PcgScalars *sc, double *upart,
                                       int nblk, int keep, cudaStream_t s, bool pf = false);
// the bookkeeping of the last update of a solve when no Ax followed it
cudaError_t launch_pcg_defer_finish(PcgScalars *sc, const double *upart, int nupd, double *hist, cudaStream_t s,
                                    const P2PMail *mail = nullptr);
cudaError_t launch_pcg_fin_p2p(PcgScalars *sc, const P2PMail &mail, double *hist, cudaStream_t s);
// device ranges whose L2 lines are demoted from evict_last after an L2-resident solve
struct L2Ranges {
    const void *ptr[10] = {};
    int64_t bytes[10] = {};
    int count = 0;
    void add(const void *p, int64_t b)
    {
        if (p && b > 0 && count < 10) { ptr[count] = p; bytes[count] = b; ++count; }
    }
};
cudaError_t launch_l2_demote(const L2Ranges &R, cudaStream_t s);
// local gather-scatter and (P2P) the halo unpack in one launch
struct HaloUnpack {
    int64_t nifc = 0;
    const int32_t *perm = nullptr, *offs = nullptr, *coffs = nullptr, *contrib = nullptr, *nbr = nullptr;
    double *partial = nullptr;
    const double *recv = nullptr;
    int64_t half = 0;
    const uint64_t *hflags = nullptr, *epochs = nullptr;
    int nnbr = 0;
    int *err = nullptr;
    uint64_t timeout_ns = 0;
    int64_t nv = 0;                      // vector length (checked build)
};
template <class T>
cudaError_t launch_gs_classes_unpack(const GsClasses &C, const HaloUnpack &U, T *v, const int *done,
                                     cudaStream_t s);   // C empty: halo unpack only
cudaError_t launch_pcg_iter_fin(PcgScalars *sc, const double *red_all, int nranks, double *hist, cudaStream_t s);
cudaError_t launch_pcg_xfinal(int64_t n, const PcgScalars *sc, const double *p, double *x, cudaStream_t s);
bool ax_has_fused(int variant, int N);
bool ax_is_v5(int variant, int N);   // the N = 7 v5 kernel (the only one with the deferred-reduction entry)
// projection space (NEXT #2)
constexpr int PROJ_MAX_VECTORS = 32;
cudaError_t launch_multidot(int64_t n, int l, const double *V, const double *y, const uint32_t *obits,
                            double *out_part, int nblk, cudaStream_t s);
cudaError_t launch_multiaxpy(int64_t n, int l, double a, double *y, const double *V, const double *c, cudaStream_t s);
cudaError_t launch_axpby(int64_t n, double alpha, const double *x, double beta, const double *y, double *z,
                         cudaStream_t s);
// NVLink peer-memory exchange (CUDA IPC mappings; see kernels.cu)
// phase: 1 = push, 2 = pull, 3 = both (see vec.cu)
cudaError_t launch_red_exchange(int channel, const P2PMail &M, const double *red_loc, double *red_all, int phase,
                                cudaStream_t s);
template <class T>
cudaError_t launch_gs_pack_p2p_fused(const int32_t *perm, const int32_t *offs, const T *v, T *partial,
                                     int64_t nslots, const int32_t *send_run, const int32_t *slot_nbr,
                                     double *const *peer_recv, const int64_t *remote_off, const int64_t *send_offs,
                                     const int64_t *remote_half, int nnbr, int me, uint64_t *const *peer_hflags,
                                     uint64_t *epochs, unsigned int *counter, const int *done, cudaStream_t s,
                                     const int4 *pack4 = nullptr);

cudaError_t launch_pcg_init_fin(PcgScalars *sc, const double *red_all, int nranks, double *hist, cudaStream_t s);
cudaError_t launch_pcg_update(int64_t n, const uint32_t *obits, const double *dinv, const double *p,
                              const double *w, double *x, double *r, const double *red_all, int nranks,
                              PcgScalars *sc, double *part, int nblk, double *dst, unsigned int *counter,
                              cudaStream_t s);
cudaError_t launch_pcg_pupdate(int64_t n, const double *dinv, const double *r, double *p, const double *red_all,
                               int nranks, PcgScalars *sc, double *hist, unsigned int *counter, int nblk,
                               cudaStream_t s);
int vec_blocks();
int upd_blocks();
int upd_blocks_deferred();   // CTAs of the single-rank deferred residual update
int device_sms();   // multiprocessors of the current device (cached per device)

// makef.cu: dealiased advection (NEXT #4)
int makef_lattice(int N);
cudaError_t makef_upload(int N);
cudaError_t launch_makef_geom(int N, int64_t E, const double *xyz, double *G9, unsigned long long *bad, cudaStream_t s);
cudaError_t launch_makef(int N, int64_t E, const double *G9, const double *u0, const double *u1, const double *u2,
                         double *f0, double *f1, double *f2, cudaStream_t s);

// pmg_kernels.cuh
template <class T>
cudaError_t launch_prolong_add(int64_t E, int Nc, int Nf, const T *J, const T *ec, T *uf, const int *done,
                               cudaStream_t s);
template <class T>
cudaError_t launch_restrict(int64_t E, int Nf, int Nc, const T *J, const T *rf, const uint32_t *obits, T *fc,
                            const int *done, cudaStream_t s);
template <class T>
cudaError_t launch_cheb(int mode, int64_t n, const T *dinv, const T *f, const T *w, double theta, double c1,
                        double c2, T *d, T *x, T *r, const int *done, cudaStream_t s);
template <class Ti, class To>
cudaError_t launch_convert(int64_t n, const Ti *in, To *out, const int *done, cudaStream_t s);
cudaError_t launch_geom_to_f32(int64_t E, int N, const double *G, float *Gf, cudaStream_t s);
cudaError_t launch_dot_owner(int64_t n, const uint32_t *obits, const double *a, const double *b, double *part,
                             int nblk, double *dst, unsigned int *counter, const int *done, cudaStream_t s);
cudaError_t launch_pcg_pupdate_z(int64_t n, const double *z, double *p, const double *red_all, int nranks,
                                 PcgScalars *sc, double *hist, unsigned int *counter, int nblk, cudaStream_t s);
cudaError_t launch_lanczos_rz(int64_t n, double alpha, const double *w, const double *dinv, double *r, double *z,
                              cudaStream_t s);
}  // namespace nekb200

struct nek_ctx {
    int device = 0;
    int64_t E = 0;
    int N = 0, Nq = 0, P3 = 0;
    int64_t n = 0;
    int rank = 0, nranks = 1;
    ncclComm_t nccl = nullptr;
    cudaStream_t s_main = nullptr, s_comm = nullptr, s_hi = nullptr;   // s_hi: high priority (boundary work)
    cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_fork2 = nullptr, ev_bnd = nullptr;
    cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
    nek_plan *plan = nullptr;
    int variant = 0;
    // geometry
    double *G = nullptr, *wJ = nullptr;
    double min_jac = 0.0;
    // maps (device)
    int32_t *perm = nullptr, *offs = nullptr;
    int64_t nruns = 0, nperm = 0;
    int32_t *gs_p2 = nullptr, *gs_p4 = nullptr, *gs_p8 = nullptr, *gs_pg = nullptr, *gs_og = nullptr;
    int32_t *gs_coff = nullptr;   // element-chunk offsets of the classes (GsClasses::coff)
    int l2keep = 0;                                 // L2-resident PCG vectors (AxLaunch::keep bits)
    bool bnd_split = true;                          // concurrent boundary/interior Ax share one wave of CTAs
    int bnd_epc = 0;                                // boundary elements per boundary CTA (NEK_BND_EPC; 0 = model)
    bool defer = true;                              // deferred reductions on the single-rank v5 path (NEK_DEFER)
    int64_t v5_pf_min = 16384;                      // AxLaunch::pf_min (NEK_V5_PF_MIN)
    double *upart = nullptr;                        // [upd_blocks][4] update partials the next Ax folds
    int64_t l2_setaside = 0, l2_setaside_max = 0;   // persisting L2 bytes granted / allowed
    bool concurrent_bnd = false;
    bool owns_streams = true, owns_nccl = true;   // false for the internal pMG level contexts
    nekb200::GsClasses gsc;
    int32_t *ifc_perm = nullptr, *ifc_offs = nullptr, *send_run = nullptr, *coffs = nullptr, *contrib = nullptr;
    int32_t *pack4 = nullptr;   // [nslots][4] local copies of each send slot's run (-1 pad; x = -2: > 4 copies)
    int64_t nifc = 0, nifc_perm = 0, nslots = 0;
    std::vector<int32_t> neighbors;
    std::vector<int64_t> send_offs;
    double *ifc_partial = nullptr, *sendbuf = nullptr, *recvbuf = nullptr;
    int32_t *elist = nullptr;
    int64_t n_boundary = 0, n_masked = 0;
    uint32_t *mbits = nullptr, *obits = nullptr;
    // work vectors
    double *vr = nullptr, *vp = nullptr, *vw = nullptr, *vx = nullptr, *vdinv = nullptr, *vtmp = nullptr;
    double *stage_in = nullptr, *stage_out = nullptr;
    double *part = nullptr;       // block partials (max of Ax and vector kernels)
    int64_t npart = 0;
    double *red_loc = nullptr, *red_all = nullptr;
    nekb200::PcgScalars *sc = nullptr, *sc_host = nullptr;
    unsigned int *counter = nullptr;   // [0] pupdate, [1] Ax, [2] init/update
    double *hist = nullptr;
    int64_t hist_cap = 0;
    // Jacobi cache
    bool dinv_valid = false;
    double dinv_h1 = 0, dinv_h2 = 0;
    // graph cache
    cudaGraphExec_t graph = nullptr;
    int graph_iters = 0;
    double graph_h1 = 0, graph_h2 = 0;
    nek_stats_t graph_stats{};
    bool graph_timing = false, capturing = false;
    std::vector<nekb200::TimedLaunch> graph_timers;   // event-record nodes of the timing graph
    // NVLink peer-memory path (nranks > 1, all peers mapped)
    bool p2p = false;
    double *mbox = nullptr;                 // [2 channels][2 parities][nranks][4]
    double **d_peer_mbox = nullptr;         // [nranks]
    uint64_t *epochs = nullptr;             // [4]: channel 0, channel 1, halo pack, halo wait
    int *p2p_err = nullptr;                 // device view of p2p_err_host (mapped pinned host memory)
    int *p2p_err_host = nullptr;            // raised by a timed-out peer wait; sticky (epochs are then out of step)
    uint64_t p2p_timeout_ns = 10000000000ull;
    // loopback group (P virtual ranks on one GPU, loopback.h)
    nekb200::LoopGroup *lb = nullptr;
    cudaEvent_t ev_lb[2] = {nullptr, nullptr};
    unsigned lb_seq = 0;
    std::vector<const double *> lb_halo_src;   // staged transport: each neighbour's send slots for this rank
    double *recv2 = nullptr;                // 2 x nslots halo receive buffer (P2P)
    double **d_peer_recv = nullptr;         // [nnbr]
    int64_t *d_remote_off = nullptr, *d_send_offs = nullptr, *d_remote_half = nullptr;
    int32_t *d_slot_nbr = nullptr, *d_nbr = nullptr;
    uint64_t *hflags = nullptr;             // [nranks], written by neighbours
    uint64_t **d_peer_hflags = nullptr;     // [nnbr]
    std::vector<void *> ipc_opened;
    // stats
    bool timing = false;
    nek_stats_t stats{};
    int64_t device_bytes = 0;
    std::string err;
};
