/*
 * nek.h -- C ABI of the B200-native SEM hot path (arXiv 2409.19119, NekRS).
 *
 * What it computes (PAPER.md = P:n, SPEC.md = S:n, readings = R#):
 *   - the matrix-free spectral-element Helmholtz operator on hexahedra of order
 *     N with GLL points,  w_e = h1 * D^T G_e D u_e + h2 * (wJ)_e u_e
 *     (Eq. 3 and "fast tensor contractions ... O(N^4) work and
 *     O(N^3) memory references"; P:148-151 the pressure Poisson system);
 *   - the gather-scatter QQ^T (direct stiffness summation; "C0
 *     continuity implies ... unit-depth stencils"), on one GPU and across GPUs
 *     as an NCCL halo exchange overlapped with interior-element work
 *     (P:391-398);
 *   - Jacobi-preconditioned conjugate gradients with device-side
 *     scalars and one reduction exchange per dot-product group.
 * All arithmetic is FP64.
 *
 * Conventions common to every call:
 *   E-vector: a field stored per element, length n_local = E*(N+1)^3, local
 *   index l = e*(N+1)^3 + i + (N+1)*j + (N+1)^2*k, i (the r direction) fastest
 *   ("local i-j-k indexing").
 *   Field pointers (u, w, v, b, x) may be DEVICE pointers on the context's
 *   device (used in stream order on `stream`, no host synchronisation) or HOST
 *   pointers (pageable or pinned; the call then stages them through internal
 *   device buffers and returns after the result is back in host memory).
 *   `stream` is a cudaStream_t (NULL = the legacy default stream).
 *   Multi-GPU (comm->nranks > 1): one process per GPU; every call below that
 *   takes a context is COLLECTIVE -- all ranks make the same calls in the same
 *   order.  Each rank passes only its own elements; a
 *   node shared between ranks carries the same gid on every rank.
 *   Ownership: the caller owns every array it passes; setup inputs are copied
 *   (they may be freed after nek_setup returns); the library owns all internal
 *   device memory until nek_free.  A context is not thread-safe.
 *   Errors: every call returns a status code (never throws, never exits);
 *   the message of the last failure is available from nek_errmsg(ctx), or from
 *   nek_last_error() when no context exists.
 */
#ifndef NEK_H
#define NEK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NEK_ABI_VERSION 1

typedef struct nek_ctx nek_ctx;

/* Status codes (SURVEY 8(b) error table). */
enum {
    NEK_OK = 0,        /* success                                                        */
    NEK_MAXIT = 1,     /* PCG reached maxit; x holds the last iterate -- not an error */
    NEK_EINVAL = -1,   /* bad argument (null pointer, E < 0, bad rank/size, ...)         */
    NEK_EORDER = -2,   /* N outside [1, 15]                                      */
    NEK_EGEOM = -3,    /* Jacobian J <= 0 at some node; message names element and node */
    NEK_ETOPO = -4,    /* copies of one gid with different coordinates (> 1e-9 * diameter)
                          or different Dirichlet flags             */
    NEK_ENOTSPD = -5,  /* PCG found <p, A p> <= 0                                */
    NEK_ENOMEM = -6,   /* device or host allocation failed                               */
    NEK_ECUDA = -7,    /* CUDA runtime error (message has the CUDA error string)          */
    NEK_ENCCL = -8,    /* NCCL error                                                     */
    NEK_ENODEV = -9    /* no CUDA device / the library was built without this arch      */
};

/* Communicator for multi-GPU runs.  nranks == 1 (or a NULL comm) = single GPU,
 * no NCCL.  nccl_id: the 128-byte ncclUniqueId produced on rank 0 by
 * nek_comm_unique_id and broadcast to every rank by the caller (the Python
 * binding uses torch.distributed).  An id bootstraps exactly one communicator:
 * every nek_setup with nranks > 1 needs a fresh id. */
typedef struct {
    int rank;
    int nranks;
    unsigned char nccl_id[128];
} nek_comm;

/*
 * Loopback group: P virtual ranks in ONE process on ONE GPU (SURVEY 4 "loopback comm backend";
 * SPEC S:196/S:235 runs its ranks under one scheduler), so the multi-rank path -- the halo exchange
 * of interface partial sums (unit-depth exchange), its overlap with interior-element work
 * and the rank-ordered reductions -- runs and is testable on a single GPU.
 *   nek_loopback_create  nranks in [1, 64]; transport 0 = the peer-memory kernels of the NVLink
 *                        path (halo pack into the neighbour's receive buffer, flag/epoch waits,
 *                        mailbox reductions), 1 = the NCCL-path kernels (pack / unpack around a
 *                        staged copy).  Returns NEK_OK / NEK_EINVAL / NEK_ENOMEM.
 *   nek_loopback_comm    fills *comm for `rank` (rank, nranks and a tag in nccl_id that names
 *                        the group); pass it to nek_setup like an NCCL communicator.
 *   nek_loopback_abort   makes every pending and later group barrier fail (NEK_ENCCL), e.g.
 *                        when one rank's thread stops early.
 *   nek_loopback_free    after every context of the group has been freed.
 * Each rank is driven by its own host thread, making the same calls as a one-process-per-GPU
 * rank would.  Inside the library every step that consumes another rank's data waits (stream
 * events swapped through the group) for that rank's producer, so no kernel spins on a rank that
 * has not launched; PCG iterations are launched directly rather than from a CUDA graph.
 * Barriers time out after NEK_LOOPBACK_TIMEOUT_S seconds (default 60).  The group object is
 * owned by the caller and must outlive its contexts.
 */
typedef struct nek_loopback nek_loopback;
int nek_loopback_create(int nranks, int transport, nek_loopback **out);
int nek_loopback_comm(nek_loopback *lb, int rank, nek_comm *comm);
int nek_loopback_abort(nek_loopback *lb);
int nek_loopback_free(nek_loopback *lb);

int nek_version(void);                 /* returns NEK_ABI_VERSION */
const char *nek_last_error(void);      /* message of the last failure without a context (thread-local) */

/* Fill id[128] with a fresh NCCL unique id (call on rank 0 only).
 * Returns NEK_OK or NEK_ENCCL. */
int nek_comm_unique_id(unsigned char id[128]);

/*
 * nek_setup -- build a context for E local elements of order N.
 *   xyz       HOST, [3][E*(N+1)^3] FP64: x, y, z of every GLL node of every
 *             element (BASELINE north_star "vertex coordinates", read as all
 *             GLL nodes -- R1; isoparametric map P:175-178).
 *   gid       HOST, [E*(N+1)^3] int64 >= 0: global node id, equal on all copies
 *             of a node (on all ranks).
 *   dirichlet HOST, [E*(N+1)^3] uint8 or NULL: 1 = homogeneous Dirichlet node;
 *             must agree on all copies (R6).
 *   comm      NULL or nranks == 1 for one GPU; else see nek_comm.
 *   device    CUDA device ordinal for this rank.
 *   stream    stream for the setup kernels.
 * Setup computes, on the device: the GLL rule and derivative matrix,
 * the 6 symmetric geometric factors plus the Jacobian weight per point
 * (G_ab = w_q J grad r_a . grad r_b, wJ = w_q J, R4), the canonical
 * gather-scatter maps (R7) and, for nranks > 1, the halo plan (one setup
 * collective: an allgather of element-surface gids).
 * On success *out holds the context; on failure *out is NULL and the status is
 * one of EINVAL, EORDER, EGEOM, ETOPO, ENOMEM, ECUDA, ENCCL, ENODEV.
 */
int nek_setup(nek_ctx **out, int64_t E, int N, const double *xyz, const int64_t *gid,
              const uint8_t *dirichlet, const nek_comm *comm, int device, void *stream);

/*
 * nek_ax -- w = M QQ^T (h1 K_L + h2 B_L) M u  (R5, R6): the local stiffness
 * apply sum_ab D_a^T G_ab D_b u_e plus h2 wJ u, the gather-scatter
 * (local runs and, for nranks > 1, the halo exchange overlapped with the Ax of
 * interior elements) and the Dirichlet mask on both sides.
 * u and w: E-vectors (device or host), must not alias.
 */
int nek_ax(nek_ctx *ctx, double h1, double h2, const double *u, double *w, void *stream);

/*
 * nek_gs -- v <- QQ^T v in place (global over all ranks).
 * Copies of a node are summed left to right in ascending local index, and
 * across ranks in ascending rank order (R7), so every copy on every rank gets
 * identical bits; at nranks == 1 the result is bit-identical to the oracle.
 */
int nek_gs(nek_ctx *ctx, double *v, void *stream);

/*
 * nek_pcg_solve -- Jacobi-preconditioned CG for (h1 K + h2 B) x = b on the
 * masked subspace, Hestenes-Stiefel form:
 *   x0 = 0, r0 = M b, z = Dinv r, p = z, rho = <r,z>
 *   repeat: stop if ||r|| <= tol ||M b||; w = A p; sigma = <p,w>; alpha = rho/sigma;
 *           x += alpha p; r -= alpha w; rho' = <r, Dinv r>; beta = rho'/rho; p = Dinv r + beta p
 * Dinv = M / diag(QQ^T (h1 K_L + h2 B_L)) uses the exact assembled diagonal (R10).
 * <.,.> is the owner-copy inner product over unique global nodes (R8).
 *   b, x      E-vectors (device or host); x is overwritten (x0 = 0, R11).
 *   tol       relative residual tolerance (R9); tol = 0 runs exactly maxit iterations.
 *   maxit     iteration cap (>= 0).
 *   iters     out (host, nullable): iterations performed.
 *   relres    out (host, nullable): ||r_k|| / ||M b|| at exit.
 *   hist      out (host, nullable): maxit+1 entries, hist[k] = ||r_k||/||M b|| for k <= iters.
 * Returns NEK_OK (converged; also b = 0 -> x = 0, iters = 0), NEK_MAXIT,
 * NEK_ENOTSPD (x holds the last iterate), or an error.  The call synchronises
 * `stream` (convergence is polled from the device after every CUDA-graph replay of
 * 20 iterations; iterations past convergence return at kernel entry).
 * Schedule (reading 25): the bookkeeping of iteration k (beta, the history
 * entry, the convergence and maxit tests) runs at the start of the iteration-(k+1)
 * operator launch, from the residual update's partial sums -- the same values as a
 * separate bookkeeping step; NEK_DEFER=0 restores the separate step.
 * L2 residency: when the PCG vectors fit in the L2 (nek_info_t.l2_keep), the
 * call raises the DEVICE-WIDE persisting-L2 limit (cudaLimitPersistingL2CacheSize)
 * for its duration and restores the previous value before returning; kernels of
 * other contexts running concurrently on the device see a smaller normal L2.
 * Multi-rank: a peer wait that times out (NEK_P2P_TIMEOUT_MS, default 10 s)
 * returns NEK_ENCCL; the error is sticky -- every later call on the context
 * returns NEK_ENCCL and the context must be rebuilt.  nek_ax / nek_gs on device
 * pointers report such a timeout at the next call (their results hold NaN in the
 * affected entries instead of stale data).
 */
int nek_pcg_solve(nek_ctx *ctx, double h1, double h2, const double *b, double *x, double tol,
                  int maxit, int *iters, double *relres, double *hist, void *stream);

/* Release every resource of the context (collective for nranks > 1). NULL is a no-op. */
int nek_free(nek_ctx *ctx);

/* Message of the context's last failure ("" if none).  Valid until the next call. */
const char *nek_errmsg(const nek_ctx *ctx);

/* ------------------------------------------------ projection initial guess */
/*
 * Fischer's projection onto prior solutions (P:513-519
 * "generate an initial guess ... by projecting onto the space of prior
 * solutions", "increasing the number of prior solutions from 8 to 30";
 * S:344-347).  A space holds up to max_vectors (<= 32)
 * A-orthonormal vectors x_i and their images A x_i (2 * max_vectors E-vectors
 * of device memory).  nek_proj_solve(b):
 *   alpha_i = <x_i, M b>; xbar = sum alpha_i x_i; db = M b - sum alpha_i A x_i;
 *   Jacobi-PCG on A dx = db to ||r|| <= tol ||M b||; x = xbar + dx;
 *   then dx is A-orthonormalised against the space (classical Gram-Schmidt,
 *   twice) and appended; when the space is full it restarts from x alone.
 * The space is reset when (h1, h2) changes.  iters = PCG iterations on db;
 * relres = ||r|| / ||M b||.  Collective for nranks > 1.  Status as
 * nek_pcg_solve.  max_vectors = 0 gives plain PCG.
 */
typedef struct nek_proj nek_proj;
int nek_proj_create(nek_ctx *ctx, int max_vectors, nek_proj **out);
int nek_proj_solve(nek_proj *proj, double h1, double h2, const double *b, double *x, double tol, int maxit,
                   int *iters, double *relres, void *stream);
int nek_proj_size(const nek_proj *proj);      /* vectors currently in the space */
int nek_proj_reset(nek_proj *proj);
int nek_proj_free(nek_proj *proj);

/* ------------------------------------------- p-multigrid preconditioned CG */
/*
 * p-multigrid V-cycle with Chebyshev smoothing as the preconditioner of the same
 * Hestenes-Stiefel PCG ("local smoothers for
 * p-multigrid", "p-multigrid schedules of p=7, 5, 3, and 1 with
 * 6th-order Chebyshev smoothing").  DESIGN.md readings P1-P7:
 *   levels    orders[0] = N > orders[1] > ... > orders[nlevels-1] = 1 (default
 *             [N,5,3,1] for N >= 7, [N,3,1] for 4 <= N < 7, [N,1] for N = 2, 3);
 *             each coarse level re-discretises the same elements: GLL-node
 *             coordinates interpolated from `xyz` (the array given to nek_setup),
 *             node ids keyed by mesh entities of the fine ids, the fine mask
 *             carried over (it must be constant on every edge / face interior:
 *             a union of closed boundary faces, else NEK_EINVAL);
 *   transfer  prolongation J x J x J per element; restriction its transpose
 *             applied to the owner copies, then QQ^T and the mask of the level;
 *   smoother  Chebyshev (Saad Alg. 12.1) of `degree` with Jacobi on
 *             [lmin_frac lam, lmax_factor lam], lam the largest Ritz value of
 *             `lanczos_steps` Jacobi-PCG steps from M hash(gid);
 *   coarse    Chebyshev of `coarse_degree` on [coarse_lo lam_min, lmax_factor lam]
 *             of the order-1 level (no host solver);
 *   V-cycle   x = S(f); r = f - A x; e = V(R r); x += P e; x = x + S(f - A x).
 * All levels run on the context's device and streams; for nranks > 1 every call
 * is collective and each level exchanges its own halo like the fine operator.
 * (h1, h2) are fixed at creation (eigenvalue bounds and diagonals depend on them).
 * Zero-valued option fields take the defaults in brackets: degree [6],
 * coarse_degree [20], lmin_frac [0.1], lmax_factor [1.1], coarse_lo [1.0],
 * lanczos_steps [20], nlevels [0 = default schedule].
 * nek_pmg_apply:  z = V(r), r and z E-vectors (device or host), not aliasing.
 * nek_pmg_solve:  PCG on A x = M b with z = V(r); arguments, stopping rule and
 *                 status as nek_pcg_solve.
 */
#define NEK_PMG_MAX_LEVELS 8
typedef struct nek_pmg nek_pmg;
typedef struct {
    int32_t nlevels;
    int32_t orders[NEK_PMG_MAX_LEVELS];
    int32_t degree, coarse_degree, lanczos_steps;
    double lmin_frac, lmax_factor, coarse_lo;
    int32_t precision;         /* 0: FP64; 1: FP32 preconditioner (NEXT #3):
                                  every level's metric factors, diagonal, transfer matrix
                                  and work vectors in single precision, r converted on
                                  entry and z on exit; the outer CG stays FP64; N <= 9 */
} nek_pmg_opts;
typedef struct {
    int32_t nlevels;
    int32_t orders[NEK_PMG_MAX_LEVELS];
    int32_t degree, coarse_degree, precision;
    int64_t n_local[NEK_PMG_MAX_LEVELS];
    double lam_min[NEK_PMG_MAX_LEVELS], lam_max[NEK_PMG_MAX_LEVELS];
    int64_t vcycles;           /* V-cycles applied so far                         */
} nek_pmg_info_t;
int nek_pmg_create(nek_ctx *ctx, const double *xyz, double h1, double h2, const nek_pmg_opts *opts, nek_pmg **out,
                   void *stream);
int nek_pmg_apply(nek_pmg *pmg, const double *r, double *z, void *stream);
int nek_pmg_solve(nek_pmg *pmg, const double *b, double *x, double tol, int maxit, int *iters, double *relres,
                  double *hist, void *stream);
int nek_pmg_info(const nek_pmg *pmg, nek_pmg_info_t *info);
int nek_pmg_free(nek_pmg *pmg);

/* ------------------------------------------------- dealiased advection makef */
/*
 * The nonlinear advection term of the velocity (P:417-420
 * "dealiased using N_q=11 quadrature points in each direction", "dealiased
 * with the 3/2's rule, the working data set per element is 12^3").
 * DESIGN.md readings M1-M4: per element, component c and GLL node l
 *   F_c(l) = - sum_q rho_q J_q phi_l(xi_q) (u . grad u_c)(xi_q)
 * on the M^3 Gauss-Legendre lattice, M = ceil(3(N+1)/2) (N = 7: M = 12), with u and
 * grad u_c from the order-N interpolant and J, dr/dx from the isoparametric map of `xyz`
 * (the nek_setup coordinates).  Output is LOCAL (unassembled, unmasked) E-vectors: apply
 * nek_gs (and a mask) as for any right-hand side.
 * nek_makef_create: M = 0 or the 3/2-rule value (else NEK_EINVAL); N <= 9 (NEK_EORDER);
 *   stores 9 M^3 FP64 factors per element (rho J dr_a/dx_b); J <= 0 at a lattice point ->
 *   NEK_EGEOM.  nek_makef_apply: u, v, w in, fu, fv, fw out (E-vectors, device or host,
 *   outputs must not alias inputs).  Element-local: no communication for nranks > 1.
 */
typedef struct nek_makef nek_makef;
int nek_makef_create(nek_ctx *ctx, const double *xyz, int M, nek_makef **out, void *stream);
int nek_makef_apply(nek_makef *mk, const double *u, const double *v, const double *w, double *fu, double *fv,
                    double *fw, void *stream);
int nek_makef_lattice(const nek_makef *mk);
int nek_makef_free(nek_makef *mk);

/* Measurement probe: FP64 FMA throughput of `device` in TFLOP/s (register-only FMA chains,
 * SURVEY 8(d)); the compute roofline denominator of makef. */
int nek_probe_dfma_tflops(int device, double *tflops);

/* Measurement probes (SURVEY 8(d) "Peaks to measure on the box"), not on the solver path:
 * FP64 streaming bandwidth of `device` over `bytes` (>= 1 MiB; split into two buffers): a double2
 * read-only kernel, a write-only kernel and a read+write copy (copy counts both directions), best of
 * five after a warm-up, in GB/s; outputs may be NULL.  NEK_EINVAL for bytes < 1 MiB, NEK_ENOMEM if
 * the buffers do not fit.  nek_probe_smem_tbps: aggregate conflict-free ld.shared.f64 bandwidth in
 * TB/s (two 1024-thread CTAs per SM). */
int nek_probe_hbm_gbps(int device, int64_t bytes, double *read_gbps, double *write_gbps, double *copy_gbps);
int nek_probe_smem_tbps(int device, double *tbps);

/* ----------------------------------------------------------- introspection */
typedef struct {
    int64_t E;                 /* local elements                                   */
    int32_t N;                 /* polynomial order                                 */
    int32_t rank, nranks;
    int64_t n_local;           /* E*(N+1)^3                                        */
    int64_t n_dof;             /* E*N^3, the paper's resolution count     */
    int64_t n_masked;          /* local Dirichlet nodes                            */
    int64_t n_runs;            /* local shared runs (local-only runs at nranks > 1) */
    int64_t n_perm;            /* local copies in those runs                       */
    int64_t n_ifc_runs;        /* runs whose gid is also on another rank           */
    int64_t n_ifc_perm;        /* local copies in interface runs                   */
    int64_t n_neighbors;       /* ranks sharing at least one gid with this rank    */
    int64_t halo_doubles;      /* FP64 values sent (= received) per gather-scatter */
    int64_t n_boundary_elems;  /* elements holding at least one interface node     */
    int64_t device_bytes;      /* device memory held by the context                */
    double  geom_min_jac;      /* min J over local nodes                           */
    int32_t transport;         /* 0 = single GPU, 1 = NCCL, 2 = NVLink peer memory (CUDA IPC) */
    int32_t l2_keep;           /* L2-resident PCG vectors: bit 0 p, r, Dinv, w, gs lists; bit 1 x  */
    int64_t l2_setaside;       /* persisting-L2 bytes in effect (device-wide limit)               */
    int64_t l2_setaside_max;   /* cudaDevAttrMaxPersistingL2CacheSize                            */
} nek_info_t;

int nek_get_info(const nek_ctx *ctx, nek_info_t *info);

/* Copy the canonical local gather-scatter map to host arrays (R7):
 * perm[n_perm] (int32 local indices, runs back to back), offs[n_runs+1]. */
int nek_get_gs_map(const nek_ctx *ctx, int32_t *perm, int64_t *offs);

/* Copy the geometric factors to host: G[E][6][(N+1)^3] (rr, rs, rt, ss, st, tt),
 * wJ[E*(N+1)^3]. Either pointer may be NULL. */
int nek_get_geom(const nek_ctx *ctx, double *G, double *wJ);

/* Jacobi inverse diagonal Dinv = M / diag(QQ^T (h1 K_L + h2 B_L)) into an
 * E-vector (device or host). */
int nek_get_dinv(nek_ctx *ctx, double h1, double h2, double *dinv, void *stream);

/* Per-kernel device timing (CUDA events on the library's stream).  When on,
 * every kernel class launched by nek_ax / nek_gs / nek_pcg_solve is bracketed
 * by events and its duration accumulated; nek_get_stats reads (and optionally
 * resets) the totals.  Launch counts are always accumulated. */
typedef struct {
    double  ax_ms, gs_ms, halo_ms, vec_ms;    /* summed device time per kernel class */
    int64_t ax_launches, gs_launches, halo_launches, vec_launches;
    int64_t launches;                          /* all kernels launched by the library */
    int64_t ax_elements;                       /* elements processed by Ax launches  */
    double  ax_bytes;                          /* algorithmic HBM bytes of those launches */
    double  axu_ms;                            /* nranks > 1: device time of each operator's whole Ax phase
                                                  (boundary launch, halo send and interior launch, which
                                                  overlap on two streams), from its first start to its
                                                  last end -- the union time of those launches   */
    int64_t axu_spans;                         /* Ax phases timed in axu_ms                            */
} nek_stats_t;

int nek_set_timing(nek_ctx *ctx, int on);
int nek_get_stats(nek_ctx *ctx, nek_stats_t *stats, int reset);

/* Ax kernel variant selection (0 = default).  For experiments and tests; other values -> NEK_EINVAL.
 *   0  default: N = 7 -> v5 (DMMA k-slabs, fused PCG prologue; TMA metric ring at 3 CTAs/SM for
 *      launches of <= 16 elements per CTA, register streaming at 4 CTAs/SM otherwise); N <= 9
 *      otherwise -> v6 (TMA-staged metric ring, line-wise contractions, fused prologue); N >= 10 -> v0
 *   1  v0 (any N, (i,j)-thread columns)       11  v6 at any N <= 9 (N = 7 included)
 *   8  v5 register streaming at 3 CTAs/SM      10  v5 TMA metric ring at 3 CTAs/SM
 *   12 v5 register streaming at 4 CTAs/SM (any size); for N != 7, 8/10/12 run v0 */
int nek_set_variant(nek_ctx *ctx, int ax_variant);

/* --------------------------------------------- host-only planning (no GPU) */
/*
 * The gather-scatter / halo plan is built by host code that needs no device;
 * these calls expose it so multi-rank logic can be tested on CPU.
 *
 * nek_plan_create: local maps for E elements of order N (same inputs as
 *   nek_setup; xyz may be NULL to skip the coordinate check).
 * nek_plan_surface_gids: sorted unique gids on element surfaces; returns the
 *   count, fills out[] when non-NULL.  These are what nek_setup allgathers.
 * nek_plan_set_ranks: give rank/nranks and every rank's surface-gid list
 *   (counts[nranks], lists[nranks] -> sorted int64 arrays); builds the halo plan.
 * nek_plan_size / nek_plan_get: size (in elements) and contents of plan arrays:
 */
typedef struct nek_plan nek_plan;
enum {
    NEK_PLAN_PERM = 0,        /* int32  local-only run copies (canonical order)           */
    NEK_PLAN_OFFS = 1,        /* int64  local-only run offsets (n_runs+1)                 */
    NEK_PLAN_IFC_PERM = 2,    /* int32  interface run copies                              */
    NEK_PLAN_IFC_OFFS = 3,    /* int64  interface run offsets (n_ifc_runs+1)              */
    NEK_PLAN_IFC_GID = 4,     /* int64  gid of each interface run                         */
    NEK_PLAN_NEIGHBORS = 5,   /* int32  neighbour ranks, ascending                        */
    NEK_PLAN_SEND_OFFS = 6,   /* int64  per-neighbour offsets into the send/recv slots    */
    NEK_PLAN_SEND_RUN = 7,    /* int32  interface run packed into each send slot          */
    NEK_PLAN_CONTRIB_OFFS = 8,/* int64  per interface run offsets into CONTRIB            */
    NEK_PLAN_CONTRIB = 9,     /* int32  summands in ascending rank order: -1 = own partial,
                                         s >= 0 = received slot s                         */
    NEK_PLAN_OWNER = 10,      /* uint8  1 on the owner copy of every local node (R8)      */
    NEK_PLAN_ELEM_ORDER = 11  /* int32  elements, boundary ones first                     */
};
int nek_plan_create(nek_plan **out, int64_t E, int N, const int64_t *gid, const uint8_t *dirichlet,
                    const double *xyz);
int64_t nek_plan_surface_gids(const nek_plan *plan, int64_t *out);
int nek_plan_set_ranks(nek_plan *plan, int rank, int nranks, const int64_t *counts,
                       const int64_t *const *lists);
int64_t nek_plan_size(const nek_plan *plan, int what);
int nek_plan_get(const nek_plan *plan, int what, void *out);
const char *nek_plan_errmsg(const nek_plan *plan);
void nek_plan_free(nek_plan *plan);

#ifdef __cplusplus
}
#endif
#endif /* NEK_H */
