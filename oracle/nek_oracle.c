/*
 * nek_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct CPU implementation of the hot path of
 * arXiv 2409.19119 (NekRS): GLL rule, derivative matrix, geometric factors,
 * the matrix-free SEM Poisson/Helmholtz operator, the gather-scatter QQ^T
 * (direct stiffness summation), the Dirichlet mask, the exact Jacobi diagonal
 * and Jacobi-preconditioned CG.  FP64 throughout ("All reported
 * FLOPS are for FP64").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code, header, table or helper with the CUDA
 * library under paper_2409_19119_b200/; neither includes the other.
 *
 * Citation key: P:n = PAPER.md line n; S:n = SPEC.md line n; "reading k" =
 * DESIGN.md section "Readings of the paper", item k.
 *
 * Parity pins: every function here is pinned by tests/test_oracle_*.py
 * against closed forms, invariants, an independent brute-force assembler
 * (oracle/assemble.py) or a dense solve -- see DESIGN.md "Oracle pins".
 */
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ GLL --- */
/* Legendre P_n(x) and its derivative by the three-term recurrence. */
static void legendre(int n, double x, double *p, double *dp)
{
    double p0 = 1.0, p1 = x, d0 = 0.0, d1 = 1.0;
    if (n == 0) { *p = 1.0; *dp = 0.0; return; }
    for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        double d2 = d0 + (2.0 * k - 1.0) * p1;   /* P_k' = P_{k-2}' + (2k-1) P_{k-1} */
        p0 = p1; p1 = p2; d0 = d1; d1 = d2;
    }
    *p = p1; *dp = d1;
}

/* q(x) = (1 - x^2) P_N'(x); its roots are the GLL nodes.  q'(x) = -N(N+1) P_N(x)
 * by Legendre's equation. */
static double gll_q(int N, double x, double *dq)
{
    double p, dp;
    legendre(N, x, &p, &dp);
    *dq = -(double)N * (N + 1) * p;
    return (1.0 - x * x) * dp;
}

/*
 * or_gll: the N+1 Gauss-Lobatto-Legendre nodes (ascending) and weights.
 * P:183-186 (Eq. 3: "Gauss-Lobatto-Legendre quadrature points").
 * Nodes: roots of (1-x^2) P_N'(x), found by Newton from Chebyshev-Gauss-Lobatto
 * guesses with a bisection fallback, then symmetrised.
 * Weights: w_i = 2 / (N (N+1) P_N(x_i)^2).
 * Returns 0, or -1 for N outside [1, 15].
 */
int or_gll(int N, double *x, double *w)
{
    if (N < 1 || N > 15) return -1;
    x[0] = -1.0; x[N] = 1.0;
    for (int i = 1; i < N; ++i) {
        /* bracket: interior GLL nodes interlace the CGL guesses well enough; use
         * a bracket between neighbouring CGL points shifted half a step. */
        double g = -cos(M_PI * i / N);
        double lo = -cos(M_PI * (i - 0.5) / N), hi = -cos(M_PI * (i + 0.5) / N);
        double t = g;
        int ok = 0;
        for (int it = 0; it < 100; ++it) {
            double dq, q = gll_q(N, t, &dq);
            double tn = t - q / dq;
            if (!(tn > lo && tn < hi)) break;
            if (fabs(tn - t) <= 1e-16) { t = tn; ok = 1; break; }
            t = tn;
        }
        if (!ok) {  /* bisection fallback on [lo, hi] */
            double dq, qlo = gll_q(N, lo, &dq);
            for (int it = 0; it < 200; ++it) {
                double mid = 0.5 * (lo + hi), qm = gll_q(N, mid, &dq);
                if ((qm < 0) == (qlo < 0)) { lo = mid; qlo = qm; } else hi = mid;
            }
            t = 0.5 * (lo + hi);
            for (int it = 0; it < 3; ++it) { double q = gll_q(N, t, &dq); t -= q / dq; }
        }
        x[i] = t;
    }
    for (int i = 0; i <= N / 2; ++i) {        /* symmetrise: x_{N-i} = -x_i */
        double s = 0.5 * (x[N - i] - x[i]);
        x[N - i] = s; x[i] = -s;
    }
    if (N % 2 == 0) x[N / 2] = 0.0;
    for (int i = 0; i <= N; ++i) {
        double p, dp;
        legendre(N, x[i], &p, &dp);
        w[i] = 2.0 / ((double)N * (N + 1) * p * p);
    }
    return 0;
}

/*
 * or_deriv: D[i][j] = h_j'(x_i), the derivative of the j-th Lagrange cardinal
 * function on the GLL nodes at node i (the h_i of Eq. 3).
 * Closed form for GLL nodes:
 *   D_ij = P_N(x_i) / (P_N(x_j) (x_i - x_j))   i != j
 *   D_00 = -N(N+1)/4,  D_NN = +N(N+1)/4,  D_ii = 0 otherwise.
 * Row-major, D[i*(N+1)+j].
 */
void or_deriv(int N, const double *x, double *D)
{
    int Nq = N + 1;
    for (int i = 0; i < Nq; ++i) {
        double pi, dpi;
        legendre(N, x[i], &pi, &dpi);
        for (int j = 0; j < Nq; ++j) {
            double pj, dpj;
            legendre(N, x[j], &pj, &dpj);
            if (i != j) D[i * Nq + j] = pi / (pj * (x[i] - x[j]));
            else if (i == 0) D[i * Nq + j] = -(double)N * (N + 1) / 4.0;
            else if (i == N) D[i * Nq + j] = (double)N * (N + 1) / 4.0;
            else D[i * Nq + j] = 0.0;
        }
    }
}

/* ------------------------------------------------------------- geometry --- */
#define IDX(i, j, k) ((i) + Nq * ((j) + Nq * (k)))

/*
 * or_geom: geometric factors of the isoparametric map x = x^e(r,s,t)
 * (reading 4).
 * At each GLL point q of element e:
 *   dx/dr etc. by applying D along each reference direction to the nodal
 *   coordinates, J = det(dx/dr), grad r_a = (cofactor rows)/J,
 *   G_ab = w_q J (grad r_a . grad r_b)  (a<=b: rr, rs, rt, ss, st, tt),
 *   wJ = w_q J,  w_q = w_i w_j w_k.
 * Layout: G[e][6][Nq^3], wJ[e][Nq^3].  xyz is [3][E*Nq^3].
 * Returns 0, or -1 if J <= 0 somewhere (first offending local index in *bad).
 */
int or_geom(int64_t E, int N, const double *D, const double *w, const double *xyz,
            double *G, double *wJ, int64_t *bad)
{
    int Nq = N + 1, P3 = Nq * Nq * Nq;
    int64_t n = E * P3;
    const double *X = xyz, *Y = xyz + n, *Z = xyz + 2 * n;
    int status = 0;
    for (int64_t e = 0; e < E; ++e) {
        const double *xe = X + e * P3, *ye = Y + e * P3, *ze = Z + e * P3;
        for (int k = 0; k < Nq; ++k)
        for (int j = 0; j < Nq; ++j)
        for (int i = 0; i < Nq; ++i) {
            double xr = 0, xs = 0, xt = 0, yr = 0, ys = 0, yt = 0, zr = 0, zs = 0, zt = 0;
            for (int m = 0; m < Nq; ++m) {
                double dr = D[i * Nq + m], ds = D[j * Nq + m], dt = D[k * Nq + m];
                xr += dr * xe[IDX(m, j, k)]; yr += dr * ye[IDX(m, j, k)]; zr += dr * ze[IDX(m, j, k)];
                xs += ds * xe[IDX(i, m, k)]; ys += ds * ye[IDX(i, m, k)]; zs += ds * ze[IDX(i, m, k)];
                xt += dt * xe[IDX(i, j, m)]; yt += dt * ye[IDX(i, j, m)]; zt += dt * ze[IDX(i, j, m)];
            }
            double J = xr * (ys * zt - yt * zs) - xs * (yr * zt - yt * zr) + xt * (yr * zs - ys * zr);
            int64_t l = e * P3 + IDX(i, j, k);
            if (!(J > 0.0)) {
                if (status == 0) { status = -1; if (bad) *bad = l; }
            }
            /* inverse metric: rows of (dx/dr)^{-1} = grad r, grad s, grad t */
            double rx = (ys * zt - yt * zs) / J, ry = -(xs * zt - xt * zs) / J, rz = (xs * yt - xt * ys) / J;
            double sx = -(yr * zt - yt * zr) / J, sy = (xr * zt - xt * zr) / J, sz = -(xr * yt - xt * yr) / J;
            double tx = (yr * zs - ys * zr) / J, ty = -(xr * zs - xs * zr) / J, tz = (xr * ys - xs * yr) / J;
            double wq = w[i] * w[j] * w[k] * J;
            double *Ge = G + e * 6 * (int64_t)P3 + IDX(i, j, k);
            Ge[0 * P3] = wq * (rx * rx + ry * ry + rz * rz);
            Ge[1 * P3] = wq * (rx * sx + ry * sy + rz * sz);
            Ge[2 * P3] = wq * (rx * tx + ry * ty + rz * tz);
            Ge[3 * P3] = wq * (sx * sx + sy * sy + sz * sz);
            Ge[4 * P3] = wq * (sx * tx + sy * ty + sz * tz);
            Ge[5 * P3] = wq * (tx * tx + ty * ty + tz * tz);
            wJ[l] = wq;
        }
    }
    return status;
}

/* ------------------------------------------------------------ operator ---- */
/*
 * or_ax_local: the local (unassembled) Helmholtz operator, element by element
 * (tensor contractions, O(N^4) work; BASELINE north_star):
 *   u_r = (I (x) I (x) D) u,  u_s = (I (x) D (x) I) u,  u_t = (D (x) I (x) I) u
 *   g_a = sum_b G_ab u_b
 *   w   = h1 (D_r^T g_r + D_s^T g_s + D_t^T g_t) + h2 wJ u
 * Plain loops in the paper's order; no blocking, no fusion.
 */
void or_ax_local(int64_t E, int N, const double *D, const double *G, const double *wJ,
                 double h1, double h2, const double *u, double *w)
{
    int Nq = N + 1, P3 = Nq * Nq * Nq;
    /* elements are independent: the OpenMP build (bench timing only) splits the element loop over
     * threads; every element's arithmetic is unchanged, so results are bitwise the same */
#pragma omp parallel
    {
    double *ur = malloc(sizeof(double) * P3), *us = malloc(sizeof(double) * P3), *ut = malloc(sizeof(double) * P3);
    double *gr = malloc(sizeof(double) * P3), *gs = malloc(sizeof(double) * P3), *gt = malloc(sizeof(double) * P3);
#pragma omp for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        const double *ue = u + e * P3;
        const double *Ge = G + e * 6 * (int64_t)P3;
        /* gradient in reference coordinates */
        for (int k = 0; k < Nq; ++k)
        for (int j = 0; j < Nq; ++j)
        for (int i = 0; i < Nq; ++i) {
            double a = 0, b = 0, c = 0;
            for (int m = 0; m < Nq; ++m) {
                a += D[i * Nq + m] * ue[IDX(m, j, k)];
                b += D[j * Nq + m] * ue[IDX(i, m, k)];
                c += D[k * Nq + m] * ue[IDX(i, j, m)];
            }
            ur[IDX(i, j, k)] = a; us[IDX(i, j, k)] = b; ut[IDX(i, j, k)] = c;
        }
        /* pointwise metric */
        for (int q = 0; q < P3; ++q) {
            double Grr = Ge[0 * P3 + q], Grs = Ge[1 * P3 + q], Grt = Ge[2 * P3 + q];
            double Gss = Ge[3 * P3 + q], Gst = Ge[4 * P3 + q], Gtt = Ge[5 * P3 + q];
            gr[q] = Grr * ur[q] + Grs * us[q] + Grt * ut[q];
            gs[q] = Grs * ur[q] + Gss * us[q] + Gst * ut[q];
            gt[q] = Grt * ur[q] + Gst * us[q] + Gtt * ut[q];
        }
        /* transposed gradient */
        for (int k = 0; k < Nq; ++k)
        for (int j = 0; j < Nq; ++j)
        for (int i = 0; i < Nq; ++i) {
            double s = 0;
            for (int m = 0; m < Nq; ++m) {
                s += D[m * Nq + i] * gr[IDX(m, j, k)];
                s += D[m * Nq + j] * gs[IDX(i, m, k)];
                s += D[m * Nq + k] * gt[IDX(i, j, m)];
            }
            int64_t l = e * P3 + IDX(i, j, k);
            w[l] = h1 * s + h2 * wJ[l] * ue[IDX(i, j, k)];
        }
    }
    free(ur); free(us); free(ut); free(gr); free(gs); free(gt);
    }
}

/* ------------------------------------------------------- gather-scatter --- */
typedef struct { int64_t gid; int64_t l; } gl_pair;
static int cmp_gl(const void *a, const void *b)
{
    const gl_pair *x = a, *y = b;
    if (x->gid != y->gid) return x->gid < y->gid ? -1 : 1;
    return (x->l > y->l) - (x->l < y->l);
}
typedef struct { int64_t first; int64_t start; int64_t len; } run_t;
static int cmp_run(const void *a, const void *b)
{
    const run_t *x = a, *y = b;
    return (x->first > y->first) - (x->first < y->first);
}

/*
 * or_gs_map: the canonical gather-scatter map of one rank (reading 7;
 * P:198-200 "C0 continuity ... unit-depth stencils").
 * A run = all local copies of one gid.  Shared runs are those with >= min_len
 * copies (min_len = 2 for a single rank).  Runs are ordered by their smallest
 * local index; copies within a run ascend in l.
 * Outputs: perm[0..nperm) = local indices of the copies in canonical order,
 * offs[0..nruns] = run starts in perm, rgid[0..nruns) = the run's gid.
 * Returns nruns.  Caller sizes perm/offs/rgid with n / n+1 / n entries.
 */
int64_t or_gs_map(int64_t n, const int64_t *gid, int64_t min_len,
                  int32_t *perm, int64_t *offs, int64_t *rgid)
{
    gl_pair *p = malloc(sizeof(gl_pair) * (n ? n : 1));
    for (int64_t l = 0; l < n; ++l) { p[l].gid = gid[l]; p[l].l = l; }
    qsort(p, n, sizeof(gl_pair), cmp_gl);
    run_t *runs = malloc(sizeof(run_t) * (n ? n : 1));
    int64_t nr = 0;
    for (int64_t a = 0; a < n;) {
        int64_t b = a + 1;
        while (b < n && p[b].gid == p[a].gid) ++b;
        if (b - a >= min_len) { runs[nr].first = p[a].l; runs[nr].start = a; runs[nr].len = b - a; ++nr; }
        a = b;
    }
    qsort(runs, nr, sizeof(run_t), cmp_run);
    int64_t o = 0;
    for (int64_t r = 0; r < nr; ++r) {
        offs[r] = o;
        rgid[r] = p[runs[r].start].gid;
        for (int64_t c = 0; c < runs[r].len; ++c) perm[o++] = (int32_t)p[runs[r].start + c].l;
    }
    offs[nr] = o;
    free(p); free(runs);
    return nr;
}

/*
 * or_gs_apply: v <- QQ^T v on one rank: for each run, s = ((v[c0]+v[c1])+v[c2])+...
 * in canonical order, then every copy gets s (reading 7).
 */
void or_gs_apply(int64_t nruns, const int32_t *perm, const int64_t *offs, double *v)
{
#pragma omp parallel for schedule(static)   /* runs are disjoint */
    for (int64_t r = 0; r < nruns; ++r) {
        double s = v[perm[offs[r]]];
        for (int64_t c = offs[r] + 1; c < offs[r + 1]; ++c) s += v[perm[c]];
        for (int64_t c = offs[r]; c < offs[r + 1]; ++c) v[perm[c]] = s;
    }
}

/* or_gs_partial: per-run left-fold partial sums only (used by the multi-rank
 * emulation in oracle/__init__.py, reading 7: totals summed in rank order). */
void or_gs_partial(int64_t nruns, const int32_t *perm, const int64_t *offs, const double *v, double *part)
{
    for (int64_t r = 0; r < nruns; ++r) {
        double s = v[perm[offs[r]]];
        for (int64_t c = offs[r] + 1; c < offs[r + 1]; ++c) s += v[perm[c]];
        part[r] = s;
    }
}

/* ------------------------------------------------------------ mask etc. --- */
/* or_mask: v[l] = 0 where mask[l] (reading 6). */
void or_mask(int64_t n, const uint8_t *mask, double *v)
{
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < n; ++l) if (mask[l]) v[l] = 0.0;
}

/*
 * or_diag_local: the diagonal of the local operator h1 K_L + h2 B_L
 * (reading 10 -- exact, including the G_rs/G_rt/G_st cross
 * terms).  With w = sum_b D_b^T (G D u)_b, the (q,q) entry at q = (i,j,k) is
 *   sum_m D_mi^2 Grr(m,j,k) + sum_m D_mj^2 Gss(i,m,k) + sum_m D_mk^2 Gtt(i,j,m)
 *   + 2 (D_ii D_jj Grs + D_ii D_kk Grt + D_jj D_kk Gst)(i,j,k)
 * times h1, plus h2 wJ.
 */
void or_diag_local(int64_t E, int N, const double *D, const double *G, const double *wJ,
                   double h1, double h2, double *d)
{
    int Nq = N + 1, P3 = Nq * Nq * Nq;
    for (int64_t e = 0; e < E; ++e) {
        const double *Ge = G + e * 6 * (int64_t)P3;
        for (int k = 0; k < Nq; ++k)
        for (int j = 0; j < Nq; ++j)
        for (int i = 0; i < Nq; ++i) {
            double s = 0;
            for (int m = 0; m < Nq; ++m) {
                s += D[m * Nq + i] * D[m * Nq + i] * Ge[0 * P3 + IDX(m, j, k)];
                s += D[m * Nq + j] * D[m * Nq + j] * Ge[3 * P3 + IDX(i, m, k)];
                s += D[m * Nq + k] * D[m * Nq + k] * Ge[5 * P3 + IDX(i, j, m)];
            }
            int q = IDX(i, j, k);
            s += 2.0 * (D[i * Nq + i] * D[j * Nq + j] * Ge[1 * P3 + q]
                      + D[i * Nq + i] * D[k * Nq + k] * Ge[2 * P3 + q]
                      + D[j * Nq + j] * D[k * Nq + k] * Ge[4 * P3 + q]);
            int64_t l = e * P3 + q;
            d[l] = h1 * s + h2 * wJ[l];
        }
    }
}

/* ------------------------------------------------------------------ PCG --- */
typedef struct {
    int64_t E; int N;
    const double *D, *G, *wJ;
    const uint8_t *mask;
    int64_t nruns; const int32_t *perm; const int64_t *offs;
    const uint8_t *owner;   /* 1 on the owner copy (smallest l) of every gid */
    double h1, h2;
} or_op;

/* w = M QQ^T (h1 K_L + h2 B_L) M u  (reading 6) */
static void op_apply(const or_op *A, const double *u, double *tmp, double *w)
{
    int64_t n = A->E * (A->N + 1) * (A->N + 1) * (A->N + 1);
    memcpy(tmp, u, sizeof(double) * n);
    or_mask(n, A->mask, tmp);
    or_ax_local(A->E, A->N, A->D, A->G, A->wJ, A->h1, A->h2, tmp, w);
    or_gs_apply(A->nruns, A->perm, A->offs, w);
    or_mask(n, A->mask, w);
}

/* owner-copy inner product sum_g x_g y_g (reading 8), evaluated as the Dot2 algorithm of Ogita,
 * Rump and Oishi ("Accurate sum and dot product", SIAM J. Sci. Comput. 26, 2005, Alg. 5.3): every
 * product is split exactly (TwoProduct via fma) and the running sum carried with its exact rounding
 * error (TwoSum), so the result is as accurate as a twice-working-precision evaluation rounded once
 * -- within an ulp of the exactly rounded definition for the well-conditioned sums of CG, and
 * independent of the summation order.  g_dot_mode (test yardsticks of reading 17, never the
 * default): 1 = the same in descending local index (order independence), 2 = plain recursive
 * summation s += x y in ascending index -- the textbook rounding of the same inner product, whose
 * distance from mode 0 is the drift two correct FP64 CG codes show on a converged solve. */
static int g_dot_mode = 0;
static void two_sum(double a, double b, double *s, double *e)
{
    const double x = a + b, z = x - a;
    *e = (a - (x - z)) + (b - z);
    *s = x;
}
static double dot_owner(int64_t n, const uint8_t *owner, const double *x, const double *y)
{
    double p = 0.0, s = 0.0;
    if (g_dot_mode == 2) {
        for (int64_t l = 0; l < n; ++l) if (owner[l]) p += x[l] * y[l];
        return p;
    }
    for (int64_t k = 0; k < n; ++k) {
        const int64_t l = g_dot_mode == 1 ? n - 1 - k : k;
        if (!owner[l]) continue;
        const double h = x[l] * y[l], r = fma(x[l], y[l], -h);   /* TwoProduct: h + r = x y exactly */
        double q;
        two_sum(p, h, &p, &q);
        s += q + r;
    }
    return p + s;
}
void or_set_dot_mode(int mode) { g_dot_mode = mode; }
static int g_upd_fma = 0;
void or_set_upd_fma(int on) { g_upd_fma = on; }

/*
 * or_pcg: Jacobi-preconditioned CG, Hestenes-Stiefel form, step by step as
 * SPEC S:353-357 / SURVEY 8(c) state it (BASELINE north_star "fused CG vector
 * updates and dot-product reductions"):
 *   x0 = 0, r0 = M b, z0 = Dinv r0, p0 = z0, rho0 = <r0,z0>, beta_b = ||M b||
 *   for k = 0,1,...: if ||r_k|| <= tol*beta_b stop
 *     w = A p; sigma = <p,w> (<= 0 -> error); alpha = rho/sigma
 *     x += alpha p; r -= alpha w; z = Dinv r; rho' = <r,z>; beta = rho'/rho
 *     p = z + beta p
 * Inner products are owner-copy sums (reading 8).  hist[k] = ||r_k||/||b||.
 * Returns 0 (converged), 1 (maxit), -5 (sigma <= 0).
 */
int or_pcg(int64_t E, int N, const double *D, const double *G, const double *wJ,
           const uint8_t *mask, int64_t nruns, const int32_t *perm, const int64_t *offs,
           const uint8_t *owner, const double *Dinv, double h1, double h2,
           const double *b, double *x, double tol, int maxit, int *iters, double *hist)
{
    or_op A = {E, N, D, G, wJ, mask, nruns, perm, offs, owner, h1, h2};
    int64_t n = E * (N + 1) * (N + 1) * (N + 1);
    double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
    double *p = malloc(sizeof(double) * n), *w = malloc(sizeof(double) * n);
    double *tmp = malloc(sizeof(double) * n);
    int status = 1;
    for (int64_t l = 0; l < n; ++l) { x[l] = 0.0; r[l] = b[l]; }
    or_mask(n, mask, r);
    for (int64_t l = 0; l < n; ++l) { z[l] = Dinv[l] * r[l]; p[l] = z[l]; }
    double rho = dot_owner(n, owner, r, z);
    double bb = sqrt(dot_owner(n, owner, r, r));
    int k = 0;
    for (;; ++k) {
        double rn = sqrt(dot_owner(n, owner, r, r));
        if (hist) hist[k] = bb > 0 ? rn / bb : 0.0;
        if (rn <= tol * bb) { status = 0; break; }
        if (k >= maxit) { status = 1; break; }
        op_apply(&A, p, tmp, w);
        double sigma = dot_owner(n, owner, p, w);
        if (!(sigma > 0.0)) { status = -5; break; }
        double alpha = rho / sigma;
        if (g_upd_fma) {
#pragma omp parallel for schedule(static)
            for (int64_t l = 0; l < n; ++l) { x[l] = fma(alpha, p[l], x[l]); r[l] = fma(-alpha, w[l], r[l]); }
        } else {
#pragma omp parallel for schedule(static)
            for (int64_t l = 0; l < n; ++l) { x[l] += alpha * p[l]; r[l] -= alpha * w[l]; }
        }
#pragma omp parallel for schedule(static)
        for (int64_t l = 0; l < n; ++l) z[l] = Dinv[l] * r[l];
        double rho1 = dot_owner(n, owner, r, z);
        double beta = rho1 / rho;
        rho = rho1;
        if (g_upd_fma) {
#pragma omp parallel for schedule(static)
            for (int64_t l = 0; l < n; ++l) p[l] = fma(beta, p[l], z[l]);
        } else {
#pragma omp parallel for schedule(static)
            for (int64_t l = 0; l < n; ++l) p[l] = z[l] + beta * p[l];
        }
    }
    *iters = k;
    free(r); free(z); free(p); free(w); free(tmp);
    return status;
}

/* or_op_apply: exported w = M QQ^T (h1 K_L + h2 B_L) M u for tests. */
void or_op_apply(int64_t E, int N, const double *D, const double *G, const double *wJ,
                 const uint8_t *mask, int64_t nruns, const int32_t *perm, const int64_t *offs,
                 double h1, double h2, const double *u, double *w)
{
    or_op A = {E, N, D, G, wJ, mask, nruns, perm, offs, NULL, h1, h2};
    int64_t n = E * (N + 1) * (N + 1) * (N + 1);
    double *tmp = malloc(sizeof(double) * n);
    op_apply(&A, u, tmp, w);
    free(tmp);
}

/* ---------------------------------------------------------- host probe --- */
/* STREAM triad a = b + 3 c over n doubles, best of `reps`, in GB/s (3 x 8 B per element; the
 * denominator of the oracle's own CPU roofline fraction).  Threads as OpenMP gives. */
#include <time.h>
double or_triad_gbps(int64_t n, int reps)
{
    double *a = malloc(sizeof(double) * n), *b = malloc(sizeof(double) * n), *c = malloc(sizeof(double) * n);
    if (!a || !b || !c) { free(a); free(b); free(c); return 0.0; }
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < n; ++l) { a[l] = 0.0; b[l] = 1.0; c[l] = 2.0; }
    double best = 1e30;
    for (int k = 0; k < reps; ++k) {
        struct timespec t0, t1;
        clock_gettime(CLOCK_MONOTONIC, &t0);
#pragma omp parallel for schedule(static)
        for (int64_t l = 0; l < n; ++l) a[l] = b[l] + 3.0 * c[l];
        clock_gettime(CLOCK_MONOTONIC, &t1);
        double dt = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
        if (dt < best) best = dt;
    }
    double chk = a[n / 2];
    free(a); free(b); free(c);
    return chk == 7.0 ? 24.0 * (double)n / best / 1e9 : 0.0;
}

int or_threads(void)
{
#ifdef _OPENMP
    int t = 1;
#pragma omp parallel
#pragma omp single
    t = omp_get_num_threads();
    return t;
#else
    return 1;
#endif
}
