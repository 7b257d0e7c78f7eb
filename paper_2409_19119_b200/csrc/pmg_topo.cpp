// pmg_topo.cpp -- host construction of the p-multigrid levels (DESIGN.md "pMG readings" P2, P3).
//
// A coarse level is the same elements at a lower order N_c.  What it needs
// from the fine level, built here on the host once at setup:
//   * node ids: every coarse node belongs to one mesh entity (vertex, edge, face, interior) and
//     is keyed by a FINE node id of that entity, so ids are global without communication and
//     agree on every element (and rank) holding the entity:
//       vertex  key = id of the vertex node                              slot 0
//       edge    key = id of the fine edge node next to the end vertex with the smaller id,
//               slot = coarse-node distance from that vertex
//       face    key = id of the fine face node diagonally next to the corner with the smallest
//               id; the first face axis points to the smaller-id neighbour corner, slot = u (Nc+1) + v
//       inside  key = id of the element's fine node (1,1,1), slot = i + (Nc+1)(j + (Nc+1)k)
//     id = key (Nc+1)^3 + slot;
//   * Dirichlet mask: the key node's mask; the fine mask must be constant over each entity's
//     interior nodes (a union of closed boundary faces / edges / vertices), else NEK_EINVAL;
//   * coordinates: Lagrange interpolation of the finest level's GLL-node coordinates to the
//     order-N_c GLL points (isoparametric rediscretisation), by sum factorisation;
//   * J: the 1-D interpolation matrix between two orders, J[I][i] = h_i^{from}(xi^{to}_I), in
//     barycentric form (exactly 1 / 0 where a target point is a source node).
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "nek_ctx.h"

namespace nekb200 {

void interp_matrix(int Nfrom, int Nto, double *J)
{
    std::vector<double> xf(Nfrom + 1), wf(Nfrom + 1), xt(Nto + 1), wt(Nto + 1), lam(Nfrom + 1);
    gll_rule(Nfrom, xf.data(), wf.data());
    gll_rule(Nto, xt.data(), wt.data());
    for (int i = 0; i <= Nfrom; ++i) {          // barycentric weights of the source nodes
        double p = 1.0;
        for (int k = 0; k <= Nfrom; ++k)
            if (k != i) p *= xf[i] - xf[k];
        lam[i] = 1.0 / p;
    }
    for (int I = 0; I <= Nto; ++I) {
        double *row = J + (size_t)I * (Nfrom + 1);
        int hit = -1;
        for (int i = 0; i <= Nfrom; ++i)
            if (xt[I] == xf[i]) hit = i;
        if (hit >= 0) {
            for (int i = 0; i <= Nfrom; ++i) row[i] = i == hit ? 1.0 : 0.0;
            continue;
        }
        double den = 0.0;
        for (int i = 0; i <= Nfrom; ++i) den += lam[i] / (xt[I] - xf[i]);
        for (int i = 0; i <= Nfrom; ++i) row[i] = lam[i] / (xt[I] - xf[i]) / den;
    }
}

// out[e] = (J x J x J) in[e] per element: in has (Nin+1)^3 points, out (Nout+1)^3, i fastest.
void interp_elements_host(int64_t E, int Nin, int Nout, const double *J, const double *in, double *out)
{
    const int a = Nin + 1, b = Nout + 1;
    std::vector<double> t1((size_t)a * a * b), t2((size_t)a * b * b);
    for (int64_t e = 0; e < E; ++e) {
        const double *u = in + e * a * a * a;
        double *v = out + e * b * b * b;
        for (int k = 0; k < a; ++k)              // i direction
            for (int j = 0; j < a; ++j)
                for (int I = 0; I < b; ++I) {
                    double s = 0.0;
                    for (int i = 0; i < a; ++i) s += J[I * a + i] * u[(k * a + j) * a + i];
                    t1[(k * a + j) * b + I] = s;
                }
        for (int k = 0; k < a; ++k)              // j direction
            for (int Jj = 0; Jj < b; ++Jj)
                for (int I = 0; I < b; ++I) {
                    double s = 0.0;
                    for (int j = 0; j < a; ++j) s += J[Jj * a + j] * t1[(k * a + j) * b + I];
                    t2[(k * b + Jj) * b + I] = s;
                }
        for (int K = 0; K < b; ++K)              // k direction
            for (int Jj = 0; Jj < b; ++Jj)
                for (int I = 0; I < b; ++I) {
                    double s = 0.0;
                    for (int k = 0; k < a; ++k) s += J[K * a + k] * t2[(k * b + Jj) * b + I];
                    v[(K * b + Jj) * b + I] = s;
                }
    }
}

int pmg_coarse_ids(int64_t E, int Nf, const int64_t *gid, const uint8_t *mask, int Nc, int64_t *gid_c,
                   uint8_t *mask_c, std::string &err)
{
    if (Nf < 2 || Nc < 1 || Nc >= Nf) { err = "pMG: coarsening needs 1 <= Nc < Nf and Nf >= 2"; return NEK_EINVAL; }
    const int a = Nf + 1, c = Nc + 1;
    const int64_t S = (int64_t)c * c * c;
    const int64_t P3f = (int64_t)a * a * a, P3c = (int64_t)c * c * c;
    auto fend = [&](int q) { return q == 0 ? 0 : Nf; };
    for (int64_t e = 0; e < E; ++e) {
        const int64_t *g = gid + e * P3f;
        const uint8_t *mk = mask ? mask + e * P3f : nullptr;
        auto F = [&](int I, int J, int K) { return (int64_t)(K * a + J) * a + I; };
        // entity-wise mask check: fine edge / face interior nodes must agree
        if (mk) {
            for (int d = 0; d < 3; ++d)
                for (int p = 0; p < 2; ++p)
                    for (int q2 = 0; q2 < 2; ++q2) {           // 12 edges
                        int idx[3];
                        uint8_t m0 = 0;
                        for (int t = 1; t < Nf; ++t) {
                            const int o1 = (d + 1) % 3, o2 = (d + 2) % 3;
                            idx[d] = t; idx[o1] = p ? Nf : 0; idx[o2] = q2 ? Nf : 0;
                            const uint8_t m = mk[F(idx[0], idx[1], idx[2])];
                            if (t == 1) m0 = m;
                            else if (m != m0) {
                                err = "pMG: Dirichlet mask not constant along an edge of element " + std::to_string(e);
                                return NEK_EINVAL;
                            }
                        }
                    }
            for (int fx = 0; fx < 3; ++fx)
                for (int side = 0; side < 2; ++side) {                // 6 faces
                    const int d1 = (fx + 1) % 3, d2 = (fx + 2) % 3;
                    uint8_t m0 = 0;
                    bool first = true;
                    for (int t2 = 1; t2 < Nf; ++t2)
                        for (int t1 = 1; t1 < Nf; ++t1) {
                            int idx[3];
                            idx[fx] = side ? Nf : 0; idx[d1] = t1; idx[d2] = t2;
                            const uint8_t m = mk[F(idx[0], idx[1], idx[2])];
                            if (first) { m0 = m; first = false; }
                            else if (m != m0) {
                                err = "pMG: Dirichlet mask not constant over a face of element " + std::to_string(e);
                                return NEK_EINVAL;
                            }
                        }
                }
        }
        for (int k = 0; k < c; ++k)
            for (int j = 0; j < c; ++j)
                for (int i = 0; i < c; ++i) {
                    const int idx[3] = {i, j, k};
                    bool end[3];
                    int ne = 0;
                    for (int t = 0; t < 3; ++t) { end[t] = idx[t] == 0 || idx[t] == Nc; ne += end[t]; }
                    int kn[3];
                    int64_t slot = 0;
                    if (ne == 3) {
                        for (int t = 0; t < 3; ++t) kn[t] = fend(idx[t]);
                    } else if (ne == 2) {
                        const int d = !end[0] ? 0 : !end[1] ? 1 : 2;
                        int A[3], B[3];
                        for (int t = 0; t < 3; ++t) A[t] = B[t] = kn[t] = end[t] ? fend(idx[t]) : 0;
                        A[d] = 0; B[d] = Nf;
                        if (g[F(A[0], A[1], A[2])] < g[F(B[0], B[1], B[2])]) { kn[d] = 1; slot = idx[d]; }
                        else { kn[d] = Nf - 1; slot = Nc - idx[d]; }
                    } else if (ne == 1) {
                        const int fx = end[0] ? 0 : end[1] ? 1 : 2;
                        const int d1 = fx == 0 ? 1 : 0, d2 = fx == 2 ? 1 : 2;
                        auto corner = [&](int o1, int o2) {
                            int p[3];
                            p[fx] = fend(idx[fx]); p[d1] = o1; p[d2] = o2;
                            return g[F(p[0], p[1], p[2])];
                        };
                        int o1 = 0, o2 = 0;
                        int64_t best = corner(0, 0);
                        for (int c2 = 0; c2 < 2; ++c2)
                            for (int c1 = 0; c1 < 2; ++c1) {
                                const int64_t v = corner(c1 ? Nf : 0, c2 ? Nf : 0);
                                if (v < best) { best = v; o1 = c1 ? Nf : 0; o2 = c2 ? Nf : 0; }
                            }
                        const int64_t n1 = corner(Nf - o1, o2), n2 = corner(o1, Nf - o2);
                        const int t1 = std::abs(idx[d1] - (o1 == 0 ? 0 : Nc)), t2 = std::abs(idx[d2] - (o2 == 0 ? 0 : Nc));
                        const int pu = n1 < n2 ? t1 : t2, pv = n1 < n2 ? t2 : t1;
                        kn[fx] = fend(idx[fx]);
                        kn[d1] = o1 == 0 ? 1 : Nf - 1;
                        kn[d2] = o2 == 0 ? 1 : Nf - 1;
                        slot = (int64_t)pu * c + pv;
                    } else {
                        kn[0] = kn[1] = kn[2] = 1;
                        slot = i + (int64_t)c * (j + (int64_t)c * k);
                    }
                    const int64_t f = F(kn[0], kn[1], kn[2]);
                    const int64_t lc = e * P3c + (k * c + j) * c + i;
                    gid_c[lc] = g[f] * S + slot;
                    mask_c[lc] = mk ? mk[f] : 0;
                }
    }
    return NEK_OK;
}

}  // namespace nekb200
