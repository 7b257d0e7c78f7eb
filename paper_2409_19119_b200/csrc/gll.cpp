// gll.cpp -- GLL rule and derivative matrix for the device path (host code).
//
// P:183-188 (Eq. 3): nodal interpolants h_i on the Gauss-Lobatto-Legendre
// points.  Route used here (independent of the oracle's):
//   nodes  -- simultaneous Newton iteration on x P_N(x) - P_{N-1}(x) for all
//             nodes at once, seeded with the Chebyshev-Gauss-Lobatto points,
//             P evaluated by the Legendre recurrence (a Vandermonde sweep);
//   weights-- w_i = 2 / (N (N+1) P_N(x_i)^2);
//   D      -- barycentric form D_ij = (lambda_j / lambda_i) / (x_i - x_j) with
//             lambda_i = 1 / prod_{k != i}(x_i - x_k), and the diagonal set by
//             the negative-row-sum identity D_ii = -sum_{j != i} D_ij, which
//             keeps D * 1 = 0 to rounding.
#include <cmath>
#include <vector>

namespace nekb200 {

void gll_rule(int N, double *x, double *w)
{
    const int Nq = N + 1;
    std::vector<double> xn(Nq), xo(Nq), P((size_t)Nq * Nq);
    for (int i = 0; i < Nq; ++i) xn[i] = -std::cos(M_PI * i / N);   // ascending CGL guess
    for (int it = 0; it < 100; ++it) {
        double delta = 0;
        for (int i = 0; i < Nq; ++i) xo[i] = xn[i];
        for (int i = 0; i < Nq; ++i) {
            double p0 = 1.0, p1 = xo[i];
            P[(size_t)i * Nq + 0] = p0;
            if (N >= 1) P[(size_t)i * Nq + 1] = p1;
            for (int k = 2; k <= N; ++k) {
                double p2 = ((2.0 * k - 1.0) * xo[i] * p1 - (k - 1.0) * p0) / k;
                P[(size_t)i * Nq + k] = p2;
                p0 = p1; p1 = p2;
            }
            double PN = P[(size_t)i * Nq + N], PN1 = P[(size_t)i * Nq + N - 1];
            xn[i] = xo[i] - (xo[i] * PN - PN1) / (Nq * PN);
            delta = std::fmax(delta, std::fabs(xn[i] - xo[i]));
        }
        if (delta <= 2.2e-16) break;
    }
    xn[0] = -1.0; xn[N] = 1.0;
    for (int i = 0; i < Nq / 2; ++i) {   // exact symmetry about 0
        double h = 0.5 * (xn[N - i] - xn[i]);
        xn[i] = -h; xn[N - i] = h;
    }
    if (N % 2 == 0) xn[N / 2] = 0.0;
    for (int i = 0; i < Nq; ++i) {
        double p0 = 1.0, p1 = xn[i];
        for (int k = 2; k <= N; ++k) {
            double p2 = ((2.0 * k - 1.0) * xn[i] * p1 - (k - 1.0) * p0) / k;
            p0 = p1; p1 = p2;
        }
        double PN = (N == 0) ? 1.0 : p1;
        x[i] = xn[i];
        w[i] = 2.0 / (N * (N + 1.0) * PN * PN);
    }
}

void deriv_matrix(int N, const double *x, double *D)
{
    const int Nq = N + 1;
    std::vector<double> lam(Nq);
    for (int i = 0; i < Nq; ++i) {
        double prod = 1.0;
        for (int k = 0; k < Nq; ++k) if (k != i) prod *= (x[i] - x[k]);
        lam[i] = 1.0 / prod;
    }
    for (int i = 0; i < Nq; ++i) {
        double rowsum = 0.0;
        for (int j = 0; j < Nq; ++j) {
            if (j == i) continue;
            double d = (lam[j] / lam[i]) / (x[i] - x[j]);
            D[i * Nq + j] = d;
            rowsum += d;
        }
        D[i * Nq + i] = -rowsum;
    }
}

}  // namespace nekb200
