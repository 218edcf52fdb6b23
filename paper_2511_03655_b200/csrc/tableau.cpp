// Host tableau generator for IRKGL16 (library side; independent of oracle/).
//
// PAPER.md P:L109-116 (Sec. 2.2): c_i = (1+x_i)/2 with x_i the zeros of the
// Legendre polynomial P_s; b and each row of A solve the collocation
// conditions  sum_j a_ij c_j^(k-1) = c_i^k/k,  sum_j b_j c_j^(k-1) = 1/k.
// P:L146-155 (Sec. 2.3): mu_ij = a_ij/b_j, rounded so that mu~_ij = 1 - mu~_ji
// (i<j) keeps the scheme exactly symplectic.  P:L165-178 (Sec. 2.4): nu, read
// as nu_ij = nu^_ij / b_j with sum_j nu^_ij (c_j-1)^(k-1) = c_i^k/k (reading R-3,
// DESIGN.md; the printed condition has c_i where c_j is meant).
//
// Algorithm (deliberately different from the oracle's bisection + Lagrange-basis
// integration): Newton on P_s from cosine guesses, then Bjorck-Pereyra solves of
// the dual Vandermonde systems, all in __float128; the checks below gate
// irk_create.
#include "tableau.h"

#include <cmath>
#include <cstdio>

namespace irk {
namespace {

typedef __float128 f128;

f128 fabsq_(f128 x) { return x < 0 ? -x : x; }

// P_s(x) and P_s'(x) by the three-term recurrence.
void legendre(int s, f128 x, f128 *p, f128 *dp) {
    f128 p0 = 1, p1 = x;
    for (int k = 1; k < s; ++k) {
        f128 p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
        p0 = p1;
        p1 = p2;
    }
    *p = (s == 0) ? p0 : p1;
    *dp = (s == 0) ? 0 : s * (x * p1 - p0) / (x * x - 1);
}

// Solve sum_j w_j x_j^k = f_k, k = 0..n-1 (Vandermonde V_kj = x_j^k) in place
// (Bjorck-Pereyra, dual system).
void bjorck_pereyra_dual(int n, const f128 *x, f128 *f) {
    for (int k = 0; k < n - 1; ++k)
        for (int i = n - 1; i >= k + 1; --i) f[i] = f[i] - x[k] * f[i - 1];
    for (int k = n - 2; k >= 0; --k) {
        for (int i = k + 1; i < n; ++i) f[i] = f[i] / (x[i] - x[i - k - 1]);
        for (int i = k; i < n - 1; ++i) f[i] = f[i] - f[i + 1];
    }
}

}  // namespace

int build_tableau(double h, Tableau *T, char *err, size_t errlen) {
    const int s = 8;
    f128 x[s], c[s], b[s], a[s][s], nu[s][s];
    // Gauss nodes: Newton from x_i ~ cos(pi (i - 1/4)/(s + 1/2)), i = 1..s
    for (int i = 0; i < s; ++i) {
        f128 xi = -std::cos(M_PI * (i + 0.75) / (s + 0.5));
        for (int it = 0; it < 100; ++it) {
            f128 p, dp;
            legendre(s, xi, &p, &dp);
            f128 dx = p / dp;
            xi -= dx;
            if (fabsq_(dx) < (f128)1e-33) break;
        }
        x[i] = xi;
    }
    for (int i = 0; i < s; ++i) c[i] = (1 + x[i]) / 2;
    for (int i = 1; i < s; ++i)
        if (!(c[i] > c[i - 1])) {
            snprintf(err, errlen, "tableau: Gauss nodes not increasing");
            return -1;
        }
    // b: sum_j b_j c_j^(k-1) = 1/k
    for (int k = 0; k < s; ++k) b[k] = (f128)1 / (k + 1);
    bjorck_pereyra_dual(s, c, b);
    // A rows: sum_j a_ij c_j^(k-1) = c_i^k / k
    for (int i = 0; i < s; ++i) {
        f128 r[s], ck = c[i];
        for (int k = 0; k < s; ++k) {
            r[k] = ck / (k + 1);
            ck *= c[i];
        }
        bjorck_pereyra_dual(s, c, r);
        for (int j = 0; j < s; ++j) a[i][j] = r[j];
    }
    // nu rows: sum_j nu^_ij (c_j - 1)^(k-1) = c_i^k / k ; nu_ij = nu^_ij / b_j
    f128 cm1[s];
    for (int j = 0; j < s; ++j) cm1[j] = c[j] - 1;
    for (int i = 0; i < s; ++i) {
        f128 r[s], ck = c[i];
        for (int k = 0; k < s; ++k) {
            r[k] = ck / (k + 1);
            ck *= c[i];
        }
        bjorck_pereyra_dual(s, cm1, r);
        for (int j = 0; j < s; ++j) nu[i][j] = r[j] / b[j];
    }
    // ---- checks: B(16), C(8), symplecticity (Eq. sym) ----
    f128 worst = 0;
    for (int k = 1; k <= 2 * s; ++k) {
        f128 acc = 0;
        for (int j = 0; j < s; ++j) {
            f128 p = 1;
            for (int e = 1; e < k; ++e) p *= c[j];
            acc += b[j] * p;
        }
        f128 r = fabsq_(acc - (f128)1 / k);
        if (r > worst) worst = r;
    }
    for (int i = 0; i < s; ++i)
        for (int k = 1; k <= s; ++k) {
            f128 acc = 0, ci = 1;
            for (int j = 0; j < s; ++j) {
                f128 p = 1;
                for (int e = 1; e < k; ++e) p *= c[j];
                acc += a[i][j] * p;
            }
            for (int e = 0; e < k; ++e) ci *= c[i];
            f128 r = fabsq_(acc - ci / k);
            if (r > worst) worst = r;
        }
    for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) {
            f128 r = fabsq_(b[i] * a[i][j] + b[j] * a[j][i] - b[i] * b[j]);
            if (r > worst) worst = r;
        }
    if (!(worst < (f128)1e-28)) {
        snprintf(err, errlen, "tableau: order/symplectic residual %.3e too large", (double)worst);
        return -1;
    }
    // ---- fp64 rounding (R-1) ----
    for (int i = 0; i < s; ++i) {
        T->c[i] = (double)c[i];
        T->b[i] = (double)b[i];
        for (int j = 0; j < s; ++j) T->nu[i][j] = (double)nu[i][j];
        for (int j = 0; j < i; ++j) T->mu[i][j] = (double)(a[i][j] / b[j]);
    }
    for (int i = 0; i < s; ++i) {
        T->mu[i][i] = 0.5;
        for (int j = i + 1; j < s; ++j) T->mu[i][j] = 1.0 - T->mu[j][i];
    }
    for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j)
            if (i != j && T->mu[i][j] + T->mu[j][i] != 1.0) {
                snprintf(err, errlen, "tableau: mu~ identity fails at (%d,%d)", i, j);
                return -1;
            }
    for (int j = 0; j < s; ++j) T->hb[j] = h * T->b[j];  // hb~_j = fl(h * b~_j)
    return 0;
}

}  // namespace irk
