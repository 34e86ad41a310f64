/*
 * oracle/exact.c -- CPU ORACLE (test infrastructure only): the exact O(n^2)
 * tsNET cost and gradient (the quantities L-tsNET approximates) and the exact
 * sparse KL attraction term, in fp64.
 *
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library.  Shares no code with the CUDA path.
 *
 * Notation: Delta_ij = X_i - X_j, r2 = |Delta_ij|^2,
 * w_ij = 1/(1 + r2), Z = sum_{k != l} w_kl.
 */
#include <stdint.h>
#include <math.h>

/* Eq. 6 first term ("analogous to attraction forces") without
 * the factor 4 lambda_KL: F_i = sum_{j in row i} p_ij w_ij Delta_ij, for the
 * rows i in [row0, row0 + nrows) (F holds those rows only). */
void oracle_attr_sparse_rows(int64_t row0, int64_t nrows, const double* X, const int64_t* indptr,
                             const int32_t* indices, const double* pval, double* F)
{
#pragma omp parallel for schedule(dynamic, 1024) if (nrows > 4096)
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = row0 + r;
        double fx = 0.0, fy = 0.0;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            int64_t j = indices[e];
            double dx = X[2 * i] - X[2 * j], dy = X[2 * i + 1] - X[2 * j + 1];
            double w = 1.0 / (1.0 + dx * dx + dy * dy);
            fx += pval[e] * w * dx;
            fy += pval[e] * w * dy;
        }
        F[2 * r] = fx;
        F[2 * r + 1] = fy;
    }
}

void oracle_attr_sparse(int64_t n, const double* X, const int64_t* indptr, const int32_t* indices,
                        const double* pval, double* F)
{
#pragma omp parallel for schedule(dynamic, 1024) if (n > 4096)
    for (int64_t i = 0; i < n; ++i) {
        double fx = 0.0, fy = 0.0;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            int64_t j = indices[e];
            double dx = X[2 * i] - X[2 * j], dy = X[2 * i + 1] - X[2 * j + 1];
            double w = 1.0 / (1.0 + dx * dx + dy * dy);
            fx += pval[e] * w * dx;
            fy += pval[e] * w * dy;
        }
        F[2 * i] = fx;
        F[2 * i + 1] = fy;
    }
}

/* Z = sum_{k != l} (1 + |X_k - X_l|^2)^-1, exact O(n^2). */
double oracle_exact_Z(int64_t n, const double* X)
{
    double Z = 0.0;
#pragma omp parallel for reduction(+ : Z) schedule(dynamic, 64) if (n > 256)
    for (int64_t i = 0; i < n; ++i) {
        double zi = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double dx = X[2 * i] - X[2 * j], dy = X[2 * i + 1] - X[2 * j + 1];
            zi += 1.0 / (1.0 + dx * dx + dy * dy);
        }
        Z += zi;
    }
    return Z;
}

/*
 * O4a. Exact gradient of C = C_KL + C_CMP + C_ENT* (Eq. 1 with readings R1-R3):
 *   g_i = 4 lkl sum_{j != i} (p_ij - w_ij / Z) w_ij Delta_ij      (Eq. 6)
 *       + (lc / n) X_i                                            (C_CMP)
 *       - (lr / n^2) sum_{j != i} Delta_ij / (eps + r2_ij)        (Eq. 8 kernel)
 * P is given in CSR (symmetric, sum 1).  Writes g (n x 2) and returns Z.
 */
double oracle_exact_grad(int64_t n, const double* X, const int64_t* indptr, const int32_t* indices,
                         const double* pval, double lkl, double lc, double lr, double eps, double* g)
{
    double Z = oracle_exact_Z(n, X);
    double nn = (double)n;
#pragma omp parallel for schedule(dynamic, 64) if (n > 256)
    for (int64_t i = 0; i < n; ++i) {
        double ax = 0.0, ay = 0.0, rx = 0.0, ry = 0.0, ex = 0.0, ey = 0.0;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            int64_t j = indices[e];
            double dx = X[2 * i] - X[2 * j], dy = X[2 * i + 1] - X[2 * j + 1];
            double w = 1.0 / (1.0 + dx * dx + dy * dy);
            ax += pval[e] * w * dx;
            ay += pval[e] * w * dy;
        }
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double dx = X[2 * i] - X[2 * j], dy = X[2 * i + 1] - X[2 * j + 1];
            double r2 = dx * dx + dy * dy;
            double w = 1.0 / (1.0 + r2);
            rx += w * w * dx;
            ry += w * w * dy;
            double ke = 1.0 / (eps + r2);
            ex += ke * dx;
            ey += ke * dy;
        }
        g[2 * i] = 4.0 * lkl * (ax - rx / Z) + (lc / nn) * X[2 * i] - (lr / (nn * nn)) * ex;
        g[2 * i + 1] = 4.0 * lkl * (ay - ry / Z) + (lc / nn) * X[2 * i + 1] - (lr / (nn * nn)) * ey;
    }
    return Z;
}

/*
 * O4b. Exact cost (the gradient above is its derivative):
 *   C_KL  = lkl sum_{p_ij > 0} p_ij ln(p_ij Z / w_ij)           (Eq. 1/4; natural log R14)
 *   C_CMP = (lc / 2n) sum_i |X_i|^2                              (Eq. 1)
 *   C_ENT* = -(lr / 4n^2) sum_{i != j} ln(eps + r2_ij)           (reading R1 of PAPER.md:90)
 * out3 = {C_KL, C_CMP, C_ENT*}.
 */
void oracle_exact_cost(int64_t n, const double* X, const int64_t* indptr, const int32_t* indices,
                       const double* pval, double lkl, double lc, double lr, double eps, double* out3)
{
    double Z = oracle_exact_Z(n, X);
    double kl = 0.0, cmp = 0.0, ent = 0.0;
    double nn = (double)n;
#pragma omp parallel for reduction(+ : kl, cmp, ent) schedule(dynamic, 64) if (n > 256)
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            if (!(pval[e] > 0.0)) continue;
            int64_t j = indices[e];
            double dx = X[2 * i] - X[2 * j], dy = X[2 * i + 1] - X[2 * j + 1];
            double w = 1.0 / (1.0 + dx * dx + dy * dy);
            kl += pval[e] * log(pval[e] * Z / w);
        }
        cmp += X[2 * i] * X[2 * i] + X[2 * i + 1] * X[2 * i + 1];
        double ei = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double dx = X[2 * i] - X[2 * j], dy = X[2 * i + 1] - X[2 * j + 1];
            ei += log(eps + dx * dx + dy * dy);
        }
        ent += ei;
    }
    out3[0] = lkl * kl;
    out3[1] = lc / (2.0 * nn) * cmp;
    out3[2] = -lr / (4.0 * nn * nn) * ent;
}
