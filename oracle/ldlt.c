/*
 * ORACLE (test infrastructure only -- see oracle/__init__.py): a plain sparse LDL^T direct
 * solver for the per-node FEM systems of the definition
 *
 *     A^{(l)} x = b,   A^{(l)} = c_I M_L + c_L (kappa^2 M_L + G)          (PAPER.md P75-78, P76)
 *
 * with a FIXED symmetric ordering chosen by the caller (oracle/ldlt.py: the edge-interior DOFs
 * first in their natural order, then the vertex block under a fill-reducing order -- SURVEY
 * §8c-O7, §7.3-5).  No pivoting: every A^{(l)} is symmetric positive definite (M_L > 0 diagonal,
 * G positive semidefinite, c_I, c_L > 0).  Nothing here knows about edges, Thomas, Schur
 * complements or PCG: it is the textbook up-looking sparse LDL^T (elimination tree from the
 * symmetric pattern, row k of L by a sparse triangular solve along the tree; the algorithm of
 * T. A. Davis, "Algorithm 849: a concise sparse Cholesky factorization package", ACM TOMS 31,
 * 2005), restated here in our own code, followed by forward / diagonal / backward substitution.
 *
 * Matrix input: the full symmetric pattern of A in compressed-column form (Ap, Ai), both
 * triangles, every diagonal entry present; values are formed from G's values, M_L and the
 * node's scalars.  perm[k] = original index of the k-th pivot, pinv its inverse.
 *
 * Built by oracle/ldlt.py with `gcc -O2 -ffp-contract=off -shared -fPIC` (no FMA contraction:
 * plain IEEE arithmetic in the order written).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Symbolic analysis of P A P^T: elimination tree parent[] and the column counts of L
 * (lnz[j] = number of off-diagonal entries in column j of L).  Returns total nnz(L). */
int64_t ldlt_symbolic(int64_t n, const int64_t* Ap, const int64_t* Ai, const int64_t* perm,
                      const int64_t* pinv, int64_t* parent, int64_t* lnz, int64_t* flag) {
    for (int64_t k = 0; k < n; ++k) {
        parent[k] = -1;
        flag[k] = k;
        lnz[k] = 0;
        const int64_t kk = perm[k];
        for (int64_t p = Ap[kk]; p < Ap[kk + 1]; ++p) {
            int64_t i = pinv[Ai[p]];
            if (i >= k) continue;               /* upper triangle of the permuted matrix only */
            for (; flag[i] != k; i = parent[i]) {  /* walk up the tree to the first marked node */
                if (parent[i] == -1) parent[i] = k;
                lnz[i]++;                        /* L(k, i) is nonzero */
                flag[i] = k;
            }
        }
    }
    int64_t tot = 0;
    for (int64_t k = 0; k < n; ++k) tot += lnz[k];
    return tot;
}

/* Numeric factorization P A P^T = L D L^T, A = cI * diag(ML) + cL * (kappa2 * diag(ML) + G)
 * where G has the pattern (Ap, Ai) and values Gx (its diagonal included).
 * Lp[n+1] column pointers (from lnz), Li / Lx columns of L (unit diagonal not stored), D[n].
 * Work: y[n] (zero on entry), pattern[n], flag[n], cnt[n].  Returns -1 on success, else the
 * pivot k where D(k) <= 0 (the matrix is not positive definite). */
int64_t ldlt_numeric(int64_t n, const int64_t* Ap, const int64_t* Ai, const double* Gx, const double* ML,
                     double cI, double cL, double kappa2, const int64_t* perm, const int64_t* pinv,
                     const int64_t* parent, const int64_t* Lp, int64_t* Li, double* Lx, double* D, double* y,
                     int64_t* pattern, int64_t* flag, int64_t* cnt) {
    for (int64_t k = 0; k < n; ++k) {
        y[k] = 0.0;
        int64_t top = n;
        flag[k] = k;
        cnt[k] = 0;
        const int64_t kk = perm[k];
        for (int64_t p = Ap[kk]; p < Ap[kk + 1]; ++p) {
            const int64_t j = Ai[p];
            int64_t i = pinv[j];
            if (i > k) continue;
            /* A(j, kk) = cL G(j, kk) + [j == kk] (cI + cL kappa2) ML(kk)   (P76) */
            double a = cL * Gx[p];
            if (j == kk) a += (cI + cL * kappa2) * ML[kk];
            y[i] += a;
            int64_t len = 0;
            for (; flag[i] != k; i = parent[i]) {  /* nonzero pattern of row k of L */
                pattern[len++] = i;
                flag[i] = k;
            }
            while (len > 0) pattern[--top] = pattern[--len];
        }
        D[k] = y[k];
        y[k] = 0.0;
        for (; top < n; ++top) {  /* sparse triangular solve L(0:k-1, 0:k-1) l = a(0:k-1) */
            const int64_t i = pattern[top];
            const double yi = y[i];
            y[i] = 0.0;
            const int64_t p2 = Lp[i] + cnt[i];
            for (int64_t p = Lp[i]; p < p2; ++p) y[Li[p]] -= Lx[p] * yi;
            const double lki = yi / D[i];
            D[k] -= lki * yi;
            Li[p2] = k;
            Lx[p2] = lki;
            cnt[i]++;
        }
        if (!(D[k] > 0.0)) return k;
    }
    return -1;
}

/* Solve A x = b for nrhs right-hand sides (row-major [nrhs][n], b and x may alias) with the
 * factors of ldlt_numeric: x = P^T L^{-T} D^{-1} L^{-1} P b.  w[n] work. */
void ldlt_solve(int64_t n, int64_t nrhs, const int64_t* perm, const int64_t* Lp, const int64_t* Li,
                const double* Lx, const double* D, const double* b, double* x, double* w) {
    for (int64_t r = 0; r < nrhs; ++r) {
        const double* br = b + r * n;
        double* xr = x + r * n;
        for (int64_t k = 0; k < n; ++k) w[k] = br[perm[k]];
        for (int64_t j = 0; j < n; ++j) {          /* L y = P b */
            const double wj = w[j];
            for (int64_t p = Lp[j]; p < Lp[j + 1]; ++p) w[Li[p]] -= Lx[p] * wj;
        }
        for (int64_t j = 0; j < n; ++j) w[j] /= D[j];  /* D z = y */
        for (int64_t j = n - 1; j >= 0; --j) {      /* L^T v = z */
            double s = w[j];
            for (int64_t p = Lp[j]; p < Lp[j + 1]; ++p) s -= Lx[p] * w[Li[p]];
            w[j] = s;
        }
        for (int64_t k = 0; k < n; ++k) xr[perm[k]] = w[k];
    }
}

/* One node of the quadrature, start to finish (convenience for the threaded driver in
 * oracle/ldlt.py; releases nothing, allocates its own factor and work arrays):
 * x[r] = (A^{(l)})^{-1} b[r].  Returns -1 on success, -2 on allocation failure, else the
 * failing pivot. */
int64_t ldlt_node_solve(int64_t n, const int64_t* Ap, const int64_t* Ai, const double* Gx, const double* ML,
                        double cI, double cL, double kappa2, const int64_t* perm, const int64_t* pinv,
                        const int64_t* parent, const int64_t* Lp, int64_t nrhs, const double* b, double* x) {
    const int64_t nnz = Lp[n];
    int64_t* Li = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    double* Lx = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    double* D = (double*)malloc(sizeof(double) * (size_t)n);
    double* y = (double*)calloc((size_t)n, sizeof(double));
    int64_t* pattern = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* flag = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t rc = -2;
    if (Li && Lx && D && y && pattern && flag && cnt) {
        rc = ldlt_numeric(n, Ap, Ai, Gx, ML, cI, cL, kappa2, perm, pinv, parent, Lp, Li, Lx, D, y, pattern, flag,
                          cnt);
        if (rc == -1) ldlt_solve(n, nrhs, perm, Lp, Li, Lx, D, b, x, y);
    }
    free(Li);
    free(Lx);
    free(D);
    free(y);
    free(pattern);
    free(flag);
    free(cnt);
    return rc;
}
