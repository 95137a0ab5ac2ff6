/*
 * gkr_svd.c -- CPU oracle (TEST INFRASTRUCTURE ONLY, never shipped or timed as
 * the product): economy SVD of a dense float64 matrix by Householder
 * bidiagonalisation followed by implicit-shift (Golub-Kahan-Reinsch) QR sweeps
 * on the bidiagonal.
 *
 * This restates the algorithm the reference's compiled backend runs
 * (/root/reference/pkg/src/rtcur/_backend/_core.pyx:24-249, contract in
 * py_kernels.py:29-54): tall case does the work (a wide input is transposed
 * and U/V swapped, _core.pyx:33-35), at most 75 sweeps per singular value
 * (_core.pyx:21) else failure, singular values made nonnegative and sorted
 * descending with a stable sort (_core.pyx:55-58).
 *
 * Storage: every matrix is column-major (Fortran order), element (i, j) of an
 * r-row matrix at [i + j * r].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#define GKR_MAX_SWEEPS 75

/* Column-space rotation: (X[:,a], X[:,b]) <- (c X[:,a] + s X[:,b], c X[:,b] - s X[:,a]). */
static void rot_cols(double *x, int64_t rows, int64_t a, int64_t b, double c, double s)
{
    double *xa = x + a * rows, *xb = x + b * rows;
    for (int64_t i = 0; i < rows; ++i) {
        double p = xa[i], q = xb[i];
        xa[i] = c * p + s * q;
        xb[i] = c * q - s * p;
    }
}

/*
 * Tall SVD: w (m x n, m >= n) is destroyed.  u: m x n, s: n, v: n x n (V, not V^T).
 * Returns 0 on success, 1 if a QR sweep did not converge.
 */
static int svd_tall(double *w, int64_t m, int64_t n, double *u, double *s, double *v)
{
    double *diag = calloc((size_t)n, sizeof(double));
    double *sup = calloc((size_t)n, sizeof(double)); /* sup[i] couples diag[i-1], diag[i] */
    unsigned char *lflag = calloc((size_t)n, 1), *rflag = calloc((size_t)n, 1);
    int status = 0;

    /* ---- Householder bidiagonalisation; reflectors kept where they annihilate ---- */
    for (int64_t k = 0; k < n; ++k) {
        double *col = w + k * m;
        double nrm2 = 0.0;
        for (int64_t i = k; i < m; ++i) nrm2 += col[i] * col[i];
        if (nrm2 > 0.0) {
            double nrm = sqrt(nrm2);
            double beta = -copysign(nrm, col[k]);
            col[k] -= beta;
            double vn2 = 0.0;
            for (int64_t i = k; i < m; ++i) vn2 += col[i] * col[i];
            double inv = 1.0 / sqrt(vn2);
            for (int64_t i = k; i < m; ++i) col[i] *= inv;
            for (int64_t j = k + 1; j < n; ++j) {
                double *cj = w + j * m, dot = 0.0;
                for (int64_t i = k; i < m; ++i) dot += col[i] * cj[i];
                dot *= 2.0;
                for (int64_t i = k; i < m; ++i) cj[i] -= dot * col[i];
            }
            lflag[k] = 1;
            diag[k] = beta;
        } else {
            diag[k] = 0.0;
        }
        if (k < n - 2) {
            /* right reflector on row k, columns k+1..n-1 (stride m) */
            double r2 = 0.0;
            for (int64_t j = k + 1; j < n; ++j) r2 += w[k + j * m] * w[k + j * m];
            if (r2 > 0.0) {
                double nrm = sqrt(r2);
                double beta = -copysign(nrm, w[k + (k + 1) * m]);
                w[k + (k + 1) * m] -= beta;
                double vn2 = 0.0;
                for (int64_t j = k + 1; j < n; ++j) vn2 += w[k + j * m] * w[k + j * m];
                double inv = 1.0 / sqrt(vn2);
                for (int64_t j = k + 1; j < n; ++j) w[k + j * m] *= inv;
                for (int64_t i = k + 1; i < m; ++i) {
                    double dot = 0.0;
                    for (int64_t j = k + 1; j < n; ++j) dot += w[i + j * m] * w[k + j * m];
                    dot *= 2.0;
                    for (int64_t j = k + 1; j < n; ++j) w[i + j * m] -= dot * w[k + j * m];
                }
                rflag[k] = 1;
                sup[k + 1] = beta;
            }
        } else if (k == n - 2) {
            sup[k + 1] = w[k + (k + 1) * m];
        }
    }

    /* ---- accumulate U = H_0 ... H_{n-1} [I_n; 0] and V = G_0 ... G_{n-3} ---- */
    memset(u, 0, sizeof(double) * (size_t)(m * n));
    for (int64_t j = 0; j < n; ++j) u[j + j * m] = 1.0;
    for (int64_t k = n - 1; k >= 0; --k) {
        if (!lflag[k]) continue;
        const double *hv = w + k * m;
        for (int64_t j = k; j < n; ++j) {
            double *uj = u + j * m, dot = 0.0;
            for (int64_t i = k; i < m; ++i) dot += hv[i] * uj[i];
            dot *= 2.0;
            for (int64_t i = k; i < m; ++i) uj[i] -= dot * hv[i];
        }
    }
    memset(v, 0, sizeof(double) * (size_t)(n * n));
    for (int64_t j = 0; j < n; ++j) v[j + j * n] = 1.0;
    for (int64_t k = n - 3; k >= 0; --k) {
        if (!rflag[k]) continue;
        for (int64_t j = k + 1; j < n; ++j) {
            double *vj = v + j * n, dot = 0.0;
            for (int64_t i = k + 1; i < n; ++i) dot += w[k + i * m] * vj[i];
            dot *= 2.0;
            for (int64_t i = k + 1; i < n; ++i) vj[i] -= dot * w[k + i * m];
        }
    }

    /* ---- implicit-shift QR on the bidiagonal ---- */
    double anorm = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double t = fabs(diag[i]) + fabs(sup[i]);
        if (t > anorm) anorm = t;
    }
    const double tol = DBL_EPSILON * anorm;

    for (int64_t k = n - 1; k >= 0 && !status; --k) {
        for (int sweep = 0; sweep < GKR_MAX_SWEEPS; ++sweep) {
            int64_t l = k;
            int cancel = 1;
            for (;;) {
                if (fabs(sup[l]) <= tol) { cancel = 0; break; }   /* sup[0] == 0 stops this */
                if (fabs(diag[l - 1]) <= tol) break;
                --l;
            }
            if (cancel) {
                /* diag[l-1] negligible: chase sup[l..k] out with left rotations */
                double c = 0.0, sn = 1.0;
                for (int64_t i = l; i <= k; ++i) {
                    double f = sn * sup[i];
                    sup[i] = c * sup[i];
                    if (fabs(f) <= tol) break;
                    double g = diag[i];
                    double h = hypot(f, g);
                    diag[i] = h;
                    c = g / h;
                    sn = -f / h;
                    rot_cols(u, m, l - 1, i, c, sn);
                }
            }
            double z = diag[k];
            if (l == k) {
                if (z < 0.0) {
                    diag[k] = -z;
                    for (int64_t i = 0; i < n; ++i) v[i + k * n] = -v[i + k * n];
                }
                break;
            }
            if (sweep == GKR_MAX_SWEEPS - 1) { status = 1; break; }

            /* shift from the trailing 2x2, then one bulge chase l..k */
            double x = diag[l], y = diag[k - 1], g = sup[k - 1], h = sup[k];
            double f = ((y - z) * (y + z) + (g - h) * (g + h)) / (2.0 * h * y);
            g = hypot(f, 1.0);
            f = ((x - z) * (x + z) + h * (y / (f + copysign(g, f)) - h)) / x;
            double c = 1.0, sn = 1.0;
            for (int64_t j = l; j < k; ++j) {
                int64_t i = j + 1;
                g = sup[i];
                y = diag[i];
                h = sn * g;
                g = c * g;
                double zz = hypot(f, h);
                sup[j] = zz;
                c = f / zz;
                sn = h / zz;
                f = x * c + g * sn;
                g = g * c - x * sn;
                h = y * sn;
                y = y * c;
                rot_cols(v, n, j, i, c, sn);
                zz = hypot(f, h);
                diag[j] = zz;
                if (zz != 0.0) {
                    zz = 1.0 / zz;
                    c = f * zz;
                    sn = h * zz;
                }
                f = c * g + sn * y;
                x = c * y - sn * g;
                rot_cols(u, m, j, i, c, sn);
            }
            sup[l] = 0.0;
            sup[k] = f;
            diag[k] = x;
        }
    }

    if (!status) {
        /* stable descending sort of the singular values, permuting U and V columns */
        int64_t *ord = malloc(sizeof(int64_t) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) ord[i] = i;
        for (int64_t i = 1; i < n; ++i) { /* insertion sort: stable, n is small */
            int64_t t = ord[i], j = i - 1;
            while (j >= 0 && diag[ord[j]] < diag[t]) { ord[j + 1] = ord[j]; --j; }
            ord[j + 1] = t;
        }
        double *ut = malloc(sizeof(double) * (size_t)(m * n));
        double *vt = malloc(sizeof(double) * (size_t)(n * n));
        for (int64_t j = 0; j < n; ++j) {
            s[j] = diag[ord[j]];
            memcpy(ut + j * m, u + ord[j] * m, sizeof(double) * (size_t)m);
            memcpy(vt + j * n, v + ord[j] * n, sizeof(double) * (size_t)n);
        }
        memcpy(u, ut, sizeof(double) * (size_t)(m * n));
        memcpy(v, vt, sizeof(double) * (size_t)(n * n));
        free(ut); free(vt); free(ord);
    }
    free(diag); free(sup); free(lflag); free(rflag);
    return status;
}

/*
 * Economy SVD: a (m x p, column-major) == u diag(s) vt.
 * u: m x q, s: q, vt: q x p, q = min(m, p), all column-major.
 * Returns 0 ok, 1 no convergence, 2 bad shape.
 */
int oracle_dense_svd(const double *a, int64_t m, int64_t p, double *u, double *s, double *vt)
{
    if (m < 1 || p < 1) return 2;
    if (m >= p) {
        double *w = malloc(sizeof(double) * (size_t)(m * p));
        double *v = malloc(sizeof(double) * (size_t)(p * p));
        memcpy(w, a, sizeof(double) * (size_t)(m * p));
        int st = svd_tall(w, m, p, u, s, v);
        /* vt = v^T */
        for (int64_t i = 0; i < p; ++i)
            for (int64_t j = 0; j < p; ++j) vt[i + j * p] = v[j + i * p];
        free(w); free(v);
        return st;
    }
    /* wide: decompose a^T (p x m) = U' S V'^T, so a = V' S U'^T */
    double *w = malloc(sizeof(double) * (size_t)(m * p));
    double *uu = malloc(sizeof(double) * (size_t)(p * m));
    double *vv = malloc(sizeof(double) * (size_t)(m * m));
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < p; ++j) w[j + i * p] = a[i + j * m];
    int st = svd_tall(w, p, m, uu, s, vv);
    memcpy(u, vv, sizeof(double) * (size_t)(m * m));            /* u = V' (m x m) */
    for (int64_t i = 0; i < m; ++i)                              /* vt = U'^T (m x p) */
        for (int64_t j = 0; j < p; ++j) vt[i + j * m] = uu[j + i * p];
    free(w); free(uu); free(vv);
    return st;
}
