/*
 * Host restatement of the synthetic-input generator jh_gen_butterfly
 * (paper_1401_2720_b200/csrc/jh_gen.cu) -- TEST INFRASTRUCTURE, NOT PRODUCT
 * CODE.  It exists so the C oracle can solve exactly the matrix the GPU
 * bench solves: tests/test_gen.py pins the GPU kernel bitwise against this
 * file, and tools/oracle_offline.py runs the whole-solve oracle on its output.
 *
 * G (m x n, column-major) = Q [diag(sigma); 0] W^T, built in place:
 *   1. G = 0, G[j][j] = sigma[j].
 *   2. column layers on the top n rows (right-multiplication by W^T):
 *      for pass in [0, passes): for l in [0, log2(cls)): within each
 *      signature class of width cls (the whole n, or the halves when
 *      n_plus = n/2), rotate columns (j, j + h), h = 2^l, for every j with
 *      bit l clear;  after every pass, when n_plus = n/2, one hyperbolic
 *      layer pairs column j with column j + n/2 (J-orthogonal mixing).
 *   3. row layers over all m rows (left-multiplication by Q): passes x
 *      log2(m) butterflies on row pairs (i, i + h).
 * Every rotation draws one 53-bit uniform u from a counter hash of
 * (seed, layer, pair) and uses only correctly rounded + - * / sqrt:
 *   t = 2u - 1 (exact);  trig: d = 1 + t*t, c = (1 - t*t)/d, s = (2t)/d,
 *   x' = c*x - s*y, y' = s*x + c*y;
 *   hyperbolic: th = tanh_max*t, ch = 1/sqrt(1 - th*th), sh = th*ch,
 *   x' = ch*x + sh*y, y' = sh*x + ch*y.
 * Compiled with -ffp-contract=off, so nothing is fused; the CUDA kernel uses
 * the same explicitly rounded operations.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double draw_t(uint64_t seed, uint64_t layer, uint64_t pair) {
    uint64_t h = mix64(mix64(seed * 0x9E3779B97F4A7C15ULL + layer) ^ (pair * 0xD1B54A32D192ED03ULL));
    double u = (double)(h >> 11) * 0x1p-53;
    return 2.0 * u - 1.0;
}

static void trig_cs(double t, double *c, double *s) {
    double t2 = t * t;
    double d = 1.0 + t2;
    *c = (1.0 - t2) / d;
    *s = (2.0 * t) / d;
}

static void hyp_cs(double t, double tanh_max, double *ch, double *sh) {
    double th = tanh_max * t;
    *ch = 1.0 / sqrt(1.0 - th * th);
    *sh = th * *ch;
}

static int ilog2(int64_t x) {
    int k = 0;
    while (((int64_t)1 << (k + 1)) <= x) k++;
    return k;
}

/* returns 0, or -1 for unsupported shapes (m, n and the class widths must be
 * powers of two, n_plus in {n, n/2}).  Rows are independent under the column
 * layers and columns under the row layers, so each phase runs all its layers
 * on one cache-resident tile at a time; per element the operation sequence is
 * the layer order above. */
int or_gen_butterfly(double *g, int64_t ldg, int64_t m, int64_t n, const double *sigma,
                     int64_t n_plus, uint64_t seed, int passes, double tanh_max) {
    if (m < n || n < 2 || (m & (m - 1)) || (n & (n - 1)) || ldg < m || passes < 1) return -1;
    if (n_plus != n && n_plus != n / 2) return -1;
    int64_t cls = (n_plus == n) ? n : n / 2;
    int lc = ilog2(cls), lr = ilog2(m);
    int hyp = cls != n;
    int ncl = passes * (lc + hyp);          /* column layers */
    int nrl = passes * lr;                  /* row layers */
    double *ccs = (double *)malloc(sizeof(double) * (size_t)ncl * (size_t)n);  /* [layer][n/2][2] */
    double *rcs = (double *)malloc(sizeof(double) * (size_t)nrl * (size_t)m);  /* [layer][m/2][2] */
    int *ckind = (int *)malloc(sizeof(int) * (size_t)ncl);  /* -1 hyperbolic, else log2 h */
    if (!ccs || !rcs || !ckind) { free(ccs); free(rcs); free(ckind); return -2; }
    uint64_t layer = 0;
    int cl = 0;
    for (int p = 0; p < passes; p++) {
        for (int l = 0; l < lc; l++, layer++, cl++) {
            ckind[cl] = l;
            for (int64_t k = 0; k < n / 2; k++)
                trig_cs(draw_t(seed, layer, (uint64_t)k), ccs + ((int64_t)cl * n + 2 * k),
                        ccs + ((int64_t)cl * n + 2 * k + 1));
        }
        if (hyp) {
            ckind[cl] = -1;
            for (int64_t k = 0; k < n / 2; k++)
                hyp_cs(draw_t(seed, layer, (uint64_t)k), tanh_max, ccs + ((int64_t)cl * n + 2 * k),
                       ccs + ((int64_t)cl * n + 2 * k + 1));
            layer++, cl++;
        }
    }
    for (int rl = 0; rl < nrl; rl++, layer++)
        for (int64_t k = 0; k < m / 2; k++)
            trig_cs(draw_t(seed, layer, (uint64_t)k), rcs + ((int64_t)rl * m + 2 * k),
                    rcs + ((int64_t)rl * m + 2 * k + 1));

    /* 1 + 2: row i of the top block starts as sigma_i e_i^T */
#pragma omp parallel
    {
        double *row = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            memset(row, 0, sizeof(double) * (size_t)n);
            row[i] = sigma[i];
            for (int c = 0; c < ncl; c++) {
                const double *cs = ccs + (int64_t)c * n;
                if (ckind[c] < 0) {
                    for (int64_t k = 0; k < n / 2; k++) {
                        double ch = cs[2 * k], sh = cs[2 * k + 1];
                        double x = row[k], y = row[k + n / 2];
                        row[k] = ch * x + sh * y;
                        row[k + n / 2] = sh * x + ch * y;
                    }
                } else {
                    int l = ckind[c];
                    int64_t h = (int64_t)1 << l;
                    for (int64_t base = 0; base < n; base += cls) {
                        for (int64_t k = 0; k < cls / 2; k++) {
                            int64_t j = base + (((k >> l) << (l + 1)) | (k & (h - 1)));
                            int64_t kk = base / 2 + k;
                            double c0 = cs[2 * kk], s0 = cs[2 * kk + 1];
                            double x = row[j], y = row[j + h];
                            row[j] = c0 * x - s0 * y;
                            row[j + h] = s0 * x + c0 * y;
                        }
                    }
                }
            }
            for (int64_t j = 0; j < n; j++) g[j * ldg + i] = row[j];
        }
        free(row);
    }
    /* 3: rows below n start at zero; the row layers mix each column */
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; j++) {
        double *col = g + j * ldg;
        for (int64_t i = n; i < m; i++) col[i] = 0.0;
        for (int rl = 0; rl < nrl; rl++) {
            int l = rl % lr;
            int64_t h = (int64_t)1 << l;
            const double *cs = rcs + (int64_t)rl * m;
            for (int64_t k = 0; k < m / 2; k++) {
                int64_t i = ((k >> l) << (l + 1)) | (k & (h - 1));
                double c0 = cs[2 * k], s0 = cs[2 * k + 1];
                double x = col[i], y = col[i + h];
                col[i] = c0 * x - s0 * y;
                col[i + h] = s0 * x + c0 * y;
            }
        }
    }
    free(ccs); free(rcs); free(ckind);
    return 0;
}
