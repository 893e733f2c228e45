/*
 * jhsvd_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the reference `jhsvd` hot path (pure Python +
 * numba in /root/reference/pkg/src/jhsvd), used only as
 *   - the parity checker of the CUDA path in tests/ and __graft_entry__.smoke(),
 *   - the CPU baseline leg of bench.py (cpu_baseline / --impl reference).
 * The product (paper_1401_2720_b200) never links, loads or calls this code.
 *
 * Every floating-point operation follows the reference's operation order:
 * fused multiply-adds where the reference calls _fp.fma (llvm.fma.f64),
 * separate multiply/add elsewhere (numba fastmath=False never contracts),
 * IEEE division and square root.  Compile with -ffp-contract=off.
 * Parity of this restatement with the reference is pinned by
 * tests/test_oracle_golden.py against fixtures generated from the reference
 * itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define EPS_U 0x1p-53
static const double MU_ = 0x1p-1022;                        /* robustnorm.py:36 */
/* ldexp(2 - 2**-52, 1022): the reference NU is 2**1023 - 2**970, half the
 * largest double (robustnorm.py:38); kept as is, it feeds safe_bounds */
static const double NU_ = 0x1.fffffffffffffp+1022;
static const double GAMMA_ = 1.0 - 0x1p-53;                 /* robustnorm.py:41 */
static const double DELTA_ = 1.0 + 0x1p-53;                 /* robustnorm.py:42 */
#define CHUNK_ 256                                          /* robustnorm.py:45 */
#define GRAM_CHUNK_ 64                                      /* blockkernel.py:27 */

/* ------------------------------------------------------------------------ */
/* double-double helpers (_fp.py:46-157), used only for safe_bounds           */

static void two_sum(double a, double b, double *s, double *e) {
    double ss = a + b, v = ss - a;
    *s = ss;
    *e = (a - (ss - v)) + (b - v);
}
static void quick_two_sum(double a, double b, double *s, double *e) {
    double ss = a + b;
    *s = ss;
    *e = b - (ss - a);
}
static void two_prod(double a, double b, double *p, double *e) {
    double pp = a * b;
    *p = pp;
    *e = fma(a, b, -pp);
}
static void dd_add(double ah, double al, double bh, double bl, double *rh, double *rl) {
    double s1, s2, t1, t2;
    two_sum(ah, bh, &s1, &s2);
    two_sum(al, bl, &t1, &t2);
    s2 += t1;
    quick_two_sum(s1, s2, &s1, &s2);
    s2 += t2;
    quick_two_sum(s1, s2, rh, rl);
}
static void dd_add_d(double ah, double al, double b, double *rh, double *rl) {
    double s1, s2;
    two_sum(ah, b, &s1, &s2);
    s2 += al;
    quick_two_sum(s1, s2, rh, rl);
}
static void dd_mul(double ah, double al, double bh, double bl, double *rh, double *rl) {
    double p1, p2;
    two_prod(ah, bh, &p1, &p2);
    p2 += ah * bl + al * bh;
    quick_two_sum(p1, p2, rh, rl);
}
static void dd_mul_d(double ah, double al, double b, double *rh, double *rl) {
    double p1, p2;
    two_prod(ah, b, &p1, &p2);
    p2 += al * b;
    quick_two_sum(p1, p2, rh, rl);
}
static void dd_div(double ah, double al, double bh, double bl, double *rh, double *rl) {
    double q1 = ah / bh, th, tl, xh, xl, q2, q3;
    dd_mul_d(bh, bl, q1, &th, &tl);
    dd_add(ah, al, -th, -tl, &xh, &xl);
    q2 = xh / bh;
    dd_mul_d(bh, bl, q2, &th, &tl);
    dd_add(xh, xl, -th, -tl, &xh, &xl);
    q3 = xh / bh;
    quick_two_sum(q1, q2, &q1, &q2);
    dd_add_d(q1, q2, q3, rh, rl);
}
static void dd_sqrt(double ah, double al, double *rh, double *rl) {
    if (ah == 0.0) { *rh = 0.0; *rl = 0.0; return; }
    double s = sqrt(ah), ph, pl, xh, xl, e;
    two_prod(s, s, &ph, &pl);
    dd_add(ah, al, -ph, -pl, &xh, &xl);
    e = xh / (2.0 * s);
    quick_two_sum(s, e, rh, rl);
}

/* ------------------------------------------------------------------------ */
/* robust norms (robustnorm.py:71-308)                                        */

static int reduction_depth(int64_t n) {              /* robustnorm.py:71-80 */
    int d = 0;
    int64_t m = n - 1;
    while (m > 0) { m >>= 1; d++; }
    return d > 1 ? d : 1;
}

void or_safe_bounds(int64_t n, double *mu_tilde, double *nu_hat) { /* :90-101 */
    int d = reduction_depth(n);
    double h, l, sh, sl;
    dd_div(MU_, 0.0, GAMMA_, 0.0, &h, &l);
    dd_sqrt(h, l, &sh, &sl);
    *mu_tilde = (sl > 0.0) ? nextafter(sh, INFINITY) : sh;
    double dh = 1.0, dl = 0.0;
    for (int i = 0; i < d + 1; i++) dd_mul(dh, dl, DELTA_, 0.0, &dh, &dl);
    dh = ldexp(dh, d);
    dl = ldexp(dl, d);
    dd_div(NU_, 0.0, dh, dl, &h, &l);
    dd_sqrt(h, l, &sh, &sl);
    *nu_hat = (sl < 0.0) ? nextafter(sh, 0.0) : sh;
}

static int scale_exponent(double f, double t, int up) { /* robustnorm.py:116-122 */
    int fe, te;
    double fy = frexp(f, &fe), ty = frexp(t, &te);
    if (up) return (te - fe) + (fy < ty ? 1 : 0);
    return (te - fe) - (fy > ty ? 1 : 0);
}

static void common_form(int64_t j, double v, int64_t *jo, double *vo) { /* :138-147 */
    if (v == 0.0) { *jo = 0; *vo = 0.0; return; }
    int fe;
    double fy = frexp(v, &fe);
    double y = 2.0 * fy;
    int64_t m = fe - 1;
    int64_t mp = (m & 1) ? -1 : 0;
    *jo = j + m - mp;
    *vo = ldexp(y, (int)mp);
}

static void add_scaled(int64_t ja, double va, int64_t jb, double vb, int64_t *jo, double *vo) {
    /* robustnorm.py:150-162 */
    if (va == 0.0) { *jo = jb; *vo = vb; return; }
    if (vb == 0.0) { *jo = ja; *vo = va; return; }
    int64_t js, jbig;
    double vs, vbig;
    if (ja < jb || (ja == jb && va <= vb)) { js = ja; vs = va; jbig = jb; vbig = vb; }
    else { js = jb; vs = vb; jbig = ja; vbig = va; }
    double shifted = ldexp(vs, (int)(js - jbig));
    *jo = jbig;
    *vo = shifted + vbig;
}

static double tree_combine(double *p, int64_t k) {   /* robustnorm.py:184-194 */
    while (k > 1) {
        int64_t half = (k + 1) / 2;
        for (int64_t i = 0; i < k / 2; i++) p[i] = p[2 * i] + p[2 * i + 1];
        if (k % 2) p[half - 1] = p[k - 1];
        k = half;
    }
    return p[0];
}

static double tree_sumsq_plain(const double *x, int64_t n, double *part) { /* :197-208 */
    int64_t nleaf = (n + CHUNK_ - 1) / CHUNK_;
    for (int64_t c = 0; c < nleaf; c++) {
        double acc = 0.0;
        int64_t end = (c + 1) * CHUNK_ < n ? (c + 1) * CHUNK_ : n;
        for (int64_t i = c * CHUNK_; i < end; i++) acc = fma(x[i], x[i], acc);
        part[c] = acc;
    }
    return tree_combine(part, nleaf);
}

static double tree_sumsq_selected(const double *x, int64_t n, double lo, double hi,
                                  int j, double *part) { /* robustnorm.py:211-226 */
    int64_t nleaf = (n + CHUNK_ - 1) / CHUNK_;
    for (int64_t c = 0; c < nleaf; c++) {
        double acc = 0.0;
        int64_t end = (c + 1) * CHUNK_ < n ? (c + 1) * CHUNK_ : n;
        for (int64_t i = c * CHUNK_; i < end; i++) {
            double a = fabs(x[i]);
            if (a > 0.0 && lo <= a && a <= hi) {
                double v = ldexp(x[i], j);
                acc = fma(v, v, acc);
            }
        }
        part[c] = acc;
    }
    return tree_combine(part, nleaf);
}

/* (scale_exp, value) in common form; robustnorm.py:242-292 */
void or_sum_squares(const double *x, int64_t n, int force_scaled, int64_t *jo, double *vo) {
    *jo = 0; *vo = 0.0;
    if (n == 0) return;
    double big = 0.0, m = NU_;
    for (int64_t i = 0; i < n; i++) {
        double a = fabs(x[i]);
        if (a > big) big = a;
        if (0.0 < a && a < m) m = a;
    }
    if (big == 0.0) return;
    double *part = (double *)malloc(sizeof(double) * (size_t)((n + CHUNK_ - 1) / CHUNK_));
    if (!force_scaled) {
        double plain = tree_sumsq_plain(x, n, part);
        if (isfinite(plain) && m * m >= MU_) {
            common_form(0, plain, jo, vo);
            free(part);
            return;
        }
    }
    double mu_tilde, nu_hat;
    or_safe_bounds(n, &mu_tilde, &nu_hat);
    int64_t js[3] = {0, 0, 0};
    double vs[3] = {0.0, 0.0, 0.0};
    int count = 0;
    if (m <= nu_hat && big >= mu_tilde) {
        double s1 = tree_sumsq_selected(x, n, mu_tilde, nu_hat, 0, part);
        if (s1 != 0.0) { common_form(0, s1, &js[count], &vs[count]); count++; }
    }
    if (big > nu_hat) {
        int j2 = scale_exponent(big, nu_hat, 0);
        double s2 = tree_sumsq_selected(x, n, nextafter(nu_hat, NU_), NU_, j2, part);
        if (s2 != 0.0) { common_form(-2 * (int64_t)j2, s2, &js[count], &vs[count]); count++; }
    }
    if (m < mu_tilde) {
        int j0 = scale_exponent(m, mu_tilde, 1);
        double s0 = tree_sumsq_selected(x, n, 0.0, nextafter(mu_tilde, 0.0), j0, part);
        if (s0 != 0.0) { common_form(-2 * (int64_t)j0, s0, &js[count], &vs[count]); count++; }
    }
    free(part);
    if (count == 0) return;
    for (int a = 0; a < count - 1; a++)
        for (int b = a + 1; b < count; b++)
            if (js[a] > js[b] || (js[a] == js[b] && vs[a] > vs[b])) {
                int64_t tj = js[a]; js[a] = js[b]; js[b] = tj;
                double tv = vs[a]; vs[a] = vs[b]; vs[b] = tv;
            }
    int64_t ja = js[0];
    double va = vs[0];
    for (int k = 1; k < count; k++) {
        common_form(ja, va, &ja, &va);
        add_scaled(ja, va, js[k], vs[k], &ja, &va);
    }
    common_form(ja, va, jo, vo);
}

/* norm2: (js, sigma) with ||x|| = sigma / 2**js; robustnorm.py:295-300 */
void or_norm2(const double *x, int64_t n, int force_scaled, int64_t *js, double *sigma) {
    int64_t j;
    double v;
    or_sum_squares(x, n, force_scaled, &j, &v);
    if (v == 0.0) { *js = 0; *sigma = 0.0; return; }
    /* j is even in common form: Python's -(j // 2) */
    int64_t q = j / 2;
    if ((j % 2) && j < 0) q -= 1;
    *js = -q;
    *sigma = sqrt(v);
}

static double norm2_unscaled(const double *x, int64_t n) { /* robustnorm.py:303-308 */
    int64_t js;
    double s;
    or_norm2(x, n, 0, &js, &s);
    return ldexp(s, (int)(-js));
}

/* ------------------------------------------------------------------------ */
/* shortening kernels (blockkernel.py:76-244)                                 */

/* h = a^T a, lower triangle by one in-order fma chain over the rows, then
 * mirrored (blockkernel.py:76-96).  The chain of every entry runs over rows
 * in ascending order; the loop nest here is reordered only across entries. */
void or_gram(const double *a, int64_t lda, int64_t m, int c, double *h) {
    double *t = (double *)malloc(sizeof(double) * (size_t)c * GRAM_CHUNK_);
    double *acc = (double *)calloc((size_t)c * c, sizeof(double)); /* acc[y*c+x] */
    for (int64_t c0 = 0; c0 < m; c0 += GRAM_CHUNK_) {
        int64_t c1 = c0 + GRAM_CHUNK_ < m ? c0 + GRAM_CHUNK_ : m;
        int64_t nr = c1 - c0;
        for (int x = 0; x < c; x++)
            for (int64_t i = 0; i < nr; i++) t[i * c + x] = a[(int64_t)x * lda + c0 + i];
        for (int64_t i = 0; i < nr; i++) {
            const double *row = t + i * c;
            for (int y = 0; y < c; y++) {
                double gy = row[y];
                double *hy = acc + (int64_t)y * c;
                for (int x = y; x < c; x++) hy[x] = fma(row[x], gy, hy[x]);
            }
        }
    }
    for (int y = 0; y < c; y++)
        for (int x = y; x < c; x++) {
            h[(int64_t)y * c + x] = acc[(int64_t)y * c + x];   /* h[x, y] */
            h[(int64_t)x * c + y] = acc[(int64_t)y * c + x];   /* h[y, x] */
        }
    free(t);
    free(acc);
}

/* forward-looking in-place Cholesky on the lower triangle; 0 or the 1-based
 * index of the bad pivot (blockkernel.py:110-127) */
int or_cholesky(double *h, int c) {
    for (int k = 0; k < c; k++) {
        double d = h[(int64_t)k * c + k];
        if (!(d > 0.0) || !isfinite(d)) return k + 1;
        double l = sqrt(d);
        h[(int64_t)k * c + k] = l;
        for (int x = k + 1; x < c; x++) h[(int64_t)k * c + x] = h[(int64_t)k * c + x] / l;
        for (int j = k + 1; j < c; j++) {
            double ljk = h[(int64_t)k * c + j];
            for (int x = j; x < c; x++)
                h[(int64_t)j * c + x] = fma(-h[(int64_t)k * c + x], ljk, h[(int64_t)j * c + x]);
        }
    }
    return 0;
}

/* R = L^T with zero strict lower triangle (blockkernel.py:454-458) */
static void lower_to_r(const double *h, int c, double *r) {
    for (int j = 0; j < c; j++)
        for (int i = 0; i < c; i++)
            r[(int64_t)j * c + i] = (i <= j) ? h[(int64_t)i * c + j] : 0.0;
}

static double hypot2(double a, double b) {            /* blockkernel.py:148-158 */
    double aa = fabs(a), ab = fabs(b);
    double big = aa >= ab ? aa : ab;
    if (big == 0.0) return 0.0;
    int e;
    frexp(big, &e);
    double as = ldexp(aa, -e), bs = ldexp(ab, -e);
    return ldexp(sqrt(fma(as, as, bs * bs)), e);
}

static void householder_qr(double *a, int c) {        /* blockkernel.py:161-188 */
#define A_(i, j) a[(int64_t)(j) * c + (i)]
    for (int k = 0; k < c - 1; k++) {
        double alpha = A_(k, k);
        double xnorm = norm2_unscaled(&A_(k + 1, k), c - k - 1);
        if (xnorm == 0.0) continue;
        double nr = hypot2(alpha, xnorm);
        double beta = alpha >= 0.0 ? -nr : nr;
        double tau = (beta - alpha) / beta;
        double denom = alpha - beta;
        for (int i = k + 1; i < c; i++) A_(i, k) = A_(i, k) / denom;
        A_(k, k) = beta;
        for (int j = k + 1; j < c; j++) {
            double z = A_(k, j);
            for (int i = k + 1; i < c; i++) z = fma(A_(i, k), A_(i, j), z);
            double tz = tau * z;
            A_(k, j) = A_(k, j) - tz;
            for (int i = k + 1; i < c; i++) A_(i, j) = fma(-tz, A_(i, k), A_(i, j));
        }
    }
    for (int j = 0; j < c; j++)
        for (int i = j + 1; i < c; i++) A_(i, j) = 0.0;
#undef A_
}

static void givens(double a, double b, double *cc, double *ss) { /* :191-201 */
    double aa = fabs(a), ab = fabs(b);
    double big = aa >= ab ? aa : ab;
    int e;
    frexp(big, &e);
    double as = ldexp(a, -e), bs = ldexp(b, -e);
    double d = sqrt(fma(as, as, bs * bs));
    *cc = as / d;
    *ss = bs / d;
}

static void peel_combine(double *r0, double *r1, int c) { /* blockkernel.py:204-220 */
    for (int k = 0; k < c; k++)
        for (int x = k; x < c; x++) {
            int xr = x - k;
            double b = r1[(int64_t)x * c + xr];
            if (b == 0.0) continue;
            double cc, ss;
            givens(r0[(int64_t)x * c + x], b, &cc, &ss);
            for (int j = x; j < c; j++) {
                double v0 = r0[(int64_t)j * c + x];
                double v1 = r1[(int64_t)j * c + xr];
                r0[(int64_t)j * c + x] = fma(ss, v1, cc * v0);
                r1[(int64_t)j * c + xr] = fma(cc, v1, -(ss * v0));
            }
        }
}

/* upper-triangular factor by per-chunk Householder QR + Givens peel-off;
 * m must be a positive multiple of c (blockkernel.py:223-244) */
int or_qr_peeloff(const double *g, int64_t ldg, int64_t m, int c, double *r0) {
    if (m % c || m < c) return -1;
    double *r1 = (double *)malloc(sizeof(double) * (size_t)c * c);
    for (int j = 0; j < c; j++)
        for (int i = 0; i < c; i++) r0[(int64_t)j * c + i] = g[(int64_t)j * ldg + i];
    householder_qr(r0, c);
    for (int64_t start = c; start < m; start += c) {
        for (int j = 0; j < c; j++)
            for (int i = 0; i < c; i++) r1[(int64_t)j * c + i] = g[(int64_t)j * ldg + start + i];
        householder_qr(r1, c);
        peel_combine(r0, r1, c);
    }
    for (int i = 0; i < c; i++)
        if (r0[(int64_t)i * c + i] < 0.0)
            for (int j = i; j < c; j++) r0[(int64_t)j * c + i] = -r0[(int64_t)j * c + i];
    free(r1);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* rotations (rotation.py:71-102) and the inner pointwise Jacobi              */

/* returns ok; *cs = cs2, *tn (rotation.py:90-102 with :71-87) */
static int rotation_core(double hpp, double hqq, double hpq, double t, double *cs, double *tn) {
    double h = hqq - t * hpp;
    double ct2 = t * (h / (2.0 * hpq));
    if (t < 0.0) {
        if (fabs(ct2) == 1.0) ct2 = ct2 > 0.0 ? 1.25 : -1.25;
        else if (fabs(ct2) < 1.0) { *cs = 0.0; *tn = 0.0; return 0; }
    }
    double a = fabs(ct2);
    double sgn = ct2 >= 0.0 ? 1.0 : -1.0;
    if (a >= 0x1p27) {                    /* _CT2_HUGE = 2**27 */
        double ct = 2.0 * a;
        *tn = sgn / ct;
        *cs = 1.0;
        return 1;
    }
    double ct;
    if (t > 0.0 && a < sqrt(0x1p-53)) ct = a + 1.0;   /* _CT2_TINY = sqrt(eps) */
    else ct = a + sqrt(fma(ct2, ct2, t));
    *tn = sgn / ct;
    /* cs1 = 1/sqrt(fma(t*tn, tn, 1)) is computed by the reference but unused */
    *cs = ct / sqrt(fma(ct, ct, t));
    return 1;
}

void or_rotation(double hpp, double hqq, double hpq, double t, double *out3) {
    double cs, tn;
    int ok = rotation_core(hpp, hqq, hpq, t, &cs, &tn);
    out3[0] = cs; out3[1] = tn; out3[2] = ok;
}

static void apply_rotation(double *mat, int c, int p, int q, double cs, double tn, int hyp) {
    /* blockkernel.py:251-266 */
    double s = hyp ? tn : -tn;
    double *cp = mat + (int64_t)p * c, *cq = mat + (int64_t)q * c;
    if (cs != 1.0) {
        for (int i = 0; i < c; i++) {
            double gp = cp[i], gq = cq[i];
            cp[i] = fma(s, gq, gp) * cs;
            cq[i] = fma(tn, gp, gq) * cs;
        }
    } else {
        for (int i = 0; i < c; i++) {
            double gp = cp[i], gq = cq[i];
            cp[i] = fma(s, gq, gp);
            cq[i] = fma(tn, gp, gq);
        }
    }
}

static void swap_columns(double *mat, int c, int p, int q) { /* blockkernel.py:269-275 */
    double *cp = mat + (int64_t)p * c, *cq = mat + (int64_t)q * c;
    for (int i = 0; i < c; i++) { double t = cp[i]; cp[i] = cq[i]; cq[i] = t; }
}

/* blockkernel.py:278-334.  steps: int32[nsteps][c/2][2], 0-based.
 * out[0..4] = rotations, proper, sweeps, status, bad_index */
void or_inner_jacobi(double *r, double *v, int c, const int32_t *steps, int nsteps,
                     const int8_t *signs, double tol_c, int max_sweeps, int64_t *out) {
    int64_t total_rot = 0, total_proper = 0, sweeps = 0;
    int half = c / 2;
    for (int sw = 0; sw < max_sweeps; sw++) {
        int64_t a_r = 0, b_r = 0;
        for (int si = 0; si < nsteps; si++)
            for (int pi = 0; pi < half; pi++) {
                int p = steps[((int64_t)si * half + pi) * 2];
                int q = steps[((int64_t)si * half + pi) * 2 + 1];
                const double *cp = r + (int64_t)p * c, *cq = r + (int64_t)q * c;
                double hpp = 0.0, hqq = 0.0, hpq = 0.0;
                for (int i = 0; i < c; i++) {
                    double gp = cp[i], gq = cq[i];
                    hpp = fma(gp, gp, hpp);
                    hqq = fma(gq, gq, hqq);
                    hpq = fma(gp, gq, hpq);
                }
                if (hpp == 0.0) { out[0] = total_rot; out[1] = total_proper; out[2] = sweeps; out[3] = 1; out[4] = p; return; }
                if (hqq == 0.0) { out[0] = total_rot; out[1] = total_proper; out[2] = sweeps; out[3] = 1; out[4] = q; return; }
                if (fabs(hpq) < tol_c * sqrt(hpp) * sqrt(hqq)) continue;
                a_r++;
                int hyp = signs[p] > 0 && signs[q] < 0;
                double t = hyp ? -1.0 : 1.0;
                double cs, tn;
                if (!rotation_core(hpp, hqq, hpq, t, &cs, &tn)) {
                    out[0] = total_rot; out[1] = total_proper; out[2] = sweeps; out[3] = 2; out[4] = p; return;
                }
                if (cs != 1.0) b_r++;
                apply_rotation(r, c, p, q, cs, tn, hyp);
                apply_rotation(v, c, p, q, cs, tn, hyp);
                if (!hyp) {
                    double h1 = fma(-tn, hpq, hpp);
                    double h2 = fma(tn, hpq, hqq);
                    if ((signs[p] > 0 && h1 < h2) || (signs[p] < 0 && h1 > h2)) {
                        swap_columns(r, c, p, q);
                        swap_columns(v, c, p, q);
                    }
                }
            }
        sweeps++;
        total_rot += a_r;
        total_proper += b_r;
        if (a_r == 0) break;
    }
    out[0] = total_rot; out[1] = total_proper; out[2] = sweeps; out[3] = 0; out[4] = -1;
}

/* out = a @ vacc, per-entry fma chain over ascending k (blockkernel.py:407-417).
 * Rows are processed in cache-sized blocks (tall pairs: a 131072-row column
 * is 1 MB); every entry's chain still runs over k = 0..c-1 in order. */
#define POST_CHUNK_ 2048
void or_postmultiply(const double *a, int64_t lda, int64_t m, int c, const double *vacc,
                     double *out, int64_t ldo) {
    for (int64_t r0 = 0; r0 < m; r0 += POST_CHUNK_) {
        const int64_t r1 = r0 + POST_CHUNK_ < m ? r0 + POST_CHUNK_ : m;
        for (int j = 0; j < c; j++) {
            double *o = out + (int64_t)j * ldo;
            for (int64_t i = r0; i < r1; i++) o[i] = 0.0;
            for (int k = 0; k < c; k++) {
                double w = vacc[(int64_t)j * c + k];
                const double *ak = a + (int64_t)k * lda;
                for (int64_t i = r0; i < r1; i++) o[i] = fma(ak[i], w, o[i]);
            }
        }
    }
}

/* R V = W back substitution (driver.py:203-211); r, w, out are n x nc */
void or_back_substitute(const double *r, int n, const double *w, int nc, double *out) {
    for (int j = 0; j < nc; j++)
        for (int i = n - 1; i >= 0; i--) {
            double acc = w[(int64_t)j * n + i];
            for (int k = i + 1; k < n; k++) acc = fma(-r[(int64_t)k * n + i], out[(int64_t)j * n + k], acc);
            out[(int64_t)j * n + i] = acc / r[(int64_t)i * n + i];
        }
}

/* ------------------------------------------------------------------------ */
/* One block sweep of run_block_jacobi_inplace (driver.py:153-196)            */

/*
 * g: m x n column-major (ld ldg), v: nv x n column-major (ld ldv) or NULL.
 * outer: int32[nsteps][b/2][2] 0-based block indices, b = n / (w/2).
 * inner: int32[w-1][w/2][2] 0-based column indices.
 * Runs p-steps [0, nsteps) of one block sweep.  Returns 0 on success, else
 * 1 (Cholesky rank deficiency), 2 (zero column in the inner kernel),
 * 3 (hyperbolic domain); err[0] = 1-based local index, err[1] = p-step,
 * err[2] = task index.  counts[0..1] += (rotations, proper).
 */
int or_block_sweep(double *g, int64_t ldg, int64_t m, int64_t n, double *v, int64_t ldv,
                   int64_t nv, int w, const int32_t *outer, int nsteps, const int32_t *inner,
                   int64_t n_plus, int inner_limit, double tol_c, int shortening,
                   int threads, int64_t *counts, int64_t *err, const int32_t *gblock) {
    int bw = w / 2;
    int64_t b = n / bw;
    int ntask = (int)(b / 2);
    int status_all = 0;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
    for (int s = 0; s < nsteps && !status_all; s++) {
        const int32_t *step = outer + (int64_t)s * ntask * 2;
        int64_t rot_s = 0, prop_s = 0;
        int first_bad = ntask, bad_status = 0;
        int64_t bad_index = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : rot_s, prop_s)
        for (int t = 0; t < ntask; t++) {
            int bp = step[2 * t], bq = step[2 * t + 1];
            int64_t cp0 = (int64_t)bp * bw, cq0 = (int64_t)bq * bw;
            double *pair = (double *)malloc(sizeof(double) * (size_t)m * w);
            double *h = (double *)malloc(sizeof(double) * (size_t)w * w);
            double *r = (double *)malloc(sizeof(double) * (size_t)w * w);
            double *vacc = (double *)malloc(sizeof(double) * (size_t)w * w);
            int8_t *sg = (int8_t *)malloc((size_t)w);
            for (int j = 0; j < bw; j++) {
                memcpy(pair + (int64_t)j * m, g + (cp0 + j) * ldg, sizeof(double) * (size_t)m);
                memcpy(pair + (int64_t)(bw + j) * m, g + (cq0 + j) * ldg, sizeof(double) * (size_t)m);
            }
            int st = 0;
            int64_t idx = 0;
            if (shortening == 0) {
                or_gram(pair, m, m, w, h);
                int info = or_cholesky(h, w);
                if (info) { st = 1; idx = info; }
                else lower_to_r(h, w, r);
            } else {
                or_qr_peeloff(pair, m, m, w, r);
            }
            if (!st) {
                for (int j = 0; j < w; j++) {
                    /* gblock: global block index of a local block-column (sharded
                     * solves; the signature follows the global column) */
                    int64_t gp0 = gblock ? (int64_t)gblock[bp] * bw : cp0;
                    int64_t gq0 = gblock ? (int64_t)gblock[bq] * bw : cq0;
                    int64_t gcol = (j < bw ? gp0 + j : gq0 + j - bw) + 1;  /* 1-based */
                    sg[j] = gcol <= n_plus ? 1 : -1;
                }
                memset(vacc, 0, sizeof(double) * (size_t)w * w);
                for (int j = 0; j < w; j++) vacc[(int64_t)j * w + j] = 1.0;
                int64_t o[5];
                or_inner_jacobi(r, vacc, w, inner, w - 1, sg, tol_c, inner_limit, o);
                if (o[3]) { st = (int)o[3] + 1; idx = o[4] + 1; }
                else {
                    rot_s += o[0];
                    prop_s += o[1];
                    if (o[0]) {
                        double *tmp = (double *)malloc(sizeof(double) * (size_t)(m > nv ? m : nv) * w);
                        or_postmultiply(pair, m, m, w, vacc, tmp, m);
                        for (int j = 0; j < bw; j++) {
                            memcpy(g + (cp0 + j) * ldg, tmp + (int64_t)j * m, sizeof(double) * (size_t)m);
                            memcpy(g + (cq0 + j) * ldg, tmp + (int64_t)(bw + j) * m, sizeof(double) * (size_t)m);
                        }
                        if (v) {
                            double *vp = (double *)malloc(sizeof(double) * (size_t)nv * w);
                            for (int j = 0; j < bw; j++) {
                                memcpy(vp + (int64_t)j * nv, v + (cp0 + j) * ldv, sizeof(double) * (size_t)nv);
                                memcpy(vp + (int64_t)(bw + j) * nv, v + (cq0 + j) * ldv, sizeof(double) * (size_t)nv);
                            }
                            or_postmultiply(vp, nv, nv, w, vacc, tmp, nv);
                            for (int j = 0; j < bw; j++) {
                                memcpy(v + (cp0 + j) * ldv, tmp + (int64_t)j * nv, sizeof(double) * (size_t)nv);
                                memcpy(v + (cq0 + j) * ldv, tmp + (int64_t)(bw + j) * nv, sizeof(double) * (size_t)nv);
                            }
                            free(vp);
                        }
                        free(tmp);
                    }
                }
            }
            if (st) {
#pragma omp critical
                {
                    if (t < first_bad) { first_bad = t; bad_status = st; bad_index = idx; }
                }
            }
            free(pair); free(h); free(r); free(vacc); free(sg);
        }
        counts[0] += rot_s;
        counts[1] += prop_s;
        if (bad_status) {
            status_all = bad_status;
            err[0] = bad_index;
            err[1] = s;
            err[2] = first_bad;
        }
    }
    return status_all;
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
