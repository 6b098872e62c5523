/*
 * tucker_oracle.c — CPU FP64 ORACLE for the Tucker/HOSVD hot path of arXiv 1711.06874.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (paper_1711_06874_b200/) never
 * imports, links or executes anything under oracle/, and this file shares no code, header, table or
 * constant generator with it.
 *
 * Plain, slow, obviously-correct C.  Every function cites the passage of
 * /root/reference/PAPER.md ("P:n" = line n) it follows; the readings of ambiguous passages are the
 * ones listed in DESIGN.md §3 ("R1".."R14").
 *
 * Build: gcc -O2 -ffp-contract=off -mfma -fopenmp -fPIC -shared (no fast-math, no BLAS/LAPACK).
 * Floating point: IEEE FP64 throughout.  Sums of products use Ogita–Rump–Oishi "Dot2"
 * (TwoProduct via fma + TwoSum), so every Gram / TTM / norm entry is as accurate as if it had been
 * accumulated in twice the working precision and rounded once.
 *
 * Parity status of each function (pins are in tests/test_oracle_*.py):
 *   orc_nodes           pinned (paper formula P:993, mirror exactness)
 *   orc_besselk_*       pinned (scipy.special.kv / mpmath, half-integer closed forms, recurrence,
 *                       Wronskian, small-z limit, overlap of regimes)
 *   orc_kernel_eval     pinned (closed forms vs general path, SPEC examples, C(0)=sigma^2;
 *                       spectral density: exact values where alpha^2+rho^2 is a power of two)
 *   orc_fill            pinned (reflection symmetry, Gaussian separability, direct evaluation)
 *   orc_unfold/orc_gram pinned (numpy BLAS Gram, trace = ||F||^2, mode invariance on cubic grids)
 *   orc_row_stats_fn    pinned (numpy max / sum of |unfolding row| of the filled tensor)
 *   orc_jacobi_eig      pinned (numpy.linalg.eigh on random SPD, residuals, orthonormality)
 *   orc_ttm_core        pinned (brute-force quadruple sum on tiny tensors, identity factors)
 *   orc_tucker_error    pinned (full-rank reconstruction, rank-1 Gaussian, ||F||^2=||b||^2+err^2)
 *   orc_hosvd           pinned (n=4 closed-form 2x2 brute force, Table 2 via orc_hooi, SVD)
 *   orc_hooi            pinned (Table 2, every cell within one unit of its last digit)
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

/* ------------------------------------------------------------------------------------------ */
/* Problem definition (the oracle's own copies; layout matches the ctypes structs in oracle.py) */

typedef struct {
    int64_t n[3];
    double lo[3], hi[3];
} orc_grid;

enum { ORC_MATERN = 0, ORC_SLATER = 1, ORC_MATERN_SPECTRAL = 2 };
enum { ORC_FORCE_GENERAL_BESSEL = 2 };

typedef struct {
    int32_t family;
    int32_t flags;
    double sigma2, ell, nu, lambda, p;
} orc_kernel;

enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_DOMAIN = 2, ORC_ERR_NOCONV = 5 };

/* ------------------------------------------------------------------------------------------ */
/* Compensated arithmetic (Ogita, Rump, Oishi 2005, "Accurate sum and dot product").           */

static inline void two_sum(double a, double b, double *s, double *e) {
    double x = a + b;
    double z = x - a;
    *e = (a - (x - z)) + (b - z);
    *s = x;
}

static inline void two_prod(double a, double b, double *p, double *e) {
    double x = a * b;
    *e = fma(a, b, -x);
    *p = x;
}

typedef struct { double s, c; } dot2_acc;

static inline void dot2_add(dot2_acc *acc, double a, double b) {
    double p, pe, s, se;
    two_prod(a, b, &p, &pe);
    two_sum(acc->s, p, &s, &se);
    acc->s = s;
    acc->c += pe + se;
}

static inline double dot2_get(const dot2_acc *acc) { return acc->s + acc->c; }

/* Dot2 of two strided vectors. */
static double dot2(int64_t len, const double *a, int64_t sa, const double *b, int64_t sb) {
    dot2_acc acc = {0.0, 0.0};
    for (int64_t t = 0; t < len; ++t) dot2_add(&acc, a[t * sa], b[t * sb]);
    return dot2_get(&acc);
}

/* ------------------------------------------------------------------------------------------ */
/* a-1  Grid nodes.  P:992-997: x_i = -b + (i-1) h, h = 2b/(n-1), on [-b,b] (and per axis
 * [lo,hi]).  Reading R2: evaluated as x_i = c + s*(2i-(n-1)), c=(lo+hi)/2,
 * s=(hi-lo)/(2(n-1)), i = 0..n-1 — the same real number, and bitwise mirror-exact when lo=-hi. */
void orc_nodes(int64_t n, double lo, double hi, double *x) {
    double c = (lo + hi) * 0.5;
    double s = (hi - lo) / (2.0 * (double)(n - 1));
    for (int64_t i = 0; i < n; ++i) {
        double m = (double)(2 * i - (n - 1));
        double sm = s * m;
        x[i] = c + sm;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Modified Bessel function K_nu(z), z > 0.  The paper uses K_nu in eq. (Matern) P:356-357 but
 * gives no algorithm.  Three textbook routes, each used only where it is accurate (reading R5):
 *   (i)   ascending series  K_nu = pi/(2 sin(nu pi)) (I_{-nu}(z) - I_nu(z))   [DLMF 10.27.4, 10.25.2]
 *   (ii)  Hankel asymptotic K_nu ~ sqrt(pi/2z) e^{-z} sum_k a_k(nu)/z^k       [DLMF 10.40.2]
 *   (iii) integral K_nu(z) = int_0^inf e^{-z cosh t} cosh(nu t) dt             [DLMF 10.32.9]
 *         by the trapezoid rule with h = 1/32 (the paper's own sinc-quadrature device).
 * All three return the exponentially scaled value e^{z} K_nu(z) to avoid underflow. */

/* (i) e^z K_nu(z) from the ascending series; valid for z <= 1 and nu not within 1e-3 of an
 * integer (the 1/sin(nu pi) cancellation).  Terms of I_mu: t_0 = (z/2)^mu / Gamma(mu+1),
 * t_{k+1} = t_k (z/2)^2 / ((k+1)(k+1+mu)). */
static double series_I(double mu, double z) {
    double h = 0.5 * z;
    double t = pow(h, mu) / tgamma(mu + 1.0);
    double q = h * h;
    double sum = 0.0, comp = 0.0;
    for (int k = 0; k < 400; ++k) {
        double s, e;
        two_sum(sum, t, &s, &e);
        sum = s;
        comp += e;
        t = t * q / ((double)(k + 1) * ((double)(k + 1) + mu));
        if (fabs(t) < 1e-18 * fabs(sum)) break;
    }
    return sum + comp;
}

double orc_besselk_series_scaled(double nu, double z) {
    double im = series_I(-nu, z);
    double ip = series_I(nu, z);
    double k = M_PI / (2.0 * sin(nu * M_PI)) * (im - ip);
    return k * exp(z);
}

/* (ii) e^z K_nu(z) from the Hankel asymptotic series, optimally truncated: a_0 = 1,
 * a_k = a_{k-1} (4nu^2 - (2k-1)^2) / (8k); stop at the smallest term.  Used for z >= 20. */
double orc_besselk_hankel_scaled(double nu, double z) {
    double mu = 4.0 * nu * nu;
    double term = 1.0, sum = 1.0, comp = 0.0;
    double prev = INFINITY;
    for (int k = 1; k < 200; ++k) {
        double nt = term * (mu - (double)(2 * k - 1) * (double)(2 * k - 1)) / (8.0 * (double)k * z);
        if (fabs(nt) >= prev || fabs(nt) < 1e-20 * fabs(sum)) break;
        double s, e;
        two_sum(sum, nt, &s, &e);
        sum = s;
        comp += e;
        prev = fabs(nt);
        term = nt;
    }
    return sqrt(M_PI / (2.0 * z)) * (sum + comp);
}

/* (iii) e^z K_nu(z) = int_0^inf exp(-z (cosh t - 1)) cosh(nu t) dt, trapezoid rule h = 1/32:
 * h [f(0)/2 + sum_{k>=1} f(kh)].  cosh t - 1 = 2 sinh^2(t/2) (no cancellation).  The sum stops
 * once the integrand is past its maximum and below 1e-18 of the running sum. */
double orc_besselk_trapz_scaled(double nu, double z) {
    const double h = 1.0 / 32.0;
    double sum = 0.5, comp = 0.0; /* f(0) = 1 */
    double prev = 1.0;
    for (int64_t k = 1; k < 100000; ++k) {
        double t = (double)k * h;
        double sh = sinh(0.5 * t);
        double f = exp(-z * 2.0 * sh * sh) * cosh(nu * t);
        double s, e;
        two_sum(sum, f, &s, &e);
        sum = s;
        comp += e;
        if (f < prev && f < 1e-18 * sum) break;
        prev = f;
    }
    return h * (sum + comp);
}

static int near_integer(double nu) { return fabs(nu - nearbyint(nu)) < 1e-3; }

/* e^z K_nu(z) by the route that is accurate at (nu, z) (reading R5). */
double orc_besselk_scaled(double nu, double z) {
    nu = fabs(nu); /* K_{-nu} = K_nu */
    if (z >= 20.0) return orc_besselk_hankel_scaled(nu, z);
    if (z <= 1.0 && !near_integer(nu)) return orc_besselk_series_scaled(nu, z);
    return orc_besselk_trapz_scaled(nu, z);
}

double orc_besselk(double nu, double z) { return orc_besselk_scaled(nu, z) * exp(-z); }

/* ------------------------------------------------------------------------------------------ */
/* a-2  Kernel families.
 * Matern, eq. (Matern): C(r) = sigma^2 2^{1-nu}/Gamma(nu) (sqrt(2nu) r/ell)^nu
 *   K_nu(sqrt(2nu) r/ell); sigma^2 per reading R3; C(0) = sigma^2 (limit, R4).
 *   nu = 1/2 gives the exponential model; nu = 3/2, 5/2 are the half-integer closed
 *   forms of the same formula ((1+z)e^{-z}, (1+z+z^2/3)e^{-z}).
 * p-Slater, eq. (exp_p): C = sigma^2 exp(-lambda r^p); p = 2 is the
 *   Gaussian.
 * Matérn spectral density, eq. (SD_matern) P:1046-1050 (NEXT f4): f(rho) = C (alpha^2 + rho^2)^{-(nu+d/2)}
 *   with d = 3, rho = ||x|| (the grid is read as a frequency grid), C = sigma^2 (reading R17) and
 *   alpha carried in the `lambda` field. */
double orc_kernel_eval(const orc_kernel *k, double r, double r2) {
    if (k->family == ORC_MATERN_SPECTRAL) {
        double a2 = k->lambda * k->lambda;
        return k->sigma2 * pow(a2 + r2, -(k->nu + 1.5));
    }
    if (k->family == ORC_SLATER) {
        double rp = (k->p == 1.0) ? r : (k->p == 2.0) ? r2 : pow(r, k->p);
        return k->sigma2 * exp(-k->lambda * rp);
    }
    if (r == 0.0) return k->sigma2;
    double nu = k->nu;
    double z = (sqrt(2.0 * nu) * r) / k->ell;
    if (!(k->flags & ORC_FORCE_GENERAL_BESSEL)) {
        if (nu == 0.5) return k->sigma2 * exp(-z);
        if (nu == 1.5) return k->sigma2 * ((1.0 + z) * exp(-z));
        if (nu == 2.5) return k->sigma2 * ((1.0 + z + z * z / 3.0) * exp(-z));
    }
    double pref = pow(2.0, 1.0 - nu) / tgamma(nu);
    /* z^nu K_nu(z) = z^nu e^{-z} (e^z K_nu(z)) */
    return k->sigma2 * (pref * (pow(z, nu) * exp(-z) * orc_besselk_scaled(nu, z)));
}

int orc_kernel_check(const orc_kernel *k) {
    if (!(k->sigma2 > 0.0)) return ORC_ERR_DOMAIN;
    if (k->family == ORC_MATERN) {
        if (!(k->nu > 0.0) || !(k->ell > 0.0)) return ORC_ERR_DOMAIN;
        return ORC_OK;
    }
    if (k->family == ORC_SLATER) {
        if (!(k->lambda > 0.0) || !(k->p > 0.0) || !(k->p <= 2.0)) return ORC_ERR_DOMAIN;
        return ORC_OK;
    }
    if (k->family == ORC_MATERN_SPECTRAL) {
        if (!(k->lambda > 0.0) || !(k->nu > 0.0)) return ORC_ERR_DOMAIN;
        return ORC_OK;
    }
    return ORC_ERR_ARG;
}

/* Collocation tensor: F[i,j,k] = C(||x_ijk||), C-order, k fastest.
 * Radius r = sqrt((x_i^2 + y_j^2) + z_k^2) in that association order (reading R2). */
int orc_fill(const orc_grid *g, const orc_kernel *k, double *F) {
    int rc = orc_kernel_check(k);
    if (rc) return rc;
    int64_t n1 = g->n[0], n2 = g->n[1], n3 = g->n[2];
    double *x = malloc(sizeof(double) * (size_t)(n1 + n2 + n3));
    double *y = x + n1, *z = y + n2;
    orc_nodes(n1, g->lo[0], g->hi[0], x);
    orc_nodes(n2, g->lo[1], g->hi[1], y);
    orc_nodes(n3, g->lo[2], g->hi[2], z);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < n1; ++i)
        for (int64_t j = 0; j < n2; ++j)
            for (int64_t l = 0; l < n3; ++l) {
                double xx = x[i] * x[i], yy = y[j] * y[j], zz = z[l] * z[l];
                double r2 = (xx + yy) + zz;
                F[(i * n2 + j) * n3 + l] = orc_kernel_eval(k, sqrt(r2), r2);
            }
    free(x);
    return ORC_OK;
}

/* Single entry of the collocation tensor (for sampled checks at sizes the oracle cannot fill). */
double orc_fill_entry(const orc_grid *g, const orc_kernel *k, int64_t i, int64_t j, int64_t l) {
    double c[3];
    int64_t idx[3] = {i, j, l};
    for (int a = 0; a < 3; ++a) {
        double cc = (g->lo[a] + g->hi[a]) * 0.5;
        double s = (g->hi[a] - g->lo[a]) / (2.0 * (double)(g->n[a] - 1));
        double m = (double)(2 * idx[a] - (g->n[a] - 1));
        double sm = s * m;
        c[a] = cc + sm;
    }
    double xx = c[0] * c[0], yy = c[1] * c[1], zz = c[2] * c[2];
    double r2 = (xx + yy) + zz;
    return orc_kernel_eval(k, sqrt(r2), r2);
}

/* ------------------------------------------------------------------------------------------ */
/* a-3  Mode-m unfolding A_(m) (Fig. "Unfolding"): rows indexed by i_m, columns by the
 * remaining two indices in increasing (slow, fast) order.  mode is 0,1,2 for modes 1,2,3. */
void orc_unfold(const double *F, const int64_t *dims, int mode, double *A) {
    int64_t n1 = dims[0], n2 = dims[1], n3 = dims[2];
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < n1; ++i)
        for (int64_t j = 0; j < n2; ++j)
            for (int64_t l = 0; l < n3; ++l) {
                double v = F[(i * n2 + j) * n3 + l];
                int64_t row, col;
                if (mode == 0) { row = i; col = j * n3 + l; }
                else if (mode == 1) { row = j; col = i * n3 + l; }
                else { row = l; col = i * n2 + j; }
                int64_t ncol = (mode == 0) ? n2 * n3 : (mode == 1) ? n1 * n3 : n1 * n2;
                A[row * ncol + col] = v;
            }
}

/* Gram G = A A^T of a rows x cols row-major matrix: the triple loop, each entry a Dot2 sum.
 * (The left singular vectors of A_(m), are the eigenvectors of G; lambda = sigma^2.) */
void orc_gram(const double *A, int64_t rows, int64_t cols, double *G) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t a = 0; a < rows; ++a)
        for (int64_t b = 0; b <= a; ++b) {
            double v = dot2(cols, A + a * cols, 1, A + b * cols, 1);
            G[a * rows + b] = v;
            G[b * rows + a] = v;
        }
}

/* Single Gram entry G_m[a][b] computed from the kernel directly (no F in memory), for sampled
 * checks at 1024^3: sum over the other two indices of C(x_a..)C(x_b..). */
double orc_gram_entry_fn(const orc_grid *g, const orc_kernel *k, int mode, int64_t a, int64_t b) {
    int64_t n1 = g->n[0], n2 = g->n[1], n3 = g->n[2];
    int64_t outer = (mode == 0) ? n2 : n1;
    int64_t inner = (mode == 2) ? n2 : n3;
    double total = 0.0, totc = 0.0;
#pragma omp parallel
    {
        dot2_acc acc = {0.0, 0.0};
#pragma omp for schedule(static)
        for (int64_t u = 0; u < outer; ++u)
            for (int64_t v = 0; v < inner; ++v) {
                double fa, fb;
                if (mode == 0) { fa = orc_fill_entry(g, k, a, u, v); fb = orc_fill_entry(g, k, b, u, v); }
                else if (mode == 1) { fa = orc_fill_entry(g, k, u, a, v); fb = orc_fill_entry(g, k, u, b, v); }
                else { fa = orc_fill_entry(g, k, u, v, a); fb = orc_fill_entry(g, k, u, v, b); }
                dot2_add(&acc, fa, fb);
            }
#pragma omp critical
        {
            double s, e;
            two_sum(total, acc.s, &s, &e);
            total = s;
            totc += e + acc.c;
        }
    }
    (void)outer;
    return total + totc;
}

/* Row statistics of the mode-m unfolding computed from the kernel directly (no F in memory):
 * out[0] = max_k |A_(m)[a,k]|, out[1] = sum_k |A_(m)[a,k]| (compensated).  Test-only: the inputs of
 * the INT8 Gram's element bound (R18) for sampled entries at sizes the oracle cannot fill. */
void orc_row_stats_fn(const orc_grid *g, const orc_kernel *k, int mode, int64_t a, double *out) {
    int64_t n1 = g->n[0], n2 = g->n[1], n3 = g->n[2];
    int64_t outer = (mode == 0) ? n2 : n1;
    int64_t inner = (mode == 2) ? n2 : n3;
    double mx = 0.0, total = 0.0, totc = 0.0;
#pragma omp parallel
    {
        double lmx = 0.0, s = 0.0, c = 0.0;
#pragma omp for schedule(static)
        for (int64_t u = 0; u < outer; ++u)
            for (int64_t v = 0; v < inner; ++v) {
                double f;
                if (mode == 0) f = orc_fill_entry(g, k, a, u, v);
                else if (mode == 1) f = orc_fill_entry(g, k, u, a, v);
                else f = orc_fill_entry(g, k, u, v, a);
                double af = fabs(f), t, e;
                lmx = fmax(lmx, af);
                two_sum(s, af, &t, &e);
                s = t;
                c += e;
            }
#pragma omp critical
        {
            double t, e;
            mx = fmax(mx, lmx);
            two_sum(total, s, &t, &e);
            total = t;
            totc += e + c;
        }
    }
    (void)n3;
    out[0] = mx;
    out[1] = total + totc;
}

/* ------------------------------------------------------------------------------------------ */
/* a-4  Symmetric eigensolver: cyclic Jacobi (Golub & Van Loan, Alg. 8.4.2 sym.schur2 rotations)
 * in parallel round-robin ordering (disjoint pairs per step).  Skip rule (reading R7):
 * rotate (p,q) only if |a_pq| > max(eps sqrt|a_pp a_qq|, eps max_i|a_ii| / n).  Stops after a
 * sweep with no rotation.  Output: eigenvalues descending (stable for ties), eigenvector columns
 * V (n x n, row-major, column k = k-th eigenvector), sign rule R6 applied. */
static void sign_fix_columns(int64_t n, int64_t ncols, double *V, int64_t ldv) {
    for (int64_t c = 0; c < ncols; ++c) {
        double mx = 0.0;
        for (int64_t i = 0; i < n; ++i) mx = fmax(mx, fabs(V[i * ldv + c]));
        int64_t istar = 0;
        for (int64_t i = 0; i < n; ++i)
            if (fabs(V[i * ldv + c]) >= 0.5 * mx) { istar = i; break; }
        if (V[istar * ldv + c] < 0.0)
            for (int64_t i = 0; i < n; ++i) V[i * ldv + c] = -V[i * ldv + c];
    }
}

void orc_sign_fix(int64_t n, int64_t ncols, double *V, int64_t ldv) { sign_fix_columns(n, ncols, V, ldv); }

int orc_jacobi_eig(int64_t n, const double *G, double *lam, double *V, int max_sweeps, int *sweeps_out) {
    double *A = malloc(sizeof(double) * (size_t)(n * n));
    memcpy(A, G, sizeof(double) * (size_t)(n * n));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) V[i * n + j] = (i == j) ? 1.0 : 0.0;
    int64_t m = n + (n & 1); /* round-robin players; index n (if present) is a dummy */
    int64_t *arr = malloc(sizeof(int64_t) * (size_t)m);
    int64_t *pp = malloc(sizeof(int64_t) * (size_t)(m / 2));
    int64_t *qq = malloc(sizeof(int64_t) * (size_t)(m / 2));
    double *cs = malloc(sizeof(double) * (size_t)m);
    double *sn = cs + m / 2;
    int rc = ORC_ERR_NOCONV, sweep;
    const double eps = DBL_EPSILON;
    for (sweep = 0; sweep < max_sweeps; ++sweep) {
        double dmax = 0.0;
        for (int64_t i = 0; i < n; ++i) dmax = fmax(dmax, fabs(A[i * n + i]));
        double floor_abs = eps * dmax / (double)n;
        int64_t rotations = 0;
        for (int64_t t = 0; t < m; ++t) arr[t] = t;
        for (int64_t step = 0; step < m - 1; ++step) {
            int64_t npairs = 0;
            for (int64_t t = 0; t < m / 2; ++t) {
                int64_t p = arr[t], q = arr[m - 1 - t];
                if (p > q) { int64_t tmp = p; p = q; q = tmp; }
                if (q >= n) continue;
                double apq = A[p * n + q], app = A[p * n + p], aqq = A[q * n + q];
                double thr = fmax(eps * sqrt(fabs(app * aqq)), floor_abs);
                if (!(fabs(apq) > thr)) continue;
                /* sym.schur2 */
                double tau = (aqq - app) / (2.0 * apq);
                double tt = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                         : -1.0 / (-tau + sqrt(1.0 + tau * tau));
                double c = 1.0 / sqrt(1.0 + tt * tt);
                pp[npairs] = p; qq[npairs] = q; cs[npairs] = c; sn[npairs] = tt * c;
                ++npairs;
            }
            rotations += npairs;
            if (npairs) {
                /* rows: A <- J^T A */
#pragma omp parallel for schedule(static)
                for (int64_t w = 0; w < npairs; ++w) {
                    double c = cs[w], s = sn[w];
                    double *rp = A + pp[w] * n, *rq = A + qq[w] * n;
                    for (int64_t j = 0; j < n; ++j) {
                        double a = rp[j], b = rq[j];
                        rp[j] = c * a - s * b;
                        rq[j] = s * a + c * b;
                    }
                }
                /* columns: A <- A J, and V <- V J */
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < n; ++i) {
                    double *ra = A + i * n, *rv = V + i * n;
                    for (int64_t w = 0; w < npairs; ++w) {
                        double c = cs[w], s = sn[w];
                        int64_t p = pp[w], q = qq[w];
                        double a = ra[p], b = ra[q];
                        ra[p] = c * a - s * b;
                        ra[q] = s * a + c * b;
                        a = rv[p]; b = rv[q];
                        rv[p] = c * a - s * b;
                        rv[q] = s * a + c * b;
                    }
                }
                for (int64_t w = 0; w < npairs; ++w) { /* annihilated by construction */
                    A[pp[w] * n + qq[w]] = 0.0;
                    A[qq[w] * n + pp[w]] = 0.0;
                }
            }
            /* rotate players 1..m-1 */
            int64_t last = arr[m - 1];
            for (int64_t t = m - 1; t > 1; --t) arr[t] = arr[t - 1];
            if (m > 1) arr[1] = last;
        }
        if (rotations == 0) { rc = ORC_OK; ++sweep; break; }
    }
    if (sweeps_out) *sweeps_out = sweep;
    /* sort descending, stable */
    int64_t *ord = malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) ord[i] = i;
    for (int64_t i = 1; i < n; ++i) {
        int64_t key = ord[i];
        double kv = A[key * n + key];
        int64_t j = i - 1;
        while (j >= 0 && A[ord[j] * n + ord[j]] < kv) { ord[j + 1] = ord[j]; --j; }
        ord[j + 1] = key;
    }
    double *W = malloc(sizeof(double) * (size_t)(n * n));
    for (int64_t k = 0; k < n; ++k) {
        lam[k] = A[ord[k] * n + ord[k]];
        for (int64_t i = 0; i < n; ++i) W[i * n + k] = V[i * n + ord[k]];
    }
    memcpy(V, W, sizeof(double) * (size_t)(n * n));
    sign_fix_columns(n, n, V, n);
    free(W); free(ord); free(cs); free(qq); free(pp); free(arr); free(A);
    return rc;
}

/* ------------------------------------------------------------------------------------------ */
/* a-5  Core by the final contraction, P:546-548 and P:578-579:
 * beta = F x_1 U1^T x_2 U2^T x_3 U3^T, evaluated as three naive mode products (Dot2 sums):
 *   T1[i,j,c] = sum_k F[i,j,k] U3[k,c];  T2[i,b,c] = sum_j U2[j,b] T1[i,j,c];
 *   beta[a,b,c] = sum_i U1[i,a] T2[i,b,c].   U_m is n_m x r_m row-major. */
void orc_ttm_core(const double *F, const int64_t *dims, const int64_t *r, const double *U1,
                  const double *U2, const double *U3, double *core) {
    int64_t n1 = dims[0], n2 = dims[1], n3 = dims[2], r1 = r[0], r2 = r[1], r3 = r[2];
    double *T1 = malloc(sizeof(double) * (size_t)(n1 * n2 * r3));
    double *T2 = malloc(sizeof(double) * (size_t)(n1 * r2 * r3));
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < n1; ++i)
        for (int64_t j = 0; j < n2; ++j)
            for (int64_t c = 0; c < r3; ++c)
                T1[(i * n2 + j) * r3 + c] = dot2(n3, F + (i * n2 + j) * n3, 1, U3 + c, r3);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < n1; ++i)
        for (int64_t b = 0; b < r2; ++b)
            for (int64_t c = 0; c < r3; ++c)
                T2[(i * r2 + b) * r3 + c] = dot2(n2, U2 + b, r2, T1 + i * n2 * r3 + c, r3);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t a = 0; a < r1; ++a)
        for (int64_t b = 0; b < r2; ++b)
            for (int64_t c = 0; c < r3; ++c)
                core[(a * r2 + b) * r3 + c] = dot2(n1, U1 + a, r1, T2 + b * r3 + c, r2 * r3);
    free(T2); free(T1);
}

/* Tucker reconstruction, eqn:Tucker_form P:532-547: Ft = beta x_1 U1 x_2 U2 x_3 U3. */
void orc_reconstruct(const int64_t *dims, const int64_t *r, const double *U1, const double *U2,
                     const double *U3, const double *core, double *Ft) {
    int64_t n1 = dims[0], n2 = dims[1], n3 = dims[2], r1 = r[0], r2 = r[1], r3 = r[2];
    double *X = malloc(sizeof(double) * (size_t)(n1 * r2 * r3));
    double *W = malloc(sizeof(double) * (size_t)(n1 * n2 * r3));
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < n1; ++i)
        for (int64_t b = 0; b < r2; ++b)
            for (int64_t c = 0; c < r3; ++c)
                X[(i * r2 + b) * r3 + c] = dot2(r1, U1 + i * r1, 1, core + b * r3 + c, r2 * r3);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < n1; ++i)
        for (int64_t j = 0; j < n2; ++j)
            for (int64_t c = 0; c < r3; ++c)
                W[(i * n2 + j) * r3 + c] = dot2(r2, U2 + j * r2, 1, X + i * r2 * r3 + c, r3);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < n1; ++i)
        for (int64_t j = 0; j < n2; ++j)
            for (int64_t l = 0; l < n3; ++l)
                Ft[(i * n2 + j) * n3 + l] = dot2(r3, W + (i * n2 + j) * r3, 1, U3 + l * r3, 1);
    free(W); free(X);
}

/* a-6  Relative Frobenius error, eq. (FNorm): E = ||F - Ft|| / ||F||.
 * out[0] = E, out[1] = ||F||, out[2] = ||F - Ft||.  Sums of squares are compensated. */
void orc_tucker_error(const double *F, const int64_t *dims, const int64_t *r, const double *U1,
                      const double *U2, const double *U3, const double *core, double *out) {
    int64_t N = dims[0] * dims[1] * dims[2];
    double *Ft = malloc(sizeof(double) * (size_t)N);
    orc_reconstruct(dims, r, U1, U2, U3, core, Ft);
    double sf = 0.0, cf = 0.0, sd = 0.0, cd = 0.0;
#pragma omp parallel
    {
        dot2_acc af = {0.0, 0.0}, ad = {0.0, 0.0};
#pragma omp for schedule(static)
        for (int64_t t = 0; t < N; ++t) {
            double d = F[t] - Ft[t];
            dot2_add(&af, F[t], F[t]);
            dot2_add(&ad, d, d);
        }
#pragma omp critical
        {
            double s, e;
            two_sum(sf, af.s, &s, &e); sf = s; cf += e + af.c;
            two_sum(sd, ad.s, &s, &e); sd = s; cd += e + ad.c;
        }
    }
    double nf = sqrt(sf + cf), nd = sqrt(sd + cd);
    out[0] = nd / nf;
    out[1] = nf;
    out[2] = nd;
    free(Ft);
}

/* ------------------------------------------------------------------------------------------ */
/* HOSVD, P:555-561 + P:578-579: for each mode, U_m = leading r_m eigenvectors of
 * G_m = A_(m) A_(m)^T (sorted, sign-fixed), sigma_m = sqrt(max(lambda,0)); then the core.
 * Also returns the full spectra lam_m (length n_m) for the tolerance reading R14.
 * U_m: n_m x r_m row-major.  Returns ORC_ERR_NOCONV if a Jacobi solve hit its cap. */
int orc_hosvd(const double *F, const int64_t *dims, const int64_t *r, double *U1, double *U2,
              double *U3, double *core, double *lam1, double *lam2, double *lam3) {
    double *U[3] = {U1, U2, U3};
    double *L[3] = {lam1, lam2, lam3};
    int64_t N = dims[0] * dims[1] * dims[2];
    int rc = ORC_OK;
    double *A = malloc(sizeof(double) * (size_t)N);
    for (int m = 0; m < 3; ++m) {
        int64_t n = dims[m];
        double *G = malloc(sizeof(double) * (size_t)(n * n));
        double *V = malloc(sizeof(double) * (size_t)(n * n));
        orc_unfold(F, dims, m, A);
        orc_gram(A, n, N / n, G);
        int sw;
        int e = orc_jacobi_eig(n, G, L[m], V, 100, &sw);
        if (e) rc = e;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t c = 0; c < r[m]; ++c) U[m][i * r[m] + c] = V[i * n + c];
        free(V); free(G);
    }
    free(A);
    orc_ttm_core(F, dims, r, U1, U2, U3, core);
    return rc;
}

/* ------------------------------------------------------------------------------------------ */
/* O7 (test-only): Tucker-ALS / HOOI sweeps.  For each mode m in turn, the
 * "single-hole" tensor Y = F x_{q != m} U_q^T (n_m x r_a x r_b) is formed by naive mode products
 * and U_m is replaced by the leading r_m left singular vectors of its unfolding Y_(m).  Those are
 * computed from the small Gram M = Y_(m)^T Y_(m) (r_a r_b square) by Jacobi: u_k = Y_(m) w_k /
 * sigma_k, followed by two passes of classical Gram-Schmidt (re-orthonormalisation).
 * U1..U3 hold the initial guess on entry (e.g. HOSVD factors) and the result on exit. */
static void single_hole(const double *F, const int64_t *dims, const int64_t *r, double *const *U,
                        int m, double *Y) {
    int64_t n1 = dims[0], n2 = dims[1], n3 = dims[2];
    if (m == 0) { /* Y[i, b, c] = sum_j sum_k F[i,j,k] U2[j,b] U3[k,c] */
        int64_t r2 = r[1], r3 = r[2];
        double *T = malloc(sizeof(double) * (size_t)(n1 * n2 * r3));
#pragma omp parallel for collapse(2) schedule(static)
        for (int64_t i = 0; i < n1; ++i)
            for (int64_t j = 0; j < n2; ++j)
                for (int64_t c = 0; c < r3; ++c)
                    T[(i * n2 + j) * r3 + c] = dot2(n3, F + (i * n2 + j) * n3, 1, U[2] + c, r3);
#pragma omp parallel for collapse(2) schedule(static)
        for (int64_t i = 0; i < n1; ++i)
            for (int64_t b = 0; b < r2; ++b)
                for (int64_t c = 0; c < r3; ++c)
                    Y[(i * r2 + b) * r3 + c] = dot2(n2, U[1] + b, r2, T + i * n2 * r3 + c, r3);
        free(T);
    } else if (m == 1) { /* Y[j, a, c] = sum_i sum_k F[i,j,k] U1[i,a] U3[k,c] */
        int64_t r1 = r[0], r3 = r[2];
        double *T = malloc(sizeof(double) * (size_t)(n1 * n2 * r3));
#pragma omp parallel for collapse(2) schedule(static)
        for (int64_t i = 0; i < n1; ++i)
            for (int64_t j = 0; j < n2; ++j)
                for (int64_t c = 0; c < r3; ++c)
                    T[(i * n2 + j) * r3 + c] = dot2(n3, F + (i * n2 + j) * n3, 1, U[2] + c, r3);
#pragma omp parallel for collapse(2) schedule(static)
        for (int64_t j = 0; j < n2; ++j)
            for (int64_t a = 0; a < r1; ++a)
                for (int64_t c = 0; c < r3; ++c)
                    Y[(j * r1 + a) * r3 + c] = dot2(n1, U[0] + a, r[0], T + j * r3 + c, n2 * r3);
        free(T);
    } else { /* Y[k, a, b] = sum_i sum_j F[i,j,k] U1[i,a] U2[j,b] */
        int64_t r1 = r[0], r2 = r[1];
        double *T = malloc(sizeof(double) * (size_t)(n1 * r2 * n3));
#pragma omp parallel for collapse(2) schedule(static)
        for (int64_t i = 0; i < n1; ++i)
            for (int64_t b = 0; b < r2; ++b)
                for (int64_t l = 0; l < n3; ++l)
                    T[(i * r2 + b) * n3 + l] = dot2(n2, U[1] + b, r2, F + i * n2 * n3 + l, n3);
#pragma omp parallel for collapse(2) schedule(static)
        for (int64_t l = 0; l < n3; ++l)
            for (int64_t a = 0; a < r1; ++a)
                for (int64_t b = 0; b < r2; ++b)
                    Y[(l * r1 + a) * r2 + b] = dot2(n1, U[0] + a, r1, T + b * n3 + l, r2 * n3);
        free(T);
    }
}

int orc_hooi(const double *F, const int64_t *dims, const int64_t *r, double *U1, double *U2,
             double *U3, int sweeps) {
    double *U[3] = {U1, U2, U3};
    int rc = ORC_OK;
    for (int s = 0; s < sweeps; ++s)
        for (int m = 0; m < 3; ++m) {
            int64_t n = dims[m];
            int64_t ra = (m == 0) ? r[1] : r[0];
            int64_t rb = (m == 2) ? r[1] : r[2];
            int64_t cols = ra * rb;
            double *Y = malloc(sizeof(double) * (size_t)(n * cols));
            single_hole(F, dims, r, U, m, Y);
            double *M = malloc(sizeof(double) * (size_t)(cols * cols));
            double *W = malloc(sizeof(double) * (size_t)(cols * cols));
            double *lam = malloc(sizeof(double) * (size_t)cols);
            for (int64_t a = 0; a < cols; ++a)
                for (int64_t b = 0; b <= a; ++b) {
                    double v = dot2(n, Y + a, cols, Y + b, cols);
                    M[a * cols + b] = v;
                    M[b * cols + a] = v;
                }
            int sw;
            int e = orc_jacobi_eig(cols, M, lam, W, 100, &sw);
            if (e) rc = e;
            int64_t rm = r[m];
            for (int64_t k = 0; k < rm; ++k) {
                double sig = sqrt(fmax(lam[k], 0.0));
                for (int64_t i = 0; i < n; ++i)
                    U[m][i * rm + k] = dot2(cols, Y + i * cols, 1, W + k, cols) / (sig > 0.0 ? sig : 1.0);
            }
            for (int pass = 0; pass < 2; ++pass) /* CGS2 re-orthonormalisation */
                for (int64_t k = 0; k < rm; ++k) {
                    for (int64_t q = 0; q < k; ++q) {
                        double h = dot2(n, U[m] + q, rm, U[m] + k, rm);
                        for (int64_t i = 0; i < n; ++i) U[m][i * rm + k] -= h * U[m][i * rm + q];
                    }
                    double nrm = sqrt(dot2(n, U[m] + k, rm, U[m] + k, rm));
                    for (int64_t i = 0; i < n; ++i) U[m][i * rm + k] /= nrm;
                }
            sign_fix_columns(n, rm, U[m], rm);
            free(lam); free(W); free(M); free(Y);
        }
    return rc;
}

/* Tucker value at one grid point: A(i,j,k) = sum_abc beta[a,b,c] U1[i,a] U2[j,b] U3[k,c]
 * (used for the origin value A(x0) of Table 2). */
double orc_tucker_point(const int64_t *r, const double *U1, const double *U2, const double *U3,
                        const double *core, int64_t i, int64_t j, int64_t l) {
    dot2_acc acc = {0.0, 0.0};
    for (int64_t a = 0; a < r[0]; ++a)
        for (int64_t b = 0; b < r[1]; ++b)
            for (int64_t c = 0; c < r[2]; ++c)
                dot2_add(&acc, core[(a * r[1] + b) * r[2] + c],
                         U1[i * r[0] + a] * U2[j * r[1] + b] * U3[l * r[2] + c]);
    return dot2_get(&acc);
}

int orc_num_threads(void) { return omp_get_max_threads(); }
void orc_set_num_threads(int t) { omp_set_num_threads(t); }
