/*
 * oracle.c -- plain, slow, obviously-correct FP64 CPU oracle for the
 * NFFT-accelerated Sinkhorn hot path (arXiv 2201.07524).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2201_07524_b200/csrc); neither side includes the other.
 *
 * Everything here is a dense, direct evaluation of a definition from the
 * paper, written in the paper's order (P:Lx = /root/reference/PAPER.md line x):
 *
 *   oracle_direct_sum     Eq. (matexp)  P:L462-465  t_i = sum_j w_j exp(-lam |x_i - y_j|^r)
 *                         Eq. (matexpt) P:L467-470  (transpose = swap the point sets)
 *                         kernel 1: c_ij exp(-lam c_ij), the integrand of the upper
 *                         divergence s~ = sum_ij pi_ij d_ij^r (Def 3.1)
 *   oracle_sinkhorn_plain Alg. 1 literally: alpha^(0)=1, alpha~^(0)=1,
 *                         odd Delta updates alpha = p / (k alpha~), even Delta
 *                         alpha~ = p~ / (k^T alpha). One "iteration" = odd + even.
 *   oracle_sinkhorn_log   the same iterates in potentials f = log(alpha)/lam,
 *                         g = log(alpha~)/lam (log-domain stabilisation, BJ north_star):
 *                         f_i = (log a_i - LSE_j lam (g_j - c_ij)) / lam, then
 *                         g_j = (log b_j - LSE_i lam (f_i - c_ij)) / lam.
 *   oracle_divergence     pi_ij = exp(lam (f_i + g_j - c_ij))   (Eq. (pi*))
 *                         s~ = sum pi_ij c_ij                     (Def 3.1)
 *                         s  = 1/lam + sum a f + sum b g - (1/lam) sum pi   (Eq. (14), P:L211;
 *                              Alg. 2 result line P:L732 with log alpha = lam f)
 *                         residuals |pi 1 - a|_1, |pi^T 1 - b|_1  (Eq. (Error))
 *                         H(pi) = -sum pi log pi                  (Def 3.1)
 *
 * Cost c_ij = d_ij^r with d_ij = |x_i - y_j| the Euclidean distance in the caller's
 * coordinates, r = 2 (squared Euclidean, the BJ hot path) or r = 1 (Euclidean,
 * SURVEY §8(f) NEXT-2); every entry point takes r. All sums are Neumaier-compensated. Rows are
 * independent and are distributed over OpenMP threads; each row is summed
 * serially in index order, so results do not depend on the thread count.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { double s, c; } kahan_t;

static inline void kadd(kahan_t* k, double v) {
    /* Neumaier's improved Kahan-Babuska summation. */
    double t = k->s + v;
    if (fabs(k->s) >= fabs(v)) k->c += (k->s - t) + v;
    else k->c += (v - t) + k->s;
    k->s = t;
}
static inline double kval(const kahan_t* k) { return k->s + k->c; }

static inline double cost(int d, int r, const double* xi, const double* yj) {
    double c = 0.0;
    for (int a = 0; a < d; ++a) { double t = xi[a] - yj[a]; c += t * t; }
    return r == 2 ? c : sqrt(c);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int nt) {
#ifdef _OPENMP
    if (nt > 0) omp_set_num_threads(nt);
#else
    (void)nt;
#endif
}

/* t[q] = sum_j w[j] K(x[rows[q]], y[j]); rows == NULL means all n rows (q = i).
 * kernel 0: K = exp(-lam c); kernel 1: K = c exp(-lam c). */
void oracle_direct_sum(int d, const double* x, long long n, const double* y, long long m,
                       const double* w, double lam, int r, int kernel,
                       const long long* rows, long long nrows, double* t) {
    long long R = rows ? nrows : n;
    #pragma omp parallel for schedule(dynamic, 16)
    for (long long q = 0; q < R; ++q) {
        long long i = rows ? rows[q] : q;
        const double* xi = x + i * d;
        kahan_t acc = {0.0, 0.0};
        for (long long j = 0; j < m; ++j) {
            double c = cost(d, r, xi, y + j * d);
            double k = exp(-lam * c);
            if (kernel == 1) k *= c;
            kadd(&acc, w[j] * k);
        }
        t[q] = kval(&acc);
    }
}

/* Alg. 1 in the plain (scaling) domain, fixed iteration count. Returns the number of
 * a non-positive / non-finite denominator (0 if none). alpha, alpha_t: out. */
int oracle_sinkhorn_plain(int d, const double* x, long long n, const double* y, long long m,
                          const double* a, const double* b, double lam, int r, int iters,
                          double* alpha, double* alpha_t) {
    int bad = 0;
    for (long long i = 0; i < n; ++i) alpha[i] = 1.0;
    for (long long j = 0; j < m; ++j) alpha_t[j] = 1.0;
    for (int it = 0; it < iters; ++it) {
        /* odd Delta: alpha_i = p_i / sum_j k_ij alpha~_j */
        #pragma omp parallel for schedule(static) reduction(+:bad)
        for (long long i = 0; i < n; ++i) {
            kahan_t acc = {0.0, 0.0};
            for (long long j = 0; j < m; ++j)
                kadd(&acc, exp(-lam * cost(d, r, x + i * d, y + j * d)) * alpha_t[j]);
            double s = kval(&acc);
            if (!(s > 0.0) || !isfinite(s)) bad += 1;
            alpha[i] = a[i] / s;
        }
        /* even Delta: alpha~_j = p~_j / sum_i k_ij alpha_i */
        #pragma omp parallel for schedule(static) reduction(+:bad)
        for (long long j = 0; j < m; ++j) {
            kahan_t acc = {0.0, 0.0};
            for (long long i = 0; i < n; ++i)
                kadd(&acc, exp(-lam * cost(d, r, x + i * d, y + j * d)) * alpha[i]);
            double s = kval(&acc);
            if (!(s > 0.0) || !isfinite(s)) bad += 1;
            alpha_t[j] = b[j] / s;
        }
    }
    return bad;
}

/* log-sum-exp of lam*(pot[j] - c(p, q_j)) over j, two passes (max, then compensated sum). */
static double lse_row(int d, int r, const double* p, const double* q, long long cnt,
                      const double* pot, double lam) {
    double mx = -INFINITY;
    for (long long j = 0; j < cnt; ++j) {
        double v = lam * (pot[j] - cost(d, r, p, q + j * d));
        if (v > mx) mx = v;
    }
    kahan_t acc = {0.0, 0.0};
    for (long long j = 0; j < cnt; ++j) {
        double v = lam * (pot[j] - cost(d, r, p, q + j * d));
        kadd(&acc, exp(v - mx));
    }
    return mx + log(kval(&acc));
}

/* Log-domain Alg. 1: g^0 = 0 (alpha~ = 1), u (f) first, fixed iters. f, g: out.
 * f_in/g_in may be NULL (cold start) or a warm start for g (f_in ignored). */
void oracle_sinkhorn_log(int d, const double* x, long long n, const double* y, long long m,
                         const double* a, const double* b, double lam, int r, int iters,
                         const double* g_in, double* f, double* g) {
    for (long long j = 0; j < m; ++j) g[j] = g_in ? g_in[j] : 0.0;
    for (long long i = 0; i < n; ++i) f[i] = 0.0;
    for (int it = 0; it < iters; ++it) {
        #pragma omp parallel for schedule(static)
        for (long long i = 0; i < n; ++i)
            f[i] = (log(a[i]) - lse_row(d, r, x + i * d, y, m, g, lam)) / lam;
        #pragma omp parallel for schedule(static)
        for (long long j = 0; j < m; ++j)
            g[j] = (log(b[j]) - lse_row(d, r, y + j * d, x, n, f, lam)) / lam;
    }
}

/* out[0] = s~ (upper, transport cost), out[1] = s (dual / lower, Eq. (14)),
 * out[2] = sum pi, out[3] = |pi 1 - a|_1, out[4] = |pi^T 1 - b|_1, out[5] = H(pi). */
void oracle_divergence(int d, const double* x, long long n, const double* y, long long m,
                       const double* a, const double* b, double lam, int r,
                       const double* f, const double* g, double* out) {
    kahan_t cost_acc = {0, 0}, mass = {0, 0}, ent = {0, 0}, rres = {0, 0}, cres = {0, 0};
    kahan_t af = {0, 0}, bg = {0, 0};
    double* colsum = (double*)calloc((size_t)m, sizeof(double));
    double* colcmp = (double*)calloc((size_t)m, sizeof(double));
    /* rows in parallel; per-row partials reduced serially afterwards (deterministic). */
    double* rc = (double*)malloc((size_t)n * 4 * sizeof(double));
    #pragma omp parallel for schedule(static)
    for (long long i = 0; i < n; ++i) {
        kahan_t sc = {0, 0}, sm = {0, 0}, se = {0, 0};
        for (long long j = 0; j < m; ++j) {
            double c = cost(d, r, x + i * d, y + j * d);
            double lp = lam * (f[i] + g[j] - c);
            double pij = exp(lp);
            kadd(&sc, pij * c);
            kadd(&sm, pij);
            kadd(&se, -pij * lp);
        }
        rc[4 * i + 0] = kval(&sc);
        rc[4 * i + 1] = kval(&sm);
        rc[4 * i + 2] = kval(&se);
    }
    for (long long i = 0; i < n; ++i) {
        kadd(&cost_acc, rc[4 * i + 0]);
        kadd(&mass, rc[4 * i + 1]);
        kadd(&ent, rc[4 * i + 2]);
        kadd(&rres, fabs(rc[4 * i + 1] - a[i]));
        kadd(&af, a[i] * f[i]);
    }
    #pragma omp parallel for schedule(static)
    for (long long j = 0; j < m; ++j) {
        kahan_t s = {0, 0};
        for (long long i = 0; i < n; ++i)
            kadd(&s, exp(lam * (f[i] + g[j] - cost(d, r, x + i * d, y + j * d))));
        colsum[j] = kval(&s);
    }
    for (long long j = 0; j < m; ++j) {
        kadd(&cres, fabs(colsum[j] - b[j]));
        kadd(&bg, b[j] * g[j]);
    }
    out[0] = kval(&cost_acc);
    out[1] = 1.0 / lam + kval(&af) + kval(&bg) - kval(&mass) / lam;
    out[2] = kval(&mass);
    out[3] = kval(&rres);
    out[4] = kval(&cres);
    out[5] = kval(&ent);
    free(rc); free(colsum); free(colcmp);
}
