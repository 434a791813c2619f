/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).  Built with
 * -O2 -ffp-contract=off: no FMA contraction, plain loops in the paper's order.
 *
 * Paper: /root/reference/PAPER.md (arXiv 1209.1910).  Every function cites the
 * passage it follows; readings of silent/garbled passages are listed in DESIGN.md.
 * Nothing here is shared with the CUDA product (paper_1209_1910_b200/csrc).
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EPS 0x1.0p-53            /* unit roundoff, reading R3/R4 */
#define MAXITS 5                 /* reading 9 */
#define NPASS 2                  /* reading 9: first pass + 1 extra */
#define MAXRESTART 2             /* reading 16 */

static double dmax(double a, double b) { return a > b ? a : b; }

/* ---------------------------------------------------------------- R1, R2, R3 */

/* R1: 1-norm of the symmetric tridiagonal T = max column sum. */
double orc_tnorm(int64_t n, const double* d, const double* e)
{
    double t = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double s = fabs(d[i]);
        if (i > 0) s += fabs(e[i - 1]);
        if (i < n - 1) s += fabs(e[i]);
        if (s > t) t = s;
    }
    return t;
}

/* R2: Alg.4 l.8 "|lambda_j - lambda_{j-1}| <= 1e-3 ||T||" chains j
 * into the current cluster; otherwise l.17 "j1 <- j" starts a new one. */
int64_t orc_clusters(int64_t n, const double* w, double tnorm, int64_t* cstart)
{
    double thr = 1e-3 * tnorm;
    int64_t nc = 0;
    for (int64_t j = 0; j < n; j++) {
        if (j == 0 || !(w[j] - w[j - 1] <= thr)) cstart[nc++] = j;
    }
    cstart[nc] = n;
    return nc;
}

/* R3 (reading 5): perturbation ladder for (near-)coincident shifts. */
void orc_shifts(int64_t n, const double* w, int64_t nclus, const int64_t* cstart, double* wt)
{
    (void)n;
    for (int64_t c = 0; c < nclus; c++) {
        int64_t j1 = cstart[c], j2 = cstart[c + 1];
        wt[j1] = w[j1];
        for (int64_t j = j1 + 1; j < j2; j++) {
            double cand = wt[j - 1] + 10.0 * EPS * fabs(w[j]);
            wt[j] = dmax(w[j], cand);
        }
    }
}

/* ---------------------------------------------------------------- RNG (reading 7) */

uint64_t orc_splitmix64(uint64_t seed, uint64_t ctr)
{
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL * ctr;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double orc_rng_uniform(uint64_t seed, uint64_t ctr)
{
    uint64_t z = orc_splitmix64(seed, ctr);
    double u = (double)(z >> 11) * 0x1.0p-53;
    return 2.0 * u - 1.0;
}

void orc_start_vector(int64_t n, uint64_t seed, int64_t j, int64_t restart, double* b)
{
    uint64_t base = 1 + ((uint64_t)restart * (uint64_t)n + (uint64_t)j) * (uint64_t)n;
    for (int64_t i = 0; i < n; i++) b[i] = orc_rng_uniform(seed, base + (uint64_t)i);
}

/* ---------------------------------------------------------------- LU (reading 6) */

static double pivot_floor(double p, double tiny)
{
    if (fabs(p) < tiny) return (p >= 0.0) ? tiny : -tiny;
    return p;
}

/* Gaussian elimination with partial pivoting on the tridiagonal T - shift I
 * (the solver of Eq.(1), unnamed by the paper).
 * Row i+1 is swapped in iff |e_i| > |current pivot| (strict). */
void orc_lu_factor(int64_t n, const double* d, const double* e, double shift, double tnorm,
                   double* l, int8_t* piv, double* u0, double* u1, double* u2)
{
    double tiny = EPS * tnorm;
    if (tiny == 0.0) tiny = DBL_MIN;
    double p = d[0] - shift;                 /* pending row: diagonal   */
    double q = (n > 1) ? e[0] : 0.0;         /* pending row: super-diag */
    for (int64_t i = 0; i < n - 1; i++) {
        double sub = e[i];
        double anext = d[i + 1] - shift;
        double enext = (i + 1 < n - 1) ? e[i + 1] : 0.0;
        if (fabs(sub) > fabs(p)) {
            double pv = pivot_floor(sub, tiny);
            piv[i] = 1;
            u0[i] = pv;
            u1[i] = anext;
            if (i < n - 2) u2[i] = enext;
            l[i] = p / pv;
            p = q - l[i] * anext;
            q = -(l[i] * enext);
        } else {
            double pv = pivot_floor(p, tiny);
            piv[i] = 0;
            u0[i] = pv;
            u1[i] = q;
            if (i < n - 2) u2[i] = 0.0;
            l[i] = sub / pv;
            p = anext - l[i] * q;
            q = enext;
        }
    }
    u0[n - 1] = pivot_floor(p, tiny);
}

void orc_lu_solve(int64_t n, const double* l, const int8_t* piv, const double* u0,
                  const double* u1, const double* u2, double* b)
{
    for (int64_t i = 0; i < n - 1; i++) {
        if (piv[i]) { double t = b[i]; b[i] = b[i + 1]; b[i + 1] = t; }
        b[i + 1] = b[i + 1] - l[i] * b[i];
    }
    b[n - 1] = b[n - 1] / u0[n - 1];
    if (n >= 2) b[n - 2] = (b[n - 2] - u1[n - 2] * b[n - 1]) / u0[n - 2];
    for (int64_t i = n - 3; i >= 0; i--)
        b[i] = (b[i] - u1[i] * b[i + 1] - u2[i] * b[i + 2]) / u0[i];
}

/* ---------------------------------------------------------------- reflector */

static double nrm2(int64_t len, const double* x)
{
    double s = 0.0;
    for (int64_t i = 0; i < len; i++) s += x[i] * x[i];
    return sqrt(s);
}

/* Eq.(2) with the §3.3.2 reduced t.
 * sgn(0) = +1 (reading 14). */
double orc_reflector(int64_t len, const double* u, double* y, double* c, double* t)
{
    double nu = nrm2(len, u);
    double sg = (u[0] >= 0.0) ? 1.0 : -1.0;
    double cc = -sg * nu;
    for (int64_t i = 0; i < len; i++) y[i] = u[i];
    y[0] = u[0] - cc;
    *c = cc;
    *t = 1.0 / (cc * cc - u[0] * cc);
    return nu;
}

/* ---------------------------------------------------------------- packed cWY */

int orc_cwy_init(orc_cwy_t* a, int64_t n, int64_t m)
{
    a->n = n; a->m = m; a->ld = n + 1; a->count = 0;
    a->P = (double*)calloc((size_t)(a->ld * m), sizeof(double));
    return a->P ? 0 : -1;
}

void orc_cwy_free(orc_cwy_t* a) { free(a->P); a->P = NULL; }

/* Y(i,k): zero above row k; yhat_k in rows k+1..n of column k.  T(l,k), l<=k. */
#define PY(a, i, k) ((a)->P[((i) + 1) + (k) * (a)->ld])
#define PT(a, l, k) ((a)->P[(l) + (k) * (a)->ld])
static double Yget(const orc_cwy_t* a, int64_t i, int64_t k) { return i >= k ? PY(a, i, k) : 0.0; }

/* Memory order of the BLAS-2 loops below.  Every output element is one dot product
 * whose terms are added in exactly the order the paper's kernel defines (k ascending for
 * the row dots of DGEMV-N / DTRMV, i or l ascending for the column dots of DGEMV-T /
 * DTRMV-T), starting from 0.0.  The row dots over the column-major packed buffer walk
 * the columns in the outer loop and keep one running sum per output row ("axpy order"):
 * the same additions in the same order per element, so the result is bit-identical to
 * the plain nested loop -- only the memory stream is contiguous.  Output elements are
 * independent, so the OpenMP splits below (over whole output elements) do not change any
 * rounding either: the result does not depend on the thread count. */

/* out[i - r0] = sum_{k=0}^{kc-1} PY(i, k) * v[k] for rows i in [r0, r1) (k ascending). */
static void rowdots_Y(const orc_cwy_t* a, int64_t r0, int64_t r1, int64_t kc, const double* v,
                      double* out)
{
#pragma omp parallel
    {
        int nt = 1, id = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads(); id = omp_get_thread_num();
#endif
        int64_t len = r1 - r0, per = (len + nt - 1) / nt;
        int64_t lo = r0 + per * id, hi = lo + per < r1 ? lo + per : r1;
        for (int64_t i = lo; i < hi; i++) out[i - r0] = 0.0;
        for (int64_t k = 0; k < kc; k++) {
            double vk = v[k];
            int64_t i0 = lo > k ? lo : k;          /* Y(i, k) = 0 above row k: only i >= k */
            for (int64_t i = i0; i < hi; i++) out[i - r0] += PY(a, i, k) * vk;
        }
    }
}

/* out[l] = sum_{k=l}^{kc-1} PT(l, k) * x[k] for l in [0, kc) (k ascending). */
static void rowdots_T(const orc_cwy_t* a, int64_t kc, const double* x, double* out)
{
#pragma omp parallel
    {
        int nt = 1, id = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads(); id = omp_get_thread_num();
#endif
        int64_t per = (kc + nt - 1) / nt;
        int64_t lo = per * id, hi = lo + per < kc ? lo + per : kc;
        for (int64_t l = lo; l < hi; l++) out[l] = 0.0;
        for (int64_t k = lo; k < kc; k++) {        /* T(l, k) = 0 below the diagonal: l <= k */
            double xk = x[k];
            int64_t l1 = hi < k + 1 ? hi : k + 1;
            for (int64_t l = lo; l < l1; l++) out[l] += PT(a, l, k) * xk;
        }
    }
}

/* §3.3.2, one reflector, in the paper's BLAS order. */
void orc_cwy_step(orc_cwy_t* a, int64_t p, const double* v, double* q, double* c, double* unorm)
{
    int64_t n = a->n;
    double* uh = (double*)malloc(sizeof(double) * (size_t)(n - p));
    double* vc = (double*)malloc(sizeof(double) * (size_t)(p + 1));
    double* vin = (double*)malloc(sizeof(double) * (size_t)(p + 1));
    double* rs = (double*)malloc(sizeof(double) * (size_t)n);

    /* u-step */
    for (int64_t i = p; i < n; i++) uh[i - p] = v[i];                         /* DCOPY */
    if (p > 0) {
        for (int64_t k = 0; k < p; k++) vin[k] = v[k];
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t k = 0; k < p; k++) {                                       /* DTRMV L_p^T */
            double s = 0.0;
            for (int64_t i = k; i < p; i++) s += PY(a, i, k) * vin[i];
            vc[k] = s;
        }
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t k = 0; k < p; k++) {                                       /* DGEMV Yhat^T vhat + vc */
            double s = 0.0;
            for (int64_t i = p; i < n; i++) s += PY(a, i, k) * v[i];
            vc[k] = s + vc[k];
        }
        for (int64_t k = 0; k < p; k++) vin[k] = vc[k];
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t k = p - 1; k >= 0; k--) {                                  /* DTRMV T_p^T */
            double s = 0.0;
            for (int64_t l = 0; l <= k; l++) s += PT(a, l, k) * vin[l];
            vc[k] = s;
        }
        rowdots_Y(a, p, n, p, vc, rs);                                          /* DGEMV uhat -= Yhat vc */
        for (int64_t i = p; i < n; i++) uh[i - p] = -rs[i - p] + uh[i - p];
    }

    /* reflector.  Reading: an exactly-zero uhat is replaced by e_1. */
    double nu0 = nrm2(n - p, uh);
    if (nu0 == 0.0) uh[0] = 1.0;
    double cc, tt;
    double* yh = (double*)malloc(sizeof(double) * (size_t)(n - p));
    orc_reflector(n - p, uh, yh, &cc, &tt);

    /* that = -t T_p Yhat_p^T yhat */
    if (p > 0) {
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t k = 0; k < p; k++) {                                       /* DGEMV */
            double s = 0.0;
            for (int64_t i = p; i < n; i++) s += PY(a, i, k) * yh[i - p];
            vin[k] = (-tt) * s;
        }
        rowdots_T(a, p, vin, vc);                                               /* DTRMV T_p */
    }
    /* append column p (rollback: any earlier trial column p is overwritten), Eq.(3) */
    for (int64_t l = 0; l < p; l++) PT(a, l, p) = vc[l];
    PT(a, p, p) = tt;
    for (int64_t i = p; i < n; i++) PY(a, i, p) = yh[i - p];
    a->count = p + 1;

    /* q = (Y T Y^T - I) e_p, with T_{p+1} (erratum for T^T) */
    for (int64_t k = 0; k <= p; k++) vin[k] = PY(a, p, k);                      /* DCOPY row p */
    rowdots_T(a, p + 1, vin, vc);                                               /* DTRMV T_{p+1} */
    rowdots_Y(a, 0, p + 1, p + 1, vc, q);                                       /* DTRMV L_{p+1} */
    rowdots_Y(a, p + 1, n, p + 1, vc, q + p + 1);                               /* DGEMV Yhat_{p+1} x */
    q[p] = q[p] - 1.0;

    *c = cc;
    *unorm = nu0;
    free(uh); free(vc); free(vin); free(rs); free(yh);
}

void orc_cwy_first(orc_cwy_t* a, const double* z)
{
    double* q = (double*)malloc(sizeof(double) * (size_t)a->n);
    double c, nu;
    orc_cwy_step(a, 0, z, q, &c, &nu);
    free(q);
}

/* Blocked application of the accepted reflectors to b vectors (Eq.(4)
 * PAPER.md:304-313, Alg. 3): builds Y_k/T_k from the first k columns of V by
 * the §3.3.2 step, then for each column x of X (n x b, column-major) writes
 *   trans = 1:  U = (I - Y T Y^T)^T x = x - Y (T^T (Y^T x))   (the u-step PAPER.md:530-538)
 *   trans = 0:  U = (I - Y T Y^T) x   = x - Y (T (Y^T x))
 * in the plain order of the definition (three GEMV loops per column).  Test oracle of the
 * blocked look-ahead; nothing on the eigenvector path calls it. */
void orc_cwy_apply_block(int64_t n, int64_t k, const double* V, int64_t b, const double* X, int trans, double* U)
{
    orc_cwy_t a;
    orc_cwy_init(&a, n, k > 0 ? k : 1);
    double* q = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < k; j++) {
        double c, nu;
        orc_cwy_step(&a, j, V + j * n, q, &c, &nu);
    }
    double* g = (double*)calloc((size_t)(k + 1), sizeof(double));
    double* h = (double*)calloc((size_t)(k + 1), sizeof(double));
    for (int64_t v = 0; v < b; v++) {
        const double* x = X + v * n;
        double* out = U + v * n;
        for (int64_t c = 0; c < k; c++) {                     /* g = Y^T x */
            double s = 0.0;
            for (int64_t i = 0; i < n; i++) s += Yget(&a, i, c) * x[i];
            g[c] = s;
        }
        for (int64_t l = 0; l < k; l++) {                     /* h = T^T g  or  T g */
            double s = 0.0;
            if (trans) for (int64_t c = 0; c <= l; c++) s += PT(&a, c, l) * g[c];
            else       for (int64_t c = l; c < k; c++) s += PT(&a, l, c) * g[c];
            h[l] = s;
        }
        for (int64_t i = 0; i < n; i++) {                     /* U = x - Y h */
            double s = 0.0;
            for (int64_t c = 0; c < k; c++) s += Yget(&a, i, c) * h[c];
            out[i] = x[i] - s;
        }
    }
    free(g); free(h); free(q);
    orc_cwy_free(&a);
}

/* ---------------------------------------------------------------- cross-checks */

/* Alg. 2, with Eq.(2)'s original t = 2/||y||^2. */
void orc_householder_orth(int64_t n, int64_t m, const double* V, double* Q)
{
    double* Yd = (double*)calloc((size_t)(n * m), sizeof(double));
    double* t = (double*)calloc((size_t)m, sizeof(double));
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < m; j++) {
        for (int64_t i = 0; i < n; i++) u[i] = V[i + j * n];
        for (int64_t r = 0; r < j; r++) {                 /* u <- (I - t_r y_r y_r^T) u */
            double s = 0.0;
            for (int64_t i = 0; i < n; i++) s += Yd[i + r * n] * u[i];
            for (int64_t i = 0; i < n; i++) u[i] -= t[r] * s * Yd[i + r * n];
        }
        double ss = 0.0;
        for (int64_t i = j; i < n; i++) ss += u[i] * u[i];
        double cc = -((u[j] >= 0.0) ? 1.0 : -1.0) * sqrt(ss);
        double yy = 0.0;
        for (int64_t i = j; i < n; i++) { Yd[i + j * n] = u[i]; }
        Yd[j + j * n] = u[j] - cc;
        for (int64_t i = j; i < n; i++) yy += Yd[i + j * n] * Yd[i + j * n];
        t[j] = 2.0 / yy;
        double* qj = Q + j * n;                          /* q_j = H_0 ... H_j e_j */
        for (int64_t i = 0; i < n; i++) qj[i] = (i == j) ? 1.0 : 0.0;
        for (int64_t r = j; r >= 0; r--) {
            double s = 0.0;
            for (int64_t i = 0; i < n; i++) s += Yd[i + r * n] * qj[i];
            for (int64_t i = 0; i < n; i++) qj[i] -= t[r] * s * Yd[i + r * n];
        }
    }
    free(Yd); free(t); free(u);
}

void orc_cwy_orth(int64_t n, int64_t m, const double* V, double* Q)
{
    orc_cwy_t a;
    orc_cwy_init(&a, n, m);
    for (int64_t j = 0; j < m; j++) {
        double c, nu;
        orc_cwy_step(&a, j, V + j * n, Q + j * n, &c, &nu);
    }
    orc_cwy_free(&a);
}

/* Runs the §3.3.2 steps on the columns of V and returns the packed buffer
 * (ld = n+1, m columns) -- lets the tests rebuild Y and T and check Eq.(3)-(4). */
void orc_cwy_build(int64_t n, int64_t m, const double* V, double* P)
{
    orc_cwy_t a;
    orc_cwy_init(&a, n, m);
    double* q = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < m; j++) {
        double c, nu;
        orc_cwy_step(&a, j, V + j * n, q, &c, &nu);
    }
    memcpy(P, a.P, sizeof(double) * (size_t)((n + 1) * m));
    free(q);
    orc_cwy_free(&a);
}

/* §3.3.1, dense Y (n x m) and T (m x m); q step uses T_j (erratum). */
void orc_cwy_ordinary_orth(int64_t n, int64_t m, const double* V, double* Q)
{
    double* Y = (double*)calloc((size_t)(n * m), sizeof(double));
    double* T = (double*)calloc((size_t)(m * m), sizeof(double));
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    double* vp = (double*)malloc(sizeof(double) * (size_t)(m + 1));
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(m + 1));
#define YD(i, k) Y[(i) + (k) * n]
#define TD(l, k) T[(l) + (k) * m]
    for (int64_t j = 0; j < m; j++) {
        for (int64_t i = 0; i < n; i++) u[i] = V[i + j * n];                  /* DCOPY */
        if (j > 0) {
            for (int64_t k = 0; k < j; k++) {                                   /* DGEMV */
                double s = 0.0;
                for (int64_t i = 0; i < n; i++) s += YD(i, k) * u[i];
                vp[k] = s;
            }
            for (int64_t k = 0; k < j; k++) {                                   /* DTRMV T^T */
                double s = 0.0;
                for (int64_t l = 0; l <= k; l++) s += TD(l, k) * vp[l];
                tmp[k] = s;
            }
            for (int64_t i = 0; i < n; i++) {                                   /* DGEMV */
                double s = 0.0;
                for (int64_t k = 0; k < j; k++) s += YD(i, k) * tmp[k];
                u[i] = -s + u[i];
            }
        }
        double ss = 0.0;                                                        /* DNRM2 */
        for (int64_t i = j; i < n; i++) ss += u[i] * u[i];
        double cc = -((u[j] >= 0.0) ? 1.0 : -1.0) * sqrt(ss);
        for (int64_t i = 0; i < n; i++) YD(i, j) = (i >= j) ? u[i] : 0.0;      /* DCOPY */
        YD(j, j) = u[j] - cc;
        double yy = 0.0;                                                        /* DNRM2 */
        for (int64_t i = 0; i < n; i++) yy += YD(i, j) * YD(i, j);
        double tt = 2.0 / yy;
        for (int64_t k = 0; k < j; k++) {                                       /* DGEMV -t Y^T y */
            double s = 0.0;
            for (int64_t i = 0; i < n; i++) s += YD(i, k) * YD(i, j);
            tmp[k] = (-tt) * s;
        }
        for (int64_t l = 0; l < j; l++) {                                       /* DTRMV T */
            double s = 0.0;
            for (int64_t k = l; k < j; k++) s += TD(l, k) * tmp[k];
            TD(l, j) = s;
        }
        TD(j, j) = tt;
        for (int64_t k = 0; k <= j; k++) vp[k] = YD(j, k);                      /* DCOPY row j */
        for (int64_t l = 0; l <= j; l++) {                                      /* DTRMV T_j */
            double s = 0.0;
            for (int64_t k = l; k <= j; k++) s += TD(l, k) * vp[k];
            tmp[l] = s;
        }
        double* qj = Q + j * n;
        for (int64_t i = 0; i < n; i++) {                                       /* DGEMV */
            double s = 0.0;
            for (int64_t k = 0; k <= j; k++) s += YD(i, k) * tmp[k];
            qj[i] = ((i == j) ? 1.0 : 0.0) - s;
        }
    }
#undef YD
#undef TD
    free(Y); free(T); free(u); free(vp); free(tmp);
}

/* ---------------------------------------------------------------- bisection (R5) */

int64_t orc_sturm_count(int64_t n, const double* d, const double* e, double x, double tnorm)
{
    double pivmin = EPS * tnorm;
    if (pivmin == 0.0) pivmin = DBL_MIN;
    int64_t cnt = 0;
    double q = d[0] - x;
    if (q == 0.0) q = -pivmin;
    if (q < 0.0) cnt++;
    for (int64_t i = 1; i < n; i++) {
        q = (d[i] - x) - (e[i - 1] * e[i - 1]) / q;
        if (q == 0.0) q = -pivmin;
        if (q < 0.0) cnt++;
    }
    return cnt;
}

void orc_bisect(int64_t n, const double* d, const double* e, double* w)
{
    double tnorm = orc_tnorm(n, d, e);
    double gl = d[0], gu = d[0];
    for (int64_t i = 0; i < n; i++) {
        double r = 0.0;
        if (i > 0) r += fabs(e[i - 1]);
        if (i < n - 1) r += fabs(e[i]);
        if (d[i] - r < gl) gl = d[i] - r;
        if (d[i] + r > gu) gu = d[i] + r;
    }
    double bn = dmax(fabs(gl), fabs(gu));
    double pad = 2.0 * (double)n * EPS * bn + 2.0 * DBL_MIN;
    if (tnorm > 0.0) pad += 2.0 * EPS * tnorm;
    gl -= pad; gu += pad;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t k = 0; k < n; k++) {
        double lo = gl, hi = gu;
        for (;;) {
            double mid = lo + 0.5 * (hi - lo);
            if (mid <= lo || mid >= hi) break;
            if (orc_sturm_count(n, d, e, mid, tnorm) > k) hi = mid; else lo = mid;
        }
        w[k] = lo + 0.5 * (hi - lo);
    }
}

/* ---------------------------------------------------------------- Alg. 4 driver */

static void finalize_vector(int64_t n, const double* b, double* z)
{
    /* Alg.4 l.20 "Normalize"; sign rule = reading 15. */
    double nb = nrm2(n, b);
    int64_t im = 0;
    double am = -1.0;
    for (int64_t i = 0; i < n; i++)
        if (fabs(b[i]) > am) { am = fabs(b[i]); im = i; }
    double s = (b[im] < 0.0) ? -1.0 : 1.0;
    for (int64_t i = 0; i < n; i++) z[i] = s * (b[i] / nb);
}

static double norm1(int64_t n, const double* x)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += fabs(x[i]);
    return s;
}

static double norminf(int64_t n, const double* x)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) if (fabs(x[i]) > s) s = fabs(x[i]);
    return s;
}

/* Alg. 1 l.10-12, the classical reorthogonalisation: modified Gram-Schmidt
 * of x against the cluster's accepted vectors V[:, 0..p-1] (column-major, ld n), in order:
 * x <- x - <x, v_i> v_i. */
static void mgs_project(int64_t n, int64_t p, const double* V, double* x)
{
    for (int64_t i = 0; i < p; i++) {
        const double* v = V + i * n;
        double dot = 0.0;
        for (int64_t r = 0; r < n; r++) dot += x[r] * v[r];
        for (int64_t r = 0; r < n; r++) x[r] = x[r] - dot * v[r];
    }
}

/* One cluster [j1, j2), vectors computed for j < jstop, written for j in [wlo, whi).
 * mgs = 0: Alg. 4 (compact WY); mgs = 1: Alg. 1 (classical MGS) with the same readings. */
static int64_t do_cluster(int64_t n, const double* d, const double* e, const double* wt,
                          double tnorm, uint64_t seed, int64_t j1, int64_t j2, int64_t jstop,
                          int64_t wlo, int64_t whi, double* Z, int64_t ldz, int32_t* iters, int mgs)
{
    int64_t m = j2 - j1;
    int64_t nflag = 0;
    double* l = (double*)malloc(sizeof(double) * (size_t)(n > 1 ? n - 1 : 1));
    int8_t* piv = (int8_t*)malloc((size_t)(n > 1 ? n - 1 : 1));
    double* u0 = (double*)malloc(sizeof(double) * (size_t)n);
    double* u1 = (double*)malloc(sizeof(double) * (size_t)(n > 1 ? n - 1 : 1));
    double* u2 = (double*)malloc(sizeof(double) * (size_t)(n > 2 ? n - 2 : 1));
    double* b = (double*)malloc(sizeof(double) * (size_t)n);
    double* x = (double*)malloc(sizeof(double) * (size_t)n);
    double* q = (double*)malloc(sizeof(double) * (size_t)n);
    double* zacc = (double*)malloc(sizeof(double) * (size_t)n);
    orc_cwy_t acc;
    acc.P = NULL;
    if (m > 1 && !mgs) orc_cwy_init(&acc, n, m);
    /* MGS: the cluster's accepted vectors, column-major n x m */
    double* V = (m > 1 && mgs) ? (double*)malloc(sizeof(double) * (size_t)n * (size_t)m) : NULL;
    double thr = sqrt(0.1 / (double)n);                /* reading 9 (DSTEIN-style) */

    for (int64_t j = j1; j < jstop; j++) {
        int64_t p = j - j1;                            /* j_c, Alg.4 l.9 */
        orc_lu_factor(n, d, e, wt[j], tnorm, l, piv, u0, u1, u2);
        double unn = fabs(u0[n - 1]);
        if (p == 1 && !mgs) orc_cwy_first(&acc, zacc); /* Alg.4 l.10-11: Y_1,T_1 from v_{j1} */
        int converged = 0, its = 0, degen_final = 0;
        for (int64_t rs = 0; rs <= MAXRESTART; rs++) {
            orc_start_vector(n, seed, j, rs, b);       /* Alg.4 l.2 */
            int passes = 0, degenerate = 0;
            for (int k = 1; k <= MAXITS; k++) {
                its++;
                double nb = nrm2(n, b);                /* l.6 Normalize */
                for (int64_t i = 0; i < n; i++) b[i] = b[i] / nb;
                double sigma = (double)n * tnorm * dmax(EPS, unn) / norm1(n, b);   /* reading 8 */
                for (int64_t i = 0; i < n; i++) x[i] = sigma * b[i];
                orc_lu_solve(n, l, piv, u0, u1, u2, x);                              /* l.7 Eq.(1) */
                double rinf;
                if (p == 0) {
                    rinf = norminf(n, x);
                    memcpy(b, x, sizeof(double) * (size_t)n);
                } else if (mgs) {
                    /* Alg.1 l.10-12: MGS against v_{j1} .. v_{j-1}; the iterate r of reading 9
                     * is the projected x (in exact arithmetic |c| q of the cWY step); the
                     * degeneracy test of reading 16 compares its norm with ||x||_2 */
                    double nx = nrm2(n, x);
                    memcpy(q, x, sizeof(double) * (size_t)n);
                    mgs_project(n, p, V, q);
                    if (nrm2(n, q) <= (double)n * EPS * nx) {
                        if (rs < MAXRESTART) { degenerate = 1; break; }
                        degen_final = 1;
                    }
                    rinf = norminf(n, q);
                    memcpy(b, q, sizeof(double) * (size_t)n);
                } else {
                    double c, nu;
                    orc_cwy_step(&acc, p, x, q, &c, &nu);                              /* l.13-16 */
                    if (nu <= (double)n * EPS * nrm2(n, x)) {          /* reading 16 */
                        if (rs < MAXRESTART) { degenerate = 1; break; }
                        degen_final = 1;
                    }
                    rinf = fabs(c) * norminf(n, q);
                    memcpy(b, q, sizeof(double) * (size_t)n);
                }
                if (rinf >= thr) passes++;
                if (passes >= NPASS) { converged = 1; break; }   /* l.19 "until ..." */
            }
            if (!degenerate) break;
        }
        if (!converged || degen_final) nflag++;
        finalize_vector(n, b, zacc);
        if (V) memcpy(V + p * n, zacc, sizeof(double) * (size_t)n);
        if (iters && j >= wlo && j < whi) iters[j] = its;
        if (j >= wlo && j < whi) memcpy(Z + j * ldz, zacc, sizeof(double) * (size_t)n);
    }
    if (m > 1 && !mgs) orc_cwy_free(&acc);
    free(V);
    free(l); free(piv); free(u0); free(u1); free(u2); free(b); free(x); free(q); free(zacc);
    return nflag;
}

static int64_t eigvecs_range(int64_t n, const double* d, const double* e, const double* w,
                             double* Z, int64_t ldz, uint64_t seed, int32_t* iters,
                             int64_t j_lo, int64_t j_hi, int mgs)
{
    if (n < 1 || ldz < n || !d || !w || !Z || (n > 1 && !e)) return -1;
    for (int64_t j = 1; j < n; j++) if (!(w[j] >= w[j - 1])) return -4;
    double tnorm = orc_tnorm(n, d, e);
    if (n == 1 || tnorm == 0.0) {                       /* special cases: Z = I */
        for (int64_t j = j_lo; j < j_hi; j++) {
            for (int64_t i = 0; i < n; i++) Z[i + j * ldz] = (i == j) ? 1.0 : 0.0;
            if (iters) iters[j] = 0;
        }
        return 0;
    }
    /* R0 (reading 21; the paper is silent on scaling): if ||T||_1 lies outside
     * [2^-200, 2^200], T and w are multiplied by the power of two 2^k that brings ||T||_1 into
     * [1, 2) -- exact, and 2^k T has the eigenvectors of T -- so that sigma (reading 8), the
     * pivot floor and the iterates' norms stay in the normal floating-point range. */
    double *dsc = NULL, *esc = NULL, *wsc = NULL;
    if (!(tnorm >= 0x1p-200 && tnorm <= 0x1p200)) {
        int ex;
        frexp(tnorm, &ex);
        const int k = 1 - ex;
        dsc = (double*)malloc(sizeof(double) * (size_t)n);
        esc = (double*)malloc(sizeof(double) * (size_t)n);
        wsc = (double*)malloc(sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; i++) { dsc[i] = ldexp(d[i], k); wsc[i] = ldexp(w[i], k); }
        for (int64_t i = 0; i + 1 < n; i++) esc[i] = ldexp(e[i], k);
        d = dsc; e = esc; w = wsc;
        tnorm = orc_tnorm(n, d, e);
    }
    int64_t* cs = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    double* wt = (double*)malloc(sizeof(double) * (size_t)n);
    int64_t nc = orc_clusters(n, w, tnorm, cs);
    orc_shifts(n, w, nc, cs, wt);
    int64_t nflag = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : nflag) if (nc > 1)
    for (int64_t c = 0; c < nc; c++) {
        int64_t j1 = cs[c], j2 = cs[c + 1];
        if (j2 <= j_lo || j1 >= j_hi) continue;
        int64_t jstop = j2 < j_hi ? j2 : j_hi;
        nflag += do_cluster(n, d, e, wt, tnorm, seed, j1, j2, jstop, j_lo, j_hi, Z, ldz, iters, mgs);
    }
    free(cs); free(wt);
    free(dsc); free(esc); free(wsc);
    return nflag;
}

int64_t orc_eigvecs_range(int64_t n, const double* d, const double* e, const double* w,
                          double* Z, int64_t ldz, uint64_t seed, int32_t* iters,
                          int64_t j_lo, int64_t j_hi)
{
    return eigvecs_range(n, d, e, w, Z, ldz, seed, iters, j_lo, j_hi, 0);
}

int64_t orc_eigvecs_mgs_range(int64_t n, const double* d, const double* e, const double* w,
                              double* Z, int64_t ldz, uint64_t seed, int32_t* iters,
                              int64_t j_lo, int64_t j_hi)
{
    return eigvecs_range(n, d, e, w, Z, ldz, seed, iters, j_lo, j_hi, 1);
}

int64_t orc_eigvecs(int64_t n, const double* d, const double* e, const double* w,
                    double* Z, int64_t ldz, uint64_t seed, int32_t* iters)
{
    return orc_eigvecs_range(n, d, e, w, Z, ldz, seed, iters, 0, n);
}
