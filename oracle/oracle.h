/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU oracle for the hot path of Ishigami, Kimura, Nakamura,
 * "On Implementation and Evaluation of Inverse Iteration Algorithm with
 * compact WY Orthogonalization" (arXiv 1209.1910, /root/reference/PAPER.md).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so.  The product (libtinv.so)
 * never includes this header, never links this library and shares no code,
 * table or constant generator with it.
 *
 * Indexing is 0-based throughout; the paper is 1-based (paper j = our j+1).
 * Readings of silent/garbled passages are the ones listed in DESIGN.md
 * ("Readings") and SURVEY.md §8(c) R1-R5.
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* R1: ||T||_1 = max_i |e_{i-1}| + |d_i| + |e_i|. */
double orc_tnorm(int64_t n, const double* d, const double* e);

/* R2: Peters-Wilkinson clusters (Alg.4 l.8 PAPER.md:692).
 * j starts a cluster iff j==0 or w_j - w_{j-1} > 1e-3*tnorm (gap <= thr chains).
 * cstart must hold n+1 entries; returns nclus and sets cstart[nclus] = n. */
int64_t orc_clusters(int64_t n, const double* w, double tnorm, int64_t* cstart);

/* R3: shift ladder inside a cluster: wt_j = max(w_j, wt_{j-1} + 10*eps*|w_j|),
 * wt_{j1} = w_{j1}; eps = 2^-53.  (Paper assumes distinct eigenvalues.) */
void orc_shifts(int64_t n, const double* w, int64_t nclus, const int64_t* cstart, double* wt);

/* Reading 7: start-vector entry ("from random numbers").
 * SplitMix64 finaliser of seed + phi64*ctr, top 53 bits -> u in [0,1), returns 2u-1. */
uint64_t orc_splitmix64(uint64_t seed, uint64_t ctr);   /* raw 64-bit output */
double orc_rng_uniform(uint64_t seed, uint64_t ctr);
/* b_i = orc_rng_uniform(seed, 1 + (restart*n + j)*n + i), i = 0..n-1. */
void orc_start_vector(int64_t n, uint64_t seed, int64_t j, int64_t restart, double* b);

/* Reading 6: LU with partial pivoting of T - shift*I (Eq.(1)).
 * l[n-1] multipliers, piv[n-1] (1 = rows i,i+1 swapped), u0[n], u1[n-1], u2[n-2]
 * (U's three diagonals).  Pivots with |p| < eps*tnorm become sign(p)*eps*tnorm (+ if p==0). */
void orc_lu_factor(int64_t n, const double* d, const double* e, double shift, double tnorm,
                   double* l, int8_t* piv, double* u0, double* u1, double* u2);
/* Solve (T - shift I) x = b with the factors; b is overwritten by x. */
void orc_lu_solve(int64_t n, const double* l, const int8_t* piv, const double* u0,
                  const double* u1, const double* u2, double* b);

/* Eq.(2) + §3.3.2 reduced t:
 * from u[0..len-1] (= rows j..n of u_j): c = -sgn(u_0)||u||_2 (sgn(0)=+1),
 * y = u with y_0 = u_0 - c, t = 1/(c^2 - u_0 c).  Returns ||u||_2. */
double orc_reflector(int64_t len, const double* u, double* y, double* c, double* t);

/* Packed compact-WY accumulator (Fig. 1 "Assignment model", PAPER.md:630-640;
 * layout per SURVEY D4): column-major (n+1) x m buffer P, column k holds
 * T[0..k-1,k] in rows 0..k-1, t_k in row k, yhat_k (rows k..n-1 of y_k) in rows k+1..n. */
typedef struct {
    int64_t n, m, ld;   /* ld = n+1 */
    int64_t count;      /* number of reflectors held (j in the paper) */
    double* P;          /* ld*m */
} orc_cwy_t;

int  orc_cwy_init(orc_cwy_t* a, int64_t n, int64_t m);
void orc_cwy_free(orc_cwy_t* a);

/* One step of Alg.3 lines 5-8 in the §3.3.2 BLAS sequence,
 * with the erratum T_j (not T_j^T) in the q step (Eq.(4), Alg.3 l.8).
 * Given v (length n) and count = p reflectors, writes reflector p into column p
 * (overwriting any previous trial column p), sets count = p+1, and returns in q the
 * sign-flipped q_p = (Y T Y^T - I) e_p, in *c the c_p of the reflector, and in
 * *unorm ||uhat||_2.  Does NOT check degeneracy. */
void orc_cwy_step(orc_cwy_t* a, int64_t p, const double* v, double* q, double* c, double* unorm);

/* Alg.4 lines 10-11: build Y_1/T_1 from the accepted z. */
void orc_cwy_first(orc_cwy_t* a, const double* z);

/* Blocked look-ahead oracle: Y_k/T_k from V's first k columns (§3.3.2
 * steps), then U[:, v] = x_v - Y (T^T (Y^T x_v)) (trans = 1) or x_v - Y (T (Y^T x_v)) (trans = 0)
 * for the b columns of X; all arrays column-major, ld n. */
void orc_cwy_apply_block(int64_t n, int64_t k, const double* V, int64_t b, const double* X, int trans, double* U);

/* Alg. 2: Householder orthogonalisation of V (n x m, column-major,
 * ld n) into Q (ordinary sign, q_j = H_1...H_j e_j).  Test cross-check only. */
void orc_householder_orth(int64_t n, int64_t m, const double* V, double* Q);
/* Alg. 3 via the packed §3.3.2 step on given columns (q sign-flipped as in the paper). */
void orc_cwy_orth(int64_t n, int64_t m, const double* V, double* Q);
/* Packed buffer after m steps on the columns of V (test access to Y and T). */
void orc_cwy_build(int64_t n, int64_t m, const double* V, double* P);
/* §3.3.1 ordinary sequence with dense Y (n x m) and T (m x m),
 * T_j (not T_j^T) in the q step.  Test cross-check only. */
void orc_cwy_ordinary_orth(int64_t n, int64_t m, const double* V, double* Q);

/* R5: Sturm count (#eigenvalues < x) and bisection of all eigenvalues (DSTEBZ's role,
 * PAPER.md:753-755).  Zero pivot -> -eps*tnorm. */
int64_t orc_sturm_count(int64_t n, const double* d, const double* e, double x, double tnorm);
void orc_bisect(int64_t n, const double* d, const double* e, double* w);

/* Alg. 4 driver, DSTEIN-cWY with the R4 rules.
 * Z column-major ldz >= n.  iters (optional, length n) receives the iteration count
 * of each vector (restarts add to it).  Returns the number of flagged
 * (non-converged) vectors, or < 0 on invalid input. */
int64_t orc_eigvecs(int64_t n, const double* d, const double* e, const double* w,
                    double* Z, int64_t ldz, uint64_t seed, int32_t* iters);

/* Same but only for the vectors j in [j_lo, j_hi) -- clusters touching that range are
 * computed from their start so the values equal the full run's.  Used for bounded
 * CPU-baseline samples and for sampled parity at full size. */
int64_t orc_eigvecs_range(int64_t n, const double* d, const double* e, const double* w,
                          double* Z, int64_t ldz, uint64_t seed, int32_t* iters,
                          int64_t j_lo, int64_t j_hi);

/* Alg. 1 (classical inverse iteration): the same
 * factorization, start vectors, scaling, stopping rule and restarts as Alg. 4, with the
 * clustered vectors reorthogonalised by MGS against the cluster's accepted vectors after
 * every solve instead of the compact-WY step.  Same arguments as orc_eigvecs_range. */
int64_t orc_eigvecs_mgs_range(int64_t n, const double* d, const double* e, const double* w,
                              double* Z, int64_t ldz, uint64_t seed, int32_t* iters,
                              int64_t j_lo, int64_t j_hi);

#ifdef __cplusplus
}
#endif
#endif
