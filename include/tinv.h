/*
 * tinv.h -- C ABI of the B200-native inverse iteration with compact-WY
 * reorthogonalisation (libtinv.so).
 *
 * Operation (§2.1, and §4 Alg. 4, lines 681-716 of
 * /root/reference/PAPER.md, arXiv 1209.1910): given a real symmetric tridiagonal
 * T = tridiag(e, d, e) of order n and its ascending (approximate) eigenvalues w,
 * compute all n eigenvectors Z (T z_j ~= w_j z_j, Z^T Z ~= I) by inverse iteration
 * (Eq. (1)); eigenvectors of each Peters-Wilkinson cluster (gap <=
 * 1e-3 ||T||_1, lines 135-139) are reorthogonalised with the compact WY Householder
 * orthogonalisation in the paper's reduced formulation (§3.3.2).
 * Readings of the points the paper leaves open (start vectors, shift perturbation,
 * solver, stopping rule, signs) are listed in DESIGN.md and are shared with the CPU
 * oracle only as rules, never as code.
 *
 * All compute runs in the library's own sm_100a kernels on the handle's stream.
 * There is no CPU fallback: on a machine without a usable CUDA device every call
 * returns TINV_ERR_CUDA.
 */
#ifndef TINV_H
#define TINV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tinv_s* tinv_t;

typedef struct {
    int         device;   /* CUDA ordinal this handle drives                                 */
    int         nranks;   /* number of cooperating ranks (processes), 1 = single GPU         */
    int         rank;     /* 0 .. nranks-1                                                    */
    const void* nccl_id;  /* 128-byte ncclUniqueId created by rank 0 and broadcast by the
                             caller, or NULL when nranks == 1                                 */
    void*       stream;   /* cudaStream_t the work is ordered on (NULL = legacy default)      */
} tinv_config_t;

/* Return codes (LAPACK INFO style).
 *   0      success
 *  -k      argument k is invalid, counting the handle as argument 1 (n < 1, NULL
 *          pointer, ldz < n, non-finite d/e/w, w not ascending)
 *  >0      number of eigenvectors that did not meet the stopping rule within MAXITS = 5
 *          iterations (they are still written, best iterate)
 *  <=-100  library failure, decode with tinv_strerror() */
#define TINV_OK            0
#define TINV_ERR_CUDA   -100
#define TINV_ERR_NOMEM  -101
#define TINV_ERR_NCCL   -102
#define TINV_ERR_HANDLE -103
#define TINV_ERR_DEVICE -104
#define TINV_ERR_UNSUPPORTED -105   /* a cluster exceeds the shared-memory staging limit, or
                                       MGS mode with a cluster the resident kernel cannot hold */

/* Create a handle bound to cfg->device and cfg->stream.  With nranks > 1 each rank
 * creates its handle with the same nccl_id (clusters are then sharded across ranks).
 * Ownership: the handle owns its device workspace (allocated lazily, cached across
 * calls, freed by tinv_destroy).  One handle per host thread. */
int tinv_create(tinv_t* h, const tinv_config_t* cfg);

/* Compute all eigenvectors.
 *   n     order of T (n >= 1)
 *   d     DEVICE pointer, n doubles: diagonal of T                       (read only)
 *   e     DEVICE pointer, n-1 doubles: off-diagonal of T; may be NULL iff n == 1
 *   w     DEVICE pointer, n doubles: eigenvalues of T, non-decreasing   (read only)
 *   Z     DEVICE pointer, ldz*n doubles, column-major: on return column j holds the unit
 *         eigenvector of w[j], sign fixed so that its largest-|.| entry (lowest index on
 *         ties) is positive.  Every column is overwritten.
 *   ldz   leading dimension of Z (ldz >= n)
 *   seed  seed of the counter-based start-vector generator (reading 7)
 * The call is synchronous with respect to the host (it returns the convergence count)
 * and stream-ordered on the handle's stream.  Special cases: n == 1 -> Z = [1];
 * ||T||_1 == 0 -> Z = I.  With nranks > 1 every rank passes identical arguments and Z
 * is complete on every rank on return. */
int tinv_eigvecs(tinv_t h, int64_t n, const double* d, const double* e, const double* w,
                 double* Z, int64_t ldz, uint64_t seed);

/* Eigenvalues of T by Sturm-count bisection (the DSTEBZ step before DSTEIN-cWY,
 * PAPER.md:753-755): w[k] = k-th smallest eigenvalue to full fp64 accuracy (bisection of the
 * padded Gershgorin interval until the midpoint equals an endpoint; Sturm count with LDL^T
 * pivots, a zero pivot replaced by -eps ||T||_1 -- DESIGN.md reading 20).  d (n), e (n-1,
 * NULL iff n == 1) and w (n, written, ascending) are DEVICE pointers.  Synchronous on the
 * handle's stream.  Returns 0 or -k for invalid argument k (n < 1, NULL pointers). */
int tinv_eigvals(tinv_t h, int64_t n, const double* d, const double* e, double* w);

/* tinv_eigvals followed by tinv_eigvecs: all eigenpairs (w, Z) of T from (d, e) alone.
 * Arguments and return codes as for tinv_eigvecs (w is written instead of read). */
int tinv_eig(tinv_t h, int64_t n, const double* d, const double* e, double* w, double* Z, int64_t ldz,
             uint64_t seed);

/* Same operation with HOST buffers (end-to-end path): the library copies d, e, w to the
 * device and runs tinv_eigvecs.  When Z is page-locked host memory mapped into the device
 * address space (cudaHostAlloc / cudaMallocHost under UVA) and nranks == 1, the kernels write
 * the finished columns straight into Z over PCIe, overlapped with the remaining compute;
 * otherwise Z is computed in a device buffer and copied back after the last kernel. */
int tinv_eigvecs_host(tinv_t h, int64_t n, const double* d, const double* e, const double* w,
                      double* Z, int64_t ldz, uint64_t seed);

/* Multi-rank partition of the eigenvectors (host only, no device needed): the clusters
 * (cstart[0..nclus], cstart[0] = 0, cstart[nclus] = n, strictly increasing: the
 * Peters-Wilkinson clusters of PAPER.md:135-139) are split into nranks contiguous,
 * cost-balanced column ranges [col_lo[r], col_hi[r]) that never cut a cluster (cost of a
 * cluster of m >= 2 vectors: m^2 n, the reorthogonalisation's HBM traffic; singletons: 1).
 * tinv_eigvecs with nranks > 1 computes exactly these columns on rank r, except the columns
 * of the row-split cluster (below), which every rank computes together.  Deterministic.
 * Returns 0, or -k for invalid argument k (n < 1; nclus outside [1, n]; cstart NULL or not a
 * valid cluster table; nranks < 1; col_lo / col_hi NULL).  Arrays are caller-owned host
 * memory of nclus + 1 and nranks entries. */
int tinv_partition(int64_t n, int64_t nclus, const int* cstart, int nranks, int* col_lo, int* col_hi);

/* tinv_partition plus the row split (SURVEY §8(e) regime 2): *split (if not NULL) receives the
 * index of the cluster whose rows are split over all ranks -- the costliest cluster when it is
 * wide (m > 64) and costs at least 1/nranks of all clusters' m^2 n -- or -1 (nranks == 1 or no
 * such cluster).  The ranges are balanced without that cluster's cost; its columns end up
 * complete on every rank.  Same return codes as tinv_partition. */
int tinv_plan(int64_t n, int64_t nclus, const int* cstart, int nranks, int* col_lo, int* col_hi, int* split);

/* Release the handle and its device workspace.  With nranks > 1 and a previous row-split
 * call (peers hold CUDA IPC mappings of this rank's workspace) it is collective: every rank
 * must call it, so that all mappings are closed (and a barrier passed) before any rank frees
 * its exported memory. */
int tinv_destroy(tinv_t h);

/* Human-readable text of a return code (static storage). */
const char* tinv_strerror(int code);

/* ---------------------------------------------------------------- introspection
 * Statistics of the last tinv_eigvecs call on this handle.  Kernel times are filled
 * only when profiling is enabled (CUDA events on the handle's stream around each
 * launch; adds a few microseconds per launch). */
#define TINV_NKERNELS 6
typedef struct {
    int64_t n;
    int64_t nclusters;          /* Peters-Wilkinson clusters (size >= 1)              */
    int64_t max_cluster;        /* largest cluster size m                             */
    int64_t n_clustered;        /* vectors with j_c >= 1 (reorthogonalised)           */
    int64_t nflagged;           /* vectors that missed the stopping rule              */
    int64_t iters_hist[8];      /* vectors by iteration count (index 7 = 7 or more)   */
    int64_t launches;           /* kernels launched by the last call                  */
    int64_t group_syncs;        /* group barrier episodes in the cWY kernel (per group max) */
    int64_t ngroups;            /* CTA groups used by the cWY kernel                  */
    int64_t cwy_ctas;           /* CTAs of the cWY kernel                             */
    int64_t resident_groups;    /* launches of the resident (DSMEM) cWY kernel        */
    double  reorth_bytes;       /* algorithmic bytes of the cWY passes, from the
                                   call's iteration counts (computed when the stats are read) */
    double  solve_bytes;        /* algorithmic bytes of the batched LU kernel         */
    double  kernel_ms[TINV_NKERNELS];     /* prep, batched_lu, finalize, cwy, misc, total */
    int64_t kernel_launches[TINV_NKERNELS];
    double  cwy_phase_ms[16];   /* group 0 of the cWY kernel, wall time per phase: first
                                   reflector, A, R1, TT, BC, R2, TN, D, test, chained solve
                                   (forward sweep), chained solve (back sweep), wait for the
                                   look-ahead pass overlapped with the back sweep; then the
                                   narrow-cluster streams: ring wait, stage compute, stage
                                   barrier; one spare.  With resident launches slots 8..15
                                   hold the resident kernel's unit-0 phases (A/R1, TT+BC,
                                   R2+TN, D+TEST, back-sweep staging, forward pass, back
                                   sweep, x copy); with no persistent launch slots 0..3 hold
                                   the batched LU's warp-0 sweeps (factor, back, forward,
                                   back) */
    int64_t dz_parked;          /* vectors whose last pass D was deferred to dz_gemm */
    int64_t dz_redo;            /* > 0: parked vectors failed their deferred test and the call
                                   was re-run without deferral; -1: re-run forced (TINV_DZ=2) */
    double  dz_ms;              /* deferred pass D kernels (dz_gemm + dz_finish, inside the cwy
                                   time of kernel_ms), profiling only                 */
} tinv_stats_t;

int tinv_set_profiling(tinv_t h, int enable);

/* Deferred final pass D (default on, single-rank calls): in the last iteration of a
 * wide cluster's vector the step's pass D (q = Y_{p+1} x' - e_p) is not
 * streamed per vector; x' is kept and one GEMM after the cWY kernel forms every such q, the
 * stopping test (Alg. 4) and z_j.  A vector whose deferred test fails makes
 * the call re-run without deferral, so results follow Alg. 4 either way.  enable = 0 turns it
 * off.  Returns 0 or TINV_ERR_HANDLE. */
int tinv_set_deferred(tinv_t h, int enable);

/* Testing aid for the multi-GPU row split on a single device: when the
 * clustered work of a tinv_eigvecs call is one cluster of more than 64 vectors, split it over
 * `nranks` virtual ranks -- groups of CTAs of the one launch, each with its own replica of
 * the workspace, exchanging through mirrored stores, partial sums read from their owner's
 * replica and the rank-replicated barrier, exactly as real ranks do over NVLink.  1 (the
 * default) disables it.  Returns 0, -2 for nranks outside [1, 16], TINV_ERR_HANDLE. */
int tinv_set_virtual_ranks(tinv_t h, int nranks);

/* Narrow clusters (m <= 64, n <= 4096) normally run in the resident kernel (one thread-block
 * cluster per eigen-cluster, Y kept in distributed shared memory); enable = 0 routes them
 * through the streaming persistent kernel instead (same results up to rounding; used to
 * compare the two paths).  Returns 0 or TINV_ERR_HANDLE. */
int tinv_set_resident(tinv_t h, int enable);

/* Reorthogonalisation of clustered vectors: mode 0 (default) = compact WY, Alg. 4
 * in the reduced BLAS sequence of §3.3.2; mode 1 = the classical inverse
 * iteration's modified Gram-Schmidt, Alg. 1, the
 * paper's comparison method: after every solve, x <- x - <x, z_i> z_i for the cluster's
 * accepted vectors in order, one cluster-wide reduction per z_i; mode 2 = compact WY in the
 * ordinary sequence of §3.3.1 (with the T_j erratum fixed; SURVEY §8(f)
 * row 4): Y^T y_j by a pass of its own instead of the reduced sequence's reuse of the BC pass.
 * Same factorization, start vectors, stopping rule and restarts; the vectors agree with mode 0
 * up to rounding.  Narrow clusters run them in the resident kernel, wide ones in the
 * persistent kernel (MGS with one group barrier per accepted vector on groups of at most
 * TINV_MGS_G = 16 CTAs); a cluster row-split over ranks (nranks > 1 or virtual ranks) makes
 * tinv_eigvecs return TINV_ERR_UNSUPPORTED in modes 1 and 2.  Returns 0, -2 for another mode,
 * TINV_ERR_HANDLE. */
int tinv_set_reorth(tinv_t h, int mode);

/* Blocked look-ahead (Eq. (4), Alg. 3 PAPER.md:314-334,
 * the u-step PAPER.md:530-538): for wide clusters (m > 64) of single-rank groups, at the start
 * of every block of b consecutive vectors k .. k+b-1 the accepted reflectors are applied to
 * the block's first iterates at once, U = (I - Y_k T_k^T Y_k^T) X = X - Y_k (T_k^T (Y_k^T X)),
 * as two skinny GEMMs and a TRMM (fp64, one pass over Y_k for each GEMM instead of two per
 * vector); vector p of the block then applies only the reflectors k .. p-1 of its own block
 * to its column of U.  Same results up to rounding.  b in 2..8 (larger values are clamped),
 * 0 or 1 = off (default; the environment variable TINV_LAB overrides).  Compact-WY modes only
 * (ignored with MGS).  Returns 0 or TINV_ERR_HANDLE. */
int tinv_set_lookahead(tinv_t h, int b);

/* Multi-rank diagnostics (SURVEY §8(e) row split; the peer-memory path of a row-split call
 * without its cross-rank barrier, so several ranks may share one GPU).
 *
 * tinv_allgather_fn: a host all-gather supplied by the caller -- every rank passes `bytes`
 * bytes at `send`; on return `recv` holds nranks * bytes, rank k's at k * bytes.  Collective;
 * returns 0 on success.  tinv_set_host_exchange(h, fn, ctx) makes the library exchange its
 * CUDA IPC handles (and run its unmap barrier) through fn instead of NCCL; fn = NULL restores
 * NCCL.  A handle may be created with nranks > 1 and nccl_id = NULL (no communicator): then
 * tinv_eigvecs returns TINV_ERR_NCCL and only these diagnostics work.
 *
 * tinv_debug_peer_map(h, bytes, tag, out): collective.  Grows the handle's cWY workspace to at
 * least `bytes` (>= 64) exactly as a row-split call does (peers unmap the old allocation,
 * collectively, before it is freed), writes `tag` into its first 8 bytes, maps every peer
 * rank's workspace through CUDA IPC (cudaIpcGetMemHandle / cudaIpcOpenMemHandle, handles
 * exchanged as above), then a kernel reads the first 8 bytes of every rank's replica through
 * those mappings into out[0 .. nranks) (HOST array; out[k] = rank k's tag).  The mappings stay
 * open until the next growth, a column-sharded call or tinv_destroy (collective).  Returns 0,
 * -2 (nranks < 2 or bytes < 64), -4 (out NULL), TINV_ERR_NCCL, TINV_ERR_CUDA. */
typedef int (*tinv_allgather_fn)(const void* send, void* recv, size_t bytes, void* ctx);
int tinv_set_host_exchange(tinv_t h, tinv_allgather_fn fn, void* ctx);
int tinv_debug_peer_map(tinv_t h, size_t bytes, uint64_t tag, uint64_t* out);
int tinv_get_stats(tinv_t h, tinv_stats_t* out);

/* Number of exported entry points (for the loader test). */
int tinv_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TINV_H */
