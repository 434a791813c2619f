// tinv_internal.h -- argument blocks shared by the host orchestrator and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tinv {
constexpr int kWidePieceW = 448;   // column block / row piece width of the wide passes (cwy.cu PW)

struct GroupBarrier;

// Small device-resident summary written by prep and the solve kernels, read back once.
struct PrepOut {
    double tnorm;
    int bad;            // bit0 d, bit1 e, bit2 w (non-finite or not ascending)
    int nclus;
    int max_cluster;
    int n_clustered;
    int nflag;          // vectors that missed the stopping rule
    int nc_pad;         // slots of the vectors the batched LU iterates, rounded up to 32
    int scale_exp;      // k of the 2^k scaling (reading 21), 0 inside the window
    int dzfail;         // parked vectors (deferred pass D) whose stopping test failed -> re-run
    int dzpark;         // parked vectors (deferred pass D) formed by dz_finish
};

struct PrepArgs {
    int64_t n;
    const double* d;
    const double* e;
    const double* w;
    double* ds;         // d and e as the kernels use them (n each): copies, scaled by 2^k when
    double* es;         // ||T||_1 is outside [2^-200, 2^200] (reading 21); es[n-1] = 0
    double* wt;         // perturbed shifts (n)
    int* cstart;        // cluster starts (n+1)
    int* cid;           // cluster of each vector (n)
    int* jc;            // position inside its cluster (n)
    // Slot permutation of the batched LU (warps hold 32 consecutive slots): the vectors it
    // iterates to convergence (cluster leaders, singletons) take slots [0, nc), the rest
    // (j_c >= 1, and leaders handed to the resident kernel) slots [nc_pad, nc_pad + n - nc);
    // the gap and the tail are dead slots (perm = -1).  perm has nslot_cap entries.
    int* slot;          // slot of each vector (n)
    int* perm;          // vector of each slot, or -1
    int64_t nslot_cap;  // roundup(n, 32) + 32
    int handover;       // leaders of clusters with 2 <= m <= handover finish in the resident kernel (0: none)
    PrepOut* out;
};

// Batched shifted LU inverse iteration: one thread per eigenvector, interleaved
// [row i][vector j] layout (element (i, j) at i*ldv + j) for coalesced warps.
struct BatchedArgs {
    int64_t n;
    int64_t ldv;        // interleave stride (>= n)
    const double* d;
    const double* e;
    const double* wt;
    const int* jc;
    const int* perm;    // vector of each slot (prep), -1 for dead slots
    uint64_t seed;
    // factors, block-row layout over slots (common.cuh bix(i, slot, n))
    double* fl;         // multipliers l_i (row i < n-1)
    int8_t* fp;         // row swap flags
    double* fr;         // 1/u0_i
    double* fb;         // u1_i/u0_i
    double* fc;         // u2_i/u0_i
    double* X;          // iterate / solution, [i][j] (iterating warps)
    double* X1c;        // x^(1) of first-solve vectors, [j][i], vector stride roundup(n, 2)
    double* unn;        // |u_{n-1,n-1}| per vector
    double* zscale;     // sign/||x||_2 of finished (j_c == 0) vectors
    int* iters;         // iteration count per vector
    PrepOut* out;
    unsigned long long* prof;   // optional sweep timers of warp 0 (ns), or NULL
    int stage_de;               // set by the launcher: d, e staged in shared memory
    int mode;                   // 0: every warp; 1: only the first-solve warps (slots >= nc_pad);
                                // 2: only the iterating warps (slots < nc_pad)
};

struct PackArgs {
    int64_t n;
    int64_t ldv;
    const int* perm;    // slots >= out->nc_pad are packed
    const PrepOut* out;
    const double* fl;
    const double* fr;
    const double* fb;
    const double* fc;
    const int8_t* fp;
    double* F;          // [j][i][4]: l, 1/u0, u1/u0, u2/u0
    int8_t* FP;         // [j][i] pivot bits
};

struct FinalizeArgs {
    int64_t n;
    int64_t ldv;
    const double* X;
    const double* zscale;
    const int* perm;    // slots < out->nc_pad are finished here
    double* Z;
    int64_t ldz;
    const PrepOut* out;
};

// Per-group workspace of the persistent compact-WY kernel.
struct GroupWS {
    double* Y;          // packed row-major Y (y_row_off(n, mcap) doubles)
    double* Tc;         // column-packed T (tcol_off(mcap))
    double* Tr;         // row-major T, row stride m2cap (mcap * m2cap)
    double* x;          // current iterate (n)
    double* q;          // orthogonalised vector (n)
    double* u;          // uhat / yhat (n)
    double* g;          // Y^T x, then T^T g   (mcap)
    double* gp;         // T^T g               (mcap)
    double* s;          // Yhat^T yhat          (mcap)
    double* xp;         // T_{p+1} y_row        (mcap + 1)
    double* P;          // partial sums [Gt][mcap] (a rank writes only its own CTAs' slots)
    double* S;          // scalar partials [Gt][16] (Gt = CTAs of the group over all ranks)
    double* P2;         // look-ahead partial sums [Gt][mcap]
    double* tyr;        // T_p yrow of the current vector (mcap), kept across its iterations
    double* ysol;       // forward-sweep workspace of the chained solve (n)
    // blocked look-ahead (CwyArgs::lab > 1, wide clusters): for the block of
    // b upcoming first iterates X = [x^(1)_k .. x^(1)_{k+b-1}]:  G = Y_k^T X,  G' = T_k^T G
    // (labG, [v][mcap]),  U = X - Y_k G'  (labU, [v][n2v], rows >= k), ||x_v||^2 (labX2 [v]);
    // labP: per-CTA partials of ||x_v||^2 [Gt][8].  NULL when the group has no block look-ahead.
    double* labG;
    double* labGp;
    double* labU;
    double* labX2;
    double* labP;
    double* labQ;       // fused in-block dots [Gt][v][q] (per CTA, from the BC pass of block vector k+q)
    double* labY0;      // y_0 of the block's vectors [8]
    double* labPB;      // streamed BL1: per (column block, CTA) partial sums [(NB + Gt)][8][448], or NULL
    GroupBarrier* bar;
    int64_t mcap;
    // Row split of one cluster over `nrk` ranks: every rank holds a full
    // replica of this workspace with the same layout; `delta[k]` (doubles) moves a pointer
    // into this replica to the same place in rank k's replica (delta[rk] = 0).  nrk == 1:
    // plain single-GPU group.  `vrt`: the ranks are virtual (groups of one launch on one
    // device sharing the caller's outputs; only rank 0 writes them).
    int nrk;
    int rk;
    int vrt;
    const int64_t* delta;
};

struct CwyArgs {
    int64_t n;
    int64_t ldv;
    const double* d;
    const double* e;
    double tnorm;
    uint64_t seed;
    const double* wt;
    const int* cstart;
    const double* fl;
    const int8_t* fp;
    const double* fr;
    const double* fb;
    const double* fc;
    const double* unn;
    const double* F;    // per-vector packed factors [j][i][4] (clustered vectors)
    const int8_t* FP;   // per-vector pivot bits [j][i]
    const double* X1c;  // x^(1) of clustered vectors, [j][i], vector stride roundup(n, 2)
    double* Z;
    int64_t ldz;
    int* iters;
    PrepOut* out;
    // schedule
    int ngroups;
    const int* g_cta0;       // first CTA of each group
    const int* g_size;       // CTAs per group
    const int* g_coff;       // offsets into g_clist
    const int* g_clist;      // cluster ids per group
    GroupWS* ws;             // per group
    long long* syncs;        // per group: barrier episodes (stats)
    unsigned long long* prof;  // optional per-group phase times [g*16 + phase] (ns), or NULL
    int64_t vcap;            // largest vector staged in shared memory (max mcap over groups)
    int nstg;                // TMA ring stages for narrow clusters (0 = ring not allocated)
    int prof_p0, prof_p1;    // phase timers count only vectors with prof_p0 <= j_c < prof_p1
    int piece_cost;          // partition cost of one wide row piece, in elements (cwy.cu part_*)
    int cta0_pm;             // per-mille cut of CTA 0's share of pass D's rows (wide clusters; cwy.cu share_bound)
    int prof_sel;            // debug: CTA whose thread 32 runs the pass timers (default: the first group's first)
    int a2;                  // fuse iteration 2's pass A behind the back sweep (TINV_A2, default 1)
    int band_ch;             // sweep chunks (256 rows) per published band (TINV_BANDCH)
    int labq;                // in-block look-ahead dots fused into the earlier vectors' BC passes (TINV_LABQ, default 1)
    int tyr;                 // keep T_p yrow across the iterations of vector p (TINV_TYR, default 1)
    int a2c;                 // fused pass A2 in the column-owner form (TINV_A2C, default 1)
    int sweep2;              // window back sweep on two threads of CTA 0: chain + TMA/store helper (TINV_SWEEP2, default 1)
    int poll_ns;             // back-off of the band polls in ns (TINV_POLLNS)
    int dbg;                 // debug build experiments (TINV_DBG bits)
    int reorth;              // 0 reduced compact WY (§3.3.2), 1 classical MGS (Alg. 1), 2 ordinary compact WY (§3.3.1)
    int lab;                 // blocked look-ahead block size b (2..8; 0/1 = off), wide clusters of single-rank groups
    int pf;                  // rows whose first pieces of the next wide pass are prefetched into L2 before a barrier (TINV_PF; 0 = off)
    unsigned long long* prof_cta;   // debug: per-CTA busy time before each phase's barrier [cta*16 + phase], or NULL
    // deferred final pass D: NULL = off.  dzc[j] = c of vector j when its last
    // pass D was deferred (0 otherwise; zeroed by the host per call); its x' is stored in
    // dzx + j * roundup(n, 2) (= X1c, the vector's dead first iterate)
    double* dzc;
    double* dzx;
};

// Deferred final pass D (dz.cu): for the parked vectors p0 <= p < m of one cluster,
// q_p = Y_{p+1} x'_p - e_p (one GEMM), the stopping test, the sign rule and z_j.
struct DzArgs {
    int64_t n;
    int64_t m;          // cluster size
    int64_t p0;         // first column that may be parked (kNarrowM)
    const double* Y;    // the group's packed Y (y_row_off(i, m) rows)
    const double* X;    // x' of column p at X + p * n2v (p + 1 entries)
    int64_t n2v;
    const double* c;    // dzc + j1: c of column p, 0 = not parked
    double* Z;          // Z + j1 * ldz: column p at Z + p * ldz
    int64_t ldz;
    double* part;       // partials [row tile][3][m - p0]
    PrepOut* out;       // dzfail (deferred test failed), counted per column
};
cudaError_t launch_dz(const DzArgs& a, cudaStream_t s);

// Resident compact-WY kernel for narrow clusters (cwy_resident.cu): one thread-block cluster
// of CS CTAs per eigen-cluster, Y kept in distributed shared memory.
struct ResArgs {
    int64_t n;
    int RL;                 // rows per CTA (even)
    int M2;                 // Y / T row stride (>= every cluster's roundup(m, 2))
    double tnorm;
    uint64_t seed;
    const int* cstart;
    const int* u_off;       // per unit: offsets into u_list
    const int* u_list;      // cluster ids
    const double* X1c;      // x^(1), [j][i], vector stride roundup(n, 2)
    const double* F;        // packed factors [j][i][4]
    const int8_t* FP;       // pivot bytes [j][i]
    const double* unn;
    double* Z;
    int64_t ldz;
    int* iters;
    PrepOut* out;
    unsigned long long* prof;   // optional 16 phase timers of unit 0 (ns), or NULL
    int handover;           // clusters with m <= handover: the batched LU stopped the leader after
                            // x^(1), iterate it here (0: none)
    int flags;              // experiments: bit 0 disables the look-ahead pass
    int mgs;                // 1: classical MGS reorthogonalisation (Alg. 1) instead of compact WY
    int ordinary;           // 1: the ordinary compact-WY sequence of §3.3.1 (separate Y^T y pass)
};
size_t resident_smem_bytes(int64_t n, int RL, int M2, int cs);
cudaError_t launch_resident(const ResArgs& a, int cs, int nunits, size_t smem, cudaStream_t s);
int resident_max_clusters(int cs, size_t smem);

void launch_prep(const PrepArgs& a, cudaStream_t s);
void launch_bisect(int64_t n, const double* d, const double* e, double* w, double* bnd, cudaStream_t s);
void launch_batched(const BatchedArgs& a, cudaStream_t s, int nsm);
int64_t batched_slot_cap(int64_t n);
void launch_finalize(const FinalizeArgs& a, cudaStream_t s);
void launch_pack(const PackArgs& a, cudaStream_t s);
void launch_identity(double* Z, int64_t n, int64_t ldz, cudaStream_t s);
void launch_peer_read(const double* base, const int64_t* delta, int nrk, uint64_t* out, cudaStream_t s);
cudaError_t launch_cwy(const CwyArgs& a, int nctas, size_t smem, cudaStream_t s);
int cwy_threads();
size_t cwy_smem_bytes(int64_t vcap, int nstg);
int cwy_narrow_max();
int cwy_ring_stages();
int cwy_max_ctas_per_sm(size_t smem);

}  // namespace tinv
