// cwy.cu -- persistent compact-WY reorthogonalisation kernel.
//
// One cooperative launch, one CTA per SM.  CTAs are partitioned into groups; each group
// owns a list of Peters-Wilkinson clusters (m >= 2) and processes their vectors
// j_c = 1..m-1 in order (Alg. 4).  Inside a group the work of one
// iteration is split by rows / columns across its G CTAs with group barriers between
// dependent phases.  Per iteration of vector p = j_c (0-based), with Y_p = [L; Yhat]
// packed row-major (zero-free, Fig. 1) and T_p held twice (column-packed and row-major):
//
//   A   g   = Y_p^T x                 column-accumulate, partials per CTA
//   R1  g   = sum of partials         deterministic, fixed CTA order
//   TT  g'  = T_p^T g                 row dots on column-packed T
//   BC  u^  = x^ - Yhat g'            row dots (own rows) fused in the same phase with
//       s'  = Yhat^T u^ (partials)    a column-accumulate over those rows
//       ||u^||^2 partials
//   R2  c = -sgn(u_0)||u^||, t = 1/(c^2 - u_0 c), y_0 = u_0 - c
//       s = s' - c Y[p,:]  (= Yhat^T yhat, the §3.3.2 reduction of Y_{j-1}^T y_j)
//   TN  [Ts, h] = T_p [s, Y[p,:]]     row dots on row-major T
//       that = -t Ts -> column p of T; x'_{<p} = h + y_0 that, x'_p = t y_0
//       (= T_{p+1} Y_{p+1}^T e_p with T, not T^T: erratum of PAPER.md:424/616)
//       yhat -> column p of Y (rollback: a repeated iteration overwrites it)
//   D   q = Y_{p+1} x' - e_p          row dots (the sign-flipped q of PAPER.md:583)
//   TEST ||c q||_inf >= sqrt(0.1/n) counts a pass; 2 passes accept (reading 9); else
//       one CTA runs the chained LU solve with rhs q (stored factors) -> next x.
// The first reflector of a cluster is built from the accepted z_{j1}.
#include "common.cuh"
#include "tinv_internal.h"

namespace tinv {

// Debug timers of the wide kernel (per-CTA busy times, vector windows; TINV_PROF_CTA,
// TINV_PROF_P0/P1): compiled in only with -DTINV_WIDE_DEBUG (`make EXTRA=-DTINV_WIDE_DEBUG`),
// since even their untaken branches cost ~3% on cfg3's short phases.
#ifdef TINV_WIDE_DEBUG
constexpr bool kWideDebug = true;
#else
constexpr bool kWideDebug = false;
#endif
constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int CFCH = 2048;   // rows whose coefficients are staged in shared memory at once
constexpr int CH = 256;                              // back-sweep ring chunk (rows)
constexpr int kRing = 4;                             // back-sweep ring depth
constexpr int64_t kSolveDoubles = kRing * 5 * CH;    // back-sweep ring slots (4 CH factor doubles + CH t)
constexpr int kVsD = 128;                            // staged vector of the short (P <= 65) passes
constexpr int kNBar = 32;                            // mbarrier slots (incl. 2 use counters), 16-B multiple
constexpr int kXFull = 27, kXEmpty = 29;             // two-thread back sweep: x staging handover (2 + 2)

// Global accesses: data produced inside this kernel by other CTAs goes through L2 (.cg,
// never a stale L1 line); explicit global-space intrinsics also let the compiler hoist
// shared-memory loads across the stores (no generic-pointer aliasing).
__device__ __forceinline__ double ld(const double* p) { return __ldcg(p); }
__device__ __forceinline__ double2 ld2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void st(double* p, double v) { __stcg(p, v); }
__device__ __forceinline__ double ldro(const double* p) { return __ldg(p); }
// bulk L2 prefetch (TMA engine; no registers held): 16-byte aligned, size multiple of 16
__device__ __forceinline__ void l2_prefetch(const double* p, int64_t ndoubles) {
    if (ndoubles <= 0) return;
    uint32_t bytes = (uint32_t)(((ndoubles * 8) + 15) & ~int64_t(15));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
constexpr int64_t kPfDist = 2048;   // doubles prefetched ahead inside a row (16 KB)
constexpr double kL2KeepBytes = 48e6;   // Y_p beyond this: single-use streams are evict_first

struct SSlots {  // scalar partial slots per CTA (ws.S[r*SST + slot])
    enum { U2 = 0, X2 = 1, Q2 = 2, QINF = 3, QARG = 4, GPN = 5, X2N = 6, Q1 = 7, FA = 8, FB = 9, MG0 = 10, MG1 = 11 };
};
constexpr int SST = 16;   // scalar slots per CTA

__device__ __forceinline__ int pow2ceil(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// smallest i in [lo, hi] with cum(i) >= target (cum non-decreasing)
template <class F>
__device__ __forceinline__ int64_t bsearch_cum(int64_t lo, int64_t hi, int64_t target, F cum) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (cum(mid) >= target) hi = mid; else lo = mid + 1;
    }
    return lo;
}
// Static partitions of the passes over the group's CTAs.  A wide pass (P > kNarrowM) costs
// a CTA its elements plus a fixed consumer cost per row piece (one TMA copy and one warp's
// dot / accumulate per piece of <= kPieceW columns), measured at several thousand elements
// (CwyArgs::piece_cost): the rows of the triangles (short rows, one or two pieces each) are
// weighted accordingly, or the CTA holding them sets the phase time.
constexpr int kPieceW = 2 * (NW - 1) * 32;   // = PW below
// sum_{i < l} floor(i / kPieceW)
__device__ __forceinline__ int64_t sum_floor_pw(int64_t l) {
    const int64_t q = (int64_t)((uint32_t)l / (uint32_t)kPieceW), rem = l - q * kPieceW;   // l < 2^31
    return (int64_t)kPieceW * q * (q - 1) / 2 + rem * q;
}
// Boundary q of G shares of the weight W when the group's first CTA takes (1000 - h0) / 1000 of a
// share (CwyArgs::cta0_pm).  Measured: in pass D CTA 0 -- the short rows of the leading triangle
// -- is 10-19% slower than the median CTA under the element + piece cost model; cutting its share
// by 12% takes 9% off D on cfg5 and 6% on cfg4 (more brings nothing: the next CTAs bound the
// pass), and does nothing for TT / TN, whose slowest CTAs are elsewhere.
__device__ __forceinline__ int64_t share_bound(int64_t W, int q, int G, int h0) {
    if (h0 == 0 || q == 0) return (W * q) / G;
    return (W * ((int64_t)q * 1000 - h0)) / ((int64_t)G * 1000 - h0);
}
// rows of A / D: row i has min(i+1, P) elements in min(floor(i / kPieceW) + 1, nblk) pieces
__device__ __forceinline__ void part_rows_weighted(int64_t n, int64_t P, int r, int G, int64_t& a, int64_t& b,
                                                   int64_t C, int h0 = 0) {
    if (P <= kNarrowM) C = 0;
    const int64_t NB = (P + kPieceW - 1) / kPieceW;
    const int64_t base = P * (P + 1) / 2 + C * ((NB > 1 ? sum_floor_pw(P) : 0) + P);
    auto cum = [P, C, NB, base](int64_t i) -> int64_t {
        if (i <= P) return i * (i + 1) / 2 + C * ((NB > 1 ? sum_floor_pw(i) : 0) + i);   // one block: 1 piece per row
        return base + (i - P) * (P + C * NB);
    };
    int64_t W = cum(n);
    a = (r == 0) ? 0 : bsearch_cum(0, n, share_bound(W, r, G, h0), cum);
    b = (r == G - 1) ? n : bsearch_cum(0, n, share_bound(W, r + 1, G, h0), cum);
}
// rows [b0, b1) of Y_P split over G CTAs by the same weights (rows of one band of the sweep)
__device__ __forceinline__ void part_band_weighted(int64_t b0, int64_t b1, int64_t P, int r, int G, int64_t& a,
                                                   int64_t& b, int64_t C) {
    if (P <= kNarrowM) C = 0;
    const int64_t NB = (P + kPieceW - 1) / kPieceW;
    const int64_t base = P * (P + 1) / 2 + C * ((NB > 1 ? sum_floor_pw(P) : 0) + P);
    auto cum = [P, C, NB, base](int64_t i) -> int64_t {
        if (i <= P) return i * (i + 1) / 2 + C * ((NB > 1 ? sum_floor_pw(i) : 0) + i);
        return base + (i - P) * (P + C * NB);
    };
    const int64_t w0 = cum(b0), W = cum(b1) - w0;
    a = (r == 0) ? b0 : bsearch_cum(b0, b1, w0 + (W * r) / G, cum);
    b = (r == G - 1) ? b1 : bsearch_cum(b0, b1, w0 + (W * (r + 1)) / G, cum);
}
__device__ __forceinline__ void part_uniform(int64_t lo, int64_t hi, int r, int G, int64_t& a, int64_t& b) {
    int64_t len = hi - lo;
    a = lo + (len * r) / G;
    b = lo + (len * (r + 1)) / G;
}
// k in [0,p): packed column k of T has k+1 elements in floor(k / kPieceW) + 1 pieces
__device__ __forceinline__ void part_tt(int64_t p, int r, int G, int64_t& a, int64_t& b, int64_t C, int h0 = 0) {
    if (p <= kNarrowM) C = 0;
    const bool multi = p > kPieceW;
    auto cum = [C, multi](int64_t k) -> int64_t { return k * (k + 1) / 2 + C * ((multi ? sum_floor_pw(k) : 0) + k); };
    int64_t W = cum(p);
    a = (r == 0) ? 0 : bsearch_cum(0, p, share_bound(W, r, G, h0), cum);
    b = (r == G - 1) ? p : bsearch_cum(0, p, share_bound(W, r + 1, G, h0), cum);
}
// l in [0,p): row l of T has p-l elements in nblk - floor(l / kPieceW) pieces
__device__ __forceinline__ void part_tn(int64_t p, int r, int G, int64_t& a, int64_t& b, int64_t C, int h0 = 0) {
    if (p <= kNarrowM) C = 0;
    const int64_t NB = (p + kPieceW - 1) / kPieceW;
    auto cum = [p, C, NB](int64_t l) -> int64_t {
        return l * p - l * (l - 1) / 2 + C * (l * NB - (NB > 1 ? sum_floor_pw(l) : 0));
    };
    int64_t W = cum(p);
    a = (r == 0) ? 0 : bsearch_cum(0, p, share_bound(W, r, G, h0), cum);
    b = (r == G - 1) ? p : bsearch_cum(0, p, share_bound(W, r + 1, G, h0), cum);
}

// dynamic shared memory carve-up
struct Smem {
    double* vs;      // staged vector of the short passes (kVsD doubles; the A2C block table)
    double* cf;      // CFCH coefficients
    double* racc;    // 2 RCH row accumulators of wide row dots
    double* vblk;    // 2 x 2 PW: column blocks of the wide row-dot vectors (double buffer)
    uint64_t* vbar;  // 2 mbarriers of the vector double buffer
    uint32_t* vuse;  // 2 use counters (shared)
    double* bring;   // back-sweep ring (kSolveDoubles), aliases the pass ring
    double2* acc;    // NT
    double* red;     // NW + 8
    uint64_t* mbar;  // kRing mbarriers (back-sweep ring)
    double* rbuf;    // partial-sum staging of reduce_partials (aliases the pass rings)
    uint64_t* rbar;  // its mbarrier
    uint32_t* rcnt;  // its use counter (phase parity)
};

// copy len doubles of a global vector into sm.vs (zero padded by 2), then barrier
__device__ __forceinline__ void stage_vec(const Smem& sm, const double* src, int64_t len) {
    for (int64_t k = threadIdx.x; k < len + 2; k += NT) sm.vs[k] = (k < len) ? ld(src + k) : 0.0;
    __syncthreads();
}

// ---------------------------------------------------------------- row dots
// For rows i in [i0,i1): dot_i = sum_{k < len(i)} R(i)[k] * vs[k] (len(i) <= P, R(i) 16-byte
// aligned, vs staged in shared memory); epi(i, dot) runs on one lane per row.  Short rows
// (P <= 64) pack several rows per warp and batch 4 rows of loads; long rows batch 8 loads
// per lane.
template <class RowPtr, class RowLen, class Epi>
__device__ __forceinline__ void rowdots(int64_t i0, int64_t i1, int64_t P, const double* vs, RowPtr rowptr,
                                        RowLen rowlen, Epi epi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (P <= 0) {
        for (int64_t i = i0 + threadIdx.x; i < i1; i += NT) epi(i, 0.0);
        return;
    }
    if (P <= 64) {
        const int LPR = pow2ceil((int)((P + 1) / 2));
        const int RPW = 32 / LPR;
        const int sub = lane / LPR, sl = lane % LPR;
        const int64_t k = 2 * sl;
        const double vx = (k < P) ? vs[k] : 0.0, vy = (k + 1 < P) ? vs[k + 1] : 0.0;
        constexpr int U = 4;
        for (int64_t ib = i0 + (int64_t)warp * RPW * U; ib < i1; ib += (int64_t)NW * RPW * U) {
            double2 a[U];
            int64_t ke[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t i = ib + u * RPW + sub;
                ke[u] = (i < i1) ? rowlen(i) : 0;
                a[u] = (k < ke[u]) ? ld2(rowptr(i) + k) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t i = ib + u * RPW + sub;
                double acc = fma(a[u].x, vx, 0.0);
                acc = fma((k + 1 < ke[u]) ? a[u].y : 0.0, vy, acc);
                for (int o = LPR >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (sl == 0 && i < i1) epi(i, acc);
            }
        }
        return;
    }
    constexpr int U = 8;
    if (lane == 0 && i0 + warp < i1) {   // prime: head of the warp's first row
        const int64_t ke0 = rowlen(i0 + warp);
        l2_prefetch(rowptr(i0 + warp), ke0 < kPfDist ? ke0 : kPfDist);
    }
    for (int64_t i = i0 + warp; i < i1; i += NW) {
        const double* row = rowptr(i);
        const int64_t ke = rowlen(i);
        if (lane == 0 && i + NW < i1) {   // head of the warp's next row
            const int64_t kn = rowlen(i + NW);
            l2_prefetch(rowptr(i + NW), kn < kPfDist ? kn : kPfDist);
        }
        double acc = 0.0;
        for (int64_t k0 = 2 * lane; k0 < ke; k0 += 64 * U) {
            if (lane == 0) {   // stay kPfDist doubles ahead inside the row
                const int64_t kp = k0 + kPfDist;
                if (kp < ke) l2_prefetch(row + kp, (ke - kp) < 64 * U ? (ke - kp) : 64 * U);
            }
            double2 a[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t k = k0 + 64 * u;
                a[u] = (k < ke) ? ld2(row + k) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t k = k0 + 64 * u;
                if (k < ke) {
                    const double2 b = *reinterpret_cast<const double2*>(vs + k);
                    acc = fma(a[u].x, b.x, acc);
                    if (k + 1 < ke) acc = fma(a[u].y, b.y, acc);
                }
            }
        }
        acc = warp_sum(acc);
        if (lane == 0) epi(i, acc);
    }
}

// ---------------------------------------------------------------- column accumulate
// out[k] = sum_{i in [i0,i1), i >= k} Y[i][k] * coef(i)  for k < P, coef(i) = cp[i*cs].
// Thread t owns a column pair (2 doubles, 16-byte loads) and a subset of the rows; the
// coefficients of a row chunk are staged in shared memory.  Returns sum coef(i)^2.
__device__ double colacc(const Smem& sm, const double* __restrict__ Y, int64_t m, int64_t i0, int64_t i1,
                         int64_t P, const double* cp, int64_t cs, double* out, int64_t ovr = -1, double ovv = 0.0) {
    const int tid = threadIdx.x;
    const int CPT = (P > 0) ? min(NT, pow2ceil((int)((P + 1) / 2))) : NT;
    const int RS = NT / CPT;
    const int cpi = tid % CPT, rs = tid / CPT;
    double c2 = 0.0;
    constexpr int U = 8;
    if (i1 <= i0) {   // no rows: this CTA's partial is zero (it is still summed by R1/R2)
        for (int64_t k = tid; k < P; k += NT) st(out + k, 0.0);
        return 0.0;
    }
    for (int64_t rc0 = i0; rc0 < i1; rc0 += CFCH) {
        const int64_t rc1 = (i1 - rc0 > CFCH) ? rc0 + CFCH : i1;
        for (int64_t i = rc0 + tid; i < rc1; i += NT) {
            const double c = (i == ovr) ? ovv : ld(cp + i * cs);   // ovr: coefficient of one row replaced
            sm.cf[i - rc0] = c;
            c2 = fma(c, c, c2);
        }
        __syncthreads();
        for (int64_t k0 = 0; k0 < P; k0 += 2 * CPT) {
            const int64_t k = k0 + 2 * cpi;
            double a0 = 0.0, a1 = 0.0;
            if (k < P) {
                const bool two = (k + 1 < P);
                const int64_t ia = (rc0 > k) ? rc0 : k;
                for (int64_t i = ia + rs; i < rc1; i += (int64_t)RS * U) {
                    double2 v[U];
                    double c[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int64_t ii = i + (int64_t)u * RS;
                        const bool ok = ii < rc1;
                        v[u] = ok ? ld2(Y + y_row_off(ii, m) + k) : make_double2(0.0, 0.0);
                        c[u] = ok ? sm.cf[ii - rc0] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int64_t ii = i + (int64_t)u * RS;
                        a0 = fma(v[u].x, c[u], a0);
                        a1 = fma((two && k + 1 <= ii) ? v[u].y : 0.0, c[u], a1);
                    }
                }
            }
            if (RS > 1) {
                sm.acc[tid] = make_double2(a0, a1);
                __syncthreads();
                if (rs == 0)
                    for (int r2 = 1; r2 < RS; r2++) {
                        const double2 t = sm.acc[cpi + r2 * CPT];
                        a0 += t.x;
                        a1 += t.y;
                    }
                __syncthreads();
            }
            if (rs == 0 && k < P) {
                if (rc0 == i0) {
                    st(out + k, a0);
                    if (k + 1 < P) st(out + k + 1, a1);
                } else {
                    st(out + k, ld(out + k) + a0);
                    if (k + 1 < P) st(out + k + 1, ld(out + k + 1) + a1);
                }
            }
        }
        __syncthreads();
    }
    return c2;
}


// ---------------------------------------------------------------- deterministic reductions
// sum over t < G of S[t*8 + slot] (fixed thread mapping + fixed tree)
__device__ __forceinline__ double reduce_slot(const Smem& sm, const double* S, int G, int slot) {
    double v = 0.0;
    for (int t = threadIdx.x; t < G; t += NT) v += ld(S + t * SST + slot);
    return block_sum<NT>(v, sm.red);
}
// max over t < G of S[t*8 + QINF] with the lowest S[t*8 + QARG] on ties
__device__ __forceinline__ void reduce_argmax(const Smem& sm, const double* S, int G, double& vmax, int64_t& arg) {
    double v = -1.0;
    int64_t ia = 0x7fffffffffffffffLL;
    for (int t = threadIdx.x; t < G; t += NT) {
        const double x = ld(S + t * SST + 3);
        const int64_t a = (int64_t)ld(S + t * SST + 4);
        if (x > v || (x == v && a < ia)) { v = x; ia = a; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const long long oa = __shfl_xor_sync(0xffffffffu, (long long)ia, o);
        if (ov > v || (ov == v && oa < ia)) { v = ov; ia = oa; }
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sm.acc[threadIdx.x >> 5] = make_double2(v, (double)ia);
    __syncthreads();
    v = -1.0;
    ia = 0x7fffffffffffffffLL;
    for (int w = 0; w < NW; w++) {
        const double2 t = sm.acc[w];
        if (t.x > v || (t.x == v && (int64_t)t.y < ia)) { v = t.x; ia = (int64_t)t.y; }
    }
    __syncthreads();
    vmax = v;
    arg = ia;
}
// out[k] = sum_{t<G} P[t*mc + k] for k in [k0, k1): threads split (k, t-group); the
// t-groups are combined in a fixed order (deterministic).
// Slot t of a rank-split group lives in the replica of rank t / Gl (delta in doubles).
struct Ranks {
    int nrk, Gl;
    const int64_t* delta;
    __device__ __forceinline__ int64_t off(int t) const { return nrk == 1 ? 0 : __ldg(delta + t / Gl); }
};
constexpr int64_t kRBufD = 21952;   // doubles of Smem::rbuf (= the wide ring, static_assert below)
template <class Post>
__device__ __forceinline__ void reduce_partials(const Smem& sm, const double* P, int64_t mc, int G, int64_t k0,
                                                int64_t k1, Post post, const Ranks& rks = Ranks{1, 1, nullptr},
                                                uint64_t* dt = nullptr) {
    const int tid = threadIdx.x;
    // Single-rank groups: the G partial slices [k0, k1) come into shared memory by TMA bulk
    // copies (one per partial, all in flight on one mbarrier), then every column is summed in
    // the fixed order t = tg, tg + TG, ... and the TG groups in order (deterministic).  Plain
    // global loads of the same slices measured ~10 us per reduction inside the kernel.
    const int64_t ka = k0 & ~int64_t(1), kw = (k1 - ka + 1) & ~int64_t(1);
    if (rks.nrk == 1 && k1 > k0 && (int64_t)G * kw <= kRBufD && G <= NT && (mc & 1) == 0) {
        const uint32_t use = *sm.rcnt;
        if (tid < G) {
            fence_proxy_async_global();   // partials stored by other CTAs (generic proxy) -> bulk copy
            const uint32_t bytes = (uint32_t)(kw * 8);
            mbar_add_tx(sm.rbar, bytes);
            bulk_g2s(sm.rbuf + (int64_t)tid * kw, P + (int64_t)tid * mc + ka, bytes, sm.rbar);
        }
        __syncthreads();
        if (tid == 0) mbar_arrive(sm.rbar);
        mbar_wait(sm.rbar, use & 1u);
        const int64_t off = k0 - ka;
        for (int64_t kb = k0; kb < k1; kb += NT) {
            const int64_t K = (k1 - kb < NT) ? (k1 - kb) : NT;
            const int KP = (int)((K + 31) & ~int64_t(31));
            const int TG = NT / KP;
            const int kk = tid % KP, tg = tid / KP;
            double acc = 0.0;
            if (tg < TG && kk < K) {
                const double* col = sm.rbuf + off + (kb - k0) + kk;
                for (int t = tg; t < G; t += TG) acc += col[(int64_t)t * kw];
            }
            if (TG > 1) {
                __syncthreads();
                sm.cf[tid] = acc;
                __syncthreads();
                if (tg == 0 && kk < K)
                    for (int u = 1; u < TG; u++) acc += sm.cf[kk + u * KP];
            }
            if (tg == 0 && kk < K) post(kb + kk, acc);
        }
        __syncthreads();   // rbuf (the pass ring) and cf free again
        if (tid == 0) *sm.rcnt = use + 1;
        __syncthreads();
        return;
    }
    for (int64_t kb = k0; kb < k1; kb += NT) {
        const uint64_t c0 = dt ? (uint64_t)clock64() : 0;
        const int64_t K = (k1 - kb < NT) ? (k1 - kb) : NT;
        const int KP = (int)((K + 31) & ~int64_t(31));
        const int TG = NT / KP;
        const int kk = tid % KP, tg = tid / KP;
        double acc = 0.0;
        if (tg < TG && kk < K) {
            const double* col = P + kb + kk;
            auto at = [&](int u) { return col + (int64_t)u * mc + rks.off(u); };
            // up to 16 independent loads in flight per thread (one L2 round trip per batch
            // instead of one per 4 partials), added in the fixed order t = tg, tg + TG, ...
            constexpr int RB = 16;
            for (int t0 = tg; t0 < G; t0 += RB * TG) {
                double v[RB];
#pragma unroll
                for (int u = 0; u < RB; u++) {
                    const int t = t0 + u * TG;
                    v[u] = (t < G) ? ld(at(t)) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < RB; u++)
                    if (t0 + u * TG < G) acc += v[u];
            }
        }
        if (dt) {
            asm volatile("" ::"d"(acc));
            const uint64_t c1 = (uint64_t)clock64();
            dt[0] += c1 - c0;
        }
        if (TG > 1) {
            __syncthreads();
            sm.cf[tid] = acc;
            __syncthreads();
            if (tg == 0 && kk < K)
                for (int u = 1; u < TG; u++) acc += sm.cf[kk + u * KP];
            __syncthreads();
        }
        if (tg == 0 && kk < K) post(kb + kk, acc);
    }
}

// ---------------------------------------------------------------- chained single-vector solve
// x = (T - wt_j I)^{-1} (sigma * rhs), sigma = n ||T||_1 max(eps,|u_nn|) / ||rhs||_1, with the
// factors stored by the batched kernel (Eq. (1); rhs = q, Alg. 4 l.16
// PAPER.md:708, or the start vector of restart `restart`).  Runs on one CTA:
//   forward  c_{i+1} = sw ? c_i - l_i b_{i+1} : b_{i+1} - l_i c_i  is first order with
//            |l_i| <= 1 (partial pivoting), so it is partitioned: one chunk of rows per
//            thread reduces to c_out = A c_in + B, a block scan of these maps gives every
//            chunk its exact incoming carry, and each chunk reruns its rows serially
//            (y_i -> t_i = s y_i / u0_i);
//   back     x_i = t_i - b_i x_{i+1} - c_i x_{i+2} stays strictly serial: its homogeneous
//            solutions grow by up to 1/eps at the near-singular pivot (that growth is the
//            inverse iteration), so any composition of row maps cancels catastrophically
//            (measured: relative errors 1e-2 .. overflow on the glued-Wilkinson config with
//            2-row blocks).  Lane 0 of warp 0 runs it out of shared memory (one dependent FMA
//            per row) while warps 1..NW-1 stage the next chunk of (t_i, b_i, c_i).
struct Aff1 {
    double a, b;   // c -> a c + b
};
__device__ __forceinline__ Aff1 comp(const Aff1& f, const Aff1& g) {   // f o g
    return Aff1{f.a * g.a, fma(f.a, g.b, f.b)};
}
__device__ __forceinline__ Aff1 shfl_up(const Aff1& f, int o) {
    return Aff1{__shfl_up_sync(0xffffffffu, f.a, o), __shfl_up_sync(0xffffffffu, f.b, o)};
}
__device__ __forceinline__ Aff1 ident(Aff1) { return Aff1{1.0, 0.0}; }

// Exclusive scan of per-thread maps in the order u = 0..NT-1 (later o earlier); returns the
// thread's exclusive prefix, `total` = composition of all NT maps.  `buf` holds NW maps.
template <class M>
__device__ __forceinline__ M block_scan_excl(M f, M* buf, M& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    M inc = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const M g = shfl_up(inc, o);
        if (lane >= o) inc = comp(inc, g);
    }
    M ex = shfl_up(inc, 1);
    if (lane == 0) ex = ident(f);
    __syncthreads();
    if (lane == 31) buf[w] = inc;
    __syncthreads();
    M pre = ident(f);
    for (int k = 0; k < w; k++) pre = comp(buf[k], pre);
    total = pre;
    for (int k = w; k < NW; k++) total = comp(buf[k], total);
    __syncthreads();
    return comp(ex, pre);
}



// Serial back substitution x_i = t_i - b_i x_{i+1} - c_i x_{i+2} (rows n-1 .. 0, x_n = x_{n+1}
// = 0) by one thread.  Its inputs stream through a kRing-deep shared-memory ring filled by TMA
// bulk copies: per chunk of CH rows the factor records F[i][0..3] (32 B/row) and t_i.  The
// same thread issues the copies and consumes them (one mbarrier per slot), so the chain only
// waits for data that was requested kRing chunks earlier.
// Band progress of the sweep (fused pass A2 behind it): rows are final bottom-up; after every
// kBandCh chunks the sweep publishes "bands 0..b done" as prog = tag + b + 1 (release), so
// the other CTAs can stream those rows while the sweep goes on.
__host__ __device__ __forceinline__ int sweep_bands(int64_t n, int bch) {
    const int64_t C = (n + 256 - 1) / 256;
    return (int)((C + bch - 1) / bch);
}
__device__ __forceinline__ void publish(unsigned int* prog, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(prog), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int acquire(const unsigned int* prog) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(prog) : "memory");
    return v;
}

__device__ void back_sweep(const CwyArgs& a, const GroupWS& ws, int64_t j, const Smem& sm, uint32_t& mbph,
                           unsigned int* prog = nullptr, unsigned int tag = 0, uint64_t* dt = nullptr) {
    // dt (debug build, TINV_DBG bit 3): SM clocks in [0] ring waits, [1] the chains, [2] the rest, [3] total
    const uint64_t d0 = dt ? (uint64_t)clock64() : 0;
    const int64_t n = a.n;
    const double* __restrict__ F = a.F + j * n * 4;
    const double* __restrict__ ts = ws.ysol;
    double* __restrict__ x = ws.x;
    double* ring = sm.bring;                                 // kRing x (4 CH + CH) doubles
    const int64_t C = (n + CH - 1) / CH;
    fence_proxy_async_global();
    auto issue = [&](int64_t k) {
        const int slot = (int)(k % kRing);
        const int64_t c = C - 1 - k;
        const int64_t lo = c * CH, hi = (lo + CH < n) ? lo + CH : n;
        const uint32_t fb = (uint32_t)((hi - lo) * 32), tb = (uint32_t)(((hi - lo + 1) & ~int64_t(1)) * 8);
        double* dst = ring + (int64_t)slot * 5 * CH;
        mbar_expect_tx(sm.mbar + slot, fb + tb);
        bulk_g2s(dst, F + lo * 4, fb, sm.mbar + slot);
        bulk_g2s(dst + 4 * CH, ts + lo, tb, sm.mbar + slot);
    };
    for (int64_t k = 0; k < C && k < kRing; k++) issue(k);
    double x1 = 0.0, x2 = 0.0;
    // x leaves through a double-buffered shared staging area and one bulk store per chunk
    // (per-row global stores on the chain cost ~16 us per 8000 rows)
    // (the wide row dots' accumulators: no wide pass runs on this CTA during the sweep)
    double* xbuf = sm.racc;   // 2 CH doubles
    for (int64_t k = 0; k < C; k++) {
        const int slot = (int)(k % kRing);
        double* xb = xbuf + (k & 1) * CH;
        const uint64_t e0 = dt ? (uint64_t)clock64() : 0;
        bulk_wait_read<1>();   // the store of chunk k-2 has read this buffer
        mbar_wait(sm.mbar + slot, (mbph >> slot) & 1u);
        mbph ^= 1u << slot;
        const uint64_t e1 = dt ? (uint64_t)clock64() : 0;
        const double* Fs = ring + (int64_t)slot * 5 * CH;
        const double* Ts = Fs + 4 * CH;
        const int64_t c = C - 1 - k;
        const int64_t lo = c * CH, hi = (lo + CH < n) ? lo + CH : n;
        const int cnt = (int)(hi - lo);
        // top remainder (only in the first chunk): scalar rows
        const int top = cnt & ~15;
        for (int u = cnt - 1; u >= top; u--) {
            const double2 bc = *reinterpret_cast<const double2*>(Fs + u * 4 + 2);
            const double xi = fma(-bc.x, x1, fma(-bc.y, x2, Ts[u]));
            xb[u] = xi;
            x2 = x1;
            x1 = xi;
        }
        // 16-row batches: the batch's loads first (independent), then the dependent chain
        // (~15 cycles/row in the kernels; the 8-row form with the next batch's loads in
        // flight measured ~19-23; tools/micro/sweep_var.cu)
        for (int u0 = top - 16; u0 >= 0; u0 -= 16) {
            double b[16], c[16], t[16], xv[16];
#pragma unroll
            for (int u = 0; u < 16; u++) {
                const double2 bc = *reinterpret_cast<const double2*>(Fs + (u0 + u) * 4 + 2);
                b[u] = bc.x; c[u] = bc.y; t[u] = Ts[u0 + u];
            }
#pragma unroll
            for (int u = 15; u >= 0; u--) {
                xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u]));
                x2 = x1;
                x1 = xv[u];
            }
#pragma unroll
            for (int u = 0; u < 16; u += 2)
                *reinterpret_cast<double2*>(xb + u0 + u) = make_double2(xv[u], xv[u + 1]);
        }
        if (cnt & 1) xb[cnt] = 0.0;   // x[n] (padding of the last, odd chunk)
        if (dt) {
            const uint64_t e2 = (uint64_t)clock64();
            dt[0] += e1 - e0;
            dt[1] += e2 - e1;
            dt[2] -= e2;   // + the chunk's end below
        }
        fence_proxy_async_smem();     // generic smem writes -> the bulk store
        bulk_s2g(x + lo, xb, (uint32_t)((cnt + 1) & ~1) * 8u);
        bulk_commit();
        if (k + kRing < C) issue(k + kRing);
        // band b = chunks [b kBandCh, (b+1) kBandCh) complete: its bulk stores are performed once
        // at most the newest group (this chunk's) is pending -- published one chunk late, so
        // the wait never stalls the chain
        if (prog && k % a.band_ch == 0 && k > 0) {
            asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
            fence_proxy_async_global();
            publish(prog, tag + (unsigned int)(k / a.band_ch));
        }
        if (dt) dt[2] += (uint64_t)clock64();
    }
    bulk_wait_all();
    fence_proxy_async_global();   // the bulk-stored x before the group barrier's release
    if (prog) publish(prog, tag + (unsigned int)sweep_bands(n, a.band_ch));
    if (dt) dt[3] += (uint64_t)clock64() - d0;
}

// One 256-row chunk of the back-sweep chain (rows cnt-1 .. 0 of the ring slot, x into xb), as a
// separate non-inlined function: the kernel's register pressure (255, spills) does not reach
// this loop (TINV_SWEEP2=2).
__device__ __noinline__ void sweep_chunk(const double* __restrict__ Fs, const double* __restrict__ Ts, double* __restrict__ xb,
                                         int cnt, double* x12) {
    double x1 = x12[0], x2 = x12[1];
    const int top = cnt & ~15;
    for (int u = cnt - 1; u >= top; u--) {
        const double2 bc = *reinterpret_cast<const double2*>(Fs + u * 4 + 2);
        const double xi = fma(-bc.x, x1, fma(-bc.y, x2, Ts[u]));
        xb[u] = xi;
        x2 = x1;
        x1 = xi;
    }
    for (int u0 = top - 16; u0 >= 0; u0 -= 16) {
        double bb[16], cc[16], tt[16], xv[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const double2 bc = *reinterpret_cast<const double2*>(Fs + (u0 + u) * 4 + 2);
            bb[u] = bc.x; cc[u] = bc.y; tt[u] = Ts[u0 + u];
        }
#pragma unroll
        for (int u = 15; u >= 0; u--) {
            xv[u] = fma(-bb[u], x1, fma(-cc[u], x2, tt[u]));
            x2 = x1;
            x1 = xv[u];
        }
#pragma unroll
        for (int u = 0; u < 16; u += 2)
            *reinterpret_cast<double2*>(xb + u0 + u) = make_double2(xv[u], xv[u + 1]);
    }
    x12[0] = x1;
    x12[1] = x2;
}

// The same sweep split over two threads of CTA 0 (the wide window, where warps 1.. of CTA 0 are
// otherwise idle): the chain thread (`helper` false) only waits for its ring slot, runs the
// 16-row batches into the x staging buffer and hands the chunk over (fence.proxy.async +
// mbarrier xfull); the helper thread (warp 1) refills the ring, issues the chunk's bulk store,
// frees the staging buffer (mbarrier xempty) once the store has read it, and publishes the
// bands.  The per-chunk TMA / bulk-store / release work (~16% of the single-thread sweep) leaves
// the dependent chain.  Same arithmetic, same order as back_sweep.  `xseq` counts the chunks
// of every such sweep (both threads keep identical copies): buffer = seq & 1, its use = seq >> 1.
__device__ void back_sweep_ws(const CwyArgs& a, const GroupWS& ws, int64_t j, const Smem& sm, uint32_t& mbph,
                              uint32_t& xseq, bool helper, unsigned int* prog, unsigned int tag, uint64_t* dt = nullptr) {
    // dt (debug build, TINV_DBG bit 3; chain thread): SM clocks in [0] buffer / ring waits, [1] the
    // chains, [2] the hand-over, [3] total
    const uint64_t d0 = dt ? (uint64_t)clock64() : 0;
    const int64_t n = a.n;
    const double* __restrict__ F = a.F + j * n * 4;
    const double* __restrict__ ts = ws.ysol;
    double* __restrict__ x = ws.x;
    double* ring = sm.bring;
    const int64_t C = (n + CH - 1) / CH;
    uint64_t* xfull = sm.mbar + kXFull;
    uint64_t* xempty = sm.mbar + kXEmpty;
    double* xbuf = sm.racc;   // 2 CH doubles
    auto rows = [&](int64_t k, int64_t& lo, int64_t& hi) {
        const int64_t c = C - 1 - k;
        lo = c * CH;
        hi = (lo + CH < n) ? lo + CH : n;
    };
    if (helper) {
        auto issue = [&](int64_t k) {
            const int slot = (int)(k % kRing);
            int64_t lo, hi;
            rows(k, lo, hi);
            const uint32_t fb = (uint32_t)((hi - lo) * 32), tb = (uint32_t)(((hi - lo + 1) & ~int64_t(1)) * 8);
            double* dst = ring + (int64_t)slot * 5 * CH;
            mbar_expect_tx(sm.mbar + slot, fb + tb);
            bulk_g2s(dst, F + lo * 4, fb, sm.mbar + slot);
            bulk_g2s(dst + 4 * CH, ts + lo, tb, sm.mbar + slot);
        };
        fence_proxy_async_global();
        for (int64_t k = 0; k < C && k < kRing; k++) issue(k);
        for (int64_t k = 0; k < C; k++) {
            const uint32_t sq = xseq + (uint32_t)k, b = sq & 1u;
            mbar_wait(xfull + b, (sq >> 1) & 1u);   // chunk k in xbuf[b]; its ring slot is consumed
            int64_t lo, hi;
            rows(k, lo, hi);
            bulk_s2g(x + lo, xbuf + b * CH, (uint32_t)((hi - lo + 1) & ~int64_t(1)) * 8u);
            bulk_commit();
            if (k + kRing < C) issue(k + kRing);
            // the buffer is free as soon as this store has read it -- during the chain of chunk
            // k+1, so chunk k+2 never waits for it (released one step later, after the wake-up
            // of the next hand-over, the chain thread stood ~0.5 us per chunk: 18% of the sweep)
            bulk_wait_read<0>();
            mbar_arrive(xempty + b);
            // band b = chunks [b band_ch, (b+1) band_ch) complete once at most the newest group
            // (this chunk's store) is pending
            if (prog && k % a.band_ch == 0 && k > 0) {
                asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
                fence_proxy_async_global();
                publish(prog, tag + (unsigned int)(k / a.band_ch));
            }
        }
        bulk_wait_all();
        fence_proxy_async_global();   // the bulk-stored x before the group barrier's release
        if (prog) publish(prog, tag + (unsigned int)sweep_bands(n, a.band_ch));
    } else {
        double x1 = 0.0, x2 = 0.0;
        for (int64_t k = 0; k < C; k++) {
            const uint32_t sq = xseq + (uint32_t)k, b = sq & 1u;
            const int slot = (int)(k % kRing);
            double* xb = xbuf + b * CH;
            const uint64_t e0 = dt ? (uint64_t)clock64() : 0;
            if (sq >= 2u) mbar_wait(xempty + b, ((sq >> 1) - 1u) & 1u);   // the store of seq - 2 read it
            mbar_wait(sm.mbar + slot, (mbph >> slot) & 1u);
            mbph ^= 1u << slot;
            const double* Fs = ring + (int64_t)slot * 5 * CH;
            const double* Ts = Fs + 4 * CH;
            int64_t lo, hi;
            rows(k, lo, hi);
            const int cnt = (int)(hi - lo);
            if (a.sweep2 == 2) {
                const uint64_t e1 = dt ? (uint64_t)clock64() : 0;
                double x12[2] = {x1, x2};
                sweep_chunk(Fs, Ts, xb, cnt, x12);
                x1 = x12[0];
                x2 = x12[1];
                const uint64_t e2 = dt ? (uint64_t)clock64() : 0;
                if (cnt & 1) xb[cnt] = 0.0;
                fence_proxy_async_smem();
                mbar_arrive(xfull + b);
                if (dt) {
                    dt[0] += e1 - e0;
                    dt[1] += e2 - e1;
                    dt[2] += (uint64_t)clock64() - e2;
                }
                continue;
            }
            const int top = cnt & ~15;
            for (int u = cnt - 1; u >= top; u--) {
                const double2 bc = *reinterpret_cast<const double2*>(Fs + u * 4 + 2);
                const double xi = fma(-bc.x, x1, fma(-bc.y, x2, Ts[u]));
                xb[u] = xi;
                x2 = x1;
                x1 = xi;
            }
            for (int u0 = top - 16; u0 >= 0; u0 -= 16) {
                double bb[16], cc[16], tt[16], xv[16];
#pragma unroll
                for (int u = 0; u < 16; u++) {
                    const double2 bc = *reinterpret_cast<const double2*>(Fs + (u0 + u) * 4 + 2);
                    bb[u] = bc.x; cc[u] = bc.y; tt[u] = Ts[u0 + u];
                }
#pragma unroll
                for (int u = 15; u >= 0; u--) {
                    xv[u] = fma(-bb[u], x1, fma(-cc[u], x2, tt[u]));
                    x2 = x1;
                    x1 = xv[u];
                }
#pragma unroll
                for (int u = 0; u < 16; u += 2)
                    *reinterpret_cast<double2*>(xb + u0 + u) = make_double2(xv[u], xv[u + 1]);
            }
            if (cnt & 1) xb[cnt] = 0.0;   // x[n] (padding of the last, odd chunk)
            fence_proxy_async_smem();     // generic smem writes -> the helper's bulk store
            mbar_arrive(xfull + b);
        }
    }
    xseq += (uint32_t)C;
    if (dt) dt[3] += (uint64_t)clock64() - d0;
}

// Composition of the forward maps of CTAs 0..cnt-1 (S slots FA, FB), applied in CTA order, by
// warp 0 (lane-serial pieces + a warp scan); broadcast through `buf`.
__device__ __forceinline__ Aff1 compose_ctas(const double* S, int cnt, Aff1* buf) {
    if ((threadIdx.x >> 5) == 0) {
        const int lane = threadIdx.x & 31;
        const int per = (cnt + 31) / 32;
        Aff1 f{1.0, 0.0};
        for (int q = lane * per; q < cnt && q < (lane + 1) * per; q++)
            f = comp(Aff1{ld(S + q * SST + SSlots::FA), ld(S + q * SST + SSlots::FB)}, f);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const Aff1 g = shfl_up(f, o);
            if (lane >= o) f = comp(f, g);
        }
        if (lane == 31) buf[0] = f;
    }
    __syncthreads();
    const Aff1 r = buf[0];
    __syncthreads();
    return r;
}

template <class Mark>
__device__ void cta_solve(const CwyArgs& a, const GroupWS& ws, int64_t j, int mode, int restart, const Smem& sm,
                          Mark mark, uint32_t& mbph) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n = a.n;
    const double* __restrict__ F = a.F + j * n * 4;      // (l, 1/u0, u1/u0, u2/u0) per row
    const int8_t* __restrict__ FP = a.FP + j * n;
    const double* __restrict__ q = ws.q;
    double* __restrict__ ts = ws.ysol;
    double* __restrict__ x = ws.x;
    auto rhs = [&](int64_t i) -> double { return mode == 0 ? ld(q + i) : start_entry(a.seed, n, j, restart, i); };
    {   // bulk L2 prefetch of the factors (32 B per row) and pivot bytes, 64 KB pieces
        const int64_t nbytes = n * 32;
        for (int64_t o = (int64_t)tid * 65536; o < nbytes; o += (int64_t)NT * 65536)
            l2_prefetch(F + o / 8, (nbytes - o < 65536 ? nbytes - o : 65536) / 8);
        if (tid == NT - 1) {
            const uintptr_t pa = reinterpret_cast<uintptr_t>(FP) & ~uintptr_t(15);
            const int64_t nb16 = (int64_t)(reinterpret_cast<uintptr_t>(FP) + n - pa + 15) / 16 * 2;
            l2_prefetch(reinterpret_cast<const double*>(pa), nb16 < 8192 ? nb16 : 8192);
        }
    }
    // ---- forward, pass 1: chunk maps and ||rhs||_1 (loads batched FB rows at a time)
    constexpr int FB = 8;
    const int64_t L = (n + NT - 1) / NT;
    const int64_t ta = min(n, (int64_t)tid * L), tb = min(n, (int64_t)(tid + 1) * L);
    const int64_t tf = tb < n - 1 ? tb : n - 1;          // forward steps [ta, tf)
    auto fetch = [&](int64_t i0, double* l, int* sw, double* bn, double* rr, bool want_r) {
#pragma unroll
        for (int u = 0; u < FB; u++) {
            const int64_t i = i0 + u;
            const bool ok = i < tf;
            l[u] = ok ? ldro(F + i * 4) : 0.0;
            sw[u] = ok ? (int)FP[i] : 0;
            bn[u] = ok ? rhs(i + 1) : 0.0;
            if (want_r) rr[u] = ok ? ldro(F + i * 4 + 1) : 0.0;
        }
    };
    double r1 = 0.0;
    Aff1 f{1.0, 0.0};
    if (ta < tb) r1 = fabs(rhs(ta));
    for (int64_t i0 = ta; i0 < tf; i0 += FB) {
        double l[FB], bn[FB], rr[FB];
        int sw[FB];
        fetch(i0, l, sw, bn, rr, false);
#pragma unroll
        for (int u = 0; u < FB; u++) {
            if (i0 + u < tf) {
                if (i0 + u + 1 < tb) r1 += fabs(bn[u]);
                if (sw[u]) f.b = fma(-l[u], bn[u], f.b);
                else { f.a = -l[u] * f.a; f.b = fma(-l[u], f.b, bn[u]); }
            }
        }
    }
    Aff1 tot;
    const Aff1 ex = block_scan_excl(f, reinterpret_cast<Aff1*>(sm.acc), tot);
    r1 = block_sum<NT>(r1, sm.red);
    const double sc = (double)n * a.tnorm * fmax(kEps, ldro(a.unn + j)) / r1;
    // ---- forward, pass 2: y_i from the exact incoming carry; t_i = s y_i / u0_i
    {
        double c = fma(ex.a, rhs(0), ex.b);
        for (int64_t i0 = ta; i0 < tf; i0 += FB) {
            double l[FB], bn[FB], rr[FB];
            int sw[FB];
            fetch(i0, l, sw, bn, rr, true);
#pragma unroll
            for (int u = 0; u < FB; u++) {
                if (i0 + u < tf) {
                    double y;
                    if (sw[u]) { y = bn[u]; c = fma(-l[u], bn[u], c); }
                    else { y = c; c = fma(-l[u], c, bn[u]); }
                    st(ts + i0 + u, sc * y * rr[u]);
                }
            }
        }
        if (tb == n && ta < tb) st(ts + n - 1, sc * c * ldro(F + (n - 1) * 4 + 1));
    }
    __syncthreads();
    mark(9);
    if (tid == 0) {
        st(ts + n, 0.0);
        back_sweep(a, ws, j, sm, mbph);
    }
}

// ---------------------------------------------------------------- TMA streaming, narrow clusters
// Clusters with m <= kNarrowM store Y with a uniform row stride m2 = roundup(m, 2) (common.cuh),
// so a CTA's rows [i0, i1) are one contiguous span.  Passes A, BC and D stream it through a
// kNStg-deep shared-memory ring of TMA bulk copies (stage = RPS whole rows + the matching
// coefficient rows x_i), one mbarrier per slot; thread 0 issues, all threads consume.
constexpr int SBD = 3584;                    // Y doubles per stage (28 KB)
constexpr int kMaxRPS = 512;                 // rows per stage cap (coefficient slots)
constexpr int SXD = kMaxRPS + 4;             // coefficient doubles per stage
constexpr int kStgD = SBD + SXD;             // doubles per ring slot
constexpr int kNStg = 4;                     // ring depth

struct Ring {
    double* base;      // kNStg slots of kStgD doubles
    uint64_t* mbar;    // kNStg mbarriers
    uint32_t* ph;      // phase bits (per thread copy)
    uint64_t* tacc;    // optional timers (wait, body, sync+issue, block end) of the timing thread, or nullptr
};

// Stream rows [i0, i1) of Y (and coef[i0, i1) if coef != nullptr) through the ring; for each
// stage call body(ra, rb, Ys, Xs) with Ys = the stage's rows (row i at Ys + (i - ra) m2) and
// Xs = coefficients (x_i at Xs[i - ra]).  All threads call; body may __syncthreads.
// Threads [T0, T0 + TN) run the stream (TN < NT: the look-ahead on warps 1.. while warp 0
// runs the chained back sweep; stage barriers are then named barrier 2 over those warps).
template <int T0, int TN>
__device__ __forceinline__ void sub_sync() {
    if (TN == NT) __syncthreads();
    else asm volatile("bar.sync 2, %0;" ::"n"(TN) : "memory");
}
template <int T0 = 0, int TN = NT, class Body>
__device__ void narrow_stream(const Ring& rg, const double* Y, int m2, int i0, int i1, const double* coef,
                              Body body) {
    if (i1 <= i0) return;
    const int tid = threadIdx.x - T0;
    const int RPS = min(kMaxRPS, SBD / m2);
    const int nst = (i1 - i0 + RPS - 1) / RPS;
    int ps = 0;   // stages issued (thread 0)
    auto issue = [&]() {
        const int slot = ps % kNStg;
        const int ra = i0 + ps * RPS, rb = min(i1, ra + RPS);
        double* dst = rg.base + slot * kStgD;
        const uint32_t yb = (uint32_t)((rb - ra) * m2 * 8);
        const int xa = ra & ~1, xb = (rb + 1) & ~1;
        const uint32_t xbytes = coef ? (uint32_t)((xb - xa) * 8) : 0u;
        mbar_expect_tx(rg.mbar + slot, yb + xbytes);
        bulk_g2s(dst, Y + (int64_t)ra * m2, yb, rg.mbar + slot);
        if (coef) bulk_g2s(dst + SBD, coef + xa, xbytes, rg.mbar + slot);
        ps++;
    };
    if (tid == 0) {
        fence_proxy_async_global();
        while (ps < nst && ps < kNStg) issue();
    }
    for (int s = 0; s < nst; s++) {
        const int slot = s % kNStg;
        const int ra = i0 + s * RPS, rb = min(i1, ra + RPS);
        const uint64_t c0 = rg.tacc ? gtime() : 0;
        mbar_wait(rg.mbar + slot, (*rg.ph >> slot) & 1u);
        *rg.ph ^= 1u << slot;
        const uint64_t c1 = rg.tacc ? gtime() : 0;
        const double* Ys = rg.base + slot * kStgD;
        double* Xs = const_cast<double*>(Ys) + SBD + (ra & 1);
        body(ra, rb, Ys, Xs);       // (a body that writes the slot fences the async proxy itself)
        const uint64_t c2 = rg.tacc ? gtime() : 0;
        sub_sync<T0, TN>();         // slot free
        if (tid == 0 && ps < nst) issue();
        if (rg.tacc) {
            rg.tacc[0] += c1 - c0;
            rg.tacc[1] += c2 - c1;
            rg.tacc[2] += gtime() - c2;
        }
    }
}

// Row dots over a stage, P <= kNarrowM: one thread per row (no shuffle reductions: the
// rows are short), vector v staged in shared memory (broadcast reads); epi(i, dot).
template <class Len, class Epi>
__device__ __forceinline__ void narrow_rowdots(int ra, int rb, int m2, const double* Ys, const double* v, Len len,
                                               Epi epi) {
    for (int i = ra + (int)threadIdx.x; i < rb; i += NT) {
        const double* row = Ys + (i - ra) * m2;
        const int le = len(i);
        double a0 = 0.0, a1 = 0.0;
        int k = 0;
        for (; k + 1 < le; k += 2) {
            const double2 y = *reinterpret_cast<const double2*>(row + k);
            const double2 w = *reinterpret_cast<const double2*>(v + k);
            a0 = fma(y.x, w.x, a0);
            a1 = fma(y.y, w.y, a1);
        }
        if (k < le) a0 = fma(row[k], v[k], a0);
        epi(i, a0 + a1);
    }
}

// Column accumulate over a stage: thread (cp, rs) adds Y[i][2cp..2cp+1] * c_i for the stage's
// rows i with (i - ra) % RS == rs into (a0, a1); columns k < len(i) only.
template <int T0 = 0, int TN = NT, class Len>
__device__ __forceinline__ void narrow_colacc(int ra, int rb, int m2, const double* Ys, const double* Xs, int CPT,
                                              Len len, double& a0, double& a1) {
    const int t = threadIdx.x - T0;
    const int RS = TN / CPT, cp = t % CPT, rs = t / CPT;
    const int k = 2 * cp;
    constexpr int U = 4;
    for (int ib = ra + rs; ib < rb; ib += RS * U) {
        double2 av[U];
        double cv[U];
        int le[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = ib + u * RS;
            le[u] = (i < rb) ? len(i) : 0;
            av[u] = (k < le[u]) ? *reinterpret_cast<const double2*>(Ys + (i - ra) * m2 + k) : make_double2(0.0, 0.0);
            cv[u] = (i < rb) ? Xs[i - ra] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (k < le[u]) a0 = fma(av[u].x, cv[u], a0);
            if (k + 1 < le[u]) a1 = fma(av[u].y, cv[u], a1);
        }
    }
}

// Fixed-order reduction of the row-slice column accumulators; writes out[k] for k < P.
template <int T0 = 0, int TN = NT>
__device__ __forceinline__ void narrow_colacc_finish(const Smem& sm, int CPT, int64_t P, double a0, double a1,
                                                     double* out) {
    const int tid = threadIdx.x - T0, RS = TN / CPT, cp = tid % CPT, rs = tid / CPT;
    sub_sync<T0, TN>();
    sm.acc[tid] = make_double2(a0, a1);
    sub_sync<T0, TN>();
    if (rs == 0) {
        for (int q = 1; q < RS; q++) {
            const double2 t = sm.acc[cp + q * CPT];
            a0 += t.x;
            a1 += t.y;
        }
        const int64_t k = 2 * cp;
        if (k < P) st(out + k, a0);
        if (k + 1 < P) st(out + k + 1, a1);
    }
    sub_sync<T0, TN>();
}

// ---------------------------------------------------------------- TMA streaming, wide passes
// Passes with more than kNarrowM columns (every pass of a cluster with m > kNarrowM once
// p > kNarrowM, and the T passes) stream their rows in column-block-major order: block kb
// covers columns [kb PW, kb PW + PW); for each block the rows that reach it are cut into
// pieces (one TMA bulk copy per row piece), PPS pieces per ring stage.  Warp-specialised:
// warp 0 only issues the copies (gated by per-slot "empty" mbarriers), warps 1..7 consume
// (full mbarriers) and release.  Row dots: consumer warp w takes piece w-1, with the current
// block of the vector(s) in shared memory (TMA double buffer, next block prefetched), and
// adds its warp sum into a per-row accumulator (fixed block order: deterministic).  Column
// accumulates: consumer thread t' owns the block's columns 2t', 2t'+1 and adds the pieces'
// rows in order.  Rows of one pass are processed in chunks of <= RCH rows.
constexpr int NCW = NW - 1;              // consumer warps
constexpr int NCT = NCW * 32;            // consumer threads
constexpr int PW = 2 * NCT;              // column block / piece width (doubles) = 448
static_assert(PW == kPieceW, "piece width of the partitions");
static_assert(PW == kWidePieceW, "piece width known to the host (workspace sizes)");
constexpr int PPS = NCW;                 // pieces per stage = consumer warps
constexpr int RCH = 1024;                // rows per chunk (row accumulators; coefficients in Smem::cf)
constexpr int kWStgD = PPS * PW;         // doubles per wide ring slot
constexpr int kWStg = 7;                 // wide ring depth
constexpr int kPfAhead = 0;              // wide stages prefetched into L2 beyond the ring (0: off;
                                         // measured slower on B200: the prefetches compete with
                                         // the ring's own bulk copies)
constexpr int64_t kRingD = (int64_t)kWStg * kWStgD > (int64_t)kNStg * kStgD ? (int64_t)kWStg * kWStgD
                                                                            : (int64_t)kNStg * kStgD;
static_assert((int64_t)kNStg * kStgD + kSolveDoubles <= kRingD, "back-sweep ring after the narrow ring");
static_assert(2 * CH <= 2 * RCH, "x staging of the back sweep in the row accumulators");
static_assert(kRBufD <= kRingD, "reduce_partials staging inside the pass rings");

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory"); }

// Row source of a wide pass: row r has valid columns [cs(r), ce(r)) stored from column 0 at
// base(r) (16-byte aligned; storage padded to an even column count).  Indices are 32-bit.
struct SrcY {      // rows of Y_P (packed row-major, zero-free)
    const double* Y;
    int m, P;
    __device__ const double* base(int r) const { return Y + y_row_off(r, m); }
    __device__ int cs(int) const { return 0; }
    __device__ int ce(int r) const { return r + 1 < P ? r + 1 : P; }
    // rows of [r0, r1) that reach block kb: ce(r) > kb PW  <=>  r >= kb PW
    __device__ void rows(int kb, int r0, int r1, int& a, int& b) const {
        a = max(r0, kb * PW);
        b = r1;
    }
    __device__ int nblk() const { return (P + PW - 1) / PW; }
    __device__ int width() const { return P; }
};
struct SrcTc {     // column-packed T: "row" k = T[0..k, k]
    const double* Tc;
    int P;
    __device__ const double* base(int k) const { return Tc + tcol_off(k); }
    __device__ int cs(int) const { return 0; }
    __device__ int ce(int k) const { return k + 1; }
    __device__ void rows(int kb, int r0, int r1, int& a, int& b) const {
        a = max(r0, kb * PW);
        b = r1;
    }
    __device__ int nblk() const { return (P + PW - 1) / PW; }
    __device__ int width() const { return P; }
};
struct SrcTr {     // row-major T: row l = T[l, l..P)
    const double* Tr;
    int m2, P;
    __device__ const double* base(int l) const { return Tr + (int64_t)l * m2; }
    __device__ int cs(int l) const { return l; }
    __device__ int ce(int) const { return P; }
    __device__ void rows(int kb, int r0, int r1, int& a, int& b) const {
        a = r0;
        b = min(r1, (kb + 1) * PW);
    }
    __device__ int nblk() const { return (P + PW - 1) / PW; }
    __device__ int width() const { return P; }
};

// Pipeline state of the wide ring: full[s] completes when stage s's bulk copies land, empty[s]
// when all NW warps released it.  Global stage counters (issued / consumed) persist across
// passes, so slot = count % kNStg and the phase parity = (count / kNStg) & 1.
struct WRing {
    double* base;
    uint64_t* full;     // kWStg (count 1 + tx)
    uint64_t* empty;    // kWStg (count NCW consumer warps)
    uint32_t* issued;   // producer warp's counter
    uint32_t* used;     // consumer threads' counter
    uint64_t* tacc;     // optional timers (wait, body, release, block end) or nullptr
};

// Piece stride of a pass: PW for multi-block passes, else the (even) row width; rows per
// stage: as many pieces as fit a slot, at most two per consumer warp.
template <class Src>
__device__ __forceinline__ int wide_pst(const Src& src) {
    return src.nblk() > 1 ? PW : ((src.width() + 1) & ~1);
}
__device__ __forceinline__ int wide_rps(int pst) { return min(2 * NCW, kWStgD / max(pst, 2)); }

// Walk (chunk of rows, block kb, stage of <= RPS rows) in the order above.  Consumers (warps
// 1..NCW) call blk_begin(kb, c0, c1) at the first stage of each block, body(kb, ra, rb, slot)
// per stage (piece q = row ra + q at slot + q PW, columns [kb PW, kb PW + PW), only the valid
// ones copied) and blk_end(kb) after its last stage; these may use consumer_sync() but not
// __syncthreads.  chunk_begin / chunk_end run on all threads around each chunk (may
// __syncthreads).
template <int CR = RCH, class Src, class Body, class BlkBegin, class BlkEnd, class ChunkBegin, class ChunkEnd>
__device__ void wide_stream(const WRing& rg, const Src& src, int r0, int r1, bool reverse_blocks, uint64_t pol,
                            ChunkBegin chunk_begin, BlkBegin blk_begin, Body body, BlkEnd blk_end,
                            ChunkEnd chunk_end) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NB = src.nblk();
    // piece stride / rows per stage: a single narrow block packs up to 32 rows per stage
    const int PST = wide_pst(src);
    const int RPS = wide_rps(PST);
    for (int c0 = r0; c0 < r1; c0 += CR) {
        const int c1 = min(r1, c0 + CR);
        chunk_begin(c0, c1);
        auto blk_of = [&](int t) { return reverse_blocks ? NB - 1 - t : t; };
        // stage cursor: block step t, next row; returns false at the end
        auto next = [&](int& t, int& row, int& ra, int& rb) -> bool {
            while (t < NB) {
                int a, b;
                src.rows(blk_of(t), c0, c1, a, b);
                row = max(row, a);
                if (row < b) {
                    ra = row;
                    rb = min(b, row + RPS);
                    row = rb;
                    return true;
                }
                t++;
                row = -1;
            }
            return false;
        };
        int t = 0, row = -1, ra = 0, rb = 0;
        if (warp == 0) {
            // ---- producer: lane q copies piece q of every stage; a second cursor kPfAhead
            // stages further on prefetches the same pieces into L2
            auto piece = [&](int kb, int r, int& a, int& b) {
                a = max(src.cs(r) & ~1, kb * PW);
                b = min((src.ce(r) + 1) & ~1, kb * PW + PW);
            };
            int ft = 0, frow = -1, fra = 0, frb = 0;
            bool fmore = true;
            auto prefetch_next = [&]() {
                if (kPfAhead == 0) return;
                if (fmore && (fmore = next(ft, frow, fra, frb))) {
                    const int r = fra + lane;
                    if (r < frb) {
                        int a, b;
                        piece(blk_of(ft), r, a, b);
                        if (b > a) l2_prefetch(src.base(r) + a, b - a);
                    }
                }
            };
            if (lane == 0) fence_proxy_async_global();
            __syncwarp();
            for (int k = 0; k < kWStg + kPfAhead; k++) prefetch_next();
            while (next(t, row, ra, rb)) {
                const int kb = blk_of(t);
                const uint32_t g = *rg.issued;
                const int slot = (int)(g % kWStg);
                if (g >= (uint32_t)kWStg) mbar_wait(rg.empty + slot, ((g / kWStg) - 1) & 1u);
                const int r = ra + lane;
                if (r < rb) {
                    int a, b;
                    piece(kb, r, a, b);
                    if (b > a) {
                        const uint32_t bytes = (uint32_t)(b - a) * 8u;
                        mbar_add_tx(rg.full + slot, bytes);
                        bulk_g2s_hint(rg.base + (int64_t)slot * kWStgD + (r - ra) * PST + (a - kb * PW),
                                      src.base(r) + a, bytes, rg.full + slot, pol);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(rg.full + slot);
                *rg.issued = g + 1;
                prefetch_next();
            }
        } else {
            // ---- consumers
            int last_kb = -1;
            while (next(t, row, ra, rb)) {
                const int kb = blk_of(t);
                const uint64_t c0t = rg.tacc ? gtime() : 0;
                if (kb != last_kb) {
                    if (last_kb >= 0) blk_end(last_kb);
                    blk_begin(kb, c0, c1);
                }
                last_kb = kb;
                const uint32_t u = *rg.used;
                const int slot = (int)(u % kWStg);
                const uint64_t c1t = rg.tacc ? gtime() : 0;
                mbar_wait(rg.full + slot, (u / kWStg) & 1u);
                const uint64_t c2t = rg.tacc ? gtime() : 0;
                body(kb, ra, rb, rg.base + (int64_t)slot * kWStgD);
                __syncwarp();
                if (lane == 0) mbar_arrive(rg.empty + slot);
                *rg.used = u + 1;
                if (rg.tacc) {
                    const uint64_t c3t = gtime();
                    rg.tacc[3] += c1t - c0t;
                    rg.tacc[0] += c2t - c1t;
                    rg.tacc[1] += c3t - c2t;
                }
            }
            if (last_kb >= 0) blk_end(last_kb);
        }
        __syncthreads();   // ring drained before the next chunk / pass
        chunk_end(c0, c1);
    }
}

// L2 prefetch of the first stages of this CTA's next wide pass (issued before the group
// barrier that precedes the pass, so its first TMA copies hit L2): the pieces of the first
// block with rows, for up to `nr` rows; lanes of warp 0, one prefetch per piece.
template <class Src>
__device__ __forceinline__ void pf_first(const Src& src, int r0, int r1, int nr) {
    if (threadIdx.x >= 32 || r1 <= r0) return;
    const int NB = src.nblk();
    for (int kb = 0; kb < NB; kb++) {
        int a, b;
        src.rows(kb, r0, r1, a, b);
        if (a >= b) continue;
        for (int r = a + (int)threadIdx.x; r < b && r < a + nr; r += 32) {
            const int lo = max(src.cs(r) & ~1, kb * PW), hi = min((src.ce(r) + 1) & ~1, kb * PW + PW);
            if (hi > lo) l2_prefetch(src.base(r) + lo, hi - lo);
        }
        return;
    }
}

// Row dots of a wide pass: dot(r) = sum_{cs(r) <= k < ce(r)} row_r[k] v[k] (and with a second
// vector w when TWO); epi(r, dot, dot2) after all blocks, one thread per row.
template <bool TWO, class Src, class Epi>
__device__ void wide_rowdots(const Smem& sm, const WRing& rg, const Src& src, int r0, int r1, const double* v,
                             const double* w, int P, uint64_t pol, Epi epi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* racc = sm.racc;           // RCH (x2 when TWO)
    int cb = 0;
    // vector blocks: TMA copies into a double buffer (buffer kb & 1), block kb + 1 prefetched
    // when block kb starts; one mbarrier per buffer; issued by consumer thread 32
    auto vfetch = [&](int kb) {
        const int buf = kb & 1;
        const int a = kb * PW, b = min(P, kb * PW + PW);
        const uint32_t bytes = (uint32_t)(((b - a + 1) & ~1) * 8);
        mbar_expect_tx(sm.vbar + buf, bytes * (TWO ? 2u : 1u));
        bulk_g2s(sm.vblk + buf * 2 * PW, v + a, bytes, sm.vbar + buf);
        if (TWO) bulk_g2s(sm.vblk + buf * 2 * PW + PW, w + a, bytes, sm.vbar + buf);
    };
    const int NB = src.nblk();
    int pre = -1;   // block prefetched into its buffer (thread 32)
    wide_stream(
        rg, src, r0, r1, false, pol,
        [&](int c0, int c1) {
            cb = c0;
            pre = -1;
            for (int i = threadIdx.x; i < c1 - c0; i += NT) {
                racc[i] = 0.0;
                if (TWO) racc[RCH + i] = 0.0;
            }
            __syncthreads();
        },
        [&](int kb, int c0, int c1) {
            consumer_sync();   // all consumers are done with the buffer that kb + 1 will overwrite
            if (threadIdx.x == 32) {
                fence_proxy_async_global();
                if (pre != kb) vfetch(kb);       // not prefetched by the previous block
                pre = -1;
                if (kb + 1 < NB) {               // blocks with rows are contiguous in the walk
                    int a, b;
                    src.rows(kb + 1, c0, c1, a, b);
                    if (a < b) {
                        vfetch(kb + 1);
                        pre = kb + 1;
                    }
                }
            }
            const uint32_t u = sm.vuse[kb & 1];
            mbar_wait(sm.vbar + (kb & 1), u & 1u);
            consumer_sync();
            if (threadIdx.x == 32) sm.vuse[kb & 1] = u + 1;
        },
        [&](int kb, int ra, int rb, const double* slot) {
            const int PST = wide_pst(src);
            for (int q = warp - 1; ra + q < rb; q += NCW) {
                const int r = ra + q;
                const int lo = src.cs(r), hi = src.ce(r);
                const double* vb = sm.vblk + (kb & 1) * 2 * PW;
                double a1 = 0.0, a2 = 0.0;
                const double* rowp = slot + q * PST;
                const int kbase = kb * PW;
                if (lo <= kbase && hi >= kbase + PW) {   // full piece: no masks
#pragma unroll
                    for (int e = 0; e < PW; e += 64) {
                        const int cl = e + 2 * lane;
                        const double2 y = *reinterpret_cast<const double2*>(rowp + cl);
                        const double2 vv = *reinterpret_cast<const double2*>(vb + cl);
                        a1 = fma(y.x, vv.x, a1);
                        a1 = fma(y.y, vv.y, a1);
                        if (TWO) {
                            const double2 ww = *reinterpret_cast<const double2*>(vb + PW + cl);
                            a2 = fma(y.x, ww.x, a2);
                            a2 = fma(y.y, ww.y, a2);
                        }
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < PW; e += 64) {   // lane: columns e + 2 lane, +1 (conflict-free)
                        const int cl = e + 2 * lane;
                        const int k = kbase + cl;
                        if (cl < PST && k + 1 >= lo && k < hi) {
                            const double2 y = *reinterpret_cast<const double2*>(rowp + cl);
                            const double2 vv = *reinterpret_cast<const double2*>(vb + cl);
                            const double y0 = (k >= lo) ? y.x : 0.0;
                            const double y1 = (k + 1 < hi) ? y.y : 0.0;
                            a1 = fma(y0, vv.x, a1);
                            a1 = fma(y1, vv.y, a1);
                            if (TWO) {
                                const double2 ww = *reinterpret_cast<const double2*>(vb + PW + cl);
                                a2 = fma(y0, ww.x, a2);
                                a2 = fma(y1, ww.y, a2);
                            }
                        }
                    }
                }
                a1 = warp_sum(a1);
                if (TWO) a2 = warp_sum(a2);
                if (lane == 0) {
                    racc[r - cb] += a1;
                    if (TWO) racc[RCH + r - cb] += a2;
                }
            }
        },
        [&](int) {},
        [&](int c0, int c1) {
            for (int r = c0 + threadIdx.x; r < c1; r += NT) {
                if (TWO) epi(r, racc[r - c0], racc[RCH + r - c0]);
                else epi(r, racc[r - c0], 0.0);
            }
            __syncthreads();
        });
}

// Column accumulate of a wide pass: out[k] = sum_r row_r[k] coef(r) for k < P over rows
// [r0, r1); coefficients staged per chunk from coef (global).  Returns sum coef^2.  TWO: a
// second coefficient vector coef2 -> out2 from the same stream (c2 sum in *c2b).  accum: add
// into out (and out2) instead of overwriting them (rows of one CTA split over several calls).
template <bool TWO = false, class Src>
__device__ double wide_colacc(const Smem& sm, const WRing& rg, const Src& src, int r0, int r1, const double* coef,
                              int P, double* out, bool reverse_blocks, uint64_t pol, bool accum = false,
                              const double* coef2 = nullptr, double* out2 = nullptr, double* c2b = nullptr,
                              int ovr = -1, double ovv = 0.0) {
    const int tid = threadIdx.x, tc = tid - 32;   // consumer thread index
    double c2 = 0.0, c2x = 0.0;
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    int cb = 0;
    // The accumulate owns columns 2tc, 2tc+1 of every block.  With one row chunk each block's
    // sums are final at its end (plain store); with several chunks they are added up (zeroed
    // first).  Blocks that no row of this CTA reaches are zero.
    const bool multi = accum || (r1 - r0) > RCH;
    if (tc >= 0 && !accum)
        for (int kb = 0; kb < src.nblk(); kb++) {
            int a, b;
            src.rows(kb, r0, r1, a, b);
            if (a < b && (r1 - r0) <= RCH) continue;   // written by blk_end
            const int k = kb * PW + 2 * tc;
            if (k < P) { st(out + k, 0.0); if (TWO) st(out2 + k, 0.0); }
            if (k + 1 < P) { st(out + k + 1, 0.0); if (TWO) st(out2 + k + 1, 0.0); }
        }
    if (TWO) *c2b = 0.0;
    if (r1 <= r0) return 0.0;
    double* cf2 = sm.racc;   // second coefficient chunk (the row accumulators are unused here)
    static_assert(2 * RCH >= CFCH, "second coefficient chunk in the row accumulators");
    // accumulating passes (several chunks / calls): the block's previous sums are loaded when the
    // block starts and added at its end, so the L2 round trip overlaps the block's stages
    // instead of stalling every block end (the fused pass A2 runs ~8 calls per vector)
    double o0 = 0.0, o1 = 0.0, o2 = 0.0, o3 = 0.0;
    wide_stream(
        rg, src, r0, r1, reverse_blocks, pol,
        [&](int c0, int c1) {
            cb = c0;
            for (int r = c0 + tid; r < c1; r += NT) {
                const double c = (r == ovr) ? ovv : ld(coef + r);   // ovr: coefficient of one row replaced
                sm.cf[r - c0] = c;
                c2 = fma(c, c, c2);
                if (TWO) {
                    const double cx = ld(coef2 + r);
                    cf2[r - c0] = cx;
                    c2x = fma(cx, cx, c2x);
                }
            }
            __syncthreads();
            a0 = a1 = b0 = b1 = 0.0;
        },
        [&](int kb, int, int) {
            if (multi) {
                const int k = kb * PW + 2 * tc;
                o0 = (k < P) ? ld(out + k) : 0.0;
                o1 = (k + 1 < P) ? ld(out + k + 1) : 0.0;
                if (TWO) {
                    o2 = (k < P) ? ld(out2 + k) : 0.0;
                    o3 = (k + 1 < P) ? ld(out2 + k + 1) : 0.0;
                }
            }
        },
        [&](int kb, int ra, int rb, const double* slot) {
            const int k = kb * PW + 2 * tc;
            const int PST = wide_pst(src);
            // every row of the stage covers the block's valid columns (SrcY: row r has
            // columns [0, min(r + 1, P))): no per-row masks
            if (src.cs(ra) == 0 && src.ce(ra) >= min(kb * PW + PW, P)) {
                if (k < P) {
                    const bool two = (k + 1 < P);
                    const double* sp = slot + 2 * tc;
                    const double* cp = sm.cf + (ra - cb);
                    const double* cp2 = cf2 + (ra - cb);
#pragma unroll 7
                    for (int q = 0; q < rb - ra; q++) {
                        const double2 y = *reinterpret_cast<const double2*>(sp + q * PST);
                        const double c = cp[q];
                        const double y1 = two ? y.y : 0.0;
                        a0 = fma(y.x, c, a0);
                        a1 = fma(y1, c, a1);
                        if (TWO) {
                            const double cx = cp2[q];
                            b0 = fma(y.x, cx, b0);
                            b1 = fma(y1, cx, b1);
                        }
                    }
                }
                return;
            }
            for (int r = ra; r < rb; r++) {
                const int lo = src.cs(r), hi = src.ce(r);
                if (k + 1 >= lo && k < hi) {
                    const double2 y = *reinterpret_cast<const double2*>(slot + (r - ra) * PST + 2 * tc);
                    const double c = sm.cf[r - cb];
                    const double y0 = (k >= lo) ? y.x : 0.0, y1 = (k + 1 < hi) ? y.y : 0.0;
                    a0 = fma(y0, c, a0);
                    a1 = fma(y1, c, a1);
                    if (TWO) {
                        const double cx = cf2[r - cb];
                        b0 = fma(y0, cx, b0);
                        b1 = fma(y1, cx, b1);
                    }
                }
            }
        },
        [&](int kb) {
            const int k = kb * PW + 2 * tc;
            if (k < P) {
                st(out + k, multi ? o0 + a0 : a0);
                if (TWO) st(out2 + k, multi ? o2 + b0 : b0);
            }
            if (k + 1 < P) {
                st(out + k + 1, multi ? o1 + a1 : a1);
                if (TWO) st(out2 + k + 1, multi ? o3 + b1 : b1);
            }
            a0 = a1 = b0 = b1 = 0.0;
        },
        [&](int, int) {});
    if (TWO) *c2b = c2x;
    return c2;
}

// ---------------------------------------------------------------- blocked look-ahead
// SURVEY §8(f) row 2 (Eq. (4), Alg. 3, u-step PAPER.md:530-538):
// for the block of NV <= kLabMax upcoming first iterates X = [x^(1)_k .. x^(1)_{k+NV-1}] (all
// computed by the batched solve), apply the k accepted reflectors at once:
//   BL1  G  = Y_k^T X            (k x NV)  columns of Y_k split over the CTAs (whole dots, no partials)
//   BL2  G' = T_k^T G            (k x NV)  columns of T (rows of T^T) split over the CTAs
//   BL3  U  = X - Y_k G'         (n x NV, rows >= k)  rows split over the CTAs
// Skinny GEMMs: 2 NV flops per 8 bytes of Y (<= 2 flop/B at NV = 8), far below the fp64 FMA
// peak per byte of HBM, so they are DFMA loops on staged operands, not fp64 tensor-core tiles.
// Operands written inside this kernel are read through L2 (ld.cg).

// Stage nseg contiguous global segments seg(s)[0, len) (16-byte aligned, produced in this kernel)
// into shared memory dst + s * dstride: one TMA bulk copy per segment (length rounded up to an
// even count), all completed on sm.rbar; every thread returns after they landed.
template <class Seg>
__device__ __forceinline__ void tma_stage(const Smem& sm, int nseg, Seg seg, int64_t len, double* dst, int64_t dstride) {
    const int tid = threadIdx.x;
    const uint32_t use = *sm.rcnt;
    const int64_t lw = (len + 1) & ~int64_t(1);
    __syncthreads();
    if (tid < nseg && lw > 0) {
        fence_proxy_async_global();
        mbar_add_tx(sm.rbar, (uint32_t)(lw * 8));
        bulk_g2s(dst + (int64_t)tid * dstride, seg(tid), (uint32_t)(lw * 8), sm.rbar);
    }
    __syncthreads();
    if (tid == 0) mbar_arrive(sm.rbar);
    mbar_wait(sm.rbar, use & 1u);
    __syncthreads();
    if (tid == 0) *sm.rcnt = use + 1;
    __syncthreads();
}

// columns [a, b) of [0, k) balanced by their row counts (column c of Y_k has rows c .. n-1)
__device__ __forceinline__ void part_cols_tri(int64_t k, int64_t n, int r, int G, int64_t& a, int64_t& b) {
    auto cum = [n](int64_t c) -> int64_t { return c * n - c * (c - 1) / 2; };
    const int64_t W = cum(k);
    a = (r == 0) ? 0 : bsearch_cum(0, k, (W * r) / G, cum);
    b = (r == G - 1) ? k : bsearch_cum(0, k, (W * (r + 1)) / G, cum);
    a &= ~int64_t(1);   // column pairs (16-byte loads): boundaries even
    b = (r == G - 1) ? k : (b & ~int64_t(1));
}

// BL1 on columns [c0, c1): G[v * ldg + c] = sum_{i >= c} Y[i][c] X_v[i]; also ||X_v||^2 over
// rows [x0, x1) into xsq[v] (this CTA's partial).  Scratch: `scr` (>= 8192 + 4096 doubles).
template <int NV>
__device__ void lab_gemm1(const Smem& sm, const double* __restrict__ Y, int64_t m, int64_t n, int64_t c0, int64_t c1,
                          const double* X, int64_t xst, int nv, double* G, int64_t ldg, double* scr, int64_t x0,
                          int64_t x1, double* xsq) {
    const int tid = threadIdx.x;
    // ||X_v||^2 partials (rows [x0, x1))
    {
        double q[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) q[v] = 0.0;
        for (int64_t i = x0 + tid; i < x1; i += NT)
#pragma unroll
            for (int v = 0; v < NV; v++) {
                const double xv = (v < nv) ? ld(X + v * xst + i) : 0.0;
                q[v] = fma(xv, xv, q[v]);
            }
#pragma unroll
        for (int v = 0; v < NV; v++) {
            const double t = block_sum<NT>(q[v], scr + 12288);
            if (tid == 0) xsq[v] = t;
        }
    }
    if (c1 <= c0) return;
    const int npair = (int)((c1 - c0 + 1) / 2);
    const int CW = min(NT, pow2ceil(npair));   // pair lanes
    const int RL = NT / CW;                    // row lanes
    constexpr int XR = 1024;                   // rows of X staged per chunk (XR * NV <= 8192)
    double* xs = scr;
    double* red = scr + 8192;
    for (int pb = 0; pb < npair; pb += CW) {
        const int cp = pb + tid % CW, rl = tid / CW;
        const int64_t c = c0 + 2 * (int64_t)cp;
        const bool act = cp < npair;
        double acc[2 * NV];
#pragma unroll
        for (int u = 0; u < 2 * NV; u++) acc[u] = 0.0;
        for (int64_t r0 = c0 + 2 * (int64_t)pb; r0 < n; r0 += XR) {
            const int64_t r1 = (r0 + XR < n) ? r0 + XR : n;
            // X rows [r0, r1) of the nv vectors by TMA (layout [v][row]); vectors >= nv: zero
            tma_stage(sm, nv, [&](int v) { return X + v * xst + r0; }, r1 - r0, xs, XR);
            for (int64_t q = tid; q < (int64_t)(NV - nv) * XR; q += NT) xs[(int64_t)nv * XR + q] = 0.0;
            __syncthreads();
            if (act) {
                constexpr int U = 16;   // 16 independent 16-byte loads per thread in flight
                for (int64_t ib = r0 + rl; ib < r1; ib += (int64_t)RL * U) {
                    double2 y[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int64_t i = ib + (int64_t)u * RL;
                        y[u] = (i < r1 && i >= c) ? ld2(Y + y_row_off(i, m) + c) : make_double2(0.0, 0.0);
                        if (i == c) y[u].y = 0.0;   // row c holds column c only
                    }
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int64_t i = ib + (int64_t)u * RL;
                        if (i < r1) {
                            const double* xr = xs + (i - r0);
#pragma unroll
                            for (int v = 0; v < NV; v++) {
                                const double xv = xr[(int64_t)v * XR];
                                acc[2 * v] = fma(y[u].x, xv, acc[2 * v]);
                                acc[2 * v + 1] = fma(y[u].y, xv, acc[2 * v + 1]);
                            }
                        }
                    }
                }
            }
        }
        // sum the row lanes in order (deterministic)
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 2 * NV; u++) red[(int64_t)u * NT + tid] = acc[u];
        __syncthreads();
        if (act && rl == 0) {
            for (int u = 0; u < 2 * NV; u++) {
                double t = 0.0;
                for (int l = 0; l < RL; l++) t += red[(int64_t)u * NT + l * CW + (tid % CW)];
                const int64_t cc = c + (u & 1);
                if (cc < c1) st(G + (int64_t)(u >> 1) * ldg + cc, t);
            }
        }
        __syncthreads();
    }
}

// BL1 streamed through the wide ring (the column split above reads ~430-byte row segments and
// reaches ~1.2 TB/s on cfg5).  Work units are (column block kb, row i) for i in [kb PW, n),
// kb < ceil(k / PW), in block-major order, split evenly over the Gt CTAs; a CTA's range is one
// or a few segments (a column block, a row range), each streamed with whole 448-column row
// pieces.  Consumer thread t' owns the block's columns 2t', 2t'+1 and accumulates them against
// the nv vectors' rows (staged per 512-row chunk) for the whole segment; the segment's sums go
// to partial slot kb + q (slots are unique: in block-major order every new (block, CTA)
// incidence starts at a block or a CTA boundary), and lab_bl1_reduce adds the slots of each
// block in CTA order (deterministic).
struct SrcYB {     // column block kb of Y_P alone: columns [kb PW, min(P, kb PW + PW))
    const double* Y;
    int m, P, kb;
    __device__ const double* base(int r) const { return Y + y_row_off(r, m) + (int64_t)kb * PW; }
    __device__ int cs(int) const { return 0; }
    __device__ int ce(int r) const { return min(r + 1, P) - kb * PW; }
    __device__ void rows(int, int r0, int r1, int& a, int& b) const {
        a = max(r0, kb * PW);
        b = r1;
    }
    __device__ int nblk() const { return 1; }
    __device__ int width() const { return min(PW, P - kb * PW); }
};
constexpr int kBl1CR = 510;   // rows per coefficient chunk
constexpr int kBl1XS = 512;   // staged rows per vector: the chunk from its even-aligned start (TMA: 16-B aligned)
static_assert(kLabMax * kBl1XS <= CFCH + 2 * RCH, "BL1 coefficient chunk in cf + racc");
__device__ __forceinline__ int64_t bl1_cum(int64_t kb, int64_t n) { return kb * n - (int64_t)PW * (kb * (kb - 1) / 2); }
__device__ __forceinline__ int64_t bl1_bound(int64_t U, int q, int Gt) { return (U * q) / Gt; }
// CTA whose unit range holds unit u
__device__ __forceinline__ int bl1_owner(int64_t U, int64_t u, int Gt) {
    int q = (int)min((int64_t)Gt - 1, (u * Gt) / (U > 0 ? U : 1));
    while (q + 1 < Gt && bl1_bound(U, q + 1, Gt) <= u) q++;
    while (q > 0 && bl1_bound(U, q, Gt) > u) q--;
    return q;
}

template <int NV>
__device__ void lab_bl1_stream(const Smem& sm, const WRing& rg, const double* __restrict__ Y, int64_t m, int64_t n,
                               int64_t k, const double* X, int64_t xst, int nv, double* PB, int q, int Gt,
                               int64_t x0, int64_t x1, double* xsq, uint64_t pol) {
    const int tid = threadIdx.x, tc = tid - 32;
    {   // ||X_v||^2 partials (rows [x0, x1))
        double qq[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) qq[v] = 0.0;
        for (int64_t i = x0 + tid; i < x1; i += NT)
#pragma unroll
            for (int v = 0; v < NV; v++) {
                const double xv = (v < nv) ? ld(X + v * xst + i) : 0.0;
                qq[v] = fma(xv, xv, qq[v]);
            }
#pragma unroll
        for (int v = 0; v < NV; v++) {
            const double t = block_sum<NT>(qq[v], sm.red);
            if (tid == 0) xsq[v] = t;
        }
    }
    const int64_t NB = (k + PW - 1) / PW;
    const int64_t U = bl1_cum(NB, n);
    int64_t u = bl1_bound(U, q, Gt);
    const int64_t ue = bl1_bound(U, q + 1, Gt);
    double* xs = sm.cf;   // [v][kBl1XS] (cf and racc are contiguous)
    while (u < ue) {
        // segment: block kb, rows [ra, rb)
        int64_t kb = 0;
        while (kb + 1 < NB && bl1_cum(kb + 1, n) <= u) kb++;
        const int64_t blk_end = bl1_cum(kb + 1, n);
        const int64_t ra = kb * PW + (u - bl1_cum(kb, n));
        const int64_t rb = ra + ((ue < blk_end ? ue : blk_end) - u);
        const int gc = (int)kb * PW + 2 * tc;   // this consumer's first column
        double acc[NV][2];
#pragma unroll
        for (int v = 0; v < NV; v++) acc[v][0] = acc[v][1] = 0.0;
        int cb = 0;
        const SrcYB src{Y, (int)m, (int)k, (int)kb};
        const int PST = wide_pst(src);
        wide_stream<kBl1CR>(
            rg, src, (int)ra, (int)rb, false, pol,
            [&](int c0, int c1) {
                cb = c0 & ~1;
                tma_stage(sm, nv, [&](int v) { return X + v * xst + cb; }, c1 - cb, xs, kBl1XS);
                for (int t = tid; t < (NV - nv) * kBl1XS; t += NT) xs[nv * kBl1XS + t] = 0.0;
                __syncthreads();
            },
            [&](int, int, int) {},
            [&](int, int sa, int sb, const double* slot) {
                if (2 * tc >= PST) return;
                // every row of the stage covers the whole (full-width) block: no masks
                const bool full = (sa >= (int)kb * PW + PW - 1) && ((int)kb * PW + PW <= (int)k);
                for (int qr = 0; qr < sb - sa; qr++) {
                    const int i = sa + qr;
                    const double2 y = *reinterpret_cast<const double2*>(slot + qr * PST + 2 * tc);
                    double y0 = y.x, y1 = y.y;
                    if (!full) {
                        y0 = (gc <= i && gc < (int)k) ? y0 : 0.0;
                        y1 = (gc + 1 <= i && gc + 1 < (int)k) ? y1 : 0.0;
                    }
                    const double* xr = xs + (i - cb);
#pragma unroll
                    for (int v = 0; v < NV; v++) {
                        const double xv = xr[v * kBl1XS];
                        acc[v][0] = fma(y0, xv, acc[v][0]);
                        acc[v][1] = fma(y1, xv, acc[v][1]);
                    }
                }
            },
            [&](int) {}, [&](int, int) {});
        if (tc >= 0) {
            double* slotp = PB + (kb + q) * (int64_t)(NV * PW);
#pragma unroll
            for (int v = 0; v < NV; v++)
                *reinterpret_cast<double2*>(slotp + v * PW + 2 * tc) = make_double2(acc[v][0], acc[v][1]);
        }
        u += rb - ra;
    }
}

// G[v][c] (ldg) for this CTA's columns: the slots of c's block summed in CTA order
template <int NV>
__device__ void lab_bl1_reduce(const double* PB, int64_t k, int64_t n, int q, int Gt, int nv, double* G, int64_t ldg) {
    const int64_t NB = (k + PW - 1) / PW;
    const int64_t U = bl1_cum(NB, n);
    int64_t c0, c1;
    part_uniform(0, k, q, Gt, c0, c1);
    for (int64_t t = threadIdx.x; t < (c1 - c0) * nv; t += NT) {
        const int v = (int)(t / (c1 - c0));
        const int64_t c = c0 + t % (c1 - c0);
        const int64_t kb = c / PW, lc = c - kb * PW;
        const int qa = bl1_owner(U, bl1_cum(kb, n), Gt), qb = bl1_owner(U, bl1_cum(kb + 1, n) - 1, Gt);
        double sum = 0.0;
        for (int r = qa; r <= qb; r++) {
            if (bl1_bound(U, r + 1, Gt) <= bl1_bound(U, r, Gt)) continue;   // empty range
            sum += ld(PB + (kb + r) * (int64_t)(NV * PW) + v * PW + lc);
        }
        st(G + v * ldg + c, sum);
    }
}

// BL2 / BL3: out_v[r] = base_v(r) - sum_{k in row r} row_r[k] V_v[k] for rows [r0, r1) (warp per
// row, vectors V staged in shared memory by chunks of CC columns, per-row sums in shared memory).
//   BL2: rows l of column-packed T (T[0..l][l]), V = G, base = 0       -> G'
//   BL3: rows i of Y_k (columns 0..k-1),          V = G', base = X_v[i] -> U
template <int NV, class RowPtr, class RowLen, class Epi>
__device__ void lab_rowdots(const Smem& sm, int64_t r0, int64_t r1, int64_t P, const double* V, int64_t ldv, int nv,
                            double* scr, RowPtr rowptr, RowLen rowlen, Epi epi) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int CC = 1024;                    // staged columns per chunk (NV * CC <= 8192)
    double* vs = scr;
    double* acc = scr + 8192;                   // [row - r0][NV]
    const int64_t R = r1 - r0;
    if (R <= 0) return;
    for (int64_t rb0 = r0; rb0 < r1; rb0 += 4096 / NV) {   // row blocks whose sums fit `acc`
        const int64_t rb1 = (rb0 + 4096 / NV < r1) ? rb0 + 4096 / NV : r1;
        for (int64_t q = tid; q < (rb1 - rb0) * NV; q += NT) acc[q] = 0.0;
        int64_t lmax = 0;   // the longest row of the block: no chunk beyond it is staged
        for (int64_t r = rb0; r < rb1; r++) lmax = max(lmax, rowlen(r));
        const int64_t Pc = (lmax < P) ? lmax : P;
        for (int64_t c0 = 0; c0 < Pc; c0 += CC) {
            const int64_t c1 = (c0 + CC < Pc) ? c0 + CC : Pc;
            // the nv vectors' columns [c0, c1) by TMA; vectors >= nv: zero
            tma_stage(sm, nv, [&](int v) { return V + v * ldv + c0; }, c1 - c0, vs, CC);
            for (int64_t q = tid; q < (int64_t)(NV - nv) * CC; q += NT) vs[(int64_t)nv * CC + q] = 0.0;
            __syncthreads();
            for (int64_t r = rb0 + warp; r < rb1; r += NW) {
                const int64_t len = rowlen(r);
                if (len <= c0) continue;
                const int64_t e1 = (len < c1) ? len : c1;
                const double* row = rowptr(r);
                double a[NV];
#pragma unroll
                for (int v = 0; v < NV; v++) a[v] = 0.0;
                constexpr int U = 8;   // (16 in flight per lane measured slower: first-iteration GEMMs 297 -> 355 ms on cfg4)
                for (int64_t k0 = c0 + 2 * lane; k0 < e1; k0 += 64 * U) {
                    double2 y[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int64_t k = k0 + 64 * u;
                        y[u] = (k < e1) ? ld2(row + k) : make_double2(0.0, 0.0);
                        if (k + 1 >= e1) y[u].y = 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int64_t k = k0 + 64 * u - c0;
                        if (k0 + 64 * u < e1) {
#pragma unroll
                            for (int v = 0; v < NV; v++) {
                                const double2 g = *reinterpret_cast<const double2*>(vs + v * CC + k);
                                a[v] = fma(y[u].x, g.x, a[v]);
                                a[v] = fma(y[u].y, g.y, a[v]);
                            }
                        }
                    }
                }
                if (NV == 8) {
                    // 8 warp sums at once: halve the values held per lane at each xor step (9
                    // shuffles instead of 40); lane L ends with the total of vector (L >> 2) & 7
                    // summed over its four-lane group, fixed order (deterministic)
#pragma unroll
                    for (int h = 0; h < 4; h++) {
                        const bool up = lane & 16;
                        const double send = up ? a[h] : a[h + 4];
                        const double keep = up ? a[h + 4] : a[h];
                        a[h] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                    }
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const bool up = lane & 8;
                        const double send = up ? a[h] : a[h + 2];
                        const double keep = up ? a[h + 2] : a[h];
                        a[h] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                    }
                    {
                        const bool up = lane & 4;
                        const double send = up ? a[0] : a[1];
                        const double keep = up ? a[1] : a[0];
                        a[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                    }
                    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
                    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
                    // lane bits 4,3,2 chose the upper halves: vector index = 4 b16 + 2 b8 + b4
                    if ((lane & 3) == 0) {
                        const int v = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                        acc[(r - rb0) * NV + v] += a[0];
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < NV; v++) {
                        const double t = warp_sum(a[v]);
                        if (lane == 0) acc[(r - rb0) * NV + v] += t;
                    }
                }
            }
        }
        __syncthreads();
        for (int64_t q = tid; q < (rb1 - rb0) * NV; q += NT) epi(rb0 + q / NV, (int)(q % NV), acc[q]);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- fused pass A2, column-owner form
// Pass A of iteration 2 (g = Y_p^T x) streamed behind the back sweep band by band.  Each of the
// Gl = G - 1 streaming CTAs owns one column block kb of Y_p (CTAs per block in proportion to
// the block's elements, at least one) and, in every band, an even share of the band's rows that
// reach the block; its 448 column sums stay in registers across all bands (no global
// read-modify-write per band and block) and are written once.  R1 then adds the few partials of
// each block in CTA order.  Needs NB <= Gl blocks.
__device__ __forceinline__ int64_t a2c_work(int64_t kb, int64_t n, int64_t P) {
    return (n - kb * PW) * (int64_t)min((int64_t)PW, P - kb * PW);
}
// first streaming CTA (0-based among the Gl) of every block: st[kb], kb = 0..NB (st[NB] = Gl),
// written by thread 0 into shared memory (the caller synchronises)
__device__ __forceinline__ void a2c_table(int64_t n, int64_t P, int Gl, int* st) {
    const int64_t NB = (P + PW - 1) / PW;
    // elements of blocks [0, b) for b <= NB - 1 (full-width blocks): PW (b n - PW b (b-1) / 2)
    auto cw = [&](int64_t b) -> int64_t { return (int64_t)PW * (b * n - (int64_t)PW * (b * (b - 1) / 2)); };
    const int64_t W = cw(NB - 1) + a2c_work(NB - 1, n, P);
    for (int64_t b = threadIdx.x; b <= NB; b += NT)
        st[b] = (b == NB) ? Gl : (int)(b + ((int64_t)(Gl - NB) * cw(b)) / W);
}
__device__ __forceinline__ void a2c_assign(int64_t P, const int* st, int rl, int& kb, int& j, int& cnt) {
    const int64_t NB = (P + PW - 1) / PW;
    kb = 0;
    while (kb + 1 < NB && st[kb + 1] <= rl) kb++;
    j = rl - st[kb];
    cnt = st[kb + 1] - st[kb];
}
// rows [i0, i1) of block kb of Y_P against coefficients x: a0, a1 (+=) for the consumer's columns
// 2t', 2t'+1 of the block; x2 (+=) the coefficients' squares when want_x2
__device__ void a2c_stream(const Smem& sm, const WRing& rg, const double* __restrict__ Y, int64_t m, int64_t P,
                           int kb, int i0, int i1, const double* x, double& a0, double& a1, double& x2, bool want_x2,
                           uint64_t pol) {
    const int tid = threadIdx.x, tc = tid - 32;
    const SrcYB src{Y, (int)m, (int)P, kb};
    const int PST = wide_pst(src);
    const int gc = kb * PW + 2 * tc;
    int cb = 0;
    wide_stream(
        rg, src, i0, i1, false, pol,
        [&](int c0, int c1) {
            cb = c0;
            for (int r = c0 + tid; r < c1; r += NT) {
                const double c = ld(x + r);
                sm.cf[r - c0] = c;
                if (want_x2) x2 = fma(c, c, x2);
            }
            __syncthreads();
        },
        [&](int, int, int) {},
        [&](int, int sa, int sb, const double* slot) {
            if (2 * tc >= PST) return;
            const bool full = (sa >= kb * PW + PW - 1) && (kb * PW + PW <= (int)P);
            const double* sp = slot + 2 * tc;
            const double* cp = sm.cf + (sa - cb);
            if (full) {
#pragma unroll 7
                for (int q = 0; q < sb - sa; q++) {
                    const double2 y = *reinterpret_cast<const double2*>(sp + q * PST);
                    const double c = cp[q];
                    a0 = fma(y.x, c, a0);
                    a1 = fma(y.y, c, a1);
                }
            } else {
                for (int q = 0; q < sb - sa; q++) {
                    const int i = sa + q;
                    const double2 y = *reinterpret_cast<const double2*>(sp + q * PST);
                    const double c = cp[q];
                    const double y0 = (gc <= i && gc < (int)P) ? y.x : 0.0;
                    const double y1 = (gc + 1 <= i && gc + 1 < (int)P) ? y.y : 0.0;
                    a0 = fma(y0, c, a0);
                    a1 = fma(y1, c, a1);
                }
            }
        },
        [&](int) {}, [&](int, int) {});
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(NT, 1) cwy_kernel(CwyArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem sm;
    {
        sm.vs = reinterpret_cast<double*>(smem_raw);
        sm.cf = sm.vs + kVsD;
        sm.racc = sm.cf + CFCH;
        sm.vblk = sm.racc + 2 * RCH;
        sm.acc = reinterpret_cast<double2*>(sm.vblk + 4 * PW);
        sm.red = reinterpret_cast<double*>(sm.acc + NT);
        sm.mbar = reinterpret_cast<uint64_t*>(sm.red + NW + 8);
    }
    // mbarriers: [0, kRing) back sweep, [kRing, +kNStg) narrow ring, then wide full, wide
    // empty, vector double buffer; vuse counters after them
    uint64_t* wfull = sm.mbar + kRing + kNStg;
    uint64_t* wempty = wfull + kWStg;
    sm.vbar = wempty + kWStg;
    sm.vuse = reinterpret_cast<uint32_t*>(sm.vbar + 2);
    double* ring_base = reinterpret_cast<double*>(sm.mbar + kNBar);   // 16-B aligned (see cwy_smem_bytes)
    // the back-sweep ring sits after the narrow ring (the single-CTA look-ahead streams the
    // narrow ring while the back sweep runs) and aliases the wide ring (never in use together)
    sm.bring = ring_base + (int64_t)kNStg * kStgD;
    sm.rbuf = ring_base;
    sm.rbar = sm.mbar + 26;
    sm.rcnt = reinterpret_cast<uint32_t*>(sm.mbar + 25);
    if (threadIdx.x == 0) {
        for (int k = 0; k < kRing + kNStg; k++) mbar_init(sm.mbar + k, 1);
        for (int k = 0; k < kWStg; k++) {
            mbar_init(wfull + k, 1);
            mbar_init(wempty + k, NCW);
        }
        mbar_init(sm.vbar, 1);
        mbar_init(sm.vbar + 1, 1);
        sm.vuse[0] = sm.vuse[1] = 0;
        mbar_init(sm.mbar + 26, 1);
        for (int k = 0; k < 2; k++) {
            mbar_init(sm.mbar + kXFull + k, 1);
            mbar_init(sm.mbar + kXEmpty + k, 1);
        }
        *reinterpret_cast<uint32_t*>(sm.mbar + 25) = 0;
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t mbph = 0;   // back-sweep ring phase bits (thread 0)
    uint32_t xseq = 0;   // chunks of the two-thread back sweeps so far (threads 0 and 32 of CTA 0)
    uint32_t rph = 0;    // pass ring phase bits (every thread)
    // pass timers (whole launch, not windowed): the first consumer thread of the first
    // group's first CTA (+ prof_sel)
    const bool timing0 = (a.prof != nullptr) && threadIdx.x == 32 && (int)blockIdx.x == a.g_cta0[0] + a.prof_sel;
    uint64_t ntim[4] = {0, 0, 0, 0};
    // debug build: SM-clock sub-timers of the reductions on thread 0 of the timed CTA (replace
    // the stream timers in prof slots 12-15: R1 partials, R1 rest, R2 scalars, R2 partials)
    const bool dsub = kWideDebug && (a.prof != nullptr) && threadIdx.x == 0 && (int)blockIdx.x == a.g_cta0[0] + a.prof_sel;
    uint64_t dtim[4] = {0, 0, 0, 0};
    uint64_t dA = 0;   // debug (TINV_DBG bit 1): SM clock at the exit of pass A's barrier
    auto dclk = [&]() -> uint64_t { return dsub ? (uint64_t)clock64() : 0; };
    const Ring rg{ring_base, sm.mbar + kRing, &rph, timing0 ? ntim : nullptr};
    uint32_t wiss = 0, wuse = 0;   // wide ring stage counters (issued: warp 0; used: all)
    const WRing wr{ring_base, wfull, wempty, &wiss, &wuse, timing0 ? ntim : nullptr};
    const int tid = threadIdx.x;
    const uint64_t pol_first = l2_policy_evict_first(), pol_norm = l2_policy_evict_normal();
    int g = 0;
    for (int t = 0; t < a.ngroups; t++)
        if ((int)blockIdx.x >= a.g_cta0[t]) g = t;
    const int r = blockIdx.x - a.g_cta0[g];
    const int G = a.g_size[g];
    if (r >= G) return;  // CTA not used by any group
    const GroupWS ws = a.ws[g];
    // row split over ranks: this CTA is cg of Gt = nrk G CTAs; work split
    // over the group uses (cg, Gt), replicated local work uses (r, G)
    const int NR = ws.nrk, RK = ws.rk;
    const int Gt = NR * G, cg = RK * G + r;
    const Ranks rks{NR, G, ws.delta};
    const bool own_out = !(ws.vrt && RK != 0);   // virtual ranks share the caller's outputs
    long long nsync = 0;
    unsigned int bar_epoch = 0;
    // debug (TINV_PROF_CTA): this CTA's busy time before each barrier, attributed to the
    // phase that the next mark() closes
    const bool ctime = kWideDebug && (a.prof_cta != nullptr) && tid == 0;
    uint64_t c_last = ctime ? gtime() : 0, c_busy = 0;
    auto gsync = [&]() {
        if (ctime) c_busy += gtime() - c_last;
        if (NR == 1) group_sync(ws.bar, G, bar_epoch);
        else group_sync_ranks(ws.bar, ws.delta, NR, Gt, bar_epoch);
        nsync++;
        if (ctime) c_last = gtime();
    };
    // mirrored store: every rank's replica of the group workspace
    auto mst = [&](double* ptr, double v) {
        if (NR == 1) st(ptr, v);
        else
            for (int k = 0; k < NR; k++) st(ptr + __ldg(ws.delta + k), v);
    };
    // optional phase timers (thread 0 of each group's first CTA; globaltimer ns)
    const bool timing = (a.prof != nullptr) && r == 0 && tid == 0;
    uint64_t tacc[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    uint64_t tmark = timing ? gtime() : 0;
    bool inwin = true;   // the current vector is inside the timed window [prof_p0, prof_p1)
    auto mark = [&](int k) {
        if (ctime) {
            if (inwin) a.prof_cta[(int64_t)blockIdx.x * 16 + k] += c_busy;
            c_busy = 0;
        }
        if (timing) {
            uint64_t _t = gtime();
            if (inwin) tacc[k] += _t - tmark;
            tmark = _t;
        }
    };
#define PH(k) mark(k)

    const int64_t n = a.n;
    const int64_t n2v = (n + 1) & ~int64_t(1);   // vector stride of X1c
    // reorthogonalisation (tinv_set_reorth): 0 the reduced compact-WY step of §3.3.2, 1 classical
    // MGS (Alg. 1; single-rank groups), 2 the ordinary compact-WY sequence of
    // §3.3.1 (Y^T y by a pass of its own)
    const int mode = a.reorth;
    const double thr = sqrt(0.1 / (double)n);
    double* __restrict__ Y = ws.Y;
    double* __restrict__ S = ws.S;
    double* __restrict__ P_ = ws.P;
    const int64_t mc = ws.mcap;

    for (int ci = a.g_coff[g]; ci < a.g_coff[g + 1]; ci++) {
        const int cl = a.g_clist[ci];
        const int64_t j1 = a.cstart[cl];
        const int64_t m = a.cstart[cl + 1] - j1;
        const int64_t m2 = (m + 1) & ~int64_t(1);
        const bool narrow = (m <= kNarrowM) && a.nstg > 0;
        const bool la_ok = ((G > 1) || narrow) && mode != 1;   // look-ahead can overlap the back sweep
        // deferred final pass D: wide clusters that are their group's last (Y stays intact after
        // the kernel), single-rank groups
        const bool dz_cl = a.dzc != nullptr && mode != 1 && NR == 1 && !narrow && m > kNarrowM + 1 &&
                           ci == a.g_coff[g + 1] - 1;
        double* __restrict__ Tc = ws.Tc;
        double* __restrict__ Tr = ws.Tr;

        // ================= first reflector from the accepted z_{j1} (p = 0)
        if (mode != 1) {
            const double* z = a.Z + j1 * a.ldz;
            int64_t i0, i1;
            part_uniform(0, n, r, G, i0, i1);
            double u2 = 0.0;
            for (int64_t i = i0 + tid; i < i1; i += NT) {
                const double zi = ld(z + i);
                st(ws.u + i, zi);
                u2 = fma(zi, zi, u2);
            }
            u2 = block_sum<NT>(u2, sm.red);
            if (tid == 0) st(S + cg * SST + SSlots::U2, u2);   // this rank's slots only (replicated work)
            gsync();
            const double un = sqrt(reduce_slot(sm, S + RK * G * SST, G, SSlots::U2));
            const double u0 = ld(ws.u);
            const double c = -((u0 >= 0.0) ? 1.0 : -1.0) * un;
            const double tt = 1.0 / (c * c - u0 * c);
            for (int64_t i = i0 + tid; i < i1; i += NT)
                st(Y + y_row_off(i, m), (i == 0) ? (u0 - c) : ld(ws.u + i));
            if (r == 0 && tid == 0) { st(Tc + tcol_off(0), tt); st(Tr, tt); }
            gsync();
            PH(0);
        }

        // ================= vectors j_c = 1 .. m-1
        bool la_have = false;   // look-ahead of this vector's first pass A is ready
        // blocked look-ahead: vectors p >= kNarrowM + 1 form blocks of a.lab
        const bool lab_cl = a.lab > 1 && ws.labU != nullptr && mode != 1 && NR == 1 && !narrow && m > kNarrowM + 1;
        constexpr int64_t kLab0 = kNarrowM + 1;
        auto in_lab = [&](int64_t q) { return lab_cl && q >= kLab0; };
        int64_t lab_k = 0;   // start of the current block
        bool lab_fused = false;   // in-block dots of this block come from the earlier vectors' BC passes
        unsigned int* sw_prog = reinterpret_cast<unsigned int*>(S + (int64_t)Gt * SST);   // sweep bands
        unsigned int sw_ep = 0;   // fused sweeps so far in this cluster (the progress tag's epoch)
        if (r == 0 && tid == 0) publish(sw_prog, 0u);   // visible after the next group barrier
        for (int64_t p = 1; p < m; p++) {
            const int64_t j = j1 + p;
            inwin = !kWideDebug || (p >= a.prof_p0 && p < a.prof_p1);
            const double* xcur = a.X1c + j * n2v;   // x^(1), contiguous copy
            int64_t xs = 1;
            int its = 1, kin = 1, passes = 0, restart = 0;
            bool done = false, flagged = false;
            bool use_la = la_have;           // first iteration: A already done in look-ahead
            bool use_a2 = false;             // pass A of this iteration fused behind the back sweep
            bool use_a2c = false;            // ... in the column-owner form (partials per column block)
            bool tyr_have = false;           // T_p yrow of this vector in ws.tyr (this CTA's TN rows)
            bool la_done = false;            // look-ahead for vector p+1 issued
            la_have = false;
            // L2 policy of the streams: once Y_p no longer fits a share of L2, the passes that read
            // their operand once stream it evict_first (the partial sums, vectors and BC's re-read
            // stay in L2); BC's first read of Yhat keeps the normal priority for its second read
            const bool ybig = 8.0 * (double)y_row_off(n, p + 1 < m ? p + 1 : m) > kL2KeepBytes;
            const uint64_t pol_once = ybig ? pol_first : pol_norm, pol_keep = pol_norm;
            // this CTA's share of every pass of vector p (the same in each iteration)
            int64_t pa0, pa1, ptt0, ptt1, ptn0, ptn1, pd0, pd1;
            part_rows_weighted(n, p, cg, Gt, pa0, pa1, a.piece_cost);
            part_tt(p, cg, Gt, ptt0, ptt1, a.piece_cost);
            part_tn(p, cg, Gt, ptn0, ptn1, a.piece_cost);
            part_rows_weighted(n, p + 1, cg, Gt, pd0, pd1, a.piece_cost, a.cta0_pm);
            bool use_lab = in_lab(p);   // first iteration from the block's U (no pass A, TT or BC rows)
            if (use_lab && (p - kLab0) % a.lab == 0) {
                // ---------------- BL1-BL3: U = X - Y_k T_k^T Y_k^T X for x^(1)_k .. x^(1)_{k+nv-1}
                lab_k = p;
                lab_fused = a.labq != 0;
                const int nv = (int)((m - p < a.lab) ? m - p : a.lab);
                const double* Xb = a.X1c + j * n2v;
                double* scr = ring_base;   // no pass ring in flight between phases
                int64_t c0, c1, x0, x1;
                part_cols_tri(p, n, cg, Gt, c0, c1);
                part_uniform(0, n, cg, Gt, x0, x1);
                if (ws.labPB != nullptr) {
                    lab_bl1_stream<kLabMax>(sm, wr, Y, m, n, p, Xb, n2v, nv, ws.labPB, cg, Gt, x0, x1,
                                            ws.labP + (int64_t)cg * kLabMax, pol_once);
                    gsync();
                    lab_bl1_reduce<kLabMax>(ws.labPB, p, n, cg, Gt, nv, ws.labG, mc);
                } else {
                    lab_gemm1<kLabMax>(sm, Y, m, n, c0, c1, Xb, n2v, nv, ws.labG, mc, scr, x0, x1, ws.labP + (int64_t)cg * kLabMax);
                }
                gsync();
                if (kWideDebug && (a.dbg & 16)) mark(12);   // debug: BL1 / BL2 in slots 12 / 13
                if (r == 0 && tid < nv) {   // ||x_v||^2 for the degeneracy test (reading 16)
                    double t = 0.0;
                    for (int q = 0; q < Gt; q++) t += ld(ws.labP + (int64_t)q * kLabMax + tid);
                    st(ws.labX2 + tid, t);
                }
                int64_t l0, l1;
                part_tt(p, cg, Gt, l0, l1, 0);
                lab_rowdots<kLabMax>(sm, l0, l1, p, ws.labG, mc, nv, scr, [&](int64_t l) { return Tc + tcol_off(l); },
                                     [&](int64_t l) -> int64_t { return l + 1; },
                                     [&](int64_t l, int v, double t) { if (v < nv) st(ws.labGp + v * mc + l, t); });
                gsync();
                if (kWideDebug && (a.dbg & 16)) mark(13);
                int64_t i0, i1;
                part_uniform(p, n, cg, Gt, i0, i1);
                lab_rowdots<kLabMax>(sm, i0, i1, p, ws.labGp, mc, nv, scr, [&](int64_t i) { return Y + y_row_off(i, m); },
                                     [&](int64_t) -> int64_t { return p; },
                                     [&](int64_t i, int v, double t) {
                                         if (v < nv) st(ws.labU + v * n2v + i, ld(Xb + v * n2v + i) - t);
                                     });
                gsync();
                PH(0);
            }
            while (!done) {
                double c = 1.0;   // the reflector's c (reduced / ordinary); 1 for MGS (r = q)
                int64_t dq0 = pd0, dq1 = pd1;   // rows of q that this CTA holds after the step
                if (mode == 1) {
                    // ---------------- MGS (Alg. 1 l.10-12): x <- x - <x, z_i> z_i
                    // for the cluster's accepted z_{j1} .. z_{j-1} in order; one group barrier per
                    // z_i (the O(m) synchronisations per vector of Table 1).  The
                    // partial dot of z_{i+1} is fused into the update with z_i; slots MG0/MG1
                    // alternate so a fast CTA never overwrites a partial still being summed.
                    part_uniform(0, n, cg, Gt, dq0, dq1);
                    const int R = (int)(dq1 - dq0);
                    double* xv = (R <= CFCH) ? sm.cf : ws.q + dq0;   // this CTA's rows of x
                    double x2 = 0.0, dp = 0.0;
                    const double* z0 = a.Z + j1 * a.ldz + dq0;
                    for (int q = tid; q < R; q += NT) {
                        const double xi = ld(xcur + (dq0 + q) * xs);
                        xv[q] = xi;
                        x2 = fma(xi, xi, x2);
                        dp = fma(xi, ld(z0 + q), dp);
                    }
                    x2 = block_sum<NT>(x2, sm.red);
                    dp = block_sum<NT>(dp, sm.red);
                    if (tid == 0) {
                        st(S + cg * SST + SSlots::X2, x2);
                        st(S + cg * SST + SSlots::MG0, dp);
                    }
                    for (int64_t i = 0; i < p; i++) {
                        gsync();
                        const double dot = reduce_slot(sm, S, Gt, (i & 1) ? SSlots::MG1 : SSlots::MG0);
                        const double* zi = a.Z + (j1 + i) * a.ldz + dq0;
                        const double* zn = a.Z + (j1 + i + 1) * a.ldz + dq0;
                        const bool nxt = i + 1 < p;
                        double dn = 0.0;
                        for (int q = tid; q < R; q += NT) {
                            const double xi = fma(-dot, ld(zi + q), xv[q]);
                            xv[q] = xi;
                            if (nxt) dn = fma(xi, ld(zn + q), dn);
                        }
                        if (nxt) {
                            dn = block_sum<NT>(dn, sm.red);
                            if (tid == 0) st(S + cg * SST + ((i & 1) ? SSlots::MG0 : SSlots::MG1), dn);
                        }
                    }
                    if (xv == sm.cf)
                        for (int q = tid; q < R; q += NT) st(ws.q + dq0 + q, xv[q]);
                    __syncthreads();
                    PH(4);
                } else {
                if (use_lab) {
                    // ---------------- block vector, iteration 1: x' = U_v = Q_k^T x^(1)_p; apply the
                    // block's own reflectors k .. p-1:  g_r = Y_{k:p}^T x',  g'_r = T_kk^T g_r (the
                    // trailing block of T_p),  uhat = rows >= p of x' - Y_{k:p} g'_r  (Eq. (4))
                    const int v = (int)(p - lab_k);
                    const double* Uv = ws.labU + v * n2v;
                    double* gr = sm.vs;          // g_r   (<= kLabMax)
                    double* grp = sm.vs + 16;    // g'_r
                    if (v > 0 && lab_fused) {
                        // g_r[q] = y0_{k+q} U_v[k+q] + sum_{i > k+q} uhat_{k+q}[i] U_v[i]: the sums were
                        // accumulated per CTA by the BC pass of vector k+q (labQ[cta][v][q]); no pass here
                        const int q = tid >> 5, lane = tid & 31;
                        if (q < v) {
                            double t = 0.0;
                            for (int u = lane; u < Gt; u += 32) t += ld(ws.labQ + ((int64_t)u * kLabMax + v) * kLabMax + q);
                            t = warp_sum(t);
                            if (lane == 0) gr[q] = fma(ld(ws.labY0 + q), ld(Uv + lab_k + q), t);
                        }
                        __syncthreads();
                        if (tid < v) {
                            const int64_t l = lab_k + tid;
                            const double* tc = Tc + tcol_off(l) + lab_k;
                            double t = 0.0;
                            for (int q2 = 0; q2 <= tid; q2++) t = fma(ld(tc + q2), gr[q2], t);
                            grp[tid] = t;
                        }
                        __syncthreads();
                        PH(1);
                    } else if (v > 0) {
                        int64_t i0, i1;
                        part_uniform(lab_k, n, cg, Gt, i0, i1);
                        double av[kLabMax];
#pragma unroll
                        for (int q = 0; q < kLabMax; q++) av[q] = 0.0;
                        for (int64_t i = i0 + tid; i < i1; i += NT) {
                            const double ui = ld(Uv + i);
                            const double* yr = Y + y_row_off(i, m) + lab_k;
#pragma unroll
                            for (int q = 0; q < kLabMax; q++)
                                if (q < v && lab_k + q <= i) av[q] = fma(ld(yr + q), ui, av[q]);
                        }
#pragma unroll
                        for (int q = 0; q < kLabMax; q++) {
                            if (q >= v) break;
                            const double t = block_sum<NT>(av[q], sm.red);
                            if (tid == 0) st(P_ + (int64_t)cg * mc + q, t);
                        }
                        gsync();
                        PH(1);
                        {   // every CTA: g_r (fixed order: lane-strided partials, warp tree), then T_kk^T g_r
                            const int q = tid >> 5, lane = tid & 31;
                            if (q < v) {
                                double t = 0.0;
                                for (int u = lane; u < Gt; u += 32) t += ld(P_ + (int64_t)u * mc + q);
                                t = warp_sum(t);
                                if (lane == 0) gr[q] = t;
                            }
                            __syncthreads();
                            if (tid < v) {
                                const int64_t l = lab_k + tid;
                                const double* tc = Tc + tcol_off(l) + lab_k;
                                double t = 0.0;
                                for (int q2 = 0; q2 <= tid; q2++) t = fma(ld(tc + q2), gr[q2], t);
                                grp[tid] = t;
                            }
                            __syncthreads();
                        }
                    }
                    int64_t i0, i1;
                    part_uniform(p, n, cg, Gt, i0, i1);
                    double u2 = 0.0;
                    for (int64_t i = i0 + tid; i < i1; i += NT) {
                        double ui = ld(Uv + i);
                        const double* yr = Y + y_row_off(i, m) + lab_k;
                        for (int q = 0; q < v; q++) ui = fma(-ld(yr + q), grp[q], ui);
                        mst(ws.u + i, ui);
                        u2 = fma(ui, ui, u2);
                    }
                    u2 = block_sum<NT>(u2, sm.red);
                    if (tid == 0) mst(S + cg * SST + SSlots::U2, u2);
                    if (mode != 2)   // s' = Yhat^T uhat (one read of Yhat)
                        wide_colacc(sm, wr, SrcY{Y, (int)m, (int)p}, (int)i0, (int)i1, ws.u, p, P_ + (int64_t)cg * mc, false, pol_once);
                    gsync();
                    PH(4);
                } else {
                if (!use_la && !use_a2) {
                    // ---------------- A: partial g = Y_p^T x, ||x||^2
                    {
                        int64_t i0, i1;
                        i0 = pa0; i1 = pa1;
                        double x2 = 0.0;
                        if (narrow) {
                            const int CPT = pow2ceil((int)((p + 1) / 2));
                            double a0 = 0.0, a1 = 0.0;
                            narrow_stream(rg, Y, (int)m2, (int)i0, (int)i1, xcur, [&](int ra, int rb, const double* Ys, double* Xs) {
                                for (int ii = tid; ii < rb - ra; ii += NT) x2 = fma(Xs[ii], Xs[ii], x2);
                                narrow_colacc(ra, rb, (int)m2, Ys, Xs, CPT, [&](int i) -> int { return i + 1 < p ? i + 1 : (int)p; }, a0, a1);
                            });
                            narrow_colacc_finish(sm, CPT, p, a0, a1, P_ + (int64_t)cg * mc);
                        } else if (p > kNarrowM) {
                            x2 = wide_colacc(sm, wr, SrcY{Y, (int)m, (int)p}, (int)i0, (int)i1, xcur, p, P_ + (int64_t)cg * mc, false, pol_once);
                        } else {
                            x2 = colacc(sm, Y, m, i0, i1, p, xcur, xs, P_ + (int64_t)cg * mc);
                        }
                        x2 = block_sum<NT>(x2, sm.red);
                        if (tid == 0) mst(S + cg * SST + SSlots::X2, x2);
                    }
                    gsync();
                    if (kWideDebug && (a.dbg & 2)) dA = dclk();
                    PH(1);
                }
                // ---------------- R1: g = sum_r partials (look-ahead: columns < p from the
                // partials of Y_{p}^T x computed during the previous vector's solve, column p-1
                // from the previous vector's last pass D)
                {
                    int64_t k0, k1;
                    const uint64_t q0 = dclk();
                    if (use_la) {
                        part_uniform(0, p - 1, cg, Gt, k0, k1);
                        reduce_partials(sm, ws.P2, mc, Gt, k0, k1, [&](int64_t k, double v) { mst(ws.g + k, v); }, rks);
                        const uint64_t q1 = dclk();
                        const bool dla = dsub && !(a.dbg & 11);
                        if (dla) dtim[0] += q1 - q0;
                        const double gl = reduce_slot(sm, S, Gt, SSlots::GPN);
                        if (r == 0 && tid == 0) st(ws.g + p - 1, gl);   // every rank, its own replica
                        if (dla) dtim[1] += dclk() - q1;
                    } else if (use_a2c) {
                        // column-owner A2: the partials of column k's block, in CTA order
                        part_uniform(0, p, cg, Gt, k0, k1);
                        int* st_tab = reinterpret_cast<int*>(sm.vs);
                        a2c_table(n, p, G - 1, st_tab);
                        __syncthreads();
                        for (int64_t k = k0 + tid; k < k1; k += NT) {
                            const int64_t kb = k / PW;
                            const int s0 = st_tab[kb], s1 = st_tab[kb + 1];
                            double t = 0.0;
                            for (int q0 = s0; q0 < s1; q0 += 8) {   // 8 independent loads per round trip
                                double v[8];
#pragma unroll
                                for (int u = 0; u < 8; u++) v[u] = (q0 + u < s1) ? ld(P_ + (int64_t)(1 + q0 + u) * mc + k) : 0.0;
#pragma unroll
                                for (int u = 0; u < 8; u++)
                                    if (q0 + u < s1) t += v[u];
                            }
                            st(ws.g + k, t);
                        }
                    } else {
                        part_uniform(0, p, cg, Gt, k0, k1);
                        reduce_partials(sm, P_, mc, Gt, k0, k1, [&](int64_t k, double v) { mst(ws.g + k, v); }, rks);
                        const uint64_t q1 = dclk();
                        if (kWideDebug && (a.dbg & 2)) {   // entry, reduce, rest, an extra barrier (every CTA)
                            __syncthreads();
                            const uint64_t q2 = dclk();
                            gsync();
                            if (dsub && dA) {
                                dtim[0] += q0 - dA;
                                dtim[1] += q1 - q0;
                                dtim[2] += q2 - q1;
                                dtim[3] += dclk() - q2;
                            }
                            dA = 0;
                        } else if (dsub && !(a.dbg & 8)) dtim[0] += q1 - q0;
                        if (kWideDebug && (a.dbg & 1)) {   // experiment: the same reduction again
                            reduce_partials(sm, P_, mc, Gt, k0, k1, [&](int64_t k, double v) { mst(ws.g + k, v); }, rks,
                                            dsub ? dtim + 2 : nullptr);
                            if (dsub) dtim[1] += dclk() - q1;
                        }
                    }
                }
                if (a.pf && p > kNarrowM) pf_first(SrcTc{Tc, (int)p}, (int)ptt0, (int)ptt1, a.pf);
                gsync();
                PH(2);
                // ---------------- TT: g' = T_p^T g
                {
                    int64_t k0, k1;
                    k0 = ptt0; k1 = ptt1;
                    if (p > kNarrowM) {
                        wide_rowdots<false>(sm, wr, SrcTc{Tc, (int)p}, (int)k0, (int)k1, ws.g, nullptr, p, pol_once,
                                            [&](int64_t k, double v, double) { mst(ws.gp + k, v); });
                    } else if (k1 > k0) {
                        stage_vec(sm, ws.g, p);
                        rowdots(k0, k1, p, sm.vs,
                                [&](int64_t k) { return Tc + tcol_off(k); },
                                [&](int64_t k) -> int64_t { return k + 1; },
                                [&](int64_t k, double v) { mst(ws.gp + k, v); });
                    }
                }
                if (a.pf && p > kNarrowM) {
                    int64_t i0, i1;
                    part_uniform(p, n, cg, Gt, i0, i1);
                    pf_first(SrcY{Y, (int)m, (int)p}, (int)i0, (int)i1, a.pf);
                }
                gsync();
                PH(3);
                // ---------------- BC: u^ = x^ - Yhat g' (rows p..n-1), s' partials, ||u^||^2
                {
                    int64_t i0, i1;
                    part_uniform(p, n, cg, Gt, i0, i1);
                    double u2 = 0.0;
                    if (narrow) {
                        // one read of Yhat per stage: row dots -> uhat (into the stage's
                        // coefficient slots), then the column accumulate with uhat
                        const int LPR = pow2ceil((int)((p + 1) / 2));
                        stage_vec(sm, ws.gp, p);
                        double a0 = 0.0, a1 = 0.0;
                        auto lenp = [&](int) -> int { return (int)p; };
                        narrow_stream(rg, Y, (int)m2, (int)i0, (int)i1, xcur, [&](int ra, int rb, const double* Ys, double* Xs) {
                            narrow_rowdots(ra, rb, (int)m2, Ys, sm.vs, lenp, [&](int i, double v) {
                                const double ui = Xs[i - ra] - v;
                                Xs[i - ra] = ui;
                                mst(ws.u + i, ui);
                                u2 = fma(ui, ui, u2);
                            });
                            __syncthreads();
                            narrow_colacc(ra, rb, (int)m2, Ys, Xs, LPR, lenp, a0, a1);
                            fence_proxy_async_smem();   // uhat written into the slot before its next bulk fill
                        });
                        narrow_colacc_finish(sm, LPR, p, a0, a1, P_ + (int64_t)cg * mc);
                        u2 = block_sum<NT>(u2, sm.red);
                        if (tid == 0) mst(S + cg * SST + SSlots::U2, u2);
                    } else if (p > kNarrowM) {
                        // vector p of a look-ahead block: dots of uhat (column p of Y below row p) with
                        // the block's later first iterates U_v, v > p - k (their in-block g_r)
                        const int jq = (int)(p - lab_k);
                        const int nvb = (int)((m - lab_k < a.lab) ? m - lab_k : a.lab);
                        const bool fq = in_lab(p) && lab_fused && jq + 1 < nvb;
                        double lq[kLabMax];
#pragma unroll
                        for (int q = 0; q < kLabMax; q++) lq[q] = 0.0;
                        wide_rowdots<false>(sm, wr, SrcY{Y, (int)m, (int)p}, (int)i0, (int)i1, ws.gp, nullptr, p, pol_keep,
                                            [&](int64_t i, double v, double) {
                                                const double ui = ld(xcur + i) - v;
                                                mst(ws.u + i, ui);
                                                u2 = fma(ui, ui, u2);
                                                if (fq && i > p) {
#pragma unroll
                                                    for (int q = 0; q < kLabMax; q++)
                                                        if (q > jq && q < nvb) lq[q] = fma(ui, ld(ws.labU + q * n2v + i), lq[q]);
                                                }
                                            });
                        if (fq) {   // CTA sums (fixed order: warp tree, then warps in order)
#pragma unroll
                            for (int q = 0; q < kLabMax; q++) lq[q] = warp_sum(lq[q]);
                            __syncthreads();
                            double* wq = reinterpret_cast<double*>(sm.acc);   // [warp][q]
                            if ((tid & 31) == 0)
#pragma unroll
                                for (int q = 0; q < kLabMax; q++) wq[(tid >> 5) * kLabMax + q] = lq[q];
                            __syncthreads();
                            if (tid > jq && tid < nvb) {
                                double t = 0.0;
                                for (int w = 0; w < NW; w++) t += wq[w * kLabMax + tid];
                                st(ws.labQ + ((int64_t)cg * kLabMax + tid) * kLabMax + jq, t);
                            }
                            __syncthreads();
                        }
                        u2 = block_sum<NT>(u2, sm.red);
                        if (tid == 0) mst(S + cg * SST + SSlots::U2, u2);
                        // second read of Yhat, blocks in reverse order (the last ones are in L2);
                        // the ordinary sequence forms Y^T y in a pass of its own after R2
                        if (mode != 2)
                            wide_colacc(sm, wr, SrcY{Y, (int)m, (int)p}, (int)i0, (int)i1, ws.u, p, P_ + (int64_t)cg * mc, true, pol_once);
                    } else {
                        stage_vec(sm, ws.gp, p);
                        rowdots(i0, i1, p, sm.vs,
                                [&](int64_t i) { return Y + y_row_off(i, m); },
                                [&](int64_t i) -> int64_t { return p; },
                                [&](int64_t i, double v) {
                                    const double ui = ld(xcur + i * xs) - v;
                                    mst(ws.u + i, ui);
                                    u2 = fma(ui, ui, u2);
                                });
                        u2 = block_sum<NT>(u2, sm.red);
                        if (tid == 0) mst(S + cg * SST + SSlots::U2, u2);
                        if (mode != 2) colacc(sm, Y, m, i0, i1, p, ws.u, 1, P_ + (int64_t)cg * mc);
                    }
                }
                gsync();
                PH(4);
                }   // block vector / regular first passes
                // ---------------- R2: scalars (every CTA, identical), s = s' - c Y[p,:]
                const uint64_t q2s = dclk();
                double un = sqrt(reduce_slot(sm, S, Gt, SSlots::U2));
                const double x2 = use_lab ? ld(ws.labX2 + (p - lab_k))
                                          : reduce_slot(sm, S, Gt, use_la ? SSlots::X2N : SSlots::X2);
                use_la = false;
                use_a2 = false;
                use_a2c = false;
                use_lab = false;
                double u0 = ld(ws.u + p);
                const bool zero_u = (un == 0.0);   // reading: exactly-zero uhat -> e_1
                if (zero_u) { u0 = 1.0; un = 1.0; }
                // degenerate iterate (reading 16): restart with a fresh start vector
                if (un <= (double)n * kEps * sqrt(x2) && restart < kMaxRestart && !zero_u) {
                    restart++;
                    its++;
                    kin = 1;
                    passes = 0;
                    if (r == 0) cta_solve(a, ws, j, 1, restart, sm, mark, mbph);
                    gsync();
                    PH(10);
                    xcur = ws.x;
                    xs = 1;
                    continue;
                }
                if (un <= (double)n * kEps * sqrt(x2)) flagged = true;
                c = -((u0 >= 0.0) ? 1.0 : -1.0) * un;
                const double tt = 1.0 / (c * c - u0 * c);
                const double y0 = u0 - c;
                if (in_lab(p)) {   // y_0 of this block vector (the last iteration's stays), fused dots void on zero uhat
                    if (r == 0 && tid == 0) st(ws.labY0 + (p - lab_k), y0);
                    if (zero_u) lab_fused = false;
                }
                const double* yrow = Y + y_row_off(p, m);
                const uint64_t q2m = dclk();
                if (dsub && !(a.dbg & 11)) dtim[2] += q2m - q2s;
                if (mode == 2) {
                    // ordinary sequence (§3.3.1): s = Y_p^T y_p by a pass of its
                    // own over rows p..n-1 (y_p = uhat with its first entry y_0), then reduced
                    int64_t i0, i1, k0, k1;
                    part_uniform(p, n, cg, Gt, i0, i1);
                    if (p > kNarrowM)
                        wide_colacc(sm, wr, SrcY{Y, (int)m, (int)p}, (int)i0, (int)i1, ws.u, p, P_ + (int64_t)cg * mc, false,
                                    pol_once, false, nullptr, nullptr, nullptr, (int)p, y0);
                    else
                        colacc(sm, Y, m, i0, i1, p, ws.u, 1, P_ + (int64_t)cg * mc, p, y0);
                    gsync();
                    part_uniform(0, p, cg, Gt, k0, k1);
                    reduce_partials(sm, P_, mc, Gt, k0, k1, [&](int64_t k, double v) { mst(ws.s + k, v); }, rks);
                } else {
                    int64_t k0, k1;
                    part_uniform(0, p, cg, Gt, k0, k1);
                    if (zero_u) {
                        for (int64_t k = k0 + tid; k < k1; k += NT) mst(ws.s + k, ld(yrow + k) - c * ld(yrow + k));
                    } else {
                        reduce_partials(sm, P_, mc, Gt, k0, k1,
                                        [&](int64_t k, double v) { mst(ws.s + k, v - c * ld(yrow + k)); }, rks);
                    }
                }
                if (dsub && !(a.dbg & 10)) dtim[3] += dclk() - q2m;
                if (a.pf && p > kNarrowM) pf_first(SrcTr{Tr, (int)m2, (int)p}, (int)ptn0, (int)ptn1, a.pf);
                gsync();
                PH(5);
                // ---------------- TN: [Ts, h] = T_p [s, yrow]; column p of T and Y; x'
                {
                    int64_t l0, l1;
                    l0 = ptn0; l1 = ptn1;
                    if (p > kNarrowM && tyr_have && a.tyr) {
                        // T_p yrow is the same in every iteration of vector p (T_p and row p of Y are
                        // final): kept from the first TN, so later TNs stream T against s alone
                        wide_rowdots<false>(sm, wr, SrcTr{Tr, (int)m2, (int)p}, (int)l0, (int)l1, ws.s, nullptr, p, pol_once,
                                            [&](int64_t l, double a1, double) {
                                                const double that = -tt * a1;
                                                mst(ws.xp + l, ld(ws.tyr + l) + y0 * that);
                                                mst(Tc + tcol_off(p) + l, that);
                                                mst(Tr + l * m2 + p, that);
                                            });
                    } else if (p > kNarrowM) {
                        wide_rowdots<true>(sm, wr, SrcTr{Tr, (int)m2, (int)p}, (int)l0, (int)l1, ws.s, yrow, p, pol_once,
                                           [&](int64_t l, double a1, double a2) {
                                               const double that = -tt * a1;
                                               st(ws.tyr + l, a2);   // this CTA's rows of T_p yrow (same rows every iteration)
                                               mst(ws.xp + l, a2 + y0 * that);
                                               mst(Tc + tcol_off(p) + l, that);
                                               mst(Tr + l * m2 + p, that);
                                           });
                        tyr_have = true;
                    } else if (l1 > l0) {
                        stage_vec(sm, ws.s, p);
                        const int lane = tid & 31, warp = tid >> 5;
                        constexpr int U = 4;
                        for (int64_t l = l0 + warp; l < l1; l += NW) {
                            const double* row = Tr + l * m2;
                            double a1 = 0.0, a2 = 0.0;
                            for (int64_t k0 = (l & ~int64_t(1)) + 2 * lane; k0 < p; k0 += 64 * U) {
                                double2 tv[U], yv[U];
#pragma unroll
                                for (int u = 0; u < U; u++) {
                                    const int64_t k = k0 + 64 * u;
                                    tv[u] = (k < p) ? ld2(row + k) : make_double2(0.0, 0.0);
                                    yv[u] = (k < p) ? ld2(yrow + k) : make_double2(0.0, 0.0);
                                }
#pragma unroll
                                for (int u = 0; u < U; u++) {
                                    const int64_t k = k0 + 64 * u;
                                    if (k < p) {
                                        const double2 sv = *reinterpret_cast<const double2*>(sm.vs + k);
                                        const bool vx = (k >= l), vy = (k + 1 < p);
                                        const double tx = vx ? tv[u].x : 0.0, ty = vy ? tv[u].y : 0.0;
                                        a1 = fma(tx, vx ? sv.x : 0.0, a1);
                                        a1 = fma(ty, vy ? sv.y : 0.0, a1);
                                        a2 = fma(tx, vx ? yv[u].x : 0.0, a2);
                                        a2 = fma(ty, vy ? yv[u].y : 0.0, a2);
                                    }
                                }
                            }
                            a1 = warp_sum(a1);
                            a2 = warp_sum(a2);
                            if (lane == 0) {
                                const double that = -tt * a1;
                                mst(ws.xp + l, a2 + y0 * that);
                                mst(Tc + tcol_off(p) + l, that);
                                mst(Tr + l * m2 + p, that);
                            }
                        }
                    }
                    if (r == 0 && tid == 0) {
                        st(ws.xp + p, tt * y0);
                        st(Tc + tcol_off(p) + p, tt);
                        st(Tr + p * m2 + p, tt);
                    }
                    int64_t i0, i1;
                    part_uniform(p, n, r, G, i0, i1);
                    for (int64_t i = i0 + tid; i < i1; i += NT)
                        st(Y + y_row_off(i, m) + p, (i == p) ? y0 : (zero_u ? 0.0 : ld(ws.u + i)));
                }
                if (a.pf && p + 1 > kNarrowM) pf_first(SrcY{Y, (int)m, (int)p + 1}, (int)pd0, (int)pd1, a.pf);
                gsync();
                PH(6);
                }   // reduced / ordinary compact-WY step
                // ---------------- deferred D (DESIGN §6 "deferred final pass D"): when a pass in
                // this iteration completes the stopping rule and nothing later reads this q (no
                // look-ahead dot for vector p+1, the cluster is its group's last), D and TEST are
                // skipped: x' is parked in the vector's dead x^(1) slot and c in dzc[j]; after the
                // kernel, dz_gemm forms q = Y_{p+1} x' - e_p for all parked vectors at once (one
                // GEMM instead of one read of Y_{p+1} per vector), runs the test and writes z_j.
                // A parked vector whose deferred test fails makes the host re-run the call
                // without deferral, so the result never depends on the guess.
                if (dz_cl && mode != 1 && p + 1 > kNarrowM && passes + 1 >= kPasses && kin < kMaxIts &&
                    !((p + 1 < m) && la_ok && !in_lab(p + 1))) {
                    int64_t k0, k1;
                    part_uniform(0, p + 1, r, G, k0, k1);
                    double* xd = a.dzx + j * n2v;
                    for (int64_t k = k0 + tid; k < k1; k += NT) st(xd + k, ld(ws.xp + k));
                    if (r == 0 && tid == 0) {
                        a.iters[j] = its;
                        if (flagged) atomicAdd(&a.out->nflag, 1);
                        a.dzc[j] = c;
                    }
                    done = true;
                    la_have = la_done;
                    PH(8);
                    continue;
                }
                // ---------------- D: q = Y_{p+1} x' - e_p, norms and argmax
                Aff1 fex{1.0, 0.0};   // forward-sweep state kept from D to the solve
                int64_t fs0 = 0, fta = 0, ftb = 0;
                bool flast = false;
                {
                    int64_t i0, i1;
                    i0 = dq0; i1 = dq1;   // D's rows (MGS: the rows of the projection)
                    double q2 = 0.0, q1 = 0.0, qinf = -1.0;
                    int64_t qarg = 0;
                    if (tid == 0) {   // this CTA's factor rows (forward sweep below, back sweep)
                        const int64_t fa = i0 > 0 ? i0 - 1 : 0;
                        if (i1 > fa) l2_prefetch(a.F + (j * n + fa) * 4, (i1 - fa) * 4);
                    }
                    // y_p^T x^(1)_{p+1}: the last column of the next vector's first pass A
                    double gpn = 0.0;
                    const bool want_gpn = (p + 1 < m) && la_ok && !in_lab(p + 1);
                    const double* xn = a.X1c + (j + 1) * n2v;
                    if (want_gpn && !narrow) {   // (narrow: fused into the D stream below)
                        for (int64_t i = (i0 > p ? i0 : p) + tid; i < i1; i += NT)
                            gpn = fma(ld(Y + y_row_off(i, m) + p), ld(xn + i), gpn);
                    }
                    auto epiq = [&](int64_t i, double v) {
                        const double qi = (i == p) ? v - 1.0 : v;
                        mst(ws.q + i, qi);
                        q2 = fma(qi, qi, q2);
                        const double aq = fabs(qi);
                        q1 += aq;
                        if (aq > qinf || (aq == qinf && i < qarg)) { qinf = aq; qarg = i; }
                    };
                    auto lend = [&](int64_t i) -> int64_t { return (i + 1 < p + 1) ? i + 1 : p + 1; };
                    if (mode == 1) {   // MGS: q (the projected x) is in place; norms and argmax
                        for (int64_t i = i0 + tid; i < i1; i += NT) {
                            const double qi = ld(ws.q + i);
                            q2 = fma(qi, qi, q2);
                            const double aq = fabs(qi);
                            q1 += aq;
                            if (aq > qinf || (aq == qinf && i < qarg)) { qinf = aq; qarg = i; }
                        }
                    } else if (narrow) {
                        stage_vec(sm, ws.xp, p + 1);
                        auto lendn = [&](int i) -> int { return (i + 1 < p + 1) ? i + 1 : (int)p + 1; };
                        // with the look-ahead, the next vector's x^(1) rides along as the stage's
                        // coefficient rows: y_p^T x^(1)_{p+1} from the same stage data
                        narrow_stream(rg, Y, (int)m2, (int)i0, (int)i1, want_gpn ? xn : nullptr,
                                      [&](int ra, int rb, const double* Ys, double* Xs) {
                            narrow_rowdots(ra, rb, (int)m2, Ys, sm.vs, lendn, [&](int i, double v) {
                                epiq(i, v);
                                if (want_gpn && i >= p) gpn = fma(Ys[(i - ra) * m2 + p], Xs[i - ra], gpn);
                            });
                        });
                    } else if (p + 1 > kNarrowM) {
                        wide_rowdots<false>(sm, wr, SrcY{Y, (int)m, (int)p + 1}, (int)i0, (int)i1, ws.xp, nullptr, p + 1, pol_once,
                                            [&](int64_t i, double v, double) { epiq(i, v); });
                    } else {
                        stage_vec(sm, ws.xp, p + 1);
                        rowdots(i0, i1, p + 1, sm.vs, [&](int64_t i) { return Y + y_row_off(i, m); }, lend, epiq);
                    }
                    gpn = block_sum<NT>(gpn, sm.red);
                    if (tid == 0) mst(S + cg * SST + SSlots::GPN, gpn);
                    q2 = block_sum<NT>(q2, sm.red);
                    q1 = block_sum<NT>(q1, sm.red);
                    // block argmax (lowest index on ties)
                    for (int o = 16; o > 0; o >>= 1) {
                        double oq = __shfl_xor_sync(0xffffffffu, qinf, o);
                        long long oa = __shfl_xor_sync(0xffffffffu, (long long)qarg, o);
                        if (oq > qinf || (oq == qinf && oa < qarg)) { qinf = oq; qarg = oa; }
                    }
                    if ((tid & 31) == 0) sm.acc[tid >> 5] = make_double2(qinf, (double)qarg);
                    __syncthreads();
                    if (tid == 0) {
                        for (int w = 1; w < NW; w++) {
                            double2 t = sm.acc[w];
                            if (t.x > qinf || (t.x == qinf && (int64_t)t.y < qarg)) { qinf = t.x; qarg = (int64_t)t.y; }
                        }
                        mst(S + cg * SST + SSlots::Q2, q2);
                        mst(S + cg * SST + SSlots::QINF, qinf);
                        mst(S + cg * SST + SSlots::QARG, (double)qarg);
                        mst(S + cg * SST + SSlots::Q1, q1);
                    }
                    // forward sweep of the chained solve with rhs q, pass 1: steps s in
                    // [i0-1, i1-1) use q_{s+1} from this CTA's rows (reduced to one map per
                    // thread and per CTA; needed only if the test below asks for another
                    // iteration)
                    __syncthreads();
                    fs0 = i0 > 0 ? i0 - 1 : 0;
                    const int64_t fs1 = (i1 - 1 < n - 1) ? i1 - 1 : n - 1;
                    const int64_t FL = fs1 > fs0 ? (fs1 - fs0 + NT - 1) / NT : 0;
                    fta = fs0 + min(fs1 > fs0 ? fs1 - fs0 : 0, (int64_t)tid * FL);
                    ftb = fs0 + min(fs1 > fs0 ? fs1 - fs0 : 0, (int64_t)(tid + 1) * FL);
                    flast = (ftb == n - 1) && (fta < ftb);
                    const double* Fj = a.F + j * n * 4;
                    const int8_t* FPj = a.FP + j * n;
                    Aff1 f{1.0, 0.0};
                    for (int64_t s0 = fta; s0 < ftb; s0 += 8) {
                        double l[8], bn[8];
                        int sw[8];
#pragma unroll
                        for (int u = 0; u < 8; u++) {
                            const bool ok = s0 + u < ftb;
                            l[u] = ok ? ldro(Fj + (s0 + u) * 4) : 0.0;
                            sw[u] = ok ? (int)FPj[s0 + u] : 0;
                            bn[u] = ok ? ld(ws.q + s0 + u + 1) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 8; u++) {
                            if (s0 + u < ftb) {
                                if (sw[u]) f.b = fma(-l[u], bn[u], f.b);
                                else { f.a = -l[u] * f.a; f.b = fma(-l[u], f.b, bn[u]); }
                            }
                        }
                    }
                    Aff1 tot;
                    fex = block_scan_excl(f, reinterpret_cast<Aff1*>(sm.acc), tot);
                    if (tid == 0) {
                        mst(S + cg * SST + SSlots::FA, tot.a);
                        mst(S + cg * SST + SSlots::FB, tot.b);
                    }
                }
                gsync();
                PH(7);
                // ---------------- TEST
                const double q2 = reduce_slot(sm, S, Gt, SSlots::Q2);
                double qinf;
                int64_t qarg;
                reduce_argmax(sm, S, Gt, qinf, qarg);
                if (mode == 1) {   // MGS: degenerate projection (reading 16) -> restart
                    const double x2 = reduce_slot(sm, S, Gt, SSlots::X2);
                    if (sqrt(q2) <= (double)n * kEps * sqrt(x2)) {
                        if (restart < kMaxRestart) {
                            restart++;
                            its++;
                            kin = 1;
                            passes = 0;
                            if (r == 0) cta_solve(a, ws, j, 1, restart, sm, mark, mbph);
                            gsync();
                            PH(10);
                            xcur = ws.x;
                            xs = 1;
                            continue;
                        }
                        flagged = true;
                    }
                }
                if (fabs(c) * qinf >= thr) passes++;
                if (passes >= kPasses) done = true;
                else if (kin >= kMaxIts) { done = true; flagged = true; }
                if (done) {
                    const double sgn = (ld(ws.q + qarg) < 0.0) ? -1.0 : 1.0;
                    const double scl = sgn / sqrt(q2);
                    int64_t i0, i1;
                    part_uniform(0, n, r, G, i0, i1);
                    double* zj = a.Z + j * a.ldz;
                    if (own_out) {   // q is complete in every rank's replica: local rows, local Z
                        for (int64_t i = i0 + tid; i < i1; i += NT) zj[i] = ld(ws.q + i) * scl;
                        if (r == 0 && tid == 0) {
                            a.iters[j] = its;
                            if (flagged) atomicAdd(&a.out->nflag, 1);
                        }
                    }
                    la_have = la_done;
                    PH(8);
                } else {
                    its++;
                    kin++;
                    PH(8);
                    // look-ahead only when it can overlap the back sweep (other CTAs of the
                    // group, or warps 1.. of a single-CTA narrow group)
                    const bool la = !la_done && p + 1 < m && la_ok && !in_lab(p + 1);
                    // fused A2 (single-rank wide groups): pass A of the next iteration (g = Y_p^T x
                    // with the solve's x) streams Y_p behind the back sweep, band by band as the
                    // rows become final, together with the look-ahead Y_p^T x^(1)_{p+1}: one read
                    // of Y_p for both (PAPER.md:534-535 for both vectors)
                    const bool a2 = a.a2 && (NR == 1) && (G > 1) && !narrow && p > kNarrowM && mode != 1;
                    if (r == 0) {
                        if (la) {   // CTA 0 of every rank solves; its look-ahead partial is zero
                            for (int64_t k = tid; k < p; k += NT) st(ws.P2 + (int64_t)cg * mc + k, 0.0);
                            if (tid == 0) mst(S + cg * SST + SSlots::X2N, 0.0);
                        }
                        if (a2) {   // ... and so is its share of the fused pass A
                            for (int64_t k = tid; k < p; k += NT) st(P_ + (int64_t)cg * mc + k, 0.0);
                            if (tid == 0) st(S + cg * SST + SSlots::X2, 0.0);
                        }
                    }
                    {   // forward sweep, pass 2: exact carries from the CTA maps -> t_s = sc y_s / u0_s
                        const double* Fj = a.F + j * n * 4;
                        const int8_t* FPj = a.FP + j * n;
                        const Aff1 pre = compose_ctas(S, cg, reinterpret_cast<Aff1*>(sm.acc));
                        const double q0 = ld(ws.q);
                        double cc = fma(fex.a, fma(pre.a, q0, pre.b), fex.b);
                        const double q1 = reduce_slot(sm, S, Gt, SSlots::Q1);
                        const double sc = (double)n * a.tnorm * fmax(kEps, ldro(a.unn + j)) / q1;
                        double* ts = ws.ysol;
                        for (int64_t s0 = fta; s0 < ftb; s0 += 8) {
                            double l[8], bn[8], rr[8];
                            int sw[8];
#pragma unroll
                            for (int u = 0; u < 8; u++) {
                                const bool ok = s0 + u < ftb;
                                l[u] = ok ? ldro(Fj + (s0 + u) * 4) : 0.0;
                                rr[u] = ok ? ldro(Fj + (s0 + u) * 4 + 1) : 0.0;
                                sw[u] = ok ? (int)FPj[s0 + u] : 0;
                                bn[u] = ok ? ld(ws.q + s0 + u + 1) : 0.0;
                            }
#pragma unroll
                            for (int u = 0; u < 8; u++) {
                                if (s0 + u < ftb) {
                                    double y;
                                    if (sw[u]) { y = bn[u]; cc = fma(-l[u], bn[u], cc); }
                                    else { y = cc; cc = fma(-l[u], cc, bn[u]); }
                                    mst(ts + s0 + u, sc * y * rr[u]);
                                }
                            }
                        }
                        if (flast) {
                            mst(ts + n - 1, sc * cc * ldro(Fj + (n - 1) * 4 + 1));
                            mst(ts + n, 0.0);
                        }
                    }
                    gsync();
                    PH(9);
                    if (G == 1 && la) {
                        // single-CTA narrow group: warps 1..NW-1 stream the look-ahead pass A
                        // of vector p+1 while lane 0 of warp 0 runs the chained back sweep
                        if (tid == 0) back_sweep(a, ws, j, sm, mbph);
                        if (tid >= 32) {
                            constexpr int LT = NT - 32;
                            const int CPT = pow2ceil((int)((p + 1) / 2));
                            double a0 = 0.0, a1 = 0.0, x2n = 0.0;
                            narrow_stream<32, LT>(rg, Y, (int)m2, 0, (int)n, a.X1c + (j + 1) * n2v,
                                                  [&](int ra, int rb, const double* Ys, double* Xs) {
                                for (int ii = tid - 32; ii < rb - ra; ii += LT) x2n = fma(Xs[ii], Xs[ii], x2n);
                                narrow_colacc<32, LT>(ra, rb, (int)m2, Ys, Xs, CPT,
                                                      [&](int i) -> int { return i + 1 < p ? i + 1 : (int)p; }, a0, a1);
                            });
                            narrow_colacc_finish<32, LT>(sm, CPT, p, a0, a1, ws.P2);
                            x2n = warp_sum(x2n);
                            if ((tid & 31) == 0) sm.red[tid >> 5] = x2n;
                            sub_sync<32, LT>();
                            if (tid == 32) {
                                double t = 0.0;
                                for (int w = 1; w < NW; w++) t += sm.red[w];
                                st(S + SSlots::X2N, t);
                                *reinterpret_cast<uint32_t*>(sm.red + NW + 7) = rph;
                            }
                        }
                        __syncthreads();
                        rph = *reinterpret_cast<volatile uint32_t*>(sm.red + NW + 7);
                    } else if (r == 0 && a.sweep2) {
                        if (tid == 0 || tid == 32)
                            back_sweep_ws(a, ws, j, sm, mbph, xseq, tid == 32, a2 ? sw_prog : nullptr, (sw_ep + 1) << 8,
                                          (kWideDebug && (a.dbg & 8) && dsub && tid == 0) ? dtim : nullptr);
                    } else if (r == 0 && tid == 0) {
                        back_sweep(a, ws, j, sm, mbph, a2 ? sw_prog : nullptr, (sw_ep + 1) << 8,
                                   (kWideDebug && (a.dbg & 8) && dsub) ? dtim : nullptr);
                    }
                    mark(10);
                    const bool a2c = a2 && !la && a.a2c && (p + PW - 1) / PW <= G - 1;
                    if (a2c && r > 0) {
                        // column-owner form: this CTA's block, its share of each band's rows
                        const unsigned int tag = (sw_ep + 1) << 8;
                        const int nbands = sweep_bands(n, a.band_ch);
                        int kb, jb, cnt;
                        int* st_tab = reinterpret_cast<int*>(sm.vs);
                        a2c_table(n, p, G - 1, st_tab);
                        __syncthreads();
                        a2c_assign(p, st_tab, r - 1, kb, jb, cnt);
                        __syncthreads();
                        double a0 = 0.0, a1 = 0.0, x2 = 0.0;
                        for (int b = 0; b < nbands; b++) {
                            const int64_t C = (n + 255) / 256;
                            const int64_t chi = C - (int64_t)b * a.band_ch, clo = chi - a.band_ch > 0 ? chi - a.band_ch : 0;
                            const int64_t b0 = clo * 256, b1 = chi * 256 < n ? chi * 256 : n;
                            const int64_t lo = b0 > (int64_t)kb * PW ? b0 : (int64_t)kb * PW;
                            if (tid == 0) {
                                uint32_t spins = 0;
                                while (acquire(sw_prog) < tag + (unsigned int)b + 1u) {
                                    if (a.poll_ns) __nanosleep(a.poll_ns);
                                    if (++spins > (1u << 30)) __trap();
                                }
                            }
                            __syncthreads();
                            if (b1 <= lo) continue;
                            int64_t i0, i1;
                            part_uniform(lo, b1, jb, cnt, i0, i1);
                            if (i1 > i0) a2c_stream(sm, wr, Y, m, p, kb, (int)i0, (int)i1, ws.x, a0, a1, x2, kb == 0, pol_once);
                        }
                        {
                            const int tc = tid - 32, c = kb * PW + 2 * tc;
                            if (tc >= 0 && 2 * tc < PW) {
                                if (c < p) st(P_ + (int64_t)cg * mc + c, a0);
                                if (c + 1 < p) st(P_ + (int64_t)cg * mc + c + 1, a1);
                            }
                        }
                        x2 = block_sum<NT>(x2, sm.red);
                        if (tid == 0) st(S + cg * SST + SSlots::X2, x2);
                    } else if (a2 && r > 0) {
                        // bands bottom-up; this CTA's rows of each band by the pass weights
                        const unsigned int tag = (sw_ep + 1) << 8;
                        const int nbands = sweep_bands(n, a.band_ch);
                        const int bch = a.band_ch;
                        const int Gl = G - 1, rl = r - 1;
                        const double* xn = a.X1c + (j + 1) * n2v;
                        double x2 = 0.0, x2n = 0.0;
                        for (int b = 0; b < nbands; b++) {
                            const int64_t C = (n + 255) / 256;
                            const int64_t chi = C - (int64_t)b * bch, clo = chi - bch > 0 ? chi - bch : 0;
                            const int64_t b0 = clo * 256, b1 = chi * 256 < n ? chi * 256 : n;
                            int64_t i0, i1;
                            part_band_weighted(b0, b1, p, rl, Gl, i0, i1, a.piece_cost);
                            if (tid == 0) {
                                uint32_t spins = 0;
                                while (acquire(sw_prog) < tag + (unsigned int)b + 1u) {
                                    if (a.poll_ns) __nanosleep(a.poll_ns);
                                    if (++spins > (1u << 30)) __trap();
                                }
                            }
                            __syncthreads();
                            if (la) {
                                double c2n = 0.0;
                                x2 += wide_colacc<true>(sm, wr, SrcY{Y, (int)m, (int)p}, (int)i0, (int)i1, ws.x, p,
                                                        P_ + (int64_t)cg * mc, false, pol_once, b > 0, xn,
                                                        ws.P2 + (int64_t)cg * mc, &c2n);
                                x2n += c2n;
                            } else {
                                x2 += wide_colacc(sm, wr, SrcY{Y, (int)m, (int)p}, (int)i0, (int)i1, ws.x, p,
                                                  P_ + (int64_t)cg * mc, false, pol_once, b > 0);
                            }
                        }
                        x2 = block_sum<NT>(x2, sm.red);
                        if (la) x2n = block_sum<NT>(x2n, sm.red);
                        if (tid == 0) {
                            st(S + cg * SST + SSlots::X2, x2);
                            if (la) st(S + cg * SST + SSlots::X2N, x2n);
                        }
                    } else if (la && r > 0) {   // G > 1: the other CTAs of the group
                        // look-ahead: Y_{p}^T x^(1)_{p+1} over the accepted columns 0..p-1,
                        // overlapped with the chained solve (PAPER.md:534-535 for vector j+1)
                        // (every rank's CTA 0 solves; the others split the rows over all ranks)
                        const int Gl = Gt - NR, rl = RK * (G - 1) + (r - 1);
                        int64_t i0, i1;
                        part_rows_weighted(n, p, rl, Gl, i0, i1, a.piece_cost);
                        double x2n = (p > kNarrowM)
                                         ? wide_colacc(sm, wr, SrcY{Y, (int)m, (int)p}, (int)i0, (int)i1, a.X1c + (j + 1) * n2v, p,
                                                       ws.P2 + (int64_t)cg * mc, false, pol_once)
                                         : colacc(sm, Y, m, i0, i1, p, a.X1c + (j + 1) * n2v, 1, ws.P2 + (int64_t)cg * mc);
                        x2n = block_sum<NT>(x2n, sm.red);
                        if (tid == 0) mst(S + cg * SST + SSlots::X2N, x2n);
                    }
                    if (la) la_done = true;
                    if (a2) { sw_ep++; use_a2 = true; use_a2c = a2c; }
                    gsync();
                    PH(11);
                    xcur = ws.x;
                    xs = 1;
                }
            }
        }
        gsync();  // workspace reuse by the next cluster of this group
    }
    if (r == 0 && tid == 0) a.syncs[g] = nsync;
    if (timing)
        for (int k = 0; k < ((kWideDebug && (a.dbg & 16)) ? 14 : 12); k++) a.prof[g * 16 + k] = tacc[k];
    if (timing0 && !kWideDebug)
        for (int k = 0; k < 4; k++) a.prof[12 + k] = ntim[k];
    if (dsub && !(a.dbg & 16))
        for (int k = 0; k < 4; k++) a.prof[12 + k] = dtim[k];
#undef PH
}

// Multi-rank diagnostic (tinv_debug_peer_map): read the first word of every rank's workspace
// replica through the peer-memory mapping, addressed as the persistent kernel addresses peer
// replicas (own base + delta[k] doubles).  Plain loads; nothing here waits on another rank.
__global__ void peer_read_kernel(const double* base, const int64_t* delta, int nrk, uint64_t* out) {
    const int k = threadIdx.x;
    if (k < nrk) {
        const double* p = base + __ldg(delta + k);
        out[k] = *reinterpret_cast<const volatile unsigned long long*>(p);
    }
}
void launch_peer_read(const double* base, const int64_t* delta, int nrk, uint64_t* out, cudaStream_t s) {
    peer_read_kernel<<<1, 32 * ((nrk + 31) / 32), 0, s>>>(base, delta, nrk, out);
}

int cwy_threads() { return NT; }
int cwy_narrow_max() { return kNarrowM; }
int cwy_ring_stages() { return kNStg; }

size_t cwy_smem_bytes(int64_t vcap, int nstg) {
    (void)vcap;
    (void)nstg;
    return sizeof(double) * (size_t)(kVsD + CFCH + 2 * RCH + 4 * PW) + sizeof(double2) * NT + sizeof(double) * (NW + 8) +
           sizeof(uint64_t) * kNBar + sizeof(double) * (size_t)kRingD;
}

int cwy_max_ctas_per_sm(size_t smem) {
    cudaFuncSetAttribute(cwy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, cwy_kernel, NT, smem);
    return nb;
}

cudaError_t launch_cwy(const CwyArgs& a, int nctas, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(cwy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void* args[] = {(void*)&a};
    return cudaLaunchCooperativeKernel((void*)cwy_kernel, dim3(nctas), dim3(NT), args, smem, s);
}

}  // namespace tinv
