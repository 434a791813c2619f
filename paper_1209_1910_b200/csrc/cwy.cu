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

constexpr int NT = 512;
constexpr int NW = NT / 32;

struct SSlots {  // scalar partial slots per CTA (ws.S[r*8 + slot])
    enum { U2 = 0, X2 = 1, Q2 = 2, QINF = 3, QARG = 4 };
};

__device__ __forceinline__ int pow2ceil(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
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

// rows of A / D weighted by their length min(i+1, P)
__device__ __forceinline__ void part_rows_weighted(int64_t n, int64_t P, int r, int G, int64_t& a, int64_t& b) {
    auto cum = [P](int64_t i) -> int64_t { return i <= P ? i * (i + 1) / 2 : P * (P + 1) / 2 + (i - P) * P; };
    int64_t W = cum(n);
    a = bsearch_cum(0, n, (W * r) / G, cum);
    b = bsearch_cum(0, n, (W * (r + 1)) / G, cum);
    if (r == G - 1) b = n;
    if (r == 0) a = 0;
}
__device__ __forceinline__ void part_uniform(int64_t lo, int64_t hi, int r, int G, int64_t& a, int64_t& b) {
    int64_t len = hi - lo;
    a = lo + (len * r) / G;
    b = lo + (len * (r + 1)) / G;
}
// k in [0,p) weighted by k+1 (T^T rows = packed columns of T)
__device__ __forceinline__ void part_tt(int64_t p, int r, int G, int64_t& a, int64_t& b) {
    auto cum = [](int64_t k) -> int64_t { return k * (k + 1) / 2; };
    int64_t W = cum(p);
    a = bsearch_cum(0, p, (W * r) / G, cum);
    b = bsearch_cum(0, p, (W * (r + 1)) / G, cum);
    if (r == G - 1) b = p;
    if (r == 0) a = 0;
}
// l in [0,p) weighted by p-l (rows of T)
__device__ __forceinline__ void part_tn(int64_t p, int r, int G, int64_t& a, int64_t& b) {
    auto cum = [p](int64_t l) -> int64_t { return l * p - l * (l - 1) / 2; };
    int64_t W = cum(p);
    a = bsearch_cum(0, p, (W * r) / G, cum);
    b = bsearch_cum(0, p, (W * (r + 1)) / G, cum);
    if (r == G - 1) b = p;
    if (r == 0) a = 0;
}

__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct Shared {
    double red[NW];
    double2 acc[NT];
};

// ---------------------------------------------------------------- column accumulate
// out[k] = sum_{i in [i0,i1), i >= k} Y[i][k] * coef(i)  for k < P   (coef(i) = cp[i*cs])
__device__ void colacc(const double* __restrict__ Y, int64_t m, int64_t i0, int64_t i1, int64_t P,
                       const double* cp, int64_t cs, double* __restrict__ out, Shared& sh) {
    if (P <= 0) return;
    const int tid = threadIdx.x;
    const int CPT = min(NT, pow2ceil((int)((P + 1) / 2)));
    const int RS = NT / CPT;
    const int cpi = tid % CPT, rs = tid / CPT;
    for (int64_t k0 = 0; k0 < P; k0 += 2 * CPT) {
        const int64_t k = k0 + 2 * cpi;
        double a0 = 0.0, a1 = 0.0;
        if (k < P) {
            const bool two = (k + 1 < P);
            int64_t ia = (i0 > k) ? i0 : k;
#pragma unroll 4
            for (int64_t i = ia + rs; i < i1; i += RS) {
                const double cf = cp[i * cs];
                const double2 v = *reinterpret_cast<const double2*>(Y + y_row_off(i, m) + k);
                a0 = fma(v.x, cf, a0);
                const double vy = (two && k + 1 <= i) ? v.y : 0.0;
                a1 = fma(vy, cf, a1);
            }
        }
        if (RS > 1) {
            __syncthreads();
            sh.acc[tid] = make_double2(a0, a1);
            __syncthreads();
            if (rs == 0) {
                for (int r2 = 1; r2 < RS; r2++) {
                    double2 t = sh.acc[cpi + r2 * CPT];
                    a0 += t.x;
                    a1 += t.y;
                }
            }
        }
        if (rs == 0 && k < P) {
            out[k] = a0;
            if (k + 1 < P) out[k + 1] = a1;
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------- row dots
// For rows i in [i0,i1): dot_i = sum_{k < L_i} R(i)[k] * v[k], L_i = min(len(i), P);
// rowptr(i) gives a 16-byte aligned row start, k0(i) the first valid column (even-aligned
// start handled by masking).  The epilogue f(i, dot) runs on one lane per row.
template <class RowPtr, class RowRange, class Epi>
__device__ __forceinline__ void rowdots(int64_t i0, int64_t i1, int64_t P, const double* __restrict__ v,
                                        RowPtr rowptr, RowRange range, Epi f) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int LPR = min(32, pow2ceil((int)((P + 1) / 2 > 0 ? (P + 1) / 2 : 1)));
    const int RPW = 32 / LPR;
    const int sub = lane / LPR, sl = lane % LPR;
    for (int64_t ib = i0 + (int64_t)warp * RPW; ib < i1; ib += (int64_t)NW * RPW) {
        const int64_t i = ib + sub;
        double acc = 0.0;
        if (i < i1) {
            const double* row = rowptr(i);
            int64_t kb, ke;
            range(i, kb, ke);  // valid columns [kb, ke)
            const int64_t kstart = kb & ~int64_t(1);
#pragma unroll 4
            for (int64_t k = kstart + 2 * sl; k < ke; k += 2 * LPR) {
                const double2 a = *reinterpret_cast<const double2*>(row + k);
                const double2 b = *reinterpret_cast<const double2*>(v + k);
                const bool vx = (k >= kb), vy = (k + 1 < ke);  // mask operands (stale slots)
                acc = fma(vx ? a.x : 0.0, vx ? b.x : 0.0, acc);
                acc = fma(vy ? a.y : 0.0, vy ? b.y : 0.0, acc);
            }
        }
        for (int o = LPR >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (sl == 0 && i < i1) f(i, acc);
    }
}

// ---------------------------------------------------------------- chained single-vector solve
// x = (T - wt_j I)^{-1} (sigma * rhs), sigma = n ||T||_1 max(eps,|u_nn|) / ||rhs||_1,
// with the factors stored by the batched kernel.  rhs = q (mode 0) or the start vector of
// restart `restart` (mode 1).  The recurrences are serial: lane 0 of warp 0 runs them out of
// shared memory while warps 1..NW-1 stage the next chunk of factors (double buffer), so the
// dependent chain is one FMA per row (forward: c <- alpha c + beta with alpha, beta
// precomputed from the pivot bit; back: x_i <- -b_i x_{i+1} + (s y_i r_i - c_i x_{i+2})).
constexpr int CH = 512;
struct SolveSmem {
    double a[2][CH];
    double b[2][CH];
    double c[2][CH];
    int8_t sw[2][CH];
};

__device__ void chain_solve(const CwyArgs& a, const GroupWS& ws, int64_t j, int mode, int restart,
                            SolveSmem& sm, double* red) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n = a.n, ld = a.ldv;
    const double* __restrict__ fl = a.fl + j;
    const int8_t* __restrict__ fp = a.fp + j;
    const double* __restrict__ fr = a.fr + j;
    const double* __restrict__ fb = a.fb + j;
    const double* __restrict__ fc = a.fc + j;
    double* __restrict__ ys = ws.ysol;
    const double* __restrict__ q = ws.q;
    auto rhs = [&](int64_t i) -> double { return mode == 0 ? q[i] : start_entry(a.seed, n, j, restart, i); };
    const int LT = NT - 32;  // loader threads
    const int lt = tid - 32;

    // ---- forward elimination: steps i = 0 .. n-2
    double r1 = 0.0;
    const int64_t nf = n - 1;
    const int64_t nchF = (nf + CH - 1) / CH;
    auto loadF = [&](int64_t ch, int buf) {
        for (int idx = lt; idx < CH; idx += LT) {
            const int64_t i = ch * CH + idx;
            if (i < nf) {
                const double l = fl[i * ld];
                const int8_t sw = fp[i * ld];
                const double bn = rhs(i + 1);
                r1 += fabs(bn);
                sm.a[buf][idx] = sw ? 1.0 : -l;
                sm.b[buf][idx] = sw ? -l * bn : bn;
                sm.c[buf][idx] = bn;
                sm.sw[buf][idx] = sw;
            }
        }
    };
    double cc = 0.0;
    if (tid == 0) { cc = rhs(0); r1 = fabs(cc); }
    if (warp > 0 && nchF > 0) loadF(0, 0);
    __syncthreads();
    for (int64_t ch = 0; ch < nchF; ch++) {
        const int buf = (int)(ch & 1);
        if (warp == 0) {
            if (lane == 0) {
                const int cnt = (int)((nf - ch * CH) < CH ? (nf - ch * CH) : CH);
                double* yo = ys + ch * CH;
#pragma unroll 8
                for (int idx = 0; idx < cnt; idx++) {
                    const double y = sm.sw[buf][idx] ? sm.c[buf][idx] : cc;
                    cc = fma(sm.a[buf][idx], cc, sm.b[buf][idx]);
                    yo[idx] = y;
                }
            }
        } else if (ch + 1 < nchF) {
            loadF(ch + 1, buf ^ 1);
        }
        __syncthreads();
    }
    if (tid == 0) ys[n - 1] = cc;
    r1 = block_sum<NT>(r1, red);   // includes the __syncthreads that publishes ys
    const double sc = (double)n * a.tnorm * fmax(kEps, a.unn[j]) / r1;

    // ---- back substitution: rows n-1 .. 0
    const int64_t nchB = (n + CH - 1) / CH;
    auto loadB = [&](int64_t ch, int buf) {
        for (int idx = lt; idx < CH; idx += LT) {
            const int64_t i = n - 1 - ch * CH - idx;
            if (i >= 0) {
                const int64_t o = i * ld;
                sm.a[buf][idx] = sc * ys[i] * fr[o];
                sm.b[buf][idx] = fb[o];
                sm.c[buf][idx] = fc[o];
            }
        }
    };
    double* __restrict__ x = ws.x;
    double xp1 = 0.0, xp2 = 0.0;
    if (warp > 0) loadB(0, 0);
    __syncthreads();
    for (int64_t ch = 0; ch < nchB; ch++) {
        const int buf = (int)(ch & 1);
        if (warp == 0) {
            if (lane == 0) {
                const int cnt = (int)((n - ch * CH) < CH ? (n - ch * CH) : CH);
                const int64_t ib = n - 1 - ch * CH;
#pragma unroll 8
                for (int idx = 0; idx < cnt; idx++) {
                    const double t = fma(-sm.c[buf][idx], xp2, sm.a[buf][idx]);
                    const double xi = fma(-sm.b[buf][idx], xp1, t);
                    x[ib - idx] = xi;
                    xp2 = xp1;
                    xp1 = xi;
                }
            }
        } else if (ch + 1 < nchB) {
            loadB(ch + 1, buf ^ 1);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(NT, 1) cwy_kernel(CwyArgs a) {
    __shared__ Shared sh;
    __shared__ SolveSmem ssm;
    const int tid = threadIdx.x;
    // locate group
    int g = 0;
    for (int t = 0; t < a.ngroups; t++)
        if ((int)blockIdx.x >= a.g_cta0[t]) g = t;
    const int r = blockIdx.x - a.g_cta0[g];
    const int G = a.g_size[g];
    if (r >= G) return;  // CTA not used by any group
    const GroupWS ws = a.ws[g];
    long long nsync = 0;
    auto gsync = [&]() { group_sync(ws.bar, G); nsync++; };
    // optional phase timers (thread 0 of each group's first CTA; globaltimer ns)
    const bool timing = (a.prof != nullptr) && r == 0 && tid == 0;
    uint64_t tacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    uint64_t tmark = timing ? gtime() : 0;
#define PH(k)                                         \
    do {                                              \
        if (timing) {                                 \
            uint64_t _t = gtime();                    \
            tacc[k] += _t - tmark;                    \
            tmark = _t;                               \
        }                                             \
    } while (0)

    const int64_t n = a.n;
    const double thr = sqrt(0.1 / (double)n);
    double* __restrict__ Y = ws.Y;
    double* __restrict__ S = ws.S;

    for (int ci = a.g_coff[g]; ci < a.g_coff[g + 1]; ci++) {
        const int cl = a.g_clist[ci];
        const int64_t j1 = a.cstart[cl];
        const int64_t m = a.cstart[cl + 1] - j1;
        const int64_t m2 = (m + 1) & ~int64_t(1);
        double* __restrict__ Tc = ws.Tc;
        double* __restrict__ Tr = ws.Tr;

        // ================= first reflector from the accepted z_{j1} (p = 0)
        {
            const double* z = a.Z + j1 * a.ldz;
            int64_t i0, i1;
            part_uniform(0, n, r, G, i0, i1);
            double u2 = 0.0;
            for (int64_t i = i0 + tid; i < i1; i += NT) {
                const double zi = z[i];
                ws.u[i] = zi;
                u2 = fma(zi, zi, u2);
            }
            u2 = block_sum<NT>(u2, sh.red);
            if (tid == 0) S[r * 8 + SSlots::U2] = u2;
            gsync();
            double un = 0.0;
            for (int t = 0; t < G; t++) un += S[t * 8 + SSlots::U2];
            un = sqrt(un);
            const double u0 = ws.u[0];
            const double c = -((u0 >= 0.0) ? 1.0 : -1.0) * un;
            const double tt = 1.0 / (c * c - u0 * c);
            for (int64_t i = i0 + tid; i < i1; i += NT)
                Y[y_row_off(i, m) + 0] = (i == 0) ? (u0 - c) : ws.u[i];
            if (r == 0 && tid == 0) { Tc[tcol_off(0)] = tt; Tr[0] = tt; }
            gsync();
            PH(0);
        }

        // ================= vectors j_c = 1 .. m-1
        for (int64_t p = 1; p < m; p++) {
            const int64_t j = j1 + p;
            const double* xcur = a.X1 + j;   // x^(1), interleaved
            int64_t xs = a.ldv;
            int its = 1, kin = 1, passes = 0, restart = 0;
            bool done = false, flagged = false;
            while (!done) {
                // ---------------- A: partial g = Y_p^T x, ||x||^2
                {
                    int64_t i0, i1;
                    part_rows_weighted(n, p, r, G, i0, i1);
                    colacc(Y, m, i0, i1, p, xcur, xs, ws.P + (int64_t)r * ws.mcap, sh);
                    double x2 = 0.0;
                    for (int64_t i = i0 + tid; i < i1; i += NT) { double xi = xcur[i * xs]; x2 = fma(xi, xi, x2); }
                    x2 = block_sum<NT>(x2, sh.red);
                    if (tid == 0) S[r * 8 + SSlots::X2] = x2;
                }
                gsync();
                PH(1);
                // ---------------- R1: g = sum_r partials
                {
                    int64_t k0, k1;
                    part_uniform(0, p, r, G, k0, k1);
                    for (int64_t k = k0 + tid; k < k1; k += NT) {
                        double s = 0.0;
                        for (int t = 0; t < G; t++) s += ws.P[(int64_t)t * ws.mcap + k];
                        ws.g[k] = s;
                    }
                }
                gsync();
                PH(2);
                // ---------------- TT: g' = T_p^T g
                {
                    int64_t k0, k1;
                    part_tt(p, r, G, k0, k1);
                    rowdots(k0, k1, p, ws.g,
                            [&](int64_t k) { return Tc + tcol_off(k); },
                            [&](int64_t k, int64_t& kb, int64_t& ke) { kb = 0; ke = k + 1; },
                            [&](int64_t k, double v) { ws.gp[k] = v; });
                }
                gsync();
                PH(3);
                // ---------------- BC: u^ = x^ - Yhat g' (rows p..n-1), s' partials, ||u^||^2
                {
                    int64_t i0, i1;
                    part_uniform(p, n, r, G, i0, i1);
                    double u2 = 0.0;
                    rowdots(i0, i1, p, ws.gp,
                            [&](int64_t i) { return Y + y_row_off(i, m); },
                            [&](int64_t i, int64_t& kb, int64_t& ke) { kb = 0; ke = p; },
                            [&](int64_t i, double v) {
                                const double ui = xcur[i * xs] - v;
                                ws.u[i] = ui;
                                u2 = fma(ui, ui, u2);
                            });
                    __syncthreads();
                    u2 = block_sum<NT>(u2, sh.red);
                    if (tid == 0) S[r * 8 + SSlots::U2] = u2;
                    colacc(Y, m, i0, i1, p, ws.u, 1, ws.P + (int64_t)r * ws.mcap, sh);
                }
                gsync();
                PH(4);
                // ---------------- R2: scalars (every CTA, identical), s = s' - c Y[p,:]
                double un = 0.0, x2 = 0.0;
                for (int t = 0; t < G; t++) { un += S[t * 8 + SSlots::U2]; x2 += S[t * 8 + SSlots::X2]; }
                un = sqrt(un);
                double u0 = ws.u[p];
                const bool zero_u = (un == 0.0);   // reading: exactly-zero uhat -> e_1
                if (zero_u) { u0 = 1.0; un = 1.0; }
                // degenerate iterate (reading 16): restart with a fresh start vector
                if (un <= (double)n * kEps * sqrt(x2) && restart < kMaxRestart && !zero_u) {
                    restart++;
                    its++;
                    kin = 1;
                    passes = 0;
                    if (r == 0) chain_solve(a, ws, j, 1, restart, ssm, sh.red);
                    gsync();
                    PH(9);
                    xcur = ws.x;
                    xs = 1;
                    continue;
                }
                if (un <= (double)n * kEps * sqrt(x2)) flagged = true;
                const double c = -((u0 >= 0.0) ? 1.0 : -1.0) * un;
                const double tt = 1.0 / (c * c - u0 * c);
                const double y0 = u0 - c;
                const double* yrow = Y + y_row_off(p, m);
                {
                    int64_t k0, k1;
                    part_uniform(0, p, r, G, k0, k1);
                    for (int64_t k = k0 + tid; k < k1; k += NT) {
                        double s = 0.0;
                        if (zero_u) s = yrow[k];
                        else for (int t = 0; t < G; t++) s += ws.P[(int64_t)t * ws.mcap + k];
                        ws.s[k] = s - c * yrow[k];
                    }
                }
                gsync();
                PH(5);
                // ---------------- TN: [Ts, h] = T_p [s, yrow]; column p of T and Y; x'
                {
                    int64_t l0, l1;
                    part_tn(p, r, G, l0, l1);
                    const int tid_ = tid, lane = tid_ & 31, warp = tid_ >> 5;
                    for (int64_t l = l0 + warp; l < l1; l += NW) {
                        const double* row = Tr + l * m2;
                        double a1 = 0.0, a2 = 0.0;
                        for (int64_t k = (l & ~int64_t(1)) + 2 * lane; k < p; k += 64) {
                            const double2 tv = *reinterpret_cast<const double2*>(row + k);
                            const double2 sv = *reinterpret_cast<const double2*>(ws.s + k);
                            const double2 yv = *reinterpret_cast<const double2*>(yrow + k);
                            const bool vx = (k >= l), vy = (k + 1 < p);
                            const double tx = vx ? tv.x : 0.0, ty = vy ? tv.y : 0.0;
                            a1 = fma(tx, vx ? sv.x : 0.0, a1); a1 = fma(ty, vy ? sv.y : 0.0, a1);
                            a2 = fma(tx, vx ? yv.x : 0.0, a2); a2 = fma(ty, vy ? yv.y : 0.0, a2);
                        }
                        a1 = warp_sum(a1);
                        a2 = warp_sum(a2);
                        if (lane == 0) {
                            const double that = -tt * a1;
                            ws.xp[l] = a2 + y0 * that;
                            Tc[tcol_off(p) + l] = that;
                            Tr[l * m2 + p] = that;
                        }
                    }
                    if (r == 0 && tid == 0) {
                        ws.xp[p] = tt * y0;
                        Tc[tcol_off(p) + p] = tt;
                        Tr[p * m2 + p] = tt;
                    }
                    int64_t i0, i1;
                    part_uniform(p, n, r, G, i0, i1);
                    for (int64_t i = i0 + tid; i < i1; i += NT)
                        Y[y_row_off(i, m) + p] = (i == p) ? y0 : (zero_u ? 0.0 : ws.u[i]);
                }
                gsync();
                PH(6);
                // ---------------- D: q = Y_{p+1} x' - e_p, norms and argmax
                {
                    int64_t i0, i1;
                    part_rows_weighted(n, p + 1, r, G, i0, i1);
                    double q2 = 0.0, qinf = -1.0;
                    int64_t qarg = 0;
                    rowdots(i0, i1, p + 1, ws.xp,
                            [&](int64_t i) { return Y + y_row_off(i, m); },
                            [&](int64_t i, int64_t& kb, int64_t& ke) { kb = 0; ke = (i + 1 < p + 1) ? i + 1 : p + 1; },
                            [&](int64_t i, double v) {
                                const double qi = (i == p) ? v - 1.0 : v;
                                ws.q[i] = qi;
                                q2 = fma(qi, qi, q2);
                                const double aq = fabs(qi);
                                if (aq > qinf || (aq == qinf && i < qarg)) { qinf = aq; qarg = i; }
                            });
                    __syncthreads();
                    q2 = block_sum<NT>(q2, sh.red);
                    // block argmax (lowest index on ties)
                    for (int o = 16; o > 0; o >>= 1) {
                        double oq = __shfl_xor_sync(0xffffffffu, qinf, o);
                        long long oa = __shfl_xor_sync(0xffffffffu, (long long)qarg, o);
                        if (oq > qinf || (oq == qinf && oa < qarg)) { qinf = oq; qarg = oa; }
                    }
                    if ((tid & 31) == 0) { sh.acc[tid >> 5] = make_double2(qinf, (double)qarg); }
                    __syncthreads();
                    if (tid == 0) {
                        for (int w = 1; w < NW; w++) {
                            double2 t = sh.acc[w];
                            if (t.x > qinf || (t.x == qinf && (int64_t)t.y < qarg)) { qinf = t.x; qarg = (int64_t)t.y; }
                        }
                        S[r * 8 + SSlots::Q2] = q2;
                        S[r * 8 + SSlots::QINF] = qinf;
                        S[r * 8 + SSlots::QARG] = (double)qarg;
                    }
                }
                gsync();
                PH(7);
                // ---------------- TEST
                double q2 = 0.0, qinf = -1.0;
                int64_t qarg = 0;
                for (int t = 0; t < G; t++) {
                    q2 += S[t * 8 + SSlots::Q2];
                    const double v = S[t * 8 + SSlots::QINF];
                    const int64_t ia = (int64_t)S[t * 8 + SSlots::QARG];
                    if (v > qinf || (v == qinf && ia < qarg)) { qinf = v; qarg = ia; }
                }
                if (fabs(c) * qinf >= thr) passes++;
                if (passes >= kPasses) done = true;
                else if (kin >= kMaxIts) { done = true; flagged = true; }
                if (done) {
                    const double sgn = (ws.q[qarg] < 0.0) ? -1.0 : 1.0;
                    const double scl = sgn / sqrt(q2);
                    int64_t i0, i1;
                    part_uniform(0, n, r, G, i0, i1);
                    double* zj = a.Z + j * a.ldz;
                    for (int64_t i = i0 + tid; i < i1; i += NT) zj[i] = ws.q[i] * scl;
                    if (r == 0 && tid == 0) {
                        a.iters[j] = its;
                        if (flagged) atomicAdd(&a.out->nflag, 1);
                    }
                    PH(8);
                } else {
                    its++;
                    kin++;
                    PH(8);
                    if (r == 0) chain_solve(a, ws, j, 0, 0, ssm, sh.red);
                    gsync();
                    PH(9);
                    xcur = ws.x;
                    xs = 1;
                }
            }
        }
        gsync();  // workspace reuse by the next cluster of this group
    }
    if (r == 0 && tid == 0) a.syncs[g] = nsync;
    if (timing)
        for (int k = 0; k < 10; k++) a.prof[g * 16 + k] = tacc[k];
#undef PH
}

int cwy_threads() { return NT; }

int cwy_max_ctas_per_sm() {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, cwy_kernel, NT, 0);
    return nb;
}

cudaError_t launch_cwy(const CwyArgs& a, int nctas, cudaStream_t s) {
    void* args[] = {(void*)&a};
    return cudaLaunchCooperativeKernel((void*)cwy_kernel, dim3(nctas), dim3(NT), args, 0, s);
}

}  // namespace tinv
