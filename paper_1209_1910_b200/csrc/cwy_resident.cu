// cwy_resident.cu -- compact-WY inverse iteration for narrow clusters with Y resident in
// distributed shared memory (Alg. 4, §3.3.2 lines
// 439-633).
//
// The clustered work of small-n problems (cfg1/cfg2: hundreds of clusters of m <= 64) is
// latency-bound: the critical path is the 2 (m-1) dependent iterations of the largest
// cluster, each a handful of passes over its Y (n x m).  Streaming Y from L2 every pass costs
// ~15 us per pass; here every eigen-cluster is owned by one thread-block cluster of CS CTAs
// (CS in {1, 2, 4, 8}, chosen by the host so that the cluster's rows fit): CTA c keeps rows
// [c RL, (c+1) RL) of Y (built column by column, never leaving shared memory), of the iterate
// and of uhat / q.  Every phase works on local rows; the few cross-CTA reductions (Y^T x,
// Yhat^T uhat, norms, the chained solve's forward maps) go through a double-buffered exchange
// area read over DSMEM in fixed CTA order (deterministic), separated by hardware cluster
// barriers.  T (m x m), g, g', s, x' are small and replicated in every CTA.
//
// Per iteration of vector p (the same algebra as cwy.cu; formulas cited there):
//   A   g = Y_p^T x                       (or the look-ahead partials for the first iteration)
//   TT  g' = T_p^T g                      (replicated)
//   BC  uhat = xhat - Yhat g', s' = Yhat^T uhat, ||uhat||^2
//   R2  c, t, y0 (reflector), s = s' - c Y[p,:]
//   TN  that = -t T_p s, x' = T_p Y[p,:]^T + y0 that (the T_j erratum fix), column p of T, Y
//   D   q = Y_{p+1} x' - e_p, norms/argmax, forward-sweep chunk maps
//   TEST, then either z_j = q/||q|| or the chained solve: exact forward carries from the
//   composed maps -> t rows (gathered in CTA 0), back substitution in CTA 0 (factor records
//   staged in shared memory by all its threads, then one thread's dependent chain), then
//   every CTA copies its x rows, while every other warp computes the look-ahead pass A of
//   vector p+1.
#include <cooperative_groups.h>

#include "common.cuh"
#include "tinv_internal.h"

namespace cgr = cooperative_groups;

namespace tinv {
namespace res {

constexpr int NT = 256;
constexpr int NW = NT / 32;
static_assert(NT >= 4 * kNarrowM, "TT / TN use four threads per column of a cluster of up to kNarrowM vectors");
constexpr int kXS = 16;          // scalar slots of the exchange area
enum { U2 = 0, X2 = 1, U0 = 2, Q2 = 3, QINF = 4, QARG = 5, Q1 = 6, FA = 7, FB = 8, X2N = 9, GPN = 10, QSGN = 11, Q0 = 12 };

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
// bulk L2 prefetch (16-byte aligned, size rounded up to 16 bytes)
__device__ __forceinline__ void l2_prefetch_(const double* p, int64_t nd) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((uint32_t)(((nd * 8) + 15) & ~int64_t(15)))
                 : "memory");
}
__device__ __forceinline__ int pow2ceil(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

struct Aff {
    double a, b;   // c -> a c + b
};
__device__ __forceinline__ Aff comp(const Aff& f, const Aff& g) { return Aff{f.a * g.a, fma(f.a, g.b, f.b)}; }

struct L {        // shared-memory carve-up (doubles unless noted)
    double* Y;    // RL x M2, local rows; the 16-byte column pairs of row i are XOR-swizzled
                  // (yo) so that a warp's loads of one pair from consecutive rows hit distinct banks
    double* xl;   // RL: current iterate
    double* ul;   // RL: uhat (BC .. TN)
    double* ql;   // RL: q (D .. the solve's forward pass / z); shares ul's storage (disjoint lives)
    double* x1l;  // RL: x^(1) of the next vector (look-ahead)
    double* T;    // M2 x TS row-major, T[l][k] (odd stride TS = M2 + 1: threads walking rows do not collide)
    double* g;    // M2 + 2
    double* gp;
    double* s;
    double* xp;
    double* yrow; // M2 + 2: row p of Y (pushed by its owner CTA)
    double* PX;   // [2][CS][XW]: exchange, double-buffered; record c written by CTA c into every CTA
    double* PXL;  // [CS][XW]: look-ahead exchange
    double* tf;   // n + 2: t rows gathered for the back sweep (CTA 0), x written in place
    double* bc;   // 2 n: (u1/u0, u2/u0) of every row, staged by CTA 0 for the back sweep
    double* red;  // 2 x NW x 6: block reductions (double-buffered)
    double* cred; // NW: colacc scalar partials
    double2* acc; // NT
};

__host__ __device__ inline size_t smem_doubles(int64_t n, int RL, int M2, int CS) {
    const size_t XW = (size_t)M2 + kXS;
    const size_t TS = M2 + 1;
    return (size_t)RL * (M2 + 3) + (size_t)M2 * TS + 1 + 5 * (size_t)(M2 + 2) + 3 * CS * XW + (n + 2) + 2 * (size_t)n +
           4 + 2 * NW * 6 + NW + 2 * NT + 8;
}

// Offset of element (i, k) of Y (row stride M2, even).  A row is U = M2/2 16-byte units; rows
// i and i' share a bank group for the same unit when (i - i') U = 0 mod 8, i.e. every 8 / 2^s
// rows with 2^s || U (s <= 3).  Unit u of row i is stored at u ^ ((i >> (3 - s)) & (2^s - 1)),
// which spreads 8 consecutive rows over distinct bank groups and stays inside the row.
struct YSw {
    int M2, sh, msk;
    __device__ explicit YSw(int m2) : M2(m2) {
        const int U = m2 >> 1;
        const int s = U ? min(3, __ffs(U) - 1) : 0;
        sh = 3 - s;
        msk = (1 << s) - 1;
    }
    __device__ __forceinline__ int x(int i) const { return (i >> sh) & msk; }                  // row's key
    __device__ __forceinline__ int pair(int i, int u) const { return i * M2 + 2 * (u ^ x(i)); }  // unit u
    __device__ __forceinline__ int at(int i, int k) const { return pair(i, k >> 1) + (k & 1); }
};

// block-wide exclusive scan of affine maps (thread order), total returned
__device__ __forceinline__ Aff scan_excl(Aff f, Aff* buf, Aff& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    Aff inc = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const Aff g{__shfl_up_sync(0xffffffffu, inc.a, o), __shfl_up_sync(0xffffffffu, inc.b, o)};
        if (lane >= o) inc = comp(inc, g);
    }
    Aff ex{__shfl_up_sync(0xffffffffu, inc.a, 1), __shfl_up_sync(0xffffffffu, inc.b, 1)};
    if (lane == 0) ex = Aff{1.0, 0.0};
    __syncthreads();
    if (lane == 31) buf[w] = inc;
    __syncthreads();
    Aff pre{1.0, 0.0};
    for (int k = 0; k < w; k++) pre = comp(buf[k], pre);
    total = pre;
    for (int k = w; k < NW; k++) total = comp(buf[k], total);
    __syncthreads();
    return comp(ex, pre);
}

// Fixed-order block reduction of K sums and, with ARG, an argmax (larger value wins, then the
// lower index) in one barrier: butterfly inside each warp, then every thread folds the NW warp
// records in warp order, so every thread holds the (bitwise identical) results.  `red` is
// double-buffered by the caller's parity `par` (every thread runs the same sequence of calls,
// and a buffer is rewritten only after the next call's barrier).
template <int K, bool ARG>
__device__ __forceinline__ void block_reduce(double (&v)[K], double& mx, long long& ix, double* red, int& par) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < K; k++) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if (ARG) {
            const double om = __shfl_xor_sync(0xffffffffu, mx, o);
            const long long oi = __shfl_xor_sync(0xffffffffu, ix, o);
            if (om > mx || (om == mx && oi < ix)) { mx = om; ix = oi; }
        }
    }
    double* B = red + par * NW * 6;
    par ^= 1;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) B[w * 6 + k] = v[k];
        if (ARG) { B[w * 6 + 4] = mx; B[w * 6 + 5] = (double)ix; }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = 0.0;
    if (ARG) { mx = -1.0; ix = 0; }
    for (int q = 0; q < NW; q++) {
#pragma unroll
        for (int k = 0; k < K; k++) v[k] += B[q * 6 + k];
        if (ARG) {
            const double m = B[q * 6 + 4];
            const long long i = (long long)B[q * 6 + 5];
            if (m > mx || (m == mx && i < ix)) { mx = m; ix = i; }
        }
    }
}

// Distributed shared memory: the shared::cluster address of `p` in CTA `cta`, and a store to it
// (explicit PTX: a 32-bit cluster address instead of a generic one).
__device__ __forceinline__ uint32_t cl_addr(const void* p, int cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(cta));
    return r;
}
__device__ __forceinline__ void st_cl(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// Column accumulate over local rows [a, b) (local indices): out(k, sum_i Y[i][k] coef(i), c) for
// k < P, Y lower-trapezoidal (row gi = r0 + i holds columns 0..gi).  Threads [t0, t0 + nth)
// (whole warps): a warp covers 32 / CPT rows per step with CPT lanes per row (two columns per
// lane), two rows per lane in flight; lanes of a row slice combine by butterfly, warps through
// shared memory in warp order (deterministic); the column sums are delivered to NC
// destinations by NC x ceil(P/2) threads (thread (pair, c) calls out(k, v, c)).  The
// per-thread scalar `s` is summed alongside and returned to every thread.
template <class Coef, class Out, class Sync>
__device__ __forceinline__ double colacc(const L& sm, const YSw& ys, int r0, int a, int b, int P, Coef coef, Out out,
                                         int NC, double s, int t0, int nth, Sync sync) {
    const int t = threadIdx.x - t0, w = t >> 5, ln = t & 31, W = nth >> 5;
    const int KP = max(1, (P + 1) >> 1);
    const int CPT = min(32, pow2ceil(KP));
    const int cp = ln & (CPT - 1), rl = ln / CPT;
    const int RS = W * (32 / CPT);
    const int k = 2 * cp;
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    auto row = [&](int i, double& x0, double& x1) {
        const int le = min(r0 + i + 1, P);
        if (k < le) {
            const double2 y = *reinterpret_cast<const double2*>(sm.Y + ys.pair(i, cp));
            const double c = coef(i);
            x0 = fma(y.x, c, x0);
            if (k + 1 < le) x1 = fma(y.y, c, x1);
        }
    };
    int i = a + w * (32 / CPT) + rl;
    // rows with global index below P - 1 hold fewer than P columns (first CTA only): checked
    for (; i < b && r0 + i + 1 < P; i += RS) row(i, a0, a1);
    if (k < P) {   // full rows: four rows' loads in flight, four accumulator pairs (the second
                   // column of the last pair may be past P: accumulated, never delivered)
        double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
        for (; i + 3 * RS < b; i += 4 * RS) {
            const double2 y0 = *reinterpret_cast<const double2*>(sm.Y + ys.pair(i, cp));
            const double2 y1 = *reinterpret_cast<const double2*>(sm.Y + ys.pair(i + RS, cp));
            const double2 y2 = *reinterpret_cast<const double2*>(sm.Y + ys.pair(i + 2 * RS, cp));
            const double2 y3 = *reinterpret_cast<const double2*>(sm.Y + ys.pair(i + 3 * RS, cp));
            const double e0 = coef(i), e1 = coef(i + RS), e2 = coef(i + 2 * RS), e3 = coef(i + 3 * RS);
            a0 = fma(y0.x, e0, a0); a1 = fma(y0.y, e0, a1);
            b0 = fma(y1.x, e1, b0); b1 = fma(y1.y, e1, b1);
            c0 = fma(y2.x, e2, c0); c1 = fma(y2.y, e2, c1);
            d0 = fma(y3.x, e3, d0); d1 = fma(y3.y, e3, d1);
        }
        for (; i < b; i += RS) {
            const double2 y = *reinterpret_cast<const double2*>(sm.Y + ys.pair(i, cp));
            const double e = coef(i);
            a0 = fma(y.x, e, a0);
            a1 = fma(y.y, e, a1);
        }
        a0 += c0; a1 += c1; b0 += d0; b1 += d1;
    }
    a0 += b0;
    a1 += b1;
    for (int o = CPT; o < 32; o <<= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    s = warp_sum(s);
    sync();   // acc / cred free
    if (rl == 0) sm.acc[w * 32 + cp] = make_double2(a0, a1);
    if (ln == 0) sm.cred[w] = s;
    sync();
    for (int u = t; u < KP * NC; u += nth) {
        const int pc = u / NC, c = u - pc * NC;
        if (2 * pc < P) {
            double v0 = 0.0, v1 = 0.0;
            for (int q = 0; q < W; q++) {
                const double2 v = sm.acc[q * 32 + pc];
                v0 += v.x;
                v1 += v.y;
            }
            out(2 * pc, v0, c);
            if (2 * pc + 1 < P) out(2 * pc + 1, v1, c);
        }
    }
    double r = 0.0;
    for (int q = 0; q < W; q++) r += sm.cred[q];
    return r;
}

// Back substitution x_i = t_i - b_i x_{i+1} - c_i x_{i+2} (rows n-1 .. 0; the row-normalised
// U of the chained solve), in place over t.  The recurrence stays sequential: expanding it
// over blocks of rows multiplies the b, c of neighbouring rows, which for nearly decoupled
// blocks (pivots ~ eps ||T||, |b| ~ 1e11 in glued Wilkinson matrices) cancels catastrophically.
// All threads of CTA 0 stage (b, c) of every row into shared memory (back_stage_async); then
// one thread runs the chain from shared memory in 16-row batches (back_sweep_smem).
// Staged asynchronously (cp.async, 16 bytes per row) when the vector starts, so the copy is
// off the critical path by the time of its first solve; the sweep waits for the group.
__device__ void back_stage_async(const double* __restrict__ F, double* bc, int64_t n) {
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < n; i += NT)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(bc + 2 * i)), "l"(F + i * 4 + 2)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ void back_sweep_smem(const double* __restrict__ bc, double* tf, int64_t n64) {
    const double2* BC = reinterpret_cast<const double2*>(bc);
    const int n = (int)n64;
    double x1 = 0.0, x2 = 0.0;
    const int top = n & ~15;
    for (int u = n - 1; u >= top; u--) {
        const double2 v = BC[u];
        const double xi = fma(-v.x, x1, fma(-v.y, x2, tf[u]));
        tf[u] = xi;
        x2 = x1;
        x1 = xi;
    }
    // 16-row batches: the batch's loads first (independent), then the dependent chain
    for (int u0 = top - 16; u0 >= 0; u0 -= 16) {
        double b[16], c[16], t[16], xv[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const double2 v = BC[u0 + u];
            b[u] = v.x; c[u] = v.y; t[u] = tf[u0 + u];
        }
#pragma unroll
        for (int u = 15; u >= 0; u--) {
            xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u]));
            x2 = x1;
            x1 = xv[u];
        }
#pragma unroll
        for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(tf + u0 + u) = make_double2(xv[u], xv[u + 1]);
    }
}

__global__ void __launch_bounds__(NT, 1) cwy_resident_kernel(ResArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cgr::cluster_group cl = cgr::this_cluster();
    const int CS = (int)cl.num_blocks();
    const int crank = (int)cl.block_rank();
    const int unit = blockIdx.x / CS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = a.n;
    const int RL = a.RL, M2 = a.M2;
    const int TS = M2 + 1;
    const YSw ys(M2);
    const int XW = M2 + kXS;
    L sm;
    {
        double* p = reinterpret_cast<double*>(smem_raw);
        sm.Y = p; p += (size_t)RL * M2;
        sm.xl = p; p += RL;
        sm.ul = p; p += RL;
        sm.ql = sm.ul;
        sm.x1l = p; p += RL;
        sm.T = p; p += (size_t)M2 * TS;
        sm.g = p; p += M2 + 2;
        sm.gp = p; p += M2 + 2;
        sm.s = p; p += M2 + 2;
        sm.xp = p; p += M2 + 2;
        sm.yrow = p; p += M2 + 2;
        sm.PX = p; p += 2 * (size_t)CS * XW;
        sm.PXL = p; p += (size_t)CS * XW;
        p += (reinterpret_cast<uintptr_t>(p) & 15) ? 1 : 0;
        sm.tf = p; p += (n + 2 + 1) & ~int64_t(1);
        sm.bc = p; p += 2 * n;
        sm.red = p; p += 2 * NW * 6;
        sm.cred = p; p += NW;
        p += (reinterpret_cast<uintptr_t>(p) & 15) ? 1 : 0;
        sm.acc = reinterpret_cast<double2*>(p);
    }
    __syncthreads();
    const double thr = sqrt(0.1 / (double)n);
    // optional phase timers (unit 0, CTA 0, thread 0; SM cycles): 0 A/R1, 1 TT, 2 BC,
    // 3 R2 (+restart), 4 TN, 5 D rows + reduction, 6 D forward maps, 7 D scan + exchange,
    // 8 TEST (+done), 9 back-sweep staging, 10 forward pass 2, 11 back sweep, 12 look-ahead,
    // 13 x push + barrier, 14 leader iterations, 15 first reflector
    const bool timing = a.prof && unit == 0 && crank == ((a.flags >> 4) & 7) && tid == 0;   // flags: timed CTA
    uint64_t tacc[16] = {};
    uint64_t tmark = 0;
    auto now = []() { return (uint64_t)clock64(); };   // SM cycles (the host converts)
    if (timing) tmark = now();
    auto PH = [&](int k) {
        if (timing) { const uint64_t t = now(); tacc[k] += t - tmark; tmark = t; }
    };
    const int64_t n2v = (n + 1) & ~int64_t(1);
    const int r0 = crank * RL, r1 = (int)min64(n, (int64_t)r0 + RL);
    const int nl = max(0, r1 - r0);
    int pxb = 0;   // exchange buffer parity
    int rpar = 0;  // block_reduce buffer parity
    // Exchange (push model): a CTA stores its record into slot [buffer][its rank] of every CTA
    // of the cluster; after the cluster barrier every read is local.
    auto PXo = [&](int c, int b) -> const double* { return sm.PX + ((size_t)b * CS + c) * XW; };
    // slot k of this CTA's record in buffer b (look-ahead area: b < 0) of CTA c
    auto pub1 = [&](int b, int k, double v, int c) {
        const double* own = (b < 0) ? sm.PXL + (size_t)crank * XW : sm.PX + ((size_t)b * CS + crank) * XW;
        st_cl(cl_addr(own + k, c), v);
    };
    // K scalars (val(k) -> slot, value; every calling thread can evaluate it) to every CTA, one
    // store per thread
    auto pubs = [&](int b, int K, auto val) {
        for (int t = tid; t < K * CS; t += NT) {
            const int k = t / CS, c = t - k * CS;
            int slot;
            const double v = val(k, slot);
            pub1(b, M2 + slot, v, c);
        }
    };
    auto csum = [&](int b, int slot) {   // sum over CTAs of a scalar slot, fixed order
        double v = 0.0;
        for (int c = 0; c < CS; c++) v += PXo(c, b)[M2 + slot];
        return v;
    };
    auto csumL = [&](int slot) {
        double v = 0.0;
        for (int c = 0; c < CS; c++) v += sm.PXL[(size_t)c * XW + M2 + slot];
        return v;
    };
    auto bsync = []() { __syncthreads(); };
    // cluster barrier; a one-CTA cluster only needs the CTA barrier (all its stores are local)
    auto csync = [&]() {
        if (CS == 1) __syncthreads();
        else cl.sync();
    };
    // x rows from CTA 0's back sweep into every CTA's `dst` (called by all threads of CTA 0)
    auto push_x = [&](double* dst) {
        for (int c = 0; c < CS; c++) {
            const uint32_t d = cl_addr(dst, c);
            const int c0 = c * RL, c1 = (int)min64(n, (int64_t)c0 + RL);
#pragma unroll 4
            for (int i = c0 + tid; i < c1; i += NT) st_cl(d + 8u * (uint32_t)(i - c0), sm.tf[i]);
        }
    };
    // forward pass 2 of a chained solve: exact carries from the composed maps (exchange buffer
    // b) -> t rows scattered into CTA 0; rhs(i) the right-hand side's row i (local rows)
    auto fwd_pass2 = [&](const double* Fj, const int8_t* FPj, int fta, int ftb, const Aff& fex, double q0, double sc,
                         int b, auto rhs) {
        Aff pre{1.0, 0.0};
        for (int c2 = 0; c2 < crank; c2++) pre = comp(Aff{PXo(c2, b)[M2 + FA], PXo(c2, b)[M2 + FB]}, pre);
        double cc = fma(fex.a, fma(pre.a, q0, pre.b), fex.b);
        const uint32_t tf0 = cl_addr(sm.tf, 0);
        auto step = [&](int s, double l, double rr, bool sw, double bn) {
            double y;
            if (sw) { y = bn; cc = fma(-l, bn, cc); }
            else { y = cc; cc = fma(-l, cc, bn); }
            st_cl(tf0 + 8u * (uint32_t)s, sc * y * rr);
        };
        int s = fta;
        for (; s + 4 <= ftb; s += 4) {   // the four steps' loads in flight together
            double2 lr[4], bn[4];
            bool sw[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                lr[u] = __ldg(reinterpret_cast<const double2*>(Fj + (int64_t)(s + u) * 4));
                sw[u] = FPj[s + u] != 0;
                bn[u].x = rhs(s + u + 1);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) step(s + u, lr[u].x, lr[u].y, sw[u], bn[u].x);
        }
        for (; s < ftb; s++) {
            const double2 lr = __ldg(reinterpret_cast<const double2*>(Fj + (int64_t)s * 4));
            step(s, lr.x, lr.y, FPj[s] != 0, rhs(s + 1));
        }
        if (ftb == n - 1 && fta < ftb) st_cl(tf0 + 8u * (uint32_t)(n - 1), sc * cc * __ldg(Fj + (n - 1) * 4 + 1));
        else if (n == 1 && tid == 0) st_cl(tf0, sc * cc * __ldg(Fj + 1));
    };
    // forward maps (pass 1) of this thread's steps [fta, ftb), rhs(i) local rows
    auto fwd_maps = [&](const double* Fj, const int8_t* FPj, int fta, int ftb, auto rhs) {
        Aff f{1.0, 0.0};
        auto step = [&](double l, bool sw, double bn) {
            if (sw) f.b = fma(-l, bn, f.b);
            else { f.a = -l * f.a; f.b = fma(-l, f.b, bn); }
        };
        int s = fta;
        for (; s + 4 <= ftb; s += 4) {   // the four steps' loads in flight together
            double l[4], bn[4];
            bool sw[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                l[u] = __ldg(Fj + (int64_t)(s + u) * 4);
                sw[u] = FPj[s + u] != 0;
                bn[u] = rhs(s + u + 1);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) step(l[u], sw[u], bn[u]);
        }
        for (; s < ftb; s++) step(__ldg(Fj + (int64_t)s * 4), FPj[s] != 0, rhs(s + 1));
        return f;
    };
    // this thread's forward steps: CTA c runs steps [max(0, r0-1), min(r1-1, n-1)), which read
    // its own rows of the right-hand side
    const int s0 = max(0, r0 - 1), s1 = (int)min64(r1 - 1, n - 1);
    const int FLn = s1 > s0 ? (s1 - s0 + NT - 1) / NT : 0;
    const int fta = s0 + min(max(s1 - s0, 0), tid * FLn), ftb = s0 + min(max(s1 - s0, 0), (tid + 1) * FLn);
    // the back sweep in CTA 0 (all its threads stage, thread 0 sweeps)
    auto sweep = [&](const double* Fj) {
        (void)Fj;
        if (crank == 0) {
            asm volatile("cp.async.wait_group 0;" ::: "memory");   // this vector's (b, c) rows
            __syncthreads();
            PH(9);
            if (tid == 0) back_sweep_smem(sm.bc, sm.tf, n);
        }
    };

    for (int ci = a.u_off[unit]; ci < a.u_off[unit + 1]; ci++) {
        const int clid = a.u_list[ci];
        const int64_t j1 = a.cstart[clid];
        const int m = (int)(a.cstart[clid + 1] - j1);

        // ================= leader z_{j1} (handover): plain inverse iteration from x^(1), the
        // batched LU's stopping rule (||x||_inf >= sqrt(0.1/n) twice, MAXITS) and chained solves
        // with its factors (Alg. 4 l.5-7 and l.20; the same arithmetic as batched_lu.cu)
        double lscl = 0.0;
        const bool lead = m <= a.handover;
        if (lead) {
            const int64_t j = j1;
            const double* Fj = a.F + j * n * 4;
            const int8_t* FPj = a.FP + j * n;
            if (crank == 0 && tid == 0)
                for (int64_t o = 0; o < n * 4; o += 8192) l2_prefetch_(Fj + o, min64(8192, n * 4 - o));
            if (crank == 0) back_stage_async(Fj, sm.bc, n);
            {
                const double* x1 = a.X1c + j * n2v;
                #pragma unroll 4
                for (int i = tid; i < nl; i += NT) sm.ql[i] = __ldcg(x1 + r0 + i);
            }
            int its = 1, passes = 0;
            while (true) {
                // norms and argmax of the iterate, forward maps of its next solve
                double v[2] = {0.0, 0.0}, qinf = -1.0;
                long long qarg = 0;
                for (int i = tid; i < nl; i += NT) {
                    const double qi = sm.ql[i];
                    v[0] = fma(qi, qi, v[0]);
                    const double aq = fabs(qi);
                    v[1] += aq;
                    if (aq > qinf) { qinf = aq; qarg = r0 + i; }
                }
                block_reduce<2, true>(v, qinf, qarg, sm.red, rpar);   // also orders ql for the maps
                const Aff f = fwd_maps(Fj, FPj, fta, ftb, [&](int64_t i) { return sm.ql[i - r0]; });
                Aff tot;
                const Aff fex = scan_excl(f, reinterpret_cast<Aff*>(sm.acc), tot);
                {
                    const double sg = (qinf >= 0.0 && sm.ql[qarg - r0] < 0.0) ? -1.0 : 1.0;
                    const double q0v = sm.ql[0];
                    pubs(pxb, crank == 0 ? 8 : 7, [&](int k, int& slot) {
                        switch (k) {
                            case 0: slot = Q2; return v[0];
                            case 1: slot = Q1; return v[1];
                            case 2: slot = QINF; return qinf;
                            case 3: slot = QARG; return (double)qarg;
                            case 4: slot = QSGN; return sg;
                            case 5: slot = FA; return tot.a;
                            case 6: slot = FB; return tot.b;
                            default: slot = Q0; return q0v;
                        }
                    });
                }
                csync();
                const double q2t = csum(pxb, Q2);
                double qi = -1.0;
                long long qa = 0;
                int own = 0;
                for (int c2 = 0; c2 < CS; c2++) {
                    const double vv = PXo(c2, pxb)[M2 + QINF];
                    const long long ia = (long long)PXo(c2, pxb)[M2 + QARG];
                    if (vv > qi || (vv == qi && ia < qa)) { qi = vv; qa = ia; own = c2; }
                }
                if (qi >= thr) passes++;
                if (passes >= kPasses || its >= kMaxIts) {
                    lscl = PXo(own, pxb)[M2 + QSGN] / sqrt(q2t);
                    double* zj = a.Z + j * a.ldz;
                    for (int i = tid; i < nl; i += NT) zj[r0 + i] = sm.ql[i] * lscl;
                    if (crank == 0 && tid == 0) {
                        a.iters[j] = its;
                        if (passes < kPasses) atomicAdd(&a.out->nflag, 1);
                    }
                    pxb ^= 1;
                    break;
                }
                its++;
                const double sc = (double)n * a.tnorm * fmax(kEps, __ldg(a.unn + j)) / csum(pxb, Q1);
                fwd_pass2(Fj, FPj, fta, ftb, fex, PXo(0, pxb)[M2 + Q0], sc, pxb, [&](int64_t i) { return sm.ql[i - r0]; });
                pxb ^= 1;
                csync();
                sweep(Fj);
                if (crank == 0) {
                    __syncthreads();
                    push_x(sm.ql);
                }
                csync();
            }
        }

        PH(14);
        // ================= first reflector from z_{j1}; MGS keeps z itself
        if (a.mgs) {
            const double* z = a.Z + j1 * a.ldz;
            for (int i = tid; i < nl; i += NT) sm.Y[ys.at(i, 0)] = lead ? sm.ql[i] * lscl : __ldcg(z + r0 + i);
            __syncthreads();
        } else {
            const double* z = a.Z + j1 * a.ldz;
            double v[1] = {0.0}, dm = 0.0;
            long long di = 0;
            for (int i = tid; i < nl; i += NT) {
                const double zi = lead ? sm.ql[i] * lscl : __ldcg(z + r0 + i);
                sm.ul[i] = zi;
                v[0] = fma(zi, zi, v[0]);
            }
            block_reduce<1, false>(v, dm, di, sm.red, rpar);
            {
                const double u0v = sm.ul[0];
                pubs(pxb, crank == 0 ? 2 : 1, [&](int k, int& slot) {
                    if (k == 0) { slot = U2; return v[0]; }
                    slot = U0;
                    return u0v;
                });
            }
            csync();
            const double un = sqrt(csum(pxb, U2));
            const double u0 = PXo(0, pxb)[M2 + U0];
            const double c = -((u0 >= 0.0) ? 1.0 : -1.0) * un;
            const double tt = 1.0 / (c * c - u0 * c);
            for (int i = tid; i < nl; i += NT) sm.Y[ys.at(i, 0)] = (r0 + i == 0) ? (u0 - c) : sm.ul[i];
            if (tid == 0) sm.T[0] = tt;
            pxb ^= 1;
            __syncthreads();
        }
        PH(15);

        bool la_have = false;
        for (int p = 1; p < m; p++) {
            const int64_t j = j1 + p;
            const double* Fj = a.F + j * n * 4;
            const int8_t* FPj = a.FP + j * n;
            int its = 1, kin = 1, passes = 0, restart = 0;
            bool done = false, flagged = false;
            bool use_la = la_have;
            bool la_done = false;
            la_have = false;
            bool first = true;
            if (crank == 0 && tid == 0 && p + 1 < m) {   // the next vector's factor records into L2
                const double* Fn = Fj + n * 4;             // (this one's were prefetched a vector ago)
                for (int64_t o = 0; o < n * 4; o += 8192) l2_prefetch_(Fn + o, min64(8192, n * 4 - o));
            }
            if (crank == 0 && tid == 0 && p == 1)
                for (int64_t o = 0; o < n * 4; o += 8192) l2_prefetch_(Fj + o, min64(8192, n * 4 - o));
            if (crank == 0) back_stage_async(Fj, sm.bc, n);   // (b, c) for its back sweeps
            if (a.mgs) {
                // ===== Alg. 1 (classical inverse iteration):
                // after every solve, modified Gram-Schmidt against the cluster's accepted
                // vectors z_{j1} .. z_{j-1} (columns 0..p-1 of Y), one cluster-wide reduction
                // per vector in order (l.10-12); then the same test, restarts and chained solve
                // as the compact-WY path.  The projected x is the iterate r of reading 9.
                {
                    const double* x1 = a.X1c + j * n2v;
#pragma unroll 4
                    for (int i = tid; i < nl; i += NT) sm.xl[i] = __ldcg(x1 + r0 + i);
                }
                __syncthreads();
                while (true) {
                    double x2 = 0.0;
                    for (int k = 0; k < p; k++) {
                        double v[2] = {0.0, 0.0}, dm = 0.0;
                        long long di = 0;
                        for (int i = tid; i < nl; i += NT) {
                            v[0] = fma(sm.Y[ys.at(i, k)], sm.xl[i], v[0]);
                            if (k == 0) v[1] = fma(sm.xl[i], sm.xl[i], v[1]);
                        }
                        block_reduce<2, false>(v, dm, di, sm.red, rpar);
                        if (tid < CS) pub1(pxb, 0, v[0], tid);
                        if (k == 0 && tid >= NT - CS) pub1(pxb, M2 + X2, v[1], tid - (NT - CS));
                        csync();
                        double dot = 0.0;
                        for (int c = 0; c < CS; c++) dot += PXo(c, pxb)[0];
                        if (k == 0) x2 = csum(pxb, X2);
                        pxb ^= 1;
                        for (int i = tid; i < nl; i += NT) sm.xl[i] = fma(-dot, sm.Y[ys.at(i, k)], sm.xl[i]);
                    }
                    // norms, argmax and sign of the projected x, forward maps of its solve
                    double v[2] = {0.0, 0.0}, qinf = -1.0;
                    long long qarg = 0;
                    for (int i = tid; i < nl; i += NT) {
                        const double qi = sm.xl[i];
                        v[0] = fma(qi, qi, v[0]);
                        const double aq = fabs(qi);
                        v[1] += aq;
                        if (aq > qinf) { qinf = aq; qarg = r0 + i; }
                    }
                    block_reduce<2, true>(v, qinf, qarg, sm.red, rpar);
                    const Aff f = fwd_maps(Fj, FPj, fta, ftb, [&](int64_t i) { return sm.xl[i - r0]; });
                    Aff tot;
                    const Aff fex = scan_excl(f, reinterpret_cast<Aff*>(sm.acc), tot);
                    {
                        const double sg = (qinf >= 0.0 && sm.xl[qarg - r0] < 0.0) ? -1.0 : 1.0;
                        const double q0v = sm.xl[0];
                        pubs(pxb, crank == 0 ? 8 : 7, [&](int k, int& slot) {
                            switch (k) {
                                case 0: slot = Q2; return v[0];
                                case 1: slot = Q1; return v[1];
                                case 2: slot = QINF; return qinf;
                                case 3: slot = QARG; return (double)qarg;
                                case 4: slot = QSGN; return sg;
                                case 5: slot = FA; return tot.a;
                                case 6: slot = FB; return tot.b;
                                default: slot = Q0; return q0v;
                            }
                        });
                    }
                    csync();
                    const double q2 = csum(pxb, Q2);
                    double qi = -1.0;
                    long long qa = 0;
                    int own = 0;
                    for (int c2 = 0; c2 < CS; c2++) {
                        const double vv = PXo(c2, pxb)[M2 + QINF];
                        const long long ia = (long long)PXo(c2, pxb)[M2 + QARG];
                        if (vv > qi || (vv == qi && ia < qa)) { qi = vv; qa = ia; own = c2; }
                    }
                    const bool degen = p > 0 && sqrt(q2) <= (double)n * kEps * sqrt(x2);   // reading 16
                    if (degen && restart < kMaxRestart) {
                        restart++;
                        its++;
                        kin = 1;
                        passes = 0;
                        const int b = pxb ^ 1;
                        auto rhs = [&](int64_t i) { return start_entry(a.seed, n, j, restart, i); };
                        double w1[1] = {0.0}, dm = 0.0;
                        long long di = 0;
                        for (int i = tid; i < nl; i += NT) w1[0] += fabs(rhs(r0 + i));
                        const Aff fr = fwd_maps(Fj, FPj, fta, ftb, rhs);
                        Aff totr;
                        const Aff exr = scan_excl(fr, reinterpret_cast<Aff*>(sm.acc), totr);
                        block_reduce<1, false>(w1, dm, di, sm.red, rpar);
                        pubs(b, 3, [&](int k, int& slot) {
                            if (k == 0) { slot = FA; return totr.a; }
                            if (k == 1) { slot = FB; return totr.b; }
                            slot = Q1;
                            return w1[0];
                        });
                        csync();
                        const double sc = (double)n * a.tnorm * fmax(kEps, __ldg(a.unn + j)) / csum(b, Q1);
                        fwd_pass2(Fj, FPj, fta, ftb, exr, rhs(0), sc, b, rhs);
                        pxb ^= 1;
                        csync();
                        sweep(Fj);
                        if (crank == 0) {
                            __syncthreads();
                            push_x(sm.xl);
                        }
                        csync();
                        continue;
                    }
                    if (degen) flagged = true;
                    if (qi >= thr) passes++;
                    bool fin = false;
                    if (passes >= kPasses) fin = true;
                    else if (kin >= kMaxIts) { fin = true; flagged = true; }
                    if (fin) {   // Alg. 1 l.14: normalise (sign rule of reading 15); z_j joins Y
                        const double scl = PXo(own, pxb)[M2 + QSGN] / sqrt(q2);
                        double* zj = a.Z + j * a.ldz;
                        for (int i = tid; i < nl; i += NT) {
                            const double zi = sm.xl[i] * scl;
                            zj[r0 + i] = zi;
                            sm.Y[ys.at(i, p)] = zi;
                        }
                        if (crank == 0 && tid == 0) {
                            a.iters[j] = its;
                            if (flagged) atomicAdd(&a.out->nflag, 1);
                        }
                        pxb ^= 1;
                        __syncthreads();
                        break;
                    }
                    its++;
                    kin++;
                    const double sc = (double)n * a.tnorm * fmax(kEps, __ldg(a.unn + j)) / csum(pxb, Q1);
                    fwd_pass2(Fj, FPj, fta, ftb, fex, PXo(0, pxb)[M2 + Q0], sc, pxb,
                              [&](int64_t i) { return sm.xl[i - r0]; });
                    pxb ^= 1;
                    csync();
                    sweep(Fj);
                    if (crank == 0) {
                        __syncthreads();
                        push_x(sm.xl);
                    }
                    csync();
                }
                continue;
            }
            // x^(1)_j into xl (the look-ahead already loaded it into x1l)
            if (use_la) {
                for (int i = tid; i < nl; i += NT) sm.xl[i] = sm.x1l[i];
            } else {
                const double* x1 = a.X1c + j * n2v;
                #pragma unroll 4
                for (int i = tid; i < nl; i += NT) sm.xl[i] = __ldcg(x1 + r0 + i);
            }
            __syncthreads();
            while (!done) {
                double x2;
                // ---------------- A / R1: g = Y_p^T x
                if (first && use_la) {
                    for (int k = tid; k < p - 1; k += NT) {
                        double v = 0.0;
                        for (int c = 0; c < CS; c++) v += sm.PXL[(size_t)c * XW + k];
                        sm.g[k] = v;
                    }
                    if (tid == 0) sm.g[p - 1] = csumL(GPN);
                    x2 = csumL(X2N);
                    __syncthreads();
                } else {
                    double s = 0.0;
                    for (int i = tid; i < nl; i += NT) s = fma(sm.xl[i], sm.xl[i], s);
                    const int b = pxb;
                    const double x2p = colacc(sm, ys, r0, 0, nl, p, [&](int i) { return sm.xl[i]; },
                                              [&](int k, double v, int c) { pub1(b, k, v, c); }, CS, s, 0, NT, bsync);
                    if (tid < CS) pub1(pxb, M2 + X2, x2p, tid);
                    csync();
                    for (int k = tid; k < p; k += NT) {
                        double v = 0.0;
                        for (int c = 0; c < CS; c++) v += PXo(c, pxb)[k];
                        sm.g[k] = v;
                    }
                    x2 = csum(pxb, X2);
                    pxb ^= 1;
                    __syncthreads();
                }
                first = false;
                use_la = false;
                PH(0);
                // ---------------- TT: g' = T_p^T g (replicated); four threads per column (p <= 64)
                {
                    const int k = tid >> 2, sub = tid & 3;
                    double v = 0.0;
                    if (k < p)
                        for (int l = sub; l <= k; l += 4) v = fma(sm.T[l * TS + k], sm.g[l], v);
                    v += __shfl_xor_sync(0xffffffffu, v, 1);
                    v += __shfl_xor_sync(0xffffffffu, v, 2);
                    if (k < p && sub == 0) sm.gp[k] = v;
                }
                __syncthreads();
                PH(1);
                // ---------------- BC: uhat (local rows >= p), s' partial, ||uhat||^2, uhat_p;
                // the owner of row p pushes Y[p, 0..p-1] to every CTA
                {
                    const int ia = max(0, p - r0);
                    double u2 = 0.0;
                    for (int i = ia + tid; i < nl; i += NT) {
                        const double* yr = sm.Y + (size_t)i * M2;
                        const int xk = ys.x(i);
                        double d0 = 0.0, d1 = 0.0;
                        int k = 0;
#pragma unroll 4
                        for (; k + 1 < p; k += 2) {
                            const double2 y = *reinterpret_cast<const double2*>(yr + 2 * ((k >> 1) ^ xk));
                            d0 = fma(y.x, sm.gp[k], d0);
                            d1 = fma(y.y, sm.gp[k + 1], d1);
                        }
                        if (k < p) d0 = fma(yr[2 * ((k >> 1) ^ xk)], sm.gp[k], d0);
                        const double ui = sm.xl[i] - (d0 + d1);
                        sm.ul[i] = ui;
                        u2 = fma(ui, ui, u2);
                    }
                    if (p >= r0 && p < r1)
                        for (int t = tid; t < p * CS; t += NT) {
                            const int k = t / CS, c = t - k * CS;
                            st_cl(cl_addr(sm.yrow + k, c), sm.Y[ys.at(p - r0, k)]);
                        }
                    __syncthreads();
                    const int b = pxb;
                    // (the ordinary sequence of §3.3.1 forms Y^T y in a pass of its own after R2)
                    const double u2s = colacc(sm, ys, r0, ia, nl, a.ordinary ? 0 : p, [&](int i) { return sm.ul[i]; },
                                              [&](int k, double v, int c) { pub1(b, k, v, c); }, CS, u2, 0, NT, bsync);
                    {
                        const double u0v = (p >= r0 && p < r1) ? sm.ul[p - r0] : 0.0;
                        pubs(pxb, 2, [&](int k, int& slot) {
                            if (k == 0) { slot = U2; return u2s; }
                            slot = U0;
                            return u0v;
                        });
                    }
                    csync();
                }
                PH(2);
                // ---------------- R2: scalars; s = s' - c Y[p,:]
                double un = sqrt(csum(pxb, U2));
                double u0 = csum(pxb, U0);
                const bool zero_u = (un == 0.0);
                if (zero_u) { u0 = 1.0; un = 1.0; }
                if (un <= (double)n * kEps * sqrt(x2) && restart < kMaxRestart && !zero_u) {
                    // degenerate iterate (reading 16): restart from a fresh start vector; its
                    // exchange uses the other buffer (the A buffer, read before the BC barrier)
                    restart++;
                    its++;
                    kin = 1;
                    passes = 0;
                    const int b = pxb ^ 1;
                    auto rhs = [&](int64_t i) { return start_entry(a.seed, n, j, restart, i); };
                    double v[1] = {0.0}, dm = 0.0;
                    long long di = 0;
                    for (int i = tid; i < nl; i += NT) v[0] += fabs(rhs(r0 + i));
                    const Aff f = fwd_maps(Fj, FPj, fta, ftb, rhs);
                    Aff tot;
                    const Aff ex = scan_excl(f, reinterpret_cast<Aff*>(sm.acc), tot);
                    block_reduce<1, false>(v, dm, di, sm.red, rpar);
                    pubs(b, 3, [&](int k, int& slot) {
                        if (k == 0) { slot = FA; return tot.a; }
                        if (k == 1) { slot = FB; return tot.b; }
                        slot = Q1;
                        return v[0];
                    });
                    csync();
                    const double sc = (double)n * a.tnorm * fmax(kEps, __ldg(a.unn + j)) / csum(b, Q1);
                    fwd_pass2(Fj, FPj, fta, ftb, ex, rhs(0), sc, b, rhs);
                    pxb ^= 1;   // the buffer used above is now the "previous" one
                    csync();
                    sweep(Fj);
                    if (crank == 0) {
                        __syncthreads();
                        push_x(sm.xl);
                    }
                    csync();
                    first = false;
                    continue;
                }
                if (un <= (double)n * kEps * sqrt(x2)) flagged = true;
                const double c = -((u0 >= 0.0) ? 1.0 : -1.0) * un;
                const double tt = 1.0 / (c * c - u0 * c);
                const double y0 = u0 - c;
                if (a.ordinary) {
                    // §3.3.1: y_j from u_j, then
                    // s = Y_{j-1}^T y_j by its own pass over Y (the DGEMV before `that`) instead of
                    // the reduced sequence's s' - c Y[p,:] from the BC pass
                    pxb ^= 1;
                    const int b = pxb;
                    const int ia = max(0, p - r0);
                    colacc(sm, ys, r0, ia, nl, p,
                           [&](int i) { return (r0 + i == p) ? y0 : (zero_u ? 0.0 : sm.ul[i]); },
                           [&](int k, double v, int cc) { pub1(b, k, v, cc); }, CS, 0.0, 0, NT, bsync);
                    csync();
                    for (int k = tid; k < p; k += NT) {
                        double v = 0.0;
                        for (int cc = 0; cc < CS; cc++) v += PXo(cc, pxb)[k];
                        sm.s[k] = v;
                    }
                } else {
                    for (int k = tid; k < p; k += NT) {
                        double v = 0.0;
                        if (!zero_u)
                            for (int cc = 0; cc < CS; cc++) v += PXo(cc, pxb)[k];
                        sm.s[k] = v - c * sm.yrow[k];
                    }
                }
                pxb ^= 1;
                __syncthreads();
                PH(3);
                // ---------------- TN (replicated): that, x', column p of T; column p of local Y;
                // four threads per row of T (p <= 64)
                {
                    const int l = tid >> 2, sub = tid & 3;
                    double a1 = 0.0, a2 = 0.0;
                    if (l < p) {
                        const double* tr = sm.T + (size_t)l * TS;
                        for (int k = l + sub; k < p; k += 4) {
                            a1 = fma(tr[k], sm.s[k], a1);
                            a2 = fma(tr[k], sm.yrow[k], a2);
                        }
                    }
                    a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
                    a2 += __shfl_xor_sync(0xffffffffu, a2, 1);
                    a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
                    a2 += __shfl_xor_sync(0xffffffffu, a2, 2);
                    if (l < p && sub == 0) {
                        const double that = -tt * a1;
                        sm.xp[l] = a2 + y0 * that;
                        sm.T[(size_t)l * TS + p] = that;
                    }
                }
                if (tid == 0) {
                    sm.xp[p] = tt * y0;
                    sm.T[(size_t)p * TS + p] = tt;
                }
                for (int i = max(0, p - r0) + tid; i < nl; i += NT)
                    sm.Y[ys.at(i, p)] = (r0 + i == p) ? y0 : (zero_u ? 0.0 : sm.ul[i]);
                __syncthreads();
                PH(4);
                // ---------------- D: q = Y_{p+1} x' - e_p, norms, argmax, look-ahead column,
                // forward-sweep chunk maps over this CTA's steps
                Aff fex{1.0, 0.0};
                {
                    double v[3] = {0.0, 0.0, 0.0}, qinf = -1.0;   // ||q||^2, ||q||_1, gpn
                    long long qarg = 0;
                    for (int i = tid; i < nl; i += NT) {
                        const int gi = r0 + i;
                        const int le = min(gi + 1, p + 1);
                        const double* yr = sm.Y + (size_t)i * M2;
                        const int xk = ys.x(i);
                        double d0 = 0.0, d1 = 0.0;
                        int k = 0;
#pragma unroll 4
                        for (; k + 1 < le; k += 2) {
                            const double2 y = *reinterpret_cast<const double2*>(yr + 2 * ((k >> 1) ^ xk));
                            d0 = fma(y.x, sm.xp[k], d0);
                            d1 = fma(y.y, sm.xp[k + 1], d1);
                        }
                        if (k < le) d0 = fma(yr[2 * ((k >> 1) ^ xk)], sm.xp[k], d0);
                        const double qi = (gi == p) ? (d0 + d1) - 1.0 : (d0 + d1);
                        sm.ql[i] = qi;
                        v[0] = fma(qi, qi, v[0]);
                        const double aq = fabs(qi);
                        v[1] += aq;
                        if (aq > qinf) { qinf = aq; qarg = gi; }
                        if (la_done && gi >= p) v[2] = fma(yr[2 * ((p >> 1) ^ xk) + (p & 1)], sm.x1l[i], v[2]);
                    }
                    block_reduce<3, true>(v, qinf, qarg, sm.red, rpar);   // also orders ql for the maps
                    PH(5);
                    const Aff f = fwd_maps(Fj, FPj, fta, ftb, [&](int64_t i) { return sm.ql[i - r0]; });
                    PH(6);
                    Aff tot;
                    fex = scan_excl(f, reinterpret_cast<Aff*>(sm.acc), tot);
                    {
                        const double sg = (qinf >= 0.0 && sm.ql[qarg - r0] < 0.0) ? -1.0 : 1.0;
                        const double q0v = sm.ql[0];
                        pubs(pxb, crank == 0 ? 8 : 7, [&](int k, int& slot) {
                            switch (k) {
                                case 0: slot = Q2; return v[0];
                                case 1: slot = Q1; return v[1];
                                case 2: slot = QINF; return qinf;
                                case 3: slot = QARG; return (double)qarg;
                                case 4: slot = QSGN; return sg;
                                case 5: slot = FA; return tot.a;
                                case 6: slot = FB; return tot.b;
                                default: slot = Q0; return q0v;
                            }
                        });
                        if (tid >= NT - CS) pub1(-1, M2 + GPN, v[2], tid - (NT - CS));
                    }
                    csync();
                    PH(7);
                }
                // ---------------- TEST (replicated)
                const double q2 = csum(pxb, Q2);
                double qinf = -1.0;
                long long qarg = 0;
                int own = 0;
                for (int c2 = 0; c2 < CS; c2++) {
                    const double vv = PXo(c2, pxb)[M2 + QINF];
                    const long long ia = (long long)PXo(c2, pxb)[M2 + QARG];
                    if (vv > qinf || (vv == qinf && ia < qarg)) { qinf = vv; qarg = ia; own = c2; }
                }
                if (fabs(c) * qinf >= thr) passes++;
                if (passes >= kPasses) done = true;
                else if (kin >= kMaxIts) { done = true; flagged = true; }
                if (done) {
                    const double scl = PXo(own, pxb)[M2 + QSGN] / sqrt(q2);
                    double* zj = a.Z + j * a.ldz;
                    for (int i = tid; i < nl; i += NT) zj[r0 + i] = sm.ql[i] * scl;
                    if (crank == 0 && tid == 0) {
                        a.iters[j] = its;
                        if (flagged) atomicAdd(&a.out->nflag, 1);
                    }
                    la_have = la_done;
                    pxb ^= 1;
                    __syncthreads();
                    PH(8);
                } else {
                    its++;
                    kin++;
                    PH(8);
                    // forward pass 2: exact carries -> t rows, gathered into CTA 0
                    const double sc = (double)n * a.tnorm * fmax(kEps, __ldg(a.unn + j)) / csum(pxb, Q1);
                    fwd_pass2(Fj, FPj, fta, ftb, fex, PXo(0, pxb)[M2 + Q0], sc, pxb,
                              [&](int64_t i) { return sm.ql[i - r0]; });
                    pxb ^= 1;
                    csync();
                    PH(10);
                    const bool la = !la_done && p + 1 < m && !(a.flags & 1);
                    sweep(Fj);
                    if (timing) PH(11);
                    if (la) {
                        // look-ahead pass A of vector p+1 (every warp except CTA 0's warp 0):
                        // columns 0..p-1 of Y_{p+1} are final
                        const bool solver = (crank == 0);
                        if (!solver || warp > 0) {
                            const int t0 = solver ? 32 : 0, nth = solver ? NT - 32 : NT;
                            auto ssync = [&]() {
                                if (solver) asm volatile("bar.sync 1, %0;" ::"n"(NT - 32) : "memory");
                                else __syncthreads();
                            };
                            const double* x1 = a.X1c + (j + 1) * n2v;
                            double x2n = 0.0;
#pragma unroll 4
                            for (int i = tid - t0; i < nl; i += nth) {
                                const double v = __ldcg(x1 + r0 + i);
                                sm.x1l[i] = v;
                                x2n = fma(v, v, x2n);
                            }
                            ssync();
                            const double x2s = colacc(sm, ys, r0, 0, nl, p, [&](int i) { return sm.x1l[i]; },
                                                      [&](int k, double v, int c) { pub1(-1, k, v, c); }, CS, x2n, t0,
                                                      nth, ssync);
                            if (tid >= t0 && tid < t0 + CS) pub1(-1, M2 + X2N, x2s, tid - t0);
                        }
                        la_done = true;
                    }
                    PH(12);
                    if (crank == 0) {
                        __syncthreads();   // x complete in CTA 0's tf
                        push_x(sm.xl);
                    }
                    csync();   // x rows in every CTA, look-ahead partials published
                    PH(13);
                }
            }
        }
        csync();   // shared workspace reuse by the unit's next cluster
    }
    if (timing)
        for (int k = 0; k < 16; k++) a.prof[k] = tacc[k];
}

}  // namespace res

size_t resident_smem_bytes(int64_t n, int RL, int M2, int cs) { return sizeof(double) * res::smem_doubles(n, RL, M2, cs); }

cudaError_t launch_resident(const ResArgs& a, int cs, int nunits, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(res::cwy_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (cs > 8) {
        e = cudaFuncSetAttribute(res::cwy_resident_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nunits * cs));
    cfg.blockDim = dim3(res::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, res::cwy_resident_kernel, a);
}

int resident_max_clusters(int cs, size_t smem) {
    cudaFuncSetAttribute(res::cwy_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cs);
    cfg.blockDim = dim3(res::NT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, res::cwy_resident_kernel, &cfg) != cudaSuccess) return 0;
    return nc;
}

}  // namespace tinv
