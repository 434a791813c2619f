// batched_lu.cu -- batched shifted tridiagonal LU inverse iteration.
//
// One lane per eigenvector j, one warp per 32 consecutive vectors.  Factors and iterates
// are interleaved [row i][vector j] so the warp's 32 vectors occupy 256 contiguous bytes
// per row.  Per vector (Eq. (1); Alg. 4 l.5-7):
//   - factor T - wt_j I by Gaussian elimination with partial pivoting (swap iff
//     |e_i| > |pivot|, pivots floored to +-eps*||T||_1), fused with the forward
//     elimination of the start vector b_i = U(-1,1)(seed, j, i) generated in registers;
//   - scale by sigma = n ||T||_1 max(eps, |u_nn|) / ||b||_1 (reading 8; the
//     2-norm normalisation of Alg. 4 l.6 cancels in this ratio) and back-substitute;
//   - vectors that start a cluster (j_c == 0, incl. singletons) keep iterating on their
//     own iterate until the stopping rule (||x||_inf >= sqrt(0.1/n) twice, MAXITS 5);
//     vectors with j_c >= 1 stop after the first solve: x^(1) and the factors go to the
//     compact-WY kernel.
// The sweeps that read stored rows (back substitutions, later forward eliminations) are
// fed by a per-warp cp.async pipeline: NS stages of RB rows x 256 B per array in shared
// memory, so ~NS*RB rows are in flight per lane while the lane runs its serial recurrence
// (one FMA per row on the dependent chain: row-normalised U, alpha/beta forward form).
#include <type_traits>

#include "common.cuh"
#include "tinv_internal.h"

namespace tinv {

constexpr int RB = 16;   // rows per stage
// start-vector ring of the factor sweep (producer warp -> solver warp), aliased onto the
// stage buffers (unused until the first back substitution): kRG slots of RR rows x 32 lanes
constexpr int RR = 32, kRG = 4;
// pipeline stages: deep when the grid has at most one warp per SM (small n, latency-bound),
// shallow when several warps share an SM
constexpr int NS_DEEP = 8, NS_SHALLOW = 2;

struct Stage {
    double v[4][RB][32];   // up to four double arrays, rows of the warp's 32 vectors
    int8_t pv[RB][32];     // pivot bits
};

// One lane issues TMA bulk copies of rows [lo, hi) of `na` arrays (block-row layout: the
// warp's rows are contiguous, 256 B each) into stage S, completing on `bar`.
__device__ __forceinline__ void stage_bulk(Stage& S, uint64_t* bar, int na, const double* const* base, int64_t lo,
                                           int64_t hi, int64_t dst_row0, const int8_t* pbase) {
    if (hi <= lo) {   // nothing to copy: complete the phase with a plain arrive
        mbar_expect_tx(bar, 0);
        return;
    }
    const uint32_t rows = (uint32_t)(hi - lo);
    mbar_expect_tx(bar, rows * 256u * (uint32_t)na + (pbase ? rows * 32u : 0u));
    for (int a = 0; a < na; a++) bulk_g2s(&S.v[a][dst_row0][0], base[a] + lo * 32, rows * 256u, bar);
    if (pbase) bulk_g2s(&S.pv[dst_row0][0], pbase + lo * 32, rows * 32u, bar);
}

// barriers: NS stage slots, d/e staging, kRG full + kRG empty ring slots, producer done
template <int NS>
constexpr int kBars = NS + 1 + 2 * kRG + 1;
template <int NS>
constexpr size_t smem_fixed() { return sizeof(Stage) * NS + ((8 * kBars<NS> + 15) & ~size_t(15)); }

// Reciprocal of a pivot (|u| in [eps ||T||_1, ~||T||_1], never subnormal or infinite): the
// hardware approximation refined by two Newton steps (error far below one ulp of the
// factorisation's own rounding), without the IEEE division's slow-path branch.
__device__ __forceinline__ double rcp_pivot(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    // one third-order step r (1 + e + e^2), e = 1 - x r: relative error delta -> delta^3
    // (three dependent FMAs instead of the four of two Newton steps)
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

// SDE: d and e staged in shared memory (compile-time, so their loads are LDS, not generic)
template <int NS, bool SDE>
__global__ void __launch_bounds__(64) batched_lu_kernel(BatchedArgs a) {
    extern __shared__ __align__(128) unsigned char bl_smem[];
    static_assert(sizeof(Stage) * NS >= sizeof(double) * (RR * kRG + 1) * 32, "start-vector ring exceeds the stages");
    Stage* stages = reinterpret_cast<Stage*>(bl_smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(bl_smem + sizeof(Stage) * NS);
    uint64_t* rfull = bars + NS + 1;
    uint64_t* rempty = rfull + kRG;
    uint64_t* rdone = rempty + kRG;
    double* ring = reinterpret_cast<double*>(bl_smem);
    // small n: d and e staged in shared memory (every warp walks them once per factor sweep;
    // from a cold L1 each 128-byte line would be an L2 round trip next to the dependent chain)
    double* sde = reinterpret_cast<double*>(bl_smem + smem_fixed<NS>());
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;   // 0: solver; 1: start-vector producer (factor sweep only)
    const int64_t n = a.n;
    // this warp's class (prep.cu slot permutation): slots < nc_pad iterate to convergence
    const int64_t ncp = __ldcg(&a.out->nc_pad);
    const bool iter_warp = (int64_t)blockIdx.x * 32 < ncp;
    if ((a.mode == 1 && iter_warp) || (a.mode == 2 && !iter_warp)) return;
    const int64_t j = a.perm[(int64_t)blockIdx.x * 32 + lane];
    const bool live = j >= 0;
    if (!__any_sync(0xffffffffu, live)) return;
    const int64_t jj = live ? j : 0;              // dead lanes shadow vector 0 (no stores)
    const double shift = a.wt[jj];
    const int p = iter_warp ? 0 : 1;              // 0: iterate; 1: hand x^(1) on
    const double tnorm = __ldcg(&a.out->tnorm);   // written by the prep kernel (same stream)
    if (a.out->bad) return;                       // invalid input: nothing is computed
    double tiny = kEps * tnorm;
    if (tiny == 0.0) tiny = 2.2250738585072014e-308;
    const double thr = sqrt(0.1 / (double)n);
    // rcp.approx.ftz flushes subnormal arguments and results: the pivots lie in
    // [eps ||T||_1, ~2 ||T||_1], so outside this range of ||T||_1 the factor sweep takes the
    // IEEE division instead (uniform over the grid)
    const bool exact_rcp = !(tnorm > 0x1p-960 && tnorm < 0x1p1000);
    // this warp's block of rows (block-row layout over slots, common.cuh bix)
    const int64_t boff = (int64_t)blockIdx.x * n * 32;
    double* __restrict__ X = a.X + boff;
    double* __restrict__ FL = a.fl + boff;
    double* __restrict__ FR = a.fr + boff;
    double* __restrict__ FB = a.fb + boff;
    double* __restrict__ FC = a.fc + boff;
    int8_t* __restrict__ FPv = a.fp + boff;
    constexpr bool stage_de = SDE;
    // d staged at sde[0, n2), e at sde[n2, n2 + n) with e[n-1] = 0 (the factor sweep's
    // enext past the last row); the bulk copies move whole 16-byte pairs inside the arrays
    const int64_t n2 = (n + 1) & ~int64_t(1);
    const int64_t dpairs = n & ~int64_t(1), epairs = (n - 1) & ~int64_t(1);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS + 1; s++) mbar_init(bars + s, 1);
        for (int s = 0; s < kRG; s++) {
            mbar_init(rfull + s, 32);
            mbar_init(rempty + s, 1);
        }
        mbar_init(rdone, 32);
        fence_mbar_init();
        if (stage_de) {
            mbar_expect_tx(bars + NS, (uint32_t)((dpairs + epairs) * 8));
            if (dpairs) bulk_g2s(sde, a.d, (uint32_t)(dpairs * 8), bars + NS);
            if (epairs) bulk_g2s(sde + n2, a.e, (uint32_t)(epairs * 8), bars + NS);
        }
    }
    __syncthreads();

    // ---------------- start-vector producer (warp 1): b_i = U(-1,1)(seed, j, i) for rows
    // 1..n-1 of the factor sweep into the ring, and ||b||_1 over those rows
    const int64_t nrow = n - 1;
    if (wid == 1) {
        double bsum = 0.0;
        int64_t k = 0;
        for (int64_t i0 = 0; i0 < nrow; i0 += RR, k++) {
            const int slot = (int)(k % kRG);
            if (k >= kRG) mbar_wait(rempty + slot, (uint32_t)((k / kRG - 1) & 1));
            double* rb = ring + (size_t)slot * RR * 32;
            const int cnt = (int)(nrow - i0 < RR ? nrow - i0 : RR);
            for (int r = 0; r < cnt; r++) {
                const double v = start_entry(a.seed, n, jj, 0, i0 + r + 1);
                rb[r * 32 + lane] = v;
                bsum += fabs(v);
            }
            mbar_arrive(rfull + slot);
        }
        ring[(size_t)kRG * RR * 32 + lane] = bsum;   // just past the ring (inside the stages)
        mbar_arrive(rdone);
        return;
    }
    if (stage_de) {
        mbar_wait(bars + NS, 0);
        if (lane == 0) {   // odd tails and the zero pad
            if (dpairs < n) sde[n - 1] = a.d[n - 1];
            if (epairs < n - 1) sde[n2 + n - 2] = a.e[n - 2];
            sde[n2 + n - 1] = 0.0;
        }
        __syncwarp();
    }
    const double* __restrict__ dd = stage_de ? sde : a.d;
    const double* __restrict__ ee = stage_de ? sde + n2 : a.e;
    uint32_t ph = 0;
    // optional sweep timers (warp 0, lane 0; globaltimer ns): factor+fwd, back 1, fwd 2, back 2
    const bool timing = a.prof && blockIdx.x == 0 && lane == 0;
    auto now = []() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
    uint64_t t_mark = timing ? now() : 0;
    int t_slot = 0;
    auto tick = [&]() {
        if (timing) { const uint64_t t = now(); if (t_slot < 8) a.prof[t_slot++] = t - t_mark; t_mark = t; }
    };

    // ---------------- iteration 1: factor + forward elimination of the random start
    double pv_last;
    double b1 = 0.0;  // ||b||_1
    {
        double pp = dd[0] - shift;
        double qq = (n > 1) ? ee[0] : 0.0;
        double c = start_entry(a.seed, n, jj, 0, 0);
        b1 = fabs(c);
        int64_t k = 0;
        for (int64_t i0 = 0; i0 < nrow; i0 += RR, k++) {
          const int slot = (int)(k % kRG);
          mbar_wait(rfull + slot, (uint32_t)((k / kRG) & 1));
          const double* rb = ring + (size_t)slot * RR * 32;
          const int cnt = (int)(nrow - i0 < RR ? nrow - i0 : RR);
          // this chunk's rows through chunk-base pointers (immediate offsets in the unrolled body)
          const double* pe = ee + i0;
          const double* pd = dd + i0 + 1;
          double* pFL = FL + i0 * 32 + lane;
          double* pFR = FR + i0 * 32 + lane;
          double* pFB = FB + i0 * 32 + lane;
          double* pFC = FC + i0 * 32 + lane;
          double* pX = X + i0 * 32 + lane;
          int8_t* pFP = FPv + i0 * 32 + lane;
          auto row = [&](int rr, auto exact) {
            const int64_t i = i0 + rr;
            const double sub = pe[rr];
            const double anext = pd[rr] - shift;
            const double enext = stage_de ? pe[rr + 1] : ((i + 1 < n - 1) ? pe[rr + 1] : 0.0);
            const double bn = rb[rr * 32 + lane];
            double u0, u1, u2, l, y;
            int8_t sw;
            // one reciprocal per row on the dependent chain (l = other * (1/pivot))
            const bool swp = fabs(sub) > fabs(pp);
            u0 = pivot_floor(swp ? sub : pp, tiny);
            double r;
            if constexpr (decltype(exact)::value) r = 1.0 / u0;   // IEEE (subnormal-safe)
            else r = rcp_pivot(u0);
            l = (swp ? pp : sub) * r;
            if (swp) {
                u1 = anext;
                u2 = enext;
                pp = qq - l * anext;
                qq = -(l * enext);
                y = bn;
                c = c - l * bn;
                sw = 1;
            } else {
                u1 = qq;
                u2 = 0.0;
                pp = anext - l * qq;
                qq = enext;
                y = c;
                c = bn - l * c;
                sw = 0;
            }
            const int o = rr * 32;   // dead lanes store too: their slots are unused
            __stcg(pFL + o, l);
            pFP[o] = sw;
            __stcg(pFR + o, r);
            __stcg(pFB + o, u1 * r);
            __stcg(pFC + o, u2 * r);
            __stcg(pX + o, y);
          };
          if (exact_rcp) {   // ||T||_1 outside [2^-960, 2^1000]: pivots may leave the normal range
            for (int rr = 0; rr < cnt; rr++) row(rr, std::true_type{});
          } else if (cnt == RR) {
#pragma unroll 8
            for (int rr = 0; rr < RR; rr++) row(rr, std::false_type{});
          } else {
            for (int rr = 0; rr < cnt; rr++) row(rr, std::false_type{});
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(rempty + slot);
        }
        mbar_wait(rdone, 0);
        b1 += ring[(size_t)kRG * RR * 32 + lane];
        pv_last = pivot_floor(pp, tiny);
        const int64_t o = (n - 1) * 32 + lane;
        __stcg(FR + o, 1.0 / pv_last);
        __stcg(FB + o, 0.0);
        __stcg(FC + o, 0.0);
        __stcg(X + o, c);
    }
    tick();
    const double unn = fabs(pv_last);
    if (live) a.unn[j] = unn;
    const double sfac = (double)n * tnorm * fmax(kEps, unn);
    // generic writes above -> bulk (async proxy) reads below; the ring's shared memory is
    // reused by the stages (async-proxy writes after generic accesses)
    fence_proxy_async_global();
    fence_proxy_async_smem();
    __syncwarp();

    // back substitution, in place: x_i = s y_i r_i - b_i x_{i+1} - c_i x_{i+2}; stage b holds
    // rows [n - (b+1) RB, n - b RB) (clipped at 0), consumed top-down
    const int64_t nblk = (n + RB - 1) / RB;
    auto back = [&](double sc, bool keep, double& xinf, double& x1, double& x2, int64_t& imax) {
        const double* arr[4] = {X, FR, FB, FC};
        double xp1 = 0.0, xp2 = 0.0;
        xinf = -1.0; x1 = 0.0; x2 = 0.0; imax = 0;
        auto issue = [&](int64_t b) {
            const int64_t hi = n - b * RB, lo = hi - RB > 0 ? hi - RB : 0;
            stage_bulk(stages[b % NS], bars + (b % NS), 4, arr, lo, hi, RB - (hi - lo), nullptr);
        };
        if (lane == 0)
            for (int64_t b = 0; b < NS && b < nblk; b++) issue(b);
        for (int64_t b = 0; b < nblk; b++) {
            mbar_wait(bars + (b % NS), (ph >> (b % NS)) & 1u);
            ph ^= 1u << (b % NS);
            const Stage& S = stages[b % NS];
            // branch-free rows (rows below 0 only occur after row 0: their values are
            // never used, only the statistics and stores are predicated), so the compiler
            // can hoist the shared-memory loads of later rows above the dependent chain; the
            // statistics (||x||_1, ||x||_2^2, argmax) are reduced per stage with fixed trees
            // instead of one dependent chain per row
            const int64_t ib = n - b * RB - RB;
            double xv[RB];
#pragma unroll
            for (int rr = RB - 1; rr >= 0; rr--) {
                const double t = fma(-S.v[3][rr][lane], xp2, sc * S.v[0][rr][lane] * S.v[1][rr][lane]);
                const double xi = fma(-S.v[2][rr][lane], xp1, t);
                xv[rr] = xi;
                xp2 = xp1;
                xp1 = xi;
            }
            if (keep && iter_warp) {
                double* Xb = X + ib * 32 + lane;   // this stage's rows (the first may be partial)
                if (ib >= 0) {
#pragma unroll
                    for (int rr = 0; rr < RB; rr++) __stcg(Xb + rr * 32, xv[rr]);
                } else {
#pragma unroll
                    for (int rr = 0; rr < RB; rr++)
                        if (ib + rr >= 0) __stcg(Xb + rr * 32, xv[rr]);
                }
            } else if (keep && live) {   // first-solve vector: x^(1) straight into its X1c row
                double* xr = a.X1c + j * ((n + 1) & ~int64_t(1)) + ib;
                if (ib >= 0 && !(ib & 1)) {
#pragma unroll
                    for (int rr = 0; rr < RB; rr += 2)
                        __stcg(reinterpret_cast<double2*>(xr + rr), make_double2(xv[rr], xv[rr + 1]));
                } else {
#pragma unroll
                    for (int rr = 0; rr < RB; rr++)
                        if (ib + rr >= 0) __stcg(xr + rr, xv[rr]);
                }
            }
            if (!iter_warp) {   // first-solve warps need no statistics (their iterate goes on)
                __syncwarp();
                if (lane == 0 && b + NS < nblk) issue(b + NS);
                continue;
            }
            double sa[RB], sq[RB];
            int ia[RB];
#pragma unroll
            for (int rr = 0; rr < RB; rr++) {
                const bool valid = ib + rr >= 0;
                sa[rr] = valid ? fabs(xv[rr]) : 0.0;
                sq[rr] = valid ? xv[rr] * xv[rr] : 0.0;
                ia[rr] = rr;
            }
            double mx[RB];
#pragma unroll
            for (int rr = 0; rr < RB; rr++) mx[rr] = (ib + rr >= 0) ? sa[rr] : -1.0;
#pragma unroll
            for (int w = 1; w < RB; w <<= 1) {
#pragma unroll
                for (int rr = 0; rr + w < RB; rr += 2 * w) {
                    sa[rr] += sa[rr + w];
                    sq[rr] += sq[rr + w];
                    // larger value wins; on ties the lower row index
                    const bool tk = mx[rr + w] > mx[rr];
                    mx[rr] = tk ? mx[rr + w] : mx[rr];
                    ia[rr] = tk ? ia[rr + w] : ia[rr];
                }
            }
            x1 += sa[0];
            x2 += sq[0];
            // this stage's rows are lower than every earlier stage's: ties go to this stage
            if (mx[0] >= xinf && mx[0] >= 0.0) {
                xinf = mx[0];
                imax = ib + ia[0];
            }
            __syncwarp();
            if (lane == 0 && b + NS < nblk) issue(b + NS);
        }
        fence_proxy_async_global();
        __syncwarp();
    };
    // forward elimination of the current iterate (rhs = x, in place): y_i, carried c; stage b
    // holds steps i in [b RB, b RB + RB): l_i, pivot bits, and x_{i+1} (in slot 1)
    auto forward = [&](bool keep) {
        double c = __ldcg(X + lane);
        const int64_t nf = n - 1;
        const int64_t nb = (nf + RB - 1) / RB;
        auto issue = [&](int64_t b) {
            const int64_t lo = b * RB, hi = lo + RB < nf ? lo + RB : nf;
            Stage& S = stages[b % NS];
            uint64_t* bar = bars + (b % NS);
            const uint32_t rows = (uint32_t)(hi - lo);
            mbar_expect_tx(bar, rows * (256u * 2u + 32u));
            bulk_g2s(&S.v[0][0][0], FL + lo * 32, rows * 256u, bar);
            bulk_g2s(&S.pv[0][0], FPv + lo * 32, rows * 32u, bar);
            bulk_g2s(&S.v[1][0][0], X + (lo + 1) * 32, rows * 256u, bar);
        };
        if (lane == 0)
            for (int64_t b = 0; b < NS && b < nb; b++) issue(b);
        for (int64_t b = 0; b < nb; b++) {
            mbar_wait(bars + (b % NS), (ph >> (b % NS)) & 1u);
            ph ^= 1u << (b % NS);
            const Stage& S = stages[b % NS];
#pragma unroll
            for (int rr = 0; rr < RB; rr++) {   // branch-free: steps past nf keep c unchanged
                const int64_t i = b * RB + rr;
                const bool valid = i < nf;
                const double l = S.v[0][rr][lane];
                const double bn = S.v[1][rr][lane];
                const bool sw = S.pv[rr][lane] != 0;
                const double y = sw ? bn : c;
                const double cn = fma(sw ? 1.0 : -l, c, sw ? -l * bn : bn);
                c = valid ? cn : c;
                if (keep && valid) __stcg(X + i * 32 + lane, y);
            }
            __syncwarp();
            if (lane == 0 && b + NS < nb) issue(b + NS);
        }
        if (keep) __stcg(X + (n - 1) * 32 + lane, c);
        fence_proxy_async_global();
        __syncwarp();
    };

    double xinf, x1, x2;
    int64_t imax;
    back(sfac / b1, true, xinf, x1, x2, imax);
    tick();
    int its = 1;
    // Vectors with j_c >= 1 (and, with handover, the leaders of resident clusters) hand x^(1)
    // to the compact-WY kernels: their warps stop here.  Iterating warps keep sweeping while
    // any lane still iterates; lanes that are done run the sweeps without storing.
    const bool active = live && p == 0;
    int passes = (xinf >= thr) ? 1 : 0;
    bool want = active && passes < kPasses && its < kMaxIts;
    while (__any_sync(0xffffffffu, want)) {
        const double sc = sfac / x1;
        forward(want);
        tick();
        double xi_inf, xi1, xi2;
        int64_t im;
        back(sc, want, xi_inf, xi1, xi2, im);
        tick();
        if (want) {
            its++;
            xinf = xi_inf; x1 = xi1; x2 = xi2; imax = im;
            if (xinf >= thr) passes++;
        }
        want = active && passes < kPasses && its < kMaxIts;
    }
    if (!live) return;
    if (p == 0) {
        if (passes < kPasses) atomicAdd(&a.out->nflag, 1);
        // Alg. 4 l.20 normalise; sign rule (reading 15)
        const double xm = __ldcg(X + imax * 32 + lane);
        a.zscale[j] = (xm < 0.0 ? -1.0 : 1.0) / sqrt(x2);
    }
    a.iters[j] = its;
}

// Per-vector contiguous copy of the factors of the first-solve vectors (slots >= nc_pad: j_c >= 1
// and handed-over leaders) for the chained solves of the compact-WY kernels:
// F[j][i] = (l_i, 1/u0_i, u1_i/u0_i, u2_i/u0_i) and the pivot byte, via 32x32 shared-memory
// tiles (coalesced on both sides).  (Their first iterates x^(1) are written per vector by the
// batched kernel's back sweep directly.)
__global__ void pack_factors_kernel(PackArgs a) {
    __shared__ double tile[4][32][33];
    __shared__ int8_t ptile[32][33];
    __shared__ int vec[32];
    const int64_t s0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
    if (s0 < __ldcg(&a.out->nc_pad)) return;   // iterating warp: nothing to pack
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    if (ty == 0) vec[tx] = a.perm[s0 + tx];
    __syncthreads();
    if (vec[0] < 0 && !__syncthreads_or(vec[tx] >= 0)) return;
    const double* src[4] = {a.fl, a.fr, a.fb, a.fc};
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = i0 + r;
        const bool ok = i < a.n;
        for (int c = 0; c < 4; c++) tile[c][r][tx] = ok ? __ldcg(src[c] + bix(i, s0 + tx, a.n)) : 0.0;
        ptile[r][tx] = ok ? a.fp[bix(i, s0 + tx, a.n)] : (int8_t)0;
    }
    __syncthreads();
    // write: vector of slot s0+r, rows i0..i0+31 -> 32 x 4 doubles contiguous (1 KB)
    for (int r = ty; r < 32; r += 8) {
        const int64_t j = vec[r];
        if (j < 0) continue;
        const int64_t i = i0 + tx;
        if (i < a.n) {
            double* dst = a.F + (j * a.n + i) * 4;
            __stcg(reinterpret_cast<double2*>(dst), make_double2(tile[0][tx][r], tile[1][tx][r]));
            __stcg(reinterpret_cast<double2*>(dst + 2), make_double2(tile[2][tx][r], tile[3][tx][r]));
            a.FP[j * a.n + i] = ptile[tx][r];
        }
    }
}

void launch_pack(const PackArgs& a, cudaStream_t s) {
    dim3 grid((unsigned)(batched_slot_cap(a.n) / 32), (unsigned)((a.n + 31) / 32));
    pack_factors_kernel<<<grid, dim3(32, 8), 0, s>>>(a);
}

// Tiled transpose + scale of finished iterates (slots < nc_pad) into column-major Z.
__global__ void finalize_kernel(FinalizeArgs a) {
    __shared__ double tile[32][33];
    __shared__ int vec[32];
    if (a.out->bad || a.out->tnorm == 0.0) return;   // invalid input / Z = I (host handles)
    const int64_t s0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
    if (s0 >= __ldcg(&a.out->nc_pad)) return;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    if (ty == 0) vec[tx] = a.perm[s0 + tx];
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = i0 + r;
        tile[r][tx] = (i < a.n) ? a.X[bix(i, s0 + tx, a.n)] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t j = vec[r], i = i0 + tx;
        if (j >= 0 && i < a.n) a.Z[j * a.ldz + i] = tile[tx][r] * a.zscale[j];
    }
}

__global__ void identity_kernel(double* Z, int64_t n, int64_t ldz) {
    int64_t j = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        Z[j * ldz + i] = (i == j) ? 1.0 : 0.0;
}

int64_t batched_slot_cap(int64_t n) { return (n + 31) / 32 * 32 + 32; }

void launch_batched(const BatchedArgs& a, cudaStream_t s, int nsm) {
    const int64_t nb = batched_slot_cap(a.n) / 32;
    BatchedArgs b = a;
    if (nb <= nsm) {
        const size_t de = (size_t)(((a.n + 1) & ~int64_t(1)) + a.n) * 8;
        size_t sm = smem_fixed<NS_DEEP>();
        b.stage_de = (sm + de <= 200 * 1024) ? 1 : 0;
        if (b.stage_de) {
            sm += de;
            cudaFuncSetAttribute(batched_lu_kernel<NS_DEEP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            batched_lu_kernel<NS_DEEP, true><<<(unsigned)nb, 64, sm, s>>>(b);
        } else {
            cudaFuncSetAttribute(batched_lu_kernel<NS_DEEP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            batched_lu_kernel<NS_DEEP, false><<<(unsigned)nb, 64, sm, s>>>(b);
        }
    } else {
        b.stage_de = 0;
        const size_t sm = smem_fixed<NS_SHALLOW>();
        cudaFuncSetAttribute(batched_lu_kernel<NS_SHALLOW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        batched_lu_kernel<NS_SHALLOW, false><<<(unsigned)nb, 64, sm, s>>>(b);
    }
}

void launch_finalize(const FinalizeArgs& a, cudaStream_t s) {
    dim3 grid((unsigned)(batched_slot_cap(a.n) / 32), (unsigned)((a.n + 31) / 32));
    finalize_kernel<<<grid, dim3(32, 8), 0, s>>>(a);
}

void launch_identity(double* Z, int64_t n, int64_t ldz, cudaStream_t s) {
    dim3 grid((unsigned)((n + 255) / 256 > 64 ? 64 : (n + 255) / 256), (unsigned)n);
    identity_kernel<<<grid, 256, 0, s>>>(Z, n, ldz);
}

}  // namespace tinv
