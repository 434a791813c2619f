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
#include "common.cuh"
#include "tinv_internal.h"

namespace tinv {

constexpr int RB = 16;   // rows per stage
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

template <int NS>
__global__ void __launch_bounds__(32) batched_lu_kernel(BatchedArgs a) {
    extern __shared__ __align__(128) unsigned char bl_smem[];
    Stage* stages = reinterpret_cast<Stage*>(bl_smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(bl_smem + sizeof(Stage) * NS);
    // small n: d and e staged in shared memory (every warp walks them once per factor sweep;
    // from a cold L1 each 128-byte line would be an L2 round trip next to the dependent chain)
    double* sde = reinterpret_cast<double*>(bl_smem + sizeof(Stage) * NS + 8 * (NS + 2));
    const int lane = threadIdx.x;
    const int64_t j0 = (int64_t)blockIdx.x * 32;
    const int64_t j = j0 + lane;
    const int64_t n = a.n;
    const bool live = j < n;
    const int64_t jj = live ? j : n - 1;          // dead lanes shadow a live vector (no stores)
    const double shift = a.wt[jj];
    const int p = a.jc[jj];
    const double tnorm = __ldcg(&a.out->tnorm);   // written by the prep kernel (same stream)
    if (a.out->bad) return;                       // invalid input: nothing is computed
    double tiny = kEps * tnorm;
    if (tiny == 0.0) tiny = 2.2250738585072014e-308;
    const double thr = sqrt(0.1 / (double)n);
    // this warp's block of rows (block-row layout, common.cuh bix)
    const int64_t boff = (int64_t)blockIdx.x * n * 32;
    double* __restrict__ X = a.X + boff;
    double* __restrict__ FL = a.fl + boff;
    double* __restrict__ FR = a.fr + boff;
    double* __restrict__ FB = a.fb + boff;
    double* __restrict__ FC = a.fc + boff;
    int8_t* __restrict__ FPv = a.fp + boff;
    const bool stage_de = a.stage_de != 0;
    if (lane == 0) {
        for (int s = 0; s < NS + 1; s++) mbar_init(bars + s, 1);
        fence_mbar_init();
        if (stage_de) {
            const uint32_t bd = (uint32_t)(((n + 1) & ~int64_t(1)) * 8), be = (uint32_t)((n & ~int64_t(1)) * 8);
            mbar_expect_tx(bars + NS, bd + be);
            bulk_g2s(sde, a.d, bd, bars + NS);
            if (be) bulk_g2s(sde + ((n + 1) & ~int64_t(1)), a.e, be, bars + NS);
        }
    }
    __syncwarp();
    if (stage_de) mbar_wait(bars + NS, 0);
    const double* __restrict__ dd = stage_de ? sde : a.d;
    const double* __restrict__ ee = stage_de ? sde + ((n + 1) & ~int64_t(1)) : a.e;
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
#pragma unroll 4
        for (int64_t i = 0; i < n - 1; i++) {
            const double sub = ee[i];
            const double anext = dd[i + 1] - shift;
            const double enext = (i + 1 < n - 1) ? ee[i + 1] : 0.0;
            const double bn = start_entry(a.seed, n, jj, 0, i + 1);
            b1 += fabs(bn);
            double u0, u1, u2, l, y;
            int8_t sw;
            // one reciprocal per row on the dependent chain (l = other * (1/pivot))
            const bool swp = fabs(sub) > fabs(pp);
            u0 = pivot_floor(swp ? sub : pp, tiny);
            const double r = 1.0 / u0;
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
            const int64_t o = i * 32 + lane;
            __stcg(FL + o, l);
            FPv[o] = sw;
            __stcg(FR + o, r);
            __stcg(FB + o, u1 * r);
            __stcg(FC + o, u2 * r);
            __stcg(X + o, y);
        }
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
    // generic writes above -> bulk (async proxy) reads below
    fence_proxy_async_global();
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
            double sa[RB], sq[RB];
            int ia[RB];
#pragma unroll
            for (int rr = 0; rr < RB; rr++) {
                const bool valid = ib + rr >= 0;
                if (keep && valid) __stcg(X + (ib + rr) * 32 + lane, xv[rr]);
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
    // Vectors with j_c >= 1 hand x^(1) to the compact-WY kernel.  The warp keeps sweeping
    // while any lane still iterates; lanes that are done run the sweeps without storing.
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

// Per-vector contiguous copy of the factors of clustered vectors (j_c >= 1) for the chained
// solves of the compact-WY kernel: F[j][i] = (l_i, 1/u0_i, u1_i/u0_i, u2_i/u0_i), the pivot
// byte, and the first iterate x^(1) (contiguous per vector, so the compact-WY passes can
// bulk-copy it), via 32x32 shared-memory tiles (coalesced on both sides).
__global__ void pack_factors_kernel(PackArgs a) {
    __shared__ double tile[5][32][33];
    __shared__ int8_t ptile[32][33];
    __shared__ int any;
    const int64_t j0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    if (tx == 0 && ty == 0) any = 0;
    __syncthreads();
    if (ty == 0 && j0 + tx < a.n && a.jc[j0 + tx] != 0) any = 1;
    __syncthreads();
    if (!any) return;
    const double* src[5] = {a.fl, a.fr, a.fb, a.fc, a.X};
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = i0 + r, j = j0 + tx;
        const bool ok = i < a.n && j < a.n;
        for (int c = 0; c < 5; c++) tile[c][r][tx] = ok ? __ldcg(src[c] + bix(i, j, a.n)) : 0.0;
        ptile[r][tx] = ok ? a.fp[bix(i, j, a.n)] : (int8_t)0;
    }
    __syncthreads();
    // write: vector j0+r, rows i0..i0+31 -> 32 x 4 doubles contiguous (1 KB)
    for (int r = ty; r < 32; r += 8) {
        const int64_t j = j0 + r;
        if (j >= a.n || a.jc[j] == 0) continue;
        const int64_t i = i0 + tx;
        if (i < a.n) {
            double* dst = a.F + (j * a.n + i) * 4;
            __stcg(reinterpret_cast<double2*>(dst), make_double2(tile[0][tx][r], tile[1][tx][r]));
            __stcg(reinterpret_cast<double2*>(dst + 2), make_double2(tile[2][tx][r], tile[3][tx][r]));
            a.FP[j * a.n + i] = ptile[tx][r];
            __stcg(a.X1c + j * ((a.n + 1) & ~int64_t(1)) + i, tile[4][tx][r]);
        }
    }
}

void launch_pack(const PackArgs& a, cudaStream_t s) {
    dim3 grid((unsigned)((a.n + 31) / 32), (unsigned)((a.n + 31) / 32));
    pack_factors_kernel<<<grid, dim3(32, 8), 0, s>>>(a);
}

// Tiled transpose + scale of finished iterates into column-major Z (j_c == 0 vectors).
__global__ void finalize_kernel(FinalizeArgs a) {
    __shared__ double tile[32][33];
    if (a.out->bad || a.out->tnorm == 0.0) return;   // invalid input / Z = I (host handles)
    const int64_t j0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        int64_t i = i0 + r, j = j0 + tx;
        tile[r][tx] = (i < a.n && j < a.n) ? a.X[bix(i, j, a.n)] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        int64_t j = j0 + r, i = i0 + tx;
        if (j < a.n && i < a.n && a.jc[j] == 0) a.Z[j * a.ldz + i] = tile[tx][r] * a.zscale[j];
    }
}

__global__ void identity_kernel(double* Z, int64_t n, int64_t ldz) {
    int64_t j = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        Z[j * ldz + i] = (i == j) ? 1.0 : 0.0;
}

void launch_batched(const BatchedArgs& a, cudaStream_t s, int nsm) {
    int64_t nb = (a.n + 31) / 32;
    BatchedArgs b = a;
    if (nb <= nsm) {
        const size_t de = (size_t)(((a.n + 1) & ~int64_t(1)) + (a.n & ~int64_t(1))) * 8;
        size_t sm = sizeof(Stage) * NS_DEEP + 8 * (NS_DEEP + 2);
        b.stage_de = (sm + de <= 200 * 1024) ? 1 : 0;
        if (b.stage_de) sm += de;
        cudaFuncSetAttribute(batched_lu_kernel<NS_DEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        batched_lu_kernel<NS_DEEP><<<(unsigned)nb, 32, sm, s>>>(b);
    } else {
        b.stage_de = 0;
        const size_t sm = sizeof(Stage) * NS_SHALLOW + 8 * (NS_SHALLOW + 2);
        cudaFuncSetAttribute(batched_lu_kernel<NS_SHALLOW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        batched_lu_kernel<NS_SHALLOW><<<(unsigned)nb, 32, sm, s>>>(b);
    }
}

void launch_finalize(const FinalizeArgs& a, cudaStream_t s) {
    dim3 grid((unsigned)((a.n + 31) / 32), (unsigned)((a.n + 31) / 32));
    finalize_kernel<<<grid, dim3(32, 8), 0, s>>>(a);
}

void launch_identity(double* Z, int64_t n, int64_t ldz, cudaStream_t s) {
    dim3 grid((unsigned)((n + 255) / 256 > 64 ? 64 : (n + 255) / 256), (unsigned)n);
    identity_kernel<<<grid, 256, 0, s>>>(Z, n, ldz);
}

}  // namespace tinv
