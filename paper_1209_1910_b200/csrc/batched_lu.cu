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

constexpr int RB = 8;    // rows per stage
// pipeline stages: deep when the grid has at most one warp per SM (small n, latency-bound),
// shallow when several warps share an SM
constexpr int NS_DEEP = 20, NS_SHALLOW = 4;

struct Stage {
    double v[4][RB][32];   // up to four double arrays
    int8_t pv[RB][32];     // pivot bits
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Stage RB rows (row(rr) for rr < RB, skipped when outside [0, n)) of `na` double arrays
// (and optionally the pivot bytes) for the warp's 32 vectors starting at column j0.
__device__ __forceinline__ void stage_rows(Stage& S, int na, const double* const* arr, const int8_t* piv,
                                           int64_t ld, int64_t j0, int64_t n, int64_t base, int dir, int lane) {
    // each 256-byte row segment is 16 chunks of 16 B: lanes 0..15 take even rows, 16..31 odd
    const int half = lane >> 4, ch = lane & 15;
    for (int a = 0; a < na; a++) {
#pragma unroll
        for (int rr = half; rr < RB; rr += 2) {
            const int64_t i = base + dir * rr;
            if (i >= 0 && i < n) cp_async16(&S.v[a][rr][ch * 2], arr[a] + i * ld + j0 + ch * 2);
        }
    }
    if (piv) {   // 32 bytes per row: lanes 0..1 of each half
        if (ch < 2) {
#pragma unroll
            for (int rr = half; rr < RB; rr += 2) {
                const int64_t i = base + dir * rr;
                if (i >= 0 && i < n) cp_async16(&S.pv[rr][ch * 16], piv + i * ld + j0 + ch * 16);
            }
        }
    }
}

template <int NS>
__global__ void __launch_bounds__(32) batched_lu_kernel(BatchedArgs a) {
    extern __shared__ __align__(16) unsigned char bl_smem[];
    Stage* stages = reinterpret_cast<Stage*>(bl_smem);
    const int lane = threadIdx.x;
    const int64_t j0 = (int64_t)blockIdx.x * 32;
    const int64_t j = j0 + lane;
    const int64_t n = a.n;
    const bool live = j < n;
    const int64_t jj = live ? j : n - 1;          // dead lanes shadow a live vector (no stores)
    const int64_t ld = a.ldv;
    const double shift = a.wt[jj];
    const int p = a.jc[jj];
    double tiny = kEps * a.tnorm;
    if (tiny == 0.0) tiny = 2.2250738585072014e-308;
    const double thr = sqrt(0.1 / (double)n);
    double* __restrict__ X = a.X;
    const double* __restrict__ dd = a.d;
    const double* __restrict__ ee = a.e;

    // ---------------- iteration 1: factor + forward elimination of the random start
    double pv_last;
    double b1 = 0.0;  // ||b||_1
    {
        double pp = __ldg(dd) - shift;
        double qq = (n > 1) ? __ldg(ee) : 0.0;
        double c = start_entry(a.seed, n, jj, 0, 0);
        b1 = fabs(c);
#pragma unroll 4
        for (int64_t i = 0; i < n - 1; i++) {
            const double sub = __ldg(ee + i);
            const double anext = __ldg(dd + i + 1) - shift;
            const double enext = (i + 1 < n - 1) ? __ldg(ee + i + 1) : 0.0;
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
            if (live) {
                const int64_t o = i * ld + j;
                __stcg(a.fl + o, l);
                a.fp[o] = sw;
                __stcg(a.fr + o, r);
                __stcg(a.fb + o, u1 * r);
                __stcg(a.fc + o, u2 * r);
                __stcg(X + o, y);
            }
        }
        pv_last = pivot_floor(pp, tiny);
        if (live) {
            const int64_t o = (n - 1) * ld + j;
            __stcg(a.fr + o, 1.0 / pv_last);
            __stcg(a.fb + o, 0.0);
            __stcg(a.fc + o, 0.0);
            __stcg(X + o, c);
        }
    }
    const double unn = fabs(pv_last);
    if (live) a.unn[j] = unn;
    const double sfac = (double)n * a.tnorm * fmax(kEps, unn);
    __syncwarp();
    __threadfence_block();

    // back substitution, in place: x_i = s y_i r_i - b_i x_{i+1} - c_i x_{i+2}
    const int64_t nblk = (n + RB - 1) / RB;
    auto back = [&](double sc, bool keep, double& xinf, double& x1, double& x2, int64_t& imax) {
        const double* arr[4] = {X, a.fr, a.fb, a.fc};
        double xp1 = 0.0, xp2 = 0.0;
        xinf = -1.0; x1 = 0.0; x2 = 0.0; imax = 0;
#pragma unroll
        for (int s = 0; s < NS - 1; s++) {
            if (s < nblk) stage_rows(stages[s], 4, arr, nullptr, ld, j0, n, n - 1 - (int64_t)s * RB, -1, lane);
            cp_async_commit();
        }
        for (int64_t b = 0; b < nblk; b++) {
            const int64_t bn = b + NS - 1;
            if (bn < nblk) stage_rows(stages[bn % NS], 4, arr, nullptr, ld, j0, n, n - 1 - bn * RB, -1, lane);
            cp_async_commit();
            cp_async_wait<NS - 1>();
            __syncwarp();
            const Stage& S = stages[b % NS];
#pragma unroll
            for (int rr = 0; rr < RB; rr++) {
                const int64_t i = n - 1 - b * RB - rr;
                if (i >= 0) {
                    const double t = fma(-S.v[3][rr][lane], xp2, sc * S.v[0][rr][lane] * S.v[1][rr][lane]);
                    const double xi = fma(-S.v[2][rr][lane], xp1, t);
                    if (keep) __stcg(X + i * ld + j, xi);
                    xp2 = xp1;
                    xp1 = xi;
                    const double ax = fabs(xi);
                    if (ax >= xinf) { xinf = ax; imax = i; }   // lowest index on ties (descending)
                    x1 += ax;
                    x2 = fma(xi, xi, x2);
                }
            }
            __syncwarp();
        }
        cp_async_wait<0>();
        __syncwarp();
    };
    // forward elimination of the current iterate (rhs = x, in place): y_i, carried c
    auto forward = [&](bool keep) {
        const double* arrL[1] = {a.fl};
        double c = __ldcg(X + jj);
        const int64_t nf = n - 1;
        const int64_t nb = (nf + RB - 1) / RB;
        const int half = lane >> 4, chk = lane & 15;
        auto issue = [&](int64_t blk) {
            Stage& S = stages[blk % NS];
            stage_rows(S, 1, arrL, a.fp, ld, j0, nf, blk * RB, 1, lane);
            for (int rr = half; rr < RB; rr += 2) {          // rhs rows i+1 -> slot 1
                const int64_t i = blk * RB + rr + 1;
                if (i < n) cp_async16(&S.v[1][rr][chk * 2], X + i * ld + j0 + chk * 2);
            }
        };
#pragma unroll
        for (int s = 0; s < NS - 1; s++) {
            if (s < nb) issue(s);
            cp_async_commit();
        }
        for (int64_t b = 0; b < nb; b++) {
            if (b + NS - 1 < nb) issue(b + NS - 1);
            cp_async_commit();
            cp_async_wait<NS - 1>();
            __syncwarp();
            const Stage& S = stages[b % NS];
#pragma unroll
            for (int rr = 0; rr < RB; rr++) {
                const int64_t i = b * RB + rr;
                if (i < nf) {
                    const double l = S.v[0][rr][lane];
                    const double bn = S.v[1][rr][lane];
                    const bool sw = S.pv[rr][lane] != 0;
                    const double y = sw ? bn : c;
                    c = fma(sw ? 1.0 : -l, c, sw ? -l * bn : bn);
                    if (keep) __stcg(X + i * ld + j, y);
                }
            }
            __syncwarp();
        }
        cp_async_wait<0>();
        if (keep) __stcg(X + (n - 1) * ld + j, c);
        __syncwarp();
        __threadfence_block();
    };

    double xinf, x1, x2;
    int64_t imax;
    back(sfac / b1, live, xinf, x1, x2, imax);
    int its = 1;
    // Vectors with j_c >= 1 hand x^(1) to the compact-WY kernel.  The warp keeps sweeping
    // while any lane still iterates; lanes that are done run the sweeps without storing.
    const bool active = live && p == 0;
    int passes = (xinf >= thr) ? 1 : 0;
    bool want = active && passes < kPasses && its < kMaxIts;
    while (__any_sync(0xffffffffu, want)) {
        const double sc = sfac / x1;
        forward(want);
        double xi_inf, xi1, xi2;
        int64_t im;
        back(sc, want, xi_inf, xi1, xi2, im);
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
        const double xm = __ldcg(X + imax * ld + j);
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
        for (int c = 0; c < 5; c++) tile[c][r][tx] = ok ? __ldcg(src[c] + i * a.ldv + j) : 0.0;
        ptile[r][tx] = ok ? a.fp[i * a.ldv + j] : (int8_t)0;
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
    const int64_t j0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        int64_t i = i0 + r, j = j0 + tx;
        tile[r][tx] = (i < a.n && j < a.n) ? a.X[i * a.ldv + j] : 0.0;
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
    if (nb <= nsm) {
        const size_t sm = sizeof(Stage) * NS_DEEP;
        cudaFuncSetAttribute(batched_lu_kernel<NS_DEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        batched_lu_kernel<NS_DEEP><<<(unsigned)nb, 32, sm, s>>>(a);
    } else {
        batched_lu_kernel<NS_SHALLOW><<<(unsigned)nb, 32, sizeof(Stage) * NS_SHALLOW, s>>>(a);
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
