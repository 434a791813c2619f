// batched_lu.cu -- batched shifted tridiagonal LU inverse iteration.
//
// One thread per eigenvector j; the factors and iterates are interleaved [row i][vector j]
// so a warp's 32 vectors touch 256 contiguous bytes per row (coalesced), and d, e are
// broadcast reads (L1/L2).  Per vector (Eq. (1); Alg. 4 l.5-7):
//   - factor T - wt_j I by Gaussian elimination with partial pivoting (swap iff
//     |e_i| > |pivot|, pivots floored to +-eps*||T||_1), fused with the forward
//     elimination of the start vector b_i = U(-1,1)(seed, j, i) generated in registers;
//   - scale by sigma = n ||T||_1 max(eps, |u_nn|) / ||b||_1 (reading 8; the
//     2-norm normalisation of Alg. 4 l.6 cancels in this ratio) and back-substitute;
//   - vectors that start a cluster (j_c == 0, incl. singletons) keep iterating on their
//     own iterate until the stopping rule (||x||_inf >= sqrt(0.1/n) twice, MAXITS 5);
//     vectors with j_c >= 1 stop after the first solve: their x^(1) and the factors go
//     to the compact-WY kernel.
// The back substitution uses the row-normalised U (1/u0, u1/u0, u2/u0) so the dependent
// chain is a single FMA per row.
#include "common.cuh"
#include "tinv_internal.h"

namespace tinv {

constexpr int kBatchThreads = 64;

__global__ void __launch_bounds__(kBatchThreads) batched_lu_kernel(BatchedArgs a) {
    const int64_t j = (int64_t)blockIdx.x * kBatchThreads + threadIdx.x;
    const int64_t n = a.n;
    if (j >= n) return;
    const int64_t ld = a.ldv;
    const double shift = a.wt[j];
    const int p = a.jc[j];
    double tiny = kEps * a.tnorm;
    if (tiny == 0.0) tiny = 2.2250738585072014e-308;
    const double thr = sqrt(0.1 / (double)n);
    double* __restrict__ X = a.X;

    // ---------------- iteration 1: factor + forward elimination of the random start
    double pv_last;
    double b1 = 0.0;  // ||b||_1
    {
        double pp = a.d[0] - shift;
        double qq = (n > 1) ? a.e[0] : 0.0;
        double c = start_entry(a.seed, n, j, 0, 0);
        b1 = fabs(c);
        for (int64_t i = 0; i < n - 1; i++) {
            const double sub = a.e[i];
            const double anext = a.d[i + 1] - shift;
            const double enext = (i + 1 < n - 1) ? a.e[i + 1] : 0.0;
            const double bn = start_entry(a.seed, n, j, 0, i + 1);
            b1 += fabs(bn);
            double u0, u1, u2, l, y;
            int8_t sw;
            if (fabs(sub) > fabs(pp)) {
                u0 = pivot_floor(sub, tiny);
                u1 = anext;
                u2 = enext;
                l = pp / u0;
                pp = qq - l * anext;
                qq = -(l * enext);
                y = bn;
                c = c - l * bn;
                sw = 1;
            } else {
                u0 = pivot_floor(pp, tiny);
                u1 = qq;
                u2 = 0.0;
                l = sub / u0;
                pp = anext - l * qq;
                qq = enext;
                y = c;
                c = bn - l * c;
                sw = 0;
            }
            const double r = 1.0 / u0;
            const int64_t o = i * ld + j;
            a.fl[o] = l;
            a.fp[o] = sw;
            a.fr[o] = r;
            a.fb[o] = u1 * r;
            a.fc[o] = u2 * r;
            X[o] = y;
        }
        pv_last = pivot_floor(pp, tiny);
        const int64_t o = (n - 1) * ld + j;
        a.fr[o] = 1.0 / pv_last;
        a.fb[o] = 0.0;
        a.fc[o] = 0.0;
        X[o] = c;
    }
    const double unn = fabs(pv_last);
    a.unn[j] = unn;
    const double sfac = (double)n * a.tnorm * fmax(kEps, unn);

    // back substitution, in place: x_i = s y_i r_i - b_i x_{i+1} - c_i x_{i+2}
    auto back = [&](double sc, double& xinf, double& x1, double& x2, int64_t& imax) {
        double xp1 = 0.0, xp2 = 0.0;
        xinf = -1.0; x1 = 0.0; x2 = 0.0; imax = 0;
        for (int64_t i = n - 1; i >= 0; i--) {
            const int64_t o = i * ld + j;
            const double t = fma(-a.fc[o], xp2, sc * X[o] * a.fr[o]);
            const double xi = fma(-a.fb[o], xp1, t);
            X[o] = xi;
            xp2 = xp1;
            xp1 = xi;
            const double ax = fabs(xi);
            if (ax >= xinf) { xinf = ax; imax = i; }   // lowest index on ties (descending loop)
            x1 += ax;
            x2 = fma(xi, xi, x2);
        }
    };
    double xinf, x1, x2;
    int64_t imax;
    back(sfac / b1, xinf, x1, x2, imax);
    int its = 1;
    if (p != 0) {          // clustered: x^(1) handed to the compact-WY kernel
        a.iters[j] = its;
        return;
    }
    int passes = (xinf >= thr) ? 1 : 0;
    while (passes < kPasses && its < kMaxIts) {
        its++;
        // forward elimination of the current iterate (rhs = x, in place)
        double c = X[j];
        for (int64_t i = 0; i < n - 1; i++) {
            const int64_t o = i * ld + j;
            const double bn = X[o + ld];
            const double l = a.fl[o];
            double y;
            if (a.fp[o]) { y = bn; c = fma(-l, bn, c); }
            else         { y = c;  c = fma(-l, c, bn); }
            X[o] = y;
        }
        X[(n - 1) * ld + j] = c;
        back(sfac / x1, xinf, x1, x2, imax);
        if (xinf >= thr) passes++;
    }
    if (passes < kPasses) atomicAdd(&a.out->nflag, 1);
    // Alg. 4 l.20 normalise; sign rule (reading 15)
    const double xm = X[imax * ld + j];
    a.zscale[j] = (xm < 0.0 ? -1.0 : 1.0) / sqrt(x2);
    a.iters[j] = its;
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

void launch_batched(const BatchedArgs& a, cudaStream_t s) {
    int64_t nb = (a.n + kBatchThreads - 1) / kBatchThreads;
    batched_lu_kernel<<<(unsigned)nb, kBatchThreads, 0, s>>>(a);
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
