// bisect.cu -- eigenvalues of the symmetric tridiagonal T by Sturm-count bisection (the
// DSTEBZ step that precedes DSTEIN-cWY).
//
// Sturm count (LDL^T pivots): q_0 = d_0 - x, q_i = (d_i - x) - e_{i-1}^2 / q_{i-1},
// a zero pivot is replaced by -eps ||T||_1 (reading 20); count(x) = #{i : q_i < 0} = number of
// eigenvalues below x.  Every eigenvalue k is bracketed by the Gershgorin interval (padded) and
// bisected until the midpoint equals an endpoint (full fp64 accuracy).  Every operation is an
// explicit round-to-nearest intrinsic in the order written here (no FMA contraction), so each
// Sturm count -- an integer decided by floating point -- is the exact count of that arithmetic.
//
// One thread per eigenvalue; a CTA's threads walk the rows in lockstep with d and e^2 staged in
// shared memory chunks (broadcast reads).
#include "common.cuh"
#include "tinv_internal.h"

namespace tinv {

constexpr int BT = 128;        // threads (eigenvalues) per CTA
constexpr int BCH = 2048;      // rows staged per chunk

// Gershgorin interval, padding, ||T||_1 (one CTA).  Out: bnd[0] = lo, bnd[1] = hi,
// bnd[2] = pivmin.
__global__ void bisect_bounds_kernel(int64_t n, const double* __restrict__ d, const double* __restrict__ e,
                                     double* bnd) {
    __shared__ double s_lo[256], s_hi[256], s_tn[256];
    double lo = d[0], hi = d[0], tn = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double ea = (i > 0) ? fabs(e[i - 1]) : 0.0, eb = (i < n - 1) ? fabs(e[i]) : 0.0;
        double r = 0.0;
        if (i > 0) r = __dadd_rn(r, ea);
        if (i < n - 1) r = __dadd_rn(r, eb);
        lo = fmin(lo, __dsub_rn(d[i], r));
        hi = fmax(hi, __dadd_rn(d[i], r));
        double s = fabs(d[i]);   // ||T||_1 row sum in the order |d_i| + |e_{i-1}| + |e_i|
        if (i > 0) s = __dadd_rn(s, ea);
        if (i < n - 1) s = __dadd_rn(s, eb);
        tn = fmax(tn, s);
    }
    s_lo[threadIdx.x] = lo;
    s_hi[threadIdx.x] = hi;
    s_tn[threadIdx.x] = tn;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int t = 1; t < (int)blockDim.x; t++) {   // min / max: exact in any order
            lo = fmin(lo, s_lo[t]);
            hi = fmax(hi, s_hi[t]);
            tn = fmax(tn, s_tn[t]);
        }
        const double bn = fmax(fabs(lo), fabs(hi));
        const double dmin = 2.2250738585072014e-308;
        double pad = __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, (double)n), kEps), bn), __dmul_rn(2.0, dmin));
        if (tn > 0.0) pad = __dadd_rn(pad, __dmul_rn(__dmul_rn(2.0, kEps), tn));
        bnd[0] = __dsub_rn(lo, pad);
        bnd[1] = __dadd_rn(hi, pad);
        double pivmin = __dmul_rn(kEps, tn);
        if (pivmin == 0.0) pivmin = dmin;
        bnd[2] = pivmin;
    }
}

__global__ void __launch_bounds__(BT) bisect_kernel(int64_t n, const double* __restrict__ d,
                                                    const double* __restrict__ e, const double* __restrict__ bnd,
                                                    double* __restrict__ w) {
    __shared__ double sd[BCH], se2[BCH];
    const int64_t k = (int64_t)blockIdx.x * BT + threadIdx.x;
    const bool live = k < n;
    const double pivmin = bnd[2];
    double lo = bnd[0], hi = bnd[1];
    // bisection; the CTA iterates while any of its eigenvalues is still open
    bool open = live;
    while (__syncthreads_or(open)) {
        double mid = __dadd_rn(lo, __dmul_rn(0.5, __dsub_rn(hi, lo)));
        if (open && (mid <= lo || mid >= hi)) open = false;
        if (!open) mid = lo;   // keeps the lockstep walk; result discarded
        int64_t cnt = 0;
        double q = 0.0;
        for (int64_t c0 = 0; c0 < n; c0 += BCH) {
            const int64_t c1 = (n - c0 < BCH) ? n : c0 + BCH;
            __syncthreads();
            for (int64_t i = c0 + threadIdx.x; i < c1; i += BT) {
                sd[i - c0] = d[i];
                se2[i - c0] = (i > 0) ? __dmul_rn(e[i - 1], e[i - 1]) : 0.0;
            }
            __syncthreads();
            int64_t i = c0;
            if (c0 == 0) {
                q = __dsub_rn(sd[0], mid);
                if (q == 0.0) q = -pivmin;
                cnt += (q < 0.0);
                i = 1;
            }
            for (; i < c1; i++) {
                q = __dsub_rn(__dsub_rn(sd[i - c0], mid), __ddiv_rn(se2[i - c0], q));
                if (q == 0.0) q = -pivmin;
                cnt += (q < 0.0);
            }
        }
        if (open) {
            if (cnt > k) hi = mid;
            else lo = mid;
        }
    }
    if (live) w[k] = __dadd_rn(lo, __dmul_rn(0.5, __dsub_rn(hi, lo)));
}

void launch_bisect(int64_t n, const double* d, const double* e, double* w, double* bnd, cudaStream_t s) {
    bisect_bounds_kernel<<<1, 256, 0, s>>>(n, d, e, bnd);
    bisect_kernel<<<(unsigned)((n + BT - 1) / BT), BT, 0, s>>>(n, d, e, bnd, w);
}

}  // namespace tinv
