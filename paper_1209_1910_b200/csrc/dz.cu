// dz.cu -- the deferred final pass D of the wide compact-WY step ("deferred final
// pass D").
//
// Pass D of the step (§3.3.2) forms
// q_p = Y_{p+1} x'_p - e_p, with x'_p = T_{p+1} Y_{p+1}[p, :]^T, then the stopping test
// |c| ||q||_inf >= sqrt(0.1/n) (Alg. 4) and, on the vector's last
// iteration, z_j = q / ||q||_2 with the sign rule.  In the last iteration nothing later reads q
// except z_j itself, so cwy_kernel parks x'_p (in the vector's dead x^(1) slot) and c instead
// of streaming Y_{p+1} once per vector; here all parked columns of a cluster are formed at once:
//
//     Q = Y X' - E,   Q[i, p] = sum_{k <= min(i, p)} Y[i, k] X'[k, p] - [i == p]
//
// (Y lower trapezoidal n x m in the kernel's packed row layout, X' upper triangular), a dense
// fp64 contraction of ~2 n m^2 / 3 flops instead of ~4 n m^2 bytes of GEMV reads.  Then per
// column: ||q||_2^2, ||q||_inf and its lowest index (the partials of each 128-row tile in a
// fixed order), the test, the sign rule, the scaling.  A parked column whose test fails is
// counted in PrepOut::dzfail and the host re-runs the call without deferral.
//
// dz_gemm_kernel: 128 x 128 output tile per 256-thread CTA, 8 x 8 accumulators per thread (DFMA:
// the measured fp64 tensor-core rate equals the DFMA rate on this part), k-slices of
// 8 through a double-buffered shared-memory stage fed by the next slice's register loads.
#include "common.cuh"
#include "tinv_internal.h"

namespace tinv {

constexpr int DBM = 128, DBN = 128, DBK = 8, DNT = 256;

__global__ void __launch_bounds__(DNT, 1) dz_gemm_kernel(DzArgs a) {
    __shared__ __align__(16) double sbuf[2 * DBK * DBM + 2 * DBK * DBN];   // 32 KB
    double* As = sbuf;                    // [buf][k][row]
    double* Bs = sbuf + 2 * DBK * DBM;    // [buf][k][col]
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    const int64_t n = a.n, m = a.m, p0 = a.p0;
    const int64_t P0 = p0 + (int64_t)blockIdx.x * DBN;
    const int64_t I0 = (int64_t)blockIdx.y * DBM;
    int any = 0;
    if (t < DBN && P0 + t < m) any = (a.c[P0 + t] != 0.0);
    if (!__syncthreads_or(any)) return;   // no parked column in this tile
    const int64_t imax = (I0 + DBM < n ? I0 + DBM : n) - 1, pmax = (P0 + DBN < m ? P0 + DBN : m) - 1;
    const int64_t K = (imax < pmax ? imax : pmax) + 1;   // k in [0, K): k <= i and k <= p

    // loader: this thread's two rows of Y and two columns of X' (fixed over the k slices)
    const int l0 = t >> 2, l1 = l0 + 64, kp = (t & 3) * 2;
    const int64_t ia = I0 + l0, ib = I0 + l1, pa = P0 + l0, pb = P0 + l1;
    const int64_t kya = ia < n ? (ia < m - 1 ? ia : m - 1) : -1;   // last valid k of the row
    const int64_t kyb = ib < n ? (ib < m - 1 ? ib : m - 1) : -1;
    const int64_t kxa = pa < m ? pa : -1, kxb = pb < m ? pb : -1;   // x'_p has p + 1 entries
    const double* ya = a.Y + y_row_off(ia < n ? ia : 0, m);
    const double* yb = a.Y + y_row_off(ib < n ? ib : 0, m);
    const double* xa = a.X + (pa < m ? pa : 0) * a.n2v;
    const double* xb = a.X + (pb < m ? pb : 0) * a.n2v;
    auto ldm = [](const double* base, int64_t k, int64_t kl) -> double2 {
        // k even; the row / column storage holds index k + 1 whenever k <= kl (even padding)
        double2 v = make_double2(0.0, 0.0);
        if (k <= kl) {
            v = __ldg(reinterpret_cast<const double2*>(base + k));
            if (k + 1 > kl) v.y = 0.0;
        }
        return v;
    };
    double2 ra, rb, rc, rd;
    auto load = [&](int64_t k0) {
        const int64_t k = k0 + kp;
        ra = ldm(ya, k, kya);
        rb = ldm(yb, k, kyb);
        rc = ldm(xa, k, kxa);
        rd = ldm(xb, k, kxb);
    };
    auto store = [&](int b) {
        double* A = As + b * DBK * DBM;
        double* B = Bs + b * DBK * DBN;
        A[kp * DBM + l0] = ra.x; A[(kp + 1) * DBM + l0] = ra.y;
        A[kp * DBM + l1] = rb.x; A[(kp + 1) * DBM + l1] = rb.y;
        B[kp * DBN + l0] = rc.x; B[(kp + 1) * DBN + l0] = rc.y;
        B[kp * DBN + l1] = rd.x; B[(kp + 1) * DBN + l1] = rd.y;
    };

    double acc[8][8];
#pragma unroll
    for (int u = 0; u < 8; u++)
#pragma unroll
        for (int v = 0; v < 8; v++) acc[u][v] = 0.0;
    const int nk = (int)((K + DBK - 1) / DBK);
    load(0);
    store(0);
    __syncthreads();
    for (int s = 0; s < nk; s++) {
        const int b = s & 1;
        if (s + 1 < nk) load((int64_t)(s + 1) * DBK);
        const double* A = As + b * DBK * DBM;
        const double* B = Bs + b * DBK * DBN;
#pragma unroll
        for (int kk = 0; kk < DBK; kk++) {
            double2 av[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; u++) av[u] = *reinterpret_cast<const double2*>(A + kk * DBM + ty * 2 + 32 * u);
#pragma unroll
            for (int v = 0; v < 4; v++) bv[v] = *reinterpret_cast<const double2*>(B + kk * DBN + tx * 2 + 32 * v);
#pragma unroll
            for (int u = 0; u < 4; u++)
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    acc[2 * u][2 * v] = fma(av[u].x, bv[v].x, acc[2 * u][2 * v]);
                    acc[2 * u][2 * v + 1] = fma(av[u].x, bv[v].y, acc[2 * u][2 * v + 1]);
                    acc[2 * u + 1][2 * v] = fma(av[u].y, bv[v].x, acc[2 * u + 1][2 * v]);
                    acc[2 * u + 1][2 * v + 1] = fma(av[u].y, bv[v].y, acc[2 * u + 1][2 * v + 1]);
                }
        }
        if (s + 1 < nk) store(b ^ 1);
        __syncthreads();
    }

    // epilogue: q = acc - [i == p] into the parked columns of Z; per-column partials of this
    // tile (sum of squares, max |q| with the lowest row index), reduced over the 16 ty rows of
    // threads in a fixed order through shared memory (the stage buffers are free now)
    double* rq2 = sbuf;                                    // [warp][col]
    double* rqi = sbuf + 8 * DBN;                          // [warp][col]
    double* rqa = sbuf + 16 * DBN;                         // [warp][col] (row index as double)
    const int NPc = (int)(m - p0);
#pragma unroll
    for (int v = 0; v < 4; v++) {
#pragma unroll
        for (int f = 0; f < 2; f++) {
            const int col = tx * 2 + 32 * v + f;
            const int64_t p = P0 + col;
            const bool parked = p < m && a.c[p < m ? p : 0] != 0.0;
            double q2 = 0.0, qi = -1.0;
            int64_t qa = 0;
            double* zc = a.Z + (parked ? p : 0) * a.ldz;
#pragma unroll
            for (int u = 0; u < 4; u++) {
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int64_t i = I0 + ty * 2 + 32 * u + e;
                    if (parked && i < n) {
                        const double q = (i == p) ? acc[2 * u + e][2 * v + f] - 1.0 : acc[2 * u + e][2 * v + f];
                        zc[i] = q;
                        q2 = fma(q, q, q2);
                        const double aq = fabs(q);
                        if (aq > qi || (aq == qi && i < qa)) { qi = aq; qa = i; }
                    }
                }
            }
            // lanes l and l ^ 16 hold the same column (ty = 2w, 2w + 1)
            const double oq2 = __shfl_xor_sync(0xffffffffu, q2, 16);
            const double oqi = __shfl_xor_sync(0xffffffffu, qi, 16);
            const long long oqa = __shfl_xor_sync(0xffffffffu, (long long)qa, 16);
            q2 += oq2;
            if (oqi > qi || (oqi == qi && oqa < qa)) { qi = oqi; qa = oqa; }
            if ((t & 16) == 0) {
                const int w = t >> 5;
                rq2[w * DBN + col] = q2;
                rqi[w * DBN + col] = qi;
                rqa[w * DBN + col] = (double)qa;
            }
        }
    }
    __syncthreads();
    if (t < DBN && P0 + t < m) {
        double q2 = 0.0, qi = -1.0, qa = 0.0;
        for (int w = 0; w < 8; w++) {
            q2 += rq2[w * DBN + t];
            const double oqi = rqi[w * DBN + t], oqa = rqa[w * DBN + t];
            if (oqi > qi || (oqi == qi && oqa < qa)) { qi = oqi; qa = oqa; }
        }
        const int64_t pc = P0 + t - p0, rt = blockIdx.y;
        a.part[(rt * 3 + 0) * NPc + pc] = q2;
        a.part[(rt * 3 + 1) * NPc + pc] = qi;
        a.part[(rt * 3 + 2) * NPc + pc] = qa;
    }
}

// One CTA per parked column: reduce the row tiles' partials, the stopping test, the sign rule
// (largest |entry| positive, lowest index on ties), z_j = sgn q / ||q||_2.
__global__ void __launch_bounds__(DNT) dz_finish_kernel(DzArgs a) {
    __shared__ double red[DNT / 32];
    __shared__ double2 amx[DNT / 32];
    __shared__ double s_scl;
    const int64_t pc = blockIdx.x, p = a.p0 + pc;
    const double c = a.c[p];
    if (c == 0.0) return;
    const int t = threadIdx.x;
    const int64_t n = a.n, NPc = a.m - a.p0, RT = (n + DBM - 1) / DBM;
    double q2 = 0.0, qi = -1.0, qa = 0.0;
    for (int64_t rt = t; rt < RT; rt += DNT) {
        q2 += a.part[(rt * 3 + 0) * NPc + pc];
        const double oqi = a.part[(rt * 3 + 1) * NPc + pc], oqa = a.part[(rt * 3 + 2) * NPc + pc];
        if (oqi > qi || (oqi == qi && oqa < qa)) { qi = oqi; qa = oqa; }
    }
    q2 = block_sum<DNT>(q2, red);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oqi = __shfl_xor_sync(0xffffffffu, qi, o), oqa = __shfl_xor_sync(0xffffffffu, qa, o);
        if (oqi > qi || (oqi == qi && oqa < qa)) { qi = oqi; qa = oqa; }
    }
    if ((t & 31) == 0) amx[t >> 5] = make_double2(qi, qa);
    __syncthreads();
    double* zc = a.Z + p * a.ldz;
    if (t == 0) {
        for (int w = 1; w < DNT / 32; w++) {
            const double2 o = amx[w];
            if (o.x > qi || (o.x == qi && o.y < qa)) { qi = o.x; qa = o.y; }
        }
        if (!(fabs(c) * qi >= sqrt(0.1 / (double)n))) atomicAdd(&a.out->dzfail, 1);   // Alg. 4 test
        atomicAdd(&a.out->dzpark, 1);
        const double sgn = (zc[(int64_t)qa] < 0.0) ? -1.0 : 1.0;
        s_scl = sgn / sqrt(q2);
    }
    __syncthreads();
    const double scl = s_scl;
    for (int64_t i = t; i < n; i += DNT) zc[i] *= scl;
}

cudaError_t launch_dz(const DzArgs& a, cudaStream_t s) {
    if (a.m <= a.p0) return cudaSuccess;
    const dim3 grid((unsigned)((a.m - a.p0 + DBN - 1) / DBN), (unsigned)((a.n + DBM - 1) / DBM));
    dz_gemm_kernel<<<grid, DNT, 0, s>>>(a);
    dz_finish_kernel<<<(unsigned)(a.m - a.p0), DNT, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace tinv
