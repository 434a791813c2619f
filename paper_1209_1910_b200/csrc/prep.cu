// prep.cu -- ||T||_1, input validation, Peters-Wilkinson cluster segmentation and the
// shift ladder.  One CTA; O(n).
//
//  R1  tnorm = max_i |d_i| + |e_{i-1}| + |e_i|
//  R2  j starts a cluster iff j == 0 or w_j - w_{j-1} > 1e-3 tnorm   (Alg. 4 l.8)
//  R3  wt_j = max(w_j, wt_{j-1} + 10 eps |w_j|) inside a cluster      (reading 5)
// The arithmetic is written with explicit _rn intrinsics so the compiler cannot contract
// it: the cluster table must equal the one the rules define, bit for bit.
#include "common.cuh"
#include "tinv_internal.h"

namespace tinv {

constexpr int kPrepThreads = 1024;

__global__ void __launch_bounds__(kPrepThreads) prep_kernel(PrepArgs a) {
    __shared__ double red[kPrepThreads / 32];
    __shared__ int sscan[kPrepThreads / 32];
    __shared__ int s_carry;
    __shared__ int s_bad;
    const int64_t n = a.n;
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_bad = 0;
        s_carry = 0;
        *a.out = PrepOut{};   // the call's summary starts from zero (the later kernels accumulate)
    }
    __syncthreads();

    // ---- R1 + validation
    double tl = 0.0;
    int bad = 0;
    for (int64_t i = tid; i < n; i += kPrepThreads) {
        double di = a.d[i];
        double s = fabs(di);
        if (i > 0) s = __dadd_rn(s, fabs(a.e[i - 1]));
        if (i < n - 1) s = __dadd_rn(s, fabs(a.e[i]));
        tl = fmax(tl, s);
        double wi = a.w[i];
        if (!isfinite(di)) bad |= 1;                          // argument d
        if (i < n - 1 && !isfinite(a.e[i])) bad |= 2;         // argument e
        if (!isfinite(wi)) bad |= 4;                          // argument w
        if (i > 0 && !(wi >= a.w[i - 1])) bad |= 4;           // w not ascending
    }
    tl = warp_max(tl);
    if ((tid & 31) == 0) red[tid >> 5] = tl;
    if (bad) atomicOr(&s_bad, bad);
    __syncthreads();
    if (tid < 32) {
        double v = red[tid];
        v = warp_max(v);
        if (tid == 0) red[0] = v;
    }
    __syncthreads();
    double tnorm = red[0];
    if (s_bad) {
        if (tid == 0) { a.out->tnorm = tnorm; a.out->bad = s_bad; }
        return;
    }
    // ---- R0 (reading 21): ||T||_1 outside [2^-200, 2^200] -> T and w scaled by
    // the power of two 2^k with 2^k ||T||_1 in [1, 2) (exact; same eigenvectors), so that the
    // solve's scaling sigma, the pivots' reciprocals and the norms stay in the normal range.
    // The kernels read d, e through the copies ds, es in either case.
    int k = 0;
    if (tnorm > 0.0 && !(tnorm >= 0x1p-200 && tnorm <= 0x1p200)) {
        int ex;
        frexp(tnorm, &ex);
        k = 1 - ex;
    }
    for (int64_t i = tid; i < n; i += kPrepThreads) {
        a.ds[i] = ldexp(a.d[i], k);
        a.es[i] = (i < n - 1) ? ldexp(a.e[i], k) : 0.0;
    }
    if (k != 0) {   // ||T||_1 of the scaled matrix, in the order of R1
        __syncthreads();
        tl = 0.0;
        for (int64_t i = tid; i < n; i += kPrepThreads) {
            double s = fabs(a.ds[i]);
            if (i > 0) s = __dadd_rn(s, fabs(a.es[i - 1]));
            if (i < n - 1) s = __dadd_rn(s, fabs(a.es[i]));
            tl = fmax(tl, s);
        }
        tl = warp_max(tl);
        __syncthreads();
        if ((tid & 31) == 0) red[tid >> 5] = tl;
        __syncthreads();
        if (tid < 32) {
            double v = red[tid];
            v = warp_max(v);
            if (tid == 0) red[0] = v;
        }
        __syncthreads();
        tnorm = red[0];
    }
    if (tid == 0) {
        a.out->tnorm = tnorm;
        a.out->bad = 0;
        a.out->scale_exp = k;
    }
    auto wv = [&](int64_t j) -> double { return ldexp(a.w[j], k); };   // exact; k = 0: w itself
    const double thr = __dmul_rn(1e-3, tnorm);

    // ---- R2: boundary flags + compaction (chunked block scan)
    for (int64_t base = 0; base < n; base += kPrepThreads) {
        int64_t j = base + tid;
        int flag = 0;
        if (j < n) flag = (j == 0) || !(__dsub_rn(wv(j), wv(j - 1)) <= thr);
        // inclusive warp scan
        int v = flag;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, v, o);
            if ((tid & 31) >= o) v += t;
        }
        if ((tid & 31) == 31) sscan[tid >> 5] = v;
        __syncthreads();
        if (tid < 32) {
            int s = sscan[tid];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int t = __shfl_up_sync(0xffffffffu, s, o);
                if (tid >= o) s += t;
            }
            sscan[tid] = s;  // inclusive over warps
        }
        __syncthreads();
        int incl = v + ((tid >> 5) > 0 ? sscan[(tid >> 5) - 1] : 0) + s_carry;
        if (j < n) {
            int cid = incl - 1;             // cluster id of j
            if (flag) a.cstart[cid] = (int)j;
            a.cid[j] = cid;
        }
        __syncthreads();
        if (tid == kPrepThreads - 1) s_carry = incl;
        __syncthreads();
    }
    const int nclus = s_carry;
    if (tid == 0) {
        a.cstart[nclus] = (int)n;
        a.out->nclus = nclus;
    }
    __syncthreads();

    // ---- jc and R3 ladder (one thread per cluster, sequential inside the cluster)
    int maxm = 0, nclustered = 0;
    for (int c = tid; c < nclus; c += kPrepThreads) {
        int j1 = a.cstart[c], j2 = a.cstart[c + 1];
        maxm = max(maxm, j2 - j1);
        nclustered += (j2 - j1) - 1;
        double prev = wv(j1);
        a.wt[j1] = prev;
        a.jc[j1] = 0;
        for (int j = j1 + 1; j < j2; j++) {
            double wj = wv(j);
            double cand = __dadd_rn(prev, __dmul_rn(10.0 * kEps, fabs(wj)));
            prev = fmax(wj, cand);
            a.wt[j] = prev;
            a.jc[j] = j - j1;
        }
    }
    // max / sum reductions of the cluster statistics
    for (int o = 16; o > 0; o >>= 1) {
        maxm = max(maxm, __shfl_xor_sync(0xffffffffu, maxm, o));
        nclustered += __shfl_xor_sync(0xffffffffu, nclustered, o);
    }
    if ((tid & 31) == 0) { atomicMax(&a.out->max_cluster, maxm); atomicAdd(&a.out->n_clustered, nclustered); }

    // ---- slot permutation of the batched LU (tinv_internal.h PrepArgs): stable compaction
    // of the vectors it iterates (class c) to the front, the first-solve vectors behind them
    // from a warp boundary, so that every warp holds one class
    __syncthreads();   // jc, cstart complete
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += kPrepThreads) {
        const int64_t j = base + tid;
        int cflag = 0;
        if (j < n && a.jc[j] == 0) {
            const int c = a.cid[j];
            const int m = a.cstart[c + 1] - a.cstart[c];
            cflag = !(m >= 2 && m <= a.handover);
        }
        int v = cflag;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if ((tid & 31) >= o) v += t;
        }
        if ((tid & 31) == 31) sscan[tid >> 5] = v;
        __syncthreads();
        if (tid < 32) {
            int s = sscan[tid];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, s, o);
                if (tid >= o) s += t;
            }
            sscan[tid] = s;
        }
        __syncthreads();
        const int incl = v + ((tid >> 5) > 0 ? sscan[(tid >> 5) - 1] : 0) + s_carry;
        const int rc = incl - cflag;   // class-c vectors before j
        // class c: its rank; first-solve: -(1 + its rank among them), resolved below
        if (j < n) a.slot[j] = cflag ? rc : -(1 + (int)(j - rc));
        __syncthreads();
        if (tid == kPrepThreads - 1) s_carry = incl;
        __syncthreads();
    }
    const int nc = s_carry;
    const int ncp = (nc + 31) & ~31;
    for (int64_t s = tid; s < a.nslot_cap; s += kPrepThreads) a.perm[s] = -1;
    __syncthreads();
    for (int64_t j = tid; j < n; j += kPrepThreads) {
        int s = a.slot[j];
        if (s < 0) s = ncp + (-s - 1);
        a.slot[j] = s;
        a.perm[s] = (int)j;
    }
    if (tid == 0) a.out->nc_pad = ncp;
}

void launch_prep(const PrepArgs& a, cudaStream_t s) {
    prep_kernel<<<1, kPrepThreads, 0, s>>>(a);
}

}  // namespace tinv
