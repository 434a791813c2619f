// Microbenchmark: the resident kernel's in-place back sweep (TMA ring of factor records from
// global memory, t in shared memory) vs the same chain over plain shared-memory arrays.
#include <cstdio>
#include <cstdint>
#include "../../paper_1209_1910_b200/csrc/common.cuh"
using namespace tinv;
constexpr int CH = 256, kRing = 4;
__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
template <int VARIANT>
__global__ void k(const double* __restrict__ F, int64_t n, long long* cyc, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    double* tf = reinterpret_cast<double*>(sm);
    double* ring = tf + n + 2 + ((n + 2) & 1);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(ring + kRing * 4 * CH);
    for (int i = threadIdx.x; i < n; i += blockDim.x) tf[i] = 1e-3 * (i % 17);
    if (threadIdx.x == 0) { for (int i = 0; i < kRing; i++) mbar_init(mbar + i, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x) return;
    uint32_t mbph = 0;
    const int64_t C = (n + CH - 1) / CH;
    auto issue = [&](int64_t kk) {
        const int slot = (int)(kk % kRing);
        const int64_t lo = (C - 1 - kk) * CH, hi = min64(lo + CH, n);
        mbar_expect_tx(mbar + slot, (uint32_t)((hi - lo) * 32));
        bulk_g2s(ring + (int64_t)slot * 4 * CH, F + lo * 4, (uint32_t)((hi - lo) * 32), mbar + slot);
    };
    long long t0 = clock64();
    for (int64_t kk = 0; kk < C && kk < kRing; kk++) issue(kk);
    double x1 = 0.0, x2 = 0.0;
    for (int64_t kk = 0; kk < C; kk++) {
        const int slot = (int)(kk % kRing);
        mbar_wait(mbar + slot, (mbph >> slot) & 1u);
        mbph ^= 1u << slot;
        const double* Fs = ring + (int64_t)slot * 4 * CH;
        const int64_t lo = (C - 1 - kk) * CH, hi = min64(lo + CH, n);
        double* Ts = tf + lo;
        const int cnt = (int)(hi - lo);
        const int top = cnt & ~7;
        if (VARIANT == 0) {
            double b[8], c[8], t[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const double2 bc = *reinterpret_cast<const double2*>(Fs + (top - 8 + u) * 4 + 2);
                b[u] = bc.x; c[u] = bc.y; t[u] = Ts[top - 8 + u];
            }
            for (int u0 = top - 8; u0 >= 0; u0 -= 8) {
                double bn[8], cn[8], tn[8], xv[8];
                const int nx = u0 >= 8 ? u0 - 8 : 0;
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const double2 bc = *reinterpret_cast<const double2*>(Fs + (nx + u) * 4 + 2);
                    bn[u] = bc.x; cn[u] = bc.y; tn[u] = Ts[nx + u];
                }
#pragma unroll
                for (int u = 7; u >= 0; u--) {
                    xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u]));
                    x2 = x1; x1 = xv[u];
                }
#pragma unroll
                for (int u = 0; u < 8; u += 2) *reinterpret_cast<double2*>(Ts + u0 + u) = make_double2(xv[u], xv[u + 1]);
#pragma unroll
                for (int u = 0; u < 8; u++) { b[u] = bn[u]; c[u] = cn[u]; t[u] = tn[u]; }
            }
        } else {
            // variant 1: 16-row batches, loads of the next 16 before the chain
            double b[16], c[16], t[16];
            const int top16 = cnt & ~15;
#pragma unroll
            for (int u = 0; u < 16; u++) {
                const double2 bc = *reinterpret_cast<const double2*>(Fs + (top16 - 16 + u) * 4 + 2);
                b[u] = bc.x; c[u] = bc.y; t[u] = Ts[top16 - 16 + u];
            }
            for (int u0 = top16 - 16; u0 >= 0; u0 -= 16) {
                double bn[16], cn[16], tn[16], xv[16];
                const int nx = u0 >= 16 ? u0 - 16 : 0;
#pragma unroll
                for (int u = 0; u < 16; u++) {
                    const double2 bc = *reinterpret_cast<const double2*>(Fs + (nx + u) * 4 + 2);
                    bn[u] = bc.x; cn[u] = bc.y; tn[u] = Ts[nx + u];
                }
#pragma unroll
                for (int u = 15; u >= 0; u--) {
                    xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u]));
                    x2 = x1; x1 = xv[u];
                }
#pragma unroll
                for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(Ts + u0 + u) = make_double2(xv[u], xv[u + 1]);
#pragma unroll
                for (int u = 0; u < 16; u++) { b[u] = bn[u]; c[u] = cn[u]; t[u] = tn[u]; }
            }
        }
        if (kk + kRing < C) issue(kk + kRing);
    }
    long long t1 = clock64();
    cyc[0] = t1 - t0;
    out[0] = x1 + tf[3];
}
template <int V>
void run(const double* F, int64_t n, long long* c, double* o) {
    size_t smem = (n + 4) * 8 + kRing * 4 * CH * 8 + 64;
    cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<V><<<1, 128, smem>>>(F, n, c, o);
    k<V><<<1, 128, smem>>>(F, n, c, o);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("variant %d n=%lld: %.2f cycles/row (%s)\n", V, (long long)n, (double)h / n, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    const int64_t n = 4096;
    double *F, *o; long long* c;
    cudaMalloc(&F, n * 32 + 64); cudaMalloc(&o, 64); cudaMalloc(&c, 64);
    cudaMemset(F, 0, n * 32);
    run<0>(F, n, c, o);
    run<1>(F, n, c, o);
    return 0;
}
