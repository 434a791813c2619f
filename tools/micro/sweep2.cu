// Microbenchmark: DFMA dependent latency by operand position, and the resident kernel's
// shared-memory back sweep (back_sweep_smem form) in isolation, cycles per row.
#include <cstdio>
#include <cstdint>
constexpr int N = 2000;
__device__ __noinline__ void sweep(const double* __restrict__ bc, double* tf, int64_t n) {
    const double2* BC = reinterpret_cast<const double2*>(bc);
    double x1 = 0.0, x2 = 0.0;
    const int64_t top = n & ~int64_t(7);
    double b[8], c[8], t[8];
#pragma unroll
    for (int u = 0; u < 8; u++) { const double2 v = BC[top - 8 + u]; b[u] = v.x; c[u] = v.y; t[u] = tf[top - 8 + u]; }
    for (int64_t u0 = top - 8; u0 >= 0; u0 -= 8) {
        double bn[8], cn[8], tn[8], xv[8];
        const int64_t nx = u0 >= 8 ? u0 - 8 : 0;
#pragma unroll
        for (int u = 0; u < 8; u++) { const double2 v = BC[nx + u]; bn[u] = v.x; cn[u] = v.y; tn[u] = tf[nx + u]; }
#pragma unroll
        for (int u = 7; u >= 0; u--) { xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
        for (int u = 0; u < 8; u += 2) *reinterpret_cast<double2*>(tf + u0 + u) = make_double2(xv[u], xv[u + 1]);
#pragma unroll
        for (int u = 0; u < 8; u++) { b[u] = bn[u]; c[u] = cn[u]; t[u] = tn[u]; }
    }
}
// variant: 32-bit indices, 16-row batches
__device__ __noinline__ void sweep16(const double* __restrict__ bc, double* tf, int n) {
    const double2* BC = reinterpret_cast<const double2*>(bc);
    double x1 = 0.0, x2 = 0.0;
    const int top = n & ~15;
    double b[16], c[16], t[16];
#pragma unroll
    for (int u = 0; u < 16; u++) { const double2 v = BC[top - 16 + u]; b[u] = v.x; c[u] = v.y; t[u] = tf[top - 16 + u]; }
    for (int u0 = top - 16; u0 >= 0; u0 -= 16) {
        double bn[16], cn[16], tn[16], xv[16];
        const int nx = u0 >= 16 ? u0 - 16 : 0;
#pragma unroll
        for (int u = 0; u < 16; u++) { const double2 v = BC[nx + u]; bn[u] = v.x; cn[u] = v.y; tn[u] = tf[nx + u]; }
#pragma unroll
        for (int u = 15; u >= 0; u--) { xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
        for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(tf + u0 + u) = make_double2(xv[u], xv[u + 1]);
#pragma unroll
        for (int u = 0; u < 16; u++) { b[u] = bn[u]; c[u] = cn[u]; t[u] = tn[u]; }
    }
}
__global__ void k(const double* g, long long* cyc, double* sink) {
    __shared__ __align__(16) double bc[2 * N];
    __shared__ __align__(16) double tf[N + 2];
    for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) bc[i] = 0.1 + 1e-3 * (i % 7);
    for (int i = threadIdx.x; i < N; i += blockDim.x) tf[i] = 1e-3 * (i % 17);
    __syncthreads();
    if (threadIdx.x) return;
    double acc = 0;
    {   // multiplicand chain
        double x = g[0], a = 0.999, b = 1e-6;
        long long t0 = clock64();
#pragma unroll 16
        for (int i = 0; i < 4096; i++) x = fma(x, a, b);
        cyc[0] = (clock64() - t0) * 1000 / 4096; acc += x;
    }
    {   // addend chain
        double x = g[0], a = 0.999, b = 1e-6;
        long long t0 = clock64();
#pragma unroll 16
        for (int i = 0; i < 4096; i++) x = fma(a, b, x);
        cyc[1] = (clock64() - t0) * 1000 / 4096; acc += x;
    }
    {   // multiplicand chain through subnormal values
        double x = 1e-310 + g[0], a = 0.999, b = 0.0;
        long long t0 = clock64();
#pragma unroll 16
        for (int i = 0; i < 4096; i++) x = fma(x, a, b);
        cyc[5] = (clock64() - t0) * 1000 / 4096; acc += x;
    }
    {   // DADD chain
        double x = g[0], b = 1e-6;
        long long t0 = clock64();
#pragma unroll 16
        for (int i = 0; i < 4096; i++) x = x + b;
        cyc[2] = (clock64() - t0) * 1000 / 4096; acc += x;
    }
    {
        long long t0 = clock64();
        sweep(bc, tf, N);
        cyc[3] = (clock64() - t0) * 1000 / N; acc += tf[3];
    }
    {
        long long t0 = clock64();
        sweep16(bc, tf, N);
        cyc[4] = (clock64() - t0) * 1000 / N; acc += tf[5];
    }
    sink[0] = acc;
}
#include <cooperative_groups.h>
// sweep by thread 0 of CTA 0 while every other thread of the 2-CTA cluster waits in
// cluster.sync (mode 1) or in __syncthreads (mode 2) or exits (mode 0)
__global__ void __cluster_dims__(2, 1, 1) kc(int mode, long long* cyc, double* sink) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ __align__(16) double bc[2 * N];
    __shared__ __align__(16) double tf[N + 2];
    for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) bc[i] = 0.1 + 1e-3 * (i % 7);
    for (int i = threadIdx.x; i < N; i += blockDim.x) tf[i] = 1e-3 * (i % 17);
    cl.sync();
    if (mode == 3 && cl.block_rank() == 1) {   // t rows written remotely by the other CTA
        double* t0p = cl.map_shared_rank(tf, 0);
        for (int i = threadIdx.x; i < N; i += blockDim.x) t0p[i] = 2e-3 * (i % 13);
    }
    if (mode == 3) cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
        long long t0 = clock64();
        sweep(bc, tf, N);
        cyc[mode] = (clock64() - t0) * 1000 / N;
        sink[mode] = tf[3];
    }
    if (mode == 1) cl.sync();
    else if (mode == 2) __syncthreads();
}
// plain (non-cluster) CTA with `blockDim` threads: thread 0 sweeps, the rest wait
__global__ void kp(int slot, long long* cyc, double* sink) {
    __shared__ __align__(16) double bc[2 * N];
    __shared__ __align__(16) double tf[N + 2];
    for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) bc[i] = 0.1 + 1e-3 * (i % 7);
    for (int i = threadIdx.x; i < N; i += blockDim.x) tf[i] = 1e-3 * (i % 17);
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        sweep(bc, tf, N);
        cyc[slot] = (clock64() - t0) * 1000 / N;
        sink[slot] = tf[3];
    }
    __syncthreads();
}
int main() {
    double *g, *s; long long* c;
    cudaMalloc(&g, 64); cudaMalloc(&s, 64); cudaMalloc(&c, 128);
    cudaMemset(g, 0, 64);
    k<<<1, 128>>>(g, c, s);
    k<<<1, 128>>>(g, c, s);
    long long h[6];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("DFMA mul-chain %.2f  add-chain %.2f  DADD %.2f  sweep8 %.2f  sweep16 %.2f cycles (%s)\n",
           h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0, cudaGetErrorString(cudaGetLastError()));
    for (int rep = 0; rep < 2; rep++)
        for (int mode = 0; mode < 4; mode++) kc<<<2, 256>>>(mode, c, s);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    for (int rep = 0; rep < 2; rep++) { kp<<<1, 32>>>(8, c, s); kp<<<1, 128>>>(9, c, s); kp<<<1, 256>>>(10, c, s); kp<<<1, 1024>>>(11, c, s); }
    long long hp[12];
    cudaMemcpy(hp, c, sizeof(hp), cudaMemcpyDeviceToHost);
    printf("plain CTA, thread 0 sweeps: 32 thr %.2f  128 thr %.2f  256 thr %.2f  1024 thr %.2f\n", hp[8] / 1000.0, hp[9] / 1000.0, hp[10] / 1000.0, hp[11] / 1000.0);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("subnormal DFMA chain %.2f\n", h[5] / 1000.0);
    printf("in a 2-CTA cluster, 256 threads: others exit %.2f  wait in cluster.sync %.2f  wait in __syncthreads %.2f  t written over DSMEM %.2f (%s)\n",
           h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, cudaGetErrorString(cudaGetLastError()));
}
