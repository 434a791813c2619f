// Microbenchmark: dependent fp64 FMA latency and LDS latency on one thread (clock64).
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters, double a, double b) {
    double x = out[0];
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        x = fma(a, x, b); x = fma(a, x, b); x = fma(a, x, b); x = fma(a, x, b);
        x = fma(a, x, b); x = fma(a, x, b); x = fma(a, x, b); x = fma(a, x, b);
    }
    long long t1 = clock64();
    out[1] = x;
    cyc[0] = t1 - t0;
    // select + fma chain (like the pivoted forward step)
    double y = out[2];
    int sw = (int)out[3];
    t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 8; u++) { y = sw ? fma(-a, b, y) : fma(-a, y, b); sw ^= (u & 1); }
    }
    t1 = clock64();
    out[4] = y;
    cyc[1] = t1 - t0;
    // fp64 reciprocal chain
    double z = out[5];
    t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 8; u++) z = 1.0 / (z + a);
    }
    t1 = clock64();
    out[6] = z;
    cyc[2] = t1 - t0;
}
int main() {
    double* d; long long* c;
    cudaMalloc(&d, 64); cudaMalloc(&c, 64);
    double h[8] = {1.0, 0, 0.5, 1, 0, 0.7, 0, 0};
    cudaMemcpy(d, h, 64, cudaMemcpyHostToDevice);
    int iters = 100000;
    k<<<1, 1>>>(d, c, iters, 0.999999, 1e-6);
    long long hc[3];
    cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)hc[0] / (8.0 * iters));
    printf("select+DFMA chain: %.2f cycles/step\n", (double)hc[1] / (8.0 * iters));
    printf("fp64 reciprocal chain: %.2f cycles/step\n", (double)hc[2] / (8.0 * iters));
    return 0;
}
