// Microbenchmark: one-thread back-substitution chain x_i = t_i - b_i x_{i+1} - c_i x_{i+2}
// fed from shared memory, in several loop forms (cycles per row).  Guides cwy.cu back_sweep.
#include <cstdio>
#include <cstdint>
constexpr int N = 1024;
__global__ void k(const double* __restrict__ g, double* __restrict__ xo, long long* cyc, double* sink) {
    __shared__ __align__(16) double F[N * 4];
    __shared__ __align__(16) double Tt[N];
    __shared__ __align__(16) double X[N];
    for (int i = threadIdx.x; i < N * 4; i += blockDim.x) F[i] = g[i];
    for (int i = threadIdx.x; i < N; i += blockDim.x) Tt[i] = g[N * 4 + i];
    __syncthreads();
    if (threadIdx.x) return;
    double acc = 0;
    // (0) DFMA dependent latency
    {
        double x = g[0], a = 0.999, b = 1e-6;
        long long t0 = clock64();
        for (int i = 0; i < 4096; i++) { x = fma(a, x, b); }
        long long t1 = clock64();
        cyc[0] = (t1 - t0) * 1000 / 4096;
        acc += x;
    }
    // (1) per-row: smem loads, chain, STG per row (global)
    {
        double x1 = 0, x2 = 0;
        long long t0 = clock64();
#pragma unroll 8
        for (int u = N - 1; u >= 0; u--) {
            const double2 bc = *reinterpret_cast<const double2*>(F + u * 4 + 2);
            const double t = fma(-bc.y, x2, Tt[u]);
            const double xi = fma(-bc.x, x1, t);
            __stcg(xo + u, xi);
            x2 = x1; x1 = xi;
        }
        long long t1 = clock64();
        cyc[1] = (t1 - t0) * 1000 / N;
        acc += x1;
    }
    // (2) per-row, stores to shared
    {
        double x1 = 0, x2 = 0;
        long long t0 = clock64();
#pragma unroll 8
        for (int u = N - 1; u >= 0; u--) {
            const double2 bc = *reinterpret_cast<const double2*>(F + u * 4 + 2);
            const double t = fma(-bc.y, x2, Tt[u]);
            const double xi = fma(-bc.x, x1, t);
            X[u] = xi;
            x2 = x1; x1 = xi;
        }
        long long t1 = clock64();
        cyc[2] = (t1 - t0) * 1000 / N;
        acc += x1 + X[5];
    }
    // (3) batch 8: loads first, chain, stores to shared
    {
        double x1 = 0, x2 = 0;
        long long t0 = clock64();
        for (int u0 = N - 8; u0 >= 0; u0 -= 8) {
            double b[8], c[8], t[8], xv[8];
#pragma unroll
            for (int u = 7; u >= 0; u--) {
                const double2 bc = *reinterpret_cast<const double2*>(F + (u0 + u) * 4 + 2);
                b[u] = bc.x; c[u] = bc.y; t[u] = Tt[u0 + u];
            }
#pragma unroll
            for (int u = 7; u >= 0; u--) {
                const double tt = fma(-c[u], x2, t[u]);
                xv[u] = fma(-b[u], x1, tt);
                x2 = x1; x1 = xv[u];
            }
#pragma unroll
            for (int u = 0; u < 8; u++) X[u0 + u] = xv[u];
        }
        long long t1 = clock64();
        cyc[3] = (t1 - t0) * 1000 / N;
        acc += x1 + X[7];
    }
    // (4) batch 8 software pipelined (next batch loads before chain), stores to shared
    {
        double x1 = 0, x2 = 0;
        double b[8], c[8], t[8];
        long long t0 = clock64();
#pragma unroll
        for (int u = 7; u >= 0; u--) {
            const double2 bc = *reinterpret_cast<const double2*>(F + (N - 8 + u) * 4 + 2);
            b[u] = bc.x; c[u] = bc.y; t[u] = Tt[N - 8 + u];
        }
        for (int u0 = N - 8; u0 >= 0; u0 -= 8) {
            double bn[8], cn[8], tn[8], xv[8];
            const int nx = u0 >= 8 ? u0 - 8 : 0;
#pragma unroll
            for (int u = 7; u >= 0; u--) {
                const double2 bc = *reinterpret_cast<const double2*>(F + (nx + u) * 4 + 2);
                bn[u] = bc.x; cn[u] = bc.y; tn[u] = Tt[nx + u];
            }
#pragma unroll
            for (int u = 7; u >= 0; u--) {
                const double tt = fma(-c[u], x2, t[u]);
                xv[u] = fma(-b[u], x1, tt);
                x2 = x1; x1 = xv[u];
            }
#pragma unroll
            for (int u = 0; u < 8; u++) { X[u0 + u] = xv[u]; b[u] = bn[u]; c[u] = cn[u]; t[u] = tn[u]; }
        }
        long long t1 = clock64();
        cyc[4] = (t1 - t0) * 1000 / N;
        acc += x1 + X[9];
    }
    // (5) like (4) but the x pairs go to global with STG.128 after each batch
    {
        double x1 = 0, x2 = 0;
        double b[8], c[8], t[8];
        long long t0 = clock64();
#pragma unroll
        for (int u = 7; u >= 0; u--) {
            const double2 bc = *reinterpret_cast<const double2*>(F + (N - 8 + u) * 4 + 2);
            b[u] = bc.x; c[u] = bc.y; t[u] = Tt[N - 8 + u];
        }
        for (int u0 = N - 8; u0 >= 0; u0 -= 8) {
            double bn[8], cn[8], tn[8], xv[8];
            const int nx = u0 >= 8 ? u0 - 8 : 0;
#pragma unroll
            for (int u = 7; u >= 0; u--) {
                const double2 bc = *reinterpret_cast<const double2*>(F + (nx + u) * 4 + 2);
                bn[u] = bc.x; cn[u] = bc.y; tn[u] = Tt[nx + u];
            }
#pragma unroll
            for (int u = 7; u >= 0; u--) {
                const double tt = fma(-c[u], x2, t[u]);
                xv[u] = fma(-b[u], x1, tt);
                x2 = x1; x1 = xv[u];
            }
#pragma unroll
            for (int u = 0; u < 8; u += 2) __stcg(reinterpret_cast<double2*>(xo + u0 + u), make_double2(xv[u], xv[u + 1]));
#pragma unroll
            for (int u = 0; u < 8; u++) { b[u] = bn[u]; c[u] = cn[u]; t[u] = tn[u]; }
        }
        long long t1 = clock64();
        cyc[5] = (t1 - t0) * 1000 / N;
        acc += x1;
    }
    // (6) 16-row body, two register halves (no copies), STG.128
    {
        double x1 = 0, x2 = 0;
        double b0[8], c0[8], t0_[8], b1[8], c1[8], t1_[8];
        auto ld8 = [&](int base, double* b, double* c, double* t) {
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const double2 bc = *reinterpret_cast<const double2*>(F + (base + u) * 4 + 2);
                b[u] = bc.x; c[u] = bc.y;
            }
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
                const double2 tt = *reinterpret_cast<const double2*>(Tt + base + u);
                t[u] = tt.x; t[u + 1] = tt.y;
            }
        };
        auto run8 = [&](int base, const double* b, const double* c, const double* t) {
            double xv[8];
#pragma unroll
            for (int u = 7; u >= 0; u--) {
                const double tt = fma(-c[u], x2, t[u]);
                xv[u] = fma(-b[u], x1, tt);
                x2 = x1; x1 = xv[u];
            }
#pragma unroll
            for (int u = 0; u < 8; u += 2) __stcg(reinterpret_cast<double2*>(xo + base + u), make_double2(xv[u], xv[u + 1]));
        };
        long long t0 = clock64();
        ld8(N - 8, b0, c0, t0_);
        for (int u0 = N - 8; u0 >= 0; u0 -= 16) {
            ld8(u0 >= 8 ? u0 - 8 : 0, b1, c1, t1_);
            run8(u0, b0, c0, t0_);
            ld8(u0 >= 16 ? u0 - 16 : 0, b0, c0, t0_);
            run8(u0 - 8, b1, c1, t1_);
        }
        long long t1 = clock64();
        cyc[6] = (t1 - t0) * 1000 / N;
        acc += x1;
    }
    sink[0] = acc;
}
int main() {
    double *g, *xo, *sink; long long* c;
    cudaMalloc(&g, sizeof(double) * N * 5); cudaMalloc(&xo, sizeof(double) * N); cudaMalloc(&sink, 64);
    cudaMalloc(&c, 64 * 8);
    double* h = new double[N * 5];
    for (int i = 0; i < N * 5; i++) h[i] = 0.3 + 1e-3 * (i % 7);
    cudaMemcpy(g, h, sizeof(double) * N * 5, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
    k<<<1, 128>>>(g, xo, c, sink);
    k<<<1, 128>>>(g, xo, c, sink);
    long long hc[8];
    cudaMemcpy(hc, c, 8 * 8, cudaMemcpyDeviceToHost);
    const char* nm[] = {"DFMA latency", "per-row STG", "per-row STS", "batch8 STS", "batch8 pipelined STS",
                        "batch8 pipelined STG.128", "16-row two-half STG.128"};
    for (int i = 0; i < 7; i++) printf("%-26s %.2f cycles/row\n", nm[i], hc[i] / 1000.0);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
