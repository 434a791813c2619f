// Floor of the back-sweep chain x_i = t_i - b_i x_{i+1} - c_i x_{i+2} on one thread (cycles/row):
//  A  x = fma(b, x, s) with b, s in registers        (one dependent DFMA per row)
//  B  the recurrence with b, c, t in registers        (outer + inner FMA per row)
//  C  the library form: 16-row batches loaded from shared memory, then the chain
//  D  as C with 32-row batches
//  E  as C, the next batch's loads issued between the chain's FMAs (manual 2-batch unroll)
//  F  as C with t scaled by 1e-310 (every x subnormal)
//  H  as C, the first 4 rows of the next batch loaded during the current one; I the same with 8-row batches
//  G  as C with t scaled by 1e-300 and |b|, |c| ~ 1e-3 (x decays through the subnormal range)
#include <cstdio>
#include <vector>
#include <random>
constexpr int R = 16;
__device__ __forceinline__ void batch16(const double2* BC, const double* tf, double* xo, int u0, double& x1, double& x2) {
    double b[16], c[16], t[16], xv[16];
#pragma unroll
    for (int u = 0; u < 16; u++) { const double2 v = BC[u0 + u]; b[u] = v.x; c[u] = v.y; t[u] = tf[u0 + u]; }
#pragma unroll
    for (int u = 15; u >= 0; u--) { xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
    for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(xo + u0 + u) = make_double2(xv[u], xv[u + 1]);
}
__global__ void probe(const double* bcg, const double* tg, int n, long long* cyc, double* sink) {
    extern __shared__ __align__(16) unsigned char raw[];
    double* tf = reinterpret_cast<double*>(raw);
    double* xo = tf + n + 2;
    double2* BC = reinterpret_cast<double2*>(xo + n + 2);
    for (int i = threadIdx.x; i < n; i += blockDim.x) { tf[i] = tg[i]; BC[i] = make_double2(bcg[2 * i], bcg[2 * i + 1]); }
    __syncthreads();
    if (threadIdx.x) return;
    double acc = 0;
    {   // A
        double b[R], s[R];
        for (int u = 0; u < R; u++) { b[u] = -BC[u].x; s[u] = tf[u]; }
        double x = 1.0;
        long long t0 = clock64();
        for (int it = 0; it < n / R; it++) {
#pragma unroll
            for (int u = 0; u < R; u++) x = fma(b[u], x, s[u]);
        }
        cyc[0] = clock64() - t0;
        acc += x;
    }
    {   // B
        double b[R], c[R], t[R];
        for (int u = 0; u < R; u++) { b[u] = BC[u].x; c[u] = BC[u].y; t[u] = tf[u]; }
        double x1 = 0.0, x2 = 0.0;
        long long t0 = clock64();
        for (int it = 0; it < n / R; it++) {
#pragma unroll
            for (int u = R - 1; u >= 0; u--) { const double xv = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv; }
        }
        cyc[1] = clock64() - t0;
        acc += x1;
    }
    {   // C
        double x1 = 0.0, x2 = 0.0;
        long long t0 = clock64();
        for (int u0 = (n & ~15) - 16; u0 >= 0; u0 -= 16) batch16(BC, tf, xo, u0, x1, x2);
        cyc[2] = clock64() - t0;
        acc += x1;
    }
    {   // D: 32-row batches
        double x1 = 0.0, x2 = 0.0;
        long long t0 = clock64();
        for (int u0 = (n & ~31) - 32; u0 >= 0; u0 -= 32) {
            double b[32], c[32], t[32], xv[32];
#pragma unroll
            for (int u = 0; u < 32; u++) { const double2 v = BC[u0 + u]; b[u] = v.x; c[u] = v.y; t[u] = tf[u0 + u]; }
#pragma unroll
            for (int u = 31; u >= 0; u--) { xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
            for (int u = 0; u < 32; u += 2) *reinterpret_cast<double2*>(xo + u0 + u) = make_double2(xv[u], xv[u + 1]);
        }
        cyc[3] = clock64() - t0;
        acc += x1;
    }
    {   // E: loads of batch k+1 interleaved with the chain of batch k (two register sets)
        double x1 = 0.0, x2 = 0.0;
        long long t0 = clock64();
        const int top = (n & ~31);
        double b0[16], c0[16], t0v[16], b1[16], c1[16], t1v[16], xv[16];
#pragma unroll
        for (int u = 0; u < 16; u++) { const double2 v = BC[top - 16 + u]; b0[u] = v.x; c0[u] = v.y; t0v[u] = tf[top - 16 + u]; }
        for (int u0 = top - 16; u0 >= 16; u0 -= 32) {
#pragma unroll
            for (int u = 15; u >= 0; u--) {
                const double2 v = BC[u0 - 16 + u]; b1[u] = v.x; c1[u] = v.y; t1v[u] = tf[u0 - 16 + u];
                xv[u] = fma(-b0[u], x1, fma(-c0[u], x2, t0v[u])); x2 = x1; x1 = xv[u];
            }
#pragma unroll
            for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(xo + u0 + u) = make_double2(xv[u], xv[u + 1]);
            const int un = u0 - 32 >= 0 ? u0 - 32 : 0;
#pragma unroll
            for (int u = 15; u >= 0; u--) {
                const double2 v = BC[un + u]; b0[u] = v.x; c0[u] = v.y; t0v[u] = tf[un + u];
                xv[u] = fma(-b1[u], x1, fma(-c1[u], x2, t1v[u])); x2 = x1; x1 = xv[u];
            }
#pragma unroll
            for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(xo + u0 - 16 + u) = make_double2(xv[u], xv[u + 1]);
        }
        cyc[4] = clock64() - t0;
        acc += x1;
    }
    {   // H: as C, the operands of the first 4 rows of the next batch loaded during this one
        double x1 = 0.0, x2 = 0.0;
        long long t0 = clock64();
        const int top = (n & ~15);
        double hb[4], hc[4], ht[4];
#pragma unroll
        for (int u = 0; u < 4; u++) { const double2 v = BC[top - 4 + u]; hb[u] = v.x; hc[u] = v.y; ht[u] = tf[top - 4 + u]; }
        for (int u0 = top - 16; u0 >= 0; u0 -= 16) {
            double b[16], c[16], t[16], xv[16];
#pragma unroll
            for (int u = 12; u < 16; u++) { b[u] = hb[u - 12]; c[u] = hc[u - 12]; t[u] = ht[u - 12]; }
#pragma unroll
            for (int u = 0; u < 12; u++) { const double2 v = BC[u0 + u]; b[u] = v.x; c[u] = v.y; t[u] = tf[u0 + u]; }
            const int un = u0 >= 16 ? u0 - 16 : 0;
#pragma unroll
            for (int u = 0; u < 4; u++) { const double2 v = BC[un + 12 + u]; hb[u] = v.x; hc[u] = v.y; ht[u] = tf[un + 12 + u]; }
#pragma unroll
            for (int u = 15; u >= 0; u--) { xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
            for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(xo + u0 + u) = make_double2(xv[u], xv[u + 1]);
        }
        cyc[7] = clock64() - t0;
        acc += x1;
    }
    {   // I: 8-row batches with the same 4-row head
        double x1 = 0.0, x2 = 0.0;
        long long t0 = clock64();
        const int top = (n & ~15);
        double hb[4], hc[4], ht[4];
#pragma unroll
        for (int u = 0; u < 4; u++) { const double2 v = BC[top - 4 + u]; hb[u] = v.x; hc[u] = v.y; ht[u] = tf[top - 4 + u]; }
        for (int u0 = top - 8; u0 >= 0; u0 -= 8) {
            double b[8], c[8], t[8], xv[8];
#pragma unroll
            for (int u = 4; u < 8; u++) { b[u] = hb[u - 4]; c[u] = hc[u - 4]; t[u] = ht[u - 4]; }
#pragma unroll
            for (int u = 0; u < 4; u++) { const double2 v = BC[u0 + u]; b[u] = v.x; c[u] = v.y; t[u] = tf[u0 + u]; }
            const int un = u0 >= 8 ? u0 - 8 : 0;
#pragma unroll
            for (int u = 0; u < 4; u++) { const double2 v = BC[un + 4 + u]; hb[u] = v.x; hc[u] = v.y; ht[u] = tf[un + 4 + u]; }
#pragma unroll
            for (int u = 7; u >= 0; u--) { xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
            for (int u = 0; u < 8; u += 2) *reinterpret_cast<double2*>(xo + u0 + u) = make_double2(xv[u], xv[u + 1]);
        }
        cyc[8] = clock64() - t0;
        acc += x1;
    }
    {   // F, G: subnormal operands
        for (int i = 0; i < n; i++) tf[i] = tg[i] * 1e-310;
        double x1 = 0.0, x2 = 0.0;
        long long t0 = clock64();
        for (int u0 = (n & ~15) - 16; u0 >= 0; u0 -= 16) batch16(BC, tf, xo, u0, x1, x2);
        cyc[5] = clock64() - t0;
        acc += x1;
        for (int i = 0; i < n; i++) { tf[i] = (i == n - 1) ? 1e-300 : 0.0; BC[i] = make_double2(BC[i].x * 2e-3, BC[i].y * 2e-3); }
        x1 = 0.0; x2 = 0.0;
        t0 = clock64();
        for (int u0 = (n & ~15) - 16; u0 >= 0; u0 -= 16) batch16(BC, tf, xo, u0, x1, x2);
        cyc[6] = clock64() - t0;
        acc += x1;
    }
    *sink = acc;
}
int main() {
    const int n = 4096;
    std::mt19937_64 g(1);
    std::uniform_real_distribution<double> U(-1, 1);
    std::vector<double> bc(2 * n), t(n);
    for (auto& v : bc) v = 0.5 * U(g);
    for (auto& v : t) v = U(g);
    double *dbc, *dt, *sink; long long* dc;
    cudaMalloc(&dbc, 16 * n); cudaMalloc(&dt, 8 * n); cudaMalloc(&dc, 128); cudaMalloc(&sink, 8);
    cudaMemcpy(dbc, bc.data(), 16 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, t.data(), 8 * n, cudaMemcpyHostToDevice);
    size_t smem = (size_t)(n + 2) * 16 + 16 * n + 64;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; rep++) probe<<<1, 256, smem>>>(dbc, dt, n, dc, sink);
    long long h[16]; cudaMemcpy(h, dc, 128, cudaMemcpyDeviceToHost);
    const char* nm[9] = {"A 1 DFMA/row, regs", "B recurrence, regs", "C 16-batch smem", "D 32-batch smem", "E 2-set interleaved",
                         "F C, subnormal x", "G C, x decaying", "H C + 4-row head", "I 8-batch + 4-row head"};
    for (int v = 0; v < 9; v++) printf("%-22s %.2f cycles/row (%s)\n", nm[v], (double)h[v] / n, cudaGetErrorString(cudaGetLastError()));
}
