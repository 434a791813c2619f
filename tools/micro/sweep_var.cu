// Back-sweep loop variants (runtime n, library compile flags), cycles per row.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
// V0: library form (int64, 8-row batches, loads of the next batch in the loop body)
__device__ __forceinline__ void v0(const double* __restrict__ bc, double* tf, int64_t n) {
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
// V1: int32 indices, t loaded as pairs
__device__ __forceinline__ void v1(const double* __restrict__ bc, double* tf, int n) {
    const double2* BC = reinterpret_cast<const double2*>(bc);
    const double2* T2 = reinterpret_cast<const double2*>(tf);
    double x1 = 0.0, x2 = 0.0;
    const int top = n & ~7;
    double b[8], c[8], t[8];
#pragma unroll
    for (int u = 0; u < 8; u++) { const double2 v = BC[top - 8 + u]; b[u] = v.x; c[u] = v.y; }
#pragma unroll
    for (int u = 0; u < 8; u += 2) { const double2 v = T2[(top - 8 + u) >> 1]; t[u] = v.x; t[u + 1] = v.y; }
    for (int u0 = top - 8; u0 >= 0; u0 -= 8) {
        double bn[8], cn[8], tn[8], xv[8];
        const int nx = u0 >= 8 ? u0 - 8 : 0;
#pragma unroll
        for (int u = 0; u < 8; u++) { const double2 v = BC[nx + u]; bn[u] = v.x; cn[u] = v.y; }
#pragma unroll
        for (int u = 0; u < 8; u += 2) { const double2 v = T2[(nx + u) >> 1]; tn[u] = v.x; tn[u + 1] = v.y; }
#pragma unroll
        for (int u = 7; u >= 0; u--) { xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
        for (int u = 0; u < 8; u += 2) *reinterpret_cast<double2*>(tf + u0 + u) = make_double2(xv[u], xv[u + 1]);
#pragma unroll
        for (int u = 0; u < 8; u++) { b[u] = bn[u]; c[u] = cn[u]; t[u] = tn[u]; }
    }
}
// V2: precomputed inner term: the chain is one FMA per row; the inner fma(-c, x2, t) needs x2
// (two rows back) -- same as V1 but written to make the two FMAs of a row independent chains
__device__ __forceinline__ void v2(const double* __restrict__ bc, double* tf, int n) {
    const double2* BC = reinterpret_cast<const double2*>(bc);
    double x1 = 0.0, x2 = 0.0;
    const int top = n & ~15;
    for (int u0 = top - 16; u0 >= 0; u0 -= 16) {
        double b[16], c[16], t[16], xv[16];
#pragma unroll
        for (int u = 0; u < 16; u++) { const double2 v = BC[u0 + u]; b[u] = v.x; c[u] = v.y; t[u] = tf[u0 + u]; }
#pragma unroll
        for (int u = 15; u >= 0; u--) { xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
        for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(tf + u0 + u) = make_double2(xv[u], xv[u + 1]);
    }
}
// V3: records [b, c, t, -] interleaved (32 B per row): two LDS.128 per row pair
__device__ __forceinline__ void v3(const double* __restrict__ rec, double* xo, int n) {
    const double4* R = reinterpret_cast<const double4*>(rec);
    double x1 = 0.0, x2 = 0.0;
    const int top = n & ~7;
    double4 r[8];
#pragma unroll
    for (int u = 0; u < 8; u++) r[u] = R[top - 8 + u];
    for (int u0 = top - 8; u0 >= 0; u0 -= 8) {
        double4 rn[8];
        double xv[8];
        const int nx = u0 >= 8 ? u0 - 8 : 0;
#pragma unroll
        for (int u = 0; u < 8; u++) rn[u] = R[nx + u];
#pragma unroll
        for (int u = 7; u >= 0; u--) { xv[u] = fma(-r[u].x, x1, fma(-r[u].y, x2, r[u].z)); x2 = x1; x1 = xv[u]; }
#pragma unroll
        for (int u = 0; u < 8; u += 2) *reinterpret_cast<double2*>(xo + u0 + u) = make_double2(xv[u], xv[u + 1]);
#pragma unroll
        for (int u = 0; u < 8; u++) r[u] = rn[u];
    }
}
// V4: 16-row batches, next batch's loads issued before the current chain (double buffer)
__device__ __forceinline__ void v4(const double* __restrict__ bc, double* tf, int n) {
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
// V5: 8-row batches, no software pipelining, int32
__device__ __forceinline__ void v5(const double* __restrict__ bc, double* tf, int n) {
    const double2* BC = reinterpret_cast<const double2*>(bc);
    double x1 = 0.0, x2 = 0.0;
    const int top = n & ~7;
    for (int u0 = top - 8; u0 >= 0; u0 -= 8) {
        double b[8], c[8], t[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) { const double2 v = BC[u0 + u]; b[u] = v.x; c[u] = v.y; t[u] = tf[u0 + u]; }
#pragma unroll
        for (int u = 7; u >= 0; u--) { xv[u] = fma(-b[u], x1, fma(-c[u], x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
        for (int u = 0; u < 8; u += 2) *reinterpret_cast<double2*>(tf + u0 + u) = make_double2(xv[u], xv[u + 1]);
    }
}
// V6: 16-row batches, inner products of the next batch precomputed: s_i = t_i - c_i x_{i+2}
// needs x_{i+2}; within a batch, the first two rows use the carried x; the chain stays 1 FMA
// per row.  (Same as V2 but the t/c loads via one LDS.128 of an interleaved [t, c] array.)
__device__ __forceinline__ void v6(const double* __restrict__ bc, double* tf, int n) {
    const double2* BC = reinterpret_cast<const double2*>(bc);
    double x1 = 0.0, x2 = 0.0;
    const int top = n & ~15;
    for (int u0 = top - 16; u0 >= 0; u0 -= 16) {
        double2 v[16];
        double t[16], xv[16];
#pragma unroll
        for (int u = 0; u < 16; u++) v[u] = BC[u0 + u];
#pragma unroll
        for (int u = 0; u < 16; u += 2) { const double2 tt = *reinterpret_cast<const double2*>(tf + u0 + u); t[u] = tt.x; t[u + 1] = tt.y; }
#pragma unroll
        for (int u = 15; u >= 0; u--) { xv[u] = fma(-v[u].x, x1, fma(-v[u].y, x2, t[u])); x2 = x1; x1 = xv[u]; }
#pragma unroll
        for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(tf + u0 + u) = make_double2(xv[u], xv[u + 1]);
    }
}
__global__ void probe(int var, const double* bcg, const double* tg, int n, long long* cyc) {
    extern __shared__ __align__(16) unsigned char raw[];
    double* tf = reinterpret_cast<double*>(raw);
    double* bc = tf + ((n + 2 + 1) & ~1);
    double* rec = bc + 2 * n;
    for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) bc[i] = bcg[i];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        tf[i] = tg[i];
        rec[4 * i] = bcg[2 * i]; rec[4 * i + 1] = bcg[2 * i + 1]; rec[4 * i + 2] = tg[i]; rec[4 * i + 3] = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        if (var == 0) v0(bc, tf, n);
        else if (var == 1) v1(bc, tf, n);
        else if (var == 2) v2(bc, tf, n);
        else if (var == 3) v3(rec, tf, n);
        else if (var == 4) v4(bc, tf, n);
        else if (var == 5) v5(bc, tf, n);
        else v6(bc, tf, n);
        cyc[var] = clock64() - t0;
    }
}
int main() {
    const int n = 2000;
    std::mt19937_64 g(1);
    std::uniform_real_distribution<double> U(-1, 1);
    std::vector<double> bc(2 * n), t(n);
    for (auto& v : bc) v = 0.5 * U(g);
    for (auto& v : t) v = U(g);
    double *dbc, *dt; long long* dc;
    cudaMalloc(&dbc, 16 * n); cudaMalloc(&dt, 8 * n); cudaMalloc(&dc, 64);
    cudaMemcpy(dbc, bc.data(), 16 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, t.data(), 8 * n, cudaMemcpyHostToDevice);
    size_t smem = (size_t)(n + 2) * 8 + 16 * n + 32 * n + 64;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int v = 0; v < 7; v++) {
        probe<<<1, 256, smem>>>(v, dbc, dt, n, dc);
        probe<<<1, 256, smem>>>(v, dbc, dt, n, dc);
        long long h[8]; cudaMemcpy(h, dc, 64, cudaMemcpyDeviceToHost);
        printf("variant %d: %.2f cycles/row (%s)\n", v, (double)h[v] / n, cudaGetErrorString(cudaGetLastError()));
    }
}
