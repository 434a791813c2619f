// Microbenchmark: the resident kernel's back sweep (tinv::res::back_sweep_smem, compiled from
// the library source) in a small kernel, with the kernel's shared-memory footprint optionally
// reserved, and data from a random tridiagonal factorisation-like distribution.
#include "../../paper_1209_1910_b200/csrc/cwy_resident.cu"
#include <cstdio>
#include <vector>
#include <random>
__global__ void probe(const double* bcg, const double* tg, int64_t n, long long* cyc) {
    extern __shared__ __align__(16) unsigned char raw[];
    double* tf = reinterpret_cast<double*>(raw);
    double* bc = tf + ((n + 2 + 1) & ~int64_t(1));
    for (int64_t i = threadIdx.x; i < 2 * n; i += blockDim.x) bc[i] = bcg[i];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) tf[i] = tg[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        tinv::res::back_sweep_smem(bc, tf, n);
        cyc[0] = clock64() - t0;
    }
}
int main() {
    const int64_t n = 2000;
    std::mt19937_64 g(1);
    std::uniform_real_distribution<double> U(-1, 1);
    std::vector<double> bc(2 * n), t(n);
    const bool konst = getenv("KONST") != nullptr;
    for (size_t i = 0; i < bc.size(); i++) bc[i] = konst ? 0.1 + 1e-3 * (i % 7) : 0.5 * U(g);
    for (size_t i = 0; i < t.size(); i++) t[i] = konst ? 1e-3 * (i % 17) : U(g);
    double *dbc, *dt; long long* dc;
    cudaMalloc(&dbc, 16 * n); cudaMalloc(&dt, 8 * n); cudaMalloc(&dc, 8);
    cudaMemcpy(dbc, bc.data(), 16 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, t.data(), 8 * n, cudaMemcpyHostToDevice);
    for (size_t smem : {size_t(64 * 1024), size_t(183 * 1024)}) {
        for (int thr : {32, 256}) {
            cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            probe<<<1, thr, smem>>>(dbc, dt, n, dc);
            probe<<<1, thr, smem>>>(dbc, dt, n, dc);
            long long h; cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
            printf("smem %zu KB, %d threads: %.2f cycles/row (%s)\n", smem / 1024, thr, (double)h / n, cudaGetErrorString(cudaGetLastError()));
        }
    }
}
