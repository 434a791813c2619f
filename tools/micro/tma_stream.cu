// Microbenchmark: one CTA streams a contiguous buffer through a shared-memory ring of TMA bulk
// copies (thread 0 issues, all threads consume) -- single-SM bytes/cycle for several ring
// shapes; and a plain ld.global.cg loop for comparison.
#include <cstdio>
#include <cstdint>
#include "../../paper_1209_1910_b200/csrc/common.cuh"
using namespace tinv;
template <int STG, int NS>
__global__ void k(const double* __restrict__ g, int64_t nd, long long* cyc, double* sink, int reps) {
    extern __shared__ __align__(128) unsigned char sm[];
    double* ring = reinterpret_cast<double*>(sm);
    uint64_t* mb = reinterpret_cast<uint64_t*>(sm + (size_t)STG * NS * 8);
    if (threadIdx.x == 0) { for (int i = 0; i < NS; i++) mbar_init(mb + i, 1); fence_mbar_init(); }
    __syncthreads();
    uint32_t ph = 0;
    double acc = 0;
    const int nst = (int)(nd / STG);
    long long t0 = clock64();
    for (int rep = 0; rep < reps; rep++) {
        int ps = 0;
        auto issue = [&]() { int sl = ps % NS; mbar_expect_tx(mb + sl, STG * 8); bulk_g2s(ring + (size_t)sl * STG, g + (int64_t)ps * STG, STG * 8, mb + sl); ps++; };
        if (threadIdx.x == 0) while (ps < nst && ps < NS) issue();
        for (int s = 0; s < nst; s++) {
            int sl = s % NS;
            mbar_wait(mb + sl, (ph >> sl) & 1u); ph ^= 1u << sl;
            const double2* p = reinterpret_cast<const double2*>(ring + (size_t)sl * STG);
            for (int i = threadIdx.x; i < STG / 2; i += blockDim.x) { double2 v = p[i]; acc += v.x + v.y; }
            __syncthreads();
            if (threadIdx.x == 0 && ps < nst) issue();
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    sink[threadIdx.x] = acc;
}
__global__ void kld(const double* __restrict__ g, int64_t nd, long long* cyc, double* sink, int reps) {
    double acc = 0;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; rep++) {
        const double2* p = reinterpret_cast<const double2*>(g);
        for (int64_t i = threadIdx.x; i < nd / 2; i += blockDim.x * 8) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) v[u] = (i + u * blockDim.x < nd / 2) ? __ldcg(p + i + u * blockDim.x) : make_double2(0, 0);
#pragma unroll
            for (int u = 0; u < 8; u++) acc += v[u].x + v[u].y;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    sink[threadIdx.x] = acc;
}
template <int STG, int NS>
void run(const char* name, double* g, int64_t nd, long long* c, double* sink) {
    size_t smem = (size_t)STG * NS * 8 + 64;
    cudaFuncSetAttribute(k<STG, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h;
    for (int reps : {1, 10}) {
        k<STG, NS><<<1, 256, smem>>>(g, nd, c, sink, reps);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-28s reps=%2d  %.1f B/cycle  (%s)\n", name, reps, (double)nd * 8 * reps / h, cudaGetErrorString(cudaGetLastError()));
    }
}
int main() {
    const int64_t nd = 416 * 1024 / 8;
    double *g, *sink; long long* c;
    cudaMalloc(&g, nd * 8 + 4096); cudaMalloc(&sink, 8192); cudaMalloc(&c, 64);
    cudaMemset(g, 0, nd * 8);
    run<4096, 4>("ring 32KB x4", g, nd, c, sink);
    run<2048, 8>("ring 16KB x8", g, nd, c, sink);
    run<1024, 8>("ring 8KB x8", g, nd, c, sink);
    run<8192, 3>("ring 64KB x3", g, nd, c, sink);
    long long h;
    for (int reps : {1, 10}) {
        kld<<<1, 256>>>(g, nd, c, sink, reps);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-28s reps=%2d  %.1f B/cycle\n", "ld.cg 8 x 16B per thread", reps, (double)nd * 8 * reps / h);
    }
    return 0;
}
