// Microbenchmark: all SMs stream a large buffer (> L2) through per-CTA shared-memory rings of
// TMA bulk copies; stage = NP pieces of PB bytes (one bulk copy each).  Reports aggregate GB/s.
#include <cstdio>
#include <cstdint>
#include "../../paper_1209_1910_b200/csrc/common.cuh"
using namespace tinv;
template <int NP, int PB, int NS>
__global__ void k(const char* __restrict__ g, int64_t bytes_per_cta, double* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int STG = NP * PB;
    uint64_t* mb = reinterpret_cast<uint64_t*>(sm + (size_t)STG * NS);
    if (threadIdx.x == 0) { for (int i = 0; i < NS; i++) mbar_init(mb + i, 1); fence_mbar_init(); }
    __syncthreads();
    const char* src = g + (int64_t)blockIdx.x * bytes_per_cta;
    const int nst = (int)(bytes_per_cta / STG);
    uint32_t ph = 0;
    double acc = 0;
    int ps = 0;
    const int lane = threadIdx.x & 31;
    auto issue = [&]() {
        const int sl = ps % NS;
        if (lane == 0) mbar_expect_tx(mb + sl, STG);
        __syncwarp();
        if (lane < NP) bulk_g2s(sm + (size_t)sl * STG + lane * PB, src + (int64_t)ps * STG + lane * PB, PB, mb + sl);
        ps++;
    };
    if (threadIdx.x < 32) while (ps < nst && ps < NS) issue();
    for (int s = 0; s < nst; s++) {
        const int sl = s % NS;
        mbar_wait(mb + sl, (ph >> sl) & 1u); ph ^= 1u << sl;
        const double2* p = reinterpret_cast<const double2*>(sm + (size_t)sl * STG);
        for (int i = threadIdx.x; i < STG / 16; i += blockDim.x) { double2 v = p[i]; acc += v.x + v.y; }
        __syncthreads();
        if (threadIdx.x < 32 && ps < nst) issue();
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void kld(const double* __restrict__ g, int64_t nd_per_cta, double* sink) {
    const double2* p = reinterpret_cast<const double2*>(g + (int64_t)blockIdx.x * nd_per_cta);
    double acc = 0;
    for (int64_t i = threadIdx.x; i < nd_per_cta / 2; i += blockDim.x * 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = (i + u * blockDim.x < nd_per_cta / 2) ? __ldcg(p + i + u * blockDim.x) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < 8; u++) acc += v[u].x + v[u].y;
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int NP, int PB, int NS>
void run(const char* g, int64_t bpc, double* sink) {
    size_t smem = (size_t)NP * PB * NS + 128;
    cudaFuncSetAttribute(k<NP, PB, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<NP, PB, NS><<<148, 256, smem>>>(g, bpc, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) k<NP, PB, NS><<<148, 256, smem>>>(g, bpc, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("TMA %2d pieces x %5d B x %d stages: %7.1f GB/s  (%s)\n", NP, PB, NS, 5.0 * 148 * bpc / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    const int64_t bpc = 8 << 20;   // 8 MB per CTA, 1.2 GB total (> L2)
    char* g; double* sink;
    cudaMalloc(&g, bpc * 148 + 4096); cudaMalloc(&sink, 148 * 1024 * 8);
    cudaMemset(g, 0, bpc * 148);
    run<8, 4096, 4>(g, bpc, sink);
    run<8, 4096, 6>(g, bpc, sink);
    run<1, 32768, 4>(g, bpc, sink);
    run<16, 2048, 4>(g, bpc, sink);
    run<8, 2048, 8>(g, bpc, sink);
    run<4, 8192, 4>(g, bpc, sink);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    kld<<<148, 256>>>((const double*)g, bpc / 8, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) kld<<<148, 256>>>((const double*)g, bpc / 8, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ld.cg 8x16B/thread, 1 CTA/SM: %7.1f GB/s\n", 5.0 * 148 * bpc / (ms * 1e-3) / 1e9);
    return 0;
}
