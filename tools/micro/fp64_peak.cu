// Micro: fp64 throughput of the two instruction paths a blocked look-ahead GEMM could use on
// B200 (sm_100a): DFMA (CUDA cores) and DMMA (mma.sync.aligned.m8n8k4 f64 tensor-core op).
// Every SM runs 4 warps x ILP independent accumulator chains; flops counted as 2 per FMA
// (DFMA: 32 lanes x 2; DMMA m8n8k4: 2 * 8*8*4 = 512 per warp instruction).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1 << 16;

template <int ILP>
__global__ void dfma_kernel(double* out, double s) {
    double a[ILP];
#pragma unroll
    for (int i = 0; i < ILP; i++) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < ILP; i++) a[i] = fma(a[i], s, 1e-9);
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < ILP; i++) t += a[i];
    if (t == 12345.0) out[0] = t;
}

template <int ILP>
__global__ void dmma_kernel(double* out, double s) {
    double acc[ILP][2];
    const double av = threadIdx.x * 1e-3 + s, bv = 1.0 - s;
#pragma unroll
    for (int i = 0; i < ILP; i++) acc[i][0] = acc[i][1] = 0.0;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < ILP; i++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(av), "d"(bv));
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < ILP; i++) t += acc[i][0] + acc[i][1];
    if (t == 12345.0) out[0] = t;
}

template <class K>
double run(K kern, int blocks, int threads, double flops_per_thread_iter) {
    double* out;
    cudaMalloc(&out, 8);
    kern<<<blocks, threads>>>(out, 0.999);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out, 0.999);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(out);
    return (double)blocks * threads * ITERS * flops_per_thread_iter / (ms * 1e-3) / 1e12;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 16}) {
        printf("DFMA  ILP=8  %2d warps/SM: %.2f TFLOP/s\n", w, run(dfma_kernel<8>, sms, 32 * w, 2.0 * 8));
        // per warp instruction 512 flops = 16 per thread
        printf("DMMA  ILP=4  %2d warps/SM: %.2f TFLOP/s\n", w, run(dmma_kernel<4>, sms, 32 * w, 16.0 * 4));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
