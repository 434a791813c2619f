// Micro: cost of the wide kernel's R1-style deterministic partial reduction.
// 148 CTAs x 256 threads (persistent), per rep: every CTA writes its P partials
// (st.cg), optional 200 MB evict stream, group barrier, reduction of columns [k0,k1)
// over G partials (the kernel's loop), group barrier.  Times per phase (globaltimer, CTA 0).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o red_micro red_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NT = 256;
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ double ld(const double* p) { return __ldcg(p); }
__device__ __forceinline__ void st(double* p, double v) { __stcg(p, v); }

__device__ void gsync(unsigned int* cnt, int G, unsigned int& ep) {
    __syncthreads();
    if (threadIdx.x == 0) {
        ep++;
        const unsigned int target = ep * (unsigned)G;
        __threadfence();
        unsigned int v = atomicAdd(cnt, 1u) + 1u;
        volatile unsigned int* vc = cnt;
        while ((int)(v - target) < 0) v = *vc;
        __threadfence();
    }
    __syncthreads();
}

template <int RB>
__device__ double red_kernel_style(const double* P, int64_t mc, int G, int64_t k0, int64_t k1, double* out, double* sh) {
    const int tid = threadIdx.x;
    double chk = 0;
    for (int64_t kb = k0; kb < k1; kb += NT) {
        const int64_t K = (k1 - kb < NT) ? (k1 - kb) : NT;
        const int KP = (int)((K + 31) & ~int64_t(31));
        const int TG = NT / KP;
        const int kk = tid % KP, tg = tid / KP;
        double acc = 0.0;
        if (tg < TG && kk < K) {
            const double* col = P + kb + kk;
            for (int t0 = tg; t0 < G; t0 += RB * TG) {
                double v[RB];
#pragma unroll
                for (int u = 0; u < RB; u++) { const int t = t0 + u * TG; v[u] = (t < G) ? ld(col + (int64_t)t * mc) : 0.0; }
#pragma unroll
                for (int u = 0; u < RB; u++) if (t0 + u * TG < G) acc += v[u];
            }
        }
        if (TG > 1) {
            __syncthreads();
            sh[tid] = acc;
            __syncthreads();
            if (tg == 0 && kk < K) for (int u = 1; u < TG; u++) acc += sh[kk + u * KP];
            __syncthreads();
        }
        if (tg == 0 && kk < K) { st(out + kb + kk, acc); chk += acc; }
    }
    return chk;
}

__global__ void __launch_bounds__(NT, 1) kern(double* P, int64_t mc, int p, double* g, const double* big, int64_t nbig,
                                              int reps, int evict, unsigned int* cnt, unsigned long long* tm) {
    __shared__ double sh[NT];
    const int G = gridDim.x, r = blockIdx.x;
    unsigned int ep = 0;
    uint64_t tw = 0, te = 0, tr = 0, tb = 0;
    double sink = 0;
    for (int it = 0; it < reps; it++) {
        uint64_t t0 = gt();
        for (int k = threadIdx.x; k < p; k += NT) st(P + (int64_t)r * mc + k, (double)(k + r + it));
        uint64_t t1 = gt();
        if (evict) {
            // touch 200 MB per rep spread over the whole buffer: 64 KB from every page-sized stride
            const int64_t npg = nbig / (1 << 18);   // 2 MB pages
            double s = 0;
            for (int64_t pg = r; pg < npg; pg += G) {
                const double2* b = reinterpret_cast<const double2*>(big + pg * (1 << 18) + ((it * 8192) & ((1 << 18) - 1)));
                for (int64_t i = threadIdx.x; i < 4096; i += NT) { double2 v = __ldcs(b + i); s += v.x + v.y; }
            }
            sink += s;
        }
        uint64_t t2 = gt();
        gsync(cnt, G, ep);
        uint64_t t3 = gt();
        int64_t k0 = (int64_t)p * r / G, k1 = (int64_t)p * (r + 1) / G;
        sink += red_kernel_style<16>(P, mc, G, k0, k1, g, sh);
        uint64_t t4 = gt();
        gsync(cnt, G, ep);
        uint64_t t5 = gt();
        tw += t1 - t0; te += t2 - t1; tb += (t3 - t2) + (t5 - t4); tr += t4 - t3;
    }
    if (threadIdx.x == 0) {
        atomicAdd(tm + 0, tw); atomicAdd(tm + 1, te); atomicAdd(tm + 2, tb); atomicAdd(tm + 3, tr);
        if (r == 0) tm[4] = tr;
    }
    if (sink == 12345.678) g[0] = sink;
}

int main(int argc, char** argv) {
    const int G = 148, reps = 200;
    int64_t mc = 8000;
    double *P, *g, *big;
    int64_t nbig = (argc > 1 ? atoll(argv[1]) : 200ll) << 20 >> 3;   // MB
    unsigned int* cnt;
    unsigned long long* tm;
    cudaMalloc(&P, sizeof(double) * G * mc);
    cudaMalloc(&g, sizeof(double) * mc);
    cudaMalloc(&big, sizeof(double) * nbig);
    cudaMemset(big, 0, sizeof(double) * nbig);
    cudaMalloc(&cnt, 4);
    cudaMalloc(&tm, 8 * 8);
    for (int evict = 0; evict < 2; evict++)
        for (int p : {500, 4000, 8000}) {
            cudaMemset(cnt, 0, 4);
            cudaMemset(tm, 0, 64);
            void* args[] = {&P, &mc, &p, &g, &big, &nbig, (void*)&reps, &evict, &cnt, &tm};
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            cudaError_t e = cudaLaunchCooperativeKernel((void*)kern, dim3(G), dim3(NT), args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            unsigned long long h[8];
            cudaMemcpy(h, tm, 64, cudaMemcpyDeviceToHost);
            printf("evict=%d p=%5d err=%d  per rep: total %.2f us  write %.2f  evict %.2f  barriers(2) %.2f  reduce %.2f (cta0 %.2f) us\n",
                   evict, p, (int)e, 1e3 * ms / reps, h[0] / 1e3 / G / reps, h[1] / 1e3 / G / reps, h[2] / 1e3 / G / reps,
                   h[3] / 1e3 / G / reps, h[4] / 1e3 / reps);
        }
    return 0;
}
