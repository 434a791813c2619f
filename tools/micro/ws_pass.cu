// Microbenchmark: one warp-specialised wide pass per CTA (warp 0 issues TMA row pieces of
// 448 doubles, 7 per stage, full/empty mbarriers; warps 1..7 consume), bytes per CTA as in
// cfg4 at p ~ 4000 (54 rows x 4000 doubles).  MODE 0: column accumulate (thread owns 2
// columns); 1: row dots, one warp per piece, one vector block in shared memory (pass D);
// 2: row dots against two vectors (pass TN).
#include <cstdio>
#include <cstdint>
#include "../../paper_1209_1910_b200/csrc/common.cuh"
using namespace tinv;
constexpr int NCW = 7, NCT = 224, PW = 448, PPS = 7, SD = PPS * PW;
__device__ __forceinline__ double wsum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <int NS, int MODE>
__global__ void __launch_bounds__(256, 1) k(const double* __restrict__ Y, int rows, int cols, double* out, int reps) {
    extern __shared__ __align__(128) unsigned char sm[];
    double* ring = reinterpret_cast<double*>(sm);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)SD * NS * 8);
    uint64_t* empty = full + NS;
    double* vb = reinterpret_cast<double*>(empty + NS);   // 2 x PW vector block(s)
    double* racc = vb + 2 * PW;                            // per-row sums
    for (int i = threadIdx.x; i < 2 * PW; i += blockDim.x) vb[i] = 1.0 / (1 + i);
    for (int i = threadIdx.x; i < 128; i += blockDim.x) racc[i] = 0.0;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) { for (int i = 0; i < NS; i++) { mbar_init(full + i, 1); mbar_init(empty + i, NCW); } fence_mbar_init(); }
    __syncthreads();
    const double* base = Y + (int64_t)blockIdx.x * rows * cols;
    const int nb = (cols + PW - 1) / PW, spb = (rows + PPS - 1) / PPS, nst = nb * spb;
    uint32_t g = 0, u = 0;
    double a0 = 0, a1 = 0;
    for (int rep = 0; rep < reps; rep++) {
        if (warp == 0) {
            for (int s = 0; s < nst; s++, g++) {
                const int kb = s / spb, ra = (s % spb) * PPS, slot = g % NS;
                if (g >= NS) mbar_wait(empty + slot, ((g / NS) - 1) & 1u);
                const int r = ra + lane;
                if (lane < PPS && r < rows) {
                    const int a = kb * PW, b = min(cols, a + PW);
                    mbar_add_tx(full + slot, (b - a) * 8);
                    bulk_g2s(ring + slot * SD + lane * PW, base + (int64_t)r * cols + a, (b - a) * 8, full + slot);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(full + slot);
            }
        } else {
            const int tc = tid - 32;
            for (int s = 0; s < nst; s++, u++) {
                const int kb = s / spb, ra = (s % spb) * PPS, slot = u % NS;
                mbar_wait(full + slot, (u / NS) & 1u);
                const double* st = ring + slot * SD;
                if (MODE == 0) {
                    for (int q = 0; q < PPS && ra + q < rows; q++) {
                        const double2 y = *reinterpret_cast<const double2*>(st + q * PW + 2 * tc);
                        const double c = 0.5 + q;
                        a0 = fma(y.x, c, a0);
                        a1 = fma(y.y, c, a1);
                    }
                } else {
                    const int q = warp - 1;
                    if (ra + q < rows) {
                        double d1 = 0.0, d2 = 0.0;
                        const double* rowp = st + q * PW;
#pragma unroll
                        for (int e = 0; e < PW; e += 64) {
                            const int cl = e + 2 * lane;
                            const double2 y = *reinterpret_cast<const double2*>(rowp + cl);
                            const double2 vv = *reinterpret_cast<const double2*>(vb + cl);
                            d1 = fma(y.x, vv.x, d1);
                            d1 = fma(y.y, vv.y, d1);
                            if (MODE == 2) {
                                const double2 ww = *reinterpret_cast<const double2*>(vb + PW + cl);
                                d2 = fma(y.x, ww.x, d2);
                                d2 = fma(y.y, ww.y, d2);
                            }
                        }
                        d1 = wsum(d1);
                        if (MODE == 2) d2 = wsum(d2);
                        if (lane == 0) { racc[ra + q] += d1; if (MODE == 2) racc[64 + ((ra + q) & 63)] += d2; }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + slot);
                if ((s + 1) % spb == 0) { out[blockIdx.x * 512 + kb % 2] = a0 + a1 + racc[lane]; }
            }
        }
        __syncthreads();
    }
}
template <int NS, int MODE = 0>
void run(double* Y, int rows, int cols, double* out) {
    size_t smem = (size_t)SD * NS * 8 + 16 * NS + 8 * (2 * PW + 128);
    cudaFuncSetAttribute(k<NS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<NS, MODE><<<148, 256, smem>>>(Y, rows, cols, out, 1);
    cudaEventRecord(a);
    k<NS, MODE><<<148, 256, smem>>>(Y, rows, cols, out, 10);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double bytes = 10.0 * 148 * rows * (double)cols * 8;
    printf("MODE=%d NS=%d rows=%d cols=%d: %.1f us/pass  %.1f GB/s (%s)\n", MODE, NS, rows, cols, ms * 1e3 / 10, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    double *Y, *out;
    const int rows = 54, cols = 4032;
    const size_t ybytes = (size_t)148 * 108 * 8064 * 8;   // the largest case below
    cudaMalloc(&Y, ybytes); cudaMalloc(&out, 148 * 512 * 8);
    cudaMemset(Y, 0, ybytes);
    run<4>(Y, rows, cols, out);
    run<7>(Y, rows, cols, out);
    run<7>(Y, 108, 8064, out);
    run<7>(Y, 27, 2016, out);
    run<7, 1>(Y, rows, cols, out);
    run<7, 2>(Y, rows, cols, out);
    run<7, 1>(Y, 108, 8064, out);
    run<7, 2>(Y, 108, 8064, out);
    return 0;
}
