// common.cuh -- device helpers shared by the libtinv kernels (sm_100a).
// Nothing here is shared with the CPU oracle (oracle/); the rules (RNG formula,
// pivot floor, shift ladder, stopping constants) are restated from DESIGN.md.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tinv {

constexpr double kEps = 1.1102230246251565404e-16;  // 2^-53, unit roundoff (R3/R4)
constexpr int kMaxIts = 5;                          // reading 9
constexpr int kPasses = 2;                          // reading 9: first pass + 1 extra
constexpr int kMaxRestart = 2;                      // reading 16

// ---------------------------------------------------------------- start vectors (reading 7)
// SplitMix64 finaliser of seed + phi64 * ctr; top 53 bits -> u in [0,1); value 2u - 1.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t ctr) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL * ctr;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double start_entry(uint64_t seed, int64_t n, int64_t j,
                                                       int64_t restart, int64_t i) {
    uint64_t ctr = 1ULL + ((uint64_t)restart * (uint64_t)n + (uint64_t)j) * (uint64_t)n + (uint64_t)i;
    uint64_t z = mix64(seed, ctr);
    double u = (double)(z >> 11) * 0x1.0p-53;
    return 2.0 * u - 1.0;  // exact in fp64
}

// pivot floor (reading 6): |p| < eps*||T||_1 -> sign(p)*eps*||T||_1, + for p == 0
__device__ __forceinline__ double pivot_floor(double p, double tiny) {
    return (fabs(p) < tiny) ? ((p >= 0.0) ? tiny : -tiny) : p;
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block sum: fixed tree over warps.  `red` needs blockDim/32 doubles.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = (lane < NT / 32) ? red[lane] : 0.0;
        r = warp_sum(r);
        if (lane == 0) red[0] = r;
    }
    __syncthreads();
    r = red[0];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------- group barrier
// A group is a contiguous range of co-resident CTAs of a persistent (cooperative)
// launch.  Sense-reversal barrier on a (count, generation) pair in global memory;
// the gpu-scope fences give the release/acquire ordering (and invalidate L1) so data
// written by any CTA before the barrier is visible to every CTA after it.
struct GroupBarrier {
    unsigned int count;   // monotonic arrival counter (episode e completes at count == e G)
    unsigned int pad;
};

// Barrier of a group whose CTAs live on nrk ranks (rank-replicated counters at bar + delta[k]
// doubles): every CTA adds 1 to every rank's counter (system-scope atomics: the replicas may
// be peer memory over NVLink), then polls its own rank's counter until all Gt CTAs of the
// episode arrived.  System-scope fences order the mirrored stores of all ranks.
__device__ __forceinline__ void group_sync_ranks(GroupBarrier* b, const int64_t* delta, int nrk, int Gt,
                                                 unsigned int& epoch) {
    __threadfence_system();   // this thread's mirrored (possibly remote) stores
    __syncthreads();
    if (threadIdx.x == 0) {
        epoch++;
        const unsigned int target = epoch * (unsigned int)Gt;
        for (int k = 0; k < nrk; k++) {
            unsigned int* c = reinterpret_cast<unsigned int*>(reinterpret_cast<double*>(&b->count) + delta[k]);
            atomicAdd_system(c, 1u);
        }
        volatile unsigned int* vc = &b->count;
        uint32_t spins = 0;
        while ((int)(*vc - target) < 0) {
            if (++spins > (1u << 30)) __trap();
        }
        __threadfence_system();
    }
    __syncthreads();
}

// `epoch` is the caller's episode counter (identical in every CTA of the group): arrive with
// one atomic, then poll until all G CTAs of this episode have arrived.  The gpu-scope fences
// give the release/acquire ordering (and invalidate L1) so data written by any CTA before the
// barrier is visible to every CTA after it.  A barrier that never completes traps.
__device__ __forceinline__ void group_sync(GroupBarrier* b, int G, unsigned int& epoch) {
    if (G == 1) {
        __syncthreads();
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        epoch++;
        const unsigned int target = epoch * (unsigned int)G;
        __threadfence();
        unsigned int v = atomicAdd(&b->count, 1u) + 1u;
        volatile unsigned int* vc = &b->count;
        uint32_t spins = 0;
        while ((int)(v - target) < 0) {
            v = *vc;
            if (++spins > (1u << 30)) __trap();
        }
        __threadfence();
    }
    __syncthreads();
}

// ---------------------------------------------------------------- batched (per-vector) arrays
// Factors and iterates of the batched solve: blocks of 32 slots (one warp; vector perm[slot],
// prep.cu), each block row-major [row i][lane] (256 B per row), blocks one after the other:
// element (i, slot) at ((slot / 32) n + i) 32 + slot % 32.  A warp's rows [a, b) are one
// contiguous span.
__host__ __device__ __forceinline__ int64_t bix(int64_t i, int64_t j, int64_t n) {
    return ((j >> 5) * n + i) * 32 + (j & 31);
}

// ---------------------------------------------------------------- packed layouts
// Y (row-major, zero-free "assignment model" of Fig. 1): row i of
// Y_m holds columns 0..min(i, m-1), padded to an even count (16-byte rows).  Narrow clusters
// (m <= kNarrowM) use a uniform row stride roundup(m, 2) instead (the padding of the leading
// triangle is < m^2/2 doubles), so any row range is one contiguous span with a fixed stride.
constexpr int kNarrowM = 64;
constexpr int kLabMax = 8;   // largest block of the blocked look-ahead (cwy.cu)
__host__ __device__ __forceinline__ int64_t y_row_off(int64_t i, int64_t m) {
    if (m <= kNarrowM) return i * ((m + 1) & ~int64_t(1));
    auto tri = [](int64_t r) -> int64_t {  // sum_{r'<r} roundup(r'+1, 2)
        int64_t a = r >> 1, b = r & 1;
        return 2 * a * (a + 1) + 2 * b * (a + 1);
    };
    if (i <= m) return tri(i);
    int64_t m2 = (m + 1) & ~int64_t(1);
    return tri(m) + (i - m) * m2;
}
// T, column-packed: column k holds T[0..k, k], padded to even.
__host__ __device__ __forceinline__ int64_t tcol_off(int64_t k) {
    int64_t a = k >> 1, b = k & 1;
    return 2 * a * (a + 1) + 2 * b * (a + 1);
}

}  // namespace tinv

// ---------------------------------------------------------------- TMA bulk copies (sm_90+ / sm_100a)
// Non-tensor bulk copies global -> shared completed on an mbarrier (transaction bytes).  A
// non-cluster launch is a cluster of one CTA, so the CTA's own shared addresses are valid
// shared::cluster addresses.
namespace tinv {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// generic-proxy global writes (possibly by other CTAs, ordered by a barrier) -> later bulk reads
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// add transaction bytes without arriving (several lanes may each announce their own copy)
__device__ __forceinline__ void mbar_add_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Waits for the phase; a wait that never completes (a pipeline bug) traps after ~10 s
// instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins > (1u << 27)) __trap();
    }
}
// bytes: multiple of 16; src, dst 16-byte aligned
// bulk shared -> global store (bulk-group completion); 16-byte aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"((uint32_t)__cvta_generic_to_shared(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N committed bulk stores may still be reading their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
// every committed bulk store complete (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// The same copy with an L2 eviction-priority hint (a policy from l2_policy_*): streams that are
// read once use evict_first, so they do not push reused data (partial sums, vectors) out of L2.
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

}  // namespace tinv
