// Round-trip cost of K3-TC/P's accumulator handshake on a CTA pair, without
// MMAs: the leader's MMA warp commits accf[d] (tcgen05.commit multicast to both
// CTAs), 16 epilogue warps per CTA wait on it, drain their 32 x 32 slice of the
// 128-column accumulator with two tcgen05.ld x16, and arrive on the leader's
// acce[d] (remote for the peer); the MMA warp waits acce before re-committing.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/handshake_bench tools/handshake_bench.cu
//
// Variants: buffers (2 or 4 accumulators in flight), ldtm (drain or not).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                 \
    do {                                                                      \
        cudaError_t e = (x);                                                  \
        if (e != cudaSuccess) {                                               \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));           \
            return 1;                                                         \
        }                                                                     \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void wait_cta(uint32_t bar, uint32_t par) {
    asm volatile(
        "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra W_%=;\n\t}" ::"r"(bar),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void wait_cl(uint32_t bar, uint32_t par) {
    asm volatile(
        "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, "
        "[%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(bar),
        "r"(par)
        : "memory");
}

template <int NBUF, bool LDTM>
__global__ void __launch_bounds__(640, 1) k_hs(int iters, int* sink) {
    __shared__ uint64_t accf[4], acce[4];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t crank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    if (threadIdx.x == 0) {
        for (int d = 0; d < 4; ++d) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&accf[d])) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(su32(&acce[d])) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         su32(&tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    uint32_t L_acce;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(L_acce) : "r"(su32(&acce[0])));
    const int cols = 256 / NBUF;
    uint32_t acc = 0;
    if (warp == 0 && crank == 0) {
        for (int t = 0; t < iters; ++t) {
            const int d = t % NBUF;
            if (t >= NBUF) wait_cl(su32(&acce[d]), ((t / NBUF) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile(
                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::"
                "cluster.b64 [%0], %1;\n\t}" ::"r"(su32(&accf[d])),
                "h"((uint16_t)3)
                : "memory");
        }
    } else if (warp >= 4) {
        const int q = warp & 3, sub = (warp - 4) >> 2;
        for (int t = 0; t < iters; ++t) {
            const int d = t % NBUF;
            wait_cta(su32(&accf[d]), (t / NBUF) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (LDTM) {
                const uint32_t a = tmem + ((uint32_t)(q * 32) << 16) + 256 + d * cols + sub * (cols / 4);
                uint32_t v[16];
                for (int h = 0; h < cols / 64; ++h) {
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"
                        "%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                          "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                          "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                        : "r"(a + 16 * h));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    for (int k = 0; k < 16; ++k) acc += v[k];
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(L_acce + 8 * d)
                             : "memory");
        }
    }
    if (acc == 0x12345u) sink[0] = 1;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

template <int NBUF, bool LDTM>
static int run(int sms, const char* name) {
    int* sink;
    CK(cudaMalloc(&sink, 4));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms / 2 * 2);
    cfg.blockDim = dim3(640);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int iters = 20000;
    CK(cudaLaunchKernelEx(&cfg, k_hs<NBUF, LDTM>, 1000, sink));
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelEx(&cfg, k_hs<NBUF, LDTM>, iters, sink));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("%s: %.1f ns per tile (%.0f clk at 1965 MHz)\n", name, ms * 1e6 / iters,
           ms * 1e-3 / iters * 1.965e9);
    cudaFree(sink);
    return 0;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    if (run<2, false>(sms, "2 buffers, no drain")) return 1;
    if (run<2, true>(sms, "2 buffers, drain")) return 1;
    if (run<4, false>(sms, "4 buffers, no drain")) return 1;
    if (run<4, true>(sms, "4 buffers, drain")) return 1;
    return 0;
}
