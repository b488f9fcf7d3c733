// Dense int8 tensor-core peak of this B200 (tcgen05.mma kind::i8, u8 x u8 -> s32),
// the denominator of K3-TC/P's roofline (bench.py `roofline`).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int8_peak tools/int8_peak.cu -lcuda
//   ./int8_peak > profiles/int8_peak.json
//
// One CTA per SM streams back-to-back MMAs with both operands resident in
// shared memory (SWIZZLE_128B, K-major) into two TMEM accumulators -- nothing
// else runs, so the MMA rate is the pipe's.  Two shapes: cta_group::1
// M=128 N=256 K=32 and cta_group::2 M=256 N=256 K=32 (the CTA-pair form
// K3-TC/P issues, N=128 there).  Timed with CUDA events after a warm-up
// launch; ops = 2*M*N*K per MMA.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                    \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// ATMEM: the A operand read from TMEM columns 256.. (tcgen05.mma ... [a_tmem]),
// as K3-TC/P does with its one-hot; N = 128 then (accumulators at 0 and 128)
template <int CG, bool ATMEM, int MODE = 0>
__global__ void __launch_bounds__(128, 1) k_peak(int iters, uint32_t idesc, int* sink) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    unsigned char* a = sm;            // 128 rows x 128 B
    unsigned char* b = sm + 16384;    // 256 rows x 128 B (CG=2: 128 rows per CTA)
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t tslot;
    for (int x = threadIdx.x; x < (16384 + 32768) / 4; x += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[x] = 0x01010101u * ((x * 2654435761u) >> 28);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             su32(&tslot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             su32(&tslot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CG == 2)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                         : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    uint32_t crank = 0;
    if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    if (threadIdx.x == 0 && crank == 0) {
        const uint64_t ad = sw128(su32(a)), bd = sw128(su32(b));
        if (MODE >= 3) {
            // K3-TC/P's triangular unit (MODE 3: tiles of 8, 7, .., 1 K blocks)
            // or full-W unit (MODE 4: 8 tiles of 8 blocks): accumulators
            // alternate per tile, the tile's first MMA overwrites, a commit per
            // tile; A = the one-hot columns 0..255, accumulators at 256 / 384
            int done = 0, t = 0;
            while (done < iters) {
                for (int I = 0; I < 8 && done < iters; ++I, ++t) {
                    const uint32_t d = tmem + 256 + (t & 1) * 128;
                    const int k0 = MODE == 3 ? I : 0;
                    for (int kb = k0; kb < 8; ++kb, ++done)
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                                "r"(tmem + kb * 32 + ks * 8), "l"(bd + 2 * ks), "r"(idesc),
                                "r"((int)(kb != k0 || ks))
                                : "memory");
                    asm volatile(
                        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                        " [%0], %1;" ::"r"(su32(&bar2)),
                        "h"((uint16_t)3)
                        : "memory");
                }
            }
        } else
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = MODE ? tmem + 256 + ((it >> 3) & 1) * 128
                                    : tmem + (it & 1) * (ATMEM ? 128 : 256);
            const uint32_t acol = MODE ? tmem + (it & 7) * 32 : tmem + 256;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                if (ATMEM)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                        "r"(acol + ks * 8), "l"(bd + 2 * ks), "r"(idesc),
                        "r"((int)((MODE ? (it & 7) : it > 1) || ks))
                        : "memory");
                else if (CG == 1)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad + 2 * ks), "l"(bd + 2 * ks), "r"(idesc), "r"((int)(it > 1 || ks))
                        : "memory");
                else
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad + 2 * ks), "l"(bd + 2 * ks), "r"(idesc), "r"((int)(it > 1 || ks))
                        : "memory");
            }
            if (MODE == 2)  // a commit per K block, as K3-TC/P's stage/tile commits
                asm volatile(
                    "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                    " [%0], %1;" ::"r"(su32(&bar2)),
                    "h"((uint16_t)3)
                    : "memory");
        }
        if (CG == 1)
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    su32(&bar))
                : "memory");
        else
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                " [%0], %1;" ::"r"(su32(&bar)),
                "h"((uint16_t)3)
                : "memory");
    }
    if (threadIdx.x == 0) {
        asm volatile(
            "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t"
            "@!P bra W_%=;\n\t}" ::"r"(su32(&bar))
            : "memory");
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (v == 0x7fffffffu) sink[0] = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CG == 2)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                         : "memory");
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// TMEM read throughput: `warps` warps per CTA, each reading its lane quadrant
// (32 lanes) x 32 columns per round with two 32x32b.x16 loads, as K3-TC/P's
// epilogue does; bytes per SM per clock
__global__ void __launch_bounds__(640, 1) k_ldtm(int rounds, int* sink) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         su32(&tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) & 3) * 32;
    uint32_t acc = 0;
    for (int r = 0; r < rounds; ++r) {
        uint32_t v[32];
        const uint32_t a = base + (uint32_t)(r & 1) * 128;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(a));
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15}, [%16];"
            : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
              "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(a + 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += v[k];
    }
    if (acc == 0x12345678u) sink[0] = 1;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

static int run_ldtm(int sms, int warps, double* bpc, float* ms_out) {
    int* sink;
    CK(cudaMalloc(&sink, 4));
    const int rounds = 20000;
    k_ldtm<<<sms, warps * 32>>>(rounds / 4, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        k_ldtm<<<sms, warps * 32>>>(rounds, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double bytes = (double)warps * 32 * 32 * 4 * rounds;  // per SM
    *bpc = bytes / (best * 1e-3 * clk * 1e3);
    *ms_out = best;
    cudaFree(sink);
    return 0;
}

template <int CG, bool ATMEM = false, int MODE = 0>
static int run(int sms, int iters, double* tops, float* ms_out) {
    const int M = CG == 1 ? 128 : 256, N = ATMEM ? 128 : 256, K = 32;
    const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const size_t smem = 1024 + 16384 + 32768;
    int* sink;
    CK(cudaMalloc(&sink, 4));
    CK(cudaFuncSetAttribute(k_peak<CG, ATMEM, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms / CG * CG);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaLaunchKernelEx(&cfg, k_peak<CG, ATMEM, MODE>, iters / 4, idesc, sink));  // warm-up
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        CK(cudaLaunchKernelEx(&cfg, k_peak<CG, ATMEM, MODE>, iters, idesc, sink));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
    }
    const double mmas = (double)(sms / CG) * iters * 4;  // per CTA (group)
    *tops = mmas * 2.0 * M * N * K / (best * 1e-3) / 1e12;
    *ms_out = best;
    cudaFree(sink);
    return 0;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    const int iters = 20000;
    double t1, t2;
    float m1, m2;
    if (run<1>(sms, iters, &t1, &m1)) return 1;
    if (run<2>(sms, iters, &t2, &m2)) return 1;
    double t3;
    float m3;
    if (run<2, true>(sms, iters, &t3, &m3)) return 1;
    double l4, l16;
    float ml4, ml16;
    if (run_ldtm(sms, 4, &l4, &ml4)) return 1;
    if (run_ldtm(sms, 16, &l16, &ml16)) return 1;
    fprintf(stderr, "ldtm bytes/clk/SM: 4 warps %.1f, 16 warps %.1f\n", l4, l16);
    double t5, t6;
    float m5, m6;
    if (run<2, true, 1>(sms, iters, &t5, &m5)) return 1;
    if (run<2, true, 2>(sms, iters, &t6, &m6)) return 1;
    fprintf(stderr, "a_tmem K3 layout: %.1f TOPS; + commit per K block: %.1f TOPS\n", t5, t6);
    double t7, t8;
    float m7, m8;
    if (run<2, true, 3>(sms, iters, &t7, &m7)) return 1;
    if (run<2, true, 4>(sms, iters, &t8, &m8)) return 1;
    fprintf(stderr, "K3 unit pattern: triangular tiles %.1f TOPS; full tiles %.1f TOPS\n", t7, t8);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"what\": \"dense int8 tensor peak, tcgen05.mma kind::i8 (u8 x u8 -> s32), operands "
           "smem-resident, one CTA per SM, best of 5 launches (CUDA events)\", "
           "\"gpu\": \"%s\", \"sms\": %d, \"iters_per_cta\": %d, "
           "\"cta_group1_m128_n256_k32\": {\"tops\": %.1f, \"ms\": %.4f}, "
           "\"cta_group2_m256_n256_k32\": {\"tops\": %.1f, \"ms\": %.4f}, "
           "\"cta_group2_m256_n128_k32_a_tmem\": {\"tops\": %.1f, \"ms\": %.4f}, "
           "\"tmem_ld_bytes_per_clk_per_sm\": {\"warps4\": %.1f, \"warps16\": %.1f}, "
           "\"int8_tops\": %.1f, \"clock_rate_khz_attr\": %d}\n",
           prop.name, sms, iters, t1, m1, t2, m2, t3, m3, l4, l16, t1 > t2 ? t1 : t2, clk);
    return 0;
}
