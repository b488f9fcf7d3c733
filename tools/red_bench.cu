// Throughput of K3-TC/P's bin update, the epilogue's per-element operation:
// G[c][r] += D[r][i] in shared memory, c = the element's cluster (< p = 20), r
// the thread's row (4 column-quarter warps share a row), 16 warps per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/red_bench tools/red_bench.cu
//
// Variants (cycles per warp-wide update per SM, 148 CTAs x 512 threads):
//   0 red.shared.add.u32 (the kernel's)
//   1 atom.shared.add.u32 (result kept)
//   2 red.shared.add.u32, every lane of a warp on ONE bank row (worst case: conflicts)
//   3 red.shared.add.u64 on [c][r] 64-bit bins
//   4 ld + add + st on per-thread private bins (no atomics; 2 private copies)
//   5 red.shared.add.u32 with 4 warps per row-group spread over 4 bin copies
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

constexpr int kP = 20, kThreads = 512, kIters = 2048;

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int V>
__global__ void __launch_bounds__(kThreads, 1) k_red(uint32_t seed, unsigned long long* cyc,
                                                     uint32_t* sink) {
    extern __shared__ __align__(16) uint32_t bins[];
    const int tid = threadIdx.x, r = tid & 127;
    const int words = V == 3 ? kP * 128 * 2 : (V == 4 ? kThreads * 2 * kP : (V == 5 ? 4 * kP * 128 : kP * 128));
    for (int x = tid; x < words; x += kThreads) bins[x] = 0;
    __syncthreads();
    uint32_t h = seed ^ (uint32_t)(tid >> 5) * 0x9E3779B9u;  // per-warp cluster stream
    const uint32_t base = su32(bins);
    const long long t0 = clock64();
    for (int it = 0; it < kIters; it += 32) {
        uint32_t cw[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            h = h * 1664525u + 1013904223u;
            // 4 cluster ids < 16 per word (cheap: the update, not this, is measured)
            cw[q] = h & 0x0F0F0F0Fu;
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint32_t c = __byte_perm(cw[k >> 2], 0u, 0x4440u + (k & 3));
            const uint32_t v = (uint32_t)(k + it);
            if (V == 0 || V == 1) {
                const uint32_t a = base + c * 512u + (uint32_t)r * 4u;
                if (V == 0)
                    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
                else {
                    uint32_t o;
                    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(o) : "r"(a), "r"(v) : "memory");
                    h ^= o & 1u;
                }
            } else if (V == 2) {
                const uint32_t a = base + c * 512u + (uint32_t)(r & 3) * 128u;
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
            } else if (V == 3) {
                const uint32_t a = base + c * 1024u + (uint32_t)r * 8u;
                asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a), "l"((unsigned long long)v) : "memory");
            } else if (V == 4) {
                // private copy k & 1 of this thread's bins: [copy][c][tid]
                uint32_t* b = bins + ((k & 1) * kP + c) * kThreads + tid;
                *reinterpret_cast<volatile uint32_t*>(b) = *reinterpret_cast<volatile uint32_t*>(b) + v;
            } else {
                const uint32_t a = base + ((uint32_t)(tid >> 7) * kP + c) * 512u + (uint32_t)r * 4u;
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
    if (tid < 32) sink[blockIdx.x * 32 + tid] = bins[tid] + h;
}

template <int V>
int run(const char* name) {
    unsigned long long* cyc;
    uint32_t* sink;
    CK(cudaMalloc(&cyc, 8));
    CK(cudaMalloc(&sink, 148 * 32 * 4));
    const int words = V == 3 ? kP * 128 * 2 : (V == 4 ? kThreads * 2 * kP : (V == 5 ? 4 * kP * 128 : kP * 128));
    const size_t smem = (size_t)words * 4;
    CK(cudaFuncSetAttribute(k_red<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(cyc, 0, 8));
        k_red<V><<<148, kThreads, smem>>>(12345u + rep, cyc, sink);
        CK(cudaDeviceSynchronize());
    }
    unsigned long long c;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    const double per_cta = (double)c / 148.0;
    const double warp_ops = (double)kIters * (kThreads / 32);
    printf("{\"variant\": %d, \"name\": \"%s\", \"cycles_per_cta\": %.0f, \"cycles_per_warp_update\": %.3f, "
           "\"element_updates_per_clk_per_sm\": %.2f}\n",
           V, name, per_cta, per_cta / warp_ops, warp_ops * 32 / per_cta);
    cudaFree(cyc);
    cudaFree(sink);
    return 0;
}

int main() {
    int rc = 0;
    rc |= run<0>("red.shared.add.u32 bins[c][r]");
    rc |= run<1>("atom.shared.add.u32 bins[c][r]");
    rc |= run<2>("red.shared.add.u32, 8 lanes per bank (conflicts)");
    rc |= run<3>("red.shared.add.u64 bins[c][r]");
    rc |= run<4>("ld+add+st private bins (2 copies)");
    rc |= run<5>("red.shared.add.u32, a bin copy per column quarter");
    return rc;
}
