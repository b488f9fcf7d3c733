// K1 on the device: the O(n^2) scans and layouts of an instance load
// (hm/model.py:55-81 holds C and W; everything here is derived from them).
//
//   k_scan_instance  one pass over C and W: min / max cost (the 16-bit
//                    allocation pre-filter's range), exact symmetry of C,
//                    whether every flow is an integer in [0, 2^32), the
//                    largest flow and the largest entry of the triangular
//                    fold, the total flow
//   k_build_planes   the u8 byte planes of W (K3-TC/P's B operand) and of its
//                    block-upper-triangular fold (symmetric costs)
//
// The host used to do these in single-threaded loops over n^2 doubles
// (n = 6000: 36 M entries, ~0.3 s per pass on one core).
#include <cstdint>

#include "hg_internal.cuh"

namespace hg {

namespace {

constexpr int kTriBlock = 128;  // the fold's block size = K3-TC/P's tile and K block

__device__ __forceinline__ unsigned long long pos_bits(double v) {
    // ordering key of a non-negative double (and -0.0 as +0.0): the IEEE bit
    // pattern of a non-negative value is monotone in the value
    return (unsigned long long)__double_as_longlong(v + 0.0);
}

// the triangular fold: W inside diagonal 128-blocks, W + W^T above them, 0 below
__device__ __forceinline__ double fold_at(const double* __restrict__ W, int n, int i, int j) {
    const int bi = i / kTriBlock, bj = j / kTriBlock;
    if (bi == bj) return W[(size_t)i * n + j];
    if (bj > bi) return W[(size_t)i * n + j] + W[(size_t)j * n + i];
    return 0.0;
}

__global__ void k_scan_instance(const double* __restrict__ C, const double* __restrict__ W, int n,
                                InstanceScan* out) {
    unsigned long long cmin = ~0ull, cmax = 0ull, wmax = 0ull, mmax = 0ull, wmin = ~0ull;
    int intw = 1, sym = 1, glsb = 1 << 30;
    double wsum = 0.0;
    const int64_t total = (int64_t)n * n;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(x / n), j = (int)(x - (int64_t)i * n);
        const double c = C[x];
        const unsigned long long cb = pos_bits(c);
        cmin = cb < cmin ? cb : cmin;
        cmax = cb > cmax ? cb : cmax;
        if (j > i && c != C[(size_t)j * n + i]) sym = 0;
        const double w = W[x];
        if (!(w >= 0.0 && w < 4294967296.0 && w == floor(w))) intw = 0;
        const unsigned long long wb = pos_bits(w >= 0.0 ? w : 0.0);
        wmax = wb > wmax ? wb : wmax;
        if (w > 0.0) {
            wmin = wb < wmin ? wb : wmin;
            // exponent of the flow's lowest set bit (w = odd * 2^e)
            const int ex = (int)((wb >> 52) & 0x7ff);
            const unsigned long long man = (wb & 0xfffffffffffffull) | (ex ? 1ull << 52 : 0ull);
            const int e = (ex ? ex : 1) - 1075 + __ffsll((long long)man) - 1;
            glsb = e < glsb ? e : glsb;
        }
        const double m = fold_at(W, n, i, j);
        const unsigned long long mb = pos_bits(m >= 0.0 ? m : 0.0);
        mmax = mb > mmax ? mb : mmax;
        wsum += w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
        cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
        wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
        mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
        wmin = min(wmin, __shfl_xor_sync(0xffffffffu, wmin, o));
        glsb = min(glsb, __shfl_xor_sync(0xffffffffu, glsb, o));
        wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    }
    intw = __all_sync(0xffffffffu, intw);
    sym = __all_sync(0xffffffffu, sym);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&out->cmin_bits, cmin);
        atomicMax(&out->cmax_bits, cmax);
        atomicMax(&out->wmax_bits, wmax);
        atomicMax(&out->mmax_bits, mmax);
        atomicMin(&out->wmin_bits, wmin);
        atomicMin(&out->lsb_exp, glsb);
        if (!intw) atomicAnd(&out->int_flows, 0);
        if (!sym) atomicAnd(&out->symmetric, 0);
        // integer flows: every partial sum is an exact integer below 2^53 for
        // any order while the total stays below 2^53 (only `< 2^32` is asked)
        atomicAdd(&out->wsum, wsum);
    }
}

// the flow as an integer multiple of the quantum: rint(w / wscale), exact for
// integer flows (wscale = 1); wscale is a power of two, so the division is exact
__device__ __forceinline__ uint64_t quant(double w, double inv) {
    return (uint64_t)rint(w * inv);
}

// plane d of W8 / M8 = byte d of Q (and of Q's triangular fold), zero in the padding
__global__ void k_build_planes(const double* __restrict__ W, int n, int nt, double inv, int P,
                               int Ptri, uint8_t* __restrict__ W8, uint8_t* __restrict__ M8) {
    const int64_t per = (int64_t)nt * nt;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < per;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(x / nt), j = (int)(x - (int64_t)i * nt);
        const bool in = i < n && j < n;
        const uint64_t q = in ? quant(W[(size_t)i * n + j], inv) : 0ull;
        for (int d = 0; d < P; ++d) W8[d * per + x] = (uint8_t)(q >> (8 * d));
        if (M8) {
            uint64_t m = 0ull;
            if (in) {
                const int bi = i / kTriBlock, bj = j / kTriBlock;
                m = bi == bj ? q : (bj > bi ? q + quant(W[(size_t)j * n + i], inv) : 0ull);
            }
            for (int d = 0; d < Ptri; ++d) M8[d * per + x] = (uint8_t)(m >> (8 * d));
        }
    }
}

unsigned grid_of(int64_t work) {
    int64_t g = (work + 255) / 256;
    return (unsigned)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

}  // namespace

int launch_scan_instance(const double* C, const double* W, int n, InstanceScan* out,
                         cudaStream_t s) {
    const InstanceScan init = {~0ull, 0ull, 0ull, 0ull, ~0ull, 0.0, 1, 1, 1 << 30};
    HG_CUDA(cudaMemcpyAsync(out, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_scan_instance<<<grid_of((int64_t)n * n), 256, 0, s>>>(C, W, n, out);
    HG_LAUNCHED();
    // the pageable source above is staged before the copy returns
    return HG_OK;
}

int launch_build_planes(const double* W, int n, int nt, double wscale, int P, int Ptri,
                        uint8_t* W8, uint8_t* M8, cudaStream_t s) {
    k_build_planes<<<grid_of((int64_t)nt * nt), 256, 0, s>>>(W, n, nt, 1.0 / wscale, P, Ptri, W8,
                                                             M8);
    HG_LAUNCHED();
    return HG_OK;
}

}  // namespace hg
