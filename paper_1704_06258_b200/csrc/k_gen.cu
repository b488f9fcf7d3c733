// Device-side instance generation and hub-set enumeration.
//
// k_gen_urand restates hm/io.py:181-210 (generate_urand) bit for bit: the
// SplitMix64 stream derived from (seed, n, p) is counter-based (draw k =
// mix64(s + k*gamma), hm/rng.py:84-89), so every matrix element computes
// its own draws.  Coordinates are draws 1..2n (x0 y0 x1 y1 ...) times
// COORD_RANGE; flows are draws 2n+1.. row-major mapped to int(u * 101),
// diagonal zeroed; distances are numpy's separate sub / mul / add / sqrt
// (hm/io.py:143-147), hence the explicit round-to-nearest intrinsics (no FMA
// contraction).
//
// k_unrank_combos writes hub sets rank0 .. rank0+B-1 of the lexicographic
// enumeration of p-subsets of [0, n) -- itertools.combinations order, the
// order restricted_optimum sweeps (hm/oracle.py:42-54).  k_argmin_raw keeps
// the first strict minimum of raw over that order: min by (raw, rank).

#include "hg_internal.cuh"

namespace hg {

namespace {

constexpr double kCoordRange = 100000.0;  // hm/io.py:39
constexpr double kFlowBound = 101.0;      // FLOW_RANGE + 1, hm/io.py:40, :205

__device__ __forceinline__ double uniform_at(uint64_t s, uint64_t k) {
    // (x >> 11) * 2^-53 (hm/rng.py:91-93): exact
    return (double)(sm_draw(s, k) >> 11) * 0x1p-53;
}

__global__ void k_gen_coords(uint64_t s, int n, double* __restrict__ xy) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 2 * n; t += gridDim.x * blockDim.x)
        xy[t] = __dmul_rn(uniform_at(s, (uint64_t)t + 1), kCoordRange);
}

__global__ void k_gen_matrices(uint64_t s, int n, const double* __restrict__ xy,
                               double* __restrict__ C, double* __restrict__ W) {
    const int64_t total = (int64_t)n * n;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(x / n), j = (int)(x - (int64_t)i * n);
        if (C) {
            const double dx = __dsub_rn(xy[2 * i], xy[2 * j]);
            const double dy = __dsub_rn(xy[2 * i + 1], xy[2 * j + 1]);
            C[x] = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
        }
        if (W) {
            const double u = uniform_at(s, (uint64_t)(2 * (int64_t)n) + (uint64_t)x + 1);
            W[x] = i == j ? 0.0 : (double)(int64_t)__dmul_rn(u, kFlowBound);
        }
    }
}

// binomial table: binom[a * (p + 1) + b] = C(a, b) for a <= n, b <= p
// (saturated at 2^62; only entries below the enumeration count are used)
__device__ __forceinline__ uint64_t binom_at(const uint64_t* bt, int p, int a, int b) {
    return (a < 0 || b < 0) ? 0 : bt[a * (p + 1) + b];
}

__global__ void k_unrank_combos(const uint64_t* __restrict__ bt, int n, int p, uint64_t rank0,
                                int64_t B, uint64_t count, int32_t* __restrict__ hubs) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint64_t r = rank0 + (uint64_t)b;
        if (r >= count) r = count - 1;  // batch tail: repeat the last set (never a new minimum)
        int x = 0;
        for (int i = 0; i < p; ++i) {
            // first element x at position i with r < #combinations starting at x
            for (;; ++x) {
                const uint64_t c = binom_at(bt, p, n - 1 - x, p - 1 - i);
                if (r < c) break;
                r -= c;
            }
            hubs[b * p + i] = x;
            ++x;
        }
    }
}

// one CTA: the batch's first strict minimum of raw (out[b][3]) in rank
// order, then merged into the running best of the earlier (lower-rank)
// batches with a strict '<' -- itertools order, hm/oracle.py:49-53
constexpr int kArgThreads = 1024;

__global__ void __launch_bounds__(kArgThreads)
k_batch_best(const double* __restrict__ out, int64_t B, uint64_t rank0, uint64_t count,
             double* __restrict__ best_raw, unsigned long long* __restrict__ best_rank) {
    __shared__ double sv[kArgThreads];
    __shared__ unsigned long long sr[kArgThreads];
    double v = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    unsigned long long r = ~0ull;
    for (int64_t b = threadIdx.x; b < B; b += kArgThreads) {
        const uint64_t rk = rank0 + (uint64_t)b;
        if (rk >= count) break;
        const double x = out[b * 4 + 3];
        if (x < v) {  // ascending ranks per thread: strict '<' keeps the first
            v = x;
            r = rk;
        }
    }
    sv[threadIdx.x] = v;
    sr[threadIdx.x] = r;
    __syncthreads();
    for (int o = kArgThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            const double x = sv[threadIdx.x + o];
            const unsigned long long rk = sr[threadIdx.x + o];
            if (x < sv[threadIdx.x] || (x == sv[threadIdx.x] && rk < sr[threadIdx.x])) {
                sv[threadIdx.x] = x;
                sr[threadIdx.x] = rk;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && sr[0] != ~0ull && (*best_rank == ~0ull || sv[0] < *best_raw)) {
        *best_raw = sv[0];
        *best_rank = sr[0];
    }
}

}  // namespace

int launch_gen_urand(uint64_t s, int n, double* xy, double* C, double* W, cudaStream_t st) {
    k_gen_coords<<<(2 * n + 255) / 256, 256, 0, st>>>(s, n, xy);
    HG_LAUNCHED();
    const int64_t total = (int64_t)n * n;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    k_gen_matrices<<<(unsigned)blocks, 256, 0, st>>>(s, n, xy, C, W);
    HG_LAUNCHED();
    return HG_OK;
}

int launch_unrank_combos(const uint64_t* binom, int n, int p, uint64_t rank0, int64_t B,
                         uint64_t count, int32_t* hubs, cudaStream_t st) {
    int64_t blocks = (B + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_unrank_combos<<<(unsigned)blocks, 256, 0, st>>>(binom, n, p, rank0, B, count, hubs);
    HG_LAUNCHED();
    return HG_OK;
}

int launch_batch_best(const double* out, int64_t B, uint64_t rank0, uint64_t count,
                      double* best_raw, unsigned long long* best_rank, cudaStream_t st) {
    k_batch_best<<<1, kArgThreads, 0, st>>>(out, B, rank0, count, best_raw, best_rank);
    HG_LAUNCHED();
    return HG_OK;
}

}  // namespace hg
