// K2 (nearest-hub allocation + spoke legs + hub-cost tables) and K3 (population
// fitness: sum_ij W_ij T_b[c_b(i)][c_b(j)]) for sm_100a.
//
// Reference: allocate_to_nearest (hm/model.py:202-207) and _components
// (hm/evaluation.py:103-120).  The transfer term is evaluated in its gather
// form S_T = sum_ij W_ij C[a_i][a_j] (the reference's own batched screen uses
// the same formulation, hm/oracle.py:126-127); it equals sum_kl F_kl C[h_k][h_l]
// up to fp64 summation order.

#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include <cstdlib>

#include <type_traits>

#include "hg_internal.cuh"

namespace hg {

// ----------------------------------------------------------------------------
// small utilities
// ----------------------------------------------------------------------------

__global__ void k_i32_to_i64(const int32_t* __restrict__ s, int64_t* __restrict__ d, int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        d[i] = s[i];
}

static int grid_for(int64_t m, int block) {
    int64_t g = ceil_div(m, block);
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return (int)g;
}

// hub sets in (int64, B x p) -> int32, validated: each row strictly increasing
// within [0, n).  *err (0 = ok) records the FIRST bad row as 0x7ffffffe - row
// via atomicMax; K2 then treats the whole batch as hubs 0..p-1 (stays in bounds);
// row0 offsets the row numbers of a batch queued in chunks
__global__ void k_hubs_in(const int64_t* __restrict__ s, int32_t* __restrict__ d, int64_t B,
                          int p, int n, int* err, int64_t row0) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < B * p;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = row0 + x / p;
        const int k = (int)(x - (b - row0) * p);
        const int64_t v = s[x];
        bool ok = v >= 0 && v < n;
        if (k > 0) ok = ok && s[x - 1] < v;
        if (!ok) atomicMax(err, (int)(0x7ffffffe - (b < 0x7ffffffe ? b : 0x7ffffffd)));
        // out-of-range entries become 0: kernels that index with the hubs
        // before seeing *err (K3-TC/P's table gather) stay in bounds
        d[x] = v >= 0 && v < n ? (int32_t)v : 0;
    }
}

// indices in [0, n) (allocations); a bad entry records its row like k_hubs_in
__global__ void k_idx_in(const int64_t* __restrict__ s, int32_t* __restrict__ d, int64_t count,
                         int n, int* err) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < count;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = s[x];
        const bool ok = v >= 0 && v < n;
        if (!ok) atomicMax(err, (int)(0x7ffffffe - (x / n < 0x7ffffffe ? x / n : 0x7ffffffd)));
        d[x] = ok ? (int32_t)v : 0;
    }
}

int launch_hubs_in(const int64_t* src, int32_t* dst, int64_t B, int p, int n, int* err,
                   cudaStream_t s, int64_t row0) {
    if (B <= 0) return HG_OK;
    k_hubs_in<<<grid_for(B * p, 256), 256, 0, s>>>(src, dst, B, p, n, err, row0);
    HG_LAUNCHED();
    return HG_OK;
}

int launch_idx_in(const int64_t* src, int32_t* dst, int64_t count, int n, int* err,
                  cudaStream_t s) {
    if (count <= 0) return HG_OK;
    k_idx_in<<<grid_for(count, 256), 256, 0, s>>>(src, dst, count, n, err);
    HG_LAUNCHED();
    return HG_OK;
}

int launch_i32_to_i64(const int32_t* src, int64_t* dst, int64_t count, cudaStream_t s) {
    if (count <= 0) return HG_OK;
    k_i32_to_i64<<<grid_for(count, 256), 256, 0, s>>>(src, dst, count);
    HG_LAUNCHED();
    return HG_OK;
}

// 32x32 smem-tiled transpose (padding column against bank conflicts)
__global__ void k_transpose(const double* __restrict__ a, double* __restrict__ t, int n) {
    __shared__ double tile[32][33];
    int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int i = by + r, j = bx + threadIdx.x;
        if (i < n && j < n) tile[r][threadIdx.x] = a[(size_t)i * n + j];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int i = bx + r, j = by + threadIdx.x;
        if (i < n && j < n) t[(size_t)i * n + j] = tile[threadIdx.x][r];
    }
}

int launch_transpose(const double* src, double* dst, int n, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
    k_transpose<<<grid, dim3(32, 8), 0, s>>>(src, dst, n);
    HG_LAUNCHED();
    return HG_OK;
}

__global__ void k_check_symmetric(const double* __restrict__ C, int n, int* flag) {
    int64_t total = (int64_t)n * n;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(x / n), j = (int)(x % n);
        if (j > i && C[x] != C[(size_t)j * n + i]) *flag = 0;
    }
}

// monotone 16-bit quantisation (x - cmin) * scale, floored and clamped: both
// IEEE operations are monotone non-decreasing, so q(a) < q(b) => a < b
__global__ void k_quantize(const double* __restrict__ Ct, uint16_t* __restrict__ Cq, int n, int nq,
                           double cmin, double scale) {
    const int64_t m = (int64_t)n * nq;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = x / nq;
        const int i = (int)(x - h * nq);
        if (i >= n) {
            Cq[x] = 0xFFFFu;  // row padding (never a minimum: masked by the readers)
            continue;
        }
        double v = floor((Ct[h * n + i] - cmin) * scale);
        v = v < 0.0 ? 0.0 : (v > 65535.0 ? 65535.0 : v);
        Cq[x] = (uint16_t)v;
    }
}

int launch_quantize(const double* Ct, uint16_t* Cq, int n, int nq, double cmin, double scale,
                    cudaStream_t s) {
    k_quantize<<<grid_for((int64_t)n * nq, 256), 256, 0, s>>>(Ct, Cq, n, nq, cmin, scale);
    HG_LAUNCHED();
    return HG_OK;
}

int launch_check_symmetric(const double* C, int n, int* flag, cudaStream_t s) {
    k_check_symmetric<<<grid_for((int64_t)n * n, 256), 256, 0, s>>>(C, n, flag);
    HG_LAUNCHED();
    return HG_OK;
}

// ----------------------------------------------------------------------------
// block reduction of two doubles in a fixed order (deterministic)
// ----------------------------------------------------------------------------

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ----------------------------------------------------------------------------
// K2 -- nearest-hub allocation (hm/model.py:202-207)
//   one WARP per individual; the argmin over the p hubs reads the 16-bit
//   quantised rows Cq[h][i] (coalesced in i), keeps the first (lowest-index)
//   minimum, and a hub node is its own hub.
//   Emits the cluster ids, the per-individual hub-cost table T and the two
//   spoke-leg sums.
// ----------------------------------------------------------------------------

constexpr int kPwRingSz = 2 * 8 * 33;  // doubles per warp: 2 streams x 8 columns x 33

// leg-sum modes: kLegsNone (allocation only), kLegsFast (a fixed-order fma
// sum per lane + butterfly: deterministic, within an ulp or so of numpy),
// kLegsExact (numpy's pairwise order, bit-identical to the reference)
constexpr int kLegsNone = 0, kLegsFast = 1, kLegsExact = 2;
template <int LM> struct K2 {
    static constexpr int threads = 256, warps = threads / 32;
    static constexpr int ring = LM == kLegsExact ? kPwRingSz : 1;
    static constexpr int stack = LM == kLegsExact ? 2 * kPwStack : 1;
};

// WARP per individual, no block barriers: the warp sweeps its individual's
// nodes in chunks of 128.  Two argmin front ends (below) feed one epilogue in
// the STRIDED layout -- lane L owns nodes c0 + 32t + L, t = 0..3 -- where
// the fp64 gathers of each node's cost to its hub touch ~2 lines per hub row
// per instruction (32 consecutive nodes), the O / D weight loads are
// coalesced, and the fp64 leg sums accumulate in one fixed order whichever
// front end ran: the two kernels' outputs are bit-identical.
// A quantised tie (two hubs at the minimal 16-bit cost q) is resolved on the
// fp64 costs: the first minimum (hm/model.py:205), and a hub node is its own
// hub (hm/model.py:206; its own q is 0 = cmin, so a competing hub at q = 0
// sends it down this path).  Quantised rows are padded to npad with 0xFFFF.

__device__ __forceinline__ void min2(unsigned& m1, unsigned& m2, unsigned key) {
    m2 = min(m2, max(m1, key));
    m1 = min(m1, key);
}

// one 128-node chunk in the strided layout: kk[t] = hub slot of node
// c0 + 32t + lane when tie[t] is false; tie[t] = quantised tie
// numpy's pairwise sum (pairwise_sum_DOUBLE: leaves of <= 128 terms, 8
// strided accumulators per leaf combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
// the last leaf's partial row added in order, leaves summed up the halving
// tree) replayed per warp, so a device sum is bit-identical to np.sum of the
// same rounded products.  A chunk's terms are staged in a ring of 32 rows x
// 8 columns per stream (2 chunks: a leaf of <= 16 rows ends in the chunk
// just staged and started in it or the one before); when a leaf is complete
// lanes 0-7 run its 8 column accumulators for stream 0 (collection), lanes
// 8-15 for stream 1 (distribution), and lanes 0 / 8 sum the leaves on a
// stack.  Column stride 33 doubles: the 16 chain lanes read 16 distinct bank
// pairs.
constexpr int kPwCol = 33;
static_assert(kPwRingSz == 2 * 8 * kPwCol, "ring size");

struct PwState {
    int leaf;    // next leaf to sum
    uint32_t e;  // its table word (prefetched)
    int depth;   // tree stack depth (warp-uniform)
};

__device__ __forceinline__ void pw_init(PwState& S, const uint32_t* __restrict__ tab,
                                        double* ring, int lane) {
    S.leaf = 0;
    S.e = __ldg(tab);
    S.depth = 0;
    if (lane < 16) ring[(lane >> 3) * 8 * kPwCol + (lane & 7) * kPwCol + 32] = 0.0;  // zero slots
    __syncwarp();
}

// every leaf whose rows are all staged (rows < row_end) is summed.  The 8
// column accumulators run branch-free over 16 rows: rows past the leaf add
// +0.0, which leaves a sum of non-negative terms unchanged bit for bit.
__device__ __forceinline__ void pw_leaves_upto(const uint32_t* __restrict__ tab, int nleaf,
                                               int nterms, int row_end, PwState& S,
                                               const double* ring, double* st, int lane) {
    const int s = lane < 8 ? 0 : 1, j = lane & 7;
    const double* col = ring + s * 8 * kPwCol + j * kPwCol;
    double* stk = st + s * kPwStack;
    const bool top = (lane & 7) == 0 && lane < 16;
    const int R = nterms >> 3, tail = nterms & 7;
    while (S.leaf < nleaf) {
        const uint32_t e = S.e;
        const int r0 = (int)(e & 0xffffu), nr = (int)((e >> 16) & 0xffu);
        const bool last = S.leaf == nleaf - 1;
        if ((last && tail ? R + 1 : r0 + nr) > row_end) break;
        if (!last) S.e = __ldg(tab + S.leaf + 1);
        // rows past the leaf read slot 32 of the column, kept at +0.0 (adding
        // it leaves a sum of non-negative terms unchanged bit for bit)
        const int s0 = r0 & 31;
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = col[q < nr ? (s0 + q) & 31 : 32];
        double acc = v[0];
#pragma unroll
        for (int q = 1; q < 16; ++q) acc = acc + v[q];
        acc = acc + __shfl_xor_sync(0xffffffffu, acc, 1);
        acc = acc + __shfl_xor_sync(0xffffffffu, acc, 2);
        acc = acc + __shfl_xor_sync(0xffffffffu, acc, 4);
        if (top) {
            if (last)  // the partial row, term by term
                for (int u = 0; u < tail; ++u)
                    acc = acc + ring[s * 8 * kPwCol + u * kPwCol + (R & 31)];
            stk[S.depth] = acc;
        }
        ++S.depth;
        for (int c = last ? S.depth - 1 : (int)(e >> 24); c > 0; --c, --S.depth)
            if (top) stk[S.depth - 2] = stk[S.depth - 2] + stk[S.depth - 1];
        ++S.leaf;
    }
}

template <int LM>
__device__ __forceinline__ void alloc_chunk_out(const DevInst& I, const int32_t* hs, int64_t b,
                                                int c0, int lane, const int (&kk)[4],
                                                const bool (&tie)[4], double& so, double& sd,
                                                PwState& S, double* ring,
                                                double* st, uint8_t* __restrict__ cl,
                                                uint16_t* __restrict__ co,
                                                int32_t* __restrict__ alloc) {
    const int n = I.n, p = I.p, nq = I.nq;
    double best[4], ow[4], dw[4];
    int c4[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {  // all loads first
        const int i = c0 + 32 * t + lane;
        const bool in = i < n;
        c4[t] = tie[t] ? 0 : kk[t];
        if (LM != kLegsNone) {
            best[t] = in ? I.Ct[(size_t)hs[c4[t]] * n + i] : 0.0;
            ow[t] = in ? I.O[i] : 0.0;
            dw[t] = in ? I.D[i] : 0.0;
        } else {
            best[t] = 0.0;
        }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int i = c0 + 32 * t + lane;
        if (i < n && tie[t]) {
            unsigned qmin = 0xFFFFu;
            for (int k2 = 0; k2 < p; ++k2)
                qmin = min(qmin, (unsigned)I.Cq[(size_t)hs[k2] * nq + i]);
            int kf = -1;
            for (int k2 = 0; k2 < p; ++k2) {
                const int h = hs[k2];
                if (I.Cq[(size_t)h * nq + i] != qmin) continue;
                if (kf < 0) {  // the first hub at qmin
                    kf = k2;
                    best[t] = I.Ct[(size_t)h * n + i];
                    if (h == i) break;
                    continue;
                }
                if (h == i) {
                    best[t] = 0.0;
                    kf = k2;
                    break;
                }
                const double d = I.Ct[(size_t)h * n + i];
                if (d < best[t]) {
                    best[t] = d;
                    kf = k2;
                }
            }
            c4[t] = kf;
        }
        // the reference's terms out_flow * legs, in_flow * legs (rounded
        // products) into the ring: node c0 + 32t + lane = row c0/8 + 4t +
        // lane/8, column lane & 7
        if (LM == kLegsFast) {
            so = fma(ow[t], best[t], so);
            sd = fma(dw[t], best[t], sd);
        }
        if (LM == kLegsExact && c0 < n) {
            // (c0/8) % 32 is 0 or 16: no wrap inside a chunk
            const int at = (lane & 7) * kPwCol + ((c0 >> 3) & 31) + 4 * t + (lane >> 3);
            ring[at] = __dmul_rn(ow[t], best[t]);
            ring[8 * kPwCol + at] = __dmul_rn(dw[t], best[t]);
        }
        if (i >= n) c4[t] = 0;
    }
    if (LM == kLegsExact && c0 < n) {
        __syncwarp();
        pw_leaves_upto(I.pwnl, I.npwnl, n, (c0 >> 3) + 16, S, ring, st, lane);
        __syncwarp();  // the ring slot is rewritten two chunks on
    }
    uint8_t* clb = cl + b * I.npad + c0 + lane;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        HG_DCHECK(c4[t] >= 0 && c4[t] < p, "K2 cluster %d of node %d outside [0, %d)", c4[t],
                  c0 + 32 * t + lane, p);
        HG_DCHECK(c0 + 32 * t + lane < I.npad, "K2 node %d past npad %d", c0 + 32 * t + lane,
                  I.npad);
        clb[32 * t] = (uint8_t)c4[t];
    }
    if (co)  // byte offsets of the columns in a T plane row (fp64 K3 only)
#pragma unroll
        for (int t = 0; t < 4; ++t) co[b * I.npad + c0 + 32 * t + lane] = (uint16_t)(c4[t] * 4);
    if (alloc)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int i = c0 + 32 * t + lane;
            if (i < n) alloc[b * n + i] = hs[c4[t]];
        }
}

// the end of one individual in K2 (warp-wide): hub-to-hub cost table T_b
// (lane = column, 8 rows per round: the 8 scattered L2 gathers are in flight
// together, not 8 round trips) and the two leg sums in a fixed order
template <int LM>
__device__ __forceinline__ void alloc_finish(const DevInst& I, const int32_t* hs, int64_t b,
                                             int lane, double so, double sd, const double* st,
                                             uint32_t* __restrict__ T, double* __restrict__ legs) {
    const int p = I.p, n = I.n;
    uint32_t* Tb = T ? T + b * 2 * (int64_t)p * I.ps : nullptr;
    for (int k0 = 0; T && k0 < p; k0 += 8) {  // T null: the fitness kernel gathers it
        for (int l = lane; l < p; l += 32) {
            const int hl = hs[l];
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = k0 + u < p ? __ldg(I.C + (size_t)hs[k0 + u] * n + hl) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < p) {
                    Tb[(k0 + u) * I.ps + l] = (uint32_t)__double2hiint(v[u]);
                    Tb[(p + k0 + u) * I.ps + l] = (uint32_t)__double2loint(v[u]);
                }
        }
    }
    if (LM == kLegsFast) {
        so = warp_sum(so);  // fixed butterfly order: deterministic
        sd = warp_sum(sd);
    }
    if (LM != kLegsNone && lane == 0) {
        legs[2 * b] = LM == kLegsExact ? st[0] : so;
        legs[2 * b + 1] = LM == kLegsExact ? st[kPwStack] : sd;
    }
}

// K2 scalar front end (any p <= 255): lane owns the 4 consecutive nodes
// c0+4*lane..+3, one 8-byte load of quantised costs per hub row.  Per node
// and hub the argmin is 4 integer ops: key = (q << 8) | k by one byte
// permute, then the two smallest keys (m1, m2) by min/max; m1's low byte is
// the first hub at the minimal q, and m2 at the same q is a tie.  The
// a warp's hub set into hs[0, p): the int32 batch, or (I.hubs64) the
// caller's int64 row read and validated here -- the fused k_hubs_in: a bad
// row records itself in *err (the first bad row wins) and runs on hubs 0..p-1
// so that every later index stays in bounds; each entry goes to I.hubs_w as
// k_hubs_in writes it (out of range -> 0) for K3
__device__ __forceinline__ void k2_load_hubs(const DevInst& I, const int32_t* __restrict__ hubs,
                                             int64_t b, int lane, int32_t* hs) {
    const int p = I.p, n = I.n;
    if (!I.hubs64) {
        const bool bad = I.err != nullptr && *I.err != 0;  // rejected input: stay in bounds
        for (int k = lane; k < p; k += 32) hs[k] = bad ? k : hubs[b * p + k];
        return;
    }
    const int64_t* row = I.hubs64 + b * p;
    bool rowbad = false;
    for (int k0 = 0; k0 < p; k0 += 32) {
        const int k = k0 + lane;
        const int64_t v = k < p ? row[k] : 0;
        int64_t prev = __shfl_up_sync(0xffffffffu, v, 1);
        if (lane == 0 && k0 > 0) prev = row[k0 - 1];
        const bool inr = v >= 0 && v < n;
        const bool ok = k >= p || (inr && (k == 0 || prev < v));
        rowbad |= __any_sync(0xffffffffu, !ok);
        if (k < p) I.hubs_w[b * p + k] = inr ? (int32_t)v : 0;
        if (k < p) hs[k] = (int32_t)v;
    }
    if (rowbad) {
        for (int k = lane; k < p; k += 32) hs[k] = k;
        if (lane == 0) {
            const int64_t r = I.hrow0 + b;
            atomicMax(const_cast<int*>(I.err), (int)(0x7ffffffe - (r < 0x7ffffffe ? r : 0x7ffffffd)));
        }
    }
}

// per-node (slot, tie) codes move to the strided layout by 8 shuffles.
template <int LM>
__global__ void __launch_bounds__(K2<LM>::threads)
k_allocate(DevInst I, int64_t B, const int32_t* __restrict__ hubs, uint8_t* __restrict__ cl,
           uint16_t* __restrict__ co, uint32_t* __restrict__ T, double* __restrict__ legs,
           int32_t* __restrict__ alloc) {
    __shared__ int32_t hs_all[K2<LM>::warps][kMaxP + 1];
    __shared__ double pwring[K2<LM>::warps][K2<LM>::ring];   // staged terms (2 streams)
    __shared__ double pwst[K2<LM>::warps][K2<LM>::stack];   // the two tree stacks
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * K2<LM>::warps + warp;
    if (b >= B || (I.dynB && b >= *I.dynB)) return;
    const int p = I.p, nq = I.nq;
    int32_t* hs = hs_all[warp];
    double* ring = pwring[warp];
    double* st = pwst[warp];
    // the fitness kernel (launched programmatically dependent) may start its
    // own set-up now; it waits for this grid before reading what it writes
    asm volatile("griddepcontrol.launch_dependents;");
    k2_load_hubs(I, hubs, b, lane, hs);
    __syncwarp();

    PwState S;
    if (LM == kLegsExact) pw_init(S, I.pwnl, ring, lane);
    double so = 0.0, sd = 0.0;
    for (int c0 = 0; c0 < I.npad; c0 += 128) {
        const int i0 = c0 + 4 * lane;
        unsigned m1[4], m2[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) m1[t] = m2[t] = 0xFFFFFFFFu;
        const uint16_t* col = I.Cq + i0;
        const int p4 = p & ~3;
        int k = 0;
        if (p4) {
            // software pipelined: the next 4 hub rows are in flight while the
            // current 4 are reduced
            uint2 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                v[u] = __ldg(reinterpret_cast<const uint2*>(col + (size_t)hs[u] * nq));
            for (; k < p4; k += 4) {
                uint2 w[4];
                const int kn = k + 4 < p4 ? k + 4 : k;  // last round: harmless reload
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    w[u] = __ldg(reinterpret_cast<const uint2*>(col + (size_t)hs[kn + u] * nq));
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const unsigned kk = (unsigned)(k + u);
                    min2(m1[0], m2[0], __byte_perm(v[u].x, kk, 0x5104));
                    min2(m1[1], m2[1], __byte_perm(v[u].x, kk, 0x5324));
                    min2(m1[2], m2[2], __byte_perm(v[u].y, kk, 0x5104));
                    min2(m1[3], m2[3], __byte_perm(v[u].y, kk, 0x5324));
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = w[u];
            }
        }
        for (; k < p; ++k) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(col + (size_t)hs[k] * nq));
            const unsigned kk = (unsigned)k;
            min2(m1[0], m2[0], __byte_perm(v.x, kk, 0x5104));
            min2(m1[1], m2[1], __byte_perm(v.x, kk, 0x5324));
            min2(m1[2], m2[2], __byte_perm(v.y, kk, 0x5104));
            min2(m1[3], m2[3], __byte_perm(v.y, kk, 0x5324));
        }
        // code per node: slot | tie << 8, two nodes per word
        unsigned cw[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            unsigned c[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int t = 2 * h + u;
                c[u] = (m1[t] & 0xffu) | ((m2[t] >> 8) == (m1[t] >> 8) ? 0x100u : 0u);
            }
            cw[h] = c[0] | (c[1] << 16);
        }
        // strided node c0 + 32t + lane = consecutive lane 8t + lane/4, slot lane&3
        int kk[4];
        bool tie[4];
        const int half = (lane >> 1) & 1, sh = (lane & 1) * 16;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int src = 8 * t + (lane >> 2);
            const unsigned x0 = __shfl_sync(0xffffffffu, cw[0], src);
            const unsigned x1 = __shfl_sync(0xffffffffu, cw[1], src);
            const unsigned c = ((half ? x1 : x0) >> sh) & 0xffffu;
            kk[t] = (int)(c & 0xffu);
            tie[t] = (c >> 8) != 0;
        }
        alloc_chunk_out<LM>(I, hs, b, c0, lane, kk, tie, so, sd, S, ring, st, cl, co, alloc);
    }
    alloc_finish<LM>(I, hs, b, lane, so, sd, st, T, legs);
}

// K2 register front end for p <= 32 (the hub rows of a pass in registers).
// Lane = 2 consecutive nodes of a 64-node pass, one u32 load of quantised
// costs per hub row (slots p..PM-1 read the all-0xFFFF row n).  qmin of both
// nodes by 16x2 SIMD min (VIMNMX3.U16x2); then per hub
// t = min_u16x2(v - qmin, 1) -- 0 exactly where the hub is at qmin, and
// v >= qmin so the 32-bit subtraction never borrows across halves -- and
// acc += t * (256 + k).  With S = sum_k (256 + k) (< 2^16 for PM <= 32),
// S - acc per half = sum over the hubs at qmin of (256 + k): the count in the
// high byte, the hub slot in the low byte when the count is 1 (a count above
// 1 is a quantised tie).  4 shuffles move the codes to the strided layout.
template <int PM, int LM>
__global__ void __launch_bounds__(K2<LM>::threads, 4)
k_allocate_r(DevInst I, int64_t B, const int32_t* __restrict__ hubs, uint8_t* __restrict__ cl,
             uint16_t* __restrict__ co, uint32_t* __restrict__ T, double* __restrict__ legs,
             int32_t* __restrict__ alloc) {
    static_assert(PM % 4 == 0 && PM <= 32, "hub slots");
    __shared__ int32_t hs_all[K2<LM>::warps][32];
    __shared__ uint32_t ro_all[K2<LM>::warps][32];  // element offset of hub slot k's row in Cq
    __shared__ double pwring[K2<LM>::warps][K2<LM>::ring];   // staged terms (2 streams)
    __shared__ double pwst[K2<LM>::warps][K2<LM>::stack];   // the two tree stacks
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * K2<LM>::warps + warp;
    if (b >= B || (I.dynB && b >= *I.dynB)) return;
    const int n = I.n, p = I.p, nq = I.nq;
    int32_t* hs = hs_all[warp];
    uint32_t* ro = ro_all[warp];
    double* ring = pwring[warp];
    double* st = pwst[warp];
    // the fitness kernel (launched programmatically dependent) may start its
    // own set-up now; it waits for this grid before reading what it writes
    asm volatile("griddepcontrol.launch_dependents;");
    k2_load_hubs(I, hubs, b, lane, hs);
    __syncwarp();
    if (lane < PM) ro[lane] = (uint32_t)(lane < p ? hs[lane] : n) * (uint32_t)nq;
    __syncwarp();
    constexpr unsigned kS = 256u * PM + PM * (PM - 1) / 2;

    PwState S;
    if (LM == kLegsExact) pw_init(S, I.pwnl, ring, lane);
    double so = 0.0, sd = 0.0;
    for (int c0 = 0; c0 < I.npad; c0 += 128) {
        unsigned wv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint16_t* col = I.Cq + c0 + 64 * h + 2 * lane;
            unsigned r[PM];
#pragma unroll
            for (int k = 0; k < PM; ++k)
                r[k] = __ldg(reinterpret_cast<const unsigned*>(col + ro[k]));
            unsigned m = r[0];
#pragma unroll
            for (int k = 1; k < PM; ++k) m = __vminu2(m, r[k]);
            unsigned acc = 0;
#pragma unroll
            for (int k = 0; k < PM; ++k) acc += __vminu2(r[k] - m, 0x00010001u) * (256u + k);
            wv[h] = kS * 0x00010001u - acc;
        }
        // strided node c0 + 32t + lane = pass t/2, lane 16(t&1) + lane/2, half lane&1
        int kk[4];
        bool tie[4];
        const int sh = (lane & 1) * 16;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const unsigned w = __shfl_sync(0xffffffffu, wv[t >> 1], 16 * (t & 1) + (lane >> 1));
            const unsigned v = (w >> sh) & 0xffffu;
            tie[t] = (v >> 8) != 1;
            kk[t] = (int)(v & 0xffu);
        }
        alloc_chunk_out<LM>(I, hs, b, c0, lane, kk, tie, so, sd, S, ring, st, cl, co, alloc);
    }
    alloc_finish<LM>(I, hs, b, lane, so, sd, st, T, legs);
}

int prepare_allocate(const DevInst&) { return HG_OK; }

// tuning / A-B override: HUBGPU_K2_SCALAR=1 keeps k_allocate for every p
static bool k2_scalar() {
    static const bool v = [] {
        const char* e = getenv("HUBGPU_K2_SCALAR");
        return e != nullptr && atoi(e) != 0;
    }();
    return v;
}

int launch_allocate(const DevInst& Iin, int64_t B, const int32_t* hubs, uint8_t* cl,
                    uint16_t* co, uint32_t* T, double* legs, int32_t* alloc, cudaStream_t s,
                    const int32_t* dynB) {
    if (B <= 0) return HG_OK;
    DevInst I = Iin;
    I.dynB = dynB;
    // legs == nullptr: the fitness kernel computes the leg sums itself
    // legs == nullptr: allocation only; else the instance's summation mode
    auto go = [&](auto mode) {
        constexpr int L = decltype(mode)::value;
        const unsigned grid = (unsigned)ceil_div(B, K2<L>::warps);
        if (I.p <= 32 && (int64_t)(I.n + 1) * I.nq < (int64_t(1) << 31) && !k2_scalar()) {
            switch ((I.p + 3) & ~3) {
#define HG_K2R(PM)                                                                                 \
    case PM:                                                                                       \
        k_allocate_r<PM, L><<<grid, K2<L>::threads, 0, s>>>(I, B, hubs, cl, co, T, legs, alloc); \
        break;
                HG_K2R(4) HG_K2R(8) HG_K2R(12) HG_K2R(16) HG_K2R(20) HG_K2R(24) HG_K2R(28)
                HG_K2R(32)
#undef HG_K2R
            }
        } else {
            k_allocate<L><<<grid, K2<L>::threads, 0, s>>>(I, B, hubs, cl, co, T, legs, alloc);
        }
    };
    if (!legs)
        go(std::integral_constant<int, kLegsNone>{});
    else if (I.exact)
        go(std::integral_constant<int, kLegsExact>{});
    else
        go(std::integral_constant<int, kLegsFast>{});
    HG_LAUNCHED();
    return HG_OK;
}

// same products for an arbitrary feasible allocation (objective() of any
// Solution, hm/evaluation.py:86-120): cluster = position of alloc[i] in hubs.
// Warp per individual through K2's epilogue (the same leg terms, the same
// pairwise sums, the same T table).
template <int LM>
__global__ void __launch_bounds__(K2<LM>::threads)
k_from_alloc(DevInst I, int64_t B, const int32_t* __restrict__ hubs,
             const int32_t* __restrict__ alloc, uint8_t* __restrict__ cl,
             uint16_t* __restrict__ co, uint32_t* __restrict__ T, double* __restrict__ legs) {
    __shared__ int32_t hs_all[K2<LM>::warps][kMaxP + 1];
    __shared__ double pwring[K2<LM>::warps][K2<LM>::ring];
    __shared__ double pwst[K2<LM>::warps][K2<LM>::stack];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * K2<LM>::warps + warp;
    if (b >= B || (I.dynB && b >= *I.dynB)) return;
    const int n = I.n, p = I.p;
    int32_t* hs = hs_all[warp];
    double* ring = pwring[warp];
    double* st = pwst[warp];
    const bool bad = I.err != nullptr && *I.err != 0;  // rejected input: stay in bounds
    for (int k = lane; k < p; k += 32) hs[k] = bad ? k : hubs[b * p + k];
    __syncwarp();
    PwState S;
    if (LM == kLegsExact) pw_init(S, I.pwnl, ring, lane);
    double so = 0.0, sd = 0.0;
    const bool notie[4] = {false, false, false, false};
    for (int c0 = 0; c0 < I.npad; c0 += 128) {
        int kk[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int i = c0 + 32 * t + lane;
            int c = 0;
            if (i < n) {
                const int a = bad ? hs[0] : alloc[b * n + i];
                int lo = 0, hi = p - 1;  // hubs sorted; a is one of them (validated by caller)
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (hs[mid] < a) lo = mid + 1; else hi = mid;
                }
                c = lo;
            }
            kk[t] = c;
        }
        alloc_chunk_out<LM>(I, hs, b, c0, lane, kk, notie, so, sd, S, ring, st, cl, co, nullptr);
    }
    alloc_finish<LM>(I, hs, b, lane, so, sd, st, T, legs);
}

int launch_from_alloc(const DevInst& I, int64_t B, const int32_t* hubs, const int32_t* alloc,
                      uint8_t* cl, uint16_t* co, uint32_t* T, double* legs, cudaStream_t s) {
    if (B <= 0) return HG_OK;
    auto go = [&](auto mode) {
        constexpr int L = decltype(mode)::value;
        k_from_alloc<L><<<(unsigned)ceil_div(B, K2<L>::warps), K2<L>::threads, 0, s>>>(
            I, B, hubs, alloc, cl, co, T, legs);
    };
    if (!legs)
        go(std::integral_constant<int, kLegsNone>{});
    else if (I.exact)
        go(std::integral_constant<int, kLegsExact>{});
    else
        go(std::integral_constant<int, kLegsFast>{});
    HG_LAUNCHED();
    return HG_OK;
}

// ----------------------------------------------------------------------------
// K3 -- population fitness, transfer term.
//
// A CTA of 16 warps owns a W tile of TR = 16*RW rows x TC = 32*CJ columns held
// in REGISTERS (warp w: rows i0+w*RW.., lane: columns j0+lane*CJ..), and streams
// individuals through it.  Per individual b the pipeline stages into smem
//   Ts[r] = T_b[c_b(i0+r)][.]   (the tile rows' hub-cost rows as hi/lo word
//                                planes, TR x 2 x ps uint32)
//   Cs[0..TC)   = c_b(j0..j0+TC)       (column cluster ids)
// with cp.async (3 stages x G individuals), and every element costs one
// smem gather Ts[r][c_b(j)] + one DFMA.  Per (b, tile) the CTA reduces in a
// fixed order and writes one partial; k_finalize sums the partials of b in a
// fixed order, so results do not depend on batch size, grid or placement.
//
// Work = (tile, group of G individuals) units, ordered chunk-major so the T
// tables of the individuals in flight stay L2-resident; each CTA takes one
// contiguous range of units (balanced to within one unit), reloading its W
// registers only when the tile changes.
// ----------------------------------------------------------------------------

constexpr int kFitWarps = 16;
constexpr int kFitThreads = kFitWarps * 32;
constexpr int kFitStages = 3;
constexpr int kFitMaxG = 8;
// The lo-word plane of the staged hub-cost rows sits at a FIXED byte offset
// from the hi-word plane, so both gathers of an element share one address
// register (LDS [R+UR] and [R+UR+kLoOff]).
constexpr int kLoOff = 96 * 1024;

struct FitArgs {
    DevInst I;
    const uint8_t* cl;
    const uint16_t* co;
    const uint32_t* T;
    double* part;
    int64_t B;
    int tcn, tiles;
    int G;
    int64_t chunk;         // individuals per chunk (multiple of G)
    int64_t full_chunks;   // B / chunk
    int64_t gpc;           // groups per full chunk per tile = chunk / G
    int64_t gl;            // groups per tile in the last (partial) chunk
    int64_t q_full;        // units in the full chunks
    int64_t q_total;
};

struct Unit {
    int tile;
    int64_t b0;
    int cnt;
};

__device__ __forceinline__ Unit decode_unit(const FitArgs& A, int64_t q) {
    Unit u;
    if (q < A.q_full) {
        int64_t per = (int64_t)A.tiles * A.gpc;
        int64_t c = q / per, r = q - c * per;
        u.tile = (int)(r / A.gpc);
        int64_t gq = r - (int64_t)u.tile * A.gpc;
        u.b0 = c * A.chunk + gq * A.G;
        u.cnt = A.G;
    } else {
        int64_t r = q - A.q_full;
        u.tile = (int)(r / A.gl);
        int64_t gq = r - (int64_t)u.tile * A.gl;
        u.b0 = A.full_chunks * A.chunk + gq * A.G;
        int64_t left = A.B - u.b0;
        u.cnt = (int)(left < A.G ? left : A.G);
    }
    return u;
}

__device__ __forceinline__ void cp16(void* dst, const void* src) {
    __pipeline_memcpy_async(dst, src, 16);
}

template <int RW, int CJ>
__device__ __forceinline__ void issue_unit(const FitArgs& A, const Unit& u, uint32_t* Ts,
                                           uint16_t* Cs) {
    constexpr int TR = kFitWarps * RW, TC = 32 * CJ;
    static_assert(TC % 16 == 0, "column tile must be a multiple of 16 bytes");
    const int ps = A.I.ps, p = A.I.p, npad = A.I.npad;
    const int tr = u.tile / A.tcn, tc = u.tile - tr * A.tcn;
    const int i0 = tr * TR, j0 = tc * TC;
    const int rowchunks = ps >> 2;           // 16 B chunks per plane row
    const int tchunks = TR * 2 * rowchunks;  // hi + lo rows
    constexpr int cchunks = TC * 2 / 16;
    const int per = tchunks + cchunks;
    const int total = u.cnt * per;
    for (int x = threadIdx.x; x < total; x += kFitThreads) {
        const int g = x / per, y = x - g * per;
        const int64_t b = u.b0 + g;
        if (y < tchunks) {
            const int r = y / (2 * rowchunks), z = y - r * 2 * rowchunks;
            const int plane = z >= rowchunks, part = z - plane * rowchunks;
            const int cid = A.cl[b * npad + i0 + r];
            const uint32_t* src =
                A.T + (((b * 2 + plane) * p + cid) * (int64_t)ps + part * 4);
            cp16(reinterpret_cast<char*>(Ts + (size_t)(g * TR + r) * ps + part * 4) +
                     plane * kLoOff, src);
        } else {
            const int k = y - tchunks;
            // chunk k (8 columns) belongs to lane k / (CJ/8); store the v-th chunk
            // of every lane contiguously so a warp's LDS.128 is conflict-free
            int slot = k;
            if constexpr (CJ >= 16) slot = (k % (CJ / 8)) * 32 + k / (CJ / 8);
            cp16(Cs + g * TC + slot * 8, A.co + b * npad + j0 + k * 8);
        }
    }
}

// CJ 16-bit column offsets of one lane, packed two per word
template <int CJ>
__device__ __forceinline__ void load_offs(const uint16_t* base, int lane,
                                          uint32_t (&cw)[(CJ + 1) / 2]) {
    const uint16_t* p = base + lane * CJ;
    if constexpr (CJ >= 16) {
#pragma unroll
        for (int v = 0; v < CJ / 8; ++v) {
            const uint4 x = reinterpret_cast<const uint4*>(base)[v * 32 + lane];
            cw[4 * v + 0] = x.x;
            cw[4 * v + 1] = x.y;
            cw[4 * v + 2] = x.z;
            cw[4 * v + 3] = x.w;
        }
    } else if constexpr (CJ == 8) {
        {
            const int v = 0;
            const uint4 x = reinterpret_cast<const uint4*>(p)[v];
            cw[4 * v + 0] = x.x;
            cw[4 * v + 1] = x.y;
            cw[4 * v + 2] = x.z;
            cw[4 * v + 3] = x.w;
        }
    } else if constexpr (CJ == 4) {
        const uint2 x = *reinterpret_cast<const uint2*>(p);
        cw[0] = x.x;
        cw[1] = x.y;
    } else if constexpr (CJ == 2) {
        cw[0] = *reinterpret_cast<const uint32_t*>(p);
    } else {
        cw[0] = *p;
    }
}

template <int RW, int CJ>
__global__ void __launch_bounds__(kFitThreads, 1) k_fitness(FitArgs A) {
    constexpr int TR = kFitWarps * RW, TC = 32 * CJ;
    extern __shared__ __align__(16) unsigned char smem[];
    const int ps = A.I.ps, n = A.I.n;
    const int G = A.G;
    const size_t ts_stage = (size_t)G * TR * ps;  // uint32 words per plane
    uint32_t* Ts0 = reinterpret_cast<uint32_t*>(smem);  // hi plane; lo plane at +kLoOff
    uint16_t* Cs0 = reinterpret_cast<uint16_t*>(smem + 2 * kLoOff);
    double* red = reinterpret_cast<double*>(Cs0 + kFitStages * G * TC + 8);  // [2][G][16]
    red = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(red) + 15) & ~uintptr_t(15));

    const int lane = threadIdx.x & 31;
    // warp index made provably warp-uniform so row bases live in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int64_t q0 = A.q_total * blockIdx.x / gridDim.x;
    const int64_t q1 = A.q_total * (blockIdx.x + 1) / gridDim.x;
    if (q0 >= q1) return;

    // prologue
#pragma unroll
    for (int s = 0; s < kFitStages - 1; ++s) {
        if (q0 + s < q1) {
            Unit u = decode_unit(A, q0 + s);
            issue_unit<RW, CJ>(A, u, Ts0 + s * ts_stage, Cs0 + s * G * TC);
        }
        __pipeline_commit();
    }

    double w[RW][CJ];
    int cur_tile = -1;
    Unit prev;
    prev.cnt = 0;
    prev.tile = 0;
    prev.b0 = 0;

    for (int64_t k = 0; q0 + k < q1; ++k) {
        const Unit u = decode_unit(A, q0 + k);
        if (u.tile != cur_tile) {
            cur_tile = u.tile;
            const int tr = u.tile / A.tcn, tc = u.tile - tr * A.tcn;
            const int jb = tc * TC + lane * CJ;
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const int i = tr * TR + warp * RW + r;
#pragma unroll
                for (int q = 0; q < CJ; ++q) {
                    const int j = jb + q;
                    w[r][q] = (i < n && j < n) ? __ldg(A.I.W + (size_t)i * n + j) : 0.0;
                }
            }
        }
        __pipeline_wait_prior(kFitStages - 2);
        __syncthreads();

        // finish the previous unit's reduction (its red buffer is complete)
        if (prev.cnt > 0 && threadIdx.x < prev.cnt) {
            const double* rp = red + ((k - 1) & 1) * kFitMaxG * kFitWarps + threadIdx.x * kFitWarps;
            double s = 0.0;
#pragma unroll
            for (int x = 0; x < kFitWarps; ++x) s += rp[x];
            A.part[(prev.b0 + threadIdx.x) * A.tiles + prev.tile] = s;
        }

        const int st = (int)(k % kFitStages);
        const uint32_t* Ts = Ts0 + st * ts_stage;
        const uint16_t* Cs = Cs0 + st * G * TC;
        double* rk = red + (k & 1) * kFitMaxG * kFitWarps;
        for (int g = 0; g < u.cnt; ++g) {
            uint32_t cw[(CJ + 1) / 2];
            load_offs<CJ>(Cs + g * TC, lane, cw);
            // two independent DFMA chains keep the FP64 pipe fed
            double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const char* Th = reinterpret_cast<const char*>(
                    Ts + (size_t)(g * TR + warp * RW + r) * ps);
                const char* Tl = Th + kLoOff;
#pragma unroll
                for (int q = 0; q < CJ; ++q) {
                    const uint32_t off = (q & 1) ? (cw[q >> 1] >> 16) : (cw[q >> 1] & 0xffffu);
                    const double t = __hiloint2double(*reinterpret_cast<const int*>(Th + off),
                                                      *reinterpret_cast<const int*>(Tl + off));
                    if (q & 1) acc1 = fma(w[r][q], t, acc1);
                    else acc0 = fma(w[r][q], t, acc0);
                }
            }
            double acc = warp_sum(acc0 + acc1);
            if (lane == 0) rk[g * kFitWarps + warp] = acc;
        }
        prev = u;

        // refill the stage consumed in the previous iteration
        const int64_t qn = q0 + k + kFitStages - 1;
        if (qn < q1) {
            const int sn = (int)((k + kFitStages - 1) % kFitStages);
            Unit un = decode_unit(A, qn);
            issue_unit<RW, CJ>(A, un, Ts0 + sn * ts_stage, Cs0 + sn * G * TC);
        }
        __pipeline_commit();
    }
    __syncthreads();
    if (prev.cnt > 0 && threadIdx.x < prev.cnt) {
        const int64_t kl = q1 - q0 - 1;
        const double* rp = red + (kl & 1) * kFitMaxG * kFitWarps + threadIdx.x * kFitWarps;
        double s = 0.0;
#pragma unroll
        for (int x = 0; x < kFitWarps; ++x) s += rp[x];
        A.part[(prev.b0 + threadIdx.x) * A.tiles + prev.tile] = s;
    }
}

// kernel table: (RW, CJ)
using FitKernel = void (*)(FitArgs);
struct FitVariant {
    int rw, cj;
    FitKernel fn;
};
static const FitVariant kVariants[] = {
    {2, 16, k_fitness<2, 16>},  // 32 x 512 tiles: n >= ~400
    {1, 32, k_fitness<1, 32>},  // 16 x 1024
    {1, 16, k_fitness<1, 16>},  // 16 x 512
    {4, 8, k_fitness<4, 8>},    // 64 x 256
    {2, 8, k_fitness<2, 8>},    // 32 x 256
    {2, 4, k_fitness<2, 4>},    // 32 x 128
    {1, 2, k_fitness<1, 2>},    // 16 x 64
    {1, 1, k_fitness<1, 1>},    // 16 x 32: tiny instances
};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

static size_t fit_hi_bytes(int rw, int g, int ps) {
    return kFitStages * (size_t)g * kFitWarps * rw * ps * sizeof(uint32_t);
}

static size_t fit_smem(int rw, int cj, int g, int ps) {
    size_t tc = 32 * cj;
    size_t bytes = 2 * (size_t)kLoOff;
    bytes += kFitStages * (size_t)g * tc * 2 + 16;
    bytes = (bytes + 15) & ~size_t(15);
    bytes += 2 * kFitMaxG * kFitWarps * sizeof(double);
    return bytes;
}

int prepare_fitness(const FitPlan& P) {
    (void)P.smem;  // every variant at the device maximum (instances differ in size)
    return set_max_dynamic_smem(reinterpret_cast<const void*>(kVariants[P.variant].fn));
}

FitPlan fitness_plan(const DevInst& I, int sm_count) {
    (void)sm_count;
    // pick the variant with the least (padded area x measured per-element cost);
    // per-element costs relative to (2,16), measured on B200 at n=1000 with
    // p=20 and p=50 (tools/sweep_variants.sh, profiles/ROUND1.md)
    static const double kCostSmallP[] = {1.00, 1.13, 1.30, 1.31, 1.40, 2.35, 7.0, 13.1};
    static const double kCostLargeP[] = {1.14, 1.00, 1.17, 1.60, 1.69, 2.9, 6.0, 11.3};
    static_assert(sizeof(kCostSmallP) / sizeof(double) == kNumVariants, "cost table");
    int best = 0;
    double best_cost = 1e300;
    for (int v = 0; v < kNumVariants; ++v) {
        const int tr = kFitWarps * kVariants[v].rw, tc = 32 * kVariants[v].cj;
        const double area = (double)round_up(I.n, tr) * (double)round_up(I.n, tc);
        const double cost = area * (I.p > 32 ? kCostLargeP[v] : kCostSmallP[v]);
        if (cost < best_cost) {
            best_cost = cost;
            best = v;
        }
    }
    if (const char* ov = getenv("HUBGPU_FIT_VARIANT")) {  // tuning override
        const int v = atoi(ov);
        if (v >= 0 && v < kNumVariants) best = v;
    }
    FitPlan P{};
    P.variant = best;
    P.rw = kVariants[best].rw;
    P.cj = kVariants[best].cj;
    P.tr = kFitWarps * P.rw;
    P.tc = 32 * P.cj;
    P.g = kFitMaxG;
    while (P.g > 1 && (fit_hi_bytes(P.rw, P.g, I.ps) > (size_t)kLoOff ||
                       fit_smem(P.rw, P.cj, P.g, I.ps) > 226 * 1024))
        P.g >>= 1;
    P.smem = fit_smem(P.rw, P.cj, P.g, I.ps);
    P.trn = (int)ceil_div(I.n, P.tr);
    P.tcn = (int)(round_up(I.n, P.tc) / P.tc);
    P.tiles = P.trn * P.tcn;
    P.blocks_per_sm = 1;
    return P;
}

int launch_fitness(const DevInst& I, const FitPlan& P, int64_t B, const uint8_t* cl,
                   const uint16_t* co, const uint32_t* T, double* part, int grid, cudaStream_t s) {
    if (B <= 0) return HG_OK;
    FitArgs A;
    A.I = I;
    A.cl = cl;
    A.co = co;
    A.T = T;
    A.part = part;
    A.B = B;
    A.tcn = P.tcn;
    A.tiles = P.tiles;
    A.G = P.g;
    // keep the T tables + cluster rows of one chunk within ~48 MB of L2
    const double per_ind = (double)I.p * I.ps * 8.0 + 3.0 * I.npad;  // 2 planes x 4 B
    int64_t chunk = (int64_t)(48.0 * 1024 * 1024 / per_ind);
    chunk = chunk / P.g * P.g;
    if (chunk < P.g) chunk = P.g;
    if (chunk > round_up(B, P.g)) chunk = round_up(B, P.g);
    A.chunk = chunk;
    A.full_chunks = B / chunk;
    A.gpc = chunk / P.g;
    const int64_t rem = B - A.full_chunks * chunk;
    A.gl = ceil_div(rem, P.g);
    A.q_full = A.full_chunks * (int64_t)P.tiles * A.gpc;
    A.q_total = A.q_full + (int64_t)P.tiles * A.gl;
    int g = grid;
    if (g > A.q_total) g = (int)A.q_total;
    FitKernel fn = kVariants[P.variant].fn;
    fn<<<g, kFitThreads, P.smem, s>>>(A);
    HG_LAUNCHED();
    return HG_OK;
}

// ----------------------------------------------------------------------------
// finalise: S_T(b) = sum over tiles in a fixed order; raw = (coll + tran) + dist
// (hm/evaluation.py:93, 110-119).  One warp per individual.
// ----------------------------------------------------------------------------

__global__ void k_finalize(DevInst I, int64_t B, int tiles, const double* __restrict__ legs,
                           const double* __restrict__ part, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (b >= B) return;
    double s = 0.0;
    for (int t = lane; t < tiles; t += 32) s += part[b * tiles + t];
    s = warp_sum(s);
    if (lane == 0) {
        const double coll = I.chi * legs[2 * b];
        const double dist = I.delta * legs[2 * b + 1];
        const double tran = I.alpha * s;
        out[4 * b + 0] = coll;
        out[4 * b + 1] = tran;
        out[4 * b + 2] = dist;
        out[4 * b + 3] = __dadd_rn(__dadd_rn(coll, tran), dist);
    }
}

int launch_finalize(const DevInst& I, int tiles, int64_t B, const double* legs,
                    const double* part, double* out, cudaStream_t s) {
    if (B <= 0) return HG_OK;
    const int threads = 256;
    const int64_t blocks = ceil_div(B * 32, threads);
    k_finalize<<<(unsigned)blocks, threads, 0, s>>>(I, B, tiles, legs, part, out);
    HG_LAUNCHED();
    return HG_OK;
}

}  // namespace hg
