// K4a-c, K5: island-GA operators on bit-packed hub masks, sm_100a.
//
// Reference: _run_island (hm/engine.py:138-167) and the operators
// crossover_hub_arrays / swap_random_hub_spoke / correct_hub_set
// (hm/operators.py:41-124).  Every random draw is replayed by INDEX on the
// counter-based SplitMix64 streams of the reference (hm/rng.py:84-89):
//   population stream: individual m (m >= 1 elitist, m >= 0 strict), swap s
//                      uses draws ctr + 2*((m-e)*strength + s) + {1, 2}
//                      (none when p == n: the swap is the identity);
//   crossover stream:  pair j uses draw ctr + j + 1 (none when n == 1);
//   mutation stream:   child c uses draws ctr + 2*o_c + {1, 2} where o_c counts
//                      the non-degenerate children before c (a child that is
//                      all-open or all-closed consumes nothing).
// so islands, pairs and children are processed in parallel yet consume
// exactly the reference's draw sequence.

#include <cub/block/block_scan.cuh>

#include "hg_internal.cuh"

namespace hg {

constexpr unsigned kFull = 0xffffffffu;

// r-th (0-based) set bit (want_set) or clear bit (!want_set) among [0, n) of
// an nw-word mask in shared memory; uniform across the warp.
__device__ int warp_select(const uint32_t* m, int nw, int n, int r, bool want_set, int lane) {
    int base = 0;
    for (int w0 = 0; w0 < nw; w0 += 32) {
        const int w = w0 + lane;
        uint32_t word = 0;
        if (w < nw) {
            word = m[w];
            if (!want_set) {
                word = ~word;
                if (w == nw - 1 && (n & 31)) word &= (1u << (n & 31)) - 1u;
            }
        }
        const int c = __popc(word);
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += v;
        }
        const int total = __shfl_sync(kFull, inc, 31);
        if (r < base + total) {
            const unsigned hit = __ballot_sync(kFull, r < base + inc);
            const int L = __ffs(hit) - 1;
            const int excl = __shfl_sync(kFull, inc - c, L);
            uint32_t wd = __shfl_sync(kFull, word, L);
            int k = r - base - excl;
            for (int t = 0; t < k; ++t) wd &= wd - 1u;
            return (w0 + L) * 32 + (__ffs(wd) - 1);
        }
        base += total;
    }
    return -1;
}

// ---------------------------------------------------------------------------
// byte masks <-> bit masks
// ---------------------------------------------------------------------------

__global__ void k_bytes_to_bits(const uint8_t* __restrict__ bytes, uint32_t* __restrict__ bits,
                                int64_t B, int n, int nw) {
    const int64_t total = B * nw;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = x / nw;
        const int w = (int)(x - b * nw);
        uint32_t v = 0;
        for (int t = 0; t < 32; ++t) {
            const int i = w * 32 + t;
            if (i < n && bytes[b * n + i]) v |= 1u << t;
        }
        bits[x] = v;
    }
}

__global__ void k_bits_to_bytes(const uint32_t* __restrict__ bits, uint8_t* __restrict__ bytes,
                                int64_t B, int n, int nw) {
    const int64_t total = B * n;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = x / n;
        const int i = (int)(x - b * n);
        bytes[x] = (bits[b * nw + (i >> 5)] >> (i & 31)) & 1u;
    }
}

static int grid_for(int64_t m, int block) {
    int64_t g = ceil_div(m, block);
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return (int)g;
}

int launch_bytes_to_bits(const uint8_t* bytes, uint32_t* bits, int64_t B, int n, int nw,
                         cudaStream_t s) {
    if (B <= 0) return HG_OK;
    k_bytes_to_bits<<<grid_for(B * nw, 256), 256, 0, s>>>(bytes, bits, B, n, nw);
    HG_LAUNCHED();
    return HG_OK;
}

int launch_bits_to_bytes(const uint32_t* bits, uint8_t* bytes, int64_t B, int n, int nw,
                         cudaStream_t s) {
    if (B <= 0) return HG_OK;
    k_bits_to_bytes<<<grid_for(B * n, 256), 256, 0, s>>>(bits, bytes, B, n, nw);
    HG_LAUNCHED();
    return HG_OK;
}

// ---------------------------------------------------------------------------
// K4c -- correction (hm/operators.py:69-101), one CTA per mask.
// ---------------------------------------------------------------------------

constexpr int kCorrThreads = 128;
using CorrScan = cub::BlockScan<int, kCorrThreads>;

// extract the set bits of the smem mask, in order, into H; returns the count
__device__ int block_extract(const uint32_t* mask, int nw, int32_t* H,
                             typename CorrScan::TempStorage& tmp, int* bcast) {
    int base = 0;
    for (int w0 = 0; w0 < nw; w0 += kCorrThreads) {
        const int w = w0 + threadIdx.x;
        const uint32_t word = w < nw ? mask[w] : 0u;
        int off, total;
        CorrScan(tmp).ExclusiveSum(__popc(word), off, total);
        uint32_t v = word;
        int k = base + off;
        while (v) {
            H[k++] = w * 32 + (__ffs(v) - 1);
            v &= v - 1u;
        }
        base += total;
        __syncthreads();
    }
    (void)bcast;
    return base;
}

// exact integer load += w (w integer-valued, totals < 2^53) on (hi, lo) words
__device__ __forceinline__ void carried_add(uint32_t* lo, uint32_t* hi, int c, double wd) {
    const uint64_t w = (uint64_t)(long long)wd;
    const uint32_t wl = (uint32_t)w, wh = (uint32_t)(w >> 32);
    const uint32_t old = atomicAdd(&lo[c], wl);
    const uint32_t up = wh + ((uint32_t)(old + wl) < old ? 1u : 0u);
    if (up) atomicAdd(&hi[c], up);
}

// position in H[0..h) of node i's hub under allocate_to_nearest
// (hm/model.py:202-207): first fp64 minimum through the exact 16-bit
// pre-filter (keys (q << 16) | k, two smallest kept; a second hub at the same
// q is a tie resolved in fp64), and a hub node is its own hub (its q is 0,
// so a competing hub at q = 0 takes the tie path, which checks for it)
__device__ __forceinline__ int corr_nearest(const DevInst& I, const int32_t* H, int h, int i) {
    unsigned m1 = 0xFFFFFFFFu, m2 = 0xFFFFFFFFu;
#pragma unroll 8
    for (int k = 0; k < h; ++k) {
        const unsigned key = ((unsigned)I.Cq[(size_t)H[k] * I.nq + i] << 16) | (unsigned)k;
        m2 = min(m2, max(m1, key));
        m1 = min(m1, key);
    }
    int kk = (int)(m1 & 0xFFFFu);
    if ((m2 >> 16) == (m1 >> 16) && H[kk] != i) {
        const unsigned qmin = m1 >> 16;
        double best = I.Ct[(size_t)H[kk] * I.n + i];
        for (int k = kk + 1; k < h; ++k) {
            if (I.Cq[(size_t)H[k] * I.nq + i] != qmin) continue;
            if (H[k] == i) return k;
            const double d = I.Ct[(size_t)H[k] * I.n + i];
            if (d < best) {
                best = d;
                kk = k;
            }
        }
    }
    return kk;
}

__global__ void __launch_bounds__(kCorrThreads)
k_correct(DevInst I, const uint32_t* __restrict__ bits, int hmax, int32_t* __restrict__ hubs_out) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ typename CorrScan::TempStorage tmp;
    __shared__ int s_kill;
    const int n = I.n, p = I.p, nw = I.nw;
    const int64_t b = blockIdx.x;
    double* carried = reinterpret_cast<double*>(sm);                 // [hmax]
    uint32_t* mask = reinterpret_cast<uint32_t*>(carried + hmax);     // [nw]
    int32_t* H = reinterpret_cast<int32_t*>(mask + nw);               // [hmax]
    int16_t* cls = reinterpret_cast<int16_t*>(H + hmax);              // [n] hub position per node
    uint16_t* nxt = reinterpret_cast<uint16_t*>(cls + n);             // [n] see below

    int h;
    if (nw <= 32) {
        // one warp counts the hubs; a child that already has p of them (the
        // common case) is extracted by that warp alone and the CTA is done
        __shared__ int s_h;
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            const uint32_t v = lane < nw ? bits[b * nw + lane] : 0u;
            if (lane < nw) mask[lane] = v;
            const int c = __popc(v);
            int pre = c;  // inclusive warp scan of the popcounts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int x = __shfl_up_sync(kFull, pre, o);
                if (lane >= o) pre += x;
            }
            const int tot = __shfl_sync(kFull, pre, 31);
            if (tot == p) {
                uint32_t w = v;
                int k = pre - c;
                while (w) {
                    hubs_out[b * p + k++] = lane * 32 + (__ffs(w) - 1);
                    w &= w - 1u;
                }
            }
            if (lane == 0) s_h = tot;
        }
        __syncthreads();
        h = s_h;
        if (h == p) return;
    } else {
        int cnt = 0;
        for (int w = threadIdx.x; w < nw; w += kCorrThreads) {
            const uint32_t v = bits[b * nw + w];
            mask[w] = v;
            cnt += __popc(v);
        }
        int dummy;
        CorrScan(tmp).ExclusiveSum(cnt, dummy, h);
        __syncthreads();
    }

    if (h < p) {
        // deficit: open closed nodes in middle-rank order (hm/operators.py:84-93)
        int need = p - h;
        for (int base = 0; need > 0 && base < n; base += kCorrThreads) {
            const int r = base + threadIdx.x;
            const int node = r < n ? I.rank[r] : -1;
            const int closed = (node >= 0 && !((mask[node >> 5] >> (node & 31)) & 1u)) ? 1 : 0;
            int pre, total;
            CorrScan(tmp).ExclusiveSum(closed, pre, total);
            if (closed && pre < need) atomicOr(&mask[node >> 5], 1u << (node & 31));
            need -= total < need ? total : need;
            __syncthreads();
        }
    }
    h = block_extract(mask, nw, H, tmp, nullptr);
    __syncthreads();

    // excess: close the least-loaded hub, one at a time (hm/operators.py:94-100)
    if (h > p && I.weights_exact) {
        // carried loads are integer-valued: exact in any order, so the nearest
        // allocation is computed once and afterwards only the nodes of the
        // closed hub move (closing a hub that is not a node's first minimum
        // leaves that node's first minimum unchanged)
        // loads as (hi, lo) 32-bit words: native shared atomics (a 64-bit
        // shared add is a compare-and-swap loop), the carry moved by hand
        uint32_t* clo = reinterpret_cast<uint32_t*>(carried);
        uint32_t* chi = clo + hmax;
        for (int k = threadIdx.x; k < h; k += kCorrThreads) clo[k] = chi[k] = 0u;
        __syncthreads();
        // 4 consecutive nodes per thread, one 8-byte load per hub row (rows are
        // padded to npad with 0xFFFF, a multiple of 16)
        // nxt[i]: node i's second-nearest hub (node id) when its three smallest
        // quantised costs are strictly ordered -- then, once its hub closes,
        // that hub (if still open) is its exact nearest, no rescan; else 0xFFFF
        for (int i0 = 4 * threadIdx.x; i0 < n; i0 += 4 * kCorrThreads) {
            unsigned m1[4], m2[4], m3[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) m1[t] = m2[t] = m3[t] = 0xFFFFFFFFu;
            const uint16_t* col = I.Cq + i0;
#pragma unroll 4
            for (int k = 0; k < h; ++k) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(col + (size_t)H[k] * I.nq));
                const unsigned q[4] = {v.x & 0xFFFFu, v.x >> 16, v.y & 0xFFFFu, v.y >> 16};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const unsigned key = (q[t] << 16) | (unsigned)k;
                    m3[t] = min(m3[t], max(m2[t], key));
                    m2[t] = min(m2[t], max(m1[t], key));
                    m1[t] = min(m1[t], key);
                }
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int i = i0 + t;
                if (i >= n) break;
                int c = (int)(m1[t] & 0xFFFFu);
                if ((m2[t] >> 16) == (m1[t] >> 16) && H[c] != i)
                    c = corr_nearest(I, H, h, i);  // quantised tie (or a hub node): exact path
                cls[i] = (int16_t)c;
                const unsigned q1 = m1[t] >> 16, q2 = m2[t] >> 16, q3 = m3[t] >> 16;
                nxt[i] = q1 < q2 && q2 < q3 && m2[t] != 0xFFFFFFFFu
                             ? (uint16_t)H[m2[t] & 0xFFFFu] : (uint16_t)0xFFFFu;
                carried_add(clo, chi, c, I.wOD[i]);
            }
        }
        __syncthreads();
        while (h > p) {
            if (threadIdx.x < 32) {
                // first minimum of the loads[0..h)
                long long bv = 0;
                int bi = -1;
                for (int k = threadIdx.x; k < h; k += 32) {
                    const long long v = (long long)(((uint64_t)chi[k] << 32) | clo[k]);
                    if (bi < 0 || v < bv) {
                        bv = v;
                        bi = k;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const long long ov = __shfl_xor_sync(kFull, bv, o);
                    const int oi = __shfl_xor_sync(kFull, bi, o);
                    if (oi >= 0 && (bi < 0 || ov < bv || (ov == bv && oi < bi))) {
                        bv = ov;
                        bi = oi;
                    }
                }
                if (threadIdx.x == 0) s_kill = bi;
                // delete position bi of H and the loads (np.delete keeps the
                // order): the warp shifts 32 entries per step
                for (int k0 = bi; k0 < h - 1; k0 += 32) {
                    const int k = k0 + (int)threadIdx.x;
                    int hv = 0;
                    uint32_t lo = 0, hi = 0;
                    if (k < h - 1) {
                        hv = H[k + 1];
                        lo = clo[k + 1];
                        hi = chi[k + 1];
                    }
                    __syncwarp();
                    if (k < h - 1) {
                        H[k] = hv;
                        clo[k] = lo;
                        chi[k] = hi;
                    }
                    __syncwarp();
                }
            }
            __syncthreads();
            const int kill = s_kill;
            --h;
            for (int i = threadIdx.x; i < n; i += kCorrThreads) {
                int c = cls[i];
                if (c == kill) {
                    const int h2 = nxt[i];
                    nxt[i] = 0xFFFFu;
                    int pos = -1;
                    if (h2 != 0xFFFF) {  // still open?  H is ascending: binary search
                        int lo = 0, hi = h - 1;
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if (H[mid] < h2) lo = mid + 1; else hi = mid;
                        }
                        if (H[lo] == h2) pos = lo;
                    }
                    c = pos >= 0 ? pos : corr_nearest(I, H, h, i);
                    carried_add(clo, chi, c, I.wOD[i]);
                } else if (c > kill) {
                    --c;
                }
                cls[i] = (int16_t)c;
            }
            __syncthreads();
        }
    }
    // fractional weights: a fresh allocation and index-ordered per-hub sums
    // each round, exactly np.bincount's order
    while (h > p) {
        for (int i = threadIdx.x; i < n; i += kCorrThreads) cls[i] = (int16_t)corr_nearest(I, H, h, i);
        __syncthreads();
        for (int k = threadIdx.x; k < h; k += kCorrThreads) {
            double acc = 0.0;
            for (int i = 0; i < n; ++i)
                if (cls[i] == k) acc += I.wOD[i];
            carried[k] = acc;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // first minimum of carried[0..h)
            double bv = 0.0;
            int bi = -1;
            for (int k = threadIdx.x; k < h; k += 32) {
                const double v = carried[k];
                if (bi < 0 || v < bv) {
                    bv = v;
                    bi = k;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(kFull, bv, o);
                const int oi = __shfl_xor_sync(kFull, bi, o);
                if (oi >= 0 && (bi < 0 || ov < bv || (ov == bv && oi < bi))) {
                    bv = ov;
                    bi = oi;
                }
            }
            for (int k0 = bi; k0 < h - 1; k0 += 32) {  // delete position bi, 32 at a time
                const int k = k0 + (int)threadIdx.x;
                const int hv = k < h - 1 ? H[k + 1] : 0;
                __syncwarp();
                if (k < h - 1) H[k] = hv;
                __syncwarp();
            }
        }
        __syncthreads();
        --h;
    }
    HG_DCHECK(h == p, "K4c left %d hubs, p = %d", h, p);
    for (int k = threadIdx.x; k < p; k += kCorrThreads) {
        HG_DCHECK(H[k] >= 0 && H[k] < n && (k == 0 || H[k] > H[k - 1]),
                  "K4c hub %d of child %lld: %d (n = %d)", k, (long long)b, H[k], n);
        hubs_out[b * p + k] = H[k];
    }
}

int launch_correct(const DevInst& I, int64_t B, const uint32_t* bits, int hmax, int32_t* hubs,
                   cudaStream_t s) {
    if (B <= 0) return HG_OK;
    if (hmax < I.p) hmax = I.p;
    size_t smem = (size_t)hmax * 8 + (size_t)I.nw * 4 + (size_t)hmax * 4;
    smem = (smem + 7) & ~size_t(7);
    smem += (size_t)I.n * 4;  // cls, nxt
    if (smem > 48 * 1024)
        HG_TRY(set_max_dynamic_smem(reinterpret_cast<const void*>(k_correct)));
    k_correct<<<(unsigned)B, kCorrThreads, smem, s>>>(I, bits, hmax, hubs);
    HG_LAUNCHED();
    return HG_OK;
}

// ---------------------------------------------------------------------------
// explicit-draw operators (single-solution API and tests)
// ---------------------------------------------------------------------------

__global__ void k_splice(int64_t B, int n, int nw, const uint32_t* __restrict__ a,
                         const uint32_t* __restrict__ bb, const int64_t* __restrict__ cuts,
                         uint32_t* __restrict__ c1, uint32_t* __restrict__ c2) {
    const int64_t total = B * nw;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = x / nw;
        const int w = (int)(x - b * nw);
        const int64_t cut = cuts[b];
        const int64_t lo = (int64_t)w * 32;
        uint32_t m;
        if (cut >= lo + 32) m = kFull;
        else if (cut <= lo) m = 0u;
        else m = (1u << (cut - lo)) - 1u;
        const uint32_t va = a[x], vb = bb[x];
        c1[x] = (va & m) | (vb & ~m);
        c2[x] = (vb & m) | (va & ~m);
    }
}

int launch_splice(int64_t B, int n, int nw, const uint32_t* a, const uint32_t* b,
                  const int64_t* cuts, uint32_t* c1, uint32_t* c2, cudaStream_t s) {
    if (B <= 0) return HG_OK;
    k_splice<<<grid_for(B * nw, 256), 256, 0, s>>>(B, n, nw, a, b, cuts, c1, c2);
    HG_LAUNCHED();
    return HG_OK;
}

constexpr int kWarpsPerBlock = 8;

__global__ void k_swap_given(int64_t B, int n, int nw, uint32_t* __restrict__ bits,
                             const int64_t* __restrict__ rc, const int64_t* __restrict__ ro) {
    extern __shared__ uint32_t wsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
    if (b >= B) return;
    uint32_t* m = wsm + warp * nw;
    for (int w = lane; w < nw; w += 32) m[w] = bits[b * nw + w];
    __syncwarp();
    if (rc[b] >= 0) {
        const int pc = warp_select(m, nw, n, (int)rc[b], true, lane);
        const int po = warp_select(m, nw, n, (int)ro[b], false, lane);
        if (lane == 0) {
            m[pc >> 5] &= ~(1u << (pc & 31));
            m[po >> 5] |= 1u << (po & 31);
        }
        __syncwarp();
    }
    for (int w = lane; w < nw; w += 32) bits[b * nw + w] = m[w];
}

int launch_swap_given(int64_t B, int n, int nw, uint32_t* bits, const int64_t* r_close,
                      const int64_t* r_open, cudaStream_t s) {
    if (B <= 0) return HG_OK;
    const unsigned blocks = (unsigned)ceil_div(B, kWarpsPerBlock);
    k_swap_given<<<blocks, kWarpsPerBlock * 32, kWarpsPerBlock * nw * 4, s>>>(B, n, nw, bits,
                                                                             r_close, r_open);
    HG_LAUNCHED();
    return HG_OK;
}

// ---------------------------------------------------------------------------
// K4a -- population build (hm/engine.py:148-153): individual 0 is the local
// ancestor (elitist), the others `strength` swaps of it.  One warp each.
// ---------------------------------------------------------------------------

__global__ void k_round_begin(GaDev G) {
    const int li = blockIdx.x;
    if (li >= G.nloc) return;
    for (int w = threadIdx.x; w < G.nw; w += blockDim.x) G.anc[(int64_t)li * G.nw + w] = 0u;
    __syncthreads();
    for (int k = threadIdx.x; k < G.p; k += blockDim.x) {
        const int h = G.inc[k];
        atomicOr(&G.anc[(int64_t)li * G.nw + (h >> 5)], 1u << (h & 31));
    }
    if (threadIdx.x == 0) G.best_raw[li] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
}

int launch_round_begin(const GaDev& G, cudaStream_t s) {
    k_round_begin<<<G.nloc, 128, 0, s>>>(G);
    HG_LAUNCHED();
    return HG_OK;
}

__global__ void k_build_pop(GaDev G) {
    extern __shared__ uint32_t wsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gid = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
    const int64_t B = (int64_t)G.nloc * G.pop;
    if (gid >= B) return;
    const int li = (int)(gid / G.pop), m = (int)(gid - (int64_t)li * G.pop);
    const int nw = G.nw, n = G.n, p = G.p;
    uint32_t* mk = wsm + warp * nw;
    for (int w = lane; w < nw; w += 32) mk[w] = G.anc[(int64_t)li * nw + w];
    __syncwarp();
    const int e = G.strict_mode ? 0 : 1;
    if (m >= e && p < n) {
        const uint64_t s = G.st[li * 3 + 0];
        const uint64_t base = G.ctr[li * 3 + 0] + (uint64_t)(m - e) * G.strength * 2;
        for (int k = 0; k < G.strength; ++k) {
            const int r1 = below(ga_draw(G.rng, s, base + 2 * k + 1), p);
            const int r2 = below(ga_draw(G.rng, s, base + 2 * k + 2), n - p);
            const int pc = warp_select(mk, nw, n, r1, true, lane);
            const int po = warp_select(mk, nw, n, r2, false, lane);
            if (lane == 0) {
                mk[pc >> 5] &= ~(1u << (pc & 31));
                mk[po >> 5] |= 1u << (po & 31);
            }
            __syncwarp();
        }
    }
    for (int w = lane; w < nw; w += 32) G.popbits[gid * nw + w] = mk[w];
}

int launch_build_pop(const GaDev& G, cudaStream_t s) {
    const int64_t B = (int64_t)G.nloc * G.pop;
    const unsigned blocks = (unsigned)ceil_div(B, kWarpsPerBlock);
    k_build_pop<<<blocks, kWarpsPerBlock * 32, kWarpsPerBlock * G.nw * 4, s>>>(G);
    HG_LAUNCHED();
    return HG_OK;
}

// ---------------------------------------------------------------------------
// K4b -- crossover (hm/operators.py:41-57) of pairs (2j, 2j+1), one warp each
// ---------------------------------------------------------------------------

__global__ void k_crossover(GaDev G) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int half = G.pop / 2;
    const int64_t gid = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
    if (gid >= (int64_t)G.nloc * half) return;
    const int li = (int)(gid / half), j = (int)(gid - (int64_t)li * half);
    const int n = G.n, nw = G.nw;
    int cut = n;  // n == 1: both children are copies, no draw
    if (n > 1)
        cut = 1 + below(ga_draw(G.rng, G.st[li * 3 + 1], G.ctr[li * 3 + 1] + j + 1), n - 1);
    const int64_t ia = (int64_t)li * G.pop + 2 * j;
    const uint32_t* a = G.popbits + ia * nw;
    const uint32_t* bb = a + nw;
    uint32_t* c1 = G.kids + ia * nw;
    uint32_t* c2 = c1 + nw;
    int n1 = 0, n2 = 0;
    for (int w = lane; w < nw; w += 32) {
        const int lo = w * 32;
        uint32_t m;
        if (cut >= lo + 32) m = kFull;
        else if (cut <= lo) m = 0u;
        else m = (1u << (cut - lo)) - 1u;
        const uint32_t va = a[w], vb = bb[w];
        const uint32_t x1 = (va & m) | (vb & ~m), x2 = (vb & m) | (va & ~m);
        c1[w] = x1;
        c2[w] = x2;
        n1 += __popc(x1);
        n2 += __popc(x2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n1 += __shfl_xor_sync(kFull, n1, o);
        n2 += __shfl_xor_sync(kFull, n2, o);
    }
    if (lane == 0) {
        G.kcount[ia] = n1;
        G.kcount[ia + 1] = n2;
    }
}

int launch_crossover(const GaDev& G, cudaStream_t s) {
    const int64_t P = (int64_t)G.nloc * (G.pop / 2);
    const unsigned blocks = (unsigned)ceil_div(P, kWarpsPerBlock);
    k_crossover<<<blocks, kWarpsPerBlock * 32, 0, s>>>(G);
    HG_LAUNCHED();
    return HG_OK;
}

// per island: exclusive count of non-degenerate children before each child
constexpr int kScanThreads = 256;
using MutScan = cub::BlockScan<int, kScanThreads>;

__global__ void k_mut_scan(GaDev G) {
    __shared__ typename MutScan::TempStorage tmp;
    const int li = blockIdx.x;
    int base = 0;
    for (int m0 = 0; m0 < G.pop; m0 += kScanThreads) {
        const int m = m0 + threadIdx.x;
        int flag = 0;
        if (m < G.pop) {
            const int c = G.kcount[(int64_t)li * G.pop + m];
            flag = (c != 0 && c != G.n) ? 1 : 0;
        }
        int off, total;
        MutScan(tmp).ExclusiveSum(flag, off, total);
        if (m < G.pop) G.moff[(int64_t)li * G.pop + m] = base + off;
        base += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) G.nondeg[li] = base;
}

int launch_mut_scan(const GaDev& G, cudaStream_t s) {
    k_mut_scan<<<G.nloc, kScanThreads, 0, s>>>(G);
    HG_LAUNCHED();
    return HG_OK;
}

// swap mutation of every child (hm/operators.py:113-124, engine.py:157)
__global__ void k_mutate(GaDev G) {
    extern __shared__ uint32_t wsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gid = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
    const int64_t B = (int64_t)G.nloc * G.pop;
    if (gid >= B) return;
    const int cnt = G.kcount[gid];
    const int n = G.n, nw = G.nw;
    if (cnt == 0 || cnt == n) return;  // identity, no draws
    const int li = (int)(gid / G.pop);
    uint32_t* mk = wsm + warp * nw;
    uint32_t* g = G.kids + gid * nw;
    for (int w = lane; w < nw; w += 32) mk[w] = g[w];
    __syncwarp();
    const uint64_t s = G.st[li * 3 + 2];
    const uint64_t base = G.ctr[li * 3 + 2] + 2ull * (uint64_t)G.moff[gid];
    const int r1 = below(ga_draw(G.rng, s, base + 1), cnt);
    const int r2 = below(ga_draw(G.rng, s, base + 2), n - cnt);
    const int pc = warp_select(mk, nw, n, r1, true, lane);
    const int po = warp_select(mk, nw, n, r2, false, lane);  // closed list before closing
    if (lane == 0) {
        mk[pc >> 5] &= ~(1u << (pc & 31));
        mk[po >> 5] |= 1u << (po & 31);
    }
    __syncwarp();
    for (int w = lane; w < nw; w += 32) g[w] = mk[w];
}

int launch_mutate(const GaDev& G, cudaStream_t s) {
    const int64_t B = (int64_t)G.nloc * G.pop;
    const unsigned blocks = (unsigned)ceil_div(B, kWarpsPerBlock);
    k_mutate<<<blocks, kWarpsPerBlock * 32, kWarpsPerBlock * G.nw * 4, s>>>(G);
    HG_LAUNCHED();
    return HG_OK;
}

// ---------------------------------------------------------------------------
// K5 -- island selection (hm/engine.py:162-166): champion = first strict
// minimum in child order; the local ancestor becomes the champion; the island
// best keeps the earliest strict minimum across generations.  Also advances
// the three stream counters by what this generation consumed.
// ---------------------------------------------------------------------------

__global__ void k_select(GaDev G) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int li = blockIdx.x * (blockDim.x >> 5) + warp;
    if (li >= G.nloc) return;
    const int pop = G.pop, p = G.p, nw = G.nw;
    double bv = 0.0;
    int bi = -1;
    for (int m = lane; m < pop; m += 32) {
        const double v = G.kraw[((int64_t)li * pop + m) * 4 + 3];
        if (bi < 0 || v < bv) {
            bv = v;
            bi = m;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, bv, o);
        const int oi = __shfl_xor_sync(kFull, bi, o);
        if (oi >= 0 && (bi < 0 || ov < bv || (ov == bv && oi < bi))) {
            bv = ov;
            bi = oi;
        }
    }
    const int32_t* ch = G.khubs + ((int64_t)li * pop + bi) * p;
    uint32_t* anc = G.anc + (int64_t)li * nw;
    for (int w = lane; w < nw; w += 32) anc[w] = 0u;
    __syncwarp();
    for (int k = lane; k < p; k += 32) {
        const int h = ch[k];
        atomicOr(&anc[h >> 5], 1u << (h & 31));
        G.champ_hubs[(int64_t)li * p + k] = h;
    }
    const bool better = bv < G.best_raw[li];
    __syncwarp();
    if (better)
        for (int k = lane; k < p; k += 32) G.best_hubs[(int64_t)li * p + k] = ch[k];
    if (lane == 0) {
        G.champ_raw[li] = bv;
        if (better) G.best_raw[li] = bv;
        const int e = G.strict_mode ? 0 : 1;
        if (p < G.n) G.ctr[li * 3 + 0] += (uint64_t)(pop - e) * G.strength * 2;
        if (G.n > 1) G.ctr[li * 3 + 1] += (uint64_t)(pop / 2);
        G.ctr[li * 3 + 2] += 2ull * (uint64_t)G.nondeg[li];
    }
}

int launch_select(const GaDev& G, cudaStream_t s) {
    const int wpb = 4;
    k_select<<<(unsigned)ceil_div(G.nloc, wpb), wpb * 32, 0, s>>>(G);
    HG_LAUNCHED();
    return HG_OK;
}

}  // namespace hg
