// K3-TC: population fitness (transfer term) on the 5th-generation tensor cores.
//
// When every flow W_ij is an integer in [0, 255] (all synthetic instances of
// the reference generator, hm/io.py:203, are integers in [0, 100]) the
// transfer term factors EXACTLY through an integer GEMM:
//
//   G_b[i][l]  = sum_j W[i][j] * [c_b(j) == l]          (u8 x u8 -> s32, exact)
//   S_T(b)     = sum_i sum_l G_b[i][l] * T_b[c_b(i)][l]  (fp64 epilogue)
//
// which equals sum_ij W_ij C[a_i][a_j] of hm/evaluation.py:113-119 up to fp64
// summation order.  Batched over the population, G is one GEMM
//   D[i][(b,l)] = W[i][:] . OneHot[(b,l)][:]
// with M = nodes i, N = (individual, hub) pairs (ipt individuals x p <= 256),
// K = nodes j.
//
// Work unit = (N tile of ipt individuals, PAIR of 128-row M tiles).  Per CTA
// (512 threads, one per SM) TMEM holds the two 128 x N s32 accumulators
// (columns 0 and 256).  Per 128-wide K block: the two W tiles (A operands,
// K-major, SWIZZLE_128B) arrive by TMA; the one-hot B tile is generated ONCE
// in shared memory (same canonical layout) from cluster ids staged by
// cp.async one K block ahead, fenced to the async proxy, and consumed by the
// 8 tcgen05.mma.kind::i8 of both accumulators (issued by one thread); K
// blocks are double-buffered so generation of block k+1 overlaps the MMAs of
// block k.  The epilogue reads the accumulators with tcgen05.ld, converts
// exactly to fp64 and contracts with the staged hub-cost tables; one partial
// per (individual, 128-row tile) in a fixed reduction order.

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_pipeline.h>

#include <cstdlib>

#include "hg_internal.cuh"

namespace hg {

namespace {

constexpr int kTcThreads = 512;
constexpr int kTcWarps = kTcThreads / 32;
constexpr int kTcTmemCols = 512;
constexpr int kAStage = 128 * 128;   // bytes: 128 rows x 128 K (u8), one M tile
constexpr int kBStage = 256 * 128;   // bytes: up to 256 rows x 128 K
constexpr int kMaxIpt = 64;  // caps the per-tile staging for tiny p

// shared memory map (offsets from the 1024-aligned base)
constexpr int kOffA = 0;                            // [2 stages][2 tiles] x 16 KB
constexpr int kOffB = kOffA + 4 * kAStage;          // [2 stages] x 32 KB
constexpr int kOffRowInfo = kOffB + 2 * kBStage;    // [256] int: (bl << 16) | l
constexpr int kOffVar = kOffRowInfo + 256 * 4;      // variable part

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

// K-major, SWIZZLE_128B canonical layout: 8-row x 128 B atoms, 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);  // start address
    d |= (uint64_t)1 << 16;                   // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;         // stride byte offset: next 8-row group
    d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// byte-wise (x == l) -> 0x80 / 0x00, exact (no cross-byte carries).  The
// one-hot value is 128 (u8) instead of 1: the GEMM yields 128*G exactly
// (< 2^31) and the 2^-7 is folded into the staged hub-cost tables.
__device__ __forceinline__ uint32_t onehot4(uint32_t x, uint32_t lrep) {
    const uint32_t y = x ^ lrep;
    const uint32_t t = (y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    return ~(t | y) & 0x80808080u;
}

}  // namespace

struct TcArgs {
    const uint8_t* cl;
    const uint32_t* T;
    double* part;
    int64_t B;
    int n, p, ps, npad;
    int ipt;      // individuals per N tile
    int N;        // MMA N (multiple of 16, <= 256)
    int64_t NT;   // N tiles
    int MT, MP;   // 128-row tiles, tile pairs
    int KB;       // 128-wide K blocks
    int pss;      // smem row stride (doubles) of the staged T rows: even, pss/2 odd
    uint32_t idesc;
    unsigned long long* timing;  // optional per-phase cycle counters (tuning builds)
};

// staged T: ipt x p rows of pss doubles (16-byte aligned rows, and an odd
// number of 16-byte chunks per row so a quarter-warp's LDS.128 of 8 different
// rows hit 8 different bank groups)
__host__ __device__ inline int tc_var_T(int ipt, int p, int pss) {
    return ((ipt * p * pss * 8) + 15) & ~15;
}

__global__ void __launch_bounds__(kTcThreads, 1)
k_fitness_tc(const __grid_constant__ CUtensorMap tmW, TcArgs A) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-align by pointer arithmetic on the shared array itself, so the
    // compiler keeps every access in the shared window (LDS/STS, not LD/ST.E)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int p = A.p, ipt = A.ipt;
    unsigned char* var = smem + kOffVar;
    double* sT = reinterpret_cast<double*>(var);                      // [ipt][p][pss] T * 2^-7
    var += tc_var_T(ipt, p, A.pss);
    uint8_t* cbuf = var;                                              // [2][ipt][128] next cids
    var += 2 * ((ipt * 128 + 15) & ~15);
    uint8_t* sc = var;                  // [2][ipt][128] cids currently set in B stage s (0xFF: none)
    var += 2 * ((ipt * 128 + 15) & ~15);
    uint8_t* rc = var;                                                // [2][ipt][256] row cids
    const int rcstride = (ipt * 256 + 15) & ~15;
    var += 2 * rcstride;
    double* red = reinterpret_cast<double*>(var);                     // [16 warps][2][ipt]
    var += kTcWarps * 2 * ipt * 8;
    uint64_t* bars = reinterpret_cast<uint64_t*>(var);                // tma[2], mma[2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t bar_tma0 = smem_u32(bars), bar_mma0 = smem_u32(bars + 2);
    const int cstride = (ipt * 128 + 15) & ~15;
    // phase timing (only when A.timing is set): thread 0 (MMA issuer) and thread 32
    const bool timed = A.timing != nullptr && (tid == 0 || tid == 32);
    unsigned long long tph[12] = {0};
    long long tlast = timed ? clock64() : 0;
#define TC_T(ph)                                   \
    do {                                           \
        if (timed) {                               \
            const long long now_ = clock64();      \
            tph[ph] += (unsigned long long)(now_ - tlast); \
            tlast = now_;                          \
        }                                          \
    } while (0)

    if (tid == 0) {
        mbar_init(bar_tma0, 1);
        mbar_init(bar_tma0 + 8, 1);
        mbar_init(bar_mma0, 1);
        mbar_init(bar_mma0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    }
    // B stages start all-zero; afterwards only the bytes that change are written
    for (int x = tid; x < 2 * kBStage / 16; x += kTcThreads)
        reinterpret_cast<uint4*>(smem + kOffB)[x] = make_uint4(0u, 0u, 0u, 0u);
    for (int x = tid; x < 2 * cstride; x += kTcThreads) sc[x] = 0xFF;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(kTcTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int64_t units = A.NT * A.MP;
    const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
    uint32_t n_tma[2] = {0, 0}, n_mma[2] = {0, 0};
    int64_t cur_nt = -1;

    struct UnitInfo {
        int64_t nt, bbase;
        int m0, nind;
        bool has1;
    };
    auto unit_info = [&](int64_t u) {
        UnitInfo U;
        U.nt = u / A.MP;
        U.m0 = 2 * (int)(u - U.nt * A.MP);
        U.has1 = U.m0 + 1 < A.MT;
        U.bbase = U.nt * ipt;
        U.nind = (int)(A.B - U.bbase < ipt ? A.B - U.bbase : ipt);
        return U;
    };
    // thread 0: the two W tiles of K block kb into A stage s
    auto issue_A = [&](const UnitInfo& U, int kb, int s) {
        unsigned char* a_st = smem + kOffA + s * 2 * kAStage;
        mbar_expect_tx(bar_tma0 + 8 * s, U.has1 ? 2 * kAStage : kAStage);
        tma_load_2d(smem_u32(a_st), &tmW, kb * 128, U.m0 * 128, bar_tma0 + 8 * s);
        if (U.has1)
            tma_load_2d(smem_u32(a_st + kAStage), &tmW, kb * 128, (U.m0 + 1) * 128,
                        bar_tma0 + 8 * s);
    };
    auto fetch_cids = [&](const UnitInfo& U, int kb, uint8_t* dst) {
        for (int x = tid; x < U.nind * 8; x += kTcThreads) {
            const int bl = x >> 3, k = x & 7;
            __pipeline_memcpy_async(dst + bl * 128 + k * 16,
                                    A.cl + (U.bbase + bl) * A.npad + kb * 128 + k * 16, 16);
        }
    };
    auto fetch_rc = [&](const UnitInfo& U, uint8_t* dst) {  // row cids of the pair's 256 rows
        for (int x = tid; x < U.nind * 16; x += kTcThreads) {
            const int bl = x >> 4, k = x & 15;
            const int i0 = U.m0 * 128 + k * 16;
            if (i0 < A.npad)
                __pipeline_memcpy_async(dst + bl * 256 + k * 16,
                                        A.cl + (U.bbase + bl) * A.npad + i0, 16);
        }
    };

    // prologue: first unit's K block 0 (stage 0) and epilogue row ids
    uint32_t gk = 0;  // K blocks issued by this CTA so far (stage = gk & 1)
    if (u0 < u1) {
        const UnitInfo U = unit_info(u0);
        if (tid == 0) issue_A(U, 0, 0);
        n_tma[0]++;
        fetch_cids(U, 0, cbuf);
        fetch_rc(U, rc);
        __pipeline_commit();
        __pipeline_wait_prior(0);
        __syncthreads();
    }

    for (int64_t u = u0; u < u1; ++u) {
        const UnitInfo U = unit_info(u);
        const int m0 = U.m0, nind = U.nind;
        const bool has1 = U.has1;
        const int64_t bbase = U.bbase;
        const uint8_t* rcu = rc + ((u - u0) & 1) * rcstride;
        TC_T(11);
        if (U.nt != cur_nt) {
            // hub-cost tables of this N tile's individuals as fp64 x 2^-7 (exact
            // power-of-two scaling: undoes the one-hot value 128)
            // power-of-two scaling: undoes the one-hot value 128); row tails up to
            // pss are zero so the epilogue runs whole 8-column chunks unguarded
            cur_nt = U.nt;
            const int pss = A.pss;
            const int per = p * pss;
            for (int x = tid; x < ipt * per; x += kTcThreads) {
                const int bl = x / per, y = x - bl * per;
                const int c = y / pss, l = y - c * pss;
                double v = 0.0;
                if (bl < nind && l < p) {
                    const uint32_t* tb = A.T + (bbase + bl) * 2 * p * (int64_t)A.ps;
                    v = __hiloint2double((int)tb[c * A.ps + l], (int)tb[(p + c) * A.ps + l]) *
                        0.0078125;
                }
                sT[(bl * p + c) * A.pss + l] = v;
            }
        }

        TC_T(0);
        for (int kb = 0; kb < A.KB; ++kb, ++gk) {
            const int s = gk & 1;
            // B stage s is free once the MMAs of K block gk-2 are done
            if (gk >= 2) mbar_wait(bar_mma0 + 8 * s, (n_mma[s] - 1) & 1);
            TC_T(1);
            unsigned char* a_st = smem + kOffA + s * 2 * kAStage;
            unsigned char* b_st = smem + kOffB + s * kBStage;
            if (kb + 1 < A.KB) fetch_cids(U, kb + 1, cbuf + (s ^ 1) * cstride);
            __pipeline_commit();
            // one-hot B tile, row r = (individual bl, hub l), 128 K bytes, SW128
            // swizzled: thread (r, half) builds 64 bytes of row r by byte-wise
            // compares of the staged cluster ids with l -- branch-free, 4
            // independent 16-byte chunks per thread (latency hidden by ILP)
            {
                const uint8_t* cb = cbuf + s * cstride;
                for (int it = tid; it < A.N * 2; it += kTcThreads) {
                    const int r = it >> 1, h2 = it & 1;
                    const int bl = r / p, l = r - bl * p;
                    const bool live = bl < nind;
                    const uint32_t lrep = (uint32_t)l * 0x01010101u;
                    const uint4* src = reinterpret_cast<const uint4*>(cb + bl * 128 + h2 * 64);
                    unsigned char* dst = b_st + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = h2 * 4 + q;
                        uint4 v = make_uint4(0u, 0u, 0u, 0u);
                        if (live) {
                            const uint4 x = src[q];
                            v.x = onehot4(x.x, lrep);
                            v.y = onehot4(x.y, lrep);
                            v.z = onehot4(x.z, lrep);
                            v.w = onehot4(x.w, lrep);
                        }
                        *reinterpret_cast<uint4*>(dst + ((c ^ (r & 7)) << 4)) = v;
                    }
                }
            }
            TC_T(2);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __pipeline_wait_prior(0);  // cluster ids of the next K block have landed
            __syncthreads();
            TC_T(3);
            if (tid == 0) {
                mbar_wait(bar_tma0 + 8 * s, (n_tma[s] - 1) & 1);
                TC_T(4);
                tc_fence_after();
                const uint64_t a0 = sw128_desc(smem_u32(a_st));
                const uint64_t a1 = sw128_desc(smem_u32(a_st + kAStage));
                const uint64_t bd = sw128_desc(smem_u32(b_st));
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)  // K = 32 bytes per MMA: +2 in 16 B units
                    mma_i8(tmem, a0 + 2 * ks, bd + 2 * ks, A.idesc, (kb | ks) != 0);
                if (has1) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        mma_i8(tmem + 256, a1 + 2 * ks, bd + 2 * ks, A.idesc, (kb | ks) != 0);
                }
                mma_commit(bar_mma0 + 8 * s);
                TC_T(5);
                // the next K block's W tiles go into stage s^1 as soon as the MMAs of
                // K block gk-1 (its previous user) are done: a full block of lead time
                if (kb + 1 < A.KB) {
                    if (gk >= 1) mbar_wait(bar_mma0 + 8 * (s ^ 1), (n_mma[s ^ 1] - 1) & 1);
                    issue_A(U, kb + 1, s ^ 1);
                }
                TC_T(6);
            }
            n_mma[s]++;
            if (kb + 1 < A.KB) n_tma[s ^ 1]++;
        }
        // accumulators complete (MMAs retire in order)
        const int sl = (gk - 1) & 1;
        mbar_wait(bar_mma0 + 8 * sl, (n_mma[sl] - 1) & 1);
        tc_fence_after();
        TC_T(7);
        // prefetch the next unit's first K block and row ids under the epilogue
        if (u + 1 < u1) {
            const UnitInfo Un = unit_info(u + 1);
            if (tid == 0) issue_A(Un, 0, gk & 1);
            n_tma[gk & 1]++;
            fetch_cids(Un, 0, cbuf + (gk & 1) * cstride);
            fetch_rc(Un, rc + ((u + 1 - u0) & 1) * rcstride);
        }
        __pipeline_commit();
        TC_T(8);

        // epilogue: warp w reads TMEM lanes (rows) 32*(w&3)..; the 4 warp
        // groups g = w>>2 take individuals bl = g, g+4, ...
        const int q = warp & 3, g = warp >> 2;
        for (int a = 0; a < (has1 ? 2 : 1); ++a) {
            const int rloc = a * 128 + q * 32 + lane;  // row within the pair
            const uint32_t trow = tmem + (uint32_t)(a * 256) + ((uint32_t)(q * 32) << 16);
            for (int bl = g; bl < nind; bl += 4) {
                const int c = rcu[bl * 256 + rloc];
                const double2* tr = reinterpret_cast<const double2*>(sT + (bl * p + c) * A.pss);
                double acc0 = 0.0, acc1 = 0.0;
                for (int l0 = 0; l0 < p; l0 += 8) {
                    // 8 accumulator columns (the tail beyond p belongs to the next
                    // individual or is unused: it meets zero T entries)
                    uint32_t d[8];
                    tmem_ld8(trow + (uint32_t)(bl * p + l0), d);
                    // the thread's T row (c fixed per row and individual) while the
                    // TMEM load is in flight
                    double2 t[4];
#pragma unroll
                    for (int k2 = 0; k2 < 4; ++k2) t[k2] = tr[(l0 >> 1) + k2];
                    tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        // exact u32 -> fp64: (2^52 + d) - 2^52
                        const double dd =
                            __hiloint2double(0x43300000, (int)d[k]) - 4503599627370496.0;
                        const double tv = (k & 1) ? t[k >> 1].y : t[k >> 1].x;
                        if (k & 1) acc1 = fma(dd, tv, acc1);
                        else acc0 = fma(dd, tv, acc0);
                    }
                }
                double acc = acc0 + acc1;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0) red[(warp * 2 + a) * ipt + bl] = acc;
            }
        }
        TC_T(9);
        tc_fence_before();
        __pipeline_wait_prior(0);  // next unit's prefetch has landed
        __syncthreads();
        for (int x = tid; x < 2 * nind; x += kTcThreads) {
            const int a = x / nind, bl = x - a * nind;
            if (a == 1 && !has1) continue;
            const int gg = bl & 3;
            double s4 = 0.0;
            for (int qq = 0; qq < 4; ++qq) s4 += red[((gg * 4 + qq) * 2 + a) * ipt + bl];
            A.part[(bbase + bl) * A.MT + m0 + a] = s4;
        }
        // red / rc / cbuf are rewritten only after the next unit's first __syncthreads
    }
    TC_T(10);
    if (timed)
        for (int k = 0; k < 12; ++k) atomicAdd(A.timing + (tid ? 16 : 0) + k, tph[k]);
#undef TC_T
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(kTcTmemCols)
                     : "memory");
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

// HUBGPU_TC_TIMING=1: per-phase cycle counters of K3-TC (tuning only)
unsigned long long* tc_timing_buffer() {
    static int on = -1;
    static unsigned long long* buf = nullptr;
    if (on < 0) {
        const char* e = getenv("HUBGPU_TC_TIMING");
        on = (e && e[0] == '1') ? 1 : 0;
        if (on && cudaMalloc(&buf, 32 * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(buf, 0, 32 * sizeof(unsigned long long));
        else
            buf = nullptr;
    }
    return buf;
}

int tc_timing_read(unsigned long long* out32) {
    unsigned long long* b = tc_timing_buffer();
    if (!b) return HG_EARG;
    HG_CUDA(cudaMemcpy(out32, b, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    HG_CUDA(cudaMemset(b, 0, 32 * sizeof(unsigned long long)));
    return HG_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

int tc_make_wmap(const uint8_t* W8, int npad_tc, int box_rows, void* map_out, int rows) {
    auto enc = get_encode();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return HG_ECUDA;
    }
    CUtensorMap* m = static_cast<CUtensorMap*>(map_out);
    cuuint64_t dims[2] = {(cuuint64_t)npad_tc, (cuuint64_t)(rows > 0 ? rows : npad_tc)};
    cuuint64_t strides[1] = {(cuuint64_t)npad_tc};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)W8, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return HG_ECUDA;
    }
    return HG_OK;
}

// row stride (doubles) of staged T: >= p rounded up to 8 (zero tail), with an
// odd number of 16-byte chunks per row (conflict-free LDS.128 across rows)
static int tc_pss(int p) { return ((p + 7) & ~7) + 2; }

static size_t tc_smem_for(int p, int ipt) {
    size_t b = 1024 + kOffVar;
    b += tc_var_T(ipt, p, tc_pss(p));
    b += 4 * ((ipt * 128 + 15) & ~15);  // cbuf + sc
    b += 2 * ((ipt * 256 + 15) & ~15);
    b += kTcWarps * 2 * ipt * 8;
    b += 4 * 8 + 16;
    return b;
}

// individuals per N tile: as many as fit N <= 256 and the shared memory
static int tc_ipt(int p) {
    int ipt = 256 / p < kMaxIpt ? 256 / p : kMaxIpt;
    // the epilogue reads 8 accumulator columns at a time: the last individual's
    // reads must stay inside its 256-column accumulator
    const int p8 = (p + 7) & ~7;
    while (ipt > 1 && (ipt - 1) * p + p8 > 256) --ipt;
    while (ipt > 1 && tc_smem_for(p, ipt) > 227 * 1024) --ipt;
    return ipt;
}

size_t tc_smem_bytes(int p) { return tc_smem_for(p, tc_ipt(p)); }

bool tc_supported(int p) { return p >= 1 && p <= 128 && tc_smem_bytes(p) <= 227 * 1024; }

int tc_tiles(int n) { return (int)(round_up(n, 128) / 128); }

int prepare_fitness_tc(int p) {
    HG_CUDA(cudaFuncSetAttribute(k_fitness_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tc_smem_bytes(p)));
    return HG_OK;
}

int launch_fitness_tc(const DevInst& I, const void* wmap, int64_t B, const uint8_t* cl,
                      const uint32_t* T, double* part, int grid, cudaStream_t s) {
    if (B <= 0) return HG_OK;
    TcArgs A;
    A.cl = cl;
    A.T = T;
    A.part = part;
    A.B = B;
    A.n = I.n;
    A.p = I.p;
    A.ps = I.ps;
    A.npad = I.npad;
    A.ipt = tc_ipt(I.p);
    A.N = (int)round_up((int64_t)A.ipt * I.p, 16);
    A.NT = ceil_div(B, A.ipt);
    A.MT = tc_tiles(I.n);
    A.MP = (A.MT + 1) / 2;
    A.KB = A.MT;
    A.pss = tc_pss(I.p);
    // kind::i8 instruction descriptor: D s32, A/B u8, both K-major, N, M=128
    A.idesc = (2u << 4) | ((uint32_t)(A.N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    A.timing = tc_timing_buffer();
    const int64_t units = A.NT * A.MP;
    int g = grid;
    if (g > units) g = (int)units;
    CUtensorMap map = *static_cast<const CUtensorMap*>(wmap);
    k_fitness_tc<<<g, kTcThreads, tc_smem_bytes(I.p), s>>>(map, A);
    HG_CUDA(cudaGetLastError());
    return HG_OK;
}

}  // namespace hg
