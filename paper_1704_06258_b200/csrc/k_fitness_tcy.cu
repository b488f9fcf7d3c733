// K3-TC/Y: population fitness (transfer term) on tcgen05 with the one-hot
// operand RESIDENT IN TENSOR MEMORY (n <= 1024).
//
// Same exact factorisation as k_fitness_tc.cu (hm/evaluation.py:113-119):
//   D[(b,l)][i] = sum_j OneHot[(b,l)][j] * W[i][j]  = 128 * G_b[i][l]   (u8 x u8 -> s32)
//   S_T(b)      = sum_i sum_l G_b[i][l] * T_b[c_b(i)][l]
// but with the roles swapped: the one-hot rows (individual b, hub l) are the
// A operand -- M = 128 TMEM lanes, all K = n columns of it generated ONCE per
// unit straight into TMEM with tcgen05.st -- and W is the B operand, streamed
// by TMA through a 6-deep shared-memory ring.  Shared memory then carries only
// W (TMA write + MMA read), a third of the traffic of the smem-resident one-hot
// design.  TMEM: A in columns [0, 256), two N=128 accumulators in [256, 512):
// the epilogue of one 128-row W tile overlaps the MMAs of the next.
//
// Warp roles (20 warps): warp 0 = MMA issuer, warp 1 = TMA producer, warps
// 4..19 = generators + epilogue (warp w reads TMEM lane quadrant w % 4, and
// the 4 warps of a quadrant split the 128 accumulator columns).

#include <cuda.h>
#include <cuda_pipeline.h>

#include <cstdlib>

#include "hg_internal.cuh"

namespace hg {

namespace {

constexpr int kYThreads = 640;
constexpr int kYWarps = kYThreads / 32;
constexpr int kYEpiWarp0 = 4;                 // first epilogue warp
constexpr int kYEpiThreads = kYThreads - 128; // 512
constexpr int kYMaxStages = 16;               // W ring depth bound (runtime: YArgs::stages)
constexpr int kYStageBytes = 128 * 128;       // 128 W rows x 128 K (u8)
constexpr int kYMaxIpt = 32;
constexpr int kYTmemCols = 512;
constexpr int kYAcc0 = 256;                   // first accumulator column
constexpr int kYCluster = kTcyCluster;        // CTAs sharing each W tile by TMA multicast

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mb_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAITY_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAITY_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// one quarter of a W tile, multicast into the same smem offset of every CTA of
// the cluster; each destination's mbarrier (same offset) gets the bytes
__device__ __forceinline__ void tma2d_mc(uint32_t dst, const CUtensorMap* map, int x, int y,
                                         uint32_t bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(bar), "h"(mask)
        : "memory");
}
// arrive on the mbarrier at this offset in every CTA of the mask once the
// issued MMAs have completed (frees a W stage cluster-wide)
__device__ __forceinline__ void commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
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
// D[tmem] (+)= A[tmem] . B[smem]^T, kind::i8
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
        : "memory");
}
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void epi_sync() {  // named barrier over the 16 epilogue warps
    asm volatile("bar.sync 1, %0;" ::"n"(kYEpiThreads) : "memory");
}
// byte-wise (x == l) -> 1 / 0.  Cluster ids and l are < 128, so every byte of
// y = x ^ l has its top bit clear and y + 0x7F per byte cannot carry: bit 7 of
// a byte of t is set exactly when that byte of y is nonzero (4 integer ops)
__device__ __forceinline__ uint32_t oh4(uint32_t x, uint32_t lrep) {
    const uint32_t y = x ^ lrep;
    const uint32_t t = y + 0x7F7F7F7Fu;
    return (~t & 0x80808080u) >> 7;
}

}  // namespace

struct YArgs {
    const uint8_t* cl;
    const uint32_t* T;
    double* part;     // [B][1]: S_T complete per individual
    int64_t B;
    int n, p, ps, npad;
    int ipt;          // individuals per unit (ipt * p <= 128)
    int64_t units;
    int IT;           // 128-row W tiles (= K blocks)
    int acols;        // TMEM columns of A = IT * 32
    int stages;       // W ring depth
    int kbs;          // 128-byte K blocks per stage
    uint32_t idesc;   // kind::i8, M=128, N=128, K-major both
    unsigned long long* timing;  // optional phase counters (HUBGPU_TC_TIMING=1)
    int dbg;                     // ablation flags (tuning only): 1 = no epilogue math, 2 = no MMA
};

__host__ __device__ inline size_t y_C_bytes(int ipt, int npad) {
    return ((size_t)ipt * npad + 15) & ~size_t(15);
}

__global__ void __launch_bounds__(kYThreads, 1)
k_fitness_tcy(const __grid_constant__ CUtensorMap tmW, YArgs A) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const int p = A.p, ipt = A.ipt, IT = A.IT;
    unsigned char* ring = smem;                                          // W stages
    const int NS = A.stages, KBS = A.kbs;
    unsigned char* var = smem + NS * KBS * kYStageBytes;
    const size_t cb = y_C_bytes(ipt, A.npad);
    // double buffer addressed arithmetically from the shared base (a pointer
    // array indexed at run time would drop to local memory and generic loads)
    unsigned char* sC0 = var;
    var += 2 * cb;
    uint32_t* bins = reinterpret_cast<uint32_t*>(var);  // [p][128] cluster-pair flow bins
    var += (size_t)p * 512;
    double* red = reinterpret_cast<double*>(var);  // [4 subs][128 rows]
    var += 4 * 128 * 8;
    uint64_t* bars = reinterpret_cast<uint64_t*>(var);
    // bars: full[16] empty[16] accfull[2] accempty[2] kbfree[4] aready[4]
    const uint32_t b_full = su32(bars), b_empty = b_full + 8 * kYMaxStages,
                   b_accf = b_empty + 8 * kYMaxStages, b_acce = b_accf + 16, b_kbf = b_acce + 16,
                   b_ard = b_kbf + 32;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kYMaxStages + 12);
    // A's K blocks are generated in 4 contiguous ranges, one per column-quarter
    // warp group: quarter h owns K blocks [kq(h), kq(h+1))
    auto kq = [&](int h) { return h * IT / 4; };

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int x = tid; x < p * 128; x += kYThreads) bins[x] = 0u;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mb_init(b_full + 8 * s, 1);
            mb_init(b_empty + 8 * s, kYCluster);  // every consumer CTA of the cluster
        }
        for (int d = 0; d < 2; ++d) {
            mb_init(b_accf + 8 * d, 1);
            mb_init(b_acce + 8 * d, kYWarps - kYEpiWarp0);
        }
        for (int h = 0; h < 4; ++h) {
            mb_init(b_kbf + 8 * h, 1);
            mb_init(b_ard + 8 * h, 4);  // the 4 lane-quadrant warps of quarter h
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(tmem_slot)),
                     "r"(kYTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    cluster_sync_all();  // peers' barriers are initialised before any multicast
    const uint32_t tmem = *tmem_slot;

    // units of this cluster, interleaved over its CTAs; every CTA runs the same
    // number of slots (a slot past the end is a dummy unit) so the multicast W
    // stream stays in lockstep
    const uint32_t crank = cluster_rank();
    const int64_t ncl = gridDim.x / kYCluster, cid = blockIdx.x / kYCluster;
    const int64_t cs0 = A.units * cid / ncl, cs1 = A.units * (cid + 1) / ncl;
    const int64_t nslots = (cs1 - cs0 + kYCluster - 1) / kYCluster;
    const uint16_t all_mask = (uint16_t)((1u << kYCluster) - 1);

    if (warp == 1) {
        // ---------------- TMA producer: W tiles (it, K-block group), same order
        // every unit; a stage holds KBS consecutive 128-byte K blocks
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            bool wrapped = false;
            const int q = (int)crank * (128 / kYCluster);
            for (int64_t j = 0; j < nslots; ++j)
                for (int it = 0; it < IT; ++it)
                    for (int kb0 = 0; kb0 < IT; kb0 += KBS) {
                        const int nk = IT - kb0 < KBS ? IT - kb0 : KBS;
                        // stage s is free in EVERY CTA of the cluster (kYCluster arrivals)
                        if (wrapped) mb_wait(b_empty + 8 * s, ph ^ 1u);
                        mb_expect_tx(b_full + 8 * s, (uint32_t)(nk * kYStageBytes));
                        const uint32_t dst = su32(ring + s * (KBS * kYStageBytes) + q * 128);
                        for (int kk = 0; kk < nk; ++kk)
                            tma2d_mc(dst + kk * kYStageBytes, &tmW, (kb0 + kk) * 128,
                                     it * 128 + q, b_full + 8 * s, all_mask);
                        if (++s == (uint32_t)NS) {
                            s = 0;
                            ph ^= 1u;
                            wrapped = true;
                        }
                    }
        }
    } else if (warp == 0) {
        // ---------------- MMA issuer
        if (lane == 0) {
            uint32_t s = 0, ph = 0, t = 0;
            const bool timed = A.timing != nullptr;
            unsigned long long w_a = 0, w_e = 0, w_f = 0, w_i = 0;
            long long c0 = timed ? clock64() : 0;
#define YT(acc_)                                    \
    do {                                            \
        if (timed) {                                \
            const long long c1_ = clock64();        \
            acc_ += (unsigned long long)(c1_ - c0); \
            c0 = c1_;                               \
        }                                           \
    } while (0)
            for (int64_t j = 0; j < nslots; ++j) {
                for (int it = 0; it < IT; ++it, ++t) {
                    const int d = t & 1;
                    if (t >= 2 && !(A.dbg & 64)) mb_wait(b_acce + 8 * d, ((t >> 1) - 1) & 1);
                    YT(w_e);
                    fence_after();
                    const uint32_t dcol = tmem + kYAcc0 + d * 128;
                    for (int kb0 = 0; kb0 < IT; kb0 += KBS) {
                        const int nk = IT - kb0 < KBS ? IT - kb0 : KBS;
                        if (it == 0 && !(A.dbg & 64)) {
                            // first use of this unit's A: its quarters must be in TMEM
                            for (int h = 0; h < 4; ++h)
                                if (kq(h) >= kb0 && kq(h) < kb0 + nk && kq(h) < kq(h + 1))
                                    mb_wait(b_ard + 8 * h, (uint32_t)(j & 1));
                            fence_after();
                            YT(w_a);
                        }
                        mb_wait(b_full + 8 * s, ph);
                        YT(w_f);
                        fence_after();
                        const uint64_t bd0 = sw128(su32(ring + s * (KBS * kYStageBytes)));
                        if (!(A.dbg & 2)) {
                            for (int kk = 0; kk < nk; ++kk) {
                                const int kb = kb0 + kk;
                                const uint64_t bd = bd0 + (uint64_t)((kk * kYStageBytes) >> 4);
#pragma unroll
                                for (int ks = 0; ks < 4; ++ks)  // K step 32 = 8 TMEM columns of A
                                    mma_ts(dcol, tmem + kb * 32 + ks * 8, bd + 2 * ks, A.idesc,
                                           (kb | ks) != 0);
                            }
                        }
                        commit_mc(b_empty + 8 * s, all_mask);
                        if (it == IT - 1)  // last use of this unit's A quarter: free it
                            for (int h = 0; h < 4; ++h)
                                if (kq(h + 1) - 1 >= kb0 && kq(h + 1) - 1 < kb0 + nk &&
                                    kq(h) < kq(h + 1))
                                    commit(b_kbf + 8 * h);
                        if (++s == (uint32_t)NS) {
                            s = 0;
                            ph ^= 1u;
                        }
                        YT(w_i);
                    }
                    commit(b_accf + 8 * d);
                }
            }
            if (timed) {
                atomicAdd(A.timing + 0, w_a);
                atomicAdd(A.timing + 1, w_e);
                atomicAdd(A.timing + 2, w_f);
                atomicAdd(A.timing + 3, w_i);
            }
        }
    } else if (warp >= kYEpiWarp0 && !(A.dbg & 64)) {
        // ---------------- generators + epilogue (16 warps)
        const int et = tid - kYEpiWarp0 * 32;           // 0..511
        const int q = warp & 3;                         // TMEM lane quadrant
        const int sub = (warp - kYEpiWarp0) >> 2;       // 0..3: column quarter
        const int r = q * 32 + lane;                    // A row / accumulator lane
        const int bl = r / p, l = r - bl * p;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        uint32_t t = 0;
        const bool timed = A.timing != nullptr && tid == kYEpiWarp0 * 32;
        unsigned long long e_st = 0, e_gen = 0, e_wait = 0, e_cmp = 0, e_red = 0, e_ld = 0;
        long long c0 = timed ? clock64() : 0;
#define ET(acc_)                                    \
    do {                                            \
        if (timed) {                                \
            const long long c1_ = clock64();        \
            acc_ += (unsigned long long)(c1_ - c0); \
            c0 = c1_;                               \
        }                                           \
    } while (0)
        // per-slot unit geometry
        auto slot_unit = [&](int64_t j, int64_t& bbase, int& nind) {
            const int64_t u = cs0 + j * kYCluster + crank;
            bbase = u * ipt;
            nind = u < cs1 ? (int)(A.B - bbase < ipt ? A.B - bbase : ipt) : 0;
        };
        // stage a unit's cluster rows into double buffer j & 1
        auto stage = [&](int64_t j) {
            int64_t bbase;
            int nind;
            slot_unit(j, bbase, nind);
            uint8_t* Cs = sC0 + (j & 1) * cb;
            const int chunks = A.npad / 16;
            for (int x = et; x < ipt * chunks; x += kYEpiThreads) {
                const int b2 = x / chunks, k = x - b2 * chunks;
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (b2 < nind)
                    v = __ldg(reinterpret_cast<const uint4*>(A.cl + (bbase + b2) * A.npad) + k);
                reinterpret_cast<uint4*>(Cs + (size_t)b2 * A.npad)[k] = v;
            }
        };
        // one-hot A of a unit into TMEM (row r = (bl, l), K = nodes); this warp
        // writes K blocks [kq(sub), kq(sub+1)) of its lane quadrant
        auto gen = [&](int64_t j) {
            int64_t bbase;
            int nind;
            slot_unit(j, bbase, nind);
            const uint8_t* Cs = sC0 + (j & 1) * cb;
            const bool live = r < ipt * p && bl < nind;
            const uint32_t lrep = (uint32_t)l * 0x01010101u;
            const uint4* crow = reinterpret_cast<const uint4*>(Cs + (size_t)(live ? bl : 0) * A.npad);
            for (int c0 = kq(sub) * 32; c0 < kq(sub + 1) * 32; c0 += 8) {
                uint32_t v[8];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint4 x = crow[(c0 >> 2) + h];  // 16 cluster ids = 4 columns
                    v[4 * h + 0] = live ? oh4(x.x, lrep) : 0u;
                    v[4 * h + 1] = live ? oh4(x.y, lrep) : 0u;
                    v[4 * h + 2] = live ? oh4(x.z, lrep) : 0u;
                    v[4 * h + 3] = live ? oh4(x.w, lrep) : 0u;
                }
                st8(tmem + lane_base + (uint32_t)c0, v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive(b_ard + 8 * sub);
        };

        if (nslots > 0) {
            stage(0);
            epi_sync();
            gen(0);
        }
        ET(e_st);
        // this thread's bin row: bins[k][r] at byte k * 512 + r * 4
        const uint32_t bin_r = su32(bins) + (uint32_t)r * 4u;
        for (int64_t j = 0; j < nslots; ++j) {
            int64_t bbase;
            int nind;
            slot_unit(j, bbase, nind);
            const bool live = r < ipt * p && bl < nind;
            const uint8_t* crow = sC0 + (j & 1) * cb + (size_t)(live ? bl : 0) * A.npad;
            if (j + 1 < nslots) {
                stage(j + 1);  // the next unit's cluster rows, under this unit's MMAs
                ET(e_st);
            }
            for (int it = 0; it < IT; ++it, ++t) {
                const int d = t & 1;
                if (j + 1 < nslots && it == IT - 1) {
                    // the next unit's one-hot, quarter by quarter as the last
                    // tile's MMAs release this unit's A
                    epi_sync();  // staging of j+1 complete
                    if (kq(sub) < kq(sub + 1)) {
                        mb_wait(b_kbf + 8 * sub, (uint32_t)(j & 1));
                        fence_after();
                    }
                    if (A.dbg & 4) {  // ablation: wait for the whole last tile
                        mb_wait(b_accf + 8 * d, (t >> 1) & 1);
                        fence_after();
                    }
                    gen(j + 1);
                    ET(e_gen);
                }
                mb_wait(b_accf + 8 * d, (t >> 1) & 1);
                ET(e_wait);
                fence_after();
                const uint32_t dcol = tmem + lane_base + kYAcc0 + d * 128 + sub * 32;
                uint32_t v0[16], v1[16];
                ld16(dcol, v0);
                ld16(dcol + 16, v1);
                // cluster ids of the 32 columns i = it*128 + sub*32 + k
                const uint4* cp = reinterpret_cast<const uint4*>(crow + it * 128 + sub * 32);
                const uint4 ca = cp[0], cz = cp[1];
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                ET(e_ld);
                fence_before();
                __syncwarp();
                if (lane == 0) mb_arrive(b_acce + 8 * d);  // accumulator may be overwritten
                if (live && !(A.dbg & 1)) {
                    // G[c_i][r] += D[r][i]: exact integer bins, this row's own
                    // (4 column-quarter warps share a row, hence the atomics)
                    const uint32_t cw[8] = {ca.x, ca.y, ca.z, ca.w, cz.x, cz.y, cz.z, cz.w};
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        const uint32_t c = __byte_perm(cw[k >> 2], 0u, 0x4440u + (k & 3));
                        const uint32_t dv = k < 16 ? v0[k] : v1[k - 16];
                        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(bin_r + c * 512u),
                                     "r"(dv)
                                     : "memory");
                    }
                }
                ET(e_cmp);
            }
            // S_T(b) = sum_l sum_k T_b[k][l] * G[k][(b,l)]; this thread takes
            // k = sub, sub + 4, ... of row r (fixed order -> deterministic).
            // The first 8 of its T values are fetched before the barrier.
            const uint32_t* tbp = A.T + (bbase + (live ? bl : 0)) * 2 * p * (int64_t)A.ps + l;
            uint32_t th[8], tl[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = sub + 4 * u;
                const bool ok = live && k < p;
                th[u] = ok ? __ldg(tbp + k * A.ps) : 0u;
                tl[u] = ok ? __ldg(tbp + (p + k) * A.ps) : 0u;
            }
            epi_sync();  // every bin of the unit is complete
            double s = 0.0;
            if (live) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int k = sub + 4 * u;
                    if (k < p) {
                        const uint32_t g = bins[k * 128 + r];
                        bins[k * 128 + r] = 0u;
                        s = fma((double)g, __hiloint2double((int)th[u], (int)tl[u]), s);
                    }
                }
                for (int k = sub + 32; k < p; k += 4) {
                    const uint32_t g = bins[k * 128 + r];
                    bins[k * 128 + r] = 0u;
                    s = fma((double)g,
                            __hiloint2double((int)__ldg(tbp + k * A.ps), (int)__ldg(tbp + (p + k) * A.ps)),
                            s);
                }
            }
            red[sub * 128 + r] = s;
            epi_sync();
            // one warp per individual: lanes stride its 4p partials, then a
            // butterfly (fixed order -> deterministic)
            for (int b2 = (warp - kYEpiWarp0); b2 < nind; b2 += kYEpiThreads / 32) {
                double acc = 0.0;
                for (int x = lane; x < 4 * p; x += 32) {
                    const int sq = x / p, ll = x - sq * p;
                    acc += red[sq * 128 + b2 * p + ll];
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                if (lane == 0) A.part[bbase + b2] = acc;
            }
            ET(e_red);
        }
        if (timed) {
            atomicAdd(A.timing + 16, e_st);
            atomicAdd(A.timing + 17, e_gen);
            atomicAdd(A.timing + 18, e_wait);
            atomicAdd(A.timing + 19, e_cmp);
            atomicAdd(A.timing + 20, e_red);
            atomicAdd(A.timing + 21, e_ld);
        }
    }
    fence_before();
    __syncthreads();
    cluster_sync_all();  // no CTA leaves while peers may still signal its barriers
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(kYTmemCols)
                     : "memory");
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static int y_ipt(int p) {
    int ipt = 128 / p;
    return ipt > kYMaxIpt ? kYMaxIpt : ipt;
}

static size_t y_fixed_bytes(int p, int npad) {  // everything but the W ring
    const int ipt = y_ipt(p);
    return 1024 + 2 * y_C_bytes(ipt, npad) + (size_t)p * 512 + 4 * 128 * 8 +
           (2 * kYMaxStages + 12) * 8 + 16;
}

// W ring depth: as deep as shared memory allows (TMA latency from L2 under load
// is well above the few hundred cycles one stage's MMAs take)
static int y_kbs() {
    const char* e = getenv("HUBGPU_TCY_KBS");  // tuning override
    const int k = e ? atoi(e) : 4;
    return k >= 1 && k <= 8 ? k : 4;
}

static int y_stages(int p, int npad) {
    const int64_t room = (int64_t)227 * 1024 - (int64_t)y_fixed_bytes(p, npad);
    int64_t s = room / ((int64_t)y_kbs() * kYStageBytes);
    if (s > kYMaxStages) s = kYMaxStages;
    const char* e = getenv("HUBGPU_TCY_STAGES");  // tuning override (shallower only)
    if (e && atoi(e) >= 2 && atoi(e) < s) s = atoi(e);
    return (int)s;
}

size_t tcy_smem_bytes(int p, int npad) {
    return y_fixed_bytes(p, npad) + (size_t)y_stages(p, npad) * y_kbs() * kYStageBytes;
}

bool tcy_supported(int n, int p, int npad) {
    return p >= 1 && p <= 128 && round_up(n, 128) <= 1024 && npad <= 1024 &&
           y_stages(p, npad) >= 2;
}

static int g_tcy_clusters = 0;  // co-resident clusters (cudaOccupancyMaxActiveClusters)

int prepare_fitness_tcy(int p, int npad) {
    HG_CUDA(cudaFuncSetAttribute(k_fitness_tcy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tcy_smem_bytes(p, npad)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kYCluster);
    cfg.blockDim = dim3(kYThreads);
    cfg.dynamicSmemBytes = tcy_smem_bytes(p, npad);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kYCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    HG_CUDA(cudaOccupancyMaxActiveClusters(&nc, k_fitness_tcy, &cfg));
    g_tcy_clusters = nc;
    return HG_OK;
}

int launch_fitness_tcy(const DevInst& I, const void* wmap, int64_t B, const uint8_t* cl,
                       const uint32_t* T, double* part, int grid, cudaStream_t s) {
    if (B <= 0) return HG_OK;
    YArgs A;
    A.cl = cl;
    A.T = T;
    A.part = part;
    A.B = B;
    A.n = I.n;
    A.p = I.p;
    A.ps = I.ps;
    A.npad = I.npad;
    A.ipt = y_ipt(I.p);
    A.units = ceil_div(B, A.ipt);
    A.IT = (int)(round_up(I.n, 128) / 128);
    A.acols = A.IT * 32;
    A.stages = y_stages(I.p, I.npad);
    A.kbs = y_kbs();
    A.idesc = (2u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    A.timing = tc_timing_buffer();
    {
        const char* e = getenv("HUBGPU_TCY_DBG");
        A.dbg = e ? atoi(e) : 0;
    }
    // whole clusters only, all co-resident (one wave): the GPCs need not hold a
    // multiple of the cluster size, so ask the occupancy API
    int g = (g_tcy_clusters > 0 ? g_tcy_clusters : grid / kYCluster) * kYCluster;
    const int64_t need = round_up(A.units, kYCluster);
    if (g > need) g = (int)need;
    if (g < kYCluster) g = kYCluster;
    CUtensorMap map = *static_cast<const CUtensorMap*>(wmap);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(kYThreads);
    cfg.dynamicSmemBytes = tcy_smem_bytes(I.p, I.npad);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kYCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HG_CUDA(cudaLaunchKernelEx(&cfg, k_fitness_tcy, map, A));
    return HG_OK;
}

}  // namespace hg
