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
constexpr int kYStages = 6;                   // W ring depth
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
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                      uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(bar)
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
// byte-wise (x == l) -> 0x80 / 0x00 (see k_fitness_tc.cu)
__device__ __forceinline__ uint32_t oh4(uint32_t x, uint32_t lrep) {
    const uint32_t y = x ^ lrep;
    const uint32_t t = (y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    return ~(t | y) & 0x80808080u;
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
    int pss;          // staged T row stride (doubles)
    uint32_t idesc;   // kind::i8, M=128, N=128, K-major both
    unsigned long long* timing;  // optional phase counters (HUBGPU_TC_TIMING=1)
    int dbg;                     // ablation flags (tuning only): 1 = no epilogue math, 2 = no MMA
};

__host__ __device__ inline size_t y_T_bytes(int ipt, int p, int pss) {
    return ((size_t)ipt * p * pss * 8 + 15) & ~size_t(15);
}
__host__ __device__ inline size_t y_C_bytes(int ipt, int npad) {
    return ((size_t)ipt * npad + 15) & ~size_t(15);
}
__host__ __device__ inline size_t y_O_bytes(int ipt, int npad) {  // u16 T-row offsets
    return ((size_t)ipt * npad * 2 + 15) & ~size_t(15);
}

__global__ void __launch_bounds__(kYThreads, 1)
k_fitness_tcy(const __grid_constant__ CUtensorMap tmW, YArgs A) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const int p = A.p, ipt = A.ipt, IT = A.IT;
    unsigned char* ring = smem;                                          // W stages
    unsigned char* var = smem + kYStages * kYStageBytes;
    const size_t tb = y_T_bytes(ipt, p, A.pss), cb = y_C_bytes(ipt, A.npad);
    // double buffers addressed arithmetically from the shared base (a pointer
    // array indexed at run time would drop to local memory and generic loads)
    unsigned char* sT0 = var;
    var += 2 * tb;
    unsigned char* sC0 = var;
    var += 2 * cb;
    const size_t ob = y_O_bytes(ipt, A.npad);
    unsigned char* sO0 = var;
    var += 2 * ob;
    double* red = reinterpret_cast<double*>(var);  // [4 subs][128 rows]
    var += 4 * 128 * 8;
    uint64_t* bars = reinterpret_cast<uint64_t*>(var);
    // bars: full[6] empty[6] accfull[2] accempty[2] aready[1]
    const uint32_t b_full = su32(bars), b_empty = b_full + 8 * kYStages,
                   b_accf = b_empty + 8 * kYStages, b_acce = b_accf + 16, b_ard = b_acce + 16;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kYStages + 5);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kYStages; ++s) {
            mb_init(b_full + 8 * s, 1);
            mb_init(b_empty + 8 * s, kYCluster);  // every consumer CTA of the cluster
        }
        for (int d = 0; d < 2; ++d) {
            mb_init(b_accf + 8 * d, 1);
            mb_init(b_acce + 8 * d, kYWarps - kYEpiWarp0);
        }
        mb_init(b_ard, kYWarps - kYEpiWarp0);
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
        // ---------------- TMA producer: W tiles (it, kb), same order every unit
        if (lane == 0) {
            uint32_t g = 0;
            for (int64_t j = 0; j < nslots; ++j)
                for (int it = 0; it < IT; ++it)
                    for (int kb = 0; kb < IT; ++kb, ++g) {
                        const int s = g % kYStages;
                        // stage s is free in EVERY CTA of the cluster (kYCluster arrivals)
                        if (g >= kYStages) mb_wait(b_empty + 8 * s, ((g / kYStages) - 1) & 1);
                        mb_expect_tx(b_full + 8 * s, kYStageBytes);
                        const int q = (int)crank * (128 / kYCluster);
                        tma2d_mc(su32(ring + s * kYStageBytes + q * 128), &tmW, kb * 128,
                                 it * 128 + q, b_full + 8 * s, all_mask);
                    }
        }
    } else if (warp == 0) {
        // ---------------- MMA issuer
        if (lane == 0) {
            uint32_t g = 0, t = 0;
            unsigned long long w_a = 0, w_e = 0, w_f = 0, w_i = 0;
            long long c0 = clock64();
#define YT(acc_)                                    \
    do {                                            \
        const long long c1_ = clock64();            \
        acc_ += (unsigned long long)(c1_ - c0);     \
        c0 = c1_;                                   \
    } while (0)
            for (int64_t j = 0; j < nslots; ++j) {
                mb_wait(b_ard, (uint32_t)(j & 1));  // A of this unit is in TMEM
                YT(w_a);
                fence_after();
                for (int it = 0; it < IT; ++it, ++t) {
                    const int d = t & 1;
                    if (t >= 2) mb_wait(b_acce + 8 * d, ((t >> 1) - 1) & 1);
                    YT(w_e);
                    fence_after();
                    const uint32_t dcol = tmem + kYAcc0 + d * 128;
                    for (int kb = 0; kb < IT; ++kb, ++g) {
                        const int s = g % kYStages;
                        mb_wait(b_full + 8 * s, (g / kYStages) & 1);
                        YT(w_f);
                        fence_after();
                        const uint64_t bd = sw128(su32(ring + s * kYStageBytes));
                        if (!(A.dbg & 2)) {
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks)  // K step 32 = 8 TMEM columns of A
                                mma_ts(dcol, tmem + kb * 32 + ks * 8, bd + 2 * ks, A.idesc,
                                       (kb | ks) != 0);
                        }
                        commit_mc(b_empty + 8 * s, all_mask);
                        YT(w_i);
                    }
                    commit(b_accf + 8 * d);
                }
            }
            if (A.timing) {
                atomicAdd(A.timing + 0, w_a);
                atomicAdd(A.timing + 1, w_e);
                atomicAdd(A.timing + 2, w_f);
                atomicAdd(A.timing + 3, w_i);
            }
        }
    } else if (warp >= kYEpiWarp0) {
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
        // stage a unit's T tables (x 2^-7, zero tails), cluster rows and the
        // epilogue's T-row offsets into double buffer `buf`
        auto stage = [&](int64_t j) {
            int64_t bbase;
            int nind;
            slot_unit(j, bbase, nind);
            const int buf = (int)(j & 1);
            double* Ts = reinterpret_cast<double*>(sT0 + buf * tb);
            uint8_t* Cs = sC0 + buf * cb;
            uint16_t* Os = reinterpret_cast<uint16_t*>(sO0 + buf * ob);
            const int pss = A.pss, per = p * pss;
            for (int x = et; x < ipt * per; x += kYEpiThreads) {
                const int b2 = x / per, y = x - b2 * per;
                const int c = y / pss, ll = y - c * pss;
                double v = 0.0;
                if (b2 < nind && ll < p) {
                    const uint32_t* tbp = A.T + (bbase + b2) * 2 * p * (int64_t)A.ps;
                    v = __hiloint2double((int)tbp[c * A.ps + ll], (int)tbp[(p + c) * A.ps + ll]) *
                        0.0078125;
                }
                Ts[(b2 * p + c) * pss + ll] = v;
            }
            const int chunks = A.npad / 16;
            for (int x = et; x < ipt * chunks; x += kYEpiThreads) {
                const int b2 = x / chunks, k = x - b2 * chunks;
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (b2 < nind)
                    v = __ldg(reinterpret_cast<const uint4*>(A.cl + (bbase + b2) * A.npad) + k);
                reinterpret_cast<uint4*>(Cs + (size_t)b2 * A.npad)[k] = v;
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                uint32_t o[8];
#pragma unroll
                for (int h = 0; h < 8; ++h) {
                    const uint32_t ca = (w[h >> 1] >> ((h & 1) * 16)) & 0xffu;
                    const uint32_t cz = (w[h >> 1] >> ((h & 1) * 16 + 8)) & 0xffu;
                    o[h] = (ca * A.pss) | ((cz * A.pss) << 16);
                }
                uint4* od = reinterpret_cast<uint4*>(Os + (size_t)b2 * A.npad + k * 16);
                od[0] = make_uint4(o[0], o[1], o[2], o[3]);
                od[1] = make_uint4(o[4], o[5], o[6], o[7]);
            }
        };
        // one-hot A of a unit into TMEM (row r = (bl, l), K = nodes); this warp
        // writes columns [sub * acols/4, (sub+1) * acols/4) of its lane quadrant
        auto gen = [&](int64_t j) {
            int64_t bbase;
            int nind;
            slot_unit(j, bbase, nind);
            const uint8_t* Cs = sC0 + (j & 1) * cb;
            const bool live = r < ipt * p && bl < nind;
            const uint32_t lrep = (uint32_t)l * 0x01010101u;
            const int cq = A.acols / 4;
            const uint4* crow = reinterpret_cast<const uint4*>(Cs + (size_t)(live ? bl : 0) * A.npad);
            for (int c0 = sub * cq; c0 < (sub + 1) * cq; c0 += 8) {
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
            if (lane == 0) mb_arrive(b_ard);
        };

        if (nslots > 0) {
            stage(0);
            epi_sync();
            gen(0);
        }
        ET(e_st);
        for (int64_t j = 0; j < nslots; ++j) {
            int64_t bbase;
            int nind;
            slot_unit(j, bbase, nind);
            const double* Ts = reinterpret_cast<const double*>(sT0 + (j & 1) * tb);
            const uint16_t* Os = reinterpret_cast<const uint16_t*>(sO0 + (j & 1) * ob);
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            const double* trow = Ts + (size_t)(r < ipt * p ? bl * p : 0) * A.pss + l;
            const uint16_t* orow = Os + (size_t)(bl < ipt ? bl : 0) * A.npad;
            for (int it = 0; it < IT; ++it, ++t) {
                const int d = t & 1;
                mb_wait(b_accf + 8 * d, (t >> 1) & 1);
                ET(e_wait);
                fence_after();
                const uint32_t dcol = tmem + lane_base + kYAcc0 + d * 128 + sub * 32;
                uint32_t v0[16], v1[16];
                ld16(dcol, v0);
                ld16(dcol + 16, v1);
                // T-row offsets of the 32 columns i = it*128 + sub*32 + k
                const uint4* op = reinterpret_cast<const uint4*>(orow + it * 128 + sub * 32);
                const uint4 o0 = op[0], o1 = op[1], o2 = op[2], o3 = op[3];
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                ET(e_ld);
                fence_before();
                __syncwarp();
                if (lane == 0) mb_arrive(b_acce + 8 * d);  // accumulator may be overwritten
                // next unit: staged early, its one-hot generated as soon as this
                // unit's last MMAs are complete (this wait), so the tensor core
                // starts on it while we finish this unit's epilogue
                if (j + 1 < nslots) {
                    if (it == 0) {
                        stage(j + 1);
                        ET(e_st);
                    }
                    if (it == IT - 1) {
                        epi_sync();  // staging of j+1 complete
                        gen(j + 1);
                        ET(e_gen);
                    }
                }
                const uint32_t ow[16] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w,
                                         o2.x, o2.y, o2.z, o2.w, o3.x, o3.y, o3.z, o3.w};
                if (A.dbg & 1) {
                    acc[0] += (double)(v0[0] + v1[15] + ow[3]);
                    continue;
                }
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const uint32_t off = (k & 1) ? (ow[k >> 1] >> 16) : (ow[k >> 1] & 0xffffu);
                    const uint32_t dv = k < 16 ? v0[k] : v1[k - 16];
                    const double dd = __hiloint2double(0x43300000, (int)dv) - 4503599627370496.0;
                    acc[k & 3] = fma(dd, trow[off], acc[k & 3]);
                }
                ET(e_cmp);
            }
            const double acc0 = acc[0] + acc[1], acc1 = acc[2] + acc[3];
            // per-individual sum over its p rows and the 4 column quarters (fixed order)
            red[sub * 128 + r] = acc0 + acc1;
            epi_sync();
            for (int b2 = et; b2 < nind; b2 += kYEpiThreads) {
                double s = 0.0;
                for (int sq = 0; sq < 4; ++sq)
                    for (int ll = 0; ll < p; ++ll) s += red[sq * 128 + b2 * p + ll];
                A.part[bbase + b2] = s;
            }
            epi_sync();
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

static int y_pss(int p) { return ((p + 7) & ~7) + 2; }

static int y_ipt(int p) {
    int ipt = 128 / p;
    return ipt > kYMaxIpt ? kYMaxIpt : ipt;
}

size_t tcy_smem_bytes(int p, int npad) {
    const int ipt = y_ipt(p);
    size_t b = 1024 + (size_t)kYStages * kYStageBytes;
    b += 2 * y_T_bytes(ipt, p, y_pss(p)) + 2 * y_C_bytes(ipt, npad) + 2 * y_O_bytes(ipt, npad);
    b += 4 * 128 * 8 + (2 * kYStages + 5) * 8 + 16;
    return b;
}

bool tcy_supported(int n, int p, int npad) {
    return p >= 1 && p <= 128 && round_up(n, 128) <= 1024 && npad <= 1024 &&
           tcy_smem_bytes(p, npad) <= 227 * 1024;
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
    A.pss = y_pss(I.p);
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
