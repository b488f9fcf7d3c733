// K3-TC/P: K3-TC/Y (k_fitness_tcy.cu) on a CTA PAIR -- tcgen05 with
// cta_group::2 (hm/evaluation.py:113-119 transfer term).
//
// Two CTAs on one TPC each hold their own unit (ipt individuals, one-hot A in
// their own TMEM lanes 0..127, integer bins, epilogue) and issue ONE stream of
// M=256 MMAs from the leader CTA: each W tile (B operand, N = 128 W rows) is
// split by rows across the pair -- each CTA TMA-loads and keeps only its 64
// rows, and the tensor cores exchange the halves.  Per SM that halves both the
// W bytes streamed from L2 and the shared-memory traffic of B, which bound the
// single-CTA kernel.  Barrier protocol (leader = cluster rank 0):
//   full[s]   leader's; both CTAs' TMA complete_tx into it, leader expects both halves
//   empty[s]  each CTA's; released by the leader's multicast tcgen05.commit
//   accf[d]   each CTA's (multicast commit); acce[d] leader's, 2 x 16 epilogue warps arrive
//   kbf[h]    each CTA's (multicast commit); ard[h] leader's, 2 x 4 generator warps arrive
//
// Any n: the K dimension is cut into chunks of 1024 nodes (the 256 TMEM
// columns of a resident one-hot).  Integer bins are linear in D, so every
// (chunk, output tile) accumulator drains into them independently, and a
// chunk's bins are folded into S_T (p fp64 FMAs per row) before the next
// chunk -- no accumulator ever spans chunks.
//
#include <cuda.h>
#include <cuda_pipeline.h>

#include <cstdlib>

#include <algorithm>
#include <cmath>

#include "hg_internal.cuh"

namespace hg {

namespace {

// warp 0 issues the MMAs, warp 1 the W loads, warps 2-3 idle, warps 4..19 are
// the epilogue (warp w reaches TMEM lanes 32 (w % 4) ..).  Registers: 96 per
// thread -- each SM sub-partition holds 5 of the 20 warps (16384 / 5 / 32)
constexpr int kYThreads = 640;
constexpr int kYWarps = kYThreads / 32;
constexpr int kYEpiWarp0 = 4;                                 // first epilogue warp
constexpr int kYEpiThreads = kYThreads - 32 * kYEpiWarp0;     // 512
constexpr int kYMaxStages = 16;               // W ring depth bound (runtime: PArgs::stages)
constexpr int kYStageBytes = 64 * 128;        // this CTA's 64 W rows x 128 K (u8)
constexpr int kYMaxIpt = 32;
constexpr int kYTmemCols = 512;
constexpr int kYAcc0 = 256;                   // first accumulator column
constexpr int kYCluster = 2;                  // the CTA pair
constexpr int kYMaxPlanes = 4;                // byte planes one launch folds together
// phase counters (HUBGPU_TC_TIMING=1) only in a timing build
// (make EXTRA=-DHG_TCP_TIMING): their accumulators cost registers
#ifdef HG_TCP_TIMING
constexpr bool kTimingBuild = true;
#else
constexpr bool kTimingBuild = false;
#endif
// timing build: an event trace of CTA 0 (clock64 stamps, code in the top
// byte) at timing[64 + role * kTraceLen ..]; roles 0 = MMA issuer, 1 = epilogue
// warp 4 (lane quadrant 0, column quarter 0), 2 = epilogue warp 19 (3, 3)
constexpr int kTraceLen = 8192;
#define TRC(role_, code_)                                                                   \
    do {                                                                                    \
        if (kTimingBuild && tr_on && tr_n < kTraceLen)                                      \
            A.timing[64 + (role_) * kTraceLen + tr_n++] =                                   \
                ((unsigned long long)(code_) << 56) | ((unsigned long long)clock64() & ((1ull << 56) - 1)); \
    } while (0)

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
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ bool mb_try(uint32_t bar, uint32_t parity) {  // non-blocking
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAITQ_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAITQ_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// this CTA's half of a W tile into its own shared memory; the bytes are
// counted on the LEADER's mbarrier (a shared::cluster address)
__device__ __forceinline__ void tma2d_pair(uint32_t dst, const CUtensorMap* map, int x, int y,
                                           uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(bar_cluster)
        : "memory");
}
// arrive on the mbarrier at this offset in both CTAs of the pair once the
// issued MMAs have completed
__device__ __forceinline__ void commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar),
        "h"((uint16_t)3)
        : "memory");
}
// the same, issued by one elected lane of a converged warp (the MMA warp runs
// its loop warp-uniformly, so descriptors stay in uniform registers)
__device__ __forceinline__ void commit_pair_w(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n\t}" ::"r"(bar),
        "h"((uint16_t)3)
        : "memory");
}
// shared::cluster address of the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mb_arrive(uint32_t bar) {  // release.cta
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// arrive once every cp.async this thread issued so far has landed (the
// barrier counts one arrival per thread: .noinc)
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void mb_wait_cl(uint32_t bar, uint32_t parity) {  // acquire.cluster
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAITP_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAITP_%=;\n\t}" ::"r"(bar),
        "r"(parity)
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
// D[tmem] (+)= A[tmem] . B[smem]^T, kind::i8, M = 256 over the pair (leader issues)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
// a K block's four K=32 MMAs (A columns a, a+8, a+16, a+24; B descriptors
// bdesc + 0, 2, 4, 6 -- 32 bytes apart in the 128-byte swizzled rows) from one
// elected lane: one election and one descriptor set-up for the four
__device__ __forceinline__ void mma4_ts_w(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {  // acc: the first MMA accumulates
    asm volatile(
        "{\n\t.reg .pred p, t, e;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b32 a1, a2, a3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 t, %4, %4;\n\t"
        "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], [a1], b1, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], [a2], b2, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], [a3], b3, %3, t;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
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

// one row's share of a plane's fold: s += sum_k G[k] * T[k][l] * sc over
// k = sub, sub + 4, ... (fixed order), zeroing the bins; out of line -- the
// epilogue's tile loop is register-bound
// lsym >= 0 (symmetric costs, the table's upper triangle only): T[k][l] for
// k > lsym = l is read as T[l][k]
__device__ __noinline__ double fold_bins(uint32_t* bp, const double* tbd, const uint32_t* tbp,
                                         int p, int ps, int sub, double sc, double s,
                                         int lsym = -1) {
    const double* trow = tbd && lsym >= 0 ? tbd - lsym + lsym * p : nullptr;
    auto tv = [&](int k) {
        return trow && k > lsym ? trow[k]
               : tbd        ? tbd[k * p]
                            : __hiloint2double((int)tbp[k * ps], (int)tbp[(p + k) * ps]);
    };
    int k = sub;
    // four bins at a time, their loads issued together (same summation order)
    for (; k + 12 < p; k += 16) {
        const uint32_t g0 = bp[k * 128], g1 = bp[(k + 4) * 128], g2 = bp[(k + 8) * 128],
                       g3 = bp[(k + 12) * 128];
        const double t0 = tv(k), t1 = tv(k + 4), t2 = tv(k + 8), t3 = tv(k + 12);
        bp[k * 128] = 0u;
        bp[(k + 4) * 128] = 0u;
        bp[(k + 8) * 128] = 0u;
        bp[(k + 12) * 128] = 0u;
        s = fma((double)g0, t0 * sc, s);
        s = fma((double)g1, t1 * sc, s);
        s = fma((double)g2, t2 * sc, s);
        s = fma((double)g3, t3 * sc, s);
    }
    for (; k < p; k += 4) {
        const uint32_t g = bp[k * 128];
        bp[k * 128] = 0u;
        s = fma((double)g, tv(k) * sc, s);
    }
    return s;
}

}  // namespace

__host__ __device__ inline size_t p_C_bytes(int ipt, int npad) {
    return ((size_t)ipt * npad + 15) & ~size_t(15);
}
__host__ __device__ inline size_t p_T_bytes(int ipt, int p) {
    return (size_t)ipt * p * p * 8;
}
__host__ __device__ inline size_t p_H_bytes(int ipt, int p) {  // 3 buffers (defer)
    return ((size_t)3 * ipt * p * 4 + 15) & ~size_t(15);
}

struct PArgs {
    const int32_t* dB;   // device-side batch size bounding B (nullptr: B)
    const uint8_t* cl;
    const uint32_t* T;   // K2's hub-cost tables (read when !tsm)
    const int32_t* hubs; // [B][p] sorted hubs (tsm: T_b gathered from C here)
    const double* C;     // the cost matrix, n x n
    int nC;
    double* part;     // [B][1]: S_T complete per individual (when out is null)
    const double* legs;  // [B][2] spoke-leg sums from K2 (finalise fused when out is set)
    double* out;         // [B][4] collection, transfer, distribution, raw
    double chi, alpha, delta;
    int64_t B;
    int n, p, ps, npad;
    int ipt;          // individuals per unit (ipt * p <= 128)
    int64_t units;
    int ITO;          // 128-row W tiles (output columns i)
    int P;            // byte planes of W (flows < 256^P): tiles per phase = P * ITO
    int nt;           // W rows per plane in the stacked u8 tensor
    int KBT;          // 128-node K blocks in all
    int NC;           // K chunks of <= 8 blocks (1024 nodes): one resident one-hot each
    int stages;       // W ring depth
    int kbs;          // 128-byte K blocks per stage
    // tri: the W tensor is the block-upper-triangular fold of a symmetric-cost
    // instance (diagonal blocks W, blocks above W + W^T, below unused): output
    // tile I runs K blocks J >= I only (see k_fitness_tcp's header)
    int tri;
    int csm;          // 1: a unit's cluster rows are staged in shared memory (they fit)
    int tsm;          // 1: a unit's hub-cost tables T_b[k][l] = C[h_k][h_l] are gathered
                      // from C into shared memory by cp.async (K2 writes none)
    // plane0: the first byte plane this launch reads (instances with more than
    // 4 planes run one launch per plane, each writing its partial S_T to part
    // with stride pstride); wscale: the weight of plane plane0 -- the flows'
    // power-of-two quantum times 256^plane0 (plane pl weighs 256^pl * that)
    int plane0, pstride;
    double wscale;
    uint32_t idesc;   // kind::i8, M=256, N=128, K-major both
    unsigned long long* timing;  // optional phase counters (HUBGPU_TC_TIMING=1)
    // ablation flags (tuning only, wrong results): 1 = no bin atomics, 2 = no
    // MMA, 4 = no chunk fold / unit reduce, 8 = no one-hot generation, 16 = the
    // MMA issuer does not wait for W (only together with 32: the ring's
    // barriers race otherwise), 32 = no W stream, 64 = no epilogue warps at all
    int dbg;
    // exact: one chunk and one plane, so the bins ARE the reference's
    // inter-cluster flows; S_T is then np.sum(inter * hub_dist) replayed in
    // numpy's pairwise order over the leaves of the p*p-term sum
    int exact;
    // defer (one K chunk, >= 4 output tiles, !exact): a unit's bins, partials,
    // T tables are double-buffered and its fold / reduce run during the next
    // unit's tiles, ordered by mbarriers instead of epilogue-wide barriers; the
    // cluster rows are triple-buffered and staged by cp.async
    int defer;
    const uint32_t* leaves;  // per leaf: first row | rows << 16 | tree sums << 24
    int nleaf;
};

constexpr int kYChunkKB = 8;  // K blocks per chunk: 8 x 128 nodes = 256 TMEM columns of A
// instruction descriptor: kind::i8, u8 x u8 -> s32, M = 256 (the pair), N = 128,
// both operands K-major (a compile-time constant: no per-MMA constant loads)
constexpr uint32_t kIdescI8 = (2u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
constexpr int kYDeferBars = 13;  // binsdone[2] folded[2] tready[2] cready[3] reduced[2] tgath[2]

// CSM: a unit's cluster rows staged in shared memory (known address space ->
// LDS) rather than read from global memory
template <bool CSM, bool EX, bool DFT = false>
__global__ void __launch_bounds__(kYThreads, 1)
k_fitness_tcp(const __grid_constant__ CUtensorMap tmW, PArgs A) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const int p = A.p, ipt = A.ipt, ITO = A.ITO, KBT = A.KBT, NC = A.NC;
    unsigned char* ring = smem;                                          // W stages
    const int NS = A.stages, KBS = A.kbs;
    unsigned char* var = smem + NS * KBS * kYStageBytes;
    // cluster rows of the current / next unit, when they fit (CSM); a double
    // buffer addressed arithmetically (a runtime-indexed pointer array would
    // drop to local memory)
    constexpr bool DF = !EX && DFT;  // (launched only with A.defer)
    const int NB = DF ? 2 : 1;  // bins / partials / T-table buffers
    const size_t cb = CSM ? p_C_bytes(ipt, A.npad) : 0;
    unsigned char* sC0 = var;
    var += (DF ? 3 : 2) * cb;
    const int PB = A.P;  // planes of bins
    // [NB][PB][p][128] cluster-pair flow bins
    uint32_t* bins = reinterpret_cast<uint32_t*>(var);
    var += (size_t)NB * PB * p * 512;
    double* red = reinterpret_cast<double*>(var);  // [NB][4 subs][128 rows]
    var += (size_t)NB * 4 * 128 * 8;
    // the unit's spoke-leg sums (finaliser), by slot parity: [2][ipt][2]
    double* sL = reinterpret_cast<double*>(var);
    var += 2 * kYMaxIpt * 2 * 8;
    // the unit's hub-cost tables T (tsm): [ipt][p][p] fp64, and its hubs (and
    // the next units': 2 buffers, defer 3) [3][ipt][p] int32
    double* sT = reinterpret_cast<double*>(var);  // [NB][ipt][p][p]
    var += A.tsm ? NB * p_T_bytes(ipt, p) : 0;
    int32_t* sH = reinterpret_cast<int32_t*>(var);
    var += A.tsm ? p_H_bytes(ipt, p) : 0;
    double* prod = reinterpret_cast<double*>(var);  // exact: [p][128] rounded terms of S_T
    var += EX ? (size_t)p * 128 * 8 : 0;
    uint64_t* bars = reinterpret_cast<uint64_t*>(var);
    // bars: full[16] empty[16] accfull[2] accempty[2] kbfree[4] aready[4], and
    // (defer) binsdone[2] folded[2] tready[2] cready[3] reduced[2]
    const uint32_t b_full = su32(bars), b_empty = b_full + 8 * kYMaxStages,
                   b_accf = b_empty + 8 * kYMaxStages, b_acce = b_accf + 16, b_kbf = b_acce + 16,
                   b_ard = b_kbf + 32, b_bdone = b_ard + 32, b_fold = b_bdone + 16,
                   b_tready = b_fold + 16, b_cready = b_tready + 16, b_rdone = b_cready + 24,
                   b_tgath = b_rdone + 16;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kYMaxStages + 12 + kYDeferBars);
    // chunk c of the K dimension: K blocks [c*8, c*8 + nkb(c)); its one-hot is
    // generated in 4 contiguous ranges of K blocks, one per column-quarter warp
    // group: quarter h owns chunk-local blocks [kq(c,h), kq(c,h+1))
    auto nkb = [&](int c) { return KBT - c * kYChunkKB < kYChunkKB ? KBT - c * kYChunkKB : kYChunkKB; };
    auto kq = [&](int c, int h) { return h * nkb(c) / 4; };
    // output tiles of chunk c (per plane), the first chunk-local K block of
    // tile I, and the tile holding the last use of chunk-local block k
    const int tri = A.tri;
    auto ntl = [&](int c) {
        return tri && c * kYChunkKB + nkb(c) < ITO ? c * kYChunkKB + nkb(c) : ITO;
    };
    auto klo = [&](int c, int I) { return tri && I > c * kYChunkKB ? I - c * kYChunkKB : 0; };
    auto klast = [&](int c, int k) { return tri ? c * kYChunkKB + k : ntl(c) - 1; };
    // the block whose last use frees A quarter h (an empty quarter: the block
    // before it) -- every kbf[h] completes exactly once per phase
    auto qrb = [&](int c, int h) {
        return kq(c, h) < kq(c, h + 1) ? kq(c, h + 1) - 1 : (kq(c, h) > 0 ? kq(c, h) - 1 : 0);
    };
    // HG_QSPLIT=1 (deferred fold, triangular fold): the last quarter -- freed
    // only by a unit's last tile, needed soon after by the next unit's first --
    // generated by the four column-quarter warps of a lane quadrant, 1/4 each,
    // its ready barrier counting 4x.  Parity-green but measured slower (0.1178
    // vs 0.1167 ms, tools/ab_k3.py): off
#ifndef HG_QSPLIT
#define HG_QSPLIT 0
#endif
    const bool qsplit = HG_QSPLIT && DF && tri && NC == 1 && kq(0, 3) < kq(0, 4);
    // 32-bit TMEM columns [lo, hi) of part s_ of the last quarter
    auto q3part = [&](int s_, int& lo, int& hi) {
        const int base = kq(0, 3) * 32, n8 = (kq(0, 4) - kq(0, 3)) * 4;
        lo = base + 8 * (n8 * s_ / 4);
        hi = base + 8 * (n8 * (s_ + 1) / 4);
    };

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int x = tid; x < NB * PB * p * 128; x += kYThreads) bins[x] = 0u;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mb_init(b_full + 8 * s, 1);
            mb_init(b_empty + 8 * s, 1);
        }
        for (int d = 0; d < 2; ++d) {
            mb_init(b_accf + 8 * d, 1);
            mb_init(b_acce + 8 * d, 2 * (kYWarps - kYEpiWarp0));  // both CTAs' epilogues
        }
        for (int h = 0; h < 4; ++h) {
            mb_init(b_kbf + 8 * h, 1);
            // the 4 lane-quadrant warps of quarter h, both CTAs (qsplit: all 16 for the last)
            mb_init(b_ard + 8 * h, h == 3 && qsplit ? 32 : 8);
        }
        for (int x = 0; x < 2; ++x) {
            mb_init(b_bdone + 8 * x, kYEpiThreads / 32);  // a warp's last atomics of a unit
            mb_init(b_fold + 8 * x, kYEpiThreads / 32);   // a warp's fold of a unit
            mb_init(b_tready + 8 * x, kYEpiThreads);      // every thread's cp.async (noinc)
        }
        for (int x = 0; x < 3; ++x) mb_init(b_cready + 8 * x, kYEpiThreads);
        for (int x = 0; x < 2; ++x) {
            mb_init(b_rdone + 8 * x, 2);   // warps 2-3
            mb_init(b_tgath + 8 * x, 64);  // warps 2-3's cp.async (noinc), a unit's T
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(tmem_slot)),
                     "r"(kYTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    cluster_sync_all();  // the peer's barriers are initialised before any remote signal
    const uint32_t tmem = *tmem_slot;
#ifdef HG_CHECKS
    if (tid == 0) {
        uint32_t dyn;
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        const size_t used = (size_t)(reinterpret_cast<unsigned char*>(tmem_slot + 1) - smem_raw);
        HG_DCHECK(used <= dyn, "K3 shared layout %llu B past the %u B launched",
                  (unsigned long long)used, dyn);
        HG_DCHECK(PB * p * 128 * 4 + (size_t)(reinterpret_cast<unsigned char*>(bins) - smem) <=
                      (size_t)dyn, "K3 bins past the launched shared memory");
    }
#endif

    // units of this pair, interleaved over its 2 CTAs; both run the same number
    // of slots (a slot past the end is a dummy unit): one MMA stream serves both.
    // A phase is (slot, chunk): one resident one-hot, ITO output tiles.
    const uint32_t crank = cluster_rank();
    const int64_t ncl = gridDim.x / kYCluster, cid = blockIdx.x / kYCluster;
    // the batch: the host's, or a device-side count bounding it (the GA's
    // distinct hub sets); units of ipt individuals
    const int64_t Bk = A.dB ? (int64_t)*A.dB : A.B;
    const int64_t units = A.dB ? (Bk + ipt - 1) / ipt : A.units;
    const int64_t cs0 = units * cid / ncl, cs1 = units * (cid + 1) / ncl;
    const int64_t nslots = (cs1 - cs0 + kYCluster - 1) / kYCluster;
    const bool leader = crank == 0;
    // the leader's barriers as shared::cluster addresses (remote for the peer)
    const uint32_t L_full = mapa(b_full, 0), L_acce = mapa(b_acce, 0), L_ard = mapa(b_ard, 0);

    // per-slot unit geometry: the first individual and the count (0: a dummy
    // slot past the pair's units)
    auto slot_unit = [&](int64_t j, int64_t& bbase, int& nind) {
        const int64_t u = cs0 + j * kYCluster + crank;
        bbase = u * ipt;
        nind = u < cs1 ? (int)(Bk - bbase < ipt ? Bk - bbase : ipt) : 0;
    };

    // a unit's S_T reduce + the finaliser (fixed order): one warp per
    // individual b2 = first, first + step, ..; lane l sums column l's 4 quarter
    // partials ((q0+q1)+(q2+q3)), columns l >= 32 folded in after, then a
    // butterfly (deterministic)
    auto reduce_rows = [&](const int64_t bbase_u, const int nind_u, const int64_t j_u, int first,
                           int step) {
        const double* lgw = sL + (j_u & 1) * kYMaxIpt * 2;
        const double* redu = red + (DF ? (j_u & 1) * 512 : 0);
        for (int b2 = first; b2 < nind_u; b2 += step) {
            double acc = 0.0;
            for (int ll = lane; ll < p; ll += 32) {
                const double* rp = redu + b2 * p + ll;
                acc += (rp[0] + rp[128]) + (rp[256] + rp[384]);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) {
                if (A.out) {
                    // the finaliser (k_finalize), fused: same operations
                    const int64_t b = bbase_u + b2;
                    const double coll = A.chi * lgw[2 * b2];
                    const double dist = A.delta * lgw[2 * b2 + 1];
                    const double tran = A.alpha * acc;
                    A.out[4 * b + 0] = coll;
                    A.out[4 * b + 1] = tran;
                    A.out[4 * b + 2] = dist;
                    A.out[4 * b + 3] = __dadd_rn(__dadd_rn(coll, tran), dist);
                } else {
                    A.part[(bbase_u + b2) * A.pstride] = acc;
                }
            }
        }
    };

    if (DF && (warp == 2 || warp == 3)) {
        // ---------------- (defer) the units' reduces, each once its folds are
        // in, and (T in smem) the units' hubs + hub-cost tables two units
        // ahead: the epilogue warps never stop draining for them
        const int t2 = tid - 64;  // 0..63
        auto sync2 = [&]() {
            __syncwarp();
            asm volatile("bar.sync 2, 64;" ::: "memory");
        };
        // unit u's hubs into sH[u % 3] (own copies awaited, then both warps)
        auto hubs_of = [&](int64_t u) {
            int64_t nb;
            int nn;
            slot_unit(u, nb, nn);
            for (int x = t2; x < nn * p; x += 64)
                cp_async4(su32(sH + (int)((uint32_t)u % 3u) * ipt * p + x), A.hubs + nb * p + x);
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_all;" ::: "memory");
            sync2();
        };
        // unit u's tables T_b[k][l] = C[h_k][h_l] into sT[u & 1] (symmetric
        // costs: the upper triangle), landing on tgath[u & 1]
        auto gather_of = [&](int64_t u) {
            int64_t nb;
            int nn;
            slot_unit(u, nb, nn);
            const uint32_t sTu = su32(sT) + (uint32_t)(u & 1) * (uint32_t)p_T_bytes(ipt, p);
            const int32_t* hsu = sH + (int)((uint32_t)u % 3u) * ipt * p;
            const int pp = p * p;
            const uint64_t mpp = (uint64_t)(0xFFFFFFFFu / (uint32_t)pp) + 1u;
            const uint64_t mp = (uint64_t)(0xFFFFFFFFu / (uint32_t)p) + 1u;
            int m = 0;
            for (int x = t2; x < nn * pp; x += 64) {
                const int b2 = (int)(((uint64_t)x * mpp) >> 32), kl = x - b2 * pp;
                const int k = (int)(((uint64_t)kl * mp) >> 32), l2 = kl - k * p;
                if (A.tri && k > l2) continue;
                const int32_t* hs = hsu + b2 * p;
                cp_async8(sTu + 8u * x, A.C + (size_t)hs[k] * A.nC + hs[l2]);
                if (++m == 16) {  // (bounded groups of copies in flight)
                    m = 0;
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            cp_async_arrive(b_tgath + 8 * (uint32_t)(u & 1));
        };
        if (A.tsm)
            for (int64_t u = 0; u < 2 && u < nslots; ++u) {
                hubs_of(u);
                gather_of(u);
            }
        for (int64_t j = 0; j < nslots; ++j) {
            mb_wait(b_fold + 8 * (uint32_t)(j & 1), (uint32_t)((j >> 1) & 1));
            int64_t pb;
            int pn;
            slot_unit(j, pb, pn);
            reduce_rows(pb, pn, j, warp - 2, 2);
            __syncwarp();
            if (lane == 0) mb_arrive(b_rdone + 8 * (uint32_t)(j & 1));
            // unit j+2's tables go where unit j's were (its fold is done)
            if (A.tsm && j + 2 < nslots) {
                hubs_of(j + 2);
                gather_of(j + 2);
            }
        }
    } else if (warp == 1) {
        // ---------------- TMA producer: per phase, the W tiles (plane, row
        // block it) in order, tile it running K blocks [klo(c, it), nkb(c));
        // a stage holds up to KBS consecutive blocks of one tile
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            bool wrapped = false;
            const int q = (int)crank * 64;  // this CTA's W rows within a tile
            for (int64_t j = 0; j < nslots; ++j)
                for (int c = 0; c < NC; ++c) {
                    const int T = ntl(c), nb = nkb(c);
                    for (int pl = 0; pl < A.P; ++pl)
                        for (int it = 0; it < T; ++it)
                            for (int kb0 = klo(c, it); kb0 < nb; kb0 += KBS) {
                                const int nk = nb - kb0 < KBS ? nb - kb0 : KBS;
                                if (A.dbg & 32) continue;  // ablation: no W stream
                                // stage s is free: the leader's MMAs reading it completed
                                if (wrapped) mb_wait(b_empty + 8 * s, ph ^ 1u);
                                if (leader)  // both halves land on the leader's barrier
                                    mb_expect_tx(b_full + 8 * s, (uint32_t)(2 * nk * kYStageBytes));
                                const uint32_t dst = su32(ring + s * (KBS * kYStageBytes));
                                for (int kk = 0; kk < nk; ++kk)
                                    tma2d_pair(dst + kk * kYStageBytes, &tmW,
                                               (c * kYChunkKB + kb0 + kk) * 128,
                                               (A.plane0 + pl) * A.nt + it * 128 + q,
                                               L_full + 8 * s);
                                if (++s == (uint32_t)NS) {
                                    s = 0;
                                    ph ^= 1u;
                                    wrapped = true;
                                }
                            }
                }
        }
    } else if (warp == 0) {
        // ---------------- MMA issuer (leader CTA only)
        if (leader) {  // the whole warp, converged; one lane issues
            uint32_t s = 0, ph = 0, t = 0, phase = 0;
            const bool timed = kTimingBuild && A.timing != nullptr;
            const bool tr_on = timed && blockIdx.x == 0 && lane == 0;
            int tr_n = 0;
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
                for (int c = 0; c < NC; ++c, ++phase) {
                    const int nb = nkb(c), T = ntl(c);
                    // per chunk-local block, 4 bits each: the A quarters whose
                    // ready barrier the block's first MMA waits on (tile 0), and
                    // the quarters its last use frees
                    uint32_t waitq = 0u, relq = 0u;
                    for (int h = 0; h < 4; ++h) {
                        if (kq(c, h) < kq(c, h + 1)) waitq |= 1u << (4 * kq(c, h) + h);
                        relq |= 1u << (4 * qrb(c, h) + h);
                    }
                    for (int pl = 0; pl < A.P; ++pl)
                        for (int it = 0; it < T; ++it, ++t) {
                            const int d = t & 1, k0 = klo(c, it);
                            const bool first = (pl | it) == 0;
                            TRC(0, 1);
                            if (t >= 2 && !(A.dbg & 64))
                                mb_wait_cl(b_acce + 8 * d, ((t >> 1) - 1) & 1);
                            TRC(0, 2);
                            YT(w_e);
                            fence_after();
                            const uint32_t dcol = tmem + kYAcc0 + d * 128;
                            // the blocks this tile is the last user of (tri: its
                            // first, block it - 8c; full W: the last tile, all)
                            const int r0 = tri ? it - c * kYChunkKB : 0;
                            const int r1 = tri ? r0 + 1 : (it == T - 1 ? nb : 0);
                            for (int kb0 = k0; kb0 < nb; kb0 += KBS) {
                                const int nk = nb - kb0 < KBS ? nb - kb0 : KBS;
                                if (!(A.dbg & 16)) mb_wait(b_full + 8 * s, ph);
                                TRC(0, 3);
                                YT(w_f);
                                fence_after();
                                const uint64_t bd0 = sw128(su32(ring + s * (KBS * kYStageBytes)));
                                for (int kk = 0; kk < nk; ++kk) {
                                    const int kb = kb0 + kk;
                                    if (first && !(A.dbg & 64)) {
                                        // first use of this phase's A: a quarter must be
                                        // in TMEM before its first block's MMAs
                                        uint32_t wq = (waitq >> (4 * kb)) & 15u;
                                        if (wq) {
                                            TRC(0, 4);
                                            for (; wq; wq &= wq - 1)
                                                mb_wait_cl(b_ard + 8 * (__ffs(wq) - 1), phase & 1u);
                                            fence_after();
                                            TRC(0, 5);
                                        }
                                        YT(w_a);
                                    }
                                    if (A.dbg & 2) continue;
                                    const uint64_t bd = bd0 + (uint64_t)((kk * kYStageBytes) >> 4);
                                    // K steps of 32 = 8 TMEM columns of A each
                                    mma4_ts_w(dcol, tmem + kb * 32, bd, kIdescI8, kb != k0);
                                }
                                commit_pair_w(b_empty + 8 * s);
                                if (pl == A.P - 1)  // last use of A quarters: free them
                                    for (int rb = r0 > kb0 ? r0 : kb0; rb < r1 && rb < kb0 + nk; ++rb)
                                        for (uint32_t m = (relq >> (4 * rb)) & 15u; m; m &= m - 1)
                                            commit_pair_w(b_kbf + 8 * (__ffs(m) - 1));
                                if (++s == (uint32_t)NS) {
                                    s = 0;
                                    ph ^= 1u;
                                }
                                YT(w_i);
                            }
                            commit_pair_w(b_accf + 8 * d);
                            TRC(0, 8);
                        }
                }
            }
            if (timed && lane == 0) {
                atomicAdd(A.timing + 0, w_a);
                atomicAdd(A.timing + 1, w_e);
                atomicAdd(A.timing + 2, w_f);
                atomicAdd(A.timing + 3, w_i);
            }
        }
    } else if (warp >= kYEpiWarp0 && !(A.dbg & 64)) {
        // ---------------- generators + epilogue (16 warps)
        // (K3 is launched programmatically dependent on K2: its set-up and the
        // first W stages overlap K2's tail; everything K2 writes -- cluster
        // ids, legs, T planes -- is read only after this)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const int q = warp & 3;                         // TMEM lane quadrant
        const int sub = (warp - kYEpiWarp0) >> 2;       // 0..3: column quarter
        const int r = q * 32 + lane;                    // A row / accumulator lane
        const int bl = r / p, l = r - bl * p;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        uint32_t t = 0;
        const bool timed = kTimingBuild && A.timing != nullptr && tid == kYEpiWarp0 * 32;
        unsigned long long e_st = 0, e_gen = 0, e_wait = 0, e_cmp = 0, e_red = 0, e_ld = 0;
        unsigned long long e_sync = 0, e_tload = 0, e_fold = 0, e_kbf = 0, e_drain = 0;
        const bool tr_on = kTimingBuild && A.timing != nullptr && blockIdx.x == 0 && lane == 0 &&
                           (warp == kYEpiWarp0 || warp == kYWarps - 1);
        const int tr_role = warp == kYEpiWarp0 ? 1 : 2;
        int tr_n = 0;
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
        // one-hot A of phase (j, c) into TMEM (row r = (bl, l), K = the chunk's
        // nodes); this warp writes chunk blocks [kq(c,sub), kq(c,sub+1)) of its
        // lane quadrant, reading the cluster rows straight from global memory
        // (lanes of one individual read the same bytes: L1 broadcasts)
        // the cluster-row buffer of unit j (defer: 3, staged by cp.async)
// the tile after which column quarter s folds the previous unit (nibble s):
// quarter 0 generates the next unit's first one-hot quarter after tile 1, so
// it folds after tile 0, the others after tile 1 (tools/ab_k3.py: tile 3 for
// quarter 0 0.1137, tile 0 0.1130, every quarter at tile 1 0.1142 ms)
#ifndef HG_FOLD_TS
#define HG_FOLD_TS 0x1110
#endif
        static_assert((HG_FOLD_TS & 0xcccc) == 0, "the deferred fold runs with >= 4 tiles");
        const int ftile = (HG_FOLD_TS >> (4 * sub)) & 15;
        auto cbuf = [&](int64_t j) { return DF ? (int)(j % 3) : (int)(j & 1); };
        // one-hot columns [lo, hi) of phase (j, c), then quarter ha's ready arrive
        auto gen = [&](int64_t j, int c, int lo, int hi, int ha) {
            int64_t bbase;
            int nind;
            slot_unit(j, bbase, nind);
            const bool live = r < ipt * p && bl < nind;
            const uint32_t lrep = (uint32_t)l * 0x01010101u;
            if (CSM && DF) mb_wait(b_cready + 8 * (uint32_t)(j % 3), (uint32_t)((j / 3) & 1));
            TRC(tr_role, 19);
            const uint8_t* rowp = CSM ? sC0 + cbuf(j) * cb + (size_t)(live ? bl : 0) * A.npad
                                        : A.cl + (bbase + (live ? bl : 0)) * A.npad;
            const uint4* crow =
                reinterpret_cast<const uint4*>(rowp + (size_t)c * kYChunkKB * 128);
#pragma unroll 4
            for (int c0 = lo; c0 < hi && !(A.dbg & 8); c0 += 8) {
                uint32_t v[8];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    // (CSM: a dead row -- padding, or past the batch -- encodes
                    // the staged row 0 or stale bytes: harmless, it only feeds
                    // its own accumulator row, which nothing reads)
                    const bool ld = CSM || live;
                    const uint4 x = ld ? crow[(c0 >> 2) + h] : make_uint4(0, 0, 0, 0);
                    v[4 * h + 0] = ld ? oh4(x.x, lrep) : 0u;
                    v[4 * h + 1] = ld ? oh4(x.y, lrep) : 0u;
                    v[4 * h + 2] = ld ? oh4(x.z, lrep) : 0u;
                    v[4 * h + 3] = ld ? oh4(x.w, lrep) : 0u;
                }
                // (.sync.aligned: the warp must be converged -- the compiler
                // does not know the asm requires it; CSM: the loop body has no
                // per-lane branch)
#ifndef HG_GEN_SYNC
#define HG_GEN_SYNC 0
#endif
                if (HG_GEN_SYNC || !CSM || !DF) __syncwarp();
                st8(tmem + lane_base + (uint32_t)c0, v);
            }
            TRC(tr_role, 25);
            __syncwarp();
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            fence_before();
            __syncwarp();
            if (lane == 0) arrive_remote(L_ard + 8 * ha);
        };

        // stage a unit's cluster rows into double buffer j & 1 (CSM)
        // (defer: by cp.async, rows of live individuals only -- nothing reads
        // the others -- completion tracked by cready[j % 3])
        auto stage = [&](int64_t j) {
            int64_t bbase;
            int nind;
            slot_unit(j, bbase, nind);
            uint8_t* Cs = sC0 + cbuf(j) * cb;
            const int chunks = A.npad / 16;
            if (DF) {
                for (int x = tid - kYEpiWarp0 * 32; x < nind * chunks; x += kYEpiThreads)
                    cp_async16(su32(Cs) + 16u * (uint32_t)x,
                               A.cl + bbase * A.npad + (size_t)x * 16);
                asm volatile("cp.async.commit_group;" ::: "memory");
                cp_async_arrive(b_cready + 8 * (uint32_t)(j % 3));
                return;
            }
            for (int x = tid - kYEpiWarp0 * 32; x < ipt * chunks; x += kYEpiThreads) {
                const int b2 = x / chunks, k = x - b2 * chunks;
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (b2 < nind)
                    v = __ldg(reinterpret_cast<const uint4*>(A.cl + (bbase + b2) * A.npad) + k);
                reinterpret_cast<uint4*>(Cs + (size_t)b2 * A.npad)[k] = v;
            }
        };
        if (nslots > 0) {
            if (A.tsm && !DF) {  // unit 0's hubs (each unit's T gather reads them; defer: warps 2-3)
                int64_t nb;
                int nn;
                slot_unit(0, nb, nn);
                for (int x = tid - kYEpiWarp0 * 32; x < nn * p; x += kYEpiThreads)
                    cp_async4(su32(sH + x), A.hubs + nb * p + x);
                asm volatile("cp.async.commit_group;" ::: "memory");
                asm volatile("cp.async.wait_all;" ::: "memory");
                epi_sync();
            }
            if (CSM) {
                stage(0);
                if (!DF) epi_sync();
            }
            int lo = kq(0, sub) * 32, hi = kq(0, sub + 1) * 32;
            if (qsplit && sub == 3) q3part(3, lo, hi);
            gen(0, 0, lo, hi, sub);
            if (qsplit && sub < 3) {
                q3part(sub, lo, hi);
                gen(0, 0, lo, hi, 3);
            }
        }
        ET(e_gen);
        // this thread's bin row: bins[k][r] at byte k * 512 + r * 4
        const uint32_t bin_r0 = su32(bins) + (uint32_t)r * 4u;
        // a unit's S_T reduce and finaliser, run during the next unit's first
        // tile (the MMA keeps its two accumulators busy meanwhile; red and prod
        // are rewritten only after the next chunk-pass barrier)
        auto reduce_unit = [&](const int64_t bbase_u, const int nind_u, const int64_t j_u) {
                const double* lgw = sL + (j_u & 1) * kYMaxIpt * 2;
                if (EX) {
                    // S_T = np.sum(inter * hub_dist) in numpy's pairwise order
                    // (hm/evaluation.py:117-118) over the terms in `prod`: one warp
                    // per individual, lane group g (8 lanes) runs leaf L0 + g's 8
                    // strided accumulators over its <= 16 rows (x = k*p + l; rows
                    // past the leaf add +0.0, exact for these non-negative terms),
                    // lane 0 sums the leaves up the halving tree on a stack in `red`
                    const int m = p * p, R8 = m & ~7;
                    const uint32_t pmag = (1u << 24) / (uint32_t)p + 1u;  // x / p for x < 2^16
                    const int g = lane >> 3, jl = lane & 7;
                    double* stk = red + (warp - kYEpiWarp0) * 32;
                    for (int b2 = (warp - kYEpiWarp0); b2 < nind_u; b2 += kYEpiThreads / 32) {
                        const double* pb = prod + b2 * p;
                        auto term = [&](uint32_t x) {
                            const int k = (int)((x * pmag) >> 24);
                            return pb[k * 128 + ((int)x - k * p)];
                        };
                        int depth = 0;
                        for (int L0 = 0; L0 < A.nleaf; L0 += 4) {
                            const int L = L0 + g;
                            const uint32_t e = L < A.nleaf ? __ldg(A.leaves + L) : 0u;
                            const int r0 = (int)(e & 0xffffu), nr = (int)((e >> 16) & 0xffu);
                            double acc = 0.0;
    #pragma unroll 4
                            for (int q = 0; q < 16; ++q) {
                                const double v = q < nr ? term(8u * (uint32_t)(r0 + q) + jl) : 0.0;
                                acc = q == 0 ? v : acc + v;
                            }
                            acc = acc + __shfl_xor_sync(0xffffffffu, acc, 1);
                            acc = acc + __shfl_xor_sync(0xffffffffu, acc, 2);
                            acc = acc + __shfl_xor_sync(0xffffffffu, acc, 4);
                            if (L == A.nleaf - 1 && jl == 0)  // the last leaf's partial row
                                for (int x = R8; x < m; ++x) acc = acc + term((uint32_t)x);
    #pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const double cu = __shfl_sync(0xffffffffu, acc, 8 * u);
                                const uint32_t eu = __shfl_sync(0xffffffffu, e, 8 * u);
                                if (lane == 0 && L0 + u < A.nleaf) {
                                    stk[depth++] = cu;
                                    for (int c2 = L0 + u == A.nleaf - 1 ? depth - 1 : (int)(eu >> 24);
                                         c2 > 0; --c2, --depth)
                                        stk[depth - 2] = stk[depth - 2] + stk[depth - 1];
                                }
                            }
                        }
                        if (lane == 0) {
                            const double st = stk[0];
                            if (A.out) {
                                const int64_t b = bbase_u + b2;
                                const double coll = A.chi * lgw[2 * b2];
                                const double dist = A.delta * lgw[2 * b2 + 1];
                                const double tran = A.alpha * st;
                                A.out[4 * b + 0] = coll;
                                A.out[4 * b + 1] = tran;
                                A.out[4 * b + 2] = dist;
                                A.out[4 * b + 3] = __dadd_rn(__dadd_rn(coll, tran), dist);
                            } else {
                                A.part[(bbase_u + b2) * A.pstride] = st;
                            }
                        }
                        __syncwarp();
                    }
                } else {
                    reduce_rows(bbase_u, nind_u, j_u, warp - kYEpiWarp0, kYEpiThreads / 32);
                }
        };
        // defer: unit jp's bins (all its warps' atomics done) into this
        // row's partial red[jp & 1][sub][r], zeroing them; then folded[jp & 1]
        auto fold_unit = [&](const int64_t jp) {
            int64_t pb;
            int pn;
            slot_unit(jp, pb, pn);
            const bool livep = r < ipt * p && bl < pn;
            const uint32_t bx = (uint32_t)(jp & 1), par = (uint32_t)((jp >> 1) & 1);
            mb_wait(b_bdone + 8 * bx, par);
            mb_wait(b_tready + 8 * bx, par);
            if (A.tsm) mb_wait(b_tgath + 8 * bx, par);  // its tables (warps 2-3)
            double sp = 0.0;
            if (livep && !(A.dbg & 4)) {
                const double* tb =
                    A.tsm ? sT + (size_t)bx * ipt * p * p + bl * p * p + l : nullptr;
                const uint32_t* tp =
                    A.tsm ? nullptr : A.T + (pb + bl) * 2 * p * (int64_t)A.ps + l;
                for (int pl = 0; pl < A.P; ++pl) {
                    const double sc =
                        A.wscale * __longlong_as_double((long long)(1023 + 8 * pl) << 52);
                    sp = fold_bins(bins + (size_t)(bx * PB + pl) * p * 128 + r, tb, tp, p,
                                   A.ps, sub, sc, sp, A.tri && A.tsm ? l : -1);
                }
            }
            red[bx * 512 + sub * 128 + r] = sp;
            __syncwarp();
            if (lane == 0) mb_arrive(b_fold + 8 * bx);
        };
        // unit j's hub-cost tables T_b[k][l] = C[h_k][h_l] into sT (defer: its
        // buffer j & 1) by cp.async, off the unit's hubs in sH[j & 1]: this
        // thread's elements x = etid + 512 m for m = part, part + parts, ..
        // ((b2, k, l2) = x by multiply-high: (x * m) >> 32 with m =
        // floor((2^32 - 1) / d) + 1 is x / d exactly while x * d < 2^32)
        auto gather_T = [&](const int64_t j, const int nind, const int part, const int parts) {
            const int etid = tid - kYEpiWarp0 * 32;
            const uint32_t sTj =
                su32(sT) + (DF ? (uint32_t)(j & 1) * (uint32_t)p_T_bytes(ipt, p) : 0u);
            const int32_t* hsj = sH + (DF ? (int)(j % 3) : (int)(j & 1)) * ipt * p;
            const int pp = p * p;
            // (32-bit divisions: inline code, no 64-bit division subroutine)
            const uint64_t mpp = (uint64_t)(0xFFFFFFFFu / (uint32_t)pp) + 1u;
            const uint64_t mp = (uint64_t)(0xFFFFFFFFu / (uint32_t)p) + 1u;
            int m = 0;
            for (int x = etid + part * kYEpiThreads; x < nind * pp; x += parts * kYEpiThreads) {
                const int b2 = (int)(((uint64_t)x * mpp) >> 32), kl = x - b2 * pp;
                const int k = (int)(((uint64_t)kl * mp) >> 32), l2 = kl - k * p;
                // (defer on symmetric costs: the upper triangle only -- the
                // fold reads T[l][k] for T[k][l] below the diagonal)
                if (DF && A.tri && k > l2) continue;
                const int32_t* hs = hsj + b2 * p;
                cp_async8(sTj + 8u * x, A.C + (size_t)hs[k] * A.nC + hs[l2]);
                // (large p: at most two groups of 16 copies in flight per thread --
                // a thread with ~40 uncommitted copies trapped in testing)
                if (++m == 16) {
                    m = 0;
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                }
            }
        };
        // (slot j's first tile runs slot j-1's reduce; phase = j * NC + c is
        // recomputed rather than carried: the loop is register-bound)
        for (int64_t j = 0; j < nslots; ++j) {
            int64_t bbase;
            int nind;
            slot_unit(j, bbase, nind);
            const bool live = r < ipt * p && bl < nind;
            // defer: unit j's bins are buffer j & 1
            const uint32_t bin_r = bin_r0 + (DF ? (uint32_t)(j & 1) * (uint32_t)(PB * p * 512) : 0u);
            uint32_t* const binsj = bins;
            const uint8_t* crow = CSM ? sC0 + cbuf(j) * cb + (size_t)(live ? bl : 0) * A.npad
                                        : A.cl + (bbase + (live ? bl : 0)) * A.npad;
            TRC(tr_role, 24);
            if (CSM && j + 1 < nslots) {
                stage(j + 1);  // the next unit's cluster rows, under this unit's MMAs
                ET(e_st);
                if (!DF) epi_sync();  // ... complete before any warp generates from them
                ET(e_sync);
            }
            // this unit's leg sums and (tsm) hub-cost tables T_b[k][l] = C[h_k][h_l]
            // into shared memory by cp.async: the tables gathered from C (row
            // (b2, k) per warp, column l per lane) off the unit's hubs, staged one
            // unit ahead; read by the fold at the unit's end (after a barrier)
            // and the deferred reduce; the previous unit's fold is done with them
            {
                const int etid = tid - kYEpiWarp0 * 32;
                if (A.tsm && !DF) {  // (defer: hubs and tables by warps 2-3)
                    gather_T(j, nind, 0, 1);
                    if (j + 1 < nslots) {
                        int64_t nb;
                        int nn;
                        slot_unit(j + 1, nb, nn);
                        for (int x = etid; x < nn * p; x += kYEpiThreads)
                            cp_async4(su32(sH + ((j + 1) & 1) * ipt * p + x), A.hubs + nb * p + x);
                    }
                }
                // defer: unit j - 2's reduce (warps 2-3) is done with sL / red
                if (DF && j >= 2)
                    mb_wait(b_rdone + 8 * (uint32_t)(j & 1), (uint32_t)(((j - 2) >> 1) & 1));
                if (A.out && etid < nind)
                    cp_async16(su32(sL + (j & 1) * kYMaxIpt * 2 + 2 * etid),
                               A.legs + 2 * (bbase + etid));
                asm volatile("cp.async.commit_group;" ::: "memory");
                // defer: this unit's T tables and legs and the next unit's hubs,
                // all issued above, land on tready[j & 1] -- no wait for the
                // unit's end (the next unit's gather and this unit's fold wait)
                if (DF) cp_async_arrive(b_tready + 8 * (uint32_t)(j & 1));
            }
            TRC(tr_role, 26);
            // this row's T column: fp64 T_b[k][l] at tbd[k * p] (tsm), else K2's
            // hi / lo planes at tbp[k * ps], tbp[(p + k) * ps]
            const double* tbd = A.tsm ? sT + (live ? bl : 0) * p * p + l : nullptr;
            const uint32_t* tbp =
                A.tsm ? nullptr : A.T + (bbase + (live ? bl : 0)) * 2 * p * (int64_t)A.ps + l;
            double s_acc = 0.0;  // this thread's share of S_T over the chunks
            // plane pl of the flows carries weight 256^pl * wscale (an exact power
            // of two): each product is the one-plane product, scaled exactly
            auto fold_plane = [&](int pl, uint32_t* bp) {
                const double sc = A.wscale * __longlong_as_double((long long)(1023 + 8 * pl) << 52);
                s_acc = fold_bins(bp + r, tbd, tbp, p, A.ps, sub, sc, s_acc);
            };
            for (int c = 0; c < NC; ++c) {
                const uint32_t phase = (uint32_t)(j * NC + c);
                const bool last_phase = j + 1 == nslots && c + 1 == NC;
                const int T = ntl(c), NT = A.P * T;
                // the next phase's one-hot quarter `sub`, generated as soon as
                // the current A frees it.  It covers blocks [kq(cn,sub), X);
                // every current-phase MMA on blocks < X must be done: wait on
                // the current quarter holding block X-1 (MMAs complete in
                // order, and a block's last use never comes after a later
                // block's) -- chunks of different sizes (the last one) have
                // different quarter boundaries.  tri: quarter h is free after
                // tile 8c + its last block, early in the phase
                int hq = -1, tt_gen = NT - 1;
                bool gen_done = false;
                if (!last_phase) {
                    const int cn = c + 1 < NC ? c + 1 : 0;
                    const int X = kq(cn, sub + 1);
                    if (kq(cn, sub) < X) {
                        const int need = X - 1 < nkb(c) ? X - 1 : nkb(c) - 1;
                        hq = 3;
                        for (int h = 0; h < 4; ++h)
                            if (kq(c, h) <= need && need < kq(c, h + 1)) {
                                hq = h;
                                break;
                            }
                        tt_gen = (A.P - 1) * T + klast(c, qrb(c, hq));
                    }
                }
#ifndef HG_GEN_T0
#define HG_GEN_T0 2
#endif
                // (deferred fold: column quarter 0 folds after tile 0, so its
                // generation waits until after tile HG_GEN_T0 <= 3: 2, tools/ab_k3.py 0.1116
                // vs 0.1127 ms at its releasing tile 1)
                if (DF && HG_GEN_T0 > 0 && sub == 0 && tt_gen < HG_GEN_T0) tt_gen = HG_GEN_T0;
                for (int tt = 0; tt < NT; ++tt, ++t) {
                    const int d = t & 1;
                    const int pl = A.P == 1 ? 0 : tt / T, it = tt - pl * T;
                    // generate as soon as the quarter is free: the MMA issuer
                    // runs up to two tiles ahead, so poll from two tiles before
                    // the releasing one (the next phase's first MMAs wait on it)
// where a warp generates its quarter of the next one-hot (deferred fold; the
// other instantiations keep 0): 2 (default) after
// the releasing tile's drain and bin atomics -- the freed accumulator goes back
// to the MMA first; 0 at the top of that tile, before its drain, polling from
// two tiles earlier (tools/ab_k3.py: 0.1208 vs 0.1238 ms)
#ifndef HG_GEN_POS
#define HG_GEN_POS 2
#endif
                    // columns [lo, hi) of the next phase's one-hot once this
                    // phase's quarter hw is free; ready arrive on quarter ha
                    auto gen_next = [&](int lo, int hi, int ha, int hw) {
                        TRC(tr_role, 11);
                        if (hw >= 0) {
                            mb_wait(b_kbf + 8 * hw, phase & 1u);
                            fence_after();
                        }
                        TRC(tr_role, 12);
                        ET(e_kbf);
                        gen(c + 1 < NC ? j : j + 1, c + 1 < NC ? c + 1 : 0, lo, hi, ha);
                        TRC(tr_role, 13);
                        ET(e_gen);
                    };
                    const int cn = c + 1 < NC ? c + 1 : 0;
                    if ((HG_GEN_POS == 0 || !DF) && !last_phase && !gen_done && tt >= tt_gen - 2 &&
                        (tt == tt_gen ||
                         (hq >= 0 && __shfl_sync(0xffffffffu,
                                                 (int)mb_try(b_kbf + 8 * hq, phase & 1u), 0)))) {
                        gen_next(kq(cn, sub) * 32, kq(cn, sub + 1) * 32, sub, hq);
                        gen_done = true;
                    }
                    // cluster ids of the 32 columns i = it*128 + sub*32 + k
                    // (CSM: a dead row reads staged bytes too; its atomics are skipped)
                    uint4 ca = make_uint4(0, 0, 0, 0), cz = ca;
                    if (CSM || live) {
                        const uint4* cp = reinterpret_cast<const uint4*>(crow + it * 128 + sub * 32);
                        ca = cp[0];
                        cz = cp[1];
                    }
                    TRC(tr_role, 14);
                    mb_wait(b_accf + 8 * d, (t >> 1) & 1);
                    TRC(tr_role, 15);
                    ET(e_wait);
                    fence_after();
                    const uint32_t dcol = tmem + lane_base + kYAcc0 + d * 128 + sub * 32;
                    uint32_t v0[16], v1[16];
                    __syncwarp();  // (.sync.aligned loads: converged warp)
                    ld16(dcol, v0);
                    ld16(dcol + 16, v1);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    ET(e_ld);
                    fence_before();
                    __syncwarp();
                    if (lane == 0) arrive_remote(L_acce + 8 * d);  // accumulator may be overwritten
                    TRC(tr_role, 16);
                    // defer: bins j & 1 were folded (zeroed) for unit j - 2
                    if (DF && tt == 0 && j >= 2)
                        mb_wait(b_fold + 8 * (uint32_t)(j & 1), (uint32_t)(((j - 2) >> 1) & 1));
                    if (live && !(A.dbg & 1)) {
                        // G[c_i][r] += D[r][i]: exact integer bins, this row's own
                        // (4 column-quarter warps share a row, hence the atomics)
                        const uint32_t cw[8] = {ca.x, ca.y, ca.z, ca.w, cz.x, cz.y, cz.z, cz.w};
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            const uint32_t cc = __byte_perm(cw[k >> 2], 0u, 0x4440u + (k & 3));
                            HG_DCHECK(cc < (uint32_t)p, "K3 cluster %u of column %d outside [0, %d)",
                                      cc, it * 128 + sub * 32 + k, p);
                            const uint32_t dv = k < 16 ? v0[k] : v1[k - 16];
                            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(
                                             bin_r + (uint32_t)pl * (uint32_t)p * 512u + cc * 512u),
                                         "r"(dv)
                                         : "memory");
                        }
                    }
                    TRC(tr_role, 17);
                    ET(e_cmp);
                    if (HG_GEN_POS == 2 && DF && !last_phase) {
                        // this warp's quarter at its releasing tile; qsplit: its
                        // part of the last quarter at the last tile
                        int lo = -1, hi = 0, ha = 3, hw = 3;
                        if (!gen_done && tt == tt_gen) {
                            lo = kq(cn, sub) * 32;
                            hi = kq(cn, sub + 1) * 32;
                            if (qsplit && sub == 3) q3part(3, lo, hi);
                            ha = sub;
                            hw = hq;
                            gen_done = true;
                        } else if (qsplit && sub < 3 && tt == NT - 1) {
                            q3part(sub, lo, hi);
                        }
                        if (lo >= 0) gen_next(lo, hi, ha, hw);
                    }
                    if (DF && tt == ftile && j > 0) {
                        // the previous unit's fold after this unit's tile 1, 0
                        // for column quarter 0 (its reduce: warps 2-3)
                        fold_unit(j - 1);
                        TRC(tr_role, 18);
                    }
                    if (!DF && c == 0 && tt == 0 && j > 0 && !(A.dbg & 4)) {  // the previous unit's reduce
                        int64_t pb;
                        int pn;
                        slot_unit(j - 1, pb, pn);
                        reduce_unit(pb, pn, j - 1);
                        TRC(tr_role, 18);
                        ET(e_red);
                    }
                }
                if (DF) {  // this warp's atomics of unit j are done; fold + reduce deferred
                    __syncwarp();
                    if (lane == 0) mb_arrive(b_bdone + 8 * (uint32_t)(j & 1));
                    continue;  // (one chunk)
                }
                // this chunk's bins into S_T: sum_k T_b[k][l] * G_c[k][(b,l)] over
                // k = sub, sub + 4, ... (fixed order -> deterministic); one chunk's
                // bins stay below 2^32 (<= 255 * 1024 * n, n <= 16384).
                TRC(tr_role, 20);
                asm volatile("cp.async.wait_all;" ::: "memory");  // T, legs: this thread's part
                auto tval = [&](int k) {
                    return tbd ? tbd[k * p]
                               : __hiloint2double((int)tbp[k * A.ps], (int)tbp[(p + k) * A.ps]);
                };
                ET(e_tload);
                epi_sync();  // every bin of the chunk is complete
                TRC(tr_role, 21);
                ET(e_sync);
                if (timed) {  // the shared-memory pipe behind the atomics (timing build only)
                    uint32_t x0;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x0) : "r"(bin_r0) : "memory");
                    asm volatile("add.u32 %0, %0, 1;" : "+r"(x0));
                    if (x0 == 0xFFFFFFFFu) A.timing[31] = 1;
                    ET(e_drain);
                }
                if (live && EX && c + 1 == NC) {
                    // the bins (every K chunk accumulated, planes weighted
                    // 256^pl) ARE the reference's inter-cluster flows, exact
                    // integers: keep each rounded term inter * T for the
                    // pairwise sums below
                    const bool one_plane = A.P == 1;
                    auto inter = [&](int k) {
                        uint32_t* bp = binsj + k * 128 + r;
                        if (one_plane) {
                            const uint32_t g = *bp;
                            *bp = 0u;
                            return (double)g;
                        }
                        uint64_t g = 0;
                        for (int pl = 0; pl < A.P; ++pl, bp += p * 128) {
                            g += (uint64_t)*bp << (8 * pl);
                            *bp = 0u;
                        }
                        return (double)g;
                    };
#pragma unroll
                    // (the bins count Q = W / wscale, wscale a power of two: exact)
                    for (int k = sub; k < p; k += 4)
                        prod[k * 128 + r] = __dmul_rn(inter(k) * A.wscale, tval(k));
                }
                if (live && !EX && !(A.dbg & 4)) {
                    for (int pl = 0; pl < A.P; ++pl) fold_plane(pl, binsj + (size_t)pl * p * 128);
                }
                if (c + 1 == NC && !EX) red[sub * 128 + r] = s_acc;
                TRC(tr_role, 22);
                ET(e_fold);
                epi_sync();  // bins zeroed before the next chunk's atomics (red / prod written)
                TRC(tr_role, 23);
                ET(e_sync);
            }
            ET(e_red);
        }
        if (nslots > 0 && DF) fold_unit(nslots - 1);  // the last unit's (reduce: warps 2-3)
        if (nslots > 0 && !DF && !(A.dbg & 4)) {  // the last unit
            int64_t pb;
            int pn;
            slot_unit(nslots - 1, pb, pn);
            reduce_unit(pb, pn, nslots - 1);
        }
        if (timed) {
            atomicAdd(A.timing + 16, e_st);
            atomicAdd(A.timing + 17, e_gen);
            atomicAdd(A.timing + 18, e_wait);
            atomicAdd(A.timing + 19, e_cmp);
            atomicAdd(A.timing + 20, e_red);
            atomicAdd(A.timing + 21, e_ld);
            atomicAdd(A.timing + 22, e_sync);
            atomicAdd(A.timing + 23, e_tload);
            atomicAdd(A.timing + 24, e_fold);
            atomicAdd(A.timing + 25, e_kbf);
            atomicAdd(A.timing + 26, e_drain);
        }
    }
    fence_before();
    __syncthreads();
    cluster_sync_all();  // no CTA leaves while its peer may still signal its barriers
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(kYTmemCols)
                     : "memory");
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static int p_ipt(int p) {
    int ipt = 128 / p;
    return ipt > kYMaxIpt ? kYMaxIpt : ipt;
}

// stage a unit's cluster rows in shared memory when the double buffer is small
static bool p_csm(int p, int npad) {
    if (env_int("HUBGPU_TCP_CSM", 1) == 0) return false;  // tuning override
    return 2 * p_C_bytes(p_ipt(p), npad) <= 48 * 1024;
}

// everything but the W ring; exact: the [p][128] fp64 terms of S_T
// planes of bins one launch holds (more planes: a launch per plane)
static int p_bin_planes(int P) { return P > kYMaxPlanes ? 1 : P; }

// df: the deferred-fold layout (cluster rows x3, bins / partials / T x2)
static size_t p_base_bytes(int p, int npad, int P, bool exact, bool df = false) {
    const int nb = df ? 2 : 1;
    return 1024 + (p_csm(p, npad) ? (df ? 3 : 2) * p_C_bytes(p_ipt(p), npad) : 0) +
           (size_t)nb * p_bin_planes(P) * p * 512 +
           (size_t)nb * 4 * 128 * 8 + 2 * kYMaxIpt * 2 * 8 + (exact ? (size_t)p * 1024 : 0) +
           (2 * kYMaxStages + 12 + kYDeferBars) * 8 + 16;
}

// the unit's T tables in shared memory when they leave room for two full W
// stages (p <= ~36 at n <= 1024)
static size_t p_tsm_bytes(int p, bool df) {
    return (df ? 2 : 1) * p_T_bytes(p_ipt(p), p) + p_H_bytes(p_ipt(p), p);
}
static bool p_tsm(int p, int npad, int P, bool exact, bool df = false) {
    if (env_int("HUBGPU_TCP_TSM", 1) == 0) return false;  // tuning override
    const int64_t room = (int64_t)227 * 1024 - (int64_t)p_base_bytes(p, npad, P, exact, df) -
                         (int64_t)p_tsm_bytes(p, df);
    return room >= 2 * 8 * (int64_t)kYStageBytes;
}

static size_t p_fixed_bytes(int p, int npad, int P, bool exact = false, bool df = false) {
    return p_base_bytes(p, npad, P, exact, df) +
           (p_tsm(p, npad, P, exact, df) ? p_tsm_bytes(p, df) : 0);
}

// K blocks per W stage: 8 (one MMA-issuer loop per 1024 K) unless that
// leaves fewer than two stages (large p / the exact mode's terms): then 4, 2, 1
static int p_kbs(int p, int npad, int P, bool exact = false, bool df = false) {
    const int ek = env_int("HUBGPU_TCP_KBS", 0);  // tuning override
    if (ek >= 1 && ek <= 8) return ek;
    const int64_t room = (int64_t)227 * 1024 - (int64_t)p_fixed_bytes(p, npad, P, exact, df);
    int k = 8;
    while (k > 1 && room < 2 * (int64_t)k * kYStageBytes) k /= 2;
    return k;
}

static int p_stages(int p, int npad, int P, bool exact = false, bool df = false) {
    const int64_t room = (int64_t)227 * 1024 - (int64_t)p_fixed_bytes(p, npad, P, exact, df);
    int64_t s = room / ((int64_t)p_kbs(p, npad, P, exact, df) * kYStageBytes);
    if (s > kYMaxStages) s = kYMaxStages;
    const int es = env_int("HUBGPU_TCP_STAGES", 0);  // tuning override (shallower only)
    if (es >= 2 && es < s) s = es;
    return (int)s;
}

// exact sums need room for the [p][128] terms next to a W ring of >= 2
// stages (p <= ~90 at n <= 1024)
static bool p_exact(int p, int npad, int P) {
    return p_stages(p, npad, P, true) >= 2;
}

// exact: the instance asks for numpy's summation order and the terms fit
size_t tcp_smem_bytes(int p, int npad, int P, bool exact, bool df) {
    const bool x = exact && p_exact(p, npad, P);
    df = df && !x;
    return p_fixed_bytes(p, npad, P, x, df) +
           (size_t)p_stages(p, npad, P, x, df) * p_kbs(p, npad, P, x, df) * kYStageBytes;
}

// the deferred fold (K3's unit-to-unit hand-off without epilogue barriers):
// one K chunk, >= 4 output tiles per plane pass (the unit-drift bound its
// buffer reuse relies on), and its layout keeps the full 8-block W stages
// and the T tables in shared memory
static bool p_defer(int p, int npad, int P, int NC, int ITO, bool exact) {
    if (exact || NC != 1 || ITO < 4 || env_int("HUBGPU_TCP_DEFER", 1) == 0) return false;
    return p_kbs(p, npad, P, false, true) == p_kbs(p, npad, P, false, false) &&
           p_stages(p, npad, P, false, true) >= 2 &&
           p_tsm(p, npad, P, false, true) == p_tsm(p, npad, P, false, false);
}

bool tcp_supported(int n, int p, int npad, int P) {
    // p <= 128: a unit's one-hot rows fit the 128 TMEM lanes; n <= 16384: a
    // chunk's u32 bins cannot overflow
    return p >= 1 && p <= 128 && n >= 1 && n <= 16384 && npad % 128 == 0 &&
           P >= 1 && P <= 8 && p_stages(p, npad, P) >= 2;
}

static int g_tcp_pairs = 0;  // co-resident clusters (cudaOccupancyMaxActiveClusters)

int prepare_fitness_tcp(int p, int npad, int P) {
    // every instantiation at the device maximum: instances of different p /
    // planes need different sizes and the attribute is per kernel
    using KernFn = void (*)(const CUtensorMap, PArgs);
    const KernFn all[6] = {k_fitness_tcp<true, true>,  k_fitness_tcp<false, true>,
                           k_fitness_tcp<true, false>, k_fitness_tcp<false, false>,
                           k_fitness_tcp<true, false, true>, k_fitness_tcp<false, false, true>};
    for (KernFn f : all) HG_TRY(set_max_dynamic_smem(reinterpret_cast<const void*>(f)));
    const KernFn kern = p_csm(p, npad) ? k_fitness_tcp<true, false> : k_fitness_tcp<false, false>;
    const size_t sm = tcp_smem_bytes(p, npad, P, false);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kYCluster);
    cfg.blockDim = dim3(kYThreads);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kYCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    HG_CUDA(cudaOccupancyMaxActiveClusters(&nc, kern, &cfg));
    g_tcp_pairs = nc;
    return HG_OK;
}

// the launch geometry and arguments (shared by the launch and the work count)
static int tcp_setup(const DevInst& I, bool tri_avail, int64_t B, int grid, PArgs& A) {
    A.chi = I.chi;
    A.alpha = I.alpha;
    A.delta = I.delta;
    A.B = B;
    A.n = I.n;
    A.p = I.p;
    A.ps = I.ps;
    A.npad = I.npad;
    A.ipt = p_ipt(I.p);
    A.units = ceil_div(B, A.ipt);
    A.ITO = (int)(round_up(I.n, 128) / 128);
    A.KBT = A.ITO;
    A.NC = (A.KBT + kYChunkKB - 1) / kYChunkKB;
    A.nt = (int)round_up(I.n, 128);
    // exact: the instance asks for numpy's order and the [p][128] terms fit
    // beside two W stages (else the fixed-order fold: tran within ~1 ulp)
    // (several K chunks or planes: the bins accumulate over all of them, exact
    // while the total flow stays below 2^32)
    A.exact = I.exact && I.int_flows && (A.NC == 1 && I.wplanes == 1 || I.bins_total_ok) &&
              p_exact(I.p, I.npad, I.wplanes) && I.pwl != nullptr;
    // the triangular fold of W (half the MMA work) whenever the bins need not
    // be the reference's own flows: symmetric costs, fixed-order sums
    A.tri = !A.exact && tri_avail && !env_int("HUBGPU_TCP_NOTRI", 0) ? 1 : 0;
    A.P = A.tri ? I.wplanes_tri : I.wplanes;
    A.defer = p_defer(I.p, I.npad, A.P, A.NC, A.ITO, A.exact) ? 1 : 0;
    A.stages = p_stages(I.p, I.npad, A.P, A.exact, A.defer);  // as tcp_smem_bytes
    A.kbs = p_kbs(I.p, I.npad, A.P, A.exact, A.defer);
    A.csm = p_csm(I.p, I.npad) ? 1 : 0;
    A.tsm = p_tsm(I.p, I.npad, A.P, A.exact, A.defer) ? 1 : 0;
    A.plane0 = 0;
    A.pstride = 1;
    A.wscale = I.wscale;
    if (A.P > kYMaxPlanes) A.P = 1;  // one launch per plane (launch_fitness_tcp)
    A.idesc = kIdescI8;
    A.timing = tc_timing_buffer();
    A.dbg = env_int("HUBGPU_TCP_DBG", 0);
    A.leaves = I.pwl;
    A.nleaf = I.npwl;
    // whole clusters only, all co-resident (one wave): the GPCs need not hold a
    // multiple of the cluster size, so ask the occupancy API
    int g = (g_tcp_pairs > 0 ? g_tcp_pairs : grid / kYCluster) * kYCluster;
    const int64_t need = round_up(A.units, kYCluster);
    if (g > need) g = (int)need;
    if (g < kYCluster) g = kYCluster;
    return g;
}

bool tcp_gathers_T(const DevInst& I, bool tri_avail, int64_t B, int grid) {
    PArgs A;
    A.dB = nullptr;
    tcp_setup(I, tri_avail, B > 0 ? B : 1, grid, A);
    return A.tsm != 0;
}

// int8 operations the tensor cores execute for one launch on B hub sets:
// every (pair slot, chunk, plane, output tile) runs its K blocks as M=256 x
// N=128 x K=128 MMAs (dummy slots of an odd unit count included)
double tcp_mma_ops(const DevInst& I, bool tri_avail, int64_t B, int grid) {
    if (B <= 0) return 0.0;
    PArgs A;
    A.dB = nullptr;
    const int g = tcp_setup(I, tri_avail, B, grid, A);
    double blocks = 0.0;  // K blocks per pair slot
    for (int c = 0; c < A.NC; ++c) {
        const int nb = A.KBT - c * kYChunkKB < kYChunkKB ? A.KBT - c * kYChunkKB : kYChunkKB;
        const int T = A.tri && c * kYChunkKB + nb < A.ITO ? c * kYChunkKB + nb : A.ITO;
        for (int it = 0; it < T; ++it)
            blocks += nb - (A.tri && it > c * kYChunkKB ? it - c * kYChunkKB : 0);
    }
    blocks *= A.tri ? I.wplanes_tri : I.wplanes;  // every plane, one launch or several
    const int64_t ncl = g / kYCluster;
    double slots = 0.0;
    for (int64_t cid = 0; cid < ncl; ++cid) {
        const int64_t u = A.units * (cid + 1) / ncl - A.units * cid / ncl;
        slots += (double)((u + kYCluster - 1) / kYCluster);
    }
    return slots * blocks * 2.0 * 256.0 * 128.0 * 128.0;
}

static int tcp_launch(const DevInst& I, const PArgs& A, int g, const void* wmap, cudaStream_t s);

int launch_fitness_tcp(const DevInst& I, const void* wmap, const void* wmap_tri, int64_t B,
                       const uint8_t* cl, const uint32_t* T, double* part, int grid,
                       cudaStream_t s, const double* legs, double* out, const int32_t* hubs,
                       const int32_t* dynB) {
    if (B <= 0) return HG_OK;
    PArgs A;
    A.dB = dynB;
    A.cl = cl;
    A.T = T;
    A.hubs = hubs;
    A.C = I.C;
    A.nC = I.n;
    A.part = part;
    A.legs = legs;
    A.out = out;
    const int g = tcp_setup(I, wmap_tri != nullptr, B, grid, A);
    const int planes = A.tri ? I.wplanes_tri : I.wplanes;
    if (planes > kYMaxPlanes) {
        // fractional flows on more than 4 planes: a launch per plane writes its
        // partial S_T (weight 256^pl * quantum), the finaliser sums them in
        // plane order
        for (int pl = 0; pl < planes; ++pl) {
            PArgs Ap = A;
            Ap.plane0 = pl;
            Ap.wscale = I.wscale * std::ldexp(1.0, 8 * pl);
            Ap.out = nullptr;
            Ap.part = part + pl;
            Ap.pstride = planes;
            HG_TRY(tcp_launch(I, Ap, g, A.tri ? wmap_tri : wmap, s));
        }
        return launch_finalize(I, planes, B, legs, part, out, s);
    }
    return tcp_launch(I, A, g, A.tri ? wmap_tri : wmap, s);
}

static int tcp_launch(const DevInst& I, const PArgs& A, int g, const void* wmap, cudaStream_t s) {
    CUtensorMap map = *static_cast<const CUtensorMap*>(wmap);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(kYThreads);
    cfg.dynamicSmemBytes = tcp_smem_bytes(I.p, I.npad, A.P, A.exact, A.defer);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kYCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch on the preceding kernel (K2): see the
    // epilogue's griddepcontrol.wait (HUBGPU_TCP_PDL=0: plain serialisation)
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = env_int("HUBGPU_TCP_PDL", 1) ? 2 : 1;
    using KernFn = void (*)(const CUtensorMap, PArgs);
    const KernFn kern = A.exact ? (A.csm ? k_fitness_tcp<true, true> : k_fitness_tcp<false, true>)
                        : A.defer ? (A.csm ? k_fitness_tcp<true, false, true>
                                           : k_fitness_tcp<false, false, true>)
                                  : (A.csm ? k_fitness_tcp<true, false> : k_fitness_tcp<false, false>);
    HG_CUDA(cudaLaunchKernelEx(&cfg, kern, map, A));
    note_launch();
    return HG_OK;
}

}  // namespace hg
