// Internal declarations shared by the libhubgpu translation units.
//
// Device data layout (all row-major, one allocation per array):
//   C   [n][n]   fp64  dist: C[i][k] = unit cost i -> k           (hm/model.py:45)
//   Ct  [n][n]   fp64  C transposed (aliases C when symmetric) -- allocation
//                      reads Ct[h][i] so a warp's 32 nodes are one 256 B line
//   W   [n][n]   fp64  flow
//   O, D, wOD [n] fp64 out/in flow and their sum (correction weights)
//   rank [n]     int32 middle-node order (hm/model.py:96-105)
// Population (capacity Bcap), see hg_pop:
//   hubs [B][p]       int32 sorted hub ids
//   cl   [B][npad]    uint8 cluster of node i = position of its hub in hubs
//                     (padding to npad is zero so padded lanes hit T row 0)
//   co   [B][npad]    uint16 4*cl: byte offset of the column in a T plane row
//   T    [B][2][p][ps] uint32 hub-to-hub cost table T[k][l] = C[h_k][h_l] as
//                     a plane of hi words and a plane of lo words
//   legs [B][2]       fp64 sum_i O_i*leg_i, sum_i D_i*leg_i (leg_i = C[i][a_i])
//   part [B][tiles]   fp64 per-W-tile partial of sum_ij W_ij T[c_i][c_j]
//   out  [B][4]       fp64 collection, transfer, distribution, raw
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdarg>
#include <cstdio>

#include "../../include/hubgpu.h"

namespace hg {

void set_error(const char* fmt, ...);

// a tuning variable of the environment as an int (absent: dflt; present but
// not a number: 1), read once per process -- launch paths call this often
int env_int(const char* name, int dflt);

#define HG_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            ::hg::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),     \
                            __FILE__, __LINE__);                                        \
            return HG_ECUDA;                                                            \
        }                                                                               \
    } while (0)

#define HG_ARG(cond, ...)                                                               \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            ::hg::set_error(__VA_ARGS__);                                               \
            return HG_EARG;                                                             \
        }                                                                               \
    } while (0)

#define HG_TRY(expr)                                                                    \
    do {                                                                                \
        int s_ = (expr);                                                                \
        if (s_ != HG_OK) return s_;                                                     \
    } while (0)

// kernels of this library launched by the host so far (graph replays add
// their kernel count): the bench's gpu_launches is a difference of two reads
void note_launch(uint64_t k = 1);
uint64_t launch_count();

#define HG_LAUNCHED()                                                                   \
    do {                                                                                \
        HG_CUDA(cudaGetLastError());                                                    \
        ::hg::note_launch();                                                            \
    } while (0)

// device-side invariant checks of the checked build (make EXTRA=-DHG_CHECKS):
// a failed check prints and traps (compute-sanitizer is closed on this pool,
// tools/checked_tests.sh runs the GPU tests on this build instead)
#ifdef HG_CHECKS
#define HG_DCHECK(cond, fmt, ...)                                                        \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            printf("HG_DCHECK %s:%d " fmt "\n", __FILE__, __LINE__, ##__VA_ARGS__);     \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define HG_DCHECK(cond, fmt, ...) \
    do {                          \
    } while (0)
#endif

constexpr int kMaxP = 255;          // cluster ids are uint8
constexpr int kMaxNga = 32768;      // GA mask kernels keep one mask per warp in smem

struct DevInst {
    int n, p;
    int nw;        // 32-bit words per hub mask
    int ps;        // row stride (uint32 words) of the T hi/lo planes: p rounded up to 4
    int npad;      // row stride (bytes) of cluster-id rows
    int weights_exact;
    int wplanes;   // byte planes of the u8 flow tensor W8 (1 when every flow < 256)
    int wplanes_tri;  // byte planes of its triangular fold (W + W^T above the diagonal blocks)
    int int_flows;    // every flow an integer below 2^32 (the planes hold W exactly)
    double wscale;    // the planes hold Q = rint(W / wscale), wscale a power of two (1: integers)
    double chi, alpha, delta;
    const double* C;
    const double* Ct;
    const double* W;
    const double* O;
    const double* D;
    const double* wOD;
    const int32_t* rank;
    // Ct quantised monotonically to 16 bits: Cq = min(65535, floor((Ct - cmin) * s)).
    // q(a) < q(b) implies a < b, so it filters the allocation argmin exactly.
    // Rows are nq = round_up(n, 8) entries (16-byte aligned, bulk-copyable).
    const uint16_t* Cq;
    int nq;
    // input-validation flag of the current host call (0 = ok, else 0x7ffffffe - bad row)
    const int* err;
    // numpy's pairwise summation order (see pw_leaf_table): the leaves of the
    // n-term leg sums and of the p*p-term transfer sum, one word per leaf
    // (first row of 8 terms | rows << 16 | tree sums after it << 24)
    const uint32_t* pwnl;
    int npwnl;
    const uint32_t* pwl;
    int npwl;
    // 1: every cost sum in numpy's pairwise order (bit-identical to the
    // reference); 0: fixed-order sums (deterministic, ~1 ulp apart)
    int exact;
    int bins_total_ok;  // total flow < 2^32: integer bins can span every K chunk
    // a device-side batch size (the GA's distinct-hub-set count) bounding a
    // launch sized for the host batch; nullptr: the host batch
    const int32_t* dynB;
    // K2 reads the batch's int64 hub sets itself (nullptr: the int32 `hubs`):
    // rows hrow0.. of the caller's batch -- typically page-locked host memory
    // read over PCIe while K2 computes, k_hubs_in fused: each row validated
    // (in [0, n), ascending) with the bad row recorded in *err, and written
    // as int32 to hubs_w for K3
    const int64_t* hubs64 = nullptr;
    int32_t* hubs_w = nullptr;
    int64_t hrow0 = 0;
};

constexpr int kPwStack = 16;  // tree depth bound (n < 2^21)

// fitness tiling chosen per instance (see fitness_plan)
struct FitPlan {
    int variant;      // index into the kernel table
    int rw, cj;       // rows per warp, columns per lane
    int tr, tc;       // tile rows (16*rw) / columns (32*cj)
    int trn, tcn, tiles;
    int g;            // individuals per pipeline stage
    int blocks_per_sm;
    size_t smem;
};

FitPlan fitness_plan(const DevInst& I, int sm_count);
int prepare_fitness(const FitPlan& P);

// ---- launchers (k_eval.cu) -------------------------------------------------
int launch_hubs_in(const int64_t* src, int32_t* dst, int64_t B, int p, int n, int* err,
                   cudaStream_t s, int64_t row0 = 0);
int launch_idx_in(const int64_t* src, int32_t* dst, int64_t count, int n, int* err,
                  cudaStream_t s);
int launch_i32_to_i64(const int32_t* src, int64_t* dst, int64_t count, cudaStream_t s);
int launch_transpose(const double* src, double* dst, int n, cudaStream_t s);
int launch_check_symmetric(const double* C, int n, int* flag, cudaStream_t s);
int launch_quantize(const double* Ct, uint16_t* Cq, int n, int nq, double cmin, double scale,
                    cudaStream_t s);
int prepare_allocate(const DevInst& I);
int launch_allocate(const DevInst& I, int64_t B, const int32_t* hubs, uint8_t* cl, uint16_t* co,
                    uint32_t* T, double* legs, int32_t* alloc, cudaStream_t s,
                    const int32_t* dynB = nullptr);
int launch_from_alloc(const DevInst& I, int64_t B, const int32_t* hubs, const int32_t* alloc,
                      uint8_t* cl, uint16_t* co, uint32_t* T, double* legs, cudaStream_t s);
int launch_fitness(const DevInst& I, const FitPlan& P, int64_t B, const uint8_t* cl,
                   const uint16_t* co, const uint32_t* T, double* part, int grid, cudaStream_t s);
int launch_finalize(const DevInst& I, int tiles, int64_t B, const double* legs,
                    const double* part, double* out, cudaStream_t s);

// ---- K1 on the device (k_load.cu) -------------------------------------------
struct InstanceScan {
    unsigned long long cmin_bits, cmax_bits;  // min / max cost (bit patterns, >= 0)
    unsigned long long wmax_bits, mmax_bits;  // max flow / max entry of the triangular fold
    unsigned long long wmin_bits;             // smallest nonzero flow
    double wsum;                              // total flow
    int int_flows;                            // 1: every flow an integer in [0, 2^32)
    int symmetric;                            // 1: C == C^T exactly
    int lsb_exp;                              // min over nonzero flows of e in w = odd * 2^e
};
int launch_scan_instance(const double* C, const double* W, int n, InstanceScan* out,
                         cudaStream_t s);
// W8: P byte planes of Q = rint(W / wscale), M8 (optional): Ptri byte planes of
// Q's triangular fold; both [planes][nt][nt] with nt = round_up(n, 128)
int launch_build_planes(const double* W, int n, int nt, double wscale, int P, int Ptri,
                        uint8_t* W8, uint8_t* M8, cudaStream_t s);

// ---- K3-TC/P helpers (tc_common.cu) ------------------------------------------
int tc_timing_read(unsigned long long* out32);
int tc_trace_read(unsigned long long* out);
unsigned long long* tc_timing_buffer();  // HUBGPU_TC_TIMING=1, else nullptr
// map_out: CUtensorMap (128 B) over the u8 W, boxes of 128 K bytes x box_rows rows
// rows: total rows of the (plane-stacked) tensor, default npad_tc
int tc_make_wmap(const uint8_t* W8, int npad_tc, int box_rows, void* map_out, int rows = 0);
inline int tc_tiles(int n) { return (int)((n + 127) / 128); }
// the largest dynamic shared memory a launch of `fn` may ask for (set once:
// the attribute is per kernel and process-wide, instances differ in size)
int set_max_dynamic_smem(const void* fn);
// K3-TC/P (k_fitness_tcp.cu): the same on CTA pairs (cta_group::2, M = 256)
// P: byte planes of W (integer flows < 256^P), stacked in the u8 tensor
bool tcp_supported(int n, int p, int npad, int P);
size_t tcp_smem_bytes(int p, int npad, int P, bool exact, bool df = false);
int prepare_fitness_tcp(int p, int npad, int P);
// legs / out set: the finaliser is fused (out gets the 4 cost terms, part unused)
// int8 tensor operations one launch on B hub sets issues (the roofline's work)
double tcp_mma_ops(const DevInst& I, bool tri_avail, int64_t B, int grid);
// wmap_tri: the map of the triangular fold (symmetric costs), or nullptr
int launch_fitness_tcp(const DevInst& I, const void* wmap, const void* wmap_tri, int64_t B,
                       const uint8_t* cl, const uint32_t* T, double* part, int grid,
                       cudaStream_t s, const double* legs, double* out, const int32_t* hubs,
                       const int32_t* dynB = nullptr);
// true: the launch gathers the hub-cost tables from C itself (K2 need not write T)
bool tcp_gathers_T(const DevInst& I, bool tri_avail, int64_t B, int grid);

// ---- k_gen.cu: device generator and hub-set enumeration ---------------------
// xy: 2n scratch; C / W: n x n (either may be null)
int launch_gen_urand(uint64_t s, int n, double* xy, double* C, double* W, cudaStream_t st);
// binom[a * (p+1) + b] = C(a, b), a <= n, b <= p
int launch_unrank_combos(const uint64_t* binom, int n, int p, uint64_t rank0, int64_t B,
                         uint64_t count, int32_t* hubs, cudaStream_t st);
int launch_batch_best(const double* out, int64_t B, uint64_t rank0, uint64_t count,
                      double* best_raw, unsigned long long* best_rank, cudaStream_t st);

// ---- k_unique.cu: duplicate-aware evaluation ---------------------------------
size_t unique_scratch_bytes(int64_t B);
// groups the B hub sets (int32 [B][p]); writes one representative per group to
// uhubs (dense, in sorted-hash order), map[b] = group of set b, and
// d_count[0] + d_count[1] = number of groups
// d_total (optional): the group count itself, written on the device
int launch_unique_groups(const int32_t* hubs, int64_t B, int p, void* scratch, size_t bytes,
                         int32_t* uhubs, int32_t* map, int32_t* d_count, cudaStream_t s,
                         int32_t* d_total = nullptr);
int launch_scatter_out(const double* uout, const int32_t* map, int64_t B, double* out,
                       cudaStream_t s);

// ---- launchers (k_ga.cu) ---------------------------------------------------
int launch_bytes_to_bits(const uint8_t* bytes, uint32_t* bits, int64_t B, int n, int nw,
                         cudaStream_t s);
int launch_bits_to_bytes(const uint32_t* bits, uint8_t* bytes, int64_t B, int n, int nw,
                         cudaStream_t s);
int launch_correct(const DevInst& I, int64_t B, const uint32_t* bits, int hmax, int32_t* hubs,
                   cudaStream_t s);
int launch_splice(int64_t B, int n, int nw, const uint32_t* a, const uint32_t* b,
                  const int64_t* cuts, uint32_t* c1, uint32_t* c2, cudaStream_t s);
int launch_swap_given(int64_t B, int n, int nw, uint32_t* bits, const int64_t* r_close,
                      const int64_t* r_open, cudaStream_t s);

struct GaDev {
    int n, p, nw;
    int nloc, pop, strength, strict_mode;
    int rng;              // HG_RNG_REPLAY / HG_RNG_PHILOX
    int island_lo;
    uint32_t* anc;        // [nloc][nw]
    uint32_t* popbits;    // [B][nw]
    uint32_t* kids;       // [B][nw]
    int32_t* kcount;      // [B]
    int32_t* moff;        // [B]
    int32_t* nondeg;      // [nloc]
    int32_t* khubs;       // [B][p]   (the population's hubs buffer)
    const double* kraw;   // [B][4]   (the population's out buffer)
    double* champ_raw;    // [nloc]
    int32_t* champ_hubs;  // [nloc][p]
    double* best_raw;     // [nloc]
    int32_t* best_hubs;   // [nloc][p]
    uint64_t* st;         // [nloc][3] stream states
    uint64_t* ctr;        // [nloc][3] draws consumed
    const int32_t* inc;   // [p] round ancestor
};

int launch_round_begin(const GaDev& G, cudaStream_t s);
int launch_build_pop(const GaDev& G, cudaStream_t s);
int launch_crossover(const GaDev& G, cudaStream_t s);
int launch_mut_scan(const GaDev& G, cudaStream_t s);
int launch_mutate(const GaDev& G, cudaStream_t s);
int launch_select(const GaDev& G, cudaStream_t s);

// ---- SplitMix64 (hm/rng.py:43-48, 84-89) --------------------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// k-th output (1-based) of the stream whose state is s
__host__ __device__ __forceinline__ uint64_t sm_draw(uint64_t s, uint64_t k) {
    return mix64(s + k * kGolden);
}

// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): 10 rounds of two
// 32x32->64 multiplies with the key bumped by the Weyl constants between rounds
__host__ __device__ __forceinline__ void philox4x32_10(uint32_t k0, uint32_t k1, uint32_t c[4]) {
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
    }
}

// the GA's k-th draw of the stream with key s: SplitMix64 replay (mode 0) or
// Philox4x32-10 keyed by s with counter (k, 0) (mode 1)
__host__ __device__ __forceinline__ uint64_t ga_draw(int mode, uint64_t s, uint64_t k) {
    if (mode == 0) return sm_draw(s, k);
    uint32_t c[4] = {(uint32_t)k, (uint32_t)(k >> 32), 0u, 0u};
    philox4x32_10((uint32_t)s, (uint32_t)(s >> 32), c);
    return (uint64_t)c[0] | ((uint64_t)c[1] << 32);
}

// int(random() * bound) with random() = (x >> 11) * 2^-53 (hm/rng.py:74-82)
__device__ __forceinline__ int below(uint64_t x, int bound) {
    double u = __dmul_rn((double)(x >> 11), 0x1p-53);
    return (int)__dmul_rn(u, (double)bound);
}

inline uint64_t host_stream_key(uint64_t seed, const uint64_t* keys, int nkeys) {
    uint64_t s = mix64(seed);
    for (int i = 0; i < nkeys; ++i) s = mix64(s ^ mix64(keys[i] + kGolden));
    return s;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace hg
