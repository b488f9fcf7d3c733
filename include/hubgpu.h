/*
 * hubgpu.h -- C-ABI of libhubgpu.so, the B200 (sm_100a) implementation of the
 * hot path of the reference package hubmedian 0.1.0 (arXiv 1704.06258):
 * score a population of hub sets and evolve it with the island GA.
 *
 * The reference is pure Python + numpy and has no FFI of its own.  Every entry
 * point below names the reference function (file:line under
 * /root/reference/pkg/src/hubmedian/) whose work it replaces; the Python
 * mirror (paper_1704_06258_b200/) binds these with ctypes and keeps the
 * reference's Python signatures, encodings and exceptions.
 *
 * Conventions
 *   - every function returns an int status: HG_OK (0) or an HG_E* code; the
 *     message is available from hg_last_error() (thread-local);
 *   - pointers are HOST pointers unless the name says _dev / the `where`
 *     argument says HG_DEVICE; host buffers are borrowed for the call only;
 *   - hub sets are sorted ascending, 0-based, int64 (the reference's
 *     Solution encoding, hm/model.py:124-138); masks are one byte per node
 *     (numpy bool);
 *   - all device work of an instance runs on the instance's stream, in order;
 *     an instance may be shared across threads (as the reference's Instance,
 *     hm/model.py:35): every call that uses an instance, or a population or
 *     GA built on it, holds that instance's mutex for its duration.
 */
#ifndef HUBGPU_H
#define HUBGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_OK 0
#define HG_EARG 1      /* invalid argument -> ValueError in the mirror       */
#define HG_ECUDA 2     /* CUDA runtime / kernel failure                       */
#define HG_ENODEV 3    /* no CUDA device visible                              */
#define HG_ESTATE 4    /* object used in the wrong state                      */

#define HG_HOST 0
#define HG_DEVICE 1

/* instance flags reported by hg_instance_info */
#define HG_FLAG_SYMMETRIC 1    /* dist == dist^T exactly: one matrix serves both */
#define HG_FLAG_WEIGHTS_EXACT 2 /* out+in flow integer-valued, total < 2^53      */
#define HG_FLAG_TENSOR_OK 4     /* flows non-negative integers < 2^32, p <= 128,
                                   n <= 16384: exact u8 tensor path on 1..4 byte
                                   planes of W                                   */

/* fitness kernel choice (hg_instance_set_fitness) */
#define HG_FIT_AUTO 0      /* tensor cores when exact, else the fp64 gather   */
#define HG_FIT_FP64 1      /* K3: fp64 smem-gather kernel (any flows)          */
#define HG_FIT_TENSOR 2    /* the tensor-core kernel (= HG_FIT_TC_PAIR)         */
/* 3 and 4 named two superseded tensor-core variants (removed; rejected)   */
#define HG_FIT_TC_PAIR 5   /* K3-TC/P: u8 one-hot GEMM on tcgen05 CTA pairs, on
                              the triangular fold of W when the costs are
                              symmetric and the sums fixed-order (half the MMAs) */
#define HG_FIT_TC_PAIR_FULL 6 /* K3-TC/P on the full W always                  */

typedef struct hg_inst hg_inst;
typedef struct hg_pop hg_pop;
typedef struct hg_ga hg_ga;

const char* hg_last_error(void);
int hg_version(void);
int hg_device_count(int* count);

/* K1 -- HBM-resident instance.  Replaces Instance.__post_init__
 * (hm/model.py:55-81) and Instance.middle_rank (hm/model.py:96-105): the
 * derived vectors are computed on the host by the reference's own numpy
 * expressions and uploaded with the n x n fp64 dist and flow matrices.
 * `stream` may be NULL (the library creates a non-blocking stream). */
int hg_instance_create(int device, int n, int p, const double* dist, const double* flow,
                       const double* out_flow, const double* in_flow, double total_flow,
                       const int64_t* middle_rank, double chi, double alpha, double delta,
                       void* stream, hg_inst** out);
void hg_instance_free(hg_inst* inst);
int hg_instance_info(const hg_inst* inst, int* n, int* p, int* flags);
/* cost sums in numpy's pairwise order (on = 1): the collection, distribution
 * and transfer sums np.sum(out_flow * legs), np.sum(in_flow * legs),
 * np.sum(inter * hub_dist) of hm/evaluation.py:110-118 reproduced bit for bit
 * (the transfer sum when the CTA-pair kernel runs and p <= ~56, with a
 * total flow below 2^32 when n > 1024 or flows >= 256).  on = 0 (default): fixed-order
 * sums, deterministic, within ~1 ulp of the reference.  Read at each launch;
 * GA objects keep the mode they were created with. */
int hg_instance_set_exact(hg_inst* inst, int on);
int hg_instance_exact(const hg_inst* inst, int* on);
/* select / query the transfer-term kernel used by hg_evaluate, hg_pop_* and
 * GA objects created afterwards (both give the same values within fp64
 * summation-order rounding) */
int hg_instance_set_fitness(hg_inst* inst, int kind);
/* the kernel the next evaluation will run: HG_FIT_FP64 or one of HG_FIT_TC_* */
int hg_instance_fitness(const hg_inst* inst, int* kind);
/* the cudaStream_t all device work of this instance is queued on */
int hg_instance_stream(const hg_inst* inst, void** stream);
int hg_synchronize(hg_inst* inst);

/* K2 -- nearest-hub allocation, bit-exact.  Replaces allocate_to_nearest
 * (hm/model.py:202-207) for B hub sets at once: argmin over hubs with the
 * first (lowest-index) minimum, then hubs allocated to themselves.
 * hubs: B x p sorted int64; alloc: B x n int64 (host). */
int hg_allocate(hg_inst* inst, int64_t B, const int64_t* hubs, int64_t* alloc);

/* K2+K3 -- population objective.  Replaces _Evaluator.evaluate
 * (hm/engine.py:116-129) -> objective / _components
 * (hm/evaluation.py:86-120) for B solutions.  alloc == NULL means nearest
 * allocation of each hub set (the GA's evaluation); otherwise alloc (B x n
 * int64) is any feasible allocation onto the given hubs (objective() of an
 * arbitrary Solution; feasibility is checked by the caller, hm/model.py:154).
 * out: B x 4 doubles = (collection, transfer, distribution, raw) with
 * raw = (collection + transfer) + distribution as hm/evaluation.py:93. */
int hg_evaluate(hg_inst* inst, int64_t B, const int64_t* hubs, const int64_t* alloc,
                double* out);

/* duplicate-aware hg_evaluate (nearest allocation): the B
 * hub sets are grouped on the device (hash, sort, equality against the sorted
 * predecessor), each distinct set is scored once and its scores are copied to
 * every member -- what the reference's memo does for repeated sets
 * (_Evaluator, hm/engine.py:102-129).  *groups = number of distinct sets. */
int hg_evaluate_unique(hg_inst* inst, int64_t B, const int64_t* hubs, double* out,
                       int64_t* groups);

/* Device-resident population (the bench's `value` path and the GA's own
 * children buffer).  hg_pop_load_hubs takes int32 hub sets (host or device);
 * hg_pop_evaluate queues K2+K3+finalise on the instance stream and returns
 * without synchronising; hg_pop_read copies the B x 4 results out. */
int hg_pop_create(hg_inst* inst, int64_t capacity, hg_pop** out);
void hg_pop_free(hg_pop* pop);
int hg_pop_load_hubs(hg_pop* pop, int64_t B, const int32_t* hubs, int where);
int hg_pop_evaluate(hg_pop* pop, int64_t B);
int hg_pop_read(hg_pop* pop, int64_t B, double* out, int where);
/* number of kernels hg_pop_evaluate launches (the bench's gpu_launches) */
int hg_pop_launches_per_evaluate(const hg_pop* pop);
/* duration (ms) of the fitness kernel K3 in the last hg_pop_evaluate,
 * measured with CUDA events on the instance stream (synchronises) */
int hg_pop_last_fitness_ms(hg_pop* pop, float* ms);
/* duration (ms) of the allocation kernel K2 in the last hg_pop_evaluate */
int hg_pop_last_allocate_ms(hg_pop* pop, float* ms);

/* int8 tensor-core operations (2 per multiply-add) the instance's fitness
 * kernel issues to score B hub sets, padding and dummy work included; 0 for
 * the fp64 kernel (the bench's roofline numerator) */
int hg_fitness_work(hg_inst* inst, int64_t B, double* mma_ops);

/* kernels this library has launched in the process so far (a CUDA-graph
 * replay adds the kernels it holds); differences of two reads count the
 * launches of a region (the bench's gpu_launches) */
int hg_launch_count(uint64_t* count);

/* tuning aid: per-phase cycle counters of K3-TC when the process runs with
 * HUBGPU_TC_TIMING=1 (32 counters, read and reset); HG_EARG otherwise */
int hg_debug_tc_timing(unsigned long long* out32);
/* Timing build only: K3-TC/P's event trace of CTA 0 (3 x 8192 words). */
int hg_debug_tc_trace(unsigned long long* out);

/* K4c -- correction.  Replaces correct_hub_set (hm/operators.py:69-101) for
 * B raw hub masks (B x n bytes): deficit opens closed nodes in middle-rank
 * order; excess closes, one at a time, the hub whose nearest-allocated nodes
 * carry the least out+in flow (first minimum), re-allocating after each
 * closure.  hubs_out: B x p int64. */
int hg_correct(hg_inst* inst, int64_t B, const uint8_t* masks, int64_t* hubs_out);

/* K4b -- single-point crossover (hm/operators.py:41-57) of B mask pairs with
 * the cut points given (cut in [1, n]; n copies the parents), and the
 * hub/spoke swap (hm/operators.py:113-124) with its two draws given as
 * indices (r_close-th open node closed, r_open-th node of the closed list
 * taken before closing opened); r_close < 0 means identity (all-open /
 * all-closed mask, no draws).  Masks are B x n bytes; no instance needed. */
int hg_crossover(int device, int n, int64_t B, const uint8_t* a, const uint8_t* b,
                 const int64_t* cuts, uint8_t* child1, uint8_t* child2);
int hg_swap(int device, int n, int64_t B, const uint8_t* masks, const int64_t* r_close,
            const int64_t* r_open, uint8_t* out);

/* K4a..K5 -- island GA on one device.  Replaces _run_island
 * (hm/engine.py:138-167) for the islands [island_lo, island_hi) of a run
 * with `islands_total` islands; per-island SplitMix64 streams are
 * derive_stream(seed, island, role) (hm/engine.py:40-54, hm/rng.py:102-107)
 * keyed by the GLOBAL island id, so any sharding replays the same draws. */
typedef struct {
    int32_t islands_total;
    int32_t island_lo;
    int32_t island_hi;
    int32_t pop_size;       /* even, >= 2                               */
    int32_t strength;       /* perturbation swaps, 1..p                 */
    int32_t strict_paper;   /* 0 elitist (default), 1 strict            */
    int32_t rng;            /* HG_RNG_REPLAY (default) or HG_RNG_PHILOX */
    uint64_t seed;          /* GaParams.seed reduced mod 2^64           */
} hg_ga_params;

/* draw generator of the island GA.  REPLAY: the reference's SplitMix64
 * streams, draw k = mix64(s + k*gamma) -- trajectories equal the reference's.
 * PHILOX: Philox4x32-10 keyed by the same per-(island, role) stream key, with
 * the draw index as counter -- the same draw accounting and operators, a
 * different (and independent) stream of numbers. */
#define HG_RNG_REPLAY 0
#define HG_RNG_PHILOX 1
/* Philox4x32-10 block (Salmon et al., SC'11), the GA's PHILOX generator;
 * host-side entry for known-answer tests */
void hg_philox4x32_10(const uint32_t key[2], const uint32_t ctr[4], uint32_t out[4]);
/* numpy's pairwise summation (pairwise_sum_DOUBLE, the order of every np.sum
 * in hm/evaluation.py:110-118) as the leaf table the exact mode replays: per
 * leaf first row of 8 terms | full rows << 16 | tree sums after it << 24;
 * host-only, for tests */
int hg_pairwise_leaves(int64_t m, uint32_t* out, int cap, int* count);

int hg_ga_create(hg_inst* inst, const hg_ga_params* params, hg_ga** out);
void hg_ga_free(hg_ga* ga);
/* restart the run with another seed: stream states derive_stream(seed, island,
 * role) and draw counters reset, buffers and the captured graph reused (a
 * solve() on the same instance and shape needs no new allocation) */
int hg_ga_reseed(hg_ga* ga, uint64_t seed);
/* start an outer round: every local island's ancestor := hubs (p sorted int64) */
int hg_ga_begin_round(hg_ga* ga, const int64_t* ancestor_hubs);
/* queue `count` generations (one CUDA graph launch each); asynchronous */
int hg_ga_generations(hg_ga* ga, int count);
/* per local island: the round result -- island best (elitist) or last
 * champion (strict); raw (n_local) and hubs (n_local x p); synchronises */
int hg_ga_round_results(hg_ga* ga, double* raw, int64_t* hubs);
/* children of the last generation in evaluation order (audit path):
 * hubs (B x p) and raw (B), B = n_local * pop_size; synchronises */
int hg_ga_last_children(hg_ga* ga, int64_t* hubs, double* raw);
/* draws consumed so far per local island and role (n_local x 3) */
int hg_ga_draw_counters(hg_ga* ga, uint64_t* counters);
/* kernels launched per generation */
int hg_ga_launches_per_generation(const hg_ga* ga);

/* page-locked host memory (cudaHostAlloc / cudaFreeHost): result buffers the
 * device can write by DMA directly (the Python layer pools them) */
int hg_host_alloc(size_t bytes, void** out);
void hg_host_free(void* p);

/* device generator.  generate_urand (hm/io.py:188-210)
 * bit for bit on the GPU: the SplitMix64 stream derive_stream(seed, n, p)
 * is counter-based, so every element computes its own draws.  Fills the host
 * arrays dist and flow (n x n row-major fp64; either may be NULL). */
int hg_generate_urand(int device, int n, int p, uint64_t seed, double* dist, double* flow);

/* restricted_optimum (hm/oracle.py:42-54) on the GPU:
 * every p-subset in itertools.combinations order through K2+K3, keeping the
 * first strict minimum of raw (lexicographically smallest hub set on ties).
 * Fails (HG_EARG) when C(n, p) > limit, as EnumerationLimitError.
 * best_hubs: p int64 (host); *count_out = C(n, p) (saturated at 2^63). */
int hg_restricted_optimum(hg_inst* inst, uint64_t limit, int64_t* best_hubs, double* best_raw,
                          uint64_t* count_out);

#ifdef __cplusplus
}
#endif
#endif /* HUBGPU_H */
