// C-ABI object layer of libhubgpu.so (see include/hubgpu.h).

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <mutex>
#include <new>
#include <vector>

#include "hg_internal.cuh"

namespace hg {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

}  // namespace hg

using namespace hg;

struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    int ensure(size_t need) {
        if (need <= bytes) return HG_OK;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        size_t cap = need + need / 4 + 256;
        HG_CUDA(cudaMalloc(&ptr, cap));
        bytes = cap;
        return HG_OK;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const { return static_cast<T*>(ptr); }
};

struct hg_pop {
    hg_inst* inst = nullptr;
    int64_t cap = 0;
    int32_t* hubs = nullptr;
    uint8_t* cl = nullptr;
    uint16_t* co = nullptr;
    uint32_t* T = nullptr;
    double* legs = nullptr;
    double* part = nullptr;
    double* out = nullptr;
    int tiles = 0;  // per-individual partials (the row stride of part)
    DevBuf alloc;  // int32 [cap][n], on demand
    cudaEvent_t evk = nullptr, ev0 = nullptr, ev1 = nullptr;  // before K2, K3, after K3
};

constexpr int kEvalChunks = 2;          // hg_evaluate pipelines batches in this many chunks
constexpr int64_t kEvalChunkMin = 2048; // ... each at least this many hub sets

struct hg_inst {
    std::atomic<int> refs{1};  // the handle itself + every hg_pop / hg_ga built on it
    // serialises every call that uses the instance's stream, scratch buffers or
    // landing slots: the reference's Instance is safe to share across threads
    // (hm/model.py:35), and ctypes releases the GIL during each call
    std::mutex mu;
    alignas(64) unsigned char wmapp[128]; // CUtensorMap of W8, 64-row boxes (half a tile per CTA)
    alignas(64) unsigned char wmapt[128]; // same over M8
    uint8_t* dW8 = nullptr;                // u8 byte planes of W, [P][npad_tc][npad_tc]
    uint8_t* dM8 = nullptr;                // u8 byte planes of W's triangular fold (symmetric C)
    bool tc_ok = false;                    // K3-TC/P runs this instance (integer flows, p, n)
    int fit_kind = HG_FIT_AUTO;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sm_count = 148;
    int flags = 0;
    DevInst I{};
    FitPlan plan{};
    double* dC = nullptr;
    double* dCt = nullptr;
    double* dW = nullptr;
    double* dO = nullptr;
    double* dD = nullptr;
    double* dwOD = nullptr;
    int32_t* drank = nullptr;
    uint8_t* dpw = nullptr;  // pairwise-sum schedules over n and p*p terms
    uint16_t* dCq = nullptr;
    int* derr = nullptr;  // input-validation flag (DevInst::err)
    int* hflag = nullptr;  // page-locked landing slots for small device->host reads
    hg_pop* scratch = nullptr;
    DevBuf t1, t2, t3, t4;
    // hg_evaluate's copy stream and per-chunk events (copies overlap compute)
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_in[kEvalChunks] = {}, ev_done[kEvalChunks] = {};
    // hg_evaluate's pipeline captured once per (batch, buffers, kernel choice)
    // and replayed with the call's host pointers patched into its copy nodes
    struct EvalGraph {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        int64_t B = -1;
        const void* P = nullptr;  // the scratch population's buffers it was captured on
        const void* Ph = nullptr;
        const void* dsrc = nullptr;
        int kind = -1, exact = -1, kernels = 0;
        bool broken = false;  // capture failed once: stream path from then on
        cudaGraphNode_t h2d[kEvalChunks] = {}, d2h[kEvalChunks] = {};
        int64_t lo[kEvalChunks + 1] = {};
        void release() {
            if (exec) cudaGraphExecDestroy(exec);
            if (graph) cudaGraphDestroy(graph);
            exec = nullptr;
            graph = nullptr;
            B = -1;
        }
    } eg;
};

namespace {

std::unique_lock<std::mutex> lock_of(hg_inst* inst) {
    return inst ? std::unique_lock<std::mutex>(inst->mu) : std::unique_lock<std::mutex>();
}

int set_device(int dev) {
    HG_CUDA(cudaSetDevice(dev));
    return HG_OK;
}

void pop_release(hg_pop* P) {
    if (!P) return;
    cudaFree(P->hubs);
    cudaFree(P->cl);
    cudaFree(P->co);
    cudaFree(P->T);
    cudaFree(P->legs);
    cudaFree(P->part);
    cudaFree(P->out);
    P->alloc.release();
    if (P->evk) cudaEventDestroy(P->evk);
    if (P->ev0) cudaEventDestroy(P->ev0);
    if (P->ev1) cudaEventDestroy(P->ev1);
    P->hubs = nullptr;
    P->cl = nullptr;
    P->co = nullptr;
    P->T = nullptr;
    P->legs = nullptr;
    P->part = nullptr;
    P->out = nullptr;
    P->evk = P->ev0 = P->ev1 = nullptr;
    P->cap = 0;
}

int pop_alloc(hg_pop* P, hg_inst* inst, int64_t cap) {
    const DevInst& I = inst->I;
    P->inst = inst;
    P->cap = 0;  // set once every buffer exists (a failed allocation leaves none usable)
    HG_CUDA(cudaMalloc(&P->hubs, (size_t)cap * I.p * sizeof(int32_t)));
    HG_CUDA(cudaMalloc(&P->cl, (size_t)cap * I.npad));
    HG_CUDA(cudaMalloc(&P->co, (size_t)cap * I.npad * sizeof(uint16_t)));
    HG_CUDA(cudaMalloc(&P->T, (size_t)cap * 2 * I.p * I.ps * sizeof(uint32_t)));
    HG_CUDA(cudaMalloc(&P->legs, (size_t)cap * 2 * sizeof(double)));
    // per-individual partials: fp64 K3 tiles, or the byte planes of K3-TC/P (<= 8)
    int tiles = inst->plan.tiles > tc_tiles(I.n) ? inst->plan.tiles : tc_tiles(I.n);
    if (tiles < 8) tiles = 8;
    HG_CUDA(cudaMalloc(&P->part, (size_t)cap * tiles * sizeof(double)));
    P->tiles = tiles;
    HG_CUDA(cudaMalloc(&P->out, (size_t)cap * 4 * sizeof(double)));
    HG_CUDA(cudaEventCreate(&P->evk));
    HG_CUDA(cudaEventCreate(&P->ev0));
    HG_CUDA(cudaEventCreate(&P->ev1));
    P->cap = cap;
    return HG_OK;
}

int scratch_pop(hg_inst* inst, int64_t B, hg_pop** out) {
    if (!inst->scratch) {
        inst->scratch = new (std::nothrow) hg_pop();
        if (!inst->scratch) {
            set_error("out of host memory");
            return HG_ECUDA;
        }
    }
    hg_pop* P = inst->scratch;
    if (P->cap < B) {
        pop_release(P);
        int64_t cap = B < 64 ? 64 : B;
        const int rc = pop_alloc(P, inst, cap);
        if (rc) {
            pop_release(P);
            return rc;
        }
    }
    *out = P;
    return HG_OK;
}

// the concrete K3 kernel for the instance's choice: HG_FIT_FP64 or HG_FIT_TC_*
// numpy's pairwise_sum_DOUBLE (PW_BLOCKSIZE 128) as a leaf table for m
// terms: the halving tree splits at n2 = m/2 - (m/2) % 8, so every leaf
// starts on a row of 8 terms, holds <= 16 full rows, and only the last leaf
// has a partial row (m % 8 terms).  Per leaf: first row | full rows << 16 |
// the tree sums that follow it << 24 (the last leaf's: all that remain).
static void pw_leaves(int64_t s, int64_t len, std::vector<int64_t>& ls, std::vector<int64_t>& ll,
                      std::vector<int>& lc) {
    if (len <= 128) {
        ls.push_back(s);
        ll.push_back(len);
        lc.push_back(0);
        return;
    }
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    pw_leaves(s, n2, ls, ll, lc);
    pw_leaves(s + n2, len - n2, ls, ll, lc);
    ++lc.back();  // this node's sum follows its right subtree's last leaf
}

static std::vector<uint32_t> pw_leaf_table(int64_t m) {
    std::vector<int64_t> ls, ll;
    std::vector<int> lc;
    pw_leaves(0, m, ls, ll, lc);
    std::vector<uint32_t> t(ls.size());
    for (size_t k = 0; k < ls.size(); ++k)
        t[k] = (uint32_t)(ls[k] / 8) | (uint32_t)(ll[k] / 8) << 16 | (uint32_t)lc[k] << 24;
    return t;
}

static int fitness_kernel(const hg_inst* inst) {
    int k = inst->fit_kind;
    if (k == HG_FIT_AUTO) k = inst->tc_ok ? HG_FIT_TENSOR : HG_FIT_FP64;
    if (k == HG_FIT_TENSOR) k = HG_FIT_TC_PAIR;
    if (k == HG_FIT_TC_PAIR && !inst->dM8) k = HG_FIT_TC_PAIR_FULL;  // asymmetric costs
    return k;
}
// the u16 column offsets K2 can emit are read only by the fp64 K3
static uint16_t* co_for(const hg_inst* inst, uint16_t* co) {
    return fitness_kernel(inst) == HG_FIT_FP64 ? co : nullptr;
}

// the hub-cost tables K2 must write: none when K3-TC/P gathers them from C
static uint32_t* T_for(const hg_inst* inst, int64_t B, uint32_t* T) {
    const int k = fitness_kernel(inst);
    if (k == HG_FIT_FP64) return T;
    return tcp_gathers_T(inst->I, k == HG_FIT_TC_PAIR, B, inst->sm_count) ? nullptr : T;
}

// K3 (fp64 gather) or K3-TC (tensor cores) + finalise, by the instance's choice
int queue_fitness(hg_inst* inst, int64_t B, const int32_t* hubs, const uint8_t* cl,
                  const uint16_t* co, const uint32_t* T, double* part, const double* legs,
                  double* out, const int32_t* dynB = nullptr) {
    const DevInst& I = inst->I;
    cudaStream_t s = inst->stream;
    const int kind = fitness_kernel(inst);
    int tiles;
    if (kind == HG_FIT_TC_PAIR || kind == HG_FIT_TC_PAIR_FULL)  // finaliser fused
        return launch_fitness_tcp(I, inst->wmapp, kind == HG_FIT_TC_PAIR ? inst->wmapt : nullptr,
                                  B, cl, T, part, inst->sm_count, s, legs, out, hubs, dynB);
    HG_ARG(dynB == nullptr, "a device-side batch bound needs the tensor kernel");
    HG_TRY(launch_fitness(I, inst->plan, B, cl, co, T, part,
                          inst->sm_count * inst->plan.blocks_per_sm, s));
    tiles = inst->plan.tiles;
    return launch_finalize(I, tiles, B, legs, part, out, s);
}

// queue K2 + K3 + finalise for individuals [b0, b0 + B) of P whose int32 hubs
// are in P->hubs (alloc32 == nullptr: nearest allocation; otherwise the given
// allocation, rows from b0); events: time K2 and K3 (hg_pop_last_*_ms)
int pop_eval_range(hg_pop* P, int64_t b0, int64_t B, const int32_t* alloc32, bool events,
                   double* out_all = nullptr) {
    hg_inst* inst = P->inst;
    const DevInst& I = inst->I;
    cudaStream_t s = inst->stream;
    const int tiles = P->tiles;
    int32_t* hubs = P->hubs + b0 * I.p;
    uint8_t* cl = P->cl + b0 * I.npad;
    uint16_t* co = co_for(inst, P->co) ? P->co + b0 * I.npad : nullptr;
    uint32_t* T = P->T + b0 * 2 * I.p * (int64_t)I.ps;
    double* legs = P->legs + 2 * b0;
    if (events) HG_CUDA(cudaEventRecord(P->evk, s));
    if (alloc32)
        HG_TRY(launch_from_alloc(I, B, hubs, alloc32 + b0 * I.n, cl, co, T_for(inst, B, T), legs,
                                 s));
    else
        HG_TRY(launch_allocate(I, B, hubs, cl, co, T_for(inst, B, T), legs, nullptr, s));
    if (events) HG_CUDA(cudaEventRecord(P->ev0, s));
    HG_TRY(queue_fitness(inst, B, hubs, cl, co, T, P->part + b0 * tiles, legs,
                         (out_all ? out_all : P->out) + 4 * b0));
    if (events) HG_CUDA(cudaEventRecord(P->ev1, s));
    return HG_OK;
}

int pop_eval_queue(hg_pop* P, int64_t B, const int32_t* alloc32) {
    return pop_eval_range(P, 0, B, alloc32, true);
}

// hg_evaluate's pipeline: chunk c's int64 hub sets cross PCIe on the copy
// stream while chunk c-1 is scored on the instance stream; chunk c's costs go
// back on the copy stream once scored.  The caller reads the flag and
// synchronises the instance stream, which waits for the last copy.
// out_d: the device address of a page-locked `out` -- the finaliser then writes
// the costs straight into it (no copies back)
int eval_pipelined(hg_inst* inst, hg_pop* P, int64_t B, const int64_t* hubs, double* out,
                   double* out_d = nullptr) {
    const DevInst& I = inst->I;
    cudaStream_t s = inst->stream;
    if (!inst->cstream) {
        HG_CUDA(cudaStreamCreateWithFlags(&inst->cstream, cudaStreamNonBlocking));
        for (int c = 0; c < kEvalChunks; ++c) {
            HG_CUDA(cudaEventCreateWithFlags(&inst->ev_in[c], cudaEventDisableTiming));
            HG_CUDA(cudaEventCreateWithFlags(&inst->ev_done[c], cudaEventDisableTiming));
        }
    }
    HG_TRY(inst->t1.ensure((size_t)B * I.p * sizeof(int64_t)));
    int64_t* dsrc = inst->t1.as<int64_t>();
    // the copy stream starts after everything queued before this call
    HG_CUDA(cudaEventRecord(inst->ev_done[kEvalChunks - 1], s));
    HG_CUDA(cudaStreamWaitEvent(inst->cstream, inst->ev_done[kEvalChunks - 1], 0));
    // equal chunks (a first chunk of one K3 wave -- 128/p hub sets per SM,
    // HUBGPU_EVAL_WAVE=1 -- measured 3 % slower end to end: two short launches)
    int64_t lo[kEvalChunks + 1];
    const int64_t ipt = I.p <= 128 ? 128 / I.p : 1;
    static const int wave_first = env_int("HUBGPU_EVAL_WAVE", 0);  // tuning override
    // HUBGPU_EVAL_FIRST=k: a first chunk of B / k (tuning override; default 2)
    static const int first_div = env_int("HUBGPU_EVAL_FIRST", 2);
    const int64_t first = wave_first ? (int64_t)inst->sm_count * ipt
                                     : B / (first_div >= 2 ? first_div : 2);
    lo[0] = 0;
    lo[1] = first < B / 2 ? first : B / 2;
    for (int c = 2; c <= kEvalChunks; ++c) lo[c] = lo[1] + (B - lo[1]) * (c - 1) / (kEvalChunks - 1);
    for (int c = 0; c <= kEvalChunks; ++c) inst->eg.lo[c] = lo[c];
    for (int c = 0; c < kEvalChunks; ++c) {
        const int64_t b0 = lo[c], nb = lo[c + 1] - lo[c];
        HG_CUDA(cudaMemcpyAsync(dsrc + b0 * I.p, hubs + b0 * I.p, (size_t)nb * I.p * sizeof(int64_t),
                                cudaMemcpyHostToDevice, inst->cstream));
        HG_CUDA(cudaEventRecord(inst->ev_in[c], inst->cstream));
    }
    for (int c = 0; c < kEvalChunks; ++c) {
        const int64_t b0 = lo[c], nb = lo[c + 1] - lo[c];
        HG_CUDA(cudaStreamWaitEvent(s, inst->ev_in[c], 0));
        HG_TRY(launch_hubs_in(dsrc + b0 * I.p, P->hubs + b0 * I.p, nb, I.p, I.n, inst->derr, s,
                              b0));
        HG_TRY(pop_eval_range(P, b0, nb, nullptr, false, out_d));
        HG_CUDA(cudaEventRecord(inst->ev_done[c], s));
    }
    if (out_d) return HG_OK;  // nothing to copy back
    // (every kernel is queued before the first copy back: a pageable `out`
    // makes that copy synchronous for the host)
    for (int c = 0; c < kEvalChunks; ++c) {
        const int64_t b0 = lo[c], nb = lo[c + 1] - lo[c];
        HG_CUDA(cudaStreamWaitEvent(inst->cstream, inst->ev_done[c], 0));
        HG_CUDA(cudaMemcpyAsync(out + 4 * b0, P->out + 4 * b0, (size_t)nb * 4 * sizeof(double),
                                cudaMemcpyDeviceToHost, inst->cstream));
    }
    // the instance stream (and its synchronisation) covers the copies back
    HG_CUDA(cudaEventRecord(inst->ev_in[0], inst->cstream));
    HG_CUDA(cudaStreamWaitEvent(s, inst->ev_in[0], 0));
    return HG_OK;
}

// hg_evaluate without copies: K2 reads the caller's page-locked int64 hub
// sets over PCIe while it computes (validating them: the fused k_hubs_in) and
// the fused finaliser writes the costs straight into the caller's page-locked
// result buffer.  hubs_d / out_d are the buffers' device addresses.
int eval_zero_copy(hg_inst* inst, hg_pop* P, int64_t B, const int64_t* hubs_d, double* out_d) {
    DevInst I = inst->I;
    cudaStream_t s = inst->stream;
    I.hubs64 = hubs_d;
    I.hubs_w = P->hubs;
    I.hrow0 = 0;
    HG_CUDA(cudaEventRecord(P->evk, s));
    HG_TRY(launch_allocate(I, B, P->hubs, P->cl, co_for(inst, P->co), T_for(inst, B, P->T),
                           P->legs, nullptr, s));
    HG_CUDA(cudaEventRecord(P->ev0, s));
    HG_TRY(queue_fitness(inst, B, P->hubs, P->cl, P->co, P->T, P->part, P->legs, out_d));
    HG_CUDA(cudaEventRecord(P->ev1, s));
    return HG_OK;
}

// the device address of a page-locked host buffer (nullptr: pageable)
const void* host_mapped(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// the pipeline of eval_pipelined (+ the error-flag read) as a CUDA graph:
// captured on first use for this batch size / scratch buffers / kernel
// choice, then replayed with the call's host pointers set into its four copy
// nodes -- one graph launch instead of ~20 stream operations (host queueing
// dominated the end-to-end overhead).  Page-locked host buffers only.
int eval_graph_run(hg_inst* inst, hg_pop* P, int64_t B, const int64_t* hubs, double* out) {
    const DevInst& I = inst->I;
    cudaStream_t s = inst->stream;
    auto& G = inst->eg;
    HG_TRY(inst->t1.ensure((size_t)B * I.p * sizeof(int64_t)));  // no allocation under capture
    const int64_t* dsrc = inst->t1.as<int64_t>();
    const int kind = fitness_kernel(inst);
    if (!G.exec || G.B != B || G.P != P->out || G.Ph != P->hubs || G.dsrc != dsrc ||
        G.kind != kind || G.exact != I.exact) {
        G.release();
        if (!inst->cstream) {  // created outside the capture
            HG_CUDA(cudaStreamCreateWithFlags(&inst->cstream, cudaStreamNonBlocking));
            for (int c = 0; c < kEvalChunks; ++c) {
                HG_CUDA(cudaEventCreateWithFlags(&inst->ev_in[c], cudaEventDisableTiming));
                HG_CUDA(cudaEventCreateWithFlags(&inst->ev_done[c], cudaEventDisableTiming));
            }
        }
        HG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const uint64_t l0 = launch_count();
        int rc = eval_pipelined(inst, P, B, hubs, out);
        if (!rc && cudaMemcpyAsync(inst->hflag, inst->derr, sizeof(int), cudaMemcpyDeviceToHost,
                                   s) != cudaSuccess)
            rc = HG_ECUDA;
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(s, &g);
        G.kernels = (int)(launch_count() - l0);  // counted again at every replay
        note_launch((uint64_t)0 - (uint64_t)G.kernels);
        if (rc || ce != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            if (!rc) set_error("evaluate graph capture: %s", cudaGetErrorString(ce));
            return rc ? rc : HG_ECUDA;
        }
        G.graph = g;
        // the copy nodes, by device-side address: chunk c's hub sets land at
        // dsrc + lo[c] p, its costs leave from P->out + 4 lo[c]
        size_t nn = 0;
        HG_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        HG_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
        int found = 0;
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            HG_CUDA(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeMemcpy) continue;
            cudaMemcpy3DParms mp = {};
            HG_CUDA(cudaGraphMemcpyNodeGetParams(nd, &mp));
            for (int c = 0; c < kEvalChunks; ++c) {
                if (mp.dstPtr.ptr == (void*)(dsrc + G.lo[c] * I.p)) {
                    G.h2d[c] = nd;
                    ++found;
                }
                if (mp.srcPtr.ptr == (void*)(P->out + 4 * G.lo[c])) {
                    G.d2h[c] = nd;
                    ++found;
                }
            }
        }
        if (found != 2 * kEvalChunks) {
            G.release();
            set_error("evaluate graph: %d of %d copy nodes found", found, 2 * kEvalChunks);
            return HG_ECUDA;
        }
        HG_CUDA(cudaGraphInstantiate(&G.exec, g, 0));
        G.B = B;
        G.P = P->out;
        G.Ph = P->hubs;
        G.dsrc = dsrc;
        G.kind = kind;
        G.exact = I.exact;
    } else {
        for (int c = 0; c < kEvalChunks; ++c) {
            const int64_t b0 = G.lo[c], nb = G.lo[c + 1] - G.lo[c];
            HG_CUDA(cudaGraphExecMemcpyNodeSetParams1D(
                G.exec, G.h2d[c], (void*)(dsrc + b0 * I.p), hubs + b0 * I.p,
                (size_t)nb * I.p * sizeof(int64_t), cudaMemcpyHostToDevice));
            HG_CUDA(cudaGraphExecMemcpyNodeSetParams1D(
                G.exec, G.d2h[c], out + 4 * b0, P->out + 4 * b0, (size_t)nb * 4 * sizeof(double),
                cudaMemcpyDeviceToHost));
        }
    }
    HG_CUDA(cudaGraphLaunch(G.exec, s));
    note_launch((uint64_t)G.kernels);
    return HG_OK;
}

bool host_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// host hub sets / allocations in, validated on the device (see k_hubs_in)
int h2d_hubs_checked(hg_inst* inst, DevBuf& tmp, const int64_t* host, int64_t B, int32_t* dst) {
    const int64_t count = B * inst->I.p;
    HG_TRY(tmp.ensure((size_t)count * sizeof(int64_t)));
    HG_CUDA(cudaMemcpyAsync(tmp.ptr, host, (size_t)count * sizeof(int64_t), cudaMemcpyHostToDevice,
                            inst->stream));
    return launch_hubs_in(tmp.as<int64_t>(), dst, B, inst->I.p, inst->I.n, inst->derr,
                          inst->stream);
}

int h2d_alloc_checked(hg_inst* inst, DevBuf& tmp, const int64_t* host, int64_t B, int32_t* dst) {
    const int64_t count = B * inst->I.n;
    HG_TRY(tmp.ensure((size_t)count * sizeof(int64_t)));
    HG_CUDA(cudaMemcpyAsync(tmp.ptr, host, (size_t)count * sizeof(int64_t), cudaMemcpyHostToDevice,
                            inst->stream));
    return launch_idx_in(tmp.as<int64_t>(), dst, count, inst->I.n, inst->derr, inst->stream);
}

// after the stream is synchronised: report (and clear) a validation failure
int check_input_flag(hg_inst* inst, int host_flag, const char* what) {
    if (host_flag == 0) return HG_OK;
    HG_CUDA(cudaMemsetAsync(inst->derr, 0, sizeof(int), inst->stream));
    HG_CUDA(cudaStreamSynchronize(inst->stream));
    set_error("%s %lld: indices must be sorted ascending, distinct and in [0, %d)", what,
              (long long)(0x7ffffffe - host_flag), inst->I.n);
    return HG_EARG;
}

int d2h_i32_as_i64(hg_inst* inst, DevBuf& tmp, const int32_t* dsrc, int64_t count, int64_t* host) {
    if (count <= 0) return HG_OK;
    HG_TRY(tmp.ensure((size_t)count * sizeof(int64_t)));
    HG_TRY(launch_i32_to_i64(dsrc, tmp.as<int64_t>(), count, inst->stream));
    HG_CUDA(cudaMemcpyAsync(host, tmp.ptr, (size_t)count * sizeof(int64_t), cudaMemcpyDeviceToHost,
                            inst->stream));
    return HG_OK;
}

}  // namespace

// ============================================================================
// exported API
// ============================================================================

extern "C" {

const char* hg_last_error(void) { return hg::g_err; }

int hg_version(void) { return 100; }

int hg_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    if (count) *count = c;
    return HG_OK;
}

int hg_instance_create(int device, int n, int p, const double* dist, const double* flow,
                       const double* out_flow, const double* in_flow, double total_flow,
                       const int64_t* middle_rank, double chi, double alpha, double delta,
                       void* stream, hg_inst** out) {
    (void)total_flow;
    HG_ARG(out != nullptr, "out is NULL");
    *out = nullptr;
    HG_ARG(n >= 1, "node count must be positive, got %d", n);
    HG_ARG(p >= 1 && p <= n, "hub count p=%d outside [1, %d]", p, n);
    HG_ARG(p <= kMaxP, "p=%d exceeds the supported maximum %d", p, kMaxP);
    HG_ARG(n <= kMaxNga, "n=%d exceeds the supported maximum %d", n, kMaxNga);
    HG_ARG(dist && flow && out_flow && in_flow && middle_rank, "NULL instance array");
    int ndev = 0;
    hg_device_count(&ndev);
    if (ndev <= 0) {
        set_error("no CUDA device visible: libhubgpu needs a B200 (sm_100a)");
        return HG_ENODEV;
    }
    HG_ARG(device >= 0 && device < ndev, "device %d outside [0, %d)", device, ndev);
    HG_TRY(set_device(device));

    hg_inst* inst = new (std::nothrow) hg_inst();
    if (!inst) {
        set_error("out of host memory");
        return HG_ECUDA;
    }
    inst->device = device;
    int rc = HG_OK;
    do {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
            set_error("cudaGetDeviceProperties failed");
            rc = HG_ECUDA;
            break;
        }
        inst->sm_count = prop.multiProcessorCount;
        if (stream) {
            inst->stream = static_cast<cudaStream_t>(stream);
        } else {
            if (cudaStreamCreateWithFlags(&inst->stream, cudaStreamNonBlocking) != cudaSuccess) {
                set_error("cudaStreamCreate failed");
                rc = HG_ECUDA;
                break;
            }
            inst->own_stream = true;
        }
        const size_t nn = (size_t)n * n;
        cudaStream_t s = inst->stream;
        auto chk = [&](cudaError_t e, const char* what) {
            if (e != cudaSuccess && rc == HG_OK) {
                set_error("%s: %s", what, cudaGetErrorString(e));
                rc = HG_ECUDA;
            }
        };
        chk(cudaMalloc(&inst->dC, nn * 8), "cudaMalloc(dist)");
        chk(cudaMalloc(&inst->dW, nn * 8), "cudaMalloc(flow)");
        // O and D zero-padded to a multiple of 4 nodes (K2 reads them 4 at a time)
        const size_t n4 = ((size_t)n + 3) & ~size_t(3);
        chk(cudaMalloc(&inst->dO, n4 * 8), "cudaMalloc");
        chk(cudaMalloc(&inst->dD, n4 * 8), "cudaMalloc");
        if (rc) break;
        chk(cudaMemsetAsync(inst->dO, 0, n4 * 8, s), "memset");
        chk(cudaMemsetAsync(inst->dD, 0, n4 * 8, s), "memset");
        chk(cudaMalloc(&inst->dwOD, (size_t)n * 8), "cudaMalloc");
        chk(cudaMalloc(&inst->drank, (size_t)n * 4), "cudaMalloc");
        if (rc) break;
        chk(cudaMemcpyAsync(inst->dC, dist, nn * 8, cudaMemcpyHostToDevice, s), "H2D dist");
        chk(cudaMemcpyAsync(inst->dW, flow, nn * 8, cudaMemcpyHostToDevice, s), "H2D flow");
        chk(cudaMemcpyAsync(inst->dO, out_flow, (size_t)n * 8, cudaMemcpyHostToDevice, s), "H2D");
        chk(cudaMemcpyAsync(inst->dD, in_flow, (size_t)n * 8, cudaMemcpyHostToDevice, s), "H2D");
        // correction weights O_i + D_i (hm/operators.py:94), exactness of order-free sums
        std::vector<double> w(n);
        std::vector<int32_t> rk(n);
        bool exact = true;
        double tot = 0.0;
        for (int i = 0; i < n; ++i) {
            w[i] = out_flow[i] + in_flow[i];
            if (!(w[i] == std::floor(w[i])) || w[i] < 0) exact = false;
            tot += w[i];
            rk[i] = (int32_t)middle_rank[i];
        }
        if (!(tot < 9007199254740992.0)) exact = false;
        chk(cudaMemcpyAsync(inst->dwOD, w.data(), (size_t)n * 8, cudaMemcpyHostToDevice, s),
            "H2D");
        chk(cudaMemcpyAsync(inst->drank, rk.data(), (size_t)n * 4, cudaMemcpyHostToDevice, s),
            "H2D");
        // one device pass over C and W (K1): cost range, symmetry, flow class
        InstanceScan* dscan = nullptr;
        chk(cudaMalloc(&dscan, sizeof(InstanceScan)), "cudaMalloc");
        if (rc) break;
        if (rc == HG_OK) rc = launch_scan_instance(inst->dC, inst->dW, n, dscan, s);
        InstanceScan scan{};
        chk(cudaMemcpyAsync(&scan, dscan, sizeof(scan), cudaMemcpyDeviceToHost, s), "D2H");
        chk(cudaStreamSynchronize(s), "sync");
        cudaFree(dscan);
        if (rc) break;
        auto from_bits = [](unsigned long long b) {
            double v;
            std::memcpy(&v, &b, sizeof(v));
            return v;
        };
        const int sym = scan.symmetric;
        if (sym) {
            inst->dCt = inst->dC;
        } else {
            chk(cudaMalloc(&inst->dCt, nn * 8), "cudaMalloc(dist^T)");
            if (rc) break;
            rc = launch_transpose(inst->dC, inst->dCt, n, s);
            if (rc) break;
        }
        inst->flags = (sym ? HG_FLAG_SYMMETRIC : 0) | (exact ? HG_FLAG_WEIGHTS_EXACT : 0);

        DevInst& I = inst->I;
        I.n = n;
        I.p = p;
        I.nw = (n + 31) / 32;
        I.ps = (p + 3) & ~3;
        I.weights_exact = exact ? 1 : 0;
        I.chi = chi;
        I.alpha = alpha;
        I.delta = delta;
        I.C = inst->dC;
        I.Ct = inst->dCt;
        I.W = inst->dW;
        I.O = inst->dO;
        I.D = inst->dD;
        I.wOD = inst->dwOD;
        I.rank = inst->drank;
        {
            const std::vector<uint32_t> pn = pw_leaf_table(n);
            const std::vector<uint32_t> pl = pw_leaf_table((int64_t)p * p);
            chk(cudaMalloc(&inst->dpw, (pn.size() + pl.size()) * 4), "cudaMalloc(pw)");
            if (rc) break;
            chk(cudaMemcpy(inst->dpw, pn.data(), pn.size() * 4, cudaMemcpyHostToDevice), "H2D pw");
            chk(cudaMemcpy(inst->dpw + pn.size() * 4, pl.data(), pl.size() * 4,
                           cudaMemcpyHostToDevice),
                "H2D pw");
            I.pwnl = reinterpret_cast<const uint32_t*>(inst->dpw);
            I.npwnl = (int)pn.size();
            I.pwl = reinterpret_cast<const uint32_t*>(inst->dpw + pn.size() * 4);
            I.npwl = (int)pl.size();
        }
        chk(cudaMalloc(&inst->derr, sizeof(int)), "cudaMalloc(err)");
        chk(cudaHostAlloc(reinterpret_cast<void**>(&inst->hflag), 4 * sizeof(int),
                          cudaHostAllocDefault), "cudaHostAlloc(flag)");
        chk(cudaMemsetAsync(inst->derr, 0, sizeof(int), s), "memset(err)");
        I.err = inst->derr;
        I.npad = 16;  // provisional for the plan
        inst->plan = fitness_plan(I, inst->sm_count);
        int64_t q = inst->plan.tr > inst->plan.tc ? inst->plan.tr : inst->plan.tc;
        if (q < 128) q = 128;  // K3-TC reads 128-wide K blocks of cluster ids
        I.npad = (int)round_up(n, q);
        {
            // 16-bit monotone quantisation of Ct: exact pre-filter for allocation
            const double cmin = from_bits(scan.cmin_bits), cmax = from_bits(scan.cmax_bits);
            const double scale = cmax > cmin ? 65535.0 / (cmax - cmin) : 0.0;
            // rows padded with 0xFFFF to nq = npad (K2 reads whole passes of
            // nodes unguarded), one all-0xFFFF row n (the register K2's
            // stand-in for hub slots >= p), plus slack for the tail
            const int nq = I.npad;
            const size_t cq_elems = (size_t)(n + 1) * nq + 2048;
            chk(cudaMalloc(&inst->dCq, cq_elems * sizeof(uint16_t)), "cudaMalloc(Cq)");
            if (rc) break;
            chk(cudaMemsetAsync(inst->dCq, 0xff, cq_elems * sizeof(uint16_t), s), "memset(Cq)");
            if (rc) break;
            rc = launch_quantize(inst->dCt, inst->dCq, n, nq, cmin, scale, s);
            if (rc) break;
            I.Cq = inst->dCq;
            I.nq = nq;
            if (rc) break;
        }
        rc = prepare_fitness(inst->plan);
        if (rc) break;
        rc = prepare_allocate(I);
        if (rc) break;
        // K3-TC eligibility.  Integer flows below 2^32 (or such integers times
        // a power of two): exact u8 GEMMs on P byte planes of W (P = 1 when
        // every flow < 256).  Other flows: the
        // planes of Q = rint(W / q), q a power of two small enough that every
        // nonzero flow keeps 2^-41 relative precision (each term W_ij * T of
        // the non-negative transfer sum then within 2^-41, so the sum too),
        // when that takes at most 8 planes.  Symmetric costs: also the planes
        // of the triangular fold of Q.
        const double wmax = from_bits(scan.wmax_bits), mmax = from_bits(scan.mmax_bits);
        const double wmin = scan.wmin_bits == ~0ull ? wmax : from_bits(scan.wmin_bits);
        // flows that are integer multiples of 2^e (e = the lowest set bit over
        // all of them) below 2^32 * 2^e: exact integers Q = W / 2^e
        int P = 1, Pt = 1;
        double qscale = 1.0;
        bool intw = scan.int_flows != 0;
        if (!intw && scan.lsb_exp < 0 && wmax > 0.0 &&
            wmax < std::ldexp(4294967296.0, scan.lsb_exp)) {
            intw = true;
            qscale = std::ldexp(1.0, scan.lsb_exp);
        }
        // every byte plane's total below 2^32: u32 bins may accumulate over
        // all K chunks (the exact transfer sum for n > 1024)
        I.bins_total_ok = intw && scan.wsum / qscale < 4294967296.0 ? 1 : 0;
        I.int_flows = intw ? 1 : 0;
        bool planes_ok = p >= 1 && p <= 128 && wmax > 0.0;
        if (intw) {
            while (P < 4 && wmax / qscale >= std::ldexp(1.0, 8 * P)) ++P;
        } else if (planes_ok) {
            const int E = std::ilogb(wmax) + 1;                       // wmax < 2^E
            const double range = std::log2(wmax / wmin);
            P = (int)std::ceil((range + 42.0) / 8.0);
            if (P < 1) P = 1;
            planes_ok = P <= 8;
            qscale = std::ldexp(1.0, E - 8 * P);                    // max Q < 2^(8P)
        }
        const double mq = mmax / qscale + 2.0;  // bound on the fold's quantised entries
        while (Pt < 9 && mq >= std::ldexp(1.0, 8 * Pt)) ++Pt;
        I.wplanes = P;
        I.wscale = qscale;
        const bool tri = sym && Pt <= 8 && !env_int("HUBGPU_TCP_NOTRI", 0);
        I.wplanes_tri = tri ? Pt : 0;
        if (planes_ok && tcp_supported(n, p, I.npad, P) &&
            (!tri || tcp_supported(n, p, I.npad, Pt))) {
            const int nt = (int)round_up(n, 128);
            const size_t plane = (size_t)nt * nt;
            chk(cudaMalloc(&inst->dW8, plane * P), "cudaMalloc(W8)");
            if (tri) chk(cudaMalloc(&inst->dM8, plane * Pt), "cudaMalloc(M8)");
            if (rc) break;
            rc = launch_build_planes(inst->dW, n, nt, qscale, P, Pt, inst->dW8,
                                     tri ? inst->dM8 : nullptr, s);
            if (rc) break;
            rc = tc_make_wmap(inst->dW8, nt, 64, inst->wmapp, P * nt);
            if (rc) break;
            if (tri) {
                rc = tc_make_wmap(inst->dM8, nt, 64, inst->wmapt, Pt * nt);
                if (rc) break;
            }
            rc = prepare_fitness_tcp(p, I.npad, tri && Pt > P ? Pt : P);
            if (rc) break;
            inst->tc_ok = true;
        }
        chk(cudaStreamSynchronize(s), "sync");
    } while (0);
    if (rc != HG_OK) {
        hg_instance_free(inst);
        return rc;
    }
    *out = inst;
    return HG_OK;
}

static void inst_destroy(hg_inst* inst) {
    cudaSetDevice(inst->device);
    if (inst->stream) cudaStreamSynchronize(inst->stream);
    if (inst->scratch) {
        pop_release(inst->scratch);
        delete inst->scratch;
    }
    if (inst->dCt && inst->dCt != inst->dC) cudaFree(inst->dCt);
    cudaFree(inst->dC);
    cudaFree(inst->dW);
    cudaFree(inst->dO);
    cudaFree(inst->dD);
    cudaFree(inst->dwOD);
    cudaFree(inst->drank);
    cudaFree(inst->dpw);
    cudaFree(inst->dCq);
    cudaFree(inst->derr);
    if (inst->hflag) cudaFreeHost(inst->hflag);
    cudaFree(inst->dW8);
    cudaFree(inst->dM8);
    inst->eg.release();
    if (inst->cstream) {
        cudaStreamSynchronize(inst->cstream);
        cudaStreamDestroy(inst->cstream);
        for (int c = 0; c < kEvalChunks; ++c) {
            cudaEventDestroy(inst->ev_in[c]);
            cudaEventDestroy(inst->ev_done[c]);
        }
    }
    inst->t1.release();
    inst->t2.release();
    inst->t3.release();
    inst->t4.release();
    if (inst->own_stream && inst->stream) cudaStreamDestroy(inst->stream);
    delete inst;
}

static void inst_release(hg_inst* inst) {
    if (inst && inst->refs.fetch_sub(1) == 1) inst_destroy(inst);
}

void hg_instance_free(hg_inst* inst) { inst_release(inst); }

int hg_instance_info(const hg_inst* inst, int* n, int* p, int* flags) {
    HG_ARG(inst != nullptr, "instance is NULL");
    if (n) *n = inst->I.n;
    if (p) *p = inst->I.p;
    if (flags) *flags = inst->flags | (inst->tc_ok ? HG_FLAG_TENSOR_OK : 0);
    return HG_OK;
}

int hg_instance_set_exact(hg_inst* inst, int on) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst != nullptr, "instance is NULL");
    inst->I.exact = on ? 1 : 0;
    return HG_OK;
}

int hg_instance_exact(const hg_inst* inst, int* on) {
    HG_ARG(inst != nullptr && on != nullptr, "NULL argument");
    *on = inst->I.exact;
    return HG_OK;
}

int hg_instance_set_fitness(hg_inst* inst, int kind) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst != nullptr, "instance is NULL");
    HG_ARG(kind == HG_FIT_AUTO || kind == HG_FIT_FP64 || kind == HG_FIT_TENSOR ||
               kind == HG_FIT_TC_PAIR || kind == HG_FIT_TC_PAIR_FULL,
           "unknown fitness kernel %d", kind);
    HG_ARG(kind < HG_FIT_TENSOR || inst->tc_ok,
           "tensor-core fitness needs p <= 128, n <= 16384 and flows whose nonzero range "
           "fits 8 byte planes at 2^-41 relative precision");
    inst->fit_kind = kind;
    return HG_OK;
}

int hg_instance_fitness(const hg_inst* inst, int* kind) {
    HG_ARG(inst && kind, "NULL argument");
    *kind = fitness_kernel(inst);
    return HG_OK;
}

int hg_instance_stream(const hg_inst* inst, void** stream) {
    HG_ARG(inst != nullptr && stream != nullptr, "NULL argument");
    *stream = inst->stream;
    return HG_OK;
}

int hg_synchronize(hg_inst* inst) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst != nullptr, "instance is NULL");
    HG_TRY(set_device(inst->device));
    HG_CUDA(cudaStreamSynchronize(inst->stream));
    return HG_OK;
}

int hg_allocate(hg_inst* inst, int64_t B, const int64_t* hubs, int64_t* alloc) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst != nullptr, "instance is NULL");
    HG_ARG(B >= 0, "negative batch");
    if (B == 0) return HG_OK;
    HG_ARG(hubs && alloc, "NULL buffer");
    HG_TRY(set_device(inst->device));
    hg_pop* P;
    HG_TRY(scratch_pop(inst, B, &P));
    const DevInst& I = inst->I;
    HG_TRY(h2d_hubs_checked(inst, inst->t1, hubs, B, P->hubs));
    HG_TRY(P->alloc.ensure((size_t)B * I.n * sizeof(int32_t)));
    HG_TRY(launch_allocate(I, B, P->hubs, P->cl, P->co, P->T, nullptr, P->alloc.as<int32_t>(),
                           inst->stream));
    HG_TRY(d2h_i32_as_i64(inst, inst->t2, P->alloc.as<int32_t>(), B * I.n, alloc));
    HG_CUDA(cudaMemcpyAsync(inst->hflag, inst->derr, sizeof(int), cudaMemcpyDeviceToHost,
                            inst->stream));
    HG_CUDA(cudaStreamSynchronize(inst->stream));
    const int flag = inst->hflag[0];
    return check_input_flag(inst, flag, "hub set");
}

int hg_evaluate(hg_inst* inst, int64_t B, const int64_t* hubs, const int64_t* alloc,
                double* out) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst != nullptr, "instance is NULL");
    HG_ARG(B >= 0, "negative batch");
    if (B == 0) return HG_OK;
    HG_ARG(hubs && out, "NULL buffer");
    HG_TRY(set_device(inst->device));
    hg_pop* P;
    HG_TRY(scratch_pop(inst, B, &P));
    const DevInst& I = inst->I;
    // HUBGPU_E2E_TRACE=1: device phase times of this call on stderr (tuning)
    static const bool trace = getenv("HUBGPU_E2E_TRACE") != nullptr;
    cudaEvent_t te[3] = {nullptr, nullptr, nullptr};
    const auto h0 = std::chrono::steady_clock::now();
    if (trace)
        for (auto& e : te) cudaEventCreate(&e);
    if (trace) cudaEventRecord(te[0], inst->stream);
    static const int chunked = env_int("HUBGPU_EVAL_CHUNKS", 1);  // tuning override: 0 = off
    const bool piped = !alloc && chunked && B >= kEvalChunks * kEvalChunkMin;
    static const int graphed = env_int("HUBGPU_EVAL_GRAPH", 1);  // tuning override: 0 = off
    // HUBGPU_EVAL_ZEROCOPY=1: no copies (measured slower end to end: K2's
    // warps all start on a PCIe read of their hub set, 313 vs 258 us per 8192)
    static const int zcopy = env_int("HUBGPU_EVAL_ZEROCOPY", 0);
    const int64_t* hubs_d = nullptr;
    double* out_d = nullptr;
    if (!alloc && zcopy) {
        hubs_d = static_cast<const int64_t*>(host_mapped(hubs));
        out_d = hubs_d ? static_cast<double*>(const_cast<void*>(host_mapped(out))) : nullptr;
    }
    const bool use_zc = hubs_d && out_d;
    const bool use_graph = !use_zc && piped && graphed && !trace && !inst->eg.broken &&
                           host_pinned(hubs) && host_pinned(out);
    if (use_zc) {
        // page-locked hub sets and results: no copies at all
        HG_TRY(eval_zero_copy(inst, P, B, hubs_d, out_d));
    } else if (use_graph) {
        // (the same pipeline, replayed as one graph; it reads the error flag too)
        if (eval_graph_run(inst, P, B, hubs, out) != HG_OK) {
            // a pipeline that cannot be captured (or replayed) here: the stream
            // path, for this and every later call on the instance
            inst->eg.release();
            inst->eg.broken = true;
            cudaGetLastError();
            HG_TRY(eval_pipelined(inst, P, B, hubs, out));
            HG_CUDA(cudaMemcpyAsync(inst->hflag, inst->derr, sizeof(int), cudaMemcpyDeviceToHost,
                                    inst->stream));
        }
    } else if (piped) {
        // the hub sets in chunks on the copy stream, each chunk scored as soon
        // as it lands and its costs copied back while the next one is scored
        // (the PCIe transfers hide under the kernels).  HUBGPU_EVAL_ZCOUT=1:
        // costs written by the finaliser into a page-locked `out` directly
        static const int zcout = env_int("HUBGPU_EVAL_ZCOUT", 0);
        double* od = zcout ? static_cast<double*>(const_cast<void*>(host_mapped(out))) : nullptr;
        HG_TRY(eval_pipelined(inst, P, B, hubs, out, od));
    } else {
        HG_TRY(h2d_hubs_checked(inst, inst->t1, hubs, B, P->hubs));
        const int32_t* a32 = nullptr;
        if (alloc) {
            HG_TRY(P->alloc.ensure((size_t)B * I.n * sizeof(int32_t)));
            HG_TRY(h2d_alloc_checked(inst, inst->t2, alloc, B, P->alloc.as<int32_t>()));
            a32 = P->alloc.as<int32_t>();
        }
        HG_TRY(pop_eval_queue(P, B, a32));
        if (trace) cudaEventRecord(te[1], inst->stream);
        HG_CUDA(cudaMemcpyAsync(out, P->out, (size_t)B * 4 * sizeof(double),
                                cudaMemcpyDeviceToHost, inst->stream));
    }
    if (!use_graph)
        HG_CUDA(cudaMemcpyAsync(inst->hflag, inst->derr, sizeof(int), cudaMemcpyDeviceToHost,
                                inst->stream));
    if (trace) cudaEventRecord(te[2], inst->stream);
    const auto h1 = std::chrono::steady_clock::now();
    HG_CUDA(cudaStreamSynchronize(inst->stream));
    if (trace) {
        const auto h2 = std::chrono::steady_clock::now();
        float in_ms = 0, k2_ms = 0, k3_ms = 0, tot_ms = 0, out_ms = 0;
        if (!piped) {
            cudaEventElapsedTime(&in_ms, te[0], P->evk);
            cudaEventElapsedTime(&k2_ms, P->evk, P->ev0);
            cudaEventElapsedTime(&k3_ms, P->ev0, P->ev1);
            cudaEventElapsedTime(&out_ms, te[1], te[2]);
        }
        cudaEventElapsedTime(&tot_ms, te[0], te[2]);
        fprintf(stderr,
                "hg_evaluate B=%lld: device: in %.1f us, K2 %.1f, K3 %.1f, out %.1f, total %.1f; "
                "host: queue %.1f us, wait %.1f us\n",
                (long long)B, in_ms * 1e3, k2_ms * 1e3, k3_ms * 1e3, out_ms * 1e3, tot_ms * 1e3,
                std::chrono::duration<double, std::micro>(h1 - h0).count(),
                std::chrono::duration<double, std::micro>(h2 - h1).count());
        for (auto& e : te) cudaEventDestroy(e);
    }
    const int flag = inst->hflag[0];
    return check_input_flag(inst, flag, alloc ? "solution" : "hub set");
}

int hg_evaluate_unique(hg_inst* inst, int64_t B, const int64_t* hubs, double* out,
                       int64_t* groups) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst != nullptr, "instance is NULL");
    HG_ARG(B >= 0, "negative batch");
    if (groups) *groups = 0;
    if (B == 0) return HG_OK;
    HG_ARG(hubs && out, "NULL buffer");
    HG_TRY(set_device(inst->device));
    hg_pop* P;
    HG_TRY(scratch_pop(inst, B, &P));
    const DevInst& I = inst->I;
    cudaStream_t s = inst->stream;
    // all hub sets (validated) -> t3; grouping scratch, map, count, full results -> t4
    HG_TRY(inst->t3.ensure((size_t)B * I.p * sizeof(int32_t)));
    int32_t* all = inst->t3.as<int32_t>();
    HG_TRY(h2d_hubs_checked(inst, inst->t1, hubs, B, all));
    const size_t gbytes = (unique_scratch_bytes(B) + 255) & ~size_t(255);
    HG_TRY(inst->t4.ensure(gbytes + (size_t)B * 4 + 16 + (size_t)B * 32 + 256));
    unsigned char* w = inst->t4.as<unsigned char>();
    int32_t* map = reinterpret_cast<int32_t*>(w + gbytes);
    int32_t* dcount = map + B + (B & 1);  // 8-byte aligned
    double* full = reinterpret_cast<double*>(
        w + ((gbytes + (size_t)B * 4 + 16 + 255) & ~size_t(255)));
    HG_TRY(launch_unique_groups(all, B, I.p, w, gbytes, P->hubs, map, dcount, s));
    int* hc = inst->hflag;
    HG_CUDA(cudaMemcpyAsync(hc, dcount, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaMemcpyAsync(hc + 2, inst->derr, sizeof(int), cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaStreamSynchronize(s));
    HG_TRY(check_input_flag(inst, hc[2], "hub set"));
    const int64_t U = (int64_t)hc[0] + hc[1];
    HG_TRY(pop_eval_queue(P, U, nullptr));
    HG_TRY(launch_scatter_out(P->out, map, B, full, s));
    HG_CUDA(cudaMemcpyAsync(out, full, (size_t)B * 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaStreamSynchronize(s));
    if (groups) *groups = U;
    return HG_OK;
}

int hg_pop_create(hg_inst* inst, int64_t capacity, hg_pop** out) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst && out, "NULL argument");
    HG_ARG(capacity >= 1, "capacity must be >= 1");
    HG_TRY(set_device(inst->device));
    hg_pop* P = new (std::nothrow) hg_pop();
    if (!P) {
        set_error("out of host memory");
        return HG_ECUDA;
    }
    int rc = pop_alloc(P, inst, capacity);
    if (rc) {
        pop_release(P);
        delete P;
        return rc;
    }
    inst->refs.fetch_add(1);
    *out = P;
    return HG_OK;
}

void hg_pop_free(hg_pop* pop) {
    if (!pop) return;
    hg_inst* inst = pop->inst;
    {
        auto lk_ = lock_of(inst);
        cudaSetDevice(inst->device);
        cudaStreamSynchronize(inst->stream);
        pop_release(pop);
        delete pop;
    }
    inst_release(inst);
}

int hg_pop_load_hubs(hg_pop* pop, int64_t B, const int32_t* hubs, int where) {
    auto lk_ = lock_of(pop ? pop->inst : nullptr);
    HG_ARG(pop && hubs, "NULL argument");
    HG_ARG(B >= 0 && B <= pop->cap, "batch %lld outside [0, %lld]", (long long)B,
           (long long)pop->cap);
    HG_TRY(set_device(pop->inst->device));
    const size_t bytes = (size_t)B * pop->inst->I.p * sizeof(int32_t);
    HG_CUDA(cudaMemcpyAsync(pop->hubs, hubs, bytes,
                            where == HG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            pop->inst->stream));
    return HG_OK;
}

int hg_pop_evaluate(hg_pop* pop, int64_t B) {
    auto lk_ = lock_of(pop ? pop->inst : nullptr);
    HG_ARG(pop != nullptr, "NULL population");
    HG_ARG(B >= 0 && B <= pop->cap, "batch outside capacity");
    if (B == 0) return HG_OK;
    HG_TRY(set_device(pop->inst->device));
    return pop_eval_queue(pop, B, nullptr);
}

int hg_pop_read(hg_pop* pop, int64_t B, double* out, int where) {
    auto lk_ = lock_of(pop ? pop->inst : nullptr);
    HG_ARG(pop && out, "NULL argument");
    HG_ARG(B >= 0 && B <= pop->cap, "batch outside capacity");
    HG_TRY(set_device(pop->inst->device));
    HG_CUDA(cudaMemcpyAsync(out, pop->out, (size_t)B * 4 * sizeof(double),
                            where == HG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                            pop->inst->stream));
    if (where != HG_DEVICE) HG_CUDA(cudaStreamSynchronize(pop->inst->stream));
    return HG_OK;
}

int hg_fitness_work(hg_inst* inst, int64_t B, double* mma_ops) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst != nullptr && mma_ops != nullptr, "NULL argument");
    HG_ARG(B >= 0, "negative batch");
    const int k = fitness_kernel(inst);
    *mma_ops = k == HG_FIT_FP64 ? 0.0
                                : tcp_mma_ops(inst->I, k == HG_FIT_TC_PAIR, B, inst->sm_count);
    return HG_OK;
}

int hg_launch_count(uint64_t* count) {
    HG_ARG(count != nullptr, "NULL argument");
    *count = launch_count();
    return HG_OK;
}

int hg_debug_tc_timing(unsigned long long* out32) {
    HG_ARG(out32 != nullptr, "NULL buffer");
    return tc_timing_read(out32);
}

int hg_debug_tc_trace(unsigned long long* out) {
    HG_ARG(out != nullptr, "NULL buffer");
    return tc_trace_read(out);
}

int hg_pop_launches_per_evaluate(const hg_pop* pop) {
    return fitness_kernel(pop->inst) == HG_FIT_FP64 ? 3 : 2;
}

int hg_pop_last_allocate_ms(hg_pop* pop, float* ms) {
    auto lk_ = lock_of(pop ? pop->inst : nullptr);
    HG_ARG(pop && ms, "NULL argument");
    HG_TRY(set_device(pop->inst->device));
    HG_CUDA(cudaEventSynchronize(pop->ev0));
    HG_CUDA(cudaEventElapsedTime(ms, pop->evk, pop->ev0));
    return HG_OK;
}

int hg_pop_last_fitness_ms(hg_pop* pop, float* ms) {
    auto lk_ = lock_of(pop ? pop->inst : nullptr);
    HG_ARG(pop && ms, "NULL argument");
    HG_TRY(set_device(pop->inst->device));
    HG_CUDA(cudaEventSynchronize(pop->ev1));
    HG_CUDA(cudaEventElapsedTime(ms, pop->ev0, pop->ev1));
    return HG_OK;
}

int hg_correct(hg_inst* inst, int64_t B, const uint8_t* masks, int64_t* hubs_out) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst != nullptr, "instance is NULL");
    HG_ARG(B >= 0, "negative batch");
    if (B == 0) return HG_OK;
    HG_ARG(masks && hubs_out, "NULL buffer");
    HG_TRY(set_device(inst->device));
    const DevInst& I = inst->I;
    cudaStream_t s = inst->stream;
    HG_TRY(inst->t1.ensure((size_t)B * I.n));
    HG_TRY(inst->t2.ensure((size_t)B * I.nw * 4));
    HG_TRY(inst->t3.ensure((size_t)B * I.p * 4));
    HG_CUDA(cudaMemcpyAsync(inst->t1.ptr, masks, (size_t)B * I.n, cudaMemcpyHostToDevice, s));
    HG_TRY(launch_bytes_to_bits(inst->t1.as<uint8_t>(), inst->t2.as<uint32_t>(), B, I.n, I.nw, s));
    HG_TRY(launch_correct(I, B, inst->t2.as<uint32_t>(), I.n, inst->t3.as<int32_t>(), s));
    HG_TRY(d2h_i32_as_i64(inst, inst->t4, inst->t3.as<int32_t>(), B * I.p, hubs_out));
    HG_CUDA(cudaStreamSynchronize(s));
    return HG_OK;
}

// per-device scratch for the instance-free operators (serialised by a mutex)
struct OpScratch {
    bool init = false;
    cudaStream_t stream = nullptr;
    DevBuf t1, t2, t3;
};
static std::mutex g_op_mutex;
static OpScratch g_op[64];

static int op_scratch(int device, OpScratch** out) {
    int ndev = 0;
    hg_device_count(&ndev);
    if (ndev <= 0) {
        set_error("no CUDA device visible: libhubgpu needs a B200 (sm_100a)");
        return HG_ENODEV;
    }
    HG_ARG(device >= 0 && device < ndev && device < 64, "device %d outside [0, %d)", device, ndev);
    HG_TRY(set_device(device));
    OpScratch& S = g_op[device];
    if (!S.init) {
        HG_CUDA(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
        S.init = true;
    }
    *out = &S;
    return HG_OK;
}

int hg_crossover(int device, int n, int64_t B, const uint8_t* a, const uint8_t* b,
                 const int64_t* cuts, uint8_t* child1, uint8_t* child2) {
    HG_ARG(n >= 1, "mask length must be positive");
    HG_ARG(B >= 0, "negative batch");
    if (B == 0) return HG_OK;
    HG_ARG(a && b && cuts && child1 && child2, "NULL buffer");
    for (int64_t x = 0; x < B; ++x)
        HG_ARG(cuts[x] >= 1 && cuts[x] <= n, "cut %lld outside [1, %d]", (long long)cuts[x], n);
    std::lock_guard<std::mutex> lock(g_op_mutex);
    OpScratch* S;
    HG_TRY(op_scratch(device, &S));
    const int nw = (n + 31) / 32;
    cudaStream_t s = S->stream;
    const size_t mb = (size_t)B * n, W = (size_t)B * nw;
    HG_TRY(S->t1.ensure(2 * mb));
    HG_TRY(S->t2.ensure(4 * W * 4));
    HG_TRY(S->t3.ensure((size_t)B * 8));
    uint8_t* dbytes = S->t1.as<uint8_t>();
    uint32_t* dbits = S->t2.as<uint32_t>();
    HG_CUDA(cudaMemcpyAsync(dbytes, a, mb, cudaMemcpyHostToDevice, s));
    HG_CUDA(cudaMemcpyAsync(dbytes + mb, b, mb, cudaMemcpyHostToDevice, s));
    HG_CUDA(cudaMemcpyAsync(S->t3.ptr, cuts, (size_t)B * 8, cudaMemcpyHostToDevice, s));
    HG_TRY(launch_bytes_to_bits(dbytes, dbits, B, n, nw, s));
    HG_TRY(launch_bytes_to_bits(dbytes + mb, dbits + W, B, n, nw, s));
    HG_TRY(launch_splice(B, n, nw, dbits, dbits + W, S->t3.as<int64_t>(), dbits + 2 * W,
                         dbits + 3 * W, s));
    HG_TRY(launch_bits_to_bytes(dbits + 2 * W, dbytes, B, n, nw, s));
    HG_TRY(launch_bits_to_bytes(dbits + 3 * W, dbytes + mb, B, n, nw, s));
    HG_CUDA(cudaMemcpyAsync(child1, dbytes, mb, cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaMemcpyAsync(child2, dbytes + mb, mb, cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaStreamSynchronize(s));
    return HG_OK;
}

int hg_swap(int device, int n, int64_t B, const uint8_t* masks, const int64_t* r_close,
            const int64_t* r_open, uint8_t* out) {
    HG_ARG(n >= 1, "mask length must be positive");
    HG_ARG(B >= 0, "negative batch");
    if (B == 0) return HG_OK;
    HG_ARG(masks && r_close && r_open && out, "NULL buffer");
    for (int64_t x = 0; x < B; ++x) {
        if (r_close[x] < 0) continue;
        int64_t on = 0;
        for (int i = 0; i < n; ++i) on += masks[x * n + i] ? 1 : 0;
        HG_ARG(on > 0 && on < n, "swap on an all-open/all-closed mask needs r_close < 0");
        HG_ARG(r_close[x] < on && r_open[x] >= 0 && r_open[x] < n - on,
               "swap draw outside its bound");
    }
    std::lock_guard<std::mutex> lock(g_op_mutex);
    OpScratch* S;
    HG_TRY(op_scratch(device, &S));
    const int nw = (n + 31) / 32;
    cudaStream_t s = S->stream;
    const size_t mb = (size_t)B * n;
    HG_TRY(S->t1.ensure(mb));
    HG_TRY(S->t2.ensure((size_t)B * nw * 4));
    HG_TRY(S->t3.ensure((size_t)B * 16));
    int64_t* dr = S->t3.as<int64_t>();
    HG_CUDA(cudaMemcpyAsync(S->t1.ptr, masks, mb, cudaMemcpyHostToDevice, s));
    HG_CUDA(cudaMemcpyAsync(dr, r_close, (size_t)B * 8, cudaMemcpyHostToDevice, s));
    HG_CUDA(cudaMemcpyAsync(dr + B, r_open, (size_t)B * 8, cudaMemcpyHostToDevice, s));
    HG_TRY(launch_bytes_to_bits(S->t1.as<uint8_t>(), S->t2.as<uint32_t>(), B, n, nw, s));
    HG_TRY(launch_swap_given(B, n, nw, S->t2.as<uint32_t>(), dr, dr + B, s));
    HG_TRY(launch_bits_to_bytes(S->t2.as<uint32_t>(), S->t1.as<uint8_t>(), B, n, nw, s));
    HG_CUDA(cudaMemcpyAsync(out, S->t1.ptr, mb, cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaStreamSynchronize(s));
    return HG_OK;
}

}  // extern "C"

// ============================================================================
// island GA
// ============================================================================

struct hg_ga {
    hg_inst* inst = nullptr;
    hg_pop* pop = nullptr;
    // per-generation duplicate grouping (the reference's memo
    // hm/engine.py:102-129): each distinct child hub set scored once
    bool dedupe = false;
    int32_t* uhubs = nullptr;  // [B][p] one representative per group
    int32_t* umap = nullptr;   // [B] group of child b
    int32_t* ucount = nullptr; // [3] slot[B-1], flag[B-1], groups
    double* uout = nullptr;    // [B][4] the groups' costs
    unsigned char* uscratch = nullptr;
    size_t uscratch_bytes = 0;
    hg_ga_params prm{};
    GaDev G{};
    int64_t B = 0;
    int32_t* inc = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int graph_kernels = 0;  // kernel launches per replay (launches captured)
    std::vector<void*> bufs;
};

namespace {

// C(n, p) saturated at 2^63
uint64_t binom_sat(int n, int p) {
    const uint64_t cap = 1ull << 63;
    uint64_t c = 1;
    for (int i = 1; i <= p; ++i) {
        // c * (n - p + i) / i stays an integer at every step
        const unsigned __int128 t = (unsigned __int128)c * (uint64_t)(n - p + i) / (uint64_t)i;
        if (t >= cap) return cap;
        c = (uint64_t)t;
    }
    return c;
}


template <class T>
int ga_alloc(hg_ga* ga, T** p, size_t count) {
    void* v = nullptr;
    HG_CUDA(cudaMalloc(&v, count * sizeof(T) + 16));
    ga->bufs.push_back(v);
    *p = static_cast<T*>(v);
    return HG_OK;
}

int ga_queue_generation(hg_ga* ga) {
    hg_inst* inst = ga->inst;
    cudaStream_t s = inst->stream;
    const GaDev& G = ga->G;
    HG_TRY(launch_build_pop(G, s));
    HG_TRY(launch_crossover(G, s));
    HG_TRY(launch_mut_scan(G, s));
    HG_TRY(launch_mutate(G, s));
    HG_TRY(launch_correct(inst->I, ga->B, G.kids, 2 * G.p, G.khubs, s));
    if (ga->dedupe) {
        // group the children's hub sets, score one per group (K2 and K3 bounded
        // by the device-side group count), copy each group's costs to its
        // members: the selection sees exactly the costs of scoring them all
        HG_TRY(launch_unique_groups(ga->pop->hubs, ga->B, G.p, ga->uscratch, ga->uscratch_bytes,
                                    ga->uhubs, ga->umap, ga->ucount, s, ga->ucount + 2));
        HG_TRY(launch_allocate(inst->I, ga->B, ga->uhubs, ga->pop->cl, co_for(inst, ga->pop->co),
                               T_for(inst, ga->B, ga->pop->T), ga->pop->legs, nullptr, s,
                               ga->ucount + 2));
        HG_TRY(queue_fitness(inst, ga->B, ga->uhubs, ga->pop->cl, ga->pop->co, ga->pop->T,
                             ga->pop->part, ga->pop->legs, ga->uout, ga->ucount + 2));
        HG_TRY(launch_scatter_out(ga->uout, ga->umap, ga->B, ga->pop->out, s));
    } else {
        HG_TRY(launch_allocate(inst->I, ga->B, ga->pop->hubs, ga->pop->cl,
                               co_for(inst, ga->pop->co), T_for(inst, ga->B, ga->pop->T),
                               ga->pop->legs, nullptr, s));
        HG_TRY(queue_fitness(inst, ga->B, ga->pop->hubs, ga->pop->cl, ga->pop->co, ga->pop->T,
                             ga->pop->part, ga->pop->legs, ga->pop->out));
    }
    HG_TRY(launch_select(G, s));
    return HG_OK;
}

// build_pop, crossover, mut_scan, mutate, correct, allocate, fitness, [finalise,] select
// (+ hash, group flags, compact, count, scatter and two CUB passes when deduplicating)
int ga_launches(const hg_ga* ga) { return ga->graph_kernels; }

void ga_release(hg_ga* ga) {
    if (ga->exec) cudaGraphExecDestroy(ga->exec);
    if (ga->graph) cudaGraphDestroy(ga->graph);
    for (void* v : ga->bufs) cudaFree(v);
    ga->bufs.clear();
    if (ga->pop) {
        pop_release(ga->pop);
        delete ga->pop;
    }
}

}  // namespace

extern "C" {

int hg_ga_create(hg_inst* inst, const hg_ga_params* prm, hg_ga** out) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst && prm && out, "NULL argument");
    *out = nullptr;
    const DevInst& I = inst->I;
    HG_ARG(prm->islands_total >= 1, "islands must be >= 1, got %d", prm->islands_total);
    HG_ARG(prm->island_lo >= 0 && prm->island_lo < prm->island_hi &&
               prm->island_hi <= prm->islands_total,
           "island range [%d, %d) invalid for %d islands", prm->island_lo, prm->island_hi,
           prm->islands_total);
    HG_ARG(prm->pop_size >= 2 && prm->pop_size % 2 == 0,
           "pop_size must be even for pairwise crossover, got %d", prm->pop_size);
    HG_ARG(prm->strength >= 1 && prm->strength <= I.p, "perturb_strength %d exceeds p=%d",
           prm->strength, I.p);
    HG_ARG(prm->rng == HG_RNG_REPLAY || prm->rng == HG_RNG_PHILOX, "unknown rng mode %d",
           prm->rng);
    HG_TRY(set_device(inst->device));
    hg_ga* ga = new (std::nothrow) hg_ga();
    if (!ga) {
        set_error("out of host memory");
        return HG_ECUDA;
    }
    ga->inst = inst;
    ga->prm = *prm;
    const int nloc = prm->island_hi - prm->island_lo;
    ga->B = (int64_t)nloc * prm->pop_size;
    int rc = HG_OK;
    do {
        ga->pop = new (std::nothrow) hg_pop();
        if (!ga->pop) {
            set_error("out of host memory");
            rc = HG_ECUDA;
            break;
        }
        if ((rc = pop_alloc(ga->pop, inst, ga->B))) break;
        GaDev& G = ga->G;
        G.n = I.n;
        G.p = I.p;
        G.nw = I.nw;
        G.nloc = nloc;
        G.pop = prm->pop_size;
        G.strength = prm->strength;
        G.strict_mode = prm->strict_paper ? 1 : 0;
        G.rng = prm->rng == HG_RNG_PHILOX ? HG_RNG_PHILOX : HG_RNG_REPLAY;
        G.island_lo = prm->island_lo;
        const size_t B = (size_t)ga->B, nw = (size_t)I.nw, p = (size_t)I.p;
        if ((rc = ga_alloc(ga, &G.anc, nloc * nw))) break;
        if ((rc = ga_alloc(ga, &G.popbits, B * nw))) break;
        if ((rc = ga_alloc(ga, &G.kids, B * nw))) break;
        if ((rc = ga_alloc(ga, &G.kcount, B))) break;
        if ((rc = ga_alloc(ga, &G.moff, B))) break;
        if ((rc = ga_alloc(ga, &G.nondeg, (size_t)nloc))) break;
        if ((rc = ga_alloc(ga, &G.champ_raw, (size_t)nloc))) break;
        if ((rc = ga_alloc(ga, &G.champ_hubs, nloc * p))) break;
        if ((rc = ga_alloc(ga, &G.best_raw, (size_t)nloc))) break;
        if ((rc = ga_alloc(ga, &G.best_hubs, nloc * p))) break;
        if ((rc = ga_alloc(ga, &G.st, (size_t)nloc * 3))) break;
        if ((rc = ga_alloc(ga, &G.ctr, (size_t)nloc * 3))) break;
        if ((rc = ga_alloc(ga, &ga->inc, p))) break;
        // per-generation duplicate grouping: off unless HUBGPU_GA_DEDUPE=1.
        // Measured (tools/ga_dedupe_probe.py, profiles/ga_dedupe_r2.json): the
        // grouping (hash, CUB sort, scan, compact, scatter) costs more than
        // scoring the duplicates at every BASELINE shape, CAB's 4x duplication
        // included -- the memo pays on the CPU, not here.  Tensor kernel only
        // (it takes the device-side group count as its batch bound).
        {
            const int fk = fitness_kernel(inst);
            ga->dedupe = (fk == HG_FIT_TC_PAIR || fk == HG_FIT_TC_PAIR_FULL) &&
                         env_int("HUBGPU_GA_DEDUPE", 0) > 0;
        }
        if (ga->dedupe) {
            ga->uscratch_bytes = unique_scratch_bytes(ga->B);
            if ((rc = ga_alloc(ga, &ga->uscratch, ga->uscratch_bytes))) break;
            if ((rc = ga_alloc(ga, &ga->uhubs, B * p))) break;
            if ((rc = ga_alloc(ga, &ga->umap, B))) break;
            if ((rc = ga_alloc(ga, &ga->ucount, 3))) break;
            if ((rc = ga_alloc(ga, &ga->uout, B * 4))) break;
        }
        G.khubs = ga->pop->hubs;
        G.kraw = ga->pop->out;
        G.inc = ga->inc;
        // streams derive_stream(seed, island, role) keyed by the GLOBAL island
        std::vector<uint64_t> st((size_t)nloc * 3), zero((size_t)nloc * 3, 0);
        for (int li = 0; li < nloc; ++li)
            for (int role = 0; role < 3; ++role) {
                uint64_t keys[2] = {(uint64_t)(prm->island_lo + li), (uint64_t)role};
                st[(size_t)li * 3 + role] = host_stream_key(prm->seed, keys, 2);
            }
        cudaStream_t s = inst->stream;
        if (cudaMemcpyAsync(G.st, st.data(), st.size() * 8, cudaMemcpyHostToDevice, s) ||
            cudaMemcpyAsync(G.ctr, zero.data(), zero.size() * 8, cudaMemcpyHostToDevice, s) ||
            cudaStreamSynchronize(s)) {
            set_error("GA state upload failed");
            rc = HG_ECUDA;
            break;
        }
        // capture one generation as a CUDA graph
        if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            set_error("cudaStreamBeginCapture failed");
            rc = HG_ECUDA;
            break;
        }
        const uint64_t l0 = launch_count();
        int qrc = ga_queue_generation(ga);
        cudaError_t ce = cudaStreamEndCapture(s, &ga->graph);
        // captured launches run on replay: count them there, not here
        ga->graph_kernels = (int)(launch_count() - l0);
        note_launch((uint64_t)0 - (uint64_t)ga->graph_kernels);
        if (qrc) {
            rc = qrc;
            break;
        }
        if (ce != cudaSuccess) {
            set_error("cudaStreamEndCapture: %s", cudaGetErrorString(ce));
            rc = HG_ECUDA;
            break;
        }
        ce = cudaGraphInstantiate(&ga->exec, ga->graph, 0);
        if (ce != cudaSuccess) {
            set_error("cudaGraphInstantiate: %s", cudaGetErrorString(ce));
            rc = HG_ECUDA;
            break;
        }
    } while (0);
    if (rc) {
        ga_release(ga);
        delete ga;
        return rc;
    }
    inst->refs.fetch_add(1);
    *out = ga;
    return HG_OK;
}

void hg_ga_free(hg_ga* ga) {
    if (!ga) return;
    hg_inst* inst = ga->inst;
    {
        auto lk_ = lock_of(inst);
        cudaSetDevice(inst->device);
        cudaStreamSynchronize(inst->stream);
        ga_release(ga);
        delete ga;
    }
    inst_release(inst);
}

int hg_ga_reseed(hg_ga* ga, uint64_t seed) {
    auto lk_ = lock_of(ga ? ga->inst : nullptr);
    HG_ARG(ga != nullptr, "GA is NULL");
    hg_inst* inst = ga->inst;
    HG_TRY(set_device(inst->device));
    const int nloc = ga->prm.island_hi - ga->prm.island_lo;
    std::vector<uint64_t> st((size_t)nloc * 3), zero((size_t)nloc * 3, 0);
    for (int li = 0; li < nloc; ++li)
        for (int role = 0; role < 3; ++role) {
            uint64_t keys[2] = {(uint64_t)(ga->prm.island_lo + li), (uint64_t)role};
            st[(size_t)li * 3 + role] = host_stream_key(seed, keys, 2);
        }
    cudaStream_t s = inst->stream;
    HG_CUDA(cudaMemcpyAsync(ga->G.st, st.data(), st.size() * 8, cudaMemcpyHostToDevice, s));
    HG_CUDA(cudaMemcpyAsync(ga->G.ctr, zero.data(), zero.size() * 8, cudaMemcpyHostToDevice, s));
    HG_CUDA(cudaStreamSynchronize(s));
    ga->prm.seed = seed;
    return HG_OK;
}

int hg_ga_begin_round(hg_ga* ga, const int64_t* ancestor_hubs) {
    auto lk_ = lock_of(ga ? ga->inst : nullptr);
    HG_ARG(ga && ancestor_hubs, "NULL argument");
    HG_TRY(set_device(ga->inst->device));
    const int p = ga->inst->I.p, n = ga->inst->I.n;
    std::vector<int32_t> h(p);
    for (int k = 0; k < p; ++k) {
        HG_ARG(ancestor_hubs[k] >= 0 && ancestor_hubs[k] < n, "ancestor hub out of range");
        HG_ARG(k == 0 || ancestor_hubs[k] > ancestor_hubs[k - 1], "ancestor hubs must be sorted");
        h[k] = (int32_t)ancestor_hubs[k];
    }
    HG_CUDA(cudaMemcpyAsync(ga->inc, h.data(), p * 4, cudaMemcpyHostToDevice, ga->inst->stream));
    HG_TRY(launch_round_begin(ga->G, ga->inst->stream));
    // the pageable H2D above is staged before return, h may go out of scope
    HG_CUDA(cudaStreamSynchronize(ga->inst->stream));
    return HG_OK;
}

int hg_ga_generations(hg_ga* ga, int count) {
    auto lk_ = lock_of(ga ? ga->inst : nullptr);
    HG_ARG(ga != nullptr, "NULL GA");
    HG_ARG(count >= 0, "negative generation count");
    HG_TRY(set_device(ga->inst->device));
    for (int g = 0; g < count; ++g) {
        HG_CUDA(cudaGraphLaunch(ga->exec, ga->inst->stream));
        note_launch((uint64_t)ga->graph_kernels);
    }
    return HG_OK;
}

int hg_ga_round_results(hg_ga* ga, double* raw, int64_t* hubs) {
    auto lk_ = lock_of(ga ? ga->inst : nullptr);
    HG_ARG(ga && raw && hubs, "NULL argument");
    HG_TRY(set_device(ga->inst->device));
    const GaDev& G = ga->G;
    const bool strict = ga->prm.strict_paper != 0;
    cudaStream_t s = ga->inst->stream;
    std::vector<int32_t> h((size_t)G.nloc * G.p);
    HG_CUDA(cudaMemcpyAsync(raw, strict ? G.champ_raw : G.best_raw, (size_t)G.nloc * 8,
                            cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaMemcpyAsync(h.data(), strict ? G.champ_hubs : G.best_hubs, h.size() * 4,
                            cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaStreamSynchronize(s));
    for (size_t x = 0; x < h.size(); ++x) hubs[x] = h[x];
    return HG_OK;
}

int hg_ga_last_children(hg_ga* ga, int64_t* hubs, double* raw) {
    auto lk_ = lock_of(ga ? ga->inst : nullptr);
    HG_ARG(ga && hubs && raw, "NULL argument");
    HG_TRY(set_device(ga->inst->device));
    cudaStream_t s = ga->inst->stream;
    const int p = ga->inst->I.p;
    std::vector<int32_t> h((size_t)ga->B * p);
    std::vector<double> o((size_t)ga->B * 4);
    HG_CUDA(cudaMemcpyAsync(h.data(), ga->pop->hubs, h.size() * 4, cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaMemcpyAsync(o.data(), ga->pop->out, o.size() * 8, cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaStreamSynchronize(s));
    for (size_t x = 0; x < h.size(); ++x) hubs[x] = h[x];
    for (int64_t b = 0; b < ga->B; ++b) raw[b] = o[(size_t)b * 4 + 3];
    return HG_OK;
}

int hg_ga_draw_counters(hg_ga* ga, uint64_t* counters) {
    auto lk_ = lock_of(ga ? ga->inst : nullptr);
    HG_ARG(ga && counters, "NULL argument");
    HG_TRY(set_device(ga->inst->device));
    HG_CUDA(cudaMemcpyAsync(counters, ga->G.ctr, (size_t)ga->G.nloc * 3 * 8,
                            cudaMemcpyDeviceToHost, ga->inst->stream));
    HG_CUDA(cudaStreamSynchronize(ga->inst->stream));
    return HG_OK;
}

int hg_host_alloc(size_t bytes, void** out) {
    HG_ARG(out != nullptr, "NULL argument");
    *out = nullptr;
    HG_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault));
    return HG_OK;
}

void hg_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

void hg_philox4x32_10(const uint32_t key[2], const uint32_t ctr[4], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    philox4x32_10(key[0], key[1], c);
    for (int i = 0; i < 4; ++i) out[i] = c[i];
}

int hg_ga_launches_per_generation(const hg_ga* ga) {
    return ga_launches(ga);
}

int hg_pairwise_leaves(int64_t m, uint32_t* out, int cap, int* count) {
    HG_ARG(m >= 0 && count != nullptr, "bad arguments");
    const std::vector<uint32_t> t = pw_leaf_table(m);
    *count = (int)t.size();
    for (int k = 0; k < cap && k < (int)t.size(); ++k) out[k] = t[k];
    return HG_OK;
}

// ---------------------------------------------------------------------------
// device generator, GPU restricted optimum
// ---------------------------------------------------------------------------

int hg_generate_urand(int device, int n, int p, uint64_t seed, double* dist, double* flow) {
    HG_ARG(n >= 1, "node count must be positive, got %d", n);
    HG_ARG(p >= 1 && p <= n, "hub count p=%d outside [1, %d]", p, n);
    HG_TRY(set_device(device));
    const uint64_t keys[2] = {(uint64_t)n, (uint64_t)p};
    const uint64_t s = host_stream_key(seed, keys, 2);  // derive_stream(seed, n, p)
    const size_t nn = (size_t)n * n;
    DevBuf xy, C, W;
    int rc = HG_OK;
    do {
        if ((rc = xy.ensure(2 * (size_t)n * sizeof(double)))) break;
        if (dist && (rc = C.ensure(nn * sizeof(double)))) break;
        if (flow && (rc = W.ensure(nn * sizeof(double)))) break;
        if ((rc = launch_gen_urand(s, n, xy.as<double>(), dist ? C.as<double>() : nullptr,
                                   flow ? W.as<double>() : nullptr, 0)))
            break;
        cudaError_t e = cudaSuccess;
        if (dist) e = cudaMemcpy(dist, C.ptr, nn * sizeof(double), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && flow)
            e = cudaMemcpy(flow, W.ptr, nn * sizeof(double), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            set_error("generate_urand copy-out failed: %s", cudaGetErrorString(e));
            rc = HG_ECUDA;
        }
    } while (0);
    xy.release();
    C.release();
    W.release();
    return rc;
}


int hg_restricted_optimum(hg_inst* inst, uint64_t limit, int64_t* best_hubs, double* best_raw,
                          uint64_t* count_out) {
    auto lk_ = lock_of(inst);
    HG_ARG(inst != nullptr, "instance is NULL");
    HG_ARG(best_hubs && best_raw, "NULL buffer");
    HG_TRY(set_device(inst->device));
    const DevInst& I = inst->I;
    const int n = I.n, p = I.p;
    const uint64_t count = binom_sat(n, p);
    if (count_out) *count_out = count;
    HG_ARG(count <= limit,
           "enumeration needs %llu candidates, over the limit of %llu; raise `limit` "
           "explicitly to allow it",
           (unsigned long long)count, (unsigned long long)limit);
    cudaStream_t s = inst->stream;
    // binomial table C(a, b), a <= n, b <= p
    std::vector<uint64_t> bt((size_t)(n + 1) * (p + 1), 0);
    for (int x = 0; x <= n; ++x)
        for (int y = 0; y <= p; ++y) bt[(size_t)x * (p + 1) + y] = y <= x ? binom_sat(x, y) : 0;
    const int64_t Bb = count < (uint64_t)65536 ? (int64_t)count : 65536;
    hg_pop* P;
    HG_TRY(scratch_pop(inst, Bb, &P));
    DevBuf dbt, dbest;
    int rc = HG_OK;
    do {
        if ((rc = dbt.ensure(bt.size() * sizeof(uint64_t)))) break;
        if ((rc = dbest.ensure(2 * sizeof(uint64_t)))) break;
        cudaError_t e = cudaMemcpyAsync(dbt.ptr, bt.data(), bt.size() * sizeof(uint64_t),
                                        cudaMemcpyHostToDevice, s);
        const unsigned long long none[2] = {0ull, ~0ull};  // raw (unused until set), rank
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(dbest.ptr, none, sizeof(none), cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(inst->derr, 0, sizeof(int), s);
        if (e != cudaSuccess) {
            set_error("restricted_optimum setup failed: %s", cudaGetErrorString(e));
            rc = HG_ECUDA;
            break;
        }
        double* d_raw = dbest.as<double>();
        unsigned long long* d_rank = reinterpret_cast<unsigned long long*>(d_raw + 1);
        for (uint64_t r0 = 0; r0 < count && rc == HG_OK; r0 += (uint64_t)Bb) {
            rc = launch_unrank_combos(dbt.as<uint64_t>(), n, p, r0, Bb, count, P->hubs, s);
            if (!rc) rc = pop_eval_queue(P, Bb, nullptr);
            if (!rc) rc = launch_batch_best(P->out, Bb, r0, count, d_raw, d_rank, s);
        }
        if (rc) break;
        unsigned long long hb[2];
        e = cudaMemcpyAsync(hb, dbest.ptr, sizeof(hb), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            set_error("restricted_optimum failed: %s", cudaGetErrorString(e));
            rc = HG_ECUDA;
            break;
        }
        double raw;
        std::memcpy(&raw, &hb[0], sizeof(raw));
        *best_raw = raw;
        // unrank the winner on the host (same lexicographic order)
        uint64_t r = hb[1];
        int x = 0;
        for (int i = 0; i < p; ++i) {
            for (;; ++x) {
                const uint64_t c = (n - 1 - x >= 0) ? bt[(size_t)(n - 1 - x) * (p + 1) + (p - 1 - i)] : 0;
                if (r < c) break;
                r -= c;
            }
            best_hubs[i] = x++;
        }
    } while (0);
    dbt.release();
    dbest.release();
    return rc;
}

}  // extern "C"
