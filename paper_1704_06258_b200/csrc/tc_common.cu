// Tensor-map and timing helpers of the tensor-core fitness kernel (K3-TC/P).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <cstdlib>

#include "hg_internal.cuh"

namespace hg {

// HUBGPU_TC_TIMING=1: per-phase cycle counters of K3-TC (tuning only)
unsigned long long* tc_timing_buffer() {
    static int on = -1;
    static unsigned long long* buf = nullptr;
    if (on < 0) {
        const char* e = getenv("HUBGPU_TC_TIMING");
        on = (e && e[0] == '1') ? 1 : 0;
        // 32 counters, 32 spare, then the K3 event trace (3 roles x 8192)
        const size_t words = 64 + 3 * 8192;
        if (on && cudaMalloc(&buf, words * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(buf, 0, words * sizeof(unsigned long long));
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

// the K3 event trace (timing build): 3 x 8192 words, cleared after the read
int tc_trace_read(unsigned long long* out) {
    unsigned long long* b = tc_timing_buffer();
    if (!b) return HG_EARG;
    HG_CUDA(cudaMemcpy(out, b + 64, 3 * 8192 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    HG_CUDA(cudaMemset(b + 64, 0, 3 * 8192 * sizeof(unsigned long long)));
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

}  // namespace hg

namespace hg {

int env_int(const char* name, int dflt) {
    static std::mutex mu;
    static std::unordered_map<std::string, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(name);
    if (it != cache.end()) return it->second;
    const char* e = getenv(name);
    int v = dflt;
    if (e) {
        char* end = nullptr;
        const long x = strtol(e, &end, 10);
        v = end != e ? (int)x : 1;
    }
    cache.emplace(name, v);
    return v;
}

static std::atomic<uint64_t> g_launches{0};

void note_launch(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

int set_max_dynamic_smem(const void* fn) {
    int dev = 0, optin = 0;
    HG_CUDA(cudaGetDevice(&dev));
    HG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    HG_CUDA(cudaFuncGetAttributes(&fa, fn));
    HG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - (int)fa.sharedSizeBytes));
    return HG_OK;
}

}  // namespace hg
