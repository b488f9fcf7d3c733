// Duplicate-aware evaluation (the reference memoises scores
// by hub set, hm/engine.py:102-129): hub sets are hashed, sorted by hash,
// grouped (equal hash AND equal hubs as the sorted predecessor), compacted to
// one representative per group, scored once, and the scores scattered back.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "hg_internal.cuh"

namespace hg {

namespace {

__global__ void k_hash_sets(const int32_t* __restrict__ hubs, int64_t B, int p,
                            uint64_t* __restrict__ keys, int32_t* __restrict__ idx) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = 0x243F6A8885A308D3ull;
        for (int k = 0; k < p; ++k) h = mix64(h ^ (uint64_t)(uint32_t)hubs[b * p + k]);
        keys[b] = h;
        idx[b] = (int32_t)b;
    }
}

__device__ __forceinline__ bool same_set(const int32_t* hubs, int p, int32_t a, int32_t b) {
    for (int k = 0; k < p; ++k)
        if (hubs[(int64_t)a * p + k] != hubs[(int64_t)b * p + k]) return false;
    return true;
}

__global__ void k_group_flags(const int32_t* __restrict__ hubs, int64_t B, int p,
                              const uint64_t* __restrict__ keys, const int32_t* __restrict__ idx,
                              int32_t* __restrict__ flag) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < B;
         s += (int64_t)gridDim.x * blockDim.x)
        flag[s] = (s == 0 || keys[s] != keys[s - 1] || !same_set(hubs, p, idx[s], idx[s - 1]))
                      ? 1
                      : 0;
}

// slot = exclusive scan of the flags: a group's representative takes slot[s];
// every member maps to slot[s] + flag[s] - 1 (its group's slot)
__global__ void k_compact_sets(const int32_t* __restrict__ hubs, int64_t B, int p,
                               const int32_t* __restrict__ idx, const int32_t* __restrict__ flag,
                               const int32_t* __restrict__ slot, int32_t* __restrict__ uhubs,
                               int32_t* __restrict__ map) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < B;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = idx[s];
        const int32_t g = slot[s] + flag[s] - 1;
        map[b] = g;
        if (flag[s])
            for (int k = 0; k < p; ++k) uhubs[(int64_t)g * p + k] = hubs[(int64_t)b * p + k];
    }
}

__global__ void k_scatter_out(const double* __restrict__ uout, const int32_t* __restrict__ map,
                              int64_t B, double* __restrict__ out) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < B * 4;
         x += (int64_t)gridDim.x * blockDim.x)
        out[x] = uout[(int64_t)map[x >> 2] * 4 + (x & 3)];
}

__global__ void k_group_total(const int32_t* __restrict__ slot, const int32_t* __restrict__ flag,
                              int64_t B, int32_t* __restrict__ total) {
    *total = slot[B - 1] + flag[B - 1];
}

int grid256(int64_t count) {
    int64_t g = (count + 255) / 256;
    return (int)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

}  // namespace

size_t unique_scratch_bytes(int64_t B) {
    size_t sort_tmp = 0, scan_tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (const uint64_t*)nullptr,
                                    (uint64_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)B);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (int)B);
    const size_t tmp = sort_tmp > scan_tmp ? sort_tmp : scan_tmp;
    // keys in/out (8 B each), idx in/out, flag, slot (4 B each), then the
    // cub temporaries at a 256-byte boundary
    return (((size_t)B * 32 + 8 + 255) & ~size_t(255)) + tmp + 256;
}

int launch_unique_groups(const int32_t* hubs, int64_t B, int p, void* scratch, size_t bytes,
                         int32_t* uhubs, int32_t* map, int32_t* d_count, cudaStream_t s,
                         int32_t* d_total) {
    HG_ARG(B < (1ll << 31), "batch too large for duplicate grouping");
    unsigned char* w = static_cast<unsigned char*>(scratch);
    uint64_t* kin = reinterpret_cast<uint64_t*>(w);
    uint64_t* kout = kin + B;
    int32_t* iin = reinterpret_cast<int32_t*>(kout + B);
    int32_t* iout = iin + B;
    int32_t* flag = iout + B;
    int32_t* slot = flag + B;
    const size_t off = ((size_t)B * 32 + 8 + 255) & ~size_t(255);
    void* tmp = w + off;
    size_t tmp_bytes = bytes > off ? bytes - off : 0;
    k_hash_sets<<<grid256(B), 256, 0, s>>>(hubs, B, p, kin, iin);
    HG_LAUNCHED();
    HG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, iin, iout, (int)B, 0, 64,
                                            s));
    k_group_flags<<<grid256(B), 256, 0, s>>>(hubs, B, p, kout, iout, flag);
    HG_LAUNCHED();
    HG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, slot, (int)B, s));
    k_compact_sets<<<grid256(B), 256, 0, s>>>(hubs, B, p, iout, flag, slot, uhubs, map);
    HG_LAUNCHED();
    // group count = slot[B-1] + flag[B-1]
    HG_CUDA(cudaMemcpyAsync(d_count, slot + B - 1, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    HG_CUDA(cudaMemcpyAsync(d_count + 1, flag + B - 1, sizeof(int32_t), cudaMemcpyDeviceToDevice,
                            s));
    if (d_total) {
        k_group_total<<<1, 1, 0, s>>>(slot, flag, B, d_total);
        HG_LAUNCHED();
    }
    return HG_OK;
}

int launch_scatter_out(const double* uout, const int32_t* map, int64_t B, double* out,
                       cudaStream_t s) {
    k_scatter_out<<<grid256(B * 4), 256, 0, s>>>(uout, map, B, out);
    HG_LAUNCHED();
    return HG_OK;
}

}  // namespace hg
