// Device-wide exclusive scan (u64) over a functor-produced sequence, plus
// small block/warp reduction helpers.  Reduce-then-scan in three launches:
// per-block sums -> one-CTA scan of the block sums -> per-block rescan.
#pragma once

#include "common.cuh"

namespace argcsr_gpu {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr uint64_t kScanTile = uint64_t(kScanThreads) * kScanItems;

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}
__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += w;
    }
    return v;
}

// Exclusive block scan of one value per thread; returns the exclusive prefix
// and writes the block total to *total (all threads).  blockDim.x % 32 == 0.
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* total) {
    __shared__ uint64_t warp_tot[32];
    __shared__ uint64_t s_total;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const uint64_t incl = warp_incl_scan_u64(v, lane);
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const uint64_t t = lane < nw ? warp_tot[lane] : 0;
        const uint64_t ti = warp_incl_scan_u64(t, lane);
        if (lane < nw) warp_tot[lane] = ti - t;
        if (lane == 31) s_total = ti;  // nw <= 32: lane 31 holds the grand total
    }
    __syncthreads();
    const uint64_t r = warp_tot[wid] + incl - v;
    *total = s_total;
    __syncthreads();
    return r;
}

__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v) {
    uint64_t tot;
    block_excl_scan_u64(v, &tot);
    return tot;
}

template <class F>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(F f, uint64_t n, uint64_t* partial) {
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile;
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const uint64_t idx = base + uint64_t(i) * kScanThreads + threadIdx.x;
        if (idx < n) s += f(idx);
    }
    s = block_sum_u64(s);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// One CTA: exclusive scan of partial[0..nb) in place; grand total to *total.
__global__ void __launch_bounds__(1024) scan_partials_kernel(uint64_t* partial, uint64_t nb, uint64_t* total);

template <class F>
__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(F f, uint64_t n, const uint64_t* partial,
                                                                  uint64_t* out) {
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile + uint64_t(threadIdx.x) * kScanItems;
    uint64_t v[kScanItems];
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = (base + i < n) ? f(base + i) : 0;
        s += v[i];
    }
    uint64_t tot;
    uint64_t run = block_excl_scan_u64(s, &tot) + partial[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
}

// out[0..n) = exclusive prefix sums of f(0..n); out[n] = total.  Stream-ordered.
template <class F>
void exclusive_scan(F f, uint64_t n, uint64_t* out, cudaStream_t s) {
    const uint64_t nb = n == 0 ? 1 : (n + kScanTile - 1) / kScanTile;
    uint64_t* partial = nullptr;
    CUDA_OK(cudaMallocAsync(&partial, nb * sizeof(uint64_t), s));
    if (n > 0) {
        scan_reduce_kernel<<<unsigned(nb), kScanThreads, 0, s>>>(f, n, partial);
        LAUNCH_OK("scan_reduce_kernel");
    } else {
        CUDA_OK(cudaMemsetAsync(partial, 0, sizeof(uint64_t), s));
    }
    scan_partials_kernel<<<1, 1024, 0, s>>>(partial, nb, out + n);
    LAUNCH_OK("scan_partials_kernel");
    if (n > 0) {
        scan_apply_kernel<<<unsigned(nb), kScanThreads, 0, s>>>(f, n, partial, out);
        LAUNCH_OK("scan_apply_kernel");
    }
    CUDA_OK(cudaFreeAsync(partial, s));
}

}  // namespace argcsr_gpu
