// ELLPACK and Sliced ELLPACK on the device: the paper's comparison formats
// (reference proj/src/ellpack.cpp, proj/include/argcsr/ellpack.hpp).
//
// One representation serves both: Sliced ELLPACK with slices of `slice_size`
// rows, each a columnwise block of its own width (slot j of local row r at
// slice_offsets[s] + j * rows_in_slice + r, padding (0.0, -1) trailing);
// ELLPACK is the single-slice case (slice_size = num_rows: width = max row
// nnz, slot j of row r at j * num_rows + r, ellpack.cpp:7-24).
//
// Kernels: conversion (per-slice width by warp/block max, offsets by scan,
// one thread per row filling its slots -- writes coalesced along rows for
// each j) and the SpMV (one thread per row, j ascending, stopping at the
// first padding slot; sum = fl(sum + fl(v * x[c])) from +0.0, the reference
// order of spmv_ellpack_rows / spmv_sliced_slices, ellpack.cpp:121-176, so
// fp64 results are bit-identical).  Both are HBM-bound; ELLPACK reads
// width * num_rows slots whatever the row lengths -- the padding the paper's
// ARG-CSR removes.
#include <algorithm>

#include "common.cuh"
#include "ellpack.cuh"
#include "scan.cuh"

namespace argcsr_gpu {

namespace {

unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 64u) {
    const uint64_t b = (n + block - 1) / block;
    return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(b, cap)));
}

// width of slice s = max row nnz over its rows (warp per slice, slices of any size)
__global__ void k_slice_width(const uint64_t* __restrict__ rp, uint64_t N, uint64_t S, uint64_t nslices,
                              uint64_t* __restrict__ width) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t s = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; s < nslices; s += nw) {
        const uint64_t first = s * S, last = min(first + S, N);
        uint64_t w = 0;
        for (uint64_t r = first + lane; r < last; r += 32) w = max(w, rp[r + 1] - rp[r]);
        w = warp_max_u64(w);
        if (lane == 0) width[s] = w;
    }
}

struct SliceSlots {  // width * rows_in_slice
    const uint64_t* width;
    uint64_t N, S;
    __device__ uint64_t operator()(uint64_t s) const {
        const uint64_t first = s * S;
        return width[s] * (min(first + S, N) - first);
    }
};

template <typename T>
__global__ void k_sell_fill(const uint64_t* __restrict__ rp, const int32_t* __restrict__ cols_in,
                            const T* __restrict__ vals_in, uint64_t N, uint64_t S, const uint64_t* __restrict__ width,
                            const uint64_t* __restrict__ offset, T* __restrict__ vals, int32_t* __restrict__ cols) {
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < N; r += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t s = r / S, first = s * S, rows = min(first + S, N) - first, local = r - first;
        const uint64_t w = width[s], base = offset[s] + local, b = rp[r], n = rp[r + 1] - b;
        for (uint64_t j = 0; j < w; ++j) {
            const uint64_t slot = base + j * rows;
            if (j < n) {
                vals[slot] = vals_in[b + j];
                cols[slot] = cols_in[b + j];
            } else {
                vals[slot] = T(0);
                cols[slot] = -1;
            }
        }
    }
}

template <typename T> __device__ __forceinline__ double load_x(const T* x, int32_t c) { return double(__ldg(x + c)); }
template <typename T> __device__ __forceinline__ T to_t(double v);
template <> __device__ __forceinline__ double to_t<double>(double v) { return v; }
template <> __device__ __forceinline__ float to_t<float>(double v) { return __double2float_rn(v); }

// One thread per row; rows of a slice are consecutive threads, so each j-step
// of a warp is one coalesced segment.  fp32: exact fp64 products, one rounding.
template <typename T>
__global__ void __launch_bounds__(256) k_sell_spmv(const T* __restrict__ vals, const int32_t* __restrict__ cols,
                                                   uint64_t N, uint64_t S, const uint64_t* __restrict__ width,
                                                   const uint64_t* __restrict__ offset, const T* __restrict__ x,
                                                   T* __restrict__ y) {
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < N; r += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t s = r / S, first = s * S, rows = min(first + S, N) - first;
        const uint64_t w = width[s];
        const T* vp = vals + offset[s] + (r - first);
        const int32_t* cp = cols + offset[s] + (r - first);
        double sum = 0.0;
        uint64_t j = 0;
        for (; j + 4 <= w; j += 4) {  // 4 steps of loads in flight
            int32_t c[4];
            T v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = __ldcs(cp + (j + q) * rows), v[q] = __ldcs(vp + (j + q) * rows);
            double xv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) xv[q] = c[q] != -1 ? load_x(x, c[q]) : 0.0;
            bool stop = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (c[q] == -1) stop = true;  // padding is trailing (ellpack.cpp:127)
                if (!stop) sum = __dadd_rn(sum, __dmul_rn(double(v[q]), xv[q]));
            }
            if (stop) break;
        }
        if (j + 4 > w) {
            for (; j < w; ++j) {
                const int32_t c = cp[j * rows];
                if (c == -1) break;
                sum = __dadd_rn(sum, __dmul_rn(double(vp[j * rows]), load_x(x, c)));
            }
        }
        y[r] = to_t<T>(sum);
    }
}

template <typename P>
struct Tmp {
    P* p = nullptr;
    cudaStream_t s;
    Tmp(size_t n, cudaStream_t st) : s(st) { CUDA_OK(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(P), s)); }
    ~Tmp() {
        if (p) cudaFreeAsync(p, s);
    }
};

template <typename T>
void convert_typed(argcsr_sell* m, const uint64_t* rp, const int32_t* cols, const T* vals, cudaStream_t s) {
    const uint64_t N = m->num_rows, S = m->slice_size;
    const uint64_t ns = (N + S - 1) / S;
    m->num_slices = ns;
    CUDA_OK(cudaMalloc(&m->width, ns * sizeof(uint64_t)));
    CUDA_OK(cudaMalloc(&m->offset, (ns + 1) * sizeof(uint64_t)));
    m->device_bytes += (2 * ns + 1) * sizeof(uint64_t);
    k_slice_width<<<grid_for(ns * 32, 256), 256, 0, s>>>(rp, N, S, ns, m->width);
    LAUNCH_OK("k_slice_width");
    exclusive_scan(SliceSlots{m->width, N, S}, ns, m->offset, s);
    CUDA_OK(cudaMemcpyAsync(&m->total_slots, m->offset + ns, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    const size_t es = sizeof(T);
    size_t free_b = 0, total_b = 0;
    CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
    if (m->total_slots && m->total_slots > (free_b / (es + 4)))
        fail(ARGCSR_E_OOM, "sliced_from_csr: " + std::to_string(m->total_slots) +
                               " slots do not fit in device memory (ELLPACK pads every row of a slice to its widest)");
    CUDA_OK(cudaMalloc(&m->values, std::max<uint64_t>(m->total_slots, 1) * es));
    CUDA_OK(cudaMalloc(&m->columns, std::max<uint64_t>(m->total_slots, 1) * sizeof(int32_t)));
    m->device_bytes += m->total_slots * (es + 4);
    if (N) {
        k_sell_fill<T><<<grid_for(N, 256), 256, 0, s>>>(rp, cols, vals, N, S, m->width, m->offset,
                                                        static_cast<T*>(m->values), m->columns);
        LAUNCH_OK("k_sell_fill");
    }
    CUDA_OK(cudaStreamSynchronize(s));
}

}  // namespace

void sell_convert(argcsr_sell* m, const uint64_t* rp, const int32_t* cols, const void* vals, cudaStream_t s) {
    if (m->dtype == ARGCSR_F64) convert_typed<double>(m, rp, cols, static_cast<const double*>(vals), s);
    else convert_typed<float>(m, rp, cols, static_cast<const float*>(vals), s);
}

void sell_spmv(const argcsr_sell* m, const void* x, void* y, cudaStream_t s) {
    if (m->num_rows == 0) return;
    const unsigned grid = grid_for(m->num_rows, 256);
    if (m->dtype == ARGCSR_F64)
        k_sell_spmv<double><<<grid, 256, 0, s>>>(static_cast<const double*>(m->values), m->columns, m->num_rows,
                                                 m->slice_size, m->width, m->offset, static_cast<const double*>(x),
                                                 static_cast<double*>(y));
    else
        k_sell_spmv<float><<<grid, 256, 0, s>>>(static_cast<const float*>(m->values), m->columns, m->num_rows,
                                                m->slice_size, m->width, m->offset, static_cast<const float*>(x),
                                                static_cast<float*>(y));
    LAUNCH_OK("k_sell_spmv");
}

}  // namespace argcsr_gpu
