// Device-side accessors of the ARG-CSR handle:
//   export_arrays  the reference layout, widened (argcsr.hpp:23-30, 52-63)
//   to_csr         csr_from_argcsr (argcsr.cpp:157-183), lossless inverse
//   padding_stats  padding_stats(const ArgCsrMatrix&) (analysis.cpp:167-184)
#include <vector>

#include "common.cuh"
#include "inverse.cuh"
#include "scan.cuh"

namespace argcsr_gpu {

namespace {

unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 64u) {
    const uint64_t b = (n + block - 1) / block;
    return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(b, cap)));
}

// GroupInfo{first_row, size, offset, chunk_size} with the reference offsets.
__global__ void k_export_groups(const GroupDesc* __restrict__ desc, const uint64_t* __restrict__ ref_off, uint64_t G,
                                uint64_t* __restrict__ out4) {
    for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < G;
         g += uint64_t(gridDim.x) * blockDim.x) {
        const GroupDesc d = desc[g];
        out4[4 * g + 0] = d.first_row;
        out4[4 * g + 1] = desc[g + 1].first_row - d.first_row;
        out4[4 * g + 2] = ref_off[g];
        out4[4 * g + 3] = d.chunk;
    }
}

// Reference-layout block of groups [g0, g1): slot (j, lane) of group g is the
// stored slot for lane < stride, else padding (+0.0, -1) (argcsr.cpp:99-104).
// Output index = ref_off[g] - ref_off[g0] + j * tpg + lane.  One CTA per group.
template <typename T>
__global__ void k_expand(const GroupDesc* __restrict__ desc, const uint64_t* __restrict__ ref_off, uint64_t g0,
                         uint64_t g1, uint64_t tpg, const T* __restrict__ vin, const int32_t* __restrict__ cin,
                         const uint32_t* __restrict__ perm, T* __restrict__ vout, int32_t* __restrict__ cout) {
    const uint64_t base = ref_off[g0];
    for (uint64_t g = g0 + blockIdx.x; g < g1; g += gridDim.x) {
        const GroupDesc d = desc[g];
        const uint64_t w = d.stride(), src = d.offset(), dst = ref_off[g] - base;
        const uint64_t n = uint64_t(d.chunk) * tpg;
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t j = i / tpg, lane = i - j * tpg;
            if (lane < w) {
                vout[dst + i] = vin[src + j * w + lane];
                const int32_t c = cin[src + j * w + lane];
                cout[dst + i] = (perm && c != -1) ? int32_t(perm[c]) : c;
            } else {
                vout[dst + i] = T(0);
                cout[dst + i] = -1;
            }
        }
    }
}

template <typename TM>
__global__ void k_widen(const TM* __restrict__ in, uint64_t n, uint64_t* __restrict__ out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = in[i];
}

// Leading non-sentinel entries of lane `lane` of a group block.
__device__ __forceinline__ uint64_t lane_len(const int32_t* cols, uint64_t off, uint64_t stride, uint32_t chunk,
                                             uint64_t lane) {
    uint64_t n = 0;
    if (lane >= stride) return 0;
    for (uint32_t j = 0; j < chunk; ++j) {
        if (cols[off + uint64_t(j) * stride + lane] == -1) break;
        ++n;
    }
    return n;
}

// Warp per group, lanes over its rows: per-row stored-element counts.
template <typename TM>
__global__ void k_row_counts(const GroupDesc* __restrict__ desc, const TM* __restrict__ tm,
                             const int32_t* __restrict__ cols, uint64_t G, uint64_t* __restrict__ cnt) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t g = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < G; g += nw) {
        const GroupDesc d = desc[g];
        const uint32_t f = d.first_row, k = desc[g + 1].first_row - f;
        for (uint32_t r = lane; r < k; r += 32) {
            const uint64_t b = r ? uint64_t(tm[f + r - 1]) : 0, e = tm[f + r];
            uint64_t n = 0;
            for (uint64_t c = b; c < e; ++c) n += lane_len(cols, d.offset(), d.stride(), d.chunk, c);
            cnt[f + r] = n;
        }
    }
}

template <typename T, typename TM>
__global__ void k_fill_csr(const GroupDesc* __restrict__ desc, const TM* __restrict__ tm,
                           const int32_t* __restrict__ cols, const T* __restrict__ vals, uint64_t G,
                           const uint64_t* __restrict__ rp, const uint32_t* __restrict__ perm,
                           int32_t* __restrict__ out_cols, T* __restrict__ out_vals) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t g = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < G; g += nw) {
        const GroupDesc d = desc[g];
        const uint32_t f = d.first_row, k = desc[g + 1].first_row - f;
        for (uint32_t r = lane; r < k; r += 32) {
            const uint64_t b = r ? uint64_t(tm[f + r - 1]) : 0, e = tm[f + r];
            uint64_t o = rp[f + r];
            for (uint64_t c = b; c < e; ++c)
                for (uint32_t j = 0; j < d.chunk; ++j) {
                    const uint64_t slot = d.offset() + uint64_t(j) * d.stride() + c;
                    const int32_t col = cols[slot];
                    if (col == -1) break;
                    out_cols[o] = perm ? int32_t(perm[col]) : col;
                    out_vals[o] = vals[slot];
                    ++o;
                }
        }
    }
}

__global__ void k_count_explicit(const int32_t* __restrict__ cols, uint64_t n, unsigned long long* __restrict__ out) {
    uint64_t c = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        c += cols[i] != -1;
    c = warp_sum_u64(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// Explicit entries of each group's stored block (one warp per group).
__global__ void k_group_nnz(const GroupDesc* __restrict__ desc, const int32_t* __restrict__ cols, uint64_t G,
                            uint64_t* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t g = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < G;
         g += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const GroupDesc d = desc[g];
        const uint64_t n = uint64_t(d.chunk) * d.stride(), base = d.offset();
        uint64_t c = 0;
        for (uint64_t i = lane; i < n; i += 32) c += cols[base + i] != -1;
        c = warp_sum_u64(c);
        if (lane == 0) out[g] = c;
    }
}

template <typename TM>
__global__ void k_assigned_slots(const GroupDesc* __restrict__ desc, const TM* __restrict__ assigned, uint64_t G,
                                 unsigned long long* __restrict__ out) {
    uint64_t c = 0;
    for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < G; g += uint64_t(gridDim.x) * blockDim.x)
        c += uint64_t(assigned[g]) * desc[g].chunk;
    c = warp_sum_u64(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

struct FromArray {
    const uint64_t* a;
    __device__ uint64_t operator()(uint64_t i) const { return a[i]; }
};

struct RefSlotsOf {  // chunk_size * threads_per_group (argcsr.cpp:151-152)
    const GroupDesc* desc;
    uint64_t tpg;
    __device__ uint64_t operator()(uint64_t g) const { return uint64_t(desc[g].chunk) * tpg; }
};

template <typename P>
struct Scratch {
    P* p = nullptr;
    cudaStream_t s;
    Scratch(size_t n, cudaStream_t st) : s(st) { CUDA_OK(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(P), s)); }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

size_t elem_size(const argcsr_dev* m) { return m->dtype == ARGCSR_F64 ? sizeof(double) : sizeof(float); }

template <typename T>
void expand_to_host(const argcsr_dev* m, const uint64_t* ref_off_dev, T* values, int32_t* columns, cudaStream_t s) {
    // Batches of whole groups, <= kBatch reference slots each (bounded scratch).
    constexpr uint64_t kBatch = uint64_t(1) << 27;
    const uint64_t G = m->num_groups;
    std::vector<uint64_t> off(G + 1);
    CUDA_OK(cudaMemcpyAsync(off.data(), ref_off_dev, (G + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    uint64_t g0 = 0;
    while (g0 < G) {
        uint64_t g1 = g0 + 1;
        while (g1 < G && off[g1 + 1] - off[g0] <= kBatch) ++g1;
        const uint64_t n = off[g1] - off[g0];
        if (n) {
            Scratch<T> v(n, s);
            Scratch<int32_t> c(n, s);
            k_expand<T><<<grid_for((g1 - g0) * 256, 256), 256, 0, s>>>(m->groups, ref_off_dev, g0, g1, m->tpg,
                                                                        static_cast<const T*>(m->values), m->columns,
                                                                        m->x_remap ? m->perm : nullptr, v.p, c.p);
            LAUNCH_OK("k_expand");
            if (values) CUDA_OK(cudaMemcpyAsync(values + off[g0], v.p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
            if (columns)
                CUDA_OK(cudaMemcpyAsync(columns + off[g0], c.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaStreamSynchronize(s));
        }
        g0 = g1;
    }
}

}  // namespace

void export_arrays(const argcsr_dev* m, uint64_t* groups4, uint64_t* tm, void* values, int32_t* columns,
                   cudaStream_t s) {
    const uint64_t G = m->num_groups, N = m->num_rows, S = m->total_slots;
    Scratch<uint64_t> ref_off(G + 1, s);
    if (G) exclusive_scan(RefSlotsOf{m->groups, m->tpg}, G, ref_off.p, s);
    if (groups4 && G) {
        Scratch<uint64_t> tmp(4 * G, s);
        k_export_groups<<<grid_for(G, 256), 256, 0, s>>>(m->groups, ref_off.p, G, tmp.p);
        LAUNCH_OK("k_export_groups");
        CUDA_OK(cudaMemcpyAsync(groups4, tmp.p, 4 * G * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
    }
    if (tm && N) {
        Scratch<uint64_t> tmp(N, s);
        k_widen<uint16_t><<<grid_for(N, 256), 256, 0, s>>>(static_cast<const uint16_t*>(m->tm), N, tmp.p);
        LAUNCH_OK("k_widen");
        CUDA_OK(cudaMemcpyAsync(tm, tmp.p, N * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
    }
    if (m->layout == kLayoutReference) {
        if (values && S) CUDA_OK(cudaMemcpyAsync(values, m->values, S * elem_size(m), cudaMemcpyDeviceToHost, s));
        if (columns && S) CUDA_OK(cudaMemcpyAsync(columns, m->columns, S * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    } else if ((values || columns) && S) {
        if (m->dtype == ARGCSR_F64) expand_to_host(m, ref_off.p, static_cast<double*>(values), columns, s);
        else expand_to_host(m, ref_off.p, static_cast<float*>(values), columns, s);
    }
    CUDA_OK(cudaStreamSynchronize(s));
}

void to_csr(const argcsr_dev* m, uint64_t* row_pointers, int32_t* columns, void* values, cudaStream_t s) {
    const uint64_t G = m->num_groups, N = m->num_rows;
    const auto* tm = static_cast<const uint16_t*>(m->tm);
    Scratch<uint64_t> cnt(N, s), rp(N + 1, s);
    k_row_counts<uint16_t><<<grid_for(G * 32, 256), 256, 0, s>>>(m->groups, tm, m->columns, G, cnt.p);
    LAUNCH_OK("k_row_counts");
    exclusive_scan(FromArray{cnt.p}, N, rp.p, s);
    uint64_t nnz = 0;
    CUDA_OK(cudaMemcpyAsync(&nnz, rp.p + N, sizeof nnz, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    Scratch<int32_t> oc(nnz, s);
    Scratch<unsigned char> ov(nnz * elem_size(m), s);
    if (m->dtype == ARGCSR_F64)
        k_fill_csr<double, uint16_t><<<grid_for(G * 32, 256), 256, 0, s>>>(
            m->groups, tm, m->columns, static_cast<const double*>(m->values), G, rp.p,
            m->x_remap ? m->perm : nullptr, oc.p,
            reinterpret_cast<double*>(ov.p));
    else
        k_fill_csr<float, uint16_t><<<grid_for(G * 32, 256), 256, 0, s>>>(
            m->groups, tm, m->columns, static_cast<const float*>(m->values), G, rp.p,
            m->x_remap ? m->perm : nullptr, oc.p,
            reinterpret_cast<float*>(ov.p));
    LAUNCH_OK("k_fill_csr");
    CUDA_OK(cudaMemcpyAsync(row_pointers, rp.p, (N + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    if (nnz) {
        CUDA_OK(cudaMemcpyAsync(columns, oc.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaMemcpyAsync(values, ov.p, nnz * elem_size(m), cudaMemcpyDeviceToHost, s));
    }
    CUDA_OK(cudaStreamSynchronize(s));
}

uint64_t to_csr_nnz(const argcsr_dev* m, cudaStream_t s) {
    const uint64_t G = m->num_groups, N = m->num_rows;
    Scratch<uint64_t> cnt(N, s), rp(N + 1, s);
    k_row_counts<uint16_t><<<grid_for(G * 32, 256), 256, 0, s>>>(m->groups, static_cast<const uint16_t*>(m->tm),
                                                                 m->columns, G, cnt.p);
    LAUNCH_OK("k_row_counts");
    exclusive_scan(FromArray{cnt.p}, N, rp.p, s);
    uint64_t nnz = 0;
    CUDA_OK(cudaMemcpyAsync(&nnz, rp.p + N, sizeof nnz, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    return nnz;
}

void balance_stats(const argcsr_dev* m, uint64_t* per_group, double* max_over_mean, double* cv, cudaStream_t s) {
    const uint64_t G = m->num_groups;
    std::vector<uint64_t> n(G);
    if (G) {
        Scratch<uint64_t> cnt(G, s);
        k_group_nnz<<<grid_for(G * 32, 256), 256, 0, s>>>(m->groups, m->columns, G, cnt.p);
        LAUNCH_OK("k_group_nnz");
        CUDA_OK(cudaMemcpyAsync(n.data(), cnt.p, G * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
    }
    if (per_group) std::copy(n.begin(), n.end(), per_group);
    // balance_of (analysis.cpp:29-55), in its order: mean of the counts, max /
    // mean, population variance summed in group order, sqrt(var) / mean; an
    // empty matrix or an all-zero one gives (1, 0).
    double mom = 1.0, c = 0.0;
    if (G) {
        uint64_t total = 0, mx = 0;
        for (uint64_t v : n) total += v, mx = std::max(mx, v);
        const double mean = double(total) / double(G);
        if (mean != 0.0) {
            mom = double(mx) / mean;
            double var = 0.0;
            for (uint64_t v : n) {
                const double d = double(v) - mean;
                var += d * d;
            }
            var /= double(G);
            c = std::sqrt(var) / mean;
        }
    }
    if (max_over_mean) *max_over_mean = mom;
    if (cv) *cv = c;
}

void padding_stats(const argcsr_dev* m, argcsr_format_stats* out, cudaStream_t s) {
    Scratch<unsigned long long> acc(2, s);
    CUDA_OK(cudaMemsetAsync(acc.p, 0, 2 * sizeof(unsigned long long), s));
    if (m->stored_slots) {
        k_count_explicit<<<grid_for(m->stored_slots, 256), 256, 0, s>>>(m->columns, m->stored_slots, acc.p);
        LAUNCH_OK("k_count_explicit");
    }
    if (m->num_groups) {
        k_assigned_slots<uint16_t><<<grid_for(m->num_groups, 256), 256, 0, s>>>(
            m->groups, static_cast<const uint16_t*>(m->assigned), m->num_groups, acc.p + 1);
        LAUNCH_OK("k_assigned_slots");
    }
    unsigned long long h[2] = {0, 0};
    CUDA_OK(cudaMemcpyAsync(h, acc.p, sizeof h, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    out->explicit_nnz = h[0];
    out->total_allocated_slots = m->total_slots;
    out->assigned_padded_slots = h[1] - h[0];
    // ratio_of (analysis.cpp:14-19)
    if (h[0] > 0) out->padding_ratio = double(m->total_slots) / double(h[0]);
    else out->padding_ratio = m->total_slots == 0 ? 1.0 : __builtin_inf();
    // kElementBytes = 8, kIndexBytes = 4 (analysis.cpp:11-12, 180-182)
    out->estimated_bytes = m->total_slots * (8 + 4) + m->num_groups * 4 * 4 + m->num_rows * 4;
}

}  // namespace argcsr_gpu
