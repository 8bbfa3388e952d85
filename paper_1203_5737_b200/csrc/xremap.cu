// x remap: keep the SpMV's x working set L2-resident when x itself does not
// fit the persisting-L2 window (B200: ~83 MB of the 126 MB L2).
//
// The lane-compact layout stores column indices in a device-internal column
// order pi: the columns the matrix actually uses come first, by popularity
// octave (floor(log2(uses)), most-used first) and by index within an octave
// (stable, so banded/stencil locality survives); unused columns get no slot.
// Every SpMV first gathers x' = x[perm[0 .. n_used)] (one small kernel), then
// runs on x', whose hot head is what the access-policy window covers.  The
// arithmetic is unchanged: each product is v * x[c] with the same x value, so
// results stay bit-identical; export, csr_from_argcsr and chunk_entries map
// stored columns back through perm, so every reference-facing array is the
// reference's.
//
// It is applied only where it pays (auto mode): x larger than the window AND
// the window, filled popularity-first, covers >= 25 points more of the nnz
// than the window over the leading columns.  A row slice of a stencil on one
// of P GPUs qualifies (it touches ~1/P of x, often none of the leading
// columns); R-MAT 2^24 does not (leading 90% vs 100%: measured, the x' gather
// costs more than the misses it saves); stencils on one GPU do
// not.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "scan.cuh"
#include "xremap.cuh"

namespace argcsr_gpu {

namespace {

unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
    const uint64_t b = (n + block - 1) / block;
    return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(b, cap)));
}

__global__ void k_col_hist(const int32_t* __restrict__ cols, uint64_t n, uint64_t num_cols, bool sentinels,
                           uint32_t* __restrict__ count, unsigned int* __restrict__ bad) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const int32_t c = cols[i];
        if (sentinels && c == -1) continue;
        if (c < 0 || uint64_t(c) >= num_cols) {
            *bad = 1u;  // the converter does not validate (argcsr.cpp:107-117): no remap then
            continue;
        }
        atomicAdd(count + c, 1u);
    }
}

// key: popularity octave, most-used first; unused columns last (255).
__global__ void k_col_keys(const uint32_t* __restrict__ count, uint64_t n, uint8_t* __restrict__ key,
                           uint32_t* __restrict__ idx, unsigned long long* __restrict__ used,
                           unsigned long long* __restrict__ lead_nnz, unsigned long long* __restrict__ total,
                           uint64_t K) {
    uint64_t u = 0, lead = 0, tot = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = count[i];
        key[i] = c == 0 ? uint8_t(255) : uint8_t(__clz(c));  // __clz(c) = 31 - floor(log2 c)
        idx[i] = uint32_t(i);
        u += c != 0;
        tot += c;
        if (i < K) lead += c;
    }
    u = warp_sum_u64(u);
    lead = warp_sum_u64(lead);
    tot = warp_sum_u64(tot);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(used, (unsigned long long)u);
        atomicAdd(lead_nnz, (unsigned long long)lead);
        atomicAdd(total, (unsigned long long)tot);
    }
}

__global__ void k_top_nnz(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ count, uint64_t K,
                          unsigned long long* __restrict__ out) {
    uint64_t t = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < K; i += uint64_t(gridDim.x) * blockDim.x)
        t += count[perm[i]];
    t = warp_sum_u64(t);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)t);
}

// Consecutive-column pairs inside long rows (>= kLongRow entries; they form
// the heavy groups): in the input order and in the remapped order.  A lane of
// a heavy group holds a contiguous run of its row, so consecutive stored
// columns let the heavy kernel load x in 16/32-byte runs (spmv.cu).
constexpr uint64_t kLongRow = 256;
__global__ void k_long_row_runs(const uint64_t* __restrict__ rp, uint64_t N, const int32_t* __restrict__ cols,
                                const int32_t* __restrict__ inv, uint64_t num_cols,
                                unsigned long long* __restrict__ acc /* long nnz, pairs, orig, remapped */) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    uint64_t ln = 0, pairs = 0, orig = 0, rem = 0;
    for (uint64_t r = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < N; r += nw) {
        const uint64_t b = rp[r], e = rp[r + 1];
        if (e - b < kLongRow) continue;
        if (lane == 0) ln += e - b;
        for (uint64_t k = b + lane; k + 1 < e; k += 32) {
            const int32_t c0 = cols[k], c1 = cols[k + 1];
            if (c0 < 0 || c1 < 0 || uint64_t(c0) >= num_cols || uint64_t(c1) >= num_cols) continue;
            ++pairs;
            orig += c1 == c0 + 1;
            rem += inv[c1] == inv[c0] + 1;
        }
    }
    ln = warp_sum_u64(ln);
    pairs = warp_sum_u64(pairs);
    orig = warp_sum_u64(orig);
    rem = warp_sum_u64(rem);
    if (lane == 0) {
        atomicAdd(acc, (unsigned long long)ln);
        atomicAdd(acc + 1, (unsigned long long)pairs);
        atomicAdd(acc + 2, (unsigned long long)orig);
        atomicAdd(acc + 3, (unsigned long long)rem);
    }
}

__global__ void k_inverse(const uint32_t* __restrict__ perm, uint64_t n_used, int32_t* __restrict__ inv) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_used;
         i += uint64_t(gridDim.x) * blockDim.x)
        inv[perm[i]] = int32_t(i);
}

template <typename T>
__global__ void k_gather_x(const T* __restrict__ x, const uint32_t* __restrict__ perm, uint64_t n,
                           T* __restrict__ xr) {
    // 8 independent gathers in flight per thread (the loop is latency-bound otherwise)
    constexpr int K = 8;
    const uint64_t step = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += K * step) {
        uint32_t p[K];
        T v[K];
#pragma unroll
        for (int k = 0; k < K; ++k) p[k] = i0 + k * step < n ? __ldg(perm + i0 + k * step) : 0u;
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = i0 + k * step < n ? __ldg(x + p[k]) : T(0);
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (i0 + k * step < n) xr[i0 + k * step] = v[k];
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

}  // namespace

int32_t* build_xremap(argcsr_dev* m, const int32_t* cols, uint64_t nnz, int mode, cudaStream_t s, bool sentinels,
                      const uint64_t* rp, const int32_t* cols_abs) {
    m->x_remap = false;
    m->n_used = m->num_cols;
    if (mode == kXRemapOff || m->layout != kLayoutCompact || m->num_cols == 0 || nnz == 0) return nullptr;
    if (m->num_cols >= 0x7fffffffull) return nullptr;  // cub item count / i32 columns
    const uint64_t C = m->num_cols;
    const size_t sv = m->dtype == ARGCSR_F64 ? sizeof(double) : sizeof(float);
    const size_t win = std::min<size_t>(size_t(m->l2_window_max), m->l2_persist_max);
    const uint64_t K = win / sv;  // x elements the window holds
    const bool fits = win == 0 || C <= K;
    if (mode == kXRemapAuto && fits && !rp) return nullptr;

    Tmp<uint32_t> count(C, s);
    Tmp<unsigned int> bad(1, s);
    Tmp<unsigned long long> acc(4, s);  // used, lead nnz, top nnz, total nnz
    CUDA_OK(cudaMemsetAsync(count.p, 0, C * sizeof(uint32_t), s));
    CUDA_OK(cudaMemsetAsync(bad.p, 0, sizeof(unsigned int), s));
    CUDA_OK(cudaMemsetAsync(acc.p, 0, 4 * sizeof(unsigned long long), s));
    k_col_hist<<<grid_for(nnz, 256), 256, 0, s>>>(cols, nnz, C, sentinels, count.p, bad.p);
    LAUNCH_OK("k_col_hist");
    Tmp<uint8_t> key(C, s), key_sorted(C, s);
    Tmp<uint32_t> idx(C, s);
    uint32_t* perm = nullptr;
    CUDA_OK(cudaMalloc(&perm, C * sizeof(uint32_t)));
    struct PermGuard {
        uint32_t*& p;
        bool keep = false;
        ~PermGuard() {
            if (!keep && p) cudaFree(p), p = nullptr;
        }
    } guard{perm};
    k_col_keys<<<grid_for(C, 256), 256, 0, s>>>(count.p, C, key.p, idx.p, acc.p, acc.p + 1, acc.p + 3, K);
    LAUNCH_OK("k_col_keys");
    size_t tmp_bytes = 0;
    CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key.p, key_sorted.p, idx.p, perm, int(C), 0, 8, s));
    Tmp<unsigned char> tmp(tmp_bytes, s);
    CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, key.p, key_sorted.p, idx.p, perm, int(C), 0, 8, s));
    k_top_nnz<<<grid_for(std::min<uint64_t>(K, C), 256), 256, 0, s>>>(perm, count.p, std::min<uint64_t>(K, C),
                                                                      acc.p + 2);
    LAUNCH_OK("k_top_nnz");
    unsigned long long h[4] = {0, 0, 0, 0};
    unsigned int hbad = 0;
    CUDA_OK(cudaMemcpyAsync(h, acc.p, sizeof h, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaMemcpyAsync(&hbad, bad.p, sizeof hbad, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    if (hbad) return nullptr;
    if (h[3] == 0) return nullptr;
    const double lead = double(h[1]) / double(h[3]), top = double(h[2]) / double(h[3]);
    const uint64_t n_used = h[0];
    int32_t* inv = nullptr;
    CUDA_OK(cudaMallocAsync(&inv, C * sizeof(int32_t), s));
    struct InvGuard {
        int32_t*& p;
        cudaStream_t s;
        bool keep = false;
        ~InvGuard() {
            if (!keep && p) cudaFreeAsync(p, s), p = nullptr;
        }
    } inv_guard{inv, s};
    k_inverse<<<grid_for(n_used, 256), 256, 0, s>>>(perm, n_used, inv);
    LAUNCH_OK("k_inverse");
    bool on = mode == kXRemapOn || (!fits && top >= lead + 0.25);
    if (!on && rp) {
        // the second reason: long rows whose columns become consecutive (the
        // heavy kernel then loads 2-4 x entries per gather, measured on C4)
        Tmp<unsigned long long> runs(4, s);
        CUDA_OK(cudaMemsetAsync(runs.p, 0, 4 * sizeof(unsigned long long), s));
        k_long_row_runs<<<grid_for(m->num_rows * 32, 256), 256, 0, s>>>(rp, m->num_rows, cols_abs, inv, C, runs.p);
        LAUNCH_OK("k_long_row_runs");
        unsigned long long r[4] = {0, 0, 0, 0};
        CUDA_OK(cudaMemcpyAsync(r, runs.p, sizeof r, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        on = r[1] > 0 && double(r[0]) >= 0.2 * double(h[3]) && double(r[3]) - double(r[2]) >= 0.5 * double(r[1]);
        m->run_pairs_orig = r[1] ? double(r[2]) / double(r[1]) : 0.0;
        m->run_pairs_remap = r[1] ? double(r[3]) / double(r[1]) : 0.0;
    }
    if (!on) return nullptr;
    inv_guard.keep = true;
    guard.keep = true;
    m->perm = perm;
    m->device_bytes += C * sizeof(uint32_t);
    CUDA_OK(cudaMalloc(&m->xbuf, std::max<uint64_t>(n_used, 1) * sv));
    m->device_bytes += std::max<uint64_t>(n_used, 1) * sv;
    m->n_used = n_used;
    m->x_remap = true;
    m->x_cover_lead = lead;
    m->x_cover_top = top;
    return inv;  // the caller frees it (stream-ordered) after the layout kernel
}

const void* xremap_apply(const argcsr_dev* m, const void* x, cudaStream_t s) {
    if (!m->x_remap) return x;
    if (m->n_used) {
        if (m->dtype == ARGCSR_F64)
            k_gather_x<double><<<grid_for(m->n_used, 256, 148u * 16u), 256, 0, s>>>(
                static_cast<const double*>(x), m->perm, m->n_used, static_cast<double*>(m->xbuf));
        else
            k_gather_x<float><<<grid_for(m->n_used, 256, 148u * 16u), 256, 0, s>>>(
                static_cast<const float*>(x), m->perm, m->n_used, static_cast<float*>(m->xbuf));
        LAUNCH_OK("k_gather_x");
    }
    return m->xbuf;
}

}  // namespace argcsr_gpu
