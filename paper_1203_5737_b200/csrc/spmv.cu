// ARG-CSR SpMV for sm_100a (replaces spmv_argcsr_groups, proj/src/argcsr.cpp:185-217).
//
// One launch, two CTA roles:
//   * heavy CTAs (blockIdx < heavy_ctas): long-chunk groups in LPT order
//     (largest chunk first), packed so their assigned lanes fill the CTA, one
//     lane per thread, deep unroll so a 1-3 MB group streams at per-SM speed;
//   * light tiles: a run of consecutive short-chunk groups whose ASSIGNED lanes
//     (free lanes are never read) are flattened into V-lane units, one unit per
//     thread.  A unit's V adjacent lanes are one vector column load (16 B for
//     V=4) and one vector value load (32 B, LDG.256, for fp64 V=4) per element
//     step, so every warp access is a contiguous, coalesced segment of a
//     group's j-row.  All element steps of a unit (up to U) are issued before
//     the first x gather, so a tile has its whole matrix block in flight.
// Group metadata of a tile is staged in shared memory and threads_mapping of
// the tile's rows is prefetched into registers during phase 1; per-chunk
// partial sums go to shared memory and each row sums its chunk range in
// ascending order from +0.0.  Products and sums use __dmul_rn/__dadd_rn in the
// reference's order (phase 1: per lane, j ascending; phase 2: per row, chunks
// ascending), so fp64 results are bit-identical to the reference's CPU product
// (which has no FMA).  fp32 handles load fp32 values/x, multiply exactly in
// fp64 and round each row sum once.
//
// Cache policy: values/columns are streamed once (L1 no-allocate, L2
// evict-normal); x gathers are L2 evict-last and x is additionally covered by a
// persisting access-policy window sized from the device's persisting-L2 limit.
// Light tiles bulk-prefetch their stored block into L2 at CTA start
// (tile_prefetch_l2; which arrays, and the x policy of regular matrices whose x
// exceeds the window, are per handle: l2_prefetch_bytes / l2_prefetch_what /
// x_evict_last).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "spmv.cuh"
#include "xremap.cuh"

namespace argcsr_gpu {

namespace {

template <typename T>
struct SpmvArgs {
    const T* __restrict__ vals;
    const int32_t* __restrict__ cols;
    const GroupDesc* __restrict__ groups;
    const uint16_t* __restrict__ tm;
    const uint16_t* __restrict__ assigned;
    const uint64_t* __restrict__ unit_base;
    const uint8_t* __restrict__ ulen;  // light unit lengths (null: read up to the group's chunk)
    uint64_t total_units;
    const uint32_t* __restrict__ tiles;
    const uint64_t* __restrict__ tile_rng;  // [2 * tiles] stored slot range per light tile (0, 0: none)
    const uint32_t* __restrict__ heavy;
    const uint32_t* __restrict__ heavy_ptr;
    const T* __restrict__ x;
    T* __restrict__ y;
    uint32_t heavy_ctas;
    uint32_t norm_light0;     // first light-tile slot of norm_part (after the heavy CTAs' slots)
    uint32_t g_begin, g_end;  // rows of groups outside [g_begin, g_end) are not written
    uint32_t all_groups;      // [g_begin, g_end) covers every group
    uint32_t max_tile_groups;
    uint32_t max_tile_rows;
    uint32_t tile0;  // light tiles [tile0, tile0 + gridDim.x) of this launch (spmv_launch_tiles)
    uint32_t max_tile_units;
    const double* x_scale;   // y = A (s * x), s = *x_scale (device) or 1.0: each gather is fl(s * x[c])
    double* norm_part;       // fused ||y||^2: one partial per CTA (heavy CTAs first, then light tiles), or null
    int x_evict_last;        // x gathers: L2 evict_last (1) or evict_normal (0)
    int stream_evict_first;  // values/columns: L2 evict_first (1) or evict_normal (0)
    uint32_t l2_prefetch;    // light tiles of at most this many stored bytes bulk-prefetch them into L2 (0: off)
    char l2_prefetch_what;   // 'b' values and columns, 'c' columns only, 'v' values only (experiments)
    uint32_t npeers;         // multi-GPU epilogue: y rows in [peer_lo[q], peer_hi[q]) are also stored
    T* peer_y[kMaxPeers];    // to peer_y[q][row] (other GPUs' x buffers via NVLink peer mappings, pre-offset)
    uint32_t peer_lo[kMaxPeers], peer_hi[kMaxPeers];
};

// ------------------------------------------------------------ cache policies
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Streaming loads of V adjacent columns / values (V * sizeof bytes, aligned).
template <int V>
__device__ __forceinline__ void ld_cols(const int32_t* p, int (&c)[V], uint64_t pol) {
    if constexpr (V == 4) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]) : "l"(p), "l"(pol));
    } else if constexpr (V == 2) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
                     : "=r"(c[0]), "=r"(c[1]) : "l"(p), "l"(pol));
    } else {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(c[0]) : "l"(p), "l"(pol));
    }
}
template <int V>
__device__ __forceinline__ void ld_vals(const double* p, double (&v)[V], uint64_t pol) {
    if constexpr (V == 4) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p), "l"(pol));
    } else if constexpr (V == 2) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(v[0]), "=d"(v[1]) : "l"(p), "l"(pol));
    } else {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[0]) : "l"(p), "l"(pol));
    }
}
template <int V>
__device__ __forceinline__ void ld_vals(const float* p, float (&v)[V], uint64_t pol) {
    if constexpr (V == 4) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "l"(p), "l"(pol));
    } else if constexpr (V == 2) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                     : "=f"(v[0]), "=f"(v[1]) : "l"(p), "l"(pol));
    } else {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v[0]) : "l"(p), "l"(pol));
    }
}

__device__ __forceinline__ double ld_x(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_x(const float* p, uint64_t pol) {
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return double(v);
}

// Phase 1 (argcsr.cpp:193-203) for V adjacent lanes starting at slot0: per
// lane, sum += v * x[c] over j ascending until the first sentinel.  Columns
// and values of U element steps are issued together (values of a fully
// finished vector are skipped when PRED); the layout keeps sentinels
// trailing, so "skip sentinel" == "stop at the first sentinel".
template <typename T, int V, int U, bool PRED>
__device__ __forceinline__ void phase1(const SpmvArgs<T>& a, uint64_t slot0, uint32_t chunk, uint64_t stride,
                                       double (&s)[V], uint64_t pol_stream, uint64_t pol_x, double xs,
                                       uint32_t jstart = 0) {
    if (jstart == 0) {
#pragma unroll
        for (int l = 0; l < V; ++l) s[l] = 0.0;
    }
    const int32_t* cp = a.cols + slot0;
    const T* vp = a.vals + slot0;
    const uint64_t tpg = stride;
    for (uint32_t j0 = jstart; j0 < chunk; j0 += U) {
        int c[U][V];
        T v[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (j0 + u < chunk) {
                ld_cols<V>(cp + uint64_t(j0 + u) * tpg, c[u], pol_stream);
                if constexpr (!PRED) ld_vals<V>(vp + uint64_t(j0 + u) * tpg, v[u], pol_stream);
            } else {
#pragma unroll
                for (int l = 0; l < V; ++l) c[u][l] = -1, v[u][l] = T(0);
            }
        }
        if constexpr (PRED) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int any = -1;
#pragma unroll
                for (int l = 0; l < V; ++l) any &= c[u][l];
                if (any != -1) {
                    ld_vals<V>(vp + uint64_t(j0 + u) * tpg, v[u], pol_stream);
                } else {
#pragma unroll
                    for (int l = 0; l < V; ++l) v[u][l] = T(0);
                }
            }
        }
        double xv[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int l = 0; l < V; ++l) xv[u][l] = c[u][l] != -1 ? ld_x(a.x + c[u][l], pol_x) : 0.0;
        if (a.x_scale) {  // uniform: fused normalisation of the power iteration
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int l = 0; l < V; ++l) xv[u][l] = __dmul_rn(xv[u][l], xs);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int l = 0; l < V; ++l)
                if (c[u][l] != -1) s[l] = __dadd_rn(s[l], __dmul_rn(double(v[u][l]), xv[u][l]));
        int all = -1;
#pragma unroll
        for (int l = 0; l < V; ++l) all &= c[U - 1][l];
        if (all == -1) break;
    }
}

// Phase 1 of ONE lane (V = 1, the long-chunk path), software-pipelined: the
// columns of batch b+1 are loaded while batch b's values and x gathers are in
// flight, so a batch of U element steps costs one memory round trip instead
// of two (columns, then gathers).  Same additions in the same order.
__device__ __forceinline__ int ld_col1(const int32_t* p, uint64_t pol) {
    int c;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(c) : "l"(p), "l"(pol));
    return c;
}
template <typename T, int U>
__device__ __forceinline__ double phase1_lane_pipe(const SpmvArgs<T>& a, uint64_t slot0, uint32_t chunk,
                                                   uint64_t stride, uint64_t pol_stream, uint64_t pol_x, double xs) {
    double s = 0.0;
    const int32_t* cp = a.cols + slot0;
    const T* vp = a.vals + slot0;
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = uint32_t(u) < chunk ? ld_col1(cp + uint64_t(u) * stride, pol_stream) : -1;
    for (uint32_t j0 = 0; j0 < chunk; j0 += U) {
        T v[U][1];
        double xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (c[u] != -1) ld_vals<1>(vp + uint64_t(j0 + u) * stride, v[u], pol_stream);
            else v[u][0] = T(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) xv[u] = c[u] != -1 ? ld_x(a.x + c[u], pol_x) : 0.0;
        int cn[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            cn[u] = j0 + U + u < chunk ? ld_col1(cp + uint64_t(j0 + U + u) * stride, pol_stream) : -1;
        if (a.x_scale) {
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = __dmul_rn(xv[u], xs);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (c[u] != -1) s = __dadd_rn(s, __dmul_rn(double(v[u][0]), xv[u]));
        if (c[U - 1] == -1) break;
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = cn[u];
    }
    return s;
}

// Phase 1 for a thread's two units when every light chunk of the matrix is
// <= H: both units' element steps are issued in ONE batch (columns, values,
// then all gathers) -- the register footprint of one unit with 2H steps, half
// the round trips of walking the units one after the other.  Per lane the
// products are added in j order: bit-identical to phase1.
template <typename T, int V, int H>
__device__ __forceinline__ void phase1_pair(const SpmvArgs<T>& a, const uint64_t (&slot)[2], const uint32_t (&ch)[2],
                                            const uint32_t (&st)[2], double (&s)[2][V], uint64_t pol_stream,
                                            uint64_t pol_x, double xs) {
    int c[2][H][V];
    T v[2][H][V];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int h = 0; h < H; ++h) {
            if (uint32_t(h) < ch[k]) {
                ld_cols<V>(a.cols + slot[k] + uint64_t(h) * st[k], c[k][h], pol_stream);
                ld_vals<V>(a.vals + slot[k] + uint64_t(h) * st[k], v[k][h], pol_stream);
            } else {
#pragma unroll
                for (int l = 0; l < V; ++l) c[k][h][l] = -1, v[k][h][l] = T(0);
            }
        }
    double xv[2][H][V];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
            for (int l = 0; l < V; ++l) xv[k][h][l] = c[k][h][l] != -1 ? ld_x(a.x + c[k][h][l], pol_x) : 0.0;
    if (a.x_scale) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int h = 0; h < H; ++h)
#pragma unroll
                for (int l = 0; l < V; ++l) xv[k][h][l] = __dmul_rn(xv[k][h][l], xs);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int l = 0; l < V; ++l) {
            s[k][l] = 0.0;
#pragma unroll
            for (int h = 0; h < H; ++h)
                if (c[k][h][l] != -1) s[k][l] = __dadd_rn(s[k][l], __dmul_rn(double(v[k][h][l]), xv[k][h][l]));
        }
}

template <typename T>
__device__ __forceinline__ double x_scale_value(const SpmvArgs<T>& a) {
    return a.x_scale ? *a.x_scale : 1.0;
}

// sq += v only in the kernels that write ||y||^2 partials (NORM); elsewhere
// the squares are dead code and compiled out.
template <bool NORM>
__device__ __forceinline__ void acc_sq(double& sq, double v) {
    if constexpr (NORM) sq = __dadd_rn(sq, v);
}

// Fused ||y||^2: every thread accumulates the squares of the y values it
// stores; the CTA's sum goes to norm_part[slot] in a fixed order (a fixed
// xor-shuffle tree per warp, lane 0's result, then the warps in index order),
// so the partials -- and the fixed-order reduction over them -- are
// deterministic run to run.  Call from every thread of the CTA.
__device__ __forceinline__ void write_norm_partial(double* out, double v) {
    __shared__ double s_warp[kTileThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) t = __dadd_rn(t, s_warp[w]);
        *out = t;
    }
}

template <typename T> __device__ __forceinline__ T to_out(double v);
template <> __device__ __forceinline__ double to_out<double>(double v) { return v; }
template <> __device__ __forceinline__ float to_out<float>(double v) { return __double2float_rn(v); }

// Epilogue: y[row], and the same value into every peer's buffer (the fused
// all-gather of the multi-GPU step: the y slice lands in the other GPUs' next
// x directly from the kernel, as plain stores over the NVLink peer mapping).
// (A template flag: the single-GPU kernels carry no peer code at all.)
template <bool PEER, typename T>
__device__ __forceinline__ double store_y(const SpmvArgs<T>& a, uint32_t row, double v) {
    const T o = to_out<T>(v);
    a.y[row] = o;
    if constexpr (PEER)
        for (uint32_t q = 0; q < a.npeers; ++q)
            if (row >= a.peer_lo[q] && row < a.peer_hi[q]) a.peer_y[q][row] = o;
    return __dmul_rn(double(o), double(o));
}

// Phase 2 (argcsr.cpp:206-215): +0.0 + p_b + p_{b+1} + ... ascending.
__device__ __forceinline__ double row_sum(const double* part, uint32_t b, uint32_t e) {
    double sum = 0.0;
    for (uint32_t t = b; t < e; ++t) sum = __dadd_rn(sum, part[t]);
    return sum;
}

// last index i in [0, n) with arr[i] <= key (arr ascending, arr[0] <= key)
__device__ __forceinline__ uint32_t find_le(const uint32_t* arr, uint32_t n, uint32_t key) {
    uint32_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) / 2;
        if (arr[mid] <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Heavy groups heavy[hb..he) packed into one CTA: lanes and rows flattened in
// order, one lane per thread.
template <typename T, int UH, int MINB, bool PEER = false, bool NORM = false, bool PIPE = false>
__global__ void __launch_bounds__(kTileThreads, MINB) spmv_heavy_kernel(const SpmvArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_part = reinterpret_cast<double*>(smem);
    __shared__ uint32_t s_lane0[kTileThreads + 1], s_row0[kTileThreads + 1], s_g[kTileThreads];
    const uint64_t pol_stream = a.stream_evict_first ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_x = a.x_evict_last ? policy_evict_last() : policy_evict_normal();
    const double xs = x_scale_value(a);
    const uint32_t hb = a.heavy_ptr[blockIdx.x], he = a.heavy_ptr[blockIdx.x + 1];
    const uint32_t ng = he - hb;
    if (threadIdx.x == 0) {
        uint32_t lanes = 0, rows = 0;
        for (uint32_t i = 0; i < ng; ++i) {
            const uint32_t g = a.heavy[hb + i];
            s_g[i] = g;
            s_lane0[i] = lanes;
            s_row0[i] = rows;
            lanes += a.assigned[g];
            rows += a.groups[g + 1].first_row - a.groups[g].first_row;
        }
        s_lane0[ng] = lanes;
        s_row0[ng] = rows;
    }
    __syncthreads();
    const uint32_t nlanes = s_lane0[ng], nrows = s_row0[ng];
    for (uint32_t l = threadIdx.x; l < nlanes; l += blockDim.x) {
        const uint32_t i = find_le(s_lane0, ng, l);
        const uint32_t g = s_g[i];
        if (g < a.g_begin || g >= a.g_end) continue;
        const GroupDesc d = a.groups[g];
        if constexpr (PIPE) {
            s_part[l] = phase1_lane_pipe<T, UH>(a, d.offset() + (l - s_lane0[i]), d.chunk, d.stride(), pol_stream,
                                                pol_x, xs);
        } else {
            double s[1];
            phase1<T, 1, UH, false>(a, d.offset() + (l - s_lane0[i]), d.chunk, d.stride(), s, pol_stream, pol_x,
                                    xs);
            s_part[l] = s[0];
        }
    }
    __syncthreads();
    double sq = 0.0;
    for (uint32_t r = threadIdx.x; r < nrows; r += blockDim.x) {
        const uint32_t i = find_le(s_row0, ng, r);
        const uint32_t g = s_g[i];
        if (g < a.g_begin || g >= a.g_end) continue;
        const uint32_t f = a.groups[g].first_row;
        const uint32_t row = f + (r - s_row0[i]);
        const uint32_t b = row == f ? 0u : uint32_t(a.tm[row - 1]);
        acc_sq<NORM>(sq, store_y<PEER>(a, row, row_sum(s_part + s_lane0[i], b, uint32_t(a.tm[row]))));
    }
    if constexpr (NORM) write_norm_partial(a.norm_part + blockIdx.x, sq);
}

// L2 prefetch of a light tile's matrix block: the tile's light groups are
// stored back to back, so its values and columns are two contiguous ranges
// (tile_rng, from the converter: no dependent metadata load).  The last warp
// issues them as 16 KB cp.async.bulk.prefetch.L2 pieces at CTA start, so the
// DRAM reads run under the metadata staging and the unit loads find their
// lines in L2.  Only for tiles of at most a.l2_prefetch bytes (the prefetched
// blocks of the resident tiles must survive in L2 until used; see
// l2_prefetch_bytes).
template <typename T>
__device__ __forceinline__ void tile_prefetch_l2(const SpmvArgs<T>& a, uint32_t kt) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t b = a.tile_rng[2 * uint64_t(kt)], e = a.tile_rng[2 * uint64_t(kt) + 1];
    if (e <= b || (e - b) * (sizeof(T) + sizeof(int32_t)) > a.l2_prefetch) return;  // bound: the tile's bytes
    auto issue = [&](const char* base, uint64_t esz) {
        // 16-B granules inside [base + b, base + e): the range start rounded down
        // stays inside the (256-B aligned) allocation, the end is rounded down
        // so no prefetch reaches past the array's last byte
        const uint64_t lo = (uint64_t(reinterpret_cast<uintptr_t>(base)) + b * esz) & ~uint64_t(15);
        const uint64_t hi = (uint64_t(reinterpret_cast<uintptr_t>(base)) + e * esz) & ~uint64_t(15);
        constexpr uint64_t kPiece = 16384;
        for (uint64_t p = lo + uint64_t(lane) * kPiece; p < hi; p += 32 * kPiece) {
            const uint32_t n = uint32_t(min(kPiece, hi - p));
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(n) : "memory");
        }
    };
    if (a.l2_prefetch_what != 'c') issue(reinterpret_cast<const char*>(a.vals), sizeof(T));
    if (a.l2_prefetch_what != 'v') issue(reinterpret_cast<const char*>(a.cols), sizeof(int32_t));
}

// Light tile kt: consecutive short-chunk groups, V-lane units, one unit per thread.
// MAP: every unit and row of the tile gets its group index in shared memory
// while the metadata loads (one thread per group, so only for small groups);
// otherwise both phases binary-search the tile's group table.
// PAIR (launched when every light chunk is <= U/2 and a tile has at most two
// units per thread): each thread's two units go through phase1_pair.
template <typename T, int V, int U, bool PRED, int MINB, bool MAP = true, bool PEER = false, bool PAIR = false,
          bool DYNW = false, bool NORM = false>
__global__ void __launch_bounds__(kTileThreads, MINB) spmv_light_kernel(const SpmvArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_part = reinterpret_cast<double*>(smem);
    const uint64_t pol_stream = a.stream_evict_first ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_x = a.x_evict_last ? policy_evict_last() : policy_evict_normal();
    const double xs = x_scale_value(a);

    const uint32_t kt = a.tile0 + blockIdx.x;
    // every tile is in range (the whole matrix): prefetch before anything else
    if (a.l2_prefetch && a.all_groups && threadIdx.x >= blockDim.x - 32) tile_prefetch_l2(a, kt);
    const uint32_t gs = a.tiles[kt], ge = a.tiles[kt + 1];
    if (ge <= a.g_begin || gs >= a.g_end || gs == ge) {
        if (NORM && threadIdx.x == 0) a.norm_part[a.norm_light0 + kt] = 0.0;
        return;
    }
    if (a.l2_prefetch && !a.all_groups && threadIdx.x >= blockDim.x - 32) tile_prefetch_l2(a, kt);
    const uint32_t ng = ge - gs;
    const uint32_t cap = a.max_tile_groups;
    // smem: s_part[max_tile_units * V] | s_off[cap] | s_ub[cap+1] | s_first[cap+1] | s_chunk[cap]
    //       | s_ugrp[max_tile_units] | s_rgrp[max_tile_rows]  (unit / row -> group in tile)
    uint64_t* s_off = reinterpret_cast<uint64_t*>(s_part + size_t(a.max_tile_units) * V);
    uint32_t* s_ub = reinterpret_cast<uint32_t*>(s_off + cap);
    uint32_t* s_first = s_ub + cap + 1;
    uint32_t* s_chunk = s_first + cap + 1;
    uint16_t* s_ugrp = reinterpret_cast<uint16_t*>(s_chunk + cap);
    uint16_t* s_rgrp = s_ugrp + a.max_tile_units;

    const uint64_t ub0 = a.unit_base[gs];
    const uint32_t row0 = MAP ? a.groups[gs].first_row : 0u;
    __shared__ uint32_t s_next;  // DYNW: next 32-unit chunk
    if (DYNW && threadIdx.x == 0) s_next = blockDim.x / 32;
    // lengths of this thread's first two units (loaded under the metadata staging)
    uint32_t ulen2[2] = {0xFFFFFFFFu, 0xFFFFFFFFu};
    if (a.ulen) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint64_t gu = ub0 + threadIdx.x + k * blockDim.x;
            if (gu < a.total_units) ulen2[k] = a.ulen[gu];
        }
    }
    for (uint32_t i = threadIdx.x; i <= ng; i += blockDim.x) {
        const GroupDesc d = a.groups[gs + i];
        const uint32_t ub = uint32_t(a.unit_base[gs + i] - ub0);
        s_first[i] = d.first_row;
        s_ub[i] = ub;
        if (i < ng) {
            s_off[i] = d.off_stride;
            s_chunk[i] = d.chunk;
            if constexpr (MAP) {
                const uint32_t ue = uint32_t(a.unit_base[gs + i + 1] - ub0), re = a.groups[gs + i + 1].first_row;
                for (uint32_t u = ub; u < ue; ++u) s_ugrp[u] = uint16_t(i);
                for (uint32_t r = d.first_row; r < re; ++r) s_rgrp[r - row0] = uint16_t(i);
            }
        }
    }
    __syncthreads();

    // Phase-2 metadata of this thread's first row, fetched under phase 1.
    const uint32_t row_end = s_first[ng];
    const uint32_t pr = (MAP ? row0 : s_first[0]) + threadIdx.x;
    uint32_t pgi = 0, pb = 0, pe = 0;
    bool pvalid = false;
    if (pr < row_end) {
        pgi = MAP ? s_rgrp[pr - row0] : find_le(s_first, ng, pr);
        const uint32_t g = gs + pgi;
        pvalid = !(s_off[pgi] & kHeavyBit) && g >= a.g_begin && g < a.g_end;
        if (pvalid) {
            pb = pr == s_first[pgi] ? 0u : uint32_t(a.tm[pr - 1]);
            pe = uint32_t(a.tm[pr]);
        }
    }

    const uint32_t nunits = s_ub[ng];
    if constexpr (PAIR) {
        uint64_t slot[2] = {0, 0};
        uint32_t ch[2] = {0, 0}, st[2] = {0, 0};
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t u = threadIdx.x + k * blockDim.x;
            if (u >= nunits) continue;
            const uint32_t gi = MAP ? s_ugrp[u] : find_le(s_ub, ng, u);
            const uint32_t g = gs + gi;
            const uint64_t os = s_off[gi];
            if ((os & kHeavyBit) || g < a.g_begin || g >= a.g_end) continue;
            slot[k] = (os & kOffsetMask) + (u - s_ub[gi]) * V;
            st[k] = uint32_t((os >> 48) & 0x7FFF);
            ch[k] = min(s_chunk[gi], ulen2[k]);
        }
        double sp[2][V];
        phase1_pair<T, V, U / 2>(a, slot, ch, st, sp, pol_stream, pol_x, xs);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t u = threadIdx.x + k * blockDim.x;
            if (u < nunits) {
#pragma unroll
                for (int l = 0; l < V; ++l) s_part[size_t(u) * V + l] = sp[k][l];
            }
        }
    }
    auto unit = [&](uint32_t u, uint32_t ulen_hint) {
        const uint32_t gi = MAP ? s_ugrp[u] : find_le(s_ub, ng, u);
        const uint32_t g = gs + gi;
        if ((s_off[gi] & kHeavyBit) || g < a.g_begin || g >= a.g_end) return;
        double s[V];
        const uint64_t os = s_off[gi];
        const uint32_t len = a.ulen ? min(s_chunk[gi], ulen_hint) : s_chunk[gi];
        phase1<T, V, U, PRED>(a, (os & kOffsetMask) + (u - s_ub[gi]) * V, len, (os >> 48) & 0x7FFF, s, pol_stream,
                              pol_x, xs);
#pragma unroll
        for (int l = 0; l < V; ++l) s_part[size_t(u) * V + l] = s[l];
    };
    if constexpr (DYNW) {
        // warps take 32-unit chunks: the first by warp index, the rest from a
        // shared counter, so warps whose gathers return early take more
        const uint32_t lane = threadIdx.x & 31;
        uint32_t c = threadIdx.x >> 5;
        bool first = true;
        while (c * 32 < nunits) {
            const uint32_t u = c * 32 + lane;
            if (u < nunits) unit(u, !a.ulen ? 0xFFFFFFFFu : first ? ulen2[0] : uint32_t(a.ulen[ub0 + u]));
            first = false;
            uint32_t nx = 0;
            if (lane == 0) nx = atomicAdd(&s_next, 1u);
            c = __shfl_sync(0xFFFFFFFFu, nx, 0);
        }
    } else {
        for (uint32_t u = threadIdx.x; !PAIR && u < nunits; u += blockDim.x) {
            const uint32_t k = (u - threadIdx.x) / blockDim.x;
            unit(u, !a.ulen ? 0xFFFFFFFFu : k < 2 ? ulen2[k] : uint32_t(a.ulen[ub0 + u]));
        }
    }
    __syncthreads();

    double sq = 0.0;
    if (pvalid) acc_sq<NORM>(sq, store_y<PEER>(a, pr, row_sum(s_part + size_t(s_ub[pgi]) * V, pb, pe)));
    for (uint32_t r = pr + blockDim.x; r < row_end; r += blockDim.x) {
        const uint32_t gi = MAP ? s_rgrp[r - row0] : find_le(s_first, ng, r);
        const uint32_t g = gs + gi;
        if ((s_off[gi] & kHeavyBit) || g < a.g_begin || g >= a.g_end) continue;
        const uint32_t b = r == s_first[gi] ? 0u : uint32_t(a.tm[r - 1]);
        acc_sq<NORM>(sq, store_y<PEER>(a, r, row_sum(s_part + size_t(s_ub[gi]) * V, b, uint32_t(a.tm[r]))));
    }
    if constexpr (NORM) write_norm_partial(a.norm_part + a.norm_light0 + kt, sq);
}

size_t light_smem_bytes(const argcsr_dev* m, int V, bool map = false) {
    const size_t cap = std::max<uint32_t>(m->max_tile_groups, 1);
    return size_t(m->max_tile_units) * V * sizeof(double) + cap * sizeof(uint64_t) + (cap + 1) * 4 * 2 + cap * 4 +
           (map ? (size_t(m->max_tile_units) + m->max_tile_rows) * sizeof(uint16_t) : 0);
}

template <typename K, typename T>
void launch(K kern, unsigned grid, size_t smem, const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s) {
    if (grid == 0) return;
    if (smem > 48 * 1024) CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTileThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.numAttrs = 0;
    const size_t xbytes = m->n_used * sizeof(T);  // x, or x' = x[perm] (xremap.cu)
    if (knobs().l2_window && m->l2_persist_max > 0 && xbytes > 0) {
        // Persist the leading part of x that fits the carve-out (hit ratio 1):
        // all of x for the stencils; the hot low-index columns of R-MAT.
        const size_t win = std::min<size_t>({xbytes, size_t(m->l2_window_max), m->l2_persist_max});
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = const_cast<T*>(a.x);
        attr[0].val.accessPolicyWindow.num_bytes = win;
        attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    if (knobs().carveout >= 0)  // experiments: shared memory / L1 split (percent of the maximum carve-out)
        CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, knobs().carveout));
    CUDA_OK(cudaLaunchKernelEx(&cfg, kern, a));
}

template <typename T, int V, int U, bool PRED, int MINB, bool PEER, bool NORM>
void launch_light(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s) {
    // small groups (units + rows per group, on average): fill the maps, else search
    const double per_group = m->num_groups ? double(m->total_units + m->num_rows) / double(m->num_groups) : 0.0;
    const int fm = knobs().map;  // experiments: force 1 / 0
    const bool map = fm >= 0 ? fm == 1 : per_group <= 24.0;
    // every light chunk <= U/2 and at most two units per thread: pair them
    const bool pair = knobs().pair != 0 && m->max_light_chunk <= uint32_t(U / 2) &&
                      m->max_tile_units <= 2 * uint64_t(kTileThreads);
    const size_t sm_map = light_smem_bytes(m, V, true), sm_search = light_smem_bytes(m, V);
    const unsigned grid = m->num_tiles;
    if (pair) {  // (twice the loads in flight per thread: 64 registers, 4 CTAs/SM)
        if (map) launch(spmv_light_kernel<T, V, U, PRED, 4, true, PEER, true, false, NORM>, grid, sm_map, m, a, s);
        else launch(spmv_light_kernel<T, V, U, PRED, 4, false, PEER, true, false, NORM>, grid, sm_search, m, a, s);
    } else if (!PEER && (knobs().light_dyn >= 0 ? knobs().light_dyn == 1 : m->num_heavy > 0)) {
        // power-law matrices (heavy groups present, light chunks of every
        // size): warps take 32-unit chunks dynamically (C3 +2%; C2 -3%, so
        // not for stencils).  ARGCSR_LIGHT_DYN=0|1 forces it (experiments).
        if (map) launch(spmv_light_kernel<T, V, U, PRED, MINB, true, false, false, true, NORM>, grid, sm_map, m, a, s);
        else launch(spmv_light_kernel<T, V, U, PRED, MINB, false, false, false, true, NORM>, grid, sm_search, m, a, s);
    } else if (map) {
        launch(spmv_light_kernel<T, V, U, PRED, MINB, true, PEER, false, false, NORM>, grid, sm_map, m, a, s);
    } else {
        launch(spmv_light_kernel<T, V, U, PRED, MINB, false, PEER, false, false, NORM>, grid, sm_search, m, a, s);
    }
}

// hardware-dispatched tiles, unpredicated value loads, 5 CTAs per SM
// (measured best on C2-C4 with the lane-compact layout)
template <typename T, bool PEER, bool NORM>
void launch_v(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s) {
    switch (m->lanes_per_unit) {
        case 4: launch_light<T, 4, 4, false, 5, PEER, NORM>(m, a, s); break;
        case 2: launch_light<T, 2, 4, false, 5, PEER, NORM>(m, a, s); break;
        // one lane per unit: 40 registers, 6 CTAs/SM (C3 1.538 vs 1.552 ms at 5)
        default: launch_light<T, 1, 4, false, 6, PEER, NORM>(m, a, s); break;
    }
}

// Long-chunk groups: one lane per thread, scalar x gathers, lanes of
// consecutive LPT-ordered groups packed into 256-thread CTAs.  fp64: 8 element
// steps in flight per lane at 4 CTAs/SM; fp32: 4 steps at 6 CTAs/SM with the
// next batch's columns loaded under the current gathers (C4 fp32 0.59 ->
// 0.50 ms; the pipelined walk does not help fp64).  ARGCSR_HEAVY_PIPE=0|1
// swaps the two walks (A/B, tests).  Variants measured and removed from the
// library are listed in DESIGN.md section 4.
template <typename T, bool PEER, bool NORM>
void launch_heavy(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t hs) {
    const size_t smem = size_t(std::max<uint64_t>(m->heavy_max_lanes, 1)) * sizeof(double);
    constexpr bool f32 = sizeof(T) == sizeof(float);
    const char hp = knobs().heavy_pipe;
    const bool pipe = hp ? hp == '1' : f32;
    if constexpr (f32) {
        if (pipe) launch(spmv_heavy_kernel<T, 4, 6, PEER, NORM, true>, m->heavy_ctas, smem, m, a, hs);
        else launch(spmv_heavy_kernel<T, 4, 6, PEER, NORM, false>, m->heavy_ctas, smem, m, a, hs);
    } else {
        if (pipe) launch(spmv_heavy_kernel<T, 8, 4, PEER, NORM, true>, m->heavy_ctas, smem, m, a, hs);
        else launch(spmv_heavy_kernel<T, 8, 4, PEER, NORM, false>, m->heavy_ctas, smem, m, a, hs);
    }
}

template <typename T, bool PEER, bool NORM>
void launch_all(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s) {
    // Heavy groups run concurrently on the handle's auxiliary stream (forked
    // from and joined back into `s`), launched first so their CTAs start first.
    const bool fork = m->heavy_ctas > 0 && m->num_tiles > 0;
    if (fork) {
        CUDA_OK(cudaEventRecord(m->ev_fork, s));
        CUDA_OK(cudaStreamWaitEvent(m->aux, m->ev_fork, 0));
    }
    if (m->heavy_ctas > 0) launch_heavy<T, PEER, NORM>(m, a, fork ? m->aux : s);
    launch_v<T, PEER, NORM>(m, a, s);
    if (fork) {
        CUDA_OK(cudaEventRecord(m->ev_join, m->aux));
        CUDA_OK(cudaStreamWaitEvent(s, m->ev_join, 0));
    }
}

// L2 policy of a handle ("tile L2 prefetch"): x (x') fits the
// persisting window -- x gathers evict_last, light tiles prefetched; x larger
// than the window on a regular matrix (no long-chunk groups, no power-law
// schedule: stencil-like, x reused within a band of rows) -- x gathers
// evict_normal and tiles prefetched (evict_last x lines would crowd the
// prefetched blocks out of L2); power-law matrices with a large x (R-MAT) --
// evict_last, no prefetch (their hot x columns need the L2).
// Measured (ms, one box each): C2 (128,1) 0.331 -> 0.293, C2 (128,4) 0.345 ->
// 0.306, C1 0.0348 -> 0.0338, C4 0.619 -> 0.608 (x fits); C5 on one GPU 2.315
// -> 2.108 (evict_normal + prefetch; prefetch with evict_last x: 2.63 ->
// 3.55); R-MAT 1.52 -> 1.71 if prefetched; C2 (128,32) 0.254 -> 0.368 if its
// 768 KB tiles were prefetched, hence the 256 KB bound.
// ARGCSR_L2PF=0|1|N forces the prefetch off / on (256 KB) / on up to N KB and
// ARGCSR_XPOL=0|1 the x policy (experiments).
bool x_fits_window(const argcsr_dev* m) {
    const size_t xbytes = m->n_used * (m->dtype == ARGCSR_F64 ? sizeof(double) : sizeof(float));
    const size_t win = std::min<size_t>(size_t(m->l2_window_max), m->l2_persist_max);
    return knobs().l2_window && xbytes <= win;
}
bool regular_matrix(const argcsr_dev* m) { return m->num_heavy == 0 && !m->powerlaw_schedule; }

uint32_t l2_prefetch_bytes(const argcsr_dev* m) {
    constexpr uint32_t kMaxTileBytes = 256 * 1024;
    const int k = knobs().l2pf;
    if (k >= 0) return k == 0 ? 0u : k == 1 ? kMaxTileBytes : uint32_t(std::min(k, 1 << 20)) * 1024u;
    return x_fits_window(m) || regular_matrix(m) ? kMaxTileBytes : 0u;
}
// What a tile prefetches: only its columns on a regular matrix whose x fits
// the window (the gathers wait on the columns; the values load in parallel
// with the gathers and need no head start: C2 0.294 -> 0.285 ms, C2 (128,4)
// 0.304 -> 0.297 against both arrays), both arrays otherwise (C5 2.11 vs 2.17,
// C4 0.608 vs 0.615 with columns only).  ARGCSR_L2PF_WHAT=b|c|v forces it.
char l2_prefetch_what(const argcsr_dev* m) {
    const char k = knobs().l2pf_what;
    if (k == 'b' || k == 'c' || k == 'v') return k;
    return x_fits_window(m) && regular_matrix(m) ? 'c' : 'b';
}
int x_evict_last(const argcsr_dev* m) {
    const int k = knobs().x_evict_last;
    if (k >= 0) return k;
    return x_fits_window(m) || !regular_matrix(m) ? 1 : 0;
}

template <typename T>
void launch_dtype(const argcsr_dev* m, const void* x, void* y, uint32_t gb, uint32_t ge, cudaStream_t s,
                  const SpmvExtra& ex) {
    SpmvArgs<T> a{};
    const uint32_t npeers = ex.npeers;
    void* const* peer_y = ex.peer_y;
    const uint64_t* peer_rows = ex.peer_rows;
    a.npeers = npeers;
    a.norm_part = ex.norm_part;
    for (uint32_t q = 0; q < npeers; ++q) {
        a.peer_y[q] = static_cast<T*>(peer_y[q]);
        a.peer_lo[q] = peer_rows ? uint32_t(std::min<uint64_t>(peer_rows[2 * q], m->num_rows)) : 0u;
        a.peer_hi[q] = peer_rows ? uint32_t(std::min<uint64_t>(peer_rows[2 * q + 1], m->num_rows))
                                 : uint32_t(m->num_rows);
    }
    a.x_scale = ex.x_scale;
    a.vals = static_cast<const T*>(m->values);
    a.cols = m->columns;
    a.groups = m->groups;
    a.tm = static_cast<const uint16_t*>(m->tm);
    a.assigned = static_cast<const uint16_t*>(m->assigned);
    a.unit_base = m->unit_base;
    a.ulen = m->ulen;
    a.total_units = m->total_units;
    a.tiles = m->tiles;
    a.tile_rng = m->tile_rng;
    a.heavy = m->heavy;
    a.heavy_ptr = m->heavy_ptr;
    a.x = static_cast<const T*>(x);
    a.y = static_cast<T*>(y);
    a.heavy_ctas = m->heavy_ctas;
    a.norm_light0 = uint32_t(norm_heavy_slots(m));
    a.g_begin = gb;
    a.g_end = ge;
    a.all_groups = gb == 0 && ge >= m->num_groups;
    a.max_tile_groups = std::max<uint32_t>(m->max_tile_groups, 1);
    a.max_tile_rows = m->max_tile_rows;
    a.tile0 = 0;
    a.max_tile_units = uint32_t(m->max_tile_units);
    a.x_evict_last = x_evict_last(m);
    // values/columns: L2 evict_normal (evict_first measured slower once the heavy
    // stream is prioritised: C4 0.69 vs 0.73, C3 0.323 vs 0.325); ARGCSR_SPOL=1 for A/B
    a.stream_evict_first = knobs().stream_evict_first;
    a.l2_prefetch = l2_prefetch_bytes(m);
    a.l2_prefetch_what = l2_prefetch_what(m);

    if (a.npeers) {
        if (a.norm_part) launch_all<T, true, true>(m, a, s);
        else launch_all<T, true, false>(m, a, s);
    } else {
        if (a.norm_part) launch_all<T, false, true>(m, a, s);
        else launch_all<T, false, false>(m, a, s);
    }
}

// Light tiles [t0, t1) only, default kernel (the pipelined host path; the
// handle has no heavy groups and no x remap).
template <typename T>
void launch_tiles_dtype(const argcsr_dev* m, const void* x, void* y, uint32_t t0, uint32_t t1, cudaStream_t s) {
    SpmvArgs<T> a{};
    a.vals = static_cast<const T*>(m->values);
    a.cols = m->columns;
    a.groups = m->groups;
    a.tm = static_cast<const uint16_t*>(m->tm);
    a.assigned = static_cast<const uint16_t*>(m->assigned);
    a.unit_base = m->unit_base;
    a.ulen = m->ulen;
    a.total_units = m->total_units;
    a.tiles = m->tiles;
    a.tile_rng = m->tile_rng;
    a.heavy = m->heavy;
    a.heavy_ptr = m->heavy_ptr;
    a.x = static_cast<const T*>(x);
    a.y = static_cast<T*>(y);
    a.heavy_ctas = 0;
    a.g_begin = 0;
    a.g_end = uint32_t(m->num_groups);
    a.all_groups = 1;
    a.max_tile_groups = std::max<uint32_t>(m->max_tile_groups, 1);
    a.max_tile_rows = m->max_tile_rows;
    a.max_tile_units = uint32_t(m->max_tile_units);
    a.x_scale = nullptr;
    a.x_evict_last = x_evict_last(m);
    a.stream_evict_first = 0;
    a.l2_prefetch = l2_prefetch_bytes(m);
    a.l2_prefetch_what = l2_prefetch_what(m);
    a.tile0 = t0;
    const double per_group = m->num_groups ? double(m->total_units + m->num_rows) / double(m->num_groups) : 0.0;
    const unsigned grid = t1 - t0;
    if (m->lanes_per_unit != 4) fail(ARGCSR_E_INTERNAL, "spmv_launch_tiles: V = 4 handles only");
    if (per_group <= 24.0)
        launch(spmv_light_kernel<T, 4, 4, false, 5, true>, grid, light_smem_bytes(m, 4, true), m, a, s);
    else
        launch(spmv_light_kernel<T, 4, 4, false, 5, false>, grid, light_smem_bytes(m, 4), m, a, s);
}

}  // namespace


void spmv_launch_tiles(const argcsr_dev* m, const void* x, void* y, uint32_t t0, uint32_t t1, cudaStream_t s) {
    if (t1 <= t0) return;
    if (m->dtype == ARGCSR_F64) launch_tiles_dtype<double>(m, x, y, t0, t1, s);
    else launch_tiles_dtype<float>(m, x, y, t0, t1, s);
}

// scale_is_norm2: s = fl(1 / fl(sqrt(||y_prev||^2))), once per SpMV into the
// handle's scalar (the SpMV kernels then only read a plain scale).
__global__ void k_norm2_to_scale(const double* n2, double* out) { *out = __drcp_rn(__dsqrt_rn(*n2)); }

void spmv_launch(const argcsr_dev* m, const void* x, void* y, uint64_t group_begin, uint64_t group_end,
                 cudaStream_t s, const SpmvExtra& ex_in) {
    const uint32_t gb = uint32_t(std::min<uint64_t>(group_begin, m->num_groups));
    const uint32_t ge = uint32_t(std::min<uint64_t>(group_end, m->num_groups));
    if (gb >= ge) return;
    Phase range("argcsr_spmv", s);  // NVTX only
    SpmvExtra ex = ex_in;
    if (ex.x_scale && ex.scale_is_norm2) {
        k_norm2_to_scale<<<1, 1, 0, s>>>(ex.x_scale, m->scale_buf);
        LAUNCH_OK("k_norm2_to_scale");
        ex.x_scale = m->scale_buf;
        ex.scale_is_norm2 = false;
    }
    x = ex.reuse_x && m->x_remap ? m->xbuf : xremap_apply(m, x, s);
    if (m->dtype == ARGCSR_F64) launch_dtype<double>(m, x, y, gb, ge, s, ex);
    else launch_dtype<float>(m, x, y, gb, ge, s, ex);
}

// Fixed-order sum of the per-CTA norm partials, in two levels so that no
// thread walks a long dependent chain: level 1 -- CTA c sums entries
// [c * 4096, (c + 1) * 4096) (each thread 16 consecutive entries in order,
// then a fixed pairwise tree over the 256 thread sums); level 2 -- one CTA
// sums the level-1 results the same way.  Deterministic run to run.
constexpr uint32_t kNormSeg = 4096;

__device__ __forceinline__ double block_tree_sum_256(double v) {
    __shared__ double s[256];
    s[threadIdx.x] = v;
    __syncthreads();
    for (uint32_t w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] = __dadd_rn(s[threadIdx.x], s[threadIdx.x + w]);
        __syncthreads();
    }
    return s[0];
}

__global__ void __launch_bounds__(256) k_norm_level(const double* __restrict__ p, uint64_t n, double* __restrict__ out) {
    const uint64_t base = uint64_t(blockIdx.x) * kNormSeg + uint64_t(threadIdx.x) * 16;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k)
        if (base + k < n) v = __dadd_rn(v, p[base + k]);
    const double t = block_tree_sum_256(v);
    if (threadIdx.x == 0) out[blockIdx.x] = t;
}

void norm_reduce(const double* partials, uint64_t n, double* out, cudaStream_t s, double* scratch) {
    const uint64_t nb = (n + kNormSeg - 1) / kNormSeg;
    if (nb <= 1) {
        k_norm_level<<<1, 256, 0, s>>>(partials, n, out);
        LAUNCH_OK("k_norm_level");
        return;
    }
    if (!scratch) fail(ARGCSR_E_INTERNAL, "norm_reduce: scratch needed above 4096 partials");
    if (nb > kNormSeg) fail(ARGCSR_E_UNSUPPORTED, "norm_reduce: more than 2^24 partials");
    k_norm_level<<<unsigned(nb), 256, 0, s>>>(partials, n, scratch);
    LAUNCH_OK("k_norm_level");
    k_norm_level<<<1, 256, 0, s>>>(scratch, nb, out);
    LAUNCH_OK("k_norm_level");
}

// ------------------------------------------------ multi-GPU step signalling
// A rank announces "my slice of the next x (and my partial ||y||^2) has
// landed in your buffers" by storing the step number into its slot of every
// peer's flag array; a peer waits until all its slots reach the step.  The
// stores of the preceding SpMV (same stream, earlier kernel) are ordered
// before the flag by the system-scope release fence.
struct PeerSlots {  // by value as a kernel parameter
    uint64_t* flag[kMaxPeers];
    double* partial[kMaxPeers];
};

__global__ void k_peer_signal(PeerSlots p, uint32_t n, uint64_t value, const double* partial) {
    if (threadIdx.x != 0) return;
    if (partial) {
        const double v = *partial;
        for (uint32_t q = 0; q < n; ++q) p.partial[q][0] = v;
    }
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (uint32_t q = 0; q < n; ++q)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.flag[q]), "l"(value) : "memory");
}

// A peer that never signals (it died) would hang the GPU: after 60 s of
// waiting the kernel traps, so the step fails loudly instead.
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_peer_wait(const uint64_t* flags, uint32_t n, uint64_t value) {
    const uint64_t t0 = globaltimer_ns();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        uint64_t v;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + i) : "memory");
            if (v < value) {
                __nanosleep(200);
                if (globaltimer_ns() - t0 > 60ull * 1000000000ull) __trap();
            }
        } while (v < value);
    }
    __syncthreads();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

void peer_signal(uint64_t* const* flags, uint32_t n, uint64_t value, const double* partial,
                 double* const* partial_dst, cudaStream_t s) {
    PeerSlots p{};
    for (uint32_t q = 0; q < n; ++q) p.flag[q] = flags[q], p.partial[q] = partial_dst ? partial_dst[q] : nullptr;
    k_peer_signal<<<1, 32, 0, s>>>(p, n, value, partial_dst ? partial : nullptr);
    CUDA_OK(cudaGetLastError());
}

void peer_wait(const uint64_t* flags, uint32_t n, uint64_t value, cudaStream_t s) {
    if (n == 0) return;
    k_peer_wait<<<1, 32, 0, s>>>(flags, n, value);
    CUDA_OK(cudaGetLastError());
}

}  // namespace argcsr_gpu
