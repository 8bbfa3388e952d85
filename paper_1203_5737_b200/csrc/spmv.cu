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
// evict-first); x gathers are L2 evict-last and x is additionally covered by a
// persisting access-policy window sized from the device's persisting-L2 limit.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "spmv.cuh"

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
    const uint32_t* __restrict__ tiles;
    const uint32_t* __restrict__ heavy;
    const uint32_t* __restrict__ heavy_ptr;
    const TileDesc* __restrict__ ttiles;  // lane-compact TMA tiles
    uint32_t num_ttiles;
    uint32_t stage_bytes;
    const T* __restrict__ x;
    T* __restrict__ y;
    uint32_t heavy_ctas;
    uint32_t g_begin, g_end;  // rows of groups outside [g_begin, g_end) are not written
    uint32_t max_tile_groups;
    uint32_t max_tile_units;
    const double* x_scale;   // y = A (s * x), s = *x_scale (device) or 1.0: each gather is fl(s * x[c])
    int x_evict_last;        // x gathers: L2 evict_last (1) or evict_normal (0)
    int stream_evict_first;  // values/columns: L2 evict_first (1) or evict_normal (0)
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
            for (int l = 0; l < V; ++l)
                xv[u][l] = c[u][l] != -1 ? ld_x(a.x + c[u][l], pol_x) : 0.0;
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

template <typename T> __device__ __forceinline__ T to_out(double v);
template <> __device__ __forceinline__ double to_out<double>(double v) { return v; }
template <> __device__ __forceinline__ float to_out<float>(double v) { return __double2float_rn(v); }

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
template <typename T, int UH>
__global__ void __launch_bounds__(kTileThreads, 2) spmv_heavy_kernel(const SpmvArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_part = reinterpret_cast<double*>(smem);
    __shared__ uint32_t s_lane0[kTileThreads + 1], s_row0[kTileThreads + 1], s_g[kTileThreads];
    const uint64_t pol_stream = a.stream_evict_first ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_x = a.x_evict_last ? policy_evict_last() : policy_evict_normal();
    const double xs = a.x_scale ? *a.x_scale : 1.0;
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
        double s[1];
        phase1<T, 1, UH, false>(a, d.offset() + (l - s_lane0[i]), d.chunk, d.stride(), s, pol_stream, pol_x, xs);
        s_part[l] = s[0];
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < nrows; r += blockDim.x) {
        const uint32_t i = find_le(s_row0, ng, r);
        const uint32_t g = s_g[i];
        if (g < a.g_begin || g >= a.g_end) continue;
        const uint32_t f = a.groups[g].first_row;
        const uint32_t row = f + (r - s_row0[i]);
        const uint32_t b = row == f ? 0u : uint32_t(a.tm[row - 1]);
        a.y[row] = to_out<T>(row_sum(s_part + s_lane0[i], b, uint32_t(a.tm[row])));
    }
}

// Light tile kt: consecutive short-chunk groups, V-lane units, one unit per thread.
template <typename T, int V, int U, bool PRED, int MINB>
__global__ void __launch_bounds__(kTileThreads, MINB) spmv_light_kernel(const SpmvArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_part = reinterpret_cast<double*>(smem);
    const uint64_t pol_stream = a.stream_evict_first ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_x = a.x_evict_last ? policy_evict_last() : policy_evict_normal();
    const double xs = a.x_scale ? *a.x_scale : 1.0;

    const uint32_t kt = blockIdx.x;
    const uint32_t gs = a.tiles[kt], ge = a.tiles[kt + 1];
    if (ge <= a.g_begin || gs >= a.g_end || gs == ge) return;
    const uint32_t ng = ge - gs;
    const uint32_t cap = a.max_tile_groups;
    // smem: s_part[max_tile_units * V] | s_off[cap] | s_ub[cap+1] | s_first[cap+1] | s_chunk[cap]
    uint64_t* s_off = reinterpret_cast<uint64_t*>(s_part + size_t(a.max_tile_units) * V);
    uint32_t* s_ub = reinterpret_cast<uint32_t*>(s_off + cap);
    uint32_t* s_first = s_ub + cap + 1;
    uint32_t* s_chunk = s_first + cap + 1;

    const uint64_t ub0 = a.unit_base[gs];
    for (uint32_t i = threadIdx.x; i <= ng; i += blockDim.x) {
        const GroupDesc d = a.groups[gs + i];
        s_first[i] = d.first_row;
        s_ub[i] = uint32_t(a.unit_base[gs + i] - ub0);
        if (i < ng) {
            s_off[i] = d.off_stride;
            s_chunk[i] = d.chunk;
        }
    }
    __syncthreads();

    // Phase-2 metadata of this thread's first row, fetched under phase 1.
    const uint32_t row0 = s_first[0], row_end = s_first[ng];
    const uint32_t pr = row0 + threadIdx.x;
    uint32_t pgi = 0, pb = 0, pe = 0;
    bool pvalid = false;
    if (pr < row_end) {
        pgi = find_le(s_first, ng, pr);
        const uint32_t g = gs + pgi;
        pvalid = !(s_off[pgi] & kHeavyBit) && g >= a.g_begin && g < a.g_end;
        if (pvalid) {
            pb = pr == s_first[pgi] ? 0u : uint32_t(a.tm[pr - 1]);
            pe = uint32_t(a.tm[pr]);
        }
    }

    const uint32_t nunits = s_ub[ng];
    for (uint32_t u = threadIdx.x; u < nunits; u += blockDim.x) {
        const uint32_t gi = find_le(s_ub, ng, u);
        const uint32_t g = gs + gi;
        if ((s_off[gi] & kHeavyBit) || g < a.g_begin || g >= a.g_end) continue;
        double s[V];
        const uint64_t os = s_off[gi];
        phase1<T, V, U, PRED>(a, (os & kOffsetMask) + (u - s_ub[gi]) * V, s_chunk[gi], (os >> 48) & 0x7FFF, s, pol_stream,
                              pol_x, xs);
#pragma unroll
        for (int l = 0; l < V; ++l) s_part[size_t(u) * V + l] = s[l];
    }
    __syncthreads();

    if (pvalid) a.y[pr] = to_out<T>(row_sum(s_part + size_t(s_ub[pgi]) * V, pb, pe));
    for (uint32_t r = pr + blockDim.x; r < row_end; r += blockDim.x) {
        const uint32_t gi = find_le(s_first, ng, r);
        const uint32_t g = gs + gi;
        if ((s_off[gi] & kHeavyBit) || g < a.g_begin || g >= a.g_end) continue;
        const uint32_t b = r == s_first[gi] ? 0u : uint32_t(a.tm[r - 1]);
        a.y[r] = to_out<T>(row_sum(s_part + size_t(s_ub[gi]) * V, b, uint32_t(a.tm[r])));
    }
}

// ---------------------------------------------------------- cp.async helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// --------------------------------------- persistent light path (prefetched metadata)
// Same per-tile work as spmv_light_kernel, but each CTA walks tiles k,
// k+gridDim.x, ... and prefetches the NEXT tile's group descriptors and unit
// bases into a second shared-memory buffer with cp.async while the current
// tile streams, so the two dependent metadata round trips leave the critical
// path (the tiles[] entries are fetched one more tile ahead into registers).
__device__ __forceinline__ uint32_t find_le64(const uint64_t* arr, uint32_t n, uint64_t key) {
    uint32_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) / 2;
        if (arr[mid] <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}
__device__ __forceinline__ uint32_t find_row(const GroupDesc* d, uint32_t n, uint32_t row) {
    uint32_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) / 2;
        if (d[mid].first_row <= row) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <typename T, int V, int U, bool PRED, int MINB, bool DYN>
__global__ void __launch_bounds__(kTileThreads, MINB) spmv_lightp_kernel(const SpmvArgs<T> a, uint32_t num_tiles,
                                                                        uint32_t* __restrict__ sched) {
    // sched[0]: next dynamic tile (offset by gridDim.x), sched[1]: CTAs done;
    // the last CTA to finish resets both, so consecutive launches reuse them.
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_grab[2];  // alternating slots: written one sync after the last read
    double* s_part = reinterpret_cast<double*>(smem);
    const uint32_t cap = a.max_tile_groups;
    const size_t part_bytes = (size_t(a.max_tile_units) * V * sizeof(double) + 15) & ~size_t(15);
    unsigned char* mbase = smem + part_bytes;
    const size_t meta_bytes = ((size_t(cap) + 1) * (sizeof(GroupDesc) + sizeof(uint64_t)) + 15) & ~size_t(15);
    auto meta_desc = [&](int b) { return reinterpret_cast<GroupDesc*>(mbase + b * meta_bytes); };
    auto meta_ub = [&](int b) { return reinterpret_cast<uint64_t*>(meta_desc(b) + cap + 1); };
    const uint64_t pol_stream = a.stream_evict_first ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_x = a.x_evict_last ? policy_evict_last() : policy_evict_normal();
    const double xs = a.x_scale ? *a.x_scale : 1.0;
    const uint32_t tid = threadIdx.x;
    auto issue_meta = [&](uint32_t gs, uint32_t ge, int b) {
        for (uint32_t i = tid; i <= ge - gs; i += blockDim.x) {
            cp_async16(smem_u32(meta_desc(b) + i), a.groups + gs + i, pol_x);
            cp_async8(smem_u32(meta_ub(b) + i), a.unit_base + gs + i);
        }
    };
    // Tile order: static round-robin (k += gridDim.x; neighbouring tiles run
    // concurrently, which keeps stencil x windows hot in L2) or dynamic.
    uint32_t static_next = blockIdx.x;
    auto grab = [&]() {
        if constexpr (DYN) return gridDim.x + atomicAdd(sched, 1u);
        static_next += gridDim.x;
        return static_next;
    };

    uint32_t k = blockIdx.x, it = 0;
    if (tid == 0) s_grab[0] = grab();
    uint32_t gs = 0, ge = 0;
    if (k < num_tiles) {
        gs = a.tiles[k], ge = a.tiles[k + 1];
        issue_meta(gs, ge, 0);
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    uint32_t kn = s_grab[0], gsn = 0, gen = 0;
    if (kn < num_tiles) gsn = a.tiles[kn], gen = a.tiles[kn + 1];
    int mb = 0;
    while (k < num_tiles) {
        const bool has_next = kn < num_tiles;
        if (has_next) issue_meta(gsn, gen, mb ^ 1);
        cp_commit();
        if (tid == 0) s_grab[(it + 1) & 1] = has_next ? grab() : num_tiles;

        const uint32_t ng = ge - gs;
        const GroupDesc* md = meta_desc(mb);
        const uint64_t* mub = meta_ub(mb);
        const bool live = ng > 0 && !(ge <= a.g_begin || gs >= a.g_end);
        const uint64_t ub0 = mub[0];
        const uint32_t row0 = md[0].first_row, row_end = live ? md[ng].first_row : row0;

        // phase-2 metadata of this thread's first row (registers)
        const uint32_t pr = row0 + tid;
        uint32_t pgi = 0, pb = 0, pe = 0;
        bool pvalid = false;
        if (pr < row_end) {
            pgi = find_row(md, ng, pr);
            const uint32_t g = gs + pgi;
            pvalid = !md[pgi].heavy() && g >= a.g_begin && g < a.g_end;
            if (pvalid) {
                pb = pr == md[pgi].first_row ? 0u : uint32_t(a.tm[pr - 1]);
                pe = uint32_t(a.tm[pr]);
            }
        }
        const uint32_t nunits = live ? uint32_t(mub[ng] - ub0) : 0u;
        for (uint32_t u = tid; u < nunits; u += blockDim.x) {
            const uint32_t gi = find_le64(mub, ng, ub0 + u);
            const uint32_t g = gs + gi;
            const GroupDesc d = md[gi];
            if (d.heavy() || g < a.g_begin || g >= a.g_end) continue;
            double sacc[V];
            phase1<T, V, U, PRED>(a, d.offset() + (ub0 + u - mub[gi]) * V, d.chunk, d.stride(), sacc, pol_stream,
                                  pol_x, xs);
#pragma unroll
            for (int l = 0; l < V; ++l) s_part[size_t(u) * V + l] = sacc[l];
        }
        cp_wait<0>();
        __syncthreads();
        const uint32_t k2 = s_grab[(it + 1) & 1];  // tile after next: its tiles[] entries load under phase 2
        uint32_t gs2 = 0, ge2 = 0;
        if (k2 < num_tiles) gs2 = a.tiles[k2], ge2 = a.tiles[k2 + 1];

        if (pvalid) a.y[pr] = to_out<T>(row_sum(s_part + size_t(mub[pgi] - ub0) * V, pb, pe));
        for (uint32_t r = pr + blockDim.x; r < row_end; r += blockDim.x) {
            const uint32_t gi = find_row(md, ng, r);
            const uint32_t g = gs + gi;
            if (md[gi].heavy() || g < a.g_begin || g >= a.g_end) continue;
            const uint32_t b = r == md[gi].first_row ? 0u : uint32_t(a.tm[r - 1]);
            a.y[r] = to_out<T>(row_sum(s_part + size_t(mub[gi] - ub0) * V, b, uint32_t(a.tm[r])));
        }
        __syncthreads();
        k = kn, gs = gsn, ge = gen;
        kn = k2, gsn = gs2, gen = ge2;
        mb ^= 1;
        ++it;
    }
    if (DYN && tid == 0) {
        __threadfence();
        if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
            sched[0] = 0;
            sched[1] = 0;
            __threadfence();
        }
    }
}

size_t lightp_smem_bytes(const argcsr_dev* m, int V) {
    const size_t cap = std::max<uint32_t>(m->max_tile_groups, 1);
    return ((size_t(m->max_tile_units) * V * sizeof(double) + 15) & ~size_t(15)) +
           2 * (((cap + 1) * (sizeof(GroupDesc) + sizeof(uint64_t)) + 15) & ~size_t(15));
}

template <typename T, int V, int U, bool PRED, int MINB, bool DYN>
void launch_lightp(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s);


// ------------------------------------------- lane-compact TMA path (default)
// Persistent CTAs (one per SM) walk the tiles k = blockIdx.x, +gridDim.x, ...
// A tile is a run of whole light groups whose value/column blocks are ONE
// contiguous stored range in the lane-compact layout.  One elected thread
// stages a tile into a shared-memory stage with five cp.async.bulk copies
// (group descriptors, unit bases, threads_mapping of its rows, columns,
// values) completing on the stage's mbarrier; `nstages` stages are kept in
// flight, so the HBM stream runs ahead of the x gathers and the reduction
// (they never wait on each other except through a full ring).  Consumers:
//   phase 1  one V-lane unit per thread and step, columns/values from shared
//            memory, 4 element steps (4V x gathers) in flight, partial sums
//            per lane to the stage's partial section;
//   phase 2  one row per thread, +0.0 + p_b + ... ascending (bit-exact order).
struct StageHdr {
    uint32_t p_desc, p_ub, p_tm, p_cols, p_vals, p_part;
    uint32_t gs, ng, row0, nrows, nunits, nslots;
    uint64_t ub0, slot_begin;
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, uint64_t src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Stage tile k: header + bulk copies (16-B aligned-down/up sections; the
// device arrays carry 16 B of tail padding for the round-up).
template <typename T, int V>
__device__ __forceinline__ void tma_issue(const SpmvArgs<T>& a, const TileDesc& t, unsigned char* stage,
                                          StageHdr* hdr, uint64_t* bar, uint64_t pol_meta, uint64_t pol_stream) {
    const uint64_t src[5] = {uint64_t(a.groups + t.gs), uint64_t(a.unit_base + t.gs), uint64_t(a.tm + t.row0),
                             uint64_t(a.cols + t.slot_begin), uint64_t(a.vals + t.slot_begin)};
    const uint64_t len[5] = {sizeof(GroupDesc) * (uint64_t(t.ng) + 1), sizeof(uint64_t) * (uint64_t(t.ng) + 1),
                             sizeof(uint16_t) * uint64_t(t.nrows), sizeof(int32_t) * uint64_t(t.nslots),
                             sizeof(T) * uint64_t(t.nslots)};
    uint64_t lo[5];
    uint32_t n[5], p[5], off = 0, total = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        lo[i] = src[i] & ~uint64_t(15);
        n[i] = len[i] ? uint32_t(((src[i] + len[i] + 15) & ~uint64_t(15)) - lo[i]) : 0u;
        p[i] = off + uint32_t(src[i] - lo[i]);
        off += n[i];
        total += n[i];
    }
    hdr->p_desc = p[0], hdr->p_ub = p[1], hdr->p_tm = p[2], hdr->p_cols = p[3], hdr->p_vals = p[4];
    hdr->p_part = off;
    hdr->gs = t.gs, hdr->ng = t.ng, hdr->row0 = t.row0, hdr->nrows = t.nrows, hdr->nunits = t.nunits;
    hdr->nslots = t.nslots;
    hdr->ub0 = t.ub0, hdr->slot_begin = t.slot_begin;
    mbar_arrive_expect_tx(bar, total);
    off = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (n[i]) bulk_g2s(stage + off, lo[i], n[i], bar, i >= 3 ? pol_stream : pol_meta);
        off += n[i];
    }
}

template <typename T, int V> struct SmemVec;
template <> struct SmemVec<double, 4> {
    static __device__ __forceinline__ void load(const double* p, double (&v)[4]) {
        const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
        v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
    }
};
template <> struct SmemVec<float, 4> {
    static __device__ __forceinline__ void load(const float* p, float (&v)[4]) {
        const float4 a = *reinterpret_cast<const float4*>(p);
        v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
    }
};

template <typename T, int V, int NT>
__global__ void __launch_bounds__(NT) spmv_tma_kernel(const SpmvArgs<T> a, uint32_t nstages) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[4];
    __shared__ StageHdr hdrs[4];
    const uint32_t tid = threadIdx.x;
    const uint32_t G = gridDim.x;
    const uint32_t SB = a.stage_bytes;
    const uint64_t pol_x = a.x_evict_last ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_meta = policy_evict_normal();
    const double xs = a.x_scale ? *a.x_scale : 1.0;
    const uint32_t mine = a.num_ttiles > blockIdx.x ? (a.num_ttiles - blockIdx.x + G - 1) / G : 0;
    if (tid == 0) {
        for (uint32_t s = 0; s < nstages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (uint32_t i = 0; i < nstages && i < mine; ++i)
            tma_issue<T, V>(a, a.ttiles[blockIdx.x + i * G], smem + size_t(i) * SB, &hdrs[i], &bars[i], pol_meta,
                            pol_stream);
    }
    __syncthreads();
    for (uint32_t i = 0; i < mine; ++i) {
        const uint32_t st = i % nstages;
        mbar_wait(&bars[st], (i / nstages) & 1);
        unsigned char* stage = smem + size_t(st) * SB;
        const StageHdr h = hdrs[st];
        // the descriptor of the tile this stage is refilled with, loaded now
        // so that its latency is off the end-of-tile critical path
        TileDesc nxt;
        const bool refill = tid == 0 && i + nstages < mine;
        if (refill) nxt = a.ttiles[blockIdx.x + (i + nstages) * G];
        const GroupDesc* sd = reinterpret_cast<const GroupDesc*>(stage + h.p_desc);
        const uint64_t* sub = reinterpret_cast<const uint64_t*>(stage + h.p_ub);
        const uint16_t* stm = reinterpret_cast<const uint16_t*>(stage + h.p_tm);
        const int32_t* scol = reinterpret_cast<const int32_t*>(stage + h.p_cols);
        const T* sval = reinterpret_cast<const T*>(stage + h.p_vals);
        double* spart = reinterpret_cast<double*>(stage + h.p_part);
        const uint32_t ns = h.nslots;

        // Phase 1 (argcsr.cpp:193-203).  A unit is V adjacent lanes of a
        // group; its steps j = 0 .. chunk-1 are the V-slot vectors
        // offset + j * stride + V * u.  Units are dealt out balanced by steps:
        // in the unit-major order of the tile's steps, thread t owns the units
        // that START in [t, t + 1) * steps / NT and runs them to the end.  A
        // thread walks its steps in batches of kB (kB * V gathers in flight),
        // batches crossing unit boundaries; each lane's sum is a sequential
        // chain over j ascending from +0.0, stopping at sentinels (which are
        // trailing), exactly the reference's.
        {
            constexpr uint32_t kB = 4;
            const uint32_t nq = ns / V;  // steps of the tile
            const uint32_t qb = uint32_t(uint64_t(nq) * tid / NT), qe = uint32_t(uint64_t(nq) * (tid + 1) / NT);
            // group holding virtual step qb: last gi with (offset - slot_begin) / V <= qb
            uint32_t gi = 0;
            {
                uint32_t lo = 0, hi = h.ng - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) / 2;
                    if (uint32_t((sd[mid].offset() - h.slot_begin) / V) <= qb) lo = mid; else hi = mid - 1;
                }
                gi = lo;
            }
            GroupDesc d = sd[gi];
            uint32_t chunk = d.chunk, wv = d.stride() / V;
            uint32_t gq0 = uint32_t((d.offset() - h.slot_begin) / V);
            uint32_t ub = uint32_t(sub[gi] - h.ub0);
            // first unit of this group starting at or after qb
            uint32_t ul = chunk ? (qb - gq0 + chunk - 1) / chunk : wv;
            uint32_t j = 0;
            bool more = qb < qe;
            auto next_group = [&]() {
                for (;;) {
                    if (++gi >= h.ng) {
                        more = false;
                        return;
                    }
                    d = sd[gi];
                    chunk = d.chunk;
                    if (chunk) break;  // all-empty group: rows give +0.0 in phase 2
                }
                wv = d.stride() / V;
                gq0 = uint32_t((d.offset() - h.slot_begin) / V);
                ub = uint32_t(sub[gi] - h.ub0);
                ul = 0;
            };
            if (more && ul >= wv) next_group();
            if (more && gq0 + ul * chunk >= qe) more = false;
            double acc[V];
            while (more) {
                uint32_t mq[kB], uid[kB], flags = 0;  // bit 2b: first step, bit 2b+1: last step
                uint32_t cnt = 0;
#pragma unroll
                for (uint32_t b = 0; b < kB; ++b) {
                    if (!more) break;
                    mq[b] = gq0 + j * wv + ul;
                    uid[b] = ub + ul;
                    if (j == 0) flags |= 1u << (2 * b);
                    if (j + 1 == chunk) flags |= 2u << (2 * b);
                    ++cnt;
                    if (++j == chunk) {
                        j = 0;
                        if (++ul >= wv) next_group();
                        if (more && gq0 + ul * chunk >= qe) more = false;
                    }
                }
                int c[kB][V];
                T v[kB][V];
#pragma unroll
                for (uint32_t b = 0; b < kB; ++b) {
                    if (b < cnt) {
                        if constexpr (V == 4) {
                            const int4 cc = reinterpret_cast<const int4*>(scol)[mq[b]];
                            c[b][0] = cc.x, c[b][1] = cc.y, c[b][2] = cc.z, c[b][3] = cc.w;
                            SmemVec<T, 4>::load(sval + 4 * mq[b], v[b]);
                        } else {
#pragma unroll
                            for (int l = 0; l < V; ++l) c[b][l] = scol[V * mq[b] + l], v[b][l] = sval[V * mq[b] + l];
                        }
                    } else {
#pragma unroll
                        for (int l = 0; l < V; ++l) c[b][l] = -1, v[b][l] = T(0);
                    }
                }
                double xv[kB][V];
#pragma unroll
                for (uint32_t b = 0; b < kB; ++b)
#pragma unroll
                    for (int l = 0; l < V; ++l) xv[b][l] = c[b][l] != -1 ? ld_x(a.x + c[b][l], pol_x) : 0.0;
                if (a.x_scale) {
#pragma unroll
                    for (uint32_t b = 0; b < kB; ++b)
#pragma unroll
                        for (int l = 0; l < V; ++l) xv[b][l] = __dmul_rn(xv[b][l], xs);
                }
#pragma unroll
                for (uint32_t b = 0; b < kB; ++b) {
                    if (b < cnt) {
                        if (flags & (1u << (2 * b))) {
#pragma unroll
                            for (int l = 0; l < V; ++l) acc[l] = 0.0;
                        }
#pragma unroll
                        for (int l = 0; l < V; ++l)
                            if (c[b][l] != -1) acc[l] = __dadd_rn(acc[l], __dmul_rn(double(v[b][l]), xv[b][l]));
                        if (flags & (2u << (2 * b))) {
#pragma unroll
                            for (int l = 0; l < V; ++l) spart[size_t(uid[b]) * V + l] = acc[l];
                        }
                    }
                }
            }
        }
        __syncthreads();

        // Phase 2 (argcsr.cpp:206-215): +0.0 + p_b + p_{b+1} + ... ascending,
        // one row per thread.
        for (uint32_t r = tid; r < h.nrows; r += NT) {
            const uint32_t row = h.row0 + r;
            const uint32_t gi = find_row(sd, h.ng, row);
            const GroupDesc d = sd[gi];
            const uint32_t g = h.gs + gi;
            if (d.heavy() || g < a.g_begin || g >= a.g_end) continue;
            double sum = 0.0;
            if (d.chunk) {
                const uint32_t b = row == d.first_row ? 0u : uint32_t(stm[r - 1]);
                sum = row_sum(spart + size_t(sub[gi] - h.ub0) * V, b, uint32_t(stm[r]));
            }
            a.y[row] = to_out<T>(sum);
        }
        __syncthreads();  // stage st fully consumed
        if (refill) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_issue<T, V>(a, nxt, stage, &hdrs[st], &bars[st], pol_meta, pol_stream);
        }
    }
}

size_t light_smem_bytes(const argcsr_dev* m, int V) {
    const size_t cap = std::max<uint32_t>(m->max_tile_groups, 1);
    return size_t(m->max_tile_units) * V * sizeof(double) + cap * sizeof(uint64_t) + (cap + 1) * 4 * 2 + cap * 4;
}

bool l2_window_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ARGCSR_L2_WINDOW");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Kernel variant for experiments: ARGCSR_SPMV_VARIANT = U<unroll>P<pred>B<min CTAs/SM>,
// one of the instantiated set below.
int variant_id() {
    static const int id = [] {
        const char* e = std::getenv("ARGCSR_SPMV_VARIANT");
        if (!e) return -1;
        const char* names[] = {"LP4P1B4", "U2P1B6", "U4P0B4", "U4P1B5", "U4P1B3", "U8P1B2", "U4P1B4", "U2P1B8",
                               "-", "-", "LP4P0B4", "LP2P1B6", "LPD4P1B4"};
        for (int i = 0; i < 13; ++i)
            if (!std::strcmp(e, names[i])) return i;
        return -1;
    }();
    return id;
}

int env_flag(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? (e[0] != '0') : dflt;
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
    const size_t xbytes = m->num_cols * sizeof(T);
    if (l2_window_enabled() && m->l2_persist_max > 0 && xbytes > 0) {
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
    CUDA_OK(cudaLaunchKernelEx(&cfg, kern, a));
}

template <typename T, int V, int U, bool PRED, int MINB>
void launch_light(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s) {
    launch(spmv_light_kernel<T, V, U, PRED, MINB>, m->num_tiles, light_smem_bytes(m, V), m, a, s);
}

template <typename T, int V, int U, bool PRED, int MINB, bool DYN>
void launch_lightp(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s) {
    int dev = 0, sms = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t smem = lightp_smem_bytes(m, V);
    auto kern = spmv_lightp_kernel<T, V, U, PRED, MINB, DYN>;
    if (smem > 48 * 1024) CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTileThreads, smem));
    const unsigned grid = unsigned(std::min<uint64_t>(m->num_tiles, uint64_t(std::max(per_sm, 1)) * sms));
    if (grid == 0) return;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTileThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.numAttrs = 0;
    const size_t xbytes = m->num_cols * sizeof(T);
    if (l2_window_enabled() && m->l2_persist_max > 0 && xbytes > 0) {
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
    CUDA_OK(cudaLaunchKernelEx(&cfg, kern, a, m->num_tiles, m->sched));
}

int tma_threads() {
    static const int nt = [] {
        const char* e = std::getenv("ARGCSR_TMA_THREADS");
        const int v = e ? std::atoi(e) : 256;
        return (v == 512 || v == 1024) ? v : 256;
    }();
    return nt;
}
int tma_ctas_per_sm() {  // resident CTAs per SM the stages are sized for
    static const int c = [] {
        const char* e = std::getenv("ARGCSR_TMA_CTAS");
        const int v = e ? std::atoi(e) : 2;
        return std::min(std::max(v, 1), 8);
    }();
    return c;
}

// Returns false when the handle has no TMA schedule or two stages do not fit.
template <typename T, int V, int NT>
bool launch_tma_nt(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s) {
    int dev = 0, sms = 0, optin = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_OK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    auto kern = spmv_tma_kernel<T, V, NT>;
    int per_sm_smem = 0;
    CUDA_OK(cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    const uint32_t SB = m->stage_bytes;
    if (SB == 0) return false;
    // stages per CTA: as many as fit (<= 4) with tma_ctas_per_sm() CTAs per SM,
    // at least 2 (fewer CTAs per SM if needed)
    uint32_t nst = 0;
    for (int ctas = tma_ctas_per_sm(); ctas >= 1 && nst < 2; --ctas) {
        const size_t budget = std::min<size_t>(size_t(optin), size_t(per_sm_smem) / ctas) - 1024;
        nst = uint32_t(std::min<size_t>(4, budget / SB));
    }
    if (nst < 2) return false;
    const size_t smem = size_t(nst) * SB;
    CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    const unsigned grid = unsigned(std::min<uint64_t>(m->num_ttiles, uint64_t(std::max(per_sm, 1)) * sms));
    if (grid == 0) return true;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.numAttrs = 0;
    const size_t xbytes = m->num_cols * sizeof(T);
    if (l2_window_enabled() && m->l2_persist_max > 0 && xbytes > 0) {
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
    CUDA_OK(cudaLaunchKernelEx(&cfg, kern, a, nst));
    return true;
}

template <typename T, int V>
bool launch_tma(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s) {
    if (m->layout != kLayoutCompact || m->num_ttiles == 0) return false;
    switch (tma_threads()) {
        case 256: return launch_tma_nt<T, V, 256>(m, a, s);
        case 1024: return launch_tma_nt<T, V, 1024>(m, a, s);
        default: return launch_tma_nt<T, V, 512>(m, a, s);
    }
}

template <typename T, int V>
void launch_v(const argcsr_dev* m, const SpmvArgs<T>& a, cudaStream_t s) {
    int vid = variant_id();
    // Opt-in experiment (measured slower): the TMA-staged kernel.
    const char* ev = std::getenv("ARGCSR_SPMV_VARIANT");
    if (ev && !std::strcmp(ev, "TMA") && launch_tma<T, V>(m, a, s)) return;
    if (vid < 0) {
        // Default: persistent CTAs with prefetched metadata and dynamic tile
        // order when there are no heavy groups (e.g. stencils); otherwise
        // hardware dispatch of independent tiles (measured best for R-MAT).
        vid = m->num_heavy == 0 ? 12 : 6;
    }
    switch (vid) {
        case 0: launch_lightp<T, V, 4, true, 4, false>(m, a, s); return;
        case 10: launch_lightp<T, V, 4, false, 4, false>(m, a, s); return;
        case 11: launch_lightp<T, V, 2, true, 6, false>(m, a, s); return;
        case 12: launch_lightp<T, V, 4, true, 4, true>(m, a, s); return;
        default: break;
    }
    switch (vid) {
        case 1: launch_light<T, V, 2, true, 6>(m, a, s); break;
        case 2: launch_light<T, V, 4, false, 4>(m, a, s); break;
        case 3: launch_light<T, V, 4, true, 5>(m, a, s); break;
        case 4: launch_light<T, V, 4, true, 3>(m, a, s); break;
        case 5: launch_light<T, V, 8, true, 2>(m, a, s); break;
        case 6: launch_light<T, V, 4, true, 4>(m, a, s); break;
        case 7: launch_light<T, V, 2, true, 8>(m, a, s); break;
        default: launch_light<T, V, 4, true, 4>(m, a, s); break;
    }
}

template <typename T>
void launch_dtype(const argcsr_dev* m, const void* x, const double* x_scale, void* y, uint32_t gb, uint32_t ge,
                  cudaStream_t s) {
    SpmvArgs<T> a;
    a.x_scale = x_scale;
    a.vals = static_cast<const T*>(m->values);
    a.cols = m->columns;
    a.groups = m->groups;
    a.tm = static_cast<const uint16_t*>(m->tm);
    a.assigned = static_cast<const uint16_t*>(m->assigned);
    a.unit_base = m->unit_base;
    a.tiles = m->tiles;
    a.heavy = m->heavy;
    a.heavy_ptr = m->heavy_ptr;
    a.ttiles = m->ttiles;
    a.num_ttiles = m->num_ttiles;
    a.stage_bytes = m->stage_bytes;
    a.x = static_cast<const T*>(x);
    a.y = static_cast<T*>(y);
    a.heavy_ctas = m->heavy_ctas;
    a.g_begin = gb;
    a.g_end = ge;
    a.max_tile_groups = std::max<uint32_t>(m->max_tile_groups, 1);
    a.max_tile_units = uint32_t(m->max_tile_units);
    a.x_evict_last = env_flag("ARGCSR_XPOL", 1);
    a.stream_evict_first = env_flag("ARGCSR_SPOL", m->num_heavy > 0 ? 1 : 0);

    // Heavy groups run concurrently on the handle's auxiliary stream (forked
    // from and joined back into `s`), launched first so their CTAs start first.
    const bool fork = m->heavy_ctas > 0 && m->num_tiles > 0;
    if (fork) {
        CUDA_OK(cudaEventRecord(m->ev_fork, s));
        CUDA_OK(cudaStreamWaitEvent(m->aux, m->ev_fork, 0));
    }
    if (m->heavy_ctas > 0) {
        const size_t smem = size_t(std::max<uint64_t>(m->heavy_max_lanes, 1)) * sizeof(double);
        launch(spmv_heavy_kernel<T, 16>, m->heavy_ctas, smem, m, a, fork ? m->aux : s);
    }
    switch (m->lanes_per_unit) {
        case 4: launch_v<T, 4>(m, a, s); break;
        case 2: launch_v<T, 2>(m, a, s); break;
        default: launch_v<T, 1>(m, a, s); break;
    }
    if (fork) {
        CUDA_OK(cudaEventRecord(m->ev_join, m->aux));
        CUDA_OK(cudaStreamWaitEvent(s, m->ev_join, 0));
    }
}

}  // namespace

void spmv_launch(const argcsr_dev* m, const void* x, void* y, uint64_t group_begin, uint64_t group_end,
                 cudaStream_t s, const double* x_scale) {
    const uint32_t gb = uint32_t(std::min<uint64_t>(group_begin, m->num_groups));
    const uint32_t ge = uint32_t(std::min<uint64_t>(group_end, m->num_groups));
    if (gb >= ge) return;
    if (m->dtype == ARGCSR_F64) launch_dtype<double>(m, x, x_scale, y, gb, ge, s);
    else launch_dtype<float>(m, x, x_scale, y, gb, ge, s);
}

}  // namespace argcsr_gpu
