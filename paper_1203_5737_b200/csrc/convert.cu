// CSR -> ARG-CSR conversion on the GPU, bit-exact with the reference
// argcsr_from_csr (proj/src/argcsr.cpp:123-155).  The two sequential greedies
// of the reference are restated data-parallel:
//
//   K1 k1_next          budget boundary next(r) per row        (argcsr.cpp:30-45 admission test)
//   K2 k2_*             group starts = orbit of row 0 under next, resolved with
//                       exact per-tile transfer tables           (argcsr.cpp:17-46)
//   K3 k3_assign        threads per row by threshold search on event keys,
//                       inclusive scan into threads_mapping      (argcsr.cpp:48-89, 141-145)
//   K4 exclusive scans  slot offsets, SpMV work units            (argcsr.cpp:151-152)
//   K5 k5_layout        per-slot gather into the columnwise block (argcsr.cpp:91-121)
//
// plus the SpMV schedule (light tiles, heavy groups in LPT order).
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "convert.cuh"
#include "scan.cuh"
#include "xremap.cuh"

namespace argcsr_gpu {

namespace {

constexpr uint32_t kTileRows = 8192;       // K2 tile length (rows)
constexpr uint32_t kMaxTiledTpg = 1024;    // K2 tile path bound (one thread per entry)
constexpr uint16_t kEnd = 0xFFFF;          // K2: chain reached num_rows
constexpr uint32_t kResolveBatch = 12000;  // K2 resolve: table entries per smem batch (< 48 KB)

__device__ __forceinline__ uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
// chunk_filling, argcsr.cpp:11-13
__device__ __forceinline__ uint64_t filling(uint64_t n, uint64_t t) { return n == 0 ? 0 : cdiv(n, t); }

// ------------------------------------------------------------------- K1
// next(r) = max(r+1, max{e <= min(r+tpg, N) : P[e]-P[r] <= budget}).  A group
// opened at r admits row e-1 iff (e-r <= tpg) and (P[e]-P[r] <= budget), the
// reference's `count + 1 > tpg || elements + cnt > budget` test; P is
// monotone, so the admissible ends form a prefix and a binary search finds it.
__global__ void k1_next(const uint64_t* __restrict__ rp, uint64_t N, uint64_t tpg, uint64_t budget,
                        uint32_t* __restrict__ next) {
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < N;
         r += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t base = rp[r];
        uint64_t e;
        if (rp[r + 1] - base > budget) {
            e = r + 1;  // oversized row: singleton group (argcsr.hpp:75-76)
        } else {
            uint64_t lo = r + 1, hi = (tpg >= N - r) ? N : r + tpg;
            while (lo < hi) {
                const uint64_t mid = lo + (hi - lo + 1) / 2;
                if (rp[mid] - base <= budget) lo = mid; else hi = mid - 1;
            }
            e = lo;
        }
        next[r] = uint32_t(e);
    }
}

// ------------------------------------------------------------------- K2
// Any chain entering tile [T, T+L) first lands in [T, T+tpg) (a jump is at
// most tpg rows), so each tile is summarised by a table over its <= tpg entry
// offsets: exit offset into the next tile and number of group starts.
__global__ void __launch_bounds__(1024) k2_tile_tables(const uint32_t* __restrict__ next, uint32_t N, uint32_t E,
                                                       uint16_t* __restrict__ exit_tab,
                                                       uint16_t* __restrict__ cnt_tab) {
    __shared__ uint32_t s_next[kTileRows];
    const uint32_t T = blockIdx.x * kTileRows;
    const uint32_t Lk = min(kTileRows, N - T);
    for (uint32_t i = threadIdx.x; i < Lk; i += blockDim.x) s_next[i] = next[T + i];
    __syncthreads();
    const uint32_t tile_end = T + Lk;
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
        uint32_t s = T + e, c = 0;
        uint16_t ex = kEnd;
        if (s < N) {
            while (s < tile_end) {
                ++c;
                s = s_next[s - T];
            }
            ex = s >= N ? kEnd : uint16_t(s - tile_end);
        }
        exit_tab[size_t(blockIdx.x) * E + e] = ex;
        cnt_tab[size_t(blockIdx.x) * E + e] = uint16_t(c);
    }
}

// One CTA composes the tile tables in order: entry/base group of every tile.
__global__ void __launch_bounds__(1024) k2_resolve(const uint16_t* __restrict__ exit_tab,
                                                   const uint16_t* __restrict__ cnt_tab, uint32_t ntiles,
                                                   uint32_t E, uint32_t* __restrict__ tile_entry,
                                                   uint32_t* __restrict__ tile_gbase,
                                                   uint32_t* __restrict__ total_groups) {
    extern __shared__ uint16_t s_tab[];  // [2][TB*E]
    const uint32_t TB = max(1u, kResolveBatch / E);
    uint16_t* s_exit = s_tab;
    uint16_t* s_cnt = s_tab + size_t(TB) * E;
    __shared__ uint32_t s_entry, s_gbase;
    if (threadIdx.x == 0) s_entry = 0, s_gbase = 0;
    for (uint32_t k0 = 0; k0 < ntiles; k0 += TB) {
        const uint32_t nb = min(TB, ntiles - k0);
        const size_t n = size_t(nb) * E;
        __syncthreads();
        for (size_t i = threadIdx.x; i < n; i += blockDim.x) {
            s_exit[i] = exit_tab[size_t(k0) * E + i];
            s_cnt[i] = cnt_tab[size_t(k0) * E + i];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t entry = s_entry, gb = s_gbase;
            for (uint32_t k = 0; k < nb; ++k) {
                tile_entry[k0 + k] = entry;
                tile_gbase[k0 + k] = gb;
                if (entry == kEnd) continue;
                gb += s_cnt[size_t(k) * E + entry];
                entry = s_exit[size_t(k) * E + entry];
            }
            s_entry = entry;
            s_gbase = gb;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *total_groups = s_gbase;
}

// Re-walk each tile's true chain and emit its group starts.
__global__ void __launch_bounds__(256) k2_emit(const uint32_t* __restrict__ next, uint32_t N,
                                               const uint32_t* __restrict__ tile_entry,
                                               const uint32_t* __restrict__ tile_gbase,
                                               uint32_t* __restrict__ first_row) {
    __shared__ uint32_t s_next[kTileRows];
    const uint32_t T = blockIdx.x * kTileRows;
    const uint32_t Lk = min(kTileRows, N - T);
    const uint32_t entry = tile_entry[blockIdx.x];
    if (entry == kEnd) return;
    for (uint32_t i = threadIdx.x; i < Lk; i += blockDim.x) s_next[i] = next[T + i];
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = T + entry, g = tile_gbase[blockIdx.x];
        const uint32_t tile_end = T + Lk;
        while (s < tile_end) {
            first_row[g++] = s;
            s = s_next[s - T];
        }
    }
}

// threads_per_group > kMaxTiledTpg: few, large groups -> one sequential walk.
__global__ void k2_sequential(const uint32_t* __restrict__ next, uint32_t N, uint32_t* __restrict__ first_row,
                              uint32_t* __restrict__ total_groups) {
    uint32_t s = 0, g = 0;
    while (s < N) {
        first_row[g++] = s;
        s = next[s];
    }
    *total_groups = g;
}

__global__ void k_set_u32(uint32_t* p, uint32_t v) { *p = v; }

// ------------------------------------------------------------------- K3
// Row r can take threads t = 1 .. T_max(n_r) where T_max is the first plateau
// of ceil(n/t) (the strict-improvement test, argcsr.cpp:71).  Each grant
// (r, t -> t+1) has key ceil(n_r/t), strictly decreasing per row, so the
// greedy grants events in (key desc, row asc) order: all events with key > K*
// for the smallest K* with A(K*) <= spare, then the remaining spare to the
// rows owning a key == K* event, ascending.  T_max is capped at spare+1.
__device__ __forceinline__ uint64_t plateau_capped(uint64_t n, uint64_t spare) {
    uint64_t t = 1;
    while (t <= spare && filling(n, t + 1) < filling(n, t)) ++t;
    return t;
}
// a_r(K): events of row r with key > K (K = 0: all of them).
__device__ __forceinline__ uint64_t events_above(uint64_t n, uint64_t tcap, uint64_t K) {
    if (K == 0) return tcap - 1;
    if (n <= K) return 0;
    const uint64_t a = cdiv(n, K) - 1;
    return a < tcap - 1 ? a : tcap - 1;
}

template <typename TM>
__global__ void __launch_bounds__(256) k3_assign(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ first_row,
                                                 uint32_t G, uint64_t tpg, uint32_t* __restrict__ tcap_buf,
                                                 TM* __restrict__ tm, uint32_t* __restrict__ chunk_out,
                                                 TM* __restrict__ assigned_out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t g = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < G; g += nwarps) {
        const uint32_t f = first_row[g];
        const uint32_t k = first_row[g + 1] - f;
        const uint64_t spare = tpg - k;
        uint64_t E = 0, maxn = 0;
        for (uint32_t i = lane; i < k; i += 32) {
            const uint64_t n = rp[f + i + 1] - rp[f + i];
            const uint64_t tc = plateau_capped(n, spare);
            tcap_buf[f + i] = uint32_t(tc);
            E += tc - 1;
            maxn = n > maxn ? n : maxn;
        }
        E = warp_sum_u64(E);
        maxn = warp_max_u64(maxn);
        uint64_t K = 0, left = 0;
        if (E > spare) {
            uint64_t lo = 1, hi = maxn;  // A(maxn) = 0 <= spare
            while (lo < hi) {
                const uint64_t mid = lo + (hi - lo) / 2;
                uint64_t A = 0;
                for (uint32_t i = lane; i < k; i += 32)
                    A += events_above(rp[f + i + 1] - rp[f + i], tcap_buf[f + i], mid);
                A = warp_sum_u64(A);
                if (A <= spare) hi = mid; else lo = mid + 1;
            }
            K = lo;
            uint64_t A = 0;
            for (uint32_t i = lane; i < k; i += 32)
                A += events_above(rp[f + i + 1] - rp[f + i], tcap_buf[f + i], K);
            left = spare - warp_sum_u64(A);
        }
        uint64_t carry = 0, chunk = 0, ties_before = 0;
        const unsigned lt_mask = (1u << lane) - 1u;
        for (uint32_t base = 0; base < k; base += 32) {
            const uint32_t i = base + lane;
            const bool valid = i < k;
            uint64_t n = 0, tc = 1, t = 0;
            if (valid) {
                n = rp[f + i + 1] - rp[f + i];
                tc = tcap_buf[f + i];
                t = 1 + events_above(n, tc, K);
            }
            if (K > 0) {
                const bool tie = valid && events_above(n, tc, K - 1) > events_above(n, tc, K);
                const unsigned bal = __ballot_sync(0xffffffffu, tie);
                const uint64_t rank = ties_before + __popc(bal & lt_mask);
                if (tie && rank < left) t += 1;
                ties_before += __popc(bal);
            }
            const uint64_t incl = warp_incl_scan_u64(t, lane) + carry;
            if (valid) {
                tm[f + i] = TM(incl);  // inclusive per-group scan, argcsr.cpp:141-145
                const uint64_t fl = filling(n, t);
                chunk = fl > chunk ? fl : chunk;
            }
            carry = __shfl_sync(0xffffffffu, incl, 31);
        }
        chunk = warp_max_u64(chunk);
        if (lane == 0) {
            chunk_out[g] = uint32_t(chunk);
            assigned_out[g] = TM(carry);
        }
    }
}

// ------------------------------------------------------------------- K4
// Lane stride of group g: threads_per_group (reference layout) or the
// assigned lanes rounded up to the vector width V (lane-compact layout).
template <typename TM>
struct StrideOf {
    const TM* assigned;
    uint64_t tpg;
    uint32_t V;
    bool compact;
    __device__ uint64_t operator()(uint64_t g) const {
        return compact ? (uint64_t(assigned[g]) + V - 1) / V * V : tpg;
    }
};

// Long-chunk groups (chunk_size > thr, default kHeavyChunk) run on the heavy path.
template <typename TM>
struct HeavyOf {
    const uint32_t* chunk;
    StrideOf<TM> stride;
    uint32_t thr;
    __device__ bool operator()(uint64_t g) const { return chunk[g] > thr; }
};

struct SlotsOf {  // chunk_size * threads_per_group (argcsr.cpp:151-152)
    const uint32_t* chunk;
    uint64_t tpg;
    __device__ uint64_t operator()(uint64_t g) const { return uint64_t(chunk[g]) * tpg; }
};

// Stored slots of the light (want_heavy = false) or heavy groups, 0 for the others.
template <typename TM>
struct ClassSlotsOf {
    HeavyOf<TM> heavy;
    bool want_heavy;
    __device__ uint64_t operator()(uint64_t g) const {
        return heavy(g) == want_heavy ? uint64_t(heavy.chunk[g]) * heavy.stride(g) : 0;
    }
};

// Descriptor of group g.  Reference layout: offset = reference offset.
// Lane-compact: light groups first (off_light), heavy groups after all light
// slots (light_total + off_heavy).
template <typename TM>
__global__ void k4_fill_desc(const uint32_t* __restrict__ first_row, const uint32_t* __restrict__ chunk,
                             const uint64_t* __restrict__ off_light, const uint64_t* __restrict__ off_heavy,
                             uint64_t light_total, HeavyOf<TM> heavy, uint32_t G, uint32_t N,
                             GroupDesc* __restrict__ desc) {
    for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g <= G;
         g += uint64_t(gridDim.x) * blockDim.x) {
        GroupDesc d;
        if (g < G) {
            const bool h = heavy(g);
            const uint64_t off = (off_heavy && h) ? light_total + off_heavy[g] : off_light[g];
            d.off_stride = off | (heavy.stride(g) << 48) | (h ? kHeavyBit : 0);
            d.first_row = first_row[g];
            d.chunk = chunk[g];
        } else {
            d.off_stride = off_heavy ? light_total + off_heavy[G] : off_light[G];
            d.first_row = N;
            d.chunk = 0;
        }
        desc[g] = d;
    }
}

template <typename TM>
struct UnitsOf {  // SpMV work units: ceil(assigned / V), heavy groups count 1
    const TM* assigned;
    HeavyOf<TM> heavy;
    uint32_t V;
    __device__ uint64_t operator()(uint64_t g) const {
        return heavy(g) ? 1 : (uint64_t(assigned[g]) + V - 1) / V;
    }
};

template <typename TM>
struct HeavyFlag {
    HeavyOf<TM> heavy;
    __device__ uint64_t operator()(uint64_t g) const { return heavy(g) ? 1 : 0; }
};

template <typename TM>
__global__ void k4_scatter_heavy(const uint32_t* __restrict__ chunk, const TM* __restrict__ assigned,
                                 HeavyOf<TM> heavy, const uint64_t* __restrict__ pos, uint32_t G,
                                 uint32_t* __restrict__ ids, uint32_t* __restrict__ chunks,
                                 uint32_t* __restrict__ lanes) {
    for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < G;
         g += uint64_t(gridDim.x) * blockDim.x) {
        if (heavy(g)) {
            ids[pos[g]] = uint32_t(g);
            chunks[pos[g]] = chunk[g];
            lanes[pos[g]] = assigned[g];
        }
    }
}

// Light tile k starts at the first group whose unit base is >= k * B.
__global__ void k4_tiles(const uint64_t* __restrict__ unit_base, uint32_t G, uint32_t ntiles, uint64_t span,
                         uint32_t* __restrict__ tiles) {
    for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k <= ntiles;
         k += uint64_t(gridDim.x) * blockDim.x) {
        if (k == ntiles) {
            tiles[k] = G;
            continue;
        }
        const uint64_t key = k * span;
        uint64_t lo = 0, hi = G;  // lower_bound over unit_base[0..G)
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if (unit_base[mid] < key) lo = mid + 1; else hi = mid;
        }
        tiles[k] = uint32_t(lo);
    }
}

// Largest tile: groups (out[0]) and rows (out[1]).
// Per light tile, the stored slot range [lo, hi) of its groups (contiguous:
// light groups are stored back to back), for the SpMV's L2 prefetch; (0, 0)
// when an end group is heavy (stored apart) or the tile is empty.
__global__ void k4_tile_ranges(const uint32_t* __restrict__ tiles, uint32_t ntiles,
                               const GroupDesc* __restrict__ desc, uint64_t* __restrict__ rng) {
    for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < ntiles;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t gs = tiles[k], ge = tiles[k + 1];
        uint64_t lo = 0, hi = 0;
        if (ge > gs) {
            const GroupDesc d0 = desc[gs], d1 = desc[ge - 1];
            if (!d0.heavy() && !d1.heavy()) {
                lo = d0.offset();
                hi = d1.offset() + uint64_t(d1.chunk) * d1.stride();
            }
        }
        rng[2 * k] = lo;
        rng[2 * k + 1] = hi;
    }
}

__global__ void k4_max_tile_groups(const uint32_t* __restrict__ tiles, uint32_t ntiles,
                                   const GroupDesc* __restrict__ desc, unsigned long long* __restrict__ out) {
    uint64_t m = 0, mr = 0;
    for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < ntiles;
         k += uint64_t(gridDim.x) * blockDim.x) {
        m = max(m, uint64_t(tiles[k + 1] - tiles[k]));
        mr = max(mr, uint64_t(desc[tiles[k + 1]].first_row - desc[tiles[k]].first_row));
    }
    m = warp_max_u64(m);
    mr = warp_max_u64(mr);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, (unsigned long long)m);
        atomicMax(out + 1, (unsigned long long)mr);
    }
}

// out[0] = max chunk_size, out[1] = max chunk_size of the light (short-chunk) groups
__global__ void k4_max_chunk(const uint32_t* __restrict__ chunk, uint32_t G, uint32_t thr,
                             unsigned long long* __restrict__ out) {
    uint64_t m = 0, ml = 0;
    for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < G;
         g += uint64_t(gridDim.x) * blockDim.x) {
        m = max(m, uint64_t(chunk[g]));
        if (chunk[g] <= thr) ml = max(ml, uint64_t(chunk[g]));
    }
    m = warp_max_u64(m);
    ml = warp_max_u64(ml);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, (unsigned long long)m);
        atomicMax(out + 1, (unsigned long long)ml);
    }
}

// Largest column each light tile reads (padding -1 ignored): for the
// pipelined host path, a tile may start once x is copied up to it.
__global__ void k_tile_cmax(const uint32_t* __restrict__ tiles, uint32_t ntiles, const GroupDesc* __restrict__ desc,
                            const int32_t* __restrict__ cols, uint32_t* __restrict__ cmax,
                            uint32_t* __restrict__ first_row) {
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t b = desc[tiles[t]].offset(), e = desc[tiles[t + 1]].offset();
        int32_t mx = 0;
        for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) mx = max(mx, cols[i]);
        mx = int32_t(warp_max_u64(uint64_t(uint32_t(mx))));
        __shared__ int32_t s_mx[32];
        if ((threadIdx.x & 31) == 0) s_mx[threadIdx.x >> 5] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            int32_t m = 0;
            for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) m = max(m, s_mx[w]);
            cmax[t] = uint32_t(m);
            first_row[t] = desc[tiles[t]].first_row;
        }
        __syncthreads();
    }
}

// Per light unit (V adjacent lanes of a group), the number of element steps
// holding an entry: 1 + the last step with a non-sentinel column in any of its
// lanes (sentinels trail per lane).  One warp per group, lanes over units,
// scanning down from the last step.  Also sums, over the light units, the
// slots the SpMV reads with and without the lengths (stop at the length vs.
// at the first U-step batch ending in an all-sentinel step), so the converter
// keeps the lengths only when they save more traffic than they cost.
__global__ void k6_unit_len(const GroupDesc* __restrict__ desc, const uint64_t* __restrict__ unit_base, uint32_t G,
                            uint32_t V, uint32_t U, const int32_t* __restrict__ cols, uint8_t* __restrict__ ulen,
                            unsigned long long* __restrict__ reads) {
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long with_len = 0, without = 0;
    for (uint64_t g = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < G;
         g += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const GroupDesc d = desc[g];
        if (d.heavy()) continue;
        const uint64_t ub = unit_base[g], ue = unit_base[g + 1];
        const uint64_t stride = d.stride();
        for (uint64_t u = ub + lane; u < ue; u += 32) {
            const uint64_t slot0 = d.offset() + (u - ub) * V;
            uint32_t len = d.chunk;
            for (; len > 0; --len) {
                bool any = false;
                for (uint32_t l = 0; l < V; ++l) any |= cols[slot0 + uint64_t(len - 1) * stride + l] != -1;
                if (any) break;
            }
            ulen[u] = uint8_t(len);
            with_len += uint64_t(len) * V;
            without += uint64_t(min(d.chunk, U * (len / U + 1))) * V;
        }
    }
    with_len = warp_sum_u64(with_len);
    without = warp_sum_u64(without);
    if (lane == 0) {
        atomicAdd(reads, with_len);
        atomicAdd(reads + 1, without);
    }
}

// ------------------------------------------------------------------- K5
// Gather form of layout_group: lane l of group g belongs to the row whose
// threads_mapping range holds l; its chunk c holds the row's elements
// [start, start+len) with the ceil/floor split, larger chunks first.  Slot
// (j, l) = value j of that run, or (+0.0, -1) padding, stored at
// offset + j * stride + l for l < stride.  Writes are coalesced along the lane
// dimension of each j-row (contiguous over the whole group when compact).
template <typename T, typename TM>
__global__ void __launch_bounds__(256) k5_layout(const uint64_t* __restrict__ rp, const int32_t* __restrict__ cols_in,
                                                 const T* __restrict__ vals_in, const GroupDesc* __restrict__ desc,
                                                 const TM* __restrict__ tm, const TM* __restrict__ assigned,
                                                 const int32_t* __restrict__ col_map, uint32_t G,
                                                 T* __restrict__ vals_out, int32_t* __restrict__ cols_out) {
    constexpr uint32_t WL = 1024;
    __shared__ uint64_t s_src[WL];
    __shared__ uint32_t s_len[WL];
    for (uint64_t g = blockIdx.x; g < G; g += gridDim.x) {
        const GroupDesc d = desc[g];
        const uint32_t f = d.first_row;
        const uint32_t k = desc[g + 1].first_row - f;
        const uint64_t chunk = d.chunk;
        if (chunk == 0) continue;  // all-empty group: zero slots
        const uint64_t asg = assigned[g];
        const uint64_t width = d.stride(), off = d.offset();
        for (uint64_t w0 = 0; w0 < width; w0 += WL) {
            const uint32_t wl = uint32_t(min(uint64_t(WL), width - w0));
            for (uint32_t l = threadIdx.x; l < wl; l += blockDim.x) {
                const uint64_t lane = w0 + l;
                uint64_t src = 0;
                uint32_t len = 0;
                if (lane < asg) {
                    uint32_t lo = 0, hi = k - 1;  // first local row with tm > lane
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) / 2;
                        if (uint64_t(tm[f + mid]) > lane) hi = mid; else lo = mid + 1;
                    }
                    const uint64_t b = lo ? uint64_t(tm[f + lo - 1]) : 0;
                    const uint64_t t = uint64_t(tm[f + lo]) - b;
                    const uint64_t c = lane - b;
                    const uint64_t n = rp[f + lo + 1] - rp[f + lo];
                    const uint64_t base = n / t, extra = n % t;
                    const uint64_t start = c < extra ? c * (base + 1) : extra * (base + 1) + (c - extra) * base;
                    len = uint32_t(base + (c < extra ? 1 : 0));
                    src = rp[f + lo] + start;
                }
                s_src[l] = src;
                s_len[l] = len;
            }
            __syncthreads();
            uint64_t j = threadIdx.x / wl;
            uint32_t l = threadIdx.x % wl;
            const uint32_t step_j = blockDim.x / wl, step_l = blockDim.x % wl;
            for (; j < chunk;) {
                const uint64_t slot = off + j * width + w0 + l;
                if (j < s_len[l]) {
                    const uint64_t src = s_src[l] + j;
                    vals_out[slot] = vals_in[src];
                    cols_out[slot] = col_map ? col_map[cols_in[src]] : cols_in[src];
                } else {
                    vals_out[slot] = T(0);
                    cols_out[slot] = -1;
                }
                j += step_j;
                l += step_l;
                if (l >= wl) {
                    l -= wl;
                    ++j;
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ bool is_pos_zero(double v) { return __double_as_longlong(v) == 0; }
__device__ __forceinline__ bool is_pos_zero(float v) { return __float_as_int(v) == 0; }

// Import (argcsr_dev_import_reference): per group, the reference block
// (chunk x tpg, argcsr.cpp:99-104) -> the stored block (stride lanes), column
// indices through the x remap.  Counts explicit entries (cnt[0]) and layout
// violations (cnt[1]): a free lane (>= assigned) must hold (+0.0, -1) and a
// lane's padding must trail its entries, as the reference converter writes.
template <typename T, typename TM>
__global__ void __launch_bounds__(256) k5_from_reference(const GroupDesc* __restrict__ desc,
                                                         const uint64_t* __restrict__ ref_off, uint64_t tpg,
                                                         const TM* __restrict__ assigned, const T* __restrict__ rv,
                                                         const int32_t* __restrict__ rc,
                                                         const int32_t* __restrict__ col_map, uint32_t G,
                                                         T* __restrict__ vals_out, int32_t* __restrict__ cols_out,
                                                         unsigned long long* __restrict__ cnt) {
    uint64_t explicit_n = 0, bad = 0;
    for (uint64_t g = blockIdx.x; g < G; g += gridDim.x) {
        const GroupDesc d = desc[g];
        const uint64_t w = d.stride(), off = d.offset(), asg = assigned[g], base = ref_off[g];
        const uint64_t n = uint64_t(d.chunk) * tpg;
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t j = i / tpg, lane = i - j * tpg;
            const int32_t c = rc[base + i];
            const T v = rv[base + i];
            if (c != -1) {
                ++explicit_n;
                if (lane >= asg || (j > 0 && rc[base + i - tpg] == -1)) ++bad;
            } else if (lane >= asg && !is_pos_zero(v)) {
                ++bad;
            }
            if (lane < w) {
                vals_out[off + j * w + lane] = v;
                cols_out[off + j * w + lane] = (c != -1 && col_map) ? col_map[c] : c;
            }
        }
    }
    explicit_n = warp_sum_u64(explicit_n);
    bad = warp_sum_u64(bad);
    if ((threadIdx.x & 31) == 0) {
        if (explicit_n) atomicAdd(cnt, (unsigned long long)explicit_n);
        if (bad) atomicAdd(cnt + 1, (unsigned long long)bad);
    }
}

// Units per light tile (default kDefaultTileUnits; a tile is one CTA of kTileThreads).
// ARGCSR_TILE_THREADS (128 .. 2048) sets the units per tile (experiments).
uint64_t tile_threads_setting(uint64_t dflt) {
    const long v = knobs().tile_threads;
    return (v >= 128 && v <= 8192 && v % 32 == 0) ? uint64_t(v) : dflt;
}

unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 64u) {
    const uint64_t b = (n + block - 1) / block;
    return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(b, cap)));
}

template <typename P>
struct DevPtr {  // stream-ordered scratch allocation
    P* p = nullptr;
    cudaStream_t s;
    DevPtr(size_t n, cudaStream_t st) : s(st) { CUDA_OK(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(P), s)); }
    ~DevPtr() {
        if (p) cudaFreeAsync(p, s);
    }
    DevPtr(const DevPtr&) = delete;
    DevPtr& operator=(const DevPtr&) = delete;
};

template <typename P>
P* dev_alloc(argcsr_dev* m, size_t n) {
    P* p = nullptr;
    CUDA_OK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(P)));
    m->device_bytes += std::max<size_t>(n, 1) * sizeof(P);
    return p;
}

template <typename T>
struct LayoutSource {
    const uint64_t* rp = nullptr;  // CSR (converter)
    const int32_t* cols = nullptr;
    const T* vals = nullptr;
    const int32_t* ref_cols = nullptr;  // reference layout (import), ref_slots entries
    const T* ref_vals = nullptr;
    uint64_t ref_slots = 0;
};

template <typename T, typename TM>
void layout_and_schedule(argcsr_dev* m, uint32_t G, const uint32_t* first_row, const uint32_t* chunk_p, TM* tm,
                         TM* assigned, const LayoutSource<T>& src, cudaStream_t s);

template <typename T, typename TM>
void convert_typed(argcsr_dev* m, const uint64_t* rp, const int32_t* cols, const T* vals, cudaStream_t s) {
    const uint64_t N = m->num_rows, tpg = m->tpg;
    const uint64_t budget = m->dcs * tpg;  // size_t product, wraps like argcsr.cpp:28
    const uint32_t N32 = uint32_t(N);

    Phase whole("argcsr_convert", s, true);
    PhaseSeq ph(s);
    ph.next("convert.k1_next");
    // K1
    DevPtr<uint32_t> next(N, s);
    k1_next<<<grid_for(N, 256), 256, 0, s>>>(rp, N, tpg, budget, next.p);
    LAUNCH_OK("k1_next");

    ph.next("convert.k2_partition");
    // K2
    DevPtr<uint32_t> first_row(N + 1, s);
    DevPtr<uint32_t> d_G(1, s);
    if (tpg <= kMaxTiledTpg) {
        const uint32_t ntiles = uint32_t((N + kTileRows - 1) / kTileRows);
        const uint32_t E = uint32_t(tpg);
        DevPtr<uint16_t> exit_tab(size_t(ntiles) * E, s), cnt_tab(size_t(ntiles) * E, s);
        DevPtr<uint32_t> tile_entry(ntiles, s), tile_gbase(ntiles, s);
        const unsigned thr = std::min<unsigned>(1024, (E + 31) / 32 * 32);
        k2_tile_tables<<<ntiles, thr, 0, s>>>(next.p, N32, E, exit_tab.p, cnt_tab.p);
        LAUNCH_OK("k2_tile_tables");
        const uint32_t TB = std::max(1u, kResolveBatch / E);
        const size_t smem = size_t(2) * TB * E * sizeof(uint16_t);
        k2_resolve<<<1, 1024, smem, s>>>(exit_tab.p, cnt_tab.p, ntiles, E, tile_entry.p, tile_gbase.p, d_G.p);
        LAUNCH_OK("k2_resolve");
        k2_emit<<<ntiles, 256, 0, s>>>(next.p, N32, tile_entry.p, tile_gbase.p, first_row.p);
        LAUNCH_OK("k2_emit");
    } else {
        k2_sequential<<<1, 1, 0, s>>>(next.p, N32, first_row.p, d_G.p);
        LAUNCH_OK("k2_sequential");
    }
    uint32_t G = 0;
    CUDA_OK(cudaMemcpyAsync(&G, d_G.p, sizeof G, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    m->num_groups = G;
    k_set_u32<<<1, 1, 0, s>>>(first_row.p + G, N32);
    LAUNCH_OK("k_set_u32");

    ph.next("convert.k3_assign");
    // K3
    TM* tm = dev_alloc<TM>(m, N);
    TM* assigned = dev_alloc<TM>(m, G);
    m->tm = tm;
    m->assigned = assigned;
    DevPtr<uint32_t> chunk(G, s), tcap(N, s);
    {
        const uint64_t threads = uint64_t(G) * 32;
        k3_assign<TM><<<grid_for(threads, 256, 148u * 256u), 256, 0, s>>>(rp, first_row.p, G, tpg, tcap.p, tm,
                                                                          chunk.p, assigned);
        LAUNCH_OK("k3_assign");
    }

    ph.end();
    layout_and_schedule<T, TM>(m, G, first_row.p, chunk.p, tm, assigned, LayoutSource<T>{rp, cols, vals}, s);
}

// K4 (offsets, descriptors, SpMV schedule) and K5 (the value/column blocks)
// for groups given by first_row [G+1] / chunk [G] and tm / assigned, from a
// CSR matrix (the converter) or from the reference arrays (import).
template <typename T, typename TM>
void layout_and_schedule(argcsr_dev* m, uint32_t G, const uint32_t* first_row, const uint32_t* chunk_p, TM* tm,
                         TM* assigned, const LayoutSource<T>& src, cudaStream_t s) {
    const uint64_t N = m->num_rows, tpg = m->tpg;
    const uint32_t N32 = uint32_t(N);
    PhaseSeq ph(s);
    ph.next("convert.k4_offsets");
    struct {
        const uint32_t* p;
    } chunk{chunk_p};
    // K4: offsets (+ total slots), descriptors.  The vector width V of the
    // SpMV also fixes the lane-compact stride granularity.
    const bool compact = m->layout == kLayoutCompact;
    // experiments: ARGCSR_HEAVY_CHUNK moves the light/heavy boundary (1..250;
    // measured on C3: 16 -> 1.79 ms, 8 -> 2.39, 4 -> 2.66 vs 1.64 at 32)
    m->heavy_chunk = knobs().heavy_chunk ? knobs().heavy_chunk : kHeavyChunk;
    {
        DevPtr<unsigned long long> mx(2, s);
        CUDA_OK(cudaMemsetAsync(mx.p, 0, 2 * sizeof(unsigned long long), s));
        k4_max_chunk<<<grid_for(G, 256), 256, 0, s>>>(chunk.p, G, m->heavy_chunk, mx.p);
        LAUNCH_OK("k4_max_chunk");
        unsigned long long mc[2] = {0, 0};
        CUDA_OK(cudaMemcpyAsync(mc, mx.p, sizeof mc, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        m->max_chunk = mc[0];
        m->max_light_chunk = uint32_t(mc[1]);
    }
    // (V divides tpg, so a compact stride never exceeds threads_per_group)
    uint32_t V = (tpg % 4 == 0) ? 4 : (tpg % 2 == 0) ? 2 : 1;
    // Power-law matrices (heavy groups AND long light lanes, chunk >= 8: R-MAT)
    // run the light tiles one lane per thread over 2048-unit tiles: C3 1.54
    // vs 1.64 ms (repeated A/B, profiles/r02/r02_vecab.jsonl); matrices with
    // short light lanes keep V = 4 (C2 0.38 vs 0.30, C4 0.72 vs 0.62 at V = 1).
    m->powerlaw_schedule = compact && knobs().vec == 0 && m->max_chunk > m->heavy_chunk && m->max_light_chunk >= 8;
    if (m->powerlaw_schedule) V = 1;
    // experiments: ARGCSR_VEC = 1 | 2 caps the unit width
    if (knobs().vec > 0 && uint32_t(knobs().vec) < V) V = uint32_t(knobs().vec);
    const StrideOf<TM> stride_of{assigned, tpg, V, compact};
    const HeavyOf<TM> heavy_of{chunk.p, stride_of, m->heavy_chunk};
    DevPtr<uint64_t> offset(uint64_t(G) + 1, s);
    exclusive_scan(SlotsOf{chunk.p, tpg}, G, offset.p, s);  // reference offsets
    uint64_t total_slots = 0;
    CUDA_OK(cudaMemcpyAsync(&total_slots, offset.p + G, sizeof total_slots, cudaMemcpyDeviceToHost, s));
    uint64_t stored_slots = 0, light_total = 0;
    DevPtr<uint64_t> off_heavy(compact ? uint64_t(G) + 1 : 1, s);
    if (compact) {
        uint64_t heavy_total = 0;
        exclusive_scan(ClassSlotsOf<TM>{heavy_of, false}, G, offset.p, s);
        exclusive_scan(ClassSlotsOf<TM>{heavy_of, true}, G, off_heavy.p, s);
        CUDA_OK(cudaMemcpyAsync(&light_total, offset.p + G, sizeof light_total, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaMemcpyAsync(&heavy_total, off_heavy.p + G, sizeof heavy_total, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        stored_slots = light_total + heavy_total;
    } else {
        CUDA_OK(cudaStreamSynchronize(s));
        stored_slots = light_total = total_slots;
    }
    if (stored_slots > kOffsetMask)
        fail(ARGCSR_E_UNSUPPORTED, "argcsr_from_csr: more than 2^48 stored slots");
    m->groups = dev_alloc<GroupDesc>(m, uint64_t(G) + 1);
    DevPtr<uint64_t> ref_off(src.ref_cols ? uint64_t(G) + 1 : 1, s);
    if (src.ref_cols) exclusive_scan(SlotsOf{chunk.p, tpg}, G, ref_off.p, s);
    k4_fill_desc<TM><<<grid_for(uint64_t(G) + 1, 256), 256, 0, s>>>(first_row, chunk.p, offset.p,
                                                                  compact ? off_heavy.p : nullptr, light_total,
                                                                  heavy_of, G, N32, m->groups);
    LAUNCH_OK("k4_fill_desc");
    m->total_slots = total_slots;
    m->stored_slots = stored_slots;
    m->light_slots = light_total;

    ph.next("convert.k4_schedule");
    // SpMV schedule: work units (V lanes), light tiles, heavy groups (LPT order).
    m->lanes_per_unit = int(V);
    m->unit_base = dev_alloc<uint64_t>(m, uint64_t(G) + 1);
    exclusive_scan(UnitsOf<TM>{assigned, heavy_of, V}, G, m->unit_base, s);
    uint64_t total_units = 0;
    CUDA_OK(cudaMemcpyAsync(&total_units, m->unit_base + G, sizeof total_units, cudaMemcpyDeviceToHost, s));
    {
        DevPtr<uint64_t> hpos(uint64_t(G) + 1, s);
        exclusive_scan(HeavyFlag<TM>{heavy_of}, G, hpos.p, s);
        uint64_t nh = 0;
        CUDA_OK(cudaMemcpyAsync(&nh, hpos.p + G, sizeof nh, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        m->num_heavy = uint32_t(nh);
        m->heavy = dev_alloc<uint32_t>(m, nh);
        std::vector<uint32_t> hptr{0};
        uint64_t max_lanes = 0;
        if (nh) {
            DevPtr<uint32_t> ids(nh, s), chs(nh, s), lns(nh, s);
            k4_scatter_heavy<TM><<<grid_for(G, 256), 256, 0, s>>>(chunk.p, assigned, heavy_of, hpos.p, G, ids.p,
                                                                  chs.p, lns.p);
            LAUNCH_OK("k4_scatter_heavy");
            std::vector<uint32_t> hid(nh), hch(nh), hln(nh);
            CUDA_OK(cudaMemcpyAsync(hid.data(), ids.p, nh * 4, cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaMemcpyAsync(hch.data(), chs.p, nh * 4, cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaMemcpyAsync(hln.data(), lns.p, nh * 4, cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaStreamSynchronize(s));
            std::vector<uint32_t> order(nh);
            std::iota(order.begin(), order.end(), 0u);
            // LPT: longest chunk first; ties by group index (deterministic)
            std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return hch[a] > hch[b]; });
            std::vector<uint32_t> sorted(nh);
            // Pack consecutive (similar-chunk) heavy groups into CTAs of <= kTileThreads lanes.
            uint64_t lanes = 0;
            for (uint64_t i = 0; i < nh; ++i) {
                sorted[i] = hid[order[i]];
                const uint64_t l = hln[order[i]];
                if (lanes > 0 && lanes + l > uint64_t(kTileThreads)) {
                    hptr.push_back(uint32_t(i));
                    max_lanes = std::max(max_lanes, lanes);
                    lanes = 0;
                }
                lanes += l;
            }
            hptr.push_back(uint32_t(nh));
            max_lanes = std::max(max_lanes, lanes);
            CUDA_OK(cudaMemcpyAsync(m->heavy, sorted.data(), nh * 4, cudaMemcpyHostToDevice, s));
        }
        m->heavy_ctas = uint32_t(hptr.size() - 1);
        m->heavy_max_lanes = max_lanes;
        m->heavy_ptr = dev_alloc<uint32_t>(m, hptr.size());
        m->scale_buf = dev_alloc<double>(m, 1);
        CUDA_OK(cudaMemcpyAsync(m->heavy_ptr, hptr.data(), hptr.size() * 4, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaStreamSynchronize(s));
    }
    // Tile keys every `span` units so that a tile (span + at most one group's
    // units - 1) fits one CTA pass when a group has at most half a CTA of units.
    const uint64_t maxu = (tpg + V - 1) / V;
    const uint64_t tt = tile_threads_setting(m->powerlaw_schedule ? 2048 : kDefaultTileUnits);
    const uint64_t span = maxu <= tt / 2 ? tt - maxu + 1 : tt;
    m->tile_span = span;
    m->tile_threads = uint32_t(tt);
    m->total_units = total_units;
    const uint64_t ntiles = (total_units + span - 1) / span;
    if (ntiles > 0x7fffffffull) fail(ARGCSR_E_UNSUPPORTED, "argcsr_from_csr: matrix too large for the tile schedule");
    m->num_tiles = uint32_t(ntiles);
    m->tiles = dev_alloc<uint32_t>(m, ntiles + 1);
    k4_tiles<<<grid_for(ntiles + 1, 256), 256, 0, s>>>(m->unit_base, G, uint32_t(ntiles), span, m->tiles);
    LAUNCH_OK("k4_tiles");
    m->tile_rng = dev_alloc<uint64_t>(m, 2 * std::max<uint64_t>(ntiles, 1));
    if (ntiles) {
        k4_tile_ranges<<<grid_for(ntiles, 256), 256, 0, s>>>(m->tiles, uint32_t(ntiles), m->groups, m->tile_rng);
        LAUNCH_OK("k4_tile_ranges");
    }
    {
        DevPtr<unsigned long long> mx(2, s);
        CUDA_OK(cudaMemsetAsync(mx.p, 0, 2 * sizeof(unsigned long long), s));
        if (ntiles) {
            k4_max_tile_groups<<<grid_for(ntiles, 256), 256, 0, s>>>(m->tiles, uint32_t(ntiles), m->groups, mx.p);
            LAUNCH_OK("k4_max_tile_groups");
        }
        unsigned long long mg[2] = {0, 0};
        CUDA_OK(cudaMemcpyAsync(mg, mx.p, sizeof mg, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        m->max_tile_groups = uint32_t(mg[0]);
        m->max_tile_rows = uint32_t(mg[1]);
        m->max_tile_units = span + maxu - 1;
    }

    ph.next("convert.k5_alloc");
    // K5
    m->values = dev_alloc<T>(m, stored_slots);
    m->columns = dev_alloc<int32_t>(m, stored_slots);
    int32_t* col_map = nullptr;
    if (src.ref_cols) {
        // import: the reference blocks, checked (free lanes all padding,
        // sentinels trailing per lane) and compacted
        col_map = build_xremap(m, src.ref_cols, src.ref_slots, m->xremap_mode, s, true);
        DevPtr<unsigned long long> cnt(2, s);
        CUDA_OK(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(unsigned long long), s));
        if (G > 0 && total_slots > 0) {
            const unsigned grid = unsigned(std::min<uint64_t>(G, 148u * 64u));
            k5_from_reference<T, TM><<<grid, 256, 0, s>>>(m->groups, ref_off.p, tpg, assigned, src.ref_vals,
                                                          src.ref_cols, col_map, G, static_cast<T*>(m->values),
                                                          m->columns, cnt.p);
            LAUNCH_OK("k5_from_reference");
        }
        unsigned long long h[2] = {0, 0};
        CUDA_OK(cudaMemcpyAsync(h, cnt.p, sizeof h, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        if (col_map) CUDA_OK(cudaFreeAsync(col_map, s));
        if (h[1]) fail(ARGCSR_E_FORMAT, "argcsr import: " + std::to_string(h[1]) +
                                            " slots break the ARG-CSR layout (free lanes must hold (0.0, -1) and "
                                            "padding must trail each lane)");
        m->nnz = h[0];
    } else {
        ph.next("convert.xremap");
        // x remap (lane-compact only): stored columns index x' = x[perm]
        uint64_t rp_ends[2] = {0, 0};
        CUDA_OK(cudaMemcpyAsync(&rp_ends[0], src.rp, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaMemcpyAsync(&rp_ends[1], src.rp + N, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        col_map = build_xremap(m, src.cols + rp_ends[0], rp_ends[1] - rp_ends[0], m->xremap_mode, s, false, src.rp,
                               src.cols);
        ph.next("convert.k5_layout");
        if (G > 0 && stored_slots > 0) {
            const unsigned grid = unsigned(std::min<uint64_t>(G, 0x7fffffffu));
            k5_layout<T, TM><<<grid, 256, 0, s>>>(src.rp, src.cols, src.vals, m->groups, tm, assigned, col_map, G,
                                                 static_cast<T*>(m->values), m->columns);
            LAUNCH_OK("k5_layout");
        }
        if (col_map) CUDA_OK(cudaFreeAsync(col_map, s));
    }
    CUDA_OK(cudaStreamSynchronize(s));
    ph.next("convert.k6_unit_len");
    // Light unit lengths (u8, light chunks <= kHeavyChunk): kept when the
    // padding steps they let the SpMV skip outweigh their own reads.
    if (G > 0 && total_units > 0 && stored_slots > 0) {
        m->ulen = dev_alloc<uint8_t>(m, total_units);
        CUDA_OK(cudaMemsetAsync(m->ulen, 0, total_units, s));
        DevPtr<unsigned long long> rd(2, s);
        CUDA_OK(cudaMemsetAsync(rd.p, 0, 2 * sizeof(unsigned long long), s));
        k6_unit_len<<<grid_for(uint64_t(G) * 32, 256), 256, 0, s>>>(m->groups, m->unit_base, G, V, 4, m->columns,
                                                                    m->ulen, rd.p);
        LAUNCH_OK("k6_unit_len");
        unsigned long long r[2] = {0, 0};
        CUDA_OK(cudaMemcpyAsync(r, rd.p, sizeof r, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        m->unit_len_saved = (r[1] - r[0]) * (sizeof(T) + sizeof(int32_t));
        const int fu = knobs().ulen;  // experiments: force 1 / 0
        const bool keep = fu >= 0 ? fu == 1 : m->unit_len_saved > 4 * total_units;
        if (!keep) {
            CUDA_OK(cudaFree(m->ulen));
            m->device_bytes -= total_units;
            m->ulen = nullptr;
        }
    }
    ph.next("convert.tile_cmax");
    // pipelined host path: tile column reach (light tiles only; no heavy groups, no remap)
    if (m->num_heavy == 0 && !m->x_remap && m->num_tiles >= 16) {
        const uint32_t nt = m->num_tiles;
        DevPtr<uint32_t> cm(nt, s), fr(nt, s);
        k_tile_cmax<<<std::min<uint32_t>(nt, 148u * 16u), 256, 0, s>>>(m->tiles, nt, m->groups, m->columns, cm.p, fr.p);
        LAUNCH_OK("k_tile_cmax");
        m->tile_cmax.resize(nt);
        m->tile_row.resize(nt + 1);
        CUDA_OK(cudaMemcpyAsync(m->tile_cmax.data(), cm.p, nt * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaMemcpyAsync(m->tile_row.data(), fr.p, nt * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        for (uint32_t t = 1; t < nt; ++t) m->tile_cmax[t] = std::max(m->tile_cmax[t], m->tile_cmax[t - 1]);
        m->tile_row[nt] = uint32_t(N);
    }
}

}  // namespace

__global__ void __launch_bounds__(1024) scan_partials_kernel(uint64_t* partial, uint64_t nb, uint64_t* total) {
    uint64_t carry = 0;
    for (uint64_t base = 0; base < nb; base += blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        const uint64_t v = i < nb ? partial[i] : 0;
        uint64_t tot;
        const uint64_t ex = block_excl_scan_u64(v, &tot);
        if (i < nb) partial[i] = ex + carry;
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

namespace {

// Import of the reference arrays (argcsr_dev_import): structural checks on the
// host (groups tile the rows in order, reference offsets, threads_mapping
// increasing within each group and <= threads_per_group), then the device
// layout and SpMV schedule exactly as after a conversion.
template <typename T>
void import_typed(argcsr_dev* m, uint64_t G, const uint64_t* g4, const uint64_t* tm64, const T* vals,
                  const int32_t* cols, uint64_t S, cudaStream_t s) {
    const uint64_t N = m->num_rows, tpg = m->tpg;
    std::vector<uint32_t> first(G + 1), chunk(G);
    std::vector<uint16_t> tm(N), asg(G);
    uint64_t row = 0, off = 0;
    for (uint64_t g = 0; g < G; ++g) {
        const uint64_t fr = g4[4 * g], size = g4[4 * g + 1], offset = g4[4 * g + 2], ch = g4[4 * g + 3];
        const std::string at = " (group " + std::to_string(g) + ")";
        if (fr != row || size == 0 || size > tpg || size > N - row)
            fail(ARGCSR_E_FORMAT, "argcsr import: groups must tile the rows in order" + at);
        if (offset != off) fail(ARGCSR_E_FORMAT, "argcsr import: offset is not threads_per_group * sum(chunk)" + at);
        if (ch > 0xFFFFFFFFull || (ch && tpg > (S - off) / ch))
            fail(ARGCSR_E_FORMAT, "argcsr import: chunk_size exceeds the value array" + at);
        uint64_t prev = 0;
        for (uint64_t r = fr; r < fr + size; ++r) {
            if (tm64[r] <= prev || tm64[r] > tpg)
                fail(ARGCSR_E_FORMAT, "argcsr import: threads_mapping must increase within a group and stay <= "
                                      "threads_per_group" + at);
            prev = tm64[r];
            tm[r] = uint16_t(prev);
        }
        first[g] = uint32_t(fr);
        chunk[g] = uint32_t(ch);
        asg[g] = uint16_t(prev);
        row += size;
        off += ch * tpg;
    }
    if (row != N) fail(ARGCSR_E_FORMAT, "argcsr import: groups cover " + std::to_string(row) + " of " +
                                            std::to_string(N) + " rows");
    if (off != S) fail(ARGCSR_E_FORMAT, "argcsr import: value/column arrays hold " + std::to_string(S) +
                                            " slots, the groups " + std::to_string(off));
    first[G] = uint32_t(N);
    m->num_groups = G;
    DevPtr<uint32_t> d_first(G + 1, s), d_chunk(G, s);
    DevPtr<int32_t> d_cols(S, s);
    DevPtr<T> d_vals(S, s);
    uint16_t* d_tm = dev_alloc<uint16_t>(m, N);
    uint16_t* d_asg = dev_alloc<uint16_t>(m, G);
    m->tm = d_tm;
    m->assigned = d_asg;
    CUDA_OK(cudaMemcpyAsync(d_first.p, first.data(), (G + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaMemcpyAsync(d_chunk.p, chunk.data(), G * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaMemcpyAsync(d_tm, tm.data(), N * sizeof(uint16_t), cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaMemcpyAsync(d_asg, asg.data(), G * sizeof(uint16_t), cudaMemcpyHostToDevice, s));
    if (S) {
        CUDA_OK(cudaMemcpyAsync(d_cols.p, cols, S * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(d_vals.p, vals, S * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    LayoutSource<T> src;
    src.ref_cols = d_cols.p;
    src.ref_vals = d_vals.p;
    src.ref_slots = S;
    layout_and_schedule<T, uint16_t>(m, uint32_t(G), d_first.p, d_chunk.p, d_tm, d_asg, src, s);
}

}  // namespace

void import_reference(argcsr_dev* m, uint64_t G, const uint64_t* groups4, const uint64_t* tm, const void* vals,
                      const int32_t* cols, uint64_t S, cudaStream_t s) {
    if (m->dtype == ARGCSR_F64) import_typed<double>(m, G, groups4, tm, static_cast<const double*>(vals), cols, S, s);
    else import_typed<float>(m, G, groups4, tm, static_cast<const float*>(vals), cols, S, s);
}

// threads_mapping and per-group assigned counts are u16 on the device
// (threads_per_group <= kMaxThreadsPerGroup < 65536); export widens to u64.
void convert_device_csr(argcsr_dev* m, const uint64_t* rp, const int32_t* cols, const void* vals, cudaStream_t s) {
    if (m->dtype == ARGCSR_F64) convert_typed<double, uint16_t>(m, rp, cols, static_cast<const double*>(vals), s);
    else convert_typed<float, uint16_t>(m, rp, cols, static_cast<const float*>(vals), s);
}

}  // namespace argcsr_gpu
