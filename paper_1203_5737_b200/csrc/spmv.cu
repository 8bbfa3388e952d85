// ARG-CSR SpMV for sm_100a (replaces spmv_argcsr_groups, proj/src/argcsr.cpp:185-217).
//
// One launch, two CTA roles:
//   * heavy CTAs (blockIdx < num_heavy): one long-chunk group each, in LPT
//     order (largest chunk first), one lane per thread with a deep unroll so a
//     1-3 MB group streams at full per-SM bandwidth;
//   * light tiles: a run of consecutive short-chunk groups whose ASSIGNED lanes
//     (free lanes are never read) are flattened into V-lane units, one unit per
//     thread.  A unit's V adjacent lanes are one 128-bit column load and
//     V*8 bytes of values per element step, so every warp access is a
//     contiguous, coalesced segment of a group's j-row.
// Group metadata of a tile is staged in shared memory; per-chunk partial sums
// go to shared memory and each row sums its chunk range in ascending order
// from +0.0.  Products and sums use __dmul_rn/__dadd_rn in the reference's
// order (phase 1: per lane, j ascending; phase 2: per row, chunks ascending),
// so fp64 results are bit-identical to the reference's CPU product (which has
// no FMA).  fp32 handles load fp32 values/x, multiply exactly in fp64 and round
// the row sum once.
//
// Streams: values/columns are read once per SpMV with evict-first loads
// (__ldcs -> LDG.E.EF); x is gathered through the read-only path and kept L2
// resident with an access-policy window sized from the device's persisting-L2
// limit.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "spmv.cuh"

namespace argcsr_gpu {

namespace {

template <typename T, typename TM>
struct SpmvArgs {
    const T* __restrict__ vals;
    const int32_t* __restrict__ cols;
    const GroupDesc* __restrict__ groups;
    const TM* __restrict__ tm;
    const TM* __restrict__ assigned;
    const uint64_t* __restrict__ unit_base;
    const uint32_t* __restrict__ tiles;
    const uint32_t* __restrict__ heavy;
    const T* __restrict__ x;
    T* __restrict__ y;
    uint64_t tpg;
    uint32_t num_heavy;
    uint32_t g_begin, g_end;  // rows of groups outside [g_begin, g_end) are not written
    uint32_t max_tile_groups;
};

// ----------------------------------------------------------------- loads
template <int V> struct IVec;
template <> struct IVec<1> { using type = int; };
template <> struct IVec<2> { using type = int2; };
template <> struct IVec<4> { using type = int4; };

template <int V>
__device__ __forceinline__ void load_cols(const int32_t* p, int (&c)[V]) {
    if constexpr (V == 4) {
        const int4 v = __ldcs(reinterpret_cast<const int4*>(p));
        c[0] = v.x, c[1] = v.y, c[2] = v.z, c[3] = v.w;
    } else if constexpr (V == 2) {
        const int2 v = __ldcs(reinterpret_cast<const int2*>(p));
        c[0] = v.x, c[1] = v.y;
    } else {
        c[0] = __ldcs(p);
    }
}

// Values of a unit, loaded only for 16-byte pieces holding a non-sentinel lane.
template <int V>
__device__ __forceinline__ void load_vals(const double* p, const int (&c)[V], double (&v)[V]) {
    if constexpr (V == 1) {
        v[0] = c[0] != -1 ? __ldcs(p) : 0.0;
    } else {
#pragma unroll
        for (int h = 0; h < V; h += 2) {
            if ((c[h] & c[h + 1]) != -1) {
                const double2 d = __ldcs(reinterpret_cast<const double2*>(p + h));
                v[h] = d.x, v[h + 1] = d.y;
            } else {
                v[h] = 0.0, v[h + 1] = 0.0;
            }
        }
    }
}
template <int V>
__device__ __forceinline__ void load_vals(const float* p, const int (&c)[V], float (&v)[V]) {
    if constexpr (V == 4) {
        if ((c[0] & c[1] & c[2] & c[3]) != -1) {
            const float4 d = __ldcs(reinterpret_cast<const float4*>(p));
            v[0] = d.x, v[1] = d.y, v[2] = d.z, v[3] = d.w;
        } else {
            v[0] = v[1] = v[2] = v[3] = 0.f;
        }
    } else if constexpr (V == 2) {
        if ((c[0] & c[1]) != -1) {
            const float2 d = __ldcs(reinterpret_cast<const float2*>(p));
            v[0] = d.x, v[1] = d.y;
        } else {
            v[0] = v[1] = 0.f;
        }
    } else {
        v[0] = c[0] != -1 ? __ldcs(p) : 0.f;
    }
}

__device__ __forceinline__ double load_x(const double* x, int c) { return c != -1 ? __ldg(x + c) : 0.0; }
__device__ __forceinline__ double load_x(const float* x, int c) { return c != -1 ? double(__ldg(x + c)) : 0.0; }

// Phase 1 (argcsr.cpp:193-203) for V adjacent lanes starting at slot0: per
// lane, sum += v * x[c] over j ascending until the first sentinel.  Columns
// of U element steps are in flight together; the layout keeps sentinels
// trailing, so "skip sentinel" == "stop at the first sentinel".
template <typename T, int V, int U>
__device__ __forceinline__ void phase1(const T* __restrict__ vals, const int32_t* __restrict__ cols,
                                       const T* __restrict__ x, uint64_t slot0, uint32_t chunk, uint64_t tpg,
                                       double (&s)[V]) {
#pragma unroll
    for (int l = 0; l < V; ++l) s[l] = 0.0;
    const int32_t* cp = cols + slot0;
    const T* vp = vals + slot0;
    for (uint32_t j0 = 0; j0 < chunk; j0 += U) {
        int c[U][V];
        T v[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (j0 + u < chunk) {
                load_cols<V>(cp + uint64_t(j0 + u) * tpg, c[u]);
            } else {
#pragma unroll
                for (int l = 0; l < V; ++l) c[u][l] = -1;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) load_vals<V>(vp + uint64_t(j0 + u) * tpg, c[u], v[u]);
        double xv[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int l = 0; l < V; ++l) xv[u][l] = load_x(x, c[u][l]);
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

// Phase 2 (argcsr.cpp:206-215): y[row] = +0.0 + p_b + p_{b+1} + ... ascending.
template <typename T, typename TM>
__device__ __forceinline__ void reduce_row(const SpmvArgs<T, TM>& a, const double* part, uint32_t row,
                                           bool first_of_group) {
    const uint32_t b = first_of_group ? 0u : uint32_t(a.tm[row - 1]);
    const uint32_t e = uint32_t(a.tm[row]);
    double sum = 0.0;
    for (uint32_t t = b; t < e; ++t) sum = __dadd_rn(sum, part[t]);
    a.y[row] = to_out<T>(sum);
}

constexpr int kUnrollLight = 2;
constexpr int kUnrollHeavy = 8;

template <typename T, typename TM, int V>
__global__ void __launch_bounds__(kTileThreads) spmv_kernel(const SpmvArgs<T, TM> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_part = reinterpret_cast<double*>(smem);

    if (blockIdx.x < a.num_heavy) {
        // ---------------------------------------------------- heavy group
        const uint32_t g = a.heavy[blockIdx.x];
        if (g < a.g_begin || g >= a.g_end) return;
        const GroupDesc d = a.groups[g];
        const uint32_t f = d.first_row, k = a.groups[g + 1].first_row - f;
        const uint32_t asg = uint32_t(a.assigned[g]);
        for (uint32_t l = threadIdx.x; l < asg; l += blockDim.x) {
            double s[1];
            phase1<T, 1, kUnrollHeavy>(a.vals, a.cols, a.x, d.offset + l, d.chunk, a.tpg, s);
            s_part[l] = s[0];
        }
        __syncthreads();
        for (uint32_t r = threadIdx.x; r < k; r += blockDim.x) reduce_row(a, s_part, f + r, r == 0);
        return;
    }

    // -------------------------------------------------------- light tile
    const uint32_t kt = blockIdx.x - a.num_heavy;
    const uint32_t gs = a.tiles[kt], ge = a.tiles[kt + 1];
    if (ge <= a.g_begin || gs >= a.g_end || gs == ge) return;
    const uint32_t ng = ge - gs;
    const uint32_t cap = a.max_tile_groups;
    // smem: s_part[(max units) * V] | s_off[cap] | s_ub[cap+1] | s_first[cap+1] | s_chunk[cap]
    const size_t part_words = size_t(kTileThreads + (a.tpg + V - 1) / V) * V;
    uint64_t* s_off = reinterpret_cast<uint64_t*>(s_part + part_words);
    uint32_t* s_ub = reinterpret_cast<uint32_t*>(s_off + cap);
    uint32_t* s_first = s_ub + cap + 1;
    uint32_t* s_chunk = s_first + cap + 1;

    const uint64_t ub0 = a.unit_base[gs];
    for (uint32_t i = threadIdx.x; i <= ng; i += blockDim.x) {
        const GroupDesc d = a.groups[gs + i];
        s_first[i] = d.first_row;
        s_ub[i] = uint32_t(a.unit_base[gs + i] - ub0);
        if (i < ng) {
            s_off[i] = d.offset;
            s_chunk[i] = d.chunk;
        }
    }
    __syncthreads();

    const uint32_t nunits = s_ub[ng];
    for (uint32_t u = threadIdx.x; u < nunits; u += blockDim.x) {
        uint32_t lo = 0, hi = ng - 1;  // last group with s_ub <= u
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) / 2;
            if (s_ub[mid] <= u) lo = mid; else hi = mid - 1;
        }
        const uint32_t gi = lo;
        const uint32_t g = gs + gi;
        if (s_chunk[gi] > kHeavyChunk || g < a.g_begin || g >= a.g_end) continue;
        const uint32_t lane0 = (u - s_ub[gi]) * V;
        double s[V];
        phase1<T, V, kUnrollLight>(a.vals, a.cols, a.x, s_off[gi] + lane0, s_chunk[gi], a.tpg, s);
#pragma unroll
        for (int l = 0; l < V; ++l) s_part[size_t(u) * V + l] = s[l];
    }
    __syncthreads();

    const uint32_t row0 = s_first[0], row_end = s_first[ng];
    for (uint32_t r = row0 + threadIdx.x; r < row_end; r += blockDim.x) {
        uint32_t lo = 0, hi = ng - 1;  // last group with s_first <= r
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) / 2;
            if (s_first[mid] <= r) lo = mid; else hi = mid - 1;
        }
        const uint32_t gi = lo;
        const uint32_t g = gs + gi;
        if (s_chunk[gi] > kHeavyChunk || g < a.g_begin || g >= a.g_end) continue;
        reduce_row(a, s_part + size_t(s_ub[gi]) * V, r, r == s_first[gi]);
    }
}

size_t light_smem_bytes(const argcsr_dev* m, int V) {
    const size_t cap = std::max<uint32_t>(m->max_tile_groups, 1);
    const size_t part = size_t(kTileThreads + (m->tpg + V - 1) / V) * V * sizeof(double);
    return part + cap * sizeof(uint64_t) + (cap + 1) * 4 * 2 + cap * 4;
}

bool l2_window_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ARGCSR_L2_WINDOW");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename T, typename TM, int V>
void launch_typed(const argcsr_dev* m, const void* x, void* y, uint32_t gb, uint32_t ge, cudaStream_t s) {
    SpmvArgs<T, TM> a;
    a.vals = static_cast<const T*>(m->values);
    a.cols = m->columns;
    a.groups = m->groups;
    a.tm = static_cast<const TM*>(m->tm);
    a.assigned = static_cast<const TM*>(m->assigned);
    a.unit_base = m->unit_base;
    a.tiles = m->tiles;
    a.heavy = m->heavy;
    a.x = static_cast<const T*>(x);
    a.y = static_cast<T*>(y);
    a.tpg = m->tpg;
    a.num_heavy = m->num_heavy;
    a.g_begin = gb;
    a.g_end = ge;
    a.max_tile_groups = std::max<uint32_t>(m->max_tile_groups, 1);

    const size_t smem = std::max(light_smem_bytes(m, V), size_t(m->tpg) * sizeof(double));
    auto kern = spmv_kernel<T, TM, V>;
    if (smem > 48 * 1024) CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const unsigned grid = m->num_heavy + m->num_tiles;
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
        int max_win = 0;
        CUDA_OK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, m->device));
        const size_t win = std::min<size_t>(xbytes, size_t(max_win));
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(x);
        attr[0].val.accessPolicyWindow.num_bytes = win;
        attr[0].val.accessPolicyWindow.hitRatio =
            float(std::min(1.0, double(m->l2_persist_max) / double(win)));
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    CUDA_OK(cudaLaunchKernelEx(&cfg, kern, a));
}

template <typename T>
void launch_dtype(const argcsr_dev* m, const void* x, void* y, uint32_t gb, uint32_t ge, cudaStream_t s) {
    switch (m->lanes_per_unit) {
        case 4: launch_typed<T, uint16_t, 4>(m, x, y, gb, ge, s); break;
        case 2: launch_typed<T, uint16_t, 2>(m, x, y, gb, ge, s); break;
        default: launch_typed<T, uint16_t, 1>(m, x, y, gb, ge, s); break;
    }
}

}  // namespace

void spmv_launch(const argcsr_dev* m, const void* x, void* y, uint64_t group_begin, uint64_t group_end,
                 cudaStream_t s) {
    const uint32_t gb = uint32_t(std::min<uint64_t>(group_begin, m->num_groups));
    const uint32_t ge = uint32_t(std::min<uint64_t>(group_end, m->num_groups));
    if (gb >= ge) return;
    if (m->dtype == ARGCSR_F64) launch_dtype<double>(m, x, y, gb, ge, s);
    else launch_dtype<float>(m, x, y, gb, ge, s);
}

}  // namespace argcsr_gpu
