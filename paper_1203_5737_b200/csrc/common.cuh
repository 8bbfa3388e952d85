// Internal definitions shared by the converter (convert.cu), the SpMV
// (spmv.cu) and the C-ABI (capi.cu).  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "argcsr_gpu.h"

namespace argcsr_gpu {

// ----------------------------------------------------------------- errors
// Host code throws Failure; the C-ABI catches it and maps it to a status.
struct Failure : std::runtime_error {
    argcsr_status status;
    Failure(argcsr_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(argcsr_status s, const std::string& msg) { throw Failure(s, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        fail(ARGCSR_E_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    }
    fail(ARGCSR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_OK(expr) ::argcsr_gpu::cuda_check((expr), #expr)
#define LAUNCH_OK(what) ::argcsr_gpu::cuda_check(cudaGetLastError(), what)

// The C-ABI's thread-local error message (argcsr_last_error).
std::string& last_error();

// Runs f and maps any exception to a status + message: nothing throws across
// the C-ABI.
template <typename F>
argcsr_status guarded(F&& f) {
    try {
        f();
        last_error().clear();
        return ARGCSR_OK;
    } catch (const Failure& e) {
        last_error() = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        last_error() = "out of host memory";
        return ARGCSR_E_OOM;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return ARGCSR_E_INTERNAL;
    }
}

// Binds a device for the duration of a call and restores the caller's current
// device afterwards.
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            fail(ARGCSR_E_CUDA, "no CUDA device available (the ARG-CSR path has no CPU fallback)");
        }
        if (dev < 0 || dev >= n) fail(ARGCSR_E_PARAMETER, "device ordinal " + std::to_string(dev) + " out of range");
        CUDA_OK(cudaGetDevice(&prev));
        if (prev != dev) CUDA_OK(cudaSetDevice(dev));
    }
    ~DeviceScope() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;
};

// ------------------------------------------------------------ device layout
// Group descriptor, 16 B, one LDG.128.  `off_stride` packs the group's slot
// offset in the STORED value/column arrays (bits 0-47), its lane stride (bits
// 48-62) and the long-chunk ("heavy") flag (bit 63): slot (j, lane) of group g
// lives at offset + j * stride + lane.
// In the reference layout stride = threads_per_group and offset is the
// reference GroupInfo offset (argcsr.hpp:23-30).  In the lane-compact layout
// (the default) stride = assigned lanes rounded up to the
// SpMV vector width: the free lanes of a group, which the reference fills with
// (0.0, -1) and never contribute, are not stored, so the matrix streams
// contiguously; export re-expands to the reference arrays.  size is
// first_row[g+1] - first_row[g] (the array carries a sentinel entry G with
// first_row = num_rows, offset = stored slots).
constexpr uint64_t kOffsetMask = (uint64_t(1) << 48) - 1;
constexpr uint64_t kHeavyBit = uint64_t(1) << 63;
struct alignas(16) GroupDesc {
    uint64_t off_stride;
    uint32_t first_row;
    uint32_t chunk;
    __host__ __device__ __forceinline__ uint64_t offset() const { return off_stride & kOffsetMask; }
    __host__ __device__ __forceinline__ uint32_t stride() const { return uint32_t(off_stride >> 48) & 0x7FFFu; }
    __host__ __device__ __forceinline__ bool heavy() const { return (off_stride & kHeavyBit) != 0; }
};


static_assert(sizeof(GroupDesc) == 16, "GroupDesc must be 16 bytes");

enum Layout : int { kLayoutCompact = 0, kLayoutReference = 1 };
enum XRemapMode : int { kXRemapAuto = 0, kXRemapOn = 1, kXRemapOff = 2 };

// Device limits (documented in DESIGN.md).  threads_per_group bounds the
// shared-memory partial-sum staging of the SpMV; rows are u32 on the device.
constexpr uint64_t kMaxThreadsPerGroup = 16384;
// Groups with chunk_size above this run on the long-chunk (heavy) path.
constexpr uint32_t kHeavyChunk = 32;
// Threads per SpMV CTA, and the default number of units (V-lane vectors) per
// light tile: a tile is walked by one CTA, two units per thread (measured best
// on the stencil and power-law configs, profiles/ and DESIGN.md §4).
// Peers a multi-GPU SpMV epilogue stores into (8 GPUs per box).
constexpr uint32_t kMaxPeers = 7;
constexpr int kTileThreads = 256;
constexpr int kDefaultTileUnits = 512;

// Experiment switches, read from the environment ONCE per process (first
// use) -- never on a launch path.  Defaults are the measured-best settings
// (DESIGN.md §4); -1 means "library decides".
struct Knobs {
    bool l2_window = true;        // ARGCSR_L2_WINDOW=0: no persisting access-policy window for x
    bool l2_persist = true;       // ARGCSR_L2_PERSIST=0: do not raise the device's persisting-L2 limit
    int x_evict_last = -1;        // ARGCSR_XPOL: x gathers L2 evict_last (1) / evict_normal (0) (-1: library decides)
    int stream_evict_first = 0;   // ARGCSR_SPOL: values/columns L2 evict_first (1) / evict_normal (0)
    int map = -1;                 // ARGCSR_MAP: unit/row -> group maps in shared memory (1/0)
    int pair = 1;                 // ARGCSR_PAIR=0: never the paired-unit light kernel
    int light_dyn = -1;           // ARGCSR_LIGHT_DYN: warp-granular dynamic light units (1/0)
    uint32_t heavy_chunk = 0;     // ARGCSR_HEAVY_CHUNK: light/heavy chunk boundary (0 = kHeavyChunk)
    char heavy_pipe = 0;          // ARGCSR_HEAVY_PIPE: '1' pipelined / '0' plain lane walk (default: fp32 pipelined)
    char aux_prio = 'h';          // ARGCSR_AUX_PRIO: heavy stream priority h(ighest) | l(owest) | d(efault)
    bool async_split = true;      // ARGCSR_ASYNC_SPLIT=0: one copy stream per direction
    int tile_threads = 0;         // ARGCSR_TILE_THREADS: light-tile size in units (multiple of 32; 0 = 512, 2048 power-law)
    int l2pf = -1;                // ARGCSR_L2PF: light-tile L2 prefetch off (0) / on (1) / on up to N KB per tile (N > 1)
    char l2pf_what = 0;           // ARGCSR_L2PF_WHAT: prefetch b(oth) / c(olumns) / v(alues) of a tile (0: library decides)
    int ulen = -1;                // ARGCSR_ULEN: per-unit lengths (1/0)
    int vec = 0;                  // ARGCSR_VEC: cap the light unit width V (1 | 2; 0 = library decides)
    int carveout = -1;            // ARGCSR_CARVEOUT: preferred shared-memory carve-out in percent (-1: driver)
    bool trace = false;           // ARGCSR_TRACE=1: per-phase host timings of the converter on stderr
};
const Knobs& knobs();
void reload_knobs();  // argcsr_reload_options (tests flip switches between cases)

// NVTX range (visible in Nsight Systems / ncu --nvtx; free when no tool is
// attached) plus, with ARGCSR_TRACE=1 and sync_timer, a synchronising
// wall-clock timer of the phase on stderr (conversion phases only: never on
// the SpMV path).
struct Phase {
    const char* name;
    cudaStream_t s;
    bool timed;
    std::chrono::steady_clock::time_point t0;
    Phase(const char* n, cudaStream_t st, bool sync_timer = false)
        : name(n), s(st), timed(sync_timer && knobs().trace) {
        nvtxRangePushA(n);
        if (timed) {
            cudaStreamSynchronize(s);
            t0 = std::chrono::steady_clock::now();
        }
    }
    ~Phase() {
        if (timed) {
            cudaStreamSynchronize(s);
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            std::fprintf(stderr, "[argcsr trace] %-28s %9.3f ms\n", name, ms);
        }
        nvtxRangePop();
    }
    Phase(const Phase&) = delete;
    Phase& operator=(const Phase&) = delete;
};

// Consecutive phases of one routine: next() closes the open phase and opens
// the following one; end() (or scope exit) closes the last.
struct PhaseSeq {
    cudaStream_t s;
    alignas(Phase) unsigned char buf[sizeof(Phase)];
    bool open = false;
    explicit PhaseSeq(cudaStream_t st) : s(st) {}
    void end() {
        if (open) reinterpret_cast<Phase*>(buf)->~Phase();
        open = false;
    }
    void next(const char* n) {
        end();
        new (buf) Phase(n, s, true);
        open = true;
    }
    ~PhaseSeq() { end(); }
    PhaseSeq(const PhaseSeq&) = delete;
    PhaseSeq& operator=(const PhaseSeq&) = delete;
};

}  // namespace argcsr_gpu

// Opaque handle behind argcsr_dev* (immutable after conversion).
struct argcsr_dev {
    int device = 0;
    argcsr_dtype dtype = ARGCSR_F64;
    uint64_t num_rows = 0, num_cols = 0, nnz = 0, tpg = 0, dcs = 0;
    uint64_t num_groups = 0, total_slots = 0, max_chunk = 0;
    uint32_t max_light_chunk = 0;         // largest chunk_size among the short-chunk (light) groups
    uint32_t heavy_chunk = 32;            // groups with chunk_size above this are heavy
    bool powerlaw_schedule = false;       // one lane per unit, 2048-unit light tiles (convert.cu)
    int layout = argcsr_gpu::kLayoutCompact;
    uint64_t stored_slots = 0;            // length of values/columns (== total_slots in the reference layout)
    bool tm16 = true;  // threads_mapping / assigned stored as u16 (tpg <= 65535)

    void* values = nullptr;               // [stored_slots] f64 | f32
    int32_t* columns = nullptr;           // [stored_slots]
    argcsr_gpu::GroupDesc* groups = nullptr;  // [num_groups + 1]
    void* tm = nullptr;                   // [num_rows]   u16 | u32
    void* assigned = nullptr;             // [num_groups] u16 | u32

    // SpMV schedule (built by the converter).
    int lanes_per_unit = 1;               // V: 4 | 2 | 1 (tpg % V == 0)
    uint64_t* unit_base = nullptr;        // [num_groups + 1] exclusive scan of light units
    uint32_t* tiles = nullptr;            // [num_tiles + 1] first group of each light tile
    uint64_t* tile_rng = nullptr;         // [2 * num_tiles] stored slot range of each light tile (L2 prefetch)
    uint32_t* heavy = nullptr;            // [num_heavy] heavy groups, chunk descending (LPT)
    uint32_t* heavy_ptr = nullptr;        // [heavy_ctas + 1] packing of `heavy` into CTAs
    uint32_t num_tiles = 0, num_heavy = 0, heavy_ctas = 0;
    uint64_t heavy_max_lanes = 0;         // lanes of the fullest heavy CTA
    uint32_t max_tile_groups = 0;         // bound used for shared-memory sizing
    uint32_t max_tile_rows = 0;
    uint64_t total_units = 0;             // light units (+1 per heavy group) of the schedule
    uint8_t* ulen = nullptr;              // [total_units] light unit lengths (steps with an entry), or null
    uint64_t unit_len_saved = 0;          // stream bytes per SpMV the lengths save (measured at conversion)
    // pipelined host path (argcsr_dev_spmv_host_staged): per light tile, the
    // largest stored column used by tiles 0..t (running max) and its first row
    std::vector<uint32_t> tile_cmax, tile_row;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_x[8] = {}, ev_c[8] = {};
    // asynchronous host SpMV (argcsr_dev_spmv_host_async): handle-owned
    // double-buffered device staging; slot b's events order buffer reuse
    void* as_x[2] = {}, *as_y[2] = {};
    cudaEvent_t as_up[2] = {}, as_mv[2] = {}, as_down[2] = {};
    bool as_used[2] = {};
    cudaStream_t as_h2d2 = nullptr, as_d2h2 = nullptr;  // second copy streams (split copies)
    cudaEvent_t as_j1[2] = {}, as_j2[2] = {};
    uint64_t as_calls = 0;           // rows of the largest light tile (heavy groups' rows included)
    uint64_t tile_span = 0;               // units between consecutive tile keys
    uint32_t tile_threads = 256;          // tiles were built for this CTA size
    uint64_t max_tile_units = 0;          // tile_span + ceil(tpg / V) - 1

    // Heavy groups run on an auxiliary stream forked from the caller's stream.
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // One SpMV in flight per handle: the x' buffer, the auxiliary stream and
    // the fork/join events are handle state, so every SpMV entry point waits
    // for the previous SpMV on this handle (whatever stream it ran on) and
    // records ev_done after its own (capi.cu SpmvSerial).
    std::mutex mu;
    cudaEvent_t ev_done = nullptr;
    bool spmv_issued = false;
    bool holds_l2_persist = false;        // counted in the device's persisting-L2 users (capi.cu)
    double* norm_scratch = nullptr;       // per-CTA ||y||^2 partials (argcsr_dev_spmv_norm2), lazily allocated
    double* scale_buf = nullptr;          // [1] 1/||y_prev|| of a scale_is_norm2 SpMV (spmv.cu)

    uint64_t light_slots = 0;             // stored slots of light groups (stored first)

    // x remap (xremap.cu): stored columns index x' = x[perm[0 .. n_used)].
    int xremap_mode = argcsr_gpu::kXRemapAuto;
    bool x_remap = false;
    uint32_t* perm = nullptr;             // [num_cols] stored column -> reference column
    void* xbuf = nullptr;                 // [n_used] x' (one SpMV in flight per handle)
    uint64_t n_used = 0;                  // columns with at least one entry (remap on) or num_cols
    double x_cover_lead = 0, x_cover_top = 0;  // nnz share of the window: leading columns / remapped
    double run_pairs_orig = 0, run_pairs_remap = 0;  // long rows: share of consecutive column pairs

    // x residency (L2 persisting window) — queried, not hard-coded.
    size_t l2_persist_max = 0;
    int l2_window_max = 0;

    size_t device_bytes = 0;
};
