// Internal definitions shared by the converter (convert.cu), the SpMV
// (spmv.cu) and the C-ABI (capi.cu).  sm_100a only.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

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

// ------------------------------------------------------------ device layout
// Group descriptor, 16 B, one LDG.128.  offset is the reference GroupInfo
// offset (argcsr.hpp:23-30); size is first_row[g+1] - first_row[g] (the
// array carries a sentinel entry G with first_row = num_rows, offset =
// total_slots).
struct alignas(16) GroupDesc {
    uint64_t offset;
    uint32_t first_row;
    uint32_t chunk;
};
static_assert(sizeof(GroupDesc) == 16, "GroupDesc must be 16 bytes");

// Device limits (documented in DESIGN.md).  threads_per_group bounds the
// shared-memory partial-sum staging of the SpMV; rows are u32 on the device.
constexpr uint64_t kMaxThreadsPerGroup = 16384;
// Groups with chunk_size above this run on the long-chunk (heavy) path.
constexpr uint32_t kHeavyChunk = 32;
// Units (V-lane quads) per light tile = threads per SpMV CTA.
constexpr int kTileThreads = 256;

}  // namespace argcsr_gpu

// Opaque handle behind argcsr_dev* (immutable after conversion).
struct argcsr_dev {
    int device = 0;
    argcsr_dtype dtype = ARGCSR_F64;
    uint64_t num_rows = 0, num_cols = 0, nnz = 0, tpg = 0, dcs = 0;
    uint64_t num_groups = 0, total_slots = 0, max_chunk = 0;
    bool tm16 = true;  // threads_mapping / assigned stored as u16 (tpg <= 65535)

    void* values = nullptr;               // [total_slots] f64 | f32
    int32_t* columns = nullptr;           // [total_slots]
    argcsr_gpu::GroupDesc* groups = nullptr;  // [num_groups + 1]
    void* tm = nullptr;                   // [num_rows]   u16 | u32
    void* assigned = nullptr;             // [num_groups] u16 | u32

    // SpMV schedule (built by the converter).
    int lanes_per_unit = 1;               // V: 4 | 2 | 1 (tpg % V == 0)
    uint64_t* unit_base = nullptr;        // [num_groups + 1] exclusive scan of light units
    uint32_t* tiles = nullptr;            // [num_tiles + 1] first group of each light tile
    uint32_t* heavy = nullptr;            // [num_heavy] heavy groups, chunk descending (LPT)
    uint32_t* heavy_ptr = nullptr;        // [heavy_ctas + 1] packing of `heavy` into CTAs
    uint32_t num_tiles = 0, num_heavy = 0, heavy_ctas = 0;
    uint64_t heavy_max_lanes = 0;         // lanes of the fullest heavy CTA
    uint32_t max_tile_groups = 0;         // bound used for shared-memory sizing
    uint64_t tile_span = 0;               // units between consecutive tile keys
    uint32_t tile_threads = 256;          // tiles were built for this CTA size
    uint64_t max_tile_units = 0;          // tile_span + ceil(tpg / V) - 1

    // Heavy groups run on an auxiliary stream forked from the caller's stream.
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    uint32_t* sched = nullptr;            // [2] dynamic tile counter + done counter (self-resetting)

    // x residency (L2 persisting window) — queried, not hard-coded.
    size_t l2_persist_max = 0;
    int l2_window_max = 0;

    size_t device_bytes = 0;
};
