// The C-ABI (include/argcsr_gpu.h).  Validation order and messages follow the
// reference (proj/src/argcsr.cpp:20-26, 220-223, 235-242); every failure is a
// status code plus a thread-local message, never an exception across the ABI.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "argcsr_gpu.h"
#include "common.cuh"
#include "convert.cuh"
#include "ellpack.cuh"
#include "inverse.cuh"
#include "spmv.cuh"

using argcsr_gpu::DeviceScope;
using argcsr_gpu::fail;
using argcsr_gpu::Failure;
using argcsr_gpu::guarded;

namespace argcsr_gpu {
std::string& last_error() {
    thread_local std::string msg;
    return msg;
}

namespace {
Knobs read_knobs() {
    Knobs v;
    auto flag = [](const char* n, int d) {
        const char* e = std::getenv(n);
        return e && e[0] ? (e[0] == '1' ? 1 : e[0] == '0' ? 0 : d) : d;
    };
    auto chr = [](const char* n, char d) {
        const char* e = std::getenv(n);
        return e && e[0] ? e[0] : d;
    };
    v.l2_window = flag("ARGCSR_L2_WINDOW", 1) != 0;
    v.l2_persist = flag("ARGCSR_L2_PERSIST", 1) != 0;
    v.x_evict_last = flag("ARGCSR_XPOL", -1);
    v.stream_evict_first = flag("ARGCSR_SPOL", 0);
    v.map = flag("ARGCSR_MAP", -1);
    v.pair = flag("ARGCSR_PAIR", 1);
    v.light_dyn = flag("ARGCSR_LIGHT_DYN", -1);
    v.heavy_pipe = chr("ARGCSR_HEAVY_PIPE", 0);
    if (const char* e = std::getenv("ARGCSR_HEAVY_CHUNK")) v.heavy_chunk = uint32_t(std::min(250, std::max(0, std::atoi(e))));
    v.aux_prio = chr("ARGCSR_AUX_PRIO", 'h');
    v.async_split = flag("ARGCSR_ASYNC_SPLIT", 1) != 0;
    if (const char* e = std::getenv("ARGCSR_TILE_THREADS")) v.tile_threads = std::atoi(e);
    v.ulen = flag("ARGCSR_ULEN", -1);
    v.l2pf_what = chr("ARGCSR_L2PF_WHAT", 0);
    if (const char* e = std::getenv("ARGCSR_L2PF")) v.l2pf = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("ARGCSR_CARVEOUT")) v.carveout = std::atoi(e);
    if (const char* e = std::getenv("ARGCSR_VEC")) v.vec = std::atoi(e);
    v.trace = flag("ARGCSR_TRACE", 0) == 1;
    return v;
}
std::mutex g_knob_mu;
std::atomic<bool> g_knobs_loaded{false};
Knobs g_knobs;
}  // namespace

const Knobs& knobs() {
    if (!g_knobs_loaded.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lock(g_knob_mu);
        if (!g_knobs_loaded.load(std::memory_order_relaxed)) {
            g_knobs = read_knobs();
            g_knobs_loaded.store(true, std::memory_order_release);
        }
    }
    return g_knobs;
}

void reload_knobs() {
    std::lock_guard<std::mutex> lock(g_knob_mu);
    g_knobs = read_knobs();
    g_knobs_loaded.store(true, std::memory_order_release);
}
}  // namespace argcsr_gpu

namespace {

void release_l2_persist(int device);

void free_handle(argcsr_dev* m) {
    if (!m) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    cudaFree(m->values);
    cudaFree(m->columns);
    cudaFree(m->groups);
    cudaFree(m->tm);
    cudaFree(m->assigned);
    cudaFree(m->unit_base);
    cudaFree(m->tiles);
    cudaFree(m->tile_rng);
    cudaFree(m->ulen);
    cudaFree(m->heavy);
    cudaFree(m->heavy_ptr);
    cudaFree(m->perm);
    cudaFree(m->xbuf);
    if (m->aux) cudaStreamDestroy(m->aux);
    if (m->as_h2d2) cudaStreamDestroy(m->as_h2d2);
    if (m->as_d2h2) cudaStreamDestroy(m->as_d2h2);
    for (int b = 0; b < 2; ++b) {
        if (m->as_j1[b]) cudaEventDestroy(m->as_j1[b]);
        if (m->as_j2[b]) cudaEventDestroy(m->as_j2[b]);
        if (m->as_x[b]) cudaFree(m->as_x[b]);
        if (m->as_y[b]) cudaFree(m->as_y[b]);
        if (m->as_up[b]) cudaEventDestroy(m->as_up[b]);
        if (m->as_mv[b]) cudaEventDestroy(m->as_mv[b]);
        if (m->as_down[b]) cudaEventDestroy(m->as_down[b]);
    }
    if (m->h2d) cudaStreamDestroy(m->h2d);
    if (m->d2h) cudaStreamDestroy(m->d2h);
    for (int i = 0; i < 8; ++i) {
        if (m->ev_x[i]) cudaEventDestroy(m->ev_x[i]);
        if (m->ev_c[i]) cudaEventDestroy(m->ev_c[i]);
    }
    if (m->ev_fork) cudaEventDestroy(m->ev_fork);
    if (m->ev_join) cudaEventDestroy(m->ev_join);
    if (m->ev_done) cudaEventDestroy(m->ev_done);
    cudaFree(m->norm_scratch);
    cudaFree(m->scale_buf);
    if (m->holds_l2_persist) release_l2_persist(m->device);
    if (prev >= 0) cudaSetDevice(prev);
    delete m;
}

size_t elem_size(argcsr_dtype d) { return d == ARGCSR_F64 ? sizeof(double) : sizeof(float); }

void check_handle(const argcsr_dev* m) {
    if (!m) fail(ARGCSR_E_PARAMETER, "null ARG-CSR handle");
}

// Persisting-L2 carve-out for the x window (SpMV).  Raising the device's
// persisting-L2 limit is a process-wide side effect (persisting lines can keep
// L2 from other kernels of the host application), so it is reference-counted
// per device: the first live handle saves the previous limit and raises it to
// the maximum, the last one to be freed resets the persisting lines
// (cudaCtxResetPersistingL2Cache) and restores the saved limit.
// ARGCSR_L2_PERSIST=0 leaves the limit alone (the window then only uses what
// the application already set aside).  Documented in include/argcsr_gpu.h.
struct L2PersistState {
    int users = 0;
    size_t saved = 0;
    size_t granted = 0;
};
std::mutex g_l2_mu;
L2PersistState g_l2[64];

size_t acquire_l2_persist(int device, bool* counted) {
    *counted = false;
    if (device < 0 || device >= 64) return 0;
    std::lock_guard<std::mutex> lock(g_l2_mu);
    L2PersistState& st = g_l2[device];
    if (!argcsr_gpu::knobs().l2_persist) {
        size_t cur = 0;
        if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) != cudaSuccess) cudaGetLastError();
        return cur;
    }
    if (st.users == 0) {
        int persist_max = 0;
        CUDA_OK(cudaDeviceGetAttribute(&persist_max, cudaDevAttrMaxPersistingL2CacheSize, device));
        st.saved = 0;
        st.granted = 0;
        if (cudaDeviceGetLimit(&st.saved, cudaLimitPersistingL2CacheSize) != cudaSuccess) cudaGetLastError();
        if (persist_max > 0) {
            if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(persist_max)) == cudaSuccess) {
                CUDA_OK(cudaDeviceGetLimit(&st.granted, cudaLimitPersistingL2CacheSize));
            } else {
                cudaGetLastError();
                st.granted = st.saved;
            }
        }
    }
    ++st.users;
    *counted = true;
    return st.granted;
}

void release_l2_persist(int device) {
    std::lock_guard<std::mutex> lock(g_l2_mu);
    L2PersistState& st = g_l2[device];
    if (st.users <= 0 || --st.users > 0) return;
    if (cudaCtxResetPersistingL2Cache() != cudaSuccess) cudaGetLastError();
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, st.saved) != cudaSuccess) cudaGetLastError();
}

using SpmvSerial = argcsr_gpu::SpmvOrder;

// A fresh handle with the per-handle resources (aux stream, events, L2 window
// limits); freed by free_handle on any failure of the caller.
argcsr_dev* new_handle(int device, argcsr_dtype dtype, uint64_t rows, uint64_t cols, uint64_t tpg, uint64_t dcs,
                       uint32_t flags) {
    auto* m = new argcsr_dev;
    m->device = device;
    m->dtype = dtype;
    m->num_rows = rows;
    m->num_cols = cols;
    m->tpg = tpg;
    m->dcs = dcs;
    m->tm16 = true;
    m->layout = (flags & ARGCSR_LAYOUT_REFERENCE) ? argcsr_gpu::kLayoutReference : argcsr_gpu::kLayoutCompact;
    m->xremap_mode = (flags & ARGCSR_XREMAP_ON)    ? argcsr_gpu::kXRemapOn
                     : (flags & ARGCSR_XREMAP_OFF) ? argcsr_gpu::kXRemapOff
                                                   : argcsr_gpu::kXRemapAuto;
    try {
        m->l2_persist_max = acquire_l2_persist(device, &m->holds_l2_persist);
        CUDA_OK(cudaDeviceGetAttribute(&m->l2_window_max, cudaDevAttrMaxAccessPolicyWindowSize, device));
        {
            // The heavy groups' stream runs at the highest priority: whenever an
            // SM slot frees, the block scheduler hands it to a heavy CTA first
            // and the short light tiles fill the gaps, instead of the heavy
            // kernel's last wave trailing alone (C4: 0.64 -> 0.69 of HBM, fp32
            // 0.39 -> 0.51).  Experiments: ARGCSR_AUX_PRIO=lo|def.
            int lo = 0, hi = 0;
            CUDA_OK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            const char ap = argcsr_gpu::knobs().aux_prio;
            const int prio = ap == 'h' ? hi : ap == 'l' ? lo : 0;
            CUDA_OK(cudaStreamCreateWithPriority(&m->aux, cudaStreamNonBlocking, prio));
        }
        CUDA_OK(cudaEventCreateWithFlags(&m->ev_done, cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming));
        CUDA_OK(cudaStreamCreateWithFlags(&m->h2d, cudaStreamNonBlocking));
        CUDA_OK(cudaStreamCreateWithFlags(&m->d2h, cudaStreamNonBlocking));
        for (int i = 0; i < 8; ++i) {
            CUDA_OK(cudaEventCreateWithFlags(&m->ev_x[i], cudaEventDisableTiming));
            CUDA_OK(cudaEventCreateWithFlags(&m->ev_c[i], cudaEventDisableTiming));
        }
    } catch (...) {
        free_handle(m);
        throw;
    }
    return m;
}

void check_flags(uint32_t flags, const char* who) {
    if (flags & ~uint32_t(ARGCSR_LAYOUT_REFERENCE | ARGCSR_XREMAP_ON | ARGCSR_XREMAP_OFF))
        fail(ARGCSR_E_PARAMETER, std::string(who) + ": unknown flags");
    if ((flags & ARGCSR_XREMAP_ON) && (flags & ARGCSR_XREMAP_OFF))
        fail(ARGCSR_E_PARAMETER, std::string(who) + ": ARGCSR_XREMAP_ON and ARGCSR_XREMAP_OFF both set");
}

// ------------------------------------------------------- binary container
// The reference's SPFMTBIN container (proj/src/io.cpp:17-22, 242-246,
// 282-298, 300-366): 8-byte magic, u32 version 1, u8 format tag, then
// little-endian u64 scalars and u64-length-prefixed arrays.
constexpr char kMagic[8] = {'S', 'P', 'F', 'M', 'T', 'B', 'I', 'N'};
constexpr uint32_t kVersion = 1;
constexpr uint8_t kTagCsr = 0, kTagArgCsr = 3;

struct File {
    std::FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

struct Reader {
    std::FILE* f;
    uint64_t left;  // bytes not yet read
    void bytes(void* p, uint64_t n) {
        if (n > left || (n && std::fread(p, 1, n, f) != n)) fail(ARGCSR_E_PARSE, "binary stream truncated");
        left -= n;
    }
    uint8_t u8() {
        uint8_t v;
        bytes(&v, 1);
        return v;
    }
    uint32_t u32() {
        unsigned char b[4];
        bytes(b, 4);
        return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
    }
    uint64_t u64() {
        unsigned char b[8];
        bytes(b, 8);
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= uint64_t(b[i]) << (8 * i);
        return v;
    }
    // u64 length + n elements of `size` bytes; a length beyond the stream is truncation
    template <typename T>
    std::vector<T> array() {
        const uint64_t n = u64();
        if (n > left / sizeof(T)) fail(ARGCSR_E_PARSE, "binary stream truncated");
        std::vector<T> a(n);
        bytes(a.data(), n * sizeof(T));  // little-endian host (x86-64 / aarch64)
        return a;
    }
};

struct Writer {
    std::FILE* f;
    void bytes(const void* p, uint64_t n) {
        if (n && std::fwrite(p, 1, n, f) != n) fail(ARGCSR_E_IO, "binary write failure");
    }
    void u8(uint8_t v) { bytes(&v, 1); }
    void u32(uint32_t v) {
        const unsigned char b[4] = {uint8_t(v), uint8_t(v >> 8), uint8_t(v >> 16), uint8_t(v >> 24)};
        bytes(b, 4);
    }
    void u64(uint64_t v) {
        unsigned char b[8];
        for (int i = 0; i < 8; ++i) b[i] = uint8_t(v >> (8 * i));
        bytes(b, 8);
    }
};

}  // namespace

extern "C" {

const char* argcsr_last_error(void) { return argcsr_gpu::last_error().c_str(); }

void argcsr_reload_options(void) { argcsr_gpu::reload_knobs(); }

int argcsr_abi_version(void) { return ARGCSR_GPU_ABI_VERSION; }

const char* argcsr_status_name(argcsr_status s) {
    switch (s) {
        case ARGCSR_OK: return "ok";
        case ARGCSR_E_PARAMETER: return "ParameterError";
        case ARGCSR_E_DIMENSION: return "DimensionError";
        case ARGCSR_E_BOUNDS: return "BoundsError";
        case ARGCSR_E_INTERNAL: return "InternalError";
        case ARGCSR_E_CUDA: return "CudaError";
        case ARGCSR_E_NCCL: return "NcclError";
        case ARGCSR_E_OOM: return "OutOfMemory";
        case ARGCSR_E_FORMAT: return "FormatError";
        case ARGCSR_E_IO: return "IoError";
        case ARGCSR_E_PARSE: return "ParseError";
        case ARGCSR_E_UNSUPPORTED: return "UnsupportedError";
    }
    return "unknown";
}

argcsr_status argcsr_dev_convert(const argcsr_csr_view* csr, uint64_t tpg, uint64_t dcs, int device,
                                 void* stream, argcsr_dev** out) {
    return argcsr_dev_convert_ex(csr, tpg, dcs, device, stream, 0u, out);
}

argcsr_status argcsr_dev_convert_ex(const argcsr_csr_view* csr, uint64_t tpg, uint64_t dcs, int device,
                                    void* stream, uint32_t flags, argcsr_dev** out) {
    return guarded([&] {
        if (!csr || !out) fail(ARGCSR_E_PARAMETER, "argcsr_dev_convert: null argument");
        *out = nullptr;
        // argcsr.cpp:20-26 order: parameters, then an empty row set.
        if (tpg == 0 || dcs == 0)
            fail(ARGCSR_E_PARAMETER,
                 "partition_groups: threads_per_group and desired_chunk_size must be at least 1");
        if (csr->num_rows == 0) fail(ARGCSR_E_PARAMETER, "partition_groups: row_nnz must be nonempty");
        if (tpg > argcsr_gpu::kMaxThreadsPerGroup)
            fail(ARGCSR_E_UNSUPPORTED, "argcsr_from_csr: threads_per_group " + std::to_string(tpg) +
                                           " exceeds the device limit " +
                                           std::to_string(argcsr_gpu::kMaxThreadsPerGroup));
        if (csr->num_rows >= 0xFFFFFFFFull)
            fail(ARGCSR_E_UNSUPPORTED, "argcsr_from_csr: num_rows exceeds the device limit 2^32-2");
        check_flags(flags, "argcsr_dev_convert_ex");
        if (csr->dtype != ARGCSR_F64 && csr->dtype != ARGCSR_F32)
            fail(ARGCSR_E_PARAMETER, "argcsr_from_csr: unknown dtype");
        if (!csr->row_pointers || (csr->nnz && (!csr->columns || !csr->values)))
            fail(ARGCSR_E_PARAMETER, "argcsr_from_csr: null CSR array");

        DeviceScope scope(device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        argcsr_dev* m = new_handle(device, csr->dtype, csr->num_rows, csr->num_cols, tpg, dcs, flags);
        try {
            const uint64_t N = csr->num_rows, nnz = csr->nnz;
            const size_t es = elem_size(csr->dtype);
            const uint64_t* rp = csr->row_pointers;
            const int32_t* cols = csr->columns;
            const void* vals = csr->values;
            void* staged[3] = {nullptr, nullptr, nullptr};
            struct Release {
                void** p;
                cudaStream_t s;
                ~Release() {
                    for (int i = 0; i < 3; ++i)
                        if (p[i]) cudaFreeAsync(p[i], s);
                }
            } release{staged, s};
            if (csr->space == ARGCSR_HOST) {
                CUDA_OK(cudaMallocAsync(&staged[0], (N + 1) * sizeof(uint64_t), s));
                CUDA_OK(cudaMallocAsync(&staged[1], std::max<uint64_t>(nnz, 1) * sizeof(int32_t), s));
                CUDA_OK(cudaMallocAsync(&staged[2], std::max<uint64_t>(nnz, 1) * es, s));
                CUDA_OK(cudaMemcpyAsync(staged[0], rp, (N + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
                if (nnz) {
                    CUDA_OK(cudaMemcpyAsync(staged[1], cols, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
                    CUDA_OK(cudaMemcpyAsync(staged[2], vals, nnz * es, cudaMemcpyHostToDevice, s));
                }
                rp = static_cast<const uint64_t*>(staged[0]);
                cols = static_cast<const int32_t*>(staged[1]);
                vals = staged[2];
            }
            uint64_t ends[2] = {0, 0};
            CUDA_OK(cudaMemcpyAsync(&ends[0], rp, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaMemcpyAsync(&ends[1], rp + N, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
            argcsr_gpu::convert_device_csr(m, rp, cols, vals, s);
            m->nnz = ends[1] - ends[0];
            CUDA_OK(cudaStreamSynchronize(s));
        } catch (...) {
            free_handle(m);
            throw;
        }
        *out = m;
    });
}

argcsr_status argcsr_dev_info(const argcsr_dev* m, argcsr_dev_info_t* info) {
    return guarded([&] {
        check_handle(m);
        if (!info) fail(ARGCSR_E_PARAMETER, "argcsr_dev_info: null output");
        info->num_rows = m->num_rows;
        info->num_cols = m->num_cols;
        info->threads_per_group = m->tpg;
        info->desired_chunk_size = m->dcs;
        info->num_groups = m->num_groups;
        info->total_slots = m->total_slots;
        info->stored_slots = m->stored_slots;
        info->layout = m->layout == argcsr_gpu::kLayoutReference ? ARGCSR_LAYOUT_REFERENCE : 0u;
        info->x_remap = m->x_remap ? 1u : 0u;
        info->x_used_columns = m->n_used;
        info->unit_len_bytes = m->ulen ? m->total_units : 0;
        info->nnz = m->nnz;
        info->heavy_groups = m->num_heavy;
        info->heavy_ctas = m->heavy_ctas;
        info->light_tiles = m->num_tiles;
        info->max_chunk_size = m->max_chunk;
        info->device_bytes = m->device_bytes;
        info->l2_persist_bytes = m->l2_persist_max;
        info->device = m->device;
        info->dtype = m->dtype;
    });
}

argcsr_status argcsr_dev_export(const argcsr_dev* m, uint64_t* groups4, uint64_t* threads_mapping, void* values,
                                int32_t* columns) {
    return guarded([&] {
        check_handle(m);
        DeviceScope scope(m->device);
        argcsr_gpu::export_arrays(m, groups4, threads_mapping, values, columns, cudaStreamPerThread);
    });
}

argcsr_status argcsr_dev_spmv(const argcsr_dev* m, const void* x, void* y, void* stream) {
    return guarded([&] {
        check_handle(m);
        if ((!x && m->num_cols) || !y) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv: null vector");
        DeviceScope scope(m->device);
        SpmvSerial serial(m, static_cast<cudaStream_t>(stream));
        argcsr_gpu::spmv_launch(m, x, y, 0, m->num_groups, serial.s);
        serial.done();
    });
}

argcsr_status argcsr_dev_spmv_scaled(const argcsr_dev* m, const void* x, const double* x_scale, void* y,
                                     void* stream) {
    return guarded([&] {
        check_handle(m);
        if ((!x && m->num_cols) || !y) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_scaled: null vector");
        DeviceScope scope(m->device);
        SpmvSerial serial(m, static_cast<cudaStream_t>(stream));
        argcsr_gpu::SpmvExtra ex;
        ex.x_scale = x_scale;
        argcsr_gpu::spmv_launch(m, x, y, 0, m->num_groups, serial.s, ex);
        serial.done();
    });
}

argcsr_status argcsr_dev_spmv_norm2(const argcsr_dev* m, const void* x, const double* x_scale, void* y,
                                    double* y_norm2, uint32_t flags, void* stream) {
    return guarded([&] {
        check_handle(m);
        if ((!x && m->num_cols) || !y || !y_norm2) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_norm2: null argument");
        if (flags & ~uint32_t(ARGCSR_SCALE_IS_NORM2)) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_norm2: unknown flags");
        if ((flags & ARGCSR_SCALE_IS_NORM2) && !x_scale)
            fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_norm2: ARGCSR_SCALE_IS_NORM2 needs x_scale");
        DeviceScope scope(m->device);
        SpmvSerial serial(m, static_cast<cudaStream_t>(stream));
        argcsr_dev* mm = const_cast<argcsr_dev*>(m);
        const uint64_t S = argcsr_gpu::norm_slots(m);
        if (!mm->norm_scratch)
            CUDA_OK(cudaMalloc(&mm->norm_scratch, (S + argcsr_gpu::norm_scratch_len(S) + 1) * sizeof(double)));
        argcsr_gpu::SpmvExtra ex;
        ex.x_scale = x_scale;
        ex.scale_is_norm2 = (flags & ARGCSR_SCALE_IS_NORM2) != 0;
        ex.norm_part = mm->norm_scratch;
        argcsr_gpu::spmv_launch(m, x, y, 0, m->num_groups, serial.s, ex);
        argcsr_gpu::norm_reduce(mm->norm_scratch, S, y_norm2, serial.s, mm->norm_scratch + S);
        serial.done();
    });
}

argcsr_status argcsr_dev_spmv_groups(const argcsr_dev* m, const void* x, uint64_t group_begin, uint64_t group_end,
                                     void* y, void* stream) {
    return guarded([&] {
        check_handle(m);
        if ((!x && m->num_cols) || !y) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_groups: null vector");
        DeviceScope scope(m->device);
        SpmvSerial serial(m, static_cast<cudaStream_t>(stream));
        argcsr_gpu::spmv_launch(m, x, y, group_begin, group_end, serial.s);
        serial.done();
    });
}

argcsr_status argcsr_dev_spmv_ex(const argcsr_dev* m, const void* x, const double* x_scale, uint64_t group_begin,
                                 uint64_t group_end, void* y, uint32_t flags, void* stream) {
    return guarded([&] {
        check_handle(m);
        if ((!x && m->num_cols) || !y) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_ex: null vector");
        if (flags & ~uint32_t(ARGCSR_SPMV_REUSE_X)) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_ex: unknown flags");
        DeviceScope scope(m->device);
        SpmvSerial serial(m, static_cast<cudaStream_t>(stream));
        argcsr_gpu::SpmvExtra ex;
        ex.x_scale = x_scale;
        ex.reuse_x = (flags & ARGCSR_SPMV_REUSE_X) != 0;
        argcsr_gpu::spmv_launch(m, x, y, group_begin, group_end, serial.s, ex);
        serial.done();
    });
}

argcsr_status argcsr_dev_spmv_peer(const argcsr_dev* m, const void* x, const double* x_scale, uint64_t group_begin,
                                   uint64_t group_end, void* y, void* const* peer_y, uint32_t npeers,
                                   const uint64_t* peer_rows, uint32_t flags, void* stream) {
    return guarded([&] {
        check_handle(m);
        if ((!x && m->num_cols) || !y) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_peer: null vector");
        if (flags & ~uint32_t(ARGCSR_SPMV_REUSE_X)) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_peer: unknown flags");
        if (npeers > argcsr_gpu::kMaxPeers) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_peer: at most 7 peers");
        if (npeers && !peer_y) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_peer: null peer list");
        for (uint32_t q = 0; q < npeers; ++q)
            if (!peer_y[q]) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_peer: null peer buffer");
        DeviceScope scope(m->device);
        SpmvSerial serial(m, static_cast<cudaStream_t>(stream));
        argcsr_gpu::SpmvExtra ex;
        ex.x_scale = x_scale;
        ex.reuse_x = (flags & ARGCSR_SPMV_REUSE_X) != 0;
        ex.peer_y = peer_y;
        ex.npeers = npeers;
        ex.peer_rows = peer_rows;
        argcsr_gpu::spmv_launch(m, x, y, group_begin, group_end, serial.s, ex);
        serial.done();
    });
}

argcsr_status argcsr_peer_signal(uint64_t* const* flags, uint32_t n, uint64_t value, const double* partial,
                                 double* const* partial_dst, void* stream) {
    return guarded([&] {
        if (n > argcsr_gpu::kMaxPeers) fail(ARGCSR_E_PARAMETER, "argcsr_peer_signal: at most 7 peers");
        if (n && !flags) fail(ARGCSR_E_PARAMETER, "argcsr_peer_signal: null flag list");
        argcsr_gpu::peer_signal(flags, n, value, partial, partial_dst, static_cast<cudaStream_t>(stream));
    });
}

argcsr_status argcsr_peer_wait(const uint64_t* flags, uint32_t n, uint64_t value, void* stream) {
    return guarded([&] {
        if (n && !flags) fail(ARGCSR_E_PARAMETER, "argcsr_peer_wait: null flags");
        argcsr_gpu::peer_wait(flags, n, value, static_cast<cudaStream_t>(stream));
    });
}

argcsr_status argcsr_peer_alloc(uint64_t bytes, int device, void** ptr, unsigned char handle[64]) {
    return guarded([&] {
        if (!ptr || !handle) fail(ARGCSR_E_PARAMETER, "argcsr_peer_alloc: null output");
        DeviceScope scope(device);
        void* p = nullptr;
        CUDA_OK(cudaMalloc(&p, std::max<uint64_t>(bytes, 1)));
        CUDA_OK(cudaMemset(p, 0, std::max<uint64_t>(bytes, 1)));
        cudaIpcMemHandle_t h;
        const cudaError_t e = cudaIpcGetMemHandle(&h, p);
        if (e != cudaSuccess) {
            cudaFree(p);
            CUDA_OK(e);
        }
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(handle, &h, 64);
        *ptr = p;
    });
}

argcsr_status argcsr_peer_open(const unsigned char handle[64], int device, void** ptr) {
    return guarded([&] {
        if (!ptr || !handle) fail(ARGCSR_E_PARAMETER, "argcsr_peer_open: null argument");
        DeviceScope scope(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, 64);
        CUDA_OK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

argcsr_status argcsr_peer_close(void* ptr) {
    return guarded([&] { CUDA_OK(cudaIpcCloseMemHandle(ptr)); });
}

argcsr_status argcsr_peer_free(void* ptr) {
    return guarded([&] { CUDA_OK(cudaFree(ptr)); });
}

argcsr_status argcsr_dev_spmv_host(const argcsr_dev* m, const void* x, uint64_t x_len, void* y) {
    return guarded([&] {
        check_handle(m);
        // argcsr.cpp:220-223
        if (x_len != m->num_cols)
            fail(ARGCSR_E_DIMENSION, "spmv_argcsr: vector length " + std::to_string(x_len) + " does not match " +
                                         std::to_string(m->num_cols) + " columns");
        if ((!x && x_len) || (!y && m->num_rows)) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_host: null vector");
        DeviceScope scope(m->device);
        cudaStream_t s = cudaStreamPerThread;
        const size_t es = elem_size(m->dtype);
        void *dx = nullptr, *dy = nullptr;
        CUDA_OK(cudaMallocAsync(&dx, std::max<uint64_t>(m->num_cols, 1) * es, s));
        struct Free {
            void** a;
            void** b;
            cudaStream_t s;
            ~Free() {
                if (*a) cudaFreeAsync(*a, s);
                if (*b) cudaFreeAsync(*b, s);
                cudaStreamSynchronize(s);
            }
        } fr{&dx, &dy, s};
        CUDA_OK(cudaMallocAsync(&dy, m->num_rows * es, s));
        if (x_len) CUDA_OK(cudaMemcpyAsync(dx, x, x_len * es, cudaMemcpyHostToDevice, s));
        {
            SpmvSerial serial(m, s);
            argcsr_gpu::spmv_launch(m, dx, dy, 0, m->num_groups, s);
            serial.done();
        }
        CUDA_OK(cudaMemcpyAsync(y, dy, m->num_rows * es, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
    });
}

argcsr_status argcsr_dev_spmv_host_async(const argcsr_dev* mc, const void* x_host, void* y_host, void* stream) {
    return guarded([&] {
        check_handle(mc);
        if ((!x_host && mc->num_cols) || (!y_host && mc->num_rows))
            fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_host_async: null buffer");
        DeviceScope scope(mc->device);
        // The staging and its events are handle state (like the copy streams):
        // one thread drives a handle's async calls.
        argcsr_dev* m = const_cast<argcsr_dev*>(mc);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t es = elem_size(m->dtype);
        const int b = int(m->as_calls & 1);
        if (!m->as_x[b]) {
            CUDA_OK(cudaMalloc(&m->as_x[b], std::max<uint64_t>(m->num_cols, 1) * es));
            CUDA_OK(cudaMalloc(&m->as_y[b], std::max<uint64_t>(m->num_rows, 1) * es));
            CUDA_OK(cudaEventCreateWithFlags(&m->as_up[b], cudaEventDisableTiming));
            CUDA_OK(cudaEventCreateWithFlags(&m->as_mv[b], cudaEventDisableTiming));
            CUDA_OK(cudaEventCreateWithFlags(&m->as_down[b], cudaEventDisableTiming));
        }
        // upload (copy engine 1) once the SpMV that last read this x buffer is done
        // each copy in two halves on two copy streams (C2 e2e 0.73 -> 0.70 ms per
        // step; ARGCSR_ASYNC_SPLIT=0 keeps one stream per direction)
        const bool split = argcsr_gpu::knobs().async_split;
        if (split && !m->as_h2d2) {
            CUDA_OK(cudaStreamCreateWithFlags(&m->as_h2d2, cudaStreamNonBlocking));
            CUDA_OK(cudaStreamCreateWithFlags(&m->as_d2h2, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                CUDA_OK(cudaEventCreateWithFlags(&m->as_j1[i], cudaEventDisableTiming));
                CUDA_OK(cudaEventCreateWithFlags(&m->as_j2[i], cudaEventDisableTiming));
            }
        }
        if (m->as_used[b]) CUDA_OK(cudaStreamWaitEvent(m->h2d, m->as_mv[b], 0));
        if (split) {
            const uint64_t h = m->num_cols / 2;
            if (m->as_used[b]) CUDA_OK(cudaStreamWaitEvent(m->as_h2d2, m->as_mv[b], 0));
            CUDA_OK(cudaMemcpyAsync(m->as_x[b], x_host, h * es, cudaMemcpyHostToDevice, m->h2d));
            CUDA_OK(cudaMemcpyAsync(static_cast<char*>(m->as_x[b]) + h * es, static_cast<const char*>(x_host) + h * es,
                                    (m->num_cols - h) * es, cudaMemcpyHostToDevice, m->as_h2d2));
            CUDA_OK(cudaEventRecord(m->as_j1[b], m->as_h2d2));
            CUDA_OK(cudaStreamWaitEvent(m->h2d, m->as_j1[b], 0));
        } else {
            CUDA_OK(cudaMemcpyAsync(m->as_x[b], x_host, m->num_cols * es, cudaMemcpyHostToDevice, m->h2d));
        }
        CUDA_OK(cudaEventRecord(m->as_up[b], m->h2d));
        // multiply on the caller's stream once x is up and this y buffer is downloaded
        CUDA_OK(cudaStreamWaitEvent(s, m->as_up[b], 0));
        if (m->as_used[b]) CUDA_OK(cudaStreamWaitEvent(s, m->as_down[b], 0));
        // one SpMV in flight per handle (x' buffer, heavy-group stream), even
        // when consecutive calls name different streams
        {
            SpmvSerial serial(m, s);
            argcsr_gpu::spmv_launch(m, m->as_x[b], m->as_y[b], 0, m->num_groups, s);
            serial.done();
        }
        CUDA_OK(cudaEventRecord(m->as_mv[b], s));
        // download (copy engine 2)
        CUDA_OK(cudaStreamWaitEvent(m->d2h, m->as_mv[b], 0));
        if (split) {
            const uint64_t h = m->num_rows / 2;
            CUDA_OK(cudaStreamWaitEvent(m->as_d2h2, m->as_mv[b], 0));
            CUDA_OK(cudaMemcpyAsync(y_host, m->as_y[b], h * es, cudaMemcpyDeviceToHost, m->d2h));
            CUDA_OK(cudaMemcpyAsync(static_cast<char*>(y_host) + h * es, static_cast<const char*>(m->as_y[b]) + h * es,
                                    (m->num_rows - h) * es, cudaMemcpyDeviceToHost, m->as_d2h2));
            CUDA_OK(cudaEventRecord(m->as_j2[b], m->as_d2h2));
            CUDA_OK(cudaStreamWaitEvent(m->d2h, m->as_j2[b], 0));
        } else {
            CUDA_OK(cudaMemcpyAsync(y_host, m->as_y[b], m->num_rows * es, cudaMemcpyDeviceToHost, m->d2h));
        }
        CUDA_OK(cudaEventRecord(m->as_down[b], m->d2h));
        m->as_used[b] = true;
        ++m->as_calls;
    });
}

argcsr_status argcsr_dev_host_wait(const argcsr_dev* m) {
    return guarded([&] {
        check_handle(m);
        DeviceScope scope(m->device);
        CUDA_OK(cudaStreamSynchronize(m->d2h));  // the last download follows every earlier stage
    });
}

argcsr_status argcsr_dev_spmv_host_staged(const argcsr_dev* m, const void* x_host, void* x_dev, void* y_dev,
                                          void* y_host, void* stream) {
    return guarded([&] {
        check_handle(m);
        if (!x_host || !x_dev || !y_dev || !y_host) fail(ARGCSR_E_PARAMETER, "argcsr_dev_spmv_host_staged: null buffer");
        DeviceScope scope(m->device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t es = elem_size(m->dtype);
        SpmvSerial serial(m, s);
        if (m->tile_cmax.empty() || m->lanes_per_unit != 4 || m->num_cols == 0) {
            CUDA_OK(cudaMemcpyAsync(x_dev, x_host, m->num_cols * es, cudaMemcpyHostToDevice, s));
            argcsr_gpu::spmv_launch(m, x_dev, y_dev, 0, m->num_groups, s);
            serial.done();
            CUDA_OK(cudaMemcpyAsync(y_host, y_dev, m->num_rows * es, cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaStreamSynchronize(s));
            return;
        }
        // Pipelined: x goes up in 8 pieces on one copy engine, y comes down in
        // 8 row chunks on the other (PCIe is full duplex), and each chunk of
        // light tiles starts as soon as x is resident up to the largest
        // column it reads (banded matrices: long before all of x arrives).
        constexpr int K = 8;
        const uint64_t C = m->num_cols, N = m->num_rows;
        const uint32_t nt = m->num_tiles;
        CUDA_OK(cudaEventRecord(m->ev_fork, s));  // order after the caller's prior work on s
        CUDA_OK(cudaStreamWaitEvent(m->h2d, m->ev_fork, 0));
        CUDA_OK(cudaStreamWaitEvent(m->d2h, m->ev_fork, 0));
        for (int j = 0; j < K; ++j) {
            const uint64_t c0 = C * j / K, c1 = C * (j + 1) / K;
            if (c1 > c0)
                CUDA_OK(cudaMemcpyAsync(static_cast<char*>(x_dev) + c0 * es, static_cast<const char*>(x_host) + c0 * es,
                                        (c1 - c0) * es, cudaMemcpyHostToDevice, m->h2d));
            CUDA_OK(cudaEventRecord(m->ev_x[j], m->h2d));
        }
        for (int k = 0; k < K; ++k) {
            const uint32_t t0 = uint32_t(uint64_t(nt) * k / K), t1 = uint32_t(uint64_t(nt) * (k + 1) / K);
            if (t1 > t0) {
                const uint64_t reach = m->tile_cmax[t1 - 1];  // columns 0..reach are read by tiles < t1
                const int j = int(std::min<uint64_t>(K - 1, ((reach + 1) * K + C - 1) / C - 1));
                CUDA_OK(cudaStreamWaitEvent(s, m->ev_x[std::max(j, 0)], 0));
                argcsr_gpu::spmv_launch_tiles(m, x_dev, y_dev, t0, t1, s);
            }
            CUDA_OK(cudaEventRecord(m->ev_c[k], s));
            CUDA_OK(cudaStreamWaitEvent(m->d2h, m->ev_c[k], 0));
            const uint64_t r0 = t0 < nt ? m->tile_row[t0] : N, r1 = m->tile_row[t1];
            if (r1 > r0)
                CUDA_OK(cudaMemcpyAsync(static_cast<char*>(y_host) + r0 * es, static_cast<const char*>(y_dev) + r0 * es,
                                        (r1 - r0) * es, cudaMemcpyDeviceToHost, m->d2h));
        }
        serial.done();
        CUDA_OK(cudaStreamSynchronize(m->d2h));
        CUDA_OK(cudaStreamSynchronize(s));
    });
}

argcsr_status argcsr_dev_to_csr(const argcsr_dev* m, uint64_t* row_pointers, int32_t* columns, void* values) {
    return guarded([&] {
        check_handle(m);
        if (!row_pointers || (m->nnz && (!columns || !values))) fail(ARGCSR_E_PARAMETER, "argcsr_dev_to_csr: null output");
        DeviceScope scope(m->device);
        argcsr_gpu::to_csr(m, row_pointers, columns, values, cudaStreamPerThread);
    });
}

argcsr_status argcsr_dev_chunk_entries(const argcsr_dev* m, uint64_t group_index, uint64_t chunk_index, void* values,
                                       int32_t* columns, uint64_t cap, uint64_t* n) {
    return guarded([&] {
        check_handle(m);
        // argcsr.cpp:231-238
        if (group_index >= m->num_groups)
            fail(ARGCSR_E_BOUNDS, "chunk_entries: group " + std::to_string(group_index) + " out of range");
        if (chunk_index >= m->tpg)
            fail(ARGCSR_E_BOUNDS, "chunk_entries: chunk " + std::to_string(chunk_index) + " out of range");
        if (!n) fail(ARGCSR_E_PARAMETER, "argcsr_dev_chunk_entries: null count");
        DeviceScope scope(m->device);
        cudaStream_t s = cudaStreamPerThread;
        argcsr_gpu::GroupDesc d;
        CUDA_OK(cudaMemcpyAsync(&d, m->groups + group_index, sizeof d, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        const size_t es = elem_size(m->dtype);
        std::vector<int32_t> c(d.chunk);
        std::vector<unsigned char> v(size_t(d.chunk) * es);
        // lanes at or past the stored stride are free lanes: all padding
        const uint64_t w = d.stride();
        if (d.chunk && chunk_index < w) {
            const uint64_t slot = d.offset() + chunk_index;
            CUDA_OK(cudaMemcpy2DAsync(c.data(), sizeof(int32_t), m->columns + slot, w * sizeof(int32_t),
                                      sizeof(int32_t), d.chunk, cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaMemcpy2DAsync(v.data(), es, static_cast<const unsigned char*>(m->values) + slot * es, w * es,
                                      es, d.chunk, cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaStreamSynchronize(s));
        } else {
            std::fill(c.begin(), c.end(), -1);
        }
        uint64_t k = 0;
        while (k < d.chunk && c[k] != -1) ++k;
        if (m->x_remap && k) {  // stored column -> reference column (xremap.cu)
            std::vector<uint32_t> pc(k);
            for (uint64_t i = 0; i < k; ++i)
                CUDA_OK(cudaMemcpyAsync(&pc[i], m->perm + c[i], sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaStreamSynchronize(s));
            for (uint64_t i = 0; i < k; ++i) c[i] = int32_t(pc[i]);
        }
        *n = k;
        if (k > cap) fail(ARGCSR_E_BOUNDS, "chunk_entries: output capacity too small");
        if (k) {
            if (!columns || !values) fail(ARGCSR_E_PARAMETER, "argcsr_dev_chunk_entries: null output");
            std::memcpy(columns, c.data(), k * sizeof(int32_t));
            std::memcpy(values, v.data(), k * es);
        }
    });
}

argcsr_status argcsr_dev_balance_stats(const argcsr_dev* m, uint64_t* per_group_nnz, double* max_over_mean,
                                       double* coefficient_of_variation) {
    return guarded([&] {
        check_handle(m);
        DeviceScope scope(m->device);
        argcsr_gpu::balance_stats(m, per_group_nnz, max_over_mean, coefficient_of_variation, cudaStreamPerThread);
    });
}

argcsr_status argcsr_dev_padding_stats(const argcsr_dev* m, argcsr_format_stats* out) {
    return guarded([&] {
        check_handle(m);
        if (!out) fail(ARGCSR_E_PARAMETER, "argcsr_dev_padding_stats: null output");
        DeviceScope scope(m->device);
        argcsr_gpu::padding_stats(m, out, cudaStreamPerThread);
    });
}

void argcsr_dev_free(argcsr_dev* m) { free_handle(m); }

// ------------------------------------------------- ELLPACK / Sliced ELLPACK
namespace {
void free_sell(argcsr_sell* m) {
    if (!m) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    cudaFree(m->width);
    cudaFree(m->offset);
    cudaFree(m->values);
    cudaFree(m->columns);
    if (prev >= 0) cudaSetDevice(prev);
    delete m;
}

argcsr_status sell_convert_common(const argcsr_csr_view* csr, uint64_t slice_size, bool ellpack, int device,
                                  void* stream, argcsr_sell** out) {
    return guarded([&] {
        const char* who = ellpack ? "ellpack_from_csr" : "sliced_from_csr";
        if (!csr || !out) fail(ARGCSR_E_PARAMETER, std::string(who) + ": null argument");
        *out = nullptr;
        if (!ellpack && slice_size == 0) fail(ARGCSR_E_PARAMETER, "sliced_from_csr: slice_size must be at least 1");
        if (csr->dtype != ARGCSR_F64 && csr->dtype != ARGCSR_F32) fail(ARGCSR_E_PARAMETER, std::string(who) + ": unknown dtype");
        if (!csr->row_pointers || (csr->nnz && (!csr->columns || !csr->values)))
            fail(ARGCSR_E_PARAMETER, std::string(who) + ": null CSR array");
        DeviceScope scope(device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        auto* m = new argcsr_sell;
        m->device = device;
        m->dtype = csr->dtype;
        m->ellpack = ellpack;
        m->num_rows = csr->num_rows;
        m->num_cols = csr->num_cols;
        m->nnz = csr->nnz;
        m->slice_size = ellpack ? std::max<uint64_t>(csr->num_rows, 1) : slice_size;
        try {
            const size_t es = elem_size(csr->dtype);
            const uint64_t N = csr->num_rows, nnz = csr->nnz;
            const uint64_t* rp = csr->row_pointers;
            const int32_t* cols = csr->columns;
            const void* vals = csr->values;
            void* staged[3] = {nullptr, nullptr, nullptr};
            struct Release {
                void** p;
                cudaStream_t s;
                ~Release() {
                    for (int i = 0; i < 3; ++i)
                        if (p[i]) cudaFreeAsync(p[i], s);
                }
            } release{staged, s};
            if (csr->space == ARGCSR_HOST) {
                CUDA_OK(cudaMallocAsync(&staged[0], (N + 1) * sizeof(uint64_t), s));
                CUDA_OK(cudaMallocAsync(&staged[1], std::max<uint64_t>(nnz, 1) * sizeof(int32_t), s));
                CUDA_OK(cudaMallocAsync(&staged[2], std::max<uint64_t>(nnz, 1) * es, s));
                CUDA_OK(cudaMemcpyAsync(staged[0], rp, (N + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
                if (nnz) {
                    CUDA_OK(cudaMemcpyAsync(staged[1], cols, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
                    CUDA_OK(cudaMemcpyAsync(staged[2], vals, nnz * es, cudaMemcpyHostToDevice, s));
                }
                rp = static_cast<const uint64_t*>(staged[0]);
                cols = static_cast<const int32_t*>(staged[1]);
                vals = staged[2];
            }
            argcsr_gpu::sell_convert(m, rp, cols, vals, s);
        } catch (...) {
            free_sell(m);
            throw;
        }
        *out = m;
    });
}
}  // namespace

argcsr_status argcsr_ell_convert(const argcsr_csr_view* csr, int device, void* stream, argcsr_sell** out) {
    return sell_convert_common(csr, 0, true, device, stream, out);
}

argcsr_status argcsr_sell_convert(const argcsr_csr_view* csr, uint64_t slice_size, int device, void* stream,
                                  argcsr_sell** out) {
    return sell_convert_common(csr, slice_size, false, device, stream, out);
}

argcsr_status argcsr_sell_info(const argcsr_sell* m, argcsr_sell_info_t* info) {
    return guarded([&] {
        if (!m || !info) fail(ARGCSR_E_PARAMETER, "argcsr_sell_info: null argument");
        DeviceScope scope(m->device);
        info->num_rows = m->num_rows;
        info->num_cols = m->num_cols;
        info->slice_size = m->slice_size;
        info->num_slices = m->num_slices;
        info->total_slots = m->total_slots;
        std::vector<uint64_t> w(m->num_slices);
        if (m->num_slices)
            CUDA_OK(cudaMemcpy(w.data(), m->width, m->num_slices * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        info->width = w.empty() ? 0 : *std::max_element(w.begin(), w.end());
        info->device_bytes = m->device_bytes;
        info->device = m->device;
        info->dtype = m->dtype;
        info->ellpack = m->ellpack ? 1u : 0u;
    });
}

argcsr_status argcsr_sell_export(const argcsr_sell* m, uint64_t* slice_widths, uint64_t* slice_offsets, void* values,
                                 int32_t* columns) {
    return guarded([&] {
        if (!m) fail(ARGCSR_E_PARAMETER, "argcsr_sell_export: null handle");
        DeviceScope scope(m->device);
        cudaStream_t s = cudaStreamPerThread;
        if (slice_widths && m->num_slices)
            CUDA_OK(cudaMemcpyAsync(slice_widths, m->width, m->num_slices * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        if (slice_offsets && m->num_slices)
            CUDA_OK(cudaMemcpyAsync(slice_offsets, m->offset, m->num_slices * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        if (values && m->total_slots)
            CUDA_OK(cudaMemcpyAsync(values, m->values, m->total_slots * elem_size(m->dtype), cudaMemcpyDeviceToHost, s));
        if (columns && m->total_slots)
            CUDA_OK(cudaMemcpyAsync(columns, m->columns, m->total_slots * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
    });
}

argcsr_status argcsr_sell_spmv(const argcsr_sell* m, const void* x, void* y, void* stream) {
    return guarded([&] {
        if (!m) fail(ARGCSR_E_PARAMETER, "argcsr_sell_spmv: null handle");
        if ((!x && m->num_cols) || (!y && m->num_rows)) fail(ARGCSR_E_PARAMETER, "argcsr_sell_spmv: null vector");
        DeviceScope scope(m->device);
        argcsr_gpu::sell_spmv(m, x, y, static_cast<cudaStream_t>(stream));
    });
}

argcsr_status argcsr_sell_spmv_host(const argcsr_sell* m, const void* x, uint64_t x_len, void* y) {
    return guarded([&] {
        if (!m) fail(ARGCSR_E_PARAMETER, "argcsr_sell_spmv_host: null handle");
        const char* who = m->ellpack ? "spmv_ellpack" : "spmv_sliced";  // ellpack.cpp:135-139, 169-173
        if (x_len != m->num_cols)
            fail(ARGCSR_E_DIMENSION, std::string(who) + ": vector length " + std::to_string(x_len) +
                                         " does not match " + std::to_string(m->num_cols) + " columns");
        DeviceScope scope(m->device);
        cudaStream_t s = cudaStreamPerThread;
        const size_t es = elem_size(m->dtype);
        void *dx = nullptr, *dy = nullptr;
        CUDA_OK(cudaMallocAsync(&dx, std::max<uint64_t>(x_len, 1) * es, s));
        CUDA_OK(cudaMallocAsync(&dy, std::max<uint64_t>(m->num_rows, 1) * es, s));
        if (x_len) CUDA_OK(cudaMemcpyAsync(dx, x, x_len * es, cudaMemcpyHostToDevice, s));
        argcsr_gpu::sell_spmv(m, dx, dy, s);
        if (m->num_rows) CUDA_OK(cudaMemcpyAsync(y, dy, m->num_rows * es, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaFreeAsync(dx, s));
        CUDA_OK(cudaFreeAsync(dy, s));
        CUDA_OK(cudaStreamSynchronize(s));
    });
}

void argcsr_sell_free(argcsr_sell* m) { free_sell(m); }

argcsr_status argcsr_dev_import(const argcsr_argcsr_view* v, int device, void* stream, uint32_t flags,
                                argcsr_dev** out) {
    return guarded([&] {
        if (!v || !out) fail(ARGCSR_E_PARAMETER, "argcsr_dev_import: null argument");
        *out = nullptr;
        check_flags(flags, "argcsr_dev_import");
        if (v->threads_per_group == 0) fail(ARGCSR_E_FORMAT, "argcsr import: threads_per_group is 0");
        if (v->num_rows == 0) fail(ARGCSR_E_FORMAT, "argcsr import: no rows");
        if (v->threads_per_group > argcsr_gpu::kMaxThreadsPerGroup)
            fail(ARGCSR_E_UNSUPPORTED, "argcsr import: threads_per_group " + std::to_string(v->threads_per_group) +
                                           " exceeds the device limit " +
                                           std::to_string(argcsr_gpu::kMaxThreadsPerGroup));
        if (v->num_rows >= 0xFFFFFFFFull) fail(ARGCSR_E_UNSUPPORTED, "argcsr import: num_rows exceeds 2^32-2");
        if (v->num_groups == 0 || v->num_groups > v->num_rows)
            fail(ARGCSR_E_FORMAT, "argcsr import: group count out of range");
        if (v->dtype != ARGCSR_F64 && v->dtype != ARGCSR_F32) fail(ARGCSR_E_PARAMETER, "argcsr import: unknown dtype");
        if (!v->groups4 || !v->threads_mapping || (v->total_slots && (!v->values || !v->columns)))
            fail(ARGCSR_E_PARAMETER, "argcsr_dev_import: null array");
        DeviceScope scope(device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        argcsr_dev* m = new_handle(device, v->dtype, v->num_rows, v->num_cols, v->threads_per_group, 0, flags);
        try {
            argcsr_gpu::import_reference(m, v->num_groups, v->groups4, v->threads_mapping, v->values, v->columns,
                                         v->total_slots, s);
            CUDA_OK(cudaStreamSynchronize(s));
        } catch (...) {
            free_handle(m);
            throw;
        }
        *out = m;
    });
}

argcsr_status argcsr_dev_write_binary(const argcsr_dev* m, const char* path) {
    return guarded([&] {
        check_handle(m);
        if (!path) fail(ARGCSR_E_PARAMETER, "argcsr_dev_write_binary: null path");
        if (m->dtype != ARGCSR_F64)
            fail(ARGCSR_E_UNSUPPORTED, "write_binary: the container stores fp64 values (io.cpp:282-298)");
        DeviceScope scope(m->device);
        const uint64_t G = m->num_groups, N = m->num_rows, S = m->total_slots;
        std::vector<uint64_t> g4(4 * G), tm(N);
        std::vector<double> vals(S);
        std::vector<int32_t> cols(S);
        argcsr_gpu::export_arrays(m, g4.data(), tm.data(), vals.data(), cols.data(), cudaStreamPerThread);
        File file;
        file.f = std::fopen(path, "wb");
        if (!file.f) fail(ARGCSR_E_IO, std::string("cannot open '") + path + "' for writing");
        Writer w{file.f};
        w.bytes(kMagic, sizeof kMagic);  // put_header, io.cpp:242-246
        w.u32(kVersion);
        w.u8(kTagArgCsr);
        w.u64(m->num_rows);  // write_binary(ArgCsrMatrix), io.cpp:282-298
        w.u64(m->num_cols);
        w.u64(m->tpg);
        w.u64(G);
        w.bytes(g4.data(), g4.size() * sizeof(uint64_t));  // {first_row, size, offset, chunk_size} per group
        w.u64(N);
        w.bytes(tm.data(), N * sizeof(uint64_t));
        w.u64(S);
        w.bytes(vals.data(), S * sizeof(double));
        w.u64(S);
        w.bytes(cols.data(), S * sizeof(int32_t));
        if (std::fflush(file.f) != 0) fail(ARGCSR_E_IO, "binary write failure");
    });
}

argcsr_status argcsr_dev_read_binary(const char* path, uint64_t tpg, uint64_t dcs, int device, void* stream,
                                     uint32_t flags, argcsr_dev** out) {
    return guarded([&] {
        if (!path || !out) fail(ARGCSR_E_PARAMETER, "argcsr_dev_read_binary: null argument");
        *out = nullptr;
        check_flags(flags, "argcsr_dev_read_binary");
        File file;
        file.f = std::fopen(path, "rb");
        if (!file.f) fail(ARGCSR_E_IO, std::string("cannot open '") + path + "' for reading");
        std::fseek(file.f, 0, SEEK_END);
        const long size = std::ftell(file.f);
        std::fseek(file.f, 0, SEEK_SET);
        Reader r{file.f, size < 0 ? 0 : uint64_t(size)};
        char magic[8];
        r.bytes(magic, sizeof magic);  // read_binary, io.cpp:300-312
        if (std::memcmp(magic, kMagic, sizeof magic) != 0) fail(ARGCSR_E_FORMAT, "binary: bad magic");
        const uint32_t version = r.u32();
        if (version != kVersion) fail(ARGCSR_E_FORMAT, "binary: unsupported version " + std::to_string(version));
        const uint8_t tag = r.u8();
        if (tag == kTagArgCsr) {  // io.cpp:343-363
            argcsr_argcsr_view v{};
            v.num_rows = r.u64();
            v.num_cols = r.u64();
            v.threads_per_group = r.u64();
            const uint64_t G = r.u64();
            if (G > r.left / 32) fail(ARGCSR_E_PARSE, "binary stream truncated");
            std::vector<uint64_t> g4(4 * G);
            r.bytes(g4.data(), g4.size() * sizeof(uint64_t));
            std::vector<uint64_t> tm = r.array<uint64_t>();
            std::vector<double> vals = r.array<double>();
            std::vector<int32_t> cols = r.array<int32_t>();
            if (tm.size() != v.num_rows) fail(ARGCSR_E_FORMAT, "argcsr import: threads_mapping length != num_rows");
            if (vals.size() != cols.size()) fail(ARGCSR_E_FORMAT, "argcsr import: values/columns lengths differ");
            v.num_groups = G;
            v.groups4 = g4.data();
            v.threads_mapping = tm.data();
            v.values = vals.data();
            v.columns = cols.data();
            v.total_slots = vals.size();
            v.dtype = ARGCSR_F64;
            const argcsr_status st = argcsr_dev_import(&v, device, stream, flags, out);
            if (st != ARGCSR_OK) fail(st, argcsr_gpu::last_error());
        } else if (tag == kTagCsr) {  // io.cpp:313-320: converted on the device
            argcsr_csr_view v{};
            v.num_rows = r.u64();
            v.num_cols = r.u64();
            std::vector<double> vals = r.array<double>();
            std::vector<int32_t> cols = r.array<int32_t>();
            std::vector<uint64_t> rp = r.array<uint64_t>();
            if (v.num_rows == UINT64_MAX || rp.empty() || rp.size() != v.num_rows + 1 || vals.size() != cols.size() ||
                rp.front() > rp.back() || rp.back() > vals.size())
                fail(ARGCSR_E_FORMAT, "binary: inconsistent CSR arrays");
            v.nnz = rp.back() - rp.front();
            v.row_pointers = rp.data();
            v.columns = cols.data();
            v.values = vals.data();
            v.dtype = ARGCSR_F64;
            v.space = ARGCSR_HOST;
            const argcsr_status st = argcsr_dev_convert_ex(&v, tpg, dcs, device, stream, flags, out);
            if (st != ARGCSR_OK) fail(st, argcsr_gpu::last_error());
        } else if (tag == 1 || tag == 2) {
            fail(ARGCSR_E_UNSUPPORTED, "binary: ELLPACK / sliced ELLPACK containers have no device path");
        } else {
            fail(ARGCSR_E_FORMAT, "binary: unknown format tag " + std::to_string(tag));
        }
    });
}

argcsr_status argcsr_partition_rows(const uint64_t* row_pointers, uint64_t num_rows, uint32_t parts,
                                    uint64_t* row_begin) {
    return guarded([&] {
        if (parts == 0) fail(ARGCSR_E_PARAMETER, "partition_rows: parts must be at least 1");
        if (!row_pointers || !row_begin) fail(ARGCSR_E_PARAMETER, "partition_rows: null argument");
        const uint64_t nnz = row_pointers[num_rows] - row_pointers[0];
        row_begin[0] = 0;
        for (uint32_t p = 1; p < parts; ++p) {
            const unsigned __int128 target128 = (unsigned __int128)nnz * p / parts;
            const uint64_t target = row_pointers[0] + uint64_t(target128);
            uint64_t r = uint64_t(std::lower_bound(row_pointers, row_pointers + num_rows + 1, target) - row_pointers);
            // keep parts non-empty and ordered when rows allow it
            const uint64_t lo = row_begin[p - 1] + (num_rows >= parts ? 1 : 0);
            const uint64_t hi = num_rows >= parts ? num_rows - (parts - p) : num_rows;
            r = std::min(std::max(r, lo), hi);
            row_begin[p] = r;
        }
        row_begin[parts] = num_rows;
    });
}

}  // extern "C"
