// Single-box multi-GPU layer behind the C-ABI
// (include/argcsr_gpu.h, argcsr_mgpu_*).  Replaces the reference's only
// parallel path, parallel_over / spmv_argcsr_parallel (proj/src/bench.cpp:
// 48-71, 109-116), which splits the GROUP range over host threads: here the
// ROWS are split into nnz-balanced contiguous slices, one per GPU, each GPU
// converts its own slice (so slice p is bit-exact with the reference
// argcsr_from_csr(slice_p)), x is replicated, and a step is the slice SpMV
// plus the exchange of the y slices into every GPU's next x.
//
// Exchanges: NCCL all-gather (in place, equal slices) / grouped broadcasts,
// the halo (grouped send/recv of only the x rows other slices read, planned at
// setup), or p2p (no collective: the SpMV epilogue stores y into the peers'
// next-x buffers over NVLink; step flags and partial norms in peer memory).
// NCCL is dlopen'ed (libnccl.so.2), so the single-GPU library has no NCCL
// dependency; every NCCL failure and every asynchronous communicator error
// (ncclCommGetAsyncError, polled each step) surfaces as ARGCSR_E_NCCL.
//
// Power iteration (config C5): ||y||^2 comes from the SpMV epilogue
// (per-CTA partials + a fixed-order reduce), is all-reduced (8 bytes), and the
// scaling 1/||y|| is fused into the next SpMV's gathers (SpmvExtra
// scale_is_norm2).  With the NCCL exchanges the exchange of step k runs on a
// collective stream under the interior groups of step k+1 (rows whose columns
// lie in the slice's own x rows); the boundary groups wait for it.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <exception>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "argcsr_gpu.h"
#include "common.cuh"
#include "spmv.cuh"

using argcsr_gpu::DeviceScope;
using argcsr_gpu::fail;
using argcsr_gpu::guarded;

namespace argcsr_gpu {
namespace {

// ------------------------------------------------------------ NCCL loader
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

const NcclApi& nccl() {
    static std::mutex mu;
    static NcclApi api;
    static bool loaded = false;
    static std::string why;
    std::lock_guard<std::mutex> lock(mu);
    if (!loaded && why.empty()) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (e.g. torch's)
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            why = std::string("NCCL not available: ") + (e ? e : "dlopen(libnccl.so.2) failed");
        } else {
            auto sym = [&](auto& fn, const char* name) {
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
                if (!fn && why.empty()) why = std::string("NCCL symbol missing: ") + name;
            };
            sym(api.GetUniqueId, "ncclGetUniqueId");
            sym(api.CommInitRank, "ncclCommInitRank");
            sym(api.CommInitAll, "ncclCommInitAll");
            sym(api.CommDestroy, "ncclCommDestroy");
            sym(api.CommAbort, "ncclCommAbort");
            sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
            sym(api.GetErrorString, "ncclGetErrorString");
            sym(api.AllReduce, "ncclAllReduce");
            sym(api.AllGather, "ncclAllGather");
            sym(api.Broadcast, "ncclBroadcast");
            sym(api.Send, "ncclSend");
            sym(api.Recv, "ncclRecv");
            sym(api.GroupStart, "ncclGroupStart");
            sym(api.GroupEnd, "ncclGroupEnd");
            loaded = why.empty();
        }
    }
    if (!loaded) fail(ARGCSR_E_NCCL, why);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess || r == ncclInProgress) return;
    const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "unknown";
    fail(ARGCSR_E_NCCL, std::string(what) + ": " + msg);
}
#define NCCL_OK(expr) nccl_check((expr), #expr)

struct NcclGroup {  // ncclGroupStart/End around the calls of every local rank
    int unwinding = std::uncaught_exceptions();
    NcclGroup() { NCCL_OK(nccl().GroupStart()); }
    ~NcclGroup() noexcept(false) {
        const ncclResult_t r = nccl().GroupEnd();
        if (std::uncaught_exceptions() == unwinding) nccl_check(r, "ncclGroupEnd");
    }
};

ncclDataType_t nccl_type(argcsr_dtype d) { return d == ARGCSR_F64 ? ncclFloat64 : ncclFloat32; }
size_t esize(argcsr_dtype d) { return d == ARGCSR_F64 ? sizeof(double) : sizeof(float); }

// ------------------------------------------------------------ small kernels
template <typename T>
__global__ void k_gather_rows(T* __restrict__ out, const T* __restrict__ x, const uint32_t* __restrict__ rows,
                              uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = x[rows[i]];
}
template <typename T>
__global__ void k_scatter_rows(T* __restrict__ x, const uint32_t* __restrict__ rows, const T* __restrict__ in,
                               uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        x[rows[i]] = in[i];
}
// out = fl(in * fl(1 / fl(sqrt(*s2))))  (the normalisation of the last x)
template <typename T>
__global__ void k_scale_norm2(T* __restrict__ out, const T* __restrict__ in, const double* s2, uint64_t n) {
    const double s = __drcp_rn(__dsqrt_rn(*s2));
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = T(__dmul_rn(double(in[i]), s));
}
__global__ void k_set_u64(uint64_t* p, uint64_t v) { *p = v; }
__global__ void k_rebase(uint64_t* __restrict__ out, const uint64_t* __restrict__ in, uint64_t n) {
    const uint64_t base = in[0];
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = in[i] - base;
}

unsigned grid_of(uint64_t n) { return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148u * 16u))); }

template <typename T>
void gather_rows(void* out, const void* x, const uint32_t* rows, uint64_t n, cudaStream_t s) {
    if (!n) return;
    k_gather_rows<T><<<grid_of(n), 256, 0, s>>>(static_cast<T*>(out), static_cast<const T*>(x), rows, n);
    LAUNCH_OK("k_gather_rows");
}
template <typename T>
void scatter_rows(void* x, const uint32_t* rows, const void* in, uint64_t n, cudaStream_t s) {
    if (!n) return;
    k_scatter_rows<T><<<grid_of(n), 256, 0, s>>>(static_cast<T*>(x), rows, static_cast<const T*>(in), n);
    LAUNCH_OK("k_scatter_rows");
}

// ------------------------------------------------------------ host planning
// nnz-balanced contiguous rows (argcsr_partition_rows' rule).
std::vector<uint64_t> partition(const uint64_t* rp, uint64_t num_rows, uint32_t parts) {
    std::vector<uint64_t> b(parts + 1, 0);
    const uint64_t nnz = rp[num_rows] - rp[0];
    for (uint32_t p = 1; p < parts; ++p) {
        const uint64_t target = rp[0] + uint64_t((unsigned __int128)nnz * p / parts);
        uint64_t r = uint64_t(std::lower_bound(rp, rp + num_rows + 1, target) - rp);
        const uint64_t lo = b[p - 1] + (num_rows >= parts ? 1 : 0);
        const uint64_t hi = num_rows >= parts ? num_rows - (parts - p) : num_rows;
        b[p] = std::min(std::max(r, lo), hi);
    }
    b[parts] = num_rows;
    return b;
}

void plan_interior(const uint64_t* rp, const int32_t* cols, uint64_t rows, const uint64_t* gfirst, uint64_t G,
                   uint64_t r0, uint64_t r1, uint64_t* ga, uint64_t* gb) {
    // row r is "bad" when it reads a column outside [r0, r1); a group is good
    // when none of its rows is bad; the longest run of good groups wins
    // (first one on ties).
    std::vector<uint8_t> bad(rows, 0);
    for (uint64_t r = 0; r < rows; ++r)
        for (uint64_t k = rp[r] - rp[0]; k < rp[r + 1] - rp[0]; ++k) {
            const int64_t c = cols[k];
            if (c < int64_t(r0) || c >= int64_t(r1)) {
                bad[r] = 1;
                break;
            }
        }
    uint64_t best_a = 0, best_b = 0, run_a = 0;
    bool in_run = false;
    for (uint64_t g = 0; g <= G; ++g) {
        bool good = false;
        if (g < G) {
            good = true;
            for (uint64_t r = gfirst[g]; r < gfirst[g + 1] && good; ++r) good = !bad[r];
        }
        if (good && !in_run) run_a = g, in_run = true;
        if (!good && in_run) {
            if (g - run_a > best_b - best_a) best_a = run_a, best_b = g;
            in_run = false;
        }
    }
    *ga = best_a;
    *gb = best_b;
}

// Distinct rows of every owner p != self that `cols` reference, ascending
// (a bitmap over the columns: O(nnz + num_cols)).
std::vector<std::vector<uint32_t>> plan_needed(const int32_t* cols, uint64_t nnz, uint64_t num_cols,
                                               const std::vector<uint64_t>& bounds, uint32_t self) {
    const uint32_t P = uint32_t(bounds.size() - 1);
    std::vector<uint64_t> bits((num_cols + 63) / 64, 0);
    const uint64_t lo = bounds[self], hi = bounds[self + 1];
    for (uint64_t k = 0; k < nnz; ++k) {
        const int64_t c = cols[k];
        if (c < 0 || uint64_t(c) >= num_cols || (uint64_t(c) >= lo && uint64_t(c) < hi)) continue;
        bits[uint64_t(c) >> 6] |= uint64_t(1) << (uint64_t(c) & 63);
    }
    std::vector<std::vector<uint32_t>> out(P);
    for (uint32_t p = 0; p < P; ++p) {
        if (p == self) continue;
        for (uint64_t c = bounds[p]; c < bounds[p + 1];) {
            const uint64_t w = bits[c >> 6] >> (c & 63);
            if (!w) {
                c = (c | 63) + 1;
                continue;
            }
            c += uint64_t(__builtin_ctzll(w));
            if (c < bounds[p + 1]) out[p].push_back(uint32_t(c));
            ++c;
        }
    }
    return out;
}

}  // namespace
}  // namespace argcsr_gpu

using namespace argcsr_gpu;

// ------------------------------------------------------------ the handle
struct MgRank {
    int device = 0, rank = 0;
    argcsr_dev* m = nullptr;
    uint64_t r0 = 0, r1 = 0;
    uint64_t ga = 0, gb = 0;      // interior groups
    ncclComm_t comm = nullptr;
    cudaStream_t cs = nullptr;    // collective stream
    cudaEvent_t ev_spmv = nullptr, ev_red = nullptr, ev_gath = nullptr;
    void* X[2] = {nullptr, nullptr};
    bool own_x = true;
    double* part = nullptr;       // 3 regions of norm_slots(m) partials, then the reduce scratch
    uint64_t part_len = 0;
    double* s2 = nullptr;         // [0] local ||y||^2, [1] all-reduced
    // halo plan
    std::vector<std::vector<uint32_t>> need_rows;  // rows this rank reads from every owner (global)
    std::vector<uint64_t> send_counts, recv_counts;
    uint32_t* send_rows = nullptr;  // local indices into the slice, owners' order
    uint32_t* recv_rows = nullptr;  // global rows, owners' order
    void* send_buf = nullptr;
    void* recv_buf = nullptr;
    uint64_t nsend = 0, nrecv = 0;
    // p2p
    void* pblock = nullptr;
    unsigned char ipc[64] = {};
    size_t off_x[2] = {0, 0}, off_flags = 0, off_partial = 0, pbytes = 0;
    std::vector<void*> peer_base;   // by global rank (nullptr: self)
    std::vector<void*> opened;      // IPC mappings (multi-process)
    std::vector<int> peers;         // global ranks, ascending
    std::vector<uint64_t> peer_rows;  // per peer: [lo, hi) local rows to store (halo)
    std::vector<void*> peer_y;      // scratch for spmv_peer
};

struct argcsr_mgpu {
    int nranks = 1;
    std::vector<MgRank> r;
    argcsr_exchange exchange = ARGCSR_EXCHANGE_NONE;
    argcsr_dtype dtype = ARGCSR_F64;
    uint64_t num_rows = 0, num_cols = 0, nnz = 0;
    std::vector<uint64_t> bounds;
    bool normalize = false, begun = false, last_full = true;
    uint64_t k = 0, k0 = 0;
    bool connected = true;  // p2p peers connected
    bool single_process = false;
};

namespace {

bool equal_slices(const argcsr_mgpu* h) {
    for (int p = 1; p < h->nranks; ++p)
        if (h->bounds[p + 1] - h->bounds[p] != h->bounds[1] - h->bounds[0]) return false;
    return true;
}

void free_rank(MgRank& R, bool abort_comm) {
    cudaSetDevice(R.device);
    for (void* p : R.opened) cudaIpcCloseMemHandle(p);
    R.opened.clear();
    if (R.pblock) cudaFree(R.pblock);
    if (R.own_x)
        for (void* x : R.X)
            if (x) cudaFree(x);
    cudaFree(R.part);
    cudaFree(R.s2);
    cudaFree(R.send_rows);
    cudaFree(R.recv_rows);
    cudaFree(R.send_buf);
    cudaFree(R.recv_buf);
    if (R.ev_spmv) cudaEventDestroy(R.ev_spmv);
    if (R.ev_red) cudaEventDestroy(R.ev_red);
    if (R.ev_gath) cudaEventDestroy(R.ev_gath);
    if (R.cs) cudaStreamDestroy(R.cs);
    if (R.comm) {
        try {
            if (abort_comm) nccl().CommAbort(R.comm);
            else nccl().CommDestroy(R.comm);
        } catch (...) {
        }
    }
    R.comm = nullptr;
    argcsr_dev_free(R.m);
    R.m = nullptr;
}

void free_handle(argcsr_mgpu* h, bool abort_comm = false) {
    if (!h) return;
    int prev = -1;
    cudaGetDevice(&prev);
    for (MgRank& R : h->r) {
        if (R.device >= 0) cudaSetDevice(R.device);
        cudaDeviceSynchronize();
    }
    for (MgRank& R : h->r) free_rank(R, abort_comm);
    if (prev >= 0) cudaSetDevice(prev);
    delete h;
}

// Convert rows [r0, r1) of A on R.device (row pointers rebased; columns and
// values are views into A).
void convert_slice(MgRank& R, const argcsr_csr_view* A, const std::vector<uint64_t>& rp_host, uint64_t tpg,
                   uint64_t dcs, uint32_t flags) {
    const uint64_t n = R.r1 - R.r0;
    const uint64_t a = rp_host[R.r0], b = rp_host[R.r1];
    argcsr_csr_view v{};
    v.num_rows = n;
    v.num_cols = A->num_cols;
    v.nnz = b - a;
    v.dtype = A->dtype;
    v.space = A->space;
    v.columns = A->columns ? A->columns + a : nullptr;
    v.values = A->values ? static_cast<const unsigned char*>(A->values) + a * esize(A->dtype) : nullptr;
    std::vector<uint64_t> rp_slice;
    uint64_t* d_rp = nullptr;
    if (A->space == ARGCSR_HOST) {
        rp_slice.resize(n + 1);
        for (uint64_t i = 0; i <= n; ++i) rp_slice[i] = rp_host[R.r0 + i] - a;
        v.row_pointers = rp_slice.data();
    } else {
        CUDA_OK(cudaMallocAsync(&d_rp, (n + 1) * sizeof(uint64_t), R.cs));
        k_rebase<<<grid_of(n + 1), 256, 0, R.cs>>>(d_rp, A->row_pointers + R.r0, n + 1);
        LAUNCH_OK("k_rebase");
        v.row_pointers = d_rp;
    }
    const argcsr_status st = argcsr_dev_convert_ex(&v, tpg, dcs, R.device, R.cs, flags, &R.m);
    if (d_rp) cudaFreeAsync(d_rp, R.cs);
    if (st != ARGCSR_OK) fail(st, last_error());
}

// Host copies of the slice's rebased row pointers and columns (planning).
void slice_host_arrays(const argcsr_csr_view* A, const std::vector<uint64_t>& rp_host, uint64_t r0, uint64_t r1,
                       std::vector<uint64_t>& rp, std::vector<int32_t>& cols, cudaStream_t s) {
    const uint64_t a = rp_host[r0], b = rp_host[r1];
    rp.resize(r1 - r0 + 1);
    for (uint64_t i = 0; i <= r1 - r0; ++i) rp[i] = rp_host[r0 + i] - a;
    cols.resize(b - a);
    if (b == a) return;
    if (A->space == ARGCSR_HOST) {
        std::memcpy(cols.data(), A->columns + a, (b - a) * sizeof(int32_t));
    } else {
        CUDA_OK(cudaMemcpyAsync(cols.data(), A->columns + a, (b - a) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
    }
}

std::vector<uint64_t> group_first_rows(const argcsr_dev* m, cudaStream_t s) {
    std::vector<GroupDesc> g(m->num_groups + 1);
    CUDA_OK(cudaMemcpyAsync(g.data(), m->groups, g.size() * sizeof(GroupDesc), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    std::vector<uint64_t> f(g.size());
    for (size_t i = 0; i < g.size(); ++i) f[i] = g[i].first_row;
    f.back() = m->num_rows;
    return f;
}

void alloc_rank_state(argcsr_mgpu* h, MgRank& R) {
    CUDA_OK(cudaEventCreateWithFlags(&R.ev_spmv, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&R.ev_red, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&R.ev_gath, cudaEventDisableTiming));
    R.part_len = 3 * norm_slots(R.m);
    CUDA_OK(cudaMalloc(&R.part, (R.part_len + norm_scratch_len(R.part_len) + 1) * sizeof(double)));
    CUDA_OK(cudaMalloc(&R.s2, 2 * sizeof(double)));
    CUDA_OK(cudaMemset(R.s2, 0, 2 * sizeof(double)));
    const size_t es = esize(h->dtype);
    if (h->exchange != ARGCSR_EXCHANGE_P2P) {
        for (void*& x : R.X) CUDA_OK(cudaMalloc(&x, std::max<uint64_t>(h->num_cols, 1) * es));
        R.own_x = true;
    } else {
        // one block shared with the peers: x[2][num_cols] | flags[P] u64 | partial[2][P] f64
        const size_t xb = ((h->num_cols * es + 255) / 256) * 256;
        R.off_x[0] = 0;
        R.off_x[1] = xb;
        R.off_flags = 2 * xb;
        R.off_partial = R.off_flags + ((size_t(h->nranks) * 8 + 255) / 256) * 256;
        R.pbytes = R.off_partial + 2 * size_t(h->nranks) * 8;
        CUDA_OK(cudaMalloc(&R.pblock, R.pbytes));
        CUDA_OK(cudaMemset(R.pblock, 0, R.pbytes));
        if (!h->single_process) {
            cudaIpcMemHandle_t ih;
            CUDA_OK(cudaIpcGetMemHandle(&ih, R.pblock));
            std::memcpy(R.ipc, &ih, 64);
        }
        R.X[0] = static_cast<char*>(R.pblock) + R.off_x[0];
        R.X[1] = static_cast<char*>(R.pblock) + R.off_x[1];
        R.own_x = false;
        R.peer_base.assign(h->nranks, nullptr);
    }
}

// p2p: peers' block addresses (and which of their rows each peer reads).
void connect_peers(argcsr_mgpu* h, MgRank& R, const std::vector<void*>& bases,
                   const std::vector<uint64_t>& need_all) {
    const int P = h->nranks;
    R.peers.clear();
    R.peer_rows.clear();
    for (int q = 0; q < P; ++q) {
        if (q == R.rank) continue;
        R.peers.push_back(q);
        R.peer_base[q] = bases[q];
        // rows q reads from me, [lo, hi) global -> local
        const uint64_t lo = need_all[(uint64_t(q) * P + R.rank) * 2], hi = need_all[(uint64_t(q) * P + R.rank) * 2 + 1];
        if (hi > lo) {
            R.peer_rows.push_back(std::max(lo, R.r0) - R.r0);
            R.peer_rows.push_back(std::min(hi, R.r1) - R.r0);
        } else {
            R.peer_rows.push_back(0);
            R.peer_rows.push_back(0);
        }
    }
    if (R.peers.size() > kMaxPeers) fail(ARGCSR_E_UNSUPPORTED, "the p2p exchange supports at most 8 GPUs");
    R.peer_y.assign(R.peers.size(), nullptr);
}

std::vector<uint64_t> need_ranges(const MgRank& R, int P) {
    std::vector<uint64_t> need(2 * size_t(P), 0);
    for (int p = 0; p < P; ++p)
        if (!R.need_rows[p].empty()) {
            need[2 * p] = R.need_rows[p].front();
            need[2 * p + 1] = uint64_t(R.need_rows[p].back()) + 1;
        }
    return need;
}

// Halo buffers from the per-owner receive lists and the per-peer send lists.
template <typename T>
void build_halo_buffers(MgRank& R, const std::vector<std::vector<uint32_t>>& send_lists) {
    std::vector<uint32_t> send, recv;
    R.send_counts.assign(send_lists.size(), 0);
    R.recv_counts.assign(send_lists.size(), 0);
    for (size_t p = 0; p < send_lists.size(); ++p) {
        R.send_counts[p] = send_lists[p].size();
        for (uint32_t g : send_lists[p]) send.push_back(g - uint32_t(R.r0));
        R.recv_counts[p] = R.need_rows[p].size();
        recv.insert(recv.end(), R.need_rows[p].begin(), R.need_rows[p].end());
    }
    R.nsend = send.size();
    R.nrecv = recv.size();
    CUDA_OK(cudaMalloc(&R.send_rows, std::max<size_t>(send.size(), 1) * 4));
    CUDA_OK(cudaMalloc(&R.recv_rows, std::max<size_t>(recv.size(), 1) * 4));
    CUDA_OK(cudaMalloc(&R.send_buf, std::max<size_t>(send.size(), 1) * sizeof(T)));
    CUDA_OK(cudaMalloc(&R.recv_buf, std::max<size_t>(recv.size(), 1) * sizeof(T)));
    if (!send.empty()) CUDA_OK(cudaMemcpy(R.send_rows, send.data(), send.size() * 4, cudaMemcpyHostToDevice));
    if (!recv.empty()) CUDA_OK(cudaMemcpy(R.recv_rows, recv.data(), recv.size() * 4, cudaMemcpyHostToDevice));
}

// The exchange the ranks agree on (every rank sees the same counts matrix).
argcsr_exchange resolve_exchange(argcsr_exchange asked, const std::vector<uint64_t>& counts_matrix, int P,
                                 uint64_t num_rows) {
    if (P == 1) return ARGCSR_EXCHANGE_NONE;
    if (asked != ARGCSR_EXCHANGE_AUTO) return asked;
    uint64_t halo = 0;
    for (uint64_t c : counts_matrix) halo += c;
    const uint64_t allgather = uint64_t(P - 1) * num_rows;  // rows received over all ranks
    return halo * 4 < allgather ? ARGCSR_EXCHANGE_HALO : ARGCSR_EXCHANGE_ALLGATHER;
}

// ------------------------------------------------------------ the step
struct Streams {
    const void* const* v;
    cudaStream_t operator[](size_t i) const { return v ? static_cast<cudaStream_t>(const_cast<void*>(v[i])) : nullptr; }
};

// Exchange of x (full length, this rank's slice already in place) on the
// collective streams of every local rank; `full`: every row (halo modes
// otherwise move only the rows others read).
template <typename T>
void exchange_nccl(argcsr_mgpu* h, void* const* xs, bool full) {
    const auto& api = nccl();
    const ncclDataType_t ty = nccl_type(h->dtype);
    const bool halo = h->exchange == ARGCSR_EXCHANGE_HALO && !full;
    if (halo) {
        for (size_t i = 0; i < h->r.size(); ++i) {
            MgRank& R = h->r[i];
            CUDA_OK(cudaSetDevice(R.device));
            gather_rows<T>(R.send_buf, static_cast<T*>(xs[i]) + R.r0, R.send_rows, R.nsend, R.cs);
        }
        {
            NcclGroup g;
            for (size_t i = 0; i < h->r.size(); ++i) {
                MgRank& R = h->r[i];
                uint64_t so = 0, ro = 0;
                for (int p = 0; p < h->nranks; ++p) {
                    if (R.send_counts[p])
                        NCCL_OK(api.Send(static_cast<T*>(R.send_buf) + so, R.send_counts[p], ty, p, R.comm, R.cs));
                    if (R.recv_counts[p])
                        NCCL_OK(api.Recv(static_cast<T*>(R.recv_buf) + ro, R.recv_counts[p], ty, p, R.comm, R.cs));
                    so += R.send_counts[p];
                    ro += R.recv_counts[p];
                }
            }
        }
        for (size_t i = 0; i < h->r.size(); ++i) {
            MgRank& R = h->r[i];
            CUDA_OK(cudaSetDevice(R.device));
            scatter_rows<T>(xs[i], R.recv_rows, R.recv_buf, R.nrecv, R.cs);
        }
        return;
    }
    NcclGroup g;
    const bool equal = equal_slices(h);
    for (size_t i = 0; i < h->r.size(); ++i) {
        MgRank& R = h->r[i];
        T* x = static_cast<T*>(xs[i]);
        if (equal) {
            NCCL_OK(api.AllGather(x + R.r0, x, R.r1 - R.r0, ty, R.comm, R.cs));
        } else {
            for (int p = 0; p < h->nranks; ++p) {
                T* seg = x + h->bounds[p];
                NCCL_OK(api.Broadcast(seg, seg, h->bounds[p + 1] - h->bounds[p], ty, p, R.comm, R.cs));
            }
        }
    }
}

void poll_comms(argcsr_mgpu* h) {
    for (MgRank& R : h->r) {
        if (!R.comm) continue;
        ncclResult_t e = ncclSuccess;
        NCCL_OK(nccl().CommGetAsyncError(R.comm, &e));
        if (e != ncclSuccess && e != ncclInProgress)
            fail(ARGCSR_E_NCCL, std::string("NCCL communicator error (rank ") + std::to_string(R.rank) +
                                    "): " + nccl().GetErrorString(e));
    }
}

template <typename T>
void step_nccl(argcsr_mgpu* h, bool last, Streams st) {
    const uint64_t k = h->k;
    const bool first = k == h->k0;
    const size_t es = sizeof(T);
    std::vector<void*> xout(h->r.size());
    for (size_t i = 0; i < h->r.size(); ++i) {
        MgRank& R = h->r[i];
        CUDA_OK(cudaSetDevice(R.device));
        const cudaStream_t s = st[i];
        void* xin = R.X[k % 2];
        xout[i] = R.X[(k + 1) % 2];
        void* y = static_cast<char*>(xout[i]) + R.r0 * es;
        SpmvExtra ex;
        if (h->normalize && !first) {
            CUDA_OK(cudaStreamWaitEvent(s, R.ev_red, 0));
            ex.x_scale = R.comm ? R.s2 + 1 : R.s2;
            ex.scale_is_norm2 = true;
        }
        SpmvOrder order(R.m, s);
        const uint64_t S = norm_slots(R.m), G = R.m->num_groups;
        const bool overlap = h->nranks > 1 && R.gb > R.ga;
        uint64_t regions = 1;
        ex.norm_part = h->normalize ? R.part : nullptr;
        if (overlap) {
            spmv_launch(R.m, xin, y, R.ga, R.gb, s, ex);                 // interior: own x rows only
            if (!first) CUDA_OK(cudaStreamWaitEvent(s, R.ev_gath, 0));  // x_k complete
            SpmvExtra e1 = ex, e2 = ex;
            if (h->normalize) e1.norm_part = R.part + S, e2.norm_part = R.part + 2 * S;
            spmv_launch(R.m, xin, y, 0, R.ga, s, e1);
            e2.reuse_x = R.ga > 0;  // x' gathered by the previous (fresh) boundary launch
            spmv_launch(R.m, xin, y, R.gb, G, s, e2);
            regions = 3;
            // groups of an empty range launch no CTA: their partials are stale
            if (h->normalize && R.ga == 0) CUDA_OK(cudaMemsetAsync(R.part + S, 0, S * sizeof(double), s));
            if (h->normalize && R.gb == G) CUDA_OK(cudaMemsetAsync(R.part + 2 * S, 0, S * sizeof(double), s));
        } else {
            if (!first && R.comm) CUDA_OK(cudaStreamWaitEvent(s, R.ev_gath, 0));
            spmv_launch(R.m, xin, y, 0, G, s, ex);
        }
        if (h->normalize) norm_reduce(R.part, regions * S, R.s2, s, R.part + R.part_len);
        order.done();
        CUDA_OK(cudaEventRecord(R.ev_spmv, s));
        CUDA_OK(cudaStreamWaitEvent(R.cs, R.ev_spmv, 0));
    }
    if (h->r[0].comm) {  // (a one-rank communicator still runs the collectives: tests, bench)
        if (h->normalize) {
            {
                NcclGroup g;
                for (MgRank& R : h->r) NCCL_OK(nccl().AllReduce(R.s2, R.s2 + 1, 1, ncclFloat64, ncclSum, R.comm, R.cs));
            }
        }
        for (MgRank& R : h->r) {
            CUDA_OK(cudaSetDevice(R.device));
            CUDA_OK(cudaEventRecord(R.ev_red, R.cs));
        }
        exchange_nccl<T>(h, xout.data(), last);
        for (MgRank& R : h->r) {
            CUDA_OK(cudaSetDevice(R.device));
            CUDA_OK(cudaEventRecord(R.ev_gath, R.cs));
        }
    } else {
        for (MgRank& R : h->r) {
            CUDA_OK(cudaSetDevice(R.device));
            CUDA_OK(cudaEventRecord(R.ev_red, R.cs));
            CUDA_OK(cudaEventRecord(R.ev_gath, R.cs));
        }
    }
}

template <typename T>
void step_p2p(argcsr_mgpu* h, bool last, Streams st) {
    const uint64_t k = h->k;
    const int P = h->nranks;
    const size_t es = sizeof(T);
    const int b = int(k % 2), nb = int((k + 1) % 2);
    for (size_t i = 0; i < h->r.size(); ++i) {
        MgRank& R = h->r[i];
        CUDA_OK(cudaSetDevice(R.device));
        const cudaStream_t s = st[i];
        char* blk = static_cast<char*>(R.pblock);
        uint64_t* flags = reinterpret_cast<uint64_t*>(blk + R.off_flags);
        double* partial = reinterpret_cast<double*>(blk + R.off_partial);
        // x_k complete here, and every peer is done reading buffer nb
        if (!R.peers.empty() && k > 0) peer_wait(flags, uint32_t(P), k, s);
        SpmvExtra ex;
        if (h->normalize && k > h->k0) {
            norm_reduce(partial + size_t(b) * P, uint64_t(P), R.s2, s);  // same order on every rank
            ex.x_scale = R.s2;
            ex.scale_is_norm2 = true;
        }
        for (size_t q = 0; q < R.peers.size(); ++q)
            R.peer_y[q] = static_cast<char*>(R.peer_base[R.peers[q]]) + R.off_x[nb] + R.r0 * es;
        ex.peer_y = R.peer_y.data();
        ex.npeers = uint32_t(R.peers.size());
        ex.peer_rows = last ? nullptr : R.peer_rows.data();
        double* own = partial + size_t(nb) * P + R.rank;
        ex.norm_part = h->normalize ? R.part : nullptr;
        {
            SpmvOrder order(R.m, s);
            spmv_launch(R.m, R.X[b], static_cast<char*>(R.X[nb]) + R.r0 * es, 0, R.m->num_groups, s, ex);
            if (h->normalize) norm_reduce(R.part, norm_slots(R.m), own, s, R.part + R.part_len);
            order.done();
        }
        if (!R.peers.empty()) {
            uint64_t* pf[kMaxPeers];
            double* pp[kMaxPeers];
            for (size_t q = 0; q < R.peers.size(); ++q) {
                char* pb = static_cast<char*>(R.peer_base[R.peers[q]]);
                pf[q] = reinterpret_cast<uint64_t*>(pb + R.off_flags) + R.rank;
                pp[q] = reinterpret_cast<double*>(pb + R.off_partial) + size_t(nb) * P + R.rank;
            }
            peer_signal(pf, uint32_t(R.peers.size()), k + 1, h->normalize ? own : nullptr,
                        h->normalize ? pp : nullptr, s);
        }
        k_set_u64<<<1, 1, 0, s>>>(flags + R.rank, k + 1);  // own slot: the wait covers all P slots
        LAUNCH_OK("k_set_u64");
    }
}

template <typename T>
void finish_typed(argcsr_mgpu* h, double* lambda, void* const* x_out, Streams st) {
    const uint64_t k = h->k;
    const int P = h->nranks;
    const size_t es = sizeof(T);
    // NCCL halo: a run whose last step moved only the halo leaves the other
    // ranks' rows stale: assemble once.
    if (h->exchange == ARGCSR_EXCHANGE_HALO && !h->last_full && P > 1) {
        std::vector<void*> xs(h->r.size());
        for (size_t i = 0; i < h->r.size(); ++i) {
            MgRank& R = h->r[i];
            CUDA_OK(cudaSetDevice(R.device));
            CUDA_OK(cudaStreamWaitEvent(R.cs, R.ev_gath, 0));
            xs[i] = R.X[k % 2];
        }
        exchange_nccl<T>(h, xs.data(), true);
        for (MgRank& R : h->r) {
            CUDA_OK(cudaSetDevice(R.device));
            CUDA_OK(cudaEventRecord(R.ev_gath, R.cs));
        }
        h->last_full = true;
    }
    double lam = 0.0;
    for (size_t i = 0; i < h->r.size(); ++i) {
        MgRank& R = h->r[i];
        CUDA_OK(cudaSetDevice(R.device));
        const cudaStream_t s = st[i];
        const double* s2 = nullptr;
        if (h->exchange == ARGCSR_EXCHANGE_P2P) {
            char* blk = static_cast<char*>(R.pblock);
            if (!R.peers.empty() && k > 0) peer_wait(reinterpret_cast<uint64_t*>(blk + R.off_flags), uint32_t(P), k, s);
            if (h->normalize) {
                norm_reduce(reinterpret_cast<double*>(blk + R.off_partial) + size_t(k % 2) * P, uint64_t(P), R.s2, s);
                s2 = R.s2;
            }
        } else {
            CUDA_OK(cudaStreamWaitEvent(s, R.ev_gath, 0));
            if (h->normalize) s2 = R.comm ? R.s2 + 1 : R.s2;
        }
        if (x_out && x_out[i]) {
            if (h->normalize && k > h->k0) {
                k_scale_norm2<T><<<grid_of(h->num_cols), 256, 0, s>>>(static_cast<T*>(x_out[i]),
                                                                       static_cast<const T*>(R.X[k % 2]), s2,
                                                                       h->num_cols);
                LAUNCH_OK("k_scale_norm2");
            } else {
                CUDA_OK(cudaMemcpyAsync(x_out[i], R.X[k % 2], h->num_cols * es, cudaMemcpyDeviceToDevice, s));
            }
        }
        double v = 0.0;
        if (s2 && k > h->k0) CUDA_OK(cudaMemcpyAsync(&v, s2, sizeof v, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        if (i == 0) lam = std::sqrt(v);
    }
    if (lambda) *lambda = lam;
}

template <typename T>
void spmv_gather_typed(argcsr_mgpu* h, const void* const* x, void* const* out, Streams st) {
    const size_t es = sizeof(T);
    for (size_t i = 0; i < h->r.size(); ++i) {
        MgRank& R = h->r[i];
        CUDA_OK(cudaSetDevice(R.device));
        const cudaStream_t s = st[i];
        {
            SpmvOrder order(R.m, s);
            spmv_launch(R.m, x[i], static_cast<char*>(out[i]) + R.r0 * es, 0, R.m->num_groups, s);
            order.done();
        }
        CUDA_OK(cudaEventRecord(R.ev_spmv, s));
        CUDA_OK(cudaStreamWaitEvent(R.cs, R.ev_spmv, 0));
    }
    if (h->r[0].comm) exchange_nccl<T>(h, out, true);
    for (size_t i = 0; i < h->r.size(); ++i) {
        MgRank& R = h->r[i];
        CUDA_OK(cudaSetDevice(R.device));
        CUDA_OK(cudaEventRecord(R.ev_gath, R.cs));
        CUDA_OK(cudaStreamWaitEvent(st[i], R.ev_gath, 0));
    }
}

void check_view(const argcsr_csr_view* A, const char* who) {
    if (!A) fail(ARGCSR_E_PARAMETER, std::string(who) + ": null matrix");
    if (A->num_rows == 0) fail(ARGCSR_E_PARAMETER, "partition_groups: row_nnz must be nonempty");
    if (A->dtype != ARGCSR_F64 && A->dtype != ARGCSR_F32) fail(ARGCSR_E_PARAMETER, std::string(who) + ": unknown dtype");
    if (!A->row_pointers || (A->nnz && (!A->columns || !A->values)))
        fail(ARGCSR_E_PARAMETER, std::string(who) + ": null CSR array");
}

std::vector<uint64_t> host_row_pointers(const argcsr_csr_view* A) {
    std::vector<uint64_t> rp(A->num_rows + 1);
    if (A->space == ARGCSR_HOST) std::memcpy(rp.data(), A->row_pointers, rp.size() * sizeof(uint64_t));
    else CUDA_OK(cudaMemcpy(rp.data(), A->row_pointers, rp.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return rp;
}

template <typename T>
void setup_halo_single_process(argcsr_mgpu* h) {
    const int P = h->nranks;
    for (int p = 0; p < P; ++p) {
        std::vector<std::vector<uint32_t>> send(P);
        for (int q = 0; q < P; ++q)
            if (q != p) send[q] = h->r[q].need_rows[p];
        CUDA_OK(cudaSetDevice(h->r[p].device));
        build_halo_buffers<T>(h->r[p], send);
    }
}

}  // namespace

extern "C" {

argcsr_status argcsr_plan_interior(const uint64_t* rp, const int32_t* columns, uint64_t rows,
                                   const uint64_t* group_first, uint64_t num_groups, uint64_t r0, uint64_t r1,
                                   uint64_t* ga, uint64_t* gb) {
    return guarded([&] {
        if (!rp || (!columns && rp[rows] > rp[0]) || !group_first || !ga || !gb)
            fail(ARGCSR_E_PARAMETER, "argcsr_plan_interior: null argument");
        plan_interior(rp, columns, rows, group_first, num_groups, r0, r1, ga, gb);
    });
}

argcsr_status argcsr_plan_needed(const int32_t* columns, uint64_t nnz, uint64_t num_cols, const uint64_t* bounds,
                                 uint32_t parts, uint32_t self, uint64_t* counts, uint64_t* rows) {
    return guarded([&] {
        if ((!columns && nnz) || !bounds || !counts || parts == 0 || self >= parts)
            fail(ARGCSR_E_PARAMETER, "argcsr_plan_needed: bad argument");
        std::vector<uint64_t> b(bounds, bounds + parts + 1);
        const auto need = plan_needed(columns, nnz, num_cols, b, self);
        uint64_t o = 0;
        for (uint32_t p = 0; p < parts; ++p) {
            counts[p] = need[p].size();
            if (rows)
                for (uint32_t r : need[p]) rows[o++] = r;
        }
    });
}

argcsr_status argcsr_mgpu_unique_id(unsigned char id[ARGCSR_NCCL_ID_BYTES]) {
    return guarded([&] {
        if (!id) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_unique_id: null output");
        static_assert(sizeof(ncclUniqueId) == ARGCSR_NCCL_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        NCCL_OK(nccl().GetUniqueId(&u));
        std::memcpy(id, &u, sizeof u);
    });
}

argcsr_status argcsr_mgpu_create_rank(const argcsr_csr_view* A, int rank, int nranks, const unsigned char* nccl_id,
                                      uint64_t tpg, uint64_t dcs, int device, uint32_t flags, argcsr_exchange exchange,
                                      argcsr_mgpu** out) {
    return guarded([&] {
        if (!out) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_create_rank: null output");
        *out = nullptr;
        if (tpg == 0 || dcs == 0)
            fail(ARGCSR_E_PARAMETER, "partition_groups: threads_per_group and desired_chunk_size must be at least 1");
        check_view(A, "argcsr_mgpu_create_rank");
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_create_rank: bad rank");
        if (exchange < ARGCSR_EXCHANGE_AUTO || exchange > ARGCSR_EXCHANGE_P2P)
            fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_create_rank: unknown exchange");
        if (nranks > 1 && !nccl_id && exchange != ARGCSR_EXCHANGE_P2P)
            fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_create_rank: the NCCL exchanges need an ncclUniqueId");
        if (exchange == ARGCSR_EXCHANGE_P2P && nranks > 8) fail(ARGCSR_E_UNSUPPORTED, "p2p exchange: at most 8 GPUs");
        DeviceScope scope(device);
        std::unique_ptr<argcsr_mgpu, void (*)(argcsr_mgpu*)> h(new argcsr_mgpu, [](argcsr_mgpu* p) {
            free_handle(p, true);
        });
        h->nranks = nranks;
        h->dtype = A->dtype;
        h->num_rows = A->num_rows;
        h->num_cols = A->num_cols;
        h->r.resize(1);
        MgRank& R = h->r[0];
        R.device = device;
        R.rank = rank;
        CUDA_OK(cudaStreamCreateWithFlags(&R.cs, cudaStreamNonBlocking));
        const std::vector<uint64_t> rp = host_row_pointers(A);
        h->nnz = rp[A->num_rows] - rp[0];
        h->bounds = partition(rp.data(), A->num_rows, uint32_t(nranks));
        R.r0 = h->bounds[rank];
        R.r1 = h->bounds[rank + 1];
        {
            Phase ph("mgpu.convert_slice", R.cs, true);
            convert_slice(R, A, rp, tpg, dcs, flags);
        }
        if (nccl_id) {
            Phase ph("mgpu.nccl_init", R.cs, true);
            ncclUniqueId u;
            std::memcpy(&u, nccl_id, sizeof u);
            NCCL_OK(nccl().CommInitRank(&R.comm, nranks, u, rank));
        }
        const int P = nranks;
        std::vector<uint64_t> counts_matrix(size_t(P) * P, 0);
        if (P > 1) {
            Phase ph("mgpu.plan", R.cs, true);
            std::vector<uint64_t> srp;
            std::vector<int32_t> scols;
            slice_host_arrays(A, rp, R.r0, R.r1, srp, scols, R.cs);
            const std::vector<uint64_t> gf = group_first_rows(R.m, R.cs);
            plan_interior(srp.data(), scols.data(), R.r1 - R.r0, gf.data(), R.m->num_groups, R.r0, R.r1, &R.ga, &R.gb);
            R.need_rows = plan_needed(scols.data(), scols.size(), A->num_cols, h->bounds, uint32_t(rank));
            if (R.comm) {  // everyone's receive counts (row p of the matrix = rank p's counts)
                uint64_t* d = nullptr;
                CUDA_OK(cudaMalloc(&d, counts_matrix.size() * sizeof(uint64_t)));
                std::vector<uint64_t> mine(P);
                for (int p = 0; p < P; ++p) mine[p] = R.need_rows[p].size();
                CUDA_OK(cudaMemcpy(d + size_t(rank) * P, mine.data(), P * sizeof(uint64_t), cudaMemcpyHostToDevice));
                NCCL_OK(nccl().AllGather(d + size_t(rank) * P, d, P, ncclUint64, R.comm, R.cs));
                CUDA_OK(cudaMemcpyAsync(counts_matrix.data(), d, counts_matrix.size() * 8, cudaMemcpyDeviceToHost, R.cs));
                CUDA_OK(cudaStreamSynchronize(R.cs));
                cudaFree(d);
            }
        }
        h->exchange = resolve_exchange(exchange, counts_matrix, P, A->num_rows);
        alloc_rank_state(h.get(), R);
        if (h->exchange == ARGCSR_EXCHANGE_HALO) {
            // the rows every peer reads from me: grouped send/recv of the lists
            std::vector<std::vector<uint32_t>> send(P);
            uint32_t *dsend = nullptr, *drecv = nullptr;
            uint64_t tot_in = 0, tot_out = 0;
            for (int p = 0; p < P; ++p) {
                tot_in += counts_matrix[size_t(p) * P + rank];
                tot_out += R.need_rows[p].size();
            }
            CUDA_OK(cudaMalloc(&dsend, std::max<uint64_t>(tot_out, 1) * 4));
            CUDA_OK(cudaMalloc(&drecv, std::max<uint64_t>(tot_in, 1) * 4));
            std::vector<uint32_t> flat;
            for (int p = 0; p < P; ++p) flat.insert(flat.end(), R.need_rows[p].begin(), R.need_rows[p].end());
            if (!flat.empty()) CUDA_OK(cudaMemcpy(dsend, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice));
            {
                NcclGroup g;
                uint64_t so = 0, ro = 0;
                for (int p = 0; p < P; ++p) {
                    const uint64_t n_out = R.need_rows[p].size(), n_in = counts_matrix[size_t(p) * P + rank];
                    if (n_out) NCCL_OK(nccl().Send(dsend + so, n_out, ncclUint32, p, R.comm, R.cs));
                    if (n_in) NCCL_OK(nccl().Recv(drecv + ro, n_in, ncclUint32, p, R.comm, R.cs));
                    so += n_out;
                    ro += n_in;
                }
            }
            std::vector<uint32_t> got(tot_in);
            if (tot_in) CUDA_OK(cudaMemcpyAsync(got.data(), drecv, tot_in * 4, cudaMemcpyDeviceToHost, R.cs));
            CUDA_OK(cudaStreamSynchronize(R.cs));
            cudaFree(dsend);
            cudaFree(drecv);
            uint64_t o = 0;
            for (int p = 0; p < P; ++p) {
                const uint64_t n_in = counts_matrix[size_t(p) * P + rank];
                send[p].assign(got.begin() + o, got.begin() + o + n_in);
                o += n_in;
            }
            if (h->dtype == ARGCSR_F64) build_halo_buffers<double>(R, send);
            else build_halo_buffers<float>(R, send);
        } else if (h->exchange == ARGCSR_EXCHANGE_P2P && P > 1) {
            h->connected = false;
            if (R.comm) {  // IPC handles and need tables over NCCL
                unsigned char* d = nullptr;
                const size_t per = 64 + 16 * size_t(P);
                CUDA_OK(cudaMalloc(&d, per * P));
                std::vector<unsigned char> mine(per);
                std::memcpy(mine.data(), R.ipc, 64);
                const std::vector<uint64_t> need = need_ranges(R, P);
                std::memcpy(mine.data() + 64, need.data(), 16 * size_t(P));
                CUDA_OK(cudaMemcpy(d + per * rank, mine.data(), per, cudaMemcpyHostToDevice));
                NCCL_OK(nccl().AllGather(d + per * rank, d, per, ncclUint8, R.comm, R.cs));
                std::vector<unsigned char> all(per * P);
                CUDA_OK(cudaMemcpyAsync(all.data(), d, all.size(), cudaMemcpyDeviceToHost, R.cs));
                CUDA_OK(cudaStreamSynchronize(R.cs));
                cudaFree(d);
                std::vector<unsigned char> handles(64 * size_t(P));
                std::vector<uint64_t> need_all(2 * size_t(P) * P);
                for (int p = 0; p < P; ++p) {
                    std::memcpy(handles.data() + 64 * p, all.data() + per * p, 64);
                    std::memcpy(need_all.data() + 2 * size_t(P) * p, all.data() + per * p + 64, 16 * size_t(P));
                }
                const argcsr_status st = argcsr_mgpu_p2p_connect(h.get(), handles.data(), need_all.data());
                if (st != ARGCSR_OK) fail(st, last_error());
            }
        }
        CUDA_OK(cudaDeviceSynchronize());
        *out = h.release();
    });
}

argcsr_status argcsr_mgpu_create(const argcsr_csr_view* A, int ngpus, const int* devices, uint64_t tpg, uint64_t dcs,
                                 argcsr_exchange exchange, argcsr_mgpu** out) {
    return guarded([&] {
        if (!out) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_create: null output");
        *out = nullptr;
        if (tpg == 0 || dcs == 0)
            fail(ARGCSR_E_PARAMETER, "partition_groups: threads_per_group and desired_chunk_size must be at least 1");
        check_view(A, "argcsr_mgpu_create");
        if (ngpus < 1 || !devices) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_create: no devices");
        if (exchange < ARGCSR_EXCHANGE_AUTO || exchange > ARGCSR_EXCHANGE_P2P)
            fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_create: unknown exchange");
        if (exchange == ARGCSR_EXCHANGE_P2P && ngpus > 8) fail(ARGCSR_E_UNSUPPORTED, "p2p exchange: at most 8 GPUs");
        std::vector<int> dl(devices, devices + ngpus);
        std::vector<int> sorted = dl;
        std::sort(sorted.begin(), sorted.end());
        const bool dup = std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end();
        if (dup && exchange != ARGCSR_EXCHANGE_P2P)
            fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_create: a device listed twice needs ARGCSR_EXCHANGE_P2P");
        DeviceScope scope(dl[0]);
        std::unique_ptr<argcsr_mgpu, void (*)(argcsr_mgpu*)> h(new argcsr_mgpu, [](argcsr_mgpu* p) {
            free_handle(p, true);
        });
        const int P = ngpus;
        h->nranks = P;
        h->single_process = true;
        h->dtype = A->dtype;
        h->num_rows = A->num_rows;
        h->num_cols = A->num_cols;
        const std::vector<uint64_t> rp = host_row_pointers(A);
        h->nnz = rp[A->num_rows] - rp[0];
        h->bounds = partition(rp.data(), A->num_rows, uint32_t(P));
        h->r.resize(P);
        std::vector<uint64_t> counts_matrix(size_t(P) * P, 0);
        for (int p = 0; p < P; ++p) {
            MgRank& R = h->r[p];
            R.device = dl[p];
            R.rank = p;
            CUDA_OK(cudaSetDevice(R.device));
            CUDA_OK(cudaStreamCreateWithFlags(&R.cs, cudaStreamNonBlocking));
            R.r0 = h->bounds[p];
            R.r1 = h->bounds[p + 1];
            convert_slice(R, A, rp, tpg, dcs, 0u);
            if (P > 1) {
                std::vector<uint64_t> srp;
                std::vector<int32_t> scols;
                slice_host_arrays(A, rp, R.r0, R.r1, srp, scols, R.cs);
                const std::vector<uint64_t> gf = group_first_rows(R.m, R.cs);
                plan_interior(srp.data(), scols.data(), R.r1 - R.r0, gf.data(), R.m->num_groups, R.r0, R.r1, &R.ga,
                              &R.gb);
                R.need_rows = plan_needed(scols.data(), scols.size(), A->num_cols, h->bounds, uint32_t(p));
                for (int q = 0; q < P; ++q) counts_matrix[size_t(p) * P + q] = R.need_rows[q].size();
            }
        }
        h->exchange = resolve_exchange(exchange, counts_matrix, P, A->num_rows);
        if (P > 1 && h->exchange != ARGCSR_EXCHANGE_P2P) {
            std::vector<ncclComm_t> comms(P);
            NCCL_OK(nccl().CommInitAll(comms.data(), P, dl.data()));
            for (int p = 0; p < P; ++p) h->r[p].comm = comms[p];
        }
        for (MgRank& R : h->r) {
            CUDA_OK(cudaSetDevice(R.device));
            alloc_rank_state(h.get(), R);
        }
        if (h->exchange == ARGCSR_EXCHANGE_HALO) {
            if (h->dtype == ARGCSR_F64) setup_halo_single_process<double>(h.get());
            else setup_halo_single_process<float>(h.get());
        } else if (h->exchange == ARGCSR_EXCHANGE_P2P && P > 1) {
            std::vector<void*> bases(P);
            std::vector<uint64_t> need_all(2 * size_t(P) * P);
            for (int p = 0; p < P; ++p) {
                bases[p] = h->r[p].pblock;
                const std::vector<uint64_t> need = need_ranges(h->r[p], P);
                std::copy(need.begin(), need.end(), need_all.begin() + 2 * size_t(P) * p);
            }
            for (int p = 0; p < P; ++p)
                for (int q = 0; q < P; ++q)
                    if (p != q && h->r[p].device != h->r[q].device) {
                        CUDA_OK(cudaSetDevice(h->r[p].device));
                        const cudaError_t e = cudaDeviceEnablePeerAccess(h->r[q].device, 0);
                        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CUDA_OK(e);
                        cudaGetLastError();
                    }
            for (MgRank& R : h->r) connect_peers(h.get(), R, bases, need_all);
        }
        for (MgRank& R : h->r) {
            CUDA_OK(cudaSetDevice(R.device));
            CUDA_OK(cudaDeviceSynchronize());
        }
        *out = h.release();
    });
}

argcsr_status argcsr_mgpu_p2p_export(const argcsr_mgpu* h, unsigned char handle[64], uint64_t* need) {
    return guarded([&] {
        if (!h || !handle || !need) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_p2p_export: null argument");
        if (h->exchange != ARGCSR_EXCHANGE_P2P || h->r.size() != 1)
            fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_p2p_export: needs a one-GPU handle with ARGCSR_EXCHANGE_P2P");
        const MgRank& R = h->r[0];
        std::memcpy(handle, R.ipc, 64);
        std::vector<uint64_t> nd(2 * size_t(h->nranks), 0);
        if (h->nranks > 1) nd = need_ranges(R, h->nranks);
        std::memcpy(need, nd.data(), nd.size() * sizeof(uint64_t));
    });
}

argcsr_status argcsr_mgpu_p2p_connect(argcsr_mgpu* h, const unsigned char* handles, const uint64_t* need_all) {
    return guarded([&] {
        if (!h || !handles || !need_all) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_p2p_connect: null argument");
        if (h->exchange != ARGCSR_EXCHANGE_P2P || h->r.size() != 1)
            fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_p2p_connect: needs a one-GPU handle with ARGCSR_EXCHANGE_P2P");
        if (h->connected) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_p2p_connect: already connected");
        MgRank& R = h->r[0];
        DeviceScope scope(R.device);
        const int P = h->nranks;
        std::vector<void*> bases(P, nullptr);
        for (int p = 0; p < P; ++p) {
            if (p == R.rank) continue;
            cudaIpcMemHandle_t ih;
            std::memcpy(&ih, handles + 64 * size_t(p), 64);
            void* ptr = nullptr;
            CUDA_OK(cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess));
            R.opened.push_back(ptr);
            bases[p] = ptr;
        }
        std::vector<uint64_t> na(need_all, need_all + 2 * size_t(P) * P);
        connect_peers(h, R, bases, na);
        h->connected = true;
    });
}

argcsr_status argcsr_mgpu_info(const argcsr_mgpu* h, argcsr_mgpu_info_t* info) {
    return guarded([&] {
        if (!h || !info) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_info: null argument");
        const MgRank& R = h->r[0];
        info->rank = R.rank;
        info->nranks = h->nranks;
        info->nlocal = int32_t(h->r.size());
        info->exchange = h->exchange;
        info->num_rows = h->num_rows;
        info->num_cols = h->num_cols;
        info->nnz = h->nnz;
        info->row_begin = R.r0;
        info->row_end = R.r1;
        info->interior_begin = R.ga;
        info->interior_end = R.gb;
        info->halo_recv_rows = R.nrecv;
        info->step = h->k;
    });
}

argcsr_status argcsr_mgpu_local(const argcsr_mgpu* h, int i, argcsr_dev** slice) {
    return guarded([&] {
        if (!h || !slice || i < 0 || size_t(i) >= h->r.size()) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_local: bad argument");
        *slice = h->r[i].m;
    });
}

argcsr_status argcsr_mgpu_begin(argcsr_mgpu* h, const void* const* x0, int normalize, void* const* streams) {
    return guarded([&] {
        if (!h || !x0) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_begin: null argument");
        if (!h->connected) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_begin: p2p peers not connected");
        Streams st{streams};
        const size_t es = esize(h->dtype);
        for (size_t i = 0; i < h->r.size(); ++i) {
            MgRank& R = h->r[i];
            DeviceScope scope(R.device);
            if (!x0[i]) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_begin: null x0");
            // the previous run's exchange into this buffer is complete first
            CUDA_OK(cudaStreamWaitEvent(st[i], R.ev_gath, 0));
            if (h->exchange == ARGCSR_EXCHANGE_P2P && !R.peers.empty() && h->k > 0)
                peer_wait(reinterpret_cast<uint64_t*>(static_cast<char*>(R.pblock) + R.off_flags),
                          uint32_t(h->nranks), h->k, st[i]);
            CUDA_OK(cudaMemcpyAsync(R.X[h->k % 2], x0[i], h->num_cols * es, cudaMemcpyDeviceToDevice, st[i]));
        }
        h->normalize = normalize != 0;
        h->k0 = h->k;
        h->begun = true;
        h->last_full = true;
    });
}

argcsr_status argcsr_mgpu_step(argcsr_mgpu* h, int last, void* const* streams) {
    return guarded([&] {
        if (!h) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_step: null handle");
        if (!h->begun) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_step: call argcsr_mgpu_begin first");
        poll_comms(h);
        nvtxRangePushA("argcsr_mgpu_step");
        int prev = -1;
        CUDA_OK(cudaGetDevice(&prev));
        struct Restore {
            int d;
            ~Restore() {
                cudaSetDevice(d);
                nvtxRangePop();
            }
        } restore{prev};
        Streams st{streams};
        const bool full = last != 0;
        if (h->exchange == ARGCSR_EXCHANGE_P2P) {
            if (h->dtype == ARGCSR_F64) step_p2p<double>(h, full, st);
            else step_p2p<float>(h, full, st);
        } else {
            if (h->dtype == ARGCSR_F64) step_nccl<double>(h, full, st);
            else step_nccl<float>(h, full, st);
        }
        h->last_full = full;
        ++h->k;
    });
}

argcsr_status argcsr_mgpu_finish(argcsr_mgpu* h, double* lambda, void* const* x_out, void* const* streams) {
    return guarded([&] {
        if (!h) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_finish: null handle");
        if (!h->begun) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_finish: call argcsr_mgpu_begin first");
        int prev = -1;
        CUDA_OK(cudaGetDevice(&prev));
        struct Restore {
            int d;
            ~Restore() { cudaSetDevice(d); }
        } restore{prev};
        Streams st{streams};
        if (h->dtype == ARGCSR_F64) finish_typed<double>(h, lambda, x_out, st);
        else finish_typed<float>(h, lambda, x_out, st);
        poll_comms(h);
    });
}

argcsr_status argcsr_mgpu_wait(argcsr_mgpu* h, void* const* streams) {
    return guarded([&] {
        if (!h) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_wait: null handle");
        int prev = -1;
        CUDA_OK(cudaGetDevice(&prev));
        struct Restore {
            int d;
            ~Restore() { cudaSetDevice(d); }
        } restore{prev};
        Streams st{streams};
        for (size_t i = 0; i < h->r.size(); ++i) {
            MgRank& R = h->r[i];
            CUDA_OK(cudaSetDevice(R.device));
            if (h->exchange == ARGCSR_EXCHANGE_P2P) {
                if (!R.peers.empty() && h->k > 0)
                    peer_wait(reinterpret_cast<uint64_t*>(static_cast<char*>(R.pblock) + R.off_flags),
                              uint32_t(h->nranks), h->k, st[i]);
            } else {
                CUDA_OK(cudaStreamWaitEvent(st[i], R.ev_gath, 0));
            }
        }
    });
}

argcsr_status argcsr_mgpu_spmv_gather(argcsr_mgpu* h, const void* const* x, void* const* out, void* const* streams) {
    return guarded([&] {
        if (!h || !x || !out) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_spmv_gather: null argument");
        if (h->nranks > 1 && !h->r[0].comm)
            fail(ARGCSR_E_UNSUPPORTED, "argcsr_mgpu_spmv_gather: needs an NCCL communicator (create with an id)");
        poll_comms(h);
        int prev = -1;
        CUDA_OK(cudaGetDevice(&prev));
        struct Restore {
            int d;
            ~Restore() { cudaSetDevice(d); }
        } restore{prev};
        Streams st{streams};
        if (h->dtype == ARGCSR_F64) spmv_gather_typed<double>(h, x, out, st);
        else spmv_gather_typed<float>(h, x, out, st);
    });
}

argcsr_status argcsr_mgpu_power_iteration(argcsr_mgpu* h, int iters, void* x_host_io, double* lambda_out) {
    return guarded([&] {
        if (!h || !x_host_io || iters < 1) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_power_iteration: bad argument");
        const size_t es = esize(h->dtype);
        std::vector<void*> x0(h->r.size()), xo(h->r.size()), streams(h->r.size(), nullptr);
        struct Tmp {
            std::vector<void*>* v;
            std::vector<int> dev;
            ~Tmp() {
                for (size_t i = 0; i < v->size(); ++i)
                    if ((*v)[i]) {
                        cudaSetDevice(dev[i]);
                        cudaFree((*v)[i]);
                    }
            }
        } tmp{&x0, {}};
        for (size_t i = 0; i < h->r.size(); ++i) {
            DeviceScope scope(h->r[i].device);
            tmp.dev.push_back(h->r[i].device);
            CUDA_OK(cudaMalloc(&x0[i], std::max<uint64_t>(h->num_cols, 1) * es));
            CUDA_OK(cudaMemcpy(x0[i], x_host_io, h->num_cols * es, cudaMemcpyHostToDevice));
            xo[i] = x0[i];
        }
        argcsr_status st = argcsr_mgpu_begin(h, x0.data(), 1, streams.data());
        for (int i = 0; st == ARGCSR_OK && i < iters; ++i) st = argcsr_mgpu_step(h, i == iters - 1, streams.data());
        if (st == ARGCSR_OK) st = argcsr_mgpu_finish(h, lambda_out, xo.data(), streams.data());
        if (st != ARGCSR_OK) fail(st, last_error());
        DeviceScope scope(h->r[0].device);
        CUDA_OK(cudaMemcpy(x_host_io, xo[0], h->num_cols * es, cudaMemcpyDeviceToHost));
    });
}

argcsr_status argcsr_mgpu_check(argcsr_mgpu* h) {
    return guarded([&] {
        if (!h) fail(ARGCSR_E_PARAMETER, "argcsr_mgpu_check: null handle");
        poll_comms(h);
    });
}

void argcsr_mgpu_free(argcsr_mgpu* h) { free_handle(h, false); }

}  // extern "C"
