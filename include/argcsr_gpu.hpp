// argcsr_gpu.hpp — C++ host API over the C-ABI (argcsr_gpu.h), mirroring the
// reference library's `namespace argcsr` (proj/include/argcsr/*.hpp): the same
// type and field names, value semantics for host objects, and the same
// exception classes (proj/include/argcsr/errors.hpp:9-66).  The one
// difference is ownership of the converted matrix: argcsr_from_csr returns a
// device-resident DeviceArgCsr (move-only RAII over argcsr_dev*); to_host()
// gives the reference's ArgCsrMatrix bit-for-bit.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "argcsr_gpu.h"

namespace argcsr_b200 {

// ------------------------------------------------------------ errors.hpp:9-66
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
class BoundsError : public Error { public: using Error::Error; };
class DimensionError : public Error { public: using Error::Error; };
class ParameterError : public Error { public: using Error::Error; };
class InternalError : public Error { public: using Error::Error; };
class ParseError : public Error { public: using Error::Error; };
class UnsupportedError : public Error { public: using Error::Error; };
class FormatError : public Error { public: using Error::Error; };
class IoError : public Error { public: using Error::Error; };
class CorrectnessError : public Error { public: using Error::Error; };
// Device-side failures are internal errors of the library.
class CudaError : public InternalError { public: using InternalError::InternalError; };
class NcclError : public InternalError { public: using InternalError::InternalError; };
class OutOfMemoryError : public InternalError { public: using InternalError::InternalError; };

[[noreturn]] inline void throw_status(argcsr_status s, const std::string& msg) {
    switch (s) {
        case ARGCSR_E_PARAMETER: throw ParameterError(msg);
        case ARGCSR_E_DIMENSION: throw DimensionError(msg);
        case ARGCSR_E_BOUNDS: throw BoundsError(msg);
        case ARGCSR_E_CUDA: throw CudaError(msg);
        case ARGCSR_E_NCCL: throw NcclError(msg);
        case ARGCSR_E_OOM: throw OutOfMemoryError(msg);
        case ARGCSR_E_FORMAT: throw FormatError(msg);
        case ARGCSR_E_IO: throw IoError(msg);
        case ARGCSR_E_PARSE: throw ParseError(msg);
        case ARGCSR_E_UNSUPPORTED: throw UnsupportedError(msg);
        default: throw InternalError(msg);
    }
}

inline void check(argcsr_status s) {
    if (s != ARGCSR_OK) throw_status(s, argcsr_last_error());
}

// --------------------------------------------------------------- core.hpp
using index_t = std::int32_t;
inline constexpr index_t kPaddingColumn = -1;

struct CsrMatrix {
    std::size_t num_rows = 0;
    std::size_t num_cols = 0;
    std::vector<double> values;
    std::vector<index_t> columns;
    std::vector<std::size_t> row_pointers;

    std::size_t nnz() const { return values.size(); }
    bool operator==(const CsrMatrix&) const = default;
};

using DenseVector = std::vector<double>;

// -------------------------------------------------------------- argcsr.hpp
struct GroupInfo {
    std::size_t first_row = 0;
    std::size_t size = 0;
    std::size_t offset = 0;
    std::size_t chunk_size = 0;
    bool operator==(const GroupInfo&) const = default;
};

struct ArgCsrMatrix {
    std::size_t num_rows = 0;
    std::size_t num_cols = 0;
    std::size_t threads_per_group = 0;
    std::vector<GroupInfo> groups;
    std::vector<double> values;
    std::vector<index_t> columns;
    std::vector<std::size_t> threads_mapping;

    std::size_t total_slots() const { return values.size(); }
    bool operator==(const ArgCsrMatrix&) const = default;
};

inline constexpr std::size_t kDefaultThreadsPerGroup = 128;
inline constexpr std::size_t kDefaultDesiredChunkSize = 1;

// analysis.hpp:14-23
struct FormatStats {
    std::size_t explicit_nnz = 0;
    std::size_t assigned_padded_slots = 0;
    std::size_t total_allocated_slots = 0;
    double padding_ratio = 1.0;
    std::size_t estimated_bytes = 0;
};

struct BalanceStats {  // analysis.hpp:26-32
    std::vector<std::size_t> per_group_nnz;
    double max_over_mean = 1.0;
    double coefficient_of_variation = 0.0;
};

static_assert(sizeof(std::size_t) == sizeof(uint64_t), "64-bit size_t required");

// ------------------------------------------------------ device ARG-CSR matrix
class DeviceArgCsr {
public:
    DeviceArgCsr() = default;
    explicit DeviceArgCsr(argcsr_dev* h, bool owned = true) : h_(h), owned_(owned) { refresh(); }
    // A view of a handle owned elsewhere (a multi-GPU slice: argcsr_mgpu_local).
    static DeviceArgCsr borrow(argcsr_dev* h) { return DeviceArgCsr(h, false); }
    DeviceArgCsr(DeviceArgCsr&& o) noexcept
        : h_(std::exchange(o.h_, nullptr)), owned_(o.owned_), info_(o.info_) {}
    DeviceArgCsr& operator=(DeviceArgCsr&& o) noexcept {
        if (this != &o) {
            reset();
            h_ = std::exchange(o.h_, nullptr);
            owned_ = o.owned_;
            info_ = o.info_;
        }
        return *this;
    }
    DeviceArgCsr(const DeviceArgCsr&) = delete;
    DeviceArgCsr& operator=(const DeviceArgCsr&) = delete;
    ~DeviceArgCsr() { reset(); }

    void reset() {
        if (h_ && owned_) argcsr_dev_free(h_);
        h_ = nullptr;
    }
    argcsr_dev* handle() const { return h_; }
    const argcsr_dev_info_t& info() const { return info_; }
    std::size_t num_rows() const { return info_.num_rows; }
    std::size_t num_cols() const { return info_.num_cols; }
    std::size_t threads_per_group() const { return info_.threads_per_group; }
    std::size_t num_groups() const { return info_.num_groups; }
    std::size_t total_slots() const { return info_.total_slots; }

    // The reference layout (argcsr.hpp:52-63), copied and widened from the device.
    ArgCsrMatrix to_host() const {
        ArgCsrMatrix M;
        M.num_rows = info_.num_rows;
        M.num_cols = info_.num_cols;
        M.threads_per_group = info_.threads_per_group;
        std::vector<uint64_t> g4(4 * info_.num_groups);
        M.threads_mapping.resize(info_.num_rows);
        if (info_.dtype != ARGCSR_F64) throw UnsupportedError("to_host: fp32 handle has no fp64 reference layout");
        M.values.resize(info_.total_slots);
        M.columns.resize(info_.total_slots);
        check(argcsr_dev_export(h_, g4.data(), reinterpret_cast<uint64_t*>(M.threads_mapping.data()),
                                M.values.data(), M.columns.data()));
        M.groups.resize(info_.num_groups);
        for (std::size_t g = 0; g < info_.num_groups; ++g)
            M.groups[g] = {g4[4 * g], g4[4 * g + 1], g4[4 * g + 2], g4[4 * g + 3]};
        return M;
    }

private:
    void refresh() {
        if (h_) check(argcsr_dev_info(h_, &info_));
    }
    argcsr_dev* h_ = nullptr;
    bool owned_ = true;
    argcsr_dev_info_t info_{};
};

// argcsr.hpp:101-104 — conversion runs on `device`; the result stays there.
inline DeviceArgCsr argcsr_from_csr(const CsrMatrix& A, std::size_t threads_per_group = kDefaultThreadsPerGroup,
                                    std::size_t desired_chunk_size = kDefaultDesiredChunkSize, int device = 0) {
    argcsr_csr_view v{};
    v.num_rows = A.num_rows;
    v.num_cols = A.num_cols;
    v.nnz = A.nnz();
    v.row_pointers = reinterpret_cast<const uint64_t*>(A.row_pointers.data());
    v.columns = A.columns.data();
    v.values = A.values.data();
    v.dtype = ARGCSR_F64;
    v.space = ARGCSR_HOST;
    if (A.row_pointers.size() != A.num_rows + 1 && A.num_rows != 0)
        throw DimensionError("argcsr_from_csr: row_pointers length does not match num_rows + 1");
    argcsr_dev* h = nullptr;
    check(argcsr_dev_convert(&v, threads_per_group, desired_chunk_size, device, nullptr, &h));
    return DeviceArgCsr(h);
}

// argcsr.hpp:110 — host vectors in and out (DimensionError on a length mismatch).
inline DenseVector spmv_argcsr(const DeviceArgCsr& M, const DenseVector& x) {
    DenseVector y(M.num_rows(), 0.0);
    check(argcsr_dev_spmv_host(M.handle(), x.data(), x.size(), y.data()));
    return y;
}

// bench.hpp:59-60 — `workers` has no meaning on the device; kept for signature parity.
inline void spmv_argcsr_parallel(const DeviceArgCsr& M, const DenseVector& x, DenseVector& y, std::size_t = 1) {
    if (x.size() != M.num_cols())
        throw DimensionError("parallel spmv: vector length " + std::to_string(x.size()) + " does not match " +
                             std::to_string(M.num_cols()) + " columns");
    y.resize(M.num_rows());
    check(argcsr_dev_spmv_host(M.handle(), x.data(), x.size(), y.data()));
}

// Device pointers, stream-ordered (the hot path).
inline void spmv_device(const DeviceArgCsr& M, const void* x, void* y, void* stream = nullptr) {
    check(argcsr_dev_spmv(M.handle(), x, y, stream));
}

// argcsr.hpp:106
inline CsrMatrix csr_from_argcsr(const DeviceArgCsr& M) {
    CsrMatrix A;
    A.num_rows = M.num_rows();
    A.num_cols = M.num_cols();
    A.row_pointers.resize(M.num_rows() + 1);
    A.values.resize(M.info().nnz);
    A.columns.resize(M.info().nnz);
    check(argcsr_dev_to_csr(M.handle(), reinterpret_cast<uint64_t*>(A.row_pointers.data()), A.columns.data(),
                            A.values.data()));
    return A;
}

// argcsr.hpp:118-121
inline std::vector<std::pair<double, index_t>> chunk_entries(const DeviceArgCsr& M, std::size_t group_index,
                                                             std::size_t chunk_index) {
    std::vector<double> v(M.info().max_chunk_size + 1);
    std::vector<index_t> c(M.info().max_chunk_size + 1);
    uint64_t n = 0;
    check(argcsr_dev_chunk_entries(M.handle(), group_index, chunk_index, v.data(), c.data(), v.size(), &n));
    std::vector<std::pair<double, index_t>> out;
    out.reserve(n);
    for (uint64_t i = 0; i < n; ++i) out.emplace_back(v[i], c[i]);
    return out;
}

// analysis.hpp:60 (ArgCsrMatrix overload)
inline FormatStats padding_stats(const DeviceArgCsr& M) {
    argcsr_format_stats s{};
    check(argcsr_dev_padding_stats(M.handle(), &s));
    return {s.explicit_nnz, s.assigned_padded_slots, s.total_allocated_slots, s.padding_ratio, s.estimated_bytes};
}

inline BalanceStats balance_stats(const DeviceArgCsr& M) {
    argcsr_dev_info_t info{};
    check(argcsr_dev_info(M.handle(), &info));
    BalanceStats b;
    b.per_group_nnz.resize(info.num_groups);
    check(argcsr_dev_balance_stats(M.handle(), reinterpret_cast<uint64_t*>(b.per_group_nnz.data()),
                                   &b.max_over_mean, &b.coefficient_of_variation));
    return b;
}

// io.hpp:37-43 — the reference's binary container, byte-identical.
inline void write_binary_file(const std::string& path, const DeviceArgCsr& M) {
    check(argcsr_dev_write_binary(M.handle(), path.c_str()));
}

// An ARG-CSR container is imported as stored (a cached conversion); a CSR
// container is converted with threads_per_group / desired_chunk_size.
inline DeviceArgCsr read_binary_file(const std::string& path, std::size_t threads_per_group = kDefaultThreadsPerGroup,
                                     std::size_t desired_chunk_size = kDefaultDesiredChunkSize, int device = 0) {
    argcsr_dev* h = nullptr;
    check(argcsr_dev_read_binary(path.c_str(), threads_per_group, desired_chunk_size, device, nullptr, 0u, &h));
    return DeviceArgCsr(h);
}

// A device handle from a host ArgCsrMatrix without re-running the converter.
inline DeviceArgCsr device_from_host(const ArgCsrMatrix& M, int device = 0) {
    std::vector<uint64_t> g4(4 * M.groups.size());
    for (std::size_t g = 0; g < M.groups.size(); ++g) {
        g4[4 * g] = M.groups[g].first_row;
        g4[4 * g + 1] = M.groups[g].size;
        g4[4 * g + 2] = M.groups[g].offset;
        g4[4 * g + 3] = M.groups[g].chunk_size;
    }
    argcsr_argcsr_view v{};
    v.num_rows = M.num_rows;
    v.num_cols = M.num_cols;
    v.threads_per_group = M.threads_per_group;
    v.num_groups = M.groups.size();
    v.groups4 = g4.data();
    v.threads_mapping = reinterpret_cast<const uint64_t*>(M.threads_mapping.data());
    v.values = M.values.data();
    v.columns = M.columns.data();
    v.total_slots = M.values.size();
    v.dtype = ARGCSR_F64;
    argcsr_dev* h = nullptr;
    check(argcsr_dev_import(&v, device, nullptr, 0u, &h));
    return DeviceArgCsr(h);
}

}  // namespace argcsr_b200
