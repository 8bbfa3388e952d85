// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Plain-C wrappers over the *unmodified* reference library (`argcsr`,
// /root/reference/proj/src/*.cpp), compiled from the sources where they lie by
// oracle/Makefile into oracle/_ref/libargcsr_ref.so.  Used to
//   * pin the C restatement in oracle/argcsr_oracle.c,
//   * generate the golden fixtures under tests/golden/ (tests/golden/make_golden.py),
//   * generate the reference test corpus (proj/tests/support.hpp:86-119) — its
//     std::uniform_*_distribution output is libstdc++-specific, so it is
//     compiled, not re-implemented,
//   * time the reference CPU path for bench.py's `cpu_baseline` leg and the
//     `--impl reference` arm (spmv_argcsr_parallel, proj/src/bench.cpp:109-116).
//
// Status codes mirror include/argcsr_gpu.h (ARGCSR_OK = 0, ...).

#include <cstdint>
#include <cstring>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "argcsr/analysis.hpp"
#include "argcsr/argcsr.hpp"
#include "argcsr/ellpack.hpp"
#include "argcsr/bench.hpp"
#include "argcsr/core.hpp"
#include "argcsr/io.hpp"
#include "support.hpp"

using namespace argcsr;

namespace {

thread_local std::string g_err;

// Same numbering as argcsr_status in include/argcsr_gpu.h.
enum : int {
    kOk = 0,
    kParameter = 1,
    kDimension = 2,
    kBounds = 3,
    kInternal = 4,
    kCuda = 5,
    kNccl = 6,
    kOom = 7,
    kFormat = 8,
    kIo = 9,
    kParse = 10,
    kUnsupported = 11,
    kCorrectness = 12,
    kUnknown = 99,
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const ParameterError& e) {
        g_err = e.what();
        return kParameter;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return kDimension;
    } catch (const BoundsError& e) {
        g_err = e.what();
        return kBounds;
    } catch (const InternalError& e) {
        g_err = e.what();
        return kInternal;
    } catch (const FormatError& e) {
        g_err = e.what();
        return kFormat;
    } catch (const IoError& e) {
        g_err = e.what();
        return kIo;
    } catch (const ParseError& e) {
        g_err = e.what();
        return kParse;
    } catch (const UnsupportedError& e) {
        g_err = e.what();
        return kUnsupported;
    } catch (const CorrectnessError& e) {
        g_err = e.what();
        return kCorrectness;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return kOom;
    } catch (const std::exception& e) {
        g_err = e.what();
        return kUnknown;
    }
}

CsrMatrix make_csr(uint64_t nrows, uint64_t ncols, uint64_t nnz, const uint64_t* rp,
                   const int32_t* cols, const double* vals) {
    CsrMatrix A;
    A.num_rows = nrows;
    A.num_cols = ncols;
    A.row_pointers.assign(rp, rp + nrows + 1);
    A.columns.assign(cols, cols + nnz);
    A.values.assign(vals, vals + nnz);
    return A;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- CSR handles
void* ref_csr_new(uint64_t nrows, uint64_t ncols, uint64_t nnz, const uint64_t* rp,
                  const int32_t* cols, const double* vals) {
    return new CsrMatrix(make_csr(nrows, ncols, nnz, rp, cols, vals));
}

int ref_csr_from_triplets(uint64_t nrows, uint64_t ncols, uint64_t n, const uint64_t* rows,
                          const uint64_t* cols, const double* vals, void** out) {
    return guarded([&] {
        std::vector<Triplet> ts(n);
        for (uint64_t i = 0; i < n; ++i) ts[i] = {rows[i], cols[i], vals[i]};
        *out = new CsrMatrix(csr_from_triplets(nrows, ncols, std::move(ts)));
    });
}

void ref_csr_shape(const void* h, uint64_t* nrows, uint64_t* ncols, uint64_t* nnz) {
    const auto* A = static_cast<const CsrMatrix*>(h);
    *nrows = A->num_rows;
    *ncols = A->num_cols;
    *nnz = A->nnz();
}

void ref_csr_copy(const void* h, uint64_t* rp, int32_t* cols, double* vals) {
    const auto* A = static_cast<const CsrMatrix*>(h);
    std::memcpy(rp, A->row_pointers.data(), A->row_pointers.size() * sizeof(uint64_t));
    if (A->nnz()) {
        std::memcpy(cols, A->columns.data(), A->nnz() * sizeof(int32_t));
        std::memcpy(vals, A->values.data(), A->nnz() * sizeof(double));
    }
}

void ref_csr_free(void* h) { delete static_cast<CsrMatrix*>(h); }

// Reference test fixtures (proj/tests/support.hpp:46-119).
void* ref_fixture_e8(void) { return new CsrMatrix(testsupport::e8_matrix()); }
void* ref_fixture_skew(uint64_t k) { return new CsrMatrix(testsupport::skew_matrix(k)); }
void* ref_fixture_uniform(uint64_t rows, uint64_t cols, uint64_t per_row) {
    return new CsrMatrix(testsupport::uniform_matrix(rows, cols, per_row));
}
void ref_probe_vector(uint64_t n, uint32_t salt, double* out) {
    const DenseVector x = testsupport::probe_vector(n, salt);
    std::memcpy(out, x.data(), n * sizeof(double));
}

void* ref_corpus_new(uint64_t count, uint32_t seed) {
    return new std::vector<CsrMatrix>(testsupport::build_corpus(count, seed));
}
uint64_t ref_corpus_size(const void* h) {
    return static_cast<const std::vector<CsrMatrix>*>(h)->size();
}
const void* ref_corpus_get(const void* h, uint64_t i) {
    return &(*static_cast<const std::vector<CsrMatrix>*>(h))[i];
}
void ref_corpus_free(void* h) { delete static_cast<std::vector<CsrMatrix>*>(h); }

// ------------------------------------------------------------ pieces of the path
int ref_partition_groups(const uint64_t* counts, uint64_t n, uint64_t tpg, uint64_t dcs,
                         uint64_t* spans2, uint64_t* nspans) {
    return guarded([&] {
        const std::vector<std::size_t> c(counts, counts + n);
        const auto spans = partition_groups(c, tpg, dcs);
        for (std::size_t i = 0; i < spans.size(); ++i) {
            spans2[2 * i] = spans[i].first_row;
            spans2[2 * i + 1] = spans[i].size;
        }
        *nspans = spans.size();
    });
}

int ref_assign_threads(const uint64_t* counts, uint64_t n, uint64_t tpg, uint64_t* tpr,
                       uint64_t* chunk, uint64_t* assigned, uint64_t* free_threads) {
    return guarded([&] {
        const std::vector<std::size_t> c(counts, counts + n);
        const ThreadAssignment ta = assign_threads(c, tpg);
        for (uint64_t i = 0; i < n; ++i) tpr[i] = ta.threads_per_row[i];
        *chunk = ta.chunk_size;
        *assigned = ta.assigned_threads;
        *free_threads = ta.free_threads;
    });
}

// --------------------------------------------------------------- ARG-CSR handles
int ref_argcsr_from_csr(const void* csr, uint64_t tpg, uint64_t dcs, void** out) {
    return guarded([&] {
        *out = new ArgCsrMatrix(argcsr_from_csr(*static_cast<const CsrMatrix*>(csr), tpg, dcs));
    });
}

void ref_argcsr_info(const void* h, uint64_t* nrows, uint64_t* ncols, uint64_t* tpg,
                     uint64_t* ngroups, uint64_t* nslots) {
    const auto* M = static_cast<const ArgCsrMatrix*>(h);
    *nrows = M->num_rows;
    *ncols = M->num_cols;
    *tpg = M->threads_per_group;
    *ngroups = M->groups.size();
    *nslots = M->total_slots();
}

void ref_argcsr_export(const void* h, uint64_t* groups4, uint64_t* tm, double* vals,
                       int32_t* cols) {
    const auto* M = static_cast<const ArgCsrMatrix*>(h);
    for (std::size_t g = 0; g < M->groups.size(); ++g) {
        groups4[4 * g + 0] = M->groups[g].first_row;
        groups4[4 * g + 1] = M->groups[g].size;
        groups4[4 * g + 2] = M->groups[g].offset;
        groups4[4 * g + 3] = M->groups[g].chunk_size;
    }
    for (std::size_t r = 0; r < M->threads_mapping.size(); ++r) tm[r] = M->threads_mapping[r];
    if (M->total_slots()) {
        std::memcpy(vals, M->values.data(), M->total_slots() * sizeof(double));
        std::memcpy(cols, M->columns.data(), M->total_slots() * sizeof(int32_t));
    }
}

// Rebuild a reference ArgCsrMatrix from exported arrays (e.g. the GPU export),
// so the reference SpMV can run on a matrix it did not convert itself.
void* ref_argcsr_import(uint64_t nrows, uint64_t ncols, uint64_t tpg, uint64_t ngroups,
                        const uint64_t* groups4, const uint64_t* tm, uint64_t nslots,
                        const double* vals, const int32_t* cols) {
    auto* M = new ArgCsrMatrix;
    M->num_rows = nrows;
    M->num_cols = ncols;
    M->threads_per_group = tpg;
    M->groups.resize(ngroups);
    for (uint64_t g = 0; g < ngroups; ++g) {
        M->groups[g] = {groups4[4 * g], groups4[4 * g + 1], groups4[4 * g + 2],
                        groups4[4 * g + 3]};
    }
    M->threads_mapping.assign(tm, tm + nrows);
    M->values.assign(vals, vals + nslots);
    M->columns.assign(cols, cols + nslots);
    return M;
}

void ref_argcsr_free(void* h) { delete static_cast<ArgCsrMatrix*>(h); }

int ref_csr_from_argcsr(const void* h, void** out) {
    return guarded([&] {
        *out = new CsrMatrix(csr_from_argcsr(*static_cast<const ArgCsrMatrix*>(h)));
    });
}

int ref_chunk_entries(const void* h, uint64_t g, uint64_t c, double* vals, int32_t* cols,
                      uint64_t* n) {
    return guarded([&] {
        const auto e = chunk_entries(*static_cast<const ArgCsrMatrix*>(h), g, c);
        for (std::size_t i = 0; i < e.size(); ++i) {
            vals[i] = e[i].first;
            cols[i] = e[i].second;
        }
        *n = e.size();
    });
}

int ref_padding_stats(const void* h, uint64_t* explicit_nnz, uint64_t* padded,
                      uint64_t* total, double* ratio, uint64_t* est_bytes) {
    return guarded([&] {
        const FormatStats fs = padding_stats(*static_cast<const ArgCsrMatrix*>(h));
        *explicit_nnz = fs.explicit_nnz;
        *padded = fs.assigned_padded_slots;
        *total = fs.total_allocated_slots;
        *ratio = fs.padding_ratio;
        *est_bytes = fs.estimated_bytes;
    });
}

int ref_balance_stats(const void* h, uint64_t* per_group, double* max_over_mean, double* cv) {
    return guarded([&] {
        const BalanceStats b = balance_stats(*static_cast<const ArgCsrMatrix*>(h));
        for (size_t i = 0; i < b.per_group_nnz.size(); ++i) per_group[i] = b.per_group_nnz[i];
        *max_over_mean = b.max_over_mean;
        *cv = b.coefficient_of_variation;
    });
}

// ------------------------------------------------------------------------ SpMV
int ref_spmv_argcsr(const void* h, const double* x, uint64_t nx, double* y) {
    return guarded([&] {
        const auto* M = static_cast<const ArgCsrMatrix*>(h);
        const DenseVector xv(x, x + nx);
        const DenseVector yv = spmv_argcsr(*M, xv);
        std::memcpy(y, yv.data(), yv.size() * sizeof(double));
    });
}

int ref_spmv_argcsr_groups(const void* h, const double* x, uint64_t nx, uint64_t gb,
                           uint64_t ge, double* y) {
    return guarded([&] {
        const auto* M = static_cast<const ArgCsrMatrix*>(h);
        const DenseVector xv(x, x + nx);
        spmv_argcsr_groups(*M, xv, gb, ge, std::span<double>(y, M->num_rows));
    });
}

int ref_spmv_csr(const void* csr, const double* x, uint64_t nx, double* y) {
    return guarded([&] {
        const auto* A = static_cast<const CsrMatrix*>(csr);
        const DenseVector xv(x, x + nx);
        const DenseVector yv = spmv_csr(*A, xv);
        std::memcpy(y, yv.data(), yv.size() * sizeof(double));
    });
}

// Timed reference CPU baseline: `iters` calls of spmv_argcsr_parallel
// (bench.cpp:109-116) with `workers` threads, x/y held as DenseVectors for the
// whole loop exactly like run_benchmark (bench.cpp:155-236). Per-call wall
// times (seconds) go to times[0..iters).
int ref_time_spmv_argcsr_parallel(const void* h, const double* x, uint64_t nx, uint64_t workers,
                                  uint64_t warmup, uint64_t iters, double* times, double* y_out) {
    return guarded([&] {
        const auto* M = static_cast<const ArgCsrMatrix*>(h);
        const DenseVector xv(x, x + nx);
        DenseVector y;
        for (uint64_t i = 0; i < warmup; ++i) spmv_argcsr_parallel(*M, xv, y, workers);
        for (uint64_t i = 0; i < iters; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            spmv_argcsr_parallel(*M, xv, y, workers);
            times[i] =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        if (y_out && !y.empty()) std::memcpy(y_out, y.data(), y.size() * sizeof(double));
    });
}

int ref_time_spmv_csr_parallel(const void* csr, const double* x, uint64_t nx, uint64_t workers,
                               uint64_t warmup, uint64_t iters, double* times) {
    return guarded([&] {
        const auto* A = static_cast<const CsrMatrix*>(csr);
        const DenseVector xv(x, x + nx);
        DenseVector y;
        for (uint64_t i = 0; i < warmup; ++i) spmv_csr_parallel(*A, xv, y, workers);
        for (uint64_t i = 0; i < iters; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            spmv_csr_parallel(*A, xv, y, workers);
            times[i] =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

// Binary container (io.cpp:282-298): byte-exact serialisation of an ArgCsrMatrix.
int ref_write_binary_argcsr(const void* h, const char* path) {
    return guarded([&] { write_binary_file(path, *static_cast<const ArgCsrMatrix*>(h)); });
}

// Binary container, CSR tag (io.cpp:250-257).
int ref_write_binary_csr(const void* csr, const char* path) {
    return guarded([&] { write_binary_file(path, *static_cast<const CsrMatrix*>(csr)); });
}

// ELLPACK / Sliced ELLPACK (ellpack.cpp): conversions, fields, SpMV.
void* ref_ellpack_from_csr(const void* csr) {
    return new EllpackMatrix(ellpack_from_csr(*static_cast<const CsrMatrix*>(csr)));
}
int ref_sliced_from_csr(const void* csr, uint64_t slice_size, void** out) {
    return guarded([&] { *out = new SlicedEllpackMatrix(sliced_from_csr(*static_cast<const CsrMatrix*>(csr), slice_size)); });
}
void ref_ell_fields(const void* h, uint64_t* width, uint64_t* slots, double* vals, int32_t* cols) {
    const auto* M = static_cast<const EllpackMatrix*>(h);
    *width = M->width;
    *slots = M->values.size();
    if (vals) std::copy(M->values.begin(), M->values.end(), vals);
    if (cols) std::copy(M->columns.begin(), M->columns.end(), cols);
}
void ref_sell_fields(const void* h, uint64_t* nslices, uint64_t* slots, uint64_t* widths, uint64_t* offsets, double* vals,
                     int32_t* cols) {
    const auto* M = static_cast<const SlicedEllpackMatrix*>(h);
    *nslices = M->num_slices();
    *slots = M->values.size();
    if (widths) std::copy(M->slice_widths.begin(), M->slice_widths.end(), widths);
    if (offsets) std::copy(M->slice_offsets.begin(), M->slice_offsets.end(), offsets);
    if (vals) std::copy(M->values.begin(), M->values.end(), vals);
    if (cols) std::copy(M->columns.begin(), M->columns.end(), cols);
}
int ref_spmv_ellpack(const void* h, const double* x, uint64_t nx, double* y) {
    return guarded([&] {
        const DenseVector r = spmv_ellpack(*static_cast<const EllpackMatrix*>(h), DenseVector(x, x + nx));
        std::copy(r.begin(), r.end(), y);
    });
}
int ref_spmv_sliced(const void* h, const double* x, uint64_t nx, double* y) {
    return guarded([&] {
        const DenseVector r = spmv_sliced(*static_cast<const SlicedEllpackMatrix*>(h), DenseVector(x, x + nx));
        std::copy(r.begin(), r.end(), y);
    });
}
void ref_ell_free(void* h) { delete static_cast<EllpackMatrix*>(h); }
void ref_sell_free(void* h) { delete static_cast<SlicedEllpackMatrix*>(h); }

uint64_t ref_hardware_threads(void) { return std::thread::hardware_concurrency(); }

}  // extern "C"
