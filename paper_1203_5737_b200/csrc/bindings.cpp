// pybind11 module `_argcsr_gpu`: the reference's Python bindings
// (proj/python/bindings.cpp:13-173) re-pointed at the C-ABI.  Names, argument
// names and defaults follow the reference module; every error surfaces as
// `Error` or one of its subclasses (bindings.cpp:15).  Large arrays cross as
// numpy buffers instead of Python lists.
#include <pybind11/numpy.h>
#include <pybind11/operators.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <algorithm>
#include <cctype>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <sstream>
#include <memory>
#include <optional>
#include <tuple>

#include "argcsr_gpu.hpp"
#include "host_io.hpp"

namespace py = pybind11;
using namespace argcsr_b200;

namespace {

template <typename T>
py::array_t<T> view_of(const std::vector<T>& v, py::handle base) {
    return py::array_t<T>({v.size()}, {sizeof(T)}, v.data(), base);
}

// A fresh, writeable 1-D float64 or float32 array of n elements.
py::array new_array(bool f64, std::size_t n) {
    if (f64) return py::array_t<double>(py::ssize_t(n));
    return py::array_t<float>(py::ssize_t(n));
}

template <typename T>
std::vector<T> vec_from(const py::array_t<T, py::array::c_style | py::array::forcecast>& a) {
    return std::vector<T>(a.data(), a.data() + a.size());
}

// Python-side ARG-CSR matrix: the device handle plus a lazily exported
// reference-layout host copy (argcsr.hpp:52-63 fields).
struct PyArgCsr {
    std::shared_ptr<DeviceArgCsr> dev;
    mutable std::optional<std::vector<uint64_t>> groups4, tm;
    mutable std::optional<py::array> values;
    mutable std::optional<std::vector<int32_t>> columns;

    const argcsr_dev_info_t& info() const { return dev->info(); }
    void need_meta() const {
        if (groups4) return;
        std::vector<uint64_t> g(4 * info().num_groups), t(info().num_rows);
        check(argcsr_dev_export(dev->handle(), g.data(), t.data(), nullptr, nullptr));
        groups4 = std::move(g);
        tm = std::move(t);
    }
    void need_slots() const {
        if (columns) return;
        const std::size_t S = info().total_slots;
        py::array v = new_array(info().dtype == ARGCSR_F64, S);
        std::vector<int32_t> c(S);
        check(argcsr_dev_export(dev->handle(), nullptr, nullptr, v.mutable_data(), c.data()));
        values = v;
        columns = std::move(c);
    }
};

// ELLPACK / Sliced ELLPACK device matrices (argcsr_sell*); the two Python
// classes share one handle type, like the reference's two structs share a
// layout (ellpack.hpp:13-45).
struct SellHandle {
    argcsr_sell* h = nullptr;
    argcsr_sell_info_t info{};
    explicit SellHandle(argcsr_sell* p) : h(p) { check(argcsr_sell_info(h, &info)); }
    ~SellHandle() { argcsr_sell_free(h); }
    SellHandle(const SellHandle&) = delete;
    SellHandle& operator=(const SellHandle&) = delete;
};
struct PySellBase {
    std::shared_ptr<SellHandle> s;
    const argcsr_sell_info_t& info() const { return s->info; }
    py::array values() const {
        const bool f64 = info().dtype == ARGCSR_F64;
        py::array v = f64 ? py::array(py::array_t<double>(py::ssize_t(info().total_slots)))
                          : py::array(py::array_t<float>(py::ssize_t(info().total_slots)));
        check(argcsr_sell_export(s->h, nullptr, nullptr, v.mutable_data(), nullptr));
        return v;
    }
    py::array_t<int32_t> columns() const {
        py::array_t<int32_t> c(py::ssize_t(info().total_slots));
        check(argcsr_sell_export(s->h, nullptr, nullptr, nullptr, c.mutable_data()));
        return c;
    }
    std::vector<uint64_t> widths() const {
        std::vector<uint64_t> w(info().num_slices);
        check(argcsr_sell_export(s->h, w.data(), nullptr, nullptr, nullptr));
        return w;
    }
    std::vector<uint64_t> offsets() const {
        std::vector<uint64_t> o(info().num_slices);
        check(argcsr_sell_export(s->h, nullptr, o.data(), nullptr, nullptr));
        return o;
    }
    // csr_from_ellpack / csr_from_sliced (ellpack.cpp:62-119): read each row's
    // slots up to the first padding, in slot order.
    CsrMatrix to_csr() const {
        if (info().dtype != ARGCSR_F64) throw UnsupportedError("csr_from_sliced: fp32 matrix");
        const uint64_t N = info().num_rows, S = info().slice_size;
        std::vector<double> v(info().total_slots);
        std::vector<int32_t> c(info().total_slots);
        std::vector<uint64_t> w = widths(), o = offsets();
        check(argcsr_sell_export(s->h, nullptr, nullptr, v.data(), c.data()));
        CsrMatrix A;
        A.num_rows = N;
        A.num_cols = info().num_cols;
        A.row_pointers.assign(N + 1, 0);
        for (uint64_t sl = 0; sl < w.size(); ++sl) {
            const uint64_t first = sl * S, rows = std::min(first + S, N) - first;
            for (uint64_t local = 0; local < rows; ++local)
                for (uint64_t j = 0; j < w[sl]; ++j) {
                    const uint64_t slot = o[sl] + j * rows + local;
                    if (c[slot] == -1) break;
                    A.values.push_back(v[slot]);
                    A.columns.push_back(c[slot]);
                    A.row_pointers[first + local + 1] += 1;
                }
        }
        for (uint64_t r = 0; r < N; ++r) A.row_pointers[r + 1] += A.row_pointers[r];
        return A;
    }
};
struct PyEllpack : PySellBase {};
struct PySliced : PySellBase {};

argcsr_csr_view host_view(const CsrMatrix& A) {
    argcsr_csr_view v{};
    v.num_rows = A.num_rows;
    v.num_cols = A.num_cols;
    v.nnz = A.nnz();
    v.row_pointers = reinterpret_cast<const uint64_t*>(A.row_pointers.data());
    v.columns = A.columns.data();
    v.values = A.values.data();
    v.dtype = ARGCSR_F64;
    v.space = ARGCSR_HOST;
    return v;
}

template <typename P>
py::array sell_spmv_host(const P& p, py::array x) {
    const bool f64 = p.info().dtype == ARGCSR_F64;
    py::array xc = f64 ? py::array(py::array_t<double, py::array::c_style | py::array::forcecast>(x))
                       : py::array(py::array_t<float, py::array::c_style | py::array::forcecast>(x));
    py::array y = new_array(f64, p.info().num_rows);
    const void* xp = xc.data();
    void* yp = y.mutable_data();
    const uint64_t n = uint64_t(xc.size());
    {
        py::gil_scoped_release nogil;
        check(argcsr_sell_spmv_host(p.s->h, xp, n, yp));
    }
    return y;
}

PyArgCsr make_handle(argcsr_dev* h) {
    PyArgCsr p;
    p.dev = std::make_shared<DeviceArgCsr>(h);
    return p;
}

PyArgCsr convert_arrays(std::size_t num_rows, std::size_t num_cols, py::array row_pointers, py::array columns,
                        py::array values, std::size_t tpg, std::size_t dcs, int device, std::uint32_t flags) {
    auto rp = py::array_t<uint64_t, py::array::c_style | py::array::forcecast>(row_pointers);
    auto cl = py::array_t<int32_t, py::array::c_style | py::array::forcecast>(columns);
    argcsr_csr_view v{};
    v.num_rows = num_rows;
    v.num_cols = num_cols;
    v.space = ARGCSR_HOST;
    v.row_pointers = rp.data();
    v.columns = cl.data();
    if (rp.size() != py::ssize_t(num_rows + 1) && num_rows != 0)
        throw DimensionError("argcsr_from_csr: row_pointers length does not match num_rows + 1");
    py::array vals;
    if (py::dtype(values.dtype()).is(py::dtype::of<float>())) {
        vals = py::array_t<float, py::array::c_style | py::array::forcecast>(values);
        v.dtype = ARGCSR_F32;
    } else {
        vals = py::array_t<double, py::array::c_style | py::array::forcecast>(values);
        v.dtype = ARGCSR_F64;
    }
    if (vals.size() != cl.size()) throw DimensionError("argcsr_from_csr: values and columns lengths differ");
    v.nnz = uint64_t(cl.size());
    v.values = vals.data();
    argcsr_dev* h = nullptr;
    {
        py::gil_scoped_release nogil;
        check(argcsr_dev_convert_ex(&v, tpg, dcs, device, nullptr, flags, &h));
    }
    return make_handle(h);
}

}  // namespace

// The multi-GPU handle (argcsr_mgpu_*): one per process in the one-process-
// per-GPU form.  Per-local-rank arguments are lists of device pointers /
// stream handles as ints.
struct PyMultiGpu {
    argcsr_mgpu* h = nullptr;
    int nlocal = 1;
    ~PyMultiGpu() { free(); }
    void free() {
        if (h) argcsr_mgpu_free(h);
        h = nullptr;
    }
    argcsr_mgpu* get() const {
        if (!h) throw ParameterError("multi-GPU handle already freed");
        return h;
    }
};

std::vector<void*> ptr_list(const std::vector<std::uintptr_t>& v, std::size_t n, const char* what) {
    if (v.size() != n) throw ParameterError(std::string(what) + ": one entry per local GPU");
    std::vector<void*> out(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = reinterpret_cast<void*>(v[i]);
    return out;
}

argcsr_csr_view view_from_ptrs(std::size_t num_rows, std::size_t num_cols, std::size_t nnz, std::uintptr_t rp,
                               std::uintptr_t cols, std::uintptr_t vals, const std::string& dtype, bool device) {
    argcsr_csr_view v{};
    v.num_rows = num_rows;
    v.num_cols = num_cols;
    v.nnz = nnz;
    v.row_pointers = reinterpret_cast<const uint64_t*>(rp);
    v.columns = reinterpret_cast<const int32_t*>(cols);
    v.values = reinterpret_cast<const void*>(vals);
    if (dtype != "float64" && dtype != "float32") throw ParameterError("dtype must be 'float64' or 'float32'");
    v.dtype = dtype == "float64" ? ARGCSR_F64 : ARGCSR_F32;
    v.space = device ? ARGCSR_DEVICE : ARGCSR_HOST;
    return v;
}

PYBIND11_MODULE(_argcsr_gpu, m) {
    m.doc() = "B200-native adaptive row-grouped CSR (ARG-CSR): GPU conversion and SpMV behind the argcsr API";

    py::register_exception_translator([](std::exception_ptr p) {
        if (!p) return;
        try {
            std::rethrow_exception(p);
        } catch (const Error& e) {
            const char* name = "Error";
            if (dynamic_cast<const ParameterError*>(&e)) name = "ParameterError";
            else if (dynamic_cast<const DimensionError*>(&e)) name = "DimensionError";
            else if (dynamic_cast<const BoundsError*>(&e)) name = "BoundsError";
            else if (dynamic_cast<const CudaError*>(&e)) name = "CudaError";
            else if (dynamic_cast<const NcclError*>(&e)) name = "NcclError";
            else if (dynamic_cast<const OutOfMemoryError*>(&e)) name = "OutOfMemoryError";
            else if (dynamic_cast<const InternalError*>(&e)) name = "InternalError";
            else if (dynamic_cast<const UnsupportedError*>(&e)) name = "UnsupportedError";
            else if (dynamic_cast<const FormatError*>(&e)) name = "FormatError";
            else if (dynamic_cast<const IoError*>(&e)) name = "IoError";
            else if (dynamic_cast<const ParseError*>(&e)) name = "ParseError";
            else if (dynamic_cast<const CorrectnessError*>(&e)) name = "CorrectnessError";
            py::object cls = py::module_::import("paper_1203_5737_b200._errors").attr(name);
            PyErr_SetString(cls.ptr(), e.what());
        }
    });

    m.attr("kDefaultThreadsPerGroup") = kDefaultThreadsPerGroup;
    m.attr("kDefaultDesiredChunkSize") = kDefaultDesiredChunkSize;
    m.attr("kPaddingColumn") = kPaddingColumn;
    m.def("abi_version", &argcsr_abi_version);

    // ------------------------------------------------ multi-GPU (argcsr_mgpu_*)
    m.def("mgpu_unique_id", [] {
        unsigned char id[ARGCSR_NCCL_ID_BYTES];
        check(argcsr_mgpu_unique_id(id));
        return py::bytes(reinterpret_cast<const char*>(id), ARGCSR_NCCL_ID_BYTES);
    });
    m.def(
        "plan_interior",
        [](py::array_t<uint64_t, py::array::c_style | py::array::forcecast> rp,
           py::array_t<int32_t, py::array::c_style | py::array::forcecast> cols,
           py::array_t<uint64_t, py::array::c_style | py::array::forcecast> group_first, uint64_t r0, uint64_t r1) {
            if (rp.size() < 1 || group_first.size() < 1) throw ParameterError("plan_interior: empty arrays");
            uint64_t ga = 0, gb = 0;
            check(argcsr_plan_interior(rp.data(), cols.data(), uint64_t(rp.size() - 1), group_first.data(),
                                       uint64_t(group_first.size() - 1), r0, r1, &ga, &gb));
            return py::make_tuple(ga, gb);
        },
        py::arg("row_pointers"), py::arg("columns"), py::arg("group_first"), py::arg("r0"), py::arg("r1"));
    m.def(
        "plan_needed",
        [](py::array_t<int32_t, py::array::c_style | py::array::forcecast> cols, uint64_t num_cols,
           py::array_t<uint64_t, py::array::c_style | py::array::forcecast> bounds, uint32_t self) {
            const uint32_t parts = uint32_t(bounds.size() - 1);
            std::vector<uint64_t> counts(parts);
            check(argcsr_plan_needed(cols.data(), uint64_t(cols.size()), num_cols, bounds.data(), parts, self,
                                     counts.data(), nullptr));
            uint64_t tot = 0;
            for (uint64_t c : counts) tot += c;
            py::array_t<uint64_t> rows(tot);
            check(argcsr_plan_needed(cols.data(), uint64_t(cols.size()), num_cols, bounds.data(), parts, self,
                                     counts.data(), rows.mutable_data()));
            py::list out;
            uint64_t o = 0;
            for (uint32_t p = 0; p < parts; ++p) {
                out.append(py::array_t<uint64_t>({counts[p]}, {sizeof(uint64_t)}, rows.data() + o));
                o += counts[p];
            }
            return out;
        },
        py::arg("columns"), py::arg("num_cols"), py::arg("bounds"), py::arg("self_rank"));

    py::class_<PyMultiGpu>(m, "MultiGpu")
        .def_static(
            "create_rank",
            [](std::size_t num_rows, std::size_t num_cols, std::size_t nnz, std::uintptr_t rp, std::uintptr_t cols,
               std::uintptr_t vals, const std::string& dtype, bool device_arrays, int rank, int nranks,
               std::optional<py::bytes> nccl_id, std::size_t tpg, std::size_t dcs, int device, std::uint32_t flags,
               int exchange) {
                argcsr_csr_view v = view_from_ptrs(num_rows, num_cols, nnz, rp, cols, vals, dtype, device_arrays);
                std::string id;
                if (nccl_id) {
                    id = *nccl_id;
                    if (id.size() != ARGCSR_NCCL_ID_BYTES) throw ParameterError("nccl_id: 128 bytes");
                }
                auto p = std::make_unique<PyMultiGpu>();
                {
                    py::gil_scoped_release nogil;
                    check(argcsr_mgpu_create_rank(&v, rank, nranks,
                                                  nccl_id ? reinterpret_cast<const unsigned char*>(id.data()) : nullptr,
                                                  tpg, dcs, device, flags, static_cast<argcsr_exchange>(exchange), &p->h));
                }
                p->nlocal = 1;
                return p;
            },
            py::arg("num_rows"), py::arg("num_cols"), py::arg("nnz"), py::arg("row_pointers_ptr"),
            py::arg("columns_ptr"), py::arg("values_ptr"), py::arg("dtype"), py::arg("device_arrays"),
            py::arg("rank"), py::arg("nranks"), py::arg("nccl_id"), py::arg("threads_per_group") = 128,
            py::arg("desired_chunk_size") = 1, py::arg("device") = 0, py::arg("flags") = 0, py::arg("exchange") = 0)
        .def_static(
            "create",
            [](std::size_t num_rows, std::size_t num_cols, std::size_t nnz, std::uintptr_t rp, std::uintptr_t cols,
               std::uintptr_t vals, const std::string& dtype, bool device_arrays, std::vector<int> devices,
               std::size_t tpg, std::size_t dcs, int exchange) {
                argcsr_csr_view v = view_from_ptrs(num_rows, num_cols, nnz, rp, cols, vals, dtype, device_arrays);
                auto p = std::make_unique<PyMultiGpu>();
                {
                    py::gil_scoped_release nogil;
                    check(argcsr_mgpu_create(&v, int(devices.size()), devices.data(), tpg, dcs,
                                             static_cast<argcsr_exchange>(exchange), &p->h));
                }
                p->nlocal = int(devices.size());
                return p;
            },
            py::arg("num_rows"), py::arg("num_cols"), py::arg("nnz"), py::arg("row_pointers_ptr"),
            py::arg("columns_ptr"), py::arg("values_ptr"), py::arg("dtype"), py::arg("device_arrays"),
            py::arg("devices"), py::arg("threads_per_group") = 128, py::arg("desired_chunk_size") = 1,
            py::arg("exchange") = 0)
        .def("info",
             [](const PyMultiGpu& p) {
                 argcsr_mgpu_info_t i{};
                 check(argcsr_mgpu_info(p.get(), &i));
                 py::dict d;
                 d["rank"] = i.rank;
                 d["nranks"] = i.nranks;
                 d["nlocal"] = i.nlocal;
                 d["exchange"] = i.exchange;
                 d["num_rows"] = i.num_rows;
                 d["num_cols"] = i.num_cols;
                 d["nnz"] = i.nnz;
                 d["row_begin"] = i.row_begin;
                 d["row_end"] = i.row_end;
                 d["interior_begin"] = i.interior_begin;
                 d["interior_end"] = i.interior_end;
                 d["halo_recv_rows"] = i.halo_recv_rows;
                 d["step"] = i.step;
                 return d;
             })
        .def(
            "local",
            [](const PyMultiGpu& p, int i) {
                argcsr_dev* s = nullptr;
                check(argcsr_mgpu_local(p.get(), i, &s));
                PyArgCsr a;
                a.dev = std::make_shared<DeviceArgCsr>(DeviceArgCsr::borrow(s));
                return a;
            },
            py::arg("index") = 0, py::keep_alive<0, 1>())
        .def("p2p_export",
             [](const PyMultiGpu& p) {
                 argcsr_mgpu_info_t i{};
                 check(argcsr_mgpu_info(p.get(), &i));
                 unsigned char hnd[64];
                 std::vector<uint64_t> need(2 * size_t(i.nranks));
                 check(argcsr_mgpu_p2p_export(p.get(), hnd, need.data()));
                 return py::make_tuple(py::bytes(reinterpret_cast<const char*>(hnd), 64), need);
             })
        .def(
            "p2p_connect",
            [](PyMultiGpu& p, const std::vector<py::bytes>& handles, const std::vector<std::vector<uint64_t>>& need_all) {
                std::string flat;
                for (const auto& hb : handles) {
                    const std::string s = hb;
                    if (s.size() != 64) throw ParameterError("p2p_connect: IPC handles are 64 bytes");
                    flat += s;
                }
                std::vector<uint64_t> na;
                for (const auto& row : need_all) na.insert(na.end(), row.begin(), row.end());
                check(argcsr_mgpu_p2p_connect(p.get(), reinterpret_cast<const unsigned char*>(flat.data()), na.data()));
            },
            py::arg("handles"), py::arg("need_all"))
        .def(
            "begin",
            [](PyMultiGpu& p, const std::vector<std::uintptr_t>& x0, bool normalize,
               const std::vector<std::uintptr_t>& streams) {
                auto xs = ptr_list(x0, p.nlocal, "begin");
                auto ss = ptr_list(streams, p.nlocal, "begin");
                check(argcsr_mgpu_begin(p.get(), xs.data(), normalize ? 1 : 0, ss.data()));
            },
            py::arg("x0"), py::arg("normalize"), py::arg("streams"))
        .def(
            "step",
            [](PyMultiGpu& p, bool last, const std::vector<std::uintptr_t>& streams) {
                auto ss = ptr_list(streams, p.nlocal, "step");
                check(argcsr_mgpu_step(p.get(), last ? 1 : 0, ss.data()));
            },
            py::arg("last"), py::arg("streams"))
        .def(
            "finish",
            [](PyMultiGpu& p, const std::vector<std::uintptr_t>& x_out, const std::vector<std::uintptr_t>& streams) {
                auto xs = ptr_list(x_out, p.nlocal, "finish");
                auto ss = ptr_list(streams, p.nlocal, "finish");
                double lam = 0.0;
                {
                    py::gil_scoped_release nogil;
                    check(argcsr_mgpu_finish(p.get(), &lam, xs.data(), ss.data()));
                }
                return lam;
            },
            py::arg("x_out"), py::arg("streams"))
        .def(
            "spmv_gather",
            [](PyMultiGpu& p, const std::vector<std::uintptr_t>& x, const std::vector<std::uintptr_t>& out,
               const std::vector<std::uintptr_t>& streams) {
                auto xs = ptr_list(x, p.nlocal, "spmv_gather");
                auto os = ptr_list(out, p.nlocal, "spmv_gather");
                auto ss = ptr_list(streams, p.nlocal, "spmv_gather");
                std::vector<const void*> xc(xs.begin(), xs.end());
                check(argcsr_mgpu_spmv_gather(p.get(), xc.data(), os.data(), ss.data()));
            },
            py::arg("x"), py::arg("out"), py::arg("streams"))
        .def(
            "power_iteration",
            [](PyMultiGpu& p, int iters, py::array x) {
                argcsr_mgpu_info_t i{};
                check(argcsr_mgpu_info(p.get(), &i));
                if (!(x.flags() & py::array::c_style) || !x.writeable() || uint64_t(x.size()) != i.num_cols)
                    throw ParameterError("power_iteration: x must be a writeable contiguous array of num_cols entries");
                double lam = 0.0;
                void* xp = x.mutable_data();
                {
                    py::gil_scoped_release nogil;
                    check(argcsr_mgpu_power_iteration(p.get(), iters, xp, &lam));
                }
                return lam;
            },
            py::arg("iters"), py::arg("x"))
        .def(
            "wait",
            [](PyMultiGpu& p, const std::vector<std::uintptr_t>& streams) {
                auto ss = ptr_list(streams, p.nlocal, "wait");
                check(argcsr_mgpu_wait(p.get(), ss.data()));
            },
            py::arg("streams"))
        .def("check", [](PyMultiGpu& p) { check(argcsr_mgpu_check(p.get())); })
        .def("free", &PyMultiGpu::free);
    m.def("reload_options", &argcsr_reload_options,
          "Re-read the ARGCSR_* experiment switches from the environment (read once otherwise).");
    // multi-GPU step over peer memory (argcsr_gpu.h: argcsr_peer_*)
    m.def(
        "peer_signal",
        [](const std::vector<std::uintptr_t>& flags, std::uint64_t value, std::uintptr_t partial,
           const std::vector<std::uintptr_t>& partial_dst, std::uintptr_t stream) {
            if (!partial_dst.empty() && partial_dst.size() != flags.size())
                throw ParameterError("peer_signal: one partial destination per flag");
            std::vector<uint64_t*> f(flags.size());
            std::vector<double*> d(partial_dst.size());
            for (size_t i = 0; i < f.size(); ++i) f[i] = reinterpret_cast<uint64_t*>(flags[i]);
            for (size_t i = 0; i < d.size(); ++i) d[i] = reinterpret_cast<double*>(partial_dst[i]);
            check(argcsr_peer_signal(f.data(), uint32_t(f.size()), value, reinterpret_cast<const double*>(partial),
                                     d.empty() ? nullptr : d.data(), reinterpret_cast<void*>(stream)));
        },
        py::arg("flag_ptrs"), py::arg("value"), py::arg("partial_ptr") = 0, py::arg("partial_dst_ptrs") = std::vector<std::uintptr_t>{},
        py::arg("stream") = 0);
    m.def(
        "peer_wait",
        [](std::uintptr_t flags, std::uint32_t n, std::uint64_t value, std::uintptr_t stream) {
            check(argcsr_peer_wait(reinterpret_cast<const uint64_t*>(flags), n, value, reinterpret_cast<void*>(stream)));
        },
        py::arg("flags_ptr"), py::arg("n"), py::arg("value"), py::arg("stream") = 0);
    m.def(
        "peer_alloc",
        [](std::uint64_t bytes, int device) {
            void* p = nullptr;
            unsigned char h[64];
            check(argcsr_peer_alloc(bytes, device, &p, h));
            return py::make_tuple(reinterpret_cast<std::uintptr_t>(p), py::bytes(reinterpret_cast<const char*>(h), 64));
        },
        py::arg("bytes"), py::arg("device"));
    m.def(
        "peer_open",
        [](const py::bytes& handle, int device) {
            const std::string h = handle;
            if (h.size() != 64) throw ParameterError("peer_open: an IPC handle is 64 bytes");
            void* p = nullptr;
            check(argcsr_peer_open(reinterpret_cast<const unsigned char*>(h.data()), device, &p));
            return reinterpret_cast<std::uintptr_t>(p);
        },
        py::arg("handle"), py::arg("device"));
    m.def("peer_close", [](std::uintptr_t p) { check(argcsr_peer_close(reinterpret_cast<void*>(p))); }, py::arg("ptr"));
    m.def("peer_free", [](std::uintptr_t p) { check(argcsr_peer_free(reinterpret_cast<void*>(p))); }, py::arg("ptr"));

    py::class_<CsrMatrix>(m, "CsrMatrix")
        .def(py::init<>())
        .def_readonly("num_rows", &CsrMatrix::num_rows)
        .def_readonly("num_cols", &CsrMatrix::num_cols)
        .def_property_readonly("values", [](py::object self) { return view_of(self.cast<const CsrMatrix&>().values, self); })
        .def_property_readonly("columns", [](py::object self) { return view_of(self.cast<const CsrMatrix&>().columns, self); })
        .def_property_readonly("row_pointers", [](py::object self) {
            const auto& rp = self.cast<const CsrMatrix&>().row_pointers;
            return py::array_t<uint64_t>({rp.size()}, {sizeof(uint64_t)}, reinterpret_cast<const uint64_t*>(rp.data()), self);
        })
        .def_property_readonly("nnz", &CsrMatrix::nnz)
        .def_static(
            "from_arrays",
            [](std::size_t num_rows, std::size_t num_cols, py::array_t<uint64_t, py::array::c_style | py::array::forcecast> rp,
               py::array_t<int32_t, py::array::c_style | py::array::forcecast> cols,
               py::array_t<double, py::array::c_style | py::array::forcecast> vals) {
                if (rp.size() != py::ssize_t(num_rows + 1)) throw DimensionError("from_arrays: row_pointers length");
                if (cols.size() != vals.size()) throw DimensionError("from_arrays: columns/values length");
                CsrMatrix A;
                A.num_rows = num_rows;
                A.num_cols = num_cols;
                A.row_pointers.assign(rp.data(), rp.data() + rp.size());
                A.columns = vec_from<int32_t>(cols);
                A.values = vec_from<double>(vals);
                return A;
            },
            py::arg("num_rows"), py::arg("num_cols"), py::arg("row_pointers"), py::arg("columns"), py::arg("values"))
        .def(py::self == py::self)
        .def("__repr__", [](const CsrMatrix& A) {
            return "CsrMatrix(" + std::to_string(A.num_rows) + "x" + std::to_string(A.num_cols) +
                   ", nnz=" + std::to_string(A.nnz()) + ")";
        });

    py::class_<GroupInfo>(m, "GroupInfo")
        .def(py::init([](std::size_t f, std::size_t s, std::size_t o, std::size_t c) { return GroupInfo{f, s, o, c}; }),
             py::arg("first_row") = 0, py::arg("size") = 0, py::arg("offset") = 0, py::arg("chunk_size") = 0)
        .def_readonly("first_row", &GroupInfo::first_row)
        .def_readonly("size", &GroupInfo::size)
        .def_readonly("offset", &GroupInfo::offset)
        .def_readonly("chunk_size", &GroupInfo::chunk_size)
        .def(py::self == py::self)
        .def("__repr__", [](const GroupInfo& g) {
            return "GroupInfo(" + std::to_string(g.first_row) + ", " + std::to_string(g.size) + ", " +
                   std::to_string(g.offset) + ", " + std::to_string(g.chunk_size) + ")";
        });

    py::class_<FormatStats>(m, "FormatStats")
        .def_readonly("explicit_nnz", &FormatStats::explicit_nnz)
        .def_readonly("assigned_padded_slots", &FormatStats::assigned_padded_slots)
        .def_readonly("total_allocated_slots", &FormatStats::total_allocated_slots)
        .def_readonly("padding_ratio", &FormatStats::padding_ratio)
        .def_readonly("estimated_bytes", &FormatStats::estimated_bytes);

    py::class_<argcsr_b200::BalanceStats>(m, "BalanceStats")  // reference bindings.cpp:77-80
        .def_readonly("per_group_nnz", &argcsr_b200::BalanceStats::per_group_nnz)
        .def_readonly("max_over_mean", &argcsr_b200::BalanceStats::max_over_mean)
        .def_readonly("coefficient_of_variation", &argcsr_b200::BalanceStats::coefficient_of_variation);

    py::class_<PyArgCsr>(m, "ArgCsrMatrix")
        .def_property_readonly("num_rows", [](const PyArgCsr& p) { return p.info().num_rows; })
        .def_property_readonly("num_cols", [](const PyArgCsr& p) { return p.info().num_cols; })
        .def_property_readonly("threads_per_group", [](const PyArgCsr& p) { return p.info().threads_per_group; })
        .def_property_readonly("desired_chunk_size", [](const PyArgCsr& p) { return p.info().desired_chunk_size; })
        .def_property_readonly("total_slots", [](const PyArgCsr& p) { return p.info().total_slots; })
        .def_property_readonly("stored_slots", [](const PyArgCsr& p) { return p.info().stored_slots; })
        .def_property_readonly("x_remap", [](const PyArgCsr& p) { return p.info().x_remap != 0; })
        .def_property_readonly("x_used_columns", [](const PyArgCsr& p) { return p.info().x_used_columns; })
        .def_property_readonly("unit_len_bytes", [](const PyArgCsr& p) { return p.info().unit_len_bytes; })
        .def_property_readonly("layout", [](const PyArgCsr& p) {
            return p.info().layout == ARGCSR_LAYOUT_REFERENCE ? "reference" : "compact";
        })
        .def_property_readonly("num_groups", [](const PyArgCsr& p) { return p.info().num_groups; })
        .def_property_readonly("nnz", [](const PyArgCsr& p) { return p.info().nnz; })
        .def_property_readonly("heavy_groups", [](const PyArgCsr& p) { return p.info().heavy_groups; })
        .def_property_readonly("heavy_ctas", [](const PyArgCsr& p) { return p.info().heavy_ctas; })
        .def_property_readonly("light_tiles", [](const PyArgCsr& p) { return p.info().light_tiles; })
        .def_property_readonly("max_chunk_size", [](const PyArgCsr& p) { return p.info().max_chunk_size; })
        .def_property_readonly("device_bytes", [](const PyArgCsr& p) { return p.info().device_bytes; })
        .def_property_readonly("l2_persist_bytes", [](const PyArgCsr& p) { return p.info().l2_persist_bytes; })
        .def_property_readonly("device", [](const PyArgCsr& p) { return p.info().device; })
        .def_property_readonly("dtype", [](const PyArgCsr& p) { return p.info().dtype == ARGCSR_F64 ? "float64" : "float32"; })
        .def_property_readonly("groups", [](const PyArgCsr& p) {
            p.need_meta();
            std::vector<GroupInfo> out(p.info().num_groups);
            const auto& g = *p.groups4;
            for (std::size_t i = 0; i < out.size(); ++i) out[i] = {g[4 * i], g[4 * i + 1], g[4 * i + 2], g[4 * i + 3]};
            return out;
        })
        .def_property_readonly("groups_array", [](py::object self) {
            const auto& p = self.cast<const PyArgCsr&>();
            p.need_meta();
            return py::array_t<uint64_t>({p.groups4->size() / 4, std::size_t(4)}, {4 * sizeof(uint64_t), sizeof(uint64_t)},
                                         p.groups4->data(), self);
        })
        .def_property_readonly("threads_mapping", [](py::object self) {
            const auto& p = self.cast<const PyArgCsr&>();
            p.need_meta();
            return view_of(*p.tm, self);
        })
        .def_property_readonly("values", [](const PyArgCsr& p) {
            p.need_slots();
            return *p.values;
        })
        .def_property_readonly("columns", [](py::object self) {
            const auto& p = self.cast<const PyArgCsr&>();
            p.need_slots();
            return view_of(*p.columns, self);
        })
        .def("spmv_device",
             [](const PyArgCsr& p, std::uintptr_t x, std::uintptr_t y, std::uintptr_t stream) {
                 check(argcsr_dev_spmv(p.dev->handle(), reinterpret_cast<const void*>(x), reinterpret_cast<void*>(y),
                                       reinterpret_cast<void*>(stream)));
             },
             py::arg("x_ptr"), py::arg("y_ptr"), py::arg("stream") = 0)
        .def("spmv_scaled_device",
             [](const PyArgCsr& p, std::uintptr_t x, std::uintptr_t scale, std::uintptr_t y, std::uintptr_t stream) {
                 check(argcsr_dev_spmv_scaled(p.dev->handle(), reinterpret_cast<const void*>(x),
                                              reinterpret_cast<const double*>(scale), reinterpret_cast<void*>(y),
                                              reinterpret_cast<void*>(stream)));
             },
             py::arg("x_ptr"), py::arg("x_scale_ptr"), py::arg("y_ptr"), py::arg("stream") = 0)
        .def("spmv_norm2_device",
             [](const PyArgCsr& p, std::uintptr_t x, std::uintptr_t scale, std::uintptr_t y, std::uintptr_t norm2,
                bool scale_is_norm2, std::uintptr_t stream) {
                 check(argcsr_dev_spmv_norm2(p.dev->handle(), reinterpret_cast<const void*>(x),
                                             reinterpret_cast<const double*>(scale), reinterpret_cast<void*>(y),
                                             reinterpret_cast<double*>(norm2), scale_is_norm2 ? ARGCSR_SCALE_IS_NORM2 : 0u,
                                             reinterpret_cast<void*>(stream)));
             },
             py::arg("x_ptr"), py::arg("x_scale_ptr"), py::arg("y_ptr"), py::arg("norm2_ptr"),
             py::arg("scale_is_norm2") = false, py::arg("stream") = 0)
        .def("spmv_peer_device",
             [](const PyArgCsr& p, std::uintptr_t x, std::uintptr_t scale, std::uint64_t gb, std::uint64_t ge,
                std::uintptr_t y, const std::vector<std::uintptr_t>& peers, const std::vector<std::uint64_t>& rows,
                std::uint32_t flags, std::uintptr_t stream) {
                 if (!rows.empty() && rows.size() != 2 * peers.size())
                     throw ParameterError("spmv_peer_device: one [lo, hi) row range per peer");
                 std::vector<void*> pp(peers.size());
                 for (size_t i = 0; i < peers.size(); ++i) pp[i] = reinterpret_cast<void*>(peers[i]);
                 check(argcsr_dev_spmv_peer(p.dev->handle(), reinterpret_cast<const void*>(x),
                                            reinterpret_cast<const double*>(scale), gb, ge, reinterpret_cast<void*>(y),
                                            pp.data(), uint32_t(pp.size()), rows.empty() ? nullptr : rows.data(),
                                            flags, reinterpret_cast<void*>(stream)));
             },
             py::arg("x_ptr"), py::arg("x_scale_ptr"), py::arg("group_begin"), py::arg("group_end"), py::arg("y_ptr"),
             py::arg("peer_y_ptrs"), py::arg("peer_rows") = std::vector<std::uint64_t>{}, py::arg("flags") = 0u,
             py::arg("stream") = 0)
        .def("spmv_ex_device",
             [](const PyArgCsr& p, std::uintptr_t x, std::uintptr_t scale, std::uint64_t gb, std::uint64_t ge,
                std::uintptr_t y, std::uint32_t flags, std::uintptr_t stream) {
                 check(argcsr_dev_spmv_ex(p.dev->handle(), reinterpret_cast<const void*>(x),
                                          reinterpret_cast<const double*>(scale), gb, ge, reinterpret_cast<void*>(y),
                                          flags, reinterpret_cast<void*>(stream)));
             },
             py::arg("x_ptr"), py::arg("x_scale_ptr"), py::arg("group_begin"), py::arg("group_end"), py::arg("y_ptr"),
             py::arg("flags") = 0u, py::arg("stream") = 0)
        .def("spmv_groups_device",
             [](const PyArgCsr& p, std::uintptr_t x, std::uint64_t gb, std::uint64_t ge, std::uintptr_t y,
                std::uintptr_t stream) {
                 check(argcsr_dev_spmv_groups(p.dev->handle(), reinterpret_cast<const void*>(x), gb, ge,
                                              reinterpret_cast<void*>(y), reinterpret_cast<void*>(stream)));
             },
             py::arg("x_ptr"), py::arg("group_begin"), py::arg("group_end"), py::arg("y_ptr"), py::arg("stream") = 0)
        .def("spmv_host_staged",
             [](const PyArgCsr& p, std::uintptr_t xh, std::uintptr_t xd, std::uintptr_t yd, std::uintptr_t yh,
                std::uintptr_t stream) {
                 py::gil_scoped_release nogil;
                 check(argcsr_dev_spmv_host_staged(p.dev->handle(), reinterpret_cast<const void*>(xh),
                                                   reinterpret_cast<void*>(xd), reinterpret_cast<void*>(yd),
                                                   reinterpret_cast<void*>(yh), reinterpret_cast<void*>(stream)));
             },
             py::arg("x_host_ptr"), py::arg("x_dev_ptr"), py::arg("y_dev_ptr"), py::arg("y_host_ptr"), py::arg("stream") = 0)
        .def("spmv_host_async",
             [](const PyArgCsr& p, std::uintptr_t xh, std::uintptr_t yh, std::uintptr_t stream) {
                 check(argcsr_dev_spmv_host_async(p.dev->handle(), reinterpret_cast<const void*>(xh),
                                                  reinterpret_cast<void*>(yh), reinterpret_cast<void*>(stream)));
             },
             py::arg("x_host_ptr"), py::arg("y_host_ptr"), py::arg("stream") = 0)
        .def("host_wait",
             [](const PyArgCsr& p) {
                 py::gil_scoped_release nogil;
                 check(argcsr_dev_host_wait(p.dev->handle()));
             })
        .def("free", [](PyArgCsr& p) { p.dev->reset(); })
        .def("__eq__", [](const PyArgCsr& a, const PyArgCsr& b) {
            if (a.info().num_rows != b.info().num_rows || a.info().num_cols != b.info().num_cols ||
                a.info().threads_per_group != b.info().threads_per_group || a.info().dtype != b.info().dtype)
                return false;
            a.need_meta(), b.need_meta(), a.need_slots(), b.need_slots();
            if (*a.groups4 != *b.groups4 || *a.tm != *b.tm || *a.columns != *b.columns) return false;
            return std::memcmp(a.values->data(), b.values->data(), a.values->nbytes()) == 0;
        })
        .def("__repr__", [](const PyArgCsr& p) {
            return "ArgCsrMatrix(" + std::to_string(p.info().num_rows) + "x" + std::to_string(p.info().num_cols) +
                   ", tpg=" + std::to_string(p.info().threads_per_group) + ", groups=" +
                   std::to_string(p.info().num_groups) + ", slots=" + std::to_string(p.info().total_slots) +
                   ", device=" + std::to_string(p.info().device) + ")";
        });

    m.def(
        "csr_from_triplets",
        [](std::size_t num_rows, std::size_t num_cols,
           const std::vector<std::tuple<std::size_t, std::size_t, double>>& entries) {
            std::vector<host_io::Entry> ts;
            ts.reserve(entries.size());
            for (const auto& [r, c, v] : entries) ts.push_back({r, c, v});
            return host_io::assemble_csr(num_rows, num_cols, ts);
        },
        py::arg("num_rows"), py::arg("num_cols"), py::arg("entries"),
        "Builds CSR from (row, col, value) tuples; duplicates are summed.");

    m.def(
        "triplets_from_csr",
        [](const CsrMatrix& A) {
            std::vector<std::tuple<std::size_t, std::size_t, double>> out;
            out.reserve(A.nnz());
            for (std::size_t r = 0; r < A.num_rows; ++r)
                for (std::size_t k = A.row_pointers[r]; k < A.row_pointers[r + 1]; ++k)
                    out.emplace_back(r, std::size_t(A.columns[k]), A.values[k]);
            return out;
        },
        py::arg("matrix"));

    m.def(
        "argcsr_from_csr",
        [](const CsrMatrix& A, std::size_t tpg, std::size_t dcs, int device, std::uint32_t flags) {
            argcsr_csr_view v{};
            v.num_rows = A.num_rows;
            v.num_cols = A.num_cols;
            v.nnz = A.nnz();
            v.row_pointers = reinterpret_cast<const uint64_t*>(A.row_pointers.data());
            v.columns = A.columns.data();
            v.values = A.values.data();
            v.dtype = ARGCSR_F64;
            v.space = ARGCSR_HOST;
            argcsr_dev* h = nullptr;
            {
                py::gil_scoped_release nogil;
                check(argcsr_dev_convert_ex(&v, tpg, dcs, device, nullptr, flags, &h));
            }
            return make_handle(h);
        },
        py::arg("matrix"), py::arg("threads_per_group") = kDefaultThreadsPerGroup,
        py::arg("desired_chunk_size") = kDefaultDesiredChunkSize, py::arg("device") = 0, py::arg("flags") = 0u);

    py::class_<PyEllpack>(m, "EllpackMatrix")
        .def_property_readonly("num_rows", [](const PyEllpack& p) { return p.info().num_rows; })
        .def_property_readonly("dtype", [](const PyEllpack& p) { return p.info().dtype == ARGCSR_F64 ? "float64" : "float32"; })
        .def_property_readonly("num_cols", [](const PyEllpack& p) { return p.info().num_cols; })
        .def_property_readonly("width", [](const PyEllpack& p) { return p.info().width; })
        .def_property_readonly("total_slots", [](const PyEllpack& p) { return p.info().total_slots; })
        .def_property_readonly("device_bytes", [](const PyEllpack& p) { return p.info().device_bytes; })
        .def_property_readonly("values", [](const PyEllpack& p) { return p.values(); })
        .def_property_readonly("columns", [](const PyEllpack& p) { return p.columns(); })
        .def("spmv_device", [](const PyEllpack& p, std::uintptr_t x, std::uintptr_t y, std::uintptr_t stream) {
            check(argcsr_sell_spmv(p.s->h, reinterpret_cast<const void*>(x), reinterpret_cast<void*>(y),
                                   reinterpret_cast<void*>(stream)));
        }, py::arg("x_ptr"), py::arg("y_ptr"), py::arg("stream") = 0);
    py::class_<PySliced>(m, "SlicedEllpackMatrix")
        .def_property_readonly("num_rows", [](const PySliced& p) { return p.info().num_rows; })
        .def_property_readonly("dtype", [](const PySliced& p) { return p.info().dtype == ARGCSR_F64 ? "float64" : "float32"; })
        .def_property_readonly("num_cols", [](const PySliced& p) { return p.info().num_cols; })
        .def_property_readonly("slice_size", [](const PySliced& p) { return p.info().slice_size; })
        .def_property_readonly("total_slots", [](const PySliced& p) { return p.info().total_slots; })
        .def_property_readonly("device_bytes", [](const PySliced& p) { return p.info().device_bytes; })
        .def("num_slices", [](const PySliced& p) { return p.info().num_slices; })
        .def_property_readonly("slice_widths", [](const PySliced& p) { return p.widths(); })
        .def_property_readonly("slice_offsets", [](const PySliced& p) { return p.offsets(); })
        .def_property_readonly("values", [](const PySliced& p) { return p.values(); })
        .def_property_readonly("columns", [](const PySliced& p) { return p.columns(); })
        .def("spmv_device", [](const PySliced& p, std::uintptr_t x, std::uintptr_t y, std::uintptr_t stream) {
            check(argcsr_sell_spmv(p.s->h, reinterpret_cast<const void*>(x), reinterpret_cast<void*>(y),
                                   reinterpret_cast<void*>(stream)));
        }, py::arg("x_ptr"), py::arg("y_ptr"), py::arg("stream") = 0);

    m.def(
        "ellpack_from_csr",
        [](const CsrMatrix& A, int device) {
            const argcsr_csr_view v = host_view(A);
            argcsr_sell* h = nullptr;
            {
                py::gil_scoped_release nogil;
                check(argcsr_ell_convert(&v, device, nullptr, &h));
            }
            PyEllpack p;
            p.s = std::make_shared<SellHandle>(h);
            return p;
        },
        py::arg("matrix"), py::arg("device") = 0);
    m.def(
        "sliced_from_csr",
        [](const CsrMatrix& A, std::size_t slice_size, int device) {
            const argcsr_csr_view v = host_view(A);
            argcsr_sell* h = nullptr;
            {
                py::gil_scoped_release nogil;
                check(argcsr_sell_convert(&v, slice_size, device, nullptr, &h));
            }
            PySliced p;
            p.s = std::make_shared<SellHandle>(h);
            return p;
        },
        py::arg("matrix"), py::arg("slice_size") = 32, py::arg("device") = 0);
    m.def(
        "sell_from_device_csr",
        [](std::uint64_t num_rows, std::uint64_t num_cols, std::uint64_t nnz, std::uintptr_t rp, std::uintptr_t cols,
           std::uintptr_t vals, const std::string& dtype, std::size_t slice_size, int device, std::uintptr_t stream) {
            argcsr_csr_view v{};
            v.num_rows = num_rows;
            v.num_cols = num_cols;
            v.nnz = nnz;
            v.row_pointers = reinterpret_cast<const uint64_t*>(rp);
            v.columns = reinterpret_cast<const int32_t*>(cols);
            v.values = reinterpret_cast<const void*>(vals);
            v.dtype = dtype == "float32" ? ARGCSR_F32 : ARGCSR_F64;
            v.space = ARGCSR_DEVICE;
            argcsr_sell* h = nullptr;
            {
                py::gil_scoped_release nogil;
                if (slice_size == 0) check(argcsr_ell_convert(&v, device, reinterpret_cast<void*>(stream), &h));
                else check(argcsr_sell_convert(&v, slice_size, device, reinterpret_cast<void*>(stream), &h));
            }
            auto hs = std::make_shared<SellHandle>(h);
            if (slice_size == 0) {
                PyEllpack p;
                p.s = hs;
                return py::cast(p);
            }
            PySliced p;
            p.s = hs;
            return py::cast(p);
        },
        py::arg("num_rows"), py::arg("num_cols"), py::arg("nnz"), py::arg("row_pointers_ptr"), py::arg("columns_ptr"),
        py::arg("values_ptr"), py::arg("dtype") = "float64", py::arg("slice_size") = 0, py::arg("device") = 0,
        py::arg("stream") = 0);
    m.def("csr_from_ellpack", [](const PyEllpack& p) { return p.to_csr(); }, py::arg("matrix"));
    m.def("csr_from_sliced", [](const PySliced& p) { return p.to_csr(); }, py::arg("matrix"));
    m.def("spmv_ellpack_host", &sell_spmv_host<PyEllpack>, py::arg("matrix"), py::arg("x"));
    m.def("spmv_sliced_host", &sell_spmv_host<PySliced>, py::arg("matrix"), py::arg("x"));

    m.def(
        "read_matrix_market",
        [](const std::string& path) { return host_io::read_matrix_market_file(path); },
        py::arg("path"));
    m.def(
        "write_matrix_market",
        [](const std::string& path, const CsrMatrix& A) { host_io::write_matrix_market_file(path, A); },
        py::arg("path"), py::arg("matrix"));

    m.def(
        "write_binary",
        [](const std::string& path, const PyArgCsr& p) {
            py::gil_scoped_release nogil;
            check(argcsr_dev_write_binary(p.dev->handle(), path.c_str()));
        },
        py::arg("path"), py::arg("matrix"));

    m.def(
        "read_binary",
        [](const std::string& path, std::size_t tpg, std::size_t dcs, int device, std::uint32_t flags) {
            argcsr_dev* h = nullptr;
            {
                py::gil_scoped_release nogil;
                check(argcsr_dev_read_binary(path.c_str(), tpg, dcs, device, nullptr, flags, &h));
            }
            return make_handle(h);
        },
        py::arg("path"), py::arg("threads_per_group") = kDefaultThreadsPerGroup,
        py::arg("desired_chunk_size") = kDefaultDesiredChunkSize, py::arg("device") = 0, py::arg("flags") = 0u);

    m.def(
        "argcsr_from_reference_arrays",
        [](std::uint64_t num_rows, std::uint64_t num_cols, std::uint64_t tpg, py::array groups, py::array tm,
           py::array values, py::array columns, int device, std::uint32_t flags) {
            auto g = py::array_t<uint64_t, py::array::c_style | py::array::forcecast>(groups);
            auto t = py::array_t<uint64_t, py::array::c_style | py::array::forcecast>(tm);
            auto c = py::array_t<int32_t, py::array::c_style | py::array::forcecast>(columns);
            py::array v;
            argcsr_argcsr_view view{};
            if (py::dtype(values.dtype()).is(py::dtype::of<float>())) {
                v = py::array_t<float, py::array::c_style | py::array::forcecast>(values);
                view.dtype = ARGCSR_F32;
            } else {
                v = py::array_t<double, py::array::c_style | py::array::forcecast>(values);
                view.dtype = ARGCSR_F64;
            }
            if (g.size() % 4) throw DimensionError("argcsr_from_reference_arrays: groups must be G x 4");
            if (t.size() != py::ssize_t(num_rows)) throw DimensionError("argcsr_from_reference_arrays: threads_mapping length");
            if (v.size() != c.size()) throw DimensionError("argcsr_from_reference_arrays: values/columns lengths differ");
            view.num_rows = num_rows;
            view.num_cols = num_cols;
            view.threads_per_group = tpg;
            view.num_groups = uint64_t(g.size() / 4);
            view.groups4 = g.data();
            view.threads_mapping = t.data();
            view.values = v.data();
            view.columns = c.data();
            view.total_slots = uint64_t(c.size());
            argcsr_dev* h = nullptr;
            {
                py::gil_scoped_release nogil;
                check(argcsr_dev_import(&view, device, nullptr, flags, &h));
            }
            return make_handle(h);
        },
        py::arg("num_rows"), py::arg("num_cols"), py::arg("threads_per_group"), py::arg("groups"),
        py::arg("threads_mapping"), py::arg("values"), py::arg("columns"), py::arg("device") = 0,
        py::arg("flags") = 0u);

    m.def("argcsr_from_csr_arrays", &convert_arrays, py::arg("num_rows"), py::arg("num_cols"), py::arg("row_pointers"),
          py::arg("columns"), py::arg("values"), py::arg("threads_per_group") = kDefaultThreadsPerGroup,
          py::arg("desired_chunk_size") = kDefaultDesiredChunkSize, py::arg("device") = 0, py::arg("flags") = 0u);

    m.def(
        "argcsr_from_device_csr",
        [](std::uint64_t num_rows, std::uint64_t num_cols, std::uint64_t nnz, std::uintptr_t rp, std::uintptr_t cols,
           std::uintptr_t vals, const std::string& dtype, std::size_t tpg, std::size_t dcs, int device,
           std::uintptr_t stream, std::uint32_t flags) {
            argcsr_csr_view v{};
            v.num_rows = num_rows;
            v.num_cols = num_cols;
            v.nnz = nnz;
            v.row_pointers = reinterpret_cast<const uint64_t*>(rp);
            v.columns = reinterpret_cast<const int32_t*>(cols);
            v.values = reinterpret_cast<const void*>(vals);
            if (dtype == "float64") v.dtype = ARGCSR_F64;
            else if (dtype == "float32") v.dtype = ARGCSR_F32;
            else throw ParameterError("argcsr_from_device_csr: dtype must be float64 or float32");
            v.space = ARGCSR_DEVICE;
            argcsr_dev* h = nullptr;
            {
                py::gil_scoped_release nogil;
                check(argcsr_dev_convert_ex(&v, tpg, dcs, device, reinterpret_cast<void*>(stream), flags, &h));
            }
            return make_handle(h);
        },
        py::arg("num_rows"), py::arg("num_cols"), py::arg("nnz"), py::arg("row_pointers_ptr"), py::arg("columns_ptr"),
        py::arg("values_ptr"), py::arg("dtype") = "float64", py::arg("threads_per_group") = kDefaultThreadsPerGroup,
        py::arg("desired_chunk_size") = kDefaultDesiredChunkSize, py::arg("device") = 0, py::arg("stream") = 0,
        py::arg("flags") = 0u);

    m.def(
        "csr_from_argcsr",
        [](const PyArgCsr& p) {
            if (p.info().dtype != ARGCSR_F64) throw UnsupportedError("csr_from_argcsr: fp32 handle");
            return argcsr_b200::csr_from_argcsr(*p.dev);
        },
        py::arg("matrix"));

    m.def(
        "csr_arrays_from_argcsr",
        [](const PyArgCsr& p) {
            const std::size_t N = p.info().num_rows, nnz = p.info().nnz;
            py::array_t<uint64_t> rp(N + 1);
            py::array_t<int32_t> cols(nnz);
            py::array vals = new_array(p.info().dtype == ARGCSR_F64, nnz);
            check(argcsr_dev_to_csr(p.dev->handle(), rp.mutable_data(), cols.mutable_data(), vals.mutable_data()));
            return py::make_tuple(rp, cols, vals);
        },
        py::arg("matrix"));

    m.def(
        "spmv_host",
        [](const PyArgCsr& p, py::array x) {
            const bool f64 = p.info().dtype == ARGCSR_F64;
            py::array xc = f64 ? py::array(py::array_t<double, py::array::c_style | py::array::forcecast>(x))
                               : py::array(py::array_t<float, py::array::c_style | py::array::forcecast>(x));
            py::array y = new_array(f64, p.info().num_rows);
            const void* xp = xc.data();
            void* yp = y.mutable_data();
            const uint64_t n = uint64_t(xc.size());
            {
                py::gil_scoped_release nogil;
                check(argcsr_dev_spmv_host(p.dev->handle(), xp, n, yp));
            }
            return y;
        },
        py::arg("matrix"), py::arg("x"));

    m.def(
        "chunk_entries",
        [](const PyArgCsr& p, std::size_t g, std::size_t c) {
            const std::size_t cap = p.info().max_chunk_size + 1;
            std::vector<double> v(cap);
            std::vector<float> vf(cap);
            std::vector<int32_t> cl(cap);
            uint64_t n = 0;
            const bool f64 = p.info().dtype == ARGCSR_F64;
            check(argcsr_dev_chunk_entries(p.dev->handle(), g, c, f64 ? static_cast<void*>(v.data()) : vf.data(),
                                           cl.data(), cap, &n));
            std::vector<std::pair<double, int32_t>> out;
            for (uint64_t i = 0; i < n; ++i) out.emplace_back(f64 ? v[i] : double(vf[i]), cl[i]);
            return out;
        },
        py::arg("matrix"), py::arg("group_index"), py::arg("chunk_index"));

    m.def(
        "padding_stats", [](const PyArgCsr& p) { return argcsr_b200::padding_stats(*p.dev); }, py::arg("matrix"));
    m.def(
        "balance_stats", [](const PyArgCsr& p) { return argcsr_b200::balance_stats(*p.dev); }, py::arg("matrix"));

    m.def(
        "partition_rows",
        [](py::array_t<uint64_t, py::array::c_style | py::array::forcecast> rp, uint32_t parts) {
            py::array_t<uint64_t> out(parts + 1);
            check(argcsr_partition_rows(rp.data(), uint64_t(rp.size()) - 1, parts, out.mutable_data()));
            return out;
        },
        py::arg("row_pointers"), py::arg("parts"));
}
