// The multi-GPU C-ABI from C++ (no Python, no torch): a row-partitioned
// power iteration (config C5's algorithm) through argcsr_mgpu_*, checked
// against a plain CPU power iteration of the same CSR.
//
//   g++ -std=c++20 -O2 -I include examples/mgpu_example.cpp
//       -L paper_1203_5737_b200 -largcsr_gpu -Wl,-rpath,$PWD/paper_1203_5737_b200 -o mgpu_example
//   ./mgpu_example [n] [iters]
//
// Runs (1) rank 0 of a 1-rank job created from an ncclUniqueId (the one-
// process-per-GPU form: the NCCL all-reduce / all-gather execute on a
// one-rank communicator), and (2) the one-process form over the visible
// devices (argcsr_mgpu_create) with the p2p exchange, virtual ranks sharing
// device 0 when fewer GPUs are visible.  Exit 0 when both match the CPU run
// (|dlambda| <= 1e-10 lambda, max|dx| <= 1e-9); 2 without a CUDA device.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "argcsr_gpu.h"

namespace {

struct Csr {
    uint64_t n = 0;
    std::vector<uint64_t> rp{0};
    std::vector<int32_t> cols;
    std::vector<double> vals;
};

// 27-point stencil on an n^3 grid, ascending columns.
Csr stencil27(uint64_t n) {
    Csr A;
    A.n = n * n * n;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < n; ++j)
            for (uint64_t k = 0; k < n; ++k) {
                for (int di = -1; di <= 1; ++di)
                    for (int dj = -1; dj <= 1; ++dj)
                        for (int dk = -1; dk <= 1; ++dk) {
                            const int64_t ii = int64_t(i) + di, jj = int64_t(j) + dj, kk = int64_t(k) + dk;
                            if (ii < 0 || jj < 0 || kk < 0 || ii >= int64_t(n) || jj >= int64_t(n) || kk >= int64_t(n))
                                continue;
                            A.cols.push_back(int32_t((ii * int64_t(n) + jj) * int64_t(n) + kk));
                            A.vals.push_back(di == 0 && dj == 0 && dk == 0 ? 26.0 : -1.0);
                        }
                A.rp.push_back(A.cols.size());
            }
    return A;
}

// CPU power iteration: x <- A x / ||A x||, lambda = ||A x_{iters-1}||.
double cpu_power_iteration(const Csr& A, std::vector<double>& x, int iters) {
    std::vector<double> y(A.n);
    double s2 = 0.0;
    for (int it = 0; it < iters; ++it) {
        s2 = 0.0;
        for (uint64_t r = 0; r < A.n; ++r) {
            double acc = 0.0;
            for (uint64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) acc += A.vals[k] * x[A.cols[k]];
            y[r] = acc;
            s2 += acc * acc;
        }
        const double s = 1.0 / std::sqrt(s2);
        for (uint64_t r = 0; r < A.n; ++r) x[r] = y[r] * s;
    }
    return std::sqrt(s2);
}

bool check(argcsr_status s, const char* what) {
    if (s == ARGCSR_OK) return true;
    std::fprintf(stderr, "%s failed: %s: %s\n", what, argcsr_status_name(s), argcsr_last_error());
    return false;
}

bool compare(const char* name, double lam, const std::vector<double>& x, double lam_ref,
             const std::vector<double>& x_ref) {
    double dx = 0.0;
    for (size_t i = 0; i < x.size(); ++i) dx = std::fmax(dx, std::fabs(x[i] - x_ref[i]));
    const bool ok = std::fabs(lam - lam_ref) <= 1e-10 * std::fabs(lam_ref) && dx <= 1e-9;
    std::printf("%s: lambda=%.15g (cpu %.15g) max|dx|=%.3e ok=%d\n", name, lam, lam_ref, dx, ok ? 1 : 0);
    return ok;
}

}  // namespace

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 24;
    const int iters = argc > 2 ? std::atoi(argv[2]) : 30;
    const Csr A = stencil27(n);
    argcsr_csr_view v{};
    v.num_rows = v.num_cols = A.n;
    v.nnz = A.cols.size();
    v.row_pointers = A.rp.data();
    v.columns = A.cols.data();
    v.values = A.vals.data();
    v.dtype = ARGCSR_F64;
    v.space = ARGCSR_HOST;

    std::vector<double> x_ref(A.n);
    for (uint64_t j = 0; j < A.n; ++j) x_ref[j] = 1.0 + 0.0625 * double(j % 13);  // bench_input
    const std::vector<double> x0 = x_ref;
    const double lam_ref = cpu_power_iteration(A, x_ref, iters);

    // (1) one-process-per-GPU form, rank 0 of 1, NCCL communicator from an id
    unsigned char id[ARGCSR_NCCL_ID_BYTES];
    argcsr_mgpu* h = nullptr;
    argcsr_status st = argcsr_mgpu_unique_id(id);
    if (st == ARGCSR_OK) st = argcsr_mgpu_create_rank(&v, 0, 1, id, 128, 1, 0, 0, ARGCSR_EXCHANGE_AUTO, &h);
    if (st == ARGCSR_E_CUDA) {
        std::fprintf(stderr, "%s\n", argcsr_last_error());
        return 2;
    }
    if (!check(st, "argcsr_mgpu_create_rank")) return 1;
    std::vector<double> x = x0;
    double lam = 0.0;
    bool ok = check(argcsr_mgpu_power_iteration(h, iters, x.data(), &lam), "argcsr_mgpu_power_iteration") &&
              compare("create_rank(1 rank, NCCL)", lam, x, lam_ref, x_ref);
    ok = ok && check(argcsr_mgpu_check(h), "argcsr_mgpu_check");
    argcsr_mgpu_free(h);

    // (2) one process, P ranks, p2p exchange (virtual ranks on device 0 if needed)
    const int P = 3;
    std::vector<int> devs(P, 0);
    argcsr_mgpu* g = nullptr;
    if (ok && check(argcsr_mgpu_create(&v, P, devs.data(), 128, 1, ARGCSR_EXCHANGE_P2P, &g), "argcsr_mgpu_create")) {
        argcsr_mgpu_info_t info{};
        check(argcsr_mgpu_info(g, &info), "argcsr_mgpu_info");
        x = x0;
        ok = check(argcsr_mgpu_power_iteration(g, iters, x.data(), &lam), "argcsr_mgpu_power_iteration(p2p)") &&
             compare("create(3 virtual ranks, p2p)", lam, x, lam_ref, x_ref) && info.nranks == P &&
             info.exchange == ARGCSR_EXCHANGE_P2P;
        argcsr_mgpu_free(g);
    } else {
        ok = false;
    }
    return ok ? 0 : 1;
}
