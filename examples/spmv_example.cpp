// A reference-style C++ program on the B200 path: include/argcsr_gpu.hpp has
// the reference's names (CsrMatrix, ArgCsrMatrix, argcsr_from_csr,
// spmv_argcsr, csr_from_argcsr, write_binary_file, ...); the converted matrix
// lives on the GPU.
//
//   g++ -std=c++20 -O2 -I include examples/spmv_example.cpp \
//       -L paper_1203_5737_b200 -largcsr_gpu -Wl,-rpath,$PWD/paper_1203_5737_b200 -o spmv_example
//   ./spmv_example [n] [out.spfmt]
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "argcsr_gpu.hpp"

using namespace argcsr_b200;

// 2-D 5-point Laplacian on an n x n grid, ascending columns.
static CsrMatrix laplacian(std::size_t n) {
    CsrMatrix A;
    A.num_rows = A.num_cols = n * n;
    A.row_pointers.push_back(0);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) {
            const std::size_t r = i * n + j;
            auto add = [&](std::size_t c, double v) { A.columns.push_back(index_t(c)), A.values.push_back(v); };
            if (i > 0) add(r - n, -1.0);
            if (j > 0) add(r - 1, -1.0);
            add(r, 4.0);
            if (j + 1 < n) add(r + 1, -1.0);
            if (i + 1 < n) add(r + n, -1.0);
            A.row_pointers.push_back(A.columns.size());
        }
    return A;
}

int main(int argc, char** argv) {
    const std::size_t n = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 256;
    try {
        const CsrMatrix A = laplacian(n);
        const DeviceArgCsr M = argcsr_from_csr(A);  // tpg 128, dcs 1 (argcsr.hpp:101-104)
        DenseVector x(A.num_cols);
        for (std::size_t j = 0; j < x.size(); ++j) x[j] = 1.0 + 0.0625 * double(j % 13);
        const DenseVector y = spmv_argcsr(M, x);
        double err = 0.0;  // against a plain host CSR product (same order: no FMA differences at 5 terms)
        for (std::size_t r = 0; r < A.num_rows; ++r) {
            double s = 0.0;
            for (std::size_t k = A.row_pointers[r]; k < A.row_pointers[r + 1]; ++k) s += A.values[k] * x[A.columns[k]];
            err = std::fmax(err, std::fabs(s - y[r]));
        }
        const CsrMatrix B = csr_from_argcsr(M);
        const bool lossless = B.row_pointers == A.row_pointers && B.columns == A.columns && B.values == A.values;
        if (argc > 2) {
            write_binary_file(argv[2], M);
            const DeviceArgCsr M2 = read_binary_file(argv[2]);
            if (spmv_argcsr(M2, x) != y) throw CorrectnessError("binary round trip changed the product");
        }
        std::printf("rows=%zu groups=%zu slots=%zu max|dy|=%.3g lossless=%d\n", M.num_rows(), M.num_groups(),
                    M.total_slots(), err, int(lossless));
        return err <= 1e-12 && lossless ? 0 : 1;
    } catch (const Error& e) {
        std::fprintf(stderr, "argcsr error: %s\n", e.what());
        return 2;
    }
}
