// TEST INFRASTRUCTURE ONLY.  The reference's read_matrix_market_file
// (proj/src/io.cpp:42-136) run in its own process: reads a Matrix Market file
// and writes the resulting CsrMatrix with the reference's write_binary_file
// (CSR container, io.cpp:250-257), or prints the error and exits 1.  A
// separate process because the reference's iostream code and the Python
// process's C++ runtime do not mix in-process (segfault in ctypes).
#include <cstdio>
#include <exception>

#include "argcsr/io.hpp"

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: ref_mm_tool in.mtx out.spfmt\n");
        return 2;
    }
    try {
        argcsr::write_binary_file(argv[2], argcsr::read_matrix_market_file(argv[1]));
    } catch (const std::exception& e) {
        std::printf("%s\n", e.what());
        return 1;
    }
    return 0;
}
