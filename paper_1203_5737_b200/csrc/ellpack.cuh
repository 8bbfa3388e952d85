// ELLPACK / Sliced ELLPACK device formats (ellpack.cu).
#pragma once

#include "common.cuh"

// Opaque handle behind argcsr_sell* (include/argcsr_gpu.h).  ELLPACK is the
// single-slice case (slice_size = num_rows).
struct argcsr_sell {
    int device = 0;
    argcsr_dtype dtype = ARGCSR_F64;
    bool ellpack = false;
    uint64_t num_rows = 0, num_cols = 0, nnz = 0, slice_size = 0, num_slices = 0, total_slots = 0;
    uint64_t* width = nullptr;   // [num_slices]
    uint64_t* offset = nullptr;  // [num_slices + 1] exclusive scan of width * rows_in_slice
    void* values = nullptr;      // [total_slots] f64 | f32, padding +0.0
    int32_t* columns = nullptr;  // [total_slots], padding -1
    size_t device_bytes = 0;
};

namespace argcsr_gpu {

// m carries device, dtype, rows, cols, slice_size; rp / cols / vals on the device.
void sell_convert(argcsr_sell* m, const uint64_t* rp, const int32_t* cols, const void* vals, cudaStream_t s);
void sell_spmv(const argcsr_sell* m, const void* x, void* y, cudaStream_t s);

}  // namespace argcsr_gpu
