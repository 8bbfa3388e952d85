// Conversion entry point (convert.cu).
#pragma once

#include "common.cuh"

namespace argcsr_gpu {

// Fills every device array of `m` from a device-resident CSR.  m->num_rows,
// num_cols, nnz, tpg, dcs and dtype must be set and validated by the caller.
void convert_device_csr(argcsr_dev* m, const uint64_t* rp, const int32_t* cols, const void* vals,
                        cudaStream_t s);

// Device handle from the reference arrays (host memory): groups as
// {first_row, size, offset, chunk_size} x G, threads_mapping [num_rows],
// values / columns [S].  m carries rows, cols, tpg, dtype, layout.
void import_reference(argcsr_dev* m, uint64_t G, const uint64_t* groups4, const uint64_t* tm, const void* vals,
                      const int32_t* cols, uint64_t S, cudaStream_t s);

}  // namespace argcsr_gpu
