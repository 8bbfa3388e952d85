// Conversion entry point (convert.cu).
#pragma once

#include "common.cuh"

namespace argcsr_gpu {

// Fills every device array of `m` from a device-resident CSR.  m->num_rows,
// num_cols, nnz, tpg, dcs and dtype must be set and validated by the caller.
void convert_device_csr(argcsr_dev* m, const uint64_t* rp, const int32_t* cols, const void* vals,
                        cudaStream_t s);

}  // namespace argcsr_gpu
