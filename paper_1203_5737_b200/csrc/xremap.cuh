// x remap (xremap.cu): device-internal column order that keeps x's working
// set L2-resident.
#pragma once

#include "common.cuh"

namespace argcsr_gpu {

// Decides and builds the remap for handle m from the column indices (device,
// n entries; with `sentinels`, -1 entries are padding and skipped).  Returns the device array inv (old column -> stored column,
// num_cols entries, cudaMallocAsync on s; the caller frees it) when the remap
// is on, else nullptr.
// rp / cols_abs (CSR input only, else nullptr): long rows are also checked
// for runs of consecutive stored columns (the heavy kernel's vector x loads).
int32_t* build_xremap(argcsr_dev* m, const int32_t* cols, uint64_t n, int mode, cudaStream_t s, bool sentinels,
                      const uint64_t* rp = nullptr, const int32_t* cols_abs = nullptr);

// x as the SpMV kernels read it: x itself, or x' = x[perm] gathered on s into
// the handle's buffer.
const void* xremap_apply(const argcsr_dev* m, const void* x, cudaStream_t s);

}  // namespace argcsr_gpu
