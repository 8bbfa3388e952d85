// SpMV launch (spmv.cu).
#pragma once

#include "common.cuh"

namespace argcsr_gpu {

// y = A x for the rows of groups [group_begin, group_end); device pointers,
// stream-ordered, no synchronisation.
void spmv_launch(const argcsr_dev* m, const void* x, void* y, uint64_t group_begin, uint64_t group_end,
                 cudaStream_t s);

}  // namespace argcsr_gpu
