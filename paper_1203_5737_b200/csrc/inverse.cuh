// Device-side accessors (inverse.cu).
#pragma once

#include "common.cuh"

namespace argcsr_gpu {

void export_arrays(const argcsr_dev* m, uint64_t* groups4, uint64_t* tm, void* values, int32_t* columns,
                   cudaStream_t s);
void to_csr(const argcsr_dev* m, uint64_t* row_pointers, int32_t* columns, void* values, cudaStream_t s);
uint64_t to_csr_nnz(const argcsr_dev* m, cudaStream_t s);
void padding_stats(const argcsr_dev* m, argcsr_format_stats* out, cudaStream_t s);
// balance_stats(const ArgCsrMatrix&) (analysis.cpp:198-208): explicit entries
// per group counted on the device, the ratios on the host in the reference's
// order (bit-identical).  per_group may be null.
void balance_stats(const argcsr_dev* m, uint64_t* per_group, double* max_over_mean, double* cv, cudaStream_t s);

}  // namespace argcsr_gpu
