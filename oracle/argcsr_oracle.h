/* TEST INFRASTRUCTURE ONLY — the CPU checker for the ARG-CSR hot path.
 *
 * A plain-C restatement of the reference algorithm (proj/src/argcsr.cpp,
 * proj/src/core.cpp, proj/src/bench.cpp of arxiv/paper_1203_5737).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it,
 * and only as the checker.  It is pinned against the compiled reference
 * (oracle/_ref) and the golden fixtures in tests/golden/.
 *
 * Arrays use the reference's widths: u64 row pointers / group fields /
 * threads_mapping, i32 columns, f64 values.  Return values are argcsr_status
 * codes (0 = OK, 1 = parameter, 2 = dimension, 3 = bounds, 4 = internal,
 * 7 = out of memory).
 */
#ifndef ARGCSR_ORACLE_H
#define ARGCSR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* argcsr.cpp:17-46 */
int orc_partition_groups(const uint64_t* counts, uint64_t n, uint64_t tpg, uint64_t dcs,
                         uint64_t* spans2, uint64_t* nspans);
/* argcsr.cpp:48-89 */
int orc_assign_threads(const uint64_t* counts, uint64_t n, uint64_t tpg, uint64_t* tpr,
                       uint64_t* chunk, uint64_t* assigned, uint64_t* free_threads);
/* argcsr.cpp:123-155: sizes first, then the arrays. */
int orc_argcsr_sizes(uint64_t nrows, const uint64_t* rp, uint64_t tpg, uint64_t dcs,
                     uint64_t* ngroups, uint64_t* nslots);
int orc_argcsr_from_csr(uint64_t nrows, const uint64_t* rp, const int32_t* cols,
                        const double* vals, uint64_t tpg, uint64_t dcs, uint64_t* groups4,
                        uint64_t* tm, double* out_vals, int32_t* out_cols);
/* argcsr.cpp:185-217 (no length check, like the reference) */
void orc_spmv_argcsr_groups(uint64_t tpg, const uint64_t* groups4, const uint64_t* tm,
                            const double* vals, const int32_t* cols, const double* x,
                            uint64_t gb, uint64_t ge, double* y);
/* argcsr.cpp:219-227 */
int orc_spmv_argcsr(uint64_t nrows, uint64_t ncols, uint64_t tpg, uint64_t ngroups,
                    const uint64_t* groups4, const uint64_t* tm, const double* vals,
                    const int32_t* cols, const double* x, uint64_t nx, double* y);
/* bench.cpp:48-71 + 109-116: contiguous group partition over `workers` pthreads. */
int orc_spmv_argcsr_parallel(uint64_t nrows, uint64_t ncols, uint64_t tpg, uint64_t ngroups,
                             const uint64_t* groups4, const uint64_t* tm, const double* vals,
                             const int32_t* cols, const double* x, uint64_t nx, double* y,
                             uint64_t workers);
/* argcsr.cpp:157-183: row_pointers first (nnz = rp[nrows]), then cols/vals. */
int orc_csr_from_argcsr_rp(uint64_t nrows, uint64_t tpg, uint64_t ngroups,
                           const uint64_t* groups4, const uint64_t* tm, const int32_t* cols,
                           uint64_t* rp);
int orc_csr_from_argcsr(uint64_t nrows, uint64_t tpg, uint64_t ngroups, const uint64_t* groups4,
                        const uint64_t* tm, const double* vals, const int32_t* cols,
                        const uint64_t* rp, int32_t* out_cols, double* out_vals);
/* core.cpp:61-81 */
int orc_spmv_csr(uint64_t nrows, uint64_t ncols, const uint64_t* rp, const int32_t* cols,
                 const double* vals, const double* x, uint64_t nx, double* y);
/* Tolerance helper (north_star): per-row sum |a_ij * x_j|. */
void orc_abs_row_sums(uint64_t nrows, const uint64_t* rp, const int32_t* cols,
                      const double* vals, const double* x, double* out);
/* analysis.cpp:167-184: padded = sum(assigned*chunk) - explicit, total = slots. */
void orc_padding_stats(uint64_t nrows, uint64_t tpg, uint64_t ngroups, const uint64_t* groups4,
                       const uint64_t* tm, uint64_t nslots, const int32_t* cols,
                       uint64_t* explicit_nnz, uint64_t* padded, uint64_t* total);

#ifdef __cplusplus
}
#endif
#endif
