/* TEST INFRASTRUCTURE ONLY — see argcsr_oracle.h.
 *
 * Plain-C restatement of the reference ARG-CSR path.  Every function cites the
 * reference file:line it follows (paths relative to /root/reference).  Built
 * with -ffp-contract=off so `sum += v * x` rounds twice, like the reference's
 * baseline-ISA x86-64 build (no FMA).
 */
#include "argcsr_oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* argcsr.cpp:9-15 */
static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
static uint64_t chunk_filling(uint64_t nnz, uint64_t threads) {
    return nnz == 0 ? 0 : ceil_div(nnz, threads);
}

/* argcsr.cpp:17-46.  `budget` is the reference's size_t product (wraps). */
int orc_partition_groups(const uint64_t* counts, uint64_t n, uint64_t tpg, uint64_t dcs,
                         uint64_t* spans2, uint64_t* nspans) {
    if (tpg == 0 || dcs == 0)
        return fail(1, "partition_groups: threads_per_group and desired_chunk_size must be at least 1");
    if (n == 0) return fail(1, "partition_groups: row_nnz must be nonempty");
    const uint64_t budget = dcs * tpg;
    uint64_t start = 0, count = 0, elements = 0, k = 0;
    for (uint64_t r = 0; r < n; ++r) {
        if (count > 0 && (count + 1 > tpg || elements + counts[r] > budget)) {
            spans2[2 * k] = start;
            spans2[2 * k + 1] = count;
            ++k;
            start = r;
            count = 0;
            elements = 0;
        }
        ++count;
        elements += counts[r];
    }
    spans2[2 * k] = start;
    spans2[2 * k + 1] = count;
    *nspans = k + 1;
    return 0;
}

/* argcsr.cpp:48-89: one thread at a time to the greatest-filling improvable
 * row, lowest index on ties (`filling <= best_filling` skip at :70, strict
 * improvement test at :71). */
int orc_assign_threads(const uint64_t* counts, uint64_t n, uint64_t tpg, uint64_t* tpr,
                       uint64_t* chunk, uint64_t* assigned, uint64_t* free_threads) {
    if (tpg == 0) return fail(1, "assign_threads: threads_per_group must be at least 1");
    if (n > tpg) return fail(1, "assign_threads: rows exceed threads");
    for (uint64_t r = 0; r < n; ++r) tpr[r] = 1;
    uint64_t spare = tpg - n;
    while (spare > 0) {
        uint64_t best = n, best_filling = 0;
        for (uint64_t r = 0; r < n; ++r) {
            const uint64_t filling = chunk_filling(counts[r], tpr[r]);
            if (filling <= best_filling) continue;
            if (chunk_filling(counts[r], tpr[r] + 1) < filling) {
                best = r;
                best_filling = filling;
            }
        }
        if (best == n) break;
        tpr[best] += 1;
        --spare;
    }
    uint64_t cs = 0;
    for (uint64_t r = 0; r < n; ++r) {
        const uint64_t f = chunk_filling(counts[r], tpr[r]);
        if (f > cs) cs = f;
    }
    *chunk = cs;
    *assigned = tpg - spare;
    *free_threads = spare;
    return 0;
}

/* row_nnz, core.cpp:83-89 */
static uint64_t* row_counts(uint64_t nrows, const uint64_t* rp) {
    uint64_t* c = (uint64_t*)malloc((nrows ? nrows : 1) * sizeof(uint64_t));
    if (!c) return NULL;
    for (uint64_t r = 0; r < nrows; ++r) c[r] = rp[r + 1] - rp[r];
    return c;
}

int orc_argcsr_sizes(uint64_t nrows, const uint64_t* rp, uint64_t tpg, uint64_t dcs,
                     uint64_t* ngroups, uint64_t* nslots) {
    if (tpg == 0 || dcs == 0)
        return fail(1, "partition_groups: threads_per_group and desired_chunk_size must be at least 1");
    if (nrows == 0) return fail(1, "partition_groups: row_nnz must be nonempty");
    uint64_t* counts = row_counts(nrows, rp);
    uint64_t* spans = (uint64_t*)malloc(2 * nrows * sizeof(uint64_t));
    uint64_t* tpr = (uint64_t*)malloc((tpg < nrows ? tpg : nrows) * sizeof(uint64_t));
    if (!counts || !spans || !tpr) {
        free(counts), free(spans), free(tpr);
        return fail(7, "out of host memory");
    }
    uint64_t ns = 0, slots = 0;
    int st = orc_partition_groups(counts, nrows, tpg, dcs, spans, &ns);
    for (uint64_t g = 0; st == 0 && g < ns; ++g) {
        uint64_t cs, as, fr;
        st = orc_assign_threads(counts + spans[2 * g], spans[2 * g + 1], tpg, tpr, &cs, &as, &fr);
        slots += cs * tpg;
    }
    free(counts), free(spans), free(tpr);
    if (st) return st;
    *ngroups = ns;
    *nslots = slots;
    return 0;
}

/* argcsr.cpp:123-155 with layout_group (argcsr.cpp:91-121) inlined: each
 * group's block is filled with (+0.0, -1) and then row r's t chunks get
 * ceil(n/t) then floor(n/t) elements, element j of chunk c at j*tpg + c. */
int orc_argcsr_from_csr(uint64_t nrows, const uint64_t* rp, const int32_t* cols,
                        const double* vals, uint64_t tpg, uint64_t dcs, uint64_t* groups4,
                        uint64_t* tm, double* out_vals, int32_t* out_cols) {
    if (tpg == 0 || dcs == 0)
        return fail(1, "partition_groups: threads_per_group and desired_chunk_size must be at least 1");
    if (nrows == 0) return fail(1, "partition_groups: row_nnz must be nonempty");
    uint64_t* counts = row_counts(nrows, rp);
    uint64_t* spans = (uint64_t*)malloc(2 * nrows * sizeof(uint64_t));
    uint64_t* tpr = (uint64_t*)malloc((tpg < nrows ? tpg : nrows) * sizeof(uint64_t));
    if (!counts || !spans || !tpr) {
        free(counts), free(spans), free(tpr);
        return fail(7, "out of host memory");
    }
    uint64_t ns = 0, offset = 0;
    int st = orc_partition_groups(counts, nrows, tpg, dcs, spans, &ns);
    for (uint64_t g = 0; st == 0 && g < ns; ++g) {
        const uint64_t first = spans[2 * g], size = spans[2 * g + 1];
        uint64_t cs, as, fr;
        st = orc_assign_threads(counts + first, size, tpg, tpr, &cs, &as, &fr);
        if (st) break;
        uint64_t scan = 0;
        for (uint64_t r = 0; r < size; ++r) {
            scan += tpr[r];
            tm[first + r] = scan; /* inclusive, argcsr.cpp:141-145 */
        }
        const uint64_t nslot = cs * tpg;
        for (uint64_t s = 0; s < nslot; ++s) {
            out_vals[offset + s] = 0.0;
            out_cols[offset + s] = -1;
        }
        uint64_t chunk = 0;
        for (uint64_t local = 0; local < size; ++local) {
            const uint64_t row = first + local;
            const uint64_t n = rp[row + 1] - rp[row];
            const uint64_t t = tpr[local];
            const uint64_t base = n / t, extra = n % t;
            uint64_t k = rp[row];
            for (uint64_t c = 0; c < t; ++c, ++chunk) {
                const uint64_t take = base + (c < extra ? 1 : 0);
                if (take > cs) {
                    st = 4;
                    fail(4, "layout_group: chunk overflow");
                    break;
                }
                for (uint64_t j = 0; j < take; ++j, ++k) {
                    out_vals[offset + j * tpg + chunk] = vals[k];
                    out_cols[offset + j * tpg + chunk] = cols[k];
                }
            }
            if (st) break;
        }
        groups4[4 * g + 0] = first;
        groups4[4 * g + 1] = size;
        groups4[4 * g + 2] = offset;
        groups4[4 * g + 3] = cs;
        offset += nslot;
    }
    free(counts), free(spans), free(tpr);
    return st;
}

/* argcsr.cpp:185-217: phase 1 per chunk until the first sentinel, phase 2 per
 * row ascending over its chunk range, both from +0.0. */
void orc_spmv_argcsr_groups(uint64_t tpg, const uint64_t* groups4, const uint64_t* tm,
                            const double* vals, const int32_t* cols, const double* x,
                            uint64_t gb, uint64_t ge, double* y) {
    double* partials = (double*)malloc(tpg * sizeof(double));
    for (uint64_t gi = gb; gi < ge; ++gi) {
        const uint64_t first = groups4[4 * gi], size = groups4[4 * gi + 1];
        const uint64_t off = groups4[4 * gi + 2], cs = groups4[4 * gi + 3];
        for (uint64_t t = 0; t < tpg; ++t) {
            double sum = 0.0;
            uint64_t slot = off + t;
            for (uint64_t j = 0; j < cs; ++j) {
                const int32_t c = cols[slot];
                if (c == -1) break;
                sum += vals[slot] * x[(uint64_t)c];
                slot += tpg;
            }
            partials[t] = sum;
        }
        for (uint64_t local = 0; local < size; ++local) {
            const uint64_t row = first + local;
            const uint64_t b = local == 0 ? 0 : tm[row - 1];
            const uint64_t e = tm[row];
            double sum = 0.0;
            for (uint64_t t = b; t < e; ++t) sum += partials[t];
            y[row] = sum;
        }
    }
    free(partials);
}

int orc_spmv_argcsr(uint64_t nrows, uint64_t ncols, uint64_t tpg, uint64_t ngroups,
                    const uint64_t* groups4, const uint64_t* tm, const double* vals,
                    const int32_t* cols, const double* x, uint64_t nx, double* y) {
    if (nx != ncols) return fail(2, "spmv_argcsr: vector length does not match columns");
    for (uint64_t r = 0; r < nrows; ++r) y[r] = 0.0;
    orc_spmv_argcsr_groups(tpg, groups4, tm, vals, cols, x, 0, ngroups, y);
    return 0;
}

struct par_job {
    uint64_t tpg, gb, ge;
    const uint64_t *groups4, *tm;
    const double *vals, *x;
    const int32_t* cols;
    double* y;
};

static void* par_body(void* p) {
    const struct par_job* j = (const struct par_job*)p;
    orc_spmv_argcsr_groups(j->tpg, j->groups4, j->tm, j->vals, j->cols, j->x, j->gb, j->ge, j->y);
    return NULL;
}

/* bench.cpp:48-71 (parallel_over) + 109-116 (spmv_argcsr_parallel). */
int orc_spmv_argcsr_parallel(uint64_t nrows, uint64_t ncols, uint64_t tpg, uint64_t ngroups,
                             const uint64_t* groups4, const uint64_t* tm, const double* vals,
                             const int32_t* cols, const double* x, uint64_t nx, double* y,
                             uint64_t workers) {
    (void)nrows;
    if (nx != ncols) return fail(2, "parallel spmv: vector length does not match columns");
    if (ngroups == 0) return 0;
    if (workers < 1) workers = 1;
    if (workers > ngroups) workers = ngroups;
    struct par_job* jobs = (struct par_job*)calloc(workers, sizeof *jobs);
    pthread_t* th = (pthread_t*)calloc(workers, sizeof *th);
    const uint64_t base = ngroups / workers, extra = ngroups % workers;
    uint64_t b = 0;
    for (uint64_t w = 0; w < workers; ++w) {
        const uint64_t e = b + base + (w < extra ? 1 : 0);
        jobs[w] = (struct par_job){tpg, b, e, groups4, tm, vals, x, cols, y};
        if (w + 1 < workers) pthread_create(&th[w], NULL, par_body, &jobs[w]);
        b = e;
    }
    par_body(&jobs[workers - 1]);
    for (uint64_t w = 0; w + 1 < workers; ++w) pthread_join(th[w], NULL);
    free(jobs), free(th);
    return 0;
}

/* argcsr.cpp:157-183 (counting pass). */
int orc_csr_from_argcsr_rp(uint64_t nrows, uint64_t tpg, uint64_t ngroups,
                           const uint64_t* groups4, const uint64_t* tm, const int32_t* cols,
                           uint64_t* rp) {
    for (uint64_t r = 0; r <= nrows; ++r) rp[r] = 0;
    for (uint64_t g = 0; g < ngroups; ++g) {
        const uint64_t first = groups4[4 * g], size = groups4[4 * g + 1];
        const uint64_t off = groups4[4 * g + 2], cs = groups4[4 * g + 3];
        for (uint64_t local = 0; local < size; ++local) {
            const uint64_t row = first + local;
            const uint64_t b = local == 0 ? 0 : tm[row - 1], e = tm[row];
            for (uint64_t c = b; c < e; ++c)
                for (uint64_t j = 0; j < cs; ++j) {
                    if (cols[off + j * tpg + c] == -1) break;
                    rp[row + 1] += 1;
                }
        }
    }
    for (uint64_t r = 0; r < nrows; ++r) rp[r + 1] += rp[r];
    return 0;
}

int orc_csr_from_argcsr(uint64_t nrows, uint64_t tpg, uint64_t ngroups, const uint64_t* groups4,
                        const uint64_t* tm, const double* vals, const int32_t* cols,
                        const uint64_t* rp, int32_t* out_cols, double* out_vals) {
    (void)nrows;
    for (uint64_t g = 0; g < ngroups; ++g) {
        const uint64_t first = groups4[4 * g], size = groups4[4 * g + 1];
        const uint64_t off = groups4[4 * g + 2], cs = groups4[4 * g + 3];
        for (uint64_t local = 0; local < size; ++local) {
            const uint64_t row = first + local;
            const uint64_t b = local == 0 ? 0 : tm[row - 1], e = tm[row];
            uint64_t k = rp[row];
            for (uint64_t c = b; c < e; ++c)
                for (uint64_t j = 0; j < cs; ++j) {
                    const uint64_t slot = off + j * tpg + c;
                    if (cols[slot] == -1) break;
                    out_cols[k] = cols[slot];
                    out_vals[k] = vals[slot];
                    ++k;
                }
        }
    }
    return 0;
}

/* core.cpp:61-81 */
int orc_spmv_csr(uint64_t nrows, uint64_t ncols, const uint64_t* rp, const int32_t* cols,
                 const double* vals, const double* x, uint64_t nx, double* y) {
    if (nx != ncols) return fail(2, "spmv_csr: vector length does not match columns");
    for (uint64_t r = 0; r < nrows; ++r) {
        double sum = 0.0;
        for (uint64_t k = rp[r]; k < rp[r + 1]; ++k) sum += vals[k] * x[(uint64_t)cols[k]];
        y[r] = sum;
    }
    return 0;
}

void orc_abs_row_sums(uint64_t nrows, const uint64_t* rp, const int32_t* cols,
                      const double* vals, const double* x, double* out) {
    for (uint64_t r = 0; r < nrows; ++r) {
        double s = 0.0;
        for (uint64_t k = rp[r]; k < rp[r + 1]; ++k) {
            double p = vals[k] * x[(uint64_t)cols[k]];
            s += p < 0 ? -p : p;
        }
        out[r] = s;
    }
}

/* analysis.cpp:167-184 */
void orc_padding_stats(uint64_t nrows, uint64_t tpg, uint64_t ngroups, const uint64_t* groups4,
                       const uint64_t* tm, uint64_t nslots, const int32_t* cols,
                       uint64_t* explicit_nnz, uint64_t* padded, uint64_t* total) {
    (void)nrows, (void)tpg;
    uint64_t ex = 0, assigned_slots = 0;
    for (uint64_t s = 0; s < nslots; ++s) ex += cols[s] != -1;
    for (uint64_t g = 0; g < ngroups; ++g) {
        const uint64_t last = groups4[4 * g] + groups4[4 * g + 1] - 1;
        assigned_slots += tm[last] * groups4[4 * g + 3];
    }
    *explicit_nnz = ex;
    *padded = assigned_slots - ex;
    *total = nslots;
}
