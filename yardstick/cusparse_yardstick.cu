// BENCH-ONLY yardstick (not part of the product library): cusparseSpMV on a
// CSR matrix, called directly so the algorithm is stated (SURVEY.md §8(d):
// CUSPARSE_SPMV_CSR_ALG1, plus ALG2 for determinism).  32-bit row pointers and
// columns (cuSPARSE needs equal index widths; every single-GPU config has
// nnz < 2^31).  bench.py loads it with
// ctypes; nothing in paper_1203_5737_b200/ links it.
#include <cuda_runtime.h>
#include <cusparse.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

namespace {
int fail(char* err, int cap, const char* what, int code) {
    if (err && cap > 0) std::snprintf(err, size_t(cap), "%s (%d)", what, code);
    return code ? code : 1;
}
}  // namespace

extern "C" int ys_spmv_csr_median_ms(int64_t rows, int64_t cols, int64_t nnz, const void* row_pointers_i32,
                                     const void* columns_i32, const void* values, int fp64, const void* x, void* y,
                                     int alg, int warmup, int iters, void* stream, double* median_ms, char* err,
                                     int errcap) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cusparseHandle_t h = nullptr;
    cusparseSpMatDescr_t A = nullptr;
    cusparseDnVecDescr_t vx = nullptr, vy = nullptr;
    void* buf = nullptr;
    int rc = 0;
    const cudaDataType dt = fp64 ? CUDA_R_64F : CUDA_R_32F;
    const cusparseSpMVAlg_t a = alg == 2 ? CUSPARSE_SPMV_CSR_ALG2 : CUSPARSE_SPMV_CSR_ALG1;
    double one64 = 1.0, zero64 = 0.0;
    float one32 = 1.0f, zero32 = 0.0f;
    const void* alpha = fp64 ? static_cast<const void*>(&one64) : static_cast<const void*>(&one32);
    const void* beta = fp64 ? static_cast<const void*>(&zero64) : static_cast<const void*>(&zero32);
    size_t bytes = 0;
    std::vector<float> t;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
#define CS(call)                                                            \
    do {                                                                    \
        cusparseStatus_t st_ = (call);                                      \
        if (st_ != CUSPARSE_STATUS_SUCCESS) {                               \
            rc = fail(err, errcap, #call, int(st_));                        \
            goto done;                                                      \
        }                                                                   \
    } while (0)
#define CU(call)                                                            \
    do {                                                                    \
        cudaError_t e_ = (call);                                            \
        if (e_ != cudaSuccess) {                                            \
            rc = fail(err, errcap, cudaGetErrorString(e_), int(e_));        \
            goto done;                                                      \
        }                                                                   \
    } while (0)
    CS(cusparseCreate(&h));
    CS(cusparseSetStream(h, s));
    CS(cusparseCreateCsr(&A, rows, cols, nnz, const_cast<void*>(row_pointers_i32), const_cast<void*>(columns_i32),
                         const_cast<void*>(values), CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO,
                         dt));
    CS(cusparseCreateDnVec(&vx, cols, const_cast<void*>(x), dt));
    CS(cusparseCreateDnVec(&vy, rows, y, dt));
    CS(cusparseSpMV_bufferSize(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, vx, beta, vy, dt, a, &bytes));
    CU(cudaMalloc(&buf, std::max<size_t>(bytes, 16)));
    CS(cusparseSpMV_preprocess(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, vx, beta, vy, dt, a, buf));
    for (int i = 0; i < warmup; ++i)
        CS(cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, vx, beta, vy, dt, a, buf));
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    t.resize(size_t(std::max(iters, 1)));
    for (int i = 0; i < iters; ++i) {
        CU(cudaEventRecord(e0, s));
        CS(cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, vx, beta, vy, dt, a, buf));
        CU(cudaEventRecord(e1, s));
        CU(cudaEventSynchronize(e1));
        CU(cudaEventElapsedTime(&t[size_t(i)], e0, e1));
    }
    std::sort(t.begin(), t.begin() + iters);
    *median_ms = iters % 2 ? t[size_t(iters / 2)] : 0.5 * (t[size_t(iters / 2 - 1)] + t[size_t(iters / 2)]);
done:
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (buf) cudaFree(buf);
    if (vx) cusparseDestroyDnVec(vx);
    if (vy) cusparseDestroyDnVec(vy);
    if (A) cusparseDestroySpMat(A);
    if (h) cusparseDestroy(h);
    return rc;
#undef CS
#undef CU
}
