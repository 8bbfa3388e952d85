// PROBE (experiment): throughput of a column stream + x gathers, no matrix
// structure, to find the gather-rate ceiling of the power-law SpMV.
#include <cuda_runtime.h>
#include <cstdint>

namespace {
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void ld_cols4(const int32_t* p, int (&c)[4], uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]) : "l"(p), "l"(pol));
}
template <int MODE>
__device__ __forceinline__ double ldx(const double* p, uint64_t pol) {
    double v;
    if constexpr (MODE == 0) asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    else if constexpr (MODE == 1)
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    else if constexpr (MODE == 2) asm("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else asm("ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

// Each thread: NV vectors of 4 columns per iteration (grid-stride), gathers, sum.
template <int NV, int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) k_gather(const int32_t* cols, uint64_t n, const double* x, double* out) {
    const uint64_t pc = pol_normal(), px = pol_last();
    double acc = 0.0;
    const uint64_t stride = uint64_t(gridDim.x) * 256 * 4 * NV;
    for (uint64_t b = (uint64_t(blockIdx.x) * 256 * NV + threadIdx.x) * 4; b < n; b += stride) {
        int c[NV][4];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const uint64_t i = b + uint64_t(q) * 1024;
            if (i + 3 < n) ld_cols4(cols + i, c[q], pc);
            else
#pragma unroll
                for (int l = 0; l < 4; ++l) c[q][l] = 0;
        }
        double xv[NV][4];
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int l = 0; l < 4; ++l) xv[q][l] = ldx<MODE>(x + c[q][l], px);
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int l = 0; l < 4; ++l) acc += xv[q][l];
    }
    if (acc == 12345.678) out[0] = acc;
}
// Same with the values streamed too (v4.f64): the structure-free SpMV ceiling.
__device__ __forceinline__ void ld_vals4(const double* p, double (&v)[4], uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p), "l"(pol));
}
template <int NV, int MINB>
__global__ void __launch_bounds__(256, MINB) k_spmv_flat(const int32_t* cols, const double* vals, uint64_t n,
                                                         const double* x, double* out) {
    const uint64_t pc = pol_normal(), px = pol_last();
    double acc = 0.0;
    const uint64_t stride = uint64_t(gridDim.x) * 256 * 4 * NV;
    for (uint64_t b = (uint64_t(blockIdx.x) * 256 * NV + threadIdx.x) * 4; b < n; b += stride) {
        int c[NV][4];
        double v[NV][4];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const uint64_t i = b + uint64_t(q) * 1024;
            if (i + 3 < n) {
                ld_cols4(cols + i, c[q], pc);
                ld_vals4(vals + i, v[q], pc);
            } else {
#pragma unroll
                for (int l = 0; l < 4; ++l) c[q][l] = 0, v[q][l] = 0.0;
            }
        }
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int l = 0; l < 4; ++l) acc += v[q][l] * ldx<0>(x + c[q][l], px);
    }
    if (acc == 12345.678) out[0] = acc;
}
}  // namespace

extern "C" int probe_spmv_flat(int variant, const int32_t* cols, const double* vals, uint64_t n, const double* x,
                               double* out, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (variant == 0) k_spmv_flat<2, 4><<<sms * 4, 256, 0, s>>>(cols, vals, n, x, out);
    else if (variant == 1) k_spmv_flat<1, 8><<<sms * 8, 256, 0, s>>>(cols, vals, n, x, out);
    else k_spmv_flat<4, 2><<<sms * 2, 256, 0, s>>>(cols, vals, n, x, out);
    return int(cudaGetLastError());
}

template <typename K>
static void go(K k, int ctas_per_sm, const int32_t* cols, uint64_t n, const double* x, double* out, cudaStream_t s) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k<<<sms * ctas_per_sm, 256, 0, s>>>(cols, n, x, out);
}

extern "C" int probe_gather(int variant, const int32_t* cols, uint64_t n, const double* x, double* out,
                            void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (variant) {
        case 0: go(k_gather<2, 0, 4>, 4, cols, n, x, out, s); break;   // 8 gathers/thread, L1 allocate
        case 1: go(k_gather<4, 0, 2>, 4, cols, n, x, out, s); break;   // 16 gathers/thread
        case 2: go(k_gather<2, 1, 4>, 4, cols, n, x, out, s); break;   // L1 no_allocate
        case 3: go(k_gather<2, 2, 4>, 4, cols, n, x, out, s); break;   // ld.cg
        case 4: go(k_gather<2, 3, 4>, 4, cols, n, x, out, s); break;   // L1 evict_last
        case 5: go(k_gather<1, 0, 8>, 8, cols, n, x, out, s); break;   // 4 gathers/thread, 8 CTAs/SM
        case 6: go(k_gather<4, 0, 2>, 8, cols, n, x, out, s); break;
        default: go(k_gather<2, 0, 4>, 8, cols, n, x, out, s); break;
    }
    return int(cudaGetLastError());
}

// Unit-walk probe on a uniform j-major layout (C2-like: groups of W lanes x C
// steps, stored j-major): thread = unit of 4 lanes, walks its C steps with
// 4-wide vector loads, gathers, sums per lane (no row sums).  IL = 0: unit u'
// holds lanes 4u'..4u'+3 (the product layout); IL = 1: lanes u' + k*W/4
// (interleaved storage: the 4 lanes of a vector are W/4 apart, so a warp's
// gather instruction covers consecutive lanes).  The storage is the same
// array; only which column/value belongs to which lane changes, so the probe
// just reads cols/vals as laid out and the lane order is a property of the
// input arrays prepared by the driver.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_unit_walk(const int32_t* cols, const double* vals, uint64_t ngroups,
                                                         uint32_t W, uint32_t C, const double* x, double* out) {
    const uint64_t pc = pol_normal(), px = pol_last();
    const uint32_t upg = W / 4;
    const uint64_t nunits = ngroups * upg;
    double acc = 0.0;
    for (uint64_t u = uint64_t(blockIdx.x) * 256 + threadIdx.x; u < nunits; u += uint64_t(gridDim.x) * 256) {
        const uint64_t g = u / upg, up = u % upg;
        const uint64_t base = g * uint64_t(W) * C + up * 4;
        int c[4][4];
        double v[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (uint32_t(j) < C) {
                ld_cols4(cols + base + uint64_t(j) * W, c[j], pc);
                ld_vals4(vals + base + uint64_t(j) * W, v[j], pc);
            } else {
#pragma unroll
                for (int l = 0; l < 4; ++l) c[j][l] = -1, v[j][l] = 0.0;
            }
        }
        double s[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int l = 0; l < 4; ++l)
                if (c[j][l] >= 0) s[l] += v[j][l] * ldx<0>(x + c[j][l], px);
        acc += s[0] + s[1] + s[2] + s[3];
    }
    if (acc == 12345.678) out[0] = acc;
}

extern "C" int probe_unit_walk(int minb, const int32_t* cols, const double* vals, uint64_t ngroups, uint32_t W,
                               uint32_t C, const double* x, double* out, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (minb == 5) k_unit_walk<5><<<sms * 5, 256, 0, s>>>(cols, vals, ngroups, W, C, x, out);
    else k_unit_walk<4><<<sms * 4, 256, 0, s>>>(cols, vals, ngroups, W, C, x, out);
    return int(cudaGetLastError());
}
