// PROTOTYPE (experiment, not product code): row-stream SpMV for ARG-CSR.
// The light part is stored in CSR order (no padding); products of a tile's
// element range go to shared memory, then each row sums its lanes (ceil/floor
// split of argcsr.cpp:86-99) in the reference order.  Long rows: one CTA per
// row, lane-major j-blocks through shared memory.
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
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void ld_cols4(const int32_t* p, int (&c)[4], uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_vals4(const double* p, double (&v)[4], uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ double ld_x(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_col1(const int32_t* p, uint64_t pol) {
    int c;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(c) : "l"(p), "l"(pol));
    return c;
}
__device__ __forceinline__ double ld_val1(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

struct TileArgs {
    const double* vals;
    const int32_t* cols;
    const uint32_t* srp;   // [N+1] short-stream row pointers
    const uint16_t* tt;    // [N] lanes per row; bit 15: long row (written by k_long)
    const uint32_t* tile_row;  // [ntiles+1]
    const double* x;
    double* y;
    uint32_t cap, rcap;
};

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_w, uint32_t& total) {
    // 256 threads
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= uint32_t(o)) inc += u;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t x = s_w[i];
        if (uint32_t(i) < w) off += x;
        tot += x;
    }
    total = tot;
    return off + inc - v;
}

// PH2: 0 = thread per row (lanes walked in order); 1 = no row sums (streaming
// ceiling, wrong results); 2 = lane-parallel lane sums in place, then rows.
template <int NV, int MINB, int PH2, int RPT>
__global__ void __launch_bounds__(256, MINB) k_tile(TileArgs a) {
    extern __shared__ double s_p[];
    const uint32_t k = blockIdx.x;
    const uint32_t r0 = a.tile_row[k], r1 = a.tile_row[k + 1];
    const uint32_t e0 = a.srp[r0], e1 = a.srp[r1];
    const uint64_t ps = pol_normal(), px = pol_last();
    const uint32_t rA = r0 + threadIdx.x;
    uint32_t mA0 = 0, mA1 = 0, tA = 0;
    if (PH2 != 2 && rA < r1) {
        mA0 = a.srp[rA];
        mA1 = a.srp[rA + 1];
        tA = a.tt[rA];
    }
    // PH2 == 2: rows [r0 + RPT*tid, +RPT) of this thread (contiguous), lane offsets by block scan
    uint32_t rs[RPT + 1], rt[RPT];
    uint32_t* s_w = nullptr;
    uint16_t* s_lrow = nullptr;
    uint32_t* s_rs = nullptr;   // [R+1] row start rel. e0
    uint32_t* s_rl = nullptr;   // [R+1] lane offset
    const uint32_t R = r1 - r0;
    if constexpr (PH2 == 2) {
        s_rs = reinterpret_cast<uint32_t*>(s_p + a.cap);
        s_rl = s_rs + a.rcap + 1;
        s_w = s_rl + a.rcap + 1;
        s_lrow = reinterpret_cast<uint16_t*>(s_w + 8);
        const uint32_t rb = r0 + RPT * threadIdx.x;
#pragma unroll
        for (int q = 0; q <= RPT; ++q) rs[q] = rb + q <= r1 ? a.srp[rb + q] : e1;
#pragma unroll
        for (int q = 0; q < RPT; ++q) rt[q] = rb + q < r1 ? a.tt[rb + q] : 0x8000u;
    }
    const uint32_t ea = e0 & ~3u;
    bool first = true;
    for (uint32_t vb = ea + 4 * threadIdx.x; vb < e1 || (PH2 == 2 && first); vb += 4 * 256 * NV) {
        int c[NV][4];
        double v[NV][4];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const uint32_t i = vb + q * 1024;
            if (i < e1) {
                ld_cols4(a.cols + i, c[q], ps);
                ld_vals4(a.vals + i, v[q], ps);
            } else {
#pragma unroll
                for (int l = 0; l < 4; ++l) c[q][l] = 0, v[q][l] = 0.0;
            }
        }
        if constexpr (PH2 == 2) {
            if (first) {  // lane offsets + lane -> row map while the loads fly
                first = false;
                uint32_t nl = 0;
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const uint32_t t = (rt[q] & 0x8000u) || rs[q + 1] == rs[q] ? 0u : rt[q];
                    nl += t;
                }
                uint32_t tot;
                uint32_t l0 = block_excl_scan(nl, s_w, tot);
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const uint32_t i = RPT * threadIdx.x + q;
                    if (i < R) {
                        const uint32_t t = (rt[q] & 0x8000u) || rs[q + 1] == rs[q] ? 0u : rt[q];
                        s_rs[i] = rs[q] - e0;
                        s_rl[i] = l0;
                        for (uint32_t c2 = 0; c2 < t; ++c2) s_lrow[l0 + c2] = uint16_t(i);
                        l0 += t;
                    }
                }
                if (threadIdx.x == 255) {
                    s_rs[R] = e1 - e0;
                    s_rl[R] = tot;
                }
            }
        }
        double xv[NV][4];
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const uint32_t i = vb + q * 1024 + l;
                xv[q][l] = (i >= e0 && i < e1) ? ld_x(a.x + c[q][l], px) : 0.0;
            }
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const uint32_t i = vb + q * 1024 + l;
                if (i >= e0 && i < e1) s_p[i - e0] = __dmul_rn(v[q][l], xv[q][l]);
            }
    }
    __syncthreads();
    if constexpr (PH2 == 1) {
        for (uint32_t r = rA; r < r1; r += 256) {
            uint32_t s0 = mA0, s1 = mA1;
            if (r != rA) s0 = a.srp[r], s1 = a.srp[r + 1];
            a.y[r] = s1 > s0 ? s_p[s0 - e0] : 0.0;
        }
        return;
    }
    if constexpr (PH2 == 2) {
        const uint32_t NL = s_rl[R];
        for (uint32_t l = threadIdx.x; l < NL; l += 256) {
            const uint32_t i = s_lrow[l];
            const uint32_t c2 = l - s_rl[i];
            const uint32_t s0 = s_rs[i], n = s_rs[i + 1] - s0, t = s_rl[i + 1] - s_rl[i];
            const uint32_t base = n / t, extra = n - base * t;
            const uint32_t st = s0 + c2 * base + min(c2, extra), len = base + (c2 < extra ? 1u : 0u);
            double ls = 0.0;
            for (uint32_t j = 0; j < len; ++j) ls = __dadd_rn(ls, s_p[st + j]);
            s_p[st] = ls;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const uint32_t i = RPT * threadIdx.x + q;
            if (i >= R || (rt[q] & 0x8000u)) continue;
            const uint32_t s0 = s_rs[i], n = s_rs[i + 1] - s0, t = rt[q];
            double y = 0.0;
            if (n) {
                const uint32_t base = n / t, extra = n - base * t;
                uint32_t st = s0;
                for (uint32_t c2 = 0; c2 < t; ++c2) {
                    y = __dadd_rn(y, s_p[st]);
                    st += base + (c2 < extra ? 1u : 0u);
                }
            }
            a.y[r0 + i] = y;
        }
        return;
    }
    for (uint32_t r = rA; r < r1; r += 256) {
        uint32_t s0 = mA0, s1 = mA1, t = tA;
        if (r != rA) {
            s0 = a.srp[r];
            s1 = a.srp[r + 1];
            t = a.tt[r];
        }
        if (t & 0x8000u) continue;
        const uint32_t n = s1 - s0;
        const uint32_t base = n / t, extra = n - base * t;
        double y = 0.0;
        uint32_t p = s0 - e0;
        for (uint32_t c = 0; c < t; ++c) {
            const uint32_t len = base + (c < extra ? 1u : 0u);
            double ls = 0.0;
            for (uint32_t j = 0; j < len; ++j) ls = __dadd_rn(ls, s_p[p + j]);
            p += len;
            y = __dadd_rn(y, ls);
        }
        a.y[r] = y;
    }
}

struct LongArgs {
    const double* vals;
    const int32_t* cols;
    const uint64_t* lrp;   // [L+1] long-region row pointers
    const uint16_t* lt;    // [L] lanes
    const uint32_t* lrow;  // [L] row index
    const uint32_t* order; // [L] CTA -> long row (LPT)
    const double* x;
    double* y;
};

// One CTA per long row; J element steps of every lane per block.
template <int J, int MINB>
__global__ void __launch_bounds__(256, MINB) k_long(LongArgs a) {
    extern __shared__ double s_p[];  // [t * J]
    __shared__ double s_ls[256];
    const uint32_t i = a.order[blockIdx.x];
    const uint32_t row = a.lrow[i];
    const uint64_t st = a.lrp[i];
    const uint32_t n = uint32_t(a.lrp[i + 1] - st);
    const uint32_t t = a.lt[i];
    const uint32_t base = n / t, extra = n - base * t;
    const uint32_t maxlen = base + (extra ? 1u : 0u);
    const uint64_t ps = pol_normal(), px = pol_last();
    const uint32_t tid = threadIdx.x;
    const uint32_t mylen = tid < t ? base + (tid < extra ? 1u : 0u) : 0u;
    double acc = 0.0;
    const uint32_t total = t * J;
    for (uint32_t j0 = 0; j0 < maxlen; j0 += J) {
        for (uint32_t f0 = 0; f0 < total; f0 += 256 * 8) {
            int c[8];
            double v[8];
            bool ok[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t f = f0 + tid + 256 * q;
                const uint32_t ln = f / J, j = f % J;
                const uint32_t len = base + (ln < extra ? 1u : 0u);
                ok[q] = f < total && j0 + j < len;
                if (ok[q]) {
                    const uint64_t pos = st + uint64_t(ln) * base + min(ln, extra) + j0 + j;
                    c[q] = ld_col1(a.cols + pos, ps);
                    v[q] = ld_val1(a.vals + pos, ps);
                } else {
                    c[q] = 0, v[q] = 0.0;
                }
            }
            double xv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) xv[q] = ok[q] ? ld_x(a.x + c[q], px) : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (ok[q]) s_p[f0 + tid + 256 * q] = __dmul_rn(v[q], xv[q]);
        }
        __syncthreads();
        if (tid < t) {
            const uint32_t m = mylen > j0 ? min(uint32_t(J), mylen - j0) : 0u;
            for (uint32_t j = 0; j < m; ++j) acc = __dadd_rn(acc, s_p[tid * J + j]);
        }
        __syncthreads();
    }
    if (tid < t) s_ls[tid] = acc;
    __syncthreads();
    if (tid == 0) {
        double y = 0.0;
        for (uint32_t c = 0; c < t; ++c) y = __dadd_rn(y, s_ls[c]);
        a.y[row] = y;
    }
}
}  // namespace

template <typename K>
static void go(K k, uint32_t grid, size_t smem, cudaStream_t s, const TileArgs& a) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, 256, smem, s>>>(a);
}

extern "C" int proto_tile(int variant, const double* vals, const int32_t* cols, const uint32_t* srp,
                          const uint16_t* tt, const uint32_t* tile_row, uint32_t ntiles, uint32_t cap, uint32_t rcap,
                          const double* x, double* y, void* stream) {
    TileArgs a{vals, cols, srp, tt, tile_row, x, y, cap, rcap};
    const size_t smem0 = size_t(cap) * sizeof(double);
    const size_t smem2 = smem0 + size_t(rcap + 1) * 8 + 32 + size_t(cap) * 2 + 16;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (variant) {
        case 0: go(k_tile<2, 4, 0, 1>, ntiles, smem0, s, a); break;
        case 1: go(k_tile<1, 5, 0, 1>, ntiles, smem0, s, a); break;
        case 4: go(k_tile<2, 4, 1, 1>, ntiles, smem0, s, a); break;
        case 5: go(k_tile<1, 5, 1, 1>, ntiles, smem0, s, a); break;
        case 6: go(k_tile<2, 4, 2, 1>, ntiles, smem2, s, a); break;
        case 7: go(k_tile<1, 5, 2, 1>, ntiles, smem2, s, a); break;
        case 8: go(k_tile<2, 4, 2, 2>, ntiles, smem2, s, a); break;
        case 9: go(k_tile<1, 4, 2, 2>, ntiles, smem2, s, a); break;
        default: go(k_tile<2, 3, 0, 1>, ntiles, smem0, s, a); break;
    }
    return int(cudaGetLastError());
}

extern "C" int proto_long(int variant, const double* vals, const int32_t* cols, const uint64_t* lrp,
                          const uint16_t* lt, const uint32_t* lrow, const uint32_t* order, uint32_t L, uint32_t maxt,
                          const double* x, double* y, void* stream) {
    LongArgs a{vals, cols, lrp, lt, lrow, order, x, y};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (L == 0) return 0;
    if (variant == 0) {
        const size_t smem = size_t(maxt) * 32 * sizeof(double);
        cudaFuncSetAttribute(k_long<32, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_long<32, 4><<<L, 256, smem, s>>>(a);
    } else {
        const size_t smem = size_t(maxt) * 16 * sizeof(double);
        cudaFuncSetAttribute(k_long<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_long<16, 4><<<L, 256, smem, s>>>(a);
    }
    return int(cudaGetLastError());
}
