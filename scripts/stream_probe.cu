// HBM read-pattern probe: the bandwidth ceilings an ARG-CSR light kernel can
// reach on this B200, per access pattern (useful bytes / time).
//   contiguous   : every byte of a 1.5 GB buffer, 32 B per thread per load
//   segments S/P : a warp-contiguous segment of S bytes every P bytes (the
//                  assigned-lane j-rows of a group: 224 B of values per 1024 B
//                  at (128,1) on the 27-pt stencil, 112 B of columns per 512 B)
//   bulk         : cp.async.bulk (TMA) of 16 KB chunks into shared memory,
//                  4-stage mbarrier ring, one elected thread per CTA
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ double g_sink;

__global__ void read_contig(const double4* __restrict__ p, size_t n4) {
    double acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) {
        double4 v;
        asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p + i));
        acc += v.x + v.w;
    }
    if (acc == 1.2345) g_sink = acc;
}

// Each warp reads segment k: bytes [k*P, k*P+S) with 32 B per lane (S <= 1024).
__global__ void read_segments(const unsigned char* __restrict__ base, size_t nseg, int S, int P) {
    double acc = 0;
    const int lane = threadIdx.x & 31;
    const size_t warp = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5;
    const size_t nwarps = (size_t(gridDim.x) * blockDim.x) >> 5;
    for (size_t k = warp; k < nseg; k += nwarps) {
        if (lane * 32 < S) {
            const double4* q = reinterpret_cast<const double4*>(base + k * P + lane * 32);
            double4 v;
            asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(q));
            acc += v.x + v.w;
        }
    }
    if (acc == 1.2345) g_sink = acc;
}

// Unrolled variant: each warp keeps 4 segments in flight.
__global__ void read_segments4(const unsigned char* __restrict__ base, size_t nseg, int S, int P) {
    double acc = 0;
    const int lane = threadIdx.x & 31;
    const size_t warp = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5;
    const size_t nwarps = (size_t(gridDim.x) * blockDim.x) >> 5;
    for (size_t k = warp; k < nseg; k += 4 * nwarps) {
        double4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const size_t kk = k + u * nwarps;
            if (lane * 32 < S && kk < nseg) {
                const double4* q = reinterpret_cast<const double4*>(base + kk * P + lane * 32);
                asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[u].x), "=d"(v[u].y), "=d"(v[u].z), "=d"(v[u].w) : "l"(q));
            } else v[u] = make_double4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].w;
    }
    if (acc == 1.2345) g_sink = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int STAGES, int CHUNK>
__global__ void read_bulk(const unsigned char* __restrict__ p, size_t nchunks) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[STAGES];
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    double acc = 0;
    // chunks of this CTA: blockIdx.x + i*gridDim.x
    size_t mine = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto issue = [&](size_t i) {
        const int s = i % STAGES;
        const size_t c = blockIdx.x + i * gridDim.x;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sm + s * CHUNK)), "l"(p + c * CHUNK), "r"(CHUNK), "r"(su32(&bar[s])) : "memory");
    };
    if (threadIdx.x == 0)
        for (size_t i = 0; i < STAGES && i < mine; ++i) issue(i);
    for (size_t i = 0; i < mine; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" ::"r"(su32(&bar[s])), "r"(ph));
        const double* d = reinterpret_cast<const double*>(sm + s * CHUNK);
        for (int k = threadIdx.x; k < CHUNK / 8; k += blockDim.x) acc += d[k];
        __syncthreads();
        if (threadIdx.x == 0 && i + STAGES < mine) issue(i + STAGES);
    }
    if (acc == 1.2345) g_sink = acc;
}

template <typename K, typename... A>
float timeit(K k, int grid, int block, size_t smem, A... a) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) k<<<grid, block, smem>>>(a...);
    cudaEventRecord(e0);
    const int R = 10;
    for (int r = 0; r < R; ++r) k<<<grid, block, smem>>>(a...);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / R;
}

int main() {
    const size_t bytes = size_t(3) << 30;  // 3 GiB >> L2
    unsigned char* buf;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 0, bytes));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int per : {4, 8, 16}) {
        float ms = timeit(read_contig, sms * per, 256, 0, (const double4*)buf, bytes / 32);
        printf("contig  grid=%d*%d  %.1f GB/s\n", sms, per, bytes / ms / 1e6);
    }
    struct P { int S, Pp; } pats[] = {{224, 1024}, {112, 512}, {1024, 1024}, {512, 1024}, {96, 1024}};
    for (auto q : pats) {
        size_t nseg = bytes / q.Pp;
        float ms = timeit(read_segments, sms * 8, 256, 0, (const unsigned char*)buf, nseg, q.S, q.Pp);
        float ms4 = timeit(read_segments4, sms * 8, 256, 0, (const unsigned char*)buf, nseg, q.S, q.Pp);
        printf("segments S=%d P=%d  useful %.1f GB/s (x1)  %.1f GB/s (x4)\n", q.S, q.Pp, nseg * q.S / ms / 1e6,
               nseg * q.S / ms4 / 1e6);
    }
    {
        constexpr int CH = 16384, ST = 4;
        auto k = read_bulk<ST, CH>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
        for (int per : {1, 2, 3}) {
            float ms = timeit(k, sms * per, 256, ST * CH, (const unsigned char*)buf, bytes / CH);
            printf("bulk 4x16KB grid=%d*%d  %.1f GB/s\n", sms, per, bytes / ms / 1e6);
        }
    }
    CK(cudaGetLastError());
    return 0;
}
