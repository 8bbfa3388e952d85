// EXPERIMENT RECORD (not compiled, not product code): the warp-specialised
// light-tile kernel tried in round 2 (TMA warp + gather warps + consumer warps
// around an mbarrier ring).  Three versions were bit-exact on the full GPU
// parity suite but slower than the register-staged light kernel on C2
// (27-pt 160^3, (128,1)): v1 register gathers 0.54 ms, v2 + two tiles in
// flight per gather thread 0.61 ms (spills), v3 cp.async gathers into shared
// memory 0.86 ms, against 0.298 ms.  ncu (profiles/r02/ncu_ws_C2.txt): the
// gather warps stall on the x gathers with only 4K in flight per SM, and the
// per-tile TMA -> gather -> consumer hand-offs serialise what the 5 resident
// CTAs of the register kernel overlap.  Kept here for the record; see
// DESIGN.md section 4.
// ------------------------------------------------ warp-specialised light tiles
// The register-staged light kernel runs every tile as one dependent chain
// (metadata -> stored slots -> x gathers -> barrier -> lane and row sums ->
// exit), so an SM has gathers in flight only part of the time.  This kernel
// gives each stage its own warps, connected by a ring of kWsRing tile buffers
// in shared memory and mbarriers:
//   * a TMA warp (one elected thread) copies a tile's stored columns and
//     values -- one contiguous range of the lane-compact arrays -- and its
//     metadata (group descriptors, unit bases, threads_mapping slices) into a
//     free ring buffer with cp.async.bulk (completion: `loaded`, expect_tx);
//   * gather warps (kWsGatherWarps) read the columns from shared memory, gather
//     x (8 slots per thread in flight) and write the exact products fl(v * x)
//     -- a signalling-NaN marker for padding slots -- over the values
//     (`full`);
//   * consumer warps (kWsConsWarps) add each lane's products in j order
//     (argcsr.cpp:193-203: from +0.0, ascending, stop at the first padding
//     slot) and each row's lane sums in ascending order (:206-215), store y and
//     release the buffer (`empty`).
// One persistent CTA per SM walks tiles blockIdx.x, + gridDim.x, ...  The
// operations and their order are the reference's: bit-identical results.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!done);
}
// global -> shared bulk copy (16-B aligned, size % 16 == 0), completes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void cons_sync() {  // consumer warps only (named barrier 1)
    asm volatile("bar.sync 1, %0;" ::"r"(kWsConsWarps * 32) : "memory");
}

// Per ring buffer: values, columns, the gathered x entries, and the metadata slices.
template <typename T>
struct WsLayout {
    static constexpr uint32_t kVals = kWsSlots * sizeof(T);
    static constexpr uint32_t kCols = kWsSlots * 4;
    static constexpr uint32_t kX = kWsSlots * 8;  // gathered x (fp32: every other float), then lane sums
    static constexpr uint32_t kGd = (kWsMaxGroups + 2) * 16;
    static constexpr uint32_t kUb = (kWsMaxGroups + 4) * 8;
    static constexpr uint32_t kTm = (kWsMaxRows + 16) * 2;
    static constexpr uint32_t kBuf = kVals + kCols + kX + kGd + kUb + kTm;
    static constexpr int kRing = kWsRing;
};
struct WsTile {  // written by the TMA thread, read after `loaded` / `full`
    uint32_t gs, ge, row0, nrows, nslots;
    uint32_t ub_skew, tm_skew;  // elements before gs / row0 in the aligned metadata copies
    uint64_t S0;
};

// x[col] -> shared memory, 8 (4) bytes, no register destination: the gather
// warps only issue; completion is tracked per thread by the `full` mbarrier.
__device__ __forceinline__ void cp_async_x(void* dst, const double* src, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_x(void* dst, const float* src, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T>
__global__ void __launch_bounds__((1 + kWsGatherWarps + kWsConsWarps) * 32, 1) spmv_ws_kernel(const SpmvArgs<T> a) {
    using L = WsLayout<T>;
    constexpr int R = L::kRing;
    extern __shared__ __align__(128) unsigned char smem[];
    uint16_t* s_rgrp = reinterpret_cast<uint16_t*>(smem + size_t(R) * L::kBuf);  // [kWsMaxRows]
    uint16_t* s_ugrp = s_rgrp + kWsMaxRows;                                     // [kWsMaxUnits]
    __shared__ uint64_t loaded[R], full[R], empty[R];
    __shared__ WsTile tinfo[R];
    auto buf = [&](int r) { return smem + size_t(r) * L::kBuf; };
    if (threadIdx.x == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            mbar_init(&loaded[r], 1);
            mbar_init(&full[r], kWsGatherWarps * 32);
            mbar_init(&empty[r], kWsConsWarps * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t nt = a.num_wtiles;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) {
        // ------------------------------------------------------------ TMA warp
        if (threadIdx.x != 0) return;
        const uint64_t pol_stream = a.stream_evict_first ? policy_evict_first() : policy_evict_normal();
        uint32_t i = 0;
        for (uint32_t k = blockIdx.x; k < nt; k += gridDim.x, ++i) {
            const int r = int(i % R);
            WsTile t;
            t.gs = a.wt_group[k], t.ge = a.wt_group[k + 1];
            t.S0 = a.wt_slot[k];
            t.nslots = uint32_t(a.wt_slot[k + 1] - t.S0);
            t.row0 = a.wt_row[k];
            t.nrows = a.wt_row[k + 1] - t.row0;
            const uint32_t ub0 = t.gs & ~1u, ub1 = (t.ge + 2) & ~1u;  // unit_base [gs, ge] in 16-B units
            const uint32_t tm0 = t.row0 & ~7u, tm1 = (t.row0 + t.nrows + 7) & ~7u;
            t.ub_skew = t.gs - ub0;
            t.tm_skew = t.row0 - tm0;
            if (i >= uint32_t(R)) mbar_wait(&empty[r], ((i / R) - 1) & 1);
            tinfo[r] = t;
            unsigned char* B = buf(r);
            const uint32_t bcols = t.nslots * 4, bvals = t.nslots * uint32_t(sizeof(T));
            const uint32_t bgd = (t.ge - t.gs + 1) * 16, bub = (ub1 - ub0) * 8, btm = (tm1 - tm0) * 2;
            mbar_arrive_tx(&loaded[r], bcols + bvals + bgd + bub + btm);
            if (t.nslots) {
                bulk_g2s(B + L::kVals, a.cols + t.S0, bcols, &loaded[r], pol_stream);
                bulk_g2s(B, a.vals + t.S0, bvals, &loaded[r], pol_stream);
            }
            unsigned char* M = B + L::kVals + L::kCols + L::kX;
            bulk_g2s(M, a.groups + t.gs, bgd, &loaded[r], pol_stream);
            bulk_g2s(M + L::kGd, a.unit_base + ub0, bub, &loaded[r], pol_stream);
            bulk_g2s(M + L::kGd + L::kUb, a.tm + tm0, btm, &loaded[r], pol_stream);
        }
        return;
    }
    if (warp <= uint32_t(kWsGatherWarps)) {
        // ------------------------------------------------ gather (issue) warps
        const uint64_t pol_x = a.x_evict_last ? policy_evict_last() : policy_evict_normal();
        const uint32_t gt = threadIdx.x - 32;
        constexpr uint32_t kG = kWsGatherWarps * 32;
        uint32_t i = 0;
        for (uint32_t k = blockIdx.x; k < nt; k += gridDim.x, ++i) {
            const int r = int(i % R);
            mbar_wait(&loaded[r], (i / R) & 1);
            const uint32_t n = tinfo[r].nslots;
            unsigned char* B = buf(r);
            const int* cs = reinterpret_cast<const int*>(B + L::kVals);
            T* xg = reinterpret_cast<T*>(B + L::kVals + L::kCols);
            constexpr uint32_t xs = sizeof(T) == 8 ? 1 : 2;  // slot stride of xg in T units
            for (uint32_t f = 4 * gt; f < n; f += 4 * kG) {
                const int4 c4 = *reinterpret_cast<const int4*>(cs + f);
                if (c4.x != -1) cp_async_x(xg + xs * f, a.x + c4.x, pol_x);
                if (c4.y != -1) cp_async_x(xg + xs * (f + 1), a.x + c4.y, pol_x);
                if (c4.z != -1) cp_async_x(xg + xs * (f + 2), a.x + c4.z, pol_x);
                if (c4.w != -1) cp_async_x(xg + xs * (f + 3), a.x + c4.w, pol_x);
            }
            cp_async_arrive(&full[r]);
        }
        return;
    }
    // -------------------------------------------------------------- consumers
    const uint32_t ct = threadIdx.x - (1 + kWsGatherWarps) * 32;
    constexpr uint32_t kCons = kWsConsWarps * 32;
    const double xs = x_scale_value(a);
    uint32_t i = 0;
    for (uint32_t k = blockIdx.x; k < nt; k += gridDim.x, ++i) {
        const int r = int(i % R);
        mbar_wait(&full[r], (i / R) & 1);
        const WsTile t = tinfo[r];
        unsigned char* B = buf(r);
        const T* vs = reinterpret_cast<const T*>(B);
        const int* cs = reinterpret_cast<const int*>(B + L::kVals);
        const T* xg = reinterpret_cast<const T*>(B + L::kVals + L::kCols);
        constexpr uint32_t xgs = sizeof(T) == 8 ? 1 : 2;
        double* part = reinterpret_cast<double*>(B + L::kVals + L::kCols);  // lane sums, in place over xg
        const unsigned char* M = B + L::kVals + L::kCols + L::kX;
        const GroupDesc* gd = reinterpret_cast<const GroupDesc*>(M);
        const uint64_t* ub = reinterpret_cast<const uint64_t*>(M + L::kGd) + t.ub_skew;
        const uint16_t* tm = reinterpret_cast<const uint16_t*>(M + L::kGd + L::kUb) + t.tm_skew;
        const uint32_t ng = t.ge - t.gs;
        const uint64_t u00 = ub[0];
        // unit / row -> group maps
        for (uint32_t q = ct; q < ng; q += kCons) {
            const uint32_t rb = gd[q].first_row - t.row0, re = gd[q + 1].first_row - t.row0;
            for (uint32_t rr = rb; rr < re; ++rr) s_rgrp[rr] = uint16_t(q);
            const uint32_t u1 = uint32_t(ub[q + 1] - u00);
            for (uint32_t u = uint32_t(ub[q] - u00); u < u1; ++u) s_ugrp[u] = uint16_t(q);
        }
        cons_sync();
        // lane sums (argcsr.cpp:193-203), four lanes (one unit) per step; the
        // sums go to a per-unit staging slot (j = 0 of the unit's lanes) once
        // every read of the unit is done
        const uint32_t nunits = uint32_t(ub[ng] - u00);
        for (uint32_t u = ct; u < nunits; u += kCons) {
            const uint32_t q = s_ugrp[u];
            const GroupDesc d = gd[q];
            const uint32_t g = t.gs + q;
            if (d.heavy() || d.chunk == 0 || g < a.g_begin || g >= a.g_end) continue;
            const uint32_t W = d.stride(), C = d.chunk;
            const uint32_t o = uint32_t(d.offset() - t.S0) + (u - uint32_t(ub[q] - u00)) * 4;
            double acc[4];
            bool live[4];
#pragma unroll
            for (int l = 0; l < 4; ++l) acc[l] = 0.0, live[l] = true;
            for (uint32_t j = 0; j < C; ++j) {
                const uint32_t sl = o + j * W;
                const int4 c4 = *reinterpret_cast<const int4*>(cs + sl);
                const int cc[4] = {c4.x, c4.y, c4.z, c4.w};
                bool any = false;
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    live[l] = live[l] && cc[l] != -1;
                    if (live[l]) {
                        const double xv = double(xg[xgs * (sl + l)]);
                        const double xx = a.x_scale ? __dmul_rn(xv, xs) : xv;
                        acc[l] = __dadd_rn(acc[l], __dmul_rn(double(vs[sl + l]), xx));
                    }
                    any |= live[l];
                }
                if (!any) break;
            }
            *reinterpret_cast<double4*>(part + o) = make_double4(acc[0], acc[1], acc[2], acc[3]);
        }
        cons_sync();
        // row sums: +0.0 + lane sums in ascending order (argcsr.cpp:206-215)
        const double* ls = part;
        for (uint32_t rr = ct; rr < t.nrows; rr += kCons) {
            const uint32_t q = s_rgrp[rr];
            const GroupDesc d = gd[q];
            const uint32_t g = t.gs + q;
            if (d.heavy() || g < a.g_begin || g >= a.g_end) continue;
            const uint32_t lb = rr == d.first_row - t.row0 ? 0u : uint32_t(tm[rr - 1]);
            const uint32_t le = tm[rr];
            double sum = 0.0;
            if (d.chunk) {
                const double* base = ls + (d.offset() - t.S0);
                for (uint32_t l = lb; l < le; ++l) sum = __dadd_rn(sum, base[l]);
            }
            store_y<false>(a, t.row0 + rr, sum);
        }
        cons_sync();  // maps and ring buffer r are free again
        mbar_arrive(&empty[r]);
    }
}

template <typename T>
size_t ws_smem_bytes() {
    return size_t(WsLayout<T>::kRing) * WsLayout<T>::kBuf + size_t(kWsMaxRows + kWsMaxUnits) * 2;
}

