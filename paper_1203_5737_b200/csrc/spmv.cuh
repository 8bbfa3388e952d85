// SpMV launch (spmv.cu).
#pragma once

#include "common.cuh"

namespace argcsr_gpu {

// y = A x for the rows of groups [group_begin, group_end); device pointers,
// stream-ordered, no synchronisation.
// y = A (s * x), s = *x_scale (a device scalar, read by the kernel; NULL:
// 1.0).  The scale is applied per gather (fl(s * x[c])), bit-identical to
// scaling x first; 1.0 is an exact no-op.
// reuse_x: an x remap handle skips its x' gather and reuses the x' of the
// previous launch on this handle (same x, stream-ordered after it).
// peer_y[0 .. npeers): every row written to y that lies in
// [peer_rows[2q], peer_rows[2q+1]) (all rows when peer_rows is null) is also
// stored to peer_y[q][row] (multi-GPU: the other GPUs' x buffers, pre-offset
// by this slice's first row; the ranges are the rows each peer reads).
// norm_part: fused ||y||^2, one partial per CTA of this launch written to
// norm_part[0 .. norm_slots(m)) (heavy CTAs, then light tiles; CTAs with no
// row of the group range write 0); reduce them with norm_reduce.
// scale_is_norm2: *x_scale holds ||y_prev||^2 and the scale is 1/sqrt of it.
struct SpmvExtra {
    const double* x_scale = nullptr;
    bool scale_is_norm2 = false;
    bool reuse_x = false;
    void* const* peer_y = nullptr;
    uint32_t npeers = 0;
    const uint64_t* peer_rows = nullptr;
    double* norm_part = nullptr;
};
void spmv_launch(const argcsr_dev* m, const void* x, void* y, uint64_t group_begin, uint64_t group_end,
                 cudaStream_t s, const SpmvExtra& ex = SpmvExtra{});

// Serialises the SpMVs of one handle (argcsr_dev::mu, ev_done): wait for the
// previous SpMV on this handle, whatever stream it ran on; done() records the
// end of this one.  Every SpMV entry point (C-ABI, multi-GPU layer) uses it.
struct SpmvOrder {
    argcsr_dev* m;
    cudaStream_t s;
    std::unique_lock<std::mutex> lock;
    SpmvOrder(const argcsr_dev* mc, cudaStream_t st) : m(const_cast<argcsr_dev*>(mc)), s(st), lock(m->mu) {
        if (m->spmv_issued) CUDA_OK(cudaStreamWaitEvent(s, m->ev_done, 0));
    }
    void done() {
        CUDA_OK(cudaEventRecord(m->ev_done, s));
        m->spmv_issued = true;
    }
};

// Heavy groups run packed into m->heavy_ctas CTAs (one norm partial each).
inline uint64_t norm_heavy_slots(const argcsr_dev* m) { return uint64_t(m->heavy_ctas); }
inline uint64_t norm_slots(const argcsr_dev* m) { return norm_heavy_slots(m) + m->num_tiles; }

// out[0] = the sum of partials[0 .. n) in a fixed order (two levels of fixed
// trees; deterministic).  scratch: norm_scratch_len(n) doubles when n > 4096.
void norm_reduce(const double* partials, uint64_t n, double* out, cudaStream_t s, double* scratch = nullptr);
inline uint64_t norm_scratch_len(uint64_t n) { return (n + 4095) / 4096; }

// Step signalling between the GPUs of a multi-GPU step (spmv.cu): store
// `value` into flags[q] (system-scope release, after *partial is copied to
// partial_dst[q] when both are given); wait until flags[0 .. n) >= value.
void peer_signal(uint64_t* const* flags, uint32_t n, uint64_t value, const double* partial,
                 double* const* partial_dst, cudaStream_t s);
void peer_wait(const uint64_t* flags, uint32_t n, uint64_t value, cudaStream_t s);

// Light tiles [t0, t1) only (handles without heavy groups or x remap): the
// pipelined host path launches the tiles whose x window has arrived.
void spmv_launch_tiles(const argcsr_dev* m, const void* x, void* y, uint32_t t0, uint32_t t1, cudaStream_t s);

}  // namespace argcsr_gpu
