/*
 * argcsr_gpu.h — C-ABI of the B200-native ARG-CSR hot path.
 *
 * Drop-in boundary for the reference library `argcsr` (arxiv/paper_1203_5737,
 * /root/reference/proj).  Each entry point names the reference interface it
 * replaces (paths relative to /root/reference).  Plain pointers and sizes only:
 * no C++ or torch types cross this boundary, so the reference's C++ API
 * (include/argcsr_gpu.hpp), its pybind11 module (paper_1203_5737_b200) and any
 * other FFI (ctypes, cgo, JNI, ...) bind the same symbols.
 *
 * Conventions
 *   - Every function returns an argcsr_status; on failure a thread-local
 *     message is available from argcsr_last_error().  The C++ shim rethrows the
 *     status as the matching proj/include/argcsr/errors.hpp class.
 *   - Validation order and messages follow the reference: threads_per_group /
 *     desired_chunk_size first (argcsr.cpp:20-23), then an empty matrix
 *     (argcsr.cpp:24-26), then vector lengths (argcsr.cpp:220-223).
 *   - A handle owns device memory on one device and its matrix is immutable
 *     after argcsr_dev_convert.  Any thread may call any entry point on any
 *     stream.  SpMVs on ONE handle are serialised in issue order: each
 *     argcsr_dev_spmv* makes its stream wait for the previous SpMV on that
 *     handle (a per-handle event), because the x-remap buffer and the
 *     heavy-group stream are per-handle scratch.  SpMVs on different handles
 *     run concurrently.  `stream` is a cudaStream_t passed as void* (NULL =
 *     the legacy default stream).
 *   - Process-wide side effect: while at least one handle lives on a device,
 *     that device's persisting-L2 limit (cudaLimitPersistingL2CacheSize) is
 *     raised to its maximum so x can be kept L2-resident through an
 *     access-policy window.  The previous limit is saved by the first handle
 *     and restored (after cudaCtxResetPersistingL2Cache) when the last one is
 *     freed.  Set ARGCSR_L2_PERSIST=0 to leave the limit untouched.
 *   - argcsr_dev_spmv* on device pointers are stream-ordered and never
 *     synchronise except to report an error.  Calls with host pointers are
 *     synchronous, like the reference's value-returning functions.
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point fails with ARGCSR_E_CUDA.
 */
#ifndef ARGCSR_GPU_H
#define ARGCSR_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ARGCSR_GPU_ABI_VERSION 2

#if defined(__GNUC__)
#define ARGCSR_API __attribute__((visibility("default")))
#else
#define ARGCSR_API
#endif

typedef enum {
    ARGCSR_OK = 0,
    ARGCSR_E_PARAMETER = 1,   /* argcsr::ParameterError   (errors.hpp:27) */
    ARGCSR_E_DIMENSION = 2,   /* argcsr::DimensionError   (errors.hpp:21) */
    ARGCSR_E_BOUNDS = 3,      /* argcsr::BoundsError      (errors.hpp:15) */
    ARGCSR_E_INTERNAL = 4,    /* argcsr::InternalError    (errors.hpp:33) */
    ARGCSR_E_CUDA = 5,        /* CUDA runtime/driver failure -> InternalError subclass */
    ARGCSR_E_NCCL = 6,        /* collective failure          -> InternalError subclass */
    ARGCSR_E_OOM = 7,         /* device or pinned-host allocation failed */
    ARGCSR_E_FORMAT = 8,      /* argcsr::FormatError      (errors.hpp:51) */
    ARGCSR_E_IO = 9,          /* argcsr::IoError          (errors.hpp:57) */
    ARGCSR_E_PARSE = 10,      /* argcsr::ParseError       (errors.hpp:39) */
    ARGCSR_E_UNSUPPORTED = 11 /* argcsr::UnsupportedError (errors.hpp:45) */
} argcsr_status;

typedef enum { ARGCSR_F64 = 0, ARGCSR_F32 = 1 } argcsr_dtype;

typedef enum { ARGCSR_HOST = 0, ARGCSR_DEVICE = 1 } argcsr_memspace;

/* A CSR matrix (proj/include/argcsr/core.hpp:31-41): row i owns
 * [row_pointers[i], row_pointers[i+1]) of columns/values.  Pointers are host
 * or device memory according to `space`.  Like the reference converter, the
 * device converter neither validates nor re-sorts entries (argcsr.cpp:107-117). */
typedef struct {
    uint64_t num_rows;
    uint64_t num_cols;
    uint64_t nnz;
    const uint64_t* row_pointers; /* [num_rows + 1] */
    const int32_t* columns;       /* [nnz] */
    const void* values;           /* [nnz] of dtype */
    argcsr_dtype dtype;
    argcsr_memspace space;
} argcsr_csr_view;

/* Opaque device-resident ARG-CSR matrix (proj/include/argcsr/argcsr.hpp:52-63). */
typedef struct argcsr_dev argcsr_dev;

typedef struct {
    uint64_t num_rows;
    uint64_t num_cols;
    uint64_t threads_per_group;
    uint64_t desired_chunk_size;
    uint64_t num_groups;       /* ArgCsrMatrix::groups.size() */
    uint64_t total_slots;      /* ArgCsrMatrix::total_slots() (argcsr.hpp:61) */
    uint64_t stored_slots;     /* slots held on the device (== total_slots in the reference layout) */
    uint64_t nnz;              /* explicit entries */
    uint64_t heavy_groups;     /* groups scheduled on the long-chunk path */
    uint64_t heavy_ctas;       /* CTAs the heavy groups are packed into */
    uint64_t light_tiles;      /* CTA tiles of the short-chunk path */
    uint64_t max_chunk_size;
    uint64_t device_bytes;     /* device memory held by the handle */
    uint64_t l2_persist_bytes; /* persisting-L2 carve-out available to the x window */
    int32_t device;
    argcsr_dtype dtype;
    uint32_t layout;           /* 0 = lane-compact (default), ARGCSR_LAYOUT_REFERENCE */
    uint32_t x_remap;          /* 1: stored columns index x' = x[perm] (see ARGCSR_XREMAP_ON) */
    uint64_t x_used_columns;   /* columns with an entry (x_remap) or num_cols */
    uint64_t unit_len_bytes;   /* per-unit step counts the SpMV stops at (0: not kept, reads to chunk_size) */
} argcsr_dev_info_t;

/* Device layout of the value/column blocks (argcsr_dev_convert_ex flags).
 * Default (0): lane-compact -- each group's block is stored with a lane stride
 * of its assigned threads rounded up to the SpMV vector width instead of
 * threads_per_group, so the free lanes the reference pads with (0.0, -1) are
 * not stored and the SpMV streams the matrix contiguously.  Groups, chunk
 * order, threads_mapping and every exported array are unchanged (export
 * re-expands to the reference layout bit-exactly).
 * ARGCSR_LAYOUT_REFERENCE: keep the reference arrays verbatim on the device
 * (stride threads_per_group, argcsr.cpp:99-104). */
#define ARGCSR_LAYOUT_REFERENCE 1u

/* x remap (lane-compact layout only).  The device stores column indices in
 * an internal order -- used columns first, most-used first by octave, index
 * order within an octave -- and every SpMV gathers x' = x[perm] (one small
 * kernel) so that x's hot head fits the persisting-L2 window.  Products and
 * sums are unchanged (bit-identical results); every exported array maps back
 * to reference column indices.  Default: automatic (on when x exceeds the
 * window and the remap raises the window's nnz coverage by >= 5 points). */
#define ARGCSR_XREMAP_ON 2u
#define ARGCSR_XREMAP_OFF 4u

/* ---------------------------------------------------------------- conversion */

/* Replaces argcsr::argcsr_from_csr(const CsrMatrix&, tpg = 128, dcs = 1)
 * (argcsr.hpp:101-104, argcsr.cpp:123-155).  Runs row_nnz, partition_groups,
 * assign_threads, the inclusive threads_mapping scan and layout_group as GPU
 * kernels on `device`; the result is bit-exact with the reference arrays
 * (see argcsr_dev_export).  Host-space inputs are copied to the device.
 * Synchronises `stream` (group and slot counts size the allocations). */
ARGCSR_API argcsr_status argcsr_dev_convert(const argcsr_csr_view* csr, uint64_t threads_per_group,
                                 uint64_t desired_chunk_size, int device, void* stream,
                                 argcsr_dev** out);

/* argcsr_dev_convert with layout flags (0 or ARGCSR_LAYOUT_REFERENCE);
 * argcsr_dev_convert(...) == argcsr_dev_convert_ex(..., 0, out). */
ARGCSR_API argcsr_status argcsr_dev_convert_ex(const argcsr_csr_view* csr, uint64_t threads_per_group,
                                    uint64_t desired_chunk_size, int device, void* stream, uint32_t flags,
                                    argcsr_dev** out);

ARGCSR_API argcsr_status argcsr_dev_info(const argcsr_dev* m, argcsr_dev_info_t* info);

/* Copies the reference layout to HOST memory, widened to the reference field
 * types (argcsr.hpp:23-30, 52-63).  Any pointer may be NULL to skip it.
 *   groups4          [num_groups * 4] u64: first_row, size, offset, chunk_size
 *   threads_mapping  [num_rows] u64 (per-group inclusive scan)
 *   values           [total_slots] f64 (or f32 for an F32 handle); padding +0.0
 *   columns          [total_slots] i32; padding -1 (core.hpp:15)           */
ARGCSR_API argcsr_status argcsr_dev_export(const argcsr_dev* m, uint64_t* groups4, uint64_t* threads_mapping,
                                void* values, int32_t* columns);

/* --------------------------------------------------------------------- SpMV */

/* y = A x on device pointers, stream-ordered: x[num_cols], y[num_rows] of the
 * handle's dtype.  Replaces spmv_argcsr / spmv_argcsr_parallel
 * (argcsr.cpp:219-227, bench.cpp:109-116).  fp64 results are bit-identical to
 * the reference (same per-chunk and per-row summation order, no FMA). */
ARGCSR_API argcsr_status argcsr_dev_spmv(const argcsr_dev* m, const void* x, void* y, void* stream);

/* y = A (s * x) with s = *x_scale, a DEVICE scalar read by the kernel (NULL:
 * s = 1.0).  The scale is applied to every gathered x value (fl(s * x[c])),
 * bit-identical to scaling x beforehand; the power iteration uses it to fuse
 * the previous step's normalisation without a host round trip. */
ARGCSR_API argcsr_status argcsr_dev_spmv_scaled(const argcsr_dev* m, const void* x, const double* x_scale, void* y,
                                                void* stream);

/* Group-range kernel (argcsr.hpp:114-116, argcsr.cpp:185-217): writes only the
 * rows of groups [group_begin, group_end); no length check, like the reference. */
ARGCSR_API argcsr_status argcsr_dev_spmv_groups(const argcsr_dev* m, const void* x, uint64_t group_begin,
                                     uint64_t group_end, void* y, void* stream);

/* The general form: rows of groups [group_begin, group_end) of y = A (s x),
 * s = *x_scale on the device (NULL: 1).  ARGCSR_SPMV_REUSE_X lets a handle
 * with the x remap on skip its x' gather and reuse the previous launch's x'
 * (the multi-GPU step runs interior then boundary groups on the same x). */
#define ARGCSR_SPMV_REUSE_X 1u
ARGCSR_API argcsr_status argcsr_dev_spmv_ex(const argcsr_dev* m, const void* x, const double* x_scale,
                                 uint64_t group_begin, uint64_t group_end, void* y, uint32_t flags,
                                 void* stream);

/* ------------------------------------------ multi-GPU step over peer memory
 * The fused form of "SpMV, then all-gather y": the kernel's
 * epilogue stores every y row both to y and to peer_y[q][row] for q < npeers
 * (npeers <= 7) -- the other GPUs' next-x buffers seen through NVLink peer
 * mappings (argcsr_peer_open), pre-offset by this slice's first row -- so the
 * y slice reaches every GPU tile by tile while the SpMV runs, with no separate
 * collective.  peer_rows (2 * npeers entries, may be NULL = all rows) limits
 * peer q to rows [peer_rows[2q], peer_rows[2q+1]): the rows its columns read
 * (a halo for banded matrices).  Otherwise argcsr_dev_spmv_ex. */
ARGCSR_API argcsr_status argcsr_dev_spmv_peer(const argcsr_dev* m, const void* x, const double* x_scale,
                                              uint64_t group_begin, uint64_t group_end, void* y,
                                              void* const* peer_y, uint32_t npeers, const uint64_t* peer_rows,
                                              uint32_t flags, void* stream);

/* Step signalling, stream-ordered one-thread kernels: store `value` into
 * *flags[q] for q < n with system-scope release semantics (after copying the
 * device scalar *partial to *partial_dst[q] when both are non-NULL); wait
 * until every flags[i] (i < n, local memory written by peers) is >= value. */
ARGCSR_API argcsr_status argcsr_peer_signal(uint64_t* const* flags, uint32_t n, uint64_t value,
                                            const double* partial, double* const* partial_dst, void* stream);
ARGCSR_API argcsr_status argcsr_peer_wait(const uint64_t* flags, uint32_t n, uint64_t value, void* stream);

/* Device buffers shared between the processes of one box (CUDA IPC): allocate
 * `bytes` (zeroed) on `device` and return its 64-byte IPC handle; open a
 * peer's handle in this process (peer access is enabled first); close/free. */
ARGCSR_API argcsr_status argcsr_peer_alloc(uint64_t bytes, int device, void** ptr, unsigned char handle[64]);
ARGCSR_API argcsr_status argcsr_peer_open(const unsigned char handle[64], int device, void** ptr);
ARGCSR_API argcsr_status argcsr_peer_close(void* ptr);
ARGCSR_API argcsr_status argcsr_peer_free(void* ptr);

/* Host-buffer form of spmv_argcsr (argcsr.cpp:219-227): checks x_len ==
 * num_cols (DimensionError, same message shape), copies x in, multiplies,
 * copies y (num_rows entries) out, synchronises. */
ARGCSR_API argcsr_status argcsr_dev_spmv_host(const argcsr_dev* m, const void* x, uint64_t x_len, void* y);

/* Same, with caller-pinned host buffers and caller-owned device staging
 * (x_dev/y_dev), on `stream`: H2D x, SpMV, D2H y, then synchronise.  The
 * end-to-end path bench.py times. */
ARGCSR_API argcsr_status argcsr_dev_spmv_host_staged(const argcsr_dev* m, const void* x_host, void* x_dev,
                                          void* y_dev, void* y_host, void* stream);

/* Non-blocking host-buffer SpMV for a stream of vectors: uploads x_host
 * (num_cols entries, pinned for a true async copy) on one copy engine,
 * multiplies on `stream`, downloads y (num_rows entries) into y_host on the
 * other copy engine, and returns at once.  The handle double-buffers its own
 * device staging, so call i+1's upload overlaps call i's SpMV and call i-1's
 * download.  x_host must stay unmodified and y_host untouched until
 * argcsr_dev_host_wait(m) returns (every earlier call is then complete).
 * One host thread drives a handle's async calls. */
ARGCSR_API argcsr_status argcsr_dev_spmv_host_async(const argcsr_dev* m, const void* x_host, void* y_host,
                                                    void* stream);
ARGCSR_API argcsr_status argcsr_dev_host_wait(const argcsr_dev* m);

/* ----------------------------------------------------------- accessors / next */

/* csr_from_argcsr (argcsr.cpp:157-183) on the device: writes the lossless CSR
 * back into HOST arrays row_pointers[num_rows+1], columns[nnz], values[nnz]. */
ARGCSR_API argcsr_status argcsr_dev_to_csr(const argcsr_dev* m, uint64_t* row_pointers, int32_t* columns,
                                void* values);

/* chunk_entries (argcsr.cpp:229-249): non-sentinel entries of chunk (g, c) in
 * storage order into host arrays of capacity `cap`; *n gets the count.
 * BoundsError on a bad group or chunk index. */
ARGCSR_API argcsr_status argcsr_dev_chunk_entries(const argcsr_dev* m, uint64_t group_index,
                                       uint64_t chunk_index, void* values, int32_t* columns,
                                       uint64_t cap, uint64_t* n);

/* padding_stats(const ArgCsrMatrix&) (analysis.cpp:167-184) reduced on the device. */
typedef struct {
    uint64_t explicit_nnz;
    uint64_t assigned_padded_slots;
    uint64_t total_allocated_slots;
    double padding_ratio;
    uint64_t estimated_bytes;
} argcsr_format_stats;
ARGCSR_API argcsr_status argcsr_dev_padding_stats(const argcsr_dev* m, argcsr_format_stats* out);

/* balance_stats(const ArgCsrMatrix&) (analysis.cpp:198-208, balance_of :29-55):
 * explicit entries per group (per_group_nnz[num_groups], may be NULL),
 * max / mean and the coefficient of variation -- bit-identical to the
 * reference (counts on the device, the ratios on the host in its order). */
ARGCSR_API argcsr_status argcsr_dev_balance_stats(const argcsr_dev* m, uint64_t* per_group_nnz,
                                                  double* max_over_mean, double* coefficient_of_variation);

ARGCSR_API void argcsr_dev_free(argcsr_dev* m);

/* ------------------------------------------- ELLPACK / Sliced ELLPACK */

/* The paper's comparison formats (proj/include/argcsr/ellpack.hpp): an
 * opaque device matrix in the reference layout -- slice s is a columnwise
 * block, slot j of local row r at slice_offsets[s] + j * rows_in_slice + r,
 * padding (0.0, -1) trailing; ELLPACK is one slice of all rows. */
typedef struct argcsr_sell argcsr_sell;

typedef struct {
    uint64_t num_rows;
    uint64_t num_cols;
    uint64_t slice_size;   /* num_rows for ELLPACK */
    uint64_t num_slices;
    uint64_t total_slots;
    uint64_t width;        /* widest slice (EllpackMatrix::width) */
    uint64_t device_bytes;
    int32_t device;
    argcsr_dtype dtype;
    uint32_t ellpack;      /* 1: made by argcsr_ell_convert */
} argcsr_sell_info_t;

/* ellpack_from_csr (ellpack.cpp:7-24) on the device. */
ARGCSR_API argcsr_status argcsr_ell_convert(const argcsr_csr_view* csr, int device, void* stream, argcsr_sell** out);
/* sliced_from_csr(A, slice_size = 32) (ellpack.cpp:26-60); slice_size 0 -> ParameterError. */
ARGCSR_API argcsr_status argcsr_sell_convert(const argcsr_csr_view* csr, uint64_t slice_size, int device,
                                  void* stream, argcsr_sell** out);
ARGCSR_API argcsr_status argcsr_sell_info(const argcsr_sell* m, argcsr_sell_info_t* info);
/* Host copies of the reference fields; any pointer may be NULL. */
ARGCSR_API argcsr_status argcsr_sell_export(const argcsr_sell* m, uint64_t* slice_widths, uint64_t* slice_offsets,
                                 void* values, int32_t* columns);
/* spmv_ellpack / spmv_sliced (ellpack.cpp:121-176), bit-identical fp64; device
 * pointers, stream-ordered. */
ARGCSR_API argcsr_status argcsr_sell_spmv(const argcsr_sell* m, const void* x, void* y, void* stream);
/* Host vectors, synchronous; x_len != num_cols -> DimensionError (ellpack.cpp:135-139). */
ARGCSR_API argcsr_status argcsr_sell_spmv_host(const argcsr_sell* m, const void* x, uint64_t x_len, void* y);
ARGCSR_API void argcsr_sell_free(argcsr_sell* m);

/* ------------------------------------------------------- import / binary */

/* The reference ArgCsrMatrix (argcsr.hpp:52-63) as host arrays. */
typedef struct {
    uint64_t num_rows;
    uint64_t num_cols;
    uint64_t threads_per_group;
    uint64_t num_groups;
    const uint64_t* groups4;         /* [num_groups * 4]: first_row, size, offset, chunk_size */
    const uint64_t* threads_mapping; /* [num_rows] */
    const void* values;              /* [total_slots] f64 (or f32) */
    const int32_t* columns;          /* [total_slots] */
    uint64_t total_slots;
    argcsr_dtype dtype;
} argcsr_argcsr_view;

/* A device handle from the reference arrays (e.g. a cached conversion),
 * without re-running the converter: the arrays are checked (groups tile the
 * rows, reference offsets, threads_mapping increasing per group, free lanes
 * all padding, padding trailing per lane; ARGCSR_E_FORMAT otherwise) and laid
 * out as after argcsr_dev_convert_ex(flags).  desired_chunk_size reads 0. */
ARGCSR_API argcsr_status argcsr_dev_import(const argcsr_argcsr_view* matrix, int device, void* stream,
                                uint32_t flags, argcsr_dev** out);

/* write_binary(ostream, const ArgCsrMatrix&) (io.cpp:282-298) to a file: the
 * reference's SPFMTBIN container, byte-identical to the reference writing
 * argcsr_from_csr of the same input.  fp64 handles only. */
ARGCSR_API argcsr_status argcsr_dev_write_binary(const argcsr_dev* m, const char* path);

/* read_binary_file (io.cpp:300-366) onto the device: an ARG-CSR container is
 * imported (argcsr_dev_import); a CSR container is converted with
 * threads_per_group / desired_chunk_size (argcsr_dev_convert_ex).  Bad magic,
 * version or tag -> ARGCSR_E_FORMAT; truncation -> ARGCSR_E_PARSE; ELLPACK
 * containers -> ARGCSR_E_UNSUPPORTED; unreadable file -> ARGCSR_E_IO. */
ARGCSR_API argcsr_status argcsr_dev_read_binary(const char* path, uint64_t threads_per_group,
                                     uint64_t desired_chunk_size, int device, void* stream,
                                     uint32_t flags, argcsr_dev** out);

/* ------------------------------------------------------ multi-GPU row slices */

/* nnz-balanced contiguous row split: row_begin[p] =
 * lower_bound(row_pointers, p*nnz/parts), row_begin[parts] = num_rows; rows of
 * each part >= 1 when num_rows >= parts.  row_pointers is host memory. */
ARGCSR_API argcsr_status argcsr_partition_rows(const uint64_t* row_pointers, uint64_t num_rows,
                                    uint32_t parts, uint64_t* row_begin);

/* ---------------------------------------------- single-GPU power iteration
 * y = A (s * x) and ||y||^2 in one pass: the SpMV epilogue accumulates the
 * squares of the stored y values into per-CTA partials that a one-CTA kernel
 * sums in a fixed order into *y_norm2 (device double) -- deterministic run to
 * run.  x_scale as argcsr_dev_spmv_scaled; with ARGCSR_SCALE_IS_NORM2 in
 * flags, *x_scale holds the previous step's ||y||^2 and the scale is
 * fl(1 / fl(sqrt(*x_scale))): the normalisation x_{k+1} = y_k / ||y_k|| of the
 * power iteration fused into the next product's gathers. */
#define ARGCSR_SCALE_IS_NORM2 2u
ARGCSR_API argcsr_status argcsr_dev_spmv_norm2(const argcsr_dev* m, const void* x, const double* x_scale,
                                               void* y, double* y_norm2, uint32_t flags, void* stream);

/* ------------------------------------------------ multi-GPU
 * Replaces the reference's only parallel path, parallel_over /
 * spmv_argcsr_parallel (proj/src/bench.cpp:48-71, 109-116; bench.hpp:59-60):
 * rows are split into contiguous nnz-balanced slices (argcsr_partition_rows),
 * each GPU converts ITS slice (bit-exact with argcsr_from_csr(slice)), x is
 * replicated, and one step is the slice SpMV plus the exchange of the y slices
 * into every GPU's next x:
 *   ARGCSR_EXCHANGE_ALLGATHER  ncclAllGather in place (equal slices), else one
 *                              ncclBroadcast per owner (grouped);
 *   ARGCSR_EXCHANGE_HALO       only the x rows other slices read (grouped
 *                              ncclSend/ncclRecv of a plan built at setup);
 *   ARGCSR_EXCHANGE_P2P        no collective: the SpMV epilogue stores y into
 *                              the peers' next x over NVLink (CUDA IPC or
 *                              peer access), step flags + partial norms in
 *                              peer memory;
 *   ARGCSR_EXCHANGE_AUTO       halo when it moves < 1/4 of the all-gather's
 *                              volume, else all-gather.
 * NCCL is loaded at run time (dlopen libnccl.so.2); collective failures and
 * asynchronous communicator errors (ncclCommGetAsyncError, polled every step)
 * return ARGCSR_E_NCCL.  The power iteration fuses ||y||^2 into the SpMV
 * epilogue, all-reduces 8 bytes, and fuses the scaling into the next SpMV.
 * With the NCCL exchanges a step overlaps the exchange of step k with the
 * interior groups (rows reading only the slice's own x rows) of step k+1. */
typedef struct argcsr_mgpu argcsr_mgpu;
typedef enum {
    ARGCSR_EXCHANGE_AUTO = 0,
    ARGCSR_EXCHANGE_ALLGATHER = 1,
    ARGCSR_EXCHANGE_HALO = 2,
    ARGCSR_EXCHANGE_P2P = 3,
    ARGCSR_EXCHANGE_NONE = 4 /* reported for one rank */
} argcsr_exchange;
#define ARGCSR_NCCL_ID_BYTES 128

typedef struct {
    int32_t rank;              /* global rank of local rank 0 */
    int32_t nranks;
    int32_t nlocal;            /* GPUs driven by this handle (1 per process in the multi-process form) */
    int32_t exchange;          /* argcsr_exchange actually used */
    uint64_t num_rows, num_cols, nnz;
    uint64_t row_begin, row_end;   /* local rank 0's slice */
    uint64_t interior_begin, interior_end;  /* its interior group range */
    uint64_t halo_recv_rows;   /* x rows it receives per step (halo exchange) */
    uint64_t step;             /* steps issued since create */
} argcsr_mgpu_info_t;

/* ncclGetUniqueId: rank 0 calls it and shares the bytes with the other ranks
 * (any channel: torch.distributed, MPI, a file). */
ARGCSR_API argcsr_status argcsr_mgpu_unique_id(unsigned char id[ARGCSR_NCCL_ID_BYTES]);

/* One process per GPU: rank `rank` of `nranks` on `device`.  `A` is the FULL
 * matrix (host or device; every rank passes the same one).  `nccl_id` may be
 * NULL only for nranks == 1 or for ARGCSR_EXCHANGE_P2P with an external
 * connection (argcsr_mgpu_p2p_export / argcsr_mgpu_p2p_connect).  Collective
 * over the ranks (NCCL communicator setup, halo plan, IPC handle exchange).
 * flags: argcsr_dev_convert_ex layout flags. */
ARGCSR_API argcsr_status argcsr_mgpu_create_rank(const argcsr_csr_view* A, int rank, int nranks,
                                                 const unsigned char* nccl_id, uint64_t threads_per_group,
                                                 uint64_t desired_chunk_size, int device, uint32_t flags,
                                                 argcsr_exchange exchange, argcsr_mgpu** out);

/* One process drives `ngpus` devices (SURVEY §8(b) signature): NCCL
 * communicators from ncclCommInitAll; collectives grouped.  A device may be
 * listed more than once only with ARGCSR_EXCHANGE_P2P (virtual ranks sharing
 * a GPU: tests). */
ARGCSR_API argcsr_status argcsr_mgpu_create(const argcsr_csr_view* A, int ngpus, const int* devices,
                                            uint64_t threads_per_group, uint64_t desired_chunk_size,
                                            argcsr_exchange exchange, argcsr_mgpu** out);

ARGCSR_API argcsr_status argcsr_mgpu_info(const argcsr_mgpu* h, argcsr_mgpu_info_t* info);
/* The slice handle of local rank i (borrowed: freed with h). */
ARGCSR_API argcsr_status argcsr_mgpu_local(const argcsr_mgpu* h, int i, argcsr_dev** slice);

/* P2P exchange without NCCL (multi-process, caller-provided channel):
 * export this rank's 64-byte IPC handle and the [lo, hi) global rows it reads
 * from every owner (need[2*p], need[2*p+1]); then connect with every rank's
 * handle (handles[64*p]) and every rank's need table (need_all[(q*nranks+p)*2]
 * = rows q reads from p).  Collective: every rank exports, exchanges, connects. */
ARGCSR_API argcsr_status argcsr_mgpu_p2p_export(const argcsr_mgpu* h, unsigned char handle[64], uint64_t* need);
ARGCSR_API argcsr_status argcsr_mgpu_p2p_connect(argcsr_mgpu* h, const unsigned char* handles,
                                                 const uint64_t* need_all);

/* Iterated SpMV / power iteration over the handle's double-buffered x (all
 * arrays below have one entry per local rank; streams may be NULL = the
 * legacy default stream).  begin: x_k <- x0 (full length, device), normalize
 * selects the power iteration; step: one step (last != 0: every row is
 * exchanged, so all GPUs end with all of x -- the halo modes otherwise move
 * only the rows others read); finish: wait, then lambda = ||A x_{k-1}||
 * (normalize) and x_out (full, device, may be NULL) = the current x
 * (normalised).  Stream-ordered except finish, which synchronises. */
ARGCSR_API argcsr_status argcsr_mgpu_begin(argcsr_mgpu* h, const void* const* x0, int normalize,
                                           void* const* streams);
ARGCSR_API argcsr_status argcsr_mgpu_step(argcsr_mgpu* h, int last, void* const* streams);
ARGCSR_API argcsr_status argcsr_mgpu_finish(argcsr_mgpu* h, double* lambda, void* const* x_out,
                                            void* const* streams);
/* Stream-ordered: `streams` wait until the last step's exchange has landed
 * (x_k complete on every local GPU) -- the end of a timed region. */
ARGCSR_API argcsr_status argcsr_mgpu_wait(argcsr_mgpu* h, void* const* streams);

/* out = A x assembled on every local rank (full-length device vectors): the
 * slice SpMV into out[row_begin:row_end] and the exchange, stream-ordered. */
ARGCSR_API argcsr_status argcsr_mgpu_spmv_gather(argcsr_mgpu* h, const void* const* x, void* const* out,
                                                 void* const* streams);

/* `iters` power-iteration steps from the host vector x_host_io
 * (num_cols entries of the matrix dtype), written back normalised; lambda =
 * ||A x_{iters-1}||.  Synchronous; every rank calls it. */
ARGCSR_API argcsr_status argcsr_mgpu_power_iteration(argcsr_mgpu* h, int iters, void* x_host_io,
                                                     double* lambda_out);

/* Poll the communicators (ncclCommGetAsyncError): ARGCSR_E_NCCL on error. */
ARGCSR_API argcsr_status argcsr_mgpu_check(argcsr_mgpu* h);
ARGCSR_API void argcsr_mgpu_free(argcsr_mgpu* h);

/* Host planning helpers of the multi-GPU layer (no device needed; the
 * create calls use them on host copies of each slice).
 * interior: the longest run [*ga, *gb) of groups (first rows group_first[0..G],
 * group_first[G] = slice rows) whose rows (slice row pointers rp, rebased)
 * reference only columns in [r0, r1).
 * needed: the distinct global rows (ascending) of owner p != self that the
 * slice's columns reference, for every owner: counts[p] (always) and, when
 * rows is non-NULL, the rows of owner 0, 1, ... concatenated. */
ARGCSR_API argcsr_status argcsr_plan_interior(const uint64_t* rp, const int32_t* columns, uint64_t rows,
                                              const uint64_t* group_first, uint64_t num_groups, uint64_t r0,
                                              uint64_t r1, uint64_t* ga, uint64_t* gb);
ARGCSR_API argcsr_status argcsr_plan_needed(const int32_t* columns, uint64_t nnz, uint64_t num_cols,
                                            const uint64_t* bounds, uint32_t parts, uint32_t self,
                                            uint64_t* counts, uint64_t* rows);

/* ------------------------------------------------------------------- errors */
ARGCSR_API const char* argcsr_last_error(void);
ARGCSR_API const char* argcsr_status_name(argcsr_status s);
ARGCSR_API int argcsr_abi_version(void);
/* Experiment switches (ARGCSR_* environment variables) are read
 * once, at first use; this re-reads them (tests flip them between cases). */
ARGCSR_API void argcsr_reload_options(void);

#ifdef __cplusplus
}
#endif
#endif /* ARGCSR_GPU_H */
