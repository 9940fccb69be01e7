/*
 * spmmm.h — C ABI of libspmmm.so, the B200 (sm_100a) CSR x CSR sparse
 * matrix-matrix product C = A·B (fp64 values, uint64 indices, sorted columns).
 *
 * This is the drop-in boundary for the reference's row-major spMMM entry point
 *     sparsemm.kernels.multiply_rowmajor(a, b, strategy=COMBINED, stats=None)
 *     (/root/reference/pkg/src/sparsemm/kernels.py:302-332)
 * The reference has no FFI of its own (it is pure Python); the ctypes binding a
 * maintainer adds on the reference side is shown in INTEGRATION.md, and the
 * Python mirror of the entry point lives in paper_1303_1651_b200/kernels.py.
 *
 * Data layout (formats.py:15-16, 40-58): CsrMatrix = (rows, cols,
 * row_ptr u64[rows+1], col_idx u64[nnz], values f64[nnz]) with strictly
 * increasing columns per row. Results follow the reference bit for bit in
 * structure; values follow its accumulation order exactly (left fold over the
 * A-row entries in ascending column order, separately rounded multiply and add,
 * exact zeros dropped: kernels.py:163-180, 285-299).
 *
 * Threading: every entry point is re-entrant per context; a context owns one
 * CUDA stream on one device. Errors are reported as status codes; the message
 * of the last failure on the calling thread is available from spmmm_last_error().
 */
#ifndef SPMMM_H
#define SPMMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPMMM_ABI_VERSION 1

/* Status codes. The Python shim maps 1 and 2 to ValueError and the rest to
 * RuntimeError (kernels.py:312-313 raises ValueError on dimension mismatch). */
typedef enum {
  SPMMM_OK = 0,
  SPMMM_ERR_DIMENSION = 1,   /* a.cols != b.rows                         (kernels.py:312-313) */
  SPMMM_ERR_INVALID = 2,     /* bad argument, malformed CSR, unknown strategy (kernels.py:77) */
  SPMMM_ERR_CUDA = 3,        /* CUDA runtime error                                          */
  SPMMM_ERR_NCCL = 4,        /* reserved for collective failures                           */
  SPMMM_ERR_OOM = 5,         /* device or host allocation failed                            */
  SPMMM_ERR_UNSUPPORTED = 6  /* shape outside the supported range (cols >= 2^32-1, ...)    */
} spmmm_status;

/* Where a CSR view's arrays live. */
typedef enum { SPMMM_MEM_HOST = 0, SPMMM_MEM_DEVICE = 1 } spmmm_memory;

/* Borrowed, read-only CSR view. For device views row_ptr[0] need not be 0:
 * a row block of a bigger matrix is passed as (row_ptr + r0, col_idx, values)
 * with `nnz` = length of the col_idx/values arrays. */
typedef struct {
  uint64_t rows;
  uint64_t cols;
  uint64_t nnz;
  const uint64_t* row_ptr;
  const uint64_t* col_idx;
  const double* values;
  int32_t memory; /* spmmm_memory */
  int32_t reserved;
} spmmm_csr;

/* Mirrors sparsemm.kernels.StrategyKind (kernels.py:38-47). Every strategy
 * yields the same bytes (kernels.py:1-17); the GPU validates and records it. */
typedef enum {
  SPMMM_STRATEGY_BFDOUBLE = 0,
  SPMMM_STRATEGY_BFBOOL = 1,
  SPMMM_STRATEGY_BFCHAR = 2,
  SPMMM_STRATEGY_MINMAX = 3,
  SPMMM_STRATEGY_MINMAXCHAR = 4,
  SPMMM_STRATEGY_SORT = 5,
  SPMMM_STRATEGY_COMBINED = 6
} spmmm_strategy;

/* spmmm_multiply flags */
#define SPMMM_FLAG_ROW_STATS 1u /* record per-row touched-range stats (KernelStats.row_choices) */
#define SPMMM_FLAG_TIMING 2u    /* record per-kernel CUDA-event durations on the context      */

typedef struct spmmm_context spmmm_context;
typedef struct spmmm_product spmmm_product;

int spmmm_abi_version(void);
const char* spmmm_last_error(void);
int spmmm_device_count(int* count);

/* One context per (device, stream). cuda_stream may be NULL (the context
 * creates its own non-blocking stream, unordered with the legacy default
 * stream) or a cudaStream_t owned by the caller — cudaStreamLegacy (0x1)
 * for the legacy default stream itself (torch's default stream). */
int spmmm_context_create(int device, void* cuda_stream, spmmm_context** out);
int spmmm_context_destroy(spmmm_context* ctx);
int spmmm_synchronize(spmmm_context* ctx);

/* C = A·B.  Replaces kernels.py:302-332 (multiply_rowmajor). A and B may be
 * host or device views; C stays device-resident in the returned product until
 * spmmm_product_destroy. Host inputs are uploaded on the context stream (A and
 * B that alias the same host arrays are uploaded once). */
int spmmm_multiply(spmmm_context* ctx, const spmmm_csr* a, const spmmm_csr* b, int strategy,
                   uint32_t flags, spmmm_product** out);

/* Shape, nnz(C) and the multiplication count (KernelStats.multiplications,
 * kernels.py:330-331 == perfmodel.count_mults). */
int spmmm_product_shape(const spmmm_product* p, uint64_t* rows, uint64_t* cols, uint64_t* nnz,
                        uint64_t* multiplications);
/* The split-mode row classes, for measurement tools (bench.py attributes the
 * products of a skewed input to the kernels that compute them):
 * out[0] products up to which a non-short row is one warp's (k_esc_warp),
 * out[1] products past which a row is cut into column-range parts,
 * out[2..4] the dominant-row rule (k_esc_dom): at most out[2] products outside
 * the row's longest B row, which has at least out[3] entries and, if out[4],
 * at least half of the row's products. */
int spmmm_row_classes(uint32_t out[5]);
/* Device bytes held by the product's arrays (their reservations: C's
 * col_idx/values are reserved before nnz(C) is known). */
int spmmm_product_reserved_bytes(const spmmm_product* p, uint64_t* bytes);
/* Device pointers of C (valid until spmmm_product_destroy). */
int spmmm_product_device_arrays(const spmmm_product* p, const uint64_t** row_ptr,
                                const uint64_t** col_idx, const double** values);
/* Copies C into caller-owned host buffers (rows+1, nnz, nnz entries). */
int spmmm_product_download(spmmm_product* p, uint64_t* row_ptr, uint64_t* col_idx,
                           double* values);

/* Result of spmmm_multiply_host: C in page-locked host memory from the
 * library's pool (return each array with spmmm_host_free). col_idx / values
 * hold `nnz` entries (their blocks may be larger). For large results row
 * pointers travel down as u32 and column indices as u32 or, when every
 * 64-entry chunk spans < 2^16 columns, as u16 deltas; host threads widen them
 * into the u64 arrays. h2d_bytes / d2h_bytes count what crossed PCIe. */
typedef struct {
  uint64_t rows, cols, nnz, mults;
  uint64_t* row_ptr;
  uint64_t* col_idx;
  double* values;
  uint64_t h2d_bytes, d2h_bytes;  /* PCIe bytes this call moved each way */
} spmmm_host_csr;

/* C = A·B for HOST operands, block-pipelined: A goes up in `blocks` row
 * blocks (<= 16) of about equal nnz — row pointers, columns, values — (for
 * A != B all of B first); there is no global count pass: block j is computed
 * as soon as the B rows it reads are resident (its own count validates it
 * and sizes its part of C) and its part of C streams down while the next block
 * computes — uploads, kernels and downloads overlap. Pageable operands go up
 * through the library's page-locked staging (several host threads). The
 * result is reserved at max(8 nnz(A), 2^20) entries of pooled page-locked
 * memory; a product past that is redone in one shot into exact-size arrays.
 * Same bytes, errors and multiplication count as spmmm_multiply +
 * spmmm_product_download (kernels.py:302-332); row stats are not available
 * here (use spmmm_multiply). Replaces, like spmmm_multiply,
 * sparsemm.kernels.multiply_rowmajor (kernels.py:302-332) for the drop-in. */
int spmmm_multiply_host(spmmm_context* ctx, const spmmm_csr* a, const spmmm_csr* b, int strategy,
                        uint32_t flags, int blocks, spmmm_host_csr* out);
/* Same, into caller-owned DEVICE buffers on the product's device (ordered on
 * the context stream; e.g. tensors that a collective then sends). */
int spmmm_product_copy_device(spmmm_product* p, uint64_t* row_ptr, uint64_t* col_idx,
                              double* values);
/* With SPMMM_FLAG_ROW_STATS: per row the smallest and largest touched column
 * and the length of the reference's touched list (kernels.py:170-178), from
 * which combined_select (kernels.py:186-191) gives row_choices. Rows that
 * touched nothing report min = UINT64_MAX, max = 0, touched = 0. */
int spmmm_product_row_stats(spmmm_product* p, uint64_t* min_col, uint64_t* max_col,
                            uint64_t* touched);
int spmmm_product_destroy(spmmm_product* p);

/* estimate_nnz (formats.py:276-289) == count_mults (perfmodel.py:63-76). */
int spmmm_estimate_nnz(spmmm_context* ctx, const spmmm_csr* a, const spmmm_csr* b,
                       uint64_t* out);
/* Inclusive prefix of per-row product counts into a host array of rows+1
 * entries (out[0] = 0): the input of product-balanced row partitioning. */
int spmmm_row_products_prefix(spmmm_context* ctx, const spmmm_csr* a, const spmmm_csr* b,
                              uint64_t* out);

/* Multi-GPU row blocks (rows of C are independent,
 * kernels.py:323-329). The product-balanced partition of A's rows into
 * `parts` (<= 64) blocks, computed on the device: bounds[g] =
 * lower_bound(P, g·T/parts) over the exclusive prefix P of per-row product
 * counts (perfmodel.py:63-76 per row), bounds[0] = 0, bounds[parts] = rows;
 * *total = T. Same result as distributed.partition_rows on the host prefix.
 * Every rank holding A and B computes the same bounds, so no collective is
 * needed to agree on them. */
int spmmm_partition_rows(spmmm_context* ctx, const spmmm_csr* a, const spmmm_csr* b, int parts,
                         uint64_t* bounds, uint64_t* total);
/* spmmm_product_download with every row pointer shifted by `offset` (the nnz
 * of the row blocks before this one): a block lands in its slice of one
 * result, row_ptr at rp + r0, columns and values at ci/v + offset. The
 * destination may be any host memory; registered (pinned) memory goes at
 * DMA speed. */
int spmmm_product_download_offset(spmmm_product* p, uint64_t offset, uint64_t* row_ptr,
                                  uint64_t* col_idx, double* values);
/* Page-lock caller memory (e.g. a shared-memory result every rank of a
 * node maps) so downloads into it run at PCIe speed; cudaHostRegister /
 * cudaHostUnregister with the portable flag. */
int spmmm_host_register(void* ptr, uint64_t bytes);
int spmmm_host_unregister(void* ptr);

/* Storage-order conversion: the product holds the CSR of M^T for the CSR view
 * M, i.e. the arrays of csr_to_csc(M) (formats.py:302-329); a CSC matrix
 * passed as the CSR view of its transpose yields csc_to_csr (formats.py:332-357).
 * Within each output slice the minor indices keep the input's major order (the
 * reference's stable scatter). Used by multiply_mixed's single conversion
 * (kernels.py:417-438); the result's device arrays can feed spmmm_multiply. */
int spmmm_transpose(spmmm_context* ctx, const spmmm_csr* m, spmmm_product** out);

/* Per-kernel timings of the last spmmm_multiply with SPMMM_FLAG_TIMING:
 * names[i] (static strings) and milliseconds ms[i], i < *count (<= cap). */
int spmmm_last_timings(spmmm_context* ctx, const char** names, double* ms, int cap, int* count);
/* Number of kernels the last spmmm_multiply launched. */
int spmmm_last_launch_count(spmmm_context* ctx, int* count);

/* Page-locked host buffers from a process-wide pool (freed blocks are kept
 * and reused by size). Downloading C into pinned memory runs at PCIe speed
 * instead of the pageable-copy rate; the Python drop-in returns CsrMatrix
 * arrays backed by these buffers. */
int spmmm_host_alloc(uint64_t bytes, void** ptr);
int spmmm_host_free(void* ptr);
/* Bytes currently held by the pool (in use + cached). */
int spmmm_host_pool_bytes(uint64_t* in_use, uint64_t* cached);

#ifdef __cplusplus
}
#endif
#endif /* SPMMM_H */
