/*
 * spmmm_mtx.h — Matrix Market coordinate I/O in libspmmm.so (host only,
 * multi-threaded). Replaces the reference's mtxio.py (save_matrix_market
 * :16-26, load_matrix_market :29-72) for the "matrix coordinate real general"
 * format: same acceptance rules (any entry order, '%' comments and blank
 * lines skipped) and the same ValueError cases (status SPMMM_ERR_INVALID)
 * with the reference's messages: unsupported header, missing / malformed size
 * line, entry outside the shape, entry count differing from the size line,
 * duplicate positions. The writer emits row-major order with "%.17g" values,
 * which round-trips every double exactly.
 */
#ifndef SPMMM_MTX_H
#define SPMMM_MTX_H

#include <stdint.h>

#include "spmmm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct spmmm_mtx spmmm_mtx;

/* Message of the last failing spmmm_mtx_* call on this thread. */
const char* spmmm_mtx_last_error(void);
/* Write a host CSR view to `path` (mtxio.py:16-26). */
int spmmm_mtx_write(const char* path, const spmmm_csr* m);
/* Parse `path` into a CSR held by the returned handle (mtxio.py:29-72). */
int spmmm_mtx_read(const char* path, spmmm_mtx** out);
int spmmm_mtx_shape(const spmmm_mtx* m, uint64_t* rows, uint64_t* cols, uint64_t* nnz);
/* Copy the CSR arrays into caller buffers of rows+1, nnz, nnz entries. */
int spmmm_mtx_copy(const spmmm_mtx* m, uint64_t* row_ptr, uint64_t* col_idx, double* values);
int spmmm_mtx_free(spmmm_mtx* m);

#ifdef __cplusplus
}
#endif
#endif /* SPMMM_MTX_H */
