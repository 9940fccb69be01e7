/*
 * spmmm_gen.h — seeded operand generators for the spMMM benchmark configs.
 *
 * Host-side C ABI exported by libspmmm.so. These are NOT on the hot path; they
 * produce the synthetic operands (BASELINE.json configs C1–C5) fast enough that
 * bench.py and the parity tests can build 2M-row matrices in well under a
 * second. All generators write plain CSR arrays (uint64 row_ptr/col_idx,
 * float64 values) into caller-owned buffers.
 *
 * Bit-identity contracts (pinned in tests/test_genmat.py against fingerprints
 * produced by the reference package itself):
 *   spmmm_splitmix64          == sparsemm.genmat.SplitMix64.next_u64   (genmat.py:28-39)
 *   spmmm_gen_fd              == sparsemm.genmat.gen_fd                (genmat.py:79-103)
 *   spmmm_gen_random_k        == sparsemm.genmat.gen_random_k          (genmat.py:106-130)
 * New generators (the reference has none for these configs):
 *   spmmm_gen_fd3             27-point stencil on a grid^3 cube (config C4)
 *   spmmm_gen_zipf            Zipf(s) row lengths clipped to [1, lmax]  (config C5)
 */
#ifndef SPMMM_GEN_H
#define SPMMM_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Writes n consecutive outputs of a splitmix64 stream seeded with `seed`. */
int spmmm_splitmix64(uint64_t seed, uint64_t n, uint64_t* out);

/* 5-point Laplacian on a grid x grid square: rows = grid^2, nnz = 5g^2 - 4g. */
int spmmm_gen_fd_size(uint64_t grid, uint64_t* rows, uint64_t* nnz);
int spmmm_gen_fd(uint64_t grid, uint64_t* row_ptr, uint64_t* col_idx, double* values);

/* 27-point stencil on a grid^3 cube, row i = x + g*y + g^2*z, diagonal 26, off -1. */
int spmmm_gen_fd3_size(uint64_t grid, uint64_t* rows, uint64_t* nnz);
int spmmm_gen_fd3(uint64_t grid, uint64_t* row_ptr, uint64_t* col_idx, double* values);

/* Device-side versions of the two stencil generators (gen_device.cu): the
 * same bytes written straight into caller-owned DEVICE arrays (sizes from the
 * *_size calls) on `stream` (a cudaStream_t, may be NULL); returns after the
 * stream has finished them. 0 ok, 2 invalid argument, 3 CUDA error. The
 * random families stay on the host: each is one sequential splitmix64 stream
 * whose draws shift with every rejected duplicate (genmat.py:106-130). */
int spmmm_gen_fd_device(uint64_t grid, uint64_t* row_ptr, uint64_t* col_idx, double* values,
                        void* stream);
int spmmm_gen_fd3_device(uint64_t grid, uint64_t* row_ptr, uint64_t* col_idx, double* values,
                         void* stream);

/* n x n, exactly k distinct uniform columns per row, values in (0,1]; nnz = n*k. */
int spmmm_gen_random_k(uint64_t n, uint64_t k, uint64_t seed,
                       uint64_t* row_ptr, uint64_t* col_idx, double* values);

/* n x n, row length L = min(Zipf(s), lmax) drawn by inverse CDF, L distinct
 * uniform columns (rejection), values uniform in [-1, 1). Two calls: the first
 * (arrays NULL) only reports nnz; the second fills the arrays. */
int spmmm_gen_zipf(uint64_t n, double s, uint64_t lmax, uint64_t seed, uint64_t* nnz,
                   uint64_t* row_ptr, uint64_t* col_idx, double* values);

#ifdef __cplusplus
}
#endif
#endif /* SPMMM_GEN_H */
