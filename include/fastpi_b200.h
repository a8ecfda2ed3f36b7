/*
 * fastpi_b200.h -- C ABI of the B200-native FastPI core (libfastpi_b200.so).
 *
 * The reference (arXiv 2011.04235, /root/reference/pkg/src/fastpi) is a pure
 * Python package with no FFI; its drop-in boundary is its public Python API.
 * Each entry point below replaces the numerical body of one reference
 * function (cited file:line); the Python package paper_2011_04235_b200
 * mirrors the reference API on top of these calls.  INTEGRATION.md shows the
 * ctypes binding.
 *
 * Conventions
 *  - Every pointer named d_* is DEVICE memory (sm_100a, the handle's device);
 *    h_* is host memory.  Dense matrices are row-major float64 with an
 *    explicit leading dimension.  CSR: int64 indptr, int32 indices, float64
 *    values, sorted indices, no duplicates, no explicit zeros.
 *  - All work is ordered on the handle's stream (fpi_set_stream); calls that
 *    return sizes or flags to the host synchronise that stream.
 *  - Return value: FPI_OK or an error code; fpi_last_error(h) has the message.
 *    FPI_EDOMAIN -> ValueError, FPI_ECAPACITY -> CapacityError,
 *    FPI_ESTRUCT -> StructuralViolationError, FPI_ECUDA / FPI_ENUMERIC ->
 *    RuntimeError (reference validation.py:22-35).
 *  - Handles are not thread-safe; use one per host thread.
 */
#ifndef FASTPI_B200_H
#define FASTPI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPI_ABI_VERSION 1

#define FPI_OK 0
#define FPI_EDOMAIN 1
#define FPI_ECAPACITY 2
#define FPI_ESTRUCT 3
#define FPI_ECUDA 4
#define FPI_ENUMERIC 5

typedef struct fpi_context* fpi_handle;

typedef struct {
  int64_t m1, n1, m2, n2;   /* spoke rows/cols, hub rows/cols (ReorderResult, reorder.py:100-120) */
  int64_t n_iterations;     /* T */
  int64_t n_spans;          /* number of BlockSpan entries */
  int64_t n_gcc;            /* len(gcc_sizes) */
} fpi_reorder_info;

typedef struct {
  int64_t nnz_a11, nnz_a12, nnz_a21, nnz_a22;
} fpi_partition_info;

typedef struct {
  int64_t rank11;           /* sum of kept ranks over non-degenerate blocks */
  int64_t nnz_u11;          /* sum over blocks of h * keep */
  int64_t nnz_vt11;         /* sum over blocks of keep * w */
  int64_t n_blocks_svd;     /* non-degenerate blocks */
  int64_t n_blocks_large;   /* blocks routed to the Gram/eigensolver tier */
} fpi_block_plan;

typedef struct {
  int32_t engine;           /* 0 none, 1 randomized, 2 dense */
  int32_t cholqr_passes;    /* 1 or 2 */
  double cond_estimate;     /* of the sketch B (randomized engine) */
  int32_t eig_sweeps[4];    /* Jacobi sweeps used per eigensolve */
  int32_t null_completed;   /* singular vectors completed for sigma == 0 */
} fpi_svd_diag;

/* ---- handle ----------------------------------------------------------- */
int fpi_abi_version(void);
int fpi_create(fpi_handle* out, int device);
int fpi_destroy(fpi_handle h);
int fpi_set_stream(fpi_handle h, void* cuda_stream);
const char* fpi_last_error(fpi_handle h);
int64_t fpi_kernel_launches(fpi_handle h);
int fpi_get_svd_diag(fpi_handle h, fpi_svd_diag* out);

/* ---- validation.py:38-55 check_csr: sum duplicates, drop zeros, sort ---- */
/* Writes at most nnz entries into the out arrays; *h_out_nnz receives the count. */
int fpi_csr_canonicalize(fpi_handle h, int64_t m, int64_t n, int64_t nnz,
                         const int64_t* d_indptr, const int32_t* d_indices, const double* d_values,
                         int64_t* d_out_indptr, int32_t* d_out_indices, double* d_out_values,
                         int64_t* h_out_nnz);

/* CSR (p x q) -> CSR of the transpose (q x p); used for A.T / to_bipartite (reorder.py:123-134). */
int fpi_csr_transpose(fpi_handle h, int64_t p, int64_t q, int64_t nnz,
                      const int64_t* d_indptr, const int32_t* d_indices, const double* d_values,
                      int64_t* d_t_indptr, int32_t* d_t_indices, double* d_t_values);

/* ---- reorder.py:158-287 reorder (Algorithm 2) --------------------------- */
/* Bit-exact hub/spoke reordering of the bipartite graph of the m x n CSR
 * pattern.  Writes forward permutations (forward[old] = new).  Spans and
 * GCC sizes stay in the handle until fpi_reorder_fetch. */
int fpi_reorder(fpi_handle h, int64_t m, int64_t n, int64_t nnz,
                const int64_t* d_indptr, const int32_t* d_indices, double k,
                int64_t* d_row_fwd, int64_t* d_col_fwd, fpi_reorder_info* h_info);
/* d_spans: n_spans * 4 int64 (row_start, row_len, col_start, col_len); h_gcc: n_gcc int64. */
int fpi_reorder_fetch(fpi_handle h, int64_t* d_spans, int64_t* h_gcc);

/* ---- reorder.py:290-337 apply_permutation + partition ------------------- */
/* Counts entries per region and checks that every spoke-region nonzero lies
 * in a block span (StructuralViolationError otherwise). */
int fpi_partition_count(fpi_handle h, int64_t m, int64_t n, int64_t nnz,
                        const int64_t* d_indptr, const int32_t* d_indices,
                        const int64_t* d_row_fwd, const int64_t* d_col_fwd,
                        int64_t m1, int64_t n1, int64_t n_spans, const int64_t* d_spans,
                        fpi_partition_info* h_info);
/* Emits, in reordered coordinates, sorted CSR of:
 *   A11 (m1 x n1), T = [A12; A22] (m x n2), T^T (n2 x m), A21 (m2 x n1), A21^T (n1 x m2).
 * Any output pointer may be NULL to skip that part. */
int fpi_partition(fpi_handle h, int64_t m, int64_t n, int64_t nnz,
                  const int64_t* d_indptr, const int32_t* d_indices, const double* d_values,
                  const int64_t* d_row_fwd, const int64_t* d_col_fwd, int64_t m1, int64_t n1,
                  int64_t n_spans, const int64_t* d_spans,
                  int64_t* a11_ptr, int32_t* a11_idx, double* a11_val,
                  int64_t* t_ptr, int32_t* t_idx, double* t_val,
                  int64_t* tt_ptr, int32_t* tt_idx, double* tt_val,
                  int64_t* a21_ptr, int32_t* a21_idx, double* a21_val,
                  int64_t* a21t_ptr, int32_t* a21t_idx, double* a21t_val);
/* Full permuted matrix (apply_permutation, reorder.py:290-307), sorted CSR m x n. */
int fpi_permute(fpi_handle h, int64_t m, int64_t n, int64_t nnz,
                const int64_t* d_indptr, const int32_t* d_indices, const double* d_values,
                const int64_t* d_row_fwd, const int64_t* d_col_fwd,
                int64_t* d_out_indptr, int32_t* d_out_indices, double* d_out_values);

/* ---- svd.py:131-132 Gaussian sketch: numpy default_rng(seed).standard_normal((rows, cols)) ---- */
/* Bit-exact with numpy 2.x PCG64 + ziggurat; seed >= 0 (SeedSequence entropy). */
int fpi_sketch_normal(fpi_handle h, int64_t seed, int64_t rows, int64_t cols, double* d_out, int64_t ld);
/* Host helper: PCG64 state after SeedSequence(seed) seeding (hi/lo words of state and inc). */
int fpi_pcg64_seed(int64_t seed, uint64_t* h_state4 /* state_hi, state_lo, inc_hi, inc_lo */);

#ifdef __cplusplus
}
#endif
#endif /* FASTPI_B200_H */
