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
 *    FPI_ESTRUCT -> StructuralViolationError, FPI_ERETRY -> (internal) retry, FPI_ECUDA / FPI_ENUMERIC ->
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
#define FPI_ERETRY 6 /* a speculative fast path did not apply: repeat the call without it */

typedef struct fpi_context* fpi_handle;

typedef struct {
  int64_t m1, n1, m2, n2;   /* spoke rows/cols, hub rows/cols (ReorderResult, reorder.py:100-120) */
  int64_t n_iterations;     /* T */
  int64_t n_spans;          /* number of BlockSpan entries */
  int64_t n_gcc;            /* len(gcc_sizes) */
  int64_t edges_visited;    /* sum over iterations of E_t: edges with both endpoints active at entry */
  int64_t nodes_visited;    /* sum over iterations of V_t: active nodes at entry (SURVEY 8(d):
                               algorithmic bytes = 24 * edges_visited + 32 * nodes_visited) */
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
/* Dense core of the last column update's sparse block T (csrc/sparse_core.cu): h_out[0..3] =
 * core rows, core columns, entries moved to the dense panel, entries left to the SpMM; all 0
 * when the product ran as a plain SpMM (sparse.py:20-39). */
int fpi_sparse_core_info(fpi_handle h, int64_t* h_out);

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

/* ---- dense FP64 kernels (DMMA tensor path) ------------------------------ */
/* C = alpha op(A) op(B) + beta C, row-major; op(A) M x K, op(B) K x N (the `@` products of
 * svd.py:133,137 and pinv.py:81,169,206). */
int fpi_gemm(fpi_handle h, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, double alpha,
             const double* d_A, int64_t lda, const double* d_B, int64_t ldb, double beta, double* d_C, int64_t ldc);
/* Y = alpha A X + beta Y, A CSR p x q, X q x k (sparse.py:20-39 multiply / multiply_transposed on A^T). */
int fpi_spmm(fpi_handle h, int64_t p, int64_t q, int64_t k, const int64_t* d_indptr, const int32_t* d_indices,
             const double* d_values, double alpha, const double* d_X, int64_t ldx, double beta, double* d_Y,
             int64_t ldy);
/* In-place lower Cholesky factor (CholeskyQR Gram); FPI_ENUMERIC if not positive definite. */
int fpi_cholesky(fpi_handle h, int64_t n, double* d_A, int64_t lda);
/* Symmetric eigendecomposition (block Jacobi): eigenvalues descending, eigenvectors as columns. */
int fpi_sym_eig(fpi_handle h, int64_t n, const double* d_A, int64_t lda, double* d_w, double* d_V, int64_t ldv,
                int32_t* h_sweeps);

/* ---- svd.py SVD engines ------------------------------------------------- */
/* svd.py:141-193 block_diagonal_svd: sizes of the block-sparse U11 / Vt11 (CSR) */
int fpi_block_svd_plan(fpi_handle h, int64_t n_spans, const int64_t* d_spans, double alpha,
                       fpi_block_plan* h_plan);
/* U11 CSR (m1 x rank11), Vt11 CSR (rank11 x n1), sigma (rank11) from the spoke CSR A11 and its spans. */
int fpi_block_svd(fpi_handle h, int64_t m1, int64_t n1, const int64_t* a11_ptr, const int32_t* a11_idx,
                  const double* a11_val, int64_t n_spans, const int64_t* d_spans, double alpha, double* d_sigma,
                  int64_t* u_ptr, int32_t* u_idx, double* u_val, int64_t* vt_ptr, int32_t* vt_idx, double* vt_val,
                  fpi_block_plan* h_plan);
/* svd.py:86-117 dense_svd + truncate: rank leading triplets of a dense p x q matrix (sorted). */
int fpi_dense_svd(fpi_handle h, int64_t p, int64_t q, const double* d_M, int64_t ldm, int64_t rank,
                  double* d_U, double* d_sigma, double* d_Vt);
/* svd.py:120-138 randomized_svd of a CSR matrix (with its transpose): U p x rank, Vt rank x q. */
int fpi_randomized_svd(fpi_handle h, int64_t p, int64_t q, const int64_t* a_ptr, const int32_t* a_idx,
                       const double* a_val, const int64_t* at_ptr, const int32_t* at_idx, const double* at_val,
                       int64_t rank, int64_t seed, double* d_U, double* d_sigma, double* d_Vt);

/* ---- pinv.py:278-347 fastpi(): the whole factorization in one call -------------------------- */
typedef struct {
  int64_t m, n, rank;             /* rank r of the final factors */
  int64_t m1, n1, m2, n2, n_iterations, n_spans;
  int64_t rank11, s;              /* block-SVD rank and row-update rank */
  int32_t row_engine, col_engine; /* 1 randomized, 2 dense, 0 none */
  int32_t rank_clamped;           /* s < ceil(alpha n1): the pinv.py:324-328 warning */
  int32_t all_filtered;           /* every sigma below the cutoff: the pinv.py:222-224 warning */
  double tolerance_used;
  int64_t n_gcc;                  /* len(gcc_sizes) (ReorderResult.gcc_sizes) */
  int64_t edges_visited, nodes_visited; /* fpi_reorder_info's work counters */
} fpi_fastpi_info;
/* check_csr + reorder + partition + block SVD + row/column updates + pinv assembly on a CSR A (m >= n;
 * for m < n factor A^T and swap the factors, pinv.py:291-303) with FastpiConfig's fields; seed is the
 * config seed (the updates use seed + 1 and seed + 2).  The factors stay on the device, owned by the
 * handle until fpi_fastpi_release or the next fpi_fastpi: U (m x r, reordered rows), sigma (r),
 * Vt (r x n, reordered columns), sigma_dagger (r), row_fwd (m), col_fwd (n) -- the inputs of
 * fpi_pinv_apply_csr / fpi_unfold.  Errors map like every entry point (ValueError / CapacityError /
 * StructuralViolationError). */
int fpi_fastpi(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr, const int32_t* d_indices,
               const double* d_values, double alpha, double k, int64_t seed, double low_rank_threshold,
               double pinv_cutoff, fpi_fastpi_info* h_info);
int fpi_fastpi_get(fpi_handle h, const double** d_U, const double** d_sigma, const double** d_Vt,
                   const double** d_sigma_dagger, const int64_t** d_row_fwd, const int64_t** d_col_fwd);
int fpi_fastpi_release(fpi_handle h);
/* fpi_fastpi with flags: FPI_FASTPI_CANONICAL = the CSR is canonical already (sorted, no duplicates,
 * no explicit zeros -- what fpi_csr_canonicalize returns), so the check_csr copy is skipped. */
#define FPI_FASTPI_CANONICAL 1
int fpi_fastpi_ex(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr, const int32_t* d_indices,
                  const double* d_values, double alpha, double k, int64_t seed, double low_rank_threshold,
                  double pinv_cutoff, int32_t flags, fpi_fastpi_info* h_info);
/* FPI_FASTPI_DEFERRED_VALUES (with FPI_FASTPI_CANONICAL): d_values is still being uploaded when the
 * call starts.  Algorithm 2 (reorder.py:158-287) reads only the sparsity pattern, so a host caller can
 * copy the values (2/3 of a CSR's bytes) to the device on another stream meanwhile.  The solve checks
 * the pattern half of check_csr (validation.py:38-55: sorted, no duplicates) first, runs the reorder,
 * then calls the hook registered with fpi_fastpi_values_hook: it blocks until the upload has been
 * ENQUEUED and returns 0 with the cudaEvent_t recorded behind it in *event_out (the solve's stream
 * waits for that event), and the value half of the check (no explicit zeros) runs before the
 * partition (reorder.py:310-337).  A CSR that fails either half returns FPI_ERETRY before any result
 * exists: canonicalize it (fpi_csr_canonicalize) and call again without the flag.  The hook is
 * cleared by every fpi_fastpi_ex call. */
#define FPI_FASTPI_DEFERRED_VALUES 2
typedef int (*fpi_values_hook)(void* ctx, void** event_out);
int fpi_fastpi_values_hook(fpi_handle h, fpi_values_hook hook, void* ctx);
/* Ownership transfer of the last fpi_fastpi result: the caller receives the device buffers below
 * (stream-ordered allocations of the handle's device pool; free each with fpi_device_free) plus,
 * optionally, the GCC sizes (h_gcc, capacity gcc_cap >= info.n_gcc) and the device time of the five
 * stages reorder, block_svd, row_update, column_update, pinv_assembly in ms (h_stage_ms[5], pinv.py:95-98;
 * waits for the solve to finish).  The handle no longer holds a result afterwards. */
typedef struct {
  double *U, *sigma, *Vt, *sigma_dagger; /* m x r, r, r x n, r */
  int64_t *row_fwd, *col_fwd;            /* m, n */
  int64_t* spans;                        /* n_spans x 4 (BlockSpan rows) */
} fpi_fastpi_buffers;
int fpi_fastpi_take(fpi_handle h, fpi_fastpi_buffers* out, int64_t* h_gcc, int64_t gcc_cap, float* h_stage_ms);
/* Stream-ordered free (on the handle stream) of a buffer handed out by fpi_fastpi_take. */
int fpi_device_free(fpi_handle h, void* d_ptr);

/* ---- dataset text format (datasets.py:81-167), host-side native parser ---------------------- */
enum fpi_dataset_error {
  FPI_DS_OK = 0,
  FPI_DS_EMPTY,           /* empty file */
  FPI_DS_HEADER_SHAPE,    /* header is not three fields */
  FPI_DS_HEADER_INT,      /* a header field is not an integer */
  FPI_DS_HEADER_RANGE,    /* a header integer exceeds int64 */
  FPI_DS_HEADER_NEG,      /* negative header count */
  FPI_DS_LINE_COUNT,      /* instance-line count differs from m */
  FPI_DS_BAD_LABEL,       /* label token is not an integer */
  FPI_DS_LABEL_RANGE,     /* label index outside [0, L) */
  FPI_DS_LABEL_DUP,       /* repeated label in a row */
  FPI_DS_FEAT_TOKEN,      /* feature token without ':value' */
  FPI_DS_FEAT_PARSE,      /* feature index / value does not parse */
  FPI_DS_FEAT_RANGE,      /* feature index outside [0, n) */
  FPI_DS_FEAT_DUP,        /* repeated feature index */
  FPI_DS_FEAT_ORDER,      /* feature indices not increasing (tok2 = previous index) */
  FPI_DS_FEAT_NONFINITE,  /* inf / nan value */
  FPI_DS_FEAT_ZERO        /* explicit zero value */
};
typedef struct {
  int64_t m, n, L, nnz_feat, nnz_lab, n_lines;
  int32_t err_kind; /* fpi_dataset_error */
  int32_t pad_;
  int64_t err_line;              /* 1-based line of the rejection */
  int64_t tok_begin, tok_end;    /* byte span of the offending token (-1 if none) */
  int64_t tok2_begin, tok2_end;  /* second span (the previous index of FPI_DS_FEAT_ORDER) */
} fpi_dataset_info;
/* Parse a dataset file image (UTF-8 bytes).  On FPI_OK *h_out holds the parsed CSR arrays (sizes in
 * *info); on FPI_EDOMAIN the rejection is described in *info (the caller renders load_dataset's
 * ParseError message).  Host-only: no handle, no device. */
int fpi_dataset_parse(const char* buf, int64_t len, void** h_out, fpi_dataset_info* info);
/* Copy the parsed arrays out: features CSR (m+1, nnz_feat, nnz_feat), labels CSR (m+1, nnz_lab). */
int fpi_dataset_fetch(void* h, int64_t* feat_ptr, int64_t* feat_idx, double* feat_val, int64_t* lab_ptr,
                      int64_t* lab_idx);
int fpi_dataset_free(void* h);

/* ---- regression harness (regression.py:89-124) -------------------------------------------- */
/* For each row of the dense score block S (rows x L): the top-kmax labels in the reference's order
 * (score descending, ties by ascending index: np.argsort(-s, kind="stable")) and whether each is in
 * the row's label set (label CSR rows x L, sorted indices).  d_hits: rows x kmax of 0/1. */
int fpi_topk_hits(fpi_handle h, int64_t rows, int64_t L, const double* d_S, int64_t lds, const int64_t* d_lab_ptr,
                  const int32_t* d_lab_idx, int32_t kmax, uint8_t* d_hits);

/* ---- building blocks of the row-sharded randomized SVD (multi-GPU, sharded.py) ------------ */
/* C = op(A) op(A)^T (n x n, symmetric: lower tiles computed and mirrored); op(A) is n x k.
 * The Gram of svd.py:134's QR (B^T B with trans_a = 1), summed across row shards by the caller. */
int fpi_gram(fpi_handle h, int trans_a, int64_t n, int64_t k, const double* d_A, int64_t lda, double* d_C,
             int64_t ldc);
/* Linv (k x k) with Q = B Linv^T orthonormal, from G = B^T B: CholeskyQR (svd.py:134's QR without
 * forming Q) or an eigen-based factor when G is not numerically positive definite. */
int fpi_orth_factor(fpi_handle h, int64_t k, const double* d_G, double* d_Linv, double* h_cond);
/* A[i, :] *= scale[i] (the diag(sigma) factors of pinv.py:133,194). */
int fpi_scale_rows(fpi_handle h, int64_t rows, int64_t cols, double* d_A, int64_t lda, const double* d_scale);
/* Sign rule applied by every SVD of the library: the largest-|.| entry of each row of Vt is made
 * positive, U's columns flipped to match (U may be a row shard: the sign depends on Vt only). */
int fpi_canonical_signs(fpi_handle h, int64_t r, int64_t p, int64_t q, double* d_U, int64_t ldu, double* d_Vt,
                        int64_t ldv);
/* At = A^T (A rows x cols). */
int fpi_transpose(fpi_handle h, int64_t rows, int64_t cols, const double* d_A, int64_t lda, double* d_At,
                  int64_t ldat);

/* ---- pinv.py FastPI stages ---------------------------------------------- */
/* pinv.py:131-171 row_update: f11 = (sigma11, U11 CSR m1 x rank11, Vt11 CSR rank11 x n1), A21 CSR m2 x n1.
 * Outputs U (m1+m2) x s, sigma s, Vt s x n1; *h_engine = 1 randomized / 2 dense. */
int fpi_row_update(fpi_handle h, int64_t m1, int64_t n1, int64_t rank11, const double* sigma11,
                   const int64_t* u_ptr, const int32_t* u_idx, const double* u_val,
                   const int64_t* v_ptr, const int32_t* v_idx, const double* v_val,
                   int64_t m2, const int64_t* a_ptr, const int32_t* a_idx, const double* a_val,
                   int64_t s, double low_rank_threshold, int64_t seed,
                   double* d_U, double* d_sigma, double* d_Vt, int32_t* h_engine);
/* pinv.py:174-208 column_update: f = (U m x s_prev, sigma, Vt s_prev x n1), T = [A12; A22] CSR m x n2 (+ T^T).
 * Outputs U m x r, sigma r, Vt r x (n1 + n2). */
int fpi_column_update(fpi_handle h, int64_t m, int64_t s_prev, int64_t n1, const double* U_prev,
                      const double* sigma_prev, const double* Vt_prev, int64_t n2,
                      const int64_t* t_ptr, const int32_t* t_idx, const double* t_val,
                      const int64_t* tt_ptr, const int32_t* tt_idx, const double* tt_val,
                      int64_t r, double low_rank_threshold, int64_t seed,
                      double* d_U, double* d_sigma, double* d_Vt, int32_t* h_engine);
/* pinv.py:211-231 pinv_from_svd: sigma_dagger = 1/sigma where sigma > cutoff*smax*max(p,q,1). */
int fpi_pinv_assemble(fpi_handle h, int64_t r, const double* d_sigma, int64_t p, int64_t q, double cutoff,
                      double* d_sigma_dagger, double* h_tol, int32_t* h_all_filtered);
/* pinv.py:271-275 + 226-228: V = Vt[:, col_fwd]^T (n x r), Ut = U[row_fwd, :]^T (r x m); either may be NULL. */
int fpi_unfold(fpi_handle h, int64_t m, int64_t n, int64_t r, const double* d_U, const double* d_Vt,
               const int64_t* d_row_fwd, const int64_t* d_col_fwd, double* d_V_out, double* d_Ut_out);
/* pinv.py:72-81 Pseudoinverse.apply / regression.py:50-70 fit: Z (n x L) = V diag(sdag) Ut Y with the factors
 * in reordered coordinates (U m x r, Vt r x n) and the row/column permutations; Y CSR m x L. */
int fpi_pinv_apply_csr(fpi_handle h, int64_t m, int64_t n, int64_t r, const double* d_U,
                       const double* d_sigma_dagger, const double* d_Vt, const int64_t* d_row_fwd,
                       const int64_t* d_col_fwd, int64_t L, int64_t nnz, const int64_t* y_ptr,
                       const int32_t* y_idx, const double* y_val, double* d_Z);
/* fpi_pinv_apply_csr with Z written to HOST memory h_Z (n x L, page-locked for overlap): the lift
 * runs in row chunks whose device->host copies overlap the next chunk's GEMM; returns when h_Z is
 * complete.  Replaces the pinv.py:72-81 apply + the host copy of its result. */
int fpi_pinv_apply_csr_host(fpi_handle h, int64_t m, int64_t n, int64_t r, const double* d_U,
                            const double* d_sigma_dagger, const double* d_Vt, const int64_t* d_row_fwd,
                            const int64_t* d_col_fwd, int64_t L, int64_t nnz, const int64_t* y_ptr,
                            const int32_t* y_idx, const double* y_val, double* h_Z);
/* One row shard of pinv.py:75's U^T Y: W (L x r) = sum over the rows of Y whose reordered index lies
 * in [r0, r0 + m_loc) of Y[i, :]^T U_loc[row_fwd[i] - r0, :]; the shards' W sum to the full product
 * (the multi-GPU all-reduce operand).  Y is CSR (m x L) in original row order. */
int fpi_pinv_project_csr(fpi_handle h, int64_t r0, int64_t m_loc, int64_t r, const double* d_U_loc,
                         const int64_t* d_row_fwd, int64_t m, int64_t L, int64_t nnz, const int64_t* y_ptr,
                         const int32_t* y_idx, const double* y_val, double* d_W);
/* pinv.py:81's lift: Z (n x L, original column order) = V diag(sigma+) W^T; W is scaled in place. */
int fpi_pinv_lift(fpi_handle h, int64_t n, int64_t r, const double* d_sigma_dagger, const double* d_Vt,
                  const int64_t* d_col_fwd, int64_t L, double* d_W, double* d_Z);
/* Dense right-hand side variant (Y m x L row-major). */
int fpi_pinv_apply_dense(fpi_handle h, int64_t m, int64_t n, int64_t r, const double* d_U,
                         const double* d_sigma_dagger, const double* d_Vt, const int64_t* d_row_fwd,
                         const int64_t* d_col_fwd, int64_t L, const double* d_Y, int64_t ldy, double* d_Z);

/* ---- measurement (bench.py) ---------------------------------------------- */
/* Record CUDA events around every kernel class launched on this handle. */
int fpi_timing_enable(fpi_handle h, int on);
/* "name\tlaunches\tms\tflops\tbytes\n" per kernel class (algorithmic flops / bytes). */
int fpi_timing_report(fpi_handle h, char* h_buf, int64_t cap, int reset);
/* FP64 tensor-pipe (DMMA) issue-rate peak of this GPU, TFLOP/s. */
int fpi_dmma_peak(fpi_handle h, double* h_tflops);

/* ---- sharded solve over several GPUs; csrc/comm.cu, csrc/sharded.cu --------------
 * One process (and handle) per GPU.  The handle owns the communicator; the exchanges are
 * stream-ordered NCCL calls (NVLink / NVSwitch) on the handle's stream. */
/* Exchange callback (host): op 0 all-reduce sum in place (send == recv), 1 all-reduce max,
 * 2 all-gather (recv holds world * count), 3 reduce to root.  Device pointers; the library has
 * synchronised its stream; return 0 once recv is written. */
typedef int (*fpi_comm_fn)(void* user, int op, const void* d_send, void* d_recv, int64_t count, int root);
/* A fresh NCCL unique id (128 bytes) for rank 0 to share with the other ranks out of band. */
int fpi_comm_nccl_id(char* h_out128, char* h_err, int64_t err_cap);
/* NCCL communicator of `world` ranks on this handle (libnccl.so.2 loaded at run time). */
int fpi_comm_init_nccl(fpi_handle h, const char* h_id128, int rank, int world);
/* Host-callback communicator (e.g. torch.distributed over gloo: several ranks on one GPU). */
int fpi_comm_init_callback(fpi_handle h, int rank, int world, fpi_comm_fn fn, void* user);
/* World of one (every exchange is the identity). */
int fpi_comm_init_self(fpi_handle h);
int fpi_comm_free(fpi_handle h);
int fpi_comm_info(fpi_handle h, int* h_rank, int* h_world);
/* In-place sum of n doubles over the ranks. */
int fpi_comm_allreduce(fpi_handle h, double* d_buf, int64_t n);
/* Ownership table h_out[world][10]: b_lo, b_hi (A11 block range), r_lo, r_hi (spoke rows), c_lo,
 * c_hi (spoke columns), h_lo, h_hi (hub rows within [0, m2)), hc_lo, hc_hi (hub columns within
 * [0, n2)); block ranges balanced by rows' work (8 + T row nnz), columns and h w min(h, w). */
int fpi_shard_plan(fpi_handle h, int64_t m, int64_t m1, int64_t n1, int64_t n2, int64_t n_spans,
                   const int64_t* d_spans, const int64_t* d_t_ptr, int world, int64_t* h_out);
/* svd.py:141-193 for the blocks [b_lo, b_hi) only (structure complete, other values zero);
 * h_keep_range[2] = the kept-rank range [k_lo, k_hi) of those blocks. */
int fpi_block_svd_range(fpi_handle h, int64_t m1, int64_t n1, const int64_t* a11_ptr, const int32_t* a11_idx,
                        const double* a11_val, int64_t n_spans, const int64_t* d_spans, double alpha, int64_t b_lo,
                        int64_t b_hi, double* d_sigma, int64_t* u_ptr, int32_t* u_idx, double* u_val,
                        int64_t* vt_ptr, int32_t* vt_idx, double* vt_val, fpi_block_plan* h_plan,
                        int64_t* h_keep_range);
/* pinv.py:131-171 on this rank's rows of [Sigma Vt11 ; A21] (kept rows [k_lo, k_lo + k_loc), U11 rows
 * [r_lo, r_lo + r_rows), A21 rows [h_lo, h_lo + m2_loc); global CSRs).  Z = inner^T B is reduced onto
 * the owners of the column ranges h_zoff[world + 1].  Out: U_loc ((r_rows + m2_loc) x s), sigma (s),
 * Vt_loc (s x own columns).  Randomized engine only. */
int fpi_row_update_shard(fpi_handle h, int64_t n1, const double* d_sigma11, const int64_t* vt_ptr,
                         const int32_t* vt_idx, const double* vt_val, int64_t k_lo, int64_t k_loc,
                         const int64_t* u_ptr, const int32_t* u_idx, const double* u_val, int64_t r_lo, int64_t r_rows,
                         const int64_t* a_ptr, const int32_t* a_idx, const double* a_val, int64_t h_lo,
                         int64_t m2_loc, int64_t p_global, int64_t s_rank, double thr, int64_t seed,
                         const int64_t* h_zoff, double* d_U, double* d_sigma, double* d_Vt);
/* pinv.py:174-208 on this rank's m_loc rows of [U Sigma | T] (T_loc and its transpose), its columns
 * of the previous Vt (s_prev x nc_loc) and its hub columns [hc_lo, hc_hi).  Out: U (m_loc x r),
 * sigma (r), Vt_loc (r x (nc_loc + hc_hi - hc_lo)).  Randomized engine only. */
int fpi_column_update_shard(fpi_handle h, int64_t m_loc, int64_t s_prev, const double* d_U_prev,
                            const double* d_sigma_prev, const double* d_Vt_prev, int64_t nc_loc, int64_t n2,
                            const int64_t* t_ptr, const int32_t* t_idx, const double* t_val, const int64_t* tt_ptr,
                            const int32_t* tt_idx, const double* tt_val, int64_t m_global, int64_t hc_lo,
                            int64_t hc_hi, int64_t r, double thr, int64_t seed, double* d_U, double* d_sigma,
                            double* d_Vt);
/* pinv.py:72-81 on this rank: W = sum over ranks of Y_i^T U_loc (all-reduce), then the rows of Z of
 * its columns, Z_loc (n_loc x L) = Vt_loc^T diag(sigma+) W^T.  Its rows are [r_lo, r_hi) then
 * [m1 + h_lo, m1 + h_hi) in reordered coordinates. */
int fpi_pinv_apply_shard(fpi_handle h, int64_t m, int64_t m1, int64_t r_lo, int64_t r_hi, int64_t h_lo,
                         int64_t h_hi, int64_t r, const double* d_U_loc, const double* d_sdag, const double* d_Vt_loc,
                         int64_t n_loc, const int64_t* d_row_fwd, int64_t L, int64_t nnz, const int64_t* y_ptr,
                         const int32_t* y_idx, const double* y_val, double* d_Z_loc);

#ifdef __cplusplus
}
#endif
#endif /* FASTPI_B200_H */
