/* libb200sp -- C ABI of the B200-native SpMV + Krylov hot path.
 *
 * This is the drop-in boundary for the reference's executor/operation plugin
 * point: the reference dispatches every numeric operation through
 *     Executor.run(op) -> _dispatch -> op.<kind>(exc)     (src/executor.py:123-154)
 * and a new backend is "a new Executor subclass plus a per-kernel Operation
 * variant". Each function below is the body of one such
 * `Operation.cuda` variant; the reference kernel it replaces is cited beside
 * it (paths relative to /root/reference/pkg/src/opalg/).
 *
 * Conventions
 *   - every pointer is a DEVICE pointer owned by the caller (borrowed for the
 *     call only, = `lend`, src/ownership.py:75-78); nothing is freed here;
 *   - sizes are int64_t, matrix indices int32_t (DEFAULT_INDEX_DTYPE,
 *     src/config.py:22), values double (_f64) or float (_f32);
 *   - `stream` is a cudaStream_t passed as void*; launches are asynchronous
 *     and stream-ordered, callers synchronise before any host read
 *     (Executor.run is observably synchronous);
 *   - return 0 (B200SP_OK) or a B200SP_E* code; b200sp_last_error() returns
 *     the thread-local message. Codes map to src/errors.py classes.
 *   - SpMV semantics, one right-hand-side column per call:
 *         x[i] = alpha * (A b)[i] + beta * x_in[i]     (x_in == NULL -> 0)
 *     alpha/beta are the host values unless the *_dev pointer is non-NULL.
 *     Strides are row strides (elements) of the (n, m) row-major Dense.
 */
#ifndef B200SP_H
#define B200SP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B200SP_ABI_VERSION 1

#define B200SP_OK 0
#define B200SP_EINVAL 1      /* ParameterError / DimensionMismatch */
#define B200SP_ECUDA 2       /* OpalgError (CUDA runtime failure)   */
#define B200SP_ESINGULAR 3   /* Singular (src/errors.py:36-37)      */
#define B200SP_EUNSUPPORTED 4 /* Unsupported (src/errors.py:18-19)  */

/* ---- runtime ---------------------------------------------------------- */
const char* b200sp_last_error(void);
long long b200sp_launch_count(void);
int b200sp_version(void);
int b200sp_device_sync(void);
/* Thread-local launch guard: SpMV / fix-up kernels launched by this host
 * thread while a guard is set return immediately when *guard != 0 (device
 * flag). Solvers set it to their "done" flag around CUDA-graph batches. */
void b200sp_set_guard(const int32_t* guard);
/* Tuning knob for benchmark sweeps (kernel variant / launch shape by name);
 * unset knobs keep the measured-best defaults. Not thread-safe against
 * concurrent set calls; not needed for correct results. */
/* b200sp_set_tuning(key, B200SP_TUNING_DEFAULT) restores a knob's built-in default */
#define B200SP_TUNING_DEFAULT (-2147483647 - 1)
int b200sp_set_tuning(const char* key, int32_t value);
int64_t b200sp_reduce_workspace_elems(void);
int64_t b200sp_scan_workspace_elems(int64_t count);
int b200sp_exclusive_scan_i32(int64_t count, const int32_t* in, int32_t* out, long long* ws, void* stream);
int b200sp_exclusive_scan_i64(int64_t count, const int32_t* in, int64_t* out, long long* ws, void* stream);
int b200sp_reduce_max_i32(int64_t count, const int32_t* in, int32_t* out, void* stream);

/* ---- BLAS-1 on Dense (n, m) blocks -------------------------------------
 * replaces CopyKernel/FillKernel/ScaleKernel/AddScaledKernel (kernels.py:30-99)
 * and DotKernel/Norm2Kernel (kernels.py:102-137). alpha_dev: (1, m) scalars. */
int b200sp_fill_f64(int64_t n, int32_t m, double* x, int64_t xs, double value, void* stream);
int b200sp_fill_f32(int64_t n, int32_t m, float* x, int64_t xs, float value, void* stream);
int b200sp_copy_f64(int64_t n, int32_t m, const double* s, int64_t ss, double* d, int64_t ds, void* stream);
int b200sp_copy_f32(int64_t n, int32_t m, const float* s, int64_t ss, float* d, int64_t ds, void* stream);
int b200sp_scale_f64(int64_t n, int32_t m, double alpha, const double* alpha_dev, double* x, int64_t xs, void* stream);
int b200sp_scale_f32(int64_t n, int32_t m, float alpha, const float* alpha_dev, float* x, int64_t xs, void* stream);
int b200sp_add_scaled_f64(int64_t n, int32_t m, double alpha, const double* alpha_dev, const double* x, int64_t xs,
                          double* y, int64_t ys, void* stream);
int b200sp_add_scaled_f32(int64_t n, int32_t m, float alpha, const float* alpha_dev, const float* x, int64_t xs,
                          float* y, int64_t ys, void* stream);
/* partials: b200sp_reduce_workspace_elems() values; counter: one zeroed uint32 */
int b200sp_dot_f64(int64_t n, int32_t m, const double* x, int64_t xs, const double* y, int64_t ys, double* out,
                   double* partials, uint32_t* counter, void* stream);
int b200sp_dot_f32(int64_t n, int32_t m, const float* x, int64_t xs, const float* y, int64_t ys, float* out,
                   float* partials, uint32_t* counter, void* stream);
int b200sp_norm2_f64(int64_t n, int32_t m, const double* x, int64_t xs, double* out, double* partials,
                     uint32_t* counter, void* stream);
int b200sp_norm2_f32(int64_t n, int32_t m, const float* x, int64_t xs, float* out, float* partials,
                     uint32_t* counter, void* stream);

/* ---- SpMV ---------------------------------------------------------------- */
/* Csr, classical strategy (sub-warp of `subwarp` lanes per row);
 * replaces CsrSpmvKernel + csr_row_sums (kernels.py:278-316).
 * `subwarp` may be OR-ed with B200SP_SUBWARP_EVEN_NNZ when the matrix has an
 * even number of entries: the kernel may then read entries in aligned pairs
 * (16-byte aligned col_idxs / vals; a pair never extends past entry nnz - 1). */
#define B200SP_SUBWARP_EVEN_NNZ 0x100
int b200sp_csr_spmv_classical_f64(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const double* vals,
                                  const double* b, int64_t b_stride, double* x, int64_t x_stride, double alpha,
                                  const double* alpha_dev, double beta, const double* beta_dev, const double* x_in,
                                  int64_t x_in_stride, int32_t subwarp, void* stream);
int b200sp_csr_spmv_classical_f32(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const float* vals,
                                  const float* b, int64_t b_stride, float* x, int64_t x_stride, float alpha,
                                  const float* alpha_dev, float beta, const float* beta_dev, const float* x_in,
                                  int64_t x_in_stride, int32_t subwarp, void* stream);
/* Csr, stream strategy: a CTA of 256 threads owns (256 / tpr) * rpt
 * consecutive rows ((tpr, rpt) in {(1,1), (2,1), (4,1), (1,2), (1,4), (1,8)});
 * their nonzeros are staged through shared memory with 128-bit loads
 * (col_idxs / vals 16-byte aligned) in chunks of chunk_cap entries (multiple
 * of 4, at most b200sp_csr_stream_capacity(); rows_per_CTA * longest_row + 4
 * keeps a block in one chunk). Same result contract as csr_row_sums
 * (kernels.py:304-316). */
int b200sp_csr_spmv_stream_f64(int64_t n, int64_t nnz, const int32_t* row_ptrs, const int32_t* col_idxs,
                               const double* vals, const double* b, int64_t b_stride, double* x, int64_t x_stride,
                               double alpha, const double* alpha_dev, double beta, const double* beta_dev,
                               const double* x_in, int64_t x_in_stride, int32_t chunk_cap, int32_t tpr,
                               int32_t rpt, int32_t gather_in_reduce, void* stream);
int b200sp_csr_spmv_stream_f32(int64_t n, int64_t nnz, const int32_t* row_ptrs, const int32_t* col_idxs,
                               const float* vals, const float* b, int64_t b_stride, float* x, int64_t x_stride,
                               float alpha, const float* alpha_dev, float beta, const float* beta_dev,
                               const float* x_in, int64_t x_in_stride, int32_t chunk_cap, int32_t tpr,
                               int32_t rpt, int32_t gather_in_reduce, void* stream);
int32_t b200sp_csr_stream_capacity(int32_t value_bytes);
/* Csr, stream strategy as a persistent TMA pipeline ("pipe"): one or two CTAs per SM
 * of `consumers` (256/512) consumer threads + 1 producer warp; tiles of
 * consumers/tpr*rpt rows, each row reduced by `tpr` (1/2/4) threads; each
 * tile's row_ptrs slice and col_idxs / vals range is bulk-copied
 * (cp.async.bulk + mbarrier) into a `stages`-deep ring of shared-memory
 * stages of `cap` entries (multiple of 4) and reduced out of shared memory.
 * Supported (consumers, tpr, rpt): (256,1,1|2|4) (256,2,1|2) (512,2,1|2) (512,4,1|2).
 * Two CTAs per SM run when 2 x stages x stage bytes fits (tuning "pipe_ctas").
 * stages * b200sp_csr_tma_stage_bytes(rows per tile) + 256 <= 226 KB. row_ptrs/col_idxs/vals 16-byte aligned. Replaces
 * the same CsrSpmvKernel as the other Csr strategies (src/kernels.py:278-316). */
int b200sp_csr_spmv_tma_f64(int64_t n, int64_t nnz, const int32_t* row_ptrs, const int32_t* col_idxs,
                            const double* vals, const double* b, int64_t b_stride, double* x, int64_t x_stride,
                            double alpha, const double* alpha_dev, double beta, const double* beta_dev,
                            const double* x_in, int64_t x_in_stride, int32_t cap, int32_t rpt, int32_t stages,
                            int32_t consumers, int32_t tpr, void* stream);
int b200sp_csr_spmv_tma_f32(int64_t n, int64_t nnz, const int32_t* row_ptrs, const int32_t* col_idxs,
                            const float* vals, const float* b, int64_t b_stride, float* x, int64_t x_stride,
                            float alpha, const float* alpha_dev, float beta, const float* beta_dev,
                            const float* x_in, int64_t x_in_stride, int32_t cap, int32_t rpt, int32_t stages,
                            int32_t consumers, int32_t tpr, void* stream);
int64_t b200sp_csr_tma_stage_bytes(int32_t value_bytes, int32_t rows_per_tile, int32_t cap);
/* Csr, load-balanced strategy: merge-path tiles of `tile` merge items (rows +
 * nonzeros) with a deterministic carry fix-up. mode 2: the tile's rows
 * reduced sub-warp-per-row from global memory, long rows and the carried-out
 * row by the whole CTA. Plan once per matrix: tile = b200sp_csr_lb_tile(vb,
 * mode), coords = 2*(num_tiles+1) int32; workspace carry_row / carry_val
 * num_tiles each. mode 3 ("nnz split", skewed rows): warp chunks of
 * tile = b200sp_csr_lb_tile(vb, 3) nonzeros reduced like Coo, rows derived
 * from row_ptrs; coords = the chunk start rows from b200sp_csr_seg_plan
 * (nchunks + 1 int32, nchunks = ceil(nnz / tile)), carry_row = nchunks int32
 * (chunk tail rows), carry_val = 2 * nchunks values. */
int32_t b200sp_csr_lb_tile(int32_t value_bytes, int32_t mode);
int b200sp_csr_seg_plan(int64_t n, int64_t nnz, const int32_t* row_ptrs, int32_t* chunk_rows, void* stream);
int64_t b200sp_csr_lb_num_tiles(int64_t n, int64_t nnz, int32_t tile);
int b200sp_csr_lb_plan(int64_t n, int64_t nnz, const int32_t* row_ptrs, int32_t tile, int32_t* coords,
                       void* stream);
int b200sp_csr_spmv_lb_f64(int64_t n, int64_t nnz, const int32_t* row_ptrs, const int32_t* col_idxs,
                           const double* vals, const double* b, int64_t b_stride, double* x, int64_t x_stride,
                           double alpha, const double* alpha_dev, double beta, const double* beta_dev,
                           const double* x_in, int64_t x_in_stride, const int32_t* coords, int32_t* carry_row,
                           double* carry_val, int32_t tile, int32_t mode, void* stream);
int b200sp_csr_spmv_lb_f32(int64_t n, int64_t nnz, const int32_t* row_ptrs, const int32_t* col_idxs,
                           const float* vals, const float* b, int64_t b_stride, float* x, int64_t x_stride,
                           float alpha, const float* alpha_dev, float beta, const float* beta_dev,
                           const float* x_in, int64_t x_in_stride, const int32_t* coords, int32_t* carry_row,
                           float* carry_val, int32_t tile, int32_t mode, void* stream);
/* Coo (entries sorted by row); replaces CooSpmvKernel / CooAdvSpmvKernel /
 * CooResidualKernel (kernels.py:163-275). Rows with no entry are NOT written:
 * the caller prefills them with b200sp_rows_scale_*. carry_head/carry_tail:
 * ceil(nnz/chunk) values each; chunk_rows (optional, NULL allowed): 2 *
 * ceil(nnz/chunk) int32, 8-byte aligned -- the kernel records each chunk's
 * first / last row there so the carry fix-up reads them contiguously. */
int b200sp_coo_spmv_f64(int64_t nnz, int32_t chunk, const int32_t* row_idxs, const int32_t* col_idxs,
                        const double* vals, const double* b, int64_t b_stride, double* x, int64_t x_stride,
                        double alpha, const double* alpha_dev, double beta, const double* beta_dev,
                        const double* x_in, int64_t x_in_stride, double* carry_head, double* carry_tail, int32_t* chunk_rows,
                        void* stream);
int b200sp_coo_spmv_f32(int64_t nnz, int32_t chunk, const int32_t* row_idxs, const int32_t* col_idxs,
                        const float* vals, const float* b, int64_t b_stride, float* x, int64_t x_stride, float alpha,
                        const float* alpha_dev, float beta, const float* beta_dev, const float* x_in,
                        int64_t x_in_stride, float* carry_head, float* carry_tail, int32_t* chunk_rows, void* stream);
int b200sp_rows_scale_f64(int64_t count, const int32_t* rows, double* x, int64_t x_stride, double beta,
                          const double* beta_dev, const double* x_in, int64_t x_in_stride, void* stream);
int b200sp_rows_scale_f32(int64_t count, const int32_t* rows, float* x, int64_t x_stride, float beta,
                          const float* beta_dev, const float* x_in, int64_t x_in_stride, void* stream);
/* Ell (column-major, padding col = -1); no reference kernel */
int b200sp_ell_spmv_f64(int64_t n, int64_t width, int64_t stride, const int32_t* col_idxs, const double* vals,
                        const double* b, int64_t b_stride, double* x, int64_t x_stride, double alpha,
                        const double* alpha_dev, double beta, const double* beta_dev, const double* x_in,
                        int64_t x_in_stride, void* stream);
int b200sp_ell_spmv_f32(int64_t n, int64_t width, int64_t stride, const int32_t* col_idxs, const float* vals,
                        const float* b, int64_t b_stride, float* x, int64_t x_stride, float alpha,
                        const float* alpha_dev, float beta, const float* beta_dev, const float* x_in,
                        int64_t x_in_stride, void* stream);
/* Sellp (slice_size rows per slice); no reference kernel */
int b200sp_sellp_spmv_f64(int64_t n, int32_t slice_size, const int32_t* slice_lengths, const int32_t* slice_sets,
                          const int32_t* col_idxs, const double* vals, const double* b, int64_t b_stride, double* x,
                          int64_t x_stride, double alpha, const double* alpha_dev, double beta,
                          const double* beta_dev, const double* x_in, int64_t x_in_stride, void* stream);
int b200sp_sellp_spmv_f32(int64_t n, int32_t slice_size, const int32_t* slice_lengths, const int32_t* slice_sets,
                          const int32_t* col_idxs, const float* vals, const float* b, int64_t b_stride, float* x,
                          int64_t x_stride, float alpha, const float* alpha_dev, float beta, const float* beta_dev,
                          const float* x_in, int64_t x_in_stride, void* stream);

/* Dense operator times one column (DenseSpmvKernel, kernels.py:319-332) */
/* matrix-free tridiagonal stencil x = tridiag(l, c, r) b on (n, m) row-major
 * blocks (StencilMatrix; StencilApplyKernel, src/kernels.py:335-363) */
int b200sp_stencil3_apply_f64(int64_t n, int32_t m, double l, double c, double r, const double* b, int64_t bs,
                              double* x, int64_t xs, void* stream);
int b200sp_stencil3_apply_f32(int64_t n, int32_t m, float l, float c, float r, const float* b, int64_t bs,
                              float* x, int64_t xs, void* stream);
int b200sp_dense_spmv_f64(int64_t n, int64_t k, const double* a, int64_t a_stride, const double* b, int64_t b_stride,
                         double* x, int64_t x_stride, void* stream);
int b200sp_dense_spmv_f32(int64_t n, int64_t k, const float* a, int64_t a_stride, const float* b, int64_t b_stride,
                         float* x, int64_t x_stride, void* stream);

/* ---- conversions (Csr hub); replaces convert/from_data/to_data
 * (formats.py:40-53, :196-221, :301-329) for the device formats ------------ */
int b200sp_csr_row_lengths(int64_t n, const int32_t* row_ptrs, int32_t* len, void* stream);
int b200sp_csr_to_coo_rows(int64_t n, const int32_t* row_ptrs, int32_t* row_idxs, void* stream);
int b200sp_coo_to_csr_ptrs(int64_t nnz, int64_t n, const int32_t* row_idxs, int32_t* row_ptrs, void* stream);
int b200sp_sellp_slice_lengths(int64_t n, const int32_t* row_ptrs, int32_t slice_size, int32_t stride_factor,
                               int32_t* slice_lengths, void* stream);
int b200sp_hybrid_overflow_counts(int64_t n, const int32_t* row_ptrs, int32_t width, int32_t* counts, void* stream);
int b200sp_ell_row_lengths(int64_t n, int64_t width, int64_t stride, const int32_t* col_idxs, int32_t* len,
                           void* stream);
int b200sp_sellp_row_lengths(int64_t n, int32_t slice_size, const int32_t* slice_lengths, const int32_t* slice_sets,
                             const int32_t* col_idxs, int32_t* len, void* stream);
int b200sp_add_csr_lengths(int64_t n, const int32_t* row_ptrs2, int32_t* len, void* stream);
int b200sp_length_histogram(int64_t n, const int32_t* row_ptrs, int32_t nbins, unsigned long long* hist,
                            void* stream);
int b200sp_empty_row_flags(int64_t n, const int32_t* row_ptrs, int32_t* flag, void* stream);
int b200sp_compact_flags(int64_t n, const int32_t* flag, const int32_t* pos, int32_t* out, void* stream);
#define B200SP_CONVERT_DECL(T, SUF)                                                                              \
    int b200sp_csr_to_ell_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, int64_t width,      \
                                int64_t stride, int32_t* ell_ci, T* ell_v, void* stream);                        \
    int b200sp_csr_to_sellp_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, int32_t slice_size, \
                                  const int32_t* slice_lengths, const int32_t* slice_sets, int32_t* sellp_ci,    \
                                  T* sellp_v, void* stream);                                                     \
    int b200sp_csr_to_hybrid_coo_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, int32_t width, \
                                       const int32_t* offsets, int32_t* coo_rows, int32_t* coo_ci, T* coo_v,      \
                                       void* stream);                                                             \
    int b200sp_ell_to_csr_fill_##SUF(int64_t n, int64_t width, int64_t stride, const int32_t* ell_ci,            \
                                     const T* ell_v, const int32_t* rp, int32_t* ci, T* v, void* stream);         \
    int b200sp_sellp_to_csr_fill_##SUF(int64_t n, int32_t slice_size, const int32_t* slice_lengths,              \
                                       const int32_t* slice_sets, const int32_t* sellp_ci, const T* sellp_v,      \
                                       const int32_t* rp, int32_t* ci, T* v, void* stream);                       \
    int b200sp_hybrid_coo_append_##SUF(int64_t n, const int32_t* rp, const int32_t* ell_len, const int32_t* coo_rp, \
                                       const int32_t* coo_ci, const T* coo_v, int32_t* ci, T* v, void* stream);   \
    int b200sp_dense_row_nnz_##SUF(int64_t n, int64_t k, const T* a, int64_t as, int32_t* len, void* stream);    \
    int b200sp_dense_to_csr_fill_##SUF(int64_t n, int64_t k, const T* a, int64_t as, const int32_t* rp,          \
                                       int32_t* ci, T* v, void* stream);                                          \
    int b200sp_csr_to_dense_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* a, int64_t as, \
                                  void* stream);
B200SP_CONVERT_DECL(double, f64)
B200SP_CONVERT_DECL(float, f32)

/* ---- generators (replace src/problems.py:11-45 at device scale) --------- */
/* rows row0 .. row0+n-1 of the global stencil (global column indices);
 * 3-D kinds: nz planes of g x g along the slowest axis (nz = g: the cube) */
int b200sp_stencil_lengths(int32_t kind, int64_t g, int64_t nz, int64_t row0, int64_t n, int32_t* len, void* stream);
int b200sp_stencil_fill_f64(int32_t kind, int64_t g, int64_t nz, double conv, int64_t row0, int64_t n,
                            const int32_t* rp, int32_t* ci, double* v, void* stream);
int b200sp_stencil_fill_f32(int32_t kind, int64_t g, int64_t nz, double conv, int64_t row0, int64_t n,
                            const int32_t* rp, int32_t* ci, float* v, void* stream);
int b200sp_powerlaw_lengths(int64_t n, uint64_t seed, const double* thresholds, int32_t max_len, int32_t* len,
                            void* stream);
int b200sp_powerlaw_fill_f64(int64_t n, uint64_t seed, const int32_t* rp, int32_t* ci, double* v, void* stream);
int b200sp_powerlaw_fill_f32(int64_t n, uint64_t seed, const int32_t* rp, int32_t* ci, float* v, void* stream);

/* ---- block-Jacobi (replaces _JacobiGenerateKernel / gauss_jordan_inverse /
 * _extract_block / _JacobiApplyKernel, precond.py:28-125, :200-208) --------
 * Generation: block sizes^2 -> exclusive scan (off64) -> invert into fp64
 * column-major blocks (bit-identical Gauss-Jordan), kappa_inf, precision
 * flag and stored byte size per block; singular: smallest singular block
 * index (init to INT64_MAX). Pack: fp64 -> mixed storage at byte offsets. */
int b200sp_jacobi_block_sizes_sq(int64_t nblocks, const int32_t* starts, int32_t* out, void* stream);
int b200sp_jacobi_invert_f64(int64_t nblocks, const int32_t* starts, const int32_t* rp, const int32_t* ci,
                             const double* vals, const int64_t* off64, double* inv64, double* cond, uint8_t* prec,
                             int32_t* nbytes, int32_t adaptive, double threshold, int64_t* singular, void* stream);
int b200sp_jacobi_invert_f32(int64_t nblocks, const int32_t* starts, const int32_t* rp, const int32_t* ci,
                             const float* vals, const int64_t* off64, double* inv64, double* cond, uint8_t* prec,
                             int32_t* nbytes, int32_t adaptive, double threshold, int64_t* singular, void* stream);
int b200sp_jacobi_pack(int64_t nblocks, const int32_t* starts, const int64_t* off64, const double* inv64,
                       const uint8_t* prec, const int64_t* offs, void* storage, void* stream);
int b200sp_jacobi_apply_f64(int64_t nblocks, const int32_t* starts, const int64_t* offs, const uint8_t* prec,
                            const void* storage, int32_t m, const double* r, int64_t rs, double* z, int64_t zs,
                            void* stream);
int b200sp_jacobi_apply_f32(int64_t nblocks, const int32_t* starts, const int64_t* offs, const uint8_t* prec,
                            const void* storage, int32_t m, const float* r, int64_t rs, float* z, int64_t zs,
                            void* stream);
/* Blocks of more than 32 rows (any block_size / block_boundaries, reference
 * src/precond.py:155-197): same arithmetic contract as the warp kernels, one
 * CTA per block with [B | I] in a caller-provided fp64 scratch of
 * slots x max_bs x 2 max_bs (slots = CTAs in flight), max_bs <=
 * b200sp_jacobi_large_max_block(). The apply takes any block sizes. */
int64_t b200sp_jacobi_large_max_block(void);
int b200sp_jacobi_invert_large_f64(int64_t nblocks, const int32_t* starts, const int32_t* rp, const int32_t* ci,
                                   const double* vals, const int64_t* off64, double* inv64, double* cond,
                                   uint8_t* prec, int32_t* nbytes, int32_t adaptive, double threshold,
                                   int64_t* singular, int32_t max_bs, double* scratch, int32_t slots, void* stream);
int b200sp_jacobi_invert_large_f32(int64_t nblocks, const int32_t* starts, const int32_t* rp, const int32_t* ci,
                                   const float* vals, const int64_t* off64, double* inv64, double* cond,
                                   uint8_t* prec, int32_t* nbytes, int32_t adaptive, double threshold,
                                   int64_t* singular, int32_t max_bs, double* scratch, int32_t slots, void* stream);
int b200sp_jacobi_apply_large_f64(int64_t nblocks, const int32_t* starts, const int64_t* offs, const uint8_t* prec,
                                  const void* storage, int32_t m, const double* r, int64_t rs, double* z, int64_t zs,
                                  void* stream);
int b200sp_jacobi_apply_large_f32(int64_t nblocks, const int32_t* starts, const int64_t* offs, const uint8_t* prec,
                                  const void* storage, int32_t m, const float* r, int64_t rs, float* z, int64_t zs,
                                  void* stream);

/* ---- device-resident Krylov iterations (m = 1) ---------------------------
 * Control block (b200sp_krylov_ctl_bytes) holds iteration count, status
 * (stopped / stopping_id / finalized), breakdown, criteria (type 1 =
 * Iteration(max), 2 = ResidualNormReduction(factor); src/stop.py:118-246)
 * and the solver scalars; part: b200sp_krylov_part_elems() doubles; hist:
 * optional per-check residual norms (hist_cap entries). Every kernel is a
 * no-op once the solve is done, so a batch of iterations can be captured in
 * one CUDA graph. JAC = (nblocks, starts, offs, prec, storage); nblocks = 0
 * means no preconditioner (z aliases r).
 *   CG       src/solvers/krylov.py:36-77:   per iteration step1, SpMV, sigma, step2
 *   BiCGSTAB src/solvers/krylov.py:190-271: step1, SpMV, gamma, step2, SpMV, tst, step3
 *   GMRES    src/solvers/gmres.py:183-340:  per Arnoldi step j: [Jacobi], SpMV,
 *            dot0, mgs(i = 0..j-1), normalize; per cycle: backsolve, combine,
 *            after_commit, residual SpMV, reset, scale_v0 */
/* Persistent cooperative CG for small Csr systems (one launch per solve,
 * two grid-wide barriers per iteration: the p update is recomputed inside
 * the SpMV and written to the other of p / p2, n values each; after
 * b200sp_cg_init_* (which fills p), no preconditioner, contiguous x). */
int b200sp_cg_coop_f64(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const double* vals, double* x,
                       double* r, double* p, double* p2, double* q, void* ctl, double* part, double* hist, void* stream);
int b200sp_cg_coop_f32(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const float* vals, float* x,
                       float* r, float* p, float* p2, float* q, void* ctl, double* part, double* hist, void* stream);
/* Persistent cooperative BiCGSTAB for small unpreconditioned Csr systems
 * (one launch per solve; after b200sp_bicgstab_init_*, y = p and z = s;
 * contiguous x): BicgstabStep1/2/3, the gamma and (t.s, t.t) reductions,
 * the mid check with finalize and the top check (src/solvers/krylov.py:
 * 190-271, steps.py:348-480), five grid barriers per cycle. */
int b200sp_bicgstab_coop_f64(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const double* vals,
                             double* x, double* r, const double* rt, double* p, double* v, double* s, double* t,
                             void* ctl, double* part, double* hist, void* stream);
int b200sp_bicgstab_coop_f32(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const float* vals,
                             float* x, float* r, const float* rt, float* p, float* v, float* s, float* t,
                             void* ctl, double* part, double* hist, void* stream);
/* Persistent cooperative FCG for small unpreconditioned Csr systems (one
 * launch per solve, after b200sp_cg_init_* + b200sp_fcg_init_ctl; z = r):
 * CgStep1, SpMV + sigma, FcgStep2 (src/solvers/krylov.py:80-125). */
int b200sp_fcg_coop_f64(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const double* vals, double* x,
                        double* r, double* p, double* q, double* t, void* ctl, double* part, double* hist,
                        void* stream);
int b200sp_fcg_coop_f32(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const float* vals, float* x,
                        float* r, float* p, float* q, float* t, void* ctl, double* part, double* hist,
                        void* stream);
/* Persistent cooperative CGS for small unpreconditioned Csr systems (one
 * launch per solve, after b200sp_bicgstab_init_*; ph = p, uh = w):
 * CgsStep1/2/3, gamma, the mid check (src/solvers/krylov.py:128-187). */
int b200sp_cgs_coop_f64(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const double* vals, double* x,
                        double* r, const double* rt, double* p, double* q, double* u, double* vh, double* w,
                        double* t, void* ctl, double* part, double* hist, void* stream);
int b200sp_cgs_coop_f32(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const float* vals, float* x,
                        float* r, const float* rt, float* p, float* q, float* u, float* vh, float* w, float* t,
                        void* ctl, double* part, double* hist, void* stream);
int64_t b200sp_krylov_ctl_bytes(void);
int64_t b200sp_krylov_part_elems(void);
int b200sp_krylov_ctl_init(void* ctl, int32_t n_crit, const int32_t* crit_type, const double* crit_param,
                           int32_t needs_residual, int32_t hist_cap, int32_t kdim, void* stream);
int b200sp_krylov_status(const void* ctl, int32_t* out_i8, double* out_d8, void* stream);
int b200sp_krylov_force_stop(void* ctl, int32_t stopping_id, int32_t gmres, void* stream);
const int32_t* b200sp_krylov_guard(const void* ctl, int32_t which);
int64_t b200sp_gmres_workspace_elems(int32_t k);
int b200sp_gmres_backsolve(void* ctl, double* gm, void* stream);
int b200sp_gmres_after_commit(void* ctl, void* stream);
#define B200SP_JAC_DECL int64_t jnb, const int32_t *jstarts, const int64_t *joffs, const uint8_t *jprec, const void *jstore
#define B200SP_KRYLOV_DECL(T, SUF)                                                                                 \
    int b200sp_cg_init_##SUF(int64_t n, const T* r, T* z, T* p, B200SP_JAC_DECL, void* ctl, double* part,           \
                             double* hist, void* stream);                                                          \
    int b200sp_cg_step1_##SUF(int64_t n, T* p, const T* z, const void* ctl, void* stream);                         \
    int b200sp_cg_sigma_##SUF(int64_t n, const T* p, const T* q, void* ctl, double* part, void* stream);            \
    int b200sp_fcg_step2_##SUF(int64_t n, T* x, int64_t xs, T* r, const T* p, const T* q, T* t, T* z,              \
                               B200SP_JAC_DECL, void* ctl, double* part, double* hist, void* stream);             \
    int b200sp_cg_step2_##SUF(int64_t n, T* x, int64_t xs, T* r, const T* p, const T* q, T* z, B200SP_JAC_DECL,     \
                              void* ctl, double* part, double* hist, void* stream);                                \
    int b200sp_bicgstab_init_##SUF(int64_t n, const T* b, int64_t bs, const T* r, T* rt, T* p, T* v, T* s, T* t,    \
                                   T* y, T* z, void* ctl, double* part, double* hist, void* stream);               \
    int b200sp_bicgstab_step1_##SUF(int64_t n, const T* r, T* p, const T* v, T* y, B200SP_JAC_DECL,                \
                                    const void* ctl, void* stream);                                                \
    int b200sp_bicgstab_gamma_##SUF(int64_t n, const T* rt, const T* v, void* ctl, double* part, void* stream);     \
    int b200sp_bicgstab_step2_##SUF(int64_t n, const T* r, const T* v, T* s, T* z, B200SP_JAC_DECL, void* ctl,     \
                                    double* part, double* hist, void* stream);                                     \
    int b200sp_bicgstab_tst_##SUF(int64_t n, const T* t, const T* s, void* ctl, double* part, void* stream);        \
    int b200sp_bicgstab_step3_##SUF(int64_t n, T* x, int64_t xs, T* r, const T* s, const T* t, const T* y,         \
                                    const T* z, const T* rt, void* ctl, double* part, double* hist, void* stream); \
    int b200sp_cgs_step1_##SUF(int64_t n, const T* r, const T* q, T* u, T* p, T* ph, B200SP_JAC_DECL,             \
                               const void* ctl, void* stream);                                                     \
    int b200sp_cgs_step2_##SUF(int64_t n, const T* u, const T* vh, T* q, T* w, T* uh, B200SP_JAC_DECL,            \
                               const void* ctl, void* stream);                                                     \
    int b200sp_cgs_step3_##SUF(int64_t n, T* x, int64_t xs, T* r, const T* t, const T* uh, const T* rt, void* ctl, \
                               double* part, double* hist, void* stream);                                          \
    int b200sp_gmres_reset_##SUF(int64_t n, const T* r, void* ctl, double* part, double* gm, double* hist,          \
                                 int32_t first, void* stream);                                                     \
    int b200sp_gmres_scale_v0_##SUF(int64_t n, const T* r, T* V, const void* ctl, void* stream);                   \
    int b200sp_gmres_dot0_##SUF(int64_t n, int32_t j, const T* V, const T* w, void* ctl, double* part, double* gm,  \
                                void* stream);                                                                     \
    int b200sp_gmres_mgs_##SUF(int64_t n, int32_t j, int32_t i, const T* V, T* w, void* ctl, double* part,          \
                               double* gm, double* hist, void* stream);                                            \
    int b200sp_gmres_normalize_##SUF(int64_t n, int32_t j, T* V, const T* w, const void* ctl, void* stream);        \
    int b200sp_gmres_combine_##SUF(int64_t n, const T* V, T* x, int64_t xs, B200SP_JAC_DECL, void* ctl,            \
                                   const double* gm, void* stream);
B200SP_KRYLOV_DECL(double, f64)
B200SP_KRYLOV_DECL(float, f32)
/* Arnoldi step j of GMRES for small systems (n <= b200sp_gmres_small_rows()):
 * dot0, every MGS step, the Givens update + check and the normalisation of
 * v_j in one single-block launch (replaces gmres_dot0 + j x gmres_mgs +
 * gmres_normalize; gmres.py:88-129). */
int32_t b200sp_gmres_small_rows(void);
int b200sp_gmres_arnoldi_small_f64(int64_t n, int32_t j, double* V, double* w, void* ctl, double* gm, double* hist,
                                   void* stream);
int b200sp_gmres_arnoldi_small_f32(int64_t n, int32_t j, float* V, float* w, void* ctl, double* gm, double* hist,
                                   void* stream);
/* A whole Arnoldi cycle (j = 1..k until a check stops it) of an
 * unpreconditioned Csr system of n <= b200sp_gmres_small_rows() rows in one
 * single-block launch: w = A v_{j-1} and the Arnoldi step above. */
int b200sp_gmres_cycle_small_f64(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const double* vals,
                                 double* V, double* w, void* ctl, double* gm, double* hist, void* stream);
int b200sp_gmres_cycle_small_f32(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const float* vals,
                                 float* V, float* w, void* ctl, double* gm, double* hist, void* stream);
/* The WHOLE restarted GMRES(k) solve of an unpreconditioned system of n <= 4
 * rows in one launch (the paper's 1x1 overhead benchmark): cycles, the
 * back-solve, x += V y, the true residual and the restart, all on chip
 * (k <= 128), after gmres_reset(first) and gmres_scale_v0 of the initial
 * residual; x is updated in place. */
int b200sp_gmres_solve_tiny_f64(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const double* vals,
                                double* x, const double* b, double* V, double* w, void* ctl, double* gm,
                                double* hist, int32_t k, void* stream);
int b200sp_gmres_solve_tiny_f32(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const float* vals,
                                float* x, const float* b, float* V, float* w, void* ctl, double* gm, double* hist,
                                int32_t k, void* stream);

/* Csr SpMV q = A p fused with the solver reduction that follows it (sub-warp
 * per row, classical layout): phase 1 = CG sigma = p.q (replaces
 * b200sp_cg_sigma), 2 = BiCGSTAB gamma = u.q with u = r_tilde (replaces
 * bicgstab_gamma), 3 = BiCGSTAB ts = q.u, tt = q.q with u = s (replaces
 * bicgstab_tst), 4 = distributed CG ghost block: q += A p (p = the ghost
 * vector) and sigma = u.q with u = the owned p. The control step (or, with a
 * distributed ctl, the parking of the local sum) runs in the last block as in the unfused
 * kernels (src/solvers/krylov.py:56-76, :233-265). `subwarp` takes the
 * B200SP_SUBWARP_EVEN_NNZ flag as for the classical SpMV. */
int b200sp_csr_spmv_dot_f64(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const double* vals,
                            const double* p, double* q, const double* u, int32_t phase, int32_t subwarp, void* ctl,
                            double* part, void* stream);
int b200sp_csr_spmv_dot_f32(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, const float* vals,
                            const float* p, float* q, const float* u, int32_t phase, int32_t subwarp, void* ctl,
                            double* part, void* stream);

/* ---- device assembly of coordinate triples (reference MatrixData.canonicalize,
 * src/formats.py:40-53, bit for bit) ------------------------------------------
 * int64 rows / cols and fp64 values (any order, duplicates allowed, indices
 * pre-validated) -> (row, col)-sorted unique int32 rows / cols and values of
 * the suffix type; *nnz_out (device int32) = number of unique coordinates.
 * Stable LSD radix sort of row * ncols + col; duplicate groups summed
 * 0.0 + v1 + v2 ... in input order when the input has any duplicate. */
int64_t b200sp_assemble_workspace_bytes(int64_t count);
int b200sp_assemble_coo_f64(int64_t count, const int64_t* rows, const int64_t* cols, const double* vals,
                            int64_t nrows, int64_t ncols, int32_t* rows_out, int32_t* cols_out, double* vals_out,
                            int32_t* nnz_out, void* ws, void* stream);
int b200sp_assemble_coo_f32(int64_t count, const int64_t* rows, const int64_t* cols, const double* vals,
                            int64_t nrows, int64_t ncols, int32_t* rows_out, int32_t* cols_out, float* vals_out,
                            int32_t* nnz_out, void* ws, void* stream);

/* ---- ParILU(0) + sparse triangular solves (reference src/precond.py:211-426,
 * src/solvers/triangular.py:18-155) -----------------------------------------
 * ilu_counts: per-row entries with col <= i (L) and col >= i (U); *nodiag =
 * first row without a stored diagonal (init INT_MAX). diag: first stored
 * diagonal per row, *zero = first row whose diagonal is 0 or missing (init
 * INT_MAX). ilu_fill: L / U patterns (row pointers from exclusive scans of
 * the counts), original values al / au and the initial iterate (l = a / a_jj,
 * l_ii = 1; u = a). parilu_sweep: one Jacobi-style fixed-point sweep from
 * (lold, uold) into (lnew, unew); lrow / urow from csr_rows. trs: sync-free
 * substitution of one column, lower (forward) or upper (backward); diag NULL
 * = unit diagonal; `ready` (n int32, zero at creation) and a fresh `epoch`
 * per call; `ticket` = one int32 of scratch; `order` = rows grouped by
 * dependency level (b200sp_trs_order) or NULL for plain row order. */
int b200sp_ilu_counts(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, int32_t* lcnt, int32_t* ucnt,
                      int32_t* nodiag, void* stream);
int b200sp_csr_rows(int64_t n, const int32_t* row_ptrs, int32_t* row_of_entry, void* stream);
/* dependency levels of a triangular factor (relaxation sweeps until
 * *changed stays 0) and the rows grouped by level (claim order of trs) */
int b200sp_trs_levels(int64_t n, const int32_t* row_ptrs, const int32_t* col_idxs, int32_t lower, int32_t* level,
                      int32_t* changed, void* stream);
int b200sp_trs_level_hist(int64_t n, const int32_t* level, int32_t* count, void* stream);
/* level-synchronous substitution of one column as one cooperative launch
 * (rows of a level in parallel, a grid barrier between levels); offs =
 * nlevels + 1 level starts in `order`; diag NULL = unit diagonal */
int b200sp_trs_coop_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, const double* diag,
                        const double* b, int64_t bs, double* x, int64_t xs, const int32_t* order, const int32_t* offs,
                        int32_t nlevels, void* stream);
int b200sp_trs_coop_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v, const float* diag,
                        const float* b, int64_t bs, float* x, int64_t xs, const int32_t* order, const int32_t* offs,
                        int32_t nlevels, void* stream);
int b200sp_trs_order(int64_t n, const int32_t* level, const int32_t* offs, int32_t* cursor, int32_t* order,
                     void* stream);
#define B200SP_ILU_DECL(T, SUF)                                                                                     \
    int b200sp_diag_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, T* diag, int32_t* zero,      \
                          void* stream);                                                                           \
    int b200sp_ilu_fill_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, const T* diag,          \
                              const int32_t* lrp, const int32_t* urp, int32_t* lci, T* al, T* lv, int32_t* uci,    \
                              T* au, T* uv, void* stream);                                                         \
    int b200sp_parilu_sweep_##SUF(int64_t n, int64_t nl, int64_t nu, const int32_t* lrow, const int32_t* lrp,       \
                                  const int32_t* lci, const T* al, const T* lold, T* lnew, const int32_t* urow,    \
                                  const int32_t* urp, const int32_t* uci, const T* au, const T* uold, T* unew,     \
                                  void* stream);                                                                   \
    int b200sp_trs_##SUF(int64_t n, const int32_t* rp, const int32_t* ci, const T* v, const T* diag,               \
                         int32_t lower, const T* b, int64_t bs, T* x, int64_t xs, int32_t* ready, int32_t epoch,   \
                         int32_t* ticket, const int32_t* order, void* stream);
B200SP_ILU_DECL(double, f64)
B200SP_ILU_DECL(float, f32)

/* ---- Matrix Market reader (host code; reference src/mmio.py:38-126) ------
 * b200sp_mm_header parses the header and size line of the file image `buf`:
 * info[7] = {array?, symmetric?, rows, cols, entries, body offset, size-line
 * number}; b200sp_mm_count sizes the output (symmetric mirrors included);
 * b200sp_mm_parse fills 0-based int64 rows / cols and vals (array files:
 * vals only, column-major) with `threads` host threads (<= 0: all cores).
 * Errors: B200SP_EINVAL = ParseError with *err_line the reference's 1-based
 * line number, B200SP_EUNSUPPORTED = Unsupported; same messages. */
int b200sp_mm_header(const char* buf, int64_t len, int64_t* info, int64_t* err_line);
int b200sp_mm_count(const char* buf, int64_t len, const int64_t* info, int32_t threads, int64_t* out_count);
int b200sp_mm_parse(const char* buf, int64_t len, const int64_t* info, int32_t threads, int64_t* rows,
                    int64_t* cols, double* vals, int64_t capacity, int64_t* out_count, int64_t* err_line);

/* ---- row-partitioned (distributed) CG ------------------------------------
 * Each rank holds rows [lo, hi) with vector layout [owned | ghosts]; the
 * reduction kernels of a ctl with dist = 1 park their local sums in the ctl's
 * red[] (byte offset b200sp_krylov_red_offset()), the caller all-reduces
 * them across ranks (NCCL) and b200sp_cg_finish runs the control step
 * (phase 0 init, 1 sigma, 2 step2). No reference counterpart: the reference
 * has no distributed matrix. */
int b200sp_krylov_set_dist(void* ctl, int32_t dist, void* stream);
int64_t b200sp_krylov_red_offset(void);
/* Peer-memory halo for the distributed CG (CUDA IPC over NVLink/NVSwitch):
 * cg_step1_put = CgStep1 (p = z + beta p, steps.py:93-119) that also stores
 * local rows [lo[k], hi[k]) into dst[k] (a peer's ghost slots, mapped) and,
 * once every CTA's stores are out, writes epoch to flag[k] (this rank's slot
 * in the peer's flag array; release, system scope). ticket: one zeroed
 * uint32. peer_wait: a one-thread kernel returning once every flags[k] >=
 * epoch (acquire) -- order the ghost SpMV after it. Both skip when the
 * solve is done. At most b200sp_peer_max() puts, twice that many waits. */
int32_t b200sp_peer_max(void);
/* epoch_dev (nullable): a device int32 holding the last epoch -- the kernels
 * then take epoch = *epoch_dev + 1 (put, all-reduce) / *epoch_dev (wait) and
 * advance it themselves, so the sequence can be captured in a CUDA graph and
 * replayed; `epoch` is ignored then. */
int b200sp_cg_step1_put_f64(int64_t n, double* p, const double* z, const void* ctl, int32_t nput, const int64_t* lo,
                            const int64_t* hi, void* const* dst, int32_t* const* flag, int32_t epoch,
                            uint32_t* ticket, int32_t* epoch_dev, void* stream);
int b200sp_cg_step1_put_f32(int64_t n, float* p, const float* z, const void* ctl, int32_t nput, const int64_t* lo,
                            const int64_t* hi, void* const* dst, int32_t* const* flag, int32_t epoch,
                            uint32_t* ticket, int32_t* epoch_dev, void* stream);
int b200sp_peer_wait(void* ctl, int32_t nwait, const int32_t* const* flags, int32_t epoch, const int32_t* epoch_dev,
                     void* stream);
/* All-reduce (sum) of red[0..k), k <= 4, across `world` <= 8 ranks through
 * peer memory: slots[j] = rank j's slot array (2 * world * 4 doubles, zeroed
 * once; mapped), flags[j] = rank j's int32 flag array (world entries, zeroed
 * once); epoch increases by one per call on every rank. Sums in rank order:
 * identical on every rank. One thread; replaces the 8-32 byte NCCL
 * all-reduces of the distributed CG. */
int b200sp_peer_allreduce(double* red, int32_t k, int32_t world, int32_t rank, double* const* slots,
                          int32_t* const* flags, int32_t epoch, int32_t* epoch_dev, void* stream);
/* The plain distributed SpMV through peer memory: peer_put copies local rows
 * [lo[k], hi[k]) of the owned x into dst[k] (a destination's ghost slots)
 * once every destination has acknowledged the previous epoch (ack_in[k]: the
 * destination's ack of this rank, in THIS rank's ack array), then raises
 * flag[k] = epoch (device-managed *epoch_dev + 1); peer_wait_plain waits for
 * the sources' flags of *epoch_dev; peer_ack (after the ghost SpMV) raises
 * ack_out[k] = *epoch_dev in every source's ack array. */
int b200sp_peer_put_f64(const double* x_owned, int32_t nput, const int64_t* lo, const int64_t* hi, void* const* dst,
                        int32_t* const* flag, int32_t nack, const int32_t* const* ack_in, int32_t* epoch_dev,
                        uint32_t* ticket, void* stream);
int b200sp_peer_put_f32(const float* x_owned, int32_t nput, const int64_t* lo, const int64_t* hi, void* const* dst,
                        int32_t* const* flag, int32_t nack, const int32_t* const* ack_in, int32_t* epoch_dev,
                        uint32_t* ticket, void* stream);
int b200sp_peer_ack(int32_t nack, const int32_t* const* ack_out, const int32_t* epoch_dev, void* stream);
int b200sp_peer_wait_plain(int32_t nwait, const int32_t* const* flags, const int32_t* epoch_dev, void* stream);
/* Spins on peer flags are bounded by b200sp_set_tuning("peer_timeout_ms", ms)
 * (default 30000): peer_wait then marks the solve broken down (code 6),
 * peer_allreduce returns NaN sums.
 *
 * CUDA IPC + explicit peer access (setup of the peer-memory paths): export a
 * device buffer as an allocation handle (b200sp_ipc_handle_bytes() bytes)
 * plus offset; open it in the caller's CURRENT device context (lazy peer
 * access, no context on the owner's device); peer_enable reports whether the
 * current device can reach `peer` (cudaDeviceCanAccessPeer) and enables it. */
int32_t b200sp_ipc_handle_bytes(void);
int b200sp_ipc_export(const void* ptr, void* handle, int64_t* offset);
int b200sp_ipc_open(const void* handle, int64_t offset, void** ptr, void** base);
int b200sp_ipc_close(void* base);
int b200sp_peer_enable(int32_t peer, int32_t* can);
int b200sp_cg_finish(void* ctl, double* hist, int32_t phase, void* stream);
/* FCG (src/solvers/krylov.py:80-125) reuses cg_init / cg_step1 / the fused
 * SpMV + sigma; fcg_init_ctl seeds rho_t = 0 after cg_init, fcg_step2 also
 * forms t = r_new - r_old and reduces (r.z, t.z, r.r). */
int b200sp_fcg_init_ctl(void* ctl, void* stream);
/* CGS (src/solvers/krylov.py:128-187) reuses bicgstab_init and the gamma
 * SpMV epilogue; cgs_mid is the mid-cycle check on the unchanged ||r||. */
int b200sp_cgs_mid(void* ctl, double* hist, void* stream);
int b200sp_flag_out_of_range(int64_t nnz, const int32_t* ci, int64_t lo, int64_t hi, int32_t* flag, void* stream);
int b200sp_compact_cols(int64_t nnz, const int32_t* ci, const int32_t* flag, const int32_t* pos, int32_t* out,
                        void* stream);
int b200sp_map_cols(int64_t nnz, int32_t* ci, int64_t lo, int64_t hi, const int32_t* ghosts, int64_t nghost,
                    void* stream);
int b200sp_split_count(int64_t n, const int32_t* rp, const int32_t* ci, int32_t thr, int32_t* len_lo,
                       int32_t* len_hi, void* stream);
int b200sp_split_fill_f64(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, int32_t thr,
                          const int32_t* rp_lo, const int32_t* rp_hi, int32_t* ci_lo, double* v_lo, int32_t* ci_hi,
                          double* v_hi, void* stream);
int b200sp_split_fill_f32(int64_t n, const int32_t* rp, const int32_t* ci, const float* v, int32_t thr,
                          const int32_t* rp_lo, const int32_t* rp_hi, int32_t* ci_lo, float* v_lo, int32_t* ci_hi,
                          float* v_hi, void* stream);
int b200sp_gather_f64(int64_t count, const int32_t* idx, const double* src, double* dst, void* stream);
int b200sp_gather_f32(int64_t count, const int32_t* idx, const float* src, float* dst, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* B200SP_H */
