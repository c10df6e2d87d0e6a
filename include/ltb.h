/*
 * ltb.h — C ABI of the B200-native *_L hot path (libltb.so).
 *
 * The reference (`ltensor`, pure Python over numpy/scipy) has no FFI; its
 * "plugin interface" is the set of Python functions re-exported by
 * pkg/src/ltensor/__init__.py:3-45.  Every entry point below replaces the
 * numerics underneath one of those functions; the Python package
 * `paper_2202_02870_b200` keeps the reference signatures and calls these
 * through ctypes (see INTEGRATION.md for the binding).
 *
 * Conventions
 *   - All functions return an ltb_status; 0 is success.  On failure
 *     ltb_ctx_last_error() holds a one-line message.  Codes map 1:1 to the
 *     reference exception classes (pkg/src/ltensor/errors.py:8-41).
 *   - Pointers named `d_*` are device pointers (allocated with ltb_malloc or
 *     by the caller, e.g. torch); `h_*` are host pointers.
 *   - Every call is stream-ordered on the context stream.  Calls that return
 *     host-visible results (norms, flags, copies to host) synchronise that
 *     stream before returning.
 *   - Dense tensors are C-order.  A tensor of shape (I1, I2, I3..IN) is a
 *     set of NT = I1*I2 "tubes" of P = I3*..*IN contiguous elements
 *     (TUBE_MAJOR).  The transform-domain slice stack is SLICE_MAJOR:
 *     element (q, i1, i2) at q*NT + i1*I2 + i2, q the C-order trailing index.
 *     (The reference's rep-stack p-order is Fortran over the trailing dims,
 *     core.py:43-74; per-slice outputs are permuted at the Python boundary.)
 *   - Complex values are interleaved (re, im) pairs of the real type.
 */
#ifndef LTB_H_
#define LTB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ltb_ctx ltb_ctx;
typedef struct ltb_spec ltb_spec;
typedef struct ltb_pga ltb_pga;

/* status codes — errors.py:8-41 (ShapeError, TransformError,
 * UnsupportedSpecError, ParameterError, NumericConsistencyError) plus device
 * failures that the reference cannot raise (mapped to DeviceError). */
enum ltb_status {
  LTB_OK = 0,
  LTB_ESHAPE = 1,
  LTB_ETRANSFORM = 2,
  LTB_EUNSUPPORTED = 3,
  LTB_EPARAM = 4,
  LTB_ENUMERIC = 5,
  LTB_ECUDA = 6,
  LTB_ENCCL = 7,
  LTB_EOOM = 8
};

/* element types */
enum ltb_dtype { LTB_F32 = 0, LTB_F64 = 1, LTB_C64 = 2, LTB_C128 = 3 };

/* layouts of a tensor's trailing (tube) index, see header comment */
enum ltb_layout { LTB_TUBE_MAJOR = 0, LTB_SLICE_MAJOR = 1 };

/* GEMM operand ops */
enum ltb_op { LTB_OP_N = 0, LTB_OP_T = 1, LTB_OP_C = 2 /* conj, no transpose */, LTB_OP_H = 3 };

/* ---------------------------------------------------------------- context */
int ltb_version(void);
int ltb_device_count(int* count);
int ltb_ctx_create(int device, ltb_ctx** out);
void ltb_ctx_destroy(ltb_ctx* ctx);
const char* ltb_ctx_last_error(const ltb_ctx* ctx);
/* adopt an external cudaStream_t (e.g. torch.cuda.current_stream()); NULL = own stream */
int ltb_ctx_set_stream(ltb_ctx* ctx, void* stream);
int ltb_ctx_synchronize(ltb_ctx* ctx);
/* per-context test / profiling options (no process-global state): value is a flag or a
 * device pointer (uint64 buffers the kernels stamp with clock values; 0 disables) */
enum ltb_option {
  LTB_OPT_FORCE_BLOCKED_SVD = 1, /* route every SVD / SVT through the blocked Jacobi tier */
  LTB_OPT_TC_TIMELINE = 2,       /* tcgen05 GEMM / transform: per-tile stamps of CTA 0 */
  LTB_OPT_QR_TIMELINE = 3,       /* QR-preconditioned Jacobi: stage stamps of CTA 0 */
  LTB_OPT_JACOBI_PAIRS = 4,      /* warm Cholesky-path Jacobi: 0 blocks of 4 columns, 1 one pair per team, 2 blocks of 2 */
  LTB_OPT_FULL_SWEEPS = 5        /* carried complex SVT: full sweeps instead of the truncated ones (cross-checks) */
};
int ltb_ctx_set_option(ltb_ctx* ctx, int option, int64_t value);
/* make ctx's device the calling host thread's current CUDA device (contexts of several
 * devices may coexist in one process; each call runs on the current device) */
int ltb_ctx_make_current(ltb_ctx* ctx);
/* number of ltb kernels launched on this context since creation */
int64_t ltb_ctx_launch_count(const ltb_ctx* ctx);
/* device-side counters (3 entries): h_out[0] = Jacobi slices solved, h_out[1] = Jacobi sweeps run,
 * h_out[2] = most sweeps of one slice */
int ltb_ctx_stats(ltb_ctx* ctx, int64_t* h_out, int reset);

/* ---------------------------------------------------------------- memory */
int ltb_malloc(ltb_ctx* ctx, int64_t bytes, void** d_out);
int ltb_free(ltb_ctx* ctx, void* d_ptr);
int ltb_memcpy_h2d(ltb_ctx* ctx, void* d_dst, const void* h_src, int64_t bytes);
int ltb_memcpy_d2h(ltb_ctx* ctx, void* h_dst, const void* d_src, int64_t bytes);
int ltb_memcpy_d2d(ltb_ctx* ctx, void* d_dst, const void* d_src, int64_t bytes);
int ltb_memset_zero(ltb_ctx* ctx, void* d_dst, int64_t bytes);
/* elementwise dtype conversion (real<->complex, single<->double); complex->real keeps .re */
int ltb_convert(ltb_ctx* ctx, int64_t n, int dtype_in, const void* d_in, int dtype_out, void* d_out);
/* TLT1 container payload (io.py:1-10, read_container io.py:54-83): reorder a
 * generalized column-major (Fortran) payload of `ndim` dims to C order on the
 * device; elem_bytes 1 (bool mask), 4 (float32), 8 (float64), 16 (complex128). */
int ltb_fortran_to_c(ltb_ctx* ctx, int ndim, const int64_t* dims, int elem_bytes, const void* d_src, void* d_dst);

/* ---------------------------------------------------------------- spec
 * Replaces TransformSpec.mode_matrix / mode_inverse (transforms.py:87-100)
 * on the device: the per-mode n x n matrices of L and L^{-1}, uploaded once.
 *   trail_dims : I3..IN (ntrail entries)
 *   axes       : transformed trailing axes, 0-based (mode m -> axis m-3), ascending
 *   fwd, inv   : concatenated row-major n_k x n_k matrices, float64; if
 *                is_complex they are interleaved complex128.
 */
int ltb_spec_create(ltb_ctx* ctx, int ntrail, const int64_t* trail_dims, int nmodes,
                    const int* axes, int is_complex, const double* h_fwd, const double* h_inv,
                    ltb_spec** out);
void ltb_spec_destroy(ltb_spec* spec);

/* ---------------------------------------------------------------- K1 / K1'
 * apply_l (transforms.py:176-192) when inverse == 0, apply_l_inv
 * (transforms.py:195-226) when inverse == 1: mode products along the spec's
 * axes (ascending forward, reversed inverse) of `ntubes` tubes.
 * If the computation is complex and dtype_out is real, the real part is
 * written and h_sumsq[0] = sum |out|^2, h_sumsq[1] = sum Im(out)^2 are
 * returned (the real-output contract check of transforms.py:217-225 is then
 * made by the caller).  h_sumsq may be NULL.
 */
int ltb_transform(ltb_ctx* ctx, const ltb_spec* spec, int64_t ntubes, int inverse,
                  int dtype_in, int layout_in, const void* d_in,
                  int dtype_out, int layout_out, void* d_out, double* h_sumsq);

/* K1 of both l_product operands (linalg.py:34-43: apply_l(a), apply_l(b)) in one
 * call: two tensors with the same tube count and dtypes, each transformed as by
 * ltb_transform (no real-output check).  On the tensor-core path the pair is
 * one launch (batch of two), so the fixed launch / pipeline-fill cost is paid
 * once. */
int ltb_transform_pair(ltb_ctx* ctx, const ltb_spec* spec, int64_t ntubes, int inverse,
                       int dtype_in, int layout_in, const void* d_in0, const void* d_in1,
                       int dtype_out, int layout_out, void* d_out0, void* d_out1);

/* mode_n_product (core.py:110-122) on a C-order view (outer, nin, inner):
 * y[o, i, l] = sum_j mat[i, j] x[o, j, l], mat nout x nin row-major (dtype_mat). */
int ltb_mode_product(ltb_ctx* ctx, int64_t outer, int64_t nin, int64_t inner, int64_t nout,
                     int dtype_in, const void* d_in, int dtype_mat, const void* d_mat,
                     int dtype_out, void* d_out);

/* ---------------------------------------------------------------- K2
 * facewise product / transform-domain GEMM (core.py:125-134, linalg.py:42):
 * C[b] = op_a(A[b]) * op_b(B[b]) for b < batch; op_a(A) is m x k, op_b(B) is k x n,
 * each stored row-major with the given leading dimension and batch stride.
 */
/* l_product (linalg.py:34-43) host to host in one pipelined call: real spec, real
 * float32 / float64 tensors A (I1 x L x trailing), B (L x I2 x trailing) -> C
 * (I1 x I2 x trailing), C-order host buffers (pinned ones let the copies overlap
 * the compute in both directions).  LTB_EUNSUPPORTED (no error text) for complex
 * transform domains, which need the real-output check of the generic path. */
int ltb_l_product_host(ltb_ctx* ctx, const ltb_spec* spec, int64_t I1, int64_t L, int64_t I2, int dtype,
                       const void* h_a, const void* h_b, void* h_c);

int ltb_slice_gemm(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n, int64_t k,
                   int op_a, const void* d_a, int64_t lda, int64_t stride_a,
                   int op_b, const void* d_b, int64_t ldb, int64_t stride_b,
                   void* d_c, int64_t ldc, int64_t stride_c);

/* The fp32 tensor-core engine underneath K1/K1'/K2 (tcgen05 kind::tf32 with the
 * 3xTF32 split when split == 3, plain TF32 when split == 1), exposed for the
 * kernel tests: C[b] (m x n, ldc) = A[b] * B[b], A stored m x k (a_mn = 0) or
 * k x m (a_mn = 1), B stored n x k (b_mn = 0) or k x n (b_mn = 1).  Leading
 * dimensions and batch strides must be multiples of 4 elements.  Returns
 * LTB_EUNSUPPORTED when the shape / alignment cannot use the tensor cores. */
int ltb_tc_gemm(ltb_ctx* ctx, int64_t batch, int64_t m, int64_t n, int64_t k, int a_mn, const void* d_a,
                int64_t lda, int64_t sa, int b_mn, const void* d_b, int64_t ldb, int64_t sb, void* d_c,
                int64_t ldc, int64_t sc, int split);

/* ---------------------------------------------------------------- K3
 * Batched one-sided Jacobi on `batch` row-major m x n slices (contiguous).
 *   ltb_slice_svt: svt's slice step (linalg.py:178-180): out = U (S - tau)_+ V^H.
 *   ltb_slice_svd: t_svd's slice step (linalg.py:111), full_matrices:
 *                  u: batch x m x m, s: batch x min(m,n) (real dtype), v: batch x n x n
 *                  (v = V, not V^H: the reference uses conj(vh^T), linalg.py:115).
 *   ltb_slice_singular_values: compute_uv=False (linalg.py:137,157,164), descending.
 */
int ltb_slice_svt(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n,
                  const void* d_a, double tau, void* d_out);

/* svt (linalg.py:168-181) on the transform-domain stack of a REAL tensor under
 * `spec` (batch == spec P): when the spec's modes are real or exactly
 * Hermitian-rowed (the DFT), slices q and its conjugate partner are solved once
 * and mirrored; otherwise identical to ltb_slice_svt. */
int ltb_spec_slice_svt(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t batch, int64_t I1, int64_t I2,
                       const void* d_a, double tau, void* d_out);
/* svt's slice step for a caller that iterates (the PGA loop of completion.py:165-172
 * run outside ltb_pga_run, e.g. by the slice-sharded multi-GPU solver): fp32 real
 * slices, warm-started from the right singular bases of the previous call.
 * d_v (batch x n x n, n = min(I1, I2)) is caller-owned: read when warm != 0 and
 * rewritten on return; pass warm = 0 on the first call.  Needs n >= 32
 * (LTB_EUNSUPPORTED otherwise: use ltb_slice_svt). */
int ltb_slice_svt_carry(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const float* d_a, double tau,
                        float* d_out, float* d_v, int warm);
/* the same for complex64 slices too large for the shared-memory Jacobi tier (the
 * block-cyclic tier; config 4's 1024 x 1024 slices): svt (linalg.py:168-181) warm-started
 * from the previous call's right singular bases.  d_vt (batch x n x n complex64, n = I2)
 * holds V^T (row j = the j-th right singular vector), caller-owned, read when warm != 0 and
 * rewritten on return.  Needs I1 >= I2 >= 32 and I2 even (LTB_EUNSUPPORTED otherwise, also
 * for slices that fit in shared memory: use ltb_slice_svt). */
int ltb_slice_svt_carry_c64(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const void* d_a, double tau,
                            void* d_out, void* d_vt, int warm);
int ltb_slice_svd(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n,
                  const void* d_a, void* d_u, void* d_s, void* d_v);
int ltb_slice_singular_values(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n,
                              const void* d_a, void* d_s);

/* ---------------------------------------------------------------- reductions
 * fro_norm / inner-product helpers (core.py:26-40): h_out[0] = sum |x - y|^2
 * (y may be NULL), h_out[1] = max(Re x) (for psnr, completion.py:63-78).
 * Deterministic (fixed-order two-stage) in float64. */
int ltb_reduce_sumsq(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const void* d_y,
                     double* h_out);

/* as ltb_reduce_sumsq, result left in device memory (d_out[0..1]) with no host
 * synchronisation (stream-ordered) */
int ltb_reduce_sumsq_device(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const void* d_y,
                            double* d_out);

/* Σ conj(x) * y in float64: h_out = {re, im} (inner_product / np.vdot, core.py:26-35) */
int ltb_reduce_dot(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const void* d_y, double* h_out);

/* ---------------------------------------------------------------- slice-stack helpers
 * ltb_embed_diag     : out[b] = diag(vals[b]) as an m x n slice (vals: batch x min(m,n), real
 *                      type of dtype_out) — _embed_diag (linalg.py:93-99), identity_tensor (:46-51)
 * ltb_slice_transpose: out[b] = A[b]^T (conj != 0: A[b]^H), A[b] m x n — l_transpose (:54-59)
 * ltb_project_omega  : out = where(mask, x, 0), mask uint8 — project_omega (completion.py:23-29)
 */
int ltb_embed_diag(ltb_ctx* ctx, int dtype_out, int64_t batch, int64_t m, int64_t n, const void* d_vals,
                   void* d_out);
int ltb_slice_transpose(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n, int conj,
                        const void* d_in, void* d_out);
int ltb_project_omega(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const uint8_t* d_mask,
                      void* d_out);

/* the PGA gradient point of completion.py:170-171 on one row shard (multi-GPU
 * driver): y = x + beta (x - x_prev), g = y - (where(mask, y, 0) - p_obs);
 * real dtype, mask uint8, y may be NULL */
int ltb_pga_gradient(ltb_ctx* ctx, int dtype, int64_t n, const void* d_xc, const void* d_xp,
                     const void* d_pobs, const uint8_t* d_mask, double beta, void* d_y, void* d_g);

/* l_product (linalg.py:34-43) on device buffers (A: I1 x L x trailing, B: L x I2 x trailing,
 * C: I1 x I2 x trailing, C-order, real dtype of a real spec).  fused != 0 runs the fp32 product
 * as ONE persistent tcgen05 kernel (forward transforms, slice GEMMs and inverse transform
 * overlapped through per-group completion counters) when the shape fits (I1 % 128 == 0,
 * P <= 96); otherwise K1(A), K1(B), K2, K1'.  d_ws: ltb_l_product_ws_bytes() bytes.
 * fused == 3: as 1, and the caller guarantees that d_ws was zero-filled once and has since
 * been used only by completed fused calls (the kernel leaves its counters zeroed), which
 * saves the per-call counter reset (a memset node in a CUDA graph).
 * Stream-ordered, no host synchronisation (CUDA-graph capturable). */
int64_t ltb_l_product_ws_bytes(const ltb_spec* spec, int64_t I1, int64_t L, int64_t I2, int dtype);
int ltb_l_product_device(ltb_ctx* ctx, const ltb_spec* spec, int64_t I1, int64_t L, int64_t I2, int dtype,
                         const void* d_a, const void* d_b, void* d_c, void* d_ws, int64_t ws_bytes, int fused);

/* ---------------------------------------------------------------- sharded PGA (multi-GPU)
 * One iteration of pga_complete (completion.py:165-197) on a rank's shard, for a caller that
 * runs the collectives between the steps: every step is
 * stream-ordered, returns without a host synchronisation, and is a no-op once
 * d_state[0] != 0, so a chunk of iterations can be enqueued and read back at its end.
 *   pack_mask : uint8 0/1 -> bit-packed words (bit e of word e/32)
 *   forward   : rows shard (ntubes tubes, tube-major) -> gradient step fused into the load
 *               (y = x + beta (x - x_prev), g = y - (P_Omega(y) - p_obs)) -> L -> slice-major
 *   svt       : the slice block; d_v (batch x n x n) carries right bases between calls for
 *               real fp32 / fp64 slices and (as V^T, complex64) for complex64 slices beyond the
 *               shared-memory Jacobi tier (warm = 0 on the first call), NULL for plain svt
 *   inverse   : slice-major rows shard -> L^-1, real part -> x_next, fused norms into
 *               d_sums[0..4] = {sum (y-x+)^2, sum x+^2, sum (x+-gt)^2, sum Im^2} (all-reduce
 *               SUM) and d_sums[4] = max x+ (all-reduce MAX); d_gt may be NULL
 *   decide    : after the all-reduces: d_rec[0..4] as ltb_pga_run's records, d_state[1] +=
 *               1, d_state[0] = 1 once rel <= tol (pobs_sumsq = the global sum p_obs^2) */
int ltb_pack_mask(ltb_ctx* ctx, int64_t n, const uint8_t* d_mask, uint32_t* d_bits);
int ltb_pga_shard_forward(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t ntubes, double beta,
                          const void* d_xc, const void* d_xp, const void* d_pobs, const uint32_t* d_bits,
                          void* d_hat, const int* d_state);
int ltb_pga_shard_svt(ltb_ctx* ctx, int dtype, int64_t batch, int64_t I1, int64_t I2, const void* d_hat, double tau,
                      void* d_out, void* d_v, int warm, const int* d_state);
int ltb_pga_shard_inverse(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t ntubes, double beta,
                          const void* d_hat, const void* d_xc, const void* d_xp, const void* d_gt, void* d_xn,
                          double* d_sums, const int* d_state);
int ltb_pga_shard_decide(ltb_ctx* ctx, const double* d_sums, double pobs_sumsq, double tol, double* d_rec,
                         int* d_state);

/* ---------------------------------------------------------------- K4 + PGA
 * pga_complete (completion.py:141-202).  The host keeps the scalar
 * recurrences: it passes, per iteration k (1-based), beta_k = (t_{k-1}-1)/t_k
 * and mu_k = max(nu^k mu0, mu_bar), computed exactly as completion.py:169-193.
 * The device runs the iterations and stops itself once rel <= tol
 * (completion.py:195-197), so no host round trip is needed per iteration.
 *   create : m (float64 host, I1 x I2 x trailing), mask (uint8 0/1 host),
 *            optional ground truth (float64 host); dtype = LTB_F32 or LTB_F64
 *            selects the compute precision.
 *   run    : iterations k0 .. k0+count-1; per-iteration records are written to
 *            h_records[(k-k0)*5 + {0..4}] = {sum (y-x+)^2, sum x+^2,
 *            sum (x+-gt)^2, max x+, sum Im(x+)^2 before the real part is
 *            taken}; *h_done = iterations executed, *h_converged = 1 once
 *            rel <= tol.
 *   fetch  : x (float64 host).  With reimpose_observed != 0, h_x must hold m
 *            on entry; observed entries of the result are m itself
 *            (completion.py:199-202).
 */
int ltb_pga_create(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t i1, int64_t i2,
                   const double* h_m, const uint8_t* h_mask, const double* h_gt,
                   ltb_pga** out);
int ltb_pga_pobs_sumsq(ltb_pga* pga, double* h_out);
int ltb_pga_run(ltb_pga* pga, int k0, int count, const double* h_beta, const double* h_mu,
                double tol, double* h_records, int* h_done, int* h_converged);
int ltb_pga_fetch(ltb_pga* pga, int reimpose_observed, double* h_x);
/* device pointer of the current iterate (compute dtype, tube-major) */
int ltb_pga_current(ltb_pga* pga, void** d_x);
void ltb_pga_destroy(ltb_pga* pga);

#ifdef __cplusplus
}
#endif

#endif /* LTB_H_ */
