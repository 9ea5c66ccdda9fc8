/*
 * hmx -- B200-native H-matrix assembly + H-matvec for the 3D Helmholtz and
 * elastodynamic (U, T) Green's tensors.  C-ABI of libhmx.so.
 *
 * Plain pointers and sizes only.  Complex arrays are interleaved (re, im)
 * float64 pairs -- numpy complex128 layout -- passed as double*.
 * All functions return an int status (HMX_OK = 0); hmx_last_error() gives
 * the message of the last failure on the calling thread.
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/pkg/src/hmatx/ unless noted; SPEC = /root/reference/SPEC.md):
 *   hmx_tree_build        geometry.py:182-220  build_cluster_tree
 *   hmx_blocks_build      geometry.py:277-295  build_block_tree  (+ BlockTree.leaves :261-268)
 *   hmx_eval_block        _kernelcore_np.py:37-130  scalar_block / elasto_u_block /
 *                         elasto_t_block (the kernel-core backend seam; the missing
 *                         Cython twin _kernelcore_cy, setup.py:13-22)
 *   hmx_assemble          SPEC:381-389  hmatrix.assemble (ACA SPEC:288-306 +
 *                         recompress SPEC:318-326 on the device)
 *   hmx_hmatrix_stats     SPEC:431-439  hmatrix.storage_report
 *   hmx_matvec            SPEC:391-399  hmatrix.matvec
 *   hmx_gmres             SPEC:497-505  solve.solve_gmres
 * Error codes map to errors.py:4-32 (see HMX_E* below).
 */
#ifndef HMX_H_
#define HMX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HMX_ABI_VERSION 3

/* status codes */
#define HMX_OK 0
#define HMX_EINVAL 1    /* invalid argument / dimension mismatch (ValueError)          */
#define HMX_ECUDA 2     /* CUDA runtime failure                                        */
#define HMX_EPIVOT 3    /* pivot exhaustion after the randomized-SVD fallback also failed (PivotExhaustionError) */
#define HMX_ESINGULAR 4 /* r == 0 pair without a self rule (SingularEvaluationError)     */
#define HMX_ENOMEM 5    /* device memory budget exceeded                               */
#define HMX_EFACTOR 6   /* singular dense diagonal leaf in the H-LU (FactorizationError)  */

/* kernel kinds (KernelSpec variant) */
#define HMX_HELMHOLTZ 0 /* e^{i kappa r}/(4 pi r); kappa = 0 is Laplace, d = 1 */
#define HMX_ELASTO_U 1  /* displacement Green's tensor, d = 3                  */
#define HMX_ELASTO_T 2  /* traction tensor with column-point normals, d = 3    */

/* recompression truncation rules (oracle/lowrank.py decision 8) */
#define HMX_TRUNC_FROBENIUS 0
#define HMX_TRUNC_SPECTRAL 1

/* ACA kernel selection for the wide (m + n >= 320 points) d = 3 leaves */
#define HMX_ACA_KERNEL_AUTO 0      /* tensor-core (DMMA) ACA, CUDA-core when its ring does not fit */
#define HMX_ACA_KERNEL_CUDA_CORE 1 /* CUDA-core ACA only                                          */

/* memory location of vector arguments */
#define HMX_HOST 0
#define HMX_DEVICE 1

typedef struct hmx_ctx hmx_ctx;
typedef struct hmx_tree hmx_tree;
typedef struct hmx_blocks hmx_blocks;
typedef struct hmx_hmatrix hmx_hmatrix;

typedef struct {
  int32_t kind;  /* HMX_HELMHOLTZ / HMX_ELASTO_U / HMX_ELASTO_T */
  int32_t pad;
  double kappa;  /* Helmholtz wavenumber */
  double kp, ks; /* P / S wavenumbers */
  double lam, mu;
  double scale;  /* 1 / (rho omega^2) */
} hmx_kernel;

typedef struct {
  double eps;            /* eps_ACA (also the recompression tolerance) */
  int64_t max_rank;      /* <= 0: min(d m, d n) per block */
  double sigma3_floor;   /* relative sigma_3 floor, default 1e-12 */
  int32_t trunc_rule;    /* HMX_TRUNC_* */
  int32_t aca_kernel;    /* HMX_ACA_KERNEL_* */
  double mem_budget_gb;  /* ACA workspace budget; <= 0: 70% of free (+ cached) device memory */
  int32_t tc_stages;     /* tensor-core ACA copy ring depth: 0 = deepest that fits, 2 or 3 */
  int32_t pad;
  int64_t rsvd_seed;     /* seed of the Gaussian test matrices of the randomized-SVD fallback */
  double eps_recompress; /* truncation tolerance of the recompression; <= 0: eps (the reference) */
} hmx_aca_cfg;

typedef struct {
  int64_t n_blocks, n_dense, n_lowrank;
  int64_t n_stored;                /* stored complex entries N_s */
  int64_t max_rank_before, max_rank_after;
  int64_t aca_steps_total;
  int64_t pairs_evaluated;         /* point pairs fed to the Green's kernels */
  int64_t n_fallback, n_unconverged, n_regularized, aca_passes;
  int64_t row_elems, v_elems, n_levels, n_tiles, n_jobs;
  double t_dense_ms, t_aca_ms, t_recompress_ms, t_form_ms, t_total_ms;
  double flops_assembly;           /* algorithmic FP64 flops */
  double matvec_bytes;             /* algorithmic bytes of one matvec */
  double dense_bytes, lowrank_bytes;
  double phase1_bytes, phase2_bytes; /* algorithmic bytes of the two streaming kernels */
} hmx_stats;

int hmx_abi_version(void);
int hmx_last_error(char* buf, int64_t cap);

/* ---- context ------------------------------------------------------------- */
int hmx_ctx_create(int32_t device, hmx_ctx** out);
/* launch on an existing cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream; 0 = legacy default stream) */
int hmx_ctx_set_stream(hmx_ctx* ctx, uint64_t stream);
int hmx_ctx_sync(hmx_ctx* ctx);
/* release device memory cached by the context's stream-ordered pool */
int hmx_ctx_release_cache(hmx_ctx* ctx);
/* opt-in arena: reserve one device region (gigabytes; 0 = 88% of the free memory) that serves every
 * request of 1 MiB and more of this context by first fit, so neither repeated assemblies nor the first
 * assembly of a new problem size call cudaMalloc / cudaFree (whose cost is ~0.1-1 ms per GB depending on
 * the box: up to 0.35 s for T65k's 150 GB).  Requests that do not fit fall back to the ordinary path.
 * hmx_ctx_release_cache returns the region to the driver once no block lives in it.  seconds (may be
 * NULL): time taken. */
int hmx_ctx_reserve(hmx_ctx* ctx, double gigabytes, double* seconds);
int hmx_ctx_destroy(hmx_ctx* ctx);

/* ---- geometry (host, bit-exact with geometry.py) -------------------------- */
int hmx_tree_build(const double* points /* n x 3 */, int64_t n, int64_t n_leaf, hmx_tree** out);
int64_t hmx_tree_num_nodes(const hmx_tree* t);
/* perm: n; nodes: nn x 5 (start, stop, level, child0, child1); boxes: nn x 6 (lo, hi) -- preorder */
int hmx_tree_export(const hmx_tree* t, int64_t* perm, int64_t* nodes, double* boxes);
void hmx_tree_free(hmx_tree* t);
int hmx_blocks_build(const hmx_tree* rows, const hmx_tree* cols, double eta, hmx_blocks** out);
int64_t hmx_blocks_count(const hmx_blocks* b);
/* table: nb x 7 (kind 0 dense / 1 admissible, r0, r1, c0, c1, row node, col node), leaves() order */
int hmx_blocks_export(const hmx_blocks* b, int64_t* table);
void hmx_blocks_free(hmx_blocks* b);

/* ---- kernel-core seam ------------------------------------------------------- */
/* out: (d m) x (d n) complex row-major.  has_shift = 0 and an r == 0 pair -> HMX_ESINGULAR */
int hmx_eval_block(hmx_ctx* ctx, const hmx_kernel* k, const double* X, int64_t m, const double* Y, int64_t n,
                   const double* NY, int32_t has_shift, double shift, double* out);

/* ---- assembly --------------------------------------------------------------- */
/* pts_tree / nrm_tree: points (normals, T only) already in cluster-tree order;
 * perm: tree slot -> original index; table: nb x 5 (kind, r0, r1, c0, c1). */
int hmx_assemble(hmx_ctx* ctx, const hmx_kernel* k, const double* pts_tree, const double* nrm_tree, int64_t n_points,
                 const int64_t* perm, const int64_t* table, int64_t nb, const hmx_aca_cfg* cfg, double self_shift,
                 hmx_hmatrix** out);
/* build an H-matrix from given payloads (parity / snapshot import):
 * dense leaf b: a[b] = (d m) x (d n) row-major; low-rank leaf: a[b] = U (d m) x r, b[b] = V (d n) x r row-major */
int hmx_hmatrix_load(hmx_ctx* ctx, int32_t d, int64_t n_points, const int64_t* perm, const int64_t* table, int64_t nb,
                     const int64_t* ranks, const double* const* a, const double* const* b, hmx_hmatrix** out);
int hmx_hmatrix_stats(const hmx_hmatrix* h, hmx_stats* st);
/* per leaf: ACA steps, rank before / after recompression, flags (bit0 converged, bit1 max_rank,
 * bit3 fallback, bit4 Cholesky regularised, bit5 QL eigen fallback, bit6 QL not converged) */
int hmx_hmatrix_block_info(const hmx_hmatrix* h, int64_t* steps, int64_t* rank_before, int64_t* rank_after,
                           int32_t* flags);
/* restore the per-leaf assembly record of an imported H (snapshot load): ACA steps,
 * rank before recompression (>= the stored rank) and flags; any pointer may be NULL (left unchanged) */
int hmx_hmatrix_set_block_info(hmx_hmatrix* h, const int64_t* steps, const int64_t* rank_before,
                               const int32_t* flags);
/* copy leaf b out (layouts as in hmx_hmatrix_load) */
int hmx_hmatrix_get_block(const hmx_hmatrix* h, int64_t b, double* a, double* v);
/* zero-copy device view of the leaf payloads (input of the H-LU, which the reference's
 * hmatrix module runs on its in-memory per-leaf payloads): per leaf b the offset of its dense block / U
 * columns in the row stream (column-major, leading dimension ld[b]) and of its V columns in the V stream
 * (column-major, leading dimension d n); bufs = {row stream device pointer, row elements, V stream device
 * pointer, V elements} (complex128 elements).  The views stay valid while h lives and must not be written. */
int hmx_hmatrix_device_layout(const hmx_hmatrix* h, int64_t* moff, int64_t* ld, int64_t* voff, uint64_t* bufs);
/* delta_{H,F} estimator kernel (SPEC.md:507-515 estimate(): "for each AdmissibleLeaf regenerate the
 * dense block from the kernel, accumulate ||A_block - U V*||_F^2").  Per leaf b:
 * err2[b] = ||A_b - U_b V_b^H||_F^2 (0 for dense leaves), norm2[b] = ||A_b||_F^2 of the regenerated
 * block (dense leaves include the self shift).  pts_tree / nrm_tree as in hmx_assemble. */
int hmx_block_errors(hmx_hmatrix* h, const hmx_kernel* k, const double* pts_tree, const double* nrm_tree,
                     int64_t n_points, double self_shift, double* err2, double* norm2);
void hmx_hmatrix_free(hmx_hmatrix* h);

/* ---- low-rank layer, one block at a time ------------------------ */
/* aca_partial (d = 1) / aca_vector (d = 3) on the block generator of (X, Y, NY) with the same device kernel
 * and pinned decisions as hmx_assemble; recompress != 0 also applies recompress
 * (SPEC.md:318-326).  U: (d m) x cap, V: (d n) x cap complex row-major (first *rank columns filled);
 * *status: bit0 converged, bit1 max_rank reached, bit3 fallback needed (returns HMX_EPIVOT). */
int hmx_aca_block(hmx_ctx* ctx, const hmx_kernel* k, const double* X, int64_t m, const double* Y, int64_t n,
                  const double* NY, int32_t has_shift, double shift, const hmx_aca_cfg* cfg, int32_t recompress,
                  int64_t cap, double* U, double* V, int64_t* rank, int64_t* steps, int32_t* status);
/* recompress(f, eps) of U (dm x K), V (dn x K) complex row-major -> Uout (dm x K),
 * Vout (dn x K) row-major with leading dimension *rank <= K */
int hmx_recompress(hmx_ctx* ctx, int64_t dm, int64_t dn, int64_t K, const double* U, const double* V, double eps,
                   int32_t trunc_rule, int64_t* rank, double* Uout, double* Vout);

/* New H-matrix = base with leaf idx[j] replaced by leaf j of sub (same leaf, e.g. re-compressed at
 * a tighter tolerance by the certification pass of ACAConfig(certify=True)); both inputs unchanged.
 * Device-side copy of every payload into a freshly laid out stream pair. */
int hmx_hmatrix_splice(const hmx_hmatrix* base, const hmx_hmatrix* sub, const int64_t* idx, hmx_hmatrix** out);

/* randomized_svd(dense, eps, oversample) (the FallbackNeeded path of aca_vector,
 * SPEC.md:302, 384-385): adaptive Gaussian range finder on a dense (m x n) complex row-major block A,
 * columns 8 + oversample, doubling until ||A - Q Q^H A||_F <= eps ||A||_F or the cap
 * min(max_rank, m, n) is reached (*converged = 0, a flagged result).  Writes U = Q (m x *k) and
 * V = (Q^H A)^H (n x *k), row-major with leading dimension *k; U and V hold cap columns.  The same
 * device routine compresses the flagged leaves inside hmx_assemble. */
int hmx_rsvd(hmx_ctx* ctx, const double* A, int64_t m, int64_t n, double eps, int32_t oversample, int64_t max_rank,
             int64_t seed, double* U, double* V, int64_t* k, int32_t* converged);

/* ---- H-matvec / GMRES ---------------------------------------------------------- */
/* y = A_H x, x and y in ORIGINAL point order (d N complex each) */
/* Batched truncation of accumulated low-rank sums on the device (the recompress of SPEC.md:318-326
 * applied to the addends that formatted_addmul collects on a low-rank target; used by
 * the H-LU).  Item i: U_i (dm_i x K_i) and V_i (dn_i x K_i), complex128, column-major, device pointers.
 * Writes U'_i = U_i W_U (dm_i x r_i) and V'_i = V_i W_V (dn_i x r_i) column-major into Uo_i / Vo_i
 * (capacity K_i columns, leading dimensions dm_i / dn_i) with U'_i V'_i^H the rank-r_i truncation of
 * U_i V_i^H (same Gram / Cholesky / Hermitian eigen-solver and truncation rule as hmx_assemble);
 * r_i -> ranks (host).  K_i <= 1020.  flags_i bit 0: the Cholesky of V_i^H V_i needed regularisation
 * (V_i numerically rank-deficient); such an item is NOT formed and the caller re-submits it in a
 * well-conditioned form (e.g. (U_i V_i^H, I)).  Launches on the context stream and returns once the
 * ranks are known (one host synchronisation per batch). */
int hmx_truncate_batch(hmx_ctx* ctx, int64_t nb, const int64_t* dm, const int64_t* dn, const int64_t* K,
                       const uint64_t* U, const uint64_t* V, const uint64_t* Uo, const uint64_t* Vo, double eps,
                       int32_t trunc_rule, int64_t* ranks, int32_t* flags);
int hmx_matvec(hmx_hmatrix* h, const double* x, double* y, int32_t mem);
/* the same on an explicit cudaStream_t (0 = legacy default stream).  Concurrency (an
 * assembled H is immutable and safe for concurrent matvec): the H is only read; every buffer a matvec
 * writes belongs to a per-stream workspace of the H (created on first use of a stream), so calls on
 * different streams run concurrently and calls from several host threads on one stream are serialised
 * by a per-workspace lock while they enqueue.  mem = HMX_DEVICE: asynchronous on `stream`;
 * HMX_HOST: returns once y is on the host.  hmx_matvec = hmx_matvec_on with the context stream. */
int hmx_matvec_on(hmx_hmatrix* h, const double* x, double* y, int32_t mem, uint64_t stream);
/* device pointers; phase_ms[4] = gather, phase 1 (V^H x), phase 2 (row GEMV), finalize */
int hmx_matvec_profile(hmx_hmatrix* h, const double* x_dev, double* y_dev, float* phase_ms);
/* live kernel timing: every matvec between begin and end records CUDA events
 * around its 4 phases on the launch stream (no extra synchronisation);
 * end returns the number of calls and the summed per-phase milliseconds */
int hmx_profile_begin(hmx_hmatrix* h);
int hmx_profile_end(hmx_hmatrix* h, int64_t* n_calls, double* phase_ms_sum);
/* FP64 DFMA throughput of the device (TFLOP/s), measured by a dependent-chain microkernel */
int hmx_bench_dfma(hmx_ctx* ctx, double* tflops);
/* read-only HBM streaming rate (GB/s), 4 GiB buffer, 16-byte streaming loads: the ceiling of read-dominated kernels */
int hmx_bench_read_bw(hmx_ctx* ctx, double* gbs);
int hmx_gmres(hmx_hmatrix* h, const double* b, double* x, double tol, int32_t restart, int64_t max_iters,
              int32_t mem, int64_t* iters, double* history, int64_t history_cap, int64_t* history_len,
              int32_t* converged);

/* ---- H-LU engine: formatted H-arithmetic, hlu, triangular solves ----------
 * Replaces the reference's hmatx.hmatrix.formatted_addmul / hlu / triangular_solve and
 * hmatx.solve.solve_direct (the module itself is absent from the mount,
 * SURVEY 0.2).  An hmx_hlu is a device factor tree over a block tree (geometry.py:277-295): dense,
 * low-rank (U V^H) and hierarchical nodes, every matrix complex128 column-major in HBM, driven from C++
 * over cuBLAS / cuSOLVER and the assembly's truncation kernels.
 *
 * Tree descriptor: nnodes rows of 8 int64 in preorder (a hierarchical node's children follow it, grid
 * row-major): kind (0 dense, 1 low-rank, 2 hierarchical, 3 low-rank from a dense block: truncated SVD
 * with eps / rule), r0, r1, c0, c1 (dof ranges, tree order), nr, nc (grid of a hierarchical node),
 * extra (dense: 1 = factored, the block is the packed LU of getrf with pivots; low-rank: rank).
 * Payload: one row of 5 uint64 per leaf, preorder: dense (p0 = block, ld0 [, p4 = int64 pidx with
 * P^T X = X[pidx] when factored]); low-rank (p0 = U, ld0, p1 = V, ld1); kind 3 (p0 = block, ld0).
 * Device pointers; hmx_hlu_build copies them (the caller's buffers may be freed afterwards). */
typedef struct hmx_hlu hmx_hlu;
typedef struct {
  int64_t n_truncations, n_truncate_calls, n_getrf, max_rank, dense_image_bytes, k_p50, k_p90, k_max;
  double t_truncate_s, t_factor_s;
} hmx_hlu_stats;
int hmx_hlu_build(hmx_ctx* ctx, int64_t nnodes, const int64_t* desc, const uint64_t* payload, double eps,
                  int32_t trunc_rule, int32_t finished, hmx_hlu** out);
int hmx_hlu_count(const hmx_hlu* h, int64_t* nnodes, int64_t* nleaves);
/* the same descriptor / payload format (payload pointers into the tree's own storage, valid until the
 * tree is modified or freed) */
int hmx_hlu_export(const hmx_hlu* h, int64_t* desc, uint64_t* payload);
/* in-place recursive H-LU: LU(A11); U12 = L11^{-1} A12; L21 = A21 U11^{-1};
 * A22 -= L21 U12 (formatted, truncation eps); recurse.  HMX_EFACTOR on a singular dense diagonal leaf. */
int hmx_hlu_factor(hmx_hlu* h, double eps, int32_t trunc_rule, hmx_hlu_stats* st);
/* mode 0: Y = U_H^{-1} L_H^{-1} X; mode 1: Y = L_H U_H X.  X, Y: device, n x nrhs
 * column-major, tree order. */
int hmx_hlu_apply(hmx_hlu* h, int32_t mode, const double* X, double* Y, int64_t n, int64_t nrhs);
/* target <- target + alpha a b in the H-format of target, low-rank targets truncated with eps */
int hmx_hlu_addmul(hmx_hlu* target, hmx_hlu* a, hmx_hlu* b, double alpha, double eps, int32_t trunc_rule);
/* dense image (device, column-major, leading dimension ld) */
int hmx_hlu_to_dense(hmx_hlu* h, double* out, int64_t ld);
/* the engine's truncation of factor pairs (direct / dense-form / range-sketch / QR + SVD routes):
 * U_i (dm_i x K_i), V_i (dn_i x K_i) column-major device -> r_i columns written into Uo_i / Vo_i
 * (capacity K_i columns, ld = dm_i / dn_i). */
int hmx_hlu_truncate(hmx_ctx* ctx, int64_t nb, const int64_t* dm, const int64_t* dn, const int64_t* K,
                     const uint64_t* U, const uint64_t* V, const uint64_t* Uo, const uint64_t* Vo, double eps,
                     int32_t trunc_rule, int64_t* ranks);
/* trim the engine's memory pool */
int hmx_hlu_release(hmx_ctx* ctx);
void hmx_hlu_free(hmx_hlu* h);

#ifdef __cplusplus
}
#endif

#endif /* HMX_H_ */
