// Internal device-side H-matrix representation and cross-module entry points.
//
// HBM layout:
//  * row stream  -- every leaf's row-side payload grouped by ROW SEGMENT (all
//    leaves sharing one row cluster [r0, r1)).  Segment g is ONE column-major
//    (d m_g) x C_g complex128 matrix: the dense leaves' (d m) x (d n) blocks and
//    the low-rank leaves' U factors (d m) x r side by side.
//  * V stream    -- low-rank V factors, (d n) x r column-major per leaf.
//  * source slots s (length sum_g C_g) -- per matvec, dense slots get the
//    leaf's x piece, low-rank slots get t = V^H x.  Phase 2 is then a plain
//    batched GEMV y_g += M_g s_g per segment, written (non-atomically) to a
//    per-level partial vector; a last pass sums the levels in fixed order and
//    scatters through the cluster-tree permutation -> deterministic y.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "green.cuh"

namespace hmx {

struct Ctx {
  int device = 0;
  cudaMemPool_t pool = nullptr;  // stream-ordered pool, never released to the driver between assemblies
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;  // second stream for concurrent launches inside assembly
  cudaStream_t rerun = nullptr;  // high-priority stream for ACA capacity-overflow reruns
  cudaStream_t side = nullptr;   // the large-K recompression class next to the classes that follow it
  bool own_stream = false;
  int num_sms = 148;
  size_t l2_bytes = 0;
  // caching allocator: freed device blocks are kept (by size) and reused by
  // later allocations of the context instead of cudaFree / cudaMalloc
  std::mutex mem_mu;
  std::multimap<size_t, void*> cache;  // size -> free block
  std::unordered_map<void*, size_t> live;  // block -> size
  size_t cached_bytes = 0;
  // opt-in arena (hmx_ctx_reserve): one reserved device region serving the large requests of every
  // assembly by first fit (free list by offset, coalescing), so steady-state and first assemblies
  // of a new problem size make no cudaMalloc / cudaFree call at all
  char* arena = nullptr;
  size_t arena_size = 0, arena_free = 0;
  std::map<size_t, size_t> arena_holes;             // offset -> length
  std::unordered_map<void*, size_t> arena_live;     // block -> length
  void* blas = nullptr;    // cublasHandle_t of the randomized-SVD fallback (rsvd.cu), lazy
  void* solver = nullptr;  // cusolverDnHandle_t, lazy
  cudaMemPool_t lu_pool = nullptr;  // stream-ordered pool of the H-LU engine (hlu.cu), lazy
};

// phase-1 job: one warp computes s[soff] = V[voff : voff+len]^H x_tree[xoff : xoff+len]
// (kind 1) or copies x_tree[xoff : xoff+len] -> s[soff : soff+len] (kind 0)
struct MvJob1 {
  int64_t voff;
  int64_t xoff;
  int64_t soff;
  int32_t len;
  int32_t kind;
};

// phase-2 tile: rows [row0, row0 + nrows) of segment g
struct MvTile2 {
  int64_t moff;    // segment matrix offset in the row stream
  int64_t soff;    // segment source offset
  int64_t yoff;    // level-buffer offset of the segment's first row (level * n + d * r0)
  int32_t ld;      // d * m_g
  int32_t ncols;   // C_g
  int32_t row0;    // first row of this tile inside the segment
  int32_t nrows;
};

// Per-stream scratch of the matvec (an assembled H is immutable and
// safe for concurrent matvec).  The H itself is read-only during a matvec; every
// buffer a matvec writes lives here, one workspace per launch stream, so calls on
// different streams never share memory and calls on one stream are ordered by it.
// `mu` is held while a call enqueues its kernels (two host threads on one stream
// cannot interleave their launches) and, for host-pointer calls, until the result
// is back on the host (the staging buffers).
struct MvWorkspace {
  cudaStream_t stream = nullptr;
  double2* d_s = nullptr;     // source slots
  double2* d_xt = nullptr;    // x in tree order
  double2* d_ylev = nullptr;  // nlevels x n partial y (rows no tile writes stay 0)
  double2* d_xio = nullptr;   // device staging for host x / y
  double2* d_yio = nullptr;
  cudaEvent_t done = nullptr;  // recorded after every call (freeing the H waits on it)
  std::mutex mu;
};

struct DeviceH {
  Ctx* ctx = nullptr;
  int kind = 0, d = 1;
  int64_t np = 0, n = 0;  // points, dofs
  int64_t nb = 0;
  std::vector<int64_t> table;  // nb x 5 (kind, r0, r1, c0, c1)
  std::vector<int64_t> steps, rank_before, rank_after;
  std::vector<int32_t> flags;
  // row-stream placement of every leaf (for export)
  std::vector<int64_t> leaf_moff, leaf_ld, leaf_voff;
  int64_t nlevels = 1;

  int64_t* d_perm = nullptr;
  double2* d_row = nullptr;  // row stream
  int64_t row_elems = 0;
  double2* d_v = nullptr;  // V stream
  int64_t v_elems = 0;
  int64_t s_elems = 0;
  // matvec scratch, one workspace per launch stream (created on first use)
  std::mutex ws_mu;
  std::vector<std::unique_ptr<MvWorkspace>> ws;
  MvJob1* d_job1 = nullptr;
  int64_t njob1 = 0;
  MvTile2* d_tile2 = nullptr;
  int64_t ntile2 = 0;
  int32_t* d_lev_cover = nullptr;  // unused placeholder
  // algorithmic traffic of one matvec (bytes), SURVEY 8(d)
  double mv_bytes = 0;
  double dense_bytes = 0, lr_bytes = 0;
  // assembly statistics
  double t_dense_ms = 0, t_aca_ms = 0, t_recomp_ms = 0, t_form_ms = 0, t_total_ms = 0;
  int64_t pairs_evaluated = 0;
  int64_t aca_passes = 0, n_fallback = 0, n_unconverged = 0, n_regularized = 0;
  double flops_assembly = 0;
  // live per-phase timing of matvec calls (hmx_profile_begin / _end)
  bool profiling = false;
  std::vector<cudaEvent_t> prof_events;  // 5 per profiled call
  double phase1_bytes = 0, phase2_bytes = 0;
};

// capi.cu: stream-ordered device memory from the context pool (no device-wide
// synchronisation, memory reused across assemblies instead of re-mapped)
void release_cache(Ctx& c);
cudaError_t dev_alloc(Ctx& c, void** p, size_t bytes);
void dev_free(Ctx& c, void* p);
template <class T>
cudaError_t dev_alloc_t(Ctx& c, T** p, size_t count) {
  return dev_alloc(c, reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1));
}
// per-file kernel warm-up (forces lazy module loading at context creation)
void warm_aca();
void warm_recompress();
void warm_dense();
void warm_matvec();
void warm_gmres();
void warm_estimate();

// matvec.cu
// Rank-independent part of the matvec plan (row segments, nesting levels);
// hmx_assemble builds it on the host while the ACA kernels run.
struct PlanPre {
  std::vector<std::pair<int64_t, int64_t>> segs;  // (r0, r1) per row segment, nesting order
  std::vector<int64_t> bseg;                      // leaf -> segment
  std::vector<int64_t> level;                     // segment -> nesting level
  int64_t nlevels = 0;
};
void build_plan_pre(const DeviceH& H, PlanPre& pre);
int build_matvec_plan(DeviceH& H, const PlanPre* pre = nullptr);
// the workspace of launch stream s (created on first use); nullptr + error set on failure
MvWorkspace* mv_workspace(DeviceH& H, cudaStream_t s, int* rc);
void free_workspaces(DeviceH& H);
// y = A_H x on stream s (device pointers); takes the stream's workspace lock while enqueueing
// (gate: optional device flag, the launches do nothing while *gate == 0)
int matvec_device(DeviceH& H, const double2* x_orig_dev, double2* y_orig_dev, float* phase_ms, cudaStream_t s,
                  const int* gate = nullptr);
// same with the workspace already locked by the caller
int matvec_enqueue(DeviceH& H, MvWorkspace& w, const double2* x_orig_dev, double2* y_orig_dev, float* phase_ms,
                   const int* gate = nullptr);

// dense.cu
int launch_dense_fill(Ctx& c, const GreenParams& P, const PointsSoA& pts, const int64_t* d_desc, int64_t ndense,
                      double2* row_stream, int32_t* d_err);
int launch_eval_block(Ctx& c, const GreenParams& P, const PointsSoA& X, const PointsSoA& Y, int64_t m, int64_t n,
                      double2* out, int32_t* d_err);

// aca.cu
struct AcaDesc {
  int64_t r0, c0;       // first row / column point (tree order)
  int32_t m, n;         // points
  int32_t kcap;         // column capacity of U / V
  int32_t max_rank;     // in scalar columns
  int64_t uoff, voff;   // workspace offsets (ld = d m, d n)
  int64_t goff;         // Gram workspace offset (two kcap x kcap matrices)
};
struct AcaOut {
  int32_t steps;
  int32_t rank;      // d * steps
  int32_t status;    // bit0 converged, bit1 max_rank, bit2 capacity overflow, bit3 fallback needed
  int32_t zero_rows;
};
// launch variants of the ACA kernel; leaves with m + n < kAcaNarrowMax points use
// the narrow variant (128 threads, 4 CTAs / SM), the others the wide one (512)
constexpr int kAcaWide = 0;
constexpr int kAcaNarrow = 1;
#ifndef HMX_ACA_NARROW_MAX
#define HMX_ACA_NARROW_MAX 320
#endif
constexpr int kAcaNarrowMax = HMX_ACA_NARROW_MAX;
// tensor-core variant for large d = 3 leaves (default; HMX_ACA_TC=0 disables); its
// per-warp Gram scratch sits behind the leaf's Gram pair: aca_tc_scratch(kcap) complex
constexpr int kAcaTensor = 2;
inline int64_t aca_tc_scratch(int64_t kcap) { return 16 * ((kcap + 7) / 8) * 64; }
int launch_aca(Ctx& c, int d, const GreenParams& P, const PointsSoA& pts, const AcaDesc* d_desc, const int32_t* d_order,
               int64_t nblk, int kcap_max, int m_max, double eps, double sigma3_floor, double2* U, double2* V,
               double2* G, AcaOut* d_out, int variant, int tc_stages);
// Routing of the admissible leaves between the ACA kernels: leaves with m + n >= wide_min points
// are "wide" (auxiliary stream; tensor-core kernel with its Gram scratch when use_tc, else the
// 512-thread CUDA-core kernel), the rest narrow.  hmx_assemble derives BOTH the workspace plan and
// the launch split from this one value.
struct AcaRoute {
  int64_t wide_min;
  bool use_tc;
  int tc_stages;  // 0: deepest ring that fits in shared memory
};
inline AcaRoute aca_route(int d, const hmx_aca_cfg* cfg) {
  AcaRoute r;
  r.wide_min = kAcaNarrowMax;
  r.use_tc = d == 3 && cfg->aca_kernel != HMX_ACA_KERNEL_CUDA_CORE;
  r.tc_stages = cfg->tc_stages;
  return r;
}

// recompress.cu
// recompress_core keeps E and the QL eigenvector matrix in shared memory up to this ACA rank
constexpr int kRecompressSmemMax = 112;
// ... and R, T / L_r as well (3 K^2 complex) up to this one
constexpr int kRecompressAllSmemMax = 0;  // measured no faster
struct RecDesc {
  int64_t goff;      // Gram pair (G_U at goff, G_V at goff + kcap*kcap), ld = kcap
  int64_t woff;      // K x K scratch workspace (2 matrices) offset
  int32_t K;         // ACA rank
  int32_t kcap;
};
int launch_recompress_core(Ctx& c, const RecDesc* d_desc, int64_t nblk, int kmax, double eps, int rule, double2* G,
                           double2* W, int32_t* d_rank, int32_t* d_flags);
struct FormDesc {
  const double2* A;  // source factor (U or V workspace), ld = lda
  const double2* W;  // K x r coefficient matrix (ld = K)
  double2* C;        // destination slot in the row stream or V stream, ld = ldc
  int32_t rows, K, r, lda, ldc;
  int32_t pad;
};
int launch_form(Ctx& c, const FormDesc* d_desc, int64_t nitems, int64_t ntiles_total, const int64_t* d_tile_start);

// estimate.cu: per-leaf ||A_b - U V^H||_F^2 and ||A_b||_F^2 by regeneration
struct ErrDesc {
  int64_t r0, c0;        // first row / column point (tree order)
  int32_t m, n, r, pad;  // points, rank (0: dense leaf -> norm only)
  const double2* U;      // d m x r, ld = ldu
  const double2* V;      // d n x r, ld = d n
  int64_t ldu;
};
int launch_block_errors(Ctx& c, int d, const GreenParams& P, const PointsSoA& pts, const ErrDesc* d_desc,
                        const int64_t* d_tile_start, int64_t nleaves, int64_t ntiles, double2* d_part,
                        double2* d_out);
int64_t err_tiles_of(int64_t m, int64_t n);

// dense.cu: FP64 peak microbenchmark
int bench_dfma(Ctx& c, double* tflops);
int bench_read_bw(Ctx& c, double* gbs);

// rsvd.cu: randomized-SVD fallback of the vector ACA.  A: m x n column-major
// dense block; U (m x cap), V (n x cap), G (2 cap^2) outputs: K columns, Gram pair at ld = K.
int rsvd_dense(Ctx& c, const double2* A, int64_t m, int64_t n, double eps, int oversample, int64_t cap, uint64_t seed,
               double2* U, double2* V, double2* G, int* K_out, int* converged);
int linalg_handles(Ctx& c, void** blas, void** solver);
// counter-based complex Gaussian fill (g1 + i g2, g ~ N(0, 1)) of `count` entries with `key`
int launch_gaussian(Ctx& c, double2* out, int64_t count, uint64_t key);

// capi.cu: batched truncation of factor pairs (hmx_truncate_batch and the H-LU engine).  Items:
// U_i (dm_i x K_i), V_i (dn_i x K_i) column-major with ld = rows, K_i <= 1020.  After the rank
// readback `outputs(ranks, flags, Uo, Vo)` fills the destinations (ld = rows, >= r_i columns) of
// every item with r_i > 0 and flags_i bit 0 clear; the U' / V' products are then launched on
// c.stream (not waited for).
using TruncOutputs = std::function<int(const int64_t* ranks, const int32_t* flags, double2** Uo, double2** Vo)>;
int truncate_pairs(Ctx& c, int64_t nb, const int64_t* dm, const int64_t* dn, const int64_t* K,
                   const double2* const* U, const double2* const* V, double eps, int32_t trunc_rule, int64_t* ranks,
                   int32_t* flags, const TruncOutputs& outputs);
void hlu_pool_destroy(Ctx& c);
void linalg_destroy(Ctx& c);

// gmres.cu
int gmres_device(DeviceH& H, const double2* b_dev, double2* x_dev, double tol, int restart, int64_t max_iters,
                 int64_t* iters, std::vector<double>& history, int* converged, cudaStream_t s);

}  // namespace hmx

struct hmx_ctx {
  hmx::Ctx c;
};
