// C-ABI of libhmx.so (include/hmx.h) and the device assembly pipeline.
//
// hmx_assemble on the device:
//   1. batched ACA over all admissible leaves (aca.cu), capacity-budgeted
//      workspaces; leaves that outgrow their column capacity are re-run in a
//      further pass with twice the capacity (deterministic -> same result);
//   2. recompression core per leaf (recompress.cu) -> rank r and the K x r
//      coefficient matrices W_U, W_V;
//   3. stream layout + matvec plan from the final ranks (matvec.cu);
//   4. dense leaves evaluated straight into the row stream (dense.cu) and
//      U' = U W_U, V' = V W_V formed straight into the row / V streams.
#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <cmath>
#include <cstring>
#include <string>
#include <map>
#include <unordered_map>
#include <vector>

#include "../../include/hmx.h"
#include "hmatrix.h"
#include "hmx_host.h"

static thread_local std::string g_last_error;

void hmx_set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}


namespace hmx {
void release_cache(Ctx& c) {
  std::lock_guard<std::mutex> lk(c.mem_mu);
  for (auto& kv : c.cache) cudaFree(kv.second);
  c.cache.clear();
  c.cached_bytes = 0;
  if (c.arena && c.arena_live.empty()) {  // the reserved region too, once nothing lives in it
    cudaFree(c.arena);
    c.arena = nullptr;
    c.arena_size = c.arena_free = 0;
    c.arena_holes.clear();
  }
}
constexpr size_t kArenaGran = size_t(2) << 20;  // 2 MiB blocks
constexpr size_t kArenaMin = size_t(1) << 20;   // smaller requests take the ordinary path
static void* arena_alloc(Ctx& c, size_t bytes) {
  bytes = (bytes + kArenaGran - 1) / kArenaGran * kArenaGran;
  for (auto it = c.arena_holes.begin(); it != c.arena_holes.end(); ++it) {  // first fit by offset
    if (it->second < bytes) continue;
    const size_t off = it->first, len = it->second;
    c.arena_holes.erase(it);
    if (len > bytes) c.arena_holes.emplace(off + bytes, len - bytes);
    c.arena_free -= bytes;
    void* p = c.arena + off;
    c.arena_live[p] = bytes;
    return p;
  }
  return nullptr;
}
static bool arena_release(Ctx& c, void* p) {
  auto it = c.arena_live.find(p);
  if (it == c.arena_live.end()) return false;
  size_t off = (size_t)(static_cast<char*>(p) - c.arena), len = it->second;
  c.arena_live.erase(it);
  c.arena_free += len;
  auto nx = c.arena_holes.lower_bound(off);
  if (nx != c.arena_holes.end() && off + len == nx->first) {  // merge with the hole behind
    len += nx->second;
    nx = c.arena_holes.erase(nx);
  }
  if (nx != c.arena_holes.begin()) {  // ... and with the one in front
    auto pv = std::prev(nx);
    if (pv->first + pv->second == off) {
      off = pv->first;
      len += pv->second;
      c.arena_holes.erase(pv);
    }
  }
  c.arena_holes.emplace(off, len);
  return true;
}
cudaError_t dev_alloc(Ctx& c, void** p, size_t bytes) {
  if (c.pool) return cudaMallocFromPoolAsync(p, bytes, c.pool, c.stream);
  if (c.arena && bytes >= kArenaMin) {
    std::lock_guard<std::mutex> lk(c.mem_mu);
    if (void* q = arena_alloc(c, bytes)) {
      *p = q;
      return cudaSuccess;
    }
  }
  // 2 MiB granularity so that repeated assemblies hit the cache
  const size_t gran = bytes >= (1u << 20) ? (size_t(2) << 20) : 256;
  bytes = (bytes + gran - 1) / gran * gran;
  {
    std::lock_guard<std::mutex> lk(c.mem_mu);
    auto it = c.cache.lower_bound(bytes);
    if (it != c.cache.end() && it->first <= 2 * bytes + (size_t(4) << 20)) {
      *p = it->second;
      c.live[*p] = it->first;
      c.cached_bytes -= it->first;
      c.cache.erase(it);
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and retry once
    cudaGetLastError();
    release_cache(c);
    e = cudaMalloc(p, bytes);
  }
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(c.mem_mu);
    c.live[*p] = bytes;
  }
  return e;
}
void dev_free(Ctx& c, void* p) {
  if (!p) return;
  if (c.pool) {
    cudaFreeAsync(p, c.stream);
    return;
  }
  // stream-ordered reuse: every later use of a cached block is issued on the
  // context stream after the work that used it (assembly joins its auxiliary
  // stream before freeing), so no device synchronisation is needed here
  std::lock_guard<std::mutex> lk(c.mem_mu);
  if (c.arena && arena_release(c, p)) return;
  auto it = c.live.find(p);
  if (it == c.live.end()) {
    cudaFree(p);
    return;
  }
  c.cache.emplace(it->second, p);
  c.cached_bytes += it->second;
  c.live.erase(it);
}
}  // namespace hmx
struct hmx_tree {
  hmx::ClusterTree t;
};
struct hmx_blocks {
  std::vector<hmx::BlockLeaf> v;
};
struct hmx_hmatrix {
  hmx::DeviceH H;
};

namespace {

using namespace hmx;

constexpr int kMaxAcaCols = 1020;  // per-leaf ACA column limit (recompress.cu vector sizes)
constexpr int kRsvdOversample = 10;  // oversampling of the randomized-SVD fallback (oracle/lowrank.py)
// share of (free + cached) HBM for the ACA workspaces U, V, G: the Grams are released
// before the final streams are allocated, so U + V + streams stay well inside 180 GB
constexpr double kAcaBudgetFrac = 0.7;

GreenParams make_params(const hmx_kernel* k, int has_shift, double shift) {
  GreenParams P;
  P.kind = k->kind;
  P.kappa = k->kappa;
  P.kp = k->kp;
  P.ks = k->ks;
  P.lam = k->lam;
  P.mu = k->mu;
  P.scale = k->scale;
  P.shift = shift;
  P.has_shift = has_shift;
  return P;
}

// device SoA copy of (n x 3) points (+ normals)
struct DevPoints {
  Ctx* ctx = nullptr;
  double* buf = nullptr;
  PointsSoA soa{};
  ~DevPoints() {
    if (buf) dev_free(*ctx, buf);
  }
  int upload(Ctx& c, const double* pts, const double* nrm, int64_t n) {
    const int nc = nrm ? 6 : 3;
    std::vector<double> h((size_t)nc * n);
    for (int64_t i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) {
        h[(size_t)k * n + i] = pts[3 * i + k];
        if (nrm) h[(size_t)(3 + k) * n + i] = nrm[3 * i + k];
      }
    ctx = &c;
    HMX_CUDA_TRY(dev_alloc(c, reinterpret_cast<void**>(&buf), sizeof(double) * h.size() + 8));
    HMX_CUDA_TRY(cudaMemcpyAsync(buf, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, c.stream));
    HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
    soa.x = buf;
    soa.y = buf + n;
    soa.z = buf + 2 * n;
    soa.nx = nrm ? buf + 3 * n : nullptr;
    soa.ny = nrm ? buf + 4 * n : nullptr;
    soa.nz = nrm ? buf + 5 * n : nullptr;
    return HMX_OK;
  }
};

template <class T>
int dev_upload(Ctx& c, T** dst, const std::vector<T>& src) {
  HMX_CUDA_TRY(dev_alloc_t(c, dst, src.size()));
  if (!src.empty())
    HMX_CUDA_TRY(cudaMemcpyAsync(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, c.stream));
  return HMX_OK;
}

struct DevBuf {
  Ctx* ctx = nullptr;
  std::vector<void*> p;
  explicit DevBuf(Ctx& c) : ctx(&c) {}
  DevBuf(DevBuf&& o) noexcept : ctx(o.ctx), p(std::move(o.p)) { o.p.clear(); }
  DevBuf(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    for (void* q : p) dev_free(*ctx, q);
    p.clear();
  }
  template <class T>
  int alloc(T** out, int64_t count) {
    void* q = nullptr;
    cudaError_t e = dev_alloc(*ctx, &q, sizeof(T) * std::max<int64_t>(count, 1));
    if (e != cudaSuccess) {
      size_t fr = 0, tot = 0;
      cudaGetLastError();
      cudaMemGetInfo(&fr, &tot);
      hmx_set_error("cudaMalloc(%lld bytes): %s (free %.2f GB of %.2f GB, context cache %.2f GB)",
                    (long long)(sizeof(T) * count), cudaGetErrorString(e), fr / 1e9, tot / 1e9,
                    ctx->cached_bytes / 1e9);
      return e == cudaErrorMemoryAllocation ? HMX_ENOMEM : HMX_ECUDA;
    }
    p.push_back(q);
    *out = static_cast<T*>(q);
    return HMX_OK;
  }
};

int recompress_device(Ctx& c, DevBuf& mem, const double2* dU, const double2* dV, int64_t dm, int64_t dn, int K,
                      double2* G, double eps, int rule, int* r_out, double2** Uo, double2** Vo);

void free_h(DeviceH& H) {
  free_workspaces(H);
  void* ptrs[] = {H.d_perm, H.d_row, H.d_v, H.d_job1, H.d_tile2};
  for (void* p : ptrs)
    if (p) dev_free(*H.ctx, p);
  H.d_perm = nullptr;
  H.d_row = H.d_v = nullptr;
  H.d_job1 = nullptr;
  H.d_tile2 = nullptr;
}

int validate_table(const int64_t* table, int64_t nb, int64_t np) {
  if (nb <= 0) {
    hmx_set_error("empty block list");
    return HMX_EINVAL;
  }
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t* t = table + 5 * b;
    if ((t[0] != 0 && t[0] != 1) || t[1] < 0 || t[2] <= t[1] || t[2] > np || t[3] < 0 || t[4] <= t[3] ||
        t[4] > np) {
      hmx_set_error("invalid block %lld: (%lld, %lld, %lld, %lld, %lld)", (long long)b, (long long)t[0],
                    (long long)t[1], (long long)t[2], (long long)t[3], (long long)t[4]);
      return HMX_EINVAL;
    }
  }
  return HMX_OK;
}

// batched strided copy (hmx_hmatrix_splice): one CTA per column block of a leaf payload
struct Copy2D {
  const double2* src;
  double2* dst;
  int64_t lds, ldd, rows, cols;
};
__global__ void __launch_bounds__(256) copy2d_batch(const Copy2D* __restrict__ items) {
  const Copy2D it = items[blockIdx.x];
  const int64_t total = it.rows * it.cols;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int64_t i = e % it.rows, j = e / it.rows;
    it.dst[i + j * it.ldd] = it.src[i + j * it.lds];
  }
}

// launches issued inside this scope go to the context's auxiliary stream
struct OnAux {
  Ctx& c;
  cudaStream_t saved;
  explicit OnAux(Ctx& cc) : c(cc), saved(cc.stream) { c.stream = c.aux; }
  ~OnAux() { c.stream = saved; }
};

struct AcaPass {
  explicit AcaPass(Ctx& c) : mem(c), gmem(c) {}
  DevBuf mem;   // U, V factor workspaces and the recompression W
  DevBuf gmem;  // Gram matrices: only needed until the recompression
  double2 *U = nullptr, *V = nullptr, *G = nullptr;
  std::vector<int64_t> blocks;  // block ids
  std::vector<AcaDesc> desc;
  std::vector<AcaOut> out;
  std::vector<double2*> wptr;  // per leaf: its W_U | W_V coefficients
  int kcap_max = 0;
};

}  // namespace

extern "C" {

int hmx_abi_version(void) { return HMX_ABI_VERSION; }

int hmx_last_error(char* buf, int64_t cap) {
  if (!buf || cap <= 0) return HMX_EINVAL;
  std::snprintf(buf, (size_t)cap, "%s", g_last_error.c_str());
  return HMX_OK;
}

int hmx_ctx_create(int32_t device, hmx_ctx** out) {
  if (!out) return HMX_EINVAL;
  int ndev = 0;
  HMX_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    hmx_set_error("device %d not available (%d devices)", device, ndev);
    return HMX_EINVAL;
  }
  HMX_CUDA_TRY(cudaSetDevice(device));
  auto* c = new hmx_ctx;
  c->c.device = device;
  cudaDeviceProp prop;
  HMX_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  c->c.num_sms = prop.multiProcessorCount;
  c->c.l2_bytes = prop.l2CacheSize;
  HMX_CUDA_TRY(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
  c->c.own_stream = true;
  HMX_CUDA_TRY(cudaStreamCreateWithFlags(&c->c.aux, cudaStreamNonBlocking));
  HMX_CUDA_TRY(cudaStreamCreateWithFlags(&c->c.side, cudaStreamNonBlocking));
  {
    int lo = 0, hi = 0;  // hi = greatest priority (numerically lowest)
    HMX_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    HMX_CUDA_TRY(cudaStreamCreateWithPriority(&c->c.rerun, cudaStreamNonBlocking, hi));
  }
  warm_aca();
  warm_recompress();
  warm_dense();
  warm_matvec();
  warm_gmres();
  warm_estimate();
  *out = c;
  return HMX_OK;
}

int hmx_ctx_set_stream(hmx_ctx* ctx, uint64_t stream) {
  if (!ctx) return HMX_EINVAL;
  HMX_CUDA_TRY(cudaSetDevice(ctx->c.device));
  HMX_CUDA_TRY(cudaStreamSynchronize(ctx->c.stream));
  if (ctx->c.own_stream && ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
  // any value is taken as a cudaStream_t; 0 is the legacy default stream
  ctx->c.stream = reinterpret_cast<cudaStream_t>(stream);
  ctx->c.own_stream = false;
  return HMX_OK;
}

int hmx_ctx_release_cache(hmx_ctx* ctx) {
  if (!ctx) return HMX_EINVAL;
  HMX_CUDA_TRY(cudaSetDevice(ctx->c.device));
  HMX_CUDA_TRY(cudaStreamSynchronize(ctx->c.stream));
  if (ctx->c.pool) HMX_CUDA_TRY(cudaMemPoolTrimTo(ctx->c.pool, 0));
  release_cache(ctx->c);
  return HMX_OK;
}

int hmx_ctx_reserve(hmx_ctx* ctx, double gigabytes, double* seconds) {
  if (!ctx || gigabytes < 0.0) return HMX_EINVAL;
  Ctx& c = ctx->c;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  const auto t0 = std::chrono::steady_clock::now();
  {
    std::lock_guard<std::mutex> lk(c.mem_mu);
    if (c.arena) {
      hmx_set_error("hmx_ctx_reserve: the context already holds a reserved region of %.2f GB", c.arena_size / 1e9);
      return HMX_EINVAL;
    }
  }
  release_cache(c);
  size_t free_b = 0, total_b = 0;
  HMX_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  // default: what the assembly's capacity model may use plus the final streams, leaving the rest
  // of the device to the libraries next to it (cuBLAS / cuSOLVER workspaces, the H-LU pool)
  size_t want = gigabytes > 0.0 ? (size_t)(gigabytes * 1e9) : (size_t)(0.88 * (double)free_b);
  want = want / hmx::kArenaGran * hmx::kArenaGran;
  if (want == 0 || want > free_b) {
    hmx_set_error("hmx_ctx_reserve: %.2f GB requested, %.2f GB free", want / 1e9, free_b / 1e9);
    return HMX_ENOMEM;
  }
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    hmx_set_error("hmx_ctx_reserve: cudaMalloc(%.2f GB): %s", want / 1e9, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? HMX_ENOMEM : HMX_ECUDA;
  }
  {
    std::lock_guard<std::mutex> lk(c.mem_mu);
    c.arena = static_cast<char*>(p);
    c.arena_size = c.arena_free = want;
    c.arena_holes.clear();
    c.arena_holes.emplace(0, want);
  }
  if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return HMX_OK;
}

int hmx_ctx_sync(hmx_ctx* ctx) {
  if (!ctx) return HMX_EINVAL;
  HMX_CUDA_TRY(cudaStreamSynchronize(ctx->c.stream));
  return HMX_OK;
}

int hmx_ctx_destroy(hmx_ctx* ctx) {
  if (!ctx) return HMX_OK;
  cudaSetDevice(ctx->c.device);
  if (ctx->c.own_stream && ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
  if (ctx->c.aux) cudaStreamDestroy(ctx->c.aux);
  if (ctx->c.rerun) cudaStreamDestroy(ctx->c.rerun);
  if (ctx->c.side) cudaStreamDestroy(ctx->c.side);
  if (ctx->c.pool) cudaMemPoolDestroy(ctx->c.pool);
  hlu_pool_destroy(ctx->c);
  linalg_destroy(ctx->c);
  release_cache(ctx->c);
  delete ctx;
  return HMX_OK;
}

// ---- geometry -----------------------------------------------------------------
int hmx_tree_build(const double* points, int64_t n, int64_t n_leaf, hmx_tree** out) {
  if (!points || !out) return HMX_EINVAL;
  if (n <= 0) {
    hmx_set_error("empty input");
    return HMX_EINVAL;
  }
  if (n_leaf < 1) {
    hmx_set_error("n_leaf must be >= 1");
    return HMX_EINVAL;
  }
  auto* t = new hmx_tree;
  build_cluster_tree(points, n, n_leaf, t->t);
  *out = t;
  return HMX_OK;
}

int64_t hmx_tree_num_nodes(const hmx_tree* t) { return t ? (int64_t)t->t.nodes.size() : -1; }

int hmx_tree_export(const hmx_tree* t, int64_t* perm, int64_t* nodes, double* boxes) {
  if (!t) return HMX_EINVAL;
  if (perm) std::memcpy(perm, t->t.perm.data(), sizeof(int64_t) * t->t.n);
  for (size_t v = 0; v < t->t.nodes.size(); ++v) {
    const TreeNode& N = t->t.nodes[v];
    if (nodes) {
      nodes[5 * v + 0] = N.start;
      nodes[5 * v + 1] = N.stop;
      nodes[5 * v + 2] = N.level;
      nodes[5 * v + 3] = N.child[0];
      nodes[5 * v + 4] = N.child[1];
    }
    if (boxes)
      for (int k = 0; k < 3; ++k) {
        boxes[6 * v + k] = N.lo[k];
        boxes[6 * v + 3 + k] = N.hi[k];
      }
  }
  return HMX_OK;
}

void hmx_tree_free(hmx_tree* t) { delete t; }

int hmx_blocks_build(const hmx_tree* rows, const hmx_tree* cols, double eta, hmx_blocks** out) {
  if (!rows || !cols || !out) return HMX_EINVAL;
  if (!(eta > 0)) {
    hmx_set_error("eta must be positive");
    return HMX_EINVAL;
  }
  auto* b = new hmx_blocks;
  build_block_leaves(rows->t, cols->t, eta, b->v);
  *out = b;
  return HMX_OK;
}

int64_t hmx_blocks_count(const hmx_blocks* b) { return b ? (int64_t)b->v.size() : -1; }

int hmx_blocks_export(const hmx_blocks* b, int64_t* table) {
  if (!b || !table) return HMX_EINVAL;
  for (size_t i = 0; i < b->v.size(); ++i) {
    const BlockLeaf& L = b->v[i];
    int64_t* t = table + 7 * i;
    t[0] = L.kind;
    t[1] = L.r0;
    t[2] = L.r1;
    t[3] = L.c0;
    t[4] = L.c1;
    t[5] = L.rnode;
    t[6] = L.cnode;
  }
  return HMX_OK;
}

void hmx_blocks_free(hmx_blocks* b) { delete b; }

// ---- kernel seam ------------------------------------------------------------------
int hmx_eval_block(hmx_ctx* ctx, const hmx_kernel* k, const double* X, int64_t m, const double* Y, int64_t n,
                   const double* NY, int32_t has_shift, double shift, double* out) {
  if (!ctx || !k || !X || !Y || !out || m <= 0 || n <= 0) return HMX_EINVAL;
  if (k->kind < 0 || k->kind > 2) return HMX_EINVAL;
  if (k->kind == HMX_ELASTO_T && !NY) {
    hmx_set_error("elasto T requires column normals");
    return HMX_EINVAL;
  }
  Ctx& c = ctx->c;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  const int d = k->kind == 0 ? 1 : 3;
  DevPoints dx, dy;
  int rc = dx.upload(c, X, nullptr, m);
  if (rc) return rc;
  rc = dy.upload(c, Y, k->kind == HMX_ELASTO_T ? NY : nullptr, n);
  if (rc) return rc;
  DevBuf mem(c);
  double2* dout;
  int32_t* derr;
  if ((rc = mem.alloc(&dout, (int64_t)d * d * m * n))) return rc;
  if ((rc = mem.alloc(&derr, 1))) return rc;
  HMX_CUDA_TRY(cudaMemsetAsync(derr, 0, sizeof(int32_t), c.stream));
  GreenParams P = make_params(k, has_shift, shift);
  if ((rc = launch_eval_block(c, P, dx.soa, dy.soa, m, n, dout, derr))) return rc;
  int32_t herr = 0;
  HMX_CUDA_TRY(cudaMemcpyAsync(&herr, derr, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
  HMX_CUDA_TRY(
      cudaMemcpyAsync(out, dout, sizeof(double2) * d * d * m * n, cudaMemcpyDeviceToHost, c.stream));
  HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  if (herr) {
    hmx_set_error("singular evaluation: coincident points without a self rule");
    return HMX_ESINGULAR;
  }
  return HMX_OK;
}

// ---- assembly --------------------------------------------------------------------------
int hmx_assemble(hmx_ctx* ctx, const hmx_kernel* k, const double* pts_tree, const double* nrm_tree, int64_t np,
                 const int64_t* perm, const int64_t* table, int64_t nb, const hmx_aca_cfg* cfg, double self_shift,
                 hmx_hmatrix** out) {
  if (!ctx || !k || !pts_tree || !perm || !table || !cfg || !out || np <= 0) return HMX_EINVAL;
  if (k->kind < 0 || k->kind > 2) return HMX_EINVAL;
  if (k->kind == HMX_ELASTO_T && !nrm_tree) {
    hmx_set_error("elasto T requires normals");
    return HMX_EINVAL;
  }
  if (!(cfg->eps > 0 && cfg->eps < 1)) {
    hmx_set_error("eps_aca must be in (0, 1)");
    return HMX_EINVAL;
  }
  int rc = validate_table(table, nb, np);
  if (rc) return rc;
  const double eps_rc = cfg->eps_recompress > 0 ? cfg->eps_recompress : cfg->eps;
  Ctx& c = ctx->c;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  const auto t_start = std::chrono::steady_clock::now();
  auto holder = new hmx_hmatrix;
  DeviceH& H = holder->H;
  H.ctx = &c;
  H.kind = k->kind;
  H.d = k->kind == 0 ? 1 : 3;
  const int d = H.d;
  H.np = np;
  H.n = d * np;
  H.nb = nb;
  H.table.assign(table, table + 5 * nb);
  H.steps.assign(nb, 0);
  H.rank_before.assign(nb, 0);
  H.rank_after.assign(nb, 0);
  H.flags.assign(nb, 0);
  auto fail = [&](int code) {
    free_h(H);
    delete holder;
    return code;
  };
  DevPoints pts;
  if ((rc = pts.upload(c, pts_tree, k->kind == HMX_ELASTO_T ? nrm_tree : nullptr, np))) return fail(rc);
  {
    std::vector<int64_t> p(perm, perm + np);
    if ((rc = dev_upload(c, &H.d_perm, p))) return fail(rc);
  }
  const GreenParams P = make_params(k, 1, self_shift);
  cudaEvent_t ev[6];
  for (auto& e : ev) HMX_CUDA_TRY(cudaEventCreate(&e));
  HMX_CUDA_TRY(cudaEventRecord(ev[0], c.stream));
  const bool verbose = std::getenv("HMX_VERBOSE") != nullptr;
  auto tick = [&](const char* what) {
    if (!verbose) return;
    cudaStreamSynchronize(c.stream);
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    std::fprintf(stderr, "[hmx] %-28s %9.2f ms   free %7.2f GB  cache %6.2f GB\n", what,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(),
                 fr / 1e9, c.cached_bytes / 1e9);
  };
  tick("upload");
  // host-only time stamps (no synchronisation), printed with the GPU timeline
  std::vector<std::pair<std::string, double>> hl;
  auto htick = [&](const char* what) {
    if (verbose)
      hl.emplace_back(what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  };
  // HMX_VERBOSE: GPU timeline of the launches (events on the issuing stream)
  std::vector<std::pair<std::string, cudaEvent_t>> tl;
  auto mark = [&](const std::string& what) {
    if (!verbose) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, c.stream);
    tl.emplace_back(what + (c.stream == c.aux ? " [aux]" : " [main]"), e);
  };

  // ---- 1. ACA passes --------------------------------------------------------------------
  std::vector<int64_t> adm;
  for (int64_t b = 0; b < nb; ++b)
    if (table[5 * b] == 1) adm.push_back(b);
  auto rows_of = [&](int64_t b) { return table[5 * b + 2] - table[5 * b + 1]; };
  auto cols_of = [&](int64_t b) { return table[5 * b + 4] - table[5 * b + 3]; };
  std::vector<int64_t> maxr(nb, 0), kcap(nb, 0);
  for (int64_t b : adm) {
    int64_t dmin = d * std::min(rows_of(b), cols_of(b));
    maxr[b] = cfg->max_rank > 0 ? std::min<int64_t>(cfg->max_rank, dmin) : dmin;
  }
  tick("aca: bounds");
  size_t free_b = 0, total_b = 0;
  HMX_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  tick("aca: meminfo");
  // memory cached by this context counts as free; U, V and the Gram matrices get
  // kAcaBudgetFrac of it (the Grams are released before the final streams are allocated)
  double avail = (double)free_b + (double)c.cached_bytes + (double)c.arena_free;
  double budget = cfg->mem_budget_gb > 0 ? cfg->mem_budget_gb * 1e9 : kAcaBudgetFrac * avail;
  auto round_d = [&](int64_t v) { return std::max<int64_t>(d, (v / d) * d); };
  // one routing decision feeds both the workspace plan (tensor-core Gram scratch) and the
  // launch split (wide prefix of the size-sorted pass): aca_route, hmatrix.h
  const AcaRoute route = aca_route(d, cfg);
  auto is_tc = [&](int64_t b) { return route.use_tc && rows_of(b) + cols_of(b) >= route.wide_min; };
  auto ws_bytes = [&](int64_t b, int64_t kc) {
    return 16.0 * ((double)d * (rows_of(b) + cols_of(b)) * kc + 2.0 * kc * kc +
                   (is_tc(b) ? (double)aca_tc_scratch(kc) : 0.0));
  };
  {
    // Column capacity per leaf from a geometric rank model: ACA ranks of these
    // kernels grow with kappa * diam (oscillatory regime) on top of a
    // frequency-independent floor (measured envelope over the five configs:
    // K <= a + 2 d kappa diam with a <= 70, docs in DESIGN.md 3).  Leaves that
    // outgrow it are re-run with twice the capacity (same result, deterministic).
    const double kap = k->kind == 0 ? std::fabs(k->kappa) : std::max(std::fabs(k->ks), std::fabs(k->kp));
    // Cluster diameters from "atom" boxes: the distinct cluster boundaries of
    // the admissible leaves cut [0, np) into atoms; one pass over the points
    // boxes every atom, and a cluster's box is the merge of its atoms' boxes.
    std::vector<int64_t> cuts;
    {
      std::vector<unsigned char> mark((size_t)np + 1, 0);  // boundaries are point indices in [0, np]
      for (int64_t b : adm)
        for (int q = 1; q <= 4; ++q) mark[(size_t)table[5 * b + q]] = 1;
      for (int64_t v = 0; v <= np; ++v)
        if (mark[(size_t)v]) cuts.push_back(v);
    }
    const size_t na = cuts.empty() ? 0 : cuts.size() - 1;
    std::vector<double> abox(6 * na);
    for (size_t a = 0; a < na; ++a) {
      double lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY, hi2 = -INFINITY;
      for (int64_t t = cuts[a]; t < cuts[a + 1]; ++t) {
        const double* q = pts_tree + 3 * t;
        lo0 = std::min(lo0, q[0]);
        hi0 = std::max(hi0, q[0]);
        lo1 = std::min(lo1, q[1]);
        hi1 = std::max(hi1, q[1]);
        lo2 = std::min(lo2, q[2]);
        hi2 = std::max(hi2, q[2]);
      }
      double* bx = &abox[6 * a];
      bx[0] = lo0, bx[1] = lo1, bx[2] = lo2, bx[3] = hi0, bx[4] = hi1, bx[5] = hi2;
    }
    auto atom = [&](int64_t v) { return (size_t)(std::lower_bound(cuts.begin(), cuts.end(), v) - cuts.begin()); };
    auto diam = [&](int64_t a0, int64_t a1) {
      double lo3[3] = {INFINITY, INFINITY, INFINITY}, hi3[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (size_t a = atom(a0), e = atom(a1); a < e; ++a)
        for (int q = 0; q < 3; ++q) {
          lo3[q] = std::min(lo3[q], abox[6 * a + q]);
          hi3[q] = std::max(hi3[q], abox[6 * a + 3 + q]);
        }
      return std::sqrt((hi3[0] - lo3[0]) * (hi3[0] - lo3[0]) + (hi3[1] - lo3[1]) * (hi3[1] - lo3[1]) +
                       (hi3[2] - lo3[2]) * (hi3[2] - lo3[2]));
    };
    // K <= a + 2 d kappa diam with a = 66 (d = 3), and at low frequency a
    // geometry-independent floor of 78 columns: tools/kcap_census.py over the
    // five configs (U131k, kappa_s = 2, needs K + 3 <= kcap at K = 66-81)
    const double floor_cols = d == 1 ? 36.0 : 66.0;
    const double floor_lo = d == 1 ? 36.0 : 78.0;
    // clusters are shared by many leaves: one diameter per distinct (start, stop)
    std::unordered_map<int64_t, double> dcache;
    dcache.reserve(2 * adm.size() + 16);
    auto diam_c = [&](int64_t a0, int64_t a1) {
      const int64_t key = a0 * (np + 1) + a1;
      auto it = dcache.find(key);
      if (it != dcache.end()) return it->second;
      const double v = diam(a0, a1);
      dcache.emplace(key, v);
      return v;
    };
    for (int64_t b : adm) {
      const double dm =
          std::max(diam_c(table[5 * b + 1], table[5 * b + 2]), diam_c(table[5 * b + 3], table[5 * b + 4]));
      const int64_t est =
          round_d((int64_t)std::ceil(std::max(floor_lo, floor_cols + 2.0 * d * kap * dm)) + d - 1);
      kcap[b] = std::min<int64_t>(maxr[b], std::min<int64_t>(est, round_d(kMaxAcaCols)));
    }
    // fit the budget: scale the model down uniformly if needed
    double need = 0;
    for (int64_t b : adm) need += ws_bytes(b, kcap[b]);
    if (need > budget && c.cached_bytes > 0 && cfg->mem_budget_gb <= 0) {
      // blocks cached for other sizes may not be reusable: hand them back and
      // size the budget from what is really free (a scaled-down capacity model
      // turns into expensive overflow reruns)
      release_cache(c);
      HMX_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
      avail = (double)free_b + (double)c.arena_free;
      budget = kAcaBudgetFrac * avail;
    }
    if (verbose)
      std::fprintf(stderr, "[hmx] ACA workspace model %.2f GB, budget %.2f GB\n", need / 1e9, budget / 1e9);
    if (need > budget) {
      const double f = budget / need;
      for (int64_t b : adm) kcap[b] = std::max<int64_t>(d, round_d((int64_t)(kcap[b] * f)));
    }
  }
  tick("aca: capacity model");
  PlanPre pre;
  std::deque<AcaPass> passes;  // stable addresses (Pending keeps pointers)
  std::vector<int64_t> todo = adm;
  const double s3f = cfg->sigma3_floor > 0 ? cfg->sigma3_floor : 1e-12;
  const int64_t nmax = route.wide_min;
  // recompression results read back once at the end
  struct Pending {
    AcaPass* ps;
    std::vector<int64_t> live;  // indices into ps->blocks
    int32_t* d_rank;
    int32_t* d_flag;
  };
  std::vector<Pending> pending;
  DevBuf rec_tmp(c);
  const cudaStream_t main_stream = c.stream;
  // Recompression of the live leaves [q0, q1) of a pass, on the current c.stream.
  auto recompress_subset = [&](AcaPass& ps, std::vector<int64_t> live) -> int {
    if (live.empty()) return HMX_OK;
    htick("consume: live list built");
    // largest K first, launched in K classes so small leaves do not pay for big shared memory
    {
      // counting sort on the rank (descending), stable in position order: the
      // order of sort(rank desc, position asc) without the comparison sort
      int kmax = 0;
      for (int64_t x : live) kmax = std::max(kmax, ps.out[x].rank);
      std::vector<int64_t> cnt((size_t)kmax + 2, 0);
      for (int64_t x : live) cnt[(size_t)(kmax - ps.out[x].rank) + 1]++;
      for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
      std::vector<int64_t> sorted(live.size());
      std::sort(live.begin(), live.end());
      for (int64_t x : live) sorted[(size_t)cnt[(size_t)(kmax - ps.out[x].rank)]++] = x;
      live.swap(sorted);
    }
    htick("consume: class sort");
    std::vector<RecDesc> rd(live.size());
    int64_t wo = 0;
    for (size_t q = 0; q < live.size(); ++q) {
      const int K = ps.out[live[q]].rank;
      rd[q].goff = ps.desc[live[q]].goff;
      rd[q].woff = wo;
      rd[q].K = K;
      rd[q].kcap = ps.desc[live[q]].kcap;
      wo += 6 * (int64_t)K * K;
    }
    double2* W;
    RecDesc* d_rd;
    int32_t *d_rank, *d_flag;
    int e;
    if ((e = ps.mem.alloc(&W, wo))) return e;
    if ((e = rec_tmp.alloc(&d_rd, (int64_t)rd.size()))) return e;
    if ((e = rec_tmp.alloc(&d_rank, (int64_t)rd.size()))) return e;
    if ((e = rec_tmp.alloc(&d_flag, (int64_t)rd.size()))) return e;
    htick("consume: descriptors + alloc");
    for (size_t q = 0; q < live.size(); ++q) ps.wptr[live[q]] = W + rd[q].woff;
    HMX_CUDA_TRY(cudaMemcpyAsync(d_rd, rd.data(), sizeof(RecDesc) * rd.size(), cudaMemcpyHostToDevice, c.stream));
    htick("consume: upload");
    mark("recompress start");
    // shared-memory size classes (smem ~ 16 K^2 bytes): more CTAs per SM for small K
    const int classes[] = {kMaxAcaCols, kRecompressSmemMax, 88, 72, 60, 48, 39, 30, 21};
    const int ncls = (int)(sizeof(classes) / sizeof(classes[0]));
    // The large-K class (one long eigen-solve chain per leaf, a tail of a few K > 200 leaves) goes to
    // the side stream when smaller classes follow: they run next to it instead of behind its tail.
    const cudaStream_t issue = c.stream;
    const bool split = c.side && rd[0].K > kRecompressSmemMax && rd.back().K <= kRecompressSmemMax;
    if (split) {
      cudaEvent_t fork;
      HMX_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      HMX_CUDA_TRY(cudaEventRecord(fork, issue));
      HMX_CUDA_TRY(cudaStreamWaitEvent(c.side, fork, 0));
      cudaEventDestroy(fork);
    }
    size_t q0 = 0;
    for (int ci = 0; ci < ncls && q0 < rd.size(); ++ci) {
      const int lim_lo = ci + 1 < ncls ? classes[ci + 1] : 0;
      size_t q1 = q0;
      while (q1 < rd.size() && (rd[q1].K > lim_lo || ci == ncls - 1)) ++q1;
      if (q1 > q0) {
        if (split && ci == 0) c.stream = c.side;
        e = launch_recompress_core(c, d_rd + q0, (int64_t)(q1 - q0), rd[q0].K, eps_rc, cfg->trunc_rule, ps.G, W,
                                   d_rank + q0, d_flag + q0);
        c.stream = issue;
        if (!(split && ci == 0))
          mark("  rc class K<=" + std::to_string(rd[q0].K) + " n=" + std::to_string(q1 - q0));
        if (e) return e;
      }
      q0 = q1;
    }
    if (split) {
      cudaEvent_t join;
      HMX_CUDA_TRY(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
      HMX_CUDA_TRY(cudaEventRecord(join, c.side));
      HMX_CUDA_TRY(cudaStreamWaitEvent(issue, join, 0));
      cudaEventDestroy(join);
      mark("  rc large-K class joined");
    }
    mark("recompress issued");
    htick("consume: classes launched");
    pending.push_back(Pending{&ps, std::move(live), d_rank, d_flag});
    return HMX_OK;
  };
  // ACA outputs of positions [q0, q1) of the pass (already on the host):
  // bookkeeping, overflow -> next pass, recompression of the rest
  std::vector<int64_t> next;
  std::vector<int64_t> fb_leaves;  // leaves whose sigma_3 pivots all fell below the floor
  auto consume = [&](AcaPass& ps, size_t q0, size_t q1) -> int {
    std::vector<int64_t> live;
    for (size_t i = q0; i < q1; ++i) {
      const int64_t b = ps.blocks[i];
      const AcaOut& o = ps.out[i];
      if (o.status & 4) {
        if (kcap[b] >= std::min<int64_t>(maxr[b], round_d(kMaxAcaCols))) {
          hmx_set_error("block %lld: ACA rank exceeds %d columns", (long long)b, kMaxAcaCols);
          return HMX_ENOMEM;
        }
        kcap[b] = std::min<int64_t>(std::min<int64_t>(maxr[b], round_d(kMaxAcaCols)), 2 * kcap[b]);
        next.push_back(b);
        ps.out[i].rank = -1;  // superseded
        continue;
      }
      H.steps[b] = o.steps;
      H.rank_before[b] = o.rank;
      H.flags[b] = o.status & 0xB;
      H.pairs_evaluated += (int64_t)o.steps * (rows_of(b) + cols_of(b)) + (int64_t)o.zero_rows * cols_of(b);
      if (o.status & 8) {  // FallbackNeeded: randomized SVD after the passes (section 1b)
        fb_leaves.push_back(b);
        continue;
      }
      live.push_back((int64_t)i);
    }
    return recompress_subset(ps, std::move(live));
  };
  // Capacity-overflow reruns (passes after the first) depend only on the
  // points and their own workspaces: they go to a high-priority stream
  // (ordered after everything issued before this assembly) and overlap the
  // first pass's remaining recompression instead of trailing it.
  cudaEvent_t ev_start;
  HMX_CUDA_TRY(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
  HMX_CUDA_TRY(cudaEventRecord(ev_start, c.stream));
  HMX_CUDA_TRY(cudaStreamWaitEvent(c.rerun, ev_start, 0));
  cudaEventDestroy(ev_start);
  struct StreamSwap {
    Ctx& c;
    cudaStream_t s0, a0;
    bool on = false;
    void enter() {
      if (!on) {
        s0 = c.stream;
        a0 = c.aux;
        c.stream = c.aux = c.rerun;
        on = true;
      }
    }
    ~StreamSwap() {
      if (on) {
        c.stream = s0;
        c.aux = a0;
      }
    }
  } rerun_swap{c, nullptr, nullptr};
  while (!todo.empty()) {
    if (H.aca_passes > 0) rerun_swap.enter();
    passes.emplace_back(c);
    AcaPass& ps = passes.back();
    {
      // LPT order (m + n descending, leaf index ascending) by a counting sort
      std::sort(todo.begin(), todo.end());
      int64_t smax = 0;
      for (int64_t b : todo) smax = std::max<int64_t>(smax, rows_of(b) + cols_of(b));
      std::vector<int64_t> cnt((size_t)smax + 2, 0);
      for (int64_t b : todo) cnt[(size_t)(smax - (rows_of(b) + cols_of(b))) + 1]++;
      for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
      std::vector<int64_t> srt(todo.size());
      for (int64_t b : todo) srt[(size_t)cnt[(size_t)(smax - (rows_of(b) + cols_of(b)))]++] = b;
      todo.swap(srt);
    }
    ps.blocks = todo;
    int64_t uo = 0, vo = 0, go = 0;
    ps.desc.resize(todo.size());
    ps.wptr.assign(todo.size(), nullptr);
    for (size_t i = 0; i < todo.size(); ++i) {
      const int64_t b = todo[i];
      AcaDesc& D = ps.desc[i];
      D.r0 = table[5 * b + 1];
      D.c0 = table[5 * b + 3];
      D.m = (int32_t)rows_of(b);
      D.n = (int32_t)cols_of(b);
      D.kcap = (int32_t)kcap[b];
      D.max_rank = (int32_t)maxr[b];
      D.uoff = uo;
      D.voff = vo;
      D.goff = go;
      uo += (int64_t)d * D.m * D.kcap;
      vo += (int64_t)d * D.n * D.kcap;
      go += 2 * (int64_t)D.kcap * D.kcap + (is_tc(b) ? aca_tc_scratch(D.kcap) : 0);
      ps.kcap_max = std::max<int>(ps.kcap_max, D.kcap);
    }
    tick("aca: descriptors");
    if ((rc = ps.mem.alloc(&ps.U, uo))) return fail(rc);
    tick("aca: alloc U");
    if ((rc = ps.mem.alloc(&ps.V, vo))) return fail(rc);
    tick("aca: alloc V");
    if ((rc = ps.gmem.alloc(&ps.G, go))) return fail(rc);
    tick("aca: alloc G");
    AcaDesc* d_desc;
    AcaOut* d_out;
    int32_t* d_order;
    if ((rc = rec_tmp.alloc(&d_desc, (int64_t)todo.size()))) return fail(rc);
    if ((rc = rec_tmp.alloc(&d_out, (int64_t)todo.size()))) return fail(rc);
    if ((rc = rec_tmp.alloc(&d_order, (int64_t)todo.size()))) return fail(rc);
    std::vector<int32_t> order(todo.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int32_t)i;
    HMX_CUDA_TRY(cudaMemcpyAsync(d_desc, ps.desc.data(), sizeof(AcaDesc) * todo.size(), cudaMemcpyHostToDevice,
                                 c.stream));
    HMX_CUDA_TRY(
        cudaMemcpyAsync(d_order, order.data(), sizeof(int32_t) * todo.size(), cudaMemcpyHostToDevice, c.stream));
    tick("aca: workspace alloc");
    // large leaves (wide CTAs, a prefix of the size-sorted list) on the
    // auxiliary stream, the many small leaves (narrow CTAs) on the main
    // stream; each side's recompression starts as soon as its own ACA is done
    size_t nwide = 0;
    while (nwide < todo.size() && rows_of(todo[nwide]) + cols_of(todo[nwide]) >= nmax) ++nwide;
    auto sub_max = [&](size_t q0, size_t q1, int& kc, int& mm) {
      kc = 1;
      mm = 1;
      for (size_t q = q0; q < q1; ++q) {
        kc = std::max<int>(kc, ps.desc[q].kcap);
        mm = std::max<int>(mm, ps.desc[q].m);
      }
    };
    cudaEvent_t fork;
    HMX_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    HMX_CUDA_TRY(cudaEventRecord(fork, c.stream));
    HMX_CUDA_TRY(cudaStreamWaitEvent(c.aux, fork, 0));
    cudaEventDestroy(fork);
    ps.out.resize(todo.size());
    int kc, mm;
    mark("aca start");
    {
      OnAux on(c);
      mark("aca wide start");
      if (nwide) {
        sub_max(0, nwide, kc, mm);
        if ((rc = launch_aca(c, d, P, pts.soa, d_desc, d_order, (int64_t)nwide, kc, mm, cfg->eps, s3f, ps.U, ps.V,
                             ps.G, d_out, route.use_tc ? kAcaTensor : kAcaWide, route.tc_stages)))
          return fail(rc);
      }
      mark("aca wide done");
      if (nwide)
        HMX_CUDA_TRY(
            cudaMemcpyAsync(ps.out.data(), d_out, sizeof(AcaOut) * nwide, cudaMemcpyDeviceToHost, c.stream));
    }
    if (todo.size() > nwide) {
      sub_max(nwide, todo.size(), kc, mm);
      if ((rc = launch_aca(c, d, P, pts.soa, d_desc, d_order + nwide, (int64_t)(todo.size() - nwide), kc, mm,
                           cfg->eps, s3f, ps.U, ps.V, ps.G, d_out, kAcaNarrow, 0)))
        return fail(rc);
      mark("aca narrow done");
    }
    // the rank-independent half of the matvec plan while the ACA runs: before the read-backs,
    // which block the host until their kernel is done (device -> pageable host copies return only
    // once complete)
    if (pre.segs.empty()) build_plan_pre(H, pre);
    htick("plan pre built");
    if (todo.size() > nwide)
      HMX_CUDA_TRY(cudaMemcpyAsync(ps.out.data() + nwide, d_out + nwide, sizeof(AcaOut) * (todo.size() - nwide),
                                   cudaMemcpyDeviceToHost, c.stream));
    // narrow leaves (main stream) first, then the wide ones (aux stream): the wide leaves'
    // large-K recompression classes then queue on aux behind the wide ACA and overlap the
    // narrow leaves' recompression on the main stream
    if (todo.size() > nwide) {
      HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
      htick("narrow ACA synced");
      if ((rc = consume(ps, nwide, todo.size()))) return fail(rc);
    }
    if (nwide) {
      HMX_CUDA_TRY(cudaStreamSynchronize(c.aux));
      OnAux on(c);
      if ((rc = consume(ps, 0, nwide))) return fail(rc);
    }
    H.aca_passes++;
    // join the auxiliary stream before the next pass / the layout
    cudaEvent_t join;
    HMX_CUDA_TRY(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    HMX_CUDA_TRY(cudaEventRecord(join, c.aux));
    HMX_CUDA_TRY(cudaStreamWaitEvent(c.stream, join, 0));
    cudaEventDestroy(join);
    todo.swap(next);
    next.clear();
  }
  if (rerun_swap.on) {  // back to the context streams; main waits for the reruns
    c.stream = rerun_swap.s0;
    c.aux = rerun_swap.a0;
    rerun_swap.on = false;
    cudaEvent_t join;
    HMX_CUDA_TRY(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    HMX_CUDA_TRY(cudaEventRecord(join, c.rerun));
    HMX_CUDA_TRY(cudaStreamWaitEvent(c.stream, join, 0));
    cudaEventDestroy(join);
  }
  // ---- 1b. randomized-SVD fallback -------------------------------
  // each flagged leaf is regenerated densely, compressed by the adaptive range finder and
  // recompressed like an ACA factor pair; its factors are copied into the streams after the
  // layout (section 3).  Pivot exhaustion is reported only if the fallback itself fails.
  struct FbOut {
    int64_t b;
    int r;
    double2 *U, *V;
  };
  std::vector<FbOut> fbo;
  DevBuf fb_mem(c);
  for (int64_t b : fb_leaves) {
    const int64_t m = rows_of(b), n = cols_of(b), dm = d * m, dn = d * n;
    const int64_t cap = std::min<int64_t>(maxr[b], kMaxAcaCols);
    DevBuf t(c);
    double2 *A, *U, *V, *G;
    int64_t* dd;
    int32_t* derr;
    if ((rc = t.alloc(&A, dm * dn)) || (rc = t.alloc(&U, dm * cap)) || (rc = t.alloc(&V, dn * cap)) ||
        (rc = t.alloc(&G, 2 * cap * cap)) || (rc = t.alloc(&dd, 6)) || (rc = t.alloc(&derr, 1)))
      return fail(rc);
    const int64_t desc[6] = {table[5 * b + 1], m, table[5 * b + 3], n, 0, dm};
    HMX_CUDA_TRY(cudaMemcpyAsync(dd, desc, sizeof(desc), cudaMemcpyHostToDevice, c.stream));
    HMX_CUDA_TRY(cudaMemsetAsync(derr, 0, sizeof(int32_t), c.stream));
    if ((rc = launch_dense_fill(c, P, pts.soa, dd, 1, A, derr))) return fail(rc);
    int K = 0, conv = 0;
    const uint64_t seed = (uint64_t)cfg->rsvd_seed * 0x9E3779B97F4A7C15ull + (uint64_t)b;
    if ((rc = rsvd_dense(c, A, dm, dn, cfg->eps, kRsvdOversample, cap, seed, U, V, G, &K, &conv))) {
      const std::string why = g_last_error;
      hmx_set_error("block %lld: FallbackNeeded and the randomized-SVD fallback failed (%s)", (long long)b,
                    why.c_str());
      return fail(HMX_EPIVOT);
    }
    int r = 0;
    double2 *Uo = nullptr, *Vo = nullptr;
    if (K > 0 && (rc = recompress_device(c, fb_mem, U, V, dm, dn, K, G, eps_rc, cfg->trunc_rule, &r, &Uo, &Vo)))
      return fail(rc);
    H.rank_before[b] = K;
    H.rank_after[b] = r;
    H.flags[b] = (H.flags[b] & ~1) | (conv ? 1 : 0) | 8 | 128;  // bit 7: factors from the rSVD fallback
    H.n_fallback++;
    H.pairs_evaluated += m * n;
    fbo.push_back(FbOut{b, r, Uo, Vo});
  }
  HMX_CUDA_TRY(cudaEventRecord(ev[1], c.stream));
  tick("aca done");
  if (verbose) {
    cudaDeviceSynchronize();
    for (auto& kv : hl) std::fprintf(stderr, "[hmx]   host %-35s %9.2f ms\n", kv.first.c_str(), kv.second);
    for (auto& kv : tl) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[0], kv.second);
      std::fprintf(stderr, "[hmx]   gpu %-36s %9.2f ms\n", kv.first.c_str(), ms);
      cudaEventDestroy(kv.second);
    }
  }
  // ---- 2. recompression results (launched per pass above) -------------------------------
  for (Pending& pd : pending) {
    std::vector<int32_t> hr(pd.live.size()), hf(pd.live.size());
    HMX_CUDA_TRY(
        cudaMemcpyAsync(hr.data(), pd.d_rank, sizeof(int32_t) * hr.size(), cudaMemcpyDeviceToHost, c.stream));
    HMX_CUDA_TRY(
        cudaMemcpyAsync(hf.data(), pd.d_flag, sizeof(int32_t) * hf.size(), cudaMemcpyDeviceToHost, c.stream));
    HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
    // pd.live was sorted by K inside recompress_subset: rebuild the same order
    std::vector<int64_t> lv = pd.live;
    for (size_t q = 0; q < lv.size(); ++q) {
      const int64_t b = pd.ps->blocks[lv[q]];
      H.rank_after[b] = hr[q];
      if (hf[q] & 1) {
        H.flags[b] |= 16;
        H.n_regularized++;
      }
      if (hf[q] & 4) H.flags[b] |= 32;  // eigenvectors from the QL fallback
      if (hf[q] & 2) H.flags[b] |= 64;  // QL did not converge
    }
  }
  HMX_CUDA_TRY(cudaEventRecord(ev[2], c.stream));
  for (AcaPass& ps : passes) ps.gmem.release();  // Gram workspaces back before the streams are allocated
  tick("recompress done");

  // ---- 3. layout + matvec plan ----------------------------------------------------------------
  if (verbose) setenv("HMX_VERBOSE_PLAN", "1", 1);
  if ((rc = build_matvec_plan(H, &pre))) return fail(rc);
  for (const FbOut& f : fbo) {
    if (f.r == 0) continue;
    const int64_t dm = d * rows_of(f.b), dn = d * cols_of(f.b);
    HMX_CUDA_TRY(cudaMemcpyAsync(H.d_row + H.leaf_moff[f.b], f.U, sizeof(double2) * dm * f.r,
                                 cudaMemcpyDeviceToDevice, c.stream));
    HMX_CUDA_TRY(cudaMemcpyAsync(H.d_v + H.leaf_voff[f.b], f.V, sizeof(double2) * dn * f.r,
                                 cudaMemcpyDeviceToDevice, c.stream));
  }

  // ---- 4a. dense leaves ---------------------------------------------------------------------
  HMX_CUDA_TRY(cudaEventRecord(ev[3], c.stream));
  tick("layout + plan");
  int32_t* d_err;
  DevBuf tmp4(c);
  if ((rc = tmp4.alloc(&d_err, 1))) return fail(rc);
  HMX_CUDA_TRY(cudaMemsetAsync(d_err, 0, sizeof(int32_t), c.stream));
  {
    std::vector<int64_t> dd;
    for (int64_t b = 0; b < nb; ++b) {
      if (table[5 * b] != 0) continue;
      dd.insert(dd.end(), {table[5 * b + 1], rows_of(b), table[5 * b + 3], cols_of(b), H.leaf_moff[b], H.leaf_ld[b]});
    }
    int64_t* d_dd;
    if ((rc = tmp4.alloc(&d_dd, (int64_t)dd.size()))) return fail(rc);
    HMX_CUDA_TRY(cudaMemcpyAsync(d_dd, dd.data(), sizeof(int64_t) * dd.size(), cudaMemcpyHostToDevice, c.stream));
    if ((rc = launch_dense_fill(c, P, pts.soa, d_dd, (int64_t)dd.size() / 6, H.d_row, d_err))) return fail(rc);
  }
  HMX_CUDA_TRY(cudaEventRecord(ev[4], c.stream));
  tick("dense leaves");

  // ---- 4b. U' = U W_U, V' = V W_V -------------------------------------------------------------
  {
    // one batched launch for every low-rank leaf of every pass, both sides
    std::vector<FormDesc> fd;
    std::vector<int64_t> ts;
    int64_t ntiles = 0;
    for (AcaPass& ps : passes)
      for (int side = 0; side < 2; ++side)
        for (size_t i = 0; i < ps.blocks.size(); ++i) {
          if (ps.out[i].rank <= 0 || !ps.wptr[i]) continue;
          const int64_t b = ps.blocks[i];
          const int K = ps.out[i].rank;
          const int r = (int)H.rank_after[b];
          if (r == 0) continue;
          FormDesc f;
          const int64_t rows = side == 0 ? d * rows_of(b) : d * cols_of(b);
          f.A = (side == 0 ? ps.U + ps.desc[i].uoff : ps.V + ps.desc[i].voff);
          f.W = ps.wptr[i] + 4 * (int64_t)K * K + (side == 0 ? 0 : (int64_t)K * r);
          f.C = side == 0 ? H.d_row + H.leaf_moff[b] : H.d_v + H.leaf_voff[b];
          f.rows = (int32_t)rows;
          f.K = K;
          f.r = r;
          f.lda = (int32_t)rows;
          f.ldc = (int32_t)rows;
          f.pad = 0;
          ts.push_back(ntiles);
          ntiles += hmx_cdiv(rows, 64) * hmx_cdiv(r, 32);
          fd.push_back(f);
        }
    if (!fd.empty()) {
      DevBuf t5(c);
      FormDesc* d_fd;
      int64_t* d_ts;
      if ((rc = t5.alloc(&d_fd, (int64_t)fd.size()))) return fail(rc);
      if ((rc = t5.alloc(&d_ts, (int64_t)ts.size()))) return fail(rc);
      HMX_CUDA_TRY(cudaMemcpyAsync(d_fd, fd.data(), sizeof(FormDesc) * fd.size(), cudaMemcpyHostToDevice, c.stream));
      HMX_CUDA_TRY(cudaMemcpyAsync(d_ts, ts.data(), sizeof(int64_t) * ts.size(), cudaMemcpyHostToDevice, c.stream));
      if ((rc = launch_form(c, d_fd, (int64_t)fd.size(), ntiles, d_ts))) return fail(rc);
    }
  }
  HMX_CUDA_TRY(cudaEventRecord(ev[5], c.stream));
  tick("form U' V'");
  int32_t herr = 0;
  HMX_CUDA_TRY(cudaMemcpyAsync(&herr, d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
  HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  if (herr) {
    hmx_set_error("singular evaluation in a dense leaf");
    return fail(HMX_ESINGULAR);
  }
  float ms[5];
  for (int i = 0; i < 5; ++i) HMX_CUDA_TRY(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
  for (auto& e : ev) cudaEventDestroy(e);
  H.t_aca_ms = ms[0];
  H.t_recomp_ms = ms[1];
  H.t_dense_ms = ms[3];
  H.t_form_ms = ms[4];
  // algorithmic FP64 flops of the factor arithmetic (pair evaluation counted separately)
  double fl = 0;
  for (int64_t b : adm) {
    const double mn = (double)(rows_of(b) + cols_of(b));
    const int64_t s = H.steps[b];
    for (int64_t kk = 0; kk < s; ++kk) {
      const double K = (double)d * kk;
      fl += 8.0 * d * d * mn * K + 8.0 * d * d * mn * (K + d);
    }
    const double K = (double)H.rank_before[b], r = (double)H.rank_after[b];
    fl += 8.0 * 22.0 * K * K * K + 8.0 * d * mn * K * r;
    if (H.flags[b] & 1) {
    } else {
      H.n_unconverged += 1;
    }
  }
  H.flops_assembly = fl;
  passes.clear();
  tick("free workspaces");
  H.t_total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  *out = holder;
  return HMX_OK;
}

int hmx_hmatrix_load(hmx_ctx* ctx, int32_t d, int64_t np, const int64_t* perm, const int64_t* table, int64_t nb,
                     const int64_t* ranks, const double* const* a, const double* const* bptr, hmx_hmatrix** out) {
  if (!ctx || !perm || !table || !a || !out || (d != 1 && d != 3) || np <= 0) return HMX_EINVAL;
  int rc = validate_table(table, nb, np);
  if (rc) return rc;
  Ctx& c = ctx->c;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  auto holder = new hmx_hmatrix;
  DeviceH& H = holder->H;
  H.ctx = &c;
  H.d = d;
  H.kind = d == 1 ? 0 : 1;
  H.np = np;
  H.n = d * np;
  H.nb = nb;
  H.table.assign(table, table + 5 * nb);
  H.steps.assign(nb, 0);
  H.rank_before.assign(nb, 0);
  H.rank_after.assign(nb, 0);
  H.flags.assign(nb, 1);
  for (int64_t b = 0; b < nb; ++b)
    if (table[5 * b] == 1) H.rank_after[b] = H.rank_before[b] = ranks ? ranks[b] : 0;
  auto fail = [&](int code) {
    free_h(H);
    delete holder;
    return code;
  };
  {
    std::vector<int64_t> p(perm, perm + np);
    if ((rc = dev_upload(c, &H.d_perm, p))) return fail(rc);
  }
  if ((rc = build_matvec_plan(H))) return fail(rc);
  std::vector<double2> row(H.row_elems), vs(std::max<int64_t>(H.v_elems, 0));
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t m = table[5 * b + 2] - table[5 * b + 1], n = table[5 * b + 4] - table[5 * b + 3];
    const int64_t dm = d * m, dn = d * n, ld = H.leaf_ld[b];
    const double2* A = reinterpret_cast<const double2*>(a[b]);
    if (table[5 * b] == 0) {
      for (int64_t i = 0; i < dm; ++i)
        for (int64_t j = 0; j < dn; ++j) row[H.leaf_moff[b] + j * ld + i] = A[i * dn + j];
    } else {
      const int64_t r = H.rank_after[b];
      if (r == 0) continue;
      const double2* Bv = reinterpret_cast<const double2*>(bptr[b]);
      for (int64_t i = 0; i < dm; ++i)
        for (int64_t l = 0; l < r; ++l) row[H.leaf_moff[b] + l * ld + i] = A[i * r + l];
      for (int64_t i = 0; i < dn; ++i)
        for (int64_t l = 0; l < r; ++l) vs[H.leaf_voff[b] + l * dn + i] = Bv[i * r + l];
    }
  }
  HMX_CUDA_TRY(cudaMemcpy(H.d_row, row.data(), sizeof(double2) * row.size(), cudaMemcpyHostToDevice));
  if (!vs.empty()) HMX_CUDA_TRY(cudaMemcpy(H.d_v, vs.data(), sizeof(double2) * vs.size(), cudaMemcpyHostToDevice));
  *out = holder;
  return HMX_OK;
}

int hmx_hmatrix_splice(const hmx_hmatrix* base, const hmx_hmatrix* sub, const int64_t* idx, hmx_hmatrix** out) {
  if (!base || !sub || !idx || !out) return HMX_EINVAL;
  const DeviceH& B = base->H;
  const DeviceH& S = sub->H;
  if (B.ctx != S.ctx || B.d != S.d || B.np != S.np) {
    hmx_set_error("hmx_hmatrix_splice: the two H-matrices differ in context, d or point count");
    return HMX_EINVAL;
  }
  std::vector<int64_t> src((size_t)B.nb, -1);  // base leaf -> sub leaf (or -1: keep the base leaf)
  for (int64_t j = 0; j < S.nb; ++j) {
    const int64_t b = idx[j];
    if (b < 0 || b >= B.nb || src[(size_t)b] >= 0 ||
        !std::equal(S.table.begin() + 5 * j, S.table.begin() + 5 * j + 5, B.table.begin() + 5 * b)) {
      hmx_set_error("hmx_hmatrix_splice: sub leaf %lld does not match base leaf %lld", (long long)j, (long long)b);
      return HMX_EINVAL;
    }
    src[(size_t)b] = j;
  }
  Ctx& c = *B.ctx;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  auto holder = new hmx_hmatrix;
  DeviceH& H = holder->H;
  H.ctx = &c;
  H.kind = B.kind;
  H.d = B.d;
  H.np = B.np;
  H.n = B.n;
  H.nb = B.nb;
  H.table = B.table;
  H.steps = B.steps;
  H.rank_before = B.rank_before;
  H.rank_after = B.rank_after;
  H.flags = B.flags;
  H.pairs_evaluated = B.pairs_evaluated + S.pairs_evaluated;
  H.aca_passes = B.aca_passes;
  H.n_fallback = B.n_fallback;
  H.n_unconverged = B.n_unconverged;
  H.n_regularized = B.n_regularized;
  H.flops_assembly = B.flops_assembly + S.flops_assembly;
  H.t_dense_ms = B.t_dense_ms;
  H.t_aca_ms = B.t_aca_ms + S.t_aca_ms;
  H.t_recomp_ms = B.t_recomp_ms + S.t_recomp_ms;
  H.t_form_ms = B.t_form_ms + S.t_form_ms;
  H.t_total_ms = B.t_total_ms + S.t_total_ms;
  for (int64_t b = 0; b < H.nb; ++b) {
    const int64_t j = src[(size_t)b];
    if (j < 0) continue;
    H.steps[b] = S.steps[j];
    H.rank_before[b] = S.rank_before[j];
    H.rank_after[b] = S.rank_after[j];
    H.flags[b] = S.flags[j] | 256;  // bit 8: re-compressed by the certification pass
    H.n_fallback += (S.flags[j] & 128) ? 1 : 0;
  }
  auto fail = [&](int code) {
    free_h(H);
    delete holder;
    return code;
  };
  int rc;
  {
    std::vector<int64_t> p((size_t)H.np);
    HMX_CUDA_TRY(cudaMemcpy(p.data(), B.d_perm, sizeof(int64_t) * H.np, cudaMemcpyDeviceToHost));
    if ((rc = dev_upload(c, &H.d_perm, p))) return fail(rc);
  }
  if ((rc = build_matvec_plan(H))) return fail(rc);
  std::vector<Copy2D> cp;
  cp.reserve(2 * (size_t)H.nb);
  for (int64_t b = 0; b < H.nb; ++b) {
    const int64_t j = src[(size_t)b];
    const DeviceH& F = j < 0 ? B : S;
    const int64_t fb = j < 0 ? b : j;
    const int64_t dm = H.d * (H.table[5 * b + 2] - H.table[5 * b + 1]);
    const int64_t dn = H.d * (H.table[5 * b + 4] - H.table[5 * b + 3]);
    if (H.table[5 * b] == 0) {
      cp.push_back(Copy2D{F.d_row + F.leaf_moff[fb], H.d_row + H.leaf_moff[b], F.leaf_ld[fb], H.leaf_ld[b], dm, dn});
    } else if (H.rank_after[b] > 0) {
      const int64_t r = H.rank_after[b];
      cp.push_back(Copy2D{F.d_row + F.leaf_moff[fb], H.d_row + H.leaf_moff[b], F.leaf_ld[fb], H.leaf_ld[b], dm, r});
      cp.push_back(Copy2D{F.d_v + F.leaf_voff[fb], H.d_v + H.leaf_voff[b], dn, dn, dn, r});
    }
  }
  if (!cp.empty()) {
    DevBuf t(c);
    Copy2D* d_cp;
    if ((rc = t.alloc(&d_cp, (int64_t)cp.size()))) return fail(rc);
    HMX_CUDA_TRY(cudaMemcpyAsync(d_cp, cp.data(), sizeof(Copy2D) * cp.size(), cudaMemcpyHostToDevice, c.stream));
    copy2d_batch<<<(unsigned)cp.size(), 256, 0, c.stream>>>(d_cp);
    HMX_CUDA_TRY(cudaGetLastError());
    HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  }
  *out = holder;
  return HMX_OK;
}

int hmx_hmatrix_stats(const hmx_hmatrix* h, hmx_stats* st) {
  if (!h || !st) return HMX_EINVAL;
  const DeviceH& H = h->H;
  std::memset(st, 0, sizeof(*st));
  st->n_blocks = H.nb;
  for (int64_t b = 0; b < H.nb; ++b) {
    const int64_t m = H.table[5 * b + 2] - H.table[5 * b + 1], n = H.table[5 * b + 4] - H.table[5 * b + 3];
    if (H.table[5 * b] == 0) {
      st->n_dense++;
      st->n_stored += (int64_t)H.d * H.d * m * n;
    } else {
      st->n_lowrank++;
      st->n_stored += H.rank_after[b] * H.d * (m + n);
      st->max_rank_before = std::max(st->max_rank_before, H.rank_before[b]);
      st->max_rank_after = std::max(st->max_rank_after, H.rank_after[b]);
      st->aca_steps_total += H.steps[b];
    }
  }
  st->pairs_evaluated = H.pairs_evaluated;
  for (int64_t b = 0; b < H.nb; ++b)
    if (H.table[5 * b] == 0)
      st->pairs_evaluated += (H.table[5 * b + 2] - H.table[5 * b + 1]) * (H.table[5 * b + 4] - H.table[5 * b + 3]);
  st->n_fallback = H.n_fallback;
  st->n_unconverged = H.n_unconverged;
  st->n_regularized = H.n_regularized;
  st->aca_passes = H.aca_passes;
  st->row_elems = H.row_elems;
  st->v_elems = H.v_elems;
  st->n_levels = H.nlevels;
  st->n_tiles = H.ntile2;
  st->n_jobs = H.njob1;
  st->t_dense_ms = H.t_dense_ms;
  st->t_aca_ms = H.t_aca_ms;
  st->t_recompress_ms = H.t_recomp_ms;
  st->t_form_ms = H.t_form_ms;
  st->t_total_ms = H.t_total_ms;
  st->flops_assembly = H.flops_assembly;
  st->matvec_bytes = H.mv_bytes;
  st->dense_bytes = H.dense_bytes;
  st->lowrank_bytes = H.lr_bytes;
  st->phase1_bytes = H.phase1_bytes;
  st->phase2_bytes = H.phase2_bytes;
  return HMX_OK;
}

int hmx_hmatrix_block_info(const hmx_hmatrix* h, int64_t* steps, int64_t* rank_before, int64_t* rank_after,
                           int32_t* flags) {
  if (!h) return HMX_EINVAL;
  const DeviceH& H = h->H;
  for (int64_t b = 0; b < H.nb; ++b) {
    if (steps) steps[b] = H.steps[b];
    if (rank_before) rank_before[b] = H.rank_before[b];
    if (rank_after) rank_after[b] = H.rank_after[b];
    if (flags) flags[b] = H.flags[b];
  }
  return HMX_OK;
}

int hmx_hmatrix_set_block_info(hmx_hmatrix* h, const int64_t* steps, const int64_t* rank_before,
                               const int32_t* flags) {
  if (!h) return HMX_EINVAL;
  DeviceH& H = h->H;
  for (int64_t b = 0; b < H.nb; ++b) {
    if (rank_before && rank_before[b] < H.rank_after[b]) {
      hmx_set_error("block %lld: rank before recompression %lld < stored rank %lld", (long long)b,
                    (long long)rank_before[b], (long long)H.rank_after[b]);
      return HMX_EINVAL;
    }
  }
  for (int64_t b = 0; b < H.nb; ++b) {
    if (steps) H.steps[b] = steps[b];
    if (rank_before) H.rank_before[b] = rank_before[b];
    if (flags) H.flags[b] = flags[b];
  }
  return HMX_OK;
}

int hmx_hmatrix_device_layout(const hmx_hmatrix* h, int64_t* moff, int64_t* ld, int64_t* voff, uint64_t* bufs) {
  if (!h || !moff || !ld || !voff || !bufs) return HMX_EINVAL;
  const DeviceH& H = h->H;
  HMX_CUDA_TRY(cudaSetDevice(H.ctx->device));
  HMX_CUDA_TRY(cudaStreamSynchronize(H.ctx->stream));
  for (int64_t b = 0; b < H.nb; ++b) {
    moff[b] = H.leaf_moff[b];
    ld[b] = H.leaf_ld[b];
    voff[b] = H.leaf_voff[b];
  }
  bufs[0] = reinterpret_cast<uint64_t>(H.d_row);
  bufs[1] = static_cast<uint64_t>(H.row_elems);
  bufs[2] = reinterpret_cast<uint64_t>(H.d_v);
  bufs[3] = static_cast<uint64_t>(H.v_elems);
  return HMX_OK;
}

int hmx_hmatrix_get_block(const hmx_hmatrix* h, int64_t b, double* a, double* v) {
  if (!h || !a || b < 0 || b >= h->H.nb) return HMX_EINVAL;
  const DeviceH& H = h->H;
  HMX_CUDA_TRY(cudaSetDevice(H.ctx->device));
  const int d = H.d;
  const int64_t m = H.table[5 * b + 2] - H.table[5 * b + 1], n = H.table[5 * b + 4] - H.table[5 * b + 3];
  const int64_t dm = d * m, dn = d * n, ld = H.leaf_ld[b];
  double2* A = reinterpret_cast<double2*>(a);
  HMX_CUDA_TRY(cudaStreamSynchronize(H.ctx->stream));
  if (H.table[5 * b] == 0) {
    std::vector<double2> t(dm * dn);
    HMX_CUDA_TRY(cudaMemcpy(t.data(), H.d_row + H.leaf_moff[b], sizeof(double2) * t.size(), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < dm; ++i)
      for (int64_t j = 0; j < dn; ++j) A[i * dn + j] = t[j * ld + i];
    return HMX_OK;
  }
  const int64_t r = H.rank_after[b];
  if (r == 0) return HMX_OK;
  if (!v) return HMX_EINVAL;
  double2* Vh = reinterpret_cast<double2*>(v);
  std::vector<double2> tu(dm * r), tv(dn * r);
  HMX_CUDA_TRY(cudaMemcpy(tu.data(), H.d_row + H.leaf_moff[b], sizeof(double2) * tu.size(), cudaMemcpyDeviceToHost));
  HMX_CUDA_TRY(cudaMemcpy(tv.data(), H.d_v + H.leaf_voff[b], sizeof(double2) * tv.size(), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < dm; ++i)
    for (int64_t l = 0; l < r; ++l) A[i * r + l] = tu[l * ld + i];
  for (int64_t i = 0; i < dn; ++i)
    for (int64_t l = 0; l < r; ++l) Vh[i * r + l] = tv[l * dn + i];
  return HMX_OK;
}

int hmx_block_errors(hmx_hmatrix* h, const hmx_kernel* k, const double* pts_tree, const double* nrm_tree,
                     int64_t n_points, double self_shift, double* err2, double* norm2) {
  if (!h || !k || !pts_tree || !err2 || !norm2) return HMX_EINVAL;
  DeviceH& H = h->H;
  Ctx& c = *H.ctx;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  const int d = k->kind == HMX_HELMHOLTZ ? 1 : 3;
  if (d != H.d || n_points != H.np) {
    hmx_set_error("hmx_block_errors: kernel / point count do not match the H-matrix");
    return HMX_EINVAL;
  }
  if (k->kind == HMX_ELASTO_T && !nrm_tree) {
    hmx_set_error("hmx_block_errors: elasto T needs normals");
    return HMX_EINVAL;
  }
  const GreenParams P = make_params(k, 1, self_shift);
  DevPoints pts;
  int rc;
  if ((rc = pts.upload(c, pts_tree, k->kind == HMX_ELASTO_T ? nrm_tree : nullptr, n_points))) return rc;
  const int64_t nb = H.nb;
  std::vector<ErrDesc> desc((size_t)nb);
  std::vector<int64_t> tile_start((size_t)nb);
  int64_t nt = 0;
  for (int64_t b = 0; b < nb; ++b) {
    ErrDesc& e = desc[b];
    e.r0 = H.table[5 * b + 1];
    e.c0 = H.table[5 * b + 3];
    e.m = (int32_t)(H.table[5 * b + 2] - H.table[5 * b + 1]);
    e.n = (int32_t)(H.table[5 * b + 4] - H.table[5 * b + 3]);
    e.pad = 0;
    const bool lowrank = H.table[5 * b] != 0;
    e.r = lowrank ? (int32_t)H.rank_after[b] : 0;
    e.U = lowrank ? H.d_row + H.leaf_moff[b] : nullptr;
    e.V = lowrank ? H.d_v + H.leaf_voff[b] : nullptr;
    e.ldu = H.leaf_ld[b];
    tile_start[b] = nt;
    nt += err_tiles_of(e.m, e.n);
  }
  if (nt >= (int64_t)INT32_MAX) {
    hmx_set_error("hmx_block_errors: %lld tiles exceed one grid", (long long)nt);
    return HMX_EINVAL;
  }
  DevBuf mem(c);
  ErrDesc* d_desc;
  int64_t* d_ts;
  double2 *d_part, *d_out;
  if ((rc = mem.alloc(&d_desc, nb)) || (rc = mem.alloc(&d_ts, nb)) || (rc = mem.alloc(&d_part, nt)) ||
      (rc = mem.alloc(&d_out, nb)))
    return rc;
  HMX_CUDA_TRY(cudaMemcpyAsync(d_desc, desc.data(), sizeof(ErrDesc) * nb, cudaMemcpyHostToDevice, c.stream));
  HMX_CUDA_TRY(cudaMemcpyAsync(d_ts, tile_start.data(), sizeof(int64_t) * nb, cudaMemcpyHostToDevice, c.stream));
  if ((rc = launch_block_errors(c, d, P, pts.soa, d_desc, d_ts, nb, nt, d_part, d_out))) return rc;
  std::vector<double2> out((size_t)nb);
  HMX_CUDA_TRY(cudaMemcpyAsync(out.data(), d_out, sizeof(double2) * nb, cudaMemcpyDeviceToHost, c.stream));
  HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  for (int64_t b = 0; b < nb; ++b) {
    err2[b] = H.table[5 * b] != 0 ? out[b].x : 0.0;  // dense leaves are stored exactly
    norm2[b] = out[b].y;
  }
  return HMX_OK;
}

void hmx_hmatrix_free(hmx_hmatrix* h) {
  if (!h) return;
  cudaSetDevice(h->H.ctx->device);
  cudaStreamSynchronize(h->H.ctx->stream);
  free_h(h->H);  // waits for the last matvec of every workspace stream
  delete h;
}

int hmx_matvec_on(hmx_hmatrix* h, const double* x, double* y, int32_t mem, uint64_t stream) {
  if (!h || !x || !y || (mem != HMX_HOST && mem != HMX_DEVICE)) return HMX_EINVAL;
  DeviceH& H = h->H;
  HMX_CUDA_TRY(cudaSetDevice(H.ctx->device));
  const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (mem == HMX_DEVICE)
    return matvec_device(H, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), nullptr, st);
  int rc = HMX_OK;
  MvWorkspace* w = mv_workspace(H, st, &rc);
  if (!w) return rc;
  std::lock_guard<std::mutex> lk(w->mu);  // the staging buffers are this call's until y is on the host
  HMX_CUDA_TRY(cudaMemcpyAsync(w->d_xio, x, sizeof(double2) * H.n, cudaMemcpyHostToDevice, st));
  if ((rc = matvec_enqueue(H, *w, w->d_xio, w->d_yio, nullptr))) return rc;
  HMX_CUDA_TRY(cudaMemcpyAsync(y, w->d_yio, sizeof(double2) * H.n, cudaMemcpyDeviceToHost, st));
  HMX_CUDA_TRY(cudaStreamSynchronize(st));
  return HMX_OK;
}

int hmx_matvec(hmx_hmatrix* h, const double* x, double* y, int32_t mem) {
  if (!h) return HMX_EINVAL;
  return hmx_matvec_on(h, x, y, mem, reinterpret_cast<uint64_t>(h->H.ctx->stream));
}

int hmx_matvec_profile(hmx_hmatrix* h, const double* x_dev, double* y_dev, float* phase_ms) {
  if (!h || !x_dev || !y_dev || !phase_ms) return HMX_EINVAL;
  HMX_CUDA_TRY(cudaSetDevice(h->H.ctx->device));
  return matvec_device(h->H, reinterpret_cast<const double2*>(x_dev), reinterpret_cast<double2*>(y_dev), phase_ms,
                       h->H.ctx->stream);
}

int hmx_profile_begin(hmx_hmatrix* h) {
  if (!h) return HMX_EINVAL;
  for (cudaEvent_t e : h->H.prof_events) cudaEventDestroy(e);
  h->H.prof_events.clear();
  h->H.profiling = true;
  return HMX_OK;
}

int hmx_profile_end(hmx_hmatrix* h, int64_t* n_calls, double* phase_ms_sum) {
  if (!h || !n_calls || !phase_ms_sum) return HMX_EINVAL;
  DeviceH& H = h->H;
  H.profiling = false;
  HMX_CUDA_TRY(cudaStreamSynchronize(H.ctx->stream));
  const size_t nc = H.prof_events.size() / 5;
  for (int i = 0; i < 4; ++i) phase_ms_sum[i] = 0.0;
  for (size_t k = 0; k < nc; ++k)
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      HMX_CUDA_TRY(cudaEventElapsedTime(&ms, H.prof_events[5 * k + i], H.prof_events[5 * k + i + 1]));
      phase_ms_sum[i] += ms;
    }
  for (cudaEvent_t e : H.prof_events) cudaEventDestroy(e);
  H.prof_events.clear();
  *n_calls = (int64_t)nc;
  return HMX_OK;
}

int hmx_bench_read_bw(hmx_ctx* ctx, double* gbs) {
  if (!ctx || !gbs) return HMX_EINVAL;
  HMX_CUDA_TRY(cudaSetDevice(ctx->c.device));
  return hmx::bench_read_bw(ctx->c, gbs);
}

int hmx_bench_dfma(hmx_ctx* ctx, double* tflops) {
  if (!ctx || !tflops) return HMX_EINVAL;
  HMX_CUDA_TRY(cudaSetDevice(ctx->c.device));
  return hmx::bench_dfma(ctx->c, tflops);
}

int hmx_gmres(hmx_hmatrix* h, const double* b, double* x, double tol, int32_t restart, int64_t max_iters,
              int32_t mem, int64_t* iters, double* history, int64_t history_cap, int64_t* history_len,
              int32_t* converged) {
  if (!h || !b || !x || !iters || !converged || restart < 1 || !(tol > 0)) return HMX_EINVAL;
  DeviceH& H = h->H;
  Ctx& c = *H.ctx;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  const double2* db = reinterpret_cast<const double2*>(b);
  double2* dx = reinterpret_cast<double2*>(x);
  DevBuf tmp(c);
  int rc;
  if (mem == HMX_HOST) {
    double2 *tb, *tx;
    if ((rc = tmp.alloc(&tb, H.n))) return rc;
    if ((rc = tmp.alloc(&tx, H.n))) return rc;
    HMX_CUDA_TRY(cudaMemcpyAsync(tb, b, sizeof(double2) * H.n, cudaMemcpyHostToDevice, c.stream));
    db = tb;
    dx = tx;
  }
  std::vector<double> hist;
  int conv = 0;
  rc = gmres_device(H, db, dx, tol, restart, max_iters, iters, hist, &conv, c.stream);
  if (rc) return rc;
  if (mem == HMX_HOST) {
    HMX_CUDA_TRY(cudaMemcpyAsync(x, dx, sizeof(double2) * H.n, cudaMemcpyDeviceToHost, c.stream));
  }
  HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  *converged = conv;
  if (history_len) *history_len = (int64_t)hist.size();
  if (history)
    for (int64_t i = 0; i < std::min<int64_t>(history_cap, (int64_t)hist.size()); ++i) history[i] = hist[i];
  return HMX_OK;
}

}  // extern "C"

// ---- single-block low-rank entry points (aca_partial /
// aca_vector on a BlockGenerator, recompress on a LowRankFactor) -------------------
// The same device kernels as the batched assembly (aca_kernel, recompress_core,
// form_gemm) run on one block, so the reference's lowrank API gets the device
// algorithm leaf by leaf.
namespace {

// G(:, :) = F^H F for a (rows x K) column-major panel, ld = rows; thread per entry
__global__ void gram_full(const double2* __restrict__ F, int64_t rows, int K, double2* __restrict__ G, int ldg) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * K) return;
  const int i = t % K, j = t / K;
  double2 s = cmk(0.0, 0.0);
  for (int64_t q = 0; q < rows; ++q) s = cfma_ca(F[q + (int64_t)i * rows], F[q + (int64_t)j * rows], s);
  if (i == j) s.y = 0.0;
  G[i + (int64_t)j * ldg] = s;
}

// row-major host (rows x cols) <-> column-major device (ld = rows)
void to_colmajor(const double2* h, int64_t rows, int64_t cols, std::vector<double2>& out) {
  out.resize((size_t)(rows * cols));
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) out[(size_t)(i + j * rows)] = h[i * cols + j];
}
void from_colmajor(const std::vector<double2>& in, int64_t rows, int64_t cols, int64_t ldh, double2* h) {
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) h[i * ldh + j] = in[(size_t)(i + j * rows)];
}

// Recompression of device factors U (dm x K), V (dn x K) with their Gram pair
// in G (kcap = K); W: 6 K^2 workspace; results into Uo (dm x r), Vo (dn x r).
int recompress_device(Ctx& c, DevBuf& mem, const double2* dU, const double2* dV, int64_t dm, int64_t dn, int K,
                      double2* G, double eps, int rule, int* r_out, double2** Uo, double2** Vo) {
  RecDesc rd;
  rd.goff = 0;
  rd.woff = 0;
  rd.K = K;
  rd.kcap = K;
  double2* W;
  RecDesc* d_rd;
  int32_t *d_rank, *d_flag;
  int rc;
  if ((rc = mem.alloc(&W, 6 * (int64_t)K * K)) || (rc = mem.alloc(&d_rd, 1)) || (rc = mem.alloc(&d_rank, 1)) ||
      (rc = mem.alloc(&d_flag, 1)))
    return rc;
  HMX_CUDA_TRY(cudaMemcpyAsync(d_rd, &rd, sizeof(RecDesc), cudaMemcpyHostToDevice, c.stream));
  if ((rc = launch_recompress_core(c, d_rd, 1, K, eps, rule, G, W, d_rank, d_flag))) return rc;
  int32_t hr = 0;
  HMX_CUDA_TRY(cudaMemcpyAsync(&hr, d_rank, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
  HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  *r_out = hr;
  if (hr == 0) return HMX_OK;
  if ((rc = mem.alloc(Uo, dm * hr)) || (rc = mem.alloc(Vo, dn * hr))) return rc;
  FormDesc fd[2];
  int64_t ts[2];
  int64_t nt = 0;
  for (int side = 0; side < 2; ++side) {
    FormDesc& f = fd[side];
    const int64_t rows = side == 0 ? dm : dn;
    f.A = side == 0 ? dU : dV;
    f.W = W + 4 * (int64_t)K * K + (side == 0 ? 0 : (int64_t)K * hr);
    f.C = side == 0 ? *Uo : *Vo;
    f.rows = (int32_t)rows;
    f.K = K;
    f.r = hr;
    f.lda = (int32_t)rows;
    f.ldc = (int32_t)rows;
    f.pad = 0;
    ts[side] = nt;
    nt += hmx_cdiv(rows, 64) * hmx_cdiv(hr, 32);
  }
  FormDesc* d_fd;
  int64_t* d_ts;
  if ((rc = mem.alloc(&d_fd, 2)) || (rc = mem.alloc(&d_ts, 2))) return rc;
  HMX_CUDA_TRY(cudaMemcpyAsync(d_fd, fd, sizeof(fd), cudaMemcpyHostToDevice, c.stream));
  HMX_CUDA_TRY(cudaMemcpyAsync(d_ts, ts, sizeof(ts), cudaMemcpyHostToDevice, c.stream));
  return launch_form(c, d_fd, 2, nt, d_ts);
}

// ---- batched truncation of accumulated factor pairs (H-arithmetic) ---------------------------
struct GramItem {
  const double2* F;  // rows x K, column-major (ld = rows)
  int64_t rows;
  int32_t K, pad;
  double2* G;  // K x K, ld = K
};

// G = F^H F, one 16 x 16 output tile per CTA; 32-row chunks of both column groups staged in shared
// memory with coalesced column reads
__global__ void __launch_bounds__(256) gram_batch(const GramItem* __restrict__ items, const int2* __restrict__ tiles) {
  __shared__ double2 sa[32][17];
  __shared__ double2 sb[32][17];
  const int2 tl = tiles[blockIdx.x];
  const GramItem it = items[tl.x];
  const int K = it.K;
  const int nt = (K + 15) / 16;
  const int i0 = (tl.y % nt) * 16, j0 = (tl.y / nt) * 16;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double2 s = cmk(0.0, 0.0);
  for (int64_t q0 = 0; q0 < it.rows; q0 += 32) {
    for (int e = threadIdx.x; e < 512; e += 256) {
      const int r = e & 31, cc = e >> 5;
      const int64_t q = q0 + r;
      sa[r][cc] = (q < it.rows && i0 + cc < K) ? it.F[q + (int64_t)(i0 + cc) * it.rows] : cmk(0.0, 0.0);
      sb[r][cc] = (q < it.rows && j0 + cc < K) ? it.F[q + (int64_t)(j0 + cc) * it.rows] : cmk(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < 32; ++r) s = cfma_ca(sa[r][ty], sb[r][tx], s);
    __syncthreads();
  }
  const int i = i0 + ty, j = j0 + tx;
  if (i < K && j < K) {
    if (i == j) s.y = 0.0;
    it.G[i + (int64_t)j * K] = s;
  }
}

}  // namespace

extern "C" {

int hmx_aca_block(hmx_ctx* ctx, const hmx_kernel* k, const double* X, int64_t m, const double* Y, int64_t n,
                  const double* NY, int32_t has_shift, double shift, const hmx_aca_cfg* cfg, int32_t recompress,
                  int64_t cap, double* U, double* V, int64_t* rank, int64_t* steps, int32_t* status) {
  if (!ctx || !k || !X || !Y || !cfg || !U || !V || !rank || !steps || !status || m <= 0 || n <= 0 || cap < 0)
    return HMX_EINVAL;
  if (k->kind == HMX_ELASTO_T && !NY) {
    hmx_set_error("hmx_aca_block: elasto T needs column normals");
    return HMX_EINVAL;
  }
  Ctx& c = ctx->c;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  const int d = k->kind == HMX_HELMHOLTZ ? 1 : 3;
  const int64_t dmin = d * std::min(m, n);
  const int64_t maxr = cfg->max_rank > 0 ? std::min<int64_t>(cfg->max_rank, dmin) : dmin;
  if (maxr > 1020) {
    hmx_set_error("hmx_aca_block: max rank %lld above the device limit 1020", (long long)maxr);
    return HMX_EINVAL;
  }
  // points of the block: rows then columns (normals only matter for columns)
  std::vector<double> pts((size_t)(3 * (m + n))), nrm;
  std::copy(X, X + 3 * m, pts.begin());
  std::copy(Y, Y + 3 * n, pts.begin() + 3 * m);
  if (NY) {
    nrm.assign((size_t)(3 * (m + n)), 0.0);
    std::copy(NY, NY + 3 * n, nrm.begin() + 3 * m);
  }
  DevPoints P3;
  int rc;
  if ((rc = P3.upload(c, pts.data(), NY ? nrm.data() : nullptr, m + n))) return rc;
  const GreenParams P = make_params(k, has_shift, shift);
  const double s3f = cfg->sigma3_floor > 0 ? cfg->sigma3_floor : 1e-12;
  int64_t kc = std::min<int64_t>(maxr, 64);
  kc = std::max<int64_t>(d, (kc / d) * d);
  for (;;) {
    DevBuf mem(c);
    AcaDesc ds;
    ds.r0 = 0;
    ds.c0 = m;
    ds.m = (int32_t)m;
    ds.n = (int32_t)n;
    ds.kcap = (int32_t)kc;
    ds.max_rank = (int32_t)maxr;
    ds.uoff = 0;
    ds.voff = 0;
    ds.goff = 0;
    double2 *dU, *dV, *G;
    AcaDesc* d_desc;
    AcaOut* d_out;
    int32_t* d_order;
    if ((rc = mem.alloc(&dU, d * m * kc)) || (rc = mem.alloc(&dV, d * n * kc)) || (rc = mem.alloc(&G, 2 * kc * kc)) ||
        (rc = mem.alloc(&d_desc, 1)) || (rc = mem.alloc(&d_out, 1)) || (rc = mem.alloc(&d_order, 1)))
      return rc;
    const int32_t zero = 0;
    HMX_CUDA_TRY(cudaMemcpyAsync(d_desc, &ds, sizeof(AcaDesc), cudaMemcpyHostToDevice, c.stream));
    HMX_CUDA_TRY(cudaMemcpyAsync(d_order, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
    const int variant = m + n < kAcaNarrowMax ? kAcaNarrow : kAcaWide;
    if ((rc = launch_aca(c, d, P, P3.soa, d_desc, d_order, 1, (int)kc, (int)m, cfg->eps, s3f, dU, dV, G, d_out,
                         variant, 0)))
      return rc;
    AcaOut o;
    HMX_CUDA_TRY(cudaMemcpyAsync(&o, d_out, sizeof(AcaOut), cudaMemcpyDeviceToHost, c.stream));
    HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
    if (o.status & 4) {  // column capacity: rerun with twice the columns (same result)
      if (kc >= maxr) {
        hmx_set_error("hmx_aca_block: capacity overflow at the maximal rank");
        return HMX_ENOMEM;
      }
      kc = std::min<int64_t>(maxr, 2 * kc);
      kc = std::max<int64_t>(d, (kc / d) * d);
      continue;
    }
    *steps = o.steps;
    *status = o.status;
    if (o.status & 8) {
      *rank = 0;
      hmx_set_error("hmx_aca_block: all sigma_3 pivots below the floor (FallbackNeeded)");
      return HMX_EPIVOT;
    }
    int K = o.rank;
    const double2* srcU = dU;
    const double2* srcV = dV;
    int64_t ldU = d * m, ldV = d * n;
    if (recompress && K > 0) {
      // the Gram pair of the ACA factors has ld kcap; recompress_core wants kcap = K
      double2* G2;
      if ((rc = mem.alloc(&G2, 2 * (int64_t)K * K))) return rc;
      HMX_CUDA_TRY(cudaMemcpy2DAsync(G2, sizeof(double2) * K, G, sizeof(double2) * kc, sizeof(double2) * K, K,
                                     cudaMemcpyDeviceToDevice, c.stream));
      HMX_CUDA_TRY(cudaMemcpy2DAsync(G2 + (int64_t)K * K, sizeof(double2) * K, G + kc * kc, sizeof(double2) * kc,
                                     sizeof(double2) * K, K, cudaMemcpyDeviceToDevice, c.stream));
      int r = 0;
      double2 *Uo = nullptr, *Vo = nullptr;
      if ((rc = recompress_device(c, mem, dU, dV, d * m, d * n, K, G2, cfg->eps_recompress > 0 ? cfg->eps_recompress : cfg->eps,
                                     cfg->trunc_rule, &r, &Uo, &Vo)))
        return rc;
      K = r;
      srcU = Uo;
      srcV = Vo;
    }
    if (K > cap) {
      hmx_set_error("hmx_aca_block: rank %d exceeds the output capacity %lld", K, (long long)cap);
      return HMX_EINVAL;
    }
    *rank = K;
    if (K > 0) {
      std::vector<double2> hu((size_t)(ldU * K)), hv((size_t)(ldV * K));
      HMX_CUDA_TRY(cudaMemcpyAsync(hu.data(), srcU, sizeof(double2) * hu.size(), cudaMemcpyDeviceToHost, c.stream));
      HMX_CUDA_TRY(cudaMemcpyAsync(hv.data(), srcV, sizeof(double2) * hv.size(), cudaMemcpyDeviceToHost, c.stream));
      HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
      from_colmajor(hu, ldU, K, cap, reinterpret_cast<double2*>(U));
      from_colmajor(hv, ldV, K, cap, reinterpret_cast<double2*>(V));
    }
    return HMX_OK;
  }
}

int hmx_recompress(hmx_ctx* ctx, int64_t dm, int64_t dn, int64_t K, const double* U, const double* V, double eps,
                   int32_t trunc_rule, int64_t* rank, double* Uout, double* Vout) {
  if (!ctx || !U || !V || !rank || !Uout || !Vout || dm <= 0 || dn <= 0 || K < 0) return HMX_EINVAL;
  if (K > 1020) {
    hmx_set_error("hmx_recompress: rank %lld above the device limit 1020", (long long)K);
    return HMX_EINVAL;
  }
  *rank = 0;
  if (K == 0) return HMX_OK;
  Ctx& c = ctx->c;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  DevBuf mem(c);
  std::vector<double2> hu, hv;
  to_colmajor(reinterpret_cast<const double2*>(U), dm, K, hu);
  to_colmajor(reinterpret_cast<const double2*>(V), dn, K, hv);
  double2 *dU, *dV, *G;
  int rc;
  if ((rc = mem.alloc(&dU, dm * K)) || (rc = mem.alloc(&dV, dn * K)) || (rc = mem.alloc(&G, 2 * K * K))) return rc;
  HMX_CUDA_TRY(cudaMemcpyAsync(dU, hu.data(), sizeof(double2) * hu.size(), cudaMemcpyHostToDevice, c.stream));
  HMX_CUDA_TRY(cudaMemcpyAsync(dV, hv.data(), sizeof(double2) * hv.size(), cudaMemcpyHostToDevice, c.stream));
  const int nthr = 128, nblk = (int)hmx_cdiv(K * K, nthr);
  gram_full<<<nblk, nthr, 0, c.stream>>>(dU, dm, (int)K, G, (int)K);
  gram_full<<<nblk, nthr, 0, c.stream>>>(dV, dn, (int)K, G + K * K, (int)K);
  HMX_CUDA_TRY(cudaGetLastError());
  int r = 0;
  double2 *Uo = nullptr, *Vo = nullptr;
  if ((rc = recompress_device(c, mem, dU, dV, dm, dn, (int)K, G, eps, trunc_rule, &r, &Uo, &Vo))) return rc;
  *rank = r;
  if (r > 0) {
    std::vector<double2> ou((size_t)(dm * r)), ov((size_t)(dn * r));
    HMX_CUDA_TRY(cudaMemcpyAsync(ou.data(), Uo, sizeof(double2) * ou.size(), cudaMemcpyDeviceToHost, c.stream));
    HMX_CUDA_TRY(cudaMemcpyAsync(ov.data(), Vo, sizeof(double2) * ov.size(), cudaMemcpyDeviceToHost, c.stream));
    HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
    from_colmajor(ou, dm, r, r, reinterpret_cast<double2*>(Uout));
    from_colmajor(ov, dn, r, r, reinterpret_cast<double2*>(Vout));
  }
  return HMX_OK;
}

int hmx_rsvd(hmx_ctx* ctx, const double* A, int64_t m, int64_t n, double eps, int32_t oversample, int64_t max_rank,
             int64_t seed, double* U, double* V, int64_t* k, int32_t* converged) {
  if (!ctx || !A || !U || !V || !k || !converged || m <= 0 || n <= 0 || oversample < 0) return HMX_EINVAL;
  if (!(eps > 0 && eps < 1)) {
    hmx_set_error("hmx_rsvd: eps must be in (0, 1)");
    return HMX_EINVAL;
  }
  Ctx& c = ctx->c;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  const int64_t cap = std::min<int64_t>(max_rank > 0 ? max_rank : std::min(m, n), std::min(m, n));
  if (cap > kMaxAcaCols) {
    hmx_set_error("hmx_rsvd: column cap %lld above the device limit %d", (long long)cap, kMaxAcaCols);
    return HMX_EINVAL;
  }
  DevBuf mem(c);
  std::vector<double2> ha;
  to_colmajor(reinterpret_cast<const double2*>(A), m, n, ha);
  double2 *dA, *dU, *dV, *G;
  int rc;
  if ((rc = mem.alloc(&dA, m * n)) || (rc = mem.alloc(&dU, m * cap)) || (rc = mem.alloc(&dV, n * cap)) ||
      (rc = mem.alloc(&G, 2 * cap * cap)))
    return rc;
  HMX_CUDA_TRY(cudaMemcpyAsync(dA, ha.data(), sizeof(double2) * ha.size(), cudaMemcpyHostToDevice, c.stream));
  int K = 0, conv = 0;
  if ((rc = rsvd_dense(c, dA, m, n, eps, oversample, cap, (uint64_t)seed, dU, dV, G, &K, &conv))) return rc;
  *k = K;
  *converged = conv;
  if (K > 0) {
    std::vector<double2> ou((size_t)(m * K)), ov((size_t)(n * K));
    HMX_CUDA_TRY(cudaMemcpyAsync(ou.data(), dU, sizeof(double2) * ou.size(), cudaMemcpyDeviceToHost, c.stream));
    HMX_CUDA_TRY(cudaMemcpyAsync(ov.data(), dV, sizeof(double2) * ov.size(), cudaMemcpyDeviceToHost, c.stream));
    HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
    from_colmajor(ou, m, K, K, reinterpret_cast<double2*>(U));
    from_colmajor(ov, n, K, K, reinterpret_cast<double2*>(V));
  }
  return HMX_OK;
}

}  // extern "C"

namespace hmx {

// Batched truncation core shared by hmx_truncate_batch and the H-LU engine (hlu.cu): Gram pairs,
// recompression K classes, rank readback (one host synchronisation), then `outputs` supplies the
// destination of every formed item (ranks / flags known) and U' = U W_U, V' = V W_V are launched.
int truncate_pairs(Ctx& c, int64_t nb, const int64_t* dm, const int64_t* dn, const int64_t* K,
                   const double2* const* U, const double2* const* V, double eps, int32_t trunc_rule, int64_t* ranks,
                   int32_t* flags, const TruncOutputs& outputs) {
  for (int64_t i = 0; i < nb; ++i) {
    ranks[i] = 0;
    flags[i] = 0;
  }
  std::vector<double2*> uo((size_t)nb, nullptr), vo((size_t)nb, nullptr);
  // items with K > 0, largest K first (the recompression launches per K class)
  std::vector<int64_t> live;
  for (int64_t i = 0; i < nb; ++i)
    if (K[i] > 0) live.push_back(i);
  if (live.empty()) return outputs(ranks, flags, uo.data(), vo.data());
  std::stable_sort(live.begin(), live.end(), [&](int64_t a, int64_t b) { return K[a] > K[b]; });
  const int64_t nl = (int64_t)live.size();
  std::vector<RecDesc> rd((size_t)nl);
  std::vector<GramItem> gi((size_t)(2 * nl));
  std::vector<int2> tiles;
  int64_t go = 0, wo = 0;
  DevBuf mem(c);
  for (int64_t q = 0; q < nl; ++q) {
    const int64_t k = K[live[q]];
    rd[q].goff = go;
    rd[q].woff = wo;
    rd[q].K = (int32_t)k;
    rd[q].kcap = (int32_t)k;
    go += 2 * k * k;
    wo += 6 * k * k;
  }
  double2 *G, *W;
  int rc;
  if ((rc = mem.alloc(&G, go)) || (rc = mem.alloc(&W, wo))) return rc;
  for (int64_t q = 0; q < nl; ++q) {
    const int64_t i = live[q], k = K[i];
    for (int side = 0; side < 2; ++side) {
      GramItem& g = gi[2 * q + side];
      g.F = side == 0 ? U[i] : V[i];
      g.rows = side == 0 ? dm[i] : dn[i];
      g.K = (int32_t)k;
      g.pad = 0;
      g.G = G + rd[q].goff + (side == 0 ? 0 : k * k);
      const int nt = (int)hmx_cdiv(k, 16);
      for (int t = 0; t < nt * nt; ++t) tiles.push_back(make_int2((int)(2 * q + side), t));
    }
  }
  // descriptors in one upload: [Gram items | recompression descriptors | tiles | rank | flag]
  const size_t b_gi = sizeof(GramItem) * gi.size(), b_rd = sizeof(RecDesc) * rd.size();
  const size_t o_rd = (b_gi + 15) / 16 * 16, o_tl = o_rd + (b_rd + 15) / 16 * 16;
  const size_t o_rk = o_tl + (sizeof(int2) * tiles.size() + 15) / 16 * 16;
  const size_t o_fl = o_rk + (sizeof(int32_t) * nl + 15) / 16 * 16;
  const size_t total = o_fl + sizeof(int32_t) * nl;
  std::vector<unsigned char> host(o_rk);
  memcpy(host.data(), gi.data(), b_gi);
  memcpy(host.data() + o_rd, rd.data(), b_rd);
  memcpy(host.data() + o_tl, tiles.data(), sizeof(int2) * tiles.size());
  unsigned char* d_blob;
  if ((rc = mem.alloc(&d_blob, (int64_t)total))) return rc;
  HMX_CUDA_TRY(cudaMemcpyAsync(d_blob, host.data(), o_rk, cudaMemcpyHostToDevice, c.stream));
  const GramItem* d_gi = reinterpret_cast<const GramItem*>(d_blob);
  const RecDesc* d_rd = reinterpret_cast<const RecDesc*>(d_blob + o_rd);
  const int2* d_tiles = reinterpret_cast<const int2*>(d_blob + o_tl);
  int32_t* d_rank = reinterpret_cast<int32_t*>(d_blob + o_rk);
  int32_t* d_flag = reinterpret_cast<int32_t*>(d_blob + o_fl);
  gram_batch<<<(unsigned)tiles.size(), 256, 0, c.stream>>>(d_gi, d_tiles);
  HMX_CUDA_TRY(cudaGetLastError());
  // K classes: > 112 (global-memory variant), 61..112, <= 60 (shared-memory variants, more CTAs per SM)
  int64_t q0 = 0;
  while (q0 < nl) {
    const int kc = rd[q0].K;
    const int lo = kc > 112 ? 112 : (kc > 60 ? 60 : 0);
    int64_t q1 = q0;
    while (q1 < nl && rd[q1].K > lo) ++q1;
    if ((rc = launch_recompress_core(c, d_rd + q0, q1 - q0, kc, eps, trunc_rule, G, W, d_rank + q0, d_flag + q0)))
      return rc;
    q0 = q1;
  }
  std::vector<int32_t> hrf((size_t)(o_fl - o_rk) / 4 + (size_t)nl);
  HMX_CUDA_TRY(cudaMemcpyAsync(hrf.data(), d_rank, total - o_rk, cudaMemcpyDeviceToHost, c.stream));
  HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  const int32_t* hr = hrf.data();
  const int32_t* hf = hrf.data() + (o_fl - o_rk) / 4;
  for (int64_t q = 0; q < nl; ++q) {
    ranks[live[q]] = hr[q];
    flags[live[q]] = hf[q];
  }
  if ((rc = outputs(ranks, flags, uo.data(), vo.data()))) return rc;
  std::vector<FormDesc> fd;
  std::vector<int64_t> ts;
  int64_t ntiles = 0;
  for (int64_t q = 0; q < nl; ++q) {
    const int64_t i = live[q], k = K[i];
    const int r = hr[q];
    if (r <= 0 || (hf[q] & 1)) continue;  // a regularised (rank-deficient V) item is not formed
    for (int side = 0; side < 2; ++side) {
      FormDesc f;
      const int64_t rows = side == 0 ? dm[i] : dn[i];
      f.A = side == 0 ? U[i] : V[i];
      f.W = W + rd[q].woff + 4 * k * k + (side == 0 ? 0 : k * r);
      f.C = side == 0 ? uo[i] : vo[i];
      f.rows = (int32_t)rows;
      f.K = (int32_t)k;
      f.r = r;
      f.lda = (int32_t)rows;
      f.ldc = (int32_t)rows;
      f.pad = 0;
      ts.push_back(ntiles);
      ntiles += hmx_cdiv(rows, 64) * hmx_cdiv(r, 32);
      fd.push_back(f);
    }
  }
  if (!fd.empty()) {
    const size_t b_fd = (sizeof(FormDesc) * fd.size() + 15) / 16 * 16;
    std::vector<unsigned char> hb(b_fd + sizeof(int64_t) * ts.size());
    memcpy(hb.data(), fd.data(), sizeof(FormDesc) * fd.size());
    memcpy(hb.data() + b_fd, ts.data(), sizeof(int64_t) * ts.size());
    unsigned char* d_f;
    if ((rc = mem.alloc(&d_f, (int64_t)hb.size()))) return rc;
    HMX_CUDA_TRY(cudaMemcpyAsync(d_f, hb.data(), hb.size(), cudaMemcpyHostToDevice, c.stream));
    if ((rc = launch_form(c, reinterpret_cast<const FormDesc*>(d_f), (int64_t)fd.size(), ntiles,
                          reinterpret_cast<const int64_t*>(d_f + b_fd))))
      return rc;
  }
  return HMX_OK;
}

}  // namespace hmx

extern "C" {

int hmx_truncate_batch(hmx_ctx* ctx, int64_t nb, const int64_t* dm, const int64_t* dn, const int64_t* K,
                       const uint64_t* U, const uint64_t* V, const uint64_t* Uo, const uint64_t* Vo, double eps,
                       int32_t trunc_rule, int64_t* ranks, int32_t* flags) {
  if (!ctx || nb < 0 || (nb > 0 && (!dm || !dn || !K || !U || !V || !Uo || !Vo || !ranks || !flags)))
    return HMX_EINVAL;
  if (nb == 0) return HMX_OK;
  for (int64_t i = 0; i < nb; ++i) {
    if (dm[i] <= 0 || dn[i] <= 0 || K[i] < 0 || (K[i] > 0 && (!U[i] || !V[i] || !Uo[i] || !Vo[i]))) {
      hmx_set_error("hmx_truncate_batch: item %lld has invalid sizes / pointers", (long long)i);
      return HMX_EINVAL;
    }
    if (K[i] > 1020) {
      hmx_set_error("hmx_truncate_batch: item %lld has %lld columns, above the device limit 1020", (long long)i,
                    (long long)K[i]);
      return HMX_EINVAL;
    }
  }
  Ctx& c = ctx->c;
  HMX_CUDA_TRY(cudaSetDevice(c.device));
  return truncate_pairs(c, nb, dm, dn, K, reinterpret_cast<const double2* const*>(U),
                        reinterpret_cast<const double2* const*>(V), eps, trunc_rule, ranks, flags,
                        [&](const int64_t*, const int32_t*, double2** uo, double2** vo) {
                          for (int64_t i = 0; i < nb; ++i) {
                            uo[i] = reinterpret_cast<double2*>(Uo[i]);
                            vo[i] = reinterpret_cast<double2*>(Vo[i]);
                          }
                          return HMX_OK;
                        });
}

}  // extern "C"
