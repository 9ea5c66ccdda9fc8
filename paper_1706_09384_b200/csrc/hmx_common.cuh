// Shared device helpers for the hmx B200 library (sm_100a).
//
// Complex numbers are double2 (x = re, y = im), the same interleaved layout as
// numpy complex128, so host buffers cross the C-ABI as plain double*.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#define HMX_HD __host__ __device__ __forceinline__
#define HMX_D __device__ __forceinline__

// ---- complex double2 -------------------------------------------------------
HMX_HD double2 cmk(double r, double i) { return make_double2(r, i); }
HMX_HD double2 cadd(double2 a, double2 b) { return cmk(a.x + b.x, a.y + b.y); }
HMX_HD double2 csub(double2 a, double2 b) { return cmk(a.x - b.x, a.y - b.y); }
HMX_HD double2 cmul(double2 a, double2 b) { return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
HMX_HD double2 cscale(double2 a, double s) { return cmk(a.x * s, a.y * s); }
HMX_HD double2 cconj(double2 a) { return cmk(a.x, -a.y); }
HMX_HD double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
// acc += a * b
HMX_HD double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc += a * conj(b)
HMX_HD double2 cfma_cj(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y);
  acc.y = fma(-a.x, b.y, acc.y);
  return acc;
}
// acc += conj(a) * b
HMX_HD double2 cfma_ca(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
HMX_HD double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm
  if (fabs(b.x) >= fabs(b.y)) {
    double rat = b.y / b.x, scl = 1.0 / (b.x + b.y * rat);
    return cmk((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
  }
  double rat = b.x / b.y, scl = 1.0 / (b.y + b.x * rat);
  return cmk((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}

// ---- warp reductions -------------------------------------------------------
HMX_D double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
HMX_D double2 warp_sum(double2 v) {
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  return v;
}
HMX_D double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (value, index) argmax with lowest-index tie-break (np.argmax semantics).
struct ArgMax {
  double v;
  int i;
};
HMX_D ArgMax argmax_pick(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
HMX_D ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    a = argmax_pick(a, b);
  }
  return a;
}

// ---- error plumbing --------------------------------------------------------
#include "../../include/hmx.h"  // HMX_OK / HMX_E* status codes

void hmx_set_error(const char* fmt, ...);

#define HMX_CUDA_TRY(expr)                                                       \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      hmx_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return HMX_ECUDA;                                                          \
    }                                                                            \
  } while (0)

static inline int64_t hmx_cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- Blackwell bulk-copy plumbing (TMA engine, async proxy) ------------------------
// cp.async.bulk moves one contiguous run global -> shared and signals completion as
// transaction bytes on an mbarrier (SASS UBLKCP / SYNCS); the issuing lane needs no
// registers for the data and no per-element address arithmetic.
HMX_D void mbar_init(unsigned a, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
HMX_D void mbar_expect_tx(unsigned a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
HMX_D void mbar_wait(unsigned a, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
HMX_D void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
// generic-proxy accesses of this thread before -> async-proxy accesses after
HMX_D void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
HMX_D void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// one lane of the (converged) warp, chosen by the hardware: the compiler issues what follows on
// the uniform datapath when its operands are warp-uniform
HMX_D bool elect_one() {
  unsigned pred;
  asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(pred));
  return pred != 0;
}

