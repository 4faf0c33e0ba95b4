// Shared helpers for the sm_100a Sinkhorn library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdio>
#include <string>

#include "otk.h"

namespace otk {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// ---- error reporting (thread-local message, returned status) ----
void set_error(const char *fmt, ...);
int cuda_status(cudaError_t e, const char *what);

#define OTK_CHECK_ARG(cond, ...)          \
  do {                                    \
    if (!(cond)) {                        \
      ::otk::set_error(__VA_ARGS__);      \
      return OTK_EINVAL;                  \
    }                                     \
  } while (0)

#define OTK_CUDA(call)                                        \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return ::otk::cuda_status(_e, #call); \
  } while (0)

#define OTK_LAUNCH_CHECK() OTK_CUDA(cudaGetLastError())

int num_sms();

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- tracing: NVTX ranges (header-only NVTX3; free unless a profiler is attached)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// ---- device math ----
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Online log2-sum-exp2 state: value = m + log2(s).  m = -inf means empty.
struct Lse2 {
  float m, s;
  __device__ __forceinline__ void init() { m = -INFINITY; s = 0.f; }
  // merge another (m2, s2)
  __device__ __forceinline__ void merge(float m2, float s2) {
    float mm = fmaxf(m, m2);
    if (mm == -INFINITY) return;
    s = s * ex2(m - mm) + s2 * ex2(m2 - mm);
    m = mm;
  }
  __device__ __forceinline__ float value() const {
    if (s != s) return s;  // NaN propagates
    return (s > 0.f) ? m + lg2(s) : -INFINITY;
  }
};

// log2-sum of a fixed-order list of partial log2 values.
__device__ __forceinline__ float combine_log2(const float *part, int nsplit, int64_t stride) {
  if (nsplit == 1) return part[0];
  float mx = -INFINITY;
  bool nan = false;
  for (int s = 0; s < nsplit; ++s) {
    float v = part[s * stride];
    nan |= (v != v);
    mx = fmaxf(mx, v);
  }
  if (nan) return __int_as_float(0x7fc00000);
  if (mx == -INFINITY) return mx;  // empty
  if (mx == INFINITY) return INFINITY;
  float acc = 0.f;
  for (int s = 0; s < nsplit; ++s) acc += ex2(part[s * stride] - mx);
  return mx + lg2(acc);
}

__device__ __forceinline__ bool bad_potential(float v) { return (v != v) || v == INFINITY; }

// The next half-step's bias kappa' * v of a solver potential v = eps (log w - ln2 L),
// from log w and L directly: kappa' v = r (log2 w - L) with r = kappa' eps ln2.
// At constant eps r is 1 but fl(kappa') fl(eps) fl(ln2) is 1 +- 1e-7, and
// multiplying every half-step's output by it is a bias of 1e-7 |L| that
// Sinkhorn never contracts along (f + c, g - c): it added up linearly with the
// iterations (9e-7 log2 units per iteration on a 48 x 40 problem).  r within
// 1e-5 of 1 is taken as 1; annealing steps (eps changes by >= 1e-3) keep r.
__device__ __forceinline__ float next_bias(float logw, float L, float eps, float kappa_next) {
  const float r = kappa_next * (eps * kLn2);
  const float b = fmaf(logw, 1.4426950408889634f, -L);
  return (fabsf(r - 1.f) < 1e-5f) ? b : r * b;
}

// Finalize of a half-step (otk_api.cu): combine the split partials, form the
// potential (mode), write the next bias / anchor, flag bad potentials.
struct FinArgs {
  const float *part;
  int nsplit;
  int64_t np;
  const float *base;
  int mode;
  float eps, kappa_next;
  float *out, *out_bias;
  int *first_bad;
  int step;
  float *anchor;  // nullable: the row's L for the next anchored half-step (NaN if not finite)
  int *repair_ws; // anchored: [0] = flagged rows, [1 + i / 128] = row-tile flags
  float lo;       // anchored: smallest L - anchor accepted (see lse_tc.cu lse_chunk_anchored)
  // multi-GPU exchange (p2p.cu): push every row's L into slot (epoch & 1, rank)
  // of every peer's exchange buffer, then flag this block on every peer
  char *xlocal;   // this rank's exchange buffer (NULL = no push)
  int xworld, xrank;
  unsigned xepoch;  // 0 = the buffer's device epoch counter (exchange_epoch)
};

// Exchange-buffer layout (p2p.cu, include/otk.h otk_exchange_*): a header
// (error word, device epoch counters), the peer pointer table, the partials
// [2][world][m_pad] float, the per-block flags [world][nblk] uint32 (nblk =
// ceil(m / 256), the finalize kernels' block size), and the check exchange:
// slots [2][world][kChkSlot] double + flags [world] uint32.
constexpr int kChkSlot = 16;
struct XLayout {
  // header words (uint32): error, completed g exchanges, combine-block ticket,
  // completed check exchanges
  static constexpr size_t ERR = 0, EPOCH = 4, TICKET = 8, CHK_EPOCH = 12;
  size_t table, data, flags, chk, chkflags, total;
  int64_t m_pad;
  int nblk;
  __host__ __device__ XLayout(int world, int64_t m) {
    m_pad = (m + 3) & ~(int64_t)3;
    nblk = (int)((m + 255) / 256);
    table = 256;
    data = table + (((size_t)world * 8 + 255) / 256) * 256;
    flags = data + (((size_t)2 * world * m_pad * 4 + 255) / 256) * 256;
    chk = flags + (((size_t)world * nblk * 4 + 255) / 256) * 256;
    chkflags = chk + (((size_t)2 * world * kChkSlot * 8 + 255) / 256) * 256;
    total = chkflags + (((size_t)world * 4 + 255) / 256) * 256;
  }
};
__device__ __forceinline__ unsigned ld_cg_u32(const void *p) {
  return __ldcg(reinterpret_cast<const unsigned *>(p));
}
// Epoch of the g exchange in flight: explicit (>= 1) or, with 0, one past the
// buffer's count of completed combines (advanced by the combine kernel's last
// block), so the same launches replay correctly inside a CUDA graph.
__device__ __forceinline__ unsigned exchange_epoch(const char *local, unsigned explicit_epoch) {
  return explicit_epoch ? explicit_epoch : ld_cg_u32(local + XLayout::EPOCH) + 1u;
}
// kind 0 = plain, 1 = after an anchored launch, 2 = after the repair launch
int finalize_launch(int kind, const FinArgs &F, cudaStream_t st);

}  // namespace otk
