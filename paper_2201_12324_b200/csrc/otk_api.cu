// Entry points of libotk_sm100.so that are not a half-step kernel:
// error plumbing, device query, K0 prep, bias, finalize (K7 local combine),
// and the K5 fused convergence check.
#include <cuda_fp16.h>

#include <cstdarg>
#include <cstring>

#include "otk_common.cuh"

namespace otk {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char *what) {
  set_error("CUDA error %s (%d) in %s", cudaGetErrorString(e), (int)e, what);
  return OTK_ECUDA;
}

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// ---------------------------------------------------------------- K0 prep
// One warp per point: |p|^2 in float64; optional split-fp16 planes and the
// per-K-block norm planes of the tcgen05 kernel (see include/otk.h).
__global__ void prep_kernel(const float *__restrict__ pts, int64_t n, int d,
                            float *__restrict__ sq, __half *__restrict__ hi,
                            __half *__restrict__ lo, __half *__restrict__ ext_a,
                            __half *__restrict__ ext_b, int dpad, float scale) {
  int64_t warp = (int64_t)(blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32);
  int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const float *row = pts + warp * d;
  double acc = 0.0;
  for (int k = lane; k < d; k += 32) {
    double v = row[k];
    acc = fma(v, v, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) sq[warp] = (float)acc;
  if (hi == nullptr) return;
  __half *hrow = hi + warp * dpad;
  __half *lrow = lo + warp * dpad;
  for (int k = lane; k < dpad; k += 32) {
    float v = (k < d) ? row[k] * scale : 0.f;
    __half h = __float2half_rn(v);
    hrow[k] = h;
    lrow[k] = __float2half_rn(v - __half2float(h));
  }
  if (ext_a == nullptr) return;
  // norm planes: -s^2 |p|^2 / 2 as three fp16 pieces times 2^15 (see include/otk.h)
  const double w = acc * (double)scale * (double)scale * (1.0 / 65536.0);
  const __half p0 = __double2half(w);
  const double r1 = w - (double)__half2float(p0);
  const __half p1 = __double2half(r1);
  const __half p2 = __double2half(r1 - (double)__half2float(p1));
  if (lane < 16) {
    const __half big = __float2half_rn(32768.f);
    const __half zero = __float2half_rn(0.f);
    __half ea = zero, eb = zero;
    if (lane < 3) {
      ea = __hneg(lane == 0 ? p0 : (lane == 1 ? p1 : p2));
      eb = big;
    } else if (lane < 6) {
      ea = big;
      eb = __hneg(lane == 3 ? p0 : (lane == 4 ? p1 : p2));
    }
    ext_a[warp * 16 + lane] = ea;
    ext_b[warp * 16 + lane] = eb;
  }
}

// ---------------------------------------------------------------- translation
// C is translation-invariant, so both point sets are shifted by one common
// centre before any kernel forms |p|^2 + |q|^2 - 2<p,q> in float32: the
// cancellation error then scales with the spread of the points, not with
// their distance from the origin.  The centre is the coordinate-wise median
// of q (over at most kMedianRows evenly strided rows): unlike the mean it is
// not dragged away from the bulk of the points by a few far outliers.
constexpr int kMedianRows = 8192;

// One block per coordinate: the strided samples in shared memory, +inf
// padded to a power of two, bitonic sort, lower median.
__global__ void __launch_bounds__(1024) column_median_kernel(const float *__restrict__ q, int64_t m,
                                                             int d, int64_t stride, int count,
                                                             int pow2, double *__restrict__ center) {
  extern __shared__ float v[];
  const int k = blockIdx.x;
  for (int i = threadIdx.x; i < pow2; i += blockDim.x)
    v[i] = (i < count) ? q[(int64_t)i * stride * d + k] : INFINITY;
  __syncthreads();
  for (int size = 2; size <= pow2; size <<= 1) {
    for (int j = size >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < pow2; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & size) == 0;
          const float a = v[i], b = v[p];
          if ((a > b) == up) {
            v[i] = b;
            v[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) center[k] = (double)v[(count - 1) / 2];
}

__global__ void shift_kernel(const float *__restrict__ p, int64_t count, int d,
                             const double *__restrict__ c, float *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)((double)p[i] - c[i % d]);
}

__global__ void absmax_kernel(const float *__restrict__ p, int64_t count, unsigned *__restrict__ out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(p[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

__global__ void bias_kernel(const float *__restrict__ pot, int64_t m, float kappa,
                            float *__restrict__ bias, int *__restrict__ first_bad, int step) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  float v = pot[j];
  if (first_bad != nullptr && bad_potential(v)) atomicMin(first_bad, step);
  bias[j] = v * kappa;
}

// Multi-GPU exchange: row i's L into slot (epoch & 1, rank) of every peer.
__device__ __forceinline__ void push_row(const FinArgs &F, int64_t i, float L) {
  const XLayout X(F.xworld, F.np);
  char *const *peers = reinterpret_cast<char *const *>(F.xlocal + X.table);
  const unsigned epoch = exchange_epoch(F.xlocal, F.xepoch);
  const int64_t off = ((int64_t)(epoch & 1u) * F.xworld + F.xrank) * X.m_pad + i;
  for (int s = 0; s < F.xworld; ++s) reinterpret_cast<float *>(peers[s] + X.data)[off] = L;
}
// After every thread of the block has pushed its rows: one release per peer
// (bar.sync orders the block's stores before thread 0's system-scope fence).
__device__ __forceinline__ void signal_block(const FinArgs &F) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const XLayout X(F.xworld, F.np);
    char *const *peers = reinterpret_cast<char *const *>(F.xlocal + X.table);
    const unsigned epoch = exchange_epoch(F.xlocal, F.xepoch);
    __threadfence_system();
    for (int s = 0; s < F.xworld; ++s) {
      unsigned *flag = reinterpret_cast<unsigned *>(peers[s] + X.flags) + (size_t)F.xrank * X.nblk + blockIdx.x;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
    }
  }
}

__device__ __forceinline__ void finalize_row(const FinArgs &F, int64_t i, float L) {
  if (F.anchor != nullptr) F.anchor[i] = isfinite(L) ? L : __int_as_float(0x7fc00000);
  if (F.xlocal != nullptr) push_row(F, i, L);
  if (F.mode == OTK_FIN_LOG2) {  // shard partial for the multi-GPU exchange
    F.out[i] = L;
    return;
  }
  const float c = F.eps * kLn2, bi = F.base[i];
  const float v = (F.mode == OTK_FIN_SOLVER) ? F.eps * bi - c * L : bi + c * L;
  F.out[i] = v;
  if (F.out_bias != nullptr)
    F.out_bias[i] = (F.mode == OTK_FIN_SOLVER) ? next_bias(bi, L, F.eps, F.kappa_next) : v * F.kappa_next;
  if (F.first_bad != nullptr && bad_potential(v)) atomicMin(F.first_bad, F.step);
}

__global__ void finalize_kernel(const FinArgs F) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < F.np) finalize_row(F, i, combine_log2(F.part + i, F.nsplit, F.np));
  if (F.xlocal != nullptr) signal_block(F);
}

// After an anchored launch: accept the row when its anchor was finite and the
// result lies in the window (lo <= L - anchor <= 120: every term within 2^-30 of the
// row's sum was above the ex2 flush threshold; an overflowing sum shows up
// as L = +inf), or when L is NaN (a NaN potential propagates exactly as in the
// running-max kernel).  Otherwise flag the row's 128-row tile for the repair
// launch and leave the row to finalize_repair_kernel.
__global__ void finalize_anchored_kernel(const FinArgs F) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= F.np) return;
  const float L = combine_log2(F.part + i, F.nsplit, F.np);
  const float S = F.anchor[i];
  const bool ok = isfinite(S) && (L != L || (isfinite(L) && L - S >= F.lo && L - S <= 120.f));
  if (!ok) {
    atomicAdd(F.repair_ws, 1);
    F.repair_ws[1 + (i >> 7)] = 1;
    return;
  }
  finalize_row(F, i, L);
}

// After the repair launch: re-finalize every row of a flagged tile from the
// running-max partials.  With a multi-GPU exchange this is the half-step's
// last kernel: it also pushes the rows finalize_anchored accepted (LOG2 mode:
// their L is already in out) and signals every block.
__global__ void finalize_repair_kernel(const FinArgs F) {
  const bool any = *reinterpret_cast<const volatile int *>(F.repair_ws) != 0;
  if (!any && F.xlocal == nullptr) return;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < F.np) {
    if (any && F.repair_ws[1 + (i >> 7)] != 0) finalize_row(F, i, combine_log2(F.part + i, F.nsplit, F.np));
    else if (F.xlocal != nullptr) push_row(F, i, F.out[i]);
  }
  if (F.xlocal != nullptr) signal_block(F);
}

int finalize_launch(int kind, const FinArgs &F, cudaStream_t st) {
  const unsigned blocks = (unsigned)((F.np + 255) / 256);
  if (kind == 0) finalize_kernel<<<blocks, 256, 0, st>>>(F);
  else if (kind == 1) finalize_anchored_kernel<<<blocks, 256, 0, st>>>(F);
  else finalize_repair_kernel<<<blocks, 256, 0, st>>>(F);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

// ---------------------------------------------------------------- geometry construction helpers
// One launch for the constructor's three questions (geometry.py:247-261): any
// non-finite coordinate in x, in y, and -- equal shapes only -- any x != y.
__global__ void points_flags_kernel(const float *__restrict__ x, int64_t cx, const float *__restrict__ y,
                                    int64_t cy, int compare, int *__restrict__ flags) {
  bool bx = false, by = false, df = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t top = cx > cy ? cx : cy;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < top; k += stride) {
    const float a = k < cx ? x[k] : 0.f, b = k < cy ? y[k] : 0.f;
    bx |= !isfinite(a);
    by |= !isfinite(b);
    df |= compare && !(a == b);
  }
  if (__syncthreads_or(bx) && threadIdx.x == 0) flags[0] = 1;
  if (__syncthreads_or(by) && threadIdx.x == 0) flags[1] = 1;
  if (__syncthreads_or(df) && threadIdx.x == 0) flags[2] = 1;
}

// Mean cost over `count` sampled pairs (geometry.py:294-312: the eps estimate),
// float64 difference form on the kernel points, fixed-order block reduction.
__global__ void __launch_bounds__(1024) mean_cost_pairs_kernel(const float *__restrict__ x,
                                                               const float *__restrict__ y,
                                                               const int64_t *__restrict__ ii,
                                                               const int64_t *__restrict__ jj, int64_t count,
                                                               int d, int eucl, int same,
                                                               double *__restrict__ out) {
  __shared__ double red[1024];
  double acc = 0.0;
  for (int64_t s = threadIdx.x; s < count; s += blockDim.x) {
    const int64_t i = ii[s], j = jj[s];
    double c = 0.0;
    for (int k = 0; k < d; ++k) {
      const double df = (double)x[i * d + k] - (double)y[j * d + k];
      c = fma(df, df, c);
    }
    if (eucl) c = sqrt(c);
    if (same && i == j) c = 0.0;
    acc += c;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0] / (double)count;
}

// ---------------------------------------------------------------- K5 check
constexpr int kCheckBlocks = 148;
constexpr int kCheckThreads = 256;
constexpr int kCheckVals = 8;

template <int N>
__device__ void block_reduce_d(double (&v)[N], double *smem /* [N][kCheckThreads] */) {
  int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < N; ++k) smem[k * kCheckThreads + t] = v[k];
  __syncthreads();
  for (int s = kCheckThreads / 2; s > 0; s >>= 1) {
    if (t < s) {
#pragma unroll
      for (int k = 0; k < N; ++k) smem[k * kCheckThreads + t] += smem[k * kCheckThreads + t + s];
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = smem[k * kCheckThreads];
}

__global__ void __launch_bounds__(kCheckThreads) check_kernel(
    const float *__restrict__ f_prev, const float *__restrict__ f_next, const float *__restrict__ a,
    int64_t n, const float *__restrict__ g, const float *__restrict__ b, int64_t m, double eps,
    double *__restrict__ out, double *__restrict__ ws, unsigned *__restrict__ counter) {
  __shared__ double smem[kCheckVals * kCheckThreads];
  __shared__ bool last;
  double v[kCheckVals] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double inv_eps = 1.0 / eps;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double fp = f_prev[i];
    double ai = a[i];
    if (f_next != nullptr) {
      double r = (ai > 0.0) ? ai * exp((fp - (double)f_next[i]) * inv_eps) : 0.0;
      v[0] += fabs(r - ai);
      v[1] += r;
    }
    if (ai > 0.0) v[2] += ai * fp;
    v[4] += (fp != fp) ? 1.0 : 0.0;
    v[6] += (fp == INFINITY) ? 1.0 : 0.0;
  }
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += stride) {
    double gj = g[j];
    double bj = b[j];
    if (bj > 0.0) v[3] += bj * gj;
    v[5] += (gj != gj) ? 1.0 : 0.0;
    v[7] += (gj == INFINITY) ? 1.0 : 0.0;
  }
  block_reduce_d(v, smem);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < kCheckVals; ++k) ws[blockIdx.x * kCheckVals + k] = v[k];
    __threadfence();
    unsigned done = atomicAdd(counter, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // Fixed-order final reduction over block partials: deterministic.
  if (threadIdx.x < kCheckVals) {
    double acc = 0.0;
    for (int blk = 0; blk < (int)gridDim.x; ++blk)
      acc += ((volatile double *)ws)[blk * kCheckVals + threadIdx.x];
    out[threadIdx.x] = acc;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

}  // namespace otk

using namespace otk;

extern "C" {

int otk_abi_version(void) { return OTK_ABI_VERSION; }

const char *otk_last_error(void) { return g_err; }

int otk_device_query(int device, int *sm_count, int *cc_major, int *cc_minor) {
  OTK_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  OTK_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  OTK_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  return OTK_OK;
}

int otk_prep_points(const float *pts, int64_t n, int32_t d, float *sqnorm, uint16_t *hi,
                    uint16_t *lo, uint16_t *ext_a, uint16_t *ext_b, int32_t dpad,
                    float split_scale, void *stream) {
  OTK_CHECK_ARG(pts && sqnorm && n > 0 && d > 0, "otk_prep_points: bad arguments");
  OTK_CHECK_ARG((hi == nullptr) == (lo == nullptr), "otk_prep_points: hi/lo must both be set");
  OTK_CHECK_ARG((ext_a == nullptr) == (ext_b == nullptr), "otk_prep_points: ext_a/ext_b must both be set");
  OTK_CHECK_ARG(ext_a == nullptr || hi != nullptr, "otk_prep_points: ext planes need hi/lo");
  OTK_CHECK_ARG(hi == nullptr || (dpad >= d && dpad % 64 == 0), "otk_prep_points: dpad must be >= d and a multiple of 64");
  const int warps = 8;
  int64_t blocks = (n + warps - 1) / warps;
  prep_kernel<<<(unsigned)blocks, warps * 32, 0, as_stream(stream)>>>(
      pts, n, d, sqnorm, reinterpret_cast<__half *>(hi), reinterpret_cast<__half *>(lo),
      reinterpret_cast<__half *>(ext_a), reinterpret_cast<__half *>(ext_b), dpad, split_scale);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_column_median(const float *q, int64_t m, int32_t d, double *center, void *stream) {
  OTK_CHECK_ARG(q && center && m > 0 && d > 0, "otk_column_median: bad arguments");
  const int64_t stride = (m + kMedianRows - 1) / kMedianRows;
  const int count = (int)((m + stride - 1) / stride);
  int pow2 = 1;
  while (pow2 < count) pow2 <<= 1;
  const size_t smem = (size_t)pow2 * sizeof(float);
  static bool attr = false;
  if (!attr) {
    OTK_CUDA(cudaFuncSetAttribute(column_median_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kMedianRows * (int)sizeof(float)));
    attr = true;
  }
  column_median_kernel<<<(unsigned)d, 1024, smem, as_stream(stream)>>>(q, m, d, stride, count, pow2,
                                                                      center);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_shift_points(const float *p, int64_t n, int32_t d, const double *center, float *out,
                     void *stream) {
  OTK_CHECK_ARG(p && center && out && n > 0 && d > 0, "otk_shift_points: bad arguments");
  const int64_t count = n * (int64_t)d;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
  shift_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(p, count, d, center, out);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

float otk_split_scale(float amax, int32_t d) {
  // largest power of two s with s*amax <= 2^12 and s^2 * d * amax^2 <= 2^31, which
  // keeps hi/lo and the fp16 norm pieces (<= s^2|p|^2/2^16) in range
  if (!(amax > 0.f) || !std::isfinite(amax) || d <= 0) return 1.f;
  const double lim = std::min(4096.0, std::pow(2.0, 15.5) / std::sqrt((double)d)) / amax;
  int e = (int)std::floor(std::log2(lim));
  e = e < -60 ? -60 : (e > 60 ? 60 : e);
  return std::ldexp(1.f, e);
}

int otk_absmax(const float *pts, int64_t count, float *out, void *stream) {
  OTK_CHECK_ARG(pts && out && count > 0, "otk_absmax: bad arguments");
  OTK_CUDA(cudaMemsetAsync(out, 0, sizeof(float), as_stream(stream)));
  int64_t blocks = (count + 255) / 256;
  if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
  absmax_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(pts, count,
                                                                  reinterpret_cast<unsigned *>(out));
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_make_bias(const float *pot, int64_t m, float kappa, float *bias, int32_t *first_bad,
                  int32_t step, void *stream) {
  OTK_CHECK_ARG(pot && bias && m > 0, "otk_make_bias: bad arguments");
  bias_kernel<<<(unsigned)((m + 255) / 256), 256, 0, as_stream(stream)>>>(pot, m, kappa, bias,
                                                                           first_bad, step);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_lse_finalize(const float *partial, int32_t nsplit, int64_t np, const float *base,
                     int32_t mode, float eps, float kappa_next, float *out_pot, float *out_bias,
                     int32_t *first_bad, int32_t step, void *stream) {
  OTK_CHECK_ARG(partial && out_pot && np > 0 && nsplit >= 1, "otk_lse_finalize: bad arguments");
  OTK_CHECK_ARG(mode == OTK_FIN_SOLVER || mode == OTK_FIN_APPLY || mode == OTK_FIN_LOG2,
                "otk_lse_finalize: bad mode");
  OTK_CHECK_ARG(base || mode == OTK_FIN_LOG2, "otk_lse_finalize: base required");
  FinArgs F{partial, nsplit, np, base, mode, eps, kappa_next, out_pot, out_bias, first_bad, step,
            nullptr, nullptr, 0.f, nullptr, 0, 0, 0u};
  return finalize_launch(0, F, as_stream(stream));
}

size_t otk_check_workspace_bytes(void) {
  return (size_t)kCheckBlocks * kCheckVals * sizeof(double) + 256;
}

int otk_check(const float *f_prev, const float *f_next, const float *a, int64_t n, const float *g,
              const float *b, int64_t m, double eps, double *out, void *ws, void *stream) {
  OTK_CHECK_ARG(f_prev && a && g && b && out && ws && n > 0 && m > 0, "otk_check: bad arguments");
  double *part = reinterpret_cast<double *>(ws);
  unsigned *counter = reinterpret_cast<unsigned *>(part + kCheckBlocks * kCheckVals);
  check_kernel<<<kCheckBlocks, kCheckThreads, 0, as_stream(stream)>>>(f_prev, f_next, a, n, g, b, m,
                                                                      eps, out, part, counter);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

}  // extern "C"

extern "C" int otk_points_flags(const float *x, int64_t nx, const float *y, int64_t ny, int32_t d,
                                int32_t compare, int32_t *flags, void *stream) {
  OTK_CHECK_ARG(x && y && flags && nx > 0 && ny > 0 && d > 0, "otk_points_flags: bad arguments");
  cudaStream_t st = as_stream(stream);
  OTK_CUDA(cudaMemsetAsync(flags, 0, 3 * sizeof(int32_t), st));
  const int64_t top = std::max(nx, ny) * d;
  const unsigned blocks = (unsigned)std::min<int64_t>((top + 255) / 256, 4 * (int64_t)num_sms());
  points_flags_kernel<<<blocks, 256, 0, st>>>(x, nx * d, y, ny * d, compare && nx == ny, flags);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

extern "C" int otk_mean_cost_pairs(const float *x, const float *y, const int64_t *ii, const int64_t *jj,
                                   int64_t count, int32_t d, int32_t flags, double *mean, void *stream) {
  OTK_CHECK_ARG(x && y && ii && jj && mean && count > 0 && d > 0, "otk_mean_cost_pairs: bad arguments");
  mean_cost_pairs_kernel<<<1, 1024, 0, as_stream(stream)>>>(x, y, ii, jj, count, d,
                                                             (flags & OTK_COST_EUCL) != 0,
                                                             (flags & OTK_SAME_POINTS) != 0, mean);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}
