// Fixed-support Wasserstein barycenter by iterative Bregman projections
// (SURVEY.md §8f row 4), the whole solve as ONE persistent cooperative kernel.
//
// Replaces reference solve_barycenter (otkit/barycenter.py:96-133), which per
// iteration makes 3K calls of apply_lse_kernel over the shared square support
// geometry.  Here the support cost is materialised once (C and C^T, fp32,
// row-major with a leading dimension padded to a multiple of 4 with +inf
// costs, otk_barycenter_pad) and every phase streams rows of one of them,
// 128-bit coalesced; one warp reduces a cost row against up to 4 histograms
// at once, so each cost chunk is loaded once per 4 histograms.  All potentials are kept in
// log2 units (x kappa = log2(e)/eps), so eps enters only through kappa:
//   F[k,i]  = log2 h_ki - LSE2_j(G[k,j] - kappa C_ij)            (barycenter.py:117)
//   B[k,j]  = LSE2_i(F[k,i] - kappa C_ij)                        (barycenter.py:118)
//   lp2_j   = sum_k w_k B[k,j]          (= log p_j / ln 2)       (barycenter.py:119)
//   err     = max_k sum_j |2^(B[k,j] + G[k,j]) - 2^lp2_j|         (barycenter.py:123-126)
//   G[k,j]  = lp2_j - B[k,j]                                     (barycenter.py:127-128)
// The marginal of coupling k on the barycenter side, exp(LSE_cols(f_k,g_k)/eps),
// equals 2^(B + G) exactly in real arithmetic (g is constant along the reduced
// axis), so the third apply of the reference costs O(K N) here, not O(K N^2).
//
// Phases are separated by grid-wide barriers (3 per iteration); the stopping
// decision is made redundantly by every CTA from the same per-CTA partials
// summed in CTA order, so all CTAs leave the loop together and the result is
// deterministic for a given grid.  Reductions over a row: one warp, per-lane
// online LSE in a fixed order, then a fixed xor butterfly.
#include <cooperative_groups.h>

#include "otk_common.cuh"

namespace cg = cooperative_groups;

namespace otk {
namespace bary {

constexpr int THREADS = 256, WARPS = THREADS / 32;
constexpr int CHUNK = 512;  // columns per warp step: 4 float4 per lane

struct Args {
  const float *C, *CT;   // [n, ld] row-major each, columns n..ld-1 = +inf
  int n, ld, K;
  const float *log2h;    // [K, n]
  const double *w;       // [K]
  float kappa;
  float *F, *G, *B;      // [K, ld] each (zero on entry, pads stay zero)
  double *lp2;           // [n]   out: log2 of the (unnormalised) barycenter
  double *part;          // [grid, K + 1]
  double *errors;        // [max_iters]
  int *state;            // [8]: iterations, converged, nan_iteration, grid, task counters x2
  double threshold;
  int max_iters;
};

// One warp reduces one cost row against KG bias rows at once:
//   res[k] = LSE2_j(bias_k[j] - kappa row[j]),  j < ld (pads: cost +inf -> -inf)
// The cost chunk is loaded once and reused for the KG histograms; all loads of
// a chunk (4 + 4 KG float4 per lane) are issued before any is used.  Bias
// rows are written inside this kernel by other CTAs, so they are read through
// L2 (ld.cg); the cost is read-only (ld.global.nc).
template <int KG>
__device__ __forceinline__ void row_lse(const float *__restrict__ row, const float *const (&bias)[KG],
                                        int ld, float kappa, float (&res)[KG]) {
  const int lane = threadIdx.x & 31;
  float m[KG], s[KG];
#pragma unroll
  for (int k = 0; k < KG; ++k) {
    m[k] = -INFINITY;
    s[k] = 0.f;
  }
  for (int j0 = 0; j0 < ld; j0 += CHUNK) {
    float4 c[4], h[KG][4];
    bool ok[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + (q * 32 + lane) * 4;
      ok[q] = j < ld;
      c[q] = __ldg(reinterpret_cast<const float4 *>(row + (ok[q] ? j : 0)));
    }
#pragma unroll
    for (int k = 0; k < KG; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = j0 + (q * 32 + lane) * 4;
        h[k][q] = __ldcg(reinterpret_cast<const float4 *>(bias[k] + (ok[q] ? j : 0)));
      }
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      float u[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        u[4 * q + 0] = ok[q] ? fmaf(-kappa, c[q].x, h[k][q].x) : -INFINITY;
        u[4 * q + 1] = ok[q] ? fmaf(-kappa, c[q].y, h[k][q].y) : -INFINITY;
        u[4 * q + 2] = ok[q] ? fmaf(-kappa, c[q].z, h[k][q].z) : -INFINITY;
        u[4 * q + 3] = ok[q] ? fmaf(-kappa, c[q].w, h[k][q].w) : -INFINITY;
      }
      float cm = -INFINITY;
#pragma unroll
      for (int e = 0; e < 16; ++e) cm = fmaxf(cm, u[e]);
      if (cm > m[k]) {
        s[k] *= ex2(m[k] - cm);
        m[k] = cm;
      }
      const float ms = (m[k] == -INFINITY) ? 0.f : m[k];
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 16; ++e) acc += ex2(u[e] - ms);
      s[k] += acc;
    }
  }
#pragma unroll
  for (int k = 0; k < KG; ++k) {
    Lse2 st;
    st.m = m[k];
    st.s = s[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, st.m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, st.s, o);
      st.merge(m2, s2);
    }
    res[k] = st.value();
  }
}

// One half-step phase: for every (row r, histogram group), out[k, r] =
// log2 h - LSE2 (rows phase) or LSE2 (cols phase).  Warps take tasks from a
// global counter (each result depends only on its task, so the schedule does
// not change any value); task order is row-major over groups so the readers
// of one cost row run side by side.  `ctr` is zero on entry; the other
// phase's counter is reset here (nobody touches it until the next barrier).
template <int KG, bool ROWS>
__device__ __forceinline__ void phase(const Args &A, const float *cost, const float *bias_base,
                                      float *out, int *ctr, int *other_ctr) {
  const int lane = threadIdx.x & 31;
  const int groups = (A.K + KG - 1) / KG;
  const int64_t tasks = (int64_t)A.n * groups;
  if (blockIdx.x == 0 && threadIdx.x == 0) *other_ctr = 0;
  for (;;) {
    int64_t task = 0;
    if (lane == 0) task = atomicAdd(ctr, 1);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= tasks) break;
    const int r = (int)(task / groups), k0 = (int)(task % groups) * KG;
    const float *bias[KG];
#pragma unroll
    for (int k = 0; k < KG; ++k) bias[k] = bias_base + (int64_t)min(k0 + k, A.K - 1) * A.ld;
    float res[KG];
    row_lse<KG>(cost + (int64_t)r * A.ld, bias, A.ld, A.kappa, res);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        if (k0 + k >= A.K) break;
        const int64_t o = (int64_t)(k0 + k) * A.ld + r;
        out[o] = ROWS ? A.log2h[(int64_t)(k0 + k) * A.n + r] - res[k] : res[k];
      }
    }
  }
}

// Fixed-order tree sum of one double per thread; result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double *red) {
  red[threadIdx.x] = v;
  __syncthreads();
#pragma unroll
  for (int s = THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// Sum over CTAs of part[b*(K+1) + col], one warp, fixed lane assignment and butterfly.
__device__ __forceinline__ double warp_sum_parts(const double *part, int K, int col) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  for (unsigned b = lane; b < gridDim.x; b += 32) v += __ldcg(part + (int64_t)b * (K + 1) + col);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int KG>
__global__ void __launch_bounds__(THREADS, 2) bary_kernel(Args A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[THREADS];
  __shared__ int s_stop;
  const int n = A.n, K = A.K, ld = A.ld;
  const int64_t gtid = (int64_t)blockIdx.x * THREADS + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * THREADS;
  for (int t = 1; t <= A.max_iters; ++t) {
    phase<KG, true>(A, A.C, A.G, A.F, A.state + 4, A.state + 5);    // f_k = eps log h_k - LSE_rows(0, g_k)
    grid.sync();
    phase<KG, false>(A, A.CT, A.F, A.B, A.state + 5, A.state + 4);  // back_k = LSE_cols(f_k, 0)
    grid.sync();
    // ---- geometric mean, marginal error, g update (O(K n))
    double nan_count = 0.0;
    for (int64_t j = gtid; j < n; j += nthreads) {
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += A.w[k] * (double)__ldcg(A.B + (int64_t)k * ld + j);
      A.lp2[j] = s;
      nan_count += (s != s) ? 1.0 : 0.0;
    }
    for (int k = 0; k < K; ++k) {
      double e = 0.0;
      for (int64_t j = gtid; j < n; j += nthreads) {
        const double lp = A.lp2[j];
        const double bk = (double)__ldcg(A.B + (int64_t)k * ld + j);
        const double gk = (double)__ldcg(A.G + (int64_t)k * ld + j);
        e += fabs(exp2(bk + gk) - exp2(lp));
        A.G[(int64_t)k * ld + j] = (float)(lp - bk);
      }
      e = block_sum(e, red);
      if (threadIdx.x == 0) A.part[(int64_t)blockIdx.x * (K + 1) + k] = e;
    }
    nan_count = block_sum(nan_count, red);
    if (threadIdx.x == 0) A.part[(int64_t)blockIdx.x * (K + 1) + K] = nan_count;
    grid.sync();
    // ---- decision (identical in every CTA: same partials, same order)
    if (threadIdx.x < 32) {
      double err = 0.0;
      for (int k = 0; k < K; ++k) err = fmax(err, warp_sum_parts(A.part, K, k));
      const double nans = warp_sum_parts(A.part, K, K);
      if (threadIdx.x == 0) {
        int stop = 0;
        if (nans > 0.0) stop = 2;
        else if (err <= A.threshold) stop = 1;
        else if (t == A.max_iters) stop = 3;
        s_stop = stop;
        if (blockIdx.x == 0) {
          A.errors[t - 1] = (nans > 0.0) ? (double)NAN : err;
          A.state[0] = t;
          A.state[1] = (stop == 1);
          A.state[2] = (stop == 2) ? t : 0;
          A.state[3] = (int)gridDim.x;
        }
      }
    }
    __syncthreads();
    if (s_stop) break;
  }
}

// Cp[i, :n] = C[i, :], CTp[j, :n] = C[:, j]; columns n..ld-1 = +inf.
__global__ void __launch_bounds__(256) pad_kernel(const float *__restrict__ C, int n, int ld,
                                                  float *__restrict__ Cp, float *__restrict__ CTp) {
  __shared__ float tile[32][33];
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + tx;
    float v = INFINITY;
    if (i < n && j < n) v = C[(int64_t)i * n + j];
    tile[r][tx] = v;
    if (i < n && j < ld) Cp[(int64_t)i * ld + j] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int j = j0 + r, i = i0 + tx;
    if (j < n && i < ld) CTp[(int64_t)j * ld + i] = tile[tx][r];
  }
}

}  // namespace bary
}  // namespace otk

using namespace otk;

// Histograms per warp task: K itself up to 4, then 4 or 3, whichever leaves
// fewer idle slots in the last group (ties -> 4).
static int bary_kg(int32_t K) {
  if (K <= 4) return K;
  const int w4 = (K + 3) / 4 * 4 - K, w3 = (K + 2) / 3 * 3 - K;
  return w3 < w4 ? 3 : 4;
}

static void *bary_kernel_for(int32_t K) {
  switch (bary_kg(K)) {
    case 1: return (void *)bary::bary_kernel<1>;
    case 2: return (void *)bary::bary_kernel<2>;
    case 3: return (void *)bary::bary_kernel<3>;
    default: return (void *)bary::bary_kernel<4>;
  }
}

static int bary_grid(int64_t n, int32_t K, int *grid) {
  int per_sm = 0;
  OTK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bary_kernel_for(K), bary::THREADS, 0));
  if (per_sm < 1) {
    set_error("bary: kernel does not fit on an SM");
    return OTK_ENOTSUP;
  }
  const int kg = bary_kg(K);
  const int64_t tasks = n * ((K + kg - 1) / kg);  // one warp per (row, histogram group)
  const int64_t want = (tasks + bary::WARPS - 1) / bary::WARPS;
  int64_t g = std::min<int64_t>((int64_t)per_sm * num_sms(), want);
  *grid = (int)std::max<int64_t>(g, 1);
  return OTK_OK;
}

extern "C" int64_t otk_barycenter_ld(int64_t n) { return (n + 3) / 4 * 4; }

extern "C" int64_t otk_barycenter_part_len(int64_t n, int32_t K) {
  int grid = 0;
  if (n <= 0 || K <= 0 || bary_grid(n, K, &grid) != OTK_OK) return -1;
  return (int64_t)grid * (K + 1);
}

extern "C" int otk_barycenter_pad(const float *cost, int64_t n, int64_t ld, float *cost_p,
                                  float *cost_tp, void *stream) {
  OTK_CHECK_ARG(cost && cost_p && cost_tp && n > 0 && ld >= n && ld % 4 == 0 && n <= (1 << 30),
                "otk_barycenter_pad: bad arguments");
  dim3 grid((unsigned)((ld + 31) / 32), (unsigned)((n + 31) / 32));
  bary::pad_kernel<<<grid, 256, 0, as_stream(stream)>>>(cost, (int)n, (int)ld, cost_p, cost_tp);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

extern "C" int otk_solve_barycenter(const float *cost_p, const float *cost_tp, int64_t n, int64_t ld,
                                    int32_t K, const float *log2_hists, const double *weights,
                                    double eps, double threshold, int32_t max_iters, float *F,
                                    float *G, float *B, double *log2_p, double *errors,
                                    int32_t *state, double *part, void *stream) {
  OTK_CHECK_ARG(cost_p && cost_tp && log2_hists && weights && F && G && B && log2_p && errors &&
                    state && part && n > 0 && K > 0 && max_iters > 0,
                "otk_solve_barycenter: bad arguments");
  OTK_CHECK_ARG(n <= (1 << 30) && ld >= n && ld % 4 == 0 && ld <= (1 << 30),
                "otk_solve_barycenter: ld must be >= n and a multiple of 4");
  OTK_CHECK_ARG(eps > 0 && threshold > 0, "otk_solve_barycenter: eps and threshold must be positive");
  int dev = 0, coop = 0;
  OTK_CUDA(cudaGetDevice(&dev));
  OTK_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  OTK_CHECK_ARG(coop, "otk_solve_barycenter: device lacks cooperative launch");
  int grid = 0;
  int rc = bary_grid(n, K, &grid);
  if (rc != OTK_OK) return rc;
  cudaStream_t st = as_stream(stream);
  const size_t plane = sizeof(float) * (size_t)K * ld;
  OTK_CUDA(cudaMemsetAsync(F, 0, plane, st));
  OTK_CUDA(cudaMemsetAsync(G, 0, plane, st));
  OTK_CUDA(cudaMemsetAsync(B, 0, plane, st));
  OTK_CUDA(cudaMemsetAsync(state, 0, sizeof(int32_t) * 8, st));
  bary::Args A{cost_p, cost_tp, (int)n, (int)ld, (int)K, log2_hists, weights,
               (float)(1.4426950408889634 / eps), F, G, B, log2_p, part, errors, state,
               threshold, (int)max_iters};
  void *params[] = {&A};
  OTK_CUDA(cudaLaunchCooperativeKernel(bary_kernel_for(K), dim3(grid), dim3(bary::THREADS), params, 0,
                                       st));
  return OTK_OK;
}
