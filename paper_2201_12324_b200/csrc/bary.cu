// Fixed-support Wasserstein barycenter by iterative Bregman projections
// (SURVEY.md §8f row 4), the whole solve as ONE persistent cooperative kernel.
//
// Replaces reference solve_barycenter (otkit/barycenter.py:96-133), which per
// iteration makes 3K calls of apply_lse_kernel over the shared square support
// geometry.  Here the support cost is materialised once (C and C^T, fp32,
// row-major, written by otk_dense_cost / otk_dense_transpose) and every phase
// streams rows of one of them, 128-bit coalesced.  All potentials are kept in
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

struct Args {
  const float *C, *CT;   // [n, n] row-major each
  int n, K;
  const float *log2h;    // [K, n]
  const double *w;       // [K]
  float kappa;
  float *F, *G, *B;      // [K, n] each (G: zero on entry)
  double *lp2;           // [n]   out: log2 of the (unnormalised) barycenter
  double *part;          // [grid, K + 1]
  double *errors;        // [max_iters]
  int *state;            // [4]: iterations, converged, nan_iteration, grid
  double threshold;
  int max_iters;
};

// LSE2 over j of bias_j - kappa * row_j, one warp, result in every lane.
// bias is written inside this kernel by other CTAs: read it through L2 (ld.cg).
__device__ __forceinline__ float warp_lse2(const float *__restrict__ row, const float *bias, int n,
                                           float kappa, bool vec) {
  const int lane = threadIdx.x & 31;
  Lse2 st;
  st.init();
  for (int j0 = 0; j0 < n; j0 += 256) {
    float u[8];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = j0 + (q * 32 + lane) * 4;
      if (vec) {
        if (j < n) {
          const float4 c = __ldg(reinterpret_cast<const float4 *>(row + j));
          const float4 h = __ldcg(reinterpret_cast<const float4 *>(bias + j));
          u[4 * q + 0] = fmaf(-kappa, c.x, h.x);
          u[4 * q + 1] = fmaf(-kappa, c.y, h.y);
          u[4 * q + 2] = fmaf(-kappa, c.z, h.z);
          u[4 * q + 3] = fmaf(-kappa, c.w, h.w);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) u[4 * q + e] = -INFINITY;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          u[4 * q + e] = (j + e < n) ? fmaf(-kappa, __ldg(row + j + e), __ldcg(bias + j + e)) : -INFINITY;
      }
    }
    float cm = -INFINITY;
#pragma unroll
    for (int e = 0; e < 8; ++e) cm = fmaxf(cm, u[e]);
    if (cm > st.m) {
      st.s *= ex2(st.m - cm);
      st.m = cm;
    }
    const float ms = (st.m == -INFINITY) ? 0.f : st.m;
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc += ex2(u[e] - ms);
    st.s += acc;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, st.m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, st.s, o);
    st.merge(m2, s2);
  }
  return st.value();
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

__global__ void __launch_bounds__(THREADS) bary_kernel(Args A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[THREADS];
  __shared__ int s_stop;
  const int n = A.n, K = A.K;
  const bool vec = (n % 4) == 0;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * THREADS + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * WARPS;
  const int64_t gtid = (int64_t)blockIdx.x * THREADS + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * THREADS;
  const int64_t tasks = (int64_t)K * n;
  for (int t = 1; t <= A.max_iters; ++t) {
    // ---- f half-step: task = i * K + k, so the K readers of row i run side by side
    for (int64_t task = gwarp; task < tasks; task += nwarps) {
      const int i = (int)(task / K), k = (int)(task % K);
      const float v = warp_lse2(A.C + (int64_t)i * n, A.G + (int64_t)k * n, n, A.kappa, vec);
      if (lane == 0) A.F[(int64_t)k * n + i] = A.log2h[(int64_t)k * n + i] - v;
    }
    grid.sync();
    // ---- back-projection: LSE over i of F - kappa C (rows of C^T)
    for (int64_t task = gwarp; task < tasks; task += nwarps) {
      const int j = (int)(task / K), k = (int)(task % K);
      const float v = warp_lse2(A.CT + (int64_t)j * n, A.F + (int64_t)k * n, n, A.kappa, vec);
      if (lane == 0) A.B[(int64_t)k * n + j] = v;
    }
    grid.sync();
    // ---- geometric mean, marginal error, g update
    double nan_count = 0.0;
    for (int64_t j = gtid; j < n; j += nthreads) {
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += A.w[k] * (double)__ldcg(A.B + (int64_t)k * n + j);
      A.lp2[j] = s;
      nan_count += (s != s) ? 1.0 : 0.0;
    }
    for (int k = 0; k < K; ++k) {
      double e = 0.0;
      for (int64_t j = gtid; j < n; j += nthreads) {
        const double lp = A.lp2[j];
        const double bk = (double)__ldcg(A.B + (int64_t)k * n + j);
        const double gk = (double)__ldcg(A.G + (int64_t)k * n + j);
        e += fabs(exp2(bk + gk) - exp2(lp));
        A.G[(int64_t)k * n + j] = (float)(lp - bk);
      }
      e = block_sum(e, red);
      if (threadIdx.x == 0) A.part[(int64_t)blockIdx.x * (K + 1) + k] = e;
    }
    nan_count = block_sum(nan_count, red);
    if (threadIdx.x == 0) A.part[(int64_t)blockIdx.x * (K + 1) + K] = nan_count;
    grid.sync();
    // ---- decision (identical in every CTA: same partials, same order)
    if (threadIdx.x == 0) {
      double err = 0.0, nans = 0.0;
      for (int k = 0; k < K; ++k) {
        double e = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) e += __ldcg(A.part + (int64_t)b * (K + 1) + k);
        err = fmax(err, e);
      }
      for (unsigned b = 0; b < gridDim.x; ++b) nans += __ldcg(A.part + (int64_t)b * (K + 1) + K);
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
    __syncthreads();
    if (s_stop) break;
  }
}

}  // namespace bary
}  // namespace otk

using namespace otk;

static int bary_grid(int64_t n, int32_t K, int *grid) {
  int per_sm = 0;
  OTK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bary::bary_kernel, bary::THREADS, 0));
  if (per_sm < 1) {
    set_error("bary: kernel does not fit on an SM");
    return OTK_ENOTSUP;
  }
  const int64_t want = ((int64_t)K * n + bary::WARPS - 1) / bary::WARPS;  // one warp per row task
  int64_t g = std::min<int64_t>((int64_t)per_sm * num_sms(), want);
  *grid = (int)std::max<int64_t>(g, 1);
  return OTK_OK;
}

extern "C" int64_t otk_barycenter_part_len(int64_t n, int32_t K) {
  int grid = 0;
  if (n <= 0 || K <= 0 || bary_grid(n, K, &grid) != OTK_OK) return -1;
  return (int64_t)grid * (K + 1);
}

extern "C" int otk_solve_barycenter(const float *cost, const float *cost_t, int64_t n, int32_t K,
                                    const float *log2_hists, const double *weights, double eps,
                                    double threshold, int32_t max_iters, float *F, float *G,
                                    float *B, double *log2_p, double *errors, int32_t *state,
                                    double *part, void *stream) {
  OTK_CHECK_ARG(cost && cost_t && log2_hists && weights && F && G && B && log2_p && errors && state &&
                    part && n > 0 && K > 0 && max_iters > 0,
                "otk_solve_barycenter: bad arguments");
  OTK_CHECK_ARG(n <= (1 << 30), "otk_solve_barycenter: support too large");
  OTK_CHECK_ARG(eps > 0 && threshold > 0, "otk_solve_barycenter: eps and threshold must be positive");
  int dev = 0, coop = 0;
  OTK_CUDA(cudaGetDevice(&dev));
  OTK_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  OTK_CHECK_ARG(coop, "otk_solve_barycenter: device lacks cooperative launch");
  int grid = 0;
  int rc = bary_grid(n, K, &grid);
  if (rc != OTK_OK) return rc;
  cudaStream_t st = as_stream(stream);
  OTK_CUDA(cudaMemsetAsync(G, 0, sizeof(float) * (size_t)K * n, st));
  OTK_CUDA(cudaMemsetAsync(state, 0, sizeof(int32_t) * 4, st));
  bary::Args A{cost, cost_t, (int)n, (int)K, log2_hists, weights,
               (float)(1.4426950408889634 / eps), F, G, B, log2_p, part, errors, state,
               threshold, (int)max_iters};
  void *params[] = {&A};
  OTK_CUDA(cudaLaunchCooperativeKernel((void *)bary::bary_kernel, dim3(grid), dim3(bary::THREADS),
                                       params, 0, st));
  return OTK_OK;
}
