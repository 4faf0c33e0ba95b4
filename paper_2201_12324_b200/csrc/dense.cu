// Materialised-cost path (DenseGeometry, reference geometry.py:171-211) for
// many independent small problems (BASELINE.json configs[2]).
//
// K4 dense_cost:  C[b,i,j] = sum_k (x_bik - y_bjk)^2  (difference form: no
//                 cancellation; exact-zero diagonal for identical sets).
// K3 dense_lse:   the log-domain kernel application over a stored C, fused
//                 with the potential update.  HBM bound: every half-step
//                 streams C once with 128-bit coalesced loads.
//   axis 0 (rows): one warp per row i, lanes stride the row with float4.
//   axis 1 (cols): one thread per 4 adjacent columns, a CTA owns a problem's
//                 column block and R row groups walk disjoint row ranges;
//                 row groups merge through shared memory in fixed order.
// Batched check and reg_ot_cost reductions run one CTA per problem with
// fixed-order float64 tree reductions (deterministic).
#include <algorithm>

#include "otk_common.cuh"

namespace otk {

// ------------------------------------------------------------------ K4
constexpr int DC_T = 32;   // transpose tile
constexpr int DC_B = 64;   // cost tile: 64 x 64 outputs per CTA, 4 x 4 per thread

// C[b,i,j] = sum_k (x_bik - y_bjk)^2 in the difference form (no cancellation).
// Also writes C^T[b, j, i] when cost_t != NULL, staged through shared memory
// so both stores are coalesced: the column half-steps then stream C^T with
// the row kernel instead of striding down the columns of C.
__global__ void __launch_bounds__(256) dense_cost_kernel(const float *__restrict__ x,
                                                         const float *__restrict__ y, int64_t n,
                                                         int64_t m, int d, int same, int eucl,
                                                         float *__restrict__ cost,
                                                         float *__restrict__ cost_t) {
  extern __shared__ float sm[];  // xs[64][d+1], ys[64][d+1]; reused as the [64][65] out tile
  const int b = blockIdx.z;
  const int64_t i0 = (int64_t)blockIdx.y * DC_B, j0 = (int64_t)blockIdx.x * DC_B;
  const float *xb = x + (int64_t)b * n * d;
  const float *yb = y + (int64_t)b * m * d;
  const int ld = d + 1;
  float *xs = sm, *ys = sm + DC_B * ld;
  for (int idx = threadIdx.x; idx < DC_B * d; idx += blockDim.x) {
    const int r = idx / d, k = idx % d;
    xs[r * ld + k] = (i0 + r < n) ? xb[(i0 + r) * d + k] : 0.f;
    ys[r * ld + k] = (j0 + r < m) ? yb[(j0 + r) * d + k] : 0.f;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // rows ty + 16*r, cols tx + 16*c
  float acc[4][4] = {};
  for (int k = 0; k < d; ++k) {
    float xv[4], yv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) xv[r] = xs[(ty + 16 * r) * ld + k];
#pragma unroll
    for (int c = 0; c < 4; ++c) yv[c] = ys[(tx + 16 * c) * ld + k];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float df = xv[r] - yv[c];
        acc[r][c] = fmaf(df, df, acc[r][c]);
      }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t i = i0 + ty + 16 * r, j = j0 + tx + 16 * c;
      if (eucl) acc[r][c] = sqrtf(acc[r][c]);
      if (same && i == j) acc[r][c] = 0.f;
      if (i < n && j < m) cost[((int64_t)b * n + i) * m + j] = acc[r][c];
    }
  if (cost_t == nullptr) return;
  __syncthreads();  // operands no longer needed: reuse smem for the output tile
  float *tile = sm;  // [64][65]
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) tile[(ty + 16 * r) * (DC_B + 1) + tx + 16 * c] = acc[r][c];
  __syncthreads();
  const int lane = threadIdx.x & 63, grp = threadIdx.x >> 6;  // 4 groups of 64 lanes
  for (int jj = grp; jj < DC_B; jj += 4) {  // row jj of C^T = column j0+jj of C
    const int64_t j = j0 + jj, i = i0 + lane;
    if (i < n && j < m) cost_t[((int64_t)b * m + j) * n + i] = tile[lane * (DC_B + 1) + jj];
  }
}

// C^T[b] = C[b]^T for a stored cost (DenseGeometry): 32x32 shared tiles.
__global__ void __launch_bounds__(256) dense_transpose_kernel(const float *__restrict__ C,
                                                              int64_t n, int64_t m,
                                                              float *__restrict__ CT) {
  __shared__ float tile[DC_T][DC_T + 1];
  const int b = blockIdx.z;
  const int64_t i0 = (int64_t)blockIdx.y * DC_T, j0 = (int64_t)blockIdx.x * DC_T;
  const int tj = threadIdx.x & 31, ti = threadIdx.x >> 5;
  for (int r = ti; r < DC_T; r += 8) {
    const int64_t i = i0 + r, j = j0 + tj;
    tile[r][tj] = (i < n && j < m) ? C[((int64_t)b * n + i) * m + j] : 0.f;
  }
  __syncthreads();
  for (int r = ti; r < DC_T; r += 8) {
    const int64_t j = j0 + r, i = i0 + tj;
    if (i < n && j < m) CT[((int64_t)b * m + j) * n + i] = tile[tj][r];
  }
}

// ------------------------------------------------------------------ K3 rows
__global__ void __launch_bounds__(256) dense_rows_kernel(
    const float *__restrict__ C, int64_t n, int64_t m, const float *__restrict__ in_bias,
    const float *__restrict__ base, int mode, const float *__restrict__ eps_arr,
    const float *__restrict__ kappa_next, const int *__restrict__ active, float *__restrict__ out,
    float *__restrict__ out_bias, int *__restrict__ first_bad, int step) {
  const int b = blockIdx.y;
  if (active != nullptr && !active[b]) return;
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (i >= n) return;
  const float eps = eps_arr[b];
  const float kappa = kLog2e / eps;
  const float *row = C + ((int64_t)b * n + i) * m;
  const float *bias = in_bias + (int64_t)b * m;
  Lse2 st;
  st.init();
  const bool vec = (m % 4 == 0);
  if (vec) {
    for (int64_t j0 = 0; j0 < m; j0 += 32 * 16) {
      float u[16];
      float cmax = -INFINITY;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t j = j0 + (q * 32 + lane) * 4;
        if (j < m) {
          float4 c4 = __ldg(reinterpret_cast<const float4 *>(row + j));
          float4 h4 = __ldg(reinterpret_cast<const float4 *>(bias + j));
          u[q * 4 + 0] = fmaf(-kappa, c4.x, h4.x);
          u[q * 4 + 1] = fmaf(-kappa, c4.y, h4.y);
          u[q * 4 + 2] = fmaf(-kappa, c4.z, h4.z);
          u[q * 4 + 3] = fmaf(-kappa, c4.w, h4.w);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) u[q * 4 + e] = -INFINITY;
        }
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) cmax = fmaxf(cmax, u[e]);
      if (cmax > st.m) {
        st.s *= ex2(st.m - cmax);
        st.m = cmax;
      }
      const float msub = (st.m == -INFINITY) ? 0.f : st.m;
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 16; ++e) acc += ex2(u[e] - msub);
      st.s += acc;
    }
  } else {
    for (int64_t j = lane; j < m; j += 32) {
      float u = fmaf(-kappa, row[j], bias[j]);
      if (u > st.m) {
        st.s *= ex2(st.m - u);
        st.m = u;
      }
      st.s += (st.m == -INFINITY) ? 0.f : ex2(u - st.m);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float m2 = __shfl_xor_sync(0xffffffffu, st.m, o);
    float s2 = __shfl_xor_sync(0xffffffffu, st.s, o);
    st.merge(m2, s2);
  }
  if (lane == 0) {
    const float L = st.value();
    const int64_t o = (int64_t)b * n + i;
    const float bo = base[o];
    float v = (mode == OTK_FIN_SOLVER) ? eps * bo - eps * kLn2 * L : bo + eps * kLn2 * L;
    out[o] = v;
    if (out_bias != nullptr)
      out_bias[o] = (mode == OTK_FIN_SOLVER) ? next_bias(bo, L, eps, kappa_next[b])
                                              : v * kappa_next[b];
    if (first_bad != nullptr && bad_potential(v)) atomicMin(first_bad + b, step);
  }
}

// ------------------------------------------------------------------ K3 cols
constexpr int DCOL_COLS = 512;  // columns per CTA (128 threads x float4)
constexpr int DCOL_GROUPS = 4;  // row groups per CTA
constexpr int DCOL_RB = 8;      // rows per online-update batch

__global__ void __launch_bounds__(128 * DCOL_GROUPS) dense_cols_kernel(
    const float *__restrict__ C, int64_t n, int64_t m, const float *__restrict__ in_bias,
    const float *__restrict__ base, int mode, const float *__restrict__ eps_arr,
    const float *__restrict__ kappa_next, const int *__restrict__ active, float *__restrict__ out,
    float *__restrict__ out_bias, int *__restrict__ first_bad, int step) {
  __shared__ float shm[DCOL_GROUPS][2][DCOL_COLS];
  const int b = blockIdx.y;
  if (active != nullptr && !active[b]) return;
  const int tc = threadIdx.x & 127, grp = threadIdx.x >> 7;
  const int64_t jbase = (int64_t)blockIdx.x * DCOL_COLS + tc * 4;
  const float eps = eps_arr[b];
  const float kappa = kLog2e / eps;
  const float *Cb = C + (int64_t)b * n * m;
  const float *bias = in_bias + (int64_t)b * n;
  float mx[4], sm[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    mx[e] = -INFINITY;
    sm[e] = 0.f;
  }
  const int64_t rows_per = (n + DCOL_GROUPS - 1) / DCOL_GROUPS;
  const int64_t r_begin = grp * rows_per, r_end = min(n, r_begin + rows_per);
  const bool vec = (m % 4 == 0) && (jbase + 3 < m);
  for (int64_t i0 = r_begin; i0 < r_end; i0 += DCOL_RB) {
    float u[DCOL_RB][4];
#pragma unroll
    for (int r = 0; r < DCOL_RB; ++r) {
      int64_t i = i0 + r;
      if (i < r_end) {
        float hb = __ldg(bias + i);
        const float *crow = Cb + i * m;
        if (vec) {
          float4 c4 = __ldg(reinterpret_cast<const float4 *>(crow + jbase));
          u[r][0] = fmaf(-kappa, c4.x, hb);
          u[r][1] = fmaf(-kappa, c4.y, hb);
          u[r][2] = fmaf(-kappa, c4.z, hb);
          u[r][3] = fmaf(-kappa, c4.w, hb);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            u[r][e] = (jbase + e < m) ? fmaf(-kappa, crow[jbase + e], hb) : -INFINITY;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) u[r][e] = -INFINITY;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float cmax = -INFINITY;
#pragma unroll
      for (int r = 0; r < DCOL_RB; ++r) cmax = fmaxf(cmax, u[r][e]);
      if (cmax > mx[e]) {
        sm[e] *= ex2(mx[e] - cmax);
        mx[e] = cmax;
      }
      const float msub = (mx[e] == -INFINITY) ? 0.f : mx[e];
      float acc = 0.f;
#pragma unroll
      for (int r = 0; r < DCOL_RB; ++r) acc += ex2(u[r][e] - msub);
      sm[e] += acc;
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    shm[grp][0][tc * 4 + e] = mx[e];
    shm[grp][1][tc * 4 + e] = sm[e];
  }
  __syncthreads();
  if (grp != 0) return;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t j = jbase + e;
    Lse2 st;
    st.m = shm[0][0][tc * 4 + e];
    st.s = shm[0][1][tc * 4 + e];
    for (int g2 = 1; g2 < DCOL_GROUPS; ++g2) st.merge(shm[g2][0][tc * 4 + e], shm[g2][1][tc * 4 + e]);
    if (j < m) {
      const float L = st.value();
      const int64_t o = (int64_t)b * m + j;
      const float bo = base[o];
      float v = (mode == OTK_FIN_SOLVER) ? eps * bo - eps * kLn2 * L : bo + eps * kLn2 * L;
      out[o] = v;
      if (out_bias != nullptr)
        out_bias[o] = (mode == OTK_FIN_SOLVER) ? next_bias(bo, L, eps, kappa_next[b])
                                                : v * kappa_next[b];
      if (first_bad != nullptr && bad_potential(v)) atomicMin(first_bad + b, step);
    }
  }
}

// transport_matrix for a stored cost: P = exp((f_i + g_j - C_ij)/eps), float64 exp.
__global__ void dense_plan_kernel(const float *__restrict__ C, int64_t n, int64_t m,
                                  const float *__restrict__ f, const float *__restrict__ g,
                                  double inv_eps, float *__restrict__ plan) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n * m) return;
  int64_t i = idx / m, j = idx % m;
  plan[idx] = (float)exp(((double)f[i] + (double)g[j] - (double)C[idx]) * inv_eps);
}

// ------------------------------------------------------------------ batched check
constexpr int BC_T = 256;

__device__ void block_sum8(double (&v)[8], double *sh /* [8][BC_T] */) {
  for (int k = 0; k < 8; ++k) sh[k * BC_T + threadIdx.x] = v[k];
  __syncthreads();
  for (int s = BC_T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < 8; ++k) sh[k * BC_T + threadIdx.x] += sh[k * BC_T + threadIdx.x + s];
    __syncthreads();
  }
  for (int k = 0; k < 8; ++k) v[k] = sh[k * BC_T];
}

__global__ void __launch_bounds__(BC_T) check_batched_kernel(
    const float *__restrict__ f_prev, const float *__restrict__ f_next,
    const float *__restrict__ a, int64_t n, const float *__restrict__ g,
    const float *__restrict__ bw, int64_t m, const float *__restrict__ eps_arr,
    const int *__restrict__ active, double *__restrict__ out) {
  __shared__ double sh[8 * BC_T];
  const int b = blockIdx.x;
  if (active != nullptr && !active[b]) return;
  const double inv_eps = 1.0 / (double)eps_arr[b];
  double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = threadIdx.x; i < n; i += BC_T) {
    const int64_t o = (int64_t)b * n + i;
    double fp = f_prev[o], ai = a[o];
    if (f_next != nullptr) {
      double r = (ai > 0.0) ? ai * exp((fp - (double)f_next[o]) * inv_eps) : 0.0;
      v[0] += fabs(r - ai);
      v[1] += r;
    }
    if (ai > 0.0) v[2] += ai * fp;
    v[4] += (fp != fp) ? 1.0 : 0.0;
    v[6] += (fp == INFINITY) ? 1.0 : 0.0;
  }
  for (int64_t j = threadIdx.x; j < m; j += BC_T) {
    const int64_t o = (int64_t)b * m + j;
    double gj = g[o], bj = bw[o];
    if (bj > 0.0) v[3] += bj * gj;
    v[5] += (gj != gj) ? 1.0 : 0.0;
    v[7] += (gj == INFINITY) ? 1.0 : 0.0;
  }
  block_sum8(v, sh);
  if (threadIdx.x < 8) out[b * 8 + threadIdx.x] = v[threadIdx.x];
}

// ------------------------------------------------------------------ batched cost
__global__ void __launch_bounds__(BC_T) dense_cost_reduce_kernel(
    const float *__restrict__ C, int64_t n, int64_t m, const float *__restrict__ f,
    const float *__restrict__ g, const float *__restrict__ eps_arr, double *__restrict__ out) {
  __shared__ double sh[8 * BC_T];
  const int b = blockIdx.x;
  const float kappa = kLog2e / eps_arr[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double tr = 0.0, ms = 0.0;
  for (int64_t i = warp; i < n; i += BC_T / 32) {
    const float fi = f[(int64_t)b * n + i];
    const float *crow = C + ((int64_t)b * n + i) * m;
    float mxv = -INFINITY, s = 0.f, t = 0.f;
    for (int64_t j = lane; j < m; j += 32) {
      float c = crow[j];
      float u = (fi + g[(int64_t)b * m + j] - c) * kappa;
      if (u > mxv) {
        float sc = ex2(mxv - u);
        s *= sc;
        t *= sc;
        mxv = u;
      }
      float p = (mxv == -INFINITY) ? 0.f : ex2(u - mxv);
      s += p;
      t = fmaf(c, p, t);
    }
    for (int o = 16; o > 0; o >>= 1) {
      float m2 = __shfl_xor_sync(0xffffffffu, mxv, o);
      float s2 = __shfl_xor_sync(0xffffffffu, s, o);
      float t2 = __shfl_xor_sync(0xffffffffu, t, o);
      float mm = fmaxf(mxv, m2);
      if (mm != -INFINITY) {
        float a1 = ex2(mxv - mm), a2 = ex2(m2 - mm);
        s = s * a1 + s2 * a2;
        t = t * a1 + t2 * a2;
        mxv = mm;
      }
    }
    if (lane == 0 && mxv != -INFINITY) {
      double w = exp2((double)mxv);
      tr += w * t;
      ms += w * s;
    }
  }
  double v[8] = {tr, ms, 0, 0, 0, 0, 0, 0};
  block_sum8(v, sh);
  if (threadIdx.x == 0) {
    out[b * 2 + 0] = v[0];
    out[b * 2 + 1] = v[1];
  }
}

}  // namespace otk

using namespace otk;

extern "C" {

int otk_dense_cost(const float *x, const float *y, int64_t batch, int64_t n, int64_t m, int32_t d,
                   int32_t flags, float *cost, float *cost_t, void *stream) {
  OTK_CHECK_ARG(x && y && cost && batch > 0 && n > 0 && m > 0 && d > 0, "otk_dense_cost: bad arguments");
  OTK_CHECK_ARG(batch <= 65535, "otk_dense_cost: batch too large");
  size_t smem = std::max(2 * DC_B * (size_t)(d + 1), (size_t)DC_B * (DC_B + 1)) * sizeof(float);
  OTK_CHECK_ARG(smem <= 200 * 1024, "otk_dense_cost: d too large");
  if (smem > 48 * 1024)
    OTK_CUDA(cudaFuncSetAttribute(dense_cost_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  dim3 grid((unsigned)((m + DC_B - 1) / DC_B), (unsigned)((n + DC_B - 1) / DC_B), (unsigned)batch);
  dense_cost_kernel<<<grid, 256, smem, as_stream(stream)>>>(x, y, n, m, d,
                                                            (flags & OTK_SAME_POINTS) ? 1 : 0,
                                                            (flags & OTK_COST_EUCL) ? 1 : 0, cost,
                                                            cost_t);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_dense_transpose(const float *cost, int64_t batch, int64_t n, int64_t m, float *cost_t,
                        void *stream) {
  OTK_CHECK_ARG(cost && cost_t && batch > 0 && batch <= 65535 && n > 0 && m > 0,
                "otk_dense_transpose: bad arguments");
  dim3 grid((unsigned)((m + DC_T - 1) / DC_T), (unsigned)((n + DC_T - 1) / DC_T), (unsigned)batch);
  dense_transpose_kernel<<<grid, 256, 0, as_stream(stream)>>>(cost, n, m, cost_t);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_dense_lse(const float *cost, int64_t batch, int64_t n, int64_t m, int32_t axis,
                  const float *in_bias, const float *base, int32_t mode, const float *eps,
                  const float *kappa_next, const int32_t *active, float *out_pot, float *out_bias,
                  int32_t *first_bad, int32_t step, void *stream) {
  OTK_CHECK_ARG(cost && in_bias && base && eps && out_pot && batch > 0 && n > 0 && m > 0,
                "otk_dense_lse: bad arguments");
  OTK_CHECK_ARG(axis == 0 || axis == 1, "otk_dense_lse: axis must be 0 (rows) or 1 (cols)");
  OTK_CHECK_ARG(out_bias == nullptr || kappa_next != nullptr, "otk_dense_lse: kappa_next missing");
  OTK_CHECK_ARG(batch <= 65535, "otk_dense_lse: batch too large");
  cudaStream_t st = as_stream(stream);
  if (axis == 0) {
    dim3 grid((unsigned)((n + 7) / 8), (unsigned)batch);
    dense_rows_kernel<<<grid, 256, 0, st>>>(cost, n, m, in_bias, base, mode, eps, kappa_next,
                                            active, out_pot, out_bias, first_bad, step);
  } else {
    dim3 grid((unsigned)((m + DCOL_COLS - 1) / DCOL_COLS), (unsigned)batch);
    dense_cols_kernel<<<grid, 128 * DCOL_GROUPS, 0, st>>>(cost, n, m, in_bias, base, mode, eps,
                                                          kappa_next, active, out_pot, out_bias,
                                                          first_bad, step);
  }
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_check_batched(const float *f_prev, const float *f_next, const float *a, int64_t n,
                      const float *g, const float *b, int64_t m, int64_t batch, const float *eps,
                      const int32_t *active, double *out, void *stream) {
  OTK_CHECK_ARG(f_prev && a && g && b && eps && out && batch > 0 && n > 0 && m > 0,
                "otk_check_batched: bad arguments");
  check_batched_kernel<<<(unsigned)batch, BC_T, 0, as_stream(stream)>>>(f_prev, f_next, a, n, g, b,
                                                                         m, eps, active, out);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_dense_plan(const float *cost, int64_t n, int64_t m, const float *f, const float *g,
                   double eps, float *plan, void *stream) {
  OTK_CHECK_ARG(cost && f && g && plan && n > 0 && m > 0 && eps > 0, "otk_dense_plan: bad arguments");
  dense_plan_kernel<<<(unsigned)((n * m + 255) / 256), 256, 0, as_stream(stream)>>>(cost, n, m, f, g,
                                                                                    1.0 / eps, plan);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_dense_cost_reduce(const float *cost, int64_t batch, int64_t n, int64_t m, const float *f,
                          const float *g, const float *eps, double *out, void *stream) {
  OTK_CHECK_ARG(cost && f && g && eps && out && batch > 0 && n > 0 && m > 0,
                "otk_dense_cost_reduce: bad arguments");
  dense_cost_reduce_kernel<<<(unsigned)batch, BC_T, 0, as_stream(stream)>>>(cost, n, m, f, g, eps,
                                                                            out);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

}  // extern "C"
