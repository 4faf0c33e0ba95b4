// Envelope gradient in the source points, online.
//
// Replaces reference sinkhorn.grad_points (sinkhorn.py:232-246), which
// materialises P = exp((f + g - C)/eps) through transport_matrix (and so
// refuses n*m > 4e6, geometry.py:46,162-168), with one streaming pass:
//     grad_i = 2 (r_i x_i - sum_j P_ij y_j),   r_i = sum_j P_ij
// P is rebuilt tile by tile from the cost (|x|^2 + |y|^2 - 2<x,y>, clamped
// at 0, exact-zero diagonal for identical sets: geometry.py:263-292) and
// exponentiated directly like the reference (converged potentials keep
// P <= 1).  The P @ Y contraction is the flash-attention-forward shape; this
// FP32 version tiles 64 rows x 64 output dims per CTA and recomputes the
// cost tile per 64-dim output chunk (d > 64), fixed reduction order.
#include "otk_common.cuh"

namespace otk {

constexpr int GP_T = 64;   // rows / columns / output dims per tile
constexpr int GP_KC = 16;  // cost-dot depth per shared-memory stage

__global__ void __launch_bounds__(256) grad_points_kernel(
    const float *__restrict__ P, const float *__restrict__ psq, int64_t np,
    const float *__restrict__ Q, const float *__restrict__ qsq, int64_t nq, int d,
    const float *__restrict__ f, const float *__restrict__ g, float kappa, int same,
    float *__restrict__ grad) {
  __shared__ __align__(16) float As[GP_KC][GP_T + 4];
  __shared__ __align__(16) float Bs[GP_KC][GP_T + 4];
  __shared__ float Pt[GP_T][GP_T + 1];   // plan tile [row][col]
  __shared__ float Yt[GP_T][GP_T + 1];   // y tile [col][dim]
  __shared__ float rmass[GP_T];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t row0 = (int64_t)blockIdx.x * GP_T;
  const int k0 = blockIdx.y * GP_T;  // output-dim chunk
  float fr[4], pr[4], rsum[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t i = row0 + ty * 4 + r;
    fr[r] = i < np ? f[i] : 0.f;
    pr[r] = i < np ? psq[i] : 0.f;
    rsum[r] = 0.f;
  }
  float acc[4][4] = {};  // rows ty*4+r, dims tx*4+c (of this chunk)
  for (int64_t col0 = 0; col0 < nq; col0 += GP_T) {
    // ---- cost tile (rows ty*4+r, cols tx*4+c)
    float dot[4][4] = {};
    for (int kc = 0; kc < d; kc += GP_KC) {
      for (int idx = tid; idx < GP_T * GP_KC; idx += 256) {
        const int r = idx / GP_KC, k = idx % GP_KC;
        const int64_t gi = row0 + r, gj = col0 + r;
        As[k][r] = (gi < np && kc + k < d) ? P[gi * d + kc + k] : 0.f;
        Bs[k][r] = (gj < nq && kc + k < d) ? Q[gj * d + kc + k] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < GP_KC; ++k) {
        const float4 a = *reinterpret_cast<const float4 *>(&As[k][ty * 4]);
        const float4 b = *reinterpret_cast<const float4 *>(&Bs[k][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) dot[r][c] = fmaf(av[r], bv[c], dot[r][c]);
      }
      __syncthreads();
    }
    // ---- plan tile
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t j = col0 + tx * 4 + c;
      const bool ok = j < nq;
      const float qj = ok ? qsq[j] : 0.f, gj = ok ? g[j] : 0.f;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t i = row0 + ty * 4 + r;
        float cij = fmaxf(pr[r] + qj - 2.f * dot[r][c], 0.f);
        if (same && i == j) cij = 0.f;
        const float pij = ok ? ex2(kappa * (fr[r] + gj - cij)) : 0.f;
        Pt[ty * 4 + r][tx * 4 + c] = pij;
        rsum[r] += pij;
      }
    }
    // ---- y tile for this output chunk: Yt[col][dim]
    for (int idx = tid; idx < GP_T * GP_T; idx += 256) {
      const int c = idx / GP_T, k = idx % GP_T;
      const int64_t j = col0 + c;
      Yt[c][k] = (j < nq && k0 + k < d) ? Q[j * d + k0 + k] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < GP_T; ++c) {
      float yv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) yv[q] = Yt[c][tx * 4 + q];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float p = Pt[ty * 4 + r][c];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[r][q] = fmaf(p, yv[q], acc[r][q]);
      }
    }
    __syncthreads();
  }
  // row masses: the 16 column-threads of a row, fixed butterfly order
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) rsum[r] += __shfl_xor_sync(0xffffffffu, rsum[r], o);
    if (tx == 0) rmass[ty * 4 + r] = rsum[r];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t i = row0 + ty * 4 + r;
    if (i >= np) continue;
    const float rm = rmass[ty * 4 + r];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = k0 + tx * 4 + q;
      if (k < d) grad[i * d + k] = 2.f * (rm * P[i * d + k] - acc[r][q]);
    }
  }
}

}  // namespace otk

using namespace otk;

extern "C" int otk_grad_points(const float *p, const float *p_sq, int64_t np, const float *q,
                               const float *q_sq, int64_t nq, int32_t d, const float *f,
                               const float *g, double eps, int32_t flags, float *grad,
                               void *stream) {
  OTK_CHECK_ARG(p && p_sq && q && q_sq && f && g && grad && np > 0 && nq > 0 && d > 0,
                "otk_grad_points: bad arguments");
  OTK_CHECK_ARG(eps > 0, "otk_grad_points: eps must be positive");
  dim3 grid((unsigned)((np + GP_T - 1) / GP_T), (unsigned)((d + GP_T - 1) / GP_T));
  grad_points_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      p, p_sq, np, q, q_sq, nq, d, f, g, (float)(1.4426950408889634 / eps),
      (flags & OTK_SAME_POINTS) ? 1 : 0, grad);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}
