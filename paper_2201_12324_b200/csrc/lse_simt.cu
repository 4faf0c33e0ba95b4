// K1 -- online squared-Euclidean cost + streaming log2-sum-exp2 half-step on
// the FP32 FMA pipe, plus the online reg_ot_cost (K6) and transport_matrix.
//
// Replaces PointCloudGeometry.apply_lse_kernel (reference geometry.py:336-354),
// whose per-block cost _cost_block (263-276) is recomputed on the fly from
//   C_ij = |p_i|^2 + |q_j|^2 - 2 <p_i, q_j>       (rank d+2)
// and never materialised.  In log2 units with kappa = log2(e)/eps:
//   (pot_j - C_ij) * kappa = u_ij - kappa*|p_i|^2,
//   u_ij = 2*kappa*<p_i,q_j> + kappa*(pot_j - |q_j|^2)      (bias_j = kappa*pot_j)
// The row term is subtracted once per row from the reduced value.  OTK_CLAMP
// applies max(C,0) exactly (u <= bias_j + kappa*|p_i|^2); OTK_SAME_POINTS
// forces the zero diagonal (geometry.py:278-292).
//
// CTA tile: 64 rows (P) x 64 columns (Q), 256 threads, 4x4 per thread.  Each
// CTA streams a contiguous column range (split) of Q through shared memory
// and keeps a per-row online (max, sum) in registers; the 16 threads sharing
// a row merge with shuffles in a fixed order (deterministic).
#include <cstdlib>

#include "otk_common.cuh"

namespace otk {

constexpr int SB_M = 64, SB_N = 64, SB_T = 256;

template <int KC, bool CLAMP, bool SAME, bool EU>
__global__ void __launch_bounds__(SB_T) lse_simt_kernel(
    const float *__restrict__ P, const float *__restrict__ psq, int64_t np,
    const float *__restrict__ Q, const float *__restrict__ qsq, int64_t nq, int d,
    const float *__restrict__ qbias, float kappa, int64_t cols_per_split,
    float *__restrict__ partial) {
  __shared__ __align__(16) float Ps[KC][SB_M + 4];
  __shared__ __align__(16) float Qs[KC][SB_N + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t row0 = (int64_t)blockIdx.x * SB_M;
  const int split = blockIdx.y;
  const int64_t c_begin = (int64_t)split * cols_per_split;
  const int64_t c_end = min(nq, c_begin + cols_per_split);
  const float two_kappa = 2.f * kappa;
  const float sk = sqrtf(kappa);
  const bool p_resident = (d <= KC);

  float cp[4];
  Lse2 st[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int64_t row = row0 + ty * 4 + r;
    cp[r] = (row < np) ? kappa * psq[row] : 0.f;
    st[r].init();
  }

  for (int64_t col0 = c_begin; col0 < c_end; col0 += SB_N) {
    float acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;

    for (int kc = 0; kc < d; kc += KC) {
      if (!p_resident || col0 == c_begin) {
        for (int idx = tid; idx < SB_M * KC; idx += SB_T) {
          int r = idx / KC, k = idx % KC;
          int64_t gr = row0 + r;
          int gk = kc + k;
          Ps[k][r] = (gr < np && gk < d) ? P[gr * d + gk] : 0.f;
        }
      }
      for (int idx = tid; idx < SB_N * KC; idx += SB_T) {
        int c = idx / KC, k = idx % KC;
        int64_t gc = col0 + c;
        int gk = kc + k;
        Qs[k][c] = (gc < c_end && gk < d) ? Q[gc * d + gk] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        float4 a = *reinterpret_cast<const float4 *>(&Ps[k][ty * 4]);
        float4 b = *reinterpret_cast<const float4 *>(&Qs[k][tx * 4]);
        float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
      }
      __syncthreads();
    }

    // epilogue: u, online log2-sum-exp2 per row
    float hb[4], cq[4];
    bool ok[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int64_t j = col0 + tx * 4 + c;
      ok[c] = j < c_end;
      cq[c] = ok[c] ? qbias[j] : 0.f;
      hb[c] = ok[c] ? fmaf(-kappa, qsq[j], EU ? 0.f : cq[c]) : 0.f;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t row = row0 + ty * 4 + r;
      float u[4];
      float cmax = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float v = fmaf(acc[r][c], two_kappa, hb[c]);
        if (EU) {  // kappa*sqrt(C) = sqrt(kappa) * sqrt(kappa*C), kappa*C = cp - v
          v = (SAME && row == col0 + tx * 4 + c) ? cq[c]
                                                  : fmaf(-sk, sqrt_approx(fmaxf(cp[r] - v, 0.f)), cq[c]);
        } else if (CLAMP) {
          float ub = cq[c] + cp[r];
          v = fminf(v, ub);
          if (SAME && row == col0 + tx * 4 + c) v = ub;
        }
        u[c] = ok[c] ? v : -INFINITY;
        cmax = fmaxf(cmax, u[c]);
      }
      if (cmax > st[r].m + 8.f) {  // lazy rescale (values may exceed m by <= 8)
        st[r].s *= ex2(st[r].m - cmax);
        st[r].m = cmax;
      }
      const float msub = (st[r].m == -INFINITY) ? 0.f : st[r].m;
#pragma unroll
      for (int c = 0; c < 4; ++c) st[r].s += ex2(u[c] - msub);
    }
  }

  // merge the 16 column-threads of each row (fixed butterfly order)
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      float m2 = __shfl_xor_sync(0xffffffffu, st[r].m, o);
      float s2 = __shfl_xor_sync(0xffffffffu, st[r].s, o);
      st[r].merge(m2, s2);
    }
    int64_t row = row0 + ty * 4 + r;
    if (tx == 0 && row < np) partial[(int64_t)split * np + row] = st[r].value() - (EU ? 0.f : cp[r]);
  }
}

// ---------------------------------------------------------------- K1 low-d
// Low-dimension variant (d <= 7): every point is one / two float4
// (coordinates, |q|^2 in slot d), staged into shared memory a chunk of
// columns at a time.  A warp owns LD_R = 4 rows whose query vectors
// p' = (2 kappa p, -kappa, 0..) live in registers, so one dot product gives
// 2 kappa <p,q> - kappa |q|^2; rows are paired so the dot products run as
// packed FFMA2 (two rows per instruction).  Lanes stride the chunk's columns
// with a per-row online log2-sum-exp2 and merge with a fixed butterfly.
constexpr int LD_T = 256, LD_WARPS = LD_T / 32, LD_R = 4, LD_CH = 512, LD_CB = 4;

template <int NV, bool CLAMP, bool SAME, bool EU>
__global__ void __launch_bounds__(LD_T) lse_lowd_kernel(
    const float *__restrict__ P, const float *__restrict__ psq, int64_t np,
    const float *__restrict__ Q, const float *__restrict__ qsq, int64_t nq, int d,
    const float *__restrict__ qbias, float kappa, int64_t cols_per_split,
    float *__restrict__ partial) {
  __shared__ float4 qs[LD_CH * NV];
  __shared__ float bs[LD_CH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = ((int64_t)blockIdx.x * LD_WARPS + warp) * LD_R;
  const int split = blockIdx.y;
  const int64_t c_begin = (int64_t)split * cols_per_split;
  const int64_t c_end = min(nq, c_begin + cols_per_split);
  const float two_k = 2.f * kappa;
  const float sk = sqrtf(kappa);
  // query vectors, two rows per float2 (rows 2t and 2t+1)
  float2 pv[LD_R / 2][4 * NV];
  float cp[LD_R], mx[LD_R], sm[LD_R];
#pragma unroll
  for (int r = 0; r < LD_R; ++r) {
    const int64_t i = min(row0 + r, np - 1);
    cp[r] = kappa * psq[i];
    mx[r] = -INFINITY;
    sm[r] = 0.f;
#pragma unroll
    for (int k = 0; k < 4 * NV; ++k) {
      const float v = (k < d) ? two_k * P[i * d + k] : (k == d ? -kappa : 0.f);
      if (r & 1) pv[r / 2][k].y = v; else pv[r / 2][k].x = v;
    }
  }
  for (int64_t j0 = c_begin; j0 < c_end; j0 += LD_CH) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < LD_CH; idx += LD_T) {
      const int64_t j = j0 + idx;
      float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      float b = -INFINITY;
      if (j < c_end) {
        for (int k = 0; k < d; ++k) v[k] = Q[j * d + k];
        v[d] = qsq[j];
        b = qbias[j];
      }
      qs[idx * NV] = make_float4(v[0], v[1], v[2], v[3]);
      if (NV == 2) qs[idx * NV + 1] = make_float4(v[4], v[5], v[6], v[7]);
      bs[idx] = b;
    }
    __syncthreads();
    const int nvalid = (int)min((int64_t)LD_CH, c_end - j0);
    for (int c0 = lane; c0 < nvalid; c0 += 32 * LD_CB) {
      float u[LD_CB][LD_R];
#pragma unroll
      for (int cb = 0; cb < LD_CB; ++cb) {
        const int c = c0 + 32 * cb;
        const int cc = min(c, LD_CH - 1);
        const float b = (c < nvalid) ? bs[cc] : -INFINITY;
        float qv[4 * NV];
        const float4 q0 = qs[cc * NV];
        qv[0] = q0.x; qv[1] = q0.y; qv[2] = q0.z; qv[3] = q0.w;
        if (NV == 2) {
          const float4 q1 = qs[cc * NV + 1];
          qv[4] = q1.x; qv[5] = q1.y; qv[6] = q1.z; qv[7] = q1.w;
        }
#pragma unroll
        for (int t = 0; t < LD_R / 2; ++t) {
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int k = 0; k < 4 * NV; ++k)
            if (k <= d || k < 4) acc = __ffma2_rn(pv[t][k], make_float2(qv[k], qv[k]), acc);
          float v0 = acc.x, v1 = acc.y;
          if (EU) {  // u = b - sqrt(kappa) sqrt(kappa C), kappa C = cp - v
            v0 = -sk * sqrt_approx(fmaxf(cp[2 * t] - v0, 0.f));
            v1 = -sk * sqrt_approx(fmaxf(cp[2 * t + 1] - v1, 0.f));
            if (SAME) {
              const int64_t j = j0 + c;
              if (j == row0 + 2 * t) v0 = 0.f;
              if (j == row0 + 2 * t + 1) v1 = 0.f;
            }
          } else {
            if (CLAMP) {
              v0 = fminf(v0, cp[2 * t]);
              v1 = fminf(v1, cp[2 * t + 1]);
            }
            if (SAME) {
              const int64_t j = j0 + c;
              if (j == row0 + 2 * t) v0 = cp[2 * t];
              if (j == row0 + 2 * t + 1) v1 = cp[2 * t + 1];
            }
          }
          u[cb][2 * t] = v0 + b;
          u[cb][2 * t + 1] = v1 + b;
        }
      }
#pragma unroll
      for (int r = 0; r < LD_R; ++r) {
        float cm = -INFINITY;
#pragma unroll
        for (int cb = 0; cb < LD_CB; ++cb) cm = fmaxf(cm, u[cb][r]);
        if (cm > mx[r] + 8.f) {
          sm[r] *= ex2(mx[r] - cm);
          mx[r] = cm;
        }
        const float ms = (mx[r] == -INFINITY) ? 0.f : mx[r];
        float acc = 0.f;
#pragma unroll
        for (int cb = 0; cb < LD_CB; ++cb) acc += ex2(u[cb][r] - ms);
        sm[r] += acc;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < LD_R; ++r) {
    Lse2 st;
    st.m = mx[r];
    st.s = sm[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, st.m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, st.s, o);
      st.merge(m2, s2);
    }
    const int64_t i = row0 + r;
    if (lane == 0 && i < np) partial[(int64_t)split * np + i] = st.value() - (EU ? 0.f : cp[r]);
  }
}

// ---------------------------------------------------------------- K6 cost
// Per (split,row): m = max u, s = sum 2^(u-m), t = sum C*2^(u-m),
// u = (f_i + g_j - C_ij)*kappa with C clamped at 0 (and zero diagonal).
template <int KC, bool SAME, bool EU>
__global__ void __launch_bounds__(SB_T) cost_simt_kernel(
    const float *__restrict__ P, const float *__restrict__ psq, int64_t np,
    const float *__restrict__ Q, const float *__restrict__ qsq, int64_t nq, int d,
    const float *__restrict__ f, const float *__restrict__ g, float kappa,
    int64_t cols_per_split, float *__restrict__ out /* [nsplit][np][3] */) {
  __shared__ __align__(16) float Ps[KC][SB_M + 4];
  __shared__ __align__(16) float Qs[KC][SB_N + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t row0 = (int64_t)blockIdx.x * SB_M;
  const int split = blockIdx.y;
  const int64_t c_begin = (int64_t)split * cols_per_split;
  const int64_t c_end = min(nq, c_begin + cols_per_split);

  float pr[4], fr[4], m[4], s[4], t[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int64_t row = row0 + ty * 4 + r;
    pr[r] = row < np ? psq[row] : 0.f;
    fr[r] = row < np ? f[row] : 0.f;
    m[r] = -INFINITY;
    s[r] = 0.f;
    t[r] = 0.f;
  }
  for (int64_t col0 = c_begin; col0 < c_end; col0 += SB_N) {
    float acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;
    for (int kc = 0; kc < d; kc += KC) {
      for (int idx = tid; idx < SB_M * KC; idx += SB_T) {
        int r = idx / KC, k = idx % KC;
        int64_t gr = row0 + r;
        int gk = kc + k;
        Ps[k][r] = (gr < np && gk < d) ? P[gr * d + gk] : 0.f;
      }
      for (int idx = tid; idx < SB_N * KC; idx += SB_T) {
        int c = idx / KC, k = idx % KC;
        int64_t gc = col0 + c;
        int gk = kc + k;
        Qs[k][c] = (gc < c_end && gk < d) ? Q[gc * d + gk] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        float4 a = *reinterpret_cast<const float4 *>(&Ps[k][ty * 4]);
        float4 b = *reinterpret_cast<const float4 *>(&Qs[k][tx * 4]);
        float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int64_t j = col0 + tx * 4 + c;
      if (j >= c_end) continue;
      float qj = qsq[j], gj = g[j];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int64_t row = row0 + ty * 4 + r;
        float cij = fmaxf(pr[r] + qj - 2.f * acc[r][c], 0.f);
        if (EU) cij = sqrtf(cij);
        if (SAME && row == j) cij = 0.f;
        float u = (fr[r] + gj - cij) * kappa;
        if (u > m[r]) {
          float sc = ex2(m[r] - u);
          s[r] *= sc;
          t[r] *= sc;
          m[r] = u;
        }
        float p = (m[r] == -INFINITY) ? 0.f : ex2(u - m[r]);
        s[r] += p;
        t[r] = fmaf(cij, p, t[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      float m2 = __shfl_xor_sync(0xffffffffu, m[r], o);
      float s2 = __shfl_xor_sync(0xffffffffu, s[r], o);
      float t2 = __shfl_xor_sync(0xffffffffu, t[r], o);
      float mm = fmaxf(m[r], m2);
      if (mm != -INFINITY) {
        float a1 = ex2(m[r] - mm), a2 = ex2(m2 - mm);
        s[r] = s[r] * a1 + s2 * a2;
        t[r] = t[r] * a1 + t2 * a2;
        m[r] = mm;
      }
    }
    int64_t row = row0 + ty * 4 + r;
    if (tx == 0 && row < np) {
      float *o = out + ((int64_t)split * np + row) * 3;
      o[0] = m[r];
      o[1] = s[r];
      o[2] = t[r];
    }
  }
}

// Deterministic float64 reduction of the (m, s, t) records into
// out[0] = sum 2^m t, out[1] = sum 2^m s.  One block, fixed order.
__global__ void __launch_bounds__(1024) cost_reduce_kernel(const float *__restrict__ rec, int64_t count,
                                                           double *__restrict__ out) {
  __shared__ double sh[2][1024];
  double tr = 0.0, ms = 0.0;
  for (int64_t k = threadIdx.x; k < count; k += blockDim.x) {
    const float *r = rec + k * 3;
    if (r[0] == -INFINITY) continue;
    double w = exp2((double)r[0]);
    tr += w * (double)r[2];
    ms += w * (double)r[1];
  }
  sh[0][threadIdx.x] = tr;
  sh[1][threadIdx.x] = ms;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + s];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sh[0][0];
    out[1] = sh[1][0];
  }
}

// transport_matrix: one thread per cell, direct formula in float64 exp.
__global__ void plan_kernel(const float *__restrict__ P, const float *__restrict__ psq, int64_t np,
                            const float *__restrict__ Q, const float *__restrict__ qsq, int64_t nq,
                            int d, const float *__restrict__ f, const float *__restrict__ g,
                            double inv_eps, int same, int eucl, float *__restrict__ plan) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= np * nq) return;
  int64_t i = idx / nq, j = idx % nq;
  float dot = 0.f;
  for (int k = 0; k < d; ++k) dot = fmaf(P[i * d + k], Q[j * d + k], dot);
  float c = fmaxf(psq[i] + qsq[j] - 2.f * dot, 0.f);
  if (eucl) c = sqrtf(c);
  if (same && i == j) c = 0.f;
  plan[idx] = (float)exp(((double)f[i] + (double)g[j] - (double)c) * inv_eps);
}

static int pick_kc(int d) { return d <= 4 ? 4 : (d <= 8 ? 8 : 16); }

int lse_simt_launch(const float *p, const float *p_sq, int64_t np, const float *q,
                    const float *q_sq, int64_t nq, int d, const float *q_bias, float kappa,
                    int flags, int nsplit, float *partial, cudaStream_t st) {
  int64_t cps = (nq + nsplit - 1) / nsplit;
  cps = (cps + SB_N - 1) / SB_N * SB_N;
  const bool clamp = flags & OTK_CLAMP, same = flags & OTK_SAME_POINTS, eu = flags & OTK_COST_EUCL;
  if (d <= 7 && !getenv("OTK_SIMT_TILED")) {
    dim3 g2((unsigned)((np + LD_WARPS * LD_R - 1) / (LD_WARPS * LD_R)), (unsigned)nsplit);
#define OTK_LOWD_CASE(NV, CL, SA, EU)                                                     \
    if ((d <= 3) == (NV == 1) && clamp == CL && same == SA && eu == EU) {                 \
      lse_lowd_kernel<NV, CL, SA, EU><<<g2, LD_T, 0, st>>>(p, p_sq, np, q, q_sq, nq, d,     \
                                                           q_bias, kappa, cps, partial);  \
      cudaError_t e = cudaGetLastError();                                                 \
      return e == cudaSuccess ? OTK_OK : cuda_status(e, "lse_lowd_kernel");               \
    }
    OTK_LOWD_CASE(1, false, false, false)
    OTK_LOWD_CASE(1, true, false, false)
    OTK_LOWD_CASE(1, true, true, false)
    OTK_LOWD_CASE(2, false, false, false)
    OTK_LOWD_CASE(2, true, false, false)
    OTK_LOWD_CASE(2, true, true, false)
    OTK_LOWD_CASE(1, true, false, true)
    OTK_LOWD_CASE(1, true, true, true)
    OTK_LOWD_CASE(2, true, false, true)
    OTK_LOWD_CASE(2, true, true, true)
#undef OTK_LOWD_CASE
    set_error("lse_simt: OTK_SAME_POINTS / OTK_COST_EUCL require OTK_CLAMP");
    return OTK_EINVAL;
  }
  dim3 grid((unsigned)((np + SB_M - 1) / SB_M), (unsigned)nsplit);
  const int kc = pick_kc(d);
#define OTK_SIMT_CASE(KC, CL, SA, EU)                                                      \
  if (kc == KC && clamp == CL && same == SA && eu == EU) {                                 \
    lse_simt_kernel<KC, CL, SA, EU><<<grid, SB_T, 0, st>>>(p, p_sq, np, q, q_sq, nq, d,     \
                                                            q_bias, kappa, cps, partial);  \
    cudaError_t e = cudaGetLastError();                                                    \
    return e == cudaSuccess ? OTK_OK : cuda_status(e, "lse_simt_kernel");                  \
  }
  OTK_SIMT_CASE(4, false, false, false)
  OTK_SIMT_CASE(4, true, false, false)
  OTK_SIMT_CASE(4, true, true, false)
  OTK_SIMT_CASE(8, false, false, false)
  OTK_SIMT_CASE(8, true, false, false)
  OTK_SIMT_CASE(8, true, true, false)
  OTK_SIMT_CASE(16, false, false, false)
  OTK_SIMT_CASE(16, true, false, false)
  OTK_SIMT_CASE(16, true, true, false)
  OTK_SIMT_CASE(4, true, false, true)
  OTK_SIMT_CASE(4, true, true, true)
  OTK_SIMT_CASE(8, true, false, true)
  OTK_SIMT_CASE(8, true, true, true)
  OTK_SIMT_CASE(16, true, false, true)
  OTK_SIMT_CASE(16, true, true, true)
#undef OTK_SIMT_CASE
  set_error("lse_simt: OTK_SAME_POINTS / OTK_COST_EUCL require OTK_CLAMP");
  return OTK_EINVAL;
}

}  // namespace otk

using namespace otk;

extern "C" {

size_t otk_cost_workspace_bytes(int64_t np, int64_t nq) {
  (void)nq;
  int nsplit = 16;
  return (size_t)nsplit * (size_t)np * 3 * sizeof(float);
}

int otk_cost_partial(const float *p, const float *p_sq, int64_t np, const float *q,
                     const float *q_sq, int64_t nq, int32_t d, const float *f, const float *g,
                     double eps, int32_t flags, double *out, void *ws, void *stream) {
  OTK_CHECK_ARG(p && p_sq && q && q_sq && f && g && out && ws && np > 0 && nq > 0 && d > 0,
                "otk_cost_partial: bad arguments");
  OTK_CHECK_ARG(eps > 0, "otk_cost_partial: eps must be positive");
  const int nsplit = 16;
  int64_t cps = (nq + nsplit - 1) / nsplit;
  cps = (cps + SB_N - 1) / SB_N * SB_N;
  dim3 grid((unsigned)((np + SB_M - 1) / SB_M), (unsigned)nsplit);
  float *rec = reinterpret_cast<float *>(ws);
  // empty splits must read as -inf records
  const float kappa = (float)(1.4426950408889634 / eps);
  const int kc = pick_kc(d);
  cudaStream_t st = as_stream(stream);
  const bool same = flags & OTK_SAME_POINTS, eu = flags & OTK_COST_EUCL;
#define OTK_COST_CASE(KC, SA, EU)                                                             \
  if (kc == KC && same == SA && eu == EU)                                                     \
    cost_simt_kernel<KC, SA, EU><<<grid, SB_T, 0, st>>>(p, p_sq, np, q, q_sq, nq, d, f, g,     \
                                                        kappa, cps, rec);
  OTK_COST_CASE(4, false, false)
  OTK_COST_CASE(4, true, false)
  OTK_COST_CASE(4, false, true)
  OTK_COST_CASE(4, true, true)
  OTK_COST_CASE(8, false, false)
  OTK_COST_CASE(8, true, false)
  OTK_COST_CASE(8, false, true)
  OTK_COST_CASE(8, true, true)
  OTK_COST_CASE(16, false, false)
  OTK_COST_CASE(16, true, false)
  OTK_COST_CASE(16, false, true)
  OTK_COST_CASE(16, true, true)
#undef OTK_COST_CASE
  OTK_LAUNCH_CHECK();
  cost_reduce_kernel<<<1, 1024, 0, st>>>(rec, (int64_t)nsplit * np, out);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_transport_matrix(const float *p, const float *p_sq, int64_t np, const float *q,
                         const float *q_sq, int64_t nq, int32_t d, const float *f, const float *g,
                         double eps, int32_t flags, float *plan, void *stream) {
  OTK_CHECK_ARG(p && p_sq && q && q_sq && f && g && plan && np > 0 && nq > 0 && d > 0,
                "otk_transport_matrix: bad arguments");
  OTK_CHECK_ARG(eps > 0, "otk_transport_matrix: eps must be positive");
  int64_t cells = np * nq;
  plan_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, as_stream(stream)>>>(
      p, p_sq, np, q, q_sq, nq, d, f, g, 1.0 / eps, (flags & OTK_SAME_POINTS) ? 1 : 0,
      (flags & OTK_COST_EUCL) ? 1 : 0, plan);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

}  // extern "C"
