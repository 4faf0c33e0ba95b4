// K1p -- the whole Sinkhorn solve of a SMALL point-cloud problem in ONE
// persistent cooperative kernel (one CTA per SM, grid-wide barriers between
// half-steps).  Replaces the reference loop sinkhorn._sinkhorn_iterations
// (reference sinkhorn.py:151-200) with apply_lse_kernel (geometry.py:336-354)
// for problems whose points fit in shared memory (BASELINE configs[0]:
// 2048^2, d = 3), where a launch per half-step costs more than the math.
//
// Every CTA keeps both point sets resident in shared memory as NV float4 per
// point: coordinates, then -kappa*|q|^2 in slot d, zeros after.  A half-step
// gives each warp R = 2 rows; a row's query vector p' = (2 kappa p, 1, 0..)
// turns one dot product into 2 kappa <p,q> - kappa |q|^2, clamped at
// kappa |p|^2 (C >= 0, geometry.py:273) and shifted by the column's
// kappa * potential.  Lanes stride the columns with an online log2-sum-exp2
// and merge in a fixed butterfly order: deterministic.
//
// The fused check (sinkhorn.py:175-189) runs inside the f_{t+1} half-step:
// r_i = a_i exp((f_t,i - f_{t+1},i)/eps); every CTA writes 8 partial sums,
// and after the barrier EVERY CTA adds all CTAs' slots in the same order, so
// all CTAs take the same converged / diverged decision (one more barrier
// keeps the first-bad marker stable while every CTA reads it).
// Constant-eps schedules only (the general loop is solve.cu).
#include <cooperative_groups.h>

#include <algorithm>

#include "otk_common.cuh"

namespace cg = cooperative_groups;

namespace otk {
namespace small {

constexpr int THREADS = 512;
constexpr int WARPS = THREADS / 32;
constexpr int R = 2;     // rows per warp (register reuse of every column load)
constexpr int CB = 8;    // columns per lane batch (online-update granularity)
constexpr int NVALS = 8;

struct Args {
  const float *x, *y, *a, *b, *la, *lb, *g_init;
  int n, m, d;
  float eps, kappa;          // float32 eps and kappa = log2(e)/eps
  double eps_d, threshold;
  int max_iters, inner_iters, max_checks;
  float *f0, *f1, *g, *bias_x, *bias_y, *f_out, *g_out;
  double *slots;             // [gridDim][8]
  int *first_bad;
  double *errors, *duals;    // [max_checks]
  int *state;                // n_checks, iterations, converged, status, fail_iter
  int probe;                 // timing probe (OTK_SMALL_PROBE): 1 = skip the half-step math
};

__device__ __forceinline__ void load_points(const float *src, int count, int d, float kappa,
                                            float4 *dst, int nv) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    double sq = 0.0;
    for (int k = 0; k < d; ++k) {
      const float c = src[(int64_t)i * d + k];
      v[k] = c;
      sq = fma((double)c, (double)c, sq);
    }
    v[d] = -kappa * (float)sq;
    dst[i * nv] = make_float4(v[0], v[1], v[2], v[3]);
    if (nv == 2) dst[i * nv + 1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

template <int NV>
__device__ __forceinline__ float dot_q(const float (&p)[4 * NV], const float4 *q) {
  float4 q0 = q[0];
  float acc = p[0] * q0.x;
  acc = fmaf(p[1], q0.y, acc);
  acc = fmaf(p[2], q0.z, acc);
  acc = fmaf(p[3], q0.w, acc);
  if (NV == 2) {
    float4 q1 = q[1];
    acc = fmaf(p[4], q1.x, acc);
    acc = fmaf(p[5], q1.y, acc);
    acc = fmaf(p[6], q1.z, acc);
    acc = fmaf(p[7], q1.w, acc);
  }
  return acc;
}

// One half-step over rows P (np) against columns Q (nq) whose kappa*potential
// is qbias (already in shared memory).  Writes out_pot = eps*logw - eps*ln2*L
// and out_bias = kappa*out_pot for the next half-step; bad outputs mark step.
// With CHECK, also accumulates the 8 check values of the rows handled here
// (f_prev = the previous f, a = weights).
//
// Work split: a CTA round covers PAIRS = WARPS/SL row pairs; the SL warps of
// a pair each take one contiguous slice of the columns (lanes stride it), so
// even a 2048-row problem keeps 16 warps per SM busy.  The slices' (max, sum)
// meet in shared memory and merge in slice order (deterministic).
constexpr int SL = 4;
constexpr int PAIRS = WARPS / SL;

template <int NV, bool SAME, bool CHECK, bool EU>
__device__ void half_step(const Args &A, const float4 *P, int np, const float4 *Q, int nq,
                          const float *qbias, const float *logw, float *out_pot, float *out_bias,
                          int step, const float *f_prev, double (&chk)[NVALS]) {
  __shared__ float part[PAIRS][R][SL][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pair = warp / SL, slice = warp % SL;
  const int per = (nq + SL - 1) / SL;
  const int c_lo = slice * per, c_hi = min(nq, c_lo + per);
  const float two_k = 2.f * A.kappa;
  const float sk = sqrtf(A.kappa);
  const int n_pairs = (A.probe == 1) ? 0 : (np + R - 1) / R;
  for (int base = blockIdx.x * PAIRS; base < n_pairs; base += gridDim.x * PAIRS) {
    const int r0 = (base + pair) * R;
    const bool live = r0 < np;
    float p[R][4 * NV], cp[R];
    float mx[R], sm[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = min(r0 + r, np - 1);
      const float *pv = reinterpret_cast<const float *>(P + i * NV);
#pragma unroll
      for (int k = 0; k < 4 * NV; ++k) p[r][k] = (k < A.d) ? two_k * pv[k] : (k == A.d ? 1.f : 0.f);
      cp[r] = -pv[A.d];  // kappa |p|^2
      mx[r] = -INFINITY;
      sm[r] = 0.f;
    }
    if (live) {
      for (int j0 = c_lo + lane; j0 < c_hi; j0 += 32 * CB) {
        float u[CB][R];
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          const int j = j0 + 32 * c;
          if (j < c_hi) {
            const float bj = qbias[j];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              float v;
              if (EU) {  // kappa sqrt(C) = sqrt(kappa) sqrt(kappa C), kappa C = cp - dot
                v = -sk * sqrt_approx(fmaxf(cp[r] - dot_q<NV>(p[r], Q + j * NV), 0.f));
                if (SAME && j == r0 + r) v = 0.f;
              } else {
                v = fminf(dot_q<NV>(p[r], Q + j * NV), cp[r]);
                if (SAME && j == r0 + r) v = cp[r];
              }
              u[c][r] = v + bj;
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) u[c][r] = -INFINITY;
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float cm = -INFINITY;
#pragma unroll
          for (int c = 0; c < CB; ++c) cm = fmaxf(cm, u[c][r]);
          if (cm > mx[r] + 8.f) {
            sm[r] *= ex2(mx[r] - cm);
            mx[r] = cm;
          }
          const float ms = (mx[r] == -INFINITY) ? 0.f : mx[r];
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < CB; ++c) acc += ex2(u[c][r] - ms);
          sm[r] += acc;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      Lse2 st;
      st.m = mx[r];
      st.s = sm[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, st.m, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, st.s, o);
        st.merge(m2, s2);
      }
      if (lane == 0) {
        part[pair][r][slice][0] = st.m;
        part[pair][r][slice][1] = st.s;
      }
    }
    __syncthreads();
    if (slice == 0 && lane < R) {
      const int r = lane, i = r0 + r;
      if (i < np) {
        Lse2 st;
        st.m = part[pair][r][0][0];
        st.s = part[pair][r][0][1];
#pragma unroll
        for (int q = 1; q < SL; ++q) st.merge(part[pair][r][q][0], part[pair][r][q][1]);
        const float L = st.value() - (EU ? 0.f : -reinterpret_cast<const float *>(P + i * NV)[A.d]);
        const float v = A.eps * logw[i] - A.eps * kLn2 * L;
        out_pot[i] = v;
        out_bias[i] = v * A.kappa;
        if (bad_potential(v)) atomicMin(A.first_bad, step);
        if (CHECK) {
          const double fp = f_prev[i], ai = A.a[i];
          const double rr = (ai > 0.0) ? ai * exp((fp - (double)v) / A.eps_d) : 0.0;
          chk[0] += fabs(rr - ai);
          chk[1] += rr;
          if (ai > 0.0) chk[2] += ai * fp;
          chk[4] += (fp != fp) ? 1.0 : 0.0;
          chk[6] += (fp == INFINITY) ? 1.0 : 0.0;
        }
      }
    }
    __syncthreads();
  }
}

__device__ void load_bias(float *dst, const float *src, int count) {
  for (int j = threadIdx.x; j < count; j += blockDim.x) dst[j] = src[j];
}

template <int NV, bool SAME, bool EU>
__global__ void __launch_bounds__(THREADS, 1) solve_small_kernel(Args A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ float4 sh4[];
  float4 *xs = sh4;
  float4 *ys = xs + A.n * NV;
  float *bias_s = reinterpret_cast<float *>(ys + A.m * NV);
  __shared__ double red[NVALS][WARPS];
  __shared__ double tot_s[NVALS];

  load_points(A.x, A.n, A.d, A.kappa, xs, NV);
  load_points(A.y, A.m, A.d, A.kappa, ys, NV);
  // initial g and its bias (h = 1 marks a bad warm start)
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.m; j += gridDim.x * blockDim.x) {
    const float g0 = A.g_init ? A.g_init[j] : 0.f;
    A.g[j] = g0;
    A.bias_y[j] = g0 * A.kappa;
    if (bad_potential(g0)) atomicMin(A.first_bad, 1);
  }
  __syncthreads();
  grid.sync();

  float *f = A.f0, *fn = A.f1;
  bool f_ready = false;
  int n_checks = 0, status = OTK_OK, fail_iter = 0, converged = 0, t;
  double chk[NVALS];
  for (t = 1; t <= A.max_iters; ++t) {
    if (!f_ready) {
      load_bias(bias_s, A.bias_y, A.m);
      __syncthreads();
      half_step<NV, SAME, false, EU>(A, xs, A.n, ys, A.m, bias_s, A.la, f, A.bias_x, 2 * t, nullptr, chk);
      grid.sync();
    }
    f_ready = false;
    load_bias(bias_s, A.bias_x, A.n);
    __syncthreads();
    half_step<NV, SAME, false, EU>(A, ys, A.m, xs, A.n, bias_s, A.lb, A.g, A.bias_y, 2 * t + 1, nullptr, chk);
    grid.sync();
    if (t % A.inner_iters == 0 || t == A.max_iters) {
      // f_{t+1} into fn, with the check of (f_t, g_t) fused in
#pragma unroll
      for (int k = 0; k < NVALS; ++k) chk[k] = 0.0;
      load_bias(bias_s, A.bias_y, A.m);
      __syncthreads();
      half_step<NV, SAME, true, EU>(A, xs, A.n, ys, A.m, bias_s, A.la, fn, A.bias_x, 2 * t + 2, f, chk);
      for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.m; j += gridDim.x * blockDim.x) {
        const double gj = A.g[j], bj = A.b[j];
        if (bj > 0.0) chk[3] += bj * gj;
        chk[5] += (gj != gj) ? 1.0 : 0.0;
        chk[7] += (gj == INFINITY) ? 1.0 : 0.0;
      }
      // fixed-order block reduction -> this CTA's slot
#pragma unroll
      for (int k = 0; k < NVALS; ++k) {
        double v = chk[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = v;
      }
      __syncthreads();
      if (threadIdx.x < NVALS) {
        double v = 0.0;
        for (int w = 0; w < WARPS; ++w) v += red[threadIdx.x][w];
        A.slots[blockIdx.x * NVALS + threadIdx.x] = v;
      }
      grid.sync();
      // every CTA reduces all slots in the same order -> identical decisions
      if (threadIdx.x < NVALS) {
        double v = 0.0;
        for (int bk = 0; bk < (int)gridDim.x; ++bk)
          v += reinterpret_cast<volatile double *>(A.slots)[bk * NVALS + threadIdx.x];
        tot_s[threadIdx.x] = v;
      }
      __syncthreads();
      const int fb = *reinterpret_cast<volatile int *>(A.first_bad);
      const double err = tot_s[0];
      // no CTA may mark first_bad again (next half-step) before all have read it
      grid.sync();
      if (fb <= 2 * t) {
        status = OTK_BAD_POTENTIAL;
        fail_iter = (fb + 1) / 2;
        break;
      }
      if (tot_s[4] > 0 || tot_s[5] > 0) {
        status = OTK_DIVERGED;
        fail_iter = t;
        break;
      }
      if (fb == 2 * t + 1) {
        status = OTK_BAD_POTENTIAL;
        fail_iter = t;
        break;
      }
      if (blockIdx.x == 0 && threadIdx.x == 0 && n_checks < A.max_checks) {
        A.errors[n_checks] = err;
        A.duals[n_checks] = tot_s[2] + tot_s[3] - A.eps_d * (tot_s[1] - 1.0);
      }
      ++n_checks;
      if (err <= A.threshold) {
        converged = 1;
        break;
      }
      if (t < A.max_iters) {
        float *tmp = f;
        f = fn;
        fn = tmp;
        f_ready = true;
      }
    }
  }
  // results (f = f_t of the last completed iteration, g = g_t)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x)
    A.f_out[i] = f[i];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.m; j += gridDim.x * blockDim.x)
    A.g_out[j] = A.g[j];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.state[0] = min(n_checks, A.max_checks);
    A.state[1] = min(t, A.max_iters);
    A.state[2] = converged;
    A.state[3] = status;
    A.state[4] = fail_iter;
  }
}

size_t smem_bytes(int n, int m, int nv) {
  return (size_t)(n + m) * nv * sizeof(float4) + (size_t)std::max(n, m) * sizeof(float);
}

}  // namespace small

// Can this problem run as one persistent kernel on this device?
bool small_solve_fits(int64_t n, int64_t m, int d) {
  if (d > 7 || n > (1 << 20) || m > (1 << 20)) return false;
  const int nv = (d + 1 + 3) / 4;
  int dev = 0, coop = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return coop && small::smem_bytes((int)n, (int)m, nv) + 4096 <= (size_t)max_smem;
}

int small_solve_launch(const small::Args &A, bool same, bool eucl, cudaStream_t st) {
  using namespace small;
  const int nv = (A.d + 1 + 3) / 4;
  const size_t smem = smem_bytes(A.n, A.m, nv);
  void *kern = nullptr;
  if (eucl) {
    if (nv == 1) kern = same ? (void *)solve_small_kernel<1, true, true> : (void *)solve_small_kernel<1, false, true>;
    else kern = same ? (void *)solve_small_kernel<2, true, true> : (void *)solve_small_kernel<2, false, true>;
  } else {
    if (nv == 1) kern = same ? (void *)solve_small_kernel<1, true, false> : (void *)solve_small_kernel<1, false, false>;
    else kern = same ? (void *)solve_small_kernel<2, true, false> : (void *)solve_small_kernel<2, false, false>;
  }
  OTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  OTK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
  if (per_sm < 1) {
    set_error("solve_small: kernel does not fit on an SM");
    return OTK_ENOTSUP;
  }
  Args args = A;
  void *params[] = {&args};
  OTK_CUDA(cudaLaunchCooperativeKernel(kern, dim3(num_sms()), dim3(THREADS), params, smem, st));
  return OTK_OK;
}

}  // namespace otk
