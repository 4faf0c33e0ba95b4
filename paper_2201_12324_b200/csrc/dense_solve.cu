// K3p -- many small stored-cost problems (BASELINE configs[2]: 512 x 512^2),
// each solved ENTIRELY by one CTA: the reference loop sinkhorn._sinkhorn_iterations
// (reference sinkhorn.py:151-200) over DenseGeometry.apply_lse_kernel
// (geometry.py:204-211) with its check (175-189) and _dual_objective (115-119),
// per problem, with no host round trip and no grid-wide synchronisation
// (problems are independent, so each CTA stops when ITS problem converges).
//
// A problem's potentials live in shared memory; its cost matrix (1 MiB at
// 512 x 512) is read from global memory once per half-step -- from L2 after
// the first touch as long as the problems in flight fit the 126 MB L2.
// Rows half-step: one warp per row, lanes stride the row with 128-bit loads,
// two rows per pass.  Columns half-step on the SAME row-major C: a warp owns
// 128 consecutive columns (a float4 per lane) for one group of rows and keeps
// a per-column online log2-sum-exp2; the row groups merge in fixed order.
// The fused check computes f_{t+1} and r_i = a_i exp((f_t - f_{t+1})/eps).
// Failure semantics follow the lock-step loop (sinkhorn._dense_loop): the
// first half-step to emit NaN/+inf is recorded by step number.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "otk_common.cuh"

namespace otk {
namespace dsolve {

#ifndef OTK_DENSE_THREADS
#define OTK_DENSE_THREADS 512
#endif
constexpr int THREADS = OTK_DENSE_THREADS, WARPS = THREADS / 32, NV = 8;

struct Args {
  const float *C;
  int64_t batch;
  int n, m;
  const float *a, *b, *la, *lb, *eps, *g_init;
  const double *eps_d;
  double threshold;
  int max_iters, inner_iters, max_checks;
  float *f_out, *g_out;
  double *errors, *duals;
  int *state;  // [B][5]: n_checks, iterations, converged, status, fail_iter
  unsigned long long *trace;  // OTK_DENSE_TRACE (trace builds): globaltimer stamps of cluster 0's first problem
};

__device__ __forceinline__ void dtrace(const Args &A, bool on, int t, int k) {
#ifdef OTK_DENSE_TRACE_BUILD  // tools/build_variant.sh ... -DOTK_DENSE_TRACE_BUILD
  if (on && A.trace && threadIdx.x == 0 && t < 64) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    A.trace[t * 8 + k] = v;
  }
#endif
}

__device__ __forceinline__ void block_sum(double (&v)[NV], double *red /* [NV][WARPS] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[k * WARPS + warp] = x;
  }
  __syncthreads();
  if (warp < NV) {  // warp k folds value k over the warps in a fixed shuffle tree
    static_assert(WARPS <= 32, "one lane per warp");
    double x = (lane < WARPS) ? red[warp * WARPS + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp * WARPS] = x;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = red[k * WARPS];
}

// rows half-step: out_i = eps log w_i - eps ln2 LSE2_j(by_j - kappa C_ij); bx_i = kappa out_i
template <bool CHECK>
__device__ void rows_half(const float *__restrict__ Cb, int n, int m, const float *by, const float *lw,
                          float eps, float kappa, float *out, float *bx, int *fbad, int step,
                          const float *fprev, const float *a, double eps_d, double (&chk)[NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i0 = warp * 2; i0 < n; i0 += WARPS * 2) {
    Lse2 st[2];
    st[0].init();
    st[1].init();
    for (int j0 = 0; j0 < m; j0 += 512) {
      float4 c4[2][4];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = j0 + (q * 32 + lane) * 4;
          const int i = min(i0 + r, n - 1);
          c4[r][q] = (j < m) ? __ldg(reinterpret_cast<const float4 *>(Cb + (int64_t)i * m + j))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        float u[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = j0 + (q * 32 + lane) * 4;
          if (j < m) {
            const float4 h = *reinterpret_cast<const float4 *>(by + j);
            u[4 * q + 0] = fmaf(-kappa, c4[r][q].x, h.x);
            u[4 * q + 1] = fmaf(-kappa, c4[r][q].y, h.y);
            u[4 * q + 2] = fmaf(-kappa, c4[r][q].z, h.z);
            u[4 * q + 3] = fmaf(-kappa, c4[r][q].w, h.w);
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) u[4 * q + e] = -INFINITY;
          }
        }
        float cm = -INFINITY;
#pragma unroll
        for (int e = 0; e < 16; ++e) cm = fmaxf(cm, u[e]);
        if (cm > st[r].m) {
          st[r].s *= ex2(st[r].m - cm);
          st[r].m = cm;
        }
        const float ms = (st[r].m == -INFINITY) ? 0.f : st[r].m;
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < 16; ++e) acc += ex2(u[e] - ms);
        st[r].s += acc;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, st[r].m, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, st[r].s, o);
        st[r].merge(m2, s2);
      }
      const int i = i0 + r;
      if (lane == 0 && i < n) {
        const float lwi = lw[i], Lr = st[r].value();
        const float v = eps * lwi - eps * kLn2 * Lr;
        out[i] = v;
        bx[i] = next_bias(lwi, Lr, eps, kappa);
        if (bad_potential(v)) atomicMin(fbad, step);
        if (CHECK) {
          const double fp = fprev[i], ai = a[i];
          const double rr = (ai > 0.0) ? ai * exp((fp - (double)v) / eps_d) : 0.0;
          chk[0] += fabs(rr - ai);
          chk[1] += rr;
          if (ai > 0.0) chk[2] += ai * fp;
          chk[4] += (fp != fp) ? 1.0 : 0.0;
          chk[6] += (fp == INFINITY) ? 1.0 : 0.0;
        }
      }
    }
  }
}

// columns half-step on row-major C: out_j = eps log b_j - eps ln2 LSE2_i(bx_i - kappa C_ij)
__device__ void cols_half(const float *__restrict__ Cb, int n, int m, const float *bx, const float *lw,
                          float eps, float kappa, float *out, float *by, int *fbad, int step,
                          float *part /* [groups x block columns][2] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int cb0 = 0; cb0 < m; cb0 += 512) {          // column block of up to 512 columns
    const int ncols = min(512, m - cb0);
    const int cwarps = (ncols + 127) / 128;          // warps per row group
    const int groups = WARPS / cwarps;               // row groups
    const int cw = warp % cwarps, rg = warp / cwarps;
    const int j = cb0 + cw * 128 + lane * 4;         // this lane's 4 columns
    const bool active = rg < groups && j < m;
    float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, sm[4] = {0.f, 0.f, 0.f, 0.f};
    if (active) {
      const int rows_per = (n + groups - 1) / groups;
      const int r0 = rg * rows_per, r1 = min(n, r0 + rows_per);
      for (int i = r0; i < r1; i += 8) {
        float4 c[8];
        float h[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int ii = min(i + k, r1 - 1);
          c[k] = __ldg(reinterpret_cast<const float4 *>(Cb + (int64_t)ii * m + j));
          h[k] = (i + k < r1) ? bx[ii] : -INFINITY;
        }
        float u[4][8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          u[0][k] = fmaf(-kappa, c[k].x, h[k]);
          u[1][k] = fmaf(-kappa, c[k].y, h[k]);
          u[2][k] = fmaf(-kappa, c[k].z, h[k]);
          u[3][k] = fmaf(-kappa, c[k].w, h[k]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float cm = -INFINITY;
#pragma unroll
          for (int k = 0; k < 8; ++k) cm = fmaxf(cm, u[e][k]);
          if (cm > mx[e]) {
            sm[e] *= ex2(mx[e] - cm);
            mx[e] = cm;
          }
          const float ms = (mx[e] == -INFINITY) ? 0.f : mx[e];
          float acc = 0.f;
#pragma unroll
          for (int k = 0; k < 8; ++k) acc += ex2(u[e][k] - ms);
          sm[e] += acc;
        }
      }
    }
    const int pstride = cwarps * 128;  // groups * pstride <= WARPS * 128
    if (rg < groups) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int jj = cw * 128 + lane * 4 + e;
        part[(rg * pstride + jj) * 2] = mx[e];
        part[(rg * pstride + jj) * 2 + 1] = sm[e];
      }
    }
    __syncthreads();
    for (int jj = threadIdx.x; jj < ncols; jj += THREADS) {
      Lse2 st;
      st.m = part[jj * 2];
      st.s = part[jj * 2 + 1];
      for (int g = 1; g < groups; ++g)
        st.merge(part[(g * pstride + jj) * 2], part[(g * pstride + jj) * 2 + 1]);
      const int jg = cb0 + jj;
      const float lwj = lw[jg], Lc = st.value();
      const float v = eps * lwj - eps * kLn2 * Lc;
      out[jg] = v;
      by[jg] = next_bias(lwj, Lc, eps, kappa);
      if (bad_potential(v)) atomicMin(fbad, step);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(THREADS, 1) dense_solve_kernel(Args A) {
  extern __shared__ __align__(16) float sh[];
  const int n = A.n, m = A.m;
  const int n4 = (n + 3) & ~3, m4 = (m + 3) & ~3;  // 16-byte aligned segments
  float *f0 = sh, *f1 = f0 + n4, *g = f1 + n4, *bx = g + m4, *by = bx + n4;
  float *part = by + m4;  // [row groups][<= 2048 columns total][2]
  __shared__ double red[NV * WARPS];
  __shared__ int fbad, decide;
  __shared__ double tot[NV];
  for (int64_t b = blockIdx.x; b < A.batch; b += gridDim.x) {
    const float *Cb = A.C + b * (int64_t)n * m;
    const float *a = A.a + b * n, *bw = A.b + b * m;
    const float *la = A.la + b * n, *lb = A.lb + b * m;
    const float eps = A.eps[b];
    const double eps_d = A.eps_d[b];
    const float kappa = kLog2e / eps;
    if (threadIdx.x == 0) fbad = 0x7fffffff;
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += THREADS) {
      const float g0 = A.g_init ? A.g_init[b * m + j] : 0.f;
      g[j] = g0;
      by[j] = g0 * kappa;
      if (bad_potential(g0)) atomicMin(&fbad, 1);
    }
    __syncthreads();
    float *f = f0, *fn = f1;
    bool f_ready = false;
    int n_checks = 0, status = OTK_OK, fail_iter = 0, converged = 0, t;
    double chk[NV];
    for (t = 1; t <= A.max_iters; ++t) {
      if (!f_ready) {
        rows_half<false>(Cb, n, m, by, la, eps, kappa, f, bx, &fbad, 2 * t, nullptr, a, eps_d, chk);
        __syncthreads();
      }
      f_ready = false;
      cols_half(Cb, n, m, bx, lb, eps, kappa, g, by, &fbad, 2 * t + 1, part);  // ends synced
      if (t % A.inner_iters == 0 || t == A.max_iters) {
#pragma unroll
        for (int k = 0; k < NV; ++k) chk[k] = 0.0;
        rows_half<true>(Cb, n, m, by, la, eps, kappa, fn, bx, &fbad, 2 * t + 2, f, a, eps_d, chk);
        for (int j = threadIdx.x; j < m; j += THREADS) {
          const double gj = g[j], bj = bw[j];
          if (bj > 0.0) chk[3] += bj * gj;
          chk[5] += (gj != gj) ? 1.0 : 0.0;
          chk[7] += (gj == INFINITY) ? 1.0 : 0.0;
        }
        block_sum(chk, red);  // contains a __syncthreads: fbad is final for this check
        if (threadIdx.x == 0) {
          int d = 0;  // 0 continue, 1 converged, 2 bad potential, 3 diverged
          if (fbad <= 2 * t) {
            d = 2;
            fail_iter = (fbad + 1) / 2;
          } else if (chk[4] > 0 || chk[5] > 0) {
            d = 3;
            fail_iter = t;
          } else if (fbad == 2 * t + 1) {
            d = 2;
            fail_iter = t;
          } else {
            if (n_checks < A.max_checks) {
              A.errors[b * A.max_checks + n_checks] = chk[0];
              A.duals[b * A.max_checks + n_checks] = chk[2] + chk[3] - eps_d * (chk[1] - 1.0);
            }
            if (chk[0] <= A.threshold) d = 1;
          }
          decide = d;
          tot[0] = (double)fail_iter;
        }
        __syncthreads();
        const int d = decide;
        if (d == 2 || d == 3) {
          status = (d == 2) ? OTK_BAD_POTENTIAL : OTK_DIVERGED;
          fail_iter = (int)tot[0];
          break;
        }
        ++n_checks;
        if (d == 1) {
          converged = 1;
          break;
        }
        if (t < A.max_iters) {
          float *tmp = f;
          f = fn;
          fn = tmp;
          f_ready = true;
        }
        __syncthreads();  // decide / tot / red reused by the next check
      }
    }
    for (int i = threadIdx.x; i < n; i += THREADS) A.f_out[b * n + i] = f[i];
    for (int j = threadIdx.x; j < m; j += THREADS) A.g_out[b * m + j] = g[j];
    if (threadIdx.x == 0) {
      int *s = A.state + b * 5;
      s[0] = min(n_checks, A.max_checks);
      s[1] = min(t, A.max_iters);
      s[2] = converged;
      s[3] = status;
      s[4] = fail_iter;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K3c
// The same per-problem loop with the problem's cost RESIDENT ON CHIP: a
// cluster of CL CTAs owns one problem at a time, each CTA keeping a slice of
// ceil(n / CL) rows of C (cfg3, CL = 6: 86 rows x 512 columns = 172 KB) in
// shared memory, loaded once per problem with bulk copies.  C is then read
// from HBM once per solve instead of once per half-step, and the loop is
// bound by the exps (MUFU), not HBM.
//   rows half-step: local (each CTA finalizes its own rows; g replicated),
//     RG threads per row with RG chosen per pass (rows_pass); an anchored
//     rows pass measured 2 % slower here (the pass is bound by the MIO queue
//     that LDS and MUFU share, not by the max / rescale instructions)
//   cols half-step: every CTA reduces its rows into one log2 partial per
//     column (anchored on its previous partial of that column), pushes it
//     into slot `rank` of EVERY CTA's shared memory (remote stores, parity
//     double-buffered), one cluster barrier, then every CTA combines the CL
//     partials of every column from its own shared memory in rank order ->
//     g is computed identically (bitwise) in every CTA of the cluster
//   check: per-CTA sums (the g terms counted by rank 0 only) and the
//     first-bad step are published the same way and reduced in rank order,
//     so every CTA takes the same decision at the same iteration.
// Parity buffers make one barrier per exchange enough: a CTA rewrites a
// parity buffer only after passing the NEXT exchange's barrier, which every
// reader of the previous use has reached after reading.

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}

// Cluster-scope push of one float into a peer CTA's shared memory that also
// counts its 4 bytes on the peer's mbarrier (st.async ... complete_tx): the
// receiver waits on its own barrier -- no cluster-wide barrier and none of the
// GPU-scope fences a release-arrive emits (measured: MEMBAR.ALL.GPU + ERRBAR
// at the column exchange's cluster.sync took ~25 % of K3c's stall samples).
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f32(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(__float_as_uint(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

// Rows half-step on the CTA's resident rows [rb, re): a group of RG (8, 16
// or 32) threads per row (each LDS.128 phase of 8 threads reads 128
// consecutive bytes of one row: no bank conflicts), each thread streaming
// every RG-th float4 of the row with an online (max, sum), then a log2(RG)-level
// shuffle merge in fixed order.  rows_pass picks RG per pass so that a CTA's
// last, partial pass still keeps most threads busy.

// 2^x for x <= 0 on the FMA pipe (two values per packed op): round-to-nearest
// split x = n + f, |f| <= 1/2, degree-5 minimax polynomial for 2^f (relative
// error 2.3e-7 in float32, the class of ex2.approx), 2^n added to the exponent
// bits; x < -125 flushes to 0 like ex2.approx.ftz.  Relieves the MIO queue
// that MUFU shares with the shared-memory loads (K3c's rows pass).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 t = __fadd2_rn(x, magic);
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 p = make_float2(0.001327647129073739f, 0.001327647129073739f);
  p = __ffma2_rn(p, f, make_float2(0.009675540961325169f, 0.009675540961325169f));
  p = __ffma2_rn(p, f, make_float2(0.05550713092088699f, 0.05550713092088699f));
  p = __ffma2_rn(p, f, make_float2(0.24022120237350464f, 0.24022120237350464f));
  p = __ffma2_rn(p, f, make_float2(0.6931469440460205f, 0.6931469440460205f));
  p = __ffma2_rn(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  const int nx = __float_as_int(t.x) - 0x4B400000, ny = __float_as_int(t.y) - 0x4B400000;
  const float vx = __int_as_float(__float_as_int(p.x) + (nx << 23));
  const float vy = __int_as_float(__float_as_int(p.y) + (ny << 23));
  return make_float2(x.x < -125.f ? 0.f : vx, x.y < -125.f ? 0.f : vy);
}

#ifndef OTK_K3C_NPOLY
#define OTK_K3C_NPOLY 0  // value pairs per 16 that take the FMA-pipe exp2 (A/B knob)
#endif

// sum_e 2^(u_e - ms) over 16 values in two chains (even / odd e), as packed
// FADD2 pairs: bitwise the scalar (a0 += ..even.., a1 += ..odd..; a0 + a1)
template <int NPOLY = 0>
__device__ __forceinline__ float sum_ex2_16(const float (&u)[16], float ms) {
  float2 acc = make_float2(0.f, 0.f);
  const float2 nms = make_float2(-ms, -ms);
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    const float2 t = __fadd2_rn(make_float2(u[e], u[e + 1]), nms);
    if (e / 2 < NPOLY) acc = __fadd2_rn(acc, ex2_poly2(t));
    else acc = __fadd2_rn(acc, make_float2(ex2(t.x), ex2(t.y)));
  }
  return acc.x + acc.y;
}
// ---- anchored passes (K3c).  Sinkhorn hands every row (column partial) a
// good shift for free: the same row's log2 result of the previous half-step
// of its role, A_i.  The anchored pass sums 2^(u_ij - A_i) directly -- no
// running max, no compare, no rescale -- and accepts the row when A_i was
// finite and lo <= L_i - A_i <= 120 (every term within 2^-30 of the row's
// sum stayed above the ex2 flush threshold, nothing overflowed; lo = -96 +
// 2 log2(#terms)) or when L_i is NaN (propagates like the running max); any
// other row is redone at once with the running max by the same threads
// (same rule as the tcgen05 kernel's anchored half-step, lse_tc.cu).
__device__ __forceinline__ bool anchor_ok(float L, float A, float lo) {
  const float dd = L - A;
  return (L != L) || (dd >= lo && dd <= 120.f);
}
__device__ __forceinline__ float nan_if_not_finite(float L) {
  return isfinite(L) ? L : __int_as_float(0x7fc00000);
}

template <bool CHECK, int RG>
__device__ void rows_local(const float *Cs, int rb, int re, int m, const float *by, const float *lw,
                           float eps, float kappa, float *out, float *bx, int *fbad, int step,
                           const float *fprev, const float *a, double eps_d, double (&chk)[NV]) {
  constexpr int RCH = 4 * RG * 4;  // columns per chunk
  const int gi = threadIdx.x / RG, gl = threadIdx.x % RG;
  constexpr int GROUPS = THREADS / RG;
  const float2 nk = make_float2(-kappa, -kappa);
  for (int i0 = rb; i0 < re; i0 += GROUPS) {
    const int i = i0 + gi;
    Lse2 st;
    st.init();
    if (i < re) {
      const float *row = Cs + (int64_t)i * m;
      for (int j0 = gl * 4; j0 < m; j0 += RCH) {  // 4 float4 per chunk
        float u[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = j0 + q * 4 * RG;
          if (j < m) {
            const float4 c = *reinterpret_cast<const float4 *>(row + j);
            const float4 h = *reinterpret_cast<const float4 *>(by + j);
            // packed FFMA2: the same IEEE results as four scalar FFMAs
            const float2 u01 = __ffma2_rn(nk, make_float2(c.x, c.y), make_float2(h.x, h.y));
            const float2 u23 = __ffma2_rn(nk, make_float2(c.z, c.w), make_float2(h.z, h.w));
            u[4 * q + 0] = u01.x;
            u[4 * q + 1] = u01.y;
            u[4 * q + 2] = u23.x;
            u[4 * q + 3] = u23.y;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) u[4 * q + e] = -INFINITY;
          }
        }
        float cm = -INFINITY;
#pragma unroll
        for (int e = 0; e < 16; ++e) cm = fmaxf(cm, u[e]);
        if (cm > st.m) {
          st.s *= ex2(st.m - cm);
          st.m = cm;
        }
        const float ms = (st.m == -INFINITY) ? 0.f : st.m;
        st.s += sum_ex2_16<OTK_K3C_NPOLY>(u, ms);
      }
    }
#pragma unroll
    for (int o = RG / 2; o > 0; o >>= 1) {  // within the row's group of RG lanes
      const float m2 = __shfl_xor_sync(0xffffffffu, st.m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, st.s, o);
      st.merge(m2, s2);
    }
    if (gl == 0 && i < re) {
      const float lwi = lw[i], Lr = st.value();
      const float v = eps * lwi - eps * kLn2 * Lr;
      out[i] = v;
      bx[i] = next_bias(lwi, Lr, eps, kappa);
      if (bad_potential(v)) atomicMin(fbad, step);
      if (CHECK) {
        const double fp = fprev[i], ai = a[i];
        const double rr = (ai > 0.0) ? ai * exp((fp - (double)v) / eps_d) : 0.0;
        chk[0] += fabs(rr - ai);
        chk[1] += rr;
        if (ai > 0.0) chk[2] += ai * fp;
        chk[4] += (fp != fp) ? 1.0 : 0.0;
        chk[6] += (fp == INFINITY) ? 1.0 : 0.0;
      }
    }
  }
}

// This CTA's log2 partial of column j over its rows, anchored on the same
// column's partial of the previous column half-step (canc[j], NaN = none),
// running max as the fallback.  Returns L (the caller publishes it).
__device__ __forceinline__ float col_partial_anchored(const float *Cs, int rows, int m, const float *bx,
                                                      float kappa, int j, float A, float lo) {
  const float *cp = Cs + j;
  if (isfinite(A)) {
    float2 acc = make_float2(0.f, 0.f);
    const float2 nk = make_float2(-kappa, -kappa), nA = make_float2(-A, -A);
    int i0 = 0;
    for (; i0 + 16 <= rows; i0 += 16) {
      float hb[16];
#pragma unroll
      for (int k = 0; k < 16; k += 4) {
        const float4 hh = *reinterpret_cast<const float4 *>(bx + i0 + k);
        hb[k] = hh.x;
        hb[k + 1] = hh.y;
        hb[k + 2] = hh.z;
        hb[k + 3] = hh.w;
      }
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        const float2 x = __fadd2_rn(__ffma2_rn(nk, make_float2(cp[(i0 + k) * m], cp[(i0 + k + 1) * m]),
                                               make_float2(hb[k], hb[k + 1])), nA);
        acc = __fadd2_rn(acc, make_float2(ex2(x.x), ex2(x.y)));
      }
    }
    if (i0 < rows) {  // last partial chunk, masked (-inf terms add 0)
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        const float x0 = (i0 + k < rows) ? fmaf(-kappa, cp[(i0 + k) * m], bx[i0 + k]) - A : -INFINITY;
        const float x1 = (i0 + k + 1 < rows) ? fmaf(-kappa, cp[(i0 + k + 1) * m], bx[i0 + k + 1]) - A : -INFINITY;
        acc = __fadd2_rn(acc, make_float2(ex2(x0), ex2(x1)));
      }
    }
    const float sm = acc.x + acc.y;
    const float L = (sm > 0.f) ? A + lg2(sm) : ((sm != sm) ? sm : -INFINITY);
    if (anchor_ok(L, A, lo)) return L;
  }
  float mx = -INFINITY, sm = 0.f;
  for (int i0 = 0; i0 < rows; i0 += 16) {
    float u[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) u[k] = (i0 + k < rows) ? fmaf(-kappa, cp[(i0 + k) * m], bx[i0 + k]) : -INFINITY;
    float cm = -INFINITY;
#pragma unroll
    for (int k = 0; k < 16; ++k) cm = fmaxf(cm, u[k]);
    if (cm > mx) {
      sm *= ex2(mx - cm);
      mx = cm;
    }
    const float ms = (mx == -INFINITY) ? 0.f : mx;
    sm += sum_ex2_16(u, ms);
  }
  Lse2 st;
  st.m = mx;
  st.s = sm;
  return st.value();
}



// ---- K3c in the scaling domain (the default) -------------------------------
// Sinkhorn's half-steps are LSEs of u_ij = b_j - kappa C_ij (rows) or
// f'_i - kappa C_ij (columns).  With the cost resident on chip, the exps can
// be taken ONCE into a stabilised kernel K_ij = 2^(beta_j - kappa C_ij - rho_i)
// (beta_j: the column potentials kappa*g_j at build time, rho_i: the row max,
// so 0 < K_ij <= 1, flushed below 2^-126 of its row's max) and every later
// half-step is a matrix-vector product in FP32 FMAs (Schmitzer's absorption,
// in log2 units):
//   rows:    L_i = rho_i + log2 sum_j K_ij v_j,          v_j = 2^(b_j - beta_j)
//   columns: P_j = -beta_j + log2 sum_{i in CTA} K_ij w_i, w_i = 2^(kappa f'_i + rho_i)
// -- one FMA and 4 B of shared memory per cell instead of one MUFU ex2 (and
// the max / rescale work around it).  Exactness guards: the kernel slice is
// rebuilt from the cost (kept in global memory, L2-resident) whenever a
// column potential drifted more than kDrift bits from its beta (v stays in
// [2^-40, 2^40], so no term that mattered can have been flushed), and a column
// partial whose FMA sum leaves [2^-90, 2^120] -- a column far from every row
// of the slice, a dead (zero-weight) column, overflow -- is recomputed exactly
// in the log domain from the global cost.  Results match the log-domain
// passes to float32 rounding (tests: K3c vs K3p, the reference fixtures).
constexpr float kDrift = 40.f;

// This CTA's kernel slice from its global cost rows Cg [rows][m]:
// beta_j = by_j, rho_i = max_j (beta_j - kappa C_ij), K_ij = 2^(.. - rho_i).
__device__ void build_kernel(const float *__restrict__ Cg, int rows, int m, const float *by,
                             float kappa, float *Ks, float *beta, float *rho) {
  for (int j = threadIdx.x; j < m; j += THREADS) beta[j] = by[j];
  __syncthreads();
  constexpr int RGB = 8, GROUPS = THREADS / RGB, RCH = 4 * RGB;
  const int gi = threadIdx.x / RGB, gl = threadIdx.x % RGB;
  for (int i0 = 0; i0 < rows; i0 += GROUPS) {
    const int i = i0 + gi;
    const bool live = i < rows;
    const float *crow = Cg + (int64_t)(live ? i : 0) * m;
    float mx = -INFINITY;
    if (live) {
      for (int j = gl * 4; j < m; j += RCH) {
        const float4 c = __ldg(reinterpret_cast<const float4 *>(crow + j));
        const float4 bb = *reinterpret_cast<const float4 *>(beta + j);
        mx = fmaxf(mx, fmaxf(fmaxf(fmaf(-kappa, c.x, bb.x), fmaf(-kappa, c.y, bb.y)),
                             fmaxf(fmaf(-kappa, c.z, bb.z), fmaf(-kappa, c.w, bb.w))));
      }
    }
#pragma unroll
    for (int o = RGB / 2; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (live) {
      const bool dead = !(mx > -INFINITY);  // every term -inf (or NaN): an all-zero row
      float *krow = Ks + (int64_t)i * m;
      for (int j = gl * 4; j < m; j += RCH) {
        const float4 c = __ldg(reinterpret_cast<const float4 *>(crow + j));
        const float4 bb = *reinterpret_cast<const float4 *>(beta + j);
        float4 k;
        k.x = dead ? 0.f : ex2(fmaf(-kappa, c.x, bb.x) - mx);
        k.y = dead ? 0.f : ex2(fmaf(-kappa, c.y, bb.y) - mx);
        k.z = dead ? 0.f : ex2(fmaf(-kappa, c.z, bb.z) - mx);
        k.w = dead ? 0.f : ex2(fmaf(-kappa, c.w, bb.w) - mx);
        *reinterpret_cast<float4 *>(krow + j) = k;
      }
      if (gl == 0) rho[i] = dead ? -INFINITY : mx;
    }
  }
  __syncthreads();
}

// v_j = 2^(by_j - beta_j) and the kernel rebuild decision: drift of a finite
// column potential beyond kDrift bits from its beta (the caller rebuilds and
// calls again).  Returns true when v is ready.
#ifdef OTK_DENSE_TRACE_BUILD
__device__ unsigned long long g_dense_rebuilds, g_dense_fallbacks;  // diagnostics (trace builds)
#endif
__device__ bool scaled_v(const float *by, const float *beta, int m, float *vv, int *flag) {
  if (threadIdx.x == 0) *flag = 0;
  __syncthreads();
  bool drift = false;
  for (int j = threadIdx.x; j < m; j += THREADS) {
    const float bt = beta[j], b = by[j];
    const float dlt = b - bt;
    if (bt > -INFINITY && fabsf(dlt) > kDrift && isfinite(dlt)) drift = true;
    vv[j] = (bt > -INFINITY) ? ex2(dlt) : 0.f;
  }
  if (__syncthreads_or(drift)) {
#ifdef OTK_DENSE_TRACE_BUILD
    if (threadIdx.x == 0) atomicAdd(&g_dense_rebuilds, 1ull);
#endif
    return false;
  }
  return true;
}

// Rows half-step as K v: one warp per row, FOUR rows in flight (rows w,
// w + WARPS, w + 2 WARPS, w + 3 WARPS, then the next four): the warp's v values
// (lane l: columns 4l + 128q, m <= 512) are loaded once per pass and kept in
// registers, so shared memory carries only K (4 B per cell); the four rows'
// partial sums leave the warp through a reduce-scatter (6 shuffles for the
// four rows instead of 20: xor 16 and xor 8 halve the rows per lane, then a
// 3-level sum) and lanes 0, 8, 16, 24 finalize one row each.  The check's
// per-row terms (a float64 exp per row) run afterwards, one thread per row.
template <bool CHECK>
__device__ void rows_pass_scaled(const float *Ks, int rows, int m, const float *vv, const float *rho,
                                 const float *lw, float eps, float kappa, float *out, float *bx,
                                 float *uw, int *fbad, int step, const float *fprev, const float *a,
                                 double eps_d, double (&chk)[NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4 v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = q * 128 + lane * 4;
    v[q] = (j < m) ? *reinterpret_cast<const float4 *>(vv + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int i0 = warp; i0 < rows; i0 += 4 * WARPS) {
    float r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k * WARPS;
      const float *kr = Ks + (int64_t)(i < rows ? i : i0) * m;
      float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = q * 128 + lane * 4;
        if (j < m) {
          const float4 x = *reinterpret_cast<const float4 *>(kr + j);
          a0 = __ffma2_rn(make_float2(x.x, x.y), make_float2(v[q].x, v[q].y), a0);
          a1 = __ffma2_rn(make_float2(x.z, x.w), make_float2(v[q].z, v[q].w), a1);
        }
      }
      const float2 s2 = __fadd2_rn(a0, a1);
      r[k] = s2.x + s2.y;
    }
    // reduce-scatter: after xor 16 lane bit 4 selects rows {0,1} / {2,3}, after
    // xor 8 lane bit 3 selects the row within the pair (fixed tree, deterministic)
    const bool hi16 = lane & 16, hi8 = lane & 8;
    float p0 = hi16 ? r[2] : r[0], p1 = hi16 ? r[3] : r[1];
    const float q0 = hi16 ? r[0] : r[2], q1 = hi16 ? r[1] : r[3];
    p0 += __shfl_xor_sync(0xffffffffu, q0, 16);
    p1 += __shfl_xor_sync(0xffffffffu, q1, 16);
    float t = hi8 ? p1 : p0;
    t += __shfl_xor_sync(0xffffffffu, hi8 ? p0 : p1, 8);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    const int k = (hi16 ? 2 : 0) + (hi8 ? 1 : 0);
    const int i = i0 + k * WARPS;
    if ((lane & 7) == 0 && i < rows) {
      const float rh = rho[i];
      const float L = rh + ((t > 0.f) ? lg2(t) : ((t != t) ? t : -INFINITY));
      const float lwi = lw[i];
      const float v_ = eps * lwi - eps * kLn2 * L;
      const float bq = next_bias(lwi, L, eps, kappa);
      out[i] = v_;
      bx[i] = bq;
      uw[i] = (rh > -INFINITY) ? ex2(bq + rh) : 0.f;
      if (bad_potential(v_)) atomicMin(fbad, step);
    }
  }
  if (CHECK) {
    __syncthreads();
    for (int i = threadIdx.x; i < rows; i += THREADS) {
      const double fp = fprev[i], ai = a[i];
      const double rr = (ai > 0.0) ? ai * exp((fp - (double)out[i]) / eps_d) : 0.0;
      chk[0] += fabs(rr - ai);
      chk[1] += rr;
      if (ai > 0.0) chk[2] += ai * fp;
      chk[4] += (fp != fp) ? 1.0 : 0.0;
      chk[6] += (fp == INFINITY) ? 1.0 : 0.0;
    }
  }
}

// This CTA's log2 partial of column j: -beta_j + log2 sum_i K_ij w_i, or the
// exact log-domain partial from the global cost when the FMA sum left its
// safe range (far / dead column, overflow).
__device__ __forceinline__ float col_partial_scaled(const float *Ks, const float *__restrict__ Cg, int rows,
                                                    int m, const float *bx, const float *uw,
                                                    const float *beta, float kappa, int j) {
  const float *kp = Ks + j;
  // four independent FFMA2 chains over 16-row chunks (the K loads of a chunk
  // are issued before its FMAs)
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                   make_float2(0.f, 0.f)};
  int i0 = 0;
  for (; i0 + 16 <= rows; i0 += 16) {
    float wb[16], kb[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) kb[k] = kp[(i0 + k) * m];
#pragma unroll
    for (int k = 0; k < 16; k += 4) {
      const float4 ww = *reinterpret_cast<const float4 *>(uw + i0 + k);
      wb[k] = ww.x;
      wb[k + 1] = ww.y;
      wb[k + 2] = ww.z;
      wb[k + 3] = ww.w;
    }
#pragma unroll
    for (int k = 0; k < 16; k += 2)
      acc[(k / 2) & 3] = __ffma2_rn(make_float2(kb[k], kb[k + 1]), make_float2(wb[k], wb[k + 1]), acc[(k / 2) & 3]);
  }
  for (; i0 < rows; ++i0) acc[0].x = fmaf(kp[i0 * m], uw[i0], acc[0].x);
  const float2 a01 = __fadd2_rn(acc[0], acc[1]), a23 = __fadd2_rn(acc[2], acc[3]);
  const float2 a4 = __fadd2_rn(a01, a23);
  const float sm = a4.x + a4.y;
  const float bt = beta[j];
  if (sm != sm) return sm;
  if (bt > -INFINITY && sm >= 0x1p-90f && sm <= 0x1p120f) return lg2(sm) - bt;
#ifdef OTK_DENSE_TRACE_BUILD
  atomicAdd(&g_dense_fallbacks, 1ull);
#endif
  // exact: running max over this CTA's rows of kappa f'_i - kappa C_ij (global cost)
  float mx = -INFINITY, s = 0.f;
  for (int i = 0; i < rows; ++i) {
    const float u = fmaf(-kappa, __ldg(Cg + (int64_t)i * m + j), bx[i]);
    if (u > mx) {
      s = (mx == -INFINITY) ? 0.f : s * ex2(mx - u);
      mx = u;
    }
    if (mx > -INFINITY) s += ex2(u - mx);
  }
  Lse2 st;
  st.m = mx;
  st.s = s;
  return st.value();
}

// Rows pass of K3c: full passes of 64 rows with 8 threads per row, then the
// remaining R rows with 8 (R > 32), 16 (R > 16) or 32 threads per row, so a
// slice of 86 rows (cfg3, CL = 6) costs 64 + 32 cells per thread instead of
// 2 x 64.
template <bool CHECK>
__device__ __forceinline__ void rows_pass(const float *Cs, int rows, int m, const float *by, const float *lw,
                                          float eps, float kappa, float *out, float *bx, int *fbad,
                                          int step, const float *fprev, const float *a, double eps_d,
                                          double (&chk)[NV]) {
  const int full = (rows / 64) * 64, rem = rows - full;
  if (full > 0) rows_local<CHECK, 8>(Cs, 0, full, m, by, lw, eps, kappa, out, bx, fbad, step, fprev, a, eps_d, chk);
  if (rem > 32) rows_local<CHECK, 8>(Cs, full, rows, m, by, lw, eps, kappa, out, bx, fbad, step, fprev, a, eps_d, chk);
  else if (rem > 16) rows_local<CHECK, 16>(Cs, full, rows, m, by, lw, eps, kappa, out, bx, fbad, step, fprev, a, eps_d, chk);
  else if (rem > 0) rows_local<CHECK, 32>(Cs, full, rows, m, by, lw, eps, kappa, out, bx, fbad, step, fprev, a, eps_d, chk);
}

template <int CL, bool SCALED>
__global__ void __launch_bounds__(THREADS, 1) dense_cluster_solve_kernel(Args A) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  extern __shared__ __align__(16) float shc[];
  const int n = A.n, m = A.m;
  const int rows_per = (n + CL - 1) / CL;
  const int rp4 = (rows_per + 3) & ~3, m4 = (m + 3) & ~3;
  float *Cs = shc;                                    // [rows_per][m]
  float *f0 = Cs + (size_t)rows_per * m, *f1 = f0 + rp4, *bx = f1 + rp4;
  float *g = bx + rp4, *by = g + m4;
  float *canc = by + m4;                              // [m4] column-partial anchors
  float *xs = canc + m4;                              // [2][CL][m4] pushed column partials
  float *las = xs + 2 * CL * m4, *lbs = las + rp4;    // log weights staged in shared memory
  // SCALED: Cs holds the kernel slice K; beta / v per column, rho / w per row
  float *beta = lbs + m4, *vv = beta + m4, *rho = vv + m4, *uw = rho + rp4;
  double *slot = reinterpret_cast<double *>(uw + rp4);  // [2][NV + 1]
  __shared__ int rebuild_flag;
  __shared__ double red[NV * WARPS];
  __shared__ double rsl[CL * (NV + 1)], rtot[NV + 1];
  __shared__ int fbad;
  __shared__ __align__(8) uint64_t lbar;
  __shared__ __align__(8) uint64_t xbar[2];  // column-partial arrivals, one per buffer parity
  const int r0 = min(n, rank * rows_per), r1 = min(n, r0 + rows_per), rows = r1 - r0;
  const int ncl = (int)(gridDim.x / CL), cid = (int)(blockIdx.x / CL);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&lbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&xbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&xbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster.sync();  // every peer's barriers are initialised before the first push
  uint32_t lphase = 0;
  uint32_t xphase = 0u;  // bit p: phase of xbar[p]
  int xpar = 0;  // parity of the next check-slot exchange
  int cpar = 0;  // parity of the next column exchange (buffer xs[cpar], barrier xbar[cpar])
  for (int64_t b = cid; b < A.batch; b += ncl) {
    const float *Cb = A.C + b * (int64_t)n * m;
    const float *a = A.a + b * n + r0, *bw = A.b + b * m;
    const float *la = las, *lb = lbs;  // the finalizes read log weights from shared memory
    const float eps = A.eps[b];
    const double eps_d = A.eps_d[b];
    const float kappa = kLog2e / eps;
    const float *Cg = Cb + (int64_t)r0 * m;  // this CTA's rows of the cost (global, L2-resident)
    // log domain: this CTA's rows of C -> shared memory (bulk copies, 32 KB pieces)
    if (!SCALED && threadIdx.x == 0 && rows > 0) {
      const size_t bytes = (size_t)rows * m * sizeof(float);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&lbar)),
                   "r"((uint32_t)bytes)
                   : "memory");
      const char *src = reinterpret_cast<const char *>(Cb + (int64_t)r0 * m);
      for (size_t off = 0; off < bytes; off += 32768)
        bulk_g2s(reinterpret_cast<char *>(Cs) + off, src + off, (uint32_t)min((size_t)32768, bytes - off),
                 &lbar);
    }
    if (threadIdx.x == 0) fbad = 0x7fffffff;
    for (int j = threadIdx.x; j < m; j += THREADS) {
      const float g0 = A.g_init ? A.g_init[b * m + j] : 0.f;
      g[j] = g0;
      by[j] = g0 * kappa;
      canc[j] = __int_as_float(0x7fc00000);  // no anchors yet: first passes run the running max
      lbs[j] = A.lb[b * m + j];
      if (bad_potential(g0)) atomicMin(&fbad, 1);
    }
    for (int i = threadIdx.x; i < rp4; i += THREADS) las[i] = (i < rows) ? A.la[b * n + r0 + i] : 0.f;
    if (!SCALED && rows > 0) {  // wait for the cost slice
      asm volatile(
          "{\n\t.reg .pred p;\nW_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra W_%=;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&lbar)),
          "r"(lphase)
          : "memory");
      lphase ^= 1;
    }
    __syncthreads();
    if constexpr (SCALED) build_kernel(Cg, rows, m, by, kappa, Cs, beta, rho);
    float *f = f0, *fn = f1;
    bool f_ready = false;
    int n_checks = 0, status = OTK_OK, fail_iter = 0, converged = 0, t;
    double chk[NV];
    const bool tr = (b == cid) && blockIdx.x == 0;
    for (t = 1; t <= A.max_iters; ++t) {
      dtrace(A, tr, t, 0);
      if (!f_ready) {
        if constexpr (SCALED) {
          while (!scaled_v(by, beta, m, vv, &rebuild_flag)) build_kernel(Cg, rows, m, by, kappa, Cs, beta, rho);
          dtrace(A, tr, t, 6);
          rows_pass_scaled<false>(Cs, rows, m, vv, rho, la, eps, kappa, f, bx, uw, &fbad, 2 * t, nullptr, a,
                                  eps_d, chk);
        } else {
          rows_pass<false>(Cs, rows, m, by, la, eps, kappa, f, bx, &fbad, 2 * t, nullptr, a, eps_d, chk);
        }
        __syncthreads();
      }
      dtrace(A, tr, t, 1);
      f_ready = false;
      // ---- columns: local partials pushed into slot `rank` of every CTA's
      // shared memory with st.async (each push counted on the receiver's
      // mbarrier), each CTA waits for its own barrier, then combines the CL
      // partials of every column from its own shared memory in rank order.
      // Buffer reuse: a CTA pushes epoch e+2 into parity (e & 1) only after its
      // own combine of e+1, which needed every peer's push of e+1, issued after
      // that peer's combine of e -- two buffers suffice, no cluster barrier.
      float *xbuf = xs + cpar * CL * m4;
      {
        const float clo = -96.f + 2.f * log2f((float)max(rows, 1));
        const uint32_t mine = (uint32_t)__cvta_generic_to_shared(xbuf + rank * m4);
        const uint32_t mybar = (uint32_t)__cvta_generic_to_shared(&xbar[cpar]);
        if (threadIdx.x == 0)  // arm: CL pushes of m floats land here this epoch
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mybar),
                       "r"((uint32_t)(CL * m * 4))
                       : "memory");
        for (int j = threadIdx.x; j < m; j += THREADS) {
          float L;
          if constexpr (SCALED) {
            L = col_partial_scaled(Cs, Cg, rows, m, bx, uw, beta, kappa, j);
          } else {
            L = (rows > 0) ? col_partial_anchored(Cs, rows, m, bx, kappa, j, canc[j], clo) : -INFINITY;
            canc[j] = nan_if_not_finite(L);
          }
#pragma unroll
          for (int r = 0; r < CL; ++r) st_async_f32(mapa_u32(mine + 4u * j, r), L, mapa_u32(mybar, r));
        }
      }
      dtrace(A, tr, t, 2);
      mbar_wait_cluster(&xbar[cpar], (xphase >> cpar) & 1u);
      xphase ^= 1u << cpar;
      dtrace(A, tr, t, 3);
      for (int j = threadIdx.x; j < m; j += THREADS) {
        float v[CL];
#pragma unroll
        for (int r = 0; r < CL; ++r) v[r] = xbuf[r * m4 + j];
        float mx = -INFINITY;
        bool nan = false;
#pragma unroll
        for (int r = 0; r < CL; ++r) {
          nan |= (v[r] != v[r]);
          mx = fmaxf(mx, v[r]);
        }
        float L;
        if (nan) {
          L = __int_as_float(0x7fc00000);
        } else if (mx == -INFINITY || mx == INFINITY) {
          L = mx;
        } else {
          float acc = 0.f;
#pragma unroll
          for (int r = 0; r < CL; ++r) acc += ex2(v[r] - mx);
          L = mx + lg2(acc);
        }
        const float lbj = lb[j];  // one read (a second one after the store to g would be a global round trip)
        const float gv = eps * lbj - eps * kLn2 * L;
        g[j] = gv;
        by[j] = next_bias(lbj, L, eps, kappa);
        if (bad_potential(gv)) atomicMin(&fbad, 2 * t + 1);
      }
      cpar ^= 1;
      __syncthreads();
      dtrace(A, tr, t, 4);
      if (t % A.inner_iters == 0 || t == A.max_iters) {
#pragma unroll
        for (int k = 0; k < NV; ++k) chk[k] = 0.0;
        if constexpr (SCALED) {
          while (!scaled_v(by, beta, m, vv, &rebuild_flag)) build_kernel(Cg, rows, m, by, kappa, Cs, beta, rho);
          rows_pass_scaled<true>(Cs, rows, m, vv, rho, la, eps, kappa, fn, bx, uw, &fbad, 2 * t + 2, f, a,
                                 eps_d, chk);
        } else {
          rows_pass<true>(Cs, rows, m, by, la, eps, kappa, fn, bx, &fbad, 2 * t + 2, f, a, eps_d, chk);
        }
        if (rank == 0) {  // g is replicated: its terms are counted once
          for (int j = threadIdx.x; j < m; j += THREADS) {
            const double gj = g[j], bj = bw[j];
            if (bj > 0.0) chk[3] += bj * gj;
            chk[5] += (gj != gj) ? 1.0 : 0.0;
            chk[7] += (gj == INFINITY) ? 1.0 : 0.0;
          }
        }
        block_sum(chk, red);  // ends with every thread holding the CTA totals
        double *myslot = slot + xpar * (NV + 1);
        __syncthreads();      // fbad final for this CTA
        if (threadIdx.x == 0) {
#pragma unroll
          for (int k = 0; k < NV; ++k) myslot[k] = chk[k];
          myslot[NV] = (double)fbad;
        }
        cluster.sync();
        // the CL slots -> shared memory (one remote load per value), then thread
        // k folds value k in rank order: identical in every CTA
        for (int e = threadIdx.x; e < CL * (NV + 1); e += THREADS)
          rsl[e] = cluster.map_shared_rank(myslot, e / (NV + 1))[e % (NV + 1)];
        __syncthreads();
        if (threadIdx.x <= NV) {
          double v = rsl[threadIdx.x];
          for (int r = 1; r < CL; ++r) {
            const double w = rsl[r * (NV + 1) + threadIdx.x];
            v = (threadIdx.x == NV) ? fmin(v, w) : v + w;
          }
          rtot[threadIdx.x] = v;
        }
        __syncthreads();
        double tot[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) tot[k] = rtot[k];
        const double fb = rtot[NV];
        xpar ^= 1;
        const int fbi = (int)fb;
        int d = 0;  // 0 continue, 1 converged, 2 bad potential, 3 diverged
        if (fbi <= 2 * t) {
          d = 2;
          fail_iter = (fbi + 1) / 2;
        } else if (tot[4] > 0 || tot[5] > 0) {
          d = 3;
          fail_iter = t;
        } else if (fbi == 2 * t + 1) {
          d = 2;
          fail_iter = t;
        } else {
          if (rank == 0 && threadIdx.x == 0 && n_checks < A.max_checks) {
            A.errors[b * A.max_checks + n_checks] = tot[0];
            A.duals[b * A.max_checks + n_checks] = tot[2] + tot[3] - eps_d * (tot[1] - 1.0);
          }
          if (tot[0] <= A.threshold) d = 1;
        }
        if (d == 2 || d == 3) {
          status = (d == 2) ? OTK_BAD_POTENTIAL : OTK_DIVERGED;
          break;
        }
        ++n_checks;
        if (d == 1) {
          converged = 1;
          break;
        }
        if (t < A.max_iters) {
          float *tmp = f;
          f = fn;
          fn = tmp;
          f_ready = true;
        }
        dtrace(A, tr, t, 5);
      }
    }
    for (int i = threadIdx.x; i < rows; i += THREADS) A.f_out[b * n + r0 + i] = f[i];
    if (rank == 0) {
      for (int j = threadIdx.x; j < m; j += THREADS) A.g_out[b * m + j] = g[j];
      if (threadIdx.x == 0) {
        int *st = A.state + b * 5;
        st[0] = min(n_checks, A.max_checks);
        st[1] = min(t, A.max_iters);
        st[2] = converged;
        st[3] = status;
        st[4] = fail_iter;
      }
    }
    // no CTA may overwrite its cost slice / partials while a peer still reads them
    cluster.sync();
  }
}

size_t cluster_smem_bytes(int n, int m, int CL) {
  const size_t rows_per = (n + CL - 1) / CL;
  const size_t rp4 = (rows_per + 3) & ~(size_t)3, m4 = (m + 3) & ~3;
  return rows_per * m * sizeof(float) + (6 * rp4 + 6 * m4 + 2 * (size_t)CL * m4) * sizeof(float) +
         2 * (NV + 1) * sizeof(double) + 64;
}

// The scaling-domain kernel holds a row's v values in registers: m <= 512;
// OTK_DENSE_DOMAIN=log forces the log-domain passes (A/B).
static bool scaled_domain(int m) {
  const char *e = getenv("OTK_DENSE_DOMAIN");
  return m <= 512 && !(e && strcmp(e, "log") == 0);
}

template <int CL>
static int cluster_try(const Args &A, int n, int m, int64_t batch, int grid, cudaStream_t st,
                       bool launch, int *sms_used) {
  int dev = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t smem = cluster_smem_bytes(n, m, CL);
  if (smem + 2048 > (size_t)max_smem) return OTK_ENOTSUP;
  auto kern = scaled_domain(m) ? dense_cluster_solve_kernel<CL, true> : dense_cluster_solve_kernel<CL, false>;
  OTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL * 64);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = CL;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl <= 0) {
    cudaGetLastError();
    return OTK_ENOTSUP;
  }
  if (grid > 0) ncl = std::min(ncl, std::max(1, grid / CL));
  ncl = (int)std::min<int64_t>(ncl, batch);
  *sms_used = ncl * CL;
  if (!launch) return OTK_OK;
  cfg.gridDim = dim3(CL * ncl);
  OTK_CUDA(cudaLaunchKernelEx(&cfg, kern, A));
  return OTK_OK;
}

// Cluster size with the most SMs in use (clusters live inside one GPC, so
// e.g. 8 x k may leave SMs idle where 6 x k or 7 x k does not; sizes whose
// cost slice does not fit shared memory drop out); ties go to the larger
// cluster (fewer rows per CTA).  OTK_DENSE_CL forces one size.
int launch_cluster_solve(const Args &A, int n, int m, int64_t batch, int grid, int want_cl,
                         cudaStream_t st) {
  int used[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  bool ok[9] = {false, false, false, false, false, false, false, false, false};
  ok[5] = (want_cl == 0 || want_cl == 5) && cluster_try<5>(A, n, m, batch, grid, st, false, &used[5]) == OTK_OK;
  ok[6] = (want_cl == 0 || want_cl == 6) && cluster_try<6>(A, n, m, batch, grid, st, false, &used[6]) == OTK_OK;
  ok[7] = (want_cl == 0 || want_cl == 7) && cluster_try<7>(A, n, m, batch, grid, st, false, &used[7]) == OTK_OK;
  ok[8] = (want_cl == 0 || want_cl == 8) && cluster_try<8>(A, n, m, batch, grid, st, false, &used[8]) == OTK_OK;
  int best = 0;
  for (int c = 5; c <= 8; ++c)
    if (ok[c] && (best == 0 || used[c] >= used[best])) best = c;
  int dummy = 0;
  switch (best) {
    case 5: return cluster_try<5>(A, n, m, batch, grid, st, true, &dummy);
    case 6: return cluster_try<6>(A, n, m, batch, grid, st, true, &dummy);
    case 7: return cluster_try<7>(A, n, m, batch, grid, st, true, &dummy);
    case 8: return cluster_try<8>(A, n, m, batch, grid, st, true, &dummy);
    default: return OTK_ENOTSUP;
  }
}

// The cluster size the batched solve would use for n x m problems and the SMs
// it would occupy (0, 0 when the cost slices do not fit: K3p streams instead).
int cluster_plan(int n, int m, int64_t batch, int *cl, int *sms) {
  Args A{};
  int used[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  bool ok[9] = {false, false, false, false, false, false, false, false, false};
  ok[5] = cluster_try<5>(A, n, m, batch, 0, nullptr, false, &used[5]) == OTK_OK;
  ok[6] = cluster_try<6>(A, n, m, batch, 0, nullptr, false, &used[6]) == OTK_OK;
  ok[7] = cluster_try<7>(A, n, m, batch, 0, nullptr, false, &used[7]) == OTK_OK;
  ok[8] = cluster_try<8>(A, n, m, batch, 0, nullptr, false, &used[8]) == OTK_OK;
  *cl = 0;
  *sms = 0;
  for (int c = 5; c <= 8; ++c)
    if (ok[c] && (*cl == 0 || used[c] >= used[*cl])) {
      *cl = c;
      *sms = used[c];
    }
  return OTK_OK;
}

size_t smem_bytes(int n, int m) {
  const size_t n4 = (n + 3) & ~3, m4 = (m + 3) & ~3;
  return (3 * n4 + 2 * m4) * sizeof(float) + (size_t)WARPS * 128 * 2 * sizeof(float);
}

}  // namespace dsolve
}  // namespace otk

using namespace otk;

extern "C" int otk_dense_cluster_plan(int64_t n, int64_t m, int64_t batch, int32_t *cluster,
                                      int32_t *sms) {
  OTK_CHECK_ARG(cluster && sms && n > 0 && m > 0 && batch > 0, "otk_dense_cluster_plan: bad arguments");
  if (!otk_dense_solve_fits(n, m)) {
    *cluster = 0;
    *sms = 0;
    return OTK_OK;
  }
  int c = 0, u = 0;
  dsolve::cluster_plan((int)n, (int)m, batch, &c, &u);
  *cluster = c;
  *sms = u;
  return OTK_OK;
}

extern "C" int otk_dense_solve_fits(int64_t n, int64_t m) {
  if (n < 1 || m < 1 || m % 4 != 0 || n > 16384 || m > 16384) return 0;
  int dev = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return dsolve::smem_bytes((int)n, (int)m) + 4096 <= (size_t)max_smem ? 1 : 0;
}

extern "C" int otk_solve_dense_batched(const float *cost, int64_t batch, int64_t n, int64_t m,
                                       const float *a, const float *b, const float *log_a,
                                       const float *log_b, const float *eps, const double *eps_d,
                                       const float *g_init, double threshold, int32_t max_iters,
                                       int32_t inner_iters, int32_t max_checks, float *f_out,
                                       float *g_out, double *errors, double *duals, int32_t *state,
                                       int32_t grid, void *stream) {
  OTK_CHECK_ARG(cost && a && b && log_a && log_b && eps && eps_d && f_out && g_out && errors &&
                    duals && state && batch > 0,
                "otk_solve_dense_batched: bad arguments");
  OTK_CHECK_ARG(otk_dense_solve_fits(n, m), "otk_solve_dense_batched: n, m unsupported (m %% 4, smem)");
  OTK_CHECK_ARG(max_iters >= 1 && inner_iters >= 1 && max_checks >= 1 && (threshold > 0 || threshold < 0),
                "otk_solve_dense_batched: bad loop parameters");
  dsolve::Args A{cost, batch, (int)n, (int)m, a, b, log_a, log_b, eps, g_init, eps_d, threshold,
                 max_iters, inner_iters, max_checks, f_out, g_out, errors, duals, state, nullptr};
  const char *trace_path = getenv("OTK_DENSE_TRACE");  // diagnostics (tools/dense_trace.py)
  if (trace_path) {
    OTK_CUDA(cudaMalloc(&A.trace, 64 * 8 * sizeof(unsigned long long)));
    OTK_CUDA(cudaMemsetAsync(A.trace, 0, 64 * 8 * sizeof(unsigned long long), as_stream(stream)));
#ifdef OTK_DENSE_TRACE_BUILD
    const unsigned long long zero = 0;
    OTK_CUDA(cudaMemcpyToSymbol(dsolve::g_dense_rebuilds, &zero, sizeof(zero)));
    OTK_CUDA(cudaMemcpyToSymbol(dsolve::g_dense_fallbacks, &zero, sizeof(zero)));
#endif
  }
  // K3c (cost resident in a cluster's shared memory) whenever a slice fits;
  // OTK_DENSE_KERNEL=cta forces the one-CTA-per-problem streaming kernel K3p
  const char *kind = getenv("OTK_DENSE_KERNEL");
  if (!(kind && strcmp(kind, "cta") == 0)) {
    const int want_cl = getenv("OTK_DENSE_CL") ? atoi(getenv("OTK_DENSE_CL")) : 0;
    int rc = dsolve::launch_cluster_solve(A, (int)n, (int)m, batch, grid, want_cl, as_stream(stream));
    if (rc != OTK_ENOTSUP) {
      if (trace_path) {
        unsigned long long h[64 * 8];
        OTK_CUDA(cudaMemcpyAsync(h, A.trace, sizeof(h), cudaMemcpyDeviceToHost, as_stream(stream)));
        OTK_CUDA(cudaStreamSynchronize(as_stream(stream)));
        cudaFree(A.trace);
#ifdef OTK_DENSE_TRACE_BUILD
        // row 63: rebuilds of kernel slices and exact column fallbacks over the whole batch
        OTK_CUDA(cudaMemcpyFromSymbol(&h[63 * 8], dsolve::g_dense_rebuilds, sizeof(h[0])));
        OTK_CUDA(cudaMemcpyFromSymbol(&h[63 * 8 + 1], dsolve::g_dense_fallbacks, sizeof(h[0])));
#endif
        if (FILE *fp = fopen(trace_path, "wb")) {
          fwrite(h, sizeof(h[0]), 64 * 8, fp);
          fclose(fp);
        }
      }
      return rc;
    }
  }
  const size_t smem = dsolve::smem_bytes((int)n, (int)m);
  OTK_CUDA(cudaFuncSetAttribute(dsolve::dense_solve_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // default: one CTA per problem (measured on cfg3, 512 problems: grid 128 / 148 / 296 / 512 ->
  // 6.13 / 6.47 / 6.31 / 5.69 ms per batched solve; the lock-step loop 8.59 ms)
  const int g = (int)std::min<int64_t>(std::min<int64_t>(batch, 65535), grid > 0 ? grid : batch);
  dsolve::dense_solve_kernel<<<g, dsolve::THREADS, smem, as_stream(stream)>>>(A);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}
