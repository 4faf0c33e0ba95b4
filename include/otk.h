/*
 * otk.h -- C ABI of the B200 (sm_100a) log-domain Sinkhorn library
 *          (libotk_sm100.so, built from paper_2201_12324_b200/csrc).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (`otkit`, /root/reference/pkg/src/otkit) is pure Python; its seam is the
 * Geometry plugin API (geometry.py:100-168) driven by the solver loop
 * sinkhorn.py:151-200.  Each entry point below names the reference function
 * it replaces.  Conventions:
 *   - every array argument is a DEVICE pointer to caller-owned, contiguous,
 *     row-major memory (float32 unless stated; fp16 planes as uint16_t);
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - the library never allocates persistent device memory: scratch space is
 *     passed in (sizes from the *_workspace_bytes queries);
 *   - return value: OTK_OK (0) or a negative error; otk_last_error() gives
 *     the message (thread-local).  Solver entries may also return the
 *     positive OTK_DIVERGED / OTK_BAD_POTENTIAL outcomes.
 * Potentials use the reference convention: -inf allowed (zero-weight
 * locations), NaN / +inf are invalid (geometry.py:65-72).
 */
#ifndef OTK_H
#define OTK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTK_ABI_VERSION 7

enum otk_status {
  OTK_OK = 0,
  OTK_EINVAL = -1,      /* invalid argument                -> ValueError   */
  OTK_ECUDA = -2,       /* CUDA runtime / launch failure   -> RuntimeError */
  OTK_ENOTSUP = -3,     /* unsupported on this device/shape                */
  OTK_ENCCL = -4,       /* NCCL failure (multi-GPU)                        */
  OTK_DIVERGED = 1,     /* NaN at a check: errors.py:10-20 DivergedError   */
  OTK_BAD_POTENTIAL = 2 /* NaN/+inf potential fed to a half-step:
                           geometry.py:65-72 ValueError                    */
};

/* flags for otk_lse_partial / otk_cost_partial */
#define OTK_SAME_POINTS 0x1 /* x and y are the same set: exact-zero diagonal (geometry.py:259-261) */
#define OTK_CLAMP 0x2       /* clamp C >= 0 (geometry.py:273)                                      */
#define OTK_COST_EUCL 0x4   /* cost_fn "eucl": C = sqrt(max(|p|^2+|q|^2-2<p,q>, 0)) (geometry.py:274-275) */
#define OTK_IMPL_SIMT 0x10  /* force the FP32 FMA kernel                                           */
#define OTK_IMPL_TC 0x20    /* force the tcgen05 split-fp16 kernel                                 */
#define OTK_IMPL_NOPERSIST 0x40 /* otk_solve_pointcloud: never use the one-kernel small-problem solve */
#define OTK_ANCHOR_INIT 0x80    /* otk_lse_step: the anchor holds no result yet (running-max kernel; anchor written) */
#define OTK_IMPL_NOANCHOR 0x100 /* otk_solve_pointcloud: never use the anchored half-step              */

/* finalize modes */
#define OTK_FIN_SOLVER 0 /* out = eps*logw - eps*ln2*L   (sinkhorn.py:173-174)                     */
#define OTK_FIN_APPLY 1  /* out = f + eps*ln2*L           (geometry.py:336-354)                     */
#define OTK_FIN_LOG2 2   /* out = L (this shard's column partial for the multi-GPU g update;
                            base, out_bias, first_bad unused)                                      */

int otk_abi_version(void);
const char *otk_last_error(void);
int otk_device_query(int device, int *sm_count, int *cc_major, int *cc_minor);

/* K0 -- per-point preparation.  Replaces the norm einsums of _cost_block
 * (geometry.py:269-270).  sqnorm[i] = |p_i|^2 (float64 accumulate).  If hi is
 * non-NULL also writes the split-fp16 operand planes of the tcgen05 kernel
 * (row pitch dpad >= d, zero padded, s = split_scale a power of two):
 *   hi = fp16(s*p), lo = fp16(s*p - hi)                      [n, dpad]
 * and the two 16-column norm planes that add -s^2 (|p_i|^2 + |q_j|^2)/2 in one
 * MMA at the end of every TC tile (so the accumulators end at -s^2 C_ij/2):
 *   ext_a[i, 0:16] = [-w0,-w1,-w2, 2^15,2^15,2^15, 0...]   (A role)
 *   ext_b[i, 0:16] = [2^15,2^15,2^15, -w0,-w1,-w2, 0...]   (B role)
 * with w0+w1+w2 = s^2 |p_i|^2 / 2^16 in three fp16 pieces.  [n, 16].
 * s must come from otk_split_scale (fp16 range of hi/lo and the pieces). */
int otk_prep_points(const float *pts, int64_t n, int32_t d, float *sqnorm,
                    uint16_t *hi, uint16_t *lo, uint16_t *ext_a, uint16_t *ext_b,
                    int32_t dpad, float split_scale, void *stream);

/* Translation (before K0).  The cost is translation-invariant; the reference
 * forms _cost_block (geometry.py:268-273) in float64, where a common offset of
 * the clouds costs nothing, but float32 |p|^2 + |q|^2 - 2<p,q> loses
 * ~ulp(|p|^2) to cancellation.  Both sets are therefore shifted by one common
 * centre before prep: otk_column_median writes center[k] = the (lower)
 * median of q[:, k] over at most 8192 evenly strided rows (robust to far
 * outliers, unlike the mean; exact float32 values, deterministic);
 * otk_shift_points writes out = fp32(p - center) (out may not alias p). */
int otk_column_median(const float *q, int64_t m, int32_t d, double *center, void *stream);
int otk_shift_points(const float *p, int64_t n, int32_t d, const double *center, float *out,
                     void *stream);

/* max |p_ik| over the array (for choosing split_scale); out is one float. */
int otk_absmax(const float *pts, int64_t count, float *out, void *stream);

/* PointCloudGeometry.__init__ (geometry.py:247-261) in one launch: flags[0] / [1] = 1
 * when x / y holds a non-finite coordinate, flags[2] = 1 when compare != 0 and the
 * sets differ anywhere (compare only with nx == ny).  flags: device int32[3]. */
int otk_points_flags(const float *x, int64_t nx, const float *y, int64_t ny, int32_t d,
                     int32_t compare, int32_t *flags, void *stream);

/* mean_cost's sampled estimate (geometry.py:294-312): the mean over `count` pairs
 * (ii[s], jj[s]) of the cost between kernel points x[ii] and y[jj] (float64
 * difference form; flags: OTK_COST_EUCL, OTK_SAME_POINTS -> exact zero for i == j).
 * ii, jj: device int64[count]; mean: device double[1]. */
int otk_mean_cost_pairs(const float *x, const float *y, const int64_t *ii, const int64_t *jj,
                        int64_t count, int32_t d, int32_t flags, double *mean, void *stream);

/* The power-of-two operand scale for point sets of dimension d whose largest
 * |coordinate| is amax (one common scale for both sets of a geometry). */
float otk_split_scale(float amax, int32_t d);

/* Scaled potential of the reduced side for the next half-step:
 * bias_j = kappa * pot_j.  NaN/+inf in pot -> atomicMin(first_bad, step). */
int otk_make_bias(const float *pot, int64_t m, float kappa, float *bias,
                  int32_t *first_bad, int32_t step, void *stream);

/* K1/K2 -- online half-step partials.  Replaces PointCloudGeometry.apply_lse_kernel
 * (geometry.py:336-354) and its _cost_rows/_cost_cols blocks (263-292), never
 * materialising C.  With kappa = log2(e)/eps and q_bias_j = kappa*pot_j:
 *     partial[s*np + i] = log2 sum_{j in split s} 2^(q_bias_j - kappa*C_ij)
 * (-inf if empty).  Columns are split into `nsplit` equal contiguous ranges
 * (fixed order).  C_ij = |p_i|^2 + |q_j|^2 - 2<p_i,q_j> from the squared norms
 * (FP32 path; OTK_CLAMP / OTK_SAME_POINTS reproduce max(C,0) and the zero
 * diagonal) or from the split planes (TC path: hi/lo/ext_a of P, hi/lo/ext_b
 * of Q, dpad % 64 == 0, split_inv = 1/s^2 with one common scale s). */
int otk_lse_partial(const float *p, const float *p_sq, const uint16_t *p_hi,
                    const uint16_t *p_lo, const uint16_t *p_ext, int64_t np,
                    const float *q, const float *q_sq, const uint16_t *q_hi,
                    const uint16_t *q_lo, const uint16_t *q_ext, int64_t nq,
                    int32_t d, int32_t dpad, float split_inv, const float *q_bias,
                    float kappa, int32_t flags, int32_t nsplit, float *partial,
                    void *stream);

/* 1 if otk_lse_partial runs the tcgen05 kernel for this d / flags (the caller
 * must then pass the split + norm planes), 0 for the FP32 FMA kernel. */
int otk_lse_uses_tc(int32_t d, int32_t flags);

/* Suggested split count for otk_lse_partial on this device. */
int otk_lse_suggest_nsplit(int64_t np, int64_t nq, int32_t d, int32_t flags);

/* Combine partials (fixed split order) and produce the potential:
 *   SOLVER: out_i = eps*base_i - eps*ln2*L_i    (base = log w; sinkhorn.py:173-174)
 *   APPLY:  out_i = base_i + eps*ln2*L_i        (base = f; apply_lse_kernel)
 *   LOG2:   out_i = L_i                         (row-sharded solve: the shard's
 *           column partial, all-gathered across ranks and combined again with
 *           nsplit = world size, rank order -- SURVEY.md §8e / K7)
 * If out_bias != NULL also writes kappa_next*out_i (this side's bias for the
 * next half-step).  NaN/+inf in out -> atomicMin(first_bad, step) (first_bad
 * may be NULL). */
int otk_lse_finalize(const float *partial, int32_t nsplit, int64_t np,
                     const float *base, int32_t mode, float eps, float kappa_next,
                     float *out_pot, float *out_bias, int32_t *first_bad,
                     int32_t step, void *stream);

/* One whole half-step = otk_lse_partial + otk_lse_finalize (same arguments,
 * same results to fp32 rounding), with an optional per-row ANCHOR that
 * replaces the running max of the streaming log-sum-exp.  anchor[np] holds
 * the log2 result L_i of this role's previous half-step (NaN = unknown) and
 * is overwritten with the new L_i.  On the tcgen05 sqeucl path
 * (otk_lse_step_anchored) each row sums 2^(u_ij - anchor_i) directly -- no
 * max, no rescale; a row whose result leaves the safe window (overflow, or
 * L_i - anchor_i outside [-96 + 2 log2(nq), 120], where terms could flush to
 * zero) is
 * recomputed by the running-max kernel inside the same call (device-side
 * decision, 4 launches, CUDA-graph capturable).  flags & OTK_ANCHOR_INIT:
 * the anchor holds nothing yet -- running-max kernel, anchor written.  With
 * anchor == NULL this is exactly otk_lse_partial + otk_lse_finalize.
 * repair_ws: otk_lse_step_workspace_bytes(np) bytes (no initialisation). */
/* Multi-GPU exchange over NVLink peer memory (row-sharded solve, the g
 * half-step).  Every rank owns one exchange buffer of
 * otk_exchange_bytes(world, m) bytes (otk_exchange_alloc: cudaMalloc, zeroed,
 * IPC-exportable), exports it (otk_ipc_handle, 64 bytes), opens the peers'
 * (otk_ipc_open) and stores the W base pointers -- its own at [rank] -- in its
 * buffer (otk_exchange_set_peers).  otk_lse_step with an otk_exchange in
 * OTK_FIN_LOG2 mode then pushes every row's log2 partial into slot
 * (epoch & 1, rank) of every peer from its last finalize kernel and releases
 * one flag per 256-row block on every peer; otk_exchange_finalize waits for
 * the W flags of each block (acquire), combines the W partials in rank order
 * and applies the finalize mode -- g bitwise equal on all ranks and to the
 * all-gather + otk_lse_finalize path.  epoch: 0 = device-counted (the push
 * and the combine use one past the buffer's count of completed combines; the
 * combine advances it -- replayable inside CUDA graphs; what every caller of
 * this library uses), or an explicit epoch >= 1 growing by one per exchange,
 * identical on all ranks (the two must not be mixed on one buffer).  A wait
 * longer than timeout_ms (0 = 10 s) sets the buffer's error word
 * (otk_exchange_status != 0) instead of hanging. */
typedef struct otk_exchange {
  void *local;         /* this rank's exchange buffer (device) */
  int32_t world, rank;
  uint32_t epoch;
} otk_exchange;
size_t otk_exchange_bytes(int32_t world, int64_t m);
int otk_exchange_alloc(size_t bytes, void **ptr);
int otk_exchange_free(void *ptr);
int otk_ipc_handle(void *ptr, void *handle);
int otk_ipc_open(const void *handle, void **ptr);
int otk_ipc_close(void *ptr);
int otk_exchange_set_peers(void *local, int32_t world, int64_t m, void *const *peers,
                           void *stream);
int otk_exchange_finalize(void *local, int32_t world, int64_t m, uint32_t epoch,
                          const float *base, int32_t mode, float eps, float kappa_next,
                          float *out_pot, float *out_bias, int32_t *first_bad, int32_t step,
                          uint32_t timeout_ms /* 0 = 10 s */, void *stream);
int otk_exchange_status(void *local, int32_t *status, void *stream);
/* Check-sum exchange of a sharded solve (sinkhorn.py:175-189 over row
 * shards): sums[0..7] = this rank's otk_check output, *first_bad = its first
 * bad step; out[0..7] = the rank-order totals every rank computes alike
 * ([3], [5], [7] -- the replicated g terms -- from rank 0), out[8] = min
 * first-bad step over ranks, out[9] = nonzero if any rank's exchange timed
 * out.  One single-block launch; epochs device-counted. */
int otk_exchange_check(void *local, int32_t world, int32_t rank, int64_t m, const double *sums,
                       const int32_t *first_bad, double *out, uint32_t timeout_ms, void *stream);

size_t otk_lse_step_workspace_bytes(int64_t np);
/* 1 if otk_lse_step anchors on this path AND the half-step is long enough for
 * it to pay (np * nq >= 2^27 cells; env OTK_ANCHOR_MIN_CELLS overrides). */
int otk_lse_step_anchored(int64_t np, int64_t nq, int32_t d, int32_t flags);
/* xchg (nullable, OTK_FIN_LOG2 only): push the rows to every rank (above). */
int otk_lse_step(const float *p, const float *p_sq, const uint16_t *p_hi,
                 const uint16_t *p_lo, const uint16_t *p_ext, int64_t np,
                 const float *q, const float *q_sq, const uint16_t *q_hi,
                 const uint16_t *q_lo, const uint16_t *q_ext, int64_t nq, int32_t d,
                 int32_t dpad, float split_inv, const float *q_bias, float kappa,
                 int32_t flags, int32_t nsplit, float *partial, const float *base,
                 int32_t mode, float eps, float kappa_next, float *out_pot,
                 float *out_bias, int32_t *first_bad, int32_t step, float *anchor,
                 int32_t *repair_ws, const otk_exchange *xchg, void *stream);

/* K5 -- fused convergence check (sinkhorn.py:175-189 + _dual_objective 115-119).
 * From f_prev = f_t, f_next = f_{t+1} (the next rows half-step) and g = g_t:
 *   r_i = a_i*exp((f_prev_i - f_next_i)/eps)  (= exp(apply_lse_kernel(f,g,rows)/eps))
 * out[0]=sum|r-a|, [1]=sum r, [2]=sum_{a>0} a f_prev, [3]=sum_{b>0} b g,
 * [4]=#NaN(f_prev), [5]=#NaN(g), [6]=#(+inf)(f_prev), [7]=#(+inf)(g).
 * f_next may be NULL (only [2..7] computed).  Deterministic float64
 * reduction; ws = otk_check_workspace_bytes() bytes of scratch. */
size_t otk_check_workspace_bytes(void);
int otk_check(const float *f_prev, const float *f_next, const float *a,
              int64_t n, const float *g, const float *b, int64_t m, double eps,
              double *out, void *ws, void *stream);

/* K6 -- online reg_ot_cost (sinkhorn.py:210-216, never materialised):
 * out[0] = sum_ij C_ij P_ij, out[1] = sum_ij P_ij with P = exp((f_i+g_j-C_ij)/eps).
 * ws: otk_cost_workspace_bytes(np) bytes. */
size_t otk_cost_workspace_bytes(int64_t np, int64_t nq);
int otk_cost_partial(const float *p, const float *p_sq, int64_t np,
                     const float *q, const float *q_sq, int64_t nq, int32_t d,
                     const float *f, const float *g, double eps, int32_t flags,
                     double *out, void *ws, void *stream);

/* transport_matrix (sinkhorn.py:203-207): P[i*m+j] = exp((f_i+g_j-C_ij)/eps). */
int otk_transport_matrix(const float *p, const float *p_sq, int64_t np,
                         const float *q, const float *q_sq, int64_t nq,
                         int32_t d, const float *f, const float *g, double eps,
                         int32_t flags, float *plan, void *stream);

/* Envelope gradient in the source points (sinkhorn.py:232-246), online, no
 * n*m cap: grad[i*d+k] = 2 (r_i p_ik - sum_j P_ij q_jk), r_i = sum_j P_ij,
 * P_ij = exp((f_i + g_j - C_ij)/eps).  FP32, [np, d] row-major output. */
int otk_grad_points(const float *p, const float *p_sq, int64_t np, const float *q,
                    const float *q_sq, int64_t nq, int32_t d, const float *f,
                    const float *g, double eps, int32_t flags, float *grad,
                    void *stream);

/* ---------------- materialised / batched path (DenseGeometry) ---------------- */

/* K4 -- C[b,i,j] = sum_k (x_bik - y_bjk)^2 (PointCloudGeometry.cost_matrix,
 * geometry.py:314-316; exact-zero diagonal with OTK_SAME_POINTS).  If cost_t
 * is non-NULL also writes C^T[b,j,i] (the column half-steps then run the
 * coalesced row kernel over C^T: otk_dense_lse(cost_t, batch, m, n, 0, ...)). */
int otk_dense_cost(const float *x, const float *y, int64_t batch, int64_t n,
                   int64_t m, int32_t d, int32_t flags, float *cost,
                   float *cost_t, void *stream);

/* C^T[b] = C[b]^T for a stored cost (DenseGeometry, geometry.py:171-211). */
int otk_dense_transpose(const float *cost, int64_t batch, int64_t n, int64_t m,
                        float *cost_t, void *stream);

/* K3 -- DenseGeometry.apply_lse_kernel (geometry.py:204-211), batched, fused
 * with the finalize step.  axis 0 ("rows"): out[b,i] from reduction over j;
 * axis 1 ("cols"): out[b,j] from reduction over i.  For problem b with
 * kappa_b = log2(e)/eps_b and u = in_bias[b,*] - kappa_b*C:
 *   SOLVER: out = eps_b*base - eps_b*ln2*L;   APPLY: out = base + eps_b*ln2*L
 * and out_bias = out*kappa_next_b (next half-step's bias) when non-NULL.
 * active[b] == 0 skips problem b (NULL = all active).  first_bad is per
 * problem: NaN/+inf in out -> atomicMin(first_bad + b, step). */
int otk_dense_lse(const float *cost, int64_t batch, int64_t n, int64_t m,
                  int32_t axis, const float *in_bias, const float *base,
                  int32_t mode, const float *eps, const float *kappa_next,
                  const int32_t *active, float *out_pot, float *out_bias,
                  int32_t *first_bad, int32_t step, void *stream);

/* Batched fused check: out[b*8 + k] as in otk_check, per problem. */
int otk_check_batched(const float *f_prev, const float *f_next, const float *a,
                      int64_t n, const float *g, const float *b, int64_t m,
                      int64_t batch, const float *eps, const int32_t *active,
                      double *out, void *stream);

/* K3p -- B independent stored-cost problems, each solved by ONE CTA from
 * start to finish (sinkhorn.py:151-200 per problem; constant eps): no host
 * round trip, each problem stops at its own convergence.  Inputs [B,n,m]
 * cost, [B,n]/[B,m] weights and log-weights, eps [B] (float32 for the
 * kernel, float64 for the check), optional g_init [B,m].  Outputs f [B,n],
 * g [B,m], errors/duals [B, max_checks] (device), state [B,5] = n_checks,
 * iterations, converged, status (OTK_OK / OTK_DIVERGED / OTK_BAD_POTENTIAL),
 * fail_iter.  grid <= 0: one CTA per problem.  Requires m % 4 == 0 and
 * otk_dense_solve_fits(n, m). */
int otk_dense_solve_fits(int64_t n, int64_t m);
/* The cluster size K3c would use for a batch of n x m problems and the SMs it
 * would occupy (both 0 when the per-CTA cost slices do not fit: K3p). */
int otk_dense_cluster_plan(int64_t n, int64_t m, int64_t batch, int32_t *cluster, int32_t *sms);
int otk_solve_dense_batched(const float *cost, int64_t batch, int64_t n, int64_t m,
                            const float *a, const float *b, const float *log_a,
                            const float *log_b, const float *eps, const double *eps_d,
                            const float *g_init, double threshold, int32_t max_iters,
                            int32_t inner_iters, int32_t max_checks, float *f_out,
                            float *g_out, double *errors, double *duals, int32_t *state,
                            int32_t grid, void *stream);

/* transport_matrix for a stored cost (sinkhorn.py:203-207), one problem. */
int otk_dense_plan(const float *cost, int64_t n, int64_t m, const float *f,
                   const float *g, double eps, float *plan, void *stream);

/* Batched dense reg_ot_cost: out[b*2+0] = sum C P, out[b*2+1] = sum P. */
int otk_dense_cost_reduce(const float *cost, int64_t batch, int64_t n,
                          int64_t m, const float *f, const float *g,
                          const float *eps, double *out, void *stream);

/* ---------------- native solver loop ---------------- */

typedef struct otk_solve_args {
  /* problem (device pointers) */
  const float *x, *y;        /* [n,d], [m,d]                                  */
  int64_t n, m;
  int32_t d;
  const float *a, *b;        /* weights [n], [m]                              */
  const float *log_a, *log_b;/* log weights (-inf where weight is 0)          */
  int32_t same_points;
  /* epsilon schedule (geometry.py:75-97): eps_t = max(target, target*init*decay^t) */
  double eps_target, eps_init_scale, eps_decay;
  double threshold;          /* > 0 (sinkhorn.py:187); < 0: never stop early (fixed-iteration measurement runs) */
  int32_t max_iters, inner_iters;
  const float *g_init;       /* nullable warm start (sinkhorn.py:166)         */
  int32_t flags;             /* OTK_IMPL_* / OTK_CLAMP / OTK_COST_EUCL        */
  int32_t use_graphs;        /* capture constant-eps check periods            */
  /* outputs */
  float *f_out, *g_out;      /* device [n], [m]                               */
  double *errors, *duals;    /* host arrays, capacity max_checks              */
  int32_t max_checks;
  int32_t n_checks, iterations, converged, fail_iter;
  int32_t launches;          /* kernels launched (graph nodes included)       */
  /* workspace (device) */
  void *workspace;
  size_t workspace_bytes;
  void *stream;
  /* nullable PINNED host buffers [n], [m]: f and g are there after the call's one
   * final synchronisation (saves the caller a second D2H sync).  The persistent
   * small-problem kernel writes them directly (zero-copy) when they are pinned
   * (cudaHostAlloc / cudaHostRegister memory); pageable buffers get a copy.
   * Note: with threshold so small that only an exact float32 fixed point
   * satisfies it (f_{t+1} == f_t bitwise, marginal error 0.0), the loop stops at
   * that iteration with converged = 1 -- every later iterate would be the same. */
  float *f_host, *g_host;
} otk_solve_args;

/* Bytes of device workspace otk_solve_pointcloud needs for these args. */
size_t otk_solve_workspace_bytes(const otk_solve_args *args);

/* Fixed-support barycenter (otkit/barycenter.py:96-133, solve_barycenter; the
 * reference's per-iteration 3K apply_lse_kernel calls, barycenter.py:116-128)
 * as ONE persistent cooperative kernel over a materialised square support
 * cost.  Layout: cost_p / cost_tp [n, ld] fp32 row-major, ld =
 * otk_barycenter_ld(n) (multiple of 4), columns n..ld-1 = +inf, written by
 * otk_barycenter_pad from a contiguous [n, n] cost.  log2_hists [K, n] fp32
 * (log2 of the histograms, -inf for zeros), weights [K] f64.  Workspaces
 * F, G, B: [K, ld] fp32 each; part: otk_barycenter_part_len doubles.
 * Outputs: log2_p [n] f64 (log2 of the unnormalised barycenter of the last
 * iteration), errors [max_iters] f64 (max_k marginal L1 error per iteration),
 * state[8] = {iterations, converged, nan_iteration (0 = none), grid, 4 x
 * scratch (task counters)}.  Stops
 * after the first iteration whose error <= threshold, on NaN in log p
 * (DivergedError at that iteration, barycenter.py:120-121) or at max_iters. */
int64_t otk_barycenter_ld(int64_t n);
int64_t otk_barycenter_part_len(int64_t n, int32_t K);
int otk_barycenter_pad(const float *cost, int64_t n, int64_t ld, float *cost_p, float *cost_tp,
                       void *stream);
int otk_solve_barycenter(const float *cost_p, const float *cost_tp, int64_t n, int64_t ld,
                         int32_t K, const float *log2_hists, const double *weights, double eps,
                         double threshold, int32_t max_iters, float *F, float *G, float *B,
                         double *log2_p, double *errors, int32_t *state, double *part,
                         void *stream);

/* Pipe throughput microbenchmarks (roofline denominators measured on the box):
 * MUFU ex2 results/s and FP32 FFMA/s (full chip, best of 3). */
int otk_bench_pipes(double *ex2_per_s, double *ffma_per_s, void *stream);

/* Streaming-read microbenchmark: best-of-5 HBM read rate (GB/s) over `bytes`
 * of `buf` -- the achievable bound of the materialised-cost half-steps. */
int otk_bench_read(const float *buf, int64_t bytes, double *gbs, void *stream);

/* Shared-memory read microbenchmark: best-of-3 full-chip LDS.128 bytes/s --
 * the roof of the scaling-domain batched solve (4 B of kernel per cell per
 * half-step from shared memory). */
int otk_bench_smem(double *bytes_per_s, void *stream);

/* Whole solve_sinkhorn (sinkhorn.py:122-200) on device.  Returns OTK_OK,
 * OTK_DIVERGED (fail_iter = t) or OTK_BAD_POTENTIAL (fail_iter = t).
 * Small FP32-path problems with a constant eps (both point sets fit in one
 * SM's shared memory, d <= 7) run as ONE persistent cooperative kernel
 * (grid-wide barriers between half-steps, fused check, launches = 1);
 * everything else runs the general loop (CUDA graphs per check period). */
int otk_solve_pointcloud(otk_solve_args *args);

/* Row-sharded whole solve, one rank per GPU: args describes
 * THIS rank's rows (x, n, a, log_a: the shard; y, b, log_b, g_init:
 * replicated; flags must include OTK_IMPL_NOPERSIST).  The g half-step's
 * column partials and the check sums travel through xchg (epoch 0) -- the
 * same loop, outputs and error outcomes as otk_solve_pointcloud, identical g
 * and check trace on every rank, no host collective, one host sync per
 * check, CUDA-graph check periods.  split_scale: the common operand scale
 * (otk_split_scale of the max |coordinate| over ALL ranks; <= 0 = this
 * rank's own).  Returns OTK_ENCCL when a peer did not answer within
 * timeout_ms (0 = 10 s) -- on every rank at the same check. */
int otk_solve_pointcloud_sharded(otk_solve_args *args, const otk_exchange *xchg,
                                 float split_scale, uint32_t timeout_ms);

#ifdef __cplusplus
}
#endif
#endif /* OTK_H */
