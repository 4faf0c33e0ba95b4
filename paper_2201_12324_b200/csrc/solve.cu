// Half-step dispatch (K1 SIMT / K2 tcgen05) and the native solver loop that
// replaces the reference's Python loop sinkhorn._sinkhorn_iterations
// (reference sinkhorn.py:151-200) for point clouds.
//
// Loop (t = 1..max_iters, eps_t from the schedule, kappa = log2(e)/eps_t):
//   f-half  h=2t-1: partial = LSE over y of (2k<x,y> + bias_y);  f = finalize(log a)
//   g-half  h=2t  : partial = LSE over x of (2k<y,x> + bias_x);  g = finalize(log b)
// Every finalize also writes the bias of its side for the next half-step and
// records the first half-step index h that would CONSUME a NaN/+inf
// potential; the reference raises ValueError at exactly that call
// (geometry.py:65-72, via apply_lse_kernel).  At a check iteration
// (t % inner == 0 or t == max_iters, sinkhorn.py:175) the next f half-step
// f_{t+1} is computed into a second buffer and the fused check kernel
// derives the row marginal r_i = a_i exp((f_t - f_{t+1})/eps), which equals
// exp(apply_lse_kernel(f_t, g_t, rows)/eps) (sinkhorn.py:183): the third
// full pass of the reference is folded into the next iteration's work.
// Constant-eps check periods are captured once as CUDA graphs and replayed.
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <vector>

#include "otk_common.cuh"

namespace otk {
int lse_simt_launch(const float *p, const float *p_sq, int64_t np, const float *q,
                    const float *q_sq, int64_t nq, int d, const float *q_bias, float kappa,
                    int flags, int nsplit, float *partial, cudaStream_t st);
int lse_tc_launch(const uint16_t *p_hi, const uint16_t *p_lo, const uint16_t *p_ext, int64_t np,
                  const uint16_t *q_hi, const uint16_t *q_lo, const uint16_t *q_ext, int64_t nq,
                  int dpad, float two_kappa_scaled, const float *q_bias, int nsplit, int same,
                  int eucl, float *partial, const float *anchor, int *repair_ws, int repair,
                  cudaStream_t st);
bool tc_available();
int tc_tile_cols(int dpad);
int tc_uses_pair(int dpad);
namespace small {
struct Args {  // solve_small.cu
  const float *x, *y, *a, *b, *la, *lb, *g_init;
  int n, m, d;
  float eps, kappa;
  double eps_d, threshold;
  int max_iters, inner_iters, max_checks;
  float *f0, *f1, *g, *f_out, *g_out;
  float *f_host, *g_host;
  double *slots;
  double *errors, *duals;
  int *state;
  int probe;
  unsigned long long *xch_x, *xch_y;
  float4 *pts;
  unsigned long long *trace;
  int trace_steps;
};
constexpr int SLOT = 20;
}  // namespace small
bool small_solve_fits(int64_t n, int64_t m, int d);
int small_solve_launch(const small::Args &A, bool same, bool eucl, cudaStream_t st);
}  // namespace otk

using namespace otk;

#define OTK_TRY_(expr)           \
  do {                           \
    int _r = (expr);             \
    if (_r != OTK_OK) return _r; \
  } while (0)

// tcgen05 kernel for every d (measured on B200 at n = m = 65536, ncu in
// profiles/r01_ncu_route_*.txt: 1.40 ms per half-step at d = 3 and 1.50 ms at
// d = 64, vs 2.27 ms for the FP32 low-d kernel at d = 3 -- issue-bound, 81 %
// issue / 52 % MUFU -- and 6.4 ms for the tiled FP32 kernel at d = 16).  The
// FP32 kernels remain for OTK_IMPL_SIMT and inside the persistent small-problem
// solve (solve_small.cu), which the solver prefers whenever it fits.
constexpr int kTcMinDim = 1;
static bool want_tc(int flags, int d) {
  if (flags & OTK_IMPL_SIMT) return false;
  if (flags & OTK_IMPL_TC) return true;
  return tc_available() && d >= kTcMinDim;
}

extern "C" int otk_lse_uses_tc(int32_t d, int32_t flags) { return want_tc(flags, d) ? 1 : 0; }

// Column-split count for the persistent TC kernel.  Its work units are
// (row tile [pair]) x (column split), dealt round-robin to min(units, SMs
// [/2]) CTAs [clusters]; the slowest CTA sets the half-step time.  Pick the
// split count (1..16) with the best modelled makespan: tiles of the busiest
// CTA plus a per-unit switch cost of ~0.4 tile (measured on B200 at cfg2:
// nsplit 1 / 2 / 3 / 4 / 8 -> 1.53 / 1.38 / 1.43 / 1.39 / 1.39 ms, i.e. 86 /
// 99 / 94 / 99 / 99 % balance).  Ties go to fewer splits (smaller partials).
static int tc_balanced_nsplit(int64_t np, int64_t nq, int dpad) {
  static std::mutex mu;
  static std::map<std::tuple<int64_t, int64_t, int>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(np, nq, dpad);
  if (auto it = cache.find(key); it != cache.end()) return it->second;
  const int bn = tc_tile_cols(dpad);
  const bool pair = tc_uses_pair(dpad) != 0;
  const int64_t row_tiles = (np + 127) / 128;
  const int64_t rows_units = pair ? (row_tiles + 1) / 2 : row_tiles;
  const int64_t ntiles = (nq + bn - 1) / bn;
  const int64_t slots = pair ? num_sms() / 2 : num_sms();
  int best = 1;
  double best_cost = 1e300;
  for (int ns = 1; ns <= 16 && ns <= ntiles; ++ns) {
    const int64_t tps = (ntiles + ns - 1) / ns;
    if ((ns - 1) * tps >= ntiles) continue;  // an empty split
    const int64_t units = rows_units * ns;
    const int64_t G = std::min<int64_t>(units, slots);
    double worst = 0.0;
    for (int64_t c = 0; c < G; ++c) {  // CTA c takes units c, c + G, ...
      double t = 0.0;
      for (int64_t u = c; u < units; u += G) {
        const int64_t split = u / rows_units;
        t += (double)(std::min(ntiles, (split + 1) * tps) - split * tps) + 0.4;
      }
      worst = std::max(worst, t);
    }
    if (worst < best_cost * (1.0 - 1e-9)) {
      best_cost = worst;
      best = ns;
    }
  }
  cache.emplace(key, best);
  return best;
}

extern "C" int otk_lse_suggest_nsplit(int64_t np, int64_t nq, int32_t d, int32_t flags) {
  const int sms = num_sms();
  if (want_tc(flags, d)) {
    if (const char *e = getenv("OTK_TC_NSPLIT")) return std::max(1, atoi(e));  // A/B knob
    return tc_balanced_nsplit(np, nq, (d + 63) / 64 * 64);
  }
  int64_t row_tiles = (np + 63) / 64;
  int64_t col_tiles = (nq + 63) / 64;
  int64_t want = (16LL * sms + row_tiles - 1) / row_tiles;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, col_tiles));
}

extern "C" int otk_lse_partial(const float *p, const float *p_sq, const uint16_t *p_hi,
                               const uint16_t *p_lo, const uint16_t *p_ext, int64_t np,
                               const float *q, const float *q_sq, const uint16_t *q_hi,
                               const uint16_t *q_lo, const uint16_t *q_ext, int64_t nq, int32_t d,
                               int32_t dpad, float split_inv, const float *q_bias, float kappa,
                               int32_t flags, int32_t nsplit, float *partial, void *stream) {
  OTK_CHECK_ARG(np > 0 && nq > 0 && d > 0 && nsplit >= 1 && q_bias && partial,
                "otk_lse_partial: bad arguments");
  OTK_CHECK_ARG(nsplit <= 65535, "otk_lse_partial: nsplit too large");
  if (want_tc(flags, d)) {
    OTK_CHECK_ARG(p_hi && p_lo && p_ext && q_hi && q_lo && q_ext && dpad % 64 == 0 && dpad >= d,
                  "otk_lse_partial: TC path needs split + norm planes with dpad %% 64 == 0");
    if (!tc_available()) {
      set_error("otk_lse_partial: tcgen05 path requires an sm_100 device");
      return OTK_ENOTSUP;
    }
    // sqeucl: u = (2 kappa / s^2) acc + bias with acc = -s^2 C / 2;
    // eucl:   u = -(kappa sqrt(2) / s) sqrt(max(-acc, 0)) + bias
    const bool eu = flags & OTK_COST_EUCL;
    const float scale = eu ? -kappa * sqrtf(2.f * split_inv) : 2.f * kappa * split_inv;
    return lse_tc_launch(p_hi, p_lo, p_ext, np, q_hi, q_lo, q_ext, nq, dpad, scale, q_bias, nsplit,
                         (flags & OTK_SAME_POINTS) ? 1 : 0, eu ? 1 : 0, partial, nullptr, nullptr, 0,
                         as_stream(stream));
  }
  OTK_CHECK_ARG(p && q && p_sq && q_sq, "otk_lse_partial: FP32 path needs points and squared norms");
  return lse_simt_launch(p, p_sq, np, q, q_sq, nq, d, q_bias, kappa, flags, nsplit, partial,
                         as_stream(stream));
}

static bool anchored_path(int32_t d, int32_t flags) {
  return want_tc(flags, d) && tc_available() && !(flags & (OTK_COST_EUCL | OTK_IMPL_NOANCHOR));
}

// The anchored step costs two extra small launches per half-step (~10 us);
// it pays off only where the half-step itself is long (measured gain ~7 % of
// the TC kernel at cfg2; break-even near 10^4 x 10^4): default threshold
// 2^27 cells (np * nq), override
// with OTK_ANCHOR_MIN_CELLS.
extern "C" int otk_lse_step_anchored(int64_t np, int64_t nq, int32_t d, int32_t flags) {
  if (!anchored_path(d, flags)) return 0;
  double min_cells = 134217728.0;
  if (const char *e = getenv("OTK_ANCHOR_MIN_CELLS")) min_cells = atof(e);
  return (double)np * (double)nq >= min_cells ? 1 : 0;
}

extern "C" size_t otk_lse_step_workspace_bytes(int64_t np) {
  return (size_t)(((np + 127) / 128) + 2) * sizeof(int32_t);
}

// One whole half-step: otk_lse_partial + otk_lse_finalize, anchored on the TC
// sqeucl path.  Launch sequence when anchored (4 launches, graph-capturable,
// no host decision): anchored partial -> finalize_anchored (accepts rows in
// the safe window, flags the tiles of the others) -> running-max partial over
// the flagged tiles only (exits at once when none) -> finalize_repair.
extern "C" int otk_lse_step(const float *p, const float *p_sq, const uint16_t *p_hi,
                            const uint16_t *p_lo, const uint16_t *p_ext, int64_t np,
                            const float *q, const float *q_sq, const uint16_t *q_hi,
                            const uint16_t *q_lo, const uint16_t *q_ext, int64_t nq, int32_t d,
                            int32_t dpad, float split_inv, const float *q_bias, float kappa,
                            int32_t flags, int32_t nsplit, float *partial, const float *base,
                            int32_t mode, float eps, float kappa_next, float *out_pot,
                            float *out_bias, int32_t *first_bad, int32_t step, float *anchor,
                            int32_t *repair_ws, const otk_exchange *xchg, void *stream) {
  OTK_CHECK_ARG(partial && out_pot && np > 0 && nq > 0 && nsplit >= 1, "otk_lse_step: bad arguments");
  OTK_CHECK_ARG(!xchg || (xchg->local && xchg->world >= 1 && xchg->rank >= 0 &&
                          xchg->rank < xchg->world && mode == OTK_FIN_LOG2),
                "otk_lse_step: the exchange needs OTK_FIN_LOG2 and a valid otk_exchange");
  OTK_CHECK_ARG(mode == OTK_FIN_SOLVER || mode == OTK_FIN_APPLY || mode == OTK_FIN_LOG2,
                "otk_lse_step: bad mode");
  OTK_CHECK_ARG(base || mode == OTK_FIN_LOG2, "otk_lse_step: base required");
  cudaStream_t st = as_stream(stream);
  FinArgs F{partial, nsplit, np, base, mode, eps, kappa_next, out_pot, out_bias, first_bad, step,
            anchor, repair_ws, 0.f, nullptr, 0, 0, 0u};
  FinArgs Fx = F;  // the half-step's LAST finalize also pushes to the peers
  if (xchg) {
    Fx.xlocal = static_cast<char *>(xchg->local);
    Fx.xworld = xchg->world;
    Fx.xrank = xchg->rank;
    Fx.xepoch = xchg->epoch;
  }
  const bool anch = anchor != nullptr && !(flags & OTK_ANCHOR_INIT) && anchored_path(d, flags);
  if (!anch) {
    OTK_TRY_(otk_lse_partial(p, p_sq, p_hi, p_lo, p_ext, np, q, q_sq, q_hi, q_lo, q_ext, nq, d, dpad,
                             split_inv, q_bias, kappa, flags, nsplit, partial, stream));
    return finalize_launch(0, Fx, st);
  }
  OTK_CHECK_ARG(repair_ws && p_hi && p_lo && p_ext && q_hi && q_lo && q_ext && dpad % 64 == 0 && dpad >= d,
                "otk_lse_step: anchored path needs the repair workspace and the split + norm planes");
  // flushed mass <= nq^2 2^(-126 - (L - anchor)) of the row's sum: <= 2^-30 for L - anchor >= lo
  F.lo = -96.f + 2.f * log2f((float)nq);
  const float scale = 2.f * kappa * split_inv;
  const int same = (flags & OTK_SAME_POINTS) ? 1 : 0;
  OTK_TRY_(lse_tc_launch(p_hi, p_lo, p_ext, np, q_hi, q_lo, q_ext, nq, dpad, scale, q_bias, nsplit,
                         same, 0, partial, anchor, repair_ws, 0, st));
  OTK_TRY_(finalize_launch(1, F, st));
  OTK_TRY_(lse_tc_launch(p_hi, p_lo, p_ext, np, q_hi, q_lo, q_ext, nq, dpad, scale, q_bias, nsplit,
                         same, 0, partial, nullptr, repair_ws, 1, st));
  return finalize_launch(2, Fx, st);
}

// ------------------------------------------------------------------ solver
namespace {

struct Carver {
  char *base;
  size_t off = 0;
  template <class T>
  T *take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
};

struct Layout {
  float *fA, *fB, *g, *xsq, *ysq, *bias_x, *bias_y, *part;
  float *lcol;                // sharded solve: this shard's log2 column partials
  double *chk_tot;            // sharded solve: rank-order check totals (10 values)
  float *anc_x, *anc_y;       // anchors of the rows / cols half-steps (otk_lse_step)
  int *rep_x, *rep_y;         // their repair workspaces
  uint16_t *xhi, *xlo, *yhi, *ylo, *xea, *xeb, *yea, *yeb;
  float *absmax;
  double *chk;
  void *chk_ws;
  int *first_bad;
  double *slots, *d_errors, *d_duals;  // persistent small-problem kernel
  unsigned long long *xch;
  float4 *pts;
  int *state;
  int nsr, nsc, dpad;
  bool tc, small;
  size_t bytes;
};

// Whole-solve persistent kernel (solve_small.cu): FP32 path, constant eps; d <= 19 within
// its cell budget, or any d <= 512 for up to 2048 points a side while the stored-kernel
// builds pay off (small_solve_fits).  OTK_IMPL_NOPERSIST / OTK_IMPL_TC force the general loop.
static bool use_small(const otk_solve_args *A) {
  if (A->flags & (OTK_IMPL_TC | OTK_IMPL_NOPERSIST)) return false;
  if (!(A->eps_init_scale <= 1.0)) return false;  // eps_t == target for every t
  return small_solve_fits(A->n, A->m, A->d);
}

Layout plan(const otk_solve_args *A, void *ws) {
  Layout L{};
  L.small = use_small(A);
  L.tc = !L.small && want_tc(A->flags, A->d);
  L.dpad = (A->d + 63) / 64 * 64;
  L.nsr = otk_lse_suggest_nsplit(A->n, A->m, A->d, A->flags);
  L.nsc = otk_lse_suggest_nsplit(A->m, A->n, A->d, A->flags);
  Carver c{reinterpret_cast<char *>(ws)};
  L.fA = c.take<float>(A->n);
  L.fB = c.take<float>(A->n);
  L.g = c.take<float>(A->m);
  L.xsq = c.take<float>(A->n);
  L.ysq = c.take<float>(A->m);
  L.bias_x = c.take<float>(A->n);
  L.bias_y = c.take<float>(A->m);
  L.part = c.take<float>(std::max((size_t)L.nsr * A->n, (size_t)L.nsc * A->m));
  L.lcol = c.take<float>(A->m);
  L.chk_tot = c.take<double>(16);
  L.anc_x = c.take<float>(A->n);
  L.anc_y = c.take<float>(A->m);
  L.rep_x = reinterpret_cast<int *>(c.take<char>(otk_lse_step_workspace_bytes(A->n)));
  L.rep_y = reinterpret_cast<int *>(c.take<char>(otk_lse_step_workspace_bytes(A->m)));
  if (L.tc) {
    L.xhi = c.take<uint16_t>((size_t)A->n * L.dpad);
    L.xlo = c.take<uint16_t>((size_t)A->n * L.dpad);
    L.yhi = c.take<uint16_t>((size_t)A->m * L.dpad);
    L.ylo = c.take<uint16_t>((size_t)A->m * L.dpad);
    L.xea = c.take<uint16_t>((size_t)A->n * 16);
    L.xeb = c.take<uint16_t>((size_t)A->n * 16);
    L.yea = c.take<uint16_t>((size_t)A->m * 16);
    L.yeb = c.take<uint16_t>((size_t)A->m * 16);
  } else {
    L.xhi = L.xlo = L.yhi = L.ylo = L.xea = L.xeb = L.yea = L.yeb = nullptr;
  }
  L.absmax = c.take<float>(2);
  L.chk = c.take<double>(8);
  L.chk_ws = c.take<char>(otk_check_workspace_bytes());
  L.first_bad = c.take<int>(1);
  if (L.small) {
    L.slots = c.take<double>((size_t)2 * num_sms() * small::SLOT + 2);  // + 2 decision words
    L.d_errors = c.take<double>(A->max_checks);
    L.d_duals = c.take<double>(A->max_checks);
    L.state = c.take<int>(8);
    L.xch = c.take<unsigned long long>(2 * (size_t)(A->n + A->m));
    // d >= 8: staged points (<= 5 float4 each); d > 19 and not a multiple of 4: both sets with rows
    // padded to a multiple of 4 coordinates (128-bit loads in the exact passes)
    L.pts = c.take<float4>((size_t)(A->n + A->m) * std::max(5, (A->d + 3) / 4));
  }
  L.bytes = c.off + 256;
  return L;
}

inline double eps_at(const otk_solve_args *A, int t) {
  return std::max(A->eps_target, A->eps_target * A->eps_init_scale * std::pow(A->eps_decay, (double)t));
}

}  // namespace

extern "C" size_t otk_solve_workspace_bytes(const otk_solve_args *A) {
  if (!A) return 0;
  return plan(A, nullptr).bytes;
}

#define OTK_TRY(expr)          \
  do {                         \
    int _r = (expr);           \
    if (_r != OTK_OK) return _r; \
  } while (0)

// Row-sharded solve (otk_solve_pointcloud_sharded): this rank holds rows
// [lo, lo + n) of x; the g half-step's column partials go to every rank
// through the peer-memory exchange (p2p.cu) and the check sums likewise.
struct ShardCtx {
  otk_exchange x;       // epoch 0: device-counted (graph-replayable)
  int64_t m;
  uint32_t timeout_ms;
};

// Half-steps go through otk_lse_step: the first of each role runs the
// running-max kernel and records the per-row anchors, every later one is
// anchored (TC sqeucl path; OTK_IMPL_NOANCHOR disables it).
struct HalfStep {
  const otk_solve_args *A;
  Layout *L;
  cudaStream_t st;
  float sinv;  // 1/s^2 for the TC operand scaling (one common scale s)
  int kflags;
  bool anchored;  // anchored path available for this problem
  const ShardCtx *sh = nullptr;
  int launches = 0;
  bool have_x = false, have_y = false;

  int rows(float kappa, float eps, float kappa_next, float *f_out, int step) {
    NvtxRange r("otk f half-step");
    const int fl = kflags | (have_x ? 0 : OTK_ANCHOR_INIT);
    launches += (anchored && have_x) ? 4 : 2;
    have_x = true;
    return otk_lse_step(A->x, L->xsq, L->xhi, L->xlo, L->xea, A->n, A->y, L->ysq, L->yhi, L->ylo,
                        L->yeb, A->m, A->d, L->dpad, sinv, L->bias_y, kappa, fl, L->nsr, L->part,
                        A->log_a, OTK_FIN_SOLVER, eps, kappa_next, f_out, L->bias_x, L->first_bad,
                        step, anchored ? L->anc_x : nullptr, L->rep_x, nullptr, st);
  }
  int cols(float kappa, float eps, float kappa_next, int step) {
    NvtxRange r("otk g half-step");
    const int fl = kflags | (have_y ? 0 : OTK_ANCHOR_INIT);
    launches += (anchored && have_y) ? 4 : 2;
    have_y = true;
    if (sh == nullptr)
      return otk_lse_step(A->y, L->ysq, L->yhi, L->ylo, L->yea, A->m, A->x, L->xsq, L->xhi, L->xlo,
                          L->xeb, A->n, A->d, L->dpad, sinv, L->bias_x, kappa, fl, L->nsc, L->part,
                          A->log_b, OTK_FIN_SOLVER, eps, kappa_next, L->g, L->bias_y, L->first_bad,
                          step, anchored ? L->anc_y : nullptr, L->rep_y, nullptr, st);
    // this shard's log2 partial per column (anchored on the shard's own previous
    // partials), pushed to every rank by the half-step's last kernel; then the W
    // partials of every column combined in rank order into g
    int rc = otk_lse_step(A->y, L->ysq, L->yhi, L->ylo, L->yea, A->m, A->x, L->xsq, L->xhi, L->xlo,
                          L->xeb, A->n, A->d, L->dpad, sinv, L->bias_x, kappa, fl, L->nsc, L->part,
                          nullptr, OTK_FIN_LOG2, 0.f, 0.f, L->lcol, nullptr, nullptr, 0,
                          anchored ? L->anc_y : nullptr, L->rep_y, &sh->x, st);
    if (rc != OTK_OK) return rc;
    launches += 1;
    NvtxRange rx("otk g exchange combine");
    return otk_exchange_finalize(sh->x.local, sh->x.world, A->m, 0u, A->log_b, OTK_FIN_SOLVER, eps,
                                 kappa_next, L->g, L->bias_y, L->first_bad, step, sh->timeout_ms, st);
  }

  // The fused check of this rank's rows; sharded: + the rank-order exchange
  // of the sums.  The host reads `out` (8 sums; sharded: [8] = first bad
  // step of any rank, [9] = exchange error) after one stream sync.
  int check(const float *f, const float *fn, double eps) {
    NvtxRange r("otk check");
    int rc = otk_check(f, fn, A->a, A->n, L->g, A->b, A->m, eps, L->chk, L->chk_ws, st);
    if (rc != OTK_OK || sh == nullptr) return rc;
    launches += 1;
    return otk_exchange_check(sh->x.local, sh->x.world, sh->x.rank, A->m, L->chk, L->first_bad,
                              L->chk_tot, sh->timeout_ms, st);
  }
  const double *check_result() const { return sh ? L->chk_tot : L->chk; }
};


static int solve_on_stream(otk_solve_args *A, Layout &L, cudaStream_t st, const ShardCtx *sh = nullptr,
                           float split_scale = 0.f);

static int solve_entry(otk_solve_args *A, const ShardCtx *sh, float split_scale);

extern "C" int otk_solve_pointcloud(otk_solve_args *A) { return solve_entry(A, nullptr, 0.f); }

// Row-sharded whole solve: A describes THIS rank's rows (x, n, a, log_a are
// the shard's; y, b, log_b, g_init are replicated).  Same loop and outputs as
// otk_solve_pointcloud, with the g half-step's column partials and the check
// sums exchanged over peer memory (p2p.cu) -- no host collective; one host
// sync per check; constant-eps check periods replayed as CUDA graphs (the
// exchange epochs are device-counted).  g_out and the check trace are
// identical on every rank; a world-1 exchange is bitwise equal to
// otk_solve_pointcloud's general loop.
extern "C" int otk_solve_pointcloud_sharded(otk_solve_args *A, const otk_exchange *xchg,
                                            float split_scale, uint32_t timeout_ms) {
  OTK_CHECK_ARG(xchg && xchg->local && xchg->world >= 1 && xchg->rank >= 0 &&
                    xchg->rank < xchg->world && xchg->epoch == 0u,
                "otk_solve_pointcloud_sharded: bad exchange (epoch must be 0: device-counted)");
  OTK_CHECK_ARG(A && (A->flags & OTK_IMPL_NOPERSIST) && A->same_points == 0,
                "otk_solve_pointcloud_sharded: needs OTK_IMPL_NOPERSIST and distinct point sets");
  ShardCtx sh{*xchg, A->m, timeout_ms};
  return solve_entry(A, &sh, split_scale);
}

static int solve_entry(otk_solve_args *A, const ShardCtx *sh, float split_scale) {
  OTK_CHECK_ARG(A && A->x && A->y && A->a && A->b && A->log_a && A->log_b && A->f_out && A->g_out,
                "otk_solve_pointcloud: missing pointers");
  OTK_CHECK_ARG(A->n > 0 && A->m > 0 && A->d > 0, "otk_solve_pointcloud: bad shape");
  OTK_CHECK_ARG(A->max_iters >= 1 && A->inner_iters >= 1, "max_iters and inner_iters must be >= 1");
  // a negative threshold never stops the loop early (fixed-iteration measurement runs)
  OTK_CHECK_ARG(A->threshold > 0 || A->threshold < 0, "threshold must be positive (or negative: never stop early)");
  OTK_CHECK_ARG(A->eps_target > 0, "eps must be positive");
  OTK_CHECK_ARG(A->errors && A->duals && A->max_checks >= 1, "otk_solve_pointcloud: no trace buffers");
  Layout L = plan(A, A->workspace);
  OTK_CHECK_ARG(A->workspace && A->workspace_bytes >= L.bytes,
                "otk_solve_pointcloud: workspace too small (%zu < %zu)", A->workspace_bytes, L.bytes);
  // Work runs on a private non-blocking stream ordered after the caller's
  // stream (graph capture is not allowed on the legacy default stream); the
  // stream and its two events are created once per host thread and device.
  struct Priv {
    int dev = -1;
    cudaStream_t st = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  };
  static thread_local Priv priv;
  int dev = 0;
  OTK_CUDA(cudaGetDevice(&dev));
  if (priv.dev != dev) {
    if (priv.st) {
      cudaEventDestroy(priv.ev_in);
      cudaEventDestroy(priv.ev_out);
      cudaStreamDestroy(priv.st);
      priv.st = nullptr;
    }
    OTK_CUDA(cudaStreamCreateWithFlags(&priv.st, cudaStreamNonBlocking));
    OTK_CUDA(cudaEventCreateWithFlags(&priv.ev_in, cudaEventDisableTiming));
    OTK_CUDA(cudaEventCreateWithFlags(&priv.ev_out, cudaEventDisableTiming));
    priv.dev = dev;
  }
  cudaStream_t caller = as_stream(A->stream);
  cudaStream_t st = priv.st;
  OTK_CUDA(cudaEventRecord(priv.ev_in, caller));
  OTK_CUDA(cudaStreamWaitEvent(st, priv.ev_in, 0));
  int rc = solve_on_stream(A, L, st, sh, split_scale);
  cudaEventRecord(priv.ev_out, st);
  cudaStreamWaitEvent(caller, priv.ev_out, 0);
  cudaStreamSynchronize(st);
  return rc;
}

static int solve_small(otk_solve_args *A, Layout &L, cudaStream_t st) {
  small::Args S{};
  S.x = A->x;
  S.y = A->y;
  S.a = A->a;
  S.b = A->b;
  S.la = A->log_a;
  S.lb = A->log_b;
  S.g_init = A->g_init;
  S.n = (int)A->n;
  S.m = (int)A->m;
  S.d = A->d;
  S.eps = (float)A->eps_target;
  S.kappa = (float)(1.4426950408889634 / A->eps_target);
  S.eps_d = A->eps_target;
  S.threshold = A->threshold;
  S.max_iters = A->max_iters;
  S.inner_iters = A->inner_iters;
  S.max_checks = A->max_checks;
  S.f0 = L.fA;
  S.f1 = L.fB;
  S.g = L.g;
  S.f_out = A->f_out;
  S.g_out = A->g_out;
  S.slots = L.slots;
  // results block in pinned host memory (per host thread, grown on demand):
  // [8 ints of state | errors | duals], written by the kernel itself
  struct HostRes {
    char *p = nullptr;
    size_t bytes = 0;
  };
  static thread_local HostRes hres;
  const size_t need = 64 + 2 * (size_t)A->max_checks * sizeof(double);
  if (hres.bytes < need) {
    if (hres.p) cudaFreeHost(hres.p);
    hres.p = nullptr;
    hres.bytes = 0;
    OTK_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&hres.p), need, cudaHostAllocDefault));
    hres.bytes = need;
  }
  double *h_err = reinterpret_cast<double *>(hres.p + 64);
  double *h_dual = h_err + A->max_checks;
  S.errors = h_err;
  S.duals = h_dual;
  S.state = reinterpret_cast<int *>(hres.p);
  std::memset(hres.p, 0, 64);
  auto pinned = [](const void *p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  S.f_host = (A->f_host && pinned(A->f_host)) ? A->f_host : nullptr;
  S.g_host = (A->g_host && pinned(A->g_host)) ? A->g_host : nullptr;
  S.probe = getenv("OTK_SMALL_PROBE") ? atoi(getenv("OTK_SMALL_PROBE")) : 0;
  S.xch_x = L.xch;
  S.xch_y = L.xch + 2 * A->n;
  S.pts = L.pts;
  const char *trace_path = getenv("OTK_SMALL_TRACE");  // diagnostics: per-CTA phase stamps
  if (trace_path) {
    S.trace_steps = 64;
    OTK_CUDA(cudaMalloc(&S.trace, (size_t)S.trace_steps * num_sms() * 8 * sizeof(unsigned long long)));
    OTK_CUDA(cudaMemsetAsync(S.trace, 0, (size_t)S.trace_steps * num_sms() * 8 * sizeof(unsigned long long), st));
  }
  OTK_TRY(small_solve_launch(S, A->same_points != 0, (A->flags & OTK_COST_EUCL) != 0, st));
  if (trace_path) {
    std::vector<unsigned long long> h((size_t)S.trace_steps * num_sms() * 8);
    OTK_CUDA(cudaMemcpyAsync(h.data(), S.trace, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost, st));
    OTK_CUDA(cudaStreamSynchronize(st));
    cudaFree(S.trace);
    if (FILE *fp = fopen(trace_path, "wb")) {
      fwrite(h.data(), sizeof(h[0]), h.size(), fp);
      fclose(fp);
    }
  }
  // one synchronisation and no copy calls: the kernel wrote its state, the
  // check trace and (when the caller's buffers are pinned) f, g straight into
  // host memory
  OTK_CUDA(cudaStreamSynchronize(st));
  if (A->f_host && !S.f_host)
    OTK_CUDA(cudaMemcpyAsync(A->f_host, A->f_out, A->n * sizeof(float), cudaMemcpyDeviceToHost, st));
  if (A->g_host && !S.g_host)
    OTK_CUDA(cudaMemcpyAsync(A->g_host, A->g_out, A->m * sizeof(float), cudaMemcpyDeviceToHost, st));
  if ((A->f_host && !S.f_host) || (A->g_host && !S.g_host)) OTK_CUDA(cudaStreamSynchronize(st));
  const int *state = reinterpret_cast<const int *>(hres.p);
  if (getenv("OTK_SMALL_DEBUG"))  // builds are counted by -DOTK_SMALL_COUNT_BUILDS libraries only (else 0 0)
    fprintf(stderr, "solve_small: %d iterations, stored-kernel builds of CTA 0: x role %d, y role %d\n", state[1],
            state[5], state[6]);
  const int nc = std::min(state[0], A->max_checks);
  std::memcpy(A->errors, h_err, (size_t)nc * sizeof(double));
  std::memcpy(A->duals, h_dual, (size_t)nc * sizeof(double));
  A->n_checks = nc;
  A->iterations = state[1];
  A->converged = state[2];
  A->fail_iter = state[4];
  A->launches = 1;
  return state[3];
}

// Host view of one check: the 8 sums of sinkhorn.py:183-186 + the first bad
// step; sharded: the rank-order totals, any rank's first bad step and the
// exchange error word, all from one D2H read after one stream sync.
struct CheckRead {
  double v[10];
  int fb;
};
static int read_check(const HalfStep &H, Layout &L, cudaStream_t st, CheckRead *cr) {
  if (H.sh) {
    OTK_CUDA(cudaMemcpyAsync(cr->v, L.chk_tot, sizeof(cr->v), cudaMemcpyDeviceToHost, st));
    OTK_CUDA(cudaStreamSynchronize(st));
    cr->fb = (int)cr->v[8];
    if (cr->v[9] != 0.0) {
      set_error("peer-memory exchange timed out waiting for another rank");
      return OTK_ENCCL;
    }
    return OTK_OK;
  }
  OTK_CUDA(cudaMemcpyAsync(cr->v, L.chk, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
  OTK_CUDA(cudaMemcpyAsync(&cr->fb, L.first_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  OTK_CUDA(cudaStreamSynchronize(st));
  return OTK_OK;
}

static int solve_on_stream(otk_solve_args *A, Layout &L, cudaStream_t st, const ShardCtx *sh,
                           float split_scale) {
  NvtxRange range(sh ? "otk_solve_pointcloud_sharded" : "otk_solve_pointcloud");
  A->n_checks = 0;
  A->iterations = 0;
  A->converged = 0;
  A->fail_iter = 0;
  if (L.small) return solve_small(A, L, st);

  // ---- prep (K0)
  float s = 1.f;  // one common power-of-two operand scale for x and y
  if (L.tc && split_scale > 0.f) {
    s = split_scale;  // sharded: common to every rank (from the global |coordinate| max)
  } else if (L.tc) {
    float amax[2];
    OTK_TRY(otk_absmax(A->x, A->n * (int64_t)A->d, L.absmax, st));
    OTK_TRY(otk_absmax(A->y, A->m * (int64_t)A->d, L.absmax + 1, st));
    OTK_CUDA(cudaMemcpyAsync(amax, L.absmax, sizeof(amax), cudaMemcpyDeviceToHost, st));
    OTK_CUDA(cudaStreamSynchronize(st));
    s = otk_split_scale(std::max(amax[0], amax[1]), A->d);
  }
  OTK_TRY(otk_prep_points(A->x, A->n, A->d, L.xsq, L.xhi, L.xlo, L.xea, L.xeb, L.dpad, s, st));
  OTK_TRY(otk_prep_points(A->y, A->m, A->d, L.ysq, L.yhi, L.ylo, L.yea, L.yeb, L.dpad, s, st));
  OTK_CUDA(cudaMemsetAsync(L.first_bad, 0x7f, sizeof(int), st));
  OTK_CUDA(cudaMemsetAsync(L.chk_ws, 0, otk_check_workspace_bytes(), st));

  HalfStep H{A, &L, st, 1.f / (s * s),
             (A->flags & (OTK_IMPL_SIMT | OTK_IMPL_TC | OTK_COST_EUCL)) | OTK_CLAMP |
                 (A->same_points ? OTK_SAME_POINTS : 0)};
  H.anchored = L.tc && !(A->flags & OTK_IMPL_NOANCHOR) && otk_lse_step_anchored(A->n, A->m, A->d, H.kflags);
  H.sh = sh;

  // ---- initial g (zeros or warm start) and its bias for h = 1
  const double e0 = eps_at(A, 0);
  if (A->g_init)
    OTK_CUDA(cudaMemcpyAsync(L.g, A->g_init, A->m * sizeof(float), cudaMemcpyDeviceToDevice, st));
  else
    OTK_CUDA(cudaMemsetAsync(L.g, 0, A->m * sizeof(float), st));
  OTK_TRY(otk_make_bias(L.g, A->m, (float)(1.4426950408889634 / e0), L.bias_y, L.first_bad, 1, st));

  float *f = L.fA, *fn = L.fB;
  bool f_ready = false;
  int t = 0;
  int status = OTK_OK;

  // CUDA graph cache for a constant-eps period (f/fn ping-pong -> 2 graphs)
  cudaGraphExec_t period_exec[2] = {nullptr, nullptr};
  int graph_launches = 0;
  const bool graphs = A->use_graphs != 0;
  int extra_launches = 2 + 1 + (L.tc ? 2 : 0);  // prep x/y, bias, absmax x/y

  for (t = 1; t <= A->max_iters; ++t) {
    const double e = eps_at(A, t - 1);
    const float kap = (float)(1.4426950408889634 / e);
    const float kap_next = (float)(1.4426950408889634 / eps_at(A, t));

    // Graph fast path: a whole constant-eps period t..t+inner-1 ending at a check.
    const int t_end = t + A->inner_iters - 1;
    if (graphs && f_ready && (t - 1) % A->inner_iters == 0 && t_end <= A->max_iters &&
        t_end % A->inner_iters == 0 && e == A->eps_target && eps_at(A, t_end) == A->eps_target) {
      const int which = (f == L.fA) ? 0 : 1;
      if (!period_exec[which]) {
        cudaGraph_t graph;
        OTK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        int rc = OTK_OK;
        const int before = H.launches;
        // steps are recorded relative; the bad-potential index is only used as a
        // "before the check" marker inside graphs (see below)
        for (int k = 0; k < A->inner_iters && rc == OTK_OK; ++k) {
          if (k > 0) rc = H.rows(kap, (float)e, kap, f, 2);
          if (rc == OTK_OK) rc = H.cols(kap, (float)e, kap, k + 1 == A->inner_iters ? 3 : 2);
        }
        if (rc == OTK_OK) rc = H.rows(kap, (float)e, kap, fn, 4);
        if (rc == OTK_OK) rc = H.check(f, fn, e);
        cudaError_t ce = cudaStreamEndCapture(st, &graph);
        graph_launches = H.launches - before + 1;
        H.launches = before;
        if (rc != OTK_OK) return rc;
        if (ce != cudaSuccess) return cuda_status(ce, "cudaStreamEndCapture");
        // Relative step ids inside the period: 2 = consumed before the check
        // (the reference raises ValueError there), 3 = g_t consumed by the
        // check itself, 4 = f_{t+1} (after the check).
        OTK_CUDA(cudaGraphInstantiate(&period_exec[which], graph, 0));
        cudaGraphDestroy(graph);
      }
      OTK_CUDA(cudaMemsetAsync(L.first_bad, 0x7f, sizeof(int), st));
      OTK_CUDA(cudaGraphLaunch(period_exec[which], st));
      extra_launches += graph_launches;
      t = t_end;
      CheckRead cr;
      if ((status = read_check(H, L, st, &cr)) != OTK_OK) break;
      const double *out = cr.v;
      const int fb = cr.fb;
      if (fb <= 2) { status = OTK_BAD_POTENTIAL; A->fail_iter = t; break; }
      if (out[4] > 0 || out[5] > 0) { status = OTK_DIVERGED; A->fail_iter = t; break; }
      if (out[7] > 0) { status = OTK_BAD_POTENTIAL; A->fail_iter = t; break; }
      const double err = out[0];
      const double dual = out[2] + out[3] - e * (out[1] - 1.0);
      if (A->n_checks < A->max_checks) {
        A->errors[A->n_checks] = err;
        A->duals[A->n_checks] = dual;
        A->n_checks++;
      }
      if (err <= A->threshold) { A->converged = 1; break; }
      if (t < A->max_iters) {
        std::swap(f, fn);
        f_ready = true;
      }
      // step ids inside graphs are relative; restore absolute numbering
      OTK_CUDA(cudaMemsetAsync(L.first_bad, 0x7f, sizeof(int), st));
      continue;
    }

    if (!f_ready) { if ((status = H.rows(kap, (float)e, kap, f, 2 * t)) != OTK_OK) break; }
    f_ready = false;
    if ((status = H.cols(kap, (float)e, kap_next, 2 * t + 1)) != OTK_OK) break;

    if (t % A->inner_iters == 0 || t == A->max_iters) {
      const bool measure = !(e > A->eps_target);
      if (measure) {
        if ((status = H.rows(kap, (float)e, kap, fn, 2 * t + 2)) != OTK_OK) break;
      }
      if ((status = H.check(f, measure ? fn : nullptr, e)) != OTK_OK) break;
      extra_launches += 1;
      CheckRead cr;
      if ((status = read_check(H, L, st, &cr)) != OTK_OK) break;
      const double *out = cr.v;
      const int fb = cr.fb;
      if (fb <= 2 * t) { status = OTK_BAD_POTENTIAL; A->fail_iter = (fb + 1) / 2; break; }
      if (out[4] > 0 || out[5] > 0) { status = OTK_DIVERGED; A->fail_iter = t; break; }
      if (!measure) continue;
      if (fb == 2 * t + 1) { status = OTK_BAD_POTENTIAL; A->fail_iter = t; break; }
      const double err = out[0];
      const double dual = out[2] + out[3] - e * (out[1] - 1.0);
      if (A->n_checks < A->max_checks) {
        A->errors[A->n_checks] = err;
        A->duals[A->n_checks] = dual;
        A->n_checks++;
      }
      if (err <= A->threshold) { A->converged = 1; break; }
      if (t < A->max_iters) {
        std::swap(f, fn);
        f_ready = true;
      }
    }
  }
  for (auto &ex : period_exec)
    if (ex) cudaGraphExecDestroy(ex);
  A->iterations = std::min(t, A->max_iters);
  A->launches = H.launches + extra_launches;
  if (status < 0) return status;
  OTK_CUDA(cudaMemcpyAsync(A->f_out, f, A->n * sizeof(float), cudaMemcpyDeviceToDevice, st));
  OTK_CUDA(cudaMemcpyAsync(A->g_out, L.g, A->m * sizeof(float), cudaMemcpyDeviceToDevice, st));
  if (A->f_host) OTK_CUDA(cudaMemcpyAsync(A->f_host, f, A->n * sizeof(float), cudaMemcpyDeviceToHost, st));
  if (A->g_host) OTK_CUDA(cudaMemcpyAsync(A->g_host, L.g, A->m * sizeof(float), cudaMemcpyDeviceToHost, st));
  OTK_CUDA(cudaStreamSynchronize(st));
  return status;
}
