// K2 -- online half-step on the 5th-generation tensor cores (sm_100a):
// tcgen05.mma with TMEM accumulators, TMA-staged shared memory, and a
// streaming log2-sum-exp2 epilogue read straight out of TMEM.
//
// Replaces PointCloudGeometry.apply_lse_kernel (reference geometry.py:336-354)
// for every d (solve.cu: want_tc).  Identical point sets: the split products
// leave C_ii at 0 only up to fp32 rounding (|C_ii| <~ 1e-6 |p_i|^2), so the
// same-points instantiation (epilogue mode EU == 2) forces the diagonal to an
// exact zero like the reference (geometry.py:278-292) with a per-register bit
// test; the default instantiation carries no such test.  Contract (include/otk.h, otk_lse_partial):
//     partial_i = log2 sum_j 2^(kappa*g_j - kappa*C_ij),  C_ij = |p_i|^2+|q_j|^2-2<p_i,q_j>
// The dot products run on the tensor cores in split-fp16 ("3xFP16"): every
// fp32 coordinate is pre-split (K0, otk_prep_points) into hi = fp16(s*x),
// lo = fp16(s*x - hi) with one power-of-two scale s for both point sets, and
//     s^2 <p,q> ~= hi_p.hi_q + hi_p.lo_q + lo_p.hi_q          (error ~2^-22)
// One more MMA per tile, issued last, adds -s^2(|p_i|^2 + |q_j|^2)/2 from the
// 16-column "norm planes" (three fp16 pieces per point times 2^15), so the
// accumulators end at -s^2 C_ij / 2 and the epilogue gets
//     u_ij = (2 kappa / s^2) * acc + kappa g_j = kappa (g_j - C_ij)
// from a single FFMA.
//
// Accuracy (measured, tools/diag_tc_bias.py): every tcgen05.mma rounds its
// fp32 accumulator toward zero (~0.3-0.5 ulp of the running sum), so a long
// chain of dot-product MMAs drifts low.  The chain is therefore split across
// several TMEM accumulators and summed in fp32 by the epilogue:
//   V1 (d <= 64):    1 accumulator, 2 tile buffers, 256-column tiles
//   V2 (d <= 256):   hi*hi | cross terms, 2 tile buffers, 128-column tiles
//   V4 (d  > 256):   hi*hi split over 3 accumulators (K-blocks round-robin) |
//                    cross terms, 1 tile buffer, 128-column tiles
// (TMEM holds 512 fp32 columns per SM: NACC * NBUF * BN = 512.)
//
// CTA = one SM, persistent over work units (row tile of 128 P rows) x
// (contiguous column split of Q).  Warp roles (384 threads):
//   warp 0      TMA producer: A (P hi/lo + norm plane, resident per unit when it
//               fits), B stages (Q hi/lo K-blocks, BN rows x 64 fp16, 128B
//               swizzle) and per-tile extras (kappa*g_j vector via 1-D TMA,
//               Q norm plane, 32B swizzle)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=BN, K=16, fp32 accumulate)
//   warps 4-11  two epilogue warpgroups: each thread owns one row (TMEM lane),
//               streams its columns with software-pipelined tcgen05.ld and
//               keeps an online (max, sum); with 2 tile buffers the groups
//               alternate tiles, with 1 buffer they split its columns.  The
//               groups merge per unit in a fixed order (deterministic).
#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <mutex>

#include "otk_common.cuh"

namespace otk {
namespace tc {

constexpr int BM = 128;                 // P rows per tile (MMA M, TMEM lanes)
constexpr int BK = 64;                  // fp16 K-block = one 128-byte swizzle row
constexpr int A_TILE = BM * BK * 2;     // 16 KB
constexpr int EXT_K = 16;               // norm-plane columns (one MMA K step)
constexpr int A_EXT = BM * EXT_K * 2;   // 4 KB
constexpr int EPI_WARP0 = 4;            // warps 0-3: TMA producer, MMA issuer, 2 spare
constexpr int NSLOT = 2;                // per-tile extras ring (bias vector + Q norm plane [+ A norm plane])

template <int V, int NG>
struct Cfg {
  static constexpr int THREADS = 32 * EPI_WARP0 + 128 * NG;  // NG epilogue warpgroups
  static constexpr int NACC = V;                    // accumulators per tile (1, 2 or 4)
  static constexpr int NBUF = (V == 4) ? 1 : 2;     // tile buffers in TMEM
  static constexpr int BN = 512 / (NACC * NBUF);    // Q rows per tile: 256, 128, 128
  static constexpr int B_TILE = BN * BK * 2;
  static constexpr int B_EXT = BN * EXT_K * 2;
  static constexpr int CH = (NG == 4 ? 16 : 32) / NACC;  // columns per epilogue chunk
  static constexpr int NCH = BN / CH;               // chunks per tile
  static constexpr int NCH_G = NCH / NG;            // chunks per epilogue group per tile
  static constexpr int EPI_ARRIVE = 128 * NG;       // every group reads every tile
  // kind::f16 instruction descriptor: D=f32 (bit 4), A=B=f16, K-major, N>>3 @17, M>>4 @24
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
template <uint32_t IDESC>
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(IDESC), "r"(accumulate));
}
// Warp-wide issue: every lane executes these (so the operands stay in the
// uniform datapath) and elect.sync picks the one lane that issues.
template <uint32_t IDESC>
__device__ __forceinline__ void umma_f16_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_w(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// K-major operand, 128-byte swizzle: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;              // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
// K-major 16-column norm plane, 32-byte swizzle: rows of 32 B, 8-row atoms 256 B apart.
__device__ __forceinline__ uint64_t sw32_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;              // SWIZZLE_32B
  return d;
}

// tcgen05.ld of 32 lanes x N consecutive 32-bit columns (async until tmem_wait).
__device__ __forceinline__ void tmem_ld_x32(uint32_t taddr, uint32_t *v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t *v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_x8(uint32_t taddr, uint32_t *v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_x4(uint32_t taddr, uint32_t *v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait16(uint32_t *v) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}
// Wait for outstanding tcgen05.ld; the 32 registers are tied in/out so the
// compiler cannot move their uses above the wait.
__device__ __forceinline__ void tmem_wait(uint32_t *v) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                 "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                 "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                 "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}

struct Params {
  int64_t np, nq;
  int kb;                 // K-blocks (dpad / 64)
  int row_tiles, ntiles, tps, nsplit, num_units;
  float c2k;              // 2*kappa/s^2 (sqeucl) or -kappa*sqrt(2)/s (eucl)
  int same;               // identical point sets (eucl: exact-zero diagonal)
  float *partial;         // [nsplit][np]
  int probe;              // pipeline probe (OTK_TC_PROBE, timing experiments only):
                          // 1 = epilogue skips the math, 2 = sums without exp,
                          // 3 = no B operand loads, 4 = one product per K step
  const float *anchor;    // FIX kernels: per-P-row anchor (log2), see lse_chunk_anchored
  int *repair_ws;         // [0] = flagged-row count, [1 + rt] = row-tile flags
  int nflags;             // row_tiles + 1 (flag slots the FIX kernel clears)
  const int *tile_mask;   // repair launch: process only flagged row tiles (NULL = all)
};

// Units skipped by a repair launch (every role walks the same live sequence,
// so barrier phases stay in step).
__device__ __forceinline__ int live_unit(const Params &prm, int u, int stride) {
  if (prm.tile_mask != nullptr)
    while (u < prm.num_units && prm.tile_mask[u % prm.row_tiles] == 0) u += stride;
  return u;
}
__device__ __forceinline__ int live_pair(const Params &prm, int u, int stride, int pair_rows, int num_pairs) {
  if (prm.tile_mask != nullptr)
    while (u < num_pairs && (prm.tile_mask[2 * (u % pair_rows)] | prm.tile_mask[2 * (u % pair_rows) + 1]) == 0)
      u += stride;
  return u;
}
// Prologue shared by both kernels: a repair launch with nothing flagged exits
// at once; a FIX launch clears the flags its finalize will set.
__device__ __forceinline__ bool repair_idle(const Params &prm) {
  return prm.tile_mask != nullptr && *reinterpret_cast<const volatile int *>(prm.repair_ws) == 0;
}
__device__ __forceinline__ void clear_repair_flags(const Params &prm) {
  if (blockIdx.x == 0 && prm.repair_ws != nullptr && prm.tile_mask == nullptr)
    for (int i = threadIdx.x; i <= prm.nflags; i += blockDim.x) prm.repair_ws[i] = 0;
}

template <int V, bool A_RES, int NS, int ABUF, int NG>
struct Plan {
  using C = Cfg<V, NG>;
  static constexpr int A_KB = 2 * A_TILE;                          // one K-block of A: hi, lo
  static constexpr int STAGE = 2 * C::B_TILE + (A_RES ? 0 : A_KB);
  static constexpr int BIAS_BYTES = ((C::BN * 4 + 1023) / 1024) * 1024;
  static constexpr int SLOT = BIAS_BYTES + C::B_EXT + (A_RES ? 0 : A_EXT);
  __host__ __device__ static constexpr int a_bytes(int kb) { return A_RES ? ABUF * (kb * A_KB + A_EXT) : 0; }
  __host__ __device__ static constexpr int smem_bytes(int kb) {
    return 1024 /*align slack*/ + a_bytes(kb) + NS * STAGE + NSLOT * SLOT + 256 /*barriers*/ +
           2 * (NG - 1) * 2 * BM * (int)sizeof(float);
  }
};

// 2^x on the FMA pipe (x <= ~8; -inf and very negative x give ~2^-125, which
// is below half an ulp of any running sum s >= 2^-8 and so adds nothing):
// round-to-nearest split x = j + f with the 1.5*2^23 shifter, a degree-5
// minimax polynomial for 2^f on [-1/2, 1/2] (max rel. error 2.3e-7 in fp32,
// same class as ex2.approx), and the exponent added back with one shift-add
// (the shifter's low mantissa bits are j in two's complement).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  const float2 lo = make_float2(-125.f, -125.f);
  x.x = fmaxf(x.x, lo.x);
  x.y = fmaxf(x.y, lo.y);
  const float2 sh = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, sh);
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-j.x, -j.y));
  float2 p = make_float2(1.327647129073739e-3f, 1.327647129073739e-3f);
  p = __ffma2_rn(p, f, make_float2(9.675541892647743e-3f, 9.675541892647743e-3f));
  p = __ffma2_rn(p, f, make_float2(5.550713092088699e-2f, 5.550713092088699e-2f));
  p = __ffma2_rn(p, f, make_float2(2.4022120237350464e-1f, 2.4022120237350464e-1f));
  p = __ffma2_rn(p, f, make_float2(6.931469440460205e-1f, 6.931469440460205e-1f));
  p = __ffma2_rn(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Online update of one row state with CH columns (accumulators already summed).
// Packed f32x2 arithmetic (FFMA2 / FADD2) halves the issue slots of the
// per-cell work; EP of every 8 column pairs take their exps from the FMA-pipe
// polynomial instead of MUFU.
//
// eucl cost (OTK_COST_EUCL, geometry.py:274-275): the accumulator holds
// -s^2 C / 2; replace it by sqrt(max(-acc, 0)) = s sqrt(C / 2) so that the
// same single FFMA with c2k = -kappa sqrt(2) / s gives kappa (g - sqrt C).
// Identical point sets: the diagonal is forced to an exact zero (the split
// products leave |C_ii| ~ 1e-6 |p|^2, whose square root would not be small).
template <int CH>
__device__ __forceinline__ void eucl_transform(float *acc, int64_t row, int64_t col0, int same) {
  const int64_t dd = row - col0;
  // bit i set <=> column i of this chunk is the diagonal (a bit test per
  // register keeps the chunk in registers; no dynamically indexed store)
  const uint32_t diag = (same && dd >= 0 && dd < CH) ? (1u << (int)dd) : 0u;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const float r = sqrt_approx(fmaxf(-acc[i], 0.f));
    acc[i] = ((diag >> i) & 1u) ? 0.f : r;
  }
}

// sqeucl, identical point sets (epilogue mode 2): acc = -s^2 C / 2 -> exactly 0
// on the diagonal (geometry.py:278-292), same bit test as eucl_transform.
template <int CH>
__device__ __forceinline__ void diag_zero(float *acc, int64_t row, int64_t col0) {
  const int64_t dd = row - col0;
  const uint32_t diag = (dd >= 0 && dd < CH) ? (1u << (int)dd) : 0u;
  if (diag == 0u) return;
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = ((diag >> i) & 1u) ? 0.f : acc[i];
}

// Epilogue cost transform: EU 0 = sqeucl, 1 = eucl, 2 = sqeucl with an exact-zero diagonal.
template <int EU, int CH>
__device__ __forceinline__ void cost_transform(float *acc, int64_t row, int64_t col0, int same) {
  if constexpr (EU == 1) eucl_transform<CH>(acc, row, col0, same);
  else if constexpr (EU == 2) diag_zero<CH>(acc, row, col0);
}

template <int CH, bool MASK, int EP>
__device__ __forceinline__ void lse_chunk(const float *acc, const float *bias, float c2k, int valid,
                                          float &m, float &s) {
  float2 u[CH / 2];
  const float2 k2 = make_float2(c2k, c2k);
#pragma unroll
  for (int i = 0; i < CH / 2; ++i) {
    u[i] = __ffma2_rn(make_float2(acc[2 * i], acc[2 * i + 1]), k2,
                      make_float2(bias[2 * i], bias[2 * i + 1]));
    if (MASK) {
      if (2 * i >= valid) u[i].x = -INFINITY;
      if (2 * i + 1 >= valid) u[i].y = -INFINITY;
    }
  }
  float cm = -INFINITY;
#pragma unroll
  for (int i = 0; i < CH / 2; ++i) cm = fmaxf(cm, fmaxf(u[i].x, u[i].y));
  if (cm > m + 8.f) {  // lazy rescale: terms may exceed m by at most 2^8
    s *= ex2(m - cm);
    m = cm;
  }
  const float ms = (m == -INFINITY) ? 0.f : m;
  const float2 nms = make_float2(-ms, -ms);
  float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int i = 0; i < CH / 2; ++i) {
    const float2 x = __fadd2_rn(u[i], nms);
    float2 e;
    if (i % 8 < EP) {
      e = ex2_poly2(x);
    } else {
      e = make_float2(ex2(x.x), ex2(x.y));
    }
    acc2[i & 1] = __fadd2_rn(acc2[i & 1], e);
  }
  const float2 t2 = __fadd2_rn(acc2[0], acc2[1]);
  s += t2.x + t2.y;
}

// Anchored chunk (FIX kernels): the row's log2-sum is accumulated against a
// FIXED per-row anchor S (the same row's result from the previous half-step
// of this role) instead of a running max: s += sum 2^(u - S).  Per cell pair
// one FFMA2, one FADD2, two MUFU ex2 and one FADD2 -- no max, no rescale
// (B200 same-box probe at cfg2: 1.42 vs 1.58 ms per half-step).  Terms
// cannot overflow unless the row's sum itself does (then s = +inf) and are
// flushed only below 2^-126 of the anchor; finalize_anchored sends every row
// whose result leaves the safe window back through the running-max kernel.
template <int CH, bool MASK, int EP = 0>
__device__ __forceinline__ void lse_chunk_anchored(const float *acc, const float *bias, float c2k,
                                                   float S, int valid, float &s) {
  const float2 k2 = make_float2(c2k, c2k);
  const float2 nS = make_float2(-S, -S);
  float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int i = 0; i < CH / 2; ++i) {
    float2 x = __ffma2_rn(make_float2(acc[2 * i], acc[2 * i + 1]), k2,
                          make_float2(bias[2 * i], bias[2 * i + 1]));
    x = __fadd2_rn(x, nS);
    if (MASK) {
      if (2 * i >= valid) x.x = -INFINITY;
      if (2 * i + 1 >= valid) x.y = -INFINITY;
    }
    float2 e;
    if (i % 8 < EP) {  // FMA-pipe exp2; x <= 126 keeps it finite (T > 120 is repaired)
      x.x = fminf(x.x, 126.f);
      x.y = fminf(x.y, 126.f);
      e = ex2_poly2(x);
      if (MASK) {
        if (2 * i >= valid) e.x = 0.f;
        if (2 * i + 1 >= valid) e.y = 0.f;
      }
    } else {
      e = make_float2(ex2(x.x), ex2(x.y));
    }
    acc2[i & 1] = __fadd2_rn(acc2[i & 1], e);
  }
  const float2 t2 = __fadd2_rn(acc2[0], acc2[1]);
  s += t2.x + t2.y;
}

// Row state -> partial.  Running max: m + log2 s.  Anchored: S + log2 s
// (s = 0 -> -inf, s = +inf -> +inf, NaN propagates).
__device__ __forceinline__ float anchored_value(float S, float s) {
  if (s != s) return s;
  return (s > 0.f) ? S + lg2(s) : -INFINITY;
}
__device__ __forceinline__ float sanitize_anchor(float S) { return isfinite(S) ? S : 0.f; }

template <int V, bool A_RES, int NS, int ABUF, int EP, int NG, int EU, bool FIX>
__global__ void __launch_bounds__(Cfg<V, NG>::THREADS, 1)
    lse_tc_kernel(const __grid_constant__ CUtensorMap tm_phi, const __grid_constant__ CUtensorMap tm_plo,
                  const __grid_constant__ CUtensorMap tm_qhi, const __grid_constant__ CUtensorMap tm_qlo,
                  const __grid_constant__ CUtensorMap tm_pext, const __grid_constant__ CUtensorMap tm_qext,
                  const __grid_constant__ CUtensorMap tm_bias, const Params prm) {
  using C = Cfg<V, NG>;
  using L = Plan<V, A_RES, NS, ABUF, NG>;
  constexpr int BN = C::BN;
  constexpr int NACC = C::NACC;
  constexpr int NBUF = C::NBUF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int kb = prm.kb;
  uint8_t *a_region = smem;                                   // [ABUF][kb x (hi, lo)][A norm plane]
  uint8_t *stage_region = smem + L::a_bytes(kb);              // [NS][B hi, B lo, (A hi, A lo)]
  uint8_t *slot_region = stage_region + NS * L::STAGE;        // [NSLOT][bias, Q norm, (P norm)]
  uint64_t *bars = reinterpret_cast<uint64_t *>(slot_region + NSLOT * L::SLOT);
  uint64_t *full = bars, *empty = bars + NS;
  uint64_t *afull = bars + 2 * NS, *aempty = afull + 2;
  uint64_t *tfull = aempty + 2, *tempty = tfull + 2;
  uint64_t *xfull = tempty + 2, *xempty = xfull + NSLOT;
  // V4 (one tile buffer): the epilogue releases the accumulator slices one by
  // one in the order the next tile first writes them -- hi*hi slice 0 on
  // tempty[0], slice 1 on s1empty, slice 2 on s2empty, cross on tempty[1] --
  // so the next tile's MMAs start after one slice has been read, not four
  uint64_t *s1empty = xempty + NSLOT, *s2empty = s1empty + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(s2empty + 1);
  float *comb = reinterpret_cast<float *>(bars + 32);          // [2][NG-1][BM][2]
  static_assert(2 * NS + 8 + 2 * NSLOT + 3 <= 32, "barrier region");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (repair_idle(prm)) return;
  if (FIX) clear_repair_flags(prm);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 1);
      mbar_init(&aempty[b], 1);
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], C::EPI_ARRIVE);
    }
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&xfull[b], 1);
      mbar_init(&xempty[b], C::EPI_ARRIVE);
    }
    mbar_init(s1empty, C::EPI_ARRIVE);
    mbar_init(s2empty, C::EPI_ARRIVE);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_phi);
    tma_prefetch_desc(&tm_plo);
    tma_prefetch_desc(&tm_qhi);
    tma_prefetch_desc(&tm_qlo);
    tma_prefetch_desc(&tm_pext);
    tma_prefetch_desc(&tm_qext);
    tma_prefetch_desc(&tm_bias);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto a_tile = [&](int buf, int k, int lo) -> uint8_t * {
    return a_region + (size_t)buf * (kb * L::A_KB + A_EXT) + (size_t)k * L::A_KB + lo * A_TILE;
  };
  auto a_ext = [&](int buf) -> uint8_t * { return a_region + (size_t)buf * (kb * L::A_KB + A_EXT) + kb * L::A_KB; };
  auto st_b = [&](int s, int lo) -> uint8_t * { return stage_region + (size_t)s * L::STAGE + lo * C::B_TILE; };
  auto st_a = [&](int s, int lo) -> uint8_t * {
    return stage_region + (size_t)s * L::STAGE + 2 * C::B_TILE + lo * A_TILE;
  };
  auto slot_bias = [&](int x) -> float * { return reinterpret_cast<float *>(slot_region + (size_t)x * L::SLOT); };
  auto slot_qext = [&](int x) -> uint8_t * { return slot_region + (size_t)x * L::SLOT + L::BIAS_BYTES; };
  auto slot_pext = [&](int x) -> uint8_t * { return slot_region + (size_t)x * L::SLOT + L::BIAS_BYTES + C::B_EXT; };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t sphase = 0;
      int uc = 0, tcount = 0;
      for (int u = live_unit(prm, blockIdx.x, gridDim.x); u < prm.num_units;
           u = live_unit(prm, u + gridDim.x, gridDim.x), ++uc) {
        const int split = u / prm.row_tiles, rt = u % prm.row_tiles;
        const int t0 = split * prm.tps, t1 = min(prm.ntiles, t0 + prm.tps);
        if (A_RES) {
          const int ab = uc % ABUF;
          mbar_wait(&aempty[ab], ((uc / ABUF) & 1) ^ 1);
          mbar_expect_tx(&afull[ab], (uint32_t)(kb * L::A_KB + A_EXT));
          for (int k = 0; k < kb; ++k) {
            tma_load_2d(a_tile(ab, k, 0), &tm_phi, &afull[ab], k * BK, rt * BM);
            tma_load_2d(a_tile(ab, k, 1), &tm_plo, &afull[ab], k * BK, rt * BM);
          }
          tma_load_2d(a_ext(ab), &tm_pext, &afull[ab], 0, rt * BM);
        }
        for (int t = t0; t < t1; ++t, ++tcount) {
          for (int k = 0; k < kb; ++k) {
            mbar_wait(&empty[stage], sphase ^ 1);
            if (prm.probe == 3) {  // timing probe: no operand traffic
              mbar_arrive(&full[stage]);
              if (++stage == NS) {
                stage = 0;
                sphase ^= 1;
              }
              continue;
            }
            mbar_expect_tx(&full[stage], (uint32_t)L::STAGE);
            tma_load_2d(st_b(stage, 0), &tm_qhi, &full[stage], k * BK, t * BN);
            tma_load_2d(st_b(stage, 1), &tm_qlo, &full[stage], k * BK, t * BN);
            if (!A_RES) {
              tma_load_2d(st_a(stage, 0), &tm_phi, &full[stage], k * BK, rt * BM);
              tma_load_2d(st_a(stage, 1), &tm_plo, &full[stage], k * BK, rt * BM);
            }
            if (++stage == NS) {
              stage = 0;
              sphase ^= 1;
            }
          }
          // per-tile extras: kappa*g_j for the epilogue, norm planes for the last MMA
          const int x = tcount % NSLOT;
          mbar_wait(&xempty[x], ((tcount / NSLOT) & 1) ^ 1);
          mbar_expect_tx(&xfull[x], (uint32_t)(BN * 4 + C::B_EXT + (A_RES ? 0 : A_EXT)));
          tma_load_1d(slot_bias(x), &tm_bias, &xfull[x], t * BN);
          tma_load_2d(slot_qext(x), &tm_qext, &xfull[x], 0, t * BN);
          if (!A_RES) tma_load_2d(slot_pext(x), &tm_pext, &xfull[x], 0, rt * BM);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (uniform control flow and operands);
    // elect.sync inside umma_f16_w / umma_commit_w issues from one lane.
    {
      int stage = 0;
      uint32_t sphase = 0;
      int tcount = 0, uc = 0;
      for (int u = live_unit(prm, blockIdx.x, gridDim.x); u < prm.num_units;
           u = live_unit(prm, u + gridDim.x, gridDim.x), ++uc) {
        const int split = u / prm.row_tiles;
        const int t0 = split * prm.tps, t1 = min(prm.ntiles, t0 + prm.tps);
        const int ab = uc % ABUF;
        if (A_RES) {
          mbar_wait(&afull[ab], (uc / ABUF) & 1);
          tc_fence_after();
        }
        for (int t = t0; t < t1; ++t, ++tcount) {
          const int buf = tcount % NBUF;
          const uint32_t tpar = ((tcount / NBUF) & 1) ^ 1;
          if (NACC != 4) {
            mbar_wait(&tempty[buf], tpar);
            tc_fence_after();
          }
          const uint32_t d0 = tmem_base + (uint32_t)(buf * NACC * BN);
          const uint32_t d_cross = d0 + (uint32_t)((NACC - 1) * BN);
          for (int k = 0; k < kb; ++k) {
            // V4 layout: hi*hi over three slices round-robin (slice = k % 3);
            // the cross terms of K-blocks 0-2 go into those hi*hi slices, later
            // ones into the cross accumulator -- so K-block k < 3 of the next
            // tile needs only slice k released, and the cross slice (read last)
            // is first written at k = 3
            const int slice = (NACC == 4) ? k % 3 : 0;
            const bool main_first = (NACC == 4) ? k < 3 : (k == 0);
            if (NACC == 4 && k < 4) {  // first write of a slice in this tile: wait for its release
              mbar_wait(k == 0 ? &tempty[0] : k == 1 ? s1empty : k == 2 ? s2empty : &tempty[1], tpar);
              tc_fence_after();
            }
            mbar_wait(&full[stage], sphase);
            tc_fence_after();
            // descriptors of the K-block; +2 (32 B >> 4) per 16-deep K step
            const uint64_t dah = sw128_desc(smem_u32(A_RES ? a_tile(ab, k, 0) : st_a(stage, 0)));
            const uint64_t dal = sw128_desc(smem_u32(A_RES ? a_tile(ab, k, 1) : st_a(stage, 1)));
            const uint64_t dbh = sw128_desc(smem_u32(st_b(stage, 0)));
            const uint64_t dbl = sw128_desc(smem_u32(st_b(stage, 1)));
            const uint32_t d_main = d0 + (uint32_t)(slice * BN);
            // cross-term target and its first write (V4: the hi*hi slice for k < 3)
            const bool cross_in_main = (NACC == 1) || (NACC == 4 && k < 3);
            const uint32_t d_cx = cross_in_main ? d_main : d_cross;
            const int cross_k0 = (NACC == 4) ? 3 : 0;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t o = (uint64_t)(2 * kk);
              const uint32_t acc_main = (main_first && kk == 0) ? 0u : 1u;
              const uint32_t acc_cross = (!cross_in_main && k == cross_k0 && kk == 0) ? 0u : 1u;
              umma_f16_w<C::IDESC>(d_main, dah + o, dbh + o, acc_main);
              if (prm.probe == 4) continue;  // timing probe: hi*hi only
              umma_f16_w<C::IDESC>(d_cx, dah + o, dbl + o, acc_cross);
              umma_f16_w<C::IDESC>(d_cx, dal + o, dbh + o, 1u);
            }
            umma_commit_w(&empty[stage]);  // smem stage free once these MMAs retire
            if (++stage == NS) {
              stage = 0;
              sphase ^= 1;
            }
          }
          // last MMA of the tile: -s^2(|p|^2 + |q|^2)/2 into the (small) cross accumulator
          const int x = tcount % NSLOT;
          mbar_wait(&xfull[x], (tcount / NSLOT) & 1);
          tc_fence_after();
          umma_f16_w<C::IDESC>(d_cross, sw32_desc(smem_u32(A_RES ? a_ext(ab) : slot_pext(x))),
                               sw32_desc(smem_u32(slot_qext(x))), 1u);
          umma_commit_w(&tfull[buf]);  // accumulators ready for the epilogue
        }
        if (A_RES) umma_commit_w(&aempty[ab]);
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ------------------------------------------------------------ epilogue
    const int eg = (warp - EPI_WARP0) >> 2;  // epilogue warpgroup 0 .. NG-1
    const int quarter = warp & 3;             // TMEM lane quarter of this warp
    const int row_local = quarter * 32 + lane;
    const uint32_t t_lane = (uint32_t)(quarter * 32) << 16;
    const float c2k = prm.c2k;
    int tcount = 0, uc = 0;
    for (int u = live_unit(prm, blockIdx.x, gridDim.x); u < prm.num_units;
         u = live_unit(prm, u + gridDim.x, gridDim.x), ++uc) {
      const int split = u / prm.row_tiles, rt = u % prm.row_tiles;
      const int t0 = split * prm.tps, t1 = min(prm.ntiles, t0 + prm.tps);
      float m = -INFINITY, s = 0.f;
      if constexpr (FIX) {  // m holds the row's anchor S for the whole unit
        const int64_t row = (int64_t)rt * BM + row_local;
        m = sanitize_anchor(row < prm.np ? prm.anchor[row] : 0.f);
      }
      for (int t = t0; t < t1; ++t, ++tcount) {
        const int buf = tcount % NBUF;
        const int x = tcount % NSLOT;
        mbar_wait(&tfull[buf], (tcount / NBUF) & 1);
        mbar_wait(&xfull[x], (tcount / NSLOT) & 1);
        tc_fence_after();
        const int64_t j0 = (int64_t)t * BN;
        const int valid = (int)(prm.nq - j0 < BN ? prm.nq - j0 : (int64_t)BN);
        const uint32_t tbase = tmem_base + (uint32_t)(buf * NACC * BN) + t_lane;
        const float *bias = slot_bias(x);
        const int cfirst = eg * C::NCH_G;  // the groups split the tile's columns
        // software pipeline: chunk c+1's tcgen05.ld is in flight while chunk c computes
        constexpr int NV = C::CH * NACC;  // registers per chunk (16 or 32)
        uint32_t va[NV], vb[NV];
        auto issue = [&](int c, uint32_t *v) {
#pragma unroll
          for (int a = 0; a < NACC; ++a) {
            const uint32_t ta = tbase + a * BN + c * C::CH;
            if (C::CH == 32) tmem_ld_x32(ta, v + a * C::CH);
            else if (C::CH == 16) tmem_ld_x16(ta, v + a * C::CH);
            else if (C::CH == 8) tmem_ld_x8(ta, v + a * C::CH);
            else tmem_ld_x4(ta, v + a * C::CH);
          }
        };
        auto wait = [&](uint32_t *v) {
          if (NV == 32) tmem_wait(v);
          else tmem_wait16(v);
        };
        auto consume = [&](int c, uint32_t *v) {
          float accv[C::CH];
#pragma unroll
          for (int i = 0; i < C::CH; ++i) {
            float a0 = __uint_as_float(v[i]);
            if (NACC == 2) a0 += __uint_as_float(v[C::CH + i]);
            if (NACC == 4)
              a0 = (__uint_as_float(v[i]) + __uint_as_float(v[C::CH + i])) +
                   (__uint_as_float(v[2 * C::CH + i]) + __uint_as_float(v[3 * C::CH + i]));
            accv[i] = a0;
          }
          const float4 *bp = reinterpret_cast<const float4 *>(bias + c * C::CH);
          float bv[C::CH];
#pragma unroll
          for (int i = 0; i < C::CH / 4; ++i) {
            float4 q = bp[i];
            bv[4 * i] = q.x;
            bv[4 * i + 1] = q.y;
            bv[4 * i + 2] = q.z;
            bv[4 * i + 3] = q.w;
          }
          if constexpr (EU != 0) cost_transform<EU, C::CH>(accv, (int64_t)rt * BM + row_local, j0 + c * C::CH, prm.same);
          if (prm.probe == 1) {
            s += accv[0];
          } else if (prm.probe == 2) {
#pragma unroll
            for (int i = 0; i < C::CH; ++i) s += fmaf(accv[i], c2k, bv[i]);
          } else if constexpr (FIX) {
            if (valid >= BN) lse_chunk_anchored<C::CH, false, EP>(accv, bv, c2k, m, 0, s);
            else lse_chunk_anchored<C::CH, true, EP>(accv, bv, c2k, m, valid - c * C::CH, s);
          } else if (valid >= BN)
            lse_chunk<C::CH, false, EP>(accv, bv, c2k, 0, m, s);
          else
            lse_chunk<C::CH, true, EP>(accv, bv, c2k, valid - c * C::CH, m, s);
        };
        if constexpr (NACC == 4) {
          // V4: read this group's 32 columns of every slice first, releasing
          // each slice to the MMA as soon as it is read (order 0, 1, 2, cross =
          // the order the next tile's K-blocks first write them), then run the
          // math on registers while the next tile's MMAs proceed.
          constexpr int GC = C::NCH_G * C::CH;
          static_assert(GC == 32, "V4 epilogue: 32 columns per group");
          const int col0 = cfirst * C::CH;
          float tot[GC];
          uint32_t v[GC];
          tmem_ld_x32(tbase + col0, v);
          tmem_wait(v);
#pragma unroll
          for (int i = 0; i < GC; ++i) tot[i] = __uint_as_float(v[i]);
          tc_fence_before();
          mbar_arrive(&tempty[0]);
          tmem_ld_x32(tbase + BN + col0, v);
          tmem_wait(v);
#pragma unroll
          for (int i = 0; i < GC; ++i) tot[i] += __uint_as_float(v[i]);
          tc_fence_before();
          mbar_arrive(s1empty);
          tmem_ld_x32(tbase + 2 * BN + col0, v);
          tmem_wait(v);
#pragma unroll
          for (int i = 0; i < GC; ++i) tot[i] += __uint_as_float(v[i]);
          tc_fence_before();
          mbar_arrive(s2empty);
          tmem_ld_x32(tbase + 3 * BN + col0, v);
          tmem_wait(v);
#pragma unroll
          for (int i = 0; i < GC; ++i) tot[i] += __uint_as_float(v[i]);
          tc_fence_before();
          mbar_arrive(&tempty[1]);
#pragma unroll
          for (int h = 0; h < GC; h += 16) {
            float *accv = tot + h;
            const float4 *bp = reinterpret_cast<const float4 *>(bias + col0 + h);
            float bv[16];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float4 q = bp[i];
              bv[4 * i] = q.x;
              bv[4 * i + 1] = q.y;
              bv[4 * i + 2] = q.z;
              bv[4 * i + 3] = q.w;
            }
            if constexpr (EU != 0) cost_transform<EU, 16>(accv, (int64_t)rt * BM + row_local, j0 + col0 + h, prm.same);
            const int vh = valid - col0 - h;
            if constexpr (FIX) {
              if (vh >= 16) lse_chunk_anchored<16, false>(accv, bv, c2k, m, 0, s);
              else lse_chunk_anchored<16, true>(accv, bv, c2k, m, vh, s);
            } else if (vh >= 16) {
              lse_chunk<16, false, 0>(accv, bv, c2k, 0, m, s);
            } else {
              lse_chunk<16, true, 0>(accv, bv, c2k, vh, m, s);
            }
          }
          mbar_arrive(&xempty[x]);
        } else {
        issue(cfirst, va);
        wait(va);
#pragma unroll
        for (int c = 0; c < C::NCH_G; c += 2) {
          issue(cfirst + c + 1, vb);
          consume(cfirst + c, va);
          wait(vb);
          if (c + 2 < C::NCH_G) issue(cfirst + c + 2, va);
          consume(cfirst + c + 1, vb);
          if (c + 2 < C::NCH_G) wait(va);
        }
        tc_fence_before();
        mbar_arrive(&tempty[buf]);
        mbar_arrive(&xempty[x]);
        }
      }
      // merge the groups' row states in a fixed order (0, 1, .., NG-1): deterministic
      float *cb = comb + (uc & 1) * ((NG - 1) * 2 * BM);
      if (eg > 0) {
        cb[((eg - 1) * BM + row_local) * 2] = m;
        cb[((eg - 1) * BM + row_local) * 2 + 1] = s;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(128 * NG) : "memory");
      if (eg == 0) {
        float val;
        if constexpr (FIX) {  // same anchor in every group: the sums add (fixed order)
#pragma unroll
          for (int g = 0; g < NG - 1; ++g) s += cb[(g * BM + row_local) * 2 + 1];
          val = anchored_value(m, s);
        } else {
          Lse2 st;
          st.m = m;
          st.s = s;
#pragma unroll
          for (int g = 0; g < NG - 1; ++g) st.merge(cb[(g * BM + row_local) * 2], cb[(g * BM + row_local) * 2 + 1]);
          val = st.value();
        }
        const int64_t row = (int64_t)rt * BM + row_local;
        if (row < prm.np) prm.partial[(int64_t)split * prm.np + row] = val;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// ---------------------------------------------------------------- CTA-pair variant
// The same half-step with the 2-SM MMA (tcgen05 cta_group::2, M = 256):
// the two CTAs of a cluster take adjacent 128-row tiles of P and the SAME
// 256-column tiles of Q.  Each CTA stages its own A rows and HALF of every B
// tile (128 of the 256 rows); the leader CTA issues M=256 x N=256 x K=16 MMAs
// that read both CTAs' shared memory and write each CTA's 128 rows into its
// own TMEM.  Per SM this halves the B operand traffic (smem reads by the
// tensor core and TMA writes): 64 instead of 96 B/clk of MMA operand reads.
// Barriers: TMA bytes of both CTAs land on the leader's full/afull barriers
// (cp.async.bulk.tensor .cta_group::2), the leader's MMA commits are
// multicast to both CTAs' empty/aempty/tfull barriers, and every epilogue
// warp of both CTAs arrives on the leader's tempty barrier.  V1 (one fp32
// accumulator, d <= 128, A resident) only.
namespace pair {

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// shared::cluster address of the same object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint32_t mbar_cluster,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
template <uint32_t IDESC>
__device__ __forceinline__ void umma2_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(IDESC), "r"(accumulate));
}
// commit the leader's outstanding MMAs to the same barrier in both CTAs
__device__ __forceinline__ void commit2_w(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

constexpr int BN = 256, HALF = 128, NS = 4, NG = 4;
constexpr int THREADS = 32 * EPI_WARP0 + 128 * NG;
constexpr int B_HALF = HALF * BK * 2;           // 16 KB (one of hi / lo)
constexpr int B_EXT_HALF = HALF * EXT_K * 2;    // 4 KB
constexpr int STAGE = 2 * B_HALF + B_EXT_HALF;  // the ext half is loaded on the last K-block
constexpr int BIAS_BYTES = BN * 4;
constexpr int CH = 16, NCH_G = BN / CH / NG;
constexpr int EPI_WARPS = 4 * NG;
// kind::f16, D f32, M = 256 (cta pair), N = 256
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);

template <int KB>
struct Plan2 {
  static constexpr int ABUF = (KB == 1) ? 2 : 1;
  static constexpr int A_BYTES = ABUF * (KB * 2 * A_TILE + A_EXT);
  static constexpr int SMEM = 1024 + A_BYTES + NS * STAGE + NSLOT * BIAS_BYTES + 256 +
                              2 * (NG - 1) * 2 * BM * (int)sizeof(float);
};

template <int KB, int EU, bool FIX>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    lse_tc_pair_kernel(const __grid_constant__ CUtensorMap tm_phi, const __grid_constant__ CUtensorMap tm_plo,
                       const __grid_constant__ CUtensorMap tm_qhi, const __grid_constant__ CUtensorMap tm_qlo,
                       const __grid_constant__ CUtensorMap tm_pext, const __grid_constant__ CUtensorMap tm_qext,
                       const __grid_constant__ CUtensorMap tm_bias, const Params prm) {
  using L = Plan2<KB>;
  constexpr int ABUF = L::ABUF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *a_region = smem;
  uint8_t *stage_region = smem + L::A_BYTES;
  uint8_t *slot_region = stage_region + NS * STAGE;
  uint64_t *bars = reinterpret_cast<uint64_t *>(slot_region + NSLOT * BIAS_BYTES);
  uint64_t *full = bars, *empty = bars + NS;
  uint64_t *afull = bars + 2 * NS, *aempty = afull + 2;
  uint64_t *tfull = aempty + 2, *tempty = tfull + 2;
  uint64_t *xfull = tempty + 2, *xempty = xfull + NSLOT;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(xempty + NSLOT);
  float *comb = reinterpret_cast<float *>(bars + 32);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  if (repair_idle(prm)) return;  // uniform over the grid: before any cluster barrier
  if (FIX) clear_repair_flags(prm);

  if (threadIdx.x == 0) {
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 1);
      mbar_init(&aempty[b], 1);
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * EPI_WARPS);  // one arrival per epilogue warp of both CTAs
    }
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&xfull[b], 1);
      mbar_init(&xempty[b], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_phi);
    tma_prefetch_desc(&tm_plo);
    tma_prefetch_desc(&tm_qhi);
    tma_prefetch_desc(&tm_qlo);
    tma_prefetch_desc(&tm_pext);
    tma_prefetch_desc(&tm_qext);
    tma_prefetch_desc(&tm_bias);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised and TMEM allocated before any remote use
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto a_tile = [&](int buf, int k, int lo) -> uint8_t * {
    return a_region + (size_t)buf * (KB * 2 * A_TILE + A_EXT) + (size_t)(2 * k + lo) * A_TILE;
  };
  auto a_ext = [&](int buf) -> uint8_t * {
    return a_region + (size_t)buf * (KB * 2 * A_TILE + A_EXT) + KB * 2 * A_TILE;
  };
  auto st_b = [&](int q, int lo) -> uint8_t * { return stage_region + (size_t)q * STAGE + lo * B_HALF; };
  auto st_ext = [&](int q) -> uint8_t * { return stage_region + (size_t)q * STAGE + 2 * B_HALF; };
  auto slot_bias = [&](int x) -> float * { return reinterpret_cast<float *>(slot_region + (size_t)x * BIAS_BYTES); };

  const int pair_rows = (prm.row_tiles + 1) / 2;
  const int num_pairs = pair_rows * prm.nsplit;
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint32_t afull_l0 = mapa(smem_u32(&afull[0]), 0), afull_l1 = mapa(smem_u32(&afull[1]), 0);
      int stage = 0;
      uint32_t sphase = 0;
      int uc = 0, tcount = 0;
      for (int u = live_pair(prm, cid, ncl, pair_rows, num_pairs); u < num_pairs;
           u = live_pair(prm, u + ncl, ncl, pair_rows, num_pairs), ++uc) {
        const int split = u / pair_rows, pr = u % pair_rows;
        const int rt = 2 * pr + (int)rank;
        const int t0 = split * prm.tps, t1 = min(prm.ntiles, t0 + prm.tps);
        const int ab = uc % ABUF;
        const uint32_t afl = ab ? afull_l1 : afull_l0;
        mbar_wait(&aempty[ab], ((uc / ABUF) & 1) ^ 1);
        if (leader) mbar_expect_tx(&afull[ab], (uint32_t)(2 * (KB * 2 * A_TILE + A_EXT)));
        for (int k = 0; k < KB; ++k) {
          tma_load_2d_pair(a_tile(ab, k, 0), &tm_phi, afl, k * BK, rt * BM);
          tma_load_2d_pair(a_tile(ab, k, 1), &tm_plo, afl, k * BK, rt * BM);
        }
        tma_load_2d_pair(a_ext(ab), &tm_pext, afl, 0, rt * BM);
        for (int t = t0; t < t1; ++t, ++tcount) {
          for (int k = 0; k < KB; ++k) {
            mbar_wait(&empty[stage], sphase ^ 1);
            const uint32_t fl = mapa(smem_u32(&full[stage]), 0);
            const bool last = (k == KB - 1);
            if (leader) mbar_expect_tx(&full[stage], (uint32_t)(2 * (2 * B_HALF + (last ? B_EXT_HALF : 0))));
            const int brow = t * BN + (int)rank * HALF;
            tma_load_2d_pair(st_b(stage, 0), &tm_qhi, fl, k * BK, brow);
            tma_load_2d_pair(st_b(stage, 1), &tm_qlo, fl, k * BK, brow);
            if (last) tma_load_2d_pair(st_ext(stage), &tm_qext, fl, 0, brow);
            if (++stage == NS) {
              stage = 0;
              sphase ^= 1;
            }
          }
          // kappa*g_j of all 256 columns for this CTA's epilogue (local)
          const int x = tcount % NSLOT;
          mbar_wait(&xempty[x], ((tcount / NSLOT) & 1) ^ 1);
          mbar_expect_tx(&xfull[x], (uint32_t)BIAS_BYTES);
          tma_load_1d(slot_bias(x), &tm_bias, &xfull[x], t * BN);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader) {
      int stage = 0;
      uint32_t sphase = 0;
      int tcount = 0, uc = 0;
      for (int u = live_pair(prm, cid, ncl, pair_rows, num_pairs); u < num_pairs;
           u = live_pair(prm, u + ncl, ncl, pair_rows, num_pairs), ++uc) {
        const int split = u / pair_rows;
        const int t0 = split * prm.tps, t1 = min(prm.ntiles, t0 + prm.tps);
        const int ab = uc % ABUF;
        mbar_wait(&afull[ab], (uc / ABUF) & 1);
        tc_fence_after();
        for (int t = t0; t < t1; ++t, ++tcount) {
          const int buf = tcount & 1;
          mbar_wait(&tempty[buf], ((tcount >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + (uint32_t)(buf * BN);
          for (int k = 0; k < KB; ++k) {
            mbar_wait(&full[stage], sphase);
            tc_fence_after();
            const uint64_t dah = sw128_desc(smem_u32(a_tile(ab, k, 0)));
            const uint64_t dal = sw128_desc(smem_u32(a_tile(ab, k, 1)));
            const uint64_t dbh = sw128_desc(smem_u32(st_b(stage, 0)));
            const uint64_t dbl = sw128_desc(smem_u32(st_b(stage, 1)));
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t o = (uint64_t)(2 * kk);
              umma2_w<IDESC>(d, dah + o, dbh + o, (k == 0 && kk == 0) ? 0u : 1u);
              umma2_w<IDESC>(d, dah + o, dbl + o, 1u);
              umma2_w<IDESC>(d, dal + o, dbh + o, 1u);
            }
            if (k == KB - 1)  // -s^2 (|p|^2 + |q|^2) / 2, last (see the file header)
              umma2_w<IDESC>(d, sw32_desc(smem_u32(a_ext(ab))), sw32_desc(smem_u32(st_ext(stage))), 1u);
            commit2_w(&empty[stage]);
            if (++stage == NS) {
              stage = 0;
              sphase ^= 1;
            }
          }
          commit2_w(&tfull[buf]);
        }
        commit2_w(&aempty[ab]);
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int eg = (warp - EPI_WARP0) >> 2;
    const int quarter = warp & 3;
    const int row_local = quarter * 32 + lane;
    const uint32_t t_lane = (uint32_t)(quarter * 32) << 16;
    const float c2k = prm.c2k;
    const uint32_t tempty_l0 = mapa(smem_u32(&tempty[0]), 0), tempty_l1 = mapa(smem_u32(&tempty[1]), 0);
    int tcount = 0, uc = 0;
    for (int u = live_pair(prm, cid, ncl, pair_rows, num_pairs); u < num_pairs;
         u = live_pair(prm, u + ncl, ncl, pair_rows, num_pairs), ++uc) {
      const int split = u / pair_rows, pr = u % pair_rows;
      const int rt = 2 * pr + (int)rank;
      const int t0 = split * prm.tps, t1 = min(prm.ntiles, t0 + prm.tps);
      float m = -INFINITY, s = 0.f;
      if constexpr (FIX) {
        const int64_t row = (int64_t)rt * BM + row_local;
        m = sanitize_anchor(row < prm.np ? prm.anchor[row] : 0.f);
      }
      for (int t = t0; t < t1; ++t, ++tcount) {
        const int buf = tcount & 1;
        const int x = tcount % NSLOT;
        mbar_wait(&tfull[buf], (tcount >> 1) & 1);
        mbar_wait(&xfull[x], (tcount / NSLOT) & 1);
        tc_fence_after();
        const int64_t j0 = (int64_t)t * BN;
        const int valid = (int)(prm.nq - j0 < BN ? prm.nq - j0 : (int64_t)BN);
        const uint32_t tbase = tmem_base + (uint32_t)(buf * BN) + t_lane;
        const float *bias = slot_bias(x);
        const int cfirst = eg * NCH_G;
        uint32_t va[16], vb[16];
        auto consume = [&](int c, uint32_t *v) {
          float accv[CH], bv[CH];
#pragma unroll
          for (int i = 0; i < CH; ++i) accv[i] = __uint_as_float(v[i]);
          if constexpr (EU != 0) cost_transform<EU, CH>(accv, (int64_t)rt * BM + row_local, j0 + c * CH, prm.same);
          const float4 *bp = reinterpret_cast<const float4 *>(bias + c * CH);
#pragma unroll
          for (int i = 0; i < CH / 4; ++i) {
            const float4 q = bp[i];
            bv[4 * i] = q.x;
            bv[4 * i + 1] = q.y;
            bv[4 * i + 2] = q.z;
            bv[4 * i + 3] = q.w;
          }
          if constexpr (FIX) {
            if (valid >= BN) lse_chunk_anchored<CH, false>(accv, bv, c2k, m, 0, s);
            else lse_chunk_anchored<CH, true>(accv, bv, c2k, m, valid - c * CH, s);
          } else if (valid >= BN)
            lse_chunk<CH, false, 0>(accv, bv, c2k, 0, m, s);
          else
            lse_chunk<CH, true, 0>(accv, bv, c2k, valid - c * CH, m, s);
        };
        tmem_ld_x16(tbase + cfirst * CH, va);
        tmem_wait16(va);
#pragma unroll
        for (int c = 0; c < NCH_G; c += 2) {
          tmem_ld_x16(tbase + (cfirst + c + 1) * CH, vb);
          consume(cfirst + c, va);
          tmem_wait16(vb);
          if (c + 2 < NCH_G) tmem_ld_x16(tbase + (cfirst + c + 2) * CH, va);
          consume(cfirst + c + 1, vb);
          if (c + 2 < NCH_G) tmem_wait16(va);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          arrive_remote(buf ? tempty_l1 : tempty_l0);  // the leader's MMA waits on both CTAs
          mbar_arrive(&xempty[x]);
        }
      }
      float *cb = comb + (uc & 1) * ((NG - 1) * 2 * BM);
      if (eg > 0) {
        cb[((eg - 1) * BM + row_local) * 2] = m;
        cb[((eg - 1) * BM + row_local) * 2 + 1] = s;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(128 * NG) : "memory");
      if (eg == 0) {
        float val;
        if constexpr (FIX) {
#pragma unroll
          for (int g = 0; g < NG - 1; ++g) s += cb[(g * BM + row_local) * 2 + 1];
          val = anchored_value(m, s);
        } else {
          Lse2 st;
          st.m = m;
          st.s = s;
#pragma unroll
          for (int g = 0; g < NG - 1; ++g) st.merge(cb[(g * BM + row_local) * 2], cb[(g * BM + row_local) * 2 + 1]);
          val = st.value();
        }
        const int64_t row = (int64_t)rt * BM + row_local;
        if (row < prm.np) prm.partial[(int64_t)split * prm.np + row] = val;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs done (the leader's MMAs wrote the peer's TMEM)
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

}  // namespace pair

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D fp16 plane [rows, cols], box = box_cols x box_rows; 128B swizzle for the 64-wide
// K-blocks, 32B swizzle for the 16-wide norm planes.
static int make_plane_map(CUtensorMap *map, const void *base, int64_t rows, int cols, int box_rows,
                          int box_cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return OTK_ENOTSUP;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  box_cols == BK ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(plane) failed (%d) rows=%lld cols=%d", (int)r, (long long)rows, cols);
    return OTK_EINVAL;
  }
  return OTK_OK;
}

// 1-D fp32 vector [n], box = box elements (OOB reads as 0; masked by the epilogue).
static int make_vec_map(CUtensorMap *map, const float *base, int64_t n, int box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return OTK_ENOTSUP;
  }
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) {
    set_error("lse_tc: bias vector must be 16-byte aligned");
    return OTK_EINVAL;
  }
  cuuint64_t dims[1] = {(cuuint64_t)n};
  cuuint64_t unused_strides[1] = {(cuuint64_t)n * 4};  // must be non-NULL even for rank 1 (probed)
  cuuint32_t boxd[1] = {(cuuint32_t)box};
  cuuint32_t estr[1] = {1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, const_cast<float *>(base), dims,
                  unused_strides, boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(bias) failed (%d) n=%lld", (int)r, (long long)n);
    return OTK_EINVAL;
  }
  return OTK_OK;
}

// exp2 split: EP of every 8 column pairs on the FMA-pipe polynomial
// (OTK_TC_EMU = 2; measured on B200 at d = 64: 0 -> 1.54 ms, 2 -> 1.59 ms,
// 4 -> 1.77 ms, 8 -> 2.27 ms per cfg2 half-step -- the epilogue is bound by
// the TMEM read path, not MUFU, so every exp stays on MUFU by default).
static int emu_pairs(int v) {
  if (v != 1) return 0;
  if (const char *e = getenv("OTK_TC_EMU")) return atoi(e);
  return 0;  // measured: the split-column epilogue is no longer MUFU-bound at d = 64
}

template <int V, bool A_RES, int NS, int ABUF, int EP, int NG, int EU = 0, bool FIX = false>
static int launch_one(const CUtensorMap (&maps)[7], const Params &prm, cudaStream_t st) {
  using L = Plan<V, A_RES, NS, ABUF, NG>;
  const int smem = L::smem_bytes(prm.kb);
  auto kern = lse_tc_kernel<V, A_RES, NS, ABUF, EP, NG, EU, FIX>;
  static bool attr_set = false;
  if (smem > 227 * 1024) {
    set_error("lse_tc: shared memory plan too large (%d B, kb=%d)", smem, prm.kb);
    return OTK_ENOTSUP;
  }
  if (!attr_set) {
    OTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set = true;
  }
  const int grid = std::min(prm.num_units, num_sms());
  kern<<<grid, Cfg<V, NG>::THREADS, smem, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], prm);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OTK_OK : cuda_status(e, "lse_tc_kernel");
}

// Epilogue warpgroups (OTK_TC_GROUPS = 2 or 4; default 4: the per-row
// LSE chain is latency-bound with two warps per SM sub-partition).
static int epi_groups() {
  if (const char *e = getenv("OTK_TC_GROUPS")) return atoi(e) == 2 ? 2 : 4;
  return 4;
}

template <int V, bool A_RES, int NS, int ABUF>
static int launch_variant(const CUtensorMap (&maps)[7], const Params &prm, int eu, bool fix,
                          cudaStream_t st) {
  if (eu == 1) return launch_one<V, A_RES, NS, ABUF, 0, 4, 1>(maps, prm, st);  // default knobs only
  if (eu == 2) {  // identical point sets: exact-zero diagonal, default knobs only
    return fix ? launch_one<V, A_RES, NS, ABUF, 0, 4, 2, true>(maps, prm, st)
               : launch_one<V, A_RES, NS, ABUF, 0, 4, 2>(maps, prm, st);
  }
  if (fix) {
    if constexpr (V == 1) {
      switch (emu_pairs(V)) {
        case 1: return launch_one<V, A_RES, NS, ABUF, 1, 4, 0, true>(maps, prm, st);
        case 2: return launch_one<V, A_RES, NS, ABUF, 2, 4, 0, true>(maps, prm, st);
        default: break;
      }
    }
    return launch_one<V, A_RES, NS, ABUF, 0, 4, 0, true>(maps, prm, st);
  }
  if constexpr (V == 4) {  // the V4 slice-release epilogue is written for 4 groups
    return launch_one<V, A_RES, NS, ABUF, 0, 4>(maps, prm, st);
  } else {
  const bool g4 = epi_groups() == 4;
  if constexpr (V == 1) {
    switch (emu_pairs(V)) {
      case 2: return g4 ? launch_one<V, A_RES, NS, ABUF, 2, 4>(maps, prm, st)
                        : launch_one<V, A_RES, NS, ABUF, 2, 2>(maps, prm, st);
      default: break;
    }
  }
  return g4 ? launch_one<V, A_RES, NS, ABUF, 0, 4>(maps, prm, st)
            : launch_one<V, A_RES, NS, ABUF, 0, 2>(maps, prm, st);
  }
}

// Same-box A/B (B200): cfg2 (d = 64, one K-block) 1.81 vs 1.50 ms per half-step
// (slower: the pair's epilogues pace each other), cfg4 (d = 128, two K-blocks)
// 19.2 / 18.9 vs 19.5 / 19.8 ms (faster: half the B operand traffic per SM).
// Default: pair for two K-blocks only; OTK_TC_PAIR=0/1 overrides.
static bool use_pair_kernel(int kb) {
  if (const char *e = getenv("OTK_TC_PAIR")) return atoi(e) == 1;
  return kb == 2;
}

template <int KB, int EU, bool FIX = false>
static int launch_pair(const CUtensorMap (&maps)[7], const Params &prm, cudaStream_t st) {
  using L = pair::Plan2<KB>;
  auto kern = pair::lse_tc_pair_kernel<KB, EU, FIX>;
  static bool attr_set = false;
  static_assert(L::SMEM <= 227 * 1024, "pair kernel shared memory plan too large");
  if (!attr_set) {
    OTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM));
    attr_set = true;
  }
  const int num_pairs = ((prm.row_tiles + 1) / 2) * prm.nsplit;
  const int grid = 2 * std::min(num_pairs, num_sms() / 2);
  kern<<<grid, pair::THREADS, L::SMEM, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5],
                                              maps[6], prm);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OTK_OK : cuda_status(e, "lse_tc_pair_kernel");
}

static int variant_for(int kb) {
  if (const char *v = getenv("OTK_TC_VARIANT")) return atoi(v);
  // V1 (one accumulator) reads 4 B of TMEM per cell -- the epilogue's binding
  // resource (tcgen05.ld ~64 B/clk/SM) -- and is accurate to ~2e-7 for d <= 128;
  // the long K chains of d > 128 need the split accumulators (V2 / V4) for
  // the 1e-5 cost tolerance (tools/diag_variants.py).
  return kb <= 2 ? 1 : (kb <= 4 ? 2 : 4);
}

}  // namespace tc

bool tc_available() {
  static int ok = -1;
  if (ok < 0) {
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    ok = (major == 10 && minor == 0 && tc::encode_fn() != nullptr) ? 1 : 0;
  }
  return ok == 1;
}

// Tile width used by the TC kernel for this depth (drives the split planning).
int tc_tile_cols(int dpad) { return tc::variant_for(dpad / tc::BK) == 1 ? 256 : 128; }
// 1 if this depth runs the CTA-pair kernel (work units are pairs of row tiles).
int tc_uses_pair(int dpad) {
  const int kb = dpad / tc::BK;
  return (tc::variant_for(kb) == 1 && kb <= 2 && tc::use_pair_kernel(kb)) ? 1 : 0;
}

// anchor != NULL: anchored (FIX) launch -- sqeucl only -- which also clears
// repair_ws[0 .. row_tiles + 1].  repair != 0: running-max launch over the
// row tiles flagged in repair_ws (exits at once when repair_ws[0] == 0).
int lse_tc_launch(const uint16_t *p_hi, const uint16_t *p_lo, const uint16_t *p_ext, int64_t np,
                  const uint16_t *q_hi, const uint16_t *q_lo, const uint16_t *q_ext, int64_t nq,
                  int dpad, float two_kappa_scaled, const float *q_bias, int nsplit,
                  int same, int eucl, float *partial, const float *anchor, int *repair_ws,
                  int repair, cudaStream_t st) {
  using namespace tc;
  if (np > (int64_t)INT32_MAX || nq > (int64_t)INT32_MAX) {
    set_error("lse_tc: too many points");
    return OTK_EINVAL;
  }
  const int kb = dpad / BK;
  const int v = variant_for(kb);
  const int bn = (v == 1) ? 256 : 128;
  if (v == 4 && kb < 3) {
    set_error("lse_tc: variant 4 needs d > 128");
    return OTK_EINVAL;
  }
  // CTA-pair (cta_group::2) variant for V1 with resident A (d <= 128), see
  // pair::lse_tc_pair_kernel and use_pair_kernel
  const bool use_pair = (v == 1 && kb <= 2 && use_pair_kernel(kb));
  const int qbox = use_pair ? pair::HALF : bn;
  CUtensorMap maps[7];
  int rc;
  if ((rc = make_plane_map(&maps[0], p_hi, np, dpad, BM, BK)) != OTK_OK) return rc;
  if ((rc = make_plane_map(&maps[1], p_lo, np, dpad, BM, BK)) != OTK_OK) return rc;
  if ((rc = make_plane_map(&maps[2], q_hi, nq, dpad, qbox, BK)) != OTK_OK) return rc;
  if ((rc = make_plane_map(&maps[3], q_lo, nq, dpad, qbox, BK)) != OTK_OK) return rc;
  if ((rc = make_plane_map(&maps[4], p_ext, np, EXT_K, BM, EXT_K)) != OTK_OK) return rc;
  if ((rc = make_plane_map(&maps[5], q_ext, nq, EXT_K, qbox, EXT_K)) != OTK_OK) return rc;
  if ((rc = make_vec_map(&maps[6], q_bias, nq, bn)) != OTK_OK) return rc;
  Params prm;
  prm.np = np;
  prm.nq = nq;
  prm.kb = kb;
  prm.row_tiles = (int)((np + BM - 1) / BM);
  prm.ntiles = (int)((nq + bn - 1) / bn);
  prm.nsplit = nsplit;
  prm.tps = (prm.ntiles + nsplit - 1) / nsplit;
  prm.num_units = prm.row_tiles * nsplit;
  prm.c2k = two_kappa_scaled;
  prm.same = same;  // eucl epilogue; sqeucl selects the exact-diagonal instantiation
  prm.partial = partial;
  prm.probe = getenv("OTK_TC_PROBE") ? atoi(getenv("OTK_TC_PROBE")) : 0;
  const int eu = eucl != 0 ? 1 : (same ? 2 : 0);
  const bool fix = anchor != nullptr && !repair;
  if (fix && eu == 1) {
    set_error("lse_tc: anchored launch needs the sqeucl epilogue");
    return OTK_EINVAL;
  }
  if ((fix || repair) && repair_ws == nullptr) {
    set_error("lse_tc: anchored / repair launch without repair workspace");
    return OTK_EINVAL;
  }
  prm.anchor = fix ? anchor : nullptr;
  prm.repair_ws = (fix || repair) ? repair_ws : nullptr;
  prm.nflags = prm.row_tiles + 1;
  prm.tile_mask = repair ? repair_ws + 1 : nullptr;
  if (use_pair) {
    if (eu == 1) return kb == 1 ? launch_pair<1, 1>(maps, prm, st) : launch_pair<2, 1>(maps, prm, st);
    if (eu == 2) {
      if (fix) return kb == 1 ? launch_pair<1, 2, true>(maps, prm, st) : launch_pair<2, 2, true>(maps, prm, st);
      return kb == 1 ? launch_pair<1, 2>(maps, prm, st) : launch_pair<2, 2>(maps, prm, st);
    }
    if (fix) return kb == 1 ? launch_pair<1, 0, true>(maps, prm, st) : launch_pair<2, 0, true>(maps, prm, st);
    return kb == 1 ? launch_pair<1, 0>(maps, prm, st) : launch_pair<2, 0>(maps, prm, st);
  }
  if (v == 1) {
    if (kb == 1) return launch_variant<1, true, 2, 2>(maps, prm, eu, fix, st);
    if (kb == 2) return launch_variant<1, true, 2, 1>(maps, prm, eu, fix, st);
    return launch_variant<1, false, 2, 1>(maps, prm, eu, fix, st);
  }
  if (v == 2) {
    if (kb <= 2) return launch_variant<2, true, 4, 1>(maps, prm, eu, fix, st);
    if (kb <= 4) return launch_variant<2, true, 2, 1>(maps, prm, eu, fix, st);
    return launch_variant<2, false, 3, 1>(maps, prm, eu, fix, st);
  }
  return launch_variant<4, false, 3, 1>(maps, prm, eu, fix, st);
}

}  // namespace otk
