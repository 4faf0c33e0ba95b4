// K2 -- online half-step on the 5th-generation tensor cores (sm_100a):
// tcgen05.mma with TMEM accumulators, TMA-staged shared memory, and a
// streaming log2-sum-exp2 epilogue read straight out of TMEM.
//
// Replaces PointCloudGeometry.apply_lse_kernel (reference geometry.py:336-354)
// for d >= 32.  Same math as the FP32 kernel (csrc/lse_simt.cu):
//     u_ij = 2*kappa*<p_i, q_j> + bias_j,   partial_i = log2 sum_j 2^u_ij
// but the dot products run on the tensor cores in split-fp16 ("3xFP16"):
// every fp32 coordinate is pre-split (K0, otk_prep_points) into
// hi = fp16(s*x), lo = fp16(s*x - hi) with a power-of-two scale s, and
//     s_p s_q <p,q> ~= hi_p.hi_q + hi_p.lo_q + lo_p.hi_q
// (error ~2^-22 |p||q|: float32 quality, SURVEY.md §7 "hard parts").
//
// CTA = one SM, persistent over work units (row tile of 128 P rows) x
// (contiguous column split of Q).  Warp roles (384 threads):
//   warp 0      TMA producer: A (P hi/lo, resident per unit) + B stages
//               (Q hi/lo K-blocks of 256 rows x 64 fp16, 128B swizzle)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=256, K=16, fp32 accumulate, 2 TMEM accumulators)
//   warps 4-11  two epilogue warpgroups, one per TMEM accumulator: each
//               thread owns one row (TMEM lane), pulls 32 columns per
//               tcgen05.ld, and keeps an online (max, sum) in registers;
//               the two groups merge per unit in a fixed order.
// Pipelines: smem full/empty mbarriers (TMA <-> MMA), tfull/tempty
// (MMA <-> epilogue), afull/aempty (A operand reuse).  Deterministic: no
// atomics, fixed reduction order.
#include <cuda.h>
#include <cuda_fp16.h>

#include <mutex>
#include <unordered_map>

#include "otk_common.cuh"

namespace otk {
namespace tc {

constexpr int BM = 128;                   // P rows per tile (MMA M, TMEM lanes)
constexpr int BN = 256;                   // Q rows per tile (MMA N, TMEM columns)
constexpr int BK = 64;                    // fp16 K-block = one 128-byte swizzle row
constexpr int A_TILE = BM * BK * 2;       // 16 KB
constexpr int B_TILE = BN * BK * 2;       // 32 KB
constexpr int THREADS = 384;
constexpr int EPI_WARP0 = 4;
constexpr int NUM_EPI = 256;
// kind::f16 instruction descriptor: D=f32 (bit 4), A=B=f16, K-major, N>>3 @17, M>>4 @24
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

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
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// K-major operand, 128-byte swizzle, rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;              // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
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
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct Params {
  int64_t np, nq;
  int kb;                 // K-blocks (dpad / 64)
  int row_tiles, ntiles, tps, nsplit, num_units;
  int order;              // MMA product order (accuracy experiments)
  const float *qbias;
  float c2k;              // 2*kappa/(s_p*s_q)
  float *partial;         // [nsplit][np]
};

template <bool A_RES, int NS, int ABUF>
struct Layout {
  static constexpr int STAGE = 2 * B_TILE + (A_RES ? 0 : 2 * A_TILE);
  __host__ __device__ static constexpr int a_bytes(int kb) { return A_RES ? ABUF * kb * 2 * A_TILE : 0; }
  __host__ __device__ static constexpr int smem_bytes(int kb) {
    return 1024 /*align slack*/ + a_bytes(kb) + NS * STAGE + 1024 /*barriers etc.*/ +
           2 * 2 * BM * (int)sizeof(float);
  }
};

template <bool A_RES, int NS, int ABUF>
__global__ void __launch_bounds__(THREADS, 1)
    lse_tc_kernel(const __grid_constant__ CUtensorMap tm_phi, const __grid_constant__ CUtensorMap tm_plo,
                  const __grid_constant__ CUtensorMap tm_qhi, const __grid_constant__ CUtensorMap tm_qlo,
                  const Params prm) {
  using L = Layout<A_RES, NS, ABUF>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int kb = prm.kb;
  uint8_t *a_region = smem;                                  // [ABUF][kb][hi,lo] 16 KB tiles
  uint8_t *stage_region = smem + L::a_bytes(kb);             // [NS][B hi, B lo, (A hi, A lo)]
  uint64_t *bars = reinterpret_cast<uint64_t *>(stage_region + NS * L::STAGE);
  uint64_t *full = bars, *empty = bars + NS;
  uint64_t *afull = bars + 2 * NS, *aempty = afull + 2;
  uint64_t *tfull = aempty + 2, *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  float *comb = reinterpret_cast<float *>(bars + 128);        // [2][BM][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 1);
      mbar_init(&aempty[b], 1);
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], NUM_EPI / 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_phi);
    tma_prefetch_desc(&tm_plo);
    tma_prefetch_desc(&tm_qhi);
    tma_prefetch_desc(&tm_qlo);
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
    return a_region + ((size_t)(buf * kb + k) * 2 + lo) * A_TILE;
  };
  auto st_b = [&](int s, int lo) -> uint8_t * { return stage_region + (size_t)s * L::STAGE + lo * B_TILE; };
  auto st_a = [&](int s, int lo) -> uint8_t * {
    return stage_region + (size_t)s * L::STAGE + 2 * B_TILE + lo * A_TILE;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t sphase = 0;
      int uc = 0;
      for (int u = blockIdx.x; u < prm.num_units; u += gridDim.x, ++uc) {
        const int split = u / prm.row_tiles, rt = u % prm.row_tiles;
        const int t0 = split * prm.tps, t1 = min(prm.ntiles, t0 + prm.tps);
        if (A_RES) {
          const int ab = uc % ABUF;
          mbar_wait(&aempty[ab], ((uc / ABUF) & 1) ^ 1);
          mbar_expect_tx(&afull[ab], (uint32_t)(kb * 2 * A_TILE));
          for (int k = 0; k < kb; ++k) {
            tma_load_2d(a_tile(ab, k, 0), &tm_phi, &afull[ab], k * BK, rt * BM);
            tma_load_2d(a_tile(ab, k, 1), &tm_plo, &afull[ab], k * BK, rt * BM);
          }
        }
        for (int t = t0; t < t1; ++t) {
          for (int k = 0; k < kb; ++k) {
            mbar_wait(&empty[stage], sphase ^ 1);
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
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t sphase = 0;
      int tcount = 0, uc = 0;
      for (int u = blockIdx.x; u < prm.num_units; u += gridDim.x, ++uc) {
        const int split = u / prm.row_tiles;
        const int t0 = split * prm.tps, t1 = min(prm.ntiles, t0 + prm.tps);
        const int ab = uc % ABUF;
        if (A_RES) {
          mbar_wait(&afull[ab], (uc / ABUF) & 1);
          tc_fence_after();
        }
        for (int t = t0; t < t1; ++t, ++tcount) {
          const int acc = tcount & 1;
          mbar_wait(&tempty[acc], ((tcount >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
          for (int k = 0; k < kb; ++k) {
            mbar_wait(&full[stage], sphase);
            tc_fence_after();
            const uint32_t ah = smem_u32(A_RES ? a_tile(ab, k, 0) : st_a(stage, 0));
            const uint32_t al = smem_u32(A_RES ? a_tile(ab, k, 1) : st_a(stage, 1));
            const uint32_t bh = smem_u32(st_b(stage, 0));
            const uint32_t bl = smem_u32(st_b(stage, 1));
            if (prm.order == 0) {
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint32_t off = kk * 32;  // 16 fp16 = 32 B along the swizzled row
                const uint64_t dah = sw128_desc(ah + off), dal = sw128_desc(al + off);
                const uint64_t dbh = sw128_desc(bh + off), dbl = sw128_desc(bl + off);
                umma_f16(d_tmem, dah, dbh, (k | kk) != 0 ? 1u : 0u);
                umma_f16(d_tmem, dah, dbl, 1u);
                umma_f16(d_tmem, dal, dbh, 1u);
              }
            } else if (prm.order == 1) {  // small cross terms first, then hi*hi
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint32_t off = kk * 32;
                umma_f16(d_tmem, sw128_desc(ah + off), sw128_desc(bl + off), (k | kk) != 0 ? 1u : 0u);
                umma_f16(d_tmem, sw128_desc(al + off), sw128_desc(bh + off), 1u);
              }
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint32_t off = kk * 32;
                umma_f16(d_tmem, sw128_desc(ah + off), sw128_desc(bh + off), 1u);
              }
            } else {  // hi*hi first, then cross terms
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint32_t off = kk * 32;
                umma_f16(d_tmem, sw128_desc(ah + off), sw128_desc(bh + off), (k | kk) != 0 ? 1u : 0u);
              }
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint32_t off = kk * 32;
                umma_f16(d_tmem, sw128_desc(ah + off), sw128_desc(bl + off), 1u);
                umma_f16(d_tmem, sw128_desc(al + off), sw128_desc(bh + off), 1u);
              }
            }
            umma_commit(&empty[stage]);  // smem stage free once these MMAs retire
            if (++stage == NS) {
              stage = 0;
              sphase ^= 1;
            }
          }
          umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        }
        if (A_RES) umma_commit(&aempty[ab]);
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ------------------------------------------------------------ epilogue
    const int eg = (warp - EPI_WARP0) >> 2;  // accumulator / warpgroup
    const int quarter = warp & 3;             // TMEM lane quarter of this warp
    const int row_local = quarter * 32 + lane;
    const uint32_t t_lane = (uint32_t)(quarter * 32) << 16;
    const float c2k = prm.c2k;
    int tcount = 0, uc = 0;
    for (int u = blockIdx.x; u < prm.num_units; u += gridDim.x, ++uc) {
      const int split = u / prm.row_tiles, rt = u % prm.row_tiles;
      const int t0 = split * prm.tps, t1 = min(prm.ntiles, t0 + prm.tps);
      float m = -INFINITY, s = 0.f;
      for (int t = t0; t < t1; ++t, ++tcount) {
        if ((tcount & 1) != eg) continue;
        mbar_wait(&tfull[eg], (tcount >> 1) & 1);
        tc_fence_after();
        const int64_t j0 = (int64_t)t * BN;
        const int valid = (int)(prm.nq - j0 < BN ? prm.nq - j0 : (int64_t)BN);
        const uint32_t taddr = tmem_base + (uint32_t)(eg * BN) + t_lane;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(taddr + c * 32, v);
          float b[32];
          const int cbase = c * 32;
          if (cbase + 32 <= valid) {
            const float4 *bp = reinterpret_cast<const float4 *>(prm.qbias + j0 + cbase);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              float4 q = __ldg(bp + i);
              b[4 * i] = q.x;
              b[4 * i + 1] = q.y;
              b[4 * i + 2] = q.z;
              b[4 * i + 3] = q.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) b[i] = (cbase + i < valid) ? prm.qbias[j0 + cbase + i] : -INFINITY;
          }
          float uu[32];
          float cm = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            uu[i] = fmaf(__uint_as_float(v[i]), c2k, b[i]);
            cm = fmaxf(cm, uu[i]);
          }
          if (cm > m + 8.f) {  // lazy rescale: terms may exceed m by at most 2^8
            s *= ex2(m - cm);
            m = cm;
          }
          const float ms = (m == -INFINITY) ? 0.f : m;
          float s0 = 0.f, s1 = 0.f;
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            s0 += ex2(uu[i] - ms);
            s1 += ex2(uu[i + 1] - ms);
          }
          s += s0 + s1;
        }
        tc_fence_before();
        mbar_arrive(&tempty[eg]);
      }
      // merge the two warpgroups' row states (fixed order: group 0 then group 1)
      float *buf = comb + (uc & 1) * (2 * BM);
      if (eg == 1) {
        buf[2 * row_local] = m;
        buf[2 * row_local + 1] = s;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (eg == 0) {
        Lse2 st;
        st.m = m;
        st.s = s;
        st.merge(buf[2 * row_local], buf[2 * row_local + 1]);
        const int64_t row = (int64_t)rt * BM + row_local;
        if (row < prm.np) prm.partial[(int64_t)split * prm.np + row] = st.value();
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

static int make_map(CUtensorMap *map, const void *base, int64_t rows, int dpad, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return OTK_ENOTSUP;
  }
  cuuint64_t dims[2] = {(cuuint64_t)dpad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)dpad * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld dpad=%d", (int)r, (long long)rows, dpad);
    return OTK_EINVAL;
  }
  return OTK_OK;
}

template <bool A_RES, int NS, int ABUF>
static int launch_variant(const CUtensorMap (&maps)[4], const Params &prm, cudaStream_t st) {
  using L = Layout<A_RES, NS, ABUF>;
  const int smem = L::smem_bytes(prm.kb);
  auto kern = lse_tc_kernel<A_RES, NS, ABUF>;
  static bool attr_set = false;
  if (!attr_set) {
    OTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set = true;
  }
  if (smem > 227 * 1024) {
    set_error("lse_tc: shared memory plan too large (%d B)", smem);
    return OTK_ENOTSUP;
  }
  const int grid = std::min(prm.num_units, num_sms());
  kern<<<grid, THREADS, smem, st>>>(maps[0], maps[1], maps[2], maps[3], prm);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OTK_OK : cuda_status(e, "lse_tc_kernel");
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

int lse_tc_launch(const uint16_t *p_hi, const uint16_t *p_lo, int64_t np, const uint16_t *q_hi,
                  const uint16_t *q_lo, int64_t nq, int dpad, float two_kappa_scaled,
                  const float *q_bias, int nsplit, float *partial, cudaStream_t st) {
  using namespace tc;
  if (np > (int64_t)INT32_MAX || nq > (int64_t)INT32_MAX) {
    set_error("lse_tc: too many points");
    return OTK_EINVAL;
  }
  CUtensorMap maps[4];
  int rc;
  if ((rc = make_map(&maps[0], p_hi, np, dpad, BM)) != OTK_OK) return rc;
  if ((rc = make_map(&maps[1], p_lo, np, dpad, BM)) != OTK_OK) return rc;
  if ((rc = make_map(&maps[2], q_hi, nq, dpad, BN)) != OTK_OK) return rc;
  if ((rc = make_map(&maps[3], q_lo, nq, dpad, BN)) != OTK_OK) return rc;
  Params prm;
  prm.np = np;
  prm.nq = nq;
  prm.kb = dpad / BK;
  prm.row_tiles = (int)((np + BM - 1) / BM);
  prm.ntiles = (int)((nq + BN - 1) / BN);
  prm.nsplit = nsplit;
  prm.tps = (prm.ntiles + nsplit - 1) / nsplit;
  prm.num_units = prm.row_tiles * nsplit;
  prm.qbias = q_bias;
  {
    const char *o = getenv("OTK_TC_ORDER");
    prm.order = o ? atoi(o) : 0;
  }
  prm.c2k = two_kappa_scaled;
  prm.partial = partial;
  if (prm.kb == 1) return launch_variant<true, 2, 2>(maps, prm, st);
  if (prm.kb == 2) return launch_variant<true, 2, 1>(maps, prm, st);
  return launch_variant<false, 2, 1>(maps, prm, st);
}

}  // namespace otk
