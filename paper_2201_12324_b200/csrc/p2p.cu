// Multi-GPU exchange of the g half-step over NVLink peer memory (SURVEY.md
// §8e; no reference equivalent -- the reference loop sinkhorn.py:151-200 is
// single-process).
//
// Row-sharded solve: every rank reduces its own rows of x into one log2
// partial per column j (the g half-step, sinkhorn.py:174), and every rank
// needs all W partials of every column to form g.  Instead of a separate
// collective, the half-step's last finalize kernel (otk_api.cu, push_row /
// signal_block) stores each column's partial straight into slot
// (epoch & 1, rank) of every peer's exchange buffer over NVLink and, per
// 256-column block, releases a flag on every peer (fence.sc.sys + st.release
// .sys).  The combine kernel here waits (ld.acquire.sys) for the W flags of
// its block, then combines the W partials in rank order -- the same fixed
// order as otk_lse_finalize, so g is bitwise identical on every rank and to
// the NCCL all-gather path.
//
// Slot reuse: rank A can write epoch e+2 into B's slot (e & 1) only after its
// own combine of e+1, which waited for B's push of e+1, which B issues after
// its combine of e finished (stream order) -- two slots suffice.
// Flags hold the epoch (monotonic, same sequence on every rank).  Epoch 0 in
// the arguments means "device-counted": the push and the combine both use one
// past the buffer's count of completed combines, and the combine's last block
// (ticket) advances the count once every block has read it -- so a captured
// CUDA graph replays the same launches epoch after epoch.  A wait that
// exceeds the timeout (default 10 s) sets the buffer's error word and gives
// up instead of hanging the GPU; otk_exchange_status reports it.
//
// The convergence check of a sharded solve (sinkhorn.py:175-189) exchanges
// its per-rank sums the same way (check_exchange_kernel): one slot of
// kChkSlot doubles per rank, a release flag per rank, fixed rank-order
// totals -- the same numbers and the same decision on every rank, with no
// host collective.
#include <cstring>

#include "otk_common.cuh"

namespace otk {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void exchange_combine_kernel(char *local, int world, int64_t m, unsigned epoch,
                                        const float *__restrict__ base, int mode, float eps,
                                        float kappa_next, float *__restrict__ out,
                                        float *__restrict__ out_bias, int *__restrict__ first_bad,
                                        int step, uint64_t timeout_ns) {
  const XLayout X(world, m);
  __shared__ int ok;
  __shared__ unsigned ep;
  const bool counted = (epoch == 0u);
  if (threadIdx.x == 0) {
    epoch = exchange_epoch(local, epoch);
    ep = epoch;
    const unsigned *flags = reinterpret_cast<const unsigned *>(local + X.flags);
    const uint64_t t0 = globaltimer_ns();
    int good = 1;
    for (int s = 0; s < world && good; ++s) {
      const unsigned *f = flags + (size_t)s * X.nblk + blockIdx.x;
      while ((int)(ld_acquire_sys(f) - epoch) < 0) {
        if (globaltimer_ns() - t0 > timeout_ns) {  // report, do not hang
          atomicExch(reinterpret_cast<unsigned *>(local), 1u);
          good = 0;
          break;
        }
      }
    }
    ok = good;
  }
  __syncthreads();
  epoch = ep;
  if (counted && threadIdx.x == 0) {
    // every block has read the epoch once it takes its ticket: the last one
    // advances the buffer's count for the next exchange
    unsigned *ticket = reinterpret_cast<unsigned *>(local + XLayout::TICKET);
    if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
      *ticket = 0u;
      __threadfence();
      atomicExch(reinterpret_cast<unsigned *>(local + XLayout::EPOCH), epoch);
    }
  }
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  // partials of this epoch, rank order; L2-only loads (peers wrote them over NVLink)
  const float *slot = reinterpret_cast<const float *>(local + X.data) +
                      (int64_t)(epoch & 1u) * world * X.m_pad + i;
  float L;
  if (!ok) {
    L = __int_as_float(0x7fc00000);
  } else if (world == 1) {
    L = __ldcg(slot);
  } else {
    float mx = -INFINITY;
    bool nan = false;
    for (int s = 0; s < world; ++s) {
      const float v = __ldcg(slot + (int64_t)s * X.m_pad);
      nan |= (v != v);
      mx = fmaxf(mx, v);
    }
    if (nan) {
      L = __int_as_float(0x7fc00000);
    } else if (mx == -INFINITY || mx == INFINITY) {
      L = mx;
    } else {
      float acc = 0.f;
      for (int s = 0; s < world; ++s) acc += ex2(__ldcg(slot + (int64_t)s * X.m_pad) - mx);
      L = mx + lg2(acc);
    }
  }
  if (mode == OTK_FIN_LOG2) {
    out[i] = L;
    return;
  }
  const float c = eps * kLn2, bi = base[i];
  const float v = (mode == OTK_FIN_SOLVER) ? eps * bi - c * L : bi + c * L;
  out[i] = v;
  if (out_bias != nullptr)
    out_bias[i] = (mode == OTK_FIN_SOLVER) ? next_bias(bi, L, eps, kappa_next) : v * kappa_next;
  if (first_bad != nullptr && bad_potential(v)) atomicMin(first_bad, step);
}

// Check-sum exchange (one block, >= world threads).  in[0..7] = this rank's
// otk_check sums, *first_bad = its first-bad step; every rank's slot gets
// {in[0..7], first_bad, own error word}, then out[0..7] = rank-order totals
// (g terms [3], [5], [7] are replicated: rank 0's), out[8] = min first_bad,
// out[9] = max error word (any rank's exchange timeout -> all ranks see it).
__global__ void check_exchange_kernel(char *local, int world, int rank, int64_t m, const double *__restrict__ in,
                                      const int *__restrict__ first_bad, double *__restrict__ out,
                                      uint64_t timeout_ns) {
  const XLayout X(world, m);
  __shared__ unsigned ep;
  __shared__ int ok;
  char *const *peers = reinterpret_cast<char *const *>(local + X.table);
  if (threadIdx.x == 0) ep = ld_cg_u32(local + XLayout::CHK_EPOCH) + 1u;
  __syncthreads();
  const unsigned epoch = ep;
  const int64_t off = ((int64_t)(epoch & 1u) * world + rank) * kChkSlot;
  for (int s = threadIdx.x; s < world; s += blockDim.x) {
    double *slot = reinterpret_cast<double *>(peers[s] + X.chk) + off;
    for (int k = 0; k < 8; ++k) slot[k] = in[k];
    slot[8] = (double)*first_bad;
    slot[9] = (double)ld_cg_u32(local + XLayout::ERR);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int s = 0; s < world; ++s) {
      unsigned *flag = reinterpret_cast<unsigned *>(peers[s] + X.chkflags) + rank;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
    }
    const unsigned *flags = reinterpret_cast<const unsigned *>(local + X.chkflags);
    const uint64_t t0 = globaltimer_ns();
    int good = 1;
    for (int s = 0; s < world && good; ++s) {
      while ((int)(ld_acquire_sys(flags + s) - epoch) < 0) {
        if (globaltimer_ns() - t0 > timeout_ns) {
          atomicExch(reinterpret_cast<unsigned *>(local), 1u);
          good = 0;
          break;
        }
      }
    }
    ok = good;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double *slots = reinterpret_cast<const double *>(local + X.chk) + (int64_t)(epoch & 1u) * world * kChkSlot;
    double tot[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (ok) {
      tot[8] = 2147483647.0;
      for (int s = 0; s < world; ++s) {  // fixed rank order: identical on every rank
        const double *v = slots + (int64_t)s * kChkSlot;
        for (int k = 0; k < 8; ++k) {
          const double x = __ldcg(v + k);
          if (k == 3 || k == 5 || k == 7) { if (s == 0) tot[k] = x; }
          else tot[k] += x;
        }
        tot[8] = fmin(tot[8], __ldcg(v + 8));
        tot[9] = fmax(tot[9], __ldcg(v + 9));
      }
    } else {
      tot[9] = 1.0;
    }
    for (int k = 0; k < 10; ++k) out[k] = tot[k];
    tot[9] = fmax(tot[9], (double)ld_cg_u32(local + XLayout::ERR));
    out[9] = tot[9];
    __threadfence();
    atomicExch(reinterpret_cast<unsigned *>(local + XLayout::CHK_EPOCH), epoch);
  }
}

}  // namespace otk

using namespace otk;

extern "C" {

size_t otk_exchange_bytes(int32_t world, int64_t m) {
  if (world < 1 || m < 1) return 0;
  return XLayout(world, m).total;
}

int otk_exchange_alloc(size_t bytes, void **ptr) {
  OTK_CHECK_ARG(ptr && bytes > 0, "otk_exchange_alloc: bad arguments");
  OTK_CUDA(cudaMalloc(ptr, bytes));
  OTK_CUDA(cudaMemset(*ptr, 0, bytes));
  return OTK_OK;
}

int otk_exchange_free(void *ptr) {
  if (ptr) OTK_CUDA(cudaFree(ptr));
  return OTK_OK;
}

int otk_ipc_handle(void *ptr, void *handle) {
  OTK_CHECK_ARG(ptr && handle, "otk_ipc_handle: bad arguments");
  cudaIpcMemHandle_t h;
  OTK_CUDA(cudaIpcGetMemHandle(&h, ptr));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, sizeof(h));
  return OTK_OK;
}

int otk_ipc_open(const void *handle, void **ptr) {
  OTK_CHECK_ARG(ptr && handle, "otk_ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  OTK_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return OTK_OK;
}

int otk_ipc_close(void *ptr) {
  if (ptr) OTK_CUDA(cudaIpcCloseMemHandle(ptr));
  return OTK_OK;
}

int otk_exchange_set_peers(void *local, int32_t world, int64_t m, void *const *peers,
                           void *stream) {
  OTK_CHECK_ARG(local && peers && world >= 1 && m >= 1, "otk_exchange_set_peers: bad arguments");
  const XLayout X(world, m);
  OTK_CUDA(cudaMemcpyAsync(static_cast<char *>(local) + X.table, peers, sizeof(void *) * world,
                           cudaMemcpyHostToDevice, as_stream(stream)));
  OTK_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return OTK_OK;
}

int otk_exchange_finalize(void *local, int32_t world, int64_t m, uint32_t epoch, const float *base,
                          int32_t mode, float eps, float kappa_next, float *out_pot,
                          float *out_bias, int32_t *first_bad, int32_t step, uint32_t timeout_ms,
                          void *stream) {
  OTK_CHECK_ARG(local && out_pot && world >= 1 && m >= 1, "otk_exchange_finalize: bad arguments");
  OTK_CHECK_ARG(mode == OTK_FIN_SOLVER || mode == OTK_FIN_APPLY || mode == OTK_FIN_LOG2,
                "otk_exchange_finalize: bad mode");
  OTK_CHECK_ARG(base || mode == OTK_FIN_LOG2, "otk_exchange_finalize: base required");
  const XLayout X(world, m);
  exchange_combine_kernel<<<X.nblk, 256, 0, as_stream(stream)>>>(
      static_cast<char *>(local), world, m, epoch, base, mode, eps, kappa_next, out_pot, out_bias,
      first_bad, step, (uint64_t)(timeout_ms ? timeout_ms : 10000u) * 1000000ull);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_exchange_check(void *local, int32_t world, int32_t rank, int64_t m, const double *sums,
                       const int32_t *first_bad, double *out, uint32_t timeout_ms, void *stream) {
  OTK_CHECK_ARG(local && sums && first_bad && out && world >= 1 && rank >= 0 && rank < world && m >= 1,
                "otk_exchange_check: bad arguments");
  check_exchange_kernel<<<1, 32, 0, as_stream(stream)>>>(
      static_cast<char *>(local), world, rank, m, sums, first_bad, out,
      (uint64_t)(timeout_ms ? timeout_ms : 10000u) * 1000000ull);
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

int otk_exchange_status(void *local, int32_t *status, void *stream) {
  OTK_CHECK_ARG(local && status, "otk_exchange_status: bad arguments");
  unsigned v = 0;
  OTK_CUDA(cudaMemcpyAsync(&v, local, sizeof(v), cudaMemcpyDeviceToHost, as_stream(stream)));
  OTK_CUDA(cudaStreamSynchronize(as_stream(stream)));
  *status = (int32_t)v;
  return OTK_OK;
}

}  // extern "C"
