// Pipe-throughput microbenchmarks used by bench.py to measure the
// denominators of the online kernel's compute roof on the box itself:
// MUFU ex2 (one per cell per half-step) and FP32 FFMA.
#include "otk_common.cuh"

namespace otk {

constexpr int PB_CHAINS = 8;

__global__ void __launch_bounds__(256) ex2_pipe_kernel(float *out, int iters, float seed) {
  float v[PB_CHAINS];
#pragma unroll
  for (int c = 0; c < PB_CHAINS; ++c) v[c] = seed * (threadIdx.x + c) * 1e-7f - 0.5f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < PB_CHAINS; ++c) v[c] = ex2(v[c]) - 1.0f;  // stays in (-0.5, 0.5)
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < PB_CHAINS; ++c) s += v[c];
  if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) fma_pipe_kernel(float *out, int iters, float seed) {
  float v[PB_CHAINS];
#pragma unroll
  for (int c = 0; c < PB_CHAINS; ++c) v[c] = seed * (threadIdx.x + c);
  const float a = 0.999999f, b = 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < PB_CHAINS; ++c) v[c] = fmaf(v[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < PB_CHAINS; ++c) s += v[c];
  if (s == 12345.f) out[threadIdx.x] = s;
}

// Streaming read of a buffer (float4, grid-stride, 8 loads in flight per thread):
// the achievable HBM READ rate that bounds the materialised-cost half-steps.
__global__ void __launch_bounds__(256) read_bw_kernel(const float4 *__restrict__ p, int64_t n4,
                                                      float *out) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(p + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  for (; i < n4; i += stride) {
    const float4 v = __ldcs(p + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

// Shared-memory read bandwidth: every thread streams LDS.128 over a 32 KB
// tile (conflict-free, 8 loads in flight) -- the roof of the scaling-domain
// batched solve, which reads 4 B of its stored kernel per cell per half-step.
__global__ void __launch_bounds__(512) smem_read_kernel(float *out, int iters) {
  __shared__ float4 tile[2048];  // 32 KB
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    tile[i] = make_float4((float)i, 1.f, 2.f, 3.f);
  __syncthreads();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = tile[(threadIdx.x + k * 512 + it) & 2047];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[threadIdx.x] = acc.x;
}

}  // namespace otk

using namespace otk;

extern "C" int otk_bench_smem(double *bytes_per_s, void *stream) {
  OTK_CHECK_ARG(bytes_per_s, "otk_bench_smem: null output");
  cudaStream_t st = as_stream(stream);
  float *scratch = nullptr;
  OTK_CUDA(cudaMallocAsync(&scratch, 512 * sizeof(float), st));
  cudaEvent_t e0, e1;
  OTK_CUDA(cudaEventCreate(&e0));
  OTK_CUDA(cudaEventCreate(&e1));
  const int blocks = num_sms() * 2, threads = 512, iters = 2048;
  const double bytes = (double)blocks * threads * iters * 8 * 16;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    smem_read_kernel<<<blocks, threads, 0, st>>>(scratch, iters);
    cudaEventRecord(e1, st);
    OTK_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::max(best, bytes / (ms * 1e-3));
  }
  *bytes_per_s = best;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  OTK_CUDA(cudaFreeAsync(scratch, st));
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

extern "C" int otk_bench_read(const float *buf, int64_t bytes, double *gbs, void *stream) {
  OTK_CHECK_ARG(buf && gbs && bytes >= 16, "otk_bench_read: bad arguments");
  cudaStream_t st = as_stream(stream);
  float *scratch = nullptr;
  OTK_CUDA(cudaMallocAsync(&scratch, sizeof(float), st));
  cudaEvent_t e0, e1;
  OTK_CUDA(cudaEventCreate(&e0));
  OTK_CUDA(cudaEventCreate(&e1));
  const int64_t n4 = bytes / 16;
  const int blocks = num_sms() * 8;
  double best = 0.0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0, st);
    read_bw_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const float4 *>(buf), n4, scratch);
    cudaEventRecord(e1, st);
    OTK_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::max(best, (double)(n4 * 16) / (ms * 1e-3) / 1e9);
  }
  *gbs = best;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  OTK_CUDA(cudaFreeAsync(scratch, st));
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}

extern "C" int otk_bench_pipes(double *ex2_per_s, double *ffma_per_s, void *stream) {
  OTK_CHECK_ARG(ex2_per_s && ffma_per_s, "otk_bench_pipes: null output");
  cudaStream_t st = as_stream(stream);
  float *scratch = nullptr;
  OTK_CUDA(cudaMallocAsync(&scratch, 256 * sizeof(float), st));
  const int blocks = num_sms() * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  OTK_CUDA(cudaEventCreate(&e0));
  OTK_CUDA(cudaEventCreate(&e1));
  float ms = 0.f;
  double ops = (double)blocks * threads * PB_CHAINS * iters;
  // warm up + measure (best of 3)
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    ex2_pipe_kernel<<<blocks, threads, 0, st>>>(scratch, iters, 1.f);
    cudaEventRecord(e1, st);
    OTK_CUDA(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::max(best, ops / (ms * 1e-3));
  }
  *ex2_per_s = best;
  best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    fma_pipe_kernel<<<blocks, threads, 0, st>>>(scratch, iters, 1.f);
    cudaEventRecord(e1, st);
    OTK_CUDA(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::max(best, ops / (ms * 1e-3));
  }
  *ffma_per_s = best;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  OTK_CUDA(cudaFreeAsync(scratch, st));
  OTK_LAUNCH_CHECK();
  return OTK_OK;
}
