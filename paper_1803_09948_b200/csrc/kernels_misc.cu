// kernels_misc.cu — vector plumbing around the FMM: caller-order <-> Morton-order permutations
// (reference solver.cpp:327-331), FP64 <-> FP32 conversion at the boundary.
#include <algorithm>

#include "device_utils.cuh"
#include "kernels.cuh"

namespace hfmm_b200 {

namespace {

__global__ void gather_charges_kernel(const double2* __restrict__ q64, const float2* __restrict__ q32,
                                      const uint32_t* __restrict__ index,
                                      const float* __restrict__ weight, float2* __restrict__ body_q,
                                      uint32_t n) {
  const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= n) return;
  const uint32_t i = index[slot];
  float2 v;
  if (q64) {
    const double2 d = q64[i];
    v = make_float2(float(d.x), float(d.y));
  } else {
    v = q32[i];
  }
  if (weight) {
    const float w = weight[i];
    v.x *= w;
    v.y *= w;
  }
  body_q[slot] = v;
}

__global__ void scatter_potentials_kernel(const float2* __restrict__ near, const float2* __restrict__ far,
                                          const uint32_t* __restrict__ index, double2* __restrict__ o64,
                                          float2* __restrict__ o32, uint32_t n) {
  const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= n) return;
  const float2 a = near[slot], b = far ? far[slot] : make_float2(0.f, 0.f);
  const uint32_t i = index[slot];
  if (o64)
    o64[i] = make_double2(double(a.x) + double(b.x), double(a.y) + double(b.y));
  else
    o32[i] = make_float2(a.x + b.x, a.y + b.y);
}

// FFMA-only probe: 16 independent chains per thread, no memory traffic.  Gives the FP32 roofline
// denominator actually reachable on this part at its running clock (MEASURED_PEAKS.json carries no
// FP32 entry; nominal is SMs x 128 lanes x 2 x clock).
__global__ void __launch_bounds__(256) fp32_peak_kernel(float* out, int iters, float a, float b) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = float(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = fmaf(v[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  if (s == 123.456f) out[0] = s;  // never true; keeps the chains alive
}

// the same with packed FFMA2 (fma.rn.f32x2, two FMAs per instruction, sm_100+): 8 chains of pairs
__global__ void __launch_bounds__(256) fp32x2_peak_kernel(float* out, int iters, float a, float b) {
  unsigned long long v[8], av, bv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(b));
#pragma unroll
  for (int i = 0; i < 8; ++i)
    asm("mov.b64 %0, {%1, %2};" : "=l"(v[i]) : "f"(float(threadIdx.x + i)), "f"(float(threadIdx.x + i + 8)));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[i]) : "l"(av), "l"(bv));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v[i]));
    s += lo + hi;
  }
  if (s == 123.456f) out[0] = s;
}

// out[s] = near[s] + far[s] + corr[index[s]] for the owned Morton slots (corr in caller order, may be null)
__global__ void combine_owned_kernel(const float2* __restrict__ near, const float2* __restrict__ far,
                                     const float2* __restrict__ corr, const uint32_t* __restrict__ index,
                                     float2* __restrict__ out, uint32_t n) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  float2 v = near[s];
  const float2 f = far[s];
  v.x += f.x;
  v.y += f.y;
  if (corr) {
    const float2 c = corr[index[s]];
    v.x += c.x;
    v.y += c.y;
  }
  out[s] = v;
}

}  // namespace

void launch_combine_owned(const float2* near, const float2* far, const float2* corr, const uint32_t* index,
                          float2* out, uint32_t n, cudaStream_t s) {
  if (!n) return;
  combine_owned_kernel<<<(n + 255) / 256, 256, 0, s>>>(near, far, corr, index, out, n);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

double run_fp32_peak_probe(cudaStream_t s, bool packed) {
  int dev = 0, sms = 0;
  HFMM_CUDA_CHECK(cudaGetDevice(&dev));
  HFMM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float* out = nullptr;
  HFMM_CUDA_CHECK(cudaMalloc(&out, 4));
  cudaEvent_t e0, e1;
  HFMM_CUDA_CHECK(cudaEventCreate(&e0));
  HFMM_CUDA_CHECK(cudaEventCreate(&e1));
  const int iters = 1 << 14, blocks = sms * 8, threads = 256;
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    HFMM_CUDA_CHECK(cudaEventRecord(e0, s));
    if (packed) fp32x2_peak_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.999f, 0.001f);
    else fp32_peak_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.999f, 0.001f);
    HFMM_CUDA_CHECK(cudaEventRecord(e1, s));
    HFMM_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0;
    HFMM_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * 16.0 * double(iters) * double(blocks) * threads;
    if (rep > 0) best = std::max(best, flops / (double(ms) * 1e-3) * 1e-12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}

void launch_gather_charges(const double2* q64, const float2* q32, const uint32_t* index,
                           const float* weight, float2* body_q, uint32_t n, cudaStream_t s) {
  if (!n) return;
  gather_charges_kernel<<<(n + 255) / 256, 256, 0, s>>>(q64, q32, index, weight, body_q, n);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

void launch_scatter_potentials(const float2* near, const float2* far, const uint32_t* index,
                               double2* o64, float2* o32, uint32_t n, cudaStream_t s) {
  if (!n) return;
  scatter_potentials_kernel<<<(n + 255) / 256, 256, 0, s>>>(near, far, index, o64, o32, n);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

namespace {
constexpr int kReduceWarps = 4;
constexpr int kMaxChunks = (kMaxOrder + 1) * (kMaxOrder + 1) / 32 + 1;

__global__ void __launch_bounds__(kReduceWarps * 32)
ordered_reduce_kernel(const float2* __restrict__ staging, const uint32_t* __restrict__ perm,
                      const uint32_t* __restrict__ seg_begin, const uint32_t* __restrict__ seg_dst,
                      uint32_t n_segs, float2* __restrict__ dst, uint32_t stride, uint32_t dim) {
  const uint32_t seg = blockIdx.x * kReduceWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (seg >= n_segs) return;
  float2* out = dst + size_t(seg_dst[seg]) * stride;
  float2 acc[kMaxChunks];
#pragma unroll
  for (int u = 0; u < kMaxChunks; ++u) {
    const uint32_t c = lane + 32u * u;
    acc[u] = c < dim ? out[c] : make_float2(0.f, 0.f);
  }
  for (uint32_t j = seg_begin[seg]; j < seg_begin[seg + 1]; ++j) {
    const float2* row = staging + size_t(perm[j]) * stride;
#pragma unroll
    for (int u = 0; u < kMaxChunks; ++u) {
      const uint32_t c = lane + 32u * u;
      if (c < dim) {
        const float2 v = row[c];
        acc[u].x += v.x;
        acc[u].y += v.y;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kMaxChunks; ++u) {
    const uint32_t c = lane + 32u * u;
    if (c < dim) out[c] = acc[u];
  }
}

__global__ void range_rows_kernel(uint32_t* out, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = i;
}
}  // namespace

void launch_ordered_reduce(const float2* staging, const uint32_t* perm, const uint32_t* seg_begin,
                           const uint32_t* seg_dst, uint32_t n_segs, float2* dst, uint32_t stride,
                           uint32_t dim, cudaStream_t s) {
  if (!n_segs) return;
  ordered_reduce_kernel<<<(n_segs + kReduceWarps - 1) / kReduceWarps, kReduceWarps * 32, 0, s>>>(
      staging, perm, seg_begin, seg_dst, n_segs, dst, stride, dim);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

void launch_range_rows(uint32_t* row_of_pair, uint64_t begin, uint32_t n, cudaStream_t s) {
  if (!n) return;
  range_rows_kernel<<<(n + 255) / 256, 256, 0, s>>>(row_of_pair + begin, n);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

}  // namespace hfmm_b200
