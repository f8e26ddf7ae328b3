// kernels_misc.cu — vector plumbing around the FMM: caller-order <-> Morton-order permutations
// (reference solver.cpp:327-331), FP64 <-> FP32 conversion at the boundary.
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
  const float2 a = near[slot], b = far[slot];
  const uint32_t i = index[slot];
  if (o64)
    o64[i] = make_double2(double(a.x) + double(b.x), double(a.y) + double(b.y));
  else
    o32[i] = make_float2(a.x + b.x, a.y + b.y);
}

}  // namespace

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

}  // namespace hfmm_b200
