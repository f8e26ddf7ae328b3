// Micro-benchmark: how well do the MUFU (XU) pipe and packed FP32 (FFMA2) overlap on sm_100a?
// Each warp runs ITER iterations of a block with NM MUFU and NF FFMA2 instructions arranged as CH
// independent chains (like one target group of the near-field kernel).  Prints clocks per block per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
using u64 = unsigned long long;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float rsq(float x) { float y; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float cosa(float x) { float y; asm volatile("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ u64 pack2(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float2 unpack2(u64 v) { float2 r; asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }

// MODE 0: 3 MUFU per value (rsq, cos, "sin"=cos) + 13 packed per pair-of-values;  MODE 1: 2 MUFU + 18 packed
template <int CH, int MODE>
__global__ void mix(float* out, int iters, long long* clk) {
  u64 acc[CH], x[CH];
  for (int c = 0; c < CH; ++c) { acc[c] = pack2(threadIdx.x * 1e-3f, 1.f); x[c] = pack2(1.f + c + threadIdx.x * 1e-4f, 2.f + c); }
  const u64 k = pack2(1.0001f, 0.9999f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      u64 r2 = x[c];
      // 6 packed: differences + r2
      r2 = fma2(r2, k, acc[c]); r2 = fma2(r2, k, x[c]); r2 = fma2(r2, r2, k);
      r2 = fma2(r2, k, k); r2 = fma2(r2, k, k); r2 = fma2(r2, k, k);
      float2 f = unpack2(r2);
      u64 ri = (MODE == 2) ? r2 : pack2(rsq(f.x), rsq(f.y));
      u64 r = fma2(r2, ri, 0ull);
      float2 g = unpack2(r);
      u64 c2 = (MODE == 2) ? r : pack2(cosa(g.x), cosa(g.y));
      u64 s2;
      if (MODE == 0) { s2 = pack2(cosa(g.x + 1.f), cosa(g.y + 1.f)); s2 = fma2(s2, ri, 0ull); }
      else if (MODE == 3) { s2 = pack2(cosa(g.x + 1.f), cosa(g.y + 1.f)); }
      else { s2 = k; for (int i = 0; i < 6; ++i) s2 = fma2(s2, r2, k); }
      c2 = fma2(c2, ri, 0ull);
      acc[c] = fma2(c2, k, acc[c]); acc[c] = fma2(s2, k, acc[c]);
      x[c] = fma2(c2, k, x[c]); x[c] = fma2(s2, k, x[c]);
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < CH; ++c) { float2 a = unpack2(acc[c]), b = unpack2(x[c]); s += a.x + a.y + b.x + b.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
template <int CH, int MODE>
void run(int warps_per_sm) {
  float* out; long long* clk; cudaMalloc(&out, 148 * 2048 * 4); cudaMalloc(&clk, 8);
  const int iters = 2000;
  // one block per SM with warps_per_sm warps
  mix<CH, MODE><<<148, warps_per_sm * 32>>>(out, iters, clk);
  mix<CH, MODE><<<148, warps_per_sm * 32>>>(out, iters, clk);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  // per SMSP: warps_per_sm/4 warps each doing iters*CH chain-bodies
  double per_chain = double(h) / (double(iters) * CH * (warps_per_sm / 4.0));
  printf("CH=%d MODE=%d warps/SMSP=%d : %.1f clk per chain-body per SMSP (MUFU-bound: %d, FMA-bound: %d)\n", CH, MODE,
         warps_per_sm / 4, per_chain, MODE == 0 ? 48 : 32, MODE == 0 ? 2 * 13 : 2 * 18);
  cudaFree(out); cudaFree(clk);
}
int main() {
  for (int w : {16, 32}) { run<4, 0>(w); run<4, 1>(w); run<4, 2>(w); run<4, 3>(w); }
  return 0;
}
