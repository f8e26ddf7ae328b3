// Shared-memory pipe cost of the access patterns the translation kernel can use for warp-shared data
// (B200, sm_100a).  One CTA of 256 threads per SM, every warp issues the same LDS in a long unrolled loop;
// cycles per instruction and SM = elapsed cycles / (instructions per warp x warps / 1) — the data pipe is
// shared by the SM's warps, so with 8 warps in flight the figure is the pipe's occupancy per instruction.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_patterns.bin lds_patterns.cu && ./lds_patterns.bin
#include <cstdio>
#include <cuda_runtime.h>

template <int WIDTH>
__device__ __forceinline__ float lds_any(unsigned addr) {
  if (WIDTH == 4) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
  } else if (WIDTH == 8) {
    float a, b;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a), "=f"(b) : "r"(addr) : "memory");
    return a + b;
  } else {
    float a, b, c, d;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(addr) : "memory");
    return a + b + c + d;
  }
}

// pattern: byte offset of a lane
//  0 uniform | 1 lane * WIDTH (contiguous) | 2 (lane >> 1) * WIDTH (adjacent lanes share) | 3 (lane & 1) * WIDTH (two addresses)
//  4 (lane >> 2) * WIDTH | 5 (lane & 3) * WIDTH (four addresses) | 6 (lane >> 4) * WIDTH (one address per half warp)
template <int WIDTH, int PATTERN>
__global__ void probe(float* out, long long* cycles, int iters) {
  extern __shared__ __align__(16) float smem[];
  for (int i = threadIdx.x; i < 8192 + 256; i += blockDim.x) smem[i] = float(i & 7);
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  unsigned off = 0;
  if (PATTERN == 1) off = lane * WIDTH;
  if (PATTERN == 2) off = (lane >> 1) * WIDTH;
  if (PATTERN == 3) off = (lane & 1) * WIDTH;
  if (PATTERN == 4) off = (lane >> 2) * WIDTH;
  if (PATTERN == 5) off = (lane & 3) * WIDTH;
  if (PATTERN == 6) off = (lane >> 4) * WIDTH;
  const unsigned base = unsigned(__cvta_generic_to_shared(smem)) + off;
  float acc = 0.f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += lds_any<WIDTH>(base + 512u * j + ((unsigned(it) & 1u) << 14));
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int WIDTH, int PATTERN>
void run(const char* name) {
  const int ctas = 148, threads = 256, iters = 2000;
  float* out;
  long long* cyc;
  cudaMalloc(&out, ctas * threads * sizeof(float));
  cudaMalloc(&cyc, ctas * sizeof(long long));
  probe<WIDTH, PATTERN><<<ctas, threads, 34816>>>(out, cyc, iters);
  probe<WIDTH, PATTERN><<<ctas, threads, 34816>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < ctas; ++i) mean += double(h[i]);
  mean /= ctas;
  const double per = mean / (double(iters) * 32 * (threads / 32));
  printf("LDS.%-3d %-28s %.2f cycles of the pipe per warp instruction\n", WIDTH * 8, name, per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<4, 0>("uniform");
  run<4, 1>("contiguous (128 B)");
  run<4, 3>("two addresses (lane & 1)");
  run<8, 0>("uniform");
  run<8, 1>("contiguous (256 B)");
  run<8, 2>("lane pairs share (128 B)");
  run<8, 3>("two addresses (lane & 1)");
  run<8, 4>("lane quads share (64 B)");
  run<8, 5>("four addresses (lane & 3)");
  run<8, 6>("one address per half warp");
  run<16, 0>("uniform");
  run<16, 1>("contiguous (512 B)");
  run<16, 2>("lane pairs share (256 B)");
  run<16, 3>("two addresses (lane & 1)");
  run<16, 4>("lane quads share (128 B)");
  run<16, 5>("four addresses (lane & 3)");
  run<16, 6>("one address per half warp");
  return 0;
}
