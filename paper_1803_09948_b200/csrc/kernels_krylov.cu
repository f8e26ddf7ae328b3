// kernels_krylov.cu — device side of the BIE operator tail and of restarted GMRES (sm_100a).
//
//   corrections : y += blockdiag(patch_block) x + CSR(near_delta) x        (solver.cpp:340-357)
//   precondition: per-patch LU solve with recorded pivots                   (solver.cpp:65-74,376-382)
//   Krylov ops  : the dot / axpy / norm / scale loops of gmres.cpp:13-23,103-113,156
// All of it is HBM-bound streaming.  Krylov basis vectors are complex FP32; every reduction
// accumulates in FP64 and lands in a device scalar, so one modified-Gram-Schmidt sweep is a chain
// of fused kernels (subtract the previous projection while dotting with the next basis vector)
// with no host round trip until the Hessenberg column is read back.
#include <algorithm>

#include "device_utils.cuh"
#include "kernels.cuh"

namespace hfmm_b200 {

namespace {

constexpr int kBlock = 256;
constexpr uint32_t kReduceBlocks = 148u * 8u;  // most blocks a reducing kernel is launched with

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum of a (re, im) pair (fixed order)
__device__ __forceinline__ void block_sum(double& re, double& im) {
  __shared__ double s_re[kBlock / 32], s_im[kBlock / 32];
  re = warp_sum_d(re);
  im = warp_sum_d(im);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // the previous use of s_re / s_im is over
  if (lane == 0) {
    s_re[warp] = re;
    s_im[warp] = im;
  }
  __syncthreads();
  re = lane < kBlock / 32 ? s_re[lane] : 0.0;
  im = lane < kBlock / 32 ? s_im[lane] : 0.0;
  re = warp_sum_d(re);
  im = warp_sum_d(im);
}

// Grid-wide sum into out[0], out[1] with a run-to-run reproducible result: every block parks its
// partial in scratch, and the block that arrives last (a ticket counter behind the partials) adds
// them up in block order — no floating-point atomics, whose order would change between runs
// (the reference accumulates in a fixed order too: gmres.cpp:13-23).
__device__ __forceinline__ void grid_accumulate(double re, double im, double* out, double* scratch) {
  __shared__ bool s_last;
  block_sum(re, im);
  unsigned* ticket = reinterpret_cast<unsigned*>(scratch + 2 * kReduceBlocks);
  if (threadIdx.x == 0) {
    scratch[2 * blockIdx.x] = re;
    scratch[2 * blockIdx.x + 1] = im;
    __threadfence();
    s_last = atomicInc(ticket, gridDim.x - 1) == gridDim.x - 1;  // wraps to 0 for the next launch
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  re = im = 0.0;
  for (uint32_t b = threadIdx.x; b < gridDim.x; b += kBlock) {
    re += __ldcg(scratch + 2 * b);
    im += __ldcg(scratch + 2 * b + 1);
  }
  block_sum(re, im);
  if (threadIdx.x == 0) {
    out[0] += re;
    out[1] += im;
  }
}

// FP64 values, FP64 accumulation: the corrections carry the near-singular part of the operator — large
// entries that cancel against the point-kernel near field — and are HBM-bound either way.  Measured on an
// ill-conditioned first-kind system (lat-long sphere, 864 unknowns): FP32 corrections alone took
// block-Jacobi GMRES(30) from 28 to 58 iterations.
__global__ void __launch_bounds__(kBlock)
corrections_kernel(uint32_t n, int ni, const double2* __restrict__ block, const uint32_t* __restrict__ off,
                   const uint32_t* __restrict__ src, const double2* __restrict__ delta,
                   const float2* __restrict__ x, float2* __restrict__ y) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ar = 0.0, ai = 0.0;
  if (block) {
    const uint32_t p = i / uint32_t(ni), r = i - p * uint32_t(ni);
    const double2* row = block + (size_t(p) * ni + r) * ni;
    const float2* xp = x + size_t(p) * ni;
    for (int c = 0; c < ni; ++c) {
      const double2 b = row[c];
      const float2 v = xp[c];
      ar += b.x * v.x - b.y * v.y;
      ai += b.x * v.y + b.y * v.x;
    }
  }
  if (delta) {
    for (uint32_t e = off[i]; e < off[i + 1]; ++e) {
      const double2 d = delta[e];
      const float2 v = x[src[e]];
      ar += d.x * v.x - d.y * v.y;
      ai += d.x * v.y + d.y * v.x;
    }
  }
  const float2 o = y[i];
  y[i] = make_float2(float(double(o.x) + ar), float(double(o.y) + ai));
}

constexpr int kMaxNi = 12;  // basis orders 1, 2, 3 -> 3, 6, 12 nodes per patch (geometry.cpp:145-171)

__global__ void __launch_bounds__(kBlock)
precondition_kernel(uint32_t npatch, int ni, const double2* __restrict__ lu, const int* __restrict__ piv,
                    const float2* __restrict__ in, float2* __restrict__ out) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npatch) return;
  double2 v[kMaxNi];  // lu_solve (solver.cpp:65-74) in FP64: the factors of small patches are badly scaled
  for (int c = 0; c < ni; ++c) {
    const float2 t = in[size_t(p) * ni + c];
    v[c] = make_double2(t.x, t.y);
  }
  const double2* a = lu + size_t(p) * ni * ni;
  const int* pv = piv + size_t(p) * ni;
  for (int c = 0; c < ni; ++c) {
    const int q = pv[c];
    if (q != c) {
      const double2 t = v[c];
      v[c] = v[q];
      v[q] = t;
    }
    for (int r = c + 1; r < ni; ++r) {
      const double2 l = a[r * ni + c];
      v[r].x -= l.x * v[c].x - l.y * v[c].y;
      v[r].y -= l.x * v[c].y + l.y * v[c].x;
    }
  }
  for (int r = ni - 1; r >= 0; --r) {
    for (int c = r + 1; c < ni; ++c) {
      const double2 u = a[r * ni + c];
      v[r].x -= u.x * v[c].x - u.y * v[c].y;
      v[r].y -= u.x * v[c].y + u.y * v[c].x;
    }
    const double2 d = a[r * ni + r];
    const double den = d.x * d.x + d.y * d.y;
    const double2 t = v[r];
    v[r] = make_double2((t.x * d.x + t.y * d.y) / den, (t.y * d.x - t.x * d.y) / den);
  }
  for (int c = 0; c < ni; ++c) out[size_t(p) * ni + c] = make_float2(float(v[c].x), float(v[c].y));
}

// w -= h_prev * v_prev (if v_prev), then out += conj(v_next) . w (if v_next)
__global__ void __launch_bounds__(kBlock)
mgs_step_kernel(uint32_t n, float2* __restrict__ w, const float2* __restrict__ v_prev,
                const double* __restrict__ h_prev, const float2* __restrict__ v_next, double* out,
                double* scratch) {
  double re = 0, im = 0;
  float hr = 0.f, hi = 0.f;
  if (v_prev) {
    hr = float(h_prev[0]);
    hi = float(h_prev[1]);
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float2 x = w[i];
    if (v_prev) {
      const float2 v = v_prev[i];
      x.x -= hr * v.x - hi * v.y;
      x.y -= hr * v.y + hi * v.x;
      w[i] = x;
    }
    if (v_next) {
      const float2 v = v_next[i];
      re += double(v.x) * x.x + double(v.y) * x.y;   // conj(v) * x
      im += double(v.x) * x.y - double(v.y) * x.x;
    }
  }
  if (v_next) grid_accumulate(re, im, out, scratch);
}

// out[0] += ||w||^2
__global__ void __launch_bounds__(kBlock)
norm2_kernel(uint32_t n, const float2* __restrict__ w, double* out, double* scratch) {
  double s = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float2 x = w[i];
    s += double(x.x) * x.x + double(x.y) * x.y;
  }
  grid_accumulate(s, 0.0, out, scratch);
}

__global__ void __launch_bounds__(kBlock)
scale_kernel(uint32_t n, const float2* __restrict__ in, float scale, float2* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float2 x = in[i];
  out[i] = make_float2(x.x * scale, x.y * scale);
}

// x += sum_i y[i] * V_i   (x in FP64, y on device as interleaved doubles)
__global__ void __launch_bounds__(kBlock)
update_solution_kernel(uint32_t n, int cols, const float2* __restrict__ basis, size_t ld,
                       const double* __restrict__ y, double2* __restrict__ x) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 acc = x[i];
  for (int c = 0; c < cols; ++c) {
    const float2 v = basis[size_t(c) * ld + i];
    const double yr = y[2 * c], yi = y[2 * c + 1];
    acc.x += yr * v.x - yi * v.y;
    acc.y += yr * v.y + yi * v.x;
  }
  x[i] = acc;
}

// r = b - ax (FP64), r32 = float(r), out[0] += ||r||^2
__global__ void __launch_bounds__(kBlock)
residual_kernel(uint32_t n, const double2* __restrict__ b, const float2* __restrict__ ax,
                float2* __restrict__ r32, double* out, double* scratch) {
  double s = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double2 bb = b[i];
    const float2 a = ax[i];
    const double rr = bb.x - double(a.x), ri = bb.y - double(a.y);
    r32[i] = make_float2(float(rr), float(ri));
    s += rr * rr + ri * ri;
  }
  grid_accumulate(s, 0.0, out, scratch);
}

__global__ void __launch_bounds__(kBlock)
narrow_kernel(uint32_t n, const double2* __restrict__ in, float2* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 v = in[i];
  out[i] = make_float2(float(v.x), float(v.y));
}

__global__ void __launch_bounds__(kBlock)
widen_kernel(uint32_t n, const float2* __restrict__ in, double2* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float2 v = in[i];
  out[i] = make_double2(double(v.x), double(v.y));
}

// plain single-layer sum at exterior points (solver.cpp:393-419): one block per observation.
// x_i - o is formed in FP64 from the FP64 points (absolute FP32 coordinates would cost a phase error of
// ulp(k |x|)); the kernel value itself is complex FP32 like the rest of the path.  touch2: squared touch
// radius per patch (0.1 x diameter, solver.cpp:399-403), or null; a sample within it raises *flag.
__global__ void __launch_bounds__(kBlock)
field_kernel(uint32_t n, const double* __restrict__ xyz, const float2* __restrict__ q, const double* __restrict__ obs,
             double k, float scale, float eps, const double* __restrict__ touch2, uint32_t ni,
             double2* __restrict__ out, int* __restrict__ flag) {
  const double ox = obs[3 * blockIdx.x], oy = obs[3 * blockIdx.x + 1], oz = obs[3 * blockIdx.x + 2];
  double re = 0, im = 0;
  bool touched = false;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double ddx = ox - xyz[3 * i], ddy = oy - xyz[3 * i + 1], ddz = oz - xyz[3 * i + 2];
    const double d2 = ddx * ddx + ddy * ddy + ddz * ddz;
    if (touch2 && d2 <= touch2[i / ni]) touched = true;
    const float2 c = q[i];
    const float dx = float(k * ddx), dy = float(k * ddy), dz = float(k * ddz);
    const float r2 = dx * dx + dy * dy + dz * dz;
    if (r2 > 0.f) {
      const float r0 = rsqrtf(r2), r = r2 * r0;
      const float rinv = eps != 0.0f ? r0 * expf(-eps * r) : r0;  // complex k: e^{-k_i R} (kernel.hpp:20)
      float sn, cs;
      sincosf(r, &sn, &cs);
      const float gr = rinv * cs, gi = rinv * sn;
      re += double(gr * c.x - gi * c.y);
      im += double(gr * c.y + gi * c.x);
    }
  }
  if (touched) *flag = 1;
  block_sum(re, im);
  if (threadIdx.x == 0) out[blockIdx.x] = make_double2(re * scale, im * scale);
}

// assemble_rhs (solver.cpp:302-312): rhs[i] = A exp(i k d.x_i), k = kr + i ki, all in FP64
__global__ void __launch_bounds__(kBlock)
assemble_rhs_kernel(uint32_t n, const double* __restrict__ xyz, double dx, double dy, double dz, double kr,
                    double ki, double ar, double ai, double2* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double t = dx * xyz[3 * i] + dy * xyz[3 * i + 1] + dz * xyz[3 * i + 2];
  // exp(i k t) = exp(-ki t) (cos(kr t) + i sin(kr t))
  double sn, cs;
  sincos(kr * t, &sn, &cs);
  const double m = exp(-ki * t);
  const double er = m * cs, ei = m * sn;
  out[i] = make_double2(ar * er - ai * ei, ar * ei + ai * er);
}

inline uint32_t grid_for(uint32_t n) { return (n + kBlock - 1) / kBlock; }
inline uint32_t reduce_grid(uint32_t n) { return std::min<uint32_t>(grid_for(n), kReduceBlocks); }

}  // namespace

size_t reduce_scratch_doubles() { return 2 * kReduceBlocks + 1; }

void launch_corrections(uint32_t n, int ni, const double2* block, const uint32_t* off, const uint32_t* src,
                        const double2* delta, const float2* x, float2* y, cudaStream_t s) {
  if (!n || (!block && !delta)) return;
  corrections_kernel<<<grid_for(n), kBlock, 0, s>>>(n, ni, block, off, src, delta, x, y);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_precondition(uint32_t npatch, int ni, const double2* lu, const int* piv, const float2* in,
                         float2* out, cudaStream_t s) {
  if (!npatch) return;
  if (ni > kMaxNi) throw Error(HFMM_ERR_CONFIG, "more than 12 basis nodes per patch");
  precondition_kernel<<<grid_for(npatch), kBlock, 0, s>>>(npatch, ni, lu, piv, in, out);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_mgs_step(uint32_t n, float2* w, const float2* v_prev, const double* h_prev,
                     const float2* v_next, double* out, double* scratch, cudaStream_t s) {
  if (!n) return;
  mgs_step_kernel<<<reduce_grid(n), kBlock, 0, s>>>(n, w, v_prev, h_prev, v_next, out, scratch);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_norm2(uint32_t n, const float2* w, double* out, double* scratch, cudaStream_t s) {
  if (!n) return;
  norm2_kernel<<<reduce_grid(n), kBlock, 0, s>>>(n, w, out, scratch);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_scale(uint32_t n, const float2* in, float scale, float2* out, cudaStream_t s) {
  if (!n) return;
  scale_kernel<<<grid_for(n), kBlock, 0, s>>>(n, in, scale, out);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_update_solution(uint32_t n, int cols, const float2* basis, size_t ld, const double* y,
                            double2* x, cudaStream_t s) {
  if (!n || !cols) return;
  update_solution_kernel<<<grid_for(n), kBlock, 0, s>>>(n, cols, basis, ld, y, x);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_residual(uint32_t n, const double2* b, const float2* ax, float2* r32, double* out,
                     double* scratch, cudaStream_t s) {
  if (!n) return;
  residual_kernel<<<reduce_grid(n), kBlock, 0, s>>>(n, b, ax, r32, out, scratch);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_field(uint32_t n, const double* xyz, const float2* q, const double* obs, uint32_t nobs, double k,
                  float scale, float eps, const double* touch2, uint32_t ni, double2* out, int* flag,
                  cudaStream_t s) {
  if (!n || !nobs) return;
  field_kernel<<<nobs, kBlock, 0, s>>>(n, xyz, q, obs, k, scale, eps, touch2, ni ? ni : 1u, out, flag);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_assemble_rhs(uint32_t n, const double* xyz, const double dir[3], double kr, double ki,
                         const double amp[2], double2* out, cudaStream_t s) {
  if (!n) return;
  assemble_rhs_kernel<<<grid_for(n), kBlock, 0, s>>>(n, xyz, dir[0], dir[1], dir[2], kr, ki, amp[0], amp[1], out);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_narrow(uint32_t n, const double2* in, float2* out, cudaStream_t s) {
  if (!n) return;
  narrow_kernel<<<grid_for(n), kBlock, 0, s>>>(n, in, out);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
void launch_widen(uint32_t n, const float2* in, double2* out, cudaStream_t s) {
  if (!n) return;
  widen_kernel<<<grid_for(n), kBlock, 0, s>>>(n, in, out);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

}  // namespace hfmm_b200
