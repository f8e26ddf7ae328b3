// kernels_translate.cu — batched M2M / M2L / L2L on level-scaled FP32 expansions (sm_100a).
//
// Replaces the reference's dense translate (src/expansion.cpp:126-139) of a Gaunt-built matrix
// (src/expansion.cpp:95-124) by the factored, truncation-identical operator of tables.hpp:
//     out += e^{-i mu phi} · E^T · Chat(k|t|) · E · e^{i m phi} · in
// applied to a BATCH of (source, destination) cell pairs that share one lattice shift, so the
// rotation block E (real Wigner-d, block diagonal in n) and the coaxial block Chat (diagonal in m)
// are staged once in shared memory and reused by every pair of the batch.  Pairs of one batch have
// different destinations, so results are accumulated with float atomics (RED) into HBM.
//
// This file holds the order-generic kernel (runtime P, operands in shared memory).
#include "device_utils.cuh"
#include "kernels.cuh"
#include "tables.hpp"

namespace hfmm_b200 {

namespace {

constexpr int kThreads = 128;
constexpr int kRow = kTranslateBatch + 1;  // padded row (float2 elements) of the operand tiles

__device__ __forceinline__ void idx_to_nm(int i, int& n, int& m) {
  n = int(sqrtf(float(i)));
  while (n * n > i) --n;
  while ((n + 1) * (n + 1) <= i) ++n;
  m = i - n * (n + 1);
}

struct SmemPlan {
  int rot_floats, coax_c, phase_c, tile_c;
  size_t bytes;
};
__host__ __device__ inline SmemPlan smem_plan(int P) {
  SmemPlan s;
  const int dim = (P + 1) * (P + 1);
  s.rot_floats = ((P + 1) * (2 * P + 1) * (2 * P + 3) / 3 + 3) & ~3;
  int c = 0;
  for (int j = 0; j <= P; ++j) c += (P + 1 - j) * (P + 1 - j);
  s.coax_c = (c + 1) & ~1;
  s.phase_c = (2 * P + 2) & ~1;
  s.tile_c = dim * kRow;
  s.bytes = size_t(s.rot_floats) * 4 + size_t(s.coax_c + s.phase_c + 2 * s.tile_c) * 8 + 32 * 4;
  return s;
}

__global__ void __launch_bounds__(kThreads) translate_generic_kernel(const TranslateArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int P = a.order, dim = (P + 1) * (P + 1);
  const SmemPlan sp = smem_plan(P);
  float* s_rot = smem;
  float2* s_coax = reinterpret_cast<float2*>(s_rot + sp.rot_floats);
  float2* s_ph = s_coax + sp.coax_c;  // e^{i m phi}, index m + P
  float2* X = s_ph + sp.phase_c;
  float2* Y = X + sp.tile_c;
  int* s_coff = reinterpret_cast<int*>(Y + sp.tile_c);  // coaxial block offsets per m

  const TranslateItem item = a.items[blockIdx.x];
  const TranslateClass cls = a.classes[item.cls];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int count = int(item.count);

  {
    const float* g_rot = a.rot_tables + size_t(cls.rot) * rot_table_size(P);
    for (int i = tid; i < rot_table_size(P); i += kThreads) s_rot[i] = g_rot[i];
    const float2* g_coax =
        reinterpret_cast<const float2*>(a.coax_tables) + size_t(cls.coax) * coax_table_size(P);
    for (int i = tid; i < coax_table_size(P); i += kThreads) s_coax[i] = g_coax[i];
    if (tid <= 2 * P) {
      const int m = tid - P, am = m < 0 ? -m : m;
      float cr = 1.f, ci = 0.f;
      for (int j = 0; j < am; ++j) {
        const float t = cr * cls.cphi - ci * cls.sphi;
        ci = ci * cls.cphi + cr * cls.sphi;
        cr = t;
      }
      s_ph[tid] = make_float2(cr, m < 0 ? -ci : ci);
    }
    if (tid == 0) {
      int off = 0;
      for (int m = 0; m <= P; ++m) {
        s_coff[m] = off;
        off += (P + 1 - m) * (P + 1 - m);
      }
    }
  }
  __syncthreads();

  // stage 1: gather sources, apply e^{i m phi}
  for (int p = warp; p < kTranslateBatch; p += kThreads / 32) {
    const bool live = p < count;
    const float2* row = live ? a.src + size_t(a.pair_src[item.pair_begin + p]) * a.stride : nullptr;
    for (int i = lane; i < dim; i += 32) {
      float2 v = make_float2(0.f, 0.f);
      if (live) {
        int n, m;
        idx_to_nm(i, n, m);
        const float2 x = row[i], ph = s_ph[m + P];
        v = make_float2(x.x * ph.x - x.y * ph.y, x.x * ph.y + x.y * ph.x);
      }
      X[i * kRow + p] = v;
    }
  }
  __syncthreads();

  // stage 2: forward rotation  Y[(n,m')] = sum_m E_n[m][m'] X[(n,m)]
  for (int i = warp; i < dim; i += kThreads / 32) {
    int n, mp;
    idx_to_nm(i, n, mp);
    const int w = 2 * n + 1;
    const float* blk = s_rot + rot_block_offset(n);
    const float2* xin = X + (n * n) * kRow + lane;
    float ar = 0.f, ai = 0.f;
    for (int m = 0; m < w; ++m) {
      const float e = blk[m * w + (mp + n)];
      const float2 x = xin[m * kRow];
      ar = fmaf(e, x.x, ar);
      ai = fmaf(e, x.y, ai);
    }
    Y[i * kRow + lane] = make_float2(ar, ai);
  }
  __syncthreads();

  // stage 3: coaxial translation  X[(nu,m)] = sum_n Chat^{|m|}[n][nu] Y[(n,m)]
  for (int i = warp; i < dim; i += kThreads / 32) {
    int nu, m;
    idx_to_nm(i, nu, m);
    const int am = m < 0 ? -m : m, w = P + 1 - am;
    const float2* blk = s_coax + s_coff[am];
    float ar = 0.f, ai = 0.f;
    for (int n = am; n <= P; ++n) {
      const float2 c = blk[(n - am) * w + (nu - am)];
      const float2 y = Y[(n * (n + 1) + m) * kRow + lane];
      ar = fmaf(c.x, y.x, ar);
      ar = fmaf(-c.y, y.y, ar);
      ai = fmaf(c.x, y.y, ai);
      ai = fmaf(c.y, y.x, ai);
    }
    X[i * kRow + lane] = make_float2(ar, ai);
  }
  __syncthreads();

  // stage 4: inverse rotation, e^{-i mu phi}, accumulate
  const bool live = lane < count;
  float2* drow = live ? a.dst + size_t(a.pair_dst[item.pair_begin + lane]) * a.stride : nullptr;
  for (int i = warp; i < dim; i += kThreads / 32) {
    int nu, mu;
    idx_to_nm(i, nu, mu);
    const int w = 2 * nu + 1;
    const float* blk = s_rot + rot_block_offset(nu) + (mu + nu) * w;
    const float2* xin = X + (nu * nu) * kRow + lane;
    float ar = 0.f, ai = 0.f;
    for (int mp = 0; mp < w; ++mp) {
      const float e = blk[mp];
      const float2 x = xin[mp * kRow];
      ar = fmaf(e, x.x, ar);
      ai = fmaf(e, x.y, ai);
    }
    if (live) {
      const float2 ph = s_ph[mu + P];  // multiply by conj
      atomicAdd(&drow[i].x, ar * ph.x + ai * ph.y);
      atomicAdd(&drow[i].y, ai * ph.x - ar * ph.y);
    }
  }
}

}  // namespace

void launch_translate(const TranslateArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  const SmemPlan sp = smem_plan(a.order);
  static int configured_for = -1;
  if (configured_for < int(sp.bytes)) {
    HFMM_CUDA_CHECK(cudaFuncSetAttribute(translate_generic_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(sp.bytes)));
    configured_for = int(sp.bytes);
  }
  translate_generic_kernel<<<a.n_items, kThreads, sp.bytes, s>>>(a);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

}  // namespace hfmm_b200
