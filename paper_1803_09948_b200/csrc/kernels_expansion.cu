// kernels_expansion.cu — P2M and L2P on level-scaled FP32 expansions (sm_100a).
//
// Replaces reference p2m (src/expansion.cpp:157-175) and the L2P half of compute_locals
// (src/expansion.cpp:283-300):
//   M_n^m  = sum_b (i k q_b) j_n(k rho_b) conj Y_n^m(rho_b^)
//   trg_b += sum_{n,m} L_n^m j_n(k |x_b|) Y_n^m(x_b^)
// in the scaled basis of tables.hpp:  Mhat = M (2n+1)!!/s^n,  Lhat = L s^n/(2n-1)!!,  with the
// scaled radial function  jhat_n(z; s) = j_n(z) (2n+1)!!/s^n = (z/s)^n * S_n(z^2),
//   S_n(z^2) = sum_j (-z^2/2)^j / (j! (2n+3)(2n+5)...(2n+2j+1))      (special.cpp:18-34's series)
// which is O(1) for every body of a leaf (z/s = rho/side <= sqrt(3)/2) at any depth of the tree.
// Y_n^m uses the reference's orthonormal Legendre recurrences (special.cpp:80-112) in FP32.
//
// One warp per leaf; lanes are bodies.  P2M reduces each coefficient across lanes with shuffles;
// L2P needs no reduction.
#include <cstdlib>
#include <cstring>

#include "device_utils.cuh"
#include "kernels.cuh"
#include "tables.hpp"

namespace hfmm_b200 {

namespace {

constexpr int kWarps = 4;
constexpr int kMaxP = kMaxOrder;
constexpr float kInvSqrt4Pi = 0.28209479177387814f;

__constant__ float c_diag[kMaxP + 1];
__constant__ float c_sub[kMaxP + 1];
__constant__ float c_a[(kMaxP + 1) * (kMaxP + 2) / 2];
__constant__ float c_b[(kMaxP + 1) * (kMaxP + 2) / 2];
// reciprocals of the series denominators j (2n + 2j + 1), n <= kMaxP, j = 1..12
constexpr int kSeriesTerms = 12;
__constant__ float c_series[(kMaxP + 1) * kSeriesTerms];
__constant__ float c_inv_odd[kMaxP + 1];  // 1 / (2n + 1)

// jhat_n(z; s), n = 0..P, written to out[n * 32] (one shared-memory column per lane)
__device__ void scaled_bessel(int P, float z, float s, float* out) {
  if (z <= 2.0f) {
    const float h = -0.5f * z * z;
    const float t = z / s;
    float tp = 1.0f;
    // |term_j / term_{j-1}| <= (z^2/2) / (j (2j+1)): 7 terms reach 1e-9 for z <= 1, 12 for z <= 2
    const int terms = z <= 1.0f ? 7 : kSeriesTerms;
    for (int n = 0; n <= P; ++n) {
      float term = 1.0f, sum = 1.0f;
      const float* inv = c_series + n * kSeriesTerms;
      for (int j = 0; j < terms; ++j) {
        term *= h * inv[j];
        sum += term;
      }
      out[n * 32] = tp * sum;
      tp *= t;
    }
    return;
  }
  // beyond the low-frequency regime (only reachable with the kd gate off): Miller's downward
  // recurrence in FP64, normalised by j_0 = sin z / z (special.cpp:36-53)
  const double zd = z;
  const int start = P + 24 + int(zd);
  double above = 0.0, cur = 1e-280;
  double keep[kMaxP + 1];
  for (int n = start; n >= 0; --n) {
    const double below = (2.0 * n + 3.0) / zd * cur - above;
    above = cur;
    cur = below;
    if (n <= P) keep[n] = cur;
    if (fabs(cur) > 1e250) {
      cur *= 1e-250;
      above *= 1e-250;
      for (int i = n < P ? n : P; i <= P; ++i) keep[i] *= 1e-250;
    }
  }
  const double scale = (sin(zd) / zd) / cur;
  double f = 1.0;  // (2n+1)!!/s^n
  for (int n = 0; n <= P; ++n) {
    out[n * 32] = float(keep[n] * scale * f);
    f *= (2.0 * n + 3.0) / double(s);
  }
}

// complex wavenumber k = k_r (1 + i eps), eps = k_i / k_r: the argument is z = kappa z' with z' = k_r rho
// the stored (real) coordinate and kappa = 1 + i eps; the same series in complex arithmetic
// (reference special.cpp:16-54 takes a complex argument throughout)
__device__ void scaled_bessel_complex(int P, float zr, float eps, float s, float* out_re, float* out_im) {
  const float zmod = zr * sqrtf(1.0f + eps * eps);
  if (zmod <= 2.0f) {
    // h = -z^2 / 2 = -(1 - eps^2 + 2 i eps) z'^2 / 2,   t = z / s
    const float hr = -0.5f * zr * zr * (1.0f - eps * eps), hi = -zr * zr * eps;
    const float tr = zr / s, ti = tr * eps;
    float pr = 1.0f, pi = 0.0f;
    const int terms = zmod <= 1.0f ? 7 : kSeriesTerms;
    for (int n = 0; n <= P; ++n) {
      float ter = 1.0f, tei = 0.0f, sr = 1.0f, si = 0.0f;
      const float* inv = c_series + n * kSeriesTerms;
      for (int j = 0; j < terms; ++j) {
        const float ar = hr * inv[j], ai = hi * inv[j];
        const float nr = ter * ar - tei * ai;
        tei = ter * ai + tei * ar;
        ter = nr;
        sr += ter;
        si += tei;
      }
      out_re[n * 32] = pr * sr - pi * si;
      out_im[n * 32] = pr * si + pi * sr;
      const float qr = pr * tr - pi * ti;
      pi = pr * ti + pi * tr;
      pr = qr;
    }
    return;
  }
  // Miller's downward recurrence in complex FP64, normalised by j_0 = sin z / z
  const double zx = zr, zy = double(zr) * eps;
  const double zn2 = zx * zx + zy * zy;
  const double ix = zx / zn2, iy = -zy / zn2;  // 1 / z
  const int start = P + 24 + int(sqrt(zn2));
  double ax = 0, ay = 0, cx = 1e-280, cy = 0;
  double kx[kMaxP + 1], ky[kMaxP + 1];
  for (int n = start; n >= 0; --n) {
    const double f = 2.0 * n + 3.0;
    const double mx = f * (ix * cx - iy * cy), my = f * (ix * cy + iy * cx);
    const double bx = mx - ax, by = my - ay;
    ax = cx;
    ay = cy;
    cx = bx;
    cy = by;
    if (n <= P) {
      kx[n] = cx;
      ky[n] = cy;
    }
    if (fabs(cx) + fabs(cy) > 1e250) {
      cx *= 1e-250; cy *= 1e-250; ax *= 1e-250; ay *= 1e-250;
      for (int i = n < P ? n : P; i <= P; ++i) {
        kx[i] *= 1e-250;
        ky[i] *= 1e-250;
      }
    }
  }
  // sin(x + i y) = sin x cosh y + i cos x sinh y
  const double snx = sin(zx) * cosh(zy), sny = cos(zx) * sinh(zy);
  const double j0x = snx * ix - sny * iy, j0y = snx * iy + sny * ix;
  // j_0 / cur with cur scaled to unit size first: |cur| ranges over 1e-280 .. 1e250, its square would
  // leave the FP64 range (the gate-off regime with wide leaves is the only one that gets here)
  const double cm = fmax(fabs(cx), fabs(cy));
  const double ux = cx / cm, uy = cy / cm, un2 = ux * ux + uy * uy;
  const double scx = (j0x * ux + j0y * uy) / un2 / cm, scy = (j0y * ux - j0x * uy) / un2 / cm;
  double f = 1.0;  // (2n+1)!!/s^n
  for (int n = 0; n <= P; ++n) {
    out_re[n * 32] = float((kx[n] * scx - ky[n] * scy) * f);
    out_im[n * 32] = float((kx[n] * scy + ky[n] * scx) * f);
    f *= (2.0 * n + 3.0) / double(s);
  }
}

struct BodyFrame {
  float ct, st, cphi, sphi, z;
};

__device__ __forceinline__ BodyFrame body_frame(const float4 p) {
  BodyFrame f;
  const float rxy2 = p.x * p.x + p.y * p.y;
  const float r2 = rxy2 + p.z * p.z;
  f.z = sqrtf(r2);
  const float rxy = sqrtf(rxy2);
  if (r2 > 0.0f) {
    f.ct = p.z / f.z;
    f.st = rxy / f.z;
  } else {
    f.ct = 1.0f;
    f.st = 0.0f;
  }
  if (rxy2 > 0.0f) {
    f.cphi = p.x / rxy;
    f.sphi = p.y / rxy;
  } else {  // atan2(0, 0) = 0 in the reference
    f.cphi = 1.0f;
    f.sphi = 0.0f;
  }
  return f;
}

// CK: complex wavenumber (radial functions and the i k q weight are complex)
template <bool CK>
__global__ void __launch_bounds__(kWarps * 32)
p2m_kernel(const LeafExpansionArgs a, const float2* __restrict__ body_q, float2* __restrict__ multipole) {
  extern __shared__ float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = a.order, dim = (P + 1) * (P + 1);
  constexpr int kPlanes = CK ? 2 : 1;
  float* s_j = smem + warp * (kPlanes * (P + 1) * 32 + 2 * dim);  // [n][lane] (+ imaginary plane)
  float* s_ji = s_j + (P + 1) * 32;
  float2* s_acc = reinterpret_cast<float2*>(s_j + kPlanes * (P + 1) * 32);
  const float eps = CK ? a.k_imag / a.k : 0.0f;
  const uint32_t li = blockIdx.x * kWarps + warp;
  if (li >= a.n_leaves) return;
  const uint32_t cell = a.leaves[li];
  const uint2 cb = a.cell_body[cell];
  const float s = a.level_scale[a.cell_geom[cell].w];
  for (int i = lane; i < dim; i += 32) s_acc[i] = make_float2(0.f, 0.f);
  __syncwarp();
  float* s_accf = reinterpret_cast<float*>(s_acc);
  const bool hi16 = (lane & 16) != 0, hi8 = (lane & 8) != 0, writer = (lane & 7) == 0;

  for (uint32_t base = 0; base < cb.y; base += 32) {
    const bool ok = base + lane < cb.y;
    const float4 p = ok ? a.body_pos[cb.x + base + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float2 q = ok ? body_q[cb.x + base + lane] : make_float2(0.f, 0.f);
    const BodyFrame f = body_frame(p);
    if (CK) scaled_bessel_complex(P, f.z, eps, s, s_j + lane, s_ji + lane);
    else scaled_bessel(P, f.z, s, s_j + lane);
    // w = i k q
    const float wr = -a.k * q.y - (CK ? a.k_imag * q.x : 0.0f), wi = a.k * q.x - (CK ? a.k_imag * q.y : 0.0f);
    float cm = 1.0f, sm = 0.0f;     // cos(m phi), sin(m phi)
    float pmm = kInvSqrt4Pi;        // Pbar_m^m
    for (int m = 0; m <= P; ++m) {
      if (m > 0) {
        pmm *= c_diag[m] * f.st;
        const float c2 = cm * f.cphi - sm * f.sphi;
        sm = sm * f.cphi + cm * f.sphi;
        cm = c2;
      }
      float p2 = 0.0f, p1 = pmm;  // Pbar_{n-2}^m, Pbar_{n-1}^m
      for (int n = m; n <= P; ++n) {
        float pn;
        if (n == m) pn = pmm;
        else if (n == m + 1) pn = c_sub[m] * f.ct * pmm;
        else pn = c_a[n * (n + 1) / 2 + m] * f.ct * p1 - c_b[n * (n + 1) / 2 + m] * p2;
        p2 = p1;
        p1 = pn;
        const float g = s_j[n * 32 + lane] * pn, gi = CK ? s_ji[n * 32 + lane] * pn : 0.0f;
        // +m: conj Y = Pbar (cm - i sm)
        const float br = wr * cm + wi * sm, bi = wi * cm - wr * sm;
        const float vr = g * br - gi * bi, vi = g * bi + gi * br;
        // -m: conj Y_n^{-m} = (-1)^m Pbar (cm + i sm)   (m = 0: slots 2, 3 carry zeros and are not stored)
        float ur = 0.0f, ui = 0.0f;
        if (m > 0) {
          const float sg = (m & 1) ? -1.0f : 1.0f;
          const float er = wr * cm - wi * sm, ei = wi * cm + wr * sm;
          ur = sg * (g * er - gi * ei);
          ui = sg * (g * ei + gi * er);
        }
        // four sums over the 32 bodies in one butterfly: the first two exchanges halve the number of
        // values a lane carries (6 shuffles instead of 20; the pairing order, hence the rounding, is
        // that of four separate reductions); lanes 0 / 8 / 16 / 24 end up with Re(+m), Im(+m), Re(-m), Im(-m)
        const float k0 = hi16 ? ur : vr, s0 = hi16 ? vr : ur, k1 = hi16 ? ui : vi, s1 = hi16 ? vi : ui;
        const float b0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16), b1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
        float c = (hi8 ? b1 : b0) + __shfl_xor_sync(0xffffffffu, hi8 ? b0 : b1, 8);
        c += __shfl_xor_sync(0xffffffffu, c, 4);
        c += __shfl_xor_sync(0xffffffffu, c, 2);
        c += __shfl_xor_sync(0xffffffffu, c, 1);
        if (writer && (m > 0 || !hi16)) s_accf[2 * (n * (n + 1) + (hi16 ? -m : m)) + (hi8 ? 1 : 0)] += c;
      }
    }
    __syncwarp();
  }
  __syncwarp();
  float2* dst = multipole + size_t(cell) * a.stride;
  for (int i = lane; i < dim; i += 32) dst[i] = s_acc[i];
}

template <bool CK>
__global__ void __launch_bounds__(kWarps * 32)
l2p_kernel(const LeafExpansionArgs a, const float2* __restrict__ local, float2* __restrict__ out) {
  extern __shared__ float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = a.order, dim = (P + 1) * (P + 1);
  constexpr int kPlanes = CK ? 2 : 1;
  float* s_j = smem + warp * (kPlanes * (P + 1) * 32 + 2 * dim);
  float* s_ji = s_j + (P + 1) * 32;
  float2* s_loc = reinterpret_cast<float2*>(s_j + kPlanes * (P + 1) * 32);
  const float eps = CK ? a.k_imag / a.k : 0.0f;
  const uint32_t li = blockIdx.x * kWarps + warp;
  if (li >= a.n_leaves) return;
  const uint32_t cell = a.leaves[li];
  const uint2 cb = a.cell_body[cell];
  const float s = a.level_scale[a.cell_geom[cell].w];
  const float2* src = local + size_t(cell) * a.stride;
  for (int i = lane; i < dim; i += 32) s_loc[i] = src[i];
  __syncwarp();

  for (uint32_t base = 0; base < cb.y; base += 32) {
    const bool ok = base + lane < cb.y;
    const float4 p = ok ? a.body_pos[cb.x + base + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    const BodyFrame f = body_frame(p);
    if (CK) scaled_bessel_complex(P, f.z, eps, s, s_j + lane, s_ji + lane);
    else scaled_bessel(P, f.z, s, s_j + lane);
    float accr = 0.0f, acci = 0.0f;
    float cm = 1.0f, sm = 0.0f, pmm = kInvSqrt4Pi;
    for (int m = 0; m <= P; ++m) {
      if (m > 0) {
        pmm *= c_diag[m] * f.st;
        const float c2 = cm * f.cphi - sm * f.sphi;
        sm = sm * f.cphi + cm * f.sphi;
        cm = c2;
      }
      float p2 = 0.0f, p1 = pmm;
      float sr = 0.0f, si = 0.0f;  // sum over n of g * (L^m, L^-m combination)
      for (int n = m; n <= P; ++n) {
        float pn;
        if (n == m) pn = pmm;
        else if (n == m + 1) pn = c_sub[m] * f.ct * pmm;
        else pn = c_a[n * (n + 1) / 2 + m] * f.ct * p1 - c_b[n * (n + 1) / 2 + m] * p2;
        p2 = p1;
        p1 = pn;
        // Lhat pairs with j_n (2n-1)!!/s^n = jhat_n / (2n+1)
        const float pw = pn * c_inv_odd[n];
        const float g = s_j[n * 32 + lane] * pw;
        const float gi = CK ? s_ji[n * 32 + lane] * pw : 0.0f;
        const float2 lp = s_loc[n * (n + 1) + m];
        if (m == 0) {
          sr += g * lp.x - gi * lp.y;
          si += g * lp.y + gi * lp.x;
        } else {
          const float2 lm = s_loc[n * (n + 1) - m];
          const float sg = (m & 1) ? -1.0f : 1.0f;
          // L^m (cm + i sm) + (-1)^m L^-m (cm - i sm)
          const float er = lp.x + sg * lm.x, ei = lp.y + sg * lm.y;   // multiplies cm
          const float dr = lp.x - sg * lm.x, di = lp.y - sg * lm.y;   // multiplies i sm
          const float xr = er * cm - di * sm, xi = ei * cm + dr * sm;
          sr += g * xr - gi * xi;
          si += g * xi + gi * xr;
        }
      }
      accr += sr;
      acci += si;
    }
    if (ok) out[cb.x + base + lane] = make_float2(accr, acci);
    __syncwarp();
  }
}

// ---- straight-line kernels for the regime every BASELINE configuration runs in ----------------------
// Real wavenumber, every body of every leaf inside the 7-term range of the series (z = k rho <= 1: with
// the reference's leaf cap k side <= kd_max = 1 the largest z is sqrt(3)/2), order known at compile time:
// the (m, n) loops are fully unrolled, so the Legendre coefficients are immediates of the constant bank,
// jhat_n lives in registers and no index arithmetic or branch is left between the multiply-adds.
// ncu on the rolled kernels: 7.5 k warp-instructions per leaf (82 per coefficient pair), issue-bound.

// jhat_n(z; s) for z <= 1, n = 0..P (same series and term count as scaled_bessel)
template <int P>
__device__ __forceinline__ void scaled_bessel_small(float z, float s, float (&jh)[P + 1]) {
  const float h = -0.5f * z * z, t = z / s;
  float tp = 1.0f;
#pragma unroll
  for (int n = 0; n <= P; ++n) {
    float term = 1.0f, sum = 1.0f;
#pragma unroll
    for (int j = 0; j < 7; ++j) {
      term *= h * c_series[n * kSeriesTerms + j];
      sum += term;
    }
    jh[n] = tp * sum;
    tp *= t;
  }
}

template <int P>
__global__ void __launch_bounds__(kWarps * 32, 4)
p2m_fast_kernel(const LeafExpansionArgs a, const float2* __restrict__ body_q, float2* __restrict__ multipole) {
  constexpr int dim = (P + 1) * (P + 1);
  __shared__ float s_all[kWarps][2 * dim];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t li = blockIdx.x * kWarps + warp;
  if (li >= a.n_leaves) return;
  float* s_accf = s_all[warp];
  const uint32_t cell = a.leaves[li];
  const uint2 cb = a.cell_body[cell];
  const float s = a.level_scale[a.cell_geom[cell].w];
  const bool hi16 = (lane & 16) != 0, hi8 = (lane & 8) != 0, writer = (lane & 7) == 0;
  // the float this lane owns after the butterfly: Re / Im (hi8) of the +m / -m (hi16) coefficient
  const int w_sign = hi16 ? -2 : 2, w_off = hi8 ? 1 : 0;
  for (int i = lane; i < 2 * dim; i += 32) s_accf[i] = 0.0f;
  __syncwarp();

  for (uint32_t base = 0; base < cb.y; base += 32) {
    const bool ok = base + lane < cb.y;
    const float4 p = ok ? a.body_pos[cb.x + base + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float2 q = ok ? body_q[cb.x + base + lane] : make_float2(0.f, 0.f);
    const BodyFrame f = body_frame(p);
    float jh[P + 1];
    scaled_bessel_small<P>(f.z, s, jh);
    const float wr = -a.k * q.y, wi = a.k * q.x;  // w = i k q
    float cm = 1.0f, sm = 0.0f, pmm = kInvSqrt4Pi;
#pragma unroll
    for (int m = 0; m <= P; ++m) {
      if (m > 0) {
        pmm *= c_diag[m] * f.st;
        const float c2 = cm * f.cphi - sm * f.sphi;
        sm = sm * f.cphi + cm * f.sphi;
        cm = c2;
      }
      // +m: w conj Y = Pbar w (cm - i sm);  -m: (-1)^m Pbar w (cm + i sm)
      const float sg = (m & 1) ? -1.0f : 1.0f;
      const float br = wr * cm + wi * sm, bi = wi * cm - wr * sm;
      const float er = sg * (wr * cm - wi * sm), ei = sg * (wi * cm + wr * sm);
      // what this lane keeps / sends in the first exchange does not depend on n
      const float kr = hi16 ? er : br, sr = hi16 ? br : er, ki = hi16 ? ei : bi, si = hi16 ? bi : ei;
      float p2 = 0.0f, p1 = pmm;
#pragma unroll
      for (int n = m; n <= P; ++n) {
        float pn;
        if (n == m) pn = pmm;
        else if (n == m + 1) pn = c_sub[m] * f.ct * pmm;
        else pn = c_a[n * (n + 1) / 2 + m] * f.ct * p1 - c_b[n * (n + 1) / 2 + m] * p2;
        p2 = p1;
        p1 = pn;
        const float g = jh[n] * pn;
        if (m == 0) {
          // two sums (Re, Im of the m = 0 coefficient): lanes 0 and 8 end up with them
          const float b0 = g * br, b1 = g * bi;
          float c = (hi8 ? b1 : b0) + __shfl_xor_sync(0xffffffffu, hi8 ? b0 : b1, 8);
          c += __shfl_xor_sync(0xffffffffu, c, 16);
          c += __shfl_xor_sync(0xffffffffu, c, 4);
          c += __shfl_xor_sync(0xffffffffu, c, 2);
          c += __shfl_xor_sync(0xffffffffu, c, 1);
          if (writer && !hi16) s_accf[2 * (n * (n + 1)) + w_off] += c;
        } else {
          // four sums over the 32 bodies in one butterfly: the first two exchanges halve the number of
          // values a lane carries; lanes 0 / 8 / 16 / 24 end up with Re(+m), Im(+m), Re(-m), Im(-m)
          const float b0 = g * kr + __shfl_xor_sync(0xffffffffu, g * sr, 16);
          const float b1 = g * ki + __shfl_xor_sync(0xffffffffu, g * si, 16);
          float c = (hi8 ? b1 : b0) + __shfl_xor_sync(0xffffffffu, hi8 ? b0 : b1, 8);
          c += __shfl_xor_sync(0xffffffffu, c, 4);
          c += __shfl_xor_sync(0xffffffffu, c, 2);
          c += __shfl_xor_sync(0xffffffffu, c, 1);
          if (writer) s_accf[2 * (n * (n + 1)) + w_sign * m + w_off] += c;
        }
      }
    }
    __syncwarp();
  }
  float2* dst = multipole + size_t(cell) * a.stride;
  const float2* s_acc = reinterpret_cast<const float2*>(s_accf);
  for (int i = lane; i < dim; i += 32) dst[i] = s_acc[i];
}

template <int P>
__global__ void __launch_bounds__(kWarps * 32, 4)
l2p_fast_kernel(const LeafExpansionArgs a, const float2* __restrict__ local, float2* __restrict__ out) {
  constexpr int dim = (P + 1) * (P + 1);
  __shared__ float2 s_all[kWarps][dim];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t li = blockIdx.x * kWarps + warp;
  if (li >= a.n_leaves) return;
  float2* s_loc = s_all[warp];
  const uint32_t cell = a.leaves[li];
  const uint2 cb = a.cell_body[cell];
  const float s = a.level_scale[a.cell_geom[cell].w];
  const float2* src = local + size_t(cell) * a.stride;
  for (int i = lane; i < dim; i += 32) s_loc[i] = src[i];
  __syncwarp();
  // fold once per leaf (the combinations are the same for every body):
  //   slot (n, +m) <- E = L^m + (-1)^m L^-m  (multiplies cos m phi),  slot (n, -m) <- D = L^m - (-1)^m L^-m  (multiplies i sin m phi)
  for (int u = lane; u < (P + 1) * (P + 2) / 2; u += 32) {
    int n = int((sqrtf(8.0f * float(u) + 1.0f) - 1.0f) * 0.5f);
    while (n * (n + 1) / 2 > u) --n;
    while ((n + 1) * (n + 2) / 2 <= u) ++n;
    const int m = u - n * (n + 1) / 2;
    if (m == 0) continue;
    const float sg = (m & 1) ? -1.0f : 1.0f;
    const float2 lp = s_loc[n * (n + 1) + m], lm = s_loc[n * (n + 1) - m];
    s_loc[n * (n + 1) + m] = make_float2(lp.x + sg * lm.x, lp.y + sg * lm.y);
    s_loc[n * (n + 1) - m] = make_float2(lp.x - sg * lm.x, lp.y - sg * lm.y);
  }
  __syncwarp();

  for (uint32_t base = 0; base < cb.y; base += 32) {
    const bool ok = base + lane < cb.y;
    const float4 p = ok ? a.body_pos[cb.x + base + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    const BodyFrame f = body_frame(p);
    float jh[P + 1];
    scaled_bessel_small<P>(f.z, s, jh);
#pragma unroll
    for (int n = 0; n <= P; ++n) jh[n] *= c_inv_odd[n];  // Lhat pairs with j_n (2n-1)!!/s^n = jhat_n / (2n+1)
    float accr = 0.0f, acci = 0.0f;
    float cm = 1.0f, sm = 0.0f, pmm = kInvSqrt4Pi;
#pragma unroll
    for (int m = 0; m <= P; ++m) {
      if (m > 0) {
        pmm *= c_diag[m] * f.st;
        const float c2 = cm * f.cphi - sm * f.sphi;
        sm = sm * f.cphi + cm * f.sphi;
        cm = c2;
      }
      float p2 = 0.0f, p1 = pmm;
      float ser = 0.0f, sei = 0.0f, sdr = 0.0f, sdi = 0.0f;  // sum_n g E, sum_n g D
#pragma unroll
      for (int n = m; n <= P; ++n) {
        float pn;
        if (n == m) pn = pmm;
        else if (n == m + 1) pn = c_sub[m] * f.ct * pmm;
        else pn = c_a[n * (n + 1) / 2 + m] * f.ct * p1 - c_b[n * (n + 1) / 2 + m] * p2;
        p2 = p1;
        p1 = pn;
        const float g = jh[n] * pn;
        const float2 e = s_loc[n * (n + 1) + m];
        ser = fmaf(g, e.x, ser);
        sei = fmaf(g, e.y, sei);
        if (m > 0) {
          const float2 d = s_loc[n * (n + 1) - m];
          sdr = fmaf(g, d.x, sdr);
          sdi = fmaf(g, d.y, sdi);
        }
      }
      // sum_n g (E cm + i D sm)
      accr += ser * cm - sdi * sm;
      acci += sei * cm + sdr * sm;
    }
    if (ok) out[cb.x + base + lane] = make_float2(accr, acci);
  }
}

size_t leaf_smem_bytes(int order, bool complex_k) {
  const int dim = (order + 1) * (order + 1);
  return size_t(kWarps) * ((complex_k ? 2 : 1) * (order + 1) * 32 + 2 * dim) * sizeof(float);
}

}  // namespace

void upload_legendre_constants(const float* diag, const float* sub, const float* a, const float* b,
                               int order) {
  const size_t tri = size_t(order + 1) * (order + 2) / 2;
  HFMM_CUDA_CHECK(cudaMemcpyToSymbol(c_diag, diag, sizeof(float) * (order + 1)));
  HFMM_CUDA_CHECK(cudaMemcpyToSymbol(c_sub, sub, sizeof(float) * (order + 1)));
  HFMM_CUDA_CHECK(cudaMemcpyToSymbol(c_a, a, sizeof(float) * tri));
  HFMM_CUDA_CHECK(cudaMemcpyToSymbol(c_b, b, sizeof(float) * tri));
  float series[(kMaxP + 1) * kSeriesTerms];
  for (int n = 0; n <= kMaxP; ++n)
    for (int j = 1; j <= kSeriesTerms; ++j)
      series[n * kSeriesTerms + j - 1] = float(1.0 / (double(j) * (2 * n + 2 * j + 1)));
  HFMM_CUDA_CHECK(cudaMemcpyToSymbol(c_series, series, sizeof(series)));
  float inv_odd[kMaxP + 1];
  for (int n = 0; n <= kMaxP; ++n) inv_odd[n] = float(1.0 / (2.0 * n + 1.0));
  HFMM_CUDA_CHECK(cudaMemcpyToSymbol(c_inv_odd, inv_odd, sizeof(inv_odd)));
}

// the straight-line kernels: real wavenumber, every leaf inside the short-series range, instantiated order
static bool leaf_fast_path(const LeafExpansionArgs& a) {
  static const bool off = [] {
    const char* e = getenv("HFMM_LEAF_KERNELS");
    return e && !strcmp(e, "rolled");
  }();
  return !off && a.small_arguments && a.k_imag == 0.0f;
}

void launch_p2m(const LeafExpansionArgs& a, const float2* body_q, float2* multipole, cudaStream_t s) {
  if (a.n_leaves == 0) return;
  const uint32_t blocks = (a.n_leaves + kWarps - 1) / kWarps;
  if (leaf_fast_path(a)) {
    bool done = true;
    switch (a.order) {
      case 8: p2m_fast_kernel<8><<<blocks, kWarps * 32, 0, s>>>(a, body_q, multipole); break;
      case 10: p2m_fast_kernel<10><<<blocks, kWarps * 32, 0, s>>>(a, body_q, multipole); break;
      case 12: p2m_fast_kernel<12><<<blocks, kWarps * 32, 0, s>>>(a, body_q, multipole); break;
      case 14: p2m_fast_kernel<14><<<blocks, kWarps * 32, 0, s>>>(a, body_q, multipole); break;
      default: done = false;
    }
    if (done) {
      HFMM_CUDA_CHECK(cudaGetLastError());
      return;
    }
  }
  if (a.k_imag != 0.0f)
    p2m_kernel<true><<<blocks, kWarps * 32, leaf_smem_bytes(a.order, true), s>>>(a, body_q, multipole);
  else
    p2m_kernel<false><<<blocks, kWarps * 32, leaf_smem_bytes(a.order, false), s>>>(a, body_q, multipole);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

void launch_l2p(const LeafExpansionArgs& a, const float2* local, float2* out, cudaStream_t s) {
  if (a.n_leaves == 0) return;
  const uint32_t blocks = (a.n_leaves + kWarps - 1) / kWarps;
  if (leaf_fast_path(a)) {
    bool done = true;
    switch (a.order) {
      case 8: l2p_fast_kernel<8><<<blocks, kWarps * 32, 0, s>>>(a, local, out); break;
      case 10: l2p_fast_kernel<10><<<blocks, kWarps * 32, 0, s>>>(a, local, out); break;
      case 12: l2p_fast_kernel<12><<<blocks, kWarps * 32, 0, s>>>(a, local, out); break;
      case 14: l2p_fast_kernel<14><<<blocks, kWarps * 32, 0, s>>>(a, local, out); break;
      default: done = false;
    }
    if (done) {
      HFMM_CUDA_CHECK(cudaGetLastError());
      return;
    }
  }
  if (a.k_imag != 0.0f)
    l2p_kernel<true><<<blocks, kWarps * 32, leaf_smem_bytes(a.order, true), s>>>(a, local, out);
  else
    l2p_kernel<false><<<blocks, kWarps * 32, leaf_smem_bytes(a.order, false), s>>>(a, local, out);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

}  // namespace hfmm_b200
