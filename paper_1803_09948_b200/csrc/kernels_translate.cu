// kernels_translate.cu — batched M2M / M2L / L2L on level-scaled FP32 expansions (sm_100a).
//
// Replaces the reference's dense translate (src/expansion.cpp:126-139) of a Gaunt-built matrix
// (src/expansion.cpp:95-124) by the factored, truncation-identical operator of tables.hpp:
//     out += e^{-i mu phi} · E^T · Chat(k|t|) · E · e^{i m phi} · in
// applied to a BATCH of 32 (source, destination) cell pairs that share one lattice shift, so the
// rotation table E (real Wigner-d, block diagonal in n) and the coaxial table Chat (diagonal in m)
// are staged once in shared memory and reused by every pair of the batch.
//
// Work layout of one CTA (8 warps, one batch):
//   * operands live in two element-major shared tiles [coefficient][pair] (ping-pong): lane = pair,
//     so a warp reads one coefficient of its 32 pairs with a conflict-free LDS.64;
//   * every stage is cut into TASKS = a block (degree n for the rotations, order |m| for the
//     coaxial step) times a tile of up to 12 (4) output rows.  A task keeps its output rows in
//     registers and runs ONE runtime loop over the block's inputs: per step one LDS.64 (the input
//     of the lane's pair) and R/4 broadcast LDS.128 (coefficients) feed 2R (8R coaxial) FFMAs;
//   * tasks are handed to the warps by a host-side longest-processing-time schedule
//     (TranslateSchedule); the code is small and loop-structured on purpose — a fully unrolled,
//     order-specialised variant measured 7x SLOWER on B200 because its 256 KB of SASS starved
//     the instruction cache (profiles/r01_notes.md);
//   * the inverse rotation reuses the same table through d^n_{mu,m'} = (-1)^{mu-m'} d^n_{m',mu};
//   * pairs of one batch have different destinations: results leave through 16-byte vector
//     reductions (RED.E.ADD.F32x4) into HBM/L2.
// FP32 work per pair: 2 * 2*sum_n (2n+1)^2 + 4*sum_m (P+1-|m|)^2 FFMAs (17.6 k at P = 12) against
// 4 (P+1)^4 = 114 k for the reference's dense complex mat-vec.
#include <algorithm>
#include <vector>

#include "device_utils.cuh"
#include "kernels.cuh"
#include "tables.hpp"

namespace hfmm_b200 {

namespace {

constexpr int kWarps = kTranslateWarps;
constexpr int kThreads = kWarps * 32;
constexpr int kRow = 34;  // float2 elements per operand row: 32 pairs + 2 pad (bank spread)

struct SmemPlan {
  int rot_floats, coax_c, phase_c, tile_c, dim;
  size_t bytes;
};
__host__ __device__ inline SmemPlan smem_plan(int P) {
  SmemPlan s;
  s.dim = (P + 1) * (P + 1);
  s.rot_floats = rot_table_size(P);
  s.coax_c = coax_table_size(P);
  s.phase_c = (2 * P + 2) & ~1;
  s.tile_c = s.dim * kRow;
  // rot | coax | phases | tile A | tile B | per-degree/order offsets (2 x 32 ints) | m-of-index
  s.bytes = size_t(s.rot_floats) * 4 + size_t(s.coax_c + s.phase_c + 2 * s.tile_c) * 8 + 64 * 4 +
            size_t((s.dim + 3) & ~3);
  return s;
}

// ---- rotation task: rows [r0, r0+R) of block n;  out[r] = sum_k E[k][r0+r] * in[k] -------------
template <int R, bool BACK>
__device__ __forceinline__ void rot_task(const float* __restrict__ E, int ws, int w,
                                         const float2* __restrict__ in, float2* __restrict__ out,
                                         const float2* __restrict__ ph, bool odd0) {
  float ar[R], ai[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ar[r] = ai[r] = 0.0f;
  constexpr int NV = (R + 3) / 4;
  // two inputs per trip; in the inverse rotation odd inputs enter negated ((-1)^k of the symmetry)
  int k = 0;
#pragma unroll 1
  for (; k + 1 < w; k += 2) {
    const float2 x0 = in[k * kRow], x1 = in[(k + 1) * kRow];
    float e0[NV * 4], e1[NV * 4];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 a = *reinterpret_cast<const float4*>(E + k * ws + 4 * v);
      const float4 b = *reinterpret_cast<const float4*>(E + (k + 1) * ws + 4 * v);
      e0[4 * v] = a.x; e0[4 * v + 1] = a.y; e0[4 * v + 2] = a.z; e0[4 * v + 3] = a.w;
      e1[4 * v] = b.x; e1[4 * v + 1] = b.y; e1[4 * v + 2] = b.z; e1[4 * v + 3] = b.w;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ar[r] = fmaf(e0[r], x0.x, ar[r]);
      ai[r] = fmaf(e0[r], x0.y, ai[r]);
      if (BACK) {
        ar[r] = fmaf(-e1[r], x1.x, ar[r]);
        ai[r] = fmaf(-e1[r], x1.y, ai[r]);
      } else {
        ar[r] = fmaf(e1[r], x1.x, ar[r]);
        ai[r] = fmaf(e1[r], x1.y, ai[r]);
      }
    }
  }
  if (k < w) {  // w is odd: one even-indexed input left
    const float2 x0 = in[k * kRow];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 a = *reinterpret_cast<const float4*>(E + k * ws + 4 * v);
      const float ev[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 * v + j < R) {
          ar[4 * v + j] = fmaf(ev[j], x0.x, ar[4 * v + j]);
          ai[4 * v + j] = fmaf(ev[j], x0.y, ai[4 * v + j]);
        }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (BACK) {
      // (-1)^{row} of the symmetry, then e^{-i mu phi}
      const bool neg = ((r & 1) != 0) != odd0;
      const float sr = neg ? -ar[r] : ar[r], si = neg ? -ai[r] : ai[r];
      const float2 p = ph[r];
      out[r * kRow] = make_float2(sr * p.x + si * p.y, si * p.x - sr * p.y);
    } else {
      out[r * kRow] = make_float2(ar[r], ai[r]);
    }
  }
}

template <bool BACK>
__device__ __forceinline__ void rot_dispatch(int R, const float* E, int ws, int w, const float2* in,
                                             float2* out, const float2* ph, bool odd0) {
  switch (R) {
    case 1: rot_task<1, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 2: rot_task<2, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 3: rot_task<3, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 4: rot_task<4, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 5: rot_task<5, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 6: rot_task<6, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 7: rot_task<7, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 8: rot_task<8, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 9: rot_task<9, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 10: rot_task<10, BACK>(E, ws, w, in, out, ph, odd0); break;
    case 11: rot_task<11, BACK>(E, ws, w, in, out, ph, odd0); break;
    default: rot_task<12, BACK>(E, ws, w, in, out, ph, odd0); break;
  }
}

// ---- coaxial task: rows nu = m + r0 .. m + r0 + R - 1 of order m, columns +m and -m -----------
template <int R, bool TWO>
__device__ __forceinline__ void coax_task(const float2* __restrict__ C, int ws, int w, int m, int r0,
                                          const float2* __restrict__ in, float2* __restrict__ out) {
  float pr[R], pi[R], qr[R], qi[R];  // +m and -m accumulators
#pragma unroll
  for (int r = 0; r < R; ++r) pr[r] = pi[r] = qr[r] = qi[r] = 0.0f;
  int idx = m * (m + 1);  // n (n+1) for n = m
#pragma unroll 1
  for (int k = 0; k < w; ++k) {
    const int n = m + k;
    const float2 xp = in[(idx + m) * kRow];
    float2 xm = make_float2(0.f, 0.f);
    if (TWO) xm = in[(idx - m) * kRow];
    idx += 2 * n + 2;
    float cr[R], ci[R];
    if (R == 1) {
      const float2 c = C[k * ws + r0];
      cr[0] = c.x; ci[0] = c.y;
    } else {
#pragma unroll
      for (int v = 0; v < (R + 1) / 2; ++v) {
        const float4 c = *reinterpret_cast<const float4*>(C + k * ws + r0 + 2 * v);
        cr[2 * v] = c.x; ci[2 * v] = c.y;
        if (2 * v + 1 < R) { cr[2 * v + 1] = c.z; ci[2 * v + 1] = c.w; }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      pr[r] = fmaf(cr[r], xp.x, pr[r]);
      pr[r] = fmaf(-ci[r], xp.y, pr[r]);
      pi[r] = fmaf(cr[r], xp.y, pi[r]);
      pi[r] = fmaf(ci[r], xp.x, pi[r]);
      if (TWO) {
        qr[r] = fmaf(cr[r], xm.x, qr[r]);
        qr[r] = fmaf(-ci[r], xm.y, qr[r]);
        qi[r] = fmaf(cr[r], xm.y, qi[r]);
        qi[r] = fmaf(ci[r], xm.x, qi[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int nu = m + r0 + r;
    out[(nu * (nu + 1) + m) * kRow] = make_float2(pr[r], pi[r]);
    if (TWO) out[(nu * (nu + 1) - m) * kRow] = make_float2(qr[r], qi[r]);
  }
}

template <bool TWO>
__device__ __forceinline__ void coax_dispatch(int R, const float2* C, int ws, int w, int m, int r0,
                                              const float2* in, float2* out) {
  switch (R) {
    case 1: coax_task<1, TWO>(C, ws, w, m, r0, in, out); break;
    case 2: coax_task<2, TWO>(C, ws, w, m, r0, in, out); break;
    case 3: coax_task<3, TWO>(C, ws, w, m, r0, in, out); break;
    default: coax_task<4, TWO>(C, ws, w, m, r0, in, out); break;
  }
}

__global__ void __launch_bounds__(kThreads, 2) translate_kernel(const TranslateArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int P = a.order;
  const SmemPlan sp = smem_plan(P);
  const int dim = sp.dim;
  float* s_rot = smem;
  float2* s_coax = reinterpret_cast<float2*>(s_rot + sp.rot_floats);
  float2* s_ph = s_coax + sp.coax_c;  // e^{i m phi}, index m + P
  float2* A = s_ph + sp.phase_c;
  float2* B = A + sp.tile_c;
  int* s_roff = reinterpret_cast<int*>(B + sp.tile_c);  // rotation block offsets per degree
  int* s_coff = s_roff + 32;                             // coaxial block offsets per order
  signed char* s_m = reinterpret_cast<signed char*>(s_coff + 32);  // order m of coefficient i

  const TranslateItem item = a.items[blockIdx.x];
  const TranslateClass cls = a.classes[item.cls];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int count = int(item.count);

  {
    const float4* g_rot = reinterpret_cast<const float4*>(a.rot_tables + size_t(cls.rot) * sp.rot_floats);
    for (int i = tid; i < sp.rot_floats / 4; i += kThreads) reinterpret_cast<float4*>(s_rot)[i] = g_rot[i];
    const float4* g_coax =
        reinterpret_cast<const float4*>(a.coax_tables + size_t(cls.coax) * sp.coax_c * 2);
    for (int i = tid; i < sp.coax_c / 2; i += kThreads) reinterpret_cast<float4*>(s_coax)[i] = g_coax[i];
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
    if (tid <= P) {
      s_roff[tid] = rot_block_offset(tid);
      s_coff[tid] = coax_block_offset(P, tid);
    }
    for (int i = tid; i < dim; i += kThreads) {
      int n = int(sqrtf(float(i)));
      while (n * n > i) --n;
      while ((n + 1) * (n + 1) <= i) ++n;
      s_m[i] = (signed char)(i - n * (n + 1));
    }
  }
  __syncthreads();

  // stage 1: gather the sources (4 pairs x 8 lanes per warp, 64-byte runs), apply e^{i m phi}
  {
    const int q = lane >> 3, e = lane & 7, p = warp * 4 + q;
    const bool live = p < count;
    const float2* row = live ? a.src + size_t(a.pair_src[item.pair_begin + p]) * a.stride : nullptr;
    for (int i = e; i < dim; i += 8) {
      float2 v = make_float2(0.f, 0.f);
      if (live) {
        const float2 x = row[i], ph = s_ph[int(s_m[i]) + P];
        v = make_float2(x.x * ph.x - x.y * ph.y, x.x * ph.y + x.y * ph.x);
      }
      A[i * kRow + p] = v;
    }
  }
  __syncthreads();

  const TranslateSchedule* sched = a.schedule;
  // stage 2: forward rotation A -> B
  for (int t = sched->rot_begin[warp]; t < sched->rot_begin[warp + 1]; ++t) {
    const uint32_t task = sched->rot_tasks[t];
    const int n = task & 0xff, r0 = (task >> 8) & 0xff, R = (task >> 16) & 0xff;
    rot_dispatch<false>(R, s_rot + s_roff[n] + r0, rot_row_stride(n), 2 * n + 1, A + n * n * kRow + lane,
                        B + (n * n + r0) * kRow + lane, nullptr, false);
  }
  __syncthreads();
  // stage 3: coaxial translation B -> A
  for (int t = sched->coax_begin[warp]; t < sched->coax_begin[warp + 1]; ++t) {
    const uint32_t task = sched->coax_tasks[t];
    const int m = task & 0xff, r0 = (task >> 8) & 0xff, R = (task >> 16) & 0xff;
    if (m == 0)
      coax_dispatch<false>(R, s_coax + s_coff[m], coax_row_stride(P, m), P + 1 - m, m, r0, B + lane, A + lane);
    else
      coax_dispatch<true>(R, s_coax + s_coff[m], coax_row_stride(P, m), P + 1 - m, m, r0, B + lane, A + lane);
  }
  __syncthreads();
  // stage 4: inverse rotation A -> B, with e^{-i mu phi}
  for (int t = sched->rot_begin[warp]; t < sched->rot_begin[warp + 1]; ++t) {
    const uint32_t task = sched->rot_tasks[t];
    const int n = task & 0xff, r0 = (task >> 8) & 0xff, R = (task >> 16) & 0xff;
    rot_dispatch<true>(R, s_rot + s_roff[n] + r0, rot_row_stride(n), 2 * n + 1, A + n * n * kRow + lane,
                       B + (n * n + r0) * kRow + lane, s_ph + (r0 - n + P), (r0 & 1) != 0);
  }
  __syncthreads();

  // stage 5: accumulate into the destinations, two coefficients (16 bytes) per reduction
  {
    const int q = lane >> 3, e = lane & 7, p = warp * 4 + q;
    if (p < count) {
      float* dst = reinterpret_cast<float*>(a.dst + size_t(a.pair_dst[item.pair_begin + p]) * a.stride);
      for (int i2 = e; i2 < dim / 2; i2 += 8) {
        const float2 lo = B[(2 * i2) * kRow + p], hi = B[(2 * i2 + 1) * kRow + p];
        atomicAdd(reinterpret_cast<float4*>(dst) + i2, make_float4(lo.x, lo.y, hi.x, hi.y));
      }
      if ((dim & 1) && e == 0) atomicAdd(reinterpret_cast<float2*>(dst) + (dim - 1), B[(dim - 1) * kRow + p]);
    }
  }
}

}  // namespace

// host side: cut the stages into tasks and hand them to the warps (longest processing time first)
void build_translate_schedule(int P, TranslateSchedule* out) {
  struct Task {
    uint32_t code;
    int cost;
  };
  auto distribute = [](std::vector<Task>& tasks, uint32_t* flat, int* begin, int cap) {
    std::stable_sort(tasks.begin(), tasks.end(), [](const Task& x, const Task& y) { return x.cost > y.cost; });
    std::vector<std::vector<uint32_t>> per(kWarps);
    long load[kWarps] = {};
    for (const Task& t : tasks) {
      int best = 0;
      for (int w = 1; w < kWarps; ++w)
        if (load[w] < load[best]) best = w;
      per[best].push_back(t.code);
      load[best] += t.cost;
    }
    int pos = 0;
    for (int w = 0; w < kWarps; ++w) {
      begin[w] = pos;
      for (uint32_t c : per[w]) {
        if (pos >= cap) throw Error(HFMM_ERR_INTERNAL, "translation schedule overflow");
        flat[pos++] = c;
      }
    }
    begin[kWarps] = pos;
  };
  std::vector<Task> rot, coax;
  for (int n = 0; n <= P; ++n) {
    const int w = 2 * n + 1;
    // tiles start at multiples of 4 (aligned 16-byte coefficient loads) and hold <= 12 rows; the
    // split minimising sum(2R + 6) (instructions per input step) is found by exhaustive search
    int best_cost = 1 << 30, best_parts[8] = {}, best_n = 0;
    for (int a = 0; a <= 12; a += 4)
      for (int b = 0; b <= 12; b += 4)
        for (int c = 0; c <= 12; c += 4) {
          const int last = w - a - b - c;
          if (last < 1 || last > 12) continue;
          if ((a == 0 && (b || c)) || (b == 0 && c)) continue;  // leading parts first
          int parts[4] = {a, b, c, last}, np = 0, cost = 0, tmp[4];
          for (int v : parts)
            if (v) {
              tmp[np++] = v;
              cost += 2 * v + 6;
            }
          if (cost < best_cost) {
            best_cost = cost;
            best_n = np;
            for (int i = 0; i < np; ++i) best_parts[i] = tmp[i];
          }
        }
    int r0 = 0;
    for (int i = 0; i < best_n; ++i) {
      const int R = best_parts[i];
      rot.push_back({uint32_t(n) | uint32_t(r0) << 8 | uint32_t(R) << 16, w * (2 * R + 6)});
      r0 += R;
    }
  }
  for (int m = 0; m <= P; ++m) {
    const int w = P + 1 - m;
    for (int r0 = 0; r0 < w; r0 += 4) {
      const int R = std::min(4, w - r0);
      coax.push_back({uint32_t(m) | uint32_t(r0) << 8 | uint32_t(R) << 16, w * ((m ? 8 : 4) * R + 8)});
    }
  }
  distribute(rot, out->rot_tasks, out->rot_begin, kTranslateMaxTasks);
  distribute(coax, out->coax_tasks, out->coax_begin, kTranslateMaxTasks);
}

int translate_batch_size(int) { return kTranslateBatch; }

void launch_translate(const TranslateArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  const SmemPlan sp = smem_plan(a.order);
  static int configured_for = -1;
  if (configured_for < int(sp.bytes)) {
    HFMM_CUDA_CHECK(cudaFuncSetAttribute(translate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sp.bytes)));
    configured_for = int(sp.bytes);
  }
  translate_kernel<<<a.n_items, kThreads, sp.bytes, s>>>(a);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

}  // namespace hfmm_b200
