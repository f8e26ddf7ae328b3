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

// Shared memory is addressed with 32-bit offsets from one base so the loops advance with a couple
// of integer adds (generic 64-bit pointer arithmetic tripled the instruction count).
__device__ __forceinline__ float2 lds2(const float* base, uint32_t off) {
  return *reinterpret_cast<const float2*>(base + off);
}
__device__ __forceinline__ float4 lds4(const float* base, uint32_t off) {
  return *reinterpret_cast<const float4*>(base + off);
}

// ---- rotation task: rows [r0, r0+R) of block n;  out[r] = sum_k E[k][r0+r] * in[k] -------------
// e_off / in_off / out_off / ph_off: float offsets into the shared-memory window `sm`
template <int R, bool BACK>
__device__ __forceinline__ void rot_task(float* __restrict__ sm, uint32_t e_off, uint32_t ws,
                                         int w, uint32_t in_off, uint32_t out_off, uint32_t ph_off,
                                         bool odd0) {
  float ar[R], ai[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ar[r] = ai[r] = 0.0f;
  constexpr int NV = (R + 3) / 4;
  constexpr uint32_t kRowF = 2 * kRow;  // floats per operand row
  // two inputs per trip; in the inverse rotation odd inputs enter negated ((-1)^k of the symmetry)
  uint32_t e1_off = e_off + ws;
  const uint32_t ws2 = 2 * ws;
#pragma unroll 1
  for (int trips = w >> 1; trips > 0; --trips) {
    const float2 x0 = lds2(sm, in_off), x1 = lds2(sm, in_off + kRowF);
    float e0[NV * 4], e1[NV * 4];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 a = lds4(sm, e_off + 4 * v);
      const float4 b = lds4(sm, e1_off + 4 * v);
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
    in_off += 2 * kRowF;
    e_off += ws2;
    e1_off += ws2;
  }
  {  // w is odd: one even-indexed input left
    const float2 x0 = lds2(sm, in_off);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 a = lds4(sm, e_off + 4 * v);
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
    float2 o;
    if (BACK) {
      // (-1)^{row} of the symmetry, then e^{-i mu phi}
      const bool neg = ((r & 1) != 0) != odd0;
      const float sr = neg ? -ar[r] : ar[r], si = neg ? -ai[r] : ai[r];
      const float2 p = lds2(sm, ph_off + 2 * r);
      o = make_float2(sr * p.x + si * p.y, si * p.x - sr * p.y);
    } else {
      o = make_float2(ar[r], ai[r]);
    }
    *reinterpret_cast<float2*>(sm + out_off + r * kRowF) = o;
  }
}

template <bool BACK>
__device__ __forceinline__ void rot_dispatch(int R, float* sm, uint32_t e_off, uint32_t ws, int w,
                                             uint32_t in_off, uint32_t out_off, uint32_t ph_off,
                                             bool odd0) {
  switch (R) {
    case 1: rot_task<1, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 2: rot_task<2, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 3: rot_task<3, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 4: rot_task<4, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 5: rot_task<5, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 6: rot_task<6, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 7: rot_task<7, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 8: rot_task<8, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 9: rot_task<9, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 10: rot_task<10, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    case 11: rot_task<11, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
    default: rot_task<12, BACK>(sm, e_off, ws, w, in_off, out_off, ph_off, odd0); break;
  }
}

// ---- coaxial task: rows nu = m + r0 .. m + r0 + R - 1 of order m, columns +m and -m -----------
// c_off: float offset of Chat^m[0][r0]; ws: row stride in floats; in_off/out_off: tile + lane
template <int R, bool TWO>
__device__ __forceinline__ void coax_task(float* __restrict__ sm, uint32_t c_off, uint32_t ws, int w,
                                          int m, int r0, uint32_t in_off, uint32_t out_off) {
  float pr[R], pi[R], qr[R], qi[R];  // +m and -m accumulators
#pragma unroll
  for (int r = 0; r < R; ++r) pr[r] = pi[r] = qr[r] = qi[r] = 0.0f;
  constexpr uint32_t kRowF = 2 * kRow;
  // input rows (n, +m) and (n, -m), n = m .. P: index n(n+1) +- m, advancing by 2n+2 rows
  uint32_t p_off = in_off + uint32_t(m * (m + 1) + m) * kRowF;
  uint32_t q_off = in_off + uint32_t(m * (m + 1) - m) * kRowF;
  uint32_t step = uint32_t(2 * m + 2) * kRowF;
#pragma unroll 1
  for (int k = w; k > 0; --k) {
    const float2 xp = lds2(sm, p_off);
    float2 xm = make_float2(0.f, 0.f);
    if (TWO) xm = lds2(sm, q_off);
    float cr[R], ci[R];
    if (R == 1) {
      const float2 c = lds2(sm, c_off);
      cr[0] = c.x; ci[0] = c.y;
    } else {
#pragma unroll
      for (int v = 0; v < (R + 1) / 2; ++v) {
        const float4 c = lds4(sm, c_off + 4 * v);
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
    p_off += step;
    q_off += step;
    step += 2 * kRowF;
    c_off += ws;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int nu = m + r0 + r;
    *reinterpret_cast<float2*>(sm + out_off + uint32_t(nu * (nu + 1) + m) * kRowF) = make_float2(pr[r], pi[r]);
    if (TWO)
      *reinterpret_cast<float2*>(sm + out_off + uint32_t(nu * (nu + 1) - m) * kRowF) = make_float2(qr[r], qi[r]);
  }
}

template <bool TWO>
__device__ __forceinline__ void coax_dispatch(int R, float* sm, uint32_t c_off, uint32_t ws, int w,
                                              int m, int r0, uint32_t in_off, uint32_t out_off) {
  switch (R) {
    case 1: coax_task<1, TWO>(sm, c_off, ws, w, m, r0, in_off, out_off); break;
    case 2: coax_task<2, TWO>(sm, c_off, ws, w, m, r0, in_off, out_off); break;
    case 3: coax_task<3, TWO>(sm, c_off, ws, w, m, r0, in_off, out_off); break;
    default: coax_task<4, TWO>(sm, c_off, ws, w, m, r0, in_off, out_off); break;
  }
}

// Persistent CTAs: each walks a contiguous range of work items (items are sorted by class, so the
// tables in shared memory are reloaded only when the class changes).  The gather of the NEXT item
// is issued into registers while the current item drains through its reductions, so the chain
// item -> pair list -> source rows never sits on the critical path.
template <int NG>  // source elements per lane of the gather: ceil((P+1)^2 / 8)
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

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t it_begin = uint32_t(uint64_t(a.n_items) * blockIdx.x / gridDim.x);
  const uint32_t it_end = uint32_t(uint64_t(a.n_items) * (blockIdx.x + 1) / gridDim.x);
  if (it_begin >= it_end) return;

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

  // gather mapping: 4 pairs x 8 lanes per warp (64-byte runs of a source row)
  const int gq = lane >> 3, ge = lane & 7, gp = warp * 4 + gq;
  float2 gx[NG];
  auto issue_gather = [&](const TranslateItem& it) {
    const bool live = gp < int(it.count);
    const float2* row = live ? a.src + size_t(a.pair_src[it.pair_begin + gp]) * a.stride : nullptr;
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const int i = ge + 8 * j;
      gx[j] = (live && i < dim) ? row[i] : make_float2(0.f, 0.f);
    }
  };

  const TranslateSchedule* sched = a.schedule;
  // float offsets of the regions inside the shared window
  const uint32_t rot_f = 0, coax_f = uint32_t(sp.rot_floats),
                 ph_f = coax_f + 2u * uint32_t(sp.coax_c),
                 a_f = ph_f + 2u * uint32_t(sp.phase_c), b_f = a_f + 2u * uint32_t(sp.tile_c);
  constexpr uint32_t kRowF = 2 * kRow;

  TranslateItem item = a.items[it_begin];
  issue_gather(item);
  uint32_t loaded_cls = 0xffffffffu;

  for (uint32_t it = it_begin; it < it_end; ++it) {
    const int count = int(item.count);
    if (item.cls != loaded_cls) {  // CTA-uniform
      // every warp is past the previous item's stage 4 (the last reader of the tables)
      const TranslateClass cls = a.classes[item.cls];
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
      loaded_cls = item.cls;
      __syncthreads();
    }

    // stage 1: apply e^{i m phi} to the gathered sources, store element-major into A
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const int i = ge + 8 * j;
      if (i < dim) {
        const float2 x = gx[j], ph = s_ph[int(s_m[i]) + P];
        A[i * kRow + gp] = make_float2(x.x * ph.x - x.y * ph.y, x.x * ph.y + x.y * ph.x);
      }
    }
    __syncthreads();
    // metadata of the next item (consumed in stage 5)
    TranslateItem next = item;
    const bool has_next = it + 1 < it_end;
    if (has_next) next = a.items[it + 1];

    // stage 2: forward rotation A -> B
    for (int t = sched->rot_begin[warp]; t < sched->rot_begin[warp + 1]; ++t) {
      const uint32_t task = sched->rot_tasks[t];
      const int n = task & 0xff, r0 = (task >> 8) & 0xff, R = (task >> 16) & 0xff;
      rot_dispatch<false>(R, smem, rot_f + s_roff[n] + r0, rot_row_stride(n), 2 * n + 1,
                          a_f + uint32_t(n * n) * kRowF + 2 * lane,
                          b_f + uint32_t(n * n + r0) * kRowF + 2 * lane, 0, false);
    }
    __syncthreads();
    // stage 3: coaxial translation B -> A
    for (int t = sched->coax_begin[warp]; t < sched->coax_begin[warp + 1]; ++t) {
      const uint32_t task = sched->coax_tasks[t];
      const int m = task & 0xff, r0 = (task >> 8) & 0xff, R = (task >> 16) & 0xff;
      const uint32_t c_off = coax_f + 2u * uint32_t(s_coff[m] + r0), cws = 2u * coax_row_stride(P, m);
      if (m == 0)
        coax_dispatch<false>(R, smem, c_off, cws, P + 1 - m, m, r0, b_f + 2 * lane, a_f + 2 * lane);
      else
        coax_dispatch<true>(R, smem, c_off, cws, P + 1 - m, m, r0, b_f + 2 * lane, a_f + 2 * lane);
    }
    __syncthreads();
    // stage 4: inverse rotation A -> B, with e^{-i mu phi}
    for (int t = sched->rot_begin[warp]; t < sched->rot_begin[warp + 1]; ++t) {
      const uint32_t task = sched->rot_tasks[t];
      const int n = task & 0xff, r0 = (task >> 8) & 0xff, R = (task >> 16) & 0xff;
      rot_dispatch<true>(R, smem, rot_f + s_roff[n] + r0, rot_row_stride(n), 2 * n + 1,
                         a_f + uint32_t(n * n) * kRowF + 2 * lane,
                         b_f + uint32_t(n * n + r0) * kRowF + 2 * lane, ph_f + 2u * uint32_t(r0 - n + P),
                         (r0 & 1) != 0);
    }
    __syncthreads();

    // stage 5: start the next item's gather, then accumulate this item into its destinations,
    // two coefficients (16 bytes) per reduction
    if (has_next) issue_gather(next);
    if (gp < count) {
      float* dst = reinterpret_cast<float*>(a.dst + size_t(a.pair_dst[item.pair_begin + gp]) * a.stride);
      for (int i2 = ge; i2 < dim / 2; i2 += 8) {
        const float2 lo = B[(2 * i2) * kRow + gp], hi = B[(2 * i2 + 1) * kRow + gp];
        atomicAdd(reinterpret_cast<float4*>(dst) + i2, make_float4(lo.x, lo.y, hi.x, hi.y));
      }
      if ((dim & 1) && ge == 0)
        atomicAdd(reinterpret_cast<float2*>(dst) + (dim - 1), B[(dim - 1) * kRow + gp]);
    }
    item = next;
    // no barrier here: the next stage 1 only writes A (last read in stage 4), and the barrier after
    // it orders this stage's reads of B before the next stage 2 overwrites B
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

namespace {
template <int NG>
void launch_translate_ng(const TranslateArgs& a, cudaStream_t s, size_t bytes, int ctas) {
  static int configured_for = -1;
  if (configured_for < int(bytes)) {
    HFMM_CUDA_CHECK(cudaFuncSetAttribute(translate_kernel<NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(bytes)));
    configured_for = int(bytes);
  }
  translate_kernel<NG><<<ctas, kThreads, bytes, s>>>(a);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
}  // namespace

void launch_translate(const TranslateArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  const SmemPlan sp = smem_plan(a.order);
  static int sm_count = 0;
  if (!sm_count) {
    int dev = 0;
    HFMM_CUDA_CHECK(cudaGetDevice(&dev));
    HFMM_CUDA_CHECK(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
  }
  // persistent grid: two CTAs per SM when their shared memory fits (227 KB per SM), else one
  const int per_sm = 2 * (sp.bytes + 1024) <= 227 * 1024 ? 2 : 1;
  const int ctas = int(std::min<uint32_t>(a.n_items, uint32_t(per_sm * sm_count)));
  const int ng = (sp.dim + 7) / 8;
  if (ng <= 11) launch_translate_ng<11>(a, s, sp.bytes, ctas);        // P <= 8
  else if (ng <= 16) launch_translate_ng<16>(a, s, sp.bytes, ctas);   // P <= 10
  else if (ng <= 22) launch_translate_ng<22>(a, s, sp.bytes, ctas);   // P <= 12
  else if (ng <= 29) launch_translate_ng<29>(a, s, sp.bytes, ctas);   // P <= 14
  else launch_translate_ng<37>(a, s, sp.bytes, ctas);                 // P <= 16
}

}  // namespace hfmm_b200
