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
//   * rotations run on FOLDED vectors (tables.hpp): the +-m symmetry of the Wigner-d blocks halves
//     their multiply-adds; vectors are folded in the gather and unfolded once before the reductions;
//   * the inverse rotation reuses the same table through d^n_{mu,m'} = (-1)^{mu-m'} d^n_{m',mu};
//   * pairs of one batch have different destinations: results leave through 16-byte vector
//     reductions (RED.E.ADD.F32x4) into HBM/L2.
// FP32 work per pair: 2 * 2*sum_n ((n+1)^2 + n^2) + 4*sum_m (P+1-|m|)^2 FFMAs (11.9 k at P = 12) against
// 4 (P+1)^4 = 114 k for the reference's dense complex mat-vec.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "device_utils.cuh"
#include "kernels.cuh"
#include "tables.hpp"

namespace hfmm_b200 {

namespace {


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
  s.phase_c = (P + 2) & ~1;
  s.tile_c = s.dim * kRow;
  // rot | coax | phases | tile A | tile B | (n, m) of every gather unit (u16)
  s.bytes = size_t(s.rot_floats) * 4 + size_t(s.coax_c + s.phase_c + 2 * s.tile_c) * 8 +
            size_t(((P + 1) * (P + 2) / 2 * 6 + 15) & ~15);
  return s;
}

// Shared memory is addressed with 32-bit BYTE addresses in the shared window (explicit
// ld.shared / st.shared), so the loops advance with one integer add per pointer and the loads use
// register + immediate addressing (generic pointers cost an address computation per access).
__device__ __forceinline__ float2 lds2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts2(uint32_t addr, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}

// warps per CTA: 8 with two CTAs per SM while two operand tile pairs fit the 227 KB of shared memory
// (P <= 12), else ONE CTA of 16 warps per SM so the SM keeps 16 resident warps (P = 13..16)
inline bool translate_two_ctas(int P) { return 2 * (smem_plan(P).bytes + 1024) <= size_t(227) * 1024; }
inline int translate_warps(int P) {
  static const int forced = [] {
    const char* e = getenv("HFMM_TRANSLATE_WARPS");
    return e ? atoi(e) : 0;
  }();
  if (forced == 8 || forced == 16) return translate_two_ctas(P) ? forced : 16;
  return translate_two_ctas(P) ? 8 : 16;
}

// ---- packed FP32 (sm_100a FFMA2): one instruction = two FMAs; with a complex accumulator held as
// a (re, im) register pair, "acc += e * x" (real e, complex x) is ONE FFMA2 with e as the scalar
// operand, and a complex multiply-add is two.  Same FLOP peak as FFMA (74.1 vs 72.4 TFLOP/s
// measured), half the issue slots — and this kernel is issue-bound.
using u64 = unsigned long long;
__device__ __forceinline__ u64 pack2(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 unpack2(u64 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// acc += x * s  (x: complex pair, s: real scalar broadcast to both halves)
__device__ __forceinline__ void fma2s(u64& acc, u64 x, float s) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(x), "l"(pack2(s, s)));
}
__device__ __forceinline__ u64 ldsp(uint32_t addr) {
  u64 v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void stsp(uint32_t addr, u64 v) {
  asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ u64 neg2(u64 v) {
  const float2 f = unpack2(v);
  return pack2(-f.x, -f.y);
}

// ---- rotation task: R output rows of one folded sub-block;  out[r] = sum_k E[k][r] * in[k] ------
// e_off / in_off / out_off: float offsets into the shared-memory window `sm`
template <int R, bool BACK>
__device__ __forceinline__ void rot_task(uint32_t e_addr, uint32_t ws_b, int w, uint32_t in_addr,
                                         uint32_t out_addr, bool odd0) {
  u64 acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0ull;
  constexpr int NV = (R + 3) / 4;
  constexpr uint32_t kRowB = 8 * kRow;  // bytes per operand row
  // two inputs per trip; in the inverse rotation odd inputs enter negated ((-1)^k of the symmetry)
  uint32_t e1_addr = e_addr + ws_b;
  const uint32_t ws2 = 2 * ws_b;
#pragma unroll 1
  for (int trips = w >> 1; trips > 0; --trips) {
    const u64 x0 = ldsp(in_addr);
    u64 x1 = ldsp(in_addr + kRowB);
    if (BACK) x1 = neg2(x1);
    float e0[NV * 4], e1[NV * 4];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 a = lds4(e_addr + 16 * v);
      const float4 b = lds4(e1_addr + 16 * v);
      e0[4 * v] = a.x; e0[4 * v + 1] = a.y; e0[4 * v + 2] = a.z; e0[4 * v + 3] = a.w;
      e1[4 * v] = b.x; e1[4 * v + 1] = b.y; e1[4 * v + 2] = b.z; e1[4 * v + 3] = b.w;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) fma2s(acc[r], x0, e0[r]);
#pragma unroll
    for (int r = 0; r < R; ++r) fma2s(acc[r], x1, e1[r]);
    in_addr += 2 * kRowB;
    e_addr += ws2;
    e1_addr += ws2;
  }
  if (w & 1) {  // one even-indexed input left
    const u64 x0 = ldsp(in_addr);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 a = lds4(e_addr + 16 * v);
      const float ev[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 * v + j < R) fma2s(acc[4 * v + j], x0, ev[j]);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    u64 o = acc[r];
    if (BACK) {  // (-1)^{row} of the symmetry
      const bool neg = ((r & 1) != 0) != odd0;
      if (neg) o = neg2(o);
    }
    stsp(out_addr + r * kRowB, o);
  }
}

template <bool BACK, int MAXR>
__device__ __forceinline__ void rot_dispatch(int R, uint32_t e_addr, uint32_t ws_b, int w,
                                             uint32_t in_addr, uint32_t out_addr, bool odd0) {
  if (MAXR == 8) {  // the 64-register variant never schedules taller tiles
    switch (R) {
      case 1: rot_task<1, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
      case 2: rot_task<2, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
      case 3: rot_task<3, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
      case 4: rot_task<4, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
      case 5: rot_task<5, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
      case 6: rot_task<6, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
      case 7: rot_task<7, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
      default: rot_task<8, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    }
    return;
  }
  switch (R) {
    case 1: rot_task<1, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 2: rot_task<2, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 3: rot_task<3, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 4: rot_task<4, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 5: rot_task<5, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 6: rot_task<6, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 7: rot_task<7, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 8: rot_task<8, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 9: rot_task<9, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 10: rot_task<10, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    case 11: rot_task<11, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
    default: rot_task<12, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0); break;
  }
}

// ---- coaxial task: rows nu = m + r0 .. m + r0 + R - 1 of order m, folded columns s_m and t_m ---
// (for m = 0 only the single column x_0).  p_off / q_off: float offsets of the first input rows
// (degree n = m) of the two columns; they advance by 2n+1 and 2n+2 rows per degree.
template <int R, bool TWO>
__device__ __forceinline__ void coax_task(uint32_t c_addr, uint32_t ws_b, int w, int m, int r0,
                                          uint32_t p_addr, uint32_t q_addr, uint32_t out_base) {
  u64 p[R], q[R];
#pragma unroll
  for (int r = 0; r < R; ++r) p[r] = q[r] = 0ull;
  constexpr uint32_t kRowB = 8 * kRow;
  uint32_t step = uint32_t(2 * m + 1) * kRowB;
#pragma unroll 1
  for (int k = w; k > 0; --k) {
    // c * x = cr * (x.re, x.im) + ci * (-x.im, x.re): two FFMA2 per complex multiply-add
    const float2 xp = lds2(p_addr);
    const u64 xpv = pack2(xp.x, xp.y), xpt = pack2(-xp.y, xp.x);
    u64 xqv = 0ull, xqt = 0ull;
    if (TWO) {
      const float2 xq = lds2(q_addr);
      xqv = pack2(xq.x, xq.y);
      xqt = pack2(-xq.y, xq.x);
    }
    float cr[R], ci[R];
    if (R == 1) {
      const float2 c = lds2(c_addr);
      cr[0] = c.x; ci[0] = c.y;
    } else {
#pragma unroll
      for (int v = 0; v < (R + 1) / 2; ++v) {
        const float4 c = lds4(c_addr + 16 * v);
        cr[2 * v] = c.x; ci[2 * v] = c.y;
        if (2 * v + 1 < R) { cr[2 * v + 1] = c.z; ci[2 * v + 1] = c.w; }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(p[r], xpv, cr[r]);
      if (TWO) fma2s(q[r], xqv, cr[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(p[r], xpt, ci[r]);
      if (TWO) fma2s(q[r], xqt, ci[r]);
    }
    p_addr += step;
    q_addr += step + kRowB;
    step += 2 * kRowB;
    c_addr += ws_b;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int nu = m + r0 + r;
    stsp(out_base + uint32_t(nu * nu + m) * kRowB, p[r]);
    if (TWO) stsp(out_base + uint32_t(nu * nu + nu + m) * kRowB, q[r]);
  }
}

template <bool TWO>
__device__ __forceinline__ void coax_dispatch(int R, uint32_t c_addr, uint32_t ws_b, int w, int m,
                                              int r0, uint32_t p_addr, uint32_t q_addr, uint32_t out_base) {
  switch (R) {
    case 1: coax_task<1, TWO>(c_addr, ws_b, w, m, r0, p_addr, q_addr, out_base); break;
    case 2: coax_task<2, TWO>(c_addr, ws_b, w, m, r0, p_addr, q_addr, out_base); break;
    case 3: coax_task<3, TWO>(c_addr, ws_b, w, m, r0, p_addr, q_addr, out_base); break;
    default: coax_task<4, TWO>(c_addr, ws_b, w, m, r0, p_addr, q_addr, out_base); break;  // tiles hold <= 4 rows
  }
}

// per-order static schedules live in constant memory: a task is four words, read with
// warp-uniform addresses, so handing a task to a warp costs two LDC.64 and no arithmetic
__constant__ TranslateSchedule c_sched[kMaxOrder + 1];

// Persistent CTAs: each walks a contiguous range of work items (items are sorted by class, so the
// tables in shared memory are reloaded only when the class changes).  The gather of the NEXT item
// is issued into registers while the current item drains through its reductions, so the chain
// item -> pair list -> source rows never sits on the critical path.
template <int NU, int WARPS, int CTAS>  // NU: (n, m >= 0) gather units per lane = ceil((P+1)(P+2)/2 / WARPS)
__global__ void __launch_bounds__(WARPS * 32, CTAS) translate_kernel(const TranslateArgs a) {
  constexpr int kThreads = WARPS * 32;
  constexpr int kMaxR = WARPS == 8 ? 12 : 8;
  constexpr int kLanesPerPair = WARPS;  // 32 pairs x WARPS lanes = all threads of the CTA
  extern __shared__ __align__(16) float smem[];
  const int P = a.order;
  const SmemPlan sp = smem_plan(P);
  const int dim = sp.dim, n_units = (P + 1) * (P + 2) / 2;
  float* s_rot = smem;
  float2* s_coax = reinterpret_cast<float2*>(s_rot + sp.rot_floats);
  float2* s_ph = s_coax + sp.coax_c;  // e^{i m phi}, m = 0..P
  float2* A = s_ph + sp.phase_c;
  float2* B = A + sp.tile_c;
  // per gather unit (n, m >= 0): raw index of (n, +m) << 16 | folded row of s_m;  t_m sits n rows
  // further, (n, -m) sits 2m raw entries back
  uint32_t* s_unit = reinterpret_cast<uint32_t*>(B + sp.tile_c);
  unsigned char* s_um = reinterpret_cast<unsigned char*>(s_unit + n_units);  // (n << 4 | m) needs 2 bytes

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t it_begin = uint32_t(uint64_t(a.n_items) * blockIdx.x / gridDim.x);
  const uint32_t it_end = uint32_t(uint64_t(a.n_items) * (blockIdx.x + 1) / gridDim.x);
  if (it_begin >= it_end) return;

  for (int u = tid; u < n_units; u += kThreads) {
    int n = int((sqrtf(8.0f * float(u) + 1.0f) - 1.0f) * 0.5f);
    while (n * (n + 1) / 2 > u) --n;
    while ((n + 1) * (n + 2) / 2 <= u) ++n;
    const int m = u - n * (n + 1) / 2;
    s_unit[u] = uint32_t(n * (n + 1) + m) << 16 | uint32_t(n * n + m);
    s_um[2 * u] = (unsigned char)n;
    s_um[2 * u + 1] = (unsigned char)m;
  }

  // gather mapping: 32/WARPS pairs x WARPS lanes per warp; a lane owns units u = ge + WARPS j, i.e.
  // the two source coefficients (n, +m) and (n, -m) it folds into s_m and t_m
  const int gq = lane / kLanesPerPair, ge = lane % kLanesPerPair, gp = warp * (32 / kLanesPerPair) + gq;
  float2 gxp[NU], gxm[NU];
  auto issue_gather = [&](const TranslateItem& it) {
    const bool live = gp < int(it.count);
    const float2* row = live ? a.src + size_t(a.pair_src[it.pair_begin + gp]) * a.stride : nullptr;
#pragma unroll
    for (int j = 0; j < NU; ++j) {
      const int u = ge + kLanesPerPair * j;
      gxp[j] = gxm[j] = make_float2(0.f, 0.f);
      if (live && u < n_units) {
        const int i = s_unit[u] >> 16, m = s_um[2 * u + 1];
        gxp[j] = row[i];
        gxm[j] = row[i - 2 * m];
      }
    }
  };

  const TranslateSchedule& sched = c_sched[P];
  // byte addresses inside the shared window
  const uint32_t win = uint32_t(__cvta_generic_to_shared(smem));
  const uint32_t a_lane = uint32_t(__cvta_generic_to_shared(A)) + 8 * lane,
                 b_lane = uint32_t(__cvta_generic_to_shared(B)) + 8 * lane;

  __syncthreads();  // s_unit
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
      if (tid <= P) {
        float cr = 1.f, ci = 0.f;
        for (int j = 0; j < tid; ++j) {
          const float t = cr * cls.cphi - ci * cls.sphi;
          ci = ci * cls.cphi + cr * cls.sphi;
          cr = t;
        }
        s_ph[tid] = make_float2(cr, ci);
      }
      loaded_cls = item.cls;
      __syncthreads();
    }

    // stage 1: e^{i m phi}, fold, store element-major into A
    //   a = x_m e^{i m phi},  b = (-1)^m x_{-m} e^{-i m phi}:   s_m = a + b,  t_m = a - b
#pragma unroll
    for (int j = 0; j < NU; ++j) {
      const int u = ge + kLanesPerPair * j;
      if (u < n_units) {
        const int n = s_um[2 * u], m = s_um[2 * u + 1], fs = s_unit[u] & 0xffff;
        const float2 ph = s_ph[m], xp = gxp[j], xm = gxm[j];
        if (m == 0) {
          A[fs * kRow + gp] = xp;
        } else {
          const float2 av = make_float2(xp.x * ph.x - xp.y * ph.y, xp.x * ph.y + xp.y * ph.x);
          float2 bv = make_float2(xm.x * ph.x + xm.y * ph.y, xm.y * ph.x - xm.x * ph.y);
          if (m & 1) bv = make_float2(-bv.x, -bv.y);
          A[fs * kRow + gp] = make_float2(av.x + bv.x, av.y + bv.y);
          A[(fs + n) * kRow + gp] = make_float2(av.x - bv.x, av.y - bv.y);
        }
      }
    }
    __syncthreads();
    // metadata of the next item (consumed in stage 5)
    TranslateItem next = item;
    const bool has_next = it + 1 < it_end;
    if (has_next) next = a.items[it + 1];

    // stage 2: forward rotation A -> B
    for (int t = sched.rot_begin[warp]; t < sched.rot_begin[warp + 1]; ++t) {
      const TranslateRotTask d = sched.rot[t];
      rot_dispatch<false, kMaxR>((d.packed >> 16) & 0xff, win + d.e_off, d.packed & 0xff, (d.packed >> 8) & 0xff,
                          a_lane + d.in_rel, b_lane + d.out_rel, false);
    }
    __syncthreads();
    // stage 3: coaxial translation B -> A
    for (int t = sched.coax_begin[warp]; t < sched.coax_begin[warp + 1]; ++t) {
      const TranslateCoaxTask d = sched.coax[t];
      const int m = (d.packed >> 16) & 0x3f, r0 = (d.packed >> 22) & 0x3f, R = d.packed >> 28;
      if (m == 0)
        coax_dispatch<false>(R, win + d.c_off, d.packed & 0xff, (d.packed >> 8) & 0xff, m, r0,
                             b_lane + d.p_rel, b_lane + d.q_rel, a_lane);
      else
        coax_dispatch<true>(R, win + d.c_off, d.packed & 0xff, (d.packed >> 8) & 0xff, m, r0,
                            b_lane + d.p_rel, b_lane + d.q_rel, a_lane);
    }
    __syncthreads();
    // stage 4: inverse rotation A -> B (same table, sign-twiddled)
    for (int t = sched.rot_begin[warp]; t < sched.rot_begin[warp + 1]; ++t) {
      const TranslateRotTask d = sched.rot[t];
      rot_dispatch<true, kMaxR>((d.packed >> 16) & 0xff, win + d.e_off, d.packed & 0xff, (d.packed >> 8) & 0xff,
                         a_lane + d.in_rel, b_lane + d.out_rel, (d.packed >> 24) & 1);
    }
    __syncthreads();
    // stage 5a: unfold B -> A in the caller's coefficient order, with e^{-i mu phi}:
    //   y_m = (u + v)/2 e^{-i m phi},   y_{-m} = (-1)^m (u - v)/2 e^{+i m phi}
    for (int u = ge; u < n_units; u += kLanesPerPair) {
      const int n = s_um[2 * u], m = s_um[2 * u + 1], fs = s_unit[u] & 0xffff;
      const float2 uu = B[fs * kRow + gp];
      if (m == 0) {
        A[(n * n + n) * kRow + gp] = uu;
      } else {
        const float2 vv = B[(fs + n) * kRow + gp], ph = s_ph[m];
        const float2 yp = make_float2(0.5f * (uu.x + vv.x), 0.5f * (uu.y + vv.y));
        float2 ym = make_float2(0.5f * (uu.x - vv.x), 0.5f * (uu.y - vv.y));
        if (m & 1) ym = make_float2(-ym.x, -ym.y);
        A[(n * n + n + m) * kRow + gp] = make_float2(yp.x * ph.x + yp.y * ph.y, yp.y * ph.x - yp.x * ph.y);
        A[(n * n + n - m) * kRow + gp] = make_float2(ym.x * ph.x - ym.y * ph.y, ym.x * ph.y + ym.y * ph.x);
      }
    }
    // a lane group reads back only what it wrote itself (same pair column gp): a warp-level
    // barrier orders the stores of the lanes of the group before the loads below
    __syncwarp();

    // stage 5b: start the next item's gather, then accumulate this item into its destinations,
    // two coefficients (16 bytes) per reduction
    if (has_next) issue_gather(next);
    if (gp < count) {
      float* dst = reinterpret_cast<float*>(a.dst + size_t(a.pair_dst[item.pair_begin + gp]) * a.stride);
      for (int i2 = ge; i2 < dim / 2; i2 += kLanesPerPair) {
        const float2 lo = A[(2 * i2) * kRow + gp], hi = A[(2 * i2 + 1) * kRow + gp];
        atomicAdd(reinterpret_cast<float4*>(dst) + i2, make_float4(lo.x, lo.y, hi.x, hi.y));
      }
      if ((dim & 1) && ge == 0)
        atomicAdd(reinterpret_cast<float2*>(dst) + (dim - 1), A[(dim - 1) * kRow + gp]);
    }
    item = next;
    // the next stage 1 overwrites A: every warp must be done reading it
    __syncthreads();
  }
}

}  // namespace

// host side: cut the stages into tasks, precompute every shared-memory offset a task needs, and
// hand the tasks to the warps (longest processing time first)
void build_translate_schedule(int P, TranslateSchedule* out) {
  const SmemPlan sp = smem_plan(P);
  const int kWarps = translate_warps(P);
  const int max_rows = kWarps == 8 ? 12 : 8;  // 16 warps need more, smaller tasks to balance
  const uint32_t kRowF = 2 * kRow, coax_f = uint32_t(sp.rot_floats);
  struct RotT {
    TranslateRotTask d;
    int cost;
  };
  struct CoaxT {
    TranslateCoaxTask d;
    int cost;
  };
  std::vector<RotT> rot;
  std::vector<CoaxT> coax;
  // rows of a sub-block are cut into tiles that start at multiples of 4 (aligned 16-byte
  // coefficient loads) and hold <= 12 rows; the split minimising sum(2R + 6) (instructions per
  // input step) is found by exhaustive search
  auto cut = [max_rows](int w, int parts[4]) {
    int best_cost = 1 << 30, best_n = 0;
    for (int a = 0; a <= max_rows; a += 4)
      for (int b = 0; b <= max_rows; b += 4)
        for (int c = 0; c <= max_rows; c += 4) {
          const int last = w - a - b - c;
          if (last < 1 || last > max_rows) continue;
          if ((a == 0 && (b || c)) || (b == 0 && c)) continue;
          int cand[4] = {a, b, c, last}, tmp[4], np = 0, cost = 0;
          for (int v : cand)
            if (v) {
              tmp[np++] = v;
              cost += 2 * v + 6;
            }
          if (cost < best_cost) {
            best_cost = cost;
            best_n = np;
            for (int i = 0; i < np; ++i) parts[i] = tmp[i];
          }
        }
    return best_n;
  };
  for (int n = 0; n <= P; ++n)
    for (int part = 0; part < 2; ++part) {  // 0: plus system (n+1 rows), 1: minus system (n rows)
      const int w = part ? n : n + 1;
      if (w == 0) continue;
      const int ws = part ? rot_minus_stride(n) : rot_plus_stride(n);
      const int base = part ? n * n + n + 1 : n * n;
      const int table = part ? rot_minus_offset(n) : rot_block_offset(n);
      int parts[4], r0 = 0;
      const int np = cut(w, parts);
      for (int i = 0; i < np; ++i) {
        const int R = parts[i];
        TranslateRotTask d;
        d.e_off = 4u * uint32_t(table + r0);
        d.in_rel = 4u * uint32_t(base) * kRowF;
        d.out_rel = 4u * uint32_t(base + r0) * kRowF;
        d.packed = 4u * uint32_t(ws) | uint32_t(w) << 8 | uint32_t(R) << 16 | uint32_t(r0 & 1) << 24;
        rot.push_back({d, w * (2 * R + 6) + 40});
        r0 += R;
      }
    }
  for (int m = 0; m <= P; ++m) {
    const int w = P + 1 - m;
    // tiles of <= 4 rows (measured: 8-row tiles balance worse over the 8 warps and are slower)
    for (int r0 = 0; r0 < w;) {
      const int R = std::min(4, w - r0);
      TranslateCoaxTask d;
      d.c_off = 4u * (coax_f + 2u * uint32_t(coax_block_offset(P, m) + r0));
      d.p_rel = 4u * uint32_t(m * m + m) * kRowF;
      d.q_rel = 4u * uint32_t(m * m + 2 * m) * kRowF;
      d.packed = 4u * uint32_t(2 * coax_row_stride(P, m)) | uint32_t(w) << 8 | uint32_t(m) << 16 |
                 uint32_t(r0) << 22 | uint32_t(R) << 28;  // R <= 8 fits bits 28..31
      coax.push_back({d, w * ((m ? 8 : 4) * R + 8) + 40});
      r0 += R;
    }
  }
  if (rot.size() > size_t(kTranslateMaxTasks) || coax.size() > size_t(kTranslateMaxTasks))
    throw Error(HFMM_ERR_INTERNAL, "translation schedule overflow");
  auto distribute = [kWarps](auto& tasks, auto* flat, int* begin) {
    std::stable_sort(tasks.begin(), tasks.end(), [](const auto& x, const auto& y) { return x.cost > y.cost; });
    std::vector<std::vector<int>> per(kWarps);
    std::vector<long> load(kWarps, 0);
    for (size_t i = 0; i < tasks.size(); ++i) {
      int best = 0;
      for (int w = 1; w < kWarps; ++w)
        if (load[w] < load[best]) best = w;
      per[best].push_back(int(i));
      load[best] += tasks[i].cost;
    }
    int pos = 0;
    for (int w = 0; w < kWarps; ++w) {
      begin[w] = pos;
      for (int i : per[w]) flat[pos++] = tasks[i].d;
    }
    for (int w = kWarps; w <= kTranslateWarps; ++w) begin[w] = pos;
  };
  *out = TranslateSchedule{};
  distribute(rot, out->rot, out->rot_begin);
  distribute(coax, out->coax, out->coax_begin);
}

void upload_translate_schedule(int order) {
  TranslateSchedule sched;
  build_translate_schedule(order, &sched);
  HFMM_CUDA_CHECK(cudaMemcpyToSymbol(c_sched, &sched, sizeof(sched), sizeof(sched) * size_t(order)));
}

int translate_batch_size(int) { return kTranslateBatch; }

namespace {
template <int NU, int WARPS, int CTAS>
void launch_translate_nu(const TranslateArgs& a, cudaStream_t s, size_t bytes, int ctas) {
  static int configured_for = -1;
  if (configured_for < int(bytes)) {
    HFMM_CUDA_CHECK(cudaFuncSetAttribute(translate_kernel<NU, WARPS, CTAS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    configured_for = int(bytes);
  }
  translate_kernel<NU, WARPS, CTAS><<<ctas, WARPS * 32, bytes, s>>>(a);
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
  // persistent grid: two 8-warp CTAs per SM, or one 16-warp CTA when the tiles are too large
  const int warps = translate_warps(a.order);
  const bool two = translate_two_ctas(a.order);
  const int ctas = int(std::min<uint32_t>(a.n_items, uint32_t((two ? 2 : 1) * sm_count)));
  const int units = (a.order + 1) * (a.order + 2) / 2;
  if (warps == 8) {
    const int nu = (units + 7) / 8;
    if (nu <= 6) launch_translate_nu<6, 8, 2>(a, s, sp.bytes, ctas);         // P <= 8
    else if (nu <= 9) launch_translate_nu<9, 8, 2>(a, s, sp.bytes, ctas);    // P <= 10
    else launch_translate_nu<12, 8, 2>(a, s, sp.bytes, ctas);                // P <= 12
  } else if (two) {
    launch_translate_nu<6, 16, 2>(a, s, sp.bytes, ctas);                     // P <= 12, 64 registers
  } else {
    const int nu = (units + 15) / 16;
    if (nu <= 8) launch_translate_nu<8, 16, 1>(a, s, sp.bytes, ctas);        // P <= 14
    else launch_translate_nu<10, 16, 1>(a, s, sp.bytes, ctas);               // P <= 16
  }
}

}  // namespace hfmm_b200
