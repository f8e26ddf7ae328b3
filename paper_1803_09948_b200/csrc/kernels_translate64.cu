// kernels_translate64.cu — batched M2M / M2L / L2L, 64 cell pairs per batch, in place (sm_100a).
//
// Same operator as kernels_translate.cu (reference: dense translate, src/expansion.cpp:126-139, of a
// Gaunt-built matrix, src/expansion.cpp:95-124), factored as
//     out += e^{-i mu phi} · E^T · Chat(k|t|) · E · e^{i m phi} · in          (tables.hpp)
// and the same tables; what changes is the work layout, chosen to spend fewer shared-memory
// wavefronts and fewer non-arithmetic instructions per multiply-add (ncu on the 32-pair kernel: the
// shared-memory data pipe at 67 % was the busiest unit, FFMA2 27 % of the instructions):
//   * a batch is 64 pairs of one table group; a LANE OWNS TWO PAIRS and ALL 32 LANES OF A WARP RUN
//     THE SAME TASK, so every coefficient load is warp-uniform (one wavefront per 16 bytes, half of
//     what two half-warp sub-tasks cost) and nothing is padded to a partner's shape;
//   * a task is a WHOLE block — the plus or minus system of one degree n in the rotations, one
//     column (s_m or t_m) of one order m in the coaxial step — so it reads every operand row once,
//     keeps all its output rows in registers (<= P+1 rows x 2 pairs) and writes them back IN PLACE:
//     one operand tile instead of a ping-pong pair, which is what lets a 64-pair batch fit twice per SM;
//   * the +-m fold with e^{i m phi} is fused into the gather (global -> registers -> tile) and the
//     unfold with e^{-i mu phi} into the scatter (tile -> registers -> RED), lane = (n, m) unit of one
//     pair: two passes over the tile and two of six barriers per batch are gone;
//   * the tile is [coefficient row][pair] with a pitch of 65 complex (520 bytes) and a lane owns the
//     pairs l and l + 32: the compute stages (two 8-byte accesses per row, 32 lanes contiguous) and the
//     transposing gather / scatter (lane = row: consecutive rows are two banks apart) are both
//     bank-conflict free, and a task addresses its rows as base register + immediate;
//   * folded layout of degree n: s_m (and x_0) at row n^2 + n + m, t_m at row n^2 + n - m — the rows of
//     the raw coefficients (n, +-m), so folding is in place per unit;
//   * a warp gathers, and later scatters, the same eight pairs of the batch: the scatter of batch i and
//     the gather of batch i + 1 touch only the warp's own tile columns and need no CTA barrier.
// Four barriers per batch: gather+fold | forward rotation | coaxial translation | inverse rotation |
// (unfold+scatter runs into the next gather).  Tasks are handed to the warps by a host-side
// longest-processing-time schedule in __constant__ memory, as before.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "device_utils.cuh"
#include "kernels.cuh"
#include "tables.hpp"

namespace hfmm_b200 {

namespace {

constexpr int kBatch64 = 64;
constexpr uint32_t kPitchB = 520;  // bytes per tile row: 64 pairs x float2 + 8 (rows two banks apart)

struct Plan64 {
  int dim, n_units, rot_floats, coax_c, phase_pitch;
  uint32_t off_coax, off_phase, off_tile, off_unit;
  size_t bytes;
};
__host__ __device__ inline Plan64 plan64(int P) {
  Plan64 s;
  s.dim = (P + 1) * (P + 1);
  s.n_units = (P + 1) * (P + 2) / 2;
  s.rot_floats = rot_table_size(P);
  s.coax_c = coax_table_size(P);
  s.phase_pitch = kBatch64;  // e^{i m phi}: [m][pair]
  s.off_coax = 4u * uint32_t(s.rot_floats);
  s.off_phase = s.off_coax + 8u * uint32_t(s.coax_c);
  s.off_tile = (s.off_phase + 8u * uint32_t((P + 1) * s.phase_pitch) + 15u) & ~15u;
  s.off_unit = (s.off_tile + kPitchB * uint32_t(s.dim) + 15u) & ~15u;
  s.bytes = size_t(s.off_unit) + size_t((4 * s.n_units + 15) & ~15);
  return s;
}

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
__device__ __forceinline__ u64 mul2s(u64 x, float s) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(pack2(s, s)));
  return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 rot90(u64 v) {  // i * v
  const float2 f = unpack2(v);
  return pack2(-f.y, f.x);
}
__device__ __forceinline__ u64 neg2(u64 v) {
  const float2 f = unpack2(v);
  return pack2(-f.x, -f.y);
}
__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ u64 lds1(uint32_t addr) {
  u64 v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts1(uint32_t addr, u64 v) {
  asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}

// the lane's two pairs (l, l + 32) of a row: 8 bytes at row * pitch + 8 l and 256 bytes further
__device__ __forceinline__ void ld_duo(uint32_t addr, u64& a, u64& b) {
  a = lds1(addr);
  b = lds1(addr + 256u);
}
__device__ __forceinline__ void st_duo(uint32_t addr, u64 a, u64 b) {
  sts1(addr, a);
  sts1(addr + 256u, b);
}

// ---- rotation task: one folded system of one degree, w inputs -> w outputs, in place -------------
// out[r] = sum_k E[k][r] in[k]  (inverse rotation: same table, (-1)^k on the inputs and (-1)^r on the
// outputs, tables.hpp).  Rows are row0 + step * index.
// `base`: byte address of the lane's first pair in row0; rows advance by stepb bytes (+- pitch).
// The loops stay rolled (two inputs per trip): fully unrolled per size the kernel was 120 KB of SASS and
// a fifth of the issue slots went to instruction-cache misses.
template <int R, bool BACK>
__device__ __forceinline__ void rot_task64(uint32_t e_addr, uint32_t ws_b, int w, uint32_t base, int stepb) {
  u64 acc0[R], acc1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc0[r] = acc1[r] = 0ull;
  constexpr int NV = (R + 3) / 4;
  uint32_t in_addr = base;
  u64 flip = 0ull;  // inverse rotation: odd inputs enter negated (sign bits toggled on the ALU pipe)
#pragma unroll 1
  for (int k = 0; k < w; ++k) {
    u64 x0, x1;
    ld_duo(in_addr, x0, x1);
    if (BACK) {
      x0 ^= flip;
      x1 ^= flip;
      flip ^= 0x8000000080000000ull;
    }
    float e[NV * 4];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 c = lds4(e_addr + 16 * v);
      e[4 * v] = c.x; e[4 * v + 1] = c.y; e[4 * v + 2] = c.z; e[4 * v + 3] = c.w;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(acc0[r], x0, e[r]);
      fma2s(acc1[r], x1, e[r]);
    }
    in_addr += stepb;
    e_addr += ws_b;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r < w) {
      u64 o0 = acc0[r], o1 = acc1[r];
      if (BACK && (r & 1)) {
        o0 = neg2(o0);
        o1 = neg2(o1);
      }
      st_duo(base + r * stepb, o0, o1);
    }
  }
}

template <bool BACK>
__device__ __forceinline__ void rot_dispatch64(int w, uint32_t e_addr, uint32_t ws_b, uint32_t base, int stepb) {
  switch (w) {
    case 1: case 2: case 3: case 4: rot_task64<4, BACK>(e_addr, ws_b, w, base, stepb); break;
    case 5: rot_task64<5, BACK>(e_addr, ws_b, w, base, stepb); break;
    case 6: rot_task64<6, BACK>(e_addr, ws_b, w, base, stepb); break;
    case 7: rot_task64<7, BACK>(e_addr, ws_b, w, base, stepb); break;
    case 8: rot_task64<8, BACK>(e_addr, ws_b, w, base, stepb); break;
    case 9: rot_task64<9, BACK>(e_addr, ws_b, w, base, stepb); break;
    case 10: rot_task64<10, BACK>(e_addr, ws_b, w, base, stepb); break;
    case 11: rot_task64<11, BACK>(e_addr, ws_b, w, base, stepb); break;
    case 12: rot_task64<12, BACK>(e_addr, ws_b, w, base, stepb); break;
    default: rot_task64<13, BACK>(e_addr, ws_b, w, base, stepb); break;
  }
}

// ---- coaxial task: one folded column of one order m, degrees n = m .. P -> nu = m .. P, in place ---
// rows: n^2 + n + sgn m, advancing by 2n + 2 per degree
// `base`: byte address of the lane's first pair in the row of degree n = m; the row of degree n + 1 is
// stepb bytes further, stepb growing by 2 pitches per degree
template <int R>
__device__ __forceinline__ void coax_task64(uint32_t c_addr, uint32_t ws_b, int w, uint32_t base, int stepb) {
  u64 p0[R], p1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) p0[r] = p1[r] = 0ull;
  constexpr int NV = (R + 1) / 2;
  uint32_t in_addr = base;
  int step = stepb;
#pragma unroll 1
  for (int k = 0; k < w; ++k) {
    u64 x0, x1;
    ld_duo(in_addr, x0, x1);
    const u64 t0 = rot90(x0), t1 = rot90(x1);
    float cr[NV * 2], ci[NV * 2];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 c = lds4(c_addr + 16 * v);
      cr[2 * v] = c.x; ci[2 * v] = c.y; cr[2 * v + 1] = c.z; ci[2 * v + 1] = c.w;
    }
    // c * x = cr * (x.re, x.im) + ci * (-x.im, x.re)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(p0[r], x0, cr[r]);
      fma2s(p1[r], x1, cr[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(p0[r], t0, ci[r]);
      fma2s(p1[r], t1, ci[r]);
    }
    in_addr += step;
    step += 2 * int(kPitchB);
    c_addr += ws_b;
  }
  uint32_t out_addr = base;
  step = stepb;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r < w) st_duo(out_addr, p0[r], p1[r]);
    out_addr += step;
    step += 2 * int(kPitchB);
  }
}

__device__ __forceinline__ void coax_dispatch64(int w, uint32_t c_addr, uint32_t ws_b, uint32_t base, int stepb) {
  switch (w) {
    case 1: case 2: coax_task64<2>(c_addr, ws_b, w, base, stepb); break;
    case 3: case 4: coax_task64<4>(c_addr, ws_b, w, base, stepb); break;
    case 5: coax_task64<5>(c_addr, ws_b, w, base, stepb); break;
    case 6: coax_task64<6>(c_addr, ws_b, w, base, stepb); break;
    case 7: coax_task64<7>(c_addr, ws_b, w, base, stepb); break;
    case 8: coax_task64<8>(c_addr, ws_b, w, base, stepb); break;
    case 9: coax_task64<9>(c_addr, ws_b, w, base, stepb); break;
    case 10: coax_task64<10>(c_addr, ws_b, w, base, stepb); break;
    case 11: coax_task64<11>(c_addr, ws_b, w, base, stepb); break;
    case 12: coax_task64<12>(c_addr, ws_b, w, base, stepb); break;
    default: coax_task64<13>(c_addr, ws_b, w, base, stepb); break;
  }
}

__constant__ Translate64Schedule c_sched64[kTranslate64MaxOrder + 1];

// STAGED: every pair owns its destination row (deterministic mode): plain stores instead of RED
template <bool STAGED>
__global__ void __launch_bounds__(kTranslate64Warps * 32, 2) translate64_kernel(const TranslateArgs a) {
  constexpr int kWarps = kTranslate64Warps, kThreads = kWarps * 32, kPairsPerWarp = kBatch64 / kWarps;
  extern __shared__ __align__(16) unsigned char smem64[];
  const int P = a.order;
  const Plan64 sp = plan64(P);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t it_begin = uint32_t(uint64_t(a.n_items) * blockIdx.x / gridDim.x);
  const uint32_t it_end = uint32_t(uint64_t(a.n_items) * (blockIdx.x + 1) / gridDim.x);
  if (it_begin >= it_end) return;

  const uint32_t win = uint32_t(__cvta_generic_to_shared(smem64));
  const uint32_t tile = win + sp.off_tile, ph_base = win + sp.off_phase, duo = tile + 8u * uint32_t(lane);
  // per unit (n, m >= 0): row of (n, +m) | m << 16; the row of (n, -m) is 2 m rows back
  uint32_t* s_unit = reinterpret_cast<uint32_t*>(smem64 + sp.off_unit);
  for (int u = tid; u < sp.n_units; u += kThreads) {
    int n = int((sqrtf(8.0f * float(u) + 1.0f) - 1.0f) * 0.5f);
    while (n * (n + 1) / 2 > u) --n;
    while ((n + 1) * (n + 2) / 2 <= u) ++n;
    const int m = u - n * (n + 1) / 2;
    s_unit[u] = uint32_t(n * n + n + m) | uint32_t(m) << 16;
  }
  // idle pair columns of a partial batch must stay finite: clear the tile once
  for (uint32_t i = tid; i < uint32_t(sp.dim) * (kPitchB / 8); i += kThreads) sts1(tile + 8u * i, 0ull);

  const Translate64Schedule& sched = c_sched64[P];
  auto fetch_tables = [&](const TranslateClass& cls) {
    const float4* g_rot = reinterpret_cast<const float4*>(a.rot_tables + size_t(cls.rot) * sp.rot_floats);
    const float4* g_coax = reinterpret_cast<const float4*>(a.coax_tables + size_t(cls.coax) * sp.coax_c * 2);
    for (int i = tid; i < sp.rot_floats / 4; i += kThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(win + 16u * i), "l"(g_rot + i) : "memory");
    for (int i = tid; i < sp.coax_c / 2; i += kThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(win + sp.off_coax + 16u * i), "l"(g_coax + i) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // the warp's pairs of a batch: source / destination rows and azimuths; lane l < 8 holds pair 8 warp + l
  const int p_first = warp * kPairsPerWarp;
  uint32_t my_src = 0, my_dst = 0;
  bool my_live = false;
  // e^{i m phi} of every pair of the batch, [m][pair]; each warp fills the columns of its own pairs
  auto load_pairs = [&](const TranslateItem& it) {
    my_live = false;
    if (lane < kPairsPerWarp) {
      const int p = p_first + lane;
      my_live = p < int(it.count);
      float cphi = 1.f, sphi = 0.f;
      if (my_live) {
        my_src = a.pair_src[it.pair_begin + p];
        my_dst = a.pair_dst[it.pair_begin + p];
        const TranslateClass c = a.classes[a.pair_cls[it.pair_begin + p]];
        cphi = c.cphi;
        sphi = c.sphi;
      }
      float cr = 1.f, ci = 0.f;
      uint32_t dst = ph_base + 8u * uint32_t(p);
      for (int m = 0; m <= P; ++m) {
        sts1(dst, pack2(cr, ci));
        dst += 8u * kBatch64;
        const float t = cr * cphi - ci * sphi;
        ci = ci * cphi + cr * sphi;
        cr = t;
      }
    }
  };

  // gather: the raw rows of the warp's pairs are copied straight into their tile columns (cp.async,
  // lane = coefficient: 256 contiguous bytes per instruction; consecutive tile rows are two banks apart)
  constexpr int kRounds = (kTranslate64MaxDim + 31) / 32;  // 32 coefficients of one pair per warp instruction
  auto issue_gather = [&]() {
#pragma unroll 1
    for (int pp = 0; pp < kPairsPerWarp; ++pp) {
      const bool live = __shfl_sync(0xffffffffu, my_live, pp);
      if (!live) continue;  // warp-uniform; the column keeps its (finite) previous contents
      const uint32_t srow = __shfl_sync(0xffffffffu, my_src, pp);
      const float2* src = a.src + size_t(srow) * a.stride + lane;
      const uint32_t dst = tile + 8u * uint32_t(p_first + pp) + kPitchB * uint32_t(lane);
#pragma unroll
      for (int r = 0; r < kRounds; ++r)
        if (32 * r + lane < sp.dim)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 32u * r * kPitchB), "l"(src + 32 * r) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // scatter: the same mapping back, tile column -> destination row (RED.64, 256 contiguous bytes each)
  auto scatter = [&]() {
#pragma unroll 1
    for (int pp = 0; pp < kPairsPerWarp; ++pp) {
      const bool live = __shfl_sync(0xffffffffu, my_live, pp);
      if (!live) continue;
      const uint32_t drow = __shfl_sync(0xffffffffu, my_dst, pp);
      float2* dst = a.dst + size_t(drow) * a.stride + lane;
      const uint32_t src = tile + 8u * uint32_t(p_first + pp) + kPitchB * uint32_t(lane);
#pragma unroll
      for (int r = 0; r < kRounds; ++r)
        if (32 * r + lane < sp.dim) {
          const float2 v = unpack2(lds1(src + 32u * r * kPitchB));
          if (STAGED) dst[32 * r] = v;
          else atomicAdd(dst + 32 * r, v);
        }
    }
  };

  // fold and unfold, in place, all 64 pairs of a unit (n, m >= 0) per warp step (a lane owns the pairs
  // l and l + 32 as in the compute stages; the unit — rows, order, sign — is warp-uniform):
  //   fold    a = x_m e^{i m phi},  b = (-1)^m x_{-m} e^{-i m phi}:   s_m = a + b -> row (n, +m),  t_m = a - b -> row (n, -m)
  //   unfold  y_m = (u + v)/2 e^{-i m phi},   y_{-m} = (-1)^m (u - v)/2 e^{+i m phi}
  const uint32_t ph_duo = ph_base + 8u * uint32_t(lane);
  auto fold = [&]() {
#pragma unroll 1
    for (int u = warp; u < sp.n_units; u += kWarps) {
      const uint32_t un = s_unit[u], rp = un & 0xffffu, m = un >> 16;
      const uint32_t ap = duo + rp * kPitchB, am = ap - 2u * m * kPitchB;
      u64 xp0, xp1;
      ld_duo(ap, xp0, xp1);
      if (m == 0) continue;  // x_0 is its own folded value (e^{i 0} = 1)
      u64 xm0, xm1, ph0, ph1;
      ld_duo(am, xm0, xm1);
      ld_duo(ph_duo + 8u * kBatch64 * m, ph0, ph1);
      const float sg = (m & 1) ? -1.0f : 1.0f;
      const float2 f0 = unpack2(ph0), f1 = unpack2(ph1);
      u64 a0 = mul2s(xp0, f0.x), a1 = mul2s(xp1, f1.x), b0 = mul2s(xm0, sg * f0.x), b1 = mul2s(xm1, sg * f1.x);
      fma2s(a0, rot90(xp0), f0.y);
      fma2s(a1, rot90(xp1), f1.y);
      fma2s(b0, rot90(xm0), -sg * f0.y);
      fma2s(b1, rot90(xm1), -sg * f1.y);
      st_duo(ap, add2(a0, b0), add2(a1, b1));
      st_duo(am, add2(a0, neg2(b0)), add2(a1, neg2(b1)));
    }
  };
  auto unfold = [&]() {
#pragma unroll 1
    for (int u = warp; u < sp.n_units; u += kWarps) {
      const uint32_t un = s_unit[u], rp = un & 0xffffu, m = un >> 16;
      if (m == 0) continue;  // y_0 = u_0
      const uint32_t ap = duo + rp * kPitchB, am = ap - 2u * m * kPitchB;
      u64 u0, u1, v0, v1, ph0, ph1;
      ld_duo(ap, u0, u1);
      ld_duo(am, v0, v1);
      ld_duo(ph_duo + 8u * kBatch64 * m, ph0, ph1);
      const float hs = (m & 1) ? -0.5f : 0.5f;
      const float2 f0 = unpack2(ph0), f1 = unpack2(ph1);
      const u64 s0 = add2(u0, v0), s1 = add2(u1, v1), d0 = add2(u0, neg2(v0)), d1 = add2(u1, neg2(v1));
      u64 yp0 = mul2s(s0, 0.5f * f0.x), yp1 = mul2s(s1, 0.5f * f1.x), ym0 = mul2s(d0, hs * f0.x), ym1 = mul2s(d1, hs * f1.x);
      fma2s(yp0, rot90(s0), -0.5f * f0.y);
      fma2s(yp1, rot90(s1), -0.5f * f1.y);
      fma2s(ym0, rot90(d0), hs * f0.y);
      fma2s(ym1, rot90(d1), hs * f1.y);
      st_duo(ap, yp0, yp1);
      st_duo(am, ym0, ym1);
    }
  };

  TranslateItem item = a.items[it_begin];
  uint32_t loaded_grp = item.group;
  fetch_tables(a.classes[a.pair_cls[item.pair_begin]]);
  __syncthreads();  // s_unit, the cleared tile
  load_pairs(item);
  issue_gather();

  for (uint32_t it = it_begin; it < it_end; ++it) {
    asm volatile("cp.async.wait_all;" ::: "memory");  // this batch's rows, this group's tables
    __syncthreads();
    fold();
    __syncthreads();
    // stage B: forward rotation, in place
    for (int t = sched.rot_begin[warp]; t < sched.rot_begin[warp + 1]; ++t) {
      const Translate64Task d = sched.rot[t];
      rot_dispatch64<false>(d.w, win + d.tab_off, d.ws_b, duo + d.row0 * kPitchB, d.step * int(kPitchB));
    }
    __syncthreads();
    // stage C: coaxial translation, in place
    for (int t = sched.coax_begin[warp]; t < sched.coax_begin[warp + 1]; ++t) {
      const Translate64Task d = sched.coax[t];
      coax_dispatch64(d.w, win + d.tab_off, d.ws_b, duo + d.row0 * kPitchB, d.step * int(kPitchB));
    }
    __syncthreads();
    // stage D: inverse rotation, in place (same table, sign-twiddled)
    for (int t = sched.rot_begin[warp]; t < sched.rot_begin[warp + 1]; ++t) {
      const Translate64Task d = sched.rot[t];
      rot_dispatch64<true>(d.w, win + d.tab_off, d.ws_b, duo + d.row0 * kPitchB, d.step * int(kPitchB));
    }
    __syncthreads();
    // the tables have had their last reader: fetch the next group's behind the unfold and the scatter
    TranslateItem next = item;
    const bool has_next = it + 1 < it_end;
    if (has_next) {
      next = a.items[it + 1];
      if (next.group != loaded_grp) {  // CTA-uniform
        fetch_tables(a.classes[a.pair_cls[next.pair_begin]]);
        loaded_grp = next.group;
      }
    }
    unfold();
    __syncthreads();
    // scatter, then this warp's columns of the next batch: a warp reads and rewrites only its own eight
    // tile columns and phase columns, so no CTA barrier separates the two
    scatter();
    if (has_next) {
      load_pairs(next);
      issue_gather();
    }
    item = next;
  }
}

}  // namespace

// host side: one task per folded system of a degree (rotations) / per folded column of an order
// (coaxial step), handed to the warps longest processing time first
void build_translate64_schedule(int P, Translate64Schedule* out) {
  const Plan64 sp = plan64(P);
  struct T {
    Translate64Task d;
    int cost;
  };
  std::vector<T> rot, coax;
  for (int n = 0; n <= P; ++n) {
    T plus{};
    plus.d.tab_off = 4u * uint32_t(rot_block_offset(n));
    plus.d.ws_b = uint16_t(4 * rot_plus_stride(n));
    plus.d.w = uint8_t(n + 1);
    plus.d.row0 = uint16_t(n * n + n);
    plus.d.step = 1;
    plus.cost = (n + 1) * (2 * (n + 1) + 6) + 2 * (n + 1) + 30;
    rot.push_back(plus);
    if (n) {
      T minus{};
      minus.d.tab_off = 4u * uint32_t(rot_minus_offset(n));
      minus.d.ws_b = uint16_t(4 * rot_minus_stride(n));
      minus.d.w = uint8_t(n);
      minus.d.row0 = uint16_t(n * n + n - 1);
      minus.d.step = -1;
      minus.cost = n * (2 * n + 6) + 2 * n + 30;
      rot.push_back(minus);
    }
  }
  for (int m = 0; m <= P; ++m) {
    const int w = P + 1 - m;
    for (int col = 0; col < (m ? 2 : 1); ++col) {
      T t{};
      t.d.tab_off = sp.off_coax + 8u * uint32_t(coax_block_offset(P, m));
      t.d.ws_b = uint16_t(8 * coax_row_stride(P, m));
      t.d.w = uint8_t(w);
      t.d.row0 = uint16_t(m * m + m + (col ? -m : m));
      t.d.step = int16_t(2 * m + 2);
      t.cost = w * (4 * w + 8) + 2 * w + 30;
      coax.push_back(t);
    }
  }
  if (rot.size() > size_t(kTranslate64MaxTasks) || coax.size() > size_t(kTranslate64MaxTasks))
    throw Error(HFMM_ERR_INTERNAL, "translation schedule overflow");
  auto distribute = [](std::vector<T>& tasks, Translate64Task* flat, int* begin) {
    std::stable_sort(tasks.begin(), tasks.end(), [](const T& x, const T& y) { return x.cost > y.cost; });
    std::vector<std::vector<int>> per(kTranslate64Warps);
    std::vector<long> load(kTranslate64Warps, 0);
    for (size_t i = 0; i < tasks.size(); ++i) {
      int best = 0;
      for (int w = 1; w < kTranslate64Warps; ++w)
        if (load[w] < load[best]) best = w;
      per[best].push_back(int(i));
      load[best] += tasks[i].cost;
    }
    int pos = 0;
    for (int w = 0; w < kTranslate64Warps; ++w) {
      begin[w] = pos;
      for (int i : per[w]) flat[pos++] = tasks[i].d;
    }
    begin[kTranslate64Warps] = pos;
  };
  *out = Translate64Schedule{};
  distribute(rot, out->rot, out->rot_begin);
  distribute(coax, out->coax, out->coax_begin);
}

void upload_translate64_schedule(int order) {
  if (!translate64_supported(order)) return;
  Translate64Schedule sched;
  build_translate64_schedule(order, &sched);
  HFMM_CUDA_CHECK(cudaMemcpyToSymbol(c_sched64, &sched, sizeof(sched), sizeof(sched) * size_t(order)));
}

// the 64-pair kernel holds one operand tile per CTA: two CTAs per SM up to P = 12
bool translate64_supported(int order) {
  const char* e = getenv("HFMM_TRANSLATE");
  if ((e && !strcmp(e, "32")) || order > kTranslate64MaxOrder) return false;
  return 2 * (plan64(order).bytes + 1024) <= size_t(227) * 1024;
}

void launch_translate64(const TranslateArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  const Plan64 sp = plan64(a.order);
  static int sm_count = 0;
  if (!sm_count) {
    int dev = 0;
    HFMM_CUDA_CHECK(cudaGetDevice(&dev));
    HFMM_CUDA_CHECK(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
  }
  static int configured_for[2] = {-1, -1};
  const int which = a.staged ? 1 : 0;
  if (configured_for[which] < int(sp.bytes)) {
    if (which) HFMM_CUDA_CHECK(cudaFuncSetAttribute(translate64_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sp.bytes)));
    else HFMM_CUDA_CHECK(cudaFuncSetAttribute(translate64_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sp.bytes)));
    configured_for[which] = int(sp.bytes);
  }
  const int ctas = int(std::min<uint32_t>(a.n_items, uint32_t(2 * sm_count)));
  if (which) translate64_kernel<true><<<ctas, kTranslate64Warps * 32, sp.bytes, s>>>(a);
  else translate64_kernel<false><<<ctas, kTranslate64Warps * 32, sp.bytes, s>>>(a);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

}  // namespace hfmm_b200
