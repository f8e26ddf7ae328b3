// kernels_translate64.cu — batched M2M / M2L / L2L, 64 cell pairs per batch, in place (sm_100a).
//
// Same operator as kernels_translate.cu (reference: dense translate, src/expansion.cpp:126-139, of a
// Gaunt-built matrix, src/expansion.cpp:95-124), factored as
//     out += e^{-i mu phi} · E^T · Chat(k|t|) · E · e^{i m phi} · in          (tables.hpp)
// and the same tables; what changes is the work layout, chosen to spend fewer shared-memory
// wavefronts and fewer non-arithmetic instructions per multiply-add:
//   * a batch is 64 pairs of one table group; a LANE OWNS TWO PAIRS and ALL 32 LANES OF A WARP RUN
//     THE SAME TASK, so every coefficient load is warp-uniform and nothing is padded to a partner's shape;
//   * a task is a WHOLE block — the plus or minus system of one degree n in the rotations, one
//     column (s_m or t_m) of one order m in the coaxial step — so it reads every operand row once,
//     keeps all its output rows in registers (<= P+1 rows x 2 pairs) and writes them back IN PLACE:
//     one operand tile instead of a ping-pong pair, which is what lets a 64-pair batch fit twice per SM
//     (P <= 12) or once (P = 13..16, sixteen warps: the largest systems are then split over two warps by
//     pair halves — columns are independent, so the split stays in place);
//   * the tile is [coefficient row][pair] with a pitch of 65 complex (520 bytes) and a lane owns the
//     pairs l and l + 32: the compute stages (two 8-byte accesses per row, 32 lanes contiguous) and the
//     transposing gather / scatter (lane = row: consecutive rows are two banks apart) are both
//     bank-conflict free, and a task addresses its rows as base register + immediate;
//   * folded layout of degree n: s_m (and x_0) at row n^2 + n + m, t_m at row n^2 + n - m — the rows of
//     the raw coefficients (n, +-m), so folding is in place per unit;
//   * the signs of the inverse rotation ((-1)^m on its inputs, (-1)^mu on its outputs, tables.hpp) are not
//     applied by the kernel: the engine folds (-1)^m into the coaxial tables it builds for this kernel
//     (coax_tables_sign_folded), and (-1)^mu is a constant of the unfold — forward and inverse rotation
//     are the same code;
//   * a warp gathers, and later scatters, the same pairs of the batch, pair by pair (scatter of pair p of
//     batch i, then the gather of pair p of batch i + 1 into the column just read): no CTA barrier
//     separates the two, and with the order a template parameter both are straight-line code;
//   * everything the end of a batch needs from global memory is fetched while the batch computes:
//     source / destination rows and azimuths of the next batch arrive through 4-byte cp.async into a
//     double-buffered metadata block, the next table group through 16-byte cp.async, and the source rows
//     are prefetched into L2.
// Six barriers per batch: gather | fold | forward rotation | coaxial translation | inverse rotation |
// unfold | (scatter + next gather).  Tasks are handed to the warps by a host-side
// longest-processing-time schedule in __constant__ memory.
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
// Register caps (measured, profiles/r02_notes.md).  Eight warps, two CTAs per SM: ptxas takes 120 registers when
// left alone; 96 (no spills) is the fastest cap tried between 80 and 128 (11.34 ms against 11.53 at 112, cfg 2).
// Sixteen warps, one CTA per SM (P = 13..16): the kernel alone is fastest at 128 (567.7 ms at cfg 4), but at 80
// (no spills, 573.8 ms) three near-field CTAs find registers and shared memory beside it and the STEP drops from
// 619 to 595 ms.
constexpr int kMaxReg8 = 96, kMaxReg16 = 80;
constexpr int kTranslate64SplitFrom = 11;  // sixteen warps: systems of this many rows or more are cut by pair halves
constexpr uint32_t kPitchB = 520;  // bytes per tile row: 64 pairs x float2 + 8 (rows two banks apart)

struct Plan64 {
  int dim, n_fold, n_units, rot_floats, coax_c;
  uint32_t off_coax, off_phase, off_tile, off_unit, off_unit_s, off_meta;
  size_t bytes;
};
// metadata of one batch: source row, destination row, class, (cos phi, sin phi) per pair
constexpr uint32_t kMetaSrc = 0, kMetaDst = 256, kMetaCls = 512, kMetaCs = 768, kMetaBytes = 1280;
__host__ __device__ constexpr Plan64 plan64(int P) {
  Plan64 s{};
  s.dim = (P + 1) * (P + 1);
  s.n_fold = P * (P + 1) / 2;  // units (n, m >= 1)
  s.n_units = (P + 1) * (P + 2) / 2;  // units (n, m >= 0)
  s.rot_floats = rot_table_size(P);
  s.coax_c = coax_table_size(P);
  s.off_coax = 4u * uint32_t(s.rot_floats);
  s.off_phase = s.off_coax + 8u * uint32_t(s.coax_c);                      // e^{i m phi}: [m][pair], tile pitch
  s.off_tile = (s.off_phase + kPitchB * uint32_t(P + 1) + 15u) & ~15u;
  s.off_unit = (s.off_tile + kPitchB * uint32_t(s.dim) + 15u) & ~15u;
  s.off_unit_s = (s.off_unit + 4u * uint32_t(s.n_fold) + 15u) & ~15u;
  s.off_meta = (s.off_unit_s + 4u * uint32_t(s.n_units) + 15u) & ~15u;
  s.bytes = size_t(s.off_meta) + 2 * kMetaBytes;
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
__device__ __forceinline__ u64 neg2(u64 v) { return v ^ 0x8000000080000000ull; }
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
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts1(uint32_t addr, u64 v) {
  asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// the lane's pairs of a row: PAIRS = 2 -> (l, l + 32), 8 bytes at row * pitch + 8 l and 256 bytes further
template <int PAIRS>
__device__ __forceinline__ void ld_duo(uint32_t addr, u64& a, u64& b) {
  a = lds1(addr);
  if (PAIRS == 2) b = lds1(addr + 256u);
}
template <int PAIRS>
__device__ __forceinline__ void st_duo(uint32_t addr, u64 a, u64 b) {
  sts1(addr, a);
  if (PAIRS == 2) sts1(addr + 256u, b);
}

// ---- rotation task: one folded system of one degree, w inputs -> w outputs, in place -------------
// out[r] = sum_k E[k][r] in[k]; forward and inverse rotation alike (the signs of the inverse live in the
// coaxial tables and in the unfold).  Rows are row0 + step * index.
// `base`: byte address of the lane's first pair in row0; rows advance by stepb bytes (+- pitch).
// The loops stay rolled: fully unrolled per size the kernel was 120 KB of SASS and a fifth of the issue
// slots went to instruction-cache misses.
template <int R, int PAIRS>
__device__ __forceinline__ void rot_task64(uint32_t e_addr, uint32_t ws_b, int w, uint32_t base, int stepb) {
  u64 acc0[R], acc1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc0[r] = acc1[r] = 0ull;
  constexpr int NV = (R + 3) / 4;
  uint32_t in_addr = base;
#pragma unroll 1
  for (int k = 0; k < w; ++k) {
    u64 x0, x1 = 0ull;
    ld_duo<PAIRS>(in_addr, x0, x1);
    float e[NV * 4];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 c = lds4(e_addr + 16 * v);
      e[4 * v] = c.x; e[4 * v + 1] = c.y; e[4 * v + 2] = c.z; e[4 * v + 3] = c.w;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(acc0[r], x0, e[r]);
      if (PAIRS == 2) fma2s(acc1[r], x1, e[r]);
    }
    in_addr += stepb;
    e_addr += ws_b;
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (r < w) st_duo<PAIRS>(base + r * stepb, acc0[r], acc1[r]);
}

// RMIN..RMAX: the widths this call site can meet (split schedules send w >= kSplitFrom to the one-pair
// tasks and everything below to the two-pair tasks): the other bodies are not instantiated
template <int PAIRS, int RMIN, int RMAX>
__device__ __forceinline__ void rot_dispatch64(int w, uint32_t e_addr, uint32_t ws_b, uint32_t base, int stepb) {
#define HFMM_ROT_CASE(R_)                                                 \
  case R_:                                                                \
    if constexpr (R_ >= RMIN && R_ <= RMAX) rot_task64<R_, PAIRS>(e_addr, ws_b, w, base, stepb); \
    break;
  switch (w) {
    case 1: case 2: case 3: case 4:
      if constexpr (RMIN <= 4) rot_task64<4, PAIRS>(e_addr, ws_b, w, base, stepb);
      break;
    HFMM_ROT_CASE(5) HFMM_ROT_CASE(6) HFMM_ROT_CASE(7) HFMM_ROT_CASE(8) HFMM_ROT_CASE(9) HFMM_ROT_CASE(10)
    HFMM_ROT_CASE(11) HFMM_ROT_CASE(12) HFMM_ROT_CASE(13) HFMM_ROT_CASE(14) HFMM_ROT_CASE(15) HFMM_ROT_CASE(16)
    HFMM_ROT_CASE(17)
    default: break;
  }
#undef HFMM_ROT_CASE
}

// ---- coaxial task: one folded column of one order m, degrees n = m .. P -> nu = m .. P, in place ---
// rows: n^2 + n + sgn m, advancing by 2n + 2 per degree
// `base`: byte address of the lane's first pair in the row of degree n = m; the row of degree n + 1 is
// stepb bytes further, stepb growing by 2 pitches per degree
template <int R, int PAIRS>
__device__ __forceinline__ void coax_task64(uint32_t c_addr, uint32_t ws_b, int w, uint32_t base, int stepb) {
  u64 p0[R], p1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) p0[r] = p1[r] = 0ull;
  constexpr int NV = (R + 1) / 2;
  uint32_t in_addr = base;
  int step = stepb;
#pragma unroll 1
  for (int k = 0; k < w; ++k) {
    u64 x0, x1 = 0ull;
    ld_duo<PAIRS>(in_addr, x0, x1);
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
      if (PAIRS == 2) fma2s(p1[r], x1, cr[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(p0[r], t0, ci[r]);
      if (PAIRS == 2) fma2s(p1[r], t1, ci[r]);
    }
    in_addr += step;
    step += 2 * int(kPitchB);
    c_addr += ws_b;
  }
  uint32_t out_addr = base;
  step = stepb;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r < w) st_duo<PAIRS>(out_addr, p0[r], p1[r]);
    out_addr += step;
    step += 2 * int(kPitchB);
  }
}

template <int PAIRS, int RMIN, int RMAX>
__device__ __forceinline__ void coax_dispatch64(int w, uint32_t c_addr, uint32_t ws_b, uint32_t base, int stepb) {
#define HFMM_COAX_CASE(R_)                                                  \
  case R_:                                                                  \
    if constexpr (R_ >= RMIN && R_ <= RMAX) coax_task64<R_, PAIRS>(c_addr, ws_b, w, base, stepb); \
    break;
  switch (w) {
    case 1: case 2:
      if constexpr (RMIN <= 2) coax_task64<2, PAIRS>(c_addr, ws_b, w, base, stepb);
      break;
    case 3: case 4:
      if constexpr (RMIN <= 4) coax_task64<4, PAIRS>(c_addr, ws_b, w, base, stepb);
      break;
    HFMM_COAX_CASE(5) HFMM_COAX_CASE(6) HFMM_COAX_CASE(7) HFMM_COAX_CASE(8) HFMM_COAX_CASE(9) HFMM_COAX_CASE(10)
    HFMM_COAX_CASE(11) HFMM_COAX_CASE(12) HFMM_COAX_CASE(13) HFMM_COAX_CASE(14) HFMM_COAX_CASE(15) HFMM_COAX_CASE(16)
    HFMM_COAX_CASE(17)
    default: break;
  }
#undef HFMM_COAX_CASE
}

__constant__ Translate64Schedule c_sched64[kTranslate64TopOrder + 1];

// one (n, m >= 1) unit of the lane's two pairs: fold, in place
//   a = x_m e^{i m phi},  b = (-1)^m x_{-m} e^{-i m phi}:   s_m = a + b -> row (n, +m),  t_m = a - b -> row (n, -m)
struct FoldUnit {
  u64 xp0, xp1, xm0, xm1, ph0, ph1;
  uint32_t ap, am;
  float sg;
};
// e^{i m phi} of the lane's two pairs, kept across the units of one order (the unit list is m-major)
struct UnitPhase {
  u64 ph0 = 0ull, ph1 = 0ull;
  uint32_t m = 0;
};
__device__ __forceinline__ void unit_load(FoldUnit& f, uint32_t un, uint32_t duo, uint32_t ph_duo, UnitPhase& ph) {
  const uint32_t m = un >> 20;
  f.ap = duo + (un & 0xfffffu);
  f.am = f.ap - m * (2u * kPitchB);
  f.xp0 = lds1(f.ap);
  f.xp1 = lds1(f.ap + 256u);
  f.xm0 = lds1(f.am);
  f.xm1 = lds1(f.am + 256u);
  if (m != ph.m) {  // warp-uniform
    ph.ph0 = lds1(ph_duo + m * kPitchB);
    ph.ph1 = lds1(ph_duo + m * kPitchB + 256u);
    ph.m = m;
  }
  f.ph0 = ph.ph0;
  f.ph1 = ph.ph1;
  f.sg = (m & 1) ? -1.0f : 1.0f;
}
__device__ __forceinline__ void fold_finish(const FoldUnit& f) {
  const float2 f0 = unpack2(f.ph0), f1 = unpack2(f.ph1);
  u64 a0 = mul2s(f.xp0, f0.x), a1 = mul2s(f.xp1, f1.x), b0 = mul2s(f.xm0, f.sg * f0.x), b1 = mul2s(f.xm1, f.sg * f1.x);
  fma2s(a0, rot90(f.xp0), f0.y);
  fma2s(a1, rot90(f.xp1), f1.y);
  fma2s(b0, rot90(f.xm0), -f.sg * f0.y);
  fma2s(b1, rot90(f.xm1), -f.sg * f1.y);
  sts1(f.ap, add2(a0, b0));
  sts1(f.ap + 256u, add2(a1, b1));
  sts1(f.am, add2(a0, neg2(b0)));
  sts1(f.am + 256u, add2(a1, neg2(b1)));
}
// unfold of the inverse rotation's outputs u' (row (n, +m)), v' (row (n, -m)), which still lack the
// (-1)^mu of the symmetry:  y_m = (-1)^m (u' + v')/2 e^{-i m phi},   y_{-m} = (u' - v')/2 e^{+i m phi}
__device__ __forceinline__ void unfold_finish(const FoldUnit& f) {
  const float hs = 0.5f * f.sg;
  const float2 f0 = unpack2(f.ph0), f1 = unpack2(f.ph1);
  const u64 s0 = add2(f.xp0, f.xm0), s1 = add2(f.xp1, f.xm1);
  const u64 d0 = add2(f.xp0, neg2(f.xm0)), d1 = add2(f.xp1, neg2(f.xm1));
  u64 yp0 = mul2s(s0, hs * f0.x), yp1 = mul2s(s1, hs * f1.x), ym0 = mul2s(d0, 0.5f * f0.x), ym1 = mul2s(d1, 0.5f * f1.x);
  fma2s(yp0, rot90(s0), -hs * f0.y);
  fma2s(yp1, rot90(s1), -hs * f1.y);
  fma2s(ym0, rot90(d0), 0.5f * f0.y);
  fma2s(ym1, rot90(d1), 0.5f * f1.y);
  sts1(f.ap, yp0);
  sts1(f.ap + 256u, yp1);
  sts1(f.am, ym0);
  sts1(f.am + 256u, ym1);
}

// PT: the order as a compile-time constant (0: run-time order, any P the launch geometry holds)
// WARPS: 8 (two CTAs per SM, P <= 12) or 16 (one CTA per SM, P <= 16; large systems split by pair halves)
// STAGED: every pair owns its destination row (deterministic mode): plain stores instead of RED
template <int PT, int WARPS, bool STAGED>
__global__ void __launch_bounds__(WARPS * 32) __maxnreg__(WARPS == 8 ? kMaxReg8 : kMaxReg16) translate64_kernel(const TranslateArgs a) {
  constexpr int kThreads = WARPS * 32, kPairsPerWarp = kBatch64 / WARPS;
  constexpr int RMAX = PT ? PT + 1 : (WARPS == 8 ? kTranslate64MaxOrder + 1 : kTranslate64TopOrder + 1);
  constexpr bool kSplit = WARPS == 16;
  extern __shared__ __align__(16) unsigned char smem64[];
  const int P = PT ? PT : a.order;
  const Plan64 sp = plan64(P);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t it_begin = uint32_t(uint64_t(a.n_items) * blockIdx.x / gridDim.x);
  const uint32_t it_end = uint32_t(uint64_t(a.n_items) * (blockIdx.x + 1) / gridDim.x);
  if (it_begin >= it_end) return;

  const uint32_t win = uint32_t(__cvta_generic_to_shared(smem64));
  const uint32_t tile = win + sp.off_tile, ph_base = win + sp.off_phase, duo = tile + 8u * uint32_t(lane);
  const uint32_t unit_base = win + sp.off_unit, unit_s_base = win + sp.off_unit_s, meta_base = win + sp.off_meta;
  // units (n, m >= 1), m-major: byte offset of row (n, +m) | m << 20; the row of (n, -m) is 2 m rows back
  {
    uint32_t* s_unit = reinterpret_cast<uint32_t*>(smem64 + sp.off_unit);
    for (int u = tid; u < sp.n_fold; u += kThreads) {
      int m = 1, first = 0;
      while (first + (P + 1 - m) <= u) {
        first += P + 1 - m;
        ++m;
      }
      const int n = m + (u - first);
      s_unit[u] = uint32_t(n * n + n + m) * kPitchB | uint32_t(m) << 20;
    }
  }
  // all units (n, m >= 0) in coefficient order, for the unfold + scatter: row of (n, +m) | m << 16
  {
    uint32_t* s_unit_s = reinterpret_cast<uint32_t*>(smem64 + sp.off_unit_s);
    for (int u = tid; u < sp.n_units; u += kThreads) {
      int n = int((sqrtf(8.0f * float(u) + 1.0f) - 1.0f) * 0.5f);
      while (n * (n + 1) / 2 > u) --n;
      while ((n + 1) * (n + 2) / 2 <= u) ++n;
      const int m = u - n * (n + 1) / 2;
      s_unit_s[u] = uint32_t(n * n + n + m) | uint32_t(m) << 16;
    }
  }
  // idle pair columns of a partial batch must stay finite: clear the tile once
  for (uint32_t i = tid; i < uint32_t(sp.dim) * (kPitchB / 8); i += kThreads) sts1(tile + 8u * i, 0ull);

  const Translate64Schedule& sched = c_sched64[P];
  auto fetch_tables = [&](uint32_t cls) {
    const TranslateClass c = a.classes[cls];
    const float4* g_rot = reinterpret_cast<const float4*>(a.rot_tables + size_t(c.rot) * sp.rot_floats);
    const float4* g_coax = reinterpret_cast<const float4*>(a.coax_tables + size_t(c.coax) * sp.coax_c * 2);
    for (int i = tid; i < sp.rot_floats / 4; i += kThreads) cp_async16(win + 16u * i, g_rot + i);
    for (int i = tid; i < sp.coax_c / 2; i += kThreads) cp_async16(win + sp.off_coax + 16u * i, g_coax + i);
  };

  // ---- batch metadata, double-buffered: thread p < 64 fetches pair p -------------------------------
  // stage A: source row, destination row, class;  stage B (after A has landed): azimuth of the class
  auto meta_a = [&](const TranslateItem& it, uint32_t mb) {
    if (tid < kBatch64) {
      const uint32_t p = min(uint32_t(tid), it.count - 1u) + it.pair_begin;  // idle columns repeat the last pair
      cp_async4(mb + kMetaSrc + 4u * tid, a.pair_src + p);
      cp_async4(mb + kMetaDst + 4u * tid, a.pair_dst + p);
      cp_async4(mb + kMetaCls + 4u * tid, a.pair_cls + p);
    }
  };
  auto meta_b = [&](uint32_t mb) {
    if (tid < kBatch64) {
      const uint32_t cls = lds32(mb + kMetaCls + 4u * tid);
      cp_async8(mb + kMetaCs + 8u * tid, &a.classes[cls].cphi);
    }
  };
  // e^{i m phi} of the warp's pairs, [m][pair]: lane = (pair, group of four orders)
  auto write_phases = [&](uint32_t mb) {
    constexpr int kGroups = 32 / kPairsPerWarp;                 // 4 (eight pairs per warp) or 8 (four)
    const int pp = lane % kPairsPerWarp, g = lane / kPairsPerWarp;
    const int per = (P + kGroups) / kGroups;                    // orders per group, ceil((P + 1) / groups)
    const float2 c1 = unpack2(lds1(mb + kMetaCs + 8u * uint32_t(warp * kPairsPerWarp + pp)));
    // e^{i (g per) phi} by binary powering
    float cr = 1.f, ci = 0.f, br = c1.x, bi = c1.y;
    for (int e = g * per; e; e >>= 1) {
      if (e & 1) {
        const float t = cr * br - ci * bi;
        ci = ci * br + cr * bi;
        cr = t;
      }
      const float t = br * br - bi * bi;
      bi = 2.f * br * bi;
      br = t;
    }
    uint32_t dst = ph_base + kPitchB * uint32_t(g * per) + 8u * uint32_t(warp * kPairsPerWarp + pp);
    for (int j = 0, m = g * per; j < per && m <= P; ++j, ++m) {
      sts1(dst, pack2(cr, ci));
      dst += kPitchB;
      const float t = cr * c1.x - ci * c1.y;
      ci = ci * c1.x + cr * c1.y;
      cr = t;
    }
  };
  // L2 prefetch of the source rows of the batch described by mb (lane = 128-byte line of a row)
  auto prefetch_rows = [&](uint32_t mb, uint32_t count) {
    const uint32_t row_bytes = 8u * uint32_t(sp.dim);
#pragma unroll 1
    for (int pp = 0; pp < kPairsPerWarp; ++pp) {
      const uint32_t p = uint32_t(warp * kPairsPerWarp + pp);
      if (p >= count) break;
      const uint32_t srow = lds32(mb + kMetaSrc + 4u * p);
      const char* row = reinterpret_cast<const char*>(a.src + size_t(srow) * a.stride);
      const uint32_t off = 128u * uint32_t(lane);
      if (off < row_bytes) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + off));
    }
  };

  // gather of pair column `col` <- source row (cp.async, lane = coefficient: 256 contiguous bytes per
  // instruction; consecutive tile rows are two banks apart); scatter: the same mapping back (RED.64)
  constexpr int kRoundsT = PT ? ((PT + 1) * (PT + 1) + 31) / 32 : 0;
  auto gather_pair = [&](uint32_t col, uint32_t srow) {
    const float2* src = a.src + size_t(srow) * a.stride + lane;
    if constexpr (PT != 0) {
#pragma unroll
      for (int r = 0; r < kRoundsT; ++r)
        if (32 * r + 32 <= (PT + 1) * (PT + 1) || 32 * r + lane < (PT + 1) * (PT + 1))
          cp_async8(col + 32u * r * kPitchB, src + 32 * r);
    } else {
      for (int r = 0; 32 * r + lane < sp.dim; ++r) cp_async8(col + 32u * r * kPitchB, src + 32 * r);
    }
  };
  auto scatter_pair = [&](uint32_t col, uint32_t drow) {
    float2* dst = a.dst + size_t(drow) * a.stride + lane;
    if constexpr (PT != 0) {
      u64 v[kRoundsT];
#pragma unroll
      for (int r = 0; r < kRoundsT; ++r)
        if (32 * r + 32 <= (PT + 1) * (PT + 1) || 32 * r + lane < (PT + 1) * (PT + 1)) v[r] = lds1(col + 32u * r * kPitchB);
#pragma unroll
      for (int r = 0; r < kRoundsT; ++r)
        if (32 * r + 32 <= (PT + 1) * (PT + 1) || 32 * r + lane < (PT + 1) * (PT + 1)) {
          if (STAGED) dst[32 * r] = unpack2(v[r]);
          else atomicAdd(dst + 32 * r, unpack2(v[r]));
        }
    } else {
      for (int r = 0; 32 * r + lane < sp.dim; ++r) {
        const float2 v = unpack2(lds1(col + 32u * r * kPitchB));
        if (STAGED) dst[32 * r] = v;
        else atomicAdd(dst + 32 * r, v);
      }
    }
  };

  // two adjacent columns at once: twice the loads in flight before the first reduction leaves
  auto scatter_two = [&](uint32_t col, uint32_t drow_a, uint32_t drow_b) {
    if constexpr (PT != 0) {
      float2* da = a.dst + size_t(drow_a) * a.stride + lane;
      float2* db = a.dst + size_t(drow_b) * a.stride + lane;
      u64 va[kRoundsT], vb[kRoundsT];
#pragma unroll
      for (int r = 0; r < kRoundsT; ++r)
        if (32 * r + 32 <= (PT + 1) * (PT + 1) || 32 * r + lane < (PT + 1) * (PT + 1)) {
          va[r] = lds1(col + 32u * r * kPitchB);
          vb[r] = lds1(col + 32u * r * kPitchB + 8u);
        }
#pragma unroll
      for (int r = 0; r < kRoundsT; ++r)
        if (32 * r + 32 <= (PT + 1) * (PT + 1) || 32 * r + lane < (PT + 1) * (PT + 1)) {
          if (STAGED) {
            da[32 * r] = unpack2(va[r]);
            db[32 * r] = unpack2(vb[r]);
          } else {
            atomicAdd(da + 32 * r, unpack2(va[r]));
            atomicAdd(db + 32 * r, unpack2(vb[r]));
          }
        }
    } else {
      scatter_pair(col, drow_a);
      scatter_pair(col + 8u, drow_b);
    }
  };

  // unfold + scatter of one pair column, lane = unit (n, m >= 0): the inverse rotation left u' in row (n, +m) and
  // v' in row (n, -m), still without the (-1)^mu of the symmetry;
  //   y_m = (-1)^m (u' + v')/2 e^{-i m phi} -> element n^2 + n + m,   y_{-m} = (u' - v')/2 e^{+i m phi} -> n^2 + n - m
  // go straight from registers to the destination row (RED.64; plain stores in deterministic mode).  Lanes read
  // different rows of one column (two banks apart: conflict free) and the phase column at the tile pitch.
  constexpr int kURoundsT = PT ? ((PT + 1) * (PT + 2) / 2 + 31) / 32 : 0;
  auto unfold_scatter_round = [&](uint32_t col, uint32_t phc, float2* dst, int u) {
    const uint32_t un = lds32(unit_s_base + 4u * uint32_t(u)), rp = un & 0xffffu, m = un >> 16;
    const u64 up = lds1(col + rp * kPitchB), vm = lds1(col + (rp - 2u * m) * kPitchB), ph = lds1(phc + m * kPitchB);
    const float2 f = unpack2(ph);
    const float hs = (m & 1) ? -0.5f : 0.5f;
    const u64 sm = m ? add2(up, vm) : add2(up, up), df = add2(up, neg2(vm));   // m = 0: y_0 = u'
    u64 yp = mul2s(sm, hs * f.x), ym = mul2s(df, 0.5f * f.x);
    fma2s(yp, rot90(sm), -hs * f.y);
    fma2s(ym, rot90(df), 0.5f * f.y);
    if (STAGED) {
      dst[rp] = unpack2(yp);
      if (m) dst[rp - 2u * m] = unpack2(ym);
    } else {
      atomicAdd(dst + rp, unpack2(yp));
      if (m) atomicAdd(dst + (rp - 2u * m), unpack2(ym));
    }
  };
  auto unfold_scatter = [&](uint32_t col, uint32_t phc, uint32_t drow) {
    float2* dst = a.dst + size_t(drow) * a.stride;
    for (int u = lane; u < sp.n_units; u += 32) unfold_scatter_round(col, phc, dst, u);
  };
  // Compile-time order: everything about a lane's unit that does not depend on the pair — tile rows, phase row,
  // destination offsets, the sign — is decoded ONCE per batch into registers (they die with the stage), and a
  // pair then costs three loads at immediate offsets, ten arithmetic instructions and one address add per
  // reduction (45 -> 19 instructions per lane, round and pair).  For m = 0 the row of v' is the row of u' itself,
  // so u' + v' = 2 u' needs no special case; only the second reduction is skipped.
  struct UnfoldRound {
    uint32_t a_up, a_vm, a_ph;  // shared-memory addresses of u', v', e^{i m phi} in the warp's first pair column
    uint32_t d_up, d_vm;        // byte offsets of (n, +m), (n, -m) in a destination row
    float hs;                   // (-1)^m / 2
    bool has_m, valid;
  };
  auto unfold_setup = [&](UnfoldRound (&ur)[kURoundsT ? kURoundsT : 1], uint32_t p0) {
#pragma unroll
    for (int r = 0; r < kURoundsT; ++r) {
      const int u = 32 * r + lane;
      ur[r].valid = 32 * r + 32 <= (PT + 1) * (PT + 2) / 2 || u < (PT + 1) * (PT + 2) / 2;
      const uint32_t un = ur[r].valid ? lds32(unit_s_base + 4u * uint32_t(u)) : 0u, rp = un & 0xffffu, m = un >> 16;
      ur[r].a_up = tile + 8u * p0 + rp * kPitchB;
      ur[r].a_vm = tile + 8u * p0 + (rp - 2u * m) * kPitchB;
      ur[r].a_ph = ph_base + 8u * p0 + m * kPitchB;
      ur[r].d_up = 8u * rp;
      ur[r].d_vm = 8u * (rp - 2u * m);
      ur[r].hs = (m & 1) ? -0.5f : 0.5f;
      ur[r].has_m = m != 0;
    }
  };
  auto unfold_scatter_fast = [&](const UnfoldRound (&ur)[kURoundsT ? kURoundsT : 1], uint32_t pp8, uint32_t drow) {
    char* dst = reinterpret_cast<char*>(a.dst + size_t(drow) * a.stride);
#pragma unroll
    for (int r = 0; r < kURoundsT; ++r) {
      if (32 * r + 32 <= (PT + 1) * (PT + 2) / 2 || ur[r].valid) {
        const u64 up = lds1(ur[r].a_up + pp8), vm = lds1(ur[r].a_vm + pp8), ph = lds1(ur[r].a_ph + pp8);
        const float2 f = unpack2(ph);
        const float hs = ur[r].hs;
        const u64 sm = add2(up, vm), df = add2(up, neg2(vm));
        u64 yp = mul2s(sm, hs * f.x), ym = mul2s(df, 0.5f * f.x);
        fma2s(yp, rot90(sm), -hs * f.y);
        fma2s(ym, rot90(df), 0.5f * f.y);
        float2* dp = reinterpret_cast<float2*>(dst + ur[r].d_up);
        float2* dm = reinterpret_cast<float2*>(dst + ur[r].d_vm);
        if (STAGED) {
          *dp = unpack2(yp);
          if (ur[r].has_m) *dm = unpack2(ym);
        } else {
          atomicAdd(dp, unpack2(yp));
          if (ur[r].has_m) atomicAdd(dm, unpack2(ym));
        }
      }
    }
  };

  // fold, in place, all 64 pairs of a unit per warp step (a lane owns the pairs l and l + 32 as
  // in the compute stages); a warp walks a contiguous chunk of the m-major unit list two units at a time
  const uint32_t ph_duo = ph_base + 8u * uint32_t(lane);
  const int u_begin = sp.n_fold * warp / WARPS, u_end = sp.n_fold * (warp + 1) / WARPS;
  auto fold_or_unfold = [&](auto finish) {
    int u = u_begin;
    UnitPhase ph;
#pragma unroll 1
    for (; u + 1 < u_end; u += 2) {
      FoldUnit fa, fb;
      unit_load(fa, lds32(unit_base + 4u * u), duo, ph_duo, ph);
      unit_load(fb, lds32(unit_base + 4u * u + 4u), duo, ph_duo, ph);
      finish(fa);
      finish(fb);
    }
    if (u < u_end) {
      FoldUnit fa;
      unit_load(fa, lds32(unit_base + 4u * u), duo, ph_duo, ph);
      finish(fa);
    }
  };

  auto run_rot = [&]() {
    for (int t = sched.rot_begin[warp]; t < sched.rot_begin[warp + 1]; ++t) {
      const Translate64Task d = sched.rot[t];
      const uint32_t base = duo + d.row0 * kPitchB;
      if (kSplit && d.half) rot_dispatch64<1, kTranslate64SplitFrom, RMAX>(d.w, win + d.tab_off, d.ws_b, base + 256u * (d.half - 1), d.step * int(kPitchB));
      else rot_dispatch64<2, 1, kSplit ? kTranslate64SplitFrom - 1 : RMAX>(d.w, win + d.tab_off, d.ws_b, base, d.step * int(kPitchB));
    }
  };
  auto run_coax = [&]() {
    for (int t = sched.coax_begin[warp]; t < sched.coax_begin[warp + 1]; ++t) {
      const Translate64Task d = sched.coax[t];
      const uint32_t base = duo + d.row0 * kPitchB;
      if (kSplit && d.half) coax_dispatch64<1, kTranslate64SplitFrom, RMAX>(d.w, win + d.tab_off, d.ws_b, base + 256u * (d.half - 1), d.step * int(kPitchB));
      else coax_dispatch64<2, 1, kSplit ? kTranslate64SplitFrom - 1 : RMAX>(d.w, win + d.tab_off, d.ws_b, base, d.step * int(kPitchB));
    }
  };

  // ---- prologue: tables and metadata of the first batch, its phases and its gather -----------------
  TranslateItem item = a.items[it_begin];
  uint32_t loaded_grp = item.group;
  uint32_t mb_cur = meta_base, mb_next = meta_base + kMetaBytes;
  fetch_tables(item.cls);
  meta_a(item, mb_cur);
  cp_commit();
  asm volatile("cp.async.wait_all;" ::: "memory");
  meta_b(mb_cur);
  cp_commit();
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();  // the unit table, the cleared tile, the metadata
  write_phases(mb_cur);
#pragma unroll 1
  for (int pp = 0; pp < kPairsPerWarp; ++pp) {
    const uint32_t p = uint32_t(warp * kPairsPerWarp + pp);
    if (p < item.count) gather_pair(tile + 8u * p + kPitchB * uint32_t(lane), lds32(mb_cur + kMetaSrc + 4u * p));
  }
  cp_commit();

  for (uint32_t it = it_begin; it < it_end; ++it) {
    const bool has_next = it + 1 < it_end;
    TranslateItem next = item;
    if (has_next) next = a.items[it + 1];
    asm volatile("cp.async.wait_all;" ::: "memory");  // this batch's rows, this group's tables
    __syncthreads();
    if (has_next) meta_a(next, mb_next);
    cp_commit();
    fold_or_unfold([](const FoldUnit& f) { fold_finish(f); });
    __syncthreads();
    run_rot();  // forward rotation, in place
    if (has_next) {
      asm volatile("cp.async.wait_all;" ::: "memory");  // own stage-A copies (long landed)
      meta_b(mb_next);
    }
    cp_commit();
    __syncthreads();
    run_coax();  // coaxial translation, in place
    __syncthreads();
    if (has_next && a.prefetch) prefetch_rows(mb_next, next.count);  // stage A is visible to every warp since the last barrier
    run_rot();  // inverse rotation, in place (same table; signs in the coaxial table and the unfold)
    asm volatile("cp.async.wait_all;" ::: "memory");  // own stage-B copies
    __syncthreads();
    // the tables have had their last reader: fetch the next group's behind the unfold and the scatter
    if (has_next && next.group != loaded_grp) {  // CTA-uniform
      fetch_tables(next.cls);
      loaded_grp = next.group;
    }
    cp_commit();
    // unfold + scatter, then this warp's columns of the next batch: a warp reads and rewrites only its own
    // tile columns and phase columns, so no CTA barrier separates the inverse rotation's barrier from the gather
    {
      uint32_t drow[kPairsPerWarp], srow[kPairsPerWarp];
#pragma unroll
      for (int v = 0; v < kPairsPerWarp / 4; ++v) {
        const float4 d4 = lds4(mb_cur + kMetaDst + 4u * uint32_t(warp * kPairsPerWarp + 4 * v));
        const float4 s4 = lds4(mb_next + kMetaSrc + 4u * uint32_t(warp * kPairsPerWarp + 4 * v));
        drow[4 * v] = __float_as_uint(d4.x); drow[4 * v + 1] = __float_as_uint(d4.y);
        drow[4 * v + 2] = __float_as_uint(d4.z); drow[4 * v + 3] = __float_as_uint(d4.w);
        srow[4 * v] = __float_as_uint(s4.x); srow[4 * v + 1] = __float_as_uint(s4.y);
        srow[4 * v + 2] = __float_as_uint(s4.z); srow[4 * v + 3] = __float_as_uint(s4.w);
      }
      const uint32_t p0 = uint32_t(warp * kPairsPerWarp);
      const uint32_t live = item.count - min(item.count, p0);  // pairs of this warp in the batch
      if constexpr (PT != 0) {
        UnfoldRound ur[kURoundsT];
        unfold_setup(ur, p0);
#pragma unroll
        for (int pp = 0; pp < kPairsPerWarp; ++pp) {
          if (uint32_t(pp) < live) unfold_scatter_fast(ur, 8u * uint32_t(pp), drow[pp]);
          // idle columns of a partial batch re-read the batch's last pair: finite, never scattered
          if (has_next) gather_pair(tile + 8u * (p0 + pp) + kPitchB * uint32_t(lane), srow[pp]);
        }
      } else {
#pragma unroll
        for (int pp = 0; pp < kPairsPerWarp; ++pp) {
          if (uint32_t(pp) < live) unfold_scatter(tile + 8u * (p0 + pp), ph_base + 8u * (p0 + pp), drow[pp]);
          if (has_next) gather_pair(tile + 8u * (p0 + pp) + kPitchB * uint32_t(lane), srow[pp]);
        }
      }
    }
    cp_commit();
    if (has_next) write_phases(mb_next);
    item = next;
    const uint32_t t = mb_cur;
    mb_cur = mb_next;
    mb_next = t;
  }
}

}  // namespace

// host side: one task per folded system of a degree (rotations) / per folded column of an order
// (coaxial step), handed to the warps longest processing time first; with sixteen warps the systems of
// more than kSplitFrom rows are cut into two tasks of 32 pairs each
void build_translate64_schedule(int P, Translate64Schedule* out) {
  const Plan64 sp = plan64(P);
  const int warps = translate64_warps(P);
  constexpr int kSplitFrom = kTranslate64SplitFrom;
  struct T {
    Translate64Task d;
    int cost;
  };
  std::vector<T> rot, coax;
  auto push = [&](std::vector<T>& v, T t) {
    if (warps == 16 && t.d.w >= kSplitFrom) {
      t.cost = t.cost / 2 + 20;
      t.d.half = 1;
      v.push_back(t);
      t.d.half = 2;
      v.push_back(t);
    } else {
      v.push_back(t);
    }
  };
  for (int n = 0; n <= P; ++n) {
    T plus{};
    plus.d.tab_off = 4u * uint32_t(rot_block_offset(n));
    plus.d.ws_b = uint16_t(4 * rot_plus_stride(n));
    plus.d.w = uint8_t(n + 1);
    plus.d.row0 = uint16_t(n * n + n);
    plus.d.step = 1;
    plus.cost = (n + 1) * (2 * std::max(n + 1, 4) + 6) + 2 * (n + 1) + 30;
    push(rot, plus);
    if (n) {
      T minus{};
      minus.d.tab_off = 4u * uint32_t(rot_minus_offset(n));
      minus.d.ws_b = uint16_t(4 * rot_minus_stride(n));
      minus.d.w = uint8_t(n);
      minus.d.row0 = uint16_t(n * n + n - 1);
      minus.d.step = -1;
      minus.cost = n * (2 * std::max(n, 4) + 6) + 2 * n + 30;
      push(rot, minus);
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
      push(coax, t);
    }
  }
  if (rot.size() > size_t(kTranslate64MaxTasks) || coax.size() > size_t(kTranslate64MaxTasks))
    throw Error(HFMM_ERR_INTERNAL, "translation schedule overflow");
  auto distribute = [&](std::vector<T>& tasks, Translate64Task* flat, int* begin) {
    std::stable_sort(tasks.begin(), tasks.end(), [](const T& x, const T& y) { return x.cost > y.cost; });
    std::vector<std::vector<int>> per(warps);
    std::vector<long> load(warps, 0);
    for (size_t i = 0; i < tasks.size(); ++i) {
      int best = 0;
      for (int w = 1; w < warps; ++w)
        if (load[w] < load[best]) best = w;
      per[best].push_back(int(i));
      load[best] += tasks[i].cost;
    }
    int pos = 0;
    for (int w = 0; w < kTranslate64MaxWarps; ++w) {
      begin[w] = pos;
      if (w < warps)
        for (int i : per[w]) flat[pos++] = tasks[i].d;
    }
    begin[kTranslate64MaxWarps] = pos;
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

// eight warps and two CTAs per SM while two operand tiles fit (P <= 12), sixteen warps and one CTA beyond
int translate64_warps(int order) {
  return order <= kTranslate64MaxOrder && 2 * (plan64(order).bytes + 1024) <= size_t(227) * 1024 ? 8 : 16;
}

bool translate64_supported(int order) {
  const char* e = getenv("HFMM_TRANSLATE");
  if ((e && !strcmp(e, "32")) || order > kTranslate64TopOrder) return false;
  if (order > kTranslate64MaxOrder && e && !strcmp(e, "64small")) return false;  // A/B: old kernel beyond P = 12
  return plan64(order).bytes + 1024 <= size_t(227) * 1024;
}

// the engine multiplies block m of the coaxial tables by (-1)^m when this kernel consumes them
bool coax_tables_sign_folded(int order) { return translate64_supported(order); }

namespace {
template <int PT, int WARPS>
void launch64(const TranslateArgs& a, cudaStream_t s, size_t bytes, int ctas) {
  static int configured_for[2] = {-1, -1};
  const int which = a.staged ? 1 : 0;
  if (configured_for[which] < int(bytes)) {
    if (which) HFMM_CUDA_CHECK(cudaFuncSetAttribute(translate64_kernel<PT, WARPS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    else HFMM_CUDA_CHECK(cudaFuncSetAttribute(translate64_kernel<PT, WARPS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    configured_for[which] = int(bytes);
  }
  if (which) translate64_kernel<PT, WARPS, true><<<ctas, WARPS * 32, bytes, s>>>(a);
  else translate64_kernel<PT, WARPS, false><<<ctas, WARPS * 32, bytes, s>>>(a);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
}  // namespace

void launch_translate64(const TranslateArgs& a_in, cudaStream_t s) {
  if (a_in.n_items == 0) return;
  const Plan64 sp = plan64(a_in.order);
  static const int prefetch = [] {
    const char* e = getenv("HFMM_T64_PREFETCH");
    return e ? atoi(e) : 1;
  }();
  TranslateArgs a = a_in;
  a.prefetch = prefetch;
  static int sm_count = 0;
  if (!sm_count) {
    int dev = 0;
    HFMM_CUDA_CHECK(cudaGetDevice(&dev));
    HFMM_CUDA_CHECK(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
  }
  const int warps = translate64_warps(a.order);
  const int ctas = int(std::min<uint32_t>(a.n_items, uint32_t((warps == 8 ? 2 : 1) * sm_count)));

  static const bool generic = [] {
    const char* e = getenv("HFMM_TRANSLATE");
    return e && !strcmp(e, "generic");
  }();
  if (warps == 8) {
    if (!generic && a.order == 12) launch64<12, 8>(a, s, sp.bytes, ctas);
    else if (!generic && a.order == 10) launch64<10, 8>(a, s, sp.bytes, ctas);
    else launch64<0, 8>(a, s, sp.bytes, ctas);
  } else {
    if (!generic && a.order == 14) launch64<14, 16>(a, s, sp.bytes, ctas);
    else launch64<0, 16>(a, s, sp.bytes, ctas);
  }
}

}  // namespace hfmm_b200
