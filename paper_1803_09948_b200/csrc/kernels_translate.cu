// kernels_translate.cu — batched M2M / M2L / L2L on level-scaled FP32 expansions (sm_100a).
//
// Replaces the reference's dense translate (src/expansion.cpp:126-139) of a Gaunt-built matrix
// (src/expansion.cpp:95-124) by the factored, truncation-identical operator of tables.hpp:
//     out += e^{-i mu phi} · E^T · Chat(k|t|) · E · e^{i m phi} · in
// applied to a BATCH of 32 (source, destination) cell pairs that share the rotation table E (real
// Wigner-d, block diagonal in n) and the coaxial table Chat (diagonal in m): one shift class, or —
// where that fills the batches better — several classes of one table group that differ only in
// azimuth (e^{i m phi} is carried per pair).  Both tables sit in shared memory for the whole group.
//
// What bounds the kernel is the shared-memory data pipe (ncu: l1tex__data_pipe_lsu_wavefronts 67-70 %
// of peak, FMA pipe 37 %): a warp-uniform coefficient LDS.128 costs two wavefronts for 16 bytes.  The
// layout below exists to spend as few wavefronts and instructions per multiply-add as possible.
//
// Work layout of one CTA (8 warps x 2 CTAs per SM up to P = 12, else 16 warps x 1), one batch:
//   * operands live in two element-major shared tiles [coefficient][pair] (ping-pong); a LANE OWNS
//     TWO PAIRS (16 lanes x 2 = 32), so one 16-byte LDS brings both operands and every broadcast
//     coefficient feeds two multiply-adds; the halves of a warp run different sub-tasks;
//   * all arithmetic is packed fma.rn.f32x2 (FFMA2): a complex accumulator is one register pair, a
//     real coefficient the scalar operand, a complex multiply-add two instructions (same FLOP rate
//     as FFMA, half the issue slots);
//   * six barrier-separated stages per batch: gather (cp.async 8-byte copies straight into tile B,
//     issued one batch ahead) | fold with e^{i m phi} (B -> A) | forward rotation (A -> B) |
//     coaxial translation (B -> A) | inverse rotation (A -> B) | unfold (B -> A) + RED.E.ADD.F32x4
//     into the destination rows;
//   * the three arithmetic stages are cut into TASKS = pairs of sub-tasks (a tile of <= 8 rows of one
//     folded rotation block, the plus system of degree n paired with the minus system of degree
//     n + 1: same shape; or a tile of <= 4 rows of one order m of the coaxial step, both folded
//     columns at once).  A sub-task keeps its output rows in registers and runs ONE runtime loop
//     over the block's inputs.  Tasks are handed to the warps by a host-side
//     longest-processing-time schedule kept in __constant__ memory (TranslateSchedule); the code is
//     small and loop-structured on purpose — a fully unrolled, order-specialised variant measured
//     3x SLOWER on B200 because its 256 KB of SASS starved the instruction cache
//     (profiles/r01_notes.md);
//   * rotations run on FOLDED vectors (tables.hpp): the +-m symmetry of the Wigner-d blocks halves
//     their multiply-adds; the inverse rotation reuses the same table through
//     d^n_{mu,m'} = (-1)^{mu-m'} d^n_{m',mu};
//   * CTAs are persistent and walk a contiguous range of batches; the next group's tables are
//     fetched with cp.async behind the unfold.
// FP32 work per pair: 2 * 2*sum_n ((n+1)^2 + n^2) + 4*sum_m (P+1-|m|)^2 FMAs (11.75 k at P = 12) against
// 4 (P+1)^4 = 114 k for the reference's dense complex mat-vec.
#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <vector>

#include "device_utils.cuh"
#include "kernels.cuh"
#include "tables.hpp"

namespace hfmm_b200 {

namespace {


constexpr int kZeroC = 4;  // complex zeros a finished half-warp keeps multiplying with (coaxial stage)
constexpr int kRow = 34;  // float2 elements per operand row: 32 pairs + 2 pad (bank spread)

struct SmemPlan {
  int rot_floats, coax_c, phase_c, unfold_c, tile_c, dim;
  size_t bytes;
};
__host__ __device__ inline SmemPlan smem_plan(int P) {
  SmemPlan s;
  s.dim = (P + 1) * (P + 1);
  s.rot_floats = rot_table_size(P);
  s.coax_c = coax_table_size(P);
  s.phase_c = (P + 1) * 32;  // e^{i m phi} of every pair of the batch: [m][pair]
  s.unfold_c = 0;
  s.tile_c = s.dim * kRow;
  // rot | coax | phases | unfold factors | zero row | tile A | tile B | (n, m) of every gather unit (u16)
  s.bytes = size_t(s.rot_floats) * 4 + size_t(s.coax_c + s.phase_c + s.unfold_c + kZeroC + 2 * s.tile_c) * 8 +
            size_t(((P + 1) * (P + 2) / 2 * 6 + 15) & ~15);
  return s;
}

// Shared memory is addressed with 32-bit BYTE addresses in the shared window (explicit
// ld.shared / st.shared), so the loops advance with one integer add per pointer and the loads use
// register + immediate addressing (generic pointers cost an address computation per access).
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
inline int translate_warps(int P) { return translate_two_ctas(P) ? 8 : 16; }

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
// x * s
__device__ __forceinline__ u64 mul2s(u64 x, float s) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(pack2(s, s)));
  return r;
}
__device__ __forceinline__ void ldsp2(uint32_t addr, u64& a, u64& b) {
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}
__device__ __forceinline__ void stsp2(uint32_t addr, u64 a, u64 b) {
  asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b) : "memory");
}
// (re, im) -> i * (re, im) = (-im, re)
__device__ __forceinline__ u64 rot90(u64 v) {
  const float2 f = unpack2(v);
  return pack2(-f.y, f.x);
}
__device__ __forceinline__ u64 neg2(u64 v) {
  const float2 f = unpack2(v);
  return pack2(-f.x, -f.y);
}

// ---- rotation task -----------------------------------------------------------------------------
// A warp runs TWO sub-tasks at once, one per half-warp: R output rows of one folded sub-block each
// (same number of inputs w), out[r] = sum_k E[k][r] * in[k].  A lane owns TWO pairs of the batch
// (16 lanes x 2 = 32 pairs), so one 16-byte LDS brings both operands and every broadcast
// coefficient feeds two FFMA2: the kernel is bound by shared-memory wavefronts (a broadcast
// LDS.128 costs two), and this halves the coefficient traffic per multiply-add.
// All addresses are per lane (they differ between the halves); rows >= nrows are not stored.
template <int R, bool BACK>
__device__ __forceinline__ void rot_task(uint32_t e_addr, uint32_t ws_b, int w, uint32_t in_addr,
                                         uint32_t out_addr, bool odd0, int nrows) {
  u64 acc0[R], acc1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc0[r] = acc1[r] = 0ull;
  constexpr int NV = (R + 3) / 4;
  constexpr uint32_t kRowB = 8 * kRow;  // bytes per operand row
  // two inputs per trip; in the inverse rotation odd inputs enter negated ((-1)^k of the symmetry)
  uint32_t e1_addr = e_addr + ws_b;
  const uint32_t ws2 = 2 * ws_b;
#pragma unroll 1
  for (int trips = w >> 1; trips > 0; --trips) {
    u64 xa0, xa1, xb0, xb1;
    ldsp2(in_addr, xa0, xa1);
    ldsp2(in_addr + kRowB, xb0, xb1);
    if (BACK) {
      xb0 = neg2(xb0);
      xb1 = neg2(xb1);
    }
    float e0[NV * 4], e1[NV * 4];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 a = lds4(e_addr + 16 * v);
      const float4 b = lds4(e1_addr + 16 * v);
      e0[4 * v] = a.x; e0[4 * v + 1] = a.y; e0[4 * v + 2] = a.z; e0[4 * v + 3] = a.w;
      e1[4 * v] = b.x; e1[4 * v + 1] = b.y; e1[4 * v + 2] = b.z; e1[4 * v + 3] = b.w;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(acc0[r], xa0, e0[r]);
      fma2s(acc1[r], xa1, e0[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(acc0[r], xb0, e1[r]);
      fma2s(acc1[r], xb1, e1[r]);
    }
    in_addr += 2 * kRowB;
    e_addr += ws2;
    e1_addr += ws2;
  }
  if (w & 1) {  // one even-indexed input left
    u64 xa0, xa1;
    ldsp2(in_addr, xa0, xa1);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 a = lds4(e_addr + 16 * v);
      const float ev[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 * v + j < R) {
          fma2s(acc0[4 * v + j], xa0, ev[j]);
          fma2s(acc1[4 * v + j], xa1, ev[j]);
        }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    u64 o0 = acc0[r], o1 = acc1[r];
    if (BACK) {  // (-1)^{row} of the symmetry
      const bool neg = ((r & 1) != 0) != odd0;
      if (neg) {
        o0 = neg2(o0);
        o1 = neg2(o1);
      }
    }
    if (r < nrows) stsp2(out_addr + r * kRowB, o0, o1);
  }
}

template <bool BACK>
__device__ __forceinline__ void rot_dispatch(int R, uint32_t e_addr, uint32_t ws_b, int w,
                                             uint32_t in_addr, uint32_t out_addr, bool odd0, int nrows) {
  switch (R) {
    case 1: rot_task<1, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0, nrows); break;
    case 2: rot_task<2, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0, nrows); break;
    case 3: rot_task<3, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0, nrows); break;
    case 4: rot_task<4, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0, nrows); break;
    case 5: rot_task<5, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0, nrows); break;
    case 6: rot_task<6, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0, nrows); break;
    case 7: rot_task<7, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0, nrows); break;
    default: rot_task<8, BACK>(e_addr, ws_b, w, in_addr, out_addr, odd0, nrows); break;
  }
}

// ---- coaxial task: rows nu = m + r0 .. m + r0 + R - 1 of order m, folded columns s_m and t_m ---
// (for m = 0 only the single column x_0).  p_off / q_off: float offsets of the first input rows
// (degree n = m) of the two columns; they advance by 2n+1 and 2n+2 rows per degree.
template <bool TWO>
__device__ __forceinline__ void coax_task(uint32_t c_addr, uint32_t ws_b, int w, int wmax, int m, int r0,
                                          int nrows, uint32_t p_addr, uint32_t q_addr, uint32_t out_base,
                                          uint32_t zero_addr, uint32_t safe_addr) {
  constexpr int R = 4;
  u64 p0[R], p1[R], q0[R], q1[R];  // columns s_m (p) and t_m (q) of the lane's two pairs
#pragma unroll
  for (int r = 0; r < R; ++r) p0[r] = p1[r] = q0[r] = q1[r] = 0ull;
  constexpr uint32_t kRowB = 8 * kRow;
  uint32_t step = uint32_t(2 * m + 1) * kRowB, dstep = 2 * kRowB, qx = kRowB;
#pragma unroll 1
  for (int k = 0; k < wmax; ++k) {
    if (k == w) {  // this half-warp's sub-task is shorter than its partner's: multiply zeros from here on
      c_addr = zero_addr;
      ws_b = 0;
      p_addr = q_addr = safe_addr;
      step = dstep = qx = 0;
    }
    // c * x = cr * (x.re, x.im) + ci * (-x.im, x.re): two FFMA2 per complex multiply-add
    u64 xp0, xp1, xq0 = 0ull, xq1 = 0ull;
    ldsp2(p_addr, xp0, xp1);
    if (TWO) ldsp2(q_addr, xq0, xq1);
    const u64 tp0 = rot90(xp0), tp1 = rot90(xp1);
    u64 tq0 = 0ull, tq1 = 0ull;
    if (TWO) {
      tq0 = rot90(xq0);
      tq1 = rot90(xq1);
    }
    float cr[R], ci[R];
#pragma unroll
    for (int v = 0; v < R / 2; ++v) {
      const float4 c = lds4(c_addr + 16 * v);
      cr[2 * v] = c.x; ci[2 * v] = c.y;
      cr[2 * v + 1] = c.z; ci[2 * v + 1] = c.w;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(p0[r], xp0, cr[r]);
      fma2s(p1[r], xp1, cr[r]);
      if (TWO) {
        fma2s(q0[r], xq0, cr[r]);
        fma2s(q1[r], xq1, cr[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      fma2s(p0[r], tp0, ci[r]);
      fma2s(p1[r], tp1, ci[r]);
      if (TWO) {
        fma2s(q0[r], tq0, ci[r]);
        fma2s(q1[r], tq1, ci[r]);
      }
    }
    p_addr += step;
    q_addr += step + qx;
    step += dstep;
    c_addr += ws_b;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int nu = m + r0 + r;
    if (r < nrows) {
      stsp2(out_base + uint32_t(nu * nu + m) * kRowB, p0[r], p1[r]);
      if (TWO) stsp2(out_base + uint32_t(nu * nu + nu + m) * kRowB, q0[r], q1[r]);
    }
  }
}

// per-order static schedules live in constant memory: a task is four words, read with
// warp-uniform addresses, so handing a task to a warp costs two LDC.64 and no arithmetic
__constant__ TranslateSchedule c_sched[kMaxOrder + 1];

// Persistent CTAs: each walks a contiguous range of work items (items are sorted by class, so the
// tables in shared memory are reloaded only when the class changes).  The gather of the NEXT item
// is issued into registers while the current item drains through its reductions, so the chain
// item -> pair list -> source rows never sits on the critical path.
// MIXED: the batches of this launch mix shift classes of one table group (per-pair azimuth phases);
// otherwise every batch holds one class and the phases are per class (broadcast)
// STAGED: every pair owns its destination row (deterministic mode): plain stores instead of RED
template <int WARPS, int CTAS, bool MIXED, bool STAGED>
__global__ void __launch_bounds__(WARPS * 32, CTAS) translate_kernel(const TranslateArgs a) {
  constexpr int kThreads = WARPS * 32;
  constexpr int kLanesPerPair = WARPS;  // 32 pairs x WARPS lanes = all threads of the CTA
  extern __shared__ __align__(16) float smem[];
  const int P = a.order;
  const SmemPlan sp = smem_plan(P);
  const int dim = sp.dim, n_units = (P + 1) * (P + 2) / 2;
  float* s_rot = smem;
  float2* s_coax = reinterpret_cast<float2*>(s_rot + sp.rot_floats);
  // e^{i m phi_p} for every pair p of the batch, [m][pair]: a batch may mix shift classes that share the
  // rotation and coaxial tables (same polar angle and distance) and differ only in azimuth
  float2* s_ph = s_coax + sp.coax_c;
  float2* s_zero = s_ph + sp.phase_c + sp.unfold_c;
  float2* A = s_zero + kZeroC;
  float2* B = A + sp.tile_c;
  // per gather unit (n, m >= 0): raw index of (n, +m) << 16 | folded row of s_m;  t_m sits n rows
  // further, (n, -m) sits 2m raw entries back
  uint32_t* s_unit = reinterpret_cast<uint32_t*>(B + sp.tile_c);
  unsigned char* s_um = reinterpret_cast<unsigned char*>(s_unit + n_units);  // (n << 4 | m) needs 2 bytes

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t it_begin = uint32_t(uint64_t(a.n_items) * blockIdx.x / gridDim.x);
  const uint32_t it_end = uint32_t(uint64_t(a.n_items) * (blockIdx.x + 1) / gridDim.x);
  if (it_begin >= it_end) return;

  if (tid < kZeroC) s_zero[tid] = make_float2(0.f, 0.f);
  for (int u = tid; u < n_units; u += kThreads) {
    int n = int((sqrtf(8.0f * float(u) + 1.0f) - 1.0f) * 0.5f);
    while (n * (n + 1) / 2 > u) --n;
    while ((n + 1) * (n + 2) / 2 <= u) ++n;
    const int m = u - n * (n + 1) / 2;
    s_unit[u] = uint32_t(n * (n + 1) + m) << 16 | uint32_t(n * n + m);
    s_um[2 * u] = (unsigned char)n;
    s_um[2 * u + 1] = (unsigned char)m;
  }

  // gather mapping: 32/WARPS pairs x WARPS lanes per warp; the lanes of a pair stream its source
  // row (64-byte runs) with asynchronous 8-byte copies straight into tile B, transposed
  // (coefficient-major, raw order): no staging registers, the copies drain under the reductions
  const int gq = lane / kLanesPerPair, ge = lane % kLanesPerPair, gp = warp * (32 / kLanesPerPair) + gq;
  const uint32_t b_gather = uint32_t(__cvta_generic_to_shared(B)) + 8u * uint32_t(ge * kRow + gp);
  auto issue_gather = [&](const TranslateItem& it) {
    uint32_t dst = b_gather;
    if (gp < int(it.count)) {
      const float2* src = a.src + size_t(a.pair_src[it.pair_begin + gp]) * a.stride + ge;
      for (int i = ge; i < dim; i += kLanesPerPair) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
        dst += 8u * kLanesPerPair * kRow;
        src += kLanesPerPair;
      }
    } else {  // a partial batch: the idle columns stay finite
      for (int i = ge; i < dim; i += kLanesPerPair) {
        sts2(dst, make_float2(0.f, 0.f));
        dst += 8u * kLanesPerPair * kRow;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto wait_gather = [&]() { asm volatile("cp.async.wait_all;" ::: "memory"); };

  const TranslateSchedule& sched = c_sched[P];
  // byte addresses inside the shared window
  const uint32_t win = uint32_t(__cvta_generic_to_shared(smem));
  // a lane owns the pairs 2l, 2l+1 (l = lane mod 16) of the batch; the halves of a warp run
  // different sub-tasks
  const int half = lane >> 4;
  constexpr uint32_t kRowB = 8 * kRow;
  const uint32_t a_duo = uint32_t(__cvta_generic_to_shared(A)) + 16 * (lane & 15),
                 b_duo = uint32_t(__cvta_generic_to_shared(B)) + 16 * (lane & 15),
                 zero_addr = uint32_t(__cvta_generic_to_shared(s_zero)),
                 ph_duo = uint32_t(__cvta_generic_to_shared(s_ph)) + (MIXED ? 16 * (lane & 15) : 0);
  constexpr uint32_t kPhaseRowB = MIXED ? 256 : 8;  // [m][pair] or [m]

  TranslateItem item = a.items[it_begin];
  issue_gather(item);
  uint32_t loaded_grp = 0xffffffffu;  // table group (rotation + coaxial table) resident in shared memory

  // Tables of a shift class: asynchronous 16-byte copies, issued as soon as the previous item has
  // left its last table-reading stage, so the fetch hides under its unfold and reductions; the
  // (P + 1) fold / unfold factor quadruples are computed by the first threads behind the unfold.
  auto fetch_tables = [&](const TranslateClass& cls) {
    const float4* g_rot = reinterpret_cast<const float4*>(a.rot_tables + size_t(cls.rot) * sp.rot_floats);
    const float4* g_coax = reinterpret_cast<const float4*>(a.coax_tables + size_t(cls.coax) * sp.coax_c * 2);
    const uint32_t rot_s = uint32_t(__cvta_generic_to_shared(s_rot)), coax_s = uint32_t(__cvta_generic_to_shared(s_coax));
    for (int i = tid; i < sp.rot_floats / 4; i += kThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(rot_s + 16u * i), "l"(g_rot + i) : "memory");
    for (int i = tid; i < sp.coax_c / 2; i += kThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(coax_s + 16u * i), "l"(g_coax + i) : "memory");
  };
  // azimuth phases of the pairs of an item: thread p < 32 walks e^{i m phi} of pair p up the orders
  uint32_t loaded_cls = 0xffffffffu;
  auto store_phases = [&](const TranslateItem& it) {
    if (!MIXED) {  // one class per batch: e^{i m phi} of the class, recomputed when the class changes
      if (it.cls == loaded_cls) return;
      loaded_cls = it.cls;
      if (tid <= P) {
        const TranslateClass c = a.classes[it.cls];
        float cr = 1.f, ci = 0.f;
        for (int j = 0; j < tid; ++j) {
          const float t = cr * c.cphi - ci * c.sphi;
          ci = ci * c.cphi + cr * c.sphi;
          cr = t;
        }
        s_ph[tid] = make_float2(cr, ci);
      }
      return;
    }
    if (tid < 32) {
      float cphi = 1.f, sphi = 0.f;
      if (tid < int(it.count)) {
        const TranslateClass c = a.classes[a.pair_cls[it.pair_begin + tid]];
        cphi = c.cphi;
        sphi = c.sphi;
      }
      float cr = 1.f, ci = 0.f;
      for (int m = 0; m <= P; ++m) {
        s_ph[m * 32 + tid] = make_float2(cr, ci);
        const float t = cr * cphi - ci * sphi;
        ci = ci * cphi + cr * sphi;
        cr = t;
      }
    }
  };
  // (c, s) of the lane's two pairs for order m
  auto load_phase = [&](int m) {
    if (MIXED) return lds4(ph_duo + kPhaseRowB * m);
    float2 p;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(p.x), "=f"(p.y) : "r"(ph_duo + kPhaseRowB * m));
    return make_float4(p.x, p.y, p.x, p.y);
  };
  {
    const TranslateClass cls = a.classes[a.pair_cls[item.pair_begin]];
    fetch_tables(cls);
    store_phases(item);
    loaded_grp = item.group;
  }
  wait_gather();    // the first item's operands and tables
  __syncthreads();  // ... and s_unit

  for (uint32_t it = it_begin; it < it_end; ++it) {
    const int count = int(item.count);

    // stage 1: e^{i m phi} and fold, B (raw) -> A:
    //   a = x_m e^{i m phi},  b = (-1)^m x_{-m} e^{-i m phi}:   s_m = a + b,  t_m = a - b
    // same mapping as the unfold below (lane = two pairs, one unit per half-warp)
    for (int up = warp; 2 * up < n_units; up += WARPS) {
      const int u = min(2 * up + half, n_units - 1);
      const int n = s_um[2 * u], m = s_um[2 * u + 1], fs = s_unit[u] & 0xffff;
      const uint32_t c0 = b_duo + uint32_t(n * n + n) * kRowB;
      u64 xp0, xp1, xm0 = 0ull, xm1 = 0ull;
      ldsp2(c0 + uint32_t(m) * kRowB, xp0, xp1);
      if (m) ldsp2(c0 - uint32_t(m) * kRowB, xm0, xm1);
      const float4 ph = load_phase(m);
      const float sg = (m & 1) ? -1.0f : 1.0f;
      u64 a0 = mul2s(xp0, ph.x), a1 = mul2s(xp1, ph.z), b0 = mul2s(xm0, sg * ph.x), b1 = mul2s(xm1, sg * ph.z);
      fma2s(a0, rot90(xp0), ph.y);
      fma2s(a1, rot90(xp1), ph.w);
      fma2s(b0, rot90(xm0), -sg * ph.y);
      fma2s(b1, rot90(xm1), -sg * ph.w);
      u64 t0 = a0, t1 = a1;
      fma2s(a0, b0, 1.0f);
      fma2s(a1, b1, 1.0f);
      fma2s(t0, b0, -1.0f);
      fma2s(t1, b1, -1.0f);
      stsp2(a_duo + uint32_t(fs) * kRowB, a0, a1);
      if (m) stsp2(a_duo + uint32_t(fs + n) * kRowB, t0, t1);
    }
    __syncthreads();
    // metadata of the next item (consumed in stage 5)
    TranslateItem next = item;
    const bool has_next = it + 1 < it_end;
    if (has_next) next = a.items[it + 1];

    // stage 2: forward rotation A -> B
    for (int t = sched.rot_begin[warp]; t < sched.rot_begin[warp + 1]; ++t) {
      const TranslateRotSub d0 = sched.rot[t].sub[0], d1 = sched.rot[t].sub[1];
      const TranslateRotSub d = half ? d1 : d0;
      rot_dispatch<false>(d0.packed >> 28, win + d.e_off, d.packed & 0xff, (d0.packed >> 8) & 0xff,
                          a_duo + d.in_rel, b_duo + d.out_rel, false, (d.packed >> 16) & 0xff);
    }
    __syncthreads();
    // stage 3: coaxial translation B -> A
    for (int t = sched.coax_begin[warp]; t < sched.coax_begin[warp + 1]; ++t) {
      const TranslateCoaxSub d0 = sched.coax[t].sub[0], d1 = sched.coax[t].sub[1];
      const TranslateCoaxSub d = half ? d1 : d0;
      const int w0 = (d0.packed >> 8) & 0xff, w1 = (d1.packed >> 8) & 0xff, wmax = max(w0, w1);
      const int m = (d.packed >> 16) & 0x3f, r0 = (d.packed >> 22) & 0x3f, nrows = d.packed >> 28;
      if (((d0.packed >> 16) & 0x3f) == 0)  // m = 0 sub-tasks are paired with each other
        coax_task<false>(win + d.c_off, d.packed & 0xff, (d.packed >> 8) & 0xff, wmax, m, r0, nrows,
                         b_duo + d.p_rel, b_duo + d.q_rel, a_duo, zero_addr, b_duo);
      else
        coax_task<true>(win + d.c_off, d.packed & 0xff, (d.packed >> 8) & 0xff, wmax, m, r0, nrows,
                        b_duo + d.p_rel, b_duo + d.q_rel, a_duo, zero_addr, b_duo);
    }
    __syncthreads();
    // stage 4: inverse rotation A -> B (same table, sign-twiddled)
    for (int t = sched.rot_begin[warp]; t < sched.rot_begin[warp + 1]; ++t) {
      const TranslateRotSub d0 = sched.rot[t].sub[0], d1 = sched.rot[t].sub[1];
      const TranslateRotSub d = half ? d1 : d0;
      rot_dispatch<true>(d0.packed >> 28, win + d.e_off, d.packed & 0xff, (d0.packed >> 8) & 0xff,
                         a_duo + d.in_rel, b_duo + d.out_rel, (d.packed >> 24) & 1, (d.packed >> 16) & 0xff);
    }
    __syncthreads();
    // the tables have had their last reader: fetch the next class's behind the unfold
    const bool new_grp = has_next && next.group != loaded_grp;  // CTA-uniform
    if (new_grp) {
      fetch_tables(a.classes[a.pair_cls[next.pair_begin]]);
      loaded_grp = next.group;
    }
    // stage 5a: unfold B -> A in the caller's coefficient order, with e^{-i mu phi}:
    //   y_m = (u + v)/2 e^{-i m phi},   y_{-m} = (-1)^m (u - v)/2 e^{+i m phi}
    // lane = two pairs, one unit (n, m) per half-warp: conflict-free 16-byte accesses, half-warp
    // uniform indices, packed arithmetic
    for (int up = warp; 2 * up < n_units; up += WARPS) {
      const int u = min(2 * up + half, n_units - 1);  // an odd unit count: the last unit is done twice
      const int n = s_um[2 * u], m = s_um[2 * u + 1], fs = s_unit[u] & 0xffff;
      u64 u0, u1, v0 = 0ull, v1 = 0ull;
      ldsp2(b_duo + uint32_t(fs) * kRowB, u0, u1);
      if (m) ldsp2(b_duo + uint32_t(fs + n) * kRowB, v0, v1);
      const float4 ph = load_phase(m);
      const float h = m ? 0.5f : 1.0f, hs = (m & 1) ? -h : h;
      u64 s0 = u0, s1 = u1, d0 = u0, d1 = u1;
      fma2s(s0, v0, 1.0f);
      fma2s(s1, v1, 1.0f);
      fma2s(d0, v0, -1.0f);
      fma2s(d1, v1, -1.0f);
      u64 yp0 = mul2s(s0, h * ph.x), yp1 = mul2s(s1, h * ph.z), ym0 = mul2s(d0, hs * ph.x), ym1 = mul2s(d1, hs * ph.z);
      fma2s(yp0, rot90(s0), -h * ph.y);
      fma2s(yp1, rot90(s1), -h * ph.w);
      fma2s(ym0, rot90(d0), hs * ph.y);
      fma2s(ym1, rot90(d1), hs * ph.w);
      const uint32_t c0 = a_duo + uint32_t(n * n + n) * kRowB;
      stsp2(c0 + uint32_t(m) * kRowB, yp0, yp1);
      stsp2(c0 - uint32_t(m) * kRowB, ym0, ym1);  // m = 0: the same row, the same value
    }
    __syncthreads();

    // stage 5b: start the next item's gather, then accumulate this item into its destinations,
    // two coefficients (16 bytes) per reduction
    if (has_next) issue_gather(next);
    if (has_next) store_phases(next);  // the unfold (last reader of the phases) is behind the barrier above
    // reduction mapping: a warp takes 4 pairs x 8 lanes, laid out so that each half-warp reads 4
    // consecutive coefficient pairs of 4 pairs (rows 2 i2 of tile A are 8 banks apart: conflict-free)
    {
      const int sq = (lane >> 2) & 3, se = (lane & 3) | ((lane >> 4) << 2), pr = 4 * (warp & 7) + sq;
      if (pr < count) {
        float* dst = reinterpret_cast<float*>(a.dst + size_t(a.pair_dst[item.pair_begin + pr]) * a.stride);
        for (int i2 = se + 8 * (warp >> 3); i2 < dim / 2; i2 += WARPS) {
          const float2 lo = A[(2 * i2) * kRow + pr], hi = A[(2 * i2 + 1) * kRow + pr];
          const float4 v = make_float4(lo.x, lo.y, hi.x, hi.y);
          if (STAGED) reinterpret_cast<float4*>(dst)[i2] = v;  // one row per pair: nothing to add to
          else atomicAdd(reinterpret_cast<float4*>(dst) + i2, v);
        }
        if ((dim & 1) && se == 0 && warp < 8) {
          if (STAGED) reinterpret_cast<float2*>(dst)[dim - 1] = A[(dim - 1) * kRow + pr];
          else atomicAdd(reinterpret_cast<float2*>(dst) + (dim - 1), A[(dim - 1) * kRow + pr]);
        }
      }
    }
    // the next item's operands (tile B is free since the unfold) must have landed
    wait_gather();
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
  constexpr int kMaxRows = 8;  // rows of a rotation tile (accumulators: 2 pairs x 8 rows x (re, im))
  const uint32_t kRowB = 8 * kRow, coax_b = 4u * uint32_t(sp.rot_floats);

  // ---- rotations: sub-task = (degree n, plus / minus system, tile of <= 8 rows starting at a
  // multiple of 4).  The plus system of degree n and the minus system of degree n + 1 have the same
  // shape ((n+1) x (n+1)), so their tiles pair up exactly; the plus system of degree P pairs its
  // own tiles.
  struct RotS {
    TranslateRotSub d;
    int w, rows;
  };
  auto rot_subs = [&](int n, int part) {
    std::vector<RotS> v;
    const int w = part ? n : n + 1;
    const int ws = part ? rot_minus_stride(n) : rot_plus_stride(n);
    const int base = part ? n * n + n + 1 : n * n;
    const int table = part ? rot_minus_offset(n) : rot_block_offset(n);
    for (int r0 = 0; r0 < w; r0 += kMaxRows) {
      const int R = std::min(kMaxRows, w - r0);
      RotS s;
      s.d.e_off = 4u * uint32_t(table + r0);
      s.d.in_rel = uint32_t(base) * kRowB;
      s.d.out_rel = uint32_t(base + r0) * kRowB;
      s.d.packed = 4u * uint32_t(ws) | uint32_t(w) << 8 | uint32_t(R) << 16 | uint32_t(r0 & 1) << 24;
      s.w = w;
      s.rows = R;
      v.push_back(s);
    }
    return v;
  };
  struct RotT {
    TranslateRotTask d;
    int cost;
  };
  std::vector<RotT> rot;
  auto add_rot = [&rot](const RotS& x, const RotS* y) {
    RotT t;
    t.d.sub[0] = x.d;
    int R = x.rows;
    if (y) {
      t.d.sub[1] = y->d;
      R = std::max(R, y->rows);
    } else {  // no partner: the second half-warp repeats the sub-task and stores nothing
      t.d.sub[1] = x.d;
      t.d.sub[1].packed &= ~(0xffu << 16);
    }
    t.d.sub[0].packed |= uint32_t(R) << 28;
    t.cost = x.w * (4 * R + 8) + 4 * R + 40;
    rot.push_back(t);
  };
  for (int n = 0; n < P; ++n) {
    const auto plus = rot_subs(n, 0), minus = rot_subs(n + 1, 1);
    for (size_t i = 0; i < plus.size(); ++i) add_rot(plus[i], &minus[i]);
  }
  {
    const auto plus = rot_subs(P, 0);
    for (size_t i = 0; i < plus.size(); i += 2) add_rot(plus[i], i + 1 < plus.size() ? &plus[i + 1] : nullptr);
  }

  // ---- coaxial step: sub-task = (order m, tile of <= 4 rows); tiles of one order pair up, the odd
  // ones out are paired by decreasing length (the shorter half multiplies zeros at the end)
  struct CoaxS {
    TranslateCoaxSub d;
    int w;
  };
  struct CoaxT {
    TranslateCoaxTask d;
    int cost;
  };
  std::vector<CoaxT> coax;
  std::vector<CoaxS> odd;
  auto add_coax = [&coax](const CoaxS& x, const CoaxS* y, bool two) {
    CoaxT t;
    t.d.sub[0] = x.d;
    int w = x.w;
    if (y) {
      t.d.sub[1] = y->d;
      w = std::max(w, y->w);
    } else {
      t.d.sub[1] = x.d;
      t.d.sub[1].packed &= ~(0xfu << 28);
    }
    t.cost = w * ((two ? 32 : 16) + 12) + 60;
    coax.push_back(t);
  };
  for (int m = 0; m <= P; ++m) {
    const int w = P + 1 - m;
    std::vector<CoaxS> tiles;
    for (int r0 = 0; r0 < w; r0 += 4) {
      const int R = std::min(4, w - r0);
      CoaxS s;
      s.d.c_off = coax_b + 8u * uint32_t(coax_block_offset(P, m) + r0);
      s.d.p_rel = uint32_t(m * m + m) * kRowB;
      s.d.q_rel = uint32_t(m * m + 2 * m) * kRowB;
      s.d.packed = 8u * uint32_t(coax_row_stride(P, m)) | uint32_t(w) << 8 | uint32_t(m) << 16 |
                   uint32_t(r0) << 22 | uint32_t(R) << 28;
      s.w = w;
      tiles.push_back(s);
    }
    size_t i = 0;
    for (; i + 1 < tiles.size(); i += 2) add_coax(tiles[i], &tiles[i + 1], m != 0);
    if (i < tiles.size()) {
      if (m == 0) add_coax(tiles[i], nullptr, false);  // x_0 column: single-column code path
      else odd.push_back(tiles[i]);
    }
  }
  std::stable_sort(odd.begin(), odd.end(), [](const CoaxS& x, const CoaxS& y) { return x.w > y.w; });
  for (size_t i = 0; i < odd.size(); i += 2) add_coax(odd[i], i + 1 < odd.size() ? &odd[i + 1] : nullptr, true);

  if (rot.size() > size_t(kTranslateMaxTasks) || coax.size() > size_t(kTranslateMaxTasks))
    throw Error(HFMM_ERR_INTERNAL, "translation schedule overflow");
  for (const auto& t : coax)
    if ((t.d.sub[0].packed & 0xff) != (8u * uint32_t(coax_row_stride(P, (t.d.sub[0].packed >> 16) & 0x3f))))
      throw Error(HFMM_ERR_INTERNAL, "coaxial row stride does not fit its field");
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
  upload_translate64_schedule(order);
  TranslateSchedule sched;
  build_translate_schedule(order, &sched);
  HFMM_CUDA_CHECK(cudaMemcpyToSymbol(c_sched, &sched, sizeof(sched), sizeof(sched) * size_t(order)));
}

int translate_batch_size(int order) { return translate64_supported(order) ? 64 : kTranslateBatch; }

namespace {
template <int WARPS, int CTAS, bool MIXED, bool STAGED>
void launch_translate_nu(const TranslateArgs& a, cudaStream_t s, size_t bytes, int ctas) {
  static int configured_for = -1;
  if (configured_for < int(bytes)) {
    HFMM_CUDA_CHECK(cudaFuncSetAttribute(translate_kernel<WARPS, CTAS, MIXED, STAGED>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    configured_for = int(bytes);
  }
  translate_kernel<WARPS, CTAS, MIXED, STAGED><<<ctas, WARPS * 32, bytes, s>>>(a);
  HFMM_CUDA_CHECK(cudaGetLastError());
}
}  // namespace

void launch_translate(const TranslateArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  if (translate64_supported(a.order)) {
    launch_translate64(a, s);
    return;
  }
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
  auto pick = [&](auto warps_c, auto ctas_c) {
    constexpr int W = decltype(warps_c)::value, C = decltype(ctas_c)::value;
    if (a.mixed) {
      if (a.staged) launch_translate_nu<W, C, true, true>(a, s, sp.bytes, ctas);
      else launch_translate_nu<W, C, true, false>(a, s, sp.bytes, ctas);
    } else {
      if (a.staged) launch_translate_nu<W, C, false, true>(a, s, sp.bytes, ctas);
      else launch_translate_nu<W, C, false, false>(a, s, sp.bytes, ctas);
    }
  };
  if (warps == 8) pick(std::integral_constant<int, 8>{}, std::integral_constant<int, 2>{});
  else pick(std::integral_constant<int, 16>{}, std::integral_constant<int, 1>{});
}

}  // namespace hfmm_b200
