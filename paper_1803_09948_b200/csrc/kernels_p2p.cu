// kernels_p2p.cu — near-field Helmholtz P2P for sm_100a.
//
// Replaces the reference's direct_groups<Real> (src/traversal.cpp:175-204) with green_t
// (include/hfmm/kernel.hpp:16-23):  trg_i += sum_j q_j e^{ikR}/(4 pi R),  R^2 == 0 skipped.
//
// Mapping (one warp per tile of <= 32 target bodies of one leaf):
//   * the 32 LANES hold 32 different SOURCE bodies, taken from the concatenation of all source
//     leaves of the tile's list, so lanes stay full however few bodies a leaf holds
//     (mean 18 per leaf at BASELINE config 2);
//   * every lane keeps one complex accumulator PER TARGET in registers (statically unrolled),
//     target coordinates are broadcast from shared memory, one array per axis;
//   * TWO targets are evaluated per packed instruction (add / mul / fma.rn.f32x2): coordinates,
//     distances and accumulators are (target 2j, target 2j+1) register pairs, only the MUFU
//     evaluations stay scalar.  ncu: the XU (MUFU) pipe is the busiest unit (65 %) — three MUFU per
//     pair (rsqrt, sin, cos) are the floor;
//   * one warp-shuffle reduction per target at the very end.
// Coordinates arrive pre-scaled by k_r and leaf-relative; the lattice offset between the two leaf
// centres is added per source body.  G = (k_r/4pi) e^{iR'}/R' with R' = k_r R, the constant applied
// once at the store; a complex wavenumber adds the amplitude 2^{-damp R'} (one more MUFU, second
// kernel instantiation).  CTAs hold two warps: one such CTA fits beside the two persistent M2L
// CTAs of an SM, which is how the near field hides under M2L (engine.cu, phase_downward).
//
// Two passes per tile (kernels.cuh, P2PArgs):
//   touching leaves (self included): compensated hi/lo coordinates, R == 0 masked — coincident
//     bodies share a key, hence a leaf, so the mask is only ever needed here;
//   all other leaves: plain FP32 coordinates, unmasked, a 1e-30 floor only guards against NaN.
#include "device_utils.cuh"
#include "kernels.cuh"

namespace hfmm_b200 {

namespace {

constexpr int kTile = 32;
constexpr int kWarpsPerBlock = 2;

__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sin_approx(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float cos_approx(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- packed FP32 (sm_100a): add / mul / fma.rn.f32x2 work on a register PAIR per instruction at
// the FP32 rate of two scalar instructions.  The kernel is issue-bound (3 MUFU + ~14 FP32
// instructions per body pair), so TWO targets are evaluated per instruction stream: every
// coordinate, distance and accumulator is a (target 2j, target 2j+1) pair; only the MUFU
// evaluations (rsqrt, sin, cos) stay scalar.
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
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ void lds_2x2(uint32_t addr, u64& a, u64& b) {
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}

// source-side constants of one lane, broadcast to both halves of a pair
struct SourceQ {
  u64 qr, qi, nqi;
};

// polynomial coefficients of the bounded near field, broadcast to both halves of a pair
struct Poly {
  u64 s[kP2PPolyDegree + 1], c[kP2PPolyDegree + 1];
};
__device__ __forceinline__ u64 horner2(const u64 (&c)[kP2PPolyDegree + 1], u64 u) {
  u64 p = c[kP2PPolyDegree];
#pragma unroll
  for (int i = kP2PPolyDegree - 1; i >= 0; --i) p = fma2(p, u, c[i]);
  return p;
}

// acc += (e^{i R'} / R') * q for a pair of targets, R'^2 = r2, rinv = 1/R'.
// MODE 0: cos and sin on the MUFU pipe (any R').  MODE 1, 2: sin(R')/R' = sinc(r2) as a polynomial
// in r2 on the FMA pipe (no 1/R' factor needed), cos on MUFU.  MODE 3: cos as a polynomial too.
// DAMP: complex wavenumber k_r + i k_i, the amplitude decays as e^{-k_i R} = 2^{-damp R'} with
// R' = k_r R (kernel.hpp:20), one more MUFU.  MASKED: r2 == 0 pairs (rinv == 0) contribute nothing.
template <bool DAMP, int MODE, bool MASKED>
__device__ __forceinline__ void green_accumulate2(u64 r2, u64 rinv, const SourceQ& q, float damp, const Poly& pl,
                                                  u64& ar, u64& ai) {
  u64 gr, gi;
  if (MODE == P2P_MODE_MUFU) {
    const float2 r = unpack2(mul2(r2, rinv));
    if (DAMP) rinv = mul2(rinv, pack2(ex2_approx(-damp * r.x), ex2_approx(-damp * r.y)));
    const u64 c = pack2(cos_approx(r.x), cos_approx(r.y)), s = pack2(sin_approx(r.x), sin_approx(r.y));
    gr = mul2(rinv, c);
    gi = mul2(rinv, s);
  } else {
    u64 c;
    float2 r;
    if (MODE != P2P_MODE_ALL_POLY || DAMP) r = unpack2(mul2(r2, rinv));
    if (MODE == P2P_MODE_ALL_POLY) c = horner2(pl.c, r2);
    else c = pack2(cos_approx(r.x), cos_approx(r.y));
    gr = mul2(rinv, c);
    gi = horner2(pl.s, r2);
    if (MASKED) {  // sinc(0) = 1: a coincident pair must not see it
      const float2 g = unpack2(gi), m = unpack2(rinv);
      gi = pack2(m.x != 0.0f ? g.x : 0.0f, m.y != 0.0f ? g.y : 0.0f);
    }
    if (DAMP) {
      const u64 e = pack2(ex2_approx(-damp * r.x), ex2_approx(-damp * r.y));
      gr = mul2(gr, e);
      gi = mul2(gi, e);
    }
  }
  ar = fma2(gr, q.qr, ar);
  ar = fma2(gi, q.nqi, ar);
  ai = fma2(gr, q.qi, ai);
  ai = fma2(gi, q.qr, ai);
}

// Targets are walked in groups of 4 (two pairs): one warp-uniform branch per group, two independent
// packed evaluations in a straight line.  Target coordinates live in shared memory as one array
// per axis, so a 16-byte broadcast load brings the four x (y, z) of a group as two pairs.
constexpr int kGroup = 4;
constexpr int kPairs = kTile / 2;

// plain path: one FP32 coordinate per axis.  nsx = (-sx, -sx) etc.  Slots past n_t inside the last
// group hold zero coordinates; their accumulators are never stored.  NP packed pairs (2 NP targets)
// are evaluated in one straight line: the independent chains hide each other's MUFU / FMA latency
// (ncu: fixed-latency waits were the top stall with two chains per basic block).
template <bool DAMP, int MODE, int NP>
__device__ __forceinline__ void plain_block(uint32_t tx, uint32_t ty, uint32_t tz, int t0, u64 nsx, u64 nsy,
                                            u64 nsz, const SourceQ& q, float damp, const Poly& pl, u64* ar,
                                            u64* ai) {
  const u64 tiny = pack2(1e-30f, 1e-30f);
  constexpr int NL = (NP + 1) / 2 * 2;  // pairs are loaded two at a time (16 bytes per axis)
  u64 x[NL], y[NL], z[NL];
#pragma unroll
  for (int v = 0; v < NL / 2; ++v) {
    lds_2x2(tx + 4 * t0 + 16 * v, x[2 * v], x[2 * v + 1]);
    lds_2x2(ty + 4 * t0 + 16 * v, y[2 * v], y[2 * v + 1]);
    lds_2x2(tz + 4 * t0 + 16 * v, z[2 * v], z[2 * v + 1]);
  }
  u64 r2[NP], rinv[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const u64 dx = add2(x[j], nsx), dy = add2(y[j], nsy), dz = add2(z[j], nsz);
    r2[j] = fma2(dz, dz, fma2(dy, dy, fma2(dx, dx, tiny)));
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const float2 r2s = unpack2(r2[j]);
    rinv[j] = pack2(rsqrt_approx(r2s.x), rsqrt_approx(r2s.y));
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) green_accumulate2<DAMP, MODE, false>(r2[j], rinv[j], q, damp, pl, ar[j], ai[j]);
}

template <bool DAMP, int MODE>
__device__ __forceinline__ void accumulate_plain(uint32_t tx, uint32_t ty, uint32_t tz, uint32_t n_t,
                                                 u64 nsx, u64 nsy, u64 nsz, const SourceQ& q, float damp,
                                                 const Poly& pl, u64 (&ar)[kPairs], u64 (&ai)[kPairs]) {
  // blocks of eight targets; the last block of a tile evaluates only its populated pairs of targets
  // (leaves hold 18 bodies on average: rounding the tail up to four targets cost 6 % of the pairs)
#pragma unroll
  for (int t0 = 0; t0 < kTile; t0 += 2 * kGroup) {
    const int rem = int(n_t) - t0;  // warp-uniform
    if (rem > 6) plain_block<DAMP, MODE, 4>(tx, ty, tz, t0, nsx, nsy, nsz, q, damp, pl, &ar[t0 / 2], &ai[t0 / 2]);
    else if (rem > 4) plain_block<DAMP, MODE, 3>(tx, ty, tz, t0, nsx, nsy, nsz, q, damp, pl, &ar[t0 / 2], &ai[t0 / 2]);
    else if (rem > 2) plain_block<DAMP, MODE, 2>(tx, ty, tz, t0, nsx, nsy, nsz, q, damp, pl, &ar[t0 / 2], &ai[t0 / 2]);
    else if (rem > 0) plain_block<DAMP, MODE, 1>(tx, ty, tz, t0, nsx, nsy, nsz, q, damp, pl, &ar[t0 / 2], &ai[t0 / 2]);
  }
}

// the same with |t - s|^2 expanded: r2 = (|t|^2 + |s|^2) - 2 t.s — four FP32 instructions instead of
// six.  Only for leaves at least one cell apart (no cancellation worth speaking of: |s|^2 / r2 <= ~8
// costs 3 bits of the 24) and bounded R'.  t2: |t|^2 per target; m2s = -2 s; s2 = |s|^2 + tiny.
template <bool DAMP, int MODE>
__device__ __forceinline__ void accumulate_expanded(uint32_t tx, uint32_t ty, uint32_t tz, uint32_t tt,
                                                    uint32_t n_t, u64 m2sx, u64 m2sy, u64 m2sz, u64 s2,
                                                    const SourceQ& q, float damp, const Poly& pl,
                                                    u64 (&ar)[kPairs], u64 (&ai)[kPairs]) {
#pragma unroll
  for (int t0 = 0; t0 < kTile; t0 += kGroup)
    if (t0 < n_t) {  // warp-uniform
      u64 x[2], y[2], z[2], w[2];
      lds_2x2(tx + 4 * t0, x[0], x[1]);
      lds_2x2(ty + 4 * t0, y[0], y[1]);
      lds_2x2(tz + 4 * t0, z[0], z[1]);
      lds_2x2(tt + 4 * t0, w[0], w[1]);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const u64 r2 = fma2(z[j], m2sz, fma2(y[j], m2sy, fma2(x[j], m2sx, add2(w[j], s2))));
        const float2 r2s = unpack2(r2);
        const u64 rinv = pack2(rsqrt_approx(r2s.x), rsqrt_approx(r2s.y));
        green_accumulate2<DAMP, MODE, false>(r2, rinv, q, damp, pl, ar[t0 / 2 + j], ai[t0 / 2 + j]);
      }
    }
}

// compensated path: d = (hi_t - hi_s) + (lo_t - lo_s); the hi difference is exact (grid multiples);
// coincident bodies (R == 0) are masked
template <bool DAMP, int MODE, int NP>
__device__ __forceinline__ void compensated_block(uint32_t thi, uint32_t tlo, int t0, u64 nhx, u64 nhy, u64 nhz,
                                                  u64 nlx, u64 nly, u64 nlz, const SourceQ& q, float damp,
                                                  const Poly& pl, u64* ar, u64* ai) {
  constexpr int NL = (NP + 1) / 2 * 2;
  u64 hx[NL], hy[NL], hz[NL], lx[NL], ly[NL], lz[NL];
#pragma unroll
  for (int v = 0; v < NL / 2; ++v) {
    lds_2x2(thi + 4 * t0 + 16 * v, hx[2 * v], hx[2 * v + 1]);
    lds_2x2(thi + 4 * (kTile + t0) + 16 * v, hy[2 * v], hy[2 * v + 1]);
    lds_2x2(thi + 4 * (2 * kTile + t0) + 16 * v, hz[2 * v], hz[2 * v + 1]);
    lds_2x2(tlo + 4 * t0 + 16 * v, lx[2 * v], lx[2 * v + 1]);
    lds_2x2(tlo + 4 * (kTile + t0) + 16 * v, ly[2 * v], ly[2 * v + 1]);
    lds_2x2(tlo + 4 * (2 * kTile + t0) + 16 * v, lz[2 * v], lz[2 * v + 1]);
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const u64 dx = add2(add2(hx[j], nhx), add2(lx[j], nlx));
    const u64 dy = add2(add2(hy[j], nhy), add2(ly[j], nly));
    const u64 dz = add2(add2(hz[j], nhz), add2(lz[j], nlz));
    const u64 r2 = fma2(dz, dz, fma2(dy, dy, mul2(dx, dx)));
    const float2 r2s = unpack2(r2);
    const u64 rinv = pack2(r2s.x > 0.0f ? rsqrt_approx(r2s.x) : 0.0f, r2s.y > 0.0f ? rsqrt_approx(r2s.y) : 0.0f);
    green_accumulate2<DAMP, MODE, true>(r2, rinv, q, damp, pl, ar[j], ai[j]);
  }
}

template <bool DAMP, int MODE>
__device__ __forceinline__ void accumulate_compensated(uint32_t thi, uint32_t tlo, uint32_t n_t, u64 nhx,
                                                       u64 nhy, u64 nhz, u64 nlx, u64 nly, u64 nlz,
                                                       const SourceQ& q, float damp, const Poly& pl,
                                                       u64 (&ar)[kPairs], u64 (&ai)[kPairs]) {
#pragma unroll
  for (int t0 = 0; t0 < kTile; t0 += kGroup) {
    const int rem = int(n_t) - t0;  // warp-uniform
    if (rem > 2)
      compensated_block<DAMP, MODE, 2>(thi, tlo, t0, nhx, nhy, nhz, nlx, nly, nlz, q, damp, pl, &ar[t0 / 2], &ai[t0 / 2]);
    else if (rem > 0)
      compensated_block<DAMP, MODE, 1>(thi, tlo, t0, nhx, nhy, nhz, nlx, nly, nlz, q, damp, pl, &ar[t0 / 2], &ai[t0 / 2]);
  }
}

struct LeafGroup {
  // one lane = one source leaf of a group of up to 32
  uint32_t count, incl, excl;
};

__device__ __forceinline__ LeafGroup scan_group(uint32_t count, int lane) {
  LeafGroup g;
  g.count = count;
  uint32_t incl = count;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  g.incl = incl;
  g.excl = incl - count;
  return g;
}

// The bodies of a group of source leaves form one flat list; a chunk is 32 consecutive entries, one
// per lane.  Which leaf owns entry c0 + lane: the leaves that START inside the chunk mark a bit
// (one warp-wide OR), `before` counts the leaves that started before it; leaves are never empty, so
// owner = before + (marks at or below the lane) - 1.  Two instructions on the critical path instead
// of a five-step shuffle search.
__device__ __forceinline__ int chunk_owner(const LeafGroup& g, uint32_t c0, uint32_t& before, uint32_t lane_le) {
  const uint32_t rel = g.excl - c0;
  const uint32_t marks = __reduce_or_sync(0xffffffffu, (g.count && rel < 32u) ? 1u << rel : 0u);
  const int j = int(before + __popc(marks & lane_le)) - 1;
  before += __popc(marks);
  return j;
}

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_f4(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// shared memory of one warp (bytes): targets | hi | lo | leaf records | staged source bodies
constexpr uint32_t kSmTgt = 0, kSmHi = 4 * kTile * 4, kSmLo = kSmHi + 3 * kTile * 4, kSmRec = kSmLo + 3 * kTile * 4,
                   kSmStage = kSmRec + 2 * 32 * 16, kSmWarp = kSmStage + 2 * 32 * 32;

// 128 registers per thread keep eight 2-warp CTAs (16 warps) per SM; measured: 134 registers cost 40 %
template <bool DAMP, int MODE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 8) p2p_kernel(const P2PArgs a) {
  constexpr bool kExpanded = MODE == P2P_MODE_SINC_POLY_EXPANDED;
  constexpr bool kPoly = MODE != P2P_MODE_MUFU;
  __shared__ __align__(16) unsigned char s_all[kWarpsPerBlock][kSmWarp];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tile_id = blockIdx.x * kWarpsPerBlock + warp;
  if (tile_id >= a.n_tiles) return;
  P2PTile tile = a.tiles[tile_id];
  tile.n_t = __shfl_sync(0xffffffffu, tile.n_t, 0);
  const int4 tg = a.cell_geom[tile.leaf];
  const uint2 tb = a.cell_body[tile.leaf];
  const uint32_t tslot = tb.x + tile.body_off + lane;
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t sm = uint32_t(__cvta_generic_to_shared(s_all[warp]));
  const uint32_t a_tgt = sm + kSmTgt, a_thi = sm + kSmHi, a_tlo = sm + kSmLo, a_rec = sm + kSmRec,
                 a_stage = sm + kSmStage + 32u * lane;
  {
    const float4 tp = lane < tile.n_t ? a.body_pos[tslot] : zero4, th = lane < tile.n_t ? a.body_hi[tslot] : zero4,
                 tl = lane < tile.n_t ? a.body_lo[tslot] : zero4;
    float* s_tgt = reinterpret_cast<float*>(s_all[warp] + kSmTgt);
    float* s_thi = reinterpret_cast<float*>(s_all[warp] + kSmHi);
    float* s_tlo = reinterpret_cast<float*>(s_all[warp] + kSmLo);
    s_tgt[lane] = tp.x; s_tgt[kTile + lane] = tp.y; s_tgt[2 * kTile + lane] = tp.z;
    s_tgt[3 * kTile + lane] = fmaf(tp.z, tp.z, fmaf(tp.y, tp.y, tp.x * tp.x));
    s_thi[lane] = th.x; s_thi[kTile + lane] = th.y; s_thi[2 * kTile + lane] = th.z;
    s_tlo[lane] = tl.x; s_tlo[kTile + lane] = tl.y; s_tlo[2 * kTile + lane] = tl.z;
  }
  const uint32_t lane_le = 0xffffffffu >> (31 - lane);

  Poly pl;
#pragma unroll
  for (int i = 0; i <= kP2PPolyDegree; ++i) {
    pl.s[i] = kPoly ? pack2(a.sinc_c[i], a.sinc_c[i]) : 0ull;
    pl.c[i] = MODE == P2P_MODE_ALL_POLY ? pack2(a.cos_c[i], a.cos_c[i]) : 0ull;
  }
  // a lane without a source body evaluates a harmless pair with zero charge: far away for the MUFU
  // path (sin / cos of anything are bounded), at the leaf centre for the polynomials (bounded R' only)
  const float pad = kPoly ? 0.0f : 1e4f;

  u64 ar[kPairs], ai[kPairs];  // accumulators of targets (2j, 2j+1)
#pragma unroll
  for (int t = 0; t < kPairs; ++t) ar[t] = ai[t] = 0ull;

  const uint32_t lb = a.p2p_offset[tile.list], lsplit = a.p2p_split[tile.list],
                 le = a.p2p_offset[tile.list + 1];

  // ---- touching leaves: compensated coordinates, masked
  for (uint32_t g0 = lb; g0 < lsplit; g0 += 32) {
    const uint32_t e = g0 + lane;
    const bool has = e < lsplit;
    const uint32_t sc = has ? a.p2p_src[e] : tile.leaf;
    const int4 sg = a.cell_geom[sc];
    const uint2 sb = a.cell_body[sc];
    const LeafGroup grp = scan_group(has ? sb.y : 0u, lane);
    // exact offset in FP64, split on the grid: o = o_hi + o_lo
    const double inv_grid = 1.0 / a.grid;
    const double odx = double(sg.x - tg.x) * a.kunit_d, ody = double(sg.y - tg.y) * a.kunit_d,
                 odz = double(sg.z - tg.z) * a.kunit_d;
    const double ohx = rint(odx * inv_grid) * a.grid, ohy = rint(ody * inv_grid) * a.grid,
                 ohz = rint(odz * inv_grid) * a.grid;
    __syncwarp();  // the previous group's records have had their last reader
    sts_f4(a_rec + 16u * lane, make_float4(float(ohx), float(ohy), float(ohz), __uint_as_float(sb.x - grp.excl)));
    sts_f4(a_rec + 512u + 16u * lane, make_float4(float(odx - ohx), float(ody - ohy), float(odz - ohz), 0.f));
    __syncwarp();
    const uint32_t total = __shfl_sync(0xffffffffu, grp.incl, 31);
    uint32_t before = 0;
    for (uint32_t c0 = 0; c0 < total; c0 += 32) {
      const uint32_t g = c0 + lane;
      const int j = chunk_owner(grp, c0, before, lane_le);
      const bool ok = g < total;
      const float4 oh = lds_f4(a_rec + 16u * j), ol = lds_f4(a_rec + 512u + 16u * j);
      const uint32_t slot = g + __float_as_uint(oh.w);
      const float4 sh = ok ? a.body_hi[slot] : zero4;
      const float4 sl = ok ? a.body_lo[slot] : zero4;
      const float2 q = ok ? a.body_q[slot] : make_float2(0.f, 0.f);
      const float hx = ok ? -(sh.x + oh.x) : -pad, hy = ok ? -(sh.y + oh.y) : -pad, hz = ok ? -(sh.z + oh.z) : -pad;
      const float lx = ok ? -(sl.x + ol.x) : 0.f, ly = ok ? -(sl.y + ol.y) : 0.f, lz = ok ? -(sl.z + ol.z) : 0.f;
      const SourceQ sq{pack2(q.x, q.x), pack2(q.y, q.y), pack2(-q.y, -q.y)};
      accumulate_compensated<DAMP, MODE>(a_thi, a_tlo, tile.n_t, pack2(hx, hx), pack2(hy, hy), pack2(hz, hz),
                                         pack2(lx, lx), pack2(ly, ly), pack2(lz, lz), sq, a.damp, pl, ar, ai);
    }
  }

  // ---- all other source leaves: plain coordinates, bodies flattened across groups of 32 leaves.
  // The bodies of chunk c + 1 are fetched with cp.async into a lane-private staging slot while chunk c
  // is evaluated (ncu: the first use of a directly loaded body was 10 % of all stall samples).
  for (uint32_t g0 = lsplit; g0 < le; g0 += 32) {
    const uint32_t e = g0 + lane;
    const bool has = e < le;
    const uint32_t sc = has ? a.p2p_src[e] : tile.leaf;
    const int4 sg = a.cell_geom[sc];
    const uint2 sb = a.cell_body[sc];
    const LeafGroup grp = scan_group(has ? sb.y : 0u, lane);
    __syncwarp();
    sts_f4(a_rec + 16u * lane, make_float4(float(sg.x - tg.x) * a.kunit, float(sg.y - tg.y) * a.kunit,
                                           float(sg.z - tg.z) * a.kunit, __uint_as_float(sb.x - grp.excl)));
    __syncwarp();
    const uint32_t total = __shfl_sync(0xffffffffu, grp.incl, 31);
    uint32_t before = 0;
    // fetch of chunk c0 into staging buffer `buf`; returns the owner leaf of the lane's entry
    auto fetch = [&](uint32_t c0, uint32_t buf) {
      const int j = chunk_owner(grp, c0, before, lane_le);
      if (c0 + lane < total) {
        const float dl = lds_f4(a_rec + 16u * j).w;
        const uint32_t slot = c0 + lane + __float_as_uint(dl);
        const uint32_t dst = a_stage + 1024u * buf;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(a.body_pos + slot) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 16u), "l"(a.body_q + slot) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      return j;
    };
    int j = fetch(0, 0);
    for (uint32_t c0 = 0, buf = 0; c0 < total; c0 += 32, buf ^= 1) {
      const bool ok = c0 + lane < total;
      asm volatile("cp.async.wait_all;" ::: "memory");
      const float4 o = lds_f4(a_rec + 16u * j);
      float4 sp = zero4;
      float2 q = make_float2(0.f, 0.f);
      if (ok) {
        sp = lds_f4(a_stage + 1024u * buf);
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(q.x), "=f"(q.y) : "r"(a_stage + 1024u * buf + 16u));
      }
      if (c0 + 32 < total) j = fetch(c0 + 32, buf ^ 1);
      const float px = ok ? sp.x + o.x : pad, py = ok ? sp.y + o.y : pad, pz = ok ? sp.z + o.z : pad;
      const SourceQ sq{pack2(q.x, q.x), pack2(q.y, q.y), pack2(-q.y, -q.y)};
      if (kExpanded) {
        const float s2 = fmaf(pz, pz, fmaf(py, py, fmaf(px, px, 1e-30f)));
        accumulate_expanded<DAMP, MODE>(a_tgt, a_tgt + 4 * kTile, a_tgt + 8 * kTile, a_tgt + 12 * kTile, tile.n_t,
                                        pack2(-2.f * px, -2.f * px), pack2(-2.f * py, -2.f * py),
                                        pack2(-2.f * pz, -2.f * pz), pack2(s2, s2), sq, a.damp, pl, ar, ai);
      } else {
        accumulate_plain<DAMP, MODE>(a_tgt, a_tgt + 4 * kTile, a_tgt + 8 * kTile, tile.n_t, pack2(-px, -px),
                                     pack2(-py, -py), pack2(-pz, -pz), sq, a.damp, pl, ar, ai);
      }
    }
  }

  // per-target reduction over the 32 source lanes; lane t keeps target t.  One butterfly for all 32
  // targets: at every exchange a lane hands over the half of its values that its partner keeps
  // (16 + 8 + 4 + 2 packed pairs, then the two halves of the last pair: 31 shuffled words per array
  // instead of 160); the pairing order — hence the rounding — is that of 32 separate reductions.
#pragma unroll
  for (int half = kPairs / 2, o = 16; half >= 1; half >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const u64 kr = up ? ar[i + half] : ar[i], sr = up ? ar[i] : ar[i + half];
      const u64 ki = up ? ai[i + half] : ai[i], si = up ? ai[i] : ai[i + half];
      ar[i] = add2(kr, __shfl_xor_sync(0xffffffffu, sr, o));
      ai[i] = add2(ki, __shfl_xor_sync(0xffffffffu, si, o));
    }
  }
  const float2 pr = unpack2(ar[0]), pi = unpack2(ai[0]);
  const bool odd = (lane & 1) != 0;
  const float out_r = (odd ? pr.y : pr.x) + __shfl_xor_sync(0xffffffffu, odd ? pr.x : pr.y, 1);
  const float out_i = (odd ? pi.y : pi.x) + __shfl_xor_sync(0xffffffffu, odd ? pi.x : pi.y, 1);
  if (lane < tile.n_t) a.out[tslot] = make_float2(out_r * a.out_scale, out_i * a.out_scale);
}

}  // namespace

namespace {
template <int MODE>
void launch_p2p_mode(const P2PArgs& a, uint32_t blocks, cudaStream_t s) {
  if (a.damp != 0.0f) p2p_kernel<true, MODE><<<blocks, kWarpsPerBlock * 32, 0, s>>>(a);
  else p2p_kernel<false, MODE><<<blocks, kWarpsPerBlock * 32, 0, s>>>(a);
}
}  // namespace

void launch_p2p(const P2PArgs& a, cudaStream_t s) {
  if (a.n_tiles == 0) return;
  const uint32_t blocks = (a.n_tiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  switch (a.mode) {
    case P2P_MODE_SINC_POLY: launch_p2p_mode<P2P_MODE_SINC_POLY>(a, blocks, s); break;
    case P2P_MODE_SINC_POLY_EXPANDED: launch_p2p_mode<P2P_MODE_SINC_POLY_EXPANDED>(a, blocks, s); break;
    case P2P_MODE_ALL_POLY: launch_p2p_mode<P2P_MODE_ALL_POLY>(a, blocks, s); break;
    default: launch_p2p_mode<P2P_MODE_MUFU>(a, blocks, s); break;
  }
  HFMM_CUDA_CHECK(cudaGetLastError());
}

// Chebyshev interpolation of f(u) on [0, U] at degree + 1 nodes (near-minimax), returned as monomial
// coefficients in u; long double throughout
void fit_p2p_polynomials(double r2_max, float sinc_c[8], float cos_c[8]) {
  constexpr int D = kP2PPolyDegree;
  const long double U = r2_max > 1e-6 ? (long double)r2_max : 1e-6L, pi = 3.14159265358979323846264338327950288L;
  for (int which = 0; which < 2; ++which) {
    long double cheb[D + 1] = {};
    for (int k = 0; k <= D; ++k) {
      const long double x = cosl(pi * (k + 0.5L) / (D + 1)), u = (x + 1) * U / 2, r = sqrtl(u);
      const long double f = which ? cosl(r) : (r > 1e-8L ? sinl(r) / r : 1 - u / 6);
      for (int j = 0; j <= D; ++j) cheb[j] += f * cosl(pi * j * (k + 0.5L) / (D + 1));
    }
    for (int j = 0; j <= D; ++j) cheb[j] *= (j ? 2.0L : 1.0L) / (D + 1);
    // sum_j cheb[j] T_j(x), x = (2/U) u - 1, expanded in powers of u
    long double tm[D + 1] = {1}, tc[D + 1] = {-1, 2 / U}, out[D + 1] = {};
    for (int i = 0; i <= D; ++i) out[i] = cheb[0] * tm[i] + (D >= 1 ? cheb[1] * tc[i] : 0);
    for (int j = 2; j <= D; ++j) {
      long double tn[D + 1] = {};
      for (int i = 0; i <= D; ++i) {
        tn[i] = -2 * tc[i] - tm[i];
        if (i) tn[i] += 2 * (2 / U) * tc[i - 1];
      }
      for (int i = 0; i <= D; ++i) {
        out[i] += cheb[j] * tn[i];
        tm[i] = tc[i];
        tc[i] = tn[i];
      }
    }
    float* dst = which ? cos_c : sinc_c;
    for (int i = 0; i < 8; ++i) dst[i] = i <= D ? float(out[i]) : 0.0f;
  }
}

}  // namespace hfmm_b200
