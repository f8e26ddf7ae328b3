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

// acc += (rinv e^{i r2 rinv}) * q for a pair of targets.  DAMP: complex wavenumber k_r + i k_i, the
// amplitude decays as e^{-k_i R} = 2^{-damp R'} with R' = k_r R (kernel.hpp:20), one more MUFU
template <bool DAMP>
__device__ __forceinline__ void green_accumulate2(u64 r2, u64 rinv, const SourceQ& q, float damp, u64& ar,
                                                  u64& ai) {
  const float2 r = unpack2(mul2(r2, rinv));
  if (DAMP) rinv = mul2(rinv, pack2(ex2_approx(-damp * r.x), ex2_approx(-damp * r.y)));
  const u64 c = pack2(cos_approx(r.x), cos_approx(r.y)), s = pack2(sin_approx(r.x), sin_approx(r.y));
  const u64 gr = mul2(rinv, c), gi = mul2(rinv, s);
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
// group hold zero coordinates; their accumulators are never stored.
template <bool DAMP>
__device__ __forceinline__ void accumulate_plain(uint32_t tx, uint32_t ty, uint32_t tz, uint32_t n_t,
                                                 u64 nsx, u64 nsy, u64 nsz, const SourceQ& q, float damp,
                                                 u64 (&ar)[kPairs], u64 (&ai)[kPairs]) {
  const u64 tiny = pack2(1e-30f, 1e-30f);
#pragma unroll
  for (int t0 = 0; t0 < kTile; t0 += kGroup)
    if (t0 < n_t) {  // warp-uniform
      u64 x[2], y[2], z[2];
      lds_2x2(tx + 4 * t0, x[0], x[1]);
      lds_2x2(ty + 4 * t0, y[0], y[1]);
      lds_2x2(tz + 4 * t0, z[0], z[1]);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const u64 dx = add2(x[j], nsx), dy = add2(y[j], nsy), dz = add2(z[j], nsz);
        const u64 r2 = fma2(dz, dz, fma2(dy, dy, fma2(dx, dx, tiny)));
        const float2 r2s = unpack2(r2);
        const u64 rinv = pack2(rsqrt_approx(r2s.x), rsqrt_approx(r2s.y));
        green_accumulate2<DAMP>(r2, rinv, q, damp, ar[t0 / 2 + j], ai[t0 / 2 + j]);
      }
    }
}

// compensated path: d = (hi_t - hi_s) + (lo_t - lo_s); the hi difference is exact (grid multiples);
// coincident bodies (R == 0) are masked
template <bool DAMP>
__device__ __forceinline__ void accumulate_compensated(uint32_t thi, uint32_t tlo, uint32_t n_t, u64 nhx,
                                                       u64 nhy, u64 nhz, u64 nlx, u64 nly, u64 nlz,
                                                       const SourceQ& q, float damp, u64 (&ar)[kPairs],
                                                       u64 (&ai)[kPairs]) {
#pragma unroll
  for (int t0 = 0; t0 < kTile; t0 += kGroup)
    if (t0 < n_t) {
      u64 hx[2], hy[2], hz[2], lx[2], ly[2], lz[2];
      lds_2x2(thi + 4 * t0, hx[0], hx[1]);
      lds_2x2(thi + 4 * (kTile + t0), hy[0], hy[1]);
      lds_2x2(thi + 4 * (2 * kTile + t0), hz[0], hz[1]);
      lds_2x2(tlo + 4 * t0, lx[0], lx[1]);
      lds_2x2(tlo + 4 * (kTile + t0), ly[0], ly[1]);
      lds_2x2(tlo + 4 * (2 * kTile + t0), lz[0], lz[1]);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const u64 dx = add2(add2(hx[j], nhx), add2(lx[j], nlx));
        const u64 dy = add2(add2(hy[j], nhy), add2(ly[j], nly));
        const u64 dz = add2(add2(hz[j], nhz), add2(lz[j], nlz));
        const u64 r2 = fma2(dz, dz, fma2(dy, dy, mul2(dx, dx)));
        const float2 r2s = unpack2(r2);
        const u64 rinv = pack2(r2s.x > 0.0f ? rsqrt_approx(r2s.x) : 0.0f, r2s.y > 0.0f ? rsqrt_approx(r2s.y) : 0.0f);
        green_accumulate2<DAMP>(r2, rinv, q, damp, ar[t0 / 2 + j], ai[t0 / 2 + j]);
      }
    }
}

struct LeafGroup {
  // one lane = one source leaf of a group of up to 32
  uint32_t first, count, incl, excl;
};

__device__ __forceinline__ LeafGroup scan_group(uint2 sb, int lane) {
  LeafGroup g;
  g.first = sb.x;
  g.count = sb.y;
  uint32_t incl = sb.y;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  g.incl = incl;
  g.excl = incl - sb.y;
  return g;
}

// lane-local: which leaf of the group owns flattened body index g (first lane with incl > g)
__device__ __forceinline__ int owner_of(uint32_t incl, uint32_t g) {
  int j = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const uint32_t v = __shfl_sync(0xffffffffu, incl, j + step - 1);
    if (v <= g) j += step;
  }
  return j;
}

// 128 registers per thread keep four CTAs (16 warps) per SM; measured: 134 registers (3 CTAs) cost 40 %
template <bool DAMP>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 8) p2p_kernel(const P2PArgs a) {
  // target coordinates, one array per axis: [x | y | z][kTile]
  __shared__ __align__(16) float s_tgt[kWarpsPerBlock][3 * kTile];
  __shared__ __align__(16) float s_thi[kWarpsPerBlock][3 * kTile];
  __shared__ __align__(16) float s_tlo[kWarpsPerBlock][3 * kTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tile_id = blockIdx.x * kWarpsPerBlock + warp;
  if (tile_id >= a.n_tiles) return;
  P2PTile tile = a.tiles[tile_id];
  tile.n_t = __shfl_sync(0xffffffffu, tile.n_t, 0);
  const int4 tg = a.cell_geom[tile.leaf];
  const uint2 tb = a.cell_body[tile.leaf];
  const uint32_t tslot = tb.x + tile.body_off + lane;
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  {
    const float4 tp = lane < tile.n_t ? a.body_pos[tslot] : zero4, th = lane < tile.n_t ? a.body_hi[tslot] : zero4,
                 tl = lane < tile.n_t ? a.body_lo[tslot] : zero4;
    s_tgt[warp][lane] = tp.x; s_tgt[warp][kTile + lane] = tp.y; s_tgt[warp][2 * kTile + lane] = tp.z;
    s_thi[warp][lane] = th.x; s_thi[warp][kTile + lane] = th.y; s_thi[warp][2 * kTile + lane] = th.z;
    s_tlo[warp][lane] = tl.x; s_tlo[warp][kTile + lane] = tl.y; s_tlo[warp][2 * kTile + lane] = tl.z;
  }
  __syncwarp();
  const uint32_t a_tgt = uint32_t(__cvta_generic_to_shared(s_tgt[warp])),
                 a_thi = uint32_t(__cvta_generic_to_shared(s_thi[warp])),
                 a_tlo = uint32_t(__cvta_generic_to_shared(s_tlo[warp]));

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
    uint2 sb = a.cell_body[sc];
    if (!has) sb.y = 0;
    // exact offset in FP64, split on the grid: o = o_hi + o_lo
    const double inv_grid = 1.0 / a.grid;
    const double odx = double(sg.x - tg.x) * a.kunit_d, ody = double(sg.y - tg.y) * a.kunit_d,
                 odz = double(sg.z - tg.z) * a.kunit_d;
    const double ohx = rint(odx * inv_grid) * a.grid, ohy = rint(ody * inv_grid) * a.grid,
                 ohz = rint(odz * inv_grid) * a.grid;
    const float fhx = float(ohx), fhy = float(ohy), fhz = float(ohz);
    const float flx = float(odx - ohx), fly = float(ody - ohy), flz = float(odz - ohz);
    const LeafGroup grp = scan_group(sb, lane);
    const uint32_t total = __shfl_sync(0xffffffffu, grp.incl, 31);
    for (uint32_t c0 = 0; c0 < total; c0 += 32) {
      const uint32_t g = c0 + lane;
      const int j = owner_of(grp.incl, g);
      const uint32_t first_j = __shfl_sync(0xffffffffu, grp.first, j);
      const uint32_t excl_j = __shfl_sync(0xffffffffu, grp.excl, j);
      const float hxj = __shfl_sync(0xffffffffu, fhx, j), hyj = __shfl_sync(0xffffffffu, fhy, j),
                  hzj = __shfl_sync(0xffffffffu, fhz, j);
      const float lxj = __shfl_sync(0xffffffffu, flx, j), lyj = __shfl_sync(0xffffffffu, fly, j),
                  lzj = __shfl_sync(0xffffffffu, flz, j);
      const bool ok = g < total;
      const uint32_t slot = first_j + (g - excl_j);
      const float4 sh = ok ? a.body_hi[slot] : make_float4(1e4f, 1e4f, 1e4f, 0.f);
      const float4 sl = ok ? a.body_lo[slot] : zero4;
      const float2 q = ok ? a.body_q[slot] : make_float2(0.f, 0.f);
      const float hx = -(sh.x + hxj), hy = -(sh.y + hyj), hz = -(sh.z + hzj);
      const float lx = -(sl.x + lxj), ly = -(sl.y + lyj), lz = -(sl.z + lzj);
      const SourceQ sq{pack2(q.x, q.x), pack2(q.y, q.y), pack2(-q.y, -q.y)};
      accumulate_compensated<DAMP>(a_thi, a_tlo, tile.n_t, pack2(hx, hx), pack2(hy, hy), pack2(hz, hz),
                                   pack2(lx, lx), pack2(ly, ly), pack2(lz, lz), sq, a.damp, ar, ai);
    }
  }

  // ---- all other source leaves: plain coordinates, bodies flattened across groups of 32 leaves
  for (uint32_t g0 = lsplit; g0 < le; g0 += 32) {
    const uint32_t e = g0 + lane;
    const bool has = e < le;
    const uint32_t sc = has ? a.p2p_src[e] : tile.leaf;
    const int4 sg = a.cell_geom[sc];
    uint2 sb = a.cell_body[sc];
    if (!has) sb.y = 0;
    const float ox = float(sg.x - tg.x) * a.kunit;
    const float oy = float(sg.y - tg.y) * a.kunit;
    const float oz = float(sg.z - tg.z) * a.kunit;
    const LeafGroup grp = scan_group(sb, lane);
    const uint32_t total = __shfl_sync(0xffffffffu, grp.incl, 31);
    for (uint32_t c0 = 0; c0 < total; c0 += 32) {
      const uint32_t g = c0 + lane;
      const int j = owner_of(grp.incl, g);
      const uint32_t first_j = __shfl_sync(0xffffffffu, grp.first, j);
      const uint32_t excl_j = __shfl_sync(0xffffffffu, grp.excl, j);
      const float oxj = __shfl_sync(0xffffffffu, ox, j);
      const float oyj = __shfl_sync(0xffffffffu, oy, j);
      const float ozj = __shfl_sync(0xffffffffu, oz, j);
      const bool ok = g < total;
      const uint32_t slot = first_j + (g - excl_j);
      const float4 sp = ok ? a.body_pos[slot] : make_float4(1e4f, 1e4f, 1e4f, 0.f);
      const float2 q = ok ? a.body_q[slot] : make_float2(0.f, 0.f);
      const float sx = -(sp.x + oxj), sy = -(sp.y + oyj), sz = -(sp.z + ozj);
      const SourceQ sq{pack2(q.x, q.x), pack2(q.y, q.y), pack2(-q.y, -q.y)};
      accumulate_plain<DAMP>(a_tgt, a_tgt + 4 * kTile, a_tgt + 8 * kTile, tile.n_t, pack2(sx, sx), pack2(sy, sy),
                             pack2(sz, sz), sq, a.damp, ar, ai);
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

void launch_p2p(const P2PArgs& a, cudaStream_t s) {
  if (a.n_tiles == 0) return;
  const uint32_t blocks = (a.n_tiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (a.damp != 0.0f) p2p_kernel<true><<<blocks, kWarpsPerBlock * 32, 0, s>>>(a);
  else p2p_kernel<false><<<blocks, kWarpsPerBlock * 32, 0, s>>>(a);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

}  // namespace hfmm_b200
