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
//     target coordinates are broadcast from shared memory;
//   * one warp-shuffle reduction per target at the very end.
// Coordinates arrive pre-scaled by k and leaf-relative; the lattice offset between the two leaf
// centres is added per source body.  G = (k/4pi) e^{iR'}/R' with R' = kR, the constant applied once
// at the store.  Per pair (plain path): 3 FADD, 3 FFMA (R'^2), MUFU.RSQ, FMUL (R'), FMUL+MUFU.SIN,
// MUFU.COS, 2 FMUL, 4 FFMA.
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
constexpr int kWarpsPerBlock = 4;

__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
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

__device__ __forceinline__ void green_accumulate(float r2, float rinv, float qr, float qi,
                                                 float& ar, float& ai) {
  const float r = r2 * rinv;
  const float gr = rinv * cos_approx(r), gi = rinv * sin_approx(r);
  ar = fmaf(gr, qr, ar);
  ar = fmaf(-gi, qi, ar);
  ai = fmaf(gr, qi, ai);
  ai = fmaf(gi, qr, ai);
}

// Targets are walked in groups of kGroup: one warp-uniform branch per group and kGroup independent
// evaluations in a straight line, so the MUFU / FMA latencies overlap.  Target coordinates are read with explicit ld.shared from a
// 32-bit shared address (register + immediate; the generic-pointer form re-derived the address in
// every group).
constexpr int kGroup = 4;

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

template <int N>
__device__ __forceinline__ void plain_group(uint32_t tgt, int t0, float sx, float sy, float sz,
                                            float qr, float qi, float (&ar)[kTile], float (&ai)[kTile]) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float4 tp = lds_f4(tgt + 16 * (t0 + j));
    const float dx = tp.x - sx, dy = tp.y - sy, dz = tp.z - sz;
    const float r2 = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, 1e-30f)));
    green_accumulate(r2, rsqrt_approx(r2), qr, qi, ar[t0 + j], ai[t0 + j]);
  }
}

// plain path: one FP32 coordinate per axis.  Slots past n_t inside the last group hold zero
// coordinates; their accumulators are never stored.
__device__ __forceinline__ void accumulate_plain(uint32_t tgt, uint32_t n_t, float sx, float sy,
                                                 float sz, float qr, float qi, float (&ar)[kTile],
                                                 float (&ai)[kTile]) {
#pragma unroll
  for (int t0 = 0; t0 < kTile; t0 += kGroup)
    if (t0 < n_t) plain_group<kGroup>(tgt, t0, sx, sy, sz, qr, qi, ar, ai);  // warp-uniform
}

template <int N>
__device__ __forceinline__ void compensated_group(uint32_t thi, uint32_t tlo, int t0, float hx, float hy,
                                                  float hz, float lx, float ly, float lz, float qr,
                                                  float qi, float (&ar)[kTile], float (&ai)[kTile]) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float4 th = lds_f4(thi + 16 * (t0 + j)), tl = lds_f4(tlo + 16 * (t0 + j));
    const float dx = (th.x - hx) + (tl.x - lx);
    const float dy = (th.y - hy) + (tl.y - ly);
    const float dz = (th.z - hz) + (tl.z - lz);
    const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    const float rinv = r2 > 0.0f ? rsqrt_approx(r2) : 0.0f;
    green_accumulate(r2, rinv, qr, qi, ar[t0 + j], ai[t0 + j]);
  }
}

// compensated path: d = (hi_t - hi_s) + (lo_t - lo_s); the hi difference is exact (grid multiples)
__device__ __forceinline__ void accumulate_compensated(uint32_t thi, uint32_t tlo, uint32_t n_t, float hx,
                                                       float hy, float hz, float lx, float ly, float lz,
                                                       float qr, float qi, float (&ar)[kTile],
                                                       float (&ai)[kTile]) {
#pragma unroll
  for (int t0 = 0; t0 < kTile; t0 += kGroup)
    if (t0 < n_t) compensated_group<kGroup>(thi, tlo, t0, hx, hy, hz, lx, ly, lz, qr, qi, ar, ai);
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
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 4) p2p_kernel(const P2PArgs a) {
  __shared__ float4 s_tgt[kWarpsPerBlock][kTile];
  __shared__ float4 s_thi[kWarpsPerBlock][kTile];
  __shared__ float4 s_tlo[kWarpsPerBlock][kTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tile_id = blockIdx.x * kWarpsPerBlock + warp;
  if (tile_id >= a.n_tiles) return;
  P2PTile tile = a.tiles[tile_id];
  tile.n_t = __shfl_sync(0xffffffffu, tile.n_t, 0);
  const int4 tg = a.cell_geom[tile.leaf];
  const uint2 tb = a.cell_body[tile.leaf];
  const uint32_t tslot = tb.x + tile.body_off + lane;
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  s_tgt[warp][lane] = lane < tile.n_t ? a.body_pos[tslot] : zero4;
  s_thi[warp][lane] = lane < tile.n_t ? a.body_hi[tslot] : zero4;
  s_tlo[warp][lane] = lane < tile.n_t ? a.body_lo[tslot] : zero4;
  __syncwarp();
  const uint32_t a_tgt = uint32_t(__cvta_generic_to_shared(s_tgt[warp])),
                 a_thi = uint32_t(__cvta_generic_to_shared(s_thi[warp])),
                 a_tlo = uint32_t(__cvta_generic_to_shared(s_tlo[warp]));

  float ar[kTile], ai[kTile];
#pragma unroll
  for (int t = 0; t < kTile; ++t) ar[t] = ai[t] = 0.0f;

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
      accumulate_compensated(a_thi, a_tlo, tile.n_t, sh.x + hxj, sh.y + hyj, sh.z + hzj,
                             sl.x + lxj, sl.y + lyj, sl.z + lzj, q.x, q.y, ar, ai);
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
      accumulate_plain(a_tgt, tile.n_t, sp.x + oxj, sp.y + oyj, sp.z + ozj, q.x, q.y, ar, ai);
    }
  }

  // per-target reduction over the 32 source lanes; lane t keeps target t
  float out_r = 0.f, out_i = 0.f;
#pragma unroll
  for (int t = 0; t < kTile; ++t) {
    if (t < tile.n_t) {
      float vr = ar[t], vi = ai[t];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        vr += __shfl_xor_sync(0xffffffffu, vr, o);
        vi += __shfl_xor_sync(0xffffffffu, vi, o);
      }
      if (lane == t) {
        out_r = vr;
        out_i = vi;
      }
    }
  }
  if (lane < tile.n_t) a.out[tslot] = make_float2(out_r * a.out_scale, out_i * a.out_scale);
}

}  // namespace

void launch_p2p(const P2PArgs& a, cudaStream_t s) {
  if (a.n_tiles == 0) return;
  const uint32_t blocks = (a.n_tiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  p2p_kernel<<<blocks, kWarpsPerBlock * 32, 0, s>>>(a);
  HFMM_CUDA_CHECK(cudaGetLastError());
}

}  // namespace hfmm_b200
