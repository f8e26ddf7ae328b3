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
// at the store.  Per pair: 3 FADD, 3 FFMA (R'^2), MUFU.RSQ, FMUL (R'), FMUL+MUFU.SIN, MUFU.COS,
// 2 FMUL, 4 FFMA.  The self leaf needs the R == 0 mask and is a separate pass; all other leaves
// cannot hold coincident bodies (same key => same leaf) and run unmasked with a 1e-30 floor that
// only guards against NaN.
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

template <bool kMasked>
__device__ __forceinline__ void pair_eval(const float4 t, float sx, float sy, float sz, float qr,
                                          float qi, float& ar, float& ai) {
  const float dx = t.x - sx, dy = t.y - sy, dz = t.z - sz;
  float r2, rinv;
  if (kMasked) {
    r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    rinv = r2 > 0.0f ? rsqrt_approx(r2) : 0.0f;
  } else {
    r2 = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, 1e-30f)));
    rinv = rsqrt_approx(r2);
  }
  const float r = r2 * rinv;
  const float gr = rinv * cos_approx(r), gi = rinv * sin_approx(r);
  ar = fmaf(gr, qr, ar);
  ar = fmaf(-gi, qi, ar);
  ai = fmaf(gr, qi, ai);
  ai = fmaf(gi, qr, ai);
}

template <bool kMasked>
__device__ __forceinline__ void accumulate_tile(const float4* __restrict__ tgt, uint32_t n_t,
                                                float sx, float sy, float sz, float qr, float qi,
                                                float (&ar)[kTile], float (&ai)[kTile]) {
#pragma unroll
  for (int t = 0; t < kTile; ++t) {
    if (t < n_t) {  // warp-uniform
      const float4 tp = tgt[t];
      pair_eval<kMasked>(tp, sx, sy, sz, qr, qi, ar[t], ai[t]);
    }
  }
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) p2p_kernel(const P2PArgs a) {
  __shared__ float4 s_tgt[kWarpsPerBlock][kTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tile_id = blockIdx.x * kWarpsPerBlock + warp;
  if (tile_id >= a.n_tiles) return;
  const P2PTile tile = a.tiles[tile_id];
  const int4 tg = a.cell_geom[tile.leaf];
  const uint2 tb = a.cell_body[tile.leaf];
  const uint32_t tslot = tb.x + tile.body_off + lane;
  s_tgt[warp][lane] = lane < tile.n_t ? a.body_pos[tslot] : make_float4(0.f, 0.f, 0.f, 0.f);
  __syncwarp();
  const float4* tgt = s_tgt[warp];

  float ar[kTile], ai[kTile];
#pragma unroll
  for (int t = 0; t < kTile; ++t) ar[t] = ai[t] = 0.0f;

  // self leaf: same frame, coincident pairs masked
  for (uint32_t base = 0; base < tb.y; base += 32) {
    const uint32_t j = base + lane;
    const bool ok = j < tb.y;
    const float4 sp = ok ? a.body_pos[tb.x + j] : make_float4(1e4f, 1e4f, 1e4f, 0.f);
    const float2 q = ok ? a.body_q[tb.x + j] : make_float2(0.f, 0.f);
    accumulate_tile<true>(tgt, tile.n_t, sp.x, sp.y, sp.z, q.x, q.y, ar, ai);
  }

  // listed source leaves, 32 leaves per group, bodies flattened across the group
  const uint32_t lb = a.p2p_offset[tile.list], le = a.p2p_offset[tile.list + 1];
  for (uint32_t g0 = lb; g0 < le; g0 += 32) {
    const uint32_t e = g0 + lane;
    const bool has = e < le;
    const uint32_t sc = has ? a.p2p_src[e] : tile.leaf;
    const int4 sg = a.cell_geom[sc];
    uint2 sb = a.cell_body[sc];
    if (!has) sb.y = 0;
    const float ox = float(sg.x - tg.x) * a.kunit;
    const float oy = float(sg.y - tg.y) * a.kunit;
    const float oz = float(sg.z - tg.z) * a.kunit;
    uint32_t incl = sb.y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t excl = incl - sb.y;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t c0 = 0; c0 < total; c0 += 32) {
      const uint32_t g = c0 + lane;
      int j = 0;  // first lane whose inclusive count exceeds g
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, j + step - 1);
        if (v <= g) j += step;
      }
      const uint32_t first_j = __shfl_sync(0xffffffffu, sb.x, j);
      const uint32_t excl_j = __shfl_sync(0xffffffffu, excl, j);
      const float oxj = __shfl_sync(0xffffffffu, ox, j);
      const float oyj = __shfl_sync(0xffffffffu, oy, j);
      const float ozj = __shfl_sync(0xffffffffu, oz, j);
      const bool ok = g < total;
      const uint32_t slot = first_j + (g - excl_j);
      const float4 sp = ok ? a.body_pos[slot] : make_float4(1e4f, 1e4f, 1e4f, 0.f);
      const float2 q = ok ? a.body_q[slot] : make_float2(0.f, 0.f);
      accumulate_tile<false>(tgt, tile.n_t, sp.x + oxj, sp.y + oyj, sp.z + ozj, q.x, q.y, ar, ai);
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
