// tree_build.cu — see tree_build.cuh
#include "tree_build.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <climits>
#include <cstdlib>
#include <tuple>
#include <cmath>

#include "common.hpp"

namespace hfmm_b200 {

namespace {

constexpr int kBlock = 256;
inline uint32_t grid_for(uint64_t n) { return uint32_t((n + kBlock - 1) / kBlock); }

struct TempStorage {
  DeviceBuffer<unsigned char> buf;
  void* get(size_t bytes) {
    if (buf.size() < bytes) buf.resize(bytes + (bytes >> 2) + 256);
    return buf.get();
  }
};

// ---- K1: keys (reference src/octree.cpp:25-51) ----------------------------------------------
__global__ void __launch_bounds__(kBlock)
morton_keys_kernel(const double* __restrict__ xyz, uint32_t n, double lox, double loy, double loz,
                   double scale, uint64_t* __restrict__ key, uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lo[3] = {lox, loy, loz};
  const long long nside = 1ll << kMaxLevel;
  uint64_t g[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    long long v = (long long)(__dmul_rn(__dsub_rn(xyz[3 * size_t(i) + a], lo[a]), scale));
    v = v < 0 ? 0 : (v >= nside ? nside - 1 : v);
    g[a] = uint64_t(v);
  }
  uint64_t k = 0;
  for (int b = kMaxLevel - 1; b >= 0; --b)
    k = k << 3 | ((g[0] >> b & 1) << 2) | ((g[1] >> b & 1) << 1) | (g[2] >> b & 1);
  key[i] = k;
  idx[i] = i;
}

// ---- K2: one level of the top-down split (reference src/octree.cpp:85-137) ------------------
struct CellArrays {
  uint8_t* level;
  uint32_t *ix, *iy, *iz, *body_first, *body_count, *child_first, *child_count, *parent;
};

__device__ __forceinline__ uint32_t lower_bound_digit(const uint64_t* key, uint32_t lo, uint32_t hi,
                                                      int shift, uint32_t digit) {
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (uint32_t((key[mid] >> shift) & 7) < digit) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kBlock)
split_count_kernel(CellArrays c, uint32_t c0, uint32_t c1, int level, int ncrit, bool over_diameter,
                   const uint64_t* __restrict__ key, uint32_t* __restrict__ nchild,
                   uint32_t* __restrict__ bounds) {
  const uint32_t i = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c1) return;
  const uint32_t first = c.body_first[i], count = c.body_count[i];
  const bool split = level < kMaxLevel && (int64_t(count) > int64_t(ncrit) || (over_diameter && count > 0));
  uint32_t nc = 0;
  if (split) {
    const int shift = 3 * (kMaxLevel - 1 - level);
    uint32_t* b = bounds + size_t(i - c0) * 9;
    b[0] = first;
    for (uint32_t d = 1; d < 8; ++d) b[d] = lower_bound_digit(key, b[d - 1], first + count, shift, d);
    b[8] = first + count;
    for (int d = 0; d < 8; ++d) nc += b[d + 1] > b[d];
  }
  nchild[i - c0] = nc;
}

__global__ void __launch_bounds__(kBlock)
write_children_kernel(CellArrays c, uint32_t c0, uint32_t c1, int level,
                      const uint32_t* __restrict__ nchild, const uint32_t* __restrict__ offs,
                      const uint32_t* __restrict__ bounds) {
  const uint32_t i = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c1) return;
  const uint32_t nc = nchild[i - c0];
  if (nc == 0) {
    c.child_first[i] = 0;
    c.child_count[i] = 0;
    return;
  }
  const uint32_t cf = c1 + offs[i - c0];
  c.child_first[i] = cf;
  c.child_count[i] = nc;
  const uint32_t* b = bounds + size_t(i - c0) * 9;
  uint32_t j = cf;
  for (uint32_t d = 0; d < 8; ++d) {
    if (b[d + 1] == b[d]) continue;
    c.level[j] = uint8_t(level + 1);
    c.ix[j] = c.ix[i] << 1 | (d >> 2 & 1);
    c.iy[j] = c.iy[i] << 1 | (d >> 1 & 1);
    c.iz[j] = c.iz[i] << 1 | (d & 1);
    c.body_first[j] = b[d];
    c.body_count[j] = b[d + 1] - b[d];
    c.parent[j] = i;
    ++j;
  }
}

template <typename T>
void grow(DeviceBuffer<T>& b, size_t keep, size_t want, cudaStream_t s) {
  if (b.size() >= want) return;
  DeviceBuffer<T> nb(want + want / 2);
  if (keep) HFMM_CUDA_CHECK(cudaMemcpyAsync(nb.get(), b.get(), keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  b = std::move(nb);
}

// ---- K3: pair frontier (reference src/traversal.cpp:45-79) -----------------------------------
struct TraversalGeom {
  double lo[3];
  double side[kMaxLevel + 1];
  double radius[kMaxLevel + 1];
  unsigned char gated[kMaxLevel + 1];  // k * diameter > kd_max at this level
  double theta;
};

struct PairSink {
  uint2* data;
  unsigned long long* count;
  unsigned long long cap;
};
// census pass of the multi-rank setup (tree_build.cuh): per-target-cell work instead of stored pairs
struct CensusSink {
  unsigned long long* cell_work = nullptr;  // [2 c] far pairs, [2 c + 1] near body pairs of target cell c: integers,
                                            // so the totals do not depend on the order of the atomics
  int* level_min = nullptr;                 // coarsest level among the SOURCES of the far pairs
};

// reserves `cnt` slots for this lane; one atomic per warp
__device__ __forceinline__ unsigned long long warp_reserve(unsigned long long* counter, uint32_t cnt) {
  const int lane = threadIdx.x & 31;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (lane == 31 && total) base = atomicAdd(counter, (unsigned long long)total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + (incl - cnt);
}

__global__ void __launch_bounds__(kBlock)
traversal_kernel(const uint2* __restrict__ frontier, unsigned long long n_front, const uint8_t* __restrict__ lvl,
                 const uint32_t* __restrict__ ix, const uint32_t* __restrict__ iy,
                 const uint32_t* __restrict__ iz, const uint32_t* __restrict__ child_first,
                 const uint32_t* __restrict__ child_count, const uint32_t* __restrict__ body_count,
                 uint32_t grain, unsigned long long* __restrict__ tasks, const TraversalGeom g, PairSink next,
                 PairSink far, PairSink near, int* __restrict__ overflow, const uint8_t* __restrict__ interest,
                 const CensusSink census) {
  const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  // pruned descent (multi-rank setup): a node none of whose two subtrees holds an owned cell is dropped
  const bool live = i < n_front && (!interest || (interest[frontier[i].x] | interest[frontier[i].y]));
  uint32_t a = 0, b = 0, n_far = 0, n_near = 0, n_next = 0;
  bool split_target = false;
  if (live) {
    const uint2 p = frontier[i];
    a = p.x;
    b = p.y;
    const int la = lvl[a], lb = lvl[b];
    bool adm = !(g.gated[la] || g.gated[lb]);
    const double ra = g.radius[la], rb = g.radius[lb];
    if (adm) {
      // centres as lo + (i + 0.5) * side, differences, norm, threshold: every operation rounded
      // on its own, the sequence of the reference (octree.cpp:116-119, traversal.cpp:49-50)
      const double sa = g.side[la], sb = g.side[lb];
      const double dx = __dsub_rn(__dadd_rn(g.lo[0], __dmul_rn(double(ix[a]) + 0.5, sa)),
                                  __dadd_rn(g.lo[0], __dmul_rn(double(ix[b]) + 0.5, sb)));
      const double dy = __dsub_rn(__dadd_rn(g.lo[1], __dmul_rn(double(iy[a]) + 0.5, sa)),
                                  __dadd_rn(g.lo[1], __dmul_rn(double(iy[b]) + 0.5, sb)));
      const double dz = __dsub_rn(__dadd_rn(g.lo[2], __dmul_rn(double(iz[a]) + 0.5, sa)),
                                  __dadd_rn(g.lo[2], __dmul_rn(double(iz[b]) + 0.5, sb)));
      const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      adm = __dsqrt_rn(d2) > __ddiv_rn(__dadd_rn(ra, rb), g.theta);
    }
    const uint32_t ca = child_count[a], cb = child_count[b];
    if (adm) n_far = 1;
    else if (ca == 0 && cb == 0) n_near = 1;
    else {
      split_target = ca != 0 && (cb == 0 || ra > rb);  // ties open the source
      n_next = split_target ? ca : cb;
    }
  }
  const unsigned long long s_far = warp_reserve(far.count, n_far);
  const unsigned long long s_near = warp_reserve(near.count, n_near);
  const unsigned long long s_next = warp_reserve(next.count, n_next);
  if (census.cell_work) {
    // census: nothing is stored; the pair's work goes to its target cell
    const unsigned long long bp = n_near ? (unsigned long long)body_count[a] * body_count[b] : 0ull;
    if (n_far) atomicAdd(census.cell_work + 2ull * a, 1ull);
    if (n_near) atomicAdd(census.cell_work + 2ull * a + 1, bp);
    // coarsest source level of the far pairs: the running minimum settles within the first levels of the walk,
    // after which no warp issues the atomic any more (the target side and the body-pair total are read off
    // cell_work on the host)
    const int ls = __reduce_min_sync(0xffffffffu, n_far ? int(lvl[b]) : kMaxLevel + 1);
    if ((threadIdx.x & 31) == 0 && ls < *reinterpret_cast<volatile int*>(census.level_min)) atomicMin(census.level_min, ls);
  } else {
    if (n_far) {
      if (s_far < far.cap) far.data[s_far] = make_uint2(a, b);
      else atomicOr(overflow, 1);
    }
    if (n_near) {
      if (s_near < near.cap) near.data[s_near] = make_uint2(a, b);
      else atomicOr(overflow, 2);
    }
  }
  if (n_next) {
    if (s_next + n_next <= next.cap) {
      const uint32_t cf = split_target ? child_first[a] : child_first[b];
      // FmmStats::tasks (traversal.cpp:56-59): a walk node opens a task when the bodies of its two cells
      // first fit the grain s — its parent node (this one) did not fit, body counts only shrink downwards
      const uint32_t other = split_target ? body_count[b] : body_count[a];
      const bool parent_open = body_count[a] + body_count[b] > grain;
      uint32_t opened = 0;
      for (uint32_t c = 0; c < n_next; ++c) {
        next.data[s_next + c] = split_target ? make_uint2(cf + c, b) : make_uint2(a, cf + c);
        if (parent_open && body_count[cf + c] + other <= grain) ++opened;
      }
      if (opened) atomicAdd(tasks, (unsigned long long)opened);
    } else {
      atomicOr(overflow, 4);
    }
  }
}

__global__ void __launch_bounds__(kBlock)
level_range_kernel(const uint2* __restrict__ pairs, unsigned long long n, const uint8_t* __restrict__ lvl,
                   int* __restrict__ out) {
  int mt = kMaxLevel + 1, ms = kMaxLevel + 1;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint2 p = pairs[i];
    mt = min(mt, int(lvl[p.x]));
    ms = min(ms, int(lvl[p.y]));
  }
  atomicMin(out, mt);
  atomicMin(out + 1, ms);
}

__global__ void __launch_bounds__(kBlock)
weights_kernel(const uint2* __restrict__ far, unsigned long long n_far, const uint2* __restrict__ near,
               unsigned long long n_near, const uint32_t* __restrict__ unit,
               const uint32_t* __restrict__ body_count, double alpha, double* __restrict__ weight) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  // alpha < 0: measured kernel-time ratio per M2L pair; alpha >= 0: the reference's per-body estimate
  // w = l + alpha r summed over the bodies of the target cell (partition.cpp:137-163)
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_far; i += stride)
    atomicAdd(weight + unit[far[i].x], alpha < 0 ? kPartitionM2lWeight : alpha * double(body_count[far[i].x]));
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_near; i += stride) {
    const uint2 p = near[i];
    atomicAdd(weight + unit[p.x], double(body_count[p.x]) * double(body_count[p.y]));
  }
}

// ---- near lists ------------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock)
near_keys_kernel(const uint2* __restrict__ near, unsigned long long n, const uint8_t* __restrict__ lvl,
                 const uint32_t* __restrict__ ix, const uint32_t* __restrict__ iy,
                 const uint32_t* __restrict__ iz, const uint32_t* __restrict__ body_count,
                 const uint32_t* __restrict__ leaf_slot, const uint8_t* __restrict__ owned, int max_level,
                 uint64_t* __restrict__ keys, unsigned long long* __restrict__ totals) {
  const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long bp = 0, obp = 0, own = 0, far2 = 0;
  if (i < n) {
    const uint2 p = near[i];
    bp = (unsigned long long)body_count[p.x] * body_count[p.y];
    uint64_t key = ~uint64_t(0);
    if (owned[p.x]) {
      own = 1;
      obp = bp;
      // cubes touch iff |centre difference| <= sum of half sides on every axis (lattice integers)
      const int ua = max_level - int(lvl[p.x]), ub = max_level - int(lvl[p.y]);
      const long long ha = 1ll << ua, hb = 1ll << ub;
      auto c = [](uint32_t v, int up) { return (long long)(2ull * v + 1) << up; };
      const long long ax = llabs(c(ix[p.x], ua) - c(ix[p.y], ub)), ay = llabs(c(iy[p.x], ua) - c(iy[p.y], ub)),
                      az = llabs(c(iz[p.x], ua) - c(iz[p.y], ub));
      const bool touch = ax <= ha + hb && ay <= ha + hb && az <= ha + hb;
      key = uint64_t(leaf_slot[p.x]) << 32 | (touch ? 0u : 0x80000000u) | p.y;
      // farthest two bodies of the two cubes can be apart, squared, in half-sides of the finest level
      const unsigned long long fx = (unsigned long long)(ax + ha + hb), fy = (unsigned long long)(ay + ha + hb),
                               fz = (unsigned long long)(az + ha + hb);
      far2 = fx * fx + fy * fy + fz * fz;
    }
    keys[i] = key;
  }
  // block totals -> three atomics per warp
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    bp += __shfl_xor_sync(0xffffffffu, bp, o);
    obp += __shfl_xor_sync(0xffffffffu, obp, o);
    own += __shfl_xor_sync(0xffffffffu, own, o);
    far2 = max(far2, __shfl_xor_sync(0xffffffffu, far2, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(totals, bp);
    atomicAdd(totals + 1, obp);
    atomicAdd(totals + 2, own);
    atomicMax(totals + 3, far2);
  }
}

__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t* a, uint32_t n, uint64_t v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kBlock)
near_offsets_kernel(const uint64_t* __restrict__ keys, uint32_t n_owned, uint32_t n_leaf,
                    uint32_t* __restrict__ offset, uint32_t* __restrict__ split) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n_leaf) return;
  offset[i] = lower_bound_u64(keys, n_owned, uint64_t(i) << 32);
  if (i < n_leaf) split[i] = lower_bound_u64(keys, n_owned, uint64_t(i) << 32 | 0x80000000u);
}

__global__ void __launch_bounds__(kBlock)
near_sources_kernel(const uint64_t* __restrict__ keys, uint32_t n_owned, uint32_t* __restrict__ src) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_owned) src[i] = uint32_t(keys[i] & 0x7fffffffu);
}

__global__ void __launch_bounds__(kBlock)
near_work_kernel(const uint32_t* __restrict__ offset, const uint32_t* __restrict__ src, uint32_t n_leaf,
                 const uint32_t* __restrict__ body_count, unsigned long long* __restrict__ work) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_leaf) return;
  unsigned long long w = 0;
  for (uint32_t e = offset[i]; e < offset[i + 1]; ++e) w += body_count[src[e]];
  work[i] = w;
}

// ---- far classes -----------------------------------------------------------------------------
// key = lt(5) | ls(5) | dx+2^17 (18) | dy+2^17 (18) | dz+2^17 (18): same (level pair, lattice shift)
// de-duplication as the reference's lattice_shift (src/traversal.cpp:152-166)
constexpr int kShiftBias = 1 << 17;

__global__ void __launch_bounds__(kBlock)
far_keys_kernel(const uint2* __restrict__ far, unsigned long long n, const uint8_t* __restrict__ lvl,
                const uint32_t* __restrict__ ix, const uint32_t* __restrict__ iy,
                const uint32_t* __restrict__ iz, const uint8_t* __restrict__ owned,
                uint64_t* __restrict__ keys, uint64_t* __restrict__ vals, long long limit) {
  const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint2 p = far[i];
  uint64_t key = ~uint64_t(0);
  if (owned[p.x]) {
    const int la = lvl[p.x], lb = lvl[p.y], lmax = max(la, lb);
    auto c = [lmax](uint32_t v, int l) { return (long long)(2ull * v + 1) << (lmax - l); };
    const long long dx = c(ix[p.x], la) - c(ix[p.y], lb), dy = c(iy[p.x], la) - c(iy[p.y], lb),
                    dz = c(iz[p.x], la) - c(iz[p.y], lb);
    // a shift beyond the packed range (a deep leaf translated straight from / to a coarse cell: level gaps of
    // fifteen and more) keeps its pair index instead: such pairs sort behind the packed keys, ahead of the
    // unowned ones, and the host groups the few of them into classes (build_far_classes_device)
    if (llabs(dx) >= limit || llabs(dy) >= limit || llabs(dz) >= limit)
      key = uint64_t(1) << 63 | uint64_t(i);
    else
      key = uint64_t(la) << 59 | uint64_t(lb) << 54 | uint64_t(dx + kShiftBias) << 36 |
            uint64_t(dy + kShiftBias) << 18 | uint64_t(dz + kShiftBias);
  }
  keys[i] = key;
  vals[i] = uint64_t(p.x) << 32 | p.y;
}

__global__ void __launch_bounds__(kBlock)
unpack_pairs_kernel(const uint64_t* __restrict__ vals, uint32_t n, uint32_t* __restrict__ src,
                    uint32_t* __restrict__ dst) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dst[i] = uint32_t(vals[i] >> 32);
  src[i] = uint32_t(vals[i]);
}

// ---- bodies ----------------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock)
leaf_bodies_kernel(const uint32_t* __restrict__ leaves, uint32_t n_leaf, const uint8_t* __restrict__ lvl,
                   const uint32_t* __restrict__ ix, const uint32_t* __restrict__ iy,
                   const uint32_t* __restrict__ iz, const uint32_t* __restrict__ body_first,
                   const uint32_t* __restrict__ body_count, const double* __restrict__ xyz,
                   const uint32_t* __restrict__ index, TraversalGeom g, double k, double grid,
                   float4* __restrict__ pos, float4* __restrict__ hi, float4* __restrict__ lo) {
  const uint32_t li = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (li >= n_leaf) return;
  const uint32_t c = leaves[li];
  const double s = g.side[lvl[c]];
  const double cx = __dadd_rn(g.lo[0], __dmul_rn(double(ix[c]) + 0.5, s)),
               cy = __dadd_rn(g.lo[1], __dmul_rn(double(iy[c]) + 0.5, s)),
               cz = __dadd_rn(g.lo[2], __dmul_rn(double(iz[c]) + 0.5, s));
  const double inv = 1.0 / grid;
  for (uint32_t b = body_first[c] + lane; b < body_first[c] + body_count[c]; b += 32) {
    const double* p = xyz + 3 * size_t(index[b]);
    const double v[3] = {__dmul_rn(k, __dsub_rn(p[0], cx)), __dmul_rn(k, __dsub_rn(p[1], cy)),
                         __dmul_rn(k, __dsub_rn(p[2], cz))};
    double h[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) h[a] = __dmul_rn(rint(__dmul_rn(v[a], inv)), grid);
    pos[b] = make_float4(float(v[0]), float(v[1]), float(v[2]), 0.f);
    hi[b] = make_float4(float(h[0]), float(h[1]), float(h[2]), 0.f);
    lo[b] = make_float4(float(v[0] - h[0]), float(v[1] - h[1]), float(v[2] - h[2]), 0.f);
  }
}

__global__ void __launch_bounds__(kBlock)
abs_bodies_kernel(const double* __restrict__ xyz, uint32_t n, double k, float4* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = make_float4(float(k * xyz[3 * size_t(i)]), float(k * xyz[3 * size_t(i) + 1]),
                       float(k * xyz[3 * size_t(i) + 2]), 0.f);
}

TraversalGeom make_geom(const TreeArrays& t, double kmag, double theta, double kd_max) {
  TraversalGeom g{};
  const double sqrt3h = std::sqrt(3.0) / 2;
  for (int a = 0; a < 3; ++a) g.lo[a] = t.lo[a];
  for (int l = 0; l <= kMaxLevel; ++l) {
    g.side[l] = t.side(l);
    g.radius[l] = g.side[l] * sqrt3h;
    g.gated[l] = kd_max > 0 && kmag * (2 * g.radius[l]) > kd_max;
  }
  g.theta = theta;
  return g;
}

}  // namespace

void DeviceCells::upload(const TreeArrays& t, cudaStream_t s) {
  level.upload(t.level, s);
  ix.upload(t.ix, s);
  iy.upload(t.iy, s);
  iz.upload(t.iz, s);
  child_first.upload(t.child_first, s);
  child_count.upload(t.child_count, s);
  body_count.upload(t.body_count, s);
}

void build_tree_device(TreeArrays& t, const double* xyz, size_t n, int ncrit, double leaf_cap,
                       DeviceBuffer<double>& d_xyz, DeviceBuffer<uint32_t>& d_index, cudaStream_t s) {
  if (n == 0) throw Error(HFMM_ERR_CONFIG, "no bodies to enclose");
  if (ncrit < 1) throw Error(HFMM_ERR_CONFIG, "leaf capacity must be at least 1");
  if (n >= (size_t(1) << 31)) throw Error(HFMM_ERR_CONFIG, "body count exceeds 31-bit indexing");
  t = TreeArrays{};
  t.n_bodies = uint32_t(n);
  enclosing_box_host(xyz, n, t.lo, t.width);
  d_xyz.upload(xyz, 3 * n, s);

  // K1
  DeviceBuffer<uint64_t> key_in(n), key_out(n);
  DeviceBuffer<uint32_t> idx_in(n);
  d_index.resize(n);
  const double scale = double(uint64_t(1) << kMaxLevel) / t.width;
  morton_keys_kernel<<<grid_for(n), kBlock, 0, s>>>(d_xyz.get(), uint32_t(n), t.lo[0], t.lo[1], t.lo[2],
                                                    scale, key_in.get(), idx_in.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  TempStorage tmp;
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, key_in.get(), key_out.get(), idx_in.get(), d_index.get(),
                                  int(n), 0, 3 * kMaxLevel, s);
  HFMM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, key_in.get(), key_out.get(),
                                                  idx_in.get(), d_index.get(), int(n), 0, 3 * kMaxLevel, s));
  key_in.release();
  idx_in.release();

  // K2
  size_t cap = std::max<size_t>(4096, n / 4 + 1024);
  DeviceBuffer<uint8_t> level(cap);
  DeviceBuffer<uint32_t> ix(cap), iy(cap), iz(cap), bf(cap), bc(cap), cf(cap), cc(cap), par(cap);
  {
    const uint32_t zero = 0, cnt = uint32_t(n);
    const uint8_t z8 = 0;
    HFMM_CUDA_CHECK(cudaMemcpyAsync(level.get(), &z8, 1, cudaMemcpyHostToDevice, s));
    for (auto* b : {&ix, &iy, &iz, &bf, &cf, &cc, &par})
      HFMM_CUDA_CHECK(cudaMemcpyAsync(b->get(), &zero, 4, cudaMemcpyHostToDevice, s));
    HFMM_CUDA_CHECK(cudaMemcpyAsync(bc.get(), &cnt, 4, cudaMemcpyHostToDevice, s));
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  DeviceBuffer<uint32_t> nchild, offs, bounds, total_dev(2);
  t.level_offset = {0, 1};
  const double sqrt3 = std::sqrt(3.0);
  uint32_t ncells = 1;
  for (int lvl = 0;; ++lvl) {
    const uint32_t c0 = t.level_offset[lvl], c1 = t.level_offset[lvl + 1], m = c1 - c0;
    const bool over_diam = leaf_cap > 0 && t.side(lvl) * sqrt3 > leaf_cap;
    if (nchild.size() < m) {
      nchild.resize(m + m / 2);
      offs.resize(m + m / 2 + 1);
      bounds.resize(size_t(9) * (m + m / 2));
    }
    CellArrays ca{level.get(), ix.get(), iy.get(), iz.get(), bf.get(), bc.get(), cf.get(), cc.get(), par.get()};
    split_count_kernel<<<grid_for(m), kBlock, 0, s>>>(ca, c0, c1, lvl, ncrit, over_diam, key_out.get(),
                                                     nchild.get(), bounds.get());
    HFMM_CUDA_CHECK(cudaGetLastError());
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, nchild.get(), offs.get(), int(m), s);
    HFMM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.get(bytes), bytes, nchild.get(), offs.get(), int(m), s));
    uint32_t last[2];
    HFMM_CUDA_CHECK(cudaMemcpyAsync(&last[0], offs.get() + (m - 1), 4, cudaMemcpyDeviceToHost, s));
    HFMM_CUDA_CHECK(cudaMemcpyAsync(&last[1], nchild.get() + (m - 1), 4, cudaMemcpyDeviceToHost, s));
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
    const uint32_t total = last[0] + last[1];
    if (size_t(c1) + total > cap) {
      cap = size_t(c1) + total;
      grow(level, c1, cap, s);
      for (auto* b : {&ix, &iy, &iz, &bf, &bc, &cf, &cc, &par}) grow(*b, c1, cap, s);
      cap = level.size();
      ca = CellArrays{level.get(), ix.get(), iy.get(), iz.get(), bf.get(), bc.get(), cf.get(), cc.get(), par.get()};
    }
    write_children_kernel<<<grid_for(m), kBlock, 0, s>>>(ca, c0, c1, lvl, nchild.get(), offs.get(), bounds.get());
    HFMM_CUDA_CHECK(cudaGetLastError());
    ncells = c1 + total;
    if (total == 0) {
      t.max_level = lvl;
      break;
    }
    t.level_offset.push_back(ncells);
  }
  // host mirror
  t.level.resize(ncells);
  for (auto* v : {&t.ix, &t.iy, &t.iz, &t.body_first, &t.body_count, &t.child_first, &t.child_count, &t.parent})
    v->resize(ncells);
  t.index.resize(n);
  level.download(t.level.data(), ncells, s);
  ix.download(t.ix.data(), ncells, s);
  iy.download(t.iy.data(), ncells, s);
  iz.download(t.iz.data(), ncells, s);
  bf.download(t.body_first.data(), ncells, s);
  bc.download(t.body_count.data(), ncells, s);
  cf.download(t.child_first.data(), ncells, s);
  cc.download(t.child_count.data(), ncells, s);
  par.download(t.parent.data(), ncells, s);
  d_index.download(t.index.data(), n, s);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  for (uint32_t c = 0; c < ncells; ++c)
    if (t.child_count[c] == 0) {
      t.leaves.push_back(c);
      if (t.level[c] == kMaxLevel && int64_t(t.body_count[c]) > int64_t(ncrit)) ++t.degenerate_leaves;
    }
}

namespace {
// the level-synchronous descent behind the three entry points below
//   census != nullptr : nothing stored, work per target cell and totals (global lists)
//   interest != nullptr: pruned to the nodes that touch an owned subtree
void run_traversal(const TreeArrays& t, const DeviceCells& cells, double kmag, double theta, double kd_max, int grain,
                   const uint8_t* d_interest, TraversalCensus* census, double alpha, DevicePairs& out, cudaStream_t s) {
  if (!(theta > 0) || theta > 1) throw Error(HFMM_ERR_CONFIG, "opening angle must satisfy 0 < theta <= 1");
  const TraversalGeom g = make_geom(t, kmag, theta, kd_max);
  const uint64_t n = t.n_bodies;
  uint64_t cap_far = 16 * n + (1 << 20), cap_near = 8 * n + (1 << 20), cap_front = 16 * n + (1 << 20);
  DeviceBuffer<unsigned long long> counters(4);
  DeviceBuffer<int> overflow(1), level_min;
  DeviceBuffer<unsigned long long> cell_work;
  if (census) {
    cell_work.resize(2 * t.n_cells());
    level_min.resize(1);
  }
  // A list that does not fit is doubled and the walk repeated, as long as the lists (8 bytes per pair, two
  // frontiers) stay within 60 % of the device memory that is free now and within the 31 / 32-bit indexing of the
  // list builders; only then is the configuration given up (a gate that forbids every coarse translation at a
  // size whose all-pairs lists no memory holds — the reference would walk them for hours).
  size_t free_b = 0, total_b = 0;
  HFMM_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
  uint64_t budget = uint64_t(0.6 * double(free_b)) + 8 * (out.far.size() + out.near.size());
  if (const char* e = getenv("HFMM_DEBUG_LIST_BUDGET_MB"))  // tests: reach the limit without filling the device
    if (atoll(e) > 0) budget = std::min<uint64_t>(budget, uint64_t(atoll(e)) << 20);
  for (;;) {
    if (!census) {
      out.far.resize(cap_far);
      out.near.resize(cap_near);
    }
    DeviceBuffer<uint2> fa(cap_front), fb(cap_front);
    counters.zero(s);
    overflow.zero(s);
    CensusSink cs;
    if (census) {
      cell_work.zero(s);
      const int init = kMaxLevel + 1;
      HFMM_CUDA_CHECK(cudaMemcpyAsync(level_min.get(), &init, sizeof(init), cudaMemcpyHostToDevice, s));
      cs.cell_work = cell_work.get();
      cs.level_min = level_min.get();
    }
    const uint2 root = make_uint2(0, 0);
    HFMM_CUDA_CHECK(cudaMemcpyAsync(fa.get(), &root, sizeof(uint2), cudaMemcpyHostToDevice, s));
    unsigned long long n_front = 1;
    uint2 *cur = fa.get(), *nxt = fb.get();
    int ovf = 0;
    const unsigned long long unbounded = ~0ull;
    while (n_front > 0 && !ovf) {
      HFMM_CUDA_CHECK(cudaMemsetAsync(counters.get() + 2, 0, sizeof(unsigned long long), s));
      PairSink next{nxt, counters.get() + 2, cap_front},
          far{census ? nullptr : out.far.get(), counters.get(), census ? unbounded : cap_far},
          near{census ? nullptr : out.near.get(), counters.get() + 1, census ? unbounded : cap_near};
      traversal_kernel<<<grid_for(n_front), kBlock, 0, s>>>(
          cur, n_front, cells.level.get(), cells.ix.get(), cells.iy.get(), cells.iz.get(),
          cells.child_first.get(), cells.child_count.get(), cells.body_count.get(), uint32_t(grain),
          counters.get() + 3, g, next, far, near, overflow.get(), d_interest, cs);
      HFMM_CUDA_CHECK(cudaGetLastError());
      unsigned long long h[4];
      HFMM_CUDA_CHECK(cudaMemcpyAsync(h, counters.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
      HFMM_CUDA_CHECK(cudaMemcpyAsync(&ovf, overflow.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
      HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
      out.n_far = h[0];
      out.n_near = h[1];
      n_front = h[2];
      // the root node opens a task itself when the whole problem fits the grain
      out.tasks = h[3] + (2 * uint64_t(t.n_bodies) <= uint64_t(grain) ? 1 : 0);
      std::swap(cur, nxt);
    }
    if (!ovf) {
      if (census) {
        census->n_far = out.n_far;
        census->n_near = out.n_near;
        census->tasks = out.tasks;
        int lm = kMaxLevel + 1;
        level_min.download(&lm, 1, s);
        std::vector<unsigned long long> work(2 * t.n_cells());
        cell_work.download(work.data(), work.size(), s);
        HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
        census->lmin_src = lm;
        census->lmin_dst = kMaxLevel + 1;
        census->body_pairs = 0;
        for (size_t c = 0; c < t.n_cells(); ++c) {
          if (work[2 * c]) census->lmin_dst = std::min(census->lmin_dst, int(t.level[c]));
          census->body_pairs += work[2 * c + 1];
        }
        // partition_weights_device's model, evaluated in a fixed order: identical on every rank
        census->cell_weight.resize(t.n_cells());
        for (size_t c = 0; c < t.n_cells(); ++c)
          census->cell_weight[c] = double(work[2 * c]) * (alpha < 0 ? kPartitionM2lWeight : alpha * double(t.body_count[c])) +
                                   double(work[2 * c + 1]);
      }
      return;
    }
    if (ovf & 1) cap_far *= 2;
    if (ovf & 2) cap_near *= 2;
    if (ovf & 4) cap_front *= 2;
    const uint64_t need = 8 * ((census ? 0 : cap_far + cap_near) + 2 * cap_front);
    if (getenv("HFMM_SETUP_TRACE"))
      fprintf(stderr, "[hfmm setup] traversal lists grown: far %llu near %llu front %llu (need %llu MB, budget %llu MB)\n",
              (unsigned long long)cap_far, (unsigned long long)cap_near, (unsigned long long)cap_front,
              (unsigned long long)(need >> 20), (unsigned long long)(budget >> 20));
    if (need > budget || cap_far > (uint64_t(1) << 31) || cap_near > (uint64_t(1) << 32))
      // the kd_max gate forbids every coarse translation (k x box >> kd_max) and the lists degenerate towards all
      // pairs of finest-level cells, as they do in the reference
      throw DeviceBuilderLimit(HFMM_ERR_STRUCTURAL,
                               "dual tree traversal: the interaction lists exceed the device memory / 32-bit indexing "
                               "(kd_max too small for this wavenumber and domain?)",
                               false);
  }
}
}  // namespace

void dual_tree_traversal_device(const TreeArrays& t, const DeviceCells& cells, double kmag, double theta,
                                double kd_max, int grain, DevicePairs& out, cudaStream_t s) {
  run_traversal(t, cells, kmag, theta, kd_max, grain, nullptr, nullptr, -1.0, out, s);
}

void dual_tree_census_device(const TreeArrays& t, const DeviceCells& cells, double kmag, double theta,
                             double kd_max, int grain, double alpha, TraversalCensus& out, cudaStream_t s) {
  DevicePairs none;
  run_traversal(t, cells, kmag, theta, kd_max, grain, nullptr, &out, alpha, none, s);
}

void dual_tree_traversal_pruned_device(const TreeArrays& t, const DeviceCells& cells, double kmag, double theta,
                                       double kd_max, const std::vector<uint8_t>& interest, DevicePairs& out,
                                       cudaStream_t s) {
  DeviceBuffer<uint8_t> d_interest;
  d_interest.upload(interest, s);
  // the grain only feeds the task counter, which the census already holds for the global lists
  run_traversal(t, cells, kmag, theta, kd_max, 0, d_interest.get(), nullptr, -1.0, out, s);
}

void far_pair_level_range(const DevicePairs& p, const DeviceCells& cells, int& lmin_dst, int& lmin_src,
                          cudaStream_t s) {
  int h[2] = {kMaxLevel + 1, kMaxLevel + 1};
  if (p.n_far) {
    DeviceBuffer<int> d(2);
    HFMM_CUDA_CHECK(cudaMemcpyAsync(d.get(), h, sizeof(h), cudaMemcpyHostToDevice, s));
    level_range_kernel<<<std::min<uint32_t>(grid_for(p.n_far), 2048), kBlock, 0, s>>>(
        p.far.get(), p.n_far, cells.level.get(), d.get());
    HFMM_CUDA_CHECK(cudaGetLastError());
    d.download(h, 2, s);
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  lmin_dst = h[0];
  lmin_src = h[1];
}

void partition_weights_device(const DevicePairs& p, const DeviceCells& cells,
                              const std::vector<uint32_t>& unit_of_cell, double alpha,
                              std::vector<double>& weight, cudaStream_t s) {
  DeviceBuffer<uint32_t> unit;
  unit.upload(unit_of_cell, s);
  DeviceBuffer<double> w(unit_of_cell.size());
  w.zero(s);
  weights_kernel<<<2048, kBlock, 0, s>>>(p.far.get(), p.n_far, p.near.get(), p.n_near, unit.get(),
                                         cells.body_count.get(), alpha, w.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  weight.resize(unit_of_cell.size());
  w.download(weight.data(), weight.size(), s);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
}

void build_near_lists_device(const DevicePairs& p, const TreeArrays& t, const DeviceCells& cells,
                             const std::vector<uint8_t>& owned, DeviceBuffer<uint32_t>& offset,
                             DeviceBuffer<uint32_t>& split, DeviceBuffer<uint32_t>& src, NearLists& out,
                             cudaStream_t s) {
  const uint32_t nleaf = uint32_t(t.leaves.size());
  if (p.n_near >= (uint64_t(1) << 32)) throw Error(HFMM_ERR_CONFIG, "near pair count exceeds 32-bit indexing");
  std::vector<uint32_t> slot(t.n_cells(), 0xffffffffu);
  for (uint32_t i = 0; i < nleaf; ++i) slot[t.leaves[i]] = i;
  DeviceBuffer<uint32_t> d_slot;
  DeviceBuffer<uint8_t> d_owned;
  d_slot.upload(slot, s);
  d_owned.upload(owned, s);
  DeviceBuffer<uint64_t> keys(std::max<uint64_t>(p.n_near, 1)), sorted(std::max<uint64_t>(p.n_near, 1));
  DeviceBuffer<unsigned long long> totals(4);
  totals.zero(s);
  if (p.n_near) {
    near_keys_kernel<<<grid_for(p.n_near), kBlock, 0, s>>>(
        p.near.get(), p.n_near, cells.level.get(), cells.ix.get(), cells.iy.get(), cells.iz.get(),
        cells.body_count.get(), d_slot.get(), d_owned.get(), t.max_level, keys.get(), totals.get());
    HFMM_CUDA_CHECK(cudaGetLastError());
    TempStorage tmp;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.get(), sorted.get(), int(p.n_near), 0, 64, s);
    HFMM_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(tmp.get(bytes), bytes, keys.get(), sorted.get(),
                                                   int(p.n_near), 0, 64, s));
  }
  unsigned long long h[4];
  totals.download(h, 4, s);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  out.body_pairs = h[0];
  out.owned_body_pairs = h[1];
  out.n_owned_pairs = h[2];
  out.max_r2_lattice = h[3];
  const uint32_t n_owned = uint32_t(h[2]);
  offset.resize(nleaf + 1);
  split.resize(std::max<uint32_t>(nleaf, 1));
  src.resize(std::max<uint32_t>(n_owned, 1));
  near_offsets_kernel<<<grid_for(nleaf + 1), kBlock, 0, s>>>(sorted.get(), n_owned, nleaf, offset.get(), split.get());
  if (n_owned) near_sources_kernel<<<grid_for(n_owned), kBlock, 0, s>>>(sorted.get(), n_owned, src.get());
  DeviceBuffer<unsigned long long> work(std::max<uint32_t>(nleaf, 1));
  near_work_kernel<<<grid_for(nleaf), kBlock, 0, s>>>(offset.get(), src.get(), nleaf, cells.body_count.get(), work.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  std::vector<unsigned long long> hw(nleaf);
  work.download(hw.data(), nleaf, s);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  out.work.assign(hw.begin(), hw.end());
}

void build_far_classes_device(const DevicePairs& p, const TreeArrays& t, const DeviceCells& cells,
                              const std::vector<uint8_t>& owned,
                              DeviceBuffer<uint32_t>& pair_src, DeviceBuffer<uint32_t>& pair_dst,
                              FarClasses& out, cudaStream_t s) {
  out = FarClasses{};
  if (p.n_far == 0) return;
  if (p.n_far >= (uint64_t(1) << 31)) throw Error(HFMM_ERR_CONFIG, "M2L pair count exceeds 31-bit indexing");
  const int n = int(p.n_far);
  DeviceBuffer<uint8_t> d_owned;
  d_owned.upload(owned, s);
  DeviceBuffer<uint64_t> k_in(n), k_out(n), v_in(n), v_out(n);
  // HFMM_DEBUG_SHIFT_LIMIT (tests): shifts from this size on take the unpacked path although they would fit
  const char* dbg = getenv("HFMM_DEBUG_SHIFT_LIMIT");
  const long long dbg_limit = dbg ? atoll(dbg) : 0;
  const long long limit = dbg_limit > 0 && dbg_limit < kShiftBias ? dbg_limit : (long long)kShiftBias;
  far_keys_kernel<<<grid_for(n), kBlock, 0, s>>>(p.far.get(), p.n_far, cells.level.get(), cells.ix.get(),
                                                 cells.iy.get(), cells.iz.get(), d_owned.get(), k_in.get(),
                                                 v_in.get(), limit);
  HFMM_CUDA_CHECK(cudaGetLastError());
  TempStorage tmp;
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k_in.get(), k_out.get(), v_in.get(), v_out.get(), n, 0, 64, s);
  HFMM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, k_in.get(), k_out.get(), v_in.get(),
                                                  v_out.get(), n, 0, 64, s));
  k_in.release();
  v_in.release();
  DeviceBuffer<uint64_t> uniq(n);
  DeviceBuffer<int> counts(n), nruns(1);
  cub::DeviceRunLengthEncode::Encode(nullptr, bytes, k_out.get(), uniq.get(), counts.get(), nruns.get(), n, s);
  HFMM_CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(tmp.get(bytes), bytes, k_out.get(), uniq.get(),
                                                     counts.get(), nruns.get(), n, s));
  int h_runs = 0;
  nruns.download(&h_runs, 1, s);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  std::vector<uint64_t> hk(h_runs);
  std::vector<int> hc(h_runs);
  uniq.download(hk.data(), h_runs, s);
  counts.download(hc.data(), h_runs, s);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  uint64_t n_unpacked = 0;
  for (int r = 0; r < h_runs; ++r) {
    if (hk[r] == ~uint64_t(0)) continue;  // pairs of targets other ranks own
    if (hk[r] >> 63) {                    // shift beyond the packed range: one run per pair, grouped below
      n_unpacked += uint64_t(hc[r]);
      continue;
    }
    out.lt.push_back(int16_t(hk[r] >> 59));
    out.ls.push_back(int16_t((hk[r] >> 54) & 31));
    out.dx.push_back(int32_t((hk[r] >> 36) & 0x3ffff) - kShiftBias);
    out.dy.push_back(int32_t((hk[r] >> 18) & 0x3ffff) - kShiftBias);
    out.dz.push_back(int32_t(hk[r] & 0x3ffff) - kShiftBias);
    out.count.push_back(uint32_t(hc[r]));
    out.n_owned_pairs += uint64_t(hc[r]);
  }
  if (n_unpacked) {
    // the unpacked pairs sit at positions [n_owned_pairs, n_owned_pairs + n_unpacked) of the sorted payloads, in
    // pair-index order: classify them on the host with the kernel's own arithmetic, sort them by class and put
    // them back, so that every class is again one contiguous range of the pair arrays
    std::vector<uint64_t> pay(n_unpacked);
    HFMM_CUDA_CHECK(cudaMemcpyAsync(pay.data(), v_out.get() + out.n_owned_pairs, n_unpacked * sizeof(uint64_t),
                                    cudaMemcpyDeviceToHost, s));
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
    struct Unpacked {
      int16_t lt, ls;
      int64_t dx, dy, dz;
      uint64_t pay;
    };
    std::vector<Unpacked> u(n_unpacked);
    for (uint64_t i = 0; i < n_unpacked; ++i) {
      const uint32_t a = uint32_t(pay[i] >> 32), b = uint32_t(pay[i]);
      const int la = t.level[a], lb = t.level[b], lmax = std::max(la, lb);
      auto c = [lmax](uint32_t v, int l) { return int64_t(2ull * v + 1) << (lmax - l); };
      u[i] = {int16_t(la), int16_t(lb), c(t.ix[a], la) - c(t.ix[b], lb), c(t.iy[a], la) - c(t.iy[b], lb),
              c(t.iz[a], la) - c(t.iz[b], lb), pay[i]};
      if (std::llabs(u[i].dx) > INT32_MAX || std::llabs(u[i].dy) > INT32_MAX || std::llabs(u[i].dz) > INT32_MAX)
        throw Error(HFMM_ERR_INTERNAL, "M2L lattice shift beyond 32 bits");  // needs a level gap of 30: kMaxLevel is 21
    }
    auto cls = [](const Unpacked& x) { return std::make_tuple(x.lt, x.ls, x.dx, x.dy, x.dz); };
    std::stable_sort(u.begin(), u.end(), [&](const Unpacked& x, const Unpacked& y) { return cls(x) < cls(y); });
    for (uint64_t i = 0; i < n_unpacked; ++i) {
      pay[i] = u[i].pay;
      if (i && cls(u[i]) == cls(u[i - 1])) {
        ++out.count.back();
      } else {
        out.lt.push_back(u[i].lt);
        out.ls.push_back(u[i].ls);
        out.dx.push_back(int32_t(u[i].dx));
        out.dy.push_back(int32_t(u[i].dy));
        out.dz.push_back(int32_t(u[i].dz));
        out.count.push_back(1);
      }
    }
    HFMM_CUDA_CHECK(cudaMemcpyAsync(v_out.get() + out.n_owned_pairs, pay.data(), n_unpacked * sizeof(uint64_t),
                                    cudaMemcpyHostToDevice, s));
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
    out.n_owned_pairs += n_unpacked;
  }
  const uint32_t no = uint32_t(out.n_owned_pairs);
  pair_src.resize(std::max<uint32_t>(no, 1));
  pair_dst.resize(std::max<uint32_t>(no, 1));
  if (no) unpack_pairs_kernel<<<grid_for(no), kBlock, 0, s>>>(v_out.get(), no, pair_src.get(), pair_dst.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
}

void build_body_arrays_device(const TreeArrays& t, const DeviceBuffer<double>& d_xyz,
                              const DeviceBuffer<uint32_t>& d_index, double k, double grid,
                              DeviceBuffer<float4>& pos, DeviceBuffer<float4>& hi, DeviceBuffer<float4>& lo,
                              DeviceBuffer<float4>& abs_pos, cudaStream_t s) {
  const uint32_t n = t.n_bodies, nleaf = uint32_t(t.leaves.size());
  pos.resize(n);
  hi.resize(n);
  lo.resize(n);
  abs_pos.resize(n);
  DeviceBuffer<uint32_t> leaves, ix, iy, iz, bf, bc;
  DeviceBuffer<uint8_t> level;
  leaves.upload(t.leaves, s);
  level.upload(t.level, s);
  ix.upload(t.ix, s);
  iy.upload(t.iy, s);
  iz.upload(t.iz, s);
  bf.upload(t.body_first, s);
  bc.upload(t.body_count, s);
  const TraversalGeom g = make_geom(t, 0, 1, 0);
  leaf_bodies_kernel<<<grid_for(uint64_t(nleaf) * 32), kBlock, 0, s>>>(
      leaves.get(), nleaf, level.get(), ix.get(), iy.get(), iz.get(), bf.get(), bc.get(), d_xyz.get(),
      d_index.get(), g, k, grid, pos.get(), hi.get(), lo.get());
  abs_bodies_kernel<<<grid_for(n), kBlock, 0, s>>>(d_xyz.get(), n, k, abs_pos.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
}

namespace {
__global__ void __launch_bounds__(kBlock)
regroup_kernel(const uint32_t* __restrict__ seg_new, const uint32_t* __restrict__ seg_old,
               const uint32_t* __restrict__ seg_cls, uint32_t n_seg, uint32_t n,
               const uint32_t* __restrict__ src_in, const uint32_t* __restrict__ dst_in,
               uint32_t* __restrict__ src_out, uint32_t* __restrict__ dst_out, uint32_t* __restrict__ cls_out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t lo = 0, hi = n_seg;  // last segment with seg_new <= i
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (seg_new[mid] <= i) lo = mid;
    else hi = mid;
  }
  const uint32_t from = seg_old[lo] + (i - seg_new[lo]);
  src_out[i] = src_in[from];
  dst_out[i] = dst_in[from];
  cls_out[i] = seg_cls[lo];
}
}  // namespace

namespace {
__global__ void iota_kernel(uint32_t n, uint32_t* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = i;
}
}  // namespace

uint32_t build_ordered_reduce_device(const uint32_t* pair_dst, uint64_t begin, uint32_t n,
                                     DeviceBuffer<uint32_t>& perm, DeviceBuffer<uint32_t>& seg_dst,
                                     DeviceBuffer<uint32_t>& seg_begin, cudaStream_t s) {
  if (!n) return 0;
  DeviceBuffer<uint32_t> idx(n), keys(n), uniq(n);
  DeviceBuffer<int> counts(n), nruns(1);
  perm.resize(n);
  iota_kernel<<<grid_for(n), kBlock, 0, s>>>(n, idx.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  TempStorage tmp;
  size_t bytes = 0;
  // LSD radix sort: stable, so the pairs of one destination stay in pair order
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, pair_dst + begin, keys.get(), idx.get(), perm.get(), int(n), 0, 32, s);
  HFMM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, pair_dst + begin, keys.get(), idx.get(),
                                                  perm.get(), int(n), 0, 32, s));
  cub::DeviceRunLengthEncode::Encode(nullptr, bytes, keys.get(), uniq.get(), counts.get(), nruns.get(), int(n), s);
  HFMM_CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(tmp.get(bytes), bytes, keys.get(), uniq.get(), counts.get(),
                                                     nruns.get(), int(n), s));
  int h_runs = 0;
  nruns.download(&h_runs, 1, s);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  seg_dst.resize(size_t(h_runs));
  seg_begin.resize(size_t(h_runs) + 1);
  HFMM_CUDA_CHECK(cudaMemcpyAsync(seg_dst.get(), uniq.get(), size_t(h_runs) * 4, cudaMemcpyDeviceToDevice, s));
  DeviceBuffer<int> offs(size_t(h_runs) + 1);
  // exclusive sum over h_runs + 1 entries: the last one is the total (counts has n >= h_runs + 1 slots
  // unless every pair has its own destination; pad through a copy)
  DeviceBuffer<int> padded(size_t(h_runs) + 1);
  padded.zero(s);
  HFMM_CUDA_CHECK(cudaMemcpyAsync(padded.get(), counts.get(), size_t(h_runs) * 4, cudaMemcpyDeviceToDevice, s));
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, padded.get(), offs.get(), h_runs + 1, s);
  HFMM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.get(bytes), bytes, padded.get(), offs.get(), h_runs + 1, s));
  HFMM_CUDA_CHECK(cudaMemcpyAsync(seg_begin.get(), offs.get(), (size_t(h_runs) + 1) * 4, cudaMemcpyDeviceToDevice, s));
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  return uint32_t(h_runs);
}

void regroup_pairs_device(const std::vector<uint32_t>& seg_new, const std::vector<uint32_t>& seg_old,
                          const std::vector<uint32_t>& seg_cls, uint64_t n_pairs,
                          DeviceBuffer<uint32_t>& pair_src, DeviceBuffer<uint32_t>& pair_dst,
                          DeviceBuffer<uint32_t>& pair_cls, cudaStream_t s) {
  pair_cls.resize(std::max<uint64_t>(n_pairs, 1));
  if (!n_pairs) return;
  DeviceBuffer<uint32_t> d_new, d_old, d_cls, src_out(n_pairs), dst_out(n_pairs);
  d_new.upload(seg_new, s);
  d_old.upload(seg_old, s);
  d_cls.upload(seg_cls, s);
  regroup_kernel<<<grid_for(n_pairs), kBlock, 0, s>>>(d_new.get(), d_old.get(), d_cls.get(), uint32_t(seg_old.size()),
                                                      uint32_t(n_pairs), pair_src.get(), pair_dst.get(), src_out.get(),
                                                      dst_out.get(), pair_cls.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  pair_src = std::move(src_out);
  pair_dst = std::move(dst_out);
}

}  // namespace hfmm_b200
