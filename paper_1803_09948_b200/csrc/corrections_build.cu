// corrections_build.cu — the BIE operator's correction arrays built on the device (sm_100a).
//
// Replaces the reference's setup loops build_patch_blocks (src/solver.cpp:80-128) and
// build_near_corrections (src/solver.cpp:132-230): the same-patch blocks with their Duffy-integrated
// self terms and LU factors, the near lists (samples of other patches inside the per-source
// threshold) and the difference between the re-integrated basis function and the plain point
// contribution for every listed pair.  All of it is FP64, evaluated in the reference's operation
// order (this file is compiled with -fmad=false: no contraction, so the geometric decisions —
// cell coordinates, R^2 <= thr^2 — fall exactly as they do on the host); only exp / sin / cos differ
// from glibc by an ulp.  The quadrature and interpolation tables are the caller's (geometry.cpp's
// rules), passed through hfmm_correction_rules.
//
//   K1  patch diameters / thresholds, sample positions (map_to_physical of the interpolation nodes)
//   K2  cell keys floor(x / h) of the hash grid, radix sort (key, sample)
//   K3  per target: scan the 27 neighbour cells (binary search in the sorted keys), count, fill;
//       segmented sort of every list (the reference sorts each list ascending)
//   K4  one thread per listed pair: Gauss sweep over the source patch for the pair's own basis
//       function, minus the plain contribution
//   K5  one thread per (patch, row): plain same-patch terms and the Duffy rule centred on the row's
//       node;  K6  one thread per patch: LU with partial pivoting (solver.cpp:45-62)
// The FP64 results stay on the device for hfmm_cuda_get_corrections; FP32 copies are installed as
// the handle's corrections, exactly what hfmm_cuda_set_corrections would have uploaded.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "device_utils.cuh"
#include "engine.hpp"

namespace hfmm_b200 {

namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;
constexpr int kMaxBasis = 12;  // LagrangeBasis: 3, 6 or 12 functions (geometry.hpp:38-40)

struct D3 {
  double x, y, z;
};
struct Z {
  double re, im;
};

// geometry.cpp:22-27, 40-45
__device__ __forceinline__ D3 map_to_physical(const double* __restrict__ node, double z, double e) {
  const double l1 = 1.0 - z - e, l2 = z, l3 = e;
  const double n[6] = {l1 * (2 * l1 - 1), l2 * (2 * l2 - 1), l3 * (2 * l3 - 1), 4 * l1 * l2, 4 * l2 * l3, 4 * l3 * l1};
  D3 r{0, 0, 0};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    r.x += n[k] * node[3 * k];
    r.y += n[k] * node[3 * k + 1];
    r.z += n[k] * node[3 * k + 2];
  }
  return r;
}
__device__ __forceinline__ double norm2(D3 a, D3 b) {
  const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  return dx * dx + dy * dy + dz * dz;
}
// kernel.hpp:16-23
__device__ __forceinline__ Z green(D3 a, D3 b, double kr, double ki) {
  const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  const double R = sqrt(dx * dx + dy * dy + dz * dz);
  const double amp = exp(-ki * R) / (4.0 * kPi * R);
  const double ph = kr * R;
  double s, c;
  sincos(ph, &s, &c);
  return Z{amp * c, amp * s};
}
// solver.cpp:13-17
__device__ __forceinline__ uint64_t cell_key(long long cx, long long cy, long long cz) {
  const uint64_t mask = (1ull << 21) - 1;
  return ((uint64_t(cx) & mask) << 42) | ((uint64_t(cy) & mask) << 21) | (uint64_t(cz) & mask);
}

// K1: geometry.cpp:9-20 (diameter), solver.cpp:40-43 (threshold), solver.cpp:283-294 (samples)
__global__ void patch_geometry_kernel(const double* __restrict__ nodes, const double* __restrict__ sample_ref,
                                      int ni, uint64_t n_patches, double near_patch_distance,
                                      double* __restrict__ thr, double* __restrict__ touch2,
                                      double* __restrict__ xyz) {
  const uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (p >= n_patches) return;
  const double* node = nodes + 18 * p;
  D3 c{0, 0, 0};
  for (int k = 0; k < 6; ++k) {
    c.x += node[3 * k];
    c.y += node[3 * k + 1];
    c.z += node[3 * k + 2];
  }
  c.x /= 6.0;
  c.y /= 6.0;
  c.z /= 6.0;
  double r = 0;
  for (int k = 0; k < 6; ++k) {
    const double dx = node[3 * k] - c.x, dy = node[3 * k + 1] - c.y, dz = node[3 * k + 2] - c.z;
    r = fmax(r, sqrt(dx * dx + dy * dy + dz * dz));
  }
  thr[p] = near_patch_distance < 0 ? 2.0 * (2.0 * r) : near_patch_distance;
  touch2[p] = (0.1 * (2.0 * r)) * (0.1 * (2.0 * r));  // evaluate_scattered_field's touch radius (solver.cpp:399-403)
  for (int j = 0; j < ni; ++j) {
    const D3 v = map_to_physical(node, sample_ref[2 * j], sample_ref[2 * j + 1]);
    xyz[3 * (p * ni + j)] = v.x;
    xyz[3 * (p * ni + j) + 1] = v.y;
    xyz[3 * (p * ni + j) + 2] = v.z;
  }
}

// K2
__global__ void cell_keys_kernel(const double* __restrict__ xyz, uint32_t n, double h, uint64_t* __restrict__ key,
                                 uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = cell_key((long long)floor(xyz[3 * i] / h), (long long)floor(xyz[3 * i + 1] / h),
                    (long long)floor(xyz[3 * i + 2] / h));
  idx[i] = i;
}

// K3: solver.cpp:159-179.  FILL = false counts, FILL = true writes the sources (unsorted)
template <bool FILL>
__global__ void near_lists_kernel(const double* __restrict__ xyz, const double* __restrict__ thr,
                                  const uint64_t* __restrict__ key, const uint32_t* __restrict__ idx, uint32_t n,
                                  int ni, double h, uint32_t* __restrict__ count, const uint32_t* __restrict__ offset,
                                  uint32_t* __restrict__ source) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  const D3 t{xyz[3 * m], xyz[3 * m + 1], xyz[3 * m + 2]};
  const long long cx = (long long)floor(t.x / h), cy = (long long)floor(t.y / h), cz = (long long)floor(t.z / h);
  const uint32_t my_patch = m / uint32_t(ni);
  uint32_t found = 0;
  const uint32_t base = FILL ? offset[m] : 0;
  for (long long dx = -1; dx <= 1; ++dx)
    for (long long dy = -1; dy <= 1; ++dy)
      for (long long dz = -1; dz <= 1; ++dz) {
        const uint64_t k = cell_key(cx + dx, cy + dy, cz + dz);
        uint32_t lo = 0, hi = n;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (key[mid] < k) lo = mid + 1;
          else hi = mid;
        }
        for (uint32_t e = lo; e < n && key[e] == k; ++e) {
          const uint32_t s = idx[e];
          const uint32_t sp = s / uint32_t(ni);
          if (sp == my_patch) continue;
          const double r2 = norm2(t, D3{xyz[3 * s], xyz[3 * s + 1], xyz[3 * s + 2]});
          if (r2 == 0.0) continue;
          const double th = thr[sp];
          if (th > 0.0 && r2 <= th * th) {
            if (FILL) source[base + found] = s;
            ++found;
          }
        }
      }
  if (!FILL) count[m] = found;
}

__global__ void entry_rows_kernel(const uint32_t* __restrict__ offset, uint32_t n, uint32_t* __restrict__ row) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  for (uint32_t e = offset[m]; e < offset[m + 1]; ++e) row[e] = m;
}

// K4: solver.cpp:194-230, one listed pair per thread (the sweep over the source patch is repeated
// for each listed basis function of it: the sums are the reference's, term for term)
__global__ void near_delta_kernel(const double* __restrict__ nodes, const double* __restrict__ xyz,
                                  const double* __restrict__ far_weight, const double* __restrict__ near_pts,
                                  const double* __restrict__ near_basis, int near_npts, int ni, double kr,
                                  double ki, const uint32_t* __restrict__ row, const uint32_t* __restrict__ source,
                                  uint64_t nnz, Z* __restrict__ delta, int* __restrict__ degenerate) {
  const uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (e >= nnz) return;
  const uint32_t m = row[e], s = source[e], sp = s / uint32_t(ni), b = s % uint32_t(ni);
  const D3 t{xyz[3 * m], xyz[3 * m + 1], xyz[3 * m + 2]};
  const double* node = nodes + 18 * size_t(sp);
  Z acc{0, 0};
  for (int q = 0; q < near_npts; ++q) {
    const D3 rp = map_to_physical(node, near_pts[3 * q], near_pts[3 * q + 1]);
    const Z g = green(t, rp, kr, ki);
    const double wl = near_pts[3 * q + 2] * near_basis[q * ni + b];
    acc.re += wl * g.re;
    acc.im += wl * g.im;
  }
  if (!(acc.re == acc.re) || !(acc.im == acc.im)) *degenerate = 1;
  const Z plain = green(t, D3{xyz[3 * s], xyz[3 * s + 1], xyz[3 * s + 2]}, kr, ki);
  const double fw = far_weight[b];
  delta[e] = Z{acc.re - plain.re * fw, acc.im - plain.im * fw};
}

// K5: solver.cpp:99-121, one (patch, row j) per thread
__global__ void patch_rows_kernel(const double* __restrict__ nodes, const double* __restrict__ sample_ref,
                                  const double* __restrict__ far_weight, const int* __restrict__ self_first,
                                  const double* __restrict__ self_pts, const double* __restrict__ self_basis,
                                  int ni, uint64_t n_patches, bool self_terms, double kr, double ki,
                                  Z* __restrict__ block, Z* __restrict__ lu) {
  const uint64_t id = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (id >= n_patches * uint64_t(ni)) return;
  const uint64_t p = id / uint64_t(ni);
  const int j = int(id % uint64_t(ni));
  const double* node = nodes + 18 * p;
  const D3 obs = map_to_physical(node, sample_ref[2 * j], sample_ref[2 * j + 1]);
  Z out[kMaxBasis], row[kMaxBasis];
  for (int n = 0; n < ni; ++n) {
    out[n] = Z{0, 0};
    row[n] = Z{0, 0};
    const D3 sn = map_to_physical(node, sample_ref[2 * n], sample_ref[2 * n + 1]);
    if (norm2(obs, sn) > 0.0) {
      const Z g = green(obs, sn, kr, ki);
      out[n] = Z{0.0 - g.re * far_weight[n], 0.0 - g.im * far_weight[n]};
    }
  }
  if (self_terms) {
    for (int q = self_first[j]; q < self_first[j + 1]; ++q) {
      const D3 rp = map_to_physical(node, self_pts[3 * q], self_pts[3 * q + 1]);
      if (norm2(obs, rp) == 0.0) continue;
      const Z g = green(obs, rp, kr, ki);
      const double w = self_pts[3 * q + 2];
      for (int n = 0; n < ni; ++n) {
        const double wl = w * self_basis[size_t(q) * ni + n];
        row[n].re += wl * g.re;
        row[n].im += wl * g.im;
      }
    }
    for (int n = 0; n < ni; ++n) {
      lu[id * ni + n] = row[n];
      out[n].re += row[n].re;
      out[n].im += row[n].im;
    }
  }
  for (int n = 0; n < ni; ++n) block[id * ni + n] = out[n];
}

__device__ __forceinline__ Z zmul(Z a, Z b) { return Z{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
// complex quotient, scaled as libgcc's __divdc3 (the host code divides std::complex<double>)
__device__ __forceinline__ Z zdiv(Z a, Z b) {
  if (fabs(b.re) < fabs(b.im)) {
    const double ratio = b.re / b.im, denom = b.re * ratio + b.im;
    return Z{(a.re * ratio + a.im) / denom, (a.im * ratio - a.re) / denom};
  }
  const double ratio = b.im / b.re, denom = b.im * ratio + b.re;
  return Z{(a.im * ratio + a.re) / denom, (a.im - a.re * ratio) / denom};
}

// K6: solver.cpp:45-62
__global__ void block_lu_kernel(Z* __restrict__ lu, int* __restrict__ piv, int ni, uint64_t n_patches,
                                int* __restrict__ singular) {
  const uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (p >= n_patches) return;
  Z* a = lu + p * uint64_t(ni) * ni;
  int* pv = piv + p * ni;
  for (int c = 0; c < ni; ++c) {
    int best = c;
    for (int r = c + 1; r < ni; ++r)
      if (hypot(a[r * ni + c].re, a[r * ni + c].im) > hypot(a[best * ni + c].re, a[best * ni + c].im)) best = r;
    pv[c] = best;
    if (best != c)
      for (int m = 0; m < ni; ++m) {
        const Z t = a[c * ni + m];
        a[c * ni + m] = a[best * ni + m];
        a[best * ni + m] = t;
      }
    if (a[c * ni + c].re == 0.0 && a[c * ni + c].im == 0.0) {
      *singular = 1;
      return;
    }
    for (int r = c + 1; r < ni; ++r) {
      a[r * ni + c] = zdiv(a[r * ni + c], a[c * ni + c]);
      for (int m = c + 1; m < ni; ++m) {
        const Z t = zmul(a[r * ni + c], a[c * ni + m]);
        a[r * ni + m].re -= t.re;
        a[r * ni + m].im -= t.im;
      }
    }
  }
}

__global__ void sample_weights_kernel(const double* __restrict__ w, int ni, uint32_t n, float* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = float(w[i % uint32_t(ni)]);
}
// largest |k x_sample - (k x)_tree| relative to max(1, |k x|): the patches must describe the points of set_points
__global__ void sample_mismatch_kernel(const double* __restrict__ xyz, const float4* __restrict__ tree_kx, uint32_t n,
                                       double k, double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 t = tree_kx[i];
  const double ax = k * xyz[3 * i], ay = k * xyz[3 * i + 1], az = k * xyz[3 * i + 2];
  const double d = fmax(fabs(ax - double(t.x)), fmax(fabs(ay - double(t.y)), fabs(az - double(t.z)))) /
                   fmax(1.0, fmax(fabs(ax), fmax(fabs(ay), fabs(az))));
  if (d > 0) atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(d));
}

inline unsigned blocks_for(uint64_t n, int threads) { return unsigned((n + threads - 1) / threads); }

}  // namespace

struct Engine::CorrectionStore {
  // FP64 results, as the reference's DiscreteSystem holds them
  DeviceBuffer<double> xyz, thr;
  DeviceBuffer<Z> patch_block, block_lu, near_delta;
  DeviceBuffer<int> block_piv;
  DeviceBuffer<uint32_t> near_offset, near_source;
  uint64_t nnz = 0;
  int ni = 0;
  bool self_terms = false;
};

void Engine::release_correction_store() { corrections64_.reset(); }

void Engine::build_corrections(const hfmm_correction_rules& r, uint64_t* nnz_out) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const int ni = r.basis_count;
  if (ni < 1 || ni > kMaxBasis) throw Error(HFMM_ERR_CONFIG, "basis_count must lie in 1..12");
  if (r.mode < 0 || r.mode > 2) throw Error(HFMM_ERR_CONFIG, "mode must be 0 (none), 1 (self_only) or 2 (self_near)");
  const uint64_t n = r.n_patches * uint64_t(ni);
  if (n != tree_.n_bodies) throw Error(HFMM_ERR_CONFIG, "n_patches x basis_count differs from the point count of set_points");
  if (!r.nodes || !r.sample_ref || !r.far_weight) throw Error(HFMM_ERR_CONFIG, "null geometry / basis arrays");
  const bool self_terms = r.mode != 0, near_terms = r.mode == 2;
  if (self_terms && (!r.self_npts || !r.self_pts || !r.self_basis)) throw Error(HFMM_ERR_CONFIG, "null self rule");
  if (near_terms && (r.near_npts < 1 || !r.near_pts || !r.near_basis)) throw Error(HFMM_ERR_CONFIG, "null near rule");
  const cudaStream_t s = stream_;
  const double kr = cfg_.wave_r, ki = cfg_.wave_i;

  auto store = std::make_shared<CorrectionStore>();
  store->ni = ni;
  store->self_terms = self_terms;
  DeviceBuffer<double> d_nodes, d_ref, d_fw, d_near_pts, d_near_basis, d_self_pts, d_self_basis;
  DeviceBuffer<int> d_self_first, d_flag(2);
  d_nodes.upload(r.nodes, size_t(r.n_patches) * 18, s);
  d_ref.upload(r.sample_ref, size_t(ni) * 2, s);
  d_fw.upload(r.far_weight, size_t(ni), s);
  d_flag.zero(s);
  std::vector<int> self_first(ni + 1, 0);
  if (self_terms) {
    for (int j = 0; j < ni; ++j) {
      if (r.self_npts[j] < 0) throw Error(HFMM_ERR_CONFIG, "negative self rule size");
      self_first[j + 1] = self_first[j] + r.self_npts[j];
    }
    d_self_pts.upload(r.self_pts, size_t(self_first[ni]) * 3, s);
    d_self_basis.upload(r.self_basis, size_t(self_first[ni]) * ni, s);
  }
  d_self_first.upload(self_first, s);

  // K1
  store->xyz.resize(n * 3);
  store->thr.resize(std::max<uint64_t>(r.n_patches, 1));
  touch2_.resize(std::max<uint64_t>(r.n_patches, 1));
  touch_ni_ = uint32_t(ni);
  patch_geometry_kernel<<<blocks_for(r.n_patches, 128), 128, 0, s>>>(d_nodes.get(), d_ref.get(), ni, r.n_patches,
                                                                      r.near_patch_distance, store->thr.get(),
                                                                      touch2_.get(), store->xyz.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  {  // the samples must be the points the tree was built on (caller order; body_abs_ holds k x in FP32)
    DeviceBuffer<double> d_diff(1);
    d_diff.zero(s);
    sample_mismatch_kernel<<<blocks_for(n, 256), 256, 0, s>>>(store->xyz.get(), body_abs_.get(), uint32_t(n),
                                                              cfg_.wave_r, d_diff.get());
    HFMM_CUDA_CHECK(cudaGetLastError());
    double diff = 0;
    d_diff.download(&diff, 1, s);
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
    if (!(diff <= 1e-5))
      throw Error(HFMM_ERR_CONFIG, "sample positions of the patches differ from the points given to set_points");
  }

  // K5 + K6
  store->patch_block.resize(n * ni);
  if (self_terms) {
    store->block_lu.resize(n * ni);
    store->block_piv.resize(n);
  }
  patch_rows_kernel<<<blocks_for(n, 64), 64, 0, s>>>(d_nodes.get(), d_ref.get(), d_fw.get(), d_self_first.get(),
                                                     d_self_pts.get(), d_self_basis.get(), ni, r.n_patches, self_terms,
                                                     kr, ki, store->patch_block.get(), store->block_lu.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  if (self_terms) {
    block_lu_kernel<<<blocks_for(r.n_patches, 64), 64, 0, s>>>(store->block_lu.get(), store->block_piv.get(), ni,
                                                               r.n_patches, d_flag.get());
    HFMM_CUDA_CHECK(cudaGetLastError());
  }

  // K2 + K3 + K4
  store->near_offset.resize(n + 1);
  store->near_offset.zero(s);
  uint64_t nnz = 0;
  if (near_terms) {
    std::vector<double> thr(r.n_patches);
    store->thr.download(thr.data(), thr.size(), s);
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
    double h = 0;
    for (double t : thr) h = std::max(h, t);
    if (h > 0.0) {
      DeviceBuffer<uint64_t> key(n), key_sorted(n);
      DeviceBuffer<uint32_t> idx(n), idx_sorted(n), count(n + 1);
      cell_keys_kernel<<<blocks_for(n, 256), 256, 0, s>>>(store->xyz.get(), uint32_t(n), h, key.get(), idx.get());
      HFMM_CUDA_CHECK(cudaGetLastError());
      size_t tmp_bytes = 0;
      HFMM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key.get(), key_sorted.get(), idx.get(),
                                                      idx_sorted.get(), int(n), 0, 63, s));
      DeviceBuffer<unsigned char> tmp(tmp_bytes);
      HFMM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, key.get(), key_sorted.get(), idx.get(),
                                                      idx_sorted.get(), int(n), 0, 63, s));
      count.zero(s);
      near_lists_kernel<false><<<blocks_for(n, 128), 128, 0, s>>>(store->xyz.get(), store->thr.get(), key_sorted.get(),
                                                                 idx_sorted.get(), uint32_t(n), ni, h, count.get(),
                                                                 nullptr, nullptr);
      HFMM_CUDA_CHECK(cudaGetLastError());
      size_t scan_bytes = 0;
      HFMM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, count.get(), store->near_offset.get(), int(n + 1), s));
      DeviceBuffer<unsigned char> scan_tmp(scan_bytes);
      HFMM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scan_tmp.get(), scan_bytes, count.get(), store->near_offset.get(),
                                                    int(n + 1), s));
      uint32_t total = 0;
      HFMM_CUDA_CHECK(cudaMemcpyAsync(&total, store->near_offset.get() + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
      // the reference's CSR offsets are 32-bit as well (solver.hpp: std::vector<std::uint32_t>)
      nnz = total;
      if (nnz) {
        DeviceBuffer<uint32_t> unsorted(nnz), row(nnz);
        store->near_source.resize(nnz);
        store->near_delta.resize(nnz);
        near_lists_kernel<true><<<blocks_for(n, 128), 128, 0, s>>>(store->xyz.get(), store->thr.get(), key_sorted.get(),
                                                                  idx_sorted.get(), uint32_t(n), ni, h, nullptr,
                                                                  store->near_offset.get(), unsorted.get());
        HFMM_CUDA_CHECK(cudaGetLastError());
        size_t seg_bytes = 0;
        HFMM_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(nullptr, seg_bytes, unsorted.get(), store->near_source.get(),
                                                           int64_t(nnz), int64_t(n), store->near_offset.get(),
                                                           store->near_offset.get() + 1, s));
        DeviceBuffer<unsigned char> seg_tmp(seg_bytes);
        HFMM_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(seg_tmp.get(), seg_bytes, unsorted.get(),
                                                           store->near_source.get(), int64_t(nnz), int64_t(n),
                                                           store->near_offset.get(), store->near_offset.get() + 1, s));
        entry_rows_kernel<<<blocks_for(n, 128), 128, 0, s>>>(store->near_offset.get(), uint32_t(n), row.get());
        HFMM_CUDA_CHECK(cudaGetLastError());
        DeviceBuffer<double> d_np, d_nb;
        d_np.upload(r.near_pts, size_t(r.near_npts) * 3, s);
        d_nb.upload(r.near_basis, size_t(r.near_npts) * ni, s);
        near_delta_kernel<<<blocks_for(nnz, 128), 128, 0, s>>>(d_nodes.get(), store->xyz.get(), d_fw.get(), d_np.get(),
                                                               d_nb.get(), r.near_npts, ni, kr, ki, row.get(),
                                                               store->near_source.get(), nnz, store->near_delta.get(),
                                                               d_flag.get() + 1);
        HFMM_CUDA_CHECK(cudaGetLastError());
        HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
      }
    }
  }
  int flags[2] = {0, 0};
  d_flag.download(flags, 2, s);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  if (flags[0]) throw Error(HFMM_ERR_SINGULAR, "patch self block is singular");  // solver.cpp:55-56
  if (flags[1]) throw Error(HFMM_ERR_STRUCTURAL, "near re-integration produced a non-finite value (degenerate patch)");
  store->nnz = nnz;

  // install the arrays as the handle's corrections (what set_corrections would upload; FP64 like there)
  ni_ = ni;
  far_weight_.resize(n);
  sample_weights_kernel<<<blocks_for(n, 256), 256, 0, s>>>(d_fw.get(), ni, uint32_t(n), far_weight_.get());
  have_weight_ = true;
  patch_block_.resize(n * ni);
  HFMM_CUDA_CHECK(cudaMemcpyAsync(patch_block_.get(), store->patch_block.get(), n * ni * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, s));
  have_block_ = true;
  have_lu_ = self_terms;
  if (self_terms) {
    block_lu_.resize(n * ni);
    HFMM_CUDA_CHECK(cudaMemcpyAsync(block_lu_.get(), store->block_lu.get(), n * ni * sizeof(double2),
                                    cudaMemcpyDeviceToDevice, s));
    block_piv_.resize(n);
    HFMM_CUDA_CHECK(cudaMemcpyAsync(block_piv_.get(), store->block_piv.get(), n * sizeof(int), cudaMemcpyDeviceToDevice, s));
  }
  have_near_ = nnz > 0;
  near_offset_.resize(n + 1);
  HFMM_CUDA_CHECK(cudaMemcpyAsync(near_offset_.get(), store->near_offset.get(), (n + 1) * sizeof(uint32_t),
                                  cudaMemcpyDeviceToDevice, s));
  if (nnz) {
    near_source_.resize(nnz);
    HFMM_CUDA_CHECK(cudaMemcpyAsync(near_source_.get(), store->near_source.get(), nnz * sizeof(uint32_t),
                                    cudaMemcpyDeviceToDevice, s));
    near_delta_.resize(nnz);
    HFMM_CUDA_CHECK(cudaMemcpyAsync(near_delta_.get(), store->near_delta.get(), nnz * sizeof(double2),
                                    cudaMemcpyDeviceToDevice, s));
  }
  HFMM_CUDA_CHECK(cudaGetLastError());
  HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
  corrections64_ = std::move(store);
  if (nnz_out) *nnz_out = nnz;
}

void Engine::get_corrections(double* patch_block, double* block_lu, int* block_piv, uint32_t* near_offset,
                             uint32_t* near_source, double* near_delta) {
  if (!corrections64_) throw Error(HFMM_ERR_CONFIG, "hfmm_cuda_build_corrections has not been called");
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const CorrectionStore& c = *corrections64_;
  const size_t n = tree_.n_bodies;
  auto fetch = [&](void* dst, const void* src, size_t bytes) {
    if (dst && bytes) HFMM_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream_));
  };
  fetch(patch_block, c.patch_block.get(), n * c.ni * sizeof(Z));
  if (c.self_terms) {
    fetch(block_lu, c.block_lu.get(), n * c.ni * sizeof(Z));
    fetch(block_piv, c.block_piv.get(), n * sizeof(int));
  }
  fetch(near_offset, c.near_offset.get(), (n + 1) * sizeof(uint32_t));
  fetch(near_source, c.near_source.get(), c.nnz * sizeof(uint32_t));
  fetch(near_delta, c.near_delta.get(), c.nnz * sizeof(Z));
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

}  // namespace hfmm_b200
