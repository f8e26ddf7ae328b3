// engine.cu — see engine.hpp
#include "engine.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cmath>
#include <complex>
#include <map>
#include <mutex>
#include <numeric>
#include <thread>
#include <unordered_map>

#include "tables.hpp"
#include "tree_build.cuh"

namespace hfmm_b200 {

cudaStream_t& alloc_stream() {
  thread_local cudaStream_t s = nullptr;
  return s;
}

namespace {
std::atomic<int> g_live_engines{0};
}

cudaMemPool_t& alloc_pool() {
  thread_local cudaMemPool_t p = nullptr;
  return p;
}

namespace {
std::mutex g_pool_mutex;
std::map<int, cudaMemPool_t> g_pools;
}  // namespace

// the library's private stream-ordered pool of `device` (null if pools are unavailable: the buffers
// then come from the device's default pool)
cudaMemPool_t library_memory_pool(int device) {
  std::lock_guard<std::mutex> lock(g_pool_mutex);
  auto it = g_pools.find(device);
  if (it != g_pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    (void)cudaGetLastError();
    pool = nullptr;
  } else {
    uint64_t keep = ~uint64_t(0);  // freed buffers stay in the pool while a handle lives
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  g_pools[device] = pool;
  return pool;
}

void trim_memory_pool(int device) {
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_pool_mutex);
    auto it = g_pools.find(device);
    if (it != g_pools.end()) pool = it->second;
  }
  if (!pool) return;
  cudaDeviceSynchronize();
  cudaMemPoolTrimTo(pool, 0);
}

std::atomic<size_t>& device_bytes_counter() {
  static std::atomic<size_t> bytes{0};
  return bytes;
}

static int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return a < 0 ? -a : a;
}

// de-duplicates rotation (by polar angle) and coaxial (by kind, levels, distance) tables
struct TableRegistry {
  struct CoaxSpec {
    CoaxKind kind;
    double dist, s_src, s_dst;
  };
  std::map<std::pair<int64_t, int64_t>, uint32_t> rot_ids;
  std::vector<double> rot_cos;
  std::map<std::tuple<int, int, int, int, int64_t>, uint32_t> coax_ids;
  std::vector<CoaxSpec> coax_specs;

  // direction (dx,dy,dz) on any lattice: key is the reduced fraction dz^2 / |d|^2 with dz's sign
  uint32_t rot(int64_t dx, int64_t dy, int64_t dz) {
    const int64_t r2 = dx * dx + dy * dy + dz * dz, z2 = dz * dz;
    const int64_t g = gcd64(z2, r2);
    const std::pair<int64_t, int64_t> key{(dz < 0 ? -1 : 1) * (z2 / g), r2 / g};
    auto [it, fresh] = rot_ids.try_emplace(key, uint32_t(rot_cos.size()));
    if (fresh) rot_cos.push_back(double(dz) / std::sqrt(double(r2)));
    return it->second;
  }
  uint32_t coax(CoaxKind kind, int lsrc, int ldst, int lunit, int64_t r2, double unit,
                double s_src, double s_dst) {
    const auto key = std::make_tuple(int(kind), lsrc, ldst, lunit, r2);
    auto [it, fresh] = coax_ids.try_emplace(key, uint32_t(coax_specs.size()));
    if (fresh) coax_specs.push_back({kind, unit * std::sqrt(double(r2)), s_src, s_dst});
    return it->second;
  }
};

static TranslateClass make_class(TableRegistry& reg, CoaxKind kind, int64_t dx, int64_t dy, int64_t dz,
                          int lsrc, int ldst, int lunit, double unit, double s_src, double s_dst) {
  TranslateClass c;
  c.rot = reg.rot(dx, dy, dz);
  c.coax = reg.coax(kind, lsrc, ldst, lunit, dx * dx + dy * dy + dz * dz, unit, s_src, s_dst);
  const double rxy = std::sqrt(double(dx * dx + dy * dy));
  c.cphi = rxy > 0 ? float(double(dx) / rxy) : 1.0f;
  c.sphi = rxy > 0 ? float(double(dy) / rxy) : 0.0f;
  return c;
}

namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;

template <typename Fn>
void parallel_for(size_t n, int threads, Fn&& fn) {
  const size_t parts = std::max<size_t>(1, std::min<size_t>(size_t(std::max(threads, 1)), n));
  if (parts <= 1) {
    for (size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> pool;
  for (size_t p = 0; p < parts; ++p)
    pool.emplace_back([&fn, n, p, parts] {
      for (size_t i = p; i < n; i += parts) fn(i);
    });
  for (auto& t : pool) t.join();
}


struct ShiftKey {
  int32_t dx, dy, dz;
  int16_t lt, ls;
  bool operator==(const ShiftKey& o) const {
    return dx == o.dx && dy == o.dy && dz == o.dz && lt == o.lt && ls == o.ls;
  }
};
struct ShiftKeyHash {
  size_t operator()(const ShiftKey& k) const {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (uint64_t v : {uint64_t(uint32_t(k.dx)), uint64_t(uint32_t(k.dy)), uint64_t(uint32_t(k.dz)),
                       uint64_t(uint16_t(k.lt)) << 16 | uint16_t(k.ls)})
      h = (h ^ v) * 0xff51afd7ed558ccdull + (h >> 29);
    return size_t(h);
  }
};

}  // namespace

Engine::Engine(const hfmm_cuda_config& cfg) : cfg_(cfg) {
  // config_error rules of the reference (traversal.cpp:16-21, 212-213; octree.cpp:144)
  if (cfg.ncrit < 1 || cfg.grain < cfg.ncrit)
    throw Error(HFMM_ERR_CONFIG, "traversal grain needs s >= c >= 1");
  if (!(cfg.theta > 0) || cfg.theta > 1)
    throw Error(HFMM_ERR_CONFIG, "opening angle must satisfy 0 < theta <= 1");
  if (cfg.order < 0) throw Error(HFMM_ERR_CONFIG, "expansion order must be non-negative");
  if (cfg.order > kMaxOrder)
    throw Error(HFMM_ERR_CONFIG, "expansion order above the supported maximum (16)");
  // complex wavenumber k = wave_r + i wave_i (common.hpp:36-40): coordinates are scaled by wave_r,
  // so the real part must be positive; wave_i (attenuation) enters the radial functions, the
  // translation tables and the near-field amplitude
  if (!(cfg.wave_r > 0)) throw Error(HFMM_ERR_CONFIG, "the real part of the wavenumber must be positive");
  if (!(cfg.wave_i == cfg.wave_i) || std::abs(cfg.wave_i) > 4.0 * cfg.wave_r)
    throw Error(HFMM_ERR_CONFIG, "wave_i must be finite with |wave_i| <= 4 wave_r");
  if (cfg.kd_max < 0) throw Error(HFMM_ERR_CONFIG, "kd_max must be non-negative");
  leaf_cap_ = cfg.leaf_cap;
  if (leaf_cap_ < 0) leaf_cap_ = cfg.kd_max > 0 ? cfg.kd_max / std::hypot(cfg.wave_r, cfg.wave_i) : 0.0;  // kd_max / |k|
  threads_ = int(std::max(1u, std::thread::hardware_concurrency()));

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(HFMM_ERR_DEVICE, "no CUDA device available (this library has no CPU fallback)");
  if (cfg.device < 0 || cfg.device >= ndev) throw Error(HFMM_ERR_CONFIG, "device ordinal out of range");
  HFMM_CUDA_CHECK(cudaSetDevice(cfg.device));
  try {
    // the far-field stream outranks the near-field stream: when both have blocks waiting, freed SM
    // resources go to the (few, persistent) M2L CTAs first and the near field fills what is left
    int prio_lo = 0, prio_hi = 0;
    HFMM_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    HFMM_CUDA_CHECK(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, prio_hi));
    HFMM_CUDA_CHECK(cudaStreamCreateWithPriority(&stream_near_, cudaStreamNonBlocking, prio_lo));
    HFMM_CUDA_CHECK(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    HFMM_CUDA_CHECK(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    ev_.assign(14, nullptr);
    for (auto& e : ev_) HFMM_CUDA_CHECK(cudaEventCreate(&e));
    user_ev_.assign(16, nullptr);
    for (auto& e : user_ev_) HFMM_CUDA_CHECK(cudaEventCreate(&e));

    const int P = cfg.order;
    const size_t tri = size_t(P + 1) * (P + 2) / 2;
    std::vector<float> diag(P + 1), sub(P + 1), a(tri), b(tri);
    build_legendre_coefficients(P, diag.data(), sub.data(), a.data(), b.data());
    upload_legendre_constants(diag.data(), sub.data(), a.data(), b.data(), P);
    upload_translate_schedule(P);
  } catch (...) {
    destroy_streams_and_events();  // a failed constructor runs no destructor: nothing may leak
    throw;
  }
  ++g_live_engines;  // last: counted only when the handle exists
}

void Engine::destroy_streams_and_events() {
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  for (auto& e : user_ev_)
    if (e) cudaEventDestroy(e);
  ev_.clear();
  user_ev_.clear();
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (stream_) cudaStreamDestroy(stream_);
  if (stream_near_) cudaStreamDestroy(stream_near_);
  ev_fork_ = ev_join_ = nullptr;
  stream_ = stream_near_ = nullptr;
}

void Engine::release_device_state() { --g_live_engines; }
bool Engine::any_engine_alive() { return g_live_engines.load() > 0; }

Engine::~Engine() {
  cudaSetDevice(cfg_.device);
  release_device_state();
  destroy_streams_and_events();
}

const char* Engine::take_stale_cuda_error() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? nullptr : cudaGetErrorName(e);
}

void Engine::require_points() const {
  if (!have_points_) throw Error(HFMM_ERR_CONFIG, "hfmm_cuda_set_points has not been called");
}

// compute_multipoles' truncation-waste scan (expansion.cpp:253-262): cells whose top radial factor
// j_P(|k| radius) vanishes in FP64.  The radius depends on the level only; j_P is evaluated as the reference
// does for small arguments (ascending series, special.cpp:17-34) — only there can it underflow to zero.
uint64_t Engine::count_starved_cells() const {
  const int P = cfg_.order;
  if (P <= 0) return 0;
  const double kmag = std::hypot(cfg_.wave_r, cfg_.wave_i);
  uint64_t starved = 0;
  for (int L = 0; L <= tree_.max_level; ++L) {
    const uint64_t cells = tree_.level_offset[L + 1] - tree_.level_offset[L];
    if (!cells) continue;
    const double z = kmag * (tree_.side(L) * std::sqrt(3.0) / 2);
    if (z >= 0.5) continue;  // Miller recurrence normalised by j_0: never exactly zero
    const double z2h = 0.5 * z * z;
    double zn = 1.0, dfact = 1.0, top = 0.0;
    for (int n = 0; n <= P; ++n) {
      double term = 1.0, sum = 1.0;
      for (int k = 1; k < 40; ++k) {
        term *= -z2h / double(k * (2 * n + 2 * k + 1));
        sum += term;
        if (std::abs(term) < 1e-18 * std::abs(sum)) break;
      }
      top = zn / dfact * sum;
      zn *= z;
      dfact *= double(2 * n + 3);
    }
    if (top == 0.0) starved += cells;
  }
  return starved;
}

// Classes that share the rotation table (polar angle) and the coaxial table (levels, distance) differ
// only in azimuth — lattice shifts related by quarter turns about z and by reflections — and are
// batched together: the kernel carries e^{i m phi} per pair.  Returns the order in which the classes
// are laid out (group by group) and the group of every class.
// batches per table group must save at least 3 % of the batches to pay for the per-pair phases
// (HFMM_BATCHING=group|class forces one layout: used by the tests to run both kernel instantiations)
static constexpr double kMixedBatchGainDefault = 0.97;
static double mixed_batch_gain() {
  const char* e = getenv("HFMM_BATCHING");
  if (e && !strcmp(e, "group")) return 1e9;
  if (e && !strcmp(e, "class")) return -1.0;
  return kMixedBatchGainDefault;
}

static void group_classes(const std::vector<TranslateClass>& classes, std::vector<uint32_t>& order,
                          std::vector<uint32_t>& group_of) {
  const size_t nc = classes.size();
  order.resize(nc);
  for (size_t c = 0; c < nc; ++c) order[c] = uint32_t(c);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
    return classes[x].rot != classes[y].rot ? classes[x].rot < classes[y].rot : classes[x].coax < classes[y].coax;
  });
  group_of.assign(nc, 0);
  uint32_t g = 0;
  for (size_t i = 0; i < nc; ++i) {
    if (i && (classes[order[i]].rot != classes[order[i - 1]].rot || classes[order[i]].coax != classes[order[i - 1]].coax)) ++g;
    group_of[order[i]] = g;
  }
}

// HFMM_FLAG_DETERMINISTIC: cut the stage into ranges of whole batches that fit the staging buffer and
// sort every range's pairs by destination (stable) for the ordered reduction (run_stage)
void Engine::plan_ordered_reduce(TranslateStage& st, const std::vector<TranslateItem>& items) {
  st.ordered.clear();
  st.row_of_pair.release();
  if (!(cfg_.flags & HFMM_FLAG_DETERMINISTIC) || items.empty()) return;
  size_t budget_mb = 4096;
  if (const char* e = getenv("HFMM_ORDERED_STAGING_MB")) budget_mb = std::max<size_t>(1, strtoull(e, nullptr, 10));
  const uint64_t row_bytes = uint64_t(stride_) * sizeof(float2);
  const uint64_t max_rows = std::max<uint64_t>(translate_batch_size(cfg_.order), (budget_mb << 20) / row_bytes);
  const uint64_t total = uint64_t(items.back().pair_begin) + items.back().count;
  st.row_of_pair.resize(total);
  uint64_t most = 0;
  for (size_t i = 0; i < items.size();) {
    TranslateStage::OrderedRange r;
    r.item_begin = uint32_t(i);
    r.pair_begin = items[i].pair_begin;
    uint64_t rows = 0;
    while (i < items.size() && rows + items[i].count <= max_rows) rows += items[i++].count;
    r.n_items = uint32_t(i) - r.item_begin;
    r.n_pairs = uint32_t(rows);
    launch_range_rows(st.row_of_pair.get(), r.pair_begin, r.n_pairs, stream_);
    r.n_segs = build_ordered_reduce_device(st.pair_dst.get(), r.pair_begin, r.n_pairs, r.perm, r.seg_dst,
                                           r.seg_begin, stream_);
    most = std::max(most, rows);
    st.ordered.push_back(std::move(r));
  }
  if (ordered_staging_.size() < most * stride_) ordered_staging_.resize(most * stride_);
}

void Engine::upload_stage(TranslateStage& st, const std::vector<uint32_t>& src,
                          const std::vector<uint32_t>& dst, const std::vector<uint32_t>& cls_of_pair,
                          const std::vector<TranslateClass>& classes, bool ordered) {
  // stable counting sort of the pairs by class (classes laid out group by group), then batches of
  // kTranslateBatch pairs cut per table group
  const size_t np = src.size(), nc = classes.size();
  std::vector<uint32_t> order, group_of;
  group_classes(classes, order, group_of);
  std::vector<uint32_t> pos_of(nc);  // position of a class in the grouped layout
  for (size_t i = 0; i < nc; ++i) pos_of[order[i]] = uint32_t(i);
  std::vector<uint64_t> start(nc + 1, 0);
  for (size_t i = 0; i < np; ++i) ++start[pos_of[cls_of_pair[i]] + 1];
  for (size_t c = 0; c < nc; ++c) start[c + 1] += start[c];
  std::vector<uint32_t> s_sorted(np), d_sorted(np), c_sorted(np);
  {
    std::vector<uint64_t> cur(start.begin(), start.end() - 1);
    for (size_t i = 0; i < np; ++i) {
      const uint64_t slot = cur[pos_of[cls_of_pair[i]]]++;
      s_sorted[slot] = src[i];
      d_sorted[slot] = dst[i];
      c_sorted[slot] = cls_of_pair[i];
    }
  }
  // batches: per table group when that saves batches (partially filled ones cost as much as full
  // ones), else per class — one class per batch keeps the cheaper per-class phases in the kernel
  const uint64_t batch = uint64_t(translate_batch_size(cfg_.order));
  auto cut = [&](bool per_group) {
    std::vector<TranslateItem> out;
    for (size_t i = 0; i < nc;) {
      size_t j = i + 1;
      while (per_group && j < nc && group_of[order[j]] == group_of[order[i]]) ++j;
      for (uint64_t b = start[i]; b < start[j]; b += batch)
        out.push_back({uint32_t(b), uint32_t(std::min<uint64_t>(batch, start[j] - b)), c_sorted[b],
                       group_of[order[i]]});
      i = j;
    }
    return out;
  };
  std::vector<TranslateItem> items = cut(true);
  st.mixed = true;
  {
    std::vector<TranslateItem> per_class = cut(false);
    if (!translate64_supported(cfg_.order) && double(items.size()) > mixed_batch_gain() * double(per_class.size())) {
      items.swap(per_class);
      st.mixed = false;
    }
  }
  if (np >= (uint64_t(1) << 32)) throw Error(HFMM_ERR_CONFIG, "pair count exceeds 32-bit indexing");
  st.n_items = uint32_t(items.size());
  st.n_pairs = np;
  st.items.upload(items, stream_);
  st.classes.upload(classes, stream_);
  st.pair_src.upload(s_sorted, stream_);
  st.pair_dst.upload(d_sorted, stream_);
  st.pair_cls.upload(c_sorted, stream_);
  if (ordered) plan_ordered_reduce(st, items);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

// M2L stage from host pair lists: one class per distinct (lattice shift, level pair), as the
// reference de-duplicates translation matrices per lattice shift (traversal.cpp:152-166, 233-250)
void Engine::build_m2l_stage_host(TableRegistry& reg, const PairLists& pairs) {
  const TreeArrays& t = tree_;
  const double k = cfg_.wave_r;
  auto scale = [&](int lvl) { return k * t.side(lvl); };
  const size_t nm2l = pairs.m2l_t.size();
  std::vector<uint32_t> cls_of_pair, own_src, own_dst;
  cls_of_pair.reserve(nm2l / size_t(nranks_) + 16);
  std::vector<TranslateClass> classes;
  std::unordered_map<ShiftKey, uint32_t, ShiftKeyHash> ids;
  ids.reserve(1 << 16);
  for (size_t e = 0; e < nm2l; ++e) {
    const uint32_t a = pairs.m2l_t[e], b = pairs.m2l_s[e];
    if (!owned_[a]) continue;  // this rank translates into its own target cells only
    const int la = t.level[a], lb = t.level[b], lmax = std::max(la, lb);
    auto c = [lmax](uint32_t i, int l) { return int64_t(2 * uint64_t(i) + 1) << (lmax - l); };
    // t = centre(target) - centre(source) in half-sides of level lmax
    const ShiftKey key{int32_t(c(t.ix[a], la) - c(t.ix[b], lb)), int32_t(c(t.iy[a], la) - c(t.iy[b], lb)),
                       int32_t(c(t.iz[a], la) - c(t.iz[b], lb)), int16_t(la), int16_t(lb)};
    auto [it, fresh] = ids.try_emplace(key, uint32_t(classes.size()));
    if (fresh)
      classes.push_back(make_class(reg, CoaxKind::m2l, key.dx, key.dy, key.dz, lb, la, lmax,
                                   t.side(lmax) / 2, scale(lb), scale(la)));
    cls_of_pair.push_back(it->second);
    own_src.push_back(b);
    own_dst.push_back(a);
  }
  stats_.m2l_shift_classes = classes.size();
  owned_m2l_pairs_ = own_src.size();
  upload_stage(m2l_, own_src, own_dst, cls_of_pair, classes, true);
}

// M2L stage from the device builder's sorted pairs + run-length-encoded shift classes
void Engine::build_m2l_stage_device(TableRegistry& reg, const FarClasses& fc) {
  const TreeArrays& t = tree_;
  const double k = cfg_.wave_r;
  auto scale = [&](int lvl) { return k * t.side(lvl); };
  const size_t nc = fc.count.size();
  std::vector<TranslateClass> classes(nc);
  for (size_t c = 0; c < nc; ++c) {
    const int la = fc.lt[c], lb = fc.ls[c], lmax = std::max(la, lb);
    classes[c] = make_class(reg, CoaxKind::m2l, fc.dx[c], fc.dy[c], fc.dz[c], lb, la, lmax,
                            t.side(lmax) / 2, scale(lb), scale(la));
  }
  // the device builder left the pairs sorted class by class; lay the classes out group by group
  // (group_classes) by moving whole class segments, and record the class of every pair
  std::vector<uint32_t> order, group_of;
  group_classes(classes, order, group_of);
  std::vector<uint64_t> old_start(nc + 1, 0);
  for (size_t c = 0; c < nc; ++c) old_start[c + 1] = old_start[c] + fc.count[c];
  std::vector<uint32_t> seg_new(nc + 1, 0), seg_old(nc), seg_cls(nc);
  std::vector<TranslateItem> items, per_class;
  const uint64_t batch = uint64_t(translate_batch_size(cfg_.order));
  uint64_t pos = 0;
  for (size_t i = 0; i < nc;) {
    size_t j = i;
    const uint64_t group_begin = pos;
    while (j < nc && group_of[order[j]] == group_of[order[i]]) {
      seg_new[j] = uint32_t(pos);
      seg_old[j] = uint32_t(old_start[order[j]]);
      seg_cls[j] = order[j];
      for (uint64_t b = 0; b < fc.count[order[j]]; b += batch)
        per_class.push_back({uint32_t(pos + b), uint32_t(std::min<uint64_t>(batch, fc.count[order[j]] - b)),
                             order[j], group_of[order[i]]});
      pos += fc.count[order[j]];
      ++j;
    }
    for (uint64_t b = group_begin; b < pos; b += batch) {
      // class of the batch's first pair: the segment that holds position b
      size_t s = i;
      while (s + 1 < j && seg_new[s + 1] <= b) ++s;
      items.push_back({uint32_t(b), uint32_t(std::min<uint64_t>(batch, pos - b)), seg_cls[s], group_of[order[i]]});
    }
    i = j;
  }
  seg_new[nc] = uint32_t(pos);
  // batches per table group only when that saves batches (see upload_stage)
  m2l_.mixed = translate64_supported(cfg_.order) || double(items.size()) <= mixed_batch_gain() * double(per_class.size());
  if (!m2l_.mixed) items.swap(per_class);
  if (pos >= (uint64_t(1) << 32)) throw Error(HFMM_ERR_CONFIG, "pair count exceeds 32-bit indexing");
  regroup_pairs_device(seg_new, seg_old, seg_cls, pos, m2l_.pair_src, m2l_.pair_dst, m2l_.pair_cls, stream_);
  stats_.m2l_shift_classes = classes.size();
  owned_m2l_pairs_ = fc.n_owned_pairs;
  m2l_.n_items = uint32_t(items.size());
  m2l_.n_pairs = fc.n_owned_pairs;
  m2l_.items.upload(items, stream_);
  m2l_.classes.upload(classes, stream_);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
  plan_ordered_reduce(m2l_, items);
}

// M2M / L2L stages per level, translation tables, leaf lists, expansion storage
void Engine::finish_far_field(TableRegistry& reg) {
  const TreeArrays& t = tree_;
  const int P = cfg_.order;
  const double k = cfg_.wave_r;
  const size_t nc = t.n_cells();
  auto scale = [&](int lvl) { return k * t.side(lvl); };
  m2m_.clear();
  l2l_.clear();
  if (!have_far_) {
    n_p2m_leaves_ = n_l2p_leaves_ = 0;
    stats_.rotation_tables = stats_.coaxial_tables = 0;
    return;
  }
  // M2M: child level L -> parent, L from the deepest level up to lmin_src+1; the 8 octant shifts
  // per level of the reference (expansion.cpp:200-222).  t = parent - child = -(+-h) per axis.
  auto level_stage = [&](int L, bool upward) {
    std::vector<uint32_t> src, dst, cls;
    std::vector<TranslateClass> cl;
    int cls_of_oct[8];
    std::fill(cls_of_oct, cls_of_oct + 8, -1);
    for (uint32_t c = t.level_offset[L]; c < t.level_offset[L + 1]; ++c) {
      if (!owned_[c]) continue;
      const int oct = int(t.ix[c] & 1) << 2 | int(t.iy[c] & 1) << 1 | int(t.iz[c] & 1);
      if (cls_of_oct[oct] < 0) {
        int64_t d[3] = {oct & 4 ? -1 : 1, oct & 2 ? -1 : 1, oct & 1 ? -1 : 1};  // parent - child
        if (!upward)
          for (auto& v : d) v = -v;
        cls_of_oct[oct] = int(cl.size());
        cl.push_back(upward ? make_class(reg, CoaxKind::m2m, d[0], d[1], d[2], L, L - 1, L,
                                         t.side(L) / 2, scale(L), scale(L - 1))
                            : make_class(reg, CoaxKind::l2l, d[0], d[1], d[2], L - 1, L, L,
                                         t.side(L) / 2, scale(L - 1), scale(L)));
      }
      src.push_back(upward ? c : t.parent[c]);
      dst.push_back(upward ? t.parent[c] : c);
      cls.push_back(uint32_t(cls_of_oct[oct]));
    }
    TranslateStage st;
    upload_stage(st, src, dst, cls, cl, upward);
    return st;
  };
  const bool trace = getenv("HFMM_SETUP_TRACE") != nullptr;
  auto t_prev = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(stream_);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[hfmm setup]   %-26s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_prev).count());
    t_prev = now;
  };
  for (int L = t.max_level; L > lmin_src_; --L) m2m_.push_back(level_stage(L, true));
  for (int L = lmin_dst_ + 1; L <= t.max_level; ++L) l2l_.push_back(level_stage(L, false));
  mark("M2M / L2L stages");

  const size_t nrot = reg.rot_cos.size(), ncoax = reg.coax_specs.size();
  stats_.rotation_tables = nrot;
  stats_.coaxial_tables = ncoax;
  std::vector<float> rot(nrot * size_t(rot_table_size(P)));
  std::vector<float> coax(ncoax * size_t(coax_table_size(P)) * 2);
  mark("table buffers");
  parallel_for(nrot, threads_, [&](size_t i) {
    build_rotation_table(P, reg.rot_cos[i], rot.data() + i * size_t(rot_table_size(P)));
  });
  mark("rotation tables");
  const CoaxBuilder& builder = CoaxBuilder::shared(P);
  const bool sign_folded = coax_tables_sign_folded(P);
  parallel_for(ncoax, threads_, [&](size_t i) {
    const auto& s = reg.coax_specs[i];
    float* tab = coax.data() + i * size_t(coax_table_size(P)) * 2;
    builder.build(s.kind, k, s.dist, s.s_src, s.s_dst, tab, cfg_.wave_i);
    if (sign_folded)  // (-1)^m of the inverse rotation's inputs, applied once here instead of per batch
      for (int m = 1; m <= P; m += 2) {
        float* blk = tab + 2 * size_t(coax_block_offset(P, m));
        const size_t cnt = 2 * size_t(P + 1 - m) * size_t(coax_row_stride(P, m));
        for (size_t e = 0; e < cnt; ++e) blk[e] = -blk[e];
      }
  });
  mark("coaxial tables");
  rot_tables_.upload(rot, stream_);
  coax_tables_.upload(coax, stream_);
  mark("table upload");

  std::vector<uint32_t> up, down;
  for (uint32_t c : t.leaves) {
    if (!owned_[c]) continue;
    if (t.level[c] >= lmin_src_) up.push_back(c);
    if (t.level[c] >= lmin_dst_) down.push_back(c);
  }
  n_p2m_leaves_ = uint32_t(up.size());
  n_l2p_leaves_ = uint32_t(down.size());
  p2m_leaves_.upload(up, stream_);
  l2p_leaves_.upload(down, stream_);
  multipole_.resize(nc * size_t(stride_));
  local_.resize(nc * size_t(stride_));
  multipole_.zero(stream_);
  local_.zero(stream_);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
  mark("leaf lists + expansions");
}

// cell geometry on the lattice, level scales, the hi/lo grid
void Engine::upload_cell_geometry(std::vector<int4>& geom) {
  const TreeArrays& t = tree_;
  const size_t nc = t.n_cells();
  const double k = cfg_.wave_r;
  const int Lf = t.max_level;
  geom.resize(nc);
  std::vector<uint2> cbody(nc);
  for (size_t c = 0; c < nc; ++c) {
    const int up = Lf - t.level[c];
    geom[c] = make_int4(int((2 * t.ix[c] + 1) << up), int((2 * t.iy[c] + 1) << up),
                        int((2 * t.iz[c] + 1) << up), int(t.level[c]));
    cbody[c] = make_uint2(t.body_first[c], t.body_count[c]);
  }
  level_scale_host_.assign(kMaxLevel + 1, 0.f);
  for (int l = 0; l <= kMaxLevel; ++l) level_scale_host_[l] = float(k * t.side(l));
  kunit_d_ = k * t.side(Lf) / 2;
  kunit_ = float(kunit_d_);
  // hi/lo split for touching leaves (kernels.cuh): every hi value, hi offset and hi difference
  // between touching leaves stays below 2^23 grid units, hence exactly representable in FP32
  double max_leaf_side = 0;
  for (uint32_t c : t.leaves) max_leaf_side = std::max(max_leaf_side, t.side(t.level[c]));
  grid_ = std::ldexp(1.0, int(std::ceil(std::log2(4.0 * k * max_leaf_side))) - 23);
  // k rho <= sqrt(3)/2 k side for every body of every leaf: inside the 7-term range of the scaled series?
  leaf_small_args_ = 0.8661 * k * max_leaf_side <= 0.999;
  cell_geom_.upload(geom, stream_);
  cell_body_.upload(cbody, stream_);
  level_scale_.upload(level_scale_host_, stream_);
}

// Near-field kernel variant (kernels.cuh, P2PArgs::mode).  max_r2_lattice bounds the squared distance
// of any evaluated body pair in half-sides of the finest level; with a leaf cap in force (the
// reference's solver path) R' = k_r R stays below ~4 and sin(R')/R' runs as a polynomial on the FMA pipe.
// HFMM_P2P_MODE=0..3 forces a variant (tests and experiments; polynomial modes need the bound).
void Engine::select_near_kernel(uint64_t max_r2_lattice) {
  near_r2_max_ = double(max_r2_lattice) * kunit_d_ * kunit_d_ * (1.0 + 1e-5);
  const bool bounded = near_r2_max_ <= double(kP2PPolyMaxR2);
  p2p_mode_ = bounded ? P2P_MODE_SINC_POLY : P2P_MODE_MUFU;
  if (const char* e = getenv("HFMM_P2P_MODE")) {
    const int m = atoi(e);
    if (m == P2P_MODE_MUFU || (bounded && m >= 0 && m <= P2P_MODE_ALL_POLY)) p2p_mode_ = m;
  }
  fit_p2p_polynomials(std::max(near_r2_max_, 1e-3), p2p_sinc_, p2p_cos_);
}

// The variant of the near-field launch that shares the machine with M2L.  On its own the bounded-range variant
// (sinc as a polynomial: 18 packed FMA-pipe instructions and two MUFU per pair of pairs) is the faster one; beside
// M2L, which lives on the FMA pipe and leaves the MUFU pipe idle, the general variant (12 + three MUFU) costs the
// step less: cfg 2 13.95 -> 13.68 ms, cfg 5's per-GPU share 73.1 -> 71.9 ms, nothing at cfg 4, +3 % at cfg 1 where
// the far field is as short as the near field — hence only when the far field clearly outweighs the near field
// (estimated kernel times: executed flops at 21 TFLOP/s against 1.0e12 body pairs per second).
int Engine::near_mode_in_step() const {
  if (getenv("HFMM_P2P_MODE") || p2p_mode_ != P2P_MODE_SINC_POLY || !have_far_) return p2p_mode_;
  const int P = cfg_.order;
  double rot = 0, coax = 0;
  for (int j = 0; j <= P; ++j) rot += double(j + 1) * (j + 1) + double(j) * j;
  for (int m = -P; m <= P; ++m) coax += double(P + 1 - std::abs(m)) * (P + 1 - std::abs(m));
  const double t_far = double(owned_m2l_pairs_) * 2.0 * (4.0 * rot + 4.0 * coax) / 21e12;
  const double t_near = double(owned_body_pairs_) / 1.0e12;
  // below half a millisecond of near field the estimates mean nothing (launch latency and tails: cfg 1)
  return t_near > 0.5e-3 && t_far > 2.0 * t_near ? int(P2P_MODE_MUFU) : p2p_mode_;
}

// tiles of <= 32 targets per owned leaf, longest first (the tail of the launch fills with short ones)
void Engine::build_tiles(const std::vector<uint64_t>& work) {
  const TreeArrays& t = tree_;
  std::vector<P2PTile> tiles;
  std::vector<uint64_t> tile_work;
  for (size_t i = 0; i < t.leaves.size(); ++i) {
    const uint32_t c = t.leaves[i];
    if (!owned_[c]) continue;
    for (uint32_t b = 0; b < t.body_count[c]; b += 32) {
      const uint32_t nt = std::min<uint32_t>(32, t.body_count[c] - b);
      tiles.push_back({c, b, nt, uint32_t(i)});
      tile_work.push_back(work[i] * nt);
    }
  }
  std::vector<uint32_t> order(tiles.size());
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t x, uint32_t y) { return tile_work[x] > tile_work[y]; });
  std::vector<P2PTile> sorted(tiles.size());
  for (size_t i = 0; i < order.size(); ++i) sorted[i] = tiles[order[i]];
  n_tiles_ = uint32_t(sorted.size());
  p2p_tiles_.upload(sorted, stream_);
}

void Engine::set_partition_alpha(double alpha) {
  if (alpha != alpha) throw Error(HFMM_ERR_CONFIG, "alpha must be a number");
  partition_alpha_ = alpha;  // takes effect at the next set_points
}

void Engine::set_partition(int rank, int nranks) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(HFMM_ERR_CONFIG, "rank out of range");
  if (nranks > 64) throw Error(HFMM_ERR_CONFIG, "at most 64 ranks (exchange masks are 64 bits wide)");
  if (rank != rank_ || nranks != nranks_) release_comm();  // a communicator belongs to one (rank, nranks)
  rank_ = rank;
  nranks_ = nranks;
  have_points_ = false;  // work lists depend on the partition: set_points must follow
}

// ownership of cells and bodies for this rank (host_tree.cpp: compute_morton_partition)
void Engine::compute_partition() {
  const size_t nc = tree_.n_cells();
  owned_.assign(nc, 1);
  own_first_ = 0;
  own_count_ = tree_.n_bodies;
  std::vector<int> cell_rank;
  std::vector<uint32_t> first, count;
  compute_morton_partition(tree_, pairs_, nranks_, partition_alpha_, cell_rank, first, count, lcut_);
  cell_rank_.assign(cell_rank.begin(), cell_rank.end());
  if (nranks_ == 1) return;
  own_first_ = first[rank_];
  own_count_ = count[rank_];
  for (size_t c = 0; c < nc; ++c) owned_[c] = cell_rank[c] == rank_;
}

void Engine::get_partition(hfmm_cuda_partition* out) {
  require_points();
  const TreeArrays& t = tree_;
  *out = hfmm_cuda_partition{};
  out->rank = rank_;
  out->nranks = nranks_;
  out->n_bodies = t.n_bodies;
  out->body_first = own_first_;
  out->body_count = own_count_;
  out->coeff_stride = uint64_t(stride_);
  out->multipole_dev = have_far_ ? multipole_.get() : nullptr;
  out->level_first = have_far_ ? lmin_src_ : 0;
  out->level_last = have_far_ ? t.max_level : -1;
  out->owned_m2l_pairs = owned_m2l_pairs_;
  out->owned_p2p_body_pairs = owned_body_pairs_;
  for (int L = 0; L <= t.max_level && L < 22; ++L) {
    out->level_cell_first[L] = t.level_offset[L];
    out->level_cell_count[L] = t.level_offset[L + 1] - t.level_offset[L];
    uint32_t f = 0xffffffffu, l = 0;
    for (uint32_t c = t.level_offset[L]; c < t.level_offset[L + 1]; ++c)
      if (owned_[c]) {
        f = std::min(f, c);
        l = std::max(l, c + 1);
      }
    out->cell_first[L] = f == 0xffffffffu ? t.level_offset[L] : f;
    out->cell_count[L] = f == 0xffffffffu ? 0 : l - f;
    // ownership follows contiguous body ranges, so the owned cells of a level at or below the
    // partition cut are contiguous too.  Above the cut a level can interleave owned leaves with
    // unowned interior cells (cell_rank -1: nobody translates into them); those levels are never
    // exchanged (level_first is the coarsest translating level), so only the exchanged ones are checked
    if (have_far_ && L >= lmin_src_)
      for (uint32_t c = out->cell_first[L]; c < out->cell_first[L] + out->cell_count[L]; ++c)
        if (!owned_[c]) throw Error(HFMM_ERR_STRUCTURAL, "owned cells of a level are not contiguous");
  }
}

// distributed matvec, phase 1: q is the FULL charge vector in Morton order (the caller gathered
// the ranks' slices); runs the near field of the owned leaves and the upward pass of the owned cells
void Engine::dist_upward(const void* q_morton_dev) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[8], stream_));
  HFMM_CUDA_CHECK(cudaMemcpyAsync(body_q_.get(), q_morton_dev, size_t(tree_.n_bodies) * sizeof(float2),
                                  cudaMemcpyDeviceToDevice, stream_));
  phase_upward();
}

// phase 2 (after the caller exchanged the owned multipole rows): M2L / L2L / L2P into the owned
// cells, then out[slot] = near + far for the owned Morton slots (other slots untouched)
void Engine::dist_downward(void* out_morton_dev) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  phase_downward();
  launch_scatter_potentials(near_.get() + own_first_, far_.get() + own_first_,
                            identity_index() + own_first_, nullptr,
                            static_cast<float2*>(out_morton_dev), own_count_, stream_);
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[9], stream_));
}

static constexpr size_t kHostFallbackBodies = size_t(1) << 18;

void Engine::set_points(const double* xyz, size_t n) {
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const auto t0 = std::chrono::steady_clock::now();
  // the buffers of the previous point set are freed in stream_'s order: nothing on the near-field
  // stream may still be reading them (a matvec joins it into stream_; a half-finished two-phase one does not)
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_near_));
  have_points_ = false;
  have_weight_ = have_block_ = have_near_ = have_lu_ = false;  // corrections belong to a point set
  release_correction_store();
  exchange_.reset();  // the index lists of the exchanges belong to a point set
  touch2_.release();
  identity_.release();
  dev_pairs_ = DevicePairs{};
  pairs_ = PairLists{};
  stride_ = coeff_stride(cfg_.order);
  m2l_ = TranslateStage{};
  host_lists_ = (cfg_.flags & HFMM_FLAG_HOST_TREE) != 0;
  if (host_lists_) {
    set_points_host(xyz, n);
  } else {
    try {
      set_points_device(xyz, n);
    } catch (const DeviceBuilderLimit& lim) {
      if (cfg_.flags & HFMM_FLAG_NO_HOST_FALLBACK) throw;  // the caller asked for the device builder or nothing
      // lists beyond the device memory / 32-bit pair indexing (a gate that forbids every coarse translation)
      // are left to the host builder for moderate sizes only: at a million points that configuration is a
      // mistake to report, not hours of host work to start
      if (!lim.any_size && n > kHostFallbackBodies) throw;
      host_lists_ = true;
      dev_pairs_ = DevicePairs{};
      pairs_ = PairLists{};
      m2l_ = TranslateStage{};
      set_points_host(xyz, n);
    }
  }
  body_index_.upload(tree_.index, stream_);
  body_q_.resize(n);
  near_.resize(n);
  far_.resize(n);
  io64_.resize(n);
  far_.zero(stream_);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));

  stats_.n_bodies = n;
  stats_.n_cells = tree_.n_cells();
  stats_.n_leaves = tree_.leaves.size();
  stats_.max_level = uint64_t(tree_.max_level);
  stats_.starved_cells = count_starved_cells();
  stats_.setup_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  stats_.device_bytes = device_bytes_counter();
  p2p_mode_late_ = near_mode_in_step();
  have_points_ = true;
}

// ---- builder on the device (default): tree_build.cu -------------------------------------------
void Engine::set_points_device(const double* xyz, size_t n) {
  const double k = cfg_.wave_r;
  // HFMM_SETUP_TRACE=1: wall time of every setup phase on stderr (synchronises after each)
  const bool trace = getenv("HFMM_SETUP_TRACE") != nullptr;
  auto t_prev = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(stream_);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[hfmm setup] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_prev).count());
    t_prev = now;
  };
  DeviceBuffer<double>& d_xyz = xyz64_;  // kept: FP64 points in caller order
  DeviceBuffer<uint32_t> d_index;
  build_tree_device(tree_, xyz, n, cfg_.ncrit, leaf_cap_, d_xyz, d_index, stream_);
  mark("tree");
  const TreeArrays& t = tree_;
  DeviceCells cells;
  cells.upload(t, stream_);
  const double kmag = std::hypot(cfg_.wave_r, cfg_.wave_i);  // the gate uses |k| (traversal.cpp:86)
  const size_t nc = t.n_cells();
  owned_.assign(nc, 1);
  own_first_ = 0;
  own_count_ = t.n_bodies;
  uint64_t global_body_pairs = 0;
  if (nranks_ == 1) {
    dual_tree_traversal_device(t, cells, kmag, cfg_.theta, cfg_.kd_max, cfg_.grain, dev_pairs_, stream_);
    stats_.tasks = dev_pairs_.tasks;
    far_pair_level_range(dev_pairs_, cells, lmin_dst_, lmin_src_, stream_);
    mark("traversal");
    stats_.m2l_pairs = dev_pairs_.n_far;
    stats_.p2p_pairs = dev_pairs_.n_near;
    std::vector<uint32_t> unit;
    lcut_ = partition_units(t, lmin_src_, lmin_dst_, unit);
    cell_rank_.assign(nc, 0);
  } else {
    // Several ranks: the pair lists are built PER RANK.  Pass 1 walks the global descent without storing a pair
    // and leaves the work of every target cell (the weights that place the Morton cuts, identical on all ranks:
    // no handshake); pass 2 repeats the descent pruned to the nodes that touch a subtree this rank owns, so the
    // stored lists, their sorts and everything derived from them are O(N / ranks + boundary).
    TraversalCensus census;
    dual_tree_census_device(t, cells, kmag, cfg_.theta, cfg_.kd_max, cfg_.grain, partition_alpha_, census, stream_);
    mark("traversal (census)");
    stats_.tasks = census.tasks;
    stats_.m2l_pairs = census.n_far;
    stats_.p2p_pairs = census.n_near;
    global_body_pairs = census.body_pairs;
    lmin_dst_ = census.lmin_dst;
    lmin_src_ = census.lmin_src;
    std::vector<uint32_t> unit;
    lcut_ = partition_units(t, lmin_src_, lmin_dst_, unit);
    std::vector<double> weight(nc, 0.0);
    for (size_t c = 0; c < nc; ++c)
      if (census.cell_weight[c] != 0.0) {
        if (unit[c] == 0xffffffffu) throw Error(HFMM_ERR_INTERNAL, "a target cell above the partition cut carries work");
        weight[unit[c]] += census.cell_weight[c];
      }
    std::vector<int> cell_rank;
    std::vector<uint32_t> first, count;
    partition_cuts(t, unit, weight, nranks_, cell_rank, first, count);
    own_first_ = first[rank_];
    own_count_ = count[rank_];
    for (size_t c = 0; c < nc; ++c) owned_[c] = cell_rank[c] == rank_;
    cell_rank_.assign(cell_rank.begin(), cell_rank.end());
    // subtrees that hold an owned cell (cells are stored level by level, parents first)
    std::vector<uint8_t> interest(owned_.begin(), owned_.end());
    for (size_t c = nc; c-- > 1;)
      if (interest[c]) interest[t.parent[c]] = 1;
    dual_tree_traversal_pruned_device(t, cells, kmag, cfg_.theta, cfg_.kd_max, interest, dev_pairs_, stream_);
    mark("traversal (pruned to the rank)");
  }
  have_far_ = stats_.m2l_pairs > 0;

  std::vector<int4> geom;
  upload_cell_geometry(geom);
  build_body_arrays_device(t, d_xyz, d_index, k, grid_, body_pos_, body_hi_, body_lo_, body_abs_, stream_);
  mark("partition + body arrays");

  NearLists nl;
  build_near_lists_device(dev_pairs_, t, cells, owned_, p2p_offset_, p2p_split_, p2p_src_, nl, stream_);
  stats_.p2p_body_pairs = nranks_ == 1 ? nl.body_pairs : global_body_pairs;  // of the global lists
  owned_body_pairs_ = nl.owned_body_pairs;
  select_near_kernel(nl.max_r2_lattice);
  build_tiles(nl.work);
  mark("near lists + tiles");

  TableRegistry reg;
  stats_.m2l_shift_classes = 0;
  owned_m2l_pairs_ = 0;
  if (have_far_) {
    FarClasses fc;
    build_far_classes_device(dev_pairs_, t, cells, owned_, m2l_.pair_src, m2l_.pair_dst, fc, stream_);
    mark("far classes (sort)");
    build_m2l_stage_device(reg, fc);
    mark("M2L stage (classes, batches)");
  }
  finish_far_field(reg);
  mark("tables + M2M/L2L + storage");
}

// ---- builder on the host (HFMM_FLAG_HOST_TREE): host_tree.cpp ---------------------------------
void Engine::set_points_host(const double* xyz, size_t n) {
  build_tree_host(tree_, xyz, n, cfg_.ncrit, leaf_cap_, threads_);
  xyz64_.upload(xyz, 3 * n, stream_);
  dual_tree_traversal_host(tree_, std::hypot(cfg_.wave_r, cfg_.wave_i), cfg_.theta, cfg_.kd_max, pairs_, threads_,
                           cfg_.grain);
  stats_.tasks = pairs_.tasks;
  const TreeArrays& t = tree_;
  const size_t nc = t.n_cells();
  const double k = cfg_.wave_r;
  const int Lf = t.max_level;
  lmin_src_ = lmin_dst_ = kMaxLevel + 1;
  for (size_t e = 0; e < pairs_.m2l_t.size(); ++e) {
    lmin_dst_ = std::min(lmin_dst_, int(t.level[pairs_.m2l_t[e]]));
    lmin_src_ = std::min(lmin_src_, int(t.level[pairs_.m2l_s[e]]));
  }
  have_far_ = !pairs_.m2l_t.empty();
  stats_.m2l_pairs = pairs_.m2l_t.size();
  stats_.p2p_pairs = pairs_.p2p_t.size();
  compute_partition();

  std::vector<int4> geom;
  upload_cell_geometry(geom);

  // bodies: leaf-relative, pre-scaled by k, plus the hi/lo split
  std::vector<float4> pos(n), pos_hi(n), pos_lo(n), abs_pos(n);
  parallel_for(t.leaves.size(), threads_, [&](size_t li) {
    const uint32_t c = t.leaves[li];
    const double s = t.side(t.level[c]);
    const double cx = t.lo[0] + (t.ix[c] + 0.5) * s, cy = t.lo[1] + (t.iy[c] + 0.5) * s,
                 cz = t.lo[2] + (t.iz[c] + 0.5) * s;
    for (uint32_t b = t.body_first[c]; b < t.body_first[c] + t.body_count[c]; ++b) {
      const double* p = xyz + 3 * size_t(t.index[b]);
      const double v[3] = {k * (p[0] - cx), k * (p[1] - cy), k * (p[2] - cz)};
      double h[3];
      for (int a = 0; a < 3; ++a) h[a] = std::rint(v[a] / grid_) * grid_;
      pos[b] = make_float4(float(v[0]), float(v[1]), float(v[2]), 0.f);
      pos_hi[b] = make_float4(float(h[0]), float(h[1]), float(h[2]), 0.f);
      pos_lo[b] = make_float4(float(v[0] - h[0]), float(v[1] - h[1]), float(v[2] - h[2]), 0.f);
    }
  });
  for (size_t i = 0; i < n; ++i)
    abs_pos[i] = make_float4(float(k * xyz[3 * i]), float(k * xyz[3 * i + 1]), float(k * xyz[3 * i + 2]), 0.f);

  // near field: CSR by target leaf, touching source leaves (self included) first
  const size_t nleaf = t.leaves.size();
  std::vector<uint32_t> leaf_slot(nc, 0xffffffffu);
  for (size_t i = 0; i < nleaf; ++i) leaf_slot[t.leaves[i]] = uint32_t(i);
  auto touching = [&](uint32_t a, uint32_t b) {
    const int64_t ha = int64_t(1) << (Lf - t.level[a]), hb = int64_t(1) << (Lf - t.level[b]);
    return std::llabs(int64_t(geom[a].x) - geom[b].x) <= ha + hb &&
           std::llabs(int64_t(geom[a].y) - geom[b].y) <= ha + hb &&
           std::llabs(int64_t(geom[a].z) - geom[b].z) <= ha + hb;
  };
  std::vector<uint32_t> off(nleaf + 1, 0), split(nleaf, 0);
  uint64_t body_pairs = 0, owned_body_pairs = 0, max_r2_lattice = 0;
  for (size_t e = 0; e < pairs_.p2p_t.size(); ++e) {
    const uint32_t a = pairs_.p2p_t[e], b = pairs_.p2p_s[e];
    body_pairs += uint64_t(t.body_count[a]) * t.body_count[b];
    if (!owned_[a]) continue;
    owned_body_pairs += uint64_t(t.body_count[a]) * t.body_count[b];
    {
      const uint64_t hs = (uint64_t(1) << (Lf - t.level[a])) + (uint64_t(1) << (Lf - t.level[b]));
      const uint64_t fx = uint64_t(std::llabs(int64_t(geom[a].x) - geom[b].x)) + hs,
                     fy = uint64_t(std::llabs(int64_t(geom[a].y) - geom[b].y)) + hs,
                     fz = uint64_t(std::llabs(int64_t(geom[a].z) - geom[b].z)) + hs;
      max_r2_lattice = std::max(max_r2_lattice, fx * fx + fy * fy + fz * fz);
    }
    ++off[leaf_slot[a] + 1];
    if (touching(a, b)) ++split[leaf_slot[a]];
  }
  for (size_t i = 0; i < nleaf; ++i) off[i + 1] += off[i];
  for (size_t i = 0; i < nleaf; ++i) split[i] += off[i];
  std::vector<uint32_t> srcs(off[nleaf]);
  std::vector<uint64_t> work(nleaf, 0);
  {
    std::vector<uint32_t> cur_touch(off.begin(), off.end() - 1), cur_far(split);
    for (size_t e = 0; e < pairs_.p2p_t.size(); ++e) {
      const uint32_t a = pairs_.p2p_t[e], b = pairs_.p2p_s[e];
      if (!owned_[a]) continue;
      work[leaf_slot[a]] += t.body_count[b];
      srcs[touching(a, b) ? cur_touch[leaf_slot[a]]++ : cur_far[leaf_slot[a]]++] = b;
    }
  }
  // source leaves in ascending cell order: neighbouring bodies, neighbouring addresses
  parallel_for(nleaf, threads_, [&](size_t i) {
    std::sort(srcs.begin() + off[i], srcs.begin() + split[i]);
    std::sort(srcs.begin() + split[i], srcs.begin() + off[i + 1]);
  });
  build_tiles(work);
  select_near_kernel(max_r2_lattice);
  stats_.p2p_body_pairs = body_pairs;
  owned_body_pairs_ = owned_body_pairs;

  body_abs_.upload(abs_pos, stream_);
  body_pos_.upload(pos, stream_);
  body_hi_.upload(pos_hi, stream_);
  body_lo_.upload(pos_lo, stream_);
  p2p_split_.upload(split, stream_);
  p2p_offset_.upload(off, stream_);
  p2p_src_.upload(srcs, stream_);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));

  TableRegistry reg;
  stats_.m2l_shift_classes = 0;
  owned_m2l_pairs_ = 0;
  if (have_far_) build_m2l_stage_host(reg, pairs_);
  finish_far_field(reg);
}

// one FMM evaluation, body_q_ (Morton order) -> near_, far_.  The near field runs on its own
// stream, concurrently with the upward / translation / downward chain.
void Engine::run_far_and_near() {
  phase_upward();
  phase_downward();
}

void Engine::phase_upward() {
  // per-kernel CUDA events are always recorded on the stream each kernel is launched on (they cost
  // nothing); HFMM_FLAG_PHASE_TIMERS additionally serialises the near field behind the far field
  // so the per-kernel durations are free of overlap
  const bool serial = (cfg_.flags & HFMM_FLAG_PHASE_TIMERS) != 0;
  launches_ = 0;
  uint64_t& launches = launches_;
  HFMM_CUDA_CHECK(cudaEventRecord(ev_fork_, stream_));
  HFMM_CUDA_CHECK(cudaStreamWaitEvent(stream_near_, ev_fork_, 0));

  P2PArgs pa{};
  pa.tiles = p2p_tiles_.get();
  pa.n_tiles = n_tiles_;
  pa.p2p_offset = p2p_offset_.get();
  pa.p2p_split = p2p_split_.get();
  pa.p2p_src = p2p_src_.get();
  pa.body_hi = body_hi_.get();
  pa.body_lo = body_lo_.get();
  pa.kunit_d = kunit_d_;
  pa.grid = grid_;
  pa.cell_geom = cell_geom_.get();
  pa.cell_body = cell_body_.get();
  pa.body_pos = body_pos_.get();
  pa.body_q = body_q_.get();
  pa.out = near_.get();
  pa.kunit = kunit_;
  pa.out_scale = float(cfg_.wave_r / (4.0 * kPi));
  pa.damp = float(cfg_.wave_i / cfg_.wave_r * 1.4426950408889634);
  pa.mode = p2p_mode_;
  std::copy(p2p_sinc_, p2p_sinc_ + 8, pa.sinc_c);
  std::copy(p2p_cos_, p2p_cos_ + 8, pa.cos_c);
  p2p_args_ = pa;
  // The near field is enqueued BEHIND the persistent M2L launch (enqueued first, its 30 k CTAs fill every SM
  // and the M2L CTAs wait for them).  Beside the one sixteen-warp M2L CTA of P >= 13 (80 registers, one tile)
  // three 2-warp near-field CTAs fit and the near field really hides under M2L (cfg 4: 619 -> 595 ms); the two
  // eight-warp CTAs of P <= 12 leave 8 KB of shared memory, less than one near-field CTA needs, and the near
  // field then runs in the gaps and behind M2L (0.4 ms gained over the serialised order at cfg 2)
  p2p_late_ = !serial && have_far_ && !(cfg_.flags & HFMM_FLAG_NEAR_FIRST);
  if (!p2p_late_) {
    cudaStream_t sn = serial ? stream_ : stream_near_;
    if (near_gate_) HFMM_CUDA_CHECK(cudaStreamWaitEvent(sn, near_gate_, 0));
    HFMM_CUDA_CHECK(cudaEventRecord(ev_[0], sn));
    launch_p2p(pa, sn);
    ++launches;
    HFMM_CUDA_CHECK(cudaEventRecord(ev_[1], sn));
  }

  if (have_far_) {
    multipole_.zero(stream_);
    local_.zero(stream_);
    LeafExpansionArgs la{};
    la.cell_geom = cell_geom_.get();
    la.cell_body = cell_body_.get();
    la.body_pos = body_pos_.get();
    la.level_scale = level_scale_.get();
    la.order = cfg_.order;
    la.stride = stride_;
    la.k = float(cfg_.wave_r);
    la.k_imag = float(cfg_.wave_i);
    la.small_arguments = leaf_small_args_;
    la.leaves = p2m_leaves_.get();
    la.n_leaves = n_p2m_leaves_;
    HFMM_CUDA_CHECK(cudaEventRecord(ev_[2], stream_));
    launch_p2m(la, body_q_.get(), multipole_.get(), stream_);
    ++launches;
    HFMM_CUDA_CHECK(cudaEventRecord(ev_[3], stream_));

    for (const auto& st : m2m_) run_stage(st, multipole_.get(), multipole_.get());
    HFMM_CUDA_CHECK(cudaEventRecord(ev_[4], stream_));
  }
}

void Engine::run_stage(const TranslateStage& st, const float2* src, float2* dst) {
  TranslateArgs ta{};
  ta.items = st.items.get();
  ta.n_items = st.n_items;
  ta.classes = st.classes.get();
  ta.pair_src = st.pair_src.get();
  ta.pair_dst = st.pair_dst.get();
  ta.pair_cls = st.pair_cls.get();
  ta.mixed = st.mixed ? 1 : 0;
  ta.rot_tables = rot_tables_.get();
  ta.coax_tables = coax_tables_.get();
  ta.src = src;
  ta.dst = dst;
  ta.order = cfg_.order;
  ta.stride = stride_;
  if (!st.ordered.empty()) {
    // deterministic accumulation: every pair writes its own staging row (plain stores in place of the
    // atomics) and the rows of a destination are then summed in pair order
    const uint32_t dim = uint32_t(cfg_.order + 1) * uint32_t(cfg_.order + 1);
    for (const auto& r : st.ordered) {
      ta.staged = 1;
      ta.items = st.items.get() + r.item_begin;
      ta.n_items = r.n_items;
      ta.pair_dst = st.row_of_pair.get();
      ta.dst = ordered_staging_.get();
      launch_translate(ta, stream_);
      launch_ordered_reduce(ordered_staging_.get(), r.perm.get(), r.seg_begin.get(), r.seg_dst.get(), r.n_segs, dst,
                            uint32_t(stride_), dim, stream_);
      launches_ += 2;
    }
    return;
  }
  launch_translate(ta, stream_);
  if (st.n_items) ++launches_;
}

void Engine::phase_downward() {
  uint64_t& launches = launches_;
  if (have_far_) {
    LeafExpansionArgs la{};
    la.cell_geom = cell_geom_.get();
    la.cell_body = cell_body_.get();
    la.body_pos = body_pos_.get();
    la.level_scale = level_scale_.get();
    la.order = cfg_.order;
    la.stride = stride_;
    la.k = float(cfg_.wave_r);
    la.k_imag = float(cfg_.wave_i);
    la.small_arguments = leaf_small_args_;
    HFMM_CUDA_CHECK(cudaEventRecord(ev_[12], stream_));
    if (p2p_late_) HFMM_CUDA_CHECK(cudaStreamWaitEvent(stream_near_, ev_[12], 0));
    run_stage(m2l_, multipole_.get(), local_.get());
    if (p2p_late_) {  // enqueued behind the persistent M2L launch: its CTAs fill what M2L leaves free
      if (near_gate_) HFMM_CUDA_CHECK(cudaStreamWaitEvent(stream_near_, near_gate_, 0));
      HFMM_CUDA_CHECK(cudaEventRecord(ev_[0], stream_near_));
      P2PArgs late = p2p_args_;
      late.mode = p2p_mode_late_;  // beside M2L: the variant that leaves it the FMA pipe (near_mode_in_step)
      launch_p2p(late, stream_near_);
      ++launches;
      HFMM_CUDA_CHECK(cudaEventRecord(ev_[1], stream_near_));
    }
    HFMM_CUDA_CHECK(cudaEventRecord(ev_[5], stream_));
    for (const auto& st : l2l_) run_stage(st, local_.get(), local_.get());
    HFMM_CUDA_CHECK(cudaEventRecord(ev_[6], stream_));
    la.leaves = l2p_leaves_.get();
    la.n_leaves = n_l2p_leaves_;
    launch_l2p(la, local_.get(), far_.get(), stream_);
    ++launches;
    HFMM_CUDA_CHECK(cudaEventRecord(ev_[7], stream_));
  }
  HFMM_CUDA_CHECK(cudaEventRecord(ev_join_, stream_near_));
  HFMM_CUDA_CHECK(cudaStreamWaitEvent(stream_, ev_join_, 0));
  stats_.kernel_launches = launches + 2;  // + gather, scatter
  timings_pending_ = true;
}

// reads the per-kernel events of the last matvec (synchronises the handle's stream)
void Engine::collect_timings() {
  if (!timings_pending_) return;
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
  auto dt = [&](int a, int b) {
    // an interval whose events were not recorded by the last call (e.g. the bracketing pair
    // after a two-phase matvec) reads as zero; drop the error so that it is not left behind
    float v = 0;
    if (cudaEventElapsedTime(&v, ev_[a], ev_[b]) != cudaSuccess) {
      (void)cudaGetLastError();
      v = 0;
    }
    return double(v) * 1e-3;
  };
  stats_.p2p_seconds = dt(0, 1);
  stats_.p2m_seconds = stats_.m2m_seconds = stats_.m2l_seconds = stats_.l2l_seconds = stats_.l2p_seconds = 0;
  if (have_far_) {
    stats_.p2m_seconds = dt(2, 3);
    stats_.m2m_seconds = dt(3, 4);
    stats_.m2l_seconds = dt(12, 5);
    stats_.l2l_seconds = dt(5, 6);
    stats_.l2p_seconds = dt(6, 7);
  }
  stats_.upward_seconds = stats_.p2m_seconds + stats_.m2m_seconds;
  stats_.interaction_seconds = stats_.m2l_seconds + stats_.p2p_seconds;
  stats_.downward_seconds = stats_.l2l_seconds + stats_.l2p_seconds;
  stats_.matvec_seconds = dt(8, 9);
  timings_pending_ = false;
}

void Engine::matvec_device(const void* q_dev, void* out_dev) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const uint32_t n = tree_.n_bodies;
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[8], stream_));
  apply_operator_device(static_cast<const float2*>(q_dev), static_cast<float2*>(out_dev));
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[9], stream_));
  (void)n;
}

void Engine::matvec_host(const double* q, double* out) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const uint32_t n = tree_.n_bodies;
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[10], stream_));
  HFMM_CUDA_CHECK(cudaMemcpyAsync(io64_.get(), q, size_t(n) * sizeof(double2), cudaMemcpyHostToDevice, stream_));
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[8], stream_));
  if (have_weight_ || have_block_ || have_near_) {
    if (x32_.size() != n) {
      x32_.resize(n);
      y32_.resize(n);
    }
    launch_narrow(n, io64_.get(), x32_.get(), stream_);
    apply_operator_device(x32_.get(), y32_.get());
    launch_widen(n, y32_.get(), io64_.get(), stream_);
  } else {
    launch_gather_charges(io64_.get(), nullptr, body_index_.get(), nullptr, body_q_.get(), n, stream_);
    run_far_and_near();
    launch_scatter_potentials(near_.get(), far_.get(), body_index_.get(), io64_.get(), nullptr, n, stream_);
  }
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[9], stream_));
  HFMM_CUDA_CHECK(cudaMemcpyAsync(out, io64_.get(), size_t(n) * sizeof(double2), cudaMemcpyDeviceToHost, stream_));
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[11], stream_));
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

double Engine::measure_fp32_peak_tflops() {
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  // the higher of the scalar-FFMA and the packed-FFMA2 probe is the roofline denominator
  return std::max(run_fp32_peak_probe(stream_, false), run_fp32_peak_probe(stream_, true));
}

void Engine::measure_fp32_probes(double out[2]) {
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  out[0] = run_fp32_peak_probe(stream_, false);
  out[1] = run_fp32_peak_probe(stream_, true);
}

void Engine::timer_record(int slot) {
  if (slot < 0 || slot >= int(user_ev_.size())) throw Error(HFMM_ERR_CONFIG, "timer slot out of range");
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  HFMM_CUDA_CHECK(cudaEventRecord(user_ev_[slot], stream_));
}

double Engine::timer_elapsed_ms(int a, int b) {
  if (a < 0 || b < 0 || a >= int(user_ev_.size()) || b >= int(user_ev_.size()))
    throw Error(HFMM_ERR_CONFIG, "timer slot out of range");
  HFMM_CUDA_CHECK(cudaEventSynchronize(user_ev_[b]));
  float ms = 0;
  HFMM_CUDA_CHECK(cudaEventElapsedTime(&ms, user_ev_[a], user_ev_[b]));
  return double(ms);
}

void Engine::flush_l2() {
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  if (flush_.size() == 0) flush_.resize(size_t(256) << 20);  // 256 MiB > 126 MB of L2
  HFMM_CUDA_CHECK(cudaMemsetAsync(flush_.get(), 1, flush_.size(), stream_));
}

const uint32_t* Engine::identity_index() {
  const uint32_t n = tree_.n_bodies;
  if (identity_.size() != n) {
    std::vector<uint32_t> id(n);
    std::iota(id.begin(), id.end(), 0u);
    identity_.upload(id, stream_);
    HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
  }
  return identity_.get();
}

void Engine::sync() {
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::get_stats(hfmm_cuda_stats* out) {
  collect_timings();
  stats_.device_bytes = device_bytes_counter();
  stats_.m2l_batches = m2l_.n_items;
  stats_.host_tree_used = host_lists_ ? 1 : 0;
  stats_.p2p_mode = uint64_t(p2p_mode_);
  stats_.p2p_mode_in_step = uint64_t(p2p_mode_late_);
  stats_.near_r2_max = near_r2_max_;
  *out = stats_;
}

void Engine::get_cells(uint32_t* out, size_t capacity) const {
  require_points();
  if (capacity < tree_.n_cells()) throw Error(HFMM_ERR_CONFIG, "cell buffer too small");
  for (size_t c = 0; c < tree_.n_cells(); ++c) {
    uint32_t* o = out + 8 * c;
    o[0] = tree_.level[c]; o[1] = tree_.ix[c]; o[2] = tree_.iy[c]; o[3] = tree_.iz[c];
    o[4] = tree_.body_first[c]; o[5] = tree_.body_count[c];
    o[6] = tree_.child_first[c]; o[7] = tree_.child_count[c];
  }
}

void Engine::get_body_order(uint32_t* out) const {
  require_points();
  std::copy(tree_.index.begin(), tree_.index.end(), out);
}

// Locally essential tree of every rank, as bit masks (reference extract_let, let.cpp:150-253, is
// sender-initiated the same way): bit p of far_mask[c] says rank p translates FROM cell c (c is a
// source of an M2L pair whose target p owns), bit p of near_mask[c] says rank p evaluates the
// bodies of leaf c directly.  Every rank holds the global lists, so all ranks compute the same
// masks and derive matching send / receive lists without communicating.
void Engine::get_exchange_masks(uint64_t* far_mask, uint64_t* near_mask, int32_t* cell_rank) const {
  require_points();
  if (nranks_ > 64) throw Error(HFMM_ERR_CONFIG, "exchange masks hold at most 64 ranks");
  const size_t nc = tree_.n_cells();
  std::fill(far_mask, far_mask + nc, uint64_t(0));
  std::fill(near_mask, near_mask + nc, uint64_t(0));
  for (size_t c = 0; c < nc; ++c) cell_rank[c] = cell_rank_.empty() ? 0 : cell_rank_[c];
  for (int which = 0; which < 2; ++which) {
    uint64_t np = 0;
    get_pairs(which, nullptr, &np);
    std::vector<uint32_t> pr(2 * np);
    if (np) get_pairs(which, pr.data(), &np);
    uint64_t* mask = which ? near_mask : far_mask;
    for (uint64_t e = 0; e < np; ++e) mask[pr[2 * e + 1]] |= uint64_t(1) << cell_rank[pr[2 * e]];
  }
}

// reference measure_weights (partition.cpp:143-163): per body, caller order;
// local = bodies of the P2P partners of its leaf, remote = M2L pairs of every cell that holds it
void Engine::measure_weights(double* local, double* remote) const {
  require_points();
  const TreeArrays& t = tree_;
  const size_t nc = t.n_cells();
  std::vector<double> partners(nc, 0.0), lists(nc, 0.0);
  for (int which = 0; which < 2; ++which) {
    uint64_t np = 0;
    get_pairs(which, nullptr, &np);
    std::vector<uint32_t> pr(2 * np);
    if (np) get_pairs(which, pr.data(), &np);
    for (uint64_t e = 0; e < np; ++e) {
      if (which) partners[pr[2 * e]] += double(t.body_count[pr[2 * e + 1]]);
      else lists[pr[2 * e]] += 1.0;
    }
  }
  // cells are stored level by level, parents first: one sweep accumulates the lists of the ancestors
  for (size_t c = 1; c < nc; ++c) lists[c] += lists[t.parent[c]];
  for (uint32_t c : t.leaves)
    for (uint32_t b = t.body_first[c]; b < t.body_first[c] + t.body_count[c]; ++b) {
      local[t.index[b]] = partners[c];
      remote[t.index[b]] = lists[c];
    }
}

void Engine::get_pairs(int which, uint32_t* out, uint64_t* count) const {
  require_points();
  if (!host_lists_) {  // lists live on the device: copy on demand
    const uint64_t np = which ? dev_pairs_.n_near : dev_pairs_.n_far;
    *count = np;
    if (!out || !np) return;
    HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
    HFMM_CUDA_CHECK(cudaMemcpy(out, (which ? dev_pairs_.near : dev_pairs_.far).get(), np * sizeof(uint2),
                               cudaMemcpyDeviceToHost));
    return;
  }
  const auto& tt = which ? pairs_.p2p_t : pairs_.m2l_t;
  const auto& ss = which ? pairs_.p2p_s : pairs_.m2l_s;
  *count = tt.size();
  if (!out) return;
  for (size_t i = 0; i < tt.size(); ++i) {
    out[2 * i] = tt[i];
    out[2 * i + 1] = ss[i];
  }
}

void Engine::get_expansions(int which, double* out) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const int P = cfg_.order, dim = nm_total(P);
  const size_t nc = tree_.n_cells();
  std::fill(out, out + 2 * nc * size_t(dim), 0.0);
  if (!have_far_) return;
  std::vector<float2> host(nc * size_t(stride_));
  (which ? local_ : multipole_).download(host.data(), host.size(), stream_);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
  // undo the level scaling: M = Mhat s^n/(2n+1)!!,  L = Lhat (2n-1)!!/s^n
  for (size_t c = 0; c < nc; ++c) {
    const long double s = (long double)cfg_.wave_r * tree_.side(tree_.level[c]);
    for (int n = 0; n <= P; ++n) {
      const long double f = which ? double_factorial(2 * n - 1) / powl(s, n)
                                  : powl(s, n) / double_factorial(2 * n + 1);
      for (int m = -n; m <= n; ++m) {
        const float2 v = host[c * size_t(stride_) + nm_index(n, m)];
        out[2 * (c * size_t(dim) + nm_index(n, m))] = double(f * v.x);
        out[2 * (c * size_t(dim) + nm_index(n, m)) + 1] = double(f * v.y);
      }
    }
  }
}

void compose_dense_from_tables(int order, double k, const double t[3], int kind, double s_src,
                               double s_dst, double* out, double k_imag) {
  using cd = std::complex<double>;
  const int P = order, dim = nm_total(P);
  const double r = std::sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  const double rxy = std::sqrt(t[0] * t[0] + t[1] * t[1]);
  const double cphi = rxy > 0 ? t[0] / rxy : 1.0, sphi = rxy > 0 ? t[1] / rxy : 0.0;
  std::vector<float> rot(rot_table_size(P)), coax(size_t(coax_table_size(P)) * 2);
  build_rotation_table(P, t[2] / r, rot.data());
  const CoaxBuilder& builder = CoaxBuilder::shared(P);
  // kind 0: M2L with (s_src, s_dst); kind 1: regular shift expressed through the M2M scaling
  builder.build(kind == 0 ? CoaxKind::m2l : CoaxKind::m2m, k, r, s_src, s_dst, coax.data(), k_imag);
  std::vector<cd> ph(2 * P + 1);
  for (int m = -P; m <= P; ++m) ph[m + P] = std::pow(cd(cphi, sphi), m);
  // R[(n,m'),(n,m)] = E_n[m][m'] e^{i m phi};  Chat[(nu,m),(n,m)]
  std::vector<cd> R(size_t(dim) * dim, 0), C(size_t(dim) * dim, 0);
  for (int n = 0; n <= P; ++n) {
    const int w = 2 * n + 1;
    std::vector<double> E(size_t(w) * w);
    unfold_rotation_block(n, rot.data(), E.data());
    for (int m = -n; m <= n; ++m)
      for (int mp = -n; mp <= n; ++mp)
        R[size_t(nm_index(n, mp)) * dim + nm_index(n, m)] = E[size_t(m + n) * w + (mp + n)] * ph[m + P];
  }
  for (int m = -P; m <= P; ++m) {
    const int am = std::abs(m), w = coax_row_stride(P, am);
    const float* blk = coax.data() + 2 * size_t(coax_block_offset(P, am));
    for (int n = am; n <= P; ++n)
      for (int nu = am; nu <= P; ++nu) {
        const size_t e = size_t(n - am) * w + (nu - am);
        // undo the scaling so the result is comparable with the reference's matrix
        long double f;
        if (kind == 0)
          f = double_factorial(2 * nu - 1) * double_factorial(2 * n + 1) /
              (powl(s_dst, nu) * powl(s_src, n));
        else
          f = powl(s_dst, nu) * double_factorial(2 * n + 1) /
              (double_factorial(2 * nu + 1) * powl(s_src, n));
        C[size_t(nm_index(nu, m)) * dim + nm_index(n, m)] =
            cd(double(f * blk[2 * e]), double(f * blk[2 * e + 1]));
      }
  }
  // T = R^H C R
  std::vector<cd> CR(size_t(dim) * dim, 0);
  for (int i = 0; i < dim; ++i)
    for (int l = 0; l < dim; ++l) {
      const cd c = C[size_t(i) * dim + l];
      if (c == cd(0)) continue;
      for (int j = 0; j < dim; ++j) CR[size_t(i) * dim + j] += c * R[size_t(l) * dim + j];
    }
  cd* T = reinterpret_cast<cd*>(out);
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j < dim; ++j) {
      cd s = 0;
      for (int l = 0; l < dim; ++l) s += std::conj(R[size_t(l) * dim + i]) * CR[size_t(l) * dim + j];
      T[size_t(i) * dim + j] = s;
    }
}

}  // namespace hfmm_b200
