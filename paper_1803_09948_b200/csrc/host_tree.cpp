// host_tree.cpp — see host_tree.hpp
#include "host_tree.hpp"

#include <algorithm>
#include <cmath>
#include <thread>

#include "common.hpp"

namespace hfmm_b200 {

namespace {

template <typename Fn>
void parallel_chunks(size_t n, int threads, Fn&& fn) {
  if (n == 0) return;
  const size_t parts = std::max<size_t>(1, std::min<size_t>(size_t(std::max(threads, 1)), n / 1024 + 1));
  if (parts == 1) {
    fn(size_t(0), n, 0);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(parts);
  for (size_t p = 0; p < parts; ++p)
    pool.emplace_back([&fn, n, p, parts] { fn(n * p / parts, n * (p + 1) / parts, int(p)); });
  for (auto& t : pool) t.join();
}

}  // namespace

// reference: src/octree.cpp:25-51 — digitise (x-lo)*2^21/width, clamp the upper face, interleave
// x (high), y, z root-first
uint64_t morton_key21(const double p[3], const double lo[3], double width) {
  for (int a = 0; a < 3; ++a)
    if (!(p[a] >= lo[a] && p[a] <= lo[a] + width))
      throw Error(HFMM_ERR_DOMAIN, "point outside the octree domain box");
  const uint64_t nside = uint64_t(1) << kMaxLevel;
  const double scale = double(nside) / width;
  uint64_t g[3];
  for (int a = 0; a < 3; ++a) {
    int64_t i = int64_t((p[a] - lo[a]) * scale);
    if (i < 0) i = 0;
    if (i >= int64_t(nside)) i = int64_t(nside) - 1;
    g[a] = uint64_t(i);
  }
  uint64_t key = 0;
  for (int b = kMaxLevel - 1; b >= 0; --b)
    key = key << 3 | ((g[0] >> b & 1) << 2) | ((g[1] >> b & 1) << 1) | (g[2] >> b & 1);
  return key;
}

void enclosing_box_host(const double* xyz, size_t n, double box_lo[3], double& width) {
  double lo[3] = {xyz[0], xyz[1], xyz[2]}, hi[3] = {xyz[0], xyz[1], xyz[2]};
  for (size_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      const double v = xyz[3 * i + a];
      if (!std::isfinite(v)) throw Error(HFMM_ERR_DOMAIN, "non-finite coordinate");
      lo[a] = std::min(lo[a], v);
      hi[a] = std::max(hi[a], v);
    }
  double w = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
  if (w <= 0) w = 1;
  w *= 1 + 1e-12;
  for (int a = 0; a < 3; ++a) box_lo[a] = (lo[a] + hi[a]) / 2.0 - w / 2;
  width = w;
}

void build_tree_host(TreeArrays& t, const double* xyz, size_t n, int ncrit, double leaf_cap,
                     int threads) {
  if (n == 0) throw Error(HFMM_ERR_CONFIG, "no bodies to enclose");
  if (ncrit < 1) throw Error(HFMM_ERR_CONFIG, "leaf capacity must be at least 1");
  if (n >= (size_t(1) << 32)) throw Error(HFMM_ERR_CONFIG, "body count exceeds 32-bit indexing");
  t = TreeArrays{};
  t.n_bodies = uint32_t(n);

  enclosing_box_host(xyz, n, t.lo, t.width);
  const double w = t.width;

  // keys, then order by (key, caller index) (reference: src/octree.cpp:164-171)
  struct KI {
    uint64_t key;
    uint32_t idx;
  };
  std::vector<KI> ki(n);
  parallel_chunks(n, threads, [&](size_t b, size_t e, int) {
    for (size_t i = b; i < e; ++i) ki[i] = {morton_key21(xyz + 3 * i, t.lo, w), uint32_t(i)};
  });
  std::sort(ki.begin(), ki.end(), [](const KI& a, const KI& b) {
    return a.key != b.key ? a.key < b.key : a.idx < b.idx;
  });
  t.key.resize(n);
  t.index.resize(n);
  for (size_t i = 0; i < n; ++i) {
    t.key[i] = ki[i].key;
    t.index[i] = ki[i].idx;
  }
  std::vector<KI>().swap(ki);

  // level-synchronous top-down split (same rule as reference src/octree.cpp:85-137): a cell
  // splits while it holds more than ncrit bodies, or its diameter exceeds leaf_cap, unless it
  // already sits at level 21; empty octants get no cell; children are contiguous
  auto push = [&](int lvl, uint32_t x, uint32_t y, uint32_t z, uint32_t bf, uint32_t bc,
                  uint32_t par) {
    t.level.push_back(uint8_t(lvl));
    t.ix.push_back(x);
    t.iy.push_back(y);
    t.iz.push_back(z);
    t.body_first.push_back(bf);
    t.body_count.push_back(bc);
    t.child_first.push_back(0);
    t.child_count.push_back(0);
    t.parent.push_back(par);
  };
  push(0, 0, 0, 0, 0, uint32_t(n), 0);
  t.level_offset = {0, 1};
  const double sqrt3 = std::sqrt(3.0);
  for (int lvl = 0;; ++lvl) {
    const uint32_t begin = t.level_offset[lvl], end = t.level_offset[lvl + 1];
    const double diameter = t.side(lvl) * sqrt3;  // 2 * radius, radius = side*sqrt(3)/2
    for (uint32_t c = begin; c < end; ++c) {
      const uint32_t first = t.body_first[c], count = t.body_count[c];
      const bool over_cap = int64_t(count) > int64_t(ncrit);
      const bool over_diam = leaf_cap > 0 && diameter > leaf_cap && count > 0;
      if ((!over_cap && !over_diam) || lvl == kMaxLevel) {
        if (lvl == kMaxLevel && over_cap) ++t.degenerate_leaves;
        t.leaves.push_back(c);
        continue;
      }
      const int shift = 3 * (kMaxLevel - 1 - lvl);
      const uint64_t* kb = t.key.data() + first;
      const uint64_t* ke = kb + count;
      const uint64_t* pos = kb;
      uint32_t nchild = 0;
      const uint32_t cf = uint32_t(t.level.size());
      for (uint32_t d = 0; d < 8; ++d) {
        const uint64_t* nxt = std::partition_point(
            pos, ke, [shift, d](uint64_t k) { return ((k >> shift) & 7) <= d; });
        if (nxt != pos) {
          push(lvl + 1, t.ix[c] << 1 | (d >> 2 & 1), t.iy[c] << 1 | (d >> 1 & 1),
               t.iz[c] << 1 | (d & 1), first + uint32_t(pos - kb), uint32_t(nxt - pos), c);
          ++nchild;
        }
        pos = nxt;
      }
      t.child_first[c] = cf;
      t.child_count[c] = nchild;
    }
    if (t.level.size() == end) {
      t.max_level = lvl;
      break;
    }
    t.level_offset.push_back(uint32_t(t.level.size()));
  }
  std::sort(t.leaves.begin(), t.leaves.end());
}

// Breadth-first pair frontier.  Each (target, source) pair is classified exactly as the
// reference's Walker::walk does (src/traversal.cpp:45-79):
//   admissible (gate k*diameter <= kd_max on both cells, |ca-cb| > (ra+rb)/theta)  -> M2L
//   both leaves                                                                    -> P2P
//   else split the target iff it is not a leaf and (source is a leaf or ra > rb),
//   ties open the source
// The pair SET equals the reference's; the order inside a target's list is not preserved (only
// floating-point summation order depends on it).
void dual_tree_traversal_host(const TreeArrays& t, double kmag, double theta, double kd_max,
                              PairLists& out, int threads, int grain) {
  if (!(theta > 0) || theta > 1)
    throw Error(HFMM_ERR_CONFIG, "opening angle must satisfy 0 < theta <= 1");
  out = PairLists{};
  struct Pair {
    uint32_t t, s;
  };
  std::vector<Pair> frontier{{0, 0}}, next;
  const double sqrt3h = std::sqrt(3.0) / 2;
  const int nthreads = std::max(threads, 1);
  struct Local {
    std::vector<Pair> next, far, near;
    uint64_t tasks = 0;
  };
  const uint32_t s_grain = uint32_t(std::max(grain, 0));
  uint64_t tasks = (t.n_cells() && 2 * uint64_t(t.n_bodies) <= s_grain) ? 1 : 0;  // the root node
  while (!frontier.empty()) {
    std::vector<Local> loc(nthreads);
    parallel_chunks(frontier.size(), nthreads, [&](size_t b, size_t e, int tid) {
      Local& L = loc[tid];
      for (size_t i = b; i < e; ++i) {
        const uint32_t a = frontier[i].t, s = frontier[i].s;
        const int la = t.level[a], ls = t.level[s];
        const double sa = t.side(la), ss = t.side(ls);
        const double ra = sa * sqrt3h, rs = ss * sqrt3h;
        bool adm = !(kd_max > 0 && (kmag * (2 * ra) > kd_max || kmag * (2 * rs) > kd_max));
        if (adm) {
          // centres exactly as the reference forms them: lo + (i + 0.5) * side
          const double dx = (t.lo[0] + (t.ix[a] + 0.5) * sa) - (t.lo[0] + (t.ix[s] + 0.5) * ss);
          const double dy = (t.lo[1] + (t.iy[a] + 0.5) * sa) - (t.lo[1] + (t.iy[s] + 0.5) * ss);
          const double dz = (t.lo[2] + (t.iz[a] + 0.5) * sa) - (t.lo[2] + (t.iz[s] + 0.5) * ss);
          adm = std::sqrt(dx * dx + dy * dy + dz * dz) > (ra + rs) / theta;
        }
        if (adm) {
          L.far.push_back({a, s});
          continue;
        }
        const bool aleaf = t.child_count[a] == 0, sleaf = t.child_count[s] == 0;
        if (aleaf && sleaf) {
          L.near.push_back({a, s});
          continue;
        }
        // a child node opens a task when its bodies first fit the grain (its parent, this node, did not)
        const bool open = t.body_count[a] + t.body_count[s] > s_grain;
        if (!aleaf && (sleaf || ra > rs)) {
          for (uint32_t c = 0; c < t.child_count[a]; ++c) {
            L.next.push_back({t.child_first[a] + c, s});
            if (open && t.body_count[t.child_first[a] + c] + t.body_count[s] <= s_grain) ++L.tasks;
          }
        } else {
          for (uint32_t c = 0; c < t.child_count[s]; ++c) {
            L.next.push_back({a, t.child_first[s] + c});
            if (open && t.body_count[a] + t.body_count[t.child_first[s] + c] <= s_grain) ++L.tasks;
          }
        }
      }
    });
    next.clear();
    for (auto& L : loc) {
      tasks += L.tasks;
      next.insert(next.end(), L.next.begin(), L.next.end());
      for (auto& p : L.far) {
        out.m2l_t.push_back(p.t);
        out.m2l_s.push_back(p.s);
      }
      for (auto& p : L.near) {
        out.p2p_t.push_back(p.t);
        out.p2p_s.push_back(p.s);
      }
    }
    frontier.swap(next);
  }
  out.tasks = tasks;
}

int partition_units(const TreeArrays& t, int lmin_src, int lmin_dst, std::vector<uint32_t>& unit) {
  const size_t nc = t.n_cells();
  const int lmin = std::min(lmin_src, lmin_dst);
  const int lcut = lmin > kMaxLevel ? 0 : lmin;  // no far field at all: the units are the leaves
  const uint32_t none = 0xffffffffu;
  unit.assign(nc, none);
  for (uint32_t c = 0; c < nc; ++c) {
    if (t.level[c] == lcut || (t.level[c] < lcut && t.child_count[c] == 0)) unit[c] = c;
    else if (t.level[c] > lcut) unit[c] = unit[t.parent[c]];
  }
  return lcut;
}

void partition_cuts(const TreeArrays& t, const std::vector<uint32_t>& unit,
                    const std::vector<double>& weight, int nranks, std::vector<int>& cell_rank,
                    std::vector<uint32_t>& first, std::vector<uint32_t>& count) {
  const size_t nc = t.n_cells();
  const uint32_t none = 0xffffffffu;
  cell_rank.assign(nc, 0);
  first.assign(nranks, 0);
  count.assign(nranks, 0);
  if (nranks <= 1) {
    count[0] = t.n_bodies;
    return;
  }
  std::vector<uint32_t> units;
  for (uint32_t c = 0; c < nc; ++c)
    if (unit[c] == c) units.push_back(c);
  std::sort(units.begin(), units.end(),
            [&](uint32_t x, uint32_t y) { return t.body_first[x] < t.body_first[y]; });
  double total = 0;
  for (uint32_t u : units) total += weight[u];
  // a unit goes to the rank whose share contains the midpoint of its weight interval; ranks are
  // monotone in Morton order, so every rank's units (and bodies) are contiguous
  std::vector<int> unit_rank(nc, -1);
  double acc = 0;
  int prev = 0;
  for (uint32_t u : units) {
    const double mid = acc + 0.5 * weight[u];
    int r = total > 0 ? int(mid / total * nranks) : 0;
    r = std::min(std::max(r, prev), nranks - 1);
    unit_rank[u] = prev = r;
    acc += weight[u];
  }
  // body ranges: rank r starts where its first unit starts; empty ranks get empty ranges
  std::vector<uint32_t> start(nranks + 1, t.n_bodies);
  for (auto it = units.rbegin(); it != units.rend(); ++it) start[unit_rank[*it]] = t.body_first[*it];
  for (int r = nranks - 1; r >= 0; --r)
    if (start[r] > start[r + 1]) start[r] = start[r + 1];
  start[0] = 0;
  for (int r = 0; r < nranks; ++r) {
    first[r] = start[r];
    count[r] = start[r + 1] - start[r];
  }
  for (uint32_t c = 0; c < nc; ++c) cell_rank[c] = unit[c] == none ? -1 : unit_rank[unit[c]];
}

void compute_morton_partition(const TreeArrays& t, const PairLists& pairs, int nranks, double alpha,
                              std::vector<int>& cell_rank, std::vector<uint32_t>& first,
                              std::vector<uint32_t>& count, int& lcut) {
  int lmin_src = kMaxLevel + 1, lmin_dst = kMaxLevel + 1;
  for (size_t e = 0; e < pairs.m2l_t.size(); ++e) {
    lmin_dst = std::min(lmin_dst, int(t.level[pairs.m2l_t[e]]));
    lmin_src = std::min(lmin_src, int(t.level[pairs.m2l_s[e]]));
  }
  std::vector<uint32_t> unit;
  lcut = partition_units(t, lmin_src, lmin_dst, unit);
  std::vector<double> weight(t.n_cells(), 0.0);
  if (nranks > 1) {
    for (size_t e = 0; e < pairs.p2p_t.size(); ++e) {
      const uint32_t a = pairs.p2p_t[e], b = pairs.p2p_s[e];
      weight[unit[a]] += kPartitionPairWeight * double(t.body_count[a]) * double(t.body_count[b]);
    }
    for (size_t e = 0; e < pairs.m2l_t.size(); ++e)
      weight[unit[pairs.m2l_t[e]]] += alpha < 0 ? kPartitionM2lWeight : alpha * double(t.body_count[pairs.m2l_t[e]]);
  }
  partition_cuts(t, unit, weight, nranks, cell_rank, first, count);
}

double partition_update_alpha(const double* alpha, const double* runtime, int n, double alpha_max) {
  if (n < 1 || !alpha || !runtime) throw Error(HFMM_ERR_CONFIG, "alpha history must not be empty");
  if (!(alpha_max > 0)) throw Error(HFMM_ERR_CONFIG, "alpha_max must be positive");
  constexpr double inv_phi = 0.6180339887498948;
  constexpr int budget = 12;
  const double tol = 1e-12 * std::max(1.0, alpha_max);
  std::vector<char> used(n, 0);
  // first unused sample measured at `a`, or -1: the search has not probed there yet
  auto take = [&](double a) {
    for (int i = 0; i < n; ++i)
      if (!used[i] && std::abs(alpha[i] - a) <= tol) {
        used[i] = 1;
        return i;
      }
    return -1;
  };
  double lo = 0, hi = alpha_max;
  double x1 = hi - inv_phi * (hi - lo), x2 = lo + inv_phi * (hi - lo);
  int s1 = take(x1);
  if (s1 < 0) return x1;
  int s2 = take(x2);
  if (s2 < 0) return x2;
  for (int probes = 2; probes < budget && hi - lo > 1e-6 * alpha_max; ++probes) {
    if (runtime[s1] < runtime[s2]) {  // the minimum lies left of x2
      hi = x2;
      x2 = x1;
      s2 = s1;
      x1 = hi - inv_phi * (hi - lo);
      if ((s1 = take(x1)) < 0) return x1;
    } else {
      lo = x1;
      x1 = x2;
      s1 = s2;
      x2 = lo + inv_phi * (hi - lo);
      if ((s2 = take(x2)) < 0) return x2;
    }
  }
  int best = 0;  // earliest minimum: a flat curve changes nothing
  for (int i = 1; i < n; ++i)
    if (runtime[i] < runtime[best]) best = i;
  return alpha[best];
}

}  // namespace hfmm_b200
