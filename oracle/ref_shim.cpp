// oracle/ref_shim.cpp — extern "C" window onto the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  This file is compiled together with the reference's own sources
// (read where they lie under /root/reference/proj/core, see oracle/Makefile) into
// oracle/_ref/libhfmm_ref.so.  tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load it through ctypes to obtain the reference's answers; the product
// library never links or loads it.
//
// Every entry point is a thin call into a reference function; no arithmetic of the path is
// restated here (the restatement lives in hfmm_oracle.c).
#include <algorithm>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "hfmm/expansion.hpp"
#include "hfmm/kernel.hpp"
#include "hfmm/let.hpp"
#include "hfmm/mesh_gen.hpp"
#include "hfmm/mesh_io.hpp"
#include "hfmm/octree.hpp"
#include "hfmm/oracle.hpp"
#include "hfmm/partition.hpp"
#include "hfmm/solver.hpp"
#include "hfmm/special.hpp"
#include "hfmm/traversal.hpp"

using namespace hfmm;

namespace {
thread_local std::string g_err;
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const config_error& e) { g_err = e.what(); return 1;
  } catch (const singular_error& e) { g_err = e.what(); return 2;
  } catch (const structural_error& e) { g_err = e.what(); return 3;
  } catch (const std::exception& e) { g_err = e.what(); return 9; }
}

std::vector<fmm::Body> make_bodies(long n, const double* xyz, const double* q) {
  std::vector<fmm::Body> b(n);
  for (long i = 0; i < n; ++i) {
    b[i].position = Vec3{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
    if (q) b[i].src = cplx(q[2 * i], q[2 * i + 1]);
  }
  return b;
}

fmm::TraversalConfig make_tcfg(int ncrit, int s, double theta, double kd_max, int threads) {
  fmm::TraversalConfig t;
  t.c = ncrit;
  t.s = s;
  t.theta = theta;
  t.kd_max = kd_max;
  t.deterministic = threads <= 1;
  t.threads = threads;
  return t;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- special functions (special.hpp:12-30) ------------------------------------------------
int ref_sph_jn(int nmax, double zr, double zi, double* out) {
  return guarded([&] {
    std::vector<cplx> v(nmax + 1);
    sf::sph_jn(nmax, cplx(zr, zi), v.data());
    std::memcpy(out, v.data(), sizeof(cplx) * v.size());
  });
}
int ref_sph_hn(int nmax, double zr, double zi, double* out) {
  return guarded([&] {
    std::vector<cplx> v(nmax + 1);
    sf::sph_hn(nmax, cplx(zr, zi), v.data());
    std::memcpy(out, v.data(), sizeof(cplx) * v.size());
  });
}
int ref_ynm(int nmax, const double* dir, double* out) {
  return guarded([&] {
    std::vector<cplx> v(sf::nm_total(nmax));
    sf::ynm(nmax, Vec3{dir[0], dir[1], dir[2]}, v.data());
    std::memcpy(out, v.data(), sizeof(cplx) * v.size());
  });
}
double ref_wigner3j(int j1, int j2, int j3, int m1, int m2, int m3) {
  return sf::wigner3j(j1, j2, j3, m1, m2, m3);
}

// ---- expansion operators (expansion.hpp:15-88) ---------------------------------------------
// radial: 0 regular (M2M/L2L), 1 singular (M2L).  out: dim*dim complex, row-major.
int ref_translation_matrix(double kr, double ki, const double* t, int order, int radial,
                           double* out) {
  return guarded([&] {
    auto m = fmm::translation_matrix(WaveNumber{kr, ki}, Vec3{t[0], t[1], t[2]}, order,
                                     radial ? fmm::Radial::singular : fmm::Radial::regular);
    std::memcpy(out, m.data(), sizeof(cplx) * m.size());
  });
}
int ref_p2m(long n, const double* xyz, const double* q, const double* center, double kr,
            double ki, int order, double* out) {
  return guarded([&] {
    auto b = make_bodies(n, xyz, q);
    fmm::Expansion m;
    m.resize(order);
    fmm::p2m(b.data(), b.size(), Vec3{center[0], center[1], center[2]}, WaveNumber{kr, ki}, m);
    std::memcpy(out, m.coeff.data(), sizeof(cplx) * m.coeff.size());
  });
}
// which: 0 eval_multipole, 1 eval_local
int ref_eval_expansion(int which, int order, const double* coeff, const double* center,
                       const double* point, double kr, double ki, double* out) {
  return guarded([&] {
    fmm::Expansion e;
    e.resize(order);
    std::memcpy(e.coeff.data(), coeff, sizeof(cplx) * e.coeff.size());
    Vec3 c{center[0], center[1], center[2]}, p{point[0], point[1], point[2]};
    cplx v = which ? fmm::eval_local(e, c, p, WaveNumber{kr, ki})
                   : fmm::eval_multipole(e, c, p, WaveNumber{kr, ki});
    out[0] = v.real();
    out[1] = v.imag();
  });
}
int ref_calibrate_order(double kr, double ki, double diameter, double theta, double tol,
                        int max_order, int* out) {
  return guarded([&] {
    *out = fmm::calibrate_order(WaveNumber{kr, ki}, diameter, theta, tol, max_order);
  });
}

// ---- tree + traversal + pipeline (octree.hpp, traversal.hpp) -------------------------------
struct RefFmm {
  fmm::Octree tree;
  fmm::TraversalPlan plan;
  fmm::TraversalConfig tcfg;
  WaveNumber k;
  int order = 0;
  fmm::FmmStats stats;
};

// builds tree (build_tree, octree.cpp:142) and plan (dual_tree_traversal, traversal.cpp:82)
int ref_fmm_create(RefFmm** out, long n, const double* xyz, double kr, double ki, int order,
                   int ncrit, double leaf_cap, int s, double theta, double kd_max, int threads) {
  return guarded([&] {
    auto h = std::make_unique<RefFmm>();
    h->k = WaveNumber{kr, ki};
    h->order = order;
    h->tcfg = make_tcfg(ncrit, s, theta, kd_max, threads);
    h->tree = fmm::build_tree(make_bodies(n, xyz, nullptr), ncrit, leaf_cap);
    h->plan = fmm::dual_tree_traversal(h->tree, h->tree, h->k, h->tcfg);
    *out = h.release();
  });
}
void ref_fmm_destroy(RefFmm* h) { delete h; }

// counts: [0] cells [1] leaves [2] m2l pairs [3] p2p leaf pairs [4] p2p body pairs
//         [5] max level [6] m2l groups [7] p2p groups [8] max m2l list [9] max p2p list
void ref_fmm_counts(const RefFmm* h, long long* c) {
  c[0] = (long long)h->tree.cells.size();
  c[1] = (long long)h->tree.leaves.size();
  c[2] = (long long)h->plan.m2l_pairs;
  c[3] = (long long)h->plan.p2p_pairs;
  long long bp = 0, mx = 0, mm = 0;
  for (const auto& g : h->plan.p2p) {
    long long ns = 0;
    for (auto s : g.sources) ns += h->tree.cells[s].body_count;
    bp += ns * h->tree.cells[g.target].body_count;
    mx = std::max<long long>(mx, (long long)g.sources.size());
  }
  for (const auto& g : h->plan.m2l) mm = std::max<long long>(mm, (long long)g.sources.size());
  c[4] = bp;
  c[5] = h->tree.max_level_used;
  c[6] = (long long)h->plan.m2l.size();
  c[7] = (long long)h->plan.p2p.size();
  c[8] = mm;
  c[9] = mx;
}
// TraversalPlan::tasks (traversal.cpp:56-59) and FmmStats::starved_cells of the last execute_plan
long long ref_fmm_tasks(const RefFmm* h) { return (long long)h->plan.tasks; }
long long ref_fmm_starved(const RefFmm* h) { return (long long)h->stats.starved_cells; }
// per cell: level, ix, iy, iz, body_first, body_count, child_first, child_count (8 x u32)
void ref_fmm_cells(const RefFmm* h, unsigned* out) {
  for (size_t i = 0; i < h->tree.cells.size(); ++i) {
    const auto& c = h->tree.cells[i];
    unsigned* o = out + 8 * i;
    o[0] = unsigned(c.level); o[1] = c.ix; o[2] = c.iy; o[3] = c.iz;
    o[4] = c.body_first; o[5] = c.body_count; o[6] = c.child_first; o[7] = c.child_count;
  }
}
void ref_fmm_box(const RefFmm* h, double* lo_w) {
  lo_w[0] = h->tree.box.lo.x; lo_w[1] = h->tree.box.lo.y; lo_w[2] = h->tree.box.lo.z;
  lo_w[3] = h->tree.box.width;
}
void ref_fmm_body_order(const RefFmm* h, unsigned* out) {
  for (size_t i = 0; i < h->tree.bodies.size(); ++i) out[i] = h->tree.bodies[i].index;
}
// flattened plan: which 0 m2l, 1 p2p.  targets[g], offsets[g+1], sources[pairs]
void ref_fmm_plan(const RefFmm* h, int which, unsigned* targets, unsigned long long* offsets,
                  unsigned* sources) {
  const auto& groups = which ? h->plan.p2p : h->plan.m2l;
  unsigned long long off = 0;
  for (size_t g = 0; g < groups.size(); ++g) {
    targets[g] = groups[g].target;
    offsets[g] = off;
    for (auto s : groups[g].sources) sources[off++] = s;
  }
  offsets[groups.size()] = off;
}
// one matvec through execute_plan (traversal.cpp:208).  q, out in CALLER order (Body::index).
// f32_p2p selects kernel::Precision::f32 for the near field (traversal.cpp:267-271).
int ref_fmm_matvec(RefFmm* h, const double* q, int f32_p2p, double* out) {
  return guarded([&] {
    for (auto& b : h->tree.bodies) b.src = cplx(q[2 * b.index], q[2 * b.index + 1]);
    kernel::KernelConfig kc;
    kc.skip_same_patch = false;
    kc.near_patch_distance = 0;
    kc.precision = f32_p2p ? kernel::Precision::f32 : kernel::Precision::f64;
    h->stats = fmm::execute_plan(h->tree, h->tree, h->plan, h->k, h->order, h->tcfg, kc);
    for (const auto& b : h->tree.bodies) {
      out[2 * b.index] = b.trg.real();
      out[2 * b.index + 1] = b.trg.imag();
    }
  });
}
// seconds: upward, interaction, downward (FmmStats, traversal.hpp:44-52)
void ref_fmm_seconds(const RefFmm* h, double* s) {
  s[0] = h->stats.upward_seconds;
  s[1] = h->stats.interaction_seconds;
  s[2] = h->stats.downward_seconds;
}
// expansions after the last matvec: which 0 multipole, 1 local; out: ncells*dim complex
void ref_fmm_expansions(const RefFmm* h, int which, double* out) {
  const size_t dim = sf::nm_total(h->order);
  for (size_t i = 0; i < h->tree.cells.size(); ++i) {
    const auto& e = which ? h->tree.cells[i].local : h->tree.cells[i].multipole;
    if (e.allocated())
      std::memcpy(out + 2 * dim * i, e.coeff.data(), sizeof(cplx) * dim);
    else
      std::memset(out + 2 * dim * i, 0, sizeof(cplx) * dim);
  }
}

// FP64 direct sum at selected targets over all sources, the reference tests' own oracle
// (tests/test_fmm.cpp:59-72) expressed through kernel::green_t (kernel.hpp:16-23).
int ref_direct_sum(long n, const double* xyz, const double* q, double kr, double ki, long nt,
                   const long long* target_index, double* out) {
  return guarded([&] {
    WaveNumber k{kr, ki};
    for (long t = 0; t < nt; ++t) {
      const long long ti = target_index ? target_index[t] : t;
      Vec3 pt{xyz[3 * ti], xyz[3 * ti + 1], xyz[3 * ti + 2]};
      cplx acc = 0;
      for (long j = 0; j < n; ++j) {
        Vec3 ps{xyz[3 * j], xyz[3 * j + 1], xyz[3 * j + 2]};
        if ((pt - ps).norm2() == 0) continue;
        acc += kernel::green_t<double>(pt, ps, k) * cplx(q[2 * j], q[2 * j + 1]);
      }
      out[2 * t] = acc.real();
      out[2 * t + 1] = acc.imag();
    }
  });
}

// simulated multi-rank matvec (let.cpp:320-362) over an ORB plan (partition.cpp:102-135)
int ref_distributed_matvec(long n, const double* xyz, const double* q, double kr, double ki,
                           int order, int ncrit, double leaf_cap, int s, double theta,
                           double kd_max, int nranks, double* out, unsigned long long* let_bytes) {
  return guarded([&] {
    auto bodies = make_bodies(n, xyz, q);
    auto plan = part::orb_partition(bodies, nranks);
    part::DistributedRunConfig cfg;
    cfg.capacity = ncrit;
    cfg.max_leaf_diameter = leaf_cap;
    cfg.order = order;
    cfg.traversal = make_tcfg(ncrit, s, theta, kd_max, 1);
    auto run = part::distributed_matvec(bodies, plan, WaveNumber{kr, ki}, cfg);
    std::memcpy(out, run.potential.data(), sizeof(cplx) * n);
    if (let_bytes)
      for (int r = 0; r < nranks; ++r) let_bytes[r] = run.let_bytes[r];
  });
}

// ---- GMRES over a C callback (gmres.cpp:35-174) --------------------------------------------
typedef void (*ref_matvec_cb)(void* user, long n, const double* x, double* y);
// report: [0] iterations [1] converged [2] breakdown [3] rhs_norm [4] final_residual
int ref_gmres(ref_matvec_cb cb, void* user, long n, const double* rhs, double rtol, int restart,
              int max_iterations, double* x, double* report, double* residuals, int residual_cap) {
  return guarded([&] {
    solver::GmresConfig cfg;
    cfg.rtol = rtol;
    cfg.restart = restart;
    cfg.max_iterations = max_iterations;
    solver::MatVec apply = [&](std::span<const cplx> v) {
      std::vector<cplx> y(v.size());
      cb(user, long(v.size()), reinterpret_cast<const double*>(v.data()),
         reinterpret_cast<double*>(y.data()));
      return y;
    };
    std::span<const cplx> b(reinterpret_cast<const cplx*>(rhs), size_t(n));
    auto [sol, rep] = solver::gmres(apply, b, cfg);
    std::memcpy(x, sol.data(), sizeof(cplx) * n);
    report[0] = rep.iterations; report[1] = rep.converged; report[2] = rep.breakdown;
    report[3] = rep.rhs_norm; report[4] = rep.final_residual;
    for (int i = 0; i < residual_cap && i < int(rep.residuals.size()); ++i)
      residuals[i] = rep.residuals[i];
  });
}

// ---- BIE system (solver.hpp:44-143) ---------------------------------------------------------
struct RefBie {
  solver::DiscreteSystem sys;
};

// patches: npatch * 18 doubles (6 nodes x xyz).  mode: 0 none, 1 self_only, 2 self_near.
int ref_bie_create(RefBie** out, long npatch, const double* nodes, int basis_order, double kr,
                   double ki, int mode, int use_tree, int order, int ncrit, int s, double theta,
                   double kd_max, double leaf_cap, int threads) {
  return guarded([&] {
    std::vector<geom::CurvilinearPatch> patches(npatch);
    for (long p = 0; p < npatch; ++p) {
      for (int j = 0; j < 6; ++j)
        patches[p].node[j] = Vec3{nodes[18 * p + 3 * j], nodes[18 * p + 3 * j + 1],
                                  nodes[18 * p + 3 * j + 2]};
      patches[p].id = std::int32_t(p);
    }
    solver::OperatorConfig op;
    op.use_tree = use_tree != 0;
    op.expansion_order = order;
    op.leaf_diameter_cap = leaf_cap;
    op.traversal = make_tcfg(ncrit, s, theta, kd_max, threads);
    auto h = std::make_unique<RefBie>();
    h->sys = solver::build_system(std::move(patches), basis_order, WaveNumber{kr, ki},
                                  solver::SingularityMode(mode), kernel::KernelConfig{}, op);
    *out = h.release();
  });
}
void ref_bie_destroy(RefBie* h) { delete h; }
// sizes: [0] n [1] basis_count [2] near nnz [3] expansion_order [4] has block_lu
void ref_bie_sizes(const RefBie* h, long long* s) {
  s[0] = (long long)h->sys.size();
  s[1] = h->sys.basis_count();
  s[2] = (long long)h->sys.near_delta.size();
  s[3] = h->sys.expansion_order;
  s[4] = h->sys.block_lu.empty() ? 0 : 1;
}
void ref_bie_samples(const RefBie* h, double* xyz, double* far_weight) {
  for (size_t i = 0; i < h->sys.size(); ++i) {
    xyz[3 * i] = h->sys.samples[i].position.x;
    xyz[3 * i + 1] = h->sys.samples[i].position.y;
    xyz[3 * i + 2] = h->sys.samples[i].position.z;
    far_weight[i] = h->sys.far_weight[i];
  }
}
void ref_bie_corrections(const RefBie* h, double* patch_block, double* block_lu, int* block_piv,
                         unsigned* near_offset, unsigned* near_source, double* near_delta) {
  const auto& s = h->sys;
  if (patch_block) std::memcpy(patch_block, s.patch_block.data(), sizeof(cplx) * s.patch_block.size());
  if (block_lu) std::memcpy(block_lu, s.block_lu.data(), sizeof(cplx) * s.block_lu.size());
  if (block_piv) std::memcpy(block_piv, s.block_piv.data(), sizeof(int) * s.block_piv.size());
  if (near_offset) std::memcpy(near_offset, s.near_offset.data(), sizeof(unsigned) * s.near_offset.size());
  if (near_source) std::memcpy(near_source, s.near_source.data(), sizeof(unsigned) * s.near_source.size());
  if (near_delta) std::memcpy(near_delta, s.near_delta.data(), sizeof(cplx) * s.near_delta.size());
}
int ref_bie_rhs(const RefBie* h, const double* dir, double kr, double ki, double* out) {
  return guarded([&] {
    solver::IncidentWave w;
    w.direction = Vec3{dir[0], dir[1], dir[2]};
    w.k = WaveNumber{kr, ki};
    auto rhs = solver::assemble_rhs(h->sys, w);
    std::memcpy(out, rhs.data(), sizeof(cplx) * rhs.size());
  });
}
int ref_bie_apply(RefBie* h, const double* x, double* y) {
  return guarded([&] {
    std::span<const cplx> xs(reinterpret_cast<const cplx*>(x), h->sys.size());
    auto r = solver::apply_operator(h->sys, xs);
    std::memcpy(y, r.data(), sizeof(cplx) * r.size());
  });
}
int ref_bie_gmres(RefBie* h, const double* rhs, double rtol, int restart, int max_iterations,
                  int precondition, double* x, double* report, double* residuals,
                  int residual_cap) {
  return guarded([&] {
    solver::GmresConfig cfg;
    cfg.rtol = rtol;
    cfg.restart = restart;
    cfg.max_iterations = max_iterations;
    cfg.precondition = precondition != 0;
    std::span<const cplx> b(reinterpret_cast<const cplx*>(rhs), h->sys.size());
    auto [sol, rep] = solver::gmres_solve(h->sys, b, cfg);
    std::memcpy(x, sol.data(), sizeof(cplx) * sol.size());
    report[0] = rep.iterations; report[1] = rep.converged; report[2] = rep.breakdown;
    report[3] = rep.rhs_norm; report[4] = rep.final_residual;
    for (int i = 0; i < residual_cap && i < int(rep.residuals.size()); ++i)
      residuals[i] = rep.residuals[i];
  });
}
int ref_bie_scattered(const RefBie* h, const double* solution, long nobs, const double* obs,
                      double kr, double ki, double* out) {
  return guarded([&] {
    std::span<const cplx> sol(reinterpret_cast<const cplx*>(solution), h->sys.size());
    std::vector<Vec3> o(nobs);
    for (long i = 0; i < nobs; ++i) o[i] = Vec3{obs[3 * i], obs[3 * i + 1], obs[3 * i + 2]};
    auto r = solver::evaluate_scattered_field(h->sys, sol, o, WaveNumber{kr, ki});
    std::memcpy(out, r.data(), sizeof(cplx) * r.size());
  });
}

// lat-long sphere mesh (mesh_gen.cpp:19-55): returns element count; nodes may be null to query
long ref_sphere_mesh(double radius, int segments, int rings, double* nodes) {
  auto mesh = meshio::sphere_mesh(radius, segments, rings);
  if (nodes)
    for (size_t e = 0; e < mesh.elements.size(); ++e)
      for (int j = 0; j < 6; ++j) {
        nodes[18 * e + 3 * j] = mesh.elements[e].node[j].x;
        nodes[18 * e + 3 * j + 1] = mesh.elements[e].node[j].y;
        nodes[18 * e + 3 * j + 2] = mesh.elements[e].node[j].z;
      }
  return long(mesh.elements.size());
}

// Mie series (oracle.cpp:11-59); obs: nobs x (r, theta, phi)
int ref_mie_soft_sphere(double radius, double kr, double ki, long nobs, const double* obs,
                        double* out) {
  return guarded([&] {
    oracle::MieConfig cfg;
    cfg.radius = radius;
    cfg.k = WaveNumber{kr, ki};
    cfg.observations.resize(nobs);
    for (long i = 0; i < nobs; ++i)
      cfg.observations[i] = oracle::SphericalPoint{obs[3 * i], obs[3 * i + 1], obs[3 * i + 2]};
    auto v = oracle::mie_soft_sphere(cfg);
    std::memcpy(out, v.data(), sizeof(cplx) * v.size());
  });
}

// quadrature / interpolation tables of geometry.cpp, the inputs of the correction builders
// (solver.cpp:80-230): exported so tests can hand the reference's own rules to the device builder
int ref_geom_basis(int order, double* nodes, double* weights) {
  const auto& b = geom::lagrange_basis(order);
  for (int j = 0; j < b.count(); ++j) {
    if (nodes) {
      nodes[2 * j] = b.nodes()[j][0];
      nodes[2 * j + 1] = b.nodes()[j][1];
    }
    if (weights) weights[j] = b.weights()[j];
  }
  return b.count();
}
void ref_geom_basis_eval(int order, double zeta, double eta, double* out) {
  const auto v = geom::lagrange_basis(order).eval(zeta, eta);
  std::memcpy(out, v.data(), sizeof(double) * v.size());
}
int ref_geom_gauss_rule(int npoints, double* pts) {  // pts: npoints x (zeta, eta, weight)
  const auto& r = geom::gauss_rule(npoints);
  if (pts)
    for (size_t i = 0; i < r.pts.size(); ++i) {
      pts[3 * i] = r.pts[i].zeta;
      pts[3 * i + 1] = r.pts[i].eta;
      pts[3 * i + 2] = r.pts[i].weight;
    }
  return int(r.pts.size());
}
int ref_geom_duffy_rule(double zeta0, double eta0, int n_per_dim, double* pts) {
  const auto r = geom::duffy_rule(zeta0, eta0, n_per_dim);
  if (pts)
    for (size_t i = 0; i < r.size(); ++i) {
      pts[3 * i] = r[i].zeta;
      pts[3 * i + 1] = r[i].eta;
      pts[3 * i + 2] = r[i].weight;
    }
  return int(r.size());
}

// repartitioning loop (partition.cpp:137-227): per-body work estimates and the alpha search
void ref_measure_weights(const RefFmm* h, double* local, double* remote) {
  const auto w = part::measure_weights(h->tree, h->plan);
  std::memcpy(local, w.local.data(), sizeof(double) * w.local.size());
  std::memcpy(remote, w.remote.data(), sizeof(double) * w.remote.size());
}
int ref_update_alpha(const double* alpha, const double* runtime, int n, double alpha_max, double* next) {
  return guarded([&] {
    std::vector<part::AlphaSample> hist(n);
    for (int i = 0; i < n; ++i) hist[i] = part::AlphaSample{alpha[i], runtime[i]};
    *next = part::update_alpha(hist, alpha_max);
  });
}

// mesh files of mesh_io.cpp written by the reference itself (fixtures for the readers of the CLI)
int ref_write_sphere_mesh(double radius, int segments, int rings, const char* gmsh_path, const char* binary_path) {
  return guarded([&] {
    const auto mesh = meshio::sphere_mesh(radius, segments, rings);
    if (gmsh_path) {
      std::ofstream f(gmsh_path);
      meshio::write_gmsh(mesh, f);
    }
    if (binary_path) {
      std::ofstream f(binary_path, std::ios::binary);
      meshio::write_binary(mesh, f);
    }
  });
}

}  // extern "C"
