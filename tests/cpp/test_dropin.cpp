// tests/cpp/test_dropin.cpp — the reference's own FMM test cases, restated against the C++ mirror
// (include/hfmm_b200.hpp) of the reference interface.  Built by __graft_entry__.build(); run by
// tests/test_gpu_cpp_mirror.py on the GPU box.  Exit 0 = all passed, 3 = no CUDA device.
//
//   pipeline vs direct sum        reference tests/test_fmm.cpp:941-961 (1000 pts, k=2, P=10)
//   linearity                     reference tests/test_fmm.cpp:985-1022
//   config errors                 reference tests/test_fmm.cpp:897-939, traversal.cpp:16-21
//   operator length check         reference tests/test_solver.cpp:180-195, solver.cpp:315-316
//   GMRES over the tree operator  reference tests/test_solver.cpp:480-494
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "hfmm_b200.hpp"

using namespace hfmm_b200;

static int failures = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    if (!(cond)) {                                                          \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);           \
      ++failures;                                                           \
    }                                                                       \
  } while (0)

static cplx green(const Vec3& a, const Vec3& b, double k) {
  const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z, R = std::sqrt(dx * dx + dy * dy + dz * dz);
  return std::polar(1.0 / (4 * 3.14159265358979323846 * R), k * R);
}

static double rel_l2(const std::vector<cplx>& a, const std::vector<cplx>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += std::norm(a[i] - b[i]);
    den += std::norm(b[i]);
  }
  return std::sqrt(num / den);
}

int main() {
  std::mt19937_64 rng(2024);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  const int n = 1000;
  const double k = 2.0;
  std::vector<fmm::Body> bodies(n);
  for (auto& b : bodies) {
    b.position = Vec3{u(rng), u(rng), u(rng)};
    b.src = cplx(u(rng), u(rng));
  }
  fmm::TraversalConfig cfg;
  cfg.s = 40;
  cfg.c = 20;
  cfg.theta = 0.5;
  try {
    fmm::fmm_evaluate(bodies, WaveNumber{k, 0}, 10, cfg, 0.5);
  } catch (const device_error& e) {
    std::printf("no CUDA device: %s\n", e.what());
    return 3;
  }
  std::vector<cplx> exact(n), got(n);
  for (int i = 0; i < n; ++i) {
    cplx acc = 0;
    for (int j = 0; j < n; ++j)
      if (j != i) acc += green(bodies[i].position, bodies[j].position, k) * bodies[j].src;
    exact[i] = acc;
    got[i] = bodies[i].trg;
  }
  const double err = rel_l2(got, exact);
  std::printf("pipeline vs direct sum: rel L2 = %.3e (reference bound 1e-6 in FP64; ours 1e-5 in FP32)\n", err);
  CHECK(err < 1e-5);

  // linearity: A(a x + y) = a A x + A y
  std::vector<Vec3> pts(n);
  for (int i = 0; i < n; ++i) pts[i] = bodies[i].position;
  fmm::DeviceTree tree(pts, WaveNumber{k, 0}, 10, cfg, 0.5);
  std::vector<cplx> x(n), y(n), z(n), ax, ay, az;
  const cplx a(0.7, -1.3);
  for (int i = 0; i < n; ++i) {
    x[i] = cplx(u(rng), u(rng));
    y[i] = cplx(u(rng), u(rng));
    z[i] = a * x[i] + y[i];
  }
  fmm::execute_plan(tree, x, ax);
  fmm::execute_plan(tree, y, ay);
  const fmm::FmmStats st = fmm::execute_plan(tree, z, az);
  for (int i = 0; i < n; ++i) ax[i] = a * ax[i] + ay[i];
  CHECK(rel_l2(az, ax) < 5e-6);
  CHECK(st.m2l_pairs > 0 && st.p2p_pairs > 0);

  // bitwise determinism (test_fmm.cpp:1024-1050): TraversalConfig::deterministic is true by default,
  // a replay and a second tree give the same bits
  std::vector<cplx> az2, az3;
  fmm::execute_plan(tree, z, az2);
  CHECK(std::memcmp(az.data(), az2.data(), n * sizeof(cplx)) == 0);
  {
    fmm::DeviceTree tree2(pts, WaveNumber{k, 0}, 10, cfg, 0.5);
    fmm::execute_plan(tree2, z, az3);
    CHECK(std::memcmp(az.data(), az3.data(), n * sizeof(cplx)) == 0);
  }

  // malformed configurations are config_error, as in the reference
  auto throws_config = [&](fmm::TraversalConfig c, int order) {
    try {
      fmm::DeviceTree t(pts, WaveNumber{k, 0}, order, c);
    } catch (const config_error&) {
      return true;
    } catch (...) {
    }
    return false;
  };
  fmm::TraversalConfig bad = cfg;
  bad.s = 10;  // s < c
  CHECK(throws_config(bad, 8));
  bad = cfg;
  bad.theta = 0;
  CHECK(throws_config(bad, 8));
  bad = cfg;
  bad.theta = 1.5;
  CHECK(throws_config(bad, 8));
  CHECK(throws_config(cfg, -1));

  // operator: length check, then GMRES over the (shifted) tree operator converges
  solver::DeviceOperator op(pts, WaveNumber{k, 0}, 8, cfg, -1.0);
  std::vector<cplx> diag(n, cplx(400.0, 0.0));
  op.set_corrections(1, {}, diag, {}, {}, {}, {}, {});
  bool threw = false;
  try {
    solver::apply_operator(op, std::vector<cplx>(n + 1));
  } catch (const config_error&) {
    threw = true;
  }
  CHECK(threw);
  solver::GmresConfig g;
  g.rtol = 1e-5;
  g.restart = 30;
  g.max_iterations = 200;
  auto [sol, rep] = solver::gmres_solve(op, y, g);
  std::printf("gmres: %d iterations, final residual %.3e\n", rep.iterations, rep.final_residual);
  CHECK(rep.converged);
  std::vector<cplx> back = solver::apply_operator(op, sol);
  CHECK(rel_l2(back, y) < 5e-5);
  solver::MatVec mv = solver::as_matvec(op);
  CHECK(rel_l2(mv(sol), back) < 1e-6);

  std::printf(failures ? "%d check(s) FAILED\n" : "all checks passed\n", failures);
  return failures ? 1 : 0;
}
