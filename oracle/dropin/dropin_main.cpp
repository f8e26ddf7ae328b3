// oracle/dropin/dropin_main.cpp — a program written against the REFERENCE's headers only (hfmm/solver.hpp,
// hfmm/mesh_gen.hpp): sphere scattering set up by the reference (mesh, patches, build_system with its CPU
// correction builders, assemble_rhs), then apply_operator and gmres_solve — which, in this binary, are the
// drop-in replacements of solver_gpu.cpp — compared with the reference's own CPU implementations of the
// same two functions (apply_operator_host / gmres_solve_host, compiled from the unmodified solver.cpp).
// Exit 0 = all checks passed, 3 = no CUDA device.  Test infrastructure; run by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "hfmm/mesh_gen.hpp"
#include "hfmm/solver.hpp"

namespace hfmm::solver {
std::vector<cplx> apply_operator_host(DiscreteSystem& sys, std::span<const cplx> x);
std::pair<std::vector<cplx>, SolveReport> gmres_solve_host(DiscreteSystem& sys, std::span<const cplx> rhs,
                                                           const GmresConfig& cfg);
void release_device(DiscreteSystem& sys);
}  // namespace hfmm::solver

using namespace hfmm;

static double rel_l2(const std::vector<cplx>& a, const std::vector<cplx>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += std::norm(a[i] - b[i]);
    den += std::norm(b[i]);
  }
  return std::sqrt(num / den);
}

static int failures = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (!(cond)) {                                                \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                 \
    }                                                             \
  } while (0)

int main(int argc, char** argv) {
  const int segments = argc > 1 ? std::atoi(argv[1]) : 12, rings = argc > 2 ? std::atoi(argv[2]) : 8;
  const double kr = argc > 3 ? std::atof(argv[3]) : 2.5;
  const WaveNumber k{kr, 0.0};
  auto mesh = meshio::sphere_mesh(1.0, segments, rings);
  solver::OperatorConfig op;
  op.use_tree = true;
  op.expansion_order = 10;
  op.traversal.s = 64;
  op.traversal.c = 32;
  op.traversal.theta = 0.4;
  op.traversal.deterministic = false;
  solver::DiscreteSystem sys = solver::build_system(mesh.as_patches(), 1, k, solver::SingularityMode::self_near,
                                                    kernel::KernelConfig{}, op);
  std::printf("reference system: %zu patches, %zu unknowns, order %d, near nnz %zu\n", sys.patches.size(),
              sys.size(), sys.expansion_order, sys.near_delta.size());
  solver::IncidentWave wave;
  wave.k = k;
  wave.direction = Vec3{0.36, 0.48, 0.8};  // a generic direction: off the symmetry axis of the lat-long mesh
  const std::vector<cplx> rhs = solver::assemble_rhs(sys, wave);

  // seam B2: apply_operator
  std::vector<cplx> y_gpu;
  try {
    y_gpu = solver::apply_operator(sys, rhs);
  } catch (const std::exception& e) {
    if (std::strstr(e.what(), "no CUDA device")) {
      std::printf("no CUDA device: %s\n", e.what());
      return 3;
    }
    throw;
  }
  const std::vector<cplx> y_cpu = solver::apply_operator_host(sys, rhs);
  const double e_apply = rel_l2(y_gpu, y_cpu);
  std::printf("apply_operator: rel L2 (GPU vs reference) = %.3e\n", e_apply);
  CHECK(e_apply < 1e-5);  // north star: 1e-5 in complex FP32
  bool threw = false;
  try {
    std::vector<cplx> shortv(sys.size() - 1);
    solver::apply_operator(sys, shortv);
  } catch (const config_error&) {
    threw = true;
  }
  CHECK(threw);  // solver.cpp:315-316

  // seam B1: gmres_solve, with and without the block-Jacobi right preconditioner
  solver::GmresConfig cfg;
  cfg.rtol = 1e-4;
  cfg.restart = 30;
  cfg.max_iterations = 400;
  for (int pre = 1; pre >= 0; --pre) {
    cfg.precondition = pre != 0;
    auto gpu = solver::gmres_solve(sys, rhs, cfg);
    auto cpu = solver::gmres_solve_host(sys, rhs, cfg);
    std::printf("gmres_solve precondition=%d: iterations GPU %d, reference %d; final residual %.3e / %.3e; "
                "solution rel L2 %.3e\n", pre, gpu.second.iterations, cpu.second.iterations,
                gpu.second.final_residual, cpu.second.final_residual, rel_l2(gpu.first, cpu.first));
    CHECK(gpu.second.converged && cpu.second.converged);
    CHECK(std::abs(gpu.second.iterations - cpu.second.iterations) <= 1);  // north star: same count +- 1
    CHECK(gpu.second.final_residual <= 1.05e-4);
    CHECK(rel_l2(gpu.first, cpu.first) < 5e-3);  // both are 1e-4-residual solutions
    CHECK(gpu.second.residuals.size() == size_t(gpu.second.iterations));
    CHECK(gpu.second.seconds.size() == size_t(gpu.second.iterations));
    CHECK(gpu.second.matvec_seconds.size() == size_t(gpu.second.iterations));
    CHECK(sys.solution.size() == sys.size());
  }

  // The degenerate case: wave along the polar axis of the lat-long mesh.  The all-FP64 solve then stays in
  // the invariant subspace of the mesh's rotational symmetry and stops early; any FP32-sized rounding breaks
  // the symmetry.  The reference's OWN single-precision near field (kernel::Precision::f32) is the yardstick:
  // the GPU path must not need more iterations than that (plus slack), and must still converge to 1e-4.
  {
    solver::IncidentWave axial;
    axial.k = k;
    const std::vector<cplx> rhs_z = solver::assemble_rhs(sys, axial);
    cfg.precondition = false;
    auto gpu = solver::gmres_solve(sys, rhs_z, cfg);
    auto cpu64 = solver::gmres_solve_host(sys, rhs_z, cfg);
    sys.kernel_cfg.precision = kernel::Precision::f32;
    auto cpu32 = solver::gmres_solve_host(sys, rhs_z, cfg);
    sys.kernel_cfg.precision = kernel::Precision::f64;
    std::printf("axial wave (symmetric problem): iterations GPU %d, reference FP64 %d, reference with its f32 near "
                "field %d\n", gpu.second.iterations, cpu64.second.iterations, cpu32.second.iterations);
    CHECK(gpu.second.converged && gpu.second.final_residual <= 1.05e-4);
    CHECK(gpu.second.iterations <= cpu32.second.iterations + cpu32.second.iterations / 4 + 2);
    CHECK(rel_l2(gpu.first, cpu64.first) < 5e-3);
  }

  // the exterior field of the reference, fed with the GPU solution
  std::vector<Vec3> obs{Vec3{0, 0, 3.0}, Vec3{2.5, 0, 0}, Vec3{0, -2.0, 2.0}};
  auto f = solver::evaluate_scattered_field(sys, sys.solution, obs, k);
  CHECK(std::isfinite(f[0].real()) && std::abs(f[0]) > 0);
  solver::release_device(sys);
  if (failures) {
    std::printf("%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("all checks passed\n");
  return 0;
}
