// oracle/dropin/solver_gpu.cpp — the binding of INTEGRATION.md section 2, applied to the ACTUAL reference.
//
// TEST INFRASTRUCTURE (like everything under oracle/): this translation unit compiles the reference's own
// solver.cpp, unmodified and where it lies (-I$(REF)/src), with its two seams renamed by the preprocessor —
//     solver::apply_operator -> solver::apply_operator_host      (solver.cpp:314-359)
//     solver::gmres_solve    -> solver::gmres_solve_host         (solver.cpp:361-391)
// — and defines those two names again, with the reference's signatures, routed through the C ABI of
// include/hfmm_cuda.h.  Every other reference object (octree, traversal, expansion, kernel, geometry, gmres,
// mesh_gen, ...) is linked unchanged, so a program written against the reference's headers — build_system,
// assemble_rhs, gmres_solve, evaluate_scattered_field — runs its matvecs and its Krylov loop on the GPU
// without a changed line.  The handle is kept in a side table because DiscreteSystem cannot gain a member
// without editing solver.hpp (the maintainer's patch adds `hfmm_cuda_t* device`).
#include <map>
#include <mutex>
#include <stdexcept>

#include "hfmm_cuda.h"

#define apply_operator apply_operator_host
#define gmres_solve gmres_solve_host
#include "solver.cpp"  // the reference's, found through -I$(REF)/src
#undef apply_operator
#undef gmres_solve

namespace hfmm::solver {

namespace {

void check(hfmm_cuda_t* h, int rc) {  // status -> the reference's own exceptions
  if (!rc) return;
  const std::string msg = hfmm_cuda_last_error(h);
  switch (rc) {
    case HFMM_ERR_CONFIG: throw config_error(msg);
    case HFMM_ERR_SINGULAR: throw singular_error(msg);
    case HFMM_ERR_STRUCTURAL: throw structural_error(msg);
    case HFMM_ERR_ACCURACY: throw accuracy_error(msg);
    case HFMM_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

std::mutex g_mutex;
std::map<const DiscreteSystem*, hfmm_cuda_t*> g_device;  // stands in for DiscreteSystem::device

hfmm_cuda_t* device_of(DiscreteSystem& sys) {
  std::lock_guard<std::mutex> lock(g_mutex);
  auto it = g_device.find(&sys);
  if (it != g_device.end()) return it->second;
  const auto& t = sys.op_cfg.traversal;
  hfmm_cuda_config c{};
  c.wave_r = sys.k.wave_r;
  c.wave_i = sys.k.wave_i;
  c.order = sys.expansion_order;  // after calibrate_order, as the reference (solver.cpp:244-257)
  c.ncrit = t.c;
  c.grain = t.s;
  c.theta = t.theta;
  c.kd_max = t.kd_max;
  c.leaf_cap = sys.op_cfg.leaf_diameter_cap > 0 ? sys.op_cfg.leaf_diameter_cap : -1.0;  // -1: kd_max/|k|
  c.flags = t.deterministic ? HFMM_FLAG_DETERMINISTIC : 0;
  hfmm_cuda_t* h = nullptr;
  check(nullptr, hfmm_cuda_create(&h, &c));
  std::vector<double> xyz(3 * sys.size());
  for (std::size_t i = 0; i < sys.size(); ++i) {
    xyz[3 * i] = sys.samples[i].position.x;
    xyz[3 * i + 1] = sys.samples[i].position.y;
    xyz[3 * i + 2] = sys.samples[i].position.z;
  }
  check(h, hfmm_cuda_set_points(h, xyz.data(), sys.size()));
  check(h, hfmm_cuda_set_corrections(
               h, sys.basis_count(), sys.far_weight.data(), reinterpret_cast<const double*>(sys.patch_block.data()),
               sys.near_offset.empty() ? nullptr : sys.near_offset.data(),
               sys.near_source.empty() ? nullptr : sys.near_source.data(),
               sys.near_delta.empty() ? nullptr : reinterpret_cast<const double*>(sys.near_delta.data()),
               sys.block_lu.empty() ? nullptr : reinterpret_cast<const double*>(sys.block_lu.data()),
               sys.block_piv.empty() ? nullptr : sys.block_piv.data()));
  std::vector<double> diam(sys.patches.size());
  for (std::size_t p = 0; p < sys.patches.size(); ++p) diam[p] = sys.patches[p].diameter();
  check(h, hfmm_cuda_set_patch_diameters(h, diam.data(), diam.size()));
  g_device[&sys] = h;
  return h;
}

}  // namespace

void release_device(DiscreteSystem& sys) {  // what ~DiscreteSystem would do with its `device` member
  std::lock_guard<std::mutex> lock(g_mutex);
  auto it = g_device.find(&sys);
  if (it == g_device.end()) return;
  hfmm_cuda_destroy(it->second);
  g_device.erase(it);
}

std::vector<cplx> apply_operator(DiscreteSystem& sys, std::span<const cplx> x) {
  if (x.size() != sys.size()) throw config_error("apply_operator: coefficient vector length mismatch");
  if (!sys.op_cfg.use_tree) return apply_operator_host(sys, x);  // the dense path stays where it is
  hfmm_cuda_t* h = device_of(sys);
  std::vector<cplx> y(x.size());
  check(h, hfmm_cuda_matvec(h, reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data())));
  return y;
}

std::pair<std::vector<cplx>, SolveReport> gmres_solve(DiscreteSystem& sys, std::span<const cplx> rhs,
                                                      const GmresConfig& cfg) {
  if (!sys.op_cfg.use_tree) return gmres_solve_host(sys, rhs, cfg);
  if (rhs.size() != sys.size()) throw config_error("gmres_solve: right-hand side length mismatch");
  hfmm_cuda_t* h = device_of(sys);  // Krylov vectors stay on the GPU
  hfmm_gmres_config c{cfg.rtol, cfg.restart, cfg.max_iterations, cfg.precondition ? 1 : 0};
  std::vector<double> res(std::size_t(std::max(cfg.max_iterations, 0)) + 1), sec(res.size()), mv(res.size());
  hfmm_gmres_report r{};
  r.seconds_history = sec.data();
  r.matvec_seconds_history = mv.data();
  r.history_cap = int(res.size());
  std::vector<cplx> x(rhs.size());
  check(h, hfmm_cuda_gmres(h, reinterpret_cast<const double*>(rhs.data()), reinterpret_cast<double*>(x.data()), &c,
                           &r, res.data(), int(res.size())));
  SolveReport rep;
  rep.iterations = r.iterations;
  rep.converged = r.converged != 0;
  rep.breakdown = r.breakdown != 0;
  rep.rhs_norm = r.rhs_norm;
  rep.final_residual = r.final_residual;
  rep.residuals.assign(res.begin(), res.begin() + r.iterations);
  rep.seconds.assign(sec.begin(), sec.begin() + r.iterations);
  rep.matvec_seconds.assign(mv.begin(), mv.begin() + r.iterations);
  sys.solution = x;
  return {std::move(x), std::move(rep)};
}

}  // namespace hfmm::solver
