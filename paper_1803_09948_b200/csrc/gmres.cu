// gmres.cu — Engine methods of the BIE layer: apply_operator, block-Jacobi preconditioner,
// restarted GMRES with device-resident Krylov vectors, exterior field evaluation.
//
// The iteration mirrors the reference's gmres (src/gmres.cpp:35-174) step for step — x0 = 0,
// modified Gram-Schmidt plus one unconditional re-orthogonalisation pass, complex Givens in FP64
// on the host, stop on |g_{j+1}| <= rtol ||b||, true residual recomputed at restarts and on exit —
// so the iteration count can be compared with the reference's (north star: same count +-1).
#include <chrono>
#include <cmath>
#include <complex>

#include "engine.hpp"

namespace hfmm_b200 {

namespace {
using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846264338327950288;

}  // namespace

void Engine::set_corrections(int ni, const double* far_weight, const double* patch_block,
                             const uint32_t* near_offset, const uint32_t* near_source,
                             const double* near_delta, const double* block_lu, const int32_t* block_piv) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const size_t n = tree_.n_bodies;
  if (ni < 1 || n % size_t(ni) != 0)
    throw Error(HFMM_ERR_CONFIG, "basis count must divide the number of unknowns");
  ni_ = ni;
  const size_t npatch = n / size_t(ni);
  have_weight_ = far_weight != nullptr;
  if (have_weight_) {
    std::vector<float> w(n);
    for (size_t i = 0; i < n; ++i) w[i] = float(far_weight[i]);
    far_weight_.upload(w, stream_);
  }
  have_block_ = patch_block != nullptr;
  if (have_block_) patch_block_.upload(reinterpret_cast<const double2*>(patch_block), npatch * ni * ni, stream_);
  have_near_ = near_offset && near_source && near_delta && near_offset[n] > 0;
  if (have_near_) {
    for (size_t i = 0; i < n; ++i)
      if (near_offset[i] > near_offset[i + 1]) throw Error(HFMM_ERR_STRUCTURAL, "near CSR offsets decrease");
    const size_t nnz = near_offset[n];
    for (size_t e = 0; e < nnz; ++e)
      if (near_source[e] >= n) throw Error(HFMM_ERR_STRUCTURAL, "near CSR source out of range");
    near_offset_.upload(near_offset, n + 1, stream_);
    near_source_.upload(near_source, nnz, stream_);
    near_delta_.upload(reinterpret_cast<const double2*>(near_delta), nnz, stream_);
  }
  have_lu_ = block_lu && block_piv;
  if (have_lu_) {
    for (size_t i = 0; i < n; ++i)
      if (block_piv[i] < 0 || block_piv[i] >= ni) throw Error(HFMM_ERR_STRUCTURAL, "pivot out of range");
    block_lu_.upload(reinterpret_cast<const double2*>(block_lu), npatch * ni * ni, stream_);
    block_piv_.upload(block_piv, n, stream_);
  }
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

// y = FMM(x * far_weight) + blockdiag x + CSR x     (reference solver.cpp:314-359), caller order
void Engine::apply_operator_device(const float2* x, float2* y) {
  const uint32_t n = tree_.n_bodies;
  launch_gather_charges(nullptr, x, body_index_.get(), have_weight_ ? far_weight_.get() : nullptr,
                        body_q_.get(), n, stream_);
  run_far_and_near();
  launch_scatter_potentials(near_.get(), far_.get(), body_index_.get(), nullptr, y, n, stream_);
  if (have_block_ || have_near_)
    launch_corrections(n, ni_, have_block_ ? patch_block_.get() : nullptr, near_offset_.get(),
                       near_source_.get(), have_near_ ? near_delta_.get() : nullptr, x, y, stream_);
}

namespace {
// body_q[first + i] = in[i] * weight[index[first + i]]: an owned Morton slice becomes the rank's charges
__global__ void __launch_bounds__(256)
owned_charges_kernel(const float2* __restrict__ in, const uint32_t* __restrict__ index, const float* __restrict__ weight,
                     float2* __restrict__ body_q, uint32_t first, uint32_t count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  float2 v = in[i];
  if (weight) {
    const float w = weight[index[first + i]];
    v.x *= w;
    v.y *= w;
  }
  body_q[first + i] = v;
}
}  // namespace

void Engine::gmres(const double* rhs, double* x_out, const hfmm_gmres_config& cfg, hfmm_gmres_report* rep,
                   double* residuals, int residual_cap) {
  gmres_impl(false, rhs, x_out, cfg, rep, residuals, residual_cap);
}

// GMRES over Morton-sharded vectors through the handle's communicator (comm.cu); see hfmm_cuda.h
void Engine::dist_solve(const double* rhs_owned, double* x_owned, const hfmm_gmres_config& cfg,
                        hfmm_gmres_report* rep, double* residuals, int residual_cap) {
  if (!transport_ && nranks_ > 1)
    throw Error(HFMM_ERR_CONFIG, "no communicator: call hfmm_cuda_comm_init_nccl / _host first");
  gmres_impl(true, rhs_owned, x_owned, cfg, rep, residuals, residual_cap);
}

// One iteration loop for both layouts.  sharded = false: vectors of all n unknowns in caller order, the
// operator is apply_operator.  sharded = true: every rank holds the slice [own_first_, own_first_ + own_count_)
// of each Krylov vector in Morton order; inner products are local FP64 reductions all-reduced IN PLACE ON THE
// DEVICE (stream-ordered, no host round trip per coefficient), the operator runs the two exchanges of comm.cu.
// All ranks see identical reduced scalars and therefore take identical branches (restart, convergence,
// breakdown).  The iteration itself is the reference's (gmres.cpp:35-174).
void Engine::gmres_impl(bool sharded, const double* rhs, double* x_out, const hfmm_gmres_config& cfg,
                        hfmm_gmres_report* rep, double* residuals, int residual_cap) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  // validation as gmres.cpp:25-31
  if (!(cfg.rtol > 0.0 && cfg.rtol < 1.0)) throw Error(HFMM_ERR_CONFIG, "gmres: rtol must lie in (0, 1)");
  if (cfg.restart < 1) throw Error(HFMM_ERR_CONFIG, "gmres: restart must be >= 1");
  if (cfg.max_iterations < 1) throw Error(HFMM_ERR_CONFIG, "gmres: max_iterations must be >= 1");
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  const uint32_t n_all = tree_.n_bodies;
  const uint32_t n = sharded ? own_count_ : n_all, first = sharded ? own_first_ : 0;
  const size_t ld = std::max<uint32_t>(n, 1);  // leading dimension of the Krylov basis
  const int m = cfg.restart;
  const bool precond = cfg.precondition && have_lu_;
  const bool corr = have_block_ || have_near_;
  const uint32_t npatch = ni_ ? n_all / uint32_t(ni_) : 0;
  const bool reduce = sharded && transport_ != nullptr;

  double* const sec_hist = rep->seconds_history;
  double* const mv_hist = rep->matvec_seconds_history;
  const int hist_cap = rep->history_cap;
  *rep = hfmm_gmres_report{};
  rep->seconds_history = sec_hist;
  rep->matvec_seconds_history = mv_hist;
  rep->history_cap = hist_cap;

  DeviceBuffer<float2> V(size_t(m + 1) * ld), w(ld), u(sharded ? 1 : n_all), r32(ld);
  DeviceBuffer<float2> full(sharded && (precond || corr) ? n_all : 1), vc(full.size()), pc(full.size()),
      yc(sharded && corr ? n_all : 1);
  DeviceBuffer<double2> b64(ld), x64(ld);
  DeviceBuffer<double> scal(size_t(2) * (2 * (m + 1) + 2)), ydev(size_t(2) * m), red(reduce_scratch_doubles());
  red.zero(stream_);
  std::vector<double> hscal(scal.size());

  double bnorm2 = 0;
  for (size_t i = 0; i < size_t(n) * 2; ++i) bnorm2 += rhs[i] * rhs[i];
  if (reduce) {  // ||b||^2 over the ranks
    scal.zero(stream_);
    HFMM_CUDA_CHECK(cudaMemcpyAsync(scal.get(), &bnorm2, sizeof(double), cudaMemcpyHostToDevice, stream_));
    comm_allreduce(scal.get(), 1);
    scal.download(&bnorm2, 1, stream_);
    HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
  }
  const double bnorm = std::sqrt(bnorm2);
  rep->rhs_norm = bnorm;
  std::fill(x_out, x_out + size_t(n) * 2, 0.0);
  if (bnorm == 0.0) {
    rep->converged = 1;
    rep->final_residual = 0;
    return;
  }
  const double target = cfg.rtol * bnorm;

  if (n) HFMM_CUDA_CHECK(cudaMemcpyAsync(b64.get(), rhs, size_t(n) * sizeof(double2), cudaMemcpyHostToDevice, stream_));
  x64.zero(stream_);
  launch_narrow(n, b64.get(), r32.get(), stream_);  // x0 = 0: the first residual is b

  std::vector<cd> H(size_t(m + 1) * m), cs(m), sn(m), g(m + 1);
  auto h = [&](int i, int j) -> cd& { return H[size_t(j) * (m + 1) + i]; };
  double matvec_s = 0;
  auto allreduce = [&](double* dev, int count) {
    if (reduce) comm_allreduce(dev, count);
  };
  // Z = A M^-1  (solver.cpp:383-387)
  auto apply = [&](const float2* in, float2* out) {
    const auto t0 = clk::now();
    if (!sharded) {
      const float2* src = in;
      if (precond) {
        launch_precondition(npatch, ni_, block_lu_.get(), block_piv_.get(), in, u.get(), stream_);
        src = u.get();
      }
      apply_operator_device(src, out);
    } else if (!(precond || corr)) {
      // plain FMM operator: the owned slice becomes the owned charges, the halo arrives through the exchange
      if (n)
        owned_charges_kernel<<<(n + 255) / 256, 256, 0, stream_>>>(in, body_index_.get(),
                                                                   have_weight_ ? far_weight_.get() : nullptr,
                                                                   body_q_.get(), first, n);
      HFMM_CUDA_CHECK(cudaGetLastError());
      dist_far_and_near();
      launch_combine_owned(near_.get() + first, far_.get() + first, nullptr, body_index_.get() + first, out, n, stream_);
    } else {
      // BIE tail: gather the operand, precondition and correct redundantly in caller order (streaming
      // kernels, < 1 % of a matvec), run the FMM over the exchanges
      if (n)
        HFMM_CUDA_CHECK(cudaMemcpyAsync(full.get() + first, in, size_t(n) * sizeof(float2), cudaMemcpyDeviceToDevice,
                                        stream_));
      comm_allgather_morton(full.get());
      launch_scatter_potentials(full.get(), nullptr, body_index_.get(), nullptr, vc.get(), n_all, stream_);
      const float2* xc = vc.get();
      if (precond) {
        launch_precondition(npatch, ni_, block_lu_.get(), block_piv_.get(), vc.get(), pc.get(), stream_);
        xc = pc.get();
      }
      launch_gather_charges(nullptr, xc, body_index_.get(), have_weight_ ? far_weight_.get() : nullptr, body_q_.get(),
                            n_all, stream_);
      dist_far_and_near();
      if (corr) {
        yc.zero(stream_);
        launch_corrections(n_all, ni_, have_block_ ? patch_block_.get() : nullptr, near_offset_.get(),
                           near_source_.get(), have_near_ ? near_delta_.get() : nullptr, xc, yc.get(), stream_);
      }
      launch_combine_owned(near_.get() + first, far_.get() + first, corr ? yc.get() : nullptr,
                           body_index_.get() + first, out, n, stream_);
    }
    HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
    matvec_s += std::chrono::duration<double>(clk::now() - t0).count();
  };

  int iterations = 0, nres = 0;
  bool done = false, breakdown = false;
  double last_est = -1, beta = bnorm, matvec_prev = 0;
  while (!done) {
    if (beta <= target || iterations >= cfg.max_iterations) break;
    launch_scale(n, r32.get(), float(1.0 / beta), V.get(), stream_);
    std::fill(g.begin(), g.end(), cd(0));
    g[0] = beta;
    int cols = 0;
    for (int j = 0; j < m; ++j) {
      if (iterations >= cfg.max_iterations) break;
      apply(V.get() + size_t(j) * ld, w.get());
      // one fused sweep: ||w||^2, two Gram-Schmidt passes, ||w||^2 again; scalars stay on the device (and are
      // all-reduced there in the sharded layout: the subtraction of a projection reads the reduced coefficient)
      scal.zero(stream_);
      double* s0 = scal.get();                  // [0]: w_scale^2
      double* h1 = s0 + 2;                      // pass 1, j+1 entries
      double* h2 = h1 + 2 * (m + 1);            // pass 2
      double* hn = h2 + 2 * (m + 1);            // ||w||^2 after both passes
      launch_norm2(n, w.get(), s0, red.get(), stream_);
      allreduce(s0, 2);
      for (int pass = 0; pass < 2; ++pass) {
        double* hp = pass ? h2 : h1;
        for (int i = 0; i <= j; ++i) {
          const float2* vprev = nullptr;
          const double* cprev = nullptr;
          if (i > 0) {
            vprev = V.get() + size_t(i - 1) * ld;
            cprev = hp + 2 * (i - 1);
          } else if (pass == 1) {
            vprev = V.get() + size_t(j) * ld;
            cprev = h1 + 2 * j;
          }
          launch_mgs_step(n, w.get(), vprev, cprev, V.get() + size_t(i) * ld, hp + 2 * i, red.get(), stream_);
          allreduce(hp + 2 * i, 2);
        }
      }
      launch_mgs_step(n, w.get(), V.get() + size_t(j) * ld, h2 + 2 * j, nullptr, nullptr, red.get(), stream_);
      launch_norm2(n, w.get(), hn, red.get(), stream_);
      allreduce(hn, 2);
      scal.download(hscal.data(), hscal.size(), stream_);
      HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
      const double w_scale = std::sqrt(hscal[0]);
      const double* c1 = hscal.data() + 2;
      const double* c2 = c1 + 2 * (m + 1);
      double hnext = std::sqrt(c2[2 * (m + 1)]);
      for (int i = 0; i <= j; ++i) h(i, j) = cd(c1[2 * i], c1[2 * i + 1]) + cd(c2[2 * i], c2[2 * i + 1]);
      const bool broke = hnext <= 1e-14 * std::max(w_scale, 1e-300);
      if (broke) hnext = 0;

      for (int i = 0; i < j; ++i) {
        const cd a = h(i, j), b = h(i + 1, j);
        h(i, j) = cs[i] * a + sn[i] * b;
        h(i + 1, j) = -std::conj(sn[i]) * a + cs[i] * b;
      }
      const cd a = h(j, j);
      const double b = hnext, r = std::hypot(std::abs(a), b);
      if (r == 0.0) {
        cs[j] = 1;
        sn[j] = 0;
      } else if (std::abs(a) == 0.0) {
        cs[j] = 0;
        sn[j] = 1;
      } else {
        cs[j] = std::abs(a) / r;
        sn[j] = (a / std::abs(a)) * (b / r);
      }
      h(j, j) = cs[j] * a + sn[j] * b;
      g[j + 1] = -std::conj(sn[j]) * g[j];
      g[j] = cs[j] * g[j];

      ++iterations;
      cols = j + 1;
      last_est = std::abs(g[j + 1]);
      if (residuals && nres < residual_cap) residuals[nres] = last_est / bnorm;
      if (nres < hist_cap) {  // SolveReport::seconds / matvec_seconds (gmres.cpp:65-71,144)
        if (sec_hist) sec_hist[nres] = std::chrono::duration<double>(clk::now() - t_start).count();
        if (mv_hist) mv_hist[nres] = matvec_s - matvec_prev;
      }
      matvec_prev = matvec_s;
      ++nres;
      if (broke) {
        breakdown = true;
        done = true;
        break;
      }
      if (last_est <= target) {
        done = true;
        break;
      }
      launch_scale(n, w.get(), float(1.0 / hnext), V.get() + size_t(j + 1) * ld, stream_);
    }
    // fold the Arnoldi columns into x, skipping trailing dead diagonals (gmres.cpp:75-85)
    while (cols > 0 && std::abs(h(cols - 1, cols - 1)) == 0.0) --cols;
    std::vector<cd> y(cols);
    for (int i = cols - 1; i >= 0; --i) {
      cd s = g[i];
      for (int l = i + 1; l < cols; ++l) s -= h(i, l) * y[l];
      y[i] = std::abs(h(i, i)) == 0.0 ? cd(0) : s / h(i, i);
    }
    if (cols > 0) {
      HFMM_CUDA_CHECK(cudaMemcpyAsync(ydev.get(), y.data(), sizeof(cd) * cols, cudaMemcpyHostToDevice, stream_));
      launch_update_solution(n, cols, V.get(), ld, ydev.get(), x64.get(), stream_);
      HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
    }
    if (!done) {  // restart boundary: true residual, not an Arnoldi step
      launch_narrow(n, x64.get(), r32.get(), stream_);
      apply(r32.get(), w.get());
      scal.zero(stream_);
      launch_residual(n, b64.get(), w.get(), r32.get(), scal.get(), red.get(), stream_);
      allreduce(scal.get(), 2);
      scal.download(hscal.data(), 2, stream_);
      HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
      beta = std::sqrt(hscal[0]);
    }
  }
  // true residual on exit (gmres.cpp:165-170)
  launch_narrow(n, x64.get(), V.get(), stream_);
  apply(V.get(), w.get());
  scal.zero(stream_);
  launch_residual(n, b64.get(), w.get(), r32.get(), scal.get(), red.get(), stream_);
  allreduce(scal.get(), 2);
  scal.download(hscal.data(), 2, stream_);
  // kept for callers that drive the restart cycles themselves (repartitioning between cycles, partition.cpp:143-227)
  if (solve_residual_.size() < ld) solve_residual_.resize(ld);
  if (n) HFMM_CUDA_CHECK(cudaMemcpyAsync(solve_residual_.get(), r32.get(), size_t(n) * sizeof(float2), cudaMemcpyDeviceToDevice, stream_));
  solve_residual_n_ = n;
  // the returned iterate maps back through M^-1 (solver.cpp:388)
  if (precond) {
    if (!sharded) {
      launch_precondition(npatch, ni_, block_lu_.get(), block_piv_.get(), V.get(), u.get(), stream_);
      launch_widen(n, u.get(), x64.get(), stream_);
    } else {  // gather the iterate, solve redundantly, keep the owned slots
      if (n)
        HFMM_CUDA_CHECK(cudaMemcpyAsync(full.get() + first, V.get(), size_t(n) * sizeof(float2), cudaMemcpyDeviceToDevice,
                                        stream_));
      comm_allgather_morton(full.get());
      launch_scatter_potentials(full.get(), nullptr, body_index_.get(), nullptr, vc.get(), n_all, stream_);
      launch_precondition(npatch, ni_, block_lu_.get(), block_piv_.get(), vc.get(), pc.get(), stream_);
      launch_gather_charges(nullptr, pc.get(), body_index_.get(), nullptr, full.get(), n_all, stream_);
      launch_widen(n, full.get() + first, x64.get(), stream_);
    }
  }
  if (n) HFMM_CUDA_CHECK(cudaMemcpyAsync(x_out, x64.get(), size_t(n) * sizeof(double2), cudaMemcpyDeviceToHost, stream_));
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
  rep->iterations = iterations;
  rep->breakdown = breakdown ? 1 : 0;
  rep->final_residual = std::sqrt(hscal[0]) / bnorm;
  rep->converged = (rep->final_residual <= cfg.rtol || (nres > 0 && last_est / bnorm <= cfg.rtol)) ? 1 : 0;
  rep->seconds = std::chrono::duration<double>(clk::now() - t_start).count();
  rep->matvec_seconds = matvec_s;
}

// fmm_evaluate(target_tree, source_tree) with targets != sources (traversal.hpp:59-67, traversal.cpp:281-287):
// the potentials of the handle's points, carrying the strengths q, at `nt` other points.  One tree over the
// union (the targets carry zero charge) runs the ordinary pipeline on a second engine; the interaction lists are
// those of the union set, not of the reference's two-tree descent, the potentials agree to the FMM's tolerance.
// The union tree is kept until the targets change (FNV-1a of their coordinates).
void Engine::evaluate_targets(const double* targets, size_t nt, const double* q, double* out) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  if (nranks_ > 1) throw Error(HFMM_ERR_CONFIG, "evaluate_targets needs a single-domain handle");
  if (!nt) return;
  if (!targets || !q || !out) throw Error(HFMM_ERR_CONFIG, "null argument");
  const size_t n = tree_.n_bodies;
  uint64_t hash = 1469598103934665603ull;
  const unsigned char* bytes = reinterpret_cast<const unsigned char*>(targets);
  for (size_t i = 0; i < nt * 3 * sizeof(double); ++i) hash = (hash ^ bytes[i]) * 1099511628211ull;
  if (!target_engine_ || target_hash_ != hash || target_count_ != nt) {
    std::vector<double> all(3 * (n + nt));
    xyz64_.download(all.data(), 3 * n, stream_);
    HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
    std::copy(targets, targets + 3 * nt, all.begin() + 3 * n);
    hfmm_cuda_config c = cfg_;
    target_engine_.reset();
    target_engine_ = std::make_unique<Engine>(c);
    AllocStreamScope scope(target_engine_->stream(), cfg_.device);
    target_engine_->set_points(all.data(), n + nt);
    target_hash_ = hash;
    target_count_ = nt;
  }
  std::vector<double> qq(2 * (n + nt), 0.0), res(2 * (n + nt));
  std::copy(q, q + 2 * n, qq.begin());
  {
    AllocStreamScope scope(target_engine_->stream(), cfg_.device);
    target_engine_->matvec_host(qq.data(), res.data());
  }
  std::copy(res.begin() + 2 * n, res.end(), out);
}

void Engine::get_solve_residual(double* out, size_t capacity) {
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  if (capacity < solve_residual_n_) throw Error(HFMM_ERR_CONFIG, "residual buffer too small");
  const uint32_t n = solve_residual_n_;
  if (!n) return;
  if (io64_.size() < n) io64_.resize(n);
  launch_widen(n, solve_residual_.get(), io64_.get(), stream_);
  HFMM_CUDA_CHECK(cudaMemcpyAsync(out, io64_.get(), size_t(n) * sizeof(double2), cudaMemcpyDeviceToHost, stream_));
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::set_patch_diameters(const double* diameter, size_t n_patches) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  if (!diameter || n_patches == 0 || tree_.n_bodies % n_patches != 0)
    throw Error(HFMM_ERR_CONFIG, "the patch count must divide the number of unknowns");
  std::vector<double> t2(n_patches);
  for (size_t p = 0; p < n_patches; ++p) {
    const double t = 0.1 * diameter[p];  // solver.cpp:399-403
    t2[p] = t * t;
  }
  touch2_.upload(t2, stream_);
  touch_ni_ = uint32_t(tree_.n_bodies / n_patches);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::assemble_rhs(const double* direction, const double* amplitude, double* out) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const double n2 = direction[0] * direction[0] + direction[1] * direction[1] + direction[2] * direction[2];
  if (!(std::abs(n2 - 1.0) <= 1e-9)) throw Error(HFMM_ERR_CONFIG, "incident direction must be unit length");
  const uint32_t n = tree_.n_bodies;
  if (io64_.size() != n) io64_.resize(n);
  launch_assemble_rhs(n, xyz64_.get(), direction, cfg_.wave_r, cfg_.wave_i, amplitude, io64_.get(), stream_);
  HFMM_CUDA_CHECK(cudaMemcpyAsync(out, io64_.get(), size_t(n) * sizeof(double2), cudaMemcpyDeviceToHost, stream_));
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::evaluate_field(const double* coeff, const double* obs, size_t nobs, double* out) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const uint32_t n = tree_.n_bodies;
  const double k = cfg_.wave_r;
  std::vector<float2> c(n);
  for (size_t i = 0; i < n; ++i)
    c[i] = make_float2(float(coeff[2 * i]), float(coeff[2 * i + 1]));
  DeviceBuffer<float2> cdev;
  cdev.upload(c, stream_);
  if (have_weight_) {  // strength = coefficient * far_weight (solver.cpp:413-414)
    launch_gather_charges(nullptr, cdev.get(), identity_index(), far_weight_.get(), body_q_.get(), n, stream_);
  } else {
    HFMM_CUDA_CHECK(cudaMemcpyAsync(body_q_.get(), cdev.get(), size_t(n) * sizeof(float2),
                                    cudaMemcpyDeviceToDevice, stream_));
  }
  DeviceBuffer<double> odev;
  odev.upload(obs, 3 * nobs, stream_);
  DeviceBuffer<double2> res(nobs);
  DeviceBuffer<int> flag(1);
  flag.zero(stream_);
  const bool test = touch2_.size() != 0;
  launch_field(n, xyz64_.get(), body_q_.get(), odev.get(), uint32_t(nobs), k, float(k / (4.0 * kPi)),
               float(cfg_.wave_i / cfg_.wave_r), test ? touch2_.get() : nullptr, touch_ni_, res.get(), flag.get(),
               stream_);
  int touched = 0;
  flag.download(&touched, 1, stream_);
  res.download(reinterpret_cast<double2*>(out), nobs, stream_);
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
  if (touched)
    throw Error(HFMM_ERR_SINGULAR, "evaluate_scattered_field: observation point touches the surface");
}

}  // namespace hfmm_b200
