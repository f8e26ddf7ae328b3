// engine.hpp — the handle behind the C ABI: owns the device-resident octree, interaction lists,
// translation tables, expansions and streams, and orchestrates one FMM matvec
// (reference fmm::execute_plan, src/traversal.cpp:208-279).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "device_utils.cuh"
#include "host_tree.hpp"
#include "kernels.cuh"
#include "tree_build.cuh"

namespace hfmm_b200 {

struct TableRegistry;

struct TranslateStage {
  // one batched-translation launch: M2L (all levels) or one level of M2M / L2L
  DeviceBuffer<TranslateItem> items;
  DeviceBuffer<TranslateClass> classes;
  DeviceBuffer<uint32_t> pair_src, pair_dst, pair_cls;  // pair_cls: shift class of every pair
  uint32_t n_items = 0;
  uint64_t n_pairs = 0;
  bool mixed = false;  // batches mix the classes of a table group (per-pair azimuth phases in the kernel)
  // HFMM_FLAG_DETERMINISTIC: the stage runs range by range (whole batches, as many pairs as the staging
  // buffer has rows) into one staging row per pair; an ordered reduction then adds the rows of every
  // destination in pair order (the reference's per-target ordered accumulation, traversal.hpp:20-22)
  struct OrderedRange {
    uint32_t item_begin = 0, n_items = 0, n_pairs = 0, n_segs = 0;
    uint64_t pair_begin = 0;
    DeviceBuffer<uint32_t> perm, seg_dst, seg_begin;
  };
  std::vector<OrderedRange> ordered;
  DeviceBuffer<uint32_t> row_of_pair;  // staging row of every pair (index inside its range)
};

class Engine {
 public:
  explicit Engine(const hfmm_cuda_config& cfg);
  ~Engine();
  cudaStream_t stream() const { return stream_; }   // the stream every allocation is ordered on
  int device() const { return cfg_.device; }
  static bool any_engine_alive();

  void set_partition(int rank, int nranks);
  void set_partition_alpha(double alpha);  // < 0: default work model
  void measure_weights(double* local, double* remote) const;
  void get_exchange_masks(uint64_t* far_mask, uint64_t* near_mask, int32_t* cell_rank) const;
  void get_partition(hfmm_cuda_partition* out);
  void dist_upward(const void* q_morton_dev);
  void dist_downward(void* out_morton_dev);
  void set_points(const double* xyz, size_t n);
  void matvec_host(const double* q, double* out);
  void matvec_device(const void* q_dev, void* out_dev);
  void sync();
  void timer_record(int slot);
  double timer_elapsed_ms(int a, int b);
  void flush_l2();
  double measure_fp32_peak_tflops();
  void measure_fp32_probes(double out[2]);  // [0] FFMA, [1] FFMA2
  void get_stats(hfmm_cuda_stats* out);
  void get_cells(uint32_t* out, size_t capacity) const;
  void get_body_order(uint32_t* out) const;
  void get_pairs(int which, uint32_t* out, uint64_t* count) const;
  void get_expansions(int which, double* out);
  void set_corrections(int ni, const double* far_weight, const double* patch_block,
                       const uint32_t* near_offset, const uint32_t* near_source,
                       const double* near_delta, const double* block_lu, const int32_t* block_piv);
  void gmres(const double* rhs, double* x, const hfmm_gmres_config& cfg, hfmm_gmres_report* rep,
             double* residuals, int residual_cap);
  // clears and returns the name of a non-sticky CUDA error left behind on this host thread (or null)
  static const char* take_stale_cuda_error();
  void evaluate_field(const double* coeff, const double* obs, size_t nobs, double* out);
  void assemble_rhs(const double* direction, const double* amplitude, double* out);
  void set_patch_diameters(const double* diameter, size_t n_patches);
  // correction builders on the device (corrections_build.cu; reference solver.cpp:80-230)
  void build_corrections(const hfmm_correction_rules& rules, uint64_t* near_nnz);
  void get_corrections(double* patch_block, double* block_lu, int* block_piv, uint32_t* near_offset,
                       uint32_t* near_source, double* near_delta);
  // multi-GPU data plane (comm.cu): communicator, locally-essential-tree exchange, sharded solver
  struct Transport;
  struct ExchangePlan;
  void comm_init_nccl(const void* unique_id_128);
  void comm_init_host(const hfmm_host_transport& cb);
  const char* comm_name() const;
  void get_exchange_volume(uint64_t* charge_bytes, uint64_t* multipole_bytes);
  // potentials at `nt` points that are not sources (fmm_evaluate with distinct target and source trees,
  // traversal.hpp:59-67): one tree over sources + targets, targets carry zero charge
  void evaluate_targets(const double* targets, size_t nt, const double* q, double* out);
  // b - Z u of the last gmres / dist_solve (the vector behind final_residual), owned slice, FP32 widened
  void get_solve_residual(double* out, size_t capacity);
  void dist_matvec(const void* q_owned_dev, void* out_owned_dev);
  void dist_solve(const double* rhs_owned, double* x_owned, const hfmm_gmres_config& cfg,
                  hfmm_gmres_report* rep, double* residuals, int residual_cap);

  std::string last_error;
  const hfmm_cuda_config& config() const { return cfg_; }
  uint32_t n_bodies() const { return tree_.n_bodies; }

 private:
  void require_points() const;
  void release_device_state();
  void destroy_streams_and_events();
  void run_far_and_near();  // body_q_ -> near_, far_
  void phase_upward();      // near field (own stream) + P2M + M2M
  void phase_downward();    // M2L + L2L + L2P, joins the near field
  void run_stage(const TranslateStage& st, const float2* src, float2* dst);
  void compute_partition();
  void gmres_impl(bool sharded, const double* rhs, double* x_out, const hfmm_gmres_config& cfg,
                  hfmm_gmres_report* rep, double* residuals, int residual_cap);
  void build_exchange_plan();
  void dist_far_and_near();   // body_q_ (owned slots) -> near_, far_ (owned slots), over the two exchanges
  void comm_allreduce(double* dev, int count);
  void comm_allgather_morton(float2* full);
  void release_comm();
  uint64_t count_starved_cells() const;
  void collect_timings();
  void apply_operator_device(const float2* x, float2* y);  // caller order, weights + corrections
  const uint32_t* identity_index();
  void set_points_host(const double* xyz, size_t n);
  void set_points_device(const double* xyz, size_t n);
  void build_m2l_stage_host(TableRegistry& reg, const PairLists& pairs);
  void build_m2l_stage_device(TableRegistry& reg, const FarClasses& fc);
  void finish_far_field(TableRegistry& reg);
  void upload_cell_geometry(std::vector<int4>& geom);
  void build_tiles(const std::vector<uint64_t>& work);
  void select_near_kernel(uint64_t max_r2_lattice);
  void plan_ordered_reduce(TranslateStage& st, const std::vector<TranslateItem>& items);
  void upload_stage(TranslateStage& st, const std::vector<uint32_t>& src,
                    const std::vector<uint32_t>& dst, const std::vector<uint32_t>& cls_of_pair,
                    const std::vector<TranslateClass>& classes, bool ordered = false);

  hfmm_cuda_config cfg_;
  double leaf_cap_ = 0;
  int threads_ = 1;
  // Morton partition (multi-GPU): this rank owns bodies [own_first_, own_first_ + own_count_)
  int rank_ = 0, nranks_ = 1, lcut_ = 0;
  uint32_t own_first_ = 0, own_count_ = 0;
  double partition_alpha_ = -1.0;
  P2PArgs p2p_args_{};
  bool p2p_late_ = false;
  cudaEvent_t near_gate_ = nullptr;  // sharded matvec: the near field waits for the halo charges
  std::shared_ptr<Transport> transport_;
  std::shared_ptr<ExchangePlan> exchange_;
  uint64_t exchange_bytes_[2] = {0, 0};
  bool host_lists_ = false;  // the pair lists of the current point set live on the host (host builder)
  std::vector<uint8_t> owned_;  // per cell
  std::vector<int32_t> cell_rank_;  // per cell: owning rank of the Morton partition
  uint64_t owned_m2l_pairs_ = 0, owned_body_pairs_ = 0, launches_ = 0;
  cudaStream_t stream_ = nullptr, stream_near_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  std::vector<cudaEvent_t> ev_;       // per-kernel timers of the last matvec
  std::vector<cudaEvent_t> user_ev_;  // caller-driven timers (hfmm_cuda_timer_*)
  bool timings_pending_ = false;
  DeviceBuffer<unsigned char> flush_;

  // host mirrors kept for introspection
  TreeArrays tree_;
  PairLists pairs_;        // host builder only
  DevicePairs dev_pairs_;  // device builder only
  bool have_points_ = false;
  hfmm_cuda_stats stats_{};

  // device tree
  DeviceBuffer<float4> body_pos_, body_hi_, body_lo_;
  DeviceBuffer<uint32_t> body_index_;
  DeviceBuffer<int4> cell_geom_;
  DeviceBuffer<uint2> cell_body_;
  DeviceBuffer<float> level_scale_;
  std::vector<float> level_scale_host_;
  // near field
  DeviceBuffer<P2PTile> p2p_tiles_;
  DeviceBuffer<uint32_t> p2p_offset_, p2p_split_, p2p_src_;
  uint32_t n_tiles_ = 0;
  int p2p_mode_ = 0;           // P2P_MODE_*: the fastest variant for the near field on its own
  int p2p_mode_late_ = 0;      // the variant of the launch that runs beside M2L (near_mode_in_step)
  int near_mode_in_step() const;
  double near_r2_max_ = 0;     // bound on R'^2 over the owned near lists
  float p2p_sinc_[8] = {}, p2p_cos_[8] = {};
  float kunit_ = 0;
  double kunit_d_ = 0, grid_ = 1;
  // far field
  int stride_ = 0;
  int lmin_src_ = 0, lmin_dst_ = 0;
  bool have_far_ = false;
  DeviceBuffer<float2> multipole_, local_;
  DeviceBuffer<float2> ordered_staging_;  // HFMM_FLAG_DETERMINISTIC: one row per pair of the largest range
  DeviceBuffer<uint32_t> p2m_leaves_, l2p_leaves_;
  uint32_t n_p2m_leaves_ = 0, n_l2p_leaves_ = 0;
  bool leaf_small_args_ = false;  // every leaf body has k rho <= 1: the unrolled P2M / L2P kernels apply
  DeviceBuffer<float> rot_tables_, coax_tables_;
  TranslateStage m2l_;
  std::vector<TranslateStage> m2m_;  // deepest level first
  std::vector<TranslateStage> l2l_;  // shallowest level first
  // BIE operator tail (set_corrections)
  struct CorrectionStore;  // FP64 results of build_corrections
  std::shared_ptr<CorrectionStore> corrections64_;  // shared_ptr: deleter bound where the type is complete
  void release_correction_store();
  int ni_ = 0;
  bool have_weight_ = false, have_block_ = false, have_near_ = false, have_lu_ = false;
  DeviceBuffer<float> far_weight_;
  DeviceBuffer<double2> patch_block_, near_delta_, block_lu_;  // FP64: see corrections_kernel
  DeviceBuffer<uint32_t> near_offset_, near_source_, identity_;
  DeviceBuffer<int> block_piv_;
  DeviceBuffer<float4> body_abs_;  // k * x, caller order
  DeviceBuffer<double> xyz64_;     // the points as given, FP64, caller order (rhs, exterior field)
  DeviceBuffer<double> touch2_;    // (0.1 patch diameter)^2 per patch: singular test of evaluate_field
  uint32_t touch_ni_ = 1;
  DeviceBuffer<float2> x32_, y32_;
  // vectors
  DeviceBuffer<float2> body_q_, near_, far_;
  DeviceBuffer<double2> io64_;
  std::unique_ptr<Engine> target_engine_;  // sources + targets of the last evaluate_targets (rebuilt when they change)
  uint64_t target_hash_ = 0;
  size_t target_count_ = 0;
  DeviceBuffer<float2> solve_residual_;  // residual vector of the last solve (restart cycles driven by the caller)
  uint32_t solve_residual_n_ = 0;
};

// FP64 composition of the factored operator into a dense (P+1)^2 x (P+1)^2 matrix in the
// reference's UNSCALED convention — used by the CPU-side table tests against
// fmm::translation_matrix (expansion.cpp:95-124).  kind: 0 M2L (singular), 1 regular.
// ncclGetUniqueId through the run-time loaded NCCL (comm.cu)
void nccl_unique_id(void* out128);

void compose_dense_from_tables(int order, double k, const double t[3], int kind, double s_src,
                               double s_dst, double* out_complex, double k_imag = 0.0);

}  // namespace hfmm_b200
