// capi.cpp — the extern "C" surface declared in include/hfmm_cuda.h.  Converts exceptions to
// status codes; nothing else lives here.
#include <cstring>
#include <new>
#include <string>

#include "device_utils.cuh"
#include "engine.hpp"
#include "hfmm_cuda.h"

using hfmm_b200::Engine;
using hfmm_b200::Error;

struct hfmm_cuda {
  Engine* engine = nullptr;
};

namespace {
thread_local std::string g_create_error;
// leftover CUDA error name of other CUDA users on this host thread (diagnosis only); thread-local like
// the CUDA error state it mirrors: handles may be driven from different host threads
thread_local std::string g_stale_error;

template <typename Fn>
int guarded(hfmm_cuda* h, Fn&& fn) {
  std::string* sink = (h && h->engine) ? &h->engine->last_error : &g_create_error;
  try {
    // the CUDA "last error" is per host thread and shared with every other CUDA user of the
    // process (torch, the caller's own code): drop what they left so that the launch checks
    // below report this call's errors only; the leftover stays readable for diagnosis
    if (const char* stale = Engine::take_stale_cuda_error()) g_stale_error = stale;
    // buffers created or dropped inside the call are ordered on the handle's stream (device_utils.cuh)
    hfmm_b200::AllocStreamScope scope((h && h->engine) ? h->engine->stream() : nullptr,
                                      (h && h->engine) ? h->engine->device() : -1);
    fn();
    return HFMM_OK;
  } catch (const Error& e) {
    *sink = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    *sink = "host allocation failed";
    return HFMM_ERR_INTERNAL;
  } catch (const std::exception& e) {
    *sink = e.what();
    return HFMM_ERR_INTERNAL;
  }
}

int need(hfmm_cuda* h) {
  if (h && h->engine) return HFMM_OK;
  g_create_error = "null handle";
  return HFMM_ERR_CONFIG;
}
}  // namespace

extern "C" {

int hfmm_cuda_create(hfmm_cuda_t** out, const hfmm_cuda_config* cfg) {
  if (!out || !cfg) {
    g_create_error = "null argument";
    return HFMM_ERR_CONFIG;
  }
  *out = nullptr;
  return guarded(nullptr, [&] {
    auto* h = new hfmm_cuda;
    try {
      h->engine = new Engine(*cfg);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void hfmm_cuda_destroy(hfmm_cuda_t* h) {
  if (!h) return;
  const int device = h->engine ? h->engine->device() : -1;
  delete h->engine;
  delete h;
  // the last handle returns the pooled device memory to the driver
  if (device >= 0 && !Engine::any_engine_alive()) hfmm_b200::trim_memory_pool(device);
}

const char* hfmm_cuda_last_error(const hfmm_cuda_t* h) {
  return (h && h->engine) ? h->engine->last_error.c_str() : g_create_error.c_str();
}

int hfmm_cuda_set_points(hfmm_cuda_t* h, const double* xyz, size_t n) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!xyz && n) throw Error(HFMM_ERR_CONFIG, "null point array");
    h->engine->set_points(xyz, n);
  });
}

int hfmm_cuda_matvec(hfmm_cuda_t* h, const double* q, double* out) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!q || !out) throw Error(HFMM_ERR_CONFIG, "null vector");
    h->engine->matvec_host(q, out);
  });
}

int hfmm_cuda_matvec_device(hfmm_cuda_t* h, const void* q_dev, void* out_dev) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!q_dev || !out_dev) throw Error(HFMM_ERR_CONFIG, "null vector");
    h->engine->matvec_device(q_dev, out_dev);
  });
}

int hfmm_cuda_sync(hfmm_cuda_t* h) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->sync(); });
}

int hfmm_cuda_timer_record(hfmm_cuda_t* h, int slot) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->timer_record(slot); });
}

int hfmm_cuda_timer_elapsed_ms(hfmm_cuda_t* h, int slot_a, int slot_b, double* ms) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { *ms = h->engine->timer_elapsed_ms(slot_a, slot_b); });
}

int hfmm_cuda_flush_l2(hfmm_cuda_t* h) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->flush_l2(); });
}

int hfmm_cuda_fp32_peak_tflops(hfmm_cuda_t* h, double* tflops) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { *tflops = h->engine->measure_fp32_peak_tflops(); });
}

int hfmm_cuda_get_stats(hfmm_cuda_t* h, hfmm_cuda_stats* out) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->get_stats(out); });
}

int hfmm_cuda_get_cells(hfmm_cuda_t* h, uint32_t* out, size_t capacity_cells) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->get_cells(out, capacity_cells); });
}

int hfmm_cuda_get_body_order(hfmm_cuda_t* h, uint32_t* out) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->get_body_order(out); });
}

int hfmm_cuda_get_pairs(hfmm_cuda_t* h, int which, uint32_t* out, uint64_t* count) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->get_pairs(which, out, count); });
}

int hfmm_cuda_get_expansions(hfmm_cuda_t* h, int which, double* out) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->get_expansions(which, out); });
}

int hfmm_cuda_set_corrections(hfmm_cuda_t* h, int ni, const double* far_weight,
                              const double* patch_block, const uint32_t* near_offset,
                              const uint32_t* near_source, const double* near_delta,
                              const double* block_lu, const int32_t* block_piv) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    h->engine->set_corrections(ni, far_weight, patch_block, near_offset, near_source, near_delta,
                               block_lu, block_piv);
  });
}

int hfmm_cuda_gmres(hfmm_cuda_t* h, const double* rhs, double* x, const hfmm_gmres_config* cfg,
                    hfmm_gmres_report* report, double* residuals, int residual_cap) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!rhs || !x || !cfg || !report) throw Error(HFMM_ERR_CONFIG, "null argument");
    h->engine->gmres(rhs, x, *cfg, report, residuals, residual_cap);
  });
}

int hfmm_cuda_evaluate_field(hfmm_cuda_t* h, const double* coeff, const double* obs, size_t nobs,
                             double* out) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!coeff || (!obs && nobs) || (!out && nobs)) throw Error(HFMM_ERR_CONFIG, "null argument");
    h->engine->evaluate_field(coeff, obs, nobs, out);
  });
}

int hfmm_cuda_assemble_rhs(hfmm_cuda_t* h, const double* direction, const double* amplitude, double* out) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!direction || !amplitude || !out) throw Error(HFMM_ERR_CONFIG, "null argument");
    h->engine->assemble_rhs(direction, amplitude, out);
  });
}

int hfmm_cuda_set_patch_diameters(hfmm_cuda_t* h, const double* diameter, size_t n_patches) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->set_patch_diameters(diameter, n_patches); });
}

int hfmm_cuda_set_partition(hfmm_cuda_t* h, int rank, int nranks) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->set_partition(rank, nranks); });
}

int hfmm_cuda_get_partition(hfmm_cuda_t* h, hfmm_cuda_partition* out) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!out) throw Error(HFMM_ERR_CONFIG, "null argument");
    h->engine->get_partition(out);
  });
}

int hfmm_cuda_dist_upward(hfmm_cuda_t* h, const void* q_morton_dev) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!q_morton_dev) throw Error(HFMM_ERR_CONFIG, "null vector");
    h->engine->dist_upward(q_morton_dev);
  });
}

int hfmm_cuda_dist_downward(hfmm_cuda_t* h, void* out_morton_dev) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!out_morton_dev) throw Error(HFMM_ERR_CONFIG, "null vector");
    h->engine->dist_downward(out_morton_dev);
  });
}

int hfmm_cuda_get_exchange_masks(hfmm_cuda_t* h, uint64_t* far_mask, uint64_t* near_mask, int32_t* cell_rank) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!far_mask || !near_mask || !cell_rank) throw Error(HFMM_ERR_CONFIG, "null mask array");
    h->engine->get_exchange_masks(far_mask, near_mask, cell_rank);
  });
}

int hfmm_cuda_set_partition_alpha(hfmm_cuda_t* h, double alpha) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->set_partition_alpha(alpha); });
}

int hfmm_cuda_measure_weights(hfmm_cuda_t* h, double* local, double* remote) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!local || !remote) throw Error(HFMM_ERR_CONFIG, "null weight array");
    h->engine->measure_weights(local, remote);
  });
}

int hfmm_partition_update_alpha(const double* alpha, const double* runtime, int n, double alpha_max, double* next) {
  return guarded(nullptr, [&] {
    if (!next) throw Error(HFMM_ERR_CONFIG, "null output");
    *next = hfmm_b200::partition_update_alpha(alpha, runtime, n, alpha_max);
  });
}

int hfmm_cuda_build_corrections(hfmm_cuda_t* h, const hfmm_correction_rules* rules, uint64_t* near_nnz) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!rules) throw Error(HFMM_ERR_CONFIG, "null rules");
    h->engine->build_corrections(*rules, near_nnz);
  });
}

int hfmm_cuda_get_corrections(hfmm_cuda_t* h, double* patch_block, double* block_lu, int32_t* block_piv,
                              uint32_t* near_offset, uint32_t* near_source, double* near_delta) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    h->engine->get_corrections(patch_block, block_lu, block_piv, near_offset, near_source, near_delta);
  });
}

int hfmm_cuda_nccl_unique_id(void* out128) {
  return guarded(nullptr, [&] {
    if (!out128) throw Error(HFMM_ERR_CONFIG, "null argument");
    hfmm_b200::nccl_unique_id(out128);
  });
}

int hfmm_cuda_comm_init_nccl(hfmm_cuda_t* h, const void* unique_id_128) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->comm_init_nccl(unique_id_128); });
}

int hfmm_cuda_comm_init_host(hfmm_cuda_t* h, const hfmm_host_transport* t) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!t) throw Error(HFMM_ERR_CONFIG, "null transport");
    h->engine->comm_init_host(*t);
  });
}

int hfmm_cuda_dist_matvec(hfmm_cuda_t* h, const void* q_owned_dev, void* out_owned_dev) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->dist_matvec(q_owned_dev, out_owned_dev); });
}

int hfmm_cuda_dist_solve(hfmm_cuda_t* h, const double* rhs_owned, double* x_owned, const hfmm_gmres_config* cfg,
                         hfmm_gmres_report* report, double* residuals, int residual_cap) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!cfg || !report) throw Error(HFMM_ERR_CONFIG, "null argument");
    h->engine->dist_solve(rhs_owned, x_owned, *cfg, report, residuals, residual_cap);
  });
}

int hfmm_cuda_evaluate_targets(hfmm_cuda_t* h, const double* targets, size_t n_targets, const double* q, double* out) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->evaluate_targets(targets, n_targets, q, out); });
}

int hfmm_cuda_get_solve_residual(hfmm_cuda_t* h, double* out, size_t capacity) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!out && capacity) throw Error(HFMM_ERR_CONFIG, "null argument");
    h->engine->get_solve_residual(out, capacity);
  });
}

int hfmm_cuda_get_exchange_volume(hfmm_cuda_t* h, uint64_t* charge_bytes, uint64_t* multipole_bytes) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] {
    if (!charge_bytes || !multipole_bytes) throw Error(HFMM_ERR_CONFIG, "null argument");
    h->engine->get_exchange_volume(charge_bytes, multipole_bytes);
  });
}

int hfmm_debug_fp32_probes(hfmm_cuda_t* h, double* out2) {
  if (int rc = need(h)) return rc;
  return guarded(h, [&] { h->engine->measure_fp32_probes(out2); });
}

const char* hfmm_debug_stale_cuda_error(void) { return g_stale_error.c_str(); }

const char* hfmm_cuda_version(void) { return "hfmm-b200 0.1 (sm_100a)"; }

// ---- host-only debug entry points for the CPU-side table tests (no device needed) ------------
// dense (P+1)^2 x (P+1)^2 matrix composed in FP64 from the FP32 device tables, unscaled.
// kind: 0 M2L, 1 regular (M2M/L2L).  Returns HFMM_OK.
int hfmm_debug_compose_translation(int order, double k, const double* t, int kind, double s_src,
                                   double s_dst, double* out) {
  return guarded(nullptr, [&] {
    if (order < 0 || order > hfmm_b200::kMaxOrder) throw Error(HFMM_ERR_CONFIG, "order out of range");
    hfmm_b200::compose_dense_from_tables(order, k, t, kind, s_src, s_dst, out);
  });
}

int hfmm_debug_compose_translation_ck(int order, double kr, double ki, const double* t, int kind, double s_src,
                                      double s_dst, double* out) {
  return guarded(nullptr, [&] {
    if (order < 0 || order > hfmm_b200::kMaxOrder) throw Error(HFMM_ERR_CONFIG, "order out of range");
    hfmm_b200::compose_dense_from_tables(order, kr, t, kind, s_src, s_dst, out, ki);
  });
}

// tree + lists of the host builder without touching a device: counts[0..4] = cells, leaves,
// m2l pairs, p2p leaf pairs, max level
int hfmm_debug_host_tree(const double* xyz, size_t n, int ncrit, double leaf_cap, double k,
                         double theta, double kd_max, uint64_t* counts, uint32_t* cells_out,
                         size_t cells_capacity, uint32_t* order_out, uint32_t* m2l_out,
                         uint32_t* p2p_out, size_t pair_capacity) {
  return guarded(nullptr, [&] {
    hfmm_b200::TreeArrays t;
    hfmm_b200::PairLists p;
    hfmm_b200::build_tree_host(t, xyz, n, ncrit, leaf_cap, 4);
    hfmm_b200::dual_tree_traversal_host(t, k, theta, kd_max, p, 4);
    counts[0] = t.n_cells();
    counts[1] = t.leaves.size();
    counts[2] = p.m2l_t.size();
    counts[3] = p.p2p_t.size();
    counts[4] = uint64_t(t.max_level);
    if (cells_out && cells_capacity >= t.n_cells())
      for (size_t c = 0; c < t.n_cells(); ++c) {
        uint32_t* o = cells_out + 8 * c;
        o[0] = t.level[c]; o[1] = t.ix[c]; o[2] = t.iy[c]; o[3] = t.iz[c];
        o[4] = t.body_first[c]; o[5] = t.body_count[c];
        o[6] = t.child_first[c]; o[7] = t.child_count[c];
      }
    if (order_out) std::memcpy(order_out, t.index.data(), sizeof(uint32_t) * n);
    if (m2l_out && pair_capacity >= p.m2l_t.size())
      for (size_t i = 0; i < p.m2l_t.size(); ++i) {
        m2l_out[2 * i] = p.m2l_t[i];
        m2l_out[2 * i + 1] = p.m2l_s[i];
      }
    if (p2p_out && pair_capacity >= p.p2p_t.size())
      for (size_t i = 0; i < p.p2p_t.size(); ++i) {
        p2p_out[2 * i] = p.p2p_t[i];
        p2p_out[2 * i + 1] = p.p2p_s[i];
      }
  });
}

// Morton partition of the host builder without a device: per-rank owned body ranges and
// (optionally) the owning rank of every cell
int hfmm_debug_partition(const double* xyz, size_t n, int ncrit, double leaf_cap, double k,
                         double theta, double kd_max, int nranks, uint32_t* first, uint32_t* count,
                         int32_t* cell_rank_out, size_t cells_capacity, int32_t* lcut_out) {
  return guarded(nullptr, [&] {
    hfmm_b200::TreeArrays t;
    hfmm_b200::PairLists p;
    hfmm_b200::build_tree_host(t, xyz, n, ncrit, leaf_cap, 4);
    hfmm_b200::dual_tree_traversal_host(t, k, theta, kd_max, p, 4);
    std::vector<int> cell_rank;
    std::vector<uint32_t> f, c;
    int lcut = 0;
    hfmm_b200::compute_morton_partition(t, p, nranks, -1.0, cell_rank, f, c, lcut);
    for (int r = 0; r < nranks; ++r) {
      first[r] = f[r];
      count[r] = c[r];
    }
    if (cell_rank_out && cells_capacity >= cell_rank.size())
      for (size_t i = 0; i < cell_rank.size(); ++i) cell_rank_out[i] = cell_rank[i];
    if (lcut_out) *lcut_out = lcut;
  });
}

}  // extern "C"
