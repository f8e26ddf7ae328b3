/* include/hfmm_cuda.h — C ABI of the B200-native FMM Helmholtz matvec (libhfmm_b200.so).
 *
 * This is the drop-in boundary for the ONE hot path of the reference: the FMM
 * matrix-vector product used inside GMRES.  The reference is a C++20 static library without an
 * FFI layer; its seams are ordinary functions.  Each entry point below names the reference
 * interface it stands in for (paths relative to /root/reference/proj/core).  The C++ mirror of
 * those interfaces (same names, argument meaning and exceptions) over this ABI is
 * include/hfmm_b200.hpp; INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Conventions: plain pointers and sizes only; complex arrays are interleaved (re, im) doubles —
 * bit-compatible with std::complex<double> / `cplx` (include/hfmm/common.hpp:14).  The caller owns
 * every host buffer; the handle owns all device memory, streams and communicators.  One call in
 * flight per handle (as "one apply at a time per system", include/hfmm/solver.hpp:92-94).
 * Every function returns an hfmm_status; no exception crosses this boundary.  There is NO CPU
 * fallback: without a CUDA device every compute call fails with HFMM_ERR_DEVICE.
 */
#ifndef HFMM_CUDA_H
#define HFMM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto the reference's error taxonomy (include/hfmm/common.hpp:43-55);
 * the C++ mirror rethrows the matching exception type. */
typedef enum {
  HFMM_OK = 0,
  HFMM_ERR_CONFIG = 1,     /* hfmm::config_error      */
  HFMM_ERR_SINGULAR = 2,   /* hfmm::singular_error    */
  HFMM_ERR_STRUCTURAL = 3, /* hfmm::structural_error  */
  HFMM_ERR_ACCURACY = 4,   /* hfmm::accuracy_error    */
  HFMM_ERR_DOMAIN = 5,     /* std::domain_error (point outside the box, octree.cpp:30-31) */
  HFMM_ERR_DEVICE = 6,     /* CUDA / NCCL failure, or no device: never falls back to the CPU */
  HFMM_ERR_INTERNAL = 9
} hfmm_status;

enum {
  /* build tree + interaction lists with the host C++ builder instead of the device builder (same
   * tree, same lists; cross-check).  The device builder has no list-size limit of its own: its pair lists grow
   * until they fit (60 % of the free device memory, 31 / 32-bit pair indexing) and lattice shifts beyond its
   * packed sort keys are classified on the host.  Only when the lists themselves exceed the device — a gate
   * that forbids every coarse translation — does set_points switch to the host builder by itself, and only up
   * to 262,144 points (hfmm_cuda_stats::host_tree_used says so; HFMM_FLAG_NO_HOST_FALLBACK forbids it) */
  HFMM_FLAG_HOST_TREE = 1 << 0,
  /* time each phase with CUDA events (fills hfmm_cuda_stats seconds); costs a few syncs */
  HFMM_FLAG_PHASE_TIMERS = 1 << 1,
  /* enqueue the near field before the far field.  Default: behind the persistent M2L launch, so that the M2L
   * CTAs own their SMs first and the near field takes what they leave (three near-field CTAs beside the one
   * sixteen-warp M2L CTA of orders 13..16; at orders <= 12 the gaps and the tail) */
  HFMM_FLAG_NEAR_FIRST = 1 << 2,
  /* run-to-run reproducible results (TraversalConfig::deterministic, traversal.hpp:11-22: per-target
   * ordered accumulation).  M2M and M2L stage one row per cell pair and add the rows of every
   * destination cell in list order instead of using floating-point atomics; costs two extra passes
   * over the staged rows (cfg 2: +22 % per matvec) and up to HFMM_ORDERED_STAGING_MB (environment,
   * default 4096) MiB of device memory.  The near field, the leaf passes and the Krylov reductions
   * are ordered in every mode. */
  HFMM_FLAG_DETERMINISTIC = 1 << 3,
  /* never switch to the host builder: when the device builder meets one of its limits (see
   * HFMM_FLAG_HOST_TREE) set_points fails with the builder's status instead.  hfmm_cuda_stats::
   * host_tree_used tells which builder produced the current tree either way. */
  HFMM_FLAG_NO_HOST_FALLBACK = 1 << 4
};

/* POD mirror of WaveNumber (common.hpp:37-40), TraversalConfig (traversal.hpp:11-18) and the
 * build_tree arguments (octree.hpp:84-90).  k = wave_r + i wave_i (WaveNumber,
 * common.hpp:36-40): wave_r > 0, |wave_i| <= 4 wave_r; wave_i > 0 is attenuation e^{-wave_i R}. */
typedef struct {
  double wave_r, wave_i;
  int order;       /* expansion order P (execute_plan `order`, traversal.hpp:59-62)           */
  int ncrit;       /* leaf capacity c                                                          */
  int grain;       /* task grain s; validated s >= c >= 1 (traversal.cpp:16-21), else unused   */
  double theta;    /* opening angle, 0 < theta <= 1                                            */
  double kd_max;   /* wavenumber gate; 0 disables (traversal.cpp:45-48)                        */
  double leaf_cap; /* max leaf diameter; 0 none; < 0: kd_max/|k| as solver.cpp:238-242         */
  int device;      /* CUDA device ordinal                                                      */
  int flags;       /* HFMM_FLAG_*                                                              */
} hfmm_cuda_config;

/* Mirror of FmmStats (traversal.hpp:44-52) plus tree/list statistics and per-kernel device times */
typedef struct {
  uint64_t n_bodies, n_cells, n_leaves, max_level;
  uint64_t m2l_pairs, p2p_pairs, p2p_body_pairs; /* cell pairs, leaf pairs, body pairs */
  uint64_t m2l_shift_classes, rotation_tables, coaxial_tables;
  uint64_t starved_cells;
  double setup_seconds;        /* tree + lists + tables + upload (once per point set)       */
  double upward_seconds;       /* P2M + M2M          (last matvec, CUDA events)              */
  double interaction_seconds;  /* M2L + P2P                                                  */
  double downward_seconds;     /* L2L + L2P                                                  */
  double p2p_seconds, m2l_seconds, p2m_seconds, m2m_seconds, l2l_seconds, l2p_seconds;
  double matvec_seconds;       /* whole device-side matvec                                   */
  uint64_t kernel_launches;    /* kernels launched by the last matvec                        */
  uint64_t device_bytes;       /* HBM held by the handle                                     */
  uint64_t m2l_batches;        /* work items of the M2L launch: <= 32 pairs of one shift class */
  uint64_t host_tree_used;     /* 1: tree and lists of this point set were built by the host builder
                                  (HFMM_FLAG_HOST_TREE, or the device builder's limits, see the flag) */
  uint64_t p2p_mode;           /* near-field kernel variant: 0 three MUFU per pair (any R'), 1..3 bounded
                                  R' with sin(R')/R' (and cos) as polynomials on the FMA pipe            */
  double near_r2_max;          /* bound on (k_r |x_i - x_j|)^2 over the near lists (selects p2p_mode)  */
  uint64_t tasks;              /* FmmStats::tasks: walk nodes where the body count first drops to the grain s
                                  (traversal.cpp:56-59)                                                 */
  uint64_t p2p_mode_in_step;   /* the variant the near field runs with INSIDE a matvec, beside the far field:
                                  0 when the far field outweighs it (the three-MUFU variant leaves the FMA pipe
                                  to M2L), else p2p_mode                                                    */
} hfmm_cuda_stats;

typedef struct hfmm_cuda hfmm_cuda_t;

/* Validates the configuration (config_error rules of traversal.cpp:16-21,212-213), selects the
 * device, creates streams.  Stands in for constructing TraversalConfig/KernelConfig. */
int hfmm_cuda_create(hfmm_cuda_t** out, const hfmm_cuda_config* cfg);
void hfmm_cuda_destroy(hfmm_cuda_t* h);
/* message of the last failure on this handle (or of the last failed create when h is NULL) */
const char* hfmm_cuda_last_error(const hfmm_cuda_t* h);

/* build_tree (octree.cpp:142-182) + dual_tree_traversal (traversal.cpp:82-97) on the same point
 * set as sources and targets: Morton order, octree, M2L/P2P lists, translation tables, all
 * device-resident afterwards.  xyz: n x 3 doubles, caller order. */
int hfmm_cuda_set_points(hfmm_cuda_t* h, const double* xyz, size_t n);

/* execute_plan (traversal.cpp:208-279): out[i] = sum_j G(x_i, x_j) q[j], j != coincident.
 * q, out: n interleaved complex doubles in CALLER order (Body::index mapping, solver.cpp:327-331).
 * Host buffers; host<->device copies happen inside the call. */
int hfmm_cuda_matvec(hfmm_cuda_t* h, const double* q, double* out);

/* Same product with operands already resident in HBM: q_dev / out_dev are device pointers to n
 * float2 (complex FP32) in caller order.  No host traffic, asynchronous on the handle's stream
 * until hfmm_cuda_sync. */
int hfmm_cuda_matvec_device(hfmm_cuda_t* h, const void* q_dev, void* out_dev);
int hfmm_cuda_sync(hfmm_cuda_t* h);

/* apply_operator tail (solver.cpp:327-328,340-357) and gmres_solve's block-Jacobi right
 * preconditioner (solver.cpp:376-382).  Any pointer group may be NULL to leave it unset.
 *   far_weight[n]                      x is scaled by it before the FMM (solver.cpp:327-328)
 *   patch_block[n/ni * ni * ni]        row-major complex blocks    (DiscreteSystem::patch_block)
 *   near_offset[n+1], near_source[nnz], near_delta[nnz]   CSR      (DiscreteSystem::near_*)
 *   block_lu[n/ni * ni * ni], block_piv[n]  LU factors + pivots    (DiscreteSystem::block_lu/piv)
 * After this call hfmm_cuda_matvec computes the full apply_operator. */
int hfmm_cuda_set_corrections(hfmm_cuda_t* h, int ni, const double* far_weight,
                              const double* patch_block, const uint32_t* near_offset,
                              const uint32_t* near_source, const double* near_delta,
                              const double* block_lu, const int32_t* block_piv);

/* GmresConfig / SolveReport (solver.hpp:97-116) */
typedef struct {
  double rtol;
  int restart;
  int max_iterations;
  int precondition; /* use block_lu as right preconditioner when set */
} hfmm_gmres_config;
typedef struct {
  int iterations;
  int converged;
  int breakdown;
  double rhs_norm;
  double final_residual;
  double seconds;
  double matvec_seconds;
  /* SolveReport::seconds / matvec_seconds (solver.hpp:106-116): optional caller buffers of history_cap
   * doubles, one entry per iteration — wall clock since the start of the solve, and the operator time
   * of that iteration (gmres.cpp:65-71,144).  Inputs; leave null / 0 when not wanted. */
  double* seconds_history;
  double* matvec_seconds_history;
  int history_cap;
} hfmm_gmres_report;

/* gmres / gmres_solve (gmres.cpp:35-174, solver.cpp:361-391) with device-resident Krylov vectors.
 * rhs, x: n interleaved complex doubles (host).  residuals (optional) receives up to
 * residual_cap per-iteration relative residual estimates. */
int hfmm_cuda_gmres(hfmm_cuda_t* h, const double* rhs, double* x, const hfmm_gmres_config* cfg,
                    hfmm_gmres_report* report, double* residuals, int residual_cap);

/* assemble_rhs (solver.cpp:302-312): rhs[i] = amplitude * exp(i k d . x_i) over the points of
 * set_points (caller order), k the handle's (complex) wavenumber; evaluated in FP64 on the device.
 * direction: 3 doubles, unit length (config_error beyond 1e-9, as the reference); amplitude: (re, im);
 * out: n interleaved complex doubles (host). */
int hfmm_cuda_assemble_rhs(hfmm_cuda_t* h, const double* direction, const double* amplitude, double* out);

/* evaluate_scattered_field (solver.cpp:393-419): plain single-layer sum at exterior points.
 * coeff: n complex (caller order, multiplied by far_weight inside); obs: nobs x 3; out: nobs complex.
 * Distances are formed in FP64 from the FP64 points.  When the patch diameters are known — after
 * hfmm_cuda_build_corrections, or hfmm_cuda_set_patch_diameters — an observation within 0.1 x patch
 * diameter of a sample fails with HFMM_ERR_SINGULAR like the reference (solver.cpp:399-413); without
 * them only coincident points are skipped (there is no geometry to test against). */
int hfmm_cuda_evaluate_field(hfmm_cuda_t* h, const double* coeff, const double* obs, size_t nobs,
                             double* out);
/* CurvilinearPatch::diameter() of every patch (n / ni of them, ni from set_corrections), for the
 * singular test of hfmm_cuda_evaluate_field when the corrections came through set_corrections */
int hfmm_cuda_set_patch_diameters(hfmm_cuda_t* h, const double* diameter, size_t n_patches);

/* Fills the statistics of the tree/lists and the per-kernel device times of the LAST matvec (CUDA
 * events recorded on the streams the kernels ran on; this call synchronises the handle). */
int hfmm_cuda_get_stats(hfmm_cuda_t* h, hfmm_cuda_stats* out);

/* ---- measurement helpers (bench.py): the handle launches on its own streams, which a caller's
 * events cannot see, so the caller drives events recorded on the handle's main stream ---------- */
int hfmm_cuda_timer_record(hfmm_cuda_t* h, int slot);                       /* slot in [0, 16) */
int hfmm_cuda_timer_elapsed_ms(hfmm_cuda_t* h, int slot_a, int slot_b, double* ms); /* waits for b */
int hfmm_cuda_flush_l2(hfmm_cuda_t* h);            /* writes a 256 MiB scratch buffer (L2 is 126 MB) */
int hfmm_cuda_fp32_peak_tflops(hfmm_cuda_t* h, double* tflops); /* FFMA-only probe, 2 flop per FFMA */

/* ---- introspection used by the parity tests (tree / list / expansion level checks) -------- */
/* cells in the library's level order: 8 x u32 per cell = level, ix, iy, iz, body_first,
 * body_count, child_first, child_count (same record as the checkers' *_fmm_cells) */
int hfmm_cuda_get_cells(hfmm_cuda_t* h, uint32_t* out, size_t capacity_cells);
/* Morton order: out[slot] = caller index (Body::index) */
int hfmm_cuda_get_body_order(hfmm_cuda_t* h, uint32_t* out);
/* which: 0 M2L cell pairs, 1 P2P leaf pairs; (target, source) u32 pairs, unspecified order.
 * Pass out == NULL to query the count only.  With nranks > 1 (device builder) the lists are built per rank:
 * exactly the pairs of the global walk whose target OR source cell this rank owns; hfmm_cuda_stats keeps the
 * counts of the global lists. */
int hfmm_cuda_get_pairs(hfmm_cuda_t* h, int which, uint32_t* out, uint64_t* count);
/* which: 0 multipole, 1 local, of the last matvec, UNSCALED back to the reference's convention
 * (M_n^m / L_n^m at index n(n+1)+m); out: n_cells x (P+1)^2 interleaved complex doubles */
int hfmm_cuda_get_expansions(hfmm_cuda_t* h, int which, double* out);

/* ---- multi-GPU: one process per GPU, Morton-partitioned ---------------------
 * Stands in for the reference's simulated-rank layer (part::distributed_matvec, let.cpp:320-362).
 * Every rank passes the GLOBAL point set to set_points after set_partition(rank, nranks): the
 * tree is identical on all ranks, the Morton order is cut into nranks contiguous body ranges balanced by
 * estimated work (a census pass of the dual tree walk that stores no pair: same cuts on every rank, no
 * handshake), and each rank then walks, stores and sorts only the pairs that touch a cell it owns — its
 * work (target owned) and what it must send (source owned).
 * hfmm_cuda_dist_matvec / hfmm_cuda_dist_solve below run the whole exchange inside the library.  The two
 * phase calls that follow are the building blocks for a caller that moves the data itself (and for the
 * single-device emulation of several ranks in the tests): all the charges in place -> dist_upward ->
 * the needed multipole rows in place (hfmm_cuda_partition, hfmm_cuda_get_exchange_masks) -> dist_downward. */
typedef struct {
  int32_t rank, nranks;
  uint64_t n_bodies, body_first, body_count;     /* owned Morton slots                           */
  int32_t level_first, level_last;               /* levels whose multipoles are exchanged        */
  uint32_t cell_first[22], cell_count[22];       /* owned cells per level: contiguous rows        */
  uint32_t level_cell_first[22], level_cell_count[22];
  uint64_t coeff_stride;                         /* complex FP32 elements per expansion row       */
  void* multipole_dev;                           /* [n_cells][coeff_stride] float2, device        */
  uint64_t owned_m2l_pairs, owned_p2p_body_pairs;
} hfmm_cuda_partition;
int hfmm_cuda_set_partition(hfmm_cuda_t* h, int rank, int nranks);   /* before set_points */
int hfmm_cuda_get_partition(hfmm_cuda_t* h, hfmm_cuda_partition* out);
/* q_morton_dev: n float2, FULL charge vector in Morton order (hfmm_cuda_get_body_order) */
int hfmm_cuda_dist_upward(hfmm_cuda_t* h, const void* q_morton_dev);
/* out_morton_dev: n float2 in Morton order; only the owned slots are written */
int hfmm_cuda_dist_downward(hfmm_cuda_t* h, void* out_morton_dev);

/* Locally essential trees (reference extract_let, let.cpp:150-253): per cell (n_cells entries, the
 * order of hfmm_cuda_get_cells), bit p of far_mask says rank p needs the cell's multipole (it is the
 * source of an M2L pair whose target p owns), bit p of near_mask says rank p needs the bodies of the
 * leaf; cell_rank is the owner (identical on all ranks).  A rank's lists hold every pair out of its own
 * cells and every pair into them, so the bits it reads — bit p of ITS OWN cells (send list) and ITS OWN bit
 * of p's cells (receive list) — are those of the global lists and the two sides match element for element
 * without any handshake; the other bits of foreign cells are not filled in.  At most 64 ranks. */
int hfmm_cuda_get_exchange_masks(hfmm_cuda_t* h, uint64_t* far_mask, uint64_t* near_mask, int32_t* cell_rank);

/* ---- repartitioning loop (reference partition.cpp:137-227) -------
 * measure_weights -> w = l + alpha r -> Morton cuts -> run -> update_alpha -> re-cut.  The work
 * estimates come from the interaction lists of the current point set; alpha is searched by the
 * caller's driver from measured matvec times (max over ranks). */
/* per body, caller order: local[i] = bodies of the P2P partner leaves of i's leaf, remote[i] = number
 * of M2L pairs of all cells holding i (measure_weights, partition.cpp:143-163).  With nranks > 1 the
 * entries of the bodies this rank owns are exact; the others only count the pairs out of this rank's cells. */
int hfmm_cuda_measure_weights(hfmm_cuda_t* h, double* local, double* remote);
/* balance the Morton cuts of hfmm_cuda_set_partition by sum(l + alpha r) (apply_weights,
 * partition.cpp:165-173); alpha < 0 (default) balances by measured kernel cost per list entry instead.
 * Takes effect at the next hfmm_cuda_set_points. */
int hfmm_cuda_set_partition_alpha(hfmm_cuda_t* h, double alpha);
/* next alpha to try given the history of (alpha, runtime) samples: golden-section replay over
 * [0, alpha_max], the best measured alpha once the bracket is tight (update_alpha,
 * partition.cpp:175-227).  config_error on an empty history or alpha_max <= 0. */
int hfmm_partition_update_alpha(const double* alpha, const double* runtime, int n, double alpha_max, double* next);

/* ---- correction builders on the device ------------------------------
 * Replace build_patch_blocks (proj/core/src/solver.cpp:80-128) and build_near_corrections
 * (solver.cpp:132-230).  The quadrature and interpolation tables are the reference's own
 * (geom::lagrange_basis, geom::gauss_rule, geom::duffy_rule of geometry.cpp), passed as arrays. */
typedef struct {
  int basis_count;            /* LagrangeBasis::count(): 3, 6 or 12 */
  int mode;                   /* SingularityMode: 0 none, 1 self_only, 2 self_near */
  uint64_t n_patches;
  const double* nodes;        /* n_patches x 6 x 3: CurvilinearPatch::node (geometry.hpp:14-15) */
  const double* sample_ref;   /* basis_count x (zeta, eta): LagrangeBasis::nodes() */
  const double* far_weight;   /* basis_count: LagrangeBasis::weights() */
  double near_patch_distance; /* KernelConfig::near_patch_distance; < 0: twice the patch diameter */
  int near_npts;              /* gauss_rule(KernelConfig::near_rule) */
  const double* near_pts;     /* near_npts x (zeta, eta, weight) */
  const double* near_basis;   /* near_npts x basis_count: basis.eval at the rule points */
  const int32_t* self_npts;   /* basis_count: size of duffy_rule centred on interpolation node j */
  const double* self_pts;     /* the Duffy rules, concatenated: sum(self_npts) x (zeta, eta, weight) */
  const double* self_basis;   /* sum(self_npts) x basis_count */
} hfmm_correction_rules;
/* Requires hfmm_cuda_set_points on the samples (patch-major: sample p * basis_count + j is
 * interpolation node j of patch p, solver.cpp:283-294).  Builds the arrays in FP64 on the device and
 * installs them as the handle's corrections (as hfmm_cuda_set_corrections would); *near_nnz receives
 * the length of the near CSR.  singular_error when a self block is singular (solver.cpp:55-56). */
int hfmm_cuda_build_corrections(hfmm_cuda_t* h, const hfmm_correction_rules* rules, uint64_t* near_nnz);
/* the FP64 arrays of the last build, in the reference's layout (DiscreteSystem, solver.hpp:60-90);
 * any pointer may be null */
int hfmm_cuda_get_corrections(hfmm_cuda_t* h, double* patch_block, double* block_lu, int32_t* block_piv,
                              uint32_t* near_offset, uint32_t* near_source, double* near_delta);

/* ---- the library's own data plane (reference let.cpp:150-362) -----------------
 * After hfmm_cuda_set_partition(rank, nranks) the handle can own a communicator:
 *   NCCL   rank 0 calls hfmm_cuda_nccl_unique_id and hands the 128 bytes to its peers by whatever bootstrap
 *          the application has (torchrun's store, MPI_Bcast, a file); every rank then calls
 *          hfmm_cuda_comm_init_nccl (ncclCommInitRank; collective).  NCCL is loaded at run time
 *          (libnccl.so.2), a single-GPU user needs none.
 *   host   the same packed buffers staged through pinned host memory, the collectives performed by two
 *          caller callbacks on HOST buffers — the MPI escape hatch, and the way two processes can share
 *          one GPU in tests (NCCL refuses two ranks on one device).
 * One matvec = pack kernel -> one grouped ncclSend/ncclRecv over all peers -> unpack kernel, for the halo
 * charges and for the multipoles of the cells the peers translate from (index lists fixed at set_points,
 * identical on both sides without a handshake), on a communication stream overlapped with the upward pass
 * and the near field.  The exchange index lists are rebuilt lazily after every hfmm_cuda_set_points. */
typedef struct {
  void* user;
  /* send / recv: host buffers; send_bytes[p] / recv_bytes[p]: bytes for / from rank p (nranks entries,
   * blocks in rank order, own entry 0).  Return 0 on success. */
  int (*alltoallv)(void* user, const void* send, const uint64_t* send_bytes, void* recv, const uint64_t* recv_bytes);
  int (*allreduce_sum)(void* user, double* values, int count);   /* host doubles, in place */
} hfmm_host_transport;
int hfmm_cuda_nccl_unique_id(void* out128);
int hfmm_cuda_comm_init_nccl(hfmm_cuda_t* h, const void* unique_id_128);
int hfmm_cuda_comm_init_host(hfmm_cuda_t* h, const hfmm_host_transport* transport);
/* plain FMM product over the ranks: q_owned_dev / out_owned_dev are device float2 arrays holding this rank's
 * slice [body_first, body_first + body_count) of the Morton-ordered vectors (hfmm_cuda_get_partition,
 * hfmm_cuda_get_body_order).  Asynchronous on the handle's streams until hfmm_cuda_sync. */
int hfmm_cuda_dist_matvec(hfmm_cuda_t* h, const void* q_owned_dev, void* out_owned_dev);
/* gmres / gmres_solve (gmres.cpp:35-174) over Morton-sharded vectors: rhs_owned / x_owned are body_count
 * interleaved complex doubles (host, Morton order).  Inner products are local FP64 reductions all-reduced
 * on the device (ncclAllReduce in stream order: no host round trip per coefficient); with corrections /
 * block-Jacobi set, the operand is all-gathered and the streaming BIE tail evaluated redundantly.  All ranks
 * see identical scalars and take identical branches. */
int hfmm_cuda_dist_solve(hfmm_cuda_t* h, const double* rhs_owned, double* x_owned, const hfmm_gmres_config* cfg,
                         hfmm_gmres_report* report, double* residuals, int residual_cap);
/* bytes this rank RECEIVES per matvec in the two exchanges (halo charges, remote multipoles) */
/* fmm_evaluate / execute_plan with DISTINCT target and source trees (traversal.hpp:59-67): out[t] = sum_j q_j
 * G(targets[t], x_j) over the handle's points x_j (strengths q, caller order, interleaved complex doubles) at
 * n_targets other points (3 doubles each); out: n_targets interleaved complex doubles.  A target that coincides
 * with a source skips that pair, as green_t does (kernel.hpp:22).  Runs the ordinary pipeline on one tree over
 * sources + targets held by a second engine inside the handle, rebuilt only when the targets change; single-domain
 * handles only.  Corrections and far weights of the handle are NOT applied (plain layer potential). */
int hfmm_cuda_evaluate_targets(hfmm_cuda_t* h, const double* targets, size_t n_targets, const double* q, double* out);
/* The residual vector b - Z u behind `final_residual` of the last hfmm_cuda_gmres / hfmm_cuda_dist_solve
 * (all unknowns in caller order, or the owned Morton slice): `capacity` interleaved complex doubles, FP32
 * values widened.  With max_iterations = restart a caller drives the restart cycles itself — solve
 * Z d = r, x += d, r <- this vector — and may re-cut the Morton partition between two cycles, which is
 * where the reference's repartitioning loop acts (partition.cpp:143-227; distributed.repartitioned_gmres). */
int hfmm_cuda_get_solve_residual(hfmm_cuda_t* h, double* out, size_t capacity);
int hfmm_cuda_get_exchange_volume(hfmm_cuda_t* h, uint64_t* charge_bytes, uint64_t* multipole_bytes);

const char* hfmm_cuda_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HFMM_CUDA_H */
