// kernels.cuh — device data layout and launcher declarations of the hand-written sm_100a kernels.
//
// HBM layout (all arrays Morton / level ordered, structure-of-arrays):
//   body_pos[slot]   float4  k * (x - centre(leaf(slot)))            leaf-relative, pre-scaled by k
//   body_q[slot]     float2  charge of the current matvec (x[index] * far_weight[index])
//   cell_geom[cell]  int4    (cx, cy, cz, level): lattice centre in half-sides of the finest level
//   cell_body[cell]  uint2   (body_first, body_count)
//   multipole/local  float2  [cell][coeff_stride(P)]  level-scaled coefficients (tables.hpp)
//   body_hi/body_lo  float4  the same coordinate split as hi + lo (hi on a power-of-two grid)
// Leaf-relative positions keep x_i - x_j accurate to ~1e-9 (absolute FP32 coordinates in a box of
// width 2 would cost 1e-7/|x_i-x_j| relative error on the nearest pairs).
// That is still not enough for the closest pairs of a random set (1e3..1e6 times closer than the
// mean spacing, and dominating the L2 norm of the potential): bodies of touching leaves are
// therefore differenced as (hi_t - hi_s - o_hi) + (lo_t - lo_s - o_lo), the first bracket exact,
// which gives x_i - x_j to FP32 RELATIVE accuracy — what the reference's Precision::f32 path gets
// by differencing in FP64 before it narrows (kernel.hpp:18).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hfmm_b200 {

// ---- P2P (near field, reference traversal.cpp:175-204 + kernel.hpp:16-23) --------------------
struct P2PTile {
  uint32_t leaf;      // target leaf cell id
  uint32_t body_off;  // first target body of this tile, relative to the leaf's body_first
  uint32_t n_t;       // targets in the tile (<= 32)
  uint32_t list;      // index into p2p_offset (source leaves of `leaf`, self excluded)
};

struct P2PArgs {
  const P2PTile* tiles;
  uint32_t n_tiles;
  // CSR over target leaves.  Entries [offset[i], split[i]) are the TOUCHING source leaves (cubes
  // share a face, edge or corner, the target leaf itself included): they can hold arbitrarily
  // close body pairs and are evaluated with compensated coordinates.  [split[i], offset[i+1]) are
  // the remaining source leaves (at least one cell apart), evaluated with plain FP32 coordinates.
  const uint32_t* p2p_offset;
  const uint32_t* p2p_split;
  const uint32_t* p2p_src;     // source leaf cell ids
  const int4* cell_geom;
  const uint2* cell_body;
  const float4* body_pos;      // float(k * x_rel)
  const float4* body_hi;       // k * x_rel rounded to the grid `grid`
  const float4* body_lo;       // k * x_rel - hi  (|lo| <= grid/2)
  const float2* body_q;
  float2* out;       // per Morton slot, overwritten (every body belongs to exactly one tile)
  float kunit;       // k * half-side of the finest level: lattice units -> scaled coordinates
  double kunit_d;    // the same in FP64 (exact offsets for the compensated path)
  double grid;       // power of two; hi parts and hi offsets are integer multiples of it
  float out_scale;   // k / (4 pi)
  float damp;        // (k_i / k_r) log2(e): complex wavenumber, amplitude 2^{-damp R'}; 0 for real k
  // Bounded near field: when every listed leaf pair keeps R'^2 = |k_r (x_i - x_j)|^2 <= r2_max (the
  // engine computes the exact bound from the lattice, set_points), sin(R')/R' is evaluated as a
  // degree-6 polynomial in R'^2 on the FMA pipe (sinc_c, fitted to [0, r2_max] at setup) and only
  // rsqrt and cos stay on the MUFU pipe: two MUFU per pair instead of three.  mode 0 keeps the
  // general three-MUFU evaluation (unbounded R': no leaf cap, gate-blocked leaves).
  int mode;          // P2P_MODE_*
  float sinc_c[8];   // sin(sqrt(u))/sqrt(u) ~ sum_i sinc_c[i] u^i on [0, r2_max]
  float cos_c[8];    // cos(sqrt(u))         ~ sum_i cos_c[i] u^i
};
enum { P2P_MODE_MUFU = 0, P2P_MODE_SINC_POLY = 1, P2P_MODE_SINC_POLY_EXPANDED = 2, P2P_MODE_ALL_POLY = 3 };
constexpr int kP2PPolyDegree = 6;
constexpr float kP2PPolyMaxR2 = 16.0f;  // beyond R' = 4 the polynomial loses to FP32 cancellation: mode 0
// least-squares-free near-minimax fit (Chebyshev interpolation) of sinc / cos in u = R'^2 on [0, r2_max]
void fit_p2p_polynomials(double r2_max, float sinc_c[8], float cos_c[8]);
void launch_p2p(const P2PArgs& a, cudaStream_t s);

// ---- P2M / L2P (reference expansion.cpp:157-175, 283-300) -----------------------------------
struct LeafExpansionArgs {
  const uint32_t* leaves;  // leaf cell ids to process
  uint32_t n_leaves;
  const int4* cell_geom;
  const uint2* cell_body;
  const float4* body_pos;
  const float* level_scale;  // s_l = k * side(l), indexed by level
  int order;
  int stride;                // coefficient row stride (complex elements)
  float k;                   // Re k
  float k_imag;              // Im k (attenuation); 0 selects the real-argument kernels
  bool small_arguments = false;  // every body of every listed leaf has k rho <= 1 (7-term series): unrolled kernels
};
void launch_p2m(const LeafExpansionArgs& a, const float2* body_q, float2* multipole, cudaStream_t s);
// out[slot] = sum over the leaf's local expansion (overwrites; bodies of unlisted leaves untouched)
void launch_l2p(const LeafExpansionArgs& a, const float2* local, float2* out, cudaStream_t s);
// Legendre recurrence coefficients -> __constant__ memory (tables.hpp build_legendre_coefficients)
void upload_legendre_constants(const float* diag, const float* sub, const float* a, const float* b,
                               int order);

// ---- batched translation: M2M / M2L / L2L (reference expansion.cpp:95-139) -------------------
struct TranslateClass {
  uint32_t rot;   // rotation table id
  uint32_t coax;  // coaxial table id
  float cphi, sphi;
};
struct TranslateItem {
  uint32_t pair_begin;
  uint32_t count;  // <= translate_batch_size(order) pairs of one table group
  uint32_t cls;    // class of the first pair
  uint32_t group;  // table group: classes with the same rotation and coaxial table (they differ in azimuth)
};
inline constexpr int kTranslateBatch = 32;   // pairs per work item (= lanes of a warp)
inline constexpr int kTranslateWarps = 16;   // most warps per CTA of the translation kernel (8 or 16)
inline constexpr int kTranslateMaxTasks = 40;

// Per-order static schedule of the translation kernel (kept in __constant__ memory): each stage is a
// list of tasks grouped per warp.  A task is a PAIR of sub-tasks, one per half-warp (a lane owns two
// of the 32 pairs of a batch); a sub-task carries every shared-memory offset it needs (bytes).
struct TranslateRotSub {
  uint32_t e_off;    // first coefficient of the sub-task's row tile (byte offset in the window)
  uint32_t in_rel;   // first input row of the folded sub-block, relative to the tile (bytes)
  uint32_t out_rel;  // first output row (bytes)
  uint32_t packed;   // row stride (bytes) | inputs << 8 | rows stored << 16 | (first row odd) << 24 | template rows << 28
};
struct TranslateRotTask {
  TranslateRotSub sub[2];
};
struct TranslateCoaxSub {
  uint32_t c_off;    // first coefficient (byte offset in the window)
  uint32_t p_rel;    // input row (n = m) of the s / x_0 column, relative to the tile (bytes)
  uint32_t q_rel;    // input row (n = m) of the t column (bytes)
  uint32_t packed;   // row stride (bytes) | inputs << 8 | m << 16 | first row << 22 | rows stored << 28
};
struct TranslateCoaxTask {
  TranslateCoaxSub sub[2];
};
struct TranslateSchedule {
  int rot_begin[kTranslateWarps + 1];
  int coax_begin[kTranslateWarps + 1];
  TranslateRotTask rot[kTranslateMaxTasks];
  TranslateCoaxTask coax[kTranslateMaxTasks];
};
void build_translate_schedule(int order, TranslateSchedule* out);
void upload_translate_schedule(int order);  // into the kernel's constant memory slot of `order`

struct TranslateArgs {
  const TranslateItem* items;
  uint32_t n_items;
  const TranslateClass* classes;
  const uint32_t* pair_src;
  const uint32_t* pair_dst;
  const uint32_t* pair_cls;  // shift class of every pair (azimuth phases)
  const float* rot_tables;   // [rot][rot_table_size(P)]
  const float* coax_tables;  // [coax][2 * coax_table_size(P)]
  const float2* src;         // expansions read
  float2* dst;               // expansions accumulated into (atomically)
  int order;
  int stride;
  int mixed;                 // batches mix classes of a table group (per-pair phases) / one class per batch
  int staged;                // every pair owns its dst row (deterministic mode): plain stores instead of atomics
  int prefetch = 0;          // 64-pair kernel: prefetch the next batch's source rows into L2
};
void launch_translate(const TranslateArgs& a, cudaStream_t s);
// pairs per work item expected by the kernel
int translate_batch_size(int order);

// ---- the 64-pair in-place translation kernel (kernels_translate64.cu), orders <= 16 ------------
inline constexpr int kTranslate64MaxOrder = 12;   // two 8-warp CTAs per SM up to here
inline constexpr int kTranslate64TopOrder = 16;   // one 16-warp CTA per SM up to here
inline constexpr int kTranslate64MaxWarps = 16;
inline constexpr int kTranslate64MaxTasks = 64;
// one whole folded system of a degree (rotations) or one folded column of an order (coaxial step)
struct Translate64Task {
  uint32_t tab_off;  // first coefficient row: byte offset in the shared-memory window
  uint16_t ws_b;     // coefficient row stride, bytes
  uint16_t row0;     // tile row of input / output 0
  int16_t step;      // rotations: +1 / -1 per index; coaxial: 2m + 2, growing by 2 per degree
  uint8_t w;         // inputs = outputs
  uint8_t half;      // 0: all 64 pairs (a lane owns two); 1 / 2: pairs 0..31 / 32..63 (a lane owns one)
};
struct Translate64Schedule {
  int rot_begin[kTranslate64MaxWarps + 1];
  int coax_begin[kTranslate64MaxWarps + 1];
  Translate64Task rot[kTranslate64MaxTasks];
  Translate64Task coax[kTranslate64MaxTasks];
};
bool translate64_supported(int order);       // HFMM_TRANSLATE=32 selects the 32-pair kernel for every order
int translate64_warps(int order);            // 8 (two CTAs per SM) or 16 (one)
// the 64-pair kernel expects block m of every coaxial table multiplied by (-1)^m (the input signs of
// the inverse rotation, tables.hpp); the 32-pair kernel applies them itself
bool coax_tables_sign_folded(int order);
void build_translate64_schedule(int order, Translate64Schedule* out);
void upload_translate64_schedule(int order);
void launch_translate64(const TranslateArgs& a, cudaStream_t s);

// ---- vector plumbing -------------------------------------------------------------------------
// body_q[slot] = float2(q[index[slot]]) * weight[index[slot]] (weight may be null)
void launch_gather_charges(const double2* q_caller, const float2* q_caller_f32,
                           const uint32_t* index, const float* weight, float2* body_q, uint32_t n,
                           cudaStream_t s);
// out[index[slot]] = near[slot] + far[slot] (far may be null); exactly one of out_f64 / out_f32 is written
void launch_scatter_potentials(const float2* near, const float2* far, const uint32_t* index,
                               double2* out_f64, float2* out_f32, uint32_t n, cudaStream_t s);

// Deterministic accumulation: dst row seg_dst[s] += the staged rows perm[seg_begin[s] .. seg_begin[s+1])
// in that order (one warp per segment; no atomics).  Rows are `stride` float2 apart, `dim` are used.
void launch_ordered_reduce(const float2* staging, const uint32_t* perm, const uint32_t* seg_begin,
                           const uint32_t* seg_dst, uint32_t n_segs, float2* dst, uint32_t stride,
                           uint32_t dim, cudaStream_t s);
// row_of_pair[i] = i - begin for i in [begin, begin + n)
void launch_range_rows(uint32_t* row_of_pair, uint64_t begin, uint32_t n, cudaStream_t s);

// ---- BIE operator tail + Krylov vector ops (kernels_krylov.cu) -------------------------------
// y += blockdiag x + CSR x and the per-patch LU solve: FP64 values and accumulation, FP32 vectors
void launch_corrections(uint32_t n, int ni, const double2* block, const uint32_t* off, const uint32_t* src,
                        const double2* delta, const float2* x, float2* y, cudaStream_t s);
void launch_precondition(uint32_t npatch, int ni, const double2* lu, const int* piv, const float2* in,
                         float2* out, cudaStream_t s);
// The reducing kernels (mgs_step, norm2, residual) sum in a fixed order (reproducible run to run):
// scratch = reduce_scratch_doubles() zero-initialised doubles, private to the stream.
size_t reduce_scratch_doubles();
// w -= h_prev * v_prev (skipped when v_prev is null); out[0..1] += <v_next, w> (skipped when null)
void launch_mgs_step(uint32_t n, float2* w, const float2* v_prev, const double* h_prev,
                     const float2* v_next, double* out, double* scratch, cudaStream_t s);
void launch_norm2(uint32_t n, const float2* w, double* out, double* scratch, cudaStream_t s);
void launch_scale(uint32_t n, const float2* in, float scale, float2* out, cudaStream_t s);
void launch_update_solution(uint32_t n, int cols, const float2* basis, size_t ld, const double* y,
                            double2* x, cudaStream_t s);
void launch_residual(uint32_t n, const double2* b, const float2* ax, float2* r32, double* out,
                     double* scratch, cudaStream_t s);
void launch_narrow(uint32_t n, const double2* in, float2* out, cudaStream_t s);
// out[o] = scale * sum_i q_i e^{i k|o-x_i|} e^{-eps k|o-x_i|}/(k|o-x_i|), distances in FP64 from the FP64
// points (caller order); touch2 (per patch of ni samples, may be null): *flag = 1 when |o-x_i|^2 <= touch2
void launch_field(uint32_t n, const double* xyz, const float2* q, const double* obs, uint32_t nobs, double k,
                  float scale, float eps, const double* touch2, uint32_t ni, double2* out, int* flag,
                  cudaStream_t s);
// out[i] = amp * exp(i (kr + i ki) dir . x_i), FP64
void launch_assemble_rhs(uint32_t n, const double* xyz, const double dir[3], double kr, double ki,
                         const double amp[2], double2* out, cudaStream_t s);
void launch_widen(uint32_t n, const float2* in, double2* out, cudaStream_t s);

// out[s] = near[s] + far[s] + corr[index[s]], s over the owned Morton slots (corr may be null)
void launch_combine_owned(const float2* near, const float2* far, const float2* corr, const uint32_t* index,
                          float2* out, uint32_t n, cudaStream_t s);

// FFMA-only micro-benchmark; returns TFLOP/s (2 flop per FFMA)
// packed: the same chains issued as FFMA2 (fma.rn.f32x2)
double run_fp32_peak_probe(cudaStream_t s, bool packed = false);

}  // namespace hfmm_b200
