// tree_build.cuh — device-side construction of the octree and the interaction lists (sm_100a).
//
// Same semantics as host_tree.cpp (which restates the reference's build_tree, src/octree.cpp:53-182,
// and dual_tree_traversal, src/traversal.cpp:36-97) — identical box, keys, cell set and pair sets —
// with the heavy loops on the GPU:
//   K1  level-21 Morton keys + stable radix sort of (key, caller index)        [bodies]
//   K2  level-synchronous top-down split: binary-search the 8 octant boundaries of every cell
//       in the sorted keys, scan the child counts, write the next level         [cells]
//   K3  breadth-first pair frontier with warp-aggregated appends: admissible -> M2L pair,
//       leaf-leaf -> P2P pair, else split the larger cell                        [cell pairs]
//   then: P2P pairs -> CSR by target leaf (touching leaves first) by one radix sort;
//         M2L pairs -> sorted by packed lattice-shift key, run-length encoded into shift classes.
// Admissibility is evaluated in FP64 with explicit round-to-nearest intrinsics (no FMA
// contraction), i.e. the same IEEE operation sequence as the host builder and the reference, so
// even exact ties (theta = 0.5 on a lattice) fall the same way.
// Radix sort / scan / run-length encoding come from CUB (setup only, never inside a matvec).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "device_utils.cuh"
#include "host_tree.hpp"

namespace hfmm_b200 {

struct DevicePairs {
  DeviceBuffer<uint2> far, near;  // (target, source) cell ids, unordered
  uint64_t n_far = 0, n_near = 0;
  uint64_t tasks = 0;  // FmmStats::tasks (traversal.cpp:56-59)
};

// K1 + K2.  Fills `tree` (host mirror: cells, leaves, index; `key` is left empty) and leaves the
// sorted keys / caller indices on the device.
void build_tree_device(TreeArrays& tree, const double* xyz_host, size_t n, int ncrit, double leaf_cap,
                       DeviceBuffer<double>& d_xyz, DeviceBuffer<uint32_t>& d_index, cudaStream_t s);

// device copy of the cell arrays the traversal and the list builders read
struct DeviceCells {
  DeviceBuffer<uint8_t> level;
  DeviceBuffer<uint32_t> ix, iy, iz, child_first, child_count, body_count;
  void upload(const TreeArrays& t, cudaStream_t s);
};

// K3
void dual_tree_traversal_device(const TreeArrays& tree, const DeviceCells& cells, double kmag,
                                double theta, double kd_max, int grain, DevicePairs& out, cudaStream_t s);

// Multi-rank setup, pass 1: the SAME global descent, but nothing is stored — every accepted pair only adds its
// work to its target cell (partition_weights_device's model) and to the totals; memory is the frontier alone.
struct TraversalCensus {
  uint64_t n_far = 0, n_near = 0, tasks = 0, body_pairs = 0;  // of the whole (global) lists
  int lmin_dst = 0, lmin_src = 0;                              // far_pair_level_range of the global lists
  std::vector<double> cell_weight;                             // per TARGET cell
};
void dual_tree_census_device(const TreeArrays& tree, const DeviceCells& cells, double kmag, double theta,
                             double kd_max, int grain, double alpha, TraversalCensus& out, cudaStream_t s);
// Multi-rank setup, pass 2: the descent pruned to one rank.  `interest[c]` != 0 iff the subtree of cell c holds a
// cell the rank owns; a node (t, s) of the walk survives iff interest[t] | interest[s], so the lists hold exactly
// the pairs whose target the rank owns (its work) or whose source it owns (what it sends: the exchange masks).
void dual_tree_traversal_pruned_device(const TreeArrays& tree, const DeviceCells& cells, double kmag, double theta,
                                       double kd_max, const std::vector<uint8_t>& interest, DevicePairs& out,
                                       cudaStream_t s);

// min level over the M2L targets / sources (kMaxLevel + 1 when there are no pairs)
void far_pair_level_range(const DevicePairs& p, const DeviceCells& cells, int& lmin_dst, int& lmin_src,
                          cudaStream_t s);

// per-unit work weights of the Morton partition (host_tree.hpp: compute_morton_partition)
// alpha < 0: default model; alpha >= 0: the reference's w = l + alpha r per body (partition.cpp:137-163)
void partition_weights_device(const DevicePairs& p, const DeviceCells& cells,
                              const std::vector<uint32_t>& unit_of_cell, double alpha,
                              std::vector<double>& weight, cudaStream_t s);

struct NearLists {
  uint64_t n_owned_pairs = 0, body_pairs = 0, owned_body_pairs = 0;
  // bound on the squared distance of any two bodies of an owned near pair, in half-sides of the
  // finest level (the cubes' farthest corners): selects the bounded near-field kernel (kernels.cuh)
  uint64_t max_r2_lattice = 0;
  std::vector<uint64_t> work;  // per leaf slot: sum of source body counts
};
// CSR by target leaf slot, touching source leaves first, sources ascending inside each part;
// pairs whose target is not owned are dropped
void build_near_lists_device(const DevicePairs& p, const TreeArrays& tree, const DeviceCells& cells,
                             const std::vector<uint8_t>& owned, DeviceBuffer<uint32_t>& offset,
                             DeviceBuffer<uint32_t>& split, DeviceBuffer<uint32_t>& src, NearLists& out,
                             cudaStream_t s);

struct FarClasses {
  // one entry per distinct (level pair, lattice shift) among the owned M2L pairs, in sorted order
  std::vector<int32_t> dx, dy, dz;
  std::vector<int16_t> lt, ls;
  std::vector<uint32_t> count;
  uint64_t n_owned_pairs = 0;
};
// pairs sorted by shift class: pair_src / pair_dst hold the owned pairs class by class
void build_far_classes_device(const DevicePairs& p, const TreeArrays& tree, const DeviceCells& cells,
                              const std::vector<uint8_t>& owned,
                              DeviceBuffer<uint32_t>& pair_src, DeviceBuffer<uint32_t>& pair_dst,
                              FarClasses& out, cudaStream_t s);

// Reorders the class-sorted pairs segment by segment: the pairs of new segment s (positions
// seg_new[s] .. seg_new[s+1]) come from old positions seg_old[s] ..; pair_cls receives seg_cls[s]
void regroup_pairs_device(const std::vector<uint32_t>& seg_new, const std::vector<uint32_t>& seg_old,
                          const std::vector<uint32_t>& seg_cls, uint64_t n_pairs,
                          DeviceBuffer<uint32_t>& pair_src, DeviceBuffer<uint32_t>& pair_dst,
                          DeviceBuffer<uint32_t>& pair_cls, cudaStream_t s);

// Deterministic accumulation (HFMM_FLAG_DETERMINISTIC): for the pairs [begin, begin + n) of a stage,
// perm = their range-relative indices sorted by destination (stable: ties keep pair order), cut into
// one segment per destination: seg_dst[s], perm slots seg_begin[s] .. seg_begin[s + 1].  Returns the
// number of segments.
uint32_t build_ordered_reduce_device(const uint32_t* pair_dst, uint64_t begin, uint32_t n,
                                     DeviceBuffer<uint32_t>& perm, DeviceBuffer<uint32_t>& seg_dst,
                                     DeviceBuffer<uint32_t>& seg_begin, cudaStream_t s);

// leaf-relative, k-scaled coordinates and their hi/lo split (kernels.cuh), plus absolute ones
void build_body_arrays_device(const TreeArrays& tree, const DeviceBuffer<double>& d_xyz,
                              const DeviceBuffer<uint32_t>& d_index, double k, double grid,
                              DeviceBuffer<float4>& pos, DeviceBuffer<float4>& hi,
                              DeviceBuffer<float4>& lo, DeviceBuffer<float4>& abs_pos, cudaStream_t s);

}  // namespace hfmm_b200
