// host_tree.hpp — host C++ octree + dual-tree-traversal builder.
//
// Mirrors the semantics of the reference's build_tree (src/octree.cpp:53-182) and
// dual_tree_traversal (src/traversal.cpp:36-97) — same box, same level-21 Morton keys, same split
// rule, same admissibility and split-larger-cell rule, hence the same cell set and the same
// (target, source) pair sets — but lays the tree out LEVEL BY LEVEL (cells of one level are
// contiguous and key-sorted, siblings adjacent), the layout the device passes want, and walks the
// two trees as a breadth-first pair frontier instead of a recursion.  This is the
// HFMM_FLAG_HOST_TREE path; the device builder (tree_build.cu) produces the same arrays.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace hfmm_b200 {

struct TreeArrays {
  double lo[3] = {0, 0, 0};
  double width = 0;
  uint32_t n_bodies = 0;
  int max_level = 0;
  size_t degenerate_leaves = 0;

  std::vector<uint64_t> key;    // level-21 key per Morton slot
  std::vector<uint32_t> index;  // Morton slot -> caller index (Body::index)

  // cells, level order; cell 0 is the root
  std::vector<uint8_t> level;
  std::vector<uint32_t> ix, iy, iz;
  std::vector<uint32_t> body_first, body_count;
  std::vector<uint32_t> child_first, child_count;
  std::vector<uint32_t> parent;
  std::vector<uint32_t> level_offset;  // cells of level L are [level_offset[L], level_offset[L+1])
  std::vector<uint32_t> leaves;        // ascending cell index

  size_t n_cells() const { return level.size(); }
  double side(int lvl) const { return width / double(uint64_t(1) << lvl); }
};

struct PairLists {
  // admissible cell pairs (M2L) and leaf pairs (P2P), as flat (target, source) arrays
  std::vector<uint32_t> m2l_t, m2l_s, p2p_t, p2p_s;
  uint64_t tasks = 0;  // FmmStats::tasks: walk nodes whose bodies first fit the grain s (traversal.cpp:56-59)
};

// level-21 key of p inside the cubified box (octree.cpp:25-51); throws Error(HFMM_ERR_DOMAIN)
uint64_t morton_key21(const double p[3], const double lo[3], double width);

// cubified bounding box with the 1e-12 pad (reference src/octree.cpp:53-70); throws on non-finite input
void enclosing_box_host(const double* xyz, size_t n, double lo[3], double& width);

// throws Error(HFMM_ERR_CONFIG) on n == 0 / ncrit < 1
void build_tree_host(TreeArrays& tree, const double* xyz, size_t n, int ncrit, double leaf_cap,
                     int threads);

void dual_tree_traversal_host(const TreeArrays& tree, double kmag, double theta, double kd_max,
                              PairLists& out, int threads, int grain = 0);

// Cuts the Morton order into nranks contiguous body ranges.  Cut points sit on the
// boundaries of PARTITION UNITS = the cells of level `lcut` (the coarsest level that takes part in
// any translation) plus the leaves above it, so every cell that owns an expansion belongs to
// exactly one rank.  Units are weighed by the work their targets attract — the idea of the
// reference's w = l + alpha r (partition.cpp:137-141) with both terms in measured kernel time:
// near-field body pairs and M2L cell pairs.
//   cell_rank[c] : owning rank, -1 for the cells above the cut (they hold no expansion)
//   first/count  : owned Morton body range per rank (ranges tile [0, n) in rank order)
// the pieces of compute_morton_partition, so the device builder can supply the weights:
//   partition_units -> unit cell of every cell (0xffffffff above the cut), returns lcut
//   partition_cuts  -> ranks from per-unit weights
inline constexpr double kPartitionPairWeight = 1.0;   // measured kernel time per near body pair ...
inline constexpr double kPartitionM2lWeight = 1600.0; // ... against one M2L cell pair
int partition_units(const TreeArrays& tree, int lmin_src, int lmin_dst, std::vector<uint32_t>& unit);
void partition_cuts(const TreeArrays& tree, const std::vector<uint32_t>& unit,
                    const std::vector<double>& weight, int nranks, std::vector<int>& cell_rank,
                    std::vector<uint32_t>& first, std::vector<uint32_t>& count);
// alpha: see partition_weights_device
void compute_morton_partition(const TreeArrays& tree, const PairLists& pairs, int nranks, double alpha,
                              std::vector<int>& cell_rank, std::vector<uint32_t>& first,
                              std::vector<uint32_t>& count, int& lcut);

// Next alpha to try: golden-section replay over [0, alpha_max] against the measured history
// (reference update_alpha, partition.cpp:175-227).  Throws config_error like the reference.
double partition_update_alpha(const double* alpha, const double* runtime, int n, double alpha_max);

}  // namespace hfmm_b200
