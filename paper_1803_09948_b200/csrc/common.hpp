// common.hpp — shared host-side types of libhfmm_b200 (status codes, config, error carrier).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "hfmm_cuda.h"

namespace hfmm_b200 {

// 3 bits per level, 21 levels in a 64-bit key (reference: include/hfmm/octree.hpp:26)
inline constexpr int kMaxLevel = 21;
// largest expansion order the tables and kernels are sized for
inline constexpr int kMaxOrder = 16;

// carries an hfmm_status through host code; capi.cpp turns it into a return code + message
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

// the pair lists of the DEVICE builder exceed the device memory / 32-bit pair indexing: Engine::set_points falls
// back to the host builder for moderate sizes (or reports it: HFMM_FLAG_NO_HOST_FALLBACK)
struct DeviceBuilderLimit : Error {
  // any_size: the host builder handles the input at the usual cost (O(N)); otherwise the lists
  // themselves are huge and the fallback is taken for moderate point counts only
  bool any_size;
  DeviceBuilderLimit(int s, const std::string& msg, bool any) : Error(s, msg), any_size(any) {}
};

inline int nm_index(int n, int m) { return n * (n + 1) + m; }
inline int nm_total(int p) { return (p + 1) * (p + 1); }
// row stride (in complex elements) of the device expansion arrays: padded to 4 complex = 32 B
inline int coeff_stride(int p) { return (nm_total(p) + 3) & ~3; }

}  // namespace hfmm_b200
