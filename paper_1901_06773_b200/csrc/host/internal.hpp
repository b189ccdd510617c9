// Helpers shared by the host planner translation units (not public API).
#pragma once

#include <cstdint>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "swapsched/api.hpp"

namespace swapsched::detail {

inline std::string slurp(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path.string());
  std::ostringstream buf;
  buf << in.rdbuf();
  return buf.str();
}

// 0 stays 0, anything else rounds up to the allocator granule
inline Bytes round_granule(Bytes raw) {
  if (raw == 0) return 0;
  return (raw + kAlignGranule - 1) / kAlignGranule * kAlignGranule;
}

std::int64_t op_delta(MemOpKind kind, std::int64_t size, bool pinned);
std::vector<Bytes> scaled_object_sizes(const Gmap& g, int k);
std::vector<char> pin_mask(const Gmap& g, const PinSet& pins);
// max(0, running-sum maximum) with the given pin mask
Bytes peak_only(const Gmap& g, const std::vector<Bytes>& sizes,
                const std::vector<char>& pinned);

}  // namespace swapsched::detail
