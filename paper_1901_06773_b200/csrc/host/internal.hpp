// Helpers shared by the host planner translation units (not public API).
#pragma once

#include <cstdint>
#include <filesystem>
#include <functional>
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

// What evaluate_minibatch computes about one k independently of the device
// budget and the host-link bandwidth (reused across re-plans, plan_session.cpp)
struct KStatic {
  std::vector<Bytes> sizes;           // k-scaled object sizes
  std::vector<std::int64_t> running;  // unpinned running sums over the GMAP ops
  Bytes top = 0;                      // their peak (the active area)
};
KStatic make_k_static(const Gmap& g, const std::vector<PhaseLayer>& phases, int k,
                      const PerfModel& model);
// the 2N phase compute times at k (throws like the reference on a model gap)
std::vector<TimeNs> k_compute_times(const Gmap& g, const std::vector<PhaseLayer>& phases, int k,
                                    const PerfModel& model);
// evaluate_minibatch from a KStatic; compute_of() supplies the phase compute
// times (called only past the memory gate)
KEvaluation evaluate_static(const Gmap& g, const KStatic& st, int k, const NetworkSpec& net,
                            const HardwareSpec& hw, double bandwidth,
                            const std::function<const std::vector<TimeNs>&()>& compute_of);
// find_efficiency_optimal_minibatch with the per-k evaluation supplied
PlanResult search_plan(const Gmap& gmap, const std::vector<PhaseLayer>& phases,
                       const NetworkSpec& net, const HardwareSpec& hw, const PerfModel& model,
                       const TrainingConfig& cfg, const PlannerOptions& opts,
                       const std::function<KEvaluation(int)>& evaluate);

}  // namespace swapsched::detail
