// swapsched-compatible host API of the B200 AccUDNN hot path.
//
// This single header declares every name the reference `swapsched` library
// exposes under /root/reference/proj/include/swapsched/*.hpp, with the same
// signatures and value semantics, so that code written against the reference
// (its CLI, its doctest suites, its acceptance binary) compiles unchanged
// against libswapsched_b200.so.  The per-module headers next to this file
// (types.hpp, model_ir.hpp, ...) only forward here.
//
// What is *different* is the implementation behind it (csrc/host/*.cpp):
// the layer-wise peak test used by the greedy pinning round is a lazy
// segment tree (O(log ops) per candidate instead of a full traversal), the
// blocked-allocation scan in Algorithm 1 is a binary search, curve queries
// bisect the knot list, and the minibatch search evaluates k values in
// parallel waves.  All integer/FP operations that feed a decision are
// evaluated in the reference's order, so k*, the pin set and t_ready are
// bit-identical (checked against the compiled reference in tests/).
#pragma once

#include <cmath>
#include <cstdint>
#include <filesystem>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace swapsched {

// ---------------------------------------------------------------------------
// Units (ref: include/swapsched/types.hpp:10-38)
// ---------------------------------------------------------------------------
using TimeNs = std::int64_t;   // all durations: integer nanoseconds
using Bytes = std::uint64_t;
using Flops = std::uint64_t;

constexpr Bytes kAlignGranule = 512;  // device allocator granule

inline double to_seconds(TimeNs t) { return static_cast<double>(t) * 1e-9; }
inline TimeNs from_seconds(double s) {
  return static_cast<TimeNs>(std::llround(s * 1e9));
}
// llround(1e9 * bytes / bw); the product is formed first, as in the reference
inline TimeNs transfer_duration(Bytes bytes, double bandwidth_bytes_per_s) {
  if (bandwidth_bytes_per_s <= 0.0)
    throw std::invalid_argument("transfer_duration: bandwidth must be > 0");
  const double scaled = 1e9 * static_cast<double>(bytes);
  return static_cast<TimeNs>(std::llround(scaled / bandwidth_bytes_per_s));
}
inline TimeNs compute_duration(Flops flops, double flops_per_s) {
  if (flops_per_s <= 0.0)
    throw std::invalid_argument("compute_duration: throughput must be > 0");
  const double scaled = 1e9 * static_cast<double>(flops);
  return static_cast<TimeNs>(std::llround(scaled / flops_per_s));
}

// Error taxonomy (ref: types.hpp:41-53).  Infeasibility is a value, never
// an exception (PlanStatus).
struct SpecError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UntrainableError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// Network description and GMAP (ref: include/swapsched/model_ir.hpp:14-150)
// ---------------------------------------------------------------------------
enum class LayerType { conv, bn, activation, pooling, fc, other };
std::string layer_type_name(LayerType t);
std::optional<LayerType> layer_type_from(const std::string& name);

struct LayerDecl {
  int index = 0;  // 1-based position in the network
  LayerType layer_type = LayerType::other;
  std::string type_tag;  // curve key for LayerType::other
  Flops flops_fwd_base = 0;
  std::optional<Flops> flops_bwd_base;
  Bytes featuremap_bytes_base = 0;  // scales with the minibatch
  Bytes param_bytes = 0;
  Bytes grad_bytes = 0;
  Bytes workspace_bytes_base = 0;   // scales with the minibatch
  std::string type_key() const;
};

struct NetworkSpec {
  std::string name;
  int num_layers = 0;
  int k_base = 1;
  double backward_flops_factor = 2.0;
  std::vector<LayerDecl> layers;
  const LayerDecl& layer(int index) const { return layers.at(index - 1); }
  Bytes param_grad_bytes_total() const;
};

enum class Direction { forward, backward };

struct PhaseLayer {
  int phase_index = 0;   // 1..2N
  int source_layer = 0;  // 1..N
  Direction direction = Direction::forward;
  Flops flops_base = 0;
  std::string type_key;
};

enum class ObjectKind { featuremap, workspace, param, grad };
using ObjectId = std::uint32_t;
using PinSet = std::set<ObjectId>;

struct MemObject {
  ObjectId id = 0;
  std::string name;
  ObjectKind kind = ObjectKind::featuremap;
  Bytes size_base = 0;
  bool scales_with_minibatch = true;
  int producer_phase = 0;
  int last_use_phase = 0;
};

enum class MemOpKind { allocate, release, offload, prefetch };
std::string mem_op_kind_name(MemOpKind k);

struct MemOp {
  MemOpKind kind = MemOpKind::allocate;
  ObjectId object = 0;
  int phase = 0;
  std::uint32_t sequence_no = 0;
};

struct Gmap {
  int num_phases = 0;
  int k_base = 1;
  std::vector<MemObject> objects;
  std::vector<MemOp> ops;                  // ascending sequence_no
  std::vector<std::uint32_t> phase_begin;  // num_phases + 1 offsets into ops

  const MemObject& object(ObjectId id) const { return objects.at(id); }
  std::pair<std::uint32_t, std::uint32_t> phase_range(int j) const {
    return {phase_begin.at(j - 1), phase_begin.at(j)};
  }
  Bytes op_bytes(const MemOp& op, int k) const;
  std::vector<ObjectId> featuremap_ids() const;
  void index_phases();
};

struct HardwareSpec {
  Bytes memory_budget = 0;
  Bytes m_others = 0;
  double delta_sync_s = 0.0;
  double pcie_nominal = 0.0;
};

NetworkSpec parse_network_spec(const std::filesystem::path& path);
NetworkSpec parse_network_spec_json(const std::string& text,
                                    const std::string& origin);
HardwareSpec parse_hardware_spec(const std::filesystem::path& path);
HardwareSpec parse_hardware_spec_json(const std::string& text,
                                      const std::string& origin);
std::string network_spec_to_json(const NetworkSpec& net);
std::string hardware_spec_to_json(const HardwareSpec& hw);
void validate_network_spec(const NetworkSpec& net);
std::vector<PhaseLayer> unfold_network(const NetworkSpec& net);
Gmap build_gmap(const std::vector<PhaseLayer>& phases, const NetworkSpec& net);
Bytes scaled_bytes(Bytes size_base, int k, int k_base, bool scales);
Bytes scale_size(const MemObject& obj, int k, int k_base);

struct PeakResult {
  Bytes peak_bytes = 0;
  std::uint32_t op_begin = 0;
  std::uint32_t op_end = 0;
  std::vector<ObjectId> live_objects;
};
PeakResult peak_layerwise_memory(const Gmap& gmap, int k, const PinSet& pins);
Bytes active_area_peak(const Gmap& gmap, int k, const PinSet& pins);
std::vector<std::string> validate_gmap(const Gmap& gmap);

// ---------------------------------------------------------------------------
// Profiles (ref: include/swapsched/profiles.hpp:13-57)
// ---------------------------------------------------------------------------
struct ComputeSample {
  int minibatch = 0;
  int phase = 0;
  std::string layer_type;
  Flops flops = 0;
  double time_s = 0.0;
};
struct TransferSample {
  int minibatch = 0;
  std::uint32_t seq_no = 0;
  Bytes bytes = 0;
  double time_s = 0.0;
};
struct ProfileSet {
  std::vector<ComputeSample> compute_samples;
  std::vector<TransferSample> transfer_samples;
  std::set<int> sampled_minibatches;
  std::vector<std::string> diagnostics;
};
struct ProfileLoadOptions {
  double min_sample_s = 1e-6;
};
ProfileSet load_profiles(const std::vector<std::filesystem::path>& paths,
                         const ProfileLoadOptions& opts = {});
ProfileSet parse_profile_csv(const std::string& text, const std::string& origin,
                             const ProfileLoadOptions& opts = {});
Flops scale_flops_count(Flops flops_base, int k, int k_base);
Flops scale_flops(const PhaseLayer& phase, int k, int k_base);
double effective_bandwidth(const std::vector<TransferSample>& samples,
                           double fallback);

// ---------------------------------------------------------------------------
// Performance model (ref: include/swapsched/perf_model.hpp:16-66)
// ---------------------------------------------------------------------------
struct ThroughputCurve {
  std::string layer_type;
  std::vector<std::pair<Flops, double>> knots;
  double plateau = 0.0;
  double efficiency = 1.0;
  double rate_at(Flops flops) const;
};
struct TrainingConfig {
  long long epochs = 1;
  long long dataset_size = 0;
  double delta_sync_s = 0.0;
};
struct PerfModel {
  std::map<std::string, ThroughputCurve> curves;
  double bandwidth_avail = 0.0;
  int k_base = 1;
  const ThroughputCurve& curve_for(const std::string& type_key) const;
};
ThroughputCurve fit_throughput_curve(const std::vector<ComputeSample>& samples,
                                     double eta);
PerfModel build_perf_model(const ProfileSet& profiles, int k_base, double eta,
                           double bandwidth_fallback);
TimeNs layer_compute_time(const PhaseLayer& phase, int k, const PerfModel& model);
std::vector<TimeNs> phase_compute_times(const std::vector<PhaseLayer>& phases,
                                        int k, const PerfModel& model);
TimeNs iteration_time(const std::vector<PhaseLayer>& phases, int k,
                      const PerfModel& model);
double whole_training_time_s(const std::vector<PhaseLayer>& phases, int k,
                             const PerfModel& model, const TrainingConfig& cfg);
TimeNs transfer_time(const Gmap& gmap, const MemOp& op, int k,
                     const PerfModel& model, const PinSet& pins);
std::string perf_model_to_json(const PerfModel& model);
PerfModel perf_model_from_json(const std::string& text, const std::string& origin);

// ---------------------------------------------------------------------------
// Memory optimizer + minibatch tuner (ref: include/swapsched/planner.hpp)
// ---------------------------------------------------------------------------
struct SwapPlan {
  int k_star = 0;
  PinSet pin_set;
  std::vector<TimeNs> t_ready;
  TimeNs predicted_iter_time = 0;
  double predicted_whole_time_s = 0.0;
  Bytes active_area_bytes = 0;
  Bytes pinned_bytes = 0;
  Bytes residual_bytes = 0;
  Bytes fixed_overhead_bytes = 0;
};
struct MemoryCheck {
  bool ok = true;
  std::optional<std::uint32_t> first_violation_seq;
  Bytes peak_bytes = 0;
};
struct ConstraintReport {
  MemoryCheck memory;
  bool stall_ok = true;
  std::vector<int> violating_phases;
  std::vector<TimeNs> slack;
};
std::vector<TimeNs> compute_t_ready(const Gmap& gmap, int k, Bytes budget,
                                    const PinSet& pins, const PerfModel& model,
                                    const std::vector<TimeNs>& compute_times);
MemoryCheck check_memory_constraint(const Gmap& gmap, int k, Bytes budget,
                                    const PinSet& pins);
std::vector<int> check_stall_constraint(const std::vector<TimeNs>& t_ready,
                                        const std::vector<TimeNs>& compute_times);
ConstraintReport build_constraint_report(const Gmap& gmap, int k, Bytes budget,
                                         const PinSet& pins,
                                         const std::vector<TimeNs>& t_ready,
                                         const std::vector<TimeNs>& compute_times);
struct KmaxResult {
  bool trainable = false;
  int k_max = 0;
  std::string reason;
};
KmaxResult max_trainable_minibatch(const Gmap& gmap, const NetworkSpec& net,
                                   const HardwareSpec& hw);
enum class PlanStatus { ok, untrainable, infeasible };
struct PlanResult {
  PlanStatus status = PlanStatus::infeasible;
  std::optional<SwapPlan> plan;
  std::string detail;
};
struct PlannerOptions {
  int step = 1;
  int k_override = 0;
};
struct KEvaluation {
  int k = 0;
  bool memory_feasible = false;
  bool stall_free = false;
  PinSet pins;
  std::vector<TimeNs> t_ready;
  std::vector<int> omega;
  Bytes active_area_bytes = 0;
  Bytes pinned_bytes = 0;
  Bytes resident_peak_bytes = 0;
};
KEvaluation evaluate_minibatch(const Gmap& gmap,
                               const std::vector<PhaseLayer>& phases, int k,
                               const NetworkSpec& net, const HardwareSpec& hw,
                               const PerfModel& model);
PlanResult find_efficiency_optimal_minibatch(const Gmap& gmap,
                                             const std::vector<PhaseLayer>& phases,
                                             const NetworkSpec& net,
                                             const HardwareSpec& hw,
                                             const PerfModel& model,
                                             const TrainingConfig& cfg,
                                             const PlannerOptions& opts = {});
long long adjust_iterations(int k_star, int k_base, long long iters_base);
std::string swap_plan_to_json(const SwapPlan& plan, const Gmap& gmap,
                              const std::vector<TimeNs>& slack);

// ---------------------------------------------------------------------------
// Learning-rate rule (ref: include/swapsched/lr_tuner.hpp)
// ---------------------------------------------------------------------------
struct LrConfig {
  double alpha_base = 0.0;
  double convexity = 0.0;
  double mu = 1.0;
  long long iters_base = 0;
  double q = 1.0;
};
double adapted_learning_rate(const LrConfig& cfg);
double contraction_residual(const LrConfig& cfg, double alpha_star);

// ---------------------------------------------------------------------------
// Three-stream iteration model (ref: include/swapsched/simulator.hpp)
// ---------------------------------------------------------------------------
enum class SimMode { naive, dynamic, resident };
std::string sim_mode_name(SimMode m);
enum class Stream { compute, swap_out, swap_in };
std::string stream_name(Stream s);
enum class EventKind {
  kernel_start,
  kernel_end,
  xfer_start,
  xfer_end,
  alloc,
  free,
  block,
  unblock
};
std::string event_kind_name(EventKind k);
struct SimEvent {
  TimeNs time = 0;
  Stream stream = Stream::compute;
  EventKind kind = EventKind::alloc;
  std::string subject;
  Bytes mem_used_after = 0;
};
struct SimConfig {
  Bytes budget = 0;
  Bytes fixed_overhead = 0;
  SimMode mode = SimMode::naive;
  double bandwidth = 0.0;
  TimeNs alloc_cost = 0;
};
struct SimSummary {
  TimeNs iter_time = 0;
  std::vector<TimeNs> per_phase_stall;
  TimeNs total_stall = 0;
  Bytes peak_mem = 0;
  std::vector<std::pair<TimeNs, Bytes>> mem_timeseries;
  bool oom = false;
  std::string oom_detail;
  std::vector<TimeNs> data_ready;
  std::vector<TimeNs> kernel_start;
  std::vector<TimeNs> kernel_end;
};
struct SimResult {
  std::vector<SimEvent> events;
  SimSummary summary;
};
SimResult simulate_iteration(const Gmap& gmap,
                             const std::vector<PhaseLayer>& phases, int k,
                             const PinSet& pins, const PerfModel& model,
                             const SimConfig& cfg);
struct StallRow {
  int phase = 0;
  TimeNs stall = 0;
};
std::vector<StallRow> stall_report(const SimSummary& summary);
struct Verdict {
  bool pass = false;
  double stall_fraction = 0.0;
  bool memory_ok = false;
  TimeNs max_ready_deviation = 0;
  std::string detail;
};
Verdict verify_plan(const SwapPlan& plan, const SimSummary& summary,
                    Bytes budget, double tolerance);
std::string trace_to_csv(const std::vector<SimEvent>& events);
std::string summary_to_json(const SimSummary& summary);
std::string mem_curves_csv(const std::vector<SimEvent>& events,
                           Bytes fixed_overhead);
std::string stall_bars_csv(const SimSummary& summary);

// ---------------------------------------------------------------------------
// (k x mode) grid (ref: include/swapsched/sweep.hpp)
// ---------------------------------------------------------------------------
struct SweepRow {
  int k = 0;
  SimMode mode = SimMode::naive;
  bool feasible = false;
  TimeNs iter_time = 0;
  double whole_time_s = 0.0;
  Bytes peak_mem = 0;
  TimeNs stall = 0;
  std::string note;
};
std::vector<SweepRow> sweep_grid(const Gmap& gmap,
                                 const std::vector<PhaseLayer>& phases,
                                 const NetworkSpec& net, const HardwareSpec& hw,
                                 const PerfModel& model, const TrainingConfig& cfg,
                                 const std::vector<int>& k_list,
                                 const std::vector<SimMode>& modes,
                                 bool parallel);
std::string sweep_to_csv(const std::vector<SweepRow>& rows);

// ---------------------------------------------------------------------------
// Seeded fixtures (ref: include/swapsched/synthetic.hpp).  The splitmix64
// stream is part of the fixture contract, so it is reproduced exactly.
// ---------------------------------------------------------------------------
struct Rng {
  std::uint64_t state;
  explicit Rng(std::uint64_t seed) : state(seed ? seed : 0x9e3779b97f4a7c15ull) {}
  std::uint64_t next();
  std::int64_t range(std::int64_t lo, std::int64_t hi);
  double uniform(double lo, double hi);
};
struct SyntheticOptions {
  int min_layers = 4;
  int max_layers = 16;
  double min_compute_transfer_ratio = 1.5;
  double max_compute_transfer_ratio = 5.0;
  double bandwidth_lo = 4e9;
  double bandwidth_hi = 16e9;
  double budget_frac_lo = 0.25;
  double budget_frac_hi = 1.1;
};
struct SyntheticInstance {
  NetworkSpec network;
  HardwareSpec hardware;
  ProfileSet profiles;
  double true_bandwidth = 0.0;
};
NetworkSpec generate_network(Rng& rng, const SyntheticOptions& opts = {});
ProfileSet generate_profiles(const NetworkSpec& net, Rng& rng, int k_ref,
                             double bandwidth);
SyntheticInstance generate_instance(std::uint64_t seed,
                                    const SyntheticOptions& opts = {});
std::string compute_profile_csv(const std::vector<ComputeSample>& samples);
std::string transfer_profile_csv(const std::vector<TransferSample>& samples);

}  // namespace swapsched
