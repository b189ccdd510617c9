// (k x mode) analysis grid: `swapsched sweep`.
//
// Behaviour contract: /root/reference/proj/src/sweep.cpp:12-111 and
// include/swapsched/sweep.hpp:12-34 -- one row per (k, mode) cell in
// canonical k-major order, the same infeasibility notes, and parallel ==
// serial bytes (reference test_sweep.cpp:42-53).
//
// Structure (B200 host build): the grid is resolved in two passes.
//   1. pin resolution -- one pin set per *distinct k* (dynamic mode runs the
//      planner's evaluate_minibatch once per k, not once per cell; the
//      resident pin set is built once for the whole grid);
//   2. simulation -- every feasible cell is simulated with its pin set.
// Both passes hand out work items from an atomic cursor to std::threads
// (parallel=true); every item writes only its own slot, so the output does
// not depend on the schedule.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <exception>
#include <optional>
#include <sstream>
#include <thread>

#include "swapsched/api.hpp"

namespace swapsched {
namespace {

// Runs body(i) for i in [0, n) on up to hardware_concurrency threads.
template <class Fn>
void for_each_item(size_t n, bool parallel, Fn&& body) {
  size_t workers = parallel ? std::max(1u, std::thread::hardware_concurrency()) : 1;
  workers = std::min(workers, n);
  if (workers <= 1) {
    for (size_t i = 0; i < n; ++i) body(i);
    return;
  }
  // an exception in an item is re-thrown on the caller (lowest index wins,
  // as the serial loop would have thrown it first)
  std::atomic<size_t> cursor{0};
  std::vector<std::exception_ptr> errors(n);
  auto drain = [&] {
    for (size_t i = cursor++; i < n; i = cursor++) {
      try {
        body(i);
      } catch (...) {
        errors[i] = std::current_exception();
      }
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(workers - 1);
  for (size_t w = 1; w < workers; ++w) pool.emplace_back(drain);
  drain();
  for (auto& t : pool) t.join();
  for (const auto& e : errors)
    if (e) std::rethrow_exception(e);
}

// Outcome of the planner for one k in dynamic mode.
struct DynamicPins {
  std::optional<PinSet> pins;  // engaged when the plan is usable
  const char* note = "";
};

DynamicPins plan_pins(const Gmap& gmap, const std::vector<PhaseLayer>& phases, int k,
                      const NetworkSpec& net, const HardwareSpec& hw,
                      const PerfModel& model) {
  KEvaluation ev = evaluate_minibatch(gmap, phases, k, net, hw, model);
  DynamicPins out;
  if (!ev.memory_feasible)
    out.note = "memory constraint violated";
  else if (!ev.stall_free)
    out.note = "stall constraint not satisfiable";
  else
    out.pins = std::move(ev.pins);
  return out;
}

// Eq. 8 whole-training time of a feasible cell (ref: sweep.cpp:51-58).
double whole_training_seconds(const TrainingConfig& cfg, const HardwareSpec& hw, int k,
                              TimeNs iter_time) {
  const long long dataset = cfg.dataset_size > 0 ? cfg.dataset_size : k;
  const long long iterations = (cfg.epochs * dataset + k - 1) / k;
  return static_cast<double>(iterations) * (to_seconds(iter_time) + hw.delta_sync_s);
}

}  // namespace

std::vector<SweepRow> sweep_grid(const Gmap& gmap,
                                 const std::vector<PhaseLayer>& phases,
                                 const NetworkSpec& net, const HardwareSpec& hw,
                                 const PerfModel& model, const TrainingConfig& cfg,
                                 const std::vector<int>& k_list,
                                 const std::vector<SimMode>& modes,
                                 bool parallel) {
  if (k_list.empty()) throw std::invalid_argument("empty minibatch grid");
  if (modes.empty()) throw std::invalid_argument("no simulation modes given");

  // pass 1: pin sets
  const bool wants_dynamic =
      std::find(modes.begin(), modes.end(), SimMode::dynamic) != modes.end();
  std::vector<int> distinct_k;
  if (wants_dynamic) {
    distinct_k = k_list;
    std::sort(distinct_k.begin(), distinct_k.end());
    distinct_k.erase(std::unique(distinct_k.begin(), distinct_k.end()), distinct_k.end());
  }
  std::vector<DynamicPins> dyn(distinct_k.size());
  for_each_item(distinct_k.size(), parallel, [&](size_t i) {
    dyn[i] = plan_pins(gmap, phases, distinct_k[i], net, hw, model);
  });
  auto dynamic_for = [&](int k) -> const DynamicPins& {
    const auto it = std::lower_bound(distinct_k.begin(), distinct_k.end(), k);
    return dyn[static_cast<size_t>(it - distinct_k.begin())];
  };
  PinSet resident;
  for (ObjectId id : gmap.featuremap_ids()) resident.insert(id);
  const PinSet none;

  // pass 2: simulate every cell (k-major, modes in the given order)
  SimConfig base;
  base.budget = hw.memory_budget;
  base.fixed_overhead = hw.m_others + net.param_grad_bytes_total();
  base.bandwidth = model.bandwidth_avail;

  std::vector<SweepRow> rows(k_list.size() * modes.size());
  for_each_item(rows.size(), parallel, [&](size_t cell) {
    SweepRow& row = rows[cell];
    row.k = k_list[cell / modes.size()];
    row.mode = modes[cell % modes.size()];
    const PinSet* pins = &none;
    if (row.mode == SimMode::resident) {
      pins = &resident;
    } else if (row.mode == SimMode::dynamic) {
      const DynamicPins& d = dynamic_for(row.k);
      if (!d.pins) {
        row.note = d.note;
        return;
      }
      pins = &*d.pins;
    }
    SimConfig sc = base;
    sc.mode = row.mode;
    const SimResult sim = simulate_iteration(gmap, phases, row.k, *pins, model, sc);
    if (sim.summary.oom) {
      row.note = "oom: " + sim.summary.oom_detail;
      return;
    }
    row.feasible = true;
    row.iter_time = sim.summary.iter_time;
    row.peak_mem = sim.summary.peak_mem;
    row.stall = sim.summary.total_stall;
    row.whole_time_s = whole_training_seconds(cfg, hw, row.k, row.iter_time);
  });
  return rows;
}

std::string sweep_to_csv(const std::vector<SweepRow>& rows) {
  std::string out = "k,mode,feasible,iter_time_s,whole_time_s,peak_mem_bytes,stall_s,note\n";
  char line[256];
  for (const SweepRow& r : rows) {
    std::snprintf(line, sizeof line, "%d,%s,%s,%.9f,%.9f,%llu,%.9f,", r.k,
                  sim_mode_name(r.mode).c_str(), r.feasible ? "true" : "false",
                  to_seconds(r.iter_time), r.whole_time_s,
                  static_cast<unsigned long long>(r.peak_mem), to_seconds(r.stall));
    out += line;
    out += r.note;
    out += '\n';
  }
  return out;
}

}  // namespace swapsched
