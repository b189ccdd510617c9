// C ABI over the swapsched host API (see include/accudnn_plan.h).
//
// This translation unit only uses the public swapsched C++ API, so the
// parity harness compiles the very same glue against the reference sources
// (oracle/Makefile, -DACCUDNN_ABI_PREFIX=oracle_) and both libraries answer
// identical document-level calls.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "swapsched/lr_tuner.hpp"
#include "swapsched/model_ir.hpp"
#include "swapsched/perf_model.hpp"
#include "swapsched/planner.hpp"
#include "swapsched/profiles.hpp"
#include "swapsched/simulator.hpp"
#include "swapsched/sweep.hpp"
#include "swapsched/synthetic.hpp"
#include "swapsched/types.hpp"

#ifndef ACCUDNN_ABI_PREFIX
#define ACCUDNN_ABI_PREFIX accudnn_
#endif
#define ABI_CAT2(a, b) a##b
#define ABI_CAT(a, b) ABI_CAT2(a, b)
#define ABI(name) ABI_CAT(ACCUDNN_ABI_PREFIX, name)
#define ABI_EXPORT extern "C" __attribute__((visibility("default")))

using namespace swapsched;
using nlohmann::json;

namespace {

thread_local std::string g_last_error;

char* dup_out(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}
void put(char** dst, const std::string& s) {
  if (dst) *dst = dup_out(s);
}

// exception -> CLI exit code (ref: tools/swapsched.cpp:654-672)
template <typename F>
int guarded(F&& body) {
  g_last_error.clear();
  try {
    return body();
  } catch (const IoError& e) {
    g_last_error = e.what();
    return 2;
  } catch (const SpecError& e) {
    g_last_error = e.what();
    return 1;
  } catch (const UntrainableError& e) {
    g_last_error = e.what();
    return 1;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return 1;
  } catch (const json::exception& e) {
    g_last_error = std::string("malformed document: ") + e.what();
    return 1;
  } catch (const std::exception& e) {
    g_last_error = std::string("internal error: ") + e.what();
    return 3;
  } catch (...) {
    g_last_error = "internal error: unknown exception";
    return 3;
  }
}

struct Loaded {
  NetworkSpec net;
  std::vector<PhaseLayer> phases;
  Gmap gmap;
  HardwareSpec hw;
  PerfModel model;
};

Loaded load(const char* net_json, const char* hw_json, const char* model_json,
            unsigned long long budget_override = 0) {
  if (!net_json || !hw_json || !model_json)
    throw std::invalid_argument("network, hardware and model documents are required");
  Loaded L;
  L.net = parse_network_spec_json(net_json, "network.json");
  L.hw = parse_hardware_spec_json(hw_json, "hardware.json");
  if (budget_override) L.hw.memory_budget = budget_override;
  L.model = perf_model_from_json(model_json, "model.json");
  L.phases = unfold_network(L.net);
  L.gmap = build_gmap(L.phases, L.net);
  return L;
}

json ns_array(const std::vector<TimeNs>& v) {
  json a = json::array();
  for (TimeNs t : v) a.push_back(t);
  return a;
}

SimMode mode_from(const std::string& name) {
  if (name == "naive") return SimMode::naive;
  if (name == "dynamic") return SimMode::dynamic;
  if (name == "resident") return SimMode::resident;
  throw SpecError("unknown mode '" + name + "'");
}

}  // namespace

ABI_EXPORT const char* ABI(last_error)(void) { return g_last_error.c_str(); }

ABI_EXPORT void ABI(free)(void* p) { std::free(p); }

ABI_EXPORT int ABI(validate)(const char* network_json, char** report) {
  return guarded([&] {
    if (!network_json) throw std::invalid_argument("network document required");
    const NetworkSpec net = parse_network_spec_json(network_json, "network.json");
    const Gmap g = build_gmap(unfold_network(net), net);
    const auto diags = validate_gmap(g);
    std::string text;
    for (const auto& d : diags) text += "diagnostic: " + d + "\n";
    if (diags.empty())
      text = "ok: " + net.name + " (" + std::to_string(net.num_layers) + " layers, " +
             std::to_string(g.ops.size()) + " memory ops)\n";
    put(report, text);
    return diags.empty() ? 0 : 1;
  });
}

ABI_EXPORT int ABI(fit)(const char* network_json, const char* const* profile_csvs,
                        int n_profiles, const char* hardware_json, double eta,
                        char** model_json) {
  return guarded([&] {
    if (!network_json) throw std::invalid_argument("network document required");
    if (n_profiles <= 0 || !profile_csvs) throw SpecError("no profile files given");
    const NetworkSpec net = parse_network_spec_json(network_json, "network.json");
    double fallback = 0.0;
    if (hardware_json)
      fallback = parse_hardware_spec_json(hardware_json, "hardware.json").pcie_nominal;
    // merge in argument order (ref: profiles.cpp:156-172)
    ProfileSet all;
    for (int i = 0; i < n_profiles; ++i) {
      ProfileSet one = parse_profile_csv(profile_csvs[i],
                                         "profile" + std::to_string(i) + ".csv");
      all.compute_samples.insert(all.compute_samples.end(), one.compute_samples.begin(),
                                 one.compute_samples.end());
      all.transfer_samples.insert(all.transfer_samples.end(),
                                  one.transfer_samples.begin(), one.transfer_samples.end());
      all.sampled_minibatches.insert(one.sampled_minibatches.begin(),
                                     one.sampled_minibatches.end());
    }
    const PerfModel model = build_perf_model(all, net.k_base, eta, fallback);
    for (const PhaseLayer& p : unfold_network(net)) model.curve_for(p.type_key);
    put(model_json, perf_model_to_json(model));
    return 0;
  });
}

ABI_EXPORT int ABI(kmax)(const char* network_json, const char* hardware_json,
                         int* k_max) {
  return guarded([&] {
    if (!network_json || !hardware_json)
      throw std::invalid_argument("network and hardware documents required");
    const NetworkSpec net = parse_network_spec_json(network_json, "network.json");
    const HardwareSpec hw = parse_hardware_spec_json(hardware_json, "hardware.json");
    const Gmap g = build_gmap(unfold_network(net), net);
    const KmaxResult r = max_trainable_minibatch(g, net, hw);
    if (k_max) *k_max = r.trainable ? r.k_max : 0;
    if (!r.trainable) g_last_error = r.reason;
    return r.trainable ? 0 : 1;
  });
}

// accudnn_plan_opts mirrors include/accudnn_plan.h; restated here so the
// glue compiles against either implementation without that header.
struct accudnn_plan_opts_t {
  int step;
  int k_override;
  long long epochs;
  long long dataset_size;
  unsigned long long budget_override;
};

ABI_EXPORT int ABI(plan)(const char* network_json, const char* hardware_json,
                         const char* model_json, const accudnn_plan_opts_t* opts,
                         char** plan_json) {
  return guarded([&] {
    accudnn_plan_opts_t o{1, 0, 1, 0, 0};
    if (opts) o = *opts;
    const Loaded L = load(network_json, hardware_json, model_json, o.budget_override);
    TrainingConfig cfg;
    cfg.epochs = o.epochs;
    cfg.dataset_size = o.dataset_size;
    cfg.delta_sync_s = L.hw.delta_sync_s;
    PlannerOptions po;
    po.step = o.step;
    po.k_override = o.k_override;
    const PlanResult res = find_efficiency_optimal_minibatch(L.gmap, L.phases, L.net,
                                                             L.hw, L.model, cfg, po);
    if (res.status != PlanStatus::ok) {
      json doc;
      doc["format_version"] = 1;
      doc["status"] = res.status == PlanStatus::untrainable ? "untrainable" : "infeasible";
      doc["detail"] = res.detail;
      put(plan_json, doc.dump(2) + "\n");
      g_last_error = doc["status"].get<std::string>() + ": " + res.detail;
      return 1;
    }
    const SwapPlan& plan = *res.plan;
    const auto compute = phase_compute_times(L.phases, plan.k_star, L.model);
    const ConstraintReport rep = build_constraint_report(
        L.gmap, plan.k_star, L.hw.memory_budget, plan.pin_set, plan.t_ready, compute);
    put(plan_json, swap_plan_to_json(plan, L.gmap, rep.slack));
    return 0;
  });
}

// the perf model's 2N phase compute times at k (perf_model.cpp:112-132),
// one "phase,time_ns" row per phase
ABI_EXPORT int ABI(phase_times)(const char* network_json, const char* model_json, int k,
                                char** times_csv) {
  return guarded([&] {
    if (!network_json || !model_json) throw std::invalid_argument("network and model required");
    const NetworkSpec net = parse_network_spec_json(network_json, "network.json");
    const PerfModel model = perf_model_from_json(model_json, "model.json");
    const auto phases = unfold_network(net);
    const auto t = phase_compute_times(phases, k, model);
    std::string out = "phase,time_ns\n";
    for (size_t j = 0; j < t.size(); ++j)
      out += std::to_string(j + 1) + "," + std::to_string(static_cast<long long>(t[j])) + "\n";
    put(times_csv, out);
    return 0;
  });
}

ABI_EXPORT int ABI(evaluate_k)(const char* network_json, const char* hardware_json,
                               const char* model_json, int k, char** eval_json) {
  return guarded([&] {
    const Loaded L = load(network_json, hardware_json, model_json);
    const KEvaluation ev = evaluate_minibatch(L.gmap, L.phases, k, L.net, L.hw, L.model);
    json doc;
    doc["k"] = ev.k;
    doc["memory_feasible"] = ev.memory_feasible;
    doc["stall_free"] = ev.stall_free;
    json pins = json::array();
    for (ObjectId id : ev.pins) pins.push_back(L.gmap.object(id).name);
    doc["pinned_objects"] = std::move(pins);
    doc["t_ready_ns"] = ns_array(ev.t_ready);
    doc["omega"] = ev.omega;
    doc["active_area_bytes"] = ev.active_area_bytes;
    doc["pinned_bytes"] = ev.pinned_bytes;
    doc["resident_peak_bytes"] = ev.resident_peak_bytes;
    put(eval_json, doc.dump() + "\n");
    return 0;
  });
}

namespace {

// One `swapsched simulate` run (ref: tools/swapsched.cpp:300-383): the
// outputs write_sim_outputs produces (swapsched.cpp:162-170) plus, with a
// plan, the verify_plan verdict document.  rc 1: deadlock or failed verdict.
struct SimRun {
  std::string summary, trace, mem_curves, stall_bars, verify;
  bool oom = false;
  int rc = 0;
};

SimRun simulate_run(const char* network_json, const char* hardware_json,
                    const char* model_json, const char* plan_json, const char* mode, int k,
                    unsigned long long budget_override, double tolerance) {
  const Loaded L = load(network_json, hardware_json, model_json, budget_override);
  const SimMode m = mode_from(mode ? mode : "naive");
  PinSet pins;
  std::optional<SwapPlan> plan;
  if (m == SimMode::dynamic) {
    if (!plan_json) throw SpecError("dynamic mode needs a plan");
    const json pj = json::parse(plan_json);
    SwapPlan p;
    p.k_star = pj.at("k_star").get<int>();
    for (const auto& name : pj.at("pinned_objects").get<std::vector<std::string>>()) {
      const auto it = std::find_if(L.gmap.objects.begin(), L.gmap.objects.end(),
                                   [&](const MemObject& o) { return o.name == name; });
      if (it == L.gmap.objects.end())
        throw SpecError("plan pins unknown object '" + name + "'");
      pins.insert(it->id);
    }
    p.pin_set = pins;
    for (double t : pj.at("t_ready_s").get<std::vector<double>>())
      p.t_ready.push_back(from_seconds(t));
    p.predicted_iter_time = from_seconds(pj.at("predicted_iter_time_s").get<double>());
    plan = std::move(p);
    if (k <= 0) k = plan->k_star;
  } else if (m == SimMode::resident) {
    for (ObjectId id : L.gmap.featuremap_ids()) pins.insert(id);
  }
  if (k <= 0) throw SpecError("k is required outside dynamic mode");
  SimConfig cfg;
  cfg.budget = L.hw.memory_budget;
  cfg.fixed_overhead = L.hw.m_others + L.net.param_grad_bytes_total();
  cfg.mode = m;
  cfg.bandwidth = L.model.bandwidth_avail;
  const SimResult sim = simulate_iteration(L.gmap, L.phases, k, pins, L.model, cfg);
  SimRun r;
  r.summary = summary_to_json(sim.summary);
  r.trace = trace_to_csv(sim.events);
  r.mem_curves = mem_curves_csv(sim.events, cfg.fixed_overhead);
  r.stall_bars = stall_bars_csv(sim.summary);
  if (sim.summary.oom) {
    g_last_error = "oom: " + sim.summary.oom_detail;
    r.oom = true;
    r.rc = 1;
    return r;
  }
  if (plan) {
    const Verdict v = verify_plan(*plan, sim.summary, cfg.budget, tolerance);
    json vj;
    vj["format_version"] = 1;
    vj["pass"] = v.pass;
    vj["stall_fraction"] = v.stall_fraction;
    vj["memory_ok"] = v.memory_ok;
    vj["max_ready_deviation_s"] = to_seconds(v.max_ready_deviation);
    r.verify = vj.dump(2);
    if (!v.pass) {
      g_last_error = "verify: fail (" + v.detail + ")";
      r.rc = 1;
    }
  }
  return r;
}

}  // namespace

ABI_EXPORT int ABI(simulate)(const char* network_json, const char* hardware_json,
                             const char* model_json, const char* plan_json,
                             const char* mode, int k, char** summary_json,
                             char** trace_csv) {
  return guarded([&] {
    const SimRun r = simulate_run(network_json, hardware_json, model_json, plan_json, mode, k,
                                  0, 0.02);
    put(summary_json, r.summary);
    put(trace_csv, r.trace);
    // the verdict is not part of this entry point's contract
    if (!r.oom) g_last_error.clear();
    return r.oom ? 1 : 0;
  });
}

ABI_EXPORT int ABI(simulate_report)(const char* network_json, const char* hardware_json,
                                    const char* model_json, const char* plan_json,
                                    const char* mode, int k,
                                    unsigned long long budget_override, double tolerance,
                                    char** summary_json, char** trace_csv,
                                    char** mem_curves_csv_out, char** stall_bars_csv_out,
                                    char** verify_json) {
  return guarded([&] {
    const SimRun r = simulate_run(network_json, hardware_json, model_json, plan_json, mode, k,
                                  budget_override, tolerance);
    put(summary_json, r.summary);
    put(trace_csv, r.trace);
    put(mem_curves_csv_out, r.mem_curves);
    put(stall_bars_csv_out, r.stall_bars);
    put(verify_json, r.verify);
    return r.rc;
  });
}

// with_digest (ref: tools/swapsched.cpp:114-118): the document re-serialised
// by the JSON library with "manifest_digest" added, indent 2, newline.
ABI_EXPORT int ABI(with_digest)(const char* doc, const char* digest, char** out) {
  return guarded([&] {
    json j = json::parse(doc ? doc : "");
    j["manifest_digest"] = digest ? digest : "";
    put(out, j.dump(2) + "\n");
    return 0;
  });
}

ABI_EXPORT int ABI(sweep)(const char* network_json, const char* hardware_json,
                          const char* model_json, const int* k_list, int n_k,
                          const char* modes_csv, int parallel, char** sweep_csv) {
  return guarded([&] {
    const Loaded L = load(network_json, hardware_json, model_json);
    std::vector<int> ks(k_list, k_list + (n_k > 0 ? n_k : 0));
    std::vector<SimMode> modes;
    std::stringstream ss(modes_csv ? modes_csv : "naive,dynamic,resident");
    std::string tok;
    while (std::getline(ss, tok, ',')) modes.push_back(mode_from(tok));
    TrainingConfig cfg;
    cfg.delta_sync_s = L.hw.delta_sync_s;
    const auto rows = sweep_grid(L.gmap, L.phases, L.net, L.hw, L.model, cfg, ks, modes,
                                 parallel != 0);
    put(sweep_csv, sweep_to_csv(rows));
    return 0;
  });
}

ABI_EXPORT int ABI(tune_lr)(double alpha_base, double convexity, double mu, double q,
                            long long iters_base, double* alpha_star, double* residual,
                            long long* adjusted_iterations) {
  return guarded([&] {
    LrConfig c;
    c.alpha_base = alpha_base;
    c.convexity = convexity;
    c.mu = mu;
    c.q = q;
    c.iters_base = iters_base;
    const double a = adapted_learning_rate(c);
    if (alpha_star) *alpha_star = a;
    if (residual) *residual = contraction_residual(c, a);
    // the CLI reports ceil(iters_base / q) in floating point
    // (ref: swapsched.cpp:432-433)
    if (adjusted_iterations)
      *adjusted_iterations =
          static_cast<long long>(std::ceil(static_cast<double>(iters_base) / q));
    return 0;
  });
}

ABI_EXPORT int ABI(generate_fixture)(unsigned long long seed, int min_layers,
                                     int max_layers, char** network_json,
                                     char** hardware_json, char** compute_csv,
                                     char** transfer_csv) {
  return guarded([&] {
    SyntheticOptions o;
    if (min_layers > 0) o.min_layers = min_layers;
    if (max_layers > 0) o.max_layers = std::max(max_layers, o.min_layers);
    const SyntheticInstance inst = generate_instance(seed, o);
    put(network_json, network_spec_to_json(inst.network));
    put(hardware_json, hardware_spec_to_json(inst.hardware));
    put(compute_csv, compute_profile_csv(inst.profiles.compute_samples));
    put(transfer_csv, transfer_profile_csv(inst.profiles.transfer_samples));
    return 0;
  });
}
