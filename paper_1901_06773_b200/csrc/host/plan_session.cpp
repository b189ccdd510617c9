// Incremental re-planning: a planning session keeps what the
// planner derives from the network and the fitted throughput curves, so a
// re-plan after the device cap or the host-link bandwidth changed (a new
// hardware.json, a re-measured link) reuses it instead of starting over.
//
// Cached per session: the parsed documents, the unfolded phases and the GMAP
// (model_ir.cpp:87-144, :289-358); per k on first use: the k-scaled object
// sizes, the unpinned running sums and their peak, and the 2N phase compute
// times (planner.cpp:255-270 and perf_model.cpp:112-132 -- none depends on
// the budget or the bandwidth).  Each re-plan runs Algorithm 2
// (planner.cpp:346-424) with the reference's scan order over these, so its
// plan.json is byte-identical to a fresh `swapsched plan` on the changed
// documents (tests/test_planner_parity.py), and a step-16 request is
// answered with the step-1 plan when `exact` is set (the coarse/fine stride
// equals the linear scan only when feasibility is monotone in k,
// planner.cpp:386-407).
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>

#include <json.hpp>

#include "swapsched/api.hpp"
#include "internal.hpp"

using namespace swapsched;
using nlohmann::json;

namespace {

thread_local std::string g_session_error;

struct Session {
  NetworkSpec net;
  HardwareSpec hw;
  PerfModel model;
  std::vector<PhaseLayer> phases;
  Gmap gmap;

  struct Entry {
    std::once_flag st_once, compute_once;
    detail::KStatic st;
    std::vector<TimeNs> compute;
  };
  std::mutex mu;
  std::unordered_map<int, std::unique_ptr<Entry>> cache;
  long long hits = 0, misses = 0;

  Entry& entry(int k) {
    std::lock_guard<std::mutex> lock(mu);
    auto& e = cache[k];
    if (!e) {
      e = std::make_unique<Entry>();
      ++misses;
    } else {
      ++hits;
    }
    return *e;
  }

  KEvaluation evaluate(int k, const HardwareSpec& h, double bandwidth) {
    Entry& e = entry(k);
    std::call_once(e.st_once, [&] { e.st = detail::make_k_static(gmap, phases, k, model); });
    return detail::evaluate_static(gmap, e.st, k, net, h, bandwidth,
                                   [&]() -> const std::vector<TimeNs>& {
                                     std::call_once(e.compute_once, [&] {
                                       e.compute = detail::k_compute_times(gmap, phases, k, model);
                                     });
                                     return e.compute;
                                   });
  }
};

template <typename F>
int session_guarded(F&& body) {
  g_session_error.clear();
  try {
    return body();
  } catch (const IoError& e) {
    g_session_error = e.what();
    return 2;
  } catch (const SpecError& e) {
    g_session_error = e.what();
    return 1;
  } catch (const UntrainableError& e) {
    g_session_error = e.what();
    return 1;
  } catch (const std::invalid_argument& e) {
    g_session_error = e.what();
    return 1;
  } catch (const json::exception& e) {
    g_session_error = std::string("malformed document: ") + e.what();
    return 1;
  } catch (const std::exception& e) {
    g_session_error = std::string("internal error: ") + e.what();
    return 3;
  }
}

char* dup_text(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

}  // namespace

struct accudnn_plan_opts_s {
  int step;
  int k_override;
  long long epochs;
  long long dataset_size;
  unsigned long long budget_override;
};

extern "C" __attribute__((visibility("default"))) const char* accudnn_session_last_error(void) {
  return g_session_error.c_str();
}

extern "C" __attribute__((visibility("default"))) int accudnn_plan_session_create(
    const char* network_json, const char* hardware_json, const char* model_json,
    void** session) {
  return session_guarded([&] {
    if (!network_json || !hardware_json || !model_json || !session)
      throw std::invalid_argument("network, hardware and model documents are required");
    auto s = std::make_unique<Session>();
    s->net = parse_network_spec_json(network_json, "network.json");
    s->hw = parse_hardware_spec_json(hardware_json, "hardware.json");
    s->model = perf_model_from_json(model_json, "model.json");
    s->phases = unfold_network(s->net);
    s->gmap = build_gmap(s->phases, s->net);
    *session = s.release();
    return 0;
  });
}

// One re-plan.  opts as accudnn_plan (budget_override != 0 replaces the
// session's memory_budget_bytes), bandwidth_override > 0 replaces the
// model's bandwidth_avail_bytes_per_s; exact != 0 answers any step with the
// step-1 scan.  Output: plan.json exactly as accudnn_plan writes it for the
// changed documents (status document and rc 1 when infeasible/untrainable).
extern "C" __attribute__((visibility("default"))) int accudnn_plan_session_plan(
    void* session, const accudnn_plan_opts_s* opts, double bandwidth_override, int exact,
    char** plan_json) {
  return session_guarded([&] {
    if (!session) throw std::invalid_argument("null planning session");
    Session& s = *static_cast<Session*>(session);
    accudnn_plan_opts_s o{1, 0, 1, 0, 0};
    if (opts) o = *opts;
    HardwareSpec hw = s.hw;
    if (o.budget_override) hw.memory_budget = o.budget_override;
    PerfModel model = s.model;
    if (bandwidth_override > 0) model.bandwidth_avail = bandwidth_override;
    TrainingConfig cfg;
    cfg.epochs = o.epochs;
    cfg.dataset_size = o.dataset_size;
    cfg.delta_sync_s = hw.delta_sync_s;
    PlannerOptions po;
    po.step = exact ? 1 : o.step;
    po.k_override = o.k_override;
    const double bw = model.bandwidth_avail;
    const PlanResult res = detail::search_plan(
        s.gmap, s.phases, s.net, hw, model, cfg, po,
        [&](int k) { return s.evaluate(k, hw, bw); });
    if (res.status != PlanStatus::ok) {
      json doc;
      doc["format_version"] = 1;
      doc["status"] = res.status == PlanStatus::untrainable ? "untrainable" : "infeasible";
      doc["detail"] = res.detail;
      if (plan_json) *plan_json = dup_text(doc.dump(2) + "\n");
      g_session_error = doc["status"].get<std::string>() + ": " + res.detail;
      return 1;
    }
    const SwapPlan& plan = *res.plan;
    Session::Entry& e = s.entry(plan.k_star);
    std::call_once(e.compute_once, [&] {
      e.compute = detail::k_compute_times(s.gmap, s.phases, plan.k_star, s.model);
    });
    const ConstraintReport rep = build_constraint_report(s.gmap, plan.k_star, hw.memory_budget,
                                                         plan.pin_set, plan.t_ready, e.compute);
    if (plan_json) *plan_json = dup_text(swap_plan_to_json(plan, s.gmap, rep.slack));
    return 0;
  });
}

// per-k cache statistics of the session: evaluations served from the cache
// and evaluations that built a cache entry
extern "C" __attribute__((visibility("default"))) int accudnn_plan_session_stats(
    void* session, long long* hits, long long* misses) {
  if (!session) return 1;
  Session& s = *static_cast<Session*>(session);
  std::lock_guard<std::mutex> lock(s.mu);
  if (hits) *hits = s.hits;
  if (misses) *misses = s.misses;
  return 0;
}

extern "C" __attribute__((visibility("default"))) void accudnn_plan_session_destroy(void* session) {
  delete static_cast<Session*>(session);
}
