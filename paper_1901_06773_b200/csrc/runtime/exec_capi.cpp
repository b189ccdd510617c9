// C ABI of the executor (include/accudnn.h).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include <json.hpp>

#include "accudnn.h"
#include "executor.h"
#include "swapsched/api.hpp"
#include "net.h"

using nlohmann::json;

struct accudnn_exec {
  std::unique_ptr<accudnn::Executor> ex;
};

namespace {

thread_local std::string g_err;

char* dup_out(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

template <typename F>
int guarded(F&& f) {
  g_err.clear();
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const json::exception& e) {
    g_err = std::string("malformed document: ") + e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// The executor's real timeline as the reference simulator's event list
// (simulator.hpp SimEvent / SimSummary): kernel_start / kernel_end per phase
// on the compute stream, xfer_start / xfer_end per copy on the swap streams,
// mem_used_after = fixed + the live instance bytes of the phase the event
// falls in; ordered by (time, stream) as simulator.cpp:56-75 orders equal
// times.  Serialised by the same functions as the simulated documents
// (simulator.cpp:419-473), so simulated and real timelines diff directly.
struct RealDocs {
  std::vector<swapsched::SimEvent> events;
  swapsched::SimSummary summary;
};

RealDocs real_docs(const accudnn::RealTimeline& tl) {
  using swapsched::EventKind;
  using swapsched::Stream;
  RealDocs d;
  const size_t P = tl.kstart.size();
  auto mem_at = [&](long long t) -> unsigned long long {
    // the last phase that started at or before t
    size_t j = static_cast<size_t>(std::upper_bound(tl.kstart.begin(), tl.kstart.end(), t) -
                                   tl.kstart.begin());
    if (j > 0) --j;
    return P ? static_cast<unsigned long long>(tl.mem_at_phase[j]) : tl.fixed;
  };
  struct Ev {
    long long t;
    int stream;
    size_t seq;
    swapsched::SimEvent e;
  };
  std::vector<Ev> ev;
  auto add = [&](long long t, Stream st, EventKind k, std::string subject) {
    swapsched::SimEvent e;
    e.time = t;
    e.stream = st;
    e.kind = k;
    e.subject = std::move(subject);
    e.mem_used_after = mem_at(t);
    ev.push_back({t, static_cast<int>(st), ev.size(), std::move(e)});
  };
  for (size_t j = 0; j < P; ++j) {
    add(tl.kstart[j], Stream::compute, EventKind::kernel_start, "phase " + std::to_string(j + 1));
    add(tl.kend[j], Stream::compute, EventKind::kernel_end, "phase " + std::to_string(j + 1));
  }
  for (const auto& c : tl.copies) {
    const Stream st = c.stream == 1 ? Stream::swap_out : Stream::swap_in;
    const std::string name = "fm" + std::to_string(c.tensor + 1);
    add(c.start, st, EventKind::xfer_start, name);
    add(c.end, st, EventKind::xfer_end, name);
  }
  std::stable_sort(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) {
    if (a.t != b.t) return a.t < b.t;
    if (a.stream != b.stream) return a.stream < b.stream;
    return a.seq < b.seq;
  });
  for (auto& e : ev) d.events.push_back(std::move(e.e));
  auto& s = d.summary;
  s.kernel_start.assign(tl.kstart.begin(), tl.kstart.end());
  s.kernel_end.assign(tl.kend.begin(), tl.kend.end());
  s.per_phase_stall.assign(P, 0);
  long long prev = 0;
  for (size_t j = 0; j < P; ++j) {
    s.per_phase_stall[j] = std::max(0LL, tl.kstart[j] - prev);
    prev = tl.kend[j];
    s.total_stall += s.per_phase_stall[j];
  }
  s.iter_time = P ? tl.kend.back() : 0;
  s.peak_mem = tl.fixed;
  for (long long m : tl.mem_at_phase) s.peak_mem = std::max<unsigned long long>(s.peak_mem, m);
  return d;
}

}  // namespace

extern "C" {

const char* accudnn_rt_last_error(void) { return g_err.c_str(); }
void accudnn_rt_free(void* p) { std::free(p); }

int accudnn_net_export(const char* arch, int image, int classes, int k_base, int lookahead,
                       char** network_json, char** describe_json) {
  return guarded([&] {
    const accudnn::Net net = accudnn::build_net(arch, image, classes);
    if (network_json) *network_json = dup_out(accudnn::export_network_json(net, k_base, lookahead));
    if (describe_json) *describe_json = dup_out(accudnn::describe_net_json(net));
    return 0;
  });
}

int accudnn_net_memory(const char* arch, int image, int classes, int k, int lookahead,
                       const char* swapped_mask, long long* live_peak, long long* arena_bytes) {
  return guarded([&] {
    const accudnn::Net net = accudnn::build_net(arch, image, classes);
    std::vector<char> sw(static_cast<size_t>(net.num_ops()), 0);
    if (swapped_mask)
      for (int i = 0; i < net.num_ops(); ++i) sw[static_cast<size_t>(i)] = swapped_mask[i] != 0;
    accudnn::LifetimeModel lm = accudnn::build_lifetimes(net, k, sw, lookahead, 512);
    if (live_peak) *live_peak = lm.peak_bytes;
    const long long arena = accudnn::plan_arena(lm);
    if (arena_bytes) *arena_bytes = arena;
    return 0;
  });
}

int accudnn_exec_create(const char* arch, int image, int classes, const char* mode,
                        const char* network_json, const char* hardware_json,
                        const char* plan_json, int k, int device, int lookahead,
                        accudnn_exec** out) {
  return guarded([&] {
    accudnn::ExecConfig cfg;
    cfg.arch = arch;
    cfg.image = image;
    cfg.classes = classes;
    cfg.device = device;
    cfg.lookahead = lookahead;
    // ACCUDNN_WGRAD_STREAM=0: weight gradients in line on the compute stream
    if (const char* e = std::getenv("ACCUDNN_WGRAD_STREAM")) cfg.wgrad_stream = std::atoi(e);
    if (const char* e = std::getenv("ACCUDNN_STREAM_PRIO")) cfg.stream_priority = std::atoi(e);
    if (const char* e = std::getenv("ACCUDNN_SIDE_CTAS")) cfg.side_ctas = std::atoi(e);
    if (const char* e = std::getenv("ACCUDNN_OVERLAP_UPDATE")) cfg.overlap_update = std::atoi(e);
    if (const char* e = std::getenv("ACCUDNN_CONV_BN_STATS")) cfg.conv_bn_stats = std::atoi(e);
    if (const char* e = std::getenv("ACCUDNN_SIDE_WS_FRAC")) cfg.side_ws_frac = std::atof(e);
    if (const char* e = std::getenv("ACCUDNN_KCOPY_D2H")) cfg.kernel_copy_max_d2h = std::strtoull(e, nullptr, 10);
    if (const char* e = std::getenv("ACCUDNN_KCOPY_H2D")) cfg.kernel_copy_max_h2d = std::strtoull(e, nullptr, 10);
    if (const char* e = std::getenv("ACCUDNN_KCOPY_CTAS")) cfg.kernel_copy_ctas = std::atoi(e);
    // ACCUDNN_PREFETCH=lookahead: fixed-lookahead swap-in instead of the queue
    if (const char* e = std::getenv("ACCUDNN_PREFETCH"))
      cfg.prefetch_queue = std::string(e) == "lookahead" ? 0 : 1;
    const accudnn::Net net = accudnn::build_net(arch, image, classes);
    const int n = net.num_ops();
    const std::string m = mode ? mode : "resident";
    std::vector<char> swapped(static_cast<size_t>(n), 0);
    if (m == "naive") {
      swapped.assign(static_cast<size_t>(n), 1);
    } else if (m == "dynamic") {
      if (!plan_json) throw std::invalid_argument("dynamic mode needs a plan");
      const json plan = json::parse(plan_json);
      if (k <= 0) k = plan.at("k_star").get<int>();
      swapped.assign(static_cast<size_t>(n), 1);
      for (const auto& name : plan.at("pinned_objects")) {
        const std::string s = name.get<std::string>();
        if (s.rfind("fm", 0) != 0) throw std::invalid_argument("plan pins a non-featuremap: " + s);
        const int layer = std::atoi(s.c_str() + 2);
        if (layer < 1 || layer > n) throw std::invalid_argument("plan pins unknown object " + s);
        swapped[static_cast<size_t>(layer - 1)] = 0;
      }
    } else if (m != "resident") {
      throw std::invalid_argument("unknown mode '" + m + "'");
    }
    if (k <= 0) throw std::invalid_argument("k must be positive");
    cfg.k = k;
    if (hardware_json) {
      const json hw = json::parse(hardware_json);
      cfg.budget = hw.at("memory_budget_bytes").get<unsigned long long>();
      unsigned long long pg = 0;
      if (network_json) {
        const json nj = json::parse(network_json);
        for (const auto& l : nj.at("layers"))
          pg += l.at("param_bytes").get<unsigned long long>() +
                l.at("grad_bytes").get<unsigned long long>();
      }
      cfg.fixed_allowance = hw.at("m_others_bytes").get<unsigned long long>() + pg;
      if (!network_json) cfg.fixed_allowance = 0;
    }
    auto h = std::make_unique<accudnn_exec>();
    h->ex = std::make_unique<accudnn::Executor>(cfg, swapped);
    *out = h.release();
    return 0;
  });
}

int accudnn_exec_destroy(accudnn_exec* ex) {
  return guarded([&] {
    delete ex;
    return 0;
  });
}

long long accudnn_exec_num_params(accudnn_exec* ex) { return ex ? ex->ex->net().n_params : -1; }
long long accudnn_exec_num_stats(accudnn_exec* ex) { return ex ? ex->ex->net().n_stats : -1; }

int accudnn_exec_set_params(accudnn_exec* ex, const float* host, long long n) {
  return guarded([&] {
    ex->ex->set_params(host, n);
    return 0;
  });
}
int accudnn_exec_get_params(accudnn_exec* ex, float* host, long long n) {
  return guarded([&] {
    ex->ex->get_params(host, n);
    return 0;
  });
}
int accudnn_exec_get_grads(accudnn_exec* ex, float* host, long long n) {
  return guarded([&] {
    ex->ex->get_grads(host, n);
    return 0;
  });
}
int accudnn_exec_get_stats(accudnn_exec* ex, float* host, long long n) {
  return guarded([&] {
    ex->ex->get_stats(host, n);
    return 0;
  });
}
int accudnn_exec_set_graph(accudnn_exec* ex, int enable) {
  ex->ex->use_graph = enable != 0;
  return 0;
}

int accudnn_exec_step(accudnn_exec* ex, const float* images, const int* labels, int host_inputs,
                      float lr, int update, int profile, accudnn_step_stats* out) {
  return guarded([&] {
    const accudnn::StepStats s = ex->ex->step(images, labels, host_inputs, lr, update, profile);
    if (out) {
      out->loss = s.loss;
      out->iter_ms = s.iter_ms;
      out->exposed_swap_ms = s.exposed_swap_ms;
      out->allreduce_ms = s.allreduce_ms;
      out->peak_bytes = s.peak_bytes;
      out->swapped_bytes = s.swapped_bytes;
      out->exposed_allreduce_ms = s.exposed_allreduce_ms;
    }
    return 0;
  });
}

int accudnn_exec_step_pipelined(accudnn_exec* ex, const float* images, const int* labels,
                                float lr, int update, const float* next_images,
                                accudnn_step_stats* out) {
  return guarded([&] {
    const accudnn::StepStats s = ex->ex->step(images, labels, 1, lr, update, 0, next_images);
    if (out) {
      out->loss = s.loss;
      out->iter_ms = s.iter_ms;
      out->exposed_swap_ms = s.exposed_swap_ms;
      out->allreduce_ms = s.allreduce_ms;
      out->peak_bytes = s.peak_bytes;
      out->swapped_bytes = s.swapped_bytes;
      out->exposed_allreduce_ms = s.exposed_allreduce_ms;
    }
    return 0;
  });
}

int accudnn_exec_memory(accudnn_exec* ex, unsigned long long* arena, unsigned long long* fixed) {
  if (arena) *arena = ex->ex->arena_bytes();
  if (fixed) *fixed = ex->ex->fixed_bytes();
  return 0;
}

int accudnn_exec_launches(accudnn_exec* ex) { return ex->ex->graph_launches(); }

int accudnn_exec_trace(accudnn_exec* ex, char** csv) {
  return guarded([&] {
    *csv = dup_out(ex->ex->trace_csv());
    return 0;
  });
}

int accudnn_exec_document(accudnn_exec* ex, const char* which, char** out) {
  return guarded([&] {
    const std::string w = which ? which : "";
    if (w == "order") {
      std::string o;
      for (const auto& line : ex->ex->copy_order()) o += line + "\n";
      *out = dup_out(o);
      return 0;
    }
    const RealDocs d = real_docs(ex->ex->timeline());
    if (w == "trace")
      *out = dup_out(swapsched::trace_to_csv(d.events));
    else if (w == "mem_curves")
      *out = dup_out(swapsched::mem_curves_csv(d.events, ex->ex->timeline().fixed));
    else if (w == "stall_bars")
      *out = dup_out(swapsched::stall_bars_csv(d.summary));
    else if (w == "summary")
      *out = dup_out(swapsched::summary_to_json(d.summary));
    else
      throw std::invalid_argument("unknown document '" + w + "'");
    return 0;
  });
}

int accudnn_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return 3;
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

int accudnn_exec_set_comm(accudnn_exec* ex, const void* uid128, int rank, int world) {
  return guarded([&] {
    ex->ex->set_comm(uid128, rank, world);
    return 0;
  });
}

unsigned long long accudnn_exec_comm_bytes(accudnn_exec* ex) { return ex ? ex->ex->comm_bytes() : 0; }

}  // extern "C"
