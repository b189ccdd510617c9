// Memory optimizer and minibatch tuner: Algorithm 1 (t_ready), Eq. 4/6
// checks, k_max, the per-k greedy pinning round and Algorithm 2.
//
// Decisions are bit-identical to /root/reference/proj/src/planner.cpp; the
// speed comes from three restatements that do not change any result:
//   * the greedy admission test "layer-wise peak with pins+{c} <= available"
//     (planner.cpp:303-312, a full GMAP traversal per candidate in the
//     reference) is a lazy segment tree over the op-indexed running sums:
//     pinning c adds +size(c) to every prefix from its offload op and
//     -size(c) from its prefetch op, so the peak is the root maximum;
//   * the blocked-allocation scan of Algorithm 1 (planner.cpp:139-148) is a
//     lower_bound over the non-decreasing free prefix;
//   * the k search (planner.cpp:376-408) evaluates waves of k values on all
//     host cores and takes the first feasible k in the reference's scan
//     order (evaluation is pure, so the answer is order-independent).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <exception>
#include <functional>
#include <numeric>

#include <thread>

#include <json.hpp>

#include "swapsched/api.hpp"
#include "internal.hpp"

namespace swapsched {

using nlohmann::json;

namespace {

Bytes fixed_overhead(const NetworkSpec& net, const HardwareSpec& hw) {
  return hw.m_others + net.param_grad_bytes_total();
}

// --- Algorithm 1 -----------------------------------------------------------
// ref: planner.cpp:34-158.  `sizes` are the k-scaled object sizes and
// `pinned` the pin mask; `compute` holds the 2N phase durations.
std::vector<TimeNs> ready_times(const Gmap& g, const std::vector<Bytes>& sizes,
                                const std::vector<char>& pinned, Bytes budget,
                                double bandwidth,
                                const std::vector<TimeNs>& compute) {
  const int phases = g.num_phases;
  const size_t P = static_cast<size_t>(phases);

  std::vector<TimeNs> cum(P + 1, 0);  // cum[j] = end of phase j's compute
  for (size_t j = 1; j <= P; ++j) cum[j] = cum[j - 1] + compute[j - 1];

  // swap-out stream: every byte-freeing op in GMAP order.  Offloads of
  // unpinned objects occupy the D2H channel; releases free at kernel end or
  // behind the transfer still draining.
  std::vector<TimeNs> free_at;
  std::vector<std::int64_t> free_prefix{0};
  std::vector<TimeNs> offload_end(g.objects.size(), 0);
  std::vector<char> offloaded(g.objects.size(), 0);
  free_at.reserve(g.ops.size());
  free_prefix.reserve(g.ops.size() + 1);
  TimeNs cursor = 0;
  for (const MemOp& op : g.ops) {
    if (op.kind != MemOpKind::offload && op.kind != MemOpKind::release) continue;
    const bool pin = pinned[op.object] != 0;
    if (op.kind == MemOpKind::offload && pin) continue;
    const Bytes sz = sizes[op.object];
    cursor = std::max(cursor, cum[static_cast<size_t>(op.phase)]);
    if (op.kind == MemOpKind::offload) {
      cursor += transfer_duration(sz, bandwidth);
      offloaded[op.object] = 1;
      offload_end[op.object] = cursor;
    }
    free_at.push_back(cursor);
    free_prefix.push_back(free_prefix.back() + static_cast<std::int64_t>(sz));
  }

  // swap-in stream: claims (allocations + unpinned prefetches) per phase and
  // the prefetch transfers in GMAP order
  struct Fetch {
    TimeNs duration;
    TimeNs earliest;
  };
  std::vector<std::int64_t> claim(P + 1, 0);
  std::vector<std::vector<Fetch>> fetches(P + 1);
  for (const MemOp& op : g.ops) {
    const size_t j = static_cast<size_t>(op.phase);
    const Bytes sz = sizes[op.object];
    if (op.kind == MemOpKind::allocate) {
      claim[j] += static_cast<std::int64_t>(sz);
    } else if (op.kind == MemOpKind::prefetch && !pinned[op.object]) {
      claim[j] += static_cast<std::int64_t>(sz);
      fetches[j].push_back(Fetch{transfer_duration(sz, bandwidth),
                                 offloaded[op.object] ? offload_end[op.object] : 0});
    }
  }
  std::vector<std::int64_t> claim_prefix(P + 1, 0);
  for (size_t j = 1; j <= P; ++j) claim_prefix[j] = claim_prefix[j - 1] + claim[j];

  const std::int64_t cap = static_cast<std::int64_t>(budget);
  const size_t nfree = free_at.size();
  std::vector<TimeNs> ready(P, 0);
  for (size_t j = 1; j <= P; ++j) {
    TimeNs start = 0;
    if (j > 1) {
      start = ready[j - 2];
      // frees landed by `start` (a free exactly at `start` counts)
      const size_t landed = static_cast<size_t>(
          std::upper_bound(free_at.begin(), free_at.end(), start) - free_at.begin());
      const std::int64_t held = claim_prefix[j - 1] - free_prefix[landed];
      const std::int64_t shortfall = held + claim[j] - cap;
      if (shortfall > 0) {
        // first m in [landed, nfree) whose cumulative frees cover the
        // shortfall, else nfree; the claim then waits for free_at[m-1]
        const std::int64_t target = free_prefix[landed] + shortfall;
        const size_t m = static_cast<size_t>(
            std::lower_bound(free_prefix.begin() + static_cast<std::ptrdiff_t>(landed),
                             free_prefix.begin() + static_cast<std::ptrdiff_t>(nfree),
                             target) -
            free_prefix.begin());
        if (m > 0) start = free_at[m - 1];
      }
    }
    TimeNs t = start;
    for (const Fetch& f : fetches[j]) t = std::max(t, f.earliest) + f.duration;
    ready[j - 1] = t;
  }
  return ready;
}

// Eq. 6 (ref: planner.cpp:188-199): violation iff t_ready[j] is strictly
// later than the sum of the computations before phase j.
std::vector<int> stall_violations(const std::vector<TimeNs>& ready,
                                  const std::vector<TimeNs>& compute) {
  std::vector<int> omega;
  TimeNs before = 0;
  for (size_t j = 0; j < ready.size(); ++j) {
    if (ready[j] > before) omega.push_back(static_cast<int>(j) + 1);
    before += compute[j];
  }
  return omega;
}

// --- O(log ops) pin admission ----------------------------------------------
// Max segment tree over the running sums S[i] (i = op index) with range add.
class PeakTree {
 public:
  explicit PeakTree(const std::vector<std::int64_t>& prefix)
      : n_(prefix.size()), mx_(4 * std::max<size_t>(n_, 1), 0),
        lz_(4 * std::max<size_t>(n_, 1), 0) {
    if (n_) build(1, 0, n_ - 1, prefix);
  }
  // add v to S[i] for every i >= from
  void add_suffix(size_t from, std::int64_t v) {
    if (from < n_) add(1, 0, n_ - 1, from, n_ - 1, v);
  }
  // layer-wise peak: the running sum starts at 0, so the peak is >= 0
  Bytes peak() const {
    return n_ == 0 ? 0 : static_cast<Bytes>(std::max<std::int64_t>(0, mx_[1]));
  }

 private:
  void build(size_t node, size_t lo, size_t hi, const std::vector<std::int64_t>& p) {
    if (lo == hi) {
      mx_[node] = p[lo];
      return;
    }
    const size_t mid = (lo + hi) / 2;
    build(2 * node, lo, mid, p);
    build(2 * node + 1, mid + 1, hi, p);
    mx_[node] = std::max(mx_[2 * node], mx_[2 * node + 1]);
  }
  void add(size_t node, size_t lo, size_t hi, size_t a, size_t b, std::int64_t v) {
    if (a <= lo && hi <= b) {
      mx_[node] += v;
      lz_[node] += v;
      return;
    }
    const size_t mid = (lo + hi) / 2;
    if (a <= mid) add(2 * node, lo, mid, a, b, v);
    if (b > mid) add(2 * node + 1, mid + 1, hi, a, b, v);
    mx_[node] = std::max(mx_[2 * node], mx_[2 * node + 1]) + lz_[node];
  }

  size_t n_;
  std::vector<std::int64_t> mx_, lz_;
};

}  // namespace

// Everything about one k that depends on neither the device budget nor the
// host-link bandwidth (detail::KStatic): k-scaled object sizes, the
// unpinned running sums and their peak, the 2N phase compute times.
detail::KStatic detail::make_k_static(const Gmap& g, const std::vector<PhaseLayer>& phases,
                                      int k, const PerfModel& model) {
  KStatic st;
  st.sizes = detail::scaled_object_sizes(g, k);
  st.running.resize(g.ops.size());
  std::int64_t s = 0;
  for (size_t i = 0; i < g.ops.size(); ++i) {
    const MemOp& op = g.ops[i];
    s += detail::op_delta(op.kind, static_cast<std::int64_t>(st.sizes[op.object]), false);
    st.running[i] = s;
  }
  std::int64_t top = 0;
  for (std::int64_t v : st.running) top = std::max(top, v);
  st.top = static_cast<Bytes>(top);
  return st;
}

std::vector<TimeNs> detail::k_compute_times(const Gmap& g, const std::vector<PhaseLayer>& phases,
                                            int k, const PerfModel& model) {
  std::vector<TimeNs> compute = phase_compute_times(phases, k, model);
  if (static_cast<int>(compute.size()) != g.num_phases)
    throw std::invalid_argument("compute_times must cover all 2N phases");
  return compute;
}

KEvaluation detail::evaluate_static(const Gmap& g, const KStatic& st, int k,
                                    const NetworkSpec& net, const HardwareSpec& hw,
                                    double bandwidth,
                                    const std::function<const std::vector<TimeNs>&()>& compute_of) {
  KEvaluation ev;
  ev.k = k;
  const std::vector<char> none(g.objects.size(), 0);
  const Bytes fixed = fixed_overhead(net, hw);
  const std::vector<Bytes>& sizes = st.sizes;
  ev.active_area_bytes = st.top;

  // C13 memory gate (ref: planner.cpp:261-266)
  if (hw.memory_budget < fixed + ev.active_area_bytes) {
    ev.memory_feasible = false;
    return ev;
  }
  ev.memory_feasible = true;

  // compute times only past the memory gate (the reference evaluates them
  // there, so a model error surfaces at the same k)
  const std::vector<TimeNs>& compute = compute_of();
  const Bytes available = hw.memory_budget - fixed;
  ev.t_ready = ready_times(g, sizes, none, available, bandwidth, compute);
  ev.omega = stall_violations(ev.t_ready, compute);
  if (ev.omega.empty()) {
    ev.stall_free = true;
    ev.resident_peak_bytes = ev.active_area_bytes;
    return ev;
  }

  // C14: prefetched featuremaps of the violating phases, first-seen order,
  // then (scaled size desc, id asc)
  std::vector<char> in_omega(static_cast<size_t>(g.num_phases) + 2, 0);
  for (int j : ev.omega) in_omega[static_cast<size_t>(j)] = 1;
  std::vector<char> seen(g.objects.size(), 0);
  std::vector<ObjectId> cand;
  for (const MemOp& op : g.ops) {
    if (op.kind != MemOpKind::prefetch) continue;
    if (op.phase < 0 || static_cast<size_t>(op.phase) >= in_omega.size() ||
        !in_omega[static_cast<size_t>(op.phase)])
      continue;
    if (!seen[op.object]) {
      seen[op.object] = 1;
      cand.push_back(op.object);
    }
  }
  std::sort(cand.begin(), cand.end(), [&](ObjectId a, ObjectId b) {
    const Bytes sa = sizes[a], sb = sizes[b];
    return sa != sb ? sa > sb : a < b;
  });

  // transfer ops per object (op index, signed effect of pinning it)
  std::vector<std::vector<std::pair<size_t, std::int64_t>>> effect(g.objects.size());
  for (ObjectId c : cand) effect[c].reserve(2);
  std::vector<char> is_cand(g.objects.size(), 0);
  for (ObjectId c : cand) is_cand[c] = 1;
  for (size_t i = 0; i < g.ops.size(); ++i) {
    const MemOp& op = g.ops[i];
    if (!is_cand[op.object]) continue;
    const auto sz = static_cast<std::int64_t>(sizes[op.object]);
    if (op.kind == MemOpKind::offload) effect[op.object].emplace_back(i, +sz);
    if (op.kind == MemOpKind::prefetch) effect[op.object].emplace_back(i, -sz);
  }

  PeakTree tree(st.running);
  Bytes pinned_peak = ev.active_area_bytes;
  std::vector<char> pinned(g.objects.size(), 0);
  for (ObjectId c : cand) {
    for (const auto& [i, v] : effect[c]) tree.add_suffix(i, v);
    const Bytes peak = tree.peak();
    if (peak <= available) {
      ev.pins.insert(c);
      pinned[c] = 1;
      ev.pinned_bytes += sizes[c];
      pinned_peak = peak;
    } else {
      for (const auto& [i, v] : effect[c]) tree.add_suffix(i, -v);
    }
  }
  ev.resident_peak_bytes = pinned_peak;
  if (!ev.pins.empty()) {
    ev.t_ready = ready_times(g, sizes, pinned, available, bandwidth, compute);
    ev.omega = stall_violations(ev.t_ready, compute);
  }
  ev.stall_free = ev.omega.empty();
  return ev;
}

namespace {

KEvaluation evaluate_k(const Gmap& g, const std::vector<PhaseLayer>& phases, int k,
                       const NetworkSpec& net, const HardwareSpec& hw, const PerfModel& model) {
  std::vector<TimeNs> compute;
  return detail::evaluate_static(g, detail::make_k_static(g, phases, k, model), k, net, hw,
                                 model.bandwidth_avail, [&]() -> const std::vector<TimeNs>& {
                                   compute = detail::k_compute_times(g, phases, k, model);
                                   return compute;
                                 });
}

// ref: planner.cpp:324-342
SwapPlan make_plan(const KEvaluation& ev, const std::vector<PhaseLayer>& phases,
                   const NetworkSpec& net, const HardwareSpec& hw,
                   const PerfModel& model, const TrainingConfig& cfg) {
  SwapPlan p;
  p.k_star = ev.k;
  p.pin_set = ev.pins;
  p.t_ready = ev.t_ready;
  p.active_area_bytes = ev.active_area_bytes;
  p.pinned_bytes = ev.pinned_bytes;
  p.fixed_overhead_bytes = fixed_overhead(net, hw);
  p.residual_bytes = hw.memory_budget - p.fixed_overhead_bytes - ev.resident_peak_bytes;
  p.predicted_iter_time = iteration_time(phases, ev.k, model);
  TrainingConfig c = cfg;
  if (c.dataset_size <= 0) c.dataset_size = ev.k;
  p.predicted_whole_time_s = whole_training_time_s(phases, ev.k, model, c);
  return p;
}

int planner_threads() {
  if (const char* s = std::getenv("ACCUDNN_PLANNER_THREADS")) {
    const int v = std::atoi(s);
    if (v > 0) return v;
  }
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? static_cast<int>(hc) : 1;
}

// First feasible k of `order` (the reference's scan order), evaluated in
// parallel waves on plain std::threads (no spinning runtime between waves).
// An exception thrown at a k that the serial scan would have reached first
// is re-thrown, so error behaviour matches too.  `cost` estimates the work
// of one evaluation; tiny instances stay on the calling thread.
std::optional<int> first_feasible(const std::vector<int>& order,
                                  const std::function<bool(int)>& feasible,
                                  size_t cost) {
  const int threads = planner_threads();
  const bool parallel = threads > 1 && cost * order.size() > 2000000;
  size_t wave = parallel ? static_cast<size_t>(threads) * 2 : 64;
  size_t pos = 0;
  while (pos < order.size()) {
    const size_t len = std::min(wave, order.size() - pos);
    std::vector<signed char> verdict(len, 0);
    std::vector<std::exception_ptr> err(len);
    auto work = [&](size_t i) {
      try {
        verdict[i] = feasible(order[pos + i]) ? 1 : 0;
      } catch (...) {
        err[i] = std::current_exception();
      }
    };
    if (parallel && len > 1) {
      std::atomic<size_t> next{0};
      const int nt = static_cast<int>(std::min<size_t>(len, static_cast<size_t>(threads)));
      std::vector<std::thread> pool;
      pool.reserve(static_cast<size_t>(nt));
      for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
          for (size_t i; (i = next.fetch_add(1)) < len;) work(i);
        });
      for (auto& th : pool) th.join();
    } else {
      for (size_t i = 0; i < len; ++i) {
        work(i);
        if (err[i] || verdict[i]) break;  // serial: stop at the first decision
      }
    }
    for (size_t i = 0; i < len; ++i) {
      if (err[i]) std::rethrow_exception(err[i]);
      if (verdict[i]) return order[pos + i];
    }
    pos += len;
    wave = std::min<size_t>(wave * 2, 4096);
  }
  return std::nullopt;
}

}  // namespace

// ---------------------------------------------------------------------------
// public API
// ---------------------------------------------------------------------------

std::vector<TimeNs> compute_t_ready(const Gmap& gmap, int k, Bytes budget,
                                    const PinSet& pins, const PerfModel& model,
                                    const std::vector<TimeNs>& compute_times) {
  if (static_cast<int>(compute_times.size()) != gmap.num_phases)
    throw std::invalid_argument("compute_times must cover all 2N phases");
  const std::vector<Bytes> sizes = detail::scaled_object_sizes(gmap, k);
  const std::vector<char> pinned = detail::pin_mask(gmap, pins);
  const Bytes needed = detail::peak_only(gmap, sizes, pinned);
  if (budget < needed)
    throw UntrainableError("budget " + std::to_string(budget) +
                           " below layer-wise peak " + std::to_string(needed));
  return ready_times(gmap, sizes, pinned, budget, model.bandwidth_avail,
                     compute_times);
}

// Eq. 4 (ref: planner.cpp:160-186)
MemoryCheck check_memory_constraint(const Gmap& gmap, int k, Bytes budget,
                                    const PinSet& pins) {
  const std::vector<Bytes> sizes = detail::scaled_object_sizes(gmap, k);
  const std::vector<char> pinned = detail::pin_mask(gmap, pins);
  MemoryCheck mc;
  std::int64_t run = 0, top = 0;
  const auto cap = static_cast<std::int64_t>(budget);
  for (const MemOp& op : gmap.ops) {
    run += detail::op_delta(op.kind, static_cast<std::int64_t>(sizes[op.object]),
                            pinned[op.object] != 0);
    top = std::max(top, run);
    if (mc.ok && run > cap) {
      mc.ok = false;
      mc.first_violation_seq = op.sequence_no;
    }
  }
  mc.peak_bytes = static_cast<Bytes>(top);
  return mc;
}

std::vector<int> check_stall_constraint(const std::vector<TimeNs>& t_ready,
                                        const std::vector<TimeNs>& compute_times) {
  if (t_ready.size() != compute_times.size())
    throw std::invalid_argument("t_ready and compute_times length mismatch");
  return stall_violations(t_ready, compute_times);
}

// ref: planner.cpp:201-216
ConstraintReport build_constraint_report(const Gmap& gmap, int k, Bytes budget,
                                         const PinSet& pins,
                                         const std::vector<TimeNs>& t_ready,
                                         const std::vector<TimeNs>& compute_times) {
  ConstraintReport r;
  r.memory = check_memory_constraint(gmap, k, budget, pins);
  r.violating_phases = check_stall_constraint(t_ready, compute_times);
  r.stall_ok = r.violating_phases.empty();
  r.slack.resize(t_ready.size());
  TimeNs before = 0;
  for (size_t j = 0; j < t_ready.size(); ++j) {
    r.slack[j] = before - t_ready[j];
    before += compute_times[j];
  }
  return r;
}

// C12 (ref: planner.cpp:218-253)
KmaxResult max_trainable_minibatch(const Gmap& gmap, const NetworkSpec& net,
                                   const HardwareSpec& hw) {
  KmaxResult res;
  const Bytes fixed = fixed_overhead(net, hw);
  const PeakResult pk = peak_layerwise_memory(gmap, net.k_base, {});
  Bytes ws = 0, fm = 0;
  for (ObjectId id : pk.live_objects) {
    const MemObject& o = gmap.object(id);
    const Bytes sz = scale_size(o, net.k_base, net.k_base);
    if (o.kind == ObjectKind::workspace) ws += sz;
    if (o.kind == ObjectKind::featuremap) fm += sz;
  }
  if (fm == 0)
    throw SpecError("peak working set holds no featuremap bytes; "
                    "the maximal minibatch is unbounded");
  if (hw.memory_budget <= fixed + ws) {
    res.reason = "memory budget does not exceed the fixed overheads";
    return res;
  }
  using u128 = unsigned __int128;
  const u128 kmax = static_cast<u128>(net.k_base) *
                    static_cast<u128>(hw.memory_budget - fixed - ws) / fm;
  if (kmax < 1) {
    res.reason = "budget cannot fit a single sample's working set";
    return res;
  }
  res.trainable = true;
  res.k_max = static_cast<int>(std::min<u128>(kmax, u128{1} << 30));
  return res;
}

KEvaluation evaluate_minibatch(const Gmap& gmap,
                               const std::vector<PhaseLayer>& phases, int k,
                               const NetworkSpec& net, const HardwareSpec& hw,
                               const PerfModel& model) {
  return evaluate_k(gmap, phases, k, net, hw, model);
}

// Algorithm 2 (ref: planner.cpp:346-424) over an evaluator of k
PlanResult detail::search_plan(const Gmap& gmap, const std::vector<PhaseLayer>& phases,
                               const NetworkSpec& net, const HardwareSpec& hw,
                               const PerfModel& model, const TrainingConfig& cfg,
                               const PlannerOptions& opts,
                               const std::function<KEvaluation(int)>& evaluate) {
  PlanResult res;
  const KmaxResult km = max_trainable_minibatch(gmap, net, hw);
  if (!km.trainable) {
    res.status = PlanStatus::untrainable;
    res.detail = km.reason;
    return res;
  }

  if (opts.k_override > 0) {
    const KEvaluation ev = evaluate(opts.k_override);
    if (ev.memory_feasible && ev.stall_free) {
      res.status = PlanStatus::ok;
      res.plan = make_plan(ev, phases, net, hw, model, cfg);
    } else {
      res.status = PlanStatus::infeasible;
      res.detail = ev.memory_feasible
                       ? "stall constraint not satisfiable at the requested k"
                       : "memory constraint violated at the requested k";
    }
    return res;
  }

  auto ok_at = [&](int k) {
    const KEvaluation ev = evaluate(k);
    return ev.memory_feasible && ev.stall_free;
  };
  auto descending = [](int from, int to, int stride) {
    std::vector<int> v;
    for (int k = from; k >= to; k -= stride) v.push_back(k);
    return v;
  };

  const size_t cost = gmap.ops.size() + phases.size();
  const int step = std::max(1, opts.step);
  std::optional<int> hit;
  if (step == 1) {
    hit = first_feasible(descending(km.k_max, 1, 1), ok_at, cost);
  } else {
    const std::optional<int> coarse = first_feasible(descending(km.k_max, 1, step), ok_at, cost);
    if (coarse) {
      hit = coarse;
      const int hi = std::min(km.k_max, *coarse + step - 1);
      if (auto fine = first_feasible(descending(hi, *coarse + 1, 1), ok_at, cost)) hit = fine;
    } else {
      hit = first_feasible(descending(km.k_max, 1, 1), ok_at, cost);
    }
  }

  if (!hit) {
    const KEvaluation one = evaluate(1);
    if (!one.memory_feasible) {
      res.status = PlanStatus::untrainable;
      res.detail = "layer-wise peak at k=1 exceeds the memory budget";
    } else {
      res.status = PlanStatus::infeasible;
      res.detail = "no minibatch size satisfies the stall constraint";
    }
    return res;
  }
  const KEvaluation best = evaluate(*hit);
  res.status = PlanStatus::ok;
  res.plan = make_plan(best, phases, net, hw, model, cfg);
  return res;
}

PlanResult find_efficiency_optimal_minibatch(const Gmap& gmap,
                                             const std::vector<PhaseLayer>& phases,
                                             const NetworkSpec& net,
                                             const HardwareSpec& hw,
                                             const PerfModel& model,
                                             const TrainingConfig& cfg,
                                             const PlannerOptions& opts) {
  return detail::search_plan(gmap, phases, net, hw, model, cfg, opts, [&](int k) {
    return evaluate_k(gmap, phases, k, net, hw, model);
  });
}

// ref: planner.cpp:426-433
long long adjust_iterations(int k_star, int k_base, long long iters_base) {
  if (k_star <= 0 || k_base <= 0 || iters_base <= 0)
    throw std::invalid_argument("adjust_iterations requires positive inputs");
  using i128 = __int128;
  const i128 num = static_cast<i128>(iters_base) * k_base;
  return static_cast<long long>((num + k_star - 1) / k_star);
}

// plan.json (ref: planner.cpp:435-456)
std::string swap_plan_to_json(const SwapPlan& plan, const Gmap& gmap,
                              const std::vector<TimeNs>& slack) {
  json doc;
  doc["format_version"] = 1;
  doc["k_star"] = plan.k_star;
  json names = json::array();
  for (ObjectId id : plan.pin_set) names.push_back(gmap.object(id).name);
  doc["pinned_objects"] = std::move(names);
  json tr = json::array();
  for (TimeNs t : plan.t_ready) tr.push_back(to_seconds(t));
  doc["t_ready_s"] = std::move(tr);
  doc["predicted_iter_time_s"] = to_seconds(plan.predicted_iter_time);
  doc["predicted_whole_time_s"] = plan.predicted_whole_time_s;
  doc["active_area_bytes"] = plan.active_area_bytes;
  doc["pinned_bytes"] = plan.pinned_bytes;
  doc["residual_bytes"] = plan.residual_bytes;
  doc["fixed_overhead_bytes"] = plan.fixed_overhead_bytes;
  json sl = json::array();
  for (TimeNs t : slack) sl.push_back(to_seconds(t));
  doc["slack_s"] = std::move(sl);
  return doc.dump(2) + "\n";
}

}  // namespace swapsched
