// Three-stream discrete-event model of one training iteration: compute,
// swap-out (D2H) and swap-in (H2D) with a bounded pool and one FIFO copy
// channel per direction.  This is the behavioural contract the CUDA
// executor realises with real streams and events, and the oracle for
// "exposed swap time".
//
// Semantics: /root/reference/proj/src/simulator.cpp:79-370 (event order,
// tie-break compute < swap_out < swap_in < schedule tick, head-of-line
// blocking on the swap-in queue, deadlock detection) -- the trace is
// byte-identical for identical inputs.
#include <algorithm>
#include <cstdio>
#include <queue>
#include <sstream>
#include <tuple>

#include <json.hpp>

#include "swapsched/api.hpp"

namespace swapsched {

using nlohmann::json;

std::string sim_mode_name(SimMode m) {
  switch (m) {
    case SimMode::naive: return "naive";
    case SimMode::dynamic: return "dynamic";
    case SimMode::resident: return "resident";
  }
  return "naive";
}

std::string stream_name(Stream s) {
  switch (s) {
    case Stream::compute: return "compute";
    case Stream::swap_out: return "swap_out";
    case Stream::swap_in: return "swap_in";
  }
  return "compute";
}

std::string event_kind_name(EventKind k) {
  static const char* const names[] = {"kernel_start", "kernel_end", "xfer_start",
                                      "xfer_end",     "alloc",      "free",
                                      "block",        "unblock"};
  const int i = static_cast<int>(k);
  return (i >= 0 && i < 8) ? names[i] : "alloc";
}

namespace {

struct QueueEntry {
  MemOpKind kind;
  ObjectId object;
  int phase;
  Bytes size;
};

enum class Completion { kernel_end, swap_in_done, swap_out_done };

struct Timer {
  TimeNs at;
  int rank;            // compute 0 < swap_out 1 < swap_in 2
  std::uint64_t tick;  // schedule order
  Completion what;
  bool operator>(const Timer& o) const {
    return std::tie(at, rank, tick) > std::tie(o.at, o.rank, o.tick);
  }
};

class IterationModel {
 public:
  IterationModel(const Gmap& g, const std::vector<PhaseLayer>& phases, int k,
                 const PinSet& pins, const PerfModel& model, const SimConfig& cfg)
      : g_(g), cfg_(cfg), P_(g.num_phases) {
    const std::vector<char> pinned = [&] {
      std::vector<char> m(g.objects.size(), 0);
      for (ObjectId id : pins) m[id] = 1;
      return m;
    }();
    waiting_.assign(static_cast<size_t>(P_) + 1, 0);
    needs_offload_.assign(g.objects.size(), 0);
    offload_done_.assign(g.objects.size(), 0);
    kernel_done_.assign(static_cast<size_t>(P_) + 1, 0);
    for (const MemOp& op : g.ops) {
      const bool pin = pinned[op.object] != 0;
      const QueueEntry e{op.kind, op.object, op.phase, g.op_bytes(op, k)};
      switch (op.kind) {
        case MemOpKind::allocate:
          in_q_.push_back(e);
          waiting_[static_cast<size_t>(op.phase)]++;
          break;
        case MemOpKind::prefetch:
          if (pin) break;
          in_q_.push_back(e);
          waiting_[static_cast<size_t>(op.phase)]++;
          break;
        case MemOpKind::offload:
          if (pin) break;
          out_q_.push_back(e);
          needs_offload_[op.object] = 1;
          break;
        case MemOpKind::release:
          out_q_.push_back(e);
          break;
      }
    }
    duration_.resize(static_cast<size_t>(P_));
    for (int j = 0; j < P_; ++j)
      duration_[static_cast<size_t>(j)] =
          layer_compute_time(phases[static_cast<size_t>(j)], k, model);
    SimSummary& s = out_.summary;
    s.per_phase_stall.assign(static_cast<size_t>(P_), 0);
    s.data_ready.assign(static_cast<size_t>(P_), 0);
    s.kernel_start.assign(static_cast<size_t>(P_), 0);
    s.kernel_end.assign(static_cast<size_t>(P_), 0);
    used_ = cfg.fixed_overhead;
    peak_ = used_;
  }

  SimResult run() {
    note_memory();
    settle();
    while (!timers_.empty()) {
      const Timer t = timers_.top();
      timers_.pop();
      now_ = t.at;
      complete(t.what);
      settle();
    }
    finish();
    return std::move(out_);
  }

 private:
  std::string name_of(ObjectId id) const { return g_.object(id).name; }

  void log(Stream s, EventKind kind, std::string subject) {
    out_.events.push_back(SimEvent{now_, s, kind, std::move(subject), used_});
  }
  void note_memory() {
    peak_ = std::max(peak_, used_);
    auto& ts = out_.summary.mem_timeseries;
    if (!ts.empty() && ts.back().first == now_)
      ts.back().second = used_;
    else
      ts.emplace_back(now_, used_);
  }
  void arm(TimeNs at, Stream s, Completion what) {
    const int rank = s == Stream::compute ? 0 : (s == Stream::swap_out ? 1 : 2);
    timers_.push(Timer{at, rank, tick_++, what});
  }
  bool try_claim(Bytes n) {
    if (used_ + n > cfg_.budget) return false;
    used_ += n;
    note_memory();
    return true;
  }
  void give_back(Bytes n) {
    used_ -= std::min(used_, n);
    note_memory();
  }
  void mark_blocked(ObjectId who) {
    if (blocked_) return;
    log(Stream::swap_in, EventKind::block, name_of(who));
    blocked_ = true;
  }
  void phase_input_landed(int phase) {
    if (--waiting_[static_cast<size_t>(phase)] == 0)
      out_.summary.data_ready[static_cast<size_t>(phase - 1)] = now_;
  }

  bool step_compute() {
    if (kernel_busy_ || next_ > P_) return false;
    if (next_ > 1 && !kernel_done_[static_cast<size_t>(next_ - 1)]) return false;
    if (waiting_[static_cast<size_t>(next_)] != 0) return false;
    kernel_busy_ = true;
    out_.summary.kernel_start[static_cast<size_t>(next_ - 1)] = now_;
    log(Stream::compute, EventKind::kernel_start, "phase " + std::to_string(next_));
    arm(now_ + duration_[static_cast<size_t>(next_ - 1)], Stream::compute,
        Completion::kernel_end);
    return true;
  }

  bool step_swap_out() {
    bool moved = false;
    while (!out_busy_ && out_head_ < out_q_.size()) {
      const QueueEntry& e = out_q_[out_head_];
      if (!kernel_done_[static_cast<size_t>(e.phase)]) break;
      moved = true;
      if (e.kind == MemOpKind::release) {
        give_back(e.size);
        log(Stream::swap_out, EventKind::free, name_of(e.object));
        ++out_head_;
        continue;
      }
      log(Stream::swap_out, EventKind::xfer_start, name_of(e.object));
      out_busy_ = true;
      arm(now_ + transfer_duration(e.size, cfg_.bandwidth), Stream::swap_out,
          Completion::swap_out_done);
    }
    return moved;
  }

  bool step_swap_in() {
    bool moved = false;
    while (!in_busy_ && in_head_ < in_q_.size()) {
      const QueueEntry& e = in_q_[in_head_];
      const bool fetch = e.kind == MemOpKind::prefetch;
      if (fetch && needs_offload_[e.object] && !offload_done_[e.object]) {
        mark_blocked(e.object);
        break;
      }
      if (!try_claim(e.size)) {
        mark_blocked(e.object);
        break;
      }
      if (blocked_) {
        log(Stream::swap_in, EventKind::unblock, name_of(e.object));
        blocked_ = false;
      }
      moved = true;
      if (fetch) {
        log(Stream::swap_in, EventKind::xfer_start, name_of(e.object));
        in_busy_ = true;
        arm(now_ + transfer_duration(e.size, cfg_.bandwidth), Stream::swap_in,
            Completion::swap_in_done);
      } else {
        log(Stream::swap_in, EventKind::alloc, name_of(e.object));
        if (cfg_.alloc_cost > 0) {
          in_busy_ = true;
          arm(now_ + cfg_.alloc_cost, Stream::swap_in, Completion::swap_in_done);
        } else {
          ++in_head_;
          phase_input_landed(e.phase);
        }
      }
    }
    return moved;
  }

  // run every stream until none can make progress at the current instant
  void settle() {
    for (;;) {
      bool any = step_compute();
      any = step_swap_out() || any;
      any = step_swap_in() || any;
      if (!any) break;
    }
  }

  void complete(Completion what) {
    switch (what) {
      case Completion::kernel_end:
        kernel_busy_ = false;
        kernel_done_[static_cast<size_t>(next_)] = 1;
        out_.summary.kernel_end[static_cast<size_t>(next_ - 1)] = now_;
        log(Stream::compute, EventKind::kernel_end, "phase " + std::to_string(next_));
        ++next_;
        break;
      case Completion::swap_out_done: {
        const QueueEntry& e = out_q_[out_head_];
        give_back(e.size);
        offload_done_[e.object] = 1;
        log(Stream::swap_out, EventKind::xfer_end, name_of(e.object));
        out_busy_ = false;
        ++out_head_;
        break;
      }
      case Completion::swap_in_done: {
        const QueueEntry& e = in_q_[in_head_];
        if (e.kind == MemOpKind::prefetch)
          log(Stream::swap_in, EventKind::xfer_end, name_of(e.object));
        in_busy_ = false;
        ++in_head_;
        phase_input_landed(e.phase);
        break;
      }
    }
  }

  void finish() {
    SimSummary& s = out_.summary;
    const bool stuck = next_ <= P_ || kernel_busy_ || in_head_ < in_q_.size() ||
                       out_head_ < out_q_.size();
    if (stuck) {
      s.oom = true;
      std::ostringstream why;
      why << "deadlock at t=" << to_seconds(now_) << "s:";
      if (next_ <= P_)
        why << " compute waits for phase " << next_ << " ("
            << waiting_[static_cast<size_t>(next_)] << " swap-in ops outstanding);";
      if (in_head_ < in_q_.size()) {
        const QueueEntry& e = in_q_[in_head_];
        why << " swap-in blocked on " << mem_op_kind_name(e.kind) << " "
            << name_of(e.object) << " (" << e.size << " B, "
            << (cfg_.budget - used_) << " B free);";
      }
      if (out_head_ < out_q_.size())
        why << " swap-out waits for phase " << out_q_[out_head_].phase << "'s kernel;";
      s.oom_detail = why.str();
    }
    s.peak_mem = peak_;
    if (!s.oom) {
      s.iter_time = s.kernel_end.back();
      TimeNs prev = 0;
      s.total_stall = 0;
      for (int j = 0; j < P_; ++j) {
        const size_t u = static_cast<size_t>(j);
        s.per_phase_stall[u] = s.kernel_start[u] - prev;
        prev = s.kernel_end[u];
        s.total_stall += s.per_phase_stall[u];
      }
    }
  }

  const Gmap& g_;
  const SimConfig& cfg_;
  const int P_;
  std::vector<QueueEntry> in_q_, out_q_;
  std::vector<int> waiting_;
  std::vector<char> needs_offload_, offload_done_, kernel_done_;
  std::vector<TimeNs> duration_;
  std::priority_queue<Timer, std::vector<Timer>, std::greater<>> timers_;
  SimResult out_;
  TimeNs now_ = 0;
  Bytes used_ = 0, peak_ = 0;
  std::uint64_t tick_ = 0;
  int next_ = 1;
  bool kernel_busy_ = false, in_busy_ = false, out_busy_ = false, blocked_ = false;
  size_t in_head_ = 0, out_head_ = 0;
};

}  // namespace

SimResult simulate_iteration(const Gmap& gmap,
                             const std::vector<PhaseLayer>& phases, int k,
                             const PinSet& pins, const PerfModel& model,
                             const SimConfig& cfg) {
  if (static_cast<int>(phases.size()) != gmap.num_phases)
    throw std::invalid_argument("phase list does not match the gmap");
  if (cfg.bandwidth <= 0.0) throw std::invalid_argument("bandwidth must be positive");
  for (ObjectId id : pins) {
    if (id >= gmap.objects.size())
      throw std::invalid_argument("pin set references unknown object");
    if (gmap.object(id).kind != ObjectKind::featuremap)
      throw std::invalid_argument("only featuremaps can be pinned");
  }
  if (cfg.mode == SimMode::naive && !pins.empty())
    throw std::invalid_argument("naive mode requires an empty pin set");
  if (cfg.mode == SimMode::resident && pins.size() != gmap.featuremap_ids().size())
    throw std::invalid_argument("resident mode requires every featuremap pinned");
  IterationModel m(gmap, phases, k, pins, model, cfg);
  return m.run();
}

std::vector<StallRow> stall_report(const SimSummary& summary) {
  if (summary.oom)
    throw std::invalid_argument("stall report requested for a deadlocked trace");
  std::vector<StallRow> rows(summary.per_phase_stall.size());
  for (size_t j = 0; j < rows.size(); ++j)
    rows[j] = StallRow{static_cast<int>(j) + 1, summary.per_phase_stall[j]};
  return rows;
}

// ref: simulator.cpp:382-407
Verdict verify_plan(const SwapPlan& plan, const SimSummary& summary,
                    Bytes budget, double tolerance) {
  Verdict v;
  if (summary.oom) {
    v.detail = "simulation deadlocked: " + summary.oom_detail;
    return v;
  }
  v.memory_ok = summary.peak_mem <= budget;
  v.stall_fraction = summary.iter_time > 0 ? to_seconds(summary.total_stall) /
                                                 to_seconds(summary.iter_time)
                                           : 0.0;
  const size_t n = std::min(plan.t_ready.size(), summary.data_ready.size());
  for (size_t j = 0; j < n; ++j) {
    const TimeNs d = summary.data_ready[j] - plan.t_ready[j];
    v.max_ready_deviation = std::max<TimeNs>(v.max_ready_deviation, d < 0 ? -d : d);
  }
  v.pass = v.memory_ok && v.stall_fraction <= tolerance;
  std::ostringstream os;
  os << "stall_fraction=" << v.stall_fraction << " peak_mem=" << summary.peak_mem
     << " budget=" << budget;
  v.detail = os.str();
  return v;
}

namespace {

std::string secs9(TimeNs t) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.9f", to_seconds(t));
  return buf;
}

}  // namespace

std::string trace_to_csv(const std::vector<SimEvent>& events) {
  std::string out = "time_s,stream,kind,subject,mem_used_bytes\n";
  for (const SimEvent& e : events) {
    out += secs9(e.time);
    out += ',';
    out += stream_name(e.stream);
    out += ',';
    out += event_kind_name(e.kind);
    out += ',';
    out += e.subject;
    out += ',';
    out += std::to_string(e.mem_used_after);
    out += '\n';
  }
  return out;
}

std::string summary_to_json(const SimSummary& summary) {
  json doc;
  doc["format_version"] = 1;
  doc["oom"] = summary.oom;
  if (summary.oom) {
    doc["oom_detail"] = summary.oom_detail;
  } else {
    doc["iter_time_s"] = to_seconds(summary.iter_time);
    doc["total_stall_s"] = to_seconds(summary.total_stall);
    json st = json::array();
    for (TimeNs s : summary.per_phase_stall) st.push_back(to_seconds(s));
    doc["per_phase_stall_s"] = std::move(st);
  }
  doc["peak_mem_bytes"] = summary.peak_mem;
  return doc.dump(2) + "\n";
}

// Fig. 6 two-curve view (ref: simulator.cpp:445-466)
std::string mem_curves_csv(const std::vector<SimEvent>& events,
                           Bytes fixed_overhead) {
  std::string out = "time_s,cum_allocated_bytes,cum_freed_bytes,mem_used_bytes\n";
  Bytes allocated = fixed_overhead, freed = 0, last = fixed_overhead;
  auto row = [&out](TimeNs t, Bytes a, Bytes f, Bytes u) {
    out += secs9(t) + ',' + std::to_string(a) + ',' + std::to_string(f) + ',' +
           std::to_string(u) + '\n';
  };
  row(0, allocated, freed, fixed_overhead);
  for (const SimEvent& e : events) {
    if (e.mem_used_after == last) continue;
    if (e.mem_used_after > last)
      allocated += e.mem_used_after - last;
    else
      freed += last - e.mem_used_after;
    last = e.mem_used_after;
    row(e.time, allocated, freed, e.mem_used_after);
  }
  return out;
}

std::string stall_bars_csv(const SimSummary& summary) {
  std::string out = "phase,stall_s\n";
  for (size_t j = 0; j < summary.per_phase_stall.size(); ++j)
    out += std::to_string(j + 1) + ',' + secs9(summary.per_phase_stall[j]) + '\n';
  return out;
}

}  // namespace swapsched
