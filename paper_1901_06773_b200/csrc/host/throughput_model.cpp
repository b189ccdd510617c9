// Profile ingestion, isotonic throughput curves, Eq. 2/3/5 timing and the
// learning-rate rule.
//
// Semantics: /root/reference/proj/src/profiles.cpp, perf_model.cpp and
// lr_tuner.cpp (cited per function).  Every floating-point expression that
// feeds a planner decision keeps the reference's operand order so that the
// rounded nanosecond durations are identical (Appendix C rules C2, C4, C6-C9).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <iterator>
#include <map>
#include <sstream>

#include <json.hpp>

#include "swapsched/api.hpp"
#include "internal.hpp"

namespace swapsched {

using nlohmann::json;

// ---------------------------------------------------------------------------
// CSV ingestion (ref: profiles.cpp:10-172)
// ---------------------------------------------------------------------------
namespace {

std::string trim_ws(const std::string& s) {
  const size_t a = s.find_first_not_of(" \t\r");
  if (a == std::string::npos) return std::string();
  const size_t b = s.find_last_not_of(" \t\r");
  return s.substr(a, b - a + 1);
}

// getline-on-',' splitting: a trailing empty field is dropped, inner empty
// fields are kept (this decides the column-count diagnostics)
std::vector<std::string> csv_fields(const std::string& line) {
  std::vector<std::string> out;
  std::stringstream in(line);
  std::string cell;
  while (std::getline(in, cell, ',')) out.push_back(trim_ws(cell));
  return out;
}

template <typename Int>
bool whole_int(const std::string& s, Int& v) {
  const char* b = s.data();
  const char* e = b + s.size();
  auto r = std::from_chars(b, e, v);
  return r.ec == std::errc() && r.ptr == e;
}

bool whole_double(const std::string& s, double& v) {
  try {
    size_t used = 0;
    v = std::stod(s, &used);
    return used == s.size();
  } catch (...) {
    return false;
  }
}

bool blank(const std::string& line) {
  return line.empty() || line.find_first_not_of(" \t\r") == std::string::npos;
}

}  // namespace

ProfileSet parse_profile_csv(const std::string& text, const std::string& origin,
                             const ProfileLoadOptions& opts) {
  static const std::vector<std::string> kComputeHeader = {
      "minibatch", "phase", "layer_type", "flops", "time_s"};
  static const std::vector<std::string> kTransferHeader = {
      "minibatch", "seq_no", "bytes", "time_s"};

  ProfileSet set;
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line)) throw SpecError(origin + ": empty profile file");
  const auto header = csv_fields(line);
  const bool compute = header == kComputeHeader;
  const bool transfer = header == kTransferHeader;
  if (!compute && !transfer)
    throw SpecError(origin +
                    ": unrecognized header; expected "
                    "'minibatch,phase,layer_type,flops,time_s' or "
                    "'minibatch,seq_no,bytes,time_s'");

  int row = 1, accepted = 0;
  while (std::getline(in, line)) {
    ++row;
    if (blank(line)) continue;
    const auto f = csv_fields(line);
    auto skip = [&](const char* why) {
      set.diagnostics.push_back(origin + ":" + std::to_string(row) + ": " + why);
    };
    // time gate shared by both kinds: positive, and above the timer noise
    auto time_ok = [&](double t) {
      if (!(t > 0.0)) {
        skip("time must be positive");
        return false;
      }
      if (t < opts.min_sample_s) {
        skip("sample below noise threshold");
        return false;
      }
      return true;
    };
    if (compute) {
      if (f.size() != 5) {
        skip("expected 5 columns");
        continue;
      }
      long long mb = 0, phase = 0;
      unsigned long long flops = 0;
      ComputeSample s;
      if (!whole_int(f[0], mb) || !whole_int(f[1], phase) ||
          !whole_int(f[3], flops) || !whole_double(f[4], s.time_s)) {
        skip("unparsable numeric field");
        continue;
      }
      s.minibatch = static_cast<int>(mb);
      s.phase = static_cast<int>(phase);
      s.layer_type = f[2];
      s.flops = flops;
      if (s.flops == 0) {
        skip("flops must be positive");
        continue;
      }
      if (!time_ok(s.time_s)) continue;
      set.sampled_minibatches.insert(s.minibatch);
      set.compute_samples.push_back(std::move(s));
    } else {
      if (f.size() != 4) {
        skip("expected 4 columns");
        continue;
      }
      long long mb = 0;
      unsigned long long seq = 0, bytes = 0;
      TransferSample s;
      if (!whole_int(f[0], mb) || !whole_int(f[1], seq) ||
          !whole_int(f[2], bytes) || !whole_double(f[3], s.time_s)) {
        skip("unparsable numeric field");
        continue;
      }
      s.minibatch = static_cast<int>(mb);
      s.seq_no = static_cast<std::uint32_t>(seq);
      s.bytes = bytes;
      if (s.bytes == 0) {
        skip("bytes must be positive");
        continue;
      }
      if (!time_ok(s.time_s)) continue;
      set.sampled_minibatches.insert(s.minibatch);
      set.transfer_samples.push_back(std::move(s));
    }
    ++accepted;
  }
  if (accepted == 0) throw SpecError(origin + ": no valid rows");
  return set;
}

ProfileSet load_profiles(const std::vector<std::filesystem::path>& paths,
                         const ProfileLoadOptions& opts) {
  if (paths.empty()) throw SpecError("no profile files given");
  ProfileSet all;
  for (const auto& p : paths) {
    ProfileSet one = parse_profile_csv(detail::slurp(p), p.string(), opts);
    all.compute_samples.insert(all.compute_samples.end(),
                               std::make_move_iterator(one.compute_samples.begin()),
                               std::make_move_iterator(one.compute_samples.end()));
    all.transfer_samples.insert(all.transfer_samples.end(),
                                one.transfer_samples.begin(),
                                one.transfer_samples.end());
    all.sampled_minibatches.insert(one.sampled_minibatches.begin(),
                                   one.sampled_minibatches.end());
    all.diagnostics.insert(all.diagnostics.end(),
                           std::make_move_iterator(one.diagnostics.begin()),
                           std::make_move_iterator(one.diagnostics.end()));
  }
  return all;
}

// C4 (ref: profiles.cpp:174-182): round half up in 128-bit integers
Flops scale_flops_count(Flops flops_base, int k, int k_base) {
  if (k <= 0) throw std::invalid_argument("minibatch must be positive");
  if (k_base <= 0) throw std::invalid_argument("k_base must be positive");
  using u128 = unsigned __int128;
  const u128 num = static_cast<u128>(flops_base) * static_cast<u128>(k);
  const u128 den = static_cast<u128>(k_base);
  return static_cast<Flops>((num + den / 2) / den);
}

Flops scale_flops(const PhaseLayer& phase, int k, int k_base) {
  return scale_flops_count(phase.flops_base, k, k_base);
}

// C6 (ref: profiles.cpp:188-198): long double totals in sample order
double effective_bandwidth(const std::vector<TransferSample>& samples,
                           double fallback) {
  if (samples.empty()) return fallback;
  long double bytes = 0.0L, seconds = 0.0L;
  for (const TransferSample& s : samples) {
    bytes += static_cast<long double>(s.bytes);
    seconds += static_cast<long double>(s.time_s);
  }
  return static_cast<double>(bytes / seconds);
}

// ---------------------------------------------------------------------------
// Throughput curves (ref: perf_model.cpp:13-111)
// ---------------------------------------------------------------------------

// C8: clamp below, plateau above, linear between neighbouring knots; x eta.
// Knot abscissae are strictly increasing (one knot per distinct FLOPs value),
// so the first knot with x >= flops is found by bisection.
double ThroughputCurve::rate_at(Flops flops) const {
  if (knots.empty()) throw std::logic_error("empty throughput curve");
  double raw;
  if (flops <= knots.front().first) {
    raw = knots.front().second;
  } else if (flops >= knots.back().first) {
    raw = plateau;
  } else {
    auto hi_it = std::lower_bound(
        knots.begin() + 1, knots.end(), flops,
        [](const std::pair<Flops, double>& kn, Flops f) { return kn.first < f; });
    const auto& lo = *(hi_it - 1);
    const auto& hi = *hi_it;
    const double x0 = static_cast<double>(lo.first);
    const double x1 = static_cast<double>(hi.first);
    const double t = (static_cast<double>(flops) - x0) / (x1 - x0);
    raw = lo.second + t * (hi.second - lo.second);
  }
  return raw * efficiency;
}

const ThroughputCurve& PerfModel::curve_for(const std::string& type_key) const {
  const auto it = curves.find(type_key);
  if (it == curves.end())
    throw SpecError("no throughput curve for layer type '" + type_key + "'");
  return it->second;
}

// C7: group by exact FLOPs (ascending), group rate = mean of flops/time,
// pool-adjacent-violators with a strict '>' merge test and weighted means.
ThroughputCurve fit_throughput_curve(const std::vector<ComputeSample>& samples,
                                     double eta) {
  if (eta <= 0.0 || eta > 1.0)
    throw std::invalid_argument("efficiency factor must be in (0, 1]");

  std::map<Flops, std::pair<double, double>> by_flops;  // (sum of rates, n)
  std::string type_key;
  for (const ComputeSample& s : samples) {
    if (type_key.empty()) type_key = s.layer_type;
    if (!(s.time_s > 0.0) || s.flops == 0)
      throw SpecError("nonpositive sample for layer type '" + s.layer_type + "'");
    auto& acc = by_flops[s.flops];
    acc.first += static_cast<double>(s.flops) / s.time_s;
    acc.second += 1.0;
  }
  if (by_flops.size() < 2)
    throw SpecError("need samples at >= 2 distinct FLOPs values for layer type '" +
                    type_key + "'");

  struct Pool {
    double mean;
    double weight;
    size_t span;
  };
  std::vector<Flops> xs;
  std::vector<Pool> pools;
  xs.reserve(by_flops.size());
  pools.reserve(by_flops.size());
  for (const auto& [x, acc] : by_flops) {
    xs.push_back(x);
    pools.push_back(Pool{acc.first / acc.second, acc.second, 1});
    while (pools.size() > 1 && pools[pools.size() - 2].mean > pools.back().mean) {
      const Pool right = pools.back();
      pools.pop_back();
      Pool& left = pools.back();
      left.mean = (left.mean * left.weight + right.mean * right.weight) /
                  (left.weight + right.weight);
      left.weight += right.weight;
      left.span += right.span;
    }
  }

  ThroughputCurve c;
  c.layer_type = type_key;
  c.efficiency = eta;
  c.knots.reserve(xs.size());
  size_t xi = 0;
  for (const Pool& p : pools)
    for (size_t r = 0; r < p.span; ++r) c.knots.emplace_back(xs[xi++], p.mean);
  c.plateau = c.knots.back().second;
  return c;
}

PerfModel build_perf_model(const ProfileSet& profiles, int k_base, double eta,
                           double bandwidth_fallback) {
  std::map<std::string, std::vector<ComputeSample>> per_type;
  for (const ComputeSample& s : profiles.compute_samples)
    per_type[s.layer_type].push_back(s);
  if (per_type.empty()) throw SpecError("no compute samples to fit");

  PerfModel m;
  m.k_base = k_base;
  for (const auto& [type, samples] : per_type)
    m.curves[type] = fit_throughput_curve(samples, eta);
  m.bandwidth_avail =
      effective_bandwidth(profiles.transfer_samples, bandwidth_fallback);
  if (m.bandwidth_avail <= 0.0)
    throw SpecError("effective bandwidth must be positive; no transfer samples "
                    "and no usable fallback");
  return m;
}

// C9 (ref: perf_model.cpp:113-117)
TimeNs layer_compute_time(const PhaseLayer& phase, int k, const PerfModel& model) {
  const Flops f = scale_flops(phase, k, model.k_base);
  return compute_duration(f, model.curve_for(phase.type_key).rate_at(f));
}

std::vector<TimeNs> phase_compute_times(const std::vector<PhaseLayer>& phases,
                                        int k, const PerfModel& model) {
  std::vector<TimeNs> t(phases.size());
  for (size_t i = 0; i < phases.size(); ++i)
    t[i] = layer_compute_time(phases[i], k, model);
  return t;
}

TimeNs iteration_time(const std::vector<PhaseLayer>& phases, int k,
                      const PerfModel& model) {
  TimeNs sum = 0;
  for (const PhaseLayer& p : phases) sum += layer_compute_time(p, k, model);
  return sum;
}

// Eq. 3 (ref: perf_model.cpp:127-144)
double whole_training_time_s(const std::vector<PhaseLayer>& phases, int k,
                             const PerfModel& model, const TrainingConfig& cfg) {
  if (k <= 0) throw std::invalid_argument("minibatch must be positive");
  if (cfg.dataset_size > 0 && k > cfg.dataset_size)
    throw std::invalid_argument("minibatch exceeds dataset size");
  const long long samples = cfg.epochs * cfg.dataset_size;
  const long long iters = (samples + k - 1) / k;
  const double one = to_seconds(iteration_time(phases, k, model)) + cfg.delta_sync_s;
  return static_cast<double>(iters) * one;
}

// ref: perf_model.cpp:146-152
TimeNs transfer_time(const Gmap& gmap, const MemOp& op, int k,
                     const PerfModel& model, const PinSet& pins) {
  if (op.kind != MemOpKind::offload && op.kind != MemOpKind::prefetch)
    throw std::invalid_argument("transfer_time requires an offload or prefetch op");
  if (pins.count(op.object)) return 0;
  return transfer_duration(gmap.op_bytes(op, k), model.bandwidth_avail);
}

// model.json (ref: perf_model.cpp:154-198)
std::string perf_model_to_json(const PerfModel& model) {
  json doc;
  doc["format_version"] = 1;
  doc["k_base"] = model.k_base;
  doc["bandwidth_avail_bytes_per_s"] = model.bandwidth_avail;
  json curves = json::object();
  for (const auto& [type, c] : model.curves) {
    json knots = json::array();
    for (const auto& [x, y] : c.knots) knots.push_back(json::array({x, y}));
    json cj;
    cj["efficiency"] = c.efficiency;
    cj["plateau"] = c.plateau;
    cj["knots"] = std::move(knots);
    curves[type] = std::move(cj);
  }
  doc["curves"] = std::move(curves);
  return doc.dump(2) + "\n";
}

PerfModel perf_model_from_json(const std::string& text,
                               const std::string& origin) {
  json doc;
  try {
    doc = json::parse(text);
  } catch (const json::exception& e) {
    throw SpecError(origin + ": malformed JSON: " + e.what());
  }
  if (!doc.contains("format_version") || doc.at("format_version").get<int>() != 1)
    throw SpecError(origin + ": missing or unsupported format_version");
  PerfModel m;
  m.k_base = doc.at("k_base").get<int>();
  m.bandwidth_avail = doc.at("bandwidth_avail_bytes_per_s").get<double>();
  for (const auto& [type, cj] : doc.at("curves").items()) {
    ThroughputCurve c;
    c.layer_type = type;
    c.efficiency = cj.at("efficiency").get<double>();
    c.plateau = cj.at("plateau").get<double>();
    for (const json& kn : cj.at("knots"))
      c.knots.emplace_back(kn.at(0).get<Flops>(), kn.at(1).get<double>());
    if (c.knots.empty()) throw SpecError(origin + ": curve without knots");
    m.curves[type] = std::move(c);
  }
  if (m.curves.empty()) throw SpecError(origin + ": model without curves");
  return m;
}

// ---------------------------------------------------------------------------
// Learning-rate rule, Eq. 8/9 (ref: lr_tuner.cpp:8-31)
// ---------------------------------------------------------------------------
double adapted_learning_rate(const LrConfig& cfg) {
  const double ac = cfg.alpha_base * cfg.convexity;
  if (!(ac > 0.0) || ac >= 1.0)
    throw std::invalid_argument(
        "alpha_base * c must lie in (0, 1) for the contraction to hold");
  if (cfg.q < 1.0)
    throw std::invalid_argument("q < 1 (shrinking minibatch) is unsupported");
  if (cfg.q == 1.0) return cfg.alpha_base;  // bit-exact identity
  return (1.0 - std::pow(1.0 - ac, cfg.q)) / cfg.convexity;
}

double contraction_residual(const LrConfig& cfg, double alpha_star) {
  const double lhs_base = 1.0 - cfg.alpha_base * cfg.convexity * cfg.mu;
  const double rhs_base = 1.0 - alpha_star * cfg.convexity * cfg.mu;
  if (!(lhs_base > 0.0) || !(rhs_base > 0.0))
    throw std::invalid_argument("contraction bases must stay positive");
  if (cfg.iters_base <= 0)
    throw std::invalid_argument("iters_base must be positive");
  const double n = static_cast<double>(cfg.iters_base);
  return std::pow(lhs_base, n - 1.0) - std::pow(rhs_base, n / cfg.q - 1.0);
}

}  // namespace swapsched
