// Seeded synthetic instances: `swapsched gen` and the parity fixtures.
//
// Contract: /root/reference/proj/src/synthetic.cpp:12-195 with
// include/swapsched/synthetic.hpp:13-56.  The splitmix64 output stream and
// the order in which draws are consumed are part of the fixture contract
// (synthetic.cpp:14), so a seed gives byte-identical documents to the
// reference; everything else is organised differently here:
//  * the RNG is a counter (state advances by the golden gamma) followed by a
//    table-driven finaliser;
//  * a layer is drawn as a fixed record of raw draws (LayerDraws) and then
//    materialised, so the draw order is visible in one place;
//  * per-type throughput curves are drawn lazily on the first phase of each
//    type key; the profile grid helper is shared by compute and transfer rows;
//  * CSV rows are formatted with one snprintf per row.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <unordered_map>

#include "swapsched/api.hpp"

namespace swapsched {
namespace {

constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ull;

// splitmix64 finaliser: two xor-shift-multiply rounds and a final xor-shift
constexpr std::uint64_t finalise(std::uint64_t z) {
  constexpr struct {
    int shift;
    std::uint64_t mul;
  } rounds[] = {{30, 0xbf58476d1ce4e5b9ull}, {27, 0x94d049bb133111ebull}};
  for (const auto& r : rounds) z = (z ^ (z >> r.shift)) * r.mul;
  return z ^ (z >> 31);
}

}  // namespace

std::uint64_t Rng::next() { return finalise(state += kGamma); }

std::int64_t Rng::range(std::int64_t lo, std::int64_t hi) {
  if (hi <= lo) return lo;
  const std::uint64_t width = static_cast<std::uint64_t>(hi - lo) + 1;
  return lo + static_cast<std::int64_t>(next() % width);
}

double Rng::uniform(double lo, double hi) {
  // top 53 bits scaled by 2^-53: a uniform double in [0, 1)
  const double unit = std::ldexp(static_cast<double>(next() >> 11), -53);
  return lo + unit * (hi - lo);
}

namespace {

// Raw draws for one synthetic layer, in consumption order.
struct LayerDraws {
  std::int64_t featuremap_granules;  // 4096..65536   (2..32 MiB)
  std::int64_t workspace_granules;   // 1024..8192    (0.5..4 MiB)
  std::int64_t param_granules;       // 0..4096       (<= 2 MiB)
  double compute_transfer_ratio;
  double backward_factor;            // 1.5..2.5 x forward FLOPs
};

LayerType synthetic_type(int index, int n) {
  static const char* const cycle[] = {"conv", "bn", "activation", "conv", "pooling"};
  return *layer_type_from(index == n ? "fc" : cycle[(index - 1) % 5]);
}

LayerDecl materialise(int index, int n, const LayerDraws& d, double nominal_rate,
                      double nominal_bw) {
  LayerDecl l;
  l.index = index;
  l.layer_type = synthetic_type(index, n);
  l.featuremap_bytes_base = static_cast<Bytes>(d.featuremap_granules) * kAlignGranule;
  l.workspace_bytes_base = static_cast<Bytes>(d.workspace_granules) * kAlignGranule;
  l.param_bytes = static_cast<Bytes>(d.param_granules) * kAlignGranule;
  l.grad_bytes = l.param_bytes;
  const double fwd = d.compute_transfer_ratio *
                     static_cast<double>(l.featuremap_bytes_base) * nominal_rate /
                     nominal_bw;
  l.flops_fwd_base = static_cast<Flops>(std::llround(fwd < 1e6 ? 1e6 : fwd));
  l.flops_bwd_base = static_cast<Flops>(
      std::llround(d.backward_factor * static_cast<double>(l.flops_fwd_base)));
  return l;
}

// 1/8, 1/4, 1/2, 2/3, 1 x k_ref, rounded, >= 1, first occurrence order
std::vector<int> profiling_grid(int k_ref) {
  static const double fractions[] = {0.125, 0.25, 0.5, 2.0 / 3.0, 1.0};
  std::vector<int> ks;
  for (double f : fractions) {
    const int k = static_cast<int>(std::max(1LL, std::llround(f * k_ref)));
    if (std::find(ks.begin(), ks.end(), k) == ks.end()) ks.push_back(k);
  }
  return ks;
}

std::string fmt_g12(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.12g", v);
  return b;
}

}  // namespace

NetworkSpec generate_network(Rng& rng, const SyntheticOptions& opts) {
  const int n = static_cast<int>(rng.range(opts.min_layers, opts.max_layers));
  NetworkSpec net;
  net.name = "synthetic-" + std::to_string(n);
  net.num_layers = n;
  net.k_base = rng.range(0, 1) != 0 ? 8 : 4;
  net.backward_flops_factor = 2.0;
  // nominal saturation rate: sizes FLOPs against the mid-band transfer time
  const double nominal_rate = rng.uniform(2e12, 6e12);
  const double nominal_bw = (opts.bandwidth_lo + opts.bandwidth_hi) / 2.0;
  net.layers.reserve(static_cast<size_t>(n));
  for (int i = 1; i <= n; ++i) {
    LayerDraws d;
    d.featuremap_granules = rng.range(4096, 65536);
    d.workspace_granules = rng.range(1024, 8192);
    d.param_granules = rng.range(0, 4096);
    d.compute_transfer_ratio =
        rng.uniform(opts.min_compute_transfer_ratio, opts.max_compute_transfer_ratio);
    d.backward_factor = rng.uniform(1.5, 2.5);
    net.layers.push_back(materialise(i, n, d, nominal_rate, nominal_bw));
  }
  return net;
}

ProfileSet generate_profiles(const NetworkSpec& net, Rng& rng, int k_ref,
                             double bandwidth) {
  const std::vector<PhaseLayer> phases = unfold_network(net);
  const Gmap gmap = build_gmap(phases, net);

  // rate(f) = plateau * f / (f + half), one curve per type key
  struct Curve {
    double plateau, half;
  };
  std::unordered_map<std::string, Curve> curves;
  for (const PhaseLayer& p : phases) {
    if (curves.find(p.type_key) != curves.end()) continue;
    const double plateau = rng.uniform(2e12, 8e12);
    const double half = rng.uniform(0.5, 3.0) * static_cast<double>(p.flops_base);
    curves.emplace(p.type_key, Curve{plateau, half});
  }
  std::vector<const MemOp*> offloads;
  for (const MemOp& op : gmap.ops)
    if (op.kind == MemOpKind::offload) offloads.push_back(&op);

  ProfileSet set;
  for (int k : profiling_grid(k_ref)) {
    for (const PhaseLayer& p : phases) {
      const Curve& c = curves.at(p.type_key);
      const Flops f = scale_flops(p, k, net.k_base);
      const double fd = static_cast<double>(f);
      set.compute_samples.push_back(
          ComputeSample{k, p.phase_index, p.type_key, f, fd / (c.plateau * fd / (fd + c.half))});
    }
    for (const MemOp* op : offloads) {
      const Bytes b = gmap.op_bytes(*op, k);
      set.transfer_samples.push_back(
          TransferSample{k, op->sequence_no, b, static_cast<double>(b) / bandwidth});
    }
    set.sampled_minibatches.insert(k);
  }
  return set;
}

SyntheticInstance generate_instance(std::uint64_t seed, const SyntheticOptions& opts) {
  Rng rng(seed);
  SyntheticInstance inst;
  inst.network = generate_network(rng, opts);
  inst.true_bandwidth = rng.uniform(opts.bandwidth_lo, opts.bandwidth_hi);

  HardwareSpec& hw = inst.hardware;
  hw.m_others = static_cast<Bytes>(rng.range(8192, 65536)) * kAlignGranule;  // 4..32 MiB
  hw.delta_sync_s = 0.0;
  hw.pcie_nominal = inst.true_bandwidth;

  // budget = fixed + peak(k=1, nothing pinned)
  //        + frac * (all-pinned peak at 8 k_base - peak(k=1))
  const Gmap gmap = build_gmap(unfold_network(inst.network), inst.network);
  const Bytes floor_peak = peak_layerwise_memory(gmap, 1, {}).peak_bytes;
  const auto ids = gmap.featuremap_ids();
  const PinSet everything(ids.begin(), ids.end());
  const Bytes ceiling_peak =
      peak_layerwise_memory(gmap, 8 * inst.network.k_base, everything).peak_bytes;
  const double frac = rng.uniform(opts.budget_frac_lo, opts.budget_frac_hi);
  hw.memory_budget = hw.m_others + inst.network.param_grad_bytes_total() + floor_peak +
                     static_cast<Bytes>(frac * static_cast<double>(ceiling_peak - floor_peak));

  const KmaxResult km = max_trainable_minibatch(gmap, inst.network, hw);
  const int k_ref = km.trainable && km.k_max > 2 ? km.k_max : 2;
  inst.profiles = generate_profiles(inst.network, rng, k_ref, inst.true_bandwidth);
  return inst;
}

std::string compute_profile_csv(const std::vector<ComputeSample>& samples) {
  std::string out = "minibatch,phase,layer_type,flops,time_s\n";
  for (const ComputeSample& s : samples)
    out += std::to_string(s.minibatch) + ',' + std::to_string(s.phase) + ',' +
           s.layer_type + ',' + std::to_string(s.flops) + ',' + fmt_g12(s.time_s) + '\n';
  return out;
}

std::string transfer_profile_csv(const std::vector<TransferSample>& samples) {
  std::string out = "minibatch,seq_no,bytes,time_s\n";
  for (const TransferSample& s : samples)
    out += std::to_string(s.minibatch) + ',' + std::to_string(s.seq_no) + ',' +
           std::to_string(s.bytes) + ',' + fmt_g12(s.time_s) + '\n';
  return out;
}

}  // namespace swapsched
