// ResNet op graphs, the network.json exporter and the lifetime model.
// See net.h for the mapping to the reference phase model.
#include "net.h"

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <cstdio>
#include <map>
#include <numeric>
#include <stdexcept>

#include <json.hpp>

namespace accudnn {

using nlohmann::json;

const char* op_kind_name(OpKind k) {
  switch (k) {
    case OpKind::conv: return "conv";
    case OpKind::bn: return "bn";
    case OpKind::bn_relu: return "bn_relu";
    case OpKind::relu: return "relu";
    case OpKind::add: return "add";
    case OpKind::maxpool: return "maxpool";
    case OpKind::avgpool: return "avgpool";
    case OpKind::fc: return "fc";
    case OpKind::xent: return "xent";
    case OpKind::bn_add_relu: return "bn_add_relu";
  }
  return "?";
}

namespace {

class Builder {
 public:
  Builder(Net& net) : net_(net) {}

  int conv(const std::string& name, int in, int cout, int k, int stride, int pad) {
    Op op;
    op.kind = OpKind::conv;
    op.name = name;
    op.in0 = in;
    const TensorShape si = in_shape(in);
    op.cin = si.c;
    op.cout = cout;
    op.r = op.s = k;
    op.stride = stride;
    op.pad = pad;
    TensorShape so{(si.h + 2 * pad - k) / stride + 1, (si.w + 2 * pad - k) / stride + 1, cout};
    return push(op, so);
  }
  int bn(const std::string& name, int in, bool relu) {
    Op op;
    op.kind = relu ? OpKind::bn_relu : OpKind::bn;
    op.name = name;
    op.in0 = in;
    op.channels = in_shape(in).c;
    return push(op, in_shape(in));
  }
  int bn_add_relu(const std::string& name, int in, int skip) {
    Op op;
    op.kind = OpKind::bn_add_relu;
    op.name = name;
    op.in0 = in;
    op.in1 = skip;
    op.channels = in_shape(in).c;
    return push(op, in_shape(in));
  }
  int relu(const std::string& name, int in) {
    Op op;
    op.kind = OpKind::relu;
    op.name = name;
    op.in0 = in;
    return push(op, in_shape(in));
  }
  int add(const std::string& name, int a, int b) {
    Op op;
    op.kind = OpKind::add;
    op.name = name;
    op.in0 = a;
    op.in1 = b;
    return push(op, in_shape(a));
  }
  int maxpool(const std::string& name, int in, int k, int stride, int pad) {
    Op op;
    op.kind = OpKind::maxpool;
    op.name = name;
    op.in0 = in;
    op.pk = k;
    op.pstride = stride;
    op.ppad = pad;
    const TensorShape si = in_shape(in);
    TensorShape so{(si.h + 2 * pad - k) / stride + 1, (si.w + 2 * pad - k) / stride + 1, si.c};
    return push(op, so);
  }
  int avgpool(const std::string& name, int in) {
    Op op;
    op.kind = OpKind::avgpool;
    op.name = name;
    op.in0 = in;
    return push(op, TensorShape{1, 1, in_shape(in).c});
  }
  int fc(const std::string& name, int in, int classes) {
    Op op;
    op.kind = OpKind::fc;
    op.name = name;
    op.in0 = in;
    op.cin = in_shape(in).c;
    op.cout = classes;
    return push(op, TensorShape{1, 1, classes});
  }
  int xent(const std::string& name, int in) {
    Op op;
    op.kind = OpKind::xent;
    op.name = name;
    op.in0 = in;
    return push(op, TensorShape{1, 1, 1});  // per-sample loss
  }

 private:
  TensorShape in_shape(int id) const {
    if (id == kImage) return TensorShape{net_.image, net_.image, net_.in_c4};
    return net_.shape.at(static_cast<size_t>(id));
  }
  int push(const Op& op, const TensorShape& s) {
    net_.ops.push_back(op);
    net_.shape.push_back(s);
    return static_cast<int>(net_.ops.size()) - 1;
  }
  Net& net_;
};

// torchvision v1.5 bottleneck (stride on the 3x3)
void imagenet_bottleneck(Net& net, const int (&blocks)[4]) {
  Builder b(net);
  int x = b.conv("stem.conv", kImage, 64, 7, 2, 3);
  x = b.bn("stem.bn", x, true);
  x = b.maxpool("stem.pool", x, 3, 2, 1);
  int cin = 64;
  for (int st = 0; st < 4; ++st) {
    const int width = 64 << st;
    for (int i = 0; i < blocks[st]; ++i) {
      const std::string p = "layer" + std::to_string(st + 1) + "." + std::to_string(i) + ".";
      const int stride = (i == 0 && st > 0) ? 2 : 1;
      const int in = x;
      int y = b.conv(p + "conv1", in, width, 1, 1, 0);
      y = b.bn(p + "bn1", y, true);
      y = b.conv(p + "conv2", y, width, 3, stride, 1);
      y = b.bn(p + "bn2", y, true);
      y = b.conv(p + "conv3", y, width * 4, 1, 1, 0);
      int sc = in;
      if (i == 0) {
        sc = b.conv(p + "downsample.conv", in, width * 4, 1, stride, 0);
        sc = b.bn(p + "downsample.bn", sc, false);
      }
      x = b.bn_add_relu(p + "bn3", y, sc);  // relu(bn3(conv3) + shortcut)
      cin = width * 4;
    }
  }
  (void)cin;
  x = b.avgpool("avgpool", x);
  x = b.fc("fc", x, net.classes);
  b.xent("loss", x);
}

// torchvision basic block (resnet18/34)
void imagenet_basic(Net& net, const int (&blocks)[4]) {
  Builder b(net);
  int x = b.conv("stem.conv", kImage, 64, 7, 2, 3);
  x = b.bn("stem.bn", x, true);
  x = b.maxpool("stem.pool", x, 3, 2, 1);
  int cin = 64;
  for (int st = 0; st < 4; ++st) {
    const int width = 64 << st;
    for (int i = 0; i < blocks[st]; ++i) {
      const std::string p = "layer" + std::to_string(st + 1) + "." + std::to_string(i) + ".";
      const int stride = (i == 0 && st > 0) ? 2 : 1;
      const int in = x;
      int y = b.conv(p + "conv1", in, width, 3, stride, 1);
      y = b.bn(p + "bn1", y, true);
      y = b.conv(p + "conv2", y, width, 3, 1, 1);
      int sc = in;
      if (stride != 1 || cin != width) {
        sc = b.conv(p + "downsample.conv", in, width, 1, stride, 0);
        sc = b.bn(p + "downsample.bn", sc, false);
      }
      x = b.bn_add_relu(p + "bn2", y, sc);  // relu(bn2(conv2) + shortcut)
      cin = width;
    }
  }
  x = b.avgpool("avgpool", x);
  x = b.fc("fc", x, net.classes);
  b.xent("loss", x);
}

// He et al. CIFAR ResNet (6n+2), basic blocks, projection shortcuts
void cifar_basic(Net& net, int n) {
  Builder b(net);
  int x = b.conv("stem.conv", kImage, 16, 3, 1, 1);
  x = b.bn("stem.bn", x, true);
  int cin = 16;
  for (int st = 0; st < 3; ++st) {
    const int width = 16 << st;
    for (int i = 0; i < n; ++i) {
      const std::string p = "stage" + std::to_string(st + 1) + "." + std::to_string(i) + ".";
      const int stride = (i == 0 && st > 0) ? 2 : 1;
      const int in = x;
      int y = b.conv(p + "conv1", in, width, 3, stride, 1);
      y = b.bn(p + "bn1", y, true);
      y = b.conv(p + "conv2", y, width, 3, 1, 1);
      int sc = in;
      if (stride != 1 || cin != width) {
        sc = b.conv(p + "shortcut.conv", in, width, 1, stride, 0);
        sc = b.bn(p + "shortcut.bn", sc, false);
      }
      x = b.bn_add_relu(p + "bn2", y, sc);  // relu(bn2(conv2) + shortcut)
      cin = width;
    }
  }
  x = b.avgpool("avgpool", x);
  x = b.fc("fc", x, net.classes);
  b.xent("loss", x);
}

// He et al. "Identity Mappings" pre-activation bottleneck (9n+2)
void cifar_preact(Net& net, int n) {
  Builder b(net);
  int x = b.conv("stem.conv", kImage, 16, 3, 1, 1);
  int cin = 16;
  for (int st = 0; st < 3; ++st) {
    const int width = 16 << st;
    for (int i = 0; i < n; ++i) {
      const std::string p = "stage" + std::to_string(st + 1) + "." + std::to_string(i) + ".";
      const int stride = (i == 0 && st > 0) ? 2 : 1;
      const int in = x;
      const int a = b.bn(p + "preact", in, true);
      int y = b.conv(p + "conv1", a, width, 1, 1, 0);
      y = b.bn(p + "bn2", y, true);
      y = b.conv(p + "conv2", y, width, 3, stride, 1);
      y = b.bn(p + "bn3", y, true);
      y = b.conv(p + "conv3", y, width * 4, 1, 1, 0);
      int sc = in;
      if (i == 0) sc = b.conv(p + "shortcut.conv", a, width * 4, 1, stride, 0);
      x = b.add(p + "add", y, sc);
      cin = width * 4;
    }
  }
  (void)cin;
  x = b.bn("final.bn", x, true);
  x = b.avgpool("avgpool", x);
  x = b.fc("fc", x, net.classes);
  b.xent("loss", x);
}

long long align4(long long v) { return (v + 3) & ~3LL; }

void finalize(Net& net) {
  const int n = net.num_ops();
  net.consumers.assign(static_cast<size_t>(n), {});
  for (int i = 0; i < n; ++i) {
    const Op& op = net.ops[static_cast<size_t>(i)];
    if (op.in0 >= 0) net.consumers[static_cast<size_t>(op.in0)].push_back(i);
    if (op.in1 >= 0) net.consumers[static_cast<size_t>(op.in1)].push_back(i);
  }
  // parameters laid out in reverse op order: backward produces gradients
  // from the front of the flat buffer, so all-reduce buckets are prefixes
  long long off = 0, stats = 0;
  for (int i = n - 1; i >= 0; --i) {
    Op& op = net.ops[static_cast<size_t>(i)];
    if (op.kind == OpKind::conv) {
      op.w_off = off;
      off = align4(off + static_cast<long long>(op.cout) * op.r * op.s * op.cin);
    } else if (op.kind == OpKind::fc) {
      op.w_off = off;
      off = align4(off + static_cast<long long>(op.cout) * op.cin);
      op.b_off = off;
      off = align4(off + op.cout);
    } else if (is_bn(op.kind)) {
      op.g_off = off;
      off = align4(off + op.channels);
      op.beta_off = off;
      off = align4(off + op.channels);
      op.stat_off = stats;
      stats += 4LL * op.channels;
      net.max_bn_channels = std::max(net.max_bn_channels, op.channels);
    }
  }
  net.n_params = align4(off);
  net.n_stats = stats;
}

}  // namespace

Net build_net(const std::string& arch, int image, int classes, int recompute) {
  Net net;
  net.arch = arch;
  net.image = image;
  net.classes = classes;
  if (classes <= 0 || (classes & 3))
    throw std::invalid_argument("classes must be a positive multiple of 4");
  static const std::map<std::string, std::vector<int>> bottleneck = {
      {"resnet50", {3, 4, 6, 3}}, {"resnet101", {3, 4, 23, 3}}, {"resnet152", {3, 8, 36, 3}}};
  static const std::map<std::string, std::vector<int>> basic = {{"resnet18", {2, 2, 2, 2}},
                                                                {"resnet34", {3, 4, 6, 3}}};
  if (auto it = bottleneck.find(arch); it != bottleneck.end()) {
    const int b[4] = {it->second[0], it->second[1], it->second[2], it->second[3]};
    imagenet_bottleneck(net, b);
  } else if (auto it2 = basic.find(arch); it2 != basic.end()) {
    const int b[4] = {it2->second[0], it2->second[1], it2->second[2], it2->second[3]};
    imagenet_basic(net, b);
  } else if (arch.rfind("resnet", 0) == 0) {
    const int depth = std::atoi(arch.c_str() + 6);
    if (depth >= 8 && (depth - 2) % 6 == 0 && depth < 164) {
      cifar_basic(net, (depth - 2) / 6);
    } else if (depth >= 11 && (depth - 2) % 9 == 0) {
      cifar_preact(net, (depth - 2) / 9);
    } else {
      throw std::invalid_argument("unsupported ResNet depth: " + arch);
    }
  } else {
    throw std::invalid_argument("unknown architecture: " + arch);
  }
  finalize(net);
  if (recompute < 0) {
    // default off (ACCUDNN_RECOMPUTE=1 turns it on).  Measured on ResNet-152
    // at 8 GiB: k* 42 -> 50 but 2360 -> 2245 img/s -- the recompute pass costs
    // as much as storing (one read + one write of the tensor) and lands on the
    // weight-gradient stream, which the critical path already waits for.  Not
    // for the CIFAR nets either way: their layer-wise memory peak of the
    // all-swapped model would fall on a transient phase, which holds no
    // featuremap bytes, and the reference's k_max formula rejects such a spec
    // (planner.cpp:232-234)
    const char* e = std::getenv("ACCUDNN_RECOMPUTE");
    recompute = e ? std::atoi(e) : 0;
  }
  if (recompute)
    for (int t = 0; t < net.num_ops(); ++t) {
      Op& op = net.ops[static_cast<size_t>(t)];
      const auto& cons = net.consumers[static_cast<size_t>(t)];
      if (op.kind == OpKind::bn_relu && cons.size() == 1 &&
          net.ops[static_cast<size_t>(cons[0])].kind == OpKind::conv) {
        op.transient = true;
        op.transient_reader = cons[0];
      }
    }
  return net;
}

bool bwd_reads_input(const Op& op) {
  switch (op.kind) {
    case OpKind::conv:
    case OpKind::fc:
    case OpKind::bn:
    case OpKind::bn_relu:
    case OpKind::bn_add_relu:  // reads both inputs (BN input + the shortcut, for the mask)
    case OpKind::relu:
    case OpKind::maxpool:
    case OpKind::xent:
      return true;
    case OpKind::add:
    case OpKind::avgpool:
      return false;
  }
  return false;
}

// ---------------------------------------------------------------------------
// lifetime model
// ---------------------------------------------------------------------------
namespace {

long long round_up(long long v, long long a) { return a > 1 ? (v + a - 1) / a * a : v; }

}  // namespace

LifetimeModel build_lifetimes(const Net& net, int k, const std::vector<char>& swapped,
                              int lookahead, long long align) {
  const int n = net.num_ops();
  LifetimeModel lm;
  lm.n = n;
  lm.act_inst.assign(static_cast<size_t>(n), -1);
  lm.pre_inst.assign(static_cast<size_t>(n), -1);
  lm.grad_inst.assign(static_cast<size_t>(n), -1);
  lm.grad_first_writer.assign(static_cast<size_t>(n), -1);

  auto bytes_of = [&](int t) {
    return round_up(4LL * k * net.shape[static_cast<size_t>(t)].per_image(), align);
  };

  // ---- activations ----
  for (int t = 0; t < n; ++t) {
    int last_fwd = fwd_step(t), first_bwd = 1 << 30, last_bwd = -1;
    for (int c : net.consumers[static_cast<size_t>(t)]) {
      last_fwd = std::max(last_fwd, fwd_step(c));
      const Op& oc = net.ops[static_cast<size_t>(c)];
      if (bwd_reads_input(oc)) {
        first_bwd = std::min(first_bwd, bwd_step(c, n));
        last_bwd = std::max(last_bwd, bwd_step(c, n));
      }
      // a transient consumer is recomputed from this tensor in its reader's backward
      if (oc.transient) {
        first_bwd = std::min(first_bwd, bwd_step(oc.transient_reader, n));
        last_bwd = std::max(last_bwd, bwd_step(oc.transient_reader, n));
      }
    }
    const Op& ot = net.ops[static_cast<size_t>(t)];
    if (ot.transient) {
      Instance a;
      a.kind = InstKind::act;
      a.tensor = t;
      a.bytes = bytes_of(t);
      a.first = fwd_step(t);
      a.last = last_fwd;
      lm.act_inst[static_cast<size_t>(t)] = static_cast<int>(lm.inst.size());
      lm.inst.push_back(a);
      Instance r = a;
      r.kind = InstKind::act_recomputed;
      r.first = r.last = bwd_step(ot.transient_reader, n);
      lm.pre_inst[static_cast<size_t>(t)] = static_cast<int>(lm.inst.size());
      lm.inst.push_back(r);
      continue;
    }
    // GMAP prefetch / release phase of fm_{t+1} (1-based) = 2N - t
    const int gmap_phase = 2 * n - t;
    Instance a;
    a.kind = InstKind::act;
    a.tensor = t;
    a.bytes = bytes_of(t);
    a.first = fwd_step(t);
    const bool sw = !swapped.empty() && swapped[static_cast<size_t>(t)];
    a.swapped = sw;
    if (!sw) {
      a.last = std::max(last_fwd, last_bwd);
      lm.act_inst[static_cast<size_t>(t)] = static_cast<int>(lm.inst.size());
      lm.inst.push_back(a);
    } else {
      a.last = last_fwd;
      lm.act_inst[static_cast<size_t>(t)] = static_cast<int>(lm.inst.size());
      lm.inst.push_back(a);
      Instance p;
      p.kind = InstKind::act_prefetched;
      p.tensor = t;
      p.bytes = a.bytes;
      const int need = std::min(gmap_phase, first_bwd);
      p.first = std::max(n + 1, need - lookahead);
      p.last = std::max(gmap_phase, last_bwd);
      lm.pre_inst[static_cast<size_t>(t)] = static_cast<int>(lm.inst.size());
      lm.inst.push_back(p);
    }
  }

  // ---- gradients ----
  // Writers of G_t: the backward of every consumer of t; reader: the
  // backward of op t.  The loss output has no gradient buffer.  An add's
  // output gradient is passed through to its inputs by aliasing their
  // gradient buffers into one group when that is exact: for every reading
  // member r of a group, every writer into the group that runs before r's
  // backward (op index > r) must be a consumer of r.  Otherwise the add
  // copies.
  std::vector<char> has_grad(static_cast<size_t>(n), 0);
  for (int t = 0; t < n; ++t)
    has_grad[static_cast<size_t>(t)] = net.ops[static_cast<size_t>(t)].kind != OpKind::xent &&
                                       !net.consumers[static_cast<size_t>(t)].empty();
  std::vector<int> group(static_cast<size_t>(n));
  std::iota(group.begin(), group.end(), 0);
  std::map<int, std::vector<int>> members;
  for (int t = 0; t < n; ++t) members[t] = {t};
  auto is_pass_through = [&](int o, int m, const std::vector<int>& grp) {
    return net.ops[static_cast<size_t>(o)].kind == OpKind::add &&
           grp[static_cast<size_t>(o)] == grp[static_cast<size_t>(m)];
  };
  // ops whose backward contributes to G_r: non-pass-through consumers of r,
  // and (recursively) the contributors of pass-through adds consuming r
  std::function<void(int, const std::vector<int>&, std::vector<int>&)> contributors =
      [&](int r, const std::vector<int>& grp, std::vector<int>& out) {
        for (int c : net.consumers[static_cast<size_t>(r)]) {
          if (is_pass_through(c, r, grp))
            contributors(c, grp, out);
          else
            out.push_back(c);
        }
      };
  auto group_ok = [&](const std::vector<int>& mem, const std::vector<int>& grp) {
    std::vector<int> writers;
    for (int m : mem)
      for (int o : net.consumers[static_cast<size_t>(m)])
        if (!is_pass_through(o, m, grp)) writers.push_back(o);
    std::sort(writers.begin(), writers.end());
    writers.erase(std::unique(writers.begin(), writers.end()), writers.end());
    for (int r : mem) {
      std::vector<int> want;
      contributors(r, grp, want);
      std::sort(want.begin(), want.end());
      want.erase(std::unique(want.begin(), want.end()), want.end());
      std::vector<int> seen;
      for (int w : writers)
        if (w > r) seen.push_back(w);
      if (seen != want) return false;
    }
    return true;
  };
  for (int c = 0; c < n; ++c) {
    const Op& op = net.ops[static_cast<size_t>(c)];
    if (op.kind != OpKind::add || !has_grad[static_cast<size_t>(c)]) continue;
    for (int x : {op.in0, op.in1}) {
      if (x < 0 || !has_grad[static_cast<size_t>(x)]) continue;
      const int gx = group[static_cast<size_t>(x)], gc = group[static_cast<size_t>(c)];
      if (gx == gc) continue;
      std::vector<int> grp = group;
      std::vector<int> merged = members[gc];
      for (int m : members[gx]) {
        grp[static_cast<size_t>(m)] = gc;
        merged.push_back(m);
      }
      if (group_ok(merged, grp)) {
        group = std::move(grp);
        members[gc] = std::move(merged);
        members.erase(gx);
      }
    }
  }
  std::map<int, int> group_inst;
  for (int t = 0; t < n; ++t) {
    if (!has_grad[static_cast<size_t>(t)]) continue;
    const int g = group[static_cast<size_t>(t)];
    int first_w = 1 << 30;
    const int reader = bwd_step(t, n);
    for (int c : net.consumers[static_cast<size_t>(t)]) first_w = std::min(first_w, bwd_step(c, n));
    auto it = group_inst.find(g);
    if (it == group_inst.end()) {
      Instance gi;
      gi.kind = InstKind::grad;
      gi.tensor = g;
      gi.bytes = bytes_of(t);
      gi.first = first_w;
      gi.last = reader;
      group_inst[g] = static_cast<int>(lm.inst.size());
      lm.inst.push_back(gi);
    } else {
      Instance& gi = lm.inst[static_cast<size_t>(it->second)];
      gi.first = std::min(gi.first, first_w);
      gi.last = std::max(gi.last, reader);
      gi.bytes = std::max(gi.bytes, bytes_of(t));
    }
    lm.grad_inst[static_cast<size_t>(t)] = group_inst[g];
  }
  // first writer (beta = 0) of every group: the writer that runs first in
  // the backward pass, i.e. the largest op index; pass-through adds and the
  // stem's missing data gradient do not write
  std::map<int, int> first;  // group -> op
  for (int c = 0; c < n; ++c) {
    const Op& op = net.ops[static_cast<size_t>(c)];
    for (int x : {op.in0, op.in1}) {
      if (x < 0 || !has_grad[static_cast<size_t>(x)]) continue;
      if (is_pass_through(c, x, group)) continue;
      const int g = group[static_cast<size_t>(x)];
      auto it = first.find(g);
      if (it == first.end() || c > it->second) first[g] = c;
    }
  }
  for (int t = 0; t < n; ++t)
    if (has_grad[static_cast<size_t>(t)]) {
      auto it = first.find(group[static_cast<size_t>(t)]);
      lm.grad_first_writer[static_cast<size_t>(t)] = it == first.end() ? -1 : it->second;
    }
  lm.grad_group = group;

  // ---- live bytes per step ----
  lm.live.assign(static_cast<size_t>(2 * n + 2), 0);
  for (const Instance& in : lm.inst)
    for (int s = in.first; s <= in.last; ++s) lm.live[static_cast<size_t>(s)] += in.bytes;
  lm.peak_bytes = *std::max_element(lm.live.begin(), lm.live.end());
  return lm;
}

void schedule_prefetches(const Net& net, LifetimeModel& lm, long long cap) {
  const int n = lm.n;
  // GMAP order of the prefetches: fm_{t+1} is prefetched in phase 2N - t,
  // so larger t first
  std::vector<int> order;
  for (int t = n - 1; t >= 0; --t) {
    const int pid = lm.pre_inst[static_cast<size_t>(t)];
    if (pid >= 0 && lm.inst[static_cast<size_t>(pid)].kind == InstKind::act_prefetched)
      order.push_back(t);
  }
  int prev_first = 1;
  for (int t : order) {
    Instance& p = lm.inst[static_cast<size_t>(lm.pre_inst[static_cast<size_t>(t)])];
    const Instance& a = lm.inst[static_cast<size_t>(lm.act_inst[static_cast<size_t>(t)])];
    // forward readers use the primary copy: the prefetched one may only
    // start after them (and after the producer, whose offload it reloads)
    const int lo = std::max({prev_first, a.last + 1, fwd_step(t) + 1});
    int s = p.first;
    while (s - 1 >= lo && lm.live[static_cast<size_t>(s - 1)] + p.bytes <= cap) {
      --s;
      lm.live[static_cast<size_t>(s)] += p.bytes;
    }
    p.first = s;
    prev_first = std::max(prev_first, s);
  }
  // a prefetch whose first backward reader comes before its GMAP phase (a
  // block input also read by the downsample convolution) may still start
  // before its queue predecessors: pull those earlier where the pool has
  // room, so the swap-in stream issues in GMAP order
  for (size_t i = order.size(); i-- > 1;) {
    Instance& p = lm.inst[static_cast<size_t>(lm.pre_inst[static_cast<size_t>(order[i - 1])])];
    const Instance& q = lm.inst[static_cast<size_t>(lm.pre_inst[static_cast<size_t>(order[i])])];
    const Instance& a = lm.inst[static_cast<size_t>(lm.act_inst[static_cast<size_t>(order[i - 1])])];
    const int lo = std::max(a.last + 1, fwd_step(order[i - 1]) + 1);
    if (q.first >= p.first || q.first < lo) continue;
    bool fits = true;
    for (int s = q.first; s < p.first; ++s)
      fits = fits && lm.live[static_cast<size_t>(s)] + p.bytes <= cap;
    if (!fits) continue;
    for (int s = q.first; s < p.first; ++s) lm.live[static_cast<size_t>(s)] += p.bytes;
    p.first = q.first;
  }
  (void)net;
  lm.peak_bytes = *std::max_element(lm.live.begin(), lm.live.end());
}

long long plan_arena(LifetimeModel& lm) {
  std::vector<int> order(lm.inst.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const Instance& x = lm.inst[static_cast<size_t>(a)];
    const Instance& y = lm.inst[static_cast<size_t>(b)];
    if (x.bytes != y.bytes) return x.bytes > y.bytes;
    return x.first < y.first;
  });
  std::vector<int> placed;
  long long arena = 0;
  for (int id : order) {
    Instance& x = lm.inst[static_cast<size_t>(id)];
    std::vector<std::pair<long long, long long>> busy;
    const int xl = std::max(x.last, x.pack_last);
    for (int p : placed) {
      const Instance& y = lm.inst[static_cast<size_t>(p)];
      if (y.first <= xl && x.first <= std::max(y.last, y.pack_last))
        busy.emplace_back(y.offset, y.offset + y.bytes);
    }
    std::sort(busy.begin(), busy.end());
    long long off = 0;
    for (const auto& [lo, hi] : busy) {
      if (off + x.bytes <= lo) break;
      off = std::max(off, hi);
    }
    x.offset = off;
    arena = std::max(arena, off + x.bytes);
    placed.push_back(id);
  }
  return arena;
}

// ---------------------------------------------------------------------------
// exporter
// ---------------------------------------------------------------------------
namespace {

struct OpCost {
  double fwd = 0, bwd = 0;  // FLOPs per image
  long long params = 0;
};

OpCost op_cost(const Net& net, int i) {
  const Op& op = net.ops[static_cast<size_t>(i)];
  const TensorShape& so = net.shape[static_cast<size_t>(i)];
  const double out = static_cast<double>(so.per_image());
  OpCost c;
  switch (op.kind) {
    case OpKind::conv: {
      c.fwd = 2.0 * so.h * so.w * op.cout * op.cin * op.r * op.s;
      c.bwd = (op.in0 == kImage ? 1.0 : 2.0) * c.fwd;
      c.params = static_cast<long long>(op.cout) * op.r * op.s * op.cin;
      break;
    }
    case OpKind::fc:
      c.fwd = 2.0 * op.cin * op.cout;
      c.bwd = 2.0 * c.fwd;
      c.params = static_cast<long long>(op.cout) * op.cin + op.cout;
      break;
    case OpKind::bn: c.fwd = 8 * out; c.bwd = 12 * out; c.params = 2LL * op.channels; break;
    case OpKind::bn_relu: c.fwd = 9 * out; c.bwd = 13 * out; c.params = 2LL * op.channels; break;
    case OpKind::bn_add_relu:
      c.fwd = 10 * out;
      c.bwd = 14 * out;
      c.params = 2LL * op.channels;
      break;
    case OpKind::relu: c.fwd = out; c.bwd = out; break;
    case OpKind::add: c.fwd = out; c.bwd = out; break;
    case OpKind::maxpool: c.fwd = out * op.pk * op.pk; c.bwd = 2 * c.fwd; break;
    case OpKind::avgpool: {
      const int in = op.in0;
      const double inn = static_cast<double>(net.shape[static_cast<size_t>(in)].per_image());
      c.fwd = inn;
      c.bwd = inn;
      break;
    }
    case OpKind::xent: c.fwd = 5.0 * net.classes; c.bwd = 5.0 * net.classes; break;
  }
  return c;
}

const char* layer_type_of(OpKind k, const char** tag) {
  *tag = nullptr;
  switch (k) {
    case OpKind::conv: return "conv";
    case OpKind::fc: return "fc";
    case OpKind::bn:
    case OpKind::bn_relu: return "bn";
    case OpKind::relu: return "activation";
    case OpKind::maxpool:
    case OpKind::avgpool: return "pooling";
    case OpKind::add: *tag = "eltwise"; return "other";
    case OpKind::xent: *tag = "loss"; return "other";
    case OpKind::bn_add_relu: *tag = "bn_add_relu"; return "other";
  }
  return "other";
}

}  // namespace

std::string export_network_json(const Net& net, int k_base, int lookahead) {
  const int n = net.num_ops();
  // worst case: every featuremap swapped; align 1 so the accounting is exact
  const std::vector<char> all(static_cast<size_t>(n), 1);
  const LifetimeModel lm = build_lifetimes(net, k_base, all, lookahead, 1);
  // bytes of the GMAP-resident featuremap at each step
  auto fm_bytes = [&](int t) {
    return net.ops[static_cast<size_t>(t)].transient
               ? 0LL
               : 4LL * k_base * net.shape[static_cast<size_t>(t)].per_image();
  };
  std::vector<long long> extra(static_cast<size_t>(2 * n + 2), 0);
  for (int s = 1; s <= 2 * n; ++s) {
    const int t = s <= n ? s - 1 : (2 * n + 1 - s) - 1;  // layer l -> tensor l-1
    extra[static_cast<size_t>(s)] = lm.live[static_cast<size_t>(s)] - fm_bytes(t);
  }

  json doc;
  doc["format_version"] = 1;
  doc["name"] = net.arch + "@" + std::to_string(net.image);
  doc["k_base"] = k_base;
  doc["backward_flops_factor"] = 2.0;
  json layers = json::array();
  for (int l = 1; l <= n; ++l) {
    const int op = l - 1;
    const OpCost own = op_cost(net, op);
    double bwd = (op + 1 < n) ? op_cost(net, op + 1).bwd : 0.0;  // shift-by-one
    if (op == 0) bwd += own.bwd;
    const char* tag = nullptr;
    const char* type = layer_type_of(net.ops[static_cast<size_t>(op)].kind, &tag);
    json lj;
    lj["index"] = l;
    lj["layer_type"] = type;
    if (tag) lj["type_tag"] = tag;
    lj["flops_fwd_base"] = static_cast<unsigned long long>(std::llround(own.fwd * k_base));
    lj["flops_bwd_base"] =
        static_cast<unsigned long long>(std::max<long long>(1, std::llround(bwd * k_base)));
    lj["featuremap_bytes_base"] = static_cast<unsigned long long>(fm_bytes(op));
    lj["param_bytes"] = static_cast<unsigned long long>(4 * own.params);
    lj["grad_bytes"] = static_cast<unsigned long long>(4 * own.params);
    const long long ws = std::max(extra[static_cast<size_t>(fwd_step(op))],
                                  extra[static_cast<size_t>(2 * n + 1 - l)]);
    lj["workspace_bytes_base"] = static_cast<unsigned long long>(std::max<long long>(0, ws));
    lj["op"] = net.ops[static_cast<size_t>(op)].name;  // informational key
    layers.push_back(std::move(lj));
  }
  doc["num_layers"] = n;
  doc["layers"] = std::move(layers);
  return doc.dump(2) + "\n";
}

std::string describe_net_json(const Net& net) {
  json doc;
  doc["arch"] = net.arch;
  doc["image"] = net.image;
  doc["in_channels"] = net.in_c;
  doc["in_channels_padded"] = net.in_c4;
  doc["classes"] = net.classes;
  doc["n_params"] = net.n_params;
  doc["n_stats"] = net.n_stats;
  json ops = json::array();
  for (int i = 0; i < net.num_ops(); ++i) {
    const Op& op = net.ops[static_cast<size_t>(i)];
    const TensorShape& s = net.shape[static_cast<size_t>(i)];
    json o;
    o["id"] = i;
    o["kind"] = op_kind_name(op.kind);
    o["name"] = op.name;
    o["in0"] = op.in0;
    o["in1"] = op.in1;
    o["out"] = {s.h, s.w, s.c};
    if (op.kind == OpKind::conv || op.kind == OpKind::fc) {
      o["cin"] = op.cin;
      o["cout"] = op.cout;
      o["r"] = op.r;
      o["stride"] = op.stride;
      o["pad"] = op.pad;
      o["w_off"] = op.w_off;
      if (op.b_off >= 0) o["b_off"] = op.b_off;
    }
    if (is_bn(op.kind)) {
      o["channels"] = op.channels;
      o["g_off"] = op.g_off;
      o["beta_off"] = op.beta_off;
      o["stat_off"] = op.stat_off;
      if (op.transient) o["transient"] = true;
    }
    if (op.kind == OpKind::maxpool) {
      o["k"] = op.pk;
      o["stride"] = op.pstride;
      o["pad"] = op.ppad;
    }
    ops.push_back(std::move(o));
  }
  doc["ops"] = std::move(ops);
  return doc.dump() + "\n";
}

}  // namespace accudnn
