// ResNet op graphs for the B200 training step, the reference-format
// network.json exporter, and the real-lifetime memory model shared by the
// exporter (workspace accounting) and the executor (static arena plan).
//
// Mapping to the reference's phase model (model_ir.cpp:238-358):
//   * one LayerDecl per executed op (conv, bn[+relu], relu, pooling, fc,
//     other:eltwise for residual adds, other:loss for softmax-xent);
//     featuremap fm_l = the output tensor of op l;
//   * "shift-by-one": backward phase 2N+1-l executes the backward of op
//     l+1, whose input fm_l is exactly the featuremap the GMAP prefetches
//     there; phase N+1 is empty and phase 2N also runs op 1's backward;
//   * every byte the executor holds besides the GMAP-resident featuremap of
//     a phase (deferred frees of inputs read while their offload drains,
//     skip tensors, gradient buffers, early prefetches of non-adjacent
//     inputs) is charged to that layer's workspace_bytes_base, computed
//     from the executor's own lifetime model with every featuremap swapped
//     (the worst case), so that real device usage <= the planner's peak for
//     any pin set the planner returns.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace accudnn {

// bn_add_relu: y = relu(bn(in0) + in1), the residual tail of a ResNet block
// as one op (its only output is the block output; bn(in0) and the sum are
// never materialised)
enum class OpKind : int { conv, bn, bn_relu, relu, add, maxpool, avgpool, fc, xent, bn_add_relu };
inline bool is_bn(OpKind k) {
  return k == OpKind::bn || k == OpKind::bn_relu || k == OpKind::bn_add_relu;
}
const char* op_kind_name(OpKind k);

constexpr int kImage = -2;  // "input" id of the network input batch

struct Op {
  OpKind kind = OpKind::conv;
  std::string name;
  int in0 = -1, in1 = -1;  // producing op ids (tensor id == op id), kImage
  // conv / fc
  int cin = 0, cout = 0, r = 1, s = 1, stride = 1, pad = 0;
  long long w_off = -1, b_off = -1;  // offsets (floats) into the flat params
  // batch norm
  int channels = 0;
  long long g_off = -1, beta_off = -1;
  long long stat_off = -1;  // [mean C][invstd C][running_mean C][running_var C]
  // pooling window
  int pk = 0, pstride = 1, ppad = 0;
  // bn_relu whose only consumer is a convolution: its output is transient
  // (lives from its forward to the conv's forward) and is recomputed from the
  // BN input and the saved statistics right before the conv's weight
  // gradient; its featuremap in the planner's model is 0 bytes
  bool transient = false;
  int transient_reader = -1;  // the consuming conv
};

struct TensorShape {
  int h = 0, w = 0, c = 0;  // per image
  long long per_image() const { return static_cast<long long>(h) * w * c; }
};

struct Net {
  std::string arch;
  int image = 0;      // input spatial size
  int in_c = 3;       // real input channels
  int in_c4 = 4;      // padded (16-byte chunks)
  int classes = 0;
  std::vector<Op> ops;
  std::vector<TensorShape> shape;           // output shape of op i
  std::vector<std::vector<int>> consumers;  // ops reading tensor i
  long long n_params = 0;                   // floats, multiple of 4
  long long n_stats = 0;                    // floats
  int max_bn_channels = 0;
  int num_ops() const { return static_cast<int>(ops.size()); }
};

// arch: resnet{18,34,50,101,152} (ImageNet layout), resnet{20,32,44,56,110}
// (CIFAR basic blocks), resnet{164,1001} (CIFAR pre-activation bottleneck).
// recompute: mark bn_relu -> conv outputs transient (see Op::transient);
// -1 = the process default (on; ACCUDNN_RECOMPUTE=0 turns it off)
Net build_net(const std::string& arch, int image, int classes, int recompute = -1);

// does the backward of `op` read its (first / second) input tensor?
bool bwd_reads_input(const Op& op);

// ---- phases ------------------------------------------------------------------
// steps are the reference's phases 1..2N (N = number of ops)
inline int fwd_step(int op) { return op + 1; }
inline int bwd_step(int op, int n) { return op == 0 ? 2 * n : 2 * n + 1 - op; }

// ---- real tensor instances ------------------------------------------------------
// act_recomputed: a transient tensor rewritten in the backward (by compute)
enum class InstKind : int { act, act_prefetched, grad, act_recomputed };
struct Instance {
  InstKind kind = InstKind::act;
  int tensor = -1;         // op id whose output (act) or output-gradient (grad)
  int first = 0, last = 0; // inclusive step interval of device residency
  long long bytes = 0;     // at the instance's k
  bool swapped = false;    // act: offloaded after production
  long long offset = -1;   // arena offset (executor)
  // packing lifetime end (>= last): a swapped activation's region may be
  // kept out of reuse while its offload drains when the budget has room
  int pack_last = -1;
};

struct LifetimeModel {
  int n = 0;                          // ops
  std::vector<Instance> inst;
  std::vector<int> act_inst;          // tensor -> primary activation instance
  std::vector<int> pre_inst;          // tensor -> prefetched / recomputed instance or -1
  std::vector<int> grad_inst;         // tensor -> gradient instance or -1 (aliases share)
  std::vector<int> grad_first_writer; // tensor -> op whose backward writes the group first
  std::vector<int> grad_group;        // tensor -> gradient alias group id
  long long peak_bytes = 0;           // max over steps of live bytes (no fragmentation)
  std::vector<long long> live;        // per step 1..2N
};

// swapped[t] = featuremap of tensor t is offloaded; lookahead = phases an
// H2D prefetch may start before its first backward use
LifetimeModel build_lifetimes(const Net& net, int k, const std::vector<char>& swapped,
                              int lookahead, long long align);

// The swap-in queue of the reference's runtime model (simulator.cpp:113-140,
// :233-285) at phase granularity: prefetches are issued in GMAP order (each
// no earlier than its predecessor in the queue -- head of line), each as
// early as the pool has room for it until its first backward reader, never
// before its offload's producer phase has finished with the featuremap.
// "Room" = live bytes of every instance at each phase + this one <= cap.
// Moves each prefetched instance's `first` step earlier (never later than
// the lookahead placement build_lifetimes gave it); recomputes live/peak.
void schedule_prefetches(const Net& net, LifetimeModel& lm, long long cap);

// static arena offsets: greedy by size, first fit against time-overlapping
// instances; returns the arena size in bytes
long long plan_arena(LifetimeModel& lm);

// reference-format network.json (format_version 1) with k_base images
std::string export_network_json(const Net& net, int k_base, int lookahead);
// layer <-> op description for host tooling and the torch oracle
std::string describe_net_json(const Net& net);

}  // namespace accudnn
