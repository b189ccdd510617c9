// Swap executor: realises one planned training iteration on a B200.
//
// Behavioural contract: /root/reference/proj/src/simulator.cpp:79-370 --
// a compute stream running the 2N phases in order, a swap-out (D2H) stream
// and a swap-in (H2D) stream working through the GMAP's offload/prefetch
// queues in order, one FIFO copy engine per direction, a hard device-memory
// cap.  Real CUDA streams and events replace the simulated ones:
//   * every tensor instance (activation, prefetched activation, gradient
//     group) gets a static offset in one capped arena (planned once per
//     (net, k, pin set)); instance lifetimes come from net.h's lifetime
//     model, the same one the exporter charged to the workspaces;
//   * a region is reused only after its previous occupant's last reader
//     (compute event) and drain (D2H event) completed;
//   * an offload starts when its producing phase's kernels finish; the
//     prefetches are issued in GMAP order, each as early as the budget
//     leaves room for its region (the simulator's swap-in queue,
//     schedule_prefetches), once its offload landed in pinned host memory
//     and its region is free;
//   * the whole iteration (kernels, copies, event edges, the bucketed NCCL
//     all-reduce and the SGD update) can be captured into one CUDA graph.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "net.h"

namespace accudnn {

struct ExecConfig {
  std::string arch = "resnet152";
  int image = 224;
  int classes = 1000;
  int k = 1;                       // per-GPU minibatch (k* of the plan)
  unsigned long long budget = 0;   // device cap (hardware.json memory_budget_bytes)
  unsigned long long fixed_allowance = 0;  // m_others + params + grads (planner's fixed)
  int lookahead = 1;
  // swap-in policy: 1 = the reference runtime's queue (simulator.cpp:113-140,
  // :233-285): prefetches in GMAP order, each as early as the budget leaves
  // room (net.h schedule_prefetches); 0 = a fixed `lookahead` phases ahead
  int prefetch_queue = 1;
  float momentum = 0.9f;
  float weight_decay = 1e-4f;
  float bn_eps = 1e-5f;
  float bn_momentum = 0.1f;
  int device = 0;
  long long bucket_bytes = 25LL << 20;
  int autotune = 1;                // tune conv tile/split-K per shape in the first (eager) step
  // batch-norm statistics from the producing conv's epilogue
  // (accudnn_conv_fwd_stats + accudnn_bn_*_fwd_stats).  Measured on ResNet-152
  // k*=42: 2218 vs 2243 img/s -- the epilogue cost exceeds the saved read --
  // so off by default.
  int conv_bn_stats = 0;
  // weight gradients on a side stream, concurrent with the data-gradient
  // chain (dgrad -> BN backward -> ...), which is the critical path; the
  // weight gradients are only needed by the all-reduce and the update.
  // Not used in profiled or autotuning (first) steps.
  int wgrad_stream = 1;
  // the compute stream (critical path) at the highest stream priority, the
  // weight-gradient stream at the lowest: pending CTAs of the critical path
  // are dispatched first (graph nodes keep their priorities)
  int stream_priority = 0;  // measured: 2333 -> 2256 img/s (the side stream starves), off
  // persistent weight-gradient grids on the side stream use at most this
  // many SMs (0 = all)
  int side_ctas = 0;
  double side_ws_frac = 0.5;  // share of the split-K workspace for the side stream
  // SGD update per gradient bucket as soon as the bucket is complete (and,
  // data parallel, all-reduced) on the communication stream, overlapping the
  // rest of the backward; 0: one update kernel after the backward.  Measured
  // on ResNet-152 k*=42 (1 GPU): 2369 -> 2339 img/s (the update kernels
  // compete with the bandwidth-bound batch norms of the critical path), off
  int overlap_update = 0;
  // featuremap transfers up to these sizes run as SM-driven copy kernels
  // through the host-mapped pinned buffer (kernels/swap_copy.cu) instead of
  // copy-engine memcpys: a memcpy pays ~3 us of issue/completion latency per
  // call (128 KB D2H: 5.8 us engine vs 2.6 us kernel; 512 KB: 13.4 vs 10.1;
  // H2D 128 KB: 5.9 vs 5.1), larger transfers are faster on the engines
  // (tools/copy_bench.py).  0 disables the kernel path for that direction.
  unsigned long long kernel_copy_max_d2h = 2ull << 20;
  unsigned long long kernel_copy_max_h2d = 512ull << 10;
  int kernel_copy_ctas = 8;
};

// The real timeline of the last profiled step, for the reference's output
// documents (exec_capi.cpp serialises it with swapsched's trace_to_csv /
// mem_curves_csv / stall_bars_csv / summary_to_json)
struct RealTimeline {
  std::vector<long long> kstart, kend;  // ns from the iteration start, phases 1..2N
  struct Copy {
    int stream = 1;  // 1 = swap_out (D2H), 2 = swap_in (H2D)
    int tensor = 0;  // featuremap fm_{tensor+1}
    long long start = 0, end = 0;
  };
  std::vector<Copy> copies;               // in stream order
  std::vector<long long> mem_at_phase;    // fixed + live instance bytes, phases 1..2N
  unsigned long long fixed = 0;
};

struct StepStats {
  float loss = 0.f;
  double iter_ms = 0;          // device time of the whole iteration
  double exposed_swap_ms = 0;  // compute-stream stall on prefetches (profiled steps)
  double allreduce_ms = 0;          // NCCL device time over the buckets (profiled steps)
  unsigned long long peak_bytes = 0;  // fixed + arena (static plan) + NCCL's device bytes
  unsigned long long swapped_bytes = 0;
  double exposed_allreduce_ms = 0;  // compute-stream wait at the all-reduce join (profiled)
};

class Executor {
 public:
  Executor(const ExecConfig& cfg, const std::vector<char>& swapped);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  const Net& net() const { return net_; }
  void set_params(const float* host, long long n);
  void get_params(float* host, long long n);
  void get_grads(float* host, long long n);
  void get_stats(float* host, long long n);
  // images: NCHW fp32 [k][3][H][W]; labels int32 [k].  host_inputs = 1 copies
  // from (pinned or pageable) host memory inside the step.  Pipelined input:
  // next_images (host) is copied H2D on a side stream as soon as this step's
  // layout kernel has consumed the staging buffer, overlapping the rest of
  // the step; the next call passes images = nullptr to use it.
  StepStats step(const void* images, const int* labels, int host_inputs, float lr, int update,
                 int profile, const void* next_images = nullptr);
  void set_comm(const void* nccl_unique_id, int rank, int world);
  bool use_graph = false;
  std::string trace_csv() const { return trace_; }
  // real timeline of the last profiled step (CUDA events on every phase
  // and copy), in the reference's simulator terms
  const RealTimeline& timeline() const { return timeline_; }
  // the copies of one iteration in stream order ("swap_out fm3", "swap_in fm7", ...)
  const std::vector<std::string>& copy_order() const { return copy_order_; }
  unsigned long long arena_bytes() const { return arena_bytes_; }
  unsigned long long fixed_bytes() const { return fixed_bytes_; }
  // device bytes NCCL allocated for the communicator (cudaMemGetInfo delta
  // around ncclCommInitRank); charged against the budget with the rest
  unsigned long long comm_bytes() const { return comm_bytes_; }
  int graph_launches() const { return kernel_launches_; }

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
  Net net_;
  ExecConfig cfg_;
  std::string trace_;
  RealTimeline timeline_;
  std::vector<std::string> copy_order_;
  unsigned long long arena_bytes_ = 0, fixed_bytes_ = 0, comm_bytes_ = 0;
  int kernel_launches_ = 0;
};

}  // namespace accudnn
