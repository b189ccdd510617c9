// Swap executor (see executor.h).
#include "executor.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>

#include "accudnn_kernels.h"

namespace accudnn {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void ckl(int rc, const char* what) { ck(static_cast<cudaError_t>(rc), what); }
void ckn(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}

constexpr long long kAlign = 512;

}  // namespace

struct Executor::Impl {
  LifetimeModel lm;
  std::vector<char> swapped;
  int n = 0;
  // device memory
  char* arena = nullptr;
  float* params = nullptr;
  float* grads = nullptr;
  float* momentum_buf = nullptr;
  float* stats = nullptr;
  void* bn_ws = nullptr;
  float* image = nullptr;        // NHWC4
  float* image_nchw = nullptr;   // staging for the host copy
  int* labels = nullptr;
  float* loss = nullptr;
  float* loss_host = nullptr;    // pinned
  void* conv_ws = nullptr;       // split-K partials of the conv kernels
  // batch-norm statistics written by the producing convolution (two slots:
  // conv o uses slot o % 2, read by its BN consumer before the slot is reused)
  float* bn_stats[2] = {nullptr, nullptr};
  size_t bn_stats_bytes = 0;
  std::vector<char> stats_from_conv;  // op -> its BN input's statistics are in a slot
  std::vector<char> stats_ok;         // op -> may produce statistics (slot not reused early)
  std::vector<float*> host_store;  // pinned host copies of swapped featuremaps
  // streams / events
  cudaStream_t compute = nullptr, d2h = nullptr, h2d = nullptr, comm_stream = nullptr;
  cudaStream_t input_stream = nullptr;  // pipelined next-batch H2D
  cudaStream_t side = nullptr;          // concurrent weight gradients
  void* side_ws = nullptr;              // its split-K workspace
  void* precise_scratch = nullptr;      // 3xTF32: operand low parts (compute stream)
  size_t precise_bytes = 0;
  std::vector<cudaEvent_t> fork_ev;     // per step: dy ready on the compute stream
  std::vector<cudaEvent_t> wg_done;     // per step: that step's weight gradient done
  std::vector<int> side_last;           // per instance: last step whose wgrad reads it
  cudaEvent_t layout_done = nullptr;    // staging buffer consumed (record node in the graph)
  cudaEvent_t input_ready = nullptr;    // next batch landed in the staging buffer
  bool prefetched = false;
  std::vector<cudaEvent_t> step_done;   // per step
  std::vector<cudaEvent_t> d2h_done;    // per tensor
  std::vector<cudaEvent_t> h2d_done;    // per tensor
  std::vector<cudaEvent_t> phase_begin, phase_end;  // profiling
  cudaEvent_t iter_begin = nullptr, iter_end = nullptr, comm_done = nullptr;
  std::vector<cudaEvent_t> bucket_ready;
  // profiled steps: all-reduce device time per bucket and the compute
  // stream's wait at the join
  std::vector<cudaEvent_t> ar_begin, ar_end;
  // profiled steps: every copy's start / end (timing events per tensor)
  std::vector<cudaEvent_t> out_b, out_e, in_b, in_e;
  cudaEvent_t bwd_done = nullptr, comm_joined = nullptr;
  // per-instance region predecessors: (instance index)
  std::vector<std::vector<int>> preds;
  // per-step actions
  std::vector<std::vector<int>> prefetch_at;  // step -> tensors to prefetch
  std::vector<std::vector<int>> offload_at;   // step -> tensors to offload
  std::vector<std::vector<int>> first_compute_write;  // step -> instances written first
  // NCCL
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  bool first_step = true;
  // CUDA graph of the iteration (fixed lr/update are baked in)
  cudaGraphExec_t graph = nullptr;
  float graph_lr = -1.f;
  int graph_update = -1;
};

Executor::Executor(const ExecConfig& cfg, const std::vector<char>& swapped)
    : impl_(std::make_unique<Impl>()), cfg_(cfg) {
  net_ = build_net(cfg.arch, cfg.image, cfg.classes);
  Impl& I = *impl_;
  I.n = net_.num_ops();
  const int n = I.n;
  if (!swapped.empty() && static_cast<int>(swapped.size()) != n)
    throw std::invalid_argument("swap mask does not match the network");
  I.swapped = swapped.empty() ? std::vector<char>(static_cast<size_t>(n), 0) : swapped;
  // transient activations are recomputed, never offloaded (0-byte featuremaps
  // in the planner's model: pinning or swapping them is the same)
  for (int t = 0; t < n; ++t)
    if (net_.ops[static_cast<size_t>(t)].transient) I.swapped[static_cast<size_t>(t)] = 0;
  ck(cudaSetDevice(cfg.device), "cudaSetDevice");

  I.lm = build_lifetimes(net_, cfg.k, I.swapped, cfg.lookahead, kAlign);

  // ---- fixed allocations (the planner's fixed overhead) ----
  const long long k = cfg.k;
  const size_t pbytes = sizeof(float) * static_cast<size_t>(net_.n_params);
  const size_t sbytes = sizeof(float) * static_cast<size_t>(std::max<long long>(4, net_.n_stats));
  const size_t wsbytes = accudnn_bn_workspace_bytes(std::max(4, net_.max_bn_channels));
  const size_t img4 = sizeof(float) * static_cast<size_t>(k) * cfg.image * cfg.image * net_.in_c4;
  const size_t img3 = sizeof(float) * static_cast<size_t>(k) * cfg.image * cfg.image * net_.in_c;
  fixed_bytes_ = 3 * pbytes + sbytes + wsbytes + img4 + img3 + sizeof(int) * k + 256;
  // conv-produced BN statistics: [2][ceil(M/32)][C] floats per slot
  {
    size_t need = 0;
    for (int o = 0; o < n; ++o) {
      const Op& op = net_.ops[static_cast<size_t>(o)];
      if (op.kind != OpKind::conv) continue;
      const auto& cons = net_.consumers[static_cast<size_t>(o)];
      if (cons.size() != 1 || !is_bn(net_.ops[static_cast<size_t>(cons[0])].kind)) continue;
      const TensorShape& so = net_.shape[static_cast<size_t>(o)];
      const long long M = static_cast<long long>(k) * so.h * so.w;
      need = std::max(need, sizeof(float) * 2 * static_cast<size_t>((M + 31) / 32) * so.c);
    }
    if (!cfg.conv_bn_stats) need = 0;
    I.bn_stats_bytes = need;
    fixed_bytes_ += 2 * need;
  }
  // 3xTF32 (fp32-accurate) convolutions on the TMA kernels: scratch for the
  // operands' low parts, sized for the largest convolution of the net at k;
  // the weight-gradient side stream is not used in this mode (one scratch)
  // (ACCUDNN_PRECISE_TMA=0: the cp.async PRECISE kernel instead, for A/B checks)
  const char* ptma = std::getenv("ACCUDNN_PRECISE_TMA");
  const bool precise = accudnn_get_conv_math() == 1 && !(ptma && std::atoi(ptma) == 0);
  size_t precise_bytes = 0;
  if (precise) {
    for (int o = 0; o < n; ++o) {
      const Op& op = net_.ops[static_cast<size_t>(o)];
      if (op.kind != OpKind::conv && op.kind != OpKind::fc) continue;
      accudnn_conv_desc d{};
      if (op.kind == OpKind::fc) {
        d = accudnn_conv_desc{static_cast<int>(k), 1, 1, op.cin, op.cout, 1, 1, 1, 0, 1, 1};
      } else {
        const int ih = op.in0 == kImage ? net_.image : net_.shape[static_cast<size_t>(op.in0)].h;
        const int iw = op.in0 == kImage ? net_.image : net_.shape[static_cast<size_t>(op.in0)].w;
        const TensorShape& so = net_.shape[static_cast<size_t>(o)];
        d = accudnn_conv_desc{static_cast<int>(k), ih, iw, op.cin, op.cout, op.r, op.s,
                              op.stride, op.pad, so.h, so.w};
      }
      precise_bytes = std::max<size_t>(precise_bytes, accudnn_conv_precise_scratch_bytes(&d));
    }
    fixed_bytes_ += precise_bytes;
  }
  // split-K workspace of the convolutions: whatever the planner's fixed
  // allowance leaves, capped at 64 MiB; the kernels pick their split
  // factors to fit it
  size_t conv_ws = 64u << 20;
  if (cfg.budget && cfg.fixed_allowance) {
    const unsigned long long used = fixed_bytes_;
    conv_ws = used >= cfg.fixed_allowance
                  ? 0
                  : std::min<size_t>(conv_ws, static_cast<size_t>(cfg.fixed_allowance - used));
    conv_ws &= ~static_cast<size_t>(4095);
  }
  fixed_bytes_ += conv_ws;
  // the side stream's weight gradients get their own share of it
  size_t side_ws = 0;
  if (cfg.wgrad_stream && conv_ws) {
    const double f = std::min(0.9, std::max(0.1, cfg.side_ws_frac));
    side_ws = static_cast<size_t>(static_cast<double>(conv_ws) * f) & ~static_cast<size_t>(4095);
    conv_ws -= side_ws;
  }
  // ---- static arena plan ----
  // The reference runtime model frees a swapped featuremap when its offload
  // lands and claims pool bytes for a prefetch as soon as they are free, in
  // GMAP order (simulator.cpp:113-140, :185-194, :233-285).  In the static
  // arena: (1) a swapped activation's region is kept out of reuse for `pad`
  // phases after its last forward reader (its offload drains) while the
  // budget has room; (2) the swap-in queue issues prefetches as early as the
  // budget leaves room (schedule_prefetches).  The largest pad whose packing
  // fits the budget wins; if first-fit packing overshoots, the room given to
  // the queue shrinks by the overshoot; the fixed lookahead placement with no
  // pad is the fallback.
  {
    bool any_swap = false;
    for (char c : I.swapped) any_swap = any_swap || c;
    long long arena = plan_arena(I.lm);
    if (cfg.prefetch_queue && any_swap && cfg.budget && fixed_bytes_ < cfg.budget) {
      const LifetimeModel base = I.lm;
      const long long base_arena = arena;
      bool ok = false;
      for (int pad : {2 * n, 16, 4, 0}) {
        LifetimeModel padded = base;
        for (Instance& x : padded.inst)
          if (x.kind == InstKind::act && x.swapped) x.pack_last = std::min(2 * n, x.last + pad);
        long long room = static_cast<long long>(cfg.budget - fixed_bytes_);
        for (int it = 0; it < 8 && room > 0 && !ok; ++it) {
          I.lm = padded;
          schedule_prefetches(net_, I.lm, room);
          arena = plan_arena(I.lm);
          const long long over = static_cast<long long>(fixed_bytes_) + arena -
                                 static_cast<long long>(cfg.budget);
          if (over <= 0)
            ok = true;
          else
            room -= over;
        }
        if (ok) break;
      }
      if (!ok) {
        I.lm = base;
        arena = base_arena;
      }
    }
    arena_bytes_ = static_cast<unsigned long long>(arena);
  }
  const long long arena = static_cast<long long>(arena_bytes_);
  // region predecessors: earlier (in time) instances sharing bytes
  I.preds.assign(I.lm.inst.size(), {});
  for (size_t a = 0; a < I.lm.inst.size(); ++a) {
    const Instance& x = I.lm.inst[a];
    for (size_t b = 0; b < I.lm.inst.size(); ++b) {
      const Instance& y = I.lm.inst[b];
      if (a == b || y.last >= x.first) continue;
      if (y.offset < x.offset + x.bytes && x.offset < y.offset + y.bytes)
        I.preds[a].push_back(static_cast<int>(b));
    }
  }
  I.prefetch_at.assign(static_cast<size_t>(2 * n + 2), {});
  I.offload_at.assign(static_cast<size_t>(2 * n + 2), {});
  I.first_compute_write.assign(static_cast<size_t>(2 * n + 2), {});
  for (int t = 0; t < n; ++t) {
    if (!I.swapped[static_cast<size_t>(t)]) continue;
    I.offload_at[static_cast<size_t>(fwd_step(t))].push_back(t);
    const Instance& p = I.lm.inst[static_cast<size_t>(I.lm.pre_inst[static_cast<size_t>(t)])];
    I.prefetch_at[static_cast<size_t>(p.first)].push_back(t);
  }
  // within a phase, the swap-in stream takes its prefetches in GMAP order
  // (fm_{t+1} is prefetched in phase 2N - t: larger t first)
  for (auto& v : I.prefetch_at) std::sort(v.begin(), v.end(), std::greater<int>());
  for (size_t i = 0; i < I.lm.inst.size(); ++i)
    if (I.lm.inst[i].kind != InstKind::act_prefetched)
      I.first_compute_write[static_cast<size_t>(I.lm.inst[i].first)].push_back(static_cast<int>(i));

  if (cfg.budget) {
    if (cfg.fixed_allowance && fixed_bytes_ > cfg.fixed_allowance)
      throw std::runtime_error("fixed device allocations (" + std::to_string(fixed_bytes_) +
                               " B) exceed the planner's fixed overhead (" +
                               std::to_string(cfg.fixed_allowance) + " B)");
    if (fixed_bytes_ + arena_bytes_ > cfg.budget)
      throw std::runtime_error("executor arena " + std::to_string(arena_bytes_) +
                               " B + fixed " + std::to_string(fixed_bytes_) +
                               " B exceed the device budget " + std::to_string(cfg.budget));
  }
  ck(cudaMalloc(&I.arena, static_cast<size_t>(std::max<long long>(arena, kAlign))), "arena");
  ck(cudaMalloc(&I.params, pbytes), "params");
  ck(cudaMalloc(&I.grads, pbytes), "grads");
  ck(cudaMalloc(&I.momentum_buf, pbytes), "momentum");
  ck(cudaMalloc(&I.stats, sbytes), "stats");
  ck(cudaMalloc(&I.bn_ws, wsbytes), "bn ws");
  ck(cudaMalloc(&I.image, img4), "image");
  ck(cudaMalloc(&I.image_nchw, img3), "image staging");
  ck(cudaMalloc(&I.labels, sizeof(int) * k), "labels");
  ck(cudaMalloc(&I.loss, 256), "loss");
  ck(cudaMallocHost(&I.loss_host, sizeof(float)), "loss host");
  if (conv_ws) ck(cudaMalloc(&I.conv_ws, conv_ws), "conv workspace");
  I.precise_bytes = precise_bytes;
  if (precise_bytes) ck(cudaMalloc(&I.precise_scratch, precise_bytes), "3xTF32 scratch");
  if (side_ws) ck(cudaMalloc(&I.side_ws, side_ws), "side conv workspace");
  if (I.bn_stats_bytes)
    for (auto& p : I.bn_stats) ck(cudaMalloc(&p, I.bn_stats_bytes), "bn stats");
  I.stats_from_conv.assign(static_cast<size_t>(n), 0);
  // a conv may hand its statistics to its BN consumer only if no other
  // statistics-producing conv of the same slot parity runs in between
  I.stats_ok.assign(static_cast<size_t>(n), 0);
  for (int o = 0; o < n; ++o) {
    const auto& cons = net_.consumers[static_cast<size_t>(o)];
    if (net_.ops[static_cast<size_t>(o)].kind != OpKind::conv || cons.size() != 1 ||
        !is_bn(net_.ops[static_cast<size_t>(cons[0])].kind))
      continue;
    bool ok = true;
    for (int q = o + 1; q < cons[0]; ++q) {
      const auto& cq = net_.consumers[static_cast<size_t>(q)];
      if (net_.ops[static_cast<size_t>(q)].kind == OpKind::conv && q % 2 == o % 2 &&
          cq.size() == 1 && is_bn(net_.ops[static_cast<size_t>(cq[0])].kind))
        ok = false;
    }
    // conv_bn_stats = 2: only the short layers (k*H*W <= 32768 rows), whose
    // batch norms are latency-bound; a large layer's BN is bandwidth-bound
    // and saves only one of its reads, less than the epilogue sums cost
    if (cfg.conv_bn_stats == 2) {
      const TensorShape& so = net_.shape[static_cast<size_t>(o)];
      if (static_cast<long long>(cfg.k) * so.h * so.w > 16LL * 2048) ok = false;
    }
    // conv_bn_stats = 3 (A/B): only the layers whose output exceeds 64 MB,
    // where the BN's second read of x comes from HBM
    if (cfg.conv_bn_stats == 3) {
      const TensorShape& so = net_.shape[static_cast<size_t>(o)];
      if (4LL * cfg.k * so.h * so.w * so.c <= (64LL << 20)) ok = false;
    }
    I.stats_ok[static_cast<size_t>(o)] = ok;
  }
  if (cfg.autotune) accudnn_conv_autotune(1);
  ck(cudaMemset(I.params, 0, pbytes), "memset");
  ck(cudaMemset(I.grads, 0, pbytes), "memset");
  ck(cudaMemset(I.momentum_buf, 0, pbytes), "memset");
  ck(cudaMemset(I.stats, 0, sbytes), "memset");
  ck(cudaMemset(I.bn_ws, 0, wsbytes), "memset");
  // running variance starts at 1
  {
    std::vector<float> st(static_cast<size_t>(std::max<long long>(4, net_.n_stats)), 0.f);
    for (const Op& op : net_.ops)
      if (op.stat_off >= 0)
        for (int c = 0; c < op.channels; ++c)
          st[static_cast<size_t>(op.stat_off + 3 * op.channels + c)] = 1.f;
    ck(cudaMemcpy(I.stats, st.data(), sbytes, cudaMemcpyHostToDevice), "stats init");
  }
  I.host_store.assign(static_cast<size_t>(n), nullptr);
  for (int t = 0; t < n; ++t)
    if (I.swapped[static_cast<size_t>(t)]) {
      const Instance& a = I.lm.inst[static_cast<size_t>(I.lm.act_inst[static_cast<size_t>(t)])];
      ck(cudaHostAlloc(reinterpret_cast<void**>(&I.host_store[static_cast<size_t>(t)]),
                       static_cast<size_t>(a.bytes), cudaHostAllocDefault),
         "pinned host store");
    }

  int prio_lo = 0, prio_hi = 0;
  ck(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "priority range");
  if (!cfg.stream_priority) prio_lo = prio_hi = 0;
  ck(cudaStreamCreateWithPriority(&I.compute, cudaStreamNonBlocking, prio_hi), "stream");
  ck(cudaStreamCreateWithFlags(&I.d2h, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&I.h2d, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&I.comm_stream, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&I.input_stream, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithPriority(&I.side, cudaStreamNonBlocking, prio_lo), "stream");
  // every stream this executor launches convolutions on owns its split-K
  // workspace (carved out of the fixed allocation, so inside the budget):
  // executors never share partials, whatever else is alive in the process
  ckl(accudnn_conv_set_stream_workspace(I.compute, I.conv_ws, I.conv_ws ? conv_ws : 0,
                                        I.conv_ws ? 0 : -1),
      "compute workspace");
  if (I.precise_scratch)
    ckl(accudnn_conv_set_precise_scratch(I.compute, I.precise_scratch, I.precise_bytes),
        "precise scratch");
  ckl(accudnn_conv_set_stream_workspace(I.side, I.side_ws, I.side_ws ? side_ws : 0,
                                        cfg.side_ctas > 0 ? cfg.side_ctas : (I.side_ws ? 0 : -1)),
      "side workspace");
  ck(cudaEventCreateWithFlags(&I.layout_done, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&I.input_ready, cudaEventDisableTiming), "event");
  auto mk = [](std::vector<cudaEvent_t>& v, size_t cnt, bool timing) {
    v.assign(cnt, nullptr);
    for (auto& e : v)
      ck(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming),
         "event");
  };
  mk(I.step_done, static_cast<size_t>(2 * n + 2), false);
  mk(I.d2h_done, static_cast<size_t>(n), false);
  mk(I.h2d_done, static_cast<size_t>(n), false);
  mk(I.fork_ev, static_cast<size_t>(2 * n + 2), false);
  mk(I.wg_done, static_cast<size_t>(2 * n + 2), false);
  // instances a side-stream weight gradient reads (its input activation as
  // the backward step sees it, and the output gradient): a later occupant of
  // their bytes must also wait for that weight gradient
  I.side_last.assign(I.lm.inst.size(), 0);
  for (int s = n + 1; s <= 2 * n; ++s)
  for (int o : {2 * n + 1 - s, s == 2 * n ? 0 : -1}) {  // the ops of step s (see step())
    if (o < 0 || o >= n || (o == 0 && s != 2 * n)) continue;
    const Op& op = net_.ops[static_cast<size_t>(o)];
    if (op.kind != OpKind::conv && op.kind != OpKind::fc) continue;
    if (op.in0 >= 0) {
      const size_t u = static_cast<size_t>(op.in0);
      int id = I.lm.act_inst[u];
      if (I.lm.pre_inst[u] >= 0 && s >= I.lm.inst[static_cast<size_t>(I.lm.pre_inst[u])].first)
        id = I.lm.pre_inst[u];
      if (id >= 0) I.side_last[static_cast<size_t>(id)] = std::max(I.side_last[static_cast<size_t>(id)], s);
      // a transient input is recomputed on the side stream from its BN input
      const Op& ob = net_.ops[u];
      if (ob.transient && ob.in0 >= 0) {
        const size_t v = static_cast<size_t>(ob.in0);
        int xi = I.lm.act_inst[v];
        if (I.lm.pre_inst[v] >= 0 && s >= I.lm.inst[static_cast<size_t>(I.lm.pre_inst[v])].first)
          xi = I.lm.pre_inst[v];
        if (xi >= 0) I.side_last[static_cast<size_t>(xi)] = std::max(I.side_last[static_cast<size_t>(xi)], s);
      }
    }
    const int g = I.lm.grad_inst[static_cast<size_t>(o)];
    if (g >= 0) I.side_last[static_cast<size_t>(g)] = std::max(I.side_last[static_cast<size_t>(g)], s);
  }
  mk(I.phase_begin, static_cast<size_t>(2 * n + 2), true);
  mk(I.phase_end, static_cast<size_t>(2 * n + 2), true);
  ck(cudaEventCreate(&I.iter_begin), "event");
  ck(cudaEventCreate(&I.iter_end), "event");
  ck(cudaEventCreateWithFlags(&I.comm_done, cudaEventDisableTiming), "event");
  mk(I.out_b, static_cast<size_t>(n), true);
  mk(I.out_e, static_cast<size_t>(n), true);
  mk(I.in_b, static_cast<size_t>(n), true);
  mk(I.in_e, static_cast<size_t>(n), true);
  mk(I.ar_begin, static_cast<size_t>(n + 2), true);
  mk(I.ar_end, static_cast<size_t>(n + 2), true);
  ck(cudaEventCreate(&I.bwd_done), "event");
  ck(cudaEventCreate(&I.comm_joined), "event");
}

Executor::~Executor() {
  Impl& I = *impl_;
  if (I.graph) cudaGraphExecDestroy(I.graph);
  if (I.comm) ncclCommDestroy(I.comm);
  if (I.side) accudnn_conv_set_stream_workspace(I.side, nullptr, 0, 0);
  if (I.precise_scratch) {
    accudnn_conv_set_precise_scratch(I.compute, nullptr, 0);
    cudaFree(I.precise_scratch);
  }
  if (I.compute) accudnn_conv_set_stream_workspace(I.compute, nullptr, 0, 0);
  for (auto* v : {&I.step_done, &I.d2h_done, &I.h2d_done, &I.phase_begin, &I.phase_end,
                  &I.bucket_ready, &I.fork_ev, &I.wg_done, &I.ar_begin, &I.ar_end, &I.out_b, &I.out_e, &I.in_b, &I.in_e})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {I.iter_begin, I.iter_end, I.comm_done, I.layout_done, I.input_ready,
                        I.bwd_done, I.comm_joined})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {I.compute, I.d2h, I.h2d, I.comm_stream, I.input_stream, I.side})
    if (s) cudaStreamDestroy(s);
  for (float* h : I.host_store)
    if (h) cudaFreeHost(h);
  if (I.loss_host) cudaFreeHost(I.loss_host);
  for (void* p : {static_cast<void*>(I.arena), static_cast<void*>(I.params),
                  static_cast<void*>(I.grads), static_cast<void*>(I.momentum_buf),
                  static_cast<void*>(I.stats), I.bn_ws, static_cast<void*>(I.image),
                  static_cast<void*>(I.image_nchw), static_cast<void*>(I.labels),
                  static_cast<void*>(I.loss), I.conv_ws, static_cast<void*>(I.bn_stats[0]),
                  static_cast<void*>(I.bn_stats[1]), I.side_ws})
    if (p) cudaFree(p);
}

void Executor::set_params(const float* host, long long n) {
  if (n != net_.n_params) throw std::invalid_argument("parameter count mismatch");
  ck(cudaMemcpy(impl_->params, host, sizeof(float) * n, cudaMemcpyHostToDevice), "set_params");
  impl_->first_step = true;
}
void Executor::get_params(float* host, long long n) {
  if (n != net_.n_params) throw std::invalid_argument("parameter count mismatch");
  ck(cudaMemcpy(host, impl_->params, sizeof(float) * n, cudaMemcpyDeviceToHost), "get_params");
}
void Executor::get_grads(float* host, long long n) {
  if (n != net_.n_params) throw std::invalid_argument("parameter count mismatch");
  ck(cudaMemcpy(host, impl_->grads, sizeof(float) * n, cudaMemcpyDeviceToHost), "get_grads");
}
void Executor::get_stats(float* host, long long n) {
  if (n != net_.n_stats) throw std::invalid_argument("stats count mismatch");
  ck(cudaMemcpy(host, impl_->stats, sizeof(float) * n, cudaMemcpyDeviceToHost), "get_stats");
}

void Executor::set_comm(const void* uid, int rank, int world) {
  Impl& I = *impl_;
  // world 1 still builds a (single-rank) communicator: the bucketed
  // all-reduce path then runs on one GPU (tests)
  if (world < 1 || rank < 0 || rank >= world)
    throw std::invalid_argument("set_comm: need 0 <= rank < world, world >= 1");
  // a captured iteration baked the previous communicator (or none) into its
  // all-reduce nodes: drop it, and the old communicator with it
  if (I.graph) cudaGraphExecDestroy(I.graph);
  I.graph = nullptr;
  I.graph_lr = -1.f;
  I.graph_update = -1;
  if (I.comm) {
    ck(cudaStreamSynchronize(I.comm_stream), "comm drain");
    ckn(ncclCommDestroy(I.comm), "ncclCommDestroy");
    I.comm = nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  // NCCL's device buffers count against the cap like every other allocation
  // (SURVEY 8e): measured as the free-memory delta around the init
  size_t free0 = 0, free1 = 0, total = 0;
  ck(cudaMemGetInfo(&free0, &total), "meminfo");
  ckn(ncclCommInitRank(&I.comm, world, id, rank), "ncclCommInitRank");
  ck(cudaDeviceSynchronize(), "comm init");
  ck(cudaMemGetInfo(&free1, &total), "meminfo");
  comm_bytes_ = free0 > free1 ? static_cast<unsigned long long>(free0 - free1) : 0ull;
  if (cfg_.budget && fixed_bytes_ + arena_bytes_ + comm_bytes_ > cfg_.budget)
    std::fprintf(stderr,
                 "[accudnn] warning: NCCL communicator holds %llu B; fixed %llu + arena %llu + "
                 "NCCL exceed the device budget %llu B (raise m_others_bytes by the NCCL "
                 "allowance before planning)\n",
                 comm_bytes_, fixed_bytes_, arena_bytes_, cfg_.budget);
  I.rank = rank;
  I.world = world;
}

StepStats Executor::step(const void* images, const int* labels, int host_inputs, float lr,
                         int update, int profile, const void* next_images) {
  Impl& I = *impl_;
  const int n = I.n;
  const int k = cfg_.k;
  const Net& net = net_;
  cudaStream_t cs = I.compute;
  void* csv = static_cast<void*>(cs);
  StepStats st;
  // (3xTF32: the weight gradients stay on the compute stream, which owns the
  // precise scratch)
  const bool use_side = cfg_.wgrad_stream && !profile && !I.first_step && !I.precise_scratch;
  int last_wg = 0;  // latest step with a side-stream weight gradient

  auto act = [&](int t, int step) -> float* {
    if (t == kImage) return I.image;
    const size_t u = static_cast<size_t>(t);
    int id = I.lm.act_inst[u];
    if (I.lm.pre_inst[u] >= 0 && step >= I.lm.inst[static_cast<size_t>(I.lm.pre_inst[u])].first)
      id = I.lm.pre_inst[u];
    return reinterpret_cast<float*>(I.arena + I.lm.inst[static_cast<size_t>(id)].offset);
  };
  auto grad = [&](int t) -> float* {
    const int id = I.lm.grad_inst[static_cast<size_t>(t)];
    if (id < 0) throw std::logic_error("tensor without gradient buffer");
    return reinterpret_cast<float*>(I.arena + I.lm.inst[static_cast<size_t>(id)].offset);
  };
  auto beta_for = [&](int x, int op) { return I.lm.grad_first_writer[static_cast<size_t>(x)] == op ? 0 : 1; };
  auto elems = [&](int t) {
    return static_cast<long long>(k) * net.shape[static_cast<size_t>(t)].per_image();
  };
  auto conv_desc = [&](const Op& op) {
    accudnn_conv_desc d{};
    if (op.kind == OpKind::fc) {
      d = accudnn_conv_desc{k, 1, 1, op.cin, op.cout, 1, 1, 1, 0, 1, 1};
      return d;
    }
    const int in_h = op.in0 == kImage ? net.image : net.shape[static_cast<size_t>(op.in0)].h;
    const int in_w = op.in0 == kImage ? net.image : net.shape[static_cast<size_t>(op.in0)].w;
    const TensorShape& so = net.shape[static_cast<size_t>(&op - net.ops.data())];
    d = accudnn_conv_desc{k, in_h, in_w, op.cin, op.cout, op.r, op.s, op.stride, op.pad, so.h, so.w};
    return d;
  };

  // ---- one forward op ----
  auto forward = [&](int o, int s) {
    const Op& op = net.ops[static_cast<size_t>(o)];
    const TensorShape& so = net.shape[static_cast<size_t>(o)];
    float* y = act(o, s);
    switch (op.kind) {
      case OpKind::conv: {
        const accudnn_conv_desc d = conv_desc(op);
        const auto& cons = net.consumers[static_cast<size_t>(o)];
        I.stats_from_conv[static_cast<size_t>(o)] = 0;
        if (I.bn_stats_bytes && I.stats_ok[static_cast<size_t>(o)]) {
          int produced = 0;
          ckl(accudnn_conv_fwd_stats(&d, act(op.in0, s), I.params + op.w_off, y,
                                     I.bn_stats[o % 2], &produced, csv),
              "conv fwd");
          I.stats_from_conv[static_cast<size_t>(o)] = static_cast<char>(produced);
        } else {
          ckl(accudnn_conv_fwd(&d, act(op.in0, s), I.params + op.w_off, y, 0, csv), "conv fwd");
        }
        break;
      }
      case OpKind::fc: {
        const accudnn_conv_desc d = conv_desc(op);
        ckl(accudnn_conv_fwd(&d, act(op.in0, s), I.params + op.w_off, y, 0, csv), "fc fwd");
        ckl(accudnn_bias_add(y, I.params + op.b_off, k, op.cout, csv), "bias");
        break;
      }
      case OpKind::bn:
      case OpKind::bn_relu: {
        const int C = op.channels;
        float* sp = I.stats + op.stat_off;
        if (op.in0 >= 0 && I.stats_from_conv[static_cast<size_t>(op.in0)])
          ckl(accudnn_bn_fwd_stats(act(op.in0, s), I.bn_stats[op.in0 % 2], elems(o) / C, C,
                                   I.params + op.g_off, I.params + op.beta_off, cfg_.bn_eps,
                                   op.kind == OpKind::bn_relu, y, sp, sp + C, sp + 2 * C,
                                   sp + 3 * C, cfg_.bn_momentum, I.bn_ws, csv),
              "bn fwd");
        else
          ckl(accudnn_bn_fwd(act(op.in0, s), elems(o) / C, C, I.params + op.g_off,
                             I.params + op.beta_off, cfg_.bn_eps, op.kind == OpKind::bn_relu, y,
                             sp, sp + C, sp + 2 * C, sp + 3 * C, cfg_.bn_momentum, I.bn_ws, csv),
              "bn fwd");
        break;
      }
      case OpKind::bn_add_relu: {
        const int C = op.channels;
        float* sp = I.stats + op.stat_off;
        if (op.in0 >= 0 && I.stats_from_conv[static_cast<size_t>(op.in0)])
          ckl(accudnn_bn_add_relu_fwd_stats(act(op.in0, s), I.bn_stats[op.in0 % 2],
                                            act(op.in1, s), elems(o) / C, C, I.params + op.g_off,
                                            I.params + op.beta_off, cfg_.bn_eps, y, sp, sp + C,
                                            sp + 2 * C, sp + 3 * C, cfg_.bn_momentum, I.bn_ws,
                                            csv),
              "bn_add_relu fwd");
        else
          ckl(accudnn_bn_add_relu_fwd(act(op.in0, s), act(op.in1, s), elems(o) / C, C,
                                      I.params + op.g_off, I.params + op.beta_off, cfg_.bn_eps, y,
                                      sp, sp + C, sp + 2 * C, sp + 3 * C, cfg_.bn_momentum,
                                      I.bn_ws, csv),
              "bn_add_relu fwd");
        break;
      }
      case OpKind::relu:
        ckl(accudnn_relu_fwd(act(op.in0, s), y, elems(o), csv), "relu fwd");
        break;
      case OpKind::add:
        ckl(accudnn_add_fwd(act(op.in0, s), act(op.in1, s), y, elems(o), csv), "add fwd");
        break;
      case OpKind::maxpool: {
        const TensorShape& si = net.shape[static_cast<size_t>(op.in0)];
        ckl(accudnn_maxpool_fwd(act(op.in0, s), k, si.h, si.w, si.c, op.pk, op.pk, op.pstride,
                                op.ppad, so.h, so.w, y, csv),
            "maxpool fwd");
        break;
      }
      case OpKind::avgpool: {
        const TensorShape& si = net.shape[static_cast<size_t>(op.in0)];
        ckl(accudnn_avgpool_fwd(act(op.in0, s), k, si.h * si.w, si.c, y, csv), "avgpool fwd");
        break;
      }
      case OpKind::xent:
        ckl(accudnn_xent_fwd(act(op.in0, s), I.labels, k, net.classes, I.loss, csv), "xent fwd");
        break;
    }
  };

  // gradient instances a side-stream weight gradient reads, by the step that
  // launched it: a later write into the same instance (an accumulating
  // writer of an aliased gradient group) must wait for that weight gradient
  std::vector<int> side_grad_reader(I.lm.inst.size(), 0);
  auto before_write = [&](int x) {
    if (x < 0) return;
    const int g = I.lm.grad_inst[static_cast<size_t>(x)];
    if (g < 0 || side_grad_reader[static_cast<size_t>(g)] == 0) return;
    ck(cudaStreamWaitEvent(cs, I.wg_done[static_cast<size_t>(side_grad_reader[static_cast<size_t>(g)])], 0),
       "wait wgrad");
    side_grad_reader[static_cast<size_t>(g)] = 0;
  };

  // ---- one backward op ----
  auto backward = [&](int o, int s) {
    const Op& op = net.ops[static_cast<size_t>(o)];
    // every gradient this op writes: its inputs' (pass-through adds write none)
    if (op.kind != OpKind::add) {
      before_write(op.in0);
      before_write(op.in1);
    } else {
      for (int x : {op.in0, op.in1})
        if (x >= 0 && I.lm.grad_group[static_cast<size_t>(x)] != I.lm.grad_group[static_cast<size_t>(o)])
          before_write(x);
    }
    switch (op.kind) {
      case OpKind::conv:
      case OpKind::fc: {
        const accudnn_conv_desc d = conv_desc(op);
        float* dy = grad(o);
        // a transient input (bn_relu output) is recomputed from the BN input
        // and its saved statistics first (on the weight-gradient stream)
        auto recompute = [&](cudaStream_t st) {
          if (op.in0 < 0 || !net.ops[static_cast<size_t>(op.in0)].transient) return;
          const Op& bn = net.ops[static_cast<size_t>(op.in0)];
          if (bn.in0 >= 0 && I.swapped[static_cast<size_t>(bn.in0)])
            ck(cudaStreamWaitEvent(st, I.h2d_done[static_cast<size_t>(bn.in0)], 0), "wait");
          const int C = bn.channels;
          const float* sp = I.stats + bn.stat_off;
          ckl(accudnn_bn_relu_apply(act(bn.in0, s), elems(op.in0) / C, C, I.params + bn.g_off,
                                    I.params + bn.beta_off, sp, sp + C, act(op.in0, s),
                                    static_cast<void*>(st)),
              "bn_relu recompute");
        };
        if (use_side) {
          ck(cudaEventRecord(I.fork_ev[static_cast<size_t>(s)], cs), "record");
          ck(cudaStreamWaitEvent(I.side, I.fork_ev[static_cast<size_t>(s)], 0), "wait");
          recompute(I.side);
          ckl(accudnn_conv_wgrad(&d, act(op.in0, s), dy, I.grads + op.w_off, 0, 0,
                                 static_cast<void*>(I.side)),
              "wgrad");
          ck(cudaEventRecord(I.wg_done[static_cast<size_t>(s)], I.side), "record");
          last_wg = s;
          side_grad_reader[static_cast<size_t>(I.lm.grad_inst[static_cast<size_t>(o)])] = s;
        } else {
          recompute(cs);
          ckl(accudnn_conv_wgrad(&d, act(op.in0, s), dy, I.grads + op.w_off, 0, 0, csv), "wgrad");
        }
        if (op.in0 != kImage)
          ckl(accudnn_conv_dgrad(&d, dy, I.params + op.w_off, grad(op.in0), beta_for(op.in0, o),
                                 csv),
              "dgrad");
        break;
      }
      case OpKind::bn:
      case OpKind::bn_relu: {
        const int C = op.channels;
        float* sp = I.stats + op.stat_off;
        ckl(accudnn_bn_bwd(act(op.in0, s), grad(o), elems(o) / C, C, I.params + op.g_off,
                           I.params + op.beta_off, sp, sp + C, op.kind == OpKind::bn_relu,
                           grad(op.in0), beta_for(op.in0, o), I.grads + op.g_off,
                           I.grads + op.beta_off, I.bn_ws, csv),
            "bn bwd");
        break;
      }
      case OpKind::bn_add_relu: {
        const int C = op.channels;
        float* sp = I.stats + op.stat_off;
        ckl(accudnn_bn_add_relu_bwd(act(op.in0, s), act(op.in1, s), grad(o), elems(o) / C, C,
                                    I.params + op.g_off, I.params + op.beta_off, sp, sp + C,
                                    grad(op.in0), beta_for(op.in0, o), grad(op.in1),
                                    beta_for(op.in1, o), I.grads + op.g_off,
                                    I.grads + op.beta_off, I.bn_ws, csv),
            "bn_add_relu bwd");
        break;
      }
      case OpKind::relu:
        ckl(accudnn_relu_bwd(act(op.in0, s), grad(o), grad(op.in0), elems(o), beta_for(op.in0, o),
                             csv),
            "relu bwd");
        break;
      case OpKind::add:
        for (int x : {op.in0, op.in1}) {
          if (x < 0) continue;
          if (I.lm.grad_group[static_cast<size_t>(x)] == I.lm.grad_group[static_cast<size_t>(o)])
            continue;  // aliased pass-through
          ckl(accudnn_copy(grad(o), grad(x), elems(o), beta_for(x, o), csv), "add bwd");
        }
        break;
      case OpKind::maxpool: {
        const TensorShape& si = net.shape[static_cast<size_t>(op.in0)];
        const TensorShape& so = net.shape[static_cast<size_t>(o)];
        if (beta_for(op.in0, o)) throw std::logic_error("maxpool input with several consumers");
        ckl(accudnn_maxpool_bwd(act(op.in0, s), grad(o), k, si.h, si.w, si.c, op.pk, op.pk,
                                op.pstride, op.ppad, so.h, so.w, grad(op.in0), csv),
            "maxpool bwd");
        break;
      }
      case OpKind::avgpool: {
        const TensorShape& si = net.shape[static_cast<size_t>(op.in0)];
        if (beta_for(op.in0, o)) throw std::logic_error("avgpool input with several consumers");
        ckl(accudnn_avgpool_bwd(grad(o), k, si.h * si.w, si.c, grad(op.in0), csv), "avgpool bwd");
        break;
      }
      case OpKind::xent: {
        const Op& fc = net.ops[static_cast<size_t>(op.in0)];
        if (fc.kind != OpKind::fc) throw std::logic_error("loss must follow the classifier");
        ckl(accudnn_xent_bwd(act(op.in0, s), I.labels, k, net.classes, grad(op.in0),
                             I.grads + fc.b_off, csv),
            "xent bwd");
        break;
      }
    }
  };

  // wait for everything a newly written instance's region depends on
  // phases whose compute waited on a copy stream (prefetch landed / offload
  // drained): the only gaps that count as exposed swap time
  std::vector<char> swap_wait(static_cast<size_t>(2 * n + 2), 0);
  int cur_step = 0;
  auto wait_region = [&](int inst, cudaStream_t stream, bool same_as_compute) {
    for (int p : I.preds[static_cast<size_t>(inst)]) {
      const Instance& y = I.lm.inst[static_cast<size_t>(p)];
      if (use_side && I.side_last[static_cast<size_t>(p)] > 0)
        ck(cudaStreamWaitEvent(stream, I.wg_done[static_cast<size_t>(I.side_last[static_cast<size_t>(p)])], 0),
           "wait wgrad");
      if (y.kind == InstKind::act && y.swapped) {
        ck(cudaStreamWaitEvent(stream, I.d2h_done[static_cast<size_t>(y.tensor)], 0), "wait");
        if (same_as_compute) swap_wait[static_cast<size_t>(cur_step)] = 1;
      }
      // a prefetched predecessor nobody read in the backward (e.g. an add's
      // input: the GMAP prefetches every featuremap) may still be landing
      if (y.kind == InstKind::act_prefetched && stream != I.h2d)
        ck(cudaStreamWaitEvent(stream, I.h2d_done[static_cast<size_t>(y.tensor)], 0), "wait");
      if (!same_as_compute) {
        ck(cudaStreamWaitEvent(stream, I.step_done[static_cast<size_t>(y.last)], 0), "wait");
      }
    }
  };

  // featuremap transfer: copy kernel through the mapped pinned buffer for
  // small transfers, copy engine for large ones (ExecConfig thresholds)
  auto transfer = [&](void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                      cudaStream_t st, const char* what) {
    const unsigned long long lim =
        kind == cudaMemcpyDeviceToHost ? cfg_.kernel_copy_max_d2h : cfg_.kernel_copy_max_h2d;
    if (bytes <= lim)
      ck(static_cast<cudaError_t>(accudnn_swap_copy(dst, src, bytes, cfg_.kernel_copy_ctas, st)),
         what);
    else
      ck(cudaMemcpyAsync(dst, src, bytes, kind, st), what);
  };

  // gradient all-reduce buckets over the completed prefix of the grads
  std::vector<long long> prefix_after_step(static_cast<size_t>(2 * n + 2), 0);
  {
    long long done = 0;
    for (int s = n + 1; s <= 2 * n; ++s) {
      const int o = 2 * n + 1 - s;
      auto extend = [&](int op_id) {
        const Op& op = net.ops[static_cast<size_t>(op_id)];
        long long end = -1;
        if (op.w_off >= 0) end = std::max(end, op.w_off + static_cast<long long>(op.cout) * op.r * op.s * op.cin);
        if (op.b_off >= 0) end = std::max(end, op.b_off + op.cout);
        if (op.beta_off >= 0) end = std::max(end, op.beta_off + op.channels);
        if (end > done) done = end;
      };
      if (o >= 1 && o < n) extend(o);
      if (s == 2 * n) extend(0);
      // bucket cuts on 16-byte boundaries (the SGD kernel is float4-wide);
      // the padding up to the next multiple of 4 belongs to the same op
      done = (done + 3) / 4 * 4;
      prefix_after_step[static_cast<size_t>(s)] = std::min(done, net.n_params);
    }
  }

  const bool overlap_update = update && cfg_.overlap_update;
  int n_buckets = 0;  // timed all-reduce buckets of a profiled step
  std::vector<std::string> order;  // copies in enqueue (= stream) order
  RealTimeline timeline;
  auto enqueue_iteration = [&](bool capture) {
    int launches = 0;
    const bool timed_copies = profile && !capture;
    order.clear();
    timeline.copies.clear();
    if (host_inputs && !capture) {
      const size_t img3 = sizeof(float) * static_cast<size_t>(k) * cfg_.image * cfg_.image * net.in_c;
      if (images)
        ck(cudaMemcpyAsync(I.image_nchw, images, img3, cudaMemcpyHostToDevice, cs), "h2d images");
      ck(cudaMemcpyAsync(I.labels, labels, sizeof(int) * k, cudaMemcpyHostToDevice, cs), "h2d labels");
    }
    const float* src = (host_inputs || capture) ? I.image_nchw : static_cast<const float*>(images);
    if (!host_inputs && !capture && labels)
      ck(cudaMemcpyAsync(I.labels, labels, sizeof(int) * k, cudaMemcpyDeviceToDevice, cs), "labels");
    // captured: the iteration's device time starts with the graph's first
    // node (the host's cudaGraphLaunch of ~1000 nodes takes longer than the
    // queued input copies, and that host latency is not device work)
    if (capture) ck(cudaEventRecordWithFlags(I.iter_begin, cs, cudaEventRecordExternal), "record");
    ckl(accudnn_nchw_to_nhwc_pad(src, k, net.in_c, cfg_.image, cfg_.image, net.in_c4, I.image, csv),
        "image layout");
    // the staging buffer is free from here on: the next batch may land in it
    ck(cudaEventRecordWithFlags(I.layout_done, cs, capture ? cudaEventRecordExternal : 0),
       "record");
    ++launches;
    long long reduced = 0;
    const long long bucket = std::max<long long>(1, cfg_.bucket_bytes / 4);
    bool comm_used = false;
    for (int s = 1; s <= 2 * n; ++s) {
      // swap-in: prefetches that may start at this step
      for (int t : I.prefetch_at[static_cast<size_t>(s)]) {
        const int pid = I.lm.pre_inst[static_cast<size_t>(t)];
        const Instance& p = I.lm.inst[static_cast<size_t>(pid)];
        ck(cudaStreamWaitEvent(I.h2d, I.d2h_done[static_cast<size_t>(t)], 0), "wait");
        // region free: every earlier occupant finished (compute) and drained
        for (int q : I.preds[static_cast<size_t>(pid)]) {
          const Instance& y = I.lm.inst[static_cast<size_t>(q)];
          if (use_side && I.side_last[static_cast<size_t>(q)] > 0)
            ck(cudaStreamWaitEvent(I.h2d, I.wg_done[static_cast<size_t>(I.side_last[static_cast<size_t>(q)])], 0),
               "wait wgrad");
          if (y.kind == InstKind::act && y.swapped)
            ck(cudaStreamWaitEvent(I.h2d, I.d2h_done[static_cast<size_t>(y.tensor)], 0), "wait");
          ck(cudaStreamWaitEvent(I.h2d, I.step_done[static_cast<size_t>(y.last)], 0), "wait");
        }
        if (timed_copies) ck(cudaEventRecord(I.in_b[static_cast<size_t>(t)], I.h2d), "rec");
        transfer(I.arena + p.offset, I.host_store[static_cast<size_t>(t)],
                 static_cast<size_t>(p.bytes), cudaMemcpyHostToDevice, I.h2d, "prefetch");
        if (timed_copies) ck(cudaEventRecord(I.in_e[static_cast<size_t>(t)], I.h2d), "rec");
        ck(cudaEventRecord(I.h2d_done[static_cast<size_t>(t)], I.h2d), "record");
        order.push_back("swap_in fm" + std::to_string(t + 1));
        timeline.copies.push_back({2, t, 0, 0});
      }
      // compute: inputs that were prefetched must have landed
      const bool fwd = s <= n;
      std::vector<int> ops;
      if (fwd) {
        ops.push_back(s - 1);
      } else {
        const int o = 2 * n + 1 - s;
        if (o >= 1 && o < n) ops.push_back(o);
        if (s == 2 * n) ops.push_back(0);
      }
      for (int o : ops) {
        const Op& op = net.ops[static_cast<size_t>(o)];
        // only inputs the backward actually reads were prefetched for it (an
        // add's backward reads none; waiting there would reference the
        // previous iteration's prefetch, which stream capture rejects)
        if (!fwd && bwd_reads_input(op))
          for (int x : {op.in0, op.in1})
            if (x >= 0 && I.swapped[static_cast<size_t>(x)]) {
              ck(cudaStreamWaitEvent(cs, I.h2d_done[static_cast<size_t>(x)], 0), "wait");
              swap_wait[static_cast<size_t>(s)] = 1;
            }
      }
      cur_step = s;
      for (int inst : I.first_compute_write[static_cast<size_t>(s)]) wait_region(inst, cs, true);
      if (profile && !capture) ck(cudaEventRecord(I.phase_begin[static_cast<size_t>(s)], cs), "rec");
      for (int o : ops) {
        if (fwd)
          forward(o, s);
        else
          backward(o, s);
        ++launches;
      }
      if (profile && !capture) ck(cudaEventRecord(I.phase_end[static_cast<size_t>(s)], cs), "rec");
      ck(cudaEventRecord(I.step_done[static_cast<size_t>(s)], cs), "record");
      // swap-out: offload what this step produced
      for (int t : I.offload_at[static_cast<size_t>(s)]) {
        const Instance& a = I.lm.inst[static_cast<size_t>(I.lm.act_inst[static_cast<size_t>(t)])];
        ck(cudaStreamWaitEvent(I.d2h, I.step_done[static_cast<size_t>(s)], 0), "wait");
        if (timed_copies) ck(cudaEventRecord(I.out_b[static_cast<size_t>(t)], I.d2h), "rec");
        transfer(I.host_store[static_cast<size_t>(t)], I.arena + a.offset,
                 static_cast<size_t>(a.bytes), cudaMemcpyDeviceToHost, I.d2h, "offload");
        if (timed_copies) ck(cudaEventRecord(I.out_e[static_cast<size_t>(t)], I.d2h), "rec");
        ck(cudaEventRecord(I.d2h_done[static_cast<size_t>(t)], I.d2h), "record");
        order.push_back("swap_out fm" + std::to_string(t + 1));
        timeline.copies.push_back({1, t, 0, 0});
      }
      // completed gradient buckets (every op whose parameters lie in the
      // prefix finished its backward on both streams): all-reduce them (data
      // parallel) and apply their update while the backward continues
      if ((I.comm || overlap_update) && !fwd) {
        const long long ready = prefix_after_step[static_cast<size_t>(s)];
        if (ready - reduced >= bucket || (s == 2 * n && ready > reduced)) {
          ck(cudaStreamWaitEvent(I.comm_stream, I.step_done[static_cast<size_t>(s)], 0), "wait");
          if (last_wg > 0)
            ck(cudaStreamWaitEvent(I.comm_stream, I.wg_done[static_cast<size_t>(last_wg)], 0), "wait");
          if (I.comm) {
            const bool timed = profile && !capture && n_buckets < static_cast<int>(I.ar_begin.size());
            if (timed) ck(cudaEventRecord(I.ar_begin[static_cast<size_t>(n_buckets)], I.comm_stream), "rec");
            ckn(ncclAllReduce(I.grads + reduced, I.grads + reduced,
                              static_cast<size_t>(ready - reduced), ncclFloat, ncclSum, I.comm,
                              I.comm_stream),
                "ncclAllReduce");
            if (timed) ck(cudaEventRecord(I.ar_end[static_cast<size_t>(n_buckets++)], I.comm_stream), "rec");
          }
          if (overlap_update) {
            ckl(accudnn_sgd_update(I.params + reduced, I.grads + reduced, I.momentum_buf + reduced,
                                   ready - reduced, lr, cfg_.momentum, cfg_.weight_decay,
                                   1.0f / static_cast<float>(I.world), I.first_step ? 1 : 0,
                                   static_cast<void*>(I.comm_stream)),
                "sgd");
            ++launches;
          }
          reduced = ready;
          comm_used = true;
        }
      }
    }
    if (comm_used) {
      const bool timed = profile && !capture && I.comm;
      if (timed) ck(cudaEventRecord(I.bwd_done, cs), "rec");
      ck(cudaEventRecord(I.comm_done, I.comm_stream), "record");
      ck(cudaStreamWaitEvent(cs, I.comm_done, 0), "wait");
      if (timed) ck(cudaEventRecord(I.comm_joined, cs), "rec");
    }
    // the weight-gradient and copy streams rejoin the compute stream (graph
    // capture needs it; the update reads every gradient)
    if (last_wg > 0) ck(cudaStreamWaitEvent(cs, I.wg_done[static_cast<size_t>(last_wg)], 0), "join");
    bool any_swap = false;
    for (char c : I.swapped) any_swap = any_swap || c;
    if (any_swap) {
      ck(cudaEventRecord(I.step_done[0], I.d2h), "record");
      ck(cudaStreamWaitEvent(cs, I.step_done[0], 0), "wait");
      ck(cudaEventRecord(I.step_done[2 * n + 1], I.h2d), "record");
      ck(cudaStreamWaitEvent(cs, I.step_done[2 * n + 1], 0), "wait");
    }
    const long long updated = overlap_update ? reduced : 0;
    if (update && updated < net.n_params) {
      ckl(accudnn_sgd_update(I.params + updated, I.grads + updated, I.momentum_buf + updated,
                             net.n_params - updated, lr, cfg_.momentum, cfg_.weight_decay,
                             1.0f / static_cast<float>(I.world), I.first_step ? 1 : 0, csv),
          "sgd");
      ++launches;
    }
    return launches;
  };

  if (!images) {
    if (!host_inputs || !I.prefetched)
      throw std::invalid_argument("step without images needs a batch prefetched by the previous step");
    ck(cudaStreamWaitEvent(cs, I.input_ready, 0), "wait input");
    I.prefetched = false;
  }
  const bool graph_ok = use_graph && !profile && update && !I.first_step;
  if (!graph_ok) ck(cudaEventRecord(I.iter_begin, cs), "record");
  if (graph_ok) {
    if (host_inputs) {
      const size_t img3 = sizeof(float) * static_cast<size_t>(k) * cfg_.image * cfg_.image * net.in_c;
      if (images)
        ck(cudaMemcpyAsync(I.image_nchw, images, img3, cudaMemcpyHostToDevice, cs), "h2d images");
      ck(cudaMemcpyAsync(I.labels, labels, sizeof(int) * k, cudaMemcpyHostToDevice, cs), "h2d labels");
    } else {
      const size_t img3 = sizeof(float) * static_cast<size_t>(k) * cfg_.image * cfg_.image * net.in_c;
      ck(cudaMemcpyAsync(I.image_nchw, images, img3, cudaMemcpyDeviceToDevice, cs), "images");
      ck(cudaMemcpyAsync(I.labels, labels, sizeof(int) * k, cudaMemcpyDeviceToDevice, cs), "labels");
    }
    if (!I.graph || I.graph_lr != lr || I.graph_update != update) {
      if (I.graph) cudaGraphExecDestroy(I.graph);
      I.graph = nullptr;
      cudaGraph_t g;
      ck(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "capture");
      kernel_launches_ = enqueue_iteration(true);
      ck(cudaStreamEndCapture(cs, &g), "end capture");
      ck(cudaGraphInstantiate(&I.graph, g,
                              cfg_.stream_priority ? cudaGraphInstantiateFlagUseNodePriority : 0),
         "instantiate");
      cudaGraphDestroy(g);
      // upload the executable graph's work to the device once: without it
      // every launch streams the ~1000 nodes in behind the first one and
      // the GPU idles ~0.9 ms per ResNet-152 step (CUPTI timeline: the gap
      // after the first node)
      ck(cudaGraphUpload(I.graph, cs), "graph upload");
      I.graph_lr = lr;
      I.graph_update = update;
    }
    ck(cudaGraphLaunch(I.graph, cs), "graph launch");
  } else {
    kernel_launches_ = enqueue_iteration(false);
  }
  if (!order.empty() || I.graph == nullptr) copy_order_ = order;
  if (next_images && host_inputs) {
    // pipelined input: the next batch's H2D overlaps the rest of this step
    const size_t img3 = sizeof(float) * static_cast<size_t>(k) * cfg_.image * cfg_.image * net.in_c;
    ck(cudaStreamWaitEvent(I.input_stream, I.layout_done, 0), "wait layout");
    ck(cudaMemcpyAsync(I.image_nchw, next_images, img3, cudaMemcpyHostToDevice, I.input_stream),
       "h2d next images");
    ck(cudaEventRecord(I.input_ready, I.input_stream), "record");
    I.prefetched = true;
  }
  ck(cudaEventRecord(I.iter_end, cs), "record");
  ck(cudaMemcpyAsync(I.loss_host, I.loss, sizeof(float), cudaMemcpyDeviceToHost, cs), "loss d2h");
  ck(cudaStreamSynchronize(cs), "step");
  if (I.prefetched) ck(cudaStreamSynchronize(I.input_stream), "input");
  if (update) I.first_step = false;

  float ms = 0.f;
  ck(cudaEventElapsedTime(&ms, I.iter_begin, I.iter_end), "elapsed");
  st.loss = *I.loss_host;
  st.iter_ms = ms;
  st.peak_bytes = fixed_bytes_ + arena_bytes_ + comm_bytes_;
  for (int t = 0; t < n; ++t)
    if (I.swapped[static_cast<size_t>(t)])
      st.swapped_bytes += static_cast<unsigned long long>(
          I.lm.inst[static_cast<size_t>(I.lm.act_inst[static_cast<size_t>(t)])].bytes);
  if (profile) {
    // exposed swap time: the compute-stream gaps in front of the phases that
    // waited on a copy stream (prefetch not landed / region not drained);
    // gaps elsewhere are launch latency of the eager profiled step
    std::string tr = "phase,begin_ms,end_ms,swap_wait\n";
    double exposed = 0;
    float prev_e = 0;
    for (int s = 1; s <= 2 * n; ++s) {
      float b = 0, e = 0;
      ck(cudaEventElapsedTime(&b, I.iter_begin, I.phase_begin[static_cast<size_t>(s)]), "t");
      ck(cudaEventElapsedTime(&e, I.iter_begin, I.phase_end[static_cast<size_t>(s)]), "t");
      if (s > 1 && swap_wait[static_cast<size_t>(s)]) exposed += std::max(0.f, b - prev_e);
      prev_e = e;
      char line[112];
      std::snprintf(line, sizeof line, "%d,%.6f,%.6f,%d\n", s, b, e,
                    static_cast<int>(swap_wait[static_cast<size_t>(s)]));
      tr += line;
    }
    st.exposed_swap_ms = exposed;
    trace_ = tr;
    // real timeline in the simulator's terms (phases and copies, ns)
    auto ns = [&](cudaEvent_t e) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, I.iter_begin, e), "t");
      return static_cast<long long>(std::llround(static_cast<double>(ms) * 1e6));
    };
    timeline.kstart.assign(static_cast<size_t>(2 * n), 0);
    timeline.kend.assign(static_cast<size_t>(2 * n), 0);
    timeline.mem_at_phase.assign(static_cast<size_t>(2 * n), 0);
    for (int s = 1; s <= 2 * n; ++s) {
      timeline.kstart[static_cast<size_t>(s - 1)] = ns(I.phase_begin[static_cast<size_t>(s)]);
      timeline.kend[static_cast<size_t>(s - 1)] = ns(I.phase_end[static_cast<size_t>(s)]);
      timeline.mem_at_phase[static_cast<size_t>(s - 1)] =
          static_cast<long long>(fixed_bytes_) + I.lm.live[static_cast<size_t>(s)];
    }
    for (auto& c : timeline.copies) {
      const size_t t = static_cast<size_t>(c.tensor);
      c.start = ns(c.stream == 1 ? I.out_b[t] : I.in_b[t]);
      c.end = ns(c.stream == 1 ? I.out_e[t] : I.in_e[t]);
    }
    timeline.fixed = fixed_bytes_;
    timeline_ = timeline;
    if (I.comm && n_buckets > 0) {
      double ar = 0;
      for (int b = 0; b < n_buckets; ++b) {
        float t = 0;
        ck(cudaEventElapsedTime(&t, I.ar_begin[static_cast<size_t>(b)], I.ar_end[static_cast<size_t>(b)]), "t");
        ar += t;
      }
      float w = 0;
      ck(cudaEventElapsedTime(&w, I.bwd_done, I.comm_joined), "t");
      st.allreduce_ms = ar;
      st.exposed_allreduce_ms = std::max(0.f, w);
    }
  }
  return st;
}

}  // namespace accudnn
