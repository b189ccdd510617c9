/*
 * accudnn.h -- C ABI of the B200 training-step executor (libaccudnn.so).
 *
 * The reference (`swapsched`) stops at the plan: its simulator
 * (/root/reference/proj/include/swapsched/simulator.hpp:73-76,
 * simulate_iteration) only *models* the runtime memory manager of the paper
 * (PAPER.md:282-289).  These entry points are that runtime on a B200:
 * network export in the reference's network.json format, an executor that
 * realises a plan.json (pin set + k*) with real compute / swap-out / swap-in
 * CUDA streams under a hard device cap, and one training step (forward,
 * backward, bucketed NCCL all-reduce, SGD) per call.  Layer kernels are in
 * accudnn_kernels.h.  Return values are cudaError_t-compatible codes; 1 =
 * invalid input / infeasible (message in accudnn_rt_last_error()).
 */
#ifndef ACCUDNN_H_
#define ACCUDNN_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct accudnn_exec accudnn_exec;

typedef struct accudnn_step_stats {
  float loss;                       /* mean softmax cross-entropy of the batch */
  double iter_ms;                   /* device time of the iteration            */
  double exposed_swap_ms;           /* compute-stream stall (profiled steps)   */
  double allreduce_ms;              /* NCCL all-reduce device time, summed over
                                       the gradient buckets (profiled steps)   */
  unsigned long long peak_bytes;    /* fixed allocations + arena (+ NCCL)      */
  unsigned long long swapped_bytes; /* featuremap bytes offloaded per step     */
  double exposed_allreduce_ms;      /* compute-stream wait at the all-reduce
                                       join after the last backward phase
                                       (profiled steps): the reference's
                                       delta_sync_s (model_ir.hpp:108)         */
} accudnn_step_stats;

const char* accudnn_rt_last_error(void);
void accudnn_rt_free(void* p);

/* reference-format network.json (workspace accounting included) and an op
 * description (JSON) for tooling / the torch oracle */
int accudnn_net_export(const char* arch, int image, int classes, int k_base, int lookahead,
                       char** network_json, char** describe_json);

/* executor memory model without a GPU: peak live bytes of the real tensor
 * instances and the static arena size for a swap mask (one char per op,
 * nonzero = featuremap offloaded) at minibatch k */
int accudnn_net_memory(const char* arch, int image, int classes, int k, int lookahead,
                       const char* swapped_mask, long long* live_peak, long long* arena_bytes);

/* mode: "resident" (nothing swapped), "naive" (every featuremap swapped) or
 * "dynamic" (plan_json's pinned_objects stay, the rest swap).  k = 0 takes
 * plan_json's k_star.  hardware_json (may be NULL) supplies the device cap
 * and m_others; network_json (may be NULL) the planner's fixed overhead. */
int accudnn_exec_create(const char* arch, int image, int classes, const char* mode,
                        const char* network_json, const char* hardware_json,
                        const char* plan_json, int k, int device, int lookahead,
                        accudnn_exec** out);
int accudnn_exec_destroy(accudnn_exec* ex);
long long accudnn_exec_num_params(accudnn_exec* ex);
long long accudnn_exec_num_stats(accudnn_exec* ex);
int accudnn_exec_set_params(accudnn_exec* ex, const float* host, long long n);
int accudnn_exec_get_params(accudnn_exec* ex, float* host, long long n);
int accudnn_exec_get_grads(accudnn_exec* ex, float* host, long long n);
int accudnn_exec_get_stats(accudnn_exec* ex, float* host, long long n);
int accudnn_exec_set_graph(accudnn_exec* ex, int enable);
/* images NCHW fp32 [k][3][H][W], labels int32 [k]; host_inputs = 1 when both
 * are host pointers (copied inside the step), 0 when device pointers */
int accudnn_exec_step(accudnn_exec* ex, const float* images, const int* labels, int host_inputs,
                      float lr, int update, int profile, accudnn_step_stats* out);
/* pipelined host input: images == NULL uses the batch the previous call
 * prefetched; next_images (host, may be NULL) is copied H2D on a side stream
 * as soon as this step's input layout kernel has consumed the staging buffer,
 * overlapping the rest of the step.  Labels are copied inside the step. */
int accudnn_exec_step_pipelined(accudnn_exec* ex, const float* images, const int* labels,
                                float lr, int update, const float* next_images,
                                accudnn_step_stats* out);
int accudnn_exec_memory(accudnn_exec* ex, unsigned long long* arena_bytes,
                        unsigned long long* fixed_bytes);
int accudnn_exec_launches(accudnn_exec* ex);
int accudnn_exec_trace(accudnn_exec* ex, char** csv);
/* documents of the last profiled step in the reference simulator's schemas
 * (/root/reference/proj/src/simulator.cpp:419-473), from CUDA events on every
 * phase and copy: which = "trace" (trace.csv), "mem_curves", "stall_bars",
 * "summary" (summary.json); "order" = the copies of an iteration in stream
 * order, one "swap_out fmN" / "swap_in fmN" per line.  Free with
 * accudnn_rt_free. */
int accudnn_exec_document(accudnn_exec* ex, const char* which, char** out);
/* data parallel: 128-byte NCCL unique id from rank 0, shared by the host */
int accudnn_nccl_unique_id(void* out128);
int accudnn_exec_set_comm(accudnn_exec* ex, const void* uid128, int rank, int world);
/* device bytes held by the NCCL communicator (0 before set_comm) */
unsigned long long accudnn_exec_comm_bytes(accudnn_exec* ex);

#ifdef __cplusplus
}
#endif

#endif /* ACCUDNN_H_ */
