/*
 * accudnn_kernels.h -- C ABI of the sm_100a layer kernels (libaccudnn.so).
 *
 * The reference has no layer implementation at all: its layers are FLOP and
 * byte descriptors (LayerType conv/bn/activation/pooling/fc/other,
 * /root/reference/proj/include/swapsched/model_ir.hpp:14-32) whose execution
 * the paper delegates to Caffe/cuDNN.  These launchers are
 * the B200 kernels behind those descriptors.  All tensors are NHWC fp32 in
 * device memory; channel counts must be multiples of 4 (16-byte chunks).
 * Every launcher is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 * default) and returns a cudaError_t value (0 = success).
 */
#ifndef ACCUDNN_KERNELS_H_
#define ACCUDNN_KERNELS_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct accudnn_conv_desc {
  int n, h, w, c;   /* input batch, height, width, channels (c % 4 == 0) */
  int k;            /* output channels (k % 4 == 0)                      */
  int r, s;         /* filter height, width                               */
  int stride, pad;  /* symmetric                                          */
  int p, q;         /* output height, width                               */
} accudnn_conv_desc;

/* implicit-GEMM convolution on tcgen05 (TF32 in, FP32 accumulate in TMEM).
 * beta = 1 accumulates into the output instead of overwriting it. */
int accudnn_conv_fwd(const accudnn_conv_desc* d, const float* x, const float* w,
                     float* y, int beta, void* stream);
/* forward convolution that also writes the batch-norm statistics of its
 * output: per-32-row column sums and sums of squares, [2][ceil(M/32)][k]
 * floats (M = n*p*q).  *produced = 0 if the shape ran on the cp.async kernel
 * (then nothing was written to `stats`). */
int accudnn_conv_fwd_stats(const accudnn_conv_desc* d, const float* x, const float* w,
                           float* y, float* stats, int* produced, void* stream);
int accudnn_conv_dgrad(const accudnn_conv_desc* d, const float* dy, const float* w,
                       float* dx, int beta, void* stream);
/* process-wide convolution math: 0 = TF32 tensor cores (default),
 * 1 = 3xTF32 (hi/lo operand split, ~FP32 accuracy, 3x MMA work) */
int accudnn_set_conv_math(int mode);
int accudnn_get_conv_math(void);
/* 3xTF32 on the TMA kernels: scratch for the operands' low parts
 * (lo = v - tf32(v)) of the convolutions launched on `stream`; with it a
 * precise convolution runs as three TF32 tcgen05 GEMMs (hi*hi + hi*lo +
 * lo*hi accumulated into the output), without it on the cp.async kernel.
 * ptr == NULL removes the entry.  accudnn_conv_precise_scratch_bytes: the
 * bytes one convolution of shape d needs (max over fwd / dgrad / wgrad). */
int accudnn_conv_set_precise_scratch(void* stream, void* ptr, unsigned long long bytes);
unsigned long long accudnn_conv_precise_scratch_bytes(const accudnn_conv_desc* d);
/* 1 = TMA-fed kernels where the shape allows (default), 0 = cp.async kernel only */
int accudnn_set_conv_impl(int impl);
/* split-K workspace of the persistent TMA kernels (deterministic fix-up:
 * partials are summed in slice order).  ptr == NULL: bytes > 0 restores a
 * lazily allocated default of that size (64 MiB initially), bytes == 0
 * disables split-K.  Splits are limited so that splits * M * N * 4 <= bytes. */
int accudnn_conv_set_workspace(void* ptr, unsigned long long bytes);
/* split-K workspace for convolutions launched on one particular stream (a
 * concurrent weight-gradient stream) and a cap on their persistent grids
 * (max_ctas SMs, 0 = all); ptr == NULL and max_ctas == 0 removes the entry */
int accudnn_conv_set_stream_workspace(void* stream, void* ptr, unsigned long long bytes,
                                      int max_ctas);
/* programmatic dependent launch for every kernel (default 0): the next
 * kernel's prologue overlaps the previous one's tail.  Returns the previous. */
int accudnn_set_pdl(int enable);
/* debug: TMA-conv launches record per-CTA clock64 stamps into buf (1024 x
 * int64 per CTA, see conv_sm100.cu); NULL turns it off */
int accudnn_conv_trace(void* buf);
/* 1: tune (tile width, split-K) per convolution shape on its first
 * overwrite (beta = 0) call outside stream capture -- every candidate is
 * timed with CUDA events and the fastest is cached for the process; 0: the
 * analytic choice.  Returns the previous setting. */
int accudnn_conv_autotune(int enable);
/* the autotuner's table as text (one "key[14] bn splits" line per shape;
 * malloc'ed, release with free) and its inverse (merges, overwriting), so a
 * tuned table can be shipped with a plan and runs are reproducible */
int accudnn_conv_tune_export(char** text);
int accudnn_conv_tune_import(const char* text);
/* test hook: force tile width (64/128/256), split-K factor and cluster size
 * (1, 2 = B tile multicast across an M-tile pair, 3 = B-stationary: the
 * N-tile's whole B kept in shared memory) for every TMA conv
 * launch; 0 fields = automatic */
int accudnn_conv_force_cfg(int bn, int splits, int cm);
/* splits <= 0 picks a split-K factor automatically (TMA path: deterministic
 * workspace fix-up; cp.async fallback: fp32 atomics) */
int accudnn_conv_wgrad(const accudnn_conv_desc* d, const float* x, const float* dy,
                       float* dw, int beta, int splits, void* stream);

/* batch normalisation over the M = n*h*w rows of an [M][C] tensor, training
 * mode; optional fused ReLU.  `ws` needs accudnn_bn_workspace_bytes(C) bytes,
 * zeroed once before first use (the reductions keep their arrival counters
 * there and re-arm them); one workspace per stream. */
unsigned long long accudnn_bn_workspace_bytes(int C);
int accudnn_bn_fwd(const float* x, long long M, int C, const float* gamma,
                   const float* beta, float eps, int relu, float* y,
                   float* save_mean, float* save_invstd, float* running_mean,
                   float* running_var, float momentum, void* ws, void* stream);
/* backward from the BN *input* x (the ReLU mask is recomputed from x) */
int accudnn_bn_bwd(const float* x, const float* dy, long long M, int C,
                   const float* gamma, const float* beta, const float* save_mean,
                   const float* save_invstd, int relu, float* dx, int dx_beta,
                   float* dgamma, float* dbeta, void* ws, void* stream);

/* the residual tail of a ResNet block as one op: y = relu(bn(x) + skip)
 * (training-mode BN over [M][C]); backward recomputes the mask from the
 * inputs and writes both gradients (dx: BN backward, dskip: masked dy;
 * each accumulates when its beta flag is 1). */
/* the forward batch norms with their statistics precomputed by
 * accudnn_conv_fwd_stats (only the normalise pass reads x) */
int accudnn_bn_fwd_stats(const float* x, const float* stats, long long M, int C,
                         const float* gamma, const float* beta, float eps, int relu, float* y,
                         float* save_mean, float* save_invstd, float* running_mean,
                         float* running_var, float momentum, void* ws, void* stream);
int accudnn_bn_add_relu_fwd_stats(const float* x, const float* stats, const float* skip,
                                  long long M, int C, const float* gamma, const float* beta,
                                  float eps, float* y, float* save_mean, float* save_invstd,
                                  float* running_mean, float* running_var, float momentum,
                                  void* ws, void* stream);
int accudnn_bn_add_relu_fwd(const float* x, const float* skip, long long M, int C,
                            const float* gamma, const float* beta, float eps, float* y,
                            float* save_mean, float* save_invstd, float* running_mean,
                            float* running_var, float momentum, void* ws, void* stream);
int accudnn_bn_add_relu_bwd(const float* x, const float* skip, const float* dy, long long M,
                            int C, const float* gamma, const float* beta,
                            const float* save_mean, const float* save_invstd, float* dx,
                            int dx_beta, float* dskip, int dskip_beta, float* dgamma,
                            float* dbeta, void* ws, void* stream);
/* y = relu(x * sc + sh), sc = gamma * save_invstd, sh = beta - save_mean * sc:
 * a bn_relu forward's output recomputed bit for bit from its saved statistics
 * (transient activations, recomputed for the consuming conv's weight gradient) */
int accudnn_bn_relu_apply(const float* x, long long M, int C, const float* gamma,
                          const float* beta, const float* save_mean, const float* save_invstd,
                          float* y, void* stream);
int accudnn_relu_fwd(const float* x, float* y, long long n, void* stream);
/* dx (+)= dy * (x > 0) */
int accudnn_relu_bwd(const float* x, const float* dy, float* dx, long long n,
                     int dx_beta, void* stream);
int accudnn_add_fwd(const float* a, const float* b, float* y, long long n, void* stream);
int accudnn_copy(const float* src, float* dst, long long n, int beta, void* stream);

/* max pooling, window kr x ks, stride, pad; NHWC */
int accudnn_maxpool_fwd(const float* x, int n, int h, int w, int c, int kr, int ks,
                        int stride, int pad, int p, int q, float* y, void* stream);
int accudnn_maxpool_bwd(const float* x, const float* dy, int n, int h, int w, int c,
                        int kr, int ks, int stride, int pad, int p, int q, float* dx,
                        void* stream);
/* global average pooling [n][hw][c] -> [n][c] and back */
int accudnn_avgpool_fwd(const float* x, int n, int hw, int c, float* y, void* stream);
int accudnn_avgpool_bwd(const float* dy, int n, int hw, int c, float* dx, void* stream);

/* y[m][j] += bias[j] */
int accudnn_bias_add(float* y, const float* bias, long long m, int n, void* stream);
/* mean softmax cross-entropy over `rows` rows of `classes` logits; writes the
 * mean loss to *loss (device scalar) */
int accudnn_xent_fwd(const float* logits, const int* labels, int rows, int classes,
                     float* loss, void* stream);
/* dlogits = (softmax - onehot) / rows ; dbias = column sums of dlogits */
int accudnn_xent_bwd(const float* logits, const int* labels, int rows, int classes,
                     float* dlogits, float* dbias, void* stream);

/* SGD with momentum and weight decay over a flat parameter buffer
 * (PyTorch semantics: buf = mu*buf + (g*grad_scale + wd*w); w -= lr*buf;
 * first_step initialises buf = d_p). */
int accudnn_sgd_update(float* w, const float* g, float* buf, long long n, float lr,
                       float momentum, float weight_decay, float grad_scale,
                       int first_step, void* stream);

/* featuremap transfer between device memory and pinned (host-mapped) host
 * memory by an SM-driven copy kernel: `bytes` from src to dst in either
 * direction, ctas <= 0 = 16 CTAs.  The swap executor's path for transfers
 * below ~2 MB (D2H) / 512 KB (H2D), where a copy-engine memcpy's per-call
 * latency dominates (kernels/swap_copy.cu). */
int accudnn_swap_copy(void* dst, const void* src, unsigned long long bytes, int ctas,
                      void* stream);

/* NCHW fp32 images with `c` channels -> NHWC with `c4` (>= c, zero padded) */
int accudnn_nchw_to_nhwc_pad(const float* x, int n, int c, int h, int w, int c4,
                             float* y, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ACCUDNN_KERNELS_H_ */
