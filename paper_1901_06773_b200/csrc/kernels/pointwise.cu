// HBM-bound layer kernels of the ResNet training step: batch norm (+ fused
// ReLU) forward/backward, ReLU, eltwise add, pooling, FC bias, softmax
// cross-entropy, SGD-momentum and the input layout conversion.
//
// All of them stream NHWC fp32 with 128-bit vector accesses; per-channel
// reductions use warp shuffles + shared memory inside a block and fp64
// atomics across blocks (the batch-norm sums run over up to k*112*112 rows,
// so the cross-block accumulation is kept in double to avoid cancellation
// in E[x^2] - E[x]^2).
#include <cuda_runtime.h>

#include <cstdint>

#include "accudnn_kernels.h"

namespace accudnn {
namespace {

constexpr int kThreads = 256;

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

int grid_for(long long work, int per_block, int cap = 148 * 16) {
  long long g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

// ---------------------------------------------------------------------------
// batch normalisation
// ---------------------------------------------------------------------------
// Workspace layout (doubles): [0,C) sum  [C,2C) sum of squares / sum(dy*xhat)
// then floats: [scale C][shift C]
struct BnWs {
  double* s1;
  double* s2;
  float* scale;
  float* shift;
};
BnWs bn_ws(void* ws, int C) {
  BnWs w;
  w.s1 = static_cast<double*>(ws);
  w.s2 = w.s1 + C;
  w.scale = reinterpret_cast<float*>(w.s2 + C);
  w.shift = w.scale + C;
  return w;
}

// Block tile: kLanes float4 channel groups x (256 / kLanes) row lanes.
// gridDim.x covers channel groups, gridDim.y splits the rows.
// mode 0: s1 += x, s2 += x^2
// mode 1: g = dy * relu_mask(x) ; s1 += g, s2 += g * xhat
template <int MODE>
__global__ void __launch_bounds__(kThreads) bn_reduce_kernel(
    const float* __restrict__ x, const float* __restrict__ dy, long long M, int C,
    int lanes, const float* __restrict__ mean, const float* __restrict__ invstd,
    const float* __restrict__ gamma, const float* __restrict__ beta, int relu,
    double* __restrict__ s1, double* __restrict__ s2) {
  __shared__ float red[2][kThreads][4];
  const int lane_c = threadIdx.x % lanes;
  const int lane_r = threadIdx.x / lanes;
  const int rows_per_pass = kThreads / lanes;
  const int c = (blockIdx.x * lanes + lane_c) * 4;
  const bool c_ok = c < C;
  const long long rows_per_block = (M + gridDim.y - 1) / gridDim.y;
  const long long r_begin = blockIdx.y * rows_per_block;
  const long long r_end = min(M, r_begin + rows_per_block);

  float a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
  float mu[4], is[4], ga[4], be[4];
  if (MODE == 1 && c_ok) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mu[j] = mean[c + j];
      is[j] = invstd[c + j];
      ga[j] = gamma[c + j];
      be[j] = beta[c + j];
    }
  }
  if (c_ok) {
    for (long long r = r_begin + lane_r; r < r_end; r += rows_per_pass) {
      const float4 v = *reinterpret_cast<const float4*>(x + r * C + c);
      const float xv[4] = {v.x, v.y, v.z, v.w};
      if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          a0[j] += xv[j];
          a1[j] += xv[j] * xv[j];
        }
      } else {
        const float4 d = *reinterpret_cast<const float4*>(dy + r * C + c);
        const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float xh = (xv[j] - mu[j]) * is[j];
          float g = dv[j];
          if (relu && (xh * ga[j] + be[j]) <= 0.f) g = 0.f;
          a0[j] += g;
          a1[j] += g * xh;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    red[0][threadIdx.x][j] = a0[j];
    red[1][threadIdx.x][j] = a1[j];
  }
  __syncthreads();
  if (lane_r == 0 && c_ok) {
    double t0[4] = {0, 0, 0, 0}, t1[4] = {0, 0, 0, 0};
    for (int rr = 0; rr < rows_per_pass; ++rr) {
      const int src = rr * lanes + lane_c;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        t0[j] += red[0][src][j];
        t1[j] += red[1][src][j];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      atomicAdd(&s1[c + j], t0[j]);
      atomicAdd(&s2[c + j], t1[j]);
    }
  }
}

__global__ void bn_fwd_finalize_kernel(int C, long long M, const float* gamma,
                                       const float* beta, float eps, double* s1, double* s2,
                                       float* scale, float* shift, float* save_mean,
                                       float* save_invstd, float* run_mean, float* run_var,
                                       float momentum) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double mean = s1[c] / static_cast<double>(M);
  double var = s2[c] / static_cast<double>(M) - mean * mean;
  if (var < 0) var = 0;
  const float inv = static_cast<float>(1.0 / sqrt(var + static_cast<double>(eps)));
  const float sc = gamma[c] * inv;
  scale[c] = sc;
  shift[c] = beta[c] - static_cast<float>(mean) * sc;
  if (save_mean) save_mean[c] = static_cast<float>(mean);
  if (save_invstd) save_invstd[c] = inv;
  if (run_mean && run_var && M > 1) {
    const double unbiased = var * static_cast<double>(M) / static_cast<double>(M - 1);
    run_mean[c] = (1.f - momentum) * run_mean[c] + momentum * static_cast<float>(mean);
    run_var[c] = (1.f - momentum) * run_var[c] + momentum * static_cast<float>(unbiased);
  }
}

__global__ void __launch_bounds__(kThreads) bn_apply_kernel(
    const float* __restrict__ x, long long total4, int C4, const float* __restrict__ scale,
    const float* __restrict__ shift, int relu, float* __restrict__ y) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C4) * 4;
    float4 v = reinterpret_cast<const float4*>(x)[i];
    const float4 sc = *reinterpret_cast<const float4*>(scale + c);
    const float4 sh = *reinterpret_cast<const float4*>(shift + c);
    v.x = v.x * sc.x + sh.x;
    v.y = v.y * sc.y + sh.y;
    v.z = v.z * sc.z + sh.z;
    v.w = v.w * sc.w + sh.w;
    if (relu) {
      v.x = fmaxf(v.x, 0.f);
      v.y = fmaxf(v.y, 0.f);
      v.z = fmaxf(v.z, 0.f);
      v.w = fmaxf(v.w, 0.f);
    }
    reinterpret_cast<float4*>(y)[i] = v;
  }
}

__global__ void bn_bwd_finalize_kernel(int C, const double* s1, const double* s2,
                                       float* dgamma, float* dbeta) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  dbeta[c] = static_cast<float>(s1[c]);
  dgamma[c] = static_cast<float>(s2[c]);
}

// dx = gamma*invstd * (g - mean(g) - xhat * mean(g*xhat))
__global__ void __launch_bounds__(kThreads) bn_bwd_dx_kernel(
    const float* __restrict__ x, const float* __restrict__ dy, long long total4, int C4,
    long long M, const float* __restrict__ gamma, const float* __restrict__ beta,
    const float* __restrict__ mean, const float* __restrict__ invstd,
    const double* __restrict__ s1, const double* __restrict__ s2, int relu,
    float* __restrict__ dx, int dx_beta) {
  const float invM = 1.f / static_cast<float>(M);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C4) * 4;
    const float4 xv4 = reinterpret_cast<const float4*>(x)[i];
    const float4 dv4 = reinterpret_cast<const float4*>(dy)[i];
    const float xv[4] = {xv4.x, xv4.y, xv4.z, xv4.w};
    const float dv[4] = {dv4.x, dv4.y, dv4.z, dv4.w};
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float is = invstd[c + j], ga = gamma[c + j];
      const float xh = (xv[j] - mean[c + j]) * is;
      float g = dv[j];
      if (relu && (xh * ga + beta[c + j]) <= 0.f) g = 0.f;
      const float mg = static_cast<float>(s1[c + j]) * invM;
      const float mgx = static_cast<float>(s2[c + j]) * invM;
      o[j] = ga * is * (g - mg - xh * mgx);
    }
    float4 r = make_float4(o[0], o[1], o[2], o[3]);
    if (dx_beta) {
      const float4 old = reinterpret_cast<float4*>(dx)[i];
      r.x += old.x;
      r.y += old.y;
      r.z += old.z;
      r.w += old.w;
    }
    reinterpret_cast<float4*>(dx)[i] = r;
  }
}

void bn_reduce_launch_dims(long long M, int C, int* lanes, dim3* grid) {
  int l = C / 4;
  if (l > 32) l = 32;
  if (l < 1) l = 1;
  *lanes = l;
  const int cgroups = (C / 4 + l - 1) / l;
  // enough row splits for ~8 blocks per SM overall, each >= 64 rows
  long long ysplit = (148LL * 8 + cgroups - 1) / cgroups;
  const long long max_split = (M + 63) / 64;
  if (ysplit > max_split) ysplit = max_split;
  if (ysplit < 1) ysplit = 1;
  *grid = dim3(cgroups, static_cast<unsigned>(ysplit));
}

// ---------------------------------------------------------------------------
// elementwise
// ---------------------------------------------------------------------------
__global__ void relu_fwd_kernel(const float4* __restrict__ x, float4* __restrict__ y,
                                long long n4) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 v = x[i];
    v.x = fmaxf(v.x, 0.f);
    v.y = fmaxf(v.y, 0.f);
    v.z = fmaxf(v.z, 0.f);
    v.w = fmaxf(v.w, 0.f);
    y[i] = v;
  }
}

__global__ void relu_bwd_kernel(const float4* __restrict__ x, const float4* __restrict__ dy,
                                float4* __restrict__ dx, long long n4, int beta) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    const float4 d = dy[i];
    float4 o = make_float4(v.x > 0.f ? d.x : 0.f, v.y > 0.f ? d.y : 0.f,
                           v.z > 0.f ? d.z : 0.f, v.w > 0.f ? d.w : 0.f);
    if (beta) {
      const float4 old = dx[i];
      o.x += old.x;
      o.y += old.y;
      o.z += old.z;
      o.w += old.w;
    }
    dx[i] = o;
  }
}

__global__ void add_kernel(const float4* __restrict__ a, const float4* __restrict__ b,
                           float4* __restrict__ y, long long n4) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 u = a[i], v = b[i];
    y[i] = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
  }
}

__global__ void copy_kernel(const float4* __restrict__ s, float4* __restrict__ d, long long n4,
                            int beta) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 v = s[i];
    if (beta) {
      const float4 o = d[i];
      v.x += o.x;
      v.y += o.y;
      v.z += o.z;
      v.w += o.w;
    }
    d[i] = v;
  }
}

// ---------------------------------------------------------------------------
// pooling
// ---------------------------------------------------------------------------
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, int n, int h, int w, int c4,
                                   int kr, int ks, int stride, int pad, int p, int q,
                                   float* __restrict__ y) {
  const long long total = static_cast<long long>(n) * p * q * c4;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cg = static_cast<int>(i % c4);
    long long t = i / c4;
    const int qq = static_cast<int>(t % q);
    t /= q;
    const int pp = static_cast<int>(t % p);
    const int nn = static_cast<int>(t / p);
    float4 best = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    for (int r = 0; r < kr; ++r) {
      const int hh = pp * stride - pad + r;
      if (hh < 0 || hh >= h) continue;
      for (int s = 0; s < ks; ++s) {
        const int ww = qq * stride - pad + s;
        if (ww < 0 || ww >= w) continue;
        const float4 v = reinterpret_cast<const float4*>(
            x)[((static_cast<long long>(nn) * h + hh) * w + ww) * c4 + cg];
        best.x = fmaxf(best.x, v.x);
        best.y = fmaxf(best.y, v.y);
        best.z = fmaxf(best.z, v.z);
        best.w = fmaxf(best.w, v.w);
      }
    }
    reinterpret_cast<float4*>(y)[i] = best;
  }
}

// gradient routed to the first maximum of each window (row-major scan),
// recomputed from the input; one thread per input element
__global__ void maxpool_bwd_kernel(const float* __restrict__ x, const float* __restrict__ dy,
                                   int n, int h, int w, int c, int kr, int ks, int stride,
                                   int pad, int p, int q, float* __restrict__ dx) {
  const long long total = static_cast<long long>(n) * h * w * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cc = static_cast<int>(i % c);
    long long t = i / c;
    const int ww = static_cast<int>(t % w);
    t /= w;
    const int hh = static_cast<int>(t % h);
    const int nn = static_cast<int>(t / h);
    float acc = 0.f;
    const int p_lo = max(0, (hh + pad - kr + stride) / stride);
    const int p_hi = min(p - 1, (hh + pad) / stride);
    const int q_lo = max(0, (ww + pad - ks + stride) / stride);
    const int q_hi = min(q - 1, (ww + pad) / stride);
    for (int pp = p_lo; pp <= p_hi; ++pp) {
      for (int qq = q_lo; qq <= q_hi; ++qq) {
        // recompute the window argmax
        float best = -INFINITY;
        int bh = -1, bw = -1;
        for (int r = 0; r < kr; ++r) {
          const int ih = pp * stride - pad + r;
          if (ih < 0 || ih >= h) continue;
          for (int s = 0; s < ks; ++s) {
            const int iw = qq * stride - pad + s;
            if (iw < 0 || iw >= w) continue;
            const float v = x[((static_cast<long long>(nn) * h + ih) * w + iw) * c + cc];
            if (v > best) {
              best = v;
              bh = ih;
              bw = iw;
            }
          }
        }
        if (bh == hh && bw == ww)
          acc += dy[((static_cast<long long>(nn) * p + pp) * q + qq) * c + cc];
      }
    }
    dx[i] = acc;
  }
}

__global__ void avgpool_fwd_kernel(const float* __restrict__ x, int n, int hw, int c,
                                   float* __restrict__ y) {
  const int total = n * c;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int nn = i / c, cc = i - nn * c;
    const float* base = x + static_cast<long long>(nn) * hw * c + cc;
    float acc = 0.f;
    for (int j = 0; j < hw; ++j) acc += base[static_cast<long long>(j) * c];
    y[i] = acc / static_cast<float>(hw);
  }
}

__global__ void avgpool_bwd_kernel(const float* __restrict__ dy, int n, int hw, int c,
                                   float* __restrict__ dx) {
  const long long total = static_cast<long long>(n) * hw * c;
  const float inv = 1.f / static_cast<float>(hw);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cc = static_cast<int>(i % c);
    const long long nn = i / (static_cast<long long>(hw) * c);
    dx[i] = dy[nn * c + cc] * inv;
  }
}

// ---------------------------------------------------------------------------
// classifier
// ---------------------------------------------------------------------------
__global__ void bias_add_kernel(float* y, const float* b, long long m, int n) {
  const long long total = m * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    y[i] += b[i % n];
}

__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one warp per row
__global__ void xent_kernel(const float* __restrict__ logits, const int* __restrict__ labels,
                            int rows, int classes, float* loss, float* dlogits,
                            float* dbias) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* z = logits + static_cast<long long>(row) * classes;
  float mx = -INFINITY;
  for (int j = lane; j < classes; j += 32) mx = fmaxf(mx, z[j]);
  mx = warp_max(mx);
  float se = 0.f;
  for (int j = lane; j < classes; j += 32) se += expf(z[j] - mx);
  se = warp_sum(se);
  const int y = labels[row];
  if (loss && lane == 0) {
    const float lse = mx + logf(se);
    atomicAdd(loss, (lse - z[y]) / static_cast<float>(rows));
  }
  if (dlogits) {
    const float inv = 1.f / se;
    float* d = dlogits + static_cast<long long>(row) * classes;
    for (int j = lane; j < classes; j += 32) {
      const float g = (expf(z[j] - mx) * inv - (j == y ? 1.f : 0.f)) / static_cast<float>(rows);
      d[j] = g;
      if (dbias) atomicAdd(&dbias[j], g);
    }
  }
}

// ---------------------------------------------------------------------------
// optimizer / layout
// ---------------------------------------------------------------------------
__global__ void sgd_kernel(float4* __restrict__ w, const float4* __restrict__ g,
                           float4* __restrict__ buf, long long n4, float lr, float mu, float wd,
                           float gscale, int first) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 wv = w[i];
    const float4 gv = g[i];
    float4 b = first ? make_float4(0, 0, 0, 0) : buf[i];
    const float d[4] = {gv.x * gscale + wd * wv.x, gv.y * gscale + wd * wv.y,
                        gv.z * gscale + wd * wv.z, gv.w * gscale + wd * wv.w};
    if (first) {
      b = make_float4(d[0], d[1], d[2], d[3]);
    } else {
      b.x = mu * b.x + d[0];
      b.y = mu * b.y + d[1];
      b.z = mu * b.z + d[2];
      b.w = mu * b.w + d[3];
    }
    wv.x -= lr * b.x;
    wv.y -= lr * b.y;
    wv.z -= lr * b.z;
    wv.w -= lr * b.w;
    buf[i] = b;
    w[i] = wv;
  }
}

__global__ void nchw_to_nhwc_kernel(const float* __restrict__ x, int n, int c, int h, int w,
                                    int c4, float* __restrict__ y) {
  const long long total = static_cast<long long>(n) * h * w * c4;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cc = static_cast<int>(i % c4);
    long long t = i / c4;
    const int ww = static_cast<int>(t % w);
    t /= w;
    const int hh = static_cast<int>(t % h);
    const int nn = static_cast<int>(t / h);
    y[i] = cc < c ? x[((static_cast<long long>(nn) * c + cc) * h + hh) * w + ww] : 0.f;
  }
}

}  // namespace
}  // namespace accudnn

using namespace accudnn;

extern "C" unsigned long long accudnn_bn_workspace_bytes(int C) {
  return static_cast<unsigned long long>(C) * (2 * sizeof(double) + 2 * sizeof(float));
}

extern "C" int accudnn_bn_fwd(const float* x, long long M, int C, const float* gamma,
                              const float* beta, float eps, int relu, float* y,
                              float* save_mean, float* save_invstd, float* running_mean,
                              float* running_var, float momentum, void* ws, void* stream) {
  if ((C & 3) || M <= 0) return static_cast<int>(cudaErrorInvalidValue);
  const BnWs w = bn_ws(ws, C);
  cudaStream_t st = S(stream);
  cudaMemsetAsync(w.s1, 0, 2 * sizeof(double) * C, st);
  int lanes;
  dim3 grid;
  bn_reduce_launch_dims(M, C, &lanes, &grid);
  bn_reduce_kernel<0><<<grid, kThreads, 0, st>>>(x, nullptr, M, C, lanes, nullptr, nullptr,
                                                 nullptr, nullptr, 0, w.s1, w.s2);
  bn_fwd_finalize_kernel<<<(C + 255) / 256, 256, 0, st>>>(
      C, M, gamma, beta, eps, w.s1, w.s2, w.scale, w.shift, save_mean, save_invstd,
      running_mean, running_var, momentum);
  const long long total4 = M * C / 4;
  bn_apply_kernel<<<grid_for(total4, kThreads), kThreads, 0, st>>>(x, total4, C / 4, w.scale,
                                                                   w.shift, relu, y);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_bn_bwd(const float* x, const float* dy, long long M, int C,
                              const float* gamma, const float* beta, const float* save_mean,
                              const float* save_invstd, int relu, float* dx, int dx_beta,
                              float* dgamma, float* dbeta, void* ws, void* stream) {
  if ((C & 3) || M <= 0) return static_cast<int>(cudaErrorInvalidValue);
  const BnWs w = bn_ws(ws, C);
  cudaStream_t st = S(stream);
  cudaMemsetAsync(w.s1, 0, 2 * sizeof(double) * C, st);
  int lanes;
  dim3 grid;
  bn_reduce_launch_dims(M, C, &lanes, &grid);
  bn_reduce_kernel<1><<<grid, kThreads, 0, st>>>(x, dy, M, C, lanes, save_mean, save_invstd,
                                                 gamma, beta, relu, w.s1, w.s2);
  if (dgamma && dbeta)
    bn_bwd_finalize_kernel<<<(C + 255) / 256, 256, 0, st>>>(C, w.s1, w.s2, dgamma, dbeta);
  const long long total4 = M * C / 4;
  bn_bwd_dx_kernel<<<grid_for(total4, kThreads), kThreads, 0, st>>>(
      x, dy, total4, C / 4, M, gamma, beta, save_mean, save_invstd, w.s1, w.s2, relu, dx,
      dx_beta);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_relu_fwd(const float* x, float* y, long long n, void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  relu_fwd_kernel<<<grid_for(n / 4, kThreads), kThreads, 0, S(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), n / 4);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_relu_bwd(const float* x, const float* dy, float* dx, long long n,
                                int dx_beta, void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  relu_bwd_kernel<<<grid_for(n / 4, kThreads), kThreads, 0, S(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(dy),
      reinterpret_cast<float4*>(dx), n / 4, dx_beta);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_add_fwd(const float* a, const float* b, float* y, long long n,
                               void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  add_kernel<<<grid_for(n / 4, kThreads), kThreads, 0, S(stream)>>>(
      reinterpret_cast<const float4*>(a), reinterpret_cast<const float4*>(b),
      reinterpret_cast<float4*>(y), n / 4);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_copy(const float* src, float* dst, long long n, int beta, void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  copy_kernel<<<grid_for(n / 4, kThreads), kThreads, 0, S(stream)>>>(
      reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), n / 4, beta);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_maxpool_fwd(const float* x, int n, int h, int w, int c, int kr, int ks,
                                   int stride, int pad, int p, int q, float* y, void* stream) {
  if (c & 3) return static_cast<int>(cudaErrorInvalidValue);
  const long long total = static_cast<long long>(n) * p * q * (c / 4);
  maxpool_fwd_kernel<<<grid_for(total, kThreads), kThreads, 0, S(stream)>>>(
      x, n, h, w, c / 4, kr, ks, stride, pad, p, q, y);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_maxpool_bwd(const float* x, const float* dy, int n, int h, int w, int c,
                                   int kr, int ks, int stride, int pad, int p, int q, float* dx,
                                   void* stream) {
  const long long total = static_cast<long long>(n) * h * w * c;
  maxpool_bwd_kernel<<<grid_for(total, kThreads), kThreads, 0, S(stream)>>>(
      x, dy, n, h, w, c, kr, ks, stride, pad, p, q, dx);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_avgpool_fwd(const float* x, int n, int hw, int c, float* y,
                                   void* stream) {
  avgpool_fwd_kernel<<<grid_for(static_cast<long long>(n) * c, kThreads), kThreads, 0,
                       S(stream)>>>(x, n, hw, c, y);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_avgpool_bwd(const float* dy, int n, int hw, int c, float* dx,
                                   void* stream) {
  avgpool_bwd_kernel<<<grid_for(static_cast<long long>(n) * hw * c, kThreads), kThreads, 0,
                       S(stream)>>>(dy, n, hw, c, dx);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_bias_add(float* y, const float* bias, long long m, int n, void* stream) {
  bias_add_kernel<<<grid_for(m * n, kThreads), kThreads, 0, S(stream)>>>(y, bias, m, n);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_xent_fwd(const float* logits, const int* labels, int rows, int classes,
                                float* loss, void* stream) {
  cudaMemsetAsync(loss, 0, sizeof(float), S(stream));
  xent_kernel<<<(rows + 7) / 8, 256, 0, S(stream)>>>(logits, labels, rows, classes, loss,
                                                    nullptr, nullptr);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_xent_bwd(const float* logits, const int* labels, int rows, int classes,
                                float* dlogits, float* dbias, void* stream) {
  if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * classes, S(stream));
  xent_kernel<<<(rows + 7) / 8, 256, 0, S(stream)>>>(logits, labels, rows, classes, nullptr,
                                                    dlogits, dbias);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_sgd_update(float* w, const float* g, float* buf, long long n, float lr,
                                  float momentum, float weight_decay, float grad_scale,
                                  int first_step, void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  sgd_kernel<<<grid_for(n / 4, kThreads), kThreads, 0, S(stream)>>>(
      reinterpret_cast<float4*>(w), reinterpret_cast<const float4*>(g),
      reinterpret_cast<float4*>(buf), n / 4, lr, momentum, weight_decay, grad_scale,
      first_step);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_nchw_to_nhwc_pad(const float* x, int n, int c, int h, int w, int c4,
                                        float* y, void* stream) {
  const long long total = static_cast<long long>(n) * h * w * c4;
  nchw_to_nhwc_kernel<<<grid_for(total, kThreads), kThreads, 0, S(stream)>>>(x, n, c, h, w, c4,
                                                                            y);
  return static_cast<int>(cudaGetLastError());
}
