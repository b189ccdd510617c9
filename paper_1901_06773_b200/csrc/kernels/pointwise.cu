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
// Per-channel reductions are deterministic (no atomics on data): the grid is
// (channel groups of <= 128 channels) x (Y row splits); every block writes
// its partial sums to its own slot part[y][2][128-channel group].  Slots are
// combined in two fixed-shape levels: the last block to arrive in each team
// of kBnTeam consecutive row splits sums the team's slots in order into a
// team slot, and the last team of a channel group sums the team slots in
// order in double precision and finalises (arrival counters are re-armed by
// the blocks that consumed them):
//   mode 0 (forward):  mean, invstd, scale = gamma*invstd, shift, running stats
//   mode 1 (backward): s1 = sum g, s2 = sum g*xhat (g = dy * relu mask) ->
//                      dbeta, dgamma and the two sums for the dx kernel.
// Workspace layout: counters (uint) [kBnMaxGroups * (1 + kBnMaxTeams)] |
//   part (float) [kBnMaxBlocks][2][128] | tpart [kBnMaxBlocks][2][128] |
//   scale[C] | shift[C] | sum1[C] | sum2[C]
constexpr int kBnGroup = 128;        // channels per channel group
constexpr int kBnMaxBlocks = 1024;   // x * Y
constexpr int kBnMaxGroups = 64;     // C <= 8192
constexpr int kBnTeam = 16;          // row splits per first-level team
constexpr int kBnMaxTeams = kBnMaxBlocks / kBnTeam;
constexpr int kBnCounters = kBnMaxGroups * (1 + kBnMaxTeams);

struct BnWs {
  float* part;
  float* tpart;
  float* scale;
  float* shift;
  float* sum1;
  float* sum2;
  unsigned* counters;
};
BnWs bn_ws(void* ws, int C) {
  // counters first: their address must not depend on the call's C (the
  // workspace is shared by layers of different widths)
  BnWs w;
  w.counters = static_cast<unsigned*>(ws);
  w.part = reinterpret_cast<float*>(w.counters + kBnCounters);
  w.tpart = w.part + static_cast<size_t>(kBnMaxBlocks) * 2 * kBnGroup;
  w.scale = w.tpart + static_cast<size_t>(kBnMaxBlocks) * 2 * kBnGroup;
  w.shift = w.scale + C;
  w.sum1 = w.shift + C;
  w.sum2 = w.sum1 + C;
  return w;
}

struct BnArgs {
  const float* x;
  const float* dy;
  long long M;
  int C, lanes, Y, relu;
  const float* gamma;
  const float* beta;
  const float* mean;     // mode 1
  const float* invstd;   // mode 1
  float eps, momentum;
  float* save_mean;      // mode 0 outputs
  float* save_invstd;
  float* run_mean;
  float* run_var;
  float* dgamma;         // mode 1 outputs
  float* dbeta;
  BnWs w;
};

template <int MODE>
__global__ void __launch_bounds__(kThreads) bn_reduce_kernel(const BnArgs a) {
  __shared__ float red[2][kThreads][4];
  __shared__ int is_last;
  const int lanes = a.lanes;
  const int lane_c = threadIdx.x % lanes;
  const int lane_r = threadIdx.x / lanes;
  const int rows_per_pass = kThreads / lanes;
  const int c = (blockIdx.x * lanes + lane_c) * 4;
  const bool c_ok = c < a.C;
  const long long rows_per_block = (a.M + a.Y - 1) / a.Y;
  const long long r_begin = blockIdx.y * rows_per_block;
  const long long r_end = min(a.M, r_begin + rows_per_block);

  float a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
  float mu[4] = {0, 0, 0, 0}, is[4] = {0, 0, 0, 0}, ga[4] = {0, 0, 0, 0},
        be[4] = {0, 0, 0, 0};
  if (MODE == 1 && c_ok) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mu[j] = a.mean[c + j];
      is[j] = a.invstd[c + j];
      ga[j] = a.gamma[c + j];
      be[j] = a.beta[c + j];
    }
  }
  auto consume = [&](const float4 v, const float4 d) {
    const float xv[4] = {v.x, v.y, v.z, v.w};
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a0[j] += xv[j];
        a1[j] += xv[j] * xv[j];
      }
    } else {
      const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float xh = (xv[j] - mu[j]) * is[j];
        float g = dv[j];
        if (a.relu && (xh * ga[j] + be[j]) <= 0.f) g = 0.f;
        a0[j] += g;
        a1[j] += g * xh;
      }
    }
  };
  if (c_ok) {
    long long r = r_begin + lane_r;
    const long long step = rows_per_pass;
    for (; r + 3 * step < r_end; r += 4 * step) {  // 4 rows in flight
      float4 v[4], d[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = __ldg(reinterpret_cast<const float4*>(a.x + (r + u * step) * a.C + c));
        if (MODE == 1) d[u] = __ldg(reinterpret_cast<const float4*>(a.dy + (r + u * step) * a.C + c));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) consume(v[u], MODE == 1 ? d[u] : v[u]);
    }
    for (; r < r_end; r += step) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(a.x + r * a.C + c));
      const float4 d = MODE == 1 ? __ldg(reinterpret_cast<const float4*>(a.dy + r * a.C + c)) : v;
      consume(v, d);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    red[0][threadIdx.x][j] = a0[j];
    red[1][threadIdx.x][j] = a1[j];
  }
  __syncthreads();
  // block partial for this block's channels (row lanes summed in order)
  const size_t slot = static_cast<size_t>(blockIdx.y * gridDim.x + blockIdx.x) * 2 * kBnGroup;
  if (lane_r == 0) {
    float t0[4] = {0, 0, 0, 0}, t1[4] = {0, 0, 0, 0};
    for (int rr = 0; rr < rows_per_pass; ++rr) {
      const int src = rr * lanes + lane_c;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        t0[j] += red[0][src][j];
        t1[j] += red[1][src][j];
      }
    }
    *reinterpret_cast<float4*>(a.w.part + slot + lane_c * 4) = make_float4(t0[0], t0[1], t0[2], t0[3]);
    *reinterpret_cast<float4*>(a.w.part + slot + kBnGroup + lane_c * 4) =
        make_float4(t1[0], t1[1], t1[2], t1[3]);
  }
  const int ch_in_group = lanes * 4;
  const int gx = gridDim.x;
  // ---- level 1: the last block of this team sums the team's slots ----
  const int team = blockIdx.y / kBnTeam;
  const int team_lo = team * kBnTeam;
  const int team_n = min(kBnTeam, static_cast<int>(gridDim.y) - team_lo);
  unsigned* tcount = a.w.counters + kBnMaxGroups + blockIdx.x * kBnMaxTeams + team;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(tcount, 1u) == static_cast<unsigned>(team_n - 1));
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int v = threadIdx.x; v < 2 * kBnGroup; v += kThreads) {
    if ((v & (kBnGroup - 1)) >= ch_in_group) continue;
    float t = 0.f;
#pragma unroll 4
    for (int y = team_lo; y < team_lo + team_n; ++y)
      t += __ldcg(a.w.part + static_cast<size_t>(y * gx + blockIdx.x) * 2 * kBnGroup + v);
    a.w.tpart[static_cast<size_t>(team * gx + blockIdx.x) * 2 * kBnGroup + v] = t;
  }
  if (threadIdx.x == 0) *tcount = 0u;  // re-arm
  // ---- level 2: the last team of the channel group finalises ----
  const int nteams = (gridDim.y + kBnTeam - 1) / kBnTeam;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    is_last = (atomicAdd(&a.w.counters[blockIdx.x], 1u) == static_cast<unsigned>(nteams - 1));
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int t = threadIdx.x; t < ch_in_group; t += kThreads) {
    const int ch = blockIdx.x * ch_in_group + t;
    if (ch >= a.C) continue;
    double s1 = 0.0, s2 = 0.0;
#pragma unroll 4
    for (int tm = 0; tm < nteams; ++tm) {
      const float* p = a.w.tpart + static_cast<size_t>(tm * gx + blockIdx.x) * 2 * kBnGroup;
      s1 += static_cast<double>(__ldcg(p + t));
      s2 += static_cast<double>(__ldcg(p + kBnGroup + t));
    }
    if (MODE == 0) {
      const double mean = s1 / static_cast<double>(a.M);
      double var = s2 / static_cast<double>(a.M) - mean * mean;
      if (var < 0) var = 0;
      const float inv = static_cast<float>(1.0 / sqrt(var + static_cast<double>(a.eps)));
      const float sc = a.gamma[ch] * inv;
      a.w.scale[ch] = sc;
      a.w.shift[ch] = a.beta[ch] - static_cast<float>(mean) * sc;
      if (a.save_mean) a.save_mean[ch] = static_cast<float>(mean);
      if (a.save_invstd) a.save_invstd[ch] = inv;
      if (a.run_mean && a.run_var && a.M > 1) {
        const double unbiased = var * static_cast<double>(a.M) / static_cast<double>(a.M - 1);
        a.run_mean[ch] = (1.f - a.momentum) * a.run_mean[ch] + a.momentum * static_cast<float>(mean);
        a.run_var[ch] = (1.f - a.momentum) * a.run_var[ch] + a.momentum * static_cast<float>(unbiased);
      }
    } else {
      a.w.sum1[ch] = static_cast<float>(s1);
      a.w.sum2[ch] = static_cast<float>(s2);
      if (a.dbeta) a.dbeta[ch] = static_cast<float>(s1);
      if (a.dgamma) a.dgamma[ch] = static_cast<float>(s2);
    }
  }
  if (threadIdx.x == 0) a.w.counters[blockIdx.x] = 0u;  // re-arm for the next launch
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

// dx = gamma*invstd * (g - mean(g) - xhat * mean(g*xhat))
__global__ void __launch_bounds__(kThreads) bn_bwd_dx_kernel(
    const float* __restrict__ x, const float* __restrict__ dy, long long total4, int C4,
    long long M, const float* __restrict__ gamma, const float* __restrict__ beta,
    const float* __restrict__ mean, const float* __restrict__ invstd,
    const float* __restrict__ s1, const float* __restrict__ s2, int relu,
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
      const float mg = s1[c + j] * invM;
      const float mgx = s2[c + j] * invM;
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

// grid of the reduction: channel groups of lanes*4 <= 128 channels, Y row
// splits so that x*Y ~ 4 blocks per SM (<= kBnMaxBlocks), >= 32 rows each
void bn_reduce_launch_dims(long long M, int C, int* lanes, dim3* grid) {
  int l = C / 4;
  if (l > kBnGroup / 4) l = kBnGroup / 4;
  if (l < 1) l = 1;
  *lanes = l;
  const int cgroups = (C / 4 + l - 1) / l;
  long long y = (148LL * 4 + cgroups - 1) / cgroups;
  const long long max_y = (M + 31) / 32;
  if (y > max_y) y = max_y;
  if (y > kBnMaxBlocks / cgroups) y = kBnMaxBlocks / cgroups;
  if (y < 1) y = 1;
  *grid = dim3(cgroups, static_cast<unsigned>(y));
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
// recomputed from the input; one thread per 4 channels of an input pixel
// (float4 gathers over the <= ceil(k/stride)^2 windows covering it)
__global__ void maxpool_bwd_kernel(const float* __restrict__ x, const float* __restrict__ dy,
                                   int n, int h, int w, int c4, int kr, int ks, int stride,
                                   int pad, int p, int q, float* __restrict__ dx) {
  const long long total = static_cast<long long>(n) * h * w * c4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* dy4 = reinterpret_cast<const float4*>(dy);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cg = static_cast<int>(i % c4);
    long long t = i / c4;
    const int ww = static_cast<int>(t % w);
    t /= w;
    const int hh = static_cast<int>(t % h);
    const int nn = static_cast<int>(t / h);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int p_lo = max(0, (hh + pad - kr + stride) / stride);
    const int p_hi = min(p - 1, (hh + pad) / stride);
    const int q_lo = max(0, (ww + pad - ks + stride) / stride);
    const int q_hi = min(q - 1, (ww + pad) / stride);
    const long long img = static_cast<long long>(nn) * h;
    for (int pp = p_lo; pp <= p_hi; ++pp) {
      for (int qq = q_lo; qq <= q_hi; ++qq) {
        // window argmax per channel (first maximum in row-major order)
        float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        int bpos[4] = {-1, -1, -1, -1};
        for (int r = 0; r < kr; ++r) {
          const int ih = pp * stride - pad + r;
          if (ih < 0 || ih >= h) continue;
          for (int s = 0; s < ks; ++s) {
            const int iw = qq * stride - pad + s;
            if (iw < 0 || iw >= w) continue;
            const float4 v = __ldg(x4 + ((img + ih) * w + iw) * c4 + cg);
            const float vv[4] = {v.x, v.y, v.z, v.w};
            const int pos = ih * w + iw;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (vv[j] > best[j]) {
                best[j] = vv[j];
                bpos[j] = pos;
              }
          }
        }
        const int me = hh * w + ww;
        if (bpos[0] == me || bpos[1] == me || bpos[2] == me || bpos[3] == me) {
          const float4 g = __ldg(dy4 + ((static_cast<long long>(nn) * p + pp) * q + qq) * c4 + cg);
          const float gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (bpos[j] == me) acc[j] += gv[j];
        }
      }
    }
    reinterpret_cast<float4*>(dx)[i] = make_float4(acc[0], acc[1], acc[2], acc[3]);
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

// Softmax cross-entropy in one block (the batch is k* rows): one warp per
// row, then the mean loss and the bias gradient (column sums of dlogits)
// are summed in row order -- deterministic, no atomics.
constexpr int kXentThreads = 1024;
__global__ void __launch_bounds__(kXentThreads) xent_kernel(
    const float* __restrict__ logits, const int* __restrict__ labels, int rows, int classes,
    float* loss, float* dlogits, float* dbias) {
  __shared__ float row_loss[kXentThreads / 32];
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const int nw = kXentThreads / 32;
  float my_loss = 0.f;  // lane 0 of each warp: sum over its rows, in order
  for (int row = warp; row < rows; row += nw) {
    const float* z = logits + static_cast<long long>(row) * classes;
    float mx = -INFINITY;
    for (int j = lane; j < classes; j += 32) mx = fmaxf(mx, z[j]);
    mx = warp_max(mx);
    float se = 0.f;
    for (int j = lane; j < classes; j += 32) se += expf(z[j] - mx);
    se = warp_sum(se);
    const int y = labels[row];
    if (lane == 0) my_loss += mx + logf(se) - z[y];
    if (dlogits) {
      const float inv = 1.f / se;
      float* d = dlogits + static_cast<long long>(row) * classes;
      for (int j = lane; j < classes; j += 32)
        d[j] = (expf(z[j] - mx) * inv - (j == y ? 1.f : 0.f)) / static_cast<float>(rows);
    }
  }
  if (lane == 0) row_loss[warp] = my_loss;
  __syncthreads();
  if (loss && threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < nw; ++w) t += row_loss[w];
    *loss = t / static_cast<float>(rows);
  }
  if (dbias && dlogits) {
    for (int j = threadIdx.x; j < classes; j += kXentThreads) {
      float t = 0.f;
      for (int row = 0; row < rows; ++row) t += dlogits[static_cast<long long>(row) * classes + j];
      dbias[j] = t;
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
  return sizeof(float) * (2ull * kBnMaxBlocks * 2 * kBnGroup + 4ull * C) +
         sizeof(unsigned) * kBnCounters;
}

extern "C" int accudnn_bn_fwd(const float* x, long long M, int C, const float* gamma,
                              const float* beta, float eps, int relu, float* y,
                              float* save_mean, float* save_invstd, float* running_mean,
                              float* running_var, float momentum, void* ws, void* stream) {
  if ((C & 3) || M <= 0 || C > kBnGroup * kBnMaxGroups) return static_cast<int>(cudaErrorInvalidValue);
  const BnWs w = bn_ws(ws, C);
  cudaStream_t st = S(stream);
  BnArgs a{};
  a.x = x;
  a.M = M;
  a.C = C;
  a.gamma = gamma;
  a.beta = beta;
  a.eps = eps;
  a.momentum = momentum;
  a.save_mean = save_mean;
  a.save_invstd = save_invstd;
  a.run_mean = running_mean;
  a.run_var = running_var;
  a.w = w;
  dim3 grid;
  bn_reduce_launch_dims(M, C, &a.lanes, &grid);
  a.Y = static_cast<int>(grid.y);
  bn_reduce_kernel<0><<<grid, kThreads, 0, st>>>(a);
  const long long total4 = M * C / 4;
  bn_apply_kernel<<<grid_for(total4, kThreads), kThreads, 0, st>>>(x, total4, C / 4, w.scale,
                                                                   w.shift, relu, y);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_bn_bwd(const float* x, const float* dy, long long M, int C,
                              const float* gamma, const float* beta, const float* save_mean,
                              const float* save_invstd, int relu, float* dx, int dx_beta,
                              float* dgamma, float* dbeta, void* ws, void* stream) {
  if ((C & 3) || M <= 0 || C > kBnGroup * kBnMaxGroups) return static_cast<int>(cudaErrorInvalidValue);
  const BnWs w = bn_ws(ws, C);
  cudaStream_t st = S(stream);
  BnArgs a{};
  a.x = x;
  a.dy = dy;
  a.M = M;
  a.C = C;
  a.relu = relu;
  a.gamma = gamma;
  a.beta = beta;
  a.mean = save_mean;
  a.invstd = save_invstd;
  a.dgamma = dgamma;
  a.dbeta = dbeta;
  a.w = w;
  dim3 grid;
  bn_reduce_launch_dims(M, C, &a.lanes, &grid);
  a.Y = static_cast<int>(grid.y);
  bn_reduce_kernel<1><<<grid, kThreads, 0, st>>>(a);
  const long long total4 = M * C / 4;
  bn_bwd_dx_kernel<<<grid_for(total4, kThreads), kThreads, 0, st>>>(
      x, dy, total4, C / 4, M, gamma, beta, save_mean, save_invstd, w.sum1, w.sum2, relu, dx,
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
  if (c & 3) return static_cast<int>(cudaErrorInvalidValue);
  const long long total = static_cast<long long>(n) * h * w * (c / 4);
  maxpool_bwd_kernel<<<grid_for(total, kThreads), kThreads, 0, S(stream)>>>(
      x, dy, n, h, w, c / 4, kr, ks, stride, pad, p, q, dx);
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
  xent_kernel<<<1, kXentThreads, 0, S(stream)>>>(logits, labels, rows, classes, loss, nullptr,
                                                 nullptr);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_xent_bwd(const float* logits, const int* labels, int rows, int classes,
                                float* dlogits, float* dbias, void* stream) {
  xent_kernel<<<1, kXentThreads, 0, S(stream)>>>(logits, labels, rows, classes, nullptr,
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
