// HBM-bound layer kernels of the ResNet training step: batch norm (+ fused
// ReLU) forward/backward, ReLU, eltwise add, pooling, FC bias, softmax
// cross-entropy, SGD-momentum and the input layout conversion.
//
// All of them stream NHWC fp32 with 128-bit vector accesses; per-channel
// reductions use warp shuffles + shared memory inside a block and fp64
// atomics across blocks (the batch-norm sums run over up to k*112*112 rows,
// so the cross-block accumulation is kept in double to avoid cancellation
// in E[x^2] - E[x]^2).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <cstdint>

#include "accudnn_kernels.h"
#include "pdl.cuh"

namespace accudnn {
int g_pdl = 0;  // measured: PDL slowed the captured step (19.6 vs 18.9 ms), off by default
float* conv_splitk_workspace(size_t bytes);  // conv_sm100.cu
void conv_select_workspace(cudaStream_t st);
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
// One cooperative kernel per BN pass (forward: statistics + normalise;
// backward: (sum g, sum g*xhat) + data gradient), deterministic, no atomics
// on data:
//   phase 1  block (channel group bx, row split by) accumulates its rows into
//            a private slot part[by*gx+bx][2][128]
//   barrier  grid-wide (all blocks are co-resident: cooperative launch)
//   phase 2  every block sums the Y slots of its channel group in a fixed
//            order (chunked over threads, chunks combined in order, fp64) --
//            all blocks of a group compute bit-identical constants; block
//            by == 0 writes the per-channel outputs
//   phase 3  the block normalises / back-propagates the same rows it reduced
//            (mostly L1/L2 hits)
// Workspace: barrier words (uint) [kBnCounters] | part (float) [kBnMaxBlocks][2][128]
constexpr int kBnThreads = 512;
constexpr int kBnGroup = 128;        // channels per channel group
constexpr int kBnMaxBlocks = 1024;   // gx * Y
constexpr int kBnMaxGroups = 256;    // 32-channel groups: C <= 8192
constexpr int kBnCounters = 64;

struct BnWs {
  unsigned* counters;  // [0] arrivals, [1] generation
  float* part;
};
BnWs bn_ws(void* ws, int C) {
  BnWs w;
  w.counters = static_cast<unsigned*>(ws);
  w.part = reinterpret_cast<float*>(w.counters + kBnCounters);
  return w;
}

struct BnArgs {
  const float* x;
  const float* dy;
  long long M;
  int C, lanes, Y, relu;
  long long rpb;  // rows per block (0: ceil(M / Y))
  const float* gamma;
  const float* beta;
  const float* mean;     // mode 1
  const float* invstd;   // mode 1
  float eps, momentum;
  float* save_mean;      // mode 0 outputs
  float* save_invstd;
  float* run_mean;
  float* run_var;
  float* y;              // mode 0: normalised output
  float* dgamma;         // mode 1 outputs
  float* dbeta;
  float* dx;             // mode 1: data gradient (+= when dx_beta)
  int dx_beta;
  const float* skip;     // SKIP: y = relu(bn(x) + skip); backward mask uses it too
  float* dskip;          // SKIP, mode 1: gradient of the shortcut (+= when dskip_beta)
  int dskip_beta;
  int mask_smem;         // SKIP backward launched with the mask buffer (dynamic smem)
  int row_cache;         // non-SKIP backward: phase 1 keeps its x / dy rows in dynamic
                         // smem for phase 3 (short layers, <= kRowCache rows per thread)
  const float* stats_in; // mode 0: the producing conv's column sums [2][P][C] (P = ceil(M/32)):
                         // phase 1 sums these instead of reading x
  BnWs w;
  long long* trace;      // debug: globaltimer stamps per block (accudnn_bn_trace)
  int l2_keep;           // phase-1 reads of the tensors phase 3 re-reads: L2 evict_last
  int l2_last;           // phase-3 (last) reads: L2 evict_first
};
long long* g_bn_trace = nullptr;
__device__ __forceinline__ long long bn_gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BN_STAMP(i)                                                                     \
  do {                                                                                  \
    if (a.trace && threadIdx.x == 0)                                                    \
      a.trace[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + (i)] = bn_gtimer();           \
  } while (0)

// 16-byte read-only loads with an L2 eviction-priority policy
__device__ __forceinline__ uint64_t l2_policy(int prio) {  // 0 normal, 1 last, 2 first
  uint64_t p;
  if (prio == 1)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (prio == 2)
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_pol(const float* ptr, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(ptr), "l"(pol));
  return v;
}

// grid-wide barrier (all blocks co-resident: cooperative launch):
// counters[0] arrivals, counters[1] generation.  (Measured: one barrier over
// the grid is faster than per-channel-group barriers here.)
__device__ __forceinline__ void grid_barrier(unsigned* counters, unsigned nblocks) {
  // bar.sync orders the block's partial writes before thread 0's fence, and
  // the fence is cumulative: one release fence per block, not per thread
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    volatile unsigned* gen = counters + 1;
    const unsigned g = *gen;
    if (atomicAdd(counters, 1u) == nblocks - 1) {
      // release first; the arrival count is reset behind it (one barrier per
      // launch, so the next arrivals are in the next kernel, after this
      // store is visible)
      atomicAdd(counters + 1, 1u);
      counters[0] = 0u;
    } else {
      // poll without sleeping first: the release usually follows within a
      // few hundred ns, and a sleep's wake-up granularity adds to every
      // barrier on the critical path
      int polls = 0;
      while (*gen == g)
        if (++polls > 64) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr int kBnPilotRows = 4;
constexpr int kRowCache = 8;  // rows per thread the backward row cache holds (2 x 64 KB)
__device__ __forceinline__ long long bn_pilot_row(long long M, int i) {
  return M * i / kBnPilotRows;
}

template <int MODE, bool SKIP>
__device__ __forceinline__ void bn_phase3(const BnArgs& a, bool c_ok, int lane_c, int lane_r,
                                          long long r_begin, long long r_end, long long step,
                                          long long first_row, bool use_mask,
                                          const float (&coef)[6][kBnGroup], const float (&mu)[4],
                                          const float (&is)[4], const float (&ga)[4],
                                          const float (&fsc)[4], const float (&fsh)[4],
                                          const uint32_t* mask_smem);

template <int MODE, bool CLUSTER, bool SKIP>
__global__ void __launch_bounds__(kBnThreads, (MODE == 0 || (CLUSTER && !SKIP)) ? 2 : 1) bn_fused_kernel(const BnArgs a) {
  pdl_wait();
  BN_STAMP(0);
  __shared__ float red[2][kBnThreads][4];
  __shared__ __align__(16) float cpart[2][kBnGroup];  // CLUSTER: this block's partial
  __shared__ double dsum[kBnThreads];
  __shared__ float coef[6][kBnGroup];
  __shared__ float pil_s[kBnGroup];  // MODE 0: the phase-1 pilot per channel of the group
  const int lanes = a.lanes;
  const int lane_c = threadIdx.x % lanes;
  const int lane_r = threadIdx.x / lanes;
  const int rows_per_pass = kBnThreads / lanes;
  const bool lane_ok = lane_r < rows_per_pass;
  const int c = (blockIdx.x * lanes + lane_c) * 4;
  const bool c_ok = lane_ok && c < a.C;
  const long long rows_per_block = a.rpb > 0 ? a.rpb : (a.M + a.Y - 1) / a.Y;
  const long long r_begin = blockIdx.y * rows_per_block;
  const long long r_end = min(a.M, r_begin + rows_per_block);
  const long long C = a.C;
  // SKIP backward: the ReLU mask of each (row, 4 channels) computed in phase 1
  // is kept as 4 bits in shared memory (kMaskWords words per thread,
  // thread-interleaved), so phase 3 need not re-read the shortcut tensor
  extern __shared__ uint32_t mask_smem[];
  float4* rcache = reinterpret_cast<float4*>(mask_smem);  // [row][x, dy][thread]
  constexpr int kMaskWords = 16;  // 128 rows per thread
  const long long first_row = r_begin + lane_r;
  const bool use_mask = MODE == 1 && SKIP && a.mask_smem &&
                        (rows_per_block + rows_per_pass - 1) / rows_per_pass <= 8 * kMaskWords;
  if (use_mask)
    for (int w = 0; w < kMaskWords; ++w) mask_smem[w * kBnThreads + threadIdx.x] = 0u;

  // per-channel parameters phase 2 needs, loaded now so their latency
  // overlaps phase 1 instead of following the statistics exchange
  float pre_g = 0.f, pre_b = 0.f, pre_rm = 0.f, pre_rv = 0.f;
  if (MODE == 0 && static_cast<int>(threadIdx.x) < lanes * 4) {
    const int chn = blockIdx.x * lanes * 4 + threadIdx.x;
    if (chn < a.C) {
      pre_g = a.gamma[chn];
      pre_b = a.beta[chn];
      if (blockIdx.y == 0 && a.run_mean && a.run_var) {
        pre_rm = a.run_mean[chn];
        pre_rv = a.run_var[chn];
      }
    }
  }

  // ---- phase 1: per-block partial sums ----
  float a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
  float mu[4] = {0, 0, 0, 0}, is[4] = {0, 0, 0, 0}, ga[4] = {0, 0, 0, 0};
  float fsc[4] = {0, 0, 0, 0}, fsh[4] = {0, 0, 0, 0};  // forward scale / shift
  // forward statistics are accumulated around a per-channel pilot (the mean
  // of 4 rows spread over the batch, the same for every block): sums of
  // (x - pilot) and (x - pilot)^2 keep E[x^2] - E[x]^2 free of cancellation
  // when |mean| >> std (shifted-data variance).  A single row is not enough:
  // row 0 is the corner pixel of image 0, which zero padding makes an
  // outlier of a convolution's output.
  // (its 8 loads are issued together with the first rows of phase 1, below)
  float pil[4] = {0, 0, 0, 0};
  auto load_pilot = [&](float4 (&pv)[kBnPilotRows]) {
#pragma unroll
    for (int i = 0; i < kBnPilotRows; ++i)
      pv[i] = __ldg(reinterpret_cast<const float4*>(a.x + bn_pilot_row(a.M, i) * C + c));
  };
  auto sum_pilot = [&](const float4 (&pv)[kBnPilotRows]) {
#pragma unroll
    for (int i = 0; i < kBnPilotRows; ++i) {
      pil[0] += pv[i].x;
      pil[1] += pv[i].y;
      pil[2] += pv[i].z;
      pil[3] += pv[i].w;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) pil[j] *= 1.f / kBnPilotRows;
  };
  if (MODE == 1 && c_ok) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mu[j] = a.mean[c + j];
      is[j] = a.invstd[c + j];
      ga[j] = a.gamma[c + j];
      fsc[j] = ga[j] * is[j];
      fsh[j] = a.beta[c + j] - mu[j] * fsc[j];
    }
  }
  auto consume = [&](const float4 v, const float4 d, const float4 sk4) -> uint32_t {
    const float xv[4] = {v.x, v.y, v.z, v.w};
    const float sk[4] = {sk4.x, sk4.y, sk4.z, sk4.w};
    uint32_t bits = 0;
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float dx = xv[j] - pil[j];
        a0[j] += dx;
        a1[j] += dx * dx;
      }
    } else {
      const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float xh = (xv[j] - mu[j]) * is[j];
        float g = dv[j];
        // the forward's pre-activation, bit for bit (scale/shift as in phase 2 of mode 0)
        if (a.relu && (xv[j] * fsc[j] + fsh[j] + (SKIP ? sk[j] : 0.f)) <= 0.f)
          g = 0.f;
        else
          bits |= 1u << j;
        a0[j] += g;
        a1[j] += g * xh;
      }
    }
    return bits;
  };
  auto keep_mask = [&](int kk, uint32_t bits) {  // kk: row index in this thread's sequence
    if (!use_mask) return;
    mask_smem[(kk >> 3) * kBnThreads + threadIdx.x] |= bits << ((kk & 7) * 4);
  };
  const long long step = rows_per_pass;
  if (MODE == 0 && a.stats_in) {
    // statistics precomputed by the conv epilogue: sum this block's share
    // of the 32-row partial slots (same fixed order as every other block)
    const long long P = (a.M + 31) / 32;
    const long long sp = (P + a.Y - 1) / a.Y;
    const long long s0 = blockIdx.y * sp, s1 = min(P, s0 + sp);
    if (c_ok)
      for (long long r = s0 + lane_r; r < s1; r += step) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(a.stats_in + r * C + c));
        const float4 q = __ldcg(reinterpret_cast<const float4*>(a.stats_in + (P + r) * C + c));
        a0[0] += v.x;
        a0[1] += v.y;
        a0[2] += v.z;
        a0[3] += v.w;
        a1[0] += q.x;
        a1[1] += q.y;
        a1[2] += q.z;
        a1[3] += q.w;
      }
  } else if (c_ok) {
    // x (and dy) are read again in phase 3: keep them in L2 ahead of the
    // shortcut, which phase 3 does not re-read when the mask is in smem
    const uint64_t p_keep = l2_policy(a.l2_keep ? 1 : 0);
    const uint64_t p_skip = l2_policy(a.l2_keep ? (use_mask ? 2 : 1) : 0);
    long long r = r_begin + lane_r;
    int kk = 0;
    if (MODE == 0) {
      // pilot: its loads and the first group's loads in flight together
      float4 pv[kBnPilotRows], v[4];
      load_pilot(pv);
      const bool group = r + 3 * step < r_end;
      if (group)
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ld_pol(a.x + (r + u * step) * C + c, p_keep);
      sum_pilot(pv);
      if (group) {
#pragma unroll
        for (int u = 0; u < 4; ++u) consume(v[u], v[u], v[u]);
        r += 4 * step;
        kk += 4;
      }
    }
    for (; r + 3 * step < r_end; r += 4 * step, kk += 4) {  // 4 rows in flight
      float4 v[4], d[4], sk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = ld_pol(a.x + (r + u * step) * C + c, p_keep);
        if (MODE == 1) d[u] = ld_pol(a.dy + (r + u * step) * C + c, p_keep);
        if (MODE == 1 && SKIP) sk[u] = ld_pol(a.skip + (r + u * step) * C + c, p_skip);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        keep_mask(kk + u,
                  consume(v[u], MODE == 1 ? d[u] : v[u], (MODE == 1 && SKIP) ? sk[u] : v[u]));
      if (MODE == 1 && !SKIP && a.row_cache)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          rcache[(2 * (kk + u)) * kBnThreads + threadIdx.x] = v[u];
          rcache[(2 * (kk + u) + 1) * kBnThreads + threadIdx.x] = d[u];
        }
    }
    for (; r < r_end; r += step, ++kk) {
      const float4 v = ld_pol(a.x + r * C + c, p_keep);
      const float4 d = MODE == 1 ? ld_pol(a.dy + r * C + c, p_keep) : v;
      const float4 sk = (MODE == 1 && SKIP) ? ld_pol(a.skip + r * C + c, p_skip) : v;
      keep_mask(kk, consume(v, d, sk));
      if (MODE == 1 && !SKIP && a.row_cache) {
        rcache[(2 * kk) * kBnThreads + threadIdx.x] = v;
        rcache[(2 * kk + 1) * kBnThreads + threadIdx.x] = d;
      }
    }
  }
  if (MODE == 0 && c_ok && !a.stats_in && lane_r == 0)
#pragma unroll
    for (int j = 0; j < 4; ++j) pil_s[lane_c * 4 + j] = pil[j];
  BN_STAMP(1);
  const int gx = gridDim.x;
  float* slot = CLUSTER ? &cpart[0][0]
                        : a.w.part + static_cast<size_t>(blockIdx.y * gx + blockIdx.x) * 2 * kBnGroup;
  if (32 % lanes == 0) {
    // row lanes of a warp: fixed xor-shuffle tree, then the 16 warp partials
    // summed in warp order by `lanes` threads (one barrier)
    for (int off = lanes; off < 32; off <<= 1) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a0[j] += __shfl_xor_sync(0xffffffffu, a0[j], off);
        a1[j] += __shfl_xor_sync(0xffffffffu, a1[j], off);
      }
    }
    const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (ln < lanes) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        red[0][wid * lanes + ln][j] = a0[j];
        red[1][wid * lanes + ln][j] = a1[j];
      }
    }
    __syncthreads();
    if (threadIdx.x < lanes) {
      float t0[4] = {0, 0, 0, 0}, t1[4] = {0, 0, 0, 0};
      for (int w = 0; w < kBnThreads / 32; ++w)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          t0[j] += red[0][w * lanes + threadIdx.x][j];
          t1[j] += red[1][w * lanes + threadIdx.x][j];
        }
      *reinterpret_cast<float4*>(slot + threadIdx.x * 4) = make_float4(t0[0], t0[1], t0[2], t0[3]);
      *reinterpret_cast<float4*>(slot + kBnGroup + threadIdx.x * 4) =
          make_float4(t1[0], t1[1], t1[2], t1[3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      red[0][threadIdx.x][j] = a0[j];
      red[1][threadIdx.x][j] = a1[j];
    }
    __syncthreads();
    // fixed-shape tree over the row lanes
    for (int n = rows_per_pass; n > 1;) {
      const int half = (n + 1) / 2;
      if (lane_r < n - half) {
        const int src = (lane_r + half) * lanes + lane_c;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          red[0][threadIdx.x][j] += red[0][src][j];
          red[1][threadIdx.x][j] += red[1][src][j];
        }
      }
      n = half;
      __syncthreads();
    }
    if (lane_r == 0) {
      *reinterpret_cast<float4*>(slot + lane_c * 4) =
          make_float4(red[0][lane_c][0], red[0][lane_c][1], red[0][lane_c][2], red[0][lane_c][3]);
      *reinterpret_cast<float4*>(slot + kBnGroup + lane_c * 4) =
          make_float4(red[1][lane_c][0], red[1][lane_c][1], red[1][lane_c][2], red[1][lane_c][3]);
    }
  }

  BN_STAMP(2);
  const int ch = lanes * 4;  // channels of this group
  const int V = 2 * ch;      // values: sum1 of ch channels, then sum2
  int T = 1;
  if constexpr (CLUSTER) {
    // ---- cluster of the group's Y row splits: partials through DSMEM ----
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    if (threadIdx.x < V) {
      const int v = threadIdx.x;
      const int off = v < ch ? v : kBnGroup + (v - ch);
      // all (<= 16) remote reads in flight at once (~200 cycles each), then
      // summed in rank order
      const unsigned nb = cluster.num_blocks();
      float pv[16];
#pragma unroll
      for (unsigned r = 0; r < 16; ++r)
        pv[r] = r < nb ? cluster.map_shared_rank(&cpart[0][0], r)[off] : 0.f;
      double t = 0.0;
#pragma unroll
      for (unsigned r = 0; r < 16; ++r)
        if (r < nb) t += static_cast<double>(pv[r]);
      dsum[v] = t;
    }
    // peers' partials must be read before any block exits: arrive now, wait
    // at the end of phase 3 (the barrier overlaps the normalisation pass)
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  } else {
    grid_barrier(a.w.counters, gridDim.x * gridDim.y);
    BN_STAMP(5);
    // ---- phase 2: the group's Y slots, chunked over threads, fixed order ----
    T = kBnThreads / V;
    const int v = threadIdx.x % V;
    const int chunk = threadIdx.x / V;
    double t = 0.0;
    if (chunk < T) {
      const int y0 = chunk * a.Y / T, y1 = (chunk + 1) * a.Y / T;  // <= 16 slots (bn_launch)
      const int off = v < ch ? v : kBnGroup + (v - ch);
      float pv[16];
#pragma unroll
      for (int k = 0; k < 16; ++k)
        pv[k] = (y0 + k < y1)
                    ? __ldcg(a.w.part + static_cast<size_t>((y0 + k) * gx + blockIdx.x) * 2 * kBnGroup + off)
                    : 0.f;
#pragma unroll
      for (int k = 0; k < 16; ++k) t += static_cast<double>(pv[k]);
    }
    dsum[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x < ch) {
    const int t = threadIdx.x;
    double s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < T; ++k) {
      s1 += dsum[k * V + t];
      s2 += dsum[k * V + ch + t];
    }
    const int chn = blockIdx.x * ch + t;
    if (chn < a.C) {
      if (MODE == 0) {
        const float pf = a.stats_in ? 0.f : pil_s[t];  // the pilot of phase 1
        const double pilot = static_cast<double>(pf);
        const double dm = s1 / static_cast<double>(a.M);
        const double mean = pilot + dm;
        double var = s2 / static_cast<double>(a.M) - dm * dm;
        if (var < 0) var = 0;
        const float inv = static_cast<float>(1.0 / sqrt(var + static_cast<double>(a.eps)));
        const float sc = pre_g * inv;
        coef[0][t] = sc;
        coef[1][t] = pre_b - static_cast<float>(mean) * sc;
        if (blockIdx.y == 0) {
          if (a.save_mean) a.save_mean[chn] = static_cast<float>(mean);
          if (a.save_invstd) a.save_invstd[chn] = inv;
          if (a.run_mean && a.run_var && a.M > 1) {
            const double unbiased = var * static_cast<double>(a.M) / static_cast<double>(a.M - 1);
            a.run_mean[chn] = (1.f - a.momentum) * pre_rm + a.momentum * static_cast<float>(mean);
            a.run_var[chn] = (1.f - a.momentum) * pre_rv + a.momentum * static_cast<float>(unbiased);
          }
        }
      } else {
        const float invM = 1.f / static_cast<float>(a.M);
        coef[0][t] = static_cast<float>(s1) * invM;  // mean(g)
        coef[1][t] = static_cast<float>(s2) * invM;  // mean(g * xhat)
        if (blockIdx.y == 0) {
          if (a.dbeta) a.dbeta[chn] = static_cast<float>(s1);
          if (a.dgamma) a.dgamma[chn] = static_cast<float>(s2);
        }
      }
    }
  }
  __syncthreads();

  BN_STAMP(3);
  pdl_trigger();  // (PDL) the successor may be scheduled during the last pass
  bn_phase3<MODE, SKIP>(a, c_ok, lane_c, lane_r, r_begin, r_end, step, first_row, use_mask, coef,
                        mu, is, ga, fsc, fsh, mask_smem);
  if constexpr (CLUSTER) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---- phase 3 of bn_fused_kernel: the block's rows again (normalise / dx) ----
template <int MODE, bool SKIP>
__device__ __forceinline__ void bn_phase3(const BnArgs& a, bool c_ok, int lane_c, int lane_r,
                                          long long r_begin, long long r_end, long long step,
                                          long long first_row, bool use_mask,
                                          const float (&coef)[6][kBnGroup], const float (&mu)[4],
                                          const float (&is)[4], const float (&ga)[4],
                                          const float (&fsc)[4], const float (&fsh)[4],
                                          const uint32_t* mask_smem) {
  const long long C = a.C;
  const int c = (blockIdx.x * a.lanes + lane_c) * 4;
  if (!c_ok) return;
  const int cl = lane_c * 4;
  // last row of this thread's phase-1 sequence r_begin + lane_r + k*step
  const long long first = r_begin + lane_r;
  if (first >= r_end) return;
  const long long r_hi = first + ((r_end - 1 - first) / step) * step;
  if (MODE == 0) {
    const float sc[4] = {coef[0][cl], coef[0][cl + 1], coef[0][cl + 2], coef[0][cl + 3]};
    const float sh[4] = {coef[1][cl], coef[1][cl + 1], coef[1][cl + 2], coef[1][cl + 3]};
    auto f = [&](float4 v, const float4 k4) {
      v.x = v.x * sc[0] + sh[0];
      v.y = v.y * sc[1] + sh[1];
      v.z = v.z * sc[2] + sh[2];
      v.w = v.w * sc[3] + sh[3];
      if (SKIP) {
        v.x += k4.x;
        v.y += k4.y;
        v.z += k4.z;
        v.w += k4.w;
      }
      if (a.relu) {
        v.x = fmaxf(v.x, 0.f);
        v.y = fmaxf(v.y, 0.f);
        v.z = fmaxf(v.z, 0.f);
        v.w = fmaxf(v.w, 0.f);
      }
      return v;
    };
    // rows in reverse: the lines read last in phase 1 are the likeliest L2 hits;
    // last reads of this step are evict_first
    const uint64_t p_last = l2_policy(a.l2_last ? 2 : 0);
    long long r = r_hi;
    for (; r - 3 * step >= r_begin; r -= 4 * step) {
      float4 v[4], kv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = ld_pol(a.x + (r - u * step) * C + c, p_last);
        kv[u] = SKIP ? ld_pol(a.skip + (r - u * step) * C + c, p_last) : v[u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        *reinterpret_cast<float4*>(a.y + (r - u * step) * C + c) = f(v[u], kv[u]);
    }
    for (; r >= r_begin; r -= step) {
      const float4 v = ld_pol(a.x + r * C + c, p_last);
      *reinterpret_cast<float4*>(a.y + r * C + c) = f(v, SKIP ? ld_pol(a.skip + r * C + c, p_last) : v);
    }
    BN_STAMP(4);
  } else {
    float mg[4], mgx[4], k0[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mg[j] = coef[0][cl + j];
      mgx[j] = coef[1][cl + j];
      k0[j] = ga[j] * is[j];
    }
    auto f = [&](const float4 xv4, const float4 dv4, const float4 k4, long long r, int kk) {
      const float xv[4] = {xv4.x, xv4.y, xv4.z, xv4.w};
      const float dv[4] = {dv4.x, dv4.y, dv4.z, dv4.w};
      const float sk[4] = {k4.x, k4.y, k4.z, k4.w};
      uint32_t mbits = 0;
      if (use_mask) mbits = mask_smem[(kk >> 3) * kBnThreads + threadIdx.x] >> ((kk & 7) * 4);
      float o[4], gg[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float xh = (xv[j] - mu[j]) * is[j];
        float g = dv[j];
        if (use_mask) {
          if (!(mbits >> j & 1u)) g = 0.f;
        } else if (a.relu && (xv[j] * fsc[j] + fsh[j] + (SKIP ? sk[j] : 0.f)) <= 0.f) {
          g = 0.f;
        }
        gg[j] = g;
        o[j] = k0[j] * (g - mg[j] - xh * mgx[j]);
      }
      auto put = [&](float* base, const float* val, int beta) {
        float4 out = make_float4(val[0], val[1], val[2], val[3]);
        float4* d = reinterpret_cast<float4*>(base + r * C + c);
        if (beta) {
          const float4 old = *d;
          out.x += old.x;
          out.y += old.y;
          out.z += old.z;
          out.w += old.w;
        }
        *d = out;
      };
      put(a.dx, o, a.dx_beta);
      if (SKIP) put(a.dskip, gg, a.dskip_beta);  // d(shortcut) = masked dy
    };
    const uint64_t p_last = l2_policy(a.l2_last ? 2 : 0);
    long long r = r_hi;  // reverse order, as above
    int kk = static_cast<int>((r_hi - first_row) / step);
    if (!SKIP && a.row_cache) {  // the rows phase 1 kept in shared memory
      const float4* rcache = reinterpret_cast<const float4*>(mask_smem);
      for (; r >= r_begin; r -= step, --kk) {
        const float4 xv = rcache[(2 * kk) * kBnThreads + threadIdx.x];
        f(xv, rcache[(2 * kk + 1) * kBnThreads + threadIdx.x], xv, r, kk);
      }
    }
    for (; r - 3 * step >= r_begin; r -= 4 * step, kk -= 4) {
      float4 xv[4], dv[4], kv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xv[u] = ld_pol(a.x + (r - u * step) * C + c, p_last);
        dv[u] = ld_pol(a.dy + (r - u * step) * C + c, p_last);
        kv[u] = (SKIP && !use_mask) ? ld_pol(a.skip + (r - u * step) * C + c, p_last) : xv[u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) f(xv[u], dv[u], kv[u], r - u * step, kk - u);
    }
    for (; r >= r_begin; r -= step, --kk) {
      const float4 xv = ld_pol(a.x + r * C + c, p_last);
      f(xv, ld_pol(a.dy + r * C + c, p_last),
        (SKIP && !use_mask) ? ld_pol(a.skip + r * C + c, p_last) : xv, r, kk);
    }
    BN_STAMP(4);
  }
}

// Launch shapes (32-channel groups, gx = C/32, 512 threads):
//  * cluster: the Y <= 16 row splits of a group form one thread-block
//    cluster and exchange partials through distributed shared memory -- no
//    global synchronisation; used for narrow layers with few rows;
//  * cooperative: Y row splits over the whole grid (all CTAs co-resident,
//    2 per SM), partials in the workspace, one grid barrier; for the large
//    early-stage layers that need every SM streaming.
// ACCUDNN_BN_ROWCACHE=0: the backward re-reads its rows from L2 in phase 3
inline bool row_cache_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("ACCUDNN_BN_ROWCACHE");
    v = e ? std::atoi(e) : 1;
  }
  return v != 0;
}

// ACCUDNN_BN_RPB=0: plain ceil(M / Y) row splits (A/B switch)
inline bool rpb_rounding() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("ACCUDNN_BN_RPB");
    v = e ? std::atoi(e) : 1;
  }
  return v != 0;
}

template <int MODE, bool SKIP>
int bn_launch(BnArgs a, cudaStream_t st) {
  // L2 eviction priorities (ACCUDNN_BN_L2HINTS: 0 off, 1 auto, 3 always,
  // 4 auto without phase-3 hints on large layers).  Measured per shape
  // (tools/bn_bench.py): evict_last on the re-read tensors pays while they
  // fit in about half the L2 and costs 3-5% above that
  static int hints = -1;
  if (hints < 0) {
    const char* e = std::getenv("ACCUDNN_BN_L2HINTS");
    hints = e ? std::atoi(e) : 1;
  }
  static double keep_mb[2] = {-1.0, -1.0};  // ACCUDNN_BN_KEEP_MB_FWD / _BWD overrides
  if (keep_mb[MODE] < 0) {
    const char* e = std::getenv(MODE == 1 ? "ACCUDNN_BN_KEEP_MB_BWD" : "ACCUDNN_BN_KEEP_MB_FWD");
    keep_mb[MODE] = e ? std::atof(e) : (MODE == 1 ? 72.0 : 48.0);
  }
  const double reread = 4.0 * static_cast<double>(a.M) * a.C * (MODE == 1 ? 2 : 1);
  const bool fits = reread <= keep_mb[MODE] * (1 << 20);
  a.l2_keep = hints == 3 || ((hints == 1 || hints == 4) && fits);
  a.l2_last = hints == 3 || hints == 1 || (hints == 4 && fits);
  static int occ = 0;
  if (!occ) {
    if (MODE == 1 && SKIP)
      cudaFuncSetAttribute(bn_fused_kernel<MODE, false, SKIP>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bn_fused_kernel<MODE, false, SKIP>,
                                                  kBnThreads, (MODE == 1 && SKIP) ? 32768 : 0);
    if (occ < 1) occ = 1;
    cudaFuncSetAttribute(bn_fused_kernel<MODE, true, SKIP>,
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int l = a.C / 4;
  if (l > 8) l = 8;
  if (l < 1) l = 1;
  a.lanes = l;
  const int gx = (a.C / 4 + l - 1) / l;
  cudaLaunchAttribute attr[2];
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kBnThreads);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (MODE == 1 && SKIP) {  // 32 KB of ReLU-mask bits (see bn_fused_kernel)
    static bool mask_attr = false;
    if (!mask_attr) {
      cudaFuncSetAttribute(bn_fused_kernel<MODE, false, SKIP>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
      cudaFuncSetAttribute(bn_fused_kernel<MODE, true, SKIP>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
      mask_attr = true;
    }
    cfg.dynamicSmemBytes = 32768;
    a.mask_smem = 1;
  }
  // measured (tools/bn_bench.py, k* = 27 shapes): clusters win for narrow
  // layers with few rows, the cooperative grid for wide or tall ones
  const long long max_blocks = std::min<long long>(static_cast<long long>(occ) * sms, kBnMaxBlocks);
  static int force = -2;  // ACCUDNN_BN_CLUSTER: 1 always, 0 never, unset: measured rule
  if (force == -2) {
    const char* e = std::getenv("ACCUDNN_BN_CLUSTER");
    force = e ? std::atoi(e) : -1;
  }
  // measured per mode (tools/bn_bench.py, k* = 42 shapes, forced both ways):
  // the forward wins with clusters on narrow short layers (14x14x256:
  // 10.4 vs 11.2 us) and tiny ones; the backward only on tiny ones -- its
  // cluster variant runs one CTA per SM with spills (14x14x256: 15.6 vs 11.1 us,
  // residual tail 22.9 vs 14.2 us)
  bool cluster = a.M < 1024 || gx > max_blocks ||
                 (MODE == 0 && a.C <= 256 && a.M <= 16LL * 2048);
  if (force == 1) cluster = true;
  if (force == 0 && gx <= max_blocks) cluster = false;
  if (cluster) {
    long long y = std::max<long long>(1, (2LL * sms + gx - 1) / gx);
    y = std::min<long long>(y, (a.M + 31) / 32);
    y = std::min<long long>(y, 16);
    if (y < 1) y = 1;
    a.Y = static_cast<int>(y);
    cfg.gridDim = dim3(gx, a.Y);
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = a.Y;
    attr[0].val.clusterDim.z = 1;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, bn_fused_kernel<MODE, true, SKIP>, a));
  }
  const int T = kBnThreads / (2 * 4 * l);
  long long y = (max_blocks + gx - 1) / gx;
  y = std::min<long long>(y, (a.M + 15) / 16);
  y = std::min<long long>(y, 16LL * T);
  y = std::min<long long>(y, max_blocks / gx);
  if (y < 1) y = 1;
  // rows per block a multiple of 4 x the rows one pass of the block covers:
  // every thread then streams whole batches of 4 rows (a ragged remainder is
  // one dependent round trip per row -- 3 of them on a 14x14 layer)
  // Taken when it saves at least two dependent round trips per thread (a
  // layer whose threads own 3-4 rows: 3 -> 1), not when it only trades one
  // for fewer CTAs streaming a large layer (measured per shape, bn_bench)
  {
    const long long rpp = kBnThreads / l;
    const long long unit = 4 * rpp;
    auto rounds = [&](long long rpb) {  // worst thread: batches of 4 + single rows
      long long worst = 0;
      for (long long rpt : {rpb / rpp, (rpb + rpp - 1) / rpp})
        worst = std::max(worst, rpt / 4 + rpt % 4);
      return worst;
    };
    const long long rpb0 = (a.M + y - 1) / y;
    const long long rpb = (rpb0 + unit - 1) / unit * unit;
    const long long y2 = (a.M + rpb - 1) / rpb;
    if (rpb_rounding() && y2 >= 1 && y2 <= y && rounds(rpb0) - rounds(rpb) >= 2) {
      y = y2;
      a.rpb = rpb;
    }
  }
  a.Y = static_cast<int>(y);
  // short backward layers: phase 1 keeps its rows in shared memory for phase 3
  // (one CTA per SM in this mode, so 128 KB of dynamic smem is free)
  if (MODE == 1 && !SKIP && row_cache_on()) {
    const long long rpp = kBnThreads / l;
    const long long rpb = a.rpb > 0 ? a.rpb : (a.M + y - 1) / y;
    if ((rpb + rpp - 1) / rpp <= kRowCache) {
      static bool attr_set = false;
      if (!attr_set) {
        cudaFuncSetAttribute(bn_fused_kernel<MODE, false, SKIP>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(float4) * 2 * kRowCache * kBnThreads));
        attr_set = true;
      }
      a.row_cache = 1;
      cfg.dynamicSmemBytes = sizeof(float4) * 2 * kRowCache * kBnThreads;
    }
  }
  cfg.gridDim = dim3(gx, a.Y);
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  return static_cast<int>(cudaLaunchKernelEx(&cfg, bn_fused_kernel<MODE, false, SKIP>, a));
}

// ---------------------------------------------------------------------------
// elementwise
// ---------------------------------------------------------------------------
__global__ void relu_fwd_kernel(const float4* __restrict__ x, float4* __restrict__ y,
                                long long n4) {
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 u = a[i], v = b[i];
    y[i] = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
  }
}

__global__ void copy_kernel(const float4* __restrict__ s, float4* __restrict__ d, long long n4,
                            int beta) {
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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

// two-pass max-pool backward: (1) the argmax tap (row-major first maximum)
// of every output window and channel as one byte; (2) every input element
// gathers dy over the <= ceil(k/stride)^2 windows covering it whose argmax
// is this element, in window order (deterministic).
// K, ST, PD > 0: compile-time window (the ResNet stem's 3x3 / 2 / 1: the
// window loops unroll and every load of a thread is in flight at once);
// 0: runtime values
template <int K, int ST, int PD>
__global__ void maxpool_argmax_kernel(const float* __restrict__ x, int n, int h, int w, int c4,
                                      int kr_, int ks_, int stride_, int pad_, int p, int q,
                                      uint8_t* __restrict__ arg, int total) {
  pdl_wait();
  pdl_trigger();
  const int kr = K ? K : kr_, ks = K ? K : ks_, stride = ST ? ST : stride_, pad = K ? PD : pad_;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // (pixel, channel float4)
  if (idx >= total) return;
  const int cg = idx % c4;
  const int pix = idx / c4;  // (n, pp, qq)
  const int qq = pix % q;
  const int pp = (pix / q) % p;
  const int nn = pix / (p * q);
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  int bt[4] = {0, 0, 0, 0};
#pragma unroll
  for (int r = 0; r < (K ? K : 16); ++r) {
    if (!K && r >= kr) break;
    const int ih = pp * stride - pad + r;
#pragma unroll
    for (int s = 0; s < (K ? K : 16); ++s) {
      if (!K && s >= ks) break;
      const int iw = qq * stride - pad + s;
      if (ih < 0 || ih >= h || iw < 0 || iw >= w) continue;
      const float4 v = __ldg(x4 + ((static_cast<long long>(nn) * h + ih) * w + iw) * c4 + cg);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (vv[j] > best[j]) {
          best[j] = vv[j];
          bt[j] = r * ks + s;
        }
    }
  }
  const uint32_t packed = static_cast<uint32_t>(bt[0]) | (static_cast<uint32_t>(bt[1]) << 8) |
                          (static_cast<uint32_t>(bt[2]) << 16) | (static_cast<uint32_t>(bt[3]) << 24);
  reinterpret_cast<uint32_t*>(arg)[static_cast<long long>(pix) * c4 + cg] = packed;
}

template <int K, int ST, int PD>
__global__ void maxpool_gather_kernel(const uint8_t* __restrict__ arg, const float* __restrict__ dy,
                                      int n, int h, int w, int c4, int kr_, int ks_, int stride_,
                                      int pad_, int p, int q, float* __restrict__ dx, int total) {
  pdl_wait();
  pdl_trigger();
  const int kr = K ? K : kr_, ks = K ? K : ks_, stride = ST ? ST : stride_, pad = K ? PD : pad_;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // (pixel, channel float4)
  if (idx >= total) return;
  const int cg = idx % c4;
  const int pix = idx / c4;  // (n, hh, ww)
  const int ww = pix % w;
  const int hh = (pix / w) % h;
  const int nn = pix / (w * h);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const int p_lo = max(0, (hh + pad - kr + stride) / stride);
  const int p_hi = min(p - 1, (hh + pad) / stride);
  const int q_lo = max(0, (ww + pad - ks + stride) / stride);
  const int q_hi = min(q - 1, (ww + pad) / stride);
  const uint32_t* a32 = reinterpret_cast<const uint32_t*>(arg);
  const float4* dy4 = reinterpret_cast<const float4*>(dy);
  // windows covering this element: at most ceil(K/ST)^2 (2x2 for the stem)
  constexpr int kW = K ? (K + ST - 1) / ST : 8;
  const int np = p_hi - p_lo + 1, nq = q_hi - q_lo + 1;
#pragma unroll
  for (int i = 0; i < kW; ++i) {
    if (i >= np) break;
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      if (j >= nq) break;
      const int pp = p_lo + i, qq = q_lo + j;
      const int tap = (hh - (pp * stride - pad)) * ks + (ww - (qq * stride - pad));
      const long long o = (static_cast<long long>(nn) * p + pp) * q + qq;
      const uint32_t packed = __ldg(a32 + o * c4 + cg);
      const float4 g = __ldg(dy4 + o * c4 + cg);  // loaded unconditionally: all in flight
      if ((packed & 0xFF) == static_cast<uint32_t>(tap)) acc[0] += g.x;
      if (((packed >> 8) & 0xFF) == static_cast<uint32_t>(tap)) acc[1] += g.y;
      if (((packed >> 16) & 0xFF) == static_cast<uint32_t>(tap)) acc[2] += g.z;
      if ((packed >> 24) == static_cast<uint32_t>(tap)) acc[3] += g.w;
    }
  }
  reinterpret_cast<float4*>(dx)[static_cast<long long>(pix) * c4 + cg] =
      make_float4(acc[0], acc[1], acc[2], acc[3]);
}

__global__ void avgpool_fwd_kernel(const float* __restrict__ x, int n, int hw, int c,
                                   float* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int total = n * c;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int nn = i / c, cc = i - nn * c;
    const float* base = x + static_cast<long long>(nn) * hw * c + cc;
    float acc = 0.f;
    for (int j = 0; j < hw; ++j) acc += base[static_cast<long long>(j) * c];
    y[i] = acc / static_cast<float>(hw);
  }
}

// dx[n][j][c] = dy[n][c] / hw; grid (channel float4 blocks, n * hw pixels)
__global__ void avgpool_bwd_kernel(const float* __restrict__ dy, int n, int hw, int c,
                                   float* __restrict__ dx) {
  pdl_wait();
  pdl_trigger();
  const int c4 = c / 4;
  const int cg = blockIdx.x * blockDim.x + threadIdx.x;
  if (cg >= c4) return;
  const int pix = blockIdx.y;  // n * hw + j
  const int nn = pix / hw;
  const float inv = 1.f / static_cast<float>(hw);
  float4 g = reinterpret_cast<const float4*>(dy)[static_cast<long long>(nn) * c4 + cg];
  g.x *= inv;
  g.y *= inv;
  g.z *= inv;
  g.w *= inv;
  reinterpret_cast<float4*>(dx)[static_cast<long long>(pix) * c4 + cg] = g;
}

// ---------------------------------------------------------------------------
// classifier
// ---------------------------------------------------------------------------
__global__ void bias_add_kernel(float* y, const float* b, long long m, int n) {
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
    // an out-of-range label poisons the loss (NaN) and contributes no target
    // term to the gradient instead of reading outside the row
    const int y = labels[row];
    const bool valid = y >= 0 && y < classes;
    if (lane == 0) my_loss += valid ? mx + logf(se) - z[y] : __int_as_float(0x7fc00000);
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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

// debug: subsequent BN launches stamp %globaltimer per block into buf
// (8 int64 per block: entry, phase-1 loop done, partial published, phase 2
// done, phase 3 done); NULL = off
extern "C" int accudnn_bn_trace(void* buf) {
  accudnn::g_bn_trace = static_cast<long long*>(buf);
  return 0;
}

extern "C" int accudnn_set_pdl(int enable) {
  const int prev = accudnn::g_pdl;
  accudnn::g_pdl = enable ? 1 : 0;
  return prev;
}

extern "C" unsigned long long accudnn_bn_workspace_bytes(int C) {
  return sizeof(unsigned) * kBnCounters + sizeof(float) * 2ull * kBnMaxBlocks * kBnGroup;
}

extern "C" int accudnn_bn_fwd(const float* x, long long M, int C, const float* gamma,
                              const float* beta, float eps, int relu, float* y,
                              float* save_mean, float* save_invstd, float* running_mean,
                              float* running_var, float momentum, void* ws, void* stream) {
  if ((C & 3) || M <= 0 || C > 32 * kBnMaxGroups) return static_cast<int>(cudaErrorInvalidValue);
  BnArgs a{};
  a.x = x;
  a.M = M;
  a.C = C;
  a.relu = relu;
  a.gamma = gamma;
  a.beta = beta;
  a.eps = eps;
  a.momentum = momentum;
  a.save_mean = save_mean;
  a.save_invstd = save_invstd;
  a.run_mean = running_mean;
  a.run_var = running_var;
  a.y = y;
  a.w = bn_ws(ws, C);
  a.trace = g_bn_trace;
  return bn_launch<0, false>(a, S(stream));
}

// forward batch norm whose statistics come from the producing convolution
// (accudnn_conv_fwd_stats): only the normalise pass reads x
namespace accudnn {
namespace {
// ---- batch norm forward from the producing conv's statistics ----------------
// With the column sums / sums of squares of every 32-row slot of x written by
// the conv epilogue ([2][P][C], accudnn_conv_fwd_stats), the forward needs no
// statistics pass over x and no grid-wide exchange: a small kernel finalises
// the per-channel scale / shift (fixed-order reduction, so every element sees
// the same coefficients) and an element-wise kernel normalises.
__global__ void __launch_bounds__(256) bn_stats_finalize_kernel(
    const float* __restrict__ stats, long long P, int C, long long M, const float* gamma,
    const float* beta, float eps, float momentum, float* run_mean, float* run_var,
    float* save_mean, float* save_invstd, float* __restrict__ coef) {
  __shared__ double red[2][256][4];
  const int c = blockIdx.x * 4;
  double s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
#pragma unroll 4
  for (long long r = threadIdx.x; r < P; r += 256) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(stats + r * C + c));
    const float4 q = __ldcg(reinterpret_cast<const float4*>(stats + (P + r) * C + c));
    s1[0] += v.x; s1[1] += v.y; s1[2] += v.z; s1[3] += v.w;
    s2[0] += q.x; s2[1] += q.y; s2[2] += q.z; s2[3] += q.w;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    red[0][threadIdx.x][j] = s1[j];
    red[1][threadIdx.x][j] = s2[j];
  }
  __syncthreads();
  for (int n = 128; n >= 1; n >>= 1) {  // fixed-shape tree
    if (static_cast<int>(threadIdx.x) < n)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        red[0][threadIdx.x][j] += red[0][threadIdx.x + n][j];
        red[1][threadIdx.x][j] += red[1][threadIdx.x + n][j];
      }
    __syncthreads();
  }
  if (threadIdx.x < 4) {
    const int j = threadIdx.x, ch = c + j;
    const double mean = red[0][0][j] / static_cast<double>(M);
    double var = red[1][0][j] / static_cast<double>(M) - mean * mean;
    if (var < 0) var = 0;
    const float inv = static_cast<float>(1.0 / sqrt(var + static_cast<double>(eps)));
    const float sc = gamma[ch] * inv;
    coef[ch] = sc;
    coef[C + ch] = beta[ch] - static_cast<float>(mean) * sc;
    if (save_mean) save_mean[ch] = static_cast<float>(mean);
    if (save_invstd) save_invstd[ch] = inv;
    if (run_mean && run_var && M > 1) {
      const double unbiased = var * static_cast<double>(M) / static_cast<double>(M - 1);
      run_mean[ch] = (1.f - momentum) * run_mean[ch] + momentum * static_cast<float>(mean);
      run_var[ch] = (1.f - momentum) * run_var[ch] + momentum * static_cast<float>(unbiased);
    }
  }
}

template <bool RELU, bool SKIP>
__global__ void __launch_bounds__(256) bn_apply_kernel(const float4* __restrict__ x,
                                                       const float4* __restrict__ skip,
                                                       const float* __restrict__ coef, int C,
                                                       long long n4, float4* __restrict__ y) {
  const int c4 = C >> 2;
  const float4* sc4 = reinterpret_cast<const float4*>(coef);
  const float4* sh4 = reinterpret_cast<const float4*>(coef + C);
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += gridDim.x * 256LL) {
    const int q = static_cast<int>(i % c4);
    const float4 sc = __ldg(sc4 + q), sh = __ldg(sh4 + q);
    float4 v = __ldcs(x + i);
    v.x = v.x * sc.x + sh.x;
    v.y = v.y * sc.y + sh.y;
    v.z = v.z * sc.z + sh.z;
    v.w = v.w * sc.w + sh.w;
    if (SKIP) {
      const float4 k = __ldcs(skip + i);
      v.x += k.x;
      v.y += k.y;
      v.z += k.z;
      v.w += k.w;
    }
    if (RELU) {
      v.x = fmaxf(v.x, 0.f);
      v.y = fmaxf(v.y, 0.f);
      v.z = fmaxf(v.z, 0.f);
      v.w = fmaxf(v.w, 0.f);
    }
    y[i] = v;
  }
}

// ACCUDNN_BN_STATS_SPLIT=0: the cooperative fused kernel with stats_in instead
bool bn_stats_split() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("ACCUDNN_BN_STATS_SPLIT");
    v = e ? std::atoi(e) : 1;
  }
  return v != 0;
}

int bn_fwd_from_stats(const float* x, const float* stats, const float* skip, long long M, int C,
                      const float* gamma, const float* beta, float eps, int relu, float* y,
                      float* save_mean, float* save_invstd, float* running_mean,
                      float* running_var, float momentum, void* ws, cudaStream_t st) {
  // coefficients in the BN workspace's partial area (2 C floats)
  float* coef = bn_ws(ws, C).part;
  const long long P = (M + 31) / 32;
  bn_stats_finalize_kernel<<<C / 4, 256, 0, st>>>(stats, P, C, M, gamma, beta, eps, momentum,
                                                  running_mean, running_var, save_mean,
                                                  save_invstd, coef);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return static_cast<int>(e);
  const long long n4 = M * C / 4;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(std::min<long long>((n4 + 255) / 256, 8LL * sms));
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* k4 = reinterpret_cast<const float4*>(skip);
  float4* y4 = reinterpret_cast<float4*>(y);
  if (skip)
    bn_apply_kernel<true, true><<<grid, 256, 0, st>>>(x4, k4, coef, C, n4, y4);
  else if (relu)
    bn_apply_kernel<true, false><<<grid, 256, 0, st>>>(x4, k4, coef, C, n4, y4);
  else
    bn_apply_kernel<false, false><<<grid, 256, 0, st>>>(x4, k4, coef, C, n4, y4);
  return static_cast<int>(cudaGetLastError());
}
}  // namespace
}  // namespace accudnn

extern "C" int accudnn_bn_fwd_stats(const float* x, const float* stats, long long M, int C,
                                    const float* gamma, const float* beta, float eps, int relu,
                                    float* y, float* save_mean, float* save_invstd,
                                    float* running_mean, float* running_var, float momentum,
                                    void* ws, void* stream) {
  if ((C & 3) || M <= 0 || C > 32 * kBnMaxGroups || !stats)
    return static_cast<int>(cudaErrorInvalidValue);
  if (bn_stats_split())
    return bn_fwd_from_stats(x, stats, nullptr, M, C, gamma, beta, eps, relu, y, save_mean,
                             save_invstd, running_mean, running_var, momentum, ws, S(stream));
  BnArgs a{};
  a.x = x;
  a.stats_in = stats;
  a.M = M;
  a.C = C;
  a.relu = relu;
  a.gamma = gamma;
  a.beta = beta;
  a.eps = eps;
  a.momentum = momentum;
  a.save_mean = save_mean;
  a.save_invstd = save_invstd;
  a.run_mean = running_mean;
  a.run_var = running_var;
  a.y = y;
  a.w = bn_ws(ws, C);
  a.trace = g_bn_trace;
  return bn_launch<0, false>(a, S(stream));
}

extern "C" int accudnn_bn_bwd(const float* x, const float* dy, long long M, int C,
                              const float* gamma, const float* beta, const float* save_mean,
                              const float* save_invstd, int relu, float* dx, int dx_beta,
                              float* dgamma, float* dbeta, void* ws, void* stream) {
  if ((C & 3) || M <= 0 || C > 32 * kBnMaxGroups) return static_cast<int>(cudaErrorInvalidValue);
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
  a.dx = dx;
  a.dx_beta = dx_beta;
  a.w = bn_ws(ws, C);
  a.trace = g_bn_trace;
  return bn_launch<1, false>(a, S(stream));
}

// y = relu(bn(x) + skip) over [M][C] (the residual tail of a ResNet block)
extern "C" int accudnn_bn_add_relu_fwd(const float* x, const float* skip, long long M, int C,
                                       const float* gamma, const float* beta, float eps, float* y,
                                       float* save_mean, float* save_invstd, float* running_mean,
                                       float* running_var, float momentum, void* ws,
                                       void* stream) {
  if ((C & 3) || M <= 0 || C > 32 * kBnMaxGroups) return static_cast<int>(cudaErrorInvalidValue);
  BnArgs a{};
  a.x = x;
  a.skip = skip;
  a.M = M;
  a.C = C;
  a.relu = 1;
  a.gamma = gamma;
  a.beta = beta;
  a.eps = eps;
  a.momentum = momentum;
  a.save_mean = save_mean;
  a.save_invstd = save_invstd;
  a.run_mean = running_mean;
  a.run_var = running_var;
  a.y = y;
  a.w = bn_ws(ws, C);
  return bn_launch<0, true>(a, S(stream));
}

extern "C" int accudnn_bn_add_relu_fwd_stats(const float* x, const float* stats,
                                             const float* skip, long long M, int C,
                                             const float* gamma, const float* beta, float eps,
                                             float* y, float* save_mean, float* save_invstd,
                                             float* running_mean, float* running_var,
                                             float momentum, void* ws, void* stream) {
  if ((C & 3) || M <= 0 || C > 32 * kBnMaxGroups || !stats)
    return static_cast<int>(cudaErrorInvalidValue);
  if (bn_stats_split())
    return bn_fwd_from_stats(x, stats, skip, M, C, gamma, beta, eps, 1, y, save_mean, save_invstd,
                             running_mean, running_var, momentum, ws, S(stream));
  BnArgs a{};
  a.x = x;
  a.stats_in = stats;
  a.skip = skip;
  a.M = M;
  a.C = C;
  a.relu = 1;
  a.gamma = gamma;
  a.beta = beta;
  a.eps = eps;
  a.momentum = momentum;
  a.save_mean = save_mean;
  a.save_invstd = save_invstd;
  a.run_mean = running_mean;
  a.run_var = running_var;
  a.y = y;
  a.w = bn_ws(ws, C);
  return bn_launch<0, true>(a, S(stream));
}

// backward of y = relu(bn(x) + skip): g = dy * [bn(x) + skip > 0] (mask
// recomputed from the inputs), dskip (+)= g, dx (+)= BN backward of g
extern "C" int accudnn_bn_add_relu_bwd(const float* x, const float* skip, const float* dy,
                                       long long M, int C, const float* gamma, const float* beta,
                                       const float* save_mean, const float* save_invstd,
                                       float* dx, int dx_beta, float* dskip, int dskip_beta,
                                       float* dgamma, float* dbeta, void* ws, void* stream) {
  if ((C & 3) || M <= 0 || C > 32 * kBnMaxGroups) return static_cast<int>(cudaErrorInvalidValue);
  BnArgs a{};
  a.x = x;
  a.skip = skip;
  a.dy = dy;
  a.M = M;
  a.C = C;
  a.relu = 1;
  a.gamma = gamma;
  a.beta = beta;
  a.mean = save_mean;
  a.invstd = save_invstd;
  a.dgamma = dgamma;
  a.dbeta = dbeta;
  a.dx = dx;
  a.dx_beta = dx_beta;
  a.dskip = dskip;
  a.dskip_beta = dskip_beta;
  a.w = bn_ws(ws, C);
  return bn_launch<1, true>(a, S(stream));
}

namespace accudnn {
namespace {
// y = relu(x * sc + sh), sc = gamma * invstd, sh = beta - mean * sc: the
// forward's batch-norm output bit for bit (the same float scale / shift and
// contraction as phase 3 of bn_fused_kernel<0>), recomputed from the saved
// statistics.  Threads own 4 channels (x) and stride over rows (y).
__global__ void bn_relu_apply_kernel(const float* __restrict__ x, long long M, int C,
                                     const float* __restrict__ gamma, const float* __restrict__ beta,
                                     const float* __restrict__ mean,
                                     const float* __restrict__ invstd, float* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (c >= C) return;
  float sc[4], sh[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    sc[j] = gamma[c + j] * invstd[c + j];
    sh[j] = beta[c + j] - mean[c + j] * sc[j];
  }
  const uint64_t p_last = l2_policy(2);
  const long long step = static_cast<long long>(blockDim.y) * gridDim.y;
  long long r = static_cast<long long>(blockIdx.y) * blockDim.y + threadIdx.y;
  for (; r + 3 * step < M; r += 4 * step) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ld_pol(x + (r + u * step) * C + c, p_last);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float4 o = v[u];
      o.x = fmaxf(o.x * sc[0] + sh[0], 0.f);
      o.y = fmaxf(o.y * sc[1] + sh[1], 0.f);
      o.z = fmaxf(o.z * sc[2] + sh[2], 0.f);
      o.w = fmaxf(o.w * sc[3] + sh[3], 0.f);
      *reinterpret_cast<float4*>(y + (r + u * step) * C + c) = o;
    }
  }
  for (; r < M; r += step) {
    float4 o = ld_pol(x + r * C + c, p_last);
    o.x = fmaxf(o.x * sc[0] + sh[0], 0.f);
    o.y = fmaxf(o.y * sc[1] + sh[1], 0.f);
    o.z = fmaxf(o.z * sc[2] + sh[2], 0.f);
    o.w = fmaxf(o.w * sc[3] + sh[3], 0.f);
    *reinterpret_cast<float4*>(y + r * C + c) = o;
  }
}
}  // namespace
}  // namespace accudnn

extern "C" int accudnn_bn_relu_apply(const float* x, long long M, int C, const float* gamma,
                                     const float* beta, const float* save_mean,
                                     const float* save_invstd, float* y, void* stream) {
  if ((C & 3) || M <= 0) return static_cast<int>(cudaErrorInvalidValue);
  const int c4 = C / 4;
  const int lanes = c4 < 32 ? c4 : 32;
  const dim3 block(lanes, 256 / lanes);
  const int gx = (c4 + lanes - 1) / lanes;
  const long long rows_per_block = static_cast<long long>(block.y) * 4;
  long long gy = (M + rows_per_block - 1) / rows_per_block;
  const long long cap = std::max<long long>(1, 148LL * 8 / gx);
  if (gy > cap) gy = cap;
  launch_pdl(bn_relu_apply_kernel, dim3(gx, static_cast<unsigned>(gy)), block, 0, S(stream), x, M, C,
             gamma, beta, save_mean, save_invstd, y);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_relu_fwd(const float* x, float* y, long long n, void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  launch_pdl(relu_fwd_kernel, grid_for(n / 4, kThreads), kThreads, 0, S(stream), 
      reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), n / 4);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_relu_bwd(const float* x, const float* dy, float* dx, long long n,
                                int dx_beta, void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  launch_pdl(relu_bwd_kernel, grid_for(n / 4, kThreads), kThreads, 0, S(stream), 
      reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(dy),
      reinterpret_cast<float4*>(dx), n / 4, dx_beta);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_add_fwd(const float* a, const float* b, float* y, long long n,
                               void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  launch_pdl(add_kernel, grid_for(n / 4, kThreads), kThreads, 0, S(stream), 
      reinterpret_cast<const float4*>(a), reinterpret_cast<const float4*>(b),
      reinterpret_cast<float4*>(y), n / 4);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_copy(const float* src, float* dst, long long n, int beta, void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  launch_pdl(copy_kernel, grid_for(n / 4, kThreads), kThreads, 0, S(stream), 
      reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), n / 4, beta);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_maxpool_fwd(const float* x, int n, int h, int w, int c, int kr, int ks,
                                   int stride, int pad, int p, int q, float* y, void* stream) {
  if (c & 3) return static_cast<int>(cudaErrorInvalidValue);
  const long long total = static_cast<long long>(n) * p * q * (c / 4);
  launch_pdl(maxpool_fwd_kernel, grid_for(total, kThreads), kThreads, 0, S(stream), 
      x, n, h, w, c / 4, kr, ks, stride, pad, p, q, y);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_maxpool_bwd(const float* x, const float* dy, int n, int h, int w, int c,
                                   int kr, int ks, int stride, int pad, int p, int q, float* dx,
                                   void* stream) {
  if (c & 3) return static_cast<int>(cudaErrorInvalidValue);
  const int c4 = c / 4;
  conv_select_workspace(S(stream));
  // argmax bytes live in the convolution split-K workspace (idle between
  // convolutions on this stream); without one, the single-pass kernel
  const long long in4 = static_cast<long long>(n) * h * w * c4;
  const long long out4 = static_cast<long long>(n) * p * q * c4;
  uint8_t* arg = (kr <= 16 && ks <= 16 && (kr + stride - 1) / stride <= 8 &&
                  (ks + stride - 1) / stride <= 8 && in4 < (1LL << 31) && out4 < (1LL << 31))
                     ? reinterpret_cast<uint8_t*>(
                           conv_splitk_workspace(static_cast<size_t>(n) * p * q * c))
                     : nullptr;
  if (arg) {
    const unsigned ga = static_cast<unsigned>((out4 + 255) / 256);
    const unsigned gg = static_cast<unsigned>((in4 + 255) / 256);
    if (kr == 3 && ks == 3 && stride == 2 && pad == 1) {
      launch_pdl(maxpool_argmax_kernel<3, 2, 1>, ga, 256, 0, S(stream), x, n, h, w, c4, kr, ks,
                 stride, pad, p, q, arg, static_cast<int>(out4));
      launch_pdl(maxpool_gather_kernel<3, 2, 1>, gg, 256, 0, S(stream), arg, dy, n, h, w, c4, kr,
                 ks, stride, pad, p, q, dx, static_cast<int>(in4));
    } else {
      launch_pdl(maxpool_argmax_kernel<0, 0, 0>, ga, 256, 0, S(stream), x, n, h, w, c4, kr, ks,
                 stride, pad, p, q, arg, static_cast<int>(out4));
      launch_pdl(maxpool_gather_kernel<0, 0, 0>, gg, 256, 0, S(stream), arg, dy, n, h, w, c4, kr,
                 ks, stride, pad, p, q, dx, static_cast<int>(in4));
    }
    return static_cast<int>(cudaGetLastError());
  }
  const long long total = static_cast<long long>(n) * h * w * c4;
  launch_pdl(maxpool_bwd_kernel, grid_for(total, kThreads), kThreads, 0, S(stream), x, dy, n, h,
             w, c4, kr, ks, stride, pad, p, q, dx);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_avgpool_fwd(const float* x, int n, int hw, int c, float* y,
                                   void* stream) {
  launch_pdl(avgpool_fwd_kernel, grid_for(static_cast<long long>(n) * c, kThreads), kThreads, 0, S(stream), x, n, hw, c, y);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_avgpool_bwd(const float* dy, int n, int hw, int c, float* dx,
                                   void* stream) {
  if (c & 3) return static_cast<int>(cudaErrorInvalidValue);
  launch_pdl(avgpool_bwd_kernel, dim3((c / 4 + 127) / 128, static_cast<unsigned>(n * hw)), 128, 0,
             S(stream), dy, n, hw, c, dx);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_bias_add(float* y, const float* bias, long long m, int n, void* stream) {
  launch_pdl(bias_add_kernel, grid_for(m * n, kThreads), kThreads, 0, S(stream), y, bias, m, n);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_xent_fwd(const float* logits, const int* labels, int rows, int classes,
                                float* loss, void* stream) {
  launch_pdl(xent_kernel, 1, kXentThreads, 0, S(stream), logits, labels, rows, classes, loss, nullptr,
                                                 nullptr);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_xent_bwd(const float* logits, const int* labels, int rows, int classes,
                                float* dlogits, float* dbias, void* stream) {
  launch_pdl(xent_kernel, 1, kXentThreads, 0, S(stream), logits, labels, rows, classes, nullptr,
                                                 dlogits, dbias);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_sgd_update(float* w, const float* g, float* buf, long long n, float lr,
                                  float momentum, float weight_decay, float grad_scale,
                                  int first_step, void* stream) {
  if (n & 3) return static_cast<int>(cudaErrorInvalidValue);
  launch_pdl(sgd_kernel, grid_for(n / 4, kThreads), kThreads, 0, S(stream), 
      reinterpret_cast<float4*>(w), reinterpret_cast<const float4*>(g),
      reinterpret_cast<float4*>(buf), n / 4, lr, momentum, weight_decay, grad_scale,
      first_step);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int accudnn_nchw_to_nhwc_pad(const float* x, int n, int c, int h, int w, int c4,
                                        float* y, void* stream) {
  const long long total = static_cast<long long>(n) * h * w * c4;
  launch_pdl(nchw_to_nhwc_kernel, grid_for(total, kThreads), kThreads, 0, S(stream), x, n, c, h, w, c4,
                                                                            y);
  return static_cast<int>(cudaGetLastError());
}
