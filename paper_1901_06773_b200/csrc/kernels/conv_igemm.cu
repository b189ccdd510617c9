// Implicit-GEMM convolution on the 5th-generation tensor cores (sm_100a).
//
// One kernel template covers the three convolution GEMMs of a training step
// (NHWC fp32 activations, weights [Cout][R][S][Cin], TF32 tensor-core math,
// FP32 accumulation in TMEM):
//
//   FWD    y[m=(n,p,q)][co]       = sum_{(r,s,ci)} x(im2col)   * w[co][(r,s,ci)]
//          A = im2col(x)  K-major      B = w            K-major
//   DGRAD  dx[m=(n,h,w)][ci]      = sum_{(r,s,co)} dy(col2im)  * w[co][r][s][ci]
//          A = gather(dy) K-major      B = w            MN-major (ci contiguous)
//   WGRAD  dw[co][(r,s,ci)]       = sum_{m=(n,p,q)} dy[m][co]  * x(im2col)[m][(r,s,ci)]
//          A = dy         MN-major     B = im2col(x)    MN-major
//
// A fully connected layer is the 1x1 conv on a 1x1 image, so FC forward /
// backward run through the same kernel.
//
// Structure (warp-specialised, one 128 x BN output tile per CTA):
//   warps 0-3  producers: gather 16-byte chunks (4 channels) straight from
//              global memory into the SWIZZLE_128B UMMA layout with
//              cp.async (zero-fill handles padding, stride holes and tails),
//              then arrive on the stage's full barrier when they land;
//              afterwards they are the epilogue (TMEM -> registers -> HBM).
//   warp 4     TMEM allocator + single-thread tcgen05.mma issuer; commits
//              free the smem stage and finally signal the accumulator.
// A 3-stage ring of 16 KB (A) + BN*128 B (B) lets two CTAs share an SM so
// one CTA's epilogue overlaps the other's main loop.  Split-K (gridDim.z)
// reduces with fp32 atomics for the small-M / huge-K weight gradients.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "accudnn_kernels.h"
#include "pdl.cuh"
#include "sm100_ptx.cuh"

namespace accudnn {
// split-K workspace + slice-order reduction (conv_sm100.cu)
float* conv_splitk_workspace(size_t bytes);
void conv_select_workspace(cudaStream_t st);
int conv_splitk_reduce(float* ws, int splits, int M, int Ng, float* out, int beta,
                       cudaStream_t st);
namespace {

constexpr int kBM = 128;        // rows per tile (UMMA M)
constexpr int kBK = 32;         // fp32 elements per 128-byte swizzle row
constexpr int kStages = 3;
constexpr int kProducers = 128; // warps 0-3
constexpr int kThreads = 160;   // + MMA warp

enum Mode : int { FWD = 0, DGRAD = 1, WGRAD = 2 };

struct Args {
  int N, H, W, C, K, R, S, stride, pad, P, Q;
  int M, Ng, Kg;       // GEMM extents
  int kb_total;        // ceil(Kg / 32)
  int kb_per_split;
  const float* a_src;  // FWD: x   DGRAD: dy  WGRAD: dy
  const float* b_src;  // FWD: w   DGRAD: w   WGRAD: x
  float* out;
  int beta;            // 1: accumulate into out
  int atomic;          // split-K partial sums (fp32 atomics into out)
  float* ws;           // split-K partials [split][M][Ng] (deterministic), or nullptr
  int mn_lbo, mn_sbo;  // MN-major descriptor strides (bytes, 0 = derived)
  int mn_layout;       // MN-major descriptor layout type (1 = SW128_BASE32B)
  int mn_kstep;        // debug override of the per-K=8 start advance
};

// byte offset of 16-byte chunk `j` of row `row` in a K-major SW128 tile
__device__ __forceinline__ uint32_t kmaj_off(int row, int j) {
  return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + ((j ^ (row & 7)) << 4));
}
// byte offset of the chunk holding MN columns [col, col+4) of K-row `kr` in
// an MN-major tile `mn` elements wide.  TF32 MN-major operands must use the
// SWIZZLE_128B_BASE32B layout: atoms of 4 K-rows x 128 bytes (32 elements)
// with Swizzle<2,5,2> (32-byte granules XOR the row).  Atoms are laid out
// MN-first: MN-atom stride 512 B (LBO), K-group stride (mn/32)*512 B (SBO).
__device__ __forceinline__ uint32_t mnmaj_off(int kr, int col, int mn) {
  const int atom = col >> 5, c16 = (col & 31) >> 2, rr = kr & 3, grp = kr >> 2;
  return static_cast<uint32_t>(grp * (mn / 32) * 512 + atom * 512 + rr * 128 +
                               (((c16 >> 1) ^ rr) << 5) + ((c16 & 1) << 4));
}

// PRECISE selects 3xTF32: each operand x is split into hi = tf32(x) and
// lo = x - hi after it lands in shared memory, and the tile product is
// hi*hi + hi*lo + lo*hi, which recovers ~fp32 accuracy at 3x the MMA work
// (the validation / "fp32-exact" mode; the training default is TF32).
template <int MODE, int BN, bool PRECISE>
__global__ void __launch_bounds__(kThreads, 1)
    conv_igemm_kernel(const Args a) {
  constexpr bool kAmn = (MODE == WGRAD);
  constexpr bool kBmn = (MODE != FWD);
  constexpr uint32_t kABytes = kBM * kBK * 4;
  constexpr uint32_t kBBytes = BN * kBK * 4;
  constexpr uint32_t kLoDelta = kABytes + kBBytes;  // hi tile -> lo tile
  constexpr uint32_t kStageBytes = kLoDelta * (PRECISE ? 2 : 1);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* accum = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kBM;
  const int n0 = blockIdx.y * BN;
  const int kb_begin = blockIdx.z * a.kb_per_split;
  const int kb_end = min(a.kb_total, kb_begin + a.kb_per_split);
  const int nkb = kb_end - kb_begin;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], kProducers);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accum, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 4) ptx::tmem_alloc<BN>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  pdl_wait();
  pdl_trigger();
  const uint32_t tmem = *tmem_slot;
  const uint32_t smem_base = ptx::smem_u32(smem);

  if (warp < 4) {
    // ============================ producers ============================
    const int t = threadIdx.x;
    // per-row state for K-major A (FWD / DGRAD): 8 rows per thread
    const int aj = t & 7;        // 16-byte chunk within the 128-byte row
    const int arow0 = t >> 3;    // 0..15
    long long a_base[8];
    int a_h[8], a_w[8];
    if constexpr (!kAmn) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = m0 + arow0 + 16 * i;
        a_base[i] = -1;
        a_h[i] = 0;
        a_w[i] = 0;
        if (m < a.M) {
          if constexpr (MODE == FWD) {
            const int pq = a.P * a.Q;
            const int n = m / pq, rem = m - n * pq;
            const int p = rem / a.Q, q = rem - p * a.Q;
            a_base[i] = static_cast<long long>(n) * a.H * a.W * a.C;
            a_h[i] = p * a.stride - a.pad;
            a_w[i] = q * a.stride - a.pad;
          } else {  // DGRAD: row = input pixel, gathers dy
            const int hw = a.H * a.W;
            const int n = m / hw, rem = m - n * hw;
            const int h = rem / a.W, w = rem - h * a.W;
            a_base[i] = static_cast<long long>(n) * a.P * a.Q * a.K;
            a_h[i] = h + a.pad;
            a_w[i] = w + a.pad;
          }
        }
      }
    }
    // WGRAD B: fixed (tap, ci) column per thread
    constexpr int kBcpr = BN / 4;             // chunks per K-row of an MN-major B tile
    constexpr int kBrowStep = kProducers / kBcpr;
    int wb_r = 0, wb_s = 0, wb_ci = 0;
    bool wb_col_ok = false;
    if constexpr (MODE == WGRAD) {
      const int col = n0 + 4 * (t % kBcpr);
      wb_col_ok = col < a.Ng;
      const int tap = col / a.C;
      wb_ci = col - tap * a.C;
      wb_r = tap / a.S;
      wb_s = tap - wb_r * a.S;
    }

    uint32_t my_dst[16];
    int n_dst = 0;
    auto put = [&](uint32_t dst, const void* src, uint32_t bytes) {
      ptx::cp_async16(dst, src, bytes);
      if constexpr (PRECISE) my_dst[n_dst++] = dst;
    };
    for (int it = 0; it < nkb; ++it) {
      const int stage = it % kStages;
      if (it >= kStages) ptx::mbar_wait(&empty[stage], ((it / kStages) - 1) & 1);
      n_dst = 0;
      const int kb = kb_begin + it;
      const uint32_t sA = smem_base + stage * kStageBytes;
      const uint32_t sB = sA + kABytes;

      // ---------------- A tile ----------------
      if constexpr (!kAmn) {
        const int kk = kb * kBK + 4 * aj;
        const bool k_ok = kk < a.Kg;
        int r = 0, s = 0, c = 0;
        if (k_ok) {
          const int cdim = (MODE == FWD) ? a.C : a.K;
          const int tap = kk / cdim;
          c = kk - tap * cdim;
          r = tap / a.S;
          s = tap - r * a.S;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = arow0 + 16 * i;
          const float* src = a.a_src;
          uint32_t bytes = 0;
          if (k_ok && a_base[i] >= 0) {
            if constexpr (MODE == FWD) {
              const int h = a_h[i] + r, w = a_w[i] + s;
              if (h >= 0 && h < a.H && w >= 0 && w < a.W) {
                src = a.a_src + a_base[i] + (static_cast<long long>(h) * a.W + w) * a.C + c;
                bytes = 16;
              }
            } else {
              const int hp = a_h[i] - r, wp = a_w[i] - s;
              if (hp >= 0 && wp >= 0) {
                int p = hp, q = wp;
                bool ok = true;
                if (a.stride != 1) {
                  ok = (hp % a.stride == 0) && (wp % a.stride == 0);
                  p = hp / a.stride;
                  q = wp / a.stride;
                }
                if (ok && p < a.P && q < a.Q) {
                  src = a.a_src + a_base[i] + (static_cast<long long>(p) * a.Q + q) * a.K + c;
                  bytes = 16;
                }
              }
            }
          }
          put(sA + kmaj_off(row, aj), src, bytes);
        }
      } else {
        // WGRAD A = dy (pixels x Cout), MN-major: K-rows are pixels
        const int col = 4 * (t & 31);
        const int co = m0 + col;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int kr = (t >> 5) + 4 * i;
          const int pix = kb * kBK + kr;
          const bool ok = pix < a.Kg && co < a.M;
          const float* src =
              ok ? a.a_src + static_cast<long long>(pix) * a.K + co : a.a_src;
          put(sA + mnmaj_off(kr, col, kBM), src, ok ? 16u : 0u);
        }
      }

      // ---------------- B tile ----------------
      if constexpr (MODE == FWD) {
        const int kk = kb * kBK + 4 * aj;
#pragma unroll
        for (int i = 0; i < BN / 16; ++i) {
          const int row = arow0 + 16 * i;
          const int co = n0 + row;
          const bool ok = co < a.K && kk < a.Kg;
          const float* src = ok ? a.b_src + static_cast<long long>(co) * a.Kg + kk : a.b_src;
          put(sB + kmaj_off(row, aj), src, ok ? 16u : 0u);
        }
      } else if constexpr (MODE == DGRAD) {
        // B[(r,s,co)][ci] = w[co][r][s][ci]
        const int col = 4 * (t % kBcpr);
        const int ci = n0 + col;
#pragma unroll
        for (int i = 0; i < kBK / kBrowStep; ++i) {
          const int kr = t / kBcpr + kBrowStep * i;
          const int kk = kb * kBK + kr;
          bool ok = kk < a.Kg && ci < a.C;
          const float* src = a.b_src;
          if (ok) {
            const int tap = kk / a.K, co = kk - tap * a.K;
            src = a.b_src + (static_cast<long long>(co) * a.R * a.S + tap) * a.C + ci;
          }
          put(sB + mnmaj_off(kr, col, BN), src, ok ? 16u : 0u);
        }
      } else {
        // WGRAD B[(r,s,ci)][pix] = x[n][p*st-pad+r][q*st-pad+s][ci]
        const int col = 4 * (t % kBcpr);
        const int pq = a.P * a.Q;
#pragma unroll
        for (int i = 0; i < kBK / kBrowStep; ++i) {
          const int kr = t / kBcpr + kBrowStep * i;
          const int pix = kb * kBK + kr;
          const float* src = a.b_src;
          uint32_t bytes = 0;
          if (wb_col_ok && pix < a.Kg) {
            const int n = pix / pq, rem = pix - n * pq;
            const int p = rem / a.Q, q = rem - p * a.Q;
            const int h = p * a.stride - a.pad + wb_r, w = q * a.stride - a.pad + wb_s;
            if (h >= 0 && h < a.H && w >= 0 && w < a.W) {
              src = a.b_src + ((static_cast<long long>(n) * a.H + h) * a.W + w) * a.C + wb_ci;
              bytes = 16;
            }
          }
          put(sB + mnmaj_off(kr, col, BN), src, bytes);
        }
      }
      if constexpr (PRECISE) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        for (int i = 0; i < n_dst; ++i) {
          uint32_t v[4], lo[4];
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                       : "r"(my_dst[i]));
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t hi = v[j] & 0xFFFFE000u;  // exactly representable in tf32
            lo[j] = __float_as_uint(__uint_as_float(v[j]) - __uint_as_float(hi));
            v[j] = hi;
          }
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(my_dst[i]), "r"(v[0]),
                       "r"(v[1]), "r"(v[2]), "r"(v[3])
                       : "memory");
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(my_dst[i] + kLoDelta),
                       "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3])
                       : "memory");
        }
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive(&full[stage]);
      } else {
        ptx::cp_async_arrive_noinc(&full[stage]);
      }
    }

    // ============================ epilogue ============================
    if (nkb > 0) {
      ptx::mbar_wait(accum, 0);
      ptx::tc_fence_after();
      const int row = warp * 32 + lane;
      const int m = m0 + row;
      const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        ptx::tmem_ld32(trow + c0, v);
        if (m < a.M) {
          float* dst = (a.ws ? a.ws + static_cast<long long>(blockIdx.z) * a.M * a.Ng : a.out) +
                       static_cast<long long>(m) * a.Ng + n0 + c0;
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            if (n0 + c0 + 4 * g >= a.Ng) break;
            float4 o = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
            float4* d4 = reinterpret_cast<float4*>(dst + 4 * g);
            if (a.ws) {
              __stcg(d4, o);
            } else if (a.atomic) {
              atomicAdd(&d4->x, o.x);
              atomicAdd(&d4->y, o.y);
              atomicAdd(&d4->z, o.z);
              atomicAdd(&d4->w, o.w);
            } else {
              if (a.beta) {
                const float4 old = *d4;
                o.x += old.x;
                o.y += old.y;
                o.z += old.z;
                o.w += old.w;
              }
              *d4 = o;
            }
          }
        }
      }
    }
  } else if (lane == 0) {
    // ============================ MMA issuer ============================
    constexpr uint32_t idesc = ptx::idesc_tf32(kBM, BN, kAmn, kBmn);
    for (int it = 0; it < nkb; ++it) {
      const int stage = it % kStages;
      ptx::mbar_wait(&full[stage], (it / kStages) & 1);
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_after();
      const uint32_t sA = smem_base + stage * kStageBytes;
      const uint32_t sB = sA + kABytes;
#pragma unroll
      for (int ks = 0; ks < kBK / 8; ++ks) {
        // one tf32 MMA consumes K = 8 (32 bytes of a K-major row, or one
        // 8-row group of an MN-major tile)
        // K-major: K=8 is 32 bytes of the 128-byte swizzled row.
        // MN-major (BASE32B): K=8 is two 4-row groups -> advance 2 * SBO.
        const uint64_t ad =
            kAmn ? ptx::smem_desc(sA + ks * (a.mn_kstep ? a.mn_kstep : 2 * (kBM / 32) * 512), a.mn_lbo,
                                  a.mn_sbo ? a.mn_sbo : (kBM / 32) * 512, a.mn_layout)
                 : ptx::smem_desc(sA + ks * 32, 16, 1024, 2);
        const uint64_t bd =
            kBmn ? ptx::smem_desc(sB + ks * (a.mn_kstep ? a.mn_kstep : 2 * (BN / 32) * 512), a.mn_lbo,
                                  a.mn_sbo ? a.mn_sbo : (BN / 32) * 512, a.mn_layout)
                 : ptx::smem_desc(sB + ks * 32, 16, 1024, 2);
        ptx::mma_tf32(tmem, ad, bd, idesc, (it > 0 || ks > 0) ? 1u : 0u);
        if constexpr (PRECISE) {
          // lo operands live kLoDelta bytes above their hi tiles
          const uint64_t lo_step = static_cast<uint64_t>(kLoDelta >> 4);
          ptx::mma_tf32(tmem, ad, bd + lo_step, idesc, 1u);
          ptx::mma_tf32(tmem, ad + lo_step, bd, idesc, 1u);
        }
      }
      ptx::mma_commit(&empty[stage]);
    }
    if (nkb > 0) ptx::mma_commit(accum);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<BN>(tmem);
  }
}

template <int MODE, int BN, bool PRECISE>
int launch(const Args& a, int splits, cudaStream_t stream) {
  constexpr size_t kStageBytes = (kBM + BN) * kBK * 4 * (PRECISE ? 2 : 1);
  const size_t smem = kStages * kStageBytes + 1024 + 256;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(conv_igemm_kernel<MODE, BN, PRECISE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  dim3 grid((a.M + kBM - 1) / kBM, (a.Ng + BN - 1) / BN, splits);
  launch_pdl(conv_igemm_kernel<MODE, BN, PRECISE>, grid, kThreads, smem, stream, a);
  return static_cast<int>(cudaGetLastError());
}

int g_conv_math = 0;  // 0 = TF32, 1 = 3xTF32

Args make_args(const accudnn_conv_desc* d, int mode) {
  Args a{};
  a.N = d->n; a.H = d->h; a.W = d->w; a.C = d->c; a.K = d->k;
  a.R = d->r; a.S = d->s; a.stride = d->stride; a.pad = d->pad; a.P = d->p; a.Q = d->q;
  if (mode == FWD) {
    a.M = a.N * a.P * a.Q; a.Ng = a.K; a.Kg = a.R * a.S * a.C;
  } else if (mode == DGRAD) {
    a.M = a.N * a.H * a.W; a.Ng = a.C; a.Kg = a.R * a.S * a.K;
  } else {
    a.M = a.K; a.Ng = a.R * a.S * a.C; a.Kg = a.N * a.P * a.Q;
  }
  a.kb_total = (a.Kg + kBK - 1) / kBK;
  a.mn_lbo = 512;
  a.mn_sbo = 0;
  a.mn_layout = 1;
  a.mn_kstep = 0;
  if (const char* e = getenv("ACCUDNN_DBG_MN")) {  // debug: "lbo,sbo,layout,kstep"
    sscanf(e, "%d,%d,%d,%d", &a.mn_lbo, &a.mn_sbo, &a.mn_layout, &a.mn_kstep);
  }
  return a;
}

int valid_desc(const accudnn_conv_desc* d) {
  if (!d || d->n <= 0 || d->c <= 0 || d->k <= 0 || d->r <= 0 || d->s <= 0 || d->stride <= 0)
    return 0;
  if ((d->c & 3) || (d->k & 3)) return 0;  // 16-byte chunks along channels
  return 1;
}

template <int MODE>
int dispatch(Args a, int splits, cudaStream_t stream) {
  a.kb_per_split = (a.kb_total + splits - 1) / splits;
  splits = (a.kb_total + a.kb_per_split - 1) / a.kb_per_split;
  a.atomic = splits > 1 ? 1 : 0;
  a.ws = nullptr;
  if (splits > 1) {  // deterministic slice-order reduction when the workspace allows
    a.ws = conv_splitk_workspace(sizeof(float) * static_cast<size_t>(splits) * a.M * a.Ng);
    if (a.ws) {
      a.atomic = 0;
      int rc;
      if (g_conv_math == 1)
        rc = a.Ng <= 64 ? launch<MODE, 64, true>(a, splits, stream)
                        : launch<MODE, 128, true>(a, splits, stream);
      else
        rc = a.Ng <= 64 ? launch<MODE, 64, false>(a, splits, stream)
                        : launch<MODE, 128, false>(a, splits, stream);
      if (rc) return rc;
      return conv_splitk_reduce(a.ws, splits, a.M, a.Ng, a.out, a.beta, stream);
    }
  }
  if (g_conv_math == 1) {
    if (a.Ng <= 64) return launch<MODE, 64, true>(a, splits, stream);
    return launch<MODE, 128, true>(a, splits, stream);
  }
  if (a.Ng <= 64) return launch<MODE, 64, false>(a, splits, stream);
  return launch<MODE, 128, false>(a, splits, stream);
}

// split-K factor: fill ~2 CTAs per SM when the output tile grid is small
int pick_splits(const Args& a, int sms) {
  const int bn = a.Ng <= 64 ? 64 : 128;
  const long long tiles = static_cast<long long>((a.M + kBM - 1) / kBM) * ((a.Ng + bn - 1) / bn);
  const long long want = 2LL * sms;
  if (tiles >= want) return 1;
  long long s = (want + tiles - 1) / tiles;
  s = s < a.kb_total / 4 ? s : a.kb_total / 4;  // keep >= 4 k-blocks per split
  return s < 1 ? 1 : static_cast<int>(s);
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

// persistent TMA kernels (conv_sm100.cu); return 0 when a shape is not eligible
int conv_tma_fwd(const accudnn_conv_desc* d, const float* x, const float* w, float* y, int beta,
                 cudaStream_t st, int* rc, float* stats = nullptr);
int conv_tma_dgrad(const accudnn_conv_desc* d, const float* dy, const float* w, float* dx,
                   int beta, cudaStream_t st, int* rc);
int conv_tma_wgrad(const accudnn_conv_desc* d, const float* x, const float* dy, float* dw,
                   int beta, cudaStream_t st, int* rc);
int g_conv_impl = 1;  // 1 = TMA kernels where eligible, 0 = cp.async kernel only

// ---- 3xTF32 on the TMA kernels --------------------------------------------
// The tensor core reads an fp32 operand as tf32 (its top 19 bits), so with
// lo(v) = v - (v & 0xFFFFE000) materialised once per operand, three TF32
// GEMMs accumulated into the output give hi*hi + hi*lo + lo*hi (~fp32
// accuracy, as the cp.async PRECISE kernel computes per tile).  The lo copies
// live in a caller-provided scratch per stream (accudnn_conv_set_precise_scratch);
// without one the cp.async PRECISE kernel runs instead.
__global__ void __launch_bounds__(256) tf32_lo_kernel(const float4* __restrict__ x,
                                                      float4* __restrict__ lo, long long n4) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += gridDim.x * 256LL) {
    const float4 v = __ldg(x + i);
    float4 o;
    o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    lo[i] = o;
  }
}

struct Scratch {
  cudaStream_t st;
  char* ptr;
  size_t bytes;
};
std::vector<Scratch> g_scratch;

const Scratch* scratch_for(cudaStream_t st) {
  for (const Scratch& e : g_scratch)
    if (e.st == st) return &e;
  return nullptr;
}

size_t align256(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }

int split_lo(const float* x, float* lo, long long n, cudaStream_t st) {
  const long long n4 = n / 4;  // every conv operand has channels % 4 == 0
  const int grid = static_cast<int>(std::min<long long>((n4 + 255) / 256, 8LL * sm_count()));
  tf32_lo_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(x),
                                       reinterpret_cast<float4*>(lo), n4);
  return static_cast<int>(cudaGetLastError());
}

// term(a, b, beta): one TF32 TMA GEMM of the mode (0 when the shape is not
// TMA-eligible); out = a*b (+ old); returns 1 when handled, rc in *rc
template <typename Term>
int precise3(cudaStream_t st, const float* a, long long na, const float* b, long long nb,
             int beta, int* rc, Term term) {
  const Scratch* sc = scratch_for(st);
  const size_t need = align256(sizeof(float) * na) + align256(sizeof(float) * nb);
  if (!sc || sc->bytes < need) return 0;
  float* a_lo = reinterpret_cast<float*>(sc->ptr);
  float* b_lo = reinterpret_cast<float*>(sc->ptr + align256(sizeof(float) * na));
  if (!term(a, b, beta, rc)) return 0;  // hi * hi (not eligible: nothing written)
  if (*rc) return 1;
  if ((*rc = split_lo(a, a_lo, na, st)) != 0) return 1;
  if ((*rc = split_lo(b, b_lo, nb, st)) != 0) return 1;
  term(a, b_lo, 1, rc);  // + hi * lo
  if (*rc) return 1;
  term(a_lo, b, 1, rc);  // + lo * hi
  return 1;
}
}  // namespace accudnn

using namespace accudnn;

extern "C" int accudnn_conv_fwd(const accudnn_conv_desc* d, const float* x, const float* w,
                                float* y, int beta, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  conv_select_workspace(stream);
  if (!valid_desc(d)) return static_cast<int>(cudaErrorInvalidValue);
  int rc = 0;
  if (g_conv_impl == 1 && g_conv_math == 0 && conv_tma_fwd(d, x, w, y, beta, stream, &rc))
    return rc;
  if (g_conv_impl == 1 && g_conv_math == 1 &&
      precise3(stream, x, 1LL * d->n * d->h * d->w * d->c, w, 1LL * d->k * d->r * d->s * d->c, beta,
               &rc, [&](const float* xa, const float* wb, int bt, int* r) {
                 return conv_tma_fwd(d, xa, wb, y, bt, stream, r);
               }))
    return rc;
  Args a = make_args(d, FWD);
  a.a_src = x; a.b_src = w; a.out = y; a.beta = beta;
  return dispatch<FWD>(a, 1, stream);
}

// forward that also writes the output's per-32-row column sums / sums of
// squares ([2][ceil(M/32)][K] floats) for the following batch norm; *produced
// = 0 when the shape runs on the cp.async kernel (no statistics written)
extern "C" int accudnn_conv_fwd_stats(const accudnn_conv_desc* d, const float* x, const float* w,
                                      float* y, float* stats, int* produced, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  conv_select_workspace(stream);
  *produced = 0;
  if (!valid_desc(d)) return static_cast<int>(cudaErrorInvalidValue);
  int rc = 0;
  if (g_conv_impl == 1 && g_conv_math == 0 && conv_tma_fwd(d, x, w, y, 0, stream, &rc, stats)) {
    *produced = (rc == 0 && d->k % 32 == 0) ? 1 : 0;  // conv_tma_fwd writes stats iff k % 32 == 0
    return rc;
  }
  return accudnn_conv_fwd(d, x, w, y, 0, stream_);
}

extern "C" int accudnn_conv_dgrad(const accudnn_conv_desc* d, const float* dy, const float* w,
                                  float* dx, int beta, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  conv_select_workspace(stream);
  if (!valid_desc(d)) return static_cast<int>(cudaErrorInvalidValue);
  int rc = 0;
  if (g_conv_impl == 1 && g_conv_math == 0 && conv_tma_dgrad(d, dy, w, dx, beta, stream, &rc))
    return rc;
  if (g_conv_impl == 1 && g_conv_math == 1 &&
      precise3(stream, dy, 1LL * d->n * d->p * d->q * d->k, w, 1LL * d->k * d->r * d->s * d->c, beta,
               &rc, [&](const float* ya, const float* wb, int bt, int* r) {
                 return conv_tma_dgrad(d, ya, wb, dx, bt, stream, r);
               }))
    return rc;
  Args a = make_args(d, DGRAD);
  a.a_src = dy; a.b_src = w; a.out = dx; a.beta = beta;
  return dispatch<DGRAD>(a, 1, stream);
}

extern "C" int accudnn_conv_wgrad(const accudnn_conv_desc* d, const float* x, const float* dy,
                                  float* dw, int beta, int splits, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  conv_select_workspace(stream);
  if (!valid_desc(d)) return static_cast<int>(cudaErrorInvalidValue);
  int rc = 0;
  if (g_conv_impl == 1 && g_conv_math == 0 && splits <= 0 &&
      conv_tma_wgrad(d, x, dy, dw, beta, stream, &rc))
    return rc;
  if (g_conv_impl == 1 && g_conv_math == 1 && splits <= 0 &&
      precise3(stream, x, 1LL * d->n * d->h * d->w * d->c, dy, 1LL * d->n * d->p * d->q * d->k, beta,
               &rc, [&](const float* xa, const float* yb, int bt, int* r) {
                 return conv_tma_wgrad(d, xa, yb, dw, bt, stream, r);
               }))
    return rc;
  Args a = make_args(d, WGRAD);
  a.a_src = dy; a.b_src = x; a.out = dw; a.beta = beta;
  if (splits <= 0) splits = pick_splits(a, sm_count());
  if (splits > 1 && !beta &&
      !conv_splitk_workspace(sizeof(float) * static_cast<size_t>(splits) * a.M * a.Ng)) {
    const cudaError_t e = cudaMemsetAsync(dw, 0, sizeof(float) * static_cast<size_t>(a.M) * a.Ng,
                                          stream);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return dispatch<WGRAD>(a, splits, stream);
}

extern "C" int accudnn_conv_set_precise_scratch(void* stream, void* ptr, unsigned long long bytes) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (size_t i = 0; i < accudnn::g_scratch.size(); ++i)
    if (accudnn::g_scratch[i].st == st) {
      accudnn::g_scratch.erase(accudnn::g_scratch.begin() + static_cast<long>(i));
      break;
    }
  if (ptr && bytes)
    accudnn::g_scratch.push_back({st, static_cast<char*>(ptr), static_cast<size_t>(bytes)});
  return 0;
}

extern "C" unsigned long long accudnn_conv_precise_scratch_bytes(const accudnn_conv_desc* d) {
  using accudnn::align256;
  if (!d) return 0;
  const size_t x = align256(sizeof(float) * d->n * d->h * d->w * d->c);
  const size_t y = align256(sizeof(float) * d->n * d->p * d->q * d->k);
  const size_t w = align256(sizeof(float) * d->k * d->r * d->s * d->c);
  return std::max({x + w, y + w, x + y});
}

extern "C" int accudnn_set_conv_math(int mode) {
  if (mode != 0 && mode != 1) return static_cast<int>(cudaErrorInvalidValue);
  accudnn::g_conv_math = mode;
  return 0;
}
extern "C" int accudnn_get_conv_math(void) { return accudnn::g_conv_math; }

extern "C" int accudnn_set_conv_impl(int impl) {
  if (impl != 0 && impl != 1) return static_cast<int>(cudaErrorInvalidValue);
  accudnn::g_conv_impl = impl;
  return 0;
}
