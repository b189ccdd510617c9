// Persistent TMA + tcgen05 implicit-GEMM convolution (sm_100a), v3.
//
// The three GEMMs of a convolution's training step on NHWC fp32 tensors with
// TF32 tensor-core math and FP32 accumulation in TMEM:
//
//   FWD    y [m=(n,p,q)][co]   = sum_{(r,s,ci)} im2col(x) * w[co][(r,s,ci)]
//          A: im2col TMA over x {C,W,H,N} (taps = im2col offsets), or a 2-D
//             tile for 1x1/stride-1; B: 2-D tile of w [Cout][R*S*Cin] (K-major)
//   DGRAD  dx[(n,h,w)][ci]     = sum_{(r,s,co)} dy(n,p,q)[co] * w[co][r][s][ci]
//          solved per output parity class (h % stride, w % stride): each class
//          is a stride-1 correlation of dy with the taps r = (h+pad) mod stride
//          (+ stride*t), i.e. an im2col TMA over dy with a (Rc x Sc) filter and
//          lower corner delta_min, whose rows scatter to (n, stride*i+a,
//          stride*j+b).  stride 1 = one class with the flipped R x S filter.
//          B: 3-D tile of w {Cin, R*S, Cout} -> MN-major (ci contiguous)
//   WGRAD  dw[co][(r,s,ci)]    = sum_{m=(n,p,q)} dy[m][co] * im2col(x)[m][(r,s,ci)]
//          A: 2-D MN-major tiles of dy [pixels][Cout]; B: im2col TMA of x with
//          32 output pixels per column (MN-major)
//
// Kernel structure (192 threads, one CTA per SM, persistent):
//   warp 0     TMA producer (one elected thread) over a STAGES-deep smem ring
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5  epilogue: TMEM -> registers -> HBM
// The CTA walks work units u = blockIdx.x + i*gridDim.x; a unit is one
// 128 x BN output tile and one K-slice of it.  The accumulator is double
// buffered in TMEM (2 x BN columns), so the epilogue of unit i overlaps the
// main loop of unit i+1.
//
// Split-K is deterministic: every K-slice writes its partial tile to its own
// workspace slice and a grid-wide reduce kernel sums the slices in slice
// order 0..S-1 (coalesced, all SMs).  No atomics anywhere: the same inputs
// give bit-identical outputs in every executor mode (resident / naive /
// dynamic swap) and every run.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "accudnn_kernels.h"
#include "sm100_ptx.cuh"

namespace accudnn {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 32;
constexpr int kThreads = 192;
constexpr int kEpiThreads = 128;

enum Mode : int { FWD = 0, DGRAD = 1, WGRAD = 2 };

struct Prob {
  // convolution geometry (original layer)
  int N, H, W, C, K, R, S, stride, pad, P, Q;
  // GEMM
  int M, Ng, kb_total;
  int tiles_m, tiles_n, splits, kb_per_split, units;
  int a_tiled;  // A is a plain 2-D tile (FWD: 1x1 s1 p0; DGRAD: class with one centred tap)
  // DGRAD parity class
  int cls_a, cls_b;    // output row / column parity
  int Hc, Wc;          // class output grid
  int Rc, Sc;          // class filter (im2col taps)
  int lo_h, lo_w;      // im2col lower corner (dy offsets of tap 0)
  int r0, s0;          // original tap of im2col tap (tr, ts) = (r0 - stride*tr, s0 - stride*ts)
  int scatter;         // rows scatter to (n, stride*i + a, stride*j + b)
  // output
  float* out;
  int beta;
  float* ws;           // split-K partials [split][M][Ng]
};

// ---- TMA PTX -------------------------------------------------------------------
__device__ __forceinline__ void tma_2d(const CUtensorMap* tm, uint32_t dst, uint64_t* bar, int c0,
                                       int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d(const CUtensorMap* tm, uint32_t dst, uint64_t* bar, int c0,
                                       int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_im2col(const CUtensorMap* tm, uint32_t dst, uint64_t* bar,
                                           int c, int w, int h, int n, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(ptx::smem_u32(bar)), "r"(c), "r"(w), "r"(h),
      "r"(n), "h"(ow), "h"(oh)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ptx::smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// global output row offset (floats) of GEMM row m
__device__ __forceinline__ long long out_row(const Prob& a, int m) {
  if (!a.scatter) return static_cast<long long>(m) * a.Ng;
  const int hw = a.Hc * a.Wc;
  const int n = m / hw;
  const int rem = m - n * hw;
  const int i = rem / a.Wc;
  const int j = rem - i * a.Wc;
  const int h = a.stride * i + a.cls_a;
  const int w = a.stride * j + a.cls_b;
  return ((static_cast<long long>(n) * a.H + h) * a.W + w) * a.C;
}

template <int MODE, int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    conv_sm100_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, const Prob a) {
  constexpr bool kAmn = (MODE == WGRAD);
  constexpr bool kBmn = (MODE != FWD);
  constexpr uint32_t kABytes = kBM * kBK * 4;
  constexpr uint32_t kBBytes = BN * kBK * 4;
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;      // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], kEpiThreads);
    }
    ptx::fence_mbar_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 1) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t smem_base = ptx::smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {
      // ============================ TMA producer ============================
      uint32_t kc = 0;  // k-blocks issued by this CTA (ring position)
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        const int split = u % a.splits;
        const int tile = u / a.splits;
        const int tm = tile % a.tiles_m;
        const int tn = tile / a.tiles_m;
        const int m0 = tm * kBM, n0 = tn * BN;
        const int kb0 = split * a.kb_per_split;
        const int kb1 = min(a.kb_total, kb0 + a.kb_per_split);
        // first output pixel of the tile (FWD: (n,p,q); DGRAD: (n,i,j) of the class grid)
        int pn = 0, pi = 0, pj = 0;
        if constexpr (MODE != WGRAD) {
          const int hh = (MODE == FWD) ? a.P : a.Hc;
          const int ww = (MODE == FWD) ? a.Q : a.Wc;
          pn = m0 / (hh * ww);
          const int rem = m0 - pn * hh * ww;
          pi = rem / ww;
          pj = rem - pi * ww;
        }
        int wt_r = 0, wt_s = 0, wt_c = 0;  // WGRAD: fixed tap / channel block of the N-tile
        if constexpr (MODE == WGRAD) {
          const int tap = n0 / a.C;
          wt_c = n0 - tap * a.C;
          wt_r = tap / a.S;
          wt_s = tap - wt_r * a.S;
        }
        for (int kb = kb0; kb < kb1; ++kb, ++kc) {
          const uint32_t stage = kc % STAGES;
          if (kc >= STAGES) ptx::mbar_wait(&empty[stage], ((kc / STAGES) - 1) & 1);
          const uint32_t sA = smem_base + stage * kStageBytes;
          const uint32_t sB = sA + kABytes;
          uint64_t* bar = &full[stage];
          mbar_expect_tx(bar, kStageBytes);
          const int kk = kb * kBK;
          if constexpr (MODE == FWD) {
            if (a.a_tiled) {
              tma_2d(&tmA, sA, bar, kk, m0);
            } else {
              const int tap = kk / a.C, c0 = kk - tap * a.C;
              const int r = tap / a.S, s = tap - r * a.S;
              tma_im2col(&tmA, sA, bar, c0, pj * a.stride - a.pad, pi * a.stride - a.pad, pn,
                         static_cast<uint16_t>(s), static_cast<uint16_t>(r));
            }
            tma_2d(&tmB, sB, bar, kk, n0);
          } else if constexpr (MODE == DGRAD) {
            const int t = kk / a.K, co0 = kk - t * a.K;
            const int tr = t / a.Sc, ts = t - tr * a.Sc;
            const int tap = (a.r0 - a.stride * tr) * a.S + (a.s0 - a.stride * ts);
            if (a.a_tiled) {
              tma_2d(&tmA, sA, bar, co0, m0);
            } else {
              tma_im2col(&tmA, sA, bar, co0, pj + a.lo_w, pi + a.lo_h, pn,
                         static_cast<uint16_t>(ts), static_cast<uint16_t>(tr));
            }
#pragma unroll
            for (int b = 0; b < BN / 32; ++b)
              tma_3d(&tmB, sB + b * 4096, bar, n0 + 32 * b, tap, co0);
          } else {
#pragma unroll
            for (int b = 0; b < kBM / 32; ++b) tma_2d(&tmA, sA + b * 4096, bar, m0 + 32 * b, kk);
            const int pq = a.P * a.Q;
            const int n = kk / pq, rem = kk - n * pq;
            const int p = rem / a.Q, q = rem - p * a.Q;
#pragma unroll
            for (int b = 0; b < BN / 32; ++b)
              tma_im2col(&tmB, sB + b * 4096, bar, wt_c + 32 * b, q * a.stride - a.pad,
                         p * a.stride - a.pad, n, static_cast<uint16_t>(wt_s),
                         static_cast<uint16_t>(wt_r));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ============================ MMA issuer ============================
      constexpr uint32_t idesc = ptx::idesc_tf32(kBM, BN, kAmn, kBmn);
      uint32_t kc = 0;
      int j = 0;  // units processed by this CTA
      for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++j) {
        const int split = u % a.splits;
        const int kb0 = split * a.kb_per_split;
        const int kb1 = min(a.kb_total, kb0 + a.kb_per_split);
        const int acc = j & 1;
        if (j >= 2) ptx::mbar_wait(&tempty[acc], ((j >> 1) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem + static_cast<uint32_t>(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++kc) {
          const uint32_t stage = kc % STAGES;
          ptx::mbar_wait(&full[stage], (kc / STAGES) & 1);
          ptx::tc_fence_after();
          const uint32_t sA = smem_base + stage * kStageBytes;
          const uint32_t sB = sA + kABytes;
#pragma unroll
          for (int ks = 0; ks < kBK / 8; ++ks) {
            const uint64_t ad = kAmn ? ptx::smem_desc(sA + ks * 1024, 4096, 512, 1)
                                     : ptx::smem_desc(sA + ks * 32, 16, 1024, 2);
            const uint64_t bd = kBmn ? ptx::smem_desc(sB + ks * 1024, 4096, 512, 1)
                                     : ptx::smem_desc(sB + ks * 32, 16, 1024, 2);
            ptx::mma_tf32(d_tmem, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&empty[stage]);
        }
        ptx::mma_commit(&tfull[acc]);
      }
    }
  } else {
    // ============================ epilogue ============================
    // Each warp drains its TMEM lane quadrant (32 rows) in 32-column chunks:
    // tcgen05.ld -> registers -> a private 4 KB smem transpose buffer (16-byte
    // granules XOR-swizzled by row) -> coalesced 128-byte row segments to HBM
    // (4 rows per instruction).  With split-K the chunk goes to the slice's
    // workspace rows instead; conv_splitk_reduce_kernel sums the slices.
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int ew = warp - 2;    // staging buffer of this warp
    float* stage_buf = reinterpret_cast<float*>(smem + STAGES * kStageBytes + 1024) + ew * 1024;
    const uint32_t sbuf = ptx::smem_u32(stage_buf);
    const int rr_lo = lane >> 3;  // read-back row within a group of 4
    const int gg = lane & 7;      // read-back 16-byte granule
    int j = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++j) {
      const int split = u % a.splits;
      const int tile = u / a.splits;
      const int tm = tile % a.tiles_m;
      const int tn = tile / a.tiles_m;
      const int m0 = tm * kBM + quad * 32, n0 = tn * BN;
      const int acc = j & 1;
      ptx::mbar_wait(&tfull[acc], (j >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t trow = tmem + static_cast<uint32_t>(acc * BN) +
                            (static_cast<uint32_t>(quad * 32) << 16);
      const int ncols = min(BN, a.Ng - n0);  // multiple of 4
      const bool partial = a.splits > 1;
      // destination row offsets of the 4 x 8 rows this lane writes
      long long drow[8];
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int m = m0 + it * 4 + rr_lo;
        drow[it] = m < a.M ? (partial ? (static_cast<long long>(split) * a.M + m) * a.Ng
                                      : out_row(a, m))
                           : -1;
      }
      float* base = partial ? a.ws : a.out;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        ptx::tmem_ld32(trow + c0, v);
        if (c0 + 32 >= BN) {  // accumulator drained: release it to the MMA warp
          ptx::tc_fence_before();
          ptx::mbar_arrive(&tempty[acc]);
        }
        if (c0 >= ncols) continue;
#pragma unroll
        for (int g = 0; g < 8; ++g)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                           sbuf + lane * 128 + ((g ^ (lane & 7)) << 4)),
                       "f"(v[4 * g]), "f"(v[4 * g + 1]), "f"(v[4 * g + 2]), "f"(v[4 * g + 3])
                       : "memory");
        __syncwarp();
        const int col = n0 + c0 + gg * 4;
        const bool col_ok = c0 + gg * 4 < ncols;
        float4 o[8];
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + rr_lo;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(o[it].x), "=f"(o[it].y), "=f"(o[it].z), "=f"(o[it].w)
                       : "r"(sbuf + rr * 128 + ((gg ^ (rr & 7)) << 4)));
        }
        __syncwarp();
        if (a.beta && !partial) {
          float4 old[8];
#pragma unroll
          for (int it = 0; it < 8; ++it)
            old[it] = (col_ok && drow[it] >= 0)
                          ? *reinterpret_cast<const float4*>(base + drow[it] + col)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            o[it].x += old[it].x;
            o[it].y += old[it].y;
            o[it].z += old[it].z;
            o[it].w += old[it].w;
          }
        }
#pragma unroll
        for (int it = 0; it < 8; ++it)
          if (col_ok && drow[it] >= 0) {
            if (partial)
              __stcg(reinterpret_cast<float4*>(base + drow[it] + col), o[it]);
            else
              *reinterpret_cast<float4*>(base + drow[it] + col) = o[it];
          }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem);
  }
}

// Deterministic split-K reduction: out[map(m)][n] (+)= sum_{s=0..S-1} ws[s][m][n],
// slices always summed in slice order.  One float4 per thread-iteration,
// grid-stride over the M x Ng/4 output vectors (coalesced rows).
__global__ void __launch_bounds__(256) conv_splitk_reduce_kernel(const Prob a) {
  const int ng4 = a.Ng >> 2;
  const long long total = static_cast<long long>(a.M) * ng4;
  const long long slice = static_cast<long long>(a.M) * a.Ng;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * 256) {
    const int m = static_cast<int>(i / ng4);
    const int c = static_cast<int>(i - static_cast<long long>(m) * ng4) * 4;
    const float* src = a.ws + static_cast<long long>(m) * a.Ng + c;
    float4 o = __ldcg(reinterpret_cast<const float4*>(src));
    for (int s = 1; s < a.splits; ++s) {
      const float4 p = __ldcg(reinterpret_cast<const float4*>(src + s * slice));
      o.x += p.x;
      o.y += p.y;
      o.z += p.z;
      o.w += p.w;
    }
    float4* d = reinterpret_cast<float4*>(a.out + out_row(a, m) + c);
    if (a.beta) {
      const float4 old = *d;
      o.x += old.x;
      o.y += old.y;
      o.z += old.z;
      o.w += old.w;
    }
    *d = o;
  }
}

// ---- host: tensor maps --------------------------------------------------------------
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using EncodeIm2col = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                  cuuint32_t, cuuint32_t, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled enc_tiled() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}
EncodeIm2col enc_im2col() {
  static EncodeIm2col fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q);
    fn = reinterpret_cast<EncodeIm2col>(p);
  }
  return fn;
}

bool tiled_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims,
               const cuuint64_t* strides_bytes, const cuuint32_t* box, CUtensorMapSwizzle sw) {
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  EncodeTiled f = enc_tiled();
  if (!f) return false;
  return f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, static_cast<cuuint32_t>(rank),
           const_cast<void*>(base), dims, strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC tensor {C, W, H, N}; the im2col walk covers dim - lower + upper
// positions per spatial dim (with traversal stride `stride`), `pixels` rows
// per column, 32 channels per pixel
bool im2col_map(CUtensorMap* m, const void* base, int n, int h, int w, int c, int lo_h, int lo_w,
                int up_h, int up_w, int stride, int pixels, CUtensorMapSwizzle sw) {
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w),
                              static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 4,
                                 static_cast<cuuint64_t>(c) * w * 4,
                                 static_cast<cuuint64_t>(c) * w * h * 4};
  const int lo[2] = {lo_w, lo_h};
  const int hi[2] = {up_w, up_h};
  const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
  EncodeIm2col f = enc_im2col();
  if (!f) return false;
  return f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, lo, hi,
           32, static_cast<cuuint32_t>(pixels), es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int g_sms = 0;
int sm_count() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

// ---- split-K workspace ------------------------------------------------------------
struct Workspace {
  float* ws = nullptr;
  size_t bytes = 0;
  bool owned = false;
};
Workspace g_ws;
size_t g_ws_default = 64ull << 20;

// lazily owned workspace when the caller did not provide one
size_t ws_capacity() {
  if (!g_ws.ws && !g_ws.bytes && g_ws_default) {
    if (cudaMalloc(&g_ws.ws, g_ws_default) == cudaSuccess) {
      g_ws.bytes = g_ws_default;
      g_ws.owned = true;
    } else {
      cudaGetLastError();
      g_ws.ws = nullptr;
    }
  }
  return g_ws.ws ? g_ws.bytes : 0;
}

// Split-K factor from a makespan model in SM cycles: a persistent CTA pays
// a prologue, then waves of units (k-blocks of 2*BN + 128 cycles each plus a
// per-unit hand-off), then the last epilogue; S > 1 adds the reduce kernel
// (launch + (S + 1 + beta) * M * Ng * 4 bytes at ~2 KB/cycle chip-wide).
int choose_splits(long long tiles, int kb_total, int bn, long long out_elems, int beta,
                  size_t ws_bytes) {
  const long long sms = sm_count();
  int best = 1;
  double best_cost = 1e30;
  const int max_s = std::max(1, std::min(kb_total, 128));
  for (int s = 1; s <= max_s; ++s) {
    if (s > 1 && static_cast<size_t>(s) * out_elems * 4 > ws_bytes) break;
    const int per = (kb_total + s - 1) / s;
    if ((kb_total + per - 1) / per != s) continue;
    const long long units = tiles * s;
    const long long waves = (units + sms - 1) / sms;
    double cost = 3000.0 + static_cast<double>(waves) * (per * (2.0 * bn + 128.0) + 300.0) +
                  4.0 * bn * 2;
    if (s > 1) cost += 2500.0 + (s + 1.0 + beta) * out_elems * 4.0 / 2000.0;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

template <int MODE, int BN, int STAGES>
int launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const Prob& a, cudaStream_t st) {
  constexpr size_t smem = STAGES * (kBM + BN) * kBK * 4 + 1024 + 1024 + 4 * 4096;
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(conv_sm100_kernel<MODE, BN, STAGES>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    configured = true;
  }
  const int grid = static_cast<int>(std::min<long long>(a.units, sm_count()));
  conv_sm100_kernel<MODE, BN, STAGES><<<grid, kThreads, smem, st>>>(ta, tb, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || a.splits == 1) return static_cast<int>(e);
  const long long vec = static_cast<long long>(a.M) * (a.Ng / 4);
  const int rgrid = static_cast<int>(std::min<long long>((vec + 255) / 256, 8LL * sm_count()));
  conv_splitk_reduce_kernel<<<rgrid, 256, 0, st>>>(a);
  return static_cast<int>(cudaGetLastError());
}

template <int MODE, int BN>
int run(const CUtensorMap& ta, const CUtensorMap& tb, Prob a, cudaStream_t st) {
  a.tiles_m = (a.M + kBM - 1) / kBM;
  a.tiles_n = (a.Ng + BN - 1) / BN;
  const long long tiles = static_cast<long long>(a.tiles_m) * a.tiles_n;
  a.splits = choose_splits(tiles, a.kb_total, BN, static_cast<long long>(a.M) * a.Ng, a.beta,
                           ws_capacity());
  a.kb_per_split = (a.kb_total + a.splits - 1) / a.splits;
  a.units = static_cast<int>(tiles * a.splits);
  a.ws = g_ws.ws;
  constexpr int kStages = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
  return launch_t<MODE, BN, kStages>(ta, tb, a, st);
}

Prob base_prob(const accudnn_conv_desc* d) {
  Prob a{};
  a.N = d->n; a.H = d->h; a.W = d->w; a.C = d->c; a.K = d->k;
  a.R = d->r; a.S = d->s; a.stride = d->stride; a.pad = d->pad; a.P = d->p; a.Q = d->q;
  return a;
}

bool geometry_ok(const accudnn_conv_desc* d) {
  return d->r == d->s && d->pad <= 64 && d->r <= 16 && d->stride <= 8 &&
         d->p == (d->h + 2 * d->pad - d->r) / d->stride + 1 &&
         d->q == (d->w + 2 * d->pad - d->s) / d->stride + 1;
}

// one spatial dimension of a DGRAD parity class (see the file comment)
struct ClassDim {
  int taps = 0;     // Rc
  int t0 = 0;       // original tap of im2col tap 0 (r_max)
  int lower = 0;    // delta_min
  int out = 0;      // Hc
};
ClassDim class_dim(int a, int stride, int pad, int R, int H, int P) {
  ClassDim c;
  c.out = (H - a + stride - 1) / stride;
  const int r_min = (a + pad) % stride;
  if (r_min >= R || c.out <= 0) return c;
  c.taps = (R - 1 - r_min) / stride + 1;
  c.t0 = r_min + (c.taps - 1) * stride;
  c.lower = (a + pad - c.t0) / stride;
  return c;
}

}  // namespace

// 0 = not eligible (caller falls back to the cp.async kernel), else launched
int conv_tma_fwd(const accudnn_conv_desc* d, const float* x, const float* w, float* y, int beta,
                 cudaStream_t st, int* rc) {
  if (!geometry_ok(d) || (d->c % 32) || (d->k % 4)) return 0;
  Prob a = base_prob(d);
  a.M = a.N * a.P * a.Q;
  a.Ng = a.K;
  const int Kg = a.R * a.S * a.C;
  a.kb_total = Kg / kBK;
  a.out = y;
  a.beta = beta;
  a.a_tiled = (a.R == 1 && a.stride == 1 && a.pad == 0);
  const int BN = a.K >= 256 ? 256 : (a.K > 64 ? 128 : 64);
  CUtensorMap ta, tb;
  bool ok;
  if (a.a_tiled) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.C), static_cast<cuuint64_t>(a.M)};
    const cuuint64_t str[1] = {static_cast<cuuint64_t>(a.C) * 4};
    const cuuint32_t box[2] = {32, kBM};
    ok = tiled_map(&ta, x, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  } else {
    const int lo = -a.pad, up = a.pad - (a.R - 1);
    ok = im2col_map(&ta, x, a.N, a.H, a.W, a.C, lo, lo, up, up, a.stride, kBM,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  }
  const cuuint64_t bd[2] = {static_cast<cuuint64_t>(Kg), static_cast<cuuint64_t>(a.K)};
  const cuuint64_t bs[1] = {static_cast<cuuint64_t>(Kg) * 4};
  const cuuint32_t bbox[2] = {32, static_cast<cuuint32_t>(BN)};
  ok = ok && tiled_map(&tb, w, 2, bd, bs, bbox, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!ok) return 0;
  *rc = BN == 256 ? run<FWD, 256>(ta, tb, a, st)
                  : (BN == 128 ? run<FWD, 128>(ta, tb, a, st) : run<FWD, 64>(ta, tb, a, st));
  return 1;
}

int conv_tma_dgrad(const accudnn_conv_desc* d, const float* dy, const float* w, float* dx,
                   int beta, cudaStream_t st, int* rc) {
  if (!geometry_ok(d) || (d->c % 32) || (d->k % 32)) return 0;
  const int s = d->stride;
  // every parity class must be expressible; classes without taps receive no
  // contribution (zero, or untouched when accumulating)
  ClassDim rows[8], cols[8];
  bool any_empty = false;
  for (int c = 0; c < s; ++c) {
    rows[c] = class_dim(c, s, d->pad, d->r, d->h, d->p);
    cols[c] = class_dim(c, s, d->pad, d->s, d->w, d->q);
    if (rows[c].out <= 0 || cols[c].out <= 0) return 0;
    if (rows[c].taps == 0 || cols[c].taps == 0) any_empty = true;
    if (rows[c].lower < -64 || cols[c].lower < -64 || rows[c].lower > 64 || cols[c].lower > 64)
      return 0;
  }
  const int BN = d->c >= 256 ? 256 : (d->c > 64 ? 128 : 64);
  if (d->c % BN && BN != 64) return 0;
  *rc = 0;
  if (any_empty && !beta) {
    const cudaError_t e = cudaMemsetAsync(
        dx, 0, sizeof(float) * static_cast<size_t>(d->n) * d->h * d->w * d->c, st);
    if (e != cudaSuccess) {
      *rc = static_cast<int>(e);
      return 1;
    }
    beta = 1;
  }
  for (int ca = 0; ca < s; ++ca) {
    for (int cb = 0; cb < s; ++cb) {
      const ClassDim& cr = rows[ca];
      const ClassDim& cc = cols[cb];
      if (cr.taps == 0 || cc.taps == 0) continue;
      Prob a = base_prob(d);
      a.cls_a = ca;
      a.cls_b = cb;
      a.Hc = cr.out;
      a.Wc = cc.out;
      a.Rc = cr.taps;
      a.Sc = cc.taps;
      a.lo_h = cr.lower;
      a.lo_w = cc.lower;
      a.r0 = cr.t0;
      a.s0 = cc.t0;
      a.scatter = s > 1;
      a.M = a.N * a.Hc * a.Wc;
      a.Ng = a.C;
      a.kb_total = a.Rc * a.Sc * a.K / kBK;
      a.out = dx;
      a.beta = beta;
      a.a_tiled = (a.Rc == 1 && a.Sc == 1 && a.lo_h == 0 && a.lo_w == 0 && a.Hc == a.P &&
                   a.Wc == a.Q);
      CUtensorMap ta, tb;
      bool ok;
      if (a.a_tiled) {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.K),
                                    static_cast<cuuint64_t>(a.N) * a.P * a.Q};
        const cuuint64_t str[1] = {static_cast<cuuint64_t>(a.K) * 4};
        const cuuint32_t box[2] = {32, kBM};
        ok = tiled_map(&ta, dy, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
      } else {
        ok = im2col_map(&ta, dy, a.N, a.P, a.Q, a.K, a.lo_h, a.lo_w, a.Hc - a.P + a.lo_h,
                        a.Wc - a.Q + a.lo_w, 1, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
      }
      const cuuint64_t bd[3] = {static_cast<cuuint64_t>(a.C), static_cast<cuuint64_t>(a.R) * a.S,
                                static_cast<cuuint64_t>(a.K)};
      const cuuint64_t bs[2] = {static_cast<cuuint64_t>(a.C) * 4,
                                static_cast<cuuint64_t>(a.C) * a.R * a.S * 4};
      const cuuint32_t bbox[3] = {32, 1, 32};
      ok = ok && tiled_map(&tb, w, 3, bd, bs, bbox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
      if (!ok) return *rc ? 1 : 0;  // nothing launched yet on the first class
      *rc = BN == 256 ? run<DGRAD, 256>(ta, tb, a, st)
                      : (BN == 128 ? run<DGRAD, 128>(ta, tb, a, st)
                                   : run<DGRAD, 64>(ta, tb, a, st));
      if (*rc) return 1;
    }
  }
  return 1;
}

int conv_tma_wgrad(const accudnn_conv_desc* d, const float* x, const float* dy, float* dw,
                   int beta, cudaStream_t st, int* rc) {
  if (!geometry_ok(d) || (d->c % 32) || (d->k % 4)) return 0;
  Prob a = base_prob(d);
  a.M = a.K;
  a.Ng = a.R * a.S * a.C;
  const int Kg = a.N * a.P * a.Q;
  // a ragged last K-block reads past the last output pixel: the im2col walk
  // and the dy tile land out of bounds there and are zero-filled by the TMA
  a.kb_total = (Kg + kBK - 1) / kBK;
  a.out = dw;
  a.beta = beta;
  const int BN = (a.C % 256 == 0) ? 256 : (a.C % 128 == 0) ? 128 : (a.C % 64 == 0 ? 64 : 0);
  if (!BN) return 0;
  CUtensorMap ta, tb;
  const cuuint64_t ad[2] = {static_cast<cuuint64_t>(a.K), static_cast<cuuint64_t>(Kg)};
  const cuuint64_t as[1] = {static_cast<cuuint64_t>(a.K) * 4};
  const cuuint32_t abox[2] = {32, 32};
  bool ok = tiled_map(&ta, dy, 2, ad, as, abox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  const int lo = -a.pad, up = a.pad - (a.R - 1);
  ok = ok && im2col_map(&tb, x, a.N, a.H, a.W, a.C, lo, lo, up, up, a.stride, 32,
                        CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!ok) return 0;
  *rc = BN == 256 ? run<WGRAD, 256>(ta, tb, a, st)
                  : (BN == 128 ? run<WGRAD, 128>(ta, tb, a, st) : run<WGRAD, 64>(ta, tb, a, st));
  return 1;
}

// shared with the cp.async kernel (conv_igemm.cu): the split-K workspace if
// it holds `bytes`, else nullptr; and the slice-order reduction on it
float* conv_splitk_workspace(size_t bytes) {
  return ws_capacity() >= bytes ? g_ws.ws : nullptr;
}
int conv_splitk_reduce(float* ws, int splits, int M, int Ng, float* out, int beta,
                       cudaStream_t st) {
  Prob a{};
  a.ws = ws;
  a.splits = splits;
  a.M = M;
  a.Ng = Ng;
  a.out = out;
  a.beta = beta;
  const long long vec = static_cast<long long>(M) * (Ng / 4);
  const int rgrid = static_cast<int>(std::min<long long>((vec + 255) / 256, 8LL * sm_count()));
  conv_splitk_reduce_kernel<<<rgrid, 256, 0, st>>>(a);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace accudnn

// caller-provided split-K workspace (e.g. carved out of an executor's fixed
// allocation so it counts against the device budget).  ptr == NULL:
// bytes > 0 restores a lazily allocated default of that size, bytes == 0
// disables split-K.
extern "C" int accudnn_conv_set_workspace(void* ptr, unsigned long long bytes) {
  using namespace accudnn;
  if (g_ws.owned && g_ws.ws) cudaFree(g_ws.ws);
  g_ws.ws = static_cast<float*>(ptr);
  g_ws.bytes = ptr ? static_cast<size_t>(bytes) : 0;
  g_ws.owned = false;
  if (!ptr) g_ws_default = static_cast<size_t>(bytes);
  return 0;
}
