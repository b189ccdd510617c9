// TMA-fed implicit-GEMM convolution on tcgen05 (sm_100a), v2.
//
// Same three GEMMs as conv_igemm.cu (FWD / DGRAD / WGRAD on NHWC fp32 with
// TF32 tensor-core math), but every operand tile is moved by the Tensor
// Memory Accelerator instead of per-thread cp.async:
//
//   FWD   A  im2col TMA over x {C,W,H,N} (taps as im2col offsets; padding and
//            stride handled by the bounding box), or a 2-D tile for 1x1/s1
//         B  2-D tile over w viewed as [Cout][R*S*Cin]            (K-major)
//   DGRAD A  im2col TMA over dy {K,Q,P,N} with flipped taps (stride 1)
//         B  3-D tile over w {Cin, R*S, Cout} -> MN-major          (ci contiguous)
//   WGRAD A  2-D tiles over dy [pixels][Cout]                      (MN-major)
//         B  im2col TMA over x with 32 output pixels per column    (MN-major)
//
// K-major tiles use SWIZZLE_128B (UMMA layout type 2); MN-major TF32 tiles
// must use SWIZZLE_128B_BASE32B (UMMA layout type 1), produced by the TMA
// swizzle mode 128B_ATOM_32B; one TMA box fills one 32-element MN atom for
// 32 K-rows (4 KB), so MN atoms sit 4 KB apart (LBO) and 4-row groups 512 B
// apart (SBO).
//
// Warp roles (192 threads): warp 0 = TMA producer (one thread), warp 1 =
// TMEM allocator + MMA issuer (one thread), warps 2-5 = epilogue (TMEM ->
// registers -> global; split-K partials with fp32 vector atomics).  A deep
// stage ring (4-6 stages, <= 192 KB) hides L2/HBM latency; split-K fills the
// 148 SMs when the output tile grid is small.
#include <cuda.h>
#include <cuda_runtime.h>

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

enum Mode : int { FWD = 0, DGRAD = 1, WGRAD = 2 };

struct TArgs {
  int N, H, W, C, K, R, S, stride, pad, P, Q;
  int M, Ng, Kg;
  int kb_total, kb_per_split;
  int a_tiled;  // FWD/DGRAD: A is a plain 2-D tile (1x1, stride 1)
  float* out;
  int beta, atomic;
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

template <int MODE, int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                    const __grid_constant__ CUtensorMap tmB, const TArgs a) {
  constexpr bool kAmn = (MODE == WGRAD);
  constexpr bool kBmn = (MODE != FWD);
  constexpr uint32_t kABytes = kBM * kBK * 4;
  constexpr uint32_t kBBytes = BN * kBK * 4;
  constexpr uint32_t kStageBytes = kABytes + kBBytes;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* accum = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kBM;
  const int n0 = blockIdx.y * BN;
  const int kb_begin = blockIdx.z * a.kb_per_split;
  const int kb_end = min(a.kb_total, kb_begin + a.kb_per_split);
  const int nkb = kb_end - kb_begin;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accum, 1);
    ptx::fence_mbar_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 1) ptx::tmem_alloc<(BN < 32 ? 32 : BN)>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t smem_base = ptx::smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {
      // ============================ TMA producer ============================
      // first output pixel of this tile (FWD: (n,p,q); DGRAD: (n,h,w))
      int tn = 0, tp = 0, tq = 0;
      if constexpr (MODE != WGRAD) {
        const int hh = (MODE == FWD) ? a.P : a.H;
        const int ww = (MODE == FWD) ? a.Q : a.W;
        tn = m0 / (hh * ww);
        const int rem = m0 - tn * hh * ww;
        tp = rem / ww;
        tq = rem - tp * ww;
      }
      // WGRAD: fixed tap / channel block of this N-tile
      int wt_r = 0, wt_s = 0, wt_c = 0;
      if constexpr (MODE == WGRAD) {
        const int tap = n0 / a.C;
        wt_c = n0 - tap * a.C;
        wt_r = tap / a.S;
        wt_s = tap - wt_r * a.S;
      }
      for (int it = 0; it < nkb; ++it) {
        const int stage = it % STAGES;
        if (it >= STAGES) ptx::mbar_wait(&empty[stage], ((it / STAGES) - 1) & 1);
        const int kb = kb_begin + it;
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
            tma_im2col(&tmA, sA, bar, c0, tq * a.stride - a.pad, tp * a.stride - a.pad, tn,
                       static_cast<uint16_t>(s), static_cast<uint16_t>(r));
          }
          tma_2d(&tmB, sB, bar, kk, n0);
        } else if constexpr (MODE == DGRAD) {
          const int tap = kk / a.K, co0 = kk - tap * a.K;
          const int r = tap / a.S, s = tap - r * a.S;
          if (a.a_tiled) {
            tma_2d(&tmA, sA, bar, co0, m0);
          } else {
            tma_im2col(&tmA, sA, bar, co0, tq + a.pad - (a.S - 1), tp + a.pad - (a.R - 1), tn,
                       static_cast<uint16_t>(a.S - 1 - s), static_cast<uint16_t>(a.R - 1 - r));
          }
#pragma unroll
          for (int b = 0; b < BN / 32; ++b) tma_3d(&tmB, sB + b * 4096, bar, n0 + 32 * b, tap, co0);
        } else {
          // A: dy[pix][co] boxes {32 co, 32 pix}
#pragma unroll
          for (int b = 0; b < kBM / 32; ++b) tma_2d(&tmA, sA + b * 4096, bar, m0 + 32 * b, kk);
          // B: im2col of x for the 32 output pixels of this K-block
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
  } else if (warp == 1) {
    if (lane == 0) {
      // ============================ MMA issuer ============================
      constexpr uint32_t idesc = ptx::idesc_tf32(kBM, BN, kAmn, kBmn);
      for (int it = 0; it < nkb; ++it) {
        const int stage = it % STAGES;
        ptx::mbar_wait(&full[stage], (it / STAGES) & 1);
        ptx::tc_fence_after();
        const uint32_t sA = smem_base + stage * kStageBytes;
        const uint32_t sB = sA + kABytes;
#pragma unroll
        for (int ks = 0; ks < kBK / 8; ++ks) {
          const uint64_t ad = kAmn ? ptx::smem_desc(sA + ks * 1024, 4096, 512, 1)
                                   : ptx::smem_desc(sA + ks * 32, 16, 1024, 2);
          const uint64_t bd = kBmn ? ptx::smem_desc(sB + ks * 1024, 4096, 512, 1)
                                   : ptx::smem_desc(sB + ks * 32, 16, 1024, 2);
          ptx::mma_tf32(tmem, ad, bd, idesc, (it > 0 || ks > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&empty[stage]);
      }
      if (nkb > 0) ptx::mma_commit(accum);
    }
  } else if (nkb > 0) {
    // ============================ epilogue ============================
    ptx::mbar_wait(accum, 0);
    ptx::tc_fence_after();
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    const int m = m0 + row;
    const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      ptx::tmem_ld32(trow + c0, v);
      if (m < a.M) {
        float* dst = a.out + static_cast<long long>(m) * a.Ng + n0 + c0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          if (n0 + c0 + 4 * g >= a.Ng) break;
          float4 o = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
          float4* d4 = reinterpret_cast<float4*>(dst + 4 * g);
          if (a.atomic) {
            atomicAdd(d4, o);
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

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<(BN < 32 ? 32 : BN)>(tmem);
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

// NHWC tensor {C, W, H, N} with `lower`/`upper` corner offsets (both spatial
// dims equal), `pixels` rows per column, 32 channels per pixel
bool im2col_map(CUtensorMap* m, const void* base, int n, int h, int w, int c, int lower,
                int upper, int stride, int pixels, CUtensorMapSwizzle sw) {
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w),
                              static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 4,
                                 static_cast<cuuint64_t>(c) * w * 4,
                                 static_cast<cuuint64_t>(c) * w * h * 4};
  const int lo[2] = {lower, lower};
  const int hi[2] = {upper, upper};
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

template <int MODE, int BN, int STAGES>
int launch_t(const CUtensorMap& ta, const CUtensorMap& tb, TArgs a, int splits,
             cudaStream_t st) {
  constexpr size_t smem = STAGES * (kBM + BN) * kBK * 4 + 1024 + 256;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(conv_tma_kernel<MODE, BN, STAGES>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  dim3 grid((a.M + kBM - 1) / kBM, (a.Ng + BN - 1) / BN, splits);
  conv_tma_kernel<MODE, BN, STAGES><<<grid, kThreads, smem, st>>>(ta, tb, a);
  return static_cast<int>(cudaGetLastError());
}

// choose the split-K factor so the grid covers ~2 waves of SMs
int choose_splits(long long tiles, int kb_total) {
  const long long want = 2LL * sm_count();
  if (tiles >= sm_count()) return 1;
  long long s = (want + tiles - 1) / tiles;
  const long long max_s = kb_total / 4 > 0 ? kb_total / 4 : 1;  // >= 4 k-blocks each
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : static_cast<int>(s);
}

template <int MODE, int BN>
int run(const CUtensorMap& ta, const CUtensorMap& tb, TArgs a, float* out, cudaStream_t st) {
  const long long tiles =
      static_cast<long long>((a.M + kBM - 1) / kBM) * ((a.Ng + BN - 1) / BN);
  int splits = choose_splits(tiles, a.kb_total);
  a.kb_per_split = (a.kb_total + splits - 1) / splits;
  splits = (a.kb_total + a.kb_per_split - 1) / a.kb_per_split;
  a.atomic = splits > 1;
  if (a.atomic && !a.beta) {
    const cudaError_t e =
        cudaMemsetAsync(out, 0, sizeof(float) * static_cast<size_t>(a.M) * a.Ng, st);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  constexpr int kStages = BN >= 256 ? 4 : 6;
  return launch_t<MODE, BN, kStages>(ta, tb, a, splits, st);
}

TArgs base_args(const accudnn_conv_desc* d) {
  TArgs a{};
  a.N = d->n; a.H = d->h; a.W = d->w; a.C = d->c; a.K = d->k;
  a.R = d->r; a.S = d->s; a.stride = d->stride; a.pad = d->pad; a.P = d->p; a.Q = d->q;
  return a;
}

bool geometry_ok(const accudnn_conv_desc* d) {
  return d->r == d->s && d->pad <= 64 && d->r <= 16 && d->stride <= 8;
}

}  // namespace

// 0 = not eligible (caller falls back to the cp.async kernel), else launched
int conv_tma_fwd(const accudnn_conv_desc* d, const float* x, const float* w, float* y, int beta,
                 cudaStream_t st, int* rc) {
  if (!geometry_ok(d) || (d->c % 32) || (d->k % 4)) return 0;
  TArgs a = base_args(d);
  a.M = a.N * a.P * a.Q;
  a.Ng = a.K;
  a.Kg = a.R * a.S * a.C;
  a.kb_total = a.Kg / kBK;
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
    ok = im2col_map(&ta, x, a.N, a.H, a.W, a.C, -a.pad, a.pad - (a.R - 1), a.stride, kBM,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  }
  const cuuint64_t bd[2] = {static_cast<cuuint64_t>(a.Kg), static_cast<cuuint64_t>(a.K)};
  const cuuint64_t bs[1] = {static_cast<cuuint64_t>(a.Kg) * 4};
  const cuuint32_t bbox[2] = {32, static_cast<cuuint32_t>(BN)};
  ok = ok && tiled_map(&tb, w, 2, bd, bs, bbox, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!ok) return 0;
  *rc = BN == 256 ? run<FWD, 256>(ta, tb, a, y, st)
                  : (BN == 128 ? run<FWD, 128>(ta, tb, a, y, st) : run<FWD, 64>(ta, tb, a, y, st));
  return 1;
}

int conv_tma_dgrad(const accudnn_conv_desc* d, const float* dy, const float* w, float* dx,
                   int beta, cudaStream_t st, int* rc) {
  if (!geometry_ok(d) || d->stride != 1 || (d->c % 32) || (d->k % 32)) return 0;
  TArgs a = base_args(d);
  a.M = a.N * a.H * a.W;
  a.Ng = a.C;
  a.Kg = a.R * a.S * a.K;
  a.kb_total = a.Kg / kBK;
  a.out = dx;
  a.beta = beta;
  a.a_tiled = (a.R == 1 && a.pad == 0);
  const int BN = a.C >= 256 ? 256 : (a.C > 64 ? 128 : 64);
  if (a.C % BN && BN != 64) return 0;
  CUtensorMap ta, tb;
  bool ok;
  if (a.a_tiled) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.K), static_cast<cuuint64_t>(a.M)};
    const cuuint64_t str[1] = {static_cast<cuuint64_t>(a.K) * 4};
    const cuuint32_t box[2] = {32, kBM};
    ok = tiled_map(&ta, dy, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  } else {
    const int lower = a.pad - (a.R - 1);
    ok = im2col_map(&ta, dy, a.N, a.P, a.Q, a.K, lower, lower + a.H - a.P, 1, kBM,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  }
  const cuuint64_t bd[3] = {static_cast<cuuint64_t>(a.C), static_cast<cuuint64_t>(a.R) * a.S,
                            static_cast<cuuint64_t>(a.K)};
  const cuuint64_t bs[2] = {static_cast<cuuint64_t>(a.C) * 4,
                            static_cast<cuuint64_t>(a.C) * a.R * a.S * 4};
  const cuuint32_t bbox[3] = {32, 1, 32};
  ok = ok && tiled_map(&tb, w, 3, bd, bs, bbox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!ok) return 0;
  *rc = BN == 256 ? run<DGRAD, 256>(ta, tb, a, dx, st)
                  : (BN == 128 ? run<DGRAD, 128>(ta, tb, a, dx, st)
                               : run<DGRAD, 64>(ta, tb, a, dx, st));
  return 1;
}

int conv_tma_wgrad(const accudnn_conv_desc* d, const float* x, const float* dy, float* dw,
                   int beta, cudaStream_t st, int* rc) {
  if (!geometry_ok(d) || (d->c % 32) || (d->k % 4)) return 0;
  TArgs a = base_args(d);
  a.M = a.K;
  a.Ng = a.R * a.S * a.C;
  a.Kg = a.N * a.P * a.Q;
  // a ragged last K-block reads past the last output pixel: the im2col walk
  // and the dy tile land out of bounds there and are zero-filled by the TMA
  a.kb_total = (a.Kg + kBK - 1) / kBK;
  a.out = dw;
  a.beta = beta;
  const int BN = (a.C % 128 == 0) ? 128 : (a.C % 64 == 0 ? 64 : 0);
  if (!BN) return 0;
  CUtensorMap ta, tb;
  const cuuint64_t ad[2] = {static_cast<cuuint64_t>(a.K), static_cast<cuuint64_t>(a.Kg)};
  const cuuint64_t as[1] = {static_cast<cuuint64_t>(a.K) * 4};
  const cuuint32_t abox[2] = {32, 32};
  bool ok = tiled_map(&ta, dy, 2, ad, as, abox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  ok = ok && im2col_map(&tb, x, a.N, a.H, a.W, a.C, -a.pad, a.pad - (a.R - 1), a.stride, 32,
                        CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!ok) return 0;
  *rc = BN == 128 ? run<WGRAD, 128>(ta, tb, a, dw, st) : run<WGRAD, 64>(ta, tb, a, dw, st);
  return 1;
}

}  // namespace accudnn
